# 3D face-kernel change check: the 3D GPU tests + the default bench
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-t3}
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_3d.py tests/test_gpu_slabs.py -x -q -p no:cacheprovider > $D/pytest_3d.log 2>&1; echo "pytest rc=$?" >> $D/pytest_3d.log
python bench.py --no-cpu --no-cases > $D/bench.json 2> $D/bench.err
tail -2 $D/pytest_3d.log
python -c "import json; d=json.load(open('$D/bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'])"
