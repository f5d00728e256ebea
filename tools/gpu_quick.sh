# quick check after a change: the GPU suite, smoke, the bench cases
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-q}
mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $D/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $D/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1
python bench.py --no-cpu > $D/bench.json 2> $D/bench.err
python bench.py --case h2o2 --no-cpu > $D/bench_h2o2.json 2>/dev/null
python bench.py --case ensemble --no-cpu > $D/bench_ens.json 2>/dev/null
python bench.py --case tgv --no-cpu > $D/bench_tgv2d.json 2>/dev/null
tail -2 $D/pytest_gpu.log
for f in bench bench_h2o2 bench_ens bench_tgv2d; do python -c "import json,sys; d=json.load(open('$D/$f.json')); print('$f', d['value'], d['ms_per_step'])"; done
