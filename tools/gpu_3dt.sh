# 3D face-kernel timing check: bench + per-kernel durations of one stage (ncu)
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-t3}
mkdir -p $D
if [ "$2" = "test" ]; then timeout 900 python -m pytest tests/test_gpu_3d.py -x -q -p no:cacheprovider > $D/pytest_3d.log 2>&1; echo "pytest rc=$?" >> $D/pytest_3d.log; tail -2 $D/pytest_3d.log; fi
python bench.py --no-cpu --no-cases > $D/bench.json 2> $D/bench.err
python -c "import json; d=json.load(open('$D/bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'])"
timeout 300 ncu --metrics gpu__time_duration.sum,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,launch__shared_mem_per_block_dynamic,launch__shared_mem_per_block_static --clock-control none -k regex:k_faces3d -c 3 --csv python tools/prof3d.py 256 2>/dev/null | grep k_faces3d | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-200
