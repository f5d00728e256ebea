# 2D face-kernel timing check: H2/O2 512^2 and TGV 2D benches + per-kernel
# durations of the H2/O2 face kernels (ncu)
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-t2}
mkdir -p $D
if [ "$2" = "test" ]; then timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_species.py tests/test_gpu_baseline_sizes.py -x -q -p no:cacheprovider > $D/pytest_2d.log 2>&1; echo "pytest rc=$?" >> $D/pytest_2d.log; tail -2 $D/pytest_2d.log; fi
python bench.py --case h2o2 --no-cpu > $D/bench_h2o2.json 2>/dev/null
python bench.py --case tgv --no-cpu > $D/bench_tgv2d.json 2>/dev/null
for f in bench_h2o2 bench_tgv2d; do python -c "import json; d=json.load(open('$D/$f.json')); print('$f', d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'])"; done
timeout 300 ncu --metrics gpu__time_duration.sum,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,launch__shared_mem_per_block_dynamic --clock-control none -k regex:k_faces3 -c 2 --csv python tools/profh2o2.py 3 2>/dev/null | grep k_faces3 | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-200
