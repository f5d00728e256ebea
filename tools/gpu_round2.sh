# round-2 measurement pass (run under gpurun): every bench case, the reference
# arm, the launch list of the default bench.  Outputs in gpurun_out/r2/.
mkdir -p gpurun_out/r2
cd $GRAFT_REPO_ROOT
python bench.py > gpurun_out/r2/bench_tgv3d.json 2> gpurun_out/r2/bench_tgv3d.err || exit 1
python bench.py --case tgv --no-cpu > gpurun_out/r2/bench_tgv2d.json 2>/dev/null
python bench.py --case h2o2 > gpurun_out/r2/bench_h2o2.json 2>/dev/null
python bench.py --case ensemble > gpurun_out/r2/bench_ensemble.json 2>/dev/null
python bench.py --case jet3d --no-cpu > gpurun_out/r2/bench_jet3d.json 2>/dev/null
python bench.py --case jet3d --nz 256 --no-cpu --steps 5 --e2e-steps 1 > gpurun_out/r2/bench_jet3d_full.json 2> gpurun_out/r2/bench_jet3d_full.err
python bench.py --impl reference > gpurun_out/r2/bench_reference.json 2>/dev/null
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > gpurun_out/r2/smi.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2/launches_tgv3d.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-cases --e2e-steps 1 > /dev/null 2>&1
echo done
