# round-2 measurement pass after the face-kernel restructure (run under
# gpurun): every bench case, the reference arm, the H2/O2 size scan against
# the ensemble, the launch list of the default bench.  Outputs in gpurun_out/r2b/.
mkdir -p gpurun_out/${R2B:-r2b}
cd $GRAFT_REPO_ROOT
D=gpurun_out/${R2B:-r2b}
python bench.py > $D/bench_tgv3d.json 2> $D/bench_tgv3d.err || exit 1
python bench.py --case tgv --no-cpu > $D/bench_tgv2d.json 2>/dev/null
python bench.py --case h2o2 > $D/bench_h2o2.json 2>/dev/null
python bench.py --case ensemble > $D/bench_ensemble.json 2>/dev/null
python bench.py --case ensemble --members 16 --no-cpu > $D/bench_ensemble16.json 2>/dev/null
python bench.py --case h2o2 --size 1024 --no-cpu > $D/bench_h2o2_1024.json 2>/dev/null
python bench.py --case h2o2 --size 2048 --no-cpu --steps 5 > $D/bench_h2o2_2048.json 2>/dev/null
python bench.py --case jet3d --no-cpu > $D/bench_jet3d.json 2>/dev/null
python bench.py --case jet3d --nz 256 --no-cpu --steps 5 --e2e-steps 1 > $D/bench_jet3d_full.json 2> $D/bench_jet3d_full.err
python bench.py --impl reference > $D/bench_reference.json 2>/dev/null
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > $D/smi.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $D/launches_tgv3d.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-cases --e2e-steps 1 > /dev/null 2>&1
echo done
