# full measurement pass: bench (3D default, 2D analogue, h2o2, ensemble), reference arm,
# launch list of the default bench, ncu --set full of the 3D faces at 256^3
mkdir -p gpurun_out/round
cd $GRAFT_REPO_ROOT
python bench.py > gpurun_out/round/bench_tgv3d.json 2> gpurun_out/round/bench_tgv3d.err || exit 1
python bench.py --case tgv --no-cpu > gpurun_out/round/bench_tgv2d.json 2>/dev/null
python bench.py --case h2o2 > gpurun_out/round/bench_h2o2.json 2>/dev/null
python bench.py --case ensemble > gpurun_out/round/bench_ensemble.json 2>/dev/null
python bench.py --case jet3d --no-cpu > gpurun_out/round/bench_jet3d.json 2>/dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_prim3|k_visc3" -c 4 -o gpurun_out/round/jet_prim_visc -f python tools/profjet.py > /dev/null 2>&1
python bench.py --impl reference > gpurun_out/round/bench_reference.json 2>/dev/null
lscpu > gpurun_out/round/lscpu.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/round/launches_tgv3d.csv python bench.py --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_faces3d -c 3 -o gpurun_out/round/faces3d_256 -f python tools/prof3d.py > /dev/null 2>&1
echo done
