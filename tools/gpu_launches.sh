# ncu launch lists (per-kernel durations, cold and serialised) of the H2/O2
# 512^2 bench and the ensemble bench; outputs in gpurun_out/launch/
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/launch
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launch/h2o2.csv python bench.py --case h2o2 --steps 2 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/launch/h2o2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launch/ens.csv python bench.py --case ensemble --steps 1 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/launch/ens.log 2>&1
echo done
