# ncu --set full (with source) of the H2/O2 512^2 ghost-fill, primitive,
# viscous and update kernels (one stage); report in gpurun_out/$1/
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-ncuo}
mkdir -p $D
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bc|k_prim|k_visc|k_assemble" -c 5 -o $D/h2o2_other python tools/profh2o2.py 3 > $D/ncu.log 2>&1
ls -la $D
