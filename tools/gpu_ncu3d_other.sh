# ncu --set full (with source) of the 3D TGV 256^3 primitive, viscous and
# update kernels (one stage); report in gpurun_out/$1/
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-ncu3o}
mkdir -p $D
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_prim3|k_visc3|k_assemble3" -c 3 -o $D/tgv3d_other python tools/prof3d.py 256 > $D/ncu.log 2>&1
ls -la $D
