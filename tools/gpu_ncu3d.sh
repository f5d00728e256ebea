# ncu --set full (with source) of the three 3D face kernels of one stage at 256^3
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-ncu3d}
mkdir -p $D
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_faces3d -c 3 -o $D/faces3d python tools/prof3d.py 256 > $D/ncu.log 2>&1
ls -la $D
