# ncu --set full (with source) of the face kernels: 3D TGV 256^3 (one stage)
# and H2/O2 512^2 (x and y); reports in gpurun_out/$1/
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-ncuf}
mkdir -p $D
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_faces3d -c 3 -o $D/faces3d python tools/prof3d.py 256 > $D/ncu3d.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_faces3 -c 2 -o $D/faces_h2o2 python tools/profh2o2.py 3 > $D/ncuh2.log 2>&1
ls -la $D
