#!/bin/bash
# dev tool: recompile the named translation units of the library (e.g.
# kernels3d_ns1) and relink, leaving the other objects as they are — for
# experiments confined to one instantiation's kernels (a header change that
# touches the others still needs the full make)
set -e
cd "$(dirname "$0")/../paper_2202_02319_b200/csrc"
NVF="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC,-ffp-contract=off -I../../include -Xptxas -warn-spills"
for u in "$@"; do nvcc $NVF -c $u.cu -o ../_build/$u.o & done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../_lib/libignis_b200.so.tmp ../_build/*.o
mv ../_lib/libignis_b200.so.tmp ../_lib/libignis_b200.so
