#!/usr/bin/env bash
# Builds the CPU oracle of record: the UNMODIFIED reference headers under
# /root/reference/proj/include compiled in place (never copied) together with
# the C-ABI shim oracle/ref_driver.cpp, into oracle/_ref/libignis_ref.so.
#
# Flags follow SURVEY.md §8(c): the reference's own -O2 (tests/CMakeLists.txt:7),
# -std=c++20, -pthread, and -ffp-contract=off so no FMA contraction can move
# results (no -march=native).  Output goes only to oracle/_ref/ (git-ignored,
# shipped to the GPU box with the gpurun snapshot).
set -euo pipefail
here="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
repo="$(dirname "$here")"
ref_inc="${IGNIS_REF_INCLUDE:-/root/reference/proj/include}"
out="$here/_ref"
if [ ! -f "$ref_inc/ignis/solver.hpp" ]; then
    if [ -f "$out/libignis_ref.so" ]; then
        echo "reference sources absent; keeping prebuilt $out/libignis_ref.so"
        exit 0
    fi
    echo "reference sources not found at $ref_inc" >&2
    exit 1
fi
mkdir -p "$out"
g++ -std=c++20 -O2 -ffp-contract=off -DNDEBUG -pthread -fPIC -shared \
    -I"$ref_inc" -I"$repo/include" \
    "$here/ref_driver.cpp" -o "$out/libignis_ref.so.tmp"
mv "$out/libignis_ref.so.tmp" "$out/libignis_ref.so"
echo "built $out/libignis_ref.so"
