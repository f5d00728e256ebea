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
# Test programs that need the reference headers, built here so they travel to
# the GPU box (where /root/reference does not exist): the reference-typed
# drop-in checked against ignis::Simulation, and the POD facade example.
lib="$repo/paper_2202_02319_b200/_lib"
if [ -f "$lib/libignis_b200.so" ]; then
    g++ -std=c++20 -O2 -ffp-contract=off -DNDEBUG -pthread \
        -I"$ref_inc" -I"$repo/include" -DREPO_DATA_DIR="\"$repo/data\"" \
        "$repo/tests/cpp/drop_in_parity.cpp" -o "$out/drop_in_parity" \
        -L"$lib" -lignis_b200 -Wl,-rpath,'$ORIGIN/../../paper_2202_02319_b200/_lib'
    g++ -std=c++17 -O2 -I"$repo/include" "$repo/tests/cpp/facade_example.cpp" \
        -o "$out/facade_example" -L"$lib" -lignis_b200 \
        -Wl,-rpath,'$ORIGIN/../../paper_2202_02319_b200/_lib'
    echo "built $out/drop_in_parity $out/facade_example"
fi
