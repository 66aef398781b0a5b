#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY. Builds the UNMODIFIED reference library straight
# from /root/reference/proj/src (nothing is copied into this repo) plus our
# extern "C" shim into oracle/_ref/libspgemm_ref.so. Flags follow the
# reference's Release build (proj/CMakeLists.txt:8-10) plus -march=native as
# the paper. The reference's own CMake build is not used.
# Output: oracle/_ref/ (git-ignored, travels to the GPU box with gpurun).
set -euo pipefail
REF=${REF:-/root/reference/proj}
HERE="$(cd "$(dirname "$0")" && pwd)"
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then
  echo "reference sources not present at $REF; keeping prebuilt $OUT" >&2
  exit 0
fi
mkdir -p "$OUT"
SRCS="$REF/src/baseline.cpp $REF/src/convert.cpp $REF/src/generate.cpp $REF/src/mmio.cpp $REF/src/pb_spgemm.cpp $REF/src/reference.cpp"
# -march=x86-64-v3: portable to the GPU box's host (AVX2), the container's
# native target may differ.
g++ -std=c++20 -O3 -march=x86-64-v3 -fopenmp -fPIC -shared -I "$REF/include" \
    $SRCS "$HERE/ref_shim.cpp" -o "$OUT/libspgemm_ref.so.tmp"
mv "$OUT/libspgemm_ref.so.tmp" "$OUT/libspgemm_ref.so"
echo "built $OUT/libspgemm_ref.so"
