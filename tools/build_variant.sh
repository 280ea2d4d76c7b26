#!/bin/bash
# Builds an alternative libebem_gpu.so with extra nvcc defines into abx/<name>.so
# (A/B timing: EBEM_GPU_LIB=abx/<name>.so python ...).  Usage:
#   tools/build_variant.sh <name> "-DEBEM_PTS_MINB=1 ..."
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; shift
B=/tmp/ebem_variant_$name
rm -rf "$B" && mkdir -p "$B" "$ROOT/abx"
cp "$ROOT"/paper_2411_18026_b200/csrc/*.{cu,cpp,h,cuh} "$ROOT"/paper_2411_18026_b200/csrc/Makefile "$B"/
sed -i "s|-I../../include|-I$ROOT/include|g; s|OUT    := ../libebem_gpu.so|OUT    := $ROOT/abx/$name.so|; s|../../include/ebem_gpu.h|$ROOT/include/ebem_gpu.h|" "$B/Makefile"
make -C "$B" -j8 EXTRA="$*" > "$B/build.log" 2>&1 || { tail -20 "$B/build.log"; exit 1; }
echo "built abx/$name.so"
