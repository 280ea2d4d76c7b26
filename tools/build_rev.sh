#!/bin/bash
# Builds libebem_gpu.so of a git revision into abx/<name>.so (bitwise / timing
# A/B against the working tree).  Usage: tools/build_rev.sh <rev> <name>
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
rev=$1; name=$2
B=/tmp/ebem_rev_$name
rm -rf "$B" && mkdir -p "$B" "$ROOT/abx"
git -C "$ROOT" archive "$rev" paper_2411_18026_b200/csrc include | tar -x -C "$B"
sed -i "s|OUT    := ../libebem_gpu.so|OUT    := $ROOT/abx/$name.so|" "$B/paper_2411_18026_b200/csrc/Makefile"
make -C "$B/paper_2411_18026_b200/csrc" -j8 > "$B/build.log" 2>&1 || { tail -20 "$B/build.log"; exit 1; }
echo "built abx/$name.so from $rev"
