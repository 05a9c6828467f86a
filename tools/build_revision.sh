#!/bin/bash
# Build libbdeg.so of a git revision (optionally with -D defines) into scratch/, for tools/ab_bench.sh:
#   bash tools/build_revision.sh 80004c9                 -> scratch/libbdeg_80004c9.so
#   bash tools/build_revision.sh HEAD BDEG_MIN_BLOCKS=3  -> scratch/libbdeg_HEAD_BDEG_MIN_BLOCKS=3.so
set -e
REV=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
git -C "$ROOT" archive "$REV" paper_1501_02237_b200/csrc include | tar -x -C "$TMP"
NAME="$REV"; DEFS=""
for d in "$@"; do NAME="${NAME}_$d"; DEFS="$DEFS -D$d"; done
mkdir -p "$ROOT/scratch"
cd "$TMP/paper_1501_02237_b200/csrc"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
  -I "$TMP/include" $DEFS -o "$ROOT/scratch/libbdeg_${NAME}.so" *.cu *.cpp -lcudart
rm -rf "$TMP"
echo "$ROOT/scratch/libbdeg_${NAME}.so"
