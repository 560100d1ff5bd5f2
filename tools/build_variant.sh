#!/bin/bash
# Build a variant of the library for A/B timing on the GPU box (dev helper).
#   tools/build_variant.sh NAME [SRC_DIR] -- EXTRA_NVCC_FLAGS...
# Output: vlib/NAME/libpagani_b200.so (git-ignored; travels with gpurun).
# Time it with: PAGANI_LIB=vlib/NAME/libpagani_b200.so python tools/variant_eval.py
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
SRC=$ROOT/paper_2104_06494_b200/csrc
if [ "$1" != "--" ]; then SRC=$1; shift; fi
shift  # --
OBJ=/tmp/vobj_$NAME
mkdir -p "$OBJ" "$ROOT/vlib/$NAME"
rm -f "$OBJ"/eval_*.o
make -s -C "$SRC" -j"$(nproc)" OBJDIR="$OBJ" OUT="$ROOT/vlib/$NAME/libpagani_b200.so" \
  HDRS= EXTRA="$*"
echo "built vlib/$NAME/libpagani_b200.so"
