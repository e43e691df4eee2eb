#!/bin/bash
# Build A/B variants of the engine library with extra nvcc defines, in-tree
# (paper_2405_20693_b200/variants/<name>.so; git-ignored, travels to the GPU box):
#   tools/variants.sh build NAME "-DSCT_K4_ACC2=1 ..."
#   tools/variants.sh run  NAME...   (quick cfg3 bench per variant, SCT_LIB_VARIANT)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
if [ "$1" = build ]; then
  name=$2; shift 2
  out=$ROOT/paper_2405_20693_b200/variants/$name.so
  mkdir -p $(dirname $out)
  make -s -C $ROOT/paper_2405_20693_b200/csrc -j8 OUT=$out BUILD=$ROOT/build/variants/$name EXTRA="$*" >/dev/null
  echo built $out
elif [ "$1" = run ]; then
  shift
  for name in "$@"; do
    lib=libsplatct_b200.so
    [ "$name" != base ] && lib=variants/$name.so
    echo -n "$name: "
    SCT_LIB_VARIANT=$lib bash $ROOT/tools/quick_bench.sh
  done
fi
