#!/bin/bash
# Build an alternative libaidw_b200.so with extra nvcc defines for kernel
# tuning:  tools/build_variant.sh <name> -DAIDW_K4_STAGES=8 ...
# -> build/variants/<name>/libaidw_b200.so (select with AIDW_LIB_PATH).
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/build/variants/$NAME
mkdir -p $OUT/obj
make -C $ROOT/paper_1601_05904_b200/csrc OBJDIR=$OUT/obj OUTDIR=$OUT NVCC="nvcc $*" -j8 >/dev/null
echo $OUT/libaidw_b200.so
