#!/bin/bash
# Build a variant of libfde_b200.so with extra nvcc flags: tools/build_variant.sh NAME "-DX=1 ..."
set -e
NAME=$1; shift
D=$(cd "$(dirname "$0")/.." && pwd)/build/var_$NAME
mkdir -p $D
make -s -j8 -C "$(dirname "$0")/../paper_1706_06844_b200/csrc" OBJDIR=$D/obj LIB=$D/libfde_b200.so EXTRA="$*" 2>&1 | grep -E "error" || true
ls $D/libfde_b200.so
