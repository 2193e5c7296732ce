#!/bin/bash
# A/B builds: tools/build_variant.sh NAME "-DFLAG=V ..." -> paper_2408_09697_b200/libhetgpu_NAME.so
# (select with HETGPU_LIB=...; delete the variants after measuring)
set -e
NAME=$1; FLAGS=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
make -C "$ROOT/paper_2408_09697_b200/csrc" -j8 OBJDIR="$ROOT/build/var_$NAME" OUTLIB="$ROOT/paper_2408_09697_b200/libhetgpu_$NAME.so" EXTRA="$FLAGS" >/dev/null
echo "$ROOT/paper_2408_09697_b200/libhetgpu_$NAME.so"
