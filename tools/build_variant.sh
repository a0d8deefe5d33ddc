#!/bin/bash
# Build an experimental variant of libnosa_b200.so into tools/bin/libnosa_<name>.so (A/B runs
# select it with NOSA_B200_LIB=...).  Usage: tools/build_variant.sh NAME [GIT_REV_FOR_FILE FILE] [-- NVCC_FLAGS...]
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
TMP=$(mktemp -d /tmp/nosa_var_XXXX)
mkdir -p "$TMP/paper_2510_13602_b200" "$TMP/include" "$ROOT/tools/bin"
cp -r "$ROOT/paper_2510_13602_b200/csrc" "$TMP/paper_2510_13602_b200/"
cp "$ROOT/include/"*.h "$TMP/include/"
rm -rf "$TMP/paper_2510_13602_b200/csrc/build"
if [ $# -ge 2 ] && [ "$1" != "--" ]; then
  git -C "$ROOT" show "$1:paper_2510_13602_b200/csrc/$2" > "$TMP/paper_2510_13602_b200/csrc/$2"; shift 2
fi
[ "$1" == "--" ] && shift
make -s -j8 -C "$TMP/paper_2510_13602_b200/csrc" FLAGS="-O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-O3 -cudart static --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a $*" > /dev/null
cp "$TMP/paper_2510_13602_b200/libnosa_b200.so" "$ROOT/tools/bin/libnosa_$NAME.so"
rm -rf "$TMP"
echo "tools/bin/libnosa_$NAME.so"
