#!/bin/bash
# Builds an A/B or probe variant of the library with extra nvcc defines into
# build_variants/<name>/liblevelrank_b200.so (load it with LR_LIB=...).
#   tools/build_variant.sh probe -DLR_LCTA_PROBE
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
dst=$root/build_variants/$name
rm -rf "$dst" && mkdir -p "$dst"
cp -r "$root/paper_1609_09068_b200/csrc" "$root/paper_1609_09068_b200/Makefile" "$dst/"
[ -e "$root/build_variants/include" ] || ln -s "$root/include" "$root/build_variants/include"
make -C "$dst" -j8 NVFLAGS="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false -Xcompiler -fPIC $*" >/dev/null
echo "$dst/liblevelrank_b200.so"
