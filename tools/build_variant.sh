#!/bin/bash
# Build an experimental variant of libbd_kvproj.so into xb/ (A/B on one box with
# BD_LIB_PATH=xb/<name>.so).   tools/build_variant.sh <name> [extra nvcc flags...]
set -e
mkdir -p "$(dirname "$0")/../xb"
name=$1; shift
cd "$(dirname "$0")/.."
C=paper_2510_01718_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  "$@" -o xb/$name.so $C/capi.cu $C/kv_proj_exact.cu $C/kv_proj_tc.cu $C/mla_attn.cu \
  $( [ -n "$WITH_DECODE" ] && echo "-DBD_WITH_DECODE_EXPERIMENT -I$C tools/experiments/kv_proj_decode_splitk.cu" )
echo xb/$name.so
