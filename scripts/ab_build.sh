#!/bin/bash
# Build an experimental variant of libmp_b200.so with extra -D flags.
# Usage: bash scripts/ab_build.sh <name> [-DFOO=1 ...]   -> build_exp/libmp_<name>.so
set -e
NAME=$1; shift
mkdir -p build_exp
cd "$(dirname "$0")/.."
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -shared -Iinclude -Ipaper_2405_02086_b200/csrc "$@" \
  paper_2405_02086_b200/csrc/mp_device.cu paper_2405_02086_b200/csrc/mp_host.cu -o build_exp/libmp_$NAME.so
echo built build_exp/libmp_$NAME.so
