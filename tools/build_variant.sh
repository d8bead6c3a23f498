#!/bin/bash
# Build paper_1408_0677_b200/libmdc_<name>.so with extra -D flags on mls_tc.cu (A/B experiments only).
# usage: tools/build_variant.sh <name> -DMDC_TC_KT=8 ...
set -e
name=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
cd "$ROOT"
make -s -j16 >/dev/null
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -diag-suppress 550"
mkdir -p build/var
$NV "$@" -c paper_1408_0677_b200/csrc/mls_tc.cu -o build/var/mls_tc_$name.o
objs=$(ls build/*.o | grep -v mls_tc.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1408_0677_b200/libmdc_$name.so $objs build/var/mls_tc_$name.o
cuobjdump -res-usage build/var/mls_tc_$name.o | grep -A1 "mls_tc_kernelILi2ELi32" | tail -1
