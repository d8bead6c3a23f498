#!/bin/bash
# Build paper_1408_0677_b200/libmdc_<name>.so with extra -D flags on layout.cu (A/B experiments only).
set -e
name=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
cd "$ROOT"
make -s -j16 >/dev/null
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -diag-suppress 550"
mkdir -p build/var
$NV "$@" -c paper_1408_0677_b200/csrc/layout.cu -o build/var/layout_$name.o
objs=$(ls build/*.o | grep -v layout.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1408_0677_b200/libmdc_$name.so $objs build/var/layout_$name.o
