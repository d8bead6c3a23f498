#!/bin/bash
# Build paper_1408_0677_b200/libmdc_<name>.so with extra -D flags on one kernel
# source (default mls_tc2.cu; SRC=mls_tc.cu for the two-pass kernel).  A/B experiments only.
# usage: [SRC=mls_tc2.cu] tools/build_variant.sh <name> -DMDC_TC2_FLUSH=8 ...
set -e
name=$1; shift
SRC=${SRC:-mls_tc2.cu}
base=${SRC%.cu}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
cd "$ROOT"
make -s -j16 >/dev/null
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -diag-suppress 550"
mkdir -p build/var
$NV "$@" -c paper_1408_0677_b200/csrc/$SRC -o build/var/${base}_$name.o
objs=$(ls build/*.o | grep -v "/$base.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1408_0677_b200/libmdc_$name.so $objs build/var/${base}_$name.o
