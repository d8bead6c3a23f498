#!/bin/bash
for L in "$@"; do
  echo "== $L"; MDC_LIB_PATH=$PWD/paper_1408_0677_b200/$L NO_SIMT=1 python tools/dbg/acc_full.py 2>&1 | grep "max normwise"
done
