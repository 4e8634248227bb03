#!/bin/bash
# Rebuild libghn.so per partition variant and time the cfg4 fit.
# VARIANTS: space-separated CHUNK_K:P1_STREAM:EXTRA_DEFINE tokens.
cd paper_2004_02290_b200/csrc
for v in ${VARIANTS:-16:0 64:1}; do
  IFS=: read ck st ex <<< "$v"
  rm -f ghn_fit.o
  make -s NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../../include -DPART_CHUNK_K=$ck -DPART_P1_STREAM=$st ${ex//,/ }" >/dev/null || exit 1
  (cd ../.. && python tools/fit_time.py "$v")
done
