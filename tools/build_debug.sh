#!/bin/bash
# Debug library (device-side PDQ_CHECK bounds/invariant asserts) at tools/libdebug.so:
#   tools/build_debug.sh && PDQ_LIB=tools/libdebug.so python tools/stress_sweep.py
cd "$(dirname "$0")/.." || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -Xcompiler -fPIC -shared -std=c++17 -Iinclude \
  -DPDQ_DEBUG -o tools/libdebug.so paper_2106_05123_b200/csrc/pdq_capi.cu
