#!/bin/bash
# Debug library (device-side PDQ_CHECK bounds/invariant asserts) at tools/libdebug.so:
#   tools/build_debug.sh && PDQ_LIB=tools/libdebug.so python tools/stress_sweep.py
cd "$(dirname "$0")/.." || exit 1
python -c "from paper_2106_05123_b200 import _lib; _lib.build(out='tools/libdebug.so', extra_flags=['-DPDQ_DEBUG'])"
