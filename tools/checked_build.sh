#!/bin/sh
# Bounds-checked build of libkmb200.so (every kernel store / cp.async load asserted inside its
# tensor's logical extent, KMB_CHECK in kmb200_kernels.cuh) into build/tmp_check/; use it with
#   KMB200_LIB=$PWD/build/tmp_check/libkmb200.so python tools/sanitize_cases.py
set -e
cd "$(dirname "$0")/../paper_2103_01691_b200/csrc"
make -j8 BUILD=../../build/tmp_check/obj LIB=../../build/tmp_check/libkmb200.so EXTRA=-DKMB_CHECK
