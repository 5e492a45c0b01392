#!/bin/bash
# Builds tools/librigidq_b200_timing.so: the product library with -DRQ_TIMING=1 (per-CTA
# clock64 phase timers, printed to stderr when RQ_TIMING is set). Use with RQ_LIB_PATH.
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
T=$(mktemp -d)
mkdir -p $T/include $T/p/csrc
cp $R/include/*.h $T/include/
cp $R/paper_1708_08427_b200/csrc/*.cu $R/paper_1708_08427_b200/csrc/*.cuh $R/paper_1708_08427_b200/csrc/*.hpp $R/paper_1708_08427_b200/csrc/Makefile $T/p/csrc/
make -s -j8 -C $T/p/csrc NVCC="/usr/local/cuda/bin/nvcc -DRQ_TIMING=${TIMING:-1} $EXTRA" OUT=$R/tools/librigidq_b200_timing${SUFFIX}.so >/dev/null 2>&1
rm -rf $T
echo built $R/tools/librigidq_b200_timing${SUFFIX}.so
