#!/bin/bash
# Experimental build of the product library with extra -D flags:
#   tools/build_variant.sh NAME -DFOO=1 ...  ->  exp/librigidq_NAME.so   (use with RQ_LIB_PATH)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
C=paper_1708_08427_b200/csrc
B=$C/build_exp_$name
mkdir -p $B exp
ARCH="-gencode arch=compute_100a,code=sm_100a"
COMMON="$ARCH -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Iinclude -I$C --expt-relaxed-constexpr"
for f in rq_setup rq_export rq_nodes; do [ -f $B/$f.o ] || cp $C/build/$f.o $B/ ; done
for f in rq_apply rq_mrhs rq_wave rq_host rq_z rq_api; do
  /usr/local/cuda/bin/nvcc $COMMON "$@" -c $C/$f.cu -o $B/$f.o &
done
wait
/usr/local/cuda/bin/nvcc $ARCH -shared -cudart static -o exp/librigidq_$name.so $B/*.o
echo built exp/librigidq_$name.so
