#!/bin/bash
# Build A/B variants of the library that differ only in knn_tc.cu compile
# definitions: tools/build_variants.sh NAME "-DFOO=1 -DBAR=2" [NAME2 "..."]...
# -> paper_2206_14148_b200/libtb_pairwise_NAME.so (never loaded by the package).
set -e
cd "$(dirname "$0")/../paper_2206_14148_b200/csrc"
ARCH="-gencode arch=compute_100a,code=sm_100a"
FLAGS="$ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr"
OTHERS="build/capi.o build/knn_kernels.o build/sgpr.o build/sgpr_i8.o build/sgpr_grad.o build/sgpr_tail.o"
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  nvcc $FLAGS $defs -c knn_tc.cu -o build/knn_tc_$name.o &
done
wait
for o in build/knn_tc_*.o; do
  n=${o#build/knn_tc_}; n=${n%.o}
  [ "$n" = trace ] && continue
  nvcc $ARCH -shared -o ../libtb_pairwise_$n.so $OTHERS $o -lcudart_static -ldl -lpthread -lrt
done
