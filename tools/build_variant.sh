#!/bin/bash
# build an experimental library variant: tools/build_variant.sh NAME -DFOO=1 ...
# -> build/exp/libbnn_NAME.so (load with BNN_LIB_PATH=...)
set -e
name=$1; shift
cd "$(dirname "$0")/.."
python -m paper_1705_09864_b200.build >/dev/null
mkdir -p build/exp
objs=$(ls build/csrc/*.o | grep -v bnn_gemm_umma.o)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
  --expt-relaxed-constexpr -Iinclude "$@" -c paper_1705_09864_b200/csrc/bnn_gemm_umma.cu \
  -o build/exp/umma_$name.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o build/exp/libbnn_$name.so \
  $objs build/exp/umma_$name.o
echo build/exp/libbnn_$name.so
