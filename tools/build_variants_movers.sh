#!/bin/bash
# Builds kernels.cu variants (compile-time knobs) into paper_2602_10940_b200/variants/<name>/
# for A/B timing of the data movers on the GPU (tools/stage_bench.py).
set -e
cd "$(dirname "$0")/../paper_2602_10940_b200"
make -j8 >/dev/null
OBJS=$(ls lib/*.o | grep -v kernels.cu.o)
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  mkdir -p variants/$name
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
    -Xptxas -v --expt-relaxed-constexpr $flags -c csrc/kernels.cu -o variants/$name/kernels.cu.o 2> variants/$name/ptxas.log
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/$name/libfastusp.so \
    variants/$name/kernels.cu.o $OBJS -lnccl -lcudart -Xlinker --no-undefined
  echo "$name: $(grep -A2 'stage_kernel' variants/$name/ptxas.log | grep -E 'registers|spill' | tr '\n' ' ')"
done
