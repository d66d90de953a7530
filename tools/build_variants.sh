#!/bin/bash
# Builds attention-kernel variants (compile-time knobs) into paper_2602_10940_b200/variants/<name>/
# for A/B timing on the GPU: FUSP_VARIANT=<name> python tools/attn_shapes.py
set -e
cd "$(dirname "$0")/../paper_2602_10940_b200"
make -j8 >/dev/null
OBJS=$(ls lib/*.o | grep -v attention_sm100)
build() {
  name=$1; shift
  mkdir -p variants/$name
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
    -Xptxas -v --expt-relaxed-constexpr "$@" -c csrc/attention_sm100.cu -o variants/$name/attention_sm100.cu.o 2> variants/$name/ptxas.log
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/$name/libfastusp.so \
    variants/$name/attention_sm100.cu.o $OBJS -lnccl -lcudart -Xlinker --no-undefined
  echo "$name: $(grep -A1 'Function properties for.*attn_fwd' variants/$name/ptxas.log | tail -1)"
}
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  build $name $flags
done
