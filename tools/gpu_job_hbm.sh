# DRAM bandwidth of the data-movement kernels on the FLUX U=8 layer (virtual mesh on one GPU):
# bf16, fp8 per-tensor, fp8 per-block, and the fused QK RMSNorm+RoPE prologue.
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum; CC=${CC:-all}
for cfg in "8 1 4608 bf16" "8 1 4608 fp8" "8 1 4608 fp8block" "8 1 4608 bf16 prologue" "2 1 4608 bf16" "8 4 16896 fp8"; do
  tag=$(echo $cfg | tr ' ' '_')
  timeout 900 ncu --metrics $M --clock-control none --cache-control $CC --csv --log-file gpurun_out/hbm_$tag.csv python tools/mesh_layer_once.py $cfg > gpurun_out/hbm_$tag.log 2>&1
done
ls -la gpurun_out/hbm_*.csv
