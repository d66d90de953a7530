# scratch GPU job: kv2 stream-K trace
mkdir -p gpurun_out
bash tools/build_variants.sh trace:-DFUSP_TRACE_BUILD=1 > gpurun_out/tmp_build.log 2>&1
for cfg in "kv2split 0" "kv2split 120" "kv2split 108" "kv2 0"; do
  echo "== $cfg"; FUSP_VARIANT=trace timeout 120 python tools/attn_trace_kv2.py 3 4608 $cfg
done > gpurun_out/tmp_trace.log 2>&1
cat gpurun_out/tmp_trace.log
