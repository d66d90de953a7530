# A/B the attention variants built by tools/build_variants.sh (outputs gpurun_out/var_*.jsonl)
mkdir -p gpurun_out
for v in "$@"; do
  modes=whole,split,auto; [ "$v" = old ] && modes=whole
  FUSP_VARIANT=$v timeout 120 python tools/attn_quick.py split 3 1024 4608 > gpurun_out/var_$v.jsonl 2>&1 || { echo "variant $v quick FAILED" >> gpurun_out/var_$v.jsonl; continue; }
  FUSP_VARIANT=$v timeout 300 python tools/attn_shapes.py $modes >> gpurun_out/var_$v.jsonl 2>&1
done
