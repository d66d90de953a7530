for v in main fake; do
  echo "== $v"
  if [ $v = main ]; then unset FUSP_VARIANT; else export FUSP_VARIANT=$v; fi
  timeout 100 python tools/attn_trace.py 24 4608 whole 2>&1 | tail -2
done
unset FUSP_VARIANT
SHAPES=flux_u1 timeout 300 python tools/ab_attn.py main fake
