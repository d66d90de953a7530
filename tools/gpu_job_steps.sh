for v in main e2 e3 e8 e64; do
  echo "== $v"
  if [ $v = main ]; then unset FUSP_VARIANT; else export FUSP_VARIANT=$v; fi
  timeout 100 python tools/attn_trace_steps.py
done
