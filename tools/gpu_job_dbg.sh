mkdir -p gpurun_out; L=gpurun_out/dbg.log; : > $L
for args in "split 3 1024 4608" "split 1 256 4608" "split 12 4608 4608" "whole 12 4608 4608" "split 6 4608 4608" "split 3 4608 4608"; do
  echo "== $args" >> $L
  timeout 60 python tools/attn_quick.py $args >> $L 2>&1; echo "rc=$?" >> $L
done
timeout 200 python -m pytest -q -x tests/test_gpu_attention_schedule.py >> $L 2>&1; echo "pytest rc=$?" >> $L
SHAPES=flux_u1,flux_u2,flux_u4,flux_u8,ring_u2r4_step,qwen_u4r2_step,qwen_u1 timeout 300 python tools/ab_attn.py old prev main neww:whole >> $L 2>&1
timeout 100 python tools/attn_trace.py 3 4608 auto >> $L 2>&1
