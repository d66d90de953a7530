mkdir -p gpurun_out
timeout 300 python tools/kv2_check.py > gpurun_out/kv2_check.jsonl 2>&1; echo "rc=$?" >> gpurun_out/kv2_check.jsonl
SHAPES=flux_u2,flux_u4,flux_u8,ring_u2r4_step,qwen_u4r2_step timeout 300 python tools/ab_attn.py main:split main:kv2 main > gpurun_out/ab_kv2.jsonl 2>&1
cat gpurun_out/kv2_check.jsonl gpurun_out/ab_kv2.jsonl
