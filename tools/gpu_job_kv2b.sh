mkdir -p gpurun_out
SHAPES=flux_u8 timeout 300 python tools/ab_attn.py main:split k4v2:kv2 k3v3:kv2 main:kv2 k3v3:kv2 k4v2:kv2 > gpurun_out/ab_kv2b.jsonl 2>&1
cat gpurun_out/ab_kv2b.jsonl
