timeout 300 python tools/kv2_check.py > gpurun_out/kv2_check.jsonl 2>&1
SHAPES=flux_u8 timeout 300 python tools/ab_attn.py main:split latek:kv2 main:kv2 k3v3e:kv2 latek:kv2 main:kv2 > gpurun_out/ab_kv2e.jsonl 2>&1
grep kv2 gpurun_out/kv2_check.jsonl | cut -c1-150; cat gpurun_out/ab_kv2e.jsonl
