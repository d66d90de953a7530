mkdir -p gpurun_out
SHAPES=flux_u1,qwen_u1,flux_u2 timeout 900 python tools/ab_attn.py main p40 u4 e5 > gpurun_out/ab_var.jsonl 2>&1; cat gpurun_out/ab_var.jsonl | cut -c1-400
