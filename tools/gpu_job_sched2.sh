mkdir -p gpurun_out
SHAPES=flux_u4,flux_u8,ring_u2r4_step,qwen_u4r2_step timeout 300 python tools/ab_attn.py main:split main:aligned main:whole main > gpurun_out/ab_sched.jsonl 2>&1
cat gpurun_out/ab_sched.jsonl
