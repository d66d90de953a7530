mkdir -p gpurun_out
ATTN_SHAPES=qwen_u1,flux_u1 timeout 600 python tools/attn_shapes.py auto,split,whole,auto,split,whole > gpurun_out/attn_shapes2.jsonl 2>&1; cat gpurun_out/attn_shapes2.jsonl
