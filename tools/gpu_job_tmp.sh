mkdir -p gpurun_out
timeout 600 python tools/block_bench.py > gpurun_out/block.jsonl 2>&1; cat gpurun_out/block.jsonl
