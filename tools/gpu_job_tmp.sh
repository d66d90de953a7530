mkdir -p gpurun_out
timeout 300 tools/cpp/movers_bench > gpurun_out/movers.jsonl 2>&1; grep -A1 "Ulysses pack" gpurun_out/movers.jsonl | cut -c1-220
