mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_wire.py tests/test_gpu_configs.py -q -p no:cacheprovider > gpurun_out/k.log 2>&1; echo "rc=$?" >> gpurun_out/k.log; tail -3 gpurun_out/k.log
timeout 300 tools/cpp/movers_bench > gpurun_out/movers.jsonl 2>&1; grep -A1 "fp8" gpurun_out/movers.jsonl | cut -c1-200
