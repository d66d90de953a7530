mkdir -p gpurun_out
tools/cpp/movers_bench > gpurun_out/movers.jsonl 2>&1
timeout 1200 python -m pytest tests/test_gpu_wire.py tests/test_gpu_protocols.py tests/test_gpu_configs.py tests/test_gpu_numerics.py -q -p no:cacheprovider > gpurun_out/t.log 2>&1; echo "rc=$?" >> gpurun_out/t.log
tail -5 gpurun_out/t.log; grep -i "ring hop" gpurun_out/movers.jsonl
