mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_protocols.py -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests_attn.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests_attn.log
for m in auto 1; do FUSP_ATTN_SPLIT=$m timeout 300 python tools/attn_shapes.py; done > gpurun_out/attn_shapes.jsonl 2> gpurun_out/attn_shapes.err
grep -E "passed|failed|FAILED" gpurun_out/gpu_tests_attn.log | tail -12; cat gpurun_out/attn_shapes.jsonl; tail -3 gpurun_out/attn_shapes.err
