mkdir -p gpurun_out
FUSP_TIMEOUT_S=30 timeout 1500 python -m pytest tests/test_gpu_peer.py tests/test_gpu_nccl_shim.py -q -p no:cacheprovider > gpurun_out/pr.log 2>&1; echo "rc=$?" >> gpurun_out/pr.log; tail -4 gpurun_out/pr.log; grep "^FAILED" gpurun_out/pr.log | head
