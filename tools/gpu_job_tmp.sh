mkdir -p gpurun_out
export FUSP_PEER_DEBUG=1
FUSP_TIMEOUT_S=20 timeout 1500 python -m pytest tests/test_gpu_peer.py tests/test_gpu_nccl_shim.py -q -p no:cacheprovider > gpurun_out/pr.log 2>&1; echo "rc=$?" >> gpurun_out/pr.log; tail -4 gpurun_out/pr.log; grep "^FAILED\|Error" gpurun_out/pr.log | head; grep "\[peer\]" gpurun_out/pr.log | sort | head -30
