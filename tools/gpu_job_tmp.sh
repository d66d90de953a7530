mkdir -p gpurun_out
FUSP_TIMEOUT_S=30 timeout 900 python -m pytest tests/test_gpu_peer.py tests/test_gpu_prologue.py -q -p no:cacheprovider > gpurun_out/pro.log 2>&1; echo "rc=$?" >> gpurun_out/pro.log; tail -15 gpurun_out/pro.log
