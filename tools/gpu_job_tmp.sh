mkdir -p gpurun_out
FUSP_TIMEOUT_S=60 timeout 1500 python -m pytest tests/test_gpu_peer.py -q -p no:cacheprovider -k "ipc" > gpurun_out/ipc.log 2>&1; echo "rc=$?" >> gpurun_out/ipc.log; tail -15 gpurun_out/ipc.log
