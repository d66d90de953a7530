mkdir -p gpurun_out
FUSP_TIMEOUT_S=60 timeout 900 python -m pytest tests/test_gpu_peer.py -q -p no:cacheprovider -k "block_graph" > gpurun_out/bg.log 2>&1; echo "rc=$?" >> gpurun_out/bg.log; tail -20 gpurun_out/bg.log
