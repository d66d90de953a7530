mkdir -p gpurun_out
FUSP_TIMEOUT_S=30 timeout 900 python -m pytest tests/test_gpu_peer.py -q -p no:cacheprovider -k "check_finite or graph" > gpurun_out/cf.log 2>&1; echo "rc=$?" >> gpurun_out/cf.log; tail -15 gpurun_out/cf.log
