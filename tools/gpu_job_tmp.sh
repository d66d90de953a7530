mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_peer.py -q -p no:cacheprovider -k "block" > gpurun_out/bg_tests.log 2>&1; echo "rc=$?" >> gpurun_out/bg_tests.log; tail -30 gpurun_out/bg_tests.log
