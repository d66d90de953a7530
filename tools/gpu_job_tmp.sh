mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_peer.py -q -p no:cacheprovider -k "dtypes" > gpurun_out/pd_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pd_tests.log; tail -5 gpurun_out/pd_tests.log
