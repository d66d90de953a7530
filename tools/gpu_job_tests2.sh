mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_wire.py tests/test_gpu_configs.py -q -p no:cacheprovider -x > gpurun_out/new_tests.log 2>&1; echo "rc=$?" >> gpurun_out/new_tests.log
tail -30 gpurun_out/new_tests.log
