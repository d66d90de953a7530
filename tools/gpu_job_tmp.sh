mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_out_proj.py tests/test_gpu_prologue.py tests/test_gpu_peer.py -q -p no:cacheprovider > gpurun_out/proj_tests.log 2>&1; echo "rc=$?" >> gpurun_out/proj_tests.log; tail -5 gpurun_out/proj_tests.log
