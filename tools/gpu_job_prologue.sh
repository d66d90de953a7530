# prologue + CLI GPU tests
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prologue.py tests/test_gpu_cli.py -q -m gpu -p no:cacheprovider > gpurun_out/gpu_prologue.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_prologue.log
tail -30 gpurun_out/gpu_prologue.log
