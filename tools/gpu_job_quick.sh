# quick iteration: attention/kernel GPU tests + default bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -p no:cacheprovider -x > gpurun_out/gpu_tests_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests_quick.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
tail -3 gpurun_out/gpu_tests_quick.log; cat gpurun_out/bench_quick.json; tail -3 gpurun_out/bench_quick.err
