mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  timeout 900 $CS --tool $tool --print-limit 5 python tools/sanitize_cases.py attention > gpurun_out/san_${tool}_attention.log 2>&1; echo "rc=$?" >> gpurun_out/san_${tool}_attention.log
done
tail -3 gpurun_out/gpu_tests.log; for f in gpurun_out/san_*_attention.log; do echo "== $f"; grep -E "SUMMARY|rc=|ok$" $f; done
