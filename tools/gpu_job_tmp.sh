mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --target-processes all --print-limit 20 python tools/sanitize_cases.py fp8pack > gpurun_out/san_${tool}_fp8pack.log 2>&1; echo "rc=$?" >> gpurun_out/san_${tool}_fp8pack.log
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|rc=|ok$" gpurun_out/san_${tool}_fp8pack.log | head -3
done
