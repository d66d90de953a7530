# compute-sanitizer over every kernel family (tools/sanitize_cases.py). Outputs gpurun_out/san_*.log
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
python tools/sanitize_cases.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/san_plain.log
for tool in memcheck synccheck racecheck initcheck; do
  for c in attention staging fp8 ring usp; do
    timeout 900 $CS --tool $tool --target-processes all --print-limit 20 python tools/sanitize_cases.py $c > gpurun_out/san_${tool}_${c}.log 2>&1
    echo "rc=$?" >> gpurun_out/san_${tool}_${c}.log
  done
done
for f in gpurun_out/san_*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|rc=|ok$|Error|error" $f | head -6; done
