mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for c in attention ring usp; do
  timeout 900 $CS --tool synccheck --print-limit 5 python tools/sanitize_cases.py $c > gpurun_out/san_synccheck_${c}.log 2>&1; echo "rc=$?" >> gpurun_out/san_synccheck_${c}.log
done
timeout 300 python tools/ab_attn.py r01 main > gpurun_out/ab_attn.jsonl 2>&1
for f in gpurun_out/san_synccheck_*.log; do echo "== $f"; grep -E "ERROR SUMMARY|rc=|ok$" $f | head -4; head -5 $f; done; cat gpurun_out/ab_attn.jsonl
