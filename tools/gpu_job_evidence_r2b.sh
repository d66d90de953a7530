# Round-2 final evidence: GPU tests, smoke, bench (both arms), ncu launch list + --set full of the
# attention launch of the bench step, movers, compute-sanitizer on the FP8 families (the one-launch
# quantize's grid barrier). Outputs in gpurun_out/ (summarised into profiles/ by hand).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpuinfo.txt 2>&1
FUSP_TIMEOUT_S=60 timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_fwd -s 3 -c 1 -o gpurun_out/attn_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/ncu_full.log 2>&1
timeout 300 tools/cpp/movers_bench > gpurun_out/movers.jsonl 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck initcheck; do
  for c in fp8 ring usp; do
    timeout 900 $CS --tool $tool --target-processes all --print-limit 20 python tools/sanitize_cases.py $c > gpurun_out/san_${tool}_${c}.log 2>&1
    echo "rc=$?" >> gpurun_out/san_${tool}_${c}.log
  done
done
tail -3 gpurun_out/gpu_tests.log; tail -3 gpurun_out/smoke.log; cut -c1-400 gpurun_out/bench.json; cut -c1-300 gpurun_out/bench_ref.json; ls -la gpurun_out/*.ncu-rep
for f in gpurun_out/san_*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|rc=" $f | head -3; done
