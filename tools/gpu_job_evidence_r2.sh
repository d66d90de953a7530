# Round-2 evidence: GPU tests, smoke, bench (both arms), ncu launch list, ncu --set full of the
# attention kernel (bench workload + FLUX U=8 split) and of the staging kernel, movers, A/B vs r01,
# virtual-mesh measurements. Outputs in gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpuinfo.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_fwd -s 3 -c 1 -o gpurun_out/attn_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_fwd -s 3 -c 1 -o gpurun_out/attn_u8_split -f python tools/attn_once.py 3 4608 auto > gpurun_out/ncu_u8.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:stage_kernel -s 2 -c 1 -o gpurun_out/stage_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/ncu_stage.log 2>&1
timeout 300 tools/cpp/movers_bench > gpurun_out/movers.jsonl 2>&1
timeout 300 python tools/ab_attn.py r01 main > gpurun_out/ab_attn.jsonl 2>&1
timeout 900 python tools/virtual_mesh_bench.py > gpurun_out/vmesh.jsonl 2> gpurun_out/vmesh.err
tail -3 gpurun_out/gpu_tests.log; tail -3 gpurun_out/smoke.log; cut -c1-400 gpurun_out/bench.json; cut -c1-300 gpurun_out/bench_ref.json; ls -la gpurun_out/*.ncu-rep
