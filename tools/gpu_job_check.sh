# Full check: GPU tests, smoke, bench, virtual-mesh measurements. Outputs in gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpuinfo.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python tools/virtual_mesh_bench.py > gpurun_out/vmesh.jsonl 2> gpurun_out/vmesh.err
tail -3 gpurun_out/gpu_tests.log; tail -4 gpurun_out/smoke.log; cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err; cut -c1-250 gpurun_out/vmesh.jsonl
