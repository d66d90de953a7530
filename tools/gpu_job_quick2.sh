mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python tools/virtual_mesh_bench.py > gpurun_out/virtual_mesh.jsonl 2> gpurun_out/virtual_mesh.err
tail -5 gpurun_out/gpu_tests.log; cat gpurun_out/virtual_mesh.jsonl; tail -5 gpurun_out/virtual_mesh.err
