mkdir -p gpurun_out
timeout 300 tools/cpp/proj_bench > gpurun_out/proj.jsonl 2>&1; cat gpurun_out/proj.jsonl
TAG=movers_r2c bash tools/gpu_job_movers_ncu.sh > /dev/null 2>&1
head -80 gpurun_out/movers_r2c_ncu.md | cut -c1-250
cat gpurun_out/movers_r2c_layer_u8.md gpurun_out/movers_r2c_layer_u2r4.md | cut -c1-200
