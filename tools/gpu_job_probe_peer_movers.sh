mkdir -p gpurun_out
timeout 120 tools/cpp/sync_probe > gpurun_out/sync_probe.jsonl 2>&1; cat gpurun_out/sync_probe.jsonl
FUSP_TIMEOUT_S=20 timeout 900 python -m pytest tests/test_gpu_peer.py tests/test_gpu_nccl_shim.py -q -p no:cacheprovider > gpurun_out/peer_tests_3.log 2>&1; echo "peer rc=$?" >> gpurun_out/peer_tests_3.log
grep -E 'FAILED|passed|failed' gpurun_out/peer_tests_3.log
TAG=movers_r2b VARIANTS=base bash tools/gpu_job_movers_ncu.sh > /dev/null 2>&1
head -60 gpurun_out/movers_r2b_ncu.md
