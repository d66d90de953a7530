mkdir -p gpurun_out
export FUSP_PEER_DEBUG=1
for i in 1 2; do
FUSP_TIMEOUT_S=20 timeout 900 python -m pytest tests/test_gpu_peer.py tests/test_gpu_nccl_shim.py -q -p no:cacheprovider > gpurun_out/peer_tests_$i.log 2>&1; echo "peer rc=$?" >> gpurun_out/peer_tests_$i.log
tail -4 gpurun_out/peer_tests_$i.log; grep "\[peer\]" gpurun_out/peer_tests_$i.log | head -5
done
timeout 900 python -m pytest tests/test_gpu_wire.py tests/test_gpu_kernels.py tests/test_gpu_configs.py -q -p no:cacheprovider > gpurun_out/fp8_tests.log 2>&1; echo "rc=$?" >> gpurun_out/fp8_tests.log; tail -4 gpurun_out/fp8_tests.log
timeout 300 tools/cpp/movers_bench > gpurun_out/movers.jsonl 2>&1; cut -c1-200 gpurun_out/movers.jsonl
