# GPU tests of the peer-memory transport (short timeout: a protocol bug shows up as a bounded
# device spin, FUSP_TIMEOUT_S), then (FULL=1) the whole suite.
mkdir -p gpurun_out
for i in 1 2; do
FUSP_TIMEOUT_S=20 timeout 900 python -m pytest tests/test_gpu_peer.py tests/test_gpu_nccl_shim.py -q -p no:cacheprovider > gpurun_out/peer_tests_$i.log 2>&1; echo "peer rc=$?" >> gpurun_out/peer_tests_$i.log
tail -12 gpurun_out/peer_tests_$i.log
done
if [ -n "$FULL" ]; then
FUSP_TIMEOUT_S=60 timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -15 gpurun_out/gpu_tests.log
fi
