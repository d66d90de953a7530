# memcheck over the 4-process peer-memory IPC test (every worker process instrumented; any error fails the test)
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
FUSP_TIMEOUT_S=300 timeout 1500 $CS --tool memcheck --target-processes all --error-exitcode 9 --print-limit 20 python -m pytest "tests/test_gpu_peer.py::test_peer_windows_across_processes_ipc[4-2-1-False-1]" -q -p no:cacheprovider > gpurun_out/san_ipc.log 2>&1; echo "rc=$?" >> gpurun_out/san_ipc.log
grep -E "ERROR SUMMARY|passed|failed|rc=" gpurun_out/san_ipc.log | head -10
