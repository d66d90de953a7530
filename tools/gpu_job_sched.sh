# Stream-K attention bring-up: quick checks (short timeouts), schedule tests, shape sweep.
mkdir -p gpurun_out
Q=gpurun_out/quick.log; : > $Q
timeout 240 python tools/attn_quick.py whole 1 256 1024 >> $Q 2>&1 || { echo "whole FAILED rc=$?" >> $Q; exit 0; }
timeout 60 python tools/attn_quick.py whole 3 1024 4608 >> $Q 2>&1 || { echo "whole2 FAILED" >> $Q; exit 0; }
timeout 60 python tools/attn_quick.py split 1 256 4608 >> $Q 2>&1 || { echo "split FAILED" >> $Q; exit 0; }
timeout 60 python tools/attn_quick.py split 3 1024 4608 >> $Q 2>&1 || { echo "split2 FAILED" >> $Q; exit 0; }
timeout 300 python -m pytest tests/test_gpu_attention_schedule.py -x -q -p no:cacheprovider > gpurun_out/sched_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sched_tests.log
timeout 300 python tools/attn_shapes.py > gpurun_out/attn_shapes.jsonl 2>&1
timeout 600 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
