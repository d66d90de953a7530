# Kernel bring-up: quick checks with short timeouts first, then tests and timing.
mkdir -p gpurun_out; Q=gpurun_out/bringup.log; : > $Q
timeout 240 python tools/attn_quick.py whole 1 256 1024 >> $Q 2>&1 || { echo "whole1 FAILED rc=$?" >> $Q; exit 0; }
timeout 60 python tools/attn_quick.py whole 3 1024 4608 >> $Q 2>&1 || { echo "whole2 FAILED" >> $Q; exit 0; }
timeout 60 python tools/attn_quick.py split 1 256 4608 >> $Q 2>&1 || { echo "split1 FAILED" >> $Q; exit 0; }
timeout 60 python tools/attn_quick.py split 3 1024 4608 >> $Q 2>&1 || { echo "split2 FAILED" >> $Q; exit 0; }
timeout 60 python tools/attn_quick.py whole 2 300 517 >> $Q 2>&1 || { echo "ragged FAILED" >> $Q; exit 0; }
SHAPES=flux_u1,flux_u2,flux_u4,flux_u8,ring_u2r4_step,qwen_u4r2_step,qwen_u1 timeout 200 python tools/ab_attn.py prev main >> $Q 2>&1
timeout 100 python tools/attn_trace.py 24 4608 whole 2>&1 | tail -2 >> $Q
timeout 300 python -m pytest -q -x tests/test_gpu_attention_schedule.py tests/test_gpu_kernels.py -p no:cacheprovider >> $Q 2>&1; echo "tests rc=$?" >> $Q
