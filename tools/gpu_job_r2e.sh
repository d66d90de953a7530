mkdir -p gpurun_out
timeout 300 python tools/ab_attn.py r01 main > gpurun_out/ab_attn.jsonl 2>&1
VDT=bf16 SHAPES=flux_u1,flux_u8 timeout 300 python tools/ab_attn.py r01 main > gpurun_out/ab_attn_vbf16.jsonl 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/ab_attn.jsonl gpurun_out/ab_attn_vbf16.jsonl; python -c "
import json;d=json.load(open('gpurun_out/bench.json'));r=d['roofline'];print(d['value'],d['ms_per_step'],r['avg_launch_us'],r['standalone_us'],d['e2e']['value'])"
