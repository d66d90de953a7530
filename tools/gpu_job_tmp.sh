mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/u8_bf16_layer.csv python tools/mesh_layer_once.py 8 1 4608 bf16 > /dev/null 2>&1
python tools/ncu_summary.py hbm gpurun_out/u8_bf16_layer.csv gpurun_out/u8_bf16_layer.md > /dev/null 2>&1; cat gpurun_out/u8_bf16_layer.md
timeout 600 ncu --set full --clock-control none -k regex:attn_kv2 -s 3 -c 1 -o gpurun_out/attn_kv2_full -f python tools/attn_once.py 3 4608 auto > /dev/null 2>&1
python tools/ncu_summary.py full gpurun_out/attn_kv2_full.ncu-rep gpurun_out/attn_kv2_full.md > /dev/null 2>&1; head -20 gpurun_out/attn_kv2_full.md
