# ncu evidence for every data mover: one --set full capture per mover launch of the movers
# micro-benchmark (MOVERS_ONCE: each op once), and a launch list (duration + DRAM bytes) of
# FP8 USP layers on a virtual mesh (ranks as threads on cuda:0): U=8 and U=2 R=4 (cfg3 mesh).
mkdir -p gpurun_out
TAG=${TAG:-movers}
MOVERS_ONCE=1 timeout 900 ncu --set full --clock-control none \
  -o gpurun_out/${TAG}_full -f tools/cpp/movers_bench > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu movers rc=$?" >> gpurun_out/${TAG}_ncu.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/${TAG}_layer_u8.csv python tools/mesh_layer_once.py 8 1 4608 fp8 > gpurun_out/${TAG}_layer_u8.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/${TAG}_layer_u2r4.csv python tools/mesh_layer_once.py 8 4 16896 fp8 > gpurun_out/${TAG}_layer_u2r4.log 2>&1
timeout 300 tools/cpp/movers_bench > gpurun_out/${TAG}.jsonl 2>&1
tail -3 gpurun_out/${TAG}_ncu.log; tail -2 gpurun_out/${TAG}_layer_u8.log; cat gpurun_out/${TAG}.jsonl | cut -c1-200
