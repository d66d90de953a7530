# ncu evidence for every data mover: one --set full capture per mover launch of the movers
# micro-benchmark (MOVERS_ONCE: each op once), summarised ON THE BOX (the .ncu-rep is too big to
# bring back), and launch lists (duration + DRAM bytes) of FP8 USP layers on a virtual mesh
# (ranks as threads on cuda:0): U=8 and U=2 R=4 (cfg3 mesh); VARIANT=base for the previous build.
mkdir -p gpurun_out
TAG=${TAG:-movers}
export MOVERS_ONCE=1
timeout 900 ncu --set full --clock-control none -k regex:'amax|quantize|pack|stage|fp8|bf16_to|peer' -o /tmp/${TAG}_full -f tools/cpp/movers_bench > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu movers rc=$?" >> gpurun_out/${TAG}_ncu.log
python tools/ncu_summary.py movers /tmp/${TAG}_full.ncu-rep gpurun_out/${TAG}_ncu.md >> gpurun_out/${TAG}_ncu.log 2>&1
unset MOVERS_ONCE
for v in "" ${VARIANTS}; do
  for cfg in "8 1 4608 fp8 u8" "8 4 16896 fp8 u2r4" "8 1 4608 fp8block u8blk"; do
    set -- $cfg
    FUSP_VARIANT=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file gpurun_out/${TAG}_layer_$5${v:+_$v}.csv python tools/mesh_layer_once.py $1 $2 $3 $4 > gpurun_out/${TAG}_layer_$5${v:+_$v}.log 2>&1
    python tools/ncu_summary.py hbm gpurun_out/${TAG}_layer_$5${v:+_$v}.csv gpurun_out/${TAG}_layer_$5${v:+_$v}.md > /dev/null 2>&1
  done
done
timeout 300 tools/cpp/movers_bench > gpurun_out/${TAG}.jsonl 2>&1
tail -3 gpurun_out/${TAG}_ncu.log; head -40 gpurun_out/${TAG}_ncu.md; cat gpurun_out/${TAG}.jsonl | cut -c1-220
