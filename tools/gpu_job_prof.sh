# Launch list of the bench step (cold, serialized) + one full capture of a named kernel.
mkdir -p gpurun_out
K=${KERNEL:-stage_kernel}
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c ${NLAUNCH:-120} --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/prof_bench.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:${K} -s ${SKIP:-2} -c 1 -o gpurun_out/kernel_full -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/prof_full.log 2>&1
python tools/ncu_summary.py launches gpurun_out/launches.csv gpurun_out/launches.md; head -40 gpurun_out/launches.md
