# ncu --set full of the attention kernel for several variants at one shape (4th launch).
# usage: H=6 S=4608 MODE=whole bash tools/gpu_job_ncu_ab.sh VARIANT...   ('main' = lib/)
mkdir -p gpurun_out
H=${H:-6}; S=${S:-4608}; MODE=${MODE:-auto}
for v in "$@"; do
  if [ "$v" = main ]; then unset FUSP_VARIANT; else export FUSP_VARIANT=$v; fi
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_fwd -s 3 -c 1 \
    -o gpurun_out/ab_${v}_$MODE -f python tools/attn_once.py $H $S $MODE > gpurun_out/ab_${v}_$MODE.log 2>&1
done
unset FUSP_VARIANT
