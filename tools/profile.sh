#!/bin/bash
# ncu evidence for profiles/: launch list of one bench run + full captures of
# the top kernels.  Run on the GPU box:  bash tools/profile.sh <tag>
TAG=${1:-r1}
export PYTHONUNBUFFERED=1
K='regex:copy_|grow_kernel|release_kernel|compact_|range_mark|decode_|prefill_|kv_append'
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv \
    --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --decode-iters 2 --no-ttft \
    > gpurun_out/ncu_launch_$TAG.log 2>&1
echo launches_rc=$?
for KN in copy_pages_kernel decode_tc_kernel copy_flat_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$KN -s 8 -c 2 \
      -o gpurun_out/prof_${TAG}_$KN \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline --decode-iters 1 --no-ttft \
      > gpurun_out/ncu_full_${TAG}_$KN.log 2>&1
  echo full_${KN}_rc=$?
done
ncu --set full --clock-control none --import-source on -k regex:prefill_tc -s 30 -c 1 \
    -o gpurun_out/prof_${TAG}_prefill_tc_kernel python tools/prefill_probe.py \
    > gpurun_out/ncu_full_${TAG}_prefill.log 2>&1
echo full_prefill_rc=$?
