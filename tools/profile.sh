#!/bin/bash
# ncu evidence for profiles/: launch list of one short bench run + full
# captures of the top kernels.  Run on the GPU box:  bash tools/profile.sh <tag>
TAG=${1:-r2}
export PYTHONUNBUFFERED=1
K='regex:copy_|grow_kernel|release_kernel|compact_|range_mark|decode_|prefill_|kv_append|hash_'
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --csv \
    --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --decode-iters 2 --no-ttft \
    > gpurun_out/ncu_launch_$TAG.log 2>&1
echo launches_rc=$?
# skip the setup / warm-up launches: copy_pages -> two bulk exchange
# launches, copy_flat -> two 2 GB slab pulls (launches 0-21 of the cycle's
# copy_flat are the restores' runs; later ones are small hand-off copies)
for KN in copy_pages_kernel copy_flat_kernel decode_tc_kernel; do
  SKIP=40
  [ "$KN" = copy_flat_kernel ] && SKIP=4
  ncu --set full --clock-control none --import-source on -k regex:$KN -s $SKIP -c 2 \
      -o gpurun_out/prof_${TAG}_$KN \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline --decode-iters 1 --no-ttft \
      > gpurun_out/ncu_full_${TAG}_$KN.log 2>&1
  echo full_${KN}_rc=$?
done
ncu --set full --clock-control none --import-source on -k regex:prefill_tc -s 30 -c 1 \
    -o gpurun_out/prof_${TAG}_prefill_tc_kernel python tools/prefill_probe.py --ncu \
    > gpurun_out/ncu_full_${TAG}_prefill.log 2>&1
echo full_prefill_rc=$?
# small-batch decode (a pipeline stage's 16 sequences)
KB_PROBE_NSEQ=16 ncu --set full --clock-control none --import-source on -k regex:decode_tc -s 20 -c 2 \
    -o gpurun_out/prof_${TAG}_decode16 python tools/decode_batch_probe.py \
    > gpurun_out/ncu_full_${TAG}_decode16.log 2>&1
echo full_decode16_rc=$?
for f in gpurun_out/prof_${TAG}_*.ncu-rep; do
  python tools/ncu_summary.py $f >> gpurun_out/${TAG}_ncu_full_summary.txt
done
python tools/launch_summary.py gpurun_out/launches_$TAG.csv "python bench.py --steps 2 --warmup 3 --no-ttft" \
    > gpurun_out/${TAG}_launch_summary.txt
