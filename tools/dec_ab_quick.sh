# decode A/B, quick: tools/decode_batch_probe.py per library variant, 3 rounds interleaved
export PYTHONUNBUFFERED=1
TAG=${1:-ab}
shift
for rep in 1 2 3; do
for v in paper_2412_18169_b200/_kb.so "$@"; do
  echo "$v $(KB_LIB_PATH=$PWD/$v timeout 300 python tools/decode_batch_probe.py 2>&1 | tail -1)" >> gpurun_out/${TAG}_dec_ab.log
done
done
cat gpurun_out/${TAG}_dec_ab.log
