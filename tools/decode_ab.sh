# decode A/B: batch probe per library variant (tools/var/*.so built on the CPU side)
export PYTHONUNBUFFERED=1
TAG=${1:-ab}
shift
for v in paper_2412_18169_b200/_kb.so "$@"; do
  echo "== $v" >> gpurun_out/${TAG}_decode_ab.log
  KB_LIB_PATH=$PWD/$v timeout 300 python tools/decode_batch_probe.py >> gpurun_out/${TAG}_decode_ab.log 2>&1
done
for m in 0 1; do
  echo "== _kb.so combine=$m forced" >> gpurun_out/${TAG}_decode_ab.log
  KB_PROBE_MERGE=$m timeout 300 python tools/decode_batch_probe.py >> gpurun_out/${TAG}_decode_ab.log 2>&1
done
echo "== _kb.so append first" >> gpurun_out/${TAG}_decode_ab.log
KB_PROBE_APPEND=1 timeout 300 python tools/decode_batch_probe.py >> gpurun_out/${TAG}_decode_ab.log 2>&1
KB_PROBE_SIZES=16,147 timeout 300 python tools/decode_trace_probe.py > gpurun_out/${TAG}_trace.log 2>&1
cat gpurun_out/${TAG}_decode_ab.log gpurun_out/${TAG}_trace.log | grep -v "^\["
