# prefill A/B: tools/pf_probe.py per library variant (tools/var/*.so built on the CPU side)
export PYTHONUNBUFFERED=1
TAG=${1:-ab}
shift
for rep in 1 2; do
for v in paper_2412_18169_b200/_kb.so "$@"; do
  KB_LIB_PATH=$PWD/$v timeout 300 python tools/pf_probe.py 2>&1 | grep '^{' >> gpurun_out/${TAG}_pf_ab.log
done
done
cat gpurun_out/${TAG}_pf_ab.log
