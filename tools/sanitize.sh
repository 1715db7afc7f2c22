# compute-sanitizer over the decode / PDL-chain parity tests (GPU box):  bash tools/sanitize.sh <tag>
TAG=${1:-r2}
export PYTHONUNBUFFERED=1
python -m paper_2412_18169_b200.build
K="${2:-paged_decode or pdl or block_tokens or prefill}"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_device.py tests/test_parity_full.py -m gpu -q -x -k "$K" > gpurun_out/${TAG}_sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|HAZARD|passed|failed" gpurun_out/${TAG}_sanitizer_$tool.log | tail -3
done
