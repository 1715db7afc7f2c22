# compute-sanitizer over the device parity suites (GPU box): bash tools/sanitize_all.sh <tag> ["memcheck racecheck synccheck"]
TAG=${1:-r2}
export PYTHONUNBUFFERED=1
export KB_SANITIZER=1  # timing-claim tests skip themselves
python -m paper_2412_18169_b200.build
TOOLS=${2:-memcheck}
FILES=${3:-tests/test_device.py tests/test_parity_full.py tests/test_cycle.py tests/test_device_scenarios.py tests/test_failure.py}
for tool in $TOOLS; do
  timeout 3000 compute-sanitizer --tool $tool --print-limit 20 python -m pytest $FILES -m gpu -q -x > gpurun_out/${TAG}_${tool}_all.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/${TAG}_${tool}_all.log | tail -3
done
