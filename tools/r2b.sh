export PYTHONUNBUFFERED=1
python -m paper_2412_18169_b200.build
timeout 900 python -m pytest tests/test_parity_full.py tests/test_device_engine.py -q -x > gpurun_out/r2b_tests.log 2>&1
echo tests_rc=$?
timeout 900 python tools/ttft_probe.py '{"kv_gib": 1.25, "base_rps": 3.0, "output_mean": 128, "policies": ["kunserve", "recompute"]}' > gpurun_out/r2b_ttft.log 2>&1
echo ttft_rc=$?
tail -c 1500 gpurun_out/r2b_tests.log
tail -c 3000 gpurun_out/r2b_ttft.log
