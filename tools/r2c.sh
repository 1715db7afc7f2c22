export PYTHONUNBUFFERED=1
python -m paper_2412_18169_b200.build
timeout 900 python -m pytest tests/test_parity_full.py tests/test_device_engine.py -q -x > gpurun_out/r2c_tests.log 2>&1
echo tests_rc=$?
timeout 900 python tools/wall_log_probe.py r2c '{"policies": ["kunserve", "recompute"]}' > gpurun_out/r2c_ttft.log 2>&1
echo ttft_rc=$?
tail -c 600 gpurun_out/r2c_tests.log
tail -c 3000 gpurun_out/r2c_ttft.log
