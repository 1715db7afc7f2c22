export PYTHONUNBUFFERED=1
python -m paper_2412_18169_b200.build
timeout 900 python -m pytest tests/test_device_scenarios.py tests/test_device_engine.py -q > gpurun_out/r2d_tests.log 2>&1
echo tests_rc=$?
timeout 900 python tools/wall_log_probe.py r2d '{"policies": ["kunserve", "recompute"]}' > gpurun_out/r2d_ttft.log 2>&1
echo ttft_rc=$?
tail -c 800 gpurun_out/r2d_tests.log
