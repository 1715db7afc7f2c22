export PYTHONUNBUFFERED=1
python -m paper_2412_18169_b200.build
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2f_gpu_tests.log 2>&1
echo tests_rc=$?
timeout 1800 bash tools/profile.sh r2f
tail -c 1000 gpurun_out/r2f_gpu_tests.log
