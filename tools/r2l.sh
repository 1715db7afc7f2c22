export PYTHONUNBUFFERED=1
python -m paper_2412_18169_b200.build
timeout 900 python -m pytest tests/test_device.py tests/test_parity_full.py -m gpu -q -x -k "decode or pdl or block_tokens" > gpurun_out/r2l_dec_tests.log 2>&1
echo dec_tests_rc=$?
tail -3 gpurun_out/r2l_dec_tests.log
bash tools/decode_ab.sh r2l tools/var/_kb_head.so
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2l_gpu_tests.log 2>&1
echo all_tests_rc=$?
tail -5 gpurun_out/r2l_gpu_tests.log
