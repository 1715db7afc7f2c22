export PYTHONUNBUFFERED=1
python -m paper_2412_18169_b200.build
timeout 900 python -m pytest tests/test_device.py tests/test_parity_full.py -m gpu -q -x -k "decode or pdl or block_tokens or two_runtimes" > gpurun_out/r2x_dec_tests.log 2>&1
echo dec_tests_rc=$?
tail -3 gpurun_out/r2x_dec_tests.log
bash tools/decode_ab.sh r2x tools/var/_kb_prev.so
