export PYTHONUNBUFFERED=1
python -m paper_2412_18169_b200.build
timeout 900 python -m pytest tests/test_device.py tests/test_parity_full.py tests/test_device_engine.py -m gpu -q -x -k "decode or pdl or block_tokens or engine" > gpurun_out/r2k_tests.log 2>&1
echo tests_rc=$?
tail -5 gpurun_out/r2k_tests.log
bash tools/decode_ab.sh r2k tools/var/_kb_head.so tools/var/_kb_ipc3.so tools/var/_kb_ipc4.so
