export PYTHONUNBUFFERED=1
python -m paper_2412_18169_b200.build
KB_LIB_PATH=$PWD/tools/var/_kb_pftiming.so timeout 300 python tools/prefill_probe.py --ncu > gpurun_out/r2t_pftiming.log 2>&1
grep "pf-timing" gpurun_out/r2t_pftiming.log | tail -12
ncu --set full --clock-control none --import-source on -k regex:prefill_tc -s 30 -c 1 \
    -o gpurun_out/prof_r2t_prefill python tools/prefill_probe.py --ncu > gpurun_out/r2t_ncu.log 2>&1
echo ncu_rc=$?
ncu -i gpurun_out/prof_r2t_prefill.ncu-rep --page source --csv > gpurun_out/r2t_prefill_source.csv 2>&1
ncu -i gpurun_out/prof_r2t_prefill.ncu-rep --page raw --csv > gpurun_out/r2t_prefill_raw.csv 2>&1
ls -la gpurun_out/ | grep r2t
