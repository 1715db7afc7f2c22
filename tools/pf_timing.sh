KB_LIB_PATH=$PWD/tools/var/_kb_pftime.so KB_PF_SQ=32768 timeout 300 python tools/pf_probe.py > gpurun_out/pftime.log 2>&1
grep "pf-timing" gpurun_out/pftime.log | sort | uniq -c | sort -rn | head -40
