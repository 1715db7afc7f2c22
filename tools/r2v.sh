export PYTHONUNBUFFERED=1
python -m paper_2412_18169_b200.build
for v in paper_2412_18169_b200/_kb.so tools/var/_kb_emu5.so tools/var/_kb_st.so tools/var/_kb_st5.so paper_2412_18169_b200/_kb.so; do
  echo "== $v"; KB_LIB_PATH=$PWD/$v timeout 300 python tools/prefill_probe.py --quick 2>&1 | tail -1
done
