export PYTHONUNBUFFERED=1
python -m paper_2412_18169_b200.build
for v in paper_2412_18169_b200/_kb.so tools/var/_kb_emu3.so tools/var/_kb_emu4.so tools/var/_kb_emu5.so tools/var/_kb_emu8.so; do
  echo "== $v"; KB_LIB_PATH=$PWD/$v timeout 300 python tools/prefill_probe.py --quick 2>&1 | tail -1
done
