# per-tile MMA / softmax timeline of one prefill CTA (variant built with -DKB_PF_TRACE)
KB_LIB_PATH=$PWD/tools/var/_kb_pft.so timeout 300 python -c "
import sys; sys.path.insert(0, '.')
import bench
from paper_2412_18169_b200 import runtime
bench.prefill_measure(runtime.Runtime(0), 1637.1, ctx=32768, chunk=32768, kv_splits=1, iters=1)
" > gpurun_out/pft.log 2>&1
grep -c pft gpurun_out/pft.log
