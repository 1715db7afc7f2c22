"""One paged-prefill configuration (config 4: Qwen2.5-14B, 32k prompt) for ncu."""
import sys
sys.path.insert(0, '.')
from paper_2412_18169_b200 import build
build.build()
import bench
from paper_2412_18169_b200 import runtime
rt = runtime.Runtime(0, max_slots=4, max_pages_per_seq=512)
print(bench.prefill_measure(rt, 1641.1, iters=1))
