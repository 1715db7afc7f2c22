"""Config-4 paged prefill (Qwen2.5-14B, 32k prompt in 2048-token chunks):
auto split choice plus a forced kv_splits sweep.  `--ncu` runs the auto
configuration once (for an ncu capture)."""
import json
import sys
sys.path.insert(0, '.')
from paper_2412_18169_b200 import build
build.build()
import bench
from paper_2412_18169_b200 import runtime
rt = runtime.Runtime(0, max_slots=4, max_pages_per_seq=512)
if "--ncu" in sys.argv:
    print(bench.prefill_measure(rt, 1641.1, iters=1))
    sys.exit(0)
out = {"auto": bench.prefill_measure(rt, 1641.1)["roofline"]["frac"]}
for s in ((1,) if "--quick" in sys.argv else range(1, 9)):
    out[s] = bench.prefill_measure(rt, 1641.1, kv_splits=s)["roofline"]["frac"]
print(json.dumps(out))
