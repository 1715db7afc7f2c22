import sys, json
sys.path.insert(0, '.')
from paper_2412_18169_b200 import build, runtime
build.build()
from paper_2412_18169_b200.core import SHAPES
from paper_2412_18169_b200.cycle import OverloadCycle
rt = runtime.Runtime(0, max_slots=512, max_pages_per_seq=256)
cyc = OverloadCycle([rt, rt], SHAPES["llama3_8b"], 16 << 30)
for b in (8, 16, 4, 1000):
    cyc.exchange_batch = b
    for _ in range(3): cyc.step()
    ms = [cyc.step().ms for _ in range(5)]
    print(b, round(sum(m["exchange"] for m in ms)/5, 3), round(sum(m["total"] for m in ms)/5, 3))
