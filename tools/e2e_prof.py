"""Host-side profile of the end-to-end overload cycle (cProfile around
cycle.step with the e2e read-back), step-return / total / device-span times.
Run on the GPU box: python tools/e2e_prof.py"""
import sys, time, cProfile, pstats, io
sys.path.insert(0, '.')
import torch
from paper_2412_18169_b200 import build, runtime
build.build()
from paper_2412_18169_b200.core import SHAPES
from paper_2412_18169_b200.cycle import OverloadCycle
rt = runtime.Runtime(0, max_slots=512, max_pages_per_seq=256)
cyc = OverloadCycle([rt, rt], SHAPES["llama3_8b"], 16 << 30)
res = torch.empty(len(cyc.tokens), dtype=torch.int32).pin_memory()
cyc.auto_refill = False
for i in range(3):
    b = cyc.burst_for(seed=100 + i); torch.cuda.synchronize()
    r = cyc.step(burst=b, light=True, on_enqueued=lambda: res.copy_(cyc.home_first_pages(), non_blocking=True)); torch.cuda.synchronize(); cyc.refill()
times = []
pr = cProfile.Profile()
for i in range(5):
    b = cyc.burst_for(seed=200 + i); torch.cuda.synchronize()
    t0 = time.perf_counter()
    pr.enable()
    r = cyc.step(burst=b, light=True, on_enqueued=lambda: res.copy_(cyc.home_first_pages(), non_blocking=True))
    t_ret = time.perf_counter()
    torch.cuda.synchronize()
    pr.disable()
    t1 = time.perf_counter()
    times.append((round((t_ret - t0) * 1e3, 2), round((t1 - t0) * 1e3, 2), round(r.ms["total"], 2)))
    cyc.refill()
print("step-return / total / device span ms:", times)
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(18); print(s.getvalue()[:4000])
