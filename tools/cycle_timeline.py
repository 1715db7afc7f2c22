"""GPU timeline of one overload-cycle step (torch.profiler / CUPTI): every
kernel and memcpy with its start offset, duration and the idle gap before
it.  Run on the GPU box:  python tools/cycle_timeline.py > gpurun_out/tl.txt"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_18169_b200 import build, runtime  # noqa: E402
from paper_2412_18169_b200.core import SHAPES  # noqa: E402
from paper_2412_18169_b200.cycle import OverloadCycle  # noqa: E402

build.build()
rt = runtime.Runtime(0, max_slots=512, max_pages_per_seq=256)
cyc = OverloadCycle([rt, rt], SHAPES["llama3_8b"], 16 << 30)
for _ in range(3):
    cyc.step()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    rep = cyc.step()
print("event ms", {k: round(v, 3) for k, v in rep.ms.items()}, "host ms",
      {k: round(v, 3) for k, v in rep.host_ms.items()})
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
prev_end = t0
busy = 0.0
for e in evs:
    s, d = e.time_range.start, e.time_range.elapsed_us()
    gap = s - prev_end
    busy += d
    print(f"{(s - t0) / 1e3:9.3f} ms  gap {gap:8.1f} us  dur {d:9.1f} us  {e.name[:60]}")
    prev_end = max(prev_end, e.time_range.end)
print(f"span {(prev_end - t0) / 1e3:.3f} ms, busy {busy / 1e3:.3f} ms")
cyc.close()
