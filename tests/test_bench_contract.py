"""bench.py's two arms report the same workload: the reference arm (CPU port)
samples the GPU arm's resident list, chosen host-side by
cycle.resident_tokens over the same KV budget (147 residents at 16 GiB per
replica -- the `residents` of the GPU bench lines)."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_reports_the_gpu_arms_workload():
    import bench
    from paper_2412_18169_b200.cycle import resident_tokens
    full = bench.host_residents(16.0)
    assert len(full) == 147
    cfg = bench.arm_config(16.0, len(full), 1)
    assert cfg["residents"] == 147 and cfg["model"] == "llama3_8b"
    # the selection fills each replica to at most 90% of its token capacity
    toks, home = resident_tokens({0: 100_000, 1: 100_000})
    for iid in (0, 1):
        assert sum(t for r, t in toks.items() if home[r] == iid) <= 90_000
    assert resident_tokens({0: 100_000, 1: 100_000}) == (toks, home)
