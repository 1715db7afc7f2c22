"""The overload cycle (cycle.OverloadCycle) end to end on device pools at a
small shape: plan -> drop -> exchange -> restore -> consolidate, nothing
waiting on the host between phases.  Every weight byte and every
long-lived resident's KV page must come back bit for bit, every step must
move the same bytes, and the pools must end where they started."""

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2412_18169_b200.core import SHAPES  # noqa: E402


@pytest.fixture(scope="module")
def rt():
    from paper_2412_18169_b200 import build
    build.build()
    from paper_2412_18169_b200 import runtime
    return runtime.Runtime(0, max_slots=512, max_pages_per_seq=256)


@pytest.mark.parametrize("shape_name", ["tiny", "llama3_8b"])
def test_cycle_round_trips_bit_exact(rt, shape_name):
    from paper_2412_18169_b200.cycle import OverloadCycle
    shape = SHAPES[shape_name]
    if shape_name == "tiny":
        cyc = OverloadCycle([rt, rt], shape, 1 << 20, kv_chunk_bytes=64 << 10,
                            param_chunk_bytes=1 << 20, input_mean=200)
    else:  # full-size layers, a small KV budget (a few residents)
        cyc = OverloadCycle([rt, rt], shape, 2 << 30, input_mean=1660)
    w0, k0 = cyc.weight_checksums(), cyc.kv_checksums()
    infos0 = {i: p.info() for i, p in cyc.pools.items()}
    reps = [cyc.step() for _ in range(2)]
    cyc.pause_merged = True
    cyc.step()
    # merged state: every member holds only its stage's layers
    layout = cyc.merged_decode_layout()
    assert len(layout) == 2 and sorted(r for r, _ in layout.values()) == [
        (0, shape.num_layers // 2), (shape.num_layers // 2, shape.num_layers)]
    reps.append(cyc.resume())
    torch.cuda.synchronize()
    assert cyc.weight_checksums() == w0
    k1 = cyc.kv_checksums()
    assert k0.keys() == k1.keys() and all(torch.equal(k0[r], k1[r]) for r in k0)
    for r in reps:
        assert r.bytes_kv_exchange > 0 and r.bytes_param > 0 and r.bytes_kv_consolidate > 0
        assert r.bytes_moved == reps[0].bytes_moved
        assert r.ms["total"] > 0
    for i, p in cyc.pools.items():
        inf = p.info()
        assert inf.extent_pages == infos0[i].extent_pages  # every slab reserved again
        assert inf.live_pages == infos0[i].live_pages
    cyc.close()
