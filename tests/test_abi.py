"""The C-ABI library builds for sm_100a, loads without a GPU, and exports
every entry point include/kunserve_b200.h declares (no compute calls)."""

import ctypes
import os
import re

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "kunserve_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(kb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2412_18169_b200 import build
    path = build.build()
    lib = ctypes.CDLL(path)
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.kb_version() == 1


def test_python_binding_covers_header():
    from paper_2412_18169_b200 import runtime
    assert set(declared_symbols()) == set(runtime.EXPORTED)


def test_header_flag_values_match_the_binding():
    """Every flag #define the header declares has the same value in the
    Python binding (the binding passes / decodes them as plain ints)."""
    from paper_2412_18169_b200 import runtime
    defs = dict(re.findall(r"#define (KB_(?:KV|DECODE)_[A-Z_0-9]+) (\d+)u?", open(HEADER).read()))
    assert {"KB_KV_V_OVERFLOW", "KB_KV_V_UNDERFLOW", "KB_KV_NO_PAGE",
            "KB_DECODE_REUSE_PLAN", "KB_DECODE_COMBINE", "KB_DECODE_FUSE"} <= set(defs)
    for name, val in defs.items():
        py = getattr(runtime, name, None)
        if py is None:
            py = getattr(runtime, name[len("KB_"):])
        assert py == int(val), name


def test_runtime_refuses_without_library(tmp_path, monkeypatch):
    # the product path must fail loudly, never fall back to the CPU
    import importlib
    import paper_2412_18169_b200.runtime as rt
    monkeypatch.setattr(rt, "LIB_PATH", str(tmp_path / "missing.so"))
    src = open(rt.__file__).read()
    ns = {"__name__": "paper_2412_18169_b200.runtime_probe", "__file__": str(tmp_path / "x.py"),
          "__package__": "paper_2412_18169_b200"}
    try:
        exec(compile(src, str(tmp_path / "x.py"), "exec"), ns)
    except ImportError as exc:
        assert "no CPU fallback" in str(exc)
    else:
        raise AssertionError("runtime imported without _kb.so")
    importlib.reload(rt)


def test_prefill_split_heuristic():
    """runtime.prefill_splits: 1 for short contexts, a wave-filling count
    for long ones, never fewer than 16 key tiles per split."""
    from paper_2412_18169_b200.runtime import prefill_splits
    assert prefill_splits(1, 40, 2048, 2048) == 1          # 16 tiles: no room to split
    assert prefill_splits(1, 40, 2048, 32768) == 4         # config 4 late chunks (B200 sweep)
    for kv in (4096, 8192, 16384, 32768):
        s = prefill_splits(1, 32, 2048, kv)
        assert 1 <= s <= 8 and (kv // 128) >= 16 * s or s == 1
    # a grid that already fills whole waves stays unsplit
    assert prefill_splits(37, 32, 256, 32768) == 1          # 37 * 32 = 8 x 148 CTAs
