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
