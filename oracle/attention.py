"""ORACLE -- fp32 CPU paged attention.  TEST INFRASTRUCTURE ONLY.

The reference has no attention math (its only trace is
the cost proxy attention_units(c, p) = p*c + (c^2+c)/2 at
pkg/src/dropsim/costmodel.py:50-57), so parity for attention is UNPINNED at
the reference level: this is a plain fp32 restatement of scaled-dot-product
attention with grouped KV heads, and the device kernels must match it within
BASELINE.json's bf16 tolerance (max-abs <= 2e-2, mean-rel <= 1e-3).

Inputs are bf16 bit patterns (uint16) so the CPU sees exactly the bytes the
GPU read; everything is computed in fp32 (numpy, all host threads via BLAS).
"""

from __future__ import annotations

import numpy as np


def bf16_to_f32(x: np.ndarray) -> np.ndarray:
    return (x.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bits."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    rounding = ((u >> 16) & 1) + 0x7FFF
    return ((u + rounding) >> 16).astype(np.uint16)


def decode_ref(q: np.ndarray, k: np.ndarray, v: np.ndarray, scale: float) -> np.ndarray:
    """One query token per sequence.  q [Hq, d]; k, v [ctx, Hkv, d] (fp32).
    Returns o [Hq, d] fp32."""
    hq, d = q.shape
    hkv = k.shape[1]
    g = hq // hkv
    out = np.empty((hq, d), dtype=np.float32)
    for h in range(hkv):
        qs = q[h * g:(h + 1) * g]                       # [g, d]
        s = (qs @ k[:, h].T) * scale                    # [g, ctx]
        s -= s.max(axis=1, keepdims=True)
        p = np.exp(s)
        p /= p.sum(axis=1, keepdims=True)
        out[h * g:(h + 1) * g] = p @ v[:, h]
    return out


def prefill_ref(q: np.ndarray, k: np.ndarray, v: np.ndarray, prefix: int,
                scale: float) -> np.ndarray:
    """Chunk of c query tokens at positions [prefix, prefix + c) attending
    causally over k, v [prefix + c, Hkv, d].  q [c, Hq, d] -> o [c, Hq, d]."""
    c, hq, d = q.shape
    hkv = k.shape[1]
    g = hq // hkv
    n = k.shape[0]
    qpos = prefix + np.arange(c)[:, None]
    kpos = np.arange(n)[None, :]
    mask = kpos <= qpos                                  # [c, n]
    out = np.empty((c, hq, d), dtype=np.float32)
    for hh in range(hq):
        h = hh // g
        s = (q[:, hh] @ k[:, h].T) * scale               # [c, n]
        s = np.where(mask, s, -np.inf)
        s -= s.max(axis=1, keepdims=True)
        p = np.exp(s)
        p /= p.sum(axis=1, keepdims=True)
        out[:, hh] = p @ v[:, h]
    return out


def check_close(got: np.ndarray, want: np.ndarray, max_abs: float = 2e-2,
                mean_rel: float = 1e-3) -> tuple[float, float]:
    """BASELINE.json tolerance: max-abs <= 2e-2 and mean-rel <= 1e-3, where
    mean-rel = mean|got - want| / mean|want|."""
    diff = np.abs(got.astype(np.float64) - want.astype(np.float64))
    ma = float(diff.max()) if diff.size else 0.0
    denom = float(np.abs(want).mean()) if want.size else 1.0
    mr = float(diff.mean() / max(denom, 1e-30)) if diff.size else 0.0
    return ma, mr
