"""Chunk / batch cost model (ref pkg/src/dropsim/costmodel.py:1-167).

cost(c new tokens over a p-token prefix) = alpha * (p*c + (c^2+c)/2)
                                          + beta * c + gamma
and a batch shares one gamma.  The engine uses it in model mode for stage
times; with real devices, measured stage times replace it and `fit`
re-derives (alpha, beta, gamma) from them.  Arithmetic order follows the
reference so model-mode event logs are byte-identical.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from .core import Chunk


@dataclass(frozen=True)
class CostCoefficients:
    alpha: float
    beta: float
    gamma: float
    batch_discount: Optional[float] = None

    def __post_init__(self) -> None:
        if self.alpha < 0 or self.beta < 0 or self.gamma < 0:
            raise ValueError("cost coefficients must be >= 0")

    @property
    def discount(self) -> float:
        return self.gamma if self.batch_discount is None else self.batch_discount


def attention_units(c: int, p: int) -> float:
    """Token pairs of attention work for a chunk (ref costmodel.py:50-52)."""
    return p * c + (c * c + c) / 2


def chunk_cost(chunk: Chunk, k: CostCoefficients) -> float:
    c = chunk.token_count
    return k.alpha * attention_units(c, chunk.prefix_len) + k.beta * c + k.gamma


def batch_cost(chunks: Sequence[Chunk], k: CostCoefficients) -> float:
    """Sum of chunk costs minus (n-1) shared discounts (ref costmodel.py:60-69)."""
    if not chunks:
        raise ValueError("batch_cost of an empty batch")
    total = sum(chunk_cost(ch, k) for ch in chunks)
    return total - (len(chunks) - 1) * k.discount


def _design(chunks) -> tuple[float, float, float]:
    return (sum(attention_units(c.token_count, c.prefix_len) for c in chunks),
            float(sum(c.token_count for c in chunks)), 1.0)


def fit_token_baseline(samples) -> tuple[CostCoefficients, float]:
    """The prefix-blind baseline fit (ref costmodel.py:97-112): alpha pinned
    to 0, (beta, gamma) least squares on token counts alone."""
    if len(samples) < 2:
        raise ValueError("insufficient profile diversity: need >= 2 samples")
    m = np.array([_design(ch)[1:] for ch, _ in samples])
    y = np.array([t for _, t in samples])
    if np.linalg.matrix_rank(m) < 2:
        raise ValueError("insufficient profile diversity: rank-deficient profile")
    sol = np.maximum(np.linalg.lstsq(m, y, rcond=None)[0], 0.0)
    rms = float(np.sqrt(np.mean((m @ sol - y) ** 2)))
    return CostCoefficients(0.0, float(sol[0]), float(sol[1])), rms


def synth_profile(compositions, truth: CostCoefficients, noise_frac: float = 0.0,
                  seed: int = 0) -> list:
    """(chunks, seconds) samples of a hidden cost model with seeded
    multiplicative gaussian noise (ref costmodel.py:115-130)."""
    import random
    rng = random.Random(seed)
    out = []
    for chunks in compositions:
        t = batch_cost(chunks, truth)
        if noise_frac > 0:
            t *= 1.0 + rng.gauss(0.0, noise_frac)
        out.append((tuple(chunks), t))
    return out


def fit(samples) -> tuple[CostCoefficients, float]:
    """Least-squares (alpha, beta, gamma) from (chunks, seconds) samples
    (ref costmodel.py:78-94); the device engine feeds measured stage times."""
    if len(samples) < 3:
        raise ValueError("insufficient profile diversity: need >= 3 samples")
    m = np.array([_design(ch) for ch, _ in samples])
    y = np.array([t for _, t in samples])
    if np.linalg.matrix_rank(m) < 3:
        raise ValueError("insufficient profile diversity: rank-deficient profile")
    sol = np.maximum(np.linalg.lstsq(m, y, rcond=None)[0], 0.0)
    rms = float(np.sqrt(np.mean((m @ sol - y) ** 2)))
    return CostCoefficients(float(sol[0]), float(sol[1]), float(sol[2])), rms


# ------------------------------------------------------------ profile CSV
# (ref costmodel.py:133-167) one row per chunk: c, p, batch_id, measured_us
PROFILE_HEADER = ["c", "p", "batch_id", "measured_us"]


def write_profile(path: str, samples) -> None:
    import csv
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(PROFILE_HEADER)
        for bid, (chunks, seconds) in enumerate(samples):
            us = int(round(seconds * 1_000_000))
            w.writerows([c.token_count, c.prefix_len, bid, us] for c in chunks)


def read_profile(path: str) -> list:
    """Samples back from a profile CSV, batches in first-seen order; a batch
    whose rows disagree on measured_us, a bad header or a non-integer field
    raise ValueError naming the line."""
    import csv
    batches: dict = {}
    with open(path, newline="") as fh:
        r = csv.DictReader(fh)
        if r.fieldnames != PROFILE_HEADER:
            raise ValueError(f"bad profile header: {r.fieldnames}")
        for lineno, row in enumerate(r, start=2):
            try:
                c, p, bid, us = (int(row[k]) for k in PROFILE_HEADER)
            except (TypeError, ValueError) as exc:
                raise ValueError(f"line {lineno}: {exc}") from exc
            chunks, seen_us = batches.setdefault(bid, ([], us))
            if seen_us != us:
                raise ValueError(f"line {lineno}: batch {bid} measured_us mismatch")
            chunks.append(Chunk(rid=0, token_count=c, prefix_len=p))
    return [(tuple(ch), us / 1_000_000) for ch, us in batches.values()]
