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


def fit(samples) -> tuple[CostCoefficients, float]:
    """Least-squares (alpha, beta, gamma) from (chunks, seconds) samples
    (ref costmodel.py:78-94); the device engine feeds measured stage times."""
    if len(samples) < 3:
        raise ValueError("insufficient profile diversity: need >= 3 samples")
    rows = [(sum(attention_units(c.token_count, c.prefix_len) for c in ch),
             float(sum(c.token_count for c in ch)), 1.0) for ch, _ in samples]
    m = np.array(rows)
    y = np.array([t for _, t in samples])
    if np.linalg.matrix_rank(m) < 3:
        raise ValueError("insufficient profile diversity: rank-deficient profile")
    sol = np.maximum(np.linalg.lstsq(m, y, rcond=None)[0], 0.0)
    rms = float(np.sqrt(np.mean((m @ sol - y) ** 2)))
    return CostCoefficients(float(sol[0]), float(sol[1]), float(sol[2])), rms
