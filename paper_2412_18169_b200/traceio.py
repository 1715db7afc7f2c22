"""Arrival traces (ref pkg/src/dropsim/traceio.py:1-155).

`synth_burst` draws exactly the same sequence as the reference for a given
seed (same `random.Random` call order), so the engine can be checked
against the reference's event logs and the benches replay the reference's
bursts.  CSV I/O keeps the reference's `arrival_s,input_len,output_len`
format.
"""

from __future__ import annotations

import csv
import math
import random
from dataclasses import dataclass

from .core import s_to_us

HEADER = ["arrival_s", "input_len", "output_len"]
# dataset presets: (input_mean, output_mean) tokens (ref config.py:20-24)
TRACE_PRESETS = {"burstgpt": (642, 262), "sharegpt": (1660, 373), "longbench": (5900, 499)}


@dataclass(frozen=True)
class TraceRecord:
    arrival_us: int
    input_len: int
    output_len: int


def _length(rng: random.Random, dist: str, mean: int, sigma: float) -> int:
    if dist == "fixed":
        return max(1, mean)
    if dist == "uniform":
        return max(1, rng.randint(max(1, mean // 2), mean + mean // 2))
    if dist == "lognormal":
        mu = math.log(mean) - sigma * sigma / 2.0
        return max(1, round(rng.lognormvariate(mu, sigma)))
    raise ValueError(f"unknown length distribution {dist!r}")


def synth_burst(duration_s: float, base_rps: float, burst_rps: float, burst_start_s: float,
                burst_end_s: float, input_mean: int, output_mean: int,
                length_dist: str = "lognormal", sigma: float = 0.6,
                seed: int = 0) -> list[TraceRecord]:
    """Poisson arrivals with a rate step inside [burst_start, burst_end)
    (ref traceio.py:132-155)."""
    if duration_s <= 0 or base_rps <= 0 or burst_rps <= 0:
        raise ValueError("duration and rates must be positive")
    rng = random.Random(seed)
    out: list[TraceRecord] = []
    t = 0.0
    while True:
        t += rng.expovariate(burst_rps if burst_start_s <= t < burst_end_s else base_rps)
        if t >= duration_s:
            return out
        inp = _length(rng, length_dist, input_mean, sigma)
        outl = _length(rng, length_dist, output_mean, sigma)
        out.append(TraceRecord(s_to_us(t), inp, outl))


def load_trace(path: str) -> list[TraceRecord]:
    recs: list[TraceRecord] = []
    with open(path, newline="") as fh:
        rows = csv.reader(fh)
        if next(rows, None) != HEADER:
            raise ValueError(f"line 1: expected header {','.join(HEADER)}")
        prev = None
        for lineno, row in enumerate(rows, start=2):
            if not row:
                continue
            if len(row) != 3:
                raise ValueError(f"line {lineno}: expected 3 columns, got {len(row)}")
            try:
                a, i, o = float(row[0]), int(row[1]), int(row[2])
            except ValueError as exc:
                raise ValueError(f"line {lineno}: {exc}") from exc
            if a < 0:
                raise ValueError(f"line {lineno}: negative arrival time")
            if i < 1 or o < 1:
                raise ValueError(f"line {lineno}: lengths must be >= 1")
            us = s_to_us(a)
            if prev is not None and us < prev:
                raise ValueError(f"line {lineno}: arrivals must be non-decreasing")
            prev = us
            recs.append(TraceRecord(us, i, o))
    return recs


def save_trace(path: str, records: list[TraceRecord]) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(HEADER)
        for r in records:
            w.writerow([f"{r.arrival_us / 1_000_000:.6f}", r.input_len, r.output_len])
