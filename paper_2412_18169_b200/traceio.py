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


def rescale(records: list[TraceRecord], factor: float, seed: int = 0) -> list[TraceRecord]:
    """Scale a trace's arrival rate, keeping its temporal shape (ref
    traceio.py:71-117).  factor < 1 keeps original i iff floor((i+1)f) >
    floor(i f); factor > 1 adds ceil(f)-1 jittered replicas per arrival
    (jitter drawn in [0, gap//2] from seed, gap = the local inter-arrival
    gap, at least 2 us) and keeps round(n f) - n of them, evenly spaced over
    the replica list; the result is sorted by (arrival, input, output)."""
    if factor <= 0:
        raise ValueError("rescale factor must be > 0")
    n = len(records)
    if n == 0 or factor == 1.0:
        return list(records)
    if factor < 1.0:
        return [r for i, r in enumerate(records)
                if math.floor((i + 1) * factor) > math.floor(i * factor)]
    rng = random.Random(seed)
    copies = math.ceil(factor) - 1
    extra: list[TraceRecord] = []
    for i, r in enumerate(records):
        if i + 1 < n:
            gap = records[i + 1].arrival_us - r.arrival_us
        else:
            gap = r.arrival_us - records[i - 1].arrival_us if i > 0 else 2
        gap = max(gap, 2)
        extra += [TraceRecord(r.arrival_us + rng.randrange(0, gap // 2 + 1), r.input_len,
                              r.output_len) for _ in range(copies)]
    want = int(round(n * factor)) - n
    if want < 0:
        raise ValueError("factor > 1 cannot shrink a trace")
    want = min(want, len(extra))
    picked = [extra[(j * len(extra)) // want] for j in range(want)]
    return sorted(list(records) + picked, key=lambda r: (r.arrival_us, r.input_len, r.output_len))
