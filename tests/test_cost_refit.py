"""the reference's cost model (alpha * attention units +
beta * tokens + gamma per microbatch, costmodel.py:50-69) refit on measured
stage times (ttft.fit_stage_samples), and the refit coefficients driving the
scheduler's planning (engine.py:389-397 microbatch formulation, 729-734
exchange chunk sizing).  Host-only: synthetic samples with known
coefficients stand in for the B200 stage timings."""

import random

import pytest

from paper_2412_18169_b200.costmodel import CostCoefficients, attention_units
from paper_2412_18169_b200.ttft import fit_stage_samples


def _samples(alpha, beta, gamma, L, n=60, noise=0.0, seed=1):
    """(tokens, units, n_decode, stage layers, us) as the engines record them:
    a stage of `layers` layers takes layers / L of the whole-model time."""
    rng = random.Random(seed)
    out = []
    for _ in range(n):
        c, p = rng.randrange(1, 2048), rng.randrange(0, 8192)
        units = attention_units(c, p)
        layers = rng.choice((L // 2, L))
        t = alpha * units + beta * c + gamma
        t *= 1.0 + noise * rng.uniform(-1, 1)
        out.append((c, units, rng.randrange(0, 64), layers, t * layers / L * 1e6))
    return out


def test_fit_recovers_known_coefficients():
    fit = fit_stage_samples(_samples(3e-9, 4e-6, 8e-3, 32), 32)
    assert fit["alpha"] == pytest.approx(3e-9, rel=1e-6)
    assert fit["beta"] == pytest.approx(4e-6, rel=1e-6)
    assert fit["gamma"] == pytest.approx(8e-3, rel=1e-6)
    assert fit["rms_s"] < 1e-12 and fit["samples"] == 60


def test_fit_with_noise_and_too_few_samples():
    fit = fit_stage_samples(_samples(2e-9, 1e-5, 5e-3, 32, n=400, noise=0.05), 32)
    assert fit["alpha"] == pytest.approx(2e-9, rel=0.1)
    assert fit["beta"] == pytest.approx(1e-5, rel=0.1)
    assert fit["gamma"] == pytest.approx(5e-3, rel=0.1)
    assert fit_stage_samples(_samples(1e-9, 1e-6, 1e-3, 32, n=2), 32) is None


def test_refit_coefficients_change_the_schedulers_plans():
    """The refit enters the reference's planning: the same trace planned with
    the reference defaults and with a refit (cheaper attention, costlier
    per-microbatch overhead) forms different rounds, and the exchange chunk
    size follows the refit's batch cost (engine.py:729-734)."""
    from paper_2412_18169_b200.config import SimConfig
    from paper_2412_18169_b200.engine import Engine
    from paper_2412_18169_b200.traceio import synth_burst
    trace = synth_burst(6.0, 2.0, 8.0, 1.5, 4.5, 400, 64, "lognormal", 0.6, 3)
    logs = {}
    chunk = {}
    for name, cost in (("default", None), ("refit", CostCoefficients(1e-9, 1e-5, 2e-2))):
        cfg = SimConfig()
        if cost is not None:
            cfg.cost = cost
        eng = Engine(cfg, trace)
        res = eng.run()
        logs[name] = [l for l in res.log_lines if " ROUND " in l]
        chunk[name] = eng._exchange_chunk_bytes()
    assert logs["default"] != logs["refit"]
    assert chunk["default"] != chunk["refit"]
