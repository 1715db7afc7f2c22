"""P99 TTFT under an overload burst on the B200 (BASELINE metric 1).

Runs the reference's scheduler on real Llama-3-8B pools against a synthetic
4x ShareGPT-shaped burst (traceio.synth_burst, the reference's generator)
with KunServe's policy and the reference's three baselines, and reports
nearest-rank P99 TTFT / P50 TPOT from the event logs (metrics.collect, the
reference's metric code path).

clock="wall" (default): realtime.WallClockEngine -- arrivals on the wall
clock, stages and transfers executing concurrently on the GPU, every token
time a CUDA-event timestamp.  clock="sim": serving.DeviceEngine -- the same
device work executed stage by stage, its measured durations fed to the
reference's discrete-event clock, links on the link model (r1's mode).
"""

from __future__ import annotations

import time

from .core import SHAPES
from .metrics import bubble_ratio, collect, percentile
from .serving import DeviceEngine, device_config
from .traceio import synth_burst


def burst_trace(duration_s: float = 20.0, base_rps: float = 1.0, burst_factor: float = 4.0,
                input_mean: int = 1660, output_mean: int = 64, seed: int = 3):
    """4x burst in the middle third of the window, ShareGPT input lengths."""
    return synth_burst(duration_s, base_rps, base_rps * burst_factor, duration_s / 4,
                       duration_s * 3 / 4, input_mean, output_mean, "lognormal", 0.6, seed)


def run_policy(policy: str, trace, shape, kv_bytes: int, runtimes=None, cost=None,
               clock: str = "wall") -> dict:
    """cost: CostCoefficients for the scheduler's planning (lookahead
    microbatch formulation, exchange chunk sizing); stage times themselves
    are always measured."""
    cfg = device_config(shape, instances=2, kv_bytes=kv_bytes)
    cfg.policy.kind = policy
    if cost is not None:
        cfg.cost = cost
    cfg.report.drain_s = 60.0
    t0 = time.perf_counter()
    if clock == "wall":
        from .realtime import WallClockEngine
        eng = WallClockEngine(cfg, trace, runtimes=runtimes)
    else:
        eng = DeviceEngine(cfg, trace, runtimes=runtimes)
    t1 = time.perf_counter()
    res = eng.run()
    wall = time.perf_counter() - t0
    st = collect(res.log_lines)
    ttfts = st.ttfts()
    # a request that never got its first token inside the run counts as
    # infinitely late in the all-requests P99 (the served-only P99 is the
    # reference's metrics.collect view)
    unserved = len(trace) - len(ttfts)
    all_sorted = sorted(ttfts) + [float("inf")] * unserved
    kinds = {}
    for line in res.log_lines:
        k = line.split(" ", 2)[1]
        kinds[k] = kinds.get(k, 0) + 1
    p99_all = percentile(all_sorted, 99) if all_sorted else None
    out = {"policy": policy, "requests": len(trace), "finished": st.finished(),
           "served": len(ttfts), "unserved": unserved,
           "p99_ttft_all_s": None if p99_all in (None, float("inf")) else round(p99_all, 4),
           "p99_ttft_s": round(percentile(ttfts, 99), 4) if ttfts else None,
           "p50_ttft_s": round(percentile(ttfts, 50), 4) if ttfts else None,
           "p50_tpot_s": round(percentile(st.tpots(), 50), 5) if st.tpots() else None,
           "drops": res.drop_events, "evictions": res.evictions,
           "exchanges": kinds.get("EXCHANGE", 0), "restores": kinds.get("RESTORE_DONE", 0),
           "rounds": kinds.get("ROUND", 0), "stages_measured": len(eng.stage_samples),
           "bubble_ratio": round(bubble_ratio(res.log_lines), 4),
           "clock": clock, "wall_s": round(wall, 1), "setup_s": round(t1 - t0, 1)}
    if hasattr(eng, "host_prof"):
        out["host_s"] = {k: round(v, 2) for k, v in eng.host_prof.items()}
    fit = fit_stage_samples(eng.stage_samples, shape.num_layers)
    if fit:
        out["cost_fit"] = {k: fit[k] for k in ("alpha", "beta", "gamma")}
    for pool in eng.pools.values():
        pool.close()
    out["_log"] = res.log_lines
    return out, eng.stage_samples


def fit_stage_samples(samples, num_layers: int) -> dict:
    """The reference's cost model (alpha*units + beta*tokens + gamma seconds
    per microbatch, costmodel.py:50-69) least-squares fitted to the measured
    B200 stage times, each scaled to the full model by L / stage layers --
    the refit SURVEY.md 8f item 2 asks for."""
    import numpy as np
    if len(samples) < 3:
        return None
    m = np.array([[units, float(n), 1.0] for n, units, nd, layers, us in samples])
    y = np.array([us * num_layers / layers / 1e6 for n, units, nd, layers, us in samples])
    sol = np.maximum(np.linalg.lstsq(m, y, rcond=None)[0], 0.0)
    rms = float(np.sqrt(np.mean((m @ sol - y) ** 2)))
    return {"alpha": float(sol[0]), "beta": float(sol[1]), "gamma": float(sol[2]),
            "rms_s": rms, "samples": len(samples),
            "reference_defaults": {"alpha": 6.6e-9, "beta": 2.8e-6, "gamma": 9.6e-3}}


def measure(kv_gib: float = 1.0, shape_name: str = "llama3_8b",
            policies=("kunserve", "recompute", "swap", "migrate"), clock: str = "wall",
            keep_logs: bool = False, **trace_kw) -> dict:
    shape = SHAPES[shape_name]
    trace = burst_trace(**trace_kw)
    # warm-up: load every kernel / cuBLAS heuristic and walk one drop cycle
    # so the measured runs see steady-state stage times
    warm = burst_trace(duration_s=4.0, base_rps=4.0, input_mean=1660, output_mean=8, seed=11)
    w, _ = run_policy("kunserve", warm, shape, int(0.25 * (1 << 30)), clock=clock)
    # the scheduler plans with the cost model refit on the warm-up's measured
    # B200 stage times (engine.py:389-397, 729-734)
    fit = w.get("cost_fit")
    cost = None
    if fit:
        from .costmodel import CostCoefficients
        cost = CostCoefficients(alpha=fit["alpha"], beta=fit["beta"], gamma=fit["gamma"])
    res = {}
    samples_all = []
    for pol in policies:
        r, samples = run_policy(pol, trace, shape, int(kv_gib * (1 << 30)), cost=cost,
                                clock=clock)
        log = r.pop("_log")
        if keep_logs:
            r["_log"] = log
        res[pol] = r
        samples_all += samples
    k, r = res["kunserve"], res["recompute"]
    ratio = (r["p99_ttft_s"] / k["p99_ttft_s"]) if k["p99_ttft_s"] and r["p99_ttft_s"] else None
    # the reference's acceptance criterion 4 (tests/test_acceptance.py:146-163)
    # on hardware: P99 TTFT ratio vs EVERY baseline, P50 TPOT ratio vs the best
    base = [p for p in policies if p != "kunserve"]
    ttft_ratio = min((res[p]["p99_ttft_s"] or 0) / k["p99_ttft_s"] for p in base) \
        if k["p99_ttft_s"] else None
    tpot_ratio = k["p50_tpot_s"] / min(res[p]["p50_tpot_s"] for p in base) \
        if k["p50_tpot_s"] else None
    return {"value": k["p99_ttft_all_s"], "unit": "s", "clock": clock,
            "note": "p99_ttft_all_s counts a request that never got its first token inside "
                    "the run (trace + 60 s drain) as infinitely late (null when such requests "
                    "fall in the top 1%); p99_ttft_s is the reference's served-only view",
            "baseline_recompute_s": r["p99_ttft_all_s"],
            "baseline_recompute_served_only_s": r["p99_ttft_s"],
            "p99_ratio_recompute_over_kunserve_served_only": round(ratio, 2) if ratio else None,
            "criterion_4": {"p99_ttft_ratio_min_over_baselines": round(ttft_ratio, 2)
                            if ttft_ratio else None,
                            "p50_tpot_ratio_vs_best_baseline": round(tpot_ratio, 3)
                            if tpot_ratio else None,
                            "bounds": "ttft ratio >= 5, tpot ratio <= 1.35 "
                                      "(reference desk config; this is a different model/trace)"},
            "planning_cost": None if cost is None else
            {"alpha": cost.alpha, "beta": cost.beta, "gamma": cost.gamma,
             "source": "refit on the warm-up run's measured stage times"},
            **{p: res[p] for p in policies},
            "trace": {"requests": len(trace), "input_mean": trace_kw.get("input_mean", 1660),
                      "output_mean": trace_kw.get("output_mean", 64), "burst": "4x",
                      "kv_budget_gib_per_replica": kv_gib},
            "timing": ("wall clock: arrivals on the host clock, every stage and transfer "
                       "executing concurrently on the B200 (two replicas = two streams on one "
                       "GPU), FIRST_TOKEN / TOKEN / STAGE times from CUDA events"
                       if clock == "wall" else
                       "simulated clock: stage times measured on the B200 one at a time (CUDA "
                       "events around each stage's Llama-3-8B layers) and fed to the "
                       "reference's event clock; links modeled at NVLink-5 900 GB/s")}
