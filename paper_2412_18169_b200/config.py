"""Serving configuration (ref pkg/src/dropsim/config.py:1-240).

Same dataclasses, field names and defaults as the reference's SimConfig so
engine runs are comparable; B200 additions live in `DeviceConfig`.
"""

from __future__ import annotations

import configparser
from dataclasses import dataclass, field
from typing import Optional

from .core import ModelSpec
from .costmodel import CostCoefficients
from .traceio import TRACE_PRESETS  # noqa: F401  (re-export, ref config.py:20-24)

POLICIES = ("kunserve", "recompute", "swap", "migrate")
FORMULATIONS = ("auto", "lookahead", "token_count")
LENGTH_DISTS = ("fixed", "uniform", "lognormal")


class ConfigError(ValueError):
    def __init__(self, fieldname: str, message: str):
        super().__init__(f"{fieldname}: {message}")
        self.fieldname = fieldname


@dataclass
class ClusterConfig:
    instances: int = 4
    hbm_bytes: int = 24_000_000_000
    nic_bandwidth: int = 25_000_000_000
    host_bandwidth: int = 32_000_000_000
    link_base_latency_us: int = 50
    map_latency_us: int = 5000
    initial_group_size: int = 1


@dataclass
class PolicyConfig:
    kind: str = "kunserve"
    formulation: str = "auto"
    token_budget: int = 2048
    min_batch_tokens: int = 256
    restore_threshold: float = 0.5
    monitor_tick_us: int = 100_000
    slo_scales: tuple = (1.25, 2.0, 4.0, 6.0, 8.0, 10.0)
    autoscale_occupancy: float = 0.9
    autoscale_window_s: float = 10.0
    swap_headroom_tokens: int = 0


@dataclass
class TraceConfig:
    source: str = "synth"
    path: str = ""
    seed: int = 7
    duration_s: float = 60.0
    base_rps: float = 4.0
    burst_rps: float = 12.0
    burst_start_s: float = 20.0
    burst_end_s: float = 40.0
    length_dist: str = "lognormal"
    input_mean: int = 600
    output_mean: int = 60
    sigma: float = 0.6
    preset: str = ""
    rescale_factor: float = 1.0


@dataclass
class ReportConfig:
    window_s: float = 1.0
    figures: bool = True
    drain_s: float = 120.0


@dataclass
class DeviceConfig:
    """B200 binding: which GPU each instance lives on and the page geometry."""

    shape: Optional[object] = None        # core.ModelShape; None = model mode
    devices: tuple = (0,)                 # instance i -> devices[i % len(devices)]
    max_slots: int = 1024
    max_pages_per_seq: int = 1024


@dataclass
class SimConfig:
    model: ModelSpec = field(default_factory=lambda: ModelSpec(
        num_layers=8, bytes_per_layer=2_000_000_000, kv_bytes_per_token=200_000))
    cost: CostCoefficients = field(default_factory=lambda: CostCoefficients(
        alpha=6.6e-9, beta=2.8e-6, gamma=9.6e-3))
    cluster: ClusterConfig = field(default_factory=ClusterConfig)
    policy: PolicyConfig = field(default_factory=PolicyConfig)
    trace: TraceConfig = field(default_factory=TraceConfig)
    report: ReportConfig = field(default_factory=ReportConfig)
    device: DeviceConfig = field(default_factory=DeviceConfig)


def validate(cfg: SimConfig) -> None:
    if cfg.policy.kind not in POLICIES:
        raise ConfigError("policy.kind", f"unknown policy {cfg.policy.kind!r}, "
                                         f"expected one of {', '.join(POLICIES)}")
    if cfg.policy.formulation not in FORMULATIONS:
        raise ConfigError("policy.formulation",
                          f"unknown formulation {cfg.policy.formulation!r}")
    if cfg.trace.source not in ("synth", "file"):
        raise ConfigError("trace.source", f"unknown source {cfg.trace.source!r}")
    if cfg.trace.source == "file" and not cfg.trace.path:
        raise ConfigError("trace.path", "required when trace.source = file")
    if cfg.trace.length_dist not in LENGTH_DISTS:
        raise ConfigError("trace.length_dist", f"unknown distribution {cfg.trace.length_dist!r}")
    if cfg.trace.preset and cfg.trace.preset not in TRACE_PRESETS:
        raise ConfigError("trace.preset", f"unknown preset {cfg.trace.preset!r}, "
                                          f"expected one of {', '.join(sorted(TRACE_PRESETS))}")
    if not 0.0 < cfg.policy.restore_threshold <= 1.0:
        raise ConfigError("policy.restore_threshold", "must be in (0, 1]")
    if cfg.cluster.instances < 1:
        raise ConfigError("cluster.instances", "must be >= 1")
    if cfg.cluster.initial_group_size < 1 or cfg.cluster.instances % cfg.cluster.initial_group_size:
        raise ConfigError("cluster.initial_group_size", "must divide cluster.instances")
    if cfg.model.param_bytes >= cfg.cluster.hbm_bytes:
        raise ConfigError("cluster.hbm_bytes", "must exceed one parameter copy")


# ---------------------------------------------------------------- INI loader
def _num(conv):
    def parse(raw: str, name: str):
        try:
            return conv(float(raw)) if conv is int else conv(raw)
        except ValueError as exc:
            raise ConfigError(name, f"not a number: {raw!r}") from exc
    return parse


def _flag(raw: str, name: str) -> bool:
    v = raw.strip().lower()
    if v in ("1", "true", "yes", "on"):
        return True
    if v in ("0", "false", "no", "off"):
        return False
    raise ConfigError(name, f"not a boolean: {raw!r}")


def _text(raw: str, name: str) -> str:
    return raw.strip()


# (section, key) -> (dataclass path, converter); ints accept scientific
# notation (hbm_bytes = 24e9), like the reference (config.py:95-99)
_FIELDS = {
    "cluster": {k: _num(int) for k in ("instances", "hbm_bytes", "nic_bandwidth", "host_bandwidth",
                                       "link_base_latency_us", "map_latency_us",
                                       "initial_group_size")},
    "policy": {"kind": _text, "formulation": _text, "token_budget": _num(int),
               "min_batch_tokens": _num(int), "restore_threshold": _num(float),
               "monitor_tick_us": _num(int), "autoscale_occupancy": _num(float),
               "autoscale_window_s": _num(float)},
    "trace": {"source": _text, "path": _text, "seed": _num(int), "duration_s": _num(float),
              "base_rps": _num(float), "burst_rps": _num(float), "burst_start_s": _num(float),
              "burst_end_s": _num(float), "length_dist": _text, "input_mean": _num(int),
              "output_mean": _num(int), "sigma": _num(float), "preset": _text,
              "rescale_factor": _num(float)},
    "report": {"window_s": _num(float), "figures": _flag, "drain_s": _num(float)},
}


def load_config(path: str) -> SimConfig:
    """INI file -> SimConfig (ref config.py:150-240): sections [model]
    [cluster] [policy] [trace] [report], every key optional over the
    desk-scale defaults; [model] also carries the cost coefficients (alpha,
    beta, gamma, batch_discount); policy.slo_scales is a comma list; a trace
    preset overrides the length means.  Bad values raise ConfigError naming
    the field; the result is validated."""
    ini = configparser.ConfigParser(inline_comment_prefixes=("#", ";"))
    if not ini.read(path):
        raise ConfigError("config", f"cannot read {path}")
    cfg = SimConfig()

    def get(section, key, conv, default):
        if not ini.has_option(section, key):
            return default
        return conv(ini.get(section, key), f"{section}.{key}")

    m, c = cfg.model, cfg.cost
    cfg.model = ModelSpec(num_layers=get("model", "num_layers", _num(int), m.num_layers),
                          bytes_per_layer=get("model", "bytes_per_layer", _num(int),
                                              m.bytes_per_layer),
                          kv_bytes_per_token=get("model", "kv_bytes_per_token", _num(int),
                                                 m.kv_bytes_per_token),
                          hidden_bytes_per_token=get("model", "hidden_bytes_per_token",
                                                     _num(int), m.hidden_bytes_per_token))
    cfg.cost = CostCoefficients(alpha=get("model", "alpha", _num(float), c.alpha),
                                beta=get("model", "beta", _num(float), c.beta),
                                gamma=get("model", "gamma", _num(float), c.gamma),
                                batch_discount=get("model", "batch_discount", _num(float),
                                                   c.batch_discount))
    for section, keys in _FIELDS.items():
        obj = getattr(cfg, section)
        for key, conv in keys.items():
            setattr(obj, key, get(section, key, conv, getattr(obj, key)))
    if ini.has_option("policy", "slo_scales"):
        raw = ini.get("policy", "slo_scales")
        cfg.policy.slo_scales = tuple(_num(float)(x.strip(), "policy.slo_scales")
                                      for x in raw.split(",") if x.strip())
    t = cfg.trace
    if t.preset:
        if t.preset not in TRACE_PRESETS:
            raise ConfigError("trace.preset", f"unknown preset {t.preset!r}")
        t.input_mean, t.output_mean = TRACE_PRESETS[t.preset]
    validate(cfg)
    return cfg
