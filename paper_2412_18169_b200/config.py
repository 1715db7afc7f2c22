"""Serving configuration (ref pkg/src/dropsim/config.py:1-240).

Same dataclasses, field names and defaults as the reference's SimConfig so
engine runs are comparable; B200 additions live in `DeviceConfig`.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

from .core import ModelSpec
from .costmodel import CostCoefficients
from .traceio import TRACE_PRESETS  # noqa: F401  (re-export, ref config.py:20-24)

POLICIES = ("kunserve", "recompute", "swap", "migrate")
FORMULATIONS = ("auto", "lookahead", "token_count")


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
    if not 0.0 < cfg.policy.restore_threshold <= 1.0:
        raise ConfigError("policy.restore_threshold", "must be in (0, 1]")
    if cfg.cluster.instances < 1:
        raise ConfigError("cluster.instances", "must be >= 1")
    if cfg.cluster.initial_group_size < 1 or cfg.cluster.instances % cfg.cluster.initial_group_size:
        raise ConfigError("cluster.initial_group_size", "must divide cluster.instances")
    if cfg.model.param_bytes >= cfg.cluster.hbm_bytes:
        raise ConfigError("cluster.hbm_bytes", "must exceed one parameter copy")
