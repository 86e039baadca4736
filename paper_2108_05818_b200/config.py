"""Hot-path configuration: hardware and policy knobs of the chunk step.

Restates the frozen dataclasses of `/root/reference/pkg/src/chunkstar/config.py:116-193`
(``HardwareSpec``, ``PolicySpec``, ``SweepSpec``, ``ScenarioConfig``) with
the same defaults and validation.  The INI grammar and its file loader
(`config.py:1-45, 245-351`) are simulator UX and out of scope: they raise.
"""

from dataclasses import dataclass, field
from typing import Optional, Sequence, Tuple

from .baselines import CHUNK, DDP, L2L, STATIC_OFFLOAD
from .chunks import DEFAULT_CAPACITY_ELEMS
from .memory import EvictionStrategy
from .model import LadderRung, ModelSchema, default_ladder, ladder_rung

KNOWN_STRATEGIES = (CHUNK, STATIC_OFFLOAD, DDP, L2L)
_OS_PLACEMENTS = ("auto", "cpu", "gpu")


class ConfigError(ValueError):
    def __init__(self, message: str, section: Optional[str] = None,
                 key: Optional[str] = None, line: Optional[int] = None):
        self.section, self.key, self.line = section, key, line
        where = "" if section is None else "[%s]%s" % (section, " " + key if key else "")
        if line is not None:
            where = (where + " (line %d)" % line).strip()
        super().__init__("%s: %s" % (where, message) if where else message)


@dataclass(frozen=True)
class HardwareSpec:
    gpu_count: int = 8
    gpu_bytes: int = 32 * 10**9
    cpu_bytes: int = 240 * 10**9
    pcie_gbps: float = 12.0
    intra_gpu_gbps: float = 100.0

    def __post_init__(self) -> None:
        if self.gpu_count < 1:
            raise ConfigError("gpu_count must be >= 1", "hardware", "gpu_count")
        if min(self.gpu_bytes, self.cpu_bytes) <= 0:
            raise ConfigError("capacities must be > 0", "hardware")
        if min(self.pcie_gbps, self.intra_gpu_gbps) <= 0:
            raise ConfigError("bandwidths must be > 0", "hardware")


@dataclass(frozen=True)
class PolicySpec:
    capacity_elems: int = DEFAULT_CAPACITY_ELEMS
    eviction: EvictionStrategy = EvictionStrategy.LATEST_NEXT_USE
    limit_fraction: float = 0.8
    checkpointing: bool = False
    strategies: Tuple[str, ...] = (CHUNK, STATIC_OFFLOAD, DDP)
    os_placement: str = "auto"

    def __post_init__(self) -> None:
        if self.capacity_elems <= 0:
            raise ConfigError("capacity_elems must be > 0", "policy", "capacity_elems")
        if not 0.0 < self.limit_fraction <= 1.0:
            raise ConfigError("limit_fraction must be in (0, 1]", "policy",
                              "limit_fraction")
        if not self.strategies:
            raise ConfigError("strategies must be non-empty", "policy", "strategies")
        unknown = [s for s in self.strategies if s not in KNOWN_STRATEGIES]
        if unknown:
            raise ConfigError("unknown strategy %r (known: %s)"
                              % (unknown[0], ", ".join(KNOWN_STRATEGIES)),
                              "policy", "strategies")
        if self.os_placement not in _OS_PLACEMENTS:
            raise ConfigError("os_placement must be auto, cpu, or gpu", "policy",
                              "os_placement")


@dataclass(frozen=True)
class SweepSpec:
    batches: Tuple[int, ...] = (4, 8, 16, 32, 64)
    gpu_counts: Tuple[int, ...] = (1, 2, 4, 8)
    rungs: Tuple[str, ...] = ()

    def __post_init__(self) -> None:
        if not self.batches or min(self.batches) < 1:
            raise ConfigError("batches must be positive", "sweep", "batches")
        if not self.gpu_counts or min(self.gpu_counts) < 1:
            raise ConfigError("gpu_counts must be positive", "sweep", "gpu_counts")

    def ladder(self) -> Sequence[LadderRung]:
        if not self.rungs:
            return default_ladder()
        try:
            return [ladder_rung(r) for r in self.rungs]
        except KeyError as exc:
            raise ConfigError("unknown ladder rung %r" % exc.args[0], "sweep",
                              "rungs") from None


@dataclass(frozen=True)
class ScenarioConfig:
    model: ModelSchema = field(default_factory=lambda: ladder_rung("1B").schema(batch=8))
    hardware: HardwareSpec = field(default_factory=HardwareSpec)
    policy: PolicySpec = field(default_factory=PolicySpec)
    sweep: SweepSpec = field(default_factory=SweepSpec)
    seed: int = 0
    iterations: int = 3

    def __post_init__(self) -> None:
        if self.iterations < 2:
            raise ConfigError("iterations must be >= 2 (1 warm-up + measured)",
                              "run", "iterations")


def parse_config(text: str, source: str = "<config>") -> ScenarioConfig:
    raise NotImplementedError("the INI scenario grammar is simulator UX and out of "
                              "scope for the B200 chunk-step build")


def load_config(path: str) -> ScenarioConfig:
    return parse_config("", path)
