"""Cache policies with the reference's per-step object API (moesim/policies.py).

`policy_step` runs one warp-level policy step on the GPU (moe_policy_step, the same device
function the offline replay and the live engine use), so the object API, the replay and
the engine cannot drift apart.  The value-style CacheState is converted to the device
arrays (resident mask, last_touch, freq) and back on every call:

* recency (most recent first)  <->  last_touch: residents get strictly increasing touch
  stamps from the oldest end; experts activated in one step share a stamp and tie-break
  to the lower id, which is exactly the reference's "higher id counts as more recent"
  insertion order (policies.py:183-185).
* freq: dict of every expert ever seen <-> dense f64 array (keys = seen experts).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Iterable, Optional, Sequence

import numpy as np

from .errors import ConfigError

LRU, LFU, LFU_AGED, OPT = "lru", "lfu", "lfu-aged", "opt"
_NAMES = (LRU, LFU, LFU_AGED, OPT)
DEFAULT_DECAY_FACTOR = 0.5
DEFAULT_DECAY_PERIOD = 16
POLICY_CODE = {LRU: 0, LFU: 1, LFU_AGED: 2, OPT: 3}


@dataclass(frozen=True)
class PolicyKind:
    """Eviction policy; decay parameters exist iff the policy is lfu-aged."""

    name: str
    decay_factor: Optional[float] = None
    decay_period: Optional[int] = None

    def __post_init__(self):
        if self.name not in _NAMES:
            raise ConfigError(f"unknown policy {self.name!r}; expected one of {_NAMES}")
        aged = self.name == LFU_AGED
        has_params = self.decay_factor is not None or self.decay_period is not None
        if not aged and has_params:
            raise ConfigError(f"decay parameters are only valid for {LFU_AGED}")
        if aged:
            if self.decay_factor is None or self.decay_period is None:
                raise ConfigError("lfu-aged requires decay_factor and decay_period")
            if not (0.0 < self.decay_factor <= 1.0):
                raise ConfigError(f"decay_factor must be in (0, 1], got {self.decay_factor}")
            if self.decay_period < 1:
                raise ConfigError(f"decay_period must be >= 1, got {self.decay_period}")

    @classmethod
    def lru(cls) -> "PolicyKind":
        return cls(LRU)

    @classmethod
    def lfu(cls) -> "PolicyKind":
        return cls(LFU)

    @classmethod
    def lfu_aged(cls, decay_factor: float = DEFAULT_DECAY_FACTOR,
                 decay_period: int = DEFAULT_DECAY_PERIOD) -> "PolicyKind":
        return cls(LFU_AGED, decay_factor, decay_period)

    @classmethod
    def opt(cls) -> "PolicyKind":
        return cls(OPT)

    @classmethod
    def parse(cls, text: str) -> "PolicyKind":
        """'lru' | 'lfu' | 'opt' | 'lfu-aged' | 'lfu-aged:<factor>:<period>' (case-insensitive)."""
        spec = text.strip().lower()
        if spec in (LRU, LFU, OPT):
            return cls(spec)
        if spec == LFU_AGED:
            return cls.lfu_aged()
        head, sep, rest = spec.partition(":")
        if head == LFU_AGED and sep:
            parts = rest.split(":")
            if len(parts) != 2:
                raise ConfigError(f"expected lfu-aged:<factor>:<period>, got {text!r}")
            try:
                factor, period = float(parts[0]), int(parts[1])
            except ValueError as exc:
                raise ConfigError(f"bad lfu-aged parameters in {text!r}") from exc
            return cls.lfu_aged(factor, period)
        raise ConfigError(f"unknown policy {text!r}")

    @property
    def code(self) -> int:
        return POLICY_CODE[self.name]

    def device_params(self) -> tuple:
        """(code, decay_factor, decay_period) with the neutral values the replay expects."""
        return (self.code, 1.0 if self.decay_factor is None else float(self.decay_factor),
                1 if self.decay_period is None else int(self.decay_period))

    def __str__(self) -> str:
        if self.name == LFU_AGED:
            return f"{LFU_AGED}:{self.decay_factor:g}:{self.decay_period}"
        return self.name


@dataclass
class CacheState:
    """One layer's cache: residents, recency (most recent first), counts of every expert
    ever activated, and the number of steps taken."""

    capacity: int
    resident: frozenset = frozenset()
    recency: tuple = ()
    freq: dict = field(default_factory=dict)
    step: int = 0


@dataclass(frozen=True)
class StepOutcome:
    hits: frozenset
    misses: frozenset
    evicted: frozenset
    loaded: frozenset
    resident_before: frozenset
    resident_after: frozenset


def warm_state(kind: PolicyKind, capacity: int) -> CacheState:
    """Cold cache (policies.py:133-137)."""
    if capacity < 1:
        raise ConfigError(f"cache capacity must be >= 1, got {capacity}")
    return CacheState(capacity=capacity)


def policy_step(state: CacheState, kind: PolicyKind, activated: Iterable[int],
                future: Optional[Sequence[Iterable[int]]] = None):
    """Advance one layer's cache by one token on the GPU; returns (new_state, outcome).

    The input state is not mutated.  `future` (the remaining activation stream) is
    required for opt and rejected otherwise (policies.py:153-160)."""
    import torch

    from . import _native

    act = sorted(frozenset(int(e) for e in activated))
    if len(act) > state.capacity:
        raise ConfigError(
            f"activated set of size {len(act)} cannot fit in capacity {state.capacity}"
        )
    if kind.name == OPT and future is None:
        raise ConfigError("opt policy requires the remaining activation stream")
    if kind.name != OPT and future is not None:
        raise ConfigError(f"future stream is only valid for opt, not {kind.name}")

    fut_sets = [sorted(frozenset(int(e) for e in s)) for s in future] if future is not None else []
    universe = set(act) | set(state.resident) | set(state.freq) | {e for s in fut_sets for e in s}
    E = max(universe) + 1 if universe else 1
    E = max(E, 1)
    if E > 256:
        raise ConfigError(f"expert ids must be < 256 for the device policy step, got {E - 1}")

    resident = np.zeros(E, np.uint8)
    touch = np.full(E, -(1 << 39), np.int64)
    freq = np.zeros(E, np.float64)
    # oldest resident gets the smallest stamp; all stamps precede the current step
    n = len(state.recency)
    for pos, e in enumerate(state.recency):
        touch[e] = state.step - n + (n - 1 - pos) - 1
    for e in state.resident:
        resident[e] = 1
    for e, v in state.freq.items():
        freq[e] = v
    offsets = np.zeros(len(fut_sets) + 1, np.int64)
    for i, s in enumerate(fut_sets):
        offsets[i + 1] = offsets[i] + len(s)
    ids = np.array([e for s in fut_sets for e in s] or [0], np.int64)

    lib = _native.lib()
    dev = torch.device("cuda")
    t_res = torch.from_numpy(resident).to(dev)
    t_touch = torch.from_numpy(touch).to(dev)
    t_freq = torch.from_numpy(freq).to(dev)
    t_act = torch.tensor(act or [0], dtype=torch.int64, device=dev)
    t_ids = torch.from_numpy(ids).to(dev)
    t_off = torch.from_numpy(offsets).to(dev)
    t_rb = torch.zeros(E, dtype=torch.uint8, device=dev)
    t_ev = torch.zeros(E, dtype=torch.uint8, device=dev)
    code, df, dp = kind.device_params()
    opt = kind.name == OPT
    _native.check(lib.moe_policy_step(
        t_res.data_ptr(), t_touch.data_ptr(), t_freq.data_ptr(), int(state.step), E,
        int(state.capacity), code, df, dp, t_act.data_ptr(), len(act),
        t_ids.data_ptr() if opt else None, t_off.data_ptr() if opt else None,
        len(fut_sets), t_rb.data_ptr(), t_ev.data_ptr(), _native.stream_ptr()))
    res_after = t_res.cpu().numpy()
    touch_after = t_touch.cpu().numpy()
    freq_after = t_freq.cpu().numpy()
    rb = frozenset(np.flatnonzero(t_rb.cpu().numpy()).tolist())
    ev = frozenset(np.flatnonzero(t_ev.cpu().numpy()).tolist())

    after = frozenset(np.flatnonzero(res_after).tolist())
    recency = tuple(sorted(after, key=lambda e: (-int(touch_after[e]), -e)))
    new_freq = {e: float(freq_after[e]) for e in sorted(set(state.freq) | set(act))}
    acts = frozenset(act)
    misses = acts - rb
    new_state = CacheState(capacity=state.capacity, resident=after, recency=recency,
                           freq=new_freq, step=state.step + 1)
    outcome = StepOutcome(hits=acts & rb, misses=misses, evicted=ev, loaded=misses,
                          resident_before=rb, resident_after=after)
    return new_state, outcome
