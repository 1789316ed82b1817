"""Drop-in for moesim.kernels: whole-layer policy replay on the B200 (K7).

`replay_policy` keeps the reference contract (kernels.py:60-67): (T, K) int64 activations
with ascending rows in, freshly allocated (resident_before, evicted) uint8 (T, E) masks
out.  The replay itself runs as one warp per layer in libmoeb200.so; numpy arrays are
staged through device memory.  There is no interpreted fallback: BACKEND names the device.
"""

from __future__ import annotations

import numpy as np

from .errors import ConfigError

P_LRU, P_LFU, P_LFU_AGED, P_OPT = 0, 1, 2, 3
BACKEND = "cuda-sm100a"


def replay_policy_layers(acts: np.ndarray, num_experts: int, capacity: int, policy: int,
                         decay_factor: float, decay_period: int):
    """Replay L independent layers at once: acts (L, T, K) -> masks (L, T, E)."""
    import torch

    from . import _native

    a = np.ascontiguousarray(acts, dtype=np.int64)
    if a.ndim != 3:
        raise ConfigError("acts must be (layers, tokens, top_k)")
    L, T, K = a.shape
    E = int(num_experts)
    if L == 0 or T == 0:
        z = np.zeros((L, T, E), np.uint8)
        return z, z.copy()
    lib = _native.lib()
    d_acts = torch.from_numpy(a).to("cuda")
    rb = torch.empty((L, T, E), dtype=torch.uint8, device="cuda")
    ev = torch.empty((L, T, E), dtype=torch.uint8, device="cuda")
    _native.check(lib.moe_replay_policy_layers(
        d_acts.data_ptr(), L, T, K, E, int(capacity), int(policy), float(decay_factor),
        int(decay_period), rb.data_ptr(), ev.data_ptr(), _native.stream_ptr()))
    return rb.cpu().numpy(), ev.cpu().numpy()


def replay_policy(acts, num_experts, capacity, policy, decay_factor, decay_period):
    """One layer: acts (T, K) -> (resident_before, evicted), each (T, E) uint8."""
    a = np.ascontiguousarray(acts, dtype=np.int64)
    if a.ndim != 2:
        raise ConfigError("acts must be (tokens, top_k)")
    rb, ev = replay_policy_layers(a[None], num_experts, capacity, policy, decay_factor,
                                  decay_period)
    return rb[0], ev[0]


def python_impl(kernel):
    """The reference exposes the uncompiled kernel here; the device kernel has none."""
    return kernel
