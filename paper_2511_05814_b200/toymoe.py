"""The reference's MoE model API (moesim/toymoe.py) backed by the B200 engine.

* ToyMoeModel draws the reference's seeded weights on the host, in the reference's order
  (gate_w, gate_b, mixing, w1, w2, then the token inputs; toymoe.py:63-83, 169).
* gate_select / speculate_next / forward_token run one fp64 device call each
  (moe_gate_topk_f64, moe_toy_forward_f64) for arbitrary user gates and models.
* run_model decodes the whole token stream through the offload engine: fp32 residual
  stream, toy tanh experts streamed from pinned host memory into an HBM cache, routing,
  speculation guess and cache policy all decided on the device.  The traces it returns
  are built from the engine's device step records.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .errors import ConfigError
from .traces import ActivationTrace, ModelShape, SpeculationTrace


@dataclass(frozen=True)
class ToyModelConfig:
    shape: ModelShape = ModelShape()
    hidden_dim: int = 16
    mixing_scale: float = 0.1
    skew: float = 1.0
    seed: int = 42
    tokens: int = 64

    def __post_init__(self):
        if self.hidden_dim < 1:
            raise ConfigError(f"hidden_dim must be >= 1, got {self.hidden_dim}")
        if self.mixing_scale < 0:
            raise ConfigError(f"mixing_scale must be >= 0, got {self.mixing_scale}")
        if self.tokens < 0:
            raise ConfigError(f"tokens must be >= 0, got {self.tokens}")


@dataclass(frozen=True)
class GatingNetwork:
    weights: np.ndarray                 # (hidden_dim, num_experts)
    bias: Optional[np.ndarray] = None   # (num_experts,)


@dataclass(frozen=True)
class HiddenState:
    values: np.ndarray  # (hidden_dim,)
    layer: int          # layer that produced it; -1 for a model input


class ToyMoeModel:
    """Seeded, immutable weights of every layer (reference draw order and scales)."""

    def __init__(self, config: ToyModelConfig, rng: np.random.Generator):
        L, E, d = config.shape.num_layers, config.shape.num_experts, config.hidden_dim
        inv = 1.0 / np.sqrt(d)
        self.config = config
        gw = rng.standard_normal((L, d, E)) * inv
        gb = rng.standard_normal((L, E)) * config.skew
        self.gates = tuple(GatingNetwork(weights=gw[l], bias=gb[l]) for l in range(L))
        self.mixing = rng.standard_normal((L, d, d))
        self.expert_w1 = rng.standard_normal((L, E, d, d)) * inv
        self.expert_w2 = rng.standard_normal((L, E, d, d)) * inv
        for arr in (gw, gb, self.mixing, self.expert_w1, self.expert_w2):
            arr.setflags(write=False)

    @classmethod
    def build(cls, config: ToyModelConfig):
        rng = np.random.default_rng(config.seed)
        return cls(config, rng), rng


def _cuda_f64(a) -> "torch.Tensor":
    import torch

    return torch.tensor(np.array(a, dtype=np.float64, copy=True), device="cuda")


def _gate_on_device(values: np.ndarray, gate: GatingNetwork, k: int):
    import torch

    from . import _native

    w = np.asarray(gate.weights, dtype=np.float64)
    v = np.asarray(values, dtype=np.float64)
    if v.shape[0] != w.shape[0]:
        raise ConfigError(
            f"hidden state of dim {v.shape[0]} does not match gate dim {w.shape[0]}")
    d, E = w.shape
    lib = _native.lib()
    order = torch.empty(max(k, 1), dtype=torch.int64, device="cuda")
    probs = torch.empty(E, dtype=torch.float64, device="cuda")
    # keep every device tensor referenced until the call returns
    t_v, t_w = _cuda_f64(v), _cuda_f64(w)
    bias = _cuda_f64(gate.bias) if gate.bias is not None else None
    _native.check(lib.moe_gate_topk_f64(
        t_v.data_ptr(), t_w.data_ptr(), bias.data_ptr() if bias is not None else None,
        d, E, int(k), order.data_ptr(), probs.data_ptr(), _native.stream_ptr()))
    return order.cpu().numpy()[:k], probs.cpu().numpy()


def gate_select(h: HiddenState, gate: GatingNetwork, k: int) -> list:
    """k most probable experts as (id, softmax prob) pairs, prob-desc, ties to the lower
    id, no renormalisation (toymoe.py:118-126)."""
    order, probs = _gate_on_device(h.values, gate, k)
    return [(int(e), float(probs[e])) for e in order]


def speculate_next(h_out_prev: HiddenState, gate_next: GatingNetwork, k: int) -> frozenset:
    """Next layer's guessed experts from the previous layer's output (toymoe.py:149-156)."""
    order, _ = _gate_on_device(h_out_prev.values, gate_next, k)
    return frozenset(int(e) for e in order)


def forward_token(model: ToyMoeModel, h_in: HiddenState, layer: int):
    """One layer for one token: mix, gate, selected experts (toymoe.py:129-146)."""
    import torch

    from . import _native

    cfg = model.config
    L, E, K = cfg.shape.num_layers, cfg.shape.num_experts, cfg.shape.top_k
    if not 0 <= layer < L:
        raise ConfigError(f"layer {layer} out of range [0, {L})")
    x = np.asarray(h_in.values, dtype=np.float64)
    d = cfg.hidden_dim
    if x.shape[0] != d:
        raise ConfigError(f"hidden state of dim {x.shape[0]} does not match gate dim {d}")
    gate = model.gates[layer]
    lib = _native.lib()
    out = torch.empty(d, dtype=torch.float64, device="cuda")
    sel = torch.empty(K, dtype=torch.int64, device="cuda")
    probs = torch.empty(E, dtype=torch.float64, device="cuda")
    bias = _cuda_f64(gate.bias) if gate.bias is not None else None
    t = [_cuda_f64(a) for a in (x, model.mixing[layer], gate.weights, model.expert_w1[layer],
                                model.expert_w2[layer])]
    _native.check(lib.moe_toy_forward_f64(
        t[0].data_ptr(), t[1].data_ptr(), t[2].data_ptr(),
        bias.data_ptr() if bias is not None else None, t[3].data_ptr(), t[4].data_ptr(),
        d, E, K, float(cfg.mixing_scale), out.data_ptr(), sel.data_ptr(), probs.data_ptr(),
        _native.stream_ptr()))
    return HiddenState(values=out.cpu().numpy(), layer=layer), frozenset(sel.cpu().tolist())


# fp32 margins below this fraction of the logit scale are re-decided in fp64 (run_model)
NEAR_TIE_REL = 1e-4


def _fp64_token(model: ToyMoeModel, x, K: int):
    """One token through every layer on the fp64 device path: (acts (L, K), guesses (L-1, K))
    sorted ascending -- the reference's run_model loop body (toymoe.py:175-185)."""
    L = model.config.shape.num_layers
    h = HiddenState(values=np.asarray(x, dtype=np.float64), layer=-1)
    acts = np.zeros((L, K), np.int64)
    guesses = np.zeros((max(L - 1, 0), K), np.int64)
    for l in range(L):
        if l >= 1:
            guesses[l - 1] = sorted(speculate_next(h, model.gates[l], K))
        h, sel = forward_token(model, h, l)
        acts[l] = sorted(sel)
    return acts, guesses


def run_model(config: ToyModelConfig, cache_size: Optional[int] = None, policy=None,
              return_engine_stats: bool = False):
    """Decode config.tokens seeded tokens through all layers on the GPU engine.

    Returns (ActivationTrace, SpeculationTrace) as toymoe.run_model does (toymoe.py:159-190).
    The engine always runs its per-layer HBM cache; by default it holds every expert
    (cache_size = E, LRU) so only compulsory misses are transferred.

    The engine computes in fp32, the reference in fp64: a selection (or guess) whose top-k
    logit margin is within fp32 reach of a tie could be ordered differently.  The engine
    records every step's margin and logit scale; each token with a margin below
    NEAR_TIE_REL x max(1, |logit|) anywhere is re-decoded on the fp64 device path
    (forward_token / speculate_next, the reference's arithmetic), so the returned traces
    are the fp64 ones wherever fp32 could not decide.
    """
    from .engine import OffloadEngine, EngineConfig
    from .policies import PolicyKind

    model, rng = ToyMoeModel.build(config)
    shape = config.shape
    T, L, K, E, d = config.tokens, shape.num_layers, shape.top_k, shape.num_experts, config.hidden_dim
    inputs = rng.standard_normal((T, d))
    if T == 0:
        empty = ActivationTrace(shape, np.zeros((0, L, K), np.int64))
        spec = SpeculationTrace(shape, np.zeros((0, max(L - 1, 0), K), np.int64),
                                np.zeros((0, max(L - 1, 0), K), np.int64))
        return (empty, spec, None) if return_engine_stats else (empty, spec)
    ecfg = EngineConfig(
        num_layers=L, num_experts=E, top_k=K, hidden_dim=d, expert_kind="toy_tanh",
        cache_size=E if cache_size is None else cache_size,
        policy=policy if policy is not None else PolicyKind.lru(),
        mixing_scale=config.mixing_scale, record_speculation=True, max_tokens=max(T, 1))
    with OffloadEngine(ecfg) as eng:
        eng.load_toy_model(model)
        eng.decode(inputs.astype(np.float32))
        rec = eng.records(0, T)
        gaps, ggaps = eng.record_gaps(0, T), eng.record_guess_gaps(0, T)
        zs = eng.record_logit_scales(0, T)
        stats = eng.stats()
    acts, guessed = rec["acts"], rec["guessed"]
    near = (gaps < NEAR_TIE_REL * np.maximum(1.0, zs[:, :, 0])).any(axis=1)
    if L >= 2:
        near |= (ggaps < NEAR_TIE_REL * np.maximum(1.0, zs[:, 1:, 1])).any(axis=1)
    for t in np.nonzero(near)[0]:
        acts[t], g = _fp64_token(model, inputs[t], K)
        if L >= 2:
            guessed[t] = g
    if L >= 2:
        actual = acts[:, 1:, :]
    else:
        guessed = actual = np.zeros((0, 0, K), np.int64)
    act_trace = ActivationTrace(shape, acts)
    spec_trace = SpeculationTrace(shape, guessed, np.ascontiguousarray(actual))
    if return_engine_stats:
        return act_trace, spec_trace, stats
    return act_trace, spec_trace
