"""OffloadEngine: the MoE-offloading decode engine behind the C ABI (include/moeb200.h).

Experts live in pinned host DRAM; each layer owns a fixed-size HBM expert cache managed
by a device-resident policy (LRU / LFU / LFU-aged, the reference's semantics); misses are
streamed over PCIe by the copy engine.  Host code here only builds configs, moves weights
in, and reads step records / statistics back.

Typical use (Mixtral-8x7B shape, synthetic weights):

    cfg = EngineConfig.mixtral_8x7b(cache_size=4, policy=PolicyKind.lfu())
    with OffloadEngine(cfg) as eng:
        eng.init_random(seed=42)
        h_out = eng.decode(h_in)            # (T, d) float32, host or CUDA
        log = eng.event_log(0, T)           # CacheEventLog (simulate.py format)
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native
from .errors import ConfigError
from .policies import OPT, PolicyKind

# Router bias spread of the synthetic Mixtral-shaped models (the reference's `skew` knob).
# With the RMS-normalised router, 0.25 reproduces the C=4 hit rates the survey / paper report
# for Mixtral (LRU ~0.55, LFU ~0.58); 1.0 makes routing bias-dominated (hit rate ~0.8).
DEFAULT_GATE_BIAS_STD = 0.25


@dataclass(frozen=True)
class EngineConfig:
    num_layers: int
    num_experts: int
    top_k: int
    hidden_dim: int
    ffn_dim: int = 0
    expert_kind: str = "swiglu"          # "swiglu" (bf16) | "toy_tanh" (f32)
    cache_size: int = 4
    policy: PolicyKind = field(default_factory=PolicyKind.lru)
    mixing_scale: float = 0.1
    prefetch: str = "off"                # "off" | "early" (gate_{l+1} on h'_l)
    renormalize: bool = False            # Mixtral routing (renormalised top-k); ref: False
    record_speculation: bool = True
    max_tokens: int = 4096
    chunk_bytes: int = 4 << 20
    prefetch_depth: int = 2
    device: int = 0
    rms_norm: bool = False               # Mixtral presets: True (RMSNorm before gate/experts)
    rms_eps: float = 1e-5
    transfer: str = "auto"               # "auto" | "copy_engine" | "sm" (see moeb200.h)
    store_layers: int = 0                # host store depth (0 = num_layers; else layers alias l % S)
    prefetch_buffers: int = 0            # staging buffers per layer with prefetch (0 = top_k)
    compress: int = 0                    # exponent-coded (lossless) demand / prefill transfers:
                                         # 0 raw, 1 raw + coded host stores, 2 coded store only

    @staticmethod
    def mixtral_8x7b(**kw) -> "EngineConfig":
        """Mixtral-8x7B shape (L=32, E=8, K=2, d=4096, f=14336), alpha = 0.1*sqrt(16/d)."""
        base = dict(num_layers=32, num_experts=8, top_k=2, hidden_dim=4096, ffn_dim=14336,
                    expert_kind="swiglu", mixing_scale=0.1 * math.sqrt(16 / 4096), rms_norm=True)
        base.update(kw)
        return EngineConfig(**base)

    @staticmethod
    def mixtral_8x22b(**kw) -> "EngineConfig":
        """Mixtral-8x22B shape (L=56, E=8, K=2, d=6144, f=16384)."""
        base = dict(num_layers=56, num_experts=8, top_k=2, hidden_dim=6144, ffn_dim=16384,
                    expert_kind="swiglu", mixing_scale=0.1 * math.sqrt(16 / 6144), rms_norm=True)
        base.update(kw)
        return EngineConfig(**base)

    @property
    def host_store_layers(self) -> int:
        return min(self.store_layers, self.num_layers) if self.store_layers > 0 else self.num_layers

    @property
    def expert_bytes(self) -> int:
        if self.expert_kind == "swiglu":
            return 3 * self.ffn_dim * self.hidden_dim * 2
        d8 = (self.hidden_dim + 7) // 8 * 8
        return 2 * d8 * d8 * 4

    def to_c(self) -> _native.EngineConfigC:
        if self.policy.name == OPT:
            raise ConfigError("the live engine cannot run opt (it needs the future stream)")
        kinds = {"toy_tanh": _native.EXPERT_TOY_TANH_F32, "swiglu": _native.EXPERT_SWIGLU_BF16}
        if self.expert_kind not in kinds:
            raise ConfigError(f"unknown expert kind {self.expert_kind!r}")
        modes = {"off": _native.PREFETCH_OFF, "early": _native.PREFETCH_EARLY}
        if self.prefetch not in modes:
            raise ConfigError(f"unknown prefetch mode {self.prefetch!r}")
        transfers = {"auto": _native.TRANSFER_AUTO, "copy_engine": _native.TRANSFER_COPY_ENGINE,
                     "sm": _native.TRANSFER_SM}
        if self.transfer not in transfers:
            raise ConfigError(f"unknown transfer mode {self.transfer!r}")
        code, df, dp = self.policy.device_params()
        return _native.EngineConfigC(
            num_layers=self.num_layers, num_experts=self.num_experts, top_k=self.top_k,
            hidden_dim=self.hidden_dim, ffn_dim=self.ffn_dim, expert_kind=kinds[self.expert_kind],
            cache_size=self.cache_size, policy=code, decay_factor=df, decay_period=dp,
            mixing_scale=self.mixing_scale, prefetch=modes[self.prefetch],
            renormalize=int(self.renormalize), record_speculation=int(self.record_speculation),
            max_tokens=self.max_tokens, chunk_bytes=self.chunk_bytes,
            prefetch_depth=self.prefetch_depth, device=self.device, rms_norm=int(self.rms_norm),
            rms_eps=self.rms_eps, transfer=transfers[self.transfer], store_layers=self.store_layers,
            prefetch_buffers=self.prefetch_buffers, compress=int(self.compress))


class OffloadEngine:
    """Owns one libmoeb200 engine (one per GPU, driven by one host thread)."""

    def __init__(self, config: EngineConfig, store=None):
        """store: optional caller-owned host expert store (replicas.SharedExpertStore) shared by
        the engines of one node; None allocates a private pinned store."""
        import torch

        self.config = config
        self._lib = _native.lib()
        self._dev = torch.device("cuda", config.device)
        self._store = store
        c = config.to_c()
        handle = ctypes.c_void_p()
        with torch.cuda.device(self._dev):
            if store is None:
                _native.check(self._lib.moe_engine_create(ctypes.byref(c), ctypes.byref(handle)))
            else:
                _native.check(self._lib.moe_engine_create_ex(
                    ctypes.byref(c), store.address, store.nbytes, ctypes.byref(handle)))
        self._h = handle
        self.tokens_done = 0
        self._inflight = []   # tensors enqueued work still reads / writes (cleared at sync)

    # -- lifetime --
    def close(self) -> None:
        if self._h:
            _native.check(self._lib.moe_engine_destroy(self._h))
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- weights --
    def init_random(self, seed: int = 42, gate_bias_std: float = DEFAULT_GATE_BIAS_STD,
                    init_experts: bool = True) -> None:
        """Synthetic Mixtral-shaped bf16 weights from the counter hash.
        init_experts=False: dense weights only (the shared store's owner wrote the experts)."""
        _native.check(self._lib.moe_engine_init_random(self._h, int(seed), float(gate_bias_std),
                                                       int(init_experts)))

    def coded_size(self) -> int:
        """Bytes of the exponent-coded store (compress=1; raw experts already written)."""
        n = ctypes.c_int64()
        _native.check(self._lib.moe_engine_coded_size(self._h, ctypes.byref(n)))
        return n.value

    def attach_coded(self, segment, build: bool) -> None:
        """Use a node-shared coded segment (replicas.SharedExpertStore): build=True encodes
        into it (the owner), build=False reads one the owner built."""
        _native.check(self._lib.moe_engine_attach_coded(self._h, segment.address, segment.nbytes,
                                                        int(build)))
        self._coded = segment

    def attach_peer_tier(self, blocks) -> None:
        """NVLink peer-HBM miss tier (include/moeb200.h moe_engine_attach_peer_tier):
        blocks maps (layer, expert) -> a CUDA uint8 tensor of expert_bytes holding that raw expert
        block, on a peer GPU (replicas.open_peer_tier) or on this one; None detaches.  Misses and
        prefetches of those experts are copied device to device instead of over PCIe; the
        decisions, traces and outputs do not change.  The tensors are kept alive here."""
        cfg = self.config
        if blocks is None:
            _native.check(self._lib.moe_engine_attach_peer_tier(self._h, None, 0))
            self._peer = None
            return
        n = cfg.num_layers * cfg.num_experts
        table = (ctypes.c_void_p * n)()
        for (l, e), t in blocks.items():
            if not (0 <= l < cfg.num_layers and 0 <= e < cfg.num_experts):
                raise ConfigError(f"peer block ({l}, {e}) out of range")
            if t.device.type != "cuda" or t.numel() * t.element_size() != cfg.expert_bytes:
                raise ConfigError("a peer block is a CUDA tensor of expert_bytes")
            table[l * cfg.num_experts + e] = t.data_ptr()
        _native.check(self._lib.moe_engine_attach_peer_tier(self._h, table, n))
        self._peer = dict(blocks)

    def load_toy_model(self, model) -> None:
        """Upload a ToyMoeModel's weights (reference layout, rounded to f32)."""
        cfg = self.config
        for l in range(cfg.num_layers):
            mix = np.ascontiguousarray(model.mixing[l], dtype=np.float32)
            gw = np.ascontiguousarray(model.gates[l].weights, dtype=np.float32)
            b = model.gates[l].bias
            gb = np.ascontiguousarray(b, dtype=np.float32) if b is not None else None
            _native.check(self._lib.moe_engine_set_dense_f32(
                self._h, l, mix.ctypes.data, gw.ctypes.data,
                gb.ctypes.data if gb is not None else None))
            for e in range(cfg.num_experts):
                w1 = np.ascontiguousarray(model.expert_w1[l, e], dtype=np.float32)
                w2 = np.ascontiguousarray(model.expert_w2[l, e], dtype=np.float32)
                _native.check(self._lib.moe_engine_set_toy_expert_f32(
                    self._h, l, e, w1.ctypes.data, w2.ctypes.data))

    def expert_block(self, layer: int, expert: int) -> np.ndarray:
        """Zero-copy uint8 view of one expert block in the pinned host store."""
        ptr, n = ctypes.c_void_p(), ctypes.c_int64()
        _native.check(self._lib.moe_engine_expert_host_ptr(self._h, layer, expert,
                                                           ctypes.byref(ptr), ctypes.byref(n)))
        buf = (ctypes.c_uint8 * n.value).from_address(ptr.value)
        return np.frombuffer(buf, dtype=np.uint8)

    def swiglu_weights(self, layer: int, expert: int):
        """(w1, w3, w2) of one SwiGLU expert as bf16-bit uint16 arrays ([f,d], [f,d], [d,f])."""
        cfg = self.config
        f, d = cfg.ffn_dim, cfg.hidden_dim
        blk = self.expert_block(layer, expert).view(np.uint16)
        return (blk[: f * d].reshape(f, d), blk[f * d: 2 * f * d].reshape(f, d),
                blk[2 * f * d:].reshape(d, f))

    def dense_weights(self, layer: int):
        """Device-layout dense weights: (mixing [d_out, d_in] as uint16 bf16 bits or f32,
        gate_w [E, d] f32, gate_b [E] f32)."""
        cfg = self.config
        D = cfg.hidden_dim if cfg.expert_kind == "swiglu" else (cfg.hidden_dim + 7) // 8 * 8
        mix = np.empty((D, D), np.uint16 if cfg.expert_kind == "swiglu" else np.float32)
        gw = np.empty((cfg.num_experts, D), np.float32)
        gb = np.empty(cfg.num_experts, np.float32)
        _native.check(self._lib.moe_engine_dense_host(self._h, layer, mix.ctypes.data,
                                                      gw.ctypes.data, gb.ctypes.data))
        return mix, gw, gb

    # -- decode --
    def reset(self) -> None:
        """Cold caches (policies.warm_state) for every layer."""
        _native.check(self._lib.moe_engine_reset(self._h))

    def _routing(self, routing, T):
        """(T, L, K) expert ids (ActivationTrace, numpy or torch) -> int32 CUDA tensor."""
        import torch

        if routing is None:
            return None
        if hasattr(routing, "activations"):
            routing = routing.activations
        cfg = self.config
        r = routing if torch.is_tensor(routing) else torch.from_numpy(np.array(routing, dtype=np.int32))
        if tuple(r.shape) != (T, cfg.num_layers, cfg.top_k):
            raise ConfigError(f"routing must be (T, L, K) = ({T}, {cfg.num_layers}, {cfg.top_k}), "
                              f"got {tuple(r.shape)}")
        return r.to(device=self._dev, dtype=torch.int32).contiguous()

    def decode_device(self, h_in, h_out=None, stream=None, routing=None):
        """Enqueue decode of h_in (T, d) float32 CUDA tensor; returns h_out without syncing.
        routing: optional (T, L, K) activation trace that replaces the gate's top-k
        (trace-driven mode: caches, transfers and FFN run as usual)."""
        import torch

        d = self.config.hidden_dim
        if h_in.dtype != torch.float32 or h_in.device.type != "cuda" or h_in.dim() != 2 or h_in.shape[1] != d:
            raise ConfigError(f"h_in must be a (T, {d}) float32 CUDA tensor")
        return self._enqueue(self._lib.moe_engine_decode_routed, h_in, h_out, stream, routing)

    def _stream(self, stream):
        """The stream work is enqueued on: the caller's, else torch's current stream of the
        ENGINE's device (not of whatever device the calling thread has current)."""
        import torch

        return stream if stream is not None else torch.cuda.current_stream(self._dev)

    def _enqueue(self, fn, h_in, h_out, stream, routing):
        """Launch fn on the engine's device and keep every tensor the enqueued kernels read or
        write alive until they ran: record_stream() for the caching allocator (the tensors may
        come from another stream) plus a per-call reference list cleared at sync()."""
        import torch

        h_in = h_in.contiguous()
        T = h_in.shape[0]
        with torch.cuda.device(self._dev):
            s = self._stream(stream)
            if h_out is None:
                h_out = torch.empty_like(h_in)
            r = self._routing(routing, T)
            _native.check(fn(self._h, h_in.data_ptr(), T, h_out.data_ptr(),
                             r.data_ptr() if r is not None else None, int(s.cuda_stream)))
            live = [x for x in (h_in, h_out, r) if x is not None]
            if s != torch.cuda.current_stream(self._dev):
                for x in live:
                    x.record_stream(s)
            self._inflight.extend(live)
        self.tokens_done += T
        return h_out

    def prefill_device(self, h_in, h_out=None, stream=None, routing=None):
        """Enqueue a batched prefill of h_in (T, d) float32 CUDA tensor (tensor-core GEMMs,
        one H2D load per needed expert per layer); returns h_out without syncing.  Step
        records / cache traces equal those of decoding the same T tokens."""
        import torch

        d = self.config.hidden_dim
        if h_in.dtype != torch.float32 or h_in.device.type != "cuda" or h_in.dim() != 2 or h_in.shape[1] != d:
            raise ConfigError(f"h_in must be a (T, {d}) float32 CUDA tensor")
        return self._enqueue(self._lib.moe_engine_prefill_routed, h_in, h_out, stream, routing)

    def _host_io(self, h_in):
        """Stage a host (T, d) array in reusable pinned buffers: returns (device input, pinned
        output view).  Pinned once and grown on demand, so a call's copies are plain DMA."""
        import torch

        a = np.ascontiguousarray(h_in, dtype=np.float32)
        T, d = a.shape
        if getattr(self, "_pin_rows", 0) < T:
            rows = max(T, 16)
            self._pin_in = torch.empty((rows, d), dtype=torch.float32, pin_memory=True)
            self._pin_out = torch.empty((rows, d), dtype=torch.float32, pin_memory=True)
            self._dev_in = torch.empty((rows, d), dtype=torch.float32, device=self._dev)
            self._dev_out = torch.empty((rows, d), dtype=torch.float32, device=self._dev)
            self._pin_rows = rows
        self._pin_in[:T].numpy()[:] = a
        x = self._dev_in[:T]
        with torch.cuda.device(self._dev):
            x.copy_(self._pin_in[:T], non_blocking=True)
        return x, self._dev_out[:T], self._pin_out[:T]

    def _run_host(self, fn, h_in, routing) -> np.ndarray:
        a = np.asarray(h_in)
        if a.ndim == 2 and a.shape[0] == 0:
            if a.shape[1] != self.config.hidden_dim:
                raise ConfigError(f"h_in must be (T, {self.config.hidden_dim})")
            return np.zeros((0, self.config.hidden_dim), np.float32)
        import torch

        x, y, out = self._host_io(h_in)
        fn(x, h_out=y, routing=routing)
        with torch.cuda.device(self._dev):
            out.copy_(y, non_blocking=True)
        self.sync()  # synchronises the device (and reports non-finite gates)
        return out.numpy().copy()

    def prefill(self, h_in, routing=None) -> np.ndarray:
        """Public prefill: host (T, d) array in, host (T, d) float32 out (copies included)."""
        return self._run_host(self.prefill_device, h_in, routing)

    def set_mode(self, policy: Optional[PolicyKind] = None, cache_size: Optional[int] = None,
                 prefetch: Optional[str] = None) -> None:
        """Switch policy / cache size (<= the allocated one) / prefetch, with cold caches."""
        import dataclasses

        cfg = dataclasses.replace(
            self.config, policy=policy or self.config.policy,
            cache_size=self.config.cache_size if cache_size is None else cache_size,
            prefetch=self.config.prefetch if prefetch is None else prefetch)
        c = cfg.to_c()
        _native.check(self._lib.moe_engine_set_mode(self._h, c.policy, c.decay_factor,
                                                    c.decay_period, c.cache_size, c.prefetch))
        self.config = cfg

    def profile(self, enable: bool = True) -> None:
        """Record CUDA events around every kernel class on the compute stream."""
        _native.check(self._lib.moe_engine_profile(self._h, int(enable)))

    def kernel_times(self) -> dict:
        k = _native.KernelTimesC()
        _native.check(self._lib.moe_engine_kernel_times(self._h, ctypes.byref(k)))
        return {name: getattr(k, name) for name, _ in _native.KernelTimesC._fields_}

    def sync(self) -> None:
        st = self._lib.moe_engine_sync(self._h)   # device-wide synchronize, then error check
        self._inflight.clear()
        _native.check(st)

    def decode(self, h_in, routing=None) -> np.ndarray:
        """Public decode: host (T, d) array in, host (T, d) float32 out (copies included).
        routing: optional (T, L, K) activation trace (trace-driven mode)."""
        return self._run_host(self.decode_device, h_in, routing)

    # -- records / stats --
    def records(self, t0: int, T: int) -> dict:
        cfg = self.config
        L, K, E = cfg.num_layers, cfg.top_k, cfg.num_experts
        acts = np.zeros((T, L, K), np.int64)
        guessed = np.zeros((T, max(L - 1, 0), K), np.int64)
        rb = np.zeros((T, L, E), np.uint8)
        ev = np.zeros((T, L, E), np.uint8)
        probs = np.zeros((T, L, K), np.float32)
        _native.check(self._lib.moe_engine_records(
            self._h, t0, T, acts.ctypes.data, guessed.ctypes.data if L > 1 else None,
            rb.ctypes.data, ev.ctypes.data, probs.ctypes.data))
        return {"acts": acts, "guessed": guessed, "resident_before": rb, "evicted": ev,
                "probs": probs}

    def record_gaps(self, t0: int, T: int) -> np.ndarray:
        """(T, L) f32 near-tie margins of the same steps: the K-th selected route logit minus
        the best unselected one (toymoe.py:99-115 ordering); +inf when K == E, NaN for
        trace-driven steps.  A margin below the fp tolerance is a selection an fp64
        evaluation could order differently (north star: ties within tolerance are stated)."""
        cfg = self.config
        gaps = np.zeros((T, cfg.num_layers), np.float32)
        _native.check(self._lib.moe_engine_record_gaps(self._h, t0, T, gaps.ctypes.data, None, None, None))
        return gaps

    def record_guess_gaps(self, t0: int, T: int) -> np.ndarray:
        """(T, L-1) margins of the reference-definition guesses (gate_l on the output of l-1,
        toymoe.py:178-180): NaN when speculation is not recorded."""
        cfg = self.config
        gg = np.full((T, max(cfg.num_layers - 1, 0)), np.nan, np.float32)
        if cfg.num_layers > 1:
            _native.check(self._lib.moe_engine_record_gaps(self._h, t0, T, None, gg.ctypes.data, None, None))
        return gg

    def record_logit_scales(self, t0: int, T: int) -> np.ndarray:
        """(T, L, 2) largest |logit| of the route and of the guess per step (0 without a
        guess): fp32 logit error grows with this scale, so near-tie tests are relative to it."""
        cfg = self.config
        zs = np.zeros((T, cfg.num_layers, 2), np.float32)
        _native.check(self._lib.moe_engine_record_gaps(self._h, t0, T, None, None, zs.ctypes.data, None))
        return zs

    def record_early_guesses(self, t0: int, T: int) -> np.ndarray:
        """(T, L-1, K) early guesses: at step (t, l) the top-k of gate_{l+1} on h'_l (ascending),
        the guess the speculative prefetch of layer l+1 acted on; -1 with prefetch off."""
        cfg = self.config
        L, K = cfg.num_layers, cfg.top_k
        early = np.full((T, max(L - 1, 0), K), -1, np.int64)
        if L > 1:
            _native.check(self._lib.moe_engine_record_gaps(self._h, t0, T, None, None, None, early.ctypes.data))
        return early

    def event_log(self, t0: int, T: int, warmup_tokens: int = 0):
        """The engine's own cache decisions as a CacheEventLog (simulate.py format)."""
        from .simulate import CacheEventLog, SimConfig
        from .traces import ModelShape

        cfg = self.config
        rec = self.records(t0, T)
        layers = tuple(range(cfg.num_layers))
        return CacheEventLog(
            config=SimConfig(policy=cfg.policy, cache_size=cfg.cache_size,
                             warmup_tokens=warmup_tokens),
            shape=ModelShape(cfg.num_layers, cfg.num_experts, cfg.top_k), layers=layers,
            activated={l: np.ascontiguousarray(rec["acts"][:, l, :]) for l in layers},
            resident_before={l: np.ascontiguousarray(rec["resident_before"][:, l, :]) for l in layers},
            evicted={l: np.ascontiguousarray(rec["evicted"][:, l, :]) for l in layers},
            num_tokens=T)

    def stats(self) -> dict:
        s = _native.StatsC()
        _native.check(self._lib.moe_engine_stats(self._h, ctypes.byref(s)))
        return {name: getattr(s, name) for name, _ in _native.StatsC._fields_}


def hash_weights(seed: int, tensor_id: int, std: float, n: int, dtype: str = "bf16"):
    """Device tensor of n synthetic values (counter hash; bf16 returned as uint16 bits)."""
    import torch

    lib = _native.lib()
    if dtype == "bf16":
        out = torch.empty(n, dtype=torch.int16, device="cuda")
        _native.check(lib.moe_hash_weights_bf16(seed, tensor_id, std, n, out.data_ptr(),
                                                _native.stream_ptr()))
    else:
        out = torch.empty(n, dtype=torch.float32, device="cuda")
        _native.check(lib.moe_hash_weights_f32(seed, tensor_id, std, n, out.data_ptr(),
                                               _native.stream_ptr()))
    return out


def tensor_id(kind: int, layer: int = 0, expert: int = 0, matrix: int = 0) -> int:
    """kind: 1 mixing, 2 gate_w, 3 gate_b, 4 expert (matrix 1 w1, 2 w3, 3 w2), 5 inputs."""
    return (kind << 40) | (layer << 16) | (expert << 4) | matrix
