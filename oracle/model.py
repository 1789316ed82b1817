"""ORACLE (test infrastructure only): numpy fp64 restatement of the reference model path.

toy_*       restate moesim/toymoe.py line by line in numpy fp64 (the reference dtype):
              draw order gate_w, gate_b, mixing, w1, w2, inputs ....... toymoe.py:73-83, 169
              _softmax ................................................ toymoe.py:93-96
              _gate_topk: z = h@W (+b), finite check, lexsort order ... toymoe.py:99-115
              _forward: h = x + a*(x@M); out = h + sum p_e tanh(h@W1)@W2 toymoe.py:138-146
              run_model loop with the guess before each layer >= 1 .... toymoe.py:175-185
MixtralRef  the same _forward with the north-star SwiGLU expert, on the engine's synthetic
            weights (counter hash, bf16-rounded, widened to fp64: "identical inputs").
            layout="ref" keeps every matrix as (d_in, d_out) and computes `h @ W` like the
            reference; layout="torch" is the tuned nn.Linear-layout fp32 variant (ii).
"""

from __future__ import annotations

import math

import numpy as np

from .native import hash_fill, hash_fill_t, replay_policy


def softmax(z: np.ndarray) -> np.ndarray:
    z = z - z.max()
    ez = np.exp(z)
    return ez / ez.sum()


def gate_topk(h: np.ndarray, W: np.ndarray, b, k: int):
    z = h @ W
    if b is not None:
        z = z + b
    if not np.isfinite(z).all():
        raise FloatingPointError("gate logits are not finite")
    E = z.shape[0]
    order = np.lexsort((np.arange(E), -z))[:k]
    return order, softmax(z), z


def toy_weights(L: int, E: int, d: int, skew: float, seed: int, tokens: int):
    rng = np.random.default_rng(seed)
    s = 1.0 / np.sqrt(d)
    w = {
        "gate_w": rng.standard_normal((L, d, E)) * s,
        "gate_b": rng.standard_normal((L, E)) * skew,
        "mixing": rng.standard_normal((L, d, d)),
        "w1": rng.standard_normal((L, E, d, d)) * s,
        "w2": rng.standard_normal((L, E, d, d)) * s,
    }
    w["inputs"] = rng.standard_normal((tokens, d))
    return w


def toy_forward(w: dict, x: np.ndarray, l: int, alpha: float, k: int):
    h = x + alpha * (x @ w["mixing"][l])
    sel, probs, z = gate_topk(h, w["gate_w"][l], w["gate_b"][l], k)
    out = h.copy()
    for e in sel:
        out = out + probs[e] * (np.tanh(h @ w["w1"][l, e]) @ w["w2"][l, e])
    return out, sel, probs, z


def toy_run_model(L, E, K, d, alpha, skew, seed, T, weights=None, return_gaps=False):
    """acts (T, L, K), guessed/actual (T, L-1, K); weights override for the
    identical-inputs protocol.  With return_gaps, also the k-th/(k+1)-th logit gap per
    (t, l) so near-ties can be reported."""
    w = weights if weights is not None else toy_weights(L, E, d, skew, seed, T)
    acts = np.zeros((T, L, K), np.int64)
    guessed = np.zeros((T, max(L - 1, 0), K), np.int64)
    gaps = np.full((T, L), np.inf)
    for t in range(T):
        h = w["inputs"][t]
        for l in range(L):
            if l >= 1:
                g, _, _ = gate_topk(h, w["gate_w"][l], w["gate_b"][l], K)
                guessed[t, l - 1] = np.sort(g)
            h, sel, _, z = toy_forward(w, h, l, alpha, K)
            acts[t, l] = np.sort(sel)
            if K < E:
                zs = np.sort(z)[::-1]
                gaps[t, l] = zs[K - 1] - zs[K]
    actual = acts[:, 1:, :].copy() if L >= 2 else np.zeros((T, 0, K), np.int64)
    if L < 2 or T == 0:
        guessed, actual = guessed[:0], actual[:0]
    if return_gaps:
        return acts, guessed, actual, gaps
    return acts, guessed, actual


def _tid(kind: int, layer: int = 0, expert: int = 0, matrix: int = 0) -> int:
    return (kind << 40) | (layer << 16) | (expert << 4) | matrix


def _std(n: int) -> float:
    return float(np.float32(1.0 / math.sqrt(n)))


class MixtralRef:
    """CPU decode of the Mixtral-shaped engine path (SwiGLU experts) on identical inputs.
    With rms_norm, h' is RMS-normalised (unit scale, as Mixtral's pre-MoE norm) before the
    gate and the experts; the residual adds to the un-normalised h'.

    Weights are regenerated from the counter hash exactly as the engine's init_random:
    mixing [d_out, d_in] bf16 std 1; gate_w [E, d] f32 std 1/sqrt(d); gate_b [E] f32 std
    gate_bias_std (default 0.25, engine.DEFAULT_GATE_BIAS_STD);
    w1, w3 [f, d] bf16 std 1/sqrt(d); w2 [d, f] bf16 std 1/sqrt(f).
    """

    def __init__(self, L, E, K, d, f, alpha, seed=42, layout="ref", threads=None,
                 layers=None, renormalize=False, rms_norm=False, rms_eps=1e-5,
                 gate_bias_std=0.25, store_layers=0):
        self.L, self.E, self.K, self.d, self.f = L, E, K, d, f
        self.alpha, self.seed, self.layout, self.threads = alpha, seed, layout, threads
        self.renormalize = renormalize
        self.rms_norm, self.rms_eps = rms_norm, rms_eps
        self.gate_bias_std = gate_bias_std
        self.store_layers = store_layers if store_layers > 0 else L  # engine store aliasing
        self.dtype = np.float64 if layout == "ref" else np.float32
        self.layers = list(range(L)) if layers is None else list(layers)
        self._dense = {}
        self._experts = {}

    def _matrix(self, tid, std, rows, cols):
        """A bf16 synthetic [rows, cols] (device layout) matrix, widened; in the reference
        layout the transpose (cols, rows) so that `h @ W` is the device's `W_dev h`."""
        if self.layout == "ref":
            return hash_fill_t(self.seed, tid, std, rows, cols, "f64", self.threads)
        return hash_fill(self.seed, tid, std, rows * cols, "f32w", self.threads).reshape(rows, cols)

    def dense(self, l):
        if l not in self._dense:
            d, E = self.d, self.E
            M = self._matrix(_tid(1, l), 1.0, d, d)
            gw = hash_fill(self.seed, _tid(2, l), _std(d), E * d, "f32", self.threads)
            gb = hash_fill(self.seed, _tid(3, l), self.gate_bias_std, E, "f32", self.threads)
            gw = gw.astype(self.dtype).reshape(E, d)
            if self.layout == "ref":   # x @ W_ref with W_ref = Wg_dev^T
                gw = np.ascontiguousarray(gw.T)
            self._dense[l] = (M, gw, gb.astype(self.dtype))
        return self._dense[l]

    def expert(self, l, e):
        l = l % self.store_layers  # layer l's experts live in store layer l % S
        if (l, e) not in self._experts:
            d, f = self.d, self.f
            self._experts[(l, e)] = (self._matrix(_tid(4, l, e, 1), _std(d), f, d),
                                     self._matrix(_tid(4, l, e, 2), _std(d), f, d),
                                     self._matrix(_tid(4, l, e, 3), _std(f), d, f))
        return self._experts[(l, e)]

    def materialize(self, layers=None):
        for l in (self.layers if layers is None else layers):
            self.dense(l)
            for e in range(self.E):
                self.expert(l, e)

    def forward(self, x: np.ndarray, l: int):
        """One layer: returns (h_out, selected prob-desc, probs over E, logits)."""
        M, gw, gb = self.dense(l)
        x = x.astype(self.dtype)
        if self.layout == "ref":
            h = x + self.alpha * (x @ M)
            hn = self._norm(h)
            z = hn @ gw + gb
        else:
            h = x + np.float32(self.alpha) * (M @ x)
            hn = self._norm(h)
            z = gw @ hn + gb
        if not np.isfinite(z).all():
            raise FloatingPointError("gate logits are not finite")
        sel = np.lexsort((np.arange(self.E), -z))[: self.K]
        p = softmax(z)
        weights = p[sel] / p[sel].sum() if self.renormalize else p[sel]
        out = h.copy()
        for e, pe in zip(sel, weights):
            w1, w3, w2 = self.expert(l, e)
            if self.layout == "ref":
                a1, a3 = hn @ w1, hn @ w3
                act = a1 / (1.0 + np.exp(-a1)) * a3
                out = out + pe * (act @ w2)
            else:
                a1, a3 = w1 @ hn, w3 @ hn
                act = a1 / (np.float32(1.0) + np.exp(-a1)) * a3
                out = out + pe * (w2 @ act)
        return out, sel, p, z

    def _norm(self, h: np.ndarray) -> np.ndarray:
        """Mixtral's RMSNorm with unit scale (engine rms_norm=1); identity otherwise."""
        if not self.rms_norm:
            return h
        return h / np.sqrt(np.mean(h * h) + self.rms_eps)

    def guess(self, h: np.ndarray, l: int):
        """Reference-definition guess for layer l from the previous layer's output."""
        _, gw, gb = self.dense(l)
        hn = self._norm(h.astype(self.dtype))
        z = hn @ gw + gb if self.layout == "ref" else gw @ hn + gb
        return np.sort(np.lexsort((np.arange(self.E), -z))[: self.K])

    @staticmethod
    def inputs(seed: int, T: int, d: int, t0: int = 0) -> np.ndarray:
        """Token inputs: f32 std 1, tensor kind 5, one tensor per token."""
        return np.stack([hash_fill(seed, _tid(5, t0 + t), 1.0, d, "f32") for t in range(T)])

    def decode(self, X: np.ndarray):
        """Run tokens through self.layers; returns (outputs, acts (T, n_layers, K))."""
        T = X.shape[0]
        acts = np.zeros((T, len(self.layers), self.K), np.int64)
        outs = []
        for t in range(T):
            h = X[t].astype(self.dtype)
            for i, l in enumerate(self.layers):
                h, sel, _, _ = self.forward(h, l)
                acts[t, i] = np.sort(sel)
            outs.append(h)
        return np.stack(outs) if outs else np.zeros((0, self.d)), acts


def decode_layerwise(ref: "MixtralRef", X: np.ndarray, forced=None, tol: float = 1e-3,
                     keep_weights: bool = False):
    """MixtralRef.decode reordered layer-major, for full-depth parity at Mixtral scale.

    Tokens are independent inputs (the reference model has no attention: run_model runs each
    token through all layers on its own, toymoe.py:175-185), so evaluating layer l for all T
    tokens before layer l+1 gives exactly MixtralRef.decode's arithmetic per token, while only
    one layer's fp64 experts are alive at a time (8x7B: 11.3 GB instead of 361 GB); each
    expert's token rows go through it as one fp64 GEMM.

    forced: optional (T, L, K) selections of the system under test (ascending ids).  Where the
    oracle's own k-th/(k+1)-th logit gap is below `tol` and its selection differs from the
    forced one, the oracle adopts the forced set for that (t, l) -- a teacher-forced near-tie --
    so a tie resolved the other way does not make the rest of the token incomparable.  A
    disagreement with a gap >= tol is never forced: it stays in the returned acts and the
    caller's equality check fails on it.

    Returns dict: outs (T, d) fp64, acts (T, L, K) sorted, gaps (T, L) route margins,
    guessed (T, L-1, K) sorted reference-definition guesses (toymoe.py:178-180), guess_gaps
    (T, L-1), forced_ties = [(t, l, gap)] where the forced set was adopted."""
    assert ref.layout == "ref"
    T, d = X.shape
    L, E, K = len(ref.layers), ref.E, ref.K
    h = X.astype(np.float64)
    acts = np.zeros((T, L, K), np.int64)
    gaps = np.full((T, L), np.inf)
    guessed = np.zeros((T, max(L - 1, 0), K), np.int64)
    guess_gaps = np.full((T, max(L - 1, 0)), np.inf)
    forced_ties = []
    ar = np.arange(E)
    for i, l in enumerate(ref.layers):
        M, gw, gb = ref.dense(l)
        if i >= 1:   # the reference guess for layer l is gate_l on the previous output
            zg = np.stack([ref._norm(r) for r in h]) @ gw + gb
            for t in range(T):
                order = np.lexsort((ar, -zg[t]))
                guessed[t, i - 1] = np.sort(order[:K])
                if K < E:
                    guess_gaps[t, i - 1] = zg[t, order[K - 1]] - zg[t, order[K]]
        hm = h + ref.alpha * (h @ M)
        hn = np.stack([ref._norm(r) for r in hm])
        z = hn @ gw + gb
        if not np.isfinite(z).all():
            raise FloatingPointError("gate logits are not finite")
        sel = np.zeros((T, K), np.int64)
        for t in range(T):
            order = np.lexsort((ar, -z[t]))
            s = order[:K]
            if K < E:
                gaps[t, i] = z[t, order[K - 1]] - z[t, order[K]]
            if forced is not None and gaps[t, i] < tol:
                f = np.asarray(forced[t, i], np.int64)
                if not np.array_equal(np.sort(s), np.sort(f)):
                    s = f[np.lexsort((f, -z[t, f]))]   # the forced set, in logit order
                    forced_ties.append((t, l, float(gaps[t, i])))
            sel[t] = s
        p = np.stack([softmax(zt) for zt in z])
        w = np.take_along_axis(p, sel, 1)
        if ref.renormalize:
            w = w / w.sum(1, keepdims=True)
        out = hm.copy()
        for e in range(E):
            rows, slots = np.nonzero(sel == e)
            if rows.size == 0:
                continue
            w1, w3, w2 = ref.expert(l, e)
            a1, a3 = hn[rows] @ w1, hn[rows] @ w3
            y = (a1 / (1.0 + np.exp(-a1)) * a3) @ w2
            out[rows] += w[rows, slots][:, None] * y
        acts[:, i] = np.sort(sel, axis=1)
        h = out
        if not keep_weights:   # one layer's fp64 weights alive at a time
            ref._dense.pop(l, None)
            for e in range(E):
                ref._experts.pop((l % ref.store_layers, e), None)
    return {"outs": h, "acts": acts, "gaps": gaps, "guessed": guessed, "guess_gaps": guess_gaps,
            "forced_ties": forced_ties}


def bf16_round(a) -> np.ndarray:
    """Round to bf16 (nearest even) through f32, returned widened to f32: the engine's
    __floats2bfloat162_rn on an f32 value."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    r = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000)
    return r.astype(np.uint32).view(np.float32)


def mixtral_prefill(ref: "MixtralRef", X: np.ndarray, return_gaps: bool = False):
    """Batched prefill restated (moe_engine_prefill): every layer over all T tokens, with the
    engine's operand roundings -- the mixing GEMM reads bf16(x), the experts read
    bf16(h' / rms(h')) and the down projection bf16(silu(w1 x) * w3 x) -- and everything else
    in fp64.  Routing / guesses as MixtralRef.forward (toymoe.py:99-115, 178-180).
    Returns (outputs (T, d), acts (T, L, K) sorted, guessed (T, L-1, K) sorted[, gaps (T, L)]),
    gaps = k-th minus (k+1)-th logit, for near-tie accounting."""
    assert ref.layout == "ref"
    T, d = X.shape
    L, E, K = len(ref.layers), ref.E, ref.K
    x = X.astype(np.float64)
    acts = np.zeros((T, L, K), np.int64)
    guessed = np.zeros((T, max(L - 1, 0), K), np.int64)
    gaps = np.zeros((T, L))
    for i, l in enumerate(ref.layers):
        M, gw, gb = ref.dense(l)
        if i >= 1:
            xn = np.stack([ref._norm(r) for r in x])
            zg = xn @ gw + gb
            guessed[:, i - 1] = np.sort(np.stack([np.lexsort((np.arange(E), -z))[:K] for z in zg]), axis=1)
        h = x + ref.alpha * (bf16_round(x).astype(np.float64) @ M)
        hn = np.stack([ref._norm(r) for r in h])
        z = hn @ gw + gb
        if not np.isfinite(z).all():
            raise FloatingPointError("gate logits are not finite")
        sel = np.stack([np.lexsort((np.arange(E), -zt))[:K] for zt in z])
        zs = -np.sort(-z, axis=1)
        gaps[:, i] = zs[:, K - 1] - zs[:, K] if K < E else np.inf
        p = np.stack([softmax(zt) for zt in z])
        w = np.take_along_axis(p, sel, 1)
        if ref.renormalize:
            w = w / w.sum(1, keepdims=True)
        an = bf16_round(hn).astype(np.float64)
        y = np.zeros((T, K, d))
        for e in range(E):
            rows, slots = np.nonzero(sel == e)
            if rows.size == 0:
                continue
            w1, w3, w2 = ref.expert(l, e)
            a1, a3 = an[rows] @ w1, an[rows] @ w3
            act = bf16_round(a1 / (1.0 + np.exp(-a1)) * a3).astype(np.float64)
            y[rows, slots] = act @ w2
        out = h.copy()
        for j in range(K):
            out = out + w[:, j:j + 1] * y[:, j]
        acts[:, i] = np.sort(sel, axis=1)
        x = out
    if return_gaps:
        return x, acts, guessed, gaps
    return x, acts, guessed


def mixtral_prefill_fp32(ref: "MixtralRef", X: np.ndarray):
    """The batched prefill as a tuned fp32 CPU port (the cpu_baseline_fp32 leg of bench.py,
    BASELINE.md variant (ii)): row-major (nn.Linear-layout) fp32 weights, BLAS sgemm over the
    token rows of each expert, same routing.  Returns outputs (T, d)."""
    assert ref.layout != "ref"
    T, d = X.shape
    E, K = ref.E, ref.K
    x = X.astype(np.float32)
    one = np.float32(1.0)
    for l in ref.layers:
        M, gw, gb = ref.dense(l)
        h = x + np.float32(ref.alpha) * (x @ M.T)
        hn = h / np.sqrt(np.mean(h * h, axis=1, keepdims=True) + np.float32(ref.rms_eps)) if ref.rms_norm else h
        z = hn @ gw.T + gb
        if not np.isfinite(z).all():
            raise FloatingPointError("gate logits are not finite")
        sel = np.argsort(-z, axis=1, kind="stable")[:, :K]
        zmax = z.max(axis=1, keepdims=True)
        p = np.exp(z - zmax)
        p /= p.sum(axis=1, keepdims=True)
        w = np.take_along_axis(p, sel, 1)
        out = h.copy()
        for e in range(E):
            rows, slots = np.nonzero(sel == e)
            if rows.size == 0:
                continue
            w1, w3, w2 = ref.expert(l, e)
            a1, a3 = hn[rows] @ w1.T, hn[rows] @ w3.T
            act = a1 / (one + np.exp(-a1)) * a3
            out[rows] += w[rows, slots][:, None] * (act @ w2.T)
        x = out
    return x


def replay_layers(acts: np.ndarray, E: int, C: int, policy: int, df=1.0, dp=1):
    """Per-layer replay of a (T, L, K) activation grid with the C oracle."""
    T, L, K = acts.shape
    rb = np.zeros((L, T, E), np.uint8)
    ev = np.zeros((L, T, E), np.uint8)
    for l in range(L):
        rb[l], ev[l] = replay_policy(np.ascontiguousarray(acts[:, l, :]), E, C, policy, df, dp)
    return rb, ev


def sample_layer(weights, T, K, uniforms, repeat_prob=None, u_retain=None):
    """ORACLE restatement of kernels.sample_zipf_layer (kernels.py:150-184) and, with
    repeat_prob / u_retain, sample_markov_layer (kernels.py:187-232): sequential renormalised
    draws without replacement, plain-Python fp64 loops in the reference's order."""
    E = len(weights)
    out = np.zeros((T, K), np.int64)
    for t in range(T):
        avail = [True] * E
        filled = 0
        if repeat_prob is not None and t > 0:
            for j in range(K):
                prev = int(out[t - 1, j])
                if u_retain[t, j] < repeat_prob:
                    out[t, filled] = prev
                    avail[prev] = False
                    filled += 1
        draws = 0
        while filled < K:
            total = 0.0
            for e in range(E):
                if avail[e]:
                    total += float(weights[e])
            x = float(uniforms[t, draws]) * total
            acc, chosen = 0.0, -1
            for e in range(E):
                if avail[e]:
                    acc += float(weights[e])
                    if x < acc:
                        chosen = e
                        break
            if chosen == -1:
                chosen = max(e for e in range(E) if avail[e])
            out[t, filled] = chosen
            avail[chosen] = False
            filled += 1
            draws += 1
        out[t] = np.sort(out[t])
    return out


def gen_trace(kind, L, E, K, T, skew, per_layer_permutation, repeat_prob, seed):
    """ORACLE restatement of tracegen.gen_zipf / gen_markov (tracegen.py:65-112), same RNG
    draw order, sampling by sample_layer.  Returns acts (T, L, K)."""
    rng = np.random.default_rng(seed)
    rank_w = np.arange(1, E + 1, dtype=np.float64) ** (-skew)
    weights = np.empty((L, E))
    shared = rng.permutation(E)
    for l in range(L):
        perm = rng.permutation(E) if per_layer_permutation else shared
        weights[l, perm] = rank_w
    acts = np.zeros((T, L, K), np.int64)
    for l in range(L):
        if kind == "zipf":
            acts[:, l] = sample_layer(weights[l], T, K, rng.random((T, K)))
        else:
            ur = rng.random((T, K))
            ud = rng.random((T, K))
            acts[:, l] = sample_layer(weights[l], T, K, ud, repeat_prob, ur)
    return acts


def prefetch_oracle(acts: np.ndarray, early: np.ndarray, resident_before: np.ndarray, nb: int):
    """The engine's speculative-prefetch rule restated for its decision counts (the
    reference models prefetch only as a cost, costmodel.py:114-132 "every guess is loaded";
    the engine loads only guesses that are not already cached).

    At step (t, l), l < L-1, the early guess for layer l+1 (top-k of gate_{l+1} on h'_l,
    ascending) is walked in order: a guess g already resident in layer l+1 (resident_before
    [t, l+1, g]) is skipped; otherwise it is staged if layer l+1 still has a buffer that is
    neither held by a resident expert nor staged in this step (nb = cache size + staging
    buffers; gate_cache_kernel's prefetch loop).  At step (t, l+1) every miss whose expert was
    staged adopts its buffer (used); the other staged buffers are cancelled (wasted).

    acts (T, L, K) ascending; early (T, L-1, K); resident_before (T, L, E) (engine layout).
    Returns (issued (T, L), used (T, L)) counts indexed by the step the prefetch serves."""
    T, L, K = acts.shape
    issued = np.zeros((T, L), np.int64)
    used = np.zeros((T, L), np.int64)
    for t in range(T):
        for l in range(L - 1):
            res = resident_before[t, l + 1]
            free = nb - int(res.sum())
            staged = []
            for g in early[t, l]:
                if g < 0 or res[g] or len(staged) >= free:
                    continue
                staged.append(int(g))
            issued[t, l + 1] = len(staged)
            used[t, l + 1] = sum(1 for e in acts[t, l + 1] if not res[e] and int(e) in staged)
    return issued, used
