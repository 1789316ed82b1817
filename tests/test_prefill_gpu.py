"""Batched prefill (moe_engine_prefill: tcgen05 grouped GEMMs) against the oracle's restatement
on identical inputs (oracle.mixtral_prefill: the engine's synthetic weights, the same bf16
operand roundings, fp64 elsewhere).

Bars: expert selections equal wherever the oracle's k-th/(k+1)-th logit gap exceeds 1e-3 (any
other disagreement is a stated near-tie); outputs within 1e-2 relative (bf16); step records /
cache traces bit-exact with the C oracle's replay of the engine's own activations (the
reference's replay_policy, kernels.py:60-147) -- including across a prefill -> decode
boundary; H2D bytes == one load per needed, uncached expert per layer."""
import math

import numpy as np
import pytest

import oracle
from oracle.model import replay_layers
from paper_2511_05814_b200.engine import EngineConfig, OffloadEngine
from paper_2511_05814_b200.errors import ConfigError
from paper_2511_05814_b200.metrics import cache_metrics
from paper_2511_05814_b200.policies import PolicyKind

pytestmark = pytest.mark.gpu

SMALL = dict(num_layers=4, num_experts=8, top_k=2, hidden_dim=512, ffn_dim=1792,
             expert_kind="swiglu", rms_norm=True)
GAP = 1e-3


def small_cfg(**kw):
    base = dict(SMALL, mixing_scale=0.1 * math.sqrt(16 / 512), max_tokens=1024)
    base.update(kw)
    return EngineConfig(**base)


def ref_for(cfg, seed):
    return oracle.MixtralRef(cfg.num_layers, cfg.num_experts, cfg.top_k, cfg.hidden_dim,
                             cfg.ffn_dim, cfg.mixing_scale, seed=seed, layout="ref",
                             renormalize=cfg.renormalize, rms_norm=cfg.rms_norm,
                             rms_eps=cfg.rms_eps)


def _check_selections(acts, ref_acts, gaps):
    diff = np.any(acts != ref_acts, axis=2)
    assert not np.any(diff & (gaps > GAP)), "selection mismatch away from a near-tie"
    return diff


def _check_trace(cfg, rec, T0=0):
    code, df, dp = cfg.policy.device_params()
    rb, ev = replay_layers(rec["acts"], cfg.num_experts, cfg.cache_size, code, df, dp)
    assert np.array_equal(rec["resident_before"], np.transpose(rb, (1, 0, 2)))
    assert np.array_equal(rec["evicted"], np.transpose(ev, (1, 0, 2)))


def _needed_loads(rec, E):
    """Experts per layer a prefill must copy: needed over the batch and not resident before."""
    acts, rb = rec["acts"], rec["resident_before"]
    total = 0
    for l in range(acts.shape[1]):
        needed = np.zeros(E, bool)
        needed[np.unique(acts[:, l])] = True
        total += int(np.sum(needed & (rb[0, l] == 0)))
    return total


@pytest.mark.parametrize("policy,C,T", [("lru", 4, 96), ("lfu", 2, 200), ("lfu-aged:0.5:16", 6, 300)])
def test_prefill_matches_oracle(policy, C, T):
    cfg = small_cfg(cache_size=C, policy=PolicyKind.parse(policy))
    X = oracle.MixtralRef.inputs(21, T, cfg.hidden_dim)
    with OffloadEngine(cfg) as eng:
        eng.init_random(21)
        out = eng.prefill(X)
        rec = eng.records(0, T)
        log = eng.event_log(0, T)
        st = eng.stats()
    ref_out, ref_acts, ref_guess, gaps = oracle.mixtral_prefill(ref_for(cfg, 21), X, return_gaps=True)
    diff = _check_selections(rec["acts"], ref_acts, gaps)
    ok = ~diff.any(axis=1)
    rel = np.abs(out[ok] - ref_out[ok]).max() / np.abs(ref_out[ok]).max()
    assert rel < 1e-2, rel
    assert diff.sum() <= 0.01 * diff.size
    g_ok = ok[:, None] & ~diff[:, 1:]
    assert np.array_equal(rec["guessed"][g_ok], ref_guess[g_ok])
    _check_trace(cfg, rec)
    m = cache_metrics(log)
    assert st["hits"] == m.total_hits and st["misses"] == m.total_misses
    assert st["prefill_tokens"] == T
    assert st["prefill_bytes"] == _needed_loads(rec, 8) * cfg.expert_bytes
    assert st["h2d_bytes"] == st["prefill_bytes"]


def test_prefill_then_decode_continues_the_cache_state():
    """Prefill 128 tokens, decode 24 more: the whole 152-step trace equals one replay."""
    cfg = small_cfg(cache_size=3, policy=PolicyKind.lfu())
    Tp, Td = 128, 24
    X = oracle.MixtralRef.inputs(8, Tp + Td, cfg.hidden_dim)
    with OffloadEngine(cfg) as eng:
        eng.init_random(8)
        out_p = eng.prefill(X[:Tp])
        out_d = eng.decode(X[Tp:])
        rec = eng.records(0, Tp + Td)
        st = eng.stats()
    _check_trace(cfg, rec)
    ref = ref_for(cfg, 8)
    ref_out_d, ref_acts_d = ref.decode(X[Tp:])
    assert np.array_equal(rec["acts"][Tp:], ref_acts_d)
    assert np.abs(out_d - ref_out_d).max() / np.abs(ref_out_d).max() < 1e-2
    # decode demand copies after the prefill: one per miss, nothing more
    dec_misses = int(sum(np.sum(rec["resident_before"][t, l][rec["acts"][t, l]] == 0)
                         for t in range(Tp, Tp + Td) for l in range(cfg.num_layers)))
    assert st["demand_bytes"] == dec_misses * cfg.expert_bytes


def test_prefill_matches_decode_trace_semantics():
    """The same tokens prefilled or decoded give the same cache decisions for the same
    activations (the policy is replayed in token order), and outputs agree within bf16."""
    cfg = small_cfg(cache_size=4, policy=PolicyKind.lru())
    T = 64
    X = oracle.MixtralRef.inputs(4, T, cfg.hidden_dim)
    with OffloadEngine(cfg) as eng:
        eng.init_random(4)
        out_d = eng.decode(X)
        rec_d = eng.records(0, T)
        eng.reset()
        out_p = eng.prefill(X)
        rec_p = eng.records(T, T)
    same = np.all(rec_d["acts"] == rec_p["acts"], axis=(1, 2))
    assert same.mean() > 0.95
    if same.all():
        for k in ("resident_before", "evicted"):
            assert np.array_equal(rec_d[k], rec_p[k]), k
    # guesses are gate_l(h_in): near-ties may flip between f32 (decode) and bf16-operand
    # (prefill) layer inputs
    assert np.mean(np.all(rec_d["guessed"] == rec_p["guessed"], axis=2)) > 0.95
    assert np.abs(out_d[same] - out_p[same]).max() / np.abs(out_d[same]).max() < 1e-2


def test_prefill_with_prefetch_engine_and_warm_cache():
    """Prefill on a warm cache of a prefetch-enabled engine: staging buffers are reclaimed,
    resident experts are computed in place and only the rest is copied."""
    cfg = small_cfg(cache_size=4, policy=PolicyKind.lfu(), prefetch="early", chunk_bytes=1 << 20)
    X = oracle.MixtralRef.inputs(13, 160, cfg.hidden_dim)
    with OffloadEngine(cfg) as eng:
        eng.init_random(13)
        eng.decode(X[:32])
        st0 = eng.stats()
        eng.prefill(X[32:])
        eng.decode(X[:8])
        rec = eng.records(0, 168)
        st1 = eng.stats()
    _check_trace(cfg, rec)
    pre = {k: v[32:160] for k, v in rec.items()}
    assert st1["prefill_bytes"] == _needed_loads(pre, 8) * cfg.expert_bytes
    assert st1["prefill_bytes"] < 4 * 8 * cfg.expert_bytes  # warm: fewer than every expert


def test_prefill_rejects_bad_shapes():
    cfg = small_cfg(max_tokens=16)
    with OffloadEngine(cfg) as eng:
        eng.init_random(1)
        with pytest.raises(ConfigError):
            eng.prefill(np.zeros((17, cfg.hidden_dim), np.float32))
    cfg = EngineConfig(num_layers=2, num_experts=8, top_k=2, hidden_dim=384, ffn_dim=768,
                       expert_kind="swiglu", rms_norm=True, mixing_scale=0.01)
    with OffloadEngine(cfg) as eng:
        with pytest.raises(ConfigError):
            eng.prefill(np.zeros((4, 384), np.float32))


def test_prefill_full_mixtral_8x7b_shape_two_layers():
    """Full d=4096, f=14336 experts, 512 tokens: tensor-core GEMMs over ~128 rows per expert."""
    cfg = EngineConfig.mixtral_8x7b(num_layers=2, cache_size=4, max_tokens=512)
    T = 512
    X = oracle.MixtralRef.inputs(42, T, 4096)
    with OffloadEngine(cfg) as eng:
        eng.init_random(42)
        eng.profile(True)
        out = eng.prefill(X)
        rec = eng.records(0, T)
        st = eng.stats()
        kt = eng.kernel_times()
    ref = oracle.MixtralRef(2, 8, 2, 4096, 14336, cfg.mixing_scale, seed=42, layout="ref", rms_norm=True)
    ref_out, ref_acts, _, gaps = oracle.mixtral_prefill(ref, X, return_gaps=True)
    diff = _check_selections(rec["acts"], ref_acts, gaps)
    ok = ~diff.any(axis=1)
    assert np.abs(out[ok] - ref_out[ok]).max() / np.abs(ref_out[ok]).max() < 1e-2
    _check_trace(cfg, rec)
    assert st["prefill_bytes"] == _needed_loads(rec, 8) * 352321536
    print(f"prefill GEMMs: {kt['gemm_launches']} launches {kt['gemm_ms']:.3f} ms "
          f"{kt['gemm_flops'] / kt['gemm_ms'] / 1e9:.1f} TFLOP/s; prefill {kt['prefill_ms']:.1f} ms")


def test_prefill_compressed_loads_bit_exact():
    cfg0 = small_cfg(cache_size=3, policy=PolicyKind.lru(), transfer="copy_engine")
    cfg1 = small_cfg(cache_size=3, policy=PolicyKind.lru(), transfer="copy_engine", compress=True)
    X = oracle.MixtralRef.inputs(31, 128, cfg0.hidden_dim)
    res = []
    for cfg in (cfg0, cfg1):
        with OffloadEngine(cfg) as eng:
            eng.init_random(31)
            out = eng.prefill(X[:100])
            out2 = eng.decode(X[100:])
            res.append((out, out2, eng.records(0, 128), eng.stats()))
    (a, a2, ra, sa), (b, b2, rb, sb) = res
    assert np.array_equal(a, b) and np.array_equal(a2, b2)
    for k in ("acts", "resident_before", "evicted", "probs"):
        assert np.array_equal(ra[k], rb[k]), k
    assert sb["prefill_bytes"] < 0.75 * sa["prefill_bytes"]


def test_prefill_single_token_and_nonfinite():
    cfg = small_cfg(cache_size=2)
    X = oracle.MixtralRef.inputs(9, 4, cfg.hidden_dim)
    with OffloadEngine(cfg) as eng:
        eng.init_random(9)
        out1 = eng.prefill(X[:1])
        rec = eng.records(0, 1)
        bad = X[1:].copy()
        bad[1, 0] = np.nan
        with pytest.raises(FloatingPointError):
            eng.prefill(bad)
    ref_out, ref_acts = ref_for(cfg, 9).decode(X[:1])
    assert np.array_equal(rec["acts"], ref_acts)
    assert np.abs(out1 - ref_out).max() / np.abs(ref_out).max() < 1e-2


@pytest.mark.parametrize("compress", [0, 1])
def test_prefill_is_deterministic_across_runs(compress):
    """The same tokens prefilled from a cold cache three times on one engine -- fresh, after a
    reset, after decode traffic in another mode -- give identical records and outputs."""
    cfg = small_cfg(cache_size=6, policy=PolicyKind.lru(), prefetch="early", compress=compress)
    T = 200
    X = oracle.MixtralRef.inputs(11, T, cfg.hidden_dim)
    runs = []
    with OffloadEngine(cfg) as eng:
        eng.init_random(11)
        for r in range(3):
            eng.set_mode(policy=PolicyKind.lru(), cache_size=4, prefetch="off")
            t0 = eng.tokens_done
            out = eng.prefill(X)
            runs.append((eng.records(t0, T), out))
            if r == 1:
                eng.set_mode(policy=PolicyKind.lfu(), cache_size=6, prefetch="early")
                eng.decode(X[:16])
    for rec, out in runs[1:]:
        for k in ("acts", "resident_before", "evicted", "guessed"):
            assert np.array_equal(rec[k], runs[0][0][k]), k
        assert np.array_equal(out, runs[0][1])


@pytest.mark.parametrize("compress", [0, 1])
def test_prefill_in_a_smaller_mode_than_allocated_matches_oracle(compress):
    """An engine allocated for C=6 + prefetch staging, switched (set_mode) to LRU C=4 without
    prefetch -- the bench's configs[3] setup -- prefills against the oracle like a C=4 engine
    (the pool keeps its allocated layer stride)."""
    cfg = small_cfg(cache_size=6, policy=PolicyKind.lru(), prefetch="early", compress=compress)
    T = 160
    X = oracle.MixtralRef.inputs(21, T, cfg.hidden_dim)
    with OffloadEngine(cfg) as eng:
        eng.init_random(21)
        eng.set_mode(policy=PolicyKind.lfu(), cache_size=6, prefetch="early")
        eng.decode(X[:24])                   # fills every buffer of the allocation
        eng.set_mode(policy=PolicyKind.lru(), cache_size=4, prefetch="off")
        t0 = eng.tokens_done
        out = eng.prefill(X)
        rec = eng.records(t0, T)
    ref_cfg = small_cfg(cache_size=4, policy=PolicyKind.lru())
    ref_out, ref_acts, _, gaps = oracle.mixtral_prefill(ref_for(ref_cfg, 21), X, return_gaps=True)
    diff = _check_selections(rec["acts"], ref_acts, gaps)
    ok = ~diff.any(axis=1)
    assert np.abs(out[ok] - ref_out[ok]).max() / np.abs(ref_out[ok]).max() < 1e-2
    _check_trace(ref_cfg, rec)
