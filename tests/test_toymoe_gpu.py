"""Model API and the engine on the tiny config, against reference-generated goldens."""
import hashlib
import json
import math

import numpy as np
import pytest

import oracle
from conftest import GOLDEN
from paper_2511_05814_b200.simulate import SimConfig, simulate
from paper_2511_05814_b200.engine import EngineConfig, OffloadEngine
from paper_2511_05814_b200.errors import ConfigError
from paper_2511_05814_b200.metrics import cache_metrics, speculation_metrics
from paper_2511_05814_b200.policies import PolicyKind
from paper_2511_05814_b200.simulate import format_event_log
from paper_2511_05814_b200.toymoe import (GatingNetwork, HiddenState, ToyModelConfig, ToyMoeModel,
                                          forward_token, gate_select, run_model, speculate_next)
from paper_2511_05814_b200.traces import ModelShape, format_trace

pytestmark = pytest.mark.gpu
MANIFEST = json.loads((GOLDEN / "manifest.json").read_text())
T1 = ToyModelConfig(ModelShape(4, 8, 2), hidden_dim=256, mixing_scale=0.1, skew=1.0, seed=42,
                    tokens=64)


def sha(b):
    return hashlib.sha256(b).hexdigest()


def ident(logits):
    d = len(logits)
    return GatingNetwork(np.eye(d)), HiddenState(np.array(logits, float), -1)


class TestGate:
    def test_order_and_ties(self):
        g, h = ident([2, 1, 0, 0, 0, 0, 0, 0])
        assert [e for e, _ in gate_select(h, g, 2)] == [0, 1]
        g, h = ident([0.0] * 8)
        assert [e for e, _ in gate_select(h, g, 2)] == [0, 1]
        g, h = ident([-0.0, 0.0, -0.0, 0.0])
        assert [e for e, _ in gate_select(h, g, 3)] == [0, 1, 2]

    def test_analytic_softmax(self):
        g, h = ident([math.log(2), math.log(1)])
        picks = gate_select(h, g, 2)
        assert picks[0][0] == 0
        assert picks[0][1] == pytest.approx(2 / 3, abs=1e-12)
        assert picks[1][1] == pytest.approx(1 / 3, abs=1e-12)

    def test_probabilities(self, rng):
        g = GatingNetwork(rng.standard_normal((6, 8)))
        picks = gate_select(HiddenState(rng.standard_normal(6), -1), g, 8)
        p = np.array([q for _, q in picks])
        assert p.sum() == pytest.approx(1.0, abs=1e-12) and (np.diff(p) <= 0).all()

    def test_errors(self):
        with pytest.raises(ConfigError):
            gate_select(HiddenState(np.zeros(5), -1), GatingNetwork(np.zeros((4, 8))), 2)
        with pytest.raises(FloatingPointError):
            gate_select(HiddenState(np.ones(2), -1), GatingNetwork(np.full((2, 4), np.inf)), 2)
        with pytest.raises(ConfigError):
            gate_select(HiddenState(np.ones(2), -1), GatingNetwork(np.ones((2, 4))), 5)


def test_forward_token_and_gate_match_reference_cases():
    z = np.load(GOLDEN / "forward_cases.npz")
    for i in range(6):
        L, E, K, d, alpha, seed, l = z[f"cfg_{i}"]
        cfg = ToyModelConfig(ModelShape(int(L), int(E), int(K)), hidden_dim=int(d),
                             mixing_scale=float(alpha), seed=int(seed))
        model, _ = ToyMoeModel.build(cfg)
        h, sel = forward_token(model, HiddenState(z[f"x_{i}"], -1), int(l))
        np.testing.assert_allclose(h.values, z[f"h_{i}"], rtol=1e-12, atol=1e-12)
        assert sorted(sel) == z[f"sel_{i}"].tolist()
        picks = gate_select(HiddenState(z[f"x_{i}"], -1), model.gates[int(l)], int(E))
        assert [e for e, _ in picks] == z[f"gate_ids_{i}"].tolist()
        np.testing.assert_allclose([p for _, p in picks], z[f"gate_p_{i}"], rtol=1e-12)


def test_forward_token_identity_and_range():
    cfg = ToyModelConfig(ModelShape(2, 4, 2), hidden_dim=4, mixing_scale=0.0, seed=3)
    model, _ = ToyMoeModel.build(cfg)
    object.__setattr__(model, "expert_w2", np.zeros_like(model.expert_w2))
    h_in = HiddenState(np.array([1.0, -2.0, 0.5, 0.0]), -1)
    out, act = forward_token(model, h_in, 0)
    assert np.array_equal(out.values, h_in.values) and len(act) == 2
    with pytest.raises(ConfigError):
        forward_token(model, h_in, 2)


def test_speculate_next_alpha_zero_exact():
    cfg = ToyModelConfig(ModelShape(2, 8, 2), mixing_scale=0.0, seed=21)
    model, rng = ToyMoeModel.build(cfg)
    h0, _ = forward_token(model, HiddenState(rng.standard_normal(16), -1), 0)
    _, actual = forward_token(model, h0, 1)
    assert speculate_next(h0, model.gates[1], 2) == actual


def test_run_model_t1_byte_identical_traces():
    act, spec = run_model(T1)
    assert format_trace(act) == (GOLDEN / "toy_t1" / "activation.jsonl").read_bytes()
    assert format_trace(spec) == (GOLDEN / "toy_t1" / "speculation.jsonl").read_bytes()
    for pol in ("lru", "lfu"):
        for C in (2, 4):
            log = simulate(act, SimConfig(PolicyKind.parse(pol), C))
            assert format_event_log(log) == (GOLDEN / "toy_t1" / f"events_{pol}_c{C}.jsonl").read_bytes()


def test_run_model_small_configs_match_reference():
    z = np.load(GOLDEN / "toy_small.npz")
    for i, (L, E, K, d, a, s, seed, T) in enumerate(z["configs"]):
        cfg = ToyModelConfig(ModelShape(int(L), int(E), int(K)), hidden_dim=int(d),
                             mixing_scale=a, skew=s, seed=int(seed), tokens=int(T))
        act, spec = run_model(cfg)
        assert np.array_equal(act.activations, z[f"acts_{i}"]), i
        assert np.array_equal(spec.guessed, z[f"guessed_{i}"]), i
        assert np.array_equal(spec.actual, z[f"actual_{i}"]), i


def test_run_model_zero_tokens_and_single_layer():
    act, spec = run_model(ToyModelConfig(ModelShape(4, 8, 2), tokens=0))
    assert act.num_tokens == 0 and spec.num_tokens == 0
    act, spec = run_model(ToyModelConfig(ModelShape(1, 8, 2), tokens=5))
    assert act.num_tokens == 5 and spec.num_tokens == 0


def test_alpha_zero_speculation_exact():
    for seed in (0, 1, 2):
        _, spec = run_model(ToyModelConfig(ModelShape(5, 8, 2), tokens=24, mixing_scale=0.0, seed=seed))
        assert speculation_metrics(spec).precision == 1.0


def test_t1_1024_engine_selections_and_live_cache_trace():
    """Configuration C1: the engine decodes 1024 tokens with its own LRU C=2 cache; its
    activations equal the reference's and its live event log is byte-identical to the
    reference's simulate() output on the same trace (teacher-forced == free-running)."""
    z = np.load(GOLDEN / "toy_t1_1024.npz")
    cfg = ToyModelConfig(ModelShape(4, 8, 2), hidden_dim=256, mixing_scale=0.1, seed=42, tokens=1024)
    model, rng = ToyMoeModel.build(cfg)
    inputs = rng.standard_normal((1024, 256)).astype(np.float32)
    for pol, C in (("lru", 2), ("lfu", 4), ("lfu-aged:0.5:16", 6), ("lru", 6)):
        ecfg = EngineConfig(num_layers=4, num_experts=8, top_k=2, hidden_dim=256,
                            expert_kind="toy_tanh", cache_size=C, policy=PolicyKind.parse(pol),
                            mixing_scale=0.1, max_tokens=1024)
        with OffloadEngine(ecfg) as eng:
            eng.load_toy_model(model)
            eng.decode(inputs)
            rec = eng.records(0, 1024)
            live = eng.event_log(0, 1024)
            st = eng.stats()
        assert np.array_equal(rec["acts"], z["acts"])
        assert np.array_equal(rec["guessed"], z["guessed"])
        want = MANIFEST["toy_t1_1024"]["event_logs"][f"{pol}_c{C}"]
        assert sha(format_event_log(live)) == want["sha256"], (pol, C)
        m = cache_metrics(live)
        assert m.total_hits == want["hits"]
        # transfer-volume identity (costmodel.py:100-110): every miss moved one expert block
        assert st["misses"] == m.total_misses
        assert st["demand_bytes"] == m.total_misses * st["expert_bytes"]
        assert st["prefetch_bytes"] == 0


def test_engine_outputs_match_oracle_fp32_tolerance():
    L, E, K, d, T = 4, 8, 2, 256, 32
    w = oracle.toy_weights(L, E, d, 1.0, 42, T)
    cfg = ToyModelConfig(ModelShape(L, E, K), hidden_dim=d, seed=42, tokens=T)
    model, _ = ToyMoeModel.build(cfg)
    with OffloadEngine(EngineConfig(num_layers=L, num_experts=E, top_k=K, hidden_dim=d,
                                    expert_kind="toy_tanh", cache_size=3, max_tokens=T)) as eng:
        eng.load_toy_model(model)
        out = eng.decode(w["inputs"].astype(np.float32))
    for t in range(T):
        h = w["inputs"][t]
        for l in range(L):
            h, _, _, _ = oracle.toy_forward(w, h, l, 0.1, K)
        np.testing.assert_allclose(out[t], h, rtol=1e-5, atol=1e-5 * np.abs(h).max())


def test_engine_nonfinite_raises():
    cfg = ToyModelConfig(ModelShape(2, 4, 2), hidden_dim=8, seed=1, tokens=2)
    model, _ = ToyMoeModel.build(cfg)
    with OffloadEngine(EngineConfig(num_layers=2, num_experts=4, top_k=2, hidden_dim=8,
                                    expert_kind="toy_tanh", cache_size=2, max_tokens=4)) as eng:
        eng.load_toy_model(model)
        with pytest.raises(FloatingPointError):
            eng.decode(np.full((1, 8), np.inf, np.float32))


def test_engine_config_errors():
    with pytest.raises(ConfigError):
        OffloadEngine(EngineConfig(num_layers=2, num_experts=8, top_k=3, hidden_dim=8,
                                   expert_kind="toy_tanh", cache_size=2))
    with pytest.raises(ConfigError):
        OffloadEngine(EngineConfig(num_layers=2, num_experts=8, top_k=2, hidden_dim=8,
                                   expert_kind="toy_tanh", cache_size=2, policy=PolicyKind.opt()))


def test_reference_suite_run_model_configs():
    """Every distinct run_model config the reference's own test suite uses (100: mixing scales
    0.1 .. 100, skew 0 / 1, 1-6 layers, up to 64 tokens), through the GPU engine: activation and
    speculation traces identical to the reference's."""
    from conftest import refsuite_run_models

    n = 0
    for (L, E, K, d, alpha, skew, seed, T), acts, guessed, actual in refsuite_run_models():
        cfg = ToyModelConfig(ModelShape(L, E, K), hidden_dim=d, mixing_scale=alpha, skew=skew,
                             seed=seed, tokens=T)
        a, s = run_model(cfg)
        key = (L, E, K, d, alpha, skew, seed, T)
        assert np.array_equal(a.activations, acts), key
        assert np.array_equal(s.guessed, guessed) and np.array_equal(s.actual, actual), key
        n += 1
    assert n == 100


def test_reference_suite_model_api_calls():
    """Every gate_select / speculate_next / forward_token call of the reference's own test suite
    (tests/golden/refsuite_toymoe_calls.json.gz, the reference's results and errors recorded):
    same ids / selected sets, probabilities and hidden states within 1e-12 relative (fp64 on the
    device vs numpy's BLAS summation order), the same exception classes."""
    from paper_2511_05814_b200 import errors

    import gzip

    with gzip.open(GOLDEN / "refsuite_toymoe_calls.json.gz", "rt") as f:
        calls = json.load(f)
    assert len(calls) >= 13
    for rec in calls:
        h = HiddenState(np.array(rec["h"], dtype=np.float64), rec["h_layer"])
        if rec["kind"] == "forward_token":
            L, E, K, d, alpha, skew, seed, T = rec["config"]
            model, _ = ToyMoeModel.build(ToyModelConfig(ModelShape(int(L), int(E), int(K)), hidden_dim=int(d),
                                                        mixing_scale=alpha, skew=skew, seed=int(seed),
                                                        tokens=int(T)))
            w = rec["weights"]   # the arrays the reference test actually used
            model.gates = tuple(GatingNetwork(np.array(gw), None if gb is None else np.array(gb))
                                for gw, gb in zip(w["gate_w"], w["gate_b"]))
            model.mixing = np.array(w["mixing"])
            model.expert_w1 = np.array(w["w1"])
            model.expert_w2 = np.array(w["w2"])
            call = lambda: forward_token(model, h, rec["layer"])  # noqa: E731
        else:
            gate = GatingNetwork(np.array(rec["w"], dtype=np.float64),
                                 None if rec["b"] is None else np.array(rec["b"], dtype=np.float64))
            fn = gate_select if rec["kind"] == "gate_select" else speculate_next
            call = lambda: fn(h, gate, rec["k"])  # noqa: E731
        if "error" in rec:
            exc = getattr(errors, rec["error"], None) or {"FloatingPointError": FloatingPointError,
                                                          "ValueError": ValueError}.get(rec["error"], Exception)
            with pytest.raises(exc):
                call()
            continue
        got = call()
        if rec["kind"] == "gate_select":
            assert [e for e, _ in got] == [e for e, _ in rec["result"]], rec
            np.testing.assert_allclose([p for _, p in got], [p for _, p in rec["result"]], rtol=1e-12)
        elif rec["kind"] == "speculate_next":
            assert sorted(got) == rec["result"], rec
        else:
            out, sel = got
            assert sorted(sel) == rec["result"]["selected"] and out.layer == rec["result"]["layer"]
            np.testing.assert_allclose(out.values, rec["result"]["values"], rtol=1e-12, atol=1e-12)


def test_run_model_near_tie_fallback_is_the_fp64_path(monkeypatch):
    """run_model re-decodes tokens with a near-tie margin on the fp64 device path.  Forcing
    every token through that path (threshold huge) reproduces the reference's traces exactly
    as the fp32 engine does (T1 and a deep, large-mixing config), and the fp32 engine's own
    margins on T1 are far above the threshold."""
    from paper_2511_05814_b200 import toymoe

    cfgs = [ToyModelConfig(ModelShape(4, 8, 2), hidden_dim=256, mixing_scale=0.1, seed=42, tokens=64),
            ToyModelConfig(ModelShape(6, 8, 2), hidden_dim=64, mixing_scale=3.0, seed=7, tokens=24)]
    base = [run_model(c) for c in cfgs]
    monkeypatch.setattr(toymoe, "NEAR_TIE_REL", 1e30)
    forced = [run_model(c) for c in cfgs]
    for (a0, s0), (a1, s1) in zip(base, forced):
        assert np.array_equal(a0.activations, a1.activations)
        assert np.array_equal(s0.guessed, s1.guessed)
    ref_acts, ref_guessed, _ = oracle.toy_run_model(4, 8, 2, 256, 0.1, 1.0, 42, 64)
    assert np.array_equal(forced[0][0].activations, ref_acts)
    assert np.array_equal(forced[0][1].guessed, ref_guessed)
