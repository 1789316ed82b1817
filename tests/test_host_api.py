"""Host-side logic of the drop-in API (no GPU): data model, JSONL formats, policy kinds,
metrics and cost identities.  Cases follow the reference's own tests (pkg/tests)."""
import io
import itertools

import numpy as np
import pytest

from conftest import random_stream
from paper_2511_05814_b200.costmodel import CostParams, estimate_latency, speculation_cost
from paper_2511_05814_b200.errors import ConfigError, TraceParseError, TraceValidationError
from paper_2511_05814_b200.metrics import cache_metrics, speculation_metrics
from paper_2511_05814_b200.policies import PolicyKind, warm_state
from paper_2511_05814_b200.simulate import (CacheEventLog, SimConfig, format_event_log,
                                            offloads_to_cache_size, read_event_log)
from paper_2511_05814_b200.traces import (ActivationTrace, ModelShape, SpeculationTrace,
                                          trace_from_bytes, trace_to_bytes)
import oracle


def rand_act(rng, shape, T):
    a = np.zeros((T, shape.num_layers, shape.top_k), np.int64)
    for t in range(T):
        for l in range(shape.num_layers):
            a[t, l] = np.sort(rng.choice(shape.num_experts, shape.top_k, replace=False))
    return ActivationTrace(shape, a)


def rand_spec(rng, shape, T):
    g = np.zeros((T, shape.num_layers - 1, shape.top_k), np.int64)
    a = np.zeros_like(g)
    for t in range(T):
        for j in range(shape.num_layers - 1):
            g[t, j] = np.sort(rng.choice(shape.num_experts, shape.top_k, replace=False))
            a[t, j] = np.sort(rng.choice(shape.num_experts, shape.top_k, replace=False))
    return SpeculationTrace(shape, g, a)


def oracle_log(trace, policy, C, warmup=0):
    kind = PolicyKind.parse(policy)
    T, L, K = trace.activations.shape if trace.num_tokens else (0, trace.shape.num_layers, trace.shape.top_k)
    E = trace.shape.num_experts
    acts, rbs, evs = {}, {}, {}
    for l in range(trace.shape.num_layers):
        a = np.ascontiguousarray(trace.activations[:, l, :])
        rbs[l], evs[l] = oracle.replay_policy(a, E, C, *kind.device_params()) if T else (
            np.zeros((0, E), np.uint8), np.zeros((0, E), np.uint8))
        acts[l] = a
    return CacheEventLog(SimConfig(kind, C, warmup), trace.shape, tuple(range(trace.shape.num_layers)),
                         acts, rbs, evs, T)


class TestModelShape:
    def test_defaults_and_validation(self):
        assert ModelShape() == ModelShape(32, 8, 2)
        for bad in [(0, 8, 2), (1, 0, 1), (1, 4, 5), (1, 4, 0)]:
            with pytest.raises(TraceValidationError):
                ModelShape(*bad)


class TestTraces:
    def test_roundtrip_byte_identical(self):
        rng = np.random.default_rng(10)
        for i in range(300):
            L, E = int(rng.integers(1, 5)), int(rng.integers(2, 9))
            K, T = int(rng.integers(1, E + 1)), int(rng.integers(0, 6))
            shape = ModelShape(L, E, K)
            if i % 2 or L < 2:
                tr = rand_act(rng, shape, T)
            else:
                tr = rand_spec(rng, shape, T)
            b = trace_to_bytes(tr)
            assert trace_to_bytes(trace_from_bytes(b)) == b
            assert trace_from_bytes(b) == tr

    def test_exact_format(self):
        shape = ModelShape(2, 8, 2)
        tr = ActivationTrace(shape, np.array([[[1, 6], [1, 2]]]))
        assert trace_to_bytes(tr) == (b'{"kind":"activation","num_layers":2,"num_experts":8,"top_k":2}\n'
                                      b'{"t":0,"l":0,"a":[1,6]}\n{"t":0,"l":1,"a":[1,2]}\n')
        sp = SpeculationTrace(shape, np.array([[[0, 1]]]), np.array([[[1, 2]]]))
        assert trace_to_bytes(sp).splitlines()[1] == b'{"t":0,"l":1,"g":[0,1],"a":[1,2]}'

    def test_records_order_irrelevant(self):
        head = '{"kind":"activation","num_layers":2,"num_experts":4,"top_k":1}\n'
        body = '{"t":0,"l":1,"a":[2]}\n{"t":0,"l":0,"a":[3]}\n'
        tr = trace_from_bytes((head + body).encode())
        assert tr.activations.tolist() == [[[3], [2]]]

    @pytest.mark.parametrize("text,exc", [
        ("", TraceParseError),
        ("not json\n", TraceParseError),
        ('{"kind":"weird","num_layers":1,"num_experts":2,"top_k":1}\n', TraceParseError),
        ('{"kind":"activation","num_layers":1,"num_experts":2}\n', TraceParseError),
        ('{"kind":"activation","num_layers":1,"num_experts":2,"top_k":1}\n[1]\n', TraceParseError),
        ('{"kind":"activation","num_layers":1,"num_experts":2,"top_k":1}\n{"t":true,"l":0,"a":[0]}\n', TraceParseError),
        ('{"kind":"activation","num_layers":1,"num_experts":2,"top_k":1}\n{"t":0,"l":0,"a":[0,0]}\n', TraceValidationError),
        ('{"kind":"activation","num_layers":1,"num_experts":2,"top_k":1}\n{"t":0,"l":0,"a":[5]}\n', TraceValidationError),
        ('{"kind":"activation","num_layers":1,"num_experts":2,"top_k":1}\n{"t":0,"l":3,"a":[1]}\n', TraceValidationError),
        ('{"kind":"activation","num_layers":1,"num_experts":2,"top_k":1}\n{"t":1,"l":0,"a":[1]}\n', TraceValidationError),
        ('{"kind":"activation","num_layers":2,"num_experts":2,"top_k":1}\n{"t":0,"l":0,"a":[1]}\n', TraceValidationError),
        ('{"kind":"speculation","num_layers":2,"num_experts":2,"top_k":1}\n{"t":0,"l":0,"g":[1],"a":[1]}\n', TraceValidationError),
    ])
    def test_reader_errors(self, text, exc):
        with pytest.raises(exc):
            trace_from_bytes(text.encode())

    def test_parse_error_carries_line(self):
        with pytest.raises(TraceParseError) as info:
            trace_from_bytes(b'{"kind":"activation","num_layers":1,"num_experts":2,"top_k":1}\n{"t":0}\n')
        assert info.value.line == 2

    def test_single_layer_speculation_is_empty(self):
        sp = SpeculationTrace(ModelShape(1, 8, 2), np.zeros((5, 0, 2)), np.zeros((5, 0, 2)))
        assert sp.num_tokens == 0 and sp.records == []


class TestPolicyKind:
    def test_parse_and_str(self):
        assert PolicyKind.parse(" LFU ") == PolicyKind.lfu()
        k = PolicyKind.parse("lfu-aged:0.25:8")
        assert (k.decay_factor, k.decay_period, str(k)) == (0.25, 8, "lfu-aged:0.25:8")
        assert PolicyKind.parse("lfu-aged") == PolicyKind.lfu_aged(0.5, 16)
        assert str(PolicyKind.lfu_aged(0.5, 16)) == "lfu-aged:0.5:16"

    @pytest.mark.parametrize("bad", ["mru", "lfu-aged:0.5", "lfu-aged:x:8", "", "lfu-aged:0:4",
                                     "lfu-aged:0.5:0", "lfu-aged:1.5:2"])
    def test_parse_rejects(self, bad):
        with pytest.raises(ConfigError):
            PolicyKind.parse(bad)

    def test_decay_params_only_for_aged(self):
        with pytest.raises(ConfigError):
            PolicyKind("lru", 0.5, 4)
        with pytest.raises(ConfigError):
            PolicyKind("lfu-aged")

    def test_warm_state(self):
        s = warm_state(PolicyKind.lru(), 4)
        assert (s.resident, s.recency, s.freq, s.step) == (frozenset(), (), {}, 0)
        with pytest.raises(ConfigError):
            warm_state(PolicyKind.lru(), 0)


class TestEventLog:
    def test_exact_lines(self):
        tr = ActivationTrace(ModelShape(1, 8, 2), np.array([[[0, 1]], [[0, 2]]]))
        lines = format_event_log(oracle_log(tr, "lru", 4)).decode().splitlines()
        assert lines[0] == ('{"kind":"events","policy":"lru","cache_size":4,"num_layers":1,'
                            '"num_experts":8,"top_k":2,"warmup_tokens":0}')
        assert lines[1] == '{"t":0,"l":0,"cached":[],"hit":[],"miss":[0,1],"evict":[]}'
        assert lines[2] == '{"t":1,"l":0,"cached":[0,1],"hit":[0],"miss":[2],"evict":[]}'

    def test_roundtrip(self):
        rng = np.random.default_rng(3)
        log = oracle_log(rand_act(rng, ModelShape(2, 8, 2), 12), "lfu-aged:0.5:16", 4, warmup=2)
        data = format_event_log(log)
        back = read_event_log(io.BytesIO(data))
        assert back == log and format_event_log(back) == data

    def test_reader_rejects(self):
        head = ('{"kind":"events","policy":"lru","cache_size":2,"num_layers":1,'
                '"num_experts":4,"top_k":1,"warmup_tokens":0}')
        for body in ['{"t":0,"l":0,"cached":[],"hit":[0],"miss":[1],"evict":[]}',
                     '{"t":1,"l":0,"cached":[],"hit":[],"miss":[1],"evict":[]}',
                     '{"t":0,"l":0,"cached":[9],"hit":[],"miss":[1],"evict":[]}']:
            with pytest.raises(TraceValidationError):
                read_event_log(io.BytesIO((head + "\n" + body + "\n").encode()))
        with pytest.raises(TraceParseError):
            read_event_log(io.BytesIO(b""))

    def test_offloads_mapping(self):
        s = ModelShape(32, 8, 2)
        assert offloads_to_cache_size(4, s) == 4 and offloads_to_cache_size(6, s) == 2
        for bad in (8, -1):
            with pytest.raises(ConfigError):
                offloads_to_cache_size(bad, s)

    def test_sim_config_validation(self):
        with pytest.raises(ConfigError):
            SimConfig(PolicyKind.lru(), 0)
        with pytest.raises(ConfigError):
            SimConfig(PolicyKind.lru(), 2, warmup_tokens=-1)


class TestMetrics:
    def test_constant_workload(self):
        tr = ActivationTrace(ModelShape(1, 8, 2), np.array([[[0, 1]]] * 5))
        log = oracle_log(tr, "lru", 4)
        assert log.miss_counts(0).tolist() == [2, 0, 0, 0, 0]
        m = cache_metrics(log)
        assert (m.total_hits, m.total_misses, m.hit_rate) == (8, 2, 0.8)
        assert m.precision == 8 / 8

    def test_warmup_excluded(self):
        tr = ActivationTrace(ModelShape(1, 8, 2), np.array([[[0, 1]]] * 5))
        m = cache_metrics(oracle_log(tr, "lru", 4, warmup=1))
        assert m.hit_rate == 1.0 and m.including_warmup["hit_rate"] == 0.8

    def test_empty(self):
        tr = ActivationTrace(ModelShape(2, 8, 2), np.zeros((0, 2, 2), np.int64))
        m = cache_metrics(oracle_log(tr, "lru", 4))
        assert m.empty and m.hit_rate == 0.0 and m.precision is None

    def test_full_cache_lock(self):
        rng = np.random.default_rng(5)
        m = cache_metrics(oracle_log(rand_act(rng, ModelShape(2, 8, 2), 200), "lfu", 4))
        fc = m.full_cache
        assert fc.recall == pytest.approx(4 / 2 * fc.precision)

    def test_speculation_fp_equals_fn(self):
        rng = np.random.default_rng(6)
        sp = rand_spec(rng, ModelShape(5, 8, 2), 30)
        m = speculation_metrics(sp)
        assert m.fp == m.fn and m.precision == m.recall
        assert m.tp + m.fp == 30 * 4 * 2

    def test_cost_identities(self):
        rng = np.random.default_rng(7)
        tr = rand_act(rng, ModelShape(3, 8, 2), 40)
        log = oracle_log(tr, "lru", 4)
        p = CostParams(expert_bytes=352321536, bandwidth_bytes_per_s=55e9, compute_s_per_layer=1e-4)
        est = estimate_latency(log, p)
        misses = sum(int(log.miss_counts(l).sum()) for l in range(3))
        assert est.bytes_transferred == misses * 352321536
        sp = rand_spec(rng, ModelShape(3, 8, 2), 10)
        sm = speculation_metrics(sp)
        moved, wasted = speculation_cost(sp, CostParams(expert_bytes=100.0))
        assert moved == (10 * 2 * 2 + sm.fn) * 100 and wasted == sm.fn * 100
        with pytest.raises(ConfigError):
            CostParams(overlap=1.5)


def test_exhaustive_lru_lfu_small_alphabet_oracle():
    """Criterion 04 (tests/test_acceptance.py:155-173) on the oracle: all 4^6 traces."""
    def straight(stream, C, pol):
        res, freq, out = [], {}, []
        for acts in stream:
            before = sorted(res)
            miss = [e for e in acts if e not in res]
            ev = []
            for _ in range(max(0, len(res) + len(miss) - C)):
                cand = [e for e in res if e not in acts]
                v = cand[0] if pol == 0 else min(cand, key=lambda e: (freq.get(e, 0), res.index(e), e))
                res.remove(v)
                ev.append(v)
            for e in acts:
                if e in res:
                    res.remove(e)
                res.append(e)
                freq[e] = freq.get(e, 0) + 1
            out.append((before, sorted(ev)))
        return out

    for assignment in itertools.product(range(4), repeat=6):
        acts = np.array(assignment, np.int64).reshape(6, 1)
        for pol in (0, 1):
            for C in (1, 2, 3):
                rb, ev = oracle.replay_policy(acts, 4, C, pol, 1.0, 1)
                for t, (before, evicted) in enumerate(straight([[a] for a in assignment], C, pol)):
                    assert np.flatnonzero(rb[t]).tolist() == before
                    assert np.flatnonzero(ev[t]).tolist() == evicted


def _ref_dump(obj):
    import json

    return json.dumps(obj, separators=(",", ":"))


def test_native_jsonl_long_traces_match_json_dumps():
    """Long traces go through the multi-threaded native path (> 64K lines): same bytes as the
    reference writers' json.dumps (traces.py:267-312, simulate.py:187-226) restated here."""
    import numpy as np

    from paper_2511_05814_b200.simulate import CacheEventLog, SimConfig, format_event_log
    from paper_2511_05814_b200.traces import ActivationTrace, ModelShape, SpeculationTrace, format_trace

    rng = np.random.default_rng(5)
    T, L, E, K = 3000, 32, 8, 2
    acts = np.sort(np.stack([rng.permutation(E)[:K] for _ in range(T * L)]), axis=1).reshape(T, L, K)
    shape = ModelShape(L, E, K)
    want = [_ref_dump({"kind": "activation", "num_layers": L, "num_experts": E, "top_k": K})]
    want += [_ref_dump({"t": t, "l": l, "a": acts[t, l].tolist()}) for t in range(T) for l in range(L)]
    assert format_trace(ActivationTrace(shape, acts)) == ("\n".join(want) + "\n").encode()
    g = np.sort(np.stack([rng.permutation(E)[:K] for _ in range(T * (L - 1))]), axis=1).reshape(T, L - 1, K)
    want = [_ref_dump({"kind": "speculation", "num_layers": L, "num_experts": E, "top_k": K})]
    want += [_ref_dump({"t": t, "l": j + 1, "g": g[t, j].tolist(), "a": acts[t, j + 1].tolist()})
             for t in range(T) for j in range(L - 1)]
    sp = SpeculationTrace(shape, g, np.ascontiguousarray(acts[:, 1:]))
    assert format_trace(sp) == ("\n".join(want) + "\n").encode()
    rb = (rng.random((L, T, E)) < 0.5).astype(np.uint8)
    ev = (rng.random((L, T, E)) < 0.2).astype(np.uint8)
    layers = tuple(range(L))
    log = CacheEventLog(config=SimConfig(policy=PolicyKind.parse("lfu-aged:0.5:16"), cache_size=4,
                                         warmup_tokens=7),
                        shape=shape, layers=layers,
                        activated={l: np.ascontiguousarray(acts[:, l]) for l in layers},
                        resident_before={l: rb[l] for l in layers},
                        evicted={l: ev[l] for l in layers}, num_tokens=T)
    want = [_ref_dump({"kind": "events", "policy": "lfu-aged:0.5:16", "cache_size": 4,
                       "num_layers": L, "num_experts": E, "top_k": K, "warmup_tokens": 7})]
    for t in range(T):
        for l in layers:
            a = set(acts[t, l].tolist())
            r = set(np.flatnonzero(rb[l, t]).tolist())
            want.append(_ref_dump({"t": t, "l": l, "cached": sorted(r), "hit": sorted(a & r),
                                   "miss": sorted(a - r), "evict": sorted(np.flatnonzero(ev[l, t]).tolist())}))
    assert format_event_log(log) == ("\n".join(want) + "\n").encode()
