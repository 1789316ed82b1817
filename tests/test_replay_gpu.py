"""K7 / policy_step on the GPU: bit-exact against the reference (golden streams generated
by moesim itself) and against the C oracle on the reference's KATs and exhaustive sets."""
import itertools

import numpy as np
import pytest

import oracle
from conftest import golden_streams, random_stream
from paper_2511_05814_b200 import kernels
from paper_2511_05814_b200.simulate import SimConfig, simulate
from paper_2511_05814_b200.errors import ConfigError
from paper_2511_05814_b200.policies import CacheState, PolicyKind, policy_step, warm_state
from paper_2511_05814_b200.traces import ActivationTrace, ModelShape

pytestmark = pytest.mark.gpu

POLICIES = [PolicyKind.lru(), PolicyKind.lfu(), PolicyKind.lfu_aged(0.5, 4), PolicyKind.opt()]


def test_replay_matches_reference_golden_streams():
    n = 0
    for E, K, C, T, code, df, dp, acts, rb, ev in golden_streams():
        grb, gev = kernels.replay_policy(acts, E, C, code, df, dp)
        assert np.array_equal(grb, rb) and np.array_equal(gev, ev), (E, K, C, T, code, df, dp)
        n += 1
    assert n == 2800


def test_replay_batched_layers_equal_single_layers(rng):
    for code, df, dp in [(0, 1.0, 1), (1, 1.0, 1), (2, 0.7, 3), (3, 1.0, 1)]:
        E, K, C, T, L = 8, 2, 4, 300, 12
        acts = np.stack([random_stream(rng, E, K, T) for _ in range(L)])
        rb, ev = kernels.replay_policy_layers(acts, E, C, code, df, dp)
        for l in range(L):
            orb, oev = oracle.replay_policy(acts[l], E, C, code, df, dp)
            assert np.array_equal(rb[l], orb) and np.array_equal(ev[l], oev)


def test_replay_large_expert_counts(rng):
    for E in (33, 64, 100, 256):
        K = min(8, E)
        C = int(rng.integers(K, E + 1))
        acts = random_stream(rng, E, K, 200)
        for code in range(4):
            got = kernels.replay_policy(acts, E, C, code, 0.5, 7)
            want = oracle.replay_policy(acts, E, C, code, 0.5, 7)
            assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1]), (E, code)


def test_exhaustive_4_to_the_6():
    """Criterion 04: all 4^6 single-expert traces x C in {1,2,3}, LRU and LFU, one launch
    per (policy, C) with every trace as its own layer."""
    allt = np.array(list(itertools.product(range(4), repeat=6)), np.int64).reshape(-1, 6, 1)
    for code in (0, 1):
        for C in (1, 2, 3):
            rb, ev = kernels.replay_policy_layers(allt, 4, C, code, 1.0, 1)
            for i in range(allt.shape[0]):
                orb, oev = oracle.replay_policy(allt[i], 4, C, code, 1.0, 1)
                assert np.array_equal(rb[i], orb) and np.array_equal(ev[i], oev)


def test_tie_break_kats():
    acts = np.array([[3, 5], [0, 1]], np.int64)
    for code in (0, 1):
        _, ev = kernels.replay_policy(acts, 8, 3, code, 1.0, 1)
        assert np.flatnonzero(ev[1]).tolist() == [3]
    acts = np.array([[1, 2], [0, 3], [1, 2]], np.int64)
    _, ev = kernels.replay_policy(acts, 4, 3, 3, 1.0, 1)
    assert np.flatnonzero(ev[1]).tolist() == [1]


def test_edge_cases():
    rb, ev = kernels.replay_policy(np.zeros((0, 2), np.int64), 8, 4, 0, 1.0, 1)
    assert rb.shape == (0, 8) and ev.shape == (0, 8)
    with pytest.raises(ConfigError):
        kernels.replay_policy(np.array([[0, 1, 2]], np.int64), 8, 2, 0, 1.0, 1)
    # C == K: every non-activated resident goes, whatever the policy
    acts = random_stream(np.random.default_rng(1), 8, 2, 50)
    outs = [kernels.replay_policy(acts, 8, 2, c, 0.5, 2) for c in range(4)]
    for o in outs[1:]:
        assert np.array_equal(o[0], outs[0][0]) and np.array_equal(o[1], outs[0][1])


def test_long_stream_lfu_aged_fp64_order():
    rng = np.random.default_rng(9)
    acts = random_stream(rng, 8, 2, 20000)
    for df, dp in [(0.3, 3), (0.9, 1), (0.999, 17)]:
        got = kernels.replay_policy(acts, 8, 4, 2, df, dp)
        want = oracle.replay_policy(acts, 8, 4, 2, df, dp)
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def _run(kind, C, stream):
    state, outs = warm_state(kind, C), []
    for i, a in enumerate(stream):
        fut = stream[i + 1:] if kind.name == "opt" else None
        state, o = policy_step(state, kind, a, fut)
        outs.append(o)
    return state, outs


class TestPolicyStepKats:
    def test_lru_textbook(self):
        state, outs = _run(PolicyKind.lru(), 4, [{0}, {1}, {2}, {3}, {4, 5}])
        assert outs[-1].evicted == {0, 1} and outs[-1].loaded == {4, 5}
        assert state.resident == {2, 3, 4, 5}

    def test_lru_hit_refresh(self):
        _, outs = _run(PolicyKind.lru(), 2, [{0}, {1}, {0}, {2}])
        assert outs[3].evicted == {1}

    def test_recency_is_resident_set(self):
        state, _ = _run(PolicyKind.lru(), 4, [{0, 1}, {2}])
        assert set(state.recency) == set(state.resident) and state.recency[0] == 2
        assert state.recency == (2, 1, 0)

    def test_lfu_displaces_despite_freq(self):
        s = CacheState(2, frozenset({0, 1}), (1, 0), {0: 5.0, 1: 1.0}, 6)
        _, o = policy_step(s, PolicyKind.lfu(), {2, 3})
        assert o.evicted == {0, 1} and o.loaded == {2, 3}

    def test_lfu_low_freq_first(self):
        _, outs = _run(PolicyKind.lfu(), 3, [{0, 1}, {0, 2}, {0, 1}, {3, 0}])
        assert outs[3].evicted == {2}

    def test_lfu_freq_tie_lru(self):
        s = CacheState(2, frozenset({3, 5}), (3, 5), {3: 2.0, 5: 2.0}, 4)
        _, o = policy_step(s, PolicyKind.lfu(), {1})
        assert o.evicted == {5}

    def test_freq_survives_eviction(self):
        state, _ = _run(PolicyKind.lfu(), 2, [{0, 1}, {2, 3}])
        assert state.freq[0] == 1.0

    def test_aged_decay(self):
        state, _ = _run(PolicyKind.lfu_aged(0.5, 2), 4, [{0}, {0}, {1}])
        assert state.freq == {0: 1.0, 1: 1.0}
        stream = [{0}] * 4 + [{1}, {2}, {3}]
        _, outs = _run(PolicyKind.lfu_aged(0.01, 4), 3, stream)
        assert outs[6].evicted == {0}
        _, outs = _run(PolicyKind.lfu(), 3, stream)
        assert outs[6].evicted == {1}

    def test_opt_belady(self):
        s = CacheState(2, frozenset({0, 1}), (1, 0), {}, 0)
        _, o = policy_step(s, PolicyKind.opt(), {2}, future=[{0}, {0}, {1}])
        assert o.evicted == {1}
        _, o = policy_step(s, PolicyKind.opt(), {2}, future=[{0}])
        assert o.evicted == {1}

    def test_opt_future_rules(self):
        s = warm_state(PolicyKind.opt(), 2)
        with pytest.raises(ConfigError):
            policy_step(s, PolicyKind.opt(), {0})
        with pytest.raises(ConfigError):
            policy_step(s, PolicyKind.lru(), {0}, future=[{0}])
        with pytest.raises(ConfigError):
            policy_step(warm_state(PolicyKind.lru(), 2), PolicyKind.lru(), {0, 1, 2})

    def test_input_not_mutated(self):
        s = CacheState(3, frozenset({0, 1, 2}), (2, 1, 0), {0: 2.0, 1: 1.0, 2: 3.0}, 5)
        snap = (s.resident, s.recency, dict(s.freq), s.step)
        outs = {policy_step(s, PolicyKind.lfu(), {3, 4})[1] for _ in range(3)}
        assert len(outs) == 1 and (s.resident, s.recency, s.freq, s.step) == snap


def test_policy_step_matches_replay(rng):
    for _ in range(40):
        E = int(rng.integers(2, 9))
        K = int(rng.integers(1, E + 1))
        C = int(rng.integers(K, E + 1))
        T = int(rng.integers(1, 20))
        acts = random_stream(rng, E, K, T)
        stream = [set(r.tolist()) for r in acts]
        for kind in POLICIES:
            rb, ev = kernels.replay_policy(acts, E, C, *kind.device_params())
            _, outs = _run(kind, C, stream)
            for t, o in enumerate(outs):
                assert frozenset(np.flatnonzero(rb[t]).tolist()) == o.resident_before
                assert frozenset(np.flatnonzero(ev[t]).tolist()) == o.evicted
                assert len(o.evicted) == max(0, len(o.resident_before) + len(o.misses) - C)


def test_simulate_on_gpu_layer_independence_and_compulsory(rng):
    shape = ModelShape(4, 8, 2)
    acts = np.stack([random_stream(rng, 8, 2, 25) for _ in range(4)], axis=1)
    tr = ActivationTrace(shape, acts)
    full = simulate(tr, SimConfig(PolicyKind.lru(), 4))
    for l in range(4):
        solo = simulate(tr, SimConfig(PolicyKind.lru(), 4, layers=(l,)))
        assert np.array_equal(solo.resident_before[l], full.resident_before[l])
    for pol in ("lru", "lfu", "lfu-aged:0.5:16", "opt"):
        log = simulate(tr, SimConfig(PolicyKind.parse(pol), 8))
        for l in range(4):
            assert int(log.miss_counts(l).sum()) == len(np.unique(acts[:, l, :]))
    with pytest.raises(ConfigError):
        simulate(tr, SimConfig(PolicyKind.lru(), 1))
    with pytest.raises(ConfigError):
        simulate(tr, SimConfig(PolicyKind.lru(), 4, layers=(7,)))


def test_reference_suite_replay_calls():
    """Every distinct replay call of the reference's own test suite (26.5 k, all four policies,
    the reference's outputs recorded by tests/golden/make_refsuite_golden.py), replayed on the
    GPU in batches of equal-shaped calls (one warp per call): bit-exact."""
    from collections import defaultdict

    from conftest import refsuite_calls

    groups = defaultdict(list)
    for acts, E, C, pol, df, dp, rb, ev in refsuite_calls():
        groups[(acts.shape, E, C, pol, df, dp)].append((acts, rb, ev))
    n = 0
    for ((T, K), E, C, pol, df, dp), items in groups.items():
        if T == 0:
            n += len(items)
            continue
        acts = np.stack([a for a, _, _ in items])
        grb, gev = kernels.replay_policy_layers(acts, E, C, pol, df, dp)
        for i, (_, rb, ev) in enumerate(items):
            assert np.array_equal(grb[i], rb) and np.array_equal(gev[i], ev), (T, K, E, C, pol, df, dp)
        n += len(items)
    assert n > 26000


def test_reference_suite_policy_steps():
    """Every distinct policy_step call of the reference's own test suite (5,084: all four
    policies, KATs, validation errors), through the GPU step: identical state, outcome sets,
    and the same error class where the reference raised one."""
    from conftest import refsuite_policy_steps

    from paper_2511_05814_b200 import errors

    n = 0
    for rec in refsuite_policy_steps():
        s = rec["state"]
        st = CacheState(capacity=s["capacity"], resident=frozenset(s["resident"]),
                        recency=tuple(s["recency"]), freq={e: f for e, f in s["freq"]}, step=s["step"])
        fut = None if rec["future"] is None else [frozenset(f) for f in rec["future"]]
        kind = PolicyKind.parse(rec["kind"])
        if "error" in rec:
            with pytest.raises(getattr(errors, rec["error"], Exception)):
                policy_step(st, kind, rec["activated"], fut)
        else:
            st2, out = policy_step(st, kind, rec["activated"], fut)
            r = rec["result"]
            assert st2.capacity == r["state"]["capacity"] and st2.step == r["state"]["step"], rec
            assert sorted(st2.resident) == r["state"]["resident"], rec
            assert list(st2.recency) == r["state"]["recency"], rec
            assert sorted([e, f] for e, f in st2.freq.items()) == r["state"]["freq"], rec
            for k in ("hits", "misses", "evicted", "loaded", "resident_before", "resident_after"):
                assert sorted(getattr(out, k)) == r[k], (k, rec)
        n += 1
    assert n > 5000
