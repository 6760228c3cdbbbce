"""The plain-C restatement (oracle/liboracle.so) against the UNMODIFIED
reference headers (oracle/_ref/libbfsim_ref.so): bit-exact step series,
request timings, admitted/completed lists and MetricsReport.

This pins the oracle before any GPU result is compared with it.
"""
import numpy as np
import pytest

from oracle.oracle import derive_lists
from paper_2601_17855_b200 import abi


def _cmp_poisson(ref, orc, sc, tr):
    rc, err, out = ref.run_poisson(sc, tr)
    assert rc == 0, err
    st, rq, metrics, completed_all = out
    rc2, res, st2, rq2 = orc.run_poisson(sc, tr)
    assert rc2 in (abi.OK, abi.PARTIAL)
    assert completed_all == (rc2 == abi.OK)
    K = len(st.loads)
    assert int(res["steps_run"]) == K
    np.testing.assert_array_equal(st2.loads, st.loads)
    np.testing.assert_array_equal(st2.dt, st.dt)
    np.testing.assert_array_equal(st2.clock_start, st.clock_start)
    np.testing.assert_array_equal(st2.max_load, st.max_load)
    np.testing.assert_array_equal(st2.active_count, st.active_count)
    np.testing.assert_array_equal(rq2["arrival_step"], rq["arrival_step"])
    np.testing.assert_array_equal(rq2["start_step"], rq["start_step"])
    np.testing.assert_array_equal(rq2["admit_clock"], rq["admit_clock"])
    np.testing.assert_array_equal(rq2["finish_clock"], rq["finish_clock"])
    rq2 = dict(rq2, decode=tr["decode"])
    adm, comp = derive_lists(rq2, K)
    assert adm == st.admitted
    assert comp == st.completed
    if metrics is None:
        assert int(res["flags"]) & abi.FLAG_EMPTY
    else:
        for k in abi.METRIC_FIELDS:
            assert float(res[k]) == metrics[k], k


@pytest.mark.parametrize("policy", [abi.FCFS, abi.JSQ, abi.BFIO_GREEDY])
@pytest.mark.parametrize("H", [0, 1, 5])
@pytest.mark.parametrize("drift", [0.0, 1.0, 2.0])
def test_poisson_small(ref, orc, policy, H, drift):
    tr = ref.sample_instance(s_max=16, p=0.15, rate=60, duration=4.0, seed=13 + H)
    sc = abi.scenario(policy=policy, workers=4, batch=4, horizon=H, drift=drift)
    _cmp_poisson(ref, orc, sc, tr)


def test_poisson_random_configs(ref, orc):
    rng = np.random.default_rng(2601)
    for t in range(60):
        G = int(rng.integers(1, 13))
        B = int(rng.integers(1, 13))
        H = int(rng.choice([0, 1, 3, 8, 20]))
        pol = int(rng.choice([abi.FCFS, abi.JSQ, abi.BFIO_GREEDY]))
        la = int(rng.choice([abi.PERFECT, abi.TRUNCATED, abi.NOISY]))
        drift = float(rng.choice([0.0, 1.0, 2.0]))
        rate = float(rng.uniform(5, 20)) * G * B / 8.0
        tr = ref.sample_instance(s_max=int(rng.integers(2, 65)), p=float(rng.uniform(0.03, 0.4)),
                                 rate=rate, duration=float(rng.uniform(0.5, 3.0)), seed=int(rng.integers(1, 1 << 30)))
        sc = abi.scenario(policy=pol, workers=G, batch=B, horizon=H, drift=drift, lookahead=la,
                          noise_sigma=float(rng.choice([0.5, 2.0])), seed=int(rng.integers(0, 1 << 40)))
        _cmp_poisson(ref, orc, sc, tr)


def test_poisson_c1_overloaded_trace(ref, orc):
    """BASELINE config C1: G=8, B=64, lambda=2000/s for 1 s, seed 1 (N=1,957)."""
    tr = ref.sample_instance(s_max=64, p=0.02, rate=2000.0, duration=1.0, seed=1)
    assert tr.shape[0] == 1957
    for pol, H in ((abi.BFIO_GREEDY, 0), (abi.BFIO_GREEDY, 20), (abi.FCFS, 0)):
        _cmp_poisson(ref, orc, abi.scenario(policy=pol, workers=8, batch=64, horizon=H), tr)


def test_poisson_max_steps_partial(ref, orc):
    tr = np.zeros(1, abi.request_dtype)
    tr[0] = (0.0, 2, 100)
    sc = abi.scenario(workers=1, batch=1, max_steps=10)
    _cmp_poisson(ref, orc, sc, tr)


def test_poisson_empty(ref, orc):
    tr = np.zeros(0, abi.request_dtype)
    sc = abi.scenario(workers=2, batch=2)
    rc, res, st, rq = orc.run_poisson(sc, tr)
    assert rc == abi.OK and int(res["steps_run"]) == 0
    assert int(res["flags"]) & abi.FLAG_EMPTY


def _stream_for(seed, n, s_max, p):
    from paper_2601_17855_b200 import host

    return host.sample_stream(seed, n, s_max=s_max, p=p)


def test_overloaded_vs_ref(ref, orc):
    """run_overloaded restated over the pre-generated stream."""
    from paper_2601_17855_b200 import host

    rng = np.random.default_rng(7)
    for t in range(24):
        G = int(rng.integers(1, 9))
        B = int(rng.integers(1, 9))
        H = int(rng.choice([0, 2, 20]))
        pol = int(rng.choice([abi.FCFS, abi.JSQ, abi.BFIO_GREEDY]))
        s_max = int(rng.integers(2, 65))
        p = float(rng.uniform(0.05, 0.4))
        drift = float(rng.choice([0.0, 1.0]))
        seed = int(rng.integers(1, 1 << 31))
        sc = abi.scenario(mode=abi.OVERLOADED, policy=pol, workers=G, batch=B, horizon=H, drift=drift,
                          steps=int(rng.integers(20, 200)), warmup=int(rng.integers(0, 50)), seed=seed,
                          backlog=float(rng.choice([1.0, 1.5])))
        rc, err, out = ref.run_overloaded(sc, s_max=s_max, p=p)
        assert rc == 0, err
        st, tm, metrics, _ = out
        stream = host.sample_stream(seed, 200000, s_max=s_max, p=p)
        rc2, res, st2, per, t2 = orc.run_overloaded(sc, stream, s_max)
        assert rc2 == abi.OK
        W = int(sc["warmup"])
        np.testing.assert_array_equal(st2.loads[W:], st.loads)
        np.testing.assert_array_equal(st2.dt[W:], st.dt)
        np.testing.assert_array_equal(st2.clock_start[W:], st.clock_start)
        np.testing.assert_array_equal(st2.active_count[W:], st.active_count)
        np.testing.assert_array_equal(t2["id"], tm["id"])
        np.testing.assert_array_equal(t2["admit_clock"], tm["admit_clock"])
        np.testing.assert_array_equal(t2["finish_clock"], tm["finish_clock"])
        for k in abi.METRIC_FIELDS:
            assert float(res[k]) == metrics[k], k


@pytest.mark.parametrize("policy", [abi.FCFS, abi.JSQ, abi.BFIO_GREEDY])
def test_assign_operator_random_steps(ref, orc, policy):
    """assign() on random steps, the shape of tests/policies_test.cpp:27-55."""
    rng = np.random.default_rng(53 + policy)
    for t in range(1500):
        H = int(rng.integers(0, 3))
        G = int(rng.integers(1, 5))
        n = int(rng.integers(0, 9))
        caps = rng.integers(0, 4, G).astype(np.int32)
        cnt = rng.integers(0, 3, G).astype(np.int32)
        fut = rng.integers(0, 20, (G, H + 1)).astype(np.float64)
        pv = rng.integers(0, 10, (n, H + 1)).astype(np.float64)
        rc, a, _ = ref.assign(policy, pv, caps, cnt, fut, H)
        rc2, b = orc.assign(policy, pv, caps, cnt, fut, H)
        assert rc == 0 and rc2 == 0
        assert a == b, (t, a, b)
