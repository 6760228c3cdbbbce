"""CUDA step engine vs the CPU oracle (and the reference build where cheap).

Bar (north_star / SURVEY §8): per-step loads, max, dt, clock, active counts
and per-request assignments bit-exact; integer metric sums exact;
energy and TPOT within 1e-9 relative (their summation order / libm pow differ).
All calls go through the C ABI (libbfsim_gpu.so) via paper_2601_17855_b200.host.
"""
import numpy as np
import pytest

from paper_2601_17855_b200 import abi, host

pytestmark = pytest.mark.gpu

EXACT = ("avg_imbalance", "throughput", "imb_total", "total_workload", "eta_sum")
TOL = 1e-9


@pytest.fixture(scope="module")
def ctx():
    c = host.Context(0)
    yield c
    c.close()


def _rel(a, b):
    return abs(a - b) / max(abs(a), abs(b), 1e-300)


def check_poisson(orc, br, i, sc, tr):
    rc, res, st, rq = orc.run_poisson(sc, tr)
    g = br.res[i]
    assert int(g["status"]) == int(res["status"])
    assert int(g["steps_run"]) == int(res["steps_run"])
    assert int(g["completed"]) == int(res["completed"])
    gs = br.steps(i)
    np.testing.assert_array_equal(gs["loads"], st.loads)
    np.testing.assert_array_equal(gs["dt"], st.dt)
    np.testing.assert_array_equal(gs["clock_start"], st.clock_start)
    np.testing.assert_array_equal(gs["max_load"], st.max_load)
    np.testing.assert_array_equal(gs["active_count"], st.active_count)
    gr = br.requests(i, tr.shape[0])
    for k in ("arrival_step", "start_step", "worker", "admit_clock", "finish_clock"):
        np.testing.assert_array_equal(gr[k], rq[k], err_msg=k)
    for k in ("imb_total_i", "total_workload_i", "tokens_i", "records"):
        assert int(g[k]) == int(res[k]), k
    assert float(g["clock"]) == float(res["clock"])
    for k in EXACT:
        assert float(g[k]) == float(res[k]), k
    for k in ("energy", "tpot"):
        assert _rel(float(g[k]), float(res[k])) <= TOL, (k, float(g[k]), float(res[k]))


def _poisson_batch(ctx, scs, traces):
    pool = host.InputPool(traces)
    for i, s in enumerate(scs):
        s["input_id"] = i
    return ctx.run_batch(np.array(scs, abi.scenario_dtype), pool, emit_steps=True, emit_requests=True)


@pytest.mark.parametrize("policy", [abi.FCFS, abi.JSQ, abi.BFIO_GREEDY])
def test_poisson_small_grid(ctx, orc, policy):
    scs, trs = [], []
    for H in (0, 1, 5):
        for drift in (0.0, 1.0, 2.0):
            for la in (abi.PERFECT, abi.TRUNCATED):
                tr = host.sample_instance(13 + H, rate=60.0, duration=4.0, s_max=16, p=0.15)
                scs.append(abi.scenario(policy=policy, workers=4, batch=4, horizon=H, drift=drift, lookahead=la))
                trs.append(tr)
    br = _poisson_batch(ctx, scs, trs)
    for i, (s, t) in enumerate(zip(br.scen, trs)):
        check_poisson(orc, br, i, s, t)


def test_poisson_random_batch(ctx, orc):
    rng = np.random.default_rng(17855)
    scs, trs = [], []
    for t in range(96):
        G = int(rng.integers(1, 70))
        B = int(rng.integers(1, 20))
        H = int(rng.choice([0, 0, 1, 3, 8, 20]))
        pol = int(rng.choice([abi.FCFS, abi.JSQ, abi.BFIO_GREEDY]))
        la = int(rng.choice([abi.PERFECT, abi.TRUNCATED]))
        drift = float(rng.choice([0.0, 1.0, 2.0]))
        rate = float(rng.uniform(3, 25)) * G * B / 8.0
        s_max = int(rng.choice([2, 7, 64, 100, 700]))
        tr = host.sample_instance(int(rng.integers(1, 1 << 30)), rate=rate, duration=float(rng.uniform(0.3, 2.0)),
                                  s_max=s_max, p=float(rng.uniform(0.03, 0.4)))
        scs.append(abi.scenario(policy=pol, workers=G, batch=B, horizon=H, drift=drift, lookahead=la))
        trs.append(tr)
    br = _poisson_batch(ctx, scs, trs)
    for i, (s, t) in enumerate(zip(br.scen, trs)):
        check_poisson(orc, br, i, s, t)


def test_poisson_c1(ctx, orc, ref):
    """BASELINE C1: G=8, B=64, lambda=2000/s, 1 s, seed 1; fcfs vs bfio-greedy H=0/20,
    checked against the oracle and the reference build."""
    tr = host.sample_instance(1, rate=2000.0, duration=1.0, s_max=64, p=0.02)
    assert tr.shape[0] == 1957
    scs = [abi.scenario(policy=p, workers=8, batch=64, horizon=H) for p, H in
           ((abi.FCFS, 0), (abi.JSQ, 0), (abi.BFIO_GREEDY, 0), (abi.BFIO_GREEDY, 20))]
    br = _poisson_batch(ctx, scs, [tr] * 4)
    for i in range(4):
        check_poisson(orc, br, i, br.scen[i], tr)
        rc, err, (st, rq, m, done) = ref.run_poisson(br.scen[i], tr)
        np.testing.assert_array_equal(br.steps(i)["loads"], st.loads)
        for k in EXACT:
            assert float(br.res[i][k]) == m[k]


def test_poisson_c2_slice(ctx, orc):
    """BASELINE C2 shape (G=16, B=64, lambda=4000/s, 2.5 s): 4 seeds x {greedy H0, jsq}."""
    scs, trs = [], []
    for seed in (1, 2, 3, 4):
        tr = host.sample_instance(seed, rate=4000.0, duration=2.5, s_max=64, p=0.02)
        for p in (abi.BFIO_GREEDY, abi.JSQ):
            scs.append(abi.scenario(policy=p, workers=16, batch=64))
            trs.append(tr)
    br = _poisson_batch(ctx, scs, trs)
    for i, (s, t) in enumerate(zip(br.scen, trs)):
        check_poisson(orc, br, i, s, t)


def test_poisson_edges(ctx, orc):
    one = np.zeros(1, abi.request_dtype)
    one[0] = (0.0, 2, 100)
    late = np.zeros(1, abi.request_dtype)
    late[0] = (5.0, 3, 2)
    hand = np.zeros(1, abi.request_dtype)
    hand[0] = (0.0, 2, 3)
    two = np.zeros(2, abi.request_dtype)
    two[0] = (0.0, 3, 4)
    two[1] = (0.0, 2, 2)
    empty = np.zeros(0, abi.request_dtype)
    cases = [
        (abi.scenario(workers=1, batch=1, max_steps=10), one),       # partial (engine_test.cpp:111-118)
        (abi.scenario(workers=2, batch=1), late),                    # idle steps (engine_test.cpp:47-54)
        (abi.scenario(workers=1, batch=1), hand),                    # loads 2,3,4 (engine_test.cpp:82-94)
        (abi.scenario(workers=2, batch=1), two),                     # x+o-1 (engine_test.cpp:142-154)
        (abi.scenario(workers=2, batch=2), empty),                   # no steps (engine_test.cpp:75-80)
        (abi.scenario(workers=3, batch=2, policy=abi.BFIO_GREEDY, horizon=4), hand),
    ]
    br = _poisson_batch(ctx, [c[0] for c in cases], [c[1] for c in cases])
    for i, (s, t) in enumerate(cases):
        check_poisson(orc, br, i, br.scen[i], t)
    assert int(br.res[0]["status"]) == abi.PARTIAL
    np.testing.assert_array_equal(br.steps(2)["loads"][:, 0], [2.0, 3.0, 4.0])
    assert int(br.res[4]["steps_run"]) == 0 and int(br.res[4]["flags"]) & abi.FLAG_EMPTY


def _ovl_check(orc, br, i, sc, stream, s_max):
    rc, res, st, per, tm = orc.run_overloaded(sc, stream, s_max)
    g = br.res[i]
    assert int(g["status"]) == abi.OK
    assert int(g["consumed"]) == int(res["consumed"])
    gs = br.steps(i)
    np.testing.assert_array_equal(gs["loads"], st.loads)
    np.testing.assert_array_equal(gs["dt"], st.dt)
    np.testing.assert_array_equal(gs["clock_start"], st.clock_start)
    np.testing.assert_array_equal(gs["active_count"], st.active_count)
    n = int(res["consumed"])
    gr = br.requests(i, stream.shape[0])
    np.testing.assert_array_equal(gr["start_step"][:n], per["start_step"][:n])
    np.testing.assert_array_equal(gr["worker"][:n], per["worker"][:n])
    for k in ("imb_total_i", "total_workload_i", "tokens_i", "records", "completed"):
        assert int(g[k]) == int(res[k]), k
    for k in EXACT:
        assert float(g[k]) == float(res[k]), k
    for k in ("energy", "tpot"):
        assert _rel(float(g[k]), float(res[k])) <= TOL, k


def test_overloaded_random_batch(ctx, orc):
    rng = np.random.default_rng(606)
    scs, streams, smaxes = [], [], []
    for t in range(48):
        G = int(rng.integers(1, 40))
        B = int(rng.integers(1, 17))
        H = int(rng.choice([0, 0, 2, 20]))
        pol = int(rng.choice([abi.FCFS, abi.JSQ, abi.BFIO_GREEDY]))
        s_max = int(rng.choice([2, 8, 64, 200]))
        p = float(rng.uniform(0.02, 0.4))
        seed = int(rng.integers(1, 1 << 31))
        steps, warm = int(rng.integers(10, 300)), int(rng.integers(0, 60))
        sc = abi.scenario(mode=abi.OVERLOADED, policy=pol, workers=G, batch=B, horizon=H,
                          drift=float(rng.choice([0.0, 1.0])), steps=steps, warmup=warm, seed=seed,
                          backlog=float(rng.choice([1.0, 2.0])))
        n = int(G * B * (3 + (steps + warm) * p * 1.6)) + 4096
        streams.append(host.sample_stream(seed, n, s_max=s_max, p=p))
        scs.append(sc)
        smaxes.append(s_max)
    pool = host.InputPool(streams)
    for i, s in enumerate(scs):
        s["input_id"] = i
    br = ctx.run_batch(np.array(scs, abi.scenario_dtype), pool, emit_steps=True, emit_requests=True)
    for i in range(len(scs)):
        _ovl_check(orc, br, i, br.scen[i], streams[i], smaxes[i])


def test_rejections(ctx):
    tr = host.sample_instance(3, rate=100.0, duration=1.0)
    pool = host.InputPool([tr])
    for bad in (dict(policy=abi.BFIO_EXACT), dict(drift=0.1), dict(drift=-1.0), dict(workers=0),
                dict(gamma=1.0), dict(per_token=0.0)):
        with pytest.raises(host.InvalidArgument):
            ctx.run_batch(np.array([abi.scenario(**bad)], abi.scenario_dtype), pool)
    # single-class prefill never satisfies Def. 1
    st = host.sample_stream(5, 5000, s_max=1, prefill_kind=1)
    with pytest.raises(host.InvalidArgument):
        ctx.run_batch(np.array([abi.scenario(mode=abi.OVERLOADED, steps=10, warmup=0)], abi.scenario_dtype),
                      host.InputPool([st]))


def test_large_worker_counts(ctx, orc):
    """G > 256 (32-worker-per-lane variant; BASELINE C4 sweeps G up to 1024)."""
    scs, trs = [], []
    for G, B, pol, H in ((300, 4, abi.BFIO_GREEDY, 0), (600, 2, abi.FCFS, 0), (1024, 2, abi.JSQ, 0),
                         (1024, 1, abi.BFIO_GREEDY, 0), (513, 3, abi.BFIO_GREEDY, 3)):
        scs.append(abi.scenario(policy=pol, workers=G, batch=B, horizon=H))
        trs.append(host.sample_instance(G + B, rate=G * B * 2.5, duration=0.6, s_max=64, p=0.1))
    br = _poisson_batch(ctx, scs, trs)
    for i, (s, t) in enumerate(zip(br.scen, trs)):
        check_poisson(orc, br, i, s, t)
    # overloaded at G = 1024 (C4 shape, short)
    stream = host.sample_stream(9, 200000, s_max=64, p=0.05)
    so = [abi.scenario(mode=abi.OVERLOADED, policy=p, workers=1024, batch=4, steps=40, warmup=10, seed=9)
          for p in (abi.FCFS, abi.BFIO_GREEDY)]
    for s in so:
        s["input_id"] = 0
    br = ctx.run_batch(np.array(so, abi.scenario_dtype), host.InputPool([stream]), emit_steps=True,
                       emit_requests=True)
    for i in range(2):
        _ovl_check(orc, br, i, br.scen[i], stream, 64)


def test_poisson_noisy_random_batch(ctx, orc):
    """Noisy lookahead (make_preview policies.hpp:67-90; per-simulation
    mt19937_64 draws in the order of engine.hpp:131/204-231) on the device:
    bit-exact against the oracle, which is pinned to the reference build in
    tests/test_oracle_vs_ref.py. Includes the variants where the draws are
    unobservable (fcfs/jsq, H = 0, sigma = 0)."""
    rng = np.random.default_rng(2026)
    scs, trs = [], []
    for t in range(80):
        G = int(rng.integers(1, 70))
        B = int(rng.integers(1, 20))
        H = int(rng.choice([1, 2, 3, 8, 20, 20]))
        pol = abi.BFIO_GREEDY
        if t % 10 == 9:
            pol = int(rng.choice([abi.FCFS, abi.JSQ]))
        if t % 10 == 8:
            H = 0
        sigma = float(rng.choice([0.0, 0.5, 2.0, 2.0, 5.0, 40.0])) if t % 10 != 7 else 0.0
        drift = float(rng.choice([0.0, 1.0, 1.0, 2.0]))
        rate = float(rng.uniform(3, 25)) * G * B / 8.0
        s_max = int(rng.choice([2, 7, 64, 100, 700]))
        tr = host.sample_instance(int(rng.integers(1, 1 << 30)), rate=rate, duration=float(rng.uniform(0.3, 2.0)),
                                  s_max=s_max, p=float(rng.uniform(0.03, 0.4)))
        scs.append(abi.scenario(policy=pol, workers=G, batch=B, horizon=H, drift=drift, lookahead=abi.NOISY,
                                noise_sigma=sigma, seed=int(rng.integers(0, 1 << 62))))
        trs.append(tr)
    br = _poisson_batch(ctx, scs, trs)
    for i, (s, t) in enumerate(zip(br.scen, trs)):
        assert not int(br.res[i]["flags"]) & abi.FLAG_NOISE_NEAR_TIE
        check_poisson(orc, br, i, s, t)


def test_poisson_c3_slice(ctx, orc, ref):
    """BASELINE C3 shape (G=64, B=64, lambda=8000/s, bfio-greedy H=20 with
    Noisy sigma=2), on a 1.5 s prefix of the trace, 3 seeds; seed 1 also
    against the reference build."""
    scs, trs = [], []
    for seed in (1, 2, 3):
        tr = host.sample_instance(seed, rate=8000.0, duration=1.5, s_max=64, p=0.02)
        scs.append(abi.scenario(policy=abi.BFIO_GREEDY, workers=64, batch=64, horizon=20,
                                lookahead=abi.NOISY, noise_sigma=2.0, seed=seed))
        trs.append(tr)
    br = _poisson_batch(ctx, scs, trs)
    for i, (s, t) in enumerate(zip(br.scen, trs)):
        check_poisson(orc, br, i, s, t)
    rc, err, (st, rq, m, done) = ref.run_poisson(br.scen[0], trs[0])
    np.testing.assert_array_equal(br.steps(0)["loads"], st.loads)
    for k in EXACT:
        assert float(br.res[0][k]) == m[k]


def test_calendar_large_slot_counts(ctx, orc):
    """G*B > 4096 switches retirement from the per-step finish-step scan to the
    completion calendar (per-owner-lane lists per finish step); every policy,
    the perfect/truncated lookahead window, noisy lists, and run_overloaded."""
    scs, trs = [], []
    cases = ((128, 40, abi.FCFS, 0, abi.PERFECT), (100, 50, abi.JSQ, 0, abi.PERFECT),
             (96, 48, abi.BFIO_GREEDY, 0, abi.PERFECT), (64, 80, abi.BFIO_GREEDY, 6, abi.PERFECT),
             (70, 64, abi.BFIO_GREEDY, 20, abi.TRUNCATED), (300, 16, abi.BFIO_GREEDY, 3, abi.PERFECT),
             (64, 72, abi.BFIO_GREEDY, 20, abi.NOISY), (520, 9, abi.BFIO_GREEDY, 0, abi.PERFECT))
    for t, (G, B, pol, H, la) in enumerate(cases):
        scs.append(abi.scenario(policy=pol, workers=G, batch=B, horizon=H, lookahead=la,
                                noise_sigma=2.0 if la == abi.NOISY else 0.0, seed=t + 1))
        trs.append(host.sample_instance(100 + t, rate=G * B * 1.5, duration=0.8, s_max=64, p=0.05))
    br = _poisson_batch(ctx, scs, trs)
    for i, (s, t) in enumerate(zip(br.scen, trs)):
        check_poisson(orc, br, i, s, t)
    stream = host.sample_stream(21, 400000, s_max=64, p=0.05)
    so = [abi.scenario(mode=abi.OVERLOADED, policy=p, workers=1024, batch=8, horizon=H, steps=40, warmup=10,
                       seed=21) for p, H in ((abi.FCFS, 0), (abi.JSQ, 0), (abi.BFIO_GREEDY, 0), (abi.BFIO_GREEDY, 2))]
    for s in so:
        s["input_id"] = 0
    br = ctx.run_batch(np.array(so, abi.scenario_dtype), host.InputPool([stream]), emit_steps=True,
                       emit_requests=True)
    for i in range(len(so)):
        _ovl_check(orc, br, i, br.scen[i], stream, 64)


def test_pinned_zero_copy_sinks_match(ctx):
    """Page-locked sinks: step records written by the kernel directly
    (zero-copy), request timings copied out per trajectory; both equal the
    staged copy path."""
    trs = [host.sample_instance(s, rate=1500.0, duration=1.0, s_max=64, p=0.05) for s in (1, 2)]
    scs = np.array([abi.scenario(policy=p, workers=8, batch=16, horizon=H, input_id=i)
                    for i in range(2) for p, H in ((abi.BFIO_GREEDY, 0), (abi.BFIO_GREEDY, 5), (abi.JSQ, 0))],
                   abi.scenario_dtype)
    pool = host.InputPool(trs)
    ref = ctx.run_batch(scs, pool, emit_steps=True, emit_requests=True)
    K = ref.res["steps_run"].astype(np.int64)
    pb = host.PinnedBatch(ctx, scs, pool, step_capacity=np.maximum(K, 1))
    res = pb.run()
    np.testing.assert_array_equal(res["imb_total_i"], ref.res["imb_total_i"])
    off = 0
    for i in range(len(scs)):
        k = int(K[i])
        np.testing.assert_array_equal(pb.steps["clock_start"][off:off + k], ref.steps(i)["clock_start"])
        np.testing.assert_array_equal(pb.steps["active_count"][off:off + k], ref.steps(i)["active_count"])
        off += max(k, 1)
    G = 8
    np.testing.assert_array_equal(pb.steps["loads"][: int(K[0]) * G].reshape(-1, G), ref.steps(0)["loads"])
    # request timings: staged in HBM, copied out per trajectory by its warp
    n0 = trs[0].shape[0]
    for key in ("arrival_step", "start_step", "worker", "admit_clock", "finish_clock"):
        np.testing.assert_array_equal(pb.reqs[key][:n0], ref.requests(0, n0)[key], err_msg=key)
        np.testing.assert_array_equal(pb.reqs[key][-trs[1].shape[0]:], ref.requests(5, trs[1].shape[0])[key],
                                      err_msg=key)


def test_empirical_inputs(ctx, orc, ref):
    """Traces / streams from Empirical prefill and decode lists
    (workload.hpp:109-118, 185-193) through the engine: Poisson against the
    oracle, run_overloaded against the unmodified reference drawing the same
    lists itself (ref_set_empirical)."""
    pv, dv = [3, 17, 17, 64, 1, 250], [1, 2, 5, 40, 40, 300, 7]
    tr = host.sample_instance(4, rate=900.0, duration=1.5, prefill_values=pv, decode_values=dv)
    scs = [abi.scenario(policy=p, workers=8, batch=12, horizon=H) for p, H in
           ((abi.FCFS, 0), (abi.BFIO_GREEDY, 0), (abi.BFIO_GREEDY, 6))]
    br = _poisson_batch(ctx, scs, [tr] * 3)
    for i in range(3):
        check_poisson(orc, br, i, br.scen[i], tr)
    ref.set_empirical(pv, dv)
    stream = host.sample_stream(11, 60000, prefill_values=pv, decode_values=dv)
    so = abi.scenario(mode=abi.OVERLOADED, policy=abi.BFIO_GREEDY, workers=8, batch=16, horizon=4, steps=80,
                      warmup=20, seed=11, input_id=0)
    br = ctx.run_batch(np.array([so], abi.scenario_dtype), host.InputPool([stream]), emit_steps=True)
    rc, err, (st, rq, m, done) = ref.run_overloaded(br.scen[0], s_max=250, prefill_kind=2, decode_kind=2)
    assert rc == 0, err
    # the reference keeps the records after warm-up (oracle.hpp:229-241); the sink has every step
    np.testing.assert_array_equal(br.steps(0)["loads"][-st.loads.shape[0]:], st.loads)
    for k in EXACT:
        assert float(br.res[0][k]) == m[k], k
