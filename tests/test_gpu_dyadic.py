"""Dyadic constant drift d = m / 2^e (hard part 2) on the GPU
path, against the unmodified reference build (oracle/_ref).

The reference builds each job's profile sequentially in fp64
(drift_profile, workload.hpp:73-85); for a dyadic d every partial sum is
exact, so the engine runs the integer problem scaled by 2^e (capi.cu
dyadic_drift) and must reproduce the reference's loads, dt, clocks, request
timings and MetricsReport bit for bit (energy / TPOT within 1e-9, as for
integer drift). Non-dyadic drift is rejected with code 1."""
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


def _check_vs_ref(br, i, st, rq, m, n_req=None, tail=False):
    g = br.steps(i)
    for k in ("loads", "dt", "clock_start", "max_load", "active_count"):
        got = g[k][-st.loads.shape[0]:] if tail else g[k]
        np.testing.assert_array_equal(got, getattr(st, k), err_msg=f"scenario {i}: {k}")
    res = br.res[i]
    for k in EXACT:
        assert float(res[k]) == m[k], (i, k, float(res[k]), m[k])
    for k in ("energy", "tpot"):
        assert _rel(float(res[k]), m[k]) <= TOL, (i, k)
    if n_req is not None:
        gr = br.requests(i, n_req)
        ids = rq["id"]
        np.testing.assert_array_equal(gr["admit_clock"][ids], rq["admit_clock"], err_msg=f"scenario {i}: admit")
        done = rq["completed"].astype(bool)
        np.testing.assert_array_equal(gr["finish_clock"][ids[done]], rq["finish_clock"][done],
                                      err_msg=f"scenario {i}: finish")


def test_poisson_dyadic_vs_reference(ctx, ref):
    """Every policy / lookahead mode at dyadic drifts; one trace shared by an
    integer-drift and several dyadic-drift scenarios (the scaled copies are
    per (input, shift))."""
    rng = np.random.default_rng(2601)
    trs = [host.sample_instance(s, rate=r, duration=1.2, s_max=sm, p=p)
           for s, r, sm, p in ((3, 900.0, 64, 0.05), (4, 2500.0, 16, 0.1), (5, 400.0, 700, 0.08))]
    combos = [(abi.FCFS, 0, abi.PERFECT), (abi.JSQ, 0, abi.PERFECT), (abi.BFIO_GREEDY, 0, abi.PERFECT),
              (abi.BFIO_GREEDY, 3, abi.PERFECT), (abi.BFIO_GREEDY, 8, abi.TRUNCATED),
              (abi.BFIO_GREEDY, 6, abi.NOISY)]
    drifts = (0.5, 0.25, 0.75, 1.5, 0.125, 3.0625, 1.0, 0.0)
    rows, tid = [], []
    for j, d in enumerate(drifts):
        for pol, H, la in combos:
            t = int(rng.integers(0, len(trs)))
            G, B = int(rng.integers(2, 20)), int(rng.integers(2, 24))
            rows.append(abi.scenario(policy=pol, workers=G, batch=B, horizon=H, drift=d, lookahead=la,
                                     noise_sigma=2.0 if la == abi.NOISY else 0.0, seed=7 + j, input_id=t))
            tid.append(t)
    scen = np.array(rows, abi.scenario_dtype)
    br = ctx.run_batch(scen, host.InputPool(trs), emit_steps=True, emit_requests=True)
    assert (br.res["status"] == abi.OK).all()
    for i in range(len(rows)):
        rc, err, (st, rq, m, done) = ref.run_poisson(br.scen[i], trs[tid[i]])
        assert rc == 0, err
        _check_vs_ref(br, i, st, rq, m, n_req=trs[tid[i]].shape[0])


def test_poisson_dyadic_large_g(ctx, ref):
    """Dyadic drift through the wide-G variants: the completion calendar
    (G*B > 4096) and the wide CTA chain (bfio-greedy H > 0 on G > 128)."""
    tr = host.sample_instance(9, rate=60000.0, duration=0.25, s_max=64, p=0.05)
    rows = [abi.scenario(policy=abi.BFIO_GREEDY, workers=200, batch=24, horizon=3, drift=0.5, input_id=0),
            abi.scenario(policy=abi.FCFS, workers=300, batch=16, drift=0.25, input_id=0),
            abi.scenario(policy=abi.BFIO_GREEDY, workers=96, batch=64, horizon=0, drift=1.5, input_id=0)]
    br = ctx.run_batch(np.array(rows, abi.scenario_dtype), host.InputPool([tr]), emit_steps=True,
                       emit_requests=True)
    for i in range(len(rows)):
        rc, err, (st, rq, m, done) = ref.run_poisson(br.scen[i], tr)
        assert rc == 0, err
        _check_vs_ref(br, i, st, rq, m, n_req=tr.shape[0])


def test_overloaded_dyadic_vs_reference(ctx, ref):
    """run_overloaded with OverloadedSpec::drift = 0.5 / 0.25 (acceptance C05's
    bfio-greedy with a window, and FCFS), the reference drawing its own pool."""
    rows = []
    for j, (pol, H, d) in enumerate(((abi.BFIO_GREEDY, 4, 0.5), (abi.FCFS, 0, 0.25), (abi.BFIO_GREEDY, 0, 0.75),
                                     (abi.JSQ, 0, 0.5))):
        rows.append(abi.scenario(mode=abi.OVERLOADED, policy=pol, workers=8, batch=16, horizon=H, drift=d,
                                 steps=120, warmup=30, seed=21 + j, input_id=j))
    streams = [host.sample_stream(21 + j, 40000, s_max=64, p=0.02) for j in range(len(rows))]
    br = ctx.run_batch(np.array(rows, abi.scenario_dtype), host.InputPool(streams), emit_steps=True)
    for i in range(len(rows)):
        rc, err, (st, rq, m, done) = ref.run_overloaded(br.scen[i], s_max=64)
        assert rc == 0, err
        _check_vs_ref(br, i, st, rq, m, tail=True)


def test_non_dyadic_drift_rejected(ctx):
    tr = host.sample_instance(1, rate=100.0, duration=0.5)
    for d in (0.1, 1.0 / 3.0, 2.0 ** -17):
        sc = np.array([abi.scenario(policy=abi.FCFS, workers=2, batch=2, drift=d, input_id=0)], abi.scenario_dtype)
        with pytest.raises(host.InvalidArgument, match="dyadic"):
            ctx.run_batch(sc, host.InputPool([tr]))
