"""The BASELINE configs at their full sizes: bit-exact
against the oracle where the CPU restatement finishes in seconds (C2, C3), and
size-independent properties everywhere (workload conservation, completion of
every request, full batches in the overloaded regime, JSQ == FCFS,
run-to-run determinism)."""
import numpy as np
import pytest

from paper_2601_17855_b200 import abi, host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = host.Context(0)
    yield c
    c.close()


def _workload(tr, d):
    s = tr["prefill"].astype(np.int64)
    o = tr["decode"].astype(np.int64)
    return int((s * o + d * o * (o - 1) // 2).sum())


def _same(orc, br, i, tr):
    rc, res, st, rq = orc.run_poisson(br.scen[i], tr)
    np.testing.assert_array_equal(br.steps(i)["loads"], st.loads)
    np.testing.assert_array_equal(br.steps(i)["clock_start"], st.clock_start)
    gr = br.requests(i, tr.shape[0])
    for k in ("start_step", "worker", "finish_clock"):
        np.testing.assert_array_equal(gr[k], rq[k], err_msg=k)
    for k in ("avg_imbalance", "throughput", "imb_total", "eta_sum"):
        assert float(br.res[i][k]) == float(res[k]), k


def test_c2_full_size(ctx, orc):
    """C2: G=16, B=64, lambda=4000/s x 2.5 s, 6 seeds x {bfio-greedy, jsq, fcfs}."""
    traces, rows = [], []
    for j, seed in enumerate((1, 2, 3, 97, 128, 256)):
        traces.append(host.sample_instance(seed, rate=4000.0, duration=2.5, s_max=64, p=0.02))
        for pol in (abi.BFIO_GREEDY, abi.JSQ, abi.FCFS):
            rows.append(abi.scenario(policy=pol, workers=16, batch=64, input_id=j))
    br = ctx.run_batch(np.array(rows, abi.scenario_dtype), host.InputPool(traces), emit_steps=True,
                       emit_requests=True)
    for i, s in enumerate(br.scen):
        tr = traces[int(s["input_id"])]
        assert int(br.res[i]["completed"]) == tr.shape[0]
        assert int(br.res[i]["total_workload_i"]) == _workload(tr, 1)
        if i % 3 == 1:  # JSQ == FCFS bit for bit
            np.testing.assert_array_equal(br.steps(i)["loads"], br.steps(i + 1)["loads"])
    for i in (0, 1, 9):
        _same(orc, br, i, traces[int(br.scen[i]["input_id"])])


def test_c3_full_size(ctx, orc):
    """C3: G=64, B=64, lambda=8000/s x 12.5 s (~100k requests), bfio-greedy
    H=20 with Noisy sigma=2; two seeds against the oracle, full length."""
    traces, rows = [], []
    for j, seed in enumerate((1, 500)):
        traces.append(host.sample_instance(seed, rate=8000.0, duration=12.5, s_max=64, p=0.02))
        rows.append(abi.scenario(policy=abi.BFIO_GREEDY, workers=64, batch=64, horizon=20, lookahead=abi.NOISY,
                                 noise_sigma=2.0, seed=seed, input_id=j))
    br = ctx.run_batch(np.array(rows, abi.scenario_dtype), host.InputPool(traces), emit_steps=True,
                       emit_requests=True)
    for i, tr in enumerate(traces):
        assert int(br.res[i]["completed"]) == tr.shape[0]
        assert not int(br.res[i]["flags"]) & abi.FLAG_NOISE_NEAR_TIE
        _same(orc, br, i, tr)


def test_c4_full_size_g1024(ctx):
    """C4 at G=1024, B=64, 2000+200 steps: every step after warm-up runs full
    batches (oracle_test.cpp:99-107), JSQ == FCFS, imbalance non-negative,
    and a re-run is identical."""
    jobs = [(p, 0, 1024, 64, 2000, 200, 7) for p in (abi.FCFS, abi.JSQ, abi.BFIO_GREEDY)]
    br, _ = host.run_overloaded_batch(ctx, jobs, emit_steps=True)
    for i in range(3):
        st = br.steps(i)
        assert (st["active_count"][200:] == 1024 * 64).all()
        ld = st["loads"]
        assert ((1024 * ld.max(axis=1) - ld.sum(axis=1)) >= 0).all()
    np.testing.assert_array_equal(br.steps(0)["loads"], br.steps(1)["loads"])
    assert br.res["avg_imbalance"][2] < br.res["avg_imbalance"][0]
    br2, _ = host.run_overloaded_batch(ctx, jobs[2:], emit_steps=True)
    np.testing.assert_array_equal(br2.steps(0)["loads"], br.steps(2)["loads"])


def test_c5_full_size_trace(ctx):
    """C5: one shared 1M-request trace (lambda=8000/s x 125 s), G=B=64, under
    fcfs and bfio-greedy H=0: every request completes, workload is conserved,
    and the run is deterministic."""
    tr = host.sample_instance(1, rate=8000.0, duration=125.0, s_max=64, p=0.02)
    assert tr.shape[0] > 990_000
    rows = [abi.scenario(policy=p, workers=64, batch=64, input_id=0) for p in (abi.FCFS, abi.BFIO_GREEDY)]
    pool = host.InputPool([tr])
    br = ctx.run_batch(np.array(rows, abi.scenario_dtype), pool)
    br2 = ctx.run_batch(np.array(rows, abi.scenario_dtype), pool)
    for i in range(2):
        assert int(br.res[i]["completed"]) == tr.shape[0]
        assert int(br.res[i]["total_workload_i"]) == _workload(tr, 1)
        assert br.res[i].tobytes() == br2.res[i].tobytes()
    assert br.res["avg_imbalance"][1] < br.res["avg_imbalance"][0]
