"""The batched policy operator (bfsim_assign_batch): assign() for all four
policies (policies.hpp:372-382), one warp per call, against the reference
build call by call -- the reference's policy unit tests
(tests/policies_test.cpp:77-224), its random-step property shapes (:27-55)
and acceptance C01's 10^4 exact-solver instances, with SearchLimitExceeded
(:158-162) surfacing as BFSIM_ELIMIT."""
import numpy as np
import pytest

from paper_2601_17855_b200 import abi, host

pytestmark = pytest.mark.gpu

POLICIES = (abi.FCFS, abi.JSQ, abi.BFIO_EXACT, abi.BFIO_GREEDY)


@pytest.fixture(scope="module")
def ctx():
    c = host.Context(0)
    yield c
    c.close()


def _random_calls(rng, n_calls, policy, max_g=3, max_b=3, max_wait=6, max_h=2, fmax=20, wmax=10):
    calls = []
    for _ in range(n_calls):
        H = int(rng.integers(0, max_h + 1))
        G = int(rng.integers(1, max_g + 1))
        n = int(rng.integers(0, max_wait + 1))
        caps = rng.integers(0, max_b + 1, G).astype(np.int32)
        cnt = rng.integers(0, 3, G).astype(np.int32)
        fut = rng.integers(0, fmax, (G, H + 1)).astype(np.float64)
        pv = rng.integers(0, wmax, (n, H + 1)).astype(np.float64)
        calls.append((policy, pv, caps, cnt, fut))
    return calls


def _check(ctx, ref, calls, limit=200000):
    got = host.assign_batch(ctx, calls, search_limit=limit)
    for k, ((pol, pv, caps, cnt, fut), (pairs, cost, st)) in enumerate(zip(calls, got)):
        H = fut.shape[1] - 1
        rc, want, wcost = ref.assign(pol, pv, caps, cnt, fut, H, limit)
        if rc == 9:  # SearchLimitExceeded (a std::runtime_error)
            assert st == abi.ELIMIT, k
            continue
        assert rc == 0 and st == abi.OK, (k, rc, st)
        assert pairs == want, (k, pol, pairs, want)
        if pol == abi.BFIO_EXACT:
            assert cost == wcost, (k, cost, wcost)


@pytest.mark.parametrize("policy", POLICIES)
def test_random_steps(ctx, ref, policy):
    """policies_test.cpp random_step shapes: G <= 3, B <= 3, <= 6 waiting, H <= 2."""
    rng = np.random.default_rng(1000 + policy)
    _check(ctx, ref, _random_calls(rng, 3000, policy))


@pytest.mark.parametrize("policy", (abi.FCFS, abi.JSQ, abi.BFIO_GREEDY))
def test_wide_steps(ctx, ref, policy):
    """Up to 32 workers, 300 waiting requests and H = 24 (phase-1 water filling active)."""
    rng = np.random.default_rng(77 + policy)
    _check(ctx, ref, _random_calls(rng, 300, policy, max_g=32, max_b=6, max_wait=300, max_h=24, fmax=400,
                                   wmax=64))


def test_c01_exact_instances(ctx, ref):
    """Acceptance C01 scale (acceptance_test.cpp:117-128): 10^4 exact-solver
    instances, every optimum and its cost equal to the reference's."""
    rng = np.random.default_rng(101)
    _check(ctx, ref, _random_calls(rng, 10000, abi.BFIO_EXACT))


def test_exact_unit_cases(ctx, ref):
    """policies_test.cpp:132-162: balance to 0, empty waiting, lexicographic
    tie, search limit."""
    calls = [
        (abi.BFIO_EXACT, np.array([[7.0], [1.0]]), np.array([1, 1]), np.array([0, 0]), np.array([[10.0], [4.0]])),
        (abi.BFIO_EXACT, np.zeros((0, 1)), np.array([1, 1]), np.array([0, 0]), np.array([[10.0], [4.0]])),
        (abi.BFIO_EXACT, np.array([[3.0], [3.0]]), np.array([1, 1]), np.array([0, 0]), np.array([[0.0], [0.0]])),
        (abi.BFIO_GREEDY, np.array([[9.0], [3.0]]), np.array([1, 1]), np.array([0, 0]), np.array([[0.0], [0.0]])),
    ]
    got = host.assign_batch(ctx, calls)
    assert got[0][0] == [(0, 1), (1, 0)] and got[0][1] == 0.0
    assert got[1][0] == [] and got[1][1] == 6.0
    assert got[2][0] == [(0, 0), (1, 1)]
    assert got[3][0] == [(0, 0), (1, 1)]
    lim = [(abi.BFIO_EXACT, np.ones((12, 1)), np.full(4, 4), np.zeros(4), np.zeros((4, 1)))]
    out = host.assign_batch(ctx, lim, search_limit=100)
    assert out[0][2] == abi.ELIMIT
    _check(ctx, ref, lim, limit=100)


def _c02_instances(rng, n):
    """Acceptance C02's instance family (acceptance_test.cpp:130-155): (G, B)
    in {(2,1), (3,1), (4,1), (2,2)}, s_max in 3..5, a pool over empty workers
    grown until Def. 1 holds for every slot (is_overloaded_at,
    workload.hpp:325-336; restarted past 9 requests), H = 0, w_0 = s."""
    combos = ((2, 1), (3, 1), (4, 1), (2, 2))
    out = []
    for _ in range(n):
        G, B = combos[int(rng.integers(0, 4))]
        s_max = 3 + int(rng.integers(0, 3))
        slots = G * B
        pool = []
        while True:
            cnt = np.bincount(np.array(pool, np.int64), minlength=s_max + 1) if pool else np.zeros(s_max + 1)
            if len(pool) - int(cnt[1:].max()) >= slots:
                break
            if len(pool) >= 9:
                pool = []
            pool.append(int(rng.integers(1, s_max + 1)))
        pv = np.array(pool, np.float64).reshape(-1, 1)
        out.append((s_max, (abi.BFIO_EXACT, pv, np.full(G, B, np.int32), np.zeros(G, np.int32),
                             np.zeros((G, 1)))))
    return out


def test_c02_smax_balance(ctx, ref):
    """Acceptance C02 (acceptance_test.cpp:130-169) on the GPU policy operator:
    1,000 overloaded pools over empty workers, bfio-exact fills every slot and
    leaves a post-admission load gap <= s_max; each optimum equals the
    reference's assign() call."""
    inst = _c02_instances(np.random.default_rng(202), 1000)
    calls = [c for _, c in inst]
    got = host.assign_batch(ctx, calls, search_limit=500000)
    for (s_max, (pol, pv, caps, cnt, fut)), (pairs, cost, st) in zip(inst, got):
        assert st == abi.OK
        G = caps.shape[0]
        assert len(pairs) == int(caps.sum())
        loads = np.zeros(G)
        for i, g in pairs:
            loads[g] += pv[i, 0]
        assert loads.max() - loads.min() <= s_max
    _check(ctx, ref, calls[:300], limit=500000)
