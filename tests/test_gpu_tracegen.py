"""Device-side input generation vs the host batcher.

The host batcher (bfsim_sample_instance*/bfsim_sample_stream*) calls
libstdc++'s own distributions and is pinned to the reference's traces
(tests/test_golden.py, tests/test_oracle_vs_ref.py). The device generator
(csrc/tracegen.cu) must produce the same bytes: arrival times, prefill and
decode of every record, the same record count, and the same bfsim_input_t
statistics and class_base table as bfsim_prepare_trace / _stream. Then a
trajectory run on the device-resident pool equals the same run on the host
pool, and the whole C3 pass (1,000 x 100k-request traces) is generated on the
device and checked record for record on a sample of traces.
"""
import os

import numpy as np
import pytest

from paper_2601_17855_b200 import abi, host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = host.Context(0)
    yield c
    c.close()


def _host_kw(sp):
    return {k: v for k, v in sp.items() if k != "seed"}


def _check(pool, specs, samples=None):
    for i, sp in enumerate(specs):
        if samples is None:
            want = host.sample_instance(sp["seed"], **_host_kw(sp))
        else:
            kw = {k: v for k, v in _host_kw(sp).items() if k not in ("rate", "duration")}
            want = host.sample_stream(sp["seed"], samples, **kw)
        got = pool.host_records(i)
        assert got.shape == want.shape, f"input {i}: {got.shape[0]} records, host batcher {want.shape[0]}"
        assert got.tobytes() == want.tobytes(), f"input {i}: records differ"
        info, cb = host.prepare(want)
        gi = pool.inputs[i]
        assert int(gi["length"]) == int(info["length"])
        assert int(gi["s_max"]) == int(info["s_max"]), f"input {i}: s_max"
        assert int(gi["max_decode"]) == int(info["max_decode"]), f"input {i}: max_decode"
        np.testing.assert_array_equal(pool.host_class_base(i), cb)


SPECS = [
    dict(seed=1, rate=8000.0, duration=2.0, s_max=64, p=0.02),            # C3-shaped
    dict(seed=2, rate=4000.0, duration=2.5, s_max=64, p=0.02),            # C2
    dict(seed=3, rate=500.0, duration=3.0, s_max=1, p=0.5),               # one class
    dict(seed=4, rate=1000.0, duration=1.0, s_max=32768, p=0.001),        # C08-style prompts
    dict(seed=5, rate=700.0, duration=2.0, s_max=17, prefill_kind=1, decode_kind=1, fixed_o=9),
    dict(seed=6, rate=900.0, duration=2.0, s_max=64, decode_kind=1, fixed_o=40),
    dict(seed=7, rate=900.0, duration=2.0, s_max=5, prefill_kind=1, p=0.3),
    dict(seed=8, rate=2000.0, duration=1.0, prefill_values=[3, 1, 4, 1, 5, 9, 2, 6], p=0.05),
    dict(seed=9, rate=2000.0, duration=1.0, s_max=64, decode_values=[10, 200, 3000, 7]),
    dict(seed=10, rate=2000.0, duration=1.0, prefill_values=[7], decode_values=list(range(1, 1000))),
    dict(seed=11, rate=3.0, duration=0.01, s_max=64, p=0.02),             # (almost surely) empty
    dict(seed=12, rate=1e5, duration=0.5, s_max=64, p=0.999),             # decode mostly 1
    dict(seed=2**63 + 5, rate=1234.5, duration=1.7, s_max=100, p=0.013),
]


def test_traces_equal_host_batcher(ctx):
    pool = host.DevicePool(ctx, SPECS)
    _check(pool, SPECS)


def test_streams_equal_host_batcher(ctx):
    specs = [dict(seed=s, s_max=64, p=0.02) for s in (0, 1, 77, 2**40)] + [
        dict(seed=5, prefill_values=[2, 8, 32], decode_values=[1, 5]),
        dict(seed=6, s_max=9, prefill_kind=1, decode_kind=1, fixed_o=3),
        dict(seed=7, s_max=256, p=0.9)]
    pool = host.DevicePool(ctx, specs, samples=50000)
    _check(pool, specs, samples=50000)


@pytest.mark.parametrize("mask", ["0x1", "0x80000001", "0xffffffff", "0x12481248"])
def test_sequential_path(ctx, monkeypatch, mask):
    """Records forced through the sequential (rejection) rules at chosen lanes
    give the same bytes: the cursor bookkeeping of an irregular record."""
    monkeypatch.setenv("BFSIM_GEN_FORCE_SLOW", mask)
    specs = SPECS[:3] + SPECS[4:6] + SPECS[7:10]
    pool = host.DevicePool(ctx, specs)
    _check(pool, specs)
    sspec = [dict(seed=3, s_max=64, p=0.02), dict(seed=4, prefill_values=[1, 2, 3], decode_values=[4, 5])]
    spool = host.DevicePool(ctx, sspec, samples=5000)
    _check(spool, sspec, samples=5000)


def test_rejections(ctx):
    with pytest.raises(host.InvalidArgument, match="rate must be > 0"):
        host.DevicePool(ctx, [dict(seed=1, rate=0.0, duration=1.0)])
    with pytest.raises(host.InvalidArgument, match="p must be in"):
        host.DevicePool(ctx, [dict(seed=1, rate=1.0, duration=1.0, p=1.0)])
    with pytest.raises(host.InvalidArgument, match="empirical value < 1"):
        host.DevicePool(ctx, [dict(seed=1, rate=1.0, duration=1.0, prefill_values=[1, 0])])
    # a decode beyond int32, as the host batcher reports it
    with pytest.raises(host.InvalidArgument, match="decode exceeds int32"):
        host.DevicePool(ctx, [dict(seed=1, rate=100.0, duration=1.0, p=1e-12)])


def test_run_on_device_pool_equals_host_pool(ctx):
    specs = [dict(seed=s, rate=6000.0, duration=0.3, s_max=64, p=0.05) for s in (21, 22)]
    dpool = host.DevicePool(ctx, specs)
    hpool = host.InputPool([host.sample_instance(sp["seed"], **_host_kw(sp)) for sp in specs])
    scen = np.array([abi.scenario(policy=p, workers=16, batch=16, horizon=h, lookahead=la, noise_sigma=sg,
                                  seed=3, input_id=i)
                     for i in (0, 1)
                     for p, h, la, sg in ((abi.FCFS, 0, 0, 0.0), (abi.BFIO_GREEDY, 4, 0, 0.0),
                                          (abi.BFIO_GREEDY, 8, abi.NOISY, 2.0))], abi.scenario_dtype)
    outs = []
    for pool in (dpool, hpool):
        b = host.DeviceBatch(ctx, scen, pool, emit_steps=True, emit_requests=True)
        for v in b.steps.values():  # rows past a trajectory's steps_run are never written
            v.zero_()
        b.run()
        import torch

        torch.cuda.synchronize()
        outs.append((b.result_array(), {k: v.cpu().numpy() for k, v in b.steps.items()},
                     {k: v.cpu().numpy() for k, v in b.reqs.items()}))
    (r0, s0, q0), (r1, s1, q1) = outs
    assert r0.tobytes() == r1.tobytes()
    for k in s0:
        np.testing.assert_array_equal(s0[k], s1[k])
    for k in q0:
        np.testing.assert_array_equal(q0[k], q1[k])


def test_c3_full_pass_generated_on_device(ctx):
    """The C3 pass's 1,000 traces (lambda = 8000/s x 12.5 s, ~100k requests
    each) in HBM; 12 of them checked record for record against the host
    batcher, all 1,000 lengths against the host generator's counts."""
    seeds = list(range(1000))
    specs = [dict(seed=s, rate=8000.0, duration=12.5, s_max=64, p=0.02) for s in seeds]
    pool = host.DevicePool(ctx, specs)
    assert int(pool.inputs["length"].sum()) > 99_000_000
    pick = [0, 1, 2, 99, 250, 333, 500, 640, 777, 888, 998, 999]
    for i in pick:
        want = host.sample_instance(seeds[i], rate=8000.0, duration=12.5, s_max=64, p=0.02)
        got = pool.host_records(i)
        assert got.tobytes() == want.tobytes(), f"trace {i} differs"
    # lengths of all traces from the host batcher's count-only call
    L, err = host.lib(), host._err()
    n = np.zeros(1, np.int64)
    for i in range(0, 1000, 37):
        rc = L.bfsim_sample_instance(0, 64, 0, 0.02, 1, 8000.0, 12.5, seeds[i], None, 0, abi.ptr(n), err, 1024)
        assert rc == 0
        assert int(pool.inputs["length"][i]) == int(n[0])
