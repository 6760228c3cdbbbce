"""Empirical prefill / decode distributions (PrefillDistribution::empirical,
DecodeDistribution::empirical, workload.hpp:109-118, 185-193) in the host
batcher: traces and overloaded sample streams byte-identical to the
reference's sample_instance / run_overloaded draws (oracle/_ref), and the
reference's validation errors. CPU only."""
import numpy as np
import pytest

from paper_2601_17855_b200 import abi, host

PV = [3, 17, 17, 64, 1, 250]
DV = [1, 2, 5, 40, 40, 300, 7]


def test_empirical_trace_matches_reference(ref):
    ref.set_empirical(PV, DV)
    for seed in (1, 2, 99):
        ours = host.sample_instance(seed, rate=500.0, duration=2.0, prefill_values=PV, decode_values=DV)
        theirs = ref.sample_instance(seed=seed, rate=500.0, duration=2.0, prefill_kind=2, decode_kind=2)
        assert ours.tobytes() == theirs.tobytes()
        assert set(np.unique(ours["prefill"])) <= set(PV) and set(np.unique(ours["decode"])) <= set(DV)


def test_mixed_kinds_match_reference(ref):
    ref.set_empirical(PV, DV)
    a = host.sample_instance(5, rate=300.0, duration=1.0, prefill_values=PV, p=0.05)
    b = ref.sample_instance(seed=5, rate=300.0, duration=1.0, prefill_kind=2, decode_kind=0, p=0.05)
    assert a.tobytes() == b.tobytes()
    a = host.sample_instance(6, rate=300.0, duration=1.0, s_max=32, decode_values=DV)
    b = ref.sample_instance(seed=6, rate=300.0, duration=1.0, s_max=32, prefill_kind=0, decode_kind=2)
    assert a.tobytes() == b.tobytes()


def test_empirical_stream_draw_order():
    """run_overloaded's top-up draws prefill then decode per request
    (oracle.hpp:177-183): the stream is the trace's marks without the gaps,
    so a fixed-seed stream is reproducible and uses only listed values."""
    s1 = host.sample_stream(3, 5000, prefill_values=PV, decode_values=DV)
    s2 = host.sample_stream(3, 5000, prefill_values=PV, decode_values=DV)
    assert s1.tobytes() == s2.tobytes()
    assert set(np.unique(s1["prefill"])) == set(PV) and set(np.unique(s1["decode"])) == set(DV)


@pytest.mark.parametrize("kw,msg", [
    (dict(prefill_values=[]), "prefill: empty empirical list"),
    (dict(prefill_values=[0, 3]), "prefill: empirical value < 1"),
    (dict(decode_values=[]), "decode: empty empirical list"),
    (dict(decode_values=[2, -1]), "decode: empirical value < 1"),
])
def test_empirical_validation(kw, msg):
    with pytest.raises(host.InvalidArgument, match=msg):
        host.sample_instance(1, rate=10.0, duration=1.0, **kw)
