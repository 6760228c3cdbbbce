"""CPU-only checks of the product library and its host batcher (no GPU needed):
the C-ABI library loads and exports every symbol include/bfsim_gpu.h declares,
the ABI record layouts match the header, and the host trace / stream
generators are byte-identical to the reference's own draws."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2601_17855_b200 import abi, host

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "bfsim_gpu.h")).read()
    return sorted(set(re.findall(r"\b(bfsim_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = host.lib()
    syms = _declared_symbols()
    assert len(syms) >= 13
    for s in syms:
        assert hasattr(L, s), s


def test_struct_layouts_match_header(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "bfsim_gpu.h"\n'
        "int main(){printf(\"%zu %zu %zu %zu %zu %zu %zu\\n\", sizeof(bfsim_request_t), sizeof(bfsim_sample_t),"
        " sizeof(bfsim_input_t), sizeof(bfsim_scenario_t), sizeof(bfsim_result_t),"
        " offsetof(bfsim_scenario_t, seed), offsetof(bfsim_result_t, avg_imbalance));}\n"
    )
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    got = list(map(int, out))
    assert got == [
        abi.request_dtype.itemsize, abi.sample_dtype.itemsize, abi.input_dtype.itemsize,
        abi.scenario_dtype.itemsize, abi.result_dtype.itemsize,
        abi.scenario_dtype.fields["seed"][1], abi.result_dtype.fields["avg_imbalance"][1],
    ]


@pytest.mark.parametrize("seed,rate,dur,smax,p", [(1, 2000.0, 1.0, 64, 0.02), (42, 10.0, 50.0, 64, 0.02),
                                                  (77, 40.0, 5.0, 16, 0.2), (1, 4000.0, 2.5, 64, 0.02)])
def test_sample_instance_byte_identical(ref, seed, rate, dur, smax, p):
    a = host.sample_instance(seed, rate=rate, duration=dur, s_max=smax, p=p)
    b = ref.sample_instance(s_max=smax, p=p, rate=rate, duration=dur, seed=seed)
    assert a.tobytes() == b.tobytes()


def test_known_answers():
    """libstdc++ known answers: a fresh mt19937_64(1) draws U[1,64] = 9 then
    1 + Geo(0.02) = 8 (checked with a standalone g++ probe; SURVEY §8(c) lists
    "29" for the uniform, which does not reproduce from a fresh engine). The C1
    trace (lambda=2000/s, 1 s, seed 1) has 1,957 requests."""
    st = host.sample_stream(1, 1, s_max=64, p=0.02)
    assert int(st[0]["prefill"]) == 9 and int(st[0]["decode"]) == 8
    assert host.sample_instance(1, rate=2000.0, duration=1.0).shape[0] == 1957


def test_stream_prefix_property():
    a = host.sample_stream(9, 1000, s_max=64, p=0.02)
    b = host.sample_stream(9, 300, s_max=64, p=0.02)
    assert a[:300].tobytes() == b.tobytes()


def test_prepare_class_base():
    tr = host.sample_instance(3, rate=500.0, duration=2.0, s_max=20, p=0.1)
    info, cb = host.prepare(tr)
    assert int(info["s_max"]) == int(tr["prefill"].max())
    assert int(info["max_decode"]) == int(tr["decode"].max())
    cnt = np.bincount(tr["prefill"], minlength=int(info["s_max"]) + 2)
    for c in range(1, int(info["s_max"]) + 2):
        assert cb[c] == cnt[:c].sum()


def test_rejects_bad_distributions():
    with pytest.raises(host.InvalidArgument):
        host.sample_instance(1, rate=-1.0, duration=1.0)
    with pytest.raises(host.InvalidArgument):
        host.sample_stream(1, 10, p=1.5)
    unsorted = np.zeros(2, abi.request_dtype)
    unsorted[0] = (1.0, 1, 1)
    unsorted[1] = (0.5, 1, 1)
    with pytest.raises(host.InvalidArgument):
        host.prepare(unsorted)


def test_iir_reducer_matches_reference_formula():
    rng = np.random.default_rng(3)
    f = rng.uniform(10, 20, (3, 5))
    b = rng.uniform(1, 5, (3, 5))
    b[2] = 0.0
    out = host.iir_reduce(f, b)
    for c in range(2):
        fm, bm = f[c].mean(), b[c].mean()
        sem = lambda v: np.sqrt(((v - v.mean()) ** 2).sum() / (len(v) - 1)) / np.sqrt(len(v))
        ratio = fm / bm
        se = ratio * np.sqrt((sem(f[c]) / fm) ** 2 + (sem(b[c]) / bm) ** 2)
        assert out[c, 2] == pytest.approx(ratio, rel=1e-14)
        assert out[c, 3] == pytest.approx(se, rel=1e-12)
    assert np.isinf(out[2, 2]) and np.isinf(out[2, 3])


def test_no_gpu_context_fails_loudly():
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    with pytest.raises(host.BfsimError):
        host.Context(0)


def test_input_pool_prefix():
    """InputPool.add_prefix: a stream prefix shares the records and carries the
    statistics and class_base of the prefix itself (the bench's C4 runs small
    G on prefixes of the large-G streams)."""
    s1 = host.sample_stream(3, 5000, s_max=64, p=0.02)
    s2 = host.sample_stream(4, 3000, s_max=16, p=0.1)
    pool = host.InputPool([s1, s2])
    n_rec = pool.records.shape[0]
    i = pool.add_prefix(1, 700)
    assert pool.records.shape[0] == n_rec and i == 2
    info, cb = host.prepare(s2[:700])
    got = pool.inputs[i]
    assert int(got["offset"]) == int(pool.inputs[1]["offset"]) and int(got["length"]) == 700
    assert int(got["s_max"]) == int(info["s_max"]) and int(got["max_decode"]) == int(info["max_decode"])
    o = int(got["class_base_offset"])
    assert np.array_equal(pool.class_base[o:o + cb.shape[0]], cb)
