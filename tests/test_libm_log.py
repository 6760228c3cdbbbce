"""The device generator's log (csrc/libm_log.cuh) is glibc's log bit for bit.

The reference's traces call glibc `log` through libstdc++ (exponential gaps,
geometric decode lengths; workload.hpp:198,252-263). libm_log.cuh restates
glibc 2.39's x86-64 __log_fma; its host twin (bfsim_libm_log_host, the same
source compiled for the host) is compared here with the host's libm on the
generator's own input domain (1 - U, U = generate_canonical<double, 53>), the
near-1 polynomial window, random positive doubles over the whole exponent
range, subnormals and the special values. The device build of the same
function is checked through the traces it produces (tests/test_gpu_tracegen.py).
"""
import ctypes

import numpy as np

from paper_2601_17855_b200 import host

_libm = ctypes.CDLL("libm.so.6")


def _glibc_log(x):
    # numpy's log is not glibc's; np.frompyfunc over ctypes calls the real one
    f = _libm.log
    f.restype, f.argtypes = ctypes.c_double, [ctypes.c_double]
    return np.frompyfunc(f, 1, 1)(x).astype(np.float64)


def _same(a, b):
    return (a.view(np.int64) == b.view(np.int64)) | (np.isnan(a) & np.isnan(b))


def test_generator_domain():
    rng = np.random.default_rng(2601)
    w = rng.integers(0, 2**64 - 1, size=300_000, dtype=np.uint64, endpoint=True)
    u = np.minimum(w.astype(np.float64) * 2.0**-64, np.nextafter(1.0, 0.0))  # generate_canonical
    x = 1.0 - u
    assert _same(host.libm_log(x), _glibc_log(x)).all()


def test_near_one_and_wide_range():
    rng = np.random.default_rng(17855)
    near = 1.0 + (rng.random(200_000) - 0.5) * 0.14
    bits = rng.integers(1, 0x7FEFFFFFFFFFFFFF, size=200_000, dtype=np.int64)
    wide = bits.view(np.float64)
    sub = np.ldexp(rng.random(20_000), -1060)
    special = np.array([1.0, np.nextafter(1.0, 0), np.nextafter(1.0, 2), 0.9375, 1.0 + float.fromhex("0x1.09p-4"), 2.0**-1074,
                        2.0**-1022, np.finfo(np.float64).max, 0.0, -0.0, -1.0, np.inf, -np.inf, np.nan])
    for x in (near, wide, sub, special):
        assert _same(host.libm_log(x), _glibc_log(x)).all()
