"""numpy / ctypes mirrors of the plain record layouts in include/bfsim_gpu.h.

These are layouts only (no behaviour): the product library, the C++ wrapper
and the test oracle all exchange the same bytes.
"""
from __future__ import annotations

import numpy as np

OK, EINVAL, ELOGIC, ECUDA, PARTIAL, ESTREAM, ELIMIT, ERANGE = 0, 1, 2, 3, 4, 5, 6, 7

# PolicyKind, policies.hpp:16
FCFS, JSQ, BFIO_EXACT, BFIO_GREEDY = 0, 1, 2, 3
POLICY_NAMES = {"fcfs": FCFS, "jsq": JSQ, "bfio-exact": BFIO_EXACT, "bfio-greedy": BFIO_GREEDY}
POLICY_LABELS = {v: k for k, v in POLICY_NAMES.items()}
# LookaheadMode, policies.hpp:36
PERFECT, TRUNCATED, NOISY = 0, 1, 2
POISSON, OVERLOADED = 0, 1

FLAG_STEP_OVERFLOW, FLAG_NOISE_NEAR_TIE, FLAG_EMPTY = 1, 2, 4

request_dtype = np.dtype([("arrival_time", "<f8"), ("prefill", "<i4"), ("decode", "<i4")])
sample_dtype = np.dtype([("prefill", "<i4"), ("decode", "<i4")])
input_dtype = np.dtype(
    [
        ("offset", "<i8"),
        ("length", "<i8"),
        ("class_base_offset", "<i8"),
        ("s_max", "<i4"),
        ("max_decode", "<i4"),
    ]
)
scenario_dtype = np.dtype(
    [
        ("mode", "<i4"),
        ("policy", "<i4"),
        ("lookahead", "<i4"),
        ("workers", "<i4"),
        ("batch", "<i4"),
        ("horizon", "<i4"),
        ("input_id", "<i4"),
        ("reserved0", "<i4"),
        ("drift", "<f8"),
        ("overhead", "<f8"),
        ("per_token", "<f8"),
        ("noise_sigma", "<f8"),
        ("p_idle", "<f8"),
        ("p_max", "<f8"),
        ("mfu_sat", "<f8"),
        ("gamma", "<f8"),
        ("backlog", "<f8"),
        ("max_steps", "<i8"),
        ("steps", "<i8"),
        ("warmup", "<i8"),
        ("seed", "<u8"),
        ("step_offset", "<i8"),
        ("step_capacity", "<i8"),
        ("load_offset", "<i8"),
        ("req_offset", "<i8"),
    ]
)
result_dtype = np.dtype(
    [
        ("status", "<i4"),
        ("flags", "<u4"),
        ("steps_run", "<i8"),
        ("records", "<i8"),
        ("completed", "<i8"),
        ("admitted", "<i8"),
        ("consumed", "<i8"),
        ("imb_total_i", "<i8"),
        ("total_workload_i", "<i8"),
        ("tokens_i", "<i8"),
        ("avg_imbalance", "<f8"),
        ("throughput", "<f8"),
        ("tpot", "<f8"),
        ("energy", "<f8"),
        ("imb_total", "<f8"),
        ("total_workload", "<f8"),
        ("eta_sum", "<f8"),
        ("clock", "<f8"),
        ("elapsed", "<f8"),
        ("tpot_sum", "<f8"),
    ]
)
METRIC_FIELDS = (
    "avg_imbalance",
    "throughput",
    "tpot",
    "energy",
    "imb_total",
    "total_workload",
    "eta_sum",
)

assert request_dtype.itemsize == 16
assert sample_dtype.itemsize == 8
assert input_dtype.itemsize == 32
assert scenario_dtype.itemsize == 168
assert result_dtype.itemsize == 152


def scenario(
    *,
    mode=POISSON,
    policy=FCFS,
    lookahead=PERFECT,
    workers=8,
    batch=16,
    horizon=0,
    input_id=0,
    drift=1.0,
    overhead=9.775e-3,
    per_token=1.005e-7,
    noise_sigma=0.0,
    p_idle=100.0,
    p_max=400.0,
    mfu_sat=0.45,
    gamma=0.7,
    backlog=1.0,
    max_steps=10_000_000,
    steps=2000,
    warmup=200,
    seed=0,
):
    """One scenario row with the reference defaults (SimConfig engine.hpp:17-30,
    OverloadedSpec oracle.hpp:121-132, PowerModel metrics_power.hpp:11-16)."""
    s = np.zeros((), dtype=scenario_dtype)
    if isinstance(policy, str):
        policy = POLICY_NAMES[policy]
    for k, v in dict(
        mode=mode, policy=policy, lookahead=lookahead, workers=workers, batch=batch,
        horizon=horizon, input_id=input_id, drift=drift, overhead=overhead,
        per_token=per_token, noise_sigma=noise_sigma, p_idle=p_idle, p_max=p_max,
        mfu_sat=mfu_sat, gamma=gamma, backlog=backlog, max_steps=max_steps, steps=steps,
        warmup=warmup, seed=seed,
    ).items():
        s[k] = v
    return s


def ptr(a):
    """ctypes void* of a numpy array (or None)."""
    import ctypes

    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return ctypes.c_void_p(a.ctypes.data)
