"""ORACLE / TEST INFRASTRUCTURE — ctypes loader for the CPU checkers.

Two checkers, both CPU:
  * RefLib    -> oracle/_ref/libbfsim_ref.so: the UNMODIFIED reference headers
                 (/root/reference/proj/include) behind oracle/ref_driver.cpp.
  * OracleLib -> oracle/liboracle.so: the plain-C restatement (bfsim_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import this
module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2601_17855_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libbfsim_ref.so")
REF_INC = "/root/reference/proj/include"

_vp, _i32, _i64, _u64, _f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double


def build():
    """Build liboracle.so (and oracle/_ref when the reference is mounted)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _errbuf():
    return C.create_string_buffer(512)


class StepSeries:
    """Per-step records as arrays (StepRecord, engine.hpp:39-48)."""

    def __init__(self, K, G):
        self.k = np.zeros(K, np.int64)
        self.clock_start = np.zeros(K)
        self.dt = np.zeros(K)
        self.max_load = np.zeros(K)
        self.active_count = np.zeros(K, np.int64)
        self.loads = np.zeros((K, G))


class OracleLib:
    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        L = self.lib
        L.oracle_run_poisson.argtypes = [_vp, _vp, _i64, _i64] + [_vp] * 10 + [_vp]
        L.oracle_run_poisson.restype = C.c_int
        L.oracle_run_overloaded.argtypes = (
            [_vp, _vp, _i64, _i32, _i64] + [_vp] * 7 + [_i64] + [_vp] * 5 + [_vp]
        )
        L.oracle_run_overloaded.restype = C.c_int
        L.oracle_assign.argtypes = [C.c_int, C.c_int, _vp, C.c_int, _vp, _vp, _vp, C.c_int, _vp, _vp]
        L.oracle_assign.restype = C.c_int
        L.oracle_mt64_seed.argtypes = [_vp, _u64]
        L.oracle_mt64_next.argtypes = [_vp]
        L.oracle_mt64_next.restype = _u64
        L.oracle_normal.argtypes = [_vp, _f64, _f64]
        L.oracle_normal.restype = _f64

    def run_poisson(self, sc, trace, step_cap=None):
        """Returns (result, steps, requests) with requests a dict of arrays."""
        sc = np.ascontiguousarray(sc, dtype=abi.scenario_dtype).reshape(())
        trace = np.ascontiguousarray(trace, dtype=abi.request_dtype)
        n = trace.shape[0]
        G = int(sc["workers"])
        if step_cap is None:
            step_cap = _poisson_step_bound(trace, sc)
        st = StepSeries(step_cap, G)
        rq = {
            "arrival_step": np.zeros(n, np.int32),
            "start_step": np.zeros(n, np.int32),
            "worker": np.zeros(n, np.int32),
            "admit_clock": np.zeros(n),
            "finish_clock": np.zeros(n),
        }
        res = np.zeros((), abi.result_dtype)
        rc = self.lib.oracle_run_poisson(
            abi.ptr(sc), abi.ptr(trace), n, step_cap,
            abi.ptr(st.clock_start), abi.ptr(st.dt), abi.ptr(st.max_load),
            abi.ptr(st.active_count), abi.ptr(st.loads),
            abi.ptr(rq["arrival_step"]), abi.ptr(rq["start_step"]), abi.ptr(rq["worker"]),
            abi.ptr(rq["admit_clock"]), abi.ptr(rq["finish_clock"]), abi.ptr(res),
        )
        K = min(int(res["steps_run"]), step_cap)
        _trim(st, K)
        return rc, res, st, rq

    def run_overloaded(self, sc, stream, s_max, step_cap=None):
        sc = np.ascontiguousarray(sc, dtype=abi.scenario_dtype).reshape(())
        stream = np.ascontiguousarray(stream, dtype=abi.sample_dtype)
        n = stream.shape[0]
        G = int(sc["workers"])
        total = int(sc["warmup"] + sc["steps"])
        if step_cap is None:
            step_cap = total
        st = StepSeries(step_cap, G)
        start = np.zeros(n, np.int32)
        worker = np.zeros(n, np.int32)
        tcap = n
        t = {
            "id": np.zeros(tcap, np.int32),
            "admit_clock": np.zeros(tcap),
            "finish_clock": np.zeros(tcap),
            "decode": np.zeros(tcap, np.int64),
        }
        nt = np.zeros(1, np.int64)
        res = np.zeros((), abi.result_dtype)
        rc = self.lib.oracle_run_overloaded(
            abi.ptr(sc), abi.ptr(stream), n, int(s_max), step_cap,
            abi.ptr(st.clock_start), abi.ptr(st.dt), abi.ptr(st.max_load),
            abi.ptr(st.active_count), abi.ptr(st.loads), abi.ptr(start), abi.ptr(worker),
            tcap, abi.ptr(t["id"]), abi.ptr(t["admit_clock"]), abi.ptr(t["finish_clock"]),
            abi.ptr(t["decode"]), abi.ptr(nt), abi.ptr(res),
        )
        _trim(st, min(int(res["steps_run"]), step_cap))
        m = int(min(nt[0], tcap))
        t = {k: v[:m] for k, v in t.items()}
        return rc, res, st, {"start_step": start, "worker": worker}, t

    def assign(self, policy, previews, caps, active_counts, futures, H):
        previews = np.ascontiguousarray(previews, np.float64).reshape(-1, H + 1)
        futures = np.ascontiguousarray(futures, np.float64).reshape(-1, H + 1)
        caps = np.ascontiguousarray(caps, np.int32)
        active_counts = np.ascontiguousarray(active_counts, np.int32)
        G = caps.shape[0]
        pairs = np.zeros(2 * max(1, int(caps.clip(min=0).sum())), np.int32)
        npairs = np.zeros(1, np.int64)
        rc = self.lib.oracle_assign(
            policy, previews.shape[0], abi.ptr(previews), G, abi.ptr(caps), abi.ptr(active_counts),
            abi.ptr(futures), H, abi.ptr(pairs), abi.ptr(npairs),
        )
        return rc, [(int(pairs[2 * j]), int(pairs[2 * j + 1])) for j in range(int(npairs[0]))]


class RefLib:
    """The unmodified reference (oracle/_ref/libbfsim_ref.so)."""

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_sample_instance.argtypes = [C.c_int, C.c_int, C.c_int, _f64, _i64, _f64, _f64, _u64, _vp, _i64, _vp, _vp, C.c_size_t]
        L.ref_set_empirical.argtypes = [_vp, _i64, _vp, _i64]
        L.ref_run_poisson.argtypes = [_vp, _vp, _i64, _vp, _vp, C.c_size_t]
        L.ref_run_poisson.restype = _vp
        L.ref_run_overloaded.argtypes = [_vp, C.c_int, C.c_int, C.c_int, _f64, _i64, _vp, _vp, C.c_size_t]
        L.ref_run_overloaded.restype = _vp
        for f in ("ref_res_steps", "ref_res_n_requests"):
            getattr(L, f).argtypes = [_vp]
            getattr(L, f).restype = _i64
        for f in ("ref_res_completed_all", "ref_res_has_metrics"):
            getattr(L, f).argtypes = [_vp]
            getattr(L, f).restype = C.c_int
        L.ref_res_step_arrays.argtypes = [_vp] * 7
        L.ref_res_list_total.argtypes = [_vp, C.c_int]
        L.ref_res_list_total.restype = _i64
        L.ref_res_list.argtypes = [_vp, C.c_int, _vp, _vp]
        L.ref_res_requests.argtypes = [_vp] * 8
        L.ref_res_metrics.argtypes = [_vp, _vp]
        L.ref_res_free.argtypes = [_vp]
        L.ref_assign.argtypes = [C.c_int, C.c_int, _vp, C.c_int, _vp, _vp, _vp, C.c_int, _i64, _vp, _vp, _vp, _vp, C.c_size_t]
        L.ref_estimate_iir.argtypes = [_vp, C.c_int, _vp, C.c_int, C.c_int, C.c_int, C.c_int, _f64, _i64, _f64, _f64, _f64, _f64, C.c_int, _i64, _i64, _u64, _vp, _vp, C.c_size_t]
        L.ref_bench_poisson.argtypes = [_vp, _i64, _vp, _vp, C.c_int, _vp]
        L.ref_bench_poisson.restype = _f64
        L.ref_bench_overloaded.argtypes = [_vp, _i64, C.c_int, C.c_int, C.c_int, _f64, _i64, C.c_int, _vp]
        L.ref_bench_overloaded.restype = _f64

    def set_empirical(self, prefill_values, decode_values):
        """Lists for the kind-2 (Empirical) distributions of the calls below."""
        self._pv = np.ascontiguousarray(prefill_values, np.int64)
        self._dv = np.ascontiguousarray(decode_values, np.int64)
        self.lib.ref_set_empirical(abi.ptr(self._pv), self._pv.shape[0], abi.ptr(self._dv), self._dv.shape[0])

    def sample_instance(self, s_max=64, p=0.02, rate=50.0, duration=10.0, seed=0,
                        prefill_kind=0, decode_kind=0, fixed_o=1):
        n = np.zeros(1, np.int64)
        err = _errbuf()
        rc = self.lib.ref_sample_instance(prefill_kind, s_max, decode_kind, p, fixed_o, rate, duration, seed, None, 0, abi.ptr(n), err, 512)
        if rc:
            raise ValueError(err.value.decode())
        out = np.zeros(int(n[0]), abi.request_dtype)
        self.lib.ref_sample_instance(prefill_kind, s_max, decode_kind, p, fixed_o, rate, duration, seed, abi.ptr(out), out.shape[0], abi.ptr(n), err, 512)
        return out

    def _collect(self, h, G):
        K = self.lib.ref_res_steps(h)
        st = StepSeries(K, G)
        if K:
            self.lib.ref_res_step_arrays(h, abi.ptr(st.k), abi.ptr(st.clock_start), abi.ptr(st.dt), abi.ptr(st.max_load), abi.ptr(st.active_count), abi.ptr(st.loads))
        lists = []
        for which in (0, 1):
            tot = self.lib.ref_res_list_total(h, which)
            off = np.zeros(K + 1, np.int64)
            ids = np.zeros(max(1, tot), np.int32)
            self.lib.ref_res_list(h, which, abi.ptr(off), abi.ptr(ids))
            lists.append([ids[off[k]:off[k + 1]].tolist() for k in range(K)])
        st.admitted, st.completed = lists
        n = self.lib.ref_res_n_requests(h)
        rq = {
            "id": np.zeros(n, np.int32),
            "arrival_step": np.zeros(n, np.int64),
            "start_step": np.zeros(n, np.int64),
            "admit_clock": np.zeros(n),
            "finish_clock": np.zeros(n),
            "decode": np.zeros(n, np.int64),
            "completed": np.zeros(n, np.uint8),
        }
        if n:
            self.lib.ref_res_requests(h, *[abi.ptr(rq[k]) for k in ("id", "arrival_step", "start_step", "admit_clock", "finish_clock", "decode", "completed")])
        m = np.zeros(7)
        has = bool(self.lib.ref_res_has_metrics(h))
        if has:
            self.lib.ref_res_metrics(h, abi.ptr(m))
        metrics = dict(zip(abi.METRIC_FIELDS, m.tolist())) if has else None
        completed_all = bool(self.lib.ref_res_completed_all(h))
        self.lib.ref_res_free(h)
        return st, rq, metrics, completed_all

    def run_poisson(self, sc, trace):
        sc = np.ascontiguousarray(sc, dtype=abi.scenario_dtype).reshape(())
        trace = np.ascontiguousarray(trace, dtype=abi.request_dtype)
        code = C.c_int(0)
        err = _errbuf()
        h = self.lib.ref_run_poisson(abi.ptr(sc), abi.ptr(trace), trace.shape[0], C.byref(code), err, 512)
        if not h:
            return code.value, err.value.decode(), None
        return 0, "", self._collect(h, int(sc["workers"]))

    def run_overloaded(self, sc, s_max=64, p=0.02, prefill_kind=0, decode_kind=0, fixed_o=1):
        sc = np.ascontiguousarray(sc, dtype=abi.scenario_dtype).reshape(())
        code = C.c_int(0)
        err = _errbuf()
        h = self.lib.ref_run_overloaded(abi.ptr(sc), prefill_kind, s_max, decode_kind, p, fixed_o, C.byref(code), err, 512)
        if not h:
            return code.value, err.value.decode(), None
        return 0, "", self._collect(h, int(sc["workers"]))

    def assign(self, policy, previews, caps, active_counts, futures, H, limit=200000):
        previews = np.ascontiguousarray(previews, np.float64).reshape(-1, H + 1)
        futures = np.ascontiguousarray(futures, np.float64).reshape(-1, H + 1)
        caps = np.ascontiguousarray(caps, np.int32)
        active_counts = np.ascontiguousarray(active_counts, np.int32)
        G = caps.shape[0]
        pairs = np.zeros(2 * max(1, int(caps.clip(min=0).sum())), np.int32)
        npairs = np.zeros(1, np.int64)
        cost = np.zeros(1)
        err = _errbuf()
        rc = self.lib.ref_assign(policy, previews.shape[0], abi.ptr(previews), G, abi.ptr(caps), abi.ptr(active_counts), abi.ptr(futures), H, limit, abi.ptr(pairs), abi.ptr(npairs), abi.ptr(cost), err, 512)
        return rc, [(int(pairs[2 * j]), int(pairs[2 * j + 1])) for j in range(int(npairs[0]))], float(cost[0])

    def estimate_iir(self, b_list, g_list, trials, steps, warmup, seed, s_max=64, p=0.02, drift=0.0,
                     overhead=9.775e-3, per_token=1.005e-7, backlog=1.0, prefill_kind=0, decode_kind=0, fixed_o=1):
        b = np.ascontiguousarray(b_list, np.int32)
        g = np.ascontiguousarray(g_list, np.int32)
        out = np.zeros((len(b) * len(g), 8))
        err = _errbuf()
        rc = self.lib.ref_estimate_iir(abi.ptr(b), len(b), abi.ptr(g), len(g), prefill_kind, s_max, decode_kind, p, fixed_o, drift, overhead, per_token, backlog, trials, steps, warmup, seed, abi.ptr(out), err, 512)
        if rc:
            raise ValueError(err.value.decode())
        return out

    def bench_overloaded(self, scen, threads, s_max=64, p=0.02, prefill_kind=0, decode_kind=0, fixed_o=1):
        scen = np.ascontiguousarray(scen, abi.scenario_dtype)
        ws = np.zeros(1, np.int64)
        sec = self.lib.ref_bench_overloaded(abi.ptr(scen), scen.shape[0], prefill_kind, s_max, decode_kind, p,
                                            fixed_o, threads, abi.ptr(ws))
        return sec, int(ws[0])

    def bench_poisson(self, scen, inputs, traces, threads):
        scen = np.ascontiguousarray(scen, abi.scenario_dtype)
        ws = np.zeros(1, np.int64)
        sec = self.lib.ref_bench_poisson(abi.ptr(scen), scen.shape[0], abi.ptr(np.ascontiguousarray(inputs, abi.input_dtype)), abi.ptr(np.ascontiguousarray(traces, abi.request_dtype)), threads, abi.ptr(ws))
        return sec, int(ws[0])


def _trim(st, K):
    for name in ("k", "clock_start", "dt", "max_load", "active_count", "loads"):
        setattr(st, name, getattr(st, name)[:K])
    st.k = np.arange(K, dtype=np.int64)


def _poisson_step_bound(trace, sc):
    """Generous cap on the Poisson step count for sink sizing (the run reports
    STEP_OVERFLOW if exceeded)."""
    n = trace.shape[0]
    if n == 0:
        return 1
    work = int(np.asarray(trace["decode"], np.int64).sum())
    G, B = int(sc["workers"]), int(sc["batch"])
    horizon_s = float(trace["arrival_time"][-1])
    steps_to_last = int(horizon_s / max(float(sc["overhead"]), 1e-6)) + 1
    return int(min(int(sc["max_steps"]), steps_to_last + work // max(1, G * B) + int(trace["decode"].max()) + 1024 + work // 8))


def derive_lists(rq, K):
    """admitted / completed per-step id lists from per-request (start_step, worker)
    data, in the reference's orders: admitted = waiting-index order (= id order in
    Poisson mode, engine.hpp:235-248); completed = worker-major then active
    insertion order (engine.hpp:149-156), insertion order = (start_step, id)."""
    admitted = [[] for _ in range(K)]
    completed = [[] for _ in range(K)]
    x = np.asarray(rq["start_step"], np.int64)
    ids = np.nonzero(x >= 0)[0]
    for i in ids:
        if x[i] < K:
            admitted[x[i]].append(int(i))
    dec = np.asarray(rq["decode"], np.int64)
    f = x + dec - 1
    key = []
    for i in ids:
        if f[i] < K:
            key.append((int(f[i]), int(rq["worker"][i]), int(x[i]), int(i)))
    key.sort()
    for fk, g, xs, i in key:
        completed[fk].append(i)
    return admitted, completed
