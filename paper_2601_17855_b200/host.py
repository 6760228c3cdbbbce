"""ctypes binding of libbfsim_gpu.so (include/bfsim_gpu.h).

This is the host-side plumbing of the product path: it loads the in-tree CUDA
library and fails loudly when it is missing. There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import abi

_LIB = None
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libbfsim_gpu.so")

_vp, _i32, _i64, _u64, _f64, _sz = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_size_t


class BfsimError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class InvalidArgument(BfsimError, ValueError):
    """std::invalid_argument in the reference."""


class LogicError(BfsimError):
    """std::logic_error in the reference."""


def _raise(code, err):
    msg = err.value.decode(errors="replace") if hasattr(err, "value") else str(err)
    if code == abi.EINVAL:
        raise InvalidArgument(code, msg)
    if code == abi.ELOGIC:
        raise LogicError(code, msg)
    raise BfsimError(code, msg)


def lib():
    """Load libbfsim_gpu.so (building it first if absent and nvcc exists)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        from . import build

        build.build()
    L = C.CDLL(LIB_PATH)
    L.bfsim_abi_version.restype = C.c_int
    L.bfsim_ctx_create.argtypes = [C.c_int, C.POINTER(_vp), _vp, _sz]
    L.bfsim_ctx_destroy.argtypes = [_vp]
    L.bfsim_sample_instance.argtypes = [C.c_int, C.c_int, C.c_int, _f64, _i64, _f64, _f64, _u64, _vp, _i64, _vp, _vp, _sz]
    L.bfsim_sample_stream.argtypes = [C.c_int, C.c_int, C.c_int, _f64, _i64, _u64, _i64, _vp, _vp, _sz]
    L.bfsim_prepare_trace.argtypes = [_vp, _i64, _vp, _vp, _vp, _sz]
    L.bfsim_prepare_stream.argtypes = [_vp, _i64, _vp, _vp, _vp, _sz]
    L.bfsim_run_batch.argtypes = [_vp, _vp, _i64, _vp, _i32, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _i64, _vp, _i64, _vp, _vp, _sz]
    L.bfsim_run_batch_device.argtypes = [_vp, _vp, _i64, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz]
    L.bfsim_last_launch_count.argtypes = [_vp]
    L.bfsim_last_launch_count.restype = _i64
    L.bfsim_last_step_kernel_ms.argtypes = [_vp]
    L.bfsim_last_step_kernel_ms.restype = _f64
    L.bfsim_iir_reduce.argtypes = [_vp, _vp, _i32, _i32, _vp, _vp, _sz]
    assert L.bfsim_abi_version() == 1
    _LIB = L
    return L


def _err():
    return C.create_string_buffer(1024)


# --------------------------------------------------------------- host batcher
def sample_instance(seed, *, rate, duration, s_max=64, p=0.02, prefill_kind=0, decode_kind=0, fixed_o=1):
    """sample_instance (workload.hpp:241-266), byte-identical traces."""
    L, err = lib(), _err()
    n = np.zeros(1, np.int64)
    rc = L.bfsim_sample_instance(prefill_kind, s_max, decode_kind, p, fixed_o, rate, duration, seed, None, 0, abi.ptr(n), err, 1024)
    if rc:
        _raise(rc, err)
    out = np.zeros(int(n[0]), abi.request_dtype)
    rc = L.bfsim_sample_instance(prefill_kind, s_max, decode_kind, p, fixed_o, rate, duration, seed, abi.ptr(out), out.shape[0], abi.ptr(n), err, 1024)
    if rc:
        _raise(rc, err)
    return out


def sample_stream(seed, n, *, s_max=64, p=0.02, prefill_kind=0, decode_kind=0, fixed_o=1):
    """The (prefill, decode) draws of run_overloaded's top-up (oracle.hpp:177-183)."""
    L, err = lib(), _err()
    out = np.zeros(int(n), abi.sample_dtype)
    rc = L.bfsim_sample_stream(prefill_kind, s_max, decode_kind, p, fixed_o, seed, int(n), abi.ptr(out), err, 1024)
    if rc:
        _raise(rc, err)
    return out


def prepare(records):
    """(bfsim_input_t, class_base) for one trace (request_dtype) or stream (sample_dtype)."""
    L, err = lib(), _err()
    records = np.ascontiguousarray(records)
    info = np.zeros((), abi.input_dtype)
    fn = L.bfsim_prepare_trace if records.dtype == abi.request_dtype else L.bfsim_prepare_stream
    rc = fn(abi.ptr(records), records.shape[0], abi.ptr(info), None, err, 1024)
    if rc:
        _raise(rc, err)
    cb = np.zeros(int(info["s_max"]) + 2, np.int32)
    rc = fn(abi.ptr(records), records.shape[0], abi.ptr(info), abi.ptr(cb), err, 1024)
    if rc:
        _raise(rc, err)
    return info, cb


class InputPool:
    """Concatenated traces or streams + their bfsim_input_t table and class_base pool."""

    def __init__(self, arrays):
        arrays = [np.ascontiguousarray(a) for a in arrays]
        self.kind = "stream" if (arrays and arrays[0].dtype == abi.sample_dtype) else "trace"
        dt = abi.sample_dtype if self.kind == "stream" else abi.request_dtype
        infos, cbs = [], []
        off = cboff = 0
        for a in arrays:
            info, cb = prepare(a)
            info["offset"] = off
            info["class_base_offset"] = cboff
            infos.append(info)
            cbs.append(cb)
            off += a.shape[0]
            cboff += cb.shape[0]
        self.records = np.concatenate(arrays) if arrays else np.zeros(0, dt)
        self.records = np.ascontiguousarray(self.records, dt)
        self.inputs = np.array(infos, abi.input_dtype) if infos else np.zeros(0, abi.input_dtype)
        self.class_base = np.concatenate(cbs).astype(np.int32) if cbs else np.zeros(1, np.int32)


# ----------------------------------------------------------------- engine
class Context:
    """One CUDA device (bfsim_ctx_t). Not thread-safe."""

    def __init__(self, device=0):
        L, err = lib(), _err()
        h = _vp()
        rc = L.bfsim_ctx_create(device, C.byref(h), err, 1024)
        if rc:
            _raise(rc, err)
        self.h = h
        self.device = device

    def close(self):
        if self.h:
            lib().bfsim_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def last_launches(self):
        return int(lib().bfsim_last_launch_count(self.h))

    @property
    def last_kernel_ms(self):
        return float(lib().bfsim_last_step_kernel_ms(self.h))

    def run_batch(self, scen, pool: InputPool, *, emit_steps=False, emit_requests=False,
                  step_capacity=None):
        """Host-pointer entry (the end-to-end path). Returns a BatchResult."""
        L, err = lib(), _err()
        scen = np.array(scen, abi.scenario_dtype, copy=True).reshape(-1)
        n = scen.shape[0]
        res = np.zeros(n, abi.result_dtype)
        steps = reqs = None
        sink_s = sink_r = None
        nrec = nload = nreq = 0
        if emit_steps:
            caps = np.array([_step_cap(s, pool, step_capacity) for s in scen], np.int64)
            scen["step_capacity"] = caps
            scen["step_offset"] = np.concatenate([[0], np.cumsum(caps)[:-1]])
            lcaps = caps * scen["workers"]
            scen["load_offset"] = np.concatenate([[0], np.cumsum(lcaps)[:-1]])
            nrec, nload = int(caps.sum()), int(lcaps.sum())
            steps = dict(clock_start=np.zeros(nrec), dt=np.zeros(nrec), max_load=np.zeros(nrec),
                         active_count=np.zeros(nrec, np.int64), loads=np.zeros(max(1, nload)))
            sink_s = _StepSink(*[abi.ptr(steps[k]) for k in ("clock_start", "dt", "max_load", "active_count", "loads")])
        if emit_requests:
            lens = pool.inputs["length"][scen["input_id"]]
            scen["req_offset"] = np.concatenate([[0], np.cumsum(lens)[:-1]])
            nreq = int(lens.sum())
            reqs = dict(arrival_step=np.zeros(nreq, np.int32), start_step=np.zeros(nreq, np.int32),
                        worker=np.zeros(nreq, np.int32), admit_clock=np.zeros(nreq), finish_clock=np.zeros(nreq))
            sink_r = _ReqSink(*[abi.ptr(reqs[k]) for k in ("arrival_step", "start_step", "worker", "admit_clock", "finish_clock")])
        is_stream = pool.kind == "stream"
        rc = L.bfsim_run_batch(
            self.h, abi.ptr(scen), n, abi.ptr(pool.inputs), pool.inputs.shape[0],
            abi.ptr(pool.class_base), pool.class_base.shape[0],
            None if is_stream else abi.ptr(pool.records), 0 if is_stream else pool.records.shape[0],
            abi.ptr(pool.records) if is_stream else None, pool.records.shape[0] if is_stream else 0,
            C.byref(sink_s) if sink_s else None, nrec, nload,
            C.byref(sink_r) if sink_r else None, nreq, abi.ptr(res), err, 1024,
        )
        if rc not in (abi.OK, abi.PARTIAL):
            _raise(rc, err)
        return BatchResult(scen, res, steps, reqs)


class _StepSink(C.Structure):
    _fields_ = [("clock_start", _vp), ("dt", _vp), ("max_load", _vp), ("active_count", _vp), ("loads", _vp)]


class _ReqSink(C.Structure):
    _fields_ = [("arrival_step", _vp), ("start_step", _vp), ("worker", _vp), ("admit_clock", _vp), ("finish_clock", _vp)]


def _step_cap(s, pool, explicit):
    if explicit is not None:
        return int(explicit)
    if s["mode"] == abi.OVERLOADED:
        return int(s["warmup"] + s["steps"])
    info = pool.inputs[s["input_id"]]
    N = int(info["length"])
    if N == 0:
        return 1
    recs = pool.records[int(info["offset"]): int(info["offset"]) + N]
    work = int(np.asarray(recs["decode"], np.int64).sum())
    G, B = int(s["workers"]), int(s["batch"])
    span = float(recs["arrival_time"][-1]) / max(float(s["overhead"]), 1e-6)
    bound = int(span) + work // max(1, G * B) + int(recs["decode"].max()) + 64 + work // 16
    return int(min(int(s["max_steps"]), bound))


class BatchResult:
    def __init__(self, scen, res, steps, reqs):
        self.scen, self.res, self._steps, self._reqs = scen, res, steps, reqs

    def __len__(self):
        return self.res.shape[0]

    def metrics(self, i):
        return {k: float(self.res[i][k]) for k in abi.METRIC_FIELDS}

    def steps(self, i):
        """Per-step arrays of scenario i (all simulated steps; overloaded includes warm-up)."""
        s = self.scen[i]
        K = int(min(self.res[i]["steps_run"], s["step_capacity"]))
        o, lo, G = int(s["step_offset"]), int(s["load_offset"]), int(s["workers"])
        d = {k: self._steps[k][o:o + K] for k in ("clock_start", "dt", "max_load", "active_count")}
        d["loads"] = self._steps["loads"][lo:lo + K * G].reshape(K, G)
        return d

    def requests(self, i, n):
        o = int(self.scen[i]["req_offset"])
        return {k: v[o:o + n] for k, v in self._reqs.items()}


def iir_reduce(fcfs_means, bfio_means):
    """estimate_iir's reducer (oracle.hpp:290-312). Inputs: [cells, trials]."""
    L, err = lib(), _err()
    f = np.ascontiguousarray(fcfs_means, np.float64)
    b = np.ascontiguousarray(bfio_means, np.float64)
    cells, trials = f.shape
    out = np.zeros((cells, 4))
    rc = L.bfsim_iir_reduce(abi.ptr(f), abi.ptr(b), trials, cells, abi.ptr(out), err, 1024)
    if rc:
        _raise(rc, err)
    return out
