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
    L.bfsim_sample_instance_dist.argtypes = [_vp, _vp, _f64, _f64, _u64, _vp, _i64, _vp, _vp, _sz]
    L.bfsim_sample_stream_dist.argtypes = [_vp, _vp, _u64, _i64, _vp, _vp, _sz]
    L.bfsim_prepare_trace.argtypes = [_vp, _i64, _vp, _vp, _vp, _sz]
    L.bfsim_prepare_stream.argtypes = [_vp, _i64, _vp, _vp, _vp, _sz]
    L.bfsim_run_batch.argtypes = [_vp, _vp, _i64, _vp, _i32, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _i64, _vp, _i64, _vp, _vp, _sz]
    L.bfsim_run_batch_device.argtypes = [_vp, _vp, _i64, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz]
    L.bfsim_last_launch_count.argtypes = [_vp]
    L.bfsim_last_launch_count.restype = _i64
    L.bfsim_last_step_kernel_ms.argtypes = [_vp]
    L.bfsim_last_step_kernel_ms.restype = _f64
    L.bfsim_iir_reduce.argtypes = [_vp, _vp, _i32, _i32, _vp, _vp, _sz]
    L.bfsim_assign_batch.argtypes = [_vp, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _vp, _i64, _i64, _vp, _i64,
                                     _vp, _vp, _vp, _vp, _sz]
    L.bfsim_generate_bounds.argtypes = [_vp, _i32, _i64, _vp, _vp, _vp, _sz]
    L.bfsim_generate_traces.argtypes = [_vp, _vp, _i32, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _sz]
    L.bfsim_generate_streams.argtypes = [_vp, _vp, _i32, _i64, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _sz]
    L.bfsim_libm_log_host.argtypes = [_vp, _vp, _i64]
    L.bfsim_libm_log_host.restype = None
    assert L.bfsim_abi_version() == 1
    _LIB = L
    return L


def _err():
    return C.create_string_buffer(1024)


# --------------------------------------------------------------- host batcher
class _Dist(C.Structure):
    _fields_ = [("kind", C.c_int32), ("reserved", C.c_int32), ("fixed", C.c_int64), ("p", C.c_double),
                ("values", C.c_void_p), ("n_values", C.c_int64)]


def _dist(kind, fixed, p, values):
    arr = None if values is None else np.ascontiguousarray(values, np.int64)
    d = _Dist(2 if arr is not None else kind, 0, int(fixed), float(p),
              arr.ctypes.data if arr is not None else None, 0 if arr is None else arr.shape[0])
    return d, arr


def sample_instance(seed, *, rate, duration, s_max=64, p=0.02, prefill_kind=0, decode_kind=0, fixed_o=1,
                    prefill_values=None, decode_values=None):
    """sample_instance (workload.hpp:241-266), byte-identical traces. prefill_values /
    decode_values select the Empirical distributions (workload.hpp:109-118, 185-193)."""
    if prefill_values is not None or decode_values is not None:
        L, err = lib(), _err()
        pd, pa = _dist(prefill_kind, s_max, 0.0, prefill_values)
        dd, da = _dist(decode_kind, fixed_o, p, decode_values)
        n = np.zeros(1, np.int64)
        rc = L.bfsim_sample_instance_dist(C.byref(pd), C.byref(dd), rate, duration, seed, None, 0, abi.ptr(n), err, 1024)
        if rc:
            _raise(rc, err)
        out = np.zeros(int(n[0]), abi.request_dtype)
        rc = L.bfsim_sample_instance_dist(C.byref(pd), C.byref(dd), rate, duration, seed, abi.ptr(out), out.shape[0],
                                          abi.ptr(n), err, 1024)
        if rc:
            _raise(rc, err)
        return out
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


def sample_stream(seed, n, *, s_max=64, p=0.02, prefill_kind=0, decode_kind=0, fixed_o=1, prefill_values=None,
                  decode_values=None):
    """The (prefill, decode) draws of run_overloaded's top-up (oracle.hpp:177-183)."""
    L, err = lib(), _err()
    out = np.zeros(int(n), abi.sample_dtype)
    if prefill_values is not None or decode_values is not None:
        pd, pa = _dist(prefill_kind, s_max, 0.0, prefill_values)
        dd, da = _dist(decode_kind, fixed_o, p, decode_values)
        rc = L.bfsim_sample_stream_dist(C.byref(pd), C.byref(dd), seed, int(n), abi.ptr(out), err, 1024)
        if rc:
            _raise(rc, err)
        return out
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
        self._arrays = arrays

    def add_prefix(self, i, length):
        """A further input: the first `length` records of input i, sharing its
        records (no copy) with its own statistics and class_base. A
        run_overloaded stream is prefix-stable (the draws of mt19937_64(seed)
        in order), so a small-G scenario can run on a short prefix of the
        stream a large-G one needs, and the engine sizes its per-trajectory
        class deques by the input it runs on. Returns the new input id."""
        length = int(min(length, self.inputs[i]["length"]))
        info, cb = prepare(self._arrays[i][:length])
        info["offset"] = self.inputs[i]["offset"]
        info["class_base_offset"] = self.class_base.shape[0]
        self.inputs = np.concatenate([self.inputs, np.array([info], abi.input_dtype)])
        self.class_base = np.concatenate([self.class_base, cb.astype(np.int32)])
        return self.inputs.shape[0] - 1


class _GenSpec(C.Structure):
    _fields_ = [("prefill", _Dist), ("decode", _Dist), ("rate", C.c_double), ("duration", C.c_double),
                ("seed", C.c_uint64)]


def libm_log(x):
    """The host twin of the device's glibc log (csrc/libm_log.cuh)."""
    x = np.ascontiguousarray(x, np.float64)
    y = np.empty_like(x)
    lib().bfsim_libm_log_host(abi.ptr(x), abi.ptr(y), x.size)
    return y


class DevicePool:
    """Traces (sample_instance, workload.hpp:241-266) or overloaded sample
    streams (oracle.hpp:177-183) generated in HBM by the device generator
    (bfsim_generate_traces / bfsim_generate_streams),
    byte-identical to sample_instance / sample_stream above. Usable wherever an
    InputPool goes into DeviceBatch; `records` / `class_base` are device
    tensors, `inputs` the host table the planner needs.

    specs: one dict per input with the keyword arguments of sample_instance
    (seed, rate, duration, s_max, p, prefill_kind, decode_kind, fixed_o,
    prefill_values, decode_values); `samples` selects stream mode."""

    def __init__(self, ctx, specs, *, samples=None, stream=None):
        import torch

        L, err = lib(), _err()
        self.kind = "stream" if samples is not None else "trace"
        keep = []
        arr = (_GenSpec * max(1, len(specs)))()
        for i, sp in enumerate(specs):
            pd, pa = _dist(sp.get("prefill_kind", 0), sp.get("s_max", 64), 0.0, sp.get("prefill_values"))
            dd, da = _dist(sp.get("decode_kind", 0), sp.get("fixed_o", 1), sp.get("p", 0.02), sp.get("decode_values"))
            keep += [pa, da]
            arr[i] = _GenSpec(pd, dd, float(sp.get("rate", 1.0)), float(sp.get("duration", 1.0)), int(sp["seed"]))
        n = len(specs)
        nrec, ncb = np.zeros(1, np.int64), np.zeros(1, np.int64)
        rc = L.bfsim_generate_bounds(arr, n, -1 if samples is None else int(samples), abi.ptr(nrec), abi.ptr(ncb),
                                     err, 1024)
        if rc:
            _raise(rc, err)
        dev = torch.device("cuda", ctx.device)
        isz = (abi.sample_dtype if samples is not None else abi.request_dtype).itemsize
        self.records = torch.empty(max(1, int(nrec[0]) * isz), dtype=torch.uint8, device=dev)
        self.class_base = torch.empty(max(1, int(ncb[0])), dtype=torch.int32, device=dev)
        self.inputs = np.zeros(n, abi.input_dtype)
        s = stream if stream is not None else torch.cuda.current_stream(ctx.device)
        if samples is None:
            rc = L.bfsim_generate_traces(ctx.h, arr, n, self.records.data_ptr(), int(nrec[0]),
                                         self.class_base.data_ptr(), int(ncb[0]), abi.ptr(self.inputs),
                                         C.c_void_p(s.cuda_stream), err, 1024)
        else:
            rc = L.bfsim_generate_streams(ctx.h, arr, n, int(samples), self.records.data_ptr(), int(nrec[0]),
                                          self.class_base.data_ptr(), int(ncb[0]), abi.ptr(self.inputs),
                                          C.c_void_p(s.cuda_stream), err, 1024)
        if rc:
            _raise(rc, err)
        self.capacity_records = int(nrec[0])

    def host_records(self, i):
        """Input i copied back to the host (request_dtype / sample_dtype)."""
        dt = abi.sample_dtype if self.kind == "stream" else abi.request_dtype
        info = self.inputs[i]
        a, b = int(info["offset"]) * dt.itemsize, int(info["offset"] + info["length"]) * dt.itemsize
        return self.records[a:b].cpu().numpy().view(dt)

    def trace_stats(self, i):
        """(sum of decode lengths, last arrival time, largest decode) of trace i,
        reduced on the device (the step-sink capacity heuristic)."""
        import torch

        info = self.inputs[i]
        a, n = int(info["offset"]), int(info["length"])
        rec = self.records[a * 16:(a + n) * 16]
        dec = rec.view(torch.int32).view(n, 4)[:, 3].to(torch.int64)
        last = float(rec.view(torch.float64).view(n, 2)[-1, 0].item())
        return int(dec.sum().item()), last, int(info["max_decode"])

    def host_class_base(self, i):
        info = self.inputs[i]
        a = int(info["class_base_offset"])
        return self.class_base[a:a + int(info["s_max"]) + 2].cpu().numpy()


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
        """Host-pointer entry (the end-to-end path). Returns a BatchResult.
        Step sinks are sized by a heuristic; if any scenario overflows it the
        batch is re-run once with the exact step counts."""
        br = self._run_batch(scen, pool, emit_steps=emit_steps, emit_requests=emit_requests,
                             step_capacity=step_capacity)
        if emit_steps and (br.res["flags"] & abi.FLAG_STEP_OVERFLOW).any():
            br = self._run_batch(scen, pool, emit_steps=emit_steps, emit_requests=emit_requests,
                                 step_capacity=np.maximum(br.res["steps_run"], 1))
        return br

    def _run_batch(self, scen, pool, *, emit_steps, emit_requests, step_capacity):
        L, err = lib(), _err()
        scen = np.array(scen, abi.scenario_dtype, copy=True).reshape(-1)
        n = scen.shape[0]
        res = np.zeros(n, abi.result_dtype)
        steps = reqs = None
        sink_s = sink_r = None
        nrec = nload = nreq = 0
        if emit_steps:
            caps = _caps(scen, pool, step_capacity)
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


def _caps(scen, pool, step_capacity):
    if step_capacity is not None and np.ndim(step_capacity) > 0:
        return np.asarray(step_capacity, np.int64).reshape(-1).copy()
    return np.array([_step_cap(s, pool, step_capacity) for s in scen], np.int64)


def _step_cap(s, pool, explicit):
    if explicit is not None:
        return int(explicit)
    if s["mode"] == abi.OVERLOADED:
        return int(s["warmup"] + s["steps"])
    info = pool.inputs[s["input_id"]]
    N = int(info["length"])
    if N == 0:
        return 1
    if isinstance(pool, DevicePool):
        work, last, omax = pool.trace_stats(int(s["input_id"]))
    else:
        recs = pool.records[int(info["offset"]): int(info["offset"]) + N]
        work = int(np.asarray(recs["decode"], np.int64).sum())
        last, omax = float(recs["arrival_time"][-1]), int(recs["decode"].max())
    G, B = int(s["workers"]), int(s["batch"])
    span = last / max(float(s["overhead"]), 1e-6)
    # heuristic capacity; run_batch re-runs any scenario that overflows it
    bound = int(span) + (3 * work) // (2 * max(1, G * B)) + omax + 64
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


class DeviceBatch:
    """A scenario batch with inputs and output sinks resident in HBM (torch
    tensors are only the allocator). run() enqueues the step kernels on the
    current torch stream via bfsim_run_batch_device."""

    def __init__(self, ctx: Context, scen, pool: InputPool, *, emit_steps=True, emit_requests=True,
                 step_capacity=None):
        import torch

        self.ctx = ctx
        dev = torch.device("cuda", ctx.device)
        scen = np.array(scen, abi.scenario_dtype, copy=True).reshape(-1)
        n = scen.shape[0]

        def dbuf(arr):
            t = torch.empty(max(1, arr.nbytes), dtype=torch.uint8, device=dev)
            if arr.nbytes:
                t[: arr.nbytes].copy_(torch.from_numpy(np.ascontiguousarray(arr).view(np.uint8).reshape(-1)))
            return t

        self._keep = []
        if isinstance(pool, DevicePool):  # already resident in HBM
            self.records, self.class_base = pool.records, pool.class_base
        else:
            self.records = dbuf(pool.records)
            self.class_base = dbuf(pool.class_base)
        self.is_stream = pool.kind == "stream"
        self.pool = pool
        self.steps = self.reqs = None
        self.sink_s = self.sink_r = None
        if emit_steps:
            caps = _caps(scen, pool, step_capacity)
            scen["step_capacity"] = caps
            scen["step_offset"] = np.concatenate([[0], np.cumsum(caps)[:-1]])
            lcaps = caps * scen["workers"]
            scen["load_offset"] = np.concatenate([[0], np.cumsum(lcaps)[:-1]])
            nrec, nload = int(caps.sum()), int(lcaps.sum())
            self.steps = {
                "clock_start": torch.empty(nrec, dtype=torch.float64, device=dev),
                "dt": torch.empty(nrec, dtype=torch.float64, device=dev),
                "max_load": torch.empty(nrec, dtype=torch.float64, device=dev),
                "active_count": torch.empty(nrec, dtype=torch.int64, device=dev),
                "loads": torch.empty(max(1, nload), dtype=torch.float64, device=dev),
            }
            self.sink_s = _StepSink(*[self.steps[k].data_ptr() for k in ("clock_start", "dt", "max_load", "active_count", "loads")])
        if emit_requests:
            lens = pool.inputs["length"][scen["input_id"]]
            scen["req_offset"] = np.concatenate([[0], np.cumsum(lens)[:-1]])
            nreq = int(lens.sum())
            self.reqs = {
                "arrival_step": torch.empty(nreq, dtype=torch.int32, device=dev),
                "start_step": torch.empty(nreq, dtype=torch.int32, device=dev),
                "worker": torch.empty(nreq, dtype=torch.int32, device=dev),
                "admit_clock": torch.empty(nreq, dtype=torch.float64, device=dev),
                "finish_clock": torch.empty(nreq, dtype=torch.float64, device=dev),
            }
            self.sink_r = _ReqSink(*[self.reqs[k].data_ptr() for k in ("arrival_step", "start_step", "worker", "admit_clock", "finish_clock")])
        self.scen = scen
        self.results = torch.empty(n * abi.result_dtype.itemsize, dtype=torch.uint8, device=dev)

    def run(self, stream=None):
        import torch

        L, err = lib(), _err()
        s = stream if stream is not None else torch.cuda.current_stream(self.ctx.device)
        rc = L.bfsim_run_batch_device(
            self.ctx.h, abi.ptr(self.scen), self.scen.shape[0], abi.ptr(self.pool.inputs),
            self.pool.inputs.shape[0], self.class_base.data_ptr(),
            None if self.is_stream else self.records.data_ptr(),
            self.records.data_ptr() if self.is_stream else None,
            C.byref(self.sink_s) if self.sink_s else None,
            C.byref(self.sink_r) if self.sink_r else None,
            self.results.data_ptr(), C.c_void_p(s.cuda_stream), err, 1024,
        )
        if rc:
            _raise(rc, err)

    def result_array(self):
        return self.results.cpu().numpy().view(abi.result_dtype)


class PinnedBatch:
    """End-to-end batch through the host-pointer entry bfsim_run_batch with
    page-locked host buffers (inputs copied H2D and all outputs D2H inside
    every call)."""

    def __init__(self, ctx: Context, scen, pool: InputPool, *, step_capacity=None, emit_requests=True):
        import torch

        def pinned(n, dtype):
            t = torch.empty(max(1, int(n) * np.dtype(dtype).itemsize), dtype=torch.uint8, pin_memory=True)
            self._keep.append(t)
            return t.numpy().view(dtype)[: int(n)]

        self._keep = []
        self.ctx = ctx
        scen = np.array(scen, abi.scenario_dtype, copy=True).reshape(-1)
        # step_capacity None: metrics and request timings only (no StepRecord sink)
        caps = (np.zeros(scen.shape[0], np.int64) if step_capacity is None
                else np.asarray(step_capacity, np.int64).reshape(-1))
        scen["step_capacity"] = caps
        scen["step_offset"] = np.concatenate([[0], np.cumsum(caps)[:-1]])
        lcaps = caps * scen["workers"]
        scen["load_offset"] = np.concatenate([[0], np.cumsum(lcaps)[:-1]])
        self.nrec, self.nload = int(caps.sum()), int(lcaps.sum())
        lens = pool.inputs["length"][scen["input_id"]]
        scen["req_offset"] = np.concatenate([[0], np.cumsum(lens)[:-1]])
        self.nreq = int(lens.sum()) if emit_requests else 0
        self.scen = pinned(scen.shape[0], abi.scenario_dtype)
        self.scen[:] = scen
        self.inputs = pinned(pool.inputs.shape[0], abi.input_dtype)
        self.inputs[:] = pool.inputs
        self.class_base = pinned(pool.class_base.shape[0], np.int32)
        self.class_base[:] = pool.class_base
        self.is_stream = pool.kind == "stream"
        self.records = pinned(pool.records.shape[0], pool.records.dtype)
        self.records[:] = pool.records
        self.steps, self.sink_s = {}, None
        if step_capacity is not None:
            self.steps = {k: pinned(self.nrec, np.float64) for k in ("clock_start", "dt", "max_load")}
            self.steps["active_count"] = pinned(self.nrec, np.int64)
            self.steps["loads"] = pinned(max(1, self.nload), np.float64)
            self.sink_s = _StepSink(*[abi.ptr(self.steps[k]) for k in ("clock_start", "dt", "max_load", "active_count", "loads")])
        self.sink_r = None
        if emit_requests:
            self.reqs = {k: pinned(self.nreq, np.int32) for k in ("arrival_step", "start_step", "worker")}
            self.reqs.update({k: pinned(self.nreq, np.float64) for k in ("admit_clock", "finish_clock")})
            self.sink_r = _ReqSink(*[abi.ptr(self.reqs[k]) for k in ("arrival_step", "start_step", "worker", "admit_clock", "finish_clock")])
        self.results = pinned(scen.shape[0], abi.result_dtype)

    @property
    def h2d_bytes(self):
        return int(self.records.nbytes + self.class_base.nbytes + self.scen.nbytes + self.inputs.nbytes)

    @property
    def d2h_bytes(self):
        b = self.results.nbytes + sum(v.nbytes for v in self.steps.values())
        if self.sink_r is not None:
            b += sum(v.nbytes for v in self.reqs.values())
        return int(b)

    def run(self):
        L, err = lib(), _err()
        st = self.is_stream
        rc = L.bfsim_run_batch(
            self.ctx.h, abi.ptr(self.scen), self.scen.shape[0], abi.ptr(self.inputs), self.inputs.shape[0],
            abi.ptr(self.class_base), self.class_base.shape[0],
            None if st else abi.ptr(self.records), 0 if st else self.records.shape[0],
            abi.ptr(self.records) if st else None, self.records.shape[0] if st else 0,
            C.byref(self.sink_s) if self.sink_s is not None else None, self.nrec, self.nload,
            C.byref(self.sink_r) if self.sink_r is not None else None, self.nreq,
            abi.ptr(self.results), err, 1024,
        )
        if rc not in (abi.OK, abi.PARTIAL):
            _raise(rc, err)
        return self.results


def run_overloaded_batch(ctx: Context, jobs, *, s_max=64, p=0.02, drift=0.0, prefill_kind=0, decode_kind=0,
                         fixed_o=1, backlog=1.0, overhead=9.775e-3, per_token=1.005e-7, emit_steps=False,
                         emit_requests=False):
    """run_overloaded (oracle.hpp:138-244) for many jobs in one batch.

    jobs: iterable of (policy, H, G, B, steps, warmup, seed). Each job's
    (prefill, decode) draws from mt19937_64(seed) are pre-generated here
    (bfsim_sample_stream; policy-independent) and shared by the
    jobs with the same seed. A stream that runs dry (code 5) is doubled and
    the batch re-run, so callers see the reference's unbounded top-up.
    Returns (BatchResult, streams by seed)."""
    jobs = list(jobs)
    mean_o = 1.0 / p if decode_kind == 0 else float(fixed_o)
    need = {}
    for (_, _, G, B, steps, warmup, seed) in jobs:
        n = int(G * B * (3 + (steps + warmup) / mean_o * 1.5)) + 4096
        need[seed] = max(need.get(seed, 0), n)
    streams = {}
    for _ in range(12):
        for seed, n in need.items():
            if seed not in streams or streams[seed].shape[0] < n:
                streams[seed] = sample_stream(seed, n, s_max=s_max, p=p, prefill_kind=prefill_kind,
                                              decode_kind=decode_kind, fixed_o=fixed_o)
        order = list(need)
        pool = InputPool([streams[s] for s in order])
        # the class structures cover the distribution's whole range
        pos = {s: i for i, s in enumerate(order)}
        scen = np.array([abi.scenario(mode=abi.OVERLOADED, policy=pol, horizon=H, workers=G, batch=B, steps=steps,
                                  warmup=warmup, seed=seed, drift=drift, backlog=backlog, overhead=overhead,
                                  per_token=per_token, input_id=pos[seed])
                         for (pol, H, G, B, steps, warmup, seed) in jobs], abi.scenario_dtype)
        try:
            br = ctx.run_batch(scen, pool, emit_steps=emit_steps, emit_requests=emit_requests)
            return br, streams
        except BfsimError as e:
            if e.code != abi.ESTREAM:
                raise
        for seed in need:  # a stream ran dry: grow them all and re-run
            need[seed] *= 2
    raise BfsimError(abi.ESTREAM, "overloaded sample stream still exhausted after 12 doublings")


def estimate_iir(ctx: Context, batch_sizes, worker_counts, trials, steps, warmup, seed, *, s_max=64, p=0.02,
                 drift=0.0, backlog=1.0, overhead=9.775e-3, per_token=1.005e-7):
    """estimate_iir (oracle.hpp:263-317) on the GPU: every (B, G, trial) x
    {FCFS, BF-IO greedy H=0} trajectory in one batch, trial seed
    seed + 1000003*t + 17*B + G (oracle.hpp:279-281), reduced with the
    reference formulas (bfsim_iir_reduce). Returns rows
    [B, G, fcfs_mean, bfio_mean, ratio, stderr, trials, outside_regime]."""
    if trials < 1:
        raise InvalidArgument(abi.EINVAL, "estimate_iir: trials must be >= 1")
    jobs, cells = [], []
    for B in batch_sizes:
        for G in worker_counts:
            cells.append((B, G))
            for t in range(trials):
                ts = (seed + 1000003 * t + 17 * B + G) & ((1 << 64) - 1)
                jobs.append((abi.FCFS, 0, G, B, steps, warmup, ts))
                jobs.append((abi.BFIO_GREEDY, 0, G, B, steps, warmup, ts))
    br, _ = run_overloaded_batch(ctx, jobs, s_max=s_max, p=p, drift=drift, backlog=backlog, overhead=overhead,
                                 per_token=per_token)
    m = br.res["avg_imbalance"].reshape(len(cells), trials, 2)
    red = iir_reduce(m[:, :, 0], m[:, :, 1])
    out = np.zeros((len(cells), 8))
    for c, (B, G) in enumerate(cells):
        out[c] = [B, G, red[c, 0], red[c, 1], red[c, 2], red[c, 3], trials, float(np.sqrt(G) > B)]
    return out


class _AssignCall(C.Structure):
    _fields_ = [("policy", C.c_int32), ("n_waiting", C.c_int32), ("workers", C.c_int32), ("horizon", C.c_int32),
                ("preview_offset", C.c_int64), ("worker_offset", C.c_int64), ("future_offset", C.c_int64),
                ("pair_offset", C.c_int64)]


def assign_batch(ctx: Context, calls, search_limit=200000):
    """Many assign() calls (policies.hpp:372-382) in one launch, one warp each.

    calls: iterable of (policy, previews [n, H+1], caps [G], active_counts [G],
    futures [G, H+1]) with integer values. Returns, per call, (pairs, cost,
    status): pairs as the reference returns them (list of (waiting idx,
    worker)), cost = bfio-exact's optimum (0 for the other policies), status
    abi.OK or abi.ELIMIT (SearchLimitExceeded)."""
    L, err = lib(), _err()
    calls = list(calls)
    n = len(calls)
    arr = (_AssignCall * max(n, 1))()
    pv_parts, fu_parts, caps_parts, cnt_parts = [], [], [], []
    pvo = fuo = wo = po = 0
    for k, (pol, pv, caps, cnt, fut) in enumerate(calls):
        caps = np.asarray(caps, np.int32).reshape(-1)
        G = caps.shape[0]
        fut = np.asarray(fut, np.float64).reshape(G, -1)
        H = fut.shape[1] - 1
        pv = np.asarray(pv, np.float64).reshape(-1, H + 1)
        nw = pv.shape[0]
        U = min(nw, int(caps.clip(min=0).sum()))
        arr[k] = _AssignCall(int(pol), nw, G, H, pvo, wo, fuo, po)
        pv_parts.append(pv.reshape(-1))
        fu_parts.append(fut.reshape(-1))
        caps_parts.append(caps)
        cnt_parts.append(np.asarray(cnt, np.int32).reshape(-1))
        pvo += pv.size
        fuo += fut.size
        wo += G
        po += 2 * U
    pv_all = np.ascontiguousarray(np.concatenate(pv_parts) if pv_parts else np.zeros(1))
    fu_all = np.ascontiguousarray(np.concatenate(fu_parts) if fu_parts else np.zeros(1))
    caps_all = np.ascontiguousarray(np.concatenate(caps_parts) if caps_parts else np.zeros(1, np.int32))
    cnt_all = np.ascontiguousarray(np.concatenate(cnt_parts) if cnt_parts else np.zeros(1, np.int32))
    pairs = np.zeros(max(po, 1), np.int32)
    npairs = np.zeros(max(n, 1), np.int64)
    cost = np.zeros(max(n, 1))
    status = np.zeros(max(n, 1), np.int32)
    rc = L.bfsim_assign_batch(ctx.h, C.byref(arr), n, abi.ptr(pv_all), pvo, abi.ptr(fu_all), fuo, abi.ptr(caps_all),
                              abi.ptr(cnt_all), wo, int(search_limit), abi.ptr(pairs), po, abi.ptr(npairs),
                              abi.ptr(cost), abi.ptr(status), err, 1024)
    if rc not in (abi.OK, abi.ELIMIT):
        _raise(rc, err)
    out = []
    for k in range(n):
        o = int(arr[k].pair_offset)
        m = int(npairs[k])
        pr = [(int(pairs[o + 2 * j]), int(pairs[o + 2 * j + 1])) for j in range(m)]
        out.append((pr, float(cost[k]), int(status[k])))
    return out
