"""Multi-GPU plumbing: scenarios are independent trajectories,
so the path shards with no data-path collective.

* shard_range: a contiguous, work-balanced slice of the scenario table per
  rank (one process per GPU).
* gather_results: the one real exchange step. Every rank's per-scenario
  bfsim_result_t rows are gathered to rank 0 in global scenario order, so the
  reduction there is deterministic and matches the single-GPU (and CPU)
  reducer bit for bit.
* allreduce_exact: exact int64 sums (imbalance totals, workload, tokens).

torch.distributed is only the transport (NCCL on B200s, gloo in the CPU tests).
"""
from __future__ import annotations

import numpy as np

from . import abi


def shard_range(work, world: int, rank: int):
    """[lo, hi) of scenarios for `rank` such that the per-rank sums of `work`
    (estimated worker-steps per scenario, in scenario order) are balanced."""
    work = np.asarray(work, dtype=np.float64)
    n = work.shape[0]
    if world <= 1:
        return 0, n
    cum = np.concatenate([[0.0], np.cumsum(work)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(cum, total * r / world, side="left")))
    cuts.append(n)
    cuts = np.maximum.accumulate(np.clip(cuts, 0, n))
    return int(cuts[rank]), int(cuts[rank + 1])


def estimated_work(scen, inputs):
    """Worker-steps estimate per scenario: overloaded = G*(warmup+steps);
    Poisson ~ G * N * E[o] / (G*B) (+1 so empty traces still count)."""
    scen = np.asarray(scen, abi.scenario_dtype)
    out = np.zeros(scen.shape[0])
    for i, s in enumerate(scen):
        if s["mode"] == abi.OVERLOADED:
            out[i] = float(s["workers"]) * float(s["warmup"] + s["steps"])
        else:
            n = float(inputs[s["input_id"]]["length"])
            out[i] = 1.0 + n * 50.0 / float(s["batch"])
    return out


def gather_results(local: np.ndarray, lo: int, n_total: int, device=None):
    """All-gather per-scenario result rows (bfsim_result_t) from every rank;
    returns the full table in global scenario order on every rank."""
    import torch
    import torch.distributed as dist

    local = np.ascontiguousarray(local, abi.result_dtype)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local
    world = dist.get_world_size()
    dev = device if device is not None else torch.device("cpu")
    raw = torch.from_numpy(local.view(np.uint8).reshape(-1).copy()).to(dev)
    meta = torch.tensor([lo, local.shape[0]], dtype=torch.int64, device=dev)
    metas = [torch.zeros_like(meta) for _ in range(world)]
    dist.all_gather(metas, meta)
    rows = max(int(m[1]) for m in metas)
    pad = torch.zeros(rows * abi.result_dtype.itemsize, dtype=torch.uint8, device=dev)
    pad[: raw.numel()] = raw
    bufs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    out = np.zeros(n_total, abi.result_dtype)
    for m, b in zip(metas, bufs):
        lo_r, cnt = int(m[0]), int(m[1])
        arr = b.cpu().numpy()[: cnt * abi.result_dtype.itemsize].view(abi.result_dtype)
        out[lo_r: lo_r + cnt] = arr
    return out


def allreduce_exact(results: np.ndarray, device=None):
    """Exact int64 sums over all ranks of imb_total_i, total_workload_i, tokens_i."""
    import torch
    import torch.distributed as dist

    res = np.asarray(results, abi.result_dtype)
    v = torch.tensor([int(res["imb_total_i"].sum()), int(res["total_workload_i"].sum()),
                      int(res["tokens_i"].sum())], dtype=torch.int64,
                     device=device if device is not None else "cpu")
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(v, op=dist.ReduceOp.SUM)
    return [int(x) for x in v.tolist()]
