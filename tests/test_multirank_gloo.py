"""world_size-2 gloo test of the multi-GPU host logic (paper_2601_17855_b200.parallel)
on CPU: each rank computes its shard of a scenario table (with the CPU oracle
standing in for its GPU, which this box does not have), then the per-scenario
results are gathered in global order and the exact sums all-reduced. The
gathered table must equal the single-process table byte for byte."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _table():
    from paper_2601_17855_b200 import abi, host

    traces = [host.sample_instance(seed, rate=300.0, duration=0.5, s_max=32, p=0.1) for seed in range(1, 7)]
    scen = []
    for j in range(6):
        for pol in (abi.FCFS, abi.BFIO_GREEDY):
            scen.append(abi.scenario(policy=pol, workers=4, batch=8, horizon=j % 3, input_id=j))
    return traces, np.array(scen, abi.scenario_dtype)


def _run_shard(lo, hi):
    from oracle.oracle import OracleLib
    from paper_2601_17855_b200 import abi

    traces, scen = _table()
    orc = OracleLib()
    out = np.zeros(hi - lo, abi.result_dtype)
    for i in range(lo, hi):
        rc, res, st, rq = orc.run_poisson(scen[i], traces[scen[i]["input_id"]])
        out[i - lo] = res
    return out


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2601_17855_b200 import host, parallel

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    traces, scen = _table()
    pool = host.InputPool(traces)
    lo, hi = parallel.shard_range(parallel.estimated_work(scen, pool.inputs), world, rank)
    local = _run_shard(lo, hi)
    full = parallel.gather_results(local, lo, scen.shape[0])
    sums = parallel.allreduce_exact(local)
    q.put((rank, lo, hi, full.tobytes(), sums))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_partitions():
    from paper_2601_17855_b200 import parallel

    rng = np.random.default_rng(0)
    for world in (1, 2, 3, 8):
        w = rng.uniform(1, 10, 37)
        cuts = [parallel.shard_range(w, world, r) for r in range(world)]
        assert cuts[0][0] == 0 and cuts[-1][1] == 37
        for a, b in zip(cuts, cuts[1:]):
            assert a[1] == b[0]
        if world > 1:
            sums = [w[lo:hi].sum() for lo, hi in cuts]
            assert max(sums) - min(sums) <= 2 * w.max() + 1e-9


def test_gloo_world2_gather_matches_single_process():
    import multiprocessing as mp

    from paper_2601_17855_b200 import abi

    traces, scen = _table()
    single = _run_shard(0, scen.shape[0])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got.sort()
    assert got[0][1] == 0 and got[1][2] == scen.shape[0] and got[0][2] == got[1][1]
    for rank, lo, hi, full, sums in got:
        assert full == single.tobytes()
        assert sums == [int(single["imb_total_i"].sum()), int(single["total_workload_i"].sum()),
                        int(single["tokens_i"].sum())]
    assert single.dtype == abi.result_dtype
