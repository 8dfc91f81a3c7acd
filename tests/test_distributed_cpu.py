"""world_size-2 gloo test of the multi-GPU plumbing on CPU (no GPU needed).

Each rank asks the library's host planner (sg_plan_query, the same code sg_plan runs) for its
shard of depth-1 subtrees, computes that shard's partial sum with the CPU oracle (standing in for
the rank's GPU), all-gathers the 2-double partials over gloo (NCCL on the GPU box) and combines them
in fixed rank order with a double-double sum, exactly as sg_finalize does.  The result must equal
the single-process oracle value: the shards partition the point set with nothing dropped or
counted twice, and the combine is order-fixed.
"""
import ctypes
import os
import socket

import mpmath as mp
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

import oracle
import sg_configs as S


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _two_sum(a, b):
    s = a + b
    bb = s - a
    return s, (a - (s - bb)) + (b - bb)


def _dd_add(x, y):
    s, e = _two_sum(x[0], y[0])
    e += x[1] + y[1]
    h = s + e
    return h, e - (h - s)


def _worker(rank, world, port, cfg, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2210_14313_b200._lib import lib, sg_options
    p = S.baseline_config(cfg)
    o = sg_options(0, 0, rank, world, 0, -1)
    sp, lo, hi = ctypes.c_ulonglong(), ctypes.c_longlong(), ctypes.c_longlong()
    rc = lib().sg_plan_query(p.d, p.q, p.rule, p.kind, ctypes.byref(o), ctypes.byref(sp), None,
                             ctypes.byref(lo), ctypes.byref(hi), None)
    assert rc == 0
    r = oracle.integrate_problem(p, lo=lo.value, hi=hi.value, include_root=(rank == 0),
                                 eval_mode=1, nthreads=2)
    assert r.npoints == sp.value
    part = torch.tensor([r.hi, r.lo], dtype=torch.float64)
    gathered = torch.zeros(2 * world, dtype=torch.float64)
    dist.all_gather_into_tensor(gathered, part)
    acc = (0.0, 0.0)
    for q in range(world):
        acc = _dd_add(acc, (float(gathered[2 * q]), float(gathered[2 * q + 1])))
    out_q.put((rank, acc, lo.value, hi.value, sp.value))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg,world", [(2, 2), (1, 2), (2, 3)])
def test_gloo_sharded_sum_equals_whole(cfg, world):
    from paper_2210_14313_b200 import build as B
    B.build()
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    res.sort()
    # every rank computed the same combined value
    assert len({r[1] for r in res}) == 1
    # contiguous, complete partition of depth-1 space, point counts add up
    assert res[0][2] == 0
    for a, b in zip(res, res[1:]):
        assert a[3] == b[2]
    p = S.baseline_config(cfg)
    whole = oracle.integrate_problem(p, eval_mode=1)
    assert sum(r[4] for r in res) == whole.npoints
    got = mp.mpf(res[0][1][0]) + mp.mpf(res[0][1][1])
    assert abs((got - mp.mpf(whole.text)) / mp.mpf(whole.text)) < 1e-28
