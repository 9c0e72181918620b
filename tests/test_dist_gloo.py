"""Multi-rank host logic on CPU (gloo, world_size 2 and 4): the global
resampling exchange plan, the all-to-all row exchange, the fixed-chunk
log-sum-exp combine and the exact fixed-point moment all-reduce.  The device
kernels are covered by the -m gpu tests; here the same collectives run on CPU
tensors so the sharded control flow is checked without GPUs."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import spa_oracle as orc
from paper_1106_0322_b200.dist import resample_plan


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("alpha", [0.05, 1.0])
def test_resample_plan_reconstructs_global_gather(world, alpha):
    rng = np.random.default_rng(world * 10 + int(alpha * 100))
    M = 512
    N = M * world
    w = rng.dirichlet(np.full(N, alpha))
    anc = orc.systematic_ancestors(w, rng.random() / N)
    B = rng.standard_normal((N, 7))
    plans = [resample_plan(anc, r, world, M) for r in range(world)]
    for r in range(world):
        # rows received by r, in source-rank order
        recv = np.concatenate([B[s * M:(s + 1) * M][plans[s]["send_rows"][r]] for s in range(world)])
        assert recv.shape[0] == plans[r]["recv_counts"].sum()
        got = recv[plans[r]["gather_idx"]]
        np.testing.assert_array_equal(got, B[anc[r * M:(r + 1) * M]])
        # contiguous ranges only: a rank never sends more than (max - min + 1) rows per peer
        for d in range(world):
            rows = plans[r]["send_rows"][d]
            if rows.size:
                assert np.all(np.diff(rows) == 1)


def _worker(rank, world, port, M, q, seed, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(seed)
        N = M * world
        B = rng.standard_normal((N, q)).astype(np.float32)
        logw = np.log(rng.dirichlet(np.full(N, 0.3)))
        mine = slice(rank * M, (rank + 1) * M)
        # 1. fixed-chunk LSE statistics, all-gathered and combined in global order
        chunk = 128
        xs = logw[mine].reshape(-1, chunk)
        mx = xs.max(1)
        st = np.stack([mx, np.exp(xs - mx[:, None]).sum(1), np.exp(2 * (xs - mx[:, None])).sum(1)], 1)
        t = torch.from_numpy(st)
        allst = torch.empty((world * t.shape[0], 3), dtype=t.dtype)
        dist.all_gather_into_tensor(allst, t)
        a = allst.numpy()
        M0 = a[:, 0].max()
        s1 = (a[:, 1] * np.exp(a[:, 0] - M0)).sum()
        s2 = (a[:, 2] * np.exp(2 * (a[:, 0] - M0))).sum()
        lse = M0 + np.log(s1)
        ess = s1 * s1 / s2
        # 2. global weights -> identical ancestors on every rank -> all-to-all rows
        wloc = torch.from_numpy(np.exp(logw[mine] - lse))
        wall = torch.empty(N, dtype=torch.float64)
        dist.all_gather_into_tensor(wall, wloc)
        anc = orc.systematic_ancestors(wall.numpy(), 0.37 / N)
        plan = resample_plan(anc, rank, world, M)
        send = torch.from_numpy(np.ascontiguousarray(B[mine][np.concatenate(plan["send_rows"])]))
        recv = torch.empty((int(plan["recv_counts"].sum()), q), dtype=torch.float32)
        dist.all_to_all_single(recv, send, output_split_sizes=[int(c) for c in plan["recv_counts"]],
                               input_split_sizes=[int(r.size) for r in plan["send_rows"]])
        new = recv.numpy()[plan["gather_idx"]]
        # 3. fixed-point moments: integer all-reduce is exact and order-free
        fix = torch.from_numpy(np.rint(B[mine].astype(np.float64).sum(0) * 2.0**48).astype(np.int64))
        dist.all_reduce(fix)
        out[rank] = dict(lse=lse, ess=ess, anc=anc[mine], new=new, fix=fix.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_sharded_lambda_step_collectives(world):
    M, q, seed = 256, 5, 11
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, M, q, seed, out), nprocs=world, join=True)
    rng = np.random.default_rng(seed)
    N = M * world
    B = rng.standard_normal((N, q)).astype(np.float32)
    logw = np.log(rng.dirichlet(np.full(N, 0.3)))
    lse = orc.logsumexp(logw)
    w = np.exp(logw - lse)
    anc = orc.systematic_ancestors(w, 0.37 / N)
    for r in range(world):
        o = out[r]
        assert o["lse"] == pytest.approx(lse, abs=1e-12)
        assert o["ess"] == pytest.approx(orc.ess(w / w.sum()), rel=1e-10)
        np.testing.assert_array_equal(o["anc"], anc[r * M:(r + 1) * M])
        np.testing.assert_array_equal(o["new"], B[anc[r * M:(r + 1) * M]])
        np.testing.assert_array_equal(o["fix"], out[0]["fix"])
    # the integer all-reduce equals the single-process fixed-point sum exactly
    ref = np.zeros(q, np.int64)
    for r in range(world):
        ref += np.rint(B[r * M:(r + 1) * M].astype(np.float64).sum(0) * 2.0**48).astype(np.int64)
    np.testing.assert_array_equal(out[0]["fix"], ref)
