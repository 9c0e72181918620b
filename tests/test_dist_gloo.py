"""Multi-rank host logic on CPU (gloo, world_size 2 and 4): the sharded
lambda step's control flow with CPU tensors standing in for device memory.

* ParticleGroup's collectives (fixed-chunk log-sum-exp statistics, exact
  fixed-point moment all-reduce, the stream barrier, max-over-ranks timing)
  run through the real class with the gloo backend;
* the peer-memory resampling exchange (spa_resample_sharded) is restated:
  every rank reads all shards' weights (here: an all-gather standing in for
  the P2P loads), scans the global vector, takes the ancestors of its own
  slots and fetches each row from its owner (dist.owner_of addressing) --
  identical to the single-process resampling for any world size.

The device kernels behind these steps are covered by -m gpu tests
(tests/test_gpu_sharded.py runs two ranks on one GPU through CUDA IPC)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import spa_oracle as orc
from paper_1106_0322_b200.dist import owner_of, shard_layout


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_layout_and_owner_addressing(world):
    M, blocks = shard_layout(512 * world, world)
    assert M == 512 and [b for _, b in blocks] == [r * M for r in range(world)]
    for j in sorted({0, M - 1, min(M, world * M - 1), world * M - 1}):
        r, row = owner_of(j, M)
        assert blocks[r][1] + row == j and 0 <= row < M
    with pytest.raises(ValueError):
        shard_layout(512 * world + 1, world + 1)  # not divisible


def _worker(rank, world, port, M, q, seed, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1106_0322_b200.dist import ParticleGroup

        g = ParticleGroup(stage_host=True)  # also builds the side-stream communicator
        assert g.side is not None and g.side.world == world
        rng = np.random.default_rng(seed)
        N = M * world
        B = rng.standard_normal((N, q)).astype(np.float32)
        logw = np.log(rng.dirichlet(np.full(N, 0.3)))
        Mr, off = g.shard(N)
        assert Mr == M and off == rank * M
        mine = slice(off, off + M)
        # 1. fixed-chunk LSE statistics, all-gathered and combined in global order
        chunk = 128
        xs = logw[mine].reshape(-1, chunk)
        mx = xs.max(1)
        st = np.stack([mx, np.exp(xs - mx[:, None]).sum(1), np.exp(2 * (xs - mx[:, None])).sum(1)], 1)
        a = g.all_gather_cat(torch.from_numpy(st)).numpy()
        M0 = a[:, 0].max()
        s1 = (a[:, 1] * np.exp(a[:, 0] - M0)).sum()
        s2 = (a[:, 2] * np.exp(2 * (a[:, 0] - M0))).sum()
        lse = M0 + np.log(s1)
        ess = s1 * s1 / s2
        # 2. the peer-memory exchange: read every shard's weights (all-gather
        #    here, P2P loads on the GPU), scan the global vector, ancestors of
        #    the own slots, each row fetched from its owner
        g.stream_barrier()
        wall = g.all_gather_cat(torch.from_numpy(np.exp(logw[mine] - lse))).numpy()
        peers_B = g.all_gather_cat(torch.from_numpy(B[mine])).numpy().reshape(world, M, q)
        anc_all = orc.systematic_ancestors(wall, 0.37 / N)
        anc = anc_all[mine]
        new = np.stack([peers_B[owner_of(int(j), M)] for j in anc])
        g.stream_barrier()
        # 3. fixed-point moments: integer all-reduce is exact and order-free
        fix = torch.from_numpy(np.rint(B[mine].astype(np.float64).sum(0) * 2.0**48).astype(np.int64))
        g.all_reduce_sum(fix)
        g.side.all_reduce_sum(side := torch.ones(1, dtype=torch.int64))
        tmax = g.max_scalar(float(rank))
        out[rank] = dict(lse=lse, ess=ess, anc=anc, new=new, fix=fix.numpy(), tmax=tmax, side=int(side.item()))
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
        assert o["tmax"] == world - 1 and o["side"] == world
    # the integer all-reduce equals the single-process fixed-point sum exactly
    ref = np.zeros(q, np.int64)
    for r in range(world):
        ref += np.rint(B[r * M:(r + 1) * M].astype(np.float64).sum(0) * 2.0**48).astype(np.int64)
    np.testing.assert_array_equal(out[0]["fix"], ref)
