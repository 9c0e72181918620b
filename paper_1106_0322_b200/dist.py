"""Particle sharding across GPUs (one process per GPU, torch.distributed).

The reference parallelises only the move step over contiguous particle
blocks and promises results independent of the partition (smc.py:298-359,
test_smc.py:280-286).  Here the particle set itself is sharded: rank r owns
global particles [r*M, (r+1)*M) (M = N / world).  Every quantity that crosses
shards is made partition-invariant by construction:

* RNG streams are keyed by the absolute particle index (smc.py:40-43);
* log-sum-exp / ESS: per fixed 4096-particle chunk statistics are
  all-gathered and combined in global chunk order (needs M % 4096 == 0 for
  bit-identity across world sizes; otherwise still correct, order = rank order);
* systematic resampling: the normalised weights are all-gathered and every
  rank runs the bit-exact sequential-cumsum ancestor kernel on the full
  vector, so all ranks agree on every ancestor; rows whose ancestor lives on
  another rank are exchanged with one all-to-all (ancestors are monotone in
  the slot index, so each rank sends one contiguous row range per peer);
* RW-cov moments are 2^-48 fixed-point integers: the all-reduce SUM is
  exact and order-independent.

The exchange plan (`resample_plan`) is pure index arithmetic and is tested on
CPU with the gloo backend (tests/test_dist_gloo.py).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist


def resample_plan(anc: np.ndarray, rank: int, world: int, shard: int):
    """Row-exchange plan for one systematic resampling step.

    anc: global ancestors [N] (monotone non-decreasing, identical on all ranks).
    Returns dict with
      send_rows[d]  : local source rows (contiguous range) this rank sends to d
      recv_counts[s]: rows received from s (concatenated in rank order)
      gather_idx    : for each local slot, its row in the receive buffer
    """
    anc = np.asarray(anc, dtype=np.int64)
    N = anc.size
    assert N == shard * world
    owner = anc // shard
    send_rows = []
    recv_counts = np.zeros(world, dtype=np.int64)
    # what does destination d need from me (rank)?
    for d in range(world):
        a = anc[d * shard:(d + 1) * shard]
        mine = a[(a // shard) == rank]
        if mine.size:
            lo, hi = int(mine.min()), int(mine.max())
            send_rows.append(np.arange(lo - rank * shard, hi - rank * shard + 1, dtype=np.int64))
        else:
            send_rows.append(np.zeros(0, dtype=np.int64))
    a = anc[rank * shard:(rank + 1) * shard]
    o = owner[rank * shard:(rank + 1) * shard]
    base = np.zeros(world, dtype=np.int64)
    lo_src = np.zeros(world, dtype=np.int64)
    for s in range(world):
        sel = a[o == s]
        if sel.size:
            lo_src[s] = sel.min()
            recv_counts[s] = sel.max() - sel.min() + 1
    base[1:] = np.cumsum(recv_counts)[:-1]
    gather_idx = base[o] + (a - lo_src[o])
    return {"send_rows": send_rows, "recv_counts": recv_counts, "gather_idx": gather_idx}


class ParticleGroup:
    """Collectives used by the sampler when particles are sharded."""

    def __init__(self, pg=None, stage_host: bool = False):
        """stage_host: run the collectives on host copies (gloo backend; used
        to test the sharded path with several ranks on one GPU, where no
        kernel may wait on another rank)."""
        self.pg = pg if pg is not None else dist.group.WORLD
        self.rank = dist.get_rank(self.pg)
        self.world = dist.get_world_size(self.pg)
        self.stage_host = stage_host

    # -- layout ----------------------------------------------------------
    def shard(self, N: int):
        if N % self.world:
            raise ValueError(f"N={N} is not divisible by the {self.world} ranks")
        M = N // self.world
        return M, self.rank * M

    # -- collectives -----------------------------------------------------
    def barrier(self):
        dist.barrier(self.pg)

    def all_gather_cat(self, t: torch.Tensor) -> torch.Tensor:
        src = t.contiguous().cpu() if self.stage_host else t.contiguous()
        out = torch.empty((self.world * src.shape[0],) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
        dist.all_gather_into_tensor(out, src, group=self.pg)
        return out.to(t.device) if self.stage_host else out

    def all_reduce_sum(self, t: torch.Tensor) -> torch.Tensor:
        if self.stage_host:
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.pg)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.pg)
        return t

    def max_scalar(self, v: float) -> float:
        t = torch.tensor([float(v)], dtype=torch.float64, device="cpu" if self.stage_host else self._dev())
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.pg)
        return float(t.item())

    def gather_to_all(self, t: torch.Tensor) -> torch.Tensor:
        return self.all_gather_cat(t)

    def zero_res(self, system):
        """res vector with lse = 0: log-weights are globally normalised."""
        r = torch.zeros(3, dtype=torch.float64, device=system.device)
        return r

    def destroy(self):
        if dist.is_initialized():
            dist.destroy_process_group()

    def _dev(self):
        return torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu")

    # -- resampling row exchange -------------------------------------------
    def exchange_rows(self, system, anc: torch.Tensor) -> None:
        """Fill system.beta_alt / ll_alt / lp_alt with the rows of this rank's
        slots' ancestors, fetching remote rows with one all-to-all."""
        from . import _lib
        from .smc import _p, _stream

        M = system.N
        plan = resample_plan(anc.cpu().numpy(), self.rank, self.world, M)
        dev = system.device
        send_idx = torch.from_numpy(np.concatenate(plan["send_rows"])).to(dev)
        send_counts = [int(r.size) for r in plan["send_rows"]]
        recv_counts = [int(c) for c in plan["recv_counts"]]
        nsend, nrecv = int(sum(send_counts)), int(sum(recv_counts))
        W = system.ldb + 4  # row payload: beta (ldb floats) + ll, lp (2 doubles as 4 floats)
        sendbuf = torch.empty((max(nsend, 1), W), dtype=torch.float32, device=dev)
        recvbuf = torch.empty((max(nrecv, 1), W), dtype=torch.float32, device=dev)
        if nsend:
            sb64 = sendbuf.view(torch.float64)  # [n, W/2] doubles view of the same storage
            ll_col = torch.empty(nsend, dtype=torch.float64, device=dev)
            lp_col = torch.empty(nsend, dtype=torch.float64, device=dev)
            _lib.call("spa_gather_rows", _p(system.beta), system.ldb, _p(sendbuf), W, system.q, _p(send_idx), 0, nsend,
                      _p(system.ll), _p(ll_col), _p(system.lp), _p(lp_col), _stream())
            sb64[:nsend, system.ldb // 2] = ll_col
            sb64[:nsend, system.ldb // 2 + 1] = lp_col
        if self.stage_host:
            rh = torch.empty((nrecv, W), dtype=torch.float32)
            dist.all_to_all_single(rh, sendbuf[:nsend].cpu(), output_split_sizes=recv_counts,
                                   input_split_sizes=send_counts, group=self.pg)
            recvbuf[:nrecv].copy_(rh)
        else:
            dist.all_to_all_single(recvbuf[:nrecv], sendbuf[:nsend], output_split_sizes=recv_counts,
                                   input_split_sizes=send_counts, group=self.pg)
        rb64 = recvbuf.view(torch.float64)
        gidx = torch.from_numpy(plan["gather_idx"]).to(dev)
        ll_in = rb64[:, system.ldb // 2].contiguous()
        lp_in = rb64[:, system.ldb // 2 + 1].contiguous()
        _lib.call("spa_gather_rows", _p(recvbuf), W, _p(system.beta_alt), system.ldb, system.q, _p(gidx), 0, M,
                  _p(ll_in), _p(system.ll_alt), _p(lp_in), _p(system.lp_alt), _stream())
