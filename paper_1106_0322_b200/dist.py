"""Particle sharding across GPUs (one process per GPU, torch.distributed).

The reference parallelises only the move step over contiguous particle
blocks and promises results independent of the partition (smc.py:298-359,
test_smc.py:280-286).  Here the particle set itself is sharded: rank r owns
global particles [r*M, (r+1)*M) (M = N / world).  Every quantity that crosses
shards is made partition-invariant by construction:

* RNG streams are keyed by the absolute particle index (smc.py:40-43);
* log-sum-exp / ESS: per fixed 4096-particle chunk statistics are
  all-gathered and combined in global chunk order (bit-identical for any
  world size when M % 4096 == 0; otherwise still correct);
* systematic resampling reads the other ranks' memory directly: every rank
  maps its peers' weight and particle buffers once (CUDA IPC), scans the
  global weight vector with the exact scan (np.cumsum's bits), searches the
  ancestors of its own slots and loads those rows from their owners over
  NVLink (spa_resample_sharded) -- gated on the device-side ESS decision, so
  a lambda step issues only fixed-size, stream-ordered collectives and never
  waits on the host;
* RW-cov moments are 2^-48 fixed-point integers: the all-reduce SUM is exact
  and order-independent;
* snapshots are assembled on rank 0 only (peer copies), not all-gathered.

Collectives run on the caller's current stream (NCCL orders them with the
surrounding kernels), the covariance-factor stream uses a second process
group so its all-reduces never interleave with the main stream's.
`stage_host=True` routes every collective through host copies (gloo): the
test harness runs several ranks on one GPU that way, where no kernel may
wait on another rank.
"""

from __future__ import annotations

import ctypes
import math

import torch
import torch.distributed as dist


def shard_layout(N: int, world: int):
    """(M, [(rank, first global index)]) of the contiguous particle blocks."""
    if N % world:
        raise ValueError(f"N={N} is not divisible by the {world} ranks")
    M = N // world
    return M, [(r, r * M) for r in range(world)]


def owner_of(j: int, M: int):
    """(rank, local row) of global particle j (the P2P gather's addressing)."""
    return j // M, j % M


class ParticleGroup:
    """Collectives and peer memory used by the sampler when particles are sharded."""

    def __init__(self, pg=None, stage_host: bool = False, _side: bool = True):
        self.pg = pg if pg is not None else dist.group.WORLD
        self.rank = dist.get_rank(self.pg)
        self.world = dist.get_world_size(self.pg)
        self.stage_host = stage_host
        self._peers = {}  # id(system) -> pointer tables
        self._opened = {}  # (rank, handle bytes) -> mapped base pointer
        self._bar = None
        # the covariance factor is built on a side stream: its collectives
        # get their own communicator (created collectively, same order on all ranks)
        self.side = None
        if _side:
            pg_side = dist.new_group(ranks=list(range(self.world)))
            self.side = ParticleGroup(pg_side, stage_host, _side=False)

    # -- layout ----------------------------------------------------------
    def shard(self, N: int):
        M, blocks = shard_layout(N, self.world)
        return M, blocks[self.rank][1]

    # -- collectives -----------------------------------------------------
    def barrier(self):
        dist.barrier(self.pg)

    def stream_barrier(self):
        """All ranks' work enqueued before this point on their current
        streams has finished before anything enqueued after it runs (a
        stream-ordered one-element all-reduce; a host barrier in stage_host
        mode)."""
        if self.stage_host:
            if torch.cuda.is_available():
                torch.cuda.synchronize()
            dist.barrier(self.pg)
            return
        if self._bar is None:
            self._bar = torch.zeros(1, dtype=torch.int32, device=self._dev())
        dist.all_reduce(self._bar, group=self.pg)

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

    def destroy(self):
        from . import _lib

        for base in self._opened.values():
            _lib.call("spa_ipc_close", ctypes.c_void_p(base))
        self._opened.clear()
        self._peers.clear()
        if dist.is_initialized():
            dist.destroy_process_group()

    def _dev(self):
        return torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu")

    # -- peer memory ---------------------------------------------------------
    def _export(self, t: torch.Tensor):
        from . import _lib

        h = (ctypes.c_uint8 * 64)()
        off = ctypes.c_uint64(0)
        _lib.call("spa_ipc_export", ctypes.c_void_p(t.data_ptr()), h, ctypes.byref(off))
        return bytes(h), int(off.value)

    def _open(self, rank: int, handle: bytes, offset: int) -> int:
        from . import _lib

        key = (rank, handle)
        if key not in self._opened:
            base = ctypes.c_void_p(0)
            _lib.call("spa_ipc_open", ctypes.create_string_buffer(handle, 64), ctypes.byref(base))
            self._opened[key] = int(base.value)
        return self._opened[key] + offset

    def setup_peers(self, system) -> None:
        """Map every rank's weight / particle buffers (system.w, beta, ll,
        lp -- fixed allocations for the life of the system) into this
        process: the pointer tables of spa_resample_sharded / snapshots."""
        names = ("w", "beta", "ll", "lp")
        mine = [self._export(getattr(system, n)) for n in names]
        blob = torch.zeros((len(names), 72), dtype=torch.uint8)
        for i, (h, off) in enumerate(mine):
            blob[i, :64] = torch.frombuffer(bytearray(h), dtype=torch.uint8)
            blob[i, 64:] = torch.tensor(list(int(off).to_bytes(8, "little")), dtype=torch.uint8)
        dev_blob = blob.to(self._dev()) if not self.stage_host else blob
        allb = self.all_gather_cat(dev_blob.view(1, len(names), 72)).cpu()
        tables = {n: (ctypes.c_void_p * self.world)() for n in names}
        for r in range(self.world):
            for i, n in enumerate(names):
                if r == self.rank:
                    tables[n][r] = getattr(system, n).data_ptr()
                else:
                    row = bytes(allb[r, i].numpy().tobytes())
                    tables[n][r] = self._open(r, row[:64], int.from_bytes(row[64:], "little"))
        tables["ptrs"] = {n: getattr(system, n).data_ptr() for n in names}
        self._peers[id(system)] = tables

    def peer_tables(self, system):
        t = self._peers.get(id(system))
        if t is None:
            raise RuntimeError("ParticleGroup.setup_peers(system) was not called")
        for n, p in t["ptrs"].items():  # the mapped buffers must not have moved
            if getattr(system, n).data_ptr() != p:
                raise RuntimeError(f"sharded particle buffer '{n}' was reallocated after setup_peers")
        return t

    # -- the exchange ----------------------------------------------------------
    def resample(self, system, gate: ctypes.c_void_p, u: float, ws: torch.Tensor, anc: torch.Tensor) -> None:
        """Device-decided global systematic resampling of the sharded set
        (gated on *gate): fence, exact global scan + own-slot ancestors + P2P
        row gather, fence, commit.  system.w must hold the globally
        normalised weights."""
        from . import _lib
        from .smc import _p, _stream

        tb = self.peer_tables(system)
        self.stream_barrier()  # every rank's weights and rows are final
        _lib.call("spa_resample_sharded", gate, tb["w"], self.world, system.N, float(u), self.rank, tb["beta"],
                  tb["ll"], tb["lp"], system.ldb, system.q, _p(system.beta_alt), _p(system.ll_alt),
                  _p(system.lp_alt), _p(anc), _p(ws), ws.numel(), _stream())
        self.stream_barrier()  # every rank has read its ancestors' rows
        _lib.call("spa_resample_commit", gate, _p(system.beta), _p(system.beta_alt), system.ldb, system.q,
                  _p(system.ll), _p(system.ll_alt), _p(system.lp), _p(system.lp_alt), _p(system.logw),
                  -math.log(system.N_total), system.N, _stream())

    def snapshot_to_rank0(self, system, w: torch.Tensor):
        """Rank 0 assembles the global (weights, particles [N][q], ll) from
        the peers' buffers; other ranks return None.  w: this rank's globally
        normalised weights (system.w)."""
        from . import _lib
        from .smc import _stream

        tb = self.peer_tables(system)
        self.stream_barrier()
        out = None
        if self.rank == 0:
            M, ldb, q = system.N, system.ldb, system.q
            dev = system.device
            W = torch.empty(M * self.world, dtype=torch.float64, device=dev)
            B = torch.empty((M * self.world, ldb), dtype=torch.float32, device=dev)
            LL = torch.empty(M * self.world, dtype=torch.float64, device=dev)
            for r in range(self.world):
                for dst, src, nb in ((W, tb["w"][r], 8 * M), (B, tb["beta"][r], 4 * M * ldb), (LL, tb["ll"][r], 8 * M)):
                    _lib.call("spa_copy_async", ctypes.c_void_p(dst.data_ptr() + r * nb), ctypes.c_void_p(src), nb,
                              _stream())
            out = (W, B[:, :q], LL)
        self.stream_barrier()  # the peers keep their buffers until rank 0 has copied
        return out
