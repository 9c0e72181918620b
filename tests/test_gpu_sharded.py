"""Sharded sampler on the one available GPU: two ranks (processes) share
cuda:0, collectives run over gloo on host copies (no kernel waits on another
rank).  Particle streams are keyed by absolute index, log-sum-exp uses fixed
4096-particle chunks, ancestors come from the full weight vector and the RW
moments are exact integer sums -- so the 2-rank run must reproduce the
1-process run bit for bit."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfg(kernel):
    from paper_1106_0322_b200 import SmcConfig

    # init_chains pinned (the automatic count scales with the number of GPUs);
    # 293 chains x 28 slots: a chain's slot block straddles the shard boundary
    return SmcConfig(N=8192, cycles=2, moves=3, seed=5, init_burn=30, init_thin=1, move_kernel=kernel,
                     ess_threshold_frac=0.9, init_chains=300, summary_levels=(0.05, 0.5, 0.95),
                     summary_deltas=(0.05,))


def _run(group, kernel):
    from paper_1106_0322_b200 import make_schedule, run_sampler
    from paper_1106_0322_b200.data import named_spec, simulate_dataset

    data, _ = simulate_dataset(named_spec("a_small"))
    return run_sampler(data, 4.0, make_schedule(2.0, 0.8, 6), _cfg(kernel), False, group)


def _worker(rank, world, port, kernel, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1106_0322_b200.dist import ParticleGroup

        res = _run(ParticleGroup(stage_host=True), kernel)
        if rank == 0:
            out["particles"] = res.steps[-1].particles
            out["weights"] = res.steps[-1].weights
            out["logz"] = [s.log_z_ratio_cum for s in res.steps]
            out["resampled"] = [s.resampled for s in res.steps]
            out["acc"] = [s.acceptance for s in res.steps]
            out["summary"] = [(s.summary["mean"], s.summary["quantiles"], s.summary["concentration"])
                              for s in res.steps]
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kernel", ["mwg", "rw"])
def test_two_ranks_reproduce_single_process(kernel):
    single = _run(None, kernel)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _port(), kernel, out), nprocs=2, join=True)
    assert any(out["resampled"]), "the schedule should exercise the cross-shard resampling"
    np.testing.assert_array_equal(out["particles"], single.steps[-1].particles)
    np.testing.assert_array_equal(out["weights"], single.steps[-1].weights)
    assert out["logz"] == [s.log_z_ratio_cum for s in single.steps]
    assert out["acc"] == [s.acceptance for s in single.steps]
    # device marginal summaries: exact integer sums all-reduced across shards
    for (m2, q2, c2), s in zip(out["summary"], single.steps):
        np.testing.assert_array_equal(m2, s.summary["mean"])
        np.testing.assert_array_equal(q2, s.summary["quantiles"])
        np.testing.assert_array_equal(c2, s.summary["concentration"])


def _nccl_worker(rank, world, port, kernel, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    try:
        from paper_1106_0322_b200.dist import ParticleGroup

        res = _run(ParticleGroup(), kernel)  # NCCL: device collectives, stream-ordered fences, side communicator
        out["particles"] = res.steps[-1].particles
        out["logz"] = [s.log_z_ratio_cum for s in res.steps]
        out["resampled"] = [s.resampled for s in res.steps]
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kernel", ["mwg", "rw"])
def test_nccl_single_rank_sharded_path_matches_unsharded(kernel):
    """The sharded code path over the NCCL backend (device-side all-gathers,
    the stream-ordered all-reduce fences around the peer-memory exchange,
    the factor stream's own communicator) with one rank -- the only NCCL
    world one GPU allows -- reproduces the unsharded run bit for bit."""
    single = _run(None, kernel)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_nccl_worker, args=(1, _port(), kernel, out), nprocs=1, join=True)
    assert any(out["resampled"])
    np.testing.assert_array_equal(out["particles"], single.steps[-1].particles)
    assert out["logz"] == [s.log_z_ratio_cum for s in single.steps]
