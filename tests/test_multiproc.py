"""Multi-process (world_size 2, gloo, CPU) coverage of bench.py's multi-GPU plumbing:
independent streams per rank, no data-path collective, barrier + max-over-ranks
timing and the whole-job aggregate value = world * frames / max time."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import bench

    d = bench.Dist("gloo")
    assert d.rank == rank and d.world == world
    d.barrier()
    # per-rank device time of its own streams (rank 1 slower): the job time is the max
    t = d.max(10.0 + 5.0 * rank)
    frames_per_rank = 40
    value = d.world * frames_per_rank / (t * 1e-3)
    out[rank] = (t, value)
    d.close()


def test_two_rank_max_timing_and_weak_scaling():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert out[0][0] == out[1][0] == 15.0
    assert abs(out[0][1] - 2 * 40 / 0.015) < 1e-6


def test_streams_are_independent_per_rank():
    # the seeds a rank uses for its streams (cfg.seed + stream) never depend on the world size,
    # so adding GPUs adds streams without changing any existing stream's outputs
    import bench  # noqa: F401

    from paper_2312_12491_b200 import stagger as sg

    a = sg.build_precompute(sg.EngineConfig(n_steps=2, d_latent=16, seed=5))
    b = sg.build_precompute(sg.EngineConfig(n_steps=2, d_latent=16, seed=5))
    assert (a.eps_cached == b.eps_cached).all()
