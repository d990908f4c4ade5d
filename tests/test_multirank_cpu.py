"""The N>1 bench logic on CPU: two ranks over gloo (127.0.0.1) exercise the max-over-ranks
timing reduction and the replica-consistency check of bench.py exactly as torchrun runs them
on a multi-GPU box (there with NCCL on cuda tensors)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    w, r, _ = bench.dist_setup()
    total, e2e, value, e2e_value = bench.aggregate_ranks(10.0 + rank, 20.0 - rank, 8, world, "cpu", dist)
    same = bench.replicas_consistent([1.0, 2.0, 3.0], "cpu", dist, world)
    differ = bench.replicas_consistent([1.0, 2.0, float(rank)], "cpu", dist, world)
    q.put((rank, w, r, total, e2e, value, e2e_value, same, differ))
    dist.destroy_process_group()


def test_two_rank_aggregation_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, w, r, total, e2e, value, e2e_value, same, differ in out:
        assert (w, r) == (2, rank)
        assert total == 11.0 and e2e == 20.0          # max over ranks
        assert value == pytest.approx(2 * 8 / 11e-3)  # whole-job aggregate
        assert e2e_value == pytest.approx(2 * 8 / 20e-3)
        assert same and not differ


def test_single_rank_is_identity():
    import bench

    total, e2e, value, _ = bench.aggregate_ranks(5.0, 6.0, 10, 1, "cpu")
    assert (total, e2e) == (5.0, 6.0) and value == pytest.approx(10 / 5e-3)
    assert bench.replicas_consistent([1.0], "cpu")
