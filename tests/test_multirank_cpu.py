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
    slowest = bench.max_over_ranks(3.0 + 4.0 * rank, "cpu", dist)  # the sharded (N > 1) line's timing
    from paper_1311_7194_b200 import shard

    uid = shard.broadcast_nccl_id(shard.DistComm())  # the sharded frame's NCCL bootstrap
    differ = bench.replicas_consistent([1.0, 2.0, float(rank)], "cpu", dist, world)
    q.put((rank, w, r, total, e2e, value, e2e_value, same, differ, slowest, uid))
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
    assert out[0][-1] == out[1][-1] and len(out[0][-1]) == 128 and any(out[0][-1])  # same NCCL id on both ranks
    for rank, w, r, total, e2e, value, e2e_value, same, differ, slowest, _ in out:
        assert (w, r) == (2, rank)
        assert slowest == 7.0
        assert total == 11.0 and e2e == 20.0          # max over ranks
        assert value == pytest.approx(2 * 8 / 11e-3)  # whole-job aggregate
        assert e2e_value == pytest.approx(2 * 8 / 20e-3)
        assert same and not differ


def test_single_rank_is_identity():
    import bench

    total, e2e, value, _ = bench.aggregate_ranks(5.0, 6.0, 10, 1, "cpu")
    assert (total, e2e) == (5.0, 6.0) and value == pytest.approx(10 / 5e-3)
    assert bench.replicas_consistent([1.0], "cpu")


def _shard_worker(rank, world, port, q):
    """The collectives of the sharded frame (paper_1311_7194_b200/shard.py DistComm) over gloo."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1311_7194_b200.shard import DistComm

    comm = DistComm()
    # global ray bounds: MIN of t_start, MAX of t_end
    ts = torch.tensor([1.0 + rank, float("inf"), 3.0 - rank])
    te = torch.tensor([2.0 + rank, float("-inf"), 4.0 - rank])
    comm.all_reduce([ts], "min")
    comm.all_reduce([te], "max")
    # composite: key MIN picks the nearest depth, then an int32 SUM of the winners' bit patterns
    depth = torch.tensor([0.5, -0.0, 2.0, 0.0]) if rank == 0 else torch.tensor([0.25, 7.0, 3.0, 0.0])
    bits = lambda d: d.view(torch.int32).to(torch.int64)  # noqa: E731
    key = torch.where(depth > 0, (bits(depth) << 32) | rank, torch.full_like(bits(depth), 2**63 - 1))
    comm.all_reduce([key], "min")
    win = (key != 2**63 - 1) & ((key & 0x7FFFFFFF) == rank)
    mine = torch.where(win, depth, torch.zeros_like(depth))
    comm.all_reduce([mine.view(torch.int32)], "sum")
    # halo exchange: variable record counts per rank
    m3 = 8
    count = 2 + 7 * rank  # rank 1 sends more records than rank 0's buffer holds
    cap = 4 if rank == 0 else 10
    keys = torch.arange(cap, dtype=torch.int32) + 100 * rank
    pays = (torch.arange(cap * m3, dtype=torch.int16).reshape(cap, m3) + 1000 * rank).contiguous()
    got = comm.exchange([(keys, pays, count)])[0]
    recs = [(k[:c].tolist(), p[:c].tolist(), c) for k, p, c in got]
    q.put((rank, ts.tolist(), te.tolist(), mine.tolist(), recs))
    dist.destroy_process_group()


def test_sharded_collectives_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ts, te, mine, recs in out:
        assert ts == [1.0, float("inf"), 2.0] and te == [3.0, float("-inf"), 4.0]
        assert mine == [0.25, 7.0, 2.0, 0.0]  # nearest positive depth per pixel, bit-copied
        other = 1 - rank
        assert len(recs) == 1
        k, p, c = recs[0]
        assert c == 2 + 7 * other and k == [100 * other + i for i in range(c)]
        assert p[0][0] == 1000 * other and len(p) == c
