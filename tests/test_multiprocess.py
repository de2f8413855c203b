"""N > 1 host logic on CPU (gloo, world_size 2): the bench's whole-job time is the max over ranks,
and every rank builds the identical replica workload ("replicas only")."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from workloads import fingerprint, make_problem
        v = bench.max_over_ranks(10.0 + 5.0 * rank, torch.device("cpu"))
        pr = make_problem("c0")
        fp = fingerprint(pr.A, pr.b)
        fps = [None] * world
        dist.all_gather_object(fps, fp)
        out[rank] = (v, len(set(fps)))
    finally:
        dist.destroy_process_group()


def test_max_over_ranks_and_identical_replicas_gloo():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert out[0] == (15.0, 1) and out[1] == (15.0, 1)


def _worker_partition(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from workloads import make_problem
        lo, hi = bench.instance_partition(rank, world, 8)
        pr = make_problem("c4", seed=lo, batch=8)
        seeds = [None] * world
        dist.all_gather_object(seeds, [int(s) for s in pr.seeds])
        out[rank] = (lo, hi, seeds)
    finally:
        dist.destroy_process_group()


def test_batched_instance_partition_gloo():
    """c4 under N ranks: disjoint instance ranges covering [0, N*batch), each rank's data drawn with
    its own instance seeds (bench.instance_partition)."""
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_partition, args=(world, port, out), nprocs=world, join=True)
    assert (out[0][0], out[0][1], out[1][0], out[1][1]) == (0, 8, 8, 16)
    allseeds = out[0][2][0] + out[0][2][1]
    assert sorted(allseeds) == list(range(16)) and out[0][2] == out[1][2]


def test_max_over_ranks_single_process():
    import bench
    assert bench.max_over_ranks(3.5, torch.device("cpu")) == 3.5
