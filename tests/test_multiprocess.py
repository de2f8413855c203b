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


def _worker_sharded(rank, world, port, out):
    """Rank r holds rows shard_rows(...) of a c0-shaped problem; the sums over ranks (gloo
    all-reduce) of the local Gram, column norms and SP right-hand sides reproduce the unsharded
    oracle's, and an SP run driven by the reduced quantities matches the oracle's iterates."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import numpy as np
        from oracle import ils_oracle as O
        from paper_2203_15340_b200.ils import shard_rows
        from workloads import make_dense
        pr = make_dense(200, 100, 50, 0.3, seed=45)
        (p0, p1), (q0, q1) = shard_rows(pr.p, pr.q, world, rank)
        A1, b1 = pr.A1[p0:p1], pr.b1[p0:p1]
        A2, b2 = pr.A2[q0:q1], pr.b2[q0:q1]

        def allsum(v):
            t = torch.from_numpy(np.ascontiguousarray(v))
            dist.all_reduce(t)
            return t.numpy()

        G = allsum(A1.T @ A1)
        N = allsum((A1 * A1).sum(axis=0))
        x = np.zeros(pr.n)
        xs = []
        for _ in range(5):
            c = allsum(O.sp_rhs(A1, A2, b1, b2, x))
            x = np.linalg.solve(G, c)
            xs.append(x)
        g = allsum(A1.T @ (b1 - A1 @ xs[-1]) - A2.T @ (b2 - A2 @ xs[-1]))
        rows = [None] * world
        dist.all_gather_object(rows, (p0, p1, q0, q1))
        out[rank] = (G, N, xs, g, rows)
    finally:
        dist.destroy_process_group()


def test_sharded_oracle_algebra_gloo():
    import numpy as np
    from oracle import ils_oracle as O
    from workloads import make_dense
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_sharded, args=(world, port, out), nprocs=world, join=True)
    pr = make_dense(200, 100, 50, 0.3, seed=45)
    G, N, xs, g, rows = out[0]
    assert rows == [(0, 100, 0, 50), (100, 200, 50, 100)]   # blocks tile the rows exactly once
    assert np.allclose(G, pr.A1.T @ pr.A1, rtol=1e-13, atol=1e-12)
    assert np.allclose(N, (pr.A1 * pr.A1).sum(axis=0), rtol=1e-13)
    ref = O.sp_solve(pr.A1, pr.A2, pr.b1, pr.b2, max_iter=5, stop=O.STOP_NONE)
    for k in range(5):
        assert np.linalg.norm(xs[k] - ref.x_hist[k]) <= 1e-10 * np.linalg.norm(ref.x_hist[k])
    gr = pr.A1.T @ (pr.b1 - pr.A1 @ xs[-1]) - pr.A2.T @ (pr.b2 - pr.A2 @ xs[-1])
    assert np.allclose(g, gr, rtol=1e-10, atol=1e-10)
    assert np.array_equal(out[1][0], G)   # every rank holds the same reduced Gram


def test_shard_rows_partition():
    from paper_2203_15340_b200.ils import shard_rows
    for p, q, world in [(10, 3, 4), (200, 0, 3), (7, 7, 7), (1000, 1, 8)]:
        covered_p, covered_q = [], []
        for r in range(world):
            (p0, p1), (q0, q1) = shard_rows(p, q, world, r)
            assert p1 > p0
            covered_p += list(range(p0, p1))
            covered_q += list(range(q0, q1))
        assert covered_p == list(range(p)) and covered_q == list(range(q))
    with pytest.raises(ValueError):
        shard_rows(3, 1, 4, 0)


def test_max_over_ranks_single_process():
    import bench
    assert bench.max_over_ranks(3.5, torch.device("cpu")) == 3.5
