"""Multi-process data parallelism on CPU (gloo, world_size 2).

The GPU run all-reduces the 10-float per-Gaussian world-frame accumulator
with NCCL between the backward and the epilogue (paper_2508_04929_b200.parallel).
Here the same host logic -- batch sharding, the accumulator all-reduce, the
global 1/B scale -- runs over gloo with the CPU oracle computing each rank's
accumulator, and must equal the single-process full-batch gradient.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT, grads_close


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(oracle):
    grid = oracle.Grid(32, 0.5, 3.0)
    params = oracle.init_random(300, 0, grid)
    rng = np.random.default_rng(4)
    params[:, 3:6] = oracle.inverse_activate(rng.uniform(1.0, 2.5, (300, 3)) * grid.pixel_width)
    params[:, 6:10] = rng.standard_normal((300, 4))
    poses = [oracle.sample_pose(np.random.default_rng(50 + i)) for i in range(6)]
    ups = [np.random.default_rng(90 + i).standard_normal((32, 32)) for i in range(6)]
    return grid, params, poses, ups


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys

    sys.path.insert(0, ROOT)
    from oracle import cgs_oracle as oracle
    from paper_2508_04929_b200 import parallel

    dist.init_process_group("gloo", rank=rank, world_size=world)
    grid, params, poses, ups = _inputs(oracle)
    batch = np.arange(len(poses))
    local = parallel.shard(batch, rank, world)
    acc = np.zeros((len(params), 10))
    for i in local:
        W, t = poses[i]
        proj = oracle.project(params, W, t, grid)
        acc += oracle.world_accumulator(proj, oracle.backward_raw_sums(params, W, t, grid, ups[i], proj))
    t_acc = torch.from_numpy(acc)
    parallel.allreduce_accumulator(t_acc)
    grads = oracle.grads_from_world_accumulator(params, t_acc.numpy()) / len(batch)
    gathered = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(gathered, torch.tensor([len(local)]))
    if rank == 0:
        np.savez(out_path, grads=grads, counts=np.array([int(g) for g in gathered]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_allreduce_matches_single_process(oracle, tmp_path):
    out = str(tmp_path / "dp.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    res = np.load(out)
    grid, params, poses, ups = _inputs(oracle)
    ref = np.zeros_like(params)
    for (W, t), up in zip(poses, ups):
        ref += oracle.rasterize_backward(params, W, t, grid, up)
    ref /= len(poses)
    assert list(res["counts"]) == [3, 3]
    grads_close(res["grads"], ref, 1e-10, 1e-12)


def test_shard_partitions_every_batch():
    from paper_2508_04929_b200 import parallel

    rng = np.random.default_rng(0)
    for B in (1, 2, 7, 256, 257):
        for world in (1, 2, 3, 8):
            idx = rng.permutation(1000)[:B]
            parts = [parallel.shard(idx, r, world) for r in range(world)]
            assert np.array_equal(np.concatenate(parts), idx)
            assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1


def test_epoch_batches_follow_reference_shuffle():
    from paper_2508_04929_b200 import parallel

    a = parallel.epoch_batches(10, 1, np.random.default_rng(3))
    b = np.random.default_rng(3).permutation(10)  # train.py:220,230
    assert [int(x[0]) for x in a] == list(b)
    c = parallel.epoch_batches(10, 4, np.random.default_rng(3))
    assert [len(x) for x in c] == [4, 4, 2]


@pytest.mark.skipif(not dist.is_available(), reason="torch.distributed unavailable")
def test_allreduce_is_noop_without_process_group():
    from paper_2508_04929_b200 import parallel

    t = torch.ones(5)
    assert parallel.allreduce_accumulator(t) is t and torch.equal(t, torch.ones(5))


def _skip_worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys

    sys.path.insert(0, ROOT)
    from paper_2508_04929_b200 import parallel

    dist.init_process_group("gloo", rank=rank, world_size=world)
    acc = torch.full((2 * 10 + 1,), float(rank + 1))
    status = torch.tensor([4 if rank == 1 else 1], dtype=torch.int32)  # rank 1: non-finite loss
    skip = parallel.allreduce_accumulator(acc, status=status)
    clean = parallel.allreduce_accumulator(torch.zeros(21), status=torch.tensor([1], dtype=torch.int32))
    out = [torch.zeros(3, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(out, torch.tensor([float(skip.item()), float(acc[0]), float(clean.item())], dtype=torch.float64))
    if rank == 0:
        np.save(out_path, torch.stack(out).numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_skip_decision_is_shared_by_all_ranks(tmp_path):
    """A non-finite loss on one rank makes every rank skip the Adam update (the flag travels in
    the accumulator all-reduce), so replicated parameters cannot diverge; a degenerate-rotation
    bit alone does not skip."""
    out = str(tmp_path / "skip.npy")
    mp.spawn(_skip_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    res = np.load(out)
    from paper_2508_04929_b200.parallel import SKIP_BITS

    assert res[:, 0].tolist() == [float(SKIP_BITS)] * 2  # SKIP_BITS on both ranks
    assert res[:, 1].tolist() == [3.0, 3.0]  # the accumulator itself is summed
    assert res[:, 2].tolist() == [0.0, 0.0]


def _exchange_layout(n, per, rank, flag):
    """What cgs_reduce_partials_sliced writes on a rank (host restatement for the CPU test):
    slices of per Gaussians (per * 10 + 2 floats), Gaussian g's 10 values = (10 g + j) * (rank + 1),
    every slice's flag slot = this rank's skip flag, padding and rows past n zero."""
    world_slices = -(-n // per)
    S = per * 10 + 2
    out = np.zeros(world_slices * S, np.float32)
    for g in range(n):
        k, r = divmod(g, per)
        out[k * S + r * 10:k * S + r * 10 + 10] = (10 * g + np.arange(10)) * (rank + 1)
    for k in range(world_slices):
        out[k * S + per * 10] = flag
    return out


def _shard_worker(rank, world, port, out_path, sharded):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import sys

    sys.path.insert(0, ROOT)
    from paper_2508_04929_b200 import parallel

    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 7
    xch = parallel.Exchange(n, sharded=sharded)
    assert not xch.capturable  # gloo: collectives stay outside captured graphs
    lay = _exchange_layout(n, xch.per, rank, 1.0 if rank == 2 else 0.0)
    xch.acc[: lay.size].copy_(torch.from_numpy(lay))
    xch.run()
    own, a, b = xch.own()
    store = torch.full((xch.per * world if sharded else n, 11), -1.0, dtype=torch.float64)
    ra, rb, per = parallel.gaussian_slice(n, rank, world)
    store[ra:rb] = float(rank)
    if sharded:
        xch.gather_rows(store)
    res = [own[: (b - a) * 10].clone().numpy(), xch.skip.clone().numpy(), store[:n].clone().numpy(),
           np.array([a, b])]
    gathered = [None] * world
    dist.all_gather_object(gathered, res)
    if rank == 0:
        np.save(out_path, np.array(gathered, dtype=object), allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("sharded", [True, False])
def test_sharded_epilogue_collectives(tmp_path, sharded):
    """parallel.Exchange on 3 ranks over gloo.  Sharded (ZeRO-1 style): each rank receives the
    rank-sum of its own Gaussian slice (ceil(7/3) = 3, 3, 1 rows) in place in the slice layout,
    the skip flag raised by one rank is shared, and the in-place all-gather leaves every rank with
    every slice's rows.  Replicated: every rank receives the whole sum."""
    out = str(tmp_path / "shard.npy")
    mp.spawn(_shard_worker, args=(3, _free_port(), out, sharded), nprocs=3, join=True)
    res = np.load(out, allow_pickle=True)
    from paper_2508_04929_b200 import parallel

    total = (10 * np.arange(7)[:, None] + np.arange(10)).ravel().astype(np.float32) * (1 + 2 + 3)
    for r in range(3):
        a, b = (int(x) for x in res[r][3])
        if sharded:
            assert (a, b) == parallel.gaussian_slice(7, r, 3)[:2]
        else:
            assert (a, b) == (0, 7)
        np.testing.assert_array_equal(res[r][0], total[a * 10:b * 10])
        assert int(res[r][1][0]) == parallel.SKIP_BITS
        if sharded:
            rows = np.concatenate([np.full((min(7, (k + 1) * 3) - min(7, k * 3), 11), float(k)) for k in range(3)])
            np.testing.assert_array_equal(res[r][2], rows)


def test_epoch_records_cover_each_batch_shard_once():
    """Per-epoch particle residency: the records a rank loads for an epoch are
    exactly its shards of that epoch's global batches (train.py:228-232 order), the ranks'
    sets partition the dataset, and every rank's count is the same every epoch (so the resident
    buffers are refilled in place)."""
    from paper_2508_04929_b200 import parallel

    for R, B, world in [(100, 8, 2), (101, 16, 3), (37, 5, 4), (1000, 256, 8)]:
        counts = None
        for seed in range(3):
            order = np.random.default_rng(seed).permutation(R)
            sets = [parallel.epoch_records(order, B, r, world) for r in range(world)]
            assert sorted(np.concatenate(sets).tolist()) == list(range(R))
            for r in range(world):
                want = np.concatenate([parallel.shard(order[i:i + B], r, world) for i in range(0, R, B)])
                assert np.array_equal(sets[r], want)
            c = [len(x) for x in sets]
            assert counts is None or c == counts
            counts = c
