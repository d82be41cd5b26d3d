"""Data parallelism over particles.

Every rank holds the full mixture (N x 11 fp64 + Adam moments) and takes a
contiguous share of each global batch; the only exchange is one all-reduce
(SUM) of the 10-float per-Gaussian world-frame accumulator per step (plus one
slot for the ranks' skip flags), after which the fused epilogue + Adam runs
identically on every rank.  With the NCCL
backend this is one ``ncclAllReduce`` over NVLink/NVSwitch (NVLS when NCCL
picks it); the same code runs on gloo for CPU tests.
"""

from __future__ import annotations

import numpy as np


def shard(indices, rank: int, world: int) -> np.ndarray:
    """Contiguous slice [B*rank/world, B*(rank+1)/world) of a global batch."""
    idx = np.asarray(indices)
    B = len(idx)
    return idx[(B * rank) // world:(B * (rank + 1)) // world]


# status bits that make the Adam epilogue skip a step (cgs_b200.h)
SKIP_BITS = 2 | 4 | 8  # CGS_STATUS_BIN_OVERFLOW | CGS_STATUS_NONFINITE_LOSS | CGS_STATUS_NONFINITE_PARAMS


def allreduce_accumulator(acc, group=None, status=None):
    """Sum the flat N*10 gradient accumulator over ranks in place (one collective).

    With ``status`` (this rank's int32 status tensor) the buffer carries one extra
    trailing slot, set to 1 when this rank must skip the step (non-finite loss or
    bin overflow) and summed with the rest, so every rank makes the same skip
    decision and the replicated parameters stay identical.  Returns the int32
    skip status for the epilogue (SKIP_BITS if any rank skips, else 0), or
    ``acc`` when ``status`` is None.
    """
    import torch
    import torch.distributed as dist

    if status is not None:
        acc[-1] = ((status[0] & SKIP_BITS) != 0).to(acc.dtype)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
    if status is None:
        return acc
    return torch.where(acc[-1:] > 0, SKIP_BITS, 0).to(torch.int32)


def epoch_batches(n_records: int, batch_size: int, rng: np.random.Generator):
    """The seeded per-epoch visiting order cut into global batches (train.py:228-232)."""
    order = rng.permutation(n_records)
    return [order[i:i + batch_size] for i in range(0, n_records, batch_size)]


def gaussian_slice(n: int, rank: int, world: int):
    """(start, stop, rows per rank) of the Gaussians whose optimizer state this rank owns in the
    sharded epilogue: equal slices of ceil(n / world) rows, the last one short."""
    per = -(-n // world)
    return min(n, rank * per), min(n, (rank + 1) * per), per


def reduce_scatter_accumulator(acc, n: int, group=None, status=None):
    """Sharded form of allreduce_accumulator (ZeRO-1 style epilogue).

    ``acc`` is the flat N*10 (+1) accumulator of this rank.  Each rank receives the sum over
    ranks of its own Gaussian slice (gaussian_slice) with one trailing skip slot, as a flat
    tensor of per*10 + 1 floats: one reduce-scatter (NCCL) instead of an all-reduce, so the
    epilogue then runs on 1/world of the Gaussians.  Returns (slice_acc, skip_status int32).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    _, _, per = gaussian_slice(n, rank, world)
    chunk = per * 10 + 1
    buf = torch.zeros(world * chunk, dtype=acc.dtype, device=acc.device)
    body = buf.view(world, chunk)
    src = acc[: n * 10]
    for k in range(world):
        a, b = min(n, k * per) * 10, min(n, (k + 1) * per) * 10
        if b > a:
            body[k, : b - a].copy_(src[a:b])
    if status is not None:
        body[:, -1] = ((status[0] & SKIP_BITS) != 0).to(acc.dtype)
    out = torch.empty(chunk, dtype=acc.dtype, device=acc.device)
    try:
        dist.reduce_scatter_tensor(out, buf, op=dist.ReduceOp.SUM, group=group)
    except (RuntimeError, NotImplementedError, ValueError):  # backends without reduce-scatter (gloo)
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
        out.copy_(body[rank])
    skip = torch.where(out[-1:] > 0, SKIP_BITS, 0).to(torch.int32)
    return out, skip


def all_gather_rows(full, per: int, group=None):
    """Every rank's rows [rank*per, rank*per + per) of ``full`` ([N][k], replicated buffer)
    gathered into all ranks' copies (one all-gather of the padded slices)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n, k = full.shape
    send = torch.zeros((per, k), dtype=full.dtype, device=full.device)
    a, b = min(n, rank * per), min(n, (rank + 1) * per)
    if b > a:
        send[: b - a].copy_(full[a:b])
    recv = torch.empty((world * per, k), dtype=full.dtype, device=full.device)
    try:
        dist.all_gather_into_tensor(recv, send, group=group)
    except (RuntimeError, NotImplementedError, ValueError):
        parts = list(recv.view(world, per, k).unbind(0))
        dist.all_gather(parts, send, group=group)
    full.copy_(recv[:n])
