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
SKIP_BITS = 2 | 4  # CGS_STATUS_BIN_OVERFLOW | CGS_STATUS_NONFINITE_LOSS


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
