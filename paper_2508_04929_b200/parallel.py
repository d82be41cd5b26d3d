"""Data parallelism over particles.

Every rank holds the full mixture (N x 11 fp64 + Adam moments) and takes a
contiguous share of each global batch (``shard``); the only exchange per step
is the 10-float per-Gaussian world-frame accumulator, summed over ranks, after
which the fused epilogue + Adam runs.  Two layouts (``Exchange``):

* replicated: one all-reduce (SUM) of the N x 10 accumulator (2 MB at 50k),
  then every rank runs the identical epilogue + Adam on all Gaussians;
* sharded (ZeRO-1 style, ``CGS_DP_SHARDED=1``): one reduce-scatter, each rank
  runs the epilogue + Adam on its own ceil(N / world) Gaussians, then one
  all-gather of the fp64 parameters.

The accumulator is written by ``cgs_reduce_partials_sliced`` directly in the
collective's layout (per-rank slices, each with this rank's skip flag), and
the parameters live in a buffer padded to world x ceil(N / world) rows, so
both collectives run in place: no send-buffer copies.  Every buffer is
preallocated, so with NCCL the whole step (kernels and collectives) is
captured in one CUDA graph; on gloo (CPU tests, or several ranks sharing one
GPU in the GPU tests) the collectives run eagerly between captured segments.

A rank's skip flag (non-finite loss, non-finite parameters, bin overflow)
travels in its slice of the summed buffer, so every rank makes the same skip
decision and the replicated parameters cannot diverge.

Particle residency (``epoch_records``): with the reference's global seeded
shuffle (train.py:228-232) a rank needs, per epoch, exactly the records of its
slices of that epoch's batches, 1/world of the dataset; ``Reconstructor`` with
``residency="epoch"`` keeps only those in HBM (and the next epoch's, while it
prefetches them).
"""

from __future__ import annotations

import numpy as np

# status bits that make the Adam epilogue skip a step (cgs_b200.h)
SKIP_BITS = 2 | 4 | 8  # CGS_STATUS_BIN_OVERFLOW | CGS_STATUS_NONFINITE_LOSS | CGS_STATUS_NONFINITE_PARAMS


def shard(indices, rank: int, world: int) -> np.ndarray:
    """Contiguous slice [B*rank/world, B*(rank+1)/world) of a global batch."""
    idx = np.asarray(indices)
    B = len(idx)
    return idx[(B * rank) // world:(B * (rank + 1)) // world]


def epoch_batches(n_records: int, batch_size: int, rng: np.random.Generator):
    """The seeded per-epoch visiting order cut into global batches (train.py:228-232)."""
    order = rng.permutation(n_records)
    return [order[i:i + batch_size] for i in range(0, n_records, batch_size)]


def epoch_records(order, batch_size: int, rank: int, world: int) -> np.ndarray:
    """The records a rank touches in one epoch: its shard of every global batch cut from
    ``order``, in step order (each record once)."""
    order = np.asarray(order)
    parts = [shard(order[i:i + batch_size], rank, world) for i in range(0, len(order), batch_size)]
    return np.concatenate(parts) if parts else np.zeros(0, dtype=order.dtype)


def gaussian_slice(n: int, rank: int, world: int):
    """(start, stop, rows per rank) of the Gaussians whose optimizer state this rank owns in the
    sharded epilogue: equal slices of ceil(n / world) rows, the last one short (or empty)."""
    per = -(-n // world)
    return min(n, rank * per), min(n, (rank + 1) * per), per


def backend_of(group=None) -> str:
    import torch.distributed as dist

    return str(dist.get_backend(group)).lower()


class Exchange:
    """Preallocated buffers and collectives of one data-parallel step.

    ``acc`` f32: the layout cgs_reduce_partials_sliced writes (slices of ``per`` Gaussians,
    ``slice`` floats each, the last two being this rank's skip flag and padding); ``skip`` int32
    [1]: SKIP_BITS when any rank flagged its step.  ``run()`` issues the collective in place;
    ``own()`` is this rank's summed slice with its row range; ``gather_rows(store)`` all-gathers a
    [world * per][k] buffer from every rank's rows (sharded mode)."""

    def __init__(self, n: int, group=None, *, sharded: bool, device=None, slice_floats=None):
        import torch
        import torch.distributed as dist

        self.n = int(n)
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.sharded = bool(sharded)
        self.backend = backend_of(group)
        self.per = gaussian_slice(self.n, self.rank, self.world)[2] if self.sharded else self.n
        self.slice = int(slice_floats) if slice_floats is not None else self.per * 10 + 2
        nslices = self.world if self.sharded else 1
        self.acc = torch.zeros(nslices * self.slice, dtype=torch.float32, device=device)
        self.skip = torch.zeros(1, dtype=torch.int32, device=device)
        self.rows = gaussian_slice(self.n, self.rank, self.world)[:2] if self.sharded else (0, self.n)

    @property
    def capturable(self) -> bool:
        """Collectives can sit inside a captured CUDA graph (NCCL)."""
        return self.backend == "nccl"

    def own(self):
        """(this rank's summed accumulator rows, first row, stop row)."""
        k = self.rank if self.sharded else 0
        return self.acc[k * self.slice:(k + 1) * self.slice], self.rows[0], self.rows[1]

    def run(self) -> None:
        """Sum the accumulator over ranks (in place), then derive the shared skip decision."""
        import torch
        import torch.distributed as dist

        # (also in a 1-rank group, CGS_DP_EXCHANGE=1: the collective path itself runs)
        if self.sharded and self.backend != "gloo":
            part = self.acc[self.rank * self.slice:(self.rank + 1) * self.slice]
            dist.reduce_scatter_tensor(part, self.acc, op=dist.ReduceOp.SUM, group=self.group)
        else:  # replicated layout, or gloo (no reduce-scatter): the own slice is summed in place
            dist.all_reduce(self.acc, op=dist.ReduceOp.SUM, group=self.group)
        part = self.own()[0]
        flag = part[self.per * 10:self.per * 10 + 1]
        self.skip.copy_(torch.where(flag > 0, SKIP_BITS, 0).to(torch.int32))

    def gather_rows(self, store) -> None:
        """All-gather [world * per][k] ``store`` in place from every rank's rows."""
        import torch.distributed as dist

        per = self.per
        mine = store[self.rank * per:(self.rank + 1) * per]
        if self.backend == "gloo":  # no in-place all_gather_into_tensor: gather into the row views
            dist.all_gather(list(store.view(self.world, per, -1).unbind(0)), mine.clone(), group=self.group)
        else:
            dist.all_gather_into_tensor(store, mine, group=self.group)


class PeerExchange(Exchange):
    """The exchange as ONE kernel over peer memory (``cgs_peer_epilogue_adam``, ``CGS_DP_PEER=1``).

    The accumulator (reduce-scatter layout), the fp64 parameter store (``store``: world x per
    rows) and a u32 [world + 1] handshake array are allocated in symmetric memory
    (``torch.distributed._symmetric_memory``) and mapped into every rank; ``acc_ptrs``,
    ``store_ptrs`` and ``flag_ptrs`` are device arrays of the peers' addresses.  Per step each
    rank's launch sums its slice of every peer's accumulator (fp64, rank order), runs the
    epilogue + Adam on it and stores the new rows into every peer's store, with a release /
    acquire handshake before and after: reduce-scatter, Adam and parameter all-gather in one
    launch, no NCCL call on the step's data path (the NCCL collectives stay for
    the rare moment gathers of ``reorder`` / ``moments_host``).  Everything is preallocated and
    the step has no host-side collective, so it is captured whole in the step's CUDA graph."""

    def __init__(self, n: int, group=None, *, device=None, slice_floats=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        super().__init__(n, group, sharded=True, device=device, slice_floats=slice_floats)
        grp = group if group is not None else dist.group.WORLD
        if hasattr(symm_mem, "is_symm_mem_enabled_for_group") and not symm_mem.is_symm_mem_enabled_for_group(
                grp.group_name):
            symm_mem.enable_symm_mem_for_group(grp.group_name)
        self.acc = symm_mem.empty(self.world * self.slice, dtype=torch.float32, device=device)
        self.store = symm_mem.empty((self.world * self.per, 11), dtype=torch.float64, device=device)
        # arrive slots + done counter, padded to 16 words
        self.flags = symm_mem.empty(max(16, self.world + 1), dtype=torch.int32, device=device)
        self.acc.zero_()
        self.store.zero_()
        self.flags.zero_()
        torch.cuda.synchronize(device)  # zeroed on every rank before any peer can signal into it
        self.acc_ptrs = self._peer_ptrs(self.acc, grp, device)
        self.store_ptrs = self._peer_ptrs(self.store, grp, device)
        self.flag_ptrs = self._peer_ptrs(self.flags, grp, device)
        dist.barrier(group=group)

    def _peer_ptrs(self, t, group, device):
        import torch
        import torch.distributed._symmetric_memory as symm_mem

        h = symm_mem.rendezvous(t, group)
        base = h.buffer_ptrs
        off = t.data_ptr() - base[self.rank]
        return torch.tensor([int(b) + off for b in base], dtype=torch.int64, device=device)

    @property
    def capturable(self) -> bool:
        return True

    def run(self) -> None:  # the exchange is inside cgs_peer_epilogue_adam
        raise RuntimeError("PeerExchange has no separate collective: the step launches cgs_peer_epilogue_adam")


def allreduce_accumulator(acc, group=None, status=None):
    """Sum a flat N*10 (+1) accumulator over ranks in place (one collective); with ``status`` the
    trailing slot carries this rank's skip flag.  Returns the int32 skip status (SKIP_BITS if any
    rank skips, else 0), or ``acc`` when ``status`` is None.  (Host-level helper; the training
    step uses ``Exchange``.)"""
    import torch
    import torch.distributed as dist

    if status is not None:
        acc[-1] = ((status[0] & SKIP_BITS) != 0).to(acc.dtype)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
    if status is None:
        return acc
    return torch.where(acc[-1:] > 0, SKIP_BITS, 0).to(torch.int32)
