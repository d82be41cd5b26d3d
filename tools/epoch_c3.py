"""C3 of SURVEY.md 8(d): one full reconstruction epoch on a 100k-particle synthetic dataset.

    python tools/epoch_c3.py [--particles 100000] [--out profiles/epoch_c3_r01.json]
    torchrun --nproc-per-node N tools/epoch_c3.py     (N ranks share each global batch)

The dataset (128^2, helix-50 truth, DefocusRange(1e4, 2.5e4), SNR 0.1) is generated on the GPU
by ``cs.simulate`` with device noise and kept in HBM (6.5 GB at 100k).  The epoch is the
reference's schedule at a fixed global batch of 256: the seeded permutation cut into 391
batches (train.py:228-232), one Reconstructor step each (50k random-init Gaussians, CTF, Adam).
Timed with CUDA events around the whole epoch, after 50 warm-up steps; the loss is read back
once at the end.  Experiment tooling: bench.py holds the headline line.
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2508_04929_b200 as cs  # noqa: E402
from paper_2508_04929_b200 import engine  # noqa: E402
from paper_2508_04929_b200.optimize import Reconstructor  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--particles", type=int, default=100_000)
    ap.add_argument("--gaussians", type=int, default=50_000)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    pg = None
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("nccl")
        pg = dist.group.WORLD
    grid = cs.GridSpec(128, 0.5, 1.5)
    spec = cs.SimSpec(truth=cs.make_phantom("helix", 50), num_particles=args.particles, grid=grid,
                      ctf_distribution=cs.DefocusRange(1e4, 2.5e4), noise=cs.NoiseModel(snr=0.1), seed=0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = cs.simulate(spec, noise="device", keep_on_device=True)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    recs = res.records
    poses = engine.pose_array(np.stack([r.pose.rotation for r in recs]))
    ctfs = engine.ctf_array([r.ctf for r in recs])
    params = cs.init_random(args.gaussians, 0, grid).params
    # one GPU: the whole stack in HBM; N ranks: each holds its shards of the epoch's batches
    rec = Reconstructor(grid, params, res.images, poses, ctfs, batch_size=args.batch, process_group=pg)
    del res
    order = np.random.default_rng(0).permutation(args.particles)  # train.py:228-232
    rec.begin_epoch(order)
    batches = [order[i:i + args.batch] for i in range(0, args.particles, args.batch)]
    # warm-up (pipelines, graphs, clocks), including the short last batch's shape (100000 = 390 x 256
    # + 160): its graph is captured here, not inside the timed epoch
    for b in batches[:50] + [batches[-1]]:
        rec.step(b, args.lr)
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    losses = []
    a.record()
    for b in batches:
        losses.append(rec.step(b, args.lr).clone())
    e.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(e)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    first = float(losses[0].mean().item())
    last = float(torch.cat([x.reshape(-1) for x in losses[-10:]]).mean().item())
    out = {"config": "C3", "particles": args.particles, "residency": rec.residency, "n_gaussians": args.gaussians, "image_px": 128,
           "global_batch": args.batch, "steps": len(batches), "n_gpus": world, "epoch_s": ms / 1e3,
           "images_per_s": args.particles / (ms / 1e3), "ms_per_step": ms / len(batches),
           "generate_s": gen_s, "generate_images_per_s": args.particles / gen_s,
           "loss_first_batch": first, "loss_last_10_batches": last, "device": torch.cuda.get_device_name()}
    if rank == 0:
        print(json.dumps(out))
        if args.out:
            json.dump(out, open(args.out, "w"), indent=1)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
