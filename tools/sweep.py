"""Throughput sweep over the SURVEY.md 8(d) configurations on one GPU.

    python tools/sweep.py [--steps K] [--out profiles/sweep_r01.json]

C1 (5k Gaussians, 64^2, B=32, no CTF), C2 (50k, 128^2, B=256, CTF), C4 per GPU
(200k, 256^2, B=64 of the 512 global batch, CTF) and the C5 Gaussian-count
sweep (10k..1M at 128^2, B=256, CTF).  Each point times K full training steps
(render, CTF, MSE, CTF^T, backward, epilogue + Adam) with CUDA events after 3
warm-up steps, on device-resident random observations (the pixel work does
not depend on their values) cycled over 8 batches, and reports images/s plus
in-ellipse pairs/s.  Experiment tooling: bench.py holds the headline line.
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2508_04929_b200 as cs  # noqa: E402
from paper_2508_04929_b200 import engine  # noqa: E402
from paper_2508_04929_b200.optimize import Reconstructor  # noqa: E402

CONFIGS = [("C1", 5000, 64, 32, False)]
CONFIGS += [("C2", 50000, 128, 256, True)]
CONFIGS += [("C4/gpu", 200000, 256, 64, True)]
CONFIGS += [(f"C5-{n // 1000}k", n, 128, 256, True) for n in (10000, 20000, 100000, 200000, 500000, 1000000)]


def point(name, n, D, B, ctf, steps):
    grid = cs.GridSpec(D, 0.5, 1.5)
    nbatch = 8
    rng = np.random.default_rng(0)
    poses = [cs.sample_pose(np.random.default_rng(1000 + i)) for i in range(nbatch * B)]
    rot = np.stack([p.rotation for p in poses])
    obs = (rng.standard_normal((nbatch * B, D, D)) * 1e-3).astype(np.float32)
    ctfs = None
    if ctf:
        d = rng.uniform(1e4, 2.5e4, nbatch * B)
        ctfs = engine.ctf_array([cs.CtfParams(float(x), float(x)) for x in d])
    mix = cs.init_random(n, 0, grid)
    rec = Reconstructor(grid, mix.params, obs, engine.pose_array(rot), ctfs, batch_size=B)
    dev = rec.ctx.device
    batches = []
    for k in range(nbatch):
        idx = torch.arange(k * B, (k + 1) * B, device=dev)
        batches.append((rec.obs.index_select(0, idx).contiguous(), rec.poses.index_select(0, idx).contiguous(),
                        None if rec.ctfs is None else rec.ctfs.index_select(0, idx).contiguous()))
    pipe = rec.pipeline(B)
    splat = engine.prepare(rec.ctx, rec.params, pipe.status)
    pairs = [int(engine.count_pairs(rec.ctx, splat, n, p, rec.gs).sum().item()) for _, p, _ in batches]
    for k in range(3):
        rec.step_batch(*batches[k % nbatch], 1e-3, global_batch=B)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(steps):
        rec.step_batch(*batches[k % nbatch], 1e-3, global_batch=B)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    p = sum(pairs[k % nbatch] for k in range(steps)) / steps
    # one more step with per-stage CUDA events (fwd = weight bound + render; ctf = K4, with the
    # per-step observation records; bwd = K5; epi = epilogue + Adam)
    ev = {s: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for s in ("fwd", "ctf", "bwd", "epi")}
    rec.step_batch(*batches[steps % nbatch], 1e-3, global_batch=B, events=ev)
    torch.cuda.synchronize()
    stage = {s: round(e[0].elapsed_time(e[1]), 4) for s, e in ev.items()}
    return {"config": name, "n_gaussians": n, "image_px": D, "batch": B, "ctf": ctf, "ms_per_step": ms,
            "images_per_s": B / (ms / 1e3), "pairs_per_image": p / B, "gpairs_per_s": p / (ms / 1e3) / 1e9,
            "stage_ms": stage}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--out", default=None)
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    res = []
    for c in CONFIGS:
        if args.only and c[0] not in args.only.split(","):
            continue
        r = point(*c, args.steps)
        print(json.dumps(r), flush=True)
        res.append(r)
    if args.out:
        json.dump({"device": torch.cuda.get_device_name(), "points": res}, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
