"""Diagnostic (experiment tooling): the training step (render, losses, gradients) at image sizes
outside the spectral K4's 64 / 128 (odd, non-power-of-two, 256) against the oracle."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import cgs_oracle as oracle
from paper_2508_04929_b200 import engine, _lib
for D in (33, 48, 96, 100, 64, 256):
    grid = oracle.Grid(D, 0.5, 1.5)
    n, B = 300, 3
    p = oracle.init_random(n, 3, grid)
    poses = [oracle.sample_pose(np.random.default_rng(8000 + i)) for i in range(B)]
    cp = [oracle.Ctf(12000.0 + 3000 * i, 14000.0, 0.2 * i) for i in range(B)]
    ctfs = np.stack([c.as_array() for c in cp])
    refs = [oracle.rasterize(p, W, t, grid)[0] for W, t in poses]
    obs = np.stack([0.7 * r for r in refs]).astype(np.float32)
    ctx = engine.DeviceContext.get(0)
    gs = _lib.grid_struct(D, 0.5, 1.5)
    pipe = engine.StepPipeline(ctx, n, B, gs)
    pt = torch.as_tensor(p).cuda()
    P = torch.as_tensor(engine.pose_array([W for W, _ in poses], [t for _, t in poses])).cuda()
    pipe.grow(pipe.measure_items(pt, P))
    pipe.forward_backward(pt, P, torch.as_tensor(obs).cuda(), torch.as_tensor(ctfs).cuda())
    rend = pipe.render_image().cpu().numpy()
    grads = engine.epilogue_grads(ctx, pipe.partial, pipe.G, pt, 0, 1.0 / B).cpu().numpy()
    ref_l, ref_g = oracle.batch_step(p, poses, grid, [oracle.ctf_evaluate(c, grid) for c in cp], obs)
    re = max(float(np.linalg.norm(rend[i] - refs[i]) / np.linalg.norm(refs[i])) for i in range(B))
    ge = max(np.linalg.norm(grads[:, j] - ref_g[:, j]) / max(np.linalg.norm(ref_g[:, j]), 1e-6 * np.linalg.norm(ref_g)) for j in range(11))
    le = float(np.max(np.abs(pipe.loss.cpu().numpy() - ref_l) / np.abs(ref_l)))
    print("D", D, "spectral" if pipe.spectral else "cufft", "render %.2e loss %.2e grad %.2e" % (re, le, ge), flush=True)
