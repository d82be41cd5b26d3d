"""Diagnostic (experiment tooling): render, loss and gradients of huge (30-100 px) and extreme
needle footprints against the oracle."""
import os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
from oracle import cgs_oracle as oracle
import paper_2508_04929_b200 as cs
import torch
from paper_2508_04929_b200 import engine, _lib
D = 128
grid = oracle.Grid(D, 0.5, 1.5)
poses = [oracle.sample_pose(np.random.default_rng(7000 + i)) for i in range(2)]
for sig in ((30, 30, 30), (60, 60, 60), (60, 2, 2), (100, 0.5, 0.5), (30, 0.3, 0.3), (14, 0.3, 0.3)):
    rng = np.random.default_rng(5)
    n = 12
    p = oracle.init_random(n, 5, grid)
    p[:, 0:3] = rng.normal(0.0, 0.2, (n, 3))
    p[:, 3:6] = oracle.inverse_activate(np.tile(np.array(sig, float), (n, 1)) * grid.pixel_width)
    p[:, 6:10] = rng.standard_normal((n, 4))
    p[:, 10] = oracle.inverse_activate(10.0 ** rng.uniform(-1.0, 0.0, n) / n)
    rend = cs.rasterize_batch(cs.GaussianMixture(p), np.stack([W for W, _ in poses]), np.stack([t for _, t in poses]), cs.GridSpec(D, 0.5, 1.5), method="direct")
    errs = [float(np.linalg.norm(rend[i] - oracle.rasterize(p, W, t, grid)[0]) / np.linalg.norm(oracle.rasterize(p, W, t, grid)[0])) for i, (W, t) in enumerate(poses)]
    # gradients through the fused step vs oracle
    obs = np.stack([0.5 * oracle.rasterize(p, W, t, grid)[0] for W, t in poses]).astype(np.float32)
    cp = [oracle.Ctf(15000.0, 15000.0) for _ in poses]
    ctfs = np.stack([c.as_array() for c in cp])
    ctx = engine.DeviceContext.get(0)
    gs = _lib.grid_struct(D, 0.5, 1.5)
    pipe = engine.StepPipeline(ctx, n, len(poses), gs)
    pt = torch.as_tensor(p).cuda()
    P = torch.as_tensor(engine.pose_array([W for W, _ in poses], [t for _, t in poses])).cuda()
    pipe.grow(pipe.measure_items(pt, P))
    pipe.forward_backward(pt, P, torch.as_tensor(obs).cuda(), torch.as_tensor(ctfs).cuda())
    grads = engine.epilogue_grads(ctx, pipe.partial, pipe.G, pt, 0, 1.0 / len(poses)).cpu().numpy()
    ref_l, ref_g = oracle.batch_step(p, poses, grid, [oracle.ctf_evaluate(c, grid) for c in cp], obs)
    cols = [np.linalg.norm(grads[:, j] - ref_g[:, j]) / max(np.linalg.norm(ref_g[:, j]), 1e-6 * np.linalg.norm(ref_g)) for j in range(11)]
    ge = max(cols)
    if os.environ.get("DIAG_COLS"):
        print("   cols", ["%.1e" % c for c in cols])
    print("sigma", sig, "render", ["%.2e" % e for e in errs], "grad col max %.2e" % ge, "loss rel %.2e" % float(np.max(np.abs(pipe.loss.cpu().numpy() - ref_l) / np.abs(ref_l))), flush=True)
