"""Diagnostic (experiment tooling): render error vs needle aspect and amplitude spread in wide/needle mixtures."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import cgs_oracle as oracle
import paper_2508_04929_b200 as cs
D = 128
grid = oracle.Grid(D, 0.5, 1.5)
poses = [oracle.sample_pose(np.random.default_rng(6000 + i)) for i in range(3)]
for minor in (0.3, 0.5, 1.0, 2.0):
    for spread in (0.0, 1.0, 2.0):
        rng = np.random.default_rng(21)
        n = 400
        p = oracle.init_random(n, 21, grid)
        p[:, 0:3] = rng.normal(0.0, 0.15, (n, 3))
        px = rng.uniform(2.0, 14.0, (n, 3))
        needles = rng.random(n) < 0.3
        px[needles] = [14.0, minor, minor]
        p[:, 3:6] = oracle.inverse_activate(px * grid.pixel_width)
        p[:, 6:10] = rng.standard_normal((n, 4))
        p[:, 10] = oracle.inverse_activate(10.0 ** rng.uniform(-spread, 0.0, n) / n)
        rend = cs.rasterize_batch(cs.GaussianMixture(p), np.stack([W for W, _ in poses]), np.stack([t for _, t in poses]), cs.GridSpec(D, 0.5, 1.5), method="direct")
        errs = []
        for i, (W, t) in enumerate(poses):
            ref = oracle.rasterize(p, W, t, grid)[0]
            errs.append(float(np.linalg.norm(rend[i] - ref) / np.linalg.norm(ref)))
        print("minor", minor, "spread", spread, "max err %.2e" % max(errs), flush=True)
