"""Diagnostic (experiment tooling): the worst case of the fixed-point range -- thousands of identical
isotropic Gaussians stacked on one point (every bound tight, every peak on one pixel)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import cgs_oracle as oracle
import paper_2508_04929_b200 as cs
D = 64
grid = oracle.Grid(D, 0.5, 1.5)
W, t = oracle.sample_pose(np.random.default_rng(1))
for n in (1, 8192, 20000, 100000):
    p = oracle.init_random(n, 0, grid)
    p[:, 0:3] = 0.0
    p[:, 3:6] = oracle.inverse_activate(np.full((n, 3), 0.8 * grid.pixel_width))
    p[:, 6:10] = [1.0, 0.0, 0.0, 0.0]
    p[:, 10] = oracle.inverse_activate(1.0 / n)
    rend = cs.rasterize_batch(cs.GaussianMixture(p), W[None], t[None], cs.GridSpec(D, 0.5, 1.5), method="direct")[0]
    ref, _ = oracle.rasterize(p[:1], W, t, grid)  # identical Gaussians: n x (1/n) = the single one
    ref = ref * n
    err = float(np.linalg.norm(rend - ref) / np.linalg.norm(ref))
    print("n", n, "rel %.2e" % err, "peak got %.6g ref %.6g" % (rend.max(), ref.max()), "min", float(rend.min()), flush=True)
