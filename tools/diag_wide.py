"""Diagnostic (experiment tooling): the direct render of wide / needle mixtures against the oracle."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import cgs_oracle as oracle
import paper_2508_04929_b200 as cs
D = 128
grid = oracle.Grid(D, 0.5, 1.5)
def mix(n, frac_needle, amp_spread, seed=21):
    rng = np.random.default_rng(seed)
    p = oracle.init_random(n, seed, grid)
    p[:, 0:3] = rng.normal(0.0, 0.15, (n, 3))
    px = rng.uniform(2.0, 14.0, (n, 3))
    needles = rng.random(n) < frac_needle
    px[needles] = [14.0, 0.3, 0.3]
    p[:, 3:6] = oracle.inverse_activate(px * grid.pixel_width)
    p[:, 6:10] = rng.standard_normal((n, 4))
    p[:, 10] = oracle.inverse_activate(10.0 ** rng.uniform(-amp_spread, 0.0, n) / n)
    return p
poses = [oracle.sample_pose(np.random.default_rng(6000 + i)) for i in range(3)]
for n, fn, sp in ((20, 1.0, 0.0), (300, 1.0, 0.0), (300, 1.0, 2.0), (400, 0.3, 0.0), (400, 0.3, 2.0), (400, 0.0, 2.0)):
    p = mix(n, fn, sp)
    rend = cs.rasterize_batch(cs.GaussianMixture(p), np.stack([W for W, _ in poses]), np.stack([t for _, t in poses]), cs.GridSpec(D, 0.5, 1.5), method="direct")
    errs = []
    for i, (W, t) in enumerate(poses):
        ref, _ = oracle.rasterize(p, W, t, grid)
        errs.append(float(np.linalg.norm(rend[i] - ref) / np.linalg.norm(ref)))
    print("n", n, "needles", fn, "amp spread 10^", sp, ["%.2e" % e for e in errs], flush=True)
p = mix(400, 0.3, 2.0)
W, t = poses[0]
rend = cs.rasterize_batch(cs.GaussianMixture(p), W[None], t[None], cs.GridSpec(D, 0.5, 1.5), method="direct")[0]
ref, _ = oracle.rasterize(p, W, t, grid)
# per-class references
rng = np.random.default_rng(21); rng.normal(0.0, 0.15, (400, 3)); rng.uniform(2.0, 14.0, (400, 3)); needles = rng.random(400) < 0.3
ref_needle, _ = oracle.rasterize(p[needles], W, t, grid)
ref_wide, _ = oracle.rasterize(p[~needles], W, t, grid)
np.savez(os.path.join(os.environ.get("OUT", "."), "diag_mix.npz"), rend=rend, ref=ref, ref_needle=ref_needle, ref_wide=ref_wide)
