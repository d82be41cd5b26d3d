"""Time K6 (cgs_epilogue_adam) alone at a config (A/B tooling; bench.py holds the headline).

    CGS_B200_LIB=... python tools/epi_probe.py [--n 50000] [--groups 24] [--iters 50]

Random image-group partials (warm in L2 after the first launch, as right after K5), random
parameters; prints us per launch (CUDA events, median of 5 blocks) for the default kernel and
the one-thread-per-Gaussian kernel (CGS_EPI_NARROW=1), and with one group only.
"""

import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2508_04929_b200 import _lib, engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=50000)
    ap.add_argument("--groups", type=int, default=24)
    ap.add_argument("--iters", type=int, default=50)
    a = ap.parse_args()
    ctx = engine.DeviceContext.get()
    rng = np.random.default_rng(0)
    part = torch.as_tensor(rng.standard_normal((a.groups, a.n, 10)).astype(np.float32) * 1e-6).cuda()
    p0 = rng.standard_normal((a.n, 11))
    p0[:, 3:6] = -5.0
    prm = torch.as_tensor(p0).cuda()
    m = torch.zeros_like(prm)
    v = torch.zeros_like(prm)
    hyper = torch.tensor([1e-3, 0.1, 0.001, 1.0], dtype=torch.float64, device="cuda")

    def run(G):
        _lib.call("cgs_epilogue_adam_dev", part.data_ptr(), G, a.n, prm.data_ptr(), m.data_ptr(), v.data_ptr(), 0,
                  1.0 / 256, 0.9, 0.999, 1e-8, hyper.data_ptr(), None, ctx.stream)

    res = {}
    for narrow in ("0", "1"):
        os.environ["CGS_EPI_NARROW"] = narrow
        for G in (a.groups, 1):
            for _ in range(3):
                run(G)
            blocks = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(a.iters):
                    run(G)
                e1.record()
                torch.cuda.synchronize()
                blocks.append(1e3 * e0.elapsed_time(e1) / a.iters)
            res[f"{'narrow' if narrow == '1' else 'wide'}_G{G}_us"] = round(statistics.median(blocks), 2)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
