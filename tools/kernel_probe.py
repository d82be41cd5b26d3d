"""Time the two raster kernels alone at a config (A/B tooling; bench.py holds the headline).

    CGS_B200_LIB=... python tools/kernel_probe.py [--n 50000] [--D 128] [--B 256] [--iters 30]

Renders (cgs_render_fixed, the training step's K3) and backward (cgs_raster_bwd from a
row-pair upstream, K5) on init_random Gaussians in Morton order with the bench's poses;
prints ms per launch (CUDA events, median of 5 blocks of `iters` launches) and a render
checksum so variants can be compared for identical output.
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

import paper_2508_04929_b200 as cs  # noqa: E402
from paper_2508_04929_b200 import _lib, engine  # noqa: E402
from paper_2508_04929_b200.optimize import morton_order  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=50000)
    ap.add_argument("--D", type=int, default=128)
    ap.add_argument("--B", type=int, default=256)
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--layout", choices=("rowpair", "natural"), default="rowpair",
                    help="upstream layout K5 reads (the spectral K4 writes row pairs at 64/128, cuFFT natural)")
    ap.add_argument("--tag", default=os.environ.get("CGS_B200_LIB", "base"))
    a = ap.parse_args()
    grid = cs.GridSpec(a.D, 0.5, 1.5)
    mix = cs.init_random(a.n, 0, grid)
    params = mix.params[morton_order(mix.params[:, :3], grid.extent)]
    ctx = engine.DeviceContext.get()
    gs = _lib.grid_struct(a.D, 0.5, 1.5)
    rot = np.stack([cs.sample_pose(np.random.default_rng(1000 + i)).rotation for i in range(a.B)])
    P = torch.as_tensor(engine.pose_array(rot)).cuda()
    p = torch.as_tensor(params).cuda()
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    splat = engine.prepare(ctx, p, status)
    out = torch.empty((a.B, a.D, a.D), dtype=torch.float32, device="cuda")
    ws = torch.zeros(ctx.lib.cgs_render_workspace_bytes(a.n) // 4 + 1, dtype=torch.float32, device="cuda")
    up = torch.randn((a.B, a.D, a.D), generator=torch.Generator(device="cuda").manual_seed(1), device="cuda") * 1e-3
    G = int(ctx.lib.cgs_bwd_groups(a.B, engine.images_per_group_auto(a.n, a.B)))
    part = torch.empty(G * a.n * 10, dtype=torch.float32, device="cuda")
    s = ctx.stream
    layout = _lib.CGS_LAYOUT_ROWPAIR if a.layout == "rowpair" else _lib.CGS_LAYOUT_NATURAL

    def fwd():
        _lib.call("cgs_render_fixed", splat.data_ptr(), a.n, P.data_ptr(), a.B, gs, out.data_ptr(), None,
                  ws.data_ptr(), s)

    def bwd():
        _lib.call("cgs_raster_bwd", splat.data_ptr(), a.n, P.data_ptr(), a.B, gs, up.data_ptr(),
                  layout, part.data_ptr(), engine.images_per_group_auto(a.n, a.B), s)

    res = {"tag": os.path.basename(a.tag), "n": a.n, "D": a.D, "B": a.B, "layout": a.layout}
    for name, fn in (("fwd", fwd), ("bwd", bwd)):
        for _ in range(3):
            fn()
        blocks = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.iters):
                fn()
            e1.record()
            torch.cuda.synchronize()
            blocks.append(e0.elapsed_time(e1) / a.iters)
        res[name + "_ms"] = round(statistics.median(blocks), 4)
    img = out.view(torch.int32).double() / ws[0].double()
    res["render_sum"] = float(img.sum())
    res["partial_sum"] = float(part.double().abs().sum())
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
