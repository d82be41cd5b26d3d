"""Time the FFT kernels alone at a config (A/B tooling; bench.py holds the headline).

    CGS_B200_LIB=... python tools/k4_probe.py [--D 128] [--B 256] [--iters 30]

Times cgs_obs_spectrum (per-step observation records, the e2e path),
cgs_ctf_mse_spectral_fixed (the training step's K4; the _fft forms at sizes without
line-FFT kernels) and the real-space cgs_ctf_mse on random images and bench-like
CTFs; prints ms per launch (CUDA events, median of 5 blocks of `iters` launches)
and checksums of the loss and upstream so variants can be compared.
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
    ap.add_argument("--D", type=int, default=128)
    ap.add_argument("--B", type=int, default=256)
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--tag", default=os.environ.get("CGS_B200_LIB", "base"))
    a = ap.parse_args()
    ctx = engine.DeviceContext.get()
    gs = _lib.grid_struct(a.D, 0.5, 1.5)
    s = ctx.stream
    rng = np.random.default_rng(0)
    ctf = np.zeros((a.B, 8))
    ctf[:, 0] = rng.uniform(1e4, 2.5e4, a.B)
    ctf[:, 1] = ctf[:, 0] + rng.uniform(-500, 500, a.B)
    ctf[:, 2] = rng.uniform(0, np.pi, a.B)
    ctf[:, 3:] = [300.0, 2.7, 0.1, 0.0, 0.0]
    ctf_t = torch.as_tensor(ctf).cuda()
    g = torch.Generator(device="cuda").manual_seed(1)
    obs = torch.randn((a.B, a.D, a.D), generator=g, device="cuda")
    # a fixed-point render as cgs_render_fixed leaves it: int32 values in unit `scale`
    scale = torch.tensor([2.0 ** 20], dtype=torch.float32, device="cuda")
    render = (torch.rand((a.B, a.D, a.D), generator=g, device="cuda") * 2.0 ** 20).to(torch.int32)
    fft = int(ctx.lib.cgs_obs_spectrum_elems(a.D, a.B)) == 0  # sizes without line-FFT kernels: the cuFFT form
    elems = ctx.lib.cgs_obs_spectrum_fft_elems(a.D, a.B) if fft else ctx.lib.cgs_obs_spectrum_elems(a.D, a.B)
    spec = torch.empty(int(elems), dtype=torch.float32, device="cuda")
    plan = ctx.plan(a.D, a.B)
    wspec = torch.empty(2 * int(ctx.lib.cgs_fft_spectrum_elems(a.D, a.B)), dtype=torch.float32, device="cuda")
    ws = torch.zeros(int(ctx.lib.cgs_spectral_fft_workspace_bytes(a.D, a.B)) + 8, dtype=torch.uint8, device="cuda")
    up = torch.empty((a.B, a.D, a.D), dtype=torch.float32, device="cuda")
    loss = torch.empty(a.B, dtype=torch.float64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")

    def obs_rec():
        if fft:
            _lib.call("cgs_obs_spectrum_fft", plan, obs.data_ptr(), ctf_t.data_ptr(), a.B, gs, wspec.data_ptr(),
                      spec.data_ptr(), s)
        else:
            _lib.call("cgs_obs_spectrum", obs.data_ptr(), ctf_t.data_ptr(), a.B, gs, spec.data_ptr(), s)

    def k4():
        if fft:
            _lib.call("cgs_ctf_mse_spectral_fft", plan, render.data_ptr(), scale.data_ptr(), spec.data_ptr(), 0,
                      a.B, gs, wspec.data_ptr(), ws.data_ptr(), up.data_ptr(), loss.data_ptr(), status.data_ptr(),
                      _lib.CGS_LAYOUT_ROWPAIR, s)
        else:
            _lib.call("cgs_ctf_mse_spectral_fixed", render.data_ptr(), scale.data_ptr(), spec.data_ptr(), a.B, gs,
                      up.data_ptr(), loss.data_ptr(), status.data_ptr(), _lib.CGS_LAYOUT_ROWPAIR, s)

    def k4_spatial():  # the real-space K4 (cgs_ctf_mse: two cuFFT transform pairs at sizes without fused kernels)
        _lib.call("cgs_ctf_mse", plan, up.data_ptr(), obs.data_ptr(), a.B, gs, ctf_t.data_ptr(), wspec.data_ptr(),
                  0, up2.data_ptr(), loss.data_ptr(), status.data_ptr(), _lib.CGS_LAYOUT_NATURAL, s)

    res = {"tag": os.path.basename(a.tag), "D": a.D, "B": a.B}
    up2 = torch.empty_like(up)
    for name, fn in (("obs_spectrum", obs_rec), ("k4", k4), ("k4_spatial", k4_spatial)):
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
        res[name + "_us"] = round(1e3 * statistics.median(blocks), 2)
    res["spec_sum"] = float(spec.double().abs().sum())
    res["loss_sum"] = float(loss.sum())
    res["up_sum"] = float(up.double().abs().sum())
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
