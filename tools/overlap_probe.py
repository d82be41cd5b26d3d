"""Probe: do the forward (K3, shared-memory atomics) and the backward (K5, FMA
pipe) overlap when launched on two streams?  Experiment tooling.

    python tools/overlap_probe.py [--reps 10]

Times K3 alone, K5 alone and both launched together on separate streams (on
independent buffers) at C2, with CUDA events.  If the together time is well
under the sum, a step pipelined over batch halves can co-schedule them.
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
from paper_2508_04929_b200 import _lib, engine  # noqa: E402
from paper_2508_04929_b200.optimize import Reconstructor  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--batch", type=int, default=256)
    args = ap.parse_args()
    n, D, B = 50000, 128, args.batch
    grid = cs.GridSpec(D, 0.5, 1.5)
    rng = np.random.default_rng(0)
    rot = np.stack([cs.sample_pose(np.random.default_rng(1000 + i)).rotation for i in range(B)])
    obs = (rng.standard_normal((B, D, D)) * 1e-3).astype(np.float32)
    d = rng.uniform(1e4, 2.5e4, B)
    ctfs = engine.ctf_array([cs.CtfParams(float(x), float(x)) for x in d])
    rec = Reconstructor(grid, cs.init_random(n, 0, grid).params, obs, engine.pose_array(rot), ctfs, batch_size=B)
    pipe = rec.pipeline(B)
    poses = rec.poses[:B].contiguous()
    pipe.forward_backward(rec.params, poses, rec.obs[:B].contiguous(), rec.ctfs[:B].contiguous())
    torch.cuda.synchronize()
    ptr = _lib._ptr if hasattr(_lib, "_ptr") else (lambda t: t.data_ptr())
    render2 = torch.empty_like(pipe.render)
    ws2 = torch.zeros_like(pipe.render_ws)
    partial2 = torch.empty_like(pipe.partial)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def fwd(st):
        _lib.call("cgs_render", pipe.splat.data_ptr(), n, poses.data_ptr(), B, pipe.grid, render2.data_ptr(),
                  None, ws2.data_ptr(), st.cuda_stream)

    def bwd(st):
        _lib.call("cgs_raster_bwd", pipe.splat.data_ptr(), n, poses.data_ptr(), B, pipe.grid,
                  pipe.upstream.data_ptr(), _lib.CGS_LAYOUT_NATURAL, partial2.data_ptr(), pipe.ipg, st.cuda_stream)

    def timed(fn):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        a.record(cur)
        for st in (s1, s2):
            st.wait_stream(cur)
        for _ in range(args.reps):
            fn()
        for st in (s1, s2):
            cur.wait_stream(st)
        b.record(cur)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / args.reps

    for _ in range(3):
        fwd(s1)
        bwd(s2)
    res = {}
    res["fwd_ms"] = timed(lambda: fwd(s1))
    res["bwd_ms"] = timed(lambda: bwd(s2))
    res["serial_ms"] = timed(lambda: (fwd(s1), bwd(s1)))
    res["together_ms"] = timed(lambda: (fwd(s1), bwd(s2)))
    res["together_bwd_first_ms"] = timed(lambda: (bwd(s2), fwd(s1)))
    res["saving_vs_sum"] = 1.0 - res["together_ms"] / (res["fwd_ms"] + res["bwd_ms"])
    print(json.dumps(res))


if __name__ == "__main__":
    main()
