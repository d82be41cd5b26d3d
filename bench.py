"""Benchmark: particle images/s for the fwd+bwd(+Adam) splatting step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[1], the metric's configuration): 50k Gaussians
(init_random(50000, 0)), 128x128 particles, batch 256 per GPU, known poses +
per-particle CTF, one full training step per "step": project, bin, render,
CTF, MSE, CTF^T, backward, all-reduce (N>1), epilogue + Adam.  Synthetic
particles (helix-50 phantom, 300 kV, defocus U(1e4, 2.5e4) A, SNR 0.1) are
generated on the device; a dataset of 2048 particles per rank (134 MB, larger
than the 126 MB L2) is cycled, so consecutive steps read different inputs.

One JSON line on rank 0: value = images/s over all ranks (device time, CUDA
events, max over ranks); e2e = the same through the public host-buffer API
(pinned H2D of each step's batch + D2H of its losses inside the timed region);
roofline for the dominant kernel (raster_bwd) against the FP32/SFU issue
roofline of SURVEY.md 8(d); cpu_baseline = the CPU oracle (fp64 NumPy + C
restatement of the reference, "port") on the host cores.  --impl reference
times that CPU path alone (the reference arm).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("MKL_NUM_THREADS", "1")

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particle images/sec (fwd+bwd step, 128² px, 50k Gaussians)"
N_GAUSS, D, BATCH_PER_GPU = 50000, 128, 256
DATASET = int(os.environ.get("CGS_BENCH_DATASET", "2048"))  # particles per rank (A/B experiments only)
GLOBAL_BATCH_STRONG = 256  # --scaling strong: C3's fixed global batch
PIXEL_A = 1.5
WORKLOAD = "C2: 50k init_random Gaussians, 128x128 particles, batch 256/GPU, known poses + CTF, fwd+bwd+Adam"
WORKLOAD_STRONG = ("C3-style strong scaling: 50k init_random Gaussians, 128x128 particles, fixed global batch 256 "
                   "split over the GPUs, known poses + CTF, fwd+bwd+all-reduce+Adam")


# ---------------------------------------------------------------------------
# CPU oracle timing (test infrastructure used as the baseline, never product)
# ---------------------------------------------------------------------------
_W = {}


def _cpu_worker_init():
    from oracle import cgs_oracle as oracle

    oracle.build_loops()
    grid = oracle.Grid(D, 0.5, PIXEL_A)
    _W["oracle"] = oracle
    _W["grid"] = grid
    _W["params"] = oracle.init_random(N_GAUSS, 0, grid)
    _W["helix"] = oracle.make_helix(50)


def _cpu_one_image(i: int) -> float:
    """The reference bench frame + loss for image i (bench.py:50-58, train.py:136-156), fp64."""
    oracle = _W["oracle"]
    grid = _W["grid"]
    W, t = oracle.sample_pose(np.random.default_rng(1000 + i))
    d = float(np.random.default_rng(3000 + i).uniform(1e4, 2.5e4))
    t0 = time.perf_counter()
    H = oracle.ctf_evaluate(oracle.Ctf(d, d), grid)
    obs = np.zeros((D, D))
    oracle.image_step(_W["params"], W, t, grid, H, obs)
    return time.perf_counter() - t0


def _cpu_sample(i0: int, seconds: float):
    """Worker: images i0, i0+1, ... until `seconds` of measured work (first one is warm-up)."""
    _cpu_one_image(i0)
    done, spent, i = 0, 0.0, i0 + 1
    while spent < seconds:
        spent += _cpu_one_image(i)
        done += 1
        i += 1
    return done, spent


# ---------------------------------------------------------------------------
# The reference itself (cryosplat, pure Python + Numba), installed into
# baseline/_ref by `pip install --no-index --no-build-isolation --no-deps --target
# baseline/_ref <copy of /root/reference/pkg>`.  One step = the
# reference's public train_step on one C2 record (ctf_evaluate + rasterize +
# apply_ctf + loss + apply_ctf + rasterize_backward + AdamState.update,
# train.py:136-191), i.e. the per-image unit of the GPU step.
# ---------------------------------------------------------------------------
REF_DIR = os.path.join(ROOT, "baseline", "_ref")
_R = {}


def reference_available() -> bool:
    if not os.path.isdir(os.path.join(REF_DIR, "cryosplat")):
        return False
    try:
        import numba  # noqa: F401
    except ImportError:
        return False
    return True


def _ref_init():
    """Import the reference and JIT its kernels once (in the parent, before forking)."""
    if _R:
        return
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/cgs_numba_cache")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import cryosplat as rc
    import cryosplat.bench  # noqa: F401  (the stock benchmark frame)

    grid = rc.GridSpec(D, 0.5, PIXEL_A)
    _R.update(rc=rc, grid=grid, mix=rc.init_random(N_GAUSS, 0, grid), cfg=rc.TrainConfig(),
              adam=rc.AdamState(N_GAUSS))
    _ref_one_image(0)  # JIT compilation (cache=True kernels), excluded from every timing


def _ref_one_image(i: int) -> float:
    rc = _R["rc"]
    pose = rc.sample_pose(np.random.default_rng(1000 + i))
    d = float(np.random.default_rng(3000 + i).uniform(1e4, 2.5e4))
    rec = rc.ParticleRecord(image=np.zeros((D, D)), pose=pose, ctf=rc.CtfParams(defocus_u=d, defocus_v=d))
    t0 = time.perf_counter()
    rc.train_step(_R["mix"], rec, _R["cfg"], _R["adam"], lr=1e-3, grid=_R["grid"])
    return time.perf_counter() - t0


def _ref_sample(i0: int, seconds: float):
    _ref_one_image(i0)
    done, spent, i = 0, 0.0, i0 + 1
    while spent < seconds:
        spent += _ref_one_image(i)
        done += 1
        i += 1
    return done, spent


def _pool_rate(init, sample, seconds: float, parent_init=None):
    import multiprocessing as mp

    cores = os.cpu_count() or 1
    if parent_init is not None:
        parent_init()
    ctx = mp.get_context("fork")
    with ctx.Pool(cores, initializer=init) as pool:
        res = pool.starmap(sample, [(100000 + 1000 * k, seconds) for k in range(cores)])
    images = sum(r[0] for r in res)
    wall = max(r[1] for r in res)
    per_img_ms = 1e3 * statistics.median(r[1] / max(r[0], 1) for r in res)
    return images / wall, images, cores, per_img_ms


def cpu_baseline(seconds: float = 12.0):
    """The CPU path on all host cores: the reference itself (baseline/_ref, kind "reference") when
    installed, beside the oracle port (kind "port", the reference's algorithm in fp64 NumPy + C)."""
    v, images, cores, ms = _pool_rate(_cpu_worker_init, _cpu_sample, seconds)
    port = {
        "value": v, "unit": "images/s", "cores": cores, "kind": "port",
        "sample": (f"{images} C2 images (50k Gaussians, 128^2, CTF, fp64 project+bin+forward+CTF+MSE+CTF^T+"
                   f"backward+chain) over {cores} fork workers x ~{seconds:.0f}s; median {ms:.0f} ms/image/core"),
        "cpu_model": _cpu_model(),
    }
    if not reference_available():
        return port
    v, images, cores, ms = _pool_rate(lambda: None, _ref_sample, seconds, parent_init=_ref_init)
    # the reference's own benchmark frame (cryosplat/bench.py:43-103: its mid-training bench
    # mixture, rasterize + CTF + backward, no Adam), one core, median of 5 after a warm-up
    stock = _R["rc"].bench.benchmark_case(N_GAUSS, D, 5, seed=0)
    return {
        "value": v, "unit": "images/s", "cores": cores, "kind": "reference",
        "sample": (f"{images} C2 records through the reference's own train_step (cryosplat from baseline/_ref, "
                   f"Numba kernels, fp64: ctf_evaluate, rasterize, apply_ctf x2, loss, rasterize_backward, Adam) "
                   f"over {cores} fork workers x ~{seconds:.0f}s; median {ms:.0f} ms/image/core"),
        "cpu_model": _cpu_model(),
        "port": port,
        "stock_bench_frame": {"ms_per_image_one_core": 1e3 * stock.median_seconds, "fps_one_core": stock.fps,
                              "what": "cryosplat.bench.benchmark_case(50000, 128, repeats=5): bench.py:43-103"},
    }


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args, rank: int, world: int):
    """The reference arm: the reference's CPU path on all host cores, K timed steps of one image
    per core (cryosplat itself from baseline/_ref when installed, else the oracle port)."""
    if rank != 0:
        return
    import multiprocessing as mp

    cores = os.cpu_count() or 1
    ref = reference_available()
    if ref:
        _ref_init()
        init, one, kind = None, _ref_one_image, "reference"
        what = "cryosplat train_step from baseline/_ref (Numba, fp64), one C2 record per core"
    else:
        init, one, kind = _cpu_worker_init, _cpu_one_image, "port"
        what = "fp64 oracle port (NumPy + C restatement of the reference), one C2 image per core"
    ctx = mp.get_context("fork")
    with ctx.Pool(cores, initializer=init) as pool:
        idx = iter(range(10**7))
        for _ in range(args.warmup):
            pool.map(one, [next(idx) for _ in range(cores)])
        t0 = time.perf_counter()
        for _ in range(args.steps):
            pool.map(one, [next(idx) for _ in range(cores)])
        dt = time.perf_counter() - t0
    value = cores * args.steps / dt
    line = {
        "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD + f" ({what} per step)", "n_gaussians": N_GAUSS, "image_px": D,
                   "images_per_step": cores},
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": cores, "kind": kind,
                         "sample": f"{args.steps} steps x {cores} images: {what}", "cpu_model": _cpu_model()},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
_POLL_SCRIPT = r"""
import json, sys, threading, time
idx, power = int(sys.argv[1]), sys.argv[2] == "1"
names = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
         ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
         ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
         ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
         ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))
import pynvml as nv
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(idx)
mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
stop = threading.Event()
threading.Thread(target=lambda: (sys.stdin.read(), stop.set()), daemon=True).start()
clk, watts, reasons = [], [], set()
print("ready", flush=True)
while not stop.is_set():
    try:
        clk.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
        if power:
            watts.append(nv.nvmlDeviceGetPowerUsage(h) / 1e3)
        m = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        for n, a in names:
            if m & getattr(nv, a, 0):
                reasons.add(n)
    except Exception:
        pass
    time.sleep(0.002)
print(json.dumps({"clk": clk, "watts": watts, "reasons": sorted(reasons), "max": mx}), flush=True)
"""


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled DURING the timed region (the
    recipe's clocks line): a child process polls NVML every 2 ms between start() and stop(),
    so the sampling does not compete with the launching thread for the GIL; optionally board
    power.  Falls back to one nvidia-smi query when NVML is missing."""

    def __init__(self, index: int, power: bool = False):
        self.index, self.power = index, power
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen([sys.executable, "-c", _POLL_SCRIPT, str(self.index), "1" if self.power else "0"],
                                         stdin=subprocess.PIPE, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                         text=True)
            if self.proc.stdout.readline().strip() != "ready":
                raise RuntimeError("sampler did not start")
        except Exception:
            if self.proc is not None:
                self.proc.kill()
            self.proc = None
        return self

    def stop(self):
        res = None
        if self.proc is not None:
            try:
                out, _ = self.proc.communicate(input="", timeout=30)
                res = json.loads(out.strip().splitlines()[-1])
            except Exception:
                self.proc.kill()
                res = None
        if not res or not res["clk"]:  # no NVML: one nvidia-smi query right after the region
            try:
                out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm", "--format=csv,noheader,nounits",
                                      "-i", str(self.index)], capture_output=True, text=True, timeout=10).stdout
                sm, mx = (float(v) for v in out.strip().split(",")[:2])
                return {"sm_mhz": sm, "sm_max_mhz": mx, "reasons": [], "samples": 1, "source": "nvidia-smi after"}
            except Exception:
                return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"], "samples": 0}
        out = {"sm_mhz": statistics.median(res["clk"]), "sm_max_mhz": res["max"], "reasons": res["reasons"],
               "samples": len(res["clk"])}
        if res["watts"]:
            out["power_w_median"] = statistics.median(res["watts"])
            out["power_w_max"] = max(res["watts"])
        return out


def _dataset(rank: int):
    import paper_2508_04929_b200 as cs
    from paper_2508_04929_b200.synth import synthetic_stack

    grid = cs.GridSpec(D, 0.5, PIXEL_A)
    base = rank * DATASET
    poses = [cs.sample_pose(np.random.default_rng(1000 + base + i)) for i in range(DATASET)]
    defocus = [float(np.random.default_rng(3000 + base + i).uniform(1e4, 2.5e4)) for i in range(DATASET)]
    rot = np.stack([p.rotation for p in poses])
    truth = cs.make_phantom("helix", 50, 0)
    obs, ctfs, sigma = synthetic_stack(truth, rot, grid, defocus=defocus, snr=0.1, noise_seed=11 + rank)
    from paper_2508_04929_b200.engine import pose_array

    return grid, obs, pose_array(rot), ctfs


def run_ours(args, rank: int, world: int, local_rank: int):
    import torch

    import paper_2508_04929_b200 as cs
    from paper_2508_04929_b200 import engine
    from paper_2508_04929_b200.optimize import Reconstructor

    if os.environ.get("CGS_BENCH_BACKEND", "nccl") != "nccl":  # test mode: ranks may share a GPU
        local_rank %= torch.cuda.device_count()
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        # CGS_BENCH_BACKEND=gloo: host-side collectives, so several ranks can share one GPU to test
        # the multi-rank bench logic (the numbers are not multi-GPU numbers)
        backend = os.environ.get("CGS_BENCH_BACKEND", "nccl")
        dist.init_process_group(backend, device_id=torch.device("cuda", local_rank) if backend == "nccl" else None)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.cpu_seconds)

    grid, obs, poses, ctfs = _dataset(rank)
    mix = cs.init_random(N_GAUSS, 0, grid)
    # weak: 256 images per GPU; strong: a fixed global batch of 256 split over the ranks
    BATCH = BATCH_PER_GPU if args.scaling == "weak" else GLOBAL_BATCH_STRONG // world
    global_batch = BATCH * world
    # each rank's synthetic particles are its own (rank-seeded), all resident in HBM
    rec = Reconstructor(grid, mix.params, obs, poses, ctfs, batch_size=global_batch, residency="full")
    dev = rec.ctx.device
    nb = DATASET // BATCH
    batches = [np.arange(k * BATCH, (k + 1) * BATCH) for k in range(nb)]
    dev_batches = []
    for b in batches:
        idx = torch.as_tensor(b, device=dev)
        dev_batches.append((rec.obs.index_select(0, idx).contiguous(), rec.poses.index_select(0, idx).contiguous(),
                            rec.ctfs.index_select(0, idx).contiguous()))
    # the dataset's observation spectra (computed once by the Reconstructor): K4 in the Fourier domain
    dev_spectra = [None if rec.obs_spec is None else rec.batch_spectra(b).contiguous() for b in batches]
    # size the tile lists once (one host read per batch shape) with 25% headroom
    pipe = rec.pipeline(BATCH)
    need = max(pipe.measure_items(rec.params, p) for _, p, _ in dev_batches)
    pipe.grow(need)
    # algorithmic work: in-ellipse (image, Gaussian, pixel) pairs of every batch
    splat = engine.prepare(rec.ctx, rec.params, pipe.status)
    pairs = [int(engine.count_pairs(rec.ctx, splat, N_GAUSS, p, rec.gs).sum().item()) for _, p, _ in dev_batches]
    # the pairs K5 evaluates: its walk stops at q < -2 ln(1e-7) (raster_bwd.cu kBwdCut)
    bwd_cut = float(rec.ctx.lib.cgs_bwd_cut_sq())
    bwd_pairs = [int(engine.count_pairs(rec.ctx, splat, N_GAUSS, p, rec.gs, cut_sq=bwd_cut).sum().item())
                 for _, p, _ in dev_batches]
    lr = 1e-3

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident timing (value) ----
    for k in range(args.warmup):
        o, p, c = dev_batches[k % nb]
        rec.step_batch(o, p, c, lr, global_batch=global_batch, obs_spec=dev_spectra[k % nb])
    barrier()
    sampler = ClockSampler(local_rank).start()
    stage = {n: [] for n in ("fwd", "ctf", "bwd", "epi")}
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    step_pairs = step_bwd_pairs = 0
    start.record()
    for k in range(args.steps):
        o, p, c = dev_batches[k % nb]
        ev = {n: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for n in stage}
        rec.step_batch(o, p, c, lr, global_batch=global_batch, events=ev, obs_spec=dev_spectra[k % nb])
        for n in stage:
            stage[n].append(ev[n])
        step_pairs += pairs[k % nb]
        step_bwd_pairs += bwd_pairs[k % nb]
    end.record()
    barrier()
    clocks = sampler.stop()
    ms = start.elapsed_time(end)
    stage_ms = {n: sum(a.elapsed_time(b) for a, b in v) / args.steps for n, v in stage.items()}
    ms_max = ms
    if dist is not None:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t.item())
    value = global_batch * args.steps / (ms_max / 1e3)
    overflow = pipe.overflowed()

    # ---- end-to-end through the public API with pinned host buffers (e2e) ----
    host = [(o.cpu().pin_memory(), p.cpu().pin_memory(), c.cpu().pin_memory()) for o, p, c in dev_batches]
    loss_host = torch.empty(BATCH, dtype=torch.float64).pin_memory()
    for k in range(args.warmup):
        o, p, c = host[k % nb]
        rec.step_host(o, p, c, lr, global_batch=global_batch, loss_out=loss_host)
    barrier()
    start.record()
    for k in range(args.steps):
        o, p, c = host[k % nb]
        rec.step_host(o, p, c, lr, global_batch=global_batch, loss_out=loss_host)
    end.record()
    barrier()
    ms_e2e = start.elapsed_time(end)
    if dist is not None:
        t = torch.tensor([ms_e2e], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
    e2e = global_batch * args.steps / (ms_e2e / 1e3)

    # ---- sustained: the device-resident step for a few seconds (clocks and power under load) ----
    sustained = None
    if args.sustained_seconds > 0:
        n_sus = max(args.steps, int(args.sustained_seconds / max(ms_max / args.steps / 1e3, 1e-6)))
        psampler = ClockSampler(local_rank, power=True).start()
        barrier()
        start.record()
        for k in range(n_sus):
            o, p, c = dev_batches[k % nb]
            rec.step_batch(o, p, c, lr, global_batch=global_batch, obs_spec=dev_spectra[k % nb])
        end.record()
        barrier()
        pclk = psampler.stop()
        ms_sus = start.elapsed_time(end)
        if dist is not None:
            t = torch.tensor([ms_sus], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_sus = float(t.item())
        sustained = {"seconds": ms_sus / 1e3, "steps": n_sus, "value": global_batch * n_sus / (ms_sus / 1e3),
                     "unit": "images/s", "clocks": pclk}
    h2d = BATCH * D * D * 4 + BATCH * 12 * 8 + BATCH * 8 * 8
    d2h = BATCH * 8

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return
    f_mhz = clocks.get("sm_mhz") or 1965.0
    pairs_per_launch = step_pairs / args.steps
    bwd_pairs_per_launch = step_bwd_pairs / args.steps
    bwd_achieved = bwd_pairs_per_launch / (stage_ms["bwd"] / 1e3) / 1e9
    bwd_peak = 8.0 * 148 * f_mhz * 1e6 / 1e9            # 128 lanes/clk/SM / 16 issue slots per pair
    step_peak = 148 * f_mhz * 1e6 / 0.164 / 1e9          # 0.164 SM-clk per pair fwd+bwd
    step_achieved = pairs_per_launch / (ms / args.steps / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "raster_bwd_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("dram_bytes_per_launch")
        except (OSError, ValueError):
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f32 (fp64 binning bbox, fp64 Adam master params)", "data": "synthetic",
        "config": {"workload": WORKLOAD if args.scaling == "weak" else WORKLOAD_STRONG, "n_gaussians": N_GAUSS,
                   "image_px": D, "batch_per_gpu": BATCH,
                   "global_batch": global_batch, "parallelism": f"dp{world}", "ctf": True,
                   "exchange": (None if world == 1 else args.exchange),
                   "l2": (f"inputs larger than L2: {DATASET}-particle dataset cycled ("
                          + (f"observation spectra {DATASET * D * (D // 2 + 1) * 8 >> 20} MiB"
                             if rec.obs_spec is not None else f"{DATASET * D * D * 4 >> 20} MiB") + ")")},
        "e2e": {"value": e2e, "unit": "images/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": (rec.pipeline(BATCH).own_launches_per_step(ctf=True, obs_spectrum=rec.obs_spec is not None)
                         * args.steps + (args.steps if world > 1 else 0)),
        "roofline": {"bound": "fp32_sfu_issue", "kernel": "raster_bwd", "achieved": bwd_achieved, "peak": bwd_peak,
                     "unit": "Gpair/s", "frac": bwd_achieved / bwd_peak, "traffic": traffic,
                     "peak_basis": (f"SURVEY.md 8(d): 1 EX2 + 15 FP32 per in-ellipse pair, 128 FP32 lanes/clk/SM "
                                    f"x 148 SMs at the sampled {f_mhz:.0f} MHz"),
                     "units_per_launch": bwd_pairs_per_launch,
                     "units": (f"(image, Gaussian, pixel) pairs K5 evaluates: q < {bwd_cut:.3f} (e >= 1e-7 of the "
                               f"peak; the reference's q < 42.25 pairs are {pairs_per_launch:.4g} per launch)"),
                     "launch_ms": stage_ms["bwd"],
                     # the same launch counted in the reference's q < 6.5^2 pairs (round 1's unit)
                     "frac_reference_pairs": pairs_per_launch / (stage_ms["bwd"] / 1e3) / 1e9 / bwd_peak},
        # the forward stage (K0 + weight bound + K3 render) against SURVEY.md 8(d)'s forward cost, 1 EX2 + 4 FP32
        # per in-ellipse pair: the SFU bound, 16 EX2 lanes/clk/SM (measured 15.6,
        # profiles/measured_fp32_sfu_peaks_r01.json).  K3 walks rows by a two-multiply recurrence instead of an
        # EX2 per pixel; what bounds it is the shared-memory atomic unit and issue
        "roofline_fwd": {"bound": "sfu", "kernel": "raster_fwd_atomic (+ weight bound)",
                         "achieved": pairs_per_launch / (stage_ms["fwd"] / 1e3) / 1e9,
                         "peak": 16.0 * 148 * f_mhz * 1e6 / 1e9, "unit": "Gpair/s",
                         "frac": (pairs_per_launch / (stage_ms["fwd"] / 1e3)) / (16.0 * 148 * f_mhz * 1e6),
                         "units": "the reference's in-ellipse (image, Gaussian, pixel) pairs, q < 6.5^2",
                         "launch_ms": stage_ms["fwd"]},
        "roofline_step": {"achieved": step_achieved, "peak": step_peak, "unit": "Gpair/s",
                          "frac": step_achieved / step_peak,
                          "peak_basis": "0.164 SM-clk per in-ellipse pair (fwd+bwd issue), SURVEY.md 8(d)"},
        "stage_ms": stage_ms,
        "clocks": clocks,
        "sustained": sustained,
        "cpu_baseline": cpu,
    }
    if overflow:
        line["warning"] = "tile-list overflow during timing"
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: 256 images per GPU (default); strong: global batch 256 split over the GPUs")
    ap.add_argument("--sustained-seconds", type=float, default=3.0,
                    help="after the timed region, run the device-resident step this long and report it as "
                         "'sustained' (clocks and power under load); 0 disables")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "peer"],
                    help="multi-GPU exchange: NCCL all-reduce (default) or the fused peer-memory kernel "
                         "(cgs_peer_epilogue_adam, CGS_DP_PEER=1)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.exchange == "peer":
        os.environ["CGS_DP_PEER"] = "1"
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
