"""Generate the golden fixtures in tests/golden/ by RUNNING THE REFERENCE.

Run in the build container only (it imports the reference package from
/root/reference, which does not exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

The fixtures pin the CPU oracle (oracle/cgs_oracle.py): tests/test_oracle_golden.py
checks the oracle against them, and the GPU parity tests check the CUDA path
against the oracle.  Every input below is generated with the reference's own
seeded generators (init_random, sample_pose, make_phantom, random_mixture of
the reference conftest), so the oracle can regenerate the inputs bit-exactly.
"""

from __future__ import annotations

import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import cryosplat as cs  # noqa: E402
from cryosplat import _kernels  # noqa: E402
from cryosplat.gmm import PARAMS_PER_GAUSSIAN, inverse_activate  # noqa: E402
from cryosplat.simulate import sample_pose  # noqa: E402
from cryosplat.splat import CLAMP_EVENTS, _Projection  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def random_mixture(rng, n, grid, scale_px=(1.0, 3.0), mean_range=0.2, amp_range=(0.3, 2.0)):
    """Same draws as the reference tests' conftest.random_mixture (conftest.py:48-62)."""
    params = np.zeros((n, PARAMS_PER_GAUSSIAN))
    params[:, 0:3] = rng.uniform(-mean_range, mean_range, (n, 3))
    params[:, 3:6] = inverse_activate(rng.uniform(*scale_px, (n, 3)) * grid.pixel_width)
    params[:, 6:10] = rng.standard_normal((n, 4))
    params[:, 10] = inverse_activate(rng.uniform(*amp_range, n))
    return cs.GaussianMixture(params)


def random_pose(rng, translation_range=0.0):
    """conftest.random_pose (conftest.py:65-67)."""
    t = rng.uniform(-translation_range, translation_range, 2) if translation_range else np.zeros(2)
    return cs.Pose.from_quaternion(rng.standard_normal(4), t)


def observed_stack(truth, poses, grid, ctfs, snr, noise_seed0):
    clean = []
    for pose, ctf in zip(poses, ctfs):
        img = cs.rasterize(truth, pose, grid)
        if ctf is not None:
            img = cs.apply_ctf(img, ctf)
        clean.append(img.pixels)
    clean = np.stack(clean)
    sigma = float(np.sqrt(clean.var() / snr))
    obs = np.stack([
        clean[i] + np.random.default_rng(noise_seed0 + i).normal(0.0, sigma, clean[i].shape)
        for i in range(len(poses))
    ]).astype(np.float32)
    return obs


def per_image(mix, pose, grid, H, obs, tile=16):
    proj = _Projection(mix, pose, grid)
    ntx = -(-grid.size // tile)
    ids, starts = _kernels.build_tile_work(proj.bbox, tile, ntx, ntx)
    rendered = cs.rasterize(mix, pose, grid).pixels
    model = rendered if H is None else cs.apply_ctf(cs.RenderedImage(grid, rendered), H).pixels
    loss = cs.loss_mse(model, obs)
    d = grid.size
    dL = (2.0 / (d * d)) * (model - obs)
    up = dL if H is None else cs.apply_ctf(cs.RenderedImage(grid, dL), H).pixels
    sums = np.zeros((len(mix), 6))
    _kernels.backward_pixels(up, proj.mean2, proj.prec, proj.bbox, grid.pixel_width,
                             grid.origin_index, 42.25, float(np.exp(-21.125)), sums)
    grads = cs.rasterize_backward(mix, pose, grid, up)
    return dict(bbox=proj.bbox, ids=ids.astype(np.int32), starts=starts, rendered=rendered,
                model=model, loss=loss, upstream=up, sums=sums, grads=grads, n_clamped=proj.n_clamped)


def stack_case(name, n, D, B, with_ctf, seed_obs=11, light=False):
    grid = cs.GridSpec(D, 0.5, 1.5)
    mix = cs.init_random(n, 0, grid)
    poses = [sample_pose(np.random.default_rng(1000 + i)) for i in range(B)]
    ctfs = []
    for i in range(B):
        if with_ctf:
            d = float(np.random.default_rng(3000 + i).uniform(1e4, 2.5e4))
            ctfs.append(cs.CtfParams(defocus_u=d, defocus_v=d))
        else:
            ctfs.append(None)
    truth = cs.make_phantom("helix", 50, 0)
    obs = observed_stack(truth, poses, grid, ctfs, 0.1, seed_obs)
    out = {"D": D, "n": n, "B": B}
    rendered, models, ups, sums, losses, grads = [], [], [], [], [], []
    ids_all, starts_all, bbox_all, clamped = [], [], [], []
    for i in range(B):
        H = None if ctfs[i] is None else cs.ctf_evaluate(ctfs[i], grid)
        r = per_image(mix, poses[i], grid, H, obs[i])
        rendered.append(r["rendered"]); models.append(r["model"]); ups.append(r["upstream"])
        sums.append(r["sums"]); losses.append(r["loss"]); grads.append(r["grads"])
        ids_all.append(r["ids"]); starts_all.append(r["starts"]); bbox_all.append(r["bbox"])
        clamped.append(r["n_clamped"])
    out["observed"] = obs
    out["rendered"] = np.stack(rendered)
    out["model"] = np.stack(models)
    out["upstream"] = np.stack(ups)
    out["losses"] = np.array(losses)
    out["grads_mean"] = np.mean(grads, axis=0)
    if not light:
        out["grads_first"] = grads[0]
        out["sums_first"] = sums[0]
    out["bbox"] = np.stack(bbox_all).astype(np.int32)
    out["tile_ids"] = np.concatenate(ids_all)
    out["tile_starts"] = np.stack(starts_all)
    out["n_clamped"] = np.array(clamped)
    out["defocus"] = np.array([np.nan if c is None else c.defocus_u for c in ctfs])
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    print(name, {k: getattr(v, "shape", v) for k, v in out.items()})


def kat_cases():
    out = {}
    grid64 = cs.GridSpec(64, 0.5, 3.0)
    # test_splat.py:298-304 dense-oracle mixture, plus tile-size variants (:317-324)
    rng = np.random.default_rng(6)
    mix = random_mixture(rng, 64, grid64)
    pose = random_pose(rng, translation_range=0.03)
    out["dense_params"] = mix.params
    out["dense_W"] = pose.rotation
    out["dense_t"] = pose.translation
    for tile in (8, 16, 32):
        out[f"dense_render_tile{tile}"] = cs.rasterize(mix, pose, grid64, tile_size=tile).pixels
        proj = _Projection(mix, pose, grid64)
        ntx = -(-64 // tile)
        ids, starts = _kernels.build_tile_work(proj.bbox, tile, ntx, ntx)
        out[f"dense_ids_tile{tile}"] = ids
        out[f"dense_starts_tile{tile}"] = starts
    up = np.random.default_rng(77).standard_normal((64, 64))
    out["dense_upstream"] = up
    out["dense_grads"] = cs.rasterize_backward(mix, pose, grid64, up)
    # eigenvalue floor (test_splat.py:347-358)
    params = np.zeros((1, PARAMS_PER_GAUSSIAN))
    params[0, 3:6] = inverse_activate(1e-6)
    params[0, 6] = 1.0
    params[0, 10] = inverse_activate(1.0)
    CLAMP_EVENTS.reset()
    out["clamp_render"] = cs.rasterize(cs.GaussianMixture(params), cs.Pose.identity(), grid64).pixels
    out["clamp_count"] = np.array(CLAMP_EVENTS.count)
    # anisotropic clamped Gaussians under random poses (needle-like)
    rng = np.random.default_rng(21)
    p = np.zeros((16, PARAMS_PER_GAUSSIAN))
    p[:, 0:3] = rng.uniform(-0.2, 0.2, (16, 3))
    p[:, 3] = inverse_activate(rng.uniform(2, 4, 16) * grid64.pixel_width)
    p[:, 4] = inverse_activate(rng.uniform(0.01, 0.05, 16) * grid64.pixel_width)
    p[:, 5] = inverse_activate(rng.uniform(0.01, 0.05, 16) * grid64.pixel_width)
    p[:, 6:10] = rng.standard_normal((16, 4))
    p[:, 10] = inverse_activate(rng.uniform(0.5, 1.5, 16))
    pose = cs.Pose(np.eye(3))
    CLAMP_EVENTS.reset()
    out["needle_params"] = p
    out["needle_render"] = cs.rasterize(cs.GaussianMixture(p), pose, grid64).pixels
    out["needle_clamp_count"] = np.array(CLAMP_EVENTS.count)
    up = np.random.default_rng(78).standard_normal((64, 64))
    out["needle_upstream"] = up
    out["needle_grads"] = cs.rasterize_backward(cs.GaussianMixture(p), pose, grid64, up)
    # softplus / Adam KATs (test_gmm.py:118-122, test_train.py:71-79)
    out["inv_act_5e-5"] = np.array(inverse_activate(5e-5))
    st = cs.AdamState(1)
    prm = np.zeros((1, 11))
    rng = np.random.default_rng(3)
    g1 = rng.standard_normal((1, 11))
    g2 = rng.standard_normal((1, 11))
    st.update(prm, g1, lr=0.01, config=cs.TrainConfig())
    st.update(prm, g2, lr=0.01, config=cs.TrainConfig())
    out["adam_g1"], out["adam_g2"], out["adam_params"] = g1, g2, prm.copy()
    np.savez_compressed(os.path.join(OUT, "kat.npz"), **out)
    print("kat", sorted(out))


def ctf_cases():
    out = {}
    specs = [
        (64, cs.CtfParams(defocus_u=15000.0, defocus_v=15000.0)),
        (64, cs.CtfParams(defocus_u=18000.0, defocus_v=14000.0, astigmatism_angle=0.7)),
        (33, cs.CtfParams(defocus_u=21000.0, defocus_v=12000.0, astigmatism_angle=2.1,
                          phase_shift=0.3, b_factor=40.0, amplitude_contrast=0.07)),
        (128, cs.CtfParams(defocus_u=24000.0, defocus_v=19000.0, astigmatism_angle=1.1,
                           voltage=200.0, spherical_aberration=2.0)),
    ]
    rng = np.random.default_rng(5)
    for i, (D, p) in enumerate(specs):
        grid = cs.GridSpec(D, 0.5, 1.5)
        H = cs.ctf_evaluate(p, grid)
        img = rng.standard_normal((D, D))
        out[f"ctf{i}_D"] = np.array(D)
        out[f"ctf{i}_params"] = np.array([p.defocus_u, p.defocus_v, p.astigmatism_angle, p.voltage,
                                          p.spherical_aberration, p.amplitude_contrast,
                                          p.phase_shift, p.b_factor])
        out[f"ctf{i}_H"] = H
        out[f"ctf{i}_img"] = img
        out[f"ctf{i}_applied"] = cs.apply_ctf(cs.RenderedImage(grid, img), H).pixels
    out["lambda_300"] = np.array(cs.electron_wavelength(300.0))
    np.savez_compressed(os.path.join(OUT, "ctf.npz"), **out)
    print("ctf", sorted(out))


def train_case():
    """A tiny deterministic train() run (train.py:194-264) with B = 1 semantics."""
    import tempfile

    grid = cs.GridSpec(32, 0.5, 3.0)
    rng = np.random.default_rng(7)
    truth = random_mixture(rng, 6, grid, amp_range=(0.5, 1.5))
    records = []
    for _ in range(3):
        pose = random_pose(rng)
        ctf = cs.CtfParams(defocus_u=15000.0, defocus_v=15000.0)
        img = cs.apply_ctf(cs.rasterize(truth, pose, grid), ctf).pixels
        records.append(cs.ParticleRecord(image=img, pose=pose, ctf=ctf))
    ds = cs.Dataset(records=records, grid=grid)
    with tempfile.TemporaryDirectory() as d:
        mix, losses = cs.train(ds, cs.TrainConfig(epochs=3, seed=0), n_gaussians=8, out_dir=d)
        trace = open(os.path.join(d, "loss_trace.txt")).read()
    out = {
        "images": np.stack([r.image for r in records]),
        "rotations": np.stack([r.pose.rotation for r in records]),
        "final_params": mix.params,
        "losses": np.stack(losses),
        "trace": np.array(trace),
    }
    np.savez_compressed(os.path.join(OUT, "train_small.npz"), **out)
    print("train_small", {k: getattr(v, "shape", v) for k, v in out.items()})


def simulate_cases():
    """cryosplat.simulate (simulate.py:204-267): two specs covering DefocusRange and
    CTF-list sampling, translations (sub-pixel and integer), pose jitter, noise."""
    from cryosplat.simulate import DefocusRange, NoiseModel, SimSpec, make_phantom, simulate

    out = {}
    grid = cs.GridSpec(64, 0.5, 1.5)
    specs = {
        "a": SimSpec(truth=make_phantom("helix", 12, 0), num_particles=5, grid=grid,
                     ctf_distribution=DefocusRange(1e4, 2.5e4), noise=NoiseModel(snr=0.5, seed=7), seed=3),
        "b": SimSpec(truth=make_phantom("blob-cluster", 10, 1), num_particles=4, grid=grid,
                     ctf_distribution=[cs.CtfParams(12000.0, 15000.0, 0.7), cs.CtfParams(20000.0, 18000.0, -0.3,
                                                                                          phase_shift=0.4)],
                     noise=NoiseModel(snr=float("inf")), translation_range=3.0, pose_jitter_deg=2.0, seed=11),
        "c": SimSpec(truth=make_phantom("two-lobe", 8, 2), num_particles=3, grid=grid,
                     ctf_distribution=DefocusRange(1.5e4, 2e4), noise=NoiseModel(snr=2.0, seed=1),
                     translation_range=2.0, integer_translations=True, seed=5),
    }
    for k, spec in specs.items():
        res = simulate(spec)
        out[f"{k}_images"] = np.stack([r.image for r in res.records])
        out[f"{k}_quaternions"] = res.quaternions
        out[f"{k}_rotations"] = np.stack([r.pose.rotation for r in res.records])
        out[f"{k}_translations"] = np.stack([r.translation for r in res.records])
        out[f"{k}_defocus"] = np.array([[r.ctf.defocus_u, r.ctf.defocus_v, r.ctf.astigmatism_angle,
                                         r.ctf.phase_shift] for r in res.records])
        out[f"{k}_sigma"] = np.array(res.noise_sigma)
    np.savez_compressed(os.path.join(OUT, "simulate.npz"), **out)
    print("simulate", sorted(out))


def io_cases():
    """Files written by the reference's io.py (MRC stack + volume, metadata table)."""
    import tempfile

    from cryosplat import io as rio

    rng = np.random.default_rng(21)
    stack = rng.standard_normal((3, 16, 16)).astype(np.float32)
    vol = rng.standard_normal((8, 8, 8)).astype(np.float32)
    quats = rng.standard_normal((3, 4))
    trans = rng.uniform(-2, 2, (3, 2))
    ctfs = [cs.CtfParams(12000.0 + 1000 * i, 15000.0 - 500 * i, 0.1 * i, phase_shift=0.05 * i, b_factor=10.0 * i)
            for i in range(3)]
    out = {"stack": stack, "volume": vol, "quats": quats, "trans": trans,
           "ctf_rows": np.array([[c.defocus_u, c.defocus_v, c.astigmatism_angle, c.voltage, c.spherical_aberration,
                                  c.amplitude_contrast, c.phase_shift, c.b_factor] for c in ctfs])}
    with tempfile.TemporaryDirectory() as d:
        rio.write_mrc(os.path.join(d, "s.mrcs"), stack, 1.37, volume=False)
        rio.write_mrc(os.path.join(d, "v.mrc"), vol, 2.5)
        rio.write_meta(os.path.join(d, "m.txt"), quats, trans, ctfs)
        for k, f in (("stack_bytes", "s.mrcs"), ("volume_bytes", "v.mrc"), ("meta_bytes", "m.txt")):
            out[k] = np.frombuffer(open(os.path.join(d, f), "rb").read(), dtype=np.uint8)
    np.savez_compressed(os.path.join(OUT, "io.npz"), **out)
    print("io", sorted(out))


def evaluate_cases():
    """evaluate.voxelize and fsc (evaluate.py:76-179) on small mixtures."""
    from cryosplat.evaluate import fsc, fsc_table, voxelize

    grid = cs.GridSpec(32, 0.5, 2.0)
    rng = np.random.default_rng(5)
    a = random_mixture(rng, 12, grid, scale_px=(0.6, 2.5), mean_range=0.35)
    b = cs.GaussianMixture(a.params + np.concatenate([rng.normal(0, 0.01, (12, 3)), rng.normal(0, 0.1, (12, 8))], 1))
    va, vb = voxelize(a, grid), voxelize(b, grid)
    c = fsc(va, vb)
    out = {"a_params": a.params, "b_params": b.params, "va": va.voxels, "vb": vb.voxels,
           "corr": c.correlations, "res": np.array([c.resolution_0143 or np.nan, c.resolution_05 or np.nan]),
           "table": np.array(fsc_table(c))}
    np.savez_compressed(os.path.join(OUT, "evaluate.npz"), **out)
    print("evaluate", sorted(out), c.resolution_0143, c.resolution_05)


def _train_records(rng, truth, grid, k, scale_of=None):
    records = []
    for i in range(k):
        pose = random_pose(rng)
        ctf = cs.CtfParams(defocus_u=15000.0, defocus_v=15000.0)
        img = cs.apply_ctf(cs.rasterize(truth, pose, grid), ctf).pixels
        if scale_of is not None:
            img = img * scale_of(i)
        records.append(cs.ParticleRecord(image=img, pose=pose, ctf=ctf))
    return records


def train_behaviour_cases():
    """train() behaviours beyond the loss values (train.py:194-264), run on the reference:
    the per-epoch CGS1 checkpoint files (gmm.py:259-265) and loss_trace.txt of the
    train_small run; an isotropic-mode run (train.py:157-159); the divergence guard on a
    non-finite loss and on 1e3 x the epoch-0 median (train.py:238-251), as the raised
    DivergenceError's (epoch, step, record_index) and message."""
    import tempfile

    from cryosplat.errors import DivergenceError

    out = {}
    grid = cs.GridSpec(32, 0.5, 3.0)
    rng = np.random.default_rng(7)
    truth = random_mixture(rng, 6, grid, amp_range=(0.5, 1.5))
    records = _train_records(rng, truth, grid, 3)
    with tempfile.TemporaryDirectory() as d:
        cs.train(cs.Dataset(records=records, grid=grid), cs.TrainConfig(epochs=3, seed=0), n_gaussians=8,
                 out_dir=d)
        for e in range(3):
            out[f"ckpt_e{e}"] = np.frombuffer(open(os.path.join(d, f"checkpoint_epoch_{e}.cgs"), "rb").read(),
                                              np.uint8)
        out["trace"] = np.array(open(os.path.join(d, "loss_trace.txt")).read())
    # isotropic mode: one shared raw scale per Gaussian
    rng = np.random.default_rng(17)
    truth = random_mixture(rng, 6, grid, amp_range=(0.5, 1.5))
    records = _train_records(rng, truth, grid, 4)
    out["iso_images"] = np.stack([r.image for r in records])
    out["iso_rotations"] = np.stack([r.pose.rotation for r in records])
    mix, losses = cs.train(cs.Dataset(records=records, grid=grid),
                           cs.TrainConfig(epochs=2, seed=3, mode="isotropic"), n_gaussians=10)
    out["iso_losses"] = np.stack(losses)
    out["iso_final_params"] = mix.params
    # divergence: one record 1e3 x brighter than the others (loss ~1e6 x)
    rng = np.random.default_rng(27)
    truth = random_mixture(rng, 6, grid, amp_range=(0.5, 1.5))
    records = _train_records(rng, truth, grid, 5, scale_of=lambda i: 1e3 if i == 2 else 1.0)
    out["big_images"] = np.stack([r.image for r in records])
    out["big_rotations"] = np.stack([r.pose.rotation for r in records])
    for seed in range(20):
        try:
            cs.train(cs.Dataset(records=records, grid=grid), cs.TrainConfig(epochs=2, seed=seed), n_gaussians=8)
        except DivergenceError as e:
            if e.step > 0:
                out["big_seed"] = np.array(seed)
                out["big_raise"] = np.array([e.epoch, e.step, e.record_index])
                out["big_message"] = np.array(str(e))
                break
    assert "big_raise" in out
    # non-finite loss: an initial mixture whose amplitude overflows the loss
    init = cs.init_random(8, 0, grid)
    init.params[3, 10] = 1e300
    out["nan_initial"] = init.params.copy()
    try:
        cs.train(cs.Dataset(records=records[:3], grid=grid), cs.TrainConfig(epochs=1, seed=4), n_gaussians=8,
                 initial=init)
        raise AssertionError("expected DivergenceError")
    except DivergenceError as e:
        out["nan_raise"] = np.array([e.epoch, e.step, e.record_index])
        out["nan_message"] = np.array(str(e))
    np.savez_compressed(os.path.join(OUT, "train_behaviour.npz"), **out)
    print("train_behaviour", {k: getattr(v, "shape", v) for k, v in out.items()})


if __name__ == "__main__" and len(sys.argv) > 1:
    for name in sys.argv[1:]:
        globals()[name]()
    sys.exit(0)

if __name__ == "__main__":
    stack_case("c1_step", 5000, 64, 4, with_ctf=False)
    stack_case("c2_slice", 50000, 128, 2, with_ctf=True, light=True)
    kat_cases()
    ctf_cases()
    train_case()
    train_behaviour_cases()
