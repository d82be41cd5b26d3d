"""CPU-only checks: the C-ABI library loads and exports every declared symbol,
host-side logic (parameter model, checkpoints, poses, configs) matches the
reference, and the product path refuses to run without a GPU (no fallback)."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT, load_golden

import paper_2508_04929_b200 as cs
from paper_2508_04929_b200 import _lib

HEADER = os.path.join(ROOT, "include", "cgs_b200.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cgs_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = _declared()
    assert len(names) >= 25
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.PROTOTYPES, f"{name} missing from the ctypes prototypes"
    assert set(_lib.PROTOTYPES) == set(names)


def test_host_only_entry_points():
    lib = _lib.load()
    assert lib.cgs_version().decode().startswith("cgs_b200")
    assert lib.cgs_error_string(1).decode() == "invalid argument"
    assert lib.cgs_bin_segments(5000) == 3
    assert lib.cgs_bin_tiles(128, 16) == 64
    assert lib.cgs_bin_tiles(33, 16) == 9
    assert lib.cgs_bwd_groups(256, 16) == 16
    assert lib.cgs_fft_spectrum_elems(128, 2) == 2 * 128 * 65
    assert lib.cgs_scan_workspace_bytes(4096) >= 8


def test_invalid_arguments_are_rejected_without_touching_the_device():
    lib = _lib.load()
    g = _lib.grid_struct(64, 0.5, 1.5)
    assert lib.cgs_prepare(None, 0, None, None, None) == 1
    assert lib.cgs_raster_fwd(None, 10, None, 1, g, 12, None, None, 0, None, 0, None) == 1
    assert lib.cgs_bin_count_bbox(None, 10, 1, 64, 16, None, None, None) == 1
    # K6 reads the accumulator as float pairs: a 4-byte-aligned pointer is refused up front
    assert lib.cgs_epilogue_grads(0x1004, 1, 10, 0x2000, 0, 1.0, 0x3000, None) == 1
    assert lib.cgs_epilogue_adam(0x1004, 1, 10, 0x2000, 0x3000, 0x4000, 0, 1.0, 1e-3, 0.9, 0.999, 1e-8,
                                 0.1, 0.001, None, None) == 1


def test_product_path_fails_loudly_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    mix = cs.init_random(10, 0, cs.GridSpec(32))
    with pytest.raises(cs.CudaUnavailableError):
        cs.rasterize(mix, cs.Pose.identity(), cs.GridSpec(32))
    with pytest.raises(cs.CudaUnavailableError):
        cs.AdamState(10)


def test_parameter_model_matches_reference_and_oracle(oracle):
    grid = cs.GridSpec(64, 0.5, 1.5)
    mix = cs.init_random(5000, 0, grid)
    assert np.array_equal(mix.params, oracle.init_random(5000, 0, oracle.Grid(64, 0.5, 1.5)))
    assert cs.inverse_activate(5e-5) == pytest.approx(-9.903462552431961, rel=1e-12)
    x = np.linspace(-50, 50, 1001)
    np.testing.assert_array_equal(cs.activate(x), oracle.activate(x))
    np.testing.assert_array_equal(cs.mixture.activate_derivative(x), oracle.activate_derivative(x))
    q = np.random.default_rng(0).standard_normal((20, 4))
    np.testing.assert_allclose(cs.mixture.quaternion_to_matrix(cs.mixture.normalize_quaternion(q)),
                               oracle.quaternion_to_matrix(oracle.normalize_quaternion(q)), rtol=0, atol=1e-15)
    with pytest.raises(cs.DegenerateRotationError):
        cs.mixture.normalize_quaternion(np.zeros(4))
    helix = cs.make_phantom("helix", 50, 0)
    np.testing.assert_array_equal(helix.params, oracle.make_helix(50))
    for kind in ("two-lobe", "blob-cluster"):
        assert cs.make_phantom(kind, 40, 3).params.shape == (40, 11)
    with pytest.raises(ValueError):
        cs.make_phantom("cube", 4)


def test_checkpoint_round_trip(tmp_path):
    mix = cs.init_random(17, 3, cs.GridSpec(32), mode="isotropic")
    path = tmp_path / "a.cgs"
    cs.save_checkpoint(mix, path)
    back = cs.load_checkpoint(path)
    assert back.mode == "isotropic" and np.array_equal(back.params, mix.params)
    blob = path.read_bytes()
    assert blob[:4] == b"CGS1" and len(blob) == 13 + 17 * 11 * 8
    (tmp_path / "bad.cgs").write_bytes(b"XXXX" + blob[4:])
    with pytest.raises(cs.DataError):
        cs.load_checkpoint(tmp_path / "bad.cgs")
    (tmp_path / "short.cgs").write_bytes(blob[:-8])
    with pytest.raises(cs.DataError):
        cs.load_checkpoint(tmp_path / "short.cgs")


def test_pose_and_config_validation():
    with pytest.raises(ValueError):
        cs.Pose(np.eye(3) * 1.1)
    with pytest.raises(ValueError):
        cs.Pose(-np.eye(3))
    rng = np.random.default_rng(0)
    p = cs.sample_pose(rng)
    assert np.allclose(p.rotation.T @ p.rotation, np.eye(3), atol=1e-12)
    assert cs.TrainConfig(batch_size=4).batch_size == 4
    with pytest.raises(ValueError):
        cs.TrainConfig(batch_size=0)
    with pytest.raises(ValueError):
        cs.TrainConfig(epochs=0)
    assert cs.TrainConfig(learning_rate=1e-3, decay_gamma=0.1).epoch_lr(2) == pytest.approx(1e-5)
    from paper_2508_04929_b200.train import half_config

    assert half_config(cs.TrainConfig(seed=7), "odd").seed == 8
    assert cs.electron_wavelength(300.0) == pytest.approx(float(load_golden("ctf")["lambda_300"]), rel=1e-15)


def test_reference_module_paths_exist():
    from paper_2508_04929_b200 import errors, gmm, optics, splat, train  # noqa: F401
    from paper_2508_04929_b200.gmm import PARAMS_PER_GAUSSIAN, inverse_activate  # noqa: F401
    from paper_2508_04929_b200.splat import CLAMP_EVENTS  # noqa: F401

    assert PARAMS_PER_GAUSSIAN == 11


def test_view_transform_and_projection_scalar_forms():
    g = cs.GaussianParams(mean=np.array([0.1, 0.0, 0.0]), raw_scale=cs.inverse_activate(np.array([0.02] * 3)),
                          quaternion=np.array([1.0, 0, 0, 0]), raw_amplitude=0.0)
    c, s = np.cos(np.pi / 2), np.sin(np.pi / 2)
    pose = cs.Pose(np.array([[c, -s, 0], [s, c, 0], [0, 0, 1.0]]), np.array([0.05, 0.0]))
    out = cs.view_transform(g, pose)
    assert np.allclose(out.mean3, [0.05, 0.1, 0.0], atol=1e-15)
    sg = cs.orthographic_project(cs.CameraSpaceGaussian(np.zeros(3), 1e-4 * np.eye(3)))
    assert float(sg.density(np.zeros(2))) == pytest.approx(1.0 / (2 * np.pi * 1e-4), rel=1e-12)
    with pytest.raises(cs.DegenerateSplatError):
        cs.orthographic_project(cs.CameraSpaceGaussian(np.zeros(3), np.diag([1.0, -1.0, 1.0])))


def _simulate_specs():
    import math

    from paper_2508_04929_b200 import synth

    grid = cs.GridSpec(64, 0.5, 1.5)
    return {
        "a": synth.SimSpec(truth=synth.make_phantom("helix", 12, 0), num_particles=5, grid=grid,
                           ctf_distribution=synth.DefocusRange(1e4, 2.5e4), noise=synth.NoiseModel(snr=0.5, seed=7),
                           seed=3),
        "b": synth.SimSpec(truth=synth.make_phantom("blob-cluster", 10, 1), num_particles=4, grid=grid,
                           ctf_distribution=[cs.CtfParams(12000.0, 15000.0, 0.7),
                                             cs.CtfParams(20000.0, 18000.0, -0.3, phase_shift=0.4)],
                           noise=synth.NoiseModel(snr=math.inf), translation_range=3.0, pose_jitter_deg=2.0, seed=11),
        "c": synth.SimSpec(truth=synth.make_phantom("two-lobe", 8, 2), num_particles=3, grid=grid,
                           ctf_distribution=synth.DefocusRange(1.5e4, 2e4), noise=synth.NoiseModel(snr=2.0, seed=1),
                           translation_range=2.0, integer_translations=True, seed=5),
    }


def test_simulate_host_draws_match_reference():
    """Per-particle pose / CTF / translation / jitter draws of simulate (simulate.py:224-239)
    are the reference's, bit for bit (tests/golden/simulate.npz from the reference itself)."""
    from paper_2508_04929_b200 import synth

    g = load_golden("simulate")
    for k, spec in _simulate_specs().items():
        true_q, rec_q, ctfs, trans = synth._draws(spec)
        assert np.array_equal(rec_q, g[f"{k}_quaternions"])
        assert np.array_equal(trans, g[f"{k}_translations"])
        d = np.array([[c.defocus_u, c.defocus_v, c.astigmatism_angle, c.phase_shift] for c in ctfs])
        assert np.array_equal(d, g[f"{k}_defocus"])
        rot = np.stack([cs.Pose.from_quaternion(q).rotation for q in rec_q])
        np.testing.assert_allclose(rot, g[f"{k}_rotations"], rtol=0, atol=1e-15)


def test_io_files_match_reference_bytes(tmp_path):
    """MRC stack / volume and the metadata table are written byte-identically to the
    reference's io.py, and the reference's files read back exactly (tests/golden/io.npz)."""
    from paper_2508_04929_b200 import io as cio

    g = load_golden("io")
    ctfs = [cs.CtfParams(*row) for row in g["ctf_rows"]]
    cio.write_mrc(tmp_path / "s.mrcs", g["stack"], 1.37, volume=False)
    cio.write_mrc(tmp_path / "v.mrc", g["volume"], 2.5)
    cio.write_meta(tmp_path / "m.txt", g["quats"], g["trans"], ctfs)
    for name, key in (("s.mrcs", "stack_bytes"), ("v.mrc", "volume_bytes"), ("m.txt", "meta_bytes")):
        assert (tmp_path / name).read_bytes() == g[key].tobytes(), name
    ref = tmp_path / "ref.mrcs"
    ref.write_bytes(g["stack_bytes"].tobytes())
    data, apix = cio.read_mrc(ref)
    assert np.array_equal(data, g["stack"]) and apix == pytest.approx(1.37, rel=1e-7)
    (tmp_path / "ref.txt").write_bytes(g["meta_bytes"].tobytes())
    rows = cio.read_meta(tmp_path / "ref.txt")
    assert np.array_equal(rows[:, 1:5], g["quats"]) and np.array_equal(rows[:, 5:7], g["trans"])
    ds = cio.load_dataset(ref, tmp_path / "ref.txt")
    assert len(ds) == 3 and ds.grid.size == 16
    assert np.array_equal(ds.records[1].translation, g["trans"][1])
    assert ds.records[2].ctf.b_factor == g["ctf_rows"][2][7]


def test_io_errors(tmp_path):
    from paper_2508_04929_b200 import io as cio

    bad = tmp_path / "bad.mrc"
    bad.write_bytes(b"\0" * 100)
    with pytest.raises(cs.DataError):
        cio.read_mrc(bad)
    cio.write_mrc(tmp_path / "ok.mrcs", np.zeros((2, 4, 4), np.float32), 1.0)
    blob = bytearray((tmp_path / "ok.mrcs").read_bytes())
    blob[12] = 1  # mode 1
    (tmp_path / "m1.mrc").write_bytes(bytes(blob))
    with pytest.raises(cs.UnsupportedModeError):
        cio.read_mrc(tmp_path / "m1.mrc")
    (tmp_path / "short.mrc").write_bytes((tmp_path / "ok.mrcs").read_bytes()[:-4])
    with pytest.raises(cs.DataError):
        cio.read_mrc(tmp_path / "short.mrc")
    (tmp_path / "meta.txt").write_text("# x\n1 0 0 0 0 0 0 1 1 0 300 2.7 0.1 0 0\n")
    with pytest.raises(cs.DataError):
        cio.read_meta(tmp_path / "meta.txt")
