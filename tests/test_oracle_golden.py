"""Pin the CPU oracle against golden vectors produced by the reference itself.

Fixtures: tests/golden/*.npz, written by tests/golden/make_golden.py (which runs
/root/reference).  CPU only.
"""

import numpy as np
import pytest

from conftest import grads_close, load_golden, rel_l2


def _stack_inputs(oracle, g):
    D, n, B = int(g["D"]), int(g["n"]), int(g["B"])
    grid = oracle.Grid(D, 0.5, 1.5)
    params = oracle.init_random(n, 0, grid)
    poses = [oracle.sample_pose(np.random.default_rng(1000 + i)) for i in range(B)]
    Hs = None
    if not np.isnan(g["defocus"][0]):
        Hs = [oracle.ctf_evaluate(oracle.Ctf(d, d), grid) for d in g["defocus"]]
    return grid, params, poses, Hs


@pytest.mark.parametrize("case", ["c1_step", "c2_slice"])
def test_oracle_matches_reference_stack(oracle, case):
    g = load_golden(case)
    grid, params, poses, Hs = _stack_inputs(oracle, g)
    B = int(g["B"])
    ntx = -(-grid.size // 16)
    off = 0
    for i, (W, t) in enumerate(poses):
        proj = oracle.project(params, W, t, grid)
        # bbox and tile lists: bit-exact
        assert np.array_equal(proj.bbox, g["bbox"][i])
        ids, starts = oracle.build_tile_work(proj.bbox, 16, ntx, ntx)
        assert np.array_equal(starts, g["tile_starts"][i])
        assert np.array_equal(ids, g["tile_ids"][off:off + len(ids)])
        off += len(ids)
        assert proj.n_clamped == g["n_clamped"][i]
        H = None if Hs is None else Hs[i]
        loss, grads, rendered, model, up, sums, _ = oracle.image_step(
            params, W, t, grid, H, g["observed"][i])
        np.testing.assert_allclose(rendered, g["rendered"][i], rtol=1e-12, atol=1e-12 * rendered.max())
        np.testing.assert_allclose(model, g["model"][i], rtol=1e-10, atol=1e-12 * np.abs(model).max())
        assert loss == pytest.approx(float(g["losses"][i]), rel=1e-12)
        if "sums_first" in g and i == 0:
            assert rel_l2(sums, g["sums_first"]) < 1e-10
            assert rel_l2(grads, g["grads_first"]) < 1e-10
    losses, grads = oracle.batch_step(params, poses, grid, Hs, g["observed"])
    np.testing.assert_allclose(losses, g["losses"], rtol=1e-12)
    grads_close(grads, g["grads_mean"], 1e-9, 1e-8)
    assert off == len(g["tile_ids"])


def test_world_accumulator_form_equals_sum_of_per_image_backward(oracle):
    """the batched 10-float form equals sum_b rasterize_backward."""
    g = load_golden("c1_step")
    grid, params, poses, _ = _stack_inputs(oracle, g)
    acc = np.zeros((len(params), 10))
    for i, (W, t) in enumerate(poses):
        proj = oracle.project(params, W, t, grid)
        sums = oracle.backward_raw_sums(params, W, t, grid, g["upstream"][i], proj)
        acc += oracle.world_accumulator(proj, sums)
    grads = oracle.grads_from_world_accumulator(params, acc) / len(poses)
    grads_close(grads, g["grads_mean"], 1e-9, 1e-8)


def test_kats(oracle):
    k = load_golden("kat")
    grid = oracle.Grid(64, 0.5, 3.0)
    W, t = k["dense_W"], k["dense_t"]
    for tile in (8, 16, 32):
        pix, _ = oracle.rasterize(k["dense_params"], W, t, grid, tile_size=tile)
        np.testing.assert_allclose(pix, k[f"dense_render_tile{tile}"], rtol=1e-12, atol=1e-12 * pix.max())
        proj = oracle.project(k["dense_params"], W, t, grid)
        ntx = -(-64 // tile)
        ids, starts = oracle.build_tile_work(proj.bbox, tile, ntx, ntx)
        assert np.array_equal(ids, k[f"dense_ids_tile{tile}"])
        assert np.array_equal(starts, k[f"dense_starts_tile{tile}"])
    gr = oracle.rasterize_backward(k["dense_params"], W, t, grid, k["dense_upstream"])
    assert rel_l2(gr, k["dense_grads"]) < 1e-10
    pix, nc = oracle.rasterize(np.asarray([[0, 0, 0, *[oracle.inverse_activate(1e-6)] * 3, 1, 0, 0, 0,
                                            oracle.inverse_activate(1.0)]], float), np.eye(3), np.zeros(2), grid)
    np.testing.assert_allclose(pix, k["clamp_render"], rtol=1e-12)
    assert nc == int(k["clamp_count"]) == 1
    pix, nc = oracle.rasterize(k["needle_params"], np.eye(3), np.zeros(2), grid)
    np.testing.assert_allclose(pix, k["needle_render"], rtol=1e-10, atol=1e-12 * pix.max())
    assert nc == int(k["needle_clamp_count"])
    gr = oracle.rasterize_backward(k["needle_params"], np.eye(3), np.zeros(2), grid, k["needle_upstream"])
    assert rel_l2(gr, k["needle_grads"]) < 1e-10
    assert float(oracle.inverse_activate(5e-5)) == pytest.approx(-9.903462552431961, rel=1e-12)
    assert float(k["inv_act_5e-5"]) == pytest.approx(-9.903462552431961, rel=1e-12)
    st = oracle.Adam(1)
    prm = np.zeros((1, 11))
    st.update(prm, k["adam_g1"], 0.01)
    st.update(prm, k["adam_g2"], 0.01)
    np.testing.assert_allclose(prm, k["adam_params"], rtol=1e-14)


def test_ctf_and_apply(oracle):
    c = load_golden("ctf")
    assert oracle.electron_wavelength(300.0) == pytest.approx(float(c["lambda_300"]), rel=1e-15)
    assert oracle.electron_wavelength(300.0) == pytest.approx(0.0196875, rel=1e-4)
    for i in range(4):
        D = int(c[f"ctf{i}_D"])
        grid = oracle.Grid(D, 0.5, 1.5)
        H = oracle.ctf_evaluate(oracle.Ctf(*c[f"ctf{i}_params"]), grid)
        np.testing.assert_allclose(H, c[f"ctf{i}_H"], rtol=1e-12, atol=1e-13)
        out = oracle.apply_ctf(c[f"ctf{i}_img"], H)
        np.testing.assert_allclose(out, c[f"ctf{i}_applied"], rtol=1e-10, atol=1e-12)


def test_nyquist_symmetrisation_matches_complex_apply(oracle):
    """for even D with astigmatism, Re(IFFT(H F x)) equals
    R2C/C2R with H_sym(k) = (H(k) + H(-k mod D)) / 2 -- the form the GPU uses."""
    c = load_golden("ctf")
    for i in range(4):
        D = int(c[f"ctf{i}_D"])
        H = c[f"ctf{i}_H"]
        img = c[f"ctf{i}_img"]
        Hu = np.fft.ifftshift(H)                      # unshifted layout, index = freq mod D
        neg = (-np.arange(D)) % D
        Hsym = 0.5 * (Hu + Hu[np.ix_(neg, neg)])
        X = np.fft.rfft2(np.fft.ifftshift(img))
        y = np.fft.fftshift(np.fft.irfft2(X * Hsym[:, : D // 2 + 1], s=(D, D)))
        np.testing.assert_allclose(y, c[f"ctf{i}_applied"], rtol=1e-9, atol=1e-12)
