/*
 * cgs_b200.h -- C ABI of the B200-native cryoGS splatting step (libcgs_b200.so).
 *
 * Every entry point takes raw DEVICE pointers, plain sizes, a cudaStream_t last
 * (passed as void* so the header needs no CUDA include), never allocates device
 * memory inside a step (FFT plans are created once up front), never
 * synchronises the host, and returns 0 on success or a CGS_ERR_* code.  All
 * launches are stream-ordered, so a whole step is CUDA-Graph capturable.
 *
 * Each function names the reference interface it replaces
 * (/root/reference/pkg/src/cryosplat/<file>:<line>).  Batched entry points take
 * B images; B = 1 reproduces the reference's one-image call.
 *
 * Data layouts (row-major, C-contiguous):
 *   params   f64 [N][11]  mean xyz | raw scale xyz | quaternion wxyz | raw amp
 *                         (gmm.py:25-29)
 *   splat    f32 [N][16]  prepared per-Gaussian record (cgs_prepare):
 *                         mean xyz, amp, M = R diag(s) (9, row-major), s xyz
 *   poses    f64 [B][12]  rotation W row-major (9), translation tx ty (2), pad
 *                         (splat.py:73-104; translation in normalised units)
 *   ctf      f64 [B][8]   defocus_u, defocus_v [A], astigmatism_angle [rad],
 *                         voltage [kV], Cs [mm], amplitude_contrast,
 *                         phase_shift [rad], b_factor [A^2]   (optics.py:39-62)
 *   images   f32 [B][D][D] in NATURAL layout (pixel (iy, ix), origin D//2) or
 *                         FFT layout (np.fft.ifftshift of natural) when
 *                         layout == CGS_LAYOUT_FFT.
 */
#ifndef CGS_B200_H
#define CGS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CGS_OK 0
#define CGS_ERR_ARG 1         /* invalid argument (sizes, null pointers) */
#define CGS_ERR_CUDA 2        /* a CUDA launch or runtime call failed */
#define CGS_ERR_CUFFT 3       /* a cuFFT call failed */
#define CGS_ERR_UNSUPPORTED 4 /* configuration outside the compiled limits */

#define CGS_LAYOUT_NATURAL 0
#define CGS_LAYOUT_FFT 1
/* rows 2j and 2j+1 interleaved: pixel (2j + t, x) at float index (j D + x) 2 + t
 * (even D; the spectral K4's upstream for the backward's region staging) */
#define CGS_LAYOUT_ROWPAIR 2

#define CGS_MODE_ANISOTROPIC 0
#define CGS_MODE_ISOTROPIC 1

#define CGS_SPLAT_STRIDE 16   /* floats per prepared splat record */
#define CGS_ACC_STRIDE 10     /* floats per world-frame gradient accumulator */
#define CGS_BIN_CHUNK 2048    /* Gaussians per binning segment */

/* GridSpec (gmm.py:38-73): D pixels over [-extent, extent]; pixel_size in A. */
typedef struct cgs_grid {
    int32_t size;
    int32_t reserved;
    double extent;
    double pixel_size;
} cgs_grid;

/* status bits written by cgs_prepare / cgs_bin_scatter into a device int32 */
#define CGS_STATUS_DEGENERATE_ROTATION 1 /* DegenerateRotationError, splat.py:191-193 */
#define CGS_STATUS_BIN_OVERFLOW 2        /* tile list exceeded the item capacity */
#define CGS_STATUS_NONFINITE_LOSS 4      /* a loss was NaN/inf: Adam skips the update (train.py:144-145) */
#define CGS_STATUS_NONFINITE_PARAMS 8    /* a mean / scale / amplitude was NaN or inf (set by cgs_prepare):
                                          * the loss kernels then report NaN losses, as the reference's
                                          * render of such a mixture does (train.py:146-149) */

const char *cgs_version(void);
const char *cgs_error_string(int code);
/* last CUDA / cuFFT error text seen by the library (host string, thread-local) */
const char *cgs_last_error_detail(void);
/* number of (kernel) launch-state entries (dynamic shared-memory opt-in,
 * resident-slot memo) the library holds for a device ordinal: the state is
 * per device, so a process may drive several GPUs (evaluate.py:182-200). */
int32_t cgs_launch_state_entries(int32_t device);

/* ---- K0: per-Gaussian preparation ---------------------------------------
 * Replaces the image-independent part of _Projection.__init__
 * (splat.py:184-196): softplus activate (gmm.py:76-80), quaternion
 * normalisation and rotation (gmm.py:101-124), M = R diag(s).
 * Writes splat[N][16] = {mean xyz, amp, M (9, row-major), s_max, s_min, s_mid}.  A zero or
 * non-finite quaternion norm sets CGS_STATUS_DEGENERATE_ROTATION in *status;
 * a non-finite mean, activated scale or amplitude (after the fp32 cast) sets
 * CGS_STATUS_NONFINITE_PARAMS. */
int cgs_prepare(const double *params, int64_t n, float *splat, int32_t *status, void *stream);

/* ---- K2: tile binning (build_tile_work, _kernels.py:17-63) ----------------
 * A stable, segmented counting sort (one LSD radix pass keyed on tile id,
 * pre-grouped by image) that reproduces the reference's per-tile ascending
 * Gaussian order bit-exactly.  Three launches: count -> scan -> scatter.
 *
 *   S      = cgs_bin_segments(n)           segments of CGS_BIN_CHUNK Gaussians
 *   T      = ceil(D/tile)^2                tiles per image
 *   counts = int32 [B*T*S + 1]             (b, tile, segment) item counts
 *   offs   = int32 [B*T*S + 1]             exclusive scan of counts; offs[B*T*S]
 *                                          = total items; tile (b,t) owns items
 *                                          [offs[(b*T+t)*S], offs[(b*T+t+1)*S])
 *   rects  = uint32 [B][n]                 packed tile rectangle per (b, g)
 */
int64_t cgs_bin_segments(int64_t n);
int64_t cgs_bin_tiles(int32_t size, int32_t tile);

/* Count pass from parameters: computes the reference's fp64 bounding box
 * (splat.py:218-226, incl. the eigenvalue-floor clamp splat.py:229-260) per
 * (image, Gaussian).  bbox_out (int32 [B][n][4], x0 x1 y0 y1) and clamp_count
 * (int32 [B], CLAMP_EVENTS, splat.py:60-70,277) are optional (may be NULL). */
int cgs_bin_count(const double *params, int64_t n, const double *poses, int32_t B, cgs_grid grid,
                  int32_t tile, uint32_t *rects, int32_t *counts, int32_t *bbox_out,
                  int32_t *clamp_count, void *stream);

/* Count pass from a caller-supplied bbox (int32 [B][n][4]); used to check the
 * binning on bit-identical input. */
int cgs_bin_count_bbox(const int32_t *bbox, int64_t n, int32_t B, int32_t size, int32_t tile,
                       uint32_t *rects, int32_t *counts, void *stream);

/* Generic int32 exclusive scan of count elements (out may alias in).  ws must
 * hold cgs_scan_workspace_bytes(count) bytes. */
size_t cgs_scan_workspace_bytes(int64_t count);
int cgs_exclusive_scan(const int32_t *in, int32_t *out, int64_t count, void *ws, void *stream);

/* Scatter pass: items[pos] = g for every (b, g, tile) in the stable order.
 * Items at or beyond capacity are dropped and CGS_STATUS_BIN_OVERFLOW is set. */
int cgs_bin_scatter(const uint32_t *rects, int64_t n, int32_t B, int32_t size, int32_t tile,
                    const int32_t *offs, int32_t *items, int64_t capacity, int32_t *status,
                    void *stream);

/* ---- K3: forward rasterizer (forward_tiles, _kernels.py:66-125; rasterize,
 * splat.py:263-298) --------------------------------------------------------
 * One CTA per (image, tile): stages the tile's Gaussians (ascending id) in
 * shared memory and accumulates sum_g w_g (exp(-q/2) - sub) per pixel, q <
 * 6.5^2, in the reference's per-pixel order.  out f32 [B][D][D]. */
int cgs_raster_fwd(const float *splat, int64_t n, const double *poses, int32_t B, cgs_grid grid,
                   int32_t tile, const int32_t *items, const int32_t *offs, int64_t capacity,
                   float *out, int32_t layout, void *stream);

/* ---- K3 (training path): binning-free render -------------------------------
 * Same image as cgs_raster_fwd without tile lists: one lane per (image,
 * Gaussian) walks its footprint and adds w e into a shared-memory image as
 * int32 fixed point.  The Gaussians split into chunks (one CTA per chunk and
 * image); a chunk's band uses its own scale 2^30 / (sum of its Gaussians'
 * view-independent weight bounds), so band sums cannot overflow, and the band
 * is added to the image in one image-wide unit (2^30 / sum over all
 * Gaussians).  Each Gaussian walks q < 6.5^2 (splat.py:49) down to 2e-5 of its
 * peak (the dropped tail bounds the render error near 1.2e-5 rel L2 at any N;
 * the reference's -sub per pixel, 6.7e-10 of the peak, is below that).
 * Integer sums make the result bitwise deterministic.
 * out f32 [B][D][D] natural layout (used as int32 scratch first); ws holds
 * cgs_render_workspace_bytes(n) bytes, zero-initialised once before its first
 * use (it carries a completion counter that every launch leaves at 0).  clamp_count (nullable, device int64)
 * is incremented by the number of (image, Gaussian) projections that hit the
 * eigenvalue floor: CLAMP_EVENTS.count += proj.n_clamped per image
 * (splat.py:276-277).  Replaces rasterize (splat.py:263-298) inside the
 * training step. */
size_t cgs_render_workspace_bytes(int64_t n);
int cgs_render(const float *splat, int64_t n, const double *poses, int32_t B, cgs_grid grid, float *out,
               int64_t *clamp_count, void *ws, void *stream);
/* cgs_render without the final conversion: out holds the int32 fixed-point
 * image; its scale (pixel value = int / scale) is the float at
 * ws + cgs_render_scale_offset(n) floats, for a consumer that converts on load
 * (cgs_ctf_mse_spectral). */
int cgs_render_fixed(const float *splat, int64_t n, const double *poses, int32_t B, cgs_grid grid, int32_t *out,
                     int64_t *clamp_count, void *ws, void *stream);
int64_t cgs_render_scale_offset(int64_t n);
/* K0 (cgs_prepare) and cgs_render_fixed in one: the Gaussians are prepared
 * into splat (and status) by the render's weight-bound pass, which visits
 * every Gaussian once in the render's scrambled chunk order; the image is
 * bitwise that of cgs_prepare + cgs_render_fixed.  Two launches + the output
 * memset (the training step's K0 + K3). */
int cgs_prepare_render_fixed(const double *params, int64_t n, float *splat, int32_t *status, const double *poses,
                             int32_t B, cgs_grid grid, int32_t *out, int64_t *clamp_count, void *ws, void *stream);

/* ---- K4: CTF, centred FFTs and MSE (optics.py:78-141, train.py:114-121,153)
 * ctf_evaluate (optics.py:93-121): H f64 [B][D][D], centred layout. */
int cgs_ctf_evaluate(const double *ctf, int32_t B, cgs_grid grid, double *H, void *stream);

/* cuFFT plans for a batch of B D x D real images (created once, reused). */
int cgs_fft_plan_create(int32_t size, int32_t B, void **plan);
int cgs_fft_plan_destroy(void *plan);
/* complex64 elements of the spectrum workspace a plan needs: B*D*(D/2+1) */
int64_t cgs_fft_spectrum_elems(int32_t size, int32_t B);

/* apply_ctf (optics.py:124-141): out = Re F^-1( H . F(in) ) per image, computed
 * as R2C -> multiply by H_sym(k) = (H(k) + H(-k mod D))/2 -> C2R (identical to
 * the reference's complex form).  H comes from ctf (f64 [B][8])
 * or, when ctf == NULL, from Harr (f64 [B][D][D], centred).  in/out may alias;
 * spectrum holds cgs_fft_spectrum_elems complex64. */
int cgs_ctf_apply(void *plan, const float *in, float *out, int32_t B, cgs_grid grid,
                  const double *ctf, const double *Harr, void *spectrum, int32_t layout,
                  void *stream);

/* loss_mse (train.py:114-121) and dL/dmodel = 2/D^2 (model - obs)
 * (train.py:153): loss f64 [B] (fp64 accumulation), resid f32 [B][D][D]
 * (may be NULL).  A non-finite loss sets CGS_STATUS_NONFINITE_LOSS in *status
 * (status may be NULL). */
int cgs_loss_residual(const float *model, const float *obs, int32_t B, int32_t size,
                      double *loss, float *resid, int32_t *status, void *stream);

/* Fused K4 of one training step: model = CTF(render); loss; upstream =
 * CTF(2/D^2 (model - obs)) (train.py:151-155).  ctf == NULL means no CTF (the
 * operator is the identity).  model may be NULL.  Images in `layout`. */
int cgs_ctf_mse(void *plan, const float *render, const float *obs, int32_t B, cgs_grid grid,
                const double *ctf, void *spectrum, float *model, float *upstream, double *loss,
                int32_t *status, int32_t layout, void *stream);

/* K4 in the Fourier domain.  cgs_obs_spectrum writes one record per
 * observation: its half spectrum F(obs) (complex64) followed by H_sym / D^2 of
 * its CTF (ctf f64 [B][8]), in an internal row order shared with the kernels;
 * cgs_obs_spectrum_elems(D, B) floats in all (D = 64 or 128, else 0 and
 * CGS_ERR_UNSUPPORTED).  A record depends only on the data, so a dataset
 * computes it once.  cgs_ctf_mse_spectral then gives the loss and upstream of
 * cgs_ctf_mse (no model image) from F(r) = H_sym F(render) - F(obs):
 * loss = sum |F(r)|^2 / D^4 by Parseval, upstream = 2/D^2 CTF^T(r), with one
 * forward and one inverse transform per image. */
int64_t cgs_obs_spectrum_elems(int32_t size, int32_t B);
int cgs_obs_spectrum(const float *obs, const double *ctf, int32_t B, cgs_grid grid, float *spec, void *stream);
int cgs_ctf_mse_spectral(const float *render, const float *obs_spec, int32_t B, cgs_grid grid, float *upstream,
                         double *loss, int32_t *status, int32_t upstream_layout, void *stream);
/* The same from a cgs_render_fixed image: render_fixed int32 [B][D][D] and its
 * scale pointer (ws + cgs_render_scale_offset(n)).  upstream_layout:
 * CGS_LAYOUT_NATURAL or CGS_LAYOUT_ROWPAIR. */
int cgs_ctf_mse_spectral_fixed(const int32_t *render_fixed, const float *render_scale, const float *obs_spec,
                               int32_t B, cgs_grid grid, float *upstream, double *loss, int32_t *status,
                               int32_t upstream_layout, void *stream);
/* The same with image b's observation record at row rows[b] (int64 [B], device)
 * of a dataset's resident records obs_spec [R][cgs_obs_spectrum_elems(D, 1)]:
 * a batch of a resident dataset needs no gathered copy of its records. */
int cgs_ctf_mse_spectral_fixed_rows(const int32_t *render_fixed, const float *render_scale, const float *obs_spec,
                                    const int64_t *rows, int32_t B, cgs_grid grid, float *upstream, double *loss,
                                    int32_t *status, int32_t upstream_layout, void *stream);
/* The spectral K4 through cuFFT (the apply_ctf -> loss_mse -> apply_ctf chain of
 * train.py:151-155, optics.py:124-141), for the other sizes (C4's 256^2 half spectrum
 * does not fit one CTA).  Records: F(obs) then H_sym / D^2, natural [ky][kx]
 * half spectrum, n = D (D/2+1): 3n floats per record, padded to an even count
 * (cgs_obs_spectrum_fft_elems(D, B) floats in all, any D >= 2); they are
 * not interchangeable with cgs_obs_spectrum's.  plan: cgs_fft_plan_create(D, B);
 * spectrum: cgs_fft_spectrum_elems(D, B) complex64 scratch; workspace:
 * cgs_spectral_fft_workspace_bytes(D, B) bytes, zero-initialised once (per-CTA
 * loss sums and self-resetting counters).  cgs_ctf_mse_spectral_fft takes a
 * cgs_render_fixed image, rows as cgs_ctf_mse_spectral_fixed_rows (NULL: row
 * b): one R2C, one filter/loss kernel, one C2R per batch (cgs_ctf_mse takes two
 * transform pairs).  upstream_layout CGS_LAYOUT_NATURAL, or CGS_LAYOUT_ROWPAIR
 * (even D; an in-place interleave after the C2R, else CGS_ERR_UNSUPPORTED). */
int64_t cgs_obs_spectrum_fft_elems(int32_t size, int32_t B);
size_t cgs_spectral_fft_workspace_bytes(int32_t size, int32_t B);
int cgs_obs_spectrum_fft(void *plan, const float *obs, const double *ctf, int32_t B, cgs_grid grid, void *spectrum,
                         float *spec, void *stream);
int cgs_ctf_mse_spectral_fft(void *plan, const int32_t *render_fixed, const float *render_scale, const float *obs_spec,
                             const int64_t *rows, int32_t B, cgs_grid grid, void *spectrum, void *workspace,
                             float *upstream, double *loss, int32_t *status, int32_t upstream_layout,
                             void *stream);

/* Batched Fourier filter out = Re ifft2(F fft2(in)), per image F = H_sym (CTF,
 * ctf f64 [B][8], may be NULL) x the sub-pixel shift ramp
 * exp(-2 pi i (fx tx + fy ty) / D) (shifts f64 [B][2] pixels, may be NULL):
 * apply_ctf (optics.py:124-141) followed by phase_shift_translate
 * (optics.py:144-159), as simulate (simulate.py:241-244) and the observed-image
 * centring (train.py:124-133) use them.  One kernel; in-place allowed.
 * Sizes 32, 64, 128 (else CGS_ERR_UNSUPPORTED). */
int cgs_fourier_filter(const float *in, float *out, int32_t B, cgs_grid grid, const double *ctf,
                       const double *shifts, void *stream);

/* ---- K8: voxelize (evaluate.voxelize, evaluate.py:76-122, and
 * voxelize_gaussians, _kernels.py:193-235) ----------------------------------
 * Samples the mixture params f64 [n][11] at the D^3 voxel centres, culled on
 * q < 6.5^2 like the rasterizer: out f64 [D][D][D] indexed [z][y][x].
 * Deterministic (int64 fixed-point accumulation).  ws: cgs_voxelize_workspace_bytes(n)
 * bytes; status gets CGS_STATUS_DEGENERATE_ROTATION (may be NULL). */
size_t cgs_voxelize_workspace_bytes(int64_t n);
int cgs_voxelize(const double *params, int64_t n, cgs_grid grid, double *out, void *ws, int32_t *status,
                 void *stream);

/* ---- K5: fused backward (backward_pixels, _kernels.py:128-190, plus the
 * per-image part of rasterize_backward, splat.py:332-349) ------------------
 * Gaussian-major: each CTA owns a chunk of Gaussians and a group of images,
 * stages each upstream image in shared memory, reduces per-Gaussian moments
 * with warp shuffles and accumulates, over its images, the 10-float
 * world-frame accumulator {cnorm sA, W2^T ac (sx, sy), W2^T (ac S) W2}
 * (SURVEY.md 8(a) row 15).  Deterministic (no atomics).
 *   partial f32 [G][n][10], G = cgs_bwd_groups(B, images_per_group). */
int64_t cgs_bwd_groups(int32_t B, int32_t images_per_group);
int cgs_raster_bwd(const float *splat, int64_t n, const double *poses, int32_t B, cgs_grid grid,
                   const float *upstream, int32_t layout, float *partial,
                   int32_t images_per_group, void *stream);

/* Data-parallel exchange buffer: the sum of partial
 * [G][n][10] over groups, in group order in fp64 (the order of the
 * single-GPU epilogue), rounded once to f32, laid out in slices of `per`
 * Gaussians: slice k = acc[k * S .. (k+1) * S), S = cgs_acc_slice_floats(n,
 * per) = per * 10 + 2 floats (8-byte aligned), Gaussian g at slice g / per,
 * offset (g % per) * 10; slot per * 10 of every slice is this rank's skip
 * flag (1.0 when *status has CGS_STATUS_BIN_OVERFLOW / _NONFINITE_LOSS /
 * _NONFINITE_PARAMS, status nullable), then one pad float; rows past n are 0.
 * per = n is the all-reduce layout (one slice); per = ceil(n / world) is the
 * reduce-scatter layout (rank k owns slice k).  G = 0 (an empty local batch)
 * writes zeros, so an idle rank still joins the collective.  acc holds
 * ceil(n / per) * S floats.  Replaces the per-image sum of rasterize_backward
 * results across a batch (train.py:136-161 for B > 1, over ranks). */
int64_t cgs_acc_slice_floats(int64_t n, int64_t per);
int cgs_reduce_partials_sliced(const float *partial, int32_t G, int64_t n, int64_t per, const int32_t *status,
                               float *acc, void *stream);
/* cgs_reduce_partials_sliced with per = n and no status: acc f32 [n][10] + 2. */
int cgs_reduce_partials(const float *partial, int32_t G, int64_t n, float *acc, void *stream);

/* Fused peer-memory exchange (data parallel over NVLink / NVSwitch): ONE
 * launch per rank does reduce-scatter + epilogue + Adam + parameter all-gather
 * for its Gaussian slice.  accs[p] (device array of `world` pointers) = rank
 * p's accumulator in the reduce-scatter layout above (per = ceil(n / world)),
 * mapped into this process; stores[p] = rank p's fp64 parameter store of
 * world * per rows x 11; flags[p] = rank p's u32 [world + 1] handshake array
 * (zero-initialised; arrive slots, done counter), or flags = nullptr for a
 * single-process simulation that launches the ranks one after another on one
 * device (no handshake).  m, v: this rank's moments for its `per` rows.
 * hyper f64 [4] on the device = (lr, bc1, bc2, epoch): the epoch is the step
 * counter, identical on every rank, +1 per step, starting at 1.  Rank r sums
 * slice r of every peer's accumulator in rank order (fp64), skips the update
 * when any peer's flag is set, runs the chain + Adam as cgs_epilogue_adam_dev
 * and stores the new rows into every peer's store.  Replaces the exchange of
 * train.py:136-161 over ranks (all-reduce or reduce-scatter, AdamState.update
 * train.py:93-111, parameter broadcast).  Every rank must launch it each step
 * with the same n, per, world (the grid is cgs_peer_blocks(per) CTAs, all
 * co-resident). */
int32_t cgs_peer_blocks(int64_t per);
int cgs_peer_epilogue_adam(const float *const *accs, double *const *stores, uint32_t *const *flags, int32_t rank,
                           int32_t world, int64_t n, int64_t per, double *m, double *v, int32_t mode, double scale,
                           double beta1, double beta2, double eps, const double *hyper, void *stream);

/* ---- particle residency -----------------------------------
 * dst[i] = src[idx[i]] for i < rows, rows of row_bytes (multiple of 16; src,
 * dst 16-byte aligned); idx int64 on the device.  src may be device memory or
 * pinned host memory (UVA, zero-copy over PCIe/C2C): it loads a rank's epoch
 * slice of a host-resident particle stack into HBM on a side stream.
 * Replaces the per-record host reads of train.py:222-223 for the slice. */
int cgs_gather_rows(const void *src, const int64_t *idx, int64_t rows, int64_t row_bytes, void *dst, void *stream);

/* ---- K6: epilogue + Adam (splat.py:344-381, train.py:157-159, train.py:101-111)
 * grads f64 [n][11] = scale * chain(acc) for the raw parameters; mode
 * isotropic sums the three raw-scale gradients (train.py:157-159).
 * acc [G][n][10] must be 8-byte aligned (read as float pairs); else CGS_ERR_ARG. */
int cgs_epilogue_grads(const float *acc, int32_t G, int64_t n, const double *params, int32_t mode,
                       double scale, double *grads, void *stream);

/* AdamState.update (train.py:101-111), fp64, in place; bc1 = 1 - beta1^t,
 * bc2 = 1 - beta2^t. */
int cgs_adam(double *params, const double *grads, double *m, double *v, int64_t count, double lr,
             double beta1, double beta2, double eps, double bc1, double bc2, void *stream);

/* Fused epilogue + Adam over acc [G][n][10].  When skip_if_status != NULL and
 * *skip_if_status has CGS_STATUS_BIN_OVERFLOW or CGS_STATUS_NONFINITE_LOSS set,
 * the update is skipped: the reference returns before Adam on a non-finite
 * loss (train.py:144-145), and an overflowed tile list is re-run larger. */
int cgs_epilogue_adam(const float *acc, int32_t G, int64_t n, double *params, double *m, double *v,
                      int32_t mode, double scale, double lr, double beta1, double beta2, double eps,
                      double bc1, double bc2, const int32_t *skip_if_status, void *stream);
/* cgs_epilogue_adam with (lr, bc1, bc2) read from device memory hyper f64 [3],
 * so a CUDA graph holding the step replays unchanged from step to step. */
int cgs_epilogue_adam_dev(const float *acc, int32_t G, int64_t n, double *params, double *m, double *v,
                          int32_t mode, double scale, double beta1, double beta2, double eps, const double *hyper,
                          const int32_t *skip_if_status, void *stream);

/* ---- measurement ----------------------------------------------------------
 * In-ellipse (image, Gaussian, pixel) pairs q < 6.5^2: the algorithmic work
 * unit of SURVEY.md 8(d).  pairs int64 [B] (accumulated, caller zeroes).
 * cgs_count_pairs_cut counts q < cut_sq instead; cgs_bwd_cut_sq() is the cut
 * of the backward's walk (q < -2 ln 1e-7, the pairs K5 evaluates). */
int cgs_count_pairs(const float *splat, int64_t n, const double *poses, int32_t B, cgs_grid grid,
                    int64_t *pairs, void *stream);
int cgs_count_pairs_cut(const float *splat, int64_t n, const double *poses, int32_t B, cgs_grid grid,
                        double cut_sq, int64_t *pairs, void *stream);
double cgs_bwd_cut_sq(void);

#ifdef __cplusplus
}
#endif
#endif /* CGS_B200_H */
