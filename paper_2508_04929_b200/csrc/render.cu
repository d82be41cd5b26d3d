// K3 (training path): binning-free forward render with deterministic
// fixed-point shared-memory accumulation.
//
// The reference renders tile by tile from per-tile Gaussian lists
// (build_tile_work + forward_tiles, _kernels.py:17-125).  On B200 the faster
// schedule for ~1 px footprints is Gaussian-major, like the backward: one
// lane per (image, Gaussian) walks its own footprint along the exact
// q < 6.5^2 row spans and adds w e into a shared-memory image.  Lanes of a
// warp hit unrelated pixels, so the adds must be atomic; shared-memory float
// atomics are CAS loops on sm_100a (3 updates/clk/SM measured), native int32
// ATOMS.ADD sustain ~10/clk/SM at random addresses
// (profiles/microbench_smem_atomics_r01.txt).  Values are therefore added as
// round-to-nearest int32 fixed point.
//
// Scales.  The Gaussians split into chunks; a CTA accumulates one chunk of
// one image into a shared-memory band in the chunk's own unit
//   scale_c = R / sum_{g in c} wb_g  (R = 2^31 - 2^20, see kFixedRange),
// wb_g >= w_g(b) for every view b, so no band sum can overflow.  A Gaussian
// brighter than 2^23 units in its view takes the rint path instead of the
// denormal one (fwd_rows_band kDen), one dimmer than 0.5 / kTailFrac units the
// dithered one (fwd_rows_band_dither).  At the end the band is added to the global
// image in the image-wide unit S = min(R / sum_g wb_g, ...) <= scale_c
// (round(v S / scale_c), one rounding per pixel and chunk), where no pixel
// can overflow either.  Integer addition makes the render bitwise
// reproducible whatever the scheduling.
//
// Precision (round 2).  Round 1 rounded every contribution in the global unit
// S, so a Gaussian's peak was only ~2^30 / N units and its tail below
// 0.5 / peak rounded away: the render error grew linearly with N (1.35e-5 rel
// L2 at 50k, 3.1e-4 at 1M).  With per-chunk units a chunk of <= 8192
// Gaussians keeps >= 2^31 / 8192 units per peak at any N, and the walk is cut
// at a fixed fraction of each Gaussian's own peak, kTailFrac = 2e-5: the
// dropped tail carries kTailFrac of the Gaussian's mass (a 2-D Gaussian
// holds a fraction t of its mass where e < t), which bounds the image error
// near 0.6 kTailFrac = 1.2e-5 rel L2 for every N (profiles/parity_margins_r02.tsv).
//
// wb_g: by eigenvalue interlacing the projected 2x2 covariance has
// lambda1 >= s_mid^2 and lambda2 >= s_min^2; with the eigenvalue floor
// (0.1 px)^2 (splat.py:207-209) det >= max(s_mid^2, f) max(s_min^2, f), so
// w = amp / (2 pi sqrt(det)) <= amp / (2 pi sqrt(that)).
//
// Along a row, e = exp(-q/2) follows e_{k+1} = e_k g_k, g_{k+1} = g_k c with
// c = 2^(2A): two FMULs per pixel instead of an MUFU.EX2, restarted every 32
// pixels so the recurrence error stays below 2e-5.
#include <algorithm>
#include <cstdlib>
#include <cmath>

#include "common.cuh"
#include "prepare.cuh"

namespace cgs {

#ifndef CGS_FWD_THREADS
#define CGS_FWD_THREADS 512
#endif
#ifndef CGS_FWD_MINB
#define CGS_FWD_MINB 2
#endif
constexpr int kRThreads = CGS_FWD_THREADS;
#ifndef CGS_FWD_CHUNK
#define CGS_FWD_CHUNK 8192
#endif
constexpr int kRChunk = CGS_FWD_CHUNK;     // max Gaussians per CTA (fwd_chunks picks the split)
constexpr int kRChunkMin = 512;
#ifndef CGS_FWD_BAND_KB
#define CGS_FWD_BAND_KB 64
#endif
constexpr int kRBandBytes = CGS_FWD_BAND_KB * 1024;  // int32 accumulator rows per CTA
#ifndef CGS_FWD_BAND_MULTI_KB
#define CGS_FWD_BAND_MULTI_KB 100
#endif
constexpr int kRBandMultiBytes = CGS_FWD_BAND_MULTI_KB * 1024;  // band budget when an image needs several
constexpr int kWbThreads = 256;  // weight-bound pass: CTA = 256 logical indices (one wave over the SMs at C2)
// Unit ranges.  A band or image pixel sums at most range x (its Gaussians' weight bounds) plus
// up to one unit per rounded contribution (<= 8192 per band pixel, <= a few thousand chunk
// flushes per image pixel), so 2^31 - 2^20 keeps every int32 sum below 2^31.  Contributions
// below 2^23 - 2^13 units take the denormal path.  Until late round 2 the unit was also capped
// at 2^22 / max wb (and the range was 2^30), which coarsened chunks whose weight bounds are
// loose (thin needles: their view-independent bound is the end-on view's peak, tens of times
// their typical view's), see test_wide_and_needle_footprints_step.
constexpr double kFixedRange = 2147483648.0 - 1048576.0;  // 2^31 - 2^20
constexpr double kContribRange = 2147483648.0 - 1048576.0;  // a single contribution: int32 (see kDen)
constexpr float kDenormalUnits = 8388608.0f - 8192.0f;      // 2^23 - 2^13: the denormal path's ceiling
#ifndef CGS_FWD_TAIL
#define CGS_FWD_TAIL 2e-5f
#endif
constexpr float kTailFrac = CGS_FWD_TAIL;      // walk each footprint down to this fraction of its peak

// View-independent peak-weight bound of one Gaussian (see the header) from
// its f32 record slots amp (3), s_min (14) and s_mid (15) (cgs_prepare).
__device__ __forceinline__ double weight_bound(float amp_f, float lo_f, float mid_f, double fl) {
    const double lo = lo_f, mid = mid_f, amp = amp_f;
    const double det = fmax(mid * mid, fl) * fmax(lo * lo, fl);
    // 1.001: headroom for the fp32 evaluation of w inside the kernels
    return 1.001 * amp / (2.0 * kPiD * sqrt(det));
}

__device__ __forceinline__ double unit_scale(double sum, double mx) {
    double sc = sum > 0.0 ? kFixedRange / sum : 1.0;
    if (mx > 0.0) sc = fmin(sc, kContribRange / mx);
    return sc;
}

// The image-wide unit S from all chunks' sub-block sums / maxima (csum, cmax:
// total values), run by one warp in a fixed order: lane l of tree w sums the
// strided entries 32 w + l + 256 k, eight xor-shuffle trees (interleaved for
// latency), then a serial sum over the trees.
__device__ __forceinline__ float image_scale(const double *__restrict__ csum, const float *__restrict__ cmax,
                                             int total) {
    const int lane = threadIdx.x & 31;
    double t[8];
    float m[8];
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        t[w] = 0.0;
        m[w] = 0.f;
        for (int i = 32 * w + lane; i < total; i += 256) {
            t[w] += __ldcg(csum + i);
            m[w] = fmaxf(m[w], __ldcg(cmax + i));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            t[w] += __shfl_xor_sync(0xffffffffu, t[w], o);
            m[w] = fmaxf(m[w], __shfl_xor_sync(0xffffffffu, m[w], o));
        }
    double s = 0.0;
    float mx = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        s += t[w];
        mx = fmaxf(mx, m[w]);
    }
    return (float)unit_scale(s, mx);
}

// Weight-bound pass.  CTA (c, sub) sums wb and takes its max over kWbThreads
// consecutive logical indices of chunk c (the chunk's scrambled order
// g = (i * A) mod n, i in [c chunk, (c+1) chunk)), one index per thread, in a
// fixed order.  The last CTA to finish (a self-resetting counter in the
// workspace) then derives the units: the image-wide S (image_scale), and per
// chunk its own unit scale_c = max(unit(chunk sum, chunk max), S) and the
// band -> image factor S / scale_c.  Deterministic: every sum has a fixed
// order.  kPrepare: the same CTA first prepares Gaussian g (K0, prepare.cuh)
// and bounds it from the values it just computed, so the training step's K0,
// weight bound and unit derivation are one launch (the scrambled order visits
// every Gaussian exactly once).
template <bool kPrepare>
__global__ void __launch_bounds__(kWbThreads) wbound_chunk_kernel(const double *__restrict__ params,
                                                                  float *__restrict__ splat, int32_t *status,
                                                                  int64_t n, double h, int64_t mulA, int chunk,
                                                                  double *__restrict__ csum, float *__restrict__ cmax,
                                                                  unsigned *__restrict__ counter,
                                                                  float *__restrict__ gscale,
                                                                  float *__restrict__ cscale,
                                                                  float *__restrict__ cratio) {
    const int64_t i0 = (int64_t)blockIdx.x * chunk, i1 = min(n, i0 + chunk);
    const int64_t i = i0 + (int64_t)blockIdx.y * kWbThreads + threadIdx.x;
    double t = 0.0;
    float m = 0.f;
    if (i < i1) {
        const int64_t g = (int64_t)(((unsigned long long)i * (unsigned long long)mulA) % (unsigned long long)n);
        float3 f;
        if (kPrepare) {
            f = prepare_one(params, g, splat, status);
        } else {
            const float *r = splat + g * CGS_SPLAT_STRIDE;
            const float2 lm = __ldg(reinterpret_cast<const float2 *>(r + 14));
            f = make_float3(__ldg(r + 3), lm.x, lm.y);
        }
        const double wb = weight_bound(f.x, f.y, f.z, (0.1 * h) * (0.1 * h));
        t = wb;
        m = (float)wb;
    }
    __shared__ double ws[kWbThreads / 32];
    __shared__ float wm[kWbThreads / 32];
    __shared__ bool last;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        t += __shfl_xor_sync(0xffffffffu, t, o);
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    }
    if ((threadIdx.x & 31) == 0) {
        ws[threadIdx.x >> 5] = t;
        wm[threadIdx.x >> 5] = m;
    }
    __syncthreads();
    const int nch = (int)gridDim.x, nsub = (int)gridDim.y;
    if (threadIdx.x < 32) {
        double s = threadIdx.x < kWbThreads / 32 ? ws[threadIdx.x] : 0.0;
        float mx = threadIdx.x < kWbThreads / 32 ? wm[threadIdx.x] : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            s += __shfl_xor_sync(0xffffffffu, s, o);
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (threadIdx.x == 0) {
            csum[(int64_t)blockIdx.x * nsub + blockIdx.y] = s;
            cmax[(int64_t)blockIdx.x * nsub + blockIdx.y] = mx;
            __threadfence();
            last = atomicAdd(counter, 1u) == (unsigned)(nch * nsub - 1);
        }
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    // every warp derives S (bitwise the same), then one warp per chunk: its nsub
    // (<= 32) sub-block values, one per lane, in a fixed xor-shuffle tree
    const float S = image_scale(csum, cmax, nch * nsub);
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        *gscale = S;
        *counter = 0u;  // ready for the next launch
    }
    for (int c = threadIdx.x >> 5; c < nch; c += kWbThreads / 32) {
        double cs = lane < nsub ? __ldcg(csum + c * nsub + lane) : 0.0;
        float cm = lane < nsub ? __ldcg(cmax + c * nsub + lane) : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            cs += __shfl_xor_sync(0xffffffffu, cs, o);
            cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, o));
        }
        if (lane == 0) {
            // scale_c >= S by construction (a chunk's sum and max are <= the image's); fmaxf guards rounding
            const float sc = fmaxf((float)unit_scale(cs, cm), S);
            cscale[c] = sc;
            cratio[c] = S / sc;
        }
    }
}

// One footprint's rows [ya, yb] into the int32 band at acc (pixel (r0, 0), row
// stride ld), columns [0, xhi], with little work per row: kRecur is chosen per
// footprint (every row shorter than 32 px -> the
// two-pixel recurrence, else one exact exp per pixel), ceil / floor run on the
// FMA pipe (adding 1.5*2^23 with directed rounding leaves the integer in the
// low mantissa bits; the clamps also absorb spans beyond +-2^22 px), and the
// row term C_k dy^2 comes from the span's own remainder,
// -log2(e)/2 k dy^2 = log2(e)/2 (rem - cut).
// Timing experiments only (wrong images): CGS_FWD_EXP 1 = non-atomic
// read-add-write, 2 = plain store, 3 = no memory op (values folded into a
// register), 4 = atomics at conflict-free addresses (bank = lane).
#if !defined(CGS_FWD_EXP) || CGS_FWD_EXP == 0 || CGS_FWD_EXP >= 5
#define CGS_BAND_ADD(p, v) atomicAdd((p), (v))
#elif CGS_FWD_EXP == 1
#define CGS_BAND_ADD(p, v) (*(volatile int *)(p) += (v))
#elif CGS_FWD_EXP == 2
#define CGS_BAND_ADD(p, v) (*(volatile int *)(p) = (v))
#elif CGS_FWD_EXP == 3
#define CGS_BAND_ADD(p, v) (g_sink ^= (v) + (int)(size_t)(p))
#elif CGS_FWD_EXP == 4
#define CGS_BAND_ADD(p, v) atomicAdd(acc + ((((p) - acc) & ~31) | (threadIdx.x & 31)), (v))
#endif
#if defined(CGS_FWD_EXP) && CGS_FWD_EXP == 3
__device__ int g_sink_dummy;
#define CGS_SINK_DECL int g_sink = 0;
#define CGS_SINK_FLUSH if (g_sink == 0x7fffffff) g_sink_dummy = g_sink;
#else
#define CGS_SINK_DECL
#define CGS_SINK_FLUSH
#endif

// kDen: contributions as denormal bit patterns (wS < 2^23, every Gaussian in the BASELINE
// configurations); otherwise (a Gaussian brighter than 2^23 units in this view, possible since
// the chunk unit is bounded by the chunk's sum of weight bounds alone) e rides unscaled and each
// contribution is converted with one rint.
template <bool kRecur, bool kDen = true>
__device__ __forceinline__ void fwd_rows_band(int *__restrict__ acc, int r0, int ld, int xhi, int ya, int yb,
                                              const Splat2 &s, float scale, float cut) {
    constexpr float kM = 12582912.0f;
    constexpr float kHalfL2e = 0.5f * 1.4426950408889634f;
    const float wS = s.w * scale;
    const float c = ex2_approx(2.f * s.A);  // g_{k+1} / g_k
    const float c2 = c * c;
    const float2 C13 = f2pack(c, c2 * c), C4 = f2pack(c2 * c2, c2 * c2);
    // Contributions land directly as integers: e is carried scaled by 2^-74 and
    // wS by 2^-75, so the product wS e 2^-149 is a denormal whose bit pattern is
    // round(wS e) (round-to-nearest-even on the 2^-149 grid, the same rounding
    // as fast_rint; explicit non-FTZ multiplies, common.cuh).  One multiply per pixel, no bias, no
    // integer fix-up.  The -wS sub term (< 0.006 units per contribution for
    // wS < 2^23) is below the rounding of each contribution and is dropped.
    const float A2 = 2.f * s.A, nHcut = -kHalfL2e * cut - (kDen ? 74.f : 0.f), xhiM = kM + (float)xhi;
    const float wSd = kDen ? wS * 0x1p-75f : wS;
    const float2 WS = f2pack(wSd, wSd);
    float dy = (float)ya - s.mpy;
    int *row = acc + (ya - r0) * ld;
    CGS_SINK_DECL
    for (int nr = yb - ya; nr >= 0; --nr, dy += 1.f, row += ld) {
        // the row centre from dy with one rounding: accumulating xcv -= slope drifted by up to
        // rows x ulp(xcv) (2.5e-4 px over a 65-row needle, a 2e-4 render error on thin footprints)
        const float xcv = fmaf(-s.slope, dy, s.mpx);
        // rem <= 0 (a row at the cut's tip) leaves an empty span or one pixel
        // at q >= cut, whose contribution rounds to 0: no branch for it
        const float rem = fmaf(-s.k * dy, dy, cut);
        const float sq = sqrt_approx(fmaxf(rem, 0.f));
        const float fa = fmaxf(__fadd_ru(fmaf(-sq, s.inv_sqrt_p00, xcv), kM), kM);
        const float fb = fminf(__fadd_rd(fmaf(sq, s.inv_sqrt_p00, xcv), kM), xhiM);
        if (fa > fb) continue;
        const int xa = __float_as_int(fa) - 0x4B400000, xb = __float_as_int(fb) - 0x4B400000;
        const float dx = (fa - kM) - xcv;
        const float Ckdy2 = fmaf(kHalfL2e, rem, nHcut);
        if (kRecur) {
            const float e0 = ex2_approx(fmaf(s.A * dx, dx, Ckdy2));
            const float g0 = ex2_approx(fmaf(A2, dx, s.A));
            const float t = g0 * g0;
            float2 E = f2pack(e0, e0 * g0);
            float2 R = f2mul(f2pack(t, t), C13);
            int x = xa;
#pragma unroll 1
            for (; x < xb; x += 2) {
                if (kDen) {
                    const float2 v = f2mul_keep_denorm(WS, E);
                    CGS_BAND_ADD(row + x, __float_as_int(v.x));
                    CGS_BAND_ADD(row + x + 1, __float_as_int(v.y));
                } else {
                    const float2 v = f2mul(WS, E);
                    CGS_BAND_ADD(row + x, __float2int_rn(v.x));
                    CGS_BAND_ADD(row + x + 1, __float2int_rn(v.y));
                }
                f2scale(E, R);
                f2scale(R, C4);
            }
            if (x == xb)
                CGS_BAND_ADD(row + x, kDen ? __float_as_int(fmul_keep_denorm(wSd, E.x)) : __float2int_rn(wSd * E.x));
        } else {
            float d = dx;
            for (int x = xa; x <= xb; ++x, d += 1.f) {
                const float e = ex2_approx(fmaf(s.A * d, d, Ckdy2));
                atomicAdd(row + x, kDen ? __float_as_int(fmul_keep_denorm(wSd, e)) : __float2int_rn(wSd * e));
            }
        }
    }
    CGS_SINK_FLUSH
}

// Dim Gaussians (w scale kTailFrac < 0.5 units).  In the chunk's unit their rounding threshold
// 0.5 / (w scale) lies above kTailFrac of the peak, and rounding each contribution to the
// nearest unit would drop the footprint beyond it: a bias, not noise.  A chunk whose unit is
// set by much brighter Gaussians -- thin needles, whose view-independent weight bound is large --
// then lost a percent of a dim blob's mass (1.4e-4 rel L2 on test_wide_and_needle_footprints_step).
// These walk down to kTailFrac like the others and round each contribution with a deterministic
// dither in [0, 1) hashed from (pixel, Gaussian): unbiased, still integer, still order-free
// (bitwise-reproducible renders).  One exact exp per pixel: dim Gaussians are rare in a step.
__device__ __forceinline__ float dither_unit(uint32_t px, uint32_t g) {
    uint32_t k = px * 0x9E3779B1u ^ g * 0x85EBCA77u;
    k ^= k >> 15;
    k *= 0x2C1B3C6Du;
    k ^= k >> 12;
    k *= 0x297A2D39u;
    k ^= k >> 15;
    return (float)(k >> 8) * 0x1p-24f;
}

__device__ __forceinline__ void fwd_rows_band_dither(int *__restrict__ acc, int r0, int ld, int D, int ya, int yb,
                                                  const Splat2 &s, float scale, float cut, uint32_t g) {
    constexpr float kHalfL2e = 0.5f * 1.4426950408889634f;
    const float wS = s.w * scale, nHcut = -kHalfL2e * cut;
    float dy = (float)ya - s.mpy;
    int *row = acc + (ya - r0) * ld;
    for (int y = ya; y <= yb; ++y, dy += 1.f, row += ld) {
        const float xcv = fmaf(-s.slope, dy, s.mpx);
        const float rem = fmaf(-s.k * dy, dy, cut);
        if (rem <= 0.f) continue;
        const float sq = sqrt_approx(rem) * s.inv_sqrt_p00;
        const int xa = max((int)ceilf(xcv - sq), 0), xb = min((int)floorf(xcv + sq), D - 1);
        const float Ckdy2 = fmaf(kHalfL2e, rem, nHcut);
        float d = (float)xa - xcv;
        for (int x = xa; x <= xb; ++x, d += 1.f) {
            const float v = wS * ex2_approx(fmaf(s.A * d, d, Ckdy2));
            const int u = __float2int_rd(v + dither_unit((uint32_t)(y * D + x), g));
            if (u) atomicAdd(row + x, u);
        }
    }
}

// CTA = (chunk of Gaussians, image, band of rows); the band's int32
// accumulator (whole 128^2 image in 64 KB) lives in shared memory, in the
// chunk's unit, and is added to the global image (image-wide unit) once at
// the end.  Lanes of a warp must hit unrelated pixels to keep ATOMS conflicts
// rare, but the device order of the Gaussians is spatial (Morton, chosen for
// the backward's region staging), so the chunk visits Gaussians in a
// scrambled order: logical index i maps to g = (i * A) mod n with
// gcd(A, n) = 1, stepped incrementally.
__global__ void __launch_bounds__(kRThreads, CGS_FWD_MINB) raster_fwd_atomic_kernel(
    const float *__restrict__ splat, int64_t n, const double *__restrict__ poses, GridF G,
    const float *__restrict__ cscale, const float *__restrict__ cratio, int HB, int64_t mulA, int chunk,
    unsigned long long *__restrict__ clamp_count, int *__restrict__ out) {
    extern __shared__ int band[];
    const int D = G.D;
    // the row stride as an opaque register value, so it is not re-read from the
    // constant bank per row (that reload's destination register would wait on
    // the row's last shared atomic reading it)
    const int ld = D + (int)(clock64() >> 62);  // = D (the counter never reaches 2^62), opaque to the compiler
    const int b = blockIdx.y;
    const int r0 = blockIdx.z * HB, r1 = min(D, r0 + HB);
    const int npx = (r1 - r0) * D;
    for (int i = threadIdx.x; i < npx; i += kRThreads) band[i] = 0;
    const PoseF P = load_pose_f(poses, b);
    const int64_t i_begin = (int64_t)blockIdx.x * chunk;
#if defined(CGS_FWD_EXP) && CGS_FWD_EXP == 6
    const int64_t i_end = i_begin;  // band init + flush only (timing experiment)
#else
    const int64_t i_end = min(n, i_begin + chunk);
#endif
    const int64_t stepA = (kRThreads * mulA) % n;
    int64_t g = ((i_begin + threadIdx.x) % n) * mulA % n;
    const float scale = cscale[blockIdx.x];
    int nclamp = 0;
    __syncthreads();
    // One projected Gaussian into the band: walk q < cut, where e(cut) is the larger of kTailFrac
    // (the precision cut, see the header) and 0.4995 / (w scale), below which a pixel rounds to 0
    // units anyway (the 1e-3 margin keeps every pixel that can round to >= 1 unit), and
    // q < 6.5^2 (splat.py:49).
    auto walk = [&](const Splat2 &s, uint32_t gid) {
        if (!(s.w > 0.f)) return;
        const float thr_round = 0.4995f * rcp_approx(s.w * scale);
        if (thr_round > kTailFrac) {  // dim in this chunk's unit: dithered rounding down to kTailFrac
            const float cut = fminf(kCutoffSq, -2.f * kLn2 * lg2_approx(kTailFrac));
            const float hy = s.hy * sqrt_approx(cut * (1.f / kCutoffSq));
            const int ylo = max(max((int)ceilf(s.mpy - hy), 0), r0);
            const int yhi = min(min((int)floorf(s.mpy + hy), D - 1), r1 - 1);
            if (ylo <= yhi) fwd_rows_band_dither(band, r0, ld, D, ylo, yhi, s, scale, cut, gid);
            return;
        }
        const float thr = fmaxf(thr_round, kTailFrac);
        if (!(thr < 1.f)) return;
        const float cut = fminf(kCutoffSq, -2.f * kLn2 * lg2_approx(thr));
        const float hy = s.hy * sqrt_approx(cut * (1.f / kCutoffSq));
        const int ylo = max(max((int)ceilf(s.mpy - hy), 0), r0);
        const int yhi = min(min((int)floorf(s.mpy + hy), D - 1), r1 - 1);
        if (ylo > yhi) return;
#if defined(CGS_FWD_EXP) && CGS_FWD_EXP == 5
        if (ylo + yhi == -12345 || cut == 1.2345f) band[0] += 1;  // projection only (timing experiment)
        return;
#endif
        // widest row = 2 sqrt(cut / p00) = 2 * 6.5 sqrt(cut / 6.5^2) / sqrt(p00)
        const bool recur = 13.f * sqrt_approx(cut * (1.f / kCutoffSq)) * s.inv_sqrt_p00 < 31.f;
        if (s.w * scale < kDenormalUnits) {
            if (recur)
                fwd_rows_band<true>(band, r0, ld, D - 1, ylo, yhi, s, scale, cut);
            else
                fwd_rows_band<false>(band, r0, ld, D - 1, ylo, yhi, s, scale, cut);
        } else if (recur) {
            fwd_rows_band<true, false>(band, r0, ld, D - 1, ylo, yhi, s, scale, cut);
        } else {
            fwd_rows_band<false, false>(band, r0, ld, D - 1, ylo, yhi, s, scale, cut);
        }
    };
    if (gridDim.z == 1) {  // the whole image in one band: every lane walks its own Gaussians
        for (int64_t i = i_begin + threadIdx.x; i < i_end; i += kRThreads) {
            const Splat2 s = project2(load_splat(splat, g), P, G);
            const uint32_t gid = (uint32_t)g;
            g += stepA;
            if (g >= n) g -= n;
            nclamp += s.clamped;
            walk(s, gid);
        }
    } else {
        // Row bands (D beyond one 64 KB band, e.g. 256^2 in 3 bands): most of a chunk's Gaussians
        // miss a band's rows, and lanes skipping them idled while the others walked (half the
        // lanes of a warp active at C4).  So a warp first sifts candidates, one per lane, and
        // stacks the survivors in shared memory; then every lane walks one stacked Gaussian.
        // Band 0 projects every candidate (each (image, Gaussian) clamp counted once) and keeps
        // those whose footprint box reaches its rows; later bands test the projected centre row
        // against a bound on the y extent (projected y variance <= max(s_max / h, 0.1 px)^2,
        // eigenvalue floor included) before any projection.  The render is bitwise the same:
        // which lane walks a Gaussian does not change the integer sums.
        int(*stk)[64] = reinterpret_cast<int(*)[64]>(band + HB * D);  // after the band (dynamic smem)
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const unsigned below = (1u << lane) - 1u;
        const float ylo_band = (float)r0, yhi_band = (float)(r1 - 1);
        int64_t i = i_begin + threadIdx.x;
        bool more = __any_sync(0xffffffffu, i < i_end);
        int depth = 0;  // warp-uniform
        while (more || depth > 0) {
            while (more && depth < 32) {
                bool keep = false;
                const int gi = (int)g;
                if (i < i_end) {
                    if (blockIdx.z == 0) {
                        const Splat2 s0 = project2(load_splat(splat, g), P, G);
                        nclamp += s0.clamped;
                        keep = s0.w > 0.f && s0.mpy - s0.hy <= yhi_band && s0.mpy + s0.hy >= ylo_band;
                    } else {
                        const float *rec = splat + g * CGS_SPLAT_STRIDE;
                        const float4 m = __ldg(reinterpret_cast<const float4 *>(rec));
                        const float yc = (P.w1[0] * m.x + P.w1[1] * m.y + P.w1[2] * m.z + P.ty) * G.inv_h + G.c0;
                        const float ry = 6.5f * 1.001f * fmaxf(__ldg(rec + 13) * G.inv_h, 0.1f) + 1.f;
                        keep = yc + ry >= ylo_band && yc - ry <= yhi_band;
                    }
                    i += kRThreads;
                    g += stepA;
                    if (g >= n) g -= n;
                }
                const unsigned bal = __ballot_sync(0xffffffffu, keep);
                if (keep) stk[warp][depth + __popc(bal & below)] = gi;
                depth += __popc(bal);
                more = __any_sync(0xffffffffu, i < i_end);
            }
            __syncwarp();
            const int take = min(depth, 32);
            const int gq = lane < take ? stk[warp][depth - take + lane] : -1;
            depth -= take;
            __syncwarp();
            if (gq >= 0) walk(project2(load_splat(splat, gq), P, G), (uint32_t)gq);
        }
    }
    if (clamp_count && blockIdx.z == 0) {  // every (image, Gaussian) projection counted once
        nclamp = __reduce_add_sync(0xffffffffu, nclamp);
        if ((threadIdx.x & 31) == 0 && nclamp) atomicAdd(clamp_count, (unsigned long long)nclamp);
    }
    __syncthreads();
    const float ratio = cratio[blockIdx.x];
    int *dst = out + (int64_t)b * D * D + (int64_t)r0 * D;
    for (int i = threadIdx.x; i < npx; i += kRThreads) {
        const int v = band[i];
        if (v) atomicAdd(dst + i, __float2int_rn((float)v * ratio));
    }
}

// int32 fixed point -> float, in place
__global__ void fixed_to_float_kernel(int *__restrict__ buf, int64_t count, const float *__restrict__ scale_ptr) {
    const float inv = 1.f / *scale_ptr;
    int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4;
    if (i + 3 < count) {
        int4 v = *reinterpret_cast<int4 *>(buf + i);
        float4 f = make_float4((float)v.x * inv, (float)v.y * inv, (float)v.z * inv, (float)v.w * inv);
        *reinterpret_cast<float4 *>(buf + i) = f;
    } else {
        for (; i < count; ++i) reinterpret_cast<float *>(buf)[i] = (float)buf[i] * inv;
    }
}

}  // namespace cgs

using namespace cgs;

// A multiplier coprime with n, near the golden ratio of n (a bijective stride)
static int64_t scramble_multiplier(int64_t n) {
    auto gcd = [](int64_t a, int64_t b) { while (b) { int64_t t = a % b; a = b; b = t; } return a; };
    if (n < 3) return 1;
    for (int64_t a = (int64_t)(0.6180339887 * (double)n) | 1; a > 1; a -= 2)
        if (gcd(a, n) == 1) return a;
    return 1;
}

// Chunks per image: equal chunks of kRChunkMin..kRChunk Gaussians, the count
// trading each CTA's band init + flush (~200 Gaussians' worth) against the
// last partial wave of CTAs over the resident slots, weighted 0.3 because CTA
// lengths vary and the tail is soft.  C2 (50k, B = 256, 296 slots): 8 chunks
// of 6250 (6.92 waves) run 2.6% faster than 13 of <= 4096 (11.24 waves).
static int64_t fwd_chunks(int64_t n, int64_t ctas_per_chunk, int slots) {
    thread_local int64_t memo[4] = {-1, -1, -1, -1};
    if (memo[0] == n && memo[1] == ctas_per_chunk && memo[2] == slots) return memo[3];
    int64_t best = (n + kRChunk - 1) / kRChunk;
    double best_cost = 1e300;
    for (int64_t nc = best; nc <= (n + kRChunkMin - 1) / kRChunkMin; ++nc) {
        const double waves = (double)(nc * ctas_per_chunk) / slots;
        const double cost = (waves + 0.3 * (std::ceil(waves) - waves)) * ((double)n / (double)nc + 200.0);
        if (cost < 0.999 * best_cost) { best_cost = cost; best = nc; }
    }
    memo[0] = n; memo[1] = ctas_per_chunk; memo[2] = slots; memo[3] = best;
    return best;
}

// Workspace: [0] image-wide scale (float), [1] the weight-bound pass's
// completion counter (u32, zero-initialised once by the caller, left 0 by every
// launch), then csum f64 [kSubMax mc], cmax f32 [kSubMax mc], cscale, cratio
// f32 [mc]; mc = the most chunks any split uses, kSubMax = the most kWbThreads-index
// sub-blocks per chunk.
static int64_t max_chunks(int64_t n) { return (n + kRChunkMin - 1) / kRChunkMin; }
constexpr int64_t kSubMax = (kRChunk + kWbThreads - 1) / kWbThreads;
static_assert(kSubMax <= 32, "the weight-bound pass reduces a chunk's sub-blocks in one warp");

extern "C" size_t cgs_render_workspace_bytes(int64_t n) {
    const int64_t mc = max_chunks(n);
    return (size_t)(8 + 12 * kSubMax * mc + 2 * 4 * mc);
}

// Two launches (+ the output memset): the weight-bound pass (with params: K0
// fused into it; its last CTA derives the units) and the render.
static int render_impl(const double *params, int32_t *status, float *splat, int64_t n, const double *poses,
                       int32_t B, cgs_grid grid, float *out, int64_t *clamp_count, void *ws, void *stream,
                       bool convert) {
    if (n <= 0 || B <= 0 || grid.size < 1 || !splat || !poses || !out || !ws || (params && !status))
        return CGS_ERR_ARG;
    const int D = grid.size;
    cudaStream_t st = (cudaStream_t)stream;
    const double h = 2.0 * grid.extent / grid.size;
    int HB = kRBandBytes / (D * (int)sizeof(int));
    if (HB < 1) return CGS_ERR_UNSUPPORTED;
    HB = HB > D ? D : HB;
    if (HB < D) {
        // Several bands: as few as a larger band allows at two CTAs per SM (kRBandMultiBytes),
        // rows split evenly.  A Gaussian cut by a band edge walks only its rows inside the band, so
        // fewer edges leave fewer lanes of a warp with short walks (C4, 256^2: 3 bands of 86 rows).
        const int hb_max = max(HB, kRBandMultiBytes / (D * (int)sizeof(int)));
        const int nb = (D + hb_max - 1) / hb_max;
        HB = (D + nb - 1) / nb;
    }
    const int bands = (D + HB - 1) / HB;
    if (bands > 1 && n > 0x7fffffff) return CGS_ERR_UNSUPPORTED;  // the banded render stacks int indices
    // banded launches also stack candidate indices per warp (64 ints per warp) after the band
    const size_t smem = (size_t)HB * D * sizeof(int) + (bands > 1 ? (size_t)kRThreads / 32 * 64 * sizeof(int) : 0);
    int rc = ensure_smem_limit((const void *)raster_fwd_atomic_kernel, smem, "raster_fwd_atomic_kernel");
    if (rc) return rc;
    int slots = 0;
    rc = resident_slots((const void *)raster_fwd_atomic_kernel, kRThreads, smem, &slots, "raster_fwd_atomic_kernel");
    if (rc) return rc;
    int64_t nchunks = fwd_chunks(n, (int64_t)B * bands, slots);
    // tests: CGS_FWD_CHUNKS forces the chunk count (clamped to chunks of kRChunkMin..kRChunk), e.g. the
    // fewest, largest chunks -- the coarsest fixed-point units -- on a batch too small to pick them
    if (const char *env = getenv("CGS_FWD_CHUNKS")) {
        const long long v = atoll(env);
        if (v > 0) nchunks = std::min<int64_t>(std::max<int64_t>(v, (n + kRChunk - 1) / kRChunk), max_chunks(n));
    }
    const int chunk = (int)((n + nchunks - 1) / nchunks);
    nchunks = (n + chunk - 1) / chunk;
    const int64_t mulA = scramble_multiplier(n);
    const int64_t mc = max_chunks(n);
    float *gscale = (float *)ws;
    double *csum = (double *)((char *)ws + 8);
    unsigned *counter = (unsigned *)ws + 1;
    float *cmax = (float *)(csum + kSubMax * mc), *cscale = cmax + kSubMax * mc, *cratio = cscale + mc;
    const int nsub = (chunk + kWbThreads - 1) / kWbThreads;
    const dim3 wg((unsigned)nchunks, (unsigned)nsub);
    if (params)
        wbound_chunk_kernel<true><<<wg, kWbThreads, 0, st>>>(params, splat, status, n, h, mulA, chunk, csum, cmax,
                                                             counter, gscale, cscale, cratio);
    else
        wbound_chunk_kernel<false><<<wg, kWbThreads, 0, st>>>(nullptr, splat, nullptr, n, h, mulA, chunk, csum,
                                                              cmax, counter, gscale, cscale, cratio);
    rc = check_launch("wbound_chunk_kernel");
    if (rc) return rc;
    const int64_t count = (int64_t)B * D * D;
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(int) * count, st);
    if (e != cudaSuccess) {
        set_error_detail("cgs_render memset", cudaGetErrorString(e));
        return CGS_ERR_CUDA;
    }
    dim3 g((unsigned)nchunks, (unsigned)B, (unsigned)bands);
    raster_fwd_atomic_kernel<<<g, kRThreads, smem, st>>>(splat, n, poses, make_grid_f(grid), cscale, cratio, HB,
                                                         mulA, chunk,
                                                         reinterpret_cast<unsigned long long *>(clamp_count),
                                                         reinterpret_cast<int *>(out));
    rc = check_launch("raster_fwd_atomic_kernel");
    if (rc || !convert) return rc;
    const int64_t threads = (count + 3) / 4;
    fixed_to_float_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(reinterpret_cast<int *>(out), count,
                                                                           gscale);
    return check_launch("fixed_to_float_kernel");
}

extern "C" int cgs_render(const float *splat, int64_t n, const double *poses, int32_t B, cgs_grid grid, float *out,
                          int64_t *clamp_count, void *ws, void *stream) {
    return render_impl(nullptr, nullptr, const_cast<float *>(splat), n, poses, B, grid, out, clamp_count, ws, stream,
                       true);
}

extern "C" int cgs_render_fixed(const float *splat, int64_t n, const double *poses, int32_t B, cgs_grid grid,
                                int32_t *out, int64_t *clamp_count, void *ws, void *stream) {
    return render_impl(nullptr, nullptr, const_cast<float *>(splat), n, poses, B, grid, reinterpret_cast<float *>(out),
                       clamp_count, ws, stream, false);
}

extern "C" int cgs_prepare_render_fixed(const double *params, int64_t n, float *splat, int32_t *status,
                                        const double *poses, int32_t B, cgs_grid grid, int32_t *out,
                                        int64_t *clamp_count, void *ws, void *stream) {
    if (!params || !status) return CGS_ERR_ARG;
    return render_impl(params, status, splat, n, poses, B, grid, reinterpret_cast<float *>(out), clamp_count, ws,
                       stream, false);
}

extern "C" int64_t cgs_render_scale_offset(int64_t) { return 0; }
