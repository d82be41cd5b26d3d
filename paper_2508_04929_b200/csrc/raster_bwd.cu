// K5: fused backward, the B200 replacement of backward_pixels
// (_kernels.py:128-190) plus the per-image part of rasterize_backward
// (splat.py:332-349), batched over images.
//
// Gaussian-major, one lane per (image, Gaussian), atomic-free.  A CTA owns
// one Gaussian per thread and a group of images; for each image the upstream
// gradient sits in shared memory and every thread walks its own Gaussian's
// footprint row by row along the exact q < 6.5^2 span (row-conditional
// coordinates, common.cuh).  Same-size footprints keep the warp's lanes in
// near lockstep, so no lane idles on another lane's rows and no cross-lane
// reduction is needed.  Per pixel it accumulates moments of ge = g e in pixel
// units (per row: sum ge, sum g, sum ge dx', sum ge dx'^2; per image the
// dy-weighted row sums), which carry the reference's six raw sums exactly
// (the default kernel drops sum g, see bwd_rowpairs):
//   sA = sum ge - sub sum g,  s_ab = 1/(2 h^2) (sum ge (Pd)_a (Pd)_b - p_ab sA),
// with (Pd)_x = p00 dx', (Pd)_y = p01 dx' + k dy.  They are converted in
// registers to the image-summable 10-float world-frame accumulator
// {cnorm sA, W2^T ac (sx, sy), W2^T (ac S) W2} and
// summed over the CTA's images.  The CTA writes its image group's partial
// once; the epilogue sums groups in a fixed order: bitwise reproducible.
//
// Kernels:
//  * raster_bwd_region_kernel (default, natural layout): per image the CTA
//    stages only the union of its Gaussians' footprint boxes (Morton order
//    keeps it small), row-pair interleaved, and walks two rows per packed step
//    (bwd_rowpairs); up to 128^2 128 threads, 70 registers, 6 CTAs per SM,
//    beyond it 256 threads, 64 registers, 4 CTAs per SM (RegShape).
//  * raster_bwd_db_kernel (CGS_BWD_KERNEL=db, D <= 160): whole upstream images
//    double-buffered with 1-D bulk async copies (TMA engine, mbarrier), one row
//    per step (bwd_rows).
//  * raster_bwd_band_kernel (FFT layout, or D beyond the region band):
//    synchronous row bands, one row per step.
#include <cstdlib>

#include "common.cuh"

namespace cgs {

constexpr int kBwdThreadsDB = 512;       // double-buffered kernel: Gaussians per CTA
constexpr int kBwdThreadsBand = 256;     // band kernel
constexpr int kBandBytes = 96 * 1024;    // upstream rows staged per band
constexpr int kDBMaxBytes = 200 * 1024;  // two whole images must fit
constexpr int kRowPad = 4;                // floats of slack after every staging buffer (bwd_rows reads ahead)

struct Moments {
    float e, g, x, y, xx, xy, yy;
};

// One pixel pair (or a single pixel when GP's high lane is 0) of a row walk:
// packed per-row sums of ge, g, ge dx', ge dx'^2.
struct RowSums {
    float2 e = {0.f, 0.f}, g = {0.f, 0.f}, x = {0.f, 0.f}, xx = {0.f, 0.f};
};

__device__ __forceinline__ void bwd_pair(RowSums &a, float2 GP, float2 E, float2 DX) {
    const float2 GE = f2mul(GP, E);
    f2acc_add(a.e, GE);
    f2acc_add(a.g, GP);
    const float2 T = f2mul(GE, DX);
    f2acc_add(a.x, T);
    f2acc_fma(a.xx, T, DX);
}

// Walk rows [ya, yb] of one footprint over upstream rows stored from row r0.
// e = 2^(A dx'^2 + Ck dy^2) along a row by the recurrence e_{k+1} = e_k g_k,
// g_{k+1} = g_k c (c = 2^(2A)), two pixels per packed f32x2 step:
// (e_k, e_k+1) *= (g_k g_k+1, g_k+1 g_k+2), that pair *= c^4 (relative error
// < 2e-5 over 32 pixels).  Rows longer than 32 pixels take an exact exp per
// pixel instead.
// img points at pixel (r0, 0) of a staged block with row stride `ld`; pixel
// columns are clipped to [xlo, xhi] (absolute image coordinates).
__device__ __forceinline__ void bwd_rows(const float *__restrict__ img, int r0, int ld, int xlo, int xhi, int ya,
                                         int yb, const Splat2 &s, float c2A, Moments &M) {
    const float c = c2A, c4 = (c * c) * (c * c);
    const float2 C4 = f2pack(c4, c4), TWO = f2pack(2.f, 2.f);
    float dy = (float)ya - s.mpy;
    const float *row = img + (ya - r0) * ld;
    for (int iy = ya; iy <= yb; ++iy, dy += 1.f, row += ld) {
        const float xcv = fmaf(-s.slope, dy, s.mpx);  // one rounding per row, no drift
        const float rem = fmaf(-s.k * dy, dy, kCutoffSq);
        if (rem <= 0.f) continue;
        const float half = sqrt_approx(rem) * s.inv_sqrt_p00;
        const int xa = max((int)ceilf(xcv - half), xlo);
        int xb = min((int)floorf(xcv + half), xhi);
        if (xa > xb) continue;
        const float dx = (float)xa - xcv;
        const float Ckdy2 = s.Ck * dy * dy;
        RowSums a;
        if (xb - xa < 32) {
            const float e0 = ex2_approx(fmaf(s.A * dx, dx, Ckdy2));
            const float g0 = ex2_approx(s.A * fmaf(2.f, dx, 1.f));
            const float g1 = g0 * c;
            float2 E = f2pack(e0, e0 * g0);
            float2 R = f2pack(g0 * g1, g1 * g1 * c);
            float2 DX = f2pack(dx, dx + 1.f);
            // software-pipelined: the next pair's loads issue before this
            // pair's math (they may read up to 2 floats past the span; every
            // staging buffer carries kRowPad floats of slack)
            const float *p = row + xa;
            float2 GP = f2pack(p[0], p[1]);
            const float *pe = row + xb;
#pragma unroll 1
            for (; p < pe; p += 2) {
                const float2 GN = f2pack(p[2], p[3]);
                bwd_pair(a, GP, E, DX);
                f2scale(E, R);
                f2scale(R, C4);
                f2acc_add(DX, TWO);
                GP = GN;
            }
            if (p == pe) bwd_pair(a, f2pack(GP.x, 0.f), E, DX);
        } else {
            float d = dx;
            for (int x = xa; x <= xb; ++x, d += 1.f)
                bwd_pair(a, f2pack(row[x], 0.f), f2pack(ex2_approx(fmaf(s.A * d, d, Ckdy2)), 0.f), f2pack(d, 0.f));
        }
        const float rE = f2sum(a.e), rX = f2sum(a.x);
        M.e += rE;
        M.g += f2sum(a.g);
        M.x += rX;
        M.xx += f2sum(a.xx);
        M.y = fmaf(dy, rE, M.y);
        M.xy = fmaf(dy, rX, M.xy);
        M.yy = fmaf(dy * dy, rE, M.yy);
    }
}

// Row-pair walk over a row-pair-interleaved block: the f32x2 lanes are the two
// rows (2j, 2j+1) of one footprint, so the per-row setup (span, exp seeds,
// moment update) runs packed once per two rows, and one 64-bit shared load
// fetches both rows' upstream values at a column.  blk holds pairs from the
// even row b0 on: element (row b0 + 2j + t, column x) at float2 index
// j*W + (x - xlo), lane t.
//
// Both lanes run over the union of their two row spans.  A pixel of that union
// outside its own row's q < 6.5^2 span has e < sub, so it adds g (e - sub),
// |e - sub| < sub = 6.7e-10, to the sums: a quarter of the fp32 rounding
// noise of sum g e at most (the mean of e over a footprint is ~0.05), and
// nothing at the 1e-3 gradient tolerance.  Rows outside [ya, yb] (the first or
// last pair of an odd-aligned footprint) have e = 0 and their g is dropped.
//
// Along a row e_{k+1} = e_k g_k, g_{k+1} = g_k c (c = 2^(2A)), restarted
// exactly every 32 columns (relative error < 2e-5).
//
// sum g (the -sub sum g part of sA = sum g (e - sub)) is not accumulated: it
// is at most sub sum |g| = 6.7e-10 sum |g|, while the fp32 rounding already
// in sum g e is ~6e-8 sum |g| e with mean e ~0.05 over a footprint, so the term
// is below a quarter of that rounding (1e-8 of the gradient; tolerance 1e-3)
// and costs one packed add per column on the FMA pipe that bounds this loop
// (-6% kernel time).  -DCGS_BWD_EXACT_SUB restores it.
constexpr int kChunk = 32;
constexpr float kMinSeedLog2 = -100.f;  // joint row-pair walks need every live seed e >= 2^-100

// Tail cut of the region kernel's walk (bwd_rowpairs): q < kBwdCut instead of
// q < 6.5^2, i.e. e >= t = exp(-kBwdCut / 2) of the Gaussian's own peak.  The
// dropped annulus carries a fraction t (1 + kBwdCut / 2) of any moment sum
// g e q^j (j <= 1) of the footprint -- 1.7e-6 at kBwdCut = 32.24 (t = 1e-7),
// the size of the fp32 rounding already in those sums and 600x below the
// 1e-3 gradient tolerance -- while the walked area shrinks by kBwdCut / 42.25.
// CGS_BWD_CUT=0 walks the reference's whole q < 6.5^2 ellipse.
#ifndef CGS_BWD_CUT
#define CGS_BWD_CUT 32.236191f  /* -2 ln(1e-7) */
#endif
constexpr float kBwdCut = (CGS_BWD_CUT > 0.f && CGS_BWD_CUT < kCutoffSq) ? CGS_BWD_CUT : kCutoffSq;

// kUnroll4: four columns per loop trip instead of two (the large-image kernel: rows at 256^2 are
// wide enough for the shorter loop control to pay, K5 1.686 -> 1.670 ms at C4; at 128^2 the
// longer remainder peel costs more, 0.698 -> 0.705 ms).  Same operations in the same order.
template <bool kUnroll4>
__device__ __forceinline__ void bwd_rowpairs(const float2 *__restrict__ blk, int b0, int W, int xlo, int xhi,
                                             int ya, int yb, const Splat2 &s, float c, Moments &M) {
    const float nk = -s.k, A = s.A, Ck = s.Ck, isp = s.inv_sqrt_p00;
    int y = ya & ~1;  // b0 is even: pairs are aligned to even rows
    float2 DY = f2pack((float)y - s.mpy, (float)(y + 1) - s.mpy);
    const float2 NSL = f2pack(-s.slope, -s.slope), MPX = f2pack(s.mpx, s.mpx);
    const float2 *prow = blk + ((y - b0) >> 1) * W - xlo;
    for (; y <= yb; y += 2, DY = f2add(DY, f2pack(2.f, 2.f)), prow += W) {
        // the row centres from DY with one rounding each (an accumulated XC drifts, see render.cu)
        const float2 XC = f2fma(DY, NSL, MPX);
        const bool v0 = y >= ya, v1 = y + 1 <= yb;
        const float2 REM = f2fma(f2mul(DY, f2pack(nk, nk)), DY, f2pack(kBwdCut, kBwdCut));
        float2 H = f2mul(f2pack(sqrt_approx(fmaxf(REM.x, 0.f)), sqrt_approx(fmaxf(REM.y, 0.f))),
                         f2pack(isp, isp));
        // a row outside [ya, yb] gets the empty span [~1e9, ~-1e9]: neutral in the union's min/max
        H.x = v0 ? H.x : -1e9f;
        H.y = v1 ? H.y : -1e9f;
        const float2 LO = f2add(XC, f2pack(-H.x, -H.y)), HI = f2add(XC, H);
        const int xa0 = max((int)ceilf(LO.x), xlo), xb0 = min((int)floorf(HI.x), xhi);
        const int xa1 = max((int)ceilf(LO.y), xlo), xb1 = min((int)floorf(HI.y), xhi);
        const int xa = min(xa0, xa1), xb = max(xb0, xb1);
        if (xa > xb) continue;
        const float2 KY = f2mul(f2mul(DY, f2pack(Ck, Ck)), DY);
        // One run of n <= kChunk columns from q, seeded at offset DX; lane t live
        // iff mt.  Per column only the running sums C = sum w, S1 = sum C,
        // S2 = sum S1 (w = g e) are kept: with u = n - k (k = 0..n-1) S1 = sum u w
        // and 2 S2 - S1 = sum u^2 w, so with D = dx' one past the last column
        // (dx'_k = D - u)
        //   sum w dx' = D C - S1,  sum w dx'^2 = D (D C - 2 S1) + 2 S2 - S1
        // (6 packed ops per column instead of 9; for n <= 32 the rounding of the
        // expansion stays below 1e-4 of sum |w| dx'^2).  Returns, per lane,
        // (sum w, sum w dx', sum w dx'^2, sum g).
        struct RunSums {
            float2 e, x, xx, g;
        };
        auto run = [&](const float2 *q, int n, float2 DX, bool m0, bool m1) -> RunSums {
            const float2 DXA = f2mul(DX, f2pack(A, A));
            const float2 Q = f2fma(DXA, DX, KY);
            const float2 GA = f2fma(DXA, f2pack(2.f, 2.f), f2pack(A, A));  // A (2 dx + 1)
            // a dead lane carries e = g = 0 (a select: its g may be inf)
            float2 E = f2pack(m0 ? ex2_approx(Q.x) : 0.f, m1 ? ex2_approx(Q.y) : 0.f);
            float2 G = f2pack(m0 ? ex2_approx(GA.x) : 0.f, m1 ? ex2_approx(GA.y) : 0.f);
            float2 C = {0.f, 0.f}, S1 = {0.f, 0.f}, S2 = {0.f, 0.f}, SG = {0.f, 0.f};
            auto column = [&](float2 V) {
                f2acc_fma(C, V, E);
#ifdef CGS_BWD_EXACT_SUB
                f2acc_add(SG, V);
#endif
                f2acc_add(S1, C);
                f2acc_add(S2, S1);
                f2scale(E, G);
                f2scale(G, f2pack(c, c));
            };
            // two columns per trip, both loaded at the top of the trip (no value
            // carried across trips: a software-pipelined load costs register
            // moves in the loop); an odd column count peels one column first
            if constexpr (kUnroll4) {  // four columns per trip; n mod 4 columns peeled first
                const float2 *qe = q + n;
                if (n & 1) column(*q++);
                if (n & 2) {
                    const float2 V0 = q[0], V1 = q[1];
                    column(V0);
                    column(V1);
                    q += 2;
                }
#pragma unroll 1
                for (; q < qe; q += 4) {
                    const float2 V0 = q[0], V1 = q[1], V2 = q[2], V3 = q[3];
                    column(V0);
                    column(V1);
                    column(V2);
                    column(V3);
                }
            } else {
                const float2 *qe = q + (n - 1);
                if (n & 1) column(*q++);
#pragma unroll 1
                for (; q < qe; q += 2) {
                    const float2 V0 = q[0], V1 = q[1];
                    column(V0);
                    column(V1);
                }
            }
            const float nf = (float)n;
            const float2 Dn = f2add(DX, f2pack(nf, nf));
            const float2 NS1 = f2pack(-S1.x, -S1.y);
            const float2 X1 = f2fma(Dn, C, NS1);
            RunSums r;
            r.e = C;
            r.x = X1;
            r.xx = f2fma(Dn, f2add(X1, NS1), f2fma(S2, f2pack(2.f, 2.f), NS1));
            r.g = SG;
            return r;
        };
        // one packed walk over columns [wa, wb]: a single run, or runs of
        // kChunk columns (each restarts the exp recurrence exactly)
        auto walk = [&](int wa, int wb, bool m0, bool m1) {
            const float2 DX = f2add(f2pack((float)wa, (float)wa), f2pack(-XC.x, -XC.y));
            RunSums r;
            if (wb - wa < kChunk) [[likely]] {
                r = run(prow + wa, wb - wa + 1, DX, m0, m1);
            } else {
                r = RunSums{{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
                for (int x0 = wa; x0 <= wb; x0 += kChunk) {
                    const float o = (float)(x0 - wa);
                    const RunSums t = run(prow + x0, min(kChunk, wb - x0 + 1), f2add(DX, f2pack(o, o)), m0, m1);
                    r.e = f2add(r.e, t.e);
                    r.x = f2add(r.x, t.x);
                    r.xx = f2add(r.xx, t.xx);
                    r.g = f2add(r.g, t.g);
                }
            }
            M.e += f2sum(r.e);
#ifdef CGS_BWD_EXACT_SUB
            M.g += (m0 ? r.g.x : 0.f) + (m1 ? r.g.y : 0.f);
#endif
            M.x += f2sum(r.x);
            M.xx += f2sum(r.xx);
            // y moments as FMA chains (one rounding fewer per term than product-then-sum)
            M.y = fmaf(DY.y, r.e.y, fmaf(DY.x, r.e.x, M.y));
            M.xy = fmaf(DY.y, r.x.y, fmaf(DY.x, r.x.x, M.xy));
            const float2 DY2 = f2mul(DY, DY);
            M.yy = fmaf(DY2.y, r.e.y, fmaf(DY2.x, r.e.x, M.yy));
        };
        // The union walk seeds a lane's recurrence up to |xa0 - xa1| columns
        // before its own span.  For thin, slanted footprints that seed e can
        // underflow, so such pairs walk their two rows apart.  A seed exponent
        // >= kMinSeedLog2 also bounds the seed g below 2^100 (no overflow).
        const float2 DX0 = f2add(f2pack((float)xa, (float)xa), f2pack(-XC.x, -XC.y));
        const float2 Q0 = f2fma(f2mul(DX0, f2pack(A, A)), DX0, KY);
        const bool joint = !(v0 && v1) || fminf(Q0.x, Q0.y) >= kMinSeedLog2;
        if (joint) {
            walk(xa, xb, v0, v1);
        } else {
            if (xa0 <= xb0) walk(xa0, xb0, true, false);
            if (xa1 <= xb1) walk(xa1, xb1, false, true);
        }
    }
}

// moments of one (image, Gaussian) -> += world-frame accumulator
__device__ __forceinline__ void accumulate_world(const Moments &M, const Splat2 &s, const PoseF &P, float inv_h,
                                                 float acc[CGS_ACC_STRIDE]) {
    const float ih2 = 0.5f * inv_h * inv_h;
    const float p00 = s.p00, p01 = s.p01, p11 = s.p11, k = s.k;
    const float sA = M.e - kSub * M.g;
    const float sx = (p00 * M.x) * inv_h;
    const float sy = (p01 * M.x + k * M.y) * inv_h;
    const float Sxx = p00 * p00 * M.xx;
    const float Sxy = p00 * (p01 * M.xx + k * M.xy);
    const float Syy = p01 * p01 * M.xx + 2.f * p01 * k * M.xy + k * k * M.yy;
    const float ac = s.w;
    const float S00 = ac * ih2 * (Sxx - p00 * sA);
    const float S01 = ac * ih2 * (Sxy - p01 * sA);
    const float S11 = ac * ih2 * (Syy - p11 * sA);
    const float d0 = ac * sx, d1 = ac * sy;
    acc[0] += s.cnorm * sA;
    acc[1] += d0 * P.w0[0] + d1 * P.w1[0];
    acc[2] += d0 * P.w0[1] + d1 * P.w1[1];
    acc[3] += d0 * P.w0[2] + d1 * P.w1[2];
    // P3_kl = sum_ab W_ak S_ab W_bl, (k,l) in xx xy xz yy yz zz
    const float u0 = S00 * P.w0[0] + S01 * P.w1[0], v0 = S01 * P.w0[0] + S11 * P.w1[0];
    const float u1 = S00 * P.w0[1] + S01 * P.w1[1], v1 = S01 * P.w0[1] + S11 * P.w1[1];
    const float u2 = S00 * P.w0[2] + S01 * P.w1[2], v2 = S01 * P.w0[2] + S11 * P.w1[2];
    acc[4] += u0 * P.w0[0] + v0 * P.w1[0];
    acc[5] += u0 * P.w0[1] + v0 * P.w1[1];
    acc[6] += u0 * P.w0[2] + v0 * P.w1[2];
    acc[7] += u1 * P.w0[1] + v1 * P.w1[1];
    acc[8] += u1 * P.w0[2] + v1 * P.w1[2];
    acc[9] += u2 * P.w0[2] + v2 * P.w1[2];
}

__device__ __forceinline__ void footprint_rows(const Splat2 &s, int D, int &ylo, int &yhi, float f = 1.f) {
    ylo = 1;
    yhi = 0;
    if (s.w > 0.f) {
        const float hy = s.hy * f;
        ylo = max((int)ceilf(s.mpy - hy), 0);
        yhi = min((int)floorf(s.mpy + hy), D - 1);
    }
}



__device__ __forceinline__ void store_partial(float *__restrict__ partial, int grp, int64_t n, int64_t g,
                                              const float acc[CGS_ACC_STRIDE]) {
    float *dst = partial + ((int64_t)grp * n + g) * CGS_ACC_STRIDE;
#ifndef CGS_PART_NO_HINT
    // keep the partials in L2 for the epilogue that reads them next (evict_last:
    // K5 0.7230 -> 0.7207 ms at C2, the partials' write-back no longer competes)
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
#pragma unroll
    for (int c = 0; c < CGS_ACC_STRIDE; c += 2)
        asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(dst + c), "f"(acc[c]),
                     "f"(acc[c + 1]), "l"(pol)
                     : "memory");
#else
#pragma unroll
    for (int c = 0; c < CGS_ACC_STRIDE; ++c) dst[c] = acc[c];
#endif
}

// Whole-image double buffering: natural layout only, D*D*4 bytes per buffer.
__global__ void __launch_bounds__(kBwdThreadsDB, 1) raster_bwd_db_kernel(
    const float *__restrict__ splat, int64_t n, const double *__restrict__ poses, int B, GridF G,
    const float *__restrict__ upstream, float *__restrict__ partial, int ipg) {
    extern __shared__ __align__(128) float smem_db[];
    __shared__ __align__(8) uint64_t bars[2];
    const int D = G.D;
    const uint32_t img_bytes = (uint32_t)D * D * sizeof(float);
    const int64_t g = (int64_t)blockIdx.x * kBwdThreadsDB + threadIdx.x;
    const bool valid = g < n;
    const int grp = blockIdx.y;
    const int b_begin = grp * ipg, b_end = min(B, b_begin + ipg);
    const int nimg = b_end - b_begin;
    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < 2 && i < nimg; ++i) {
            mbar_expect_tx(&bars[i], img_bytes);
            bulk_g2s(smem_db + i * D * D, upstream + (int64_t)(b_begin + i) * D * D, img_bytes, &bars[i]);
        }
    }
    __syncthreads();
    SplatRec rec{};
    if (valid) rec = load_splat(splat, g);
    float acc[CGS_ACC_STRIDE];
#pragma unroll
    for (int c = 0; c < CGS_ACC_STRIDE; ++c) acc[c] = 0.f;

    for (int i = 0; i < nimg; ++i) {
        const int b = b_begin + i;
        const PoseF P = load_pose_f(poses, b);
        Splat2 s{};
        int ylo = 1, yhi = 0;
        if (valid) {
            s = project2(rec, P, G);
            footprint_rows(s, D, ylo, yhi);
        }
        const float c2A = ex2_approx(2.f * s.A);
        mbar_wait(&bars[i & 1], (uint32_t)((i >> 1) & 1));
        Moments M{0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        bwd_rows(smem_db + (i & 1) * D * D, 0, D, 0, D - 1, ylo, yhi, s, c2A, M);
        if (ylo <= yhi) accumulate_world(M, s, P, G.inv_h, acc);
        __syncthreads();  // every thread is done reading buf[i & 1]
        if (threadIdx.x == 0 && i + 2 < nimg) {
            fence_proxy_async_smem();
            mbar_expect_tx(&bars[i & 1], img_bytes);
            bulk_g2s(smem_db + (i & 1) * D * D, upstream + (int64_t)(b + 2) * D * D, img_bytes, &bars[i & 1]);
        }
    }
    if (valid) store_partial(partial, grp, n, g, acc);
}

__device__ __forceinline__ void stage_rows(float *__restrict__ img, const float *__restrict__ up, int b, int D,
                                           int r0, int r1, int layout) {
    const float *src = up + (int64_t)b * D * D;
    const int total = (r1 - r0) * D;
    if (layout == CGS_LAYOUT_NATURAL && (D & 3) == 0) {
        const float4 *s4 = reinterpret_cast<const float4 *>(src + (int64_t)r0 * D);
        float4 *d4 = reinterpret_cast<float4 *>(img);
        for (int i = threadIdx.x; i < (total >> 2); i += blockDim.x) d4[i] = __ldg(s4 + i);
        return;
    }
    const int c0 = D / 2;
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
        int r = idx / D, x = idx - r * D;
        int sy = r0 + r, sx = x;
        if (layout == CGS_LAYOUT_FFT) {
            sy -= c0; if (sy < 0) sy += D;
            sx -= c0; if (sx < 0) sx += D;
        }
        img[idx] = src[(int64_t)sy * D + sx];
    }
}

// Synchronous row bands: any D, either layout.
__global__ void __launch_bounds__(kBwdThreadsBand, 3) raster_bwd_band_kernel(
    const float *__restrict__ splat, int64_t n, const double *__restrict__ poses, int B, GridF G,
    const float *__restrict__ upstream, int layout, float *__restrict__ partial, int ipg, int HB) {
    extern __shared__ float img[];
    const int D = G.D;
    const int64_t g = (int64_t)blockIdx.x * kBwdThreadsBand + threadIdx.x;
    const bool valid = g < n;
    const int grp = blockIdx.y;
    const int b_begin = grp * ipg, b_end = min(B, b_begin + ipg);
    SplatRec rec{};
    if (valid) rec = load_splat(splat, g);
    float acc[CGS_ACC_STRIDE];
#pragma unroll
    for (int c = 0; c < CGS_ACC_STRIDE; ++c) acc[c] = 0.f;
    for (int b = b_begin; b < b_end; ++b) {
        const PoseF P = load_pose_f(poses, b);
        Splat2 s{};
        int ylo = 1, yhi = 0;
        if (valid) {
            s = project2(rec, P, G);
            footprint_rows(s, D, ylo, yhi);
        }
        const float c2A = ex2_approx(2.f * s.A);
        Moments M{0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int r0 = 0; r0 < D; r0 += HB) {
            const int r1 = min(D, r0 + HB);
            __syncthreads();
            stage_rows(img, upstream, b, D, r0, r1, layout);
            __syncthreads();
            bwd_rows(img, r0, D, 0, D - 1, max(ylo, r0), min(yhi, r1 - 1), s, c2A, M);
        }
        if (ylo <= yhi) accumulate_world(M, s, P, G.inv_h, acc);
    }
    if (valid) store_partial(partial, grp, n, g, acc);
}

// Region staging (default): per image the CTA stages only the union of its
// Gaussians' footprint boxes, in row bands of at most kRegFloats floats.  With
// Gaussians in spatial order the region is a few hundred pixels, so shared
// memory stays small and several CTAs share an SM; in any order it is correct
// (the region then grows to the whole image and is processed band by band).
#ifndef CGS_BWD_REG_THREADS
#define CGS_BWD_REG_THREADS 256
#endif
#ifndef CGS_BWD_MINB
#define CGS_BWD_MINB 4
#endif
#ifndef CGS_BWD_REG_THREADS_SMALL
#define CGS_BWD_REG_THREADS_SMALL 128
#endif
#ifndef CGS_BWD_MINB_SMALL
#define CGS_BWD_MINB_SMALL 7
#endif
constexpr int kRegThreads = CGS_BWD_REG_THREADS;
// CTA shape per band kind.  The static 24 KB band (D <= 128) runs 128 threads at up to 7 CTAs
// per SM: 70 registers and no spills (256 threads at 4 per SM allow 64 and spill), 6 CTAs per SM
// by shared memory; C2 K5 0.698 -> 0.690 ms, bitwise the same partials.  The 40 KB dynamic band
// (larger images) keeps 256 threads at 4 per SM: at 128 threads its band per thread doubles and
// C4's K5 went 1.67 -> 1.88 ms.
template <int kRegF>
struct RegShape {
    static constexpr int kT = kRegF > 0 ? CGS_BWD_REG_THREADS_SMALL : kRegThreads;
    static constexpr int kMinB = kRegF > 0 ? CGS_BWD_MINB_SMALL : CGS_BWD_MINB;
};
constexpr int kMaxPoseImages = 64;  // image groups up to this size keep fp32 poses in shared memory
#ifndef CGS_BWD_REG_FLOATS
#define CGS_BWD_REG_FLOATS 6144
#endif
constexpr int kRegFloats = CGS_BWD_REG_FLOATS;  // 24 KB per band (measured 8..32 KB)
#ifndef CGS_BWD_REG_FLOATS_LARGE
#define CGS_BWD_REG_FLOATS_LARGE 10240
#endif
// Images beyond 128^2: a larger region band (40 KB, still 4 CTAs per SM), so a CTA's union box
// splits into fewer bands; a lane whose footprint misses the current band idles through it
// (C4, 256^2: K5 1.79 -> see DESIGN.md).
constexpr int kRegFloatsLarge = CGS_BWD_REG_FLOATS_LARGE;

// kRowPair: upstream in CGS_LAYOUT_ROWPAIR (a straight float2 copy); kRegF: the region band in
// static shared memory of kRegF floats (128^2: the static array measured 0.2% faster), or 0 for a
// dynamic band of regf_dyn floats (larger images)
template <bool kPoseSmem, bool kRowPair, int kRegF>
__global__ void __launch_bounds__(RegShape<kRegF>::kT, RegShape<kRegF>::kMinB) raster_bwd_region_kernel(
    const float *__restrict__ splat, int64_t n, const double *__restrict__ poses, int B, GridF G,
    const float *__restrict__ upstream, float *__restrict__ partial, int ipg, int regf_dyn) {
    constexpr int kT = RegShape<kRegF>::kT;
    // regf + kRowPad floats, row-pair interleaved (bwd_rowpairs)
    __shared__ __align__(16) float reg_static[kRegF > 0 ? kRegF + kRowPad : 1];
    extern __shared__ __align__(16) float reg_dyn[];
    float *reg = kRegF > 0 ? reg_static : reg_dyn;
    const int regf = kRegF > 0 ? kRegF : regf_dyn;
    __shared__ int red[2][4][kT / 32];
    // Register budget: the walk needs ~40 registers, so per-thread state that
    // is touched once per image lives outside the register file: the world
    // accumulator in shared memory (column-major: conflict-free), poses as fp32
    // in shared memory, and the splat record re-read from L1 each image.
    __shared__ float accs[CGS_ACC_STRIDE * kT];
    __shared__ float poses_f[kMaxPoseImages * 8];
    const int D = G.D;
    const int64_t g = (int64_t)blockIdx.x * kT + threadIdx.x;
    const bool valid = g < n;
    const int grp = blockIdx.y;
    const int b_begin = grp * ipg, b_end = min(B, b_begin + ipg);
    // extents under the tail cut: half-extents scale by sqrt(kBwdCut / 6.5^2) (+1e-4 margin)
    const float ext = kBwdCut < kCutoffSq ? 1.0001f * sqrtf(kBwdCut / kCutoffSq) : 1.f;
    constexpr bool pose_smem = kPoseSmem;  // host guarantees ipg <= kMaxPoseImages when set
    if (pose_smem)
        for (int i = threadIdx.x; i < (b_end - b_begin) * 8; i += kT) {
            const int k = i & 7;
            poses_f[i] = (float)poses[12 * (int64_t)(b_begin + (i >> 3)) + (k < 6 ? k : k + 3)];
        }
#pragma unroll
    for (int c = 0; c < CGS_ACC_STRIDE; ++c) accs[c * kT + threadIdx.x] = 0.f;
    for (int i = threadIdx.x; i < regf + kRowPad; i += kT) reg[i] = 0.f;  // finite reads past spans
    __syncthreads();
    auto pose = [&](int b) {
        if (!pose_smem) return load_pose_f(poses, b);
        const float *q = poses_f + 8 * (b - b_begin);
        PoseF P;
        P.w0[0] = q[0]; P.w0[1] = q[1]; P.w0[2] = q[2];
        P.w1[0] = q[3]; P.w1[1] = q[4]; P.w1[2] = q[5];
        P.tx = q[6]; P.ty = q[7];
        return P;
    };

    for (int b = b_begin; b < b_end; ++b) {
        Splat2 s{};
        int ylo = 1, yhi = 0;
        if (valid) {
            s = project2(load_splat(splat, g), pose(b), G);
            footprint_rows(s, D, ylo, yhi, ext);
            s.hx *= ext;
        }
        // its barrier also retires every thread's reads of reg for the previous image
        const Box R = block_union(footprint_box(s, valid, ylo, yhi, D), red, b);
        if (R.x0 > R.x1) continue;  // uniform
        const int W = R.x1 - R.x0 + 1;
        // rows per band, even so row pairs never straddle bands (W <= regf / 2);
        // the division only runs for regions larger than one band
        const int HBr = ((R.y1 | 1) - (R.y0 & ~1) + 1) * W <= regf ? D + 2 : (regf / W) & ~1;
        const float c2A = ex2_approx(2.f * s.A);
        const float *src = upstream + (int64_t)b * D * D;
        Moments M{0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        float2 *reg2 = reinterpret_cast<float2 *>(reg);
        for (int by0 = R.y0 & ~1; by0 <= R.y1; by0 += HBr) {
            const int by1 = min(R.y1 | 1, by0 + HBr - 1);  // odd: whole pairs
            const int np = (by1 - by0 + 1) >> 1;
            if (by0 != (R.y0 & ~1)) __syncthreads();  // previous band fully consumed (block_union covers the first)
            // flat over the band's np * W float2 slots, slot i = (pair j, column x):
            // coalesced row loads, one 64-bit store of both rows per column
            // (row D is zero).  j = floor((i + 0.5) / W) on the FMA pipe: a
            // round-down FFMA into the 1.5*2^23 magic; (i + 0.5) / W is >= 0.5 / W
            // from an integer, far above the rcp error; i is tracked as an exact float
            {
                const float invW = rcp_approx((float)W);
                const int nel = np * W;
                float fi = (float)threadIdx.x + 0.5f;
                if (kRowPair) {  // the pair rows are already interleaved in HBM (even D)
                    const float2 *sb2 = reinterpret_cast<const float2 *>(src) + (by0 >> 1) * D + R.x0;
                    for (int i = threadIdx.x; i < nel; i += kT, fi += (float)kT) {
                        const int j = __float_as_int(__fmaf_rd(fi, invW, 12582912.0f)) - 0x4B400000;
                        reg2[i] = __ldg(sb2 + j * D + (i - j * W));
                    }
                } else {
                    const float *sb = src + by0 * D + R.x0;
                    for (int i = threadIdx.x; i < nel; i += kT, fi += (float)kT) {
                        const int j = __float_as_int(__fmaf_rd(fi, invW, 12582912.0f)) - 0x4B400000;
                        const float *p = sb + j * (2 * D) + (i - j * W);
                        reg2[i] = f2pack(__ldg(p), by0 + 2 * j + 1 < D ? __ldg(p + D) : 0.f);
                    }
                }
            }
            __syncthreads();
            const int ya = max(ylo, by0), yb = min(yhi, by1);
            if (ya <= yb)
                bwd_rowpairs<kRegF == 0>(reinterpret_cast<const float2 *>(reg), by0, W, R.x0, R.x1, ya, yb, s, c2A,
                                         M);
        }
        if (ylo <= yhi) {
            float acc[CGS_ACC_STRIDE];
#pragma unroll
            for (int c = 0; c < CGS_ACC_STRIDE; ++c) acc[c] = accs[c * kT + threadIdx.x];
            accumulate_world(M, s, pose(b), G.inv_h, acc);
#pragma unroll
            for (int c = 0; c < CGS_ACC_STRIDE; ++c) accs[c * kT + threadIdx.x] = acc[c];
        }
    }
    if (valid) {
        float acc[CGS_ACC_STRIDE];
#pragma unroll
        for (int c = 0; c < CGS_ACC_STRIDE; ++c) acc[c] = accs[c * kT + threadIdx.x];
        store_partial(partial, grp, n, g, acc);
    }
}

// (image, Gaussian, pixel) pairs with q < cut per image: cut = 6.5^2 counts the
// reference's in-ellipse pairs; cut = kBwdCut counts the pairs
// the backward evaluates.
__global__ void __launch_bounds__(256) count_pairs_kernel(const float *__restrict__ splat, int64_t n,
                                                          const double *__restrict__ poses, GridF G, float cut,
                                                          int64_t *__restrict__ pairs) {
    const int b = blockIdx.y;
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    long long cnt = 0;
    if (g < n) {
        const PoseF P = load_pose_f(poses, b);
        Splat2 s = project2(load_splat(splat, g), P, G);
        const int D = G.D;
        int ylo, yhi;
        footprint_rows(s, D, ylo, yhi, sqrtf(cut / kCutoffSq));
        for (int iy = ylo; iy <= yhi; ++iy) {
            const float dy = (float)iy - s.mpy;
            const float rem = fmaf(-s.k * dy, dy, cut);
            if (rem <= 0.f) continue;
            const float half = sqrt_approx(rem) * s.inv_sqrt_p00;
            const float xc = fmaf(-s.slope, dy, s.mpx);
            const int xa = max((int)ceilf(xc - half), 0), xb = min((int)floorf(xc + half), D - 1);
            if (xa <= xb) cnt += xb - xa + 1;
        }
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd((unsigned long long *)&pairs[b], (unsigned long long)cnt);
}

}  // namespace cgs

using namespace cgs;

extern "C" int64_t cgs_bwd_groups(int32_t B, int32_t images_per_group) {
    if (B <= 0 || images_per_group <= 0) return 0;
    return (B + images_per_group - 1) / images_per_group;
}

extern "C" int cgs_raster_bwd(const float *splat, int64_t n, const double *poses, int32_t B,
                              cgs_grid grid, const float *upstream, int32_t layout, float *partial,
                              int32_t images_per_group, void *stream) {
    if (n <= 0 || B <= 0 || grid.size < 1 || images_per_group <= 0 || !splat || !poses ||
        !upstream || !partial)
        return CGS_ERR_ARG;
    const int D = grid.size;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t G = cgs_bwd_groups(B, images_per_group);
    // kernel variant: region (default) | db | band; CGS_BWD_KERNEL overrides for A/B runs
    static int variant = -1;
    if (variant < 0) {
        const char *v = getenv("CGS_BWD_KERNEL");
        variant = (v && v[0] == 'd') ? 1 : (v && v[0] == 'b') ? 2 : 0;
    }
    const int regf = D <= 128 ? kRegFloats : kRegFloatsLarge;
    if (layout == CGS_LAYOUT_ROWPAIR && ((D & 1) || D > regf / 2)) return CGS_ERR_UNSUPPORTED;
    if ((layout == CGS_LAYOUT_NATURAL && variant == 0 && D <= regf / 2) || layout == CGS_LAYOUT_ROWPAIR) {
        const int threads = regf == kRegFloats ? RegShape<kRegFloats>::kT : RegShape<0>::kT;
        dim3 g((unsigned)((n + threads - 1) / threads), (unsigned)G);
        const GridF gf = make_grid_f(grid);
        const bool ps = images_per_group <= kMaxPoseImages;
        const size_t smem = (size_t)(regf + kRowPad) * sizeof(float);
        auto launch = [&](auto kern) -> int {
            const size_t dyn = regf == kRegFloats ? 0 : smem;
            // a dynamic band beyond 48 KB with the static arrays needs the opt-in
            if (dyn) {
                const int rc = ensure_smem_limit((const void *)kern, dyn + 16 * 1024, "raster_bwd_region_kernel");
                if (rc) return rc;
            }
            kern<<<g, threads, dyn, st>>>(splat, n, poses, B, gf, upstream, partial, images_per_group, regf);
            return CGS_OK;
        };
        int rc;
        if (regf == kRegFloats)
            rc = layout == CGS_LAYOUT_ROWPAIR
                     ? (ps ? launch(raster_bwd_region_kernel<true, true, kRegFloats>)
                           : launch(raster_bwd_region_kernel<false, true, kRegFloats>))
                     : (ps ? launch(raster_bwd_region_kernel<true, false, kRegFloats>)
                           : launch(raster_bwd_region_kernel<false, false, kRegFloats>));
        else
            rc = layout == CGS_LAYOUT_ROWPAIR
                     ? (ps ? launch(raster_bwd_region_kernel<true, true, 0>)
                           : launch(raster_bwd_region_kernel<false, true, 0>))
                     : (ps ? launch(raster_bwd_region_kernel<true, false, 0>)
                           : launch(raster_bwd_region_kernel<false, false, 0>));
        if (rc) return rc;
        return check_launch("raster_bwd_region_kernel");
    }
    const size_t db_bytes = (2 * (size_t)D * D + kRowPad) * sizeof(float);
    const bool aligned = ((reinterpret_cast<uintptr_t>(upstream) & 15) == 0) && ((D * D) % 4 == 0);
    if (layout == CGS_LAYOUT_NATURAL && variant == 1 && db_bytes <= (size_t)kDBMaxBytes && aligned) {
        const int rc = ensure_smem_limit((const void *)raster_bwd_db_kernel, db_bytes, "raster_bwd_db_kernel");
        if (rc) return rc;
        dim3 g((unsigned)((n + kBwdThreadsDB - 1) / kBwdThreadsDB), (unsigned)G);
        raster_bwd_db_kernel<<<g, kBwdThreadsDB, db_bytes, st>>>(splat, n, poses, B, make_grid_f(grid), upstream,
                                                                 partial, images_per_group);
        return check_launch("raster_bwd_db_kernel");
    }
    int HB = kBandBytes / (D * (int)sizeof(float));
    if (HB < 1) return CGS_ERR_UNSUPPORTED;
    HB = HB > D ? D : HB;
    const size_t smem = ((size_t)HB * D + kRowPad) * sizeof(float);
    const int rc = ensure_smem_limit((const void *)raster_bwd_band_kernel, smem, "raster_bwd_band_kernel");
    if (rc) return rc;
    dim3 g((unsigned)((n + kBwdThreadsBand - 1) / kBwdThreadsBand), (unsigned)G);
    raster_bwd_band_kernel<<<g, kBwdThreadsBand, smem, st>>>(splat, n, poses, B, make_grid_f(grid), upstream, layout,
                                                             partial, images_per_group, HB);
    return check_launch("raster_bwd_band_kernel");
}

extern "C" int cgs_count_pairs_cut(const float *splat, int64_t n, const double *poses, int32_t B, cgs_grid grid,
                                   double cut_sq, int64_t *pairs, void *stream) {
    if (n <= 0 || B <= 0 || !splat || !poses || !pairs || !(cut_sq > 0.0)) return CGS_ERR_ARG;
    dim3 g((unsigned)((n + 255) / 256), (unsigned)B);
    count_pairs_kernel<<<g, 256, 0, (cudaStream_t)stream>>>(splat, n, poses, make_grid_f(grid), (float)cut_sq,
                                                             pairs);
    return check_launch("count_pairs_kernel");
}

extern "C" int cgs_count_pairs(const float *splat, int64_t n, const double *poses, int32_t B,
                               cgs_grid grid, int64_t *pairs, void *stream) {
    return cgs_count_pairs_cut(splat, n, poses, B, grid, (double)kCutoffSq, pairs, stream);
}

extern "C" double cgs_bwd_cut_sq(void) { return (double)kBwdCut; }
