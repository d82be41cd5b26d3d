// Shared device helpers for the sm_100a cryoGS kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "cgs_b200.h"

namespace cgs {

constexpr double kCullSigma = 6.5;                 // splat.py:49
constexpr double kCutoffSqD = kCullSigma * kCullSigma;
constexpr float kCutoffSq = 42.25f;
constexpr double kPiD = 3.14159265358979323846;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr float kEigenFloorPx2 = 0.01f;            // (EIGEN_FLOOR_FRACTION * h)^2 / h^2, splat.py:55
// sub = exp(-cutoff_sq / 2) (splat.py:51) as the fp32 boundary value
constexpr float kSub = 6.6915861e-10f;
// the same boundary in log2 units: log2(sub) = -21.125 * log2(e)
constexpr float kL2Cut = -21.125f * 1.4426950408889634f;

void set_error_detail(const char *what, const char *detail);
int check_launch(const char *what);
// per-device dynamic shared-memory opt-in (cudaFuncSetAttribute) for func, checked
int ensure_smem_limit(const void *func, size_t bytes, const char *what);
// SMs x resident CTAs of func on the current device, memoised per (device, func)
int resident_slots(const void *func, int threads, size_t smem, int *slots, const char *what);

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float lg2_approx(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float sqrt_approx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// one MUFU each, no denormal fix-up code (projection inputs are >= (0.1 px)^2)
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float rsqrt_approx(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Image-independent geometry of one Gaussian, written by cgs_prepare:
// rec[0..2] mean, rec[3] amp, rec[4..12] M = R diag(s) row-major.
struct SplatRec {
    float mx, my, mz, amp;
    float M[9];
};

__device__ __forceinline__ SplatRec load_splat(const float *__restrict__ splat, int64_t g) {
    const float4 *p = reinterpret_cast<const float4 *>(splat + g * CGS_SPLAT_STRIDE);
    float4 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2), d = __ldg(p + 3);
    SplatRec r;
    r.mx = a.x; r.my = a.y; r.mz = a.z; r.amp = a.w;
    r.M[0] = b.x; r.M[1] = b.y; r.M[2] = b.z; r.M[3] = b.w;
    r.M[4] = c.x; r.M[5] = c.y; r.M[6] = c.z; r.M[7] = c.w;
    r.M[8] = d.x;
    return r;
}

// Pose of one image in fp32 for the raster kernels: rows 0/1 of W and t.
struct PoseF {
    float w0[3], w1[3], tx, ty;
};

__device__ __forceinline__ PoseF load_pose_f(const double *__restrict__ poses, int b) {
    const double *p = poses + 12 * (int64_t)b;
    PoseF q;
    q.w0[0] = (float)p[0]; q.w0[1] = (float)p[1]; q.w0[2] = (float)p[2];
    q.w1[0] = (float)p[3]; q.w1[1] = (float)p[4]; q.w1[2] = (float)p[5];
    q.tx = (float)p[9]; q.ty = (float)p[10];
    return q;
}

// Grid constants in the units the raster kernels use (pixels).
struct GridF {
    int D;
    float c0;      // origin pixel index D//2
    float inv_h;   // 1 / pixel_width
    float inv_2pi_h2;  // 1 / (2 pi h^2): cnorm in normalised units from a px^2 det
};

__host__ __forceinline__ GridF make_grid_f(const cgs_grid &g) {
    GridF f;
    f.D = g.size;
    f.c0 = (float)(g.size / 2);
    double h = 2.0 * g.extent / g.size;
    f.inv_h = (float)(1.0 / h);
    f.inv_2pi_h2 = (float)(1.0 / (2.0 * kPiD * h * h));
    return f;
}

// Screen-space Gaussian of one (image, Gaussian) pair in pixel units: the
// fp32 restatement of _Projection.__init__ (splat.py:184-226) and
// _clamp_eigenvalues (splat.py:229-260).
//   q(dx, dy) = p00 dx^2 + 2 p01 dx dy + p11 dy^2, d = pixel - mean  [pixels]
//   l = -q/2 * log2(e) = A dx^2 + Bc dx dy + C dy^2   (exp(-q/2) = 2^l)
//
// Rows are walked in row-conditional coordinates: on pixel row dy the
// ellipse is centred at x_c(dy) = mpx - (p01/p00) dy and, with dx' = x - x_c,
//   q = p00 dx'^2 + k dy^2,   k = p11 - p01^2/p00 = 1/c11,
// a sum of two non-negative terms.  Expanding (p00 dx + p01 dy)^2 instead
// cancels catastrophically in fp32 for thin diagonal footprints.
struct Splat2 {
    float mpx, mpy;        // mean in pixel-index coordinates
    float p00, p01, p11;   // precision in px^-2
    float A, Bc, C;        // log2-scaled quadratic form: l = A dx^2 + Bc dx dy + C dy^2
    float slope;           // p01 / p00: x_c(dy) = mpx - slope * dy
    float k, Ck;           // k = 1/c11 [px^-2]; Ck = -log2(e)/2 * k
    float inv_sqrt_p00;    // row half-span = sqrt((cut - k dy^2) / p00)
    float cnorm;           // 1 / (2 pi sqrt(det)) in normalised units
    float w;               // amp * cnorm
    float hx, hy;          // half-extents of the q < cutoff ellipse [px]
    int clamped;           // 1 when the small eigenvalue hit the floor (CLAMP_EVENTS, splat.py:277)
};

// fast approximate rcp/sqrt (MUFU, ~1 ulp): the raster tolerances are 1e-4/1e-3
__device__ __forceinline__ Splat2 project2(const SplatRec &r, const PoseF &P, const GridF &G) {
    Splat2 s;
    // B2 = W[:2] M, mean2 = W[:2] mu + t  (splat.py:197-200), in pixel units
    float b0[3], b1[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        b0[j] = (P.w0[0] * r.M[j] + P.w0[1] * r.M[3 + j] + P.w0[2] * r.M[6 + j]) * G.inv_h;
        b1[j] = (P.w1[0] * r.M[j] + P.w1[1] * r.M[3 + j] + P.w1[2] * r.M[6 + j]) * G.inv_h;
    }
    s.mpx = (P.w0[0] * r.mx + P.w0[1] * r.my + P.w0[2] * r.mz + P.tx) * G.inv_h + G.c0;
    s.mpy = (P.w1[0] * r.mx + P.w1[1] * r.my + P.w1[2] * r.mz + P.ty) * G.inv_h + G.c0;
    // cov2 = B2 B2^T (splat.py:202-206); det by Cauchy-Binet (sum of squared
    // 2x2 minors) so thin footprints keep full relative precision
    float c00 = b0[0] * b0[0] + b0[1] * b0[1] + b0[2] * b0[2];
    float c01 = b0[0] * b1[0] + b0[1] * b1[1] + b0[2] * b1[2];
    float c11 = b1[0] * b1[0] + b1[1] * b1[1] + b1[2] * b1[2];
    float m01 = b0[0] * b1[1] - b0[1] * b1[0];
    float m02 = b0[0] * b1[2] - b0[2] * b1[0];
    float m12 = b0[1] * b1[2] - b0[2] * b1[1];
    float det = m01 * m01 + m02 * m02 + m12 * m12;
    float mid = 0.5f * (c00 + c11);
    float hd = 0.5f * (c00 - c11);
    float rad = sqrt_approx(hd * hd + c01 * c01);
    float l1 = mid + rad;
    float l2 = l1 > 0.f ? det * rcp_approx(l1) : 0.f;
    s.clamped = l2 < kEigenFloorPx2;
    if (s.clamped) {
        // floor the small eigenvalue, keep the eigenvector (splat.py:245-259)
        float a1 = fmaxf(l1, kEigenFloorPx2), a2 = kEigenFloorPx2;
        float vx = c01, vy = l1 - c00;
        float ux = l1 - c11, uy = c01;
        if (ux * ux + uy * uy > vx * vx + vy * vy) { vx = ux; vy = uy; }
        float nn2 = vx * vx + vy * vy;
        if (nn2 == 0.f) { vx = 1.f; vy = 0.f; } else { const float inn = rsqrt_approx(nn2); vx *= inn; vy *= inn; }
        c00 = a1 * vx * vx + a2 * vy * vy;
        c01 = (a1 - a2) * vx * vy;
        c11 = a1 * vy * vy + a2 * vx * vx;
        det = a1 * a2;
    }
    float inv_det = rcp_approx(det);
    s.p00 = c11 * inv_det;
    s.p01 = -c01 * inv_det;
    s.p11 = c00 * inv_det;
    s.cnorm = G.inv_2pi_h2 * rsqrt_approx(det);
    s.w = r.amp * s.cnorm;
    s.A = -0.5f * kLog2e * s.p00;
    s.Bc = -kLog2e * s.p01;
    s.C = -0.5f * kLog2e * s.p11;
    s.hx = sqrt_approx(kCutoffSq * c00);
    s.hy = sqrt_approx(kCutoffSq * c11);
    s.slope = s.p01 * rcp_approx(s.p00);
    s.k = rcp_approx(c11);
    s.Ck = -0.5f * kLog2e * s.k;
    s.inv_sqrt_p00 = rsqrt_approx(s.p00);
    return s;
}

// Pixel span [xa, xb] of row dy (clipped to [xlo, xhi]) inside q < cutoff,
// and the row-conditional offset dx' of xa.  Returns false for an empty row.
__device__ __forceinline__ bool row_span(const Splat2 &s, float dy, int xlo, int xhi, int &xa, int &xb,
                                         float &dxa) {
    const float rem = fmaf(-s.k * dy, dy, kCutoffSq);
    if (rem <= 0.f) return false;
    // approximate sqrt: a boundary pixel it might flip carries ~sub of the peak
    const float half = sqrt_approx(rem) * s.inv_sqrt_p00;
    const float xc = fmaf(-s.slope, dy, s.mpx);
    xa = max((int)ceilf(xc - half), xlo);
    xb = min((int)floorf(xc + half), xhi);
    dxa = (float)xa - xc;
    return xa <= xb;
}

// ---- footprint boxes and their CTA-wide union -----------------------------
// With Gaussians in spatial (Morton) order, the footprints of a CTA's
// Gaussians in one image cover a small region, so the kernels stage (or
// accumulate into) only that region of the image in shared memory.
struct Box {
    int x0, x1, y0, y1;  // inclusive pixel bounds; empty when x0 > x1
};

__device__ __forceinline__ Box footprint_box(const Splat2 &s, bool live, int ylo, int yhi, int D) {
    Box b{0x7fffffff, -1, 0x7fffffff, -1};
    if (live && ylo <= yhi) {
        b.x0 = max((int)floorf(s.mpx - s.hx) - 1, 0);
        b.x1 = min((int)ceilf(s.mpx + s.hx) + 1, D - 1);
        b.y0 = ylo;
        b.y1 = yhi;
    }
    return b;
}

// Union of every thread's box.  red is shared scratch [2][4][warps] used in
// two halves by call parity, so one barrier per call suffices:
// the half written now was last read two calls ago, before the previous call's
// barrier.  That barrier also orders everything each thread did before the
// call ahead of everything after it (callers rely on it).  Needs blockDim <= 1024.
template <int NW>  // warps per CTA
__device__ __forceinline__ Box block_union(const Box &b, int (&red)[2][4][NW], int parity) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int x0 = __reduce_min_sync(0xffffffffu, b.x0), y0 = __reduce_min_sync(0xffffffffu, b.y0);
    const int x1 = __reduce_max_sync(0xffffffffu, b.x1), y1 = __reduce_max_sync(0xffffffffu, b.y1);
    int (&rr)[4][NW] = red[parity & 1];
    if (lane == 0) {
        rr[0][warp] = x0;
        rr[1][warp] = x1;
        rr[2][warp] = y0;
        rr[3][warp] = y1;
    }
    __syncthreads();
    const bool in = lane < NW;
    const int l = in ? lane : 0;
    Box r;
    r.x0 = __reduce_min_sync(0xffffffffu, in ? rr[0][l] : 0x7fffffff);
    r.x1 = __reduce_max_sync(0xffffffffu, in ? rr[1][l] : -1);
    r.y0 = __reduce_min_sync(0xffffffffu, in ? rr[2][l] : 0x7fffffff);
    r.y1 = __reduce_max_sync(0xffffffffu, in ? rr[3][l] : -1);
    return r;
}

// ---- packed f32x2 arithmetic (sm_100a FFMA2 / FMUL2 / FADD2) --------------
// One instruction updates two fp32 lanes: same FMA-pipe throughput as two
// FFMAs but half the issue slots (profiles/microbench_ffma2_r01.txt), which
// is what the issue-bound pixel loops need.  CUDA 12.8+ intrinsics on float2.
__device__ __forceinline__ float2 f2pack(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 f2mul(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 f2add(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ void f2acc_add(float2 &acc, float2 a) { acc = __fadd2_rn(acc, a); }
__device__ __forceinline__ void f2acc_fma(float2 &acc, float2 a, float2 b) { acc = __ffma2_rn(a, b, acc); }
__device__ __forceinline__ void f2scale(float2 &a, float2 b) { a = __fmul2_rn(a, b); }

// Multiplies whose results are meant to be denormal (render.cu: integer
// contributions as denormal bit patterns): explicit non-FTZ PTX, so a -ftz=true
// or --use_fast_math build cannot flush them to zero.
__device__ __forceinline__ float2 f2mul_keep_denorm(float2 a, float2 b) {
    unsigned long long ua, ub, ud;
    memcpy(&ua, &a, 8);
    memcpy(&ub, &b, 8);
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(ud) : "l"(ua), "l"(ub));
    float2 d;
    memcpy(&d, &ud, 8);
    return d;
}
__device__ __forceinline__ float fmul_keep_denorm(float a, float b) {
    float d;
    asm("mul.rn.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}
__device__ __forceinline__ float f2sum(float2 v) { return v.x + v.y; }

// float -> nearest int32 on the FMA/ALU pipes (no F2I on the XU pipe):
// valid for |x| < 2^22; returns round-to-nearest-even(x).
__device__ __forceinline__ int fast_rint(float x) {
    return __float_as_int(x + 12582912.0f) - 0x4B400000;
}

// ---- mbarrier + 1D bulk async copy (TMA engine), CTA scope ----------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global -> shared bulk copy of `bytes` (multiple of 16, 16B-aligned), completing on `bar`
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// order this thread's prior generic-proxy shared accesses before async-proxy writes
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// A step whose parameters were non-finite (cgs_prepare sets CGS_STATUS_NONFINITE_PARAMS)
// reports a NaN loss, as the reference's fp64 render of such a mixture would
// (train.py:146-149 -> DivergenceError); the loss kernels pass each image's
// loss through this before they store it.
__device__ __forceinline__ double poison_loss(double l, const int32_t *status) {
    if (status && (*(volatile const int32_t *)status & CGS_STATUS_NONFINITE_PARAMS)) return __longlong_as_double(0x7ff8000000000000ll);
    return l;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace cgs
