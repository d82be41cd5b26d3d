// K3 (training path): binning-free forward render with deterministic
// fixed-point shared-memory accumulation.
//
// The reference renders tile by tile from per-tile Gaussian lists
// (build_tile_work + forward_tiles, _kernels.py:17-125).  On B200 the faster
// schedule for ~1 px footprints is Gaussian-major, like the backward: one
// lane per (image, Gaussian) walks its own footprint along the exact
// q < 6.5^2 row spans and adds w (e - sub) into a shared-memory image.  Lanes
// of a warp hit unrelated pixels, so the adds must be atomic; shared-memory
// float atomics are CAS loops on sm_100a (3 updates/clk/SM measured), native
// int32 ATOMS.ADD sustain ~10/clk/SM at random addresses
// (profiles/microbench_smem_atomics_r01.txt).  Values are therefore added as
// round-to-nearest int32 fixed point with one scale per step:
//   scale = 2^30 / sum_g wb_g,   wb_g >= w_g(b) for every view b,
// so no pixel sum can overflow, and integer addition makes the render
// bitwise reproducible regardless of scheduling.  One ulp is sum wb / 2^30,
// ~1e-6 of the image's total peak weight (render tolerance is 1e-4 rel L2).
//
// wb_g: by eigenvalue interlacing the projected 2x2 covariance has
// lambda1 >= s_mid^2 and lambda2 >= s_min^2; with the eigenvalue floor
// (0.1 px)^2 (splat.py:207-209) det >= max(s_mid^2, f) max(s_min^2, f), so
// w = amp / (2 pi sqrt(det)) <= amp / (2 pi sqrt(that)).
//
// Along a row, e = exp(-q/2) follows e_{k+1} = e_k g_k, g_{k+1} = g_k c with
// c = 2^(2A): two FMULs per pixel instead of an MUFU.EX2, restarted every 32
// pixels so the recurrence error stays below 2e-5.  Rounding to int uses the
// FMA-pipe magic-number trick (common.cuh fast_rint) instead of F2I on the XU.
#include <algorithm>
#include <cmath>

#include "common.cuh"

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
constexpr int kWbBlock = 1024;
constexpr float kFixedRange = 1073741824.f;  // 2^30
constexpr float kContribRange = 4194304.f;   // 2^22

__global__ void __launch_bounds__(kWbBlock) wbound_partial_kernel(const float *__restrict__ splat, int64_t n,
                                                                  double h, float *__restrict__ part) {
    const int64_t g = blockIdx.x * (int64_t)kWbBlock + threadIdx.x;
    float wb = 0.f;
    if (g < n) {
        const float *r = splat + g * CGS_SPLAT_STRIDE;
        const double s0 = r[13], s1 = r[14], s2 = r[15], amp = r[3];
        const double lo = fmin(s0, fmin(s1, s2)), hi = fmax(s0, fmax(s1, s2));
        const double mid = s0 + s1 + s2 - lo - hi;
        const double fl = (0.1 * h) * (0.1 * h);
        const double det = fmax(mid * mid, fl) * fmax(lo * lo, fl);
        // 1.001: headroom for the fp32 evaluation of w inside the kernels
        wb = (float)(1.001 * amp / (2.0 * kPiD * sqrt(det)));
    }
    __shared__ float ws[kWbBlock / 32], wm[kWbBlock / 32];
    float v = warp_sum(wb), m = wb;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) {
        ws[threadIdx.x >> 5] = v;
        wm[threadIdx.x >> 5] = m;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        float t = warp_sum(ws[threadIdx.x]), mm = wm[threadIdx.x];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mm = fmaxf(mm, __shfl_xor_sync(0xffffffffu, mm, o));
        if (threadIdx.x == 0) {
            part[blockIdx.x] = t;
            part[gridDim.x + blockIdx.x] = mm;
        }
    }
}

// scale = min(2^30 / sum wb, 2^22 / max wb) -> part[2 nparts]; fixed-order
// reduction.  The first bound keeps every pixel sum below 2^30; the second
// keeps every single contribution below 2^22, where fast_rint is exact.
__global__ void __launch_bounds__(256) wbound_scale_kernel(float *part, int nparts) {
    __shared__ double ws[8];
    __shared__ float wm[8];
    double t = 0.0;
    float m = 0.f;
    for (int i = threadIdx.x; i < nparts; i += 256) {
        t += part[i];
        m = fmaxf(m, part[nparts + i]);
    }
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
    if (threadIdx.x == 0) {
        double s = 0.0;
        float mx = 0.f;
        for (int w = 0; w < 8; ++w) {
            s += ws[w];
            mx = fmaxf(mx, wm[w]);
        }
        double sc = s > 0.0 ? (double)kFixedRange / s : 1.0;
        if (mx > 0.f) sc = fmin(sc, (double)kContribRange / mx);
        part[2 * nparts] = (float)sc;
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
template <bool kRecur>
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
    // integer fix-up.  The -wS sub term (< 0.003 units per contribution for
    // wS <= 2^22) is below the rounding of each contribution and is dropped.
    const float A2 = 2.f * s.A, nHcut = -kHalfL2e * cut - 74.f, xhiM = kM + (float)xhi;
    const float wSd = wS * 0x1p-75f;
    const float2 WS = f2pack(wSd, wSd);
    float dy = (float)ya - s.mpy;
    float xcv = fmaf(-s.slope, dy, s.mpx);
    int *row = acc + (ya - r0) * ld;
    for (int nr = yb - ya; nr >= 0; --nr, dy += 1.f, xcv -= s.slope, row += ld) {
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
                const float2 v = f2mul_keep_denorm(WS, E);
                atomicAdd(row + x, __float_as_int(v.x));
                atomicAdd(row + x + 1, __float_as_int(v.y));
                f2scale(E, R);
                f2scale(R, C4);
            }
            if (x == xb) atomicAdd(row + x, __float_as_int(fmul_keep_denorm(wSd, E.x)));
        } else {
            float d = dx;
            for (int x = xa; x <= xb; ++x, d += 1.f)
                atomicAdd(row + x, __float_as_int(fmul_keep_denorm(wSd, ex2_approx(fmaf(s.A * d, d, Ckdy2)))));
        }
    }
}

// CTA = (chunk of kRChunk Gaussians, image, band of rows); the band's int32
// accumulator (whole 128^2 image in 64 KB) lives in shared memory and is
// added to the global image once at the end.  Lanes of a warp must hit
// unrelated pixels to keep ATOMS conflicts rare, but the device order of the
// Gaussians is spatial (Morton, chosen for the backward's region staging), so
// the chunk visits Gaussians in a scrambled order: logical index i maps to
// g = (i * A) mod n with gcd(A, n) = 1, stepped incrementally.
__global__ void __launch_bounds__(kRThreads, CGS_FWD_MINB) raster_fwd_atomic_kernel(
    const float *__restrict__ splat, int64_t n, const double *__restrict__ poses, GridF G,
    const float *__restrict__ scale_ptr, int HB, int64_t mulA, int chunk, int *__restrict__ out) {
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
    const float scale = *scale_ptr;
    const PoseF P = load_pose_f(poses, b);
    const int64_t i_begin = (int64_t)blockIdx.x * chunk;
    const int64_t i_end = min(n, i_begin + chunk);
    const int64_t stepA = (kRThreads * mulA) % n;
    int64_t g = ((i_begin + threadIdx.x) % n) * mulA % n;
    __syncthreads();
    for (int64_t i = i_begin + threadIdx.x; i < i_end; i += kRThreads) {
        const Splat2 s = project2(load_splat(splat, g), P, G);
        g += stepA;
        if (g >= n) g -= n;
        if (!(s.w > 0.f)) continue;
        // Contribution-exact footprint: a pixel adds round(wS e) units, which is
        // 0 wherever e < 0.5 / wS.  Walk only q < cut with e(cut) = 0.4995 / wS
        // (the 1e-3 margin keeps every pixel that can round to >= 1 unit) and
        // q < 6.5^2: the same integer image as the whole culled ellipse, far
        // fewer updates.
        const float thr = fmaxf(0.4995f * rcp_approx(s.w * scale), kSub);  // >= sub: no denormals
        if (!(thr < 1.f)) continue;
        const float cut = fminf(kCutoffSq, -2.f * kLn2 * lg2_approx(thr));
        const float hy = s.hy * sqrt_approx(cut * (1.f / kCutoffSq));
        const int ylo = max(max((int)ceilf(s.mpy - hy), 0), r0);
        const int yhi = min(min((int)floorf(s.mpy + hy), D - 1), r1 - 1);
        if (ylo > yhi) continue;
        // widest row = 2 sqrt(cut / p00) = 2 * 6.5 sqrt(cut / 6.5^2) / sqrt(p00)
        if (13.f * sqrt_approx(cut * (1.f / kCutoffSq)) * s.inv_sqrt_p00 < 31.f)
            fwd_rows_band<true>(band, r0, ld, D - 1, ylo, yhi, s, scale, cut);
        else
            fwd_rows_band<false>(band, r0, ld, D - 1, ylo, yhi, s, scale, cut);
    }
    __syncthreads();
    int *dst = out + (int64_t)b * D * D + (int64_t)r0 * D;
    for (int i = threadIdx.x; i < npx; i += kRThreads) {
        const int v = band[i];
        if (v) atomicAdd(dst + i, v);
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

extern "C" size_t cgs_render_workspace_bytes(int64_t n) {
    int64_t parts = (n + kWbBlock - 1) / kWbBlock;
    return (size_t)(2 * parts + 1) * sizeof(float);
}

static int render_impl(const float *splat, int64_t n, const double *poses, int32_t B, cgs_grid grid, float *out,
                          void *ws, void *stream, bool convert) {
    if (n <= 0 || B <= 0 || grid.size < 1 || !splat || !poses || !out || !ws) return CGS_ERR_ARG;
    const int D = grid.size;
    cudaStream_t st = (cudaStream_t)stream;
    const int parts = (int)((n + kWbBlock - 1) / kWbBlock);
    float *part = (float *)ws;
    const double h = 2.0 * grid.extent / grid.size;
    wbound_partial_kernel<<<parts, kWbBlock, 0, st>>>(splat, n, h, part);
    wbound_scale_kernel<<<1, 256, 0, st>>>(part, parts);
    int HB = kRBandBytes / (D * (int)sizeof(int));
    if (HB < 1) return CGS_ERR_UNSUPPORTED;
    HB = HB > D ? D : HB;
    const int bands = (D + HB - 1) / HB;
    const size_t smem = (size_t)HB * D * sizeof(int);
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        cudaFuncSetAttribute(raster_fwd_atomic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = smem;
    }
    const int64_t count = (int64_t)B * D * D;
    cudaMemsetAsync(out, 0, sizeof(int) * count, st);
    thread_local int slots = 0;
    thread_local size_t slots_smem = 0;
    if (slots == 0 || slots_smem != smem) {
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, raster_fwd_atomic_kernel, kRThreads, smem);
        slots = std::max(1, sms * per_sm);
        slots_smem = smem;
    }
    int64_t nchunks = fwd_chunks(n, (int64_t)B * bands, slots);
    const int chunk = (int)((n + nchunks - 1) / nchunks);
    nchunks = (n + chunk - 1) / chunk;
    dim3 g((unsigned)nchunks, (unsigned)B, (unsigned)bands);
    raster_fwd_atomic_kernel<<<g, kRThreads, smem, st>>>(splat, n, poses, make_grid_f(grid), part + 2 * parts, HB,
                                                         scramble_multiplier(n), chunk, reinterpret_cast<int *>(out));
    int rc = check_launch("raster_fwd_atomic_kernel");
    if (rc || !convert) return rc;
    const int64_t threads = (count + 3) / 4;
    fixed_to_float_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(reinterpret_cast<int *>(out), count,
                                                                           part + 2 * parts);
    return check_launch("fixed_to_float_kernel");
}

extern "C" int cgs_render(const float *splat, int64_t n, const double *poses, int32_t B, cgs_grid grid, float *out,
                          void *ws, void *stream) {
    return render_impl(splat, n, poses, B, grid, out, ws, stream, true);
}

extern "C" int cgs_render_fixed(const float *splat, int64_t n, const double *poses, int32_t B, cgs_grid grid,
                                int32_t *out, void *ws, void *stream) {
    return render_impl(splat, n, poses, B, grid, reinterpret_cast<float *>(out), ws, stream, false);
}

extern "C" int64_t cgs_render_scale_offset(int64_t n) { return 2 * ((n + kWbBlock - 1) / kWbBlock); }
