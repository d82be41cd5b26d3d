// K5: fused backward, the B200 replacement of backward_pixels
// (_kernels.py:128-190) plus the per-image part of rasterize_backward
// (splat.py:332-349), batched over images.
//
// Gaussian-major, one lane per (image, Gaussian), atomic-free.  A CTA owns
// kGPC Gaussians (one per thread) and a group of images; for each image it
// stages the upstream gradient in shared memory, and every thread walks its
// own Gaussian's footprint row by row along the exact q < 6.5^2 span.  Same-
// size footprints keep the warp's lanes in near lockstep, so no lane sits idle
// on another lane's rows and no cross-lane reduction is needed.  Per pixel it
// accumulates moments of ge = g e in pixel units:
//   per row:   sum ge, sum g, sum ge dx, sum ge dx^2
//   per image: + dy-weighted row sums -> 7 moments
// which carry the reference's six raw sums exactly
//   sA = sum ge - sub sum g,   s_ab = 1/(2 h^2) (sum ge pd_a pd_b - p_ab sA),
// then converts them, in registers, to the image-summable 10-float world-frame
// accumulator {cnorm sA, W2^T ac (sx, sy), W2^T (ac S) W2} (SURVEY.md 8(a)
// row 15) and keeps summing that over the CTA's images.  The CTA writes its
// image group's partial once; the epilogue sums groups in fixed order, so the
// gradient is bitwise reproducible.
#include "common.cuh"

namespace cgs {

constexpr int kBwdThreads = 256;
constexpr int kGPC = kBwdThreads;        // Gaussians per CTA, one per thread
constexpr int kBandBytes = 96 * 1024;    // upstream rows staged per band

__device__ __forceinline__ void stage_rows(float *__restrict__ img, const float *__restrict__ up,
                                           int b, int D, int r0, int r1, int layout) {
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

struct Moments {
    float e, g, x, y, xx, xy, yy;
};

// one pixel of the row walk in row-conditional coordinates (common.cuh):
// e = 2^l, l = A dx'^2 + Ck dy^2
__device__ __forceinline__ void bwd_pixel(float gp, float dx, float A, float Ckdy2,
                                          float &rE, float &rG, float &rX, float &rXX) {
    const float e = ex2_approx(fmaf(A * dx, dx, Ckdy2));
    const float ge = gp * e;
    rE += ge;
    rG += gp;
    const float t = ge * dx;
    rX += t;
    rXX = fmaf(t, dx, rXX);
}

__global__ void __launch_bounds__(kBwdThreads, 2) raster_bwd_kernel(
    const float *__restrict__ splat, int64_t n, const double *__restrict__ poses, int B, GridF G,
    const float *__restrict__ upstream, int layout, float *__restrict__ partial, int ipg, int HB) {
    extern __shared__ float img[];
    const int D = G.D;
    const int64_t g = (int64_t)blockIdx.x * kGPC + threadIdx.x;
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
            if (s.w > 0.f) {
                ylo = max((int)ceilf(s.mpy - s.hy), 0);
                yhi = min((int)floorf(s.mpy + s.hy), D - 1);
            }
        }
        Moments M{0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int r0 = 0; r0 < D; r0 += HB) {
            const int r1 = min(D, r0 + HB);
            __syncthreads();
            stage_rows(img, upstream, b, D, r0, r1, layout);
            __syncthreads();
            const int ya = max(ylo, r0), yb = min(yhi, r1 - 1);
            for (int iy = ya; iy <= yb; ++iy) {
                const float dy = (float)iy - s.mpy;
                int xa, xb;
                float dx;
                if (!row_span(s, dy, 0, D - 1, xa, xb, dx)) continue;
                const float Ckdy2 = s.Ck * dy * dy;
                const float *row = img + (iy - r0) * D;
                float rE = 0.f, rG = 0.f, rX = 0.f, rXX = 0.f, rE2 = 0.f, rG2 = 0.f, rX2 = 0.f, rXX2 = 0.f;
                int x = xa;
                for (; x < xb; x += 2) {  // two independent chains per iteration
                    bwd_pixel(row[x], dx, s.A, Ckdy2, rE, rG, rX, rXX);
                    bwd_pixel(row[x + 1], dx + 1.f, s.A, Ckdy2, rE2, rG2, rX2, rXX2);
                    dx += 2.f;
                }
                if (x == xb) bwd_pixel(row[x], dx, s.A, Ckdy2, rE, rG, rX, rXX);
                M.xx += rXX + rXX2;
                rE += rE2;
                rG += rG2;
                rX += rX2;
                M.e += rE;
                M.g += rG;
                M.x += rX;
                M.y = fmaf(dy, rE, M.y);
                M.xy = fmaf(dy, rX, M.xy);
                M.yy = fmaf(dy * dy, rE, M.yy);
            }
        }
        if (ylo <= yhi) {
            // moments -> the reference's raw sums (normalised units), then the
            // world-frame accumulator for this image
            const float ih2 = 0.5f * G.inv_h * G.inv_h;
            const float p00 = s.p00, p01 = s.p01, p11 = s.p11;
            // row-conditional moments: (P d)_x = p00 dx', (P d)_y = p01 dx' + k dy
            const float k = s.k;
            const float sA = M.e - kSub * M.g;
            const float sx = (p00 * M.x) * G.inv_h;
            const float sy = (p01 * M.x + k * M.y) * G.inv_h;
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
    }
    if (valid) {
        float *dst = partial + ((int64_t)grp * n + g) * CGS_ACC_STRIDE;
#pragma unroll
        for (int c = 0; c < CGS_ACC_STRIDE; ++c) dst[c] = acc[c];
    }
}

// In-ellipse pair count per image (same row spans as the backward).
__global__ void __launch_bounds__(256) count_pairs_kernel(const float *__restrict__ splat, int64_t n,
                                                          const double *__restrict__ poses, GridF G,
                                                          int64_t *__restrict__ pairs) {
    const int b = blockIdx.y;
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    long long cnt = 0;
    if (g < n) {
        const PoseF P = load_pose_f(poses, b);
        Splat2 s = project2(load_splat(splat, g), P, G);
        const int D = G.D;
        int ylo = max((int)ceilf(s.mpy - s.hy), 0), yhi = min((int)floorf(s.mpy + s.hy), D - 1);
        if (s.w > 0.f) {
            for (int iy = ylo; iy <= yhi; ++iy) {
                int xa, xb;
                float dx;
                if (row_span(s, (float)iy - s.mpy, 0, D - 1, xa, xb, dx)) cnt += xb - xa + 1;
            }
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
    int HB = kBandBytes / (D * (int)sizeof(float));
    if (HB < 1) return CGS_ERR_UNSUPPORTED;
    HB = HB > D ? D : HB;
    size_t smem = (size_t)HB * D * sizeof(float);
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        cudaFuncSetAttribute(raster_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = smem;
    }
    int64_t G = cgs_bwd_groups(B, images_per_group);
    dim3 g((unsigned)((n + kGPC - 1) / kGPC), (unsigned)G);
    raster_bwd_kernel<<<g, kBwdThreads, smem, (cudaStream_t)stream>>>(
        splat, n, poses, B, make_grid_f(grid), upstream, layout, partial, images_per_group, HB);
    return check_launch("raster_bwd_kernel");
}

extern "C" int cgs_count_pairs(const float *splat, int64_t n, const double *poses, int32_t B,
                               cgs_grid grid, int64_t *pairs, void *stream) {
    if (n <= 0 || B <= 0 || !splat || !poses || !pairs) return CGS_ERR_ARG;
    dim3 g((unsigned)((n + 255) / 256), (unsigned)B);
    count_pairs_kernel<<<g, 256, 0, (cudaStream_t)stream>>>(splat, n, poses, make_grid_f(grid), pairs);
    return check_launch("count_pairs_kernel");
}
