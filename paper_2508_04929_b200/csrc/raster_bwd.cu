// K5: fused backward, the B200 replacement of backward_pixels
// (_kernels.py:128-190) plus the per-image part of rasterize_backward
// (splat.py:332-349), batched over images.
//
// Gaussian-major and atomic-free: a CTA owns kGPC Gaussians and a group of
// images.  For each image it stages the upstream gradient (natural layout,
// padded rows) in shared memory; each Gaussian is handled by kLPG lanes, lane
// i walking rows i, i+kLPG, ... of the footprint along the exact q < 6.5^2
// row span.  Per pixel it accumulates seven moments of g*e in pixel units
// (sum ge, sum g, sum ge dx, ge dx^2 and per row ge dy, ge dx dy, ge dy^2),
// which carry the reference's six raw sums exactly:
//   sA = sum ge - sub sum g,  s_ab = 1/(2h^2) (sum ge pd_a pd_b - p_ab sA), ...
// The kLPG lanes reduce them with xor shuffles, convert them to the
// image-summable 10-float world-frame accumulator
//   {cnorm sA, W2^T ac (sx, sy), W2^T (ac S) W2}
// and add it to a per-CTA shared accumulator that exactly one lane group owns.
// The CTA writes its image group's partial once; cgs_epilogue_* sums groups in
// a fixed order, so the gradient is bitwise reproducible.
#include "common.cuh"

namespace cgs {

constexpr int kLPG = 8;                  // lanes per Gaussian
constexpr int kGPW = 32 / kLPG;          // Gaussians per warp per pass
constexpr int kBwdThreads = 256;
constexpr int kGPC = 256;                // Gaussians per CTA
constexpr int kBandBytes = 96 * 1024;    // upstream rows staged per band

__device__ __forceinline__ void stage_rows(float *__restrict__ img, const float *__restrict__ up,
                                           int b, int D, int r0, int r1, int layout) {
    const int ld = D + 1, c0 = D / 2;
    const int total = (r1 - r0) * D;
    const float *src = up + (int64_t)b * D * D;
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
        int r = idx / D, x = idx - r * D;
        int iy = r0 + r;
        int sy = iy, sx = x;
        if (layout == CGS_LAYOUT_FFT) {
            sy = iy - c0; if (sy < 0) sy += D;
            sx = x - c0; if (sx < 0) sx += D;
        }
        img[r * ld + x] = src[(int64_t)sy * D + sx];
    }
}

__global__ void __launch_bounds__(kBwdThreads) raster_bwd_kernel(
    const float *__restrict__ splat, int64_t n, const double *__restrict__ poses, int B, GridF G,
    const float *__restrict__ upstream, int layout, float *__restrict__ partial, int ipg, int HB) {
    extern __shared__ float sm[];
    const int D = G.D, ld = D + 1;
    float *img = sm;
    float *acc = sm + HB * ld;
    const int64_t g0 = (int64_t)blockIdx.x * kGPC;
    const int grp = blockIdx.y;
    const int b_begin = grp * ipg, b_end = min(B, b_begin + ipg);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sub = lane / kLPG, li = lane % kLPG;
    for (int i = threadIdx.x; i < kGPC * CGS_ACC_STRIDE; i += blockDim.x) acc[i] = 0.f;

    for (int b = b_begin; b < b_end; ++b) {
        const PoseF P = load_pose_f(poses, b);
        for (int r0 = 0; r0 < D; r0 += HB) {
            const int r1 = min(D, r0 + HB);
            __syncthreads();
            stage_rows(img, upstream, b, D, r0, r1, layout);
            __syncthreads();
            for (int k = warp * kGPW + sub; k < kGPC; k += (kBwdThreads / 32) * kGPW) {
                const int64_t g = g0 + k;
                Splat2 s{};
                int ylo = 1, yhi = 0;
                if (g < n) {
                    s = project2(load_splat(splat, g), P, G);
                    if (s.w > 0.f) {
                        ylo = max(max((int)ceilf(s.mpy - s.hy), r0), 0);
                        yhi = min(min((int)floorf(s.mpy + s.hy), r1 - 1), D - 1);
                    }
                }
                float Me = 0.f, Mg = 0.f, Mx = 0.f, My = 0.f, Mxx = 0.f, Mxy = 0.f, Myy = 0.f;
                for (int iy = ylo + li; iy <= yhi; iy += kLPG) {
                    const float dy = (float)iy - s.mpy;
                    // exact span of q < cutoff on this row:
                    // p00 dx^2 + 2 (p01 dy) dx + (p11 dy^2 - cut) < 0
                    const float bq = s.p01 * dy;
                    const float cq = fmaf(s.p11 * dy, dy, -kCutoffSq);
                    const float disc = fmaf(bq, bq, -s.p00 * cq);
                    if (disc <= 0.f) continue;
                    const float root = sqrtf(disc);
                    const float inv = 1.f / s.p00;
                    const int xa = max((int)ceilf(s.mpx + (-bq - root) * inv), 0);
                    const int xb = min((int)floorf(s.mpx + (-bq + root) * inv), D - 1);
                    const float Bdy = s.Bc * dy, Cdy2 = s.C * dy * dy;
                    const float *row = img + (iy - r0) * ld;
                    float rE = 0.f, rG = 0.f, rX = 0.f;
                    float dx = (float)xa - s.mpx;
                    for (int x = xa; x <= xb; ++x) {
                        const float e = ex2_approx(fmaf(fmaf(s.A, dx, Bdy), dx, Cdy2));
                        const float gp = row[x];
                        const float ge = gp * e;
                        rE += ge;
                        rG += gp;
                        const float tq = ge * dx;
                        rX += tq;
                        Mxx = fmaf(tq, dx, Mxx);
                        dx += 1.f;
                    }
                    Me += rE;
                    Mg += rG;
                    Mx += rX;
                    My = fmaf(dy, rE, My);
                    Mxy = fmaf(dy, rX, Mxy);
                    Myy = fmaf(dy * dy, rE, Myy);
                }
#pragma unroll
                for (int o = kLPG / 2; o > 0; o >>= 1) {
                    Me += __shfl_xor_sync(0xffffffffu, Me, o);
                    Mg += __shfl_xor_sync(0xffffffffu, Mg, o);
                    Mx += __shfl_xor_sync(0xffffffffu, Mx, o);
                    My += __shfl_xor_sync(0xffffffffu, My, o);
                    Mxx += __shfl_xor_sync(0xffffffffu, Mxx, o);
                    Mxy += __shfl_xor_sync(0xffffffffu, Mxy, o);
                    Myy += __shfl_xor_sync(0xffffffffu, Myy, o);
                }
                if (ylo <= yhi) {
                    // moments -> the reference's raw sums (normalised units)
                    const float ih2 = 0.5f * G.inv_h * G.inv_h;
                    const float p00 = s.p00, p01 = s.p01, p11 = s.p11;
                    const float sA = Me - kSub * Mg;
                    const float sx = (p00 * Mx + p01 * My) * G.inv_h;
                    const float sy = (p01 * Mx + p11 * My) * G.inv_h;
                    const float Sxx = p00 * p00 * Mxx + 2.f * p00 * p01 * Mxy + p01 * p01 * Myy;
                    const float Sxy = p00 * p01 * Mxx + (p00 * p11 + p01 * p01) * Mxy + p01 * p11 * Myy;
                    const float Syy = p01 * p01 * Mxx + 2.f * p01 * p11 * Mxy + p11 * p11 * Myy;
                    const float ac = s.w;
                    const float S00 = ac * ih2 * (Sxx - p00 * sA);
                    const float S01 = ac * ih2 * (Sxy - p01 * sA);
                    const float S11 = ac * ih2 * (Syy - p11 * sA);
                    const float d0 = ac * sx, d1 = ac * sy;
                    float *a = acc + k * CGS_ACC_STRIDE;
#pragma unroll
                    for (int c = li; c < CGS_ACC_STRIDE; c += kLPG) {
                        float v;
                        switch (c) {
                            case 0: v = s.cnorm * sA; break;
                            case 1: v = d0 * P.w0[0] + d1 * P.w1[0]; break;
                            case 2: v = d0 * P.w0[1] + d1 * P.w1[1]; break;
                            case 3: v = d0 * P.w0[2] + d1 * P.w1[2]; break;
                            default: {
                                // P3_kl = sum_ab W_ak S_ab W_bl for (k,l) in xx xy xz yy yz zz
                                const int kk = (c == 4 || c == 5 || c == 6) ? 0 : (c == 9 ? 2 : 1);
                                const int ll = (c == 4) ? 0 : (c == 5 || c == 7) ? 1 : 2;
                                v = S00 * P.w0[kk] * P.w0[ll] +
                                    S01 * (P.w0[kk] * P.w1[ll] + P.w1[kk] * P.w0[ll]) +
                                    S11 * P.w1[kk] * P.w1[ll];
                            }
                        }
                        a[c] += v;
                    }
                }
            }
        }
    }
    __syncthreads();
    const int64_t cnt = min((int64_t)kGPC, n - g0);
    float *dst = partial + ((int64_t)grp * n + g0) * CGS_ACC_STRIDE;
    for (int64_t i = threadIdx.x; i < cnt * CGS_ACC_STRIDE; i += blockDim.x) dst[i] = acc[i];
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
                const float dy = (float)iy - s.mpy;
                const float bq = s.p01 * dy;
                const float cq = fmaf(s.p11 * dy, dy, -kCutoffSq);
                const float disc = fmaf(bq, bq, -s.p00 * cq);
                if (disc <= 0.f) continue;
                const float root = sqrtf(disc), inv = 1.f / s.p00;
                const int xa = max((int)ceilf(s.mpx + (-bq - root) * inv), 0);
                const int xb = min((int)floorf(s.mpx + (-bq + root) * inv), D - 1);
                if (xb >= xa) cnt += xb - xa + 1;
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
    int HB = kBandBytes / ((D + 1) * (int)sizeof(float));
    if (HB < 1) return CGS_ERR_UNSUPPORTED;
    HB = HB > D ? D : HB;
    size_t smem = ((size_t)HB * (D + 1) + (size_t)kGPC * CGS_ACC_STRIDE) * sizeof(float);
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
