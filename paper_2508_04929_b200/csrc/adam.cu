// K6: per-Gaussian epilogue and Adam.
// Replaces the per-Gaussian chain of rasterize_backward (splat.py:344-381),
// the isotropic tie (train.py:157-159) and AdamState.update (train.py:101-111).
//
// Input is the 10-float world-frame accumulator summed over images
// {a, dmean (3), P (xx xy xz yy yz zz)}: dM = 2 P M with M = R diag(s)
// image-independent, so the chain runs once per Gaussian per step instead of
// once per (image, Gaussian).  fp64 throughout (parameters and moments are
// fp64 master copies, so tiny late-epoch updates survive as in the reference).
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include <algorithm>

#include "common.cuh"

namespace cgs {

__device__ __forceinline__ double softplus_e(double x) { return fmax(x, 0.0) + log1p(exp(-fabs(x))); }
__device__ __forceinline__ double sigmoid_e(double x) {
    double e = exp(-fabs(x));  // gmm.py:83-88
    return x >= 0.0 ? 1.0 / (1.0 + e) : e / (1.0 + e);
}

// The transcendental part of the chain for one Gaussian (softplus / sigmoid of
// the scales, sigmoid of the amplitude, the normalised quaternion): gmm.py:76-124.
struct ChainPre {
    double s[3], sig[3], sig_amp, inv, w, x, y, z;
};

__device__ __forceinline__ void chain_pre_scale(const double *__restrict__ raw, int j, double &s, double &sig) {
    s = softplus_e(raw[3 + j]);
    sig = sigmoid_e(raw[3 + j]);
}

__device__ __forceinline__ void chain_pre_quat(const double *__restrict__ raw, ChainPre &c) {
    double qw = raw[6], qx = raw[7], qy = raw[8], qz = raw[9];
    double qnorm = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
    bool ok = qnorm > 0.0 && isfinite(qnorm);
    double inv = ok ? 1.0 / qnorm : 0.0;
    c.inv = inv;
    c.w = ok ? qw * inv : 1.0;
    c.x = qx * inv;
    c.y = qy * inv;
    c.z = qz * inv;
}

// grads[11] = scale * chain(acc) from the transcendentals (splat.py:344-381)
__device__ __forceinline__ void chain_post(const ChainPre &c, const double acc[10], double scale, int mode,
                                           double out[11]) {
    const double w = c.w, x = c.x, y = c.y, z = c.z, inv = c.inv;
    const double *s = c.s, *sig = c.sig;
    double R[9];
    R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z);     R[2] = 2 * (x * z + w * y);
    R[3] = 2 * (x * y + w * z);     R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
    R[6] = 2 * (x * z - w * y);     R[7] = 2 * (y * z + w * x);     R[8] = 1 - 2 * (x * x + y * y);
    double P[9] = {acc[4], acc[5], acc[6], acc[5], acc[7], acc[8], acc[6], acc[8], acc[9]};
    // dM = 2 P M, M = R diag(s)
    double dM[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            dM[3 * i + j] = 2.0 * (P[3 * i] * R[j] + P[3 * i + 1] * R[3 + j] + P[3 * i + 2] * R[6 + j]) * s[j];
    double dscale[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) dscale[j] = R[j] * dM[j] + R[3 + j] * dM[3 + j] + R[6 + j] * dM[6 + j];
    double r[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) r[3 * i + j] = dM[3 * i + j] * s[j];
    // d R(qn) / d qn contracted with dR (splat.py:351-372)
    double d0 = 2 * (-z * r[1] + y * r[2] + z * r[3] - x * r[5] - y * r[6] + x * r[7]);
    double d1 = 2 * (y * r[1] + z * r[2] + y * r[3] - 2 * x * r[4] - w * r[5] + z * r[6] + w * r[7] - 2 * x * r[8]);
    double d2 = 2 * (-2 * y * r[0] + x * r[1] + w * r[2] + x * r[3] + z * r[5] - w * r[6] + z * r[7] - 2 * y * r[8]);
    double d3 = 2 * (-2 * z * r[0] - w * r[1] + x * r[2] + w * r[3] - 2 * z * r[4] + y * r[5] + x * r[6] + y * r[7]);
    double dot = d0 * w + d1 * x + d2 * y + d3 * z;  // splat.py:374
    out[0] = scale * acc[1];
    out[1] = scale * acc[2];
    out[2] = scale * acc[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) out[3 + j] = scale * dscale[j] * sig[j];
    out[6] = scale * (d0 - dot * w) * inv;
    out[7] = scale * (d1 - dot * x) * inv;
    out[8] = scale * (d2 - dot * y) * inv;
    out[9] = scale * (d3 - dot * z) * inv;
    out[10] = scale * acc[0] * c.sig_amp;
    if (mode == CGS_MODE_ISOTROPIC) {  // train.py:157-159
        double t = out[3] + out[4] + out[5];
        out[3] = out[4] = out[5] = t;
    }
}

// grads[11] = scale * chain(acc) for one Gaussian
__device__ void chain_grads(const double *__restrict__ raw, const double acc[10], double scale,
                            int mode, double out[11]) {
    ChainPre c;
#pragma unroll
    for (int j = 0; j < 3; ++j) chain_pre_scale(raw, j, c.s[j], c.sig[j]);
    chain_pre_quat(raw, c);
    c.sig_amp = sigmoid_e(raw[10]);
    chain_post(c, acc, scale, mode, out);
}

__device__ __forceinline__ void sum_groups(const float *__restrict__ part, int G, int64_t n,
                                           int64_t g, double acc[10]) {
#pragma unroll
    for (int c = 0; c < 10; ++c) acc[c] = 0.0;
    // groups in order (fixed fp64 summation order), loads issued 4 groups ahead as
    // 8-byte vectors: the kernel is bound by the latency of these 52 MB of reads
    const float2 *base = reinterpret_cast<const float2 *>(part + g * CGS_ACC_STRIDE);
    const int64_t gstride = n * (CGS_ACC_STRIDE / 2);
    int k = 0;
    for (; k + 4 <= G; k += 4) {
        float2 v[4][5];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int c = 0; c < 5; ++c) v[u][c] = __ldg(base + (k + u) * gstride + c);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int c = 0; c < 5; ++c) {
                acc[2 * c] += (double)v[u][c].x;
                acc[2 * c + 1] += (double)v[u][c].y;
            }
    }
    for (; k < G; ++k)
#pragma unroll
        for (int c = 0; c < 5; ++c) {
            const float2 w = __ldg(base + k * gstride + c);
            acc[2 * c] += (double)w.x;
            acc[2 * c + 1] += (double)w.y;
        }
}

// AdamState.update for one element, operation order as train.py:103-111
__device__ __forceinline__ void adam_elem(double &p, double g, double &m, double &v, double lr,
                                          double b1, double b2, double eps, double bc1, double bc2) {
    m = __dadd_rn(__dmul_rn(m, b1), __dmul_rn(1.0 - b1, g));
    v = __dadd_rn(__dmul_rn(v, b2), __dmul_rn(__dmul_rn(1.0 - b2, g), g));
    double mh = m / bc1;
    double vh = v / bc2;
    p = __dsub_rn(p, __dmul_rn(lr, mh) / __dadd_rn(sqrt(vh), eps));
}

// Sum of the G partial groups in fp64, in group order (the order of the
// single-GPU epilogue's sum_groups), rounded once to fp32.  Gaussian g's 10
// floats land in slice g / per at offset (g % per) * 10; a slice is
// per * 10 + 2 floats (8-byte aligned), slot per * 10 carries the rank's skip
// flag (1 when status has a skip bit) and the last slot is padding.  per = n
// is the dense all-reduce layout; per = ceil(n / world) feeds a reduce-scatter
// whose rank k receives slice k in place.
__global__ void reduce_partials_kernel(const float *__restrict__ part, int G, int64_t n, int64_t per,
                                       const int32_t *__restrict__ status, float *__restrict__ acc) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t chunk = per * CGS_ACC_STRIDE + 2;
    const int64_t slices = (n + per - 1) / per;
    if (i < slices) {
        const bool skip = status && (*status & (CGS_STATUS_BIN_OVERFLOW | CGS_STATUS_NONFINITE_LOSS |
                                                CGS_STATUS_NONFINITE_PARAMS));
        acc[i * chunk + per * CGS_ACC_STRIDE] = skip ? 1.f : 0.f;
        acc[i * chunk + per * CGS_ACC_STRIDE + 1] = 0.f;
    }
    if (i >= n * CGS_ACC_STRIDE) return;
    double s = 0.0;
    for (int k = 0; k < G; ++k) s += (double)part[(int64_t)k * n * CGS_ACC_STRIDE + i];
    const int64_t g = i / CGS_ACC_STRIDE;
    acc[(g / per) * chunk + (g % per) * CGS_ACC_STRIDE + i % CGS_ACC_STRIDE] = (float)s;
}

// slices of the padded tail (rows n .. slices * per) stay zero
__global__ void zero_tail_kernel(float *__restrict__ acc, int64_t n, int64_t per) {
    const int64_t chunk = per * CGS_ACC_STRIDE + 2;
    const int64_t slices = (n + per - 1) / per;
    const int64_t tail0 = n - (slices - 1) * per;  // rows used in the last slice
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < (per - tail0) * CGS_ACC_STRIDE) acc[(slices - 1) * chunk + tail0 * CGS_ACC_STRIDE + i] = 0.f;
}

__global__ void epilogue_grads_kernel(const float *__restrict__ part, int G, int64_t n,
                                      const double *__restrict__ params, int mode, double scale,
                                      double *__restrict__ grads) {
    int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= n) return;
    double acc[10], out[11];
    sum_groups(part, G, n, g, acc);
    chain_grads(params + 11 * g, acc, scale, mode, out);
#pragma unroll
    for (int j = 0; j < 11; ++j) grads[11 * g + j] = out[j];
}

__global__ void adam_kernel(double *__restrict__ params, const double *__restrict__ grads,
                            double *__restrict__ m, double *__restrict__ v, int64_t count,
                            double lr, double b1, double b2, double eps, double bc1, double bc2) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= count) return;
    double p = params[i], mm = m[i], vv = v[i];
    adam_elem(p, grads[i], mm, vv, lr, b1, b2, eps, bc1, bc2);
    params[i] = p;
    m[i] = mm;
    v[i] = vv;
}

__global__ void epilogue_adam_kernel(const float *__restrict__ part, int G, int64_t n,
                                     double *__restrict__ params, double *__restrict__ m,
                                     double *__restrict__ v, int mode, double scale, double lr,
                                     double b1, double b2, double eps, double bc1, double bc2,
                                     const int32_t *__restrict__ skip, const double *__restrict__ hyper) {
    if (skip && (*skip & (CGS_STATUS_BIN_OVERFLOW | CGS_STATUS_NONFINITE_LOSS | CGS_STATUS_NONFINITE_PARAMS))) return;
    if (hyper) {  // device-resident (lr, bc1, bc2): one launch serves every step of a captured graph
        lr = hyper[0];
        bc1 = hyper[1];
        bc2 = hyper[2];
    }
    int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= n) return;
    double acc[10], gr[11];
    sum_groups(part, G, n, g, acc);
    double *p = params + 11 * g;
    chain_grads(p, acc, scale, mode, gr);
    double *mg = m + 11 * g, *vg = v + 11 * g;
#pragma unroll
    for (int j = 0; j < 11; ++j) {
        double pj = p[j], mj = mg[j], vj = vg[j];
        adam_elem(pj, gr[j], mj, vj, lr, b1, b2, eps, bc1, bc2);
        p[j] = pj;
        mg[j] = mj;
        vg[j] = vj;
    }
}

// The epilogue + Adam spread over a CTA of 256 threads per 64 Gaussians (the
// default; epilogue_adam_kernel above runs one thread per Gaussian end to end).
// One thread per Gaussian left only ~10 warps per SM with ~3000 dependent
// instructions each (26-group sums, seven fp64 transcendentals, 11 x Adam's
// divisions and square root), so the launch was latency-bound (25 us at C2).
// Here the work splits by kind, with the same arithmetic in the same order
// (bitwise the same parameters):
//  (1) transcendentals, 4 threads per Gaussian: scale j's softplus / sigmoid
//      (j < 3), or the amplitude's sigmoid and the normalised quaternion;
//  (2) group sums, coalesced: float f of the block's 64 x 10 contiguous
//      accumulator floats, summed over the groups in order in fp64;
//  (3) the chain's algebra, one thread per Gaussian;
//  (4) Adam, one thread per element of the block's 64 x 11 contiguous
//      parameters (coalesced p, m, v).
#ifndef CGS_EPI_GAUSS
#define CGS_EPI_GAUSS 64
#endif
#ifndef CGS_EPI_UNROLL
#define CGS_EPI_UNROLL 4
#endif
constexpr int kEpiThreads = 256, kEpiGauss = CGS_EPI_GAUSS, kEpiUnroll = CGS_EPI_UNROLL;
static_assert(4 * kEpiGauss <= kEpiThreads, "phase (1): four threads per Gaussian");
#ifndef CGS_EPI_MINB
#define CGS_EPI_MINB 4
#endif

__global__ void __launch_bounds__(kEpiThreads, CGS_EPI_MINB) epilogue_adam_wide_kernel(
    const float *__restrict__ part, int G, int64_t n, double *__restrict__ params, double *__restrict__ m,
    double *__restrict__ v, int mode, double scale, double lr, double b1, double b2, double eps, double bc1,
    double bc2, const int32_t *__restrict__ skip, const double *__restrict__ hyper) {
    if (skip && (*skip & (CGS_STATUS_BIN_OVERFLOW | CGS_STATUS_NONFINITE_LOSS | CGS_STATUS_NONFINITE_PARAMS))) return;
    if (hyper) {
        lr = hyper[0];
        bc1 = hyper[1];
        bc2 = hyper[2];
    }
    __shared__ double sacc[kEpiGauss * 10];
    __shared__ double sgr[kEpiGauss * 11];
    __shared__ double ss[3][kEpiGauss], ssig[3][kEpiGauss], sq[6][kEpiGauss];
    const int tid = threadIdx.x;
    const int64_t g0 = (int64_t)blockIdx.x * kEpiGauss;
    const int ng = (int)min((int64_t)kEpiGauss, n - g0);
    {  // (1)
        const int j = tid / kEpiGauss, i = tid - j * kEpiGauss;
        if (j < 4 && i < ng) {
            const double *raw = params + (g0 + i) * 11;
            if (j < 3) {
                chain_pre_scale(raw, j, ss[j][i], ssig[j][i]);
            } else {
                ChainPre c;
                chain_pre_quat(raw, c);
                sq[0][i] = c.inv;
                sq[1][i] = c.w;
                sq[2][i] = c.x;
                sq[3][i] = c.y;
                sq[4][i] = c.z;
                sq[5][i] = sigmoid_e(raw[10]);
            }
        }
    }
    {  // (2): kFpt accumulator floats per thread, independent chains, kEpiUnroll groups of loads in flight
        constexpr int kFpt = (kEpiGauss * 10 + kEpiThreads - 1) / kEpiThreads;
        const int nf = ng * 10;
        const float *base = part + g0 * 10;
        const int64_t gs = n * 10;
        double a[kFpt];
        bool u[kFpt];
#pragma unroll
        for (int q = 0; q < kFpt; ++q) {
            a[q] = 0.0;
            u[q] = tid + q * kEpiThreads < nf;
        }
        int k = 0;
        for (; k + kEpiUnroll <= G; k += kEpiUnroll) {
            float x[kEpiUnroll][kFpt];
#pragma unroll
            for (int r = 0; r < kEpiUnroll; ++r)
#pragma unroll
                for (int q = 0; q < kFpt; ++q)
                    x[r][q] = u[q] ? __ldg(base + (k + r) * gs + tid + q * kEpiThreads) : 0.f;
#pragma unroll
            for (int r = 0; r < kEpiUnroll; ++r)
#pragma unroll
                for (int q = 0; q < kFpt; ++q) a[q] += (double)x[r][q];
        }
        for (; k < G; ++k)
#pragma unroll
            for (int q = 0; q < kFpt; ++q)
                a[q] += (double)(u[q] ? __ldg(base + k * gs + tid + q * kEpiThreads) : 0.f);
#pragma unroll
        for (int q = 0; q < kFpt; ++q)
            if (u[q]) sacc[tid + q * kEpiThreads] = a[q];
    }
    __syncthreads();
    if (tid < ng) {  // (3)
        ChainPre c;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            c.s[j] = ss[j][tid];
            c.sig[j] = ssig[j][tid];
        }
        c.inv = sq[0][tid];
        c.w = sq[1][tid];
        c.x = sq[2][tid];
        c.y = sq[3][tid];
        c.z = sq[4][tid];
        c.sig_amp = sq[5][tid];
        double acc[10], gr[11];
#pragma unroll
        for (int j = 0; j < 10; ++j) acc[j] = sacc[tid * 10 + j];
        chain_post(c, acc, scale, mode, gr);
#pragma unroll
        for (int j = 0; j < 11; ++j) sgr[tid * 11 + j] = gr[j];
    }
    __syncthreads();
    double *pb = params + g0 * 11, *mb = m + g0 * 11, *vb = v + g0 * 11;
    for (int e = tid; e < ng * 11; e += kEpiThreads) {  // (4)
        double pj = pb[e], mj = mb[e], vj = vb[e];
        adam_elem(pj, sgr[e], mj, vj, lr, b1, b2, eps, bc1, bc2);
        pb[e] = pj;
        mb[e] = mj;
        vb[e] = vj;
    }
}

// ---- fused peer-memory exchange: reduce-scatter + epilogue + Adam + parameter broadcast ----
//
// Data parallel over NVLink / NVSwitch without NCCL on the step's data path
// (SURVEY.md 8(e)).  Every rank's accumulator (the cgs_reduce_partials_sliced
// layout, one slice of `per` Gaussians per rank, each slice carrying the
// rank's skip flag) and its fp64 parameter store (world x per rows) are mapped
// into every peer (symmetric memory).  Rank r's launch:
//   1. arrive: block 0 stores the step's epoch into slot r of every peer's
//      flag array (release, system scope); every block waits until its own
//      array shows the epoch for all peers (acquire): every accumulator is
//      complete (each was written by the kernel before this one on its rank);
//   2. reads slice r of every peer's accumulator over peer memory and sums it
//      in fp64 in rank order (deterministic), runs the chain + Adam for those
//      Gaussians (the owner keeps their moments) and stores the new parameter
//      rows into every peer's store;
//   3. done: each block adds 1 to every peer's done counter (release), and
//      block 0 returns only when its own counter has every block of every rank
//      for this epoch (acquire): no rank starts its next step (K0 reads the
//      parameters; the exchange rewrites the accumulator peers read) before
//      all writes into it and all reads from it are finished.
// One launch replaces reduce-scatter + epilogue + parameter all-gather.  The
// epoch is hyper[3] (the step counter, identical on every rank and advanced
// by the host before each step or graph replay), so counters never reset.
// Flags per rank: u32 [world] arrive slots, then the done counter.
// With flags == nullptr the launch skips both handshakes: a single-process
// simulation of `world` ranks (ranks launched one after another on one
// device) that checks the arithmetic and the layouts.
__device__ __forceinline__ void st_release_sys(uint32_t *p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_sys_add(uint32_t *p, uint32_t v) {
    asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_at_least(const uint32_t *p, uint32_t target) {
    while ((int32_t)(ld_acquire_sys(p) - target) < 0) __nanosleep(64);
}

constexpr int kPeerThreads = 128;
constexpr int kPeerMaxWorld = 64;

__global__ void __launch_bounds__(kPeerThreads) peer_epilogue_adam_kernel(
    const float *const *__restrict__ accs, double *const *__restrict__ stores, uint32_t *const *__restrict__ flags,
    int rank, int world, int64_t n, int64_t per, double *__restrict__ m, double *__restrict__ v, int mode,
    double scale, double b1, double b2, double eps, const double *__restrict__ hyper) {
    const uint32_t epoch = (uint32_t)hyper[3];
    if (flags) {
        if (blockIdx.x == 0 && threadIdx.x < world) {
            __threadfence_system();
            st_release_sys(flags[threadIdx.x] + rank, epoch);
        }
        if (threadIdx.x == 0)
            for (int p = 0; p < world; ++p) wait_at_least(flags[rank] + p, epoch);
        __syncthreads();
    }
    const int64_t slice = per * CGS_ACC_STRIDE + 2;
    const int64_t off = (int64_t)rank * slice;
    bool skip = false;
    for (int p = 0; p < world; ++p) skip |= accs[p][off + per * CGS_ACC_STRIDE] > 0.f;
    const int64_t a = (int64_t)rank * per;
    const int64_t rows = a < n ? min(per, n - a) : 0;
    if (!skip) {
        const double lr = hyper[0], bc1 = hyper[1], bc2 = hyper[2];
        const double *own = stores[rank];
        for (int64_t i = blockIdx.x * (int64_t)kPeerThreads + threadIdx.x; i < rows;
             i += (int64_t)gridDim.x * kPeerThreads) {
            double acc[10];
#pragma unroll
            for (int c = 0; c < 10; ++c) acc[c] = 0.0;
            for (int p = 0; p < world; ++p) {  // rank order: the same sum on every run
                const float2 *src = reinterpret_cast<const float2 *>(accs[p] + off + i * CGS_ACC_STRIDE);
#pragma unroll
                for (int c = 0; c < 5; ++c) {
                    const float2 w = src[c];
                    acc[2 * c] += (double)w.x;
                    acc[2 * c + 1] += (double)w.y;
                }
            }
            double raw[11], gr[11];
#pragma unroll
            for (int j = 0; j < 11; ++j) raw[j] = own[(a + i) * 11 + j];
            chain_grads(raw, acc, scale, mode, gr);
            double *mg = m + i * 11, *vg = v + i * 11;
#pragma unroll
            for (int j = 0; j < 11; ++j) {
                double mj = mg[j], vj = vg[j];
                adam_elem(raw[j], gr[j], mj, vj, lr, b1, b2, eps, bc1, bc2);
                mg[j] = mj;
                vg[j] = vj;
            }
            for (int q = 0; q < world; ++q) {  // the row into every rank's store (own included)
                double *dst = stores[q] + (a + i) * 11;
#pragma unroll
                for (int j = 0; j < 11; ++j) dst[j] = raw[j];
            }
        }
    }
    if (flags) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence_system();
            for (int q = 0; q < world; ++q) red_release_sys_add(flags[q] + world, 1u);
            if (blockIdx.x == 0) wait_at_least(flags[rank] + world, epoch * (uint32_t)world * gridDim.x);
        }
    }
}

}  // namespace cgs

using namespace cgs;

// A/B switch: CGS_EPI_NARROW=1 runs the one-thread-per-Gaussian epilogue
static bool getenv_flag(const char *name) {
    const char *v = getenv(name);
    return v && v[0] == '1';
}

extern "C" int32_t cgs_peer_blocks(int64_t per) {
    if (per <= 0) return 0;
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return (int32_t)std::min<int64_t>((per + kPeerThreads - 1) / kPeerThreads, sms);
}

extern "C" int cgs_peer_epilogue_adam(const float *const *accs, double *const *stores, uint32_t *const *flags,
                                      int32_t rank, int32_t world, int64_t n, int64_t per, double *m, double *v,
                                      int32_t mode, double scale, double beta1, double beta2, double eps,
                                      const double *hyper, void *stream) {
    if (!accs || !stores || !m || !v || !hyper || world < 1 || world > kPeerMaxWorld || rank < 0 ||
        rank >= world || n <= 0 || per <= 0 || per * world < n)
        return CGS_ERR_ARG;
    const int32_t blocks = cgs_peer_blocks(per);
    peer_epilogue_adam_kernel<<<blocks, kPeerThreads, 0, (cudaStream_t)stream>>>(
        accs, stores, flags, rank, world, n, per, m, v, mode, scale, beta1, beta2, eps, hyper);
    return check_launch("peer_epilogue_adam_kernel");
}

extern "C" int64_t cgs_acc_slice_floats(int64_t n, int64_t per) {
    if (n <= 0 || per <= 0) return 0;
    return per * CGS_ACC_STRIDE + 2;
}

extern "C" int cgs_reduce_partials_sliced(const float *partial, int32_t G, int64_t n, int64_t per,
                                          const int32_t *status, float *acc, void *stream) {
    if (G < 0 || n <= 0 || per <= 0 || !acc || (G > 0 && !partial)) return CGS_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t slices = (n + per - 1) / per;
    if (G == 0) {  // an empty local batch: a zero accumulator (and a clear flag) joins the exchange
        cudaError_t e = cudaMemsetAsync(acc, 0, sizeof(float) * slices * (per * CGS_ACC_STRIDE + 2), st);
        if (e != cudaSuccess) {
            set_error_detail("cgs_reduce_partials_sliced memset", cudaGetErrorString(e));
            return CGS_ERR_CUDA;
        }
        return CGS_OK;
    }
    const int64_t tot = std::max(n * CGS_ACC_STRIDE, slices);
    reduce_partials_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(partial, G, n, per, status, acc);
    int rc = check_launch("reduce_partials_kernel");
    if (rc) return rc;
    const int64_t pad = (slices * per - n) * CGS_ACC_STRIDE;
    if (pad > 0) {
        zero_tail_kernel<<<(unsigned)((pad + 255) / 256), 256, 0, st>>>(acc, n, per);
        rc = check_launch("zero_tail_kernel");
    }
    return rc;
}

extern "C" int cgs_reduce_partials(const float *partial, int32_t G, int64_t n, float *acc, void *stream) {
    if (G <= 0 || n <= 0 || !partial || !acc) return CGS_ERR_ARG;
    // dense layout: one slice of n rows, then the flag slot (left 0: no status)
    return cgs_reduce_partials_sliced(partial, G, n, n, nullptr, acc, stream);
}

extern "C" int cgs_epilogue_grads(const float *acc, int32_t G, int64_t n, const double *params,
                                  int32_t mode, double scale, double *grads, void *stream) {
    if (G <= 0 || n <= 0 || !acc || !params || !grads || (reinterpret_cast<uintptr_t>(acc) & 7)) return CGS_ERR_ARG;
    epilogue_grads_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        acc, G, n, params, mode, scale, grads);
    return check_launch("epilogue_grads_kernel");
}

extern "C" int cgs_adam(double *params, const double *grads, double *m, double *v, int64_t count,
                        double lr, double beta1, double beta2, double eps, double bc1, double bc2,
                        void *stream) {
    if (count <= 0 || !params || !grads || !m || !v) return CGS_ERR_ARG;
    adam_kernel<<<(unsigned)((count + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        params, grads, m, v, count, lr, beta1, beta2, eps, bc1, bc2);
    return check_launch("adam_kernel");
}

extern "C" int cgs_epilogue_adam(const float *acc, int32_t G, int64_t n, double *params, double *m,
                                 double *v, int32_t mode, double scale, double lr, double beta1,
                                 double beta2, double eps, double bc1, double bc2,
                                 const int32_t *skip_if_status, void *stream) {
    if (G <= 0 || n <= 0 || !acc || !params || !m || !v || (reinterpret_cast<uintptr_t>(acc) & 7)) return CGS_ERR_ARG;
    if (getenv_flag("CGS_EPI_NARROW")) {
        epilogue_adam_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
            acc, G, n, params, m, v, mode, scale, lr, beta1, beta2, eps, bc1, bc2, skip_if_status, nullptr);
        return check_launch("epilogue_adam_kernel");
    }
    epilogue_adam_wide_kernel<<<(unsigned)((n + kEpiGauss - 1) / kEpiGauss), kEpiThreads, 0, (cudaStream_t)stream>>>(
        acc, G, n, params, m, v, mode, scale, lr, beta1, beta2, eps, bc1, bc2, skip_if_status, nullptr);
    return check_launch("epilogue_adam_wide_kernel");
}

extern "C" int cgs_epilogue_adam_dev(const float *acc, int32_t G, int64_t n, double *params, double *m, double *v,
                                     int32_t mode, double scale, double beta1, double beta2, double eps,
                                     const double *hyper, const int32_t *skip_if_status, void *stream) {
    if (G <= 0 || n <= 0 || !acc || !params || !m || !v || !hyper || (reinterpret_cast<uintptr_t>(acc) & 7))
        return CGS_ERR_ARG;
    if (getenv_flag("CGS_EPI_NARROW")) {
        epilogue_adam_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
            acc, G, n, params, m, v, mode, scale, 0.0, beta1, beta2, eps, 1.0, 1.0, skip_if_status, hyper);
        return check_launch("epilogue_adam_kernel");
    }
    epilogue_adam_wide_kernel<<<(unsigned)((n + kEpiGauss - 1) / kEpiGauss), kEpiThreads, 0, (cudaStream_t)stream>>>(
        acc, G, n, params, m, v, mode, scale, 0.0, beta1, beta2, eps, 1.0, 1.0, skip_if_status, hyper);
    return check_launch("epilogue_adam_wide_kernel");
}
