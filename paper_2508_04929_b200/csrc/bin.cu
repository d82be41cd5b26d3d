// K2: tile binning, the B200 replacement of build_tile_work (_kernels.py:17-63).
//
// The reference runs a serial counting scatter per image: count items per
// tile, cumsum, then scatter Gaussian ids in ascending order.  Here the same
// stable order comes from one LSD counting-sort pass keyed on the tile id:
//
//   count   : grid (segment s, image b).  Each thread computes the reference's
//             fp64 bbox of one (b, g) (splat.py:218-226), packs its tile
//             rectangle, and the warp counts items per tile with one ballot per
//             tile of the warp's union rectangle.  Writes counts[(b,t,s)].
//   scan    : exclusive scan over (b, t, s) -> global item offsets.  Items are
//             ordered by image, then tile, then segment, i.e. by (b, t, g).
//   scatter : same grid; within a segment, 256-Gaussian sub-chunks are ranked
//             per warp (ballot + popc of lower lanes) and per CTA (prefix over
//             warps), so every tile list ends up in ascending Gaussian order.
#include <cmath>

#include "common.cuh"

namespace cgs {

constexpr uint32_t kEmptyRect = 0x000000FFu;  // tx0 = 255 > tx1 = 0
constexpr int kMaxTilesPerDim = 255;
constexpr int kMaxTiles = 8192;

__device__ __forceinline__ uint32_t pack_rect(int tx0, int tx1, int ty0, int ty1) {
    return (uint32_t)tx0 | ((uint32_t)tx1 << 8) | ((uint32_t)ty0 << 16) | ((uint32_t)ty1 << 24);
}

// -------------------------------------------------------------------------
// fp64 bounding box exactly as _Projection computes it (splat.py:184-226,
// 229-260), operation by operation with no FMA contraction, so the tile lists
// match the reference bit for bit.
// -------------------------------------------------------------------------
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

__device__ __forceinline__ double softplus_ref(double x) {
    return dadd(fmax(x, 0.0), log1p(exp(-fabs(x))));  // gmm.py:79
}

struct BBox {
    int x0, x1, y0, y1;
    bool clamped;
};

__device__ BBox bbox_fp64(const double *__restrict__ p, const double *__restrict__ W, double h,
                          double c0, int D, double floor_) {
    double s[3] = {softplus_ref(p[3]), softplus_ref(p[4]), softplus_ref(p[5])};
    double qw = p[6], qx = p[7], qy = p[8], qz = p[9];
    double qnorm = sqrt(dadd(dadd(dadd(dmul(qw, qw), dmul(qx, qx)), dmul(qy, qy)), dmul(qz, qz)));
    double w = qw / qnorm, x = qx / qnorm, y = qy / qnorm, z = qz / qnorm;
    double R[9];
    R[0] = dsub(1.0, dmul(2.0, dadd(dmul(y, y), dmul(z, z))));
    R[1] = dmul(2.0, dsub(dmul(x, y), dmul(w, z)));
    R[2] = dmul(2.0, dadd(dmul(x, z), dmul(w, y)));
    R[3] = dmul(2.0, dadd(dmul(x, y), dmul(w, z)));
    R[4] = dsub(1.0, dmul(2.0, dadd(dmul(x, x), dmul(z, z))));
    R[5] = dmul(2.0, dsub(dmul(y, z), dmul(w, x)));
    R[6] = dmul(2.0, dsub(dmul(x, z), dmul(w, y)));
    R[7] = dmul(2.0, dadd(dmul(y, z), dmul(w, x)));
    R[8] = dsub(1.0, dmul(2.0, dadd(dmul(x, x), dmul(y, y))));
    double M[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) M[3 * i + j] = dmul(R[3 * i + j], s[j]);
    double B[2][3];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            B[a][j] = dadd(dadd(dmul(W[3 * a], M[j]), dmul(W[3 * a + 1], M[3 + j])),
                           dmul(W[3 * a + 2], M[6 + j]));
    double mean[2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
        mean[a] = dadd(dadd(dadd(dmul(p[0], W[3 * a]), dmul(p[1], W[3 * a + 1])), dmul(p[2], W[3 * a + 2])),
                       W[9 + a]);
    double ca = dadd(dadd(dmul(B[0][0], B[0][0]), dmul(B[0][1], B[0][1])), dmul(B[0][2], B[0][2]));
    double cb = dadd(dadd(dmul(B[0][0], B[1][0]), dmul(B[0][1], B[1][1])), dmul(B[0][2], B[1][2]));
    double cd = dadd(dadd(dmul(B[1][0], B[1][0]), dmul(B[1][1], B[1][1])), dmul(B[1][2], B[1][2]));
    double mid = dmul(0.5, dadd(ca, cd));
    double amd = dsub(ca, cd);
    double rad = sqrt(fmax(dadd(dmul(0.25, dmul(amd, amd)), dmul(cb, cb)), 0.0));
    double lam1 = dadd(mid, rad);
    double lam2 = dsub(mid, rad);
    BBox bb;
    bb.clamped = lam2 < floor_;
    double lam_max = fmax(lam1, floor_);
    double radius = dmul(kCullSigma, sqrt(lam_max)) / h;
    double px = dadd(mean[0] / h, c0);
    double py = dadd(mean[1] / h, c0);
    double fx0 = fmax(ceil(dsub(px, radius)), 0.0);
    double fx1 = fmin(floor(dadd(px, radius)), (double)(D - 1));
    double fy0 = fmax(ceil(dsub(py, radius)), 0.0);
    double fy1 = fmin(floor(dadd(py, radius)), (double)(D - 1));
    if (!(fx0 <= fx1) || !(fy0 <= fy1)) {  // empty (or non-finite) footprint
        bb.x0 = 1; bb.x1 = 0; bb.y0 = 1; bb.y1 = 0;
        // keep the reference's values when finite so bbox_out can be compared
        if (isfinite(fx0) && isfinite(fx1) && isfinite(fy0) && isfinite(fy1) &&
            fabs(fx0) < 2e9 && fabs(fx1) < 2e9 && fabs(fy0) < 2e9 && fabs(fy1) < 2e9) {
            bb.x0 = (int)fx0; bb.x1 = (int)fx1; bb.y0 = (int)fy0; bb.y1 = (int)fy1;
        }
    } else {
        bb.x0 = (int)fx0; bb.x1 = (int)fx1; bb.y0 = (int)fy0; bb.y1 = (int)fy1;
    }
    return bb;
}

// -------------------------------------------------------------------------
// Warp-cooperative walk over the union of the lanes' tile rectangles:
// f(tile, ballot_mask, mine) is called once per tile that any lane covers.
// -------------------------------------------------------------------------
template <typename F>
__device__ __forceinline__ void warp_tile_walk(uint32_t rect, int ntx, F &&f) {
    int tx0 = rect & 0xFF, tx1 = (rect >> 8) & 0xFF, ty0 = (rect >> 16) & 0xFF, ty1 = rect >> 24;
    bool empty = tx0 > tx1;
    unsigned ux0 = __reduce_min_sync(0xffffffffu, empty ? 0xFFFFu : (unsigned)tx0);
    unsigned ux1 = __reduce_max_sync(0xffffffffu, empty ? 0u : (unsigned)tx1);
    unsigned uy0 = __reduce_min_sync(0xffffffffu, empty ? 0xFFFFu : (unsigned)ty0);
    unsigned uy1 = __reduce_max_sync(0xffffffffu, empty ? 0u : (unsigned)ty1);
    for (unsigned ty = uy0; ty <= uy1; ++ty) {
        bool row = !empty && (int)ty >= ty0 && (int)ty <= ty1;
        if (__ballot_sync(0xffffffffu, row) == 0u) continue;
        for (unsigned tx = ux0; tx <= ux1; ++tx) {
            bool mine = row && (int)tx >= tx0 && (int)tx <= tx1;
            unsigned m = __ballot_sync(0xffffffffu, mine);
            if (m) f((int)(ty * ntx + tx), m, mine);
        }
    }
}

__device__ __forceinline__ uint32_t rect_from_bbox(const BBox &bb, int tile) {
    if (bb.x0 > bb.x1 || bb.y0 > bb.y1) return kEmptyRect;
    return pack_rect(bb.x0 / tile, bb.x1 / tile, bb.y0 / tile, bb.y1 / tile);
}

template <bool kFromParams>
__global__ void __launch_bounds__(256) bin_count_kernel(
    const double *__restrict__ params, const int32_t *__restrict__ bbox_in, int64_t n,
    const double *__restrict__ poses, int D, double h, double c0, double floor_, int tile, int ntx,
    int T, int S, uint32_t *__restrict__ rects, int32_t *__restrict__ counts,
    int32_t *__restrict__ bbox_out, int32_t *__restrict__ clamp_count) {
    extern __shared__ int hist[];
    const int b = blockIdx.y, s = blockIdx.x;
    const int64_t g_begin = (int64_t)s * CGS_BIN_CHUNK;
    const int64_t g_end = min(n, g_begin + CGS_BIN_CHUNK);
    for (int t = threadIdx.x; t < T; t += blockDim.x) hist[t] = 0;
    __syncthreads();
    double W[12];
    if (kFromParams) {
#pragma unroll
        for (int k = 0; k < 12; ++k) W[k] = poses[12 * (int64_t)b + k];
    }
    int nclamped = 0;
    for (int64_t g0 = g_begin; g0 < g_end; g0 += blockDim.x) {
        int64_t g = g0 + threadIdx.x;
        uint32_t rect = kEmptyRect;
        if (g < g_end) {
            BBox bb;
            if (kFromParams) {
                bb = bbox_fp64(params + 11 * g, W, h, c0, D, floor_);
                nclamped += bb.clamped;
                if (bbox_out) {
                    int4 v = make_int4(bb.x0, bb.x1, bb.y0, bb.y1);
                    reinterpret_cast<int4 *>(bbox_out)[(int64_t)b * n + g] = v;
                }
            } else {
                int4 v = reinterpret_cast<const int4 *>(bbox_in)[(int64_t)b * n + g];
                bb.x0 = v.x; bb.x1 = v.y; bb.y0 = v.z; bb.y1 = v.w; bb.clamped = false;
            }
            rect = rect_from_bbox(bb, tile);
            rects[(int64_t)b * n + g] = rect;
        }
        warp_tile_walk(rect, ntx, [&](int t, unsigned m, bool) {
            if ((threadIdx.x & 31) == 0) atomicAdd(&hist[t], __popc(m));
        });
    }
    __syncthreads();
    for (int t = threadIdx.x; t < T; t += blockDim.x)
        counts[((int64_t)b * T + t) * S + s] = hist[t];
    if (kFromParams && clamp_count) {
        int c = __reduce_add_sync(0xffffffffu, nclamped);
        if ((threadIdx.x & 31) == 0 && c) atomicAdd(&clamp_count[b], c);
    }
}

__global__ void __launch_bounds__(256) bin_scatter_kernel(
    const uint32_t *__restrict__ rects, int64_t n, int ntx, int T, int S,
    const int32_t *__restrict__ offs, int32_t *__restrict__ items, int64_t capacity,
    int32_t *status) {
    extern __shared__ int smem[];
    int *cursor = smem;            // [T]
    int *whist = smem + T;         // [8][T]
    const int b = blockIdx.y, s = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t g_begin = (int64_t)s * CGS_BIN_CHUNK;
    const int64_t g_end = min(n, g_begin + CGS_BIN_CHUNK);
    for (int t = threadIdx.x; t < T; t += blockDim.x) cursor[t] = offs[((int64_t)b * T + t) * S + s];
    bool overflow = false;
    for (int64_t g0 = g_begin; g0 < g_end; g0 += blockDim.x) {
        int64_t g = g0 + threadIdx.x;
        uint32_t rect = g < g_end ? rects[(int64_t)b * n + g] : kEmptyRect;
        int *wh = whist + warp * T;
        for (int t = lane; t < T; t += 32) wh[t] = 0;
        __syncwarp();
        warp_tile_walk(rect, ntx, [&](int t, unsigned m, bool) {
            if (lane == 0) wh[t] = __popc(m);
        });
        __syncthreads();
        for (int t = threadIdx.x; t < T; t += blockDim.x) {
            int run = cursor[t];
#pragma unroll
            for (int w = 0; w < 8; ++w) {
                int c = whist[w * T + t];
                whist[w * T + t] = run;
                run += c;
            }
            cursor[t] = run;
        }
        __syncthreads();
        warp_tile_walk(rect, ntx, [&](int t, unsigned m, bool mine) {
            if (mine) {
                int64_t pos = (int64_t)wh[t] + __popc(m & lt);
                if (pos < capacity) items[pos] = (int32_t)g;
                else overflow = true;
            }
        });
        __syncthreads();
    }
    if (__any_sync(0xffffffffu, overflow) && lane == 0) atomicOr(status, CGS_STATUS_BIN_OVERFLOW);
}

// -------------------------------------------------------------------------
// int32 exclusive scan: reduce -> scan block sums -> scan with offsets
// -------------------------------------------------------------------------
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ int block_exclusive_scan(int v, int *total) {
    __shared__ int wsum[kScanThreads / 32];
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int w = lane < kScanThreads / 32 ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < kScanThreads / 32) wsum[lane] = w;
    }
    __syncthreads();
    int warp_off = warp ? wsum[warp - 1] : 0;
    if (total) *total = wsum[kScanThreads / 32 - 1];
    int res = warp_off + x - v;
    __syncthreads();
    return res;
}

__global__ void __launch_bounds__(kScanThreads) scan_reduce_kernel(const int32_t *__restrict__ in,
                                                                   int64_t count, int32_t *bsum) {
    int64_t base = (int64_t)blockIdx.x * kScanTile;
    int acc = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        int64_t i = base + k * kScanThreads + threadIdx.x;
        if (i < count) acc += in[i];
    }
    int total;
    block_exclusive_scan(acc, &total);
    if (threadIdx.x == 0) bsum[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kScanThreads) scan_blocksums_kernel(int32_t *bsum, int64_t nb) {
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int64_t base = 0; base < nb; base += kScanThreads) {
        int64_t i = base + threadIdx.x;
        int v = i < nb ? bsum[i] : 0;
        int total;
        int ex = block_exclusive_scan(v, &total);
        int c = carry;
        if (i < nb) bsum[i] = c + ex;
        __syncthreads();
        if (threadIdx.x == 0) carry = c + total;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kScanThreads) scan_apply_kernel(const int32_t *__restrict__ in,
                                                                  int32_t *out, int64_t count,
                                                                  const int32_t *__restrict__ bsum) {
    int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    int v[kScanItems];
    int local = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        int64_t i = base + k;
        v[k] = i < count ? in[i] : 0;
        local += v[k];
    }
    int ex = block_exclusive_scan(local, nullptr) + bsum[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        int64_t i = base + k;
        if (i < count) out[i] = ex;
        ex += v[k];
    }
}

}  // namespace cgs

using namespace cgs;

extern "C" int64_t cgs_bin_segments(int64_t n) { return (n + CGS_BIN_CHUNK - 1) / CGS_BIN_CHUNK; }

extern "C" int64_t cgs_bin_tiles(int32_t size, int32_t tile) {
    if (size <= 0 || tile <= 0) return 0;
    int64_t nt = (size + tile - 1) / tile;
    return nt * nt;
}

static int bin_args_ok(int64_t n, int32_t B, int32_t size, int32_t tile) {
    if (n <= 0 || B <= 0 || size < 1 || tile < 1) return CGS_ERR_ARG;
    int ntx = (size + tile - 1) / tile;
    if (ntx > kMaxTilesPerDim || (int64_t)ntx * ntx > kMaxTiles) return CGS_ERR_UNSUPPORTED;
    if (n > (int64_t)INT32_MAX) return CGS_ERR_UNSUPPORTED;
    return CGS_OK;
}

extern "C" int cgs_bin_count(const double *params, int64_t n, const double *poses, int32_t B,
                             cgs_grid grid, int32_t tile, uint32_t *rects, int32_t *counts,
                             int32_t *bbox_out, int32_t *clamp_count, void *stream) {
    int rc = bin_args_ok(n, B, grid.size, tile);
    if (rc) return rc;
    if (!params || !poses || !rects || !counts) return CGS_ERR_ARG;
    int ntx = (grid.size + tile - 1) / tile, T = ntx * ntx;
    int S = (int)cgs_bin_segments(n);
    double h = 2.0 * grid.extent / grid.size;
    double fl = (0.1 * h) * (0.1 * h);  // (EIGEN_FLOOR_FRACTION * pixel_width)^2, splat.py:207
    cudaStream_t st = (cudaStream_t)stream;
    // the trailing element of counts is the scan's total slot
    cudaMemsetAsync(counts + (int64_t)B * T * S, 0, sizeof(int32_t), st);
    dim3 g(S, B);
    bin_count_kernel<true><<<g, 256, T * sizeof(int), st>>>(
        params, nullptr, n, poses, grid.size, h, (double)(grid.size / 2), fl, tile, ntx, T, S, rects,
        counts, bbox_out, clamp_count);
    return check_launch("bin_count_kernel");
}

extern "C" int cgs_bin_count_bbox(const int32_t *bbox, int64_t n, int32_t B, int32_t size,
                                  int32_t tile, uint32_t *rects, int32_t *counts, void *stream) {
    int rc = bin_args_ok(n, B, size, tile);
    if (rc) return rc;
    if (!bbox || !rects || !counts) return CGS_ERR_ARG;
    int ntx = (size + tile - 1) / tile, T = ntx * ntx;
    int S = (int)cgs_bin_segments(n);
    cudaStream_t st = (cudaStream_t)stream;
    cudaMemsetAsync(counts + (int64_t)B * T * S, 0, sizeof(int32_t), st);
    dim3 g(S, B);
    bin_count_kernel<false><<<g, 256, T * sizeof(int), st>>>(
        nullptr, bbox, n, nullptr, size, 0.0, 0.0, 0.0, tile, ntx, T, S, rects, counts, nullptr,
        nullptr);
    return check_launch("bin_count_kernel<bbox>");
}

extern "C" size_t cgs_scan_workspace_bytes(int64_t count) {
    int64_t nb = (count + kScanTile - 1) / kScanTile;
    return (size_t)(nb > 0 ? nb : 1) * sizeof(int32_t);
}

extern "C" int cgs_exclusive_scan(const int32_t *in, int32_t *out, int64_t count, void *ws,
                                  void *stream) {
    if (count <= 0 || !in || !out || !ws) return CGS_ERR_ARG;
    int64_t nb = (count + kScanTile - 1) / kScanTile;
    cudaStream_t st = (cudaStream_t)stream;
    int32_t *bsum = (int32_t *)ws;
    scan_reduce_kernel<<<(unsigned)nb, kScanThreads, 0, st>>>(in, count, bsum);
    scan_blocksums_kernel<<<1, kScanThreads, 0, st>>>(bsum, nb);
    scan_apply_kernel<<<(unsigned)nb, kScanThreads, 0, st>>>(in, out, count, bsum);
    return check_launch("exclusive_scan");
}

extern "C" int cgs_bin_scatter(const uint32_t *rects, int64_t n, int32_t B, int32_t size,
                               int32_t tile, const int32_t *offs, int32_t *items, int64_t capacity,
                               int32_t *status, void *stream) {
    int rc = bin_args_ok(n, B, size, tile);
    if (rc) return rc;
    if (!rects || !offs || !items || !status) return CGS_ERR_ARG;
    int ntx = (size + tile - 1) / tile, T = ntx * ntx;
    int S = (int)cgs_bin_segments(n);
    size_t smem = (size_t)T * 9 * sizeof(int);
    cudaStream_t st = (cudaStream_t)stream;
    rc = ensure_smem_limit((const void *)bin_scatter_kernel, smem, "bin_scatter_kernel");
    if (rc) return rc;
    dim3 g(S, B);
    bin_scatter_kernel<<<g, 256, smem, st>>>(rects, n, ntx, T, S, offs, items, capacity, status);
    return check_launch("bin_scatter_kernel");
}
