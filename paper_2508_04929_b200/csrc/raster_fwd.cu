// K3: forward rasterizer, the B200 replacement of forward_tiles
// (_kernels.py:66-125) and rasterize (splat.py:263-298).
//
// One CTA per (tile, image), one thread per pixel.  The tile's Gaussian list
// (ascending id, from the binning) is processed in batches of blockDim items:
// every thread projects one listed Gaussian (fp32, pixel units) into shared
// memory, then each warp owns a 4 x 8 pixel block, ballots which batch items
// touch its block (tight ellipse AABB) and walks only those, in list order,
// so each pixel accumulates sum_g w_g (2^l - sub)^+ in the reference's
// per-pixel order (ascending g) -- deterministic.
#include "common.cuh"

namespace cgs {

struct __align__(16) FwdItem {
    float mpx, mpy, A, slope;  // mean [px]; l = A (dx + slope dy)^2 + Ck dy^2
    float Ck, w, pad0, pad1;
    float xlo, xhi, ylo, yhi;  // conservative ellipse AABB [px]
};

template <int TILE>
__global__ void __launch_bounds__(TILE *TILE) raster_fwd_kernel(
    const float *__restrict__ splat, const double *__restrict__ poses, GridF G, int ntx, int T,
    int S, const int32_t *__restrict__ items, const int32_t *__restrict__ offs, int64_t capacity,
    float *__restrict__ out, int layout) {
    constexpr int NT = TILE * TILE;
    constexpr int BC = TILE / 8;  // warp blocks per tile row
    __shared__ FwdItem sitem[NT];
    const int t = blockIdx.x, b = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tx = t % ntx, ty = t / ntx;
    const int bcol = (warp % BC) * 8, brow = (warp / BC) * 4;
    const int ix = tx * TILE + bcol + (lane & 7);
    const int iy = ty * TILE + brow + (lane >> 3);
    const float fx = (float)ix, fy = (float)iy;
    // the warp's pixel block, as float bounds for the AABB test
    const float bx0 = (float)(tx * TILE + bcol), bx1 = bx0 + 7.f;
    const float by0 = (float)(ty * TILE + brow), by1 = by0 + 3.f;

    int64_t lo = offs[((int64_t)b * T + t) * S];
    int64_t hi = offs[((int64_t)b * T + t + 1) * S];
    hi = min(hi, capacity);
    const PoseF P = load_pose_f(poses, b);
    float acc = 0.f;
    for (int64_t base = lo; base < hi; base += NT) {
        const int cnt = (int)min((int64_t)NT, hi - base);
        __syncthreads();
        if ((int)threadIdx.x < cnt) {
            int g = items[base + threadIdx.x];
            Splat2 s = project2(load_splat(splat, g), P, G);
            FwdItem it;
            it.mpx = s.mpx; it.mpy = s.mpy; it.A = s.A; it.slope = s.slope;
            it.Ck = s.Ck; it.w = s.w; it.pad0 = 0.f; it.pad1 = 0.f;
            // +0.01 px keeps the AABB conservative under fp32 rounding
            it.xlo = s.mpx - s.hx - 0.01f; it.xhi = s.mpx + s.hx + 0.01f;
            it.ylo = s.mpy - s.hy - 0.01f; it.yhi = s.mpy + s.hy + 0.01f;
            sitem[threadIdx.x] = it;
        }
        __syncthreads();
        for (int j0 = 0; j0 < cnt; j0 += 32) {
            bool hit = false;
            if (j0 + lane < cnt) {
                float4 bb = *reinterpret_cast<const float4 *>(&sitem[j0 + lane].xlo);
                hit = bb.x <= bx1 && bb.y >= bx0 && bb.z <= by1 && bb.w >= by0;
            }
            unsigned m = __ballot_sync(0xffffffffu, hit);
            while (m) {
                const int k = j0 + __ffs(m) - 1;
                m &= m - 1;
                const float4 p0 = *reinterpret_cast<const float4 *>(&sitem[k].mpx);
                const float4 p1 = *reinterpret_cast<const float4 *>(&sitem[k].Ck);
                const float dx = fx - p0.x, dy = fy - p0.y;
                const float dxp = fmaf(p0.w, dy, dx);  // row-conditional offset
                const float l = fmaf(p0.z * dxp, dxp, (p1.x * dy) * dy);
                // q < cutoff  <=>  2^l > sub; outside the ellipse the term is 0
                const float v = fmaxf(ex2_approx(l) - kSub, 0.f);
                acc = fmaf(p1.y, v, acc);
            }
        }
    }
    const int D = G.D;
    if (ix < D && iy < D) {
        int oy = iy, ox = ix;
        if (layout == CGS_LAYOUT_FFT) {
            const int c0 = D / 2;
            oy = iy - c0; if (oy < 0) oy += D;
            ox = ix - c0; if (ox < 0) ox += D;
        }
        out[((int64_t)b * D + oy) * D + ox] = acc;
    }
}

// ---------------------------------------------------------------------------
// 32 x 32 tiles: row-owner scatter into half-warp-private accumulators.
//
// The gather above evaluates every pixel of a 4 x 8 warp block for every
// listed Gaussian that touches the block: ~5 slots per in-ellipse pair for
// ~1 px footprints.  Here each half-warp takes one listed Gaussian at a time,
// one lane per footprint row, and walks exactly the q < 6.5^2 span of its row,
// adding w (2^l - sub) into a shared-memory tile accumulator private to the
// half-warp (lanes own distinct rows, so no two lanes of a half ever write the
// same word and no atomics are needed).  The 16 private tiles are summed in a
// fixed order at the end, so the result is deterministic.
// ---------------------------------------------------------------------------
constexpr int kST = 32;          // tile side
constexpr int kSThreads = 256;   // 8 warps, 16 half-warps
constexpr int kSHalves = kSThreads / 16;

struct __align__(16) ScatItem {
    float mpx, mpy, A, Ck;       // mean [px, tile-relative]; l = A dx'^2 + Ck dy^2
    float w, slope, k, isp;      // weight; row centre slope, 1/c11, 1/sqrt(p00)
    float y0, y1, pad0, pad1;    // rows [y0, y1] of the ellipse AABB (tile-relative, float)
};

__global__ void __launch_bounds__(kSThreads) raster_fwd_scatter_kernel(
    const float *__restrict__ splat, const double *__restrict__ poses, GridF G, int ntx, int T, int S,
    const int32_t *__restrict__ items, const int32_t *__restrict__ offs, int64_t capacity,
    float *__restrict__ out, int layout) {
    extern __shared__ float smem[];
    float *acc = smem;                                                   // [16][32 x][32 y]
    ScatItem *sitem = reinterpret_cast<ScatItem *>(smem + kSHalves * kST * kST);  // [256]
    const int t = blockIdx.x, b = blockIdx.y;
    const int tx0 = (t % ntx) * kST, ty0 = (t / ntx) * kST;
    const int D = G.D;
    const int half = threadIdx.x >> 4, li = threadIdx.x & 15;
    const int xmax = min(kST, D - tx0) - 1, ymax = min(kST, D - ty0) - 1;  // tile-relative clip
    float *my = acc + half * kST * kST;
    const int skew = (half & 1) * 16;  // the two halves of a warp use opposite bank halves
    for (int i = threadIdx.x; i < kSHalves * kST * kST; i += kSThreads) acc[i] = 0.f;

    int64_t lo = offs[((int64_t)b * T + t) * S];
    int64_t hi = min((int64_t)offs[((int64_t)b * T + t + 1) * S], capacity);
    const PoseF P = load_pose_f(poses, b);
    for (int64_t base = lo; base < hi; base += kSThreads) {
        const int cnt = (int)min((int64_t)kSThreads, hi - base);
        __syncthreads();
        if ((int)threadIdx.x < cnt) {
            Splat2 s = project2(load_splat(splat, items[base + threadIdx.x]), P, G);
            ScatItem it;
            it.mpx = s.mpx - tx0; it.mpy = s.mpy - ty0;
            it.A = s.A; it.Ck = s.Ck; it.w = s.w;
            it.slope = s.slope; it.k = s.k; it.isp = s.inv_sqrt_p00;
            it.pad0 = 0.f; it.pad1 = 0.f;
            it.y0 = fmaxf(ceilf(it.mpy - s.hy), 0.f);
            it.y1 = fminf(floorf(it.mpy + s.hy), (float)ymax);
            if (!(s.w > 0.f)) it.y1 = -1.f;
            sitem[threadIdx.x] = it;
        }
        __syncthreads();
        for (int j = half; j < cnt; j += kSHalves) {
            const ScatItem it = sitem[j];
            const int y0 = (int)it.y0, y1 = (int)it.y1;
            const float ws = it.w * kSub;
            for (int iy = y0 + li; iy <= y1; iy += 16) {
                // row-conditional span (common.cuh row_span)
                const float dy = (float)iy - it.mpy;
                const float rem = fmaf(-it.k * dy, dy, kCutoffSq);
                if (rem <= 0.f) continue;
                const float hw = sqrtf(rem) * it.isp;
                const float xc = fmaf(-it.slope, dy, it.mpx);
                const int xa = max((int)ceilf(xc - hw), 0);
                const int xb = min((int)floorf(xc + hw), xmax);
                const float Ckdy2 = it.Ck * dy * dy;
                float *col = my + ((iy + skew) & (kST - 1));
                float dx = (float)xa - xc;
                for (int x = xa; x <= xb; ++x) {
                    const float e = ex2_approx(fmaf(it.A * dx, dx, Ckdy2));
                    col[x * kST] += fmaf(it.w, e, -ws);
                    dx += 1.f;
                }
            }
        }
    }
    __syncthreads();
    // fixed-order sum of the 16 private tiles (y fastest: conflict-free), staged
    // transposed through shared memory so the global store is row-coalesced
    float *tileT = reinterpret_cast<float *>(sitem);  // [32 y][33]
    for (int p = threadIdx.x; p < kST * kST; p += kSThreads) {
        const int y = p % kST, x = p / kST;
        float v = 0.f;
#pragma unroll
        for (int h = 0; h < kSHalves; ++h) v += acc[h * kST * kST + x * kST + ((y + (h & 1) * 16) & (kST - 1))];
        tileT[y * (kST + 1) + x] = v;
    }
    __syncthreads();
    for (int p = threadIdx.x; p < kST * kST; p += kSThreads) {
        const int y = p / kST, x = p % kST;
        const float v = tileT[y * (kST + 1) + x];
        const int iy = ty0 + y, ix = tx0 + x;
        if (iy < D && ix < D) {
            int oy = iy, ox = ix;
            if (layout == CGS_LAYOUT_FFT) {
                const int c0 = D / 2;
                oy = iy - c0; if (oy < 0) oy += D;
                ox = ix - c0; if (ox < 0) ox += D;
            }
            out[((int64_t)b * D + oy) * D + ox] = v;
        }
    }
}

}  // namespace cgs

using namespace cgs;

extern "C" int cgs_raster_fwd(const float *splat, int64_t n, const double *poses, int32_t B,
                              cgs_grid grid, int32_t tile, const int32_t *items,
                              const int32_t *offs, int64_t capacity, float *out, int32_t layout,
                              void *stream) {
    if (n <= 0 || B <= 0 || grid.size < 1 || !splat || !poses || !items || !offs || !out)
        return CGS_ERR_ARG;
    if (tile != 8 && tile != 16 && tile != 32) return CGS_ERR_UNSUPPORTED;
    int ntx = (grid.size + tile - 1) / tile, T = ntx * ntx;
    int S = (int)cgs_bin_segments(n);
    GridF G = make_grid_f(grid);
    dim3 g(T, B);
    cudaStream_t st = (cudaStream_t)stream;
    switch (tile) {
        case 8:
            raster_fwd_kernel<8><<<g, 64, 0, st>>>(splat, poses, G, ntx, T, S, items, offs, capacity, out, layout);
            break;
        case 16:
            raster_fwd_kernel<16><<<g, 256, 0, st>>>(splat, poses, G, ntx, T, S, items, offs, capacity, out, layout);
            break;
        default: {
            const size_t smem = (size_t)kSHalves * kST * kST * sizeof(float) + kSThreads * sizeof(ScatItem);
            const int rc = ensure_smem_limit((const void *)raster_fwd_scatter_kernel, smem, "raster_fwd_scatter_kernel");
            if (rc) return rc;
            raster_fwd_scatter_kernel<<<g, kSThreads, smem, st>>>(splat, poses, G, ntx, T, S, items, offs, capacity,
                                                                  out, layout);
            break;
        }
    }
    return check_launch("raster_fwd_kernel");
}
