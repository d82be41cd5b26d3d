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
    float mpx, mpy, A, Bc;     // mean [px], log2 quadratic form
    float C, w, pad0, pad1;
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
            it.mpx = s.mpx; it.mpy = s.mpy; it.A = s.A; it.Bc = s.Bc;
            it.C = s.C; it.w = s.w; it.pad0 = 0.f; it.pad1 = 0.f;
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
                const float4 p1 = *reinterpret_cast<const float4 *>(&sitem[k].C);
                const float dx = fx - p0.x, dy = fy - p0.y;
                const float l = fmaf(dx, fmaf(p0.z, dx, p0.w * dy), (p1.x * dy) * dy);
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
        default:
            raster_fwd_kernel<32><<<g, 1024, 0, st>>>(splat, poses, G, ntx, T, S, items, offs, capacity, out, layout);
            break;
    }
    return check_launch("raster_fwd_kernel");
}
