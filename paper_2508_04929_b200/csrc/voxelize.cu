// K8: voxelize a mixture onto the D^3 grid (evaluate.voxelize, evaluate.py:76-122,
// and voxelize_gaussians, _kernels.py:193-235), for FSC.
//
// Per Gaussian (fp64, voxel_prep_kernel): s = softplus(raw_s), amp =
// softplus(raw_A), R(q/|q|); cov = R diag(s^2) R^T has eigenvalues s^2, so
// prec = R diag(1/s^2) R^T, sqrt(det) = s0 s1 s2, weight = amp / ((2 pi)^1.5
// s0 s1 s2) and the cull radius is 6.5 max(s), all in closed form.  The bbox
// is the reference's: ceil/floor of centre_px -+ radius/h, clipped.
//
// Accumulation (voxelize_kernel): one CTA per Gaussian, one thread per (y, z)
// row of its bbox.  The row's q < 6.5^2 span is solved from the quadratic,
// widened by one voxel each side and every voxel re-tested with the
// reference's q < cutoff, so the voxel set is exactly the reference's.
// Contributions w (exp(-q/2) - sub) >= 0 are added as int64 fixed point with
// one power-of-two scale, 2^62 / sum_g w_g rounded down, so no voxel can
// overflow and the integer sums make the volume bitwise reproducible; one
// unit is ~1e-19 of the total weight.  fp64 throughout, like the reference.
#include <cmath>

#include "common.cuh"

namespace cgs {

constexpr double kSubD = 6.691586091292782e-10;  // exp(-21.125), splat.py:51

struct VoxGauss {
    double c[3];     // centre in voxel units (x, y, z)
    double m[3];     // mean (x, y, z), normalised units
    double p[6];     // p00 p01 p02 p11 p12 p22
    double w;        // amp / ((2 pi)^1.5 sqrt det)
    int box[6];      // x0 x1 y0 y1 z0 z1 (inclusive; empty if x0 > x1)
};

__device__ __forceinline__ double softplus_v(double x) { return fmax(x, 0.0) + log1p(exp(-fabs(x))); }

__global__ void __launch_bounds__(256) voxel_prep_kernel(const double *__restrict__ params, int64_t n, double h,
                                                         int c0, int D, VoxGauss *__restrict__ out,
                                                         int32_t *status) {
    const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= n) return;
    const double *q = params + 11 * g;
    const double s[3] = {softplus_v(q[3]), softplus_v(q[4]), softplus_v(q[5])};
    const double amp = softplus_v(q[10]);
    double qw = q[6], qx = q[7], qy = q[8], qz = q[9];
    const double qn = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
    VoxGauss v;
    if (!(qn > 0.0) || !isfinite(qn)) {
        if (status) atomicOr(status, CGS_STATUS_DEGENERATE_ROTATION);
        for (int k = 0; k < 6; k += 2) { v.box[k] = 1; v.box[k + 1] = 0; }
        v.w = 0.0;
        out[g] = v;
        return;
    }
    qw /= qn; qx /= qn; qy /= qn; qz /= qn;
    const double R[9] = {1 - 2 * (qy * qy + qz * qz), 2 * (qx * qy - qw * qz),     2 * (qx * qz + qw * qy),
                         2 * (qx * qy + qw * qz),     1 - 2 * (qx * qx + qz * qz), 2 * (qy * qz - qw * qx),
                         2 * (qx * qz - qw * qy),     2 * (qy * qz + qw * qx),     1 - 2 * (qx * qx + qy * qy)};
    const double is2[3] = {1.0 / (s[0] * s[0]), 1.0 / (s[1] * s[1]), 1.0 / (s[2] * s[2])};
    auto P = [&](int a, int b) { return R[3 * a] * is2[0] * R[3 * b] + R[3 * a + 1] * is2[1] * R[3 * b + 1] +
                                        R[3 * a + 2] * is2[2] * R[3 * b + 2]; };
    v.p[0] = P(0, 0); v.p[1] = P(0, 1); v.p[2] = P(0, 2);
    v.p[3] = P(1, 1); v.p[4] = P(1, 2); v.p[5] = P(2, 2);
    v.w = amp / (pow(2.0 * kPiD, 1.5) * (s[0] * s[1] * s[2]));
    const double rad = kCullSigma * fmax(s[0], fmax(s[1], s[2]));
    for (int a = 0; a < 3; ++a) {
        v.m[a] = q[a];
        v.c[a] = q[a] / h + c0;
        v.box[2 * a] = (int)fmax(ceil(v.c[a] - rad / h), 0.0);
        v.box[2 * a + 1] = (int)fmin(floor(v.c[a] + rad / h), (double)(D - 1));
    }
    out[g] = v;
}

// scale = 2^floor(log2(2^62 / sum w)), one block, fixed order: deterministic
__global__ void __launch_bounds__(1024) voxel_scale_kernel(const VoxGauss *__restrict__ gs, int64_t n,
                                                           double *__restrict__ scale) {
    __shared__ double part[32];
    double t = 0.0;
    for (int64_t g = threadIdx.x; g < n; g += blockDim.x) t += gs[g].w;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += part[w];
        *scale = s > 0.0 ? exp2(floor(log2(4.611686018427388e18 / s))) : 1.0;
    }
}

__global__ void __launch_bounds__(128) voxelize_kernel(const VoxGauss *__restrict__ gs, double h, int c0, int D,
                                                       const double *__restrict__ scale_ptr,
                                                       unsigned long long *__restrict__ vox) {
    const VoxGauss &G = gs[blockIdx.x];
    const int x0 = G.box[0], x1 = G.box[1], y0 = G.box[2], y1 = G.box[3], z0 = G.box[4], z1 = G.box[5];
    if (x0 > x1 || y0 > y1 || z0 > z1) return;
    const double scale = *scale_ptr, wS = G.w * scale;
    const double p00 = G.p[0], p01 = G.p[1], p02 = G.p[2], p11 = G.p[3], p12 = G.p[4], p22 = G.p[5];
    const int ny = y1 - y0 + 1, rows = ny * (z1 - z0 + 1);
    for (int r = threadIdx.x; r < rows; r += blockDim.x) {
        const int iz = z0 + r / ny, iy = y0 + r % ny;
        const double dz = (iz - c0) * h - G.m[2], dy = (iy - c0) * h - G.m[1];
        const double qyz = p11 * dy * dy + 2.0 * p12 * dy * dz + p22 * dz * dz;
        const double bx = 2.0 * (p01 * dy + p02 * dz);
        // q(dx) = p00 dx^2 + bx dx + qyz < cutoff  <=>  dx inside the roots
        const double disc = bx * bx - 4.0 * p00 * (qyz - kCutoffSqD);
        if (disc < 0.0) continue;
        const double sq = sqrt(disc), inv = 0.5 / p00;
        const int xa = max(x0, (int)floor(((-bx - sq) * inv + G.m[0]) / h + c0) - 1);
        const int xb = min(x1, (int)ceil(((-bx + sq) * inv + G.m[0]) / h + c0) + 1);
        unsigned long long *row = vox + ((int64_t)iz * D + iy) * D;
        for (int ix = xa; ix <= xb; ++ix) {
            const double dx = (ix - c0) * h - G.m[0];
            const double q = p00 * dx * dx + bx * dx + qyz;
            if (q < kCutoffSqD) atomicAdd(row + ix, (unsigned long long)llrint(wS * (exp(-0.5 * q) - kSubD)));
        }
    }
}

__global__ void voxel_to_double_kernel(double *__restrict__ buf, int64_t count, const double *__restrict__ scale) {
    const double inv = 1.0 / *scale;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < count) buf[i] = (double)reinterpret_cast<unsigned long long *>(buf)[i] * inv;
}

}  // namespace cgs

using namespace cgs;

extern "C" size_t cgs_voxelize_workspace_bytes(int64_t n) { return (size_t)n * sizeof(VoxGauss) + 16; }

extern "C" int cgs_voxelize(const double *params, int64_t n, cgs_grid grid, double *out, void *ws, int32_t *status,
                            void *stream) {
    if (n <= 0 || grid.size < 1 || !params || !out || !ws) return CGS_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const int D = grid.size;
    const double h = 2.0 * grid.extent / D;
    VoxGauss *gs = reinterpret_cast<VoxGauss *>(ws);
    double *scale = reinterpret_cast<double *>(reinterpret_cast<char *>(ws) + (size_t)n * sizeof(VoxGauss));
    voxel_prep_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(params, n, h, D / 2, D, gs, status);
    voxel_scale_kernel<<<1, 1024, 0, st>>>(gs, n, scale);
    const int64_t count = (int64_t)D * D * D;
    cudaMemsetAsync(out, 0, sizeof(double) * count, st);
    voxelize_kernel<<<(unsigned)n, 128, 0, st>>>(gs, h, D / 2, D, scale, reinterpret_cast<unsigned long long *>(out));
    voxel_to_double_kernel<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(out, count, scale);
    return check_launch("voxelize_kernel");
}
