// K0 per-Gaussian preparation as a device function: shared by cgs_prepare
// (prepare.cu) and the fused prepare + weight-bound pass of the training
// render (render.cu).
#pragma once
#include <cmath>

#include "common.cuh"

namespace cgs {

__device__ __forceinline__ double softplus_d(double x) {
    // max(x, 0) + log1p(exp(-|x|))   (gmm.py:79)
    return fmax(x, 0.0) + log1p(exp(-fabs(x)));
}

// Prepare Gaussian g: splat[g] = {mean, amp, M = R diag(s) (row-major), s_max,
// s_min, s_mid} in f32; status bits for a degenerate rotation or non-finite
// parameters.  Returns the f32 record slots (amp, s_min, s_mid) the render's
// weight bound reads.
__device__ __forceinline__ float3 prepare_one(const double *__restrict__ params, int64_t g, float *__restrict__ splat,
                                              int32_t *status) {
    const double *p = params + g * 11;
    double s0 = softplus_d(p[3]), s1 = softplus_d(p[4]), s2 = softplus_d(p[5]);
    double amp = softplus_d(p[10]);
    double qw = p[6], qx = p[7], qy = p[8], qz = p[9];
    double qn = sqrt(qw * qw + qx * qx + qy * qy + qz * qz);
    if (!(qn > 0.0) || !isfinite(qn)) {
        atomicOr(status, CGS_STATUS_DEGENERATE_ROTATION);
        qn = 1.0;
        qw = 1.0; qx = qy = qz = 0.0;
    }
    double w = qw / qn, x = qx / qn, y = qy / qn, z = qz / qn;
    double R[9];
    R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z);     R[2] = 2 * (x * z + w * y);
    R[3] = 2 * (x * y + w * z);     R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
    R[6] = 2 * (x * z - w * y);     R[7] = 2 * (y * z + w * x);     R[8] = 1 - 2 * (x * x + y * y);
    float4 *o = reinterpret_cast<float4 *>(splat + g * CGS_SPLAT_STRIDE);
    o[0] = make_float4((float)p[0], (float)p[1], (float)p[2], (float)amp);
    o[1] = make_float4((float)(R[0] * s0), (float)(R[1] * s1), (float)(R[2] * s2), (float)(R[3] * s0));
    o[2] = make_float4((float)(R[4] * s1), (float)(R[5] * s2), (float)(R[6] * s0), (float)(R[7] * s1));
    // slots 14 / 15 carry the smallest and middle activated scale for cgs_render's weight bound
    const double lo = fmin(s0, fmin(s1, s2)), hi = fmax(s0, fmax(s1, s2));
    const float flo = (float)lo, fmid = (float)(s0 + s1 + s2 - lo - hi);
    o[3] = make_float4((float)(R[8] * s2), (float)hi, flo, fmid);
    const float chk = (float)p[0] + (float)p[1] + (float)p[2] + (float)amp + (float)s0 + (float)s1 + (float)s2;
    if (!isfinite(chk)) atomicOr(status, CGS_STATUS_NONFINITE_PARAMS);
    return make_float3((float)amp, flo, fmid);
}

}  // namespace cgs
