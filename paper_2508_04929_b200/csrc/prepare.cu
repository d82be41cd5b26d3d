// K0 cgs_prepare: per-Gaussian, image-independent geometry.
// Replaces the first half of _Projection.__init__ (splat.py:184-196):
// s = softplus(raw_scale), amp = softplus(raw_amp) (gmm.py:76-80),
// qn = q/|q| (splat.py:190-194), R(qn) (gmm.py:110-124), M = R diag(s).
#include "prepare.cuh"

namespace cgs {

__global__ void __launch_bounds__(256) prepare_kernel(const double *__restrict__ params, int64_t n,
                                                      float *__restrict__ splat, int32_t *status) {
    int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= n) return;
    prepare_one(params, g, splat, status);
}

}  // namespace cgs

extern "C" int cgs_prepare(const double *params, int64_t n, float *splat, int32_t *status,
                           void *stream) {
    if (n <= 0 || !params || !splat || !status) return CGS_ERR_ARG;
    int64_t blocks = (n + 255) / 256;
    cgs::prepare_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(params, n, splat, status);
    return cgs::check_launch("prepare_kernel");
}
