// Record gather for the per-epoch particle residency (optimize.Reconstructor,
// residency "epoch"): dst[i] = src[idx[i]] for rows of
// row_bytes.  src may be device memory or pinned host memory (UVA): a kernel
// reading pinned host memory pulls the records straight over PCIe / C2C
// (zero-copy), so a rank's epoch slice of a host-resident dataset lands in HBM
// without a host-side gather or a staging copy, on a side stream while the
// training step runs.  One CTA per row, 16-byte loads.
#include <algorithm>

#include "common.cuh"

namespace cgs {

constexpr int kGatherThreads = 256;

__global__ void __launch_bounds__(kGatherThreads) gather_rows_kernel(const int4 *__restrict__ src,
                                                                     const int64_t *__restrict__ idx,
                                                                     int64_t rows, int64_t vec_per_row,
                                                                     int4 *__restrict__ dst) {
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const int4 *s = src + idx[r] * vec_per_row;
        int4 *d = dst + r * vec_per_row;
        for (int64_t k = threadIdx.x; k < vec_per_row; k += kGatherThreads) d[k] = s[k];
    }
}

}  // namespace cgs

extern "C" int cgs_gather_rows(const void *src, const int64_t *idx, int64_t rows, int64_t row_bytes, void *dst,
                               void *stream) {
    if (rows < 0 || row_bytes <= 0 || (row_bytes & 15) || !src || !dst || (rows > 0 && !idx)) return CGS_ERR_ARG;
    if ((reinterpret_cast<uintptr_t>(src) & 15) || (reinterpret_cast<uintptr_t>(dst) & 15)) return CGS_ERR_ARG;
    if (rows == 0) return CGS_OK;
    // a pinned host source is read through its device mapping (an unmapped host
    // pointer is an error here, not a fault in the kernel)
    cudaPointerAttributes attr;
    cudaError_t e = cudaPointerGetAttributes(&attr, src);
    if (e != cudaSuccess) {
        cgs::set_error_detail("cgs_gather_rows", cudaGetErrorString(e));
        return CGS_ERR_CUDA;
    }
    if (attr.type == cudaMemoryTypeHost) {
        void *dsrc = nullptr;
        e = cudaHostGetDevicePointer(&dsrc, const_cast<void *>(src), 0);
        if (e != cudaSuccess || !dsrc) {
            cgs::set_error_detail("cgs_gather_rows (host source not mapped)", cudaGetErrorString(e));
            return CGS_ERR_CUDA;
        }
        src = dsrc;
    } else if (attr.type == cudaMemoryTypeUnregistered) {
        cgs::set_error_detail("cgs_gather_rows", "source is pageable host memory (pin it)");
        return CGS_ERR_ARG;
    }
    const unsigned grid = (unsigned)std::min<int64_t>(rows, 4 * 148);
    cgs::gather_rows_kernel<<<grid, cgs::kGatherThreads, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const int4 *>(src), idx, rows, row_bytes / 16, reinterpret_cast<int4 *>(dst));
    return cgs::check_launch("gather_rows_kernel");
}
