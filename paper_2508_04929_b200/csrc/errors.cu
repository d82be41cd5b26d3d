// Error reporting and version strings of the C ABI.
#include <cstdio>
#include <cstring>

#include "common.cuh"

namespace cgs {

static thread_local char g_detail[256] = "";

void set_error_detail(const char *what, const char *detail) {
    snprintf(g_detail, sizeof(g_detail), "%s: %s", what, detail);
}

int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) return CGS_OK;
    set_error_detail(what, cudaGetErrorString(e));
    return CGS_ERR_CUDA;
}

}  // namespace cgs

extern "C" const char *cgs_version(void) { return "cgs_b200 0.1.0 sm_100a"; }

extern "C" const char *cgs_error_string(int code) {
    switch (code) {
        case CGS_OK: return "ok";
        case CGS_ERR_ARG: return "invalid argument";
        case CGS_ERR_CUDA: return "CUDA error";
        case CGS_ERR_CUFFT: return "cuFFT error";
        case CGS_ERR_UNSUPPORTED: return "unsupported configuration";
        default: return "unknown error";
    }
}

extern "C" const char *cgs_last_error_detail(void) { return cgs::g_detail; }
