// K4: CTF evaluation, CTF application around batched cuFFT, and the MSE
// loss / residual.  Replaces ctf_evaluate (optics.py:93-121), apply_ctf
// (optics.py:124-141, incl. fft_centered/ifft_centered :78-90), loss_mse
// (train.py:114-121) and dL/dmodel (train.py:153).
//
// apply_ctf multiplies the spectrum by a frequency-domain filter, which
// commutes with circular shifts, so fftshift(ifft2(ifftshift(H) fft2(
// ifftshift(x)))) == ifft2(ifftshift(H) fft2(x)) in any consistent layout: the
// images stay in natural layout and no shift is ever materialised.  The
// reference keeps Re() of a complex inverse, which equals R2C -> H_sym -> C2R
// with H_sym(k) = (H(k) + H(-k mod D)) / 2; H_sym != H only on the Nyquist
// row/column of an even-D astigmatic CTF.
#include <cufft.h>

#include <cmath>
#include <cstdio>

#include "common.cuh"

namespace cgs {

struct CtfConst {
    double lam, cs, du, dv, c2a, s2a, s1mw2, w, phase, bfac, dA;
    double inv_dA, pl, cs3;  // 1/(D A), pi lambda, pi/2 Cs lambda^3 (fast path)
};

__host__ __device__ inline double electron_wavelength_A(double kv) {
    // optics.py:30-36 (CODATA 2018)
    const double h = 6.62607015e-34, m = 9.1093837015e-31, e = 1.602176634e-19, c = 299792458.0;
    double ev = e * kv * 1e3;
    return h / sqrt(2.0 * m * ev * (1.0 + ev / (2.0 * m * c * c))) * 1e10;
}

__device__ __forceinline__ CtfConst load_ctf(const double *__restrict__ p, int D, double pix) {
    CtfConst c;
    c.du = p[0];
    c.dv = p[1];
    double ang = p[2];
    c.lam = electron_wavelength_A(p[3]);
    c.cs = p[4] * 1e7;  // mm -> A
    c.w = p[5];
    c.s1mw2 = sqrt(1.0 - c.w * c.w);
    c.phase = p[6];
    c.bfac = p[7];
    c.c2a = cos(2.0 * ang);
    c.s2a = sin(2.0 * ang);
    c.dA = (double)D * pix;
    return c;
}

// H at centred frequency index (fy, fx) (optics.py:104-121)
__device__ __forceinline__ double ctf_value(const CtfConst &c, int fy, int fx) {
    double kx = fx / c.dA, ky = fy / c.dA;
    double k2 = kx * kx + ky * ky;
    // cos(2 (theta - theta_a)) with theta = atan2(ky, kx); theta(0, 0) = 0
    double cosv;
    if (k2 > 0.0) {
        double c2t = (kx * kx - ky * ky) / k2, s2t = 2.0 * kx * ky / k2;
        cosv = c2t * c.c2a + s2t * c.s2a;
    } else {
        cosv = c.c2a;
    }
    double defocus = 0.5 * ((c.du + c.dv) + (c.du - c.dv) * cosv);
    double chi = kPiD * c.lam * defocus * k2 - 0.5 * kPiD * c.cs * c.lam * c.lam * c.lam * k2 * k2 + c.phase;
    double sn, cs;
    sincos(chi, &sn, &cs);
    double H = -(c.s1mw2 * sn + c.w * cs);
    if (c.bfac > 0.0) H *= exp(-c.bfac * k2 / 4.0);
    return H;
}

__global__ void ctf_eval_kernel(const double *__restrict__ ctf, int D, double pix, double *__restrict__ H) {
    const int b = blockIdx.y;
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= D * D) return;
    const int iy = idx / D, ix = idx - iy * D, c0 = D / 2;
    CtfConst c = load_ctf(ctf + 8 * (int64_t)b, D, pix);
    H[(int64_t)b * D * D + idx] = ctf_value(c, iy - c0, ix - c0);
}

__device__ __forceinline__ int wrap_freq(int f, int D, int c0) {
    // map -f into the centred range [-c0, D-1-c0]
    int v = -f;
    if (v > D - 1 - c0) v -= D;
    if (v < -c0) v += D;
    return v;
}

// H for the step's multiply: chi in fp64 without divisions (k^2 cos 2(theta -
// theta_a) = (kx^2 - ky^2) cos 2theta_a + 2 kx ky sin 2theta_a), reduced mod
// 2 pi in fp64, then an fp32 sincos; |H - H_ref| < 1e-6 (fp32 pipeline).
__device__ __forceinline__ float ctf_value_fast(const CtfConst &c, int fy, int fx) {
    const double kx = fx * c.inv_dA, ky = fy * c.inv_dA;
    const double k2 = kx * kx + ky * ky;
    const double ck2 = (kx * kx - ky * ky) * c.c2a + 2.0 * kx * ky * c.s2a;
    const double dk2 = 0.5 * ((c.du + c.dv) * k2 + (c.du - c.dv) * ck2);
    double chi = c.pl * dk2 - c.cs3 * k2 * k2 + c.phase;
    chi -= 6.283185307179586 * rint(chi * 0.15915494309189535);
    float sn, cs;
    sincosf((float)chi, &sn, &cs);
    float H = -((float)c.s1mw2 * sn + (float)c.w * cs);
    if (c.bfac > 0.0) H *= __expf((float)(-c.bfac * k2 * 0.25));
    return H;
}

// spectrum[b][jy][jx] *= H_sym(fy, fx) / D^2 over the R2C half spectrum
__global__ void __launch_bounds__(256) ctf_multiply_kernel(float2 *__restrict__ spec, int D, double pix,
                                                           const double *__restrict__ ctf,
                                                           const double *__restrict__ Harr) {
    const int b = blockIdx.y;
    const int W = D / 2 + 1;
    __shared__ CtfConst cc;
    if (ctf) {  // per-image constants once per block (wavelength, 2 theta_a trig)
        if (threadIdx.x == 0) {
            cc = load_ctf(ctf + 8 * (int64_t)b, D, pix);
            cc.inv_dA = 1.0 / cc.dA;
            cc.pl = kPiD * cc.lam;
            cc.cs3 = 0.5 * kPiD * cc.cs * cc.lam * cc.lam * cc.lam;
        }
        __syncthreads();
    }
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= D * W) return;
    const int jy = idx / W, jx = idx - jy * W, c0 = D / 2;
    const int fy = jy < D - c0 ? jy : jy - D;
    const int fx = jx < D - c0 ? jx : jx - D;
    const bool nyq = (D % 2 == 0) && (fy == -c0 || fx == -c0);
    double H;
    if (ctf) {
        H = ctf_value_fast(cc, fy, fx);
        if (nyq) H = 0.5 * (H + ctf_value_fast(cc, wrap_freq(fy, D, c0), wrap_freq(fx, D, c0)));
    } else {
        const double *Hb = Harr + (int64_t)b * D * D;
        H = Hb[(fy + c0) * D + fx + c0];
        if (nyq) H = 0.5 * (H + Hb[(wrap_freq(fy, D, c0) + c0) * D + wrap_freq(fx, D, c0) + c0]);
    }
    const float s = (float)(H / ((double)D * (double)D));
    float2 v = spec[(int64_t)b * D * W + idx];
    v.x *= s;
    v.y *= s;
    spec[(int64_t)b * D * W + idx] = v;
}

// loss_b = mean((model - obs)^2) in fp64; resid = 2/D^2 (model - obs)
__global__ void __launch_bounds__(1024) loss_resid_kernel(const float *__restrict__ model,
                                                          const float *__restrict__ obs, int D,
                                                          double *__restrict__ loss,
                                                          float *__restrict__ resid,
                                                          int32_t *status) {
    const int b = blockIdx.x;
    const int64_t off = (int64_t)b * D * D;
    const int npix = D * D;
    const float sc = 2.f / (float)npix;
    double acc = 0.0;
    int i0 = 0;
    if ((npix & 3) == 0) {  // vectorised main part
        const float4 *m4 = reinterpret_cast<const float4 *>(model + off);
        const float4 *o4 = reinterpret_cast<const float4 *>(obs + off);
        float4 *r4 = reinterpret_cast<float4 *>(resid + off);
        for (int i = threadIdx.x; i < (npix >> 2); i += blockDim.x) {
            const float4 m = m4[i], o = o4[i];
            const float4 d = make_float4(m.x - o.x, m.y - o.y, m.z - o.z, m.w - o.w);
            acc += (double)d.x * d.x + (double)d.y * d.y + (double)d.z * d.z + (double)d.w * d.w;
            if (resid) r4[i] = make_float4(sc * d.x, sc * d.y, sc * d.z, sc * d.w);
        }
        i0 = npix;
    }
    for (int i = i0 + threadIdx.x; i < npix; i += blockDim.x) {
        float d = model[off + i] - obs[off + i];
        acc += (double)d * (double)d;
        if (resid) resid[off + i] = sc * d;
    }
    __shared__ double ws[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
        double l = t / (double)npix;
        loss[b] = l;
        if (status && !isfinite(l)) atomicOr(status, CGS_STATUS_NONFINITE_LOSS);
    }
}

struct FftPlan {
    cufftHandle r2c, c2r;
    int D, B;
};

static int cufft_check(cufftResult r, const char *what) {
    if (r == CUFFT_SUCCESS) return CGS_OK;
    char buf[64];
    snprintf(buf, sizeof(buf), "cufftResult %d", (int)r);
    set_error_detail(what, buf);
    return CGS_ERR_CUFFT;
}

}  // namespace cgs

using namespace cgs;

extern "C" int cgs_ctf_evaluate(const double *ctf, int32_t B, cgs_grid grid, double *H, void *stream) {
    if (B <= 0 || grid.size < 1 || !ctf || !H || !(grid.pixel_size > 0)) return CGS_ERR_ARG;
    int D = grid.size;
    dim3 g((D * D + 255) / 256, B);
    ctf_eval_kernel<<<g, 256, 0, (cudaStream_t)stream>>>(ctf, D, grid.pixel_size, H);
    return check_launch("ctf_eval_kernel");
}

extern "C" int64_t cgs_fft_spectrum_elems(int32_t size, int32_t B) {
    return (int64_t)B * size * (size / 2 + 1);
}

extern "C" int cgs_fft_plan_create(int32_t size, int32_t B, void **plan) {
    if (size < 2 || B <= 0 || !plan) return CGS_ERR_ARG;
    FftPlan *p = new FftPlan();
    p->D = size;
    p->B = B;
    int nn[2] = {size, size};
    int rc = cufft_check(cufftPlanMany(&p->r2c, 2, nn, nullptr, 1, size * size, nullptr, 1,
                                       size * (size / 2 + 1), CUFFT_R2C, B),
                         "cufftPlanMany(R2C)");
    if (rc) { delete p; return rc; }
    rc = cufft_check(cufftPlanMany(&p->c2r, 2, nn, nullptr, 1, size * (size / 2 + 1), nullptr, 1,
                                   size * size, CUFFT_C2R, B),
                     "cufftPlanMany(C2R)");
    if (rc) { cufftDestroy(p->r2c); delete p; return rc; }
    *plan = p;
    return CGS_OK;
}

extern "C" int cgs_fft_plan_destroy(void *plan) {
    if (!plan) return CGS_ERR_ARG;
    FftPlan *p = (FftPlan *)plan;
    cufftDestroy(p->r2c);
    cufftDestroy(p->c2r);
    delete p;
    return CGS_OK;
}

extern "C" int cgs_ctf_apply(void *plan, const float *in, float *out, int32_t B, cgs_grid grid,
                             const double *ctf, const double *Harr, void *spectrum, int32_t layout,
                             void *stream) {
    (void)layout;  // the filter commutes with the centring shift (see header comment)
    FftPlan *p = (FftPlan *)plan;
    if (!p || !in || !out || !spectrum || (!ctf && !Harr)) return CGS_ERR_ARG;
    if (p->D != grid.size || p->B != B) return CGS_ERR_ARG;
    if (ctf && !(grid.pixel_size > 0)) return CGS_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    int D = grid.size;
    int rc = cufft_check(cufftSetStream(p->r2c, st), "cufftSetStream");
    if (rc) return rc;
    rc = cufft_check(cufftSetStream(p->c2r, st), "cufftSetStream");
    if (rc) return rc;
    rc = cufft_check(cufftExecR2C(p->r2c, (cufftReal *)in, (cufftComplex *)spectrum), "cufftExecR2C");
    if (rc) return rc;
    int W = D / 2 + 1;
    dim3 g((D * W + 255) / 256, B);
    ctf_multiply_kernel<<<g, 256, 0, st>>>((float2 *)spectrum, D, grid.pixel_size, ctf, Harr);
    rc = check_launch("ctf_multiply_kernel");
    if (rc) return rc;
    return cufft_check(cufftExecC2R(p->c2r, (cufftComplex *)spectrum, (cufftReal *)out), "cufftExecC2R");
}

extern "C" int cgs_loss_residual(const float *model, const float *obs, int32_t B, int32_t size,
                                 double *loss, float *resid, int32_t *status, void *stream) {
    if (B <= 0 || size < 1 || !model || !obs || !loss) return CGS_ERR_ARG;
    loss_resid_kernel<<<B, 1024, 0, (cudaStream_t)stream>>>(model, obs, size, loss, resid, status);
    return check_launch("loss_resid_kernel");
}

extern "C" int cgs_ctf_mse(void *plan, const float *render, const float *obs, int32_t B,
                           cgs_grid grid, const double *ctf, void *spectrum, float *model,
                           float *upstream, double *loss, int32_t *status, int32_t layout,
                           void *stream) {
    if (!render || !obs || !upstream || !loss) return CGS_ERR_ARG;
    const float *m = render;
    if (ctf) {
        float *dst = model ? model : upstream;
        int rc = cgs_ctf_apply(plan, render, dst, B, grid, ctf, nullptr, spectrum, layout, stream);
        if (rc) return rc;
        m = dst;
    } else if (model && model != render) {
        cudaMemcpyAsync(model, render, sizeof(float) * (size_t)B * grid.size * grid.size,
                        cudaMemcpyDeviceToDevice, (cudaStream_t)stream);
    }
    int rc = cgs_loss_residual(m, obs, B, grid.size, loss, upstream, status, stream);
    if (rc) return rc;
    if (ctf) return cgs_ctf_apply(plan, upstream, upstream, B, grid, ctf, nullptr, spectrum, layout, stream);
    return CGS_OK;
}
