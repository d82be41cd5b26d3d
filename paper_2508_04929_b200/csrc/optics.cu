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
#include <cstdlib>
#include <cstdio>

#include "common.cuh"
#include "linefft.cuh"

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
    __sincosf((float)chi, &sn, &cs);  // |chi| <= pi: MUFU sin/cos, abs error < 6e-7
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
        double l = poison_loss(t / (double)npix, status);
        loss[b] = l;
        if (status && !isfinite(l)) atomicOr(status, CGS_STATUS_NONFINITE_LOSS);
    }
}

// ---------------------------------------------------------------------------
// Fused CTF -> MSE -> CTF^T for D = 32 R (R = 1, 2, 4), one CTA per PAIR of
// images, everything in shared memory: render + obs in, upstream + loss out.
// cuFFT needs 4 passes over HBM per transform plus the multiply kernels
// (~0.15 ms for a 256-image C2 batch); this kernel reads each input once and
// writes the upstream once.
//
// Two real images share one complex transform: z = a + i b.  With
// Z = FFT2(z), A(k) = (Z(k) + conj Z(-k)) / 2, B(k) = (Z(k) - conj Z(-k)) / 2i,
// and the real, even filters H1, H2 (H_sym, see top of file):
//   W(k) = H1 A + i H2 B = P Z(k) + Q conj Z(-k),  P = (H1+H2)/2, Q = (H1-H2)/2
// so IFFT2(W) = filt_H1(a) + i filt_H2(b) exactly: the reference's
// Re(ifft2(H fft2(x))) for both images from one forward and one inverse
// transform.  The residuals (2/D^2 (model - obs), train.py:153) are packed the
// same way for the CTF^T pass (H is real and even, so CTF^T = CTF).
//
// 1-D transforms run one per warp on a row or column of the padded smem array:
// lane l holds x[l + 32 j], j < R; a radix-R DIF step in registers (with
// twiddles W_D^{l m}) then a 32-point DIF across lanes by shuffles leaves
// X[m + R bitrev5(l)] in lane l, element m, stored back where it was loaded
// from.  The spectrum therefore lives in that permuted order, and the inverse
// runs the exact mirror network (DIT, conjugate twiddles), which takes the
// permuted order back to natural order.  The 1/D^2 of the inverse is folded
// into P and Q.
template <int R>
struct WarpFft {
    float2 tw1[R];  // W_D^{l m}
    float2 tws[5];  // lane stage s = 16 >> st: W_{2s}^{l mod s} on upper lanes, 1 on lower
    float sg[5];    // +1 lower lane, -1 upper lane

    __device__ __forceinline__ void init(int lane) {
        constexpr int D = 32 * R;
#pragma unroll
        for (int m = 0; m < R; ++m) {
            float sn, cs;
            sincospif(-2.f * (float)(lane * m) / (float)D, &sn, &cs);
            tw1[m] = make_float2(cs, sn);
        }
#pragma unroll
        for (int st = 0; st < 5; ++st) {
            const int s = 16 >> st;
            const bool up = (lane & s) != 0;
            float sn = 0.f, cs = 1.f;
            if (up) sincospif(-(float)(lane & (s - 1)) / (float)s, &sn, &cs);
            tws[st] = make_float2(cs, sn);
            sg[st] = up ? -1.f : 1.f;
        }
    }
    static __device__ __forceinline__ float2 cmul(float2 a, float2 b) {
        return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
    }
    static __device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
        return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
    }
    static __device__ __forceinline__ float2 shfl(float2 v, int s) {
        return make_float2(__shfl_xor_sync(0xffffffffu, v.x, s), __shfl_xor_sync(0xffffffffu, v.y, s));
    }
    // radix-R DFT across the register elements, sign -1 (forward) or +1 (inverse, unscaled)
    template <int SIGN>
    static __device__ __forceinline__ void dft_r(float2 v[R]) {
        if constexpr (R == 2) {
            const float2 a = v[0], b = v[1];
            v[0] = make_float2(a.x + b.x, a.y + b.y);
            v[1] = make_float2(a.x - b.x, a.y - b.y);
        } else if constexpr (R == 4) {
            const float2 a = v[0], b = v[1], c = v[2], d = v[3];
            const float2 s0 = make_float2(a.x + c.x, a.y + c.y), d0 = make_float2(a.x - c.x, a.y - c.y);
            const float2 s1 = make_float2(b.x + d.x, b.y + d.y), d1 = make_float2(b.x - d.x, b.y - d.y);
            // SIGN -1: X1 = d0 - i d1, X3 = d0 + i d1; SIGN +1 swaps them
            const float2 mi = make_float2(d0.x + d1.y, d0.y - d1.x), pi = make_float2(d0.x - d1.y, d0.y + d1.x);
            v[0] = make_float2(s0.x + s1.x, s0.y + s1.y);
            v[2] = make_float2(s0.x - s1.x, s0.y - s1.y);
            v[1] = SIGN < 0 ? mi : pi;
            v[3] = SIGN < 0 ? pi : mi;
        }
    }
    __device__ __forceinline__ void fwd(float2 v[R]) const {
        dft_r<-1>(v);
#pragma unroll
        for (int m = 1; m < R; ++m) v[m] = cmul(v[m], tw1[m]);
#pragma unroll
        for (int st = 0; st < 5; ++st) {
#pragma unroll
            for (int m = 0; m < R; ++m) {
                const float2 p = shfl(v[m], 16 >> st);
                const float2 t = make_float2(fmaf(sg[st], v[m].x, p.x), fmaf(sg[st], v[m].y, p.y));
                v[m] = cmul(t, tws[st]);
            }
        }
    }
    __device__ __forceinline__ void inv(float2 v[R]) const {  // unscaled: D x the inverse DFT
#pragma unroll
        for (int st = 4; st >= 0; --st) {
#pragma unroll
            for (int m = 0; m < R; ++m) {
                const float2 t = cmulc(v[m], tws[st]);
                const float2 p = shfl(t, 16 >> st);
                v[m] = make_float2(fmaf(sg[st], t.x, p.x), fmaf(sg[st], t.y, p.y));
            }
        }
#pragma unroll
        for (int m = 1; m < R; ++m) v[m] = cmulc(v[m], tw1[m]);
        dft_r<1>(v);
    }
};

__device__ __forceinline__ int bitrev5(int l) { return (int)(__brev((unsigned)l) >> 27); }

constexpr int kFusedThreads = 512;

// One pass of 1-D transforms over all rows (COLS = false) or columns of Z.
template <int R, bool INV, bool COLS>
__device__ __forceinline__ void fft_pass(float2 *Z, int P, const WarpFft<R> &F) {
    constexpr int D = 32 * R;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    auto addr = [&](int r, int j) { return COLS ? (lane + 32 * j) * P + r : r * P + lane + 32 * j; };
    // the next line's loads issue before this line's transform
    float2 nx[R];
#pragma unroll
    for (int j = 0; j < R; ++j) nx[j] = Z[addr(warp, j)];
    for (int r = warp; r < D; r += kFusedThreads / 32) {
        float2 v[R];
#pragma unroll
        for (int j = 0; j < R; ++j) v[j] = nx[j];
        const int rn = r + kFusedThreads / 32;
        if (rn < D) {
#pragma unroll
            for (int j = 0; j < R; ++j) nx[j] = Z[addr(rn, j)];
        }
        if (INV) F.inv(v); else F.fwd(v);
#pragma unroll
        for (int j = 0; j < R; ++j) Z[addr(r, j)] = v[j];
    }
}

// position p (0..D-1) of the permuted spectrum <-> frequency index k
template <int R>
__device__ __forceinline__ int perm_k(int p) { return (p >> 5) + R * bitrev5(p & 31); }
template <int R>
__device__ __forceinline__ int perm_p(int k) { return bitrev5(k / R) + 32 * (k % R); }

// H_sym at frequency index (ky, kx) of the full D x D grid
__device__ __forceinline__ float ctf_sym(const CtfConst &c, int D, int ky, int kx) {
    const int c0 = D / 2;
    const int fy = ky < D - c0 ? ky : ky - D, fx = kx < D - c0 ? kx : kx - D;
    float H = ctf_value_fast(c, fy, fx);
    if ((D % 2 == 0) && (fy == -c0 || fx == -c0))
        H = 0.5f * (H + ctf_value_fast(c, wrap_freq(fy, D, c0), wrap_freq(fx, D, c0)));
    return H;
}

// W(k) = P Z(k) + Q conj Z(-k) over the permuted spectrum, pairs (k, -k) at once
template <int R>
__device__ __forceinline__ void ctf_combine(float2 *Z, int P, const CtfConst *cc, bool two, float norm) {
    constexpr int D = 32 * R;
    for (int idx = threadIdx.x; idx < D * D; idx += kFusedThreads) {
        const int py = idx / D, px = idx - py * D;
        const int ky = perm_k<R>(py), kx = perm_k<R>(px);
        const int ny = ky ? D - ky : 0, nx = kx ? D - kx : 0;
        const int qy = perm_p<R>(ny), qx = perm_p<R>(nx);
        const int idx2 = qy * D + qx;
        if (idx2 < idx) continue;  // the partner's thread handles the pair
        const float h1 = ctf_sym(cc[0], D, ky, kx), h2 = two ? ctf_sym(cc[1], D, ky, kx) : 0.f;
        const float Pc = 0.5f * (h1 + h2) * norm, Qc = 0.5f * (h1 - h2) * norm;
        const float2 z1 = Z[py * P + px], z2 = Z[qy * P + qx];
        Z[py * P + px] = make_float2(Pc * z1.x + Qc * z2.x, Pc * z1.y - Qc * z2.y);
        if (idx2 != idx) Z[qy * P + qx] = make_float2(Pc * z2.x + Qc * z1.x, Pc * z2.y - Qc * z1.y);
    }
}

__device__ __forceinline__ double block_sum_f64(double v, double *scratch) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < kFusedThreads / 32; ++w) t += scratch[w];
    return t;
}

template <int R>
__global__ void __launch_bounds__(kFusedThreads, 1) ctf_mse_fused_kernel(
    const float *__restrict__ render, const float *__restrict__ obs, int B, double pix,
    const double *__restrict__ ctf, float *__restrict__ model, float *__restrict__ upstream,
    double *__restrict__ loss, int32_t *status) {
    constexpr int D = 32 * R, P = D + 1;  // padded rows: conflict-free column passes
    extern __shared__ float2 Z[];
    __shared__ CtfConst cc[2];
    __shared__ double scratch[kFusedThreads / 32];
    const int b0 = 2 * blockIdx.x;
    const bool two = b0 + 1 < B;
    if (threadIdx.x < 2 && (threadIdx.x == 0 || two)) {
        CtfConst c = load_ctf(ctf + 8 * (int64_t)(b0 + threadIdx.x), D, pix);
        c.inv_dA = 1.0 / c.dA;
        c.pl = kPiD * c.lam;
        c.cs3 = 0.5 * kPiD * c.cs * c.lam * c.lam * c.lam;
        cc[threadIdx.x] = c;
    }
    WarpFft<R> F;
    F.init(threadIdx.x & 31);
    {  // warm L2 with the observations, read only after the first CTF pass
        const char *ob = reinterpret_cast<const char *>(obs + (int64_t)b0 * D * D);
        const int bytes = (two ? 2 : 1) * D * D * (int)sizeof(float);
        for (int off = threadIdx.x * 128; off < bytes; off += kFusedThreads * 128)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(ob + off));
    }
    const float *r1 = render + (int64_t)b0 * D * D, *r2 = r1 + D * D;
    for (int i = threadIdx.x; i < D * D; i += kFusedThreads) {
        const int y = i / D, x = i - y * D;
        Z[y * P + x] = make_float2(r1[i], two ? r2[i] : 0.f);
    }
    __syncthreads();
    const float norm = 1.f / (float)(D * D);
    // model = CTF (render)
    fft_pass<R, false, false>(Z, P, F);
    __syncthreads();
    fft_pass<R, false, true>(Z, P, F);
    __syncthreads();
    ctf_combine<R>(Z, P, cc, two, norm);
    __syncthreads();
    fft_pass<R, true, true>(Z, P, F);
    __syncthreads();
    fft_pass<R, true, false>(Z, P, F);
    __syncthreads();
    // residual 2/D^2 (model - obs), loss = mean (model - obs)^2 in fp64
    const float *o1 = obs + (int64_t)b0 * D * D, *o2 = o1 + D * D;
    const float sc = 2.f * norm;
    double a1 = 0.0, a2 = 0.0;
    for (int i = threadIdx.x; i < D * D; i += kFusedThreads) {
        const int y = i / D, x = i - y * D;
        const float2 m = Z[y * P + x];
        if (model) {
            model[(int64_t)b0 * D * D + i] = m.x;
            if (two) model[(int64_t)(b0 + 1) * D * D + i] = m.y;
        }
        const float d1 = m.x - o1[i], d2 = two ? m.y - o2[i] : 0.f;
        a1 += (double)d1 * d1;
        a2 += (double)d2 * d2;
        Z[y * P + x] = make_float2(sc * d1, sc * d2);
    }
    a1 = block_sum_f64(a1, scratch);
    a2 = block_sum_f64(a2, scratch);
    if (threadIdx.x == 0) {
        const double l1 = poison_loss(a1 / (double)(D * D), status), l2 = poison_loss(a2 / (double)(D * D), status);
        loss[b0] = l1;
        if (two) loss[b0 + 1] = l2;
        if (status && (!isfinite(l1) || (two && !isfinite(l2)))) atomicOr(status, CGS_STATUS_NONFINITE_LOSS);
    }
    // upstream = CTF^T (residual)
    fft_pass<R, false, false>(Z, P, F);
    __syncthreads();
    fft_pass<R, false, true>(Z, P, F);
    __syncthreads();
    ctf_combine<R>(Z, P, cc, two, norm);
    __syncthreads();
    fft_pass<R, true, true>(Z, P, F);
    __syncthreads();
    fft_pass<R, true, false>(Z, P, F);
    __syncthreads();
    float *u1 = upstream + (int64_t)b0 * D * D, *u2 = u1 + D * D;
    for (int i = threadIdx.x; i < D * D; i += kFusedThreads) {
        const int y = i / D, x = i - y * D;
        const float2 u = Z[y * P + x];
        u1[i] = u.x;
        if (two) u2[i] = u.y;
    }
}

// ---------------------------------------------------------------------------
// General Fourier filter on image pairs: out = Re ifft2(F . fft2(in)) with, per
// image, F = H_sym (CTF, optional) x exp(-2 pi i (fx tx + fy ty) / D) (a
// sub-pixel shift by (tx, ty) pixels, optional; phase_shift_translate,
// optics.py:144-159).  Same packed-pair scheme as ctf_mse_fused_kernel with a
// complex filter: only the Hermitian part Fh(k) = (F(k) + conj F(-k)) / 2 of a
// filter reaches the real output, and with it W(k) = P Z(k) + Q conj Z(-k),
// P, Q = (Fh1 +- Fh2) / 2, W(-k) = conj(P) Z(-k) + conj(Q) conj Z(k).
// Centred and natural layouts give the same result (the filter is a circular
// convolution), so images stay in natural layout.
__device__ __forceinline__ float2 shift_ramp(float tx, float ty, int D, int fy, int fx) {
    float sn, cs;
    // exp(-2 pi i (fx tx + fy ty) / D), phase reduced in fp32 turns first
    float t = (fx * tx + fy * ty) / (float)D;
    t -= rintf(t);
    sincospif(-2.f * t, &sn, &cs);
    return make_float2(cs, sn);
}

struct FilterSpec {
    bool ctf, shift;
    CtfConst cc;
    float tx, ty;
};

// Fh(k) at frequency index (ky, kx); 1 when the image has no filter part
__device__ __forceinline__ float2 filter_h(const FilterSpec &f, int D, int ky, int kx) {
    const int c0 = D / 2;
    const int fy = ky < D - c0 ? ky : ky - D, fx = kx < D - c0 ? kx : kx - D;
    float h = f.ctf ? ctf_sym(f.cc, D, ky, kx) : 1.f;
    if (!f.shift) return make_float2(h, 0.f);
    const float2 r = shift_ramp(f.tx, f.ty, D, fy, fx);
    float2 rh = r;
    if ((D % 2 == 0) && (fy == -c0 || fx == -c0)) {  // -k wraps onto the grid: average with conj F(-k)
        const float2 rm = shift_ramp(f.tx, f.ty, D, wrap_freq(fy, D, c0), wrap_freq(fx, D, c0));
        rh = make_float2(0.5f * (r.x + rm.x), 0.5f * (r.y - rm.y));
    }
    return make_float2(h * rh.x, h * rh.y);
}

template <int R>
__device__ __forceinline__ void filter_combine(float2 *Z, int P, const FilterSpec *fs, bool two, float norm) {
    constexpr int D = 32 * R;
    for (int idx = threadIdx.x; idx < D * D; idx += kFusedThreads) {
        const int py = idx / D, px = idx - py * D;
        const int ky = perm_k<R>(py), kx = perm_k<R>(px);
        const int ny = ky ? D - ky : 0, nx = kx ? D - kx : 0;
        const int qy = perm_p<R>(ny), qx = perm_p<R>(nx);
        const int idx2 = qy * D + qx;
        if (idx2 < idx) continue;
        const float2 f1 = filter_h(fs[0], D, ky, kx);
        const float2 f2 = two ? filter_h(fs[1], D, ky, kx) : make_float2(0.f, 0.f);
        const float2 Pc = make_float2(0.5f * (f1.x + f2.x) * norm, 0.5f * (f1.y + f2.y) * norm);
        const float2 Qc = make_float2(0.5f * (f1.x - f2.x) * norm, 0.5f * (f1.y - f2.y) * norm);
        const float2 z1 = Z[py * P + px], z2 = Z[qy * P + qx];
        const float2 z2c = make_float2(z2.x, -z2.y), z1c = make_float2(z1.x, -z1.y);
        // W(k) = P z1 + Q conj(z2)
        Z[py * P + px] = make_float2(Pc.x * z1.x - Pc.y * z1.y + Qc.x * z2c.x - Qc.y * z2c.y,
                                     Pc.x * z1.y + Pc.y * z1.x + Qc.x * z2c.y + Qc.y * z2c.x);
        if (idx2 != idx)  // W(-k) = conj(P) z2 + conj(Q) conj(z1)
            Z[qy * P + qx] = make_float2(Pc.x * z2.x + Pc.y * z2.y + Qc.x * z1c.x + Qc.y * z1c.y,
                                         Pc.x * z2.y - Pc.y * z2.x + Qc.x * z1c.y - Qc.y * z1c.x);
    }
}

template <int R>
__global__ void __launch_bounds__(kFusedThreads, 1) fourier_filter_kernel(const float *__restrict__ in,
                                                                          float *__restrict__ out, int B, double pix,
                                                                          const double *__restrict__ ctf,
                                                                          const double *__restrict__ shifts) {
    constexpr int D = 32 * R, P = D + 1;
    extern __shared__ float2 Z[];
    __shared__ FilterSpec fs[2];
    const int b0 = 2 * blockIdx.x;
    const bool two = b0 + 1 < B;
    if (threadIdx.x < 2 && (threadIdx.x == 0 || two)) {
        const int b = b0 + threadIdx.x;
        FilterSpec f;
        f.ctf = ctf != nullptr;
        if (f.ctf) {
            CtfConst c = load_ctf(ctf + 8 * (int64_t)b, D, pix);
            c.inv_dA = 1.0 / c.dA;
            c.pl = kPiD * c.lam;
            c.cs3 = 0.5 * kPiD * c.cs * c.lam * c.lam * c.lam;
            f.cc = c;
        }
        f.tx = shifts ? (float)shifts[2 * (int64_t)b] : 0.f;
        f.ty = shifts ? (float)shifts[2 * (int64_t)b + 1] : 0.f;
        f.shift = f.tx != 0.f || f.ty != 0.f;
        fs[threadIdx.x] = f;
    }
    WarpFft<R> F;
    F.init(threadIdx.x & 31);
    const float *i1 = in + (int64_t)b0 * D * D, *i2 = i1 + D * D;
    for (int i = threadIdx.x; i < D * D; i += kFusedThreads) {
        const int y = i / D, x = i - y * D;
        Z[y * P + x] = make_float2(i1[i], two ? i2[i] : 0.f);
    }
    __syncthreads();
    fft_pass<R, false, false>(Z, P, F);
    __syncthreads();
    fft_pass<R, false, true>(Z, P, F);
    __syncthreads();
    filter_combine<R>(Z, P, fs, two, 1.f / (float)(D * D));
    __syncthreads();
    fft_pass<R, true, true>(Z, P, F);
    __syncthreads();
    fft_pass<R, true, false>(Z, P, F);
    __syncthreads();
    float *o1 = out + (int64_t)b0 * D * D, *o2 = o1 + D * D;
    for (int i = threadIdx.x; i < D * D; i += kFusedThreads) {
        const int y = i / D, x = i - y * D;
        const float2 u = Z[y * P + x];
        o1[i] = u.x;
        if (two) o2[i] = u.y;
    }
}

template <int R>
static int launch_fourier_filter(const float *in, float *out, int B, double pix, const double *ctf,
                                 const double *shifts, cudaStream_t st) {
    constexpr int D = 32 * R;
    const size_t smem = (size_t)D * (D + 1) * sizeof(float2);
    const int rc = ensure_smem_limit((const void *)fourier_filter_kernel<R>, smem, "fourier_filter_kernel");
    if (rc) return rc;
    fourier_filter_kernel<R><<<(B + 1) / 2, kFusedThreads, smem, st>>>(in, out, B, pix, ctf, shifts);
    return check_launch("fourier_filter_kernel");
}

// ---------------------------------------------------------------------------
// K4, one image per CTA (the training step's default for D = 64 / 128).
//
// The pair kernel above needs a full D x (D+1) complex array per CTA (132 KB at
// D = 128: one CTA per SM, 128 CTAs for 148 SMs).  Here each CTA keeps one
// image's half spectrum, D rows x (D/2 + 1) complex (66.5 KB) plus its filter
// table (33 KB): two CTAs per SM, 256 CTAs.  Real transforms by the two-for-one trick:
//  * rows, forward: rows 2j and 2j+1 go through one complex FFT as
//    z = x_2j + i x_2j+1; with Z(-k) from the same transform,
//    X_2j(k) = (Z(k) + conj Z(-k)) / 2, X_2j+1(k) = (Z(k) - conj Z(-k)) / 2i,
//    for k = 0..D/2 (the rest is their conjugate mirror);
//  * columns: D/2 + 1 complex FFTs (permuted order along y, as in WarpFft);
//  * filter: H_sym / D^2 per half-spectrum element, evaluated once per image
//    (fp64 chi) into a shared-memory table used by both CTF passes;
//  * columns inverse (mirror network, natural order), then rows inverse:
//    Z(k) = X_2j(k) + i X_2j+1(k) over all k (conjugate mirror above D/2)
//    through one complex inverse FFT gives rows 2j and 2j+1 as real and imag.
// The real rows live in the same shared array (a row of D/2 + 1 float2 holds
// D + 2 floats), each warp rewriting only its own row pairs.
#ifndef CGS_R2C_THREADS
#define CGS_R2C_THREADS 384
#endif
constexpr int kR2cThreads = CGS_R2C_THREADS;
#ifndef CGS_SPEC_MINB
#define CGS_SPEC_MINB 2
#endif

// forward real 2-D FFT of the real image held row-wise (floats, row stride 2P)
// in X: afterwards X[py][kx] = spectrum at (perm_k(py), kx), kx <= D/2
template <int R>
__device__ __forceinline__ void r2c_2d(float2 *X, const WarpFft<R> &F) {
    constexpr int D = 32 * R, P = D / 2 + 1, NW = kR2cThreads / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float *Xf = reinterpret_cast<float *>(X);
    for (int j = warp; j < D / 2; j += NW) {
        float2 v[R];
#pragma unroll
        for (int t = 0; t < R; ++t) v[t] = make_float2(Xf[(2 * j) * 2 * P + lane + 32 * t],
                                                       Xf[(2 * j + 1) * 2 * P + lane + 32 * t]);
        F.fwd(v);
        // park Z(k): k <= D/2 in row 2j slot k, k > D/2 in row 2j+1 slot k - D/2
        __syncwarp();
#pragma unroll
        for (int m = 0; m < R; ++m) {
            const int k = m + R * bitrev5(lane);
            X[k <= D / 2 ? (2 * j) * P + k : (2 * j + 1) * P + (k - D / 2)] = v[m];
        }
        __syncwarp();
        float2 a[3], c[3];
#pragma unroll
        for (int u = 0; u < 3; ++u) {
            const int k = lane + 32 * u;
            if (k > D / 2) break;
            const int nk = (D - k) % D;
            const float2 zk = X[(2 * j) * P + k];
            const float2 zn = nk <= D / 2 ? X[(2 * j) * P + nk] : X[(2 * j + 1) * P + (nk - D / 2)];
            a[u] = make_float2(0.5f * (zk.x + zn.x), 0.5f * (zk.y - zn.y));  // (Z(k) + conj Z(-k)) / 2
            c[u] = make_float2(0.5f * (zk.y + zn.y), 0.5f * (zn.x - zk.x));  // (Z(k) - conj Z(-k)) / 2i
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 3; ++u) {
            const int k = lane + 32 * u;
            if (k > D / 2) break;
            X[(2 * j) * P + k] = a[u];
            X[(2 * j + 1) * P + k] = c[u];
        }
    }
    __syncthreads();
    for (int col = warp; col < P; col += NW) {  // columns: DIF, permuted along y
        float2 v[R];
#pragma unroll
        for (int t = 0; t < R; ++t) v[t] = X[(lane + 32 * t) * P + col];
        F.fwd(v);
#pragma unroll
        for (int t = 0; t < R; ++t) X[(lane + 32 * t) * P + col] = v[t];
    }
}

// inverse: columns (mirror network, natural order), then rows back to real
// (unscaled: D^2 x the inverse DFT; the filter carries 1/D^2)
template <int R>
__device__ __forceinline__ void c2r_2d(float2 *X, const WarpFft<R> &F) {
    constexpr int D = 32 * R, P = D / 2 + 1, NW = kR2cThreads / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int col = warp; col < P; col += NW) {
        float2 v[R];
#pragma unroll
        for (int t = 0; t < R; ++t) v[t] = X[(lane + 32 * t) * P + col];
        F.inv(v);
#pragma unroll
        for (int t = 0; t < R; ++t) X[(lane + 32 * t) * P + col] = v[t];
    }
    __syncthreads();
    float *Xf = reinterpret_cast<float *>(X);
    for (int j = warp; j < D / 2; j += NW) {
        float2 v[R];
#pragma unroll
        for (int m = 0; m < R; ++m) {  // lane l, element m carries Z(m + R bitrev5(l))
            const int k = m + R * bitrev5(lane);
            const bool lo = k <= D / 2;
            const int kk = lo ? k : D - k;
            float2 a = X[(2 * j) * P + kk], c = X[(2 * j + 1) * P + kk];
            if (!lo) { a.y = -a.y; c.y = -c.y; }
            v[m] = make_float2(a.x - c.y, a.y + c.x);  // X_2j(k) + i X_2j+1(k)
        }
        F.inv(v);
        __syncwarp();
#pragma unroll
        for (int t = 0; t < R; ++t) {
            Xf[(2 * j) * 2 * P + lane + 32 * t] = v[t].x;
            Xf[(2 * j + 1) * 2 * P + lane + 32 * t] = v[t].y;
        }
    }
    __syncthreads();
}

template <int R>
__device__ __forceinline__ void half_filter(float2 *X, const float *__restrict__ Hh) {
    constexpr int D = 32 * R, P = D / 2 + 1;
    for (int i = threadIdx.x; i < D * P; i += kR2cThreads) {
        const int py = i / P, kx = i - py * P;
        const float h = Hh[perm_k<R>(py) * P + kx];
        const float2 z = X[i];
        X[i] = make_float2(z.x * h, z.y * h);
    }
    __syncthreads();
}

template <int R>
__global__ void __launch_bounds__(kR2cThreads, 2) ctf_mse_r2c_kernel(
    const float *__restrict__ render, const float *__restrict__ obs, const double *__restrict__ ctf, double pix,
    float *__restrict__ model, float *__restrict__ upstream, double *__restrict__ loss, int32_t *status) {
    constexpr int D = 32 * R, P = D / 2 + 1;
    extern __shared__ float2 X[];
    float *hb = reinterpret_cast<float *>(X + D * P);  // H_sym / D^2 over the half spectrum
    __shared__ double scratch[kR2cThreads / 32];
    __shared__ CtfConst cc;
    float *Xf = reinterpret_cast<float *>(X);
    const int b = blockIdx.x;
    if (threadIdx.x == 0) {
        CtfConst c = load_ctf(ctf + 8 * (int64_t)b, D, pix);
        c.inv_dA = 1.0 / c.dA;
        c.pl = kPiD * c.lam;
        c.cs3 = 0.5 * kPiD * c.cs * c.lam * c.lam * c.lam;
        cc = c;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < D * P; i += kR2cThreads) {
        const int ky = i / P, kx = i - ky * P;
        hb[i] = ctf_sym(cc, D, ky, kx) * (1.f / ((float)D * (float)D));
    }
    WarpFft<R> F;
    F.init(threadIdx.x & 31);
    {  // warm L2 with the observation, read only after the first CTF pass
        const char *ob = reinterpret_cast<const char *>(obs + (int64_t)b * D * D);
        for (int off = threadIdx.x * 128; off < D * D * (int)sizeof(float); off += kR2cThreads * 128)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(ob + off));
    }
    const float4 *r4 = reinterpret_cast<const float4 *>(render + (int64_t)b * D * D);
    for (int i = threadIdx.x; i < D * D / 4; i += kR2cThreads) {
        const int y = (4 * i) / D, x = 4 * i - y * D;
        const float4 v = __ldg(r4 + i);
        float *row = Xf + y * 2 * P + x;
        row[0] = v.x; row[1] = v.y; row[2] = v.z; row[3] = v.w;
    }
    __syncthreads();
    r2c_2d<R>(X, F);
    __syncthreads();
    half_filter<R>(X, hb);
    c2r_2d<R>(X, F);
    // residual 2/D^2 (model - obs), loss = mean (model - obs)^2 in fp64
    const float sc = 2.f / (float)(D * D);
    const float *o = obs + (int64_t)b * D * D;
    double acc = 0.0;
    for (int i = threadIdx.x; i < D * D; i += kR2cThreads) {
        const int y = i / D, x = i - y * D;
        const float m = Xf[y * 2 * P + x];
        if (model) model[(int64_t)b * D * D + i] = m;
        const float d = m - __ldg(o + i);
        acc += (double)d * d;
        Xf[y * 2 * P + x] = sc * d;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kR2cThreads / 32; ++w) t += scratch[w];
        const double l = poison_loss(t / (double)(D * D), status);
        loss[b] = l;
        if (status && !isfinite(l)) atomicOr(status, CGS_STATUS_NONFINITE_LOSS);
    }
    // upstream = CTF^T (residual)
    r2c_2d<R>(X, F);
    __syncthreads();
    half_filter<R>(X, hb);
    c2r_2d<R>(X, F);
    float4 *u4 = reinterpret_cast<float4 *>(upstream + (int64_t)b * D * D);
    for (int i = threadIdx.x; i < D * D / 4; i += kR2cThreads) {
        const int y = (4 * i) / D, x = 4 * i - y * D;
        const float *row = Xf + y * 2 * P + x;
        u4[i] = make_float4(row[0], row[1], row[2], row[3]);
    }
}

// K4 in the Fourier domain (the training step's default when the observation
// spectra are available, D = 64 / 128).  With O = F(obs) computed once per
// observation (obs_spectrum_kernel, same half-spectrum layout as r2c_2d), the
// residual's spectrum is F(r) = H_sym F(render) - O, so
//   loss = mean r^2 = sum_k w_k |F(r)_k|^2 / D^4      (Parseval; w = 1 on the
//          kx = 0 and kx = D/2 columns of the half spectrum, 2 elsewhere)
//   upstream = 2/D^2 CTF^T(r) = c2r(H_sym / D^2 * 2/D^2 * F(r))
// One forward and one inverse 2-D transform per image instead of two of each,
// and the model image is never formed.
// Per observation record (obs_spectrum_kernel): the half spectrum O = F(obs),
// D x P complex in r2c_2d's layout, then H_sym / D^2 as D x P floats in the
// same (permuted-row) layout, so the step reads both with coalesced loads.
template <int R>
__global__ void __launch_bounds__(kR2cThreads, 2) obs_spectrum_kernel(const float *__restrict__ obs,
                                                                       const double *__restrict__ ctf, double pix,
                                                                       float2 *__restrict__ spec) {
    constexpr int D = 32 * R, P = D / 2 + 1;
    extern __shared__ float2 X[];
    __shared__ CtfConst cc;
    float *Xf = reinterpret_cast<float *>(X);
    const int b = blockIdx.x;
    if (threadIdx.x == 0) {
        CtfConst c = load_ctf(ctf + 8 * (int64_t)b, D, pix);
        c.inv_dA = 1.0 / c.dA;
        c.pl = kPiD * c.lam;
        c.cs3 = 0.5 * kPiD * c.cs * c.lam * c.lam * c.lam;
        cc = c;
    }
    WarpFft<R> F;
    F.init(threadIdx.x & 31);
    const float4 *o4 = reinterpret_cast<const float4 *>(obs + (int64_t)b * D * D);
    for (int i = threadIdx.x; i < D * D / 4; i += kR2cThreads) {
        const int y = (4 * i) / D, x = 4 * i - y * D;
        const float4 v = __ldg(o4 + i);
        float *row = Xf + y * 2 * P + x;
        row[0] = v.x; row[1] = v.y; row[2] = v.z; row[3] = v.w;
    }
    __syncthreads();
    r2c_2d<R>(X, F);
    __syncthreads();
    float2 *dst = spec + (int64_t)b * (3 * D * P / 2);
    for (int i = threadIdx.x; i < D * P; i += kR2cThreads) dst[i] = X[i];
    float *hd = reinterpret_cast<float *>(dst + D * P);
    for (int i = threadIdx.x; i < D * P; i += kR2cThreads) {
        const int py = i / P, kx = i - py * P;
        hd[i] = ctf_sym(cc, D, perm_k<R>(py), kx) * (1.f / ((float)D * (float)D));
    }
}

template <int R, bool kFixed, bool kRowPair>  // kFixed: render is cgs_render_fixed's int32 image, converted
                                              // on load; kRowPair: upstream in CGS_LAYOUT_ROWPAIR
__global__ void __launch_bounds__(kR2cThreads, CGS_SPEC_MINB) ctf_mse_spec_kernel(
    const float *__restrict__ render, const float *__restrict__ render_scale, const float2 *__restrict__ obs_spec,
    float *__restrict__ upstream, double *__restrict__ loss, int32_t *status) {
    constexpr int D = 32 * R, P = D / 2 + 1;
    extern __shared__ float2 X[];
    __shared__ double scratch[kR2cThreads / 32];
    float *Xf = reinterpret_cast<float *>(X);
    const int b = blockIdx.x;
    WarpFft<R> F;
    F.init(threadIdx.x & 31);
    const float2 *O = obs_spec + (int64_t)b * (3 * D * P / 2);
    const float *Hh = reinterpret_cast<const float *>(O + D * P);  // H_sym / D^2, X's layout
    {  // warm L2 with the observation record, read after the forward transform
        const char *ob = reinterpret_cast<const char *>(O);
        for (int off = threadIdx.x * 128; off < 3 * D * P * (int)sizeof(float); off += kR2cThreads * 128)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(ob + off));
    }
    const float4 *r4 = reinterpret_cast<const float4 *>(render + (int64_t)b * D * D);
    const float inv_scale = kFixed ? 1.f / __ldg(render_scale) : 1.f;
    for (int i = threadIdx.x; i < D * D / 4; i += kR2cThreads) {
        const int y = (4 * i) / D, x = 4 * i - y * D;
        float4 v = __ldg(r4 + i);
        if (kFixed) {
            v = make_float4((float)__float_as_int(v.x) * inv_scale, (float)__float_as_int(v.y) * inv_scale,
                            (float)__float_as_int(v.z) * inv_scale, (float)__float_as_int(v.w) * inv_scale);
        }
        float *row = Xf + y * 2 * P + x;
        row[0] = v.x; row[1] = v.y; row[2] = v.z; row[3] = v.w;
    }
    __syncthreads();
#if !defined(CGS_SPEC_EXP) || !(CGS_SPEC_EXP & 1)  // timing experiments only: 1 skips the forward, 2 the inverse
    r2c_2d<R>(X, F);
#endif
    __syncthreads();
    // F(r) = H F(render) - O (H = Hh D^2, exact: D^2 is a power of two); loss; then
    // the CTF^T filter and the 2/D^2 residual scale in place
    const float d2 = (float)(D * D), sc = 2.f / (float)(D * D);
    double acc = 0.0;
    for (int i = threadIdx.x; i < D * P; i += kR2cThreads) {
        const int kx = i % P;
        const float h = __ldg(Hh + i);
        const float2 z = X[i], o = __ldg(O + i);
        const float hd = h * d2;
        const float rx = fmaf(hd, z.x, -o.x), ry = fmaf(hd, z.y, -o.y);
        const double m2 = (double)rx * rx + (double)ry * ry;
        acc += (kx == 0 || kx == D / 2) ? m2 : 2.0 * m2;
        const float hs = h * sc;
        X[i] = make_float2(hs * rx, hs * ry);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kR2cThreads / 32; ++w) t += scratch[w];
        const double l = poison_loss(t / ((double)D * D * (double)D * D), status);
        loss[b] = l;
        if (status && !isfinite(l)) atomicOr(status, CGS_STATUS_NONFINITE_LOSS);
    }
#if !defined(CGS_SPEC_EXP) || !(CGS_SPEC_EXP & 2)
    c2r_2d<R>(X, F);
#else
    __syncthreads();
#endif
    float4 *u4 = reinterpret_cast<float4 *>(upstream + (int64_t)b * D * D);
    if (kRowPair) {  // float4 i = pixels (2j, x), (2j+1, x), (2j, x+1), (2j+1, x+1)
        for (int i = threadIdx.x; i < D * D / 4; i += kR2cThreads) {
            const int j = (2 * i) / D, x = 2 * i - j * D;
            const float *r0 = Xf + (2 * j) * 2 * P + x, *r1 = r0 + 2 * P;
            u4[i] = make_float4(r0[0], r1[0], r0[1], r1[1]);
        }
    } else {
        for (int i = threadIdx.x; i < D * D / 4; i += kR2cThreads) {
            const int y = (4 * i) / D, x = 4 * i - y * D;
            const float *row = Xf + y * 2 * P + x;
            u4[i] = make_float4(row[0], row[1], row[2], row[3]);
        }
    }
}

// ---------------------------------------------------------------------------
// The spectral K4 and its observation records on line FFTs (linefft.cuh):
// one length-D complex transform per group of 8 threads, natural order.
// Shared memory: X complex [D][S], S = D/2 + 2, and the step-A twiddles.
// Forward real 2-D transform of a real image:
//  * rows: pair row j (rows 2j, 2j+1) sits in slots [2jS, 2jS + D) as
//    z[x] = (img[2j][x], img[2j+1][x]); one line FFT gives Z = X_2j + i X_2j+1,
//    separated into X_2j(k) = (Z(k) + conj Z(-k)) / 2 -> slot 2jS + k and
//    X_2j+1(k) = (Z(k) - conj Z(-k)) / 2i -> slot (2j+1)S + k, k = 0..D/2;
//  * columns kx = 1..D/2-1: one line each (natural ky).  Columns 0 and D/2
//    are real sequences in y (the DC and Nyquist bins of real rows), so they
//    share one line, z = X(., 0) + i X(., D/2), whose spectrum
//    Zp = F0 + i F_D/2 stays packed in column 0: D/2 lines per pass, one per
//    group of a CTA of 4D threads.
// The filter acts on the packed column as on the pair kernel's two images
// (ctf_mse_fused_kernel): H0 F0 + i HN F_D/2 = Pc Zp(ky) + Qc conj Zp(-ky)
// with Pc, Qc = (H(ky, 0) +- H(ky, D/2)) / 2, and Parseval gives
// sum_ky |F0|^2 + |F_D/2|^2 = sum_ky |Zp|^2.  The inverse runs the columns
// (the packed line unpacks into columns 0 and D/2) and then the pair rows,
// whose line output z[x] = (row 2j, row 2j+1) at x is exactly the row-pair
// upstream layout.
// Bank layout: S = D/2 + 2 = 2 mod 16 puts the 8 rows a column group reads
// at once on distinct bank pairs, and pair rows j, j + 2 (the two groups of a
// half warp in the row passes) 16 banks apart.
template <int D>
struct SpecLf {
    static constexpr int V = D / 8, S = D / 2 + 2, P = D / 2 + 1, NT = 4 * D;
    static constexpr size_t smem = (size_t)(D * S + V * 8) * sizeof(float2);
    static __device__ __forceinline__ int pair_row() {  // this group's pair row, interleaved per warp
        const int g = threadIdx.x >> 3, q = g & 3;
        return (g & ~3) + ((q & 1) << 1) + (q >> 1);
    }
};

// load pair rows: (img[2j][x], img[2j+1][x]) -> slot 2jS + x (float4 loads, 16-byte stores)
template <int D, bool kFixed>
__device__ __forceinline__ void lf_load_pairs(float2 *X, const float *__restrict__ img, float inv_scale) {
    using G = SpecLf<D>;
    const float4 *r4 = reinterpret_cast<const float4 *>(img);
    for (int i = threadIdx.x; i < D * D / 8; i += G::NT) {
        const int j = i / (D / 4), x = 4 * (i - j * (D / 4));
        const float4 a = __ldg(r4 + (2 * j) * (D / 4) + x / 4), b = __ldg(r4 + (2 * j + 1) * (D / 4) + x / 4);
        float4 u, w;
        if (kFixed) {
            u = make_float4((float)__float_as_int(a.x) * inv_scale, (float)__float_as_int(b.x) * inv_scale,
                            (float)__float_as_int(a.y) * inv_scale, (float)__float_as_int(b.y) * inv_scale);
            w = make_float4((float)__float_as_int(a.z) * inv_scale, (float)__float_as_int(b.z) * inv_scale,
                            (float)__float_as_int(a.w) * inv_scale, (float)__float_as_int(b.w) * inv_scale);
        } else {
            u = make_float4(a.x, b.x, a.y, b.y);
            w = make_float4(a.z, b.z, a.w, b.w);
        }
        float4 *dst = reinterpret_cast<float4 *>(X + 2 * j * G::S + x);
        dst[0] = u;
        dst[1] = w;
    }
}

template <int D>
__device__ __forceinline__ void lf_rows_forward(float2 *X, const float2 *twt) {
    using G = SpecLf<D>;
    constexpr int S = G::S, NK = D / 16 + 1;
    const int t = threadIdx.x & 7;
    float2 *reg = X + 2 * G::pair_row() * S;
    lfft::line<D, -1, true>(
        t, twt, [&](int n) { return reg[n]; }, [&](int s) { return reg + s; },
        [&](int k, float2 v) { reg[k] = v; });
    __syncwarp();
    float2 a[NK], c[NK];
#pragma unroll
    for (int m = 0; m < NK; ++m) {
        const int k = t + 8 * m;
        if (k <= D / 2) {
            const float2 zk = reg[k], zn = reg[(D - k) & (D - 1)];
            a[m] = make_float2(0.5f * (zk.x + zn.x), 0.5f * (zk.y - zn.y));  // (Z(k) + conj Z(-k)) / 2
            c[m] = make_float2(0.5f * (zk.y + zn.y), 0.5f * (zn.x - zk.x));  // (Z(k) - conj Z(-k)) / 2i
        }
    }
    __syncwarp();
#pragma unroll
    for (int m = 0; m < NK; ++m) {
        const int k = t + 8 * m;
        if (k <= D / 2) {
            reg[k] = a[m];
            reg[S + k] = c[m];
        }
    }
}

template <int D, int SIGN>
__device__ __forceinline__ void lf_cols(float2 *X, const float2 *twt) {
    using G = SpecLf<D>;
    constexpr int S = G::S;
    const int c = threadIdx.x >> 3, t = threadIdx.x & 7;
    float2 *col = X + c;
    lfft::line<D, SIGN, true>(
        t, twt,
        [&](int n) {
            float2 v = col[n * S];
            if (SIGN < 0 && c == 0) v.y = col[n * S + D / 2].x;  // pack the real columns 0 and D/2
            return v;
        },
        [&](int s) { return col + s * S; },
        [&](int k, float2 v) {
            if (SIGN > 0 && c == 0) {  // unpack
                col[k * S] = make_float2(v.x, 0.f);
                col[k * S + D / 2] = make_float2(v.y, 0.f);
            } else {
                col[k * S] = v;
            }
        });
}

// inverse pair rows (unscaled) straight to the upstream image in HBM
template <int D, bool kRowPair>
__device__ __forceinline__ void lf_rows_inverse(float2 *X, const float2 *twt, float *__restrict__ up) {
    using G = SpecLf<D>;
    constexpr int S = G::S;
    const int t = threadIdx.x & 7, j = G::pair_row();
    float2 *reg = X + 2 * j * S;
    lfft::line<D, 1, false>(
        t, twt,
        [&](int k) {
            const bool lo = k <= D / 2;
            const int kk = lo ? k : D - k;
            float2 a = reg[kk], c = reg[S + kk];
            if (!lo) {
                a.y = -a.y;
                c.y = -c.y;
            }
            return make_float2(a.x - c.y, a.y + c.x);  // X_2j(k) + i X_2j+1(k)
        },
        [&](int s) { return reg + s; },
        [&](int x, float2 v) {
            if (kRowPair) {
                reinterpret_cast<float2 *>(up)[j * D + x] = v;
            } else {
                up[(2 * j) * D + x] = v.x;
                up[(2 * j + 1) * D + x] = v.y;
            }
        });
}

template <int D>
__global__ void __launch_bounds__(SpecLf<D>::NT, 2) obs_spectrum_lf_kernel(const float *__restrict__ obs,
                                                                            const double *__restrict__ ctf,
                                                                            double pix, float2 *__restrict__ spec) {
    using G = SpecLf<D>;
    constexpr int S = G::S, P = G::P;
    extern __shared__ float2 X[];
    float2 *twt = X + D * S;
    __shared__ CtfConst cc;
    const int b = blockIdx.x;
    if (threadIdx.x == 0) {
        CtfConst c = load_ctf(ctf + 8 * (int64_t)b, D, pix);
        c.inv_dA = 1.0 / c.dA;
        c.pl = kPiD * c.lam;
        c.cs3 = 0.5 * kPiD * c.cs * c.lam * c.lam * c.lam;
        cc = c;
    }
    lfft::init_twiddles<D>(twt, threadIdx.x, G::NT);
    lf_load_pairs<D, false>(X, obs + (int64_t)b * D * D, 1.f);
    __syncthreads();
#if !defined(CGS_SPEC_EXP) || !(CGS_SPEC_EXP & 1)
    lf_rows_forward<D>(X, twt);
    __syncthreads();
    lf_cols<D, -1>(X, twt);
#endif
    __syncthreads();
    // record: F(obs) [D][P] natural (the packed column in kx = 0, kx = D/2 zero), then H_sym / D^2 [D][P]
    float2 *dst = spec + (int64_t)b * (3 * D * P / 2);
    float *hd = reinterpret_cast<float *>(dst + D * P);
    for (int i = threadIdx.x; i < D * P; i += G::NT) {
        const int ky = i / P, kx = i - ky * P;
        dst[i] = kx == D / 2 ? make_float2(0.f, 0.f) : X[ky * S + kx];
#if !defined(CGS_SPEC_EXP) || !(CGS_SPEC_EXP & 4)  // 4: no H table (timing experiment)
        hd[i] = ctf_sym(cc, D, ky, kx) * (1.f / ((float)D * (float)D));
#endif
    }
}

template <int D, bool kFixed, bool kRowPair>
__global__ void __launch_bounds__(SpecLf<D>::NT, 2) ctf_mse_spec_lf_kernel(
    const float *__restrict__ render, const float *__restrict__ render_scale, const float2 *__restrict__ obs_spec,
    const int64_t *__restrict__ rows, float *__restrict__ upstream, double *__restrict__ loss, int32_t *status) {
    using G = SpecLf<D>;
    constexpr int S = G::S, P = G::P;
    extern __shared__ float2 X[];
    float2 *twt = X + D * S;
    __shared__ double scratch[G::NT / 32];
    const int b = blockIdx.x;
    // image b's record: row b of obs_spec, or row rows[b] of a dataset's resident records
    const float2 *O = obs_spec + (rows ? __ldg(rows + b) : (int64_t)b) * (3 * D * P / 2);
    const float *Hh = reinterpret_cast<const float *>(O + D * P);  // H_sym / D^2, natural [ky][kx]
    {  // warm L2 with the observation record, read after the forward transform
        const char *ob = reinterpret_cast<const char *>(O);
        for (int off = threadIdx.x * 128; off < 3 * D * P * (int)sizeof(float); off += G::NT * 128)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(ob + off));
    }
    lfft::init_twiddles<D>(twt, threadIdx.x, G::NT);
    lf_load_pairs<D, kFixed>(X, render + (int64_t)b * D * D, kFixed ? 1.f / __ldg(render_scale) : 1.f);
    __syncthreads();
#if !defined(CGS_SPEC_EXP) || !(CGS_SPEC_EXP & 1)  // timing experiments only: 1 skips the forward, 2 the inverse
    lf_rows_forward<D>(X, twt);
    __syncthreads();
    lf_cols<D, -1>(X, twt);
#endif
    __syncthreads();
    // F(r) = H F(render) - O (H = Hh D^2, exact: D^2 is a power of two); loss by
    // Parseval (weight 2 on kx = 1..D/2-1, 1 on the packed column); then CTF^T
    // and the 2/D^2 residual scale in place
    const float d2 = (float)(D * D), sc = 2.f / (float)(D * D);
    double acc = 0.0;
    for (int i = threadIdx.x; i < D * P; i += G::NT) {
        const int ky = i / P, kx = i - ky * P;
        if (kx == 0 || kx == D / 2) continue;
        const float h = __ldg(Hh + i);
        const float2 z = X[ky * S + kx], o = __ldg(O + i);
        const float hd = h * d2;
        const float rx = fmaf(hd, z.x, -o.x), ry = fmaf(hd, z.y, -o.y);
        acc += 2.0 * ((double)rx * rx + (double)ry * ry);
        const float hs = h * sc;
        X[ky * S + kx] = make_float2(hs * rx, hs * ry);
    }
    for (int ky = threadIdx.x; ky <= D / 2; ky += G::NT) {  // packed column, pairs (ky, -ky)
        const int ny = (D - ky) & (D - 1);
        const float2 zk = X[ky * S], zn = X[ny * S], ok = __ldg(O + ky * P), on = __ldg(O + ny * P);
        const float h0k = __ldg(Hh + ky * P), hnk = __ldg(Hh + ky * P + D / 2);
        const float h0n = __ldg(Hh + ny * P), hnn = __ldg(Hh + ny * P + D / 2);
        const float pk = 0.5f * (h0k + hnk), qk = 0.5f * (h0k - hnk);
        const float pn = 0.5f * (h0n + hnn), qn = 0.5f * (h0n - hnn);
        // r(k) = d2 (Pc Zp(k) + Qc conj Zp(-k)) - Op(k)
        const float2 rk = make_float2(fmaf(d2, fmaf(pk, zk.x, qk * zn.x), -ok.x),
                                      fmaf(d2, fmaf(pk, zk.y, -qk * zn.y), -ok.y));
        const float2 rn = make_float2(fmaf(d2, fmaf(pn, zn.x, qn * zk.x), -on.x),
                                      fmaf(d2, fmaf(pn, zn.y, -qn * zk.y), -on.y));
        acc += (double)rk.x * rk.x + (double)rk.y * rk.y;
        if (ny != ky) acc += (double)rn.x * rn.x + (double)rn.y * rn.y;
        // CTF^T on the packed residual, the same way, times 2/D^2
        X[ky * S] = make_float2(sc * fmaf(pk, rk.x, qk * rn.x), sc * fmaf(pk, rk.y, -qk * rn.y));
        if (ny != ky) X[ny * S] = make_float2(sc * fmaf(pn, rn.x, qn * rk.x), sc * fmaf(pn, rn.y, -qn * rk.y));
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double tsum = 0.0;
        for (int w = 0; w < G::NT / 32; ++w) tsum += scratch[w];
        const double l = poison_loss(tsum / ((double)D * D * (double)D * D), status);
        loss[b] = l;
        if (status && !isfinite(l)) atomicOr(status, CGS_STATUS_NONFINITE_LOSS);
    }
#if !defined(CGS_SPEC_EXP) || !(CGS_SPEC_EXP & 2)
    lf_cols<D, 1>(X, twt);
    __syncthreads();
    lf_rows_inverse<D, kRowPair>(X, twt, upstream + (int64_t)b * D * D);
#else
    __syncthreads();
    for (int i = threadIdx.x; i < D * D / 2; i += G::NT)
        reinterpret_cast<float2 *>(upstream + (int64_t)b * D * D)[i] = X[(i / D) * 2 * S + (i % D)];
#endif
}

template <int R>
static int launch_obs_spectrum(const float *obs, const double *ctf, double pix, float *spec, int B,
                               cudaStream_t st) {
    constexpr int D = 32 * R, P = D / 2 + 1;
    const size_t smem = (size_t)D * P * sizeof(float2);
    const int rc = ensure_smem_limit((const void *)obs_spectrum_kernel<R>, smem, "obs_spectrum_kernel");
    if (rc) return rc;
#ifdef CGS_SPEC_V1
    obs_spectrum_kernel<R><<<B, kR2cThreads, smem, st>>>(obs, ctf, pix, reinterpret_cast<float2 *>(spec));
    return check_launch("obs_spectrum_kernel");
#else
    (void)smem;
    using G = SpecLf<D>;
    const int rc2 = ensure_smem_limit((const void *)obs_spectrum_lf_kernel<D>, G::smem, "obs_spectrum_lf_kernel");
    if (rc2) return rc2;
    obs_spectrum_lf_kernel<D><<<B, G::NT, G::smem, st>>>(obs, ctf, pix, reinterpret_cast<float2 *>(spec));
    return check_launch("obs_spectrum_lf_kernel");
#endif
}

template <int R, bool kFixed, bool kRowPair>
static int launch_ctf_mse_spec_t(const float *render, const float *render_scale, const float *spec,
                                 const int64_t *rows, int B, float *upstream, double *loss, int32_t *status,
                                 cudaStream_t st) {
    constexpr int D = 32 * R, P = D / 2 + 1;
    const size_t smem = (size_t)D * P * sizeof(float2);
    const int rc = ensure_smem_limit((const void *)ctf_mse_spec_kernel<R, kFixed, kRowPair>, smem, "ctf_mse_spec_kernel");
    if (rc) return rc;
#ifdef CGS_SPEC_V1
    if (rows) return CGS_ERR_UNSUPPORTED;
    ctf_mse_spec_kernel<R, kFixed, kRowPair><<<B, kR2cThreads, smem, st>>>(
        render, render_scale, reinterpret_cast<const float2 *>(spec), upstream, loss, status);
    return check_launch("ctf_mse_spec_kernel");
#else
    (void)smem;
    using G = SpecLf<D>;
    const int rc2 = ensure_smem_limit((const void *)ctf_mse_spec_lf_kernel<D, kFixed, kRowPair>, G::smem,
                                      "ctf_mse_spec_lf_kernel");
    if (rc2) return rc2;
    ctf_mse_spec_lf_kernel<D, kFixed, kRowPair><<<B, G::NT, G::smem, st>>>(
        render, render_scale, reinterpret_cast<const float2 *>(spec), rows, upstream, loss, status);
    return check_launch("ctf_mse_spec_lf_kernel");
#endif
}

template <int R, bool kFixed>
static int launch_ctf_mse_spec(const float *render, const float *render_scale, const float *spec,
                               const int64_t *rows, int B, float *upstream, double *loss, int32_t *status,
                               int layout, cudaStream_t st) {
    if (layout == CGS_LAYOUT_ROWPAIR)
        return launch_ctf_mse_spec_t<R, kFixed, true>(render, render_scale, spec, rows, B, upstream, loss, status, st);
    if (layout == CGS_LAYOUT_NATURAL)
        return launch_ctf_mse_spec_t<R, kFixed, false>(render, render_scale, spec, rows, B, upstream, loss, status,
                                                       st);
    return CGS_ERR_ARG;
}

template <int R>
static int launch_ctf_mse_r2c(const float *render, const float *obs, int B, double pix, const double *ctf,
                              float *model, float *upstream, double *loss, int32_t *status, cudaStream_t st) {
    constexpr int D = 32 * R, P = D / 2 + 1;
    const size_t smem = (size_t)D * P * (sizeof(float2) + sizeof(float));
    const int rc = ensure_smem_limit((const void *)ctf_mse_r2c_kernel<R>, smem, "ctf_mse_r2c_kernel");
    if (rc) return rc;
    ctf_mse_r2c_kernel<R><<<B, kR2cThreads, smem, st>>>(render, obs, ctf, pix, model, upstream, loss, status);
    return check_launch("ctf_mse_r2c_kernel");
}

template <int R>
static int launch_ctf_mse_fused(const float *render, const float *obs, int B, double pix, const double *ctf,
                                float *model, float *upstream, double *loss, int32_t *status, cudaStream_t st) {
    constexpr int D = 32 * R;
    const size_t smem = (size_t)D * (D + 1) * sizeof(float2);
    const int rc = ensure_smem_limit((const void *)ctf_mse_fused_kernel<R>, smem, "ctf_mse_fused_kernel");
    if (rc) return rc;
    ctf_mse_fused_kernel<R><<<(B + 1) / 2, kFusedThreads, smem, st>>>(render, obs, B, pix, ctf, model, upstream,
                                                                      loss, status);
    return check_launch("ctf_mse_fused_kernel");
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


// ---- spectral K4 through cuFFT, for the sizes without a one-CTA line-FFT
// kernel (C4: a 256^2 half spectrum is 264 KB, more than one CTA's shared
// memory).  Same records and loss as the line-FFT path, natural [ky][kx] half
// spectrum: F(obs) then H_sym / D^2.  Per step: int32 render -> float (scale),
// R2C, one filter/loss kernel over the half spectrum, C2R -- one transform
// pair instead of cgs_ctf_mse's two, and H from the records.
constexpr int kSpecFftThreads = 256, kSpecFftElems = 8 * kSpecFftThreads;  // half-spectrum elements per CTA

__host__ __device__ inline int spec_fft_ctas(int D) { return (D * (D / 2 + 1) + kSpecFftElems - 1) / kSpecFftElems; }
// record stride in float2: F (n complex) + H (n floats), padded to an even float count (odd D: n odd)
__host__ __device__ inline int64_t spec_fft_record_f2(int D) {
    const int64_t n = (int64_t)D * (D / 2 + 1);
    return (3 * n + (n & 1)) / 2;
}

// out = in / scale (the fixed-point render as floats, the R2C's input)
__global__ void __launch_bounds__(256) fixed_scale_kernel(const int *__restrict__ in, float *__restrict__ out,
                                                          int64_t count, const float *__restrict__ scale_ptr) {
    const float inv = 1.f / __ldg(scale_ptr);
    const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4;
    if (i + 3 < count) {
        const int4 v = __ldg(reinterpret_cast<const int4 *>(in + i));
        *reinterpret_cast<float4 *>(out + i) = make_float4((float)v.x * inv, (float)v.y * inv, (float)v.z * inv,
                                                           (float)v.w * inv);
    } else {
        for (int64_t j = i; j < count; ++j) out[j] = (float)in[j] * inv;
    }
}

// record b: F(obs) as cuFFT left it, then H_sym / D^2 (grid: CTAs per image x B)
__global__ void __launch_bounds__(kSpecFftThreads) obs_record_fft_kernel(const float2 *__restrict__ spectrum,
                                                                         const double *__restrict__ ctf, int D,
                                                                         double pix, float2 *__restrict__ rec) {
    const int b = blockIdx.y, P = D / 2 + 1, n = D * P;
    __shared__ CtfConst cc;
    if (threadIdx.x == 0) {
        CtfConst c = load_ctf(ctf + 8 * (int64_t)b, D, pix);
        c.inv_dA = 1.0 / c.dA;
        c.pl = kPiD * c.lam;
        c.cs3 = 0.5 * kPiD * c.cs * c.lam * c.lam * c.lam;
        cc = c;
    }
    __syncthreads();
    const float2 *src = spectrum + (int64_t)b * n;
    float2 *dst = rec + (int64_t)b * spec_fft_record_f2(D);
    float *hd = reinterpret_cast<float *>(dst + n);
    const float inv_d2 = 1.f / ((float)D * (float)D);
    const int end = min(n, (int)(blockIdx.x + 1) * kSpecFftElems);
    for (int i = blockIdx.x * kSpecFftElems + threadIdx.x; i < end; i += kSpecFftThreads) {
        const int ky = i / P, kx = i - ky * P;
        dst[i] = src[i];
        hd[i] = ctf_sym(cc, D, ky, kx) * inv_d2;
    }
}

// r = H F(render) - F(obs) over the half spectrum in place of F(render), then
// CTF^T and the 2/D^2 residual scale (C2R is unnormalised: Hh = H / D^2 gives
// the 1/D^2).  Loss by Parseval, weight 1 on the self-conjugate columns kx = 0
// and D/2 (even D), 2 elsewhere; per-CTA fp64 sums, the image's last CTA adds
// them in CTA order (deterministic) and resets its counter.
__global__ void __launch_bounds__(kSpecFftThreads) ctf_mse_spec_fft_kernel(
    float2 *__restrict__ spectrum, const float2 *__restrict__ obs_spec, const int64_t *__restrict__ rows, int D,
    double *__restrict__ part, unsigned *__restrict__ count, double *__restrict__ loss, int32_t *status) {
    const int b = blockIdx.y, P = D / 2 + 1, n = D * P, K = gridDim.x;
    const float2 *O = obs_spec + (rows ? __ldg(rows + b) : (int64_t)b) * spec_fft_record_f2(D);
    const float *Hh = reinterpret_cast<const float *>(O + n);
    float2 *Z = spectrum + (int64_t)b * n;
    const float d2 = (float)D * (float)D, sc = 2.f / d2;
    constexpr int kPer = kSpecFftElems / kSpecFftThreads;
    const int i0 = blockIdx.x * kSpecFftElems + threadIdx.x;
    // all loads of the thread's elements first: one DRAM round trip, not kPer
    float2 z[kPer], o[kPer];
    float h[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const int i = i0 + j * kSpecFftThreads;
        if (i < n) {
            z[j] = Z[i];
            o[j] = __ldg(O + i);
            h[j] = __ldg(Hh + i);
        }
    }
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const int i = i0 + j * kSpecFftThreads;
        if (i < n) {
            const int kx = i % P;
            const float hd = h[j] * d2;
            const float rx = fmaf(hd, z[j].x, -o[j].x), ry = fmaf(hd, z[j].y, -o[j].y);
            const double w = (kx == 0 || (!(D & 1) && kx == D / 2)) ? 1.0 : 2.0;
            acc += w * ((double)rx * rx + (double)ry * ry);
            const float hs = h[j] * sc;
            Z[i] = make_float2(hs * rx, hs * ry);
        }
    }
    __shared__ double scratch[kSpecFftThreads / 32];
    __shared__ bool last;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kSpecFftThreads / 32; ++w) t += scratch[w];
        part[(int64_t)b * K + blockIdx.x] = t;
        __threadfence();
        last = atomicAdd(count + b, 1u) == (unsigned)(K - 1);
        if (last) {
            __threadfence();
            double s = 0.0;
            for (int k = 0; k < K; ++k) s += *(volatile const double *)(part + (int64_t)b * K + k);
            const double l = poison_loss(s / ((double)d2 * (double)d2), status);
            loss[b] = l;
            if (status && !isfinite(l)) atomicOr(status, CGS_STATUS_NONFINITE_LOSS);
            count[b] = 0;
        }
    }
}

// natural -> CGS_LAYOUT_ROWPAIR in place, one CTA per row pair (even D): the
// backward's region staging then copies float2 pairs (2% of K5 at 256^2)
constexpr int kInterleaveThreads = 128;
__global__ void __launch_bounds__(kInterleaveThreads) rowpair_interleave_kernel(float *__restrict__ buf, int D) {
    extern __shared__ float rows[];  // [2][D]
    float *p = buf + (int64_t)blockIdx.x * 2 * D;
    for (int x = threadIdx.x; x < 2 * D; x += kInterleaveThreads) rows[x] = p[x];
    __syncthreads();
    float2 *q = reinterpret_cast<float2 *>(p);
    for (int x = threadIdx.x; x < D; x += kInterleaveThreads) q[x] = make_float2(rows[x], rows[D + x]);
}

static int spec_fft_setup(FftPlan *p, int32_t B, cgs_grid grid, cudaStream_t st) {
    if (!p || p->D != grid.size || p->B != B) return CGS_ERR_ARG;
    if (B > 65535) {  // images on the grid's y dimension
        set_error_detail("cgs spectral fft", "batch above 65535 images");
        return CGS_ERR_UNSUPPORTED;
    }
    int rc = cufft_check(cufftSetStream(p->r2c, st), "cufftSetStream");
    if (rc) return rc;
    return cufft_check(cufftSetStream(p->c2r, st), "cufftSetStream");
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
    // fused single-kernel path for D = 32 / 64 / 128 (CGS_CTF_CUFFT=1 forces cuFFT, for A/B)
    static const bool force_cufft = getenv("CGS_CTF_CUFFT") && getenv("CGS_CTF_CUFFT")[0] == '1';
    if (ctf && !force_cufft && render != upstream && grid.pixel_size > 0 && B > 0) {
        cudaStream_t st = (cudaStream_t)stream;
        static const bool pair_kernel = getenv("CGS_CTF_PAIR") && getenv("CGS_CTF_PAIR")[0] == '1';
        if (!pair_kernel && (grid.size == 128 || grid.size == 64)) {
            if (grid.size == 128)
                return launch_ctf_mse_r2c<4>(render, obs, B, grid.pixel_size, ctf, model, upstream, loss, status, st);
            return launch_ctf_mse_r2c<2>(render, obs, B, grid.pixel_size, ctf, model, upstream, loss, status, st);
        }
        if (grid.size == 128)
            return launch_ctf_mse_fused<4>(render, obs, B, grid.pixel_size, ctf, model, upstream, loss, status, st);
        if (grid.size == 64)
            return launch_ctf_mse_fused<2>(render, obs, B, grid.pixel_size, ctf, model, upstream, loss, status, st);
        if (grid.size == 32)
            return launch_ctf_mse_fused<1>(render, obs, B, grid.pixel_size, ctf, model, upstream, loss, status, st);
    }
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

extern "C" int64_t cgs_obs_spectrum_elems(int32_t size, int32_t B) {
    if (size != 64 && size != 128) return 0;
    return (int64_t)B * 3 * size * (size / 2 + 1);  // floats: F(obs) complex + H_sym / D^2
}

extern "C" int cgs_obs_spectrum(const float *obs, const double *ctf, int32_t B, cgs_grid grid, float *spec,
                                void *stream) {
    if (!obs || !ctf || !spec || B <= 0 || !(grid.pixel_size > 0)) return CGS_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    if (grid.size == 128) return launch_obs_spectrum<4>(obs, ctf, grid.pixel_size, spec, B, st);
    if (grid.size == 64) return launch_obs_spectrum<2>(obs, ctf, grid.pixel_size, spec, B, st);
    set_error_detail("cgs_obs_spectrum", "image size must be 64 or 128");
    return CGS_ERR_UNSUPPORTED;
}

extern "C" int cgs_ctf_mse_spectral(const float *render, const float *obs_spec, int32_t B, cgs_grid grid,
                                    float *upstream, double *loss, int32_t *status, int32_t upstream_layout,
                                    void *stream) {
    if (!render || !obs_spec || !upstream || !loss || B <= 0 || render == upstream) return CGS_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    if (grid.size == 128)
        return launch_ctf_mse_spec<4, false>(render, nullptr, obs_spec, nullptr, B, upstream, loss, status, upstream_layout, st);
    if (grid.size == 64)
        return launch_ctf_mse_spec<2, false>(render, nullptr, obs_spec, nullptr, B, upstream, loss, status, upstream_layout, st);
    set_error_detail("cgs_ctf_mse_spectral", "image size must be 64 or 128");
    return CGS_ERR_UNSUPPORTED;
}

extern "C" int cgs_ctf_mse_spectral_fixed(const int32_t *render_fixed, const float *render_scale,
                                          const float *obs_spec, int32_t B, cgs_grid grid, float *upstream,
                                          double *loss, int32_t *status, int32_t upstream_layout, void *stream) {
    const float *r = reinterpret_cast<const float *>(render_fixed);
    if (!r || !render_scale || !obs_spec || !upstream || !loss || B <= 0 || r == upstream) return CGS_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    if (grid.size == 128)
        return launch_ctf_mse_spec<4, true>(r, render_scale, obs_spec, nullptr, B, upstream, loss, status, upstream_layout, st);
    if (grid.size == 64)
        return launch_ctf_mse_spec<2, true>(r, render_scale, obs_spec, nullptr, B, upstream, loss, status, upstream_layout, st);
    set_error_detail("cgs_ctf_mse_spectral_fixed", "image size must be 64 or 128");
    return CGS_ERR_UNSUPPORTED;
}

extern "C" int cgs_ctf_mse_spectral_fixed_rows(const int32_t *render_fixed, const float *render_scale,
                                               const float *obs_spec, const int64_t *rows, int32_t B, cgs_grid grid,
                                               float *upstream, double *loss, int32_t *status,
                                               int32_t upstream_layout, void *stream) {
    const float *r = reinterpret_cast<const float *>(render_fixed);
    if (!r || !render_scale || !obs_spec || !rows || !upstream || !loss || B <= 0 || r == upstream)
        return CGS_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    if (grid.size == 128)
        return launch_ctf_mse_spec<4, true>(r, render_scale, obs_spec, rows, B, upstream, loss, status, upstream_layout,
                                            st);
    if (grid.size == 64)
        return launch_ctf_mse_spec<2, true>(r, render_scale, obs_spec, rows, B, upstream, loss, status, upstream_layout,
                                            st);
    set_error_detail("cgs_ctf_mse_spectral_fixed_rows", "image size must be 64 or 128");
    return CGS_ERR_UNSUPPORTED;
}

extern "C" int64_t cgs_obs_spectrum_fft_elems(int32_t size, int32_t B) {
    if (size < 2 || B < 0) return 0;
    return (int64_t)B * 2 * spec_fft_record_f2(size);
}

extern "C" size_t cgs_spectral_fft_workspace_bytes(int32_t size, int32_t B) {
    if (size < 2 || B <= 0) return 0;
    return (size_t)B * spec_fft_ctas(size) * sizeof(double) + (size_t)B * sizeof(unsigned);
}

extern "C" int cgs_obs_spectrum_fft(void *plan, const float *obs, const double *ctf, int32_t B, cgs_grid grid,
                                    void *spectrum, float *spec, void *stream) {
    if (!obs || !ctf || !spec || !spectrum || B <= 0 || !(grid.pixel_size > 0)) return CGS_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    int rc = spec_fft_setup((FftPlan *)plan, B, grid, st);
    if (rc) return rc;
    FftPlan *p = (FftPlan *)plan;
    rc = cufft_check(cufftExecR2C(p->r2c, (cufftReal *)obs, (cufftComplex *)spectrum), "cufftExecR2C");
    if (rc) return rc;
    const int D = grid.size;
    obs_record_fft_kernel<<<dim3(spec_fft_ctas(D), B), kSpecFftThreads, 0, st>>>(
        (const float2 *)spectrum, ctf, D, grid.pixel_size, (float2 *)spec);
    return check_launch("obs_record_fft_kernel");
}

extern "C" int cgs_ctf_mse_spectral_fft(void *plan, const int32_t *render_fixed, const float *render_scale,
                                        const float *obs_spec, const int64_t *rows, int32_t B, cgs_grid grid,
                                        void *spectrum, void *workspace, float *upstream, double *loss,
                                        int32_t *status, int32_t upstream_layout, void *stream) {
    if (!render_fixed || !render_scale || !obs_spec || !spectrum || !workspace || !upstream || !loss || B <= 0 ||
        (const void *)render_fixed == (const void *)upstream)
        return CGS_ERR_ARG;
    if (upstream_layout != CGS_LAYOUT_NATURAL && upstream_layout != CGS_LAYOUT_ROWPAIR) return CGS_ERR_ARG;
    if (upstream_layout == CGS_LAYOUT_ROWPAIR && (grid.size & 1)) return CGS_ERR_UNSUPPORTED;
    cudaStream_t st = (cudaStream_t)stream;
    int rc = spec_fft_setup((FftPlan *)plan, B, grid, st);
    if (rc) return rc;
    FftPlan *p = (FftPlan *)plan;
    const int D = grid.size, K = spec_fft_ctas(D);
    const int64_t count = (int64_t)B * D * D;
    fixed_scale_kernel<<<(unsigned)(((count + 3) / 4 + 255) / 256), 256, 0, st>>>(render_fixed, upstream, count,
                                                                                 render_scale);
    rc = check_launch("fixed_scale_kernel");
    if (rc) return rc;
    rc = cufft_check(cufftExecR2C(p->r2c, (cufftReal *)upstream, (cufftComplex *)spectrum), "cufftExecR2C");
    if (rc) return rc;
    double *part = (double *)workspace;
    unsigned *cnt = (unsigned *)(part + (int64_t)B * K);
    ctf_mse_spec_fft_kernel<<<dim3(K, B), kSpecFftThreads, 0, st>>>((float2 *)spectrum, (const float2 *)obs_spec,
                                                                   rows, D, part, cnt, loss, status);
    rc = check_launch("ctf_mse_spec_fft_kernel");
    if (rc) return rc;
    rc = cufft_check(cufftExecC2R(p->c2r, (cufftComplex *)spectrum, (cufftReal *)upstream), "cufftExecC2R");
    if (rc || upstream_layout == CGS_LAYOUT_NATURAL) return rc;
    rowpair_interleave_kernel<<<(unsigned)((int64_t)B * D / 2), kInterleaveThreads, 2 * D * sizeof(float), st>>>(
        upstream, D);
    return check_launch("rowpair_interleave_kernel");
}

extern "C" int cgs_fourier_filter(const float *in, float *out, int32_t B, cgs_grid grid, const double *ctf,
                                  const double *shifts, void *stream) {
    if (!in || !out || B <= 0 || grid.size < 1) return CGS_ERR_ARG;
    if (ctf && !(grid.pixel_size > 0)) return CGS_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    if (grid.size == 128) return launch_fourier_filter<4>(in, out, B, grid.pixel_size, ctf, shifts, st);
    if (grid.size == 64) return launch_fourier_filter<2>(in, out, B, grid.pixel_size, ctf, shifts, st);
    if (grid.size == 32) return launch_fourier_filter<1>(in, out, B, grid.pixel_size, ctf, shifts, st);
    set_error_detail("cgs_fourier_filter", "image size must be 32, 64 or 128");
    return CGS_ERR_UNSUPPORTED;
}
