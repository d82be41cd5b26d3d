// Line FFTs for the spectral K4 (optics.cu): one length-D complex transform
// per group of 8 threads, D = 8 V (V = 8 or 16 values per thread).
//
// Round 1's WarpFft ran one transform per warp with D / 32 values per lane and
// did five of its seven radix-2 stages across lanes by shuffles (~200 warp
// instructions per 128-point line, a long dependent shuffle chain).  Here a
// line is two register steps and one exchange through the line's own
// shared-memory slots (four-step FFT, D = V x 8):
//   A: thread t (0..7) holds x[t + 8 n1], n1 < V, and takes a V-point DFT in
//      registers; then multiplies element k1 by W_D^(t k1) (a table);
//   exchange: element k1 goes to slot 8 k1 + ((t + k1) & 7) (the rotation
//      keeps the reads below conflict-free);
//   B: thread t reads rows k1 = t + 8 h (h < V / 8) of all 8 threads and takes
//      8-point DFTs: X[k1 + V k2] = sum_t' W_8^(t' k2) Y_t'[k1].
// Inputs and outputs are in natural order.  The small DFTs are fully unrolled
// Cooley-Tukey (decimation in time) with compile-time twiddles, the trivial
// ones (1, -1, +-i, (1 +- i)/sqrt 2) as adds and swaps.  The inverse (SIGN =
// +1) is the same network with conjugate twiddles, unscaled.
#pragma once

#include <type_traits>

#include "common.cuh"

namespace cgs {
namespace lfft {

template <int I, int N, class F>
__device__ __forceinline__ void static_for(F &&f) {
    if constexpr (I < N) {
        f(std::integral_constant<int, I>{});
        static_for<I + 1, N>(f);
    }
}

__host__ __device__ constexpr float cos16(int m) {  // cos(2 pi m / 16)
    m &= 15;
    return m == 0 ? 1.f
         : m == 1 || m == 15 ? 0.92387953251128674f
         : m == 2 || m == 14 ? 0.70710678118654752f
         : m == 3 || m == 13 ? 0.38268343236508977f
         : m == 4 || m == 12 ? 0.f
         : m == 5 || m == 11 ? -0.38268343236508977f
         : m == 6 || m == 10 ? -0.70710678118654752f
         : m == 7 || m == 9 ? -0.92387953251128674f
                             : -1.f;
}

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a conj(b)
    return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}

// v W_N^E, W_N = exp(SIGN 2 pi i / N), N | 16, E compile time
template <int N, int E, int SIGN>
__device__ __forceinline__ float2 tw(float2 v) {
    constexpr int e = ((E % N) + N) % N;
    constexpr int m = e * (16 / N);  // in units of 2 pi / 16
    if constexpr (m == 0) {
        return v;
    } else if constexpr (m == 8) {
        return make_float2(-v.x, -v.y);
    } else if constexpr (m == 4 || m == 12) {
        // exp(SIGN i pi / 2) = SIGN i for m = 4; its negative for m = 12
        constexpr int s = (m == 4 ? SIGN : -SIGN);
        return s > 0 ? make_float2(-v.y, v.x) : make_float2(v.y, -v.x);
    } else if constexpr (m == 2 || m == 6 || m == 10 || m == 14) {
        // (c, SIGN s) with |c| = |s| = 1/sqrt 2
        constexpr float c = cos16(m), s = SIGN * cos16(m - 4);
        constexpr float a = c < 0.f ? -c : c;
        const float re = (c > 0.f ? v.x : -v.x) - (s > 0.f ? v.y : -v.y);
        const float im = (c > 0.f ? v.y : -v.y) + (s > 0.f ? v.x : -v.x);
        return make_float2(a * re, a * im);
    } else {
        constexpr float c = cos16(m), s = SIGN * cos16(m - 4);
        return make_float2(fmaf(v.x, c, -v.y * s), fmaf(v.x, s, v.y * c));
    }
}

// in-place DFT of N = 2, 4, 8 or 16 registers, natural order in and out
template <int N, int SIGN>
__device__ __forceinline__ void dft(float2 *v) {
    if constexpr (N == 2) {
        const float2 a = v[0], b = v[1];
        v[0] = cadd(a, b);
        v[1] = csub(a, b);
    } else if constexpr (N == 4) {
        const float2 a = cadd(v[0], v[2]), b = csub(v[0], v[2]);
        const float2 c = cadd(v[1], v[3]), d = tw<4, 1, SIGN>(csub(v[1], v[3]));
        v[0] = cadd(a, c);
        v[2] = csub(a, c);
        v[1] = cadd(b, d);
        v[3] = csub(b, d);
    } else {
        // N = R M, decimation in time: Y_r = DFT_M(x[R m + r]),
        // X[k1 + M k2] = DFT_R over r of W_N^(r k1) Y_r[k1]
        constexpr int R = 4, M = N / R;
        float2 y[R][M];
        static_for<0, R>([&](auto r) {
            static_for<0, M>([&](auto m) { y[r][m] = v[R * m + r]; });
            dft<M, SIGN>(y[r]);
        });
        static_for<0, M>([&](auto k1) {
            float2 z[R];
            static_for<0, R>([&](auto r) { z[r] = tw<N, decltype(r)::value * decltype(k1)::value, SIGN>(y[r][k1]); });
            dft<R, SIGN>(z);
            static_for<0, R>([&](auto k2) { v[k1 + M * k2] = z[k2]; });
        });
    }
}

// Twiddles of step A: table[k1 * 8 + t] = W_D^(t k1) (forward sign), k1 < V.
template <int D>
__device__ __forceinline__ void init_twiddles(float2 *table, int tid, int nthreads) {
    constexpr int V = D / 8;
    for (int i = tid; i < V * 8; i += nthreads) {
        const int k1 = i >> 3, t = i & 7;
        float sn, cs;
        sincospif(-2.f * (float)(t * k1) / (float)D, &sn, &cs);
        table[i] = make_float2(cs, sn);
    }
}

// One length-D transform by the 8 threads of a group (t = 0..7, all in one warp).
//   in(n)    -> float2   input element n
//   slot(s)  -> float2 * exchange storage s in [0, D) (the line's own slots)
//   out(k, v)             output element k (natural order)
// Every in() read happens before any slot() write; with kOutInPlace every
// exchange read happens before any out() write (out() may then reuse the slots).
template <int D, int SIGN, bool kOutInPlace, class In, class Slot, class Out>
__device__ __forceinline__ void line(int t, const float2 *__restrict__ twt, In in, Slot slot, Out out) {
    constexpr int V = D / 8, H = V / 8;
    float2 v[V];
#pragma unroll
    for (int n = 0; n < V; ++n) v[n] = in(t + 8 * n);
    dft<V, SIGN>(v);
#pragma unroll
    for (int k1 = 1; k1 < V; ++k1) {
        const float2 w = twt[k1 * 8 + t];
        v[k1] = SIGN < 0 ? cmul(v[k1], w) : cmulc(v[k1], w);
    }
    __syncwarp();
#pragma unroll
    for (int k1 = 0; k1 < V; ++k1) *slot(8 * k1 + ((t + k1) & 7)) = v[k1];
    __syncwarp();
#pragma unroll
    for (int h = 0; h < H; ++h) {
        const int k1 = t + 8 * h;
#pragma unroll
        for (int u = 0; u < 8; ++u) v[8 * h + u] = *slot(8 * k1 + ((u + k1) & 7));
    }
    if (kOutInPlace) __syncwarp();
#pragma unroll
    for (int h = 0; h < H; ++h) {
        dft<8, SIGN>(v + 8 * h);
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) out(t + 8 * h + V * k2, v[8 * h + k2]);
    }
}

}  // namespace lfft
}  // namespace cgs
