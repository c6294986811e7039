// Device helpers shared by every stencil kernel: the per-point arithmetic of the three
// forms, the fused epilogue (store, peer store, source injection, max|u|).
#pragma once
#include <cuda_runtime.h>

#include "swb_internal.h"
#include <climits>

namespace swb {

// Runtime selection among three pointers without dynamic indexing of a parameter array
// (which would force a local-memory copy of the kernel parameters).
template <typename T>
__device__ __forceinline__ T pick3(T a, T b, T c, int i) {
    return i == 0 ? a : (i == 1 ? b : c);
}

__device__ __forceinline__ unsigned abs_bits(float v) { return __float_as_uint(v) & 0x7fffffffu; }

// mine = max(mine, |x|, |y|, |z|, |w|) on the max|u| bits: two FMNMX3.NAN with |.| source
// modifiers instead of four masks and three integer max.  For non-NaN values this is the
// integer max of abs_bits (non-negative floats order like their bits); any NaN gives NaN,
// which is still above +inf as bits.
__device__ __forceinline__ unsigned fold_abs4(unsigned mine, float x, float y, float z, float w) {
    float r, r2;
    asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(fabsf(x)), "f"(fabsf(y)), "f"(__uint_as_float(mine)));
    asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r2) : "f"(fabsf(z)), "f"(fabsf(w)), "f"(r));
    return __float_as_uint(r2);
}

// Block-wide max of `mine`, then one conditional atomicMax per block into *dst.
// Non-negative floats order like their bit patterns; |NaN| > +inf in that order, so a
// non-finite cell always wins and the host maps bits >= 0x7f800000 to NaN
// (max_abs_interior returns NaN for any non-finite cell, src/executor.cpp:526-544).
__device__ __forceinline__ void block_max_commit(unsigned mine, unsigned* dst) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine = max(mine, __shfl_xor_sync(0xffffffffu, mine, o));
    __shared__ unsigned red[32];
    const int lane = threadIdx.x & 31;
    const int warp = (threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z)) >> 5;
    const int nwarps = (blockDim.x * blockDim.y * blockDim.z + 31) >> 5;
    if (lane == 0) red[warp] = mine;
    __syncthreads();
    if (warp == 0) {
        unsigned v = lane < nwarps ? red[lane] : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (lane == 0 && v > *reinterpret_cast<volatile unsigned*>(dst)) atomicMax(dst, v);
    }
}

// Source injection, exactly the reference's point cluster (src/wave_model.cpp:117-124 solved
// as u[t+1] = u[t+1] + dt*dt*src_amp/m, evaluated in double with one division,
// src/executor.cpp:255-283) applied to the already FP32-rounded stencil value: two roundings,
// as in the reference where the stencil store precedes the injection store.
__device__ __forceinline__ float inject_source(float v, float amp, float m, double dtd) {
    double t = __dmul_rn(__dmul_rn(dtd, dtd), static_cast<double>(amp));
    t = __ddiv_rn(t, static_cast<double>(m));
    return static_cast<float>(__dadd_rn(static_cast<double>(v), t));
}

// ---- plain (basic DSE) form, FP64, bit-exact with the interpreter -------------------
// Term order and grouping of the solved update (see oracle/port/wave_port.c point_update):
//   2*m*u/(dt*dt*I) - m*up/(dt*dt*I) + 1/2*damp*up/(dt*I) + sum_d sum_k (+-)|c_k|*u_k/(h_d*h_d*I)
// with I = m/(dt*dt) + 1/2*damp/dt.  __d*_rn intrinsics forbid FMA contraction, matching the
// FMA-free x86 interpreter (src/executor.cpp:448-451).
template <int H>
__device__ __forceinline__ float plain_f64_point(const float* __restrict__ ut, long long i,
                                                 long long s0, long long s1, float u0f,
                                                 float upf, float mf, float df, const Coef& K) {
    const double dt = static_cast<double>(K.dt);
    const double m = mf, dmp = df, u0 = u0f, up = upf;
    const double dtdt = __dmul_rn(dt, dt);
    const double I = __dadd_rn(__ddiv_rn(m, dtdt), __ddiv_rn(__dmul_rn(0.5, dmp), dt));
    const double dden = __dmul_rn(dtdt, I);
    double acc = __ddiv_rn(__dmul_rn(__dmul_rn(2.0, m), u0), dden);
    acc = __dsub_rn(acc, __ddiv_rn(__dmul_rn(m, up), dden));
    acc = __dadd_rn(acc, __ddiv_rn(__dmul_rn(__dmul_rn(0.5, dmp), up), __dmul_rn(dt, I)));
    const long long st[3] = {s0, s1, 1};
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const double hh = static_cast<double>(K.h[d]);
        const double den = __dmul_rn(__dmul_rn(hh, hh), I);
#pragma unroll
        for (int k = -H; k <= H; ++k) {
            const float cf = K.c[k < 0 ? -k : k];
            const double ca = static_cast<double>(fabsf(cf));
            const double v = static_cast<double>(k == 0 ? u0f : ut[i + k * st[d]]);
            const double t = __ddiv_rn(__dmul_rn(ca, v), den);
            acc = cf < 0.f ? __dsub_rn(acc, t) : __dadd_rn(acc, t);
        }
    }
    return static_cast<float>(acc);
}

// ---- plain form, FP32 term by term (the paper's OPS user kernel k0 in C float) --------
template <int H>
__device__ __forceinline__ float plain_f32_point(const float* __restrict__ ut, long long i,
                                                 long long s0, long long s1, float u0,
                                                 float up, float m, float dmp, const Coef& K) {
    const float dt = K.dt;
    const float dtdt = __fmul_rn(dt, dt);
    const float I = __fadd_rn(__fdiv_rn(m, dtdt), __fdiv_rn(__fmul_rn(0.5f, dmp), dt));
    const float dden = __fmul_rn(dtdt, I);
    float acc = __fdiv_rn(__fmul_rn(__fmul_rn(2.0f, m), u0), dden);
    acc = __fsub_rn(acc, __fdiv_rn(__fmul_rn(m, up), dden));
    acc = __fadd_rn(acc, __fdiv_rn(__fmul_rn(__fmul_rn(0.5f, dmp), up), __fmul_rn(dt, I)));
    const long long st[3] = {s0, s1, 1};
    // (the axes are not unrolled at the widest stencils: all 3(2H+1) hoisted loads would not
    // fit the register file; the term order is unchanged)
#pragma unroll(H >= 7 ? 1 : 3)
    for (int d = 0; d < 3; ++d) {
        const float hh = K.h[d];
        const float den = __fmul_rn(__fmul_rn(hh, hh), I);
#pragma unroll
        for (int k = -H; k <= H; ++k) {
            const float cf = K.c[k < 0 ? -k : k];
            const float v = k == 0 ? u0 : ut[i + k * st[d]];
            const float t = __fdiv_rn(__fmul_rn(fabsf(cf), v), den);
            acc = cf < 0.f ? __fsub_rn(acc, t) : __fadd_rn(acc, t);
        }
    }
    return acc;
}

// ---- factorised form: FP32 Laplacian, k=1 ring in difference form, FP64 combine ------
// One space dimension of sum_k c_k u(x+k e_d) rewritten as
//   c1*((u_-1 - u0) + (u_+1 - u0)) + sum_{k>=2} c_k*(u_-k + u_+k)   [+ (c0 + 2 c1) u0, added in FP64]
// summed far-to-near so the small terms accumulate first.  `get(k)` returns u(x + k e_d).
template <int H, typename Get>
__device__ __forceinline__ float lap_axis(const Coef& K, float u0, Get get) {
    float s = 0.f;
#pragma unroll
    for (int k = H; k >= 2; --k) s = fmaf(K.c[k], get(-k) + get(k), s);
    return fmaf(K.c[1], (get(-1) - u0) + (get(1) - u0), s);
}

// Final combine of the corrected aggressive form (src/pipeline.cpp:467-512 with the sign fix):
//   u+ = (a(2u - up) + b up + L) / (a + b),  a = m/dt^2, b = damp/(2dt),  L = sum_d S_d/h_d^2
// in FP64, so the only FP32 rounding besides the final store is inside the S_d sums.
__device__ __forceinline__ float combine_f64(const Coef& K, double L, float u0, float up, float m,
                                             float dmp) {
    const double a = static_cast<double>(m) * K.inv_dt2;
    const double b = static_cast<double>(dmp) * K.half_inv_dt;
    const double num = fma(2.0 * a, static_cast<double>(u0), fma(-(a - b), static_cast<double>(up), L));
    return static_cast<float>(num / (a + b));
}

// FP32 combine with no systematic coefficient rounding:
//   u+ - u = [ (m - g)(u - up) + Lr*(dt/h)^2 ] / (m + g),   g = damp*dt/2,
// where Lr = S + 3R*u is the raw (unscaled) Laplacian sum and (dt/h)^2 is applied as an
// exact hi+lo float pair; the quotient is an IEEE division and the final add is the only
// rounding at the scale of u (the interpreter's one final store rounding).
__device__ __forceinline__ float combine_f32(float Lr, float u0, float up, float m, float dmp,
                                             float kap_hi, float kap_lo, float half_dt) {
    const float Lk = fmaf(Lr, kap_hi, Lr * kap_lo);
    const float g = dmp * half_dt;
    const float num = fmaf(m - g, u0 - up, Lk);
    return u0 + __fdiv_rn(num, m + g);
}

__device__ __forceinline__ double lap_total(const Coef& K, float s0, float s1, float s2, float u0) {
    if (K.iso) {
        const float s = (s0 + s1) + s2;
        return fma(3.0 * K.R_d, static_cast<double>(u0), static_cast<double>(s)) * K.inv_h2[0];
    }
    double L = fma(K.R_d, static_cast<double>(u0), static_cast<double>(s0)) * K.inv_h2[0];
    L = fma(fma(K.R_d, static_cast<double>(u0), static_cast<double>(s1)), K.inv_h2[1], L);
    L = fma(fma(K.R_d, static_cast<double>(u0), static_cast<double>(s2)), K.inv_h2[2], L);
    return L;
}

}  // namespace swb
