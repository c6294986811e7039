// Device helpers of the TMA stencil kernel (k_tma.cu): mbarrier/TMA PTX
// wrappers, packed FP32x2 arithmetic, tensor-map bundle, work schedule.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "k_common.cuh"
#include "kernels.h"

namespace swb {
namespace tma {

constexpr int kT2 = 64;  // output cols per tile (16 lanes x float4)

struct Maps {
    CUtensorMap u[3];     // halo box (W2, T1+2H, 1)
    CUtensorMap a[3];     // aux box (64, T1, 1) over the u levels (for u[t-1])
    CUtensorMap m;        // aux box over m
    CUtensorMap damp;     // aux box over damp
};

struct Sched {
    int nyt, nzt, ncol;   // column tiles
    int np;               // planes to update per column
    int nchunk;           // dim-0 chunks per column (work items = ncol * nchunk)
    int y0, y1, z0, z1, zs, x0;
    const unsigned char* dflag;  // [ncol][np]: damp tile non-zero (null = always load damp)
};

__device__ __forceinline__ unsigned smem_addr(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// try_wait with a suspend-time hint: the waiting warp sleeps in hardware until the phase
// completes (or the hint expires) instead of waking to re-poll and taking issue slots.
#ifndef SWB_MBAR_SUSPEND_NS
#define SWB_MBAR_SUSPEND_NS 20000
#endif
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(bar),
        "r"(parity), "r"(SWB_MBAR_SUSPEND_NS)
        : "memory");
}
__device__ __forceinline__ void tma_load3(unsigned dst, const CUtensorMap* map, int c0, int c1,
                                          int c2, unsigned bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_load3_hint(unsigned dst, const CUtensorMap* map, int c0, int c1,
                                               int c2, unsigned bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ float4 lds4(unsigned addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(addr));
    return v;
}
__device__ __forceinline__ float comp(const float4& v, int e) {
    return e == 0 ? v.x : (e == 1 ? v.y : (e == 2 ? v.z : v.w));
}
__device__ __forceinline__ void set_comp(float4& v, int e, float x) {
    if (e == 0) v.x = x;
    else if (e == 1) v.y = x;
    else if (e == 2) v.z = x;
    else v.w = x;
}

template <int H, int R1, int T1, int YW = 0>
struct Cfg {
    static constexpr int A = (H + 3) / 4 * 4;         // dim-2 halo rounded to float4
    static constexpr int W2 = kT2 + 2 * A;             // smem row length (floats)
    static constexpr int ROWS = T1 + 2 * H;            // smem rows per plane
    static constexpr int UPLANE = (ROWS * W2 * 4 + 127) / 128 * 128;
    static constexpr int ATILE = T1 * kT2 * 4;         // one aux tile (bytes)
    static constexpr int NCW = (T1 / R1) * 16 / 32;    // consumer warps
    static constexpr int NTHREADS = 32 * (NCW + 1 + YW);  // + YW y-pencil warps (k_tma.cu)
    static constexpr int NQ = 2 * H + 1;               // queue depth
};

// ---- packed FP32x2 arithmetic (FADD2 / FFMA2 / FMUL2 on sm_100a) --------------------
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    return __ffma2_rn(b, make_float2(-1.f, -1.f), a);  // a - b, one rounding
}
__device__ __forceinline__ float2 splat(float v) { return make_float2(v, v); }
__device__ __forceinline__ float2 lo2(const float4& v) { return make_float2(v.x, v.y); }
__device__ __forceinline__ float2 hi2(const float4& v) { return make_float2(v.z, v.w); }
__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// n / d with one Newton step on MUFU.RCP: error <= 1 ulp of the quotient (the quotient is the
// per-step increment, ~0.1 |u|, so this is ~0.1 ulp of u; see DESIGN.md numerics).
__device__ __forceinline__ float2 div2(float2 n, float2 d) {
    const float2 r = make_float2(rcp_approx(d.x), rcp_approx(d.y));
    const float2 q = mul2(n, r);
    const float2 e = fma2(make_float2(-d.x, -d.y), q, n);
    return fma2(e, r, q);
}

// The time update with the per-point coefficient fields of K1 (tma_update_coefs):
//   u+ = u + A (u - u-) + B Lk,   A = (m - g)/(m + g),  B = 1/(m + g),  g = damp dt/2,
// which is u + [(m - g)(u - u-) + Lk]/(m + g) without a division; A = 1 where no damping.
// (measured alternatives: the increment formed first, or an E/D division instead of
// the B field, gave the same accuracy once B's rounding is dithered, and the division costs 2-3 %)
__device__ __forceinline__ float2 update2(float2 u, float2 um, float2 Lk, float2 a, float2 b) {
    return fma2(b, Lk, fma2(a, sub2(u, um), u));
}

// Advance a ring position (stage, phase) by one.
template <int S>
__device__ __forceinline__ void ring_next(unsigned& st, unsigned& ph) {
    if (++st == S) {
        st = 0;
        ph ^= 1u;
    }
}

// Per-item state shared by the consumer's per-plane steps.
struct Item {
    int xa, xb, dir, q0, nq, yt, zc;
    bool zfull, rows_ok;
    unsigned zmask;    // bit e set: element zc+e lies in the updated z range
    unsigned rowmask;  // bit i set: tile row yt+i lies in the updated y range
    int s0;            // [s0, s0+sn): planes of the item whose epilogue is not the plain store
    unsigned sn;       // (slab-boundary planes, the source plane; one covering range)
    long long gcol;
    long long xrun;   // offset of the next output plane's element (running, K1 register queue)
};

// Per-lane validity mask of the float4 at zc against the updated range [z0, z1).
__device__ __forceinline__ unsigned zmask_of(int zc, int z0, int z1) {
    unsigned m = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) m |= (zc + e >= z0 && zc + e < z1) ? (1u << e) : 0u;
    return m;
}

// Store one output float4 row and fold it into the max|u| bits.  Full lanes take one
// STG.128; boundary lanes predicated scalar stores; no per-element branches (the partial
// case only exists on the first/last z tile).
// kHoist: the L2 policy comes from a non-volatile asm with no inputs, so it is computed once and
// hoisted out of the plane loop (2 registers) instead of rebuilt by ~6 uniform ops at every
// store; the plain-store plane path of the variants with H % 4 == 0 takes it.
template <bool kHoist = false>
__device__ __forceinline__ void store_row(float* dst, const float4& o, unsigned zmask, unsigned& mine) {
    if (zmask == 0xFu) {
        // u[t+1] is next step's u[t] (halo re-reads by the neighbouring tiles): keep it in L2
        // (evict_last; measured +1.1 % at SO 8, neutral on the predicated-store variants)
        if constexpr (kHoist) {
            uint64_t pol;
            asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
            asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;"
                         ::"l"(dst), "f"(o.x), "f"(o.y), "f"(o.z), "f"(o.w), "l"(pol) : "memory");
        } else {
            asm volatile(
                "{\n\t.reg .b64 pol;\n\t"
                "createpolicy.fractional.L2::evict_last.b64 pol, 1.0;\n\t"
                "st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, pol;\n\t}"
                ::"l"(dst), "f"(o.x), "f"(o.y), "f"(o.z), "f"(o.w) : "memory");
        }
        mine = fold_abs4(mine, o.x, o.y, o.z, o.w);
    } else if (zmask) {
        if (zmask & 1u) dst[0] = o.x;
        if (zmask & 2u) dst[1] = o.y;
        if (zmask & 4u) dst[2] = o.z;
        if (zmask & 8u) dst[3] = o.w;
        mine = fold_abs4(mine, (zmask & 1u) ? o.x : 0.f, (zmask & 2u) ? o.y : 0.f, (zmask & 4u) ? o.z : 0.f,
                         (zmask & 8u) ? o.w : 0.f);
    }
}

// Same, for grids whose interior z bounds cut a float4 lane (z0 or z1 not a multiple of 4):
// full lanes STG.128, half lanes (masks 0b0011 / 0b1100: even bounds) one STG.64, all as
// predicated stores with a select-masked max, so the warp holding the edge lane does not take
// the divergent per-element path every plane (that cost the edge-tile CTAs ~5 % at SO 4 and 12).
// Other masks (odd bounds) still use per-element stores.
__device__ __forceinline__ void store_row_pred(float* dst, const float4& o, unsigned zmask, unsigned& mine) {
    asm volatile(
        "{\n\t.reg .pred pf, pl, ph;\n\t"
        "setp.eq.u32 pf, %0, 15;\n\t"
        "setp.eq.u32 pl, %0, 3;\n\t"
        "setp.eq.u32 ph, %0, 12;\n\t"
        "@pf st.global.v4.f32 [%1], {%2, %3, %4, %5};\n\t"
        "@pl st.global.v2.f32 [%1], {%2, %3};\n\t"
        "@ph st.global.v2.f32 [%1+8], {%4, %5};\n\t"
        "}" ::"r"(zmask), "l"(dst), "f"(o.x), "f"(o.y), "f"(o.z), "f"(o.w)
        : "memory");
    if (zmask != 0xFu && zmask != 0x3u && zmask != 0xCu && zmask != 0u) {
        if (zmask & 1u) dst[0] = o.x;
        if (zmask & 2u) dst[1] = o.y;
        if (zmask & 4u) dst[2] = o.z;
        if (zmask & 8u) dst[3] = o.w;
    }
    mine = fold_abs4(mine, (zmask & 1u) ? o.x : 0.f, (zmask & 2u) ? o.y : 0.f, (zmask & 4u) ? o.z : 0.f,
                     (zmask & 8u) ? o.w : 0.f);
}

// One arrival step of a consumer thread: take plane q's centre values into queue slot U,
// and (after the 2H warm-up planes) produce output plane p = q - dir*H, whose queue slot is
// (U - H) mod NQ.  All queue indices are compile-time.
// Spin (acquire, system scope) until *flag >= need; bounded at ~20 s, then record an error
// instead of hanging.  Followed by a proxy fence: the caller's next reads are TMA (async proxy).
__device__ __forceinline__ void wait_counter(const unsigned long long* flag, unsigned long long need,
                                             unsigned* err) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
    if (v < need) {
        const unsigned long long t0 = gtimer();
        while (true) {
            __nanosleep(200);
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
            if (v >= need) break;
            if (gtimer() - t0 > 20000000000ull) {
                atomicExch(err, 1u);
                break;
            }
        }
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// End-of-CTA signal for the fused halo exchange (after the CTA barrier in block_max_commit).
__device__ __forceinline__ void signal_neighbours(const Ctl& c) {
    if (threadIdx.x == 0 && (c.sig_lo || c.sig_hi)) {
        __threadfence_system();
        if (c.sig_lo) atomicAdd(c.sig_lo, 1ull);
        if (c.sig_hi) atomicAdd(c.sig_hi, 1ull);
    }
}

// Launch a stencil kernel with programmatic stream serialization (PDL): the next step's
// CTAs start their prologue while this step drains; they block in griddepcontrol.wait.
inline cudaError_t launch_pdl_args(const void* fn, int grid, int threads, size_t smem, cudaStream_t s,
                                   void** args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelExC(&cfg, fn, args);
}
// k_tma kernels: (Maps, Geo, Coef, Ctl, Peer, Sched)
inline cudaError_t launch_pdl(const void* fn, int grid, int threads, size_t smem, cudaStream_t s,
                              const Maps& maps, const Geo& g, const Coef& K, const Ctl& c, const Peer& p,
                              const Sched& sc) {
    void* args[] = {const_cast<Maps*>(&maps), const_cast<Geo*>(&g), const_cast<Coef*>(&K),
                    const_cast<Ctl*>(&c), const_cast<Peer*>(&p), const_cast<Sched*>(&sc)};
    return launch_pdl_args(fn, grid, threads, smem, s, args);
}

}  // namespace tma
}  // namespace swb
