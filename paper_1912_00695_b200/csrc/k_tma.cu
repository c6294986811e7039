// K1: TMA-staged 2.5D factorised stencil for sm_100a.
//
// One persistent CTA per SM strides over work items (column tile x dim-0 chunk): a column
// tile is T1 rows (dim 1) x 64 cols (dim 2) of output points; the CTA streams it along dim 0
// (the reference's slowest axis "x"; the north star's "z-slab" axis) over the chunk's planes.
// Warp 0 is the TMA producer (lane 0: u ring, lane 1: aux ring); warps 1..NCW are consumers.
//
//   u ring  : halo-padded planes of u[t] ((T1+2H) x (64+2A) floats) loaded by
//             cp.async.bulk.tensor.3d; a plane stays resident from its arrival (when the
//             consumers take its centre values into the register queue) until the output
//             plane with the same index has used it for the in-plane (dim 1 / dim 2) stencil,
//             H planes later.  Depth S_U = H + 1 + prefetch.
//   aux ring: u[t-1], B, A tiles (T1 x 64) of the output plane, one TMA each (A only where
//             the tile is damped); B and A are the coefficient fields that replace m and damp.
//   register queue: each consumer thread keeps u[t] of its R1 x 4 points for the 2H+1
//             planes around the output plane (the dim-0 stencil never touches smem).
//
// Arithmetic per point (factorised form, src/pipeline.cpp:467-512 with the sign fix):
//   S  = sum_k>=2 c_k (u_-k + u_+k) over the three axes + c_1 sum((u_-1 - u) + (u_+1 - u))
//   Lr = S + 3 (c_0 + 2 c_1) u
//   u+ = u + A (u - u-) + B Lr (dt/h)^2,   A = (m - g)/(m + g),  B = 1/(m + g),  g = damp dt/2
// (update2 in k_tma_common.cuh; the one-thread-per-point kernels divide instead, combine_f32
// in k_common.cuh), then the fused epilogue: source injection with the reference's two
// roundings, 128-bit stores, peer stores of slab-boundary planes, and the per-step max|u| /
// non-finite flag.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <cstdint>
#include <cstring>

#include "k_tma_common.cuh"

namespace swb {
namespace {
using namespace tma;

#ifndef SWB_UNROLL_MAXH
#define SWB_UNROLL_MAXH 4  // rotate the register queue by renaming up to this halo (measured: +1 % at SO 8; I-cache misses beyond)
#endif
#ifndef SWB_LAP
#define SWB_LAP 0  // development: Laplacian summation variants (probe_combine.py)
#endif
#ifndef SWB_TB_LEAD
#define SWB_TB_LEAD 4
#endif
constexpr int kTbLead = SWB_TB_LEAD;  // K3: planes stage 1 must be ahead of stage 2's request

// K3 stage-1 progress publication: a plane counts as done once every consumer warp has
// stored its rows of it (warps drift apart by up to SU-H planes, so a per-plane smem tally
// over a ring of 16 slots finds the last warp, which publishes with atomicMax).
struct Pub {
    unsigned long long* cnt;  // this item's global counter (null: not publishing)
    unsigned long long base;  // epoch tag
    unsigned* done;           // smem [16] per-plane warp tallies, [16] = (seq << 16) | planes complete
    unsigned seq;             // this CTA's item sequence number (tags `complete`)
    int H;                    // halo (output plane n of an item arrives at step n + 2H)
    int ncw;                  // consumer warps of the CTA
};

// The dim-2 window of one output float4: w[i] = row[i - A] for the indices the stencil reads,
// [A - H, A + 4 + H).  The smem row is padded to A >= H floats per side (A a multiple of 4 keeps
// the centre float4 aligned); only the needed part is loaded, 128-bit where aligned and 64/32-bit
// at the ends (SO 12: 3 LDS.128 + 2 LDS.64 instead of 5 LDS.128).
template <int A, int I, int HI, int N>
__device__ __forceinline__ void window_step(const float* rowc, float (&w)[N]) {
    if constexpr (I < HI) {
        if constexpr (I % 4 == 0 && I + 4 <= HI) {
            const float4 v = *reinterpret_cast<const float4*>(rowc - A + I);
            w[I] = v.x;
            w[I + 1] = v.y;
            w[I + 2] = v.z;
            w[I + 3] = v.w;
            window_step<A, I + 4, HI>(rowc, w);
        } else if constexpr (I % 2 == 0 && I + 2 <= HI) {
            const float2 v = *reinterpret_cast<const float2*>(rowc - A + I);
            w[I] = v.x;
            w[I + 1] = v.y;
            window_step<A, I + 2, HI>(rowc, w);
        } else {
            w[I] = rowc[I - A];
            window_step<A, I + 1, HI>(rowc, w);
        }
    }
}
template <int H, int A>
__device__ __forceinline__ void load_window(const float* rowc, float (&w)[4 + 2 * A]) {
    window_step<A, A - H, A + 4 + H>(rowc, w);
}

// Fused epilogue of one output plane: 128-bit stores (plus peer stores into the neighbours'
// ghost planes, and the source injection with the reference's two roundings), the max|u|
// fold, and the K3 stage-1 progress publication.
template <int H, int R1>
__device__ __forceinline__ void epilogue_store(const float4* out, int p, long long xoff,
                                               const Item& it, unsigned& mine, float* un, float* lo_peer,
                                               float* hi_peer, const Geo& g, const Coef& K, const Ctl& c,
                                               const Peer& pr, const Pub& pub, int j) {
    if (static_cast<unsigned>(p - it.s0) >= it.sn) {
        // common path: plain stores (rows past the interior are skipped warp-uniformly)
#pragma unroll
        for (int i = 0; i < R1; ++i)
            if ((it.rowmask >> i) & 1u) {
                // H not a multiple of 4: the interior's z bounds cut a lane on (even-extent) grids,
                // so take the branch-free predicated stores (compile-time choice per variant)
                if constexpr (H % 4 != 0)
                    store_row_pred(un + xoff + static_cast<long long>(i) * g.P2, out[i], it.zmask, mine);
                else
                    store_row(un + xoff + static_cast<long long>(i) * g.P2, out[i], it.zmask, mine);
            }
    } else {
        // slab-boundary planes (also stored into the neighbour's ghost plane, 128-bit, same
        // lane masks) and the source plane (the one injected element is patched first)
        const bool lo_m = p >= pr.lo_first && p < pr.lo_last;
        const bool hi_m = p >= pr.hi_first && p < pr.hi_last;
        const bool src_plane = c.has_src && p == c.src_x;
#pragma unroll
        for (int i = 0; i < R1; ++i) {
            const int y = it.yt + i;
            float4 o = out[i];
            if (y >= g.y1) continue;
            if (src_plane && y == c.src_y && static_cast<unsigned>(c.src_z - it.zc) < 4u) {
                const int e = c.src_z - it.zc;
                set_comp(o, e, inject_source(comp(o, e), c.wavelet[c.step], c.src_m, static_cast<double>(K.dt)));
            }
            const long long idx = xoff + static_cast<long long>(i) * g.P2;
            store_row(un + idx, o, it.zmask, mine);
            unsigned dummy = 0u;
            if (lo_m) store_row(lo_peer + idx + static_cast<long long>(pr.lo_shift) * g.plane, o, it.zmask, dummy);
            if (hi_m) store_row(hi_peer + idx + static_cast<long long>(pr.hi_shift) * g.plane, o, it.zmask, dummy);
        }
    }
    // Temporal blocking, stage 1: publish "this warp has stored one more u[t+1] plane"
    // (the stage-2 CTAs wait on these counters before reading the plane through TMA).
    if (pub.cnt) {
        // A plane is done when its last warp tallies it; that warp records it in `complete`
        // (CTA scope).  The gpu-scope release (fence + red.max) is paid by the FIRST warp to
        // finish a later plane -- a warp that is ahead of the others, so the fence does not
        // stall the slowest warp (which gates the whole CTA through the rings).  The item's
        // final plane is published by its last warp.
        __syncwarp();  // orders the warp's stores before lane 0's tally (bar.warp.sync)
        if ((threadIdx.x & 31) == 0) {
            const int n = j - 2 * pub.H;  // output plane index within the item
            unsigned old;
            asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                         : "=r"(old) : "r"(smem_addr(pub.done + (n & 15))) : "memory");
            const unsigned tag = pub.seq << 16;
            if (old == static_cast<unsigned>(pub.ncw - 1)) {  // last warp for plane n
                pub.done[n & 15] = 0u;
                asm volatile("red.release.cta.shared::cta.max.u32 [%0], %1;"
                             :: "r"(smem_addr(pub.done + 16)), "r"(tag | static_cast<unsigned>(n + 1)) : "memory");
                if (n + 1 == it.xb - it.xa) {  // the item's final plane
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                    asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;"
                                 :: "l"(pub.cnt), "l"(pub.base + static_cast<unsigned long long>(n + 1)) : "memory");
                }
            } else if (old == 0u && n > 0) {  // first warp for plane n: publish what is complete
                unsigned done_;
                asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];"
                             : "=r"(done_) : "r"(smem_addr(pub.done + 16)) : "memory");
                if ((done_ & ~0xffffu) == tag && (done_ & 0xffffu) != 0u) {
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                    asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;"
                                 :: "l"(pub.cnt), "l"(pub.base + static_cast<unsigned long long>(done_ & 0xffffu))
                                 : "memory");
                }
            }
        }
    }
}

template <int H, int R1, int T1, int SU, int SA, int QN, int U>
__device__ __forceinline__ void consumer_step(float4 (&Q)[R1][QN], int j, Item& it,
                                              const float* ucol, const float* acol,
                                              const unsigned* aflag, unsigned full_u,
                                              unsigned empty_u, unsigned full_a, unsigned empty_a,
                                              unsigned& su, unsigned& pu, unsigned& sp,
                                              unsigned& sa, unsigned& pa_, unsigned& mine,
                                              float* un, float* lo_peer, float* hi_peer,
                                              const Geo& g, const Coef& K, const Ctl& c,
                                              const Peer& pr, const Pub& pub) {
    using C = Cfg<H, R1, T1>;
    constexpr int NQ = QN;  // queue slots; plane j-m sits in slot (U - m) mod QN
    const int q = it.q0 + it.dir * j;
    mbar_wait(full_u + 8 * su, pu);
    const float* plane_q = ucol + su * (C::UPLANE / 4);
#pragma unroll
    for (int i = 0; i < R1; ++i) Q[i][U] = *reinterpret_cast<const float4*>(plane_q + i * C::W2);
    if (!(q >= it.xa && q < it.xb))  // only needed for its centre values
        mbar_arrive(empty_u + 8 * su);
    ring_next<SU>(su, pu);
    if (j < 2 * H) return;
    // ---- output plane p (arrived H planes ago, smem stage sp) ----
    const int p = q - it.dir * H;
    constexpr int UC = (U + NQ - H) % NQ;  // queue slot of plane p
    const float* pp = ucol + sp * (C::UPLANE / 4);
    float2 acc[R1][2];
#pragma unroll
    for (int i = 0; i < R1; ++i) {
        const float* rowc = pp + i * C::W2;
        float w[4 + 2 * C::A];
        load_window<H, C::A>(rowc, w);
        float2 al = splat(0.f), ah = splat(0.f);
#if SWB_LAP == 2
        const float2 cl = lo2(Q[i][UC]), chh = hi2(Q[i][UC]);
#endif
#pragma unroll
        for (int k = H; k >= 2; --k) {
            const float2 ck = splat(K.c[k]);
            const float4 ym = *reinterpret_cast<const float4*>(rowc - k * C::W2);
            const float4 yp = *reinterpret_cast<const float4*>(rowc + k * C::W2);
            const float4& xm = Q[i][(UC + NQ - k) % NQ];
            const float4& xp = Q[i][(UC + k) % NQ];
#if SWB_LAP == 2
            // full difference form: every neighbour minus the centre first
            const float2 zl = make_float2((w[C::A - k] - cl.x) + (w[C::A + k] - cl.x),
                                          (w[C::A + 1 - k] - cl.y) + (w[C::A + 1 + k] - cl.y));
            const float2 zh = make_float2((w[C::A + 2 - k] - chh.x) + (w[C::A + 2 + k] - chh.x),
                                          (w[C::A + 3 - k] - chh.y) + (w[C::A + 3 + k] - chh.y));
            const float2 sl = add2(add2(sub2(lo2(xm), cl), sub2(lo2(xp), cl)),
                                   add2(add2(sub2(lo2(ym), cl), sub2(lo2(yp), cl)), zl));
            const float2 sh = add2(add2(sub2(hi2(xm), chh), sub2(hi2(xp), chh)),
                                   add2(add2(sub2(hi2(ym), chh), sub2(hi2(yp), chh)), zh));
#else
            float2 zl, zh;
            if ((k & 1) == 0) {  // register-pair aligned: packed adds
                zl = add2(make_float2(w[C::A - k], w[C::A + 1 - k]), make_float2(w[C::A + k], w[C::A + 1 + k]));
                zh = add2(make_float2(w[C::A + 2 - k], w[C::A + 3 - k]),
                          make_float2(w[C::A + 2 + k], w[C::A + 3 + k]));
            } else {
                zl = make_float2(w[C::A - k] + w[C::A + k], w[C::A + 1 - k] + w[C::A + 1 + k]);
                zh = make_float2(w[C::A + 2 - k] + w[C::A + 2 + k], w[C::A + 3 - k] + w[C::A + 3 + k]);
            }
#if SWB_LAP == 1
            // per-axis grouping (pairs of one axis first, as the one-thread-per-point kernels)
            const float2 sl = add2(add2(add2(lo2(xm), lo2(xp)), add2(lo2(ym), lo2(yp))), zl);
            const float2 sh = add2(add2(add2(hi2(xm), hi2(xp)), add2(hi2(ym), hi2(yp))), zh);
#else
            const float2 sl = add2(add2(lo2(xm), lo2(xp)), add2(add2(lo2(ym), lo2(yp)), zl));
            const float2 sh = add2(add2(hi2(xm), hi2(xp)), add2(add2(hi2(ym), hi2(yp)), zh));
#endif
#endif
            al = fma2(ck, sl, al);
            ah = fma2(ck, sh, ah);
        }
        // k = 1 ring in difference form, all three axes
        const float4 u0 = Q[i][UC];
        const float4 ym = *reinterpret_cast<const float4*>(rowc - C::W2);
        const float4 yp = *reinterpret_cast<const float4*>(rowc + C::W2);
        const float4& xm = Q[i][(UC + NQ - 1) % NQ];
        const float4& xp = Q[i][(UC + 1) % NQ];
        const float2 ul = lo2(u0), uh = hi2(u0);
        float dz[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float ue = comp(u0, e);
            dz[e] = (w[C::A + e - 1] - ue) + (w[C::A + e + 1] - ue);
        }
        float2 dl = add2(sub2(lo2(xm), ul), sub2(lo2(xp), ul));
        dl = add2(dl, add2(sub2(lo2(ym), ul), sub2(lo2(yp), ul)));
        dl = add2(dl, make_float2(dz[0], dz[1]));
        float2 dh = add2(sub2(hi2(xm), uh), sub2(hi2(xp), uh));
        dh = add2(dh, add2(sub2(hi2(ym), uh), sub2(hi2(yp), uh)));
        dh = add2(dh, make_float2(dz[2], dz[3]));
        const float2 c1 = splat(K.c[1]);
        acc[i][0] = fma2(c1, dl, al);
        acc[i][1] = fma2(c1, dh, ah);
    }
    // ---- aux tiles: u[t-1], m, damp ----
    mbar_wait(full_a + 8 * sa, pa_);
    const float* aux = acol + sa * (3 * C::ATILE / 4);
    const bool has_damp = aflag[sa] != 0u;
    float4 upv[R1], bv[R1], av[R1];
#pragma unroll
    for (int i = 0; i < R1; ++i) {
        upv[i] = *reinterpret_cast<const float4*>(aux + i * kT2);
        bv[i] = *reinterpret_cast<const float4*>(aux + C::ATILE / 4 + i * kT2);
#if SWB_COMBINE == 2
        av[i] = has_damp ? *reinterpret_cast<const float4*>(aux + C::ATILE / 2 + i * kT2) : bv[i];
#else
        av[i] = has_damp ? *reinterpret_cast<const float4*>(aux + C::ATILE / 2 + i * kT2)
                         : make_float4(1.f, 1.f, 1.f, 1.f);
#endif
    }
    mbar_arrive(empty_a + 8 * sa);
    mbar_arrive(empty_u + 8 * sp);  // plane p is no longer needed
    ring_next<SA>(sa, pa_);
    if (++sp == SU) sp = 0;
    // ---- combine: u+ = u + A (u - u-) + B Lr (dt/h)^2 (coefficient fields, tma_update_coefs) ----
#if SWB_LAP == 2
    const float2 R3 = splat(K.R3f), khi = splat(K.kap_hi), klo = splat(K.kap_lo);
#else
    const float2 R3 = splat(K.R3), khi = splat(K.kap_hi), klo = splat(K.kap_lo);
#endif
    float4 out[R1];
#pragma unroll
    for (int i = 0; i < R1; ++i) {
        const float4 u0 = Q[i][UC];
        float2 res[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float2 ucv = h ? hi2(u0) : lo2(u0);
            const float2 um = h ? hi2(upv[i]) : lo2(upv[i]);
            const float2 Lr = fma2(R3, ucv, acc[i][h]);
            const float2 Lk = fma2(Lr, khi, mul2(Lr, klo));
            res[h] = update2(ucv, um, Lk, h ? hi2(av[i]) : lo2(av[i]), h ? hi2(bv[i]) : lo2(bv[i]));
        }
        out[i] = make_float4(res[0].x, res[0].y, res[1].x, res[1].y);
    }
    // output offset p * plane + gcol: kept running (one 64-bit add per plane instead of the
    // multiply-add), except at SO 12, whose 15-warp variant is at its register cap and spills
    // with the two extra registers (measured: SO 16 +2.7 %, SO 12 -1.3 % with it)
    long long xoff;
    if constexpr (H != 6) {
        xoff = it.xrun;
        it.xrun += it.dir > 0 ? g.plane : -g.plane;
    } else {
        xoff = static_cast<long long>(p) * g.plane + it.gcol;
    }
    epilogue_store<H, R1>(out, p, xoff, it, mine, un, lo_peer, hi_peer, g, K, c, pr, pub, j);
}

// ---- K1 with the dim-0 queue in tensor memory (UNR == 0 variants) -----------------------
// Each consumer thread owns one TMEM lane (its warp's lane quadrant) and a 128-column block
// (4 warps share a quadrant): a ring of 32 float4 slots holding u[t] of its 4 points for the
// last 32 planes.  The x-stencil reads its 2H neighbours with tcgen05.ld instead of keeping
// 2H+UNR float4 in registers, so the register queue (and its shift moves) disappears and the
// plane loop needs no unrolling.  TMEM is an extra on-chip store with its own datapath: the
// loads do not use the shared-memory pipe that the y/z stencil saturates.
__device__ __forceinline__ void tm_st4(unsigned addr, const float4& v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
}
__device__ __forceinline__ float4 tm_ld4(unsigned addr) {
    float4 v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(addr)
                 : "memory");
    return v;
}
// tcgen05.wait::ld, with the loaded values routed through the asm so that no use of them can
// be scheduled before the wait (the loads' outputs are otherwise "ready" at issue).
template <int N>
__device__ __forceinline__ void tm_wait_ld(float4 (&v)[N]) {
    static_assert(N <= 7, "at most 28 asm operands per wait");
    if constexpr (N == 0) {
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    } else if constexpr (N == 1) {
        asm volatile("tcgen05.wait::ld.sync.aligned;" : "+f"(v[0].x), "+f"(v[0].y), "+f"(v[0].z), "+f"(v[0].w) :: "memory");
    } else {
        asm volatile("tcgen05.wait::ld.sync.aligned;" : "+f"(v[0].x), "+f"(v[0].y), "+f"(v[0].z), "+f"(v[0].w),
                     "+f"(v[1].x), "+f"(v[1].y), "+f"(v[1].z), "+f"(v[1].w) :: "memory");
#pragma unroll
        for (int i = 2; i < N; ++i)
            asm volatile("" : "+f"(v[i].x), "+f"(v[i].y), "+f"(v[i].z), "+f"(v[i].w) :: "memory");
    }
}

template <int H, int R1, int T1, int SU, int SA>
__device__ __forceinline__ void consumer_step_tq(unsigned tq, int j, const Item& it, const float* ucol,
                                                 const float* acol, const unsigned* aflag, unsigned full_u,
                                                 unsigned empty_u, unsigned full_a, unsigned empty_a, unsigned& su,
                                                 unsigned& pu, unsigned& sp, unsigned& sa, unsigned& pa_,
                                                 unsigned& mine, float* un, float* lo_peer, float* hi_peer,
                                                 const Geo& g, const Coef& K, const Ctl& c, const Peer& pr,
                                                 const Pub& pub) {
    static_assert(R1 == 1 && H >= 2 && 2 * H + 1 <= 32, "TMEM queue: one row per thread, ring of 32 planes");
    using C = Cfg<H, R1, T1>;
    const int q = it.q0 + it.dir * j;
    mbar_wait(full_u + 8 * su, pu);
    const float* plane_q = ucol + su * (C::UPLANE / 4);
    const float4 cq = *reinterpret_cast<const float4*>(plane_q);
    tm_st4(tq + 4u * static_cast<unsigned>(j & 31), cq);
    if (!(q >= it.xa && q < it.xb)) mbar_arrive(empty_u + 8 * su);
    ring_next<SU>(su, pu);
    if (j < 2 * H) return;
    const int p = q - it.dir * H;
    const int jc = j - H;  // step index of plane p
    const float* rowc = ucol + sp * (C::UPLANE / 4);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");  // earlier planes' stores landed
    float w[4 + 2 * C::A];
    load_window<H, C::A>(rowc, w);
    float2 al = splat(0.f), ah = splat(0.f);
    // far half of the x-neighbours: k = H .. KB+1 (plane p+H is the one that just arrived)
    constexpr int KB = H / 2;
    {
        float4 xv[2 * (H - KB) - 1];
#pragma unroll
        for (int k = H; k > KB; --k) {
            xv[H - k] = tm_ld4(tq + 4u * static_cast<unsigned>((jc - k) & 31));
            if (k != H) xv[2 * (H - KB) - 1 - (H - k)] = tm_ld4(tq + 4u * static_cast<unsigned>((jc + k) & 31));
        }
        tm_wait_ld(xv);
#pragma unroll
        for (int k = H; k > KB; --k) {
            const float2 ck = splat(K.c[k]);
            const float4 ym = *reinterpret_cast<const float4*>(rowc - k * C::W2);
            const float4 yp = *reinterpret_cast<const float4*>(rowc + k * C::W2);
            const float4 xm = xv[H - k];
            const float4 xp = k == H ? cq : xv[2 * (H - KB) - 1 - (H - k)];
            float2 zl, zh;
            if ((k & 1) == 0) {
                zl = add2(make_float2(w[C::A - k], w[C::A + 1 - k]), make_float2(w[C::A + k], w[C::A + 1 + k]));
                zh = add2(make_float2(w[C::A + 2 - k], w[C::A + 3 - k]),
                          make_float2(w[C::A + 2 + k], w[C::A + 3 + k]));
            } else {
                zl = make_float2(w[C::A - k] + w[C::A + k], w[C::A + 1 - k] + w[C::A + 1 + k]);
                zh = make_float2(w[C::A + 2 - k] + w[C::A + 2 + k], w[C::A + 3 - k] + w[C::A + 3 + k]);
            }
            const float2 sl = add2(add2(lo2(xm), lo2(xp)), add2(add2(lo2(ym), lo2(yp)), zl));
            const float2 sh = add2(add2(hi2(xm), hi2(xp)), add2(add2(hi2(ym), hi2(yp)), zh));
            al = fma2(ck, sl, al);
            ah = fma2(ck, sh, ah);
        }
    }
    float4 u0;
    float4 xm1, xp1;
    {
        // near half: k = KB .. 2, then the k = 1 ring and the centre
        float4 xv[2 * KB + 1];
#pragma unroll
        for (int k = KB; k >= 1; --k) {
            xv[KB - k] = tm_ld4(tq + 4u * static_cast<unsigned>((jc - k) & 31));
            xv[2 * KB - (KB - k)] = tm_ld4(tq + 4u * static_cast<unsigned>((jc + k) & 31));
        }
        xv[KB] = tm_ld4(tq + 4u * static_cast<unsigned>(jc & 31));
        if constexpr (2 * KB + 1 <= 7) {
            tm_wait_ld(xv);
        } else {
            float4 (&a)[7] = *reinterpret_cast<float4 (*)[7]>(&xv[0]);
            tm_wait_ld(a);
#pragma unroll
            for (int i = 7; i < 2 * KB + 1; ++i)
                asm volatile("" : "+f"(xv[i].x), "+f"(xv[i].y), "+f"(xv[i].z), "+f"(xv[i].w) :: "memory");
        }
#pragma unroll
        for (int k = KB; k >= 2; --k) {
            const float2 ck = splat(K.c[k]);
            const float4 ym = *reinterpret_cast<const float4*>(rowc - k * C::W2);
            const float4 yp = *reinterpret_cast<const float4*>(rowc + k * C::W2);
            const float4 xm = xv[KB - k];
            const float4 xp = xv[2 * KB - (KB - k)];
            float2 zl, zh;
            if ((k & 1) == 0) {
                zl = add2(make_float2(w[C::A - k], w[C::A + 1 - k]), make_float2(w[C::A + k], w[C::A + 1 + k]));
                zh = add2(make_float2(w[C::A + 2 - k], w[C::A + 3 - k]),
                          make_float2(w[C::A + 2 + k], w[C::A + 3 + k]));
            } else {
                zl = make_float2(w[C::A - k] + w[C::A + k], w[C::A + 1 - k] + w[C::A + 1 + k]);
                zh = make_float2(w[C::A + 2 - k] + w[C::A + 2 + k], w[C::A + 3 - k] + w[C::A + 3 + k]);
            }
            const float2 sl = add2(add2(lo2(xm), lo2(xp)), add2(add2(lo2(ym), lo2(yp)), zl));
            const float2 sh = add2(add2(hi2(xm), hi2(xp)), add2(add2(hi2(ym), hi2(yp)), zh));
            al = fma2(ck, sl, al);
            ah = fma2(ck, sh, ah);
        }
        u0 = xv[KB];
        xm1 = xv[KB - 1];
        xp1 = xv[KB + 1];
    }
    float2 acc[2];
    {
        // k = 1 ring in difference form, all three axes
        const float4 ym = *reinterpret_cast<const float4*>(rowc - C::W2);
        const float4 yp = *reinterpret_cast<const float4*>(rowc + C::W2);
        const float4& xm = xm1;
        const float4& xp = xp1;
        const float2 ul = lo2(u0), uh = hi2(u0);
        float dz[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float ue = comp(u0, e);
            dz[e] = (w[C::A + e - 1] - ue) + (w[C::A + e + 1] - ue);
        }
        float2 dl = add2(sub2(lo2(xm), ul), sub2(lo2(xp), ul));
        dl = add2(dl, add2(sub2(lo2(ym), ul), sub2(lo2(yp), ul)));
        dl = add2(dl, make_float2(dz[0], dz[1]));
        float2 dh = add2(sub2(hi2(xm), uh), sub2(hi2(xp), uh));
        dh = add2(dh, add2(sub2(hi2(ym), uh), sub2(hi2(yp), uh)));
        dh = add2(dh, make_float2(dz[2], dz[3]));
        const float2 c1 = splat(K.c[1]);
        acc[0] = fma2(c1, dl, al);
        acc[1] = fma2(c1, dh, ah);
    }
    // ---- aux tiles: u[t-1], m, damp ----
    mbar_wait(full_a + 8 * sa, pa_);
    const float* aux = acol + sa * (3 * C::ATILE / 4);
    const bool has_damp = aflag[sa] != 0u;
    const float4 upv = *reinterpret_cast<const float4*>(aux);
    const float4 bv = *reinterpret_cast<const float4*>(aux + C::ATILE / 4);
    const float4 av = has_damp ? *reinterpret_cast<const float4*>(aux + C::ATILE / 2) : make_float4(1.f, 1.f, 1.f, 1.f);
    mbar_arrive(empty_a + 8 * sa);
    mbar_arrive(empty_u + 8 * sp);  // plane p is no longer needed
    ring_next<SA>(sa, pa_);
    if (++sp == SU) sp = 0;
    // ---- combine (as consumer_step) ----
    const float2 R3 = splat(K.R3), khi = splat(K.kap_hi), klo = splat(K.kap_lo);
    float4 out;
    {
        float2 res[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float2 ucv = h ? hi2(u0) : lo2(u0);
            const float2 um = h ? hi2(upv) : lo2(upv);
            const float2 Lr = fma2(R3, ucv, acc[h]);
            const float2 Lk = fma2(Lr, khi, mul2(Lr, klo));
            res[h] = update2(ucv, um, Lk, h ? hi2(av) : lo2(av), h ? hi2(bv) : lo2(bv));
        }
        out = make_float4(res[0].x, res[0].y, res[1].x, res[1].y);
    }
    epilogue_store<H, R1>(&out, p, static_cast<long long>(p) * g.plane + it.gcol, it, mine, un, lo_peer,
                          hi_peer, g, K, c, pr, pub, j);
}

template <int H, int R1, int T1, int SU, int SA, int U>
struct Unrolled {
    __device__ __forceinline__ static void run(float4 (&Q)[R1][2 * H + 1], int jb, Item& it,
                                               const float* ucol, const float* acol,
                                               const unsigned* aflag, unsigned full_u, unsigned empty_u,
                                               unsigned full_a, unsigned empty_a, unsigned& su,
                                               unsigned& pu, unsigned& sp, unsigned& sa, unsigned& pa_,
                                               unsigned& mine, float* un, float* lo_peer,
                                               float* hi_peer, const Geo& g, const Coef& K,
                                               const Ctl& c, const Peer& pr, const Pub& pub) {
        if (jb + U < it.nq) {
            consumer_step<H, R1, T1, SU, SA, 2 * H + 1, U>(Q, jb + U, it, ucol, acol, aflag, full_u, empty_u,
                                                full_a, empty_a, su, pu, sp, sa, pa_, mine, un,
                                                lo_peer, hi_peer, g, K, c, pr, pub);
            Unrolled<H, R1, T1, SU, SA, U + 1>::run(Q, jb, it, ucol, acol, aflag, full_u, empty_u,
                                                    full_a, empty_a, su, pu, sp, sa, pa_, mine, un,
                                                    lo_peer, hi_peer, g, K, c, pr, pub);
        }
    }
};
template <int H, int R1, int T1, int SU, int SA>
struct Unrolled<H, R1, T1, SU, SA, 2 * H + 1> {
    __device__ __forceinline__ static void run(float4 (&)[R1][2 * H + 1], int, Item&,
                                               const float*, const float*, const unsigned*, unsigned,
                                               unsigned, unsigned, unsigned, unsigned&, unsigned&,
                                               unsigned&, unsigned&, unsigned&, unsigned&, float*,
                                               float*, float*, const Geo&, const Coef&, const Ctl&,
                                               const Peer&, const Pub&) {}
};

template <int H, int R1, int T1, int SU, int SA, int UNR, int U>
struct ShiftBlock {
    __device__ __forceinline__ static void run(float4 (&Q)[R1][2 * H + UNR], int jb, Item& it,
                                               const float* ucol, const float* acol,
                                               const unsigned* aflag, unsigned full_u, unsigned empty_u,
                                               unsigned full_a, unsigned empty_a, unsigned& su,
                                               unsigned& pu, unsigned& sp, unsigned& sa, unsigned& pa_,
                                               unsigned& mine, float* un, float* lo_peer,
                                               float* hi_peer, const Geo& g, const Coef& K,
                                               const Ctl& c, const Peer& pr, const Pub& pub) {
        if (jb + U < it.nq) {
            consumer_step<H, R1, T1, SU, SA, 2 * H + UNR, 2 * H + U>(
                Q, jb + U, it, ucol, acol, aflag, full_u, empty_u, full_a, empty_a, su, pu, sp, sa, pa_,
                mine, un, lo_peer, hi_peer, g, K, c, pr, pub);
            ShiftBlock<H, R1, T1, SU, SA, UNR, U + 1>::run(Q, jb, it, ucol, acol, aflag, full_u, empty_u,
                                                           full_a, empty_a, su, pu, sp, sa, pa_, mine, un,
                                                           lo_peer, hi_peer, g, K, c, pr, pub);
        }
    }
};
template <int H, int R1, int T1, int SU, int SA, int UNR>
struct ShiftBlock<H, R1, T1, SU, SA, UNR, UNR> {
    __device__ __forceinline__ static void run(float4 (&)[R1][2 * H + UNR], int, Item&, const float*,
                                               const float*, const unsigned*, unsigned, unsigned, unsigned,
                                               unsigned, unsigned&, unsigned&, unsigned&, unsigned&,
                                               unsigned&, unsigned&, float*, float*, float*, const Geo&,
                                               const Coef&, const Ctl&, const Peer&, const Pub&) {}
};

// The kernel body.  role 0: one time step (K1).  Temporal blocking of two steps (K3) runs
// two roles in one launch: role 1 CTAs compute u[t+1] (level (s+1)%3) for their item plus H
// overlap planes on each dim-0 side, publishing per-plane progress; role 2 CTAs compute
// u[t+2] from it (c.step already advanced by one), their TMA producer waiting on the progress
// counters of the 3x3 neighbouring stage-1 columns before each u[t+1] plane, and before
// overwriting u[t-1] planes that a neighbouring chunk's stage 1 still reads.
template <int H, int R1, int T1, int SU, int SA, int UNR, int TB>
__device__ __forceinline__ void tma_body(const Maps& maps, const Geo& g, const Coef& K, const Ctl& c,
                                         const Peer& pr, const Sched& sc, const TbCtl& tb, int role) {
    using C = Cfg<H, R1, T1>;
    constexpr int NQ = C::NQ;
    // Small halos: unroll the plane loop by the queue depth so the register queue rotates by
    // renaming; large halos: shift the queue (keeps the loop body small for the I-cache).
    constexpr bool kTQ = UNR == 0;  // dim-0 queue in tensor memory
    constexpr bool kUnroll = !kTQ && H <= SWB_UNROLL_MAXH;
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char* uring = smem;
    unsigned char* aring = smem + SU * C::UPLANE;
    uint64_t* bars = reinterpret_cast<uint64_t*>(aring + SA * 3 * C::ATILE);
    unsigned* aflag = reinterpret_cast<unsigned*>(bars + 2 * (SU + SA));  // damp-present per aux stage
    unsigned* tally = aflag + SA;  // K3: per-plane warp tallies [16] + complete-plane word
    const unsigned full_u = smem_addr(bars), empty_u = full_u + 8 * SU;
    const unsigned full_a = empty_u + 8 * SU, empty_a = full_a + 8 * SA;
    const unsigned uring_s = smem_addr(uring), aring_s = smem_addr(aring);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < SU; ++i) {
            mbar_init(full_u + 8 * i, 1);
            mbar_init(empty_u + 8 * i, 32 * C::NCW);  // every consumer thread arrives
        }
        for (int i = 0; i < SA; ++i) {
            mbar_init(full_a + 8 * i, 1);
            mbar_init(empty_a + 8 * i, 32 * C::NCW);
        }
        for (int i = 0; i < 17; ++i) tally[i] = 0u;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __shared__ unsigned tmem_base;
    if constexpr (kTQ) {
        // all 512 TMEM columns: 4 warps per lane quadrant x 128 columns (32 float4 slots) each
        if ((threadIdx.x >> 5) == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                smem_addr(&tmem_base)) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    }
    __syncthreads();
    if constexpr (kTQ) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // Programmatic dependent launch: everything above overlapped the previous step's tail;
    // u[t], u[t-1] written by that step are only touched after this point.
    asm volatile("griddepcontrol.wait;" ::: "memory");

    const int lt = c.step % 3, ln = (c.step + 1) % 3, lp = (c.step + 2) % 3;
    const int nitems = sc.ncol * sc.nchunk;
    // K1: persistent CTAs stride over the items; K3: one item per CTA and role.
    const int first = TB ? static_cast<int>(blockIdx.x) - (role == 2 ? tb.ctas : 0) : static_cast<int>(blockIdx.x);
    const int G = TB ? tb.ctas : static_cast<int>(gridDim.x);
    const unsigned long long epoch = TB ? (tb.epoch << 32) : 0ull;
    if (TB) {
        // reset this item's stage-1 progress for this launch (after griddepcontrol.wait: the
        // previous launch's stage-2 CTAs are done polling it), ordered before every
        // consumer's increments by the CTA barrier
        if (role == 1 && threadIdx.x == 0) {
            for (int item = first; item < nitems; item += G) atomicExch(tb.cnt + item, epoch);
            __threadfence();
        }
        __syncthreads();
    }
    unsigned mine = 0u;
    if (c.trace && threadIdx.x == 0) c.trace[4 * blockIdx.x] = gtimer();

    if (warp == 0) {
        // ===== TMA producers: lane 0 feeds the u ring, lane 1 the aux ring, each limited
        // only by its own ring (independent progress of diverged lanes, sm_70+) =====
        if (lane < 2) {
            const CUtensorMap* mu = &maps.u[lt];
            const CUtensorMap* ma = &maps.a[lp];
            if (lane == 0) {
                prefetch_map(mu);
            } else {
                prefetch_map(ma);
                prefetch_map(&maps.m);
                prefetch_map(&maps.damp);
            }
            uint64_t pol_first;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
            unsigned st = 0, ph = 0;
            bool lo_ready = c.ghost_lo_end <= 0 || c.need_lo == 0, hi_ready = !c.flags || c.need_hi == 0;
            if (!c.flags) lo_ready = hi_ready = true;
            for (int item = first; item < nitems; item += G) {
                const int col = item % sc.ncol, chunk = item / sc.ncol;
                int xa = sc.x0 + static_cast<int>(static_cast<long long>(sc.np) * chunk / sc.nchunk);
                int xb = sc.x0 + static_cast<int>(static_cast<long long>(sc.np) * (chunk + 1) / sc.nchunk);
                const int dir = (chunk & 1) ? 1 : -1;   // even chunks descend, odd ascend
                // stage-1 range of a chunk: its planes plus H overlap planes per side
                const int xa1 = max(xa - H, sc.x0), xb1 = min(xb + H, sc.x0 + sc.np);
                if (TB && role == 1) {
                    xa = xa1;
                    xb = xb1;
                }
                const int yt = sc.y0 + (col / sc.nzt) * T1;
                const int zt = sc.zs + (col % sc.nzt) * kT2;
                if (lane == 0) {
                    const int q0 = dir > 0 ? xa - H : xb - 1 + H;
                    const int nq = xb - xa + 2 * H;
                    unsigned long long seen = 0;  // K3 stage 2: min progress seen among neighbours
                    for (int j = 0; j < nq; ++j) {
                        const int q = q0 + dir * j;
                        if (q < c.ghost_lo_end && !lo_ready) {  // lower neighbour's step must be done
                            wait_counter(c.flags, c.need_lo, c.err);
                            lo_ready = true;
                        }
                        if (q >= c.ghost_hi_begin && !hi_ready) {
                            wait_counter(c.flags + 1, c.need_hi, c.err);
                            hi_ready = true;
                        }
                        if (TB && role == 2 && q >= xa1 && q < xb1) {
                            // u[t+1] plane q (with its y/z halo) must be stored by the stage-1
                            // CTAs of this column tile and its 3x3 neighbours (same chunk, same
                            // order); `seen` caches the smallest counter observed so far.
                            // Ask for kTbLead planes more than needed (capped at the stage-1
                            // item's end): stage 2 then trails stage 1 by a few planes instead of
                            // running dry at its edge, so its TMA ring stays primed.
                            const int idx = dir > 0 ? q - xa1 + 1 : xb1 - q;
                            const unsigned long long need_min = epoch + static_cast<unsigned long long>(idx);
                            const unsigned long long need =
                                epoch + static_cast<unsigned long long>(min(idx + kTbLead, xb1 - xa1));
                            if (seen < need_min) {
                                const int cy = col / sc.nzt, cz = col % sc.nzt;
                                const int ya = max(cy - 1, 0), yb = min(cy + 1, sc.nyt - 1);
                                const int za = max(cz - 1, 0), zb = min(cz + 1, sc.nzt - 1);
                                const unsigned long long* base = tb.cnt + chunk * sc.ncol;
                                const unsigned long long t0 = gtimer();
                                while (true) {  // all neighbour counters polled concurrently
                                    unsigned long long lo = ~0ull;
                                    for (int ny = ya; ny <= yb; ++ny)
                                        for (int nz = za; nz <= zb; ++nz) {
                                            unsigned long long v;
                                            asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];"
                                                         : "=l"(v) : "l"(base + ny * sc.nzt + nz) : "memory");
                                            lo = v < lo ? v : lo;
                                        }
                                    seen = lo;
                                    if (lo >= need) break;
                                    if (gtimer() - t0 > 20000000000ull) {
                                        atomicExch(c.err, 1u);
                                        break;
                                    }
                                    __nanosleep(64);
                                }
                                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                                asm volatile("fence.proxy.async.global;" ::: "memory");
                            }
                        }
                        mbar_wait(empty_u + 8 * st, ph ^ 1u);
                        mbar_expect_tx(full_u + 8 * st, C::ROWS * C::W2 * 4);
                        tma_load3(uring_s + st * C::UPLANE, mu, zt - C::A, yt - H, q, full_u + 8 * st);
                        ring_next<SU>(st, ph);
                    }
                } else {
                    const unsigned char* dfl =
                        sc.dflag ? sc.dflag + static_cast<long long>(col) * sc.np - sc.x0 : nullptr;
                    const int p0 = dir > 0 ? xa : xb - 1;
                    for (int j = 0; j < xb - xa; ++j) {
                        const int p = p0 + dir * j;
                        if (TB && role == 2) {
                            // u[t+2] overwrites u[t-1]: the neighbouring chunks' stage 1 reads
                            // u[t-1] on its H overlap planes; it must be past plane p first.
                            if (chunk > 0 && p < xa + H) {
                                const int xa0 = sc.x0 + static_cast<int>(static_cast<long long>(sc.np) * (chunk - 1) / sc.nchunk);
                                const int pa1 = max(xa0 - H, sc.x0), pb1 = min(xa + H, sc.x0 + sc.np);
                                const int n = ((chunk - 1) & 1) ? p - pa1 + 1 : pb1 - p;
                                wait_gpu(tb.cnt + (chunk - 1) * sc.ncol + col, epoch + static_cast<unsigned long long>(n),
                                         c.err);
                            }
                            if (chunk + 1 < sc.nchunk && p >= xb - H) {
                                const int xb2 = sc.x0 + static_cast<int>(static_cast<long long>(sc.np) * (chunk + 2) / sc.nchunk);
                                const int pa1 = max(xb - H, sc.x0), pb1 = min(xb2 + H, sc.x0 + sc.np);
                                const int n = ((chunk + 1) & 1) ? p - pa1 + 1 : pb1 - p;
                                wait_gpu(tb.cnt + (chunk + 1) * sc.ncol + col, epoch + static_cast<unsigned long long>(n),
                                         c.err);
                            }
                        }
                        mbar_wait(empty_a + 8 * st, ph ^ 1u);
                        const unsigned need_damp = (!dfl || dfl[p]) ? 1u : 0u;
                        aflag[st] = need_damp;  // published by the arrive below (release)
                        mbar_expect_tx(full_a + 8 * st, (need_damp ? 3 : 2) * C::ATILE);
                        const unsigned dst = aring_s + st * 3 * C::ATILE;
                        tma_load3_hint(dst, ma, zt, yt, p, full_a + 8 * st, pol_first);
                        // B (1/(m+g)) is re-read every step: default L2 policy (evict_first measured
                        // -3 % at 512^3 SO 8); u[t-1] and A stay evict_first
                        tma_load3(dst + C::ATILE, &maps.m, zt, yt, p, full_a + 8 * st);
                        if (need_damp)
                            tma_load3_hint(dst + 2 * C::ATILE, &maps.damp, zt, yt, p, full_a + 8 * st,
                                           pol_first);
                        ring_next<SA>(st, ph);
                    }
                }
            }
        }
    } else {
        // ===== consumers =====
        const int ct = threadIdx.x - 32;
        const int tz = ct & 15;
        const int ty = ct >> 4;
        const int r0 = ty * R1;  // first tile row of this thread
        float* un = pick3(g.lev[0], g.lev[1], g.lev[2], ln);
        float* lo_peer = pick3(pr.lo_lev[0], pr.lo_lev[1], pr.lo_lev[2], ln);
        float* hi_peer = pick3(pr.hi_lev[0], pr.hi_lev[1], pr.hi_lev[2], ln);
        // this thread's column inside a u plane / an aux tile (floats)
        const float* ucol = reinterpret_cast<const float*>(uring) + (r0 + H) * C::W2 + C::A + 4 * tz;
        const float* acol = reinterpret_cast<const float*>(aring) + r0 * kT2 + 4 * tz;
        float4 Q[R1][kUnroll ? NQ : 1];   // rotating register queue (H <= 3)
        float4 Qs[R1][(kUnroll || kTQ) ? 1 : 2 * H + UNR];  // shifting register queue
        unsigned su = 0, pu = 0, sp = 0, sa = 0, pa_ = 0;
        for (int item = first; item < nitems; item += G) {
            Pub pub;
            pub.cnt = (TB && role == 1) ? tb.cnt + item : nullptr;
            pub.base = epoch;
            pub.done = tally;
            pub.seq = static_cast<unsigned>((item - first) / G + 1);
            pub.H = H;
            pub.ncw = C::NCW;
            const int col = item % sc.ncol, chunk = item / sc.ncol;
            Item it;
            it.xa = sc.x0 + static_cast<int>(static_cast<long long>(sc.np) * chunk / sc.nchunk);
            it.xb = sc.x0 + static_cast<int>(static_cast<long long>(sc.np) * (chunk + 1) / sc.nchunk);
            if (TB && role == 1) {
                it.xa = max(it.xa - H, sc.x0);
                it.xb = min(it.xb + H, sc.x0 + sc.np);
            }
            it.dir = (chunk & 1) ? 1 : -1;
            it.q0 = it.dir > 0 ? it.xa - H : it.xb - 1 + H;
            it.nq = it.xb - it.xa + 2 * H;
            it.yt = sc.y0 + (col / sc.nzt) * T1 + r0;
            const int zt = sc.zs + (col % sc.nzt) * kT2;
            it.zc = zt + 4 * tz;  // first z of this thread's float4
            it.zfull = it.zc >= sc.z0 && it.zc + 3 < sc.z1;
            it.zmask = zmask_of(it.zc, sc.z0, sc.z1);
            it.rows_ok = it.yt + R1 - 1 < sc.y1;
            it.rowmask = 0u;
#pragma unroll
            for (int i = 0; i < R1; ++i) it.rowmask |= (it.yt + i < sc.y1) ? (1u << i) : 0u;
            {
                // one range covering the item's special planes (the epilogue re-tests them exactly)
                int s_lo = it.xb, s_hi = it.xa;
                const int ra[3] = {pr.lo_first, pr.hi_first, c.has_src ? c.src_x : 0};
                const int rb[3] = {pr.lo_last, pr.hi_last, c.has_src ? c.src_x + 1 : 0};
#pragma unroll
                for (int r = 0; r < 3; ++r) {
                    const int a = max(ra[r], it.xa), b = min(rb[r], it.xb);
                    if (a < b) {
                        s_lo = min(s_lo, a);
                        s_hi = max(s_hi, b);
                    }
                }
                it.s0 = s_lo;
                it.sn = s_lo < s_hi ? static_cast<unsigned>(s_hi - s_lo) : 0u;
            }
            it.gcol = static_cast<long long>(it.yt) * g.P2 + it.zc;
            it.xrun = static_cast<long long>(it.q0 + it.dir * H) * g.plane + it.gcol;  // first output plane
            sp = (su + H) % SU;  // stage of plane j = H, the first output plane of this item
            if (c.trace && ct == 0 && item == first) {
                // time when the first output plane's data is complete (end of warm-up)
                unsigned s2 = (su + 2 * H) % SU, p2 = pu ^ (((su + 2 * H) / SU) & 1u);
                mbar_wait(full_u + 8 * s2, p2);
                c.trace[4 * blockIdx.x + 1] = gtimer();
            }
            if constexpr (kTQ) {
                const unsigned tq = tmem_base + (static_cast<unsigned>(32 * (warp & 3)) << 16) +
                                    128u * static_cast<unsigned>(warp >> 2);
#pragma unroll 1
                for (int j = 0; j < it.nq; ++j)
                    consumer_step_tq<H, R1, T1, SU, SA>(tq, j, it, ucol, acol, aflag, full_u, empty_u, full_a,
                                                        empty_a, su, pu, sp, sa, pa_, mine, un, lo_peer, hi_peer,
                                                        g, K, c, pr, pub);
            } else if constexpr (kUnroll) {
#pragma unroll 1
                for (int jb = 0; jb < it.nq; jb += NQ)
                    Unrolled<H, R1, T1, SU, SA, 0>::run(Q, jb, it, ucol, acol, aflag, full_u, empty_u,
                                                        full_a, empty_a, su, pu, sp, sa, pa_, mine,
                                                        un, lo_peer, hi_peer, g, K, c, pr, pub);
            } else {
                // Partial unroll by UNR with a queue of 2H+UNR slots: plane j-m lives in slot
                // 2H+u-m inside a block, and the queue shifts down by UNR once per block
                // (2H/UNR float4 moves per plane instead of 2H).
#pragma unroll 1
                for (int jb = 0; jb < it.nq; jb += UNR) {
                    ShiftBlock<H, R1, T1, SU, SA, UNR, 0>::run(Qs, jb, it, ucol, acol, aflag, full_u, empty_u,
                                                             full_a, empty_a, su, pu, sp, sa, pa_, mine, un,
                                                             lo_peer, hi_peer, g, K, c, pr, pub);
#pragma unroll
                    for (int i = 0; i < R1; ++i)
#pragma unroll
                        for (int k = 0; k < 2 * H; ++k) Qs[i][k] = Qs[i][k + UNR];
                }
            }
        }
    }
    __syncwarp();
    // (peer stores reach system scope through thread 0's __threadfence_system in
    // signal_neighbours, after the CTA barrier in block_max_commit: fence cumulativity)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (c.trace && threadIdx.x == 32) c.trace[4 * blockIdx.x + 2] = gtimer();
    if constexpr (kTQ) asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    block_max_commit(mine, c.smax + c.slot);  // (contains the CTA barrier)
    if constexpr (kTQ) {
        if ((threadIdx.x >> 5) == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
        }
    }
    signal_neighbours(c);
    if (c.trace && threadIdx.x == 0) c.trace[4 * blockIdx.x + 3] = gtimer();
}

template <int H, int R1, int T1, int SU, int SA, int UNR, int TB>
__global__ void __launch_bounds__(Cfg<H, R1, T1>::NTHREADS, 1)
    k_tma(const __grid_constant__ Maps maps, Geo g, Coef K, Ctl c, Peer pr, Sched sc, TbCtl tb) {
    if constexpr (TB) {
        const int role = static_cast<int>(blockIdx.x) >= tb.ctas ? 2 : 1;
        Ctl cc = c;
        if (role == 2) {  // the second of the two steps
            ++cc.step;
            ++cc.slot;
        }
        tma_body<H, R1, T1, SU, SA, UNR, 1>(maps, g, K, cc, pr, sc, tb, role);
    } else {
        tma_body<H, R1, T1, SU, SA, UNR, 0>(maps, g, K, c, pr, sc, tb, 0);
    }
}

template <int H, int R1, int T1, int SU, int SA>
size_t smem_bytes() {
    using C = Cfg<H, R1, T1>;
    return static_cast<size_t>(SU) * C::UPLANE + static_cast<size_t>(SA) * 3 * C::ATILE +
           16 * (SU + SA) + 4 * SA + 4 * 17;
}

// Variant table: (H, R1, T1, SU, SA) chosen per space order to fit 227 KB of smem.
// (H, R1, T1, SU, SA, UNR): rows per thread, tile rows, u-ring stages, aux-ring stages,
// queue unroll (ignored for H <= 3, which rotates the queue by renaming).
#define SWB_TMA_VARIANTS(X)      \
    X(1, 1, 30, 5, 4, 1)         \
    X(2, 1, 30, 6, 4, 1)         \
    X(3, 1, 30, 7, 4, 1)         \
    X(4, 1, 30, 8, 4, 4)         \
    X(4, 1, 30, 11, 4, 4)        \
    X(5, 1, 30, 10, 4, 2)        \
    X(6, 1, 30, 10, 3, 2)        \
    X(6, 1, 30, 11, 3, 2)        \
    X(7, 1, 22, 14, 3, 2)        \
    X(8, 1, 22, 11, 3, 4)        \
    X(8, 1, 22, 14, 3, 4)        \
    X(1, 1, 28, 5, 4, 1)         \
    X(2, 1, 28, 6, 4, 1)         \
    X(3, 1, 28, 7, 4, 1)         \
    X(4, 1, 28, 8, 4, 4)         \
    X(5, 1, 28, 10, 4, 2)        \
    X(6, 1, 28, 10, 3, 2)        \
    X(6, 1, 26, 10, 3, 2)        \
    X(6, 1, 28, 10, 3, 4)        \
    X(8, 1, 30, 10, 2, 0)        \
    X(6, 1, 30, 10, 3, 0)        \
    X(8, 1, 20, 11, 3, 4)

using KernelFn = void (*)(Maps, Geo, Coef, Ctl, Peer, Sched, TbCtl);

struct Variant {
    int H, R1, T1, SU, SA, UNR;
    KernelFn fn;     // one step per launch (K1)
    KernelFn fn_tb;  // two steps per launch (K3)
    size_t smem;
    int threads;
};

#define SWB_VARIANT_ENTRY(h, r1, t1, su, sa, unr)                                                     \
    {h, r1, t1, su, sa, unr, k_tma<h, r1, t1, su, sa, unr, 0>, k_tma<h, r1, t1, su, sa, unr, 1>,   \
     smem_bytes<h, r1, t1, su, sa>(), Cfg<h, r1, t1>::NTHREADS},

// Rows per consumer thread: R1 = 1 doubles the consumer warps per SM (more latency hiding)
// at the cost of re-reading the y-neighbour rows per row; SWB_R1=1|2 overrides the default.
int preferred_r1(int H) {
    const char* env = std::getenv("SWB_R1");
    if (env && (env[0] == '1' || env[0] == '2')) return env[0] - '0';
    (void)H;
    return 1;
}

int preferred_unr(int H) {
    const char* env = std::getenv("SWB_UNR");
    if (env && env[0] >= '0' && env[0] <= '9') return env[0] - '0';  // 0: TMEM queue variants
    // measured on B200 at 256^3 and 512^3: 4 for SO 8, 12 and 16, 2 for SO 10/14
    // (SO 8 runs the rotating queue, which ignores UNR)
    return H == 4 || H == 6 || H == 8 ? 4 : (H >= 5 ? 2 : 1);
}

int preferred_su(int H) {
    const char* env = std::getenv("SWB_SU");
    if (env && env[0] >= '1' && env[0] <= '9') return std::atoi(env);
    (void)H;
    return 0;  // 0: first matching variant
}

int preferred_t1(int H) {
    const char* env = std::getenv("SWB_T1");
    if (env && std::atoi(env) > 0) return std::atoi(env);
    (void)H;
    return 0;  // 0: first matching variant
}

// t1_want: tile height chosen by tma_plan (0: any); SWB_T1 overrides it.
const Variant* find_variant(int H, int t1_want = 0) {
    static const Variant table[] = {SWB_TMA_VARIANTS(SWB_VARIANT_ENTRY)};
    const int r1 = preferred_r1(H), unr = preferred_unr(H), su = preferred_su(H);
    const int t1 = preferred_t1(H) ? preferred_t1(H) : t1_want;
    for (const auto& v : table)
        if (v.H == H && v.R1 == r1 && v.UNR == unr && (su == 0 || v.SU == su) && (t1 == 0 || v.T1 == t1)) return &v;
    for (const auto& v : table)
        if (v.H == H && v.R1 == r1 && (unr == 0 || v.UNR == unr) && (t1 == 0 || v.T1 == t1)) return &v;
    for (const auto& v : table)
        if (v.H == H && v.R1 == r1 && v.UNR == unr && (su == 0 || v.SU == su)) return &v;
    for (const auto& v : table)
        if (v.H == H && v.R1 == r1 && v.UNR == unr) return &v;
    for (const auto& v : table)
        if (v.H == H && v.R1 == r1) return &v;
    for (const auto& v : table)
        if (v.H == H) return &v;
    return nullptr;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

bool encode(CUtensorMap* map, const float* base, int n2, int n1, int nl0, int P2, int box0,
            int box1) {
    auto fn = get_encode();
    if (!fn) return false;
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(n2), static_cast<cuuint64_t>(n1),
                          static_cast<cuuint64_t>(nl0)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(P2) * 4,
                             static_cast<cuuint64_t>(P2) * 4 * static_cast<cuuint64_t>(n1)};
    cuuint32_t box[3] = {static_cast<cuuint32_t>(box0), static_cast<cuuint32_t>(box1), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides,
                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace

bool sq_variant(int H, int* T1, int* threads, int* smem, const void** fn);
cudaError_t launch_sq(const TmaPlan& plan, const void* maps, const Geo& g, const Coef& K, const Ctl& c,
                      const Peer& p, const void* sched, cudaStream_t s);

// Kernel choice: the register-queue variant (this file) by default -- measured faster than
// the smem-queue variant (k_sq.cu) at every SO (equal at SO 4/8 on 256^3, +40% at 512^3 SO 8,
// +30% at SO 16); SWB_KERNEL=sq selects the smem-queue variant.
TmaPlan tma_plan(int H, const Geo& g, int num_sms) {
    TmaPlan p{};
    p.ok = 0;
    p.H = H;
    p.num_sms = num_sms;
    const char* env = std::getenv("SWB_KERNEL");
    const bool want_rq = !(env && std::strcmp(env, "sq") == 0);
    int T1 = 0, threads = 0, smem = 0;
    const void* fn = nullptr;
    if (!want_rq && sq_variant(H, &T1, &threads, &smem, &fn)) {
        p.kind = 1;
        p.variant = 2000 + H;
    } else {
        // Tile height: among the K1 heights for this halo, the one whose row tiles waste the
        // fewest rows of the interior (measured +1-2 % at 256^3 SO 4/8/12 and 512^3 SO 8 over a
        // fixed height; heights below 28 lose warps and are not auto-selected).
        int t1_best = 0;
        double eff_best = -1.0;
        const int rows = g.y1 - g.y0;
        for (int cand : {30, 28, 22}) {
            if ((H <= 6) != (cand >= 28)) continue;
            const double eff = static_cast<double>(rows) / (static_cast<double>(ceil_div(rows, cand)) * cand);
            if (eff > eff_best + 1e-9) {
                eff_best = eff;
                t1_best = cand;
            }
        }
        const Variant* v = find_variant(H, t1_best);
        if (!v) return p;
        T1 = v->T1;
        threads = v->threads;
        smem = static_cast<int>(v->smem);
        fn = reinterpret_cast<const void*>(v->fn);
        p.kind = 0;
        p.variant = 1000 + 100 * (v->R1 - 1) + 10 * v->UNR + H + 100000 * v->T1;
    }
    p.T1 = T1;
    p.T2 = kT2;
    p.A = (H + 3) / 4 * 4;
    p.threads = threads;
    p.smem_bytes = smem;
    const int zs = g.z0 & ~3;
    p.zs = zs;
    p.tiles_y = ceil_div(g.y1 - g.y0, T1);
    p.tiles_z = ceil_div(g.z1 - zs, kT2);
    p.columns = p.tiles_y * p.tiles_z;
    const int np = g.x1 - g.x0;
    p.work = static_cast<long long>(p.columns) * np;
    if (np <= 0 || p.columns <= 0) return p;
    // Work items: column tiles x dim-0 chunks.  Chunk boundaries line up across columns and
    // alternate direction (even chunks descend, odd ascend), so CTAs meeting at a chunk
    // boundary read the shared planes at the same time (L2 hits), and neighbouring columns
    // stream the same planes concurrently (halo re-reads hit L2).  The chunk count minimises
    // the estimated makespan: rounds of items over the persistent CTAs x (chunk length +
    // warm-up of 2H planes, which cost about half an output plane each).
    int best = 1;
    double best_cost = 1e300;
    for (int nc = 1; nc <= 32 && nc <= np; ++nc) {
        const long long items = static_cast<long long>(p.columns) * nc;
        const long long rounds = (items + num_sms - 1) / num_sms;
        const double len = static_cast<double>(np) / nc;
        const double cost = static_cast<double>(rounds) * (std::ceil(len) + 0.5 * 2 * H);
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best = nc;
        }
    }
    if (const char* env_nc = std::getenv("SWB_NCHUNK")) {  // development override
        const int v = std::atoi(env_nc);
        if (v >= 1 && v <= np) best = v;
    }
    p.nchunk = best;
    p.grid = static_cast<int>(std::min<long long>(num_sms, static_cast<long long>(p.columns) * best));
    // K3 (two steps per launch): half the SMs run stage 1, half stage 2, all co-resident (the
    // stage-2 CTAs spin on stage-1 progress).  Stage 1 also computes H overlap planes per
    // chunk side; chunks are at least H planes long (the overlap only reaches the next chunk).
    {
        const int half = num_sms / 2;
        int tb_best = 0;
        double tb_cost = 1e300;
        for (int nc = 1; nc <= 32 && nc * std::max(H, 4) <= np; ++nc) {
            const long long items = static_cast<long long>(p.columns) * nc;
            const long long rounds = (items + half - 1) / half;
            const double len = static_cast<double>(np) / nc;
            const double cost = static_cast<double>(rounds) * (std::ceil(len) + 0.5 * 2 * H + 2 * H);
            if (cost < tb_cost - 1e-9) {
                tb_cost = cost;
                tb_best = nc;
            }
        }
        p.nchunk_tb = tb_best;
        p.tb_items = tb_best > 0 ? p.columns * tb_best : 0;
        p.tb_ok = (p.kind == 0 && tb_best > 0 && half >= 1) ? 1 : 0;
    }
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) {
        cudaGetLastError();
        return p;
    }
    if (p.tb_ok && p.kind == 0) {
        const Variant* v = find_variant(H, p.T1);
        if (cudaFuncSetAttribute(reinterpret_cast<const void*>(v->fn_tb),
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) {
            cudaGetLastError();
            p.tb_ok = 0;
        }
    }
    p.ok = 1;
    return p;
}

cudaError_t tma_make_maps(const TmaPlan& plan, const Geo& g, int nl0, void* out) {
    Maps* maps = static_cast<Maps*>(out);
    std::memset(maps, 0, sizeof(Maps));
    const int W2 = kT2 + 2 * plan.A;
    for (int l = 0; l < 3; ++l) {
        if (!encode(&maps->u[l], g.lev[l], g.n2, g.n1, nl0, g.P2, W2, plan.T1 + 2 * plan.H))
            return cudaErrorInvalidValue;
        if (!encode(&maps->a[l], g.lev[l], g.n2, g.n1, nl0, g.P2, kT2, plan.T1))
            return cudaErrorInvalidValue;
    }
    if (!encode(&maps->m, g.m, g.n2, g.n1, nl0, g.P2, kT2, plan.T1)) return cudaErrorInvalidValue;
    if (!encode(&maps->damp, g.damp, g.n2, g.n1, nl0, g.P2, kT2, plan.T1))
        return cudaErrorInvalidValue;
    return cudaSuccess;
}

static_assert(sizeof(Maps) == kTmaMapsBytes, "tensor-map block size");

namespace {
__global__ void k_update_coefs(float* __restrict__ m, float* __restrict__ damp, long long n, float half_dt) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const float mf = m[i];
        const float g = damp[i] * half_dt;  // fl(damp dt/2), as the update has always rounded it
        float b = 0.f, a = 0.f;
#if SWB_COMBINE == 2
        b = mf + g;  // D
        a = mf - g;  // E
#else
        if (mf != 0.f) {
            const double mp = static_cast<double>(mf) + static_cast<double>(g);
            b = static_cast<float>(1.0 / mp);
            a = static_cast<float>((static_cast<double>(mf) - static_cast<double>(g)) / mp);
        }
#endif
        m[i] = b;
        damp[i] = a;
    }
}

// flags[col * np + (x - x0)] = any damp != 0 over the output points of that tile and plane
__global__ void k_damp_flags(const float* __restrict__ damp, long long plane, int P2, int x0, int np,
                             int y0, int y1, int z0, int z1, int zs, int T1, int tiles_z,
                             unsigned char* flags) {
    const int col = blockIdx.y, x = x0 + blockIdx.x;
    const int yt = y0 + (col / tiles_z) * T1, zt = zs + (col % tiles_z) * kT2;
    const int ya = yt, yb = min(yt + T1, y1), za = max(zt, z0), zb = min(zt + kT2, z1);
    int any = 0;
    for (int t = threadIdx.x; t < (yb - ya) * kT2; t += blockDim.x) {
        const int y = ya + t / kT2, z = zt + t % kT2;
        if (z >= za && z < zb && damp[x * plane + static_cast<long long>(y) * P2 + z] != 0.0f) any = 1;
    }
    any = __syncthreads_or(any);
    if (threadIdx.x == 0) flags[static_cast<long long>(col) * np + blockIdx.x] = static_cast<unsigned char>(any);
}
}  // namespace

cudaError_t tma_update_coefs(float* m, float* damp, long long n, float half_dt, cudaStream_t s) {
    k_update_coefs<<<device_sm_count() * 8, 256, 0, s>>>(m, damp, n, half_dt);
    return cudaGetLastError();
}


cudaError_t tma_damp_flags_device(const TmaPlan& plan, const Geo& g, unsigned char* flags, cudaStream_t s) {
    const int np = g.x1 - g.x0;
    if (np <= 0 || plan.columns <= 0) return cudaSuccess;
    dim3 grid(np, plan.columns);
    k_damp_flags<<<grid, 256, 0, s>>>(g.damp, g.plane, g.P2, g.x0, np, g.y0, g.y1, g.z0, g.z1, plan.zs,
                                     plan.T1, plan.tiles_z, flags);
    return cudaGetLastError();
}

void tma_damp_flags(const TmaPlan& plan, const Geo& g, const float* damp, int n1, int n2,
                    unsigned char* flags) {
    const int np = g.x1 - g.x0;
    for (int col = 0; col < plan.columns; ++col) {
        const int yt = g.y0 + (col / plan.tiles_z) * plan.T1;
        const int zt = plan.zs + (col % plan.tiles_z) * kT2;
        const int ya = yt, yb = std::min(yt + plan.T1, g.y1);
        const int za = std::max(zt, g.z0), zb = std::min(zt + kT2, g.z1);
        for (int x = g.x0; x < g.x1; ++x) {
            unsigned char f = 0;
            if (damp) {
                const float* pl = damp + static_cast<long long>(x + g.xg_off) * n1 * n2;
                for (int y = ya; y < yb && !f; ++y)
                    for (int z = za; z < zb; ++z)
                        if (pl[static_cast<long long>(y) * n2 + z] != 0.0f) {
                            f = 1;
                            break;
                        }
            }
            flags[static_cast<long long>(col) * np + (x - g.x0)] = f;
        }
    }
}

cudaError_t launch_tma(const TmaPlan& plan, const void* maps, const Geo& g, const Coef& K,
                       const Ctl& c, const Peer& p, cudaStream_t s) {
    const Variant* v = find_variant(plan.H, plan.T1);
    if (!plan.ok || (plan.kind == 0 && !v)) return cudaErrorInvalidValue;
    Sched sc;
    sc.nyt = plan.tiles_y;
    sc.nzt = plan.tiles_z;
    sc.ncol = plan.columns;
    sc.np = g.x1 - g.x0;
    sc.nchunk = plan.nchunk;
    sc.dflag = plan.dflag;
    sc.y0 = g.y0;
    sc.y1 = g.y1;
    sc.z0 = g.z0;
    sc.z1 = g.z1;
    sc.zs = plan.zs;
    sc.x0 = g.x0;
    if (plan.kind == 1) return launch_sq(plan, maps, g, K, c, p, &sc, s);
    TbCtl tb{};
    return launch_pdl(reinterpret_cast<const void*>(v->fn), plan.grid, v->threads, v->smem, s,
                      *static_cast<const Maps*>(maps), g, K, c, p, sc, tb);
}

cudaError_t launch_tma_tb(const TmaPlan& plan, const void* maps, const Geo& g, const Coef& K,
                          const Ctl& c, const TbCtl& tb_in, cudaStream_t s) {
    const Variant* v = find_variant(plan.H, plan.T1);
    if (!plan.ok || !plan.tb_ok || plan.kind != 0 || !v || !tb_in.cnt) return cudaErrorInvalidValue;
    Sched sc;
    sc.nyt = plan.tiles_y;
    sc.nzt = plan.tiles_z;
    sc.ncol = plan.columns;
    sc.np = g.x1 - g.x0;
    sc.nchunk = plan.nchunk_tb;
    sc.dflag = plan.dflag;
    sc.y0 = g.y0;
    sc.y1 = g.y1;
    sc.z0 = g.z0;
    sc.z1 = g.z1;
    sc.zs = plan.zs;
    sc.x0 = g.x0;
    TbCtl tb = tb_in;
    tb.ctas = tb_ctas(plan);
    Peer none{};
    return launch_pdl(reinterpret_cast<const void*>(v->fn_tb), 2 * tb.ctas, v->threads, v->smem, s,
                      *static_cast<const Maps*>(maps), g, K, c, none, sc, tb);
}

}  // namespace swb
