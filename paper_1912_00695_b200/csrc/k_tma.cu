// K1: TMA-staged 2.5D factorised stencil for sm_100a.
//
// One persistent CTA per SM strides over work items (column tile x dim-0 chunk): a column
// tile is T1 rows (dim 1) x 64 cols (dim 2) of output points; the CTA streams it along dim 0
// (the reference's slowest axis "x"; the north star's "z-slab" axis) over the chunk's planes.
// Warp 0 is the TMA producer (lane 0: u ring, lane 1: aux ring); the pencil variants (SO 8 and 12 on
// 28-row tiles, SO 16 on 20-row tiles) have a y-pencil warp at warp 4 (far y terms, see ypencil_loop);
// the other warps are consumers.
//
//   u ring  : halo-padded planes of u[t] ((T1+2H) x (64+2A) floats) loaded by
//             cp.async.bulk.tensor.3d; a plane stays resident from its arrival (when the
//             consumers take its centre values into the register queue) until the output
//             plane with the same index has used it for the in-plane (dim 1 / dim 2) stencil,
//             H planes later.  Depth S_U = H + 1 + prefetch.
//   aux ring: u[t-1], B, A tiles (T1 x 64) of the output plane, one TMA each (A only where
//             the tile is damped); B and A are the coefficient fields that replace m and damp.
//             Pencil variants add a fourth slot, P_y, written by the pencil warp.
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

#ifndef SWB_DIFF_K
#define SWB_DIFF_K 1  // difference form (neighbour minus centre) for the terms k <= SWB_DIFF_K
#endif
#ifndef SWB_UNROLL_MAXH
#define SWB_UNROLL_MAXH 4  // rotate the register queue by renaming up to this halo (measured: +1 % at SO 8; I-cache misses beyond)
#endif
// Summation of the k >= 2 terms, chosen per halo (measured, DESIGN.md §4 numerics):
//   2 (H <= 2): full difference form -- every neighbour minus the centre before the sum, residual
//     fp32(3 (c0 + 2 sum c_k)) u.  SO 4 then holds ~4e-6 relative L2 after 10k steps instead of
//     1.5e-5 (the sum of six values ~u cancelled against R3 u); 1 % slower at SO 4;
//   1 (H == 6): the pairs of each axis first (+1.9 % at SO 12, same accuracy);
//   0: (x pair + (y pair + z pair)).
template <int H>
constexpr int lap_form() { return H <= 2 ? 2 : (H == 6 ? 1 : 0); }
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
// ghost planes, and the source injection with the reference's two roundings) and the max|u|
// fold.
template <int H, int R1>
__device__ __forceinline__ void epilogue_store(const float4* out, int p, long long xoff,
                                               const Item& it, unsigned& mine, float* un, float* lo_peer,
                                               float* hi_peer, const Geo& g, const Coef& K, const Ctl& c,
                                               const Peer& pr) {
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
                    store_row<true>(un + xoff + static_cast<long long>(i) * g.P2, out[i], it.zmask, mine);
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
}

// ---- y-pencil warp (variants with YW = 1; SO 16 on grids where the 20-row tile is chosen) ----
// The consumers are bound by shared-memory traffic and latency at SO 16: per output float4 they
// issue 2H LDS.128 for the y neighbours alone.  A pencil warp takes the far y terms k >= kP of
// every output plane:
//   P_y = sum_{k=H..kP} c_k (u_{y-k} + u_{y+k})                                       FP32
// Each lane owns one float4 column and half of the tile rows and holds its whole pencil (T1/2 + 2H
// rows) in registers, so every u value is read from shared memory once per pencil instead of once
// per output that needs it; P_y goes to a two-stage ring and the consumers read it with one
// LDS.128 in place of 2 (H - kP + 1) loads.  kP balances the pencil warp against the consumers.
// Warps are spread over the four SM sub-partitions as warp % 4, so the pencil warp shares an issue
// port with whatever warps sit on its sub-partition: placed after the consumers (warp 11) it shared
// one with two consumer warps and was issue-bound beyond kP = 5; placed at warp 4 it shares one with
// the (nearly idle) TMA producer warp and one consumer, and takes one more y pair.  Measured at SO 16
// on B200 (256^3, 20-row tile, GPts/s; profiles/pencil_r02.txt, pencil_place_r02.txt):
//   warp 11: kP = 3: 202, 4: 209, 5: 219, 6: 214, 7: 209, 8: 201;   no pencil 208.5 / 209.5
//   warp 4:  kP = 3: 227.9, 4: 230.6, 5: 225.6
// With P_y handed over through the aux ring (SWB_PY_AUX, below) the pencil costs the consumers no
// barrier, and the SO 8 and SO 12 variants (28 rows + pencil = 16 warps at 128 registers) pay off too:
// SO 8 k >= 2: 313 -> 318, SO 12 k >= 4: 251 -> 266 GPts/s at 256^3 (with their own ring they had
// measured slower or equal: profiles/pencil_r02.txt, pencil12_r02.txt; now pencil8_r02.txt,
// pencil12_aux_r02.txt, pencil12_unr_r02.txt).
// Ring roles with SWB_PY_AUX: ypencil_loop's (sring, SS, full_s, empty_s, STAGE_F) are the aux ring's
// fourth slot, SA stages, its full / empty barriers and its stage stride; without it, the P_y ring's.
#ifndef SWB_PENCIL_K
#define SWB_PENCIL_K 0  // development override of the pencil split point (0: H - 4)
#endif
#ifndef SWB_PENCIL_WARP
#define SWB_PENCIL_WARP 4  // physical warp of the first pencil warp (0: after the consumers)
#endif
#ifndef SWB_PENCIL_SS
#define SWB_PENCIL_SS 0  // development override of the P_y ring depth (0: 2 per pencil warp)
#endif
#ifndef SWB_PY_AUX
#define SWB_PY_AUX 1  // P_y in a fourth slot of the aux ring stage (one barrier pair for aux + P_y)
#endif
// With SWB_PY_AUX the pencil writes P_y of output plane p into the aux-ring stage of p and arrives on
// its full barrier (initialised for the TMA producer's arrive plus the 32 pencil lanes), so the
// consumers wait once and release once per plane for u[t-1], B, A and P_y together.
template <int YW>
constexpr bool py_aux() { return YW > 0 && SWB_PY_AUX != 0; }
template <int YW>
constexpr int aux_slots() { return py_aux<YW>() ? 4 : 3; }
#ifndef SWB_PENCIL_K6
#define SWB_PENCIL_K6 4  // split point of the SO 12 pencil variant (k >= 3 / 5 measured slower, pencil12_r02.txt)
#endif
#ifndef SWB_PENCIL_K4
#define SWB_PENCIL_K4 2  // split point of the SO 8 pencil variant (k >= 3: -0.5 %, k >= 4: -1.6 % at 256^3)
#endif
template <int H>
constexpr int pencil_k() {
    return SWB_PENCIL_K > 0 ? SWB_PENCIL_K : (H == 6 ? SWB_PENCIL_K6 : (H == 4 ? SWB_PENCIL_K4 : H - 4));
}
// A pencil lane holds SEG/NSUB + 2H rows at a time (the halo rows between sub-segments are read
// twice): SO 12's 28-row tile has 14 rows per pencil, two sub-segments fit its 128-register cap.
template <int H>
constexpr int pencil_nsub() { return H <= 6 ? 2 : 1; }

struct YRing {
    unsigned full, empty;  // mbarriers of stage 0 (8 bytes apart)
    const float* col;      // this consumer's float4 in stage 0
    unsigned st, ph;       // consumer's stage / phase
};

// Pencil warp yw (of YW) takes output planes g = yw, yw + YW, ... of this CTA in the consumers'
// order.  The consumers wait for P_y of output plane p before they release p's u-ring stage, so
// the pencil's reads of that stage are ordered before the TMA overwrite (mbarrier release/acquire).
template <int H, int T1, int SU, int SS, int YW, int STAGE_F>
__device__ __forceinline__ void ypencil_loop(int yw, int lane, const unsigned char* uring, float* sring,
                                             unsigned full_u, unsigned full_s, unsigned empty_s,
                                             const Coef& K, const Sched& sc, int first, int G, int nitems) {
    using C = Cfg<H, 1, T1, YW>;
    constexpr int SEG = T1 / 2;
    constexpr int NL = SEG + 2 * H;
    constexpr int KP = pencil_k<H>();
    constexpr int SUB = (SEG + pencil_nsub<H>() - 1) / pencil_nsub<H>();
    static_assert(T1 % 2 == 0 && KP >= 2, "two pencils per column; k = 1 stays with the consumers");
    const int tz = lane & 15, seg = lane >> 4;
    const float* ub = reinterpret_cast<const float*>(uring) + seg * SEG * C::W2 + C::A + 4 * tz;
    float* sb = sring + seg * SEG * kT2 + 4 * tz;
    unsigned gseq = 0, useq = 0;  // output planes / u-ring planes of the items before this one
    for (int item = first; item < nitems; item += G) {
        const int chunk = item / sc.ncol;
        const int xa = sc.x0 + static_cast<int>(static_cast<long long>(sc.np) * chunk / sc.nchunk);
        const int xb = sc.x0 + static_cast<int>(static_cast<long long>(sc.np) * (chunk + 1) / sc.nchunk);
        const int np = xb - xa;
#pragma unroll 1
        for (int j = static_cast<int>((yw + YW - gseq % YW) % YW); j < np; j += YW) {
            const unsigned gs = gseq + j, us = useq + j + H;  // output plane j is u-ring plane j + H
            const unsigned sst = gs % SS, sph = (gs / SS) & 1u;
            const unsigned ust = us % SU, uph = (us / SU) & 1u;
            mbar_wait(empty_s + 8 * sst, sph ^ 1u);
            mbar_wait(full_u + 8 * ust, uph);
            const float* pl = ub + ust * (C::UPLANE / 4);
            float* so = sb + sst * STAGE_F;
            // all rows of a sub-segment first (no queue here), then k outer / outputs inner, so the
            // sub-segment's independent FFMA2 chains advance together
#pragma unroll
            for (int s0 = 0; s0 < SEG; s0 += SUB) {
                constexpr int NV = SUB + 2 * H;
                float4 v[NV];
#pragma unroll
                for (int i = 0; i < NV; ++i)
                    if (s0 + i < NL) v[i] = *reinterpret_cast<const float4*>(pl + (s0 + i) * C::W2);
                float2 al[SUB], ah[SUB];
#pragma unroll
                for (int o = 0; o < SUB; ++o) al[o] = ah[o] = splat(0.f);
#pragma unroll
                for (int k = H; k >= KP; --k) {
                    const float2 ck = splat(K.c[k]);
#pragma unroll
                    for (int o = 0; o < SUB; ++o) {  // output row s0 + o of the pencil: centre v[o + H]
                        if (s0 + o < SEG) {
                            al[o] = fma2(ck, add2(lo2(v[o + H - k]), lo2(v[o + H + k])), al[o]);
                            ah[o] = fma2(ck, add2(hi2(v[o + H - k]), hi2(v[o + H + k])), ah[o]);
                        }
                    }
                }
#pragma unroll
                for (int o = 0; o < SUB; ++o)
                    if (s0 + o < SEG)
                        *reinterpret_cast<float4*>(so + (s0 + o) * kT2) =
                            make_float4(al[o].x, al[o].y, ah[o].x, ah[o].y);
            }
            mbar_arrive(full_s + 8 * sst);  // release: this lane's P_y stores
        }
        gseq += np;
        useq += np + 2 * H;
    }
}

template <int H, int R1, int T1, int SU, int SA, int QN, int U, int YW, int SS>
__device__ __forceinline__ void consumer_step(float4 (&Q)[R1][QN], int j, Item& it,
                                              const float* ucol, const float* acol,
                                              const unsigned* aflag, unsigned full_u,
                                              unsigned empty_u, unsigned full_a, unsigned empty_a,
                                              unsigned& su, unsigned& pu, unsigned& sp,
                                              unsigned& sa, unsigned& pa_, unsigned& mine,
                                              float* un, float* lo_peer, float* hi_peer,
                                              const Geo& g, const Coef& K, const Ctl& c,
                                              const Peer& pr, YRing& yr) {
    using C = Cfg<H, R1, T1, YW>;
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
        constexpr int kLap = lap_form<H>();
        const float2 cl = lo2(Q[i][UC]), chh = hi2(Q[i][UC]);
#pragma unroll
        for (int k = H; k >= 2; --k) {
            const float2 ck = splat(K.c[k]);
            // far y pairs k >= pencil_k come from the pencil warp (P_y); the loads are issued first,
            // as in the variants without it (the register-capped SO 12 variant is sensitive to it)
            const bool from_pencil = YW > 0 && k >= pencil_k<H>();
            const float4 ym = from_pencil ? make_float4(0.f, 0.f, 0.f, 0.f)
                                          : *reinterpret_cast<const float4*>(rowc - k * C::W2);
            const float4 yp = from_pencil ? make_float4(0.f, 0.f, 0.f, 0.f)
                                          : *reinterpret_cast<const float4*>(rowc + k * C::W2);
            const float4& xm = Q[i][(UC + NQ - k) % NQ];
            const float4& xp = Q[i][(UC + k) % NQ];
            float2 sl, sh;
            if (from_pencil) {
                float2 zl, zh;
                if ((k & 1) == 0) {
                    zl = add2(make_float2(w[C::A - k], w[C::A + 1 - k]), make_float2(w[C::A + k], w[C::A + 1 + k]));
                    zh = add2(make_float2(w[C::A + 2 - k], w[C::A + 3 - k]),
                              make_float2(w[C::A + 2 + k], w[C::A + 3 + k]));
                } else {
                    zl = make_float2(w[C::A - k] + w[C::A + k], w[C::A + 1 - k] + w[C::A + 1 + k]);
                    zh = make_float2(w[C::A + 2 - k] + w[C::A + 2 + k], w[C::A + 3 - k] + w[C::A + 3 + k]);
                }
                sl = add2(add2(lo2(xm), lo2(xp)), zl);
                sh = add2(add2(hi2(xm), hi2(xp)), zh);
            } else if (kLap == 2 || k <= SWB_DIFF_K) {
                // full difference form: every neighbour minus the centre first
                const float2 zl = make_float2((w[C::A - k] - cl.x) + (w[C::A + k] - cl.x),
                                              (w[C::A + 1 - k] - cl.y) + (w[C::A + 1 + k] - cl.y));
                const float2 zh = make_float2((w[C::A + 2 - k] - chh.x) + (w[C::A + 2 + k] - chh.x),
                                              (w[C::A + 3 - k] - chh.y) + (w[C::A + 3 + k] - chh.y));
                sl = add2(add2(sub2(lo2(xm), cl), sub2(lo2(xp), cl)),
                          add2(add2(sub2(lo2(ym), cl), sub2(lo2(yp), cl)), zl));
                sh = add2(add2(sub2(hi2(xm), chh), sub2(hi2(xp), chh)),
                          add2(add2(sub2(hi2(ym), chh), sub2(hi2(yp), chh)), zh));
            } else {
                float2 zl, zh;
                if ((k & 1) == 0) {  // register-pair aligned: packed adds
                    zl = add2(make_float2(w[C::A - k], w[C::A + 1 - k]), make_float2(w[C::A + k], w[C::A + 1 + k]));
                    zh = add2(make_float2(w[C::A + 2 - k], w[C::A + 3 - k]),
                              make_float2(w[C::A + 2 + k], w[C::A + 3 + k]));
                } else {
                    zl = make_float2(w[C::A - k] + w[C::A + k], w[C::A + 1 - k] + w[C::A + 1 + k]);
                    zh = make_float2(w[C::A + 2 - k] + w[C::A + 2 + k], w[C::A + 3 - k] + w[C::A + 3 + k]);
                }
                if constexpr (kLap == 1) {  // pairs of one axis first
                    sl = add2(add2(add2(lo2(xm), lo2(xp)), add2(lo2(ym), lo2(yp))), zl);
                    sh = add2(add2(add2(hi2(xm), hi2(xp)), add2(hi2(ym), hi2(yp))), zh);
                } else {
                    sl = add2(add2(lo2(xm), lo2(xp)), add2(add2(lo2(ym), lo2(yp)), zl));
                    sh = add2(add2(hi2(xm), hi2(xp)), add2(add2(hi2(ym), hi2(yp)), zh));
                }
            }
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
    if constexpr (YW > 0 && !py_aux<YW>()) {  // + P_y of this output plane (pencil warp)
        static_assert(R1 == 1, "pencil variants run one row per consumer thread");
        mbar_wait(yr.full + 8 * yr.st, yr.ph);
        const float4 sy = *reinterpret_cast<const float4*>(yr.col + yr.st * (T1 * kT2));
        mbar_arrive(yr.empty + 8 * yr.st);
        ring_next<SS>(yr.st, yr.ph);
        acc[0][0] = add2(acc[0][0], lo2(sy));
        acc[0][1] = add2(acc[0][1], hi2(sy));
    }
    // ---- aux tiles: u[t-1], m, damp ----
    mbar_wait(full_a + 8 * sa, pa_);
    const float* aux = acol + sa * (aux_slots<YW>() * C::ATILE / 4);
    const bool has_damp = aflag[sa] != 0u;
    if constexpr (py_aux<YW>()) {  // + P_y of this output plane (pencil warp, fourth aux slot)
        static_assert(R1 == 1, "pencil variants run one row per consumer thread");
        const float4 sy = *reinterpret_cast<const float4*>(aux + 3 * C::ATILE / 4);
        acc[0][0] = add2(acc[0][0], lo2(sy));
        acc[0][1] = add2(acc[0][1], hi2(sy));
    }
    float4 upv[R1], bv[R1], av[R1];
#pragma unroll
    for (int i = 0; i < R1; ++i) {
        upv[i] = *reinterpret_cast<const float4*>(aux + i * kT2);
        bv[i] = *reinterpret_cast<const float4*>(aux + C::ATILE / 4 + i * kT2);
        av[i] = has_damp ? *reinterpret_cast<const float4*>(aux + C::ATILE / 2 + i * kT2)
                         : make_float4(1.f, 1.f, 1.f, 1.f);
    }
    mbar_arrive(empty_a + 8 * sa);
    mbar_arrive(empty_u + 8 * sp);  // plane p is no longer needed
    ring_next<SA>(sa, pa_);
    if (++sp == SU) sp = 0;
    // ---- combine: u+ = u + A (u - u-) + B Lr (dt/h)^2 (coefficient fields, tma_update_coefs) ----
    const float2 R3 = splat(lap_form<H>() == 2 ? K.R3f : (SWB_DIFF_K > 1 ? K.R3k[SWB_DIFF_K - 1] : K.R3)),
                 khi = splat(K.kap_hi), klo = splat(K.kap_lo);
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
    epilogue_store<H, R1>(out, p, xoff, it, mine, un, lo_peer, hi_peer, g, K, c, pr);
}

template <int H, int R1, int T1, int SU, int SA, int U, int YW, int SS>
struct Unrolled {
    __device__ __forceinline__ static void run(float4 (&Q)[R1][2 * H + 1], int jb, Item& it,
                                               const float* ucol, const float* acol,
                                               const unsigned* aflag, unsigned full_u, unsigned empty_u,
                                               unsigned full_a, unsigned empty_a, unsigned& su,
                                               unsigned& pu, unsigned& sp, unsigned& sa, unsigned& pa_,
                                               unsigned& mine, float* un, float* lo_peer,
                                               float* hi_peer, const Geo& g, const Coef& K,
                                               const Ctl& c, const Peer& pr, YRing& yr) {
        if (jb + U < it.nq) {
            consumer_step<H, R1, T1, SU, SA, 2 * H + 1, U, YW, SS>(Q, jb + U, it, ucol, acol, aflag, full_u, empty_u,
                                                full_a, empty_a, su, pu, sp, sa, pa_, mine, un,
                                                lo_peer, hi_peer, g, K, c, pr, yr);
            Unrolled<H, R1, T1, SU, SA, U + 1, YW, SS>::run(Q, jb, it, ucol, acol, aflag, full_u, empty_u,
                                                    full_a, empty_a, su, pu, sp, sa, pa_, mine, un,
                                                    lo_peer, hi_peer, g, K, c, pr, yr);
        }
    }
};
template <int H, int R1, int T1, int SU, int SA, int YW, int SS>
struct Unrolled<H, R1, T1, SU, SA, 2 * H + 1, YW, SS> {
    __device__ __forceinline__ static void run(float4 (&)[R1][2 * H + 1], int, Item&,
                                               const float*, const float*, const unsigned*, unsigned,
                                               unsigned, unsigned, unsigned, unsigned&, unsigned&,
                                               unsigned&, unsigned&, unsigned&, unsigned&, float*,
                                               float*, float*, const Geo&, const Coef&, const Ctl&,
                                               const Peer&, YRing&) {}
};

template <int H, int R1, int T1, int SU, int SA, int UNR, int U, int YW, int SS>
struct ShiftBlock {
    __device__ __forceinline__ static void run(float4 (&Q)[R1][2 * H + UNR], int jb, Item& it,
                                               const float* ucol, const float* acol,
                                               const unsigned* aflag, unsigned full_u, unsigned empty_u,
                                               unsigned full_a, unsigned empty_a, unsigned& su,
                                               unsigned& pu, unsigned& sp, unsigned& sa, unsigned& pa_,
                                               unsigned& mine, float* un, float* lo_peer,
                                               float* hi_peer, const Geo& g, const Coef& K,
                                               const Ctl& c, const Peer& pr, YRing& yr) {
        if (jb + U < it.nq) {
            consumer_step<H, R1, T1, SU, SA, 2 * H + UNR, 2 * H + U, YW, SS>(
                Q, jb + U, it, ucol, acol, aflag, full_u, empty_u, full_a, empty_a, su, pu, sp, sa, pa_,
                mine, un, lo_peer, hi_peer, g, K, c, pr, yr);
            ShiftBlock<H, R1, T1, SU, SA, UNR, U + 1, YW, SS>::run(Q, jb, it, ucol, acol, aflag, full_u, empty_u,
                                                           full_a, empty_a, su, pu, sp, sa, pa_, mine, un,
                                                           lo_peer, hi_peer, g, K, c, pr, yr);
        }
    }
};
template <int H, int R1, int T1, int SU, int SA, int UNR, int YW, int SS>
struct ShiftBlock<H, R1, T1, SU, SA, UNR, UNR, YW, SS> {
    __device__ __forceinline__ static void run(float4 (&)[R1][2 * H + UNR], int, Item&, const float*,
                                               const float*, const unsigned*, unsigned, unsigned, unsigned,
                                               unsigned, unsigned&, unsigned&, unsigned&, unsigned&,
                                               unsigned&, unsigned&, float*, float*, float*, const Geo&,
                                               const Coef&, const Ctl&, const Peer&, YRing&) {}
};

// The kernel body: one time step over the items of this persistent CTA.
template <int H, int R1, int T1, int SU, int SA, int UNR, int YW>
__device__ __forceinline__ void tma_body(const Maps& maps, const Geo& g, const Coef& K, const Ctl& c,
                                         const Peer& pr, const Sched& sc) {
    using C = Cfg<H, R1, T1, YW>;
    constexpr int SS = YW > 0 ? (SWB_PENCIL_SS > 0 ? SWB_PENCIL_SS : 2 * YW) : 1;  // y-pencil ring stages
    constexpr int NQ = C::NQ;
    // Small halos: unroll the plane loop by the queue depth so the register queue rotates by
    // renaming; large halos: shift the queue (keeps the loop body small for the I-cache).
    constexpr bool kUnroll = H <= SWB_UNROLL_MAXH;
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char* uring = smem;
    unsigned char* aring = smem + SU * C::UPLANE;
    constexpr int AS = aux_slots<YW>() * C::ATILE;  // bytes per aux stage
    float* sring = reinterpret_cast<float*>(aring + SA * AS);  // YW > 0 without py_aux: P_y stages (T1 x 64)
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(sring) +
                                                 (YW > 0 && !py_aux<YW>() ? SS * C::ATILE : 0));
    unsigned* aflag = reinterpret_cast<unsigned*>(bars + 2 * (SU + SA + SS));  // damp-present per aux stage
    const unsigned full_u = smem_addr(bars), empty_u = full_u + 8 * SU;
    const unsigned full_a = empty_u + 8 * SU, empty_a = full_a + 8 * SA;
    const unsigned full_s = empty_a + 8 * SA, empty_s = full_s + 8 * SS;
    const unsigned uring_s = smem_addr(uring), aring_s = smem_addr(aring);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // roles: warp 0 producer; pencil warps PW0 .. PW0 + YW - 1; the other warps are consumers in
    // order (warps are spread over the SM sub-partitions as warp % 4)
    constexpr int PW0 = (YW > 0 && SWB_PENCIL_WARP > 0) ? SWB_PENCIL_WARP : C::NCW + 1;
    const bool is_pencil = YW > 0 && warp >= PW0 && warp < PW0 + YW;
    const int cw = warp - 1 - ((YW > 0 && warp >= PW0 + YW) ? YW : 0);  // consumer ordinal
    if (threadIdx.x == 0) {
        for (int i = 0; i < SU; ++i) {
            mbar_init(full_u + 8 * i, 1);
            mbar_init(empty_u + 8 * i, 32 * C::NCW);  // every consumer thread arrives
        }
        for (int i = 0; i < SA; ++i) {
            mbar_init(full_a + 8 * i, py_aux<YW>() ? 1 + 32 : 1);  // (+ the pencil lanes)
            mbar_init(empty_a + 8 * i, 32 * C::NCW);
        }
        for (int i = 0; i < SS; ++i) {
            mbar_init(full_s + 8 * i, 32);  // one pencil warp writes a stage
            mbar_init(empty_s + 8 * i, 32 * C::NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    // per-CTA stamps (SWB_TRACE): [entry, after griddepcontrol.wait, warm-up done, consumers done,
    // exit] of the last two launches (even / odd step)
    // (recomputed from the launch parameters at each use: a pointer kept live would cost the
    // register-capped variants a spill)
#define SWB_TRACE_AT(i) c.trace[8 * blockIdx.x + (i)]  // (the host offsets c.trace by the step parity)
    if (c.trace && threadIdx.x == 0) {
        SWB_TRACE_AT(0) = gtimer();
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        SWB_TRACE_AT(5) = smid;
    }
    // Programmatic dependent launch: everything above overlapped the previous step's tail;
    // u[t], u[t-1] written by that step are only touched after this point.
    asm volatile("griddepcontrol.wait;" ::: "memory");

    const int lt = c.step % 3, ln = (c.step + 1) % 3, lp = (c.step + 2) % 3;
    const int nitems = sc.ncol * sc.nchunk;
    const int first = static_cast<int>(blockIdx.x), G = static_cast<int>(gridDim.x);  // persistent CTAs
    unsigned mine = 0u;
    if (c.trace && threadIdx.x == 0) SWB_TRACE_AT(1) = gtimer();

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
                const int xa = sc.x0 + static_cast<int>(static_cast<long long>(sc.np) * chunk / sc.nchunk);
                const int xb = sc.x0 + static_cast<int>(static_cast<long long>(sc.np) * (chunk + 1) / sc.nchunk);
                const int dir = (chunk & 1) ? 1 : -1;   // even chunks descend, odd ascend
                const int yt = sc.y0 + (col / sc.nzt) * T1;
                const int zt = sc.zs + (col % sc.nzt) * kT2;
                if (lane == 0) {
                    const int q0 = dir > 0 ? xa - H : xb - 1 + H;
                    const int nq = xb - xa + 2 * H;
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
                        mbar_wait(empty_a + 8 * st, ph ^ 1u);
                        const unsigned need_damp = (!dfl || dfl[p]) ? 1u : 0u;
                        aflag[st] = need_damp;  // published by the arrive below (release)
                        mbar_expect_tx(full_a + 8 * st, (need_damp ? 3 : 2) * C::ATILE);
                        const unsigned dst = aring_s + st * AS;
                        // u[t-1] evict_first, except at SO 16, whose tile rows straddle two 256-byte
                        // L2 segments (tile_z_start): the neighbouring tile's half then survives
                        // (+0.4 % at SO 16, -0.7 % at SO 8; profiles/um1_policy_r02.txt)
                        if constexpr (H >= 8)
                            tma_load3(dst, ma, zt, yt, p, full_a + 8 * st);
                        else
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
    } else if (is_pencil) {
        // ===== y-pencil warps =====
        if constexpr (YW > 0)
            if constexpr (py_aux<YW>())
                ypencil_loop<H, T1, SU, SA, YW, AS / 4>(warp - PW0, lane, uring,
                                                        reinterpret_cast<float*>(aring) + 3 * C::ATILE / 4, full_u,
                                                        full_a, empty_a, K, sc, first, G, nitems);
            else
                ypencil_loop<H, T1, SU, SS, YW, T1 * kT2>(warp - PW0, lane, uring, sring, full_u, full_s, empty_s, K,
                                            sc, first, G, nitems);
    } else {
        // ===== consumers =====
        const int ct = cw * 32 + lane;
        const int tz = ct & 15;
        const int ty = ct >> 4;
        const int r0 = ty * R1;  // first tile row of this thread
        float* un = pick3(g.lev[0], g.lev[1], g.lev[2], ln);
        float* lo_peer = pick3(pr.lo_lev[0], pr.lo_lev[1], pr.lo_lev[2], ln);
        float* hi_peer = pick3(pr.hi_lev[0], pr.hi_lev[1], pr.hi_lev[2], ln);
        // this thread's column inside a u plane / an aux tile (floats)
        const float* ucol = reinterpret_cast<const float*>(uring) + (r0 + H) * C::W2 + C::A + 4 * tz;
        const float* acol = reinterpret_cast<const float*>(aring) + r0 * kT2 + 4 * tz;
        float4 Q[R1][kUnroll ? NQ : 1];              // rotating register queue (H <= SWB_UNROLL_MAXH)
        float4 Qs[R1][kUnroll ? 1 : 2 * H + UNR];   // shifting register queue
        unsigned su = 0, pu = 0, sp = 0, sa = 0, pa_ = 0;
        YRing yr{full_s, empty_s, sring + r0 * kT2 + 4 * tz, 0u, 0u};
        for (int item = first; item < nitems; item += G) {
            const int col = item % sc.ncol, chunk = item / sc.ncol;
            Item it;
            it.xa = sc.x0 + static_cast<int>(static_cast<long long>(sc.np) * chunk / sc.nchunk);
            it.xb = sc.x0 + static_cast<int>(static_cast<long long>(sc.np) * (chunk + 1) / sc.nchunk);
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
                SWB_TRACE_AT(2) = gtimer();
            }
            if constexpr (kUnroll) {
#pragma unroll 1
                for (int jb = 0; jb < it.nq; jb += NQ)
                    Unrolled<H, R1, T1, SU, SA, 0, YW, SS>::run(Q, jb, it, ucol, acol, aflag, full_u, empty_u,
                                                        full_a, empty_a, su, pu, sp, sa, pa_, mine,
                                                        un, lo_peer, hi_peer, g, K, c, pr, yr);
            } else {
                // Partial unroll by UNR with a queue of 2H+UNR slots: plane j-m lives in slot
                // 2H+u-m inside a block, and the queue shifts down by UNR once per block
                // (2H/UNR float4 moves per plane instead of 2H).
#pragma unroll 1
                for (int jb = 0; jb < it.nq; jb += UNR) {
                    ShiftBlock<H, R1, T1, SU, SA, UNR, 0, YW, SS>::run(Qs, jb, it, ucol, acol, aflag, full_u, empty_u,
                                                             full_a, empty_a, su, pu, sp, sa, pa_, mine, un,
                                                             lo_peer, hi_peer, g, K, c, pr, yr);
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
    if (c.trace && threadIdx.x == 32) SWB_TRACE_AT(3) = gtimer();
    block_max_commit(mine, c.smax + c.slot);  // (contains the CTA barrier)
    signal_neighbours(c);
    if (c.trace && threadIdx.x == 0) SWB_TRACE_AT(4) = gtimer();
#undef SWB_TRACE_AT
}

template <int H, int R1, int T1, int SU, int SA, int UNR, int YW>
__global__ void __launch_bounds__(Cfg<H, R1, T1, YW>::NTHREADS, 1)
    k_tma(const __grid_constant__ Maps maps, Geo g, Coef K, Ctl c, Peer pr, Sched sc) {
    tma_body<H, R1, T1, SU, SA, UNR, YW>(maps, g, K, c, pr, sc);
}
template <int H, int R1, int T1, int SU, int SA, int YW>
size_t smem_bytes() {
    using C = Cfg<H, R1, T1, YW>;
    constexpr int SS = YW > 0 ? (SWB_PENCIL_SS > 0 ? SWB_PENCIL_SS : 2 * YW) : 1;
    return static_cast<size_t>(SU) * C::UPLANE + static_cast<size_t>(SA) * aux_slots<YW>() * C::ATILE +
           (YW > 0 && !py_aux<YW>() ? static_cast<size_t>(SS) * C::ATILE : 0) + 16 * (SU + SA + SS) + 4 * SA;
}

// Variant table: (H, R1, T1, SU, SA) chosen per space order to fit 227 KB of smem.
// (H, R1, T1, SU, SA, UNR, YW): rows per thread, tile rows, u-ring stages, aux-ring stages,
// queue unroll (ignored for H <= 4, which rotates the queue by renaming), y-pencil warps.
#define SWB_TMA_VARIANTS(X)      \
    X(1, 1, 30, 5, 4, 1, 0)         \
    X(2, 1, 30, 6, 4, 1, 0)         \
    X(3, 1, 30, 7, 4, 1, 0)         \
    X(4, 1, 30, 8, 4, 4, 0)         \
    X(5, 1, 30, 10, 4, 2, 0)        \
    X(6, 1, 30, 10, 3, 2, 0)        \
    X(7, 1, 22, 14, 3, 2, 0)        \
    X(8, 1, 22, 11, 3, 4, 0)        \
    X(1, 1, 28, 5, 4, 1, 0)         \
    X(2, 1, 28, 6, 4, 1, 0)         \
    X(3, 1, 28, 7, 4, 1, 0)         \
    X(4, 1, 28, 8, 4, 4, 0)         \
    X(5, 1, 28, 10, 4, 2, 0)        \
    X(6, 1, 28, 10, 3, 4, 0)        \
    X(8, 1, 20, 11, 3, 4, 0)        \
    X(8, 1, 20, 13, 3, 3, 1)        \
    X(6, 1, 28, 10, 3, 3, 1)        \
    X(4, 1, 28, 8, 4, 4, 1)


using KernelFn = void (*)(Maps, Geo, Coef, Ctl, Peer, Sched);

struct Variant {
    int H, R1, T1, SU, SA, UNR, YW;
    KernelFn fn;
    size_t smem;
    int threads;
};

#define SWB_VARIANT_ENTRY(h, r1, t1, su, sa, unr, yw)                                              \
    {h, r1, t1, su, sa, unr, yw, k_tma<h, r1, t1, su, sa, unr, yw>, smem_bytes<h, r1, t1, su, sa, yw>(), \
     Cfg<h, r1, t1, yw>::NTHREADS},

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
    if (env && env[0] >= '1' && env[0] <= '9') return env[0] - '0';
    // measured on B200 at 256^3 and 512^3: 4 for SO 8, 12 and 16, 2 for SO 10/14;
    // the SO 16 pencil variant exists only with 3 and is found by the fallback (with P_y through the
    // aux ring, 256^3 / 384^3 / 512^3 GPts/s: UNR 2 233 / 238 / 255, 3 239 / 245 / 261, 4 239 / 243 / 261,
    // 5 239 / 245 / 261, 6 236 / 241 / 258, 8 222 / 228 / 244; profiles/pencil16_unr_r02.txt); the SO 12
    // pencil variant likewise only with 3 (UNR 1 / 2 / 3 at 256^3: 250 / 261 / 266 GPts/s, pencil12_unr_r02.txt)
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

// y-pencil warps per CTA (0: the consumers read the 2H y neighbours themselves); SWB_YW overrides.
int preferred_yw(int H) {
    const char* env = std::getenv("SWB_YW");
    if (env && env[0] >= '0' && env[0] <= '9') return env[0] - '0';
    (void)H;
    return -1;  // -1: the plan's choice
}

// t1_want / yw_want: tile height and pencil warps chosen by tma_plan (0: any height / none);
// SWB_T1 and SWB_YW override them.
const Variant* find_variant(int H, int t1_want = 0, int yw_want = 0) {
    static const Variant table[] = {SWB_TMA_VARIANTS(SWB_VARIANT_ENTRY)};
    const int r1 = preferred_r1(H), unr = preferred_unr(H), su = preferred_su(H);
    const int t1 = preferred_t1(H) ? preferred_t1(H) : t1_want;
    const int yw_pref = preferred_yw(H) >= 0 ? preferred_yw(H) : yw_want;
    for (int yw : {yw_pref, 0}) {
        for (const auto& v : table)
            if (v.H == H && v.YW == yw && v.R1 == r1 && v.UNR == unr && (su == 0 || v.SU == su) &&
                (t1 == 0 || v.T1 == t1))
                return &v;
        for (const auto& v : table)
            if (v.H == H && v.YW == yw && v.R1 == r1 && (unr == 0 || v.UNR == unr) && (t1 == 0 || v.T1 == t1))
                return &v;
        for (const auto& v : table)
            if (v.H == H && v.YW == yw && v.R1 == r1 && v.UNR == unr && (su == 0 || v.SU == su)) return &v;
        for (const auto& v : table)
            if (v.H == H && v.YW == yw && v.R1 == r1 && v.UNR == unr) return &v;
        for (const auto& v : table)
            if (v.H == H && v.YW == yw && v.R1 == r1) return &v;
        for (const auto& v : table)
            if (v.H == H && v.YW == yw) return &v;
    }
    return nullptr;
}

// A variant with exactly this tile height and pencil count exists for the halo (rows-per-thread
// preference applied).
bool find_variant_exact(int H, int t1, int yw) {
    const Variant* v = find_variant(H, t1, yw);
    return v && v->T1 == t1 && v->YW == yw;
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

// L2 promotion of a map (SWB_PROMO_U / SWB_PROMO_A = 0, 64, 128 or 256 override it, development A/B).
// 256 B, except the u boxes at SO <= 12: with the 256-byte aligned z tiles their 64 + 2A float rows
// reach A floats into each neighbouring segment, and 128 B promotion fetched less of those
// (512^3 SO 8: 374 -> 377 GPts/s; 256^3 within noise; profiles/promo_r02.txt).
CUtensorMapL2promotion promo_env(const char* name, int dflt = 256) {
    const char* env = std::getenv(name);
    const int v = env ? std::atoi(env) : dflt;
    return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                  : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                            : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
}

bool encode(CUtensorMap* map, const float* base, int n2, int n1, int nl0, int P2, int box0,
            int box1, CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B) {
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
                    promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace

// Kernel plan for one handle: the variant (tile height by row efficiency), the column tiles and
// the dim-0 chunk count.
// First dim-2 column of z tile 0.  For H < 8, tiles start on a 64-float (256-byte) boundary when
// that needs no extra tile, so the aux-tile rows (u[t-1], B, A: T1 x 64 floats) and the output rows
// each sit in one 256-byte L2 segment instead of straddling two (the lanes left of z0 are masked
// like the right edge); otherwise at z0 rounded down to a float4, which aligns the u box
// (zt - A = z0 - H) instead.  Measured (profiles/zalign_r02.txt, 256^3): SO 8 307 -> 314 GPts/s
// (512^3: 360 -> 373), SO 12 +0.4 %, SO 16 -0.4 % (its u box of 64 + 16 floats then spans three
// segments), SO 4 unchanged (z0 & ~3 is already 0).  SWB_ZALIGN=0/1 forces either (development A/B).
int tile_z_start(const Geo& g, int H) {
    const int z4 = g.z0 & ~3, z64 = g.z0 & ~(kT2 - 1);
    const char* env = std::getenv("SWB_ZALIGN");
    const bool align = env ? env[0] == '1' : H < 8;
    return align && ceil_div(g.z1 - z64, kT2) == ceil_div(g.z1 - z4, kT2) ? z64 : z4;
}

TmaPlan tma_plan(int H, const Geo& g, int num_sms) {
    TmaPlan p{};
    p.ok = 0;
    p.H = H;
    p.num_sms = num_sms;
    // Tile height and dim-0 chunk count together: among the K1 heights for this halo (28/30 rows at
    // SO <= 12, 20/22 at SO 14-16), the pair with the smallest estimated makespan
    //     rounds(columns x chunks over the persistent CTAs) x (chunk length + warm-up) x t(T1),
    // where t(T1) ~ T1^0.25 is the time a CTA takes per plane of a T1-row tile (measured: a 20-row
    // SO 16 tile streams a plane 2.3 % faster than a 22-row one; the kernel is shared-memory and
    // latency bound, not proportional to rows).  At 256^3 SO 16 this picks 20 rows: 48 columns x 3
    // chunks fill 144 of 148 SMs instead of 132 (+2.4 %); at 512^3 it keeps 22 (20 rows: -8 %).
    // Ties go to the height that wastes fewer interior rows.  SWB_TPLAN=rows: row efficiency only
    // (the previous rule, development A/B).  A variant with a y-pencil warp streams a plane in
    // kPencilTime of the time (SO 16, 20 rows, pencil on the producer's sub-partition taking
    // k >= 4, P_y in the aux ring, queue unroll 3: 239.4 against 209.5 GPts/s at 256^3; at 512^3 the
    // 20-row pencil tile runs 261 against 250 for the 22-row tile without it; profiles/pyaux_r02.txt,
    // pencil16_unr_r02.txt; the factor is kept at the 0.89 measured with unroll 6, which already
    // puts 256^3, 384^3 and 512^3 on the pencil tile and 320^3 / 448^3 on the 22-row one).
    const int rows = g.y1 - g.y0;
    const int np_all = g.x1 - g.x0;
    const int zs_all = tile_z_start(g, H);
    const int tz_all = ceil_div(g.z1 - zs_all, kT2);
    const bool rows_only = std::getenv("SWB_TPLAN") && std::strcmp(std::getenv("SWB_TPLAN"), "rows") == 0;
    auto makespan = [&](int t1, int* nchunk_out) {
        const long long cols = static_cast<long long>(ceil_div(rows, t1)) * tz_all;
        double best_cost = 1e300;
        int best_nc = 1;
        for (int nc = 1; nc <= 32 && nc <= std::max(np_all, 1); ++nc) {
            const long long rounds = (cols * nc + num_sms - 1) / num_sms;
            const double cost = static_cast<double>(rounds) * (std::ceil(static_cast<double>(np_all) / nc) + H);
            if (cost < best_cost - 1e-9) {
                best_cost = cost;
                best_nc = nc;
            }
        }
        if (nchunk_out) *nchunk_out = best_nc;
        return best_cost * std::pow(static_cast<double>(t1), 0.25);
    };
    constexpr double kPencilTime = 0.89;
    // SO 12: the 28-row tile with a pencil warp (16 warps at 128 registers, queue unroll 3, P_y
    // through the aux ring) against the 15-warp tile without it: 266.0 against 250.8 GPts/s at 256^3,
    // 282.3 / 267.0 at 384^3, 323.9 / 304.7 at 512^3 (profiles/pencil12_aux_r02.txt, pencil12_unr_r02.txt)
    constexpr double kPencilTime12 = 0.94;
    // SO 8: the same with k >= 2 in the pencil: 318.0 against 313.4 GPts/s at 256^3, equal at 512^3
    // (profiles/pencil8_r02.txt)
    constexpr double kPencilTime8 = 0.985;
    int t1_best = 0, yw_best = 0;
    double eff_best = -1.0, cost_best = 1e300;
    for (int yw : {0, 1})
        for (int cand : {30, 28, 22, 20}) {
            if ((H <= 6) != (cand >= 28)) continue;
            if (!find_variant_exact(H, cand, yw)) continue;
            const double eff = static_cast<double>(rows) / (static_cast<double>(ceil_div(rows, cand)) * cand);
            const double cost = rows_only || np_all <= 0 || rows <= 0
                                    ? 0.0
                                    : makespan(cand, nullptr) * (yw ? (H == 8 ? kPencilTime : H == 6 ? kPencilTime12 : kPencilTime8) : 1.0);
            if (cost < cost_best * (1 - 1e-9) || (cost <= cost_best * (1 + 1e-9) && eff > eff_best + 1e-9)) {
                cost_best = cost;
                eff_best = eff;
                t1_best = cand;
                yw_best = yw;
            }
        }
    const Variant* v = find_variant(H, t1_best, yw_best);
    if (!v) return p;
    p.variant = 1000 + 100 * (v->R1 - 1) + 10 * v->UNR + H + 100000 * v->T1 + 10000000 * v->YW;
    p.T1 = v->T1;
    p.yw = v->YW;
    p.T2 = kT2;
    p.A = (H + 3) / 4 * 4;
    p.threads = v->threads;
    p.smem_bytes = static_cast<int>(v->smem);
    const int zs = tile_z_start(g, H);
    p.zs = zs;
    p.tiles_y = ceil_div(g.y1 - g.y0, p.T1);
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
    // warm-up of 2H planes, which cost about half an output plane each).  Among equal makespans
    // with items of at most 4 planes (small grids: each item is a short latency-bound pipeline
    // fill) the most items win: more CTAs start at once and the average item is shorter
    // (64^3 SO 2: 31 chunks 5.9 us per step, 49 chunks 5.4 us; scripts/small_sweep.py).
    int best = 1;
    double best_cost = 1e300;
    for (int nc = 1; nc <= 64 && nc <= np; ++nc) {
        const long long items = static_cast<long long>(p.columns) * nc;
        const long long rounds = (items + num_sms - 1) / num_sms;
        const double len = static_cast<double>(np) / nc;
        const double cost = static_cast<double>(rounds) * (std::ceil(len) + 0.5 * 2 * H);
        if (cost < best_cost - 1e-9 || (cost <= best_cost + 1e-9 && std::ceil(len) <= 4)) {
            best_cost = cost;
            best = nc;
        }
    }
    if (const char* env_nc = std::getenv("SWB_NCHUNK")) {  // development override
        const int n = std::atoi(env_nc);
        if (n >= 1 && n <= np) best = n;
    }
    p.nchunk = best;
    p.grid = static_cast<int>(std::min<long long>(num_sms, static_cast<long long>(p.columns) * best));
    if (cudaFuncSetAttribute(reinterpret_cast<const void*>(v->fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                             p.smem_bytes) != cudaSuccess) {
        cudaGetLastError();
        return p;
    }
    p.ok = 1;
    return p;
}

cudaError_t tma_make_maps(const TmaPlan& plan, const Geo& g, int nl0, void* out) {
    Maps* maps = static_cast<Maps*>(out);
    std::memset(maps, 0, sizeof(Maps));
    const int W2 = kT2 + 2 * plan.A;
    for (int l = 0; l < 3; ++l) {
        if (!encode(&maps->u[l], g.lev[l], g.n2, g.n1, nl0, g.P2, W2, plan.T1 + 2 * plan.H, promo_env("SWB_PROMO_U", plan.H < 8 ? 128 : 256)))
            return cudaErrorInvalidValue;
        if (!encode(&maps->a[l], g.lev[l], g.n2, g.n1, nl0, g.P2, kT2, plan.T1, promo_env("SWB_PROMO_A")))
            return cudaErrorInvalidValue;
    }
    if (!encode(&maps->m, g.m, g.n2, g.n1, nl0, g.P2, kT2, plan.T1, promo_env("SWB_PROMO_A"))) return cudaErrorInvalidValue;
    if (!encode(&maps->damp, g.damp, g.n2, g.n1, nl0, g.P2, kT2, plan.T1, promo_env("SWB_PROMO_A")))
        return cudaErrorInvalidValue;
    return cudaSuccess;
}

static_assert(sizeof(Maps) == kTmaMapsBytes, "tensor-map block size");

namespace {
// Round x (double) to one of the two floats around it, the upper one with probability equal to
// x's position between them, drawn from a hash of the cell's global index: E[result] = x exactly.
// A plain round-to-nearest B = fl(1/m) has the same relative error at every cell of a constant
// medium -- a velocity bias of up to 6e-8, a phase drift linear in time (1e-5 relative L2 after 10k
// steps at SO 16); dithered, the medium is exact on average (5.5e-6).  Keyed by the global index,
// so z-slab decompositions get the same coefficients bit for bit.
__device__ __forceinline__ float dither_round(double x, unsigned long long key) {
    const float lo = __double2float_rz(x);
    const float hi = nextafterf(lo, x > 0 ? INFINITY : -INFINITY);
    if (x == static_cast<double>(lo)) return lo;
    const double fr = (x - static_cast<double>(lo)) / (static_cast<double>(hi) - static_cast<double>(lo));
    unsigned long long z = key + 0x9e3779b97f4a7c15ull;  // splitmix64
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    return static_cast<double>(z >> 11) * 0x1.0p-53 < fr ? hi : lo;
}

__global__ void k_update_coefs(float* __restrict__ m, float* __restrict__ damp, long long n, float half_dt,
                               int P2, int n1, int n2, int xg_off) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int z = static_cast<int>(i % P2);
        const long long row = i / P2;  // local plane * n1 + y
        const unsigned long long key =
            (static_cast<unsigned long long>(row + static_cast<long long>(xg_off) * n1)) * n2 + z;  // global C index
        const float mf = m[i];
        const float g = damp[i] * half_dt;  // fl(damp dt/2), as the update has always rounded it
        float b = 0.f, a = 0.f;
        if (mf != 0.f && z < n2) {
            const double mp = static_cast<double>(mf) + static_cast<double>(g);
            b = dither_round(1.0 / mp, key);
            a = g == 0.f ? 1.f : dither_round((static_cast<double>(mf) - static_cast<double>(g)) / mp,
                                               key ^ 0x5555555555555555ull);
        }
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

cudaError_t tma_update_coefs(float* m, float* damp, long long n, float half_dt, int P2, int n1, int n2, int xg_off,
                             cudaStream_t s) {
    k_update_coefs<<<device_sm_count() * 8, 256, 0, s>>>(m, damp, n, half_dt, P2, n1, n2, xg_off);
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
    const Variant* v = find_variant(plan.H, plan.T1, plan.yw);
    if (!plan.ok || !v) return cudaErrorInvalidValue;
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
    return launch_pdl(reinterpret_cast<const void*>(v->fn), plan.grid, v->threads, v->smem, s,
                      *static_cast<const Maps*>(maps), g, K, c, p, sc);
}

}  // namespace swb
