// K1: TMA-staged 2.5D factorised stencil for sm_100a.
//
// One persistent CTA per SM walks a contiguous, balanced range of (column tile, plane)
// work: a column tile is T1 rows (dim 1) x 64 cols (dim 2) of output points; the CTA
// streams it along dim 0 (the reference's slowest axis "x"; the north star's "z-slab"
// axis).  Warp 0 is the TMA producer; warps 1..NC are consumers.
//
//   u ring  : halo-padded planes of u[t] ((T1+2H) x (64+2A) floats) loaded by
//             cp.async.bulk.tensor.3d; a plane stays resident from its arrival (when the
//             consumers take its centre values into the register queue) until the output
//             plane with the same index has used it for the in-plane (dim 1 / dim 2) stencil,
//             H planes later.  Depth S_U = H + 1 + prefetch.
//   aux ring: u[t-1], m, damp tiles (T1 x 64) of the output plane, one TMA each.
//   register queue: each consumer thread keeps u[t] of its R1 x 4 points for the 2H+1
//             planes around the output plane (the dim-0 stencil never touches smem).
//
// Arithmetic per point (factorised form, src/pipeline.cpp:467-512 with the sign fix):
//   S  = sum_k>=2 c_k (u_-k + u_+k) over the three axes + c_1 sum((u_-1 - u) + (u_+1 - u))
//   Lr = S + 3 (c_0 + 2 c_1) u
//   u+ = u + [ (m - g)(u - u-) + Lr (dt/h)^2 ] / (m + g),   g = damp dt/2
// (see combine_f32 in k_common.cuh), then the fused epilogue: source injection with the
// reference's two roundings, 128-bit stores, peer stores of slab-boundary planes, and the
// per-step max|u| / non-finite flag.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>

#include "k_common.cuh"
#include "kernels.h"

namespace swb {
namespace {

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
    long long work;       // ncol * np
    int y0, y1, z0, z1, zs, x0;
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
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
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

// Walk the segments [col, p_lo, p_hi) of this CTA's balanced work range.
struct SegIter {
    long long u, end;
    int np;
    __device__ SegIter(long long work, int np_, int cta, int ncta) : np(np_) {
        u = work * cta / ncta;
        end = work * (cta + 1) / ncta;
    }
    __device__ bool next(int& col, int& pa, int& pb) {
        if (u >= end) return false;
        col = static_cast<int>(u / np);
        pa = static_cast<int>(u % np);
        const long long cend = static_cast<long long>(col + 1) * np;
        const long long e = end < cend ? end : cend;
        pb = static_cast<int>(e - static_cast<long long>(col) * np);
        u = e;
        return true;
    }
};

template <int H, int R1, int T1>
struct Cfg {
    static constexpr int A = (H + 3) / 4 * 4;         // dim-2 halo rounded to float4
    static constexpr int W2 = kT2 + 2 * A;             // smem row length (floats)
    static constexpr int ROWS = T1 + 2 * H;            // smem rows per plane
    static constexpr int UPLANE = (ROWS * W2 * 4 + 127) / 128 * 128;
    static constexpr int ATILE = T1 * kT2 * 4;         // one aux tile (bytes)
    static constexpr int NCW = (T1 / R1) * 16 / 32;    // consumer warps
    static constexpr int NTHREADS = 32 * (NCW + 1);
    static constexpr int NQ = 2 * H + 1;               // queue depth
};

template <int H, int R1, int T1, int SU, int SA>
__global__ void __launch_bounds__(Cfg<H, R1, T1>::NTHREADS, 1)
    k_tma(const __grid_constant__ Maps maps, Geo g, Coef K, Ctl c, Peer pr, Sched sc) {
    using C = Cfg<H, R1, T1>;
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char* uring = smem;
    unsigned char* aring = smem + SU * C::UPLANE;
    uint64_t* bars = reinterpret_cast<uint64_t*>(aring + SA * 3 * C::ATILE);
    const unsigned full_u = smem_addr(bars), empty_u = full_u + 8 * SU;
    const unsigned full_a = empty_u + 8 * SU, empty_a = full_a + 8 * SA;
    const unsigned uring_s = smem_addr(uring), aring_s = smem_addr(aring);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < SU; ++i) {
            mbar_init(full_u + 8 * i, 1);
            mbar_init(empty_u + 8 * i, C::NCW);
        }
        for (int i = 0; i < SA; ++i) {
            mbar_init(full_a + 8 * i, 1);
            mbar_init(empty_a + 8 * i, C::NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();

    const int lt = c.step % 3, ln = (c.step + 1) % 3, lp = (c.step + 2) % 3;
    const int ncta = gridDim.x;
    unsigned mine = 0u;

    if (warp == 0) {
        // ===== TMA producer (one elected lane) =====
        if (lane == 0) {
            const CUtensorMap* mu = &maps.u[lt];
            const CUtensorMap* ma = &maps.a[lp];
            prefetch_map(mu);
            prefetch_map(ma);
            prefetch_map(&maps.m);
            prefetch_map(&maps.damp);
            constexpr int DA = SA - 1 < 2 ? SA - 1 : 2;  // aux prefetch distance (planes)
            unsigned nu = 0, na = 0;
            SegIter it(sc.work, sc.np, blockIdx.x, ncta);
            int col, pa, pb;
            while (it.next(col, pa, pb)) {
                const int yt = sc.y0 + (col / sc.nzt) * T1;
                const int zt = sc.zs + (col % sc.nzt) * kT2;
                const int xa = sc.x0 + pa, xb = sc.x0 + pb;  // local output planes [xa, xb)
                for (int q = xa - H; q < xb + H; ++q) {
                    const unsigned st = nu % SU, ph = (nu / SU) & 1u;
                    mbar_wait(empty_u + 8 * st, ph ^ 1u);
                    mbar_expect_tx(full_u + 8 * st, C::ROWS * C::W2 * 4);
                    tma_load3(uring_s + st * C::UPLANE, mu, zt - C::A, yt - H, q, full_u + 8 * st);
                    ++nu;
                    const int p = q - H + DA;
                    if (p >= xa && p < xb) {
                        const unsigned sa = na % SA, pha = (na / SA) & 1u;
                        mbar_wait(empty_a + 8 * sa, pha ^ 1u);
                        mbar_expect_tx(full_a + 8 * sa, 3 * C::ATILE);
                        const unsigned dst = aring_s + sa * 3 * C::ATILE;
                        tma_load3(dst, ma, zt, yt, p, full_a + 8 * sa);
                        tma_load3(dst + C::ATILE, &maps.m, zt, yt, p, full_a + 8 * sa);
                        tma_load3(dst + 2 * C::ATILE, &maps.damp, zt, yt, p, full_a + 8 * sa);
                        ++na;
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
        float4 Q[R1][C::NQ];  // register queue along dim 0
        unsigned nu = 0, na = 0;
        SegIter it(sc.work, sc.np, blockIdx.x, ncta);
        int col, pa, pb;
        while (it.next(col, pa, pb)) {
            const int yt = sc.y0 + (col / sc.nzt) * T1;
            const int zt = sc.zs + (col % sc.nzt) * kT2;
            const int xa = sc.x0 + pa, xb = sc.x0 + pb;
            const int zc = zt + 4 * tz;  // first z of this thread's float4
            const unsigned base_u = nu;  // sequence number of plane xa - H
#pragma unroll 1
            for (int q = xa - H; q < xb + H; ++q) {
                const unsigned st = nu % SU, ph = (nu / SU) & 1u;
                mbar_wait(full_u + 8 * st, ph);
                const unsigned plane_q = uring_s + st * C::UPLANE;
                // shift the queue and append the centre values of plane q
#pragma unroll
                for (int i = 0; i < R1; ++i) {
#pragma unroll
                    for (int k = 0; k < C::NQ - 1; ++k) Q[i][k] = Q[i][k + 1];
                    Q[i][C::NQ - 1] =
                        lds4(plane_q + 4 * ((r0 + i + H) * C::W2 + C::A + 4 * tz));
                }
                ++nu;
                const bool keep = q >= xa && q < xb;  // needed later for an in-plane stencil
                if (!keep) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(empty_u + 8 * st);
                }
                const int p = q - H;
                if (p < xa) continue;
                // ---- output plane p: in-plane stencil from its smem stage ----
                const unsigned sp = (base_u + static_cast<unsigned>(p - (xa - H))) % SU;
                const unsigned plane_p = uring_s + sp * C::UPLANE;
                float4 acc[R1];
#pragma unroll
                for (int i = 0; i < R1; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
                // far terms (k >= 2): dim 0 from the queue, dim 1 / dim 2 from smem
#pragma unroll
                for (int k = H; k >= 2; --k) {
                    const float ck = K.c[k];
#pragma unroll
                    for (int i = 0; i < R1; ++i) {
                        const float4 a0 = Q[i][H - k], b0 = Q[i][H + k];
                        const float4 a1 = lds4(plane_p + 4 * ((r0 + i + H - k) * C::W2 + C::A + 4 * tz));
                        const float4 b1 = lds4(plane_p + 4 * ((r0 + i + H + k) * C::W2 + C::A + 4 * tz));
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            float s = (comp(a0, e) + comp(b0, e)) + (comp(a1, e) + comp(b1, e));
                            set_comp(acc[i], e, fmaf(ck, s, comp(acc[i], e)));
                        }
                    }
                }
                // dim 2 far terms from a (4 + 2A)-wide window of the centre row
#pragma unroll
                for (int i = 0; i < R1; ++i) {
                    float w[4 + 2 * C::A];
#pragma unroll
                    for (int j = 0; j < (4 + 2 * C::A) / 4; ++j) {
                        const float4 v = lds4(plane_p + 4 * ((r0 + i + H) * C::W2 + 4 * tz + 4 * j));
                        w[4 * j] = v.x;
                        w[4 * j + 1] = v.y;
                        w[4 * j + 2] = v.z;
                        w[4 * j + 3] = v.w;
                    }
                    const float4 u0 = Q[i][H];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        float a = comp(acc[i], e);
#pragma unroll
                        for (int k = H; k >= 2; --k)
                            a = fmaf(K.c[k], w[C::A + e - k] + w[C::A + e + k], a);
                        const float uc = comp(u0, e);
                        // k = 1 ring of all three axes in difference form
                        const float4 xm = Q[i][H - 1], xp = Q[i][H + 1];
                        float d1 = (comp(xm, e) - uc) + (comp(xp, e) - uc);
                        d1 += (w[C::A + e - 1] - uc) + (w[C::A + e + 1] - uc);
                        set_comp(acc[i], e, a);
                        // dim 1 k=1 handled below (needs the neighbour rows)
                        set_comp(acc[i], e, fmaf(K.c[1], d1, comp(acc[i], e)));
                    }
                    const float4 ym = lds4(plane_p + 4 * ((r0 + i + H - 1) * C::W2 + C::A + 4 * tz));
                    const float4 yp = lds4(plane_p + 4 * ((r0 + i + H + 1) * C::W2 + C::A + 4 * tz));
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float uc = comp(u0, e);
                        set_comp(acc[i], e,
                                 fmaf(K.c[1], (comp(ym, e) - uc) + (comp(yp, e) - uc), comp(acc[i], e)));
                    }
                }
                // ---- aux tiles: u[t-1], m, damp ----
                const unsigned sa = na % SA, pha = (na / SA) & 1u;
                mbar_wait(full_a + 8 * sa, pha);
                const unsigned aux = aring_s + sa * 3 * C::ATILE;
                float4 upv[R1], mv[R1], dv[R1];
#pragma unroll
                for (int i = 0; i < R1; ++i) {
                    const unsigned off = 4 * ((r0 + i) * kT2 + 4 * tz);
                    upv[i] = lds4(aux + off);
                    mv[i] = lds4(aux + C::ATILE + off);
                    dv[i] = lds4(aux + 2 * C::ATILE + off);
                }
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(empty_a + 8 * sa);
                    mbar_arrive(empty_u + 8 * sp);  // plane p is no longer needed
                }
                ++na;
                // ---- combine + fused epilogue ----
                const long long xoff = static_cast<long long>(p) * g.plane;
#pragma unroll
                for (int i = 0; i < R1; ++i) {
                    const int y = yt + r0 + i;
                    float4 out;
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float uc = comp(Q[i][H], e);
                        const float Lr = fmaf(K.R3, uc, comp(acc[i], e));
                        set_comp(out, e,
                                 combine_f32(Lr, uc, comp(upv[i], e), comp(mv[i], e), comp(dv[i], e),
                                             K.kap_hi, K.kap_lo, K.half_dt));
                    }
                    if (y < sc.y1) {
                        if (c.has_src && p == c.src_x && y == c.src_y &&
                            static_cast<unsigned>(c.src_z - zc) < 4u) {
                            const int e = c.src_z - zc;
                            set_comp(out, e, inject_source(comp(out, e), c.wavelet[c.step],
                                                           comp(mv[i], e), static_cast<double>(K.dt)));
                        }
                        const long long idx = xoff + static_cast<long long>(y) * g.P2 + zc;
                        const bool full = zc >= sc.z0 && zc + 3 < sc.z1;
                        const bool lo_m = p >= pr.lo_first && p < pr.lo_last;
                        const bool hi_m = p >= pr.hi_first && p < pr.hi_last;
                        if (full) {
                            *reinterpret_cast<float4*>(un + idx) = out;
                            if (lo_m)
                                *reinterpret_cast<float4*>(
                                    lo_peer + idx + static_cast<long long>(pr.lo_shift) * g.plane) = out;
                            if (hi_m)
                                *reinterpret_cast<float4*>(
                                    hi_peer + idx + static_cast<long long>(pr.hi_shift) * g.plane) = out;
                            mine = max(mine, max(max(abs_bits(out.x), abs_bits(out.y)),
                                                 max(abs_bits(out.z), abs_bits(out.w))));
                        } else {
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const int z = zc + e;
                                if (z >= sc.z0 && z < sc.z1) {
                                    const float v = comp(out, e);
                                    un[idx + e] = v;
                                    if (lo_m) lo_peer[idx + e + static_cast<long long>(pr.lo_shift) * g.plane] = v;
                                    if (hi_m) hi_peer[idx + e + static_cast<long long>(pr.hi_shift) * g.plane] = v;
                                    mine = max(mine, abs_bits(v));
                                }
                            }
                        }
                    }
                }
            }
        }
    }
    __syncwarp();
    block_max_commit(mine, c.smax + c.slot);
}

template <int H, int R1, int T1, int SU, int SA>
size_t smem_bytes() {
    using C = Cfg<H, R1, T1>;
    return static_cast<size_t>(SU) * C::UPLANE + static_cast<size_t>(SA) * 3 * C::ATILE +
           16 * (SU + SA);
}

// Variant table: (H, R1, T1, SU, SA) chosen per space order to fit 227 KB of smem.
#define SWB_TMA_VARIANTS(X)         \
    X(1, 2, 28, 4, 3)               \
    X(2, 2, 28, 5, 3)               \
    X(3, 2, 28, 6, 3)               \
    X(4, 2, 28, 7, 3)               \
    X(5, 2, 28, 8, 3)               \
    X(6, 2, 28, 9, 3)               \
    X(7, 2, 28, 10, 2)              \
    X(8, 2, 28, 11, 2)

using KernelFn = void (*)(Maps, Geo, Coef, Ctl, Peer, Sched);

struct Variant {
    int H, R1, T1, SU, SA;
    KernelFn fn;
    size_t smem;
    int threads;
};

#define SWB_VARIANT_ENTRY(h, r1, t1, su, sa) \
    {h, r1, t1, su, sa, k_tma<h, r1, t1, su, sa>, smem_bytes<h, r1, t1, su, sa>(), Cfg<h, r1, t1>::NTHREADS},

const Variant* find_variant(int H) {
    static const Variant table[] = {SWB_TMA_VARIANTS(SWB_VARIANT_ENTRY)};
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

TmaPlan tma_plan(int H, const Geo& g, int num_sms) {
    TmaPlan p{};
    p.ok = 0;
    p.H = H;
    const Variant* v = find_variant(H);
    if (!v) return p;
    p.T1 = v->T1;
    p.T2 = kT2;
    p.A = (H + 3) / 4 * 4;
    p.stages = v->SU;
    p.threads = v->threads;
    p.smem_bytes = static_cast<int>(v->smem);
    const int zs = g.z0 & ~3;
    p.zs = zs;
    p.tiles_y = ceil_div(g.y1 - g.y0, v->T1);
    p.tiles_z = ceil_div(g.z1 - zs, kT2);
    p.columns = p.tiles_y * p.tiles_z;
    const int np = g.x1 - g.x0;
    p.work = static_cast<long long>(p.columns) * np;
    if (np <= 0 || p.columns <= 0) return p;
    p.grid = static_cast<int>(std::min<long long>(num_sms, p.work));
    p.variant = 1000 + H;
    if (cudaFuncSetAttribute(v->fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(v->smem)) != cudaSuccess) {
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

cudaError_t launch_tma(const TmaPlan& plan, const void* maps, const Geo& g, const Coef& K,
                       const Ctl& c, const Peer& p, cudaStream_t s) {
    const Variant* v = find_variant(plan.H);
    if (!v || !plan.ok) return cudaErrorInvalidValue;
    Sched sc;
    sc.nyt = plan.tiles_y;
    sc.nzt = plan.tiles_z;
    sc.ncol = plan.columns;
    sc.np = g.x1 - g.x0;
    sc.work = plan.work;
    sc.y0 = g.y0;
    sc.y1 = g.y1;
    sc.z0 = g.z0;
    sc.z1 = g.z1;
    sc.zs = plan.zs;
    sc.x0 = g.x0;
    v->fn<<<plan.grid, v->threads, v->smem, s>>>(*static_cast<const Maps*>(maps), g, K, c, p, sc);
    return cudaGetLastError();
}

}  // namespace swb
