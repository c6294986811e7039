// K1 (smem-queue variant): TMA-staged 2.5D factorised stencil whose dim-0 neighbours are
// read from the shared-memory plane ring instead of a per-thread register queue.
//
// Why: the register queue of k_tma.cu costs 2H+1 float4 per thread row (72 registers at
// SO 8) and 64-128 register moves per plane.  Here the u ring keeps every plane from its
// arrival until the output plane H planes later no longer needs it (2H+1 resident planes +
// prefetch), so u(x+-k) for the dim-0 stencil are plain LDS.128 from neighbouring stages.
// u[t-1], m and damp are not staged in smem at all: each consumer thread streams its own
// float4s with LDG.128 (evict-first) two output planes ahead, in registers.  The freed
// registers and smem buy a taller tile (more consumer warps per SM).
//
// Same arithmetic and fused epilogue as k_tma.cu (see the header comment there).
#include <algorithm>
#include <cstdint>
#include <cstring>

#include "k_tma_common.cuh"

namespace swb {
namespace {
using namespace tma;

template <int H, int R1, int T1, int SU>
struct SqCfg {
    static constexpr int A = (H + 3) / 4 * 4;
    static constexpr int W2 = kT2 + 2 * A;
    static constexpr int ROWS = T1 + 2 * H;
    static constexpr int UPLANE = (ROWS * W2 * 4 + 127) / 128 * 128;
    static constexpr int NCW = (T1 / R1) * 16 / 32;
    static constexpr int NTHREADS = 32 * (NCW + 1);
    static constexpr size_t SMEM = static_cast<size_t>(SU) * UPLANE + 16 * SU;
    static_assert(SU >= 2 * H + 2, "ring must hold 2H+1 planes plus one in flight");
};

struct AuxRegs {
    float4 up[2], m[2], d[2];  // R1 <= 2
};

__device__ __forceinline__ float4 ldg_stream(const float* p) { return __ldcs(reinterpret_cast<const float4*>(p)); }

// Issue the aux loads (u[t-1], m, damp) of one output plane into registers.  idx_row[i] is
// the in-plane index of row i, clamped into the allocation for rows past the grid.
template <int R1>
__device__ __forceinline__ void load_aux(AuxRegs& a, const float* um_lvl, const Geo& g, long long xoff,
                                         const long long (&idx_row)[2], bool damp) {
#pragma unroll
    for (int i = 0; i < R1; ++i) {
        const long long idx = xoff + idx_row[i];
        a.up[i] = ldg_stream(um_lvl + idx);
        a.m[i] = ldg_stream(g.m + idx);
        a.d[i] = damp ? ldg_stream(g.damp + idx) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

// Stage index helpers (ring of SU stages, unsigned wrap trick: min(x, x - SU)).
template <int SU>
__device__ __forceinline__ unsigned stage_add(unsigned s, unsigned k) {
    const unsigned x = s + k;
    return min(x, x - SU);
}
template <int SU>
__device__ __forceinline__ unsigned stage_sub(unsigned s, unsigned k) {
    const unsigned x = s - k;
    return min(x, x + SU);
}

template <int H, int R1, int T1, int SU>
__device__ __forceinline__ void sq_output(const float* ring, unsigned sc, const AuxRegs& ax, bool has_damp,
                                          int p, const Item& it, unsigned& mine, float* un,
                                          float* lo_peer, float* hi_peer, const Geo& g, const Coef& K,
                                          const Ctl& c, const Peer& pr) {
    using C = SqCfg<H, R1, T1, SU>;
    constexpr int PL = C::UPLANE / 4;
    const float* pc = ring + sc * PL;
    float2 acc[R1][2];
#pragma unroll
    for (int i = 0; i < R1; ++i) {
        const float* rowc = pc + i * C::W2;
        float w[4 + 2 * C::A];
#pragma unroll
        for (int jj = 0; jj < (4 + 2 * C::A) / 4; ++jj) {
            const float4 v = *reinterpret_cast<const float4*>(rowc - C::A + 4 * jj);
            w[4 * jj] = v.x;
            w[4 * jj + 1] = v.y;
            w[4 * jj + 2] = v.z;
            w[4 * jj + 3] = v.w;
        }
        float2 al = splat(0.f), ah = splat(0.f);
#pragma unroll
        for (int k = H; k >= 2; --k) {
            const float2 ck = splat(K.c[k]);
            const float4 xm = *reinterpret_cast<const float4*>(ring + stage_sub<SU>(sc, k) * PL + i * C::W2);
            const float4 xp = *reinterpret_cast<const float4*>(ring + stage_add<SU>(sc, k) * PL + i * C::W2);
            const float4 ym = *reinterpret_cast<const float4*>(rowc - k * C::W2);
            const float4 yp = *reinterpret_cast<const float4*>(rowc + k * C::W2);
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
        const float4 u0 = make_float4(w[C::A], w[C::A + 1], w[C::A + 2], w[C::A + 3]);
        const float4 xm = *reinterpret_cast<const float4*>(ring + stage_sub<SU>(sc, 1) * PL + i * C::W2);
        const float4 xp = *reinterpret_cast<const float4*>(ring + stage_add<SU>(sc, 1) * PL + i * C::W2);
        const float4 ym = *reinterpret_cast<const float4*>(rowc - C::W2);
        const float4 yp = *reinterpret_cast<const float4*>(rowc + C::W2);
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
    // ---- combine ----
    const float2 R3 = splat(K.R3), khi = splat(K.kap_hi), klo = splat(K.kap_lo);
    float4 out[R1];
#pragma unroll
    for (int i = 0; i < R1; ++i) {
        const float4 u0 = *reinterpret_cast<const float4*>(pc + i * C::W2);
        float2 res[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const float2 ucv = h ? hi2(u0) : lo2(u0);
            const float2 um = h ? hi2(ax.up[i]) : lo2(ax.up[i]);
            const float2 m = h ? hi2(ax.m[i]) : lo2(ax.m[i]);
            const float2 Lr = fma2(R3, ucv, acc[i][h]);
            const float2 Lk = fma2(Lr, khi, mul2(Lr, klo));
            if (has_damp) {
                const float2 gg = mul2(h ? hi2(ax.d[i]) : lo2(ax.d[i]), splat(K.half_dt));
                const float2 num = fma2(sub2(m, gg), sub2(ucv, um), Lk);
                res[h] = add2(ucv, div2(num, add2(m, gg)));
            } else {
                // damp == 0: u+ = u + ((u - u-) + Lk / m)
                res[h] = add2(ucv, add2(sub2(ucv, um), div2(Lk, m)));
            }
        }
        out[i] = make_float4(res[0].x, res[0].y, res[1].x, res[1].y);
    }
    // ---- fused epilogue ----
    const long long xoff = static_cast<long long>(p) * g.plane + it.gcol;
    const bool lo_m = p >= pr.lo_first && p < pr.lo_last;
    const bool hi_m = p >= pr.hi_first && p < pr.hi_last;
    const bool src_plane = c.has_src && p == c.src_x;
    if (!(lo_m || hi_m || src_plane)) {
        // common path: plain stores (rows past the interior are skipped warp-uniformly)
#pragma unroll
        for (int i = 0; i < R1; ++i)
            if (it.rows_ok || it.yt + i < g.y1)
                store_row(un + xoff + static_cast<long long>(i) * g.P2, out[i], it.zmask, mine);
        return;
    }
#pragma unroll
    for (int i = 0; i < R1; ++i) {
        const int y = it.yt + i;
        float4 o = out[i];
        if (y >= g.y1) continue;
        if (src_plane && y == c.src_y && static_cast<unsigned>(c.src_z - it.zc) < 4u) {
            const int e = c.src_z - it.zc;
            set_comp(o, e, inject_source(comp(o, e), c.wavelet[c.step], comp(ax.m[i], e),
                                         static_cast<double>(K.dt)));
        }
        const long long idx = xoff + static_cast<long long>(i) * g.P2;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int z = it.zc + e;
            if (z >= g.z0 && z < g.z1) {
                const float v = comp(o, e);
                un[idx + e] = v;
                if (lo_m) lo_peer[idx + e + static_cast<long long>(pr.lo_shift) * g.plane] = v;
                if (hi_m) hi_peer[idx + e + static_cast<long long>(pr.hi_shift) * g.plane] = v;
                mine = max(mine, abs_bits(v));
            }
        }
    }
}

template <int H, int R1, int T1, int SU>
__global__ void __launch_bounds__(SqCfg<H, R1, T1, SU>::NTHREADS, 1)
    k_sq(const __grid_constant__ Maps maps, Geo g, Coef K, Ctl c, Peer pr, Sched sc) {
    using C = SqCfg<H, R1, T1, SU>;
    constexpr int PL = C::UPLANE / 4;
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SU * C::UPLANE);
    const unsigned full_u = smem_addr(bars), empty_u = full_u + 8 * SU;
    const unsigned ring_s = smem_addr(smem);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < SU; ++i) {
            mbar_init(full_u + 8 * i, 1);
            mbar_init(empty_u + 8 * i, 32 * C::NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    // Programmatic dependent launch: everything above overlapped the previous step's tail;
    // u[t], u[t-1] written by that step are only touched after this point.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int lt = c.step % 3, ln = (c.step + 1) % 3, lp = (c.step + 2) % 3;
    const int G = gridDim.x;
    const int nitems = sc.ncol * sc.nchunk;
    unsigned mine = 0u;

    if (warp == 0) {
        if (lane == 0) {  // ===== TMA producer: halo-padded u[t] planes =====
            const CUtensorMap* mu = &maps.u[lt];
            prefetch_map(mu);
            unsigned st = 0, ph = 0;
            for (int item = blockIdx.x; item < nitems; item += G) {
                const int col = item % sc.ncol, chunk = item / sc.ncol;
                const int xa = sc.x0 + static_cast<int>(static_cast<long long>(sc.np) * chunk / sc.nchunk);
                const int xb = sc.x0 + static_cast<int>(static_cast<long long>(sc.np) * (chunk + 1) / sc.nchunk);
                const int dir = (chunk & 1) ? 1 : -1;
                const int yt = sc.y0 + (col / sc.nzt) * T1;
                const int zt = sc.zs + (col % sc.nzt) * kT2;
                const int q0 = dir > 0 ? xa - H : xb - 1 + H;
                const int nq = xb - xa + 2 * H;
                for (int j = 0; j < nq; ++j) {
                    mbar_wait(empty_u + 8 * st, ph ^ 1u);
                    mbar_expect_tx(full_u + 8 * st, C::ROWS * C::W2 * 4);
                    tma_load3(ring_s + st * C::UPLANE, mu, zt - C::A, yt - H, q0 + dir * j, full_u + 8 * st);
                    ring_next<SU>(st, ph);
                }
            }
        }
    } else {  // ===== consumers =====
        const int ct = threadIdx.x - 32;
        const int tz = ct & 15, ty = ct >> 4;
        const int r0 = ty * R1;
        float* un = pick3(g.lev[0], g.lev[1], g.lev[2], ln);
        const float* um_lvl = pick3(g.lev[0], g.lev[1], g.lev[2], lp);
        float* lo_peer = pick3(pr.lo_lev[0], pr.lo_lev[1], pr.lo_lev[2], ln);
        float* hi_peer = pick3(pr.hi_lev[0], pr.hi_lev[1], pr.hi_lev[2], ln);
        const float* ring = reinterpret_cast<const float*>(smem) + (r0 + H) * C::W2 + C::A + 4 * tz;
        unsigned su = 0, pu = 0;  // next arrival's stage / phase
        for (int item = blockIdx.x; item < nitems; item += G) {
            const int col = item % sc.ncol, chunk = item / sc.ncol;
            Item it;
            it.xa = sc.x0 + static_cast<int>(static_cast<long long>(sc.np) * chunk / sc.nchunk);
            it.xb = sc.x0 + static_cast<int>(static_cast<long long>(sc.np) * (chunk + 1) / sc.nchunk);
            it.dir = (chunk & 1) ? 1 : -1;
            it.q0 = it.dir > 0 ? it.xa - H : it.xb - 1 + H;
            it.nq = it.xb - it.xa + 2 * H;
            it.yt = sc.y0 + (col / sc.nzt) * T1 + r0;
            const int zt = sc.zs + (col % sc.nzt) * kT2;
            it.zc = zt + 4 * tz;
            it.zfull = it.zc >= sc.z0 && it.zc + 3 < sc.z1;
            it.zmask = zmask_of(it.zc, sc.z0, sc.z1);
            it.rows_ok = it.yt + R1 - 1 < sc.y1;
            it.gcol = static_cast<long long>(it.yt) * g.P2 + it.zc;
            // aux loads: per-row in-plane index, clamped into the allocation for masked rows /
            // columns (their values are never stored)
            long long lrow[2];
            const int zl = min(it.zc, g.P2 - 4);
#pragma unroll
            for (int i = 0; i < 2; ++i) lrow[i] = static_cast<long long>(min(it.yt + i, g.n1 - 1)) * g.P2 + zl;
            // does any plane of this item carry damping? (warp vote over the item's flags)
            bool damp = true;
            if (sc.dflag) {
                const unsigned char* f = sc.dflag + static_cast<long long>(col) * sc.np + (it.xa - sc.x0);
                bool any = false;
                for (int x = lane; x < it.xb - it.xa; x += 32) any |= f[x] != 0;
                damp = __any_sync(0xffffffffu, any);
            }
            const int nout = it.xb - it.xa;
            const int p0 = it.dir > 0 ? it.xa : it.xb - 1;
            // warm-up: planes 0 .. 2H-1 of the item
            for (int j = 0; j < 2 * H; ++j) {
                mbar_wait(full_u + 8 * su, pu);
                ring_next<SU>(su, pu);
            }
            AuxRegs ax[2];
            load_aux<R1>(ax[0], um_lvl, g, static_cast<long long>(p0) * g.plane, lrow, damp);
            if (nout > 1)
                load_aux<R1>(ax[1], um_lvl, g, static_cast<long long>(p0 + it.dir) * g.plane, lrow, damp);
            // centre stage of output 0 = arrival H of this item
            unsigned sc_ = stage_sub<SU>(su, H);
#pragma unroll 1
            for (int o = 0; o < nout; o += 2) {
#pragma unroll
                for (int b = 0; b < 2; ++b) {
                    const int oo = o + b;
                    if (oo < nout) {
                        mbar_wait(full_u + 8 * su, pu);  // newest plane needed: centre + H
                        ring_next<SU>(su, pu);
                        const int p = p0 + it.dir * oo;
                        sq_output<H, R1, T1, SU>(ring, sc_, ax[b], damp, p, it, mine, un, lo_peer, hi_peer,
                                                 g, K, c, pr);
                        // the oldest plane (centre - H) is no longer needed by any output
                        mbar_arrive(empty_u + 8 * stage_sub<SU>(sc_, H));
                        sc_ = stage_add<SU>(sc_, 1);
                        if (oo + 2 < nout)
                            load_aux<R1>(ax[b], um_lvl, g, static_cast<long long>(p + 2 * it.dir) * g.plane,
                                         lrow, damp);
                    }
                }
            }
            // release the last 2H planes of the item
            for (int k = 2 * H; k >= 1; --k) mbar_arrive(empty_u + 8 * stage_sub<SU>(su, k));
        }
    }
    __syncwarp();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    block_max_commit(mine, c.smax + c.slot);
}

#define SWB_SQ_VARIANTS(X) \
    X(1, 2, 44, 6)          \
    X(2, 2, 44, 8)          \
    X(3, 2, 44, 10)         \
    X(4, 2, 44, 12)         \
    X(5, 2, 28, 14)         \
    X(6, 2, 28, 16)         \
    X(7, 2, 28, 17)         \
    X(8, 2, 20, 19)

using SqFn = void (*)(Maps, Geo, Coef, Ctl, Peer, Sched);
struct SqVariant {
    int H, R1, T1, SU;
    SqFn fn;
    size_t smem;
    int threads;
};
#define SWB_SQ_ENTRY(h, r1, t1, su) \
    {h, r1, t1, su, k_sq<h, r1, t1, su>, SqCfg<h, r1, t1, su>::SMEM, SqCfg<h, r1, t1, su>::NTHREADS},

const SqVariant* find_sq(int H) {
    static const SqVariant table[] = {SWB_SQ_VARIANTS(SWB_SQ_ENTRY)};
    for (const auto& v : table)
        if (v.H == H) return &v;
    return nullptr;
}

}  // namespace

bool sq_variant(int H, int* T1, int* threads, int* smem, const void** fn) {
    const SqVariant* v = find_sq(H);
    if (!v) return false;
    *T1 = v->T1;
    *threads = v->threads;
    *smem = static_cast<int>(v->smem);
    *fn = reinterpret_cast<const void*>(v->fn);
    return true;
}

cudaError_t launch_sq(const TmaPlan& plan, const void* maps, const Geo& g, const Coef& K, const Ctl& c,
                      const Peer& p, const void* sched, cudaStream_t s) {
    const SqVariant* v = find_sq(plan.H);
    if (!v) return cudaErrorInvalidValue;
    return launch_pdl(reinterpret_cast<const void*>(v->fn), plan.grid, v->threads, v->smem, s,
                      *static_cast<const Maps*>(maps), g, K, c, p, *static_cast<const Sched*>(sched));
}

}  // namespace swb
