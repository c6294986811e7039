// One-thread-per-point stencil kernels (all three forms) and the small auxiliary kernels.
//
// The plain forms (basic DSE) are arithmetic-bound by design (3*SO+3 IEEE divisions per
// point, the paper's OI comparison, BASELINE config 3); the factorised "simple" variant is
// the kernel-choice baseline for the TMA 2.5D kernel in k_tma.cu.
#include <cuda_runtime.h>

#include <atomic>

#include "k_common.cuh"
#include "kernels.h"

namespace swb {

template <int H, int FORM>
__global__ void __launch_bounds__(128) k_simple(Geo g, Coef K, Ctl c, Peer p) {
    const int z = g.z0 + blockIdx.x * blockDim.x + threadIdx.x;
    const int y = g.y0 + blockIdx.y;
    const int x = g.x0 + blockIdx.z;
    const int lt = c.step % 3, ln = (c.step + 1) % 3, lp = (c.step + 2) % 3;
    const float* __restrict__ ut = pick3(g.lev[0], g.lev[1], g.lev[2], lt);
    const float* __restrict__ um = pick3(g.lev[0], g.lev[1], g.lev[2], lp);
    float* __restrict__ un = pick3(g.lev[0], g.lev[1], g.lev[2], ln);
    unsigned mine = 0u;
    if (z < g.z1) {
        const long long s0 = g.plane, s1 = g.P2;
        const long long i = x * s0 + y * s1 + z;
        const float u0 = ut[i], up = um[i], m = g.m[i], dmp = g.damp[i];
        float v;
        if constexpr (FORM == 1) {
            v = plain_f64_point<H>(ut, i, s0, s1, u0, up, m, dmp, K);
        } else if constexpr (FORM == 2) {
            v = plain_f32_point<H>(ut, i, s0, s1, u0, up, m, dmp, K);
        } else {
            const float sx = lap_axis<H>(K, u0, [&](int k) { return ut[i + k * s0]; });
            const float sy = lap_axis<H>(K, u0, [&](int k) { return ut[i + k * s1]; });
            const float sz = lap_axis<H>(K, u0, [&](int k) { return ut[i + k]; });
            if (FORM == 3 && K.iso) {
                const float Lr = fmaf(K.R3, u0, (sx + sy) + sz);
                v = combine_f32(Lr, u0, up, m, dmp, K.kap_hi, K.kap_lo, K.half_dt);
            } else {
                v = combine_f64(K, lap_total(K, sx, sy, sz, u0), u0, up, m, dmp);
            }
        }
        if (c.has_src && x == c.src_x && y == c.src_y && z == c.src_z)
            v = inject_source(v, c.wavelet[c.step], m, static_cast<double>(K.dt));
        un[i] = v;
        if (x >= p.lo_first && x < p.lo_last)
            pick3(p.lo_lev[0], p.lo_lev[1], p.lo_lev[2], ln)[(x + p.lo_shift) * s0 + y * s1 + z] = v;
        if (x >= p.hi_first && x < p.hi_last)
            pick3(p.hi_lev[0], p.hi_lev[1], p.hi_lev[2], ln)[(x + p.hi_shift) * s0 + y * s1 + z] = v;
        mine = abs_bits(v);
    }
    block_max_commit(mine, c.smax + c.slot);
}

template <int H>
static cudaError_t launch_simple_h(int form, const Geo& g, const Coef& K, const Ctl& c,
                                   const Peer& p, cudaStream_t s) {
    dim3 block(128);
    dim3 grid(ceil_div(g.z1 - g.z0, 128), g.y1 - g.y0, g.x1 - g.x0);
    if (grid.z == 0 || grid.y == 0) return cudaSuccess;
    switch (form) {
        case 1: k_simple<H, 1><<<grid, block, 0, s>>>(g, K, c, p); break;
        case 2: k_simple<H, 2><<<grid, block, 0, s>>>(g, K, c, p); break;
        case 3: k_simple<H, 3><<<grid, block, 0, s>>>(g, K, c, p); break;
        default: k_simple<H, 0><<<grid, block, 0, s>>>(g, K, c, p); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_simple(int H, int form, const Geo& g, const Coef& K, const Ctl& c,
                          const Peer& p, cudaStream_t s) {
    switch (H) {
        case 1: return launch_simple_h<1>(form, g, K, c, p, s);
        case 2: return launch_simple_h<2>(form, g, K, c, p, s);
        case 3: return launch_simple_h<3>(form, g, K, c, p, s);
        case 4: return launch_simple_h<4>(form, g, K, c, p, s);
        case 5: return launch_simple_h<5>(form, g, K, c, p, s);
        case 6: return launch_simple_h<6>(form, g, K, c, p, s);
        case 7: return launch_simple_h<7>(form, g, K, c, p, s);
        case 8: return launch_simple_h<8>(form, g, K, c, p, s);
        case 9: return launch_simple_h<9>(form, g, K, c, p, s);
        case 10: return launch_simple_h<10>(form, g, K, c, p, s);
        case 11: return launch_simple_h<11>(form, g, K, c, p, s);
        case 12: return launch_simple_h<12>(form, g, K, c, p, s);
        default: return cudaErrorInvalidValue;
    }
}

// ---- auxiliary kernels ---------------------------------------------------------------

// max|u| and non-finite detection over the cells of one level that the stencil never
// writes (the ring of width H inside the grid plus, for a slab, nothing else): these stay
// constant for the whole run, so the per-step whole-grid max of the reference
// (src/executor.cpp:526-544) is max(ring_max[level], max over the updated points).
__global__ void k_ring_max(const float* __restrict__ u, long long plane, int P2, int nx0, int nx1,
                           int n1, int n2, int x_in0, int x_in1, int y_in0, int y_in1, int z_in0,
                           int z_in1, unsigned* out) {
    // Reads the ring only (about 6 % of a 256^3 level at SO 8), as two flat index spaces with
    // independent loads: (B) every cell of the rows outside the interior in x or y, (A) the
    // z ends of the interior rows.
    unsigned mine = 0u;
    const int xi0 = max(x_in0, nx0), xi1 = max(min(x_in1, nx1), xi0);
    const int nxl = xi0 - nx0, nxo = nxl + (nx1 - xi1), nxi = xi1 - xi0;
    const int yi0 = min(y_in0, n1), yi1 = max(min(y_in1, n1), yi0);
    const int nyl = yi0, nyo = nyl + (n1 - yi1), nyi = yi1 - yi0;
    const int zlo = min(z_in0, n2), zhi = max(min(z_in1, n2), zlo), edge = zlo + (n2 - zhi);
    const long long rowsB = static_cast<long long>(nxo) * n1 + static_cast<long long>(nxi) * nyo;
    const long long totB = rowsB * n2, totA = static_cast<long long>(nxi) * nyi * edge;
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < totB + totA; t += stride) {
        int x, y, z;
        if (t < totB) {
            const long long r = t / n2;
            z = static_cast<int>(t % n2);
            if (r < static_cast<long long>(nxo) * n1) {
                const int i = static_cast<int>(r / n1);
                x = i < nxl ? nx0 + i : xi1 + (i - nxl);
                y = static_cast<int>(r % n1);
            } else {
                const long long r2 = r - static_cast<long long>(nxo) * n1;
                const int j = static_cast<int>(r2 % nyo);
                x = xi0 + static_cast<int>(r2 / nyo);
                y = j < nyl ? j : yi1 + (j - nyl);
            }
        } else {
            const long long t2 = t - totB;
            const long long r = t2 / edge;
            const int e = static_cast<int>(t2 % edge);
            x = xi0 + static_cast<int>(r / nyi);
            y = yi0 + static_cast<int>(r % nyi);
            z = e < zlo ? e : zhi + (e - zlo);
        }
        mine = max(mine, abs_bits(u[x * plane + static_cast<long long>(y) * P2 + z]));
    }
    block_max_commit(mine, out);
}

// Receiver sampling: u of the newest level at on-grid points, after injection — what the
// reference's on_step(step, u, newest) callback observes (src/executor.cpp:595-596).
__global__ void k_receivers(const float* __restrict__ un, const long long* __restrict__ idx, int n,
                            float* __restrict__ out) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) {
        const long long j = idx[r];
        out[r] = j >= 0 ? un[j] : 0.0f;
    }
}

// Receiver sampling through 8-corner stencils (on-grid receivers: one corner of weight 1, so the
// trace is exactly u; off-grid: trilinear weights).  Double accumulation in a fixed order, no
// FMA, so the result is bit-identical to the C oracle's restatement.  Corners not owned by this
// slab have index -1 (their partial sums are added across slabs by the caller).
__global__ void k_samplers(const float* __restrict__ un, const long long* __restrict__ idx,
                           const double* __restrict__ w, int n, float* __restrict__ out) {
    // Launched with programmatic stream serialization: wait for the stencil step (the previous
    // grid) to complete, and let the next step's stencil kernel start its prologue right away.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) {
        double v = 0.0;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const long long j = idx[8 * r + c];
            if (j >= 0) v = __dadd_rn(v, __dmul_rn(w[8 * r + c], static_cast<double>(un[j])));
        }
        out[r] = static_cast<float>(v);
    }
}

// Adjoint of the receiver sampling: spread each receiver's datum onto its corners with the
// weights w (trilinear weight / (m + damp dt/2), zero outside the update interior).
__global__ void k_inject(float* __restrict__ un, const long long* __restrict__ idx, const double* __restrict__ w,
                         int n, const float* __restrict__ data) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const double d = static_cast<double>(data[r]);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const long long j = idx[8 * r + c];
        const double wc = w[8 * r + c];
        if (j < 0 || wc == 0.0) continue;
        const double inc = __dmul_rn(wc, d);
        unsigned* a = reinterpret_cast<unsigned*>(un + j);
        unsigned old = *a, assumed;
        do {
            assumed = old;
            const float nv = static_cast<float>(__dadd_rn(static_cast<double>(__uint_as_float(assumed)), inc));
            old = atomicCAS(a, assumed, __float_as_uint(nv));
        } while (old != assumed);
    }
}

cudaError_t launch_inject(float* un, const long long* idx, const double* w, int n, const float* data,
                          cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    k_inject<<<ceil_div(n, 128), 128, 0, s>>>(un, idx, w, n, data);
    return cudaGetLastError();
}

// Receiver samples of up to three consecutive steps in one launch: the three u levels hold the
// outputs of the last three steps, so the per-step sampler launch (2-3 us at small grids, where
// the stencil step itself is ~6 us) is needed only every third step.  Row b of `out` (n floats)
// is sampled from lev[b]; the arithmetic per sample is k_samplers'.
struct SampleLevels {
    const float* lev[3];
};
__global__ void k_samplers_batch(const SampleLevels L, int nb, const long long* __restrict__ idx,
                                 const double* __restrict__ w, int n, float* __restrict__ out) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n * nb) {
        const int b = t / n, r = t - b * n;
        const float* un = b == 0 ? L.lev[0] : (b == 1 ? L.lev[1] : L.lev[2]);
        double v = 0.0;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const long long j = idx[8 * r + c];
            if (j >= 0) v = __dadd_rn(v, __dmul_rn(w[8 * r + c], static_cast<double>(un[j])));
        }
        out[t] = static_cast<float>(v);
    }
}

cudaError_t launch_samplers_batch(const float* const* lev, int nb, const long long* idx, const double* w, int n,
                                  float* out, cudaStream_t s) {
    if (n <= 0 || nb <= 0) return cudaSuccess;
    SampleLevels L{{lev[0], nb > 1 ? lev[1] : lev[0], nb > 2 ? lev[2] : lev[0]}};
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ceil_div(n * nb, 128));
    cfg.blockDim = dim3(128);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_samplers_batch, L, nb, idx, w, n, out);
}

cudaError_t launch_samplers(const float* un, const long long* idx, const double* w, int n, float* out,
                            cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ceil_div(n, 128));
    cfg.blockDim = dim3(128);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_samplers, un, idx, w, n, out);
}

// Halo-exchange ordering: spin until every linked neighbour has completed at least
// `need` steps (counters live in this handle's memory and are written by the neighbours).
// Bounded: after `timeout_ns` the kernel records an error instead of hanging the device.
__global__ void k_wait_flags(const volatile unsigned long long* flags, int mask,
                             unsigned long long need, unsigned long long timeout_ns,
                             unsigned* err) {
    if (threadIdx.x < 2 && ((mask >> threadIdx.x) & 1)) {
        unsigned long long t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        while (flags[threadIdx.x] < need) {
            __nanosleep(100);
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > timeout_ns) {
                atomicExch(err, 1u);
                break;
            }
        }
    }
    __syncthreads();
    __threadfence_system();
}

// Publish "I completed `done` steps" into each neighbour's flag slot (after the stencil
// kernel in stream order, so all peer stores of that step are complete and visible).
__global__ void k_signal_flags(unsigned long long* lo_flag, unsigned long long* hi_flag,
                               unsigned long long done) {
    __threadfence_system();
    if (threadIdx.x == 0) {
        if (lo_flag) atomicExch(lo_flag, done);
        if (hi_flag) atomicExch(hi_flag, done);
    }
    __threadfence_system();
}

int device_sm_count() {
    static std::atomic<int> cache[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64) {
        const int c = cache[dev].load(std::memory_order_relaxed);
        if (c > 0) return c;
    }
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
        cudaGetLastError();
        n = 1;
    }
    if (dev >= 0 && dev < 64) cache[dev].store(n, std::memory_order_relaxed);
    return n;
}

namespace {
// m = 1.0f / (c * c) as IEEE FP32 (the reference's host expression has no contraction: a
// product, then a division)
__global__ void k_m_from_velocity(float* __restrict__ m, long long n, int P2, int n2) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        if (static_cast<int>(i % P2) >= n2) continue;  // row padding stays 0
        const float c = m[i];
        m[i] = __fdiv_rn(1.0f, __fmul_rn(c, c));
    }
}

// damp_data: dist = cells to the nearest face (global coordinates), damp_max (1 - dist/width)
// for dist < width, else 0 (src/wave_model.cpp:25-45)
__global__ void k_damp_taper(float* __restrict__ damp, int nl0, int n1, int P2, int xg_off, int n0, int n2,
                             float damp_max, int width) {
    const long long n = static_cast<long long>(nl0) * n1 * P2;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int z = static_cast<int>(i % P2);
        const int y = static_cast<int>((i / P2) % n1);
        const int x = static_cast<int>(i / (static_cast<long long>(P2) * n1)) + xg_off;
        float v = 0.0f;
        if (z < n2) {
            const int dist = min(min(min(x, n0 - 1 - x), min(y, n1 - 1 - y)), min(z, n2 - 1 - z));
            if (dist < width)
                v = __fmul_rn(damp_max, __fsub_rn(1.0f, __fdiv_rn(static_cast<float>(dist), static_cast<float>(width))));
        }
        damp[i] = v;
    }
}
}  // namespace

cudaError_t launch_m_from_velocity(float* m, long long n, int P2, int n2, cudaStream_t s) {
    k_m_from_velocity<<<device_sm_count() * 8, 256, 0, s>>>(m, n, P2, n2);
    return cudaGetLastError();
}

cudaError_t launch_damp_taper(float* damp, int nl0, int n1, int P2, int xg_off, int n0, int gn1, int n2,
                              float damp_max, int width, cudaStream_t s) {
    (void)gn1;
    k_damp_taper<<<device_sm_count() * 8, 256, 0, s>>>(damp, nl0, n1, P2, xg_off, n0, n2, damp_max, width);
    return cudaGetLastError();
}

cudaError_t launch_ring_max(const float* u, long long plane, int P2, int nx0, int nx1, int n1,
                            int n2, int x_in0, int x_in1, int y_in0, int y_in1, int z_in0,
                            int z_in1, unsigned* out, cudaStream_t s) {
    if (nx1 <= nx0) return cudaSuccess;
    k_ring_max<<<device_sm_count() * 8, 256, 0, s>>>(u, plane, P2, nx0, nx1, n1, n2, x_in0, x_in1, y_in0, y_in1,
                                       z_in0, z_in1, out);
    return cudaGetLastError();
}

cudaError_t launch_receivers(const float* un, const long long* idx, int n, float* out,
                             cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    k_receivers<<<ceil_div(n, 128), 128, 0, s>>>(un, idx, n, out);
    return cudaGetLastError();
}

cudaError_t launch_wait_flags(const unsigned long long* flags, int mask,
                              unsigned long long need, unsigned* err, cudaStream_t s) {
    k_wait_flags<<<1, 32, 0, s>>>(flags, mask, need, 20000000000ull, err);
    return cudaGetLastError();
}

cudaError_t launch_signal_flags(unsigned long long* lo_flag, unsigned long long* hi_flag,
                                unsigned long long done, cudaStream_t s) {
    k_signal_flags<<<1, 32, 0, s>>>(lo_flag, hi_flag, done);
    return cudaGetLastError();
}

}  // namespace swb
