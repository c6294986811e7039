// Internal types shared by the runtime (runtime.cu) and the kernels (k_*.cu).
//
// HBM layout (per handle):
//   u       : 3 levels x [nl0][n1][P2] FP32, P2 = round_up(n2, 32) so every row starts
//             128 B aligned (TMA needs 16 B strides; coalesced 128 B rows).
//   m, damp : [nl0][n1][P2] FP32, same indexing as one u level.
//   nl0     : owned planes of the z-slab plus SO/2 ghost planes on each side that has a
//             neighbour (single GPU: nl0 = n0, no ghosts).
// Local plane j <-> global plane x = j + xg_off.
#pragma once
#include <cstdint>

namespace swb {

constexpr int kMaxH = 12;  // space orders 2..24

// Geometry of one step: where to read/write and which points to update.
struct Geo {
    float* lev[3];          // base of u level 0,1,2 (local plane 0)
    const float* m;
    const float* damp;
    long long plane;        // floats per plane = n1 * P2
    int P2;                 // row pitch (floats)
    int n1, n2;
    int x0, x1;             // local planes to update [x0, x1)
    int y0, y1;             // rows to update [y0, y1)   (= [H, n1-H))
    int z0, z1;             // cols to update [z0, z1)   (= [H, n2-H))
    int xg_off;             // global x = local x + xg_off
};

// Stencil constants (passed by value -> kernel-parameter constant bank).
struct Coef {
    float c[kMaxH + 1];     // float(c_k), k = 0..H  (signed; c_{-k} = c_k)
    float R;                // fp32(double(c0) + 2 double(c1)): residual of the k=1 difference form
    float h[3];             // float spacing
    float dt;
    double inv_h2[3];       // 1 / (double(h)^2)
    double R_d;             // double(c0) + 2 double(c1)
    double inv_dt2;         // 1 / (double(dt)^2)
    double half_inv_dt;     // 0.5 / double(dt)
    double inject;          // double(dt) * double(dt)   (source scale numerator)
    float R3;               // fp32(3 (c0 + 2 c1))  (isotropic residual)
    float R3f;              // fp32(3 (c0 + 2 sum_k>=1 c_k)) in double: residual of the full difference form
    float R3k[4];           // fp32(3 (c0 + 2 sum_{k<=d+1} c_k)): residual with the difference form for k <= d+1
    float kap_hi, kap_lo;   // (dt/h)^2 as an exact-ish float pair (isotropic)
    float half_dt;          // dt/2 (exact)
    int iso;                // h[0]==h[1]==h[2]
};

// Per-step control data (device pointers + the absolute step).
struct Ctl {
    const float* wavelet;   // device, indexed by absolute step
    int wavelet_len;
    int has_src;            // source owned by this handle
    int src_x, src_y, src_z;  // LOCAL coordinates of the source
    float src_m;              // m at the source point (the injection's dt^2 amp / m)
    unsigned* smax;         // [nt] per-step max|u| bits (atomicMax over non-negative floats)
    int step;               // absolute step
    int slot;               // index into smax / traces for this step
    unsigned long long* trace;  // optional per-CTA timestamps [gridDim][4] (SWB_TRACE), or null
    // Fused halo-exchange ordering (TMA kernel on linked z-slabs; all null/0 otherwise):
    // every CTA bumps sig_lo / sig_hi (counters in the neighbours' memory) once it has
    // finished the step, and a producer about to TMA-load a ghost plane first waits until
    // flags[0] (lower neighbour) / flags[1] (upper) reach need_lo / need_hi.
    unsigned long long* sig_lo;
    unsigned long long* sig_hi;
    const unsigned long long* flags;
    unsigned long long need_lo, need_hi;
    int ghost_lo_end;           // local planes < ghost_lo_end are lower ghosts (0: none)
    int ghost_hi_begin;         // local planes >= ghost_hi_begin are upper ghosts (INT_MAX: none)
    unsigned* err;              // set to 1 if a wait timed out
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Peer (halo) exchange: boundary planes written straight into neighbour ghosts.
struct Peer {
    float* lo_lev[3];       // lower neighbour's u levels (its local plane 0), or null
    float* hi_lev[3];       // upper neighbour's u levels, or null
    int lo_first, lo_last;  // my local planes [lo_first, lo_last) mirrored to the lower neighbour
    int lo_shift;           // neighbour local plane = my local plane + lo_shift
    int hi_first, hi_last;
    int hi_shift;
};

inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace swb
