// Kernel launchers (host-callable) implemented in k_simple.cu and k_tma.cu.
#pragma once
#include <cuda_runtime.h>

#include "swb_internal.h"

namespace swb {

// SMs of the current device (cached per device; grid sizing of the element-wise kernels).
int device_sm_count();

// Model fields on the device (bit-identical to WaveProblem::m_data / damp_data,
// src/wave_model.cpp:16-45): m <- 1.0f/(c*c) in place over a level-sized buffer holding the
// velocity (row padding stays 0); damp <- the boundary taper for local planes [0, nl0) at global
// plane offset xg_off of an n0 x n1 x n2 grid.
cudaError_t launch_m_from_velocity(float* m, long long n, int P2, int n2, cudaStream_t s);
cudaError_t launch_damp_taper(float* damp, int nl0, int n1, int P2, int xg_off, int n0, int gn1, int n2,
                              float damp_max, int width, cudaStream_t s);

// One-thread-per-point stencil step; form: 0 factorised, 1 plain FP64, 2 plain FP32.
cudaError_t launch_simple(int H, int form, const Geo& g, const Coef& K, const Ctl& c,
                          const Peer& p, cudaStream_t s);

// TMA 2.5D factorised stencil (k_tma.cu).  `plan` is produced by tma_plan().
struct TmaPlan {
    int ok;
    int H;
    int T1, T2;           // output tile rows (dim 1) and cols (dim 2)
    int yw;               // y-pencil warps of the variant (0 or 1)
    int A;                // dim-2 halo rounded up to a multiple of 4
    int stages;           // u-plane ring depth
    int threads;
    int smem_bytes;
    int tiles_y, tiles_z, columns;  // column tiles
    int zs;               // first (aligned) dim-2 column of tile 0
    int grid;             // persistent CTAs
    long long work;       // column tiles x planes
    int nchunk;           // dim-0 chunks per column
    const unsigned char* dflag;  // device [columns][planes] damp-tile-nonzero flags (or null)
    int variant;
    int num_sms;
};
// Host-side damp tile flags for a plan: flags[col * np + (x - x0)] = any damp != 0 in the tile.
void tma_damp_flags(const TmaPlan& plan, const Geo& g, const float* damp_host_local, int n1, int n2,
                    unsigned char* flags);
// Same flags computed on the device from the uploaded damp field.
cudaError_t tma_damp_flags_device(const TmaPlan& plan, const Geo& g, unsigned char* flags, cudaStream_t s);
TmaPlan tma_plan(int H, const Geo& g, int num_sms);
// In place: m -> B = 1/(m + g), damp -> A = (m - g)/(m + g), g = fl(damp * half_dt), computed in
// double and rounded once, to a neighbouring float chosen by a hash of the global cell index so
// that the rounding is unbiased over a medium (cells with m == 0, row padding, get 0; A = 1 exactly
// where g == 0).  For K1 handles only.  Buffer: [nl0][n1][P2], local plane 0 = global xg_off.
cudaError_t tma_update_coefs(float* m, float* damp, long long n, float half_dt, int P2, int n1, int n2, int xg_off,
                             cudaStream_t s);
// Encodes the tensor maps for the three u levels (once per handle).
constexpr int kTmaMapsBytes = 8 * 128;  // 8 CUtensorMaps
cudaError_t tma_make_maps(const TmaPlan& plan, const Geo& g, int nl0, void* maps /*kTmaMapsBytes*/);
cudaError_t launch_tma(const TmaPlan& plan, const void* maps, const Geo& g, const Coef& K,
                       const Ctl& c, const Peer& p, cudaStream_t s);
cudaError_t launch_ring_max(const float* u, long long plane, int P2, int nx0, int nx1, int n1,
                            int n2, int x_in0, int x_in1, int y_in0, int y_in1, int z_in0,
                            int z_in1, unsigned* out, cudaStream_t s);
cudaError_t launch_receivers(const float* un, const long long* idx, int n, float* out,
                             cudaStream_t s);
cudaError_t launch_samplers(const float* un, const long long* idx, const double* w, int n, float* out,
                            cudaStream_t s);
cudaError_t launch_samplers_batch(const float* const* lev, int nb, const long long* idx, const double* w, int n,
                                  float* out, cudaStream_t s);
// Adjoint receiver injection: un[idx] += w * data[r] (8 corners per receiver, one rounding of the
// double sum per corner, CAS loop so coinciding corners accumulate).
cudaError_t launch_inject(float* un, const long long* idx, const double* w, int n, const float* data,
                          cudaStream_t s);
cudaError_t launch_wait_flags(const unsigned long long* flags, int mask,
                              unsigned long long need, unsigned* err, cudaStream_t s);
cudaError_t launch_signal_flags(unsigned long long* lo_flag, unsigned long long* hi_flag,
                                unsigned long long done, cudaStream_t s);

}  // namespace swb
