/*
 * swb.h — C-ABI of the B200-native acoustic wave-equation operator
 *         (the drop-in boundary for the reference's hot path).
 *
 * The reference's hot path is the C++ call
 *     stencilc::exec::RunResult stencilc::exec::run(const pipeline::IetNodePtr& iet,
 *                                                   const WaveProblem& problem,
 *                                                   const RunOptions& options);
 *     (/root/reference/proj/include/stencilc/executor.hpp:90-91, src/executor.cpp:610-613)
 * which builds an Engine over halo-padded FP32 Fields (src/executor.cpp:28-88, 142-148),
 * steps the time loop (src/executor.cpp:546-606) and returns all three u levels plus
 * per-step max|u| (include/stencilc/executor.hpp:81-87).  Every entry point below replaces
 * one piece of that call; INTEGRATION.md shows the replacement exec::run that a maintainer
 * drops into the reference tree (it calls exactly these functions, in this order).
 *
 * Conventions
 *   - Grids are rank 3, C order: dim 0 = reference "x" (slowest), dim 2 = "z" (unit stride),
 *     as in Field (src/executor.cpp:32-37).  Host arrays are grid-sized (no halo), the
 *     layout of Field::interior()/fill_interior() (src/executor.cpp:56-88).
 *   - All pointers are borrowed for the duration of the call.  The library owns device
 *     memory, streams and CUDA graphs.  Calls on one handle are synchronous unless named
 *     *_async; a handle is not re-entrant (like the reference Engine).
 *   - Return codes: SWB_OK, SWB_EINVAL (the reference throws std::invalid_argument),
 *     SWB_ECUDA (device/driver failure), SWB_EUNSTABLE (the reference throws
 *     InstabilityError{step}, include/stencilc/executor.hpp:62-70), SWB_ERANGE (the reference
 *     throws std::out_of_range under RunOptions::check_bounds).  swb_last_error() gives
 *     the message of the last failing call on this thread.
 *   - There is no CPU fallback: without a usable sm_100 device swb_create fails with SWB_ECUDA.
 */
#ifndef SWB_H
#define SWB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SWB_OK 0
#define SWB_EINVAL 1
#define SWB_ECUDA 2
#define SWB_EUNSTABLE 3
#define SWB_ERANGE 4   /* RunOptions::check_bounds: an access leaves the allocation (std::out_of_range) */

/* Stencil form.  The reference has two IETs for the same problem (pipeline::DseLevel,
 * include/stencilc/pipeline.hpp:17; src/pipeline.cpp:467-512):
 *   basic      -> the solved update term by term, 3*SO+3 divisions per point.
 *   aggressive -> factorised/CSE form (its shipped version has a sign bug,
 *                 src/pipeline.cpp:246-248; we implement the corrected algebra).
 * SWB_FORM_FACTORISED : aggressive algebra, FP32 Laplacian (difference form on the k=1 ring).
 *                       The production kernel (TMA 2.5D, isotropic spacing, SO >= 2) combines in
 *                       FP32 with per-point coefficient fields B = 1/(m+g), A = (m-g)/(m+g),
 *                       g = damp dt/2 (computed once per handle in FP64, rounded once to a
 *                       neighbouring float chosen by a hash of the cell: unbiased):
 *                       u+ = u + A (u - u-) + B Lr (dt/h)^2.  Anisotropic spacing takes the
 *                       one-thread-per-point fallback with an FP64 final combine.
 * SWB_FORM_PLAIN_F64  : basic form evaluated exactly as the interpreter does (double,
 *                       same term order, one division per product, no FMA): bit-exact.
 * SWB_FORM_PLAIN_F32  : basic form in FP32 term by term (the paper's OPS kernel, src/opsgen.cpp:327-355).
 * SWB_FORM_FACTORISED_SIMPLE : FP32 Laplacian + FP64 combine, one thread per point, no TMA
 *                       (kernel-choice baseline).
 * SWB_FORM_FACTORISED_SIMPLE_F32C : same, with the all-FP32 combine of the TMA kernel. */
enum swb_form {
    SWB_FORM_FACTORISED = 0,
    SWB_FORM_PLAIN_F64 = 1,
    SWB_FORM_PLAIN_F32 = 2,
    SWB_FORM_FACTORISED_SIMPLE = 3,
    SWB_FORM_FACTORISED_SIMPLE_F32C = 4
};

/* Everything exec::run reads from WaveProblem + the IET (src/executor.cpp:189-199, 383-403,
 * 577-597) flattened to plain data. */
typedef struct swb_problem {
    int32_t shape[3];          /* Grid::shape()                                            */
    float spacing[3];          /* float(Grid::spacing()[d]) — bound as float (src/executor.cpp:193-194) */
    int32_t space_order;       /* even, 2..24 (GridFunction u space_order)                 */
    float dt;                  /* WaveProblem::dt                                          */
    const float* m;            /* grid-sized WaveProblem::m_data(); NULL = from velocity (below) */
    const float* damp;         /* grid-sized WaveProblem::damp_data(); NULL = from damp_max/width (below) */
    const float* weights;      /* space_order+1 floats float(c_k), k=-SO/2..SO/2, of
                                  fd_coefficients(2, SO) (src/executor.cpp:136-138); NULL = computed */
    int32_t has_source;        /* WaveProblem::source engaged                              */
    int32_t source[3];         /* SourceSpec::point                                        */
    const float* wavelet;      /* SourceSpec::wavelet, >= wavelet_len samples              */
    int32_t wavelet_len;
    int32_t n_receivers;       /* on-grid receivers (new; the reference samples via on_step) */
    const int32_t* receivers;  /* [n_receivers][3] grid coordinates                        */
    int32_t form;              /* enum swb_form                                            */
    int32_t time_block;        /* 1 (or 0): one launch per step.  The temporal-blocking kernel
                                  (2 steps per launch) was measured 0.53-0.74x of the single-step
                                  kernel on B200 and is retired; other values are SWB_EINVAL. */
    int32_t device;            /* CUDA device ordinal                                      */
    /* z-slab (reference dim 0) decomposition: this handle updates planes [slab_lo, slab_hi)
     * of the global grid; slab_hi <= 0 means the whole grid.  See swb_link_neighbours. */
    int32_t slab_lo;
    int32_t slab_hi;
    /* Off-grid receivers (new; Devito-style trilinear interpolation): physical coordinates
     * [n_coord_receivers][3] with grid index 0 at coordinate 0.  Their traces follow the
     * on-grid receivers' in rec_traces.  Value = sum over the 8 surrounding cells, in
     * (a,b,c) lexicographic order, of ((wx_a*wy_b)*wz_c)*u in double, w0 = 1-f, w1 = f. */
    int32_t n_coord_receivers;
    const double* coord_receivers;
    /* RunOptions::check_bounds (include/stencilc/executor.hpp:74; src/executor.cpp:233, 333,
     * 417-428): validate every access of the operator -- the stencil reach of the update interior,
     * the source point's u and m accesses, the receivers -- against the reference's padded
     * allocation (u padded by SO/2, m and damp by 1) before anything runs; the first access
     * outside fails with SWB_ERANGE and the interpreter's message ("access to u leaves the
     * allocation in x at step 0").  Without it, a source outside the update interior is
     * SWB_EINVAL. */
    int32_t check_bounds;
    /* Model fields computed on the device instead of uploaded (the reference computes them on the
     * host, src/wave_model.cpp:16-45; the device results are bit-identical):
     *   m == NULL:    velocity (grid-sized) is uploaded and m = 1.0f/(c*c) per cell (m_data);
     *   damp == NULL: damp_max > 0 and damp_width > 0 give the boundary taper
     *                 damp_max * (1 - dist/damp_width) within damp_width cells of a face
     *                 (damp_data); otherwise damp is zero. */
    const float* velocity;
    float damp_max;
    int32_t damp_width;
} swb_problem;

typedef struct swb_handle swb_handle;

typedef struct swb_stats {
    double device_ms;          /* CUDA-event time of the last apply's time loop            */
    uint64_t point_updates;    /* RunResult::point_updates accumulated by this handle      */
    uint64_t kernel_launches;  /* launches of this library's kernels in the last apply     */
    int32_t kernel_variant;    /* internal id of the stencil kernel chosen                 */
    int32_t launch_steps;      /* time steps per stencil launch (1)                        */
    /* linked z-slabs: neighbour device ordinals in this process's enumeration (-1: none, -2: not
     * visible to this process) and whether the halo exchange with
     * each neighbour is ordered inside the stencil kernel (1) or by wait/signal kernels (0) */
    int32_t peer_lo, peer_hi;
    int32_t fused_lo, fused_hi;
    int32_t grid;              /* persistent CTAs of the stencil launch (0: not the TMA kernel) */
} swb_stats;

/* Engine construction (src/executor.cpp:142-148, 383-403): validates the problem, allocates
 * the three u levels (zeroed, as Field's constructor does) plus m and damp in HBM, uploads
 * m/damp, selects the kernel. */
int swb_create(const swb_problem* problem, swb_handle** out);

/* RunOptions::initial_u[level] (src/executor.cpp:387-393): grid-sized host data. */
int swb_set_level(swb_handle* h, int level, const float* grid_sized);

/* Field::interior(level) (src/executor.cpp:56-71) of the current state. */
int swb_get_level(swb_handle* h, int level, float* grid_sized);

/* Field::level_data(level) filled in place (src/executor.cpp:28-44: halo-padded C-order levels):
 * the grid-sized level lands at offset `halo` in every dim of a (n0+2h) x (n1+2h) x (n2+2h)
 * host block; the padding is not touched.  One pitched copy, no host repacking. */
int swb_get_level_padded(swb_handle* h, int level, float* padded, int halo);

/* The time loop (src/executor.cpp:577-597) for steps step0 .. step0+nt-1; level rotation
 * (step+toff) mod 3 as in resolve_channels (src/executor.cpp:407-415).  Outputs (each
 * nullable): step_max_abs[nt] (max|u| of the newest level over the whole grid, NaN if any
 * cell is non-finite, src/executor.cpp:526-544), *first_bad_step (-1 if all finite; the
 * call then returns SWB_EUNSTABLE), rec_traces[nt][n_receivers] (u of the newest level at
 * each receiver after injection — what on_step sees).  wavelet[] is indexed by absolute
 * step.  Synchronous. */
int swb_apply(swb_handle* h, int step0, int nt, float* step_max_abs, int32_t* first_bad_step,
              float* rec_traces);

/* Adjoint operator (new; the reference has none -- PAPER.md:350 lists adjoint/RTM as future
 * work).  The forward map of swb_apply from the source wavelet w to the receiver traces d is
 * linear: D u[n+1] = (2M + dt^2 L) u[n] - E u[n-1] + S w[n], d[n] = R u[n+1] with
 * D = m + damp dt/2, E = m - damp dt/2, S = e_s dt^2/m_s.  Its transpose is the same stencil run
 * backwards in time: starting from zero, for k = nt..1
 *     z[k] = stencil(z[k+1], z[k+2]) + D^-1 R^T rec_data[k-1],
 *     src_trace[k-1] = dt^2 (m_s + g_s)/m_s * z[k][source],
 * with the handle's receivers (on-grid and trilinear) as injection points.  rec_data is
 * [nt][n_receivers + n_coord_receivers]; the handle's levels are overwritten (zeroed first).
 * Single-domain handles only.  step_max_abs / first_bad_step as in swb_apply (adjoint-step order).
 * Restated on the CPU by oracle/port/wave_port.c port_adjoint (tests/test_oracle_adjoint.py). */
int swb_apply_adjoint(swb_handle* h, int nt, const float* rec_data, float* src_trace, float* step_max_abs,
                      int32_t* first_bad_step);

/* swb_apply plus wavefield snapshots (the reference's route is
 * RunOptions::on_step + write_snapshot, src/executor.cpp:595-596, 816-837, which costs a full
 * synchronous download per step).  After every `every` steps the newest level is copied
 * device-to-device into a staging ring in HBM (the compute stream only waits for that copy,
 * and only before the step that would overwrite the level) and drained to snaps[i]
 * (grid-sized, reference interior layout; pinned memory for full PCIe speed) on a separate
 * copy stream, overlapping the following steps.  n_snaps must equal nt / every; snapshot i is
 * the state after step step0 + (i+1)*every - 1.  Other outputs as swb_apply.  Linked slabs of
 * one process driven from several threads need pinned snaps[] buffers: a pageable copy can
 * block its thread inside the driver while the other slabs still have steps to enqueue. */
int swb_apply_snapshots(swb_handle* h, int step0, int nt, int every, float* const* snaps, int n_snaps,
                        float* step_max_abs, int32_t* first_bad_step, float* rec_traces);

/* Asynchronous halves of swb_apply for callers that time on the device: enqueue the time
 * loop on the handle's stream, then collect the same outputs. */
int swb_apply_async(swb_handle* h, int step0, int nt);
int swb_collect(swb_handle* h, float* step_max_abs, int32_t* first_bad_step, float* rec_traces);

/* The handle's CUDA stream (cudaStream_t as void*), for event timing by the caller. */
void* swb_stream(swb_handle* h);

int swb_get_stats(swb_handle* h, swb_stats* out);

int swb_destroy(swb_handle* h);

const char* swb_last_error(void);

/* ---- multi-GPU z-slabs (new; the reference only emits ops_partition(""), src/opsgen.cpp:561) ----
 * One handle per GPU/process owns [slab_lo, slab_hi) plus SO/2 ghost planes per side for u.
 * swb_export_ghosts returns an opaque blob (cudaIpcMemHandle_t + offsets, <= 256 bytes)
 * that a neighbour passes to swb_link_neighbours; after linking, each step's boundary
 * planes are written straight into the neighbours' ghost planes by the stencil kernel
 * (peer stores over NVLink) and a per-step flag in peer memory orders the exchange. */
int swb_export_ghosts(swb_handle* h, void* blob, size_t* blob_len);
int swb_link_neighbours(swb_handle* h, const void* lower_blob, size_t lower_len,
                        const void* upper_blob, size_t upper_len);
/* Same, for two handles living in one process (single-process multi-slab, tests). */
int swb_link_local(swb_handle* lower, swb_handle* upper);

/* ---- model helpers (host; same results as the reference's wave_model.cpp) ---- */
/* fd_coefficients(2, so) as exact fractions, offsets -so/2..so/2 (src/fd_coefficients.cpp:40-83). */
int swb_fd_weights(int derivative_order, int space_order, int64_t* num, int64_t* den);
/* cfl_dt (src/wave_model.cpp:146-154) for a rank-r grid. */
double swb_cfl_dt(int rank, const double* spacing, double max_velocity, int space_order);
/* ricker_wavelet (src/wave_model.cpp:134-144). */
int swb_ricker_wavelet(double peak_frequency, double dt, int steps, float* out);
/* m_data (src/wave_model.cpp:16-23) and damp_data (src/wave_model.cpp:25-45), rank 3. */
int swb_m_data(const float* velocity, size_t n, float* m);
int swb_damp_data(const int32_t* shape, float damp_max, int damp_width, float* out);

/* Version / build info string. */
const char* swb_version(void);

/* Debug: with SWB_TRACE=1 in the environment at swb_create, copy the per-CTA globaltimer
 * stamps of the last K1 launch of an even and of an odd step: out[parity][cta][8] =
 * {entry, after griddepcontrol.wait, warm-up done, compute done, exit, SM id, 0, 0}
 * (out holds 2 * 8 * max_ctas values).  Returns the number of CTAs (or a negative error). */
int swb_debug_trace(swb_handle* h, unsigned long long* out, int max_ctas);

#ifdef __cplusplus
}
#endif
#endif /* SWB_H */
