/* ORACLE TEST INFRASTRUCTURE ONLY — a CPU restatement of the reference's hot path,
 * used by tests/ (as the parity checker), __graft_entry__.smoke() (as the checker)
 * and bench.py (as the `cpu_baseline` / `--impl reference` arm when oracle/_ref is
 * not built).  It is never called by the product path.
 *
 * What it restates (reference = /root/reference/proj):
 *   - fd weights for d^2/dx^2        src/fd_coefficients.cpp:40-83 (closed form of the Taylor solve)
 *   - cfl_dt                         src/wave_model.cpp:146-154
 *   - ricker_amplitude / wavelet     src/wave_model.cpp:128-144
 *   - m_data / damp_data             src/wave_model.cpp:16-45
 *   - make_wave_problem validation   src/wave_model.cpp:47-104
 *   - the DseLevel::basic update exactly as exec::run evaluates it:
 *       solved form of wave_equations (src/wave_model.cpp:106-126, src/symbolic.cpp:542-621)
 *       canonical term order, one division per product, FP32-rounded literals in double
 *       (src/executor.cpp:136-138, 216-286, 430-468); interior bounds src/pipeline.cpp:79-88
 *   - source cluster after the interior cluster (src/pipeline.cpp:89-113, src/executor.cpp:583-586)
 *   - 3-level rotation and per-step max|u| / InstabilityError (src/executor.cpp:407-415, 526-597)
 * It is bit-identical to exec::run on the basic IET (checked in tests/test_oracle.py).
 * Compile with -ffp-contract=off: the interpreter performs every +,-,*,/ as a
 * separately rounded double operation (no FMA).
 */
#include <math.h>
#include <stdio.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct port_config {
    int32_t rank;                 /* must be 3 for the port */
    int32_t shape[3];
    double spacing[3];
    int32_t space_order;
    double dt;                    /* <= 0 -> cfl_dt */
    int32_t steps;
    double velocity;
    const float* velocity_field;  /* nullable */
    double damp_max;
    int32_t damp_width;
    int32_t with_source;
    int32_t source_point[3];      /* -1 -> centre */
    double source_frequency;
    const float* source_wavelet;  /* nullable */
    int32_t source_wavelet_len;
} port_config;

typedef struct port_run_out {
    float* levels;        /* [3][n] */
    float* step_max_abs;  /* [steps] */
    float* rec_traces;    /* [steps][n_rec] */
    double wall_seconds;
    uint64_t point_updates;
    int32_t final_level;
    int32_t bad_step;
} port_run_out;

static char g_err[256];
const char* port_last_error(void) { return g_err; }

static int64_t gcd64(int64_t a, int64_t b) {
    if (a < 0) a = -a;
    while (b) { int64_t t = a % b; a = b; b = t; }
    return a ? a : 1;
}

/* Exact central weights of d^2/dx^2, offsets -M..M, as reduced int64 fractions
 * (src/fd_coefficients.cpp:40-83; closed form, see oracle/shim/fd_coefficients_closed.cpp). */
int port_fd_weights(int so, int64_t* num, int64_t* den) {
    if (so < 2 || so % 2) return 1;
    int M = so / 2;
    int64_t pn = 1, pd = 1, sn = 0, sd = 1;
    for (int k = 1; k <= M; ++k) {
        pn *= (M - k + 1); pd *= (M + k);
        int64_t g = gcd64(pn, pd); pn /= g; pd /= g;
        int64_t cn = 2 * pn * ((k % 2) ? 1 : -1), cd = pd * (int64_t)k * k;
        g = gcd64(cn, cd); cn /= g; cd /= g;
        num[M + k] = num[M - k] = cn; den[M + k] = den[M - k] = cd;
        /* sum += c_k (128-bit intermediates; the reduced sum fits in int64 up to SO 24) */
        __int128 nn = (__int128)sn * cd + (__int128)cn * sd, dd = (__int128)sd * cd;
        __int128 a = nn < 0 ? -nn : nn, b = dd;
        while (b) { __int128 t = a % b; a = b; b = t; }
        if (a == 0) a = 1;
        sn = (int64_t)(nn / a); sd = (int64_t)(dd / a);
    }
    int64_t c0n = -2 * sn, c0d = sd, g = gcd64(c0n, c0d);
    num[M] = c0n / g; den[M] = c0d / g;
    return 0;
}

/* src/wave_model.cpp:146-154 */
double port_cfl_dt(const port_config* c, const float* velocity) {
    double min_h = c->spacing[0];
    for (int d = 1; d < c->rank; ++d) if (c->spacing[d] < min_h) min_h = c->spacing[d];
    size_t n = 1;
    for (int d = 0; d < c->rank; ++d) n *= (size_t)c->shape[d];
    double max_c = velocity[0];
    for (size_t i = 1; i < n; ++i) if (velocity[i] > max_c) max_c = velocity[i];
    double base = (min_h / max_c) / sqrt((double)c->rank) * 0.9;
    int64_t num[64], den[64];
    port_fd_weights(c->space_order, num, den);
    double sum = 0.0;
    for (int i = 0; i <= c->space_order; ++i) sum += fabs((double)num[i] / (double)den[i]);
    return base * (4.0 / sum);
}

/* src/wave_model.cpp:128-132 */
double port_ricker_amplitude(double f, double tau) {
    double a = 3.14159265358979323846 * f * tau;
    a *= a;
    return (1.0 - 2.0 * a) * exp(-a);
}

/* src/wave_model.cpp:134-144 */
void port_ricker_wavelet(double f, double dt, int steps, float* out) {
    double shift = 1.0 / f;
    for (int i = 0; i < steps; ++i) out[i] = (float)port_ricker_amplitude(f, i * dt - shift);
}

/* src/wave_model.cpp:16-23 */
void port_m_data(const float* vel, size_t n, float* m) {
    for (size_t i = 0; i < n; ++i) { float c = vel[i]; m[i] = 1.0f / (c * c); }
}

/* src/wave_model.cpp:25-45 */
void port_damp_data(const int32_t* shape, float damp_max, int width, float* out) {
    size_t n = (size_t)shape[0] * shape[1] * shape[2];
    memset(out, 0, n * sizeof(float));
    if (damp_max <= 0.0f || width <= 0) return;
    for (int x = 0; x < shape[0]; ++x)
        for (int y = 0; y < shape[1]; ++y)
            for (int z = 0; z < shape[2]; ++z) {
                int p[3] = {x, y, z};
                int dist = INT32_MAX;
                for (int d = 0; d < 3; ++d) {
                    if (p[d] < dist) dist = p[d];
                    if (shape[d] - 1 - p[d] < dist) dist = shape[d] - 1 - p[d];
                }
                if (dist < width)
                    out[((size_t)x * shape[1] + y) * shape[2] + z] =
                        damp_max * (1.0f - (float)dist / (float)width);
            }
}

typedef struct port_problem {
    int n0, n1, n2, so, H, steps;
    float dt;
    float h[3];
    float* m;
    float* damp;
    float* wavelet;  /* NULL when no source */
    int src[3];
    double coef[33]; /* |float(c_k)| widened, offsets -H..H */
    int neg[33];     /* sign of c_k */
    int unit[33];    /* |c_k| == 1: no literal multiply (src/executor.cpp:261) */
} port_problem;

static void port_free(port_problem* p) {
    free(p->m); free(p->damp); free(p->wavelet);
}

/* make_wave_problem (src/wave_model.cpp:47-104) restated for rank 3. */
static int port_make(const port_config* c, port_problem* p) {
    memset(p, 0, sizeof *p);
    if (c->rank != 3) { strcpy(g_err, "port oracle supports rank 3 only"); return 1; }
    if (c->space_order < 2 || c->space_order % 2) {
        strcpy(g_err, "space_order must be an even integer >= 2"); return 1; }
    if (c->space_order > 32) { strcpy(g_err, "space_order too large for the port"); return 1; }
    if (c->steps < 1) { strcpy(g_err, "steps must be >= 1"); return 1; }
    for (int d = 0; d < 3; ++d)
        if (c->shape[d] < 1 || !(c->spacing[d] > 0)) { strcpy(g_err, "bad grid"); return 1; }
    p->n0 = c->shape[0]; p->n1 = c->shape[1]; p->n2 = c->shape[2];
    p->so = c->space_order; p->steps = c->steps;
    p->H = p->so / 2 > 1 ? p->so / 2 : 1;  /* widest halo among u (so/2), m, damp (1) */
    size_t n = (size_t)p->n0 * p->n1 * p->n2;
    float* vel = (float*)malloc(n * sizeof(float));
    if (c->velocity_field) memcpy(vel, c->velocity_field, n * sizeof(float));
    else for (size_t i = 0; i < n; ++i) vel[i] = (float)c->velocity;
    for (size_t i = 0; i < n; ++i)
        if (!(vel[i] > 0.0f) || !isfinite(vel[i])) {
            free(vel); strcpy(g_err, "velocity must be positive and finite everywhere"); return 1; }
    p->m = (float*)malloc(n * sizeof(float));
    p->damp = (float*)malloc(n * sizeof(float));
    port_m_data(vel, n, p->m);
    port_damp_data(c->shape, (float)c->damp_max, c->damp_width, p->damp);
    p->dt = (float)(c->dt > 0.0 ? c->dt : port_cfl_dt(c, vel));
    free(vel);
    for (int d = 0; d < 3; ++d) p->h[d] = (float)c->spacing[d];
    int64_t num[65], den[65];
    port_fd_weights(p->so, num, den);
    int M = p->so / 2;
    for (int k = -M; k <= M; ++k) {
        double w = (double)num[M + k] / (double)den[M + k];
        double aw = fabs(w);
        p->coef[M + k] = (double)(float)aw;
        p->neg[M + k] = w < 0;
        p->unit[M + k] = (num[M + k] == den[M + k]) || (num[M + k] == -den[M + k]);
    }
    if (c->with_source) {
        for (int d = 0; d < 3; ++d)
            p->src[d] = c->source_point[0] >= 0 ? c->source_point[d] : c->shape[d] / 2;
        int hu = p->so / 2;
        for (int d = 0; d < 3; ++d)
            if (p->src[d] < hu || p->src[d] > c->shape[d] - 1 - hu) {
                port_free(p); strcpy(g_err, "source point must lie in the updatable interior"); return 1; }
        p->wavelet = (float*)malloc((size_t)p->steps * sizeof(float));
        if (c->source_wavelet) {
            if (c->source_wavelet_len < p->steps) {
                port_free(p); strcpy(g_err, "source wavelet shorter than the number of steps"); return 1; }
            memcpy(p->wavelet, c->source_wavelet, (size_t)p->steps * sizeof(float));
        } else {
            port_ricker_wavelet(c->source_frequency, p->dt, p->steps, p->wavelet);
        }
    }
    return 0;
}

int port_problem_info(const port_config* c, float* dt, float* wavelet, float* m, float* damp,
                      int32_t* src_point) {
    port_problem p;
    int rc = port_make(c, &p);
    if (rc) return rc;
    size_t n = (size_t)p.n0 * p.n1 * p.n2;
    if (dt) *dt = p.dt;
    if (wavelet && p.wavelet) memcpy(wavelet, p.wavelet, (size_t)p.steps * sizeof(float));
    if (m) memcpy(m, p.m, n * sizeof(float));
    if (damp) memcpy(damp, p.damp, n * sizeof(float));
    if (src_point) for (int d = 0; d < 3; ++d) src_point[d] = p.src[d];
    port_free(&p);
    return 0;
}

/* One interior point of the basic (solved, undistributed-by-DSE) update, term by term:
 *   2*m*u/(dt*dt*I) - m*u_prev/(dt*dt*I) + 1/2*damp*u_prev/(dt*I)
 *   + sum_d sum_k (+-)|c_k|*u[.. x_d+k ..]/(h_d*h_d*I),   I = m/(dt*dt) + 1/2*damp/dt
 * with the interpreter's grouping: ((c*a)*b)/((p*q)*r), left-to-right sums. */
static inline float point_update(const port_problem* p, const float* ut, const float* up,
                                 size_t idx, size_t s0, size_t s1, double m, double dmp) {
    const double dt = (double)p->dt;
    const double half = 0.5;
    double inner = m / (dt * dt) + (half * dmp) / dt;
    double acc = ((2.0 * m) * (double)ut[idx]) / ((dt * dt) * inner);
    acc = acc - (m * (double)up[idx]) / ((dt * dt) * inner);
    acc = acc + ((half * dmp) * (double)up[idx]) / (dt * inner);
    const int M = p->so / 2;
    const size_t stride[3] = {s0, s1, 1};
    for (int d = 0; d < 3; ++d) {
        const double hh = (double)p->h[d];
        const double den = (hh * hh) * inner;
        for (int k = -M; k <= M; ++k) {
            double v = (double)ut[(ptrdiff_t)idx + (ptrdiff_t)k * (ptrdiff_t)stride[d]];
            double t = p->unit[M + k] ? v : p->coef[M + k] * v;
            t = t / den;
            acc = p->neg[M + k] ? acc - t : acc + t;
        }
    }
    return (float)acc;
}

/* Trilinear receiver sampling restated for the off-grid receivers (an addition: the reference
 * samples only through on_step at grid points).  Index position g = X/h (h = float spacing
 * widened), i0 = floor(g) clamped to n-2, f = g - i0, weights w0 = 1-f, w1 = f; the value is
 * sum over corners (a,b,c) in lexicographic order of ((wx*wy)*wz)*u, in double, no FMA. */
static int crec_stencil(const port_problem* p, const double* X, size_t* idx, double* w) {
    const int n[3] = {p->n0, p->n1, p->n2};
    int i0[3];
    double f[3];
    for (int d = 0; d < 3; ++d) {
        double g = X[d] / (double)p->h[d];
        if (!(g >= 0.0) || g > (double)(n[d] - 1)) return 1;
        int i = (int)floor(g);
        if (i >= n[d] - 1) i = n[d] - 2;
        i0[d] = i;
        f[d] = g - (double)i;
    }
    int c = 0;
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
            for (int e = 0; e < 2; ++e, ++c) {
                double wa = a ? f[0] : 1.0 - f[0], wb = b ? f[1] : 1.0 - f[1], we = e ? f[2] : 1.0 - f[2];
                w[c] = (wa * wb) * we;
                idx[c] = ((size_t)(i0[0] + a) * n[1] + (size_t)(i0[1] + b)) * n[2] + (size_t)(i0[2] + e);
            }
    return 0;
}

int port_run2(const port_config* c, int threads, const float* const* initial_u, int n_initial,
              int n_rec, const int32_t* rec, int n_crec, const double* crec, float* crec_traces,
              port_run_out* out);

/* exec::run on the basic IET, restated.  levels: caller-owned [3][n]; initial_u optional. */
int port_run(const port_config* c, int threads, const float* const* initial_u, int n_initial,
             int n_rec, const int32_t* rec, port_run_out* out) {
    return port_run2(c, threads, initial_u, n_initial, n_rec, rec, 0, NULL, NULL, out);
}

int port_run2(const port_config* c, int threads, const float* const* initial_u, int n_initial,
              int n_rec, const int32_t* rec, int n_crec, const double* crec, float* crec_traces,
              port_run_out* out) {
    port_problem p;
    int rc = port_make(c, &p);
    if (rc) return rc;
    const int n0 = p.n0, n1 = p.n1, n2 = p.n2, H = p.H;
    const size_t n = (size_t)n0 * n1 * n2, s0 = (size_t)n1 * n2, s1 = (size_t)n2;
    for (int d = 0; d < 3; ++d)
        if (c->shape[d] - 1 - H < H) {
            port_free(&p); strcpy(g_err, "grid extent is too small for halo"); return 1; }
    size_t* cidx = NULL;
    double* cw = NULL;
    if (n_crec > 0) {
        cidx = (size_t*)malloc(sizeof(size_t) * 8 * (size_t)n_crec);
        cw = (double*)malloc(sizeof(double) * 8 * (size_t)n_crec);
        for (int r = 0; r < n_crec; ++r)
            if (crec_stencil(&p, crec + 3 * r, cidx + 8 * r, cw + 8 * r)) {
                free(cidx); free(cw); port_free(&p);
                snprintf(g_err, sizeof g_err, "receiver coordinate %d lies outside the grid", r);
                return 1;
            }
    }
    float* u = (float*)calloc(3 * n, sizeof(float));
    if (initial_u)
        for (int l = 0; l < n_initial && l < 3; ++l) memcpy(u + n * l, initial_u[l], n * sizeof(float));
    if (threads <= 0) {
#ifdef _OPENMP
        threads = omp_get_max_threads();
#else
        threads = 1;
#endif
    }
    const uint64_t interior = (uint64_t)(n0 - 2 * H) * (n1 - 2 * H) * (n2 - 2 * H);
    uint64_t updates = 0;
    out->bad_step = -1;
    double t0 = 0;
#ifdef _OPENMP
    t0 = omp_get_wtime();
#endif
    for (int step = 0; step < p.steps; ++step) {
        float* up1 = u + n * ((step + 1) % 3);
        const float* ut = u + n * (step % 3);
        const float* um = u + n * ((step + 2) % 3);
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(threads)
#endif
        for (int x = H; x <= n0 - 1 - H; ++x)
            for (int y = H; y <= n1 - 1 - H; ++y)
                for (int z = H; z <= n2 - 1 - H; ++z) {
                    size_t idx = (size_t)x * s0 + (size_t)y * s1 + (size_t)z;
                    up1[idx] = point_update(&p, ut, um, idx, s0, s1, (double)p.m[idx],
                                            (double)p.damp[idx]);
                }
        updates += interior;
        if (p.wavelet) {
            size_t si = (size_t)p.src[0] * s0 + (size_t)p.src[1] * s1 + (size_t)p.src[2];
            double dt = (double)p.dt;
            double inj = ((dt * dt) * (double)p.wavelet[step]) / (double)p.m[si];
            up1[si] = (float)((double)up1[si] + inj);
            updates += 1;
        }
        /* max_abs_interior over the whole grid of the newest level (src/executor.cpp:526-544) */
        float best = 0.0f;
        int finite = 1;
        for (size_t i = 0; i < n; ++i) {
            float v = up1[i];
            if (!isfinite(v)) finite = 0;
            float a = fabsf(v);
            if (a > best) best = a;
        }
        if (!finite) {
            out->bad_step = step;
            free(u); free(cidx); free(cw); port_free(&p);
            snprintf(g_err, sizeof g_err, "non-finite wave field at step %d (unstable dt?)", step);
            return 3;
        }
        if (out->step_max_abs) out->step_max_abs[step] = best;
        if (out->rec_traces)
            for (int r = 0; r < n_rec; ++r)
                out->rec_traces[(size_t)step * n_rec + r] =
                    up1[(size_t)rec[3 * r] * s0 + (size_t)rec[3 * r + 1] * s1 + (size_t)rec[3 * r + 2]];
        if (crec_traces)
            for (int r = 0; r < n_crec; ++r) {
                double v = 0.0;
                for (int k = 0; k < 8; ++k) v = v + cw[8 * r + k] * (double)up1[cidx[8 * r + k]];
                crec_traces[(size_t)step * n_crec + r] = (float)v;
            }
    }
    double t1 = 0;
#ifdef _OPENMP
    t1 = omp_get_wtime();
#endif
    if (out->levels) memcpy(out->levels, u, 3 * n * sizeof(float));
    out->wall_seconds = t1 - t0;
    out->point_updates = updates;
    out->final_level = p.steps % 3;
    free(u);
    free(cidx);
    free(cw);
    port_free(&p);
    return 0;
}

/* Adjoint of the forward operator above, restated (an addition: the reference has no adjoint;
 * PAPER.md:350 lists it as future work).  The forward map is w -> d with
 *   D u[n+1] = (2M + dt^2 L) u[n] - E u[n-1]  (+ S w[n] after the stencil),  d[n] = R u[n+1],
 * D = m + damp*dt/2, E = m - damp*dt/2, S = e_s dt^2/m_s, R = receiver sampling (on-grid or
 * trilinear).  L is symmetric on the interior (zero ring), so the transpose of the block
 * lower-triangular time-stepping system is the same recurrence run backwards in time:
 *   z[k] = stencil(z[k+1], z[k+2]) + D^{-1} R^T d[k-1],   (F^T d)[k-1] = (dt^2 (m_s+g_s)/m_s) z[k][s]
 * for k = nt .. 1 from z = 0.  R^T only reaches interior points: the ring of width SO/2 is never
 * written by the forward operator, so receivers (or trilinear corners) there have no adjoint.  Step s' = nt-k uses the forward level rotation; the stencil is the
 * basic form (point_update).  rec_data is [steps][n_rec + n_crec]; src_trace is [steps]. */
int port_adjoint(const port_config* c, int threads, int n_rec, const int32_t* rec, int n_crec,
                 const double* crec, const float* rec_data, float* src_trace) {
    port_problem p;
    int rc = port_make(c, &p);
    if (rc) return rc;
    const int n0 = p.n0, n1 = p.n1, n2 = p.n2, H = p.H;
    const size_t n = (size_t)n0 * n1 * n2, s0 = (size_t)n1 * n2, s1 = (size_t)n2;
    const int nr = n_rec + (n_crec > 0 ? n_crec : 0);
    if (!c->with_source) { port_free(&p); strcpy(g_err, "the adjoint samples at the source point"); return 1; }
    size_t* ridx = (size_t*)malloc(sizeof(size_t) * 8 * (size_t)(nr > 0 ? nr : 1));
    double* rw = (double*)malloc(sizeof(double) * 8 * (size_t)(nr > 0 ? nr : 1));
    int* ncorner = (int*)malloc(sizeof(int) * (size_t)(nr > 0 ? nr : 1));
    for (int r = 0; r < n_rec; ++r) {
        ridx[8 * r] = (size_t)rec[3 * r] * s0 + (size_t)rec[3 * r + 1] * s1 + (size_t)rec[3 * r + 2];
        rw[8 * r] = 1.0;
        ncorner[r] = 1;
    }
    for (int r = 0; r < n_crec; ++r) {
        if (crec_stencil(&p, crec + 3 * r, ridx + 8 * (n_rec + r), rw + 8 * (n_rec + r))) {
            free(ridx); free(rw); free(ncorner); port_free(&p);
            snprintf(g_err, sizeof g_err, "receiver coordinate %d lies outside the grid", r);
            return 1;
        }
        ncorner[n_rec + r] = 8;
    }
    if (threads <= 0) {
#ifdef _OPENMP
        threads = omp_get_max_threads();
#else
        threads = 1;
#endif
    }
    const double dt = (double)p.dt;
    const size_t si = (size_t)p.src[0] * s0 + (size_t)p.src[1] * s1 + (size_t)p.src[2];
    const double ws = ((dt * dt) * ((double)p.m[si] + 0.5 * (double)p.damp[si] * dt)) / (double)p.m[si];
    float* z = (float*)calloc(3 * n, sizeof(float));
    for (int sp = 0; sp < p.steps; ++sp) {
        const int k = p.steps - sp;
        float* zn = z + n * ((sp + 1) % 3);
        const float* zc = z + n * (sp % 3);
        const float* zp = z + n * ((sp + 2) % 3);
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(threads)
#endif
        for (int x = H; x <= n0 - 1 - H; ++x)
            for (int y = H; y <= n1 - 1 - H; ++y)
                for (int zz = H; zz <= n2 - 1 - H; ++zz) {
                    size_t idx = (size_t)x * s0 + (size_t)y * s1 + (size_t)zz;
                    zn[idx] = point_update(&p, zc, zp, idx, s0, s1, (double)p.m[idx], (double)p.damp[idx]);
                }
        const float* drow = rec_data + (size_t)(k - 1) * nr;
        for (int r = 0; r < nr; ++r)
            for (int q = 0; q < ncorner[r]; ++q) {
                const size_t j = ridx[8 * r + q];
                /* points outside the update interior are never written by the forward
                 * operator (the ring keeps its values), so they carry no adjoint */
                const int jx = (int)(j / s0), jy = (int)((j / s1) % (size_t)n1), jz = (int)(j % s1);
                if (jx < H || jx > n0 - 1 - H || jy < H || jy > n1 - 1 - H || jz < H || jz > n2 - 1 - H)
                    continue;
                const double den = (double)p.m[j] + 0.5 * (double)p.damp[j] * dt;
                zn[j] = (float)((double)zn[j] + (rw[8 * r + q] * (double)drow[r]) / den);
            }
        src_trace[k - 1] = (float)(ws * (double)zn[si]);
    }
    free(z); free(ridx); free(rw); free(ncorner);
    port_free(&p);
    return 0;
}

int port_omp_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
