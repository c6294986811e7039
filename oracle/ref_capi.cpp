// ORACLE TEST INFRASTRUCTURE ONLY — never linked into, or called by, the product path.
//
// A thin extern "C" wrapper around the reference's OWN, unmodified sources
// (/root/reference/proj/src/{symbolic,pipeline,opsgen,reference_emit,executor,wave_model}.cpp,
// compiled in place by oracle/Makefile into oracle/_ref/libstencilc_ref.so).  It exists
// so that pytest (ctypes) and bench.py's `--impl reference` arm can drive the
// reference CPU path exactly as a reference user would:
//
//   make_wave_problem (src/wave_model.cpp:47-104)
//   -> wave_equations (src/wave_model.cpp:106-126)
//   -> pipeline::lower (src/pipeline.cpp:48-140)
//   -> pipeline::optimize_all(DseLevel) (src/pipeline.cpp:514-524)
//   -> pipeline::build_iet(ocs, steps, time_order) (src/pipeline.cpp:541-600)
//   -> exec::run / exec::reference_run (src/executor.cpp:610-613, 731-814)
//
// Receiver traces are sampled through the reference's only hook for it,
// RunOptions::on_step (include/stencilc/executor.hpp:78), at on-grid points.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "stencilc/executor.hpp"
#include "stencilc/opsgen.hpp"
#include "stencilc/pipeline.hpp"
#include "stencilc/wave_model.hpp"

using namespace stencilc;

extern "C" {

// Mirrors exec::WaveProblemConfig (include/stencilc/wave_model.hpp:41-56) for rank 1-3.
struct ref_config {
    int32_t rank;
    int32_t shape[3];
    double spacing[3];
    int32_t space_order;
    double dt;              // <= 0 -> cfl_dt
    int32_t steps;
    double velocity;
    const float* velocity_field;  // nullable, grid-sized
    double damp_max;
    int32_t damp_width;
    int32_t with_source;
    int32_t source_point[3];  // -1 -> grid centre default
    double source_frequency;
    const float* source_wavelet;  // nullable
    int32_t source_wavelet_len;
};

struct ref_run_out {
    float* levels;          // [3][n] grid-sized interior per level (nullable)
    float* step_max_abs;    // [steps] (nullable)
    float* rec_traces;      // [steps][n_rec] (nullable)
    double wall_seconds;
    uint64_t point_updates;
    int32_t final_level;
    int32_t bad_step;       // InstabilityError::step(), -1 if none
};

}  // extern "C"

namespace {

thread_local std::string g_err;

exec::WaveProblemConfig to_cfg(const ref_config* c) {
    exec::WaveProblemConfig cfg;
    size_t cells = 1;
    for (int d = 0; d < c->rank; ++d) {
        cfg.shape.push_back(c->shape[d]);
        cfg.spacing.push_back(c->spacing[d]);
        cells *= static_cast<size_t>(c->shape[d]);
    }
    cfg.space_order = c->space_order;
    cfg.time_order = 2;
    cfg.dt = c->dt;
    cfg.steps = c->steps;
    cfg.velocity = c->velocity;
    if (c->velocity_field) cfg.velocity_field.assign(c->velocity_field, c->velocity_field + cells);
    cfg.damp_max = c->damp_max;
    cfg.damp_width = c->damp_width;
    cfg.with_source = c->with_source != 0;
    if (c->source_point[0] >= 0)
        for (int d = 0; d < c->rank; ++d) cfg.source_point.push_back(c->source_point[d]);
    cfg.source_frequency = c->source_frequency;
    if (c->source_wavelet)
        cfg.source_wavelet.assign(c->source_wavelet, c->source_wavelet + c->source_wavelet_len);
    return cfg;
}

pipeline::IetNodePtr make_iet(const exec::WaveProblem& p, int dse) {
    auto eqs = exec::wave_equations(p);
    auto cl = pipeline::lower(eqs.equations, eqs.targets, eqs.points);
    auto ocs = pipeline::optimize_all(cl, dse ? pipeline::DseLevel::aggressive
                                              : pipeline::DseLevel::basic);
    return pipeline::build_iet(ocs, p.steps, p.time_order);
}

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// Problem-level facts the GPU path must reproduce bit-exactly: dt, wavelet,
// source point, m/damp fields, FD weights (as exact rationals), IET hashes and
// the reference's flop counts per form.
int ref_problem_info(const ref_config* c, float* dt, float* wavelet, float* m, float* damp,
                     int32_t* src_point, int64_t* w_num, int64_t* w_den,
                     uint64_t* hash_basic, uint64_t* hash_aggr, int64_t* flops_basic,
                     int64_t* flops_aggr) {
    try {
        auto p = exec::make_wave_problem(to_cfg(c));
        if (dt) *dt = p.dt;
        if (wavelet && p.source)
            std::memcpy(wavelet, p.source->wavelet.data(), sizeof(float) * p.steps);
        if (src_point && p.source)
            for (int d = 0; d < c->rank; ++d) src_point[d] = p.source->point[d];
        if (m) {
            auto v = p.m_data();
            std::memcpy(m, v.data(), sizeof(float) * v.size());
        }
        if (damp) {
            auto v = p.damp_data();
            std::memcpy(damp, v.data(), sizeof(float) * v.size());
        }
        if (w_num && w_den) {
            auto w = sym::fd_coefficients(2, c->space_order);
            for (size_t i = 0; i < w.size(); ++i) {
                w_num[i] = w[i].second.num();
                w_den[i] = w[i].second.den();
            }
        }
        auto eqs = exec::wave_equations(p);
        auto cl = pipeline::lower(eqs.equations, eqs.targets, eqs.points);
        auto ob = pipeline::optimize_all(cl, pipeline::DseLevel::basic);
        auto oa = pipeline::optimize_all(cl, pipeline::DseLevel::aggressive);
        if (hash_basic) *hash_basic = pipeline::iet_hash(pipeline::build_iet(ob, p.steps, 2));
        if (hash_aggr) *hash_aggr = pipeline::iet_hash(pipeline::build_iet(oa, p.steps, 2));
        if (flops_basic) *flops_basic = ob.empty() ? 0 : ob[0].flops;
        if (flops_aggr) *flops_aggr = oa.empty() ? 0 : oa[0].flops;
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, 1);
    } catch (const std::exception& e) {
        return fail(e, 2);
    }
}

// exec::run (serial_ref == 0) or exec::reference_run (serial_ref != 0) on the
// IET the reference builds for the problem at DSE level `dse` (0 basic, 1 aggressive).
// Return codes: 0 ok, 1 invalid_argument, 2 other error, 3 InstabilityError.
int ref_run(const ref_config* c, int dse, int threads, int serial_ref,
            const float* const* initial_u, int n_initial, int n_rec, const int32_t* rec,
            ref_run_out* out) {
    try {
        auto p = exec::make_wave_problem(to_cfg(c));
        auto iet = make_iet(p, dse);
        exec::RunOptions opt;
        opt.threads = threads;
        size_t cells = p.cell_count();
        if (initial_u && n_initial > 0) {
            std::vector<std::vector<float>> init;
            for (int l = 0; l < n_initial; ++l)
                init.emplace_back(initial_u[l], initial_u[l] + cells);
            opt.initial_u = std::move(init);
        }
        if (n_rec > 0 && out->rec_traces) {
            float* traces = out->rec_traces;
            int rank = c->rank;
            opt.on_step = [=](int step, const exec::Field& u, int newest) {
                for (int r = 0; r < n_rec; ++r) {
                    std::vector<int> pt(rec + r * rank, rec + (r + 1) * rank);
                    traces[static_cast<size_t>(step) * n_rec + r] = u.at(newest, pt);
                }
            };
        }
        out->bad_step = -1;
        exec::RunResult res = serial_ref ? exec::reference_run(iet, p, opt)
                                         : exec::run(iet, p, opt);
        if (out->levels)
            for (int l = 0; l < res.u.levels(); ++l) {
                auto v = res.u.interior(l);
                std::memcpy(out->levels + cells * l, v.data(), sizeof(float) * cells);
            }
        if (out->step_max_abs)
            std::memcpy(out->step_max_abs, res.step_max_abs.data(),
                        sizeof(float) * res.step_max_abs.size());
        out->wall_seconds = res.wall_seconds;
        out->point_updates = res.point_updates;
        out->final_level = res.final_level;
        return 0;
    } catch (const exec::InstabilityError& e) {
        out->bad_step = e.step();
        return fail(e, 3);
    } catch (const std::invalid_argument& e) {
        return fail(e, 1);
    } catch (const std::exception& e) {
        return fail(e, 2);
    }
}

// The reference's own emitted plain-C loop nest (src/reference_emit.cpp:133-232)
// for inspection of the interpreter's evaluation order.  Returns the needed size.
int64_t ref_emit_reference_c(const ref_config* c, int dse, char* buf, int64_t cap) {
    try {
        auto p = exec::make_wave_problem(to_cfg(c));
        auto s = opsgen::emit_reference_c(make_iet(p, dse), p, "acoustic");
        if (buf && cap > 0) {
            int64_t n = std::min<int64_t>(cap - 1, static_cast<int64_t>(s.size()));
            std::memcpy(buf, s.data(), static_cast<size_t>(n));
            buf[n] = 0;
        }
        return static_cast<int64_t>(s.size()) + 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int ref_omp_max_threads(void);

}  // extern "C"

#ifdef STENCILC_HAVE_OPENMP
#include <omp.h>
int ref_omp_max_threads(void) { return omp_get_max_threads(); }
#else
int ref_omp_max_threads(void) { return 1; }
#endif
