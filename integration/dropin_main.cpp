// Exercise exec::run exactly as a reference user calls it:
//   make_wave_problem -> wave_equations -> lower -> optimize_all(dse) -> build_iet -> exec::run
// Linked against the drop-in executor (integration/_build/dropin_run, B200) or against the
// reference's own interpreter (oracle/_ref/ref_main, the checker).
//
// Usage: <exe> <basic|aggressive> <n0> <n1> <n2> <so> <steps> <damp_max> <out.bin|-> [dt]
//   out.bin receives: int32 final_level, uint64 point_updates, float step_max_abs[steps],
//   float levels[3][n] (Field::interior of each level); "-" writes nothing (timing runs).
// Environment (optional):
//   DROPIN_SRC=x,y,z        move the source point after make_wave_problem (a hand-edited problem)
//   DROPIN_BOUNDS=d,lo,hi   replace cluster 0's iteration range in dim d (a hand-edited tree)
//   DROPIN_CHECK_BOUNDS=1   RunOptions::check_bounds
//   DROPIN_ON_STEP=1        RunOptions::on_step callback that checks the levels it is shown
//   DROPIN_REPS=n           call exec::run n times (after one untimed call) and report the median
// stdout: "ok wall=<RunResult.wall_seconds> run=<seconds of the exec::run call> setup=<seconds of
//   problem + IET construction>" on success.
// Exit codes: 0 ok, 3 exec::InstabilityError ("instability step=<s>"), 4 std::out_of_range
// ("out_of_range <what>"), 1 other exception ("error <what>").
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "stencilc/executor.hpp"
#include "stencilc/pipeline.hpp"
#include "stencilc/wave_model.hpp"

using namespace stencilc;

int main(int argc, char** argv) {
    if (argc != 9 && argc != 10) {
        std::fprintf(stderr, "usage: %s dse n0 n1 n2 so steps damp_max out|- [dt]\n", argv[0]);
        return 2;
    }
    exec::WaveProblemConfig cfg;
    cfg.shape = {std::atoi(argv[2]), std::atoi(argv[3]), std::atoi(argv[4])};
    cfg.spacing = {10.0, 10.0, 10.0};
    cfg.space_order = std::atoi(argv[5]);
    cfg.steps = std::atoi(argv[6]);
    cfg.damp_max = std::atof(argv[7]);
    cfg.damp_width = 4;
    if (argc == 10) cfg.dt = std::atof(argv[9]);  // <= 0: the CFL step (the reference default)
    const std::string out = argv[8];
    try {
        using clk = std::chrono::steady_clock;
        const auto t0 = clk::now();
        auto p = exec::make_wave_problem(cfg);
        if (const char* s = std::getenv("DROPIN_SRC")) {
            int x, y, z;
            if (std::sscanf(s, "%d,%d,%d", &x, &y, &z) == 3 && p.source) p.source->point = {x, y, z};
        }
        auto eqs = exec::wave_equations(p);
        auto cl = pipeline::lower(eqs.equations, eqs.targets, eqs.points);
        auto ocs = pipeline::optimize_all(cl, pipeline::parse_dse_level(argv[1]));
        if (const char* b = std::getenv("DROPIN_BOUNDS")) {  // hand-edited iteration space of cluster 0
            int d, lo, hi;
            if (std::sscanf(b, "%d,%d,%d", &d, &lo, &hi) == 3 && !ocs.empty() && d >= 0 &&
                d < static_cast<int>(ocs[0].cluster.bounds.size()))
                ocs[0].cluster.bounds[static_cast<size_t>(d)] = {lo, hi};
        }
        auto iet = pipeline::build_iet(ocs, p.steps, p.time_order);
        exec::RunOptions opts;
        if (const char* cb = std::getenv("DROPIN_CHECK_BOUNDS")) opts.check_bounds = cb[0] == '1';
        // DROPIN_ON_STEP=1: a callback that checks what it is shown -- the newest level's max|u|
        // must be step_max_abs[step], and the level before it must be the previous step's newest
        std::vector<float> cb_max;
        std::vector<double> cb_sum;
        int cb_bad = -1;
        if (const char* os = std::getenv("DROPIN_ON_STEP"); os && os[0] == '1') {
            opts.on_step = [&](int step, const exec::Field& u, int newest) {
                auto stats = [&](int l, float& mx, double& sum) {
                    const float* d = u.level_data(l);
                    mx = 0.f;
                    sum = 0.0;
                    for (std::size_t i = 0; i < u.cells_per_level(); ++i) {
                        mx = std::max(mx, std::fabs(d[i]));
                        sum += d[i];
                    }
                };
                float mx, mp;
                double sm, sp;
                stats(newest, mx, sm);
                if (step > 0) {
                    stats((newest + 2) % 3, mp, sp);
                    if (sp != cb_sum.back() && cb_bad < 0) cb_bad = step;
                }
                cb_max.push_back(mx);
                cb_sum.push_back(sm);
            };
        }
        const double setup = std::chrono::duration<double>(clk::now() - t0).count();
        int reps = 1;
        if (const char* r = std::getenv("DROPIN_REPS")) reps = std::max(1, std::atoi(r));
        if (reps > 1) exec::run(iet, p, opts);  // untimed first call (process start-up costs)
        std::vector<double> runs;
        double wall = 0.0;
        exec::RunResult r = [&] {
            for (int i = 0;; ++i) {
                const auto a = clk::now();
                exec::RunResult res = exec::run(iet, p, opts);
                runs.push_back(std::chrono::duration<double>(clk::now() - a).count());
                wall = res.wall_seconds;
                if (i + 1 == reps) return res;
            }
        }();
        std::sort(runs.begin(), runs.end());
        if (out != "-") {
            FILE* f = std::fopen(out.c_str(), "wb");
            int32_t fl = r.final_level;
            std::fwrite(&fl, 4, 1, f);
            std::fwrite(&r.point_updates, 8, 1, f);
            std::fwrite(r.step_max_abs.data(), 4, r.step_max_abs.size(), f);
            for (int l = 0; l < 3; ++l) {
                auto v = r.u.interior(l);
                std::fwrite(v.data(), 4, v.size(), f);
            }
            std::fclose(f);
        }
        std::printf("ok wall=%.6f run=%.6f setup=%.6f point_updates=%llu\n", wall, runs[runs.size() / 2], setup,
                    static_cast<unsigned long long>(r.point_updates));
        if (opts.on_step) {
            for (std::size_t i = 0; i < r.step_max_abs.size() && cb_bad < 0; ++i)
                if (i >= cb_max.size() || cb_max[i] != r.step_max_abs[i]) cb_bad = static_cast<int>(i);
            std::printf("on_step %s %d\n", cb_bad < 0 ? "match" : "mismatch", cb_bad);
        }
    } catch (const exec::InstabilityError& e) {
        std::printf("instability step=%d\n", e.step());
        return 3;
    } catch (const std::out_of_range& e) {
        std::printf("out_of_range %s\n", e.what());
        return 4;
    } catch (const std::exception& e) {
        std::printf("error %s\n", e.what());
        return 1;
    }
    return 0;
}
