// Exercise the drop-in executor exactly as a reference user calls exec::run:
//   make_wave_problem -> wave_equations -> lower -> optimize_all(dse) -> build_iet -> exec::run
// Usage: dropin_run <basic|aggressive> <n0> <n1> <n2> <so> <steps> <damp_max> <out.bin> [dt]
// Writes: int32 final_level, uint64 point_updates, float step_max_abs[steps], float levels[3][n].
// Exit codes: 0 ok, 3 exec::InstabilityError (prints the step), 1 other exception.
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "stencilc/executor.hpp"
#include "stencilc/pipeline.hpp"
#include "stencilc/wave_model.hpp"

using namespace stencilc;

int main(int argc, char** argv) {
    if (argc != 9 && argc != 10) {
        std::fprintf(stderr, "usage: %s dse n0 n1 n2 so steps damp_max out [dt]\n", argv[0]);
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
    try {
        auto p = exec::make_wave_problem(cfg);
        auto eqs = exec::wave_equations(p);
        auto cl = pipeline::lower(eqs.equations, eqs.targets, eqs.points);
        auto ocs = pipeline::optimize_all(cl, pipeline::parse_dse_level(argv[1]));
        auto iet = pipeline::build_iet(ocs, p.steps, p.time_order);
        exec::RunResult r = exec::run(iet, p, {});
        FILE* f = std::fopen(argv[8], "wb");
        int32_t fl = r.final_level;
        std::fwrite(&fl, 4, 1, f);
        std::fwrite(&r.point_updates, 8, 1, f);
        std::fwrite(r.step_max_abs.data(), 4, r.step_max_abs.size(), f);
        for (int l = 0; l < 3; ++l) {
            auto v = r.u.interior(l);
            std::fwrite(v.data(), 4, v.size(), f);
        }
        std::fclose(f);
        std::printf("ok wall=%.6f\n", r.wall_seconds);
    } catch (const exec::InstabilityError& e) {
        std::printf("instability step=%d\n", e.step());
        return 3;
    } catch (const std::exception& e) {
        std::printf("error %s\n", e.what());
        return 1;
    }
    return 0;
}
