// The reference's code-generation path, retargeted: make_wave_problem -> wave_equations -> lower ->
// optimize_all(dse) -> outline_kernel per cluster (/root/reference/proj/src/opsgen.cpp:250-312),
// then BOTH the reference's OPS program (opsgen::emit_program, :371-614) and the B200 program
// (opsgen::b200::emit_program, integration/opsgen_b200.cpp) are written to <outdir>.
//
// Usage: opsgen_b200 <basic|aggressive> <n0> <n1> <n2> <so> <steps> <damp_max> <outdir> <name> [hetero]
//   hetero: a smooth heterogeneous velocity (1500..3000 m/s); <outdir>/<name>_m.f32 then holds
//   m_data() (the file both host programs read) and <outdir>/<name>_velocity.f32 the velocity.
// Environment: OPSGEN_TAMPER=1 widens kernel k0's iteration range by one plane before emission (a
//   hand-edited kernel list the B200 emitter must reject).
// Exit codes: 0 ok ("ok <basic|aggressive> <kernels file> <host file>"), 2 std::invalid_argument, 1 other.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "opsgen_b200.hpp"
#include "stencilc/opsgen.hpp"
#include "stencilc/pipeline.hpp"
#include "stencilc/wave_model.hpp"

using namespace stencilc;

static void write_file(const std::string& path, const std::string& text) {
    std::ofstream f(path, std::ios::binary);
    if (!f || !(f << text)) throw std::runtime_error("cannot write " + path);
}

int main(int argc, char** argv) {
    if (argc != 10 && argc != 11) {
        std::fprintf(stderr, "usage: %s dse n0 n1 n2 so steps damp_max outdir name [hetero]\n", argv[0]);
        return 1;
    }
    try {
        exec::WaveProblemConfig cfg;
        cfg.shape = {std::atoi(argv[2]), std::atoi(argv[3]), std::atoi(argv[4])};
        cfg.spacing = {10.0, 10.0, 10.0};
        cfg.space_order = std::atoi(argv[5]);
        cfg.steps = std::atoi(argv[6]);
        cfg.damp_max = std::atof(argv[7]);
        cfg.damp_width = 4;
        const std::string outdir = argv[8], name = argv[9];
        const bool hetero = argc == 11 && std::string(argv[10]) == "hetero";
        if (hetero) {
            const size_t n = static_cast<size_t>(cfg.shape[0]) * cfg.shape[1] * cfg.shape[2];
            cfg.velocity_field.resize(n);
            for (size_t i = 0; i < n; ++i) {
                const double x = static_cast<double>(i / (static_cast<size_t>(cfg.shape[1]) * cfg.shape[2])) / cfg.shape[0];
                cfg.velocity_field[i] = static_cast<float>(1500.0 + 1500.0 * (0.5 + 0.5 * std::sin(6.283185307179586 * x)));
            }
        }
        auto p = exec::make_wave_problem(cfg);
        auto eqs = exec::wave_equations(p);
        auto cl = pipeline::lower(eqs.equations, eqs.targets, eqs.points);
        auto ocs = pipeline::optimize_all(cl, pipeline::parse_dse_level(argv[1]));
        std::vector<opsgen::OpsKernel> kernels;
        for (size_t i = 0; i < ocs.size(); ++i) kernels.push_back(opsgen::outline_kernel(ocs[i], "k" + std::to_string(i)));
        if (std::getenv("OPSGEN_TAMPER")) kernels[0].iteration_range[0].hi += 1;
        // the reference's own OPS program, for comparison
        auto ops = opsgen::emit_program(kernels, p, name);
        write_file(outdir + "/ops_" + ops.kernels_file, ops.kernels_source);
        write_file(outdir + "/ops_" + ops.host_file, ops.host_source);
        // the B200 program
        auto b = opsgen::b200::emit_program(kernels, p, name);
        write_file(outdir + "/" + b.kernels_file, b.kernels_source);
        write_file(outdir + "/" + b.host_file, b.host_source);
        if (hetero) {
            const auto m = p.m_data();
            std::ofstream f(outdir + "/" + name + "_m.f32", std::ios::binary);
            f.write(reinterpret_cast<const char*>(m.data()), static_cast<std::streamsize>(m.size() * sizeof(float)));
            std::ofstream v(outdir + "/" + name + "_velocity.f32", std::ios::binary);
            v.write(reinterpret_cast<const char*>(p.velocity.data()),
                    static_cast<std::streamsize>(p.velocity.size() * sizeof(float)));
        }
        std::printf("ok %s %s %s\n",
                    opsgen::b200::classify_kernels(kernels, p) == pipeline::DseLevel::basic ? "basic" : "aggressive",
                    b.kernels_file.c_str(), b.host_file.c_str());
        return 0;
    } catch (const std::invalid_argument& e) {
        std::printf("invalid_argument %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::printf("error %s\n", e.what());
        return 1;
    }
}
