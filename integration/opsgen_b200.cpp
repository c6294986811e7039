// OPS-text retargeting for B200 (see opsgen_b200.hpp).  Replaces, for this repo's operator, the
// OPS host-program emission of /root/reference/proj/src/opsgen.cpp:371-614: same inputs (outlined
// kernels + WaveProblem), same two-file output shape, a host program that calls include/swb.h.
#include "opsgen_b200.hpp"

#include <cmath>
#include <cstdio>
#include <sstream>
#include <stdexcept>

namespace stencilc::opsgen::b200 {
namespace {

const char* mode_name(AccessMode m) {
    switch (m) {
        case AccessMode::read: return "read";
        case AccessMode::write: return "write";
        case AccessMode::read_write: return "rw";
    }
    return "?";
}

// Everything that defines what an outlined kernel computes, except its name: argument list
// (dat, mode, stencil points), scalar parameters, per-point temps, stores, iteration range.
std::string fingerprint(const OpsKernel& k) {
    std::ostringstream os;
    for (const auto& a : k.ctx.args) {
        os << "arg " << a.dat_name << ' ' << mode_name(a.mode) << ' ' << a.time_offset << " pts";
        for (const auto& p : a.stencil_points) {
            os << " (";
            for (int o : p) os << o << ',';
            os << ')';
        }
        os << '\n';
    }
    for (const auto& s : k.ctx.scalar_params) os << "scalar " << s.name << '\n';
    for (const auto& b : k.point_temps) os << "temp " << b.temp->name << " = " << render_ops_expr(b.value, k.ctx) << '\n';
    for (const auto& a : k.stores)
        os << "store " << render_ops_expr(a.target, k.ctx) << " = " << render_ops_expr(a.update, k.ctx) << '\n';
    for (const auto& b : k.iteration_range) os << "range " << b.lo << ' ' << b.hi << '\n';
    return os.str();
}

std::string upper(std::string s) {
    for (auto& c : s) c = static_cast<char>(std::toupper(static_cast<unsigned char>(c)));
    return s;
}

// Exact float literal (C99 hex float), so the emitted program carries the problem's bits.
std::string hexf(float v) {
    char buf[48];
    std::snprintf(buf, sizeof buf, "%aF", static_cast<double>(v));
    return buf;
}

bool valid_ident(const std::string& s) {
    if (s.empty() || std::isdigit(static_cast<unsigned char>(s[0]))) return false;
    for (char c : s)
        if (!(std::isalnum(static_cast<unsigned char>(c)) || c == '_')) return false;
    return true;
}

}  // namespace

std::vector<OpsKernel> canonical_kernels(const exec::WaveProblem& problem, pipeline::DseLevel level) {
    auto eqs = exec::wave_equations(problem);
    auto cl = pipeline::lower(eqs.equations, eqs.targets, eqs.points);
    auto ocs = pipeline::optimize_all(cl, level);
    std::vector<OpsKernel> ks;
    for (size_t i = 0; i < ocs.size(); ++i) ks.push_back(outline_kernel(ocs[i], "k" + std::to_string(i)));
    return ks;
}

pipeline::DseLevel classify_kernels(const std::vector<OpsKernel>& kernels, const exec::WaveProblem& problem) {
    if (kernels.empty()) throw std::invalid_argument("emit_program_b200: need at least one kernel");
    for (const auto& k : kernels)
        if (k.stores.empty()) throw std::invalid_argument("emit_program_b200: kernel " + k.name + " has an empty body");
    if (!problem.grid || problem.grid->rank() != 3)
        throw std::invalid_argument("emit_program_b200: the B200 operator supports rank-3 grids");
    for (auto level : {pipeline::DseLevel::basic, pipeline::DseLevel::aggressive}) {
        const auto canon = canonical_kernels(problem, level);
        if (canon.size() != kernels.size()) continue;
        bool same = true;
        for (size_t i = 0; i < canon.size() && same; ++i) same = fingerprint(canon[i]) == fingerprint(kernels[i]);
        if (same) return level;
    }
    throw std::invalid_argument(
        "emit_program_b200: the kernels are not the acoustic wave operator of this problem at DseLevel basic or "
        "aggressive (the B200 program runs precompiled sm_100a kernels; there is no OPS fallback)");
}

OpsProgram emit_program(const std::vector<OpsKernel>& kernels, const exec::WaveProblem& problem,
                        const std::string& name) {
    if (!valid_ident(name)) throw std::invalid_argument("emit_program_b200: name must be a C identifier");
    const pipeline::DseLevel level = classify_kernels(kernels, problem);
    const sym::Grid& grid = *problem.grid;
    const int so = problem.space_order;
    const bool basic = level == pipeline::DseLevel::basic;
    const std::string N = upper(name);
    OpsProgram out;
    out.kernels_file = name + "_kernels.h";
    out.host_file = name + "_host.c";
    const std::size_t cells = problem.cell_count();

    // ---- stencil descriptors (what the OPS kernels file defined as user kernels) ----
    {
        std::ostringstream os;
        const std::string guard = N + "_KERNELS_H";
        os << "/* " << out.kernels_file << "\n"
           << " * Stencil descriptors of the " << name << " stencil program, retargeted from the OPS user\n"
           << " * kernels to the B200 operator library (include/swb.h).  Generated; do not edit.\n"
           << " *\n"
           << " * The OPS kernels were recognised as the acoustic wave operator at DseLevel "
           << (basic ? "basic" : "aggressive") << ":\n";
        for (size_t i = 0; i < kernels.size(); ++i) {
            const bool point = kernels[i].iteration_range.size() == 3 &&
                               kernels[i].iteration_range[0].lo == kernels[i].iteration_range[0].hi &&
                               kernels[i].iteration_range[1].lo == kernels[i].iteration_range[1].hi &&
                               kernels[i].iteration_range[2].lo == kernels[i].iteration_range[2].hi;
            os << " *   " << kernels[i].name << " ("
               << (point ? "point source" : "stencil") << ") -> "
               << (point ? "fused into the stencil launch's epilogue (two roundings, as exec::run)"
                         : (basic ? "SWB_FORM_PLAIN_F64 (bit-exact with exec::run)"
                                  : "SWB_FORM_FACTORISED (TMA 2.5D sm_100a kernel, sign-corrected algebra)"))
               << "\n";
        }
        os << " */\n"
           << "#ifndef " << guard << "\n#define " << guard << "\n\n"
           << "#define " << N << "_SPACE_ORDER " << so << "\n"
           << "#define " << N << "_STEPS " << problem.steps << "\n"
           << "#define " << N << "_FORM " << (basic ? "SWB_FORM_PLAIN_F64" : "SWB_FORM_FACTORISED") << "\n\n";
        os << "/* float(c_k) of fd_coefficients(2, " << so << "), k = -" << so / 2 << " .. " << so / 2 << " */\n"
           << "static const float " << name << "_weights[" << so + 1 << "] = {";
        int i = 0;
        for (const auto& [off, r] : sym::fd_coefficients(2, so))
            os << (i++ ? ", " : "") << hexf(static_cast<float>(r.to_double()));
        os << "};\n\n";
        for (const auto& k : kernels) {
            os << "/* " << k.name << ": iteration range (exclusive upper bounds) and stencil points per argument */\n"
               << "static const int " << name << "_" << k.name << "_range[6] = {";
            for (int d = 0; d < 3; ++d)
                os << (d ? ", " : "") << k.iteration_range[d].lo << ", " << k.iteration_range[d].hi + 1;
            os << "};\n";
            for (const auto& a : k.ctx.args) {
                os << "static const int " << name << "_" << k.name << "_" << a.dat_name << "_pts[] = {";
                bool first = true;
                for (const auto& p : a.stencil_points)
                    for (int o : p) {
                        os << (first ? "" : ", ") << o;
                        first = false;
                    }
                os << "};  /* " << a.stencil_points.size() << " points, " << mode_name(a.mode) << " */\n";
            }
        }
        if (problem.source) {
            const auto& w = problem.source->wavelet;
            os << "\n/* source wavelet (SourceSpec::wavelet, exact) */\n"
               << "static const int " << name << "_source[3] = {" << problem.source->point[0] << ", "
               << problem.source->point[1] << ", " << problem.source->point[2] << "};\n"
               << "static const float " << name << "_wavelet[" << w.size() << "] = {";
            for (size_t j = 0; j < w.size(); ++j) os << (j ? (j % 6 ? ", " : ",\n  ") : "\n  ") << hexf(w[j]);
            os << "};\n";
        }
        os << "\n#endif /* " << guard << " */\n";
        out.kernels_source = os.str();
    }

    // ---- host program (what the OPS host file did with ops_init .. ops_end) ----
    std::ostringstream os;
    bool uniform = true;
    for (float c : problem.velocity) uniform &= c == problem.velocity.front();
    os << "/* " << out.host_file << "\n"
       << " * B200 host program for the " << name << " stencil problem (retargeted from the OPS host\n"
       << " * program: one swb_apply over the time loop instead of one ops_par_loop per kernel and step).\n"
       << " * Generated; do not edit.\n"
       << " *   usage: " << name << "_host [device] [result.f32]\n"
       << " *   exit: 0 ok, 3 instability (non-finite field), 1 other error\n"
       << " */\n"
       << "#include <stdio.h>\n#include <stdlib.h>\n#include <string.h>\n#include <math.h>\n\n"
       << "#include \"swb.h\"\n"
       << "#include \"" << out.kernels_file << "\"\n\n"
       << "int main(int argc, const char **argv)\n{\n"
       << "  const int device = argc > 1 ? atoi(argv[1]) : 0;\n"
       << "  const char *result_path = argc > 2 ? argv[2] : NULL;\n"
       << "  const size_t cells = " << cells << "u;\n"
       << "  swb_problem p;\n"
       << "  memset(&p, 0, sizeof p);\n";
    for (int d = 0; d < 3; ++d)
        os << "  p.shape[" << d << "] = " << grid.shape()[d] << ";  p.spacing[" << d << "] = "
           << hexf(static_cast<float>(grid.spacing()[d])) << ";  /* " << grid.space_dims()[d].spacing_symbol
           << " */\n";
    os << "  p.space_order = " << N << "_SPACE_ORDER;\n"
       << "  p.dt = " << hexf(problem.dt) << ";  /* " << grid.time_dim().spacing_symbol << " */\n"
       << "  p.weights = " << name << "_weights;\n"
       << "  p.form = " << N << "_FORM;\n"
       << "  p.time_block = 1;\n"
       << "  p.device = device;\n";
    // coefficient fields: the OPS host filled m_data (uniform) or read <name>_m.f32; the B200
    // program uploads the velocity (the device computes m = 1.0f/(c*c), bit-identical to m_data)
    // or reads the same m file, and the device computes the damp taper (bit-identical to damp_data)
    os << "  float *field = (float *)malloc(cells * sizeof(float));\n"
       << "  if (!field) { fprintf(stderr, \"out of memory\\n\"); return 1; }\n";
    if (uniform) {
        os << "  for (size_t i = 0; i < cells; ++i)\n"
           << "    field[i] = " << hexf(problem.velocity.front()) << ";  /* velocity, m/s */\n"
           << "  p.velocity = field;\n";
    } else {
        os << "  {\n"
           << "    FILE *f = fopen(\"" << name << "_m.f32\", \"rb\");\n"
           << "    if (!f || fread(field, sizeof(float), cells, f) != cells) {\n"
           << "      fprintf(stderr, \"cannot read " << name << "_m.f32\\n\");\n"
           << "      return 1;\n"
           << "    }\n"
           << "    fclose(f);\n"
           << "  }\n"
           << "  p.m = field;\n";
    }
    os << "  p.damp_max = " << hexf(problem.damp_max) << ";\n"
       << "  p.damp_width = " << problem.damp_width << ";\n";
    if (problem.source) {
        os << "  p.has_source = 1;\n"
           << "  memcpy(p.source, " << name << "_source, sizeof p.source);\n"
           << "  p.wavelet = " << name << "_wavelet;\n"
           << "  p.wavelet_len = " << problem.source->wavelet.size() << ";\n";
    }
    os << "\n  swb_handle *h = NULL;\n"
       << "  if (swb_create(&p, &h) != SWB_OK) {\n"
       << "    fprintf(stderr, \"swb_create: %s\\n\", swb_last_error());\n"
       << "    return 1;\n"
       << "  }\n"
       << "  /* the time loop: " << kernels.size() << " OPS kernel(s) per step -> one fused launch per step */\n"
       << "  int32_t bad = -1;\n"
       << "  int rc = swb_apply(h, 0, " << N << "_STEPS, NULL, &bad, NULL);\n"
       << "  if (rc == SWB_EUNSTABLE) {\n"
       << "    fprintf(stderr, \"instability at step %d\\n\", (int)bad);\n"
       << "    swb_destroy(h);\n"
       << "    return 3;\n"
       << "  }\n"
       << "  if (rc != SWB_OK) {\n"
       << "    fprintf(stderr, \"swb_apply: %s\\n\", swb_last_error());\n"
       << "    swb_destroy(h);\n"
       << "    return 1;\n"
       << "  }\n\n"
       << "  /* result fetch: u_levels[" << problem.steps % 3 << "], as ops_dat_fetch_data */\n"
       << "  if (swb_get_level(h, " << problem.steps % 3 << ", field) != SWB_OK) {\n"
       << "    fprintf(stderr, \"swb_get_level: %s\\n\", swb_last_error());\n"
       << "    swb_destroy(h);\n"
       << "    return 1;\n"
       << "  }\n"
       << "  float u_max = 0.0F;\n"
       << "  for (size_t i = 0; i < cells; ++i) {\n"
       << "    float a = fabsf(field[i]);\n"
       << "    if (a > u_max) u_max = a;\n"
       << "  }\n"
       << "  printf(\"max |u| = %g after " << problem.steps << " steps\\n\", u_max);\n"
       << "  if (result_path) {\n"
       << "    FILE *f = fopen(result_path, \"wb\");\n"
       << "    if (!f || fwrite(field, sizeof(float), cells, f) != cells) {\n"
       << "      fprintf(stderr, \"cannot write %s\\n\", result_path);\n"
       << "      return 1;\n"
       << "    }\n"
       << "    fclose(f);\n"
       << "  }\n"
       << "  free(field);\n"
       << "  swb_destroy(h);\n"
       << "  return 0;\n"
       << "}\n";
    out.host_source = os.str();
    return out;
}

}  // namespace stencilc::opsgen::b200
