// OPS-text retargeting for B200: the reference's code generator path (the Devito -> OPS
// translation of PAPER.md §2.3) emits an OPS host program whose time loop issues one
// ops_par_loop per outlined kernel (/root/reference/proj/src/opsgen.cpp:371-614, kernels from
// outline_kernel :250-312).  emit_program_b200 takes the SAME inputs -- the outlined kernels and
// the WaveProblem -- and emits a program with the same two-file shape that runs on a B200
// through this repo's C-ABI (include/swb.h) instead of the OPS runtime:
//
//   <name>_kernels.h   stencil descriptor of each outlined kernel: the OPS iteration range
//                      (exclusive upper bounds, as the OPS host's <kernel>_range), the stencil
//                      points of every argument (as its ops_decl_stencil), the FD weights
//                      float(c_k), the source wavelet (exact hex-float literals) and the form the
//                      kernels were recognised as;
//   <name>_host.c      swb_problem filled from the problem, swb_create, one swb_apply over the time
//                      loop (the stencil kernel and the point-source kernel of every step become one
//                      fused sm_100a launch), the result fetch of level steps % 3 and the same
//                      "max |u| = %g after N steps" line as the OPS host program; optional argv:
//                      device ordinal, and a path that receives the fetched level (float32).
//
// The kernels are recognised, not compiled: a B200 program runs precompiled sm_100a kernels, so
// each given kernel must equal (argument list, stencil points, temps, stores, iteration range) the
// kernel outline_kernel produces for this problem's own IET at DseLevel basic or aggressive --
// the same classification the drop-in exec::run makes with iet_hash (integration/executor_b200.cpp).
// Anything else throws std::invalid_argument (there is no OPS or CPU fallback).  basic maps to
// SWB_FORM_PLAIN_F64 (bit-exact with exec::run), aggressive to SWB_FORM_FACTORISED (the
// sign-corrected algebra; the reference's aggressive output is wrong).
#pragma once

#include <string>
#include <vector>

#include "stencilc/opsgen.hpp"
#include "stencilc/pipeline.hpp"
#include "stencilc/wave_model.hpp"

namespace stencilc::opsgen::b200 {

// Which canonical acoustic IET the kernels were outlined from.
pipeline::DseLevel classify_kernels(const std::vector<OpsKernel>& kernels, const exec::WaveProblem& problem);

// The retargeted program (same OpsProgram shape as opsgen::emit_program).
OpsProgram emit_program(const std::vector<OpsKernel>& kernels, const exec::WaveProblem& problem,
                        const std::string& name);

// The kernels opsgen would outline for this problem at `level`, named k0, k1, ... (cluster order:
// the stencil, then the point source) -- what a reference user passes to emit_program.
std::vector<OpsKernel> canonical_kernels(const exec::WaveProblem& problem, pipeline::DseLevel level);

}  // namespace stencilc::opsgen::b200
