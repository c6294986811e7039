"""B200-native acoustic wave-equation FD operator (hot path of arxiv/paper_1912_00695).

Drop-in for the reference's exec::run on the acoustic IET: the time-stepped 3-D damped
wave update with Ricker point injection, executed by hand-written sm_100a CUDA kernels
behind the C-ABI in include/swb.h.  See DESIGN.md.
"""
from .wave import (DseLevel, Field, InstabilityError, Operator, OutOfRangeError, RunOptions, RunResult,
                   SourceSpec, WaveProblem, WaveProblemConfig, cfl_dt, fd_coefficients,
                   form_for, make_wave_problem, parse_dse_level, ricker_amplitude,
                   ricker_wavelet, rounded_weights, run, write_snapshot, read_snapshot,
                   write_checkpoint)

__all__ = [
    "DseLevel", "Field", "InstabilityError", "Operator", "OutOfRangeError", "RunOptions", "RunResult",
    "SourceSpec", "WaveProblem", "WaveProblemConfig", "cfl_dt", "fd_coefficients", "form_for",
    "make_wave_problem", "parse_dse_level", "ricker_amplitude", "ricker_wavelet",
    "rounded_weights", "run", "write_snapshot", "read_snapshot", "write_checkpoint",
]
