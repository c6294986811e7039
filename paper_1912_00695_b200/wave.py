"""Python mirror of the reference operator API for the acoustic hot path.

Reference interface (C++, /root/reference/proj/include/stencilc):
  * WaveProblemConfig / WaveProblem / make_wave_problem / ricker_wavelet / cfl_dt
    (wave_model.hpp:14-85, src/wave_model.cpp)
  * Field / InstabilityError / RunOptions / RunResult / run / write_snapshot
    (executor.hpp:21-103, src/executor.cpp)
  * DseLevel basic|aggressive (pipeline.hpp:17)
Same names, argument meaning and error behaviour (ValueError where the reference throws
std::invalid_argument, InstabilityError(step) for a non-finite field).  Execution goes
through the C-ABI of libswb.so (include/swb.h) — there is no CPU path here.

Additions the reference lacks (north star): ``Operator(problem).apply(nt)`` with a step
offset, on-grid receivers, a choice of stencil form and z-slab multi-GPU handles.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import os
import time
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N


class DseLevel(enum.Enum):
    """pipeline::DseLevel (include/stencilc/pipeline.hpp:17)."""
    basic = "basic"
    aggressive = "aggressive"


def parse_dse_level(text: str) -> DseLevel:
    """pipeline::parse_dse_level (src/pipeline.cpp:20-24)."""
    if text == "basic":
        return DseLevel.basic
    if text == "aggressive":
        return DseLevel.aggressive
    raise ValueError(f"unknown dse level '{text}' (basic|aggressive)")


class InstabilityError(RuntimeError):
    """exec::InstabilityError (include/stencilc/executor.hpp:62-70)."""

    def __init__(self, step: int, what: str):
        super().__init__(what)
        self._step = step

    def step(self) -> int:
        return self._step


class OutOfRangeError(IndexError):
    """std::out_of_range of the interpreter's RunOptions::check_bounds (src/executor.cpp:417-428)."""


def _check(rc: int, step: int = -1) -> None:
    if rc == N.SWB_OK:
        return
    msg = N.last_error()
    if rc == N.SWB_EINVAL:
        raise ValueError(msg)
    if rc == N.SWB_ERANGE:
        raise OutOfRangeError(msg)
    if rc == N.SWB_EUNSTABLE:
        raise InstabilityError(step, msg)
    raise N.CudaError(msg)


# ---- model helpers (wave_model.cpp) ----------------------------------------------------

def fd_coefficients(derivative_order: int, accuracy_order: int) -> List[Tuple[int, Fraction]]:
    """sym::fd_coefficients (src/fd_coefficients.cpp:40-83): exact central weights."""
    if derivative_order < 1 or derivative_order > 2:
        raise ValueError("fd_coefficients: derivative order must be 1 or 2")
    if accuracy_order < 2 or accuracy_order % 2 != 0:
        raise ValueError("fd_coefficients: accuracy order must be even and >= 2")
    if accuracy_order > 24:
        raise ValueError("fd_coefficients: accuracy order above 24 is not supported")
    n = accuracy_order + 1
    num = (C.c_int64 * n)()
    den = (C.c_int64 * n)()
    _check(N.lib.swb_fd_weights(derivative_order, accuracy_order, num, den))
    half = accuracy_order // 2
    return [(j - half, Fraction(num[j], den[j])) for j in range(n)]


def rounded_weights(space_order: int) -> np.ndarray:
    """float(c_k) for k = -SO/2..SO/2, rounded like exec's rounded_const (src/executor.cpp:136-138)."""
    return np.array([np.float32(float(w.numerator) / float(w.denominator))
                     for _, w in fd_coefficients(2, space_order)], dtype=np.float32)


def ricker_amplitude(peak_frequency: float, tau: float) -> float:
    """src/wave_model.cpp:128-132."""
    a = math.pi * peak_frequency * tau
    a *= a
    return (1.0 - 2.0 * a) * math.exp(-a)


def ricker_wavelet(peak_frequency: float, dt: float, steps: int) -> np.ndarray:
    """src/wave_model.cpp:134-144 (computed by the C library for bit-identical exp())."""
    if not peak_frequency > 0.0:
        raise ValueError("ricker peak frequency must be positive")
    if not dt > 0.0:
        raise ValueError("ricker dt must be positive")
    out = np.zeros(max(int(steps), 0), np.float32)
    _check(N.lib.swb_ricker_wavelet(float(peak_frequency), float(dt), int(out.size), N.fptr(out)))
    return out


@dataclass
class SourceSpec:
    """exec::SourceSpec (include/stencilc/wave_model.hpp:14-18)."""
    point: List[int]
    wavelet: np.ndarray
    frequency: float = 0.0


@dataclass
class WaveProblemConfig:
    """exec::WaveProblemConfig (include/stencilc/wave_model.hpp:41-56)."""
    shape: Sequence[int]
    spacing: Sequence[float]
    space_order: int = 8
    time_order: int = 2
    dt: float = 0.0
    steps: int = 100
    velocity: float = 1500.0
    velocity_field: Optional[np.ndarray] = None
    damp_max: float = 0.0
    damp_width: int = 10
    with_source: bool = True
    source_point: Optional[Sequence[int]] = None
    source_frequency: float = 10.0
    source_wavelet: Optional[np.ndarray] = None


@dataclass
class WaveProblem:
    """exec::WaveProblem (include/stencilc/wave_model.hpp:20-39)."""
    shape: Tuple[int, int, int]
    spacing: Tuple[float, float, float]
    space_order: int
    time_order: int
    dt: np.float32
    steps: int
    velocity: np.ndarray
    damp_max: np.float32
    damp_width: int
    source: Optional[SourceSpec]

    def cell_count(self) -> int:
        return int(np.prod(self.shape))

    def halo(self) -> int:
        """GridFunction u halo = space_order/2 (include/stencilc/symbolic.hpp:64)."""
        return self.space_order // 2

    def m_data(self) -> np.ndarray:
        """1/velocity^2 per cell in FP32 (src/wave_model.cpp:16-23)."""
        v = np.ascontiguousarray(self.velocity, np.float32).reshape(-1)
        out = np.empty_like(v)
        _check(N.lib.swb_m_data(N.fptr(v), v.size, N.fptr(out)))
        return out.reshape(self.shape)

    def damp_data(self) -> np.ndarray:
        """Linear boundary taper (src/wave_model.cpp:25-45)."""
        out = np.empty(self.shape, np.float32)
        shp = (C.c_int32 * 3)(*self.shape)
        _check(N.lib.swb_damp_data(shp, C.c_float(float(self.damp_max)), int(self.damp_width),
                                   N.fptr(out)))
        return out


def cfl_dt(problem: WaveProblem) -> float:
    """src/wave_model.cpp:146-154."""
    sp = (C.c_double * 3)(*problem.spacing)
    return float(N.lib.swb_cfl_dt(3, sp, float(np.max(problem.velocity)), problem.space_order))


def make_wave_problem(config: WaveProblemConfig) -> WaveProblem:
    """exec::make_wave_problem (src/wave_model.cpp:47-104), rank-3 grids."""
    shape = tuple(int(s) for s in config.shape)
    spacing = tuple(float(h) for h in config.spacing)
    if len(shape) != 3 or len(spacing) != 3:
        raise ValueError("the B200 operator supports rank-3 grids (shape and spacing of length 3)")
    if any(s < 1 for s in shape):
        raise ValueError("grid shape must be positive")
    if any(not h > 0 for h in spacing):
        raise ValueError("grid spacing must be positive")
    if config.space_order < 2 or config.space_order % 2 != 0:
        raise ValueError("space_order must be an even integer >= 2")
    if config.time_order != 2:
        raise ValueError("time_order must be 2 for the second-order wave model")
    if config.steps < 1:
        raise ValueError("steps must be >= 1")
    damp_max = np.float32(config.damp_max)
    if damp_max < 0:
        raise ValueError("damp_max must be nonnegative")
    cells = int(np.prod(shape))
    if config.velocity_field is not None:
        vel = np.ascontiguousarray(config.velocity_field, np.float32).reshape(-1)
        if vel.size != cells:
            raise ValueError("velocity field size does not match the grid")
        vel = vel.reshape(shape)
    else:
        if not config.velocity > 0.0:
            raise ValueError("velocity must be positive")
        vel = np.full(shape, np.float32(config.velocity), np.float32)
    if not (np.all(vel > 0) and np.all(np.isfinite(vel))):
        raise ValueError("velocity must be positive and finite everywhere")
    p = WaveProblem(shape, spacing, int(config.space_order), 2, np.float32(0), int(config.steps),
                    vel, damp_max, int(config.damp_width), None)
    p.dt = np.float32(config.dt if config.dt > 0.0 else cfl_dt(p))
    if not p.dt > 0:
        raise ValueError("dt must be positive")
    if config.with_source:
        point = list(config.source_point) if config.source_point is not None else [s // 2 for s in shape]
        if len(point) != 3:
            raise ValueError("source point rank does not match the grid")
        halo = p.halo()
        for d in range(3):
            if point[d] < halo or point[d] > shape[d] - 1 - halo:
                raise ValueError("source point must lie in the updatable interior")
        if config.source_wavelet is not None:
            wav = np.ascontiguousarray(config.source_wavelet, np.float32).reshape(-1)
        else:
            wav = ricker_wavelet(config.source_frequency, float(p.dt), p.steps)
        if wav.size < p.steps:
            raise ValueError("source wavelet shorter than the number of steps")
        p.source = SourceSpec(point, wav, float(config.source_frequency))
    return p


# ---- executor types (executor.hpp) ----------------------------------------------------

class Field:
    """exec::Field (include/stencilc/executor.hpp:25-60) for u: 3 time levels of the grid.

    The reference stores halo-padded levels; the padded cells are never read or written by
    the operator, so this mirror keeps the grid-sized interiors and reports the reference's
    padded_shape/halo for API compatibility.
    """

    def __init__(self, problem: WaveProblem, levels: Optional[np.ndarray] = None):
        self._shape = tuple(problem.shape)
        self._halo = problem.halo()
        self._data = (np.zeros((3,) + self._shape, np.float32) if levels is None
                      else np.ascontiguousarray(levels, np.float32).reshape((3,) + self._shape))

    def levels(self) -> int:
        return 3

    def halo(self) -> int:
        return self._halo

    def padded_shape(self) -> List[int]:
        return [s + 2 * self._halo for s in self._shape]

    def at(self, level: int, point: Sequence[int]) -> float:
        return float(self._data[level][tuple(point)])

    def interior(self, level: int) -> np.ndarray:
        return self._data[level].reshape(-1).copy()

    def fill_interior(self, level: int, values: np.ndarray) -> None:
        v = np.asarray(values, np.float32).reshape(-1)
        if v.size != int(np.prod(self._shape)):
            raise ValueError("interior data size does not match the grid")
        self._data[level] = v.reshape(self._shape)

    @property
    def data(self) -> np.ndarray:
        """[3, n0, n1, n2] view of the three levels."""
        return self._data


@dataclass
class RunOptions:
    """exec::RunOptions (include/stencilc/executor.hpp:72-79).  ``threads`` is accepted for
    compatibility (the device decides the parallelism).  ``check_bounds`` validates every access
    of the operator against the reference's padded allocation before stepping and raises
    OutOfRangeError (std::out_of_range) with the interpreter's message at the first one outside
    (only a source point moved after make_wave_problem can get there)."""
    threads: int = 1
    check_bounds: bool = False
    initial_u: Optional[Sequence[np.ndarray]] = None
    on_step: Optional[Callable[[int, Field, int], None]] = None


@dataclass
class RunResult:
    """exec::RunResult (include/stencilc/executor.hpp:81-87) plus receiver traces."""
    u: Field
    step_max_abs: np.ndarray
    wall_seconds: float = 0.0
    point_updates: int = 0
    final_level: int = 0
    rec_traces: Optional[np.ndarray] = None
    device_seconds: float = 0.0


_FORMS = {"factorised": N.FORM_FACTORISED, "plain_f64": N.FORM_PLAIN_F64,
          "plain_f32": N.FORM_PLAIN_F32, "factorised_simple": N.FORM_FACTORISED_SIMPLE,
          "factorised_simple_f32c": N.FORM_FACTORISED_SIMPLE_F32C}


def form_for(dse: DseLevel) -> str:
    """basic IET -> bit-exact plain FP64 kernel; aggressive IET -> factorised TMA kernel."""
    return "plain_f64" if dse == DseLevel.basic else "factorised"


class Operator:
    """The time-stepped acoustic operator on one B200 (or one z-slab of it).

    ``Operator(problem).apply(nt)`` runs nt steps from the current state, like
    exec::run's time loop (src/executor.cpp:577-597) but resumable (``step0``).
    """

    def __init__(self, problem: WaveProblem, dse: DseLevel = DseLevel.aggressive, *,
                 form: Optional[str] = None, receivers: Optional[np.ndarray] = None,
                 receiver_coords: Optional[np.ndarray] = None,
                 device: int = 0, time_block: int = 1,
                 slab: Optional[Tuple[int, int]] = None,
                 m: Optional[np.ndarray] = None, damp: Optional[np.ndarray] = None,
                 check_bounds: bool = False):
        self.problem = problem
        self.form = form or form_for(dse)
        if self.form not in _FORMS:
            raise ValueError(f"unknown stencil form '{self.form}'")
        self._keep = []
        p = N.SwbProblem()
        for d in range(3):
            p.shape[d] = problem.shape[d]
            p.spacing[d] = np.float32(problem.spacing[d])
        p.space_order = problem.space_order
        p.dt = float(problem.dt)
        # m / damp may be passed precomputed (e.g. pinned host buffers); they must equal
        # problem.m_data() / problem.damp_data().  Otherwise the device computes them from the
        # velocity and the taper parameters (bit-identical; swb.h swb_problem.velocity).
        w = rounded_weights(problem.space_order)
        self._keep.append(w)
        if m is None:
            vel = np.ascontiguousarray(problem.velocity, np.float32)
            if vel.size != problem.cell_count():
                raise ValueError("velocity size does not match the grid")
            self._keep.append(vel)
            p.m = N.fptr(None)
            p.velocity = N.fptr(vel)
        else:
            m = np.ascontiguousarray(m, np.float32)
            if m.size != problem.cell_count():
                raise ValueError("m size does not match the grid")
            self._keep.append(m)
            p.m = N.fptr(m)
        p.damp_max = float(problem.damp_max)
        p.damp_width = int(problem.damp_width)
        if damp is None or float(problem.damp_max) == 0.0:
            # NULL: the taper on the device (zero without a layer, src/wave_model.cpp:29) --
            # nothing crosses PCIe for it
            p.damp = N.fptr(None)
        else:
            damp = np.ascontiguousarray(damp, np.float32)
            if damp.size != problem.cell_count():
                raise ValueError("damp size does not match the grid")
            self._keep.append(damp)
            p.damp = N.fptr(damp)
        p.weights = N.fptr(w)
        if problem.source is not None:
            wav = np.ascontiguousarray(problem.source.wavelet, np.float32)
            self._keep.append(wav)
            p.has_source = 1
            for d in range(3):
                p.source[d] = int(problem.source.point[d])
            p.wavelet = N.fptr(wav)
            p.wavelet_len = wav.size
        self.receivers = None
        if receivers is not None:
            rec = np.ascontiguousarray(receivers, np.int32).reshape(-1, 3)
            self._keep.append(rec)
            self.receivers = rec
            p.n_receivers = rec.shape[0]
            p.receivers = rec.ctypes.data_as(C.POINTER(C.c_int32))
        self.receiver_coords = None
        if receiver_coords is not None:
            rc = np.ascontiguousarray(receiver_coords, np.float64).reshape(-1, 3)
            self._keep.append(rc)
            self.receiver_coords = rc
            p.n_coord_receivers = rc.shape[0]
            p.coord_receivers = rc.ctypes.data_as(C.POINTER(C.c_double))
        p.form = _FORMS[self.form]
        p.check_bounds = 1 if check_bounds else 0
        p.time_block = int(time_block)
        p.device = int(device)
        if slab is not None:
            p.slab_lo, p.slab_hi = int(slab[0]), int(slab[1])
        self.slab = (0, problem.shape[0]) if slab is None else (int(slab[0]), int(slab[1]))
        self._h = C.c_void_p()
        _check(N.lib.swb_create(C.byref(p), C.byref(self._h)))
        self._keep.append(p)
        self.step = 0

    # -- state ---------------------------------------------------------------------------
    def set_level(self, level: int, values: np.ndarray) -> None:
        v = np.ascontiguousarray(values, np.float32).reshape(-1)
        if v.size != self.problem.cell_count():
            raise ValueError("interior data size does not match the grid")
        _check(N.lib.swb_set_level(self._h, int(level), N.fptr(v)))

    def get_level(self, level: int, out: Optional[np.ndarray] = None) -> np.ndarray:
        if out is None:
            out = np.zeros(self.problem.shape, np.float32)
        elif (not isinstance(out, np.ndarray) or out.dtype != np.float32
              or out.size != self.problem.cell_count() or not out.flags.c_contiguous):
            # the library writes a whole grid of float32 through this pointer
            raise ValueError("out must be a grid-sized C-contiguous float32 array")
        _check(N.lib.swb_get_level(self._h, int(level), N.fptr(out)))
        return out

    def levels(self) -> np.ndarray:
        return np.stack([self.get_level(l) for l in range(3)])

    # -- stepping ------------------------------------------------------------------------
    def apply(self, nt: Optional[int] = None, step0: Optional[int] = None) -> RunResult:
        nt = self.problem.steps if nt is None else int(nt)
        step0 = self.step if step0 is None else int(step0)
        smax = np.zeros(nt, np.float32)
        bad = C.c_int32(-1)
        n_rec = (0 if self.receivers is None else self.receivers.shape[0]) + \
            (0 if self.receiver_coords is None else self.receiver_coords.shape[0])
        traces = np.zeros((nt, n_rec), np.float32) if n_rec else None
        t0 = time.perf_counter()
        rc = N.lib.swb_apply(self._h, step0, nt, N.fptr(smax), C.byref(bad),
                             N.fptr(traces) if traces is not None else N.fptr(None))
        wall = time.perf_counter() - t0
        if rc != N.SWB_OK:
            _check(rc, bad.value)
        self.step = step0 + nt
        st = self.stats()
        return RunResult(Field(self.problem), smax, wall, 0, (step0 + nt) % 3, traces,
                         st.device_ms * 1e-3)

    def restore(self, directory: str, stem: str, step: int) -> None:
        """Resume from write_checkpoint(directory, stem, op) taken at ``step``: loads u[step]
        and u[step-1] into the levels the next step reads; apply() continues at ``step``."""
        cur, mc = read_snapshot(os.path.join(directory, f"{stem}_{step:06d}"))
        prev, mp = read_snapshot(os.path.join(directory, f"{stem}_{step - 1:06d}"))
        if mc["shape"] != tuple(self.problem.shape) or mp["step"] != step - 1 or mc["step"] != step:
            raise ValueError("checkpoint does not match this problem/step")
        self.set_level(step % 3, cur)
        self.set_level((step + 2) % 3, prev)
        self.step = step

    def apply_snapshots(self, nt: int, every: int, step0: Optional[int] = None,
                        out: Optional[list] = None) -> Tuple[RunResult, list]:
        """apply(nt) plus a snapshot of the newest level after every ``every`` steps, drained
        to host memory on a copy stream while the following steps run (swb_apply_snapshots).
        ``out`` may supply the nt // every grid-sized float32 host buffers (pinned for full
        PCIe bandwidth).  Returns (the RunResult of apply, the snapshot arrays)."""
        nt, every = int(nt), int(every)
        step0 = self.step if step0 is None else int(step0)
        ns = nt // every
        snaps = out if out is not None else [np.zeros(self.problem.shape, np.float32) for _ in range(ns)]
        if len(snaps) != ns:
            raise ValueError(f"need {ns} snapshot buffers")
        for a in snaps:
            if a.dtype != np.float32 or a.size != self.problem.cell_count() or not a.flags.c_contiguous:
                raise ValueError("snapshot buffers must be grid-sized C-contiguous float32")
        arr = (C.POINTER(C.c_float) * max(ns, 1))(*[N.fptr(a) for a in snaps])
        smax = np.zeros(nt, np.float32)
        bad = C.c_int32(-1)
        n_rec = (0 if self.receivers is None else self.receivers.shape[0]) + \
            (0 if self.receiver_coords is None else self.receiver_coords.shape[0])
        traces = np.zeros((nt, n_rec), np.float32) if n_rec else None
        t0 = time.perf_counter()
        rc = N.lib.swb_apply_snapshots(self._h, step0, nt, every, arr, ns, N.fptr(smax), C.byref(bad),
                                       N.fptr(traces) if traces is not None else N.fptr(None))
        wall = time.perf_counter() - t0
        if rc != N.SWB_OK:
            _check(rc, bad.value)
        self.step = step0 + nt
        st = self.stats()
        return (RunResult(Field(self.problem), smax, wall, 0, (step0 + nt) % 3, traces, st.device_ms * 1e-3),
                snaps)

    def apply_adjoint(self, rec_data: np.ndarray) -> np.ndarray:
        """Adjoint of the map source wavelet -> receiver traces (an addition; the reference has
        no adjoint): inject ``rec_data[nt][n_receivers]`` (on-grid receivers
        first, then ``receiver_coords``) backwards in time from a zero field and return the
        source-point trace ``[nt]`` such that <apply traces, rec_data> == <wavelet, result>.
        Overwrites the operator's levels.  See swb_apply_adjoint in include/swb.h."""
        n_rec = (0 if self.receivers is None else self.receivers.shape[0]) + \
            (0 if self.receiver_coords is None else self.receiver_coords.shape[0])
        data = np.ascontiguousarray(rec_data, np.float32)
        if data.ndim != 2 or data.shape[1] != n_rec:
            raise ValueError(f"rec_data must be [nt][{n_rec}]")
        nt = data.shape[0]
        out = np.zeros(nt, np.float32)
        smax = np.zeros(nt, np.float32)
        bad = C.c_int32(-1)
        rc = N.lib.swb_apply_adjoint(self._h, nt, N.fptr(data), N.fptr(out), N.fptr(smax), C.byref(bad))
        if rc != N.SWB_OK:
            _check(rc, bad.value)
        return out

    def apply_async(self, nt: int, step0: int) -> None:
        _check(N.lib.swb_apply_async(self._h, int(step0), int(nt)))
        self.step = step0 + nt

    def collect(self, nt: int):
        smax = np.zeros(nt, np.float32)
        bad = C.c_int32(-1)
        rc = N.lib.swb_collect(self._h, N.fptr(smax), C.byref(bad), N.fptr(None))
        if rc != N.SWB_OK:
            _check(rc, bad.value)
        return smax

    def stream_ptr(self) -> int:
        return int(N.lib.swb_stream(self._h) or 0)

    def stats(self) -> N.SwbStats:
        s = N.SwbStats()
        _check(N.lib.swb_get_stats(self._h, C.byref(s)))
        return s

    # -- multi-GPU z-slabs -----------------------------------------------------------------
    def export_ghosts(self) -> bytes:
        n = C.c_size_t(0)
        N.lib.swb_export_ghosts(self._h, None, C.byref(n))
        buf = C.create_string_buffer(n.value)
        _check(N.lib.swb_export_ghosts(self._h, buf, C.byref(n)))
        return buf.raw[: n.value]

    def link_neighbours(self, lower: Optional[bytes], upper: Optional[bytes]) -> None:
        lb = C.create_string_buffer(lower, len(lower)) if lower else None
        ub = C.create_string_buffer(upper, len(upper)) if upper else None
        _check(N.lib.swb_link_neighbours(self._h, lb, len(lower) if lower else 0,
                                         ub, len(upper) if upper else 0))

    @staticmethod
    def link_local(lower: "Operator", upper: "Operator") -> None:
        _check(N.lib.swb_link_local(lower._h, upper._h))

    def close(self) -> None:
        if self._h:
            N.lib.swb_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run(problem: WaveProblem, options: Optional[RunOptions] = None,
        dse: DseLevel = DseLevel.aggressive, *, form: Optional[str] = None,
        receivers: Optional[np.ndarray] = None, receiver_coords: Optional[np.ndarray] = None,
        device: int = 0) -> RunResult:
    """exec::run (include/stencilc/executor.hpp:90-91, src/executor.cpp:546-613).

    The IET argument of the reference is identified by its DSE level: the acoustic IET
    built by lower -> optimize_all(dse) -> build_iet for this problem.
    """
    options = options or RunOptions()
    op = Operator(problem, dse, form=form, receivers=receivers, receiver_coords=receiver_coords,
                  device=device, check_bounds=options.check_bounds)
    try:
        if options.initial_u is not None:
            if len(options.initial_u) > 3:
                raise ValueError("more initial levels than storage levels")
            for l, v in enumerate(options.initial_u):
                op.set_level(l, v)
        per_step = 1
        for s in problem.shape:
            per_step *= s - 2 * max(problem.halo(), 1)
        per_step += 1 if problem.source is not None else 0
        if options.on_step is None:
            res = op.apply(problem.steps, 0)
        else:
            # slow path: the callback sees the newest level after every step
            smax, traces, wall = [], [], 0.0
            for s in range(problem.steps):
                r = op.apply(1, s)
                wall += r.wall_seconds
                smax.append(r.step_max_abs[0])
                if r.rec_traces is not None:
                    traces.append(r.rec_traces[0])
                # step s writes only level (s+1)%3: one level per step after the first download
                if s == 0:
                    lv = op.levels()
                else:
                    op.get_level((s + 1) % 3, lv[(s + 1) % 3])
                options.on_step(s, Field(problem, lv), (s + 1) % 3)
            res = RunResult(Field(problem), np.array(smax, np.float32), wall, 0,
                            problem.steps % 3, np.array(traces) if traces else None)
        res.u = Field(problem, op.levels())
        res.point_updates = per_step * problem.steps
        res.final_level = problem.steps % 3
        return res
    finally:
        op.close()


def write_snapshot(directory: str, stem: str, step: int, field: Field, level: int,
                   problem: WaveProblem) -> str:
    """exec::write_snapshot (src/executor.cpp:816-837): <stem>_<step:06d>.f32 (LE FP32,
    C order interior) plus a .meta sidecar with shape=, spacing=, step=."""
    os.makedirs(directory, exist_ok=True)
    base = os.path.join(directory, f"{stem}_{step:06d}")
    field.interior(level).astype("<f4").tofile(base + ".f32")
    with open(base + ".meta", "w") as f:
        f.write("shape=" + ",".join(str(s) for s in problem.shape) + "\n")
        f.write("spacing=" + ",".join(_fmt_double(h) for h in problem.spacing) + "\n")
        f.write(f"step={step}\n")
    return base


def read_snapshot(base: str) -> Tuple[np.ndarray, dict]:
    """Inverse of write_snapshot: the grid-sized FP32 level stored at ``<base>.f32`` and the
    sidecar's ``shape``/``spacing``/``step`` (an addition: the reference only writes snapshots)."""
    meta = {}
    with open(base + ".meta") as f:
        for line in f:
            if "=" in line:
                k, v = line.strip().split("=", 1)
                meta[k] = v
    shape = tuple(int(x) for x in meta["shape"].split(","))
    meta = {"shape": shape, "spacing": tuple(float(x) for x in meta["spacing"].split(",")),
            "step": int(meta["step"])}
    data = np.fromfile(base + ".f32", dtype="<f4")
    if data.size != int(np.prod(shape)):
        raise ValueError(f"{base}.f32 holds {data.size} values, the sidecar says {shape}")
    return data.reshape(shape).astype(np.float32), meta


def write_checkpoint(directory: str, stem: str, op: "Operator") -> Tuple[str, str]:
    """Restart point of an Operator at its current step s, as two reference-format snapshots:
    u[s] (``<stem>_<s>``) and u[s-1] (``<stem>_<s-1>``) -- the two levels the next step reads
    (RunOptions::initial_u semantics, src/executor.cpp:387-393)."""
    s = op.step
    if s < 1:
        raise ValueError("a checkpoint needs at least one completed step")
    f = Field(op.problem, op.levels())
    a = write_snapshot(directory, stem, s, f, s % 3, op.problem)
    b = write_snapshot(directory, stem, s - 1, f, (s + 2) % 3, op.problem)
    return a, b


def _fmt_double(v: float) -> str:
    """std::ostream default formatting of a double (%g with 6 significant digits)."""
    return f"{v:g}"
