"""ORACLE TEST INFRASTRUCTURE ONLY — ctypes bindings for the two CPU checkers.

* ``ref_*``  drive the reference's OWN C++ sources (oracle/_ref/libstencilc_ref.so,
  built by ``make -C oracle ref`` from /root/reference/proj/src; see oracle/ref_capi.cpp).
* ``port_*`` drive the C restatement (oracle/port/libwave_port.so, ``make -C oracle port``).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference arm may
import this module, and only as the checker or the timed CPU baseline.  The product
(paper_1912_00695_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libstencilc_ref.so")
PORT_SO = os.path.join(HERE, "port", "libwave_port.so")


class _Config(C.Structure):
    # Layout shared by ref_config (oracle/ref_capi.cpp) and port_config (oracle/port/wave_port.c).
    _fields_ = [
        ("rank", C.c_int32), ("shape", C.c_int32 * 3), ("spacing", C.c_double * 3),
        ("space_order", C.c_int32), ("dt", C.c_double), ("steps", C.c_int32),
        ("velocity", C.c_double), ("velocity_field", C.POINTER(C.c_float)),
        ("damp_max", C.c_double), ("damp_width", C.c_int32), ("with_source", C.c_int32),
        ("source_point", C.c_int32 * 3), ("source_frequency", C.c_double),
        ("source_wavelet", C.POINTER(C.c_float)), ("source_wavelet_len", C.c_int32),
    ]


class _RunOut(C.Structure):
    _fields_ = [
        ("levels", C.POINTER(C.c_float)), ("step_max_abs", C.POINTER(C.c_float)),
        ("rec_traces", C.POINTER(C.c_float)), ("wall_seconds", C.c_double),
        ("point_updates", C.c_uint64), ("final_level", C.c_int32), ("bad_step", C.c_int32),
    ]


@dataclass
class OracleConfig:
    """Mirror of exec::WaveProblemConfig (include/stencilc/wave_model.hpp:41-56)."""
    shape: Sequence[int]
    spacing: Sequence[float] = (10.0, 10.0, 10.0)
    space_order: int = 8
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
    _keep: list = field(default_factory=list, repr=False)

    def to_c(self) -> _Config:
        c = _Config()
        c.rank = len(self.shape)
        for d in range(c.rank):
            c.shape[d] = int(self.shape[d])
            c.spacing[d] = float(self.spacing[d])
        c.space_order = int(self.space_order)
        c.dt = float(self.dt)
        c.steps = int(self.steps)
        c.velocity = float(self.velocity)
        self._keep = []
        if self.velocity_field is not None:
            vf = np.ascontiguousarray(self.velocity_field, dtype=np.float32)
            self._keep.append(vf)
            c.velocity_field = vf.ctypes.data_as(C.POINTER(C.c_float))
        c.damp_max = float(self.damp_max)
        c.damp_width = int(self.damp_width)
        c.with_source = 1 if self.with_source else 0
        if self.source_point is None:
            c.source_point[0] = -1
        else:
            for d in range(c.rank):
                c.source_point[d] = int(self.source_point[d])
        c.source_frequency = float(self.source_frequency)
        if self.source_wavelet is not None:
            w = np.ascontiguousarray(self.source_wavelet, dtype=np.float32)
            self._keep.append(w)
            c.source_wavelet = w.ctypes.data_as(C.POINTER(C.c_float))
            c.source_wavelet_len = int(w.size)
        return c

    @property
    def ncells(self) -> int:
        return int(np.prod(self.shape))


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str, step: int = -1):
        super().__init__(msg)
        self.code = code
        self.step = step


_libs: dict = {}


def build(which: str = "port") -> None:
    """Build the checker library (``port`` always; ``ref`` needs /root/reference)."""
    subprocess.run(["make", "-s", "-C", HERE, which], check=True)


def _lib(which: str):
    if which in _libs:
        return _libs[which]
    path = REF_SO if which == "ref" else PORT_SO
    if not os.path.exists(path):
        if which == "port":
            build("port")
        else:
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
    lib = C.CDLL(path)
    pre = "ref_" if which == "ref" else "port_"
    getattr(lib, pre + "last_error").restype = C.c_char_p
    getattr(lib, pre + "omp_max_threads").restype = C.c_int
    _libs[which] = lib
    return lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _fptr(a: Optional[np.ndarray]):
    if a is None:
        return C.POINTER(C.c_float)()
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _run(which: str, cfg: OracleConfig, *, dse: str = "basic", threads: int = 0,
         serial: bool = False, initial_u=None, receivers=None, receiver_coords=None) -> dict:
    lib = _lib(which)
    c = cfg.to_c()
    n = cfg.ncells
    levels = np.zeros((3, n), np.float32)
    smax = np.zeros(cfg.steps, np.float32)
    rec = None if receivers is None else np.ascontiguousarray(receivers, np.int32).reshape(-1, len(cfg.shape))
    n_rec = 0 if rec is None else rec.shape[0]
    traces = np.zeros((cfg.steps, max(n_rec, 1)), np.float32)
    out = _RunOut()
    out.levels = _fptr(levels)
    out.step_max_abs = _fptr(smax)
    out.rec_traces = _fptr(traces) if n_rec else C.POINTER(C.c_float)()
    init_keep = []
    init_arr = None
    n_init = 0
    if initial_u is not None:
        n_init = len(initial_u)
        init_keep = [np.ascontiguousarray(a, np.float32).reshape(-1) for a in initial_u]
        init_arr = (C.POINTER(C.c_float) * n_init)(*[_fptr(a) for a in init_keep])
    rec_ptr = rec.ctypes.data_as(C.POINTER(C.c_int32)) if n_rec else C.POINTER(C.c_int32)()
    if which == "ref":
        rc = lib.ref_run(C.byref(c), 1 if dse == "aggressive" else 0, int(threads),
                         1 if serial else 0, init_arr, n_init, n_rec, rec_ptr, C.byref(out))
        err = lib.ref_last_error
    else:
        crec = None if receiver_coords is None else np.ascontiguousarray(receiver_coords, np.float64).reshape(-1, 3)
        n_crec = 0 if crec is None else crec.shape[0]
        ctr = np.zeros((cfg.steps, max(n_crec, 1)), np.float32)
        rc = lib.port_run2(C.byref(c), int(threads), init_arr, n_init, n_rec, rec_ptr, n_crec,
                           crec.ctypes.data_as(C.POINTER(C.c_double)) if n_crec else C.POINTER(C.c_double)(),
                           _fptr(ctr) if n_crec else C.POINTER(C.c_float)(), C.byref(out))
        err = lib.port_last_error
    if rc != 0:
        raise OracleError(rc, err().decode(), out.bad_step)
    shape = tuple(cfg.shape)
    coord_traces = None
    if which == "port" and receiver_coords is not None:
        coord_traces = ctr[:, :n_crec]
    return {
        "coord_traces": coord_traces,
        "levels": levels.reshape((3,) + shape),
        "step_max_abs": smax,
        "rec_traces": traces[:, :n_rec] if n_rec else None,
        "wall_seconds": out.wall_seconds,
        "point_updates": int(out.point_updates),
        "final_level": int(out.final_level),
    }


def ref_run(cfg: OracleConfig, **kw) -> dict:
    """exec::run (or exec::reference_run with serial=True) of the reference itself."""
    if kw.get("receiver_coords") is not None:
        raise ValueError("the reference has no off-grid receivers (use port_run)")
    kw.pop("receiver_coords", None)
    return _run("ref", cfg, **kw)


def port_run(cfg: OracleConfig, **kw) -> dict:
    """The C restatement of exec::run on the basic IET."""
    kw.pop("dse", None)
    kw.pop("serial", None)
    return _run("port", cfg, **kw)


def ref_info(cfg: OracleConfig) -> dict:
    lib = _lib("ref")
    c = cfg.to_c()
    n = cfg.ncells
    dt = C.c_float()
    wav = np.zeros(cfg.steps, np.float32)
    m = np.zeros(n, np.float32)
    damp = np.zeros(n, np.float32)
    src = (C.c_int32 * 3)()
    so = cfg.space_order
    wn = (C.c_int64 * (so + 1))()
    wd = (C.c_int64 * (so + 1))()
    hb, ha = C.c_uint64(), C.c_uint64()
    fb, fa = C.c_int64(), C.c_int64()
    rc = lib.ref_problem_info(C.byref(c), C.byref(dt), _fptr(wav), _fptr(m), _fptr(damp), src,
                              wn, wd, C.byref(hb), C.byref(ha), C.byref(fb), C.byref(fa))
    if rc:
        raise OracleError(rc, lib.ref_last_error().decode())
    return {
        "dt": dt.value, "wavelet": wav, "m": m.reshape(tuple(cfg.shape)),
        "damp": damp.reshape(tuple(cfg.shape)), "source_point": tuple(src[: len(cfg.shape)]),
        "weights": [(wn[i], wd[i]) for i in range(so + 1)],
        "iet_hash_basic": hb.value, "iet_hash_aggressive": ha.value,
        "flops_basic": fb.value, "flops_aggressive": fa.value,
    }


def port_info(cfg: OracleConfig) -> dict:
    lib = _lib("port")
    c = cfg.to_c()
    n = cfg.ncells
    dt = C.c_float()
    wav = np.zeros(cfg.steps, np.float32)
    m = np.zeros(n, np.float32)
    damp = np.zeros(n, np.float32)
    src = (C.c_int32 * 3)()
    rc = lib.port_problem_info(C.byref(c), C.byref(dt), _fptr(wav), _fptr(m), _fptr(damp), src)
    if rc:
        raise OracleError(rc, lib.port_last_error().decode())
    so = cfg.space_order
    wn = (C.c_int64 * (so + 1))()
    wd = (C.c_int64 * (so + 1))()
    lib.port_fd_weights(so, wn, wd)
    return {
        "dt": dt.value, "wavelet": wav, "m": m.reshape(tuple(cfg.shape)),
        "damp": damp.reshape(tuple(cfg.shape)), "source_point": tuple(src[:3]),
        "weights": [(wn[i], wd[i]) for i in range(so + 1)],
    }


def ref_emit_c(cfg: OracleConfig, dse: str = "basic") -> str:
    lib = _lib("ref")
    lib.ref_emit_reference_c.restype = C.c_int64
    c = cfg.to_c()
    need = lib.ref_emit_reference_c(C.byref(c), 1 if dse == "aggressive" else 0, None, 0)
    buf = C.create_string_buffer(int(need))
    lib.ref_emit_reference_c(C.byref(c), 1 if dse == "aggressive" else 0, buf, need)
    return buf.value.decode()


def omp_threads(which: str = "port") -> int:
    lib = _lib(which)
    return int(getattr(lib, ("ref_" if which == "ref" else "port_") + "omp_max_threads")())


def port_adjoint(cfg: OracleConfig, rec_data: np.ndarray, *, receivers=None, receiver_coords=None,
                 threads: int = 0) -> np.ndarray:
    """Adjoint of the C restatement's forward map (source wavelet -> receiver traces): the
    receiver data rec_data[steps][n_rec + n_coord] is injected backwards in time and the
    source-point trace [steps] is returned (see port_adjoint in port/wave_port.c)."""
    lib = _lib("port")
    c = cfg.to_c()
    rec = None if receivers is None else np.ascontiguousarray(receivers, np.int32).reshape(-1, 3)
    n_rec = 0 if rec is None else rec.shape[0]
    crec = None if receiver_coords is None else np.ascontiguousarray(receiver_coords, np.float64).reshape(-1, 3)
    n_crec = 0 if crec is None else crec.shape[0]
    data = np.ascontiguousarray(rec_data, np.float32).reshape(cfg.steps, n_rec + n_crec)
    out = np.zeros(cfg.steps, np.float32)
    rc = lib.port_adjoint(C.byref(c), int(threads), n_rec,
                          rec.ctypes.data_as(C.POINTER(C.c_int32)) if n_rec else C.POINTER(C.c_int32)(),
                          n_crec, crec.ctypes.data_as(C.POINTER(C.c_double)) if n_crec else C.POINTER(C.c_double)(),
                          _fptr(data), _fptr(out))
    if rc != 0:
        raise OracleError(rc, lib.port_last_error().decode())
    return out
