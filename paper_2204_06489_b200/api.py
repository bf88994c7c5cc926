"""Python mirror of the reference's operator/solver API over the C ABI.

Names, argument meaning and error behaviour follow the reference
(include/fwi/kkt.hpp, include/fwi/krylov.hpp, include/fwi/lu.hpp,
include/fwi/ilu.hpp); the work happens in libfwi_b200.so (sm_100a CUDA).
There is no CPU fallback: if the library or a GPU is missing, calls raise.

    state = GnState(problem, exact=True, ilu_level=4)      # make_gn_state
    xi = KktVector.from_host(state, flat)                  # KktVector
    out = kkt_apply(state, xi)                             # kkt_apply
    b = kkt_rhs(state)                                     # kkt_rhs
    z = precond_apply(state, xi, PrecondMode.exact)        # precond_apply
    ds, log = fsgn_gmres_step(state, FsgnOptions(...))     # fsgn_gmres_step
"""
from __future__ import annotations

import ctypes as C
import enum
import os
import subprocess
import threading
from dataclasses import dataclass

import numpy as np

from . import _abi
from .krylov import ConvergenceLog
from .problem import Problem

HERE = os.path.dirname(os.path.abspath(__file__))
# FWI_B200_LIB: another build of the same library (binary A/B runs, tools/ab_lib.py)
LIB_PATH = os.environ.get("FWI_B200_LIB") or os.path.join(HERE, "libfwi_b200.so")

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_vp = C.c_void_p


# ---------------------------------------------------------------------------
# errors (the reference's exception types)
# ---------------------------------------------------------------------------
class FwiError(RuntimeError):
    code = -1


class InvalidArgument(FwiError, ValueError):
    """std::invalid_argument"""
    code = _abi.FWI_ERR_INVALID_ARGUMENT


class SingularPivotError(FwiError):
    """fwi::SingularPivotError (include/fwi/lu.hpp:11-16)"""
    code = _abi.FWI_ERR_SINGULAR_PIVOT

    def __init__(self, msg, index):
        super().__init__(msg)
        self.index = index


class ZeroPivotError(FwiError):
    """fwi::ZeroPivotError (include/fwi/ilu.hpp:11-17)"""
    code = _abi.FWI_ERR_ZERO_PIVOT

    def __init__(self, msg, index):
        super().__init__(msg)
        self.index = index


class CudaError(FwiError):
    code = _abi.FWI_ERR_CUDA


class CgBreakdownError(FwiError):
    """fwi::CgBreakdownError (include/fwi/krylov.hpp:35-37)"""
    code = 7


class PrecondMode(enum.IntEnum):
    exact = _abi.FWI_PRECOND_EXACT
    ilu = _abi.FWI_PRECOND_ILU


# ---------------------------------------------------------------------------
# library loading
# ---------------------------------------------------------------------------
_lib = None
_lock = threading.Lock()


def build_library(force: bool = False) -> str:
    """Compile csrc/ for sm_100a into libfwi_b200.so (in-tree)."""
    if force or not os.path.exists(LIB_PATH):
        out = subprocess.run(["make", "-C", os.path.join(HERE, "csrc"), "-j16"], capture_output=True,
                             text=True)
        if out.returncode != 0:
            raise RuntimeError("CUDA library build failed:\n" + out.stdout[-6000:] + out.stderr[-6000:])
    return LIB_PATH


def lib() -> C.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                build_library()
            L = C.CDLL(LIB_PATH)
            sig = {
                "fwi_dev_ctx_create": [C.c_void_p, C.POINTER(_vp)],
                "fwi_dev_ctx_destroy": [_vp],
                "fwi_dev_ctx_info": [_vp, C.c_void_p],
                "fwi_dev_ctx_set_epsilon": [_vp, C.c_double],
                "fwi_dev_ctx_set_drop_reg_term": [_vp, C.c_int],
                "fwi_dev_ctx_synchronize": [_vp],
                "fwi_dev_ctx_get_u": [_vp, _dp],
                "fwi_dev_ctx_get_residual": [_vp, _dp],
                "fwi_dev_ctx_get_dpred": [_vp, _dp],
                "fwi_dev_ctx_get_stencil": [_vp, _dp, _dp, _dp],
                "fwi_dev_factor_exact": [_vp],
                "fwi_dev_factor_ilu": [_vp, C.c_int, C.c_double],
                "fwi_dev_solve": [_vp, C.c_int, C.c_int, C.c_int, _dp, _dp],
                "fwi_dev_vec_create": [_vp, C.c_int, C.POINTER(_vp)],
                "fwi_dev_vec_destroy": [_vp],
                "fwi_dev_vec_precision": [_vp],
                "fwi_dev_vec_upload": [_vp, _dp],
                "fwi_dev_vec_download": [_vp, _dp],
                "fwi_dev_vec_upload_f32": [_vp, _fp],
                "fwi_dev_vec_download_f32": [_vp, _fp],
                "fwi_dev_vec_copy": [_vp, _vp],
                "fwi_dev_vec_zero": [_vp],
                "fwi_dev_vec_dot": [_vp, _vp, _dp],
                "fwi_dev_vec_norm": [_vp, _dp],
                "fwi_dev_vec_axpy": [C.c_double, _vp, _vp],
                "fwi_dev_vec_scal": [C.c_double, _vp],
                "fwi_dev_vec_device_ptr": [_vp, C.POINTER(_vp)],
                "fwi_dev_kkt_apply": [_vp, _vp, _vp],
                "fwi_dev_kkt_rhs": [_vp, _vp],
                "fwi_dev_kkt_apply_host": [_vp, _dp, _dp],
                "fwi_dev_gn_step": [C.c_void_p, C.c_void_p, _dp, C.c_void_p, C.c_void_p],
                "fwi_dev_rsgn_cg_step": [_vp, C.c_double, C.c_int, _dp, C.c_void_p],
                "fwi_dev_gradient": [_vp, _dp],
                "fwi_dev_hessian_apply": [_vp, _dp, _dp],
                "fwi_dev_precond_apply": [_vp, C.c_int, _vp, _vp],
                "fwi_dev_fsgn_gmres_step": [_vp, C.c_void_p, _dp, C.c_void_p],
                "fwi_dev_gmres_generic": [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, _vp, _vp, _vp,
                                          C.c_int, C.c_double, C.c_int, C.c_void_p],
                "fwi_dev_malloc": [C.POINTER(_vp), C.c_int64],
                "fwi_dev_free": [_vp],
                "fwi_dev_memcpy_h2d": [_vp, _vp, C.c_int64],
                "fwi_dev_memcpy_d2h": [_vp, _vp, C.c_int64],
                "fwi_dev_ctx_stream": [_vp, C.POINTER(_vp)],
                "fwi_host_register": [_vp, C.c_int64],
                "fwi_host_unregister": [_vp],
                "fwi_host_alloc": [C.POINTER(_vp), C.c_int64],
                "fwi_host_free": [_vp],
            }
            for name, args in sig.items():
                f = getattr(L, name)
                f.argtypes = args
                f.restype = C.c_int
            L.fwi_dev_last_error.restype = C.c_char_p
            L.fwi_dev_last_error_index.restype = C.c_int
            L.fwi_dev_version.restype = C.c_char_p
            L.fwi_dev_solve_count.argtypes = [_vp, C.c_int]
            L.fwi_dev_solve_count.restype = C.c_int64
            L.fwi_dev_reset_solve_count.argtypes = [_vp, C.c_int]
            L.fwi_dev_reset_solve_count.restype = None
            L.fwi_dev_kkt_kernel.argtypes = [_vp, C.c_int]
            L.fwi_dev_kkt_kernel.restype = C.c_char_p
            _lib = L
    return _lib


def _check(code: int) -> None:
    if code == 0:
        return
    L = lib()
    msg = L.fwi_dev_last_error().decode()
    idx = L.fwi_dev_last_error_index()
    if code == _abi.FWI_ERR_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if code == _abi.FWI_ERR_SINGULAR_PIVOT:
        raise SingularPivotError(msg, idx)
    if code == _abi.FWI_ERR_ZERO_PIVOT:
        raise ZeroPivotError(msg, idx)
    if code == _abi.FWI_ERR_CUDA:
        raise CudaError(msg)
    if code == 7:
        raise CgBreakdownError(msg)
    e = FwiError(f"[{code}] {msg}")
    e.code = code
    raise e


def _p(a):
    return a.ctypes.data_as(_dp)


# ---------------------------------------------------------------------------
# GnState / KktVector
# ---------------------------------------------------------------------------
class GnState:
    """Device-resident fwi::GnState (make_gn_state, src/reduced_space.cpp:40-86)."""

    def __init__(self, problem: Problem, *, exact: bool = True, ilu_level: int = -1,
                 ilu_diag_shift: float = 0.0, c64: bool = False):
        L = lib()
        self.problem = problem
        d, self._keep = problem.desc(exact_factor=exact, ilu_level=ilu_level,
                                     ilu_diag_shift=ilu_diag_shift,
                                     precision_mask=(1 << _abi.FWI_C64) if c64 else 0)
        h = _vp()
        _check(L.fwi_dev_ctx_create(C.byref(d), C.byref(h)))
        self.h = h
        self._info()

    def _info(self):
        info = _abi.StateInfo()
        _check(lib().fwi_dev_ctx_info(self.h, C.byref(info)))
        self.n, self.K, self.num_data = info.n, info.num_sources, info.num_data
        self.omega, self.epsilon = info.omega, info.epsilon
        self.vec_len = int(info.vec_doubles)
        self.device_bytes = int(info.device_bytes)
        self.has_exact, self.has_ilu = bool(info.has_exact), bool(info.has_ilu)
        self.exact_factor_bytes, self.ilu_factor_bytes = int(info.exact_factor_bytes), int(info.ilu_factor_bytes)
        self.exact_probe_residual = float(info.exact_probe_residual)

    def close(self):
        if getattr(self, "h", None):
            lib().fwi_dev_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def model_size(self):
        return self.n

    def num_sources(self):
        return self.K

    def set_epsilon(self, e):
        _check(lib().fwi_dev_ctx_set_epsilon(self.h, e))
        self._info()

    def set_drop_reg_term(self, d: bool):
        _check(lib().fwi_dev_ctx_set_drop_reg_term(self.h, int(d)))

    def synchronize(self):
        _check(lib().fwi_dev_ctx_synchronize(self.h))

    def stream_ptr(self) -> int:
        s = _vp()
        _check(lib().fwi_dev_ctx_stream(self.h, C.byref(s)))
        return s.value or 0

    def u(self):
        out = np.empty(self.K * self.n, np.complex128)
        _check(lib().fwi_dev_ctx_get_u(self.h, _p(out)))
        return out

    def residual(self):
        out = np.empty(max(self.num_data, 1), np.complex128)
        _check(lib().fwi_dev_ctx_get_residual(self.h, _p(out)))
        return out[: self.num_data]

    def d_pred(self):
        out = np.empty(max(self.num_data, 1), np.complex128)
        _check(lib().fwi_dev_ctx_get_dpred(self.h, _p(out)))
        return out[: self.num_data]

    def stencil(self):
        d, e, s = (np.empty(self.n, np.complex128) for _ in range(3))
        _check(lib().fwi_dev_ctx_get_stencil(self.h, _p(d), _p(e), _p(s)))
        return d, e, s

    def factor_exact(self):
        _check(lib().fwi_dev_factor_exact(self.h))
        self._info()

    def factor_ilu(self, level: int, diag_shift: float = 0.0):
        _check(lib().fwi_dev_factor_ilu(self.h, level, diag_shift))
        self._info()

    def kkt_kernel(self, precision=None) -> str:
        """Name of the K1 kernel the last kkt_apply at this precision launched."""
        prec = _abi.FWI_C128 if precision is None else precision
        return lib().fwi_dev_kkt_kernel(self.h, int(prec)).decode()

    def solve_count(self, mode=PrecondMode.exact) -> int:
        return lib().fwi_dev_solve_count(self.h, int(mode))

    def reset_solve_count(self, mode=PrecondMode.exact):
        lib().fwi_dev_reset_solve_count(self.h, int(mode))

    def solve(self, b: np.ndarray, mode=PrecondMode.exact, adjoint=False) -> np.ndarray:
        """LuFactors::solve / IluFactors::solve for one or several (stacked) RHS."""
        b = np.ascontiguousarray(b, np.complex128)
        nrhs = b.size // self.n
        x = np.empty_like(b)
        _check(lib().fwi_dev_solve(self.h, int(mode), int(adjoint), nrhs, _p(b), _p(x)))
        return x


class KktVector:
    """Device-resident fwi::KktVector (include/fwi/kkt.hpp:12-19), one flat buffer."""

    def __init__(self, state: GnState, precision: int = _abi.FWI_C128):
        self.state = state
        self.precision = precision
        h = _vp()
        _check(lib().fwi_dev_vec_create(state.h, precision, C.byref(h)))
        self.h = h

    @staticmethod
    def zeros(state: GnState, precision: int = _abi.FWI_C128) -> "KktVector":
        return KktVector(state, precision)

    @staticmethod
    def from_host(state: GnState, flat: np.ndarray, precision: int = _abi.FWI_C128) -> "KktVector":
        v = KktVector(state, precision)
        v.upload(flat)
        return v

    def upload(self, flat: np.ndarray):
        if self.precision == _abi.FWI_C128:
            flat = np.ascontiguousarray(flat, np.float64)
            assert flat.size == self.state.vec_len
            _check(lib().fwi_dev_vec_upload(self.h, _p(flat)))
        else:
            flat = np.ascontiguousarray(flat, np.float32)
            assert flat.size == self.state.vec_len
            _check(lib().fwi_dev_vec_upload_f32(self.h, flat.ctypes.data_as(_fp)))

    def to_host(self, out: np.ndarray | None = None) -> np.ndarray:
        if self.precision == _abi.FWI_C128:
            out = np.empty(self.state.vec_len) if out is None else out
            _check(lib().fwi_dev_vec_download(self.h, _p(out)))
        else:
            out = np.empty(self.state.vec_len, np.float32) if out is None else out
            _check(lib().fwi_dev_vec_download_f32(self.h, out.ctypes.data_as(_fp)))
        return out

    def device_ptr(self) -> int:
        p = _vp()
        _check(lib().fwi_dev_vec_device_ptr(self.h, C.byref(p)))
        return p.value

    def copy(self) -> "KktVector":
        v = KktVector(self.state, self.precision)
        _check(lib().fwi_dev_vec_copy(v.h, self.h))
        return v

    def close(self):
        if getattr(self, "h", None):
            lib().fwi_dev_vec_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def dot(x: KktVector, y: KktVector) -> float:
    out = C.c_double()
    _check(lib().fwi_dev_vec_dot(x.h, y.h, C.byref(out)))
    return out.value


def norm(x: KktVector) -> float:
    out = C.c_double()
    _check(lib().fwi_dev_vec_norm(x.h, C.byref(out)))
    return out.value


def axpy(a: float, x: KktVector, y: KktVector) -> None:
    _check(lib().fwi_dev_vec_axpy(float(a), x.h, y.h))


def scal(a: float, x: KktVector) -> None:
    _check(lib().fwi_dev_vec_scal(float(a), x.h))


def kkt_apply(state: GnState, xi: KktVector, out: KktVector | None = None) -> KktVector:
    out = KktVector(state, xi.precision) if out is None else out
    _check(lib().fwi_dev_kkt_apply(state.h, xi.h, out.h))
    return out


def kkt_apply_host(state: GnState, xi: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
    """kkt_apply on host arrays (flat 4Kn+n doubles), streamed through the GPU
    with copy/compute overlap (fwi_dev_kkt_apply_host)."""
    xi = np.ascontiguousarray(xi, np.float64)
    out = np.empty(state.vec_len) if out is None else out
    _check(lib().fwi_dev_kkt_apply_host(state.h, _p(xi), _p(out)))
    return out


def gradient(state: GnState) -> np.ndarray:
    """fwi::gradient (src/reduced_space.cpp:141-152): Re(J^H W^T W r) - eps s."""
    out = np.empty(state.n)
    _check(lib().fwi_dev_gradient(state.h, _p(out)))
    return out


def hessian_apply(state: GnState, v: np.ndarray) -> np.ndarray:
    """fwi::hessian_apply (src/reduced_space.cpp:120-139): Re(J^H W^T W J v) + eps v."""
    v = np.ascontiguousarray(v, np.float64)
    out = np.empty(state.n)
    _check(lib().fwi_dev_hessian_apply(state.h, _p(v), _p(out)))
    return out


def kkt_rhs(state: GnState) -> KktVector:
    out = KktVector(state)
    _check(lib().fwi_dev_kkt_rhs(state.h, out.h))
    return out


def precond_apply(state: GnState, v: KktVector, mode=PrecondMode.exact,
                  out: KktVector | None = None) -> KktVector:
    out = KktVector(state) if out is None else out
    _check(lib().fwi_dev_precond_apply(state.h, int(mode), v.h, out.h))
    return out


@dataclass
class FsgnOptions:
    """fwi::FsgnOptions (include/fwi/kkt.hpp:47-57), same defaults."""
    mode: PrecondMode = PrecondMode.exact
    restart: int = 30
    tol: float = 1e-10
    maxit: int = 30
    ecg_stride: int = 1
    ecg_stop_tol: float = 0.0


def fsgn_gmres_step(state: GnState, options: FsgnOptions = FsgnOptions()):
    """Returns (delta_s, ConvergenceLog) like fwi::fsgn_gmres_step."""
    o = _abi.FsgnOptions(int(options.mode), options.restart, options.tol, options.maxit,
                         options.ecg_stride, options.ecg_stop_tol)
    ds = np.empty(state.n)
    lb = _abi.LogBuffer(options.maxit + 2)
    _check(lib().fwi_dev_fsgn_gmres_step(state.h, C.byref(o), _p(ds), C.byref(lb.c)))
    return ds, lb.to_log()


def host_register(a: np.ndarray) -> None:
    """Page-lock a numpy buffer (cudaHostRegister) for DMA-speed transfers."""
    _check(lib().fwi_host_register(a.ctypes.data, a.nbytes))


def host_unregister(a: np.ndarray) -> None:
    _check(lib().fwi_host_unregister(a.ctypes.data))


class _PinnedOwner:
    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        try:
            lib().fwi_host_free(self.ptr)
        except Exception:
            pass


def host_empty(n: int, dtype=np.float64) -> np.ndarray:
    """A numpy array backed by page-locked memory from cudaHostAlloc (freed with the array)."""
    dt = np.dtype(dtype)
    p = _vp()
    _check(lib().fwi_host_alloc(C.byref(p), max(int(n) * dt.itemsize, 1)))
    buf = (C.c_char * (int(n) * dt.itemsize)).from_address(p.value)
    a = np.frombuffer(buf, dtype=dt, count=int(n))
    a.setflags(write=True)
    owner = _PinnedOwner(p.value)
    buf._owner = owner  # keep the allocation alive as long as the array
    return a


def simulate(problem: Problem, s: np.ndarray | None = None) -> np.ndarray:
    """Observed data Q A(s)^{-1} f on model s (default problem.s_true), computed
    with the device's exact block solver (fixtures::simulate_blocks analogue)."""
    from dataclasses import replace
    q = replace(problem, s=problem.s_true if s is None else s, u=None, r=None, d_obs=None)
    st = GnState(q, exact=True)
    try:
        return st.d_pred()
    finally:
        st.close()


def rsgn_cg_step(state: GnState, tol: float, maxit: int):
    """fwi::rsgn_cg_step (src/reduced_space.cpp:163-170) on the device."""
    ds = np.empty(state.n)
    lb = _abi.LogBuffer(maxit + 2)
    _check(lib().fwi_dev_rsgn_cg_step(state.h, tol, maxit, _p(ds), C.byref(lb.c)))
    return ds, lb.to_log()


# ---------------------------------------------------------------------------
# Gauss-Newton driver (src/driver.cpp:65-155)
# ---------------------------------------------------------------------------
@dataclass
class FwiConfig:
    """The fields of fwi::FwiConfig (include/fwi/driver.hpp:17-42) this path uses."""
    solver: str = "fsgn-gmres-exact"
    max_inner: int = 30
    inner_tol: float = 1e-12
    gmres_restart: int = 30
    ilu_level: int = 4
    ilu_diag_shift: float = 0.0
    v_min: float = 300.0
    v_max: float = 8000.0
    ecg_stride: int = 0
    ecg_stop_tol: float = 0.0


@dataclass
class GnStepResult:
    freq_hz: float
    epsilon: float
    s: np.ndarray
    log: ConvergenceLog
    misfit_ini: float
    misfit_fin: float
    update_relnorm: float
    wall_seconds: float
    setup_seconds: float = 0.0       # linearisation (incl. the host ILU(p) factorisation)
    ilu_factor_seconds: float = 0.0
    krylov_seconds: float = 0.0
    final_seconds: float = 0.0       # re-solve at the updated model


def gn_step(problem: Problem, s: np.ndarray, freq_hz: float, epsilon: float, config: FwiConfig = FwiConfig()):
    """fwi::gn_step: linearise at s, solve the KKT system on the device, clamp, re-solve.
    problem.d_obs must hold the observed data at freq_hz."""
    from dataclasses import replace
    solver = {"rsgn-cg": 0, "fsgn-gmres-exact": _abi.FWI_SOLVER_FSGN_EXACT,
              "fsgn-gmres-ilu": _abi.FWI_SOLVER_FSGN_ILU}
    if config.solver not in solver:
        raise InvalidArgument(f"unknown inner solver '{config.solver}' on this path")
    q = replace(problem, s=np.ascontiguousarray(s, np.float64), freq_hz=freq_hz, epsilon=epsilon, u=None, r=None)
    d, keep = q.desc()
    o = _abi.GnOptions(solver[config.solver], config.max_inner, config.inner_tol, config.gmres_restart,
                       config.ilu_level, config.ilu_diag_shift, config.v_min, config.v_max, config.ecg_stride,
                       config.ecg_stop_tol)
    s_out = np.empty(problem.n)
    res = _abi.GnResult()
    lb = _abi.LogBuffer(config.max_inner + 2)
    _check(lib().fwi_dev_gn_step(C.byref(d), C.byref(o), _p(s_out), C.byref(res), C.byref(lb.c)))
    return GnStepResult(freq_hz, epsilon, s_out, lb.to_log(), res.misfit_ini, res.misfit_fin,
                        res.update_relnorm, res.wall_seconds, res.setup_seconds, res.ilu_factor_seconds,
                        res.krylov_seconds, res.final_seconds)


def fwi_run(problem: Problem, observed: dict, s0: np.ndarray, epsilons: dict, config: FwiConfig = FwiConfig(),
            steps_per_frequency: int = 1):
    """fwi::fwi_run (src/driver.cpp:129-155): ascending frequencies, each consuming the
    previous model; steps_per_frequency > 1 repeats gn_step (BASELINE configs 3-4)."""
    from dataclasses import replace
    report, s = [], np.asarray(s0, np.float64)
    for f in sorted(observed):
        q = replace(problem, d_obs=observed[f])
        for _ in range(steps_per_frequency):
            r = gn_step(q, s, f, epsilons[f], config)
            report.append(r)
            s = r.s
    return report


# ---------------------------------------------------------------------------
# generic GMRES over flat real device vectors (gmres<Vec,OpA,OpM>)
# ---------------------------------------------------------------------------
_OP = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p)
_OBS = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p)


def gmres(apply, precond, b: np.ndarray, restart: int, tol: float, maxit: int, observer=None):
    """fwi::gmres (include/fwi/krylov.hpp:128-269) over a real vector of even
    length, driven by the device GMRES core. `apply`/`precond`/`observer` are
    host callables on numpy arrays (test-size operators)."""
    L = lib()
    b = np.ascontiguousarray(b, np.float64)
    n = b.size
    nb = n * 8
    bd, xd = _vp(), _vp()
    _check(L.fwi_dev_malloc(C.byref(bd), nb))
    _check(L.fwi_dev_malloc(C.byref(xd), nb))
    err: list[BaseException] = []

    def wrap(fn):
        def cb(user, src, dst):
            try:
                x = np.empty(n)
                _check(L.fwi_dev_memcpy_d2h(x.ctypes.data, src, nb))
                y = np.ascontiguousarray(fn(x), np.float64)
                _check(L.fwi_dev_memcpy_h2d(dst, y.ctypes.data, nb))
                return 0
            except BaseException as e:  # noqa: BLE001
                err.append(e)
                return 1
        return _OP(cb)

    def obs(user, it, src):
        try:
            x = np.empty(n)
            _check(L.fwi_dev_memcpy_d2h(x.ctypes.data, src, nb))
            return int(bool(observer(it, x)))
        except BaseException as e:  # noqa: BLE001
            err.append(e)
            return 1

    ca, cp = wrap(apply), wrap(precond)
    co = _OBS(obs) if observer else None
    try:
        _check(L.fwi_dev_memcpy_h2d(bd, b.ctypes.data, nb))
        lb = _abi.LogBuffer(maxit + 2)
        code = L.fwi_dev_gmres_generic(n, C.cast(ca, C.c_void_p), C.cast(cp, C.c_void_p),
                                       C.cast(co, C.c_void_p) if co else None, None, bd, xd, restart,
                                       tol, maxit, C.byref(lb.c))
        if err:
            raise err[0]
        _check(code)
        x = np.empty(n)
        _check(L.fwi_dev_memcpy_d2h(x.ctypes.data, xd, nb))
        return x, lb.to_log()
    finally:
        L.fwi_dev_free(bd)
        L.fwi_dev_free(xd)


__all__ = ["GnState", "KktVector", "PrecondMode", "FsgnOptions", "ConvergenceLog", "kkt_apply",
           "kkt_rhs", "precond_apply", "fsgn_gmres_step", "gmres", "dot", "norm", "axpy", "scal",
           "FwiError", "InvalidArgument", "SingularPivotError", "ZeroPivotError", "CudaError"]
