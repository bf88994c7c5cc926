"""TEST INFRASTRUCTURE ONLY — Python bindings of the two CPU checkers:

* ``Ref``  : the unmodified reference core (oracle/_ref/libfwiref.so, built by
             oracle/Makefile from /root/reference/proj/src + ref_harness.cpp);
* ``Orc``  : our plain-C restatement (oracle/liboracle.so from fwi_oracle.c).

Only tests/, __graft_entry__.smoke() (as the checker) and bench.py's
cpu_baseline / ``--impl reference`` leg import this module. The product
package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2204_06489_b200 import _abi
from paper_2204_06489_b200.problem import Problem

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libfwiref.so")
ORC_SO = os.path.join(HERE, "liboracle.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


def build(quiet: bool = True) -> None:
    """Compile the checkers (make -C oracle). The reference part is skipped
    when /root/reference is absent (GPU box): the prebuilt _ref travels."""
    out = subprocess.run(["make", "-C", HERE, "all", "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout[-4000:] + out.stderr[-4000:])


def _load(path: str) -> C.CDLL:
    if not os.path.exists(path):
        build()
    return C.CDLL(path)


_ref_lib = None
_orc_lib = None


def ref_lib() -> C.CDLL:
    global _ref_lib
    if _ref_lib is None:
        lib = _load(REF_SO)
        vp = C.c_void_p
        lib.ref_last_error.restype = C.c_char_p
        for name, args in {
            "ref_make_state": [C.c_void_p, C.POINTER(vp)],
            "ref_make_state_direct": [C.c_void_p, C.POINTER(vp)],
            "ref_kkt_apply": [vp, _dp, _dp],
            "ref_kkt_rhs": [vp, _dp],
            "ref_precond_apply": [vp, C.c_int, _dp, _dp],
            "ref_solve": [vp, C.c_int, C.c_int, _dp, _dp],
            "ref_fsgn": [vp, C.c_void_p, _dp, C.c_void_p],
            "ref_simulate": [C.c_void_p, _dp],
            "ref_gradient": [vp, _dp],
            "ref_hessian_apply": [vp, _dp, _dp],
            "ref_ilu_factor_status": [vp, C.c_int, C.c_double],
            "ref_kkt_apply_bench": [vp, _dp, C.c_int, C.c_int, _dp],
            "ref_ilu_export": [vp, _ip, _ip, _ip, _ip, _dp, _ip, _ip, _dp],
            "ref_rsgn": [vp, C.c_double, C.c_int, _dp, C.c_void_p],
            "ref_gn_step": [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                            C.c_double, C.c_double, _dp, _dp, _dp, C.c_void_p],
        }.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = C.c_int
        lib.ref_free.argtypes = [vp]
        lib.ref_free.restype = None
        lib.ref_state_info.argtypes = [vp, _ip, _ip, _ip, _ip, _dp]
        lib.ref_state_info.restype = None
        for name in ("ref_get_u", "ref_get_residual", "ref_get_dpred"):
            getattr(lib, name).argtypes = [vp, _dp]
            getattr(lib, name).restype = None
        lib.ref_get_csr.argtypes = [vp, _ip, _ip, _dp]
        lib.ref_get_csr.restype = None
        lib.ref_solve_count.argtypes = [vp, C.c_int]
        lib.ref_solve_count.restype = C.c_longlong
        lib.ref_reset_solve_count.argtypes = [vp, C.c_int]
        lib.ref_reset_solve_count.restype = None
        lib.ref_set_epsilon.argtypes = [vp, C.c_double]
        lib.ref_set_drop.argtypes = [vp, C.c_int]
        _ref_lib = lib
    return _ref_lib


class CheckerError(RuntimeError):
    def __init__(self, code: int, msg: str, index: int = -1):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.index = index


def _ck(lib, code: int, prefix="ref"):
    if code != 0:
        msg = getattr(lib, f"{prefix}_last_error")().decode()
        raise CheckerError(code, msg, getattr(lib, f"{prefix}_last_error_index")())


def _p(a):
    return a.ctypes.data_as(_dp)


class Ref:
    """A reference fwi::GnState driven through the reference's own API."""

    def __init__(self, p: Problem, *, full: bool = True, exact: bool = True, ilu_level: int = -1,
                 ilu_shift: float = 0.0):
        lib = ref_lib()
        self.lib, self.p = lib, p
        d, self._keep = p.desc(exact_factor=exact, ilu_level=ilu_level, ilu_diag_shift=ilu_shift)
        h = C.c_void_p()
        fn = lib.ref_make_state if full else lib.ref_make_state_direct
        _ck(lib, fn(C.byref(d), C.byref(h)))
        self.h = h
        n, K, nd, nnz = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        om = C.c_double()
        lib.ref_state_info(h, C.byref(n), C.byref(K), C.byref(nd), C.byref(nnz), C.byref(om))
        self.n, self.K, self.num_data, self.nnz, self.omega = n.value, K.value, nd.value, nnz.value, om.value

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_free(self.h)
            self.h = None

    @property
    def vec_len(self):
        return 4 * self.K * self.n + self.n

    def u(self):
        out = np.empty(self.K * self.n, np.complex128)
        self.lib.ref_get_u(self.h, _p(out))
        return out

    def residual(self):
        out = np.empty(self.num_data, np.complex128)
        self.lib.ref_get_residual(self.h, _p(out))
        return out

    def dpred(self):
        out = np.empty(self.num_data, np.complex128)
        self.lib.ref_get_dpred(self.h, _p(out))
        return out

    def csr(self):
        rp = np.empty(self.n + 1, np.int32)
        ci = np.empty(self.nnz, np.int32)
        va = np.empty(self.nnz, np.complex128)
        self.lib.ref_get_csr(self.h, rp.ctypes.data_as(_ip), ci.ctypes.data_as(_ip), _p(va))
        return rp, ci, va

    def set_epsilon(self, e):
        self.lib.ref_set_epsilon(self.h, e)

    def set_drop(self, d):
        self.lib.ref_set_drop(self.h, int(d))

    def kkt_apply(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty(self.vec_len)
        _ck(self.lib, self.lib.ref_kkt_apply(self.h, _p(x), _p(out)))
        return out

    def kkt_rhs(self) -> np.ndarray:
        out = np.empty(self.vec_len)
        _ck(self.lib, self.lib.ref_kkt_rhs(self.h, _p(out)))
        return out

    def precond_apply(self, x: np.ndarray, mode: int) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty(self.vec_len)
        _ck(self.lib, self.lib.ref_precond_apply(self.h, mode, _p(x), _p(out)))
        return out

    def solve(self, b: np.ndarray, mode: int, adjoint: bool) -> np.ndarray:
        b = np.ascontiguousarray(b, np.complex128)
        out = np.empty(self.n, np.complex128)
        _ck(self.lib, self.lib.ref_solve(self.h, mode, int(adjoint), _p(b), _p(out)))
        return out

    def solve_count(self, mode):
        return self.lib.ref_solve_count(self.h, mode)

    def reset_solve_count(self, mode):
        self.lib.ref_reset_solve_count(self.h, mode)

    def gradient(self):
        out = np.empty(self.n)
        _ck(self.lib, self.lib.ref_gradient(self.h, _p(out)))
        return out

    def hessian_apply(self, v):
        v = np.ascontiguousarray(v, np.float64)
        out = np.empty(self.n)
        _ck(self.lib, self.lib.ref_hessian_apply(self.h, _p(v), _p(out)))
        return out

    def fsgn(self, mode=_abi.FWI_PRECOND_EXACT, restart=30, tol=1e-10, maxit=30, ecg_stride=0,
             ecg_stop_tol=0.0):
        o = _abi.FsgnOptions(mode, restart, tol, maxit, ecg_stride, ecg_stop_tol)
        ds = np.empty(self.n)
        lb = _abi.LogBuffer(maxit + 2)
        _ck(self.lib, self.lib.ref_fsgn(self.h, C.byref(o), _p(ds), C.byref(lb.c)))
        return ds, lb.to_log()

    def rsgn(self, tol, maxit):
        ds = np.empty(self.n)
        lb = _abi.LogBuffer(maxit + 2)
        _ck(self.lib, self.lib.ref_rsgn(self.h, tol, maxit, _p(ds), C.byref(lb.c)))
        return ds, lb.to_log()

    def ilu_factors(self):
        nl, nu = C.c_int(), C.c_int()
        z = None
        self.lib.ref_ilu_export(self.h, C.byref(nl), C.byref(nu), z, z, z, z, z, z)
        lp = np.empty(self.n + 1, np.int32)
        li = np.empty(nl.value, np.int32)
        lv = np.empty(nl.value, np.complex128)
        up = np.empty(self.n + 1, np.int32)
        ui = np.empty(nu.value, np.int32)
        uv = np.empty(nu.value, np.complex128)
        ip = lambda a: a.ctypes.data_as(_ip)  # noqa: E731
        self.lib.ref_ilu_export(self.h, C.byref(nl), C.byref(nu), ip(lp), ip(li), _p(lv), ip(up),
                                ip(ui), _p(uv))
        return (lp, li, lv), (up, ui, uv)

    def ilu_factor_status(self, level, shift):
        code = self.lib.ref_ilu_factor_status(self.h, level, shift)
        if code:
            return code, self.lib.ref_last_error_index()
        return 0, -1

    def bench_kkt_apply(self, x, nthreads, napplies):
        x = np.ascontiguousarray(x, np.float64)
        sec = C.c_double()
        _ck(self.lib, self.lib.ref_kkt_apply_bench(self.h, _p(x), nthreads, napplies, C.byref(sec)))
        return sec.value


def ref_simulate(p: Problem, s: np.ndarray | None = None) -> np.ndarray:
    """Observed data on model s (default p.s_true) via the reference LU."""
    lib = ref_lib()
    q = Problem(**{**p.__dict__, "s": p.s_true if s is None else s})
    d, keep = q.desc()
    out = np.empty(p.survey.num_data, np.complex128)
    _ck(lib, lib.ref_simulate(C.byref(d), _p(out)))
    return out


def ref_gn_step(p: Problem, solver=1, max_inner=30, inner_tol=1e-12, restart=30, ilu_level=4,
                v_min=300.0, v_max=8000.0):
    lib = ref_lib()
    d, keep = p.desc()
    s_out = np.empty(p.n)
    mi, mf = C.c_double(), C.c_double()
    lb = _abi.LogBuffer(max_inner + 2)
    _ck(lib, lib.ref_gn_step(C.byref(d), solver, max_inner, inner_tol, restart, ilu_level, v_min,
                             v_max, _p(s_out), C.byref(mi), C.byref(mf), C.byref(lb.c)))
    return s_out, mi.value, mf.value, lb.to_log()


# ---------------------------------------------------------------------------
# our plain-C restatement (oracle/fwi_oracle.c)
# ---------------------------------------------------------------------------
def orc_lib() -> C.CDLL:
    global _orc_lib
    if _orc_lib is None:
        lib = _load(ORC_SO)
        vp = C.c_void_p
        lib.orc_last_error.restype = C.c_char_p
        lib.orc_last_error_index.restype = C.c_int
        for name, args in {
            "orc_state_create": [C.c_void_p, C.POINTER(vp)],
            "orc_kkt_apply": [vp, _dp, _dp],
            "orc_kkt_rhs": [vp, _dp],
            "orc_precond_apply": [vp, C.c_int, _dp, _dp],
            "orc_solve": [vp, C.c_int, C.c_int, _dp, _dp],
            "orc_ilu_factor": [vp, C.c_int, C.c_double],
            "orc_gradient": [vp, _dp],
            "orc_hessian_apply": [vp, _dp, _dp],
            "orc_fsgn": [vp, C.c_void_p, _dp, C.c_void_p],
        }.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = C.c_int
        for name in ("orc_get_u", "orc_get_residual", "orc_get_dpred"):
            getattr(lib, name).argtypes = [vp, _dp]
            getattr(lib, name).restype = None
        lib.orc_get_csr.argtypes = [vp, _ip, _ip, _dp]
        lib.orc_get_csr.restype = None
        lib.orc_state_info.argtypes = [vp, _ip, _ip, _ip, _ip, _dp]
        lib.orc_state_info.restype = None
        lib.orc_state_free.argtypes = [vp]
        lib.orc_state_free.restype = None
        lib.orc_solve_count.argtypes = [vp, C.c_int]
        lib.orc_solve_count.restype = C.c_longlong
        lib.orc_set_epsilon.argtypes = [vp, C.c_double]
        lib.orc_set_epsilon.restype = None
        lib.orc_set_drop.argtypes = [vp, C.c_int]
        lib.orc_set_drop.restype = None
        _orc_lib = lib
    return _orc_lib


class Orc(Ref):
    """Same interface as Ref, backed by the plain-C restatement."""

    def __init__(self, p: Problem, *, exact: bool = True, ilu_level: int = -1, ilu_shift: float = 0.0):
        lib = orc_lib()
        self.lib, self.p = lib, p
        d, self._keep = p.desc(exact_factor=exact, ilu_level=ilu_level, ilu_diag_shift=ilu_shift)
        h = C.c_void_p()
        _ck(lib, lib.orc_state_create(C.byref(d), C.byref(h)), prefix="orc")
        self.h = h
        n, K, nd, nnz = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        om = C.c_double()
        lib.orc_state_info(h, C.byref(n), C.byref(K), C.byref(nd), C.byref(nnz), C.byref(om))
        self.n, self.K, self.num_data, self.nnz, self.omega = n.value, K.value, nd.value, nnz.value, om.value

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.orc_state_free(self.h)
            self.h = None

    def _c(self, code):
        _ck(self.lib, code, prefix="orc")

    def u(self):
        out = np.empty(self.K * self.n, np.complex128)
        self.lib.orc_get_u(self.h, _p(out))
        return out

    def residual(self):
        out = np.empty(max(self.num_data, 1), np.complex128)
        self.lib.orc_get_residual(self.h, _p(out))
        return out[: self.num_data]

    def dpred(self):
        out = np.empty(max(self.num_data, 1), np.complex128)
        self.lib.orc_get_dpred(self.h, _p(out))
        return out[: self.num_data]

    def csr(self):
        rp = np.empty(self.n + 1, np.int32)
        ci = np.empty(self.nnz, np.int32)
        va = np.empty(self.nnz, np.complex128)
        self.lib.orc_get_csr(self.h, rp.ctypes.data_as(_ip), ci.ctypes.data_as(_ip), _p(va))
        return rp, ci, va

    def set_epsilon(self, e):
        self.lib.orc_set_epsilon(self.h, e)

    def set_drop(self, d):
        self.lib.orc_set_drop(self.h, int(d))

    def kkt_apply(self, x):
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty(self.vec_len)
        self._c(self.lib.orc_kkt_apply(self.h, _p(x), _p(out)))
        return out

    def kkt_rhs(self):
        out = np.empty(self.vec_len)
        self._c(self.lib.orc_kkt_rhs(self.h, _p(out)))
        return out

    def precond_apply(self, x, mode):
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty(self.vec_len)
        self._c(self.lib.orc_precond_apply(self.h, mode, _p(x), _p(out)))
        return out

    def solve(self, b, mode, adjoint):
        b = np.ascontiguousarray(b, np.complex128)
        out = np.empty(self.n, np.complex128)
        self._c(self.lib.orc_solve(self.h, mode, int(adjoint), _p(b), _p(out)))
        return out

    def solve_count(self, mode):
        return self.lib.orc_solve_count(self.h, mode)

    def gradient(self):
        out = np.empty(self.n)
        self._c(self.lib.orc_gradient(self.h, _p(out)))
        return out

    def hessian_apply(self, v):
        v = np.ascontiguousarray(v, np.float64)
        out = np.empty(self.n)
        self._c(self.lib.orc_hessian_apply(self.h, _p(v), _p(out)))
        return out

    def ilu_factor_status(self, level, shift):
        code = self.lib.orc_ilu_factor(self.h, level, shift)
        return (code, self.lib.orc_last_error_index()) if code else (0, -1)

    def fsgn(self, mode=_abi.FWI_PRECOND_EXACT, restart=30, tol=1e-10, maxit=30, ecg_stride=0,
             ecg_stop_tol=0.0):
        o = _abi.FsgnOptions(mode, restart, tol, maxit, ecg_stride, ecg_stop_tol)
        ds = np.empty(self.n)
        lb = _abi.LogBuffer(maxit + 2)
        self._c(self.lib.orc_fsgn(self.h, C.byref(o), _p(ds), C.byref(lb.c)))
        return ds, lb.to_log()
