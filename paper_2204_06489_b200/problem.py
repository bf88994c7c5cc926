"""Problem descriptions (grid, PML profile, survey, model) and the seeded
synthetic BASELINE configurations.

Mirrors the reference's value types: Grid2D / PmlProfile
(include/fwi/grid.hpp:11-42), Survey (include/fwi/forward.hpp:16-33),
SlownessModel (include/fwi/helmholtz.hpp:13-19) and the GnState inputs of
make_gn_state (include/fwi/reduced_space.hpp:43-54). No public dataset is used:
every configuration below is generated from a seed with the shapes and value
distributions BASELINE.json states (decisions it leaves open follow
SURVEY.md §8(d) and are listed in DESIGN.md).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _abi


@dataclass
class Grid:
    """fwi::Grid2D (grid.hpp:11-35) + fwi::PmlProfile (grid.hpp:40-43)."""
    nx: int
    nz: int
    h: float
    n_pml: int
    sigma_max: float = 0.0
    power: float = 2.0

    @property
    def n(self) -> int:
        return self.nx * self.nz

    def index(self, ix: int, iz: int) -> int:
        return iz * self.nx + ix

    def on_boundary(self, ix: int, iz: int) -> bool:
        return ix == 0 or iz == 0 or ix == self.nx - 1 or iz == self.nz - 1

    def in_core(self, ix: int, iz: int) -> bool:
        p = self.n_pml
        return p <= ix < self.nx - p and p <= iz < self.nz - p

    def usable_node(self, ix: int, iz: int) -> bool:
        return self.in_core(ix, iz) and not self.on_boundary(ix, iz)

    @property
    def core_nx(self) -> int:
        return self.nx - 2 * self.n_pml

    def validate(self) -> None:
        """build_grid's checks (src/grid.cpp:9-19)."""
        if self.nx < 3 or self.nz < 3:
            raise ValueError("build_grid: need nx >= 3 and nz >= 3")
        if not self.h > 0:
            raise ValueError("build_grid: spacing h must be positive")
        if self.n_pml < 0:
            raise ValueError("build_grid: n_pml must be non-negative")
        if 2 * self.n_pml >= min(self.nx, self.nz):
            raise ValueError("build_grid: PML frame consumes the whole domain")


def pml_sigma_max(grid: Grid, c_ref: float) -> float:
    """make_pml_profile (src/grid.cpp:21-33): sigma_max = 3 c_ref ln(1e3) / (2 L_pml).
    Evaluated with the same IEEE operations in the same order."""
    if not c_ref > 0:
        raise ValueError("make_pml_profile: c_ref must be positive")
    if grid.n_pml == 0:
        return 0.0
    l_pml = grid.n_pml * grid.h
    return 3.0 * c_ref * math.log(1e3) / (2.0 * l_pml)


def omega_of(freq_hz: float) -> float:
    """st.omega = 2*pi*f (src/reduced_space.cpp:55)."""
    return 2.0 * math.pi * freq_hz


@dataclass
class Survey:
    """fwi::Survey flattened: per-source position/amplitude + receiver lists."""
    src_ix: np.ndarray
    src_iz: np.ndarray
    recv_offset: np.ndarray
    recv_ix: np.ndarray
    recv_iz: np.ndarray
    src_amp: np.ndarray | None = None
    weight_mode: int = _abi.FWI_WEIGHT_IDENTITY

    @property
    def num_sources(self) -> int:
        return int(self.src_ix.size)

    @property
    def num_data(self) -> int:
        return int(self.recv_offset[-1])

    @staticmethod
    def shared(src: list[tuple[int, int]], recv: list[tuple[int, int]], **kw) -> "Survey":
        k = len(src)
        r = len(recv)
        return Survey(
            src_ix=np.array([s[0] for s in src], np.int32),
            src_iz=np.array([s[1] for s in src], np.int32),
            recv_offset=np.arange(k + 1, dtype=np.int32) * r,
            recv_ix=np.tile(np.array([p[0] for p in recv], np.int32), k),
            recv_iz=np.tile(np.array([p[1] for p in recv], np.int32), k), **kw)

    @staticmethod
    def per_source(src: list[tuple[int, int]], recvs: list[list[tuple[int, int]]], **kw) -> "Survey":
        off = np.zeros(len(src) + 1, np.int32)
        off[1:] = np.cumsum([len(r) for r in recvs])
        flat = [p for r in recvs for p in r]
        return Survey(
            src_ix=np.array([s[0] for s in src], np.int32),
            src_iz=np.array([s[1] for s in src], np.int32),
            recv_offset=off,
            recv_ix=np.array([p[0] for p in flat] or [0], np.int32)[: len(flat)].copy(),
            recv_iz=np.array([p[1] for p in flat] or [0], np.int32)[: len(flat)].copy(), **kw)

    def weights(self) -> np.ndarray:
        """build_weights (src/forward.cpp:43-62)."""
        w = np.ones(self.num_data)
        if self.weight_mode == _abi.FWI_WEIGHT_IDENTITY:
            return w
        for k in range(self.num_sources):
            for j in range(self.recv_offset[k], self.recv_offset[k + 1]):
                dx = float(self.recv_ix[j] - self.src_ix[k])
                dz = float(self.recv_iz[j] - self.src_iz[k])
                w[j] = math.sqrt(dx * dx + dz * dz)
        mx = w.max() if w.size else 0.0
        return w / mx if mx > 0 else w


@dataclass
class Problem:
    """Everything make_gn_state consumes, as host arrays."""
    grid: Grid
    survey: Survey
    freq_hz: float
    epsilon: float
    s: np.ndarray                      # squared slowness, n
    drop_reg_term: bool = False
    u: np.ndarray | None = None        # K*n complex128 (source-major) or None
    r: np.ndarray | None = None        # num_data complex128
    d_obs: np.ndarray | None = None    # num_data complex128
    s_true: np.ndarray | None = None   # the truth model (for simulating d_obs)
    name: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return self.grid.n

    @property
    def K(self) -> int:
        return self.survey.num_sources

    @property
    def omega(self) -> float:
        return omega_of(self.freq_hz)

    @property
    def vec_len(self) -> int:
        """Doubles in one flat KKT vector: 4*K*n + n."""
        return 4 * self.K * self.n + self.n

    def desc(self, *, exact_factor: bool = False, ilu_level: int = -1, ilu_diag_shift: float = 0.0,
             precision_mask: int = 0, with_u: bool = True, with_r: bool = True,
             with_dobs: bool = True):
        """Build a StateDesc; returns (desc, keepalive)."""
        g, sv = self.grid, self.survey
        keep = []

        def arr(a, dt):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dtype=dt)
            keep.append(a)
            return a

        s = arr(self.s, np.float64)
        u = arr(self.u, np.complex128) if with_u else None
        r = arr(self.r, np.complex128) if with_r else None
        dobs = arr(self.d_obs, np.complex128) if with_dobs else None
        sx, sz = arr(sv.src_ix, np.int32), arr(sv.src_iz, np.int32)
        ro, rx, rz = arr(sv.recv_offset, np.int32), arr(sv.recv_ix, np.int32), arr(sv.recv_iz, np.int32)
        amp = arr(sv.src_amp, np.float64)
        d = _abi.StateDesc()
        d.grid = _abi.GridDesc(g.nx, g.nz, g.h, g.n_pml, g.sigma_max, g.power)
        d.survey = _abi.SurveyDesc(sv.num_sources, _abi.iptr(sx), _abi.iptr(sz), _abi.dptr(amp),
                                   _abi.iptr(ro), _abi.iptr(rx), _abi.iptr(rz), sv.weight_mode)
        d.freq_hz = self.freq_hz
        d.epsilon = self.epsilon
        d.drop_reg_term = int(bool(self.drop_reg_term))
        d.s = _abi.dptr(s)
        d.u = _abi.dptr(u)
        d.r = _abi.dptr(r)
        d.d_obs = _abi.dptr(dobs)
        d.exact_factor = int(bool(exact_factor))
        d.ilu_level = int(ilu_level)
        d.ilu_diag_shift = float(ilu_diag_shift)
        d.precision_mask = int(precision_mask)
        return d, keep


# --------------------------------------------------------------------------
# seeded synthetic inputs
# --------------------------------------------------------------------------

def _gauss_smooth(a: np.ndarray, sigma: float) -> np.ndarray:
    from scipy.ndimage import gaussian_filter
    return gaussian_filter(a, sigma=sigma, mode="nearest")


def random_kkt(p: Problem, seed: int, dtype=np.float64) -> np.ndarray:
    """Flat KKT vector with du, lambda ~ CN (re, im each N(0,1)) and ds ~ N(0,1)
    (BASELINE config 2's input distribution)."""
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(p.vec_len)
    return v.astype(dtype)


def c1_problem(seed: int = 1234) -> Problem:
    """BASELINE config 1: 128x64, h=25 m, 10-cell PML, 5 Hz, 8 sources, 64 receivers.

    Rows: "z=2" lies inside the PML (rejected by Survey::validate,
    src/forward.cpp:23-41), so sources/receivers use the core-relative row
    iz = n_pml + 2. Receivers: 64 distinct core nodes
    (every 2nd node of the row cannot fit 64 in the 108-node core).
    eps = 1e10 with drop_reg_term (the reference default eps=1
    does not converge)."""
    g = Grid(128, 64, 25.0, 10)
    rng = np.random.default_rng(seed)
    iz = np.arange(g.nz)[:, None] * np.ones((1, g.nx))
    ixg = np.ones((g.nz, 1)) * np.arange(g.nx)[None, :]
    v = 1500.0 + 2000.0 * iz / (g.nz - 1)
    for _ in range(3):
        cx = rng.uniform(g.n_pml + 10, g.nx - g.n_pml - 10)
        cz = rng.uniform(g.n_pml + 8, g.nz - g.n_pml - 5)
        sign = 1.0 if rng.uniform() < 0.5 else -1.0
        v = v * (1.0 + sign * 0.10 * np.exp(-((ixg - cx) ** 2 + (iz - cz) ** 2) / (2 * 5.0 ** 2)))
    v0 = _gauss_smooth(v, 10.0)
    g.sigma_max = pml_sigma_max(g, float(v0.mean()))
    row = g.n_pml + 2
    src = [(g.n_pml + int(round((k + 0.5) * g.core_nx / 8)), row) for k in range(8)]
    rec = [(g.n_pml + (j * g.core_nx) // 64, row) for j in range(64)]
    sv = Survey.shared(src, rec)
    return Problem(grid=g, survey=sv, freq_hz=5.0, epsilon=1e10, drop_reg_term=True,
                   s=(1.0 / v0 ** 2).ravel(), s_true=(1.0 / v ** 2).ravel(), name="C1",
                   meta={"v_true": v, "v0": v0})


def c2_problem(seed: int = 2024, K: int = 64, R: int = 256) -> Problem:
    """BASELINE config 2: 512x256, 20-cell PML, 8 Hz, 64 sources / 256 receivers on the
    top core row. h = 20 m (unstated). v = 1500->4500 linear plus a seeded +/-5%
    i.i.d. field smoothed with a 4-cell Gaussian. u_k and r are seeded CN(0,1)
    (the apply's cost and arithmetic do not depend on the physics)."""
    g = Grid(512, 256, 20.0, 20)
    rng = np.random.default_rng(seed)
    iz = np.arange(g.nz)[:, None] * np.ones((1, g.nx))
    pert = _gauss_smooth(rng.standard_normal((g.nz, g.nx)), 4.0)
    pert *= 0.05 / np.abs(pert).max()
    v = (1500.0 + 3000.0 * iz / (g.nz - 1)) * (1.0 + pert)
    g.sigma_max = pml_sigma_max(g, float(v.mean()))
    row = g.n_pml
    src = [(g.n_pml + int(round((k + 0.5) * g.core_nx / K)), row) for k in range(K)]
    rec = [(g.n_pml + (j * g.core_nx) // R, row) for j in range(R)]
    sv = Survey.shared(src, rec)
    u = (rng.standard_normal((K, g.n)) + 1j * rng.standard_normal((K, g.n))).ravel()
    r = rng.standard_normal(sv.num_data) + 1j * rng.standard_normal(sv.num_data)
    return Problem(grid=g, survey=sv, freq_hz=8.0, epsilon=1.0, s=(1.0 / v ** 2).ravel(),
                   u=u, r=r, name="C2")


def layered_fault_velocity(nx: int, nz: int, seed: int, water_cells: int = 10, n_layers: int = 40,
                           n_faults: int = 3, vmin: float = 1500.0, vmax: float = 4700.0,
                           fault_throw=(5, 15)) -> np.ndarray:
    """Marmousi-like synthetic section (BASELINE config 3): a water layer at 1500 m/s,
    `n_layers` seeded dipping layers with velocities drawn from U(vmin, vmax) and
    sorted to trend upward with depth, and `n_faults` seeded normal faults whose
    hanging wall is shifted down by 5-15 cells. The reference has only layered and
    lens generators (src/model_io.cpp:437-487), so this one is ours."""
    rng = np.random.default_rng(seed)
    depth = nz - water_cells
    vel_layers = np.sort(rng.uniform(vmin, vmax, n_layers))
    # interface depths (cells below the water) and per-interface dips (cells per column)
    tops = np.sort(rng.uniform(0, depth, n_layers - 1))
    dips = rng.uniform(-0.08, 0.08, n_layers - 1)
    ix = np.arange(nx)[None, :]
    iz = np.arange(depth)[:, None].astype(float)
    # layer index at (z, x): number of interfaces above
    layer = np.zeros((depth, nx), np.int64)
    for t, d in zip(tops, dips):
        layer += (iz >= t + d * (ix - nx / 2)).astype(np.int64)
    v = vel_layers[np.clip(layer, 0, n_layers - 1)]
    for _ in range(n_faults):  # normal faults: shift the hanging wall down
        x0 = rng.uniform(0.15 * nx, 0.85 * nx)
        slope = rng.uniform(0.4, 1.2) * (1 if rng.uniform() < 0.5 else -1)
        throw = int(rng.integers(fault_throw[0], fault_throw[1] + 1))
        hang = (ix - x0) * slope > iz - depth / 2 + 0 * ix  # one side of a dipping fault plane
        hang = np.broadcast_to(hang, (depth, nx))
        shifted = np.empty_like(v)
        shifted[throw:] = v[:-throw]
        shifted[:throw] = v[:1]
        v = np.where(hang, shifted, v)
    out = np.empty((nz, nx))
    out[:water_cells] = 1500.0
    out[water_cells:] = v
    return out


def c3_problem(freq_hz: float = 3.0, seed: int = 33, K: int = 48, R: int = 192, nx: int = 384, nz: int = 128,
               h: float = 20.0, n_pml: int = 20) -> Problem:
    """BASELINE config 3/4: 384x128, h=20 m, ⚑ 20-cell PML, 10-cell water layer, 40 seeded
    dipping layers and 3 normal faults; 48 sources and 192 receivers on the top core
    row; the start model is the truth smoothed with a 10-cell Gaussian; frequencies
    3, 5, 7 Hz. ⚑ eps calibrated as in config 1 (1e10 with drop_reg_term)."""
    g = Grid(nx, nz, h, n_pml)
    vt = layered_fault_velocity(nx, nz, seed)
    v0 = _gauss_smooth(vt, 10.0)
    v0[:10] = 1500.0
    g.sigma_max = pml_sigma_max(g, float(v0.mean()))
    row = g.n_pml + 1
    src = [(g.n_pml + 1 + int(round((k + 0.5) * (g.core_nx - 2) / K)), row) for k in range(K)]
    rec = [(g.n_pml + 1 + (j * (g.core_nx - 2)) // R, row) for j in range(R)]
    sv = Survey.shared(src, rec)
    return Problem(grid=g, survey=sv, freq_hz=freq_hz, epsilon=1e10, drop_reg_term=True,
                   s=(1.0 / v0 ** 2).ravel(), s_true=(1.0 / vt ** 2).ravel(), name="C3",
                   meta={"v_true": vt, "v0": v0})


def c5_problem(freq_hz: float = 10.0, seed: int = 55, K: int = 256, R: int = 1024, nx: int = 2048,
               nz: int = 1024, h: float = 10.0, n_pml: int = 30, with_u: bool = False) -> Problem:
    """BASELINE config 5: 2048x1024, h=10 m, 30-cell PML, 10 Hz, 256 surface sources and
    1024 receivers on the top core row; the model is config 3's construction scaled to
    this grid (water layer, dipping layers, fault throws and the start-model smoothing
    all x8 in cells, i.e. the same depths in metres at half the spacing).
    ⚑ eps calibrated as for config 1, eps ~ 1e-2 ||J^H W^T W J||: the power-iteration
    estimate at the start model is 1.1e14 (tools/jhj_norm.py), so eps = 1e12 with
    drop_reg_term. With `with_u`, u_k and r are seeded CN(0,1) (8.6 GB of host memory)
    for apply-only measurements, as in config 2."""
    g = Grid(nx, nz, h, n_pml)
    sc = nz / 128.0
    vt = layered_fault_velocity(nx, nz, seed, water_cells=int(round(10 * sc)),
                                fault_throw=(int(round(5 * sc)), int(round(15 * sc))))
    v0 = _gauss_smooth(vt, 10.0 * sc)
    v0[:int(round(10 * sc))] = 1500.0
    g.sigma_max = pml_sigma_max(g, float(v0.mean()))
    row = g.n_pml + 1
    src = [(g.n_pml + 1 + int(round((k + 0.5) * (g.core_nx - 2) / K)), row) for k in range(K)]
    rec = [(g.n_pml + 1 + (j * (g.core_nx - 2)) // R, row) for j in range(R)]
    sv = Survey.shared(src, rec)
    u = r = None
    if with_u:
        rng = np.random.default_rng(seed + 1)
        u = rng.standard_normal(2 * K * g.n).view(np.complex128)
        r = rng.standard_normal(2 * sv.num_data).view(np.complex128)
    return Problem(grid=g, survey=sv, freq_hz=freq_hz, epsilon=1e12, drop_reg_term=True,
                   s=(1.0 / v0 ** 2).ravel(), s_true=(1.0 / vt ** 2).ravel(), u=u, r=r, name="C5",
                   meta={"v_true": vt, "v0": v0})


def small_problem(nx=24, nz=18, n_pml=3, K=3, R=5, freq=6.0, h=20.0, seed=7, eps=1e-2,
                  duplicate_receiver=False, weight_mode=_abi.FWI_WEIGHT_IDENTITY) -> Problem:
    """Small desk-scale instance for parity tests (seconds on the CPU oracle)."""
    g = Grid(nx, nz, h, n_pml)
    rng = np.random.default_rng(seed)
    v = 2000.0 + 300.0 * rng.standard_normal((nz, nx)).clip(-2, 2)
    v = _gauss_smooth(v, 1.5)
    g.sigma_max = pml_sigma_max(g, float(v.mean()))
    row = n_pml + 1
    src = [(n_pml + 1 + (k * (g.core_nx - 3)) // max(K - 1, 1), row) for k in range(K)]
    recvs = []
    for k in range(K):
        rr = [(n_pml + 1 + (j * (g.core_nx - 3)) // max(R - 1, 1), nz - n_pml - 2) for j in range(R)]
        if duplicate_receiver and rr:
            rr.append(rr[0])
        recvs.append(rr)
    sv = Survey.per_source(src, recvs, weight_mode=weight_mode)
    u = (rng.standard_normal((K, g.n)) + 1j * rng.standard_normal((K, g.n))).ravel()
    r = rng.standard_normal(sv.num_data) + 1j * rng.standard_normal(sv.num_data)
    return Problem(grid=g, survey=sv, freq_hz=freq, epsilon=eps, s=(1.0 / v ** 2).ravel(),
                   u=u, r=r, name=f"small{nx}x{nz}")


def standard_instance() -> Problem:
    """fixtures::standard_instance (tests/support/fixtures.hpp:48-81) restated:
    12x12, h=1, n_pml=2, c_ref=1, 0.15 Hz, 2 sources x 6 receivers, eps=1e-2;
    truth = lens (make_lens_model, src/model_io.cpp:465-487), start = constant 1."""
    g = Grid(12, 12, 1.0, 2)
    g.sigma_max = pml_sigma_max(g, 1.0)
    ix = np.arange(12)[None, :].astype(float)
    iz = np.arange(12)[:, None].astype(float)
    vt = 1.0 + 0.15 * np.exp(-((ix - 5.5) ** 2 + (iz - 5.5) ** 2) / (2.0 * 2.0 * 2.0))
    recv = [(x, 8) for x in range(3, 9)]
    sv = Survey.per_source([(3, 3), (8, 3)], [recv, recv])
    return Problem(grid=g, survey=sv, freq_hz=0.15, epsilon=1e-2, s=np.ones(g.n),
                   s_true=(1.0 / vt ** 2).ravel(), name="standard")


def no_receiver_instance() -> Problem:
    """no_receiver_instance (tests/test_kkt.cpp:29-46): two sources, no receivers."""
    g = Grid(12, 12, 1.0, 2)
    g.sigma_max = pml_sigma_max(g, 1.0)
    sv = Survey.per_source([(5, 5), (7, 6)], [[], []])
    return Problem(grid=g, survey=sv, freq_hz=0.15, epsilon=1e-2, s=np.ones(g.n),
                   r=np.zeros(0, np.complex128), d_obs=np.zeros(0, np.complex128), name="norecv")


def cancelling_slowness(freq_hz: float) -> float:
    """Squared slowness whose stencil diagonal 4/h^2 - w^2 s X Z cancels exactly on an h = 1
    grid without PML (X = Z = 1): fl(w^2 * s) == 4 (assemble_helmholtz, src/helmholtz.cpp:52-53)."""
    w2 = omega_of(freq_hz) ** 2
    s = 4.0 / w2
    for _ in range(64):
        if w2 * s == 4.0:
            return s
        s = math.nextafter(s, 0.0 if w2 * s > 4.0 else 10.0)
    raise RuntimeError("no exactly cancelling slowness found")


def zero_pivot_instance(freq_hz: float = 0.15) -> Problem:
    """A Helmholtz instance with an exact zero ILU pivot (tests/test_ilu.cpp:107-120 on a real
    operator): 7x6 grid, h = 1, no PML, node (1,1)'s diagonal cancels exactly; its earlier
    neighbours are Dirichlet, so its ILU pivot is the bare diagonal -> ZeroPivotError(8).
    The full operator is nonsingular (the exact LU pivots past it)."""
    g = Grid(7, 6, 1.0, 0, sigma_max=0.0)
    s = np.ones(g.n)
    s[g.index(1, 1)] = cancelling_slowness(freq_hz)
    sv = Survey.per_source([(3, 3)], [[(4, 3), (2, 4)]])
    K = 1
    u = np.linspace(0.1, 1.0, K * g.n) * (1.0 - 0.5j)
    return Problem(grid=g, survey=sv, freq_hz=freq_hz, epsilon=1.0, s=s, u=u,
                   r=np.array([0.5 - 0.25j, -0.125 + 1.0j]), name="zero_pivot")


def singular_instance(freq_hz: float = 0.15) -> Problem:
    """A singular Helmholtz operator with a zero row (tests/test_lu.cpp:44-47 on a real
    operator): 3x3 grid, h = 1, no PML; the only interior node's couplings all go to
    Dirichlet columns and its diagonal cancels -> SingularPivotError(4)."""
    g = Grid(3, 3, 1.0, 0, sigma_max=0.0)
    s = np.ones(g.n)
    s[g.index(1, 1)] = cancelling_slowness(freq_hz)
    sv = Survey.per_source([(1, 1)], [[(1, 1)]])
    return Problem(grid=g, survey=sv, freq_hz=freq_hz, epsilon=1.0, s=s, u=np.ones(g.n, np.complex128),
                   r=np.ones(1, np.complex128), name="singular")
