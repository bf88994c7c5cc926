// ref_harness.cpp — TEST INFRASTRUCTURE ONLY (checker, never shipped or measured
// as the product). An extern "C" harness over the UNMODIFIED reference library
// compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libfwiref.so. It lets the Python tests, the golden-vector script
// and bench.py's reference arm drive the reference's own public API
// (make_gn_state, kkt_apply, precond_apply, fsgn_gmres_step, gn_step, ...)
// on the same seeded inputs the CUDA path sees.
//
// Only tests/, __graft_entry__.smoke() (as checker) and bench.py's
// cpu_baseline / --impl reference leg load this library.
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <numbers>
#include <string>
#include <thread>
#include <vector>

#include "fwi/driver.hpp"
#include "fwi/kkt.hpp"
#include "fwi/model_io.hpp"
#include "fwi_b200.h"  // shared plain-C descriptor structs only

using namespace fwi;

namespace {

thread_local std::string g_err;
thread_local int g_err_index = -1;

struct RefCtx {
    GnState st;
};

int fail(const std::exception& e) {
    g_err = e.what();
    g_err_index = -1;
    if (auto* p = dynamic_cast<const SingularPivotError*>(&e)) {
        g_err_index = p->index;
        return FWI_ERR_SINGULAR_PIVOT;
    }
    if (auto* p = dynamic_cast<const ZeroPivotError*>(&e)) {
        g_err_index = p->index;
        return FWI_ERR_ZERO_PIVOT;
    }
    if (dynamic_cast<const std::invalid_argument*>(&e)) return FWI_ERR_INVALID_ARGUMENT;
    return FWI_ERR_NOT_SUPPORTED;
}

template <class F>
static int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

Grid2D grid_of(const fwi_grid_desc& g) { return build_grid(g.nx, g.nz, g.h, g.n_pml); }

PmlProfile profile_of(const fwi_grid_desc& g) {
    PmlProfile p;
    p.sigma_max = g.pml_sigma_max;
    p.power = g.pml_power;
    return p;
}

Survey survey_of(const fwi_survey_desc& s, double freq_hz) {
    Survey sv;
    sv.frequencies_hz = {freq_hz};
    sv.weight_mode = s.weight_mode == FWI_WEIGHT_OFFSET ? WeightMode::offset : WeightMode::identity;
    for (int k = 0; k < s.num_sources; ++k) {
        Survey::Source src;
        src.ix = s.src_ix[k];
        src.iz = s.src_iz[k];
        src.amplitude = s.src_amp ? s.src_amp[k] : 1.0;
        for (int j = s.recv_offset[k]; j < s.recv_offset[k + 1]; ++j)
            src.receivers.emplace_back(s.recv_ix[j], s.recv_iz[j]);
        sv.sources.push_back(std::move(src));
    }
    return sv;
}

ComplexVector cvec(const double* p, std::size_t n) {
    ComplexVector v(n);
    if (p) std::memcpy(static_cast<void*>(v.data()), p, n * sizeof(Complex));
    return v;
}

void put(const ComplexVector& v, double* out) {
    std::memcpy(out, static_cast<const void*>(v.data()), v.size() * sizeof(Complex));
}

KktVector from_flat(const GnState& st, const double* f) {
    const int K = st.num_sources(), n = st.model_size();
    KktVector v = KktVector::zeros(K, n, n);
    std::size_t off = 0;
    for (int k = 0; k < K; ++k, off += 2 * n)
        std::memcpy(static_cast<void*>(v.du[k].data()), f + off, n * sizeof(Complex));
    std::memcpy(v.ds.data(), f + off, n * sizeof(double));
    off += n;
    for (int k = 0; k < K; ++k, off += 2 * n)
        std::memcpy(static_cast<void*>(v.lambda[k].data()), f + off, n * sizeof(Complex));
    return v;
}

void to_flat(const KktVector& v, double* f) {
    const int n = static_cast<int>(v.ds.size());
    std::size_t off = 0;
    for (const auto& b : v.du) {
        put(b, f + off);
        off += 2 * n;
    }
    std::memcpy(f + off, v.ds.data(), n * sizeof(double));
    off += n;
    for (const auto& b : v.lambda) {
        put(b, f + off);
        off += 2 * n;
    }
}

void fill_log(const ConvergenceLog& lg, fwi_convergence_log* out) {
    if (!out) return;
    out->count = 0;
    for (const auto& e : lg.entries) {
        if (out->count >= out->capacity) break;
        fwi_log_entry& d = out->entries[out->count++];
        d.iteration = e.iteration;
        d.residual_norm = e.residual_norm;
        d.has_precond_residual = e.precond_residual.has_value();
        d.precond_residual = e.precond_residual.value_or(0.0);
        d.has_normal_residual = e.normal_residual.has_value();
        d.normal_residual = e.normal_residual.value_or(0.0);
        d.wall_time = e.wall_time;
    }
    out->converged = lg.converged;
    out->stagnated = lg.stagnated;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
int ref_last_error_index(void) { return g_err_index; }

// Full make_gn_state (src/reduced_space.cpp:40-86): assembly, exact LU,
// optional ILU, forward fields, residual from d_obs.
int ref_make_state(const fwi_state_desc* d, void** out) {
    try {
        const Grid2D grid = grid_of(d->grid);
        const Survey sv = survey_of(d->survey, d->freq_hz);
        SlownessModel m;
        m.s.assign(d->s, d->s + grid.num_nodes());
        GnStateOptions o;
        o.epsilon = d->epsilon;
        o.drop_reg_term = d->drop_reg_term != 0;
        o.weight_mode = sv.weight_mode;
        if (d->ilu_level >= 0) {
            o.ilu_level = d->ilu_level;
            o.ilu_diag_shift = d->ilu_diag_shift;
        }
        const DataVector dobs = cvec(d->d_obs, sv.num_data());
        auto c = std::make_unique<RefCtx>();
        c->st = make_gn_state(grid, profile_of(d->grid), m, sv, d->freq_hz, dobs, o);
        *out = c.release();
        return FWI_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// GnState built member by member without the LU (the C2 apply benchmark:
// u and r are given). ILU is built if requested.
int ref_make_state_direct(const fwi_state_desc* d, void** out) {
    try {
        const Grid2D grid = grid_of(d->grid);
        const Survey sv = survey_of(d->survey, d->freq_hz);
        auto c = std::make_unique<RefCtx>();
        GnState& st = c->st;
        st.grid = grid;
        st.profile = profile_of(d->grid);
        st.model.s.assign(d->s, d->s + grid.num_nodes());
        st.freq_hz = d->freq_hz;
        st.omega = 2.0 * std::numbers::pi * d->freq_hz;
        st.epsilon = d->epsilon;
        st.drop_reg_term = d->drop_reg_term != 0;
        st.survey = sv;
        st.weights = build_weights(sv, sv.weight_mode);
        st.op = assemble_helmholtz(grid, st.profile, st.model, st.omega);
        if (d->ilu_level >= 0)
            st.ilu = std::make_shared<IluFactors>(
                IluFactors::factor(st.op.a, d->ilu_level, d->ilu_diag_shift));
        if (d->exact_factor) st.lu = std::make_shared<LuFactors>(LuFactors::factor(st.op.a));
        const int n = grid.num_nodes();
        st.u.per_source.resize(sv.num_sources());
        for (int k = 0; k < sv.num_sources(); ++k)
            st.u.per_source[k] = cvec(d->u ? d->u + 2 * static_cast<std::size_t>(k) * n : nullptr, n);
        st.r = cvec(d->r, sv.num_data());
        st.d_obs = DataVector(sv.num_data(), 0.0);
        st.d_pred = DataVector(sv.num_data(), 0.0);
        st.offset = sv.data_offsets();
        for (const auto& s : sv.sources) {
            st.src_node.push_back(grid.index(s.ix, s.iz));
            std::vector<int> nodes;
            for (const auto& [rx, rz] : s.receivers) nodes.push_back(grid.index(rx, rz));
            st.recv_node.push_back(std::move(nodes));
        }
        *out = c.release();
        return FWI_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

void ref_free(void* h) { delete static_cast<RefCtx*>(h); }

void ref_state_info(void* h, int* n, int* K, int* ndata, int* nnz, double* omega) {
    const GnState& st = static_cast<RefCtx*>(h)->st;
    *n = st.model_size();
    *K = st.num_sources();
    *ndata = st.survey.num_data();
    *nnz = st.op.a.nnz();
    *omega = st.omega;
}

void ref_set_epsilon(void* h, double eps) { static_cast<RefCtx*>(h)->st.epsilon = eps; }
void ref_set_drop(void* h, int drop) { static_cast<RefCtx*>(h)->st.drop_reg_term = drop != 0; }

void ref_get_u(void* h, double* out) {
    const GnState& st = static_cast<RefCtx*>(h)->st;
    const int n = st.model_size();
    for (int k = 0; k < st.num_sources(); ++k)
        put(st.u.per_source[k], out + 2 * static_cast<std::size_t>(k) * n);
}
void ref_get_residual(void* h, double* out) { put(static_cast<RefCtx*>(h)->st.r, out); }
void ref_get_dpred(void* h, double* out) { put(static_cast<RefCtx*>(h)->st.d_pred, out); }

void ref_get_csr(void* h, int* row_ptr, int* col_idx, double* values) {
    const auto& a = static_cast<RefCtx*>(h)->st.op.a;
    std::memcpy(row_ptr, a.row_ptr.data(), a.row_ptr.size() * sizeof(int));
    std::memcpy(col_idx, a.col_idx.data(), a.col_idx.size() * sizeof(int));
    put(a.values, values);
}

int ref_kkt_apply(void* h, const double* in, double* out) {
    try {
        const GnState& st = static_cast<RefCtx*>(h)->st;
        to_flat(kkt_apply(st, from_flat(st, in)), out);
        return FWI_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_kkt_rhs(void* h, double* out) {
    try {
        to_flat(kkt_rhs(static_cast<RefCtx*>(h)->st), out);
        return FWI_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_precond_apply(void* h, int mode, const double* in, double* out) {
    try {
        const GnState& st = static_cast<RefCtx*>(h)->st;
        to_flat(precond_apply(st, from_flat(st, in),
                              mode == FWI_PRECOND_ILU ? PrecondMode::ilu : PrecondMode::exact),
                out);
        return FWI_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_solve(void* h, int mode, int adjoint, const double* in, double* out) {
    try {
        const GnState& st = static_cast<RefCtx*>(h)->st;
        const ComplexVector b = cvec(in, st.model_size());
        put(mode == FWI_PRECOND_ILU ? st.ilu->solve(b, adjoint != 0) : st.lu->solve(b, adjoint != 0),
            out);
        return FWI_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

long long ref_solve_count(void* h, int mode) {
    const GnState& st = static_cast<RefCtx*>(h)->st;
    if (mode == FWI_PRECOND_ILU) return st.ilu ? st.ilu->solve_count() : -1;
    return st.lu ? st.lu->solve_count() : -1;
}

void ref_reset_solve_count(void* h, int mode) {
    const GnState& st = static_cast<RefCtx*>(h)->st;
    if (mode == FWI_PRECOND_ILU && st.ilu) st.ilu->reset_solve_count();
    if (mode == FWI_PRECOND_EXACT && st.lu) st.lu->reset_solve_count();
}

// ILU factors in CSR (lower unit WITHOUT the implicit diagonal, upper with the
// diagonal first), for pinning the C restatement. Call with NULL arrays to get sizes.
int ref_ilu_export(void* h, int* nnz_l, int* nnz_u, int* lptr, int* lidx, double* lval,
                   int* uptr, int* uidx, double* uval) {
    const GnState& st = static_cast<RefCtx*>(h)->st;
    if (!st.ilu) return FWI_ERR_INVALID_ARGUMENT;
    const SparseMatrixCSR l = st.ilu->lower_unit();
    const SparseMatrixCSR u = st.ilu->upper();
    const int n = l.rows;
    *nnz_l = l.nnz() - n;
    *nnz_u = u.nnz();
    if (!lptr) return FWI_OK;
    int p = 0;
    lptr[0] = 0;
    for (int i = 0; i < n; ++i) {
        for (int q = l.row_ptr[i]; q < l.row_ptr[i + 1]; ++q) {
            if (l.col_idx[q] == i) continue;
            lidx[p] = l.col_idx[q];
            lval[2 * p] = l.values[q].real();
            lval[2 * p + 1] = l.values[q].imag();
            ++p;
        }
        lptr[i + 1] = p;
    }
    std::memcpy(uptr, u.row_ptr.data(), (n + 1) * sizeof(int));
    std::memcpy(uidx, u.col_idx.data(), u.nnz() * sizeof(int));
    put(u.values, uval);
    return FWI_OK;
}

// Standalone ILU factor of the state's operator with a given level/shift
// (reports ZeroPivotError like the reference).
int ref_ilu_factor_status(void* h, int level, double shift) {
    try {
        const GnState& st = static_cast<RefCtx*>(h)->st;
        (void)IluFactors::factor(st.op.a, level, shift);
        return FWI_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_gradient(void* h, double* out) {
    try {
        const RealVector g = gradient(static_cast<RefCtx*>(h)->st);
        std::memcpy(out, g.data(), g.size() * sizeof(double));
        return FWI_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_hessian_apply(void* h, const double* v, double* out) {
    try {
        const GnState& st = static_cast<RefCtx*>(h)->st;
        const RealVector r = hessian_apply(st, RealVector(v, v + st.model_size()));
        std::memcpy(out, r.data(), r.size() * sizeof(double));
        return FWI_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_fsgn(void* h, const fwi_fsgn_options* o, double* ds_out, fwi_convergence_log* log) {
    try {
        const GnState& st = static_cast<RefCtx*>(h)->st;
        FsgnOptions fo;
        fo.mode = o->mode == FWI_PRECOND_ILU ? PrecondMode::ilu : PrecondMode::exact;
        fo.restart = o->restart;
        fo.tol = o->tol;
        fo.maxit = o->maxit;
        fo.ecg_stride = o->ecg_stride;
        fo.ecg_stop_tol = o->ecg_stop_tol;
        const StepResult r = fsgn_gmres_step(st, fo);
        std::memcpy(ds_out, r.delta_s.data(), r.delta_s.size() * sizeof(double));
        fill_log(r.log, log);
        return FWI_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int ref_rsgn(void* h, double tol, int maxit, double* ds_out, fwi_convergence_log* log) {
    try {
        const StepResult r = rsgn_cg_step(static_cast<RefCtx*>(h)->st, tol, maxit);
        std::memcpy(ds_out, r.delta_s.data(), r.delta_s.size() * sizeof(double));
        fill_log(r.log, log);
        return FWI_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Forward data d = Q A(s)^{-1} f for the state's geometry at model s
// (fixtures::simulate_blocks, tests/support/fixtures.hpp:12-23).
int ref_simulate(const fwi_state_desc* d, double* d_out) {
    try {
        const Grid2D grid = grid_of(d->grid);
        const Survey sv = survey_of(d->survey, d->freq_hz);
        SlownessModel m;
        m.s.assign(d->s, d->s + grid.num_nodes());
        const double omega = 2.0 * std::numbers::pi * d->freq_hz;
        const HelmholtzOperator op = assemble_helmholtz(grid, profile_of(d->grid), m, omega);
        const LuFactors lu = LuFactors::factor(op.a);
        put(observe(grid, sv, solve_forward(lu, grid, sv)), d_out);
        return FWI_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// One reference gn_step (src/driver.cpp:65-127) at the desc's frequency.
int ref_gn_step(const fwi_state_desc* d, int solver, int max_inner, double inner_tol,
                int restart, int ilu_level, double v_min, double v_max, double* s_out,
                double* misfit_ini, double* misfit_fin, fwi_convergence_log* log) {
    try {
        FwiProblem p;
        p.grid = grid_of(d->grid);
        p.profile = profile_of(d->grid);
        p.survey = survey_of(d->survey, d->freq_hz);
        p.observed = {cvec(d->d_obs, p.survey.num_data())};
        SlownessModel m;
        m.s.assign(d->s, d->s + p.grid.num_nodes());
        FwiConfig cfg;
        cfg.solver = solver == 0   ? InnerSolver::rsgn_cg
                     : solver == 1 ? InnerSolver::fsgn_gmres_exact
                                   : InnerSolver::fsgn_gmres_ilu;
        cfg.max_inner = max_inner;
        cfg.inner_tol = inner_tol;
        cfg.gmres_restart = restart;
        cfg.ilu_level = ilu_level;
        cfg.drop_reg_term = d->drop_reg_term != 0;
        cfg.v_min = v_min;
        cfg.v_max = v_max;
        cfg.ecg_stride = 0;
        const GnStepResult r = gn_step(p, m, d->freq_hz, d->epsilon, cfg);
        std::memcpy(s_out, r.model.s.data(), r.model.s.size() * sizeof(double));
        *misfit_ini = r.misfit_ini;
        *misfit_fin = r.misfit_fin;
        fill_log(r.log, log);
        return FWI_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// CPU baseline: `napplies` kkt_apply calls spread over `nthreads` host
// threads (each call is the reference's serial kkt_apply; threads run
// independent applies on the shared read-only state). Returns wall seconds.
int ref_kkt_apply_bench(void* h, const double* in, int nthreads, int napplies, double* seconds) {
    try {
        const GnState& st = static_cast<RefCtx*>(h)->st;
        const KktVector xi = from_flat(st, in);
        std::atomic<int> next{0};
        std::atomic<bool> failed{false};
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int t = 0; t < nthreads; ++t) {
            pool.emplace_back([&] {
                try {
                    while (next.fetch_add(1) < napplies) {
                        KktVector out = kkt_apply(st, xi);
                        if (!std::isfinite(out.ds[0])) failed = true;
                    }
                } catch (...) {
                    failed = true;
                }
            });
        }
        for (auto& th : pool) th.join();
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return failed ? FWI_ERR_NOT_SUPPORTED : FWI_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}


// ---- on-disk formats (src/model_io.cpp): the reference's own writers and
// readers, for parity of paper_2204_06489_b200/model_io.py
int ref_format_double(double v, char* buf, int cap) {
    const std::string s = format_double(v);
    if (int(s.size()) + 1 > cap) return -1;
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return int(s.size());
}

int ref_write_model(const char* path, int nx, int nz, double h, int n_pml, int kind, const double* values) {
    return guard([&] {
        ModelFile m;
        m.grid = build_grid(nx, nz, h, n_pml);
        m.kind = kind ? ModelKind::slowness_sq : ModelKind::velocity_mps;
        m.values.assign(values, values + std::size_t(nx) * nz);
        write_model(path, m);
    });
}

// the reference's model generators (src/model_io.cpp:437-487): kind 0 layered, 1 lens;
// values out (nx*nz velocities)
int ref_make_model(int kind, int nx, int nz, double h, int n_pml, const double* vel, int nvel, const int* ifc,
                   int nifc, double bg, double amp, double cx, double cz, double rad, double* values) {
    return guard([&] {
        const Grid2D g = build_grid(nx, nz, h, n_pml);
        const ModelFile m = kind == 0 ? make_layered_model(g, std::vector<double>(vel, vel + nvel),
                                                           std::vector<int>(ifc, ifc + nifc))
                                      : make_lens_model(g, bg, amp, cx, cz, rad);
        std::memcpy(values, m.values.data(), m.values.size() * sizeof(double));
    });
}

int ref_write_heatmap(const char* path, int nx, int nz, double h, int n_pml, const double* values) {
    return guard([&] {
        const Grid2D g = build_grid(nx, nz, h, n_pml);
        write_heatmap(path, g, RealVector(values, values + std::size_t(nx) * nz));
    });
}

// status: 0 ok, 1 ParseError, 2 IoError, 3 other; header out = nx, nz, n_pml, kind; h; values (cap doubles)
int ref_read_model(const char* path, int* hdr, double* h, double* values, long cap) {
    try {
        const ModelFile m = read_model(path);
        hdr[0] = m.grid.nx;
        hdr[1] = m.grid.nz;
        hdr[2] = m.grid.n_pml;
        hdr[3] = m.kind == ModelKind::slowness_sq ? 1 : 0;
        *h = m.grid.h;
        if (values && long(m.values.size()) <= cap) std::memcpy(values, m.values.data(), m.values.size() * 8);
        return 0;
    } catch (const ParseError& e) {
        g_err = e.what();
        return 1;
    } catch (const IoError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

namespace {
Survey survey_from(int nf, const double* freqs, int weight_mode, int K, const int* sx, const int* sz,
                   const double* amp, const int* off, const int* rx, const int* rz) {
    Survey s;
    s.frequencies_hz.assign(freqs, freqs + nf);
    s.weight_mode = weight_mode ? WeightMode::offset : WeightMode::identity;
    for (int k = 0; k < K; ++k) {
        Survey::Source src;
        src.ix = sx[k];
        src.iz = sz[k];
        if (amp) src.amplitude = amp[k];
        for (int j = off[k]; j < off[k + 1]; ++j) src.receivers.emplace_back(rx[j], rz[j]);
        s.sources.push_back(src);
    }
    return s;
}
}  // namespace

int ref_write_survey(const char* path, int nf, const double* freqs, int weight_mode, int K, const int* sx,
                     const int* sz, const double* amp, const int* off, const int* rx, const int* rz) {
    return guard([&] { write_survey(path, survey_from(nf, freqs, weight_mode, K, sx, sz, amp, off, rx, rz)); });
}

// counts[0..3] = nf, weight_mode, K, num_data; arrays filled when non-null (capacities from a first call)
int ref_read_survey(const char* path, int* counts, double* freqs, int* sx, int* sz, double* amp, int* off, int* rx,
                    int* rz) {
    try {
        const Survey s = read_survey(path);
        counts[0] = int(s.frequencies_hz.size());
        counts[1] = s.weight_mode == WeightMode::offset ? 1 : 0;
        counts[2] = s.num_sources();
        counts[3] = s.num_data();
        if (freqs) {
            int j = 0;
            for (std::size_t i = 0; i < s.frequencies_hz.size(); ++i) freqs[i] = s.frequencies_hz[i];
            for (int k = 0; k < s.num_sources(); ++k) {
                sx[k] = s.sources[k].ix;
                sz[k] = s.sources[k].iz;
                amp[k] = s.sources[k].amplitude;
                off[k] = j;
                for (const auto& [a, b] : s.sources[k].receivers) {
                    rx[j] = a;
                    rz[j] = b;
                    ++j;
                }
            }
            off[s.num_sources()] = j;
        }
        return 0;
    } catch (const ParseError& e) {
        g_err = e.what();
        return 1;
    } catch (const IoError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

// blocks: nf x num_data complex (re, im)
int ref_write_data(const char* path, const char* survey_path, const double* blocks) {
    return guard([&] {
        const Survey s = read_survey(survey_path);
        std::vector<DataVector> b(s.frequencies_hz.size());
        const int nd = s.num_data();
        for (std::size_t f = 0; f < b.size(); ++f) {
            b[f].resize(nd);
            for (int j = 0; j < nd; ++j)
                b[f][j] = Complex(blocks[2 * (f * nd + j)], blocks[2 * (f * nd + j) + 1]);
        }
        write_data(path, s, b);
    });
}

int ref_read_data(const char* path, const char* survey_path, double* blocks) {
    try {
        const Survey s = read_survey(survey_path);
        const auto b = read_data(path, s);
        const int nd = s.num_data();
        for (std::size_t f = 0; f < b.size(); ++f)
            for (int j = 0; j < nd; ++j) {
                blocks[2 * (f * nd + j)] = b[f][j].real();
                blocks[2 * (f * nd + j) + 1] = b[f][j].imag();
            }
        return 0;
    } catch (const ParseError& e) {
        g_err = e.what();
        return 1;
    } catch (const IoError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

// FwiConfig fields: d[0..10] = epsilon_start, epsilon_end, inner_tol, ilu_diag_shift, v_min, v_max,
// ecg_stop_tol, pml_power, pml_c_ref (NaN if unset), pml_sigma_max (NaN if unset), unused;
// i[0..7] = solver, max_inner, gmres_restart, ilu_level, drop_reg_term, weight_mode (-1 unset),
// ecg_stride, nfreq; i[8] = neps; freqs / eps (capacity 64 each)
int ref_read_config(const char* path, double* d, int* i, double* freqs, double* eps) {
    try {
        const FwiConfig c = read_config(path);
        const double nan = std::nan("");
        d[0] = c.epsilon_start;
        d[1] = c.epsilon_end;
        d[2] = c.inner_tol;
        d[3] = c.ilu_diag_shift;
        d[4] = c.v_min;
        d[5] = c.v_max;
        d[6] = c.ecg_stop_tol;
        d[7] = c.pml_power;
        d[8] = c.pml_c_ref.value_or(nan);
        d[9] = c.pml_sigma_max.value_or(nan);
        i[0] = int(c.solver);
        i[1] = c.max_inner;
        i[2] = c.gmres_restart;
        i[3] = c.ilu_level;
        i[4] = c.drop_reg_term ? 1 : 0;
        i[5] = c.weight_mode ? (*c.weight_mode == WeightMode::offset ? 1 : 0) : -1;
        i[6] = c.ecg_stride;
        i[7] = int(c.frequencies_hz.size());
        i[8] = int(c.epsilon_list.size());
        for (std::size_t k = 0; k < c.frequencies_hz.size() && k < 64; ++k) freqs[k] = c.frequencies_hz[k];
        for (std::size_t k = 0; k < c.epsilon_list.size() && k < 64; ++k) eps[k] = c.epsilon_list[k];
        return 0;
    } catch (const ParseError& e) {
        g_err = e.what();
        return 1;
    } catch (const IoError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

}  // extern "C"
