// fwi_b200/kkt.hpp — header-only C++ mirror of the reference's KKT/Krylov API
// (namespace fwi in /root/reference/proj/include/fwi/{kkt,krylov,lu,ilu}.hpp)
// on top of the plain C ABI in fwi_b200.h. Same names, argument meaning,
// defaults and exception types; the objects live on the GPU.
//
//   reference (CPU)                          this header (B200)
//   fwi::GnState  make_gn_state(...)         fwi::gpu::make_gn_state(...) (same arguments),
//                                            fwi::gpu::gn_state_from_reference(ref_state),
//                                            fwi::gpu::GnState(desc)
//   fwi::KktVector                           fwi::gpu::KktVector (one flat device buffer)
//   dot / norm / axpy / scal                 same names, same semantics
//   kkt_apply(state, xi)                     kkt_apply(state, xi)
//   kkt_rhs(state)                           kkt_rhs(state)
//   precond_apply(state, v, mode)            precond_apply(state, v, mode)
//   fsgn_gmres_step(state, options)          fsgn_gmres_step(state, options)
//   SingularPivotError / ZeroPivotError      same, with .index
#pragma once

#include <complex>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "fwi_b200.h"

namespace fwi::gpu {

struct SingularPivotError : std::runtime_error {
    int index;
    SingularPivotError(const std::string& m, int i) : std::runtime_error(m), index(i) {}
};
struct ZeroPivotError : std::runtime_error {
    int index;
    ZeroPivotError(const std::string& m, int i) : std::runtime_error(m), index(i) {}
};
struct DeviceError : std::runtime_error {
    int code;
    DeviceError(const std::string& m, int c) : std::runtime_error(m), code(c) {}
};

inline void check(int code) {
    if (code == FWI_OK) return;
    const std::string msg = fwi_dev_last_error();
    switch (code) {
        case FWI_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case FWI_ERR_SINGULAR_PIVOT: throw SingularPivotError(msg, fwi_dev_last_error_index());
        case FWI_ERR_ZERO_PIVOT: throw ZeroPivotError(msg, fwi_dev_last_error_index());
        default: throw DeviceError(msg, code);
    }
}

enum class PrecondMode { exact = FWI_PRECOND_EXACT, ilu = FWI_PRECOND_ILU };

// fwi::GnState on the device (make_gn_state, src/reduced_space.cpp:40-86)
class GnState {
public:
    explicit GnState(const fwi_state_desc& d) { check(fwi_dev_ctx_create(&d, &h_)); }
    GnState(const GnState&) = delete;
    GnState& operator=(const GnState&) = delete;
    GnState(GnState&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
    ~GnState() {
        if (h_) fwi_dev_ctx_destroy(h_);
    }
    fwi_dev_ctx* handle() const { return h_; }
    fwi_state_info info() const {
        fwi_state_info i{};
        check(fwi_dev_ctx_info(h_, &i));
        return i;
    }
    int model_size() const { return info().n; }
    // u_n (K x n, source-major) and r = d_obs - d_pred, as the device holds them
    std::vector<std::complex<double>> u() const {
        const fwi_state_info i = info();
        std::vector<std::complex<double>> v(size_t(i.num_sources) * size_t(i.n));
        check(fwi_dev_ctx_get_u(h_, reinterpret_cast<double*>(v.data())));
        return v;
    }
    std::vector<std::complex<double>> residual() const {
        std::vector<std::complex<double>> v(size_t(info().num_data));
        check(fwi_dev_ctx_get_residual(h_, reinterpret_cast<double*>(v.data())));
        return v;
    }
    int num_sources() const { return info().num_sources; }
    void set_epsilon(double e) { check(fwi_dev_ctx_set_epsilon(h_, e)); }
    void set_drop_reg_term(bool d) { check(fwi_dev_ctx_set_drop_reg_term(h_, d ? 1 : 0)); }
    void factor_ilu(int level, double diag_shift = 0.0) { check(fwi_dev_factor_ilu(h_, level, diag_shift)); }
    std::int64_t solve_count(PrecondMode m = PrecondMode::exact) const {
        return fwi_dev_solve_count(h_, int(m));
    }
    void reset_solve_count(PrecondMode m = PrecondMode::exact) { fwi_dev_reset_solve_count(h_, int(m)); }
    // LuFactors::solve / IluFactors::solve for one RHS
    std::vector<std::complex<double>> solve(const std::vector<std::complex<double>>& b,
                                            PrecondMode m = PrecondMode::exact, bool adjoint = false) {
        if (b.size() != size_t(model_size())) throw std::invalid_argument("solve: right-hand side length mismatch");
        std::vector<std::complex<double>> x(b.size());
        check(fwi_dev_solve(h_, int(m), adjoint ? 1 : 0, 1, reinterpret_cast<const double*>(b.data()),
                            reinterpret_cast<double*>(x.data())));
        return x;
    }

private:
    fwi_dev_ctx* h_ = nullptr;
};

namespace detail {
// The reference's Grid2D / PmlProfile / Survey (include/fwi/grid.hpp:11-42,
// include/fwi/forward.hpp:16-33) flattened into the C descriptor; the arrays live
// as long as this object (ctx_create copies them).
struct FlatSurvey {
    std::vector<int> sx, sz, off, rx, rz;
    std::vector<double> amp;
    fwi_state_desc d{};
    template <class Grid, class Profile, class SurveyT>
    FlatSurvey(const Grid& grid, const Profile& profile, const SurveyT& survey, int weight_mode) {
        off.push_back(0);
        for (const auto& src : survey.sources) {
            sx.push_back(src.ix);
            sz.push_back(src.iz);
            amp.push_back(src.amplitude);
            for (const auto& [x, z] : src.receivers) {
                rx.push_back(x);
                rz.push_back(z);
            }
            off.push_back(int(rx.size()));
        }
        d.grid = fwi_grid_desc{grid.nx, grid.nz, grid.h, grid.n_pml, profile.sigma_max, profile.power};
        d.survey = fwi_survey_desc{int(sx.size()), sx.data(), sz.data(), amp.data(), off.data(),
                                   rx.data(), rz.data(), weight_mode};
    }
};
}  // namespace detail

// fwi::make_gn_state (include/fwi/reduced_space.hpp:51-54, src/reduced_space.cpp:40-86) taking the
// reference's own argument types (Grid2D, PmlProfile, SlownessModel, Survey, DataVector,
// GnStateOptions — or any types with those members). Assembly, the exact factorisation, the
// optional ILU(p), the K forward solves, d_pred and r = d_obs - d_pred are built on the device.
// Same argument checks and exception types as the reference.
template <class Grid, class Profile, class Model, class SurveyT, class Data, class Options>
GnState make_gn_state(const Grid& grid, const Profile& profile, const Model& model, const SurveyT& survey,
                      double freq_hz, const Data& d_obs, const Options& options) {
    if (!(freq_hz > 0.0)) throw std::invalid_argument("make_gn_state: frequency must be positive");
    if (!(options.epsilon > 0.0)) throw std::invalid_argument("make_gn_state: epsilon must be positive");
    if (model.s.size() != size_t(grid.nx) * size_t(grid.nz))
        throw std::invalid_argument("SlownessModel: size does not match the grid");
    detail::FlatSurvey f(grid, profile, survey, int(options.weight_mode));
    if (d_obs.size() != size_t(f.off.back()))
        throw std::invalid_argument("make_gn_state: observed data length mismatch");
    fwi_state_desc d = f.d;
    d.freq_hz = freq_hz;
    d.epsilon = options.epsilon;
    d.drop_reg_term = options.drop_reg_term ? 1 : 0;
    d.s = model.s.data();
    d.u = nullptr;  // computed on the device (solve_forward)
    d.r = nullptr;  // r = d_obs - d_pred on the device
    d.d_obs = reinterpret_cast<const double*>(d_obs.data());
    d.exact_factor = 1;
    d.ilu_level = options.ilu_level ? int(*options.ilu_level) : -1;
    d.ilu_diag_shift = options.ilu_diag_shift;
    return GnState(d);
}

// A device GnState holding exactly the linearisation point of a reference fwi::GnState
// (include/fwi/reduced_space.hpp:15-41): its model, survey, weights mode, epsilon, drop
// flag, background fields u and residual r are uploaded as they are (no re-solve; the weight
// mode is recovered from the weights: all ones = identity), and the
// device factorisations are built from the same operator. ilu_level < 0: no ILU factors.
template <class RefState>
GnState gn_state_from_reference(const RefState& st, int ilu_level = -1, double ilu_diag_shift = 0.0,
                                bool exact_factor = true) {
    // GnState keeps the weights, not the mode they were built with (build_weights,
    // src/forward.cpp:43-62): identity weights are all 1
    bool identity = true;
    for (double w : st.weights.w) identity = identity && w == 1.0;
    detail::FlatSurvey f(st.grid, st.profile, st.survey, identity ? FWI_WEIGHT_IDENTITY : FWI_WEIGHT_OFFSET);
    std::vector<std::complex<double>> u;
    u.reserve(size_t(st.num_sources()) * size_t(st.model_size()));
    for (const auto& uk : st.u.per_source) u.insert(u.end(), uk.begin(), uk.end());
    fwi_state_desc d = f.d;
    d.freq_hz = st.freq_hz;
    d.epsilon = st.epsilon;
    d.drop_reg_term = st.drop_reg_term ? 1 : 0;
    d.s = st.model.s.data();
    d.u = reinterpret_cast<const double*>(u.data());
    d.r = reinterpret_cast<const double*>(st.r.data());
    d.d_obs = reinterpret_cast<const double*>(st.d_obs.data());
    d.exact_factor = exact_factor ? 1 : 0;
    d.ilu_level = ilu_level;
    d.ilu_diag_shift = ilu_diag_shift;
    return GnState(d);
}

// fwi::KktVector on the device: one flat buffer [du_0..du_{K-1} | ds | la_0..la_{K-1}].
// A vector keeps the precision it was created with (FWI_C128, or FWI_C64 for the
// complex64 apply); copies and kkt_apply results inherit it.
class KktVector {
public:
    static KktVector zeros(GnState& s, int precision = FWI_C128) { return KktVector(s, precision); }
    KktVector(GnState& s, int precision = FWI_C128) : state_(&s) {
        check(fwi_dev_vec_create(s.handle(), precision, &h_));
    }
    KktVector(const KktVector& o) : state_(o.state_) {
        check(fwi_dev_vec_create(state_->handle(), o.precision(), &h_));
        check(fwi_dev_vec_copy(h_, o.h_));
    }
    KktVector& operator=(const KktVector& o) {
        if (this == &o) return *this;
        if (!h_ || state_ != o.state_ || precision() != o.precision()) {
            KktVector t(o);
            swap(t);
        } else {
            check(fwi_dev_vec_copy(h_, o.h_));
        }
        return *this;
    }
    KktVector(KktVector&& o) noexcept : state_(o.state_), h_(std::exchange(o.h_, nullptr)) {}
    KktVector& operator=(KktVector&& o) noexcept {
        swap(o);
        return *this;
    }
    ~KktVector() {
        if (h_) fwi_dev_vec_destroy(h_);
    }
    void swap(KktVector& o) noexcept {
        std::swap(state_, o.state_);
        std::swap(h_, o.h_);
    }
    fwi_dev_vec* handle() const { return h_; }
    GnState& state() const { return *state_; }
    int precision() const { return fwi_dev_vec_precision(h_); }
    // number of doubles in the flat host form: 4Kn + n (check_shape, src/kkt.cpp:43-47)
    size_t size() const { return size_t(state_->info().vec_doubles); }
    void upload(const std::vector<double>& flat) {
        if (flat.size() != size()) throw std::invalid_argument("KktVector::upload: size mismatch");
        if (precision() == FWI_C64) {
            const std::vector<float> f(flat.begin(), flat.end());
            check(fwi_dev_vec_upload_f32(h_, f.data()));
        } else {
            check(fwi_dev_vec_upload(h_, flat.data()));
        }
    }
    std::vector<double> download() const {
        if (precision() == FWI_C64) {
            std::vector<float> f(size());
            check(fwi_dev_vec_download_f32(h_, f.data()));
            return std::vector<double>(f.begin(), f.end());
        }
        std::vector<double> f(size());
        check(fwi_dev_vec_download(h_, f.data()));
        return f;
    }
    // any type with the reference KktVector's members (du, ds, lambda)
    template <class RefKkt>
    void upload_from(const RefKkt& v) {
        check_shape(v);
        std::vector<double> f;
        f.reserve(size());
        for (const auto& b : v.du) append(f, b);
        f.insert(f.end(), v.ds.begin(), v.ds.end());
        for (const auto& b : v.lambda) append(f, b);
        upload(f);
    }
    template <class RefKkt>
    void download_into(RefKkt& v) const {
        check_shape(v);
        const std::vector<double> f = download();
        size_t o = 0;
        for (auto& b : v.du) o = take(f, o, b);
        for (auto& d : v.ds) d = f[o++];
        for (auto& b : v.lambda) o = take(f, o, b);
    }

private:
    template <class C>
    static void append(std::vector<double>& f, const C& b) {
        for (const auto& z : b) {
            f.push_back(z.real());
            f.push_back(z.imag());
        }
    }
    template <class C>
    static size_t take(const std::vector<double>& f, size_t o, C& b) {
        for (auto& z : b) {
            z = {f[o], f[o + 1]};
            o += 2;
        }
        return o;
    }
    template <class RefKkt>
    void check_shape(const RefKkt& v) const {
        const fwi_state_info i = state_->info();
        bool ok = int(v.du.size()) == i.num_sources && int(v.lambda.size()) == i.num_sources &&
                  int(v.ds.size()) == i.n;
        for (const auto& b : v.du) ok = ok && int(b.size()) == i.n;
        for (const auto& b : v.lambda) ok = ok && int(b.size()) == i.n;
        if (!ok) throw std::invalid_argument("KktVector: shape mismatch");
    }
    GnState* state_;
    fwi_dev_vec* h_ = nullptr;
};

inline double dot(const KktVector& x, const KktVector& y) {
    double r = 0;
    check(fwi_dev_vec_dot(x.handle(), y.handle(), &r));
    return r;
}
inline double norm(const KktVector& x) {
    double r = 0;
    check(fwi_dev_vec_norm(x.handle(), &r));
    return r;
}
inline void axpy(double a, const KktVector& x, KktVector& y) { check(fwi_dev_vec_axpy(a, x.handle(), y.handle())); }
inline void scal(double a, KktVector& x) { check(fwi_dev_vec_scal(a, x.handle())); }

inline KktVector kkt_apply(GnState& s, const KktVector& xi) {
    KktVector out(s, xi.precision());  // complex64 in, complex64 out
    check(fwi_dev_kkt_apply(s.handle(), xi.handle(), out.handle()));
    return out;
}
inline KktVector kkt_rhs(GnState& s) {
    KktVector out(s);
    check(fwi_dev_kkt_rhs(s.handle(), out.handle()));
    return out;
}
inline KktVector precond_apply(GnState& s, const KktVector& v, PrecondMode mode) {
    if (v.precision() != FWI_C128)
        throw std::invalid_argument("precond_apply: complex128 vector required (complex64 is kkt_apply only)");
    KktVector out(s);
    check(fwi_dev_precond_apply(s.handle(), int(mode), v.handle(), out.handle()));
    return out;
}

// fwi::FsgnOptions (include/fwi/kkt.hpp:47-57), same defaults
struct FsgnOptions {
    PrecondMode mode = PrecondMode::exact;
    int restart = 30;
    double tol = 1e-10;
    int maxit = 30;
    int ecg_stride = 1;
    double ecg_stop_tol = 0.0;
};

// fwi::ConvergenceLog (include/fwi/krylov.hpp:17-33)
struct ConvergenceLog {
    struct Entry {
        int iteration = 0;
        double residual_norm = 0.0;
        std::optional<double> normal_residual;
        std::optional<double> precond_residual;
        double wall_time = 0.0;
    };
    std::vector<Entry> entries;
    bool converged = false;
    bool stagnated = false;
    int iterations() const { return entries.empty() ? 0 : entries.back().iteration; }
    double final_residual() const { return entries.empty() ? 0.0 : entries.back().residual_norm; }
};

struct StepResult {
    std::vector<double> delta_s;
    ConvergenceLog log;
};

inline StepResult fsgn_gmres_step(GnState& s, const FsgnOptions& o = {}) {
    fwi_fsgn_options co{int(o.mode), o.restart, o.tol, o.maxit, o.ecg_stride, o.ecg_stop_tol};
    std::vector<fwi_log_entry> buf(size_t(o.maxit) + 2);
    fwi_convergence_log cl{buf.data(), int(buf.size()), 0, 0, 0};
    StepResult r;
    r.delta_s.resize(size_t(s.model_size()));
    check(fwi_dev_fsgn_gmres_step(s.handle(), &co, r.delta_s.data(), &cl));
    for (int i = 0; i < cl.count; ++i) {
        ConvergenceLog::Entry e;
        e.iteration = buf[i].iteration;
        e.residual_norm = buf[i].residual_norm;
        if (buf[i].has_normal_residual) e.normal_residual = buf[i].normal_residual;
        if (buf[i].has_precond_residual) e.precond_residual = buf[i].precond_residual;
        e.wall_time = buf[i].wall_time;
        r.log.entries.push_back(e);
    }
    r.log.converged = cl.converged != 0;
    r.log.stagnated = cl.stagnated != 0;
    return r;
}

// fwi::gradient / fwi::hessian_apply (include/fwi/reduced_space.hpp; src/reduced_space.cpp:
// 120-152): the reduced-space building blocks of the E_cg metric and the RSGN path.
inline std::vector<double> gradient(GnState& s) {
    std::vector<double> g(size_t(s.model_size()));
    check(fwi_dev_gradient(s.handle(), g.data()));
    return g;
}
inline std::vector<double> hessian_apply(GnState& s, const std::vector<double>& v) {
    if (v.size() != size_t(s.model_size())) throw std::invalid_argument("hessian_apply: size mismatch");
    std::vector<double> out(v.size());
    check(fwi_dev_hessian_apply(s.handle(), v.data(), out.data()));
    return out;
}

}  // namespace fwi::gpu
