// driver.cu — gn_step on the device (src/driver.cpp:65-127): the caller of
// the hot path. Linearisation (assembly, exact block factorisation, forward
// fields, residual) happens in the device context; the inner solve is the
// device fsgn_gmres_step; the clamp and the misfits follow the reference's
// arithmetic (std::clamp, std::norm sums in data order).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <limits>
#include <memory>

#include "ctx.cuh"

namespace fwi_b200 {

void rsgn_cg_step(Ctx& c, double tol, int maxit, double* ds_host, fwi_convergence_log* log);

namespace {

// relative_misfit (src/forward.cpp:114-124)
double relative_misfit(const std::vector<std::complex<double>>& pred, const std::complex<double>* obs, int nd) {
    double num = 0.0, den = 0.0;
    for (int i = 0; i < nd; ++i) {
        num += std::norm(pred[i] - obs[i]);
        den += std::norm(obs[i]);
    }
    if (den == 0.0) return std::sqrt(num) == 0.0 ? 0.0 : std::numeric_limits<double>::infinity();
    return std::sqrt(num / den);
}

std::vector<std::complex<double>> dpred_of(const Ctx& c) {
    std::vector<std::complex<double>> d(std::max(c.ndata, 1));
    CK(cudaStreamSynchronize(c.stream));
    if (c.ndata) CK(cudaMemcpy(d.data(), c.dpred.p, c.ndata * sizeof(double2), cudaMemcpyDeviceToHost));
    d.resize(c.ndata);
    return d;
}

}  // namespace

void gn_step(const fwi_state_desc& d0, const fwi_gn_options& o, double* s_out, fwi_gn_result* res,
             fwi_convergence_log* log) {
    require(o.solver == FWI_SOLVER_RSGN_CG || o.solver == FWI_SOLVER_FSGN_EXACT || o.solver == FWI_SOLVER_FSGN_ILU,
            "gn_step: unknown inner solver");
    require(o.max_inner >= 1, "FwiConfig: max_inner must be >= 1");
    require(o.v_min > 0.0 && o.v_max > o.v_min, "FwiConfig: need 0 < v_min < v_max");
    require(d0.d_obs != nullptr || d0.survey.recv_offset[d0.survey.num_sources] == 0,
            "gn_step: observed data required");
    const auto t0 = std::chrono::steady_clock::now();
    fwi_state_desc d = d0;
    d.u = nullptr;  // linearisation: fields from the device's own forward solves
    d.r = nullptr;
    d.exact_factor = 1;
    // make_gn_state builds the ILU factors only for the ILU solver (src/driver.cpp:78-83), and
    // IluFactors::factor rejects a negative fill level (src/ilu.cpp:9-10)
    require(o.solver != FWI_SOLVER_FSGN_ILU || o.ilu_level >= 0, "IluFactors::factor: fill level must be >= 0");
    d.ilu_level = o.solver == FWI_SOLVER_FSGN_ILU ? o.ilu_level : -1;
    d.ilu_diag_shift = o.ilu_diag_shift;
    std::unique_ptr<Ctx> c(ctx_create(d));
    const auto t1 = std::chrono::steady_clock::now();
    res->setup_seconds = std::chrono::duration<double>(t1 - t0).count();
    res->ilu_factor_seconds = c->t_ilu_factor;
    const int nd = c->ndata, n = c->n;
    const auto* obs = reinterpret_cast<const std::complex<double>*>(d0.d_obs);
    res->misfit_ini = relative_misfit(dpred_of(*c), obs, nd);

    fwi_fsgn_options fo;
    fo.mode = o.solver == FWI_SOLVER_FSGN_EXACT ? FWI_PRECOND_EXACT : FWI_PRECOND_ILU;
    fo.restart = o.gmres_restart;
    fo.tol = o.inner_tol;
    fo.maxit = o.max_inner;
    fo.ecg_stride = o.ecg_stride;
    fo.ecg_stop_tol = o.ecg_stop_tol;
    std::vector<double> ds(n);
    if (o.solver == FWI_SOLVER_RSGN_CG)
        rsgn_cg_step(*c, o.inner_tol, o.max_inner, ds.data(), log);
    else
        fsgn_gmres_step(*c, fo, ds.data(), log);
    c.reset();
    const auto t2 = std::chrono::steady_clock::now();
    res->krylov_seconds = std::chrono::duration<double>(t2 - t1).count();

    // clamp (src/driver.cpp:108-113)
    const double s_lo = 1.0 / (o.v_max * o.v_max), s_hi = 1.0 / (o.v_min * o.v_min);
    std::vector<double> s1(n);
    double nds = 0.0, ns = 0.0;
    for (int i = 0; i < n; ++i) {
        s1[i] = std::clamp(d0.s[i] + ds[i], s_lo, s_hi);
        nds += ds[i] * ds[i];
        ns += d0.s[i] * d0.s[i];
    }
    res->update_relnorm = std::sqrt(nds) / std::sqrt(ns);
    std::copy(s1.begin(), s1.end(), s_out);

    // final misfit at the updated model (src/driver.cpp:116-122)
    fwi_state_desc d2 = d;
    d2.s = s1.data();
    d2.ilu_level = -1;
    std::unique_ptr<Ctx> c2(ctx_create(d2));
    res->misfit_fin = relative_misfit(dpred_of(*c2), obs, nd);
    const auto t3 = std::chrono::steady_clock::now();
    res->final_seconds = std::chrono::duration<double>(t3 - t2).count();
    res->wall_seconds = std::chrono::duration<double>(t3 - t0).count();
}

}  // namespace fwi_b200
