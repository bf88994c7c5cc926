// gmres.cu — restarted, left-preconditioned GMRES on device-resident vectors
// (the reference's template, include/fwi/krylov.hpp:128-269, with S = double
// as the KKT inner product is real) and fsgn_gmres_step
// (src/kkt.cpp:137-171).
//
// Control flow, Hessenberg/Givens arithmetic, the triangular y-solve,
// stagnation and best-iterate rules are the reference's, on the host, in
// double. Every vector pass runs on the device: the MGS steps are fused
// "w -= h_{i-1} v_{i-1}; h_i = <v_i, w>" kernels whose h values stay in device
// memory until one D2H copy per iteration; x_cand = x + V y is one fused pass
// with the reference's per-basis-vector rounding order; the true residual
// ||b - A x_cand|| is a KKT apply plus one fused difference-norm pass.
#include <chrono>
#include <cmath>
#include <functional>
#include <optional>

#include "ctx.cuh"

namespace fwi_b200 {

void reduced_gradient(Ctx& c, double* g_dev);
void reduced_hessian(Ctx& c, const double* v_dev, double* out_dev);

namespace {

struct Entry {
    int iteration;
    double residual_norm;
    std::optional<double> normal_residual;
    std::optional<double> precond_residual;
    double wall_time;
};

struct Log {
    std::vector<Entry> entries;
    bool converged = false;
    bool stagnated = false;
};

struct GmresOps {
    int64_t len = 0;
    cudaStream_t st = nullptr;
    std::function<void(const double*, double*)> apply, precond;
    std::function<bool(int, const double*)> observer;  // may be empty
};

struct Scratch {
    DevBuf<double> partials, out;
    DevBuf<unsigned> ticket;
    Scratch() {
        partials.alloc(4096);
        out.alloc(256);
        ticket.alloc(64);
        CK(cudaMemset(ticket.p, 0, 64 * sizeof(unsigned)));
    }
};

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

double dnorm(Scratch& s, cudaStream_t st, const double* x, int64_t len) {
    dev_dot_async(st, x, x, s.out.p, s.partials.p, s.ticket.p, len);
    double h = 0;
    CK(cudaMemcpyAsync(&h, s.out.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return std::sqrt(h);
}

// x (device, len) receives the solution.
Log gmres_core(GmresOps& ops, const double* b, double* x, int restart, double tol, int maxit) {
    if (restart < 1) throw FwiError(FWI_ERR_INVALID_ARGUMENT, "gmres: restart must be >= 1");
    const auto t0 = std::chrono::steady_clock::now();
    double observer_time = 0.0;
    auto elapsed = [&] { return seconds_since(t0) - observer_time; };
    const int64_t len = ops.len;
    const size_t bytes = size_t(len) * sizeof(double);
    cudaStream_t st = ops.st;
    Scratch sc;

    CK(cudaMemsetAsync(x, 0, bytes, st));
    Log log;
    const double bnorm = dnorm(sc, st, b, len);
    if (bnorm == 0.0) {
        log.entries.push_back({0, 0.0, {}, {}, elapsed()});
        log.converged = true;
        return log;
    }
    DevBuf<double> tmp(len), w(len), xc(len), best(len);
    ops.precond(b, w.p);
    const double pbnorm = dnorm(sc, st, w.p, len);
    if (pbnorm == 0.0)
        throw FwiError(FWI_ERR_INVALID_ARGUMENT, "gmres: preconditioner annihilates the right-hand side");
    log.entries.push_back({0, 1.0, {}, 1.0, elapsed()});

    CK(cudaMemsetAsync(best.p, 0, bytes, st));
    double best_res = 1.0, true_res = 1.0;
    int iter = 0;
    bool stop_requested = false;
    const int nbasis = std::min(restart, std::max(maxit, 1)) + 1;
    std::vector<DevBuf<double>> V(nbasis);
    DevBuf<double> hdev(size_t(restart) + 2), ydev(size_t(restart) + 1);
    std::vector<double> hh(restart + 2);

    while (iter < maxit && !log.converged && !stop_requested) {
        // r0 = M^{-1}(b - A x)
        ops.apply(x, tmp.p);
        CK(cudaMemcpyAsync(xc.p, b, bytes, cudaMemcpyDeviceToDevice, st));
        dev_axpy(st, -1.0, tmp.p, xc.p, len);
        if (!V[0].p) V[0].alloc(len);
        ops.precond(xc.p, V[0].p);
        const double beta = dnorm(sc, st, V[0].p, len);
        const double cycle_start_res = true_res;
        if (beta == 0.0) break;
        dev_scal(st, 1.0 / beta, V[0].p, len);

        std::vector<std::vector<double>> hcols;
        std::vector<double> gs_c, gs_s, g(1, beta);
        CK(cudaMemcpyAsync(xc.p, x, bytes, cudaMemcpyDeviceToDevice, st));
        bool happy = false;
        int nv = 1;

        for (int j = 0; j < restart && iter < maxit; ++j) {
            ++iter;
            ops.apply(V[j].p, tmp.p);
            ops.precond(tmp.p, w.p);
            // MGS: h_i = <v_i, w>; w -= h_i v_i  (fused pairwise)
            for (int i = 0; i <= j; ++i)
                dev_mgs_step(st, w.p, i > 0 ? V[i - 1].p : nullptr, hdev.p + (i - 1), V[i].p,
                             hdev.p + i, sc.partials.p, sc.ticket.p, len);
            dev_mgs_step(st, w.p, V[j].p, hdev.p + j, nullptr, hdev.p + j + 1, sc.partials.p,
                         sc.ticket.p, len);
            CK(cudaMemcpyAsync(hh.data(), hdev.p, (j + 2) * sizeof(double), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            std::vector<double> h(hh.begin(), hh.begin() + j + 2);
            const double wn = std::sqrt(h[j + 1]);
            h[j + 1] = wn;

            for (int i = 0; i < j; ++i) {
                const double t = gs_c[i] * h[i] + gs_s[i] * h[i + 1];
                h[i + 1] = -gs_s[i] * h[i] + gs_c[i] * h[i + 1];
                h[i] = t;
            }
            double c, s, rr;
            {
                const double an = std::abs(h[j]), bn = std::abs(h[j + 1]);
                const double t = std::sqrt(an * an + bn * bn);
                if (bn == 0.0) {
                    c = 1.0;
                    s = 0.0;
                    rr = h[j];
                } else if (an == 0.0) {
                    c = 0.0;
                    s = h[j + 1] / bn;
                    rr = bn;
                } else {
                    c = an / t;
                    s = (h[j] / an) * h[j + 1] / t;
                    rr = (h[j] / an) * t;
                }
            }
            gs_c.push_back(c);
            gs_s.push_back(s);
            h[j] = rr;
            h[j + 1] = 0.0;
            g.push_back(-s * g[j]);
            g[j] = c * g[j];
            hcols.push_back(h);
            const double prec_res = std::abs(g[j + 1]) / pbnorm;

            std::vector<double> y(j + 1);
            for (int i = j; i >= 0; --i) {
                double acc = g[i];
                for (int k2 = i + 1; k2 <= j; ++k2) acc -= hcols[k2][i] * y[k2];
                y[i] = acc / hcols[i][i];
            }
            CK(cudaMemcpyAsync(ydev.p, y.data(), (j + 1) * sizeof(double), cudaMemcpyHostToDevice, st));
            std::vector<const double*> vp(j + 1);
            for (int i = 0; i <= j; ++i) vp[i] = V[i].p;
            dev_multi_axpy(st, xc.p, x, vp.data(), ydev.p, j + 1, len);

            ops.apply(xc.p, tmp.p);
            dev_sub_norm2(st, b, tmp.p, sc.out.p, sc.partials.p, sc.ticket.p, len);
            double r2 = 0;
            CK(cudaMemcpyAsync(&r2, sc.out.p, sizeof(double), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            true_res = std::sqrt(r2) / bnorm;
            log.entries.push_back({iter, true_res, {}, prec_res, elapsed()});
            if (true_res < best_res) {
                best_res = true_res;
                CK(cudaMemcpyAsync(best.p, xc.p, bytes, cudaMemcpyDeviceToDevice, st));
            }
            if (ops.observer) {
                const auto to0 = std::chrono::steady_clock::now();
                stop_requested = ops.observer(iter, xc.p);
                observer_time += seconds_since(to0);
            }
            if (true_res <= tol) log.converged = true;
            if (wn == 0.0) happy = true;
            if (log.converged || stop_requested || happy) break;
            // v_{j+1} = w / ||w||  (buffer rotation, no copy)
            dev_scal(st, 1.0 / wn, w.p, len);
            std::swap(V[j + 1], w);
            if (!w.p) w.alloc(len);
            nv = j + 2;
        }
        (void)nv;
        CK(cudaMemcpyAsync(x, xc.p, bytes, cudaMemcpyDeviceToDevice, st));
        if (!log.converged && !stop_requested && true_res >= cycle_start_res * (1.0 - 1e-12)) {
            log.stagnated = true;
            CK(cudaMemcpyAsync(x, best.p, bytes, cudaMemcpyDeviceToDevice, st));
            break;
        }
        if (happy && !log.converged && !stop_requested) {
            log.stagnated = true;
            CK(cudaMemcpyAsync(x, best.p, bytes, cudaMemcpyDeviceToDevice, st));
            break;
        }
    }
    CK(cudaStreamSynchronize(st));
    return log;
}

void fill_log(const Log& lg, fwi_convergence_log* out) {
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
        d.pad_ = 0;
    }
    out->converged = lg.converged;
    out->stagnated = lg.stagnated;
}

}  // namespace

void fsgn_gmres_step(Ctx& c, const fwi_fsgn_options& o, double* ds_host, fwi_convergence_log* log) {
    require(o.mode == FWI_PRECOND_EXACT || o.mode == FWI_PRECOND_ILU, "fsgn_gmres_step: unknown mode");
    if (o.mode == FWI_PRECOND_ILU) require(c.ilu != nullptr, "precond_apply: state has no ILU factorization");
    if (o.mode == FWI_PRECOND_EXACT)
        require(c.exact != nullptr, "precond_apply: state has no exact factorization");
    const int64_t len = c.vec_len;
    const int64_t n = c.n;
    cudaStream_t st = c.stream;
    // b = kkt_rhs
    Vec bv;
    bv.ctx = &c;
    bv.d.alloc(len);
    kkt_rhs(c, bv);
    DevBuf<double> xv(len);
    // g = gradient(state): K adjoint solves (src/kkt.cpp:139-141). It only
    // normalises the E_cg metric; without the exact factorisation the metric
    // column is left unset.
    DevBuf<double> g(c.ds_stride), hds(c.ds_stride);
    CK(cudaMemsetAsync(g.p, 0, g.bytes(), st));
    CK(cudaMemsetAsync(hds.p, 0, hds.bytes(), st));
    double gnorm = 0.0;
    if (c.exact) {
        reduced_gradient(c, g.p);
        Scratch sc;
        gnorm = dnorm(sc, st, g.p, c.ds_stride);
    }
    std::vector<std::pair<int, double>> metric;
    GmresOps ops;
    ops.len = len;
    ops.st = st;
    ops.apply = [&c](const double* in, double* out) { kkt_apply_raw(c, in, out); };
    const int mode = o.mode;
    ops.precond = [&c, mode](const double* in, double* out) { precond_apply_raw(c, mode, in, out); };
    if (o.ecg_stride > 0) {
        require(c.exact != nullptr, "fsgn_gmres_step: the normal-equation metric needs the exact factorization");
        ops.observer = [&](int iter, const double* xi) {
            if (iter % o.ecg_stride != 0) return false;
            // normal_residual (src/reduced_space.cpp:154-161)
            reduced_hessian(c, c.ds_of(const_cast<double*>(xi)), hds.p);
            dev_axpy(st, -1.0, g.p, hds.p, c.ds_stride);
            Scratch sc;
            const double rn = dnorm(sc, st, hds.p, c.ds_stride);
            double e;
            if (gnorm == 0.0)
                e = rn == 0.0 ? 0.0 : INFINITY;
            else
                e = rn / gnorm;
            metric.emplace_back(iter, e);
            return o.ecg_stop_tol > 0.0 && e <= o.ecg_stop_tol;
        };
    }
    Log lg = gmres_core(ops, bv.d.p, xv.p, o.restart, o.tol, o.maxit);
    if (!lg.entries.empty() && c.exact) lg.entries.front().normal_residual = gnorm > 0.0 ? 1.0 : 0.0;
    for (const auto& [it, e] : metric)
        for (auto& en : lg.entries)
            if (en.iteration == it) {
                en.normal_residual = e;
                break;
            }
    if (ds_host)
        CK(cudaMemcpyAsync(ds_host, c.ds_of(xv.p), n * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    fill_log(lg, log);
}

// rsgn_cg_step (src/reduced_space.cpp:163-170) over cg<RealVector>
// (include/fwi/krylov.hpp:79-120): CG on H ds = g, H = Re(J^H W^T W J) + eps I.
void rsgn_cg_step(Ctx& c, double tol, int maxit, double* ds_host, fwi_convergence_log* log) {
    require(c.exact != nullptr, "rsgn_cg_step: state has no exact factorization");
    const auto t0 = std::chrono::steady_clock::now();
    const int64_t len = c.ds_stride;
    cudaStream_t st = c.stream;
    Scratch sc;
    auto ddot = [&](const double* a, const double* b) {
        dev_dot_async(st, a, b, sc.out.p, sc.partials.p, sc.ticket.p, len);
        double h = 0;
        CK(cudaMemcpyAsync(&h, sc.out.p, sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        return h;
    };
    DevBuf<double> g(len), x(len), r(len), p(len), ap(len);
    for (auto* b : {&g, &x, &r, &p, &ap}) CK(cudaMemsetAsync(b->p, 0, b->bytes(), st));
    reduced_gradient(c, g.p);
    Log lg;
    const double bnorm = std::sqrt(ddot(g.p, g.p));
    if (bnorm == 0.0) {
        lg.entries.push_back({0, 0.0, {}, {}, seconds_since(t0)});
        lg.converged = true;
    } else {
        lg.entries.push_back({0, 1.0, {}, {}, seconds_since(t0)});
        CK(cudaMemcpyAsync(r.p, g.p, len * sizeof(double), cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(p.p, g.p, len * sizeof(double), cudaMemcpyDeviceToDevice, st));
        double rho = ddot(r.p, r.p);
        for (int it = 1; it <= maxit; ++it) {
            reduced_hessian(c, p.p, ap.p);
            const double pap = ddot(p.p, ap.p);
            if (!(pap > 0.0))
                throw FwiError(FWI_ERR_CG_BREAKDOWN, "cg: non-positive curvature, operator is not HPD");
            const double alpha = rho / pap;
            dev_axpy(st, alpha, p.p, x.p, len);
            dev_axpy(st, -alpha, ap.p, r.p, len);
            const double rn = std::sqrt(ddot(r.p, r.p)) / bnorm;
            lg.entries.push_back({it, rn, {}, {}, seconds_since(t0)});
            if (rn <= tol) {
                lg.converged = true;
                break;
            }
            const double rho_new = ddot(r.p, r.p);
            const double beta = rho_new / rho;
            rho = rho_new;
            dev_scal(st, beta, p.p, len);
            dev_axpy(st, 1.0, r.p, p.p, len);
        }
    }
    for (auto& e : lg.entries) e.normal_residual = e.residual_norm;  // src/reduced_space.cpp:166-168
    if (ds_host) CK(cudaMemcpyAsync(ds_host, x.p, c.n * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    fill_log(lg, log);
}

void gmres_generic(int64_t n, fwi_op_cb apply, fwi_op_cb precond, fwi_observer_cb observer, void* user,
                   const double* b, double* x, int restart, double tol, int maxit,
                   fwi_convergence_log* log) {
    require(n > 0 && n % 2 == 0, "gmres_generic: vector length must be positive and even");
    GmresOps ops;
    ops.len = n;
    ops.st = nullptr;  // legacy stream: callbacks may use any stream-ordered API
    ops.apply = [&](const double* in, double* out) {
        CK(cudaStreamSynchronize(nullptr));
        if (apply(user, in, out) != 0) throw FwiError(FWI_ERR_INVALID_ARGUMENT, "gmres: apply callback failed");
    };
    ops.precond = [&](const double* in, double* out) {
        CK(cudaStreamSynchronize(nullptr));
        if (precond(user, in, out) != 0)
            throw FwiError(FWI_ERR_INVALID_ARGUMENT, "gmres: precond callback failed");
    };
    if (observer)
        ops.observer = [&](int it, const double* xc) {
            CK(cudaStreamSynchronize(nullptr));
            return observer(user, it, xc) != 0;
        };
    Log lg = gmres_core(ops, b, x, restart, tol, maxit);
    fill_log(lg, log);
}

}  // namespace fwi_b200
