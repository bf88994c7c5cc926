// capi.cu — the extern "C" boundary (include/fwi_b200.h). Exceptions never
// cross it: every entry point maps FwiError / std::exception to a status code
// and a thread-local message (+ pivot index for SingularPivotError /
// ZeroPivotError, include/fwi/lu.hpp:11-16, include/fwi/ilu.hpp:11-17).
#include <cstring>

#include "ctx.cuh"

using namespace fwi_b200;

struct fwi_dev_ctx {
    Ctx* c;
};
struct fwi_dev_vec {
    Vec v;
};

namespace fwi_b200 {
void rsgn_cg_step(Ctx& c, double tol, int maxit, double* ds_host, fwi_convergence_log* log);
void reduced_gradient(Ctx& c, double* g_dev);
void reduced_hessian(Ctx& c, const double* v_dev, double* out_dev);
void gn_step(const fwi_state_desc& d0, const fwi_gn_options& o, double* s_out, fwi_gn_result* res,
             fwi_convergence_log* log);
void gmres_generic(int64_t n, fwi_op_cb apply, fwi_op_cb precond, fwi_observer_cb observer, void* user,
                   const double* b, double* x, int restart, double tol, int maxit,
                   fwi_convergence_log* log);
}

namespace {
thread_local std::string g_err;
thread_local int g_err_index = -1;

template <class F>
int guard(F&& f) {
    try {
        f();
        return FWI_OK;
    } catch (const FwiError& e) {
        g_err = e.what();
        g_err_index = e.index;
        return e.code;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        g_err_index = -1;
        return FWI_ERR_INVALID_ARGUMENT;
    } catch (const std::bad_alloc& e) {
        g_err = e.what();
        g_err_index = -1;
        return FWI_ERR_OUT_OF_MEMORY;
    } catch (const std::exception& e) {
        g_err = e.what();
        g_err_index = -1;
        return FWI_ERR_NOT_SUPPORTED;
    }
}

void need(const void* p, const char* what) {
    if (!p) throw FwiError(FWI_ERR_INVALID_ARGUMENT, std::string(what) + ": null pointer");
}

// host flat (4Kn+n) <-> device flat (4Kn + ds_stride)
template <class T>
void copy_flat(const Ctx& c, T* dst, const T* src, bool to_device) {
    const size_t kn2 = size_t(2) * c.K * c.n;
    const auto kind = to_device ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
    const size_t dev_la = kn2 + c.ds_stride, host_la = kn2 + c.n;
    if (to_device) {
        CK(cudaMemcpyAsync(dst, src, kn2 * sizeof(T), kind, c.stream));
        CK(cudaMemcpyAsync(dst + kn2, src + kn2, size_t(c.n) * sizeof(T), kind, c.stream));
        CK(cudaMemcpyAsync(dst + dev_la, src + host_la, kn2 * sizeof(T), kind, c.stream));
    } else {
        CK(cudaMemcpyAsync(dst, src, kn2 * sizeof(T), kind, c.stream));
        CK(cudaMemcpyAsync(dst + kn2, src + kn2, size_t(c.n) * sizeof(T), kind, c.stream));
        CK(cudaMemcpyAsync(dst + host_la, src + dev_la, kn2 * sizeof(T), kind, c.stream));
    }
    CK(cudaStreamSynchronize(c.stream));
}
}  // namespace

extern "C" {

const char* fwi_dev_last_error(void) { return g_err.c_str(); }
int fwi_dev_last_error_index(void) { return g_err_index; }
const char* fwi_dev_version(void) { return "fwi_b200 0.1 sm_100a"; }

int fwi_dev_ctx_create(const fwi_state_desc* desc, fwi_dev_ctx** out) {
    return guard([&] {
        need(desc, "fwi_dev_ctx_create");
        need(out, "fwi_dev_ctx_create");
        *out = nullptr;
        Ctx* c = ctx_create(*desc);
        *out = new fwi_dev_ctx{c};
    });
}

int fwi_dev_ctx_destroy(fwi_dev_ctx* ctx) {
    return guard([&] {
        if (!ctx) return;
        delete ctx->c;
        delete ctx;
    });
}

int fwi_dev_ctx_info(const fwi_dev_ctx* ctx, fwi_state_info* o) {
    return guard([&] {
        need(ctx, "ctx");
        need(o, "info");
        const Ctx& c = *ctx->c;
        o->nx = c.nx;
        o->nz = c.nz;
        o->n = c.n;
        o->num_sources = c.K;
        o->num_data = c.ndata;
        o->omega = c.omega;
        o->epsilon = c.eps;
        o->drop_reg_term = c.drop;
        o->has_exact = c.exact != nullptr;
        o->has_ilu = c.ilu != nullptr;
        o->vec_doubles = 4 * int64_t(c.K) * c.n + c.n;
        o->device_bytes = int64_t(c.diag.bytes() * 3 + c.u.bytes() + c.u32.bytes() + c.s.bytes() +
                                  exact_bytes(c.exact) + ilu_bytes(c.ilu) + c.work_a.bytes() + c.work_b.bytes() +
                                  c.work_c.bytes());
        o->exact_factor_bytes = exact_bytes(c.exact);
        o->ilu_factor_bytes = ilu_bytes(c.ilu);
        o->exact_probe_residual = exact_probe_residual(c.exact);
    });
}

int fwi_dev_ctx_set_epsilon(fwi_dev_ctx* ctx, double e) {
    return guard([&] {
        need(ctx, "ctx");
        require(e > 0.0, "make_gn_state: epsilon must be positive");
        ctx->c->eps = e;
    });
}

int fwi_dev_ctx_set_drop_reg_term(fwi_dev_ctx* ctx, int d) {
    return guard([&] {
        need(ctx, "ctx");
        ctx->c->drop = d != 0;
    });
}

int fwi_dev_ctx_synchronize(fwi_dev_ctx* ctx) {
    return guard([&] {
        need(ctx, "ctx");
        CK(cudaStreamSynchronize(ctx->c->stream));
    });
}

int fwi_dev_ctx_stream(const fwi_dev_ctx* ctx, void** stream) {
    return guard([&] {
        need(ctx, "ctx");
        need(stream, "stream");
        *stream = static_cast<void*>(ctx->c->stream);
    });
}

int fwi_dev_ctx_get_u(const fwi_dev_ctx* ctx, double* host) {
    return guard([&] {
        need(ctx, "ctx");
        need(host, "host");
        const Ctx& c = *ctx->c;
        CK(cudaStreamSynchronize(c.stream));
        CK(cudaMemcpy(host, c.u.p, c.u.bytes(), cudaMemcpyDeviceToHost));
    });
}

int fwi_dev_ctx_get_residual(const fwi_dev_ctx* ctx, double* host) {
    return guard([&] {
        need(ctx, "ctx");
        const Ctx& c = *ctx->c;
        CK(cudaStreamSynchronize(c.stream));
        if (c.ndata) CK(cudaMemcpy(host, c.r.p, c.ndata * sizeof(double2), cudaMemcpyDeviceToHost));
    });
}

int fwi_dev_ctx_get_dpred(const fwi_dev_ctx* ctx, double* host) {
    return guard([&] {
        need(ctx, "ctx");
        const Ctx& c = *ctx->c;
        CK(cudaStreamSynchronize(c.stream));
        if (c.ndata) CK(cudaMemcpy(host, c.dpred.p, c.ndata * sizeof(double2), cudaMemcpyDeviceToHost));
    });
}

int fwi_dev_ctx_get_stencil(const fwi_dev_ctx* ctx, double* diag, double* east, double* south) {
    return guard([&] {
        need(ctx, "ctx");
        stencil_to_host(*ctx->c, diag, east, south);
    });
}

int fwi_dev_factor_exact(fwi_dev_ctx* ctx) {
    return guard([&] {
        need(ctx, "ctx");
        exact_factor(*ctx->c);
    });
}

int fwi_dev_factor_ilu(fwi_dev_ctx* ctx, int level, double shift) {
    return guard([&] {
        need(ctx, "ctx");
        ilu_factor(*ctx->c, level, shift);
    });
}

int64_t fwi_dev_solve_count(const fwi_dev_ctx* ctx, int mode) {
    if (!ctx || (mode != FWI_PRECOND_EXACT && mode != FWI_PRECOND_ILU)) return -1;
    return ctx->c->solve_count[mode];
}

const char* fwi_dev_kkt_kernel(const fwi_dev_ctx* ctx, int precision) {
    if (!ctx) return "";
    return ctx->c->kkt_kernel[precision == FWI_C64 ? 1 : 0];
}

void fwi_dev_reset_solve_count(fwi_dev_ctx* ctx, int mode) {
    if (ctx && (mode == FWI_PRECOND_EXACT || mode == FWI_PRECOND_ILU)) ctx->c->solve_count[mode] = 0;
}

int fwi_dev_solve(fwi_dev_ctx* ctx, int mode, int adjoint, int nrhs, const double* b, double* x) {
    return guard([&] {
        need(ctx, "ctx");
        need(b, "b");
        need(x, "x");
        require(nrhs >= 1, "fwi_dev_solve: nrhs must be >= 1");
        Ctx& c = *ctx->c;
        const size_t m = size_t(nrhs) * c.n;
        DevBuf<double2> db(m), dx(m);
        CK(cudaMemcpyAsync(db.p, b, m * sizeof(double2), cudaMemcpyHostToDevice, c.stream));
        block_solve(c, mode, adjoint != 0, db.p, dx.p, nrhs);
        CK(cudaMemcpyAsync(x, dx.p, m * sizeof(double2), cudaMemcpyDeviceToHost, c.stream));
        CK(cudaStreamSynchronize(c.stream));
    });
}

int fwi_dev_vec_create(fwi_dev_ctx* ctx, int precision, fwi_dev_vec** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(out, "out");
        require(precision == FWI_C128 || precision == FWI_C64, "fwi_dev_vec_create: unknown precision");
        Ctx& c = *ctx->c;
        auto v = std::make_unique<fwi_dev_vec>();
        v->v.ctx = &c;
        v->v.prec = precision;
        if (precision == FWI_C128) {
            v->v.d.alloc(c.vec_len);
            CK(cudaMemsetAsync(v->v.d.p, 0, v->v.d.bytes(), c.stream));
        } else {
            v->v.f.alloc(c.vec_len);
            CK(cudaMemsetAsync(v->v.f.p, 0, v->v.f.bytes(), c.stream));
        }
        CK(cudaStreamSynchronize(c.stream));
        *out = v.release();
    });
}

int fwi_dev_vec_destroy(fwi_dev_vec* v) {
    return guard([&] { delete v; });
}

int fwi_dev_vec_precision(const fwi_dev_vec* v) { return v ? v->v.prec : -1; }

int fwi_dev_vec_upload(fwi_dev_vec* v, const double* h) {
    return guard([&] {
        need(v, "vec");
        need(h, "host");
        require(v->v.prec == FWI_C128, "upload: complex128 vector expected");
        copy_flat(*v->v.ctx, v->v.d.p, h, true);
    });
}

int fwi_dev_vec_download(const fwi_dev_vec* v, double* h) {
    return guard([&] {
        need(v, "vec");
        need(h, "host");
        require(v->v.prec == FWI_C128, "download: complex128 vector expected");
        copy_flat(*v->v.ctx, h, v->v.d.p, false);
    });
}

int fwi_dev_vec_upload_f32(fwi_dev_vec* v, const float* h) {
    return guard([&] {
        need(v, "vec");
        need(h, "host");
        require(v->v.prec == FWI_C64, "upload_f32: complex64 vector expected");
        copy_flat(*v->v.ctx, v->v.f.p, h, true);
    });
}

int fwi_dev_vec_download_f32(const fwi_dev_vec* v, float* h) {
    return guard([&] {
        need(v, "vec");
        need(h, "host");
        require(v->v.prec == FWI_C64, "download_f32: complex64 vector expected");
        copy_flat(*v->v.ctx, h, v->v.f.p, false);
    });
}

int fwi_dev_vec_copy(fwi_dev_vec* dst, const fwi_dev_vec* src) {
    return guard([&] {
        need(dst, "dst");
        need(src, "src");
        require(dst->v.ctx == src->v.ctx && dst->v.prec == src->v.prec, "vec_copy: shape mismatch");
        const Ctx& c = *src->v.ctx;
        if (src->v.prec == FWI_C128)
            CK(cudaMemcpyAsync(dst->v.d.p, src->v.d.p, src->v.d.bytes(), cudaMemcpyDeviceToDevice, c.stream));
        else
            CK(cudaMemcpyAsync(dst->v.f.p, src->v.f.p, src->v.f.bytes(), cudaMemcpyDeviceToDevice, c.stream));
    });
}

int fwi_dev_vec_zero(fwi_dev_vec* v) {
    return guard([&] {
        need(v, "vec");
        const Ctx& c = *v->v.ctx;
        if (v->v.prec == FWI_C128)
            CK(cudaMemsetAsync(v->v.d.p, 0, v->v.d.bytes(), c.stream));
        else
            CK(cudaMemsetAsync(v->v.f.p, 0, v->v.f.bytes(), c.stream));
    });
}

int fwi_dev_vec_dot(const fwi_dev_vec* x, const fwi_dev_vec* y, double* out) {
    return guard([&] {
        need(x, "x");
        need(y, "y");
        need(out, "out");
        require(x->v.ctx == y->v.ctx, "KktVector dot: block mismatch");
        require(x->v.prec == FWI_C128 && y->v.prec == FWI_C128, "dot: complex128 vectors required");
        Ctx& c = *x->v.ctx;
        *out = dev_dot(&c, c.stream, x->v.d.p, y->v.d.p, c.vec_len);
    });
}

int fwi_dev_vec_norm(const fwi_dev_vec* x, double* out) {
    return guard([&] {
        need(x, "x");
        need(out, "out");
        require(x->v.prec == FWI_C128, "norm: complex128 vector required");
        Ctx& c = *x->v.ctx;
        *out = std::sqrt(dev_dot(&c, c.stream, x->v.d.p, x->v.d.p, c.vec_len));
    });
}

int fwi_dev_vec_axpy(double a, const fwi_dev_vec* x, fwi_dev_vec* y) {
    return guard([&] {
        need(x, "x");
        need(y, "y");
        require(x->v.ctx == y->v.ctx && x->v.prec == FWI_C128 && y->v.prec == FWI_C128,
                "axpy: shape mismatch");
        Ctx& c = *x->v.ctx;
        dev_axpy(c.stream, a, x->v.d.p, y->v.d.p, c.vec_len);
    });
}

int fwi_dev_vec_scal(double a, fwi_dev_vec* x) {
    return guard([&] {
        need(x, "x");
        require(x->v.prec == FWI_C128, "scal: complex128 vector required");
        Ctx& c = *x->v.ctx;
        dev_scal(c.stream, a, x->v.d.p, c.vec_len);
    });
}

int fwi_dev_vec_device_ptr(const fwi_dev_vec* v, void** out) {
    return guard([&] {
        need(v, "vec");
        need(out, "out");
        *out = v->v.prec == FWI_C128 ? static_cast<void*>(v->v.d.p) : static_cast<void*>(v->v.f.p);
    });
}

int fwi_dev_kkt_apply(fwi_dev_ctx* ctx, const fwi_dev_vec* xi, fwi_dev_vec* out) {
    return guard([&] {
        need(ctx, "ctx");
        need(xi, "xi");
        need(out, "out");
        kkt_apply(*ctx->c, xi->v, out->v);
    });
}

int fwi_dev_kkt_apply_host(fwi_dev_ctx* ctx, const double* xi_host, double* out_host) {
    return guard([&] {
        need(ctx, "ctx");
        need(xi_host, "xi");
        need(out_host, "out");
        kkt_apply_host(*ctx->c, xi_host, out_host);
    });
}

int fwi_dev_kkt_rhs(fwi_dev_ctx* ctx, fwi_dev_vec* out) {
    return guard([&] {
        need(ctx, "ctx");
        need(out, "out");
        kkt_rhs(*ctx->c, out->v);
    });
}

int fwi_dev_precond_apply(fwi_dev_ctx* ctx, int mode, const fwi_dev_vec* v, fwi_dev_vec* out) {
    return guard([&] {
        need(ctx, "ctx");
        need(v, "v");
        need(out, "out");
        precond_apply(*ctx->c, mode, v->v, out->v);
    });
}

int fwi_dev_fsgn_gmres_step(fwi_dev_ctx* ctx, const fwi_fsgn_options* opt, double* ds, fwi_convergence_log* log) {
    return guard([&] {
        need(ctx, "ctx");
        need(opt, "options");
        fsgn_gmres_step(*ctx->c, *opt, ds, log);
    });
}

int fwi_dev_gradient(fwi_dev_ctx* ctx, double* g_host) {
    return guard([&] {
        need(ctx, "ctx");
        need(g_host, "g");
        Ctx& c = *ctx->c;
        require(c.exact != nullptr, "gradient: state has no exact factorization");
        DevBuf<double> g(c.n);
        reduced_gradient(c, g.p);
        CK(cudaMemcpyAsync(g_host, g.p, c.n * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
        CK(cudaStreamSynchronize(c.stream));
    });
}

int fwi_dev_hessian_apply(fwi_dev_ctx* ctx, const double* v_host, double* out_host) {
    return guard([&] {
        need(ctx, "ctx");
        need(v_host, "v");
        need(out_host, "out");
        Ctx& c = *ctx->c;
        require(c.exact != nullptr, "hessian_apply: state has no exact factorization");
        DevBuf<double> v(c.n), h(c.n);
        CK(cudaMemcpyAsync(v.p, v_host, c.n * sizeof(double), cudaMemcpyHostToDevice, c.stream));
        reduced_hessian(c, v.p, h.p);
        CK(cudaMemcpyAsync(out_host, h.p, c.n * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
        CK(cudaStreamSynchronize(c.stream));
    });
}

int fwi_dev_rsgn_cg_step(fwi_dev_ctx* ctx, double tol, int maxit, double* ds, fwi_convergence_log* log) {
    return guard([&] {
        need(ctx, "ctx");
        rsgn_cg_step(*ctx->c, tol, maxit, ds, log);
    });
}

int fwi_dev_gn_step(const fwi_state_desc* desc, const fwi_gn_options* opt, double* s_out,
                    fwi_gn_result* result, fwi_convergence_log* log) {
    return guard([&] {
        need(desc, "desc");
        need(opt, "options");
        need(s_out, "s_out");
        need(result, "result");
        gn_step(*desc, *opt, s_out, result, log);
    });
}

int fwi_dev_gmres_generic(int64_t n, fwi_op_cb apply, fwi_op_cb precond, fwi_observer_cb observer,
                          void* user, const double* b, double* x, int restart, double tol, int maxit,
                          fwi_convergence_log* log) {
    return guard([&] {
        need(reinterpret_cast<const void*>(apply), "apply");
        need(reinterpret_cast<const void*>(precond), "precond");
        need(b, "b");
        need(x, "x");
        gmres_generic(n, apply, precond, observer, user, b, x, restart, tol, maxit, log);
    });
}

int fwi_dev_malloc(void** out, int64_t bytes) {
    return guard([&] {
        need(out, "out");
        CK(cudaMalloc(out, size_t(bytes)));
    });
}

int fwi_dev_free(void* p) {
    return guard([&] { CK(cudaFree(p)); });
}

int fwi_dev_memcpy_h2d(void* dst, const void* src, int64_t bytes) {
    return guard([&] { CK(cudaMemcpy(dst, src, size_t(bytes), cudaMemcpyHostToDevice)); });
}

int fwi_dev_memcpy_d2h(void* dst, const void* src, int64_t bytes) {
    return guard([&] { CK(cudaMemcpy(dst, src, size_t(bytes), cudaMemcpyDeviceToHost)); });
}

int fwi_host_register(void* host, int64_t bytes) {
    return guard([&] { CK(cudaHostRegister(host, size_t(bytes), cudaHostRegisterDefault)); });
}

int fwi_host_unregister(void* host) {
    return guard([&] { CK(cudaHostUnregister(host)); });
}

int fwi_host_alloc(void** out, int64_t bytes) {
    return guard([&] {
        need(out, "out");
        require(bytes >= 0, "fwi_host_alloc: negative size");
        *out = pinned_alloc(size_t(bytes));
    });
}

int fwi_host_free(void* host) {
    return guard([&] {
        if (!pinned_free(host)) CK(cudaFreeHost(host));
    });
}

}  // extern "C"
