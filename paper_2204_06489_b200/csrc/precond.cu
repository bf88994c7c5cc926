// precond.cu — the block-triangular preconditioner (precond_apply,
// src/kkt.cpp:114-135) and the reduced-space actions the E_cg observer needs
// (gradient / hessian_apply / normal_residual, src/reduced_space.cpp:120-161).
//
//   (1) lambda_k = A^{-H} v.du_k                      all K sources in one batched solve
//   (2) ds       = (v.ds + sum_k Re(w^2 conj(u_k) lambda_k)) / eps   (k in order)
//   (3) du_k     = A^{-1} (w^2 u_k ds + v.la_k)       RHS built in one fused pass
//
// Steps (2) and (3)'s RHS follow the reference's rounding order exactly; the
// block solves are the exact block solver (exact.cu) or the bit-faithful ILU
// sweeps (ilu.cu). Each batched solve advances the solve counter by K, so one
// apply costs exactly 2K solve pairs as the reference's cost contract states
// (tests/test_kkt.cpp:153-159).
#include "ctx.cuh"

namespace fwi_b200 {

namespace {

__global__ void precond_ds_kernel(int K, int64_t n, double w2, double eps,
                                  const double2* __restrict__ u, const double2* __restrict__ la,
                                  const double* __restrict__ vds, double* __restrict__ ods) {
    pdl_enter();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        double pl = 0.0;
#pragma unroll 8
        for (int k = 0; k < K; ++k) {
            const double2 uc = u[int64_t(k) * n + i], z = la[int64_t(k) * n + i];
            const double a = __dmul_rn(uc.x, w2), b = __dmul_rn(-uc.y, w2);
            pl = __dadd_rn(pl, __dsub_rn(__dmul_rn(a, z.x), __dmul_rn(b, z.y)));
        }
        ods[i] = __ddiv_rn(__dadd_rn(vds[i], pl), eps);
    }
}

// rhs_k = (w2 * u_k) * ds + v.la_k
__global__ void precond_rhs_kernel(int64_t kn, int64_t n, double w2, const double2* __restrict__ u,
                                   const double* __restrict__ ds, const double2* __restrict__ vla,
                                   double2* __restrict__ rhs) {
    pdl_enter();
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < kn;
         t += int64_t(gridDim.x) * blockDim.x) {
        const double2 uc = u[t];
        const double d = ds[t % n];
        const double2 p = make_double2(__dmul_rn(__dmul_rn(w2, uc.x), d), __dmul_rn(__dmul_rn(w2, uc.y), d));
        rhs[t] = cadd(p, vla[t]);
    }
}

// hessian_apply / gradient building blocks ---------------------------------

// rhs_k = P_k v = (w2 u_k) v
__global__ void apply_p_kernel(int64_t kn, int64_t n, double w2, const double2* __restrict__ u,
                               const double* __restrict__ v, double2* __restrict__ out) {
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < kn;
         t += int64_t(gridDim.x) * blockDim.x) {
        const double2 uc = u[t];
        const double d = v[t % n];
        out[t] = make_double2(__dmul_rn(__dmul_rn(w2, uc.x), d), __dmul_rn(__dmul_rn(w2, uc.y), d));
    }
}

// y_k = Q_k^H (W^2 Q_k x_k)  (hessian)   or   y_k = Q_k^H (W^2 r_k)  (gradient);
// one thread per source keeps the data order for duplicate receivers.
__global__ void weighted_scatter_kernel(int K, int64_t n, const int* __restrict__ off,
                                        const int* __restrict__ node, const double* __restrict__ w,
                                        const double2* __restrict__ x, const double2* __restrict__ r,
                                        double2* __restrict__ y) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    for (int j = off[k]; j < off[k + 1]; ++j) {
        const double ww = __dmul_rn(w[j], w[j]);
        const double2 d = x ? x[int64_t(k) * n + node[j]] : r[j];
        double2& t = y[int64_t(k) * n + node[j]];
        t = cadd(t, rmul(ww, d));
    }
}

// out = Re(sum_k w2 conj(u_k) z_k) (+ eps v | - eps s)
__global__ void reduce_padj_kernel(int K, int64_t n, double w2, const double2* __restrict__ u,
                                   const double2* __restrict__ z, const double* __restrict__ add_v,
                                   double add_scale, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        double2 acc = make_double2(0.0, 0.0);
        for (int k = 0; k < K; ++k) {
            const double2 uc = u[int64_t(k) * n + i];
            const double2 a = make_double2(__dmul_rn(w2, uc.x), __dmul_rn(w2, -uc.y));
            acc = cadd(acc, cmul(a, z[int64_t(k) * n + i]));
        }
        double r = acc.x;
        if (add_v) r = __dadd_rn(r, __dmul_rn(add_scale, add_v[i]));
        out[i] = r;
    }
}

int ew(int64_t m) { return grid_blocks(m, 256, 16 * sm_count()); }

}  // namespace

void block_solve(Ctx& c, int mode, bool adjoint, const double2* b, double2* x, int nrhs) {
    if (mode == FWI_PRECOND_ILU)
        ilu_solve_batch(c, adjoint, b, x, nrhs);
    else if (mode == FWI_PRECOND_EXACT)
        exact_solve_batch(c, adjoint, b, x, nrhs);
    else
        throw FwiError(FWI_ERR_INVALID_ARGUMENT, "precond_apply: unknown mode");
}

void precond_apply_raw(Ctx& c, int mode, const double* v, double* out) {
    if (mode == FWI_PRECOND_ILU) require(c.ilu != nullptr, "precond_apply: state has no ILU factorization");
    if (mode == FWI_PRECOND_EXACT) require(c.exact != nullptr, "precond_apply: state has no exact factorization");
    const int K = c.K;
    const int64_t n = c.n, kn = int64_t(K) * n;
    double* vv = const_cast<double*>(v);
    // (1)
    block_solve(c, mode, true, c.du_of(vv), c.la_of(out), K);
    // (2)
    launch_pdl<kPdlPrecond>(precond_ds_kernel, dim3(ew(n)), dim3(256), 0, c.stream, K, n, c.w2, c.eps, c.u.p,
                            c.la_of(out), c.ds_of(vv), c.ds_of(out));
    CK_LAUNCH();
    // (3)
    // the right-hand side is built in out.du and solved in place (both block solvers
    // read their whole input before writing)
    launch_pdl<kPdlPrecond>(precond_rhs_kernel, dim3(ew(kn)), dim3(256), 0, c.stream, kn, n, c.w2, c.u.p, c.ds_of(out),
                            c.la_of(vv), c.du_of(out));
    CK_LAUNCH();
    block_solve(c, mode, false, c.du_of(out), c.du_of(out), K);
}

void precond_apply(Ctx& c, int mode, const Vec& v, Vec& out) {
    require(v.ctx == &c && out.ctx == &c, "KktVector does not conform to the state");
    require(v.prec == FWI_C128 && out.prec == FWI_C128, "precond_apply: complex128 vectors required");
    require(&v != &out, "precond_apply: output must not alias the input");
    precond_apply_raw(c, mode, v.d.p, out.d.p);
}

// g = Re(J^H W^T W r) - eps s (gradient, src/reduced_space.cpp:141-152)
void reduced_gradient(Ctx& c, double* g_dev) {
    const int K = c.K;
    const int64_t n = c.n, kn = int64_t(K) * n;
    // scratch of its own (freed on return): the gradient runs once per Newton step and
    // must not keep K x n of HBM from the Krylov basis at config 5
    DevBuf<double2> a(kn);
    CK(cudaMemsetAsync(a.p, 0, kn * sizeof(double2), c.stream));
    if (c.ndata)
        weighted_scatter_kernel<<<(K + 127) / 128, 128, 0, c.stream>>>(
            K, n, c.recv_offset.p, c.recv_node.p, c.w.p, nullptr, c.r.p, a.p);
    CK_LAUNCH();
    exact_solve_batch(c, true, a.p, a.p, K);  // in place
    reduce_padj_kernel<<<ew(n), 256, 0, c.stream>>>(K, n, c.w2, c.u.p, a.p, c.drop ? nullptr : c.s.p, -c.eps,
                                                   g_dev);
    CK_LAUNCH();
    CK(cudaStreamSynchronize(c.stream));
}

// H v = Re(J^H W^T W J v) + eps v (hessian_apply, src/reduced_space.cpp:120-139)
void reduced_hessian(Ctx& c, const double* v_dev, double* out_dev) {
    c.ensure_work(Ctx::kWorkA | Ctx::kWorkB);
    const int K = c.K;
    const int64_t n = c.n, kn = int64_t(K) * n;
    apply_p_kernel<<<ew(kn), 256, 0, c.stream>>>(kn, n, c.w2, c.u.p, v_dev, c.work_a.p);
    CK_LAUNCH();
    exact_solve_batch(c, false, c.work_a.p, c.work_b.p, K);
    CK(cudaMemsetAsync(c.work_a.p, 0, kn * sizeof(double2), c.stream));
    if (c.ndata)
        weighted_scatter_kernel<<<(K + 127) / 128, 128, 0, c.stream>>>(
            K, n, c.recv_offset.p, c.recv_node.p, c.w.p, c.work_b.p, nullptr, c.work_a.p);
    CK_LAUNCH();
    exact_solve_batch(c, true, c.work_a.p, c.work_b.p, K);
    reduce_padj_kernel<<<ew(n), 256, 0, c.stream>>>(K, n, c.w2, c.u.p, c.work_b.p, v_dev, c.eps, out_dev);
    CK_LAUNCH();
}

}  // namespace fwi_b200
