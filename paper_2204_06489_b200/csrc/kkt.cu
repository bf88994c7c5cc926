// kkt.cu — K1: the fused, source-batched KKT operator apply and the KKT
// right-hand side.
//
// Reference: kkt_apply (src/kkt.cpp:78-96) with apply_f (:50-58),
// apply_p (:60-66), accumulate_re_p_adjoint (:68-74) and spmv
// (src/sparse.cpp:69-91); kkt_rhs (src/kkt.cpp:98-112).
//
//   out.du_k = F_k du_k + A^H lambda_k
//   out.la_k = A du_k - w^2 u_k * ds
//   out.ds   = eps ds - sum_k Re(w^2 conj(u_k) lambda_k)      (k = 0..K-1 in order)
//
// One pass: each thread owns one grid node, loads its five stencil
// coefficients once, then walks the K sources in order, reading du_k, la_k and
// u_k at the node (and du_k, la_k at the 4 neighbours, served from L1 by the
// neighbouring threads of the CTA tile), writing out.du_k and out.la_k, and
// carrying the ds row's K-sum in a register. A(i,i-1) and A(i,i-nx) come from
// the east/south planes of the neighbours (exact complex symmetry),
// and A^H lambda is a gather with conjugated coefficients in ascending row
// order — the same summation order as the reference's column scatter, so the
// complex128 result is bit-identical to the reference.
#include "arith.cuh"
#include <cstdlib>

#include "ctx.cuh"

#include <algorithm>

namespace fwi_b200 {

namespace {

template <class A>
__global__ void __launch_bounds__(256) kkt_apply_kernel(
    int nx, int nz, int K, int64_t n, typename A::R w2, typename A::R eps,
    const typename A::T* __restrict__ diag, const typename A::T* __restrict__ east,
    const typename A::T* __restrict__ south, const typename A::T* __restrict__ u,
    const int* __restrict__ nrec_ptr, const int* __restrict__ nrec_k,
    const double* __restrict__ nrec_w2, const typename A::T* __restrict__ du,
    const typename A::R* __restrict__ ds, const typename A::T* __restrict__ la,
    typename A::T* __restrict__ odu, typename A::R* __restrict__ ods, typename A::T* __restrict__ ola,
    int k0, int k1, typename A::R* __restrict__ plbuf) {
    pdl_enter();
    // Sources [k0, k1) only (the pipelined host-buffer apply streams source
    // chunks); the ds row's running sum continues from plbuf when k0 > 0 and
    // is written back to plbuf unless the chunk ends at K.
    using T = typename A::T;
    using R = typename A::R;
    const int ix = blockIdx.x * blockDim.x + threadIdx.x;
    const int iz = blockIdx.y * blockDim.y + threadIdx.y;
    if (ix >= nx || iz >= nz) return;
    const int64_t c = int64_t(iz) * nx + ix;
    const bool bnd = on_boundary(ix, iz, nx, nz);
    const bool hN = !bnd && !on_boundary(ix, iz - 1, nx, nz);
    const bool hW = !bnd && !on_boundary(ix - 1, iz, nx, nz);
    const bool hE = !bnd && !on_boundary(ix + 1, iz, nx, nz);
    const bool hS = !bnd && !on_boundary(ix, iz + 1, nx, nz);
    const T cD = diag[c];
    const T cN = hN ? south[c - nx] : A::zero();
    const T cW = hW ? east[c - 1] : A::zero();
    const T cE = hE ? east[c] : A::zero();
    const T cS = hS ? south[c] : A::zero();
    const R dsv = ds[c];
    int q = nrec_ptr[c];
    const int qe = nrec_ptr[c + 1];
    while (q < qe && nrec_k[q] < k0) ++q;
    R pl = k0 > 0 ? plbuf[c] : R(0);
    for (int k = k0; k < k1; ++k) {
        const int64_t o = int64_t(k) * n + c;
        // row 3: A du - P ds (ascending column order: -nx, -1, 0, +1, +nx)
        T s = A::zero();
        T t = A::zero();
        if (hN) {
            s = A::add(s, A::mul(cN, du[o - nx]));
            t = A::add(t, A::mulc(cN, la[o - nx]));
        }
        if (hW) {
            s = A::add(s, A::mul(cW, du[o - 1]));
            t = A::add(t, A::mulc(cW, la[o - 1]));
        }
        const T duc = du[o];
        const T lac = la[o];
        s = A::add(s, A::mul(cD, duc));
        t = A::add(t, A::mulc(cD, lac));
        if (hE) {
            s = A::add(s, A::mul(cE, du[o + 1]));
            t = A::add(t, A::mulc(cE, la[o + 1]));
        }
        if (hS) {
            s = A::add(s, A::mul(cS, du[o + nx]));
            t = A::add(t, A::mulc(cS, la[o + nx]));
        }
        const T uc = u[o];
        ola[o] = A::sub(s, A::pmul(w2, uc, dsv));
        // row 1: F du + A^H lambda; F accumulates duplicate receivers in data order
        if (q < qe && nrec_k[q] == k) {
            T f = A::zero();
            while (q < qe && nrec_k[q] == k) {
                f = A::add(f, A::rm(R(nrec_w2[q]), duc));
                ++q;
            }
            t = A::add(f, t);
        }
        odu[o] = t;
        // row 2 partial sum, sources in order
        pl = A::radd(pl, A::re_pconj(w2, uc, lac));
    }
    if (k1 == K)
        ods[c] = A::rsub(A::rmulr(eps, dsv), pl);
    else
        plbuf[c] = pl;
}

// The same apply for small problems with the sources spread over threads: one thread per (node,
// source slot), a CTA = 32 nodes of a row x 8 source slots (config 1: 256 CTAs instead of 32 with
// the node-per-thread kernel, whose threads walk all K sources). Each (node, source) output is
// computed exactly as above; the ds row's K-sum is taken in source order from shared memory by the
// slot-0 thread of each node, so the result is bit-identical.
constexpr int kKsNodes = 32, kKsSlots = 8, kKsMaxK = 64;
template <class A>
__global__ void __launch_bounds__(kKsNodes * kKsSlots) kkt_apply_ks_kernel(
    int nx, int nz, int K, int64_t n, typename A::R w2, typename A::R eps,
    const typename A::T* __restrict__ diag, const typename A::T* __restrict__ east,
    const typename A::T* __restrict__ south, const typename A::T* __restrict__ u,
    const int* __restrict__ nrec_ptr, const int* __restrict__ nrec_k,
    const double* __restrict__ nrec_w2, const typename A::T* __restrict__ du,
    const typename A::R* __restrict__ ds, const typename A::T* __restrict__ la,
    typename A::T* __restrict__ odu, typename A::R* __restrict__ ods, typename A::T* __restrict__ ola) {
    pdl_enter();
    using T = typename A::T;
    using R = typename A::R;
    __shared__ R pterm[kKsMaxK][kKsNodes];
    const int lx = threadIdx.x, ks = threadIdx.y;
    const int ix = blockIdx.x * kKsNodes + lx, iz = blockIdx.y;
    const bool in = ix < nx;
    const int64_t c = int64_t(iz) * nx + (in ? ix : 0);
    if (in) {
        const bool bnd = on_boundary(ix, iz, nx, nz);
        const bool hN = !bnd && !on_boundary(ix, iz - 1, nx, nz);
        const bool hW = !bnd && !on_boundary(ix - 1, iz, nx, nz);
        const bool hE = !bnd && !on_boundary(ix + 1, iz, nx, nz);
        const bool hS = !bnd && !on_boundary(ix, iz + 1, nx, nz);
        const T cD = diag[c];
        const T cN = hN ? south[c - nx] : A::zero();
        const T cW = hW ? east[c - 1] : A::zero();
        const T cE = hE ? east[c] : A::zero();
        const T cS = hS ? south[c] : A::zero();
        const R dsv = ds[c];
        const int q0 = nrec_ptr[c], qe = nrec_ptr[c + 1];
        for (int k = ks; k < K; k += kKsSlots) {
            const int64_t o = int64_t(k) * n + c;
            T s_ = A::zero();
            T t_ = A::zero();
            if (hN) {
                s_ = A::add(s_, A::mul(cN, du[o - nx]));
                t_ = A::add(t_, A::mulc(cN, la[o - nx]));
            }
            if (hW) {
                s_ = A::add(s_, A::mul(cW, du[o - 1]));
                t_ = A::add(t_, A::mulc(cW, la[o - 1]));
            }
            const T duc = du[o];
            const T lac = la[o];
            s_ = A::add(s_, A::mul(cD, duc));
            t_ = A::add(t_, A::mulc(cD, lac));
            if (hE) {
                s_ = A::add(s_, A::mul(cE, du[o + 1]));
                t_ = A::add(t_, A::mulc(cE, la[o + 1]));
            }
            if (hS) {
                s_ = A::add(s_, A::mul(cS, du[o + nx]));
                t_ = A::add(t_, A::mulc(cS, la[o + nx]));
            }
            const T uc = u[o];
            ola[o] = A::sub(s_, A::pmul(w2, uc, dsv));
            int q = q0;
            while (q < qe && nrec_k[q] < k) ++q;
            if (q < qe && nrec_k[q] == k) {
                T f = A::zero();
                while (q < qe && nrec_k[q] == k) {
                    f = A::add(f, A::rm(R(nrec_w2[q]), duc));
                    ++q;
                }
                t_ = A::add(f, t_);
            }
            odu[o] = t_;
            pterm[k][lx] = A::re_pconj(w2, uc, lac);
        }
    }
    __syncthreads();
    if (in && ks == 0) {
        R pl = R(0);
        for (int k = 0; k < K; ++k) pl = A::radd(pl, pterm[k][lx]);
        ods[c] = A::rsub(A::rmulr(eps, ds[c]), pl);
    }
}

// kkt_rhs (src/kkt.cpp:98-112): b = (Q^H W^T W r scattered per source,
// -eps s or 0, 0). One thread per source keeps the reference's data order
// for duplicate receivers.
__global__ void kkt_rhs_scatter(int K, int64_t n, const int* __restrict__ off,
                                const int* __restrict__ node, const double* __restrict__ w,
                                const double2* __restrict__ r, double2* __restrict__ du) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    for (int j = off[k]; j < off[k + 1]; ++j) {
        const double ww = __dmul_rn(w[j], w[j]);
        double2& d = du[int64_t(k) * n + node[j]];
        d = cadd(d, rmul(ww, r[j]));
    }
}

__global__ void kkt_rhs_ds(int64_t n, double neg_eps, const double* __restrict__ s,
                           double* __restrict__ ds) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        ds[i] = __dmul_rn(neg_eps, s[i]);
}

}  // namespace

void kkt_apply_raw(Ctx& c, const double* xi, double* out) {
    if (c.kkt_variant != 1 && kkt_apply_tma(c, false, xi, out)) return;
    double* x = const_cast<double*>(xi);
    // small problems: sources over threads (FWI_KKT_KS=0 keeps the node-per-thread kernel)
    const bool ks_off = std::getenv("FWI_KKT_KS") && std::atoi(std::getenv("FWI_KKT_KS")) == 0;
    if (!ks_off && c.K <= kKsMaxK) {
        launch_pdl<kPdlKkt>(kkt_apply_ks_kernel<F64>, dim3((c.nx + kKsNodes - 1) / kKsNodes, c.nz),
                            dim3(kKsNodes, kKsSlots), 0, c.stream, c.nx, c.nz, c.K, c.n, c.w2, c.eps, c.diag.p,
                            c.east.p, c.south.p, c.u.p, c.nrec_ptr.p, c.nrec_k.p, c.nrec_w2.p, c.du_of(x),
                            c.ds_of(x), c.la_of(x), c.du_of(out), c.ds_of(out), c.la_of(out));
        CK_LAUNCH();
        c.kkt_kernel[0] = "kkt_apply_ks_kernel<F64> (plain K1, sources over threads, csrc/kkt.cu)";
        return;
    }
    dim3 blk(32, 8), grd((c.nx + 31) / 32, (c.nz + 7) / 8);
    launch_pdl<kPdlKkt>(kkt_apply_kernel<F64>, dim3(grd), dim3(blk), 0, c.stream, c.nx, c.nz, c.K, c.n, c.w2, c.eps,
                        c.diag.p, c.east.p, c.south.p, c.u.p, c.nrec_ptr.p, c.nrec_k.p, c.nrec_w2.p, c.du_of(x),
                        c.ds_of(x), c.la_of(x), c.du_of(out), c.ds_of(out), c.la_of(out), 0, c.K, nullptr);
    CK_LAUNCH();
    c.kkt_kernel[0] = "kkt_apply_kernel<F64> (plain K1, csrc/kkt.cu)";
}

void kkt_apply_raw_on(Ctx& c, const double* xi, double* out, cudaStream_t s) {
    // the chunked tile kernel's plan holds its work counters: a concurrent apply needs its own
    struct Swap {
        Ctx& c;
        cudaStream_t s0;
        Swap(Ctx& cc, cudaStream_t s) : c(cc), s0(cc.stream) {
            c.stream = s;
            std::swap(c.kplan, c.kplan_alt);
        }
        ~Swap() {
            std::swap(c.kplan, c.kplan_alt);
            c.stream = s0;
        }
    } sw(c, s);
    kkt_apply_raw(c, xi, out);
}

// kkt_apply on host buffers (the reference's own signature,
// src/kkt.cpp:78): the flat input is streamed in source chunks on one copy
// stream, each chunk is applied as soon as it lands, and its output block
// streams back on a second copy stream, so H2D, compute and D2H overlap. The
// ds row's K-sum is carried across chunks in source order (bit-exact).
void kkt_apply_host(Ctx& c, const double* in, double* out) {
    const int K = c.K;
    const int64_t n = c.n, kn2 = 2 * int64_t(K) * n;
    if (!c.hx.p) {
        c.hx.alloc(c.vec_len);
        c.hy.alloc(c.vec_len);
        c.hpl.alloc(c.ds_stride);
        CK(cudaMemset(c.hx.p, 0, c.hx.bytes()));
        CK(cudaMemset(c.hy.p, 0, c.hy.bytes()));
        CK(cudaStreamCreateWithFlags(&c.s_h2d, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&c.s_d2h, cudaStreamNonBlocking));
        for (int i = 0; i < Ctx::kMaxChunks; ++i) {
            CK(cudaEventCreateWithFlags(&c.ev_in[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&c.ev_out[i], cudaEventDisableTiming));
        }
    }
    static const int want = std::getenv("FWI_HOST_CHUNKS") ? std::atoi(std::getenv("FWI_HOST_CHUNKS")) : 16;
    const int nch = std::max(1, std::min(K, std::min(want, Ctx::kMaxChunks)));
    double* x = c.hx.p;
    double* y = c.hy.p;
    const size_t cb = sizeof(double2);
    const int64_t dev_la = kn2 + c.ds_stride, host_la = kn2 + n;
    // the previous call's D2H must be done before this call reuses y (stream order)
    CK(cudaMemcpyAsync(c.ds_of(x), in + kn2, n * sizeof(double), cudaMemcpyHostToDevice, c.s_h2d));
    dim3 blk(32, 8), grd((c.nx + 31) / 32, (c.nz + 7) / 8);
    for (int ch = 0; ch < nch; ++ch) {
        const int k0 = int(int64_t(K) * ch / nch), k1 = int(int64_t(K) * (ch + 1) / nch);
        const size_t off = size_t(k0) * n, cnt = size_t(k1 - k0) * n;
        CK(cudaMemcpyAsync(c.du_of(x) + off, in + 2 * off, cnt * cb, cudaMemcpyHostToDevice, c.s_h2d));
        CK(cudaMemcpyAsync(c.la_of(x) + off, in + host_la + 2 * off, cnt * cb, cudaMemcpyHostToDevice,
                           c.s_h2d));
        CK(cudaEventRecord(c.ev_in[ch], c.s_h2d));
        CK(cudaStreamWaitEvent(c.stream, c.ev_in[ch], 0));
        launch_pdl<kPdlKkt>(kkt_apply_kernel<F64>, dim3(grd), dim3(blk), 0, c.stream, c.nx, c.nz, K, n, c.w2, c.eps,
                            c.diag.p, c.east.p, c.south.p, c.u.p, c.nrec_ptr.p, c.nrec_k.p, c.nrec_w2.p, c.du_of(x),
                            c.ds_of(x), c.la_of(x), c.du_of(y), c.ds_of(y), c.la_of(y), k0, k1, c.hpl.p);
        CK_LAUNCH();
        CK(cudaEventRecord(c.ev_out[ch], c.stream));
        CK(cudaStreamWaitEvent(c.s_d2h, c.ev_out[ch], 0));
        CK(cudaMemcpyAsync(out + 2 * off, c.du_of(y) + off, cnt * cb, cudaMemcpyDeviceToHost, c.s_d2h));
        CK(cudaMemcpyAsync(out + host_la + 2 * off, c.la_of(y) + off, cnt * cb, cudaMemcpyDeviceToHost,
                           c.s_d2h));
    }
    CK(cudaMemcpyAsync(out + kn2, c.ds_of(y), n * sizeof(double), cudaMemcpyDeviceToHost, c.s_d2h));
    CK(cudaStreamSynchronize(c.s_d2h));
    (void)dev_la;
}

void kkt_apply(Ctx& c, const Vec& xi, Vec& out) {
    require(xi.ctx == &c && out.ctx == &c, "KktVector does not conform to the state");
    require(xi.prec == out.prec, "kkt_apply: precision mismatch");
    require(&xi != &out, "kkt_apply: output must not alias the input");
    if (xi.prec == FWI_C128) {
        kkt_apply_raw(c, xi.d.p, out.d.p);
        return;
    }
    require(c.u32.p != nullptr, "kkt_apply: context was created without the complex64 copy");
    if (c.kkt_variant != 1 && kkt_apply_tma(c, true, xi.f.p, out.f.p)) return;
    dim3 blk(32, 8), grd((c.nx + 31) / 32, (c.nz + 7) / 8);
    const int64_t kn2 = 2 * int64_t(c.K) * c.n;
    float* x = const_cast<float*>(xi.f.p);
    float* o = out.f.p;
    launch_pdl<kPdlKkt>(kkt_apply_kernel<F32>, dim3(grd), dim3(blk), 0, c.stream, c.nx, c.nz, c.K, c.n, float(c.w2),
                        float(c.eps), c.diag32.p, c.east32.p, c.south32.p, c.u32.p, c.nrec_ptr.p, c.nrec_k.p,
                        c.nrec_w2.p, reinterpret_cast<float2*>(x), x + kn2,
                        reinterpret_cast<float2*>(x + kn2 + c.ds_stride), reinterpret_cast<float2*>(o), o + kn2,
                        reinterpret_cast<float2*>(o + kn2 + c.ds_stride), 0, c.K, nullptr);
    CK_LAUNCH();
    c.kkt_kernel[1] = "kkt_apply_kernel<F32> (plain K1, csrc/kkt.cu)";
}

void kkt_rhs(Ctx& c, Vec& out) {
    require(out.ctx == &c && out.prec == FWI_C128, "kkt_rhs: complex128 vector of this state required");
    CK(cudaMemsetAsync(out.d.p, 0, out.d.bytes(), c.stream));
    if (c.ndata)
        kkt_rhs_scatter<<<(c.K + 127) / 128, 128, 0, c.stream>>>(c.K, c.n, c.recv_offset.p,
                                                                 c.recv_node.p, c.w.p, c.r.p,
                                                                 c.du_of(out.d.p));
    if (!c.drop)
        kkt_rhs_ds<<<grid_blocks(c.n, 256, 4 * sm_count()), 256, 0, c.stream>>>(
            c.n, -c.eps, c.s.p, c.ds_of(out.d.p));
    CK_LAUNCH();
}

}  // namespace fwi_b200
