// ilu.cu — ILU(p) block solver: host factorisation + batched, level-scheduled
// triangular sweeps on the device (K2/K4, inexact mode).
//
// Reference: IluFactors::factor (src/ilu.cpp:8-106), build_transposes
// (:108-129), solve (:131-174).
//
// The factorisation is per-Newton-step setup. It runs on the host in the
// same operation order as the reference (level-of-fill symbolic phase, IKJ
// numeric phase with the `lij == 0` skip, libgcc complex division), so the
// factors are bit-identical to the reference's and the inexact
// preconditioner reproduces the reference's output exactly. The four
// triangular sweeps (L, U forward; U^H, L^H adjoint) run on the device for
// all sources at once, one CTA per source (ilu_sweep_tma): rows grouped into
// dependency levels, each level in two phases — every thread forms products
// (lane per entry), then each row's owner subtracts them in the reference's
// entry order (bit-faithful) — with the level data streamed into shared
// memory by TMA bulk copies several levels ahead. The vector lives in shared
// memory (config 1), or in a ring indexed by level-ordered position when it
// is too large (config 3/4: operands lie < 700 positions behind their rows).
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <complex>
#include <cstdio>
#include <queue>
#include <string>

#include "ctx.cuh"

namespace fwi_b200 {

using cplx = std::complex<double>;

constexpr int kIluBatch = 8;  // entries per batch of the sweep kernels (row padding unit)
constexpr int kIluThreads = 256;  // sweep kernel block
constexpr int kIluEpl = 2;        // entries per thread and level (a level holds <= kIluThreads * kIluEpl)
constexpr int kIluRows = 128;     // rows per (sub-)level
constexpr int kIluRing = 4;       // TMA stage ring
constexpr int kIluAhead = 3;      // levels staged ahead
constexpr int kIluRingW = 2048;   // operand ring (positions) of the ring sweep, a power of two

struct Sweep {          // one triangular sweep in CSR form + its level schedule
    DevBuf<int> ptr, idx, lvl_ptr, lvl_rows;
    DevBuf<double2> val;
    // the same entries regrouped in level order: row lvl_rows[r] owns
    // entries [rstart[r], rstart[r+1]) of (lidx, lval), in the row's own order
    // (entries padded per row to a multiple of kIluBatch; diagonals of U / U^T in ldiag;
    // levels wider than the kernel are cut into consecutive sub-levels)
    DevBuf<int> rstart, lidx;
    DevBuf<int4> recs;      // per level-ordered row: {row, first entry, end entry (level-relative), position}
    DevBuf<int> lpos;       // operand level-ordered positions (ring sweep), -1 for padding
    bool ring_ok = false;
    DevBuf<double2> lval;
    DevBuf<double4> ldiag;  // per level-ordered row: divisor {ratio, denominator, |c| < |d|, 0}
    DevBuf<int4> lmeta;  // per level: first row, end row, first entry, end entry
    int nlev = 0;            // (sub-)levels of the two-phase kernel
    int nlev0 = 0;           // dependency levels (lvl_ptr)
    int ecap = 0, rcap = 0;  // max entries / rows of one (sub-)level
};

struct IluFactor {
    int level = 0;
    Sweep L, U, Ut, Lt;  // Ut/Lt: transposes for the adjoint
    int64_t bytes = 0;
    DevBuf<double2> zslot;  // the padding entries' operand (+0) when the vector is in global memory
    DevBuf<double2> blo;    // right-hand sides in level order (ring sweep scratch, nrhs x n)
};

void ilu_free(IluFactor* f) { delete f; }
int64_t ilu_bytes(const IluFactor* f) { return f ? f->bytes : 0; }

namespace {

// Host CSR of the assembled operator, built from the device stencil planes
// in ascending column order (as SparseMatrixCSR::from_triplets sorts them).
void host_csr(const Ctx& c, std::vector<int>& rp, std::vector<int>& ci, std::vector<cplx>& va) {
    std::vector<double2> d(c.n), e(c.n), s(c.n);
    stencil_to_host(c, &d[0].x, &e[0].x, &s[0].x);
    rp.assign(c.n + 1, 0);
    ci.clear();
    va.clear();
    ci.reserve(size_t(c.n) * 5);
    va.reserve(size_t(c.n) * 5);
    const int nx = c.nx, nz = c.nz;
    auto push = [&](int col, double2 v) {
        ci.push_back(col);
        va.emplace_back(v.x, v.y);
    };
    for (int iz = 0; iz < nz; ++iz)
        for (int ix = 0; ix < nx; ++ix) {
            const int i = iz * nx + ix;
            if (on_boundary(ix, iz, nx, nz)) {
                push(i, d[i]);
            } else {
                if (!on_boundary(ix, iz - 1, nx, nz)) push(i - nx, s[i - nx]);
                if (!on_boundary(ix - 1, iz, nx, nz)) push(i - 1, e[i - 1]);
                push(i, d[i]);
                if (!on_boundary(ix + 1, iz, nx, nz)) push(i + 1, e[i]);
                if (!on_boundary(ix, iz + 1, nx, nz)) push(i + nx, s[i]);
            }
            rp[i + 1] = int(ci.size());
        }
}

// levels of a DAG whose row i depends on the columns listed in (ptr, idx)
// excluding i itself; forward = dependencies point to smaller indices.
void build_levels(int n, const std::vector<int>& ptr, const std::vector<int>& idx, bool forward,
                  std::vector<int>& lvl_ptr, std::vector<int>& rows, int& nlev) {
    std::vector<int> lv(n, 0);
    nlev = 0;
    auto visit = [&](int i) {
        int l = 0;
        for (int p = ptr[i]; p < ptr[i + 1]; ++p) {
            const int j = idx[p];
            if (j != i) l = std::max(l, lv[j] + 1);
        }
        lv[i] = l;
        nlev = std::max(nlev, l + 1);
    };
    if (forward)
        for (int i = 0; i < n; ++i) visit(i);
    else
        for (int i = n - 1; i >= 0; --i) visit(i);
    lvl_ptr.assign(nlev + 1, 0);
    for (int i = 0; i < n; ++i) lvl_ptr[lv[i] + 1]++;
    for (int l = 0; l < nlev; ++l) lvl_ptr[l + 1] += lvl_ptr[l];
    std::vector<int> pos(lvl_ptr.begin(), lvl_ptr.end() - 1);
    rows.resize(n);
    for (int i = 0; i < n; ++i) rows[pos[lv[i]]++] = i;
}

void upload_sweep(Sweep& s, int n, const std::vector<int>& ptr, const std::vector<int>& idx,
                  const std::vector<cplx>& val, bool forward, bool has_diag, cudaStream_t st, int64_t& bytes) {
    std::vector<int> lp, rows;
    build_levels(n, ptr, idx, forward, lp, rows, s.nlev);
    s.nlev0 = s.nlev;
    auto up = [&](auto& buf, const auto& v) {
        using T = typename std::remove_reference_t<decltype(buf)>;
        (void)sizeof(T);
        buf.alloc(std::max<size_t>(v.size(), 1));
        if (!v.empty())
            CK(cudaMemcpyAsync(buf.p, v.data(), v.size() * sizeof(v[0]), cudaMemcpyHostToDevice, st));
        bytes += int64_t(v.size() * sizeof(v[0]));
    };
    up(s.ptr, ptr);
    up(s.idx, idx);
    up(s.lvl_ptr, lp);
    up(s.lvl_rows, rows);
    {
        // level order; per row the off-diagonal entries in the row's own order, padded to a
        // multiple of kIluBatch with (n, 0) entries; the diagonal (U: first, U^T: last) apart
        std::vector<int> rst(n + 1, 0), li;
        std::vector<cplx> lv, dg(n, cplx(1.0, 0.0));
        li.reserve(idx.size() + size_t(n) * kIluBatch);
        lv.reserve(val.size() + size_t(n) * kIluBatch);
        for (int r = 0; r < n; ++r) {
            const int i = rows[r];
            for (int q = ptr[i]; q < ptr[i + 1]; ++q) {
                if (idx[q] == i && has_diag) {
                    dg[r] = val[q];
                    continue;
                }
                li.push_back(idx[q]);
                lv.push_back(val[q]);
            }
            while (li.size() % kIluBatch) {
                li.push_back(n);
                lv.push_back(cplx(0.0, 0.0));
            }
            rst[r + 1] = int(li.size());
        }
        up(s.rstart, rst);
        // sub-levels: at most kIluThreads rows and kIluThreads * kIluEpl entries each
        std::vector<int> sp{0};
        for (int l = 0; l < s.nlev; ++l) {
            int r = lp[l];
            while (r < lp[l + 1]) {
                const int r0 = r;
                while (r < lp[l + 1] && r - r0 < kIluRows && rst[r + 1] - rst[r0] <= kIluThreads * kIluEpl) ++r;
                if (r == r0)
                    throw FwiError(FWI_ERR_NOT_SUPPORTED, "ILU sweep: a factor row holds more than " +
                                                             std::to_string(kIluThreads * kIluEpl) + " entries");
                sp.push_back(r);
            }
        }
        lp.swap(sp);
        s.nlev = int(lp.size()) - 1;
        s.ecap = s.rcap = 1;
        std::vector<int4> rec(n);
        for (int l = 0; l < s.nlev; ++l) {
            s.rcap = std::max(s.rcap, lp[l + 1] - lp[l]);
            s.ecap = std::max(s.ecap, rst[lp[l + 1]] - rst[lp[l]]);
            for (int r = lp[l]; r < lp[l + 1]; ++r)
                rec[r] = make_int4(rows[r], rst[r] - rst[lp[l]], rst[r + 1] - rst[lp[l]], r);
        }
        s.ecap = (s.ecap + kIluBatch - 1) / kIluBatch * kIluBatch;
        up(s.recs, rec);
        std::vector<int4> meta(s.nlev);
        for (int l = 0; l < s.nlev; ++l) meta[l] = make_int4(lp[l], lp[l + 1], rst[lp[l]], rst[lp[l + 1]]);
        up(s.lmeta, meta);
        up(s.lidx, li);
        // operand positions for the ring sweep (padding: -1) and whether the ring holds them
        {
            std::vector<int> pos(n + 1, -1), lpos(li.size());
            for (int r = 0; r < n; ++r) pos[rows[r]] = r;
            int maxd = 0;
            for (int r = 0; r < n; ++r)
                for (int q = rst[r]; q < rst[r + 1]; ++q) {
                    lpos[q] = pos[li[q]];
                    if (li[q] < n) maxd = std::max(maxd, r - pos[li[q]]);
                }
            s.ring_ok = maxd + kIluRows < kIluRingW;
            up(s.lpos, lpos);
        }
        s.lval.alloc(std::max<size_t>(lv.size(), 1));
        if (!lv.empty())
            CK(cudaMemcpyAsync(s.lval.p, lv.data(), lv.size() * sizeof(cplx), cudaMemcpyHostToDevice, st));
        bytes += int64_t(lv.size() * sizeof(cplx));
        if (has_diag) {
            // divisor of each row: U(i,i) (forward U sweep) or conj(U(i,i)) (the U^H sweep)
            std::vector<double4> q(n);
            for (int r = 0; r < n; ++r) {
                const double c = dg[r].real(), d = forward ? -dg[r].imag() : dg[r].imag();
                double rr, den;
                const bool small_c = host_cdiv_prep(c, d, rr, den);
                q[r] = make_double4(rr, den, small_c ? 1.0 : 0.0, 0.0);
            }
            s.ldiag.alloc(size_t(n));
            CK(cudaMemcpyAsync(s.ldiag.p, q.data(), size_t(n) * sizeof(double4), cudaMemcpyHostToDevice, st));
            CK(cudaStreamSynchronize(st));
            bytes += int64_t(n) * int64_t(sizeof(double4));
        }
    }
    s.val.alloc(std::max<size_t>(val.size(), 1));
    if (!val.empty())
        CK(cudaMemcpyAsync(s.val.p, val.data(), val.size() * sizeof(cplx), cudaMemcpyHostToDevice, st));
    bytes += int64_t(val.size() * sizeof(cplx));
    CK(cudaStreamSynchronize(st));
}

void transpose_csr(int n, const std::vector<int>& ptr, const std::vector<int>& idx,
                   const std::vector<cplx>& val, std::vector<int>& tp, std::vector<int>& ti,
                   std::vector<cplx>& tv) {
    tp.assign(n + 1, 0);
    for (int c : idx) tp[c + 1]++;
    for (int j = 0; j < n; ++j) tp[j + 1] += tp[j];
    ti.resize(idx.size());
    tv.resize(idx.size());
    std::vector<int> nx(tp.begin(), tp.end() - 1);
    for (int i = 0; i < n; ++i)  // rows ascending -> ascending order within each transposed row
        for (int p = ptr[i]; p < ptr[i + 1]; ++p) {
            const int q = nx[idx[p]]++;
            ti[q] = i;
            tv[q] = val[p];
        }
}

enum SweepKind { kLfwd = 0, kUbwd = 1, kUtfwd = 2, kLtbwd = 3 };

// One CTA per group of `kg` right-hand sides; levels in order with a barrier
// between them; each (row, rhs) item follows the reference's entry order.
template <int KIND>
__global__ void __launch_bounds__(256) ilu_sweep_kernel(int64_t n, int nrhs, int kg, int nlev,
                                                       const int* __restrict__ lvl_ptr,
                                                       const int* __restrict__ lvl_rows,
                                                       const int* __restrict__ ptr,
                                                       const int* __restrict__ idx,
                                                       const double2* __restrict__ val, double2* x) {
    const int k0 = blockIdx.x * kg;
    const int kc = min(kg, nrhs - k0);
    if (kc <= 0) return;
    for (int l = 0; l < nlev; ++l) {
        const int r0 = lvl_ptr[l], r1 = lvl_ptr[l + 1];
        const int items = (r1 - r0) * kc;
        for (int it = threadIdx.x; it < items; it += blockDim.x) {
            const int i = lvl_rows[r0 + it / kc];
            double2* xk = x + int64_t(k0 + it % kc) * n;
            double2 s = xk[i];
            const int p0 = ptr[i], p1 = ptr[i + 1];
            if (KIND == kLfwd || KIND == kLtbwd) {
                for (int p = p0; p < p1; ++p) {
                    const double2 a = val[p];
                    const double2 xv = xk[idx[p]];
                    s = csub(s, KIND == kLfwd ? cmul(a, xv) : cmulc(a, xv));
                }
                xk[i] = s;
            } else if (KIND == kUbwd) {  // diagonal first
                for (int p = p0 + 1; p < p1; ++p) s = csub(s, cmul(val[p], xk[idx[p]]));
                xk[i] = cdiv(s, val[p0]);
            } else {  // kUtfwd: row i of U^T, diagonal last
                double2 dg = make_double2(0.0, 0.0);
                for (int p = p0; p < p1; ++p) {
                    const int k = idx[p];
                    if (k == i)
                        dg = val[p];
                    else
                        s = csub(s, cmulc(val[p], xk[k]));
                }
                xk[i] = cdiv(s, make_double2(dg.x, -dg.y));
            }
        }
        __syncthreads();
    }
}

// Two-phase level sweep (the default). One CTA per right-hand side, kIluThreads threads, one
// barrier pair per level:
//   phase A  every thread forms the products a_e * x[k_e] of up to kIluEpl of the level's
//            entries (lane per entry: the level's ~240 products of config 1's ILU(21) take one
//            product's latency instead of a 40-long per-row sequence) into shared memory;
//   phase B  thread t owns the level's row t and subtracts its products from b_i in the
//            reference's entry order (a chain of dependent subtractions: the irreducible
//            part), divides by the diagonal of U / U^T, and stores x_i.
// The level's entry indices / values and row records are loaded into registers one level
// ahead (they do not depend on x), so the only memory reads on the critical path are the x
// operands (shared memory, or L1/L2 for vectors beyond shared memory) and the products.
// Entries are the padded rows of the level-ordered arrays (padding: operand +0 at slot n,
// value 0 -> product +0, which leaves the running sum bit-for-bit unchanged).
template <int KIND, bool XS>
__global__ void __launch_bounds__(kIluThreads) ilu_sweep_2p(int n, int nlev, const int4* __restrict__ lmeta,
                                                           const int4* __restrict__ recs,
                                                           const int* __restrict__ idx,
                                                           const double2* __restrict__ val,
                                                           const double4* __restrict__ ldiag, double2* x,
                                                           const double2* __restrict__ zslot, long long* trace) {
    extern __shared__ __align__(16) double2 dyn[];
    constexpr bool kHasDiag = KIND == kUbwd || KIND == kUtfwd;
    constexpr int T = kIluThreads, E = kIluEpl;
    double2* xk = x + int64_t(blockIdx.x) * n;
    double2* xs = XS ? dyn : xk;
    double2* prod = dyn + (XS ? n + 1 : 0);  // [T * E] products of the current level
    const double2* zero = XS ? xs + n : zslot;
    const int tid = threadIdx.x;
    if (XS) {
        for (int i = tid; i < n; i += T) xs[i] = xk[i];
        if (tid == 0) xs[n] = make_double2(0.0, 0.0);
    }
    // level l's operands in registers (loaded during level l-1)
    int kc[E];
    double2 ac[E];
    int4 rc = make_int4(-1, 0, 0, 0);
    double4 dc = make_double4(0, 0, 0, 0);
    int4 m = nlev > 0 ? __ldg(lmeta) : make_int4(0, 0, 0, 0);
    auto load_level = [&](const int4 mm, int (&kk)[E], double2 (&aa)[E], int4& rr, double4& dd) {
#pragma unroll
        for (int j = 0; j < E; ++j) {
            const int e = mm.z + tid + j * T;
            kk[j] = e < mm.w ? __ldg(idx + e) : -1;
            aa[j] = e < mm.w ? __ldg(val + e) : make_double2(0.0, 0.0);
        }
        const int r = mm.x + tid;
        rr = r < mm.y ? __ldg(recs + r) : make_int4(-1, 0, 0, 0);
        if (kHasDiag && r < mm.y) {
            const double2 d0 = __ldg(reinterpret_cast<const double2*>(ldiag + r));
            const double2 d1 = __ldg(reinterpret_cast<const double2*>(ldiag + r) + 1);
            dd = make_double4(d0.x, d0.y, d1.x, d1.y);
        }
    };
    // one level: prefetch level l+1 into (kn, an, rn, dn), phase A and phase B of level l
    // from (kc, ac, rc, dc). The loop is unrolled by two with the register sets in turn, so
    // the prefetched loads are first consumed a whole level later.
    int4 mnext = nlev > 1 ? __ldg(lmeta + 1) : make_int4(0, 0, 0, 0);  // level l+1's bounds, loaded during l-1
    auto step = [&](int l, int (&kc)[E], double2 (&ac)[E], int4& rc, double4& dc, int (&kn)[E], double2 (&an)[E],
                    int4& rn, double4& dn) {
        const bool tr = trace && blockIdx.x == 0 && tid == 0;  // diagnostics (FWI_ILU_TRACE)
        if (tr) trace[5 * l] = clock64();
        const int4 mn = l + 1 < nlev ? mnext : make_int4(0, 0, 0, 0);
        mnext = l + 2 < nlev ? __ldg(lmeta + l + 2) : make_int4(0, 0, 0, 0);
        load_level(mn, kn, an, rn, dn);
        // phase A: products of level l
#pragma unroll
        for (int j = 0; j < E; ++j) {
            if (kc[j] >= 0) {
                const double2 xv = XS ? xs[kc[j]] : *(kc[j] < n ? xk + kc[j] : zero);
                const int e = tid + j * T;  // level-relative entry; one skew slot per 8 (bank spread)
                prod[e + (e >> 3)] = (KIND == kLfwd || KIND == kUbwd) ? cmul(ac[j], xv) : cmulc(ac[j], xv);
            }
        }
        if (tr) trace[5 * l + 1] = clock64();
        __syncthreads();
        if (tr) trace[5 * l + 2] = clock64();
        // phase B: the rows of level l, entries in the reference's order
        if (rc.x >= 0) {
            const int i = rc.x;
            double2 s = XS ? xs[i] : xk[i];
            for (int p = rc.y; p < rc.z; p += kIluBatch) {
                double2 t[kIluBatch];
#pragma unroll
                for (int u = 0; u < kIluBatch; ++u) t[u] = prod[p + (p >> 3) + u];
#pragma unroll
                for (int u = 0; u < kIluBatch; ++u) s = csub(s, t[u]);
            }
            if (kHasDiag)  // libgcc __divdc3 with the divisor's ratio and denominator precomputed
                s = dc.z != 0.0 ? make_double2(__ddiv_rn(__dadd_rn(__dmul_rn(s.x, dc.x), s.y), dc.y),
                                               __ddiv_rn(__dsub_rn(__dmul_rn(s.y, dc.x), s.x), dc.y))
                                : make_double2(__ddiv_rn(__dadd_rn(__dmul_rn(s.y, dc.x), s.x), dc.y),
                                               __ddiv_rn(__dsub_rn(s.y, __dmul_rn(s.x, dc.x)), dc.y));
            if (XS)
                xs[i] = s;
            else
                xk[i] = s;
        }
        if (tr) trace[5 * l + 3] = clock64();
        __syncthreads();
        if (tr) trace[5 * l + 4] = clock64();
    };
    int kb[E];
    double2 ab[E];
    int4 rb = make_int4(-1, 0, 0, 0);
    double4 db = make_double4(0, 0, 0, 0);
    load_level(m, kc, ac, rc, dc);
    __syncthreads();
    for (int l = 0; l < nlev; l += 2) {
        step(l, kc, ac, rc, dc, kb, ab, rb, db);
        if (l + 1 < nlev) step(l + 1, kb, ab, rb, db, kc, ac, rc, dc);
    }
    if (XS)
        for (int i = tid; i < n; i += T) xk[i] = xs[i];
}

// Two-phase level sweep (the default). One CTA per right-hand side, kIluThreads threads, one
// barrier pair per level:
//   phase A  every thread forms the products a_e * x[k_e] of up to kIluEpl of the level's
//            entries (lane per entry: the ~240 products of a config-1 ILU(21) level take one
//            product's latency instead of a 40-long per-row sequence) into shared memory;
//   phase B  thread t owns the level's row t and subtracts its products from b_i in the
//            reference's entry order (the chain of dependent subtractions, the irreducible
//            part), divides by the diagonal of U / U^T, and stores x_i.
// A level's entry indices and values, row records and divisors are contiguous in the
// level-ordered arrays; thread 0 streams them into a ring of kIluStages shared-memory stages
// with TMA bulk copies (cp.async.bulk + mbarrier) kIluStages levels ahead, so no global load
// is waited on inside the level loop except the x operands of vectors beyond shared memory.
// Entries are the padded rows of the level-ordered arrays (padding: operand +0 at slot n,
// value 0 -> product +0, which leaves the running sum bit-for-bit unchanged).
__device__ __forceinline__ uint32_t ilu_smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void ilu_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     ilu_smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(ilu_smem_addr(b))
                 : "memory");
}
__device__ __forceinline__ void ilu_bar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            ilu_smem_addr(b)),
        "r"(parity)
        : "memory");
}

struct IluStageLayout {  // byte offsets inside one stage
    static constexpr uint32_t kE = kIluThreads * kIluEpl, kR = kIluRows;
    static constexpr uint32_t hdr = 0, vals = 16, diag = vals + kE * 16, recs = diag + kR * 32, bseg = recs + kR * 16,
                              idx = bseg + kR * 16;
    static constexpr uint32_t bytes = idx + kE * 4;
};

// the 8 products of one batch, issued back to back (the chain then never waits on a load)
__device__ __forceinline__ void ilu_lds8(double2 (&t)[kIluBatch], const double2* p) {
    static_assert(kIluBatch == 8, "ilu_lds8 loads 8 products");
    asm volatile(
        "ld.shared.v2.f64 {%0, %1}, [%16];\n\t"
        "ld.shared.v2.f64 {%2, %3}, [%16+16];\n\t"
        "ld.shared.v2.f64 {%4, %5}, [%16+32];\n\t"
        "ld.shared.v2.f64 {%6, %7}, [%16+48];\n\t"
        "ld.shared.v2.f64 {%8, %9}, [%16+64];\n\t"
        "ld.shared.v2.f64 {%10, %11}, [%16+80];\n\t"
        "ld.shared.v2.f64 {%12, %13}, [%16+96];\n\t"
        "ld.shared.v2.f64 {%14, %15}, [%16+112];"
        : "=d"(t[0].x), "=d"(t[0].y), "=d"(t[1].x), "=d"(t[1].y), "=d"(t[2].x), "=d"(t[2].y), "=d"(t[3].x),
          "=d"(t[3].y), "=d"(t[4].x), "=d"(t[4].y), "=d"(t[5].x), "=d"(t[5].y), "=d"(t[6].x), "=d"(t[6].y),
          "=d"(t[7].x), "=d"(t[7].y)
        : "r"(ilu_smem_addr(p))
        : "memory");
}

// MODE: 0 = the vector in global memory (operands through L1/L2), 1 = the whole vector in
// shared memory, 2 = a ring of kIluRingW shared-memory slots indexed by level-ordered position
// (operand indices remapped to positions at factorisation time; the right-hand side gathered
// into level order first and staged with the level, x_i written through to global memory):
// operands lie at most a few hundred positions behind the rows that read them (config 3:
// 658), so the ring holds every live operand of vectors far beyond shared memory.
template <int KIND, int MODE>
__global__ void __launch_bounds__(kIluThreads) ilu_sweep_tma(int n, int nlev, const int4* __restrict__ lmeta,
                                                            const int4* __restrict__ recs,
                                                            const int* __restrict__ idx,
                                                            const double2* __restrict__ val,
                                                            const double4* __restrict__ ldiag, double2* x,
                                                            const double2* __restrict__ zslot,
                                                            const double2* __restrict__ blo, long long* trace) {
    extern __shared__ __align__(128) unsigned char sraw[];
    constexpr bool XS = MODE == 1, RING = MODE == 2;
    constexpr bool kHasDiag = KIND == kUbwd || KIND == kUtfwd;
    constexpr int T = kIluThreads, E = kIluEpl, R = kIluRing, A = kIluAhead;
    static_assert(A < R, "the stage being refilled must not be the one being read");
    using SL = IluStageLayout;
    unsigned char* stage0 = sraw;
    uint64_t* full = reinterpret_cast<uint64_t*>(sraw + R * SL::bytes);  // [R]
    double2* prod = reinterpret_cast<double2*>(full + 2 * R);             // [T*E*9/8]
    double2* xk = x + int64_t(blockIdx.x) * n;
    double2* xs = (XS || RING) ? prod + T * E * 9 / 8 : xk;             // [n + 1] or the ring [kIluRingW + 1]
    const double2* zero = XS ? xs + n : RING ? xs + kIluRingW : zslot;
    const double2* bk = RING ? blo + int64_t(blockIdx.x) * n : nullptr;
    const int tid = threadIdx.x;
    const bool producer = tid == T - 1;  // never owns a row (rows per level <= kIluRows < T)
    if (XS) {
        for (int i = tid; i < n; i += T) xs[i] = xk[i];
        if (tid == 0) xs[n] = make_double2(0.0, 0.0);
    }
    if (RING && tid == 0) xs[kIluRingW] = make_double2(0.0, 0.0);
    if (producer) {
        for (int s = 0; s < R; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(ilu_smem_addr(full + s)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int l, int4 m) {  // producer: level l (bounds m) into stage l % R
        unsigned char* st = stage0 + (l % R) * SL::bytes;
        uint64_t* b = full + (l % R);
        const uint32_t ne = uint32_t(m.w - m.z), nr = uint32_t(m.y - m.x);
        const uint32_t tx = 16 + ne * 20 + nr * ((kHasDiag ? 48 : 16) + (RING ? 16 : 0));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ilu_smem_addr(b)), "r"(tx)
                     : "memory");
        ilu_bulk_g2s(st + SL::hdr, lmeta + l, 16, b);
        if (ne) {
            ilu_bulk_g2s(st + SL::vals, val + m.z, ne * 16, b);
            ilu_bulk_g2s(st + SL::idx, idx + m.z, ne * 4, b);
        }
        if (nr) {
            ilu_bulk_g2s(st + SL::recs, recs + m.x, nr * 16, b);
            if (kHasDiag) ilu_bulk_g2s(st + SL::diag, ldiag + m.x, nr * 32, b);
            if (RING) ilu_bulk_g2s(st + SL::bseg, bk + m.x, nr * 16, b);
        }
    };
    int4 mpre = make_int4(0, 0, 0, 0);  // producer: bounds of the next level to issue
    if (producer) {
        for (int l = 0; l < A && l < nlev; ++l) issue(l, __ldg(lmeta + l));
        if (A < nlev) mpre = __ldg(lmeta + A);
    }
    for (int l = 0; l < nlev; ++l) {
        const bool tr = trace && blockIdx.x == 0 && tid == 0;  // diagnostics (FWI_ILU_TRACE)
        if (tr) trace[5 * l] = clock64();
        const unsigned char* st = stage0 + (l % R) * SL::bytes;
        ilu_bar_wait(full + (l % R), uint32_t(l / R) & 1u);
        const int4 m = *reinterpret_cast<const int4*>(st + SL::hdr);
        const int ne = m.w - m.z, nr = m.y - m.x;
        // phase A: products of level l (branch-free: entries past the level read the zero slot)
        const int* ki = reinterpret_cast<const int*>(st + SL::idx);
        const double2* av = reinterpret_cast<const double2*>(st + SL::vals);
        int kk[E];
#pragma unroll
        for (int j = 0; j < E; ++j) {
            const int e = tid + j * T;
            const int kr = ki[e];
            kk[j] = RING ? (e < ne && kr >= 0 ? (kr & (kIluRingW - 1)) : kIluRingW) : (e < ne ? kr : n);
        }
        double2 xv[E], a[E];
#pragma unroll
        for (int j = 0; j < E; ++j) {
            xv[j] = (XS || RING) ? xs[kk[j]] : *(kk[j] < n ? xk + kk[j] : zero);
            a[j] = av[tid + j * T];
        }
#pragma unroll
        for (int j = 0; j < E; ++j) {
            const int e = tid + j * T;
            prod[e + (e >> 3)] = (KIND == kLfwd || KIND == kUbwd) ? cmul(a[j], xv[j]) : cmulc(a[j], xv[j]);
        }
        if (tr) trace[5 * l + 1] = clock64();
        __syncthreads();
        if (tr) trace[5 * l + 2] = clock64();
        // phase B: the rows of level l, entries in the reference's order; meanwhile the
        // producer refills the stage of level l-1 with level l+A
        if (tid < nr) {
            const int4 rc = reinterpret_cast<const int4*>(st + SL::recs)[tid];
            const int i = rc.x;
            double2 s = RING ? reinterpret_cast<const double2*>(st + SL::bseg)[tid] : xs[i];
            if (rc.y < rc.z) {
                double2 tc[kIluBatch], tn[kIluBatch];
                ilu_lds8(tc, prod + rc.y + (rc.y >> 3));
                for (int p = rc.y + kIluBatch; p < rc.z; p += kIluBatch) {
                    ilu_lds8(tn, prod + p + (p >> 3));  // next batch in flight during this chain
#pragma unroll
                    for (int u = 0; u < kIluBatch; ++u) s = csub(s, tc[u]);
#pragma unroll
                    for (int u = 0; u < kIluBatch; ++u) tc[u] = tn[u];
                }
#pragma unroll
                for (int u = 0; u < kIluBatch; ++u) s = csub(s, tc[u]);
            }
            if (kHasDiag) {  // libgcc __divdc3 with the divisor's ratio and denominator precomputed
                const double4 dc = reinterpret_cast<const double4*>(st + SL::diag)[tid];
                s = dc.z != 0.0 ? make_double2(__ddiv_rn(__dadd_rn(__dmul_rn(s.x, dc.x), s.y), dc.y),
                                               __ddiv_rn(__dsub_rn(__dmul_rn(s.y, dc.x), s.x), dc.y))
                                : make_double2(__ddiv_rn(__dadd_rn(__dmul_rn(s.y, dc.x), s.x), dc.y),
                                               __ddiv_rn(__dsub_rn(s.y, __dmul_rn(s.x, dc.x)), dc.y));
            }
            if (RING) {
                xs[rc.w & (kIluRingW - 1)] = s;
                xk[i] = s;
            } else {
                xs[i] = s;
            }
        } else if (producer && l + A < nlev) {
            issue(l + A, mpre);
            if (l + A + 1 < nlev) mpre = __ldg(lmeta + l + A + 1);
        }
        if (tr) trace[5 * l + 3] = clock64();
        __syncthreads();  // level l's rows written; stage l % R consumed
        if (tr) trace[5 * l + 4] = clock64();
    }
    if (XS)
        for (int i = tid; i < n; i += T) xk[i] = xs[i];
}

long long* g_ilu_trace = nullptr;  // FWI_ILU_TRACE diagnostics: clock64 samples of the first sweep

// blo[k][r] = x[k][rows[r]]: right-hand sides in a sweep's level order (ring sweep)
__global__ void ilu_gather(int n, const int* __restrict__ rows, const double2* __restrict__ x, double2* __restrict__ blo) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int64_t o = int64_t(blockIdx.y) * n;
    blo[o + r] = x[o + __ldg(rows + r)];
}

template <int KIND>
void run_sweep(const Sweep& s, int64_t n, int nrhs, double2* x, cudaStream_t st, const double2* zslot,
               double2* blo) {
    const size_t prod = size_t(kIluThreads) * kIluEpl * 9 / 8 * sizeof(double2);
    const size_t smem = size_t(n + 1) * sizeof(double2) + prod;
    const char* mode = std::getenv("FWI_ILU_GLOBAL");  // diagnostics: "1" = the unstaged one-row-per-thread kernel
    static const bool no_tma = std::getenv("FWI_ILU_NOTMA") != nullptr;  // diagnostics: register-prefetch kernel
    {
        const size_t base = size_t(kIluRing) * IluStageLayout::bytes + 16 * kIluRing +
                            size_t(kIluThreads) * kIluEpl * 9 / 8 * sizeof(double2);
        const size_t with_x = base + size_t(n + 1) * sizeof(double2);
        const size_t with_ring = base + size_t(kIluRingW + 1) * sizeof(double2);
        static const bool no_ring = std::getenv("FWI_ILU_NORING") != nullptr;  // diagnostics
        if (!mode && !no_tma && base <= 220 * 1024) {
            const int md = with_x <= 220 * 1024 ? 1 : (s.ring_ok && !no_ring && blo) ? 2 : 0;
            const size_t sm = md == 1 ? with_x : md == 2 ? with_ring : base;
            static size_t set[3] = {0, 0, 0};  // per (KIND, MODE): the attribute only ever grows
            auto launch = [&](auto kern, const int* ix) {
                if (sm > set[md]) {
                    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
                    set[md] = sm;
                }
                kern<<<nrhs, kIluThreads, sm, st>>>(int(n), s.nlev, s.lmeta.p, s.recs.p, ix, s.lval.p, s.ldiag.p, x,
                                                    zslot, blo, g_ilu_trace);
            };
            if (md == 1) {
                launch(ilu_sweep_tma<KIND, 1>, s.lidx.p);
            } else if (md == 2) {
                // the right-hand sides gathered into the sweep's level order
                ilu_gather<<<dim3((unsigned(n) + 255) / 256, unsigned(nrhs)), 256, 0, st>>>(int(n), s.lvl_rows.p, x,
                                                                                            blo);
                CK_LAUNCH();
                launch(ilu_sweep_tma<KIND, 2>, s.lpos.p);
            } else {
                launch(ilu_sweep_tma<KIND, 0>, s.lidx.p);
            }
            CK_LAUNCH();
            return;
        }
    }
    if (!mode) {
        if (smem <= 220 * 1024) {
            static size_t set = 0;
            if (smem > set) {
                CK(cudaFuncSetAttribute(ilu_sweep_2p<KIND, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(smem)));
                set = smem;
            }
            ilu_sweep_2p<KIND, true><<<nrhs, kIluThreads, smem, st>>>(int(n), s.nlev, s.lmeta.p, s.recs.p, s.lidx.p,
                                                                     s.lval.p, s.ldiag.p, x, zslot, g_ilu_trace);
        } else {
            ilu_sweep_2p<KIND, false><<<nrhs, kIluThreads, prod, st>>>(int(n), s.nlev, s.lmeta.p, s.recs.p, s.lidx.p,
                                                                      s.lval.p, s.ldiag.p, x, zslot, g_ilu_trace);
        }
        CK_LAUNCH();
        return;
    }
    const int kg = 1;
    ilu_sweep_kernel<KIND><<<(nrhs + kg - 1) / kg, 256, 0, st>>>(n, nrhs, kg, s.nlev0, s.lvl_ptr.p,
                                                                s.lvl_rows.p, s.ptr.p, s.idx.p,
                                                                s.val.p, x);
    CK_LAUNCH();
}

}  // namespace

void ilu_factor(Ctx& c, int level, double shift) {
    require(level >= 0, "IluFactors::factor: fill level must be >= 0");
    const auto t_start = std::chrono::steady_clock::now();
    std::vector<int> arp, aci;
    std::vector<cplx> ava;
    host_csr(c, arp, aci, ava);
    const int n = c.n;

    // ---- symbolic phase: levels of fill (src/ilu.cpp:19-50). Row i starts
    // from A's pattern at level 0; pivot rows j < i are visited in ascending
    // order (a min-heap, since fill created through j only lands at k > j),
    // and fill (i,k) via j gets lev(i,j) + lev(j,k) + 1 if <= level.
    std::vector<std::vector<int>> lpat(n), upat(n);
    std::vector<std::vector<std::pair<int, int>>> ulev(n);
    std::vector<int> lev(n, 0), stamp(n, -1), cols;
    for (int i = 0; i < n; ++i) {
        cols.clear();
        std::priority_queue<int, std::vector<int>, std::greater<int>> todo;
        bool has_diag = false;
        for (int p = arp[i]; p < arp[i + 1]; ++p) {
            const int j = aci[p];
            stamp[j] = i;
            lev[j] = 0;
            cols.push_back(j);
            if (j < i) todo.push(j);
            has_diag |= (j == i);
        }
        if (!has_diag)
            throw FwiError(FWI_ERR_INVALID_ARGUMENT,
                           "IluFactors::factor: missing diagonal at row " + std::to_string(i));
        while (!todo.empty()) {
            const int j = todo.top();
            todo.pop();
            const int lj = lev[j];
            for (const auto& [k, lu] : ulev[j]) {
                const int nl = lj + lu + 1;
                if (nl > level) continue;
                if (stamp[k] != i) {
                    stamp[k] = i;
                    lev[k] = nl;
                    cols.push_back(k);
                    if (k < i) todo.push(k);
                } else if (nl < lev[k]) {
                    lev[k] = nl;
                }
            }
        }
        std::sort(cols.begin(), cols.end());
        for (int cc : cols) {
            if (cc < i)
                lpat[i].push_back(cc);
            else
                upat[i].push_back(cc);
            if (cc > i) ulev[i].emplace_back(cc, lev[cc]);
        }
    }

    // ---- numeric phase (src/ilu.cpp:52-104), IKJ on the fixed pattern
    std::vector<int> lp(n + 1, 0), up(n + 1, 0);
    for (int i = 0; i < n; ++i) {
        lp[i + 1] = lp[i] + int(lpat[i].size());
        up[i + 1] = up[i] + int(upat[i].size());
    }
    std::vector<int> li(lp[n]), ui(up[n]);
    std::vector<cplx> lv(lp[n]), uv(up[n]);
    std::vector<cplx> w(n, 0.0);
    std::fill(stamp.begin(), stamp.end(), -1);
    for (int i = 0; i < n; ++i) {
        for (int cc : lpat[i]) { stamp[cc] = i; w[cc] = 0.0; }
        for (int cc : upat[i]) { stamp[cc] = i; w[cc] = 0.0; }
        for (int p = arp[i]; p < arp[i + 1]; ++p) w[aci[p]] += ava[p];
        w[i] += shift;
        for (int j : lpat[i]) {
            const int ud = up[j];
            w[j] /= uv[ud];
            const cplx lij = w[j];
            if (lij == 0.0) continue;
            for (int p = ud + 1; p < up[j + 1]; ++p) {
                const int k = ui[p];
                if (stamp[k] == i) w[k] -= lij * uv[p];
            }
        }
        if (w[i] == 0.0) throw FwiError(FWI_ERR_ZERO_PIVOT,
                                        "ILU: zero pivot at row " + std::to_string(i) +
                                            " (consider a diagonal shift)", i);
        int p = lp[i];
        for (int cc : lpat[i]) { li[p] = cc; lv[p] = w[cc]; ++p; }
        p = up[i];
        for (int cc : upat[i]) { ui[p] = cc; uv[p] = w[cc]; ++p; }
    }

    auto f = std::make_unique<IluFactor>();
    f->level = level;
    std::vector<int> ltp, lti, utp, uti;
    std::vector<cplx> ltv, utv;
    transpose_csr(n, lp, li, lv, ltp, lti, ltv);
    transpose_csr(n, up, ui, uv, utp, uti, utv);
    upload_sweep(f->L, n, lp, li, lv, true, false, c.stream, f->bytes);
    upload_sweep(f->U, n, up, ui, uv, false, true, c.stream, f->bytes);
    upload_sweep(f->Ut, n, utp, uti, utv, true, true, c.stream, f->bytes);
    upload_sweep(f->Lt, n, ltp, lti, ltv, false, false, c.stream, f->bytes);
    f->zslot.alloc(1);
    CK(cudaMemsetAsync(f->zslot.p, 0, sizeof(double2), c.stream));
    if (c.ilu) ilu_free(c.ilu);
    c.ilu = f.release();
    c.t_ilu_factor = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
}

// x = M^{-1} b (or M^{-H} b) for nrhs source-major right-hand sides.
void ilu_solve_batch(Ctx& c, bool adjoint, const double2* b, double2* x, int nrhs) {
    require(c.ilu != nullptr, "precond_apply: state has no ILU factorization");
    const int64_t n = c.n;
    if (x != b)
        CK(cudaMemcpyAsync(x, b, size_t(nrhs) * n * sizeof(double2), cudaMemcpyDeviceToDevice, c.stream));
    IluFactor& f = *c.ilu;
    // level-ordered right-hand sides of the ring sweep (vectors beyond shared memory)
    double2* blo = nullptr;
    if (size_t(n + 1) * sizeof(double2) > 100 * 1024) {
        if (f.blo.count < size_t(nrhs) * size_t(n)) f.blo.alloc(size_t(nrhs) * size_t(n));
        blo = f.blo.p;
    }
    const char* tpath = std::getenv("FWI_ILU_TRACE");
    DevBuf<long long> tb;
    if (tpath) {
        tb.alloc(size_t(5) * (adjoint ? f.Ut : f.L).nlev);
        CK(cudaMemsetAsync(tb.p, 0, tb.bytes(), c.stream));
        g_ilu_trace = tb.p;
    }
    if (!adjoint) {
        run_sweep<kLfwd>(f.L, n, nrhs, x, c.stream, f.zslot.p, blo);
        g_ilu_trace = nullptr;
        run_sweep<kUbwd>(f.U, n, nrhs, x, c.stream, f.zslot.p, blo);
    } else {
        run_sweep<kUtfwd>(f.Ut, n, nrhs, x, c.stream, f.zslot.p, blo);
        g_ilu_trace = nullptr;
        run_sweep<kLtbwd>(f.Lt, n, nrhs, x, c.stream, f.zslot.p, blo);
    }
    if (tpath) {
        std::vector<long long> h(tb.count);
        CK(cudaMemcpyAsync(h.data(), tb.p, tb.bytes(), cudaMemcpyDeviceToHost, c.stream));
        CK(cudaStreamSynchronize(c.stream));
        if (FILE* fp = std::fopen(tpath, "wb")) {
            std::fwrite(h.data(), 8, h.size(), fp);
            std::fclose(fp);
        }
    }
    c.solve_count[FWI_PRECOND_ILU] += nrhs;
}

}  // namespace fwi_b200
