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
// all sources at once: rows are grouped into dependency levels, one CTA owns
// a group of sources, and each (row, source) item evaluates its row in the
// reference's entry order (bit-faithful), with a CTA barrier between levels.
#include <algorithm>
#include <cstdlib>
#include <complex>
#include <queue>

#include "ctx.cuh"

namespace fwi_b200 {

using cplx = std::complex<double>;

struct Sweep {          // one triangular sweep in CSR form + its level schedule
    DevBuf<int> ptr, idx, lvl_ptr, lvl_rows;
    DevBuf<double2> val;
    // the same entries regrouped in level order: row lvl_rows[r] owns
    // entries [rstart[r], rstart[r+1]) of (lidx, lval), in the row's own order
    DevBuf<int> rstart, lidx;
    DevBuf<double2> lval;
    DevBuf<int4> lmeta;  // per level: first row, end row, first entry, end entry
    int nlev = 0;
    int ecap = 0, rcap = 0;  // max entries / rows of one level
};

struct IluFactor {
    int level = 0;
    Sweep L, U, Ut, Lt;  // Ut/Lt: transposes for the adjoint
    int64_t bytes = 0;
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
                  const std::vector<cplx>& val, bool forward, cudaStream_t st, int64_t& bytes) {
    std::vector<int> lp, rows;
    build_levels(n, ptr, idx, forward, lp, rows, s.nlev);
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
        std::vector<int> rst(n + 1, 0), li;
        std::vector<cplx> lv;
        li.reserve(idx.size());
        lv.reserve(val.size());
        for (int r = 0; r < n; ++r) {
            const int i = rows[r];
            for (int q = ptr[i]; q < ptr[i + 1]; ++q) {
                li.push_back(idx[q]);
                lv.push_back(val[q]);
            }
            rst[r + 1] = int(li.size());
        }
        up(s.rstart, rst);
        s.ecap = s.rcap = 1;
        for (int l = 0; l < s.nlev; ++l) {
            s.rcap = std::max(s.rcap, lp[l + 1] - lp[l]);
            s.ecap = std::max(s.ecap, rst[lp[l + 1]] - rst[lp[l]]);
        }
        s.ecap = (s.ecap + 1) / 2 * 2;
        std::vector<int4> meta(s.nlev);
        for (int l = 0; l < s.nlev; ++l) meta[l] = make_int4(lp[l], lp[l + 1], rst[lp[l]], rst[lp[l + 1]]);
        up(s.lmeta, meta);
        up(s.lidx, li);
        s.lval.alloc(std::max<size_t>(lv.size(), 1));
        if (!lv.empty())
            CK(cudaMemcpyAsync(s.lval.p, lv.data(), lv.size() * sizeof(cplx), cudaMemcpyHostToDevice, st));
        bytes += int64_t(lv.size() * sizeof(cplx));
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

// Shared-memory variant (n * 16 B fits): one CTA per right-hand side keeps
// its whole vector in shared memory. The rows of each level and their entries
// are contiguous in the level-ordered arrays; they are staged into a ring of
// shared-memory buffers with cp.async three levels ahead, so the dependency
// chain of a level only touches shared memory.
constexpr int kLvlBuf = 4;

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// XS = false: the vector stays in global memory (L2-resident; loaded with
// ld.global.cg so a CTA always sees its own earlier levels' stores) and only the
// level metadata is staged — for vectors beyond shared memory (config 3/4:
// n = 49,152 -> 786 KB per right-hand side).
// x operands: shared memory (XS), or global memory through L1 (L1) or L2 only. The
// rows of one level read what this CTA's threads wrote before the level barrier, so
// L1-cached loads see it (CTA-scope ordering of bar.sync).
__device__ __forceinline__ double2 xload(const double2* p, bool glob) { return glob ? __ldcg(p) : *p; }

template <int KIND, bool XS, bool L1 = false>
__global__ void __launch_bounds__(256) ilu_sweep_smem(int n, int nlev, const int4* __restrict__ lmeta,
                                                     int meta_smem, const int* __restrict__ lvl_rows,
                                                     const int* __restrict__ rstart,
                                                     const int* __restrict__ idx,
                                                     const double2* __restrict__ val, double2* x, int ecap,
                                                     int rcap) {
    extern __shared__ __align__(16) double2 dyn[];
    double2* xs = XS ? dyn : x + int64_t(blockIdx.x) * n;
    double2* vb = dyn + (XS ? n : 0);                         // [kLvlBuf][ecap]
    int* ib = reinterpret_cast<int*>(vb + size_t(kLvlBuf) * ecap);  // [kLvlBuf][ecap]
    int* rib = ib + kLvlBuf * ecap;                           // [kLvlBuf][rcap] row ids
    int* rpb = rib + kLvlBuf * rcap;                          // [kLvlBuf][rcap + 1] entry starts
    int4* ms = reinterpret_cast<int4*>(rpb + kLvlBuf * (rcap + 1) + 3 - ((kLvlBuf * (rcap + 1) + 3) & 3));
    double2* xk = x + int64_t(blockIdx.x) * n;
    const int tid = threadIdx.x, nt = blockDim.x;
    // level bounds in shared memory: the prefetch of level l+3 then issues its copies
    // without a dependent chain of global loads on every level's critical path
    if (meta_smem)
        for (int l = tid; l < nlev; l += nt) ms[l] = lmeta[l];
    const int4* mt = meta_smem ? ms : lmeta;
    __syncthreads();
    // The last warp stages level metadata (cp.async, kLvlBuf-1 levels ahead) while the
    // other warps evaluate the current level: one barrier per level, and the staging
    // of level l+3 overlaps the rows of level l.
    const int pw0 = nt - 32;  // first thread of the staging warp
    const bool stager = tid >= pw0;
    const int ct = stager ? 0 : tid, cn = pw0;  // compute threads 0..pw0-1
    auto prefetch = [&](int l) {
        if (!stager) return;
        if (l < nlev) {
            const int b = l % kLvlBuf;
            const int4 m = mt[l];
            const int r0 = m.x, r1 = m.y;
            const int e0 = m.z, e1 = m.w;
            for (int t = tid - pw0; t < e1 - e0; t += 32) {
                cp_async16(vb + b * ecap + t, val + e0 + t);
                cp_async4(ib + b * ecap + t, idx + e0 + t);
            }
            for (int t = tid - pw0; t < r1 - r0; t += 32) cp_async4(rib + b * rcap + t, lvl_rows + r0 + t);
            for (int t = tid - pw0; t <= r1 - r0; t += 32) cp_async4(rpb + b * (rcap + 1) + t, rstart + r0 + t);
        }
        cp_commit();  // (possibly empty) group per level keeps the counting uniform
    };
    if (XS)
        for (int i = tid; i < n; i += nt) xs[i] = xk[i];
#pragma unroll
    for (int l = 0; l < kLvlBuf - 1; ++l) prefetch(l);
    for (int l = 0; l < nlev; ++l) {
        if (stager) cp_wait<kLvlBuf - 2>();
        __syncthreads();  // level l staged; level l-1's rows written
        prefetch(l + kLvlBuf - 1);  // into level l-1's buffer, free now
        if (stager) continue;
        const int b = l % kLvlBuf;
        const int nrow = mt[l].y - mt[l].x;
        const int* rp = rpb + b * (rcap + 1);
        const int e0 = rp[0];
        const double2* vl = vb + b * ecap;
        const int* il = ib + b * ecap;
        for (int t = ct; t < nrow; t += cn) {
            const int i = rib[b * rcap + t];
            const int p0 = rp[t] - e0, p1 = rp[t + 1] - e0;
            double2 s = xload(xs + i, !XS && !L1);
            double2 dg = make_double2(0.0, 0.0);
            // Entries in the reference's order. A batch of 8 loads its indices, values and x
            // operands first, forms the 8 products independently, then runs the dependent
            // subtraction chain with selects (no per-entry branches, so the loads overlap).
            constexpr int BT = 8;
            const int q0 = (KIND == kUbwd) ? p0 + 1 : p0;
            for (int pb = q0; pb < p1; pb += BT) {
                double2 xv[BT], av[BT];
                int kv[BT];
#pragma unroll
                for (int u = 0; u < BT; ++u) {
                    const int pp = min(pb + u, p1 - 1);  // clamped: in range, result discarded
                    kv[u] = il[pp];
                    av[u] = vl[pp];
                }
#pragma unroll
                for (int u = 0; u < BT; ++u) xv[u] = xload(xs + kv[u], !XS && !L1);
                double2 tv[BT];
#pragma unroll
                for (int u = 0; u < BT; ++u)
                    tv[u] = (KIND == kLfwd || KIND == kUbwd) ? cmul(av[u], xv[u]) : cmulc(av[u], xv[u]);
#pragma unroll
                for (int u = 0; u < BT; ++u) {
                    const bool valid = pb + u < p1;
                    bool use = valid;
                    if (KIND == kUtfwd) {
                        const bool diag = valid && kv[u] == i;
                        dg = diag ? av[u] : dg;
                        use = valid && !diag;
                    }
                    const double2 sn = csub(s, tv[u]);
                    s = use ? sn : s;
                }
            }
            if (KIND == kLfwd || KIND == kLtbwd)
                xs[i] = s;
            else if (KIND == kUbwd)
                xs[i] = cdiv(s, vl[p0]);
            else
                xs[i] = cdiv(s, make_double2(dg.x, -dg.y));
        }
    }
    cp_wait<0>();
    __syncthreads();
    if (XS)
        for (int t = tid; t < n; t += nt) xk[t] = xs[t];
}

template <int KIND>
void run_sweep(const Sweep& s, int64_t n, int nrhs, double2* x, cudaStream_t st) {
    size_t meta = size_t(kLvlBuf) * s.ecap * (sizeof(double2) + 4) + size_t(kLvlBuf) * (2 * s.rcap + 1) * 4 + 64;
    const size_t lm = size_t(s.nlev) * sizeof(int4);
    const int meta_smem = (lm <= 48 * 1024) ? 1 : 0;
    if (meta_smem) meta += lm + 16;
    const size_t smem = size_t(n) * sizeof(double2) + meta;
    const char* mode = std::getenv("FWI_ILU_GLOBAL");  // diagnostics: "1" = unstaged global kernel
    static const int nthr = std::getenv("FWI_ILU_THREADS") ? std::atoi(std::getenv("FWI_ILU_THREADS")) : 256;
    if (smem <= 220 * 1024 && !mode) {
        static size_t set = 0;
        if (smem > set) {
            CK(cudaFuncSetAttribute(ilu_sweep_smem<KIND, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(smem)));
            set = smem;
        }
        ilu_sweep_smem<KIND, true><<<nrhs, nthr, smem, st>>>(int(n), s.nlev, s.lmeta.p, meta_smem, s.lvl_rows.p,
                                                           s.rstart.p, s.lidx.p, s.lval.p, x, s.ecap, s.rcap);
        CK_LAUNCH();
        return;
    }
    if (meta <= 220 * 1024 && !mode) {  // vector in global memory, level metadata staged in shared memory
        static const bool l2only = std::getenv("FWI_ILU_L2") != nullptr;  // diagnostics: bypass L1
        static size_t set = 0;
        if (meta > set) {
            CK(cudaFuncSetAttribute(ilu_sweep_smem<KIND, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(meta)));
            CK(cudaFuncSetAttribute(ilu_sweep_smem<KIND, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(meta)));
            set = meta;
        }
        if (l2only)
            ilu_sweep_smem<KIND, false, false><<<nrhs, nthr, meta, st>>>(int(n), s.nlev, s.lmeta.p, meta_smem,
                                                                       s.lvl_rows.p, s.rstart.p, s.lidx.p, s.lval.p,
                                                                       x, s.ecap, s.rcap);
        else
            ilu_sweep_smem<KIND, false, true><<<nrhs, nthr, meta, st>>>(int(n), s.nlev, s.lmeta.p, meta_smem,
                                                                      s.lvl_rows.p, s.rstart.p, s.lidx.p, s.lval.p,
                                                                      x, s.ecap, s.rcap);
        CK_LAUNCH();
        return;
    }
    const int kg = 1;
    ilu_sweep_kernel<KIND><<<(nrhs + kg - 1) / kg, 256, 0, st>>>(n, nrhs, kg, s.nlev, s.lvl_ptr.p,
                                                                s.lvl_rows.p, s.ptr.p, s.idx.p,
                                                                s.val.p, x);
    CK_LAUNCH();
}

}  // namespace

void ilu_factor(Ctx& c, int level, double shift) {
    require(level >= 0, "IluFactors::factor: fill level must be >= 0");
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
    upload_sweep(f->L, n, lp, li, lv, true, c.stream, f->bytes);
    upload_sweep(f->U, n, up, ui, uv, false, c.stream, f->bytes);
    upload_sweep(f->Ut, n, utp, uti, utv, true, c.stream, f->bytes);
    upload_sweep(f->Lt, n, ltp, lti, ltv, false, c.stream, f->bytes);
    if (c.ilu) ilu_free(c.ilu);
    c.ilu = f.release();
}

// x = M^{-1} b (or M^{-H} b) for nrhs source-major right-hand sides.
void ilu_solve_batch(Ctx& c, bool adjoint, const double2* b, double2* x, int nrhs) {
    require(c.ilu != nullptr, "precond_apply: state has no ILU factorization");
    const int64_t n = c.n;
    if (x != b)
        CK(cudaMemcpyAsync(x, b, size_t(nrhs) * n * sizeof(double2), cudaMemcpyDeviceToDevice, c.stream));
    const IluFactor& f = *c.ilu;
    if (!adjoint) {
        run_sweep<kLfwd>(f.L, n, nrhs, x, c.stream);
        run_sweep<kUbwd>(f.U, n, nrhs, x, c.stream);
    } else {
        run_sweep<kUtfwd>(f.Ut, n, nrhs, x, c.stream);
        run_sweep<kLtbwd>(f.Lt, n, nrhs, x, c.stream);
    }
    c.solve_count[FWI_PRECOND_ILU] += nrhs;
}

}  // namespace fwi_b200
