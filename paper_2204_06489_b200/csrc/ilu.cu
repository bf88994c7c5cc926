// ilu.cu — ILU(p) block solver: factorisation + batched, level-scheduled triangular sweeps on
// the device (K2/K4, inexact mode).
//
// Reference: IluFactors::factor (src/ilu.cpp:8-106), build_transposes (:108-129), solve
// (:131-174).
//
// The factorisation is per-Newton-step setup; the factors must be bit-identical to the
// reference's for the inexact preconditioner to reproduce its output exactly.
//  * symbolic phase (level-of-fill patterns, host, the reference's rules) and everything that
//    depends only on the pattern — level schedules, the level-ordered sweep layouts, the
//    numeric phase's update lists — are built once per (grid, fill level) and cached across
//    contexts (a Newton sweep re-factors the same pattern every step);
//  * numeric phase on the device (ilu_numeric), the reference's IKJ order exactly: rows in
//    dependency levels, one warp per row; for each j of row i's L pattern in ascending
//    order, w_j /= U_jj (libgcc complex division), skipped if zero, then the row's entries
//    k in U_j's pattern updated in parallel (each k once per j, so the order of the updates
//    to every w_k is the reference's); zero pivots raise ZeroPivotError(row) with the
//    smallest failing row, the one the reference reports;
//  * the four sweeps' value arrays (L, U forward; U^H, L^H adjoint) gathered from the factor
//    in their level-ordered layouts, and U's divisors prepared (ilu_sweep_vals).
// The sweeps run for all sources at once, one CTA per source (ilu_sweep_tma): rows grouped
// into dependency levels, each level in two phases — every thread forms products (lane per
// entry), then each row's owner subtracts them in the reference's entry order (bit-faithful)
// — with the level data streamed into shared memory by TMA bulk copies several levels ahead.
// The vector lives in shared memory (config 1), or in a ring indexed by level-ordered
// position when it is too large (config 3/4: operands lie < 700 positions behind their rows).
#include <algorithm>
#include <chrono>
#include <climits>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <mutex>
#include <queue>
#include <string>

#include "ctx.cuh"

namespace fwi_b200 {

using cplx = std::complex<double>;

constexpr int kIluBatch = 8;      // entries per batch of the sweep kernels (row padding unit)
constexpr int kIluThreads = 256;  // sweep kernel block
constexpr int kIluEpl = 2;        // entries per thread and level (a level holds <= kIluThreads * kIluEpl)
constexpr int kIluRows = 128;     // rows per (sub-)level
constexpr int kIluRing = 4;       // TMA stage ring
constexpr int kIluAhead = 3;      // levels staged ahead
constexpr int kIluRingW = 2048;   // operand ring (positions) of the ring sweep, a power of two

// One triangular sweep's pattern-only data: the entries regrouped in level order (row
// lvl_rows[r] owns entries [rstart[r], rstart[r+1]) in the row's own order, padded to a
// multiple of kIluBatch; the diagonals of U / U^T apart; levels wider than the kernel cut into
// consecutive sub-levels) and where each entry's value comes from in the factor.
struct Sweep {
    DevBuf<int> lvl_rows, lidx, lpos;  // rows in level order; operand node / level position (-1: padding)
    DevBuf<int4> recs;                 // per level-ordered row: {row, first entry, end entry, position}
    DevBuf<int4> lmeta;                // per (sub-)level: first row, end row, first entry, end entry
    DevBuf<int> vmap;                  // per entry: index of its value in the factor (-1: padding)
    DevBuf<int> dmap;                  // per level-ordered row: index of its divisor (sweeps with one)
    bool has_diag = false, conj_diag = false;
    bool ring_ok = false;
    int nlev = 0, nent = 0;
    int maxrow = 0;
};

// Everything that depends only on the pattern of one (grid, fill level).
struct IluPattern {
    int nx = 0, nz = 0, n = 0, level = 0;
    int64_t nfv = 0;                                   // factor values: row i at [rowoff[i], rowoff[i+1]): L then U
    int maxcnt = 0, maxnl = 0, maxupd = 0;             // longest factor row, L row, row update list
    DevBuf<int> rowoff, nl, arp, aslot, lp, jdiag, updptr, frows;
    DevBuf<int2> upd;                                  // (slot in row i, factor index of U_jk)
    std::vector<int> flvl;                             // numeric phase levels (host) over frows
    Sweep L, U, Ut, Lt;
    int64_t bytes = 0;
};

struct IluFactor {
    int level = 0;
    std::shared_ptr<IluPattern> pat;
    DevBuf<double2> fv;                                // L | U per row
    DevBuf<double2> lval[4];                           // per sweep (L, U, Ut, Lt)
    DevBuf<double4> ldiag[4];                          // per sweep with a divisor (U, Ut)
    int64_t bytes = 0;
    DevBuf<double2> zslot;  // the padding entries' operand (+0) when the vector is in global memory
    DevBuf<double2> blo;    // right-hand sides in level order (ring sweep scratch, nrhs x n)
    DevBuf<int> status;
};

void ilu_free(IluFactor* f) { delete f; }
int64_t ilu_bytes(const IluFactor* f) { return f ? f->bytes + (f->pat ? f->pat->bytes : 0) : 0; }

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

template <class T>
void upload(DevBuf<T>& buf, const std::vector<T>& v, cudaStream_t st, int64_t& bytes) {
    buf.alloc(std::max<size_t>(v.size(), 1));
    if (!v.empty()) CK(cudaMemcpyAsync(buf.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
    bytes += int64_t(v.size() * sizeof(T));
}

// The sweep layout of one triangular factor given in CSR (ptr, idx) with src[p] = index of
// entry p's value in the factor; has_diag: the row's diagonal is its divisor (kept apart).
void build_sweep(Sweep& s, int n, const std::vector<int>& ptr, const std::vector<int>& idx,
                 const std::vector<int>& src, bool forward, bool has_diag, bool conj_diag, cudaStream_t st,
                 int64_t& bytes) {
    std::vector<int> lp, rows;
    int nlev0 = 0;
    build_levels(n, ptr, idx, forward, lp, rows, nlev0);
    s.has_diag = has_diag;
    s.conj_diag = conj_diag;
    upload(s.lvl_rows, rows, st, bytes);
    // level order; per row the off-diagonal entries in the row's own order, padded to a
    // multiple of kIluBatch with (n, -1) entries; the diagonal (U: first, U^T: last) apart
    std::vector<int> rst(n + 1, 0), li, vm, dm(n, -1);
    li.reserve(idx.size() + size_t(n) * kIluBatch);
    vm.reserve(idx.size() + size_t(n) * kIluBatch);
    for (int r = 0; r < n; ++r) {
        const int i = rows[r];
        for (int q = ptr[i]; q < ptr[i + 1]; ++q) {
            if (idx[q] == i && has_diag) {
                dm[r] = src[q];
                continue;
            }
            li.push_back(idx[q]);
            vm.push_back(src[q]);
        }
        while (li.size() % kIluBatch) {
            li.push_back(n);
            vm.push_back(-1);
        }
        rst[r + 1] = int(li.size());
        s.maxrow = std::max(s.maxrow, rst[r + 1] - rst[r]);
    }
    // sub-levels: at most kIluRows rows and kIluThreads * kIluEpl entries each
    std::vector<int> sp{0};
    for (int l = 0; l < nlev0; ++l) {
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
    s.nent = int(li.size());
    std::vector<int4> rec(n);
    for (int l = 0; l < s.nlev; ++l)
        for (int r = lp[l]; r < lp[l + 1]; ++r)
            rec[r] = make_int4(rows[r], rst[r] - rst[lp[l]], rst[r + 1] - rst[lp[l]], r);
    upload(s.recs, rec, st, bytes);
    std::vector<int4> meta(s.nlev);
    for (int l = 0; l < s.nlev; ++l) meta[l] = make_int4(lp[l], lp[l + 1], rst[lp[l]], rst[lp[l + 1]]);
    upload(s.lmeta, meta, st, bytes);
    upload(s.lidx, li, st, bytes);
    upload(s.vmap, vm, st, bytes);
    if (has_diag) upload(s.dmap, dm, st, bytes);
    // operand positions for the ring sweep (padding: -1) and whether the ring holds them
    std::vector<int> pos(n + 1, -1), lpos(li.size());
    for (int r = 0; r < n; ++r) pos[rows[r]] = r;
    int maxd = 0;
    for (int r = 0; r < n; ++r)
        for (int q = rst[r]; q < rst[r + 1]; ++q) {
            lpos[q] = pos[li[q]];
            if (li[q] < n) maxd = std::max(maxd, r - pos[li[q]]);
        }
    s.ring_ok = maxd + kIluRows < kIluRingW;
    upload(s.lpos, lpos, st, bytes);
}

// transpose of a CSR pattern; tsrc[q] = source entry index of transposed entry q
void transpose_pattern(int n, const std::vector<int>& ptr, const std::vector<int>& idx, std::vector<int>& tp,
                       std::vector<int>& ti, std::vector<int>& tsrc) {
    tp.assign(n + 1, 0);
    for (int c : idx) tp[c + 1]++;
    for (int j = 0; j < n; ++j) tp[j + 1] += tp[j];
    ti.resize(idx.size());
    tsrc.resize(idx.size());
    std::vector<int> nx(tp.begin(), tp.end() - 1);
    for (int i = 0; i < n; ++i)  // rows ascending -> ascending order within each transposed row
        for (int p = ptr[i]; p < ptr[i + 1]; ++p) {
            const int q = nx[idx[p]]++;
            ti[q] = i;
            tsrc[q] = p;
        }
}

// The pattern of ILU(level) on the operand's pattern (rp, ci) and all pattern-only data.
std::shared_ptr<IluPattern> build_pattern(const Ctx& c, int level, const std::vector<int>& arp,
                                          const std::vector<int>& aci) {
    auto P = std::make_shared<IluPattern>();
    P->nx = c.nx;
    P->nz = c.nz;
    P->level = level;
    const int n = c.n;
    P->n = n;
    const cudaStream_t st = c.stream;
    // ---- symbolic phase: levels of fill (src/ilu.cpp:19-50). Row i starts from A's pattern
    // at level 0; pivot rows j < i are visited in ascending order (a min-heap, since fill
    // created through j only lands at k > j), and fill (i,k) via j gets lev(i,j) + lev(j,k) + 1
    // if <= level.
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
    // ---- factor layout: row i = [L entries | U entries (diagonal first)]
    std::vector<int> lp(n + 1, 0), up(n + 1, 0), rowoff(n + 1, 0), nl(n);
    for (int i = 0; i < n; ++i) {
        lp[i + 1] = lp[i] + int(lpat[i].size());
        up[i + 1] = up[i] + int(upat[i].size());
        nl[i] = int(lpat[i].size());
        rowoff[i + 1] = rowoff[i] + int(lpat[i].size() + upat[i].size());
    }
    P->nfv = rowoff[n];
    for (int i = 0; i < n; ++i) {
        P->maxcnt = std::max(P->maxcnt, rowoff[i + 1] - rowoff[i]);
        P->maxnl = std::max(P->maxnl, nl[i]);
    }
    std::vector<int> li(lp[n]), ui(up[n]);
    for (int i = 0; i < n; ++i) {
        std::copy(lpat[i].begin(), lpat[i].end(), li.begin() + lp[i]);
        std::copy(upat[i].begin(), upat[i].end(), ui.begin() + up[i]);
    }
    auto lsrc = [&](int i, int p) { return rowoff[i] + (p - lp[i]); };
    auto usrc = [&](int i, int p) { return rowoff[i] + nl[i] + (p - up[i]); };
    // ---- numeric phase data (src/ilu.cpp:52-104): A's entries scattered into row slots; per
    // L entry (i, j): the index of U_jj and the updates w_k -= l_ij u_jk for k in U_j's pattern
    // that row i holds (the stamp test)
    std::vector<int> aslot(arp[n]), jdiag(lp[n]), updptr(lp[n] + 1, 0);
    std::vector<int2> upd;
    std::vector<int> slot(n, -1);
    for (int i = 0; i < n; ++i) {
        int q = 0;
        for (int cc : lpat[i]) slot[cc] = q++;
        for (int cc : upat[i]) slot[cc] = q++;
        for (int p = arp[i]; p < arp[i + 1]; ++p) aslot[p] = slot[aci[p]];
        for (int t = 0; t < nl[i]; ++t) {
            const int j = lpat[i][t], pl = lp[i] + t;
            jdiag[pl] = usrc(j, up[j]);
            for (int p = up[j] + 1; p < up[j + 1]; ++p) {
                const int k = ui[p];
                if (slot[k] >= 0) upd.push_back(make_int2(slot[k], usrc(j, p)));
            }
            updptr[pl + 1] = int(upd.size());
        }
        for (int cc : lpat[i]) slot[cc] = -1;
        for (int cc : upat[i]) slot[cc] = -1;
    }
    for (int i = 0; i < n; ++i) P->maxupd = std::max(P->maxupd, updptr[lp[i + 1]] - updptr[lp[i]]);
    std::vector<int> flp, frows;
    int fnlev = 0;
    build_levels(n, lp, li, true, flp, frows, fnlev);
    P->flvl = flp;
    upload(P->rowoff, rowoff, st, P->bytes);
    upload(P->nl, nl, st, P->bytes);
    upload(P->arp, arp, st, P->bytes);
    upload(P->aslot, aslot, st, P->bytes);
    upload(P->lp, lp, st, P->bytes);
    upload(P->jdiag, jdiag, st, P->bytes);
    upload(P->updptr, updptr, st, P->bytes);
    upload(P->upd, upd, st, P->bytes);
    upload(P->frows, frows, st, P->bytes);
    // ---- the four sweeps (build_transposes, src/ilu.cpp:108-129)
    std::vector<int> ls(lp[n]), us(up[n]);
    for (int i = 0; i < n; ++i) {
        for (int p = lp[i]; p < lp[i + 1]; ++p) ls[p] = lsrc(i, p);
        for (int p = up[i]; p < up[i + 1]; ++p) us[p] = usrc(i, p);
    }
    std::vector<int> tp, ti, tsrc, ts;
    build_sweep(P->L, n, lp, li, ls, true, false, false, st, P->bytes);
    build_sweep(P->U, n, up, ui, us, false, true, false, st, P->bytes);
    transpose_pattern(n, up, ui, tp, ti, tsrc);
    ts.resize(tsrc.size());
    for (size_t q = 0; q < tsrc.size(); ++q) ts[q] = us[tsrc[q]];
    build_sweep(P->Ut, n, tp, ti, ts, true, true, true, st, P->bytes);
    transpose_pattern(n, lp, li, tp, ti, tsrc);
    ts.resize(tsrc.size());
    for (size_t q = 0; q < tsrc.size(); ++q) ts[q] = ls[tsrc[q]];
    build_sweep(P->Lt, n, tp, ti, ts, false, false, false, st, P->bytes);
    CK(cudaStreamSynchronize(st));
    return P;
}

// ---- numeric phase kernels --------------------------------------------------

// One warp per row of one level: the reference's IKJ loop (src/ilu.cpp:66-103) on row i,
// everything the row reads staged in shared memory first — w, U_jj of every j, and every
// update entry (slot, u_jk) of the row, loaded together in one coalesced pass (they come
// from earlier, final rows) — so the j loop runs from shared memory: lane 0 forms
// l_ij = w_j / U_jj (libgcc division), then the lanes apply j's updates (distinct slots).
struct NumericSmem {  // per-warp layout (double2 units, then ints)
    int maxcnt, maxnl, maxupd;
    __host__ __device__ size_t d2() const { return size_t(maxcnt) + maxnl + maxupd; }
    __host__ __device__ size_t ints() const { return size_t(maxupd) + maxnl + 1; }
    __host__ __device__ size_t bytes() const { return d2() * 16 + (ints() * 4 + 15) / 16 * 16; }
};

__global__ void __launch_bounds__(128) ilu_numeric(int r0, int r1, const int* __restrict__ frows,
                                                   const int* __restrict__ rowoff, const int* __restrict__ nl,
                                                   const int* __restrict__ arp, const int* __restrict__ aslot,
                                                   const double2* __restrict__ ava, double shift,
                                                   const int* __restrict__ lp, const int* __restrict__ jdiag,
                                                   const int* __restrict__ updptr, const int2* __restrict__ upd,
                                                   double2* fv, int* status, NumericSmem L) {
    extern __shared__ __align__(16) unsigned char nraw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double2* w = reinterpret_cast<double2*>(nraw + size_t(wid) * L.bytes());
    double2* ujj = w + L.maxcnt;
    double2* uval = ujj + L.maxnl;
    int* uslot = reinterpret_cast<int*>(uval + L.maxupd);
    int* uptr = uslot + L.maxupd;
    const int r = r0 + int(blockIdx.x) * (blockDim.x >> 5) + wid;
    if (r >= r1) return;
    const int i = frows[r];
    const int base = rowoff[i], cnt = rowoff[i + 1] - base, nli = nl[i], l0 = lp[i];
    const int e0 = updptr[l0], ne = updptr[l0 + nli] - e0;
    for (int t = lane; t < cnt; t += 32) w[t] = make_double2(0.0, 0.0);
    for (int q = lane; q < nli; q += 32) ujj[q] = fv[jdiag[l0 + q]];  // U_jj of every j (final rows)
    for (int q = lane; q <= nli; q += 32) uptr[q] = updptr[l0 + q] - e0;
    for (int e = lane; e < ne; e += 32) {
        const int2 u = upd[e0 + e];
        uslot[e] = u.x;
        uval[e] = fv[u.y];
    }
    __syncwarp();
    for (int p = arp[i] + lane; p < arp[i + 1]; p += 32) w[aslot[p]] = cadd(w[aslot[p]], ava[p]);  // w[col] += a
    __syncwarp();
    if (lane == 0) w[nli].x = __dadd_rn(w[nli].x, shift);  // w[i] += shift
    __syncwarp();
    for (int q = 0; q < nli; ++q) {
        double2 lij = make_double2(0.0, 0.0);
        if (lane == 0) {
            lij = cdiv(w[q], ujj[q]);  // w[j] /= uv[ud]
            w[q] = lij;
        }
        lij.x = __shfl_sync(0xffffffffu, lij.x, 0);
        lij.y = __shfl_sync(0xffffffffu, lij.y, 0);
        if (lij.x == 0.0 && lij.y == 0.0) continue;  // if (lij == 0.0) continue;
        for (int e = uptr[q] + lane; e < uptr[q + 1]; e += 32)
            w[uslot[e]] = csub(w[uslot[e]], cmul(lij, uval[e]));  // w[k] -= lij * uv[p]
        __syncwarp();
    }
    __syncwarp();
    if (lane == 0 && w[nli].x == 0.0 && w[nli].y == 0.0) atomicMin(status, i);
    for (int t = lane; t < cnt; t += 32) fv[base + t] = w[t];
}

// sweep values from the factor: lval[e] = fv[vmap[e]] (padding: +0); divisors (U / U^H):
// cdiv's ratio and denominator (host_cdiv_prep) of U_ii or conj(U_ii)
__global__ void ilu_sweep_vals(int nent, const int* __restrict__ vmap, const double2* __restrict__ fv,
                               double2* __restrict__ lval, int n, const int* __restrict__ dmap, bool conj_diag,
                               double4* __restrict__ ldiag) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < nent) {
        const int v = vmap[t];
        lval[t] = v >= 0 ? fv[v] : make_double2(0.0, 0.0);
    }
    if (ldiag && t < n) {
        const double2 d = fv[dmap[t]];
        const double cc = d.x, dd = conj_diag ? -d.y : d.y;
        double r, den, small;
        if (fabs(cc) < fabs(dd)) {
            r = __ddiv_rn(cc, dd);
            den = __dadd_rn(__dmul_rn(cc, r), dd);
            small = 1.0;
        } else {
            r = __ddiv_rn(dd, cc);
            den = __dadd_rn(__dmul_rn(dd, r), cc);
            small = 0.0;
        }
        ldiag[t] = make_double4(r, den, small, 0.0);
    }
}

enum SweepKind { kLfwd = 0, kUbwd = 1, kUtfwd = 2, kLtbwd = 3 };

// Two-phase level sweep (the default). One CTA per right-hand side, kIluThreads threads, one
// barrier pair per level:
//   phase A  every thread forms the products a_e * x[k_e] of up to kIluEpl of the level's
//            entries (lane per entry: the ~240 products of a config-1 ILU(21) level take one
//            product's latency instead of a 40-long per-row sequence) into shared memory;
//   phase B  thread t owns the level's row t and subtracts its products from b_i in the
//            reference's entry order (the chain of dependent subtractions, the irreducible
//            part), divides by the diagonal of U / U^T, and stores x_i.
// A level's entry indices and values, row records and divisors are contiguous in the
// level-ordered arrays; a thread without a row streams them into a ring of kIluRing shared-
// memory stages with TMA bulk copies (cp.async.bulk + mbarrier) kIluAhead levels ahead, so no
// global load is waited on inside the level loop except the x operands of vectors beyond
// shared memory.
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
void run_sweep(const Sweep& s, const double2* lval, const double4* ldiag, int64_t n, int nrhs, double2* x,
               cudaStream_t st, const double2* zslot, double2* blo) {
    const size_t base = size_t(kIluRing) * IluStageLayout::bytes + 16 * kIluRing +
                        size_t(kIluThreads) * kIluEpl * 9 / 8 * sizeof(double2);
    const size_t with_x = base + size_t(n + 1) * sizeof(double2);
    const size_t with_ring = base + size_t(kIluRingW + 1) * sizeof(double2);
    static const bool no_ring = std::getenv("FWI_ILU_NORING") != nullptr;  // diagnostics
    const int md = with_x <= 220 * 1024 ? 1 : (s.ring_ok && !no_ring && blo) ? 2 : 0;
    const size_t sm = md == 1 ? with_x : md == 2 ? with_ring : base;
    static size_t set[3] = {0, 0, 0};  // per (KIND, MODE): the attribute only ever grows
    auto launch = [&](auto kern, const int* ix) {
        if (sm > set[md]) {
            CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
            set[md] = sm;
        }
        kern<<<nrhs, kIluThreads, sm, st>>>(int(n), s.nlev, s.lmeta.p, s.recs.p, ix, lval, ldiag, x, zslot, blo,
                                            g_ilu_trace);
    };
    if (md == 1) {
        launch(ilu_sweep_tma<KIND, 1>, s.lidx.p);
    } else if (md == 2) {
        // the right-hand sides gathered into the sweep's level order
        ilu_gather<<<dim3((unsigned(n) + 255) / 256, unsigned(nrhs)), 256, 0, st>>>(int(n), s.lvl_rows.p, x, blo);
        CK_LAUNCH();
        launch(ilu_sweep_tma<KIND, 2>, s.lpos.p);
    } else {
        launch(ilu_sweep_tma<KIND, 0>, s.lidx.p);
    }
    CK_LAUNCH();
}

}  // namespace

// ILU(level) of the context's operator with diagonal shift `shift` (IluFactors::factor,
// src/ilu.cpp:8-106): the pattern from the cache (or built), the numeric phase on the device.
void ilu_factor(Ctx& c, int level, double shift) {
    require(level >= 0, "IluFactors::factor: fill level must be >= 0");
    const auto t_start = std::chrono::steady_clock::now();
    std::vector<int> arp, aci;
    std::vector<cplx> ava;
    host_csr(c, arp, aci, ava);
    const int n = c.n;
    // pattern cache: the operator's pattern depends on the grid only (Dirichlet ring), so a
    // Newton sweep re-factors one pattern per fill level
    static std::mutex mu;
    static std::vector<std::shared_ptr<IluPattern>> cache;
    std::shared_ptr<IluPattern> P;
    {
        std::lock_guard<std::mutex> lk(mu);
        for (auto& e : cache)
            if (e->nx == c.nx && e->nz == c.nz && e->level == level) P = e;
    }
    const auto t_pat0 = std::chrono::steady_clock::now();
    if (!P) {
        P = build_pattern(c, level, arp, aci);
        std::lock_guard<std::mutex> lk(mu);
        cache.push_back(P);
        if (cache.size() > 4) cache.erase(cache.begin());
    }
    const auto t_pat1 = std::chrono::steady_clock::now();
    auto f = std::make_unique<IluFactor>();
    f->level = level;
    f->pat = P;
    f->fv.alloc(size_t(std::max<int64_t>(P->nfv, 1)));
    f->status.alloc(1);
    DevBuf<double2> a(ava.size());
    CK(cudaMemcpyAsync(a.p, ava.data(), ava.size() * sizeof(cplx), cudaMemcpyHostToDevice, c.stream));
    const int big = INT_MAX;
    CK(cudaMemcpyAsync(f->status.p, &big, sizeof(int), cudaMemcpyHostToDevice, c.stream));
    // numeric phase, level by level (a row's L pattern are its dependencies)
    const NumericSmem ns{std::max(P->maxcnt, 1), std::max(P->maxnl, 1), std::max(P->maxupd, 1)};
    const size_t nsm = size_t(4) * ns.bytes();
    require(nsm <= 220 * 1024, "ILU: factor rows too long for the device numeric phase");
    static size_t nsm_set = 0;
    if (nsm > 48 * 1024 && nsm > nsm_set) {
        CK(cudaFuncSetAttribute(ilu_numeric, cudaFuncAttributeMaxDynamicSharedMemorySize, int(nsm)));
        nsm_set = nsm;
    }
    for (size_t l = 0; l + 1 < P->flvl.size(); ++l) {
        const int r0 = P->flvl[l], r1 = P->flvl[l + 1];
        const int warps = 4;
        ilu_numeric<<<(r1 - r0 + warps - 1) / warps, 32 * warps, nsm, c.stream>>>(
            r0, r1, P->frows.p, P->rowoff.p, P->nl.p, P->arp.p, P->aslot.p, a.p, shift, P->lp.p, P->jdiag.p,
            P->updptr.p, P->upd.p, f->fv.p, f->status.p, ns);
        CK_LAUNCH();
    }
    int st = big;
    CK(cudaMemcpyAsync(&st, f->status.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    if (st != big)
        throw FwiError(FWI_ERR_ZERO_PIVOT, "ILU: zero pivot at row " + std::to_string(st) + " (consider a diagonal shift)",
                       st);
    const auto t_num = std::chrono::steady_clock::now();
    const Sweep* sw[4] = {&P->L, &P->U, &P->Ut, &P->Lt};
    for (int k = 0; k < 4; ++k) {
        const Sweep& s = *sw[k];
        f->lval[k].alloc(size_t(std::max(s.nent, 1)));
        if (s.has_diag) f->ldiag[k].alloc(size_t(n));
        f->bytes += int64_t(f->lval[k].bytes() + f->ldiag[k].bytes());
        const int work = std::max(s.nent, n);
        ilu_sweep_vals<<<(work + 255) / 256, 256, 0, c.stream>>>(s.nent, s.vmap.p, f->fv.p, f->lval[k].p, n,
                                                                s.has_diag ? s.dmap.p : nullptr, s.conj_diag,
                                                                s.has_diag ? f->ldiag[k].p : nullptr);
        CK_LAUNCH();
    }
    f->zslot.alloc(1);
    CK(cudaMemsetAsync(f->zslot.p, 0, sizeof(double2), c.stream));
    f->bytes += f->fv.bytes();
    CK(cudaStreamSynchronize(c.stream));
    if (c.ilu) ilu_free(c.ilu);
    c.ilu = f.release();
    const auto t_end = std::chrono::steady_clock::now();
    c.t_ilu_factor = std::chrono::duration<double>(t_end - t_start).count();
    if (std::getenv("FWI_ILU_TIMING"))
        std::fprintf(stderr, "[fwi] ILU(%d) factor: operator %.3f s, pattern %.3f s%s, numeric (device) %.3f s, "
                             "sweep values %.3f s\n",
                     level, std::chrono::duration<double>(t_pat0 - t_start).count(),
                     std::chrono::duration<double>(t_pat1 - t_pat0).count(),
                     t_pat1 - t_pat0 > std::chrono::milliseconds(1) ? " (built)" : " (cached)",
                     std::chrono::duration<double>(t_num - t_pat1).count(),
                     std::chrono::duration<double>(t_end - t_num).count());
}

// x = M^{-1} b (or M^{-H} b) for nrhs source-major right-hand sides.
void ilu_solve_batch(Ctx& c, bool adjoint, const double2* b, double2* x, int nrhs) {
    require(c.ilu != nullptr, "precond_apply: state has no ILU factorization");
    const int64_t n = c.n;
    if (x != b)
        CK(cudaMemcpyAsync(x, b, size_t(nrhs) * n * sizeof(double2), cudaMemcpyDeviceToDevice, c.stream));
    IluFactor& f = *c.ilu;
    const IluPattern& P = *f.pat;
    // level-ordered right-hand sides of the ring sweep (vectors beyond shared memory)
    double2* blo = nullptr;
    if (size_t(n + 1) * sizeof(double2) > 100 * 1024) {
        if (f.blo.count < size_t(nrhs) * size_t(n)) f.blo.alloc(size_t(nrhs) * size_t(n));
        blo = f.blo.p;
    }
    const char* tpath = std::getenv("FWI_ILU_TRACE");  // diagnostics: clock64 trace of the first sweep
    DevBuf<long long> tb;
    if (tpath) {
        tb.alloc(size_t(5) * (adjoint ? P.Ut : P.L).nlev);
        CK(cudaMemsetAsync(tb.p, 0, tb.bytes(), c.stream));
        g_ilu_trace = tb.p;
    }
    if (!adjoint) {
        run_sweep<kLfwd>(P.L, f.lval[0].p, nullptr, n, nrhs, x, c.stream, f.zslot.p, blo);
        g_ilu_trace = nullptr;
        run_sweep<kUbwd>(P.U, f.lval[1].p, f.ldiag[1].p, n, nrhs, x, c.stream, f.zslot.p, blo);
    } else {
        run_sweep<kUtfwd>(P.Ut, f.lval[2].p, f.ldiag[2].p, n, nrhs, x, c.stream, f.zslot.p, blo);
        g_ilu_trace = nullptr;
        run_sweep<kLtbwd>(P.Lt, f.lval[3].p, nullptr, n, nrhs, x, c.stream, f.zslot.p, blo);
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
