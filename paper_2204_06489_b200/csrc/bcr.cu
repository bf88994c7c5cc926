// bcr.cu — block cyclic reduction: the exact block solver with a log-depth solve
// (K2/K4 exact mode for the config-3/4 geometry).
//
// Reference semantics: LuFactors::factor / solve (src/lu.cpp:37-209), x = A^{-1} b.
// exact.cu factors the block-tridiagonal A (L lines of nb nodes, tridiagonal blocks
// T_i, diagonal couplings E_i = A(i, i+1) = A(i+1, i)) as a Schur recursion along the
// lines, so a solve is a chain of 2L dependent line steps; a line step is latency-bound
// (~1.8 us at config 3), which leaves the GPU mostly idle. Cyclic reduction removes the
// chain: at every level the even blocks are eliminated at once and the odd blocks form a
// block-tridiagonal system of half the size,
//
//   M_j   = D_j^{-1}                         (even j, batched Gauss-Jordan)
//   D'    = D_j - U_{j-1}^T M_{j-1} U_{j-1} - U_j M_{j+1} U_j^T      (odd j)
//   U'    = -U_j M_{j+1} U_{j+1}                                       (odd j, j+2)
//
// down to one block (log2 L levels). A solve is log2 L levels of batched products down
// and up, each a strided-batched complex GEMM on the FP64 tensor cores (cgemm_batched):
//
//   down  t_j = M_j b_j (even);  b_j -= U_{j-1}^T t_{j-1} + U_j t_{j+1}   (odd)
//   up    x_j = t_j - P_j x_{j-1} - Q_j x_{j+1}   (even; P_j = M_j U_{j-1}^T, Q_j = M_j U_j)
//
// Level 0 keeps the couplings diagonal (elementwise updates, no P/Q). Storage: M, P, Q,
// U per level, ~3.5 L nb^2 complex (config 3: ~200 MB); solve work ~3.5 L nb^2 K complex
// multiply-adds (against 2 L nb^2 K for the sweeps), in ~5 log2 L launches.
// Pivoting: partial pivoting over each whole block (the block Gauss-Jordan of the long-
// line path restricts it to 64-wide diagonal blocks); exact.cu's residual probe checks
// every factorisation.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "ctx.cuh"
#include "dense.cuh"

namespace fwi_b200 {

struct BcrLevel {
    int m = 0;            // blocks at this level
    int line0 = 0, step = 0;  // block j <-> grid line line0 + j * step
    int ne = 0, no = 0;   // eliminated (even) and kept (odd) blocks
    double2 *M = nullptr, *P = nullptr, *Q = nullptr, *U = nullptr;  // ne, ne, ne, m-1 blocks of nb^2
    size_t t_off = 0;     // this level's t_j (ne blocks of nrhs x nb) in the solve scratch
};

struct BcrFactor {
    int nb = 0, L = 0;
    std::vector<BcrLevel> lv;
    DevBuf<double2> store;  // M, P, Q, U of every level
    DevBuf<double2> t, r;   // solve scratch (grown to the widest batch)
    DevBuf<double2> part;   // split-K partial tiles of the narrow GEMMs
    // level 0: the even blocks are the lines' tridiagonal T_{2b}; their LU with partial pivoting
    // (LAPACK zgttrf form: dl, 1/d, du, du2 per block, row interchanges in tpiv) replaces the dense
    // M_b products of the level-0 solve by O(nb) sweeps (M_b stays for the factorisation)
    DevBuf<double2> tri;
    DevBuf<unsigned char> tpiv;
    bool tri_ok = false;
    size_t t_blocks = 0;    // sum over levels of ne
    int nrhs_cap = 0;
};

void bcr_free(BcrFactor* f) { delete f; }

// one-product levels of at least this many blocks use the tiled DMMA kernel (shared-memory
// operand reuse), narrower ones the warp-tile kernel (every SM busy)
// (FWI_BCR_TILED_MIN=<batch> moves both switch points)
static int bcr_tiled_min() {
    static const int v = std::getenv("FWI_BCR_TILED_MIN") ? std::atoi(std::getenv("FWI_BCR_TILED_MIN")) : 64;
    return v;
}
#define kBcrTiledBatch bcr_tiled_min()
#define kBcrTiledBatch2 bcr_tiled_min()
constexpr size_t kTriSmem = 112 * 1024;  // level-0 tridiagonal solve: shared memory per CTA (2 CTAs/SM)
int64_t bcr_bytes(const BcrFactor* f) {
    return f ? int64_t(f->store.bytes() + f->t.bytes() + f->r.bytes() + f->part.bytes()) : 0;
}

namespace {

__device__ __forceinline__ int64_t node_of(bool col_lines, int nx, int line, int m) {
    return col_lines ? int64_t(m) * nx + line : int64_t(line) * nx + m;
}
__device__ __forceinline__ double2 cm(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// T_line as a dense nb x nb block (the line's tridiagonal stencil rows)
__device__ __forceinline__ double2 tri(bool col_lines, int nx, int nb, int line, int a, int b,
                                       const double2* __restrict__ diag, const double2* __restrict__ east,
                                       const double2* __restrict__ south) {
    if (a == b) return diag[node_of(col_lines, nx, line, a)];
    if (b == a + 1) {
        const int64_t na = node_of(col_lines, nx, line, a);
        return col_lines ? south[na] : east[na];
    }
    if (a == b + 1) {
        const int64_t nbn = node_of(col_lines, nx, line, b);
        return col_lines ? south[nbn] : east[nbn];
    }
    return make_double2(0.0, 0.0);
}

// level 0, even blocks: D = T_{2b}
__global__ void l0_even(bool col_lines, int nx, int nb, int ne, const double2* __restrict__ diag,
                        const double2* __restrict__ east, const double2* __restrict__ south, double2* __restrict__ M) {
    const int64_t nn = int64_t(nb) * nb;
    const int b = blockIdx.y;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < nn; t += int64_t(gridDim.x) * blockDim.x) {
        const int a = int(t / nb), c = int(t % nb);
        M[b * nn + t] = tri(col_lines, nx, nb, 2 * b, a, c, diag, east, south);
    }
}

// level 0 -> 1: for odd j = 2b+1, D'_b = T_j - E_{j-1} M_b E_{j-1} - E_j M_{b+1} E_j and
// U'_b = -E_j M_{b+1} E_{j+1} (couplings diagonal: E_i = coup[i], rows a / columns c)
__global__ void l0_schur(bool col_lines, int nx, int nb, int m, int no, const double2* __restrict__ diag,
                         const double2* __restrict__ east, const double2* __restrict__ south,
                         const double2* __restrict__ coup, const double2* __restrict__ M, double2* __restrict__ D1,
                         double2* __restrict__ U1) {
    const int64_t nn = int64_t(nb) * nb;
    const int b = blockIdx.y;
    const int j = 2 * b + 1;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < nn; t += int64_t(gridDim.x) * blockDim.x) {
        const int a = int(t / nb), c = int(t % nb);
        double2 v = tri(col_lines, nx, nb, j, a, c, diag, east, south);
        const double2* El = coup + int64_t(j - 1) * nb;
        const double2 w = cm(cm(El[a], M[b * nn + t]), El[c]);
        v.x -= w.x;
        v.y -= w.y;
        if (j + 1 < m) {
            const double2* Er = coup + int64_t(j) * nb;
            const double2 w2 = cm(cm(Er[a], M[(b + 1) * nn + t]), Er[c]);
            v.x -= w2.x;
            v.y -= w2.y;
            if (b + 1 < no) {
                const double2* Enn = coup + int64_t(j + 1) * nb;
                const double2 u = cm(cm(Er[a], M[(b + 1) * nn + t]), Enn[c]);
                U1[b * nn + t] = make_double2(-u.x, -u.y);
            }
        }
        D1[b * nn + t] = v;
    }
}

// strided block copy: dst[b] = src[b * sstride] (nn elements per block)
__global__ void copy_blocks(int64_t nn, int nblk, const double2* __restrict__ src, int64_t sstride,
                            double2* __restrict__ dst, int64_t dstride) {
    pdl_enter();
    const int b = blockIdx.y;
    if (b >= nblk) return;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < nn; t += int64_t(gridDim.x) * blockDim.x)
        dst[b * dstride + t] = src[b * sstride + t];
}

// batched transpose of nb x nb blocks
__global__ void transpose_blocks(int nb, const double2* __restrict__ src, double2* __restrict__ dst) {
    __shared__ double2 tile[32][33];
    const int64_t nn = int64_t(nb) * nb;
    const int b = blockIdx.z;
    const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int r = r0 + i, c = c0 + threadIdx.x;
        if (r < nb && c < nb) tile[i][threadIdx.x] = src[b * nn + int64_t(r) * nb + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int r = c0 + i, c = r0 + threadIdx.x;
        if (r < nb && c < nb) dst[b * nn + int64_t(r) * nb + c] = tile[threadIdx.x][i];
    }
}

// In-place Gauss-Jordan inverse of a batch of nb x nb blocks (one CTA per block, the block
// in global memory / L2), partial pivoting over the whole column. A zero pivot records
// status = 1 + line * nb + k (the block's grid line, exact.cu maps it to the node).
__global__ void __launch_bounds__(512) gj_batched(int nb, double2* __restrict__ Ab, int line0, int lstep,
                                                  int* status) {
    extern __shared__ double2 gsm[];
    double2* prow = gsm;
    double2* pcol = gsm + nb;
    int* piv = reinterpret_cast<int*>(gsm + 2 * nb);
    __shared__ double red_v[16];
    __shared__ int red_i[16];
    __shared__ int s_p;
    __shared__ double2 s_pivinv;
    const int64_t nn = int64_t(nb) * nb;
    double2* A = Ab + blockIdx.x * nn;
    const int line = line0 + int(blockIdx.x) * lstep;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
    for (int k = 0; k < nb; ++k) {
        double best = -1.0;
        int bi = nb;
        for (int r = k + tid; r < nb; r += nt) {
            const double2 v = A[int64_t(r) * nb + k];
            const double m2 = v.x * v.x + v.y * v.y;
            if (m2 > best || (m2 == best && r < bi)) {
                best = m2;
                bi = r;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_down_sync(0xffffffffu, best, o);
            const int oi = __shfl_down_sync(0xffffffffu, bi, o);
            if (ov > best || (ov == best && oi < bi)) {
                best = ov;
                bi = oi;
            }
        }
        if (lane == 0) {
            red_v[wid] = best;
            red_i[wid] = bi;
        }
        __syncthreads();
        if (tid == 0) {
            double bv = -1.0;
            int bb = nb;
            for (int w = 0; w < nw; ++w)
                if (red_v[w] > bv || (red_v[w] == bv && red_i[w] < bb)) {
                    bv = red_v[w];
                    bb = red_i[w];
                }
            if (!(bv > 0.0)) {
                atomicCAS(status, 0, line * nb + k + 1);
                bb = k;
            }
            s_p = bb;
            piv[k] = bb;
            const double2 d = A[int64_t(bb) * nb + k];
            s_pivinv = (d.x == 0.0 && d.y == 0.0) ? make_double2(0.0, 0.0) : cdiv(make_double2(1.0, 0.0), d);
        }
        __syncthreads();
        const int p = s_p;
        const double2 pinv = s_pivinv;
        // the scaled pivot row (old row p) and the pivot column as it stands after rows k and
        // p are swapped (row p then holds old row k), read before anything is written
        for (int j = tid; j < nb; j += nt) {
            const double2 a = (j == k) ? make_double2(1.0, 0.0) : A[int64_t(p) * nb + j];
            prow[j] = cm(a, pinv);
        }
        for (int r = tid; r < nb; r += nt)
            pcol[r] = (r == k) ? make_double2(0.0, 0.0) : A[int64_t(r == p ? k : r) * nb + k];
        __syncthreads();
        for (int j = tid; j < nb; j += nt) {
            const double2 ak = A[int64_t(k) * nb + j];
            if (p != k) A[int64_t(p) * nb + j] = ak;
            A[int64_t(k) * nb + j] = prow[j];
        }
        __syncthreads();
        for (int r = wid; r < nb; r += nw) {
            if (r == k) continue;
            const double2 f = pcol[r];
            for (int j = lane; j < nb; j += 32) {
                double2 v = (j == k) ? make_double2(0.0, 0.0) : A[int64_t(r) * nb + j];
                const double2 pr = prow[j];
                v.x -= f.x * pr.x - f.y * pr.y;
                v.y -= f.x * pr.y + f.y * pr.x;
                A[int64_t(r) * nb + j] = v;
            }
        }
        __syncthreads();
    }
    // undo the column permutation (reverse order)
    for (int k = nb - 1; k >= 0; --k) {
        const int p = piv[k];
        if (p != k)
            for (int r = tid; r < nb; r += nt) {
                const double2 t = A[int64_t(r) * nb + k];
                A[int64_t(r) * nb + k] = A[int64_t(r) * nb + p];
                A[int64_t(r) * nb + p] = t;
            }
        __syncthreads();
    }
}

// level-0 solve updates, W[line][k][m] (blk = nrhs * nb per line), T[b][k][m]:
// down, odd j = 2b+1: b_j -= E_{j-1} t_b + E_j t_{b+1}
__global__ void l0_down(int nb, int m, int64_t blk, const double2* __restrict__ coup, const double2* __restrict__ T,
                        double2* __restrict__ W) {
    pdl_enter();
    const int b = blockIdx.y, j = 2 * b + 1;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < blk; e += int64_t(gridDim.x) * blockDim.x) {
        const int c = int(e % nb);
        double2 v = W[j * blk + e];
        const double2 w = cm(coup[int64_t(j - 1) * nb + c], T[b * blk + e]);
        v.x -= w.x;
        v.y -= w.y;
        if (j + 1 < m) {
            const double2 w2 = cm(coup[int64_t(j) * nb + c], T[(b + 1) * blk + e]);
            v.x -= w2.x;
            v.y -= w2.y;
        }
        W[j * blk + e] = v;
    }
}
// up, even j = 2b: R_b = E_{j-1} x_{j-1} + E_j x_{j+1}  (then x_j = t_b - M_b R_b)
__global__ void l0_up_rhs(int nb, int m, int64_t blk, const double2* __restrict__ coup, const double2* __restrict__ W,
                          double2* __restrict__ R) {
    pdl_enter();
    const int b = blockIdx.y, j = 2 * b;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < blk; e += int64_t(gridDim.x) * blockDim.x) {
        const int c = int(e % nb);
        double2 v = make_double2(0.0, 0.0);
        if (j > 0) v = cm(coup[int64_t(j - 1) * nb + c], W[(j - 1) * blk + e]);
        if (j + 1 < m) {
            const double2 w = cm(coup[int64_t(j) * nb + c], W[(j + 1) * blk + e]);
            v.x += w.x;
            v.y += w.y;
        }
        R[b * blk + e] = v;
    }
}

__device__ __forceinline__ double cabs1(double2 z) { return fabs(z.x) + fabs(z.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// LU with partial pivoting of every level-0 even block T_{2b} (one thread per block; LAPACK's
// zgttrf: interchange rows i, i+1 when |dl_i| > |d_i| in the 1-norm of re/im, one extra
// superdiagonal du2 of fill). Stores dl (multipliers), 1/d, du/d, du2/d as trf[b][4][nb].
__global__ void l0_gttrf(bool col_lines, int nx, int nb, int ne, const double2* __restrict__ diag,
                         const double2* __restrict__ east, const double2* __restrict__ south,
                         double2* __restrict__ trf, unsigned char* __restrict__ piv) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= ne) return;
    const int line = 2 * b;
    double2* dl = trf + int64_t(b) * 4 * nb;
    double2* dv = dl + nb;
    double2* du = dv + nb;
    double2* du2 = du + nb;
    unsigned char* pv = piv + int64_t(b) * nb;
    for (int i = 0; i < nb; ++i) {
        dv[i] = tri(col_lines, nx, nb, line, i, i, diag, east, south);
        du[i] = i + 1 < nb ? tri(col_lines, nx, nb, line, i, i + 1, diag, east, south) : make_double2(0.0, 0.0);
        dl[i] = i + 1 < nb ? tri(col_lines, nx, nb, line, i + 1, i, diag, east, south) : make_double2(0.0, 0.0);
        du2[i] = make_double2(0.0, 0.0);
        pv[i] = 0;
    }
    for (int i = 0; i + 1 < nb; ++i) {
        if (cabs1(dv[i]) >= cabs1(dl[i])) {
            if (dv[i].x != 0.0 || dv[i].y != 0.0) {
                const double2 f = cdiv(dl[i], dv[i]);
                dl[i] = f;
                dv[i + 1] = csub(dv[i + 1], cm(f, du[i]));
            }
        } else {
            const double2 f = cdiv(dv[i], dl[i]);
            dv[i] = dl[i];
            dl[i] = f;
            const double2 t = du[i];
            du[i] = dv[i + 1];
            dv[i + 1] = csub(t, cm(f, dv[i + 1]));
            if (i + 2 < nb) {
                du2[i] = du[i + 1];
                du[i + 1] = make_double2(-f.x * du[i + 1].x + f.y * du[i + 1].y, -f.x * du[i + 1].y - f.y * du[i + 1].x);
            }
            pv[i] = 1;
        }
    }
    // 1/d and the rows of U scaled by it: x_i = x_i / d_i - (du_i / d_i) x_{i+1} - (du2_i / d_i) x_{i+2}
    for (int i = 0; i < nb; ++i) {
        const double2 r =
            (dv[i].x == 0.0 && dv[i].y == 0.0) ? make_double2(0.0, 0.0) : cdiv(make_double2(1.0, 0.0), dv[i]);
        dv[i] = r;
        du[i] = cm(du[i], r);
        du2[i] = cm(du2[i], r);
    }
}

// Level-0 solves with the tridiagonal factors: one CTA per (even block b, chunk of kc right-hand
// sides). UP = false (down): T[b] = T_{2b}^{-1} W[2b]. UP = true: W[2b] = T_{2b}^{-1}(W[2b] -
// E_{2b-1} x_{2b-1} - E_{2b} x_{2b+1}) with the odd neighbours' solutions already in W. The
// chunk's columns are staged in shared memory (row pitch nb + 1: conflict-free per-thread
// walks) by all threads with several loads in flight; one thread per column then runs the
// forward and back substitution, carrying the running values in registers so the only
// dependent chain is one complex multiply-subtract per row.
constexpr int kTriThreads = 256;
constexpr int kTriCols = 16;
template <bool UP>
__global__ void __launch_bounds__(kTriThreads, 4) l0_tri_solve(int nb, int m, int kc, int nrhs, int64_t blk,
                                                            const double2* __restrict__ trf,
                                                            const unsigned char* __restrict__ piv,
                                                            const double2* __restrict__ coup,
                                                            double2* __restrict__ W, double2* __restrict__ T) {
    pdl_enter();
    extern __shared__ double2 ts[];
    const int b = blockIdx.x, j = 2 * b, k0 = blockIdx.y * kc;
    const int kn = min(kc, nrhs - k0);
    const int pitch = nb + 1;
    double2* f = ts;            // dl, 1/d, du, du2
    double2* xs = ts + 4 * nb;  // kn columns
    unsigned char* ps = reinterpret_cast<unsigned char*>(xs + int64_t(kc) * pitch);
    const double2* fb = trf + int64_t(b) * 4 * nb;
    for (int i = threadIdx.x; i < 4 * nb; i += blockDim.x) f[i] = fb[i];
    for (int i = threadIdx.x; i < nb; i += blockDim.x) ps[i] = piv[int64_t(b) * nb + i];
    const int64_t off = int64_t(k0) * nb;
    const double2* wj = W + int64_t(j) * blk + off;
    const double2* wl = W + int64_t(j - 1) * blk + off;
    const double2* wr = W + int64_t(j + 1) * blk + off;
    const double2* el = coup + int64_t(j - 1) * nb;
    const double2* er = coup + int64_t(j) * nb;
    const bool hl = UP && j > 0, hr = UP && j + 1 < m;
    const int tot = kn * nb;
    constexpr int U = UP ? 2 : 4;  // loads in flight per thread and array (64 registers)
    for (int e0 = threadIdx.x; e0 < tot; e0 += U * kTriThreads) {
        double2 v[U], l[U], r[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
            const int e = e0 + q * kTriThreads;
            if (e < tot) {
                v[q] = wj[e];
                if (hl) l[q] = wl[e];
                if (hr) r[q] = wr[e];
            }
        }
#pragma unroll
        for (int q = 0; q < U; ++q) {
            const int e = e0 + q * kTriThreads;
            if (e >= tot) continue;
            const int c = e % nb;
            double2 x = v[q];
            if (UP) {
                double2 s = make_double2(0.0, 0.0);
                if (hl) s = cm(el[c], l[q]);
                if (hr) {
                    const double2 w2 = cm(er[c], r[q]);
                    s.x += w2.x;
                    s.y += w2.y;
                }
                x = csub(x, s);
            }
            xs[(e / nb) * pitch + c] = x;
        }
    }
    __syncthreads();
    const double2 *dl = f, *di = f + nb, *ud = f + 2 * nb, *ud2 = f + 3 * nb;
    for (int k = threadIdx.x; k < kn; k += blockDim.x) {
        double2* x = xs + k * pitch;
        // forward: the interchanges and L; cur = the running row i (rows < i are final)
        double2 cur = x[0];
#pragma unroll 4
        for (int i = 0; i + 1 < nb; ++i) {
            // row i's final value s (the next row when rows i, i+1 were interchanged) and the
            // running row i+1: o - l s (branch-free: the selects sit beside the chain)
            const double2 nxt = x[i + 1], d = dl[i];
            const bool p = ps[i] != 0;
            const double2 s = p ? nxt : cur, o = p ? cur : nxt;
            x[i] = s;
            cur = make_double2(fma(-d.x, s.x, fma(d.y, s.y, o.x)), fma(-d.x, s.y, fma(-d.y, s.x, o.y)));
        }
        // back: x_i = x_i / d_i - (du_i / d_i) x_{i+1} - (du2_i / d_i) x_{i+2}
        double2 x1 = cm(cur, di[nb - 1]), x2 = make_double2(0.0, 0.0);
        x[nb - 1] = x1;
#pragma unroll 4
        for (int i = nb - 2; i >= 0; --i) {
            const double2 a = csub(cm(x[i], di[i]), cm(ud2[i], x2));  // off the x1 chain
            const double2 u = ud[i];
            const double2 v =
                make_double2(fma(-u.x, x1.x, fma(u.y, x1.y, a.x)), fma(-u.x, x1.y, fma(-u.y, x1.x, a.y)));
            x[i] = v;
            x2 = x1;
            x1 = v;
        }
    }
    __syncthreads();
    double2* out = UP ? W + int64_t(j) * blk + off : T + int64_t(b) * blk + off;
    for (int e = threadIdx.x; e < tot; e += blockDim.x) out[e] = xs[(e / nb) * pitch + e % nb];
}

dim3 ew_grid(int64_t work, int batch) {
    int64_t g = (work + 255) / 256;
    if (g > 1024) g = 1024;
    return dim3(unsigned(g), unsigned(batch));
}

}  // namespace

// Factorisation (exact.cu chooses it for short lines and many of them). col_lines / nx
// describe the line geometry, coup the level-0 couplings (L x nb). status: exact.cu's.
BcrFactor* bcr_factor(Ctx& c, bool col_lines, int nb, int L, const double2* coup, int* status) {
    auto f = std::make_unique<BcrFactor>();
    f->nb = nb;
    f->L = L;
    const int64_t nn = int64_t(nb) * nb;
    // level geometry and storage
    size_t blocks = 0;
    {
        int m = L, line0 = 0, step = 1;
        for (;;) {
            BcrLevel v;
            v.m = m;
            v.line0 = line0;
            v.step = step;
            v.ne = (m + 1) / 2;
            v.no = m / 2;
            v.t_off = f->t_blocks;
            f->t_blocks += v.ne;
            const bool l0 = f->lv.empty();
            blocks += v.ne + (l0 ? 0 : 2 * size_t(v.ne) + size_t(std::max(m - 1, 0)));
            f->lv.push_back(v);
            if (m == 1) break;
            m = v.no;
            line0 = line0 + step;
            step *= 2;
        }
    }
    f->store.alloc(blocks * nn);
    {
        double2* p = f->store.p;
        for (size_t l = 0; l < f->lv.size(); ++l) {
            BcrLevel& v = f->lv[l];
            v.M = p;
            p += v.ne * nn;
            if (l > 0) {
                v.P = p;
                p += v.ne * nn;
                v.Q = p;
                p += v.ne * nn;
                v.U = p;
                p += std::max(v.m - 1, 0) * nn;
            }
        }
    }
    // scratch for the next level's D (and the level's U^T, U_j M_{j+1})
    DevBuf<double2> D(size_t(std::max(L / 2, 1)) * nn), S1(size_t(std::max(L / 2, 1)) * nn),
        S2(size_t(std::max(L / 2, 1)) * nn);
    const size_t gsm = size_t(2 * nb) * sizeof(double2) + size_t((nb + 3) & ~3) * sizeof(int);
    CK(cudaFuncSetAttribute(gj_batched, cudaFuncAttributeMaxDynamicSharedMemorySize, int(gsm)));
    const cudaStream_t st = c.stream;
    auto gj = [&](double2* A, int count, int line0, int lstep) {
        if (count <= 0) return;
        gj_batched<<<count, 512, gsm, st>>>(nb, A, line0, lstep, status);
        CK_LAUNCH();
    };
    // level 0
    {
        BcrLevel& v = f->lv[0];
        l0_even<<<ew_grid(nn, v.ne), 256, 0, st>>>(col_lines, c.nx, nb, v.ne, c.diag.p, c.east.p, c.south.p, v.M);
        CK_LAUNCH();
        gj(v.M, v.ne, 0, 2);
        // FWI_BCR_L0=gemm keeps the dense M_b products at level 0 (diagnostics)
        const char* e0 = std::getenv("FWI_BCR_L0");
        if (!(e0 && std::string(e0) == "gemm") && size_t(4 * nb) * sizeof(double2) + size_t(nb) + 8 * size_t(nb + 1) *
                                                     sizeof(double2) <= kTriSmem) {
            f->tri.alloc(size_t(v.ne) * 4 * nb);
            f->tpiv.alloc(size_t(v.ne) * nb);
            l0_gttrf<<<(v.ne + 63) / 64, 64, 0, st>>>(col_lines, c.nx, nb, v.ne, c.diag.p, c.east.p, c.south.p,
                                                      f->tri.p, f->tpiv.p);
            CK_LAUNCH();
            f->tri_ok = true;
        }
        if (v.no > 0) {
            BcrLevel& w = f->lv[1];
            l0_schur<<<ew_grid(nn, v.no), 256, 0, st>>>(col_lines, c.nx, nb, v.m, v.no, c.diag.p, c.east.p, c.south.p,
                                                       coup, v.M, D.p, w.U);
            CK_LAUNCH();
        }
    }
    // levels >= 1: D (m blocks, in D), U (m-1 blocks, in lv[l].U)
    for (size_t l = 1; l < f->lv.size(); ++l) {
        BcrLevel& v = f->lv[l];
        const int m = v.m;
        // M_b = D_{2b}^{-1}
        launch_pdl<kPdlDense>(copy_blocks, dim3(ew_grid(nn, v.ne)), dim3(256), 0, st, nn, v.ne, D.p, 2 * nn, v.M, nn);
        CK_LAUNCH();
        gj(v.M, v.ne, v.line0, 2 * v.step);
        // P_b = M_b U_{2b-1}^T (b >= 1), Q_b = M_b U_{2b} (2b < m-1)
        if (v.ne > 1)
            cgemm_batched(st, true, nb, nb, nb, 1.0, v.M + nn, nb, nn, v.U + nn, nb, 2 * nn, nullptr, 0, 0, v.P + nn,
                          nb, nn, v.ne - 1);
        const int nq = (m - 1 + 1) / 2;  // b with 2b < m-1
        if (nq > 0)
            cgemm_batched(st, false, nb, nb, nb, 1.0, v.M, nb, nn, v.U, nb, 2 * nn, nullptr, 0, 0, v.Q, nb, nn, nq);
        if (v.no == 0) break;
        BcrLevel& w = f->lv[l + 1];
        // D'_b = D_{2b+1} - U_{2b}^T Q_b - U_{2b+1} P_{b+1}
        transpose_blocks<<<dim3((nb + 31) / 32, (nb + 31) / 32, unsigned(m - 1)), dim3(32, 8), 0, st>>>(nb, v.U, S1.p);
        CK_LAUNCH();
        // (the odd D blocks move to S2 first: D is rewritten as the next level's D)
        launch_pdl<kPdlDense>(copy_blocks, dim3(ew_grid(nn, v.no)), dim3(256), 0, st, nn, v.no, D.p + nn, 2 * nn, S2.p,
                              nn);
        CK_LAUNCH();
        cgemm_batched(st, false, nb, nb, nb, -1.0, S1.p, nb, 2 * nn, v.Q, nb, nn, S2.p, nb, nn, D.p, nb, nn, v.no);
        const int np = std::min(v.no, v.ne - 1);  // b with 2b+2 < m
        if (np > 0)
            cgemm_batched(st, false, nb, nb, nb, -1.0, v.U + nn, nb, 2 * nn, v.P + nn, nb, nn, D.p, nb, nn, D.p, nb, nn,
                          np);
        // U'_b = -(U_{2b+1} M_{b+1}) U_{2b+2}, b < no - 1
        if (v.no > 1) {
            cgemm_batched(st, false, nb, nb, nb, 1.0, v.U + nn, nb, 2 * nn, v.M + nn, nb, nn, nullptr, 0, 0, S1.p, nb,
                          nn, v.no - 1);
            cgemm_batched(st, false, nb, nb, nb, -1.0, S1.p, nb, nn, v.U + 2 * nn, nb, 2 * nn, nullptr, 0, 0, w.U, nb,
                          nn, v.no - 1);
        }
    }
    return f.release();
}

// Solve for nrhs right-hand sides in the line-major buffer W (W[line][k][m], overwritten
// by the solution).
void bcr_solve(Ctx& c, BcrFactor& f, const double2* coup, double2* W, int nrhs) {
    const int nb = f.nb;
    const int64_t nn = int64_t(nb) * nb, blk = int64_t(nrhs) * nb;
    if (f.nrhs_cap < nrhs) {
        f.t.alloc(f.t_blocks * size_t(blk));
        f.r.alloc(size_t(f.lv[0].ne) * size_t(blk));
        // split-K partials: the narrow levels (< ~2 x SMs tiles), K / 32 chunks each
        // (a split GEMM has fewer than 2 x SMs tiles, so at most that many batch entries)
        f.part.alloc(size_t(std::min(f.lv[0].ne, 2 * sm_count())) * size_t((nb + 31) / 32) * size_t(blk));
        f.nrhs_cap = nrhs;
    }

    const cudaStream_t st = c.stream;
    double2* T = f.t.p;
    auto Wl = [&](const BcrLevel& v, int j) { return W + int64_t(v.line0 + j * v.step) * blk; };
    // FWI_BCR_GEMM=tiled: the tiled DMMA kernel for the t = M b products (diagnostics)
    static const bool tiled = std::getenv("FWI_BCR_GEMM") && std::string(std::getenv("FWI_BCR_GEMM")) == "tiled";
    static const bool warp_only = std::getenv("FWI_BCR_GEMM") && std::string(std::getenv("FWI_BCR_GEMM")) == "warp";
    auto term = [](const double2* A, int64_t sA, const double2* B, int64_t sB, double alpha, bool bt, int lo, int hi,
                   int nb_) {
        return CgemmTerm{A, nb_, sA, B, nb_, sB, alpha, bt, lo, hi};
    };
    auto emit = [&](const CgemmTerm& ta, const CgemmTerm* tb, const double2* C0, int64_t sC0, double2* C, int64_t sC,
                    int batch) { cgemm2(st, nrhs, nb, nb, ta, tb, C0, nb, sC0, C, nb, sC, batch); };
    // level-0 tridiagonal solves: column chunks of kc right-hand sides per CTA
    auto tri_solve = [&](bool up, const BcrLevel& v, double2* Tl) {
        const size_t fixed = size_t(4 * nb) * sizeof(double2) + size_t(nb + 15) / 16 * 16;
        const size_t fit = (kTriSmem - fixed) / (size_t(nb + 1) * sizeof(double2));
        const int kc = int(std::min<size_t>(std::min(nrhs, kTriCols), fit));
        const size_t smem = fixed + size_t(kc) * (nb + 1) * sizeof(double2);
        static bool attr = false;
        if (!attr) {
            CK(cudaFuncSetAttribute(l0_tri_solve<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kTriSmem)));
            CK(cudaFuncSetAttribute(l0_tri_solve<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kTriSmem)));
            attr = true;
        }
        const dim3 g(unsigned(v.ne), unsigned((nrhs + kc - 1) / kc));
        if (up)
            launch_pdl<kPdlDense>(l0_tri_solve<true>, dim3(g), dim3(kTriThreads), smem, st, nb, v.m, kc, nrhs, blk,
                                  f.tri.p, f.tpiv.p, coup, W, Tl);
        else
            launch_pdl<kPdlDense>(l0_tri_solve<false>, dim3(g), dim3(kTriThreads), smem, st, nb, v.m, kc, nrhs, blk,
                                  f.tri.p, f.tpiv.p, coup, W, Tl);
        CK_LAUNCH();
    };
    // down
    for (size_t l = 0; l < f.lv.size(); ++l) {
        const BcrLevel& v = f.lv[l];
        double2* Tl = T + v.t_off * blk;
        const int64_t sw = 2 * int64_t(v.step) * blk;  // W stride between same-parity blocks
        // t_b = M_b b_{2b} (rows k of b times M^T); level 0: the tridiagonal factors
        if (l == 0 && f.tri_ok)
            tri_solve(false, v, Tl);
        else if (tiled || (v.ne >= kBcrTiledBatch && !warp_only))
            cgemm_batched(st, true, nrhs, nb, nb, 1.0, Wl(v, 0), nb, sw, v.M, nb, nn, nullptr, 0, 0, Tl, nb, blk, v.ne,
                          f.part.p, f.part.count);
        else
            emit(term(Wl(v, 0), sw, v.M, nn, 1.0, true, 0, v.ne, nb), nullptr, nullptr, 0, Tl, blk, v.ne);
        if (v.no == 0) break;
        if (l == 0) {
            launch_pdl<kPdlDense>(l0_down, dim3(ew_grid(blk, v.no)), dim3(256), 0, st, nb, v.m, blk, coup, Tl, W);
            CK_LAUNCH();
        } else {
            // b_{2b+1} -= U_{2b}^T t_b (rows: t_b U_{2b}) + U_{2b+1} t_{b+1} (rows: t_{b+1} U_{2b+1}^T)
            const int np = std::min(v.no, v.ne - 1);
            if (v.no >= kBcrTiledBatch2 && !warp_only) {
                cgemm_batched(st, false, nrhs, nb, nb, -1.0, Tl, nb, blk, v.U, nb, 2 * nn, Wl(v, 1), nb, sw, Wl(v, 1),
                              nb, sw, v.no, f.part.p, f.part.count);
                if (np > 0)
                    cgemm_batched(st, true, nrhs, nb, nb, -1.0, Tl + blk, nb, blk, v.U + nn, nb, 2 * nn, Wl(v, 1), nb,
                                  sw, Wl(v, 1), nb, sw, np, f.part.p, f.part.count);
            } else {
                const CgemmTerm ta = term(Tl, blk, v.U, 2 * nn, -1.0, false, 0, v.no, nb);
                const CgemmTerm tb = term(Tl + blk, blk, v.U + nn, 2 * nn, -1.0, true, 0, np, nb);
                emit(ta, np > 0 ? &tb : nullptr, Wl(v, 1), sw, Wl(v, 1), sw, v.no);
            }
        }
    }
    // up
    for (size_t li = f.lv.size(); li-- > 0;) {
        const BcrLevel& v = f.lv[li];
        double2* Tl = T + v.t_off * blk;
        const int64_t sw = 2 * int64_t(v.step) * blk;
        if (li == 0 && f.tri_ok) {  // x_{2b} = T_{2b}^{-1}(b_{2b} - E x_{2b-1} - E x_{2b+1})
            tri_solve(true, v, Tl);
        } else if (li == 0) {
            if (v.m > 1) {
                launch_pdl<kPdlDense>(l0_up_rhs, dim3(ew_grid(blk, v.ne)), dim3(256), 0, st, nb, v.m, blk, coup, W,
                                      f.r.p);
                CK_LAUNCH();
            } else {
                CK(cudaMemsetAsync(f.r.p, 0, size_t(blk) * sizeof(double2), st));
            }
            // x_{2b} = t_b - R_b M_b^T
            if (v.ne >= kBcrTiledBatch && !warp_only)
                cgemm_batched(st, true, nrhs, nb, nb, -1.0, f.r.p, nb, blk, v.M, nb, nn, Tl, nb, blk, Wl(v, 0), nb, sw,
                              v.ne, f.part.p, f.part.count);
            else
                cgemm2(st, nrhs, nb, nb, term(f.r.p, blk, v.M, nn, -1.0, true, 0, v.ne, nb), nullptr, Tl, nb, blk,
                       Wl(v, 0), nb, sw, v.ne);
        } else {
            // x_{2b} = t_b - x_{2b-1} P_b^T (b >= 1) - x_{2b+1} Q_b^T (2b+1 < m)
            const int nq = v.m / 2;
            if (v.ne >= kBcrTiledBatch2 && !warp_only) {  // copy t, then both products in place
                launch_pdl<kPdlDense>(copy_blocks, dim3(ew_grid(blk, v.ne)), dim3(256), 0, st, blk, v.ne, Tl, blk,
                                      Wl(v, 0), sw);
                CK_LAUNCH();
                if (v.ne > 1)
                    cgemm_batched(st, true, nrhs, nb, nb, -1.0, Wl(v, 1), nb, sw, v.P + nn, nb, nn, Wl(v, 2), nb, sw,
                                  Wl(v, 2), nb, sw, v.ne - 1, f.part.p, f.part.count);
                if (nq > 0)
                    cgemm_batched(st, true, nrhs, nb, nb, -1.0, Wl(v, 1), nb, sw, v.Q, nb, nn, Wl(v, 0), nb, sw, Wl(v, 0),
                                  nb, sw, nq, f.part.p, f.part.count);
                continue;
            }
            const CgemmTerm tp = term(Wl(v, 1), sw, v.P + nn, nn, -1.0, true, 1, v.ne, nb);
            const CgemmTerm tq = term(Wl(v, 1), sw, v.Q, nn, -1.0, true, 0, nq, nb);
            if (v.ne > 1)
                emit(tp, nq > 0 ? &tq : nullptr, Tl, blk, Wl(v, 0), sw, v.ne);
            else
                emit(tq, nullptr, Tl, blk, Wl(v, 0), sw, v.ne);  // (tq empty when nq = 0: x = t)
        }
    }
}

}  // namespace fwi_b200
