// exact.cu — the exact Helmholtz block solver of the block-triangular
// preconditioner (K2/K4, exact mode) and of the forward/adjoint field solves.
//
// Reference semantics: LuFactors::solve (src/lu.cpp:168-209) — x = A^{-1} b,
// or A^{-H} b — with a factorisation done once per Newton step
// (LuFactors::factor, src/lu.cpp:37-166). The reference uses a natural-order
// sparse LU whose solve DAG is a chain; that is the wrong shape
// for a GPU. Here the grid is cut into L lines of nb = min(nx, nz) nodes
// (along the shorter axis), which makes A block-tridiagonal with tridiagonal
// diagonal blocks T_i and diagonal couplings E_i. The exact block LU
//
//     S_0 = T_0,   S_i = T_i - E_{i-1} S_{i-1}^{-1} E_{i-1},   G_i = S_i^{-1}
//
// is built on the device (one Gauss-Jordan inversion per line, partial
// pivoting), and a solve for K right-hand sides is two sweeps of dense
// (nb x nb) x (nb x K) products:
//
//     forward  y_i = G_i (b_i - E_{i-1} y_{i-1})
//     backward x_i = y_i - G_i E_i x_{i+1}
//
// The adjoint uses exact complex symmetry (A^T = A bitwise):
// A^{-H} b = conj(A^{-1} conj(b)). Storage: L * nb^2 complex128
// (C1: 8.4 MB, C3: 100 MB, C5: 34 GB), read twice per solve.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>
#include <array>
#include <chrono>
#include <mutex>
#include <type_traits>
#include <cstdio>
#include <vector>

#include "ctx.cuh"
#include "dense.cuh"

namespace fwi_b200 {

struct ExactFactor {
    int L = 0, nb = 0;
    bool col_lines = true;  // lines are grid columns (fixed ix) when nz <= nx
    int gp = 0;             // row pitch of G (nb + 1: padded against smem bank conflicts)
    DevBuf<double2> G;      // L x nb x gp, G[i][m][j] = (S_i^{-1})[m][j]
    DevBuf<double2> coup;   // L x nb, coupling line i -> i+1 at position m
    DevBuf<double2> work;   // nb x nb scratch (global-memory inversion)
    DevBuf<double2> ybuf;   // forward-sweep results of the cluster sweep
    DevBuf<int> status;
    bool dense = false;     // long lines: GEMM line sweeps (dense.cu)
    bool dense_factor = false;  // whole-GPU block Gauss-Jordan per line (dense.cu)
    bool twisted = false;       // factored from both ends towards line `mid` (two sweep chains)
    double probe_residual = -1; // ||b - A A^{-1} b|| / ||b|| of the post-factorisation probe
    bool refactored = false;    // the probe forced whole-line pivoting
    int mid = 0;
    DenseWork dwork;
    DevBuf<double2> tbuf;   // dense sweep operand (nrhs x nb)
    // the second chain of a twisted dense factor / sweep runs on its own stream
    cudaStream_t s2 = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    DenseWork dwork2;
    DevBuf<double2> tbuf2;
    BcrFactor* bcr = nullptr;  // block cyclic reduction (bcr.cu) instead of the Schur sweeps
    void ensure_side() {
        if (s2) return;
        CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    }
    ~ExactFactor() {
        if (bcr) bcr_free(bcr);
        if (s2) {
            cudaStreamSynchronize(s2);
            cudaStreamDestroy(s2);
        }
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
    }
};

void exact_free(ExactFactor* f) { delete f; }
int64_t exact_bytes(const ExactFactor* f) {
    return f ? int64_t(f->G.bytes() + f->coup.bytes()) + bcr_bytes(f->bcr) : 0;
}

namespace {

__device__ __forceinline__ int64_t line_node(bool col_lines, int nx, int i, int m) {
    return col_lines ? int64_t(m) * nx + i : int64_t(i) * nx + m;
}

__device__ __forceinline__ double2 fmul(double2 a, double2 b) {  // fast complex multiply
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 fdiv(double2 a, double2 b) { return cdiv(a, b); }

// coupling planes of each line
__global__ void extract_lines(bool col_lines, int nx, int L, int nb, const double2* __restrict__ east,
                              const double2* __restrict__ south, double2* __restrict__ coup) {
    const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (t >= int64_t(L) * nb) return;
    const int i = int(t / nb), m = int(t % nb);
    const int64_t node = line_node(col_lines, nx, i, m);
    coup[t] = col_lines ? east[node] : south[node];
}

// S_i = T_i - E_a G_a E_a - E_b G_b E_b into A (row pitch gp), one thread per entry;
// (cA, GA) is the neighbour already eliminated on one side (the previous line of a
// sweep), (cB, GB) the other side (the twisted factorisation's middle line), either null.
__global__ void form_schur(bool col_lines, int nx, int nb, int line, const double2* __restrict__ diag,
                           const double2* __restrict__ east, const double2* __restrict__ south,
                           const double2* __restrict__ cA, const double2* __restrict__ GA,
                           const double2* __restrict__ cB, const double2* __restrict__ GB, int gp,
                           double2* __restrict__ A) {
    const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (t >= int64_t(nb) * nb) return;
    const int a = int(t / nb), b = int(t % nb);
    double2 v = make_double2(0.0, 0.0);
    const int64_t na = line_node(col_lines, nx, line, a);
    if (a == b) v = diag[na];
    else if (b == a + 1) v = col_lines ? south[na] : east[na];
    else if (a == b + 1) v = col_lines ? south[line_node(col_lines, nx, line, b)]
                                       : east[line_node(col_lines, nx, line, b)];
    if (GA) {
        const double2 t2 = fmul(fmul(cA[a], GA[int64_t(a) * gp + b]), cA[b]);
        v.x -= t2.x;
        v.y -= t2.y;
    }
    if (GB) {
        const double2 t2 = fmul(fmul(cB[a], GB[int64_t(a) * gp + b]), cB[b]);
        v.x -= t2.x;
        v.y -= t2.y;
    }
    A[int64_t(a) * gp + b] = v;
}

// Form S_i (row-major, in A) from the line's tridiagonal block and G_{i-1},
// then invert it in place by Gauss-Jordan with partial pivoting and write
// G_i transposed into GT_i. A lives in shared memory (small nb) or in a
// global scratch (large nb). One CTA per line; lines are launched in order.
template <bool SMEM>
__global__ void __launch_bounds__(512) line_factor_kernel(
    bool col_lines, int nx, int nb, int line, const double2* __restrict__ diag,
    const double2* __restrict__ east, const double2* __restrict__ south,
    const double2* __restrict__ coup, const double2* __restrict__ Gprev, double2* __restrict__ Gout, int gp,
    double2* gwork, int* status) {
    extern __shared__ double2 dsm[];
    double2* prow = dsm;
    double2* pcol = dsm + nb;
    int* piv = reinterpret_cast<int*>(dsm + 2 * nb);
    double2* A = SMEM ? reinterpret_cast<double2*>(piv + ((nb + 3) & ~3)) : gwork;
    __shared__ double red_v[32];
    __shared__ int red_i[32];
    __shared__ int s_p;
    __shared__ double2 s_pivinv;
    const int tid = threadIdx.x, nt = blockDim.x;

    // ---- S_i = T_i - E_{i-1} G_{i-1} E_{i-1}
    const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
    for (int a = wid; a < nb; a += nw)
        for (int b = lane; b < nb; b += 32) {
            double2 v = make_double2(0.0, 0.0);
            const int64_t na = line_node(col_lines, nx, line, a);
            if (a == b) v = diag[na];
            else if (b == a + 1) v = col_lines ? south[na] : east[na];
            else if (a == b + 1) v = col_lines ? south[line_node(col_lines, nx, line, b)]
                                               : east[line_node(col_lines, nx, line, b)];
            if (line > 0) {
                const double2 ea = coup[int64_t(line - 1) * nb + a], eb = coup[int64_t(line - 1) * nb + b];
                const double2 g = Gprev[int64_t(a) * gp + b];  // G_{i-1}[a][b]
                const double2 t2 = fmul(fmul(ea, g), eb);
                v.x -= t2.x;
                v.y -= t2.y;
            }
            A[a * nb + b] = v;
        }
    __syncthreads();

    // ---- Gauss-Jordan inversion with row pivoting
    for (int k = 0; k < nb; ++k) {
        double best = -1.0;
        int bi = nb;
        for (int r = k + tid; r < nb; r += nt) {
            const double2 v = A[int64_t(r) * nb + k];
            const double m2 = v.x * v.x + v.y * v.y;
            if (m2 > best || (m2 == best && r < bi)) { best = m2; bi = r; }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_down_sync(0xffffffffu, best, o);
            const int oi = __shfl_down_sync(0xffffffffu, bi, o);
            if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
        }
        if ((tid & 31) == 0) { red_v[tid >> 5] = best; red_i[tid >> 5] = bi; }
        __syncthreads();
        if (tid == 0) {
            double bv = -1.0;
            int b = nb;
            for (int w = 0; w < (nt + 31) / 32; ++w)
                if (red_v[w] > bv || (red_v[w] == bv && red_i[w] < b)) { bv = red_v[w]; b = red_i[w]; }
            if (!(bv > 0.0)) {
                atomicCAS(status, 0, line * nb + k + 1);
                b = k;
            }
            s_p = b;
            piv[k] = b;
        }
        __syncthreads();
        const int p = s_p;
        if (p != k)
            for (int j = tid; j < nb; j += nt) {
                const double2 t = A[int64_t(k) * nb + j];
                A[int64_t(k) * nb + j] = A[int64_t(p) * nb + j];
                A[int64_t(p) * nb + j] = t;
            }
        __syncthreads();
        if (tid == 0) {
            const double2 d = A[int64_t(k) * nb + k];
            s_pivinv = (d.x == 0.0 && d.y == 0.0) ? make_double2(0.0, 0.0)
                                                  : fdiv(make_double2(1.0, 0.0), d);
        }
        __syncthreads();
        const double2 pinv = s_pivinv;
        for (int j = tid; j < nb; j += nt) {
            const double2 a = (j == k) ? make_double2(1.0, 0.0) : A[int64_t(k) * nb + j];
            const double2 v = fmul(a, pinv);
            prow[j] = v;
            A[int64_t(k) * nb + j] = v;
            pcol[j] = (j == k) ? make_double2(0.0, 0.0) : A[int64_t(j) * nb + k];
        }
        __syncthreads();
        for (int r = wid; r < nb; r += nw) {
            if (r == k) continue;
            const double2 f = pcol[r];
            for (int j = lane; j < nb; j += 32) {
                double2 v = (j == k) ? make_double2(0.0, 0.0) : A[r * nb + j];
                const double2 pr = prow[j];
                v.x -= f.x * pr.x - f.y * pr.y;
                v.y -= f.x * pr.y + f.y * pr.x;
                A[r * nb + j] = v;
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
    for (int m = wid; m < nb; m += nw)
        for (int j = lane; j < nb; j += 32) Gout[int64_t(m) * gp + j] = A[m * nb + j];
}

// source-major b_k[node]  ->  line-major W[i][k][m] (optionally conjugated)
// and back. A 32x32 tile transpose in shared memory keeps both sides
// coalesced for column lines; row lines are a plain strided copy.
__global__ void gather_lines(bool col_lines, int nx, int nz, int L, int nb, int nrhs, bool conj,
                             const double2* __restrict__ src, double2* __restrict__ W) {
    pdl_enter();
    __shared__ double2 tile[32][33];
    const int k = blockIdx.z;
    const int64_t n = int64_t(nx) * nz;
    const double sg = conj ? -1.0 : 1.0;
    if (col_lines) {
        // node = m*nx + i ; read along i (x), write along m
        const int i0 = blockIdx.x * 32, m0 = blockIdx.y * 32;
        for (int r = threadIdx.y; r < 32; r += blockDim.y) {
            const int m = m0 + r, i = i0 + threadIdx.x;
            if (m < nb && i < L) {
                const double2 v = src[int64_t(k) * n + int64_t(m) * nx + i];
                tile[r][threadIdx.x] = make_double2(v.x, sg * v.y);
            }
        }
        __syncthreads();
        for (int r = threadIdx.y; r < 32; r += blockDim.y) {
            const int i = i0 + r, m = m0 + threadIdx.x;
            if (m < nb && i < L) W[(int64_t(i) * nrhs + k) * nb + m] = tile[threadIdx.x][r];
        }
    } else {
        const int m0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
        for (int r = threadIdx.y; r < 32; r += blockDim.y) {
            const int i = i0 + r, m = m0 + threadIdx.x;
            if (m < nb && i < L) {
                const double2 v = src[int64_t(k) * n + int64_t(i) * nx + m];
                W[(int64_t(i) * nrhs + k) * nb + m] = make_double2(v.x, sg * v.y);
            }
        }
    }
}

__global__ void scatter_lines(bool col_lines, int nx, int nz, int L, int nb, int nrhs, bool conj,
                              const double2* __restrict__ W, double2* __restrict__ dst) {
    pdl_enter();
    __shared__ double2 tile[32][33];
    const int k = blockIdx.z;
    const int64_t n = int64_t(nx) * nz;
    const double sg = conj ? -1.0 : 1.0;
    if (col_lines) {
        const int i0 = blockIdx.x * 32, m0 = blockIdx.y * 32;
        for (int r = threadIdx.y; r < 32; r += blockDim.y) {
            const int i = i0 + r, m = m0 + threadIdx.x;
            if (m < nb && i < L) tile[threadIdx.x][r] = W[(int64_t(i) * nrhs + k) * nb + m];
        }
        __syncthreads();
        for (int r = threadIdx.y; r < 32; r += blockDim.y) {
            const int m = m0 + r, i = i0 + threadIdx.x;
            if (m < nb && i < L) {
                const double2 v = tile[r][threadIdx.x];
                dst[int64_t(k) * n + int64_t(m) * nx + i] = make_double2(v.x, sg * v.y);
            }
        }
    } else {
        const int m0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
        for (int r = threadIdx.y; r < 32; r += blockDim.y) {
            const int i = i0 + r, m = m0 + threadIdx.x;
            if (m < nb && i < L) {
                const double2 v = W[(int64_t(i) * nrhs + k) * nb + m];
                dst[int64_t(k) * n + int64_t(i) * nx + m] = make_double2(v.x, sg * v.y);
            }
        }
    }
}

// Forward + backward block sweep for a group of KG right-hand sides, in place
// on the line-major W. Thread layout: nb rows x S segments of the inner
// dimension (S = 256/nb when nb <= 256), partial sums combined in fixed order.
template <int KG>
__global__ void __launch_bounds__(256) sweep_kernel(int L, int nb, int nrhs,
                                                    const double2* __restrict__ GT, int gp,
                                                    const double2* __restrict__ coup, double2* W) {
    extern __shared__ double2 sm[];
    double2* wv = sm;                 // KG x nb   operand
    double2* yv = sm + KG * nb;       // KG x nb   previous solution line
    double2* part = sm + 2 * KG * nb; // S x KG x nb partials
    const int k0 = blockIdx.x * KG;
    const int kc = min(KG, nrhs - k0);
    if (kc <= 0) return;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int S = nb <= nt ? nt / nb : 1;
    const int seg = (nb + S - 1) / S;
    const int my_s = nb <= nt ? tid / nb : 0;

    auto matvec = [&](const double2* G, bool subtract_into_y, int line) {
        // acc[k][m] = sum_j G[m][j] wv[k][j]  over this thread's (m, segment)
        for (int m0 = (nb <= nt ? tid % nb : tid); m0 < nb; m0 += (nb <= nt ? nb : nt)) {
            if (nb <= nt && tid >= S * nb) break;
            double2 acc[KG];
#pragma unroll
            for (int k = 0; k < KG; ++k) acc[k] = make_double2(0.0, 0.0);
            const int j0 = my_s * seg, j1 = min(nb, j0 + seg);
#pragma unroll 4
            for (int j = j0; j < j1; ++j) {
                const double2 g = __ldg(G + int64_t(m0) * gp + j);
#pragma unroll
                for (int k = 0; k < KG; ++k) {
                    const double2 w = wv[k * nb + j];
                    acc[k].x += g.x * w.x - g.y * w.y;
                    acc[k].y += g.x * w.y + g.y * w.x;
                }
            }
            if (S > 1) {
#pragma unroll
                for (int k = 0; k < KG; ++k) part[(my_s * KG + k) * nb + m0] = acc[k];
            } else {
#pragma unroll
                for (int k = 0; k < KG; ++k) {
                    if (k >= kc) break;
                    double2 r = acc[k];
                    if (subtract_into_y) {
                        const double2 y = yv[k * nb + m0];
                        r = make_double2(y.x - r.x, y.y - r.y);
                    }
                    part[k * nb + m0] = r;  // staged; committed after the barrier
                }
            }
        }
        __syncthreads();
        for (int t = tid; t < kc * nb; t += nt) {
            const int k = t / nb, m = t % nb;
            double2 r;
            if (S > 1) {
                r = make_double2(0.0, 0.0);
                for (int s = 0; s < S; ++s) {
                    const double2 p = part[(s * KG + k) * nb + m];
                    r.x += p.x;
                    r.y += p.y;
                }
                if (subtract_into_y) {
                    const double2 y = yv[k * nb + m];
                    r = make_double2(y.x - r.x, y.y - r.y);
                }
            } else {
                r = part[k * nb + m];
            }
            yv[k * nb + m] = r;
            W[(int64_t(line) * nrhs + k0 + k) * nb + m] = r;
        }
        __syncthreads();
    };

    // forward: y_i = G_i (b_i - E_{i-1} y_{i-1})
    for (int i = 0; i < L; ++i) {
        for (int t = tid; t < kc * nb; t += nt) {
            const int k = t / nb, m = t % nb;
            double2 b = W[(int64_t(i) * nrhs + k0 + k) * nb + m];
            if (i > 0) {
                const double2 e = coup[int64_t(i - 1) * nb + m];
                const double2 y = yv[k * nb + m];
                b.x -= e.x * y.x - e.y * y.y;
                b.y -= e.x * y.y + e.y * y.x;
            }
            wv[k * nb + m] = b;
        }
        __syncthreads();
        matvec(GT + int64_t(i) * nb * gp, false, i);
    }
    // backward: x_i = y_i - G_i E_i x_{i+1}; yv holds x_{i+1}
    for (int i = L - 2; i >= 0; --i) {
        for (int t = tid; t < kc * nb; t += nt) {
            const int k = t / nb, m = t % nb;
            const double2 e = coup[int64_t(i) * nb + m];
            const double2 x = yv[k * nb + m];
            wv[k * nb + m] = make_double2(e.x * x.x - e.y * x.y, e.x * x.y + e.y * x.x);
        }
        __syncthreads();
        // yv <- y_i (stored in W by the forward sweep) before subtracting
        for (int t = tid; t < kc * nb; t += nt) {
            const int k = t / nb, m = t % nb;
            yv[k * nb + m] = W[(int64_t(i) * nrhs + k0 + k) * nb + m];
        }
        __syncthreads();
        matvec(GT + int64_t(i) * nb * gp, true, i);
    }
}

// ---------------------------------------------------------------------------
// Cluster sweep: one thread-block cluster of CS CTAs carries a group of KG
// right-hand sides through all lines. CTA r owns rows [r*R, (r+1)*R) of every
// G_i; per line it computes its slab of y_i = G_i w and pushes it into the
// double-buffered full-vector copy of every CTA of the cluster through
// distributed shared memory, followed by one cluster barrier. The next line's
// G slab, coupling row and right-hand-side block are prefetched with bulk
// async copies (cp.async.bulk + mbarrier) while the current line computes.
// ---------------------------------------------------------------------------
struct SweepArgs {
    int L, nb, nrhs, gp, R;
    const double2* G;
    const double2* coup;
    double2* W;   // line-major RHS in, solution out
    double2* Y;   // line-major forward-sweep results (separate: W is still being read)
    uint32_t off_e, off_b, stage_bytes, off_y, off_w, off_part, off_bar;
    int nseg, nst;  // inner-dimension segments, pipeline stages (2..4)
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint64_t* b) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
            smem_addr(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(b))
                 : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t map_rank(uint32_t local_addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
    return r;
}
// remote store that completes 16 bytes on the receiver's mbarrier (no fence)
__device__ __forceinline__ void st_async16(uint32_t addr, double2 v, uint32_t remote_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(addr),
                 "d"(v.x), "d"(v.y), "r"(remote_bar)
                 : "memory");
}

template <int KG, int CS>
__global__ void __launch_bounds__(256) sweep_cluster_kernel(const SweepArgs a) {
    extern __shared__ __align__(128) unsigned char csm[];
    const int tid = threadIdx.x;
    const uint32_t rank = cluster_rank();
    const int grp = blockIdx.x / CS;
    const int nb = a.nb, L = a.L, R = a.R, gp = a.gp, nrhs = a.nrhs;
    const int nbp = nb + 1;
    const int k0 = grp * KG;
    const int kc = min(KG, nrhs - k0);
    const int r0 = int(rank) * R;
    const int rows = max(0, min(nb, r0 + R) - r0);
    double2* yfull = reinterpret_cast<double2*>(csm + a.off_y);  // [2][KG][nbp]
    double2* wv = reinterpret_cast<double2*>(csm + a.off_w);     // [KG][nbp]
    double2* part = reinterpret_cast<double2*>(csm + a.off_part);
    uint64_t* bar = reinterpret_cast<uint64_t*>(csm + a.off_bar);
    const int O = R * KG;  // outputs (row, rhs) per CTA
    const int nsteps = 2 * L - 1;

    // step s: forward line s (s < L), backward line 2L-2-s (s >= L)
    auto line_of = [&](int st) { return st < L ? st : 2 * L - 2 - st; };
    auto issue = [&](int st) {
        if (st >= nsteps) return;
        const int sb = st % a.nst;
        unsigned char* buf = csm + sb * a.stage_bytes;
        const int i = line_of(st);
        const bool fwd = st < L;
        const uint32_t gbytes = uint32_t(rows) * gp * sizeof(double2);
        const bool has_e = fwd ? i > 0 : true;
        const uint32_t ebytes = has_e ? uint32_t(nb) * sizeof(double2) : 0u;
        const uint32_t bbytes = fwd ? uint32_t(kc) * nb * sizeof(double2) : 0u;
        bar_expect(&bar[sb], gbytes + ebytes + bbytes);
        if (gbytes) bulk_g2s(buf, a.G + (int64_t(i) * nb + r0) * gp, gbytes, &bar[sb]);
        if (ebytes) bulk_g2s(buf + a.off_e, a.coup + int64_t(fwd ? i - 1 : i) * nb, ebytes, &bar[sb]);
        if (bbytes) bulk_g2s(buf + a.off_b, a.W + (int64_t(i) * nrhs + k0) * nb, bbytes, &bar[sb]);
    };
    uint64_t* rbar = bar + 4;  // receive barriers of the two y buffers
    const uint32_t recv_bytes = uint32_t(kc) * nb * sizeof(double2);
    if (tid == 0) {
        for (int q = 0; q < a.nst; ++q) bar_init(&bar[q]);
        bar_init(&rbar[0]);
        bar_init(&rbar[1]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int q = 0; q < a.nst; ++q) issue(q);
    }
    __syncthreads();
    cluster_sync_all();  // peers' barriers are initialised before any remote arrive

    for (int st = 0; st < nsteps; ++st) {
        const int i = line_of(st);
        const bool fwd = st < L;
        const unsigned char* buf = csm + (st % a.nst) * a.stage_bytes;
        const double2* Gs = reinterpret_cast<const double2*>(buf);
        const double2* es = reinterpret_cast<const double2*>(buf + a.off_e);
        const double2* bs = reinterpret_cast<const double2*>(buf + a.off_b);
        bar_wait(&bar[st % a.nst], (st / a.nst) & 1);
        // arm this step's receive buffer, then wait for all slabs of step st-1
        if (tid == 0 && st + 1 < nsteps) bar_expect(&rbar[st & 1], recv_bytes);
        if (st > 0) bar_wait(&rbar[(st - 1) & 1], ((st - 1) >> 1) & 1);
        const double2* yprev = yfull + ((st + 1) & 1) * KG * nbp;  // written at step st-1
        // w = b_i - E_{i-1} y_{i-1}  (forward)  |  w = E_i x_{i+1}  (backward)
        for (int t = tid; t < KG * nb; t += blockDim.x) {
            const int k = t / nb, m = t - k * nb;
            double2 v = make_double2(0.0, 0.0);
            if (k < kc) {
                if (fwd) {
                    v = bs[k * nb + m];
                    if (i > 0) {
                        const double2 e = es[m], y = yprev[k * nbp + m];
                        v.x -= e.x * y.x - e.y * y.y;
                        v.y -= e.x * y.y + e.y * y.x;
                    }
                } else {
                    const double2 e = es[m], x = yprev[k * nbp + m];
                    v = make_double2(e.x * x.x - e.y * x.y, e.x * x.y + e.y * x.x);
                }
            }
            wv[k * nbp + m] = v;
        }
        __syncthreads();
        // slab matvec: output o = (row, rhs), segments of the inner dimension
        const int seglen = (nb + a.nseg - 1) / a.nseg;
        for (int t = tid; t < O * a.nseg; t += blockDim.x) {
            const int o = t % O, seg = t / O;
            const int row = o / KG, k = o - row * KG;
            double2 acc = make_double2(0.0, 0.0), acc2 = make_double2(0.0, 0.0);
            if (row < rows) {
                const double2* g = Gs + row * gp;
                const double2* w = wv + k * nbp;
                const int j0 = seg * seglen, j1 = min(nb, j0 + seglen);
                int j = j0;
                for (; j + 1 < j1; j += 2) {  // two independent accumulator chains
                    const double2 g0 = g[j], x0 = w[j], g1 = g[j + 1], x1 = w[j + 1];
                    acc.x += g0.x * x0.x - g0.y * x0.y;
                    acc.y += g0.x * x0.y + g0.y * x0.x;
                    acc2.x += g1.x * x1.x - g1.y * x1.y;
                    acc2.y += g1.x * x1.y + g1.y * x1.x;
                }
                if (j < j1) {
                    const double2 g0 = g[j], x0 = w[j];
                    acc.x += g0.x * x0.x - g0.y * x0.y;
                    acc.y += g0.x * x0.y + g0.y * x0.x;
                }
            }
            part[seg * O + o] = make_double2(acc.x + acc2.x, acc.y + acc2.y);
        }
        __syncthreads();
        double2* ynext_local = yfull + (st & 1) * KG * nbp;
        for (int o = tid; o < O; o += blockDim.x) {
            const int row = o / KG, k = o - row * KG;
            if (row >= rows || k >= kc) continue;
            double2 v = make_double2(0.0, 0.0);
            for (int sg = 0; sg < a.nseg; ++sg) {
                const double2 pv = part[sg * O + o];
                v.x += pv.x;
                v.y += pv.y;
            }
            const int64_t gi = (int64_t(i) * nrhs + k0 + k) * nb + r0 + row;
            if (fwd) {
                a.Y[gi] = v;
            } else {
                const double2 y = a.Y[gi];  // y_i from the forward sweep
                v = make_double2(y.x - v.x, y.y - v.y);
                a.W[gi] = v;
            }
            if (fwd && i == L - 1) a.W[gi] = v;  // x_{L-1} = y_{L-1}
            if (st + 1 < nsteps) {  // the last step's slabs have no consumer
                const uint32_t la = smem_addr(ynext_local + k * nbp + r0 + row);
                const uint32_t lb = smem_addr(&rbar[st & 1]);
#pragma unroll
                for (int q = 0; q < CS; ++q) st_async16(map_rank(la, uint32_t(q)), v, map_rank(lb, uint32_t(q)));
            }
        }
        __syncthreads();  // stage (st % nst) and the partials are free
        if (tid == 0) issue(st + a.nst);
    }
    cluster_sync_all();  // no CTA leaves while peers may still address its shared memory
}

uint32_t al128(size_t b) { return uint32_t((b + 127) / 128 * 128); }

// ---------------------------------------------------------------------------
// Warp-specialised cluster sweep (v2). A cluster of CS CTAs owns KG right-hand
// sides; CTA `rank` owns rows [rank*R, rank*R+R) of every line block. Each
// consumer warp owns KR right-hand sides: it builds its own w_k = b_i - E y_{i-1}
// (or E_i x_{i+1}), multiplies the CTA's G slab with it (lane = (row, column
// residue class), fixed-order shuffle reduction over the classes) and pushes its
// slab of y_k to every peer with st.async, completing on a per-warp receive
// mbarrier there. A warp only ever waits for its own right-hand sides' data, so
// a line step needs no CTA barrier; the producer warp streams G slabs, coupling
// rows and RHS blocks into a ring of stages released by per-stage "empty"
// mbarriers. Per line step the critical path is: receive wake-up -> w -> matvec
// -> butterfly -> st.async (DSMEM latency ~200 cycles).
//
// Shared-memory traffic per step (the bound at large KG): G is read once per
// warp, i.e. KG/KR times, and each G element feeds KR complex MACs; columns are
// dealt to lanes round-robin (j = cls + ncls*t) so a warp's G and w loads hit
// distinct bank groups.
// ---------------------------------------------------------------------------
constexpr int kWMaxStages = 8;

// A chain of line steps over lines first, first+dir, ... (count lines):
//   mode 0: forward over the chain, then backward over it (the classical sweep);
//   mode 1: forward only (y_i into Y);
//   mode 2: backward only, starting from the boundary solution xin of the line
//           before `first` (x_i into W).
// The twisted solve runs two chains per launch (top and bottom half of the lines).
struct SweepChain {
    int first = 0, count = 0, dir = 1, mode = 0;
    const double2* xin = nullptr;  // mode 2: boundary line's solution, [k][m]
};

struct WSweepArgs {
    int L, nb, nrhs, gp, R, Rp, nst;
    const double2* G;
    const double2* coup;
    double2* W;
    double2* Y;
    uint32_t off_e, off_b, stage_bytes, off_y, off_w, off_bar;
    unsigned long long* trace;  // diagnostics: per-step clock64 stamps of CTA 0 / warp 0, or null
    SweepChain chain[2];        // clusters [0, groups0) run chain[0], the rest chain[1]
    int groups0;
};

__host__ __device__ __forceinline__ int chain_steps(const SweepChain& c) {
    return c.mode == 0 ? 2 * c.count - 1 : c.count;
}
__host__ __device__ __forceinline__ int chain_line(const SweepChain& c, int st) {
    return c.first + c.dir * ((c.mode == 0 && st >= c.count) ? 2 * c.count - 2 - st : st);
}
__host__ __device__ __forceinline__ bool chain_fwd(const SweepChain& c, int st) {
    return c.mode == 1 || (c.mode == 0 && st < c.count);
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %clock64;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void bar_init_n(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
// producer-side wait: polls with a back-off so the spinning warp leaves the issue
// slots of its sub-partition to the consumer warps on the critical path
__device__ __forceinline__ void bar_wait_lazy(uint64_t* b, uint32_t parity) {
    uint32_t done = 0;
    for (;;) {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_addr(b)), "r"(parity)
            : "memory");
        if (done) return;
        __nanosleep(128);
    }
}

__device__ __forceinline__ void cmac(double2& c, const double2 g, const double2 x) {
    c.x = fma(g.x, x.x, c.x);
    c.y = fma(g.x, x.y, c.y);
    c.x = fma(-g.y, x.y, c.x);
    c.y = fma(g.y, x.x, c.y);
}

template <int CS, int KG, int KR, bool TRACE, bool EVEN>
__global__ void __launch_bounds__((KG / KR + 1) * 32) sweep_warp_kernel(const WSweepArgs a) {
    pdl_enter();
    constexpr int NW = KG / KR;  // consumer warps
    extern __shared__ __align__(128) unsigned char wsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const int cid = blockIdx.x / CS;
    const int chn = cid < a.groups0 ? 0 : 1;
    const SweepChain C = a.chain[chn];
    const int grp = chn == 0 ? cid : cid - a.groups0;
    const int nb = a.nb, gp = a.gp, nrhs = a.nrhs, R = a.R, Rp = a.Rp;
    const int S = a.nst, smask = a.nst - 1;  // power of two
    const int nbp = nb + 1;
    const int k0 = grp * KG;
    const int kc = min(KG, nrhs - k0);
    const int r0 = int(rank) * R;
    const int rows = max(0, min(nb, r0 + R) - r0);
    double2* yfull = reinterpret_cast<double2*>(wsm + a.off_y);  // [2][KG][nbp]
    uint64_t* full = reinterpret_cast<uint64_t*>(wsm + a.off_bar);
    uint64_t* empty = full + kWMaxStages;
    uint64_t* rbar = empty + kWMaxStages;  // [2][NW]
    const int nsteps = chain_steps(C);
    const int last_fwd_line = C.first + C.dir * (C.count - 1);

    if (threadIdx.x == 0) {
        for (int q = 0; q < S; ++q) {
            bar_init(&full[q]);
            bar_init_n(&empty[q], NW);
        }
        for (int q = 0; q < 2 * NW; ++q) bar_init(&rbar[q]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    cluster_sync_all();  // peers' barriers exist before any remote arrive

    if (warp == NW) {  // ---- producer
        if (lane == 0) {
            const uint32_t gbytes = uint32_t(rows) * gp * sizeof(double2);
            const uint32_t ebytes = uint32_t(rows) * sizeof(double2);
            const uint32_t bbytes = uint32_t(kc) * nb * sizeof(double2);
            for (int st = 0; st < nsteps; ++st) {
                const int sb = st & smask;
                if (st >= S) bar_wait_lazy(&empty[sb], ((st - S) / S) & 1);
                unsigned char* buf = wsm + sb * a.stage_bytes;
                const bool fwd = chain_fwd(C, st);
                const int i = chain_line(C, st);
                // coupling that scales this step's result before it is pushed: the one
                // between this line and the chain's next line
                const int cidx = st + 1 < nsteps ? min(i, chain_line(C, st + 1)) : 0;
                const uint32_t eb = (st + 1 < nsteps) ? ebytes : 0u;
                const uint32_t bb = fwd ? bbytes : 0u;
                bar_expect(&full[sb], gbytes + eb + bb);
                if (gbytes) bulk_g2s(buf, a.G + (int64_t(i) * nb + r0) * gp, gbytes, &full[sb]);
                if (eb) bulk_g2s(buf + a.off_e, a.coup + int64_t(cidx) * nb + r0, eb, &full[sb]);
                if (bb) bulk_g2s(buf + a.off_b, a.W + (int64_t(i) * nrhs + k0) * nb, bb, &full[sb]);
            }
        }
    } else {  // ---- consumer warp: right-hand sides k0 + warp*KR + [0, KR)
        const int w = warp;
        const int kw = w * KR;                    // first local RHS of this warp
        const int kr = max(0, min(KR, kc - kw));  // active RHS of this warp
        const int ncls = 32 / Rp;
        const int row = lane & (Rp - 1), cls = lane / Rp;
        const bool has_row = row < rows;
        const int nj = (nb - cls + ncls - 1) / ncls;  // columns j = cls + ncls*t of this lane
        const bool tr = TRACE && blockIdx.x == 0 && w == 0 && lane == 0;
        // per-lane constant addresses
        const uint32_t rb_local0 = smem_addr(&rbar[w]), rb_local1 = smem_addr(&rbar[NW + w]);
        const uint32_t y_local0 = smem_addr(yfull + kw * nbp + r0 + row);
        const uint32_t y_buf_bytes = uint32_t(KG * nbp * sizeof(double2)), y_q_bytes = uint32_t(nbp * sizeof(double2));
        const int pfirst = cls, pstep = ncls;  // the row's lanes share the pushes to the CS peers
        double2* Yrow = a.Y + int64_t(k0 + kw) * nb + r0 + row;  // + i*nrhs*nb + q*nb
        double2* Wrow = a.W + int64_t(k0 + kw) * nb + r0 + row;
        const int64_t line_stride = int64_t(nrhs) * nb;
        const uint32_t rbytes = uint32_t(kr * nb) * 16u;

        // Received vectors are pre-scaled by the coupling (z = E y), so a step is
        //   forward   y_i = G_i (b_i - z_{i-1}),   backward  x_i = y_i - G_i z'_{i+1},
        // and the CTA scales its own rows of the result before pushing them.
        // EVEN: every lane owns a row and nj is a multiple of 4 (no element guards).
        if (C.mode == 2 && kr > 0) {
            // the chain's first step receives E (x of the boundary line) from global memory
            const int bl = C.first - C.dir;
            const double2* e = a.coup + int64_t(min(C.first, bl)) * nb;
            for (int q = 0; q < kr; ++q) {
                double2* dst = yfull + (KG + kw + q) * nbp;  // the buffer step 0 reads
                const double2* src = C.xin + int64_t(k0 + kw + q) * nb;
                for (int m = lane; m < nb; m += 32) {
                    const double2 ev = e[m], xv = src[m];
                    dst[m] = make_double2(ev.x * xv.x - ev.y * xv.y, ev.x * xv.y + ev.y * xv.x);
                }
            }
            __syncwarp();
        }
        int sb = 0;
        uint32_t fph = 0;
        auto step = [&](auto fwd_tag, auto first_tag, const int st, const int i) {
            constexpr bool fwd = decltype(fwd_tag)::value;
            constexpr bool first = decltype(first_tag)::value;
            if (tr) a.trace[8 * st] = gtimer();
            // backward: this thread wrote its rows of y_i itself in the forward sweep; load early
            double2 yown[KR];
            if (!fwd) {
#pragma unroll
                for (int q = 0; q < KR; ++q)
                    yown[q] = (q < kr && has_row) ? Yrow[i * line_stride + q * nb] : make_double2(0.0, 0.0);
            }
            bar_wait(&full[sb], fph);
            if (tr) a.trace[8 * st + 1] = gtimer();
            const unsigned char* buf = wsm + sb * a.stage_bytes;
            const double2* Gs = reinterpret_cast<const double2*>(buf);
            const double2* es = reinterpret_cast<const double2*>(buf + a.off_e);
            const double2* bs = reinterpret_cast<const double2*>(buf + a.off_b);
            if (kr > 0) {
                if (lane == 0 && st + 1 < nsteps)
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((st & 1) ? rb_local1
                                                                                                    : rb_local0),
                                 "r"(rbytes)
                                 : "memory");
                const double2* g = Gs + row * gp + cls;
                const double2* z = yfull + (((st + 1) & 1) * KG + kw) * nbp + cls;
                const double2* bq = bs + kw * nb + cls;
                const double2 esc = has_row && st + 1 < nsteps ? es[row] : make_double2(0.0, 0.0);
                if (!first && st > 0) bar_wait(&rbar[((st - 1) & 1) * NW + w], ((st - 1) >> 1) & 1);
                if (tr) a.trace[8 * st + 2] = gtimer();
                if (tr) a.trace[8 * st + 3] = gtimer();
                // w_j = b_j - z_j (forward) | b_j (first line) | z_j (backward)
                auto wval = [&](int q, int j) {
                    if constexpr (first) return bq[q * nb + j];
                    if constexpr (!fwd) return z[q * nbp + j];
                    const double2 b = bq[q * nb + j], zz = z[q * nbp + j];
                    return make_double2(b.x - zz.x, b.y - zz.y);
                };
                double2 acc[KR][4];
#pragma unroll
                for (int q = 0; q < KR; ++q) acc[q][0] = acc[q][1] = acc[q][2] = acc[q][3] = make_double2(0.0, 0.0);
                if constexpr (EVEN) {
#pragma unroll 2
                    for (int t = 0; t < nj; t += 4) {
                        double2 g4[4], w4[4][KR];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            g4[u] = g[(t + u) * ncls];
#pragma unroll
                            for (int q = 0; q < KR; ++q) w4[u][q] = wval(q, (t + u) * ncls);
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u)
#pragma unroll
                            for (int q = 0; q < KR; ++q) cmac(acc[q][u], g4[u], w4[u][q]);
                    }
                } else if (has_row) {
                    for (int t = 0; t < nj; ++t) {
                        const double2 g0 = g[t * ncls];
#pragma unroll
                        for (int q = 0; q < KR; ++q) cmac(acc[q][0], g0, wval(q, t * ncls));
                    }
                }
                double2 v[KR];
#pragma unroll
                for (int q = 0; q < KR; ++q) {
                    v[q] = make_double2((acc[q][0].x + acc[q][2].x) + (acc[q][1].x + acc[q][3].x),
                                        (acc[q][0].y + acc[q][2].y) + (acc[q][1].y + acc[q][3].y));
                    for (int off = Rp; off < 32; off <<= 1) {  // fixed-order class reduction
                        v[q].x += __shfl_xor_sync(0xffffffffu, v[q].x, off);
                        v[q].y += __shfl_xor_sync(0xffffffffu, v[q].y, off);
                    }
                }
                if (tr) a.trace[8 * st + 4] = gtimer();
                if (has_row) {  // every class lane holds the row totals after the butterfly
#pragma unroll
                    for (int q = 0; q < KR; ++q) {
                        if (q < kr) {
                            if (!fwd) v[q] = make_double2(yown[q].x - v[q].x, yown[q].y - v[q].y);
                            if (st + 1 < nsteps) {
                                const double2 zo = make_double2(esc.x * v[q].x - esc.y * v[q].y,
                                                                esc.x * v[q].y + esc.y * v[q].x);
                                const uint32_t la = y_local0 + ((st & 1) ? y_buf_bytes : 0u) + q * y_q_bytes;
                                const uint32_t lb = (st & 1) ? rb_local1 : rb_local0;
                                for (int p = pfirst; p < CS; p += pstep)
                                    st_async16(map_rank(la, uint32_t(p)), zo, map_rank(lb, uint32_t(p)));
                            }
                            if (cls == q % ncls) {
                                const int64_t off = i * line_stride + q * nb;
                                if (fwd) {
                                    Yrow[off] = v[q];
                                    if (C.mode == 0 && i == last_fwd_line) Wrow[off] = v[q];
                                } else {
                                    Wrow[off] = v[q];
                                }
                            }
                        }
                    }
                }
                if (tr) a.trace[8 * st + 5] = gtimer();
            }
            __syncwarp();
            if (lane == 0) bar_arrive(&empty[sb]);
            if (++sb == S) {
                sb = 0;
                fph ^= 1u;
            }
        };
        if (C.mode != 2) {
            step(std::true_type{}, std::true_type{}, 0, chain_line(C, 0));
            for (int st = 1; st < C.count; ++st) step(std::true_type{}, std::false_type{}, st, chain_line(C, st));
        }
        for (int st = (C.mode == 2 ? 0 : C.count); C.mode != 1 && st < nsteps; ++st)
            step(std::false_type{}, std::false_type{}, st, chain_line(C, st));
    }
    __syncthreads();
    cluster_sync_all();
}

// twisted solve, middle line: T[k][m] = b[k][m] - eA[m] yA[k][m] - eB[m] yB[k][m]
__global__ void middle_rhs(int nb, int64_t blk, const double2* __restrict__ b, const double2* __restrict__ eA,
                           const double2* __restrict__ yA, const double2* __restrict__ eB,
                           const double2* __restrict__ yB, double2* __restrict__ T) {
    pdl_enter();
    const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (t >= blk) return;
    const int m = int(t % nb);
    const double2 a = eA[m], ya = yA[t], e = eB[m], yb = yB[t];
    double2 v = b[t];
    v.x -= (a.x * ya.x - a.y * ya.y) + (e.x * yb.x - e.y * yb.y);
    v.y -= (a.x * ya.y + a.y * ya.x) + (e.x * yb.y + e.y * yb.x);
    T[t] = v;
}

// twisted solve, middle line for few right-hand sides: X[k][r] = sum_j G[r][j] T[k][j],
// one warp per row r (lanes split j, fixed-order butterfly), all k in registers
template <int KMAX>
__global__ void __launch_bounds__(256) middle_gemv(int nb, int nrhs, const double2* __restrict__ G, int gp,
                                                   const double2* __restrict__ T, double2* __restrict__ X) {
    pdl_enter();
    const int lane = threadIdx.x & 31;
    const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (r >= nb) return;
    double2 acc[KMAX];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) acc[k] = make_double2(0.0, 0.0);
    for (int j = lane; j < nb; j += 32) {
        const double2 g = G[int64_t(r) * gp + j];
#pragma unroll
        for (int k = 0; k < KMAX; ++k)
            if (k < nrhs) {
                const double2 t = T[int64_t(k) * nb + j];
                acc[k].x = fma(g.x, t.x, acc[k].x);
                acc[k].y = fma(g.x, t.y, acc[k].y);
                acc[k].x = fma(-g.y, t.y, acc[k].x);
                acc[k].y = fma(g.y, t.x, acc[k].y);
            }
    }
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
        for (int o = 16; o > 0; o >>= 1) {
            acc[k].x += __shfl_xor_sync(0xffffffffu, acc[k].x, o);
            acc[k].y += __shfl_xor_sync(0xffffffffu, acc[k].y, o);
        }
        if (lane == 0 && k < nrhs) X[int64_t(k) * nb + r] = acc[k];
    }
}

struct WarpPlan {
    WSweepArgs a;
    int CS = 0, KG = 0, KR = 0;
    bool even = false;  // every lane owns a row and an equal multiple-of-4 column count
    size_t smem = 0;
    double est = 0;
};

bool warp_layout(int nb, int L, int gp, int nrhs, int CS, int KG, int KR, WarpPlan& p) {
    const int R = (nb + CS - 1) / CS;
    if (R > 32) return false;
    int Rp = 1;
    while (Rp < R) Rp <<= 1;
    WSweepArgs& a = p.a;
    a = WSweepArgs{};
    a.L = L;
    a.chain[0].first = 0;
    a.chain[0].count = L;
    a.chain[0].dir = 1;
    a.chain[0].mode = 0;
    a.chain[1].count = 0;
    a.nb = nb;
    a.nrhs = nrhs;
    a.gp = gp;
    a.R = R;
    a.Rp = Rp;
    const size_t gbytes = size_t(R) * gp * sizeof(double2);
    a.off_e = al128(gbytes);
    a.off_b = a.off_e + al128(size_t(R) * sizeof(double2));
    a.stage_bytes = a.off_b + al128(size_t(KG) * nb * sizeof(double2));
    const size_t yb = al128(size_t(2) * KG * (nb + 1) * sizeof(double2));
    const size_t wb = 0;  // w is formed in registers
    const char* ns = std::getenv("FWI_EXACT_STAGES");
    a.nst = ns ? std::max(2, std::min(kWMaxStages, std::atoi(ns))) : kWMaxStages;
    while (a.nst & (a.nst - 1)) --a.nst;  // power of two: the kernel masks the step index
    while (a.nst > 2 && size_t(a.nst) * a.stage_bytes + yb + wb + 512 > 220 * 1024) a.nst /= 2;
    a.off_y = a.nst * a.stage_bytes;
    a.off_w = a.off_y + yb;
    a.off_bar = a.off_w + wb;
    p.smem = a.off_bar + 512;
    p.CS = CS;
    p.KG = KG;
    p.KR = KR;
    p.even = (R == Rp) && (nb % CS == 0) && (nb % (4 * (32 / Rp)) == 0);
    return p.smem <= 220 * 1024;
}

template <int CS, int KG, int KR, bool TRACE, bool EVEN>
bool warp_prepare(const WarpPlan& p, int* max_clusters) {
    auto kern = sweep_warp_kernel<CS, KG, KR, TRACE, EVEN>;
    static size_t set = 0;
    if (p.smem > set) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(p.smem)) != cudaSuccess)
            return false;
        if (CS > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
            return false;
        set = p.smem;
    }
    if (max_clusters) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(CS);
        cfg.blockDim = dim3((KG / KR + 1) * 32);
        cfg.dynamicSmemBytes = p.smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CS;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n < 1) {
            cudaGetLastError();
            return false;
        }
        *max_clusters = n;
    }
    return true;
}

template <int CS, int KG, int KR, bool TRACE, bool EVEN>
bool warp_launch(const WarpPlan& p, int nrhs, cudaStream_t st) {
    if (!warp_prepare<CS, KG, KR, TRACE, EVEN>(p, nullptr)) return false;
    const int groups = (nrhs + KG - 1) / KG;
    const int chains = p.a.chain[1].count > 0 ? 2 : 1;
    WSweepArgs args = p.a;
    args.groups0 = groups;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(chains * groups * CS);
    cfg.blockDim = dim3((KG / KR + 1) * 32);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // pdl_enter() in the kernel
    attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    CK(cudaLaunchKernelEx(&cfg, sweep_warp_kernel<CS, KG, KR, TRACE, EVEN>, args));
    return true;
}

#define FWI_WARP_VARIANTS(X)                                                                      \
    X(16, 8, 2) X(16, 8, 1) X(16, 6, 1) X(16, 4, 2) X(16, 4, 1) X(16, 2, 1) X(16, 1, 1) X(8, 8, 2) X(8, 8, 1) \
    X(8, 4, 2) X(8, 2, 1) X(8, 1, 1)

bool warp_dispatch_prepare(const WarpPlan& p, int* maxc) {
#define X(cs, kg, kr) \
    if (p.CS == cs && p.KG == kg && p.KR == kr)                                          \
        return p.even ? warp_prepare<cs, kg, kr, false, true>(p, maxc) : warp_prepare<cs, kg, kr, false, false>(p, maxc);
    FWI_WARP_VARIANTS(X)
#undef X
    return false;
}

bool warp_dispatch_launch(const WarpPlan& p, int nrhs, cudaStream_t st) {
#define X(cs, kg, kr) \
    if (p.CS == cs && p.KG == kg && p.KR == kr)                     \
        return !p.even ? warp_launch<cs, kg, kr, false, false>(p, nrhs, st)                         \
                       : (p.a.trace ? warp_launch<cs, kg, kr, true, true>(p, nrhs, st)                   \
                                    : warp_launch<cs, kg, kr, false, true>(p, nrhs, st));
    FWI_WARP_VARIANTS(X)
#undef X
    return false;
}

// Pick (CS, KG, KR) by a model of one line step, fitted to clock64 traces of the
// kernel on B200 (tools/sweep_trace.py, tools/sweep_grid.sh): a consumer warp's step
// is bound by its dependent instruction stream, ~1400 cycles of fixed work (barrier
// wake-ups, butterfly, pushes, DSMEM flight) plus ~35 cycles per column element per
// RHS it owns, plus ~4.5 cycles per element for every consumer warp beyond two that
// shares the SM; clusters beyond the resident limit run in further waves.
bool warp_plan(int nb, int L, int gp, int nrhs, WarpPlan& best, int chains = 1, int steps = -1) {
    if (steps < 0) steps = 2 * L - 1;
    const char* ecs = std::getenv("FWI_EXACT_CS");
    const char* ekg = std::getenv("FWI_EXACT_KG");
    const char* ekr = std::getenv("FWI_EXACT_KR");
    const int want_cs = ecs ? std::atoi(ecs) : 0, want_kg = ekg ? std::atoi(ekg) : 0, want_kr = ekr ? std::atoi(ekr) : 0;
    bool found = false;
    struct V {
        int cs, kg, kr;
    };
    static const V variants[] = {
#define X(cs, kg, kr) {cs, kg, kr},
        FWI_WARP_VARIANTS(X)
#undef X
    };
    for (const V& v : variants) {
        const int cs = v.cs, kg = v.kg, kr = v.kr;
        if (true) {
            if ((want_cs && cs != want_cs) || (want_kg && kg != want_kg) || (want_kr && kr != want_kr)) continue;
            WarpPlan p;
            if (!warp_layout(nb, L, gp, nrhs, cs, kg, kr, p)) continue;
            int maxc = 0;
            if (!warp_dispatch_prepare(p, &maxc)) continue;
            const int groups = chains * ((nrhs + kg - 1) / kg);
            const int waves = (groups + maxc - 1) / maxc;
            const int ncls = 32 / p.a.Rp;
            const double per_lane = double((nb + ncls - 1) / ncls);
            const int nw = kg / kr;
            p.est = double(waves) * double(steps) *
                    (1400.0 + 35.0 * per_lane * kr + 4.5 * per_lane * kr * std::max(0, nw - 2));
            if (!found || p.est < best.est - 1e-9) {
                best = p;
                found = true;
            }
        }
    }
    return found;
}

struct ClusterPlan {
    bool ok = false;
    int KG = 0, CS = 0, R = 0, nseg = 0;
    SweepArgs a{};
    size_t smem = 0;
};

template <int KG, int CS>
bool cluster_launch(const ClusterPlan& cp, int nrhs, cudaStream_t st) {
    static size_t set = 0;
    if (cp.smem > set) {
        if (cudaFuncSetAttribute(sweep_cluster_kernel<KG, CS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(cp.smem)) != cudaSuccess)
            return false;
        if (CS > 8 && cudaFuncSetAttribute(sweep_cluster_kernel<KG, CS>,
                                           cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
            return false;
        set = cp.smem;
    }
    const int groups = (nrhs + KG - 1) / KG;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(groups * CS);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = cp.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SweepArgs a = cp.a;
    a.nrhs = nrhs;
    CK(cudaLaunchKernelEx(&cfg, sweep_cluster_kernel<KG, CS>, a));
    return true;
}

// pick (KG, CS) whose shared-memory footprint fits; nb <= 256 only
bool cluster_plan(int nb, int L, int gp, int nrhs, ClusterPlan& cp) {
    const int cands[][2] = {{8, 8}, {4, 8}, {8, 16}, {4, 16}, {2, 16}, {1, 16}};
    for (const auto& c : cands) {
        const int KG = c[0], CS = c[1];
        if (KG > 1 && nrhs < KG && KG != 8) continue;
        const int R = (nb + CS - 1) / CS;
        const int O = R * KG;
        const int nseg = std::max(1, std::min(8, 256 / std::max(O, 1)));
        SweepArgs a{};
        a.L = L;
        a.nb = nb;
        a.gp = gp;
        a.R = R;
        a.nseg = nseg;
        const size_t gbytes = size_t(R) * gp * sizeof(double2);
        a.off_e = al128(gbytes);
        a.off_b = a.off_e + al128(size_t(nb) * sizeof(double2));
        a.stage_bytes = a.off_b + al128(size_t(KG) * nb * sizeof(double2));
        const size_t rest = al128(size_t(2) * KG * (nb + 1) * sizeof(double2)) +
                            al128(size_t(KG) * (nb + 1) * sizeof(double2)) +
                            al128(size_t(nseg) * O * sizeof(double2)) + 128;
        a.nst = 4;
        while (a.nst > 2 && size_t(a.nst) * a.stage_bytes + rest > 220 * 1024) --a.nst;
        a.off_y = a.nst * a.stage_bytes;
        a.off_w = a.off_y + al128(size_t(2) * KG * (nb + 1) * sizeof(double2));
        a.off_part = a.off_w + al128(size_t(KG) * (nb + 1) * sizeof(double2));
        a.off_bar = a.off_part + al128(size_t(nseg) * O * sizeof(double2));
        const size_t smem = a.off_bar + 128;
        if (smem <= 220 * 1024) {
            cp.ok = true;
            cp.KG = KG;
            cp.CS = CS;
            cp.R = R;
            cp.nseg = nseg;
            cp.a = a;
            cp.smem = smem;
            return true;
        }
    }
    return false;
}

constexpr int kSweepKG = 2;

size_t sweep_smem(int nb) {
    const int S = nb <= 256 ? 256 / nb : 1;
    return size_t(2 * kSweepKG * nb + S * kSweepKG * nb) * sizeof(double2);
}

}  // namespace

// cyclic reduction for nb-node lines, L of them (FWI_EXACT_BCR=1|0 forces it on or off)
static bool bcr_wanted(bool line_pivot, int nb, int L) {
    const char* eb = std::getenv("FWI_EXACT_BCR");
    return !line_pivot && nb <= 512 && L >= 2 && (eb ? std::string(eb) == "1" : (L >= kBcrMinLines && nb >= 32));
}

// line_pivot: factor every line with the one-CTA Gauss-Jordan, partial pivoting over the
// whole line (the fallback when the residual probe rejects the block Gauss-Jordan, whose
// pivot search is restricted to 64-wide diagonal blocks)
static void exact_factor_once(Ctx& c, bool line_pivot) {
    const auto t_host0 = std::chrono::steady_clock::now();
    auto f = std::make_unique<ExactFactor>();
    f->col_lines = c.nz <= c.nx;  // short lines by default (least factor work and storage)
    // A line step is latency-bound (fixed dependent chain + work per column), so
    // fewer, longer lines can sweep faster: take the long-line orientation when the
    // sweep model says so (config 1: 64 lines of 128 instead of 128 lines of 64).
    {
        const int nbs = std::min(c.nx, c.nz), nbl = std::max(c.nx, c.nz);
        const char* eo = std::getenv("FWI_EXACT_LINES");  // "short" | "long" (diagnostics)
        const std::string o = eo ? eo : "";
        WarpPlan ps, pl;
        if (o == "long" && nbl <= 512) {
            f->col_lines = !f->col_lines;
        } else if (o.empty() && nbl <= 512 && nbs != nbl && !bcr_wanted(line_pivot, nbs, nbl) &&
                   warp_plan(nbs, nbl, nbs + 1, c.K, ps) && warp_plan(nbl, nbs, nbl + 1, c.K, pl) &&
                   pl.est < 0.9 * ps.est) {
            f->col_lines = !f->col_lines;
        }
    }
    f->nb = f->col_lines ? c.nz : c.nx;
    f->L = f->col_lines ? c.nx : c.nz;
    const int nb = f->nb, L = f->L;
    require(nb <= 2048, "exact block factorisation: line length above 2048 is not supported");
    f->gp = nb + 1;
    f->coup.alloc(size_t(L) * nb);
    f->status.alloc(1);
    CK(cudaMemsetAsync(f->status.p, 0, sizeof(int), c.stream));
    extract_lines<<<grid_blocks(int64_t(L) * nb, 256, 1 << 20), 256, 0, c.stream>>>(
        f->col_lines, c.nx, L, nb, c.east.p, c.south.p, f->coup.p);
    CK_LAUNCH();
    // Block cyclic reduction (bcr.cu) when the line chain is long: a Schur sweep is 2L
    // latency-bound line steps, cyclic reduction log2 L levels of batched tensor-core GEMMs.
    // FWI_EXACT_BCR=1|0 forces it on or off (diagnostics).
    {
        if (bcr_wanted(line_pivot, nb, L)) f->bcr = bcr_factor(c, f->col_lines, nb, L, f->coup.p, f->status.p);
    }
    if (!f->bcr) {
    f->G.alloc(size_t(L) * nb * f->gp);
    // Sweeps: GEMM per line beyond the cluster kernel's reach (nb > 512). Factor: the
    // whole-GPU block Gauss-Jordan whenever a line does not fit one CTA's shared memory
    // (nb > 112; ~8x faster than the one-CTA global-memory Gauss-Jordan at nb = 128).
    // FWI_EXACT_DENSE=1 forces both; FWI_EXACT_FACTOR=cta keeps the one-CTA factor.
    const bool force_dense = std::getenv("FWI_EXACT_DENSE") != nullptr;
    const char* ef = std::getenv("FWI_EXACT_FACTOR");
    f->dense = nb > 512 || force_dense;
    f->dense_factor = f->dense || (nb > 112 && !(ef && std::string(ef) == "cta"));
    if (line_pivot && !f->dense) f->dense_factor = false;
    if (!line_pivot && !f->dense && std::getenv("FWI_EXACT_TWISTED") &&
        std::string(std::getenv("FWI_EXACT_TWISTED")) == "1")
        f->dense_factor = true;  // the twisted factorisation is built with the block Gauss-Jordan
    // Twisted factorisation: Schur recursions from both ends meet at the middle line,
    // so a solve is two concurrent sweep chains of ~L/2 lines each (then a dense
    // solve of the middle line) instead of one chain of L: a line step is latency-
    // bound, so this halves the sweep. Used when the step model says it pays.
    if (f->dense_factor && L >= 8) {
        const char* et = line_pivot ? nullptr : std::getenv("FWI_EXACT_TWISTED");
        if (et) {
            f->twisted = std::string(et) == "1";
        } else if (f->dense) {
            // GEMM sweeps: two concurrent chains fill the GPU (one C5 step GEMM has 128 tiles)
            f->twisted = true;
        } else {
            WarpPlan p1, p2;
            const int m = L / 2;
            const int steps2 = 2 * std::max(m, L - 1 - m);
            f->twisted = warp_plan(nb, L, nb + 1, c.K, p1) && warp_plan(nb, L, nb + 1, c.K, p2, 2, steps2) &&
                         p2.est + 40000.0 < 0.9 * p1.est;
        }
    }
    if (f->dense_factor) {
        const int64_t nn = int64_t(nb) * nb;
        auto Gl = [&](int i) { return f->G.p + i * int64_t(nb) * f->gp; };
        auto cl = [&](int i) { return f->coup.p + int64_t(i) * nb; };  // coupling of lines i, i+1
        auto line = [&](cudaStream_t st, DenseWork& dw, int i, const double2* cA, const double2* GA,
                        const double2* cB, const double2* GB) {
            form_schur<<<int((nn + 255) / 256), 256, 0, st>>>(f->col_lines, c.nx, nb, i, c.diag.p, c.east.p,
                                                              c.south.p, cA, GA, cB, GB, f->gp, Gl(i));
            CK_LAUNCH();
            dense_invert(st, nb, Gl(i), f->gp, dw, f->status.p, i * nb);
        };
        if (!f->twisted) {
            for (int i = 0; i < L; ++i)
                line(c.stream, f->dwork, i, i > 0 ? cl(i - 1) : nullptr, i > 0 ? Gl(i - 1) : nullptr, nullptr, nullptr);
        } else {
            // the two recursions are independent: top chain on the context stream, bottom
            // chain on the factor's second stream, then the middle line
            const int m = L / 2;
            f->mid = m;
            f->ensure_side();
            CK(cudaEventRecord(f->ev_fork, c.stream));
            CK(cudaStreamWaitEvent(f->s2, f->ev_fork, 0));
            // launches alternate between the chains: the launch queue fills up, so
            // enqueueing one whole chain first would serialise them
            for (int r = 0; r < std::max(m, L - 1 - m); ++r) {
                if (r < m)
                    line(c.stream, f->dwork, r, r > 0 ? cl(r - 1) : nullptr, r > 0 ? Gl(r - 1) : nullptr, nullptr,
                         nullptr);
                const int i = L - 1 - r;
                if (i > m)
                    line(f->s2, f->dwork2, i, i < L - 1 ? cl(i) : nullptr, i < L - 1 ? Gl(i + 1) : nullptr, nullptr,
                         nullptr);
            }
            CK(cudaEventRecord(f->ev_join, f->s2));
            CK(cudaStreamWaitEvent(c.stream, f->ev_join, 0));
            line(c.stream, f->dwork, m, cl(m - 1), Gl(m - 1), cl(m), Gl(m + 1));
        }
    } else {
    const bool smem = nb <= 112;
    const size_t base = size_t(2 * nb) * sizeof(double2) + size_t((nb + 3) & ~3) * sizeof(int);
    const size_t shm = base + (smem ? size_t(nb) * nb * sizeof(double2) : 0);
    if (!smem) f->work.alloc(size_t(nb) * nb);
    const int threads = nb <= 64 ? 256 : 512;
    if (smem)
        CK(cudaFuncSetAttribute(line_factor_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm)));
    else
        CK(cudaFuncSetAttribute(line_factor_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm)));
    for (int i = 0; i < L; ++i) {
        const double2* prev = i > 0 ? f->G.p + (i - 1) * int64_t(nb) * f->gp : nullptr;
        if (smem)
            line_factor_kernel<true><<<1, threads, shm, c.stream>>>(
                f->col_lines, c.nx, nb, i, c.diag.p, c.east.p, c.south.p, f->coup.p, prev,
                f->G.p + i * int64_t(nb) * f->gp, f->gp, nullptr, f->status.p);
        else
            line_factor_kernel<false><<<1, threads, shm, c.stream>>>(
                f->col_lines, c.nx, nb, i, c.diag.p, c.east.p, c.south.p, f->coup.p, prev,
                f->G.p + i * int64_t(nb) * f->gp, f->gp, f->work.p, f->status.p);
        CK_LAUNCH();
    }
    }
    }  // !f->bcr
    int st = 0;
    CK(cudaMemcpyAsync(&st, f->status.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    if (std::getenv("FWI_EXACT_PLAN_LOG"))
        std::fprintf(stderr, "[fwi] exact factor nb=%d L=%d dense=%d twisted=%d bcr=%d: %.3f s\n", nb, L,
                     int(f->dense), int(f->twisted), int(f->bcr != nullptr),
                     std::chrono::duration<double>(std::chrono::steady_clock::now() - t_host0).count());
    if (st != 0) {
        // status = line * nb + (position in the line) + 1. Reported as the grid node, the
        // reference's elimination-column numbering (natural order, src/lu.cpp:113); which node
        // of a singular operator meets the zero pivot first depends on the elimination order,
        // and for a zero row (tests/test_lu.cpp:44-47) both name that row.
        const int line = (st - 1) / nb, m = (st - 1) % nb;
        const int node = f->col_lines ? m * c.nx + line : line * c.nx + m;
        throw FwiError(FWI_ERR_SINGULAR_PIVOT,
                       "LU: singular pivot at node " + std::to_string(node) + " (exact block factorisation, line " +
                           std::to_string(line) + ")",
                       node);
    }
    if (c.exact) exact_free(c.exact);
    c.exact = f.release();
}

namespace {
// r = b - A x with the assembled 5-point planes (A(i,i-1) = east[i-1], A(i,i-nx) =
// south[i-nx]: exact complex symmetry)
__global__ void stencil_residual(int nx, int64_t n, const double2* __restrict__ diag,
                                 const double2* __restrict__ east, const double2* __restrict__ south,
                                 const double2* __restrict__ x, const double2* __restrict__ b,
                                 double2* __restrict__ r) {
    const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    double2 acc = fmul(diag[i], x[i]);
    auto add = [&](double2 a, double2 v) {
        const double2 t = fmul(a, v);
        acc.x += t.x;
        acc.y += t.y;
    };
    if (i + 1 < n) add(east[i], x[i + 1]);
    if (i >= 1) add(east[i - 1], x[i - 1]);
    if (i + nx < n) add(south[i], x[i + nx]);
    if (i >= nx) add(south[i - nx], x[i - nx]);
    r[i] = make_double2(b[i].x - acc.x, b[i].y - acc.y);
}
}  // namespace

double exact_probe_residual(const ExactFactor* f) { return f ? f->probe_residual : -1.0; }

// ||b - A A^{-1} b|| / ||b|| for one seeded random right-hand side
double exact_residual_probe(Ctx& c) {
    std::vector<double2> hb(size_t(c.n));
    uint64_t z = 0x9e3779b97f4a7c15ull;
    auto rnd = [&] {  // splitmix64 -> [-1, 1)
        z += 0x9e3779b97f4a7c15ull;
        uint64_t t = z;
        t = (t ^ (t >> 30)) * 0xbf58476d1ce4e5b9ull;
        t = (t ^ (t >> 27)) * 0x94d049bb133111ebull;
        t ^= t >> 31;
        return double(t >> 11) * (2.0 / 9007199254740992.0) - 1.0;
    };
    for (auto& v : hb) v = make_double2(rnd(), rnd());
    DevBuf<double2> b(c.n), x(c.n), r(c.n);
    CK(cudaMemcpyAsync(b.p, hb.data(), b.bytes(), cudaMemcpyHostToDevice, c.stream));
    const int64_t cnt = c.solve_count[FWI_PRECOND_EXACT];
    exact_solve_batch(c, false, b.p, x.p, 1);
    c.solve_count[FWI_PRECOND_EXACT] = cnt;  // not a caller's solve
    stencil_residual<<<int((c.n + 255) / 256), 256, 0, c.stream>>>(c.nx, c.n, c.diag.p, c.east.p, c.south.p, x.p,
                                                                   b.p, r.p);
    CK_LAUNCH();
    const double rr = dev_dot(&c, c.stream, reinterpret_cast<const double*>(r.p),
                              reinterpret_cast<const double*>(r.p), 2 * int64_t(c.n));
    const double bb = dev_dot(&c, c.stream, reinterpret_cast<const double*>(b.p),
                              reinterpret_cast<const double*>(b.p), 2 * int64_t(c.n));
    return std::sqrt(rr / bb);
}

// The exact factorisation with a residual guard. The block
// factorisations pivot within a line, or within 64-wide diagonal blocks of a line (the
// block Gauss-Jordan, nb > 112), never across lines as the reference's sparse LU does
// (src/lu.cpp:56-133). One seeded right-hand side is solved after every factorisation;
// above kProbeTol the lines are re-factored with partial pivoting over each whole line
// (nb <= 512), and if that also fails, or for longer lines, SingularPivotError is raised
// rather than returning an inaccurate factor. FWI_EXACT_PROBE=0 skips the probe.
void exact_factor(Ctx& c) {
    constexpr double kProbeTol = 1e-8;
    exact_factor_once(c, false);
    const char* ep = std::getenv("FWI_EXACT_PROBE");
    if (ep && std::string(ep) == "0") return;
    double res = exact_residual_probe(c);
    c.exact->probe_residual = res;
    if (!(res <= kProbeTol) && c.exact->nb <= 512 && c.exact->dense_factor) {
        exact_factor_once(c, true);
        res = exact_residual_probe(c);
        c.exact->probe_residual = res;
        c.exact->refactored = true;
    }
    if (std::getenv("FWI_EXACT_PLAN_LOG"))
        std::fprintf(stderr, "[fwi] exact factor residual probe %.3e%s\n", res,
                     c.exact->refactored ? " (after whole-line pivoting)" : "");
    if (!(res <= kProbeTol)) {
        char buf[160];
        std::snprintf(buf, sizeof buf,
                      "LU: exact block factorisation failed its residual probe (||b - A x|| / ||b|| = %.3e)", res);
        exact_free(c.exact);
        c.exact = nullptr;
        throw FwiError(FWI_ERR_SINGULAR_PIVOT, buf, -1);
    }
}

void exact_solve_batch(Ctx& c, bool adjoint, const double2* b, double2* x, int nrhs) {
    require(c.exact != nullptr, "precond_apply: state has no exact factorization");
    const ExactFactor& f = *c.exact;
    c.ensure_work(Ctx::kWorkC);
    DevBuf<double2> tmp;  // only for batches larger than K (freed synchronously)
    double2* W = c.work_c.p;
    if (size_t(nrhs) * c.n > c.work_c.count) {
        tmp.alloc(size_t(nrhs) * c.n);
        W = tmp.p;
    }
    // the attribute is per kernel (process-wide): only ever raise it
    static size_t smem_set = 0;
    if (sweep_smem(f.nb) > smem_set) {
        CK(cudaFuncSetAttribute(sweep_kernel<kSweepKG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(sweep_smem(f.nb))));
        smem_set = sweep_smem(f.nb);
    }
    dim3 tb(32, 8);
    dim3 tg = f.col_lines ? dim3((f.L + 31) / 32, (f.nb + 31) / 32, nrhs)
                          : dim3((f.nb + 31) / 32, (f.L + 31) / 32, nrhs);
    launch_pdl<kPdlExact>(gather_lines, dim3(tg), dim3(tb), 0, c.stream, f.col_lines, c.nx, c.nz, f.L, f.nb, nrhs,
                          adjoint, b, W);
    CK_LAUNCH();
    bool done = false;
    if (f.bcr) {
        bcr_solve(c, *f.bcr, f.coup.p, W, nrhs);
        done = true;
    }
    if (!done && f.dense) {
        ExactFactor& fm = const_cast<ExactFactor&>(f);
        if (fm.tbuf.count < size_t(nrhs) * f.nb) fm.tbuf.alloc(size_t(nrhs) * f.nb);
        if (f.twisted) {
            if (fm.tbuf2.count < size_t(nrhs) * f.nb) fm.tbuf2.alloc(size_t(nrhs) * f.nb);
            dense_sweep_twisted(c.stream, fm.s2, fm.ev_fork, fm.ev_join, f.L, f.mid, f.nb, nrhs, f.G.p, f.gp,
                                f.coup.p, W, fm.tbuf.p, fm.tbuf2.p);
        } else {
            dense_sweep(c.stream, f.L, f.nb, nrhs, f.G.p, f.gp, f.coup.p, W, fm.tbuf.p);
        }
        done = true;
    }
    const char* sw = std::getenv("FWI_EXACT_SWEEP");  // "warp" (default) | "cta" | "legacy"
    if (done) sw = "none";
    const std::string sweep = sw ? sw : "warp";
    if (!done && sweep == "warp") {
        // plans are cached per (nb, L, nrhs) (the model queries cluster occupancy);
        // process-wide, so guarded for contexts driven from several host threads
        static std::mutex mu;
        static std::vector<std::pair<std::array<int, 4>, WarpPlan>> cache;
        const bool forced = std::getenv("FWI_EXACT_CS") || std::getenv("FWI_EXACT_KG") || std::getenv("FWI_EXACT_KR");
        const std::array<int, 4> key{f.nb, f.L, nrhs, f.twisted ? 1 : 0};
        const int m = f.mid;
        const int chains = f.twisted ? 2 : 1;
        const int steps = f.twisted ? 2 * std::max(m, f.L - 1 - m) : 2 * f.L - 1;
        bool have = false;
        WarpPlan plan;
        {
            std::lock_guard<std::mutex> lk(mu);
            for (auto& e : cache)
                if (e.first == key && !forced) {
                    plan = e.second;
                    have = true;
                }
            if (!have && warp_plan(f.nb, f.L, f.gp, nrhs, plan, chains, steps)) {
                if (!forced) cache.emplace_back(key, plan);
                have = true;
                if (std::getenv("FWI_EXACT_PLAN_LOG"))
                    std::fprintf(stderr, "[fwi] exact plan nb=%d L=%d nrhs=%d twisted=%d: CS=%d KG=%d KR=%d est=%.0f\n",
                                 f.nb, f.L, nrhs, int(f.twisted), plan.CS, plan.KG, plan.KR, plan.est);
            }
        }
        if (have) {
            WarpPlan p = plan;
            p.a.G = f.G.p;
            p.a.coup = f.coup.p;
            p.a.W = W;
            if (f.ybuf.count < size_t(nrhs) * c.n) const_cast<ExactFactor&>(f).ybuf.alloc(size_t(nrhs) * c.n);
            p.a.Y = f.ybuf.p;
            const char* tpath = std::getenv("FWI_SWEEP_TRACE");  // diagnostics only
            DevBuf<unsigned long long> tbuf;
            if (tpath) {
                tbuf.alloc(size_t(8) * (2 * f.L - 1));
                CK(cudaMemsetAsync(tbuf.p, 0, tbuf.count * 8, c.stream));
                p.a.trace = tbuf.p;
            }
            if (!f.twisted) {
                done = warp_dispatch_launch(p, nrhs, c.stream);
            } else {
                // (1) both halves forward, concurrently: y_i for lines 0..m-1 and L-1..m+1
                p.a.trace = nullptr;
                p.a.chain[0] = SweepChain{0, m, 1, 1, nullptr};
                p.a.chain[1] = SweepChain{f.L - 1, f.L - 1 - m, -1, 1, nullptr};
                done = warp_dispatch_launch(p, nrhs, c.stream);
                if (done) {
                    // (2) middle line: x_m = G_m (b_m - E_{m-1} y_{m-1} - E_m y_{m+1})
                    ExactFactor& fm = const_cast<ExactFactor&>(f);
                    if (fm.tbuf.count < size_t(nrhs) * f.nb) fm.tbuf.alloc(size_t(nrhs) * f.nb);
                    const int64_t blk = int64_t(nrhs) * f.nb;
                    launch_pdl<kPdlExact>(middle_rhs, dim3(int((blk + 255) / 256)), dim3(256), 0, c.stream, f.nb, blk,
                                          W + m * blk, f.coup.p + int64_t(m - 1) * f.nb, f.ybuf.p + (m - 1) * blk,
                                          f.coup.p + int64_t(m) * f.nb, f.ybuf.p + (m + 1) * blk, fm.tbuf.p);
                    CK_LAUNCH();
                    const double2* Gm = f.G.p + int64_t(m) * f.nb * f.gp;
                    if (nrhs <= 8) {
                        launch_pdl<kPdlExact>(middle_gemv<8>, dim3((f.nb + 7) / 8), dim3(256), 0, c.stream, f.nb, nrhs,
                                              Gm, f.gp, fm.tbuf.p, W + m * blk);
                        CK_LAUNCH();
                    } else {
                        cgemm(c.stream, true, nrhs, f.nb, f.nb, 1.0, fm.tbuf.p, f.nb, Gm, f.gp, nullptr, 0, W + m * blk,
                              f.nb);
                    }
                    // (3) both halves backward from the middle line outwards
                    p.a.chain[0] = SweepChain{m - 1, m, -1, 2, W + m * blk};
                    p.a.chain[1] = SweepChain{m + 1, f.L - 1 - m, 1, 2, W + m * blk};
                    done = warp_dispatch_launch(p, nrhs, c.stream);
                    if (!done) throw FwiError(FWI_ERR_CUDA, "exact solve: twisted backward sweep could not launch");
                }
            }
            if (tpath && done && !f.twisted) {
                std::vector<unsigned long long> h(tbuf.count);
                CK(cudaMemcpyAsync(h.data(), tbuf.p, tbuf.count * 8, cudaMemcpyDeviceToHost, c.stream));
                CK(cudaStreamSynchronize(c.stream));
                if (FILE* fp = std::fopen(tpath, "ab")) {
                    std::fwrite(h.data(), 8, h.size(), fp);
                    std::fclose(fp);
                }
                std::fprintf(stderr, "[fwi] exact sweep plan CS=%d KG=%d KR=%d nst=%d smem=%zu est=%.0f\n", p.CS,
                             p.KG, p.KR, p.a.nst, p.smem, p.est);
            }
        }
    }
    if (!done && sweep != "legacy" && sweep != "none") {
        ClusterPlan cp;
        if (cluster_plan(f.nb, f.L, f.gp, nrhs, cp)) {
            cp.a.G = f.G.p;
            cp.a.coup = f.coup.p;
            cp.a.W = W;
            if (f.ybuf.count < size_t(nrhs) * c.n) const_cast<ExactFactor&>(f).ybuf.alloc(size_t(nrhs) * c.n);
            cp.a.Y = f.ybuf.p;
            switch (cp.KG * 100 + cp.CS) {
                case 808: done = cluster_launch<8, 8>(cp, nrhs, c.stream); break;
                case 408: done = cluster_launch<4, 8>(cp, nrhs, c.stream); break;
                case 816: done = cluster_launch<8, 16>(cp, nrhs, c.stream); break;
                case 416: done = cluster_launch<4, 16>(cp, nrhs, c.stream); break;
                case 216: done = cluster_launch<2, 16>(cp, nrhs, c.stream); break;
                case 116: done = cluster_launch<1, 16>(cp, nrhs, c.stream); break;
                default: break;
            }
        }
    }
    if (!done && sweep != "none") {
        sweep_kernel<kSweepKG><<<(nrhs + kSweepKG - 1) / kSweepKG, 256, sweep_smem(f.nb), c.stream>>>(
            f.L, f.nb, nrhs, f.G.p, f.gp, f.coup.p, W);
        CK_LAUNCH();
    }
    launch_pdl<kPdlExact>(scatter_lines, dim3(tg), dim3(tb), 0, c.stream, f.col_lines, c.nx, c.nz, f.L, f.nb, nrhs,
                          adjoint, W, x);
    CK_LAUNCH();
    c.solve_count[FWI_PRECOND_EXACT] += nrhs;
}

}  // namespace fwi_b200
