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

#include "ctx.cuh"

namespace fwi_b200 {

struct ExactFactor {
    int L = 0, nb = 0;
    bool col_lines = true;  // lines are grid columns (fixed ix) when nz <= nx
    DevBuf<double2> GT;     // L x nb x nb, GT[i][j][m] = G_i[m][j]
    DevBuf<double2> coup;   // L x nb, coupling line i -> i+1 at position m
    DevBuf<double2> work;   // nb x nb scratch (global-memory inversion)
    DevBuf<int> status;
};

void exact_free(ExactFactor* f) { delete f; }
int64_t exact_bytes(const ExactFactor* f) { return f ? int64_t(f->GT.bytes() + f->coup.bytes()) : 0; }

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

// Form S_i (row-major, in A) from the line's tridiagonal block and G_{i-1},
// then invert it in place by Gauss-Jordan with partial pivoting and write
// G_i transposed into GT_i. A lives in shared memory (small nb) or in a
// global scratch (large nb). One CTA per line; lines are launched in order.
template <bool SMEM>
__global__ void __launch_bounds__(512) line_factor_kernel(
    bool col_lines, int nx, int nb, int line, const double2* __restrict__ diag,
    const double2* __restrict__ east, const double2* __restrict__ south,
    const double2* __restrict__ coup, const double2* __restrict__ GTprev, double2* __restrict__ GTout,
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
    const int64_t nn = int64_t(nb) * nb;

    // ---- S_i = T_i - E_{i-1} G_{i-1} E_{i-1}
    for (int64_t t = tid; t < nn; t += nt) {
        const int a = int(t / nb), b = int(t % nb);
        double2 v = make_double2(0.0, 0.0);
        const int64_t na = line_node(col_lines, nx, line, a);
        if (a == b) v = diag[na];
        else if (b == a + 1) v = col_lines ? south[na] : east[na];
        else if (a == b + 1) v = col_lines ? south[line_node(col_lines, nx, line, b)]
                                           : east[line_node(col_lines, nx, line, b)];
        if (line > 0) {
            const double2 ea = coup[int64_t(line - 1) * nb + a], eb = coup[int64_t(line - 1) * nb + b];
            const double2 g = GTprev[int64_t(b) * nb + a];  // G_{i-1}[a][b]
            const double2 t2 = fmul(fmul(ea, g), eb);
            v.x -= t2.x;
            v.y -= t2.y;
        }
        A[t] = v;
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
                if (*status == 0) *status = line * nb + k + 1;
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
        for (int64_t t = tid; t < nn; t += nt) {
            const int r = int(t / nb), j = int(t % nb);
            if (r == k) continue;
            const double2 f = pcol[r];
            double2 v = (j == k) ? make_double2(0.0, 0.0) : A[t];
            const double2 pr = prow[j];
            v.x -= f.x * pr.x - f.y * pr.y;
            v.y -= f.x * pr.y + f.y * pr.x;
            A[t] = v;
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
    // GT[j][m] = G[m][j]
    for (int64_t t = tid; t < nn; t += nt) {
        const int m = int(t / nb), j = int(t % nb);
        GTout[int64_t(j) * nb + m] = A[t];
    }
}

// source-major b_k[node]  ->  line-major W[i][k][m] (optionally conjugated)
// and back. A 32x32 tile transpose in shared memory keeps both sides
// coalesced for column lines; row lines are a plain strided copy.
__global__ void gather_lines(bool col_lines, int nx, int nz, int L, int nb, int nrhs, bool conj,
                             const double2* __restrict__ src, double2* __restrict__ W) {
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
                                                    const double2* __restrict__ GT,
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
    const int64_t nn = int64_t(nb) * nb;

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
                const double2 g = __ldg(G + int64_t(j) * nb + m0);
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
        matvec(GT + int64_t(i) * nn, false, i);
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
        matvec(GT + int64_t(i) * nn, true, i);
    }
}

constexpr int kSweepKG = 2;

size_t sweep_smem(int nb) {
    const int S = nb <= 256 ? 256 / nb : 1;
    return size_t(2 * kSweepKG * nb + S * kSweepKG * nb) * sizeof(double2);
}

}  // namespace

void exact_factor(Ctx& c) {
    auto f = std::make_unique<ExactFactor>();
    f->col_lines = c.nz <= c.nx;
    f->nb = f->col_lines ? c.nz : c.nx;
    f->L = f->col_lines ? c.nx : c.nz;
    const int nb = f->nb, L = f->L;
    require(nb <= 2048, "exact block factorisation: line length above 2048 is not supported");
    f->GT.alloc(size_t(L) * nb * nb);
    f->coup.alloc(size_t(L) * nb);
    f->status.alloc(1);
    CK(cudaMemsetAsync(f->status.p, 0, sizeof(int), c.stream));
    extract_lines<<<grid_blocks(int64_t(L) * nb, 256, 1 << 20), 256, 0, c.stream>>>(
        f->col_lines, c.nx, L, nb, c.east.p, c.south.p, f->coup.p);
    CK_LAUNCH();
    const bool smem = nb <= 112;
    const size_t base = size_t(2 * nb) * sizeof(double2) + size_t((nb + 3) & ~3) * sizeof(int);
    const size_t shm = base + (smem ? size_t(nb) * nb * sizeof(double2) : 0);
    if (!smem) f->work.alloc(size_t(nb) * nb);
    const int threads = nb <= 64 ? 256 : 512;
    if (smem)
        CK(cudaFuncSetAttribute(line_factor_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm)));
    else
        CK(cudaFuncSetAttribute(line_factor_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm)));
    const int64_t nn = int64_t(nb) * nb;
    for (int i = 0; i < L; ++i) {
        const double2* prev = i > 0 ? f->GT.p + (i - 1) * nn : nullptr;
        if (smem)
            line_factor_kernel<true><<<1, threads, shm, c.stream>>>(
                f->col_lines, c.nx, nb, i, c.diag.p, c.east.p, c.south.p, f->coup.p, prev,
                f->GT.p + i * nn, nullptr, f->status.p);
        else
            line_factor_kernel<false><<<1, threads, shm, c.stream>>>(
                f->col_lines, c.nx, nb, i, c.diag.p, c.east.p, c.south.p, f->coup.p, prev,
                f->GT.p + i * nn, f->work.p, f->status.p);
        CK_LAUNCH();
    }
    int st = 0;
    CK(cudaMemcpyAsync(&st, f->status.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    if (st != 0)
        throw FwiError(FWI_ERR_SINGULAR_PIVOT,
                       "LU: singular pivot at elimination step " + std::to_string(st - 1), st - 1);
    if (c.exact) exact_free(c.exact);
    c.exact = f.release();
}

void exact_solve_batch(Ctx& c, bool adjoint, const double2* b, double2* x, int nrhs) {
    require(c.exact != nullptr, "precond_apply: state has no exact factorization");
    const ExactFactor& f = *c.exact;
    c.ensure_work();
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
    gather_lines<<<tg, tb, 0, c.stream>>>(f.col_lines, c.nx, c.nz, f.L, f.nb, nrhs, adjoint, b, W);
    CK_LAUNCH();
    sweep_kernel<kSweepKG><<<(nrhs + kSweepKG - 1) / kSweepKG, 256, sweep_smem(f.nb), c.stream>>>(
        f.L, f.nb, nrhs, f.GT.p, f.coup.p, W);
    CK_LAUNCH();
    scatter_lines<<<tg, tb, 0, c.stream>>>(f.col_lines, c.nx, c.nz, f.L, f.nb, nrhs, adjoint, W, x);
    CK_LAUNCH();
    c.solve_count[FWI_PRECOND_EXACT] += nrhs;
}

}  // namespace fwi_b200
