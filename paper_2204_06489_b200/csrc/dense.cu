// dense.cu — the exact block solver for long lines (nb > 512, BASELINE config 5:
// nb = 1024, L = 2048, K = 256 right-hand sides).
//
// Same algebra as exact.cu (block-tridiagonal Schur factorisation along lines,
// G_i = S_i^{-1}, forward/backward line sweeps), but every line-level operation
// is a whole-GPU dense product instead of a one-cluster kernel:
//
//   factor, per line i (in order):
//     S_i = T_i - E_{i-1} G_{i-1} E_{i-1}                      (elementwise)
//     G_i = S_i^{-1} by block Gauss-Jordan, 64-wide blocks:
//       D^{-1} of the 64x64 diagonal block (partial pivoting inside the block)
//       R = D^{-1} A[K,:] (K columns := I),  A -= F R with F = A[:,K] (K rows := 0),
//       A[K,:] = R                                              (two cgemm launches)
//   sweep for nrhs right-hand sides (W[i][k][m] line-major):
//     forward   y_i = G_i (b_i - E_{i-1} y_{i-1})      prologue + cgemm (B = G_i^T)
//     backward  x_i = y_i - G_i (E_i x_{i+1})          prologue + cgemm with C0 = y_i
//
// Pivoting is restricted to the 64x64 diagonal blocks (block pivoting); the
// solve is validated by its residual ||A x - b|| in the tests and by parity with
// the reference LU on small grids (FWI_EXACT_DENSE=1 forces this path).
//
// cgemm is a SIMT FP64 complex GEMM (B200 FP64: 64 DFMA/clk/SM, measured by
// tools/fp64_probe.cu; the FP64 tensor path has the same peak, so DFMA with
// register tiling is the right unit): 64x64 or 32x64 output tiles, 16-deep K
// slabs staged through shared memory with register prefetch, 4 DFMA per
// complex multiply-add.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "dense.cuh"

namespace fwi_b200 {
namespace {

constexpr int kBN = 64, kBK = 16, kGemmThreads = 256;
constexpr int kInvSmem = 64 * 65 * int(sizeof(double2));

__device__ __forceinline__ void cmac4(double2& c, const double2 a, const double2 b) {
    c.x = fma(a.x, b.x, c.x);
    c.y = fma(a.x, b.y, c.y);
    c.x = fma(-a.y, b.y, c.x);
    c.y = fma(a.y, b.x, c.y);
}

// C[m][n] = (C0 ? C0[m][n] : 0) + alpha * sum_k A[m][k] B(k,n)
// A row-major (lda); B(k,n) = B[k*ldb + n] (BT = false) or B[n*ldb + k] (BT = true).
template <int BM, bool BT>
__global__ void __launch_bounds__(kGemmThreads) cgemm_kernel(int M, int N, int K, double alpha,
                                                             const double2* __restrict__ A, int64_t lda,
                                                             const double2* __restrict__ B, int64_t ldb,
                                                             const double2* C0, int64_t ldc0, double2* C,
                                                             int64_t ldc) {
    constexpr int TM = BM / 16;  // rows per thread
    constexpr int TN = 4;        // columns per thread (strided by 16)
    constexpr int A_PER = BM * kBK / kGemmThreads;
    constexpr int B_PER = kBK * kBN / kGemmThreads;
    __shared__ double2 As[kBK][BM];
    __shared__ double2 Bs[kBK][kBN];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * kBN;

    double2 ra[A_PER], rb[B_PER];
    auto load = [&](int k0) {
#pragma unroll
        for (int q = 0; q < A_PER; ++q) {  // A tile: k fastest (contiguous rows of A)
            const int e = tid + q * kGemmThreads;
            const int kk = e % kBK, mm = e / kBK;
            const int m = m0 + mm, k = k0 + kk;
            ra[q] = (m < M && k < K) ? A[int64_t(m) * lda + k] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int q = 0; q < B_PER; ++q) {
            const int e = tid + q * kGemmThreads;
            int kk, nn;
            if (BT) { kk = e % kBK; nn = e / kBK; }
            else { nn = e % kBN; kk = e / kBN; }
            const int n = n0 + nn, k = k0 + kk;
            rb[q] = (n < N && k < K) ? (BT ? B[int64_t(n) * ldb + k] : B[int64_t(k) * ldb + n])
                                     : make_double2(0.0, 0.0);
        }
    };
    auto store = [&]() {
#pragma unroll
        for (int q = 0; q < A_PER; ++q) {
            const int e = tid + q * kGemmThreads;
            As[e % kBK][e / kBK] = ra[q];
        }
#pragma unroll
        for (int q = 0; q < B_PER; ++q) {
            const int e = tid + q * kGemmThreads;
            if (BT) Bs[e % kBK][e / kBK] = rb[q];
            else Bs[e / kBN][e % kBN] = rb[q];
        }
    };

    double2 acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = make_double2(0.0, 0.0);

    load(0);
    for (int k0 = 0; k0 < K; k0 += kBK) {
        __syncthreads();
        store();
        __syncthreads();
        if (k0 + kBK < K) load(k0 + kBK);  // next slab in flight during the products
#pragma unroll 4
        for (int kk = 0; kk < kBK; ++kk) {
            double2 a[TM], b[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) a[i] = As[kk][ty * TM + i];
#pragma unroll
            for (int j = 0; j < TN; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) cmac4(acc[i][j], a[i], b[j]);
        }
    }
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int m = m0 + ty * TM + i;
        if (m >= M) continue;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int n = n0 + tx + 16 * j;
            if (n >= N) continue;
            double2 v = make_double2(alpha * acc[i][j].x, alpha * acc[i][j].y);
            if (C0) {
                const double2 c = C0[int64_t(m) * ldc0 + n];
                v.x += c.x;
                v.y += c.y;
            }
            C[int64_t(m) * ldc + n] = v;
        }
    }
}

// Inverse of one b x b diagonal block (b <= 64) by Gauss-Jordan with partial
// pivoting inside the block, in shared memory; one CTA.
__global__ void __launch_bounds__(256) block_inverse_kernel(int b, const double2* __restrict__ D, int64_t ldd,
                                                            double2* __restrict__ out, int64_t ldo, int* status,
                                                            int status_base) {
    extern __shared__ double2 bsm[];
    double2(*A)[65] = reinterpret_cast<double2(*)[65]>(bsm);  // [64][65]
    __shared__ double2 prow[64], pcol[64];
    __shared__ int piv[64];
    __shared__ int s_p;
    __shared__ double2 s_inv;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (int e = tid; e < b * b; e += blockDim.x) A[e / b][e % b] = D[int64_t(e / b) * ldd + e % b];
    __syncthreads();
    for (int k = 0; k < b; ++k) {
        if (wid == 0) {  // pivot: max |A[r][k]|, r >= k (ties: lowest row)
            double best = -1.0;
            int bi = b;
            for (int r = k + lane; r < b; r += 32) {
                const double m2 = A[r][k].x * A[r][k].x + A[r][k].y * A[r][k].y;
                if (m2 > best) { best = m2; bi = r; }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_down_sync(0xffffffffu, best, o);
                const int oi = __shfl_down_sync(0xffffffffu, bi, o);
                if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
            }
            if (lane == 0) {
                if (!(best > 0.0)) {
                    if (*status == 0) *status = status_base + k + 1;
                    bi = k;
                }
                s_p = bi;
                piv[k] = bi;
            }
        }
        __syncthreads();
        const int p = s_p;
        if (p != k)
            for (int j = tid; j < b; j += blockDim.x) {
                const double2 t = A[k][j];
                A[k][j] = A[p][j];
                A[p][j] = t;
            }
        __syncthreads();
        if (tid == 0) {
            const double2 d = A[k][k];
            s_inv = (d.x == 0.0 && d.y == 0.0) ? make_double2(0.0, 0.0) : cdiv(make_double2(1.0, 0.0), d);
        }
        __syncthreads();
        const double2 pinv = s_inv;
        for (int j = tid; j < b; j += blockDim.x) {
            const double2 a = (j == k) ? make_double2(1.0, 0.0) : A[k][j];
            const double2 v = make_double2(a.x * pinv.x - a.y * pinv.y, a.x * pinv.y + a.y * pinv.x);
            prow[j] = v;
            pcol[j] = (j == k) ? make_double2(0.0, 0.0) : A[j][k];
        }
        __syncthreads();
        for (int e = tid; e < b * b; e += blockDim.x) {
            const int r = e / b, j = e % b;
            if (r == k) {
                A[r][j] = prow[j];
            } else {
                const double2 f = pcol[r];
                double2 v = (j == k) ? make_double2(0.0, 0.0) : A[r][j];
                const double2 pr = prow[j];
                v.x -= f.x * pr.x - f.y * pr.y;
                v.y -= f.x * pr.y + f.y * pr.x;
                A[r][j] = v;
            }
        }
        __syncthreads();
    }
    for (int k = b - 1; k >= 0; --k) {  // undo the column permutation
        const int p = piv[k];
        if (p != k)
            for (int r = tid; r < b; r += blockDim.x) {
                const double2 t = A[r][k];
                A[r][k] = A[r][p];
                A[r][p] = t;
            }
        __syncthreads();
    }
    for (int e = tid; e < b * b; e += blockDim.x) out[int64_t(e / b) * ldo + e % b] = A[e / b][e % b];
}

// F = A[:, K] with rows K zeroed (nb x bs, ld kBlk), then A[:, K] = 0
__global__ void take_panel(int nb, int kb, int bs, double2* A, int64_t lda, double2* F) {
    const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (t >= int64_t(nb) * bs) return;
    const int r = int(t / bs), c = int(t % bs);
    double2& a = A[int64_t(r) * lda + kb + c];
    F[int64_t(r) * kDenseBlk + c] = (r >= kb && r < kb + bs) ? make_double2(0.0, 0.0) : a;
    a = make_double2(0.0, 0.0);
}

// Ablk = A[K, :] with the K columns replaced by the identity (bs x nb, ld nb)
__global__ void take_rows(int nb, int kb, int bs, const double2* A, int64_t lda, double2* Ablk) {
    const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (t >= int64_t(bs) * nb) return;
    const int c = int(t / nb), j = int(t % nb);
    Ablk[t] = (j >= kb && j < kb + bs) ? make_double2(j - kb == c ? 1.0 : 0.0, 0.0)
                                       : A[int64_t(kb + c) * lda + j];
}

__global__ void put_rows(int nb, int kb, int bs, const double2* R, double2* A, int64_t lda) {
    const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (t >= int64_t(bs) * nb) return;
    A[int64_t(kb + t / nb) * lda + t % nb] = R[t];
}

// sweep prologue: T[k][m] = bsel ? b[k][m] - e[m] v[k][m] : e[m] v[k][m]   (v may be null)
__global__ void sweep_prologue(int nb, int nrhs, const double2* __restrict__ b, const double2* __restrict__ e,
                               const double2* __restrict__ v, double2* __restrict__ T) {
    const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (t >= int64_t(nb) * nrhs) return;
    const int m = int(t % nb);
    double2 r = make_double2(0.0, 0.0);
    if (v) {
        const double2 ee = e[m], vv = v[t];
        r = make_double2(ee.x * vv.x - ee.y * vv.y, ee.x * vv.y + ee.y * vv.x);
    }
    if (b) r = make_double2(b[t].x - r.x, b[t].y - r.y);
    T[t] = r;
}

template <bool BT>
void cgemm_launch(cudaStream_t st, int M, int N, int K, double alpha, const double2* A, int64_t lda,
                  const double2* B, int64_t ldb, const double2* C0, int64_t ldc0, double2* C, int64_t ldc) {
    const int gx = (N + kBN - 1) / kBN;
    const int big = gx * ((M + 63) / 64);
    if (big >= sm_count()) {
        cgemm_kernel<64, BT><<<dim3(gx, (M + 63) / 64), kGemmThreads, 0, st>>>(M, N, K, alpha, A, lda, B, ldb,
                                                                                C0, ldc0, C, ldc);
    } else {
        cgemm_kernel<32, BT><<<dim3(gx, (M + 31) / 32), kGemmThreads, 0, st>>>(M, N, K, alpha, A, lda, B, ldb,
                                                                                C0, ldc0, C, ldc);
    }
    CK_LAUNCH();
}

inline int blocks_for(int64_t n) { return int((n + 255) / 256); }

}  // namespace

void cgemm(cudaStream_t st, bool bt, int M, int N, int K, double alpha, const double2* A, int64_t lda,
           const double2* B, int64_t ldb, const double2* C0, int64_t ldc0, double2* C, int64_t ldc) {
    if (bt) cgemm_launch<true>(st, M, N, K, alpha, A, lda, B, ldb, C0, ldc0, C, ldc);
    else cgemm_launch<false>(st, M, N, K, alpha, A, lda, B, ldb, C0, ldc0, C, ldc);
}

void DenseWork::ensure(int nb) {
    if (nb_ >= nb) return;
    F.alloc(size_t(nb) * kDenseBlk);
    Ablk.alloc(size_t(kDenseBlk) * nb);
    R.alloc(size_t(kDenseBlk) * nb);
    Dinv.alloc(size_t(kDenseBlk) * kDenseBlk);
    nb_ = nb;
}

void dense_invert(cudaStream_t st, int nb, double2* A, int64_t lda, DenseWork& w, int* status, int status_base) {
    w.ensure(nb);
    static bool attr = false;
    if (!attr) {
        CK(cudaFuncSetAttribute(block_inverse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kInvSmem));
        attr = true;
    }
    for (int kb = 0; kb < nb; kb += kDenseBlk) {
        const int bs = std::min(kDenseBlk, nb - kb);
        block_inverse_kernel<<<1, 256, kInvSmem, st>>>(bs, A + int64_t(kb) * lda + kb, lda, w.Dinv.p, kDenseBlk,
                                                       status, status_base + kb);
        CK_LAUNCH();
        take_rows<<<blocks_for(int64_t(bs) * nb), 256, 0, st>>>(nb, kb, bs, A, lda, w.Ablk.p);
        CK_LAUNCH();
        take_panel<<<blocks_for(int64_t(nb) * bs), 256, 0, st>>>(nb, kb, bs, A, lda, w.F.p);
        CK_LAUNCH();
        // R = D^{-1} Ablk
        cgemm_launch<false>(st, bs, nb, bs, 1.0, w.Dinv.p, kDenseBlk, w.Ablk.p, nb, nullptr, 0, w.R.p, nb);
        // A -= F R   (rows K of F are zero; columns K of A were zeroed)
        cgemm_launch<false>(st, nb, nb, bs, -1.0, w.F.p, kDenseBlk, w.R.p, nb, A, lda, A, lda);
        put_rows<<<blocks_for(int64_t(bs) * nb), 256, 0, st>>>(nb, kb, bs, w.R.p, A, lda);
        CK_LAUNCH();
    }
}

void dense_sweep(cudaStream_t st, int L, int nb, int nrhs, const double2* G, int64_t gp, const double2* coup,
                 double2* W, double2* T) {
    // y_i overwrites b_i in W (b_i is consumed by the prologue of its own step), and
    // x_i overwrites y_i in the backward sweep (each entry read, then written, by one thread).
    const int64_t blk = int64_t(nrhs) * nb;
    const int nbk = blocks_for(blk);
    for (int i = 0; i < L; ++i) {  // forward: y_i = G_i (b_i - E_{i-1} y_{i-1})
        sweep_prologue<<<nbk, 256, 0, st>>>(nb, nrhs, W + i * blk, i > 0 ? coup + int64_t(i - 1) * nb : nullptr,
                                            i > 0 ? W + (i - 1) * blk : nullptr, T);
        CK_LAUNCH();
        cgemm_launch<true>(st, nrhs, nb, nb, 1.0, T, nb, G + int64_t(i) * nb * gp, gp, nullptr, 0, W + i * blk, nb);
    }
    for (int i = L - 2; i >= 0; --i) {  // backward: x_i = y_i - G_i (E_i x_{i+1})
        sweep_prologue<<<nbk, 256, 0, st>>>(nb, nrhs, nullptr, coup + int64_t(i) * nb, W + (i + 1) * blk, T);
        CK_LAUNCH();
        cgemm_launch<true>(st, nrhs, nb, nb, -1.0, T, nb, G + int64_t(i) * nb * gp, gp, W + i * blk, nb,
                           W + i * blk, nb);
    }
}

}  // namespace fwi_b200
