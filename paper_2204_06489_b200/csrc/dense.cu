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
// cgemm runs on the FP64 tensor cores by default (zgemm_pipe_kernel: DMMA
// m8n8k4, Gauss's three-product form, a 3-stage cp.async ring; FWI_CGEMM picks
// the older variants): 32.2 TFLOP/s effective on 1024^3 against 26.5 for cuBLAS
// ZGEMM. The SIMT DFMA kernel (cgemm_kernel, FWI_CGEMM=simt,
// 64x64 or 32x64 tiles with register prefetch, 4 DFMA per complex
// multiply-add) is kept as the reference point (12.5 TFLOP/s).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>

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
// pivoting inside the block; one CTA of 256 threads. Thread (cj, rg) keeps entries
// (rg + 4i, cj), i < 16, of the working matrix in registers, so a pivot step moves
// only O(b) values through shared memory (the pivot column, the candidates, the
// pivot row and the row it swaps with; double-buffered, two barriers per step)
// instead of the whole 64 KB block. The column permutation is applied on output.
__global__ void __launch_bounds__(256) block_inverse_kernel(int b, const double2* __restrict__ D, int64_t ldd,
                                                            double2* __restrict__ out, int64_t ldo, int* status,
                                                            int status_base) {
    extern __shared__ double2 bsm[];
    double2(*A)[65] = reinterpret_cast<double2(*)[65]>(bsm);  // [64][65], only for the final permutation
    __shared__ double2 colk[2][64], rowp[2][64], rowk[2][64];
    __shared__ double cbest[2][4];
    __shared__ int crow[2][4];
    __shared__ int piv[64], perm[64];
    const int tid = threadIdx.x;
    const int cj = tid & 63, rg = tid >> 6;  // column; rows rg, rg+4, ...
    double2 a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int r = rg + 4 * i;
        a[i] = (r < b && cj < b) ? D[int64_t(r) * ldd + cj] : make_double2(0.0, 0.0);
    }
    for (int k = 0; k < b; ++k) {
        const int buf = k & 1;
        // (1) the four owners of column k publish it and their best candidate (rows >= k)
        if (cj == k) {
            double best = -1.0;
            int bi = b;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int r = rg + 4 * i;
                colk[buf][r] = a[i];
                const double m2 = a[i].x * a[i].x + a[i].y * a[i].y;
                if (r >= k && r < b && m2 > best) {  // rows ascend: ties keep the lowest
                    best = m2;
                    bi = r;
                }
            }
            cbest[buf][rg] = best;
            crow[buf][rg] = bi;
        }
        __syncthreads();
        // (2) every thread picks the same pivot (max |.|^2, ties: lowest row)
        double best = cbest[buf][0];
        int p = crow[buf][0];
#pragma unroll
        for (int q = 1; q < 4; ++q) {
            const double v = cbest[buf][q];
            const int r = crow[buf][q];
            if (v > best || (v == best && r < p)) {
                best = v;
                p = r;
            }
        }
        if (!(best > 0.0)) p = k;
        if (tid == 0) {
            piv[k] = p;
            if (!(best > 0.0)) atomicCAS(status, 0, status_base + k + 1);
        }
        // owners of rows p and k publish them (pre-swap); register index by unrolled select
        const int ip = p >> 2, ik = k >> 2;
        if ((p & 3) == rg) {
            double2 v = a[0];
#pragma unroll
            for (int i = 1; i < 16; ++i)
                if (i == ip) v = a[i];
            rowp[buf][cj] = v;
        }
        if ((k & 3) == rg) {
            double2 v = a[0];
#pragma unroll
            for (int i = 1; i < 16; ++i)
                if (i == ik) v = a[i];
            rowk[buf][cj] = v;
        }
        __syncthreads();
        // (3) swap rows k <-> p, scale the pivot row, eliminate column k everywhere
        const double2 d = colk[buf][p];
        const double m2 = d.x * d.x + d.y * d.y;
        const double rr = m2 > 0.0 ? 1.0 / m2 : 0.0;
        const double2 pinv = make_double2(d.x * rr, -d.y * rr);
        const double2 ap = (cj == k) ? make_double2(1.0, 0.0) : rowp[buf][cj];
        const double2 pr = make_double2(ap.x * pinv.x - ap.y * pinv.y, ap.x * pinv.y + ap.y * pinv.x);
        const bool colk_thread = (cj == k);
#pragma unroll
        for (int i = 0; i < 16; ++i) {  // common path: a -= f * pr (column k starts from 0)
            const double2 f = colk[buf][rg + 4 * i];
            double2 v = colk_thread ? make_double2(0.0, 0.0) : a[i];
            v.x -= f.x * pr.x - f.y * pr.y;
            v.y -= f.x * pr.y + f.y * pr.x;
            a[i] = v;
        }
        if ((p & 3) == rg && p != k) {  // row p now holds the old row k
            const double2 f = colk[buf][k];
            double2 v = colk_thread ? make_double2(0.0, 0.0) : rowk[buf][cj];
            v.x -= f.x * pr.x - f.y * pr.y;
            v.y -= f.x * pr.y + f.y * pr.x;
#pragma unroll
            for (int i = 0; i < 16; ++i)
                if (i == ip) a[i] = v;
        }
        if ((k & 3) == rg) {  // the pivot row
#pragma unroll
            for (int i = 0; i < 16; ++i)
                if (i == ik) a[i] = pr;
        }
    }
    // undoing the column swaps in reverse order = one permutation, applied through shared memory
    if (tid == 0) {
        for (int j = 0; j < b; ++j) perm[j] = j;
        for (int k = b - 1; k >= 0; --k) {
            const int t = perm[k];
            perm[k] = perm[piv[k]];
            perm[piv[k]] = t;
        }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) A[rg + 4 * i][cj] = a[i];
    __syncthreads();
    if (cj < b)
        for (int r = rg; r < b; r += 4) out[int64_t(r) * ldo + cj] = A[r][perm[cj]];
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

// twisted middle line: T[k][m] = b[k][m] - e1[m] v1[k][m] - e2[m] v2[k][m]
__global__ void sweep_middle(int nb, int nrhs, const double2* __restrict__ b, const double2* __restrict__ e1,
                             const double2* __restrict__ v1, const double2* __restrict__ e2,
                             const double2* __restrict__ v2, double2* __restrict__ T) {
    const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (t >= int64_t(nb) * nrhs) return;
    const int m = int(t % nb);
    const double2 a = e1[m], x = v1[t], c = e2[m], y = v2[t];
    T[t] = make_double2(b[t].x - (a.x * x.x - a.y * x.y) - (c.x * y.x - c.y * y.y),
                        b[t].y - (a.x * x.y + a.y * x.x) - (c.x * y.y + c.y * y.x));
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

// ---------------------------------------------------------------------------
// FP64 tensor-core variant: mma.sync m8n8k4 (DMMA). Complex products as four real
// MMAs into three accumulators: P = Ar Br, Q = Ai Bi, I = Ar Bi + Ai Br (C = P - Q + iI).
// 32x64 output tile per CTA, 8 warps in a 2x4 grid of 16x16 warp tiles (2x2 MMA tiles),
// 16-deep complex K slabs staged in shared memory as separate re/im planes (k-major)
// with a register prefetch of the next slab.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

constexpr int kTBM = 32, kTBN = 64, kTBK = 16, kTPadM = kTBM + 4, kTPadN = kTBN + 4;

template <bool BT>
__global__ void __launch_bounds__(256) zgemm_dmma_kernel(int M, int N, int K, double alpha,
                                                         const double2* __restrict__ A, int64_t lda,
                                                         const double2* __restrict__ B, int64_t ldb,
                                                         const double2* C0, int64_t ldc0, double2* C, int64_t ldc) {
    __shared__ double Ar[kTBK][kTPadM], Ai[kTBK][kTPadM], Br[kTBK][kTPadN], Bi[kTBK][kTPadN];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp & 1, wn = warp >> 1;  // 2 x 4 warp grid of 16 x 16 tiles
    const int m0 = blockIdx.y * kTBM, n0 = blockIdx.x * kTBN;
    constexpr int A_PER = kTBM * kTBK / 256, B_PER = kTBN * kTBK / 256;  // 2, 4
    double2 ra[A_PER], rb[B_PER];
    auto load = [&](int k0) {
#pragma unroll
        for (int q = 0; q < A_PER; ++q) {
            const int e = tid + q * 256, kk = e % kTBK, mm = e / kTBK;
            const int m = m0 + mm, k = k0 + kk;
            ra[q] = (m < M && k < K) ? A[int64_t(m) * lda + k] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int q = 0; q < B_PER; ++q) {
            const int e = tid + q * 256;
            int kk, nn;
            if (BT) { kk = e % kTBK; nn = e / kTBK; }
            else { nn = e % kTBN; kk = e / kTBN; }
            const int n = n0 + nn, k = k0 + kk;
            rb[q] = (n < N && k < K) ? (BT ? B[int64_t(n) * ldb + k] : B[int64_t(k) * ldb + n])
                                     : make_double2(0.0, 0.0);
        }
    };
    auto store = [&]() {
#pragma unroll
        for (int q = 0; q < A_PER; ++q) {
            const int e = tid + q * 256, kk = e % kTBK, mm = e / kTBK;
            Ar[kk][mm] = ra[q].x;
            Ai[kk][mm] = ra[q].y;
        }
#pragma unroll
        for (int q = 0; q < B_PER; ++q) {
            const int e = tid + q * 256;
            int kk, nn;
            if (BT) { kk = e % kTBK; nn = e / kTBK; }
            else { nn = e % kTBN; kk = e / kTBN; }
            Br[kk][nn] = rb[q].x;
            Bi[kk][nn] = rb[q].y;
        }
    };
    double P[2][2][2] = {}, Q[2][2][2] = {}, I[2][2][2] = {};
    const int g = lane >> 2, t4 = lane & 3;
    load(0);
    for (int k0 = 0; k0 < K; k0 += kTBK) {
        __syncthreads();
        store();
        __syncthreads();
        if (k0 + kTBK < K) load(k0 + kTBK);
#pragma unroll
        for (int ks = 0; ks < kTBK; ks += 4) {
            double ar[2], ai[2], br[2], bi[2];
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                ar[t] = Ar[ks + t4][wm * 16 + t * 8 + g];
                ai[t] = Ai[ks + t4][wm * 16 + t * 8 + g];
                br[t] = Br[ks + t4][wn * 16 + t * 8 + g];
                bi[t] = Bi[ks + t4][wn * 16 + t * 8 + g];
            }
#pragma unroll
            for (int t = 0; t < 2; ++t)
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    dmma(P[t][u], ar[t], br[u]);
                    dmma(Q[t][u], ai[t], bi[u]);
                    dmma(I[t][u], ar[t], bi[u]);
                    dmma(I[t][u], ai[t], br[u]);
                }
        }
    }
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int m = m0 + wm * 16 + t * 8 + g, n = n0 + wn * 16 + u * 8 + 2 * t4 + e;
                if (m >= M || n >= N) continue;
                double2 v = make_double2(alpha * (P[t][u][e] - Q[t][u][e]), alpha * I[t][u][e]);
                if (C0) {
                    const double2 c = C0[int64_t(m) * ldc0 + n];
                    v.x += c.x;
                    v.y += c.y;
                }
                C[int64_t(m) * ldc + n] = v;
            }
}

// ---------------------------------------------------------------------------
// Pipelined DMMA variant (default): BM x 64 output tile per CTA (BM = 32 or 64),
// 8 warps in a 2 x 4 grid, complex operands staged interleaved (re, im) in a
// 3-stage cp.async ring so one 16-byte shared load yields both planes of a
// fragment element; fragments for the next k4 step are loaded while the current
// one issues its DMMAs. One block barrier per 16-deep K slab.
// ---------------------------------------------------------------------------
constexpr int kPBN = 64, kPBK = 16, kPStages = 3, kPPitchK = kPBK + 4;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(gmem), "r"(pred ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int BM, bool BT, int BN = kPBN, int NS = kPStages>
constexpr int zgemm_pipe_smem() {
    // A: [BM][kPPitchK]; B: BT ? [BN][kPPitchK] : [kPBK][BN + 2]   (double2 elements)
    return NS * (BM * kPPitchK + (BT ? BN * kPPitchK : kPBK * (BN + 2))) * 16;
}

// G3: Gauss's three-product form, S = (Ar+Ai)(Br+Bi): real = P - Q, imag = S - P - Q
// (3 DMMA per complex k-step instead of 4; operand sums formed as the fragments load)
// batch strides: blockIdx.z selects A + z sA, B + z sB, C0 + z sC0, C + z sC (cgemm_batched)
struct GemmStrides {
    int64_t a = 0, b = 0, c0 = 0, c = 0;
};

// BN: the CTA's N tile (64, or 32 for narrow batches: twice the CTAs, so a batch of ~100
// products spreads over the SMs more evenly); warps 2 (m) x 4 (n), warp tile (BM/2) x (BN/4)
template <int BM, bool BT, bool G3, int BN = kPBN, int NS = kPStages>
__global__ void __launch_bounds__(256) zgemm_pipe_kernel(int M, int N, int K, double alpha,
                                                         const double2* __restrict__ A, int64_t lda,
                                                         const double2* __restrict__ B, int64_t ldb,
                                                         const double2* C0, int64_t ldc0, double2* C, int64_t ldc,
                                                         GemmStrides bs) {
    pdl_enter();
    extern __shared__ __align__(16) double2 psm[];
    A += blockIdx.z * bs.a;
    B += blockIdx.z * bs.b;
    if (C0) C0 += blockIdx.z * bs.c0;
    C += blockIdx.z * bs.c;
    constexpr int PN = BN + 2;  // B row pitch (non-transposed)
    constexpr int ASZ = BM * kPPitchK, BSZ = BT ? BN * kPPitchK : kPBK * PN;
    constexpr int TM = BM / 16;  // m8 tiles per warp (warp tile (BM/2) x (BN/4))
    constexpr int UN = BN / 32;  // n8 tiles per warp
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp & 1, wn = warp >> 1;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int g = lane >> 2, t4 = lane & 3;
    const int KT = (K + kPBK - 1) / kPBK;

    auto load_stage = [&](int stage, int k0) {
        double2* As = psm + stage * (ASZ + BSZ);
        double2* Bs = As + ASZ;
#pragma unroll
        for (int q = 0; q < BM * kPBK / 256; ++q) {
            const int e = tid + q * 256, kk = e % kPBK, mm = e / kPBK;
            const int m = m0 + mm, k = k0 + kk;
            const bool ok = m < M && k < K;
            cp_async16(As + mm * kPPitchK + kk, ok ? A + int64_t(m) * lda + k : A, ok);
        }
#pragma unroll
        for (int q = 0; q < BN * kPBK / 256; ++q) {
            const int e = tid + q * 256;
            if (BT) {
                const int kk = e % kPBK, nn = e / kPBK, n = n0 + nn, k = k0 + kk;
                const bool ok = n < N && k < K;
                cp_async16(Bs + nn * kPPitchK + kk, ok ? B + int64_t(n) * ldb + k : B, ok);
            } else {
                const int nn = e % BN, kk = e / BN, n = n0 + nn, k = k0 + kk;
                const bool ok = n < N && k < K;
                cp_async16(Bs + kk * PN + nn, ok ? B + int64_t(k) * ldb + n : B, ok);
            }
        }
    };

    double P[TM][UN][2] = {}, Q[TM][UN][2] = {}, I[TM][UN][2] = {};
#pragma unroll
    for (int s = 0; s < NS - 1; ++s) {
        if (s < KT) load_stage(s, s * kPBK);
        cp_async_commit();
    }
    for (int kt = 0; kt < KT; ++kt) {
        cp_async_wait<NS - 2>();
        __syncthreads();  // stage kt landed for every thread; stage kt-1 is free
        {
            const int nk = kt + NS - 1;
            if (nk < KT) load_stage(nk % NS, nk * kPBK);
            cp_async_commit();
        }
        const double2* As = psm + (kt % NS) * (ASZ + BSZ);
        const double2* Bs = As + ASZ;
        double2 fa[2][TM], fb[2][UN];
        double sa[2][TM], sb[2][UN];  // G3 operand sums
        auto frag = [&](int buf, int ks) {
#pragma unroll
            for (int t = 0; t < TM; ++t) {
                fa[buf][t] = As[(wm * (BM / 2) + t * 8 + g) * kPPitchK + ks + t4];
                if (G3) sa[buf][t] = fa[buf][t].x + fa[buf][t].y;
            }
#pragma unroll
            for (int u = 0; u < UN; ++u) {
                fb[buf][u] = BT ? Bs[(wn * (BN / 4) + u * 8 + g) * kPPitchK + ks + t4]
                                : Bs[(ks + t4) * PN + wn * (BN / 4) + u * 8 + g];
                if (G3) sb[buf][u] = fb[buf][u].x + fb[buf][u].y;
            }
        };
        frag(0, 0);
#pragma unroll
        for (int k4 = 0; k4 < kPBK / 4; ++k4) {
            const int cur = k4 & 1;
            if (k4 + 1 < kPBK / 4) frag(cur ^ 1, (k4 + 1) * 4);
#pragma unroll
            for (int t = 0; t < TM; ++t)
#pragma unroll
                for (int u = 0; u < UN; ++u) {
                    dmma(P[t][u], fa[cur][t].x, fb[cur][u].x);
                    dmma(Q[t][u], fa[cur][t].y, fb[cur][u].y);
                    if (G3) {
                        dmma(I[t][u], sa[cur][t], sb[cur][u]);
                    } else {
                        dmma(I[t][u], fa[cur][t].x, fb[cur][u].y);
                        dmma(I[t][u], fa[cur][t].y, fb[cur][u].x);
                    }
                }
        }
    }
    cp_async_wait<0>();
#pragma unroll
    for (int t = 0; t < TM; ++t)
#pragma unroll
        for (int u = 0; u < UN; ++u)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int m = m0 + wm * (BM / 2) + t * 8 + g, n = n0 + wn * (BN / 4) + u * 8 + 2 * t4 + e;
                if (m >= M || n >= N) continue;
                const double im = G3 ? I[t][u][e] - P[t][u][e] - Q[t][u][e] : I[t][u][e];
                double2 v = make_double2(alpha * (P[t][u][e] - Q[t][u][e]), alpha * im);
                if (C0) {
                    const double2 c = C0[int64_t(m) * ldc0 + n];
                    v.x += c.x;
                    v.y += c.y;
                }
                C[int64_t(m) * ldc + n] = v;
            }
}

template <int BM, bool BT, bool G3, int BN = kPBN, int NS = kPStages>
void zgemm_pipe_launch(cudaStream_t st, int M, int N, int K, double alpha, const double2* A, int64_t lda,
                       const double2* B, int64_t ldb, const double2* C0, int64_t ldc0, double2* C, int64_t ldc,
                       GemmStrides bs = {}, int batch = 1) {
    constexpr int smem = zgemm_pipe_smem<BM, BT, BN, NS>();
    static bool attr = false;
    if (!attr) {
        CK(cudaFuncSetAttribute(zgemm_pipe_kernel<BM, BT, G3, BN, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                smem));
        attr = true;
    }
    launch_pdl<kPdlDense>(zgemm_pipe_kernel<BM, BT, G3, BN, NS>, dim3((N + BN - 1) / BN, (M + BM - 1) / BM, batch),
                          dim3(256), smem, st, M, N, K, alpha, A, lda, B, ldb, C0, ldc0, C, ldc, bs);
    CK_LAUNCH();
}

template <bool BT>
void cgemm_launch(cudaStream_t st, int M, int N, int K, double alpha, const double2* A, int64_t lda,
                  const double2* B, int64_t ldb, const double2* C0, int64_t ldc0, double2* C, int64_t ldc) {
    // FWI_CGEMM: "pipe3" (default: Gauss's 3-product form, 3 DMMA per complex k-step; sweep shape
    // 85.5 -> 78.4 us, 1024^3 27.4 -> 32.2 TFLOP/s, relative error 1.9e-15 against 1.7e-15),
    // "pipe" (4-product form), "dmma" (the unpipelined DMMA kernel), "simt"
    static const int variant = [] {
        const char* e = std::getenv("FWI_CGEMM");
        if (!e) return 3;
        const std::string v(e);
        return v == "simt" ? 2 : v == "dmma" ? 1 : v == "pipe" ? 0 : 3;
    }();
    if (variant == 0 || variant == 3) {
        // 64-row tiles only when they still give every SM a tile
        const int tiles64 = ((N + kPBN - 1) / kPBN) * ((M + 63) / 64);
        if (variant == 3) {
            if (tiles64 >= sm_count())
                zgemm_pipe_launch<64, BT, true>(st, M, N, K, alpha, A, lda, B, ldb, C0, ldc0, C, ldc);
            else
                zgemm_pipe_launch<32, BT, true>(st, M, N, K, alpha, A, lda, B, ldb, C0, ldc0, C, ldc);
            return;
        }
        if (tiles64 >= sm_count())
            zgemm_pipe_launch<64, BT, false>(st, M, N, K, alpha, A, lda, B, ldb, C0, ldc0, C, ldc);
        else
            zgemm_pipe_launch<32, BT, false>(st, M, N, K, alpha, A, lda, B, ldb, C0, ldc0, C, ldc);
        return;
    }
    if (variant == 1) {
        zgemm_dmma_kernel<BT><<<dim3((N + kTBN - 1) / kTBN, (M + kTBM - 1) / kTBM), 256, 0, st>>>(
            M, N, K, alpha, A, lda, B, ldb, C0, ldc0, C, ldc);
        CK_LAUNCH();
        return;
    }
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

namespace {
// Split-K strided-batched complex GEMM for a few narrow products (the upper levels of the
// cyclic reduction: M = nrhs, N = K = nb, batch 1..50, where the tiled kernel leaves most
// SMs idle and each CTA runs its whole K at one SM's DMMA rate): one warp per 8x8 output
// tile and K chunk of kc, operands straight from L2 into DMMA fragments (Gauss's three-
// product form), partial tiles to part[(z S + s)][M][N]; zgemm_splitk_reduce sums them in
// chunk order (deterministic) and applies alpha and C0.
template <bool BT>
__global__ void __launch_bounds__(128) zgemm_splitk_kernel(int M, int N, int K, int kc, int S,
                                                          const double2* __restrict__ A, int64_t lda, int64_t sA,
                                                          const double2* __restrict__ B, int64_t ldb, int64_t sB,
                                                          double2* __restrict__ part) {
    pdl_enter();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int n0 = (blockIdx.x * 4 + w) * 8, m0 = blockIdx.y * 8;
    const int z = blockIdx.z / S, s = blockIdx.z % S;
    if (n0 >= N) return;
    A += z * sA;
    B += z * sB;
    const int g = lane >> 2, t4 = lane & 3;
    const int k0 = s * kc, k1 = min(K, k0 + kc);
    const int m = m0 + g, n = n0 + g;
    const bool mok = m < M, nok = n < N;
    double P[2] = {0.0, 0.0}, Q[2] = {0.0, 0.0}, I[2] = {0.0, 0.0};
#pragma unroll 8
    for (int k = k0; k < k1; k += 4) {
        const int kk = k + t4;
        const bool kok = kk < k1;
        const double2 a = (mok && kok) ? __ldg(A + int64_t(m) * lda + kk) : make_double2(0.0, 0.0);
        const double2 b = (nok && kok) ? __ldg(BT ? B + int64_t(n) * ldb + kk : B + int64_t(kk) * ldb + n)
                                       : make_double2(0.0, 0.0);
        dmma(P, a.x, b.x);
        dmma(Q, a.y, b.y);
        dmma(I, a.x + a.y, b.x + b.y);
    }
    double2* out = part + int64_t(blockIdx.z) * M * N;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int mm = m0 + g, nn = n0 + 2 * t4 + e;
        if (mm < M && nn < N) out[int64_t(mm) * N + nn] = make_double2(P[e] - Q[e], I[e] - P[e] - Q[e]);
    }
}

// Up to two products in one launch, for the cyclic-reduction solve levels:
//   C_z = C0_z + sum_t alpha_t A_{t,z} B_{t,z}    (term t present for z in [lo_t, hi_t))
// one warp per 8x8 output tile over the whole K (M = nrhs, N = K = nb), operands from L2
// into DMMA fragments (Gauss's three-product form), C0 read in the epilogue. Fewer launches
// than one tiled GEMM per product plus reductions, and every SM busy on narrow batches.
struct Gemm2Term {
    const double2* A;
    int64_t lda, sA;
    const double2* B;
    int64_t ldb, sB;
    double alpha;
    int bt, lo, hi;
};

// one 8x8 output tile (rows m0.., columns n0.., batch entry z) of C_z = C0_z + sum_t alpha_t A B
template <int CH>
__device__ __forceinline__ void zgemm2_tile(int M, int N, int K, const Gemm2Term& t0, const Gemm2Term& t1, int nterms,
                                            const double2* C0, int64_t ldc0, int64_t sC0, double2* C, int64_t ldc,
                                            int64_t sC, int m0, int n0, int z, int lane) {
    const int g = lane >> 2, t4 = lane & 3;
    const int m = m0 + g, n = n0 + g;
    const bool mok = m < M, nok = n < N;
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};  // (re, im) x 2 columns
    for (int tt = 0; tt < nterms; ++tt) {
        const Gemm2Term& T = tt == 0 ? t0 : t1;
        if (z < T.lo || z >= T.hi) continue;
        const double2* A = T.A + (z - T.lo) * T.sA;
        const double2* B = T.B + (z - T.lo) * T.sB;
        double P[2] = {0.0, 0.0}, Q[2] = {0.0, 0.0}, I[2] = {0.0, 0.0};
        // chunks of CH k4-steps: the next chunk's loads are issued before this chunk's DMMAs
        double2 ca[CH], cb[CH], na[CH], nb_[CH];
        auto load = [&](int k0, double2 (&ra)[CH], double2 (&rb)[CH]) {
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                const int kk = k0 + 4 * q + t4;
                const bool kok = kk < K;
                ra[q] = (mok && kok) ? __ldg(A + int64_t(m) * T.lda + kk) : make_double2(0.0, 0.0);
                rb[q] = (nok && kok) ? __ldg(T.bt ? B + int64_t(n) * T.ldb + kk : B + int64_t(kk) * T.ldb + n)
                                     : make_double2(0.0, 0.0);
            }
        };
        load(0, ca, cb);
        for (int k0 = 0; k0 < K; k0 += 4 * CH) {
            if (k0 + 4 * CH < K) load(k0 + 4 * CH, na, nb_);
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                dmma(P, ca[q].x, cb[q].x);
                dmma(Q, ca[q].y, cb[q].y);
                dmma(I, ca[q].x + ca[q].y, cb[q].x + cb[q].y);
            }
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                ca[q] = na[q];
                cb[q] = nb_[q];
            }
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            acc[e][0] += T.alpha * (P[e] - Q[e]);
            acc[e][1] += T.alpha * (I[e] - P[e] - Q[e]);
        }
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int mm = m0 + g, nn = n0 + 2 * t4 + e;
        if (mm >= M || nn >= N) continue;
        double2 v = make_double2(acc[e][0], acc[e][1]);
        if (C0) {
            const double2 c = C0[z * sC0 + int64_t(mm) * ldc0 + nn];
            v.x += c.x;
            v.y += c.y;
        }
        C[z * sC + int64_t(mm) * ldc + nn] = v;
    }
}

// CH: k4-steps per prefetched chunk; MINB: CTAs per SM the register budget is cut for (the kernel
// is latency-bound: more resident warps beat deeper per-warp prefetch, C3 1.92 -> 1.86 ms per
// GMRES iteration with CH = 4 at four CTAs per SM against CH = 8 at three)
template <int CH, int MINB>
__global__ void __launch_bounds__(128, MINB) zgemm2_warp_kernel(int M, int N, int K, Gemm2Term t0, Gemm2Term t1,
                                                               int nterms, const double2* C0, int64_t ldc0,
                                                               int64_t sC0, double2* C, int64_t ldc, int64_t sC) {
    pdl_enter();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int n0 = (blockIdx.x * 4 + w) * 8, m0 = blockIdx.y * 8, z = blockIdx.z;
    if (n0 >= N) return;
    zgemm2_tile<CH>(M, N, K, t0, t1, nterms, C0, ldc0, sC0, C, ldc, sC, m0, n0, z, lane);
}

// The same products for narrow batches (the upper cyclic-reduction levels: a few products, so
// a warp's walk over K — chunks of operands from DRAM/L2 one after another — is the launch's
// latency): one CTA per 8x8 output tile, its four warps each take a quarter of K with all of
// their operand loads issued at once, and warp 0 sums the quarters in warp order (deterministic)
// before alpha, C0 and the store.
__global__ void __launch_bounds__(128) zgemm2_splitk_tile_kernel(int M, int N, int K, Gemm2Term t0, Gemm2Term t1,
                                                                int nterms, const double2* C0, int64_t ldc0,
                                                                int64_t sC0, double2* C, int64_t ldc, int64_t sC) {
    pdl_enter();
    __shared__ double red[2][4][32][6];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int n0 = blockIdx.x * 8, m0 = blockIdx.y * 8, z = blockIdx.z;
    const int g = lane >> 2, t4 = lane & 3;
    const int m = m0 + g, n = n0 + g;
    const bool mok = m < M, nok = n < N;
    const int kq = ((K + 15) / 16) * 4;  // a warp's quarter of K, a multiple of 4
    const int k0 = w * kq, k1 = min(K, k0 + kq);
    constexpr int CH = 8;                 // k4-steps per warp held in registers (K <= 128 in one pass)
    for (int tt = 0; tt < nterms; ++tt) {
        const Gemm2Term& T = tt == 0 ? t0 : t1;
        double P[2] = {0.0, 0.0}, Q[2] = {0.0, 0.0}, I[2] = {0.0, 0.0};
        if (z >= T.lo && z < T.hi) {
            const double2* A = T.A + (z - T.lo) * T.sA;
            const double2* B = T.B + (z - T.lo) * T.sB;
            for (int kb = k0; kb < k1; kb += 4 * CH) {
                double2 ra[CH], rb[CH];
#pragma unroll
                for (int q = 0; q < CH; ++q) {
                    const int kk = kb + 4 * q + t4;
                    const bool kok = kk < k1;
                    ra[q] = (mok && kok) ? __ldg(A + int64_t(m) * T.lda + kk) : make_double2(0.0, 0.0);
                    rb[q] = (nok && kok) ? __ldg(T.bt ? B + int64_t(n) * T.ldb + kk : B + int64_t(kk) * T.ldb + n)
                                         : make_double2(0.0, 0.0);
                }
#pragma unroll
                for (int q = 0; q < CH; ++q) {
                    dmma(P, ra[q].x, rb[q].x);
                    dmma(Q, ra[q].y, rb[q].y);
                    dmma(I, ra[q].x + ra[q].y, rb[q].x + rb[q].y);
                }
            }
        }
        double* r = red[tt][w][lane];
        r[0] = P[0];
        r[1] = P[1];
        r[2] = Q[0];
        r[3] = Q[1];
        r[4] = I[0];
        r[5] = I[1];
    }
    __syncthreads();
    if (w != 0) return;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        double re = 0.0, im = 0.0;
        for (int tt = 0; tt < nterms; ++tt) {
            const Gemm2Term& T = tt == 0 ? t0 : t1;
            if (z < T.lo || z >= T.hi) continue;
            double P = 0.0, Q = 0.0, I = 0.0;
            for (int q = 0; q < 4; ++q) {
                P += red[tt][q][lane][e];
                Q += red[tt][q][lane][2 + e];
                I += red[tt][q][lane][4 + e];
            }
            re += T.alpha * (P - Q);
            im += T.alpha * (I - P - Q);
        }
        const int mm = m0 + g, nn = n0 + 2 * t4 + e;
        if (mm >= M || nn >= N) continue;
        double2 v = make_double2(re, im);
        if (C0) {
            const double2 c = C0[z * sC0 + int64_t(mm) * ldc0 + nn];
            v.x += c.x;
            v.y += c.y;
        }
        C[z * sC + int64_t(mm) * ldc + nn] = v;
    }
}

__global__ void zgemm_splitk_reduce(int M, int N, int S, double alpha, const double2* __restrict__ part,
                                    const double2* C0, int64_t ldc0, int64_t sC0, double2* C, int64_t ldc,
                                    int64_t sC) {
    pdl_enter();
    const int z = blockIdx.y;
    const int64_t mn = int64_t(M) * N;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < mn; t += int64_t(gridDim.x) * blockDim.x) {
        const int m = int(t / N), n = int(t % N);
        double2 acc = make_double2(0.0, 0.0);
        for (int s = 0; s < S; ++s) {
            const double2 p = part[(int64_t(z) * S + s) * mn + t];
            acc.x += p.x;
            acc.y += p.y;
        }
        double2 v = make_double2(alpha * acc.x, alpha * acc.y);
        if (C0) {
            const double2 c = C0[z * sC0 + int64_t(m) * ldc0 + n];
            v.x += c.x;
            v.y += c.y;
        }
        C[z * sC + int64_t(m) * ldc + n] = v;
    }
}
}  // namespace

void cgemm_batched(cudaStream_t st, bool bt, int M, int N, int K, double alpha, const double2* A, int64_t lda,
                   int64_t sA, const double2* B, int64_t ldb, int64_t sB, const double2* C0, int64_t ldc0,
                   int64_t sC0, double2* C, int64_t ldc, int64_t sC, int batch, double2* scratch,
                   size_t scratch_count) {
    if (batch <= 0) return;
    require(batch <= 65535, "cgemm_batched: batch above 65535");
    // few tiles: split K over warps (see zgemm_splitk_kernel); FWI_CGEMM_SPLITK_CTAS moves the
    // switch point (tiled CTAs below which the split-K form runs)
    static const int64_t split_below = std::getenv("FWI_CGEMM_SPLITK_CTAS")
                                           ? std::atoll(std::getenv("FWI_CGEMM_SPLITK_CTAS"))
                                           : 2 * int64_t(sm_count());
    const int64_t ctas32 = int64_t((N + kPBN - 1) / kPBN) * ((M + 31) / 32) * batch;
    if (scratch && ctas32 < split_below) {
        const int kc = 32, S = (K + kc - 1) / kc;
        const size_t need = size_t(batch) * S * size_t(M) * N;
        if (need <= scratch_count && int64_t(batch) * S <= 65535) {
            const dim3 g((N + 31) / 32, (M + 7) / 8, unsigned(batch * S));
            if (bt)
                launch_pdl<kPdlDense>(zgemm_splitk_kernel<true>, dim3(g), dim3(128), 0, st, M, N, K, kc, S, A, lda, sA,
                                      B, ldb, sB, scratch);
            else
                launch_pdl<kPdlDense>(zgemm_splitk_kernel<false>, dim3(g), dim3(128), 0, st, M, N, K, kc, S, A, lda, sA,
                                      B, ldb, sB, scratch);
            CK_LAUNCH();
            const int64_t mn = int64_t(M) * N;
            launch_pdl<kPdlDense>(zgemm_splitk_reduce,
                                  dim3(dim3(unsigned(std::min<int64_t>((mn + 255) / 256, 64)), unsigned(batch))),
                                  dim3(256), 0, st, M, N, S, alpha, scratch, C0, ldc0, sC0, C, ldc, sC);
            CK_LAUNCH();
            return;
        }
    }
    GemmStrides bs;
    bs.a = sA;
    bs.b = sB;
    bs.c0 = sC0;
    bs.c = sC;
    // 48-row tiles for 48 rows (config 3's 48 right-hand sides: no padded rows); otherwise
    // 64-row tiles only when they still give every SM a tile (Gauss's 3-product form)
    if (M == 48) {
        // 32-wide N tiles when 64-wide ones would leave the last wave of SMs short (a batch of
        // ~100 products: 192 tiles on 148 SMs take two tile-times, 384 half tiles ~1.5);
        // FWI_CGEMM_BN=32|64 forces the width
        static const int bn_env = std::getenv("FWI_CGEMM_BN") ? std::atoi(std::getenv("FWI_CGEMM_BN")) : 0;
        const int64_t t64 = int64_t((N + 63) / 64) * batch;
        const int sms = sm_count();
        const int64_t w64 = 2 * ((t64 + sms - 1) / sms), w32 = (2 * t64 + sms - 1) / sms;  // in half tiles
        const bool narrow = bn_env ? bn_env == 32 : 5 * w32 <= 4 * w64;
        // narrow tiles keep two stages (51 KB: four CTAs per SM; C3 537 -> 551 it/s against three
        // stages at two CTAs per SM); FWI_CGEMM_NS=3 restores three
        static const int ns_env = std::getenv("FWI_CGEMM_NS") ? std::atoi(std::getenv("FWI_CGEMM_NS")) : 2;
        if (narrow && ns_env == 2) {
            if (bt)
                zgemm_pipe_launch<48, true, true, 32, 2>(st, M, N, K, alpha, A, lda, B, ldb, C0, ldc0, C, ldc, bs,
                                                         batch);
            else
                zgemm_pipe_launch<48, false, true, 32, 2>(st, M, N, K, alpha, A, lda, B, ldb, C0, ldc0, C, ldc, bs,
                                                          batch);
        } else if (narrow) {
            if (bt)
                zgemm_pipe_launch<48, true, true, 32>(st, M, N, K, alpha, A, lda, B, ldb, C0, ldc0, C, ldc, bs, batch);
            else
                zgemm_pipe_launch<48, false, true, 32>(st, M, N, K, alpha, A, lda, B, ldb, C0, ldc0, C, ldc, bs, batch);
        } else if (bt) {
            zgemm_pipe_launch<48, true, true>(st, M, N, K, alpha, A, lda, B, ldb, C0, ldc0, C, ldc, bs, batch);
        } else {
            zgemm_pipe_launch<48, false, true>(st, M, N, K, alpha, A, lda, B, ldb, C0, ldc0, C, ldc, bs, batch);
        }
        return;
    }
    const int64_t tiles64 = int64_t((N + kPBN - 1) / kPBN) * ((M + 63) / 64) * batch;
    if (bt) {
        if (tiles64 >= sm_count() && M > 32)
            zgemm_pipe_launch<64, true, true>(st, M, N, K, alpha, A, lda, B, ldb, C0, ldc0, C, ldc, bs, batch);
        else
            zgemm_pipe_launch<32, true, true>(st, M, N, K, alpha, A, lda, B, ldb, C0, ldc0, C, ldc, bs, batch);
    } else {
        if (tiles64 >= sm_count() && M > 32)
            zgemm_pipe_launch<64, false, true>(st, M, N, K, alpha, A, lda, B, ldb, C0, ldc0, C, ldc, bs, batch);
        else
            zgemm_pipe_launch<32, false, true>(st, M, N, K, alpha, A, lda, B, ldb, C0, ldc0, C, ldc, bs, batch);
    }
}

void cgemm2(cudaStream_t st, int M, int N, int K, const CgemmTerm& a, const CgemmTerm* b, const double2* C0,
            int64_t ldc0, int64_t sC0, double2* C, int64_t ldc, int64_t sC, int batch) {
    if (batch <= 0) return;
    require(batch <= 65535, "cgemm2: batch above 65535");
    auto conv = [](const CgemmTerm& t) {
        Gemm2Term g;
        g.A = t.A;
        g.lda = t.lda;
        g.sA = t.sA;
        g.B = t.B;
        g.ldb = t.ldb;
        g.sB = t.sB;
        g.alpha = t.alpha;
        g.bt = t.bt ? 1 : 0;
        g.lo = t.lo;
        g.hi = t.hi;
        return g;
    };
    const Gemm2Term t0 = conv(a), t1 = b ? conv(*b) : t0;
    // narrow batches (a launch's warps fewer than ~4 per SM): the split-K tile kernel
    // (FWI_CGEMM2_SPLIT=<batch> moves the switch point, 0 disables it)
    static const int split_max = std::getenv("FWI_CGEMM2_SPLIT") ? std::atoi(std::getenv("FWI_CGEMM2_SPLIT")) : 12;
    if (batch <= split_max && K <= 4 * 4 * 32) {
        const dim3 g((N + 7) / 8, (M + 7) / 8, unsigned(batch));
        launch_pdl<kPdlDense>(zgemm2_splitk_tile_kernel, dim3(g), dim3(128), 0, st, M, N, K, t0, t1, b ? 2 : 1, C0,
                              ldc0, sC0, C, ldc, sC);
        CK_LAUNCH();
        return;
    }
    const dim3 g((N + 31) / 32, (M + 7) / 8, unsigned(batch));
    // FWI_ZG2=<CH>,<MINB> picks the variant (diagnostics): 8,1 / 4,4 (default) / 4,5 / 2,6
    static const int var = [] {
        const char* e = std::getenv("FWI_ZG2");
        if (!e) return 1;
        const std::string v(e);
        return v == "8,1" ? 0 : v == "4,5" ? 2 : v == "2,6" ? 3 : 1;
    }();
    auto go = [&](auto kern) {
        launch_pdl<kPdlDense>(kern, g, dim3(128), 0, st, M, N, K, t0, t1, b ? 2 : 1, C0, ldc0, sC0, C, ldc, sC);
    };
    if (var == 0)
        go(zgemm2_warp_kernel<8, 1>);
    else if (var == 2)
        go(zgemm2_warp_kernel<4, 5>);
    else if (var == 3)
        go(zgemm2_warp_kernel<2, 6>);
    else
        go(zgemm2_warp_kernel<4, 4>);
    CK_LAUNCH();
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

void dense_sweep_twisted(cudaStream_t st, cudaStream_t st2, cudaEvent_t fork, cudaEvent_t join, int L, int m, int nb,
                         int nrhs, const double2* G, int64_t gp, const double2* coup, double2* W, double2* T,
                         double2* T2) {
    const int64_t blk = int64_t(nrhs) * nb;
    const int nbk = blocks_for(blk);
    auto Gl = [&](int i) { return G + int64_t(i) * nb * gp; };
    auto cl = [&](int i) { return coup + int64_t(i) * nb; };  // lines i, i+1
    CK(cudaEventRecord(fork, st));
    CK(cudaStreamWaitEvent(st2, fork, 0));
    // launches alternate between the chains (a full launch queue would otherwise
    // serialise them)
    const int R = std::max(m, L - 1 - m);
    for (int r = 0; r < R; ++r) {
        if (r < m) {  // top, forward: y_i = G_i (b_i - E_{i-1} y_{i-1})
            const int i = r;
            sweep_prologue<<<nbk, 256, 0, st>>>(nb, nrhs, W + i * blk, i > 0 ? cl(i - 1) : nullptr,
                                                i > 0 ? W + (i - 1) * blk : nullptr, T);
            CK_LAUNCH();
            cgemm_launch<true>(st, nrhs, nb, nb, 1.0, T, nb, Gl(i), gp, nullptr, 0, W + i * blk, nb);
        }
        const int i = L - 1 - r;
        if (i > m) {  // bottom, forward: y_i = G_i (b_i - E_i y_{i+1})
            sweep_prologue<<<nbk, 256, 0, st2>>>(nb, nrhs, W + i * blk, i < L - 1 ? cl(i) : nullptr,
                                                 i < L - 1 ? W + (i + 1) * blk : nullptr, T2);
            CK_LAUNCH();
            cgemm_launch<true>(st2, nrhs, nb, nb, 1.0, T2, nb, Gl(i), gp, nullptr, 0, W + i * blk, nb);
        }
    }
    CK(cudaEventRecord(join, st2));
    CK(cudaStreamWaitEvent(st, join, 0));
    // middle: x_m = G_m (b_m - E_{m-1} y_{m-1} - E_m y_{m+1})
    sweep_middle<<<nbk, 256, 0, st>>>(nb, nrhs, W + m * blk, cl(m - 1), W + (m - 1) * blk, cl(m), W + (m + 1) * blk, T);
    CK_LAUNCH();
    cgemm_launch<true>(st, nrhs, nb, nb, 1.0, T, nb, Gl(m), gp, nullptr, 0, W + m * blk, nb);
    CK(cudaEventRecord(fork, st));
    CK(cudaStreamWaitEvent(st2, fork, 0));
    for (int r = 0; r < R; ++r) {
        const int it = m - 1 - r, ib = m + 1 + r;
        if (it >= 0) {  // top, backward: x_i = y_i - G_i (E_i x_{i+1})
            sweep_prologue<<<nbk, 256, 0, st>>>(nb, nrhs, nullptr, cl(it), W + (it + 1) * blk, T);
            CK_LAUNCH();
            cgemm_launch<true>(st, nrhs, nb, nb, -1.0, T, nb, Gl(it), gp, W + it * blk, nb, W + it * blk, nb);
        }
        if (ib < L) {  // bottom, backward: x_i = y_i - G_i (E_{i-1} x_{i-1})
            sweep_prologue<<<nbk, 256, 0, st2>>>(nb, nrhs, nullptr, cl(ib - 1), W + (ib - 1) * blk, T2);
            CK_LAUNCH();
            cgemm_launch<true>(st2, nrhs, nb, nb, -1.0, T2, nb, Gl(ib), gp, W + ib * blk, nb, W + ib * blk, nb);
        }
    }
    CK(cudaEventRecord(join, st2));
    CK(cudaStreamWaitEvent(st, join, 0));
}

}  // namespace fwi_b200
