// dense.cuh — whole-GPU dense kernels of the long-line exact solver (dense.cu).
#pragma once

#include <vector>

#include "common.cuh"

namespace fwi_b200 {

constexpr int kDenseBlk = 64;  // Gauss-Jordan block width

// C = (C0 ? C0 : 0) + alpha * A B, complex double; B(k,n) = B[k*ldb+n] or, with bt, B[n*ldb+k]
void cgemm(cudaStream_t st, bool bt, int M, int N, int K, double alpha, const double2* A, int64_t lda,
           const double2* B, int64_t ldb, const double2* C0, int64_t ldc0, double2* C, int64_t ldc);

// strided-batched cgemm: for z < batch, C_z = C0_z + alpha A_z B_z with X_z = X + z sX.
// scratch (scratch_count complex): partial tiles of the split-K form used for few tiles;
// without it the tiled kernel always runs.
void cgemm_batched(cudaStream_t st, bool bt, int M, int N, int K, double alpha, const double2* A, int64_t lda,
                   int64_t sA, const double2* B, int64_t ldb, int64_t sB, const double2* C0, int64_t ldc0,
                   int64_t sC0, double2* C, int64_t ldc, int64_t sC, int batch, double2* scratch = nullptr,
                   size_t scratch_count = 0);

// One term of cgemm2: alpha A_z B_z (B transposed when bt) for batch entries z in [lo, hi),
// the operands at A + (z - lo) sA, B + (z - lo) sB.
struct CgemmTerm {
    const double2* A;
    int64_t lda, sA;
    const double2* B;
    int64_t ldb, sB;
    double alpha;
    bool bt;
    int lo, hi;
};
// C_z = C0_z + term a (+ term b), z < batch: up to two products in one launch (warp tiles)
void cgemm2(cudaStream_t st, int M, int N, int K, const CgemmTerm& a, const CgemmTerm* b, const double2* C0,
            int64_t ldc0, int64_t sC0, double2* C, int64_t ldc, int64_t sC, int batch);

struct DenseWork {
    DevBuf<double2> F, Ablk, R, Dinv;
    int nb_ = 0;
    void ensure(int nb);
};

// A (nb x nb, row pitch lda) <- A^{-1}; block Gauss-Jordan with pivoting inside the
// 64-wide diagonal blocks. A zero pivot sets *status = status_base + column + 1.
void dense_invert(cudaStream_t st, int nb, double2* A, int64_t lda, DenseWork& w, int* status, int status_base);

// Forward/backward line sweeps for nrhs right-hand sides in W[i][k][m] (overwritten
// in place by y, then by the solution); T is nrhs x nb scratch.
// Twisted sweeps (factor built from both ends towards line m): the top chain
// (lines 0..m-1) on st, the bottom chain (L-1..m+1) on st2, then the middle line,
// then both backward chains outwards again. T, T2: nrhs x nb scratch per chain.
void dense_sweep_twisted(cudaStream_t st, cudaStream_t st2, cudaEvent_t fork, cudaEvent_t join, int L, int m, int nb,
                         int nrhs, const double2* G, int64_t gp, const double2* coup, double2* W, double2* T,
                         double2* T2);

void dense_sweep(cudaStream_t st, int L, int nb, int nrhs, const double2* G, int64_t gp, const double2* coup,
                 double2* W, double2* T);

}  // namespace fwi_b200
