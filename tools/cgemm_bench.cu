// Standalone timing of the long-line solver's FP64 complex GEMM (dense.cu) at the
// config-5 shapes: sweep step (256 x 1024 x 1024, B transposed) and the block
// Gauss-Jordan update (1024 x 1024 x 64).
#include <cstdio>
#include <vector>

#include "../paper_2204_06489_b200/csrc/dense.cu"

namespace fwi_b200 {
int sm_count() {
    static int n = 0;
    if (!n) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, 0);
    return n;
}
}  // namespace fwi_b200

using namespace fwi_b200;

static double bench(bool bt, int M, int N, int K, int reps) {
    double2 *A, *B, *C;
    cudaMalloc(&A, sizeof(double2) * size_t(M) * K);
    cudaMalloc(&B, sizeof(double2) * size_t(K) * N);
    cudaMalloc(&C, sizeof(double2) * size_t(M) * N);
    cudaMemset(A, 0, sizeof(double2) * size_t(M) * K);
    cudaMemset(B, 0, sizeof(double2) * size_t(K) * N);
    cudaStream_t st;
    cudaStreamCreate(&st);
    const int64_t ldb = bt ? K : N;
    for (int i = 0; i < 3; ++i) cgemm(st, bt, M, N, K, 1.0, A, K, B, ldb, nullptr, 0, C, N);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    for (int i = 0; i < reps; ++i) cgemm(st, bt, M, N, K, 1.0, A, K, B, ldb, nullptr, 0, C, N);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / reps;
    const double tf = 8.0 * M * N * K / (us * 1e-6) / 1e12;
    printf("cgemm %s M=%d N=%d K=%d: %.1f us  %.2f TFLOP/s\n", bt ? "NT" : "NN", M, N, K, us, tf);
    cudaFree(A);
    cudaFree(B);
    cudaFree(C);
    return tf;
}

int main() {
    bench(true, 256, 1024, 1024, 50);   // C5 sweep step
    bench(true, 512, 1024, 1024, 50);   // two sweep steps batched (twisted sweep, one launch)
    bench(true, 1024, 1024, 1024, 20);  // large
    bench(false, 1024, 1024, 64, 100);  // C5 Gauss-Jordan update
    bench(false, 64, 1024, 64, 100);    // D^{-1} row block
    bench(true, 48, 128, 128, 200);     // C3-sized (dense path forced)
    return 0;
}
