// Correctness + timing of the long-line solver's complex GEMM variants (dense.cu):
// compares the DMMA kernel with the SIMT kernel on random data.
#include <cmath>
#include <cstdio>
#include <cstdlib>
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

static void run(bool bt, int M, int N, int K, double alpha, bool c0) {
    std::vector<double2> hA(size_t(M) * K), hB(size_t(K) * N), hC0(size_t(M) * N);
    srand(1);
    auto rnd = [] { return double(rand()) / RAND_MAX - 0.5; };
    for (auto& v : hA) v = make_double2(rnd(), rnd());
    for (auto& v : hB) v = make_double2(rnd(), rnd());
    for (auto& v : hC0) v = make_double2(rnd(), rnd());
    double2 *A, *B, *C0, *C;
    cudaMalloc(&A, hA.size() * 16);
    cudaMalloc(&B, hB.size() * 16);
    cudaMalloc(&C0, hC0.size() * 16);
    cudaMalloc(&C, hC0.size() * 16);
    cudaMemcpy(A, hA.data(), hA.size() * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(B, hB.data(), hB.size() * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(C0, hC0.data(), hC0.size() * 16, cudaMemcpyHostToDevice);
    const int64_t ldb = bt ? K : N;
    cudaStream_t st;
    cudaStreamCreate(&st);
    // reference on the host (double accumulation, natural order)
    std::vector<double2> ref(size_t(M) * N);
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double re = 0, im = 0;
            for (int k = 0; k < K; ++k) {
                const double2 a = hA[size_t(m) * K + k];
                const double2 b = bt ? hB[size_t(n) * K + k] : hB[size_t(k) * N + n];
                re += a.x * b.x - a.y * b.y;
                im += a.x * b.y + a.y * b.x;
            }
            ref[size_t(m) * N + n] = make_double2(alpha * re + (c0 ? hC0[size_t(m) * N + n].x : 0),
                                                  alpha * im + (c0 ? hC0[size_t(m) * N + n].y : 0));
        }
    cgemm(st, bt, M, N, K, alpha, A, K, B, ldb, c0 ? C0 : nullptr, N, C, N);
    cudaStreamSynchronize(st);
    std::vector<double2> got(ref.size());
    cudaMemcpy(got.data(), C, got.size() * 16, cudaMemcpyDeviceToHost);
    double num = 0, den = 0;
    for (size_t i = 0; i < got.size(); ++i) {
        num += std::pow(got[i].x - ref[i].x, 2) + std::pow(got[i].y - ref[i].y, 2);
        den += ref[i].x * ref[i].x + ref[i].y * ref[i].y;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int reps = 20;
    cudaEventRecord(e0, st);
    for (int i = 0; i < reps; ++i) cgemm(st, bt, M, N, K, alpha, A, K, B, ldb, c0 ? C0 : nullptr, N, C, N);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / reps;
    printf("%s M=%d N=%d K=%d alpha=%g C0=%d: rel err %.2e   %.1f us  %.2f TFLOP/s\n", bt ? "NT" : "NN", M, N, K,
           alpha, c0, std::sqrt(num / den), us, 8.0 * M * N * K / (us * 1e-6) / 1e12);
    cudaFree(A);
    cudaFree(B);
    cudaFree(C0);
    cudaFree(C);
}

int main() {
    run(true, 256, 1024, 1024, 1.0, false);
    run(true, 256, 1024, 1024, -1.0, true);
    run(false, 1024, 1024, 64, -1.0, true);
    run(false, 64, 1024, 64, 1.0, false);
    run(true, 37, 70, 45, -1.0, true);
    run(false, 70, 37, 45, 1.0, false);
    run(true, 1024, 1024, 256, -1.0, true);   // 64-row tiles
    run(true, 150, 200, 75, 1.0, true);       // ragged
    run(false, 1030, 1000, 70, -1.0, true);   // ragged, 64-row tiles
    return 0;
}
