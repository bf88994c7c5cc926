// Latency/throughput probe for FP64 on sm_100a (diagnostics for the exact sweep design).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_dfma(double* out, long long* cyc, int n, double a, double b) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, a, b);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_dadd(double* out, long long* cyc, int n, double a) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = x + a;
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// throughput: 8 independent chains per thread
__global__ void thr_dfma(double* out, long long* cyc, int n, double a, double b) {
    double x[8];
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    long long t1 = clock64();
    double s = 0;
    for (int k = 0; k < 8; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lat_lds(double* out, long long* cyc, int n) {
    __shared__ int idx[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i + 1) & 1023;
    __syncthreads();
    int j = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) j = idx[j];
    long long t1 = clock64();
    out[threadIdx.x] = j;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    double* o;
    long long* c;
    cudaMalloc(&o, 1 << 24);
    cudaMalloc(&c, 8);
    long long h;
    const int n = 4096;
    for (int w : {32, 64, 128, 256}) {
        lat_dfma<<<1, w>>>(o, c, n, 1.0000001, 1e-9);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("DFMA dependent latency (block %d): %.1f cyc\n", w, double(h) / n);
    }
    lat_dadd<<<1, 32>>>(o, c, n, 1e-9);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DADD dependent latency: %.1f cyc\n", double(h) / n);
    lat_lds<<<1, 32>>>(o, c, n);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("LDS dependent latency: %.1f cyc\n", double(h) / n);
    for (int w : {32, 128, 256, 512, 1024}) {
        thr_dfma<<<1, w>>>(o, c, n, 1.0000001, 1e-9);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("DFMA throughput (1 CTA x %d thr): %.2f DFMA/cyc/SM\n", w, double(n) * 8 * w / double(h));
    }
    return 0;
}
