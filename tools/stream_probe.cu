// Memory-system probe: the byte mix of the C2 KKT apply (3 reads + 2 writes of
// K*n complex128 per apply) as plain streaming loops, to find the ceiling the
// tiled TMA kernel should be compared with. Not part of the product.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void mix(const double2* __restrict__ a, const double2* __restrict__ b, const double2* __restrict__ c,
                    double2* __restrict__ o1, double2* __restrict__ o2, long m) {
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < m; i += long(gridDim.x) * blockDim.x) {
        const double2 x = a[i], y = b[i], z = c[i];
        o1[i] = make_double2(x.x + z.x, x.y + z.y);
        o2[i] = make_double2(y.x - z.x, y.y - z.y);
    }
}
__global__ void rd(const double2* __restrict__ a, const double2* __restrict__ b, const double2* __restrict__ c,
                   double2* __restrict__ o, long m) {
    double s = 0;
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < m; i += long(gridDim.x) * blockDim.x) {
        const double2 x = a[i], y = b[i], z = c[i];
        s += x.x + y.y + z.x;
    }
    if (s == 12345.678) o[0] = make_double2(s, s);
}
__global__ void wr(double2* __restrict__ o1, double2* __restrict__ o2, long m) {
    for (long i = blockIdx.x * long(blockDim.x) + threadIdx.x; i < m; i += long(gridDim.x) * blockDim.x) {
        o1[i] = make_double2(1.0, 2.0);
        o2[i] = make_double2(3.0, 4.0);
    }
}

int main() {
    const long m = 64L * 131072;  // K*n
    double2 *a, *b, *c, *o1, *o2;
    cudaMalloc(&a, m * 16); cudaMalloc(&b, m * 16); cudaMalloc(&c, m * 16);
    cudaMalloc(&o1, m * 16); cudaMalloc(&o2, m * 16);
    cudaMemset(a, 0, m * 16); cudaMemset(b, 0, m * 16); cudaMemset(c, 0, m * 16);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    // (grid, block): one 512-thread CTA per SM is the source-major K1's shape
    int grids[][2] = {{148, 512}, {144, 512}, {296, 512}, {148, 1024}, {148 * 4, 256}, {148 * 8, 256},
                      {148 * 16, 256}, {148 * 32, 256}};
    for (auto& gb : grids) {
        const int g = gb[0], bs = gb[1];
        for (int rep = 0; rep < 3; ++rep) mix<<<g, bs>>>(a, b, c, o1, o2, m);
        cudaEventRecord(e0);
        for (int rep = 0; rep < 20; ++rep) mix<<<g, bs>>>(a, b, c, o1, o2, m);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 20;
        printf("mix3r2w grid %5d x %4d: %.4f ms  %.0f GB/s\n", g, bs, ms, 5.0 * m * 16 / ms / 1e6);
        cudaEventRecord(e0);
        for (int rep = 0; rep < 20; ++rep) rd<<<g, bs>>>(a, b, c, o1, m);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1); ms /= 20;
        printf("read3     grid %5d: %.4f ms  %.0f GB/s\n", g, ms, 3.0 * m * 16 / ms / 1e6);
        cudaEventRecord(e0);
        for (int rep = 0; rep < 20; ++rep) wr<<<g, bs>>>(o1, o2, m);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1); ms /= 20;
        printf("write2    grid %5d: %.4f ms  %.0f GB/s\n", g, ms, 2.0 * m * 16 / ms / 1e6);
    }
    return 0;
}
