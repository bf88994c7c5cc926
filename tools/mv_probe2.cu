// Latency decomposition for 8-element complex dot products in one warp.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void cmac(double2& c, const double2 g, const double2 x) {
    c.x = fma(g.x, x.x, c.x);
    c.y = fma(g.x, x.y, c.y);
    c.x = fma(-g.y, x.y, c.x);
    c.y = fma(g.y, x.x, c.y);
}

template <int MODE>
__global__ void probe(double2* out, long long* cyc, int iters) {
    __shared__ double2 G[8 * 65 + 8];
    __shared__ double2 wv[72];
    const int lane = threadIdx.x & 31;
    for (int t = threadIdx.x; t < 8 * 65; t += blockDim.x) G[t] = make_double2(t * 1e-3, 1.0 - t * 1e-3);
    for (int t = threadIdx.x; t < 72; t += blockDim.x) wv[t] = make_double2(1.0 / (t + 1), 0.5);
    __syncthreads();
    const int row = lane & 3, cls = lane >> 2;
    const double2* g = G + row * 65 + cls;
    double2 tot = make_double2(0, 0);
    double2 gr[8], xr[8];
    for (int u = 0; u < 8; ++u) { gr[u] = g[u * 8]; xr[u] = wv[cls + u * 8]; }
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const double2* x = wv + cls + (it & 1);
        double2 acc[2] = {make_double2(0, 0), make_double2(0, 0)};
        if (MODE == 0) {  // loads + fma
            double2 gv[8], xv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) { gv[u] = g[u * 8]; xv[u] = x[u * 8]; }
#pragma unroll
            for (int u = 0; u < 8; ++u) cmac(acc[u & 1], gv[u], xv[u]);
        } else if (MODE == 1) {  // loads only (sum one component)
            double2 gv[8], xv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) { gv[u] = g[u * 8]; xv[u] = x[u * 8]; }
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[u & 1].x += gv[u].x + xv[u].y;
        } else if (MODE == 2) {  // fma only from registers (x depends on it)
            const double s = tot.x * 1e-300;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                double2 xv = make_double2(xr[u].x + s, xr[u].y);
                cmac(acc[u & 1], gr[u], xv);
            }
        } else if (MODE == 3) {  // 4 accumulators
            double2 gv[8], xv[8];
            double2 a4[4] = {make_double2(0, 0), make_double2(0, 0), make_double2(0, 0), make_double2(0, 0)};
#pragma unroll
            for (int u = 0; u < 8; ++u) { gv[u] = g[u * 8]; xv[u] = x[u * 8]; }
#pragma unroll
            for (int u = 0; u < 8; ++u) cmac(a4[u & 3], gv[u], xv[u]);
            acc[0] = make_double2(a4[0].x + a4[2].x, a4[0].y + a4[2].y);
            acc[1] = make_double2(a4[1].x + a4[3].x, a4[1].y + a4[3].y);
        }
        double2 v = make_double2(acc[0].x + acc[1].x, acc[0].y + acc[1].y);
        tot.x += v.x;
        tot.y += v.y;
    }
    long long t1 = clock64();
    out[threadIdx.x] = tot;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    double2* o;
    long long* c;
    cudaMalloc(&o, 1 << 20);
    cudaMalloc(&c, 8);
    long long h;
    const char* names[] = {"loads+cmac", "loads only", "cmac only (regs)", "loads+cmac 4 acc"};
#define RUN(M)                                                          \
    probe<M><<<1, 32>>>(o, c, 1000);                                   \
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);                      \
    printf("%-20s %.0f cyc/iter\n", names[M], h / 1000.0);
    RUN(0) RUN(1) RUN(2) RUN(3)
    return 0;
}
