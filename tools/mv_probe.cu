// Latency probe: one warp runs the exact-sweep matvec section (R=4 rows x 8 classes,
// nb=64, interleaved columns, butterfly) repeatedly from shared memory.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void cmac(double2& c, const double2 g, const double2 x) {
    c.x = fma(g.x, x.x, c.x);
    c.y = fma(g.x, x.y, c.y);
    c.x = fma(-g.y, x.y, c.x);
    c.y = fma(g.y, x.x, c.y);
}

template <int MODE>
__global__ void probe(double2* out, long long* cyc, int iters, int nb, int Rp) {
    __shared__ double2 G[8 * 65 + 8];
    __shared__ double2 wv[72];
    const int lane = threadIdx.x & 31;
    for (int t = threadIdx.x; t < 8 * 65; t += blockDim.x) G[t] = make_double2(t * 1e-3, 1.0 - t * 1e-3);
    for (int t = threadIdx.x; t < 72; t += blockDim.x) wv[t] = make_double2(1.0 / (t + 1), 0.5);
    __syncthreads();
    const int ncls = 32 / Rp, row = lane & (Rp - 1), cls = lane / Rp, gp = nb + 1;
    const int nj = (nb - cls + ncls - 1) / ncls;
    double2 tot = make_double2(0, 0);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        double2 acc[2] = {make_double2(0, 0), make_double2(0, 0)};
        const double2* g = G + row * gp + cls;
        const double2* x = wv + cls;
        int t = 0;
#pragma unroll 2
        for (; t + 4 <= nj; t += 4) {
            double2 gv[4], xv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                gv[u] = g[(t + u) * ncls];
                xv[u] = x[(t + u) * ncls];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) cmac(acc[u & 1], gv[u], xv[u]);
        }
        for (; t < nj; ++t) cmac(acc[0], g[t * ncls], x[t * ncls]);
        double2 v = make_double2(acc[0].x + acc[1].x, acc[0].y + acc[1].y);
        if (MODE == 1) {
            for (int off = Rp; off < 32; off <<= 1) {
                v.x += __shfl_xor_sync(0xffffffffu, v.x, off);
                v.y += __shfl_xor_sync(0xffffffffu, v.y, off);
            }
        }
        // feed back so iterations serialise like line steps
        if (lane == 0) wv[it & 63] = v;
        __syncwarp();
        tot.x += v.x;
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
    for (int Rp : {4, 8}) {
        probe<0><<<1, 32>>>(o, c, 1000, 64, Rp);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("Rp=%d matvec only: %.0f cyc/iter\n", Rp, h / 1000.0);
        probe<1><<<1, 32>>>(o, c, 1000, 64, Rp);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("Rp=%d matvec+butterfly: %.0f cyc/iter\n", Rp, h / 1000.0);
    }
    return 0;
}
