// Latency of the ILU phase-B chain (diagnostics): one warp, `lanes` active lanes, each
// subtracts `ne` complex products from shared memory in order (2 dependent DADD chains).
#include <cstdio>
#include <cuda_runtime.h>

template <int NE>
__global__ void chain(double2* out, long long* cyc, int lanes, int reps) {
    __shared__ double2 prod[32 * 64];
    for (int i = threadIdx.x; i < 32 * 64; i += blockDim.x) prod[i] = make_double2(1e-3 * i, -2e-3 * i);
    __syncthreads();
    double2 s = make_double2(threadIdx.x, 1.0);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        if (threadIdx.x < lanes) {
            const double2* p = prod + threadIdx.x * 64 + (r & 7);
#pragma unroll
            for (int u = 0; u < NE; ++u) {
                const double2 t = p[u];
                s.x = __dsub_rn(s.x, t.x);
                s.y = __dsub_rn(s.y, t.y);
            }
        }
        __syncwarp();
    }
    long long t1 = clock64();
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    double2* o;
    long long* c;
    cudaMalloc(&o, 1 << 16);
    cudaMalloc(&c, 8);
    long long h;
    const int reps = 1000;
    for (int lanes : {1, 6, 32}) {
        chain<8><<<1, 32>>>(o, c, lanes, reps);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("lanes %2d  8 entries: %.1f cyc/rep (%.1f per entry)\n", lanes, double(h) / reps, double(h) / reps / 8);
        chain<40><<<1, 32>>>(o, c, lanes, reps);
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("lanes %2d 40 entries: %.1f cyc/rep (%.1f per entry)\n", lanes, double(h) / reps, double(h) / reps / 40);
    }
    return 0;
}
