// TMA read-throughput probe: persistent CTAs stream 4-D boxes of a 3-D field
// [K][nz][nx] complex128 (viewed as (8-complex groups, x/8, z, k)) through an
// S-stage mbarrier pipeline, mimicking the KKT apply's loads without compute.
// Reports aggregate GB/s for several box heights / CTA counts. Not product code.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t sa(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

template <int S>
__global__ void __launch_bounds__(256, 1) probe(const __grid_constant__ CUtensorMap tm, int nsteps, int tiles_x,
                                               int tiles_z, int rows, int K, uint32_t box_bytes, double* sink,
                                               int order) {
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + S * box_bytes);
    const int tid = threadIdx.x;
    auto issue = [&](int j) {
        const int g = blockIdx.x + j * gridDim.x;  // global step id
        const int nt = tiles_x * tiles_z;
        const int k = order ? (g / nt) % K : g % K, t = order ? g % nt : (g / K) % nt;
        const int tx = t % tiles_x, tz = t / tiles_x;
        const int s = j % S;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[s])), "r"(box_bytes) : "memory");
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                     ::"r"(sa(sm + s * box_bytes)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(tx * 16), "r"(tz * rows), "r"(k),
                     "r"(sa(&bar[s])) : "memory");
    };
    if (tid == 0) {
        for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int j = 0; j < S && j < nsteps; ++j) issue(j);
    }
    __syncthreads();
    double acc = 0;
    for (int j = 0; j < nsteps; ++j) {
        const int s = j % S;
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(sa(&bar[s])), "r"((j / S) & 1) : "memory");
        acc += reinterpret_cast<const double*>(sm + s * box_bytes)[tid];
        __syncthreads();
        if (tid == 0 && j + S < nsteps) issue(j + S);
    }
    if (acc == 1234.5) sink[0] = acc;
}

int main() {
    const int nx = 512, nz = 256, K = 64;
    const size_t n = size_t(nx) * nz * K;
    double* f; cudaMalloc(&f, n * 16); cudaMemset(f, 0, n * 16);
    double* sink; cudaMalloc(&sink, 8);
    void* fn = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int order : {0, 1}) for (int rows : {8, 10}) for (int ctas_per_sm : {1, 2}) {
        CUtensorMap tm;
        cuuint64_t dims[4] = {16, cuuint64_t(nx / 8), cuuint64_t(nz), cuuint64_t(K)};
        cuuint64_t str[3] = {128, cuuint64_t(nx) * 16, cuuint64_t(nx) * nz * 16};
        cuuint32_t box[4] = {16, 16, cuuint32_t(rows), 1};
        cuuint32_t es[4] = {1, 1, 1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, f, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const uint32_t bb = 16 * 16 * rows * 8;
        const int S = 4;
        const size_t smem = S * bb + 64;
        cudaFuncSetAttribute(probe<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        const int grid = sms * ctas_per_sm;
        const int tiles_x = nx / 128, tiles_z = nz / rows;
        const long total_steps = long(tiles_x) * tiles_z * K * 4;  // 4 passes over the field
        const int nsteps = int(total_steps / grid);
        probe<4><<<grid, 256, smem>>>(tm, nsteps, tiles_x, tiles_z, rows, K, bb, sink, order);
        cudaEventRecord(e0);
        probe<4><<<grid, 256, smem>>>(tm, nsteps, tiles_x, tiles_z, rows, K, bb, sink, order);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = double(nsteps) * grid * bb;
        printf("order %s box 128x%-2d  ctas/SM %d  stage %6u B: %.3f ms  %.0f GB/s  (%s)\n", order ? "same-k" : "k-fastest", rows, ctas_per_sm, bb, ms,
               bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        (void)0;
    }
    return 0;
}
