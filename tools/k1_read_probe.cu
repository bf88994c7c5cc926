// Read-path probe for the tile-TMA KKT apply (K1): persistent CTAs stream the
// K1 stage pattern — du and la boxes with a one-node halo, u without — of three
// distinct K x nz x nx complex128 fields (C2 shape) through an S-stage
// mbarrier ring, no arithmetic, no stores. Sweeps tile height, halo, stages
// and CTAs per SM to find which shape of the read path reaches the streaming
// rate (tools/stream_probe: ~6.7 TB/s for three plain read streams).
// Reports algorithmic GB/s (3 x 16 B per node and source). Not product code.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t sa(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

struct Args {
    int tiles_x, tiles_z, rows, K, KC, S, halo, gr;
    uint32_t hb, ub, stage, tx;
    double* sink;
};

__global__ void __launch_bounds__(512, 1) probe(const __grid_constant__ CUtensorMap tdu, const __grid_constant__ CUtensorMap tla,
                                               const __grid_constant__ CUtensorMap tu, const Args a) {
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + a.S * a.stage);
    const int tid = threadIdx.x;
    const int T = a.tiles_x * a.tiles_z, C = a.K / a.KC, U = T * C;
    const int nunits = (U - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int nsteps = nunits * a.KC;
    auto issue = [&](int j) {
        const int u = blockIdx.x + (j / a.KC) * gridDim.x;
        const int t = u % T, c = u / T;
        const int k = c * a.KC + j % a.KC;
        const int tx = t % a.tiles_x, tz = t / a.tiles_x;
        const int s = j % a.S;
        unsigned char* st = sm + s * a.stage;
        const int gx = tx * (128 / a.gr) - (a.halo ? 1 : 0), gz = tz * a.rows - (a.halo ? 1 : 0);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[s])), "r"(a.tx) : "memory");
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                     ::"r"(sa(st)), "l"(reinterpret_cast<uint64_t>(&tdu)), "r"(0), "r"(gx), "r"(gz), "r"(k), "r"(sa(&bar[s])) : "memory");
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                     ::"r"(sa(st + a.hb)), "l"(reinterpret_cast<uint64_t>(&tla)), "r"(0), "r"(gx), "r"(gz), "r"(k), "r"(sa(&bar[s])) : "memory");
        asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                     ::"r"(sa(st + 2 * a.hb)), "l"(reinterpret_cast<uint64_t>(&tu)), "r"(0), "r"(tx * (128 / a.gr)), "r"(tz * a.rows), "r"(k), "r"(sa(&bar[s])) : "memory");
    };
    if (tid == 0) {
        for (int s = 0; s < a.S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int j = 0; j < a.S && j < nsteps; ++j) issue(j);
    }
    __syncthreads();
    double acc = 0;
    for (int j = 0; j < nsteps; ++j) {
        const int s = j % a.S;
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(sa(&bar[s])), "r"((j / a.S) & 1) : "memory");
        acc += reinterpret_cast<const double*>(sm + s * a.stage)[tid];
        __syncthreads();
        if (tid == 0 && j + a.S < nsteps) issue(j + a.S);
    }
    if (acc == 1234.5) a.sink[0] = acc;
}

static PFN_cuTensorMapEncodeTiled_v12000 enc;

static void mk(CUtensorMap* tm, void* base, int nx, int nz, int K, int gr, int box_groups, int box_rows) {
    cuuint64_t dims[4] = {cuuint64_t(2 * gr), cuuint64_t(nx / gr), cuuint64_t(nz), cuuint64_t(K)};
    cuuint64_t str[3] = {cuuint64_t(gr) * 16, cuuint64_t(nx) * 16, cuuint64_t(nx) * nz * 16};
    cuuint32_t box[4] = {cuuint32_t(2 * gr), cuuint32_t(box_groups), cuuint32_t(box_rows), 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", int(r));
}

int main() {
    const int nx = 512, nz = 256, K = 64;
    const size_t m = size_t(nx) * nz * K;
    double *du, *la, *u, *sink;
    cudaMalloc(&du, m * 16); cudaMalloc(&la, m * 16); cudaMalloc(&u, m * 16); cudaMalloc(&sink, 8);
    cudaMemset(du, 0, m * 16); cudaMemset(la, 0, m * 16); cudaMemset(u, 0, m * 16);
    void* fn = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int gr = 8;
    struct Cfg { int rows, halo, S, cps, KC; };
    const Cfg cfgs[] = {{8, 1, 2, 1, 8}, {8, 0, 2, 1, 8}, {8, 1, 3, 1, 8}, {8, 0, 3, 1, 8}, {8, 0, 4, 1, 8},
                        {16, 1, 2, 1, 8}, {16, 0, 2, 1, 8}, {4, 1, 4, 1, 8}, {4, 0, 4, 1, 8}, {4, 1, 2, 2, 8},
                        {8, 1, 1, 2, 8}, {4, 1, 6, 1, 8}, {8, 1, 2, 1, 64}, {8, 0, 2, 1, 64}};
    for (const Cfg& c : cfgs) {
        const int bh = c.rows + (c.halo ? 2 : 0), bg = 128 / gr + (c.halo ? 2 : 0);
        CUtensorMap tdu, tla, tu;
        mk(&tdu, du, nx, nz, K, gr, bg, bh);
        mk(&tla, la, nx, nz, K, gr, bg, bh);
        mk(&tu, u, nx, nz, K, gr, 128 / gr, c.rows);
        Args a;
        a.tiles_x = nx / 128; a.tiles_z = nz / c.rows; a.rows = c.rows; a.K = K; a.KC = c.KC; a.S = c.S;
        a.halo = c.halo; a.gr = gr; a.sink = sink;
        a.hb = uint32_t((bg * gr * 16 * bh + 127) / 128 * 128);
        a.ub = uint32_t(128 * 16 * c.rows);
        a.stage = 2 * a.hb + a.ub;
        a.tx = uint32_t(2 * bg * gr * 16 * bh + 128 * 16 * c.rows);
        const size_t smem = size_t(c.S) * a.stage + 64;
        if (smem > 227 * 1024 / c.cps) { printf("rows %2d halo %d S %d ctas/SM %d: smem %zu too big\n", c.rows, c.halo, c.S, c.cps, smem); continue; }
        cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        const int grid = sms * c.cps;
        for (int w = 0; w < 3; ++w) probe<<<grid, 512 / c.cps, smem>>>(tdu, tla, tu, a);
        cudaEventRecord(e0);
        const int reps = 20;
        for (int w = 0; w < reps; ++w) probe<<<grid, 512 / c.cps, smem>>>(tdu, tla, tu, a);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
        printf("rows %2d halo %d S %d ctas/SM %d KC %2d stage %6u B: %.4f ms  %5.0f GB/s algorithmic  (%s)\n", c.rows, c.halo,
               c.S, c.cps, c.KC, a.stage, ms, 3.0 * m * 16 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
