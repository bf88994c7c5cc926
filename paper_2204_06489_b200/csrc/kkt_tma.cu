// kkt_tma.cu — K1, the production KKT apply: a persistent, load-balanced,
// TMA-pipelined kernel (same arithmetic as kkt.cu's reference-faithful
// kernel, see there for the operator and the reference citations).
//
// Work decomposition. The grid is cut into G ~= #SMs rectangles of equal area
// (x-strips of <= 128 columns, each split into z-bands), one CTA per SM,
// 512 threads = 128 columns x 4 row slots, two rows per thread. A CTA walks
// its rectangle in sub-tiles of 8 rows and, for each sub-tile, the K sources
// in order; the ds row's K-sum stays in registers, so the complex128 result
// is bit-identical to the reference.
//
// Data movement. For every (sub-tile, k) step one elected thread issues six
// cp.async.bulk.tensor loads into a shared-memory stage: du_k and la_k with a
// one-node halo (two 65-column boxes each, out-of-range halo zero-filled by
// the TMA unit) and u_k (two 64-column boxes), completing on an mbarrier.
// Up to 3-4 stages are in flight, so HBM streams while the FP64 pipes work;
// outputs are written with streaming (evict-first) stores straight from
// registers. Stencil coefficients are loaded once per sub-tile.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <climits>
#include <vector>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "arith.cuh"
#include "ctx.cuh"

namespace fwi_b200 {

namespace {

#ifndef FWI_KKT_THREADS
#define FWI_KKT_THREADS 512
#endif
#ifndef FWI_KKT_COLS
#define FWI_KKT_COLS 128
#endif
constexpr int kThreads = FWI_KKT_THREADS;
constexpr int kCols = FWI_KKT_COLS;                   // tile width (columns)
constexpr int kSlots = kThreads / kCols;              // row slots (2 rows per thread)
constexpr int kColShift = kCols == 256 ? 8 : kCols == 128 ? 7 : kCols == 64 ? 6 : 5;
constexpr int kCtasPerSm = kThreads <= 256 ? 2 : 1;
constexpr int kRows = 2 * kSlots;  // rows per tile
constexpr int kBH = kRows + 2;
constexpr int kMaxStages = 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
        "%4, %5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}

template <class A>
struct TmaArgs {
    using T = typename A::T;
    using R = typename A::R;
    int nx, nz, K;
    int64_t n;
    R w2, eps;
    const T *diag, *east, *south;
    const int *nrec_ptr, *nrec_k;
    const double* nrec_w2;
    const R* ds;
    T *odu, *ola;
    R* ods;
    const int4* tiles;     // x0, w, z0, h   (w <= 128, h <= 8)
    int T_, C;             // tiles, K-chunks (units = T_ * C, chunk-major)
    unsigned* sched;       // [0] next unit, [1] finished CTAs
    unsigned* flags;       // per tile: chunks completed (epoch-based)
    unsigned base;         // epoch * C
    int RP, UP;            // smem row pitch (complex) of the halo tiles / of the u tile
    int stages;
    int memonly;           // diagnostics: move the data, skip the arithmetic
    int nofold;            // diagnostics: skip the ordered ds fold (wrong ds)
    int nostore, nou;      // diagnostics: skip the output stores / the u load
    int gr;                // complex numbers per innermost TMA element group
    uint32_t dub, ub, stage_bytes, tx_bytes, ub_bytes;
};

template <class T>
__device__ __forceinline__ void st_stream(T* p, T v);
template <>
__device__ __forceinline__ void st_stream<double2>(double2* p, double2 v) {
#ifdef FWI_TILE_STCS
    __stcs(p, v);
#else
    // not allocated in the L1 (the chunked kernel's shared memory leaves little of it)
    asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
#endif
}
template <>
__device__ __forceinline__ void st_stream<float2>(float2* p, float2 v) { __stcs(p, v); }

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

constexpr int kRing = 8;

// barrier over the consumer threads only (the producer warp never joins)
template <int WS>
__device__ __forceinline__ void consumer_sync() {
    if (WS == 1)
        asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory");
    else
        __syncthreads();
}

// Units = (tile, chunk of KC sources), claimed dynamically in chunk-major
// order by persistent CTAs. A unit's ds contribution is folded into the
// tile's running partial sum (kept in out.ds) strictly in source order: the
// unit waits for the tile's previous chunk, so the complex128 result stays
// bit-identical to the reference's sequential sum.
// One node, one source: the three block rows of the KKT operator with the
// reference's rounding order. FULL: all four neighbours present (interior
// fast path, no per-term predication).
template <class A, bool FULL>
__device__ __forceinline__ void node_step(const typename A::T* dr, const typename A::T* lr, int RP,
                                          bool hN, bool hW, bool hE, bool hS, typename A::T cD,
                                          typename A::T cN, typename A::T cW, typename A::T cE,
                                          typename A::T cS, typename A::T& s_, typename A::T& t_) {
    using T = typename A::T;
    // Warps that touch the Dirichlet ring (FULL = false) run the same straight-line code on
    // operands selected to +0 where the reference has no stencil entry (the coefficient is +0
    // there too): 0 * 0 = +0 and a running sum that started at +0 is never -0, so s + (+0) == s
    // bit for bit, for non-finite inputs as well — identical to skipping the term, without the
    // four divergent branches (the per-CTA timeline showed the edge strips ending 4 % (complex128)
    // to 11 % (complex64) after the interior ones).
    const T z = A::zero();
    const T dN = (FULL || hN) ? dr[-RP] : z, lN = (FULL || hN) ? lr[-RP] : z;
    const T dW = (FULL || hW) ? dr[-1] : z, lW = (FULL || hW) ? lr[-1] : z;
    const T dE = (FULL || hE) ? dr[1] : z, lE = (FULL || hE) ? lr[1] : z;
    const T dS = (FULL || hS) ? dr[RP] : z, lS = (FULL || hS) ? lr[RP] : z;
    s_ = A::madd(z, cN, dN);
    t_ = A::maddc(z, cN, lN);
    s_ = A::madd(s_, cW, dW);
    t_ = A::maddc(t_, cW, lW);
    s_ = A::madd(s_, cD, dr[0]);
    t_ = A::maddc(t_, cD, lr[0]);
    s_ = A::madd(s_, cE, dE);
    t_ = A::maddc(t_, cE, lE);
    s_ = A::madd(s_, cS, dS);
    t_ = A::maddc(t_, cS, lS);
    (void)sizeof(T);
}

// Units = (tile, chunk of KC sources), claimed dynamically in chunk-major
// order by persistent CTAs. A unit's ds contribution is folded into the
// tile's running partial sum (kept in out.ds) strictly in source order: the
// unit waits for the tile's previous chunk, so the complex128 result stays
// bit-identical to the reference's sequential sum. S (stages) divides KC, so
// stage indices and mbarrier parities are compile-time within a unit.
//
// WS = 1 (warp-specialised): a 17th warp is the producer. It waits on
// per-stage "empty" mbarriers (one arrive per consumer warp) instead of the
// block-wide barrier after every step, and hands the claimed unit id over
// through the stage's "full" mbarrier (release/acquire). The 17th warp caps
// the register budget at 96 per thread (5 warps on one SM sub-partition), so
// it suits the complex64 kernel. WS = 2: same empty barriers, no extra warp —
// thread 0 waits for the stage to drain and refills it, the other warps run
// ahead within the ring. WS = 0: a block barrier after every step.
template <class A, int KC, int S, int WS>
__global__ void __launch_bounds__(WS == 1 ? kThreads + 32 : kThreads, kCtasPerSm)
    kkt_tma_kernel(const __grid_constant__ CUtensorMap tdu, const __grid_constant__ CUtensorMap tla,
                   const __grid_constant__ CUtensorMap tu, const TmaArgs<A> P) {
    static_assert(KC % S == 0, "stages must divide the chunk");
    using T = typename A::T;
    using R = typename A::R;
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + size_t(S) * P.stage_bytes);
    uint64_t* empty = bar + kMaxStages;
    int* ring = reinterpret_cast<int*>(bar + 2 * kMaxStages);
    // this chunk's Re(w^2 conj(u_k) lambda_k) terms, [KC][2][kThreads]
    R* terms = reinterpret_cast<R*>(sm + size_t(S) * P.stage_bytes + 128);
    const int nx = P.nx, nz = P.nz, Tn = P.T_;
    const int U = Tn * P.C;
    const int tid = threadIdx.x, lx = tid & (kCols - 1), zs = tid >> kColShift;
    const int RP = P.RP, UP = P.UP;
    const int64_t n = P.n;

    // producer (thread 0): claims units lazily, issues one step = 3 TMA boxes
    int nclaimed = 0;
    auto issue = [&](int j) -> bool {
        const int qq = j / KC;
        while (nclaimed <= qq) {
            const unsigned u = atomicAdd(P.sched, 1u);
            ring[nclaimed % kRing] = u < unsigned(U) ? int(u) : -1;
            ++nclaimed;
        }
        const int u = ring[qq % kRing];
        if (u < 0) {
            if (WS == 1) mbar_arrive(&bar[j % S]);  // wakes the consumers, who read the end marker
            return false;
        }
        const int t = u % Tn, c = u / Tn;
        const int k = c * KC + j % KC;
        const int4 tl = P.tiles[t];
        const int s = j % S;
        unsigned char* st = sm + size_t(s) * P.stage_bytes;
        mbar_expect_tx(&bar[s], P.nou ? P.tx_bytes - P.ub_bytes : P.tx_bytes);
        // halo tiles start one complex pair (two nodes) left of the tile, so a
        // smem row holds x0-2 .. x0+RP-3
        tma_load_4d(st, &tdu, 0, tl.x / P.gr - 1, tl.z - 1, k, &bar[s]);
        tma_load_4d(st + P.dub, &tla, 0, tl.x / P.gr - 1, tl.z - 1, k, &bar[s]);
        if (!P.nou) tma_load_4d(st + 2 * P.dub, &tu, 0, tl.x / P.gr, tl.z, k, &bar[s]);
        return true;
    };

    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&bar[s], 1);
            if (WS) mbar_init(&empty[s], kThreads / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (WS != 1)
            for (int j = 0; j < S; ++j) issue(j);
    }
    __syncthreads();
    if (WS == 1 && tid >= kThreads) {
        if (tid == kThreads)
            for (int j = 0;; ++j) {
                if (j >= S) mbar_wait(&empty[j % S], ((j / S) - 1) & 1);
                if (!issue(j)) break;
            }
        return;
    }

    for (int q = 0;; ++q) {
        if (WS == 1) mbar_wait(&bar[0], (q * (KC / S)) & 1);  // the unit's first stage carries its id
        const int u = ring[q % kRing];
        if (u < 0) break;
        const int t = u % Tn, c = u / Tn;
        const int4 tl = P.tiles[t];
        const int x0 = tl.x, w = tl.y, zt = tl.z, ht = tl.w;
        const int k0 = c * KC;
        bool act[2], hN[2], hW[2], hE[2], hS[2];
        T cD[2], cN[2], cW[2], cE[2], cS[2];
        R dsv[2];
        int qr[2], qe[2];
        int64_t cnode[2];
        bool full = true;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int row = zs + kSlots * r;
            act[r] = lx < w && row < ht;
            const int ix = x0 + lx, iz = zt + row;
            const int64_t cc = act[r] ? int64_t(iz) * nx + ix : 0;
            cnode[r] = cc;
            const bool bnd = on_boundary(ix, iz, nx, nz);
            hN[r] = act[r] && !bnd && !on_boundary(ix, iz - 1, nx, nz);
            hW[r] = act[r] && !bnd && !on_boundary(ix - 1, iz, nx, nz);
            hE[r] = act[r] && !bnd && !on_boundary(ix + 1, iz, nx, nz);
            hS[r] = act[r] && !bnd && !on_boundary(ix, iz + 1, nx, nz);
            full = full && act[r] && hN[r] && hW[r] && hE[r] && hS[r];
            cD[r] = act[r] ? P.diag[cc] : A::zero();
            cN[r] = hN[r] ? P.south[cc - nx] : A::zero();
            cW[r] = hW[r] ? P.east[cc - 1] : A::zero();
            cE[r] = hE[r] ? P.east[cc] : A::zero();
            cS[r] = hS[r] ? P.south[cc] : A::zero();
            dsv[r] = act[r] ? P.ds[cc] : R(0);
            int qq = act[r] ? P.nrec_ptr[cc] : 0;
            qe[r] = act[r] ? P.nrec_ptr[cc + 1] : 0;
            while (qq < qe[r] && P.nrec_k[qq] < k0) ++qq;
            qr[r] = qq;
        }
        const bool warp_full = __all_sync(0xffffffffu, full);
        const int par0 = (q * (KC / S)) & 1;
#pragma unroll
        for (int kk = 0; kk < KC; ++kk) {
            const int k = k0 + kk;
            constexpr int dummy = 0;
            (void)dummy;
            const int s = kk % S;  // compile-time
            mbar_wait(&bar[s], (par0 + kk / S) & 1);
            const unsigned char* st = sm + size_t(s) * P.stage_bytes;
            const T* dus = reinterpret_cast<const T*>(st) + lx + P.gr;
            const T* las = reinterpret_cast<const T*>(st + P.dub) + lx + P.gr;
            const T* us = reinterpret_cast<const T*>(st + 2 * P.dub) + lx;
            T s_[2], t_[2];
            if (P.memonly) {
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    s_[r] = dus[(zs + kSlots * r + 1) * RP];
                    t_[r] = las[(zs + kSlots * r + 1) * RP];
                }
            } else if (warp_full) {
#pragma unroll
                for (int r = 0; r < 2; ++r)
                    node_step<A, true>(dus + (zs + kSlots * r + 1) * RP, las + (zs + kSlots * r + 1) * RP, RP, true, true,
                                       true, true, cD[r], cN[r], cW[r], cE[r], cS[r], s_[r], t_[r]);
            } else {
#pragma unroll
                for (int r = 0; r < 2; ++r)
                    node_step<A, false>(dus + (zs + kSlots * r + 1) * RP, las + (zs + kSlots * r + 1) * RP, RP, hN[r],
                                        hW[r], hE[r], hS[r], cD[r], cN[r], cW[r], cE[r], cS[r], s_[r], t_[r]);
            }
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int row = zs + kSlots * r;
                const T duc = dus[(row + 1) * RP];
                const T lac = las[(row + 1) * RP];
                const T uc = us[row * UP];
                terms[(kk * 2 + r) * kThreads + tid] = A::re_pconj(P.w2, uc, lac);
                if (!act[r] || P.nostore) continue;
                const int64_t o = int64_t(k) * n + cnode[r];
                st_stream(P.ola + o, A::sub(s_[r], A::pmul(P.w2, uc, dsv[r])));
                T tv = t_[r];
                if (qr[r] < qe[r] && P.nrec_k[qr[r]] == k) {
                    T f = A::zero();
                    while (qr[r] < qe[r] && P.nrec_k[qr[r]] == k) {
                        f = A::add(f, A::rm(R(P.nrec_w2[qr[r]]), duc));
                        ++qr[r];
                    }
                    tv = A::add(f, tv);
                }
                st_stream(P.odu + o, tv);
            }
            if (WS) {
                __syncwarp();
                if ((tid & 31) == 0) mbar_arrive(&empty[s]);  // this warp is done with stage s
                if (WS == 2 && tid == 0) {
                    mbar_wait(&empty[s], (par0 + kk / S) & 1);
                    issue(q * KC + kk + S);
                }
            } else {
                __syncthreads();  // every thread is done with stage s
                if (tid == 0) issue(q * KC + kk + S);
            }
        }
        // fold this chunk into the tile's running ds sum, in source order
        if (tid == 0 && c > 0 && !P.nofold)
            while (ld_acquire(P.flags + t) != P.base + unsigned(c)) __nanosleep(64);
        consumer_sync<WS>();
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            if (!act[r]) continue;
            R pl = c > 0 ? __ldcg(P.ods + cnode[r]) : R(0);
#pragma unroll
            for (int kk = 0; kk < KC; ++kk) pl = A::radd(pl, terms[(kk * 2 + r) * kThreads + tid]);
            P.ods[cnode[r]] = (c == P.C - 1) ? A::rsub(A::rmulr(P.eps, dsv[r]), pl) : pl;
        }
        consumer_sync<WS>();
        if (tid == 0) {
            __threadfence();
            st_release(P.flags + t, P.base + unsigned(c) + 1u);
        }
    }
    // last CTA out resets the scheduler for the next launch
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(P.sched + 1, 1u) == gridDim.x - 1) {
            P.sched[0] = 0u;
            P.sched[1] = 0u;
            __threadfence();
        }
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

uint32_t align128(size_t b) { return uint32_t((b + 127) / 128 * 128); }

}  // namespace

struct KktPlan {
    bool ok = false;
    int G = 0, T = 0, C = 0, KC = 0, RP = 0, UP = 0, stages = 0, gr = 2;
    int ws = 0;  // stage hand-off (kernel WS parameter; FWI_KKT_WS)
    uint32_t dub = 0, ub = 0, stage_bytes = 0, tx_bytes = 0;
    unsigned epoch = 0;
    size_t smem = 0;
    DevBuf<int4> tiles;
    DevBuf<unsigned> sched, flags;
    CUtensorMap tm_u;
};

void kkt_plan_free(KktPlan* p) { delete p; }

namespace {

CUtensorMapL2promotion l2promo() {
    const char* e = std::getenv("FWI_KKT_L2PROMO");
    if (!e) return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    const int v = std::atoi(e);
    return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
         : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
}

// 4-D view of a source-major field: (complex pair, x/2, z, source). Each
// element is 8 bytes: a double (complex128: 4 per pair) or a whole complex64
// (2 per pair; the copy engine does not interpret the payload).
bool encode(CUtensorMap* tm, bool f32, const void* base, int nx, int nz, int K, int gr, int box_pairs,
            int box_rows, int box_sources = 1) {
    auto fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t e = cuuint64_t(gr) * (f32 ? 1 : 2);  // 8-byte elements per group
    const cuuint64_t cb = f32 ? 8 : 16;  // bytes per complex
    cuuint64_t dims[4] = {e, cuuint64_t(nx / gr), cuuint64_t(nz), cuuint64_t(K)};
    cuuint64_t strides[3] = {cuuint64_t(gr) * cb, cuuint64_t(nx) * cb, cuuint64_t(nx) * nz * cb};
    cuuint32_t box[4] = {cuuint32_t(e), cuuint32_t(box_pairs), cuuint32_t(box_rows), cuuint32_t(box_sources)};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = fn(tm, f32 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4,
                          const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, l2promo(),
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <class A, int KC, int S, int WS>
void set_smem(size_t smem) {
    static size_t smem_set = 0;  // per-kernel, process-wide attribute: only ever raise it
    if (smem > smem_set) {
        CK(cudaFuncSetAttribute(kkt_tma_kernel<A, KC, S, WS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                int(smem)));
        smem_set = smem;
    }
}

// (KC, S) instantiations: KC in {1,2,4,8}, S in {1,2,4} with S | KC and S <= KC
#define FWI_KKT_DISPATCH(KCv, Sv, CALL)                      \
    switch (KCv * 16 + Sv) {                                 \
        case 1 * 16 + 1: CALL(1, 1); break;                  \
        case 2 * 16 + 2: CALL(2, 2); break;                  \
        case 4 * 16 + 2: CALL(4, 2); break;                  \
        case 4 * 16 + 4: CALL(4, 4); break;                  \
        case 8 * 16 + 2: CALL(8, 2); break;                  \
        default: CALL(8, 4); break;                          \
    }

template <class A>
KktPlan* build_plan(Ctx& c, bool f32) {
    auto p = std::make_unique<KktPlan>();
    const int nx = c.nx, nz = c.nz, K = c.K;
    const int es = f32 ? 8 : 16;  // bytes per complex
    if (nx % 2 != 0) return p.release();  // pair view needs an even row length
    if (!encode_fn()) return p.release();
    const int nsx = (nx + kCols - 1) / kCols;
    const int W = ((nx + nsx - 1) / nsx + 1) / 2 * 2;  // even strip width <= 128
    // innermost TMA element group: 8 complex (128 B for complex128) measured
    // best on B200 (request size vs. halo width); 2 as the general fallback
    int gr = 8;
    if (const char* e = std::getenv("FWI_KKT_GRP")) gr = std::max(1, std::atoi(e));
    if (nx % gr != 0 || W % gr != 0) gr = 2;
    const int RP = W + 2 * gr, UP = W;  // halo row: x0-gr .. x0+W+gr-1
    p->gr = gr;
    // tiles of <= 128 x 8 nodes, row-block major
    std::vector<int4> tiles;
    for (int z0 = 0; z0 < nz; z0 += kRows)
        for (int sx = 0; sx < nsx; ++sx) {
            const int x0 = sx * W;
            tiles.push_back(make_int4(x0, std::min(W, nx - x0), z0, std::min(kRows, nz - z0)));
        }
    p->T = int(tiles.size());
    // K-chunk per unit: the largest power of two dividing K that still gives every
    // CTA a unit. Smaller chunks do not balance better: a tile's chunks fold in
    // order, and each fold costs a wait (config 3, 48 tiles x K=48: KC=8 58.8 us,
    // KC=4 64.1 us, KC=2 88.5 us per apply; tools/apply_sizes.py)
    const int G0 = sm_count() * kCtasPerSm;
    int kc = 8;
    while (kc > 1 && (K % kc != 0 || int64_t(p->T) * (K / kc) < int64_t(G0))) kc /= 2;
    if (const char* e = std::getenv("FWI_KKT_KC")) {
        const int v = std::atoi(e);
        if ((v == 1 || v == 2 || v == 4 || v == 8) && K % v == 0) kc = v;
    }
    p->KC = kc;
    p->C = K / kc;
    p->G = int(std::min<int64_t>(G0, int64_t(p->T) * p->C));
    p->tiles.alloc(tiles.size());
    CK(cudaMemcpy(p->tiles.p, tiles.data(), tiles.size() * sizeof(int4), cudaMemcpyHostToDevice));
    p->sched.alloc(2);
    p->flags.alloc(tiles.size());
    CK(cudaMemset(p->sched.p, 0, 2 * sizeof(unsigned)));
    CK(cudaMemset(p->flags.p, 0, tiles.size() * sizeof(unsigned)));
    p->RP = RP;
    p->UP = UP;
    p->dub = align128(size_t(RP) * kBH * es);
    p->ub = align128(size_t(UP) * kRows * es);
    p->stage_bytes = 2 * p->dub + p->ub;
    p->tx_bytes = uint32_t(2 * size_t(RP) * kBH * es + size_t(UP) * kRows * es);
    const size_t tail = 128 + size_t(kc) * 2 * kThreads * (f32 ? 4 : 8);  // mbarriers, unit ring, terms
    const size_t budget = (kCtasPerSm == 1 ? 227 * 1024 : 113 * 1024) - tail;
    // four stages when they fit and divide the chunk, else two
    int st = 4;
    if (const char* e = std::getenv("FWI_KKT_STAGES")) st = std::atoi(e) >= 4 ? 4 : 2;
    while (st > 1 && (size_t(st) * p->stage_bytes > budget || kc % st != 0)) st /= 2;
    if (kc == 1) st = 1;
    p->stages = st;
    p->ws = f32 ? 1 : 0;
    if (const char* e = std::getenv("FWI_KKT_WS")) p->ws = std::atoi(e);
    if (size_t(st) * p->stage_bytes > budget) return p.release();
    p->smem = size_t(p->stages) * p->stage_bytes + tail;
#define FWI_SET(KCc, Sc) \
    set_smem<A, KCc, Sc, 0>(p->smem), set_smem<A, KCc, Sc, 1>(p->smem), set_smem<A, KCc, Sc, 2>(p->smem)
    FWI_KKT_DISPATCH(kc, st, FWI_SET)
#undef FWI_SET
    const void* ubase = f32 ? static_cast<const void*>(c.u32.p) : static_cast<const void*>(c.u.p);
    if (!ubase || !encode(&p->tm_u, f32, ubase, nx, nz, K, gr, UP / gr, kRows)) return p.release();
    p->ok = true;
    return p.release();
}

template <class A>
bool launch(Ctx& c, KktPlan* p, const typename A::T* du, const typename A::R* ds, const typename A::T* la,
            typename A::T* odu, typename A::R* ods, typename A::T* ola, bool f32) {
    CUtensorMap tdu, tla;
    if (!encode(&tdu, f32, du, c.nx, c.nz, c.K, p->gr, p->RP / p->gr, kBH)) return false;
    if (!encode(&tla, f32, la, c.nx, c.nz, c.K, p->gr, p->RP / p->gr, kBH)) return false;
    TmaArgs<A> a;
    a.nx = c.nx;
    a.nz = c.nz;
    a.K = c.K;
    a.n = c.n;
    a.w2 = typename A::R(c.w2);
    a.eps = typename A::R(c.eps);
    if (f32) {
        a.diag = reinterpret_cast<const typename A::T*>(c.diag32.p);
        a.east = reinterpret_cast<const typename A::T*>(c.east32.p);
        a.south = reinterpret_cast<const typename A::T*>(c.south32.p);
    } else {
        a.diag = reinterpret_cast<const typename A::T*>(c.diag.p);
        a.east = reinterpret_cast<const typename A::T*>(c.east.p);
        a.south = reinterpret_cast<const typename A::T*>(c.south.p);
    }
    a.nrec_ptr = c.nrec_ptr.p;
    a.nrec_k = c.nrec_k.p;
    a.nrec_w2 = c.nrec_w2.p;
    a.ds = ds;
    a.odu = odu;
    a.ola = ola;
    a.ods = ods;
    a.tiles = p->tiles.p;
    a.T_ = p->T;
    a.C = p->C;
    a.sched = p->sched.p;
    a.flags = p->flags.p;
    ++p->epoch;
    a.base = p->epoch * unsigned(p->C);
    a.RP = p->RP;
    a.UP = p->UP;
    a.stages = p->stages;
    a.memonly = std::getenv("FWI_KKT_MEMONLY") ? 1 : 0;
    a.nofold = std::getenv("FWI_KKT_NOFOLD") ? 1 : 0;
    a.nostore = std::getenv("FWI_KKT_NOSTORE") ? 1 : 0;
    a.nou = std::getenv("FWI_KKT_NOU") ? 1 : 0;
    a.ub_bytes = uint32_t(size_t(p->UP) * kRows * (f32 ? 8 : 16));
    a.gr = p->gr;
    a.dub = p->dub;
    a.ub = p->ub;
    a.stage_bytes = p->stage_bytes;
    a.tx_bytes = p->tx_bytes;
#define FWI_LAUNCH(KCc, Sc)                                                                            \
    (p->ws == 1   ? kkt_tma_kernel<A, KCc, Sc, 1><<<p->G, kThreads + 32, p->smem, c.stream>>>(tdu, tla, p->tm_u, a) \
     : p->ws == 2 ? kkt_tma_kernel<A, KCc, Sc, 2><<<p->G, kThreads, p->smem, c.stream>>>(tdu, tla, p->tm_u, a)      \
                  : kkt_tma_kernel<A, KCc, Sc, 0><<<p->G, kThreads, p->smem, c.stream>>>(tdu, tla, p->tm_u, a))
    FWI_KKT_DISPATCH(p->KC, p->stages, FWI_LAUNCH)
#undef FWI_LAUNCH
    CK_LAUNCH();
    c.kkt_kernel[f32 ? 1 : 0] = f32 ? "kkt_tma_kernel<F32> (chunked tile-TMA K1, csrc/kkt_tma.cu)"
                                    : "kkt_tma_kernel<F64> (chunked tile-TMA K1, csrc/kkt_tma.cu)";
    return true;
}

// ---------------------------------------------------------------------------
// Source-major K1 (`kkt_km_kernel`, the default when every CTA's share of the
// grid fits its threads). The grid is cut into G ~= #SMs rectangles of W <= COLS
// columns and h or h+1 rows (equal areas to one row), one per CTA, 512 threads
// = COLS columns x (512/COLS) row slots, two rows per thread. Every CTA walks
// the K sources in order over its own rectangle, so:
//  * the ds row's K-sum stays in a register per node (the reference's
//    sequential sum, bit-identical) — no cross-CTA ordering, no fold;
//  * the stencil, ds and receiver pointers are loaded once per apply;
//  * at any moment all SMs read the same few source planes, so the DRAM
//    stream stays coherent and the halo rows a CTA shares with its neighbours
//    are L2 hits.
// Per source one elected thread issues three TMA boxes (du_k, la_k with a
// one-node halo, u_k) into an S-stage ring, one block barrier per step.
// ---------------------------------------------------------------------------
template <class A>
struct KmArgs {
    using T = typename A::T;
    using R = typename A::R;
    int nx, nz, K, per_strip, W, gr, RP, nbands;
    int64_t n;
    R w2, eps;
    const T *diag, *east, *south;
    const int *nrec_ptr, *nrec_k;
    const double* nrec_w2;
    const R* ds;
    T *odu, *ola;
    R* ods;
    int hlo;                          // rectangle heights are hlo or hlo + 1
    uint32_t hb[2], ub[2], tx[2];     // halo box bytes (128-aligned), u box bytes, stage fill (h = hlo, hlo+1)
    uint32_t pb[2];                   // bytes of one source plane of a halo box
    // one-band kernel (kkt_km1_kernel): a rectangle per CTA and up to kKmShapes box shapes
    uint32_t shb[4], stx[4], spb[4];  // per shape: halo box bytes, stage fill, plane bytes
    int srp[4];                       // per shape: shared-memory row pitch (complex)
    const int4* rects;                // per CTA: x0, w, z0, h
    const unsigned char* rshape;      // per CTA: its box shape
    uint32_t stage_bytes;
    const T* u;                       // u through registers instead of a TMA box (ul = 1)
    int ul;
    int stmode;                       // output store flavour (st_mode)
    unsigned long long* trace;        // diagnostics (FWI_KKT_KM_TRACE): per CTA start, loop start, loop end, end, smid
    int rdup;                         // some node holds two receiver entries of one source (Ctx::nrec_dup)
};

__device__ __forceinline__ unsigned long long km_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// output store flavours (FWI_KKT_KM_ST): 0 st.global.cs, 1 st.global.L1::no_allocate,
// 2 st.global (default policy)
template <class T>
__device__ __forceinline__ void st_mode(T* p, T v, int mode);
template <>
__device__ __forceinline__ void st_mode<double2>(double2* p, double2 v, int mode) {
    if (mode == 1)
        asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
    else if (mode == 2)
        *p = v;
    else
        __stcs(p, v);
}
template <>
__device__ __forceinline__ void st_mode<float2>(float2* p, float2 v, int mode) {
    if (mode == 1)
        asm volatile("st.global.L1::no_allocate.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
    else if (mode == 2)
        *p = v;
    else
        __stcs(p, v);
}

// u_k at one node, read once: non-coherent, no L1 allocation (the L1 space is what
// keeps the TMA loads in flight)
template <class T>
__device__ __forceinline__ T ldg_na(const T* p);
template <>
__device__ __forceinline__ double2 ldg_na<double2>(const double2* p) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
template <>
__device__ __forceinline__ float2 ldg_na<float2>(const float2* p) {
    float2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
    return v;
}

// One band per CTA (config 2): the single-band form of kkt_km_kernel below, kept separate because
// the band loop costs it ~2.5 % (127.5 against 124.5 us on config 2).
// WS = 0: one block barrier per step, then thread 0 refills the drained stage.
// WS = 2: per-stage "empty" mbarriers (one arrival per warp) instead of the block barrier: the
//   last warp to finish a stage refills it (a shared counter per stage elects it), so no warp
//   waits for the others — warps run up to S - 1 steps apart within the ring.
// KS: sources per stage (one TMA box KS planes deep, K % KS == 0): complex64 moves half the
//   bytes of complex128 per source, so KS = 2 gives its steps the same size.
constexpr int kKmShapes = 4;
struct KmMaps {  // TMA descriptors of the one-band kernel's box shapes (du, lambda)
    CUtensorMap du[kKmShapes], la[kKmShapes];
};

template <class A, int COLS, int S, int WS, int KS, int THR>
__global__ void __launch_bounds__(THR, 1)
    kkt_km1_kernel(const __grid_constant__ KmMaps M, const KmArgs<A> P) {
    using T = typename A::T;
    using R = typename A::R;
    constexpr int kSl = THR / COLS;  // row slots; a thread owns rows slot (and slot + kSl when RPT = 2)
    constexpr int RPT = 1024 / THR;  // rows per thread: 2 with 512 threads, 1 with 1024
    // output stores: no L1 allocation, except complex64 with one source per stage (.cs); a
    // compile-time choice, so the store sites carry no branch (FWI_KKT_KM_ST applies to the
    // banded kernel only)
    constexpr int kStm = (sizeof(T) == 8 && KS == 1) ? 0 : 1;
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + size_t(S) * P.stage_bytes);
    unsigned* done = reinterpret_cast<unsigned*>(bar + S);  // WS = 2: warps finished with stage s
    const int tid = threadIdx.x, lx = tid % COLS, zs = tid / COLS;
    const int nx = P.nx, nz = P.nz, K = P.K;
    const int64_t n = P.n;
    // this CTA's rectangle and its box shape (the plan balances the rectangles' areas)
    const int4 rc = P.rects[blockIdx.x];
    const int shp = P.rshape[blockIdx.x];
    const int x0 = rc.x, w = rc.y, z0 = rc.z, h = rc.w;
    const int RP = P.srp[shp];
    const CUtensorMap* tdu = &M.du[shp];
    const CUtensorMap* tla = &M.la[shp];
    const uint32_t hb = P.shb[shp], tx = P.stx[shp], pb = P.spb[shp];
    const int steps = K / KS;
    if (P.trace && tid == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        P.trace[5 * blockIdx.x] = km_now();
        P.trace[5 * blockIdx.x + 4] = smid;
    }
    auto issue = [&](int g) {  // step g: sources [g KS, g KS + KS)
        const int s = g % S;
        unsigned char* st = sm + size_t(s) * P.stage_bytes;
        mbar_expect_tx(&bar[s], tx);
        tma_load_4d(st, tdu, 0, x0 / P.gr - 1, z0 - 1, g * KS, &bar[s]);
        tma_load_4d(st + hb, tla, 0, x0 / P.gr - 1, z0 - 1, g * KS, &bar[s]);
    };
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&bar[s], 1);
            if (WS == 2) done[s] = 0u;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int g = 0; g < S && g < steps; ++g) issue(g);
    }
    bool act[RPT], hN[RPT], hW[RPT], hE[RPT], hS[RPT];
    T cD[RPT], cN[RPT], cW[RPT], cE[RPT], cS[RPT];
    R dsv[RPT], pl[RPT];
    int qr[RPT], qe[RPT];
    int64_t cnode[RPT];
    bool full = true;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
        const int row = zs + kSl * r;
        act[r] = lx < w && row < h;
        const int ix = x0 + lx, iz = z0 + row;
        const int64_t cc = act[r] ? int64_t(iz) * nx + ix : 0;
        cnode[r] = cc;
        const bool bnd = on_boundary(ix, iz, nx, nz);
        hN[r] = act[r] && !bnd && !on_boundary(ix, iz - 1, nx, nz);
        hW[r] = act[r] && !bnd && !on_boundary(ix - 1, iz, nx, nz);
        hE[r] = act[r] && !bnd && !on_boundary(ix + 1, iz, nx, nz);
        hS[r] = act[r] && !bnd && !on_boundary(ix, iz + 1, nx, nz);
        full = full && act[r] && hN[r] && hW[r] && hE[r] && hS[r];
        cD[r] = act[r] ? P.diag[cc] : A::zero();
        cN[r] = hN[r] ? P.south[cc - nx] : A::zero();
        cW[r] = hW[r] ? P.east[cc - 1] : A::zero();
        cE[r] = hE[r] ? P.east[cc] : A::zero();
        cS[r] = hS[r] ? P.south[cc] : A::zero();
        dsv[r] = act[r] ? P.ds[cc] : R(0);
        qr[r] = act[r] ? P.nrec_ptr[cc] : 0;
        qe[r] = act[r] ? P.nrec_ptr[cc + 1] : 0;
        pl[r] = R(0);
    }
    const bool warp_full = __all_sync(0xffffffffu, full);
    const int lxs = min(lx, w - 1);  // lanes beyond the rectangle read (and drop) its last column
    T un[KS][RPT];  // u of the next step's sources, loaded one step ahead (u is read once per node)
#pragma unroll
    for (int kk = 0; kk < KS; ++kk)
#pragma unroll
        for (int r = 0; r < RPT; ++r) un[kk][r] = act[r] ? ldg_na(P.u + int64_t(kk) * n + cnode[r]) : A::zero();
    // receiver entries one step ahead (one-band kernel, tables without duplicate (node, source)
    // entries): the entry at qr[r] sits in registers, so a receiver row's warps do not wait for
    // two dependent table loads inside every step (the per-CTA timeline showed the receiver
    // bands ending 15 us after the others at C2)
    const bool rfast = !P.rdup;
    int pk[RPT];
    double pw[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
        pk[r] = -1;
        pw[r] = 0.0;
        if (rfast && qr[r] < qe[r]) {
            pk[r] = P.nrec_k[qr[r]];
            pw[r] = P.nrec_w2[qr[r]];
        }
    }
    __syncthreads();
    if (P.trace && tid == 0) P.trace[5 * blockIdx.x + 1] = km_now();
    for (int g = 0; g < steps; ++g) {
        T ucur[KS][RPT];
#pragma unroll
        for (int kk = 0; kk < KS; ++kk)
#pragma unroll
            for (int r = 0; r < RPT; ++r) ucur[kk][r] = un[kk][r];
        if (g + 1 < steps)
#pragma unroll
            for (int kk = 0; kk < KS; ++kk)
#pragma unroll
                for (int r = 0; r < RPT; ++r)
                    if (act[r]) un[kk][r] = ldg_na(P.u + int64_t((g + 1) * KS + kk) * n + cnode[r]);
        const int s = g % S;
        mbar_wait(&bar[s], (g / S) & 1);
        const unsigned char* st = sm + size_t(s) * P.stage_bytes;
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
            const int k = g * KS + kk;
            const T* dus = reinterpret_cast<const T*>(st + kk * pb) + P.gr + lxs;
            const T* las = reinterpret_cast<const T*>(st + hb + kk * pb) + P.gr + lxs;
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                const int row = zs + kSl * r;
                if (row >= h) continue;  // CTA-uniform per slot: the rectangle's last rows
                T s_, t_;
                const T* dr = dus + (row + 1) * RP;
                const T* lr = las + (row + 1) * RP;
                if (warp_full)
                    node_step<A, true>(dr, lr, RP, true, true, true, true, cD[r], cN[r], cW[r], cE[r], cS[r], s_, t_);
                else
                    node_step<A, false>(dr, lr, RP, hN[r], hW[r], hE[r], hS[r], cD[r], cN[r], cW[r], cE[r], cS[r],
                                        s_, t_);
                const T duc = dr[0], lac = lr[0], uc = ucur[kk][r];
                pl[r] = A::radd(pl[r], A::re_pconj(P.w2, uc, lac));
                if (!act[r]) continue;
                const int64_t o = int64_t(k) * n + cnode[r];
                st_mode(P.ola + o, A::sub(s_, A::pmul(P.w2, uc, dsv[r])), kStm);
                if (rfast) {
                    if (pk[r] == k) {  // at most one entry per (node, source): same sum, 0 + w2 du
                        t_ = A::add(A::add(A::zero(), A::rm(R(pw[r]), duc)), t_);
                        ++qr[r];
                        pk[r] = -1;
                        if (qr[r] < qe[r]) {
                            pk[r] = P.nrec_k[qr[r]];
                            pw[r] = P.nrec_w2[qr[r]];
                        }
                    }
                } else if (qr[r] < qe[r] && P.nrec_k[qr[r]] == k) {
                    T f = A::zero();
                    while (qr[r] < qe[r] && P.nrec_k[qr[r]] == k) {
                        f = A::add(f, A::rm(R(P.nrec_w2[qr[r]]), duc));
                        ++qr[r];
                    }
                    t_ = A::add(f, t_);
                }
                st_mode(P.odu + o, t_, kStm);
            }
        }
        if constexpr (WS == 2) {
            // this warp is done with stage s; the last of the 16 refills it with step g + S
            __syncwarp();
            if ((tid & 31) == 0) {
                unsigned old;
                asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                             : "=r"(old) : "r"(smem_u32(&done[s])) : "memory");
                if (old % unsigned(THR / 32) == unsigned(THR / 32 - 1) && g + S < steps) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    issue(g + S);
                }
            }
        } else {
            __syncthreads();  // every thread is done with stage s
            if (tid == 0 && g + S < steps) issue(g + S);
        }
    }
    if (P.trace && tid == 0) P.trace[5 * blockIdx.x + 2] = km_now();
#pragma unroll
    for (int r = 0; r < RPT; ++r)
        if (act[r]) P.ods[cnode[r]] = A::rsub(A::rmulr(P.eps, dsv[r]), pl[r]);
    if (P.trace && tid == 0) P.trace[5 * blockIdx.x + 3] = km_now();
}
template <class A, int COLS, int S, bool MB>
__global__ void __launch_bounds__(512, 1)
    kkt_km_kernel(const __grid_constant__ CUtensorMap tdu0, const __grid_constant__ CUtensorMap tla0,
                  const __grid_constant__ CUtensorMap tu0, const __grid_constant__ CUtensorMap tdu1,
                  const __grid_constant__ CUtensorMap tla1, const __grid_constant__ CUtensorMap tu1,
                  const KmArgs<A> P) {
    using T = typename A::T;
    using R = typename A::R;
    constexpr int kSl = 512 / COLS;  // row slots; a thread owns rows slot and slot + kSl
    extern __shared__ __align__(1024) unsigned char sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + size_t(S) * P.stage_bytes);
    const int tid = threadIdx.x, lx = tid % COLS, zs = tid / COLS;
    const int nx = P.nx, nz = P.nz, K = P.K, RP = P.RP;
    const int64_t n = P.n;
    // bands of this CTA: q = blockIdx.x + j * gridDim.x, band q = strip q / per_strip, rows
    // [z0, z1) of it; one band per CTA when the grid is small enough (config 2), several otherwise
    const int nmine = MB ? (P.nbands - int(blockIdx.x) + int(gridDim.x) - 1) / int(gridDim.x) : 1;
    const int64_t nsteps = int64_t(nmine) * K;
    struct Band {
        int x0, w, z0, h, hi;
    };
    auto band = [&](int j) {
        const int q = int(blockIdx.x) + j * int(gridDim.x);
        const int strip = q / P.per_strip, i = q % P.per_strip;
        Band bd;
        bd.z0 = int(int64_t(i) * nz / P.per_strip);
        bd.h = int(int64_t(i + 1) * nz / P.per_strip) - bd.z0;
        bd.hi = bd.h - P.hlo;  // 0 or 1: which box shape
        bd.x0 = strip * P.W;
        bd.w = min(P.W, nx - bd.x0);
        return bd;
    };
    // producer state (thread 0): the next step to issue, walked in order
    int ij = 0, ik = 0, is = 0;
    Band ib = band(0);
    auto issue_next = [&]() {
        unsigned char* st = sm + size_t(is) * P.stage_bytes;
        const uint32_t hbi = P.hb[ib.hi];
        mbar_expect_tx(&bar[is], P.tx[ib.hi]);
        tma_load_4d(st, ib.hi ? &tdu1 : &tdu0, 0, ib.x0 / P.gr - 1, ib.z0 - 1, ik, &bar[is]);
        tma_load_4d(st + hbi, ib.hi ? &tla1 : &tla0, 0, ib.x0 / P.gr - 1, ib.z0 - 1, ik, &bar[is]);
        if (!P.ul) tma_load_4d(st + 2 * hbi, ib.hi ? &tu1 : &tu0, 0, ib.x0 / P.gr, ib.z0, ik, &bar[is]);
        is = is + 1 == S ? 0 : is + 1;
        if (++ik == K) {
            ik = 0;
            if (++ij < nmine) ib = band(ij);
        }
    };
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int64_t g = 0; g < S && g < nsteps; ++g) issue_next();
    }
    int cs = 0;        // consumer: stage of the next step
    uint32_t cph = 0;  // and its phase
    __syncthreads();
    const int UP = P.W;                // u box row pitch (complex)
    const int lxs = min(lx, P.W - 1);  // lanes beyond the strip read (and drop) its last column
    for (int j = 0; j < nmine; ++j) {
        const Band bd = band(j);
        const int x0 = bd.x0, w = bd.w, z0 = bd.z0, h = bd.h;
        const uint32_t hb = P.hb[bd.hi];
        bool act[2], hN[2], hW[2], hE[2], hS[2];
        T cD[2], cN[2], cW[2], cE[2], cS[2];
        R dsv[2], pl[2];
        int qr[2], qe[2];
        int64_t cnode[2];
        bool full = true;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int row = zs + kSl * r;
            act[r] = lx < w && row < h;
            const int ix = x0 + lx, iz = z0 + row;
            const int64_t cc = act[r] ? int64_t(iz) * nx + ix : 0;
            cnode[r] = cc;
            const bool bnd = on_boundary(ix, iz, nx, nz);
            hN[r] = act[r] && !bnd && !on_boundary(ix, iz - 1, nx, nz);
            hW[r] = act[r] && !bnd && !on_boundary(ix - 1, iz, nx, nz);
            hE[r] = act[r] && !bnd && !on_boundary(ix + 1, iz, nx, nz);
            hS[r] = act[r] && !bnd && !on_boundary(ix, iz + 1, nx, nz);
            full = full && act[r] && hN[r] && hW[r] && hE[r] && hS[r];
            cD[r] = act[r] ? P.diag[cc] : A::zero();
            cN[r] = hN[r] ? P.south[cc - nx] : A::zero();
            cW[r] = hW[r] ? P.east[cc - 1] : A::zero();
            cE[r] = hE[r] ? P.east[cc] : A::zero();
            cS[r] = hS[r] ? P.south[cc] : A::zero();
            dsv[r] = act[r] ? P.ds[cc] : R(0);
            qr[r] = act[r] ? P.nrec_ptr[cc] : 0;
            qe[r] = act[r] ? P.nrec_ptr[cc + 1] : 0;
            pl[r] = R(0);
        }
        const bool warp_full = __all_sync(0xffffffffu, full);
        T un[2] = {A::zero(), A::zero()};  // ul: u_k of the next step, loaded one step ahead
        if (P.ul)
#pragma unroll
            for (int r = 0; r < 2; ++r)
                if (act[r]) un[r] = ldg_na(P.u + cnode[r]);
        for (int k = 0; k < K; ++k) {
            T ucur[2] = {un[0], un[1]};
            if (P.ul && k + 1 < K)
#pragma unroll
                for (int r = 0; r < 2; ++r)
                    if (act[r]) un[r] = ldg_na(P.u + int64_t(k + 1) * n + cnode[r]);
            const int64_t g = int64_t(j) * K + k;
            const int s = cs;
            mbar_wait(&bar[s], cph);
            if (++cs == S) {
                cs = 0;
                cph ^= 1u;
            }
            const unsigned char* st = sm + size_t(s) * P.stage_bytes;
            const T* dus = reinterpret_cast<const T*>(st) + P.gr + lxs;
            const T* las = reinterpret_cast<const T*>(st + hb) + P.gr + lxs;
            const T* us = reinterpret_cast<const T*>(st + 2 * hb) + lxs;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const int row = zs + kSl * r;
            if (row >= h) continue;  // CTA-uniform per slot: the rectangle's last rows
            T s_, t_;
            const T* dr = dus + (row + 1) * RP;
            const T* lr = las + (row + 1) * RP;
            if (warp_full)
                node_step<A, true>(dr, lr, RP, true, true, true, true, cD[r], cN[r], cW[r], cE[r], cS[r], s_, t_);
            else
                node_step<A, false>(dr, lr, RP, hN[r], hW[r], hE[r], hS[r], cD[r], cN[r], cW[r], cE[r], cS[r], s_,
                                    t_);
            const T duc = dr[0], lac = lr[0], uc = P.ul ? ucur[r] : us[row * UP];
            pl[r] = A::radd(pl[r], A::re_pconj(P.w2, uc, lac));
            if (!act[r]) continue;
            const int64_t o = int64_t(k) * n + cnode[r];
            st_mode(P.ola + o, A::sub(s_, A::pmul(P.w2, uc, dsv[r])), P.stmode);
            if (qr[r] < qe[r] && P.nrec_k[qr[r]] == k) {
                T f = A::zero();
                while (qr[r] < qe[r] && P.nrec_k[qr[r]] == k) {
                    f = A::add(f, A::rm(R(P.nrec_w2[qr[r]]), duc));
                    ++qr[r];
                }
                t_ = A::add(f, t_);
            }
            st_mode(P.odu + o, t_, P.stmode);
        }
            __syncthreads();  // every thread is done with stage s
            if (tid == 0 && g + S < nsteps) issue_next();
        }
#pragma unroll
        for (int r = 0; r < 2; ++r)
            if (act[r]) P.ods[cnode[r]] = A::rsub(A::rmulr(P.eps, dsv[r]), pl[r]);
    }
}

}  // namespace

struct KktKmPlan {
    bool ok = false;
    int cols = 128, stages = 0, G = 0, per_strip = 0, W = 0, gr = 8, RP = 0, hlo = 0, ul = 1, nbands = 0;
    int ws = 0, ks = 1;  // one-band kernel: ring discipline, sources per stage
    int thr = 512;       // one-band kernel: threads per CTA (1024: one row per thread)
    uint32_t hb[2] = {0, 0}, ub[2] = {0, 0}, tx[2] = {0, 0}, pb[2] = {0, 0}, stage_bytes = 0;
    size_t smem = 0;
    CUtensorMap tm_u[2];
    // one-band kernel: a rectangle per CTA, box shapes (box width in columns, rows)
    int nshapes = 0, shw[4] = {0, 0, 0, 0}, shh[4] = {0, 0, 0, 0};
    uint32_t shb[4] = {0, 0, 0, 0}, stx[4] = {0, 0, 0, 0}, spb[4] = {0, 0, 0, 0};
    int max_area = 0;  // largest rectangle (nodes): the apply's time follows it (C2, round 2)
    DevBuf<int4> rects;
    DevBuf<unsigned char> rshape;
    DevBuf<unsigned long long> trace;  // FWI_KKT_KM_TRACE
};

void kkt_km_plan_free(KktKmPlan* p) { delete p; }

namespace {

// instantiations: (COLS, S, MB, WS, KS); MB: several bands per CTA (kkt_km_kernel), else the
// one-band kkt_km1_kernel with its ring discipline WS and sources per stage KS
#define FWI_KM_KEY(COLSv, Sv, MBv, WSv, KSv, THRv) \
    ((((((COLSv) * 16 + (Sv)) * 2 + (MBv)) * 4 + (WSv)) * 4 + (KSv)) * 2 + ((THRv) == 1024 ? 1 : 0))
#define FWI_KM_DISPATCH(COLSv, Sv, MBv, WSv, KSv, THRv, CALL)                             \
    switch (FWI_KM_KEY(COLSv, Sv, MBv, WSv, KSv, THRv)) {                                 \
        case FWI_KM_KEY(128, 2, 0, 0, 1, 512): CALL(128, 2, false, 0, 1, 512); break;     \
        case FWI_KM_KEY(128, 3, 0, 0, 1, 512): CALL(128, 3, false, 0, 1, 512); break;     \
        case FWI_KM_KEY(64, 3, 0, 0, 1, 512): CALL(64, 3, false, 0, 1, 512); break;       \
        case FWI_KM_KEY(64, 4, 0, 0, 1, 512): CALL(64, 4, false, 0, 1, 512); break;       \
        case FWI_KM_KEY(32, 2, 0, 0, 1, 512): CALL(32, 2, false, 0, 1, 512); break;       \
        case FWI_KM_KEY(32, 3, 0, 0, 1, 512): CALL(32, 3, false, 0, 1, 512); break;       \
        case FWI_KM_KEY(64, 2, 0, 2, 1, 512): CALL(64, 2, false, 2, 1, 512); break;       \
        case FWI_KM_KEY(64, 3, 0, 2, 1, 512): CALL(64, 3, false, 2, 1, 512); break;       \
        case FWI_KM_KEY(64, 4, 0, 2, 1, 512): CALL(64, 4, false, 2, 1, 512); break;       \
        case FWI_KM_KEY(64, 2, 0, 0, 2, 512): CALL(64, 2, false, 0, 2, 512); break;       \
        case FWI_KM_KEY(64, 3, 0, 0, 2, 512): CALL(64, 3, false, 0, 2, 512); break;       \
        case FWI_KM_KEY(64, 2, 0, 2, 2, 512): CALL(64, 2, false, 2, 2, 512); break;       \
        case FWI_KM_KEY(64, 3, 0, 2, 2, 512): CALL(64, 3, false, 2, 2, 512); break;       \
        case FWI_KM_KEY(64, 4, 0, 2, 2, 512): CALL(64, 4, false, 2, 2, 512); break;       \
        case FWI_KM_KEY(64, 2, 0, 0, 1, 1024): CALL(64, 2, false, 0, 1, 1024); break;     \
        case FWI_KM_KEY(64, 3, 0, 0, 1, 1024): CALL(64, 3, false, 0, 1, 1024); break;     \
        case FWI_KM_KEY(64, 2, 0, 0, 2, 1024): CALL(64, 2, false, 0, 2, 1024); break;     \
        case FWI_KM_KEY(64, 3, 0, 0, 2, 1024): CALL(64, 3, false, 0, 2, 1024); break;     \
        case FWI_KM_KEY(64, 2, 1, 0, 1, 512): CALL(64, 2, true, 0, 1, 512); break;        \
        case FWI_KM_KEY(64, 3, 1, 0, 1, 512): CALL(64, 3, true, 0, 1, 512); break;        \
        default: CALL(64, 2, false, 0, 1, 512); break;                                    \
    }

// Area-balanced rectangles for the one-band kernel (FWI_KKT_KM_BALANCED=1, an experiment). Every
// CTA walks all K sources over its own rectangle and the CTAs cannot share work (each node's
// K-sum is one CTA's), so the apply takes as long as the slowest CTA: on C2, 128 CTAs of 16 x 64
// nodes take 136.9 us against 125.2 us for 144 CTAs of at most 15 x 64. Strips of two widths
// (multiples of the 8-complex TMA group), each cut into equal bands of 8..maxrows rows, bring the
// largest rectangle to the smallest area achievable (C2: one 64-column strip of 19 bands and
// eight 56-column strips of 16 bands = 147 CTAs of at most 896 nodes, against 960) — and measure
// 137.0 us: a CTA's time follows its rows x 64 lanes (its warp-rows), not its area, so the
// 56-column strips cost what 64-column ones do (tools/exp_km_rects.sh). Returns the strips as
// (width, bands) pairs left to right, or an empty list.
std::vector<std::pair<int, int>> balanced_strips(int nx, int nz, int sms, int cols, int maxrows, int minrows,
                                                 int gr, int& area) {
    std::vector<int> widths;
    for (int w = cols; w >= gr; w -= gr) widths.push_back(w);
    std::vector<int> targets;
    for (int w : widths)
        for (int h = minrows; h <= maxrows; ++h) targets.push_back(w * h);
    std::sort(targets.begin(), targets.end());
    targets.erase(std::unique(targets.begin(), targets.end()), targets.end());
    for (int M : targets) {
        if (int64_t(M) * sms < int64_t(nx) * nz) continue;
        auto bands = [&](int w) {  // fewest bands of <= M nodes, or 0 when the rows fall short
            const int h = std::min(maxrows, M / w);
            if (h < minrows) return 0;
            const int b = (nz + h - 1) / h;
            return nz / b >= minrows ? b : 0;
        };
        int best = INT_MAX;
        std::vector<std::pair<int, int>> pick;
        for (int wa : widths) {
            const int ba = bands(wa);
            if (!ba) continue;
            for (int wb : widths) {
                if (wb > wa) continue;
                const int bb = bands(wb);
                if (!bb) continue;
                for (int na = 1; na * wa <= nx; ++na) {
                    const int rem = nx - na * wa;
                    if (wb == wa ? rem != 0 : (rem == 0 || rem % wb != 0)) continue;
                    const int nb = wb == wa ? 0 : rem / wb;
                    const int total = na * ba + nb * bb;
                    if (total <= sms && total < best) {
                        best = total;
                        pick.assign(size_t(na), {wa, ba});
                        for (int q = 0; q < nb; ++q) pick.push_back({wb, bb});
                    }
                }
            }
        }
        if (!pick.empty()) {
            area = M;
            return pick;
        }
    }
    return {};
}

template <class A>
KktKmPlan* build_km_plan(Ctx& c, bool f32) {
    auto p = std::make_unique<KktKmPlan>();
    const int nx = c.nx, nz = c.nz, K = c.K;
    const int es = f32 ? 8 : 16;
    if (nx % 2 != 0 || !encode_fn()) return p.release();
    const int sms = sm_count();
    const bool force = std::getenv("FWI_KKT_KM_FORCE") != nullptr;
    // Rectangles of <= 2 x (512 / COLS) rows. 64-column strips (measured best on C2 with equal
    // strips: 128 us per apply against 142 us with 128 columns and 131 us with 32); the kernel is
    // chosen only when the rectangles have >= 8 rows — shorter ones spend too much on halo rows.
    // One rectangle per CTA when the grid fits (config 2: 8 strips x 18 bands of 14-15 rows);
    // otherwise bands of ~15 rows, several per CTA, each walked over all sources (config 5: 32
    // strips x 69 bands on 148 CTAs). FWI_KKT_KM_ROWS sets a uniform band height (tests: several
    // bands per CTA on small grids). FWI_KKT_KM_BALANCED=1 plans area-balanced strips of two
    // widths instead (balanced_strips; measured slower, kept as the documented experiment).
    int cols = 64;
    const char* ecols = std::getenv("FWI_KKT_KM_COLS");
    if (ecols) cols = std::atoi(ecols) == 128 ? 128 : std::atoi(ecols) == 32 ? 32 : 64;
    int maxrows = 2 * (512 / cols);
    const int nsx = (nx + cols - 1) / cols;
    int per = std::min(sms / nsx, nz);
    if (per < 1 || (nz + per - 1) / per > maxrows) per = (nz + 14) / 15;
    const bool rows_env = std::getenv("FWI_KKT_KM_ROWS") != nullptr;
    if (rows_env) per = (nz + std::max(1, std::atoi(std::getenv("FWI_KKT_KM_ROWS"))) - 1) /
                        std::max(1, std::atoi(std::getenv("FWI_KKT_KM_ROWS")));
    per = std::max(1, std::min(per, nz));
    const int W = ((nx + nsx - 1) / nsx + 1) / 2 * 2;  // even strip width <= cols
    int gr = 8;
    if (const char* e = std::getenv("FWI_KKT_GRP")) gr = std::max(1, std::atoi(e));
    if (nx % gr != 0 || W % gr != 0) gr = 2;
    bool uniform_ok = (nz + per - 1) / per <= maxrows && (nz / per >= 8 || force) && W <= cols;
    int uniform_area = W * ((nz + per - 1) / per);
    int G = std::min(sms, nsx * per);
    if (const char* e = std::getenv("FWI_KKT_KM_G")) G = std::max(1, std::min(G, std::atoi(e)));  // tests
    bool mb = G < nsx * per;
    // balanced one-rectangle-per-CTA layout (strips of two widths, multiples of the TMA group)
    std::vector<std::pair<int, int>> strips;
    int bal_area = 0;
    if (std::getenv("FWI_KKT_KM_BALANCED") && !rows_env && !std::getenv("FWI_KKT_KM_G") && nx % 8 == 0 &&
        !std::getenv("FWI_KKT_GRP")) {
        const int bcols = ecols ? cols : 64;
        strips = balanced_strips(nx, nz, sms, std::min(bcols, 64), 2 * (512 / std::min(bcols, 64)), force ? 1 : 8, 8,
                                 bal_area);
        if (!strips.empty() && uniform_ok && !mb && bal_area >= uniform_area) strips.clear();
    }
    if (!strips.empty()) {
        int wmax = 0;
        for (auto& sb : strips) wmax = std::max(wmax, sb.first);
        if (wmax <= 32 && !ecols) cols = 32;  // every lane of a 32-column CTA has a column
        maxrows = 2 * (512 / cols);
        gr = 8;
        mb = false;
    } else if (!uniform_ok) {
        return p.release();
    }
    p->cols = cols;
    p->gr = gr;
    p->ul = 1;
    // u through registers (non-allocating loads) rather than a third TMA box: shared memory is
    // carved out of the L1, and the L1 space is what keeps the TMA loads in flight (unused extra
    // shared memory alone slows the C2 apply: +30 KB 128 -> 140 us, +60 KB 154 us). The banded
    // kernel keeps the TMA form as a diagnostic (FWI_KKT_KM_ULDG=0).
    if (mb)
        if (const char* e = std::getenv("FWI_KKT_KM_ULDG")) p->ul = std::atoi(e) != 0;
    if (!mb) {
        // complex64: two sources per stage, so a step moves the bytes of a complex128 step
        // (C2: 91.6 -> 82.9 us with non-allocating stores, tools/exp_km_c64.sh); the per-stage
        // empty barriers (WS = 2) measured within noise of the block barrier (124.6 vs 125.2 us
        // at 3 stages for complex128, slower for complex64), so the block barrier stays
        p->ks = f32 ? 2 : 1;
        if (const char* e = std::getenv("FWI_KKT_KM_WS")) p->ws = std::atoi(e) == 2 ? 2 : 0;
        if (const char* e = std::getenv("FWI_KKT_KM_KS")) p->ks = std::atoi(e) == 2 ? 2 : 1;
        // 1024 threads, one row per thread (twice the warps to hide latency; the register budget
        // halves to 64)
        if (const char* e = std::getenv("FWI_KKT_KM_THR")) p->thr = std::atoi(e) == 1024 ? 1024 : 512;
        if (cols != 64) p->ws = 0, p->ks = 1;
        if (p->ws != 0) p->thr = 512;
        if (K % p->ks != 0) p->ks = 1;
        // the rectangles and their box shapes
        std::vector<int4> rc;
        std::vector<unsigned char> rs;
        auto shape_of = [&](int wbox, int h) {
            for (int q = 0; q < p->nshapes; ++q)
                if (p->shw[q] == wbox && p->shh[q] == h) return q;
            if (p->nshapes == kKmShapes) return -1;
            p->shw[p->nshapes] = wbox;
            p->shh[p->nshapes] = h;
            return p->nshapes++;
        };
        auto add_strip = [&](int x0, int w, int wbox, int bands) {
            for (int b = 0; b < bands; ++b) {
                const int z0 = int(int64_t(b) * nz / bands), z1 = int(int64_t(b + 1) * nz / bands);
                const int q = shape_of(wbox, z1 - z0);
                if (q < 0) return false;
                rc.push_back(make_int4(x0, w, z0, z1 - z0));
                rs.push_back((unsigned char)q);
                p->max_area = std::max(p->max_area, w * (z1 - z0));
            }
            return true;
        };
        bool okr = true;
        if (!strips.empty()) {
            int x0 = 0;
            for (auto& sb : strips) {
                okr = okr && add_strip(x0, sb.first, sb.first, sb.second);
                x0 += sb.first;
            }
        } else {
            for (int q = 0; q < nsx; ++q) okr = okr && add_strip(q * W, std::min(W, nx - q * W), W, per);
        }
        if (!okr || int(rc.size()) > sms) return p.release();
        p->G = int(rc.size());
        p->nbands = p->G;
        p->rects.alloc(rc.size());
        p->rshape.alloc(rs.size());
        CK(cudaMemcpy(p->rects.p, rc.data(), rc.size() * sizeof(int4), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(p->rshape.p, rs.data(), rs.size(), cudaMemcpyHostToDevice));
        for (int q = 0; q < p->nshapes; ++q) {
            const int rp = p->shw[q] + 2 * gr;
            p->spb[q] = uint32_t(size_t(rp) * (p->shh[q] + 2) * es);
            p->shb[q] = align128(size_t(p->ks) * p->spb[q]);
            p->stx[q] = 2 * p->ks * p->spb[q];
            p->stage_bytes = std::max(p->stage_bytes, 2 * p->shb[q]);
        }
    } else {
        p->per_strip = per;
        p->nbands = nsx * per;
        p->G = G;
        p->W = W;
        p->RP = W + 2 * gr;
        p->hlo = nz / per;
        for (int v = 0; v < 2; ++v) {
            const int h = p->hlo + v;
            p->pb[v] = uint32_t(size_t(p->RP) * (h + 2) * es);
            p->hb[v] = align128(size_t(p->pb[v]));
            p->ub[v] = p->ul ? 0 : align128(size_t(W) * h * es);
            p->tx[v] = uint32_t(2 * size_t(p->pb[v]) + (p->ul ? 0 : size_t(W) * h * es));
            p->stage_bytes = std::max(p->stage_bytes, 2 * p->hb[v] + p->ub[v]);
        }
    }
    const size_t budget = 227 * 1024 - 128;
    // two stages in flight (three for complex64 with one source per stage): deeper rings are
    // measurably slower with the output stores sharing the memory system (C2: 3 stages 181 us,
    // 4 stages 209 us against 129 us, with L1-allocating stores)
    int st = (f32 && p->ks == 1) ? 3 : 2;
    if (const char* e = std::getenv("FWI_KKT_KM_STAGES")) st = std::atoi(e);
    auto valid = [&](int v) {
        if (mb) return cols == 64 && (v == 2 || v == 3);
        if (p->ks == 2 && p->ws == 0) return v == 2 || v == 3;
        if (p->ws == 2) return v >= 2 && v <= 4;
        return cols == 32 ? (v == 2 || v == 3) : cols == 128 ? (v == 2 || v == 3) : (v >= 2 && v <= 4);
    };
    while (st > 2 && (!valid(st) || size_t(st) * p->stage_bytes > budget)) --st;
    if (!valid(st)) return p.release();
    if (size_t(st) * p->stage_bytes > budget) return p.release();
    p->stages = st;
    p->smem = size_t(st) * p->stage_bytes + 128;
    if (const char* e = std::getenv("FWI_KKT_KM_PAD_KB"))  // diagnostics: unused extra shared memory
        p->smem = std::min<size_t>(227 * 1024, p->smem + size_t(std::atoi(e)) * 1024);
#define FWI_KM_ATTR(COLSc, Sc, MBc, WSc, KSc, THRc)                                                       \
    CK(MBc ? cudaFuncSetAttribute(kkt_km_kernel<A, COLSc, Sc, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                  int(p->smem))                                                             \
           : cudaFuncSetAttribute(kkt_km1_kernel<A, COLSc, Sc, WSc, KSc, THRc>,                               \
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, int(p->smem)))
    FWI_KM_DISPATCH(cols, st, mb ? 1 : 0, p->ws, p->ks, p->thr, FWI_KM_ATTR);
#undef FWI_KM_ATTR
    if (mb) {
        const void* ubase = f32 ? static_cast<const void*>(c.u32.p) : static_cast<const void*>(c.u.p);
        for (int v = 0; v < 2; ++v)
            if (!ubase || !encode(&p->tm_u[v], f32, ubase, nx, nz, K, gr, W / gr, p->hlo + v)) return p.release();
    }
    if (std::getenv("FWI_KKT_KM_LOG")) {
        std::fprintf(stderr, "[fwi] K1 plan %dx%d K=%d %s: cols %d, %d CTAs, stages %d, ks %d, ws %d, ", nx, nz, K,
                     f32 ? "c64" : "c128", cols, p->G, st, p->ks, p->ws);
        if (mb)
            std::fprintf(stderr, "%d bands of %d-%d rows x %d columns\n", p->nbands, p->hlo, p->hlo + 1, W);
        else {
            std::fprintf(stderr, "largest rectangle %d nodes, shapes", p->max_area);
            for (int q = 0; q < p->nshapes; ++q) std::fprintf(stderr, " %dx%d", p->shw[q], p->shh[q]);
            std::fprintf(stderr, "\n");
        }
    }
    p->ok = true;
    return p.release();
}

template <class A>
bool launch_km(Ctx& c, KktKmPlan* p, const typename A::T* du, const typename A::R* ds, const typename A::T* la,
               typename A::T* odu, typename A::R* ods, typename A::T* ola, bool f32) {
    const bool mb = p->G < p->nbands;
    CUtensorMap tdu[2], tla[2];
    KmMaps maps;
    if (mb) {
        for (int v = 0; v < 2; ++v) {
            if (!encode(&tdu[v], f32, du, c.nx, c.nz, c.K, p->gr, p->RP / p->gr, p->hlo + v + 2)) return false;
            if (!encode(&tla[v], f32, la, c.nx, c.nz, c.K, p->gr, p->RP / p->gr, p->hlo + v + 2)) return false;
        }
    } else {
        for (int q = 0; q < p->nshapes; ++q) {
            const int pairs = (p->shw[q] + 2 * p->gr) / p->gr;
            if (!encode(&maps.du[q], f32, du, c.nx, c.nz, c.K, p->gr, pairs, p->shh[q] + 2, p->ks)) return false;
            if (!encode(&maps.la[q], f32, la, c.nx, c.nz, c.K, p->gr, pairs, p->shh[q] + 2, p->ks)) return false;
        }
    }
    KmArgs<A> a;
    a.nx = c.nx;
    a.nz = c.nz;
    a.K = c.K;
    a.per_strip = p->per_strip;
    a.nbands = p->nbands;
    a.W = p->W;
    a.gr = p->gr;
    a.RP = p->RP;
    a.n = c.n;
    a.w2 = typename A::R(c.w2);
    a.eps = typename A::R(c.eps);
    if (f32) {
        a.diag = reinterpret_cast<const typename A::T*>(c.diag32.p);
        a.east = reinterpret_cast<const typename A::T*>(c.east32.p);
        a.south = reinterpret_cast<const typename A::T*>(c.south32.p);
    } else {
        a.diag = reinterpret_cast<const typename A::T*>(c.diag.p);
        a.east = reinterpret_cast<const typename A::T*>(c.east.p);
        a.south = reinterpret_cast<const typename A::T*>(c.south.p);
    }
    a.nrec_ptr = c.nrec_ptr.p;
    a.nrec_k = c.nrec_k.p;
    a.nrec_w2 = c.nrec_w2.p;
    a.ds = ds;
    a.odu = odu;
    a.ola = ola;
    a.ods = ods;
    a.hlo = p->hlo;
    for (int v = 0; v < 2; ++v) {
        a.hb[v] = p->hb[v];
        a.ub[v] = p->ub[v];
        a.tx[v] = p->tx[v];
        a.pb[v] = p->pb[v];
    }
    for (int q = 0; q < kKmShapes; ++q) {
        a.shb[q] = p->shb[q];
        a.stx[q] = p->stx[q];
        a.spb[q] = p->spb[q];
        a.srp[q] = p->shw[q] + 2 * p->gr;
    }
    a.rects = p->rects.p;
    a.rshape = p->rshape.p;
    a.stage_bytes = p->stage_bytes;
    a.ul = p->ul;
    // complex128 outputs bypass the L1 (st.global.L1::no_allocate): with L1-allocating streaming
    // stores the apply needs free L1 (unused shared memory and deeper rings slowed it); without
    // allocation it does not, 126 -> 124.7 us. complex64 with one source per stage keeps .cs (0.088 vs 0.090 ms); with two, no_allocate (82.9 vs 85.0 us).
    a.stmode = (f32 && p->ks == 1) ? 0 : 1;
    if (const char* e = std::getenv("FWI_KKT_KM_ST")) a.stmode = std::atoi(e);
    a.u = reinterpret_cast<const typename A::T*>(f32 ? static_cast<const void*>(c.u32.p)
                                                    : static_cast<const void*>(c.u.p));
    // diagnostics: FWI_KKT_KM_TRACE=<file> writes each launch's per-CTA timeline (globaltimer ns:
    // start, loop start, loop end, end; SM id), synchronising after the launch — never set in production
    const char* trace_path = mb ? nullptr : std::getenv("FWI_KKT_KM_TRACE");
    a.rdup = (c.nrec_dup || std::getenv("FWI_KKT_KM_RDUP")) ? 1 : 0;  // env: force the general loop (tests, A/B)
    a.trace = nullptr;
    if (trace_path) {
        if (!p->trace.p) p->trace.alloc(size_t(5) * p->G);
        a.trace = p->trace.p;
    }
#define FWI_KM_LAUNCH(COLSc, Sc, MBc, WSc, KSc, THRc)                                                      \
    ((MBc ? kkt_km_kernel<A, COLSc, Sc, true><<<p->G, 512, p->smem, c.stream>>>(tdu[0], tla[0], p->tm_u[0],     \
                                                                              tdu[1], tla[1], p->tm_u[1], a)  \
          : kkt_km1_kernel<A, COLSc, Sc, WSc, KSc, THRc><<<p->G, THRc, p->smem, c.stream>>>(maps, a)),        \
     c.kkt_kernel[f32 ? 1 : 0] = MBc ? (f32 ? "kkt_km_kernel<F32, " #COLSc ", " #Sc ", bands> (source-major TMA K1, csrc/kkt_tma.cu)" \
                                           : "kkt_km_kernel<F64, " #COLSc ", " #Sc ", bands> (source-major TMA K1, csrc/kkt_tma.cu)") \
                                     : (f32 ? "kkt_km1_kernel<F32, " #COLSc ", " #Sc ", " #WSc ", " #KSc ", " #THRc "> (source-major TMA K1, one band per CTA, csrc/kkt_tma.cu)" \
                                           : "kkt_km1_kernel<F64, " #COLSc ", " #Sc ", " #WSc ", " #KSc ", " #THRc "> (source-major TMA K1, one band per CTA, csrc/kkt_tma.cu)"))
    FWI_KM_DISPATCH(p->cols, p->stages, mb ? 1 : 0, p->ws, p->ks, p->thr, FWI_KM_LAUNCH);
#undef FWI_KM_LAUNCH
    CK_LAUNCH();
    if (trace_path) {
        std::vector<unsigned long long> h(size_t(5) * p->G);
        CK(cudaStreamSynchronize(c.stream));
        CK(cudaMemcpy(h.data(), p->trace.p, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        if (FILE* f = std::fopen(trace_path, "w")) {
            for (int b = 0; b < p->G; ++b)
                std::fprintf(f, "%d %llu %llu %llu %llu %llu\n", b, h[5 * b], h[5 * b + 1], h[5 * b + 2], h[5 * b + 3],
                             h[5 * b + 4]);
            std::fclose(f);
        }
    }
    return true;
}

}  // namespace

// Returns false when the TMA path does not apply (the caller then runs the
// plain kernel of kkt.cu): small problems (the single-pass plain kernel wins
// when everything is L2-resident) and layouts TMA cannot describe.
bool kkt_apply_tma(Ctx& c, bool f32, const void* xi, void* out) {
    // (FWI_KKT_F32_TMA=0 keeps the complex64 apply on the plain kernel)
    if (f32) {
        const char* e = std::getenv("FWI_KKT_F32_TMA");
        if (e && std::atoi(e) == 0) return false;
    }
    if (int64_t(c.K) * c.n < (int64_t(1) << 21) && !std::getenv("FWI_KKT_FORCE_TMA")) return false;
    const int64_t kn2s = 2 * int64_t(c.K) * c.n;
    if (c.kkt_variant == 0) {  // source-major kernel first
        KktKmPlan*& sp = c.kmplan[f32 ? 1 : 0];
        if (!sp) sp = f32 ? build_km_plan<F32>(c, true) : build_km_plan<F64>(c, false);
        if (sp->ok) {
            if (f32) {
                const float* x = static_cast<const float*>(xi);
                float* o = static_cast<float*>(out);
                return launch_km<F32>(c, sp, reinterpret_cast<const float2*>(x), x + kn2s,
                                      reinterpret_cast<const float2*>(x + kn2s + c.ds_stride),
                                      reinterpret_cast<float2*>(o), o + kn2s,
                                      reinterpret_cast<float2*>(o + kn2s + c.ds_stride), true);
            }
            const double* x = static_cast<const double*>(xi);
            double* o = static_cast<double*>(out);
            return launch_km<F64>(c, sp, reinterpret_cast<const double2*>(x), x + kn2s,
                                  reinterpret_cast<const double2*>(x + kn2s + c.ds_stride),
                                  reinterpret_cast<double2*>(o), o + kn2s,
                                  reinterpret_cast<double2*>(o + kn2s + c.ds_stride), false);
        }
    }
    KktPlan*& p = c.kplan[f32 ? 1 : 0];
    if (!p) p = f32 ? build_plan<F32>(c, true) : build_plan<F64>(c, false);
    if (!p->ok) return false;
    const int64_t kn2 = 2 * int64_t(c.K) * c.n;
    if (f32) {
        const float* x = static_cast<const float*>(xi);
        float* o = static_cast<float*>(out);
        return launch<F32>(c, p, reinterpret_cast<const float2*>(x), x + kn2,
                           reinterpret_cast<const float2*>(x + kn2 + c.ds_stride), reinterpret_cast<float2*>(o),
                           o + kn2, reinterpret_cast<float2*>(o + kn2 + c.ds_stride), true);
    }
    const double* x = static_cast<const double*>(xi);
    double* o = static_cast<double*>(out);
    return launch<F64>(c, p, reinterpret_cast<const double2*>(x), x + kn2,
                       reinterpret_cast<const double2*>(x + kn2 + c.ds_stride), reinterpret_cast<double2*>(o),
                       o + kn2, reinterpret_cast<double2*>(o + kn2 + c.ds_stride), false);
}

}  // namespace fwi_b200
