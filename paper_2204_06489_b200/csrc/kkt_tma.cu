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

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "arith.cuh"
#include "ctx.cuh"

namespace fwi_b200 {

namespace {

constexpr int kThreads = 512;
constexpr int kCols = 128;  // max strip width (columns per CTA)
constexpr int kRows = 8;    // rows per sub-tile (4 slots x 2 rows per thread)
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
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
        "%4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
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
    const int4* regions;  // x0, w, z0, h
    int BW, BWU;          // halo box width / u box width (complex elements)
    int stages, cm;
    uint32_t dub, ub, stage_bytes, tx_bytes;
};

template <class T>
__device__ __forceinline__ void st_stream(T* p, T v);
template <>
__device__ __forceinline__ void st_stream<double2>(double2* p, double2 v) { __stcs(p, v); }
template <>
__device__ __forceinline__ void st_stream<float2>(float2* p, float2 v) { __stcs(p, v); }

template <class A>
__global__ void __launch_bounds__(kThreads, 1)
    kkt_tma_kernel(const __grid_constant__ CUtensorMap tdu, const __grid_constant__ CUtensorMap tla,
                   const __grid_constant__ CUtensorMap tu, const TmaArgs<A> P) {
    using T = typename A::T;
    using R = typename A::R;
    extern __shared__ __align__(1024) unsigned char sm[];
    // mbarriers live in the dynamic allocation, after the stages (explicit layout)
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + size_t(P.stages) * P.stage_bytes);
    const int4 rg = P.regions[blockIdx.x];
    const int x0 = rg.x, w = rg.y, z0 = rg.z, h = rg.w;
    const int K = P.K, nx = P.nx, nz = P.nz, S = P.stages;
    const int nsub = (h + kRows - 1) / kRows;
    const int nsteps = nsub * K;
    const int tid = threadIdx.x, lx = tid & (kCols - 1), zs = tid >> 7;
    const int BW = P.BW, BWU = P.BWU;

    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    auto issue = [&](int j) {
        const int s = j % S;
        const int sub = j / K, k = j - sub * K;
        const int zt = z0 + kRows * sub;
        unsigned char* st = sm + size_t(s) * P.stage_bytes;
        mbar_expect_tx(&bar[s], P.tx_bytes);
        const int cm = P.cm;  // tensor elements per complex number
        tma_load_3d(st, &tdu, cm * (x0 - 1), zt - 1, k, &bar[s]);
        tma_load_3d(st + P.dub, &tdu, cm * (x0 - 1 + BW), zt - 1, k, &bar[s]);
        tma_load_3d(st + 2 * P.dub, &tla, cm * (x0 - 1), zt - 1, k, &bar[s]);
        tma_load_3d(st + 3 * P.dub, &tla, cm * (x0 - 1 + BW), zt - 1, k, &bar[s]);
        tma_load_3d(st + 4 * P.dub, &tu, cm * x0, zt, k, &bar[s]);
        tma_load_3d(st + 4 * P.dub + P.ub, &tu, cm * (x0 + BWU), zt, k, &bar[s]);
    };
    if (tid == 0)
        for (int j = 0; j < S && j < nsteps; ++j) issue(j);

    // per-node state for the current sub-tile (two rows per thread)
    bool act[2], hN[2], hW[2], hE[2], hS[2];
    T cD[2], cN[2], cW[2], cE[2], cS[2];
    R dsv[2], pl[2];
    int q[2], qe[2];
    int64_t cnode[2];

    for (int j = 0; j < nsteps; ++j) {
        const int sub = j / K, k = j - sub * K;
        if (k == 0) {
            const int zt = z0 + kRows * sub;
            const int ht = min(kRows, h - kRows * sub);
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int row = zs + 4 * r;
                act[r] = lx < w && row < ht;
                const int ix = x0 + lx, iz = zt + row;
                const int64_t c = act[r] ? int64_t(iz) * nx + ix : 0;
                cnode[r] = c;
                const bool bnd = on_boundary(ix, iz, nx, nz);
                hN[r] = act[r] && !bnd && !on_boundary(ix, iz - 1, nx, nz);
                hW[r] = act[r] && !bnd && !on_boundary(ix - 1, iz, nx, nz);
                hE[r] = act[r] && !bnd && !on_boundary(ix + 1, iz, nx, nz);
                hS[r] = act[r] && !bnd && !on_boundary(ix, iz + 1, nx, nz);
                cD[r] = act[r] ? P.diag[c] : A::zero();
                cN[r] = hN[r] ? P.south[c - nx] : A::zero();
                cW[r] = hW[r] ? P.east[c - 1] : A::zero();
                cE[r] = hE[r] ? P.east[c] : A::zero();
                cS[r] = hS[r] ? P.south[c] : A::zero();
                dsv[r] = act[r] ? P.ds[c] : R(0);
                q[r] = act[r] ? P.nrec_ptr[c] : 0;
                qe[r] = act[r] ? P.nrec_ptr[c + 1] : 0;
                pl[r] = R(0);
            }
        }
        const int s = j % S;
        mbar_wait(&bar[s], (j / S) & 1);
        const unsigned char* st = sm + size_t(s) * P.stage_bytes;
        const T* du0 = reinterpret_cast<const T*>(st);
        const T* du1 = reinterpret_cast<const T*>(st + P.dub);
        const T* la0 = reinterpret_cast<const T*>(st + 2 * P.dub);
        const T* la1 = reinterpret_cast<const T*>(st + 3 * P.dub);
        const T* u0 = reinterpret_cast<const T*>(st + 4 * P.dub);
        const T* u1 = reinterpret_cast<const T*>(st + 4 * P.dub + P.ub);
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            if (!act[r]) continue;
            const int row = zs + 4 * r;  // smem halo row = row + 1
            auto at = [&](const T* b0, const T* b1, int col, int ri) -> T {
                return col < BW ? b0[ri * BW + col] : b1[ri * BW + col - BW];
            };
            const int col = lx + 1;
            T s_ = A::zero(), t_ = A::zero();
            if (hN[r]) {
                s_ = A::add(s_, A::mul(cN[r], at(du0, du1, col, row)));
                t_ = A::add(t_, A::mulc(cN[r], at(la0, la1, col, row)));
            }
            if (hW[r]) {
                s_ = A::add(s_, A::mul(cW[r], at(du0, du1, col - 1, row + 1)));
                t_ = A::add(t_, A::mulc(cW[r], at(la0, la1, col - 1, row + 1)));
            }
            const T duc = at(du0, du1, col, row + 1);
            const T lac = at(la0, la1, col, row + 1);
            s_ = A::add(s_, A::mul(cD[r], duc));
            t_ = A::add(t_, A::mulc(cD[r], lac));
            if (hE[r]) {
                s_ = A::add(s_, A::mul(cE[r], at(du0, du1, col + 1, row + 1)));
                t_ = A::add(t_, A::mulc(cE[r], at(la0, la1, col + 1, row + 1)));
            }
            if (hS[r]) {
                s_ = A::add(s_, A::mul(cS[r], at(du0, du1, col, row + 2)));
                t_ = A::add(t_, A::mulc(cS[r], at(la0, la1, col, row + 2)));
            }
            const T uc = lx < BWU ? u0[row * BWU + lx] : u1[row * BWU + lx - BWU];
            const int64_t o = int64_t(k) * P.n + cnode[r];
            st_stream(P.ola + o, A::sub(s_, A::pmul(P.w2, uc, dsv[r])));
            if (q[r] < qe[r] && P.nrec_k[q[r]] == k) {
                T f = A::zero();
                while (q[r] < qe[r] && P.nrec_k[q[r]] == k) {
                    f = A::add(f, A::rm(R(P.nrec_w2[q[r]]), duc));
                    ++q[r];
                }
                t_ = A::add(f, t_);
            }
            st_stream(P.odu + o, t_);
            pl[r] = A::radd(pl[r], A::re_pconj(P.w2, uc, lac));
            if (k == K - 1) P.ods[cnode[r]] = A::rsub(A::rmulr(P.eps, dsv[r]), pl[r]);
        }
        __syncthreads();  // every thread is done with stage s
        if (tid == 0 && j + S < nsteps) issue(j + S);
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
    int G = 0, BW = 0, BWU = 0, stages = 0;
    uint32_t dub = 0, ub = 0, stage_bytes = 0, tx_bytes = 0;
    size_t smem = 0;
    DevBuf<int4> regions;
    CUtensorMap tm_u;
};

void kkt_plan_free(KktPlan* p) { delete p; }

namespace {

bool encode(CUtensorMap* tm, bool f32, const void* base, int nx, int nz, int K, int box_cplx, int box_rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    // complex128: two FLOAT64 elements per number; complex64: one 8-byte
    // element per number (the copy engine does not interpret the payload)
    const int cm = f32 ? 1 : 2;
    cuuint64_t dims[3] = {cuuint64_t(cm) * nx, cuuint64_t(nz), cuuint64_t(K)};
    cuuint64_t strides[2] = {cuuint64_t(nx) * (f32 ? 8 : 16), cuuint64_t(nx) * nz * (f32 ? 8 : 16)};
    cuuint32_t box[3] = {cuuint32_t(cm * box_cplx), cuuint32_t(box_rows), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    const CUresult r = fn(tm, f32 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                          const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <class A>
KktPlan* build_plan(Ctx& c, bool f32) {
    auto p = std::make_unique<KktPlan>();
    const int nx = c.nx, nz = c.nz;
    const int es = f32 ? 8 : 16;  // bytes per complex
    // TMA constraints: 16-byte global strides, 16-byte box rows
    if ((int64_t(2) * nx * (es / 2)) % 16 != 0) return p.release();
    if (!encode_fn()) return p.release();
    const int nsx = (nx + kCols - 1) / kCols;
    const int W = (nx + nsx - 1) / nsx;
    int BW = (W + 2 + 1) / 2, BWU = (W + 1) / 2;
    if (f32) {  // box rows must be multiples of 16 bytes
        BW = (BW + 1) / 2 * 2;
        BWU = (BWU + 1) / 2 * 2;
    }
    // regions: distribute the SMs over the strips in proportion to their width,
    // then split each strip's rows evenly among its bands
    const int G0 = sm_count();
    std::vector<int4> regs;
    int given = 0;
    for (int sidx = 0; sidx < nsx; ++sidx) {
        const int x0 = sidx * W, ws = std::min(W, nx - x0);
        int bands = (sidx == nsx - 1) ? G0 - given
                                      : int(std::lround(double(G0) * (x0 + ws) / nx)) - given;
        bands = std::max(1, std::min(bands, nz));
        given += bands;
        for (int b = 0; b < bands; ++b) {
            const int za = int(int64_t(nz) * b / bands), zb = int(int64_t(nz) * (b + 1) / bands);
            if (zb > za) regs.push_back(make_int4(x0, ws, za, zb - za));
        }
    }
    p->G = int(regs.size());
    p->regions.alloc(regs.size());
    CK(cudaMemcpy(p->regions.p, regs.data(), regs.size() * sizeof(int4), cudaMemcpyHostToDevice));
    p->BW = BW;
    p->BWU = BWU;
    p->dub = align128(size_t(BW) * kBH * es);
    p->ub = align128(size_t(BWU) * kRows * es);
    p->stage_bytes = 4 * p->dub + 2 * p->ub;
    p->tx_bytes = uint32_t(4 * size_t(BW) * kBH * es + 2 * size_t(BWU) * kRows * es);
    const size_t budget = 227 * 1024 - 256;
    p->stages = int(std::min<size_t>(kMaxStages, budget / p->stage_bytes));
    if (const char* e = std::getenv("FWI_KKT_STAGES")) p->stages = std::min(p->stages, std::max(1, std::atoi(e)));
    if (p->stages < 2) return p.release();
    p->smem = size_t(p->stages) * p->stage_bytes + kMaxStages * sizeof(uint64_t);
    // the attribute is per kernel and process-wide: only ever raise it
    static size_t smem_set = 0;
    if (p->smem > smem_set) {
        CK(cudaFuncSetAttribute(kkt_tma_kernel<A>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(p->smem)));
        smem_set = p->smem;
    }
    const void* ubase = f32 ? static_cast<const void*>(c.u32.p) : static_cast<const void*>(c.u.p);
    if (!ubase || !encode(&p->tm_u, f32, ubase, nx, nz, c.K, BWU, kRows)) return p.release();
    p->ok = true;
    return p.release();
}

template <class A>
bool launch(Ctx& c, KktPlan* p, const typename A::T* du, const typename A::R* ds, const typename A::T* la,
            typename A::T* odu, typename A::R* ods, typename A::T* ola, bool f32) {
    CUtensorMap tdu, tla;
    if (!encode(&tdu, f32, du, c.nx, c.nz, c.K, p->BW, kBH)) return false;
    if (!encode(&tla, f32, la, c.nx, c.nz, c.K, p->BW, kBH)) return false;
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
    a.regions = p->regions.p;
    a.BW = p->BW;
    a.BWU = p->BWU;
    a.stages = p->stages;
    a.cm = f32 ? 1 : 2;
    a.dub = p->dub;
    a.ub = p->ub;
    a.stage_bytes = p->stage_bytes;
    a.tx_bytes = p->tx_bytes;
    kkt_tma_kernel<A><<<p->G, kThreads, p->smem, c.stream>>>(tdu, tla, p->tm_u, a);
    CK_LAUNCH();
    return true;
}

}  // namespace

// Returns false when the TMA path does not apply (the caller then runs the
// plain kernel of kkt.cu).
bool kkt_apply_tma(Ctx& c, bool f32, const void* xi, void* out) {
    // The complex64 instantiation faults (illegal instruction) as soon as more
    // than one pipeline stage is in flight; until that is understood the
    // complex64 apply runs the plain kernel (FWI_KKT_F32_TMA=1 re-enables it).
    if (f32 && !std::getenv("FWI_KKT_F32_TMA")) return false;
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
