// common.cuh — shared device helpers and the device-side GnState.
//
// Bit-faithful complex arithmetic: the reference computes with libstdc++
// std::complex<double> built by g++ (no FMA on x86-64): a*b = (ac-bd, ad+bc)
// with every product and sum rounded, and a/b through libgcc's __divdc3
// (Smith's method). The helpers below use the __d*_rn intrinsics, which nvcc
// never contracts into FMA, so kernels that follow the reference's operation
// order reproduce its results bit for bit.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "fwi_b200.h"

namespace fwi_b200 {

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
struct FwiError : std::runtime_error {
    int code;
    int index;
    FwiError(int c, const std::string& m, int idx = -1) : std::runtime_error(m), code(c), index(idx) {}
};

[[noreturn]] inline void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
    const int code = (e == cudaErrorMemoryAllocation) ? FWI_ERR_OUT_OF_MEMORY : FWI_ERR_CUDA;
    throw FwiError(code, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                             std::to_string(line) + ")");
}

#define CK(x)                                                              \
    do {                                                                   \
        cudaError_t e__ = (x);                                             \
        if (e__ != cudaSuccess) ::fwi_b200::throw_cuda(e__, #x, __FILE__, __LINE__); \
    } while (0)

#define CK_LAUNCH() CK(cudaGetLastError())

inline void require(bool ok, const std::string& msg) {
    if (!ok) throw FwiError(FWI_ERR_INVALID_ARGUMENT, msg);
}

// ---------------------------------------------------------------------------
// programmatic dependent launch (the Krylov iteration's chain of short kernels)
// ---------------------------------------------------------------------------
// A kernel launched with launch_pdl may be scheduled while the previous kernel in the stream
// is still draining; pdl_enter() lets the next kernel be scheduled likewise and then waits
// until the previous grid has completed and its memory is visible (griddepcontrol.wait), so
// the kernel's own reads and writes are ordered exactly as in a plain stream launch. In a
// kernel launched without the attribute both instructions are no-ops. FWI_PDL=0 disables it.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}
// kernel groups (FWI_PDL_OFF=<mask> turns PDL off per group: 1 Krylov vector passes, 2 exact
// line solver, 4 cyclic reduction and dense GEMMs, 8 KKT apply, 16 preconditioner glue, 32 the fused
// MGS sweep)
enum { kPdlVec = 1, kPdlExact = 2, kPdlDense = 4, kPdlKkt = 8, kPdlPrecond = 16, kPdlMgs = 32 };
bool pdl_enabled(int group = 0);
template <int G, typename... KA, typename... A>
void launch_pdl(void (*k)(KA...), dim3 g, dim3 b, size_t smem, cudaStream_t st, A... args) {
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled(G) ? 1 : 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = g;
    cfg.blockDim = b;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k, static_cast<KA>(args)...));
}

// ---------------------------------------------------------------------------
// device buffers
// ---------------------------------------------------------------------------
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t count = 0;
    DevBuf() = default;
    explicit DevBuf(size_t n) { alloc(n); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), count(o.count) { o.p = nullptr; o.count = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; count = o.count; o.p = nullptr; o.count = 0; }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t n) {
        release();
        if (n) CK(cudaMalloc(&p, n * sizeof(T)));
        count = n;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        count = 0;
    }
    size_t bytes() const { return count * sizeof(T); }
    T* get() const { return p; }
};

// ---------------------------------------------------------------------------
// bit-faithful complex helpers (double2 = {re, im})
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ double2 cz() { return make_double2(0.0, 0.0); }

#ifdef __CUDACC__
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
    return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
    return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
}
// a * b  (libstdc++ / GCC expansion: re = ac - bd, im = ad + bc)
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                        __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
// conj(a) * b  ==  (ar br + ai bi, ar bi - ai br), bitwise equal to the
// expansion of std::conj(a) * b.
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
    return make_double2(__dadd_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                        __dsub_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
// real scalar * complex (each part multiplied once)
__device__ __forceinline__ double2 rmul(double r, double2 a) {
    return make_double2(__dmul_rn(r, a.x), __dmul_rn(r, a.y));
}
// libgcc __divdc3 (a+bi)/(c+di) for finite, normal-range operands (the
// power-of-two rescaling branches of libgcc are exact and do not change the
// result in that range).
__device__ __forceinline__ double2 cdiv(double2 n, double2 dd) {
    const double a = n.x, b = n.y, c = dd.x, d = dd.y;
    double x, y;
    if (fabs(c) < fabs(d)) {
        const double r = __ddiv_rn(c, d);
        const double den = __dadd_rn(__dmul_rn(c, r), d);
        x = __ddiv_rn(__dadd_rn(__dmul_rn(a, r), b), den);
        y = __ddiv_rn(__dsub_rn(__dmul_rn(b, r), a), den);
    } else {
        const double r = __ddiv_rn(d, c);
        const double den = __dadd_rn(__dmul_rn(d, r), c);
        x = __ddiv_rn(__dadd_rn(__dmul_rn(b, r), a), den);
        y = __ddiv_rn(__dsub_rn(b, __dmul_rn(a, r)), den);
    }
    return make_double2(x, y);
}
#endif

// the divisor-only part of cdiv / host_cdiv: returns |c| < |d| with r and den as cdiv forms them
inline bool host_cdiv_prep(double c, double d, double& r, double& den) {
    if (std::fabs(c) < std::fabs(d)) {
        r = c / d;
        den = c * r + d;
        return true;
    }
    r = d / c;
    den = d * r + c;
    return false;
}

// host twin of cdiv (used by the host-side ILU factorisation)
inline void host_cdiv(double a, double b, double c, double d, double& x, double& y) {
    if (std::fabs(c) < std::fabs(d)) {
        const double r = c / d;
        const double den = c * r + d;
        x = (a * r + b) / den;
        y = (b * r - a) / den;
    } else {
        const double r = d / c;
        const double den = d * r + c;
        x = (b * r + a) / den;
        y = (b - a * r) / den;
    }
}

// ---------------------------------------------------------------------------
// grid helpers
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ bool on_boundary(int ix, int iz, int nx, int nz) {
    return ix == 0 || iz == 0 || ix == nx - 1 || iz == nz - 1;
}

inline int grid_blocks(int64_t work, int threads, int max_blocks) {
    int64_t b = (work + threads - 1) / threads;
    if (b > max_blocks) b = max_blocks;
    if (b < 1) b = 1;
    return static_cast<int>(b);
}

int sm_count();
// page-locked host memory (host_mem.cu): huge-page mapping, parallel first touch,
// cudaHostRegister; zero-filled. pinned_free returns false for foreign pointers.
void* pinned_alloc(size_t bytes);
bool pinned_free(void* p);

}  // namespace fwi_b200
