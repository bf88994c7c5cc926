// vec.cu — K5: Krylov vector algebra on flat KKT vectors.
//
// Reference: KktVector dot/norm/axpy/scal (src/kkt.cpp:15-39) over
// vec.hpp:16-58, and the GMRES vector passes (include/fwi/krylov.hpp:181-237).
// By F4 a KKT vector is a flat array of 4Kn+n doubles and the KKT
// inner product is the plain real dot product of that array, so every
// operation here is real BLAS-1 on one contiguous buffer.
//
// Reductions are deterministic: a fixed grid (reduce_blocks()), fixed
// per-thread strides, a fixed shuffle tree, and the last CTA to finish sums
// the per-CTA partials in index order. Element-wise updates keep the
// reference's rounding (no FMA: y + (a*x) rounded twice).
#include <cstdlib>

#include "ctx.cuh"

namespace fwi_b200 {

namespace {

constexpr int kRedThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

// block sum in a fixed order; result valid in thread 0
__device__ __forceinline__ double block_sum(double v, double* sh) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double r = 0.0;
    if (wid == 0) {
        r = lane < (blockDim.x >> 5) ? sh[lane] : 0.0;
        r = warp_sum(r);
    }
    __syncthreads();
    return r;
}

// Combine per-CTA partials: the last CTA (ticket) sums them in index order.
__device__ __forceinline__ void finish_reduction(double part, double* partials, unsigned* ticket,
                                                 double* out) {
    __shared__ bool last;
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = part;
        __threadfence();
        const unsigned t = atomicAdd(ticket, 1u);
        last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    __shared__ double sh[32];
    double v = 0.0;
    for (int i = threadIdx.x; i < gridDim.x; i += blockDim.x) v += __ldcg(partials + i);
    v = block_sum(v, sh);
    if (threadIdx.x == 0) {
        *out = v;
        *ticket = 0u;
    }
}

__global__ void __launch_bounds__(kRedThreads) dot_kernel(const double2* __restrict__ x,
                                                          const double2* __restrict__ y, int64_t m,
                                                          double* partials, unsigned* ticket,
                                                          double* out) {
    pdl_enter();
    __shared__ double sh[32];
    double acc = 0.0;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    for (; i + 3 * stride < m; i += 4 * stride) {  // loads first, same accumulation order
        double2 a[4], b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            a[u] = x[i + u * stride];
            b[u] = y[i + u * stride];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc += a[u].x * b[u].x + a[u].y * b[u].y;
    }
    for (; i < m; i += stride) {
        const double2 a = x[i], b = y[i];
        acc += a.x * b.x + a.y * b.y;
    }
    acc = block_sum(acc, sh);
    finish_reduction(acc, partials, ticket, out);
}

__global__ void axpy_kernel(double a, const double2* __restrict__ x, double2* __restrict__ y, int64_t m) {
    pdl_enter();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m;
         i += int64_t(gridDim.x) * blockDim.x) {
        const double2 xv = x[i];
        double2 yv = y[i];
        yv.x = __dadd_rn(yv.x, __dmul_rn(a, xv.x));
        yv.y = __dadd_rn(yv.y, __dmul_rn(a, xv.y));
        y[i] = yv;
    }
}

__global__ void scal_kernel(double a, double2* __restrict__ x, int64_t m) {
    pdl_enter();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m;
         i += int64_t(gridDim.x) * blockDim.x) {
        double2 v = x[i];
        v.x = __dmul_rn(a, v.x);
        v.y = __dmul_rn(a, v.y);
        x[i] = v;
    }
}


// One thread's share of an MGS step, w -= h_{i-1} v_{i-1}; acc += <v_i, w>, over its
// grid-stride elements in order. The loads of U elements are issued before any of
// them is used (memory-level parallelism); the accumulation order is unchanged.
constexpr int kMgsUnroll = 8;
__device__ __forceinline__ void mgs_elem(double2& wv, const double2& pv, const double2& nv, double nh, bool prev,
                                         bool next, double& acc) {
    if (prev) {
        wv.x = __dadd_rn(wv.x, __dmul_rn(nh, pv.x));
        wv.y = __dadd_rn(wv.y, __dmul_rn(nh, pv.y));
    }
    const double2 n = next ? nv : wv;
    acc += n.x * wv.x + n.y * wv.y;
}
// L2 hints for the device-resident sweep: w (read and written by every step) is kept
// in L2 (evict_last) while the basis vectors stream through (evict_first), so a step
// costs ~2 vector reads of DRAM instead of 4 when w fits in L2 (config 3: 76 MB of 126).
__device__ __forceinline__ uint64_t l2_policy_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double2 ld_hint(const double2* p, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_hint(double2* p, double2 v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y),
                 "l"(pol)
                 : "memory");
}
// streamed once: no L1 allocation (stores allocating in the L1 cost bandwidth on this part)
__device__ __forceinline__ void st_na(double2* p, double2 v) {
    asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ double2 ld_na(const double2* p) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}

template <bool HINT = false, int U = kMgsUnroll>
__device__ __forceinline__ double mgs_pass(double2* __restrict__ w, const double2* __restrict__ vprev, double nh,
                                           const double2* __restrict__ vnext, int64_t m, int64_t t0, int64_t stride,
                                           bool release = false, double acc0 = 0.0) {
    double acc = acc0;
    int64_t t = t0;
    uint64_t keep = 0, stream = 0;
    if (HINT) {
        // the sweep's last step hands w back to normal priority for the kernels after it
        keep = release ? l2_policy_first() : l2_policy_last();
        stream = l2_policy_first();
    }
    for (; t + (U - 1) * stride < m; t += U * stride) {
        double2 wv[U], pv[U], nv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            wv[u] = HINT ? ld_hint(w + t + u * stride, keep) : w[t + u * stride];
            pv[u] = vprev ? (HINT ? ld_hint(vprev + t + u * stride, stream) : vprev[t + u * stride])
                          : make_double2(0.0, 0.0);
            nv[u] = vnext ? (HINT ? ld_hint(vnext + t + u * stride, stream) : vnext[t + u * stride])
                          : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            mgs_elem(wv[u], pv[u], nv[u], nh, vprev != nullptr, vnext != nullptr, acc);
            if (vprev) {
                if (HINT) st_hint(w + t + u * stride, wv[u], keep);
                else w[t + u * stride] = wv[u];
            }
        }
    }
    for (; t < m; t += stride) {
        double2 wv = w[t];
        const double2 pv = vprev ? vprev[t] : make_double2(0.0, 0.0);
        const double2 nv = vnext ? vnext[t] : make_double2(0.0, 0.0);
        mgs_elem(wv, pv, nv, nh, vprev != nullptr, vnext != nullptr, acc);
        if (vprev) w[t] = wv;
    }
    return acc;
}

// MGS step (krylov.hpp:183-186), fused: w -= h_{i-1} v_{i-1} (h read from
// device memory, no host round trip), then h_i = <v_i, w> (or <w, w> when
// vnext is null, for ||w||).
__global__ void __launch_bounds__(kRedThreads) mgs_kernel(double2* __restrict__ w,
                                                          const double2* __restrict__ vprev,
                                                          const double* __restrict__ hprev,
                                                          const double2* __restrict__ vnext, int64_t m,
                                                          double* partials, unsigned* ticket,
                                                          double* out) {
    pdl_enter();
    __shared__ double sh[32];
    const double nh = vprev ? -*hprev : 0.0;
    double acc = mgs_pass(w, vprev, nh, vnext, m, blockIdx.x * int64_t(blockDim.x) + threadIdx.x,
                          int64_t(gridDim.x) * blockDim.x);
    acc = block_sum(acc, sh);
    finish_reduction(acc, partials, ticket, out);
}

// The same fused MGS step over one chunk of the vector, leaving its per-CTA
// partial sums in partials_out (host-resident basis: chunks are staged through
// device buffers and the partials of all chunks are summed in order afterwards).
__global__ void __launch_bounds__(kRedThreads) mgs_partial_kernel(double2* __restrict__ w,
                                                                  const double2* __restrict__ vprev,
                                                                  const double* __restrict__ hprev,
                                                                  const double2* __restrict__ vnext, int64_t m,
                                                                  double* partials_out) {
    pdl_enter();
    __shared__ double sh[32];
    const double nh = vprev ? -*hprev : 0.0;
    double acc = mgs_pass(w, vprev, nh, vnext, m, blockIdx.x * int64_t(blockDim.x) + threadIdx.x,
                          int64_t(gridDim.x) * blockDim.x);
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) partials_out[blockIdx.x] = acc;
}

__global__ void __launch_bounds__(kRedThreads) sum_ordered_kernel(const double* __restrict__ p, int count,
                                                                  double* out) {
    pdl_enter();
    __shared__ double sh[32];
    double v = 0.0;
    for (int i = threadIdx.x; i < count; i += blockDim.x) v += p[i];
    v = block_sum(v, sh);
    if (threadIdx.x == 0) *out = v;
}

// The whole MGS sweep of one GMRES iteration in one launch (device-resident
// basis): for i = 0..m, w -= h_{i-1} v_{i-1}; h_i = <v_i, w> (v_m := w, the norm).
// Every step is the same grid-stride pass and the same ordered partial sum as
// mgs_kernel, so the h values are bit-identical to m+1 separate launches; the
// steps are separated by a software grid barrier (the grid is sized to be
// co-resident): the last CTA of a step sums the partials and publishes h_i.
struct MgsAllArgs {
    const double2* v[64];
};

// QS > 0 (streaming form, vectors far beyond the registers): the first QS of a thread's
// grid-stride elements of w live in shared memory for the whole sweep, so only the rest of w
// streams through L2 (config 3: 16 of 62 elements) and fewer of its dirty lines are written back
// between steps. Same elements, same accumulation order (bit-identical to the plain streaming form).
template <int QMAX, int QS = 0>
__global__ void __launch_bounds__(kRedThreads, 2) mgs_all_kernel(double2* __restrict__ w, MgsAllArgs a, int m,
                                                              int64_t len2, double* partials, unsigned* ticket,
                                                              volatile unsigned* flag, unsigned epoch, double* h) {
    pdl_enter();
    __shared__ double sh[32];
    __shared__ bool last;
    extern __shared__ double2 wsm[];  // QS > 0: [QS][blockDim.x]
    // QMAX > 0: this thread's grid-stride elements of w (at most QMAX) stay in registers
    // for the whole sweep and the next basis vector's elements are loaded before the
    // grid barrier; same elements, same order of accumulation as the streaming form.
    const int64_t stride = int64_t(gridDim.x) * blockDim.x, t0 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    double2 wq[QMAX > 0 ? QMAX : 1], nq[QMAX > 0 ? QMAX : 1], pq[QMAX > 0 ? QMAX : 1];
    if constexpr (QMAX > 0) {
#pragma unroll
        for (int q = 0; q < QMAX; ++q) {
            const int64_t t = t0 + q * stride;
            wq[q] = t < len2 ? w[t] : make_double2(0.0, 0.0);
            nq[q] = (t < len2 && m > 0) ? a.v[0][t] : make_double2(0.0, 0.0);
        }
    }
    if constexpr (QS > 0) {
        for (int q = 0; q < QS; ++q) {
            const int64_t t = t0 + q * stride;
            wsm[q * blockDim.x + threadIdx.x] = t < len2 ? w[t] : make_double2(0.0, 0.0);
        }
    }
    for (int i = 0; i <= m; ++i) {
        const double2* vprev = i > 0 ? a.v[i - 1] : nullptr;
        const double2* vnext = i < m ? a.v[i] : nullptr;
        const double nh = vprev ? -__ldcg(h + i - 1) : 0.0;  // published by another CTA: bypass L1
        double acc = 0.0;
        if constexpr (QMAX > 0) {
#pragma unroll
            for (int q = 0; q < QMAX; ++q) {
                const int64_t t = t0 + q * stride;
                if (t < len2) {
                    double2 wv = wq[q];
                    if (vprev) {
                        const double2 pv = pq[q];  // v_{i-1}: the previous step's vnext
                        wv.x = __dadd_rn(wv.x, __dmul_rn(nh, pv.x));
                        wv.y = __dadd_rn(wv.y, __dmul_rn(nh, pv.y));
                        wq[q] = wv;
                    }
                    const double2 nv = vnext ? nq[q] : wv;
                    acc += nv.x * wv.x + nv.y * wv.y;
                }
            }
#pragma unroll
            for (int q = 0; q < QMAX; ++q) {  // v_i becomes the next step's vprev; prefetch v_{i+1}
                const int64_t t = t0 + q * stride;
                pq[q] = nq[q];
                if (i + 1 < m && t < len2) nq[q] = a.v[i + 1][t];
            }
        } else if constexpr (QS > 0) {
            const uint64_t stream = l2_policy_first();
            constexpr int U = 4;
#pragma unroll 1
            for (int q0 = 0; q0 < QS; q0 += U) {
                double2 pv[U], nv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t t = t0 + int64_t(q0 + u) * stride;
                    const bool ok = q0 + u < QS && t < len2;
                    pv[u] = (vprev && ok) ? ld_hint(vprev + t, stream) : make_double2(0.0, 0.0);
                    nv[u] = (vnext && ok) ? ld_hint(vnext + t, stream) : make_double2(0.0, 0.0);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t t = t0 + int64_t(q0 + u) * stride;
                    if (q0 + u >= QS || t >= len2) continue;
                    double2& ws = wsm[(q0 + u) * blockDim.x + threadIdx.x];
                    double2 wv = ws;
                    mgs_elem(wv, pv[u], nv[u], nh, vprev != nullptr, vnext != nullptr, acc);
                    if (vprev) ws = wv;
                }
            }
            acc = mgs_pass<true>(w, vprev, nh, vnext, len2, t0 + int64_t(QS) * stride, stride, i == m, acc);
        } else {
            acc = mgs_pass<true>(w, vprev, nh, vnext, len2, t0, stride, i == m);
        }
        acc = block_sum(acc, sh);
        if (threadIdx.x == 0) {
            partials[blockIdx.x] = acc;
            __threadfence();
            last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
        }
        __syncthreads();
        if (last) {  // same ordered combine as finish_reduction
            __threadfence();
            double v = 0.0;
            for (int q = threadIdx.x; q < gridDim.x; q += blockDim.x) v += __ldcg(partials + q);
            v = block_sum(v, sh);
            if (threadIdx.x == 0) {
                h[i] = v;
                *ticket = 0u;
                __threadfence();
                flag[0] = epoch + unsigned(i) + 1u;
            }
        }
        if (threadIdx.x == 0)
            while (flag[0] < epoch + unsigned(i) + 1u) __nanosleep(32);
        __syncthreads();
        __threadfence();
    }
    if constexpr (QMAX > 0) {
#pragma unroll
        for (int q = 0; q < QMAX; ++q) {
            const int64_t t = t0 + q * stride;
            if (t < len2) w[t] = wq[q];
        }
    }
    if constexpr (QS > 0) {
        for (int q = 0; q < QS; ++q) {
            const int64_t t = t0 + q * stride;
            if (t < len2) w[t] = wsm[q * blockDim.x + threadIdx.x];
        }
    }
}

struct MultiAxpyArgs {
    const double2* v[64];
};

// x_cand = x + sum_i y_i v_i with the reference's sequential rounding
// (krylov.hpp:231-232: one axpy per basis vector, in order).
__global__ void multi_axpy_kernel(double2* __restrict__ out, const double2* __restrict__ x,
                                  MultiAxpyArgs args, const double* __restrict__ y, int mvec,
                                  int64_t m) {
    pdl_enter();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m;
         i += int64_t(gridDim.x) * blockDim.x) {
        double2 acc = x ? ld_na(x + i) : make_double2(0.0, 0.0);
        for (int j = 0; j < mvec; ++j) {
            const double yj = y[j];
            const double2 v = ld_na(args.v[j] + i);
            acc.x = __dadd_rn(acc.x, __dmul_rn(yj, v.x));
            acc.y = __dadd_rn(acc.y, __dmul_rn(yj, v.y));
        }
        st_na(out + i, acc);
    }
}

// ||b - ax||^2 without materialising the residual (krylov.hpp:234-237)
__global__ void __launch_bounds__(kRedThreads) sub_norm2_kernel(const double2* __restrict__ b,
                                                                const double2* __restrict__ ax, int64_t m,
                                                                double* partials, unsigned* ticket,
                                                                double* out) {
    pdl_enter();
    __shared__ double sh[32];
    double acc = 0.0;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    for (; i + 3 * stride < m; i += 4 * stride) {  // loads first, same accumulation order
        double2 bv[4], av[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            bv[u] = b[i + u * stride];
            av[u] = ax[i + u * stride];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double rx = __dsub_rn(bv[u].x, av[u].x), ry = __dsub_rn(bv[u].y, av[u].y);
            acc += rx * rx + ry * ry;
        }
    }
    for (; i < m; i += stride) {
        const double2 bv = b[i], av = ax[i];
        const double rx = __dsub_rn(bv.x, av.x), ry = __dsub_rn(bv.y, av.y);
        acc += rx * rx + ry * ry;
    }
    acc = block_sum(acc, sh);
    finish_reduction(acc, partials, ticket, out);
}

}  // namespace

int reduce_blocks() { return 2 * sm_count(); }

static int ew_blocks(int64_t m) { return grid_blocks(m, 256, 16 * sm_count()); }

void dev_dot_async(cudaStream_t st, const double* x, const double* y, double* out_dev,
                   double* partials, unsigned* ticket, int64_t len) {
    launch_pdl<kPdlVec>(dot_kernel, dim3(reduce_blocks()), dim3(kRedThreads), 0, st,
                        reinterpret_cast<const double2*>(x), reinterpret_cast<const double2*>(y), len / 2, partials,
                        ticket, out_dev);
    CK_LAUNCH();
}

double dev_dot(Ctx* c, cudaStream_t st, const double* x, const double* y, int64_t len) {
    dev_dot_async(st, x, y, c->red_out.p, c->red_partials.p, c->red_ticket.p, len);
    double h = 0.0;
    CK(cudaMemcpyAsync(&h, c->red_out.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return h;
}

void dev_axpy(cudaStream_t st, double a, const double* x, double* y, int64_t len) {
    launch_pdl<kPdlVec>(axpy_kernel, dim3(ew_blocks(len / 2)), dim3(256), 0, st, a, reinterpret_cast<const double2*>(x),
                        reinterpret_cast<double2*>(y), len / 2);
    CK_LAUNCH();
}

void dev_scal(cudaStream_t st, double a, double* x, int64_t len) {
    launch_pdl<kPdlVec>(scal_kernel, dim3(ew_blocks(len / 2)), dim3(256), 0, st, a, reinterpret_cast<double2*>(x),
                        len / 2);
    CK_LAUNCH();
}

// x *= 1 / sqrt(*h2): the basis normalisation v_{j+1} = w / ||w|| with ||w||^2 read from the
// device (the MGS kernel's last h), rounded as the host's 1.0 / std::sqrt(h2)
__global__ void scal_rsqrt_kernel(const double* __restrict__ h2, double2* __restrict__ x, int64_t m) {
    pdl_enter();
    const double a = __ddiv_rn(1.0, __dsqrt_rn(__ldg(h2)));
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m;
         i += int64_t(gridDim.x) * blockDim.x) {
        double2 v = x[i];
        v.x = __dmul_rn(a, v.x);
        v.y = __dmul_rn(a, v.y);
        x[i] = v;
    }
}

void dev_scal_rsqrt(cudaStream_t st, const double* h2_dev, double* x, int64_t len) {
    launch_pdl<kPdlVec>(scal_rsqrt_kernel, dim3(ew_blocks(len / 2)), dim3(256), 0, st, h2_dev,
                        reinterpret_cast<double2*>(x), len / 2);
    CK_LAUNCH();
}

void dev_mgs_step(cudaStream_t st, double* w, const double* vprev, const double* hprev_dev,
                  const double* vnext, double* h_out_dev, double* partials, unsigned* ticket,
                  int64_t len) {
    launch_pdl<kPdlVec>(mgs_kernel, dim3(reduce_blocks()), dim3(kRedThreads), 0, st, reinterpret_cast<double2*>(w),
                        reinterpret_cast<const double2*>(vprev), hprev_dev, reinterpret_cast<const double2*>(vnext),
                        len / 2, partials, ticket, h_out_dev);
    CK_LAUNCH();
}

void dev_mgs_step_parts(cudaStream_t st, double* w, const double* vprev, const double* hprev_dev,
                        const double* vnext, double* partials_out, int64_t len) {
    launch_pdl<kPdlVec>(mgs_partial_kernel, dim3(reduce_blocks()), dim3(kRedThreads), 0, st,
                        reinterpret_cast<double2*>(w), reinterpret_cast<const double2*>(vprev), hprev_dev,
                        reinterpret_cast<const double2*>(vnext), len / 2, partials_out);
    CK_LAUNCH();
}

bool dev_mgs_all(cudaStream_t st, double* w, const double* const* v, int m, double* h_dev, double* partials,
                 unsigned* ticket, unsigned* flag, unsigned& epoch, int64_t len) {
    if (m + 1 > 64) return false;
    // co-residency of the software grid barrier: reduce_blocks() CTAs of 256 threads
    // (every variant that may launch: the grid barrier needs all its CTAs resident at once)
    // shared-memory-resident elements of w per thread in the streaming form (FWI_MGS_QS=16|24, 0 =
    // off): C3 560 -> 588 it/s with either (w's L2 footprint 76 -> 57 or 47 MB)
    static const int qsel = std::getenv("FWI_MGS_QS") ? std::atoi(std::getenv("FWI_MGS_QS")) : 16;
    const int kQS = qsel == 16 ? 16 : qsel == 24 ? 24 : 0;
    const size_t kQSmem = size_t(kQS) * kRedThreads * sizeof(double2);
    using MgsKern = void (*)(double2*, MgsAllArgs, int, int64_t, double*, unsigned*, volatile unsigned*, unsigned,
                             double*);
    const MgsKern qs_kernel = kQS == 24 ? mgs_all_kernel<0, 24> : mgs_all_kernel<0, 16>;
    static int ok = -1, ok_qs = -1;
    if (ok < 0) {
        ok = 1;
        for (const void* k : {reinterpret_cast<const void*>(mgs_all_kernel<0>),
                              reinterpret_cast<const void*>(mgs_all_kernel<2>),
                              reinterpret_cast<const void*>(mgs_all_kernel<4>)}) {
            int per_sm = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kRedThreads, 0) != cudaSuccess ||
                per_sm * sm_count() < reduce_blocks())
                ok = 0;
        }
        int per_sm = 0;
        ok_qs = kQS > 0 &&
                cudaFuncSetAttribute(qs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kQSmem)) ==
                    cudaSuccess &&
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qs_kernel, kRedThreads, kQSmem) ==
                    cudaSuccess &&
                per_sm * sm_count() >= reduce_blocks();
        cudaGetLastError();
    }
    if (!ok) return false;
    MgsAllArgs a{};
    for (int i = 0; i < m; ++i) a.v[i] = reinterpret_cast<const double2*>(v[i]);
    const int64_t len2 = len / 2, per = int64_t(reduce_blocks()) * kRedThreads;
    auto go = [&](auto kern) {
        launch_pdl<kPdlMgs>(kern, dim3(reduce_blocks()), dim3(kRedThreads), 0, st, reinterpret_cast<double2*>(w), a, m,
                            len2, partials, ticket, flag, epoch, h_dev);
    };
    if (len2 <= 2 * per) {
        go(mgs_all_kernel<2>);
    } else if (len2 <= 4 * per) {
        go(mgs_all_kernel<4>);
    } else if (ok_qs && len2 >= int64_t(2 * kQS) * per) {
        launch_pdl<kPdlMgs>(qs_kernel, dim3(reduce_blocks()), dim3(kRedThreads), kQSmem, st,
                            reinterpret_cast<double2*>(w), a, m, len2, partials, ticket, flag, epoch, h_dev);
    } else {
        go(mgs_all_kernel<0>);
    }
    CK_LAUNCH();
    epoch += unsigned(m) + 1u;
    return true;
}

void dev_sum_ordered(cudaStream_t st, const double* partials, int count, double* out_dev) {
    launch_pdl<kPdlVec>(sum_ordered_kernel, dim3(1), dim3(kRedThreads), 0, st, partials, count, out_dev);
    CK_LAUNCH();
}

void dev_multi_axpy(cudaStream_t st, double* out, const double* x, const double* const* v,
                    const double* y_dev, int m, int64_t len) {
    MultiAxpyArgs a{};
    require(m <= 64, "gmres: restart larger than 63 is not supported by the fused update");
    for (int i = 0; i < m; ++i) a.v[i] = reinterpret_cast<const double2*>(v[i]);
    launch_pdl<kPdlVec>(multi_axpy_kernel, dim3(ew_blocks(len / 2)), dim3(256), 0, st, reinterpret_cast<double2*>(out),
                        reinterpret_cast<const double2*>(x), a, y_dev, m, len / 2);
    CK_LAUNCH();
}

void dev_sub_norm2(cudaStream_t st, const double* b, const double* ax, double* out_dev,
                   double* partials, unsigned* ticket, int64_t len) {
    launch_pdl<kPdlVec>(sub_norm2_kernel, dim3(reduce_blocks()), dim3(kRedThreads), 0, st,
                        reinterpret_cast<const double2*>(b), reinterpret_cast<const double2*>(ax), len / 2, partials,
                        ticket, out_dev);
    CK_LAUNCH();
}

}  // namespace fwi_b200
