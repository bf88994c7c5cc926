// gmres.cu — restarted, left-preconditioned GMRES on device-resident vectors
// (the reference's template, include/fwi/krylov.hpp:128-269, with S = double
// as the KKT inner product is real) and fsgn_gmres_step
// (src/kkt.cpp:137-171).
//
// Control flow, Hessenberg/Givens arithmetic, the triangular y-solve,
// stagnation and best-iterate rules are the reference's, on the host, in
// double. Every vector pass runs on the device: the MGS steps are fused
// "w -= h_{i-1} v_{i-1}; h_i = <v_i, w>" kernels whose h values stay in device
// memory until one D2H copy per iteration; x_cand = x + V y is one fused pass
// with the reference's per-basis-vector rounding order; the true residual
// ||b - A x_cand|| is a KKT apply plus one fused difference-norm pass.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <cmath>
#include <functional>
#include <memory>
#include <future>
#include <optional>

#include "ctx.cuh"

namespace fwi_b200 {

void reduced_gradient(Ctx& c, double* g_dev);
void reduced_hessian(Ctx& c, const double* v_dev, double* out_dev);

namespace {

struct Entry {
    int iteration;
    double residual_norm;
    std::optional<double> normal_residual;
    std::optional<double> precond_residual;
    double wall_time;
};

struct Log {
    std::vector<Entry> entries;
    bool converged = false;
    bool stagnated = false;
};

struct GmresOps {
    int64_t len = 0;
    cudaStream_t st = nullptr;
    std::function<void(const double*, double*)> apply, precond;
    // optional: the operator on a second stream, concurrent with apply/precond on st (lets the
    // pipelined loop run x_cand and the true residual beside the next iteration)
    std::function<void(const double*, double*, cudaStream_t)> apply_alt;
    std::function<bool(int, const double*)> observer;  // may be empty
};

struct Scratch {
    DevBuf<double> partials, out;
    DevBuf<unsigned> ticket, flag;
    unsigned epoch = 0;  // grid-barrier generation of the fused MGS kernel
    Scratch() {
        partials.alloc(4096);
        out.alloc(256);
        ticket.alloc(64);
        flag.alloc(1);
        CK(cudaMemset(ticket.p, 0, 64 * sizeof(unsigned)));
        CK(cudaMemset(flag.p, 0, sizeof(unsigned)));
    }
};

}  // namespace

// Krylov buffers kept by a context between solves: cudaMalloc/cudaFree serialise the
// device, and a solve allocates ~restart+6 vectors (≈10 ms of allocation at config 1,
// where a whole GMRES iteration takes ~0.7 ms). Host-basis solves (config 5) do not keep
// their 17 GB vectors.
struct GmresWork {
    int64_t len = 0;
    std::vector<DevBuf<double>> vecs;
    DevBuf<double> hdev, ydev;
    Scratch sc;
    // device-side Givens state of the pipelined loop (gmres_core): Hessenberg columns, rotations,
    // g; per-iteration status slots (||b - A x_cand||^2, ||w||, |g_{j+1}|) copied to pinned memory
    DevBuf<double> gst, stat;
    double* hstat = nullptr;
    cudaEvent_t ev_stat[2] = {nullptr, nullptr};
    int gst_restart = 0;
    // the residual branch's stream (x_cand, A x_cand, its norm), its reduction scratch, and the
    // events ordering it against the main chain
    cudaStream_t s2 = nullptr;
    std::unique_ptr<Scratch> sc2;
    cudaEvent_t ev_mgs[2] = {nullptr, nullptr}, ev_x = nullptr;
    ~GmresWork() {
        if (s2) cudaStreamSynchronize(s2);
        if (hstat) cudaFreeHost(hstat);
        for (auto& e : ev_stat)
            if (e) cudaEventDestroy(e);
        for (auto& e : ev_mgs)
            if (e) cudaEventDestroy(e);
        if (ev_x) cudaEventDestroy(ev_x);
        if (s2) cudaStreamDestroy(s2);
    }
    void second_stream() {
        if (s2) return;
        CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
        sc2 = std::make_unique<Scratch>();
        for (auto& e : ev_mgs) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ev_x, cudaEventDisableTiming));
    }
    void pipeline(int restart) {
        if (gst_restart < restart) {
            gst.alloc(size_t(restart) * (restart + 2) + 3 * size_t(restart) + 4);
            gst_restart = restart;
        }
        if (!hstat) {
            stat.alloc(8);
            CK(cudaHostAlloc(reinterpret_cast<void**>(&hstat), 8 * sizeof(double), cudaHostAllocDefault));
            for (auto& e : ev_stat) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
    }
    DevBuf<double> take(int64_t n) {
        if (n != len) {
            vecs.clear();
            len = n;
        }
        if (!vecs.empty()) {
            DevBuf<double> b = std::move(vecs.back());
            vecs.pop_back();
            return b;
        }
        return DevBuf<double>(size_t(n));
    }
    void give(DevBuf<double>&& b) {
        if (b.p && int64_t(b.count) == len) vecs.push_back(std::move(b));
    }
    void small(int restart) {
        if (hdev.count < 2 * (size_t(restart) + 2)) hdev.alloc(2 * (size_t(restart) + 2));  // two slots
        if (ydev.count < size_t(restart) + 1) ydev.alloc(size_t(restart) + 1);
    }
};

void gmres_work_free(GmresWork* w) { delete w; }

namespace {

// The reference's Givens step and triangular y-solve (include/fwi/krylov.hpp:190-230, S = double)
// for column j, on the device so the iteration needs no host round trip: the same operations
// in the same order as the host code in gmres_core, each rounded explicitly (no contraction),
// so h, the rotations, g and y are bit-identical to it. h_dev: the MGS kernel's h_0..h_{j+1}
// (h_{j+1} = ||w||^2). Layout of gst (restart R): H (column-major, R+2 per column), c[R], s[R],
// g[R+2]. stat: [1] = ||w||, [2] = |g_{j+1}|; y_dev: y_0..y_j.
__global__ void __launch_bounds__(32) givens_kernel(const double* __restrict__ h_dev, int j, int R,
                                                    double* __restrict__ gst, double* __restrict__ y_dev,
                                                    double* __restrict__ stat) {
    pdl_enter();
    // the warp stages columns 0..j of H (rows 0..j+1), the rotations and g in shared memory
    // (one round of loads instead of a dependent global load per operation); lane 0 computes
    extern __shared__ double gs_sm[];
    const int P = R + 2;
    double* Hs = gs_sm;                       // (j+1) columns of pitch P
    double* cs = Hs + size_t(j + 1) * P;      // c[0..j], s[0..j]
    double* ss = cs + (j + 1);
    double* gg = ss + (j + 1);                // g[0..j+1]
    double* ys = gg + (j + 2);                // y[0..j]
    double* H = gst;
    double* gc = gst + size_t(R) * P;
    double* gsn = gc + R;
    double* g = gsn + R;
    const int lane = threadIdx.x;
    for (int q = lane; q < j * P; q += 32) Hs[q] = H[q];  // columns 0..j-1
    for (int q = lane; q <= j + 1; q += 32) Hs[size_t(j) * P + q] = h_dev[q];
    for (int q = lane; q < j; q += 32) {
        cs[q] = gc[q];
        ss[q] = gsn[q];
    }
    for (int q = lane; q <= j; q += 32) gg[q] = g[q];
    __syncwarp();
    if (lane == 0) {
        double* h = Hs + size_t(j) * P;
        const double wn = __dsqrt_rn(h[j + 1]);
        h[j + 1] = wn;
        for (int i = 0; i < j; ++i) {
            const double t = __dadd_rn(__dmul_rn(cs[i], h[i]), __dmul_rn(ss[i], h[i + 1]));
            h[i + 1] = __dadd_rn(__dmul_rn(-ss[i], h[i]), __dmul_rn(cs[i], h[i + 1]));
            h[i] = t;
        }
        double c, s, rr;
        const double an = fabs(h[j]), bn = fabs(h[j + 1]);
        const double t = __dsqrt_rn(__dadd_rn(__dmul_rn(an, an), __dmul_rn(bn, bn)));
        if (bn == 0.0) {
            c = 1.0;
            s = 0.0;
            rr = h[j];
        } else if (an == 0.0) {
            c = 0.0;
            s = __ddiv_rn(h[j + 1], bn);
            rr = bn;
        } else {
            c = __ddiv_rn(an, t);
            s = __ddiv_rn(__dmul_rn(__ddiv_rn(h[j], an), h[j + 1]), t);
            rr = __dmul_rn(__ddiv_rn(h[j], an), t);
        }
        cs[j] = c;
        ss[j] = s;
        h[j] = rr;
        h[j + 1] = 0.0;
        gg[j + 1] = __dmul_rn(-s, gg[j]);
        gg[j] = __dmul_rn(c, gg[j]);
        for (int i = j; i >= 0; --i) {
            double acc = gg[i];
            for (int k2 = i + 1; k2 <= j; ++k2) acc = __dsub_rn(acc, __dmul_rn(Hs[size_t(k2) * P + i], ys[k2]));
            ys[i] = __ddiv_rn(acc, Hs[size_t(i) * P + i]);
        }
        gc[j] = c;
        gsn[j] = s;
        g[j] = gg[j];
        g[j + 1] = gg[j + 1];
        stat[1] = wn;
        stat[2] = fabs(gg[j + 1]);
    }
    __syncwarp();
    for (int q = lane; q <= j + 1; q += 32) H[size_t(j) * P + q] = Hs[size_t(j) * P + q];
    for (int q = lane; q <= j; q += 32) y_dev[q] = ys[q];
}

__global__ void givens_init_kernel(double* gst, int R, double beta) {
    gst[size_t(R) * (R + 2) + 2 * size_t(R)] = beta;  // g_0
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

double dnorm(Scratch& s, cudaStream_t st, const double* x, int64_t len) {
    dev_dot_async(st, x, x, s.out.p, s.partials.p, s.ticket.p, len);
    double h = 0;
    CK(cudaMemcpyAsync(&h, s.out.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return std::sqrt(h);
}

// Krylov basis storage. Normally every basis vector is a device buffer. When the
// working set does not fit in HBM (BASELINE config 5: one KKT vector is 17.2 GB,
// SURVEY §7 hard part 3) the basis vectors beyond the device budget live in
// pinned host memory and are streamed through two device staging chunks; the
// newest basis vector is always kept on the device as well (it feeds the next
// operator apply and the last MGS step), and the best iterate is kept on the
// host. Arithmetic is unchanged except for the reduction order of the chunked
// dot products (per-chunk partials summed in chunk order).
struct Basis {
    int64_t len = 0;
    cudaStream_t st = nullptr;
    std::vector<DevBuf<double>> dev;  // device slots (index < ndev)
    std::vector<double*> host;        // pinned slots (index >= ndev)
    int ndev = 0;
    DevBuf<double> vlast;             // device copy of the newest host-resident vector
    int vlast_index = -1;
    // a free full-length device buffer during MGS + x_cand (host mode: the x_cand buffer):
    // holds the last host vector the MGS sweep streamed in, so the next step and x_cand
    // do not stream it again
    double* cache = nullptr;
    int cache_index = -1;
    DevBuf<double> stage[2], parts;
    int64_t chunk = 0;
    int nchunks = 0;
    // device-to-host copies (new basis vectors, the best iterate) run on their own
    // stream, overlapping the next iteration; events order every later use
    cudaStream_t cs = nullptr;
    std::vector<cudaEvent_t> ev_slot;  // copy into host[i] done
    cudaEvent_t ev_ready = nullptr, ev_vlast = nullptr;

    void init_copies() {
        CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        ev_slot.assign(host.size(), nullptr);
        for (auto& e : ev_slot) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ev_ready, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ev_vlast, cudaEventDisableTiming));
        CK(cudaEventRecord(ev_vlast, cs));
        for (auto& e : ev_slot) CK(cudaEventRecord(e, cs));
    }
    std::future<void> prealloc;  // host slots mapped in the background (host mode)
    ~Basis() {
        if (prealloc.valid()) prealloc.wait();
        if (cs) cudaStreamSynchronize(cs);
        for (auto& e : ev_slot)
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : {ev_ready, ev_vlast})
            if (e) cudaEventDestroy(e);
        if (cs) cudaStreamDestroy(cs);
        for (double* h : host)
            if (h) pinned_free(h);
    }
    bool on_host(int i) const { return i >= ndev; }
    void ensure_host(int i) {
        if (prealloc.valid()) prealloc.get();  // rethrows an allocation failure
        if (!host[i]) host[i] = static_cast<double*>(pinned_alloc(size_t(len) * sizeof(double)));
    }
    // device pointer of v_i if it is device-resident (or the cached newest vector), else null
    const double* dptr(int i) const {
        if (!on_host(i)) return dev[i].p;
        if (i == vlast_index) return vlast.p;
        return cache && i == cache_index ? cache : nullptr;
    }
    const double* stage_chunk(int slot, int i, int64_t off, int64_t cl) {
        if (const double* d = dptr(i)) return d + off;
        if (cs && off == 0) CK(cudaStreamWaitEvent(st, ev_slot[i], 0));  // host[i] fully written
        CK(cudaMemcpyAsync(stage[slot].p, host[i] + off, size_t(cl) * sizeof(double), cudaMemcpyHostToDevice, st));
        return stage[slot].p;
    }
};

// w -= h_{i-1} v_{i-1}; h_i = <v_i, w>  (vi < 0: <w, w>)
void mgs_step_any(Scratch& sc, Basis& B, double* w, int iprev, const double* hprev, int inext, double* hout) {
    const bool dev_prev = iprev < 0 || B.dptr(iprev), dev_next = inext < 0 || B.dptr(inext);
    // host mode (nchunks > 1) always reduces chunk by chunk, so h does not depend on which
    // basis vectors happen to be device-resident
    if (dev_prev && dev_next && B.nchunks <= 1) {
        dev_mgs_step(B.st, w, iprev >= 0 ? B.dptr(iprev) : nullptr, hprev, inext >= 0 ? B.dptr(inext) : nullptr,
                     hout, sc.partials.p, sc.ticket.p, B.len);
        return;
    }
    const int rb = reduce_blocks();
    const bool keep = B.cache && !dev_next;  // v_inext streams in: keep it for the next step
    for (int c = 0; c < B.nchunks; ++c) {
        const int64_t off = c * B.chunk, cl = std::min(B.chunk, B.len - off);
        const double* pv = iprev >= 0 ? B.stage_chunk(0, iprev, off, cl) : nullptr;
        const double* nv = inext >= 0 ? B.stage_chunk(1, inext, off, cl) : nullptr;
        dev_mgs_step_parts(B.st, w + off, pv, hprev, nv, B.parts.p + int64_t(c) * rb, cl);
        // chunk c of the cached v_iprev has been consumed: replace it by v_inext's
        if (keep)
            CK(cudaMemcpyAsync(B.cache + off, nv, size_t(cl) * sizeof(double), cudaMemcpyDeviceToDevice, B.st));
    }
    if (keep) B.cache_index = inext;
    dev_sum_ordered(B.st, B.parts.p, B.nchunks * rb, hout);
}

// out = x + sum_i y_i v_i, one basis vector at a time in index order (the fused
// kernel's rounding order)
void multi_axpy_any(Basis& B, double* out, const double* x, const std::vector<double>& y, const double* ydev,
                    int m) {
    bool all_dev = true;
    int staged = 0;
    for (int i = 0; i < m; ++i) {
        all_dev = all_dev && B.dptr(i);
        staged += B.dptr(i) ? 0 : 1;
    }
    if (all_dev && !(B.cache && out == B.cache)) {
        std::vector<const double*> vp(m);
        for (int i = 0; i < m; ++i) vp[i] = B.dptr(i);
        dev_multi_axpy(B.st, out, x, vp.data(), ydev, m, B.len);
        B.cache_index = -1;
        return;
    }
    if (staged <= 2) {
        // chunk-major: every element still sums x + y_0 v_0 + y_1 v_1 + ... in index order;
        // chunk c of a cached vector is read before out's chunk c (possibly the cache
        // buffer itself) is written
        std::vector<const double*> vp(m);
        for (int c = 0; c < B.nchunks; ++c) {
            const int64_t off = c * B.chunk, cl = std::min(B.chunk, B.len - off);
            int s = 0;
            for (int i = 0; i < m; ++i) vp[i] = B.dptr(i) ? B.dptr(i) + off : B.stage_chunk(s++, i, off, cl);
            dev_multi_axpy(B.st, out + off, x + off, vp.data(), ydev, m, cl);
        }
        B.cache_index = -1;
        return;
    }
    B.cache_index = -1;  // out may be the cache buffer: stream every host vector
    CK(cudaMemcpyAsync(out, x, size_t(B.len) * sizeof(double), cudaMemcpyDeviceToDevice, B.st));
    for (int i = 0; i < m; ++i) {
        if (const double* d = B.dptr(i)) {
            dev_axpy(B.st, y[i], d, out, B.len);
            continue;
        }
        for (int c = 0; c < B.nchunks; ++c) {
            const int64_t off = c * B.chunk, cl = std::min(B.chunk, B.len - off);
            dev_axpy(B.st, y[i], B.stage_chunk(c & 1, i, off, cl), out + off, cl);
        }
    }
}

// x (device, len) receives the solution.
Log gmres_core(GmresOps& ops, const double* b, double* x, int restart, double tol, int maxit, GmresWork& WS) {
    if (restart < 1) throw FwiError(FWI_ERR_INVALID_ARGUMENT, "gmres: restart must be >= 1");
    const auto t0 = std::chrono::steady_clock::now();
    double observer_time = 0.0;
    auto elapsed = [&] { return seconds_since(t0) - observer_time; };
    const int64_t len = ops.len;
    const size_t bytes = size_t(len) * sizeof(double);
    cudaStream_t st = ops.st;
    Scratch& sc = WS.sc;

    CK(cudaMemsetAsync(x, 0, bytes, st));
    Log log;
    const double bnorm = dnorm(sc, st, b, len);
    if (bnorm == 0.0) {
        log.entries.push_back({0, 0.0, {}, {}, elapsed()});
        log.converged = true;
        return log;
    }
    const int nbasis = std::min(restart, std::max(maxit, 1)) + 1;
    // ---- storage plan: tmp, w, xc (+ best, + basis) on the device if they fit
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    const size_t margin = size_t(2) << 30;
    const bool force_host = std::getenv("FWI_GMRES_HOST_BASIS") != nullptr;
    const bool host_mode = force_host || (size_t(4 + nbasis + 1) * bytes + margin > free_b);
    Basis B;
    B.len = len;
    B.st = st;
    B.dev.resize(nbasis);
    B.host.assign(nbasis, nullptr);
    double* best_host = nullptr;
    DevBuf<double> tmp, w, xc, best, xc2, axb;  // pipelined loop: second x_cand, A x_cand (second stream)
    // buffers come from (and go back to) the context's workspace unless the basis spills to the host
    struct Giveback {
        GmresWork& ws;
        bool keep;
        std::vector<DevBuf<double>*> bufs;
        ~Giveback() {
            if (keep)
                for (auto* b : bufs) ws.give(std::move(*b));
        }
    } gb{WS, !host_mode, {}};
    auto grab = [&](DevBuf<double>& d) {
        d = host_mode ? DevBuf<double>(size_t(len)) : WS.take(len);
        // KKT vectors carry a zero pad after the ds block that the flat dot products read
        CK(cudaMemsetAsync(d.p, 0, bytes, st));
        gb.bufs.push_back(&d);
    };
    // host mode keeps three vector buffers (w, xc and the newest basis vector's device
    // copy) and rotates their roles; the device mode also has tmp
    if (!host_mode) grab(tmp);
    grab(w);
    grab(xc);
    if (!host_mode) {
        grab(best);
        B.ndev = nbasis;
        // all slots up front: put_basis() then only rotates buffers (no allocation inside
        // the iteration, which would serialise the device)
        for (int i = 0; i < nbasis; ++i) grab(B.dev[i]);
    } else {
        B.chunk = std::min<int64_t>(len, int64_t(32) << 20);
        B.chunk -= B.chunk % 2;
        B.nchunks = int((len + B.chunk - 1) / B.chunk);
        B.stage[0].alloc(B.chunk);
        B.stage[1].alloc(B.chunk);
        B.parts.alloc(size_t(B.nchunks) * reduce_blocks());
        B.vlast.alloc(len);
        CK(cudaMemGetInfo(&free_b, &total_b));
        const int fit = free_b > margin ? int((free_b - margin) / bytes) : 0;
        B.ndev = force_host ? std::min(1, std::min(fit, nbasis)) : std::min(fit, nbasis);
        for (int i = 0; i < B.ndev; ++i) B.dev[i].alloc(len);
        B.init_copies();
        // mapping 17 GB of page-locked memory takes ~0.65 s: do it while the device works
        B.prealloc = std::async(std::launch::async, [&B, nbasis, bytes] {
            for (int i = B.ndev; i < nbasis; ++i) B.host[i] = static_cast<double*>(pinned_alloc(bytes));
        });
    }
    // FWI_GMRES_TRACE: per-iteration phase times (events on the solver stream) to stderr
    struct Trace {
        bool on = std::getenv("FWI_GMRES_TRACE") != nullptr;
        cudaEvent_t ev[8] = {};
        int n = 0;
        Trace() {
            if (on)
                for (auto& e : ev) CK(cudaEventCreate(&e));
        }
        ~Trace() {
            for (auto& e : ev)
                if (e) cudaEventDestroy(e);
        }
        void mark(cudaStream_t s) {
            if (on && n < 8) CK(cudaEventRecord(ev[n++], s));
        }
        void report(int iter, int j) {
            if (!on) return;
            CK(cudaEventSynchronize(ev[n - 1]));
            std::fprintf(stderr, "gmres-trace it %d j %d ms:", iter, j);
            for (int i = 1; i < n; ++i) {
                float ms = 0;
                CK(cudaEventElapsedTime(&ms, ev[i - 1], ev[i]));
                std::fprintf(stderr, " %.1f", ms);
            }
            std::fprintf(stderr, "\n");
            n = 0;
        }
    } trace;
    if (trace.on)
        std::fprintf(stderr, "gmres-trace host_mode %d ndev %d nbasis %d free %.1f GB vec %.1f GB\n", int(host_mode),
                     B.ndev, nbasis, double(free_b) / 1e9, double(bytes) / 1e9);
    // The best iterate (returned on stagnation). Device mode: a device copy. Host mode:
    // kept recoverable without a 17 GB copy per improvement. best_kind 1: the cycle-start
    // x (the x buffer itself); 2: iterate best_j of the current cycle, x + V y_best,
    // recomputed from the basis when needed (same arithmetic, so bit-identical); 3: a
    // page-locked host copy, made only when x moves on while the best lies elsewhere.
    int best_kind = 1, best_j = -1, last_j = -1;
    std::vector<double> best_y;
    struct HostFree {
        double*& p;
        ~HostFree() {
            if (p) pinned_free(p);
        }
    } best_guard{best_host};
    auto save_best = [&](const double* src) {
        CK(cudaMemcpyAsync(best.p, src, bytes, cudaMemcpyDeviceToDevice, st));
    };
    auto load_best = [&](double* dst) {
        CK(cudaMemcpyAsync(dst, best.p, bytes, cudaMemcpyDeviceToDevice, st));
    };
    auto recompute_best = [&](double* dst) {
        B.cache_index = -1;
        CK(cudaMemcpyAsync(WS.ydev.p, best_y.data(), best_y.size() * sizeof(double), cudaMemcpyHostToDevice, st));
        multi_axpy_any(B, dst, x, best_y, WS.ydev.p, best_j + 1);
    };
    auto materialise = [&](const double* src) {
        if (!best_host) best_host = static_cast<double*>(pinned_alloc(bytes));
        CK(cudaMemcpyAsync(best_host, src, bytes, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        best_kind = 3;
    };
    // store the normalised vector in `src` (a device buffer we own) as basis vector i
    auto put_basis = [&](int i, DevBuf<double>& src) {
        if (!B.on_host(i)) {
            std::swap(B.dev[i], src);
        } else {
            B.ensure_host(i);
            CK(cudaEventRecord(B.ev_ready, st));
            CK(cudaStreamWaitEvent(B.cs, B.ev_ready, 0));
            CK(cudaMemcpyAsync(B.host[i], src.p, bytes, cudaMemcpyDeviceToHost, B.cs));
            CK(cudaEventRecord(B.ev_slot[i], B.cs));
            // src takes the previous newest vector's buffer, whose own host copy must be
            // finished before it is overwritten
            CK(cudaStreamWaitEvent(st, B.ev_vlast, 0));
            CK(cudaEventRecord(B.ev_vlast, B.cs));
            std::swap(B.vlast, src);  // device copy of the newest vector; src reuses the old one
            B.vlast_index = i;
        }
    };

    ops.precond(b, w.p);
    const double pbnorm = dnorm(sc, st, w.p, len);
    if (pbnorm == 0.0)
        throw FwiError(FWI_ERR_INVALID_ARGUMENT, "gmres: preconditioner annihilates the right-hand side");
    log.entries.push_back({0, 1.0, {}, 1.0, elapsed()});

    if (!host_mode) CK(cudaMemsetAsync(best.p, 0, bytes, st));
    double best_res = 1.0, true_res = 1.0;
    int iter = 0;
    bool stop_requested = false;
    WS.small(restart);
    DevBuf<double>& hdev = WS.hdev;
    DevBuf<double>& ydev = WS.ydev;
    std::vector<double> hh(restart + 2);

    // Pipelined loop (device-resident basis, no observer): the Givens step runs on the device
    // (givens_kernel, bit-identical to the host code below), the basis normalisation reads ||w||
    // from the device, and iteration j + 1 is enqueued before the host waits for iteration j's
    // residual — the device never idles on the host's convergence test. A speculative iteration
    // past convergence writes only buffers the result does not use (x_cand alternates between two
    // buffers) and is dropped. With a second-stream operator (ops.apply_alt) iteration j's
    // residual branch — Givens step, x_cand = x + V y, A x_cand and its norm — runs on its own
    // stream beside iteration j + 1's operator and preconditioner (h in two slots by iteration
    // parity). FWI_GMRES_SYNC=1 selects the synchronous loop below, FWI_GMRES_ONESTREAM=1 keeps
    // the residual branch on the main stream.
    if (!host_mode && !ops.observer && restart + 1 <= 63 && !std::getenv("FWI_GMRES_SYNC")) {
        WS.pipeline(restart);
        const bool two = bool(ops.apply_alt) && !std::getenv("FWI_GMRES_ONESTREAM");
        if (two) WS.second_stream();
        const cudaStream_t sb = two ? WS.s2 : st;  // the residual branch's stream
        Scratch& scb = two ? *WS.sc2 : sc;
        // on every exit (an error included) the residual branch is drained before its buffers go
        // back to the context's pool
        struct Drain {
            cudaStream_t s;
            ~Drain() {
                if (s) cudaStreamSynchronize(s);
            }
        } drain{two ? sb : nullptr};
        grab(xc2);
        if (two) grab(axb);
        DevBuf<double>* xcb[2] = {&xc, &xc2};
        const int hp = restart + 2;  // h slot pitch
        auto hslot = [&](int j) { return hdev.p + (two ? (j & 1) * hp : 0); };
        auto copy_best = [&](const double* src) {
            CK(cudaMemcpyAsync(best.p, src, bytes, cudaMemcpyDeviceToDevice, sb));
        };
        double res_prev = 1.0, rate = 1.0;  // last true residual and reduction factor (prediction)
        while (iter < maxit && !log.converged) {
            // r0 = M^{-1}(b - A x)
            ops.apply(x, w.p);
            CK(cudaMemcpyAsync(xc.p, b, bytes, cudaMemcpyDeviceToDevice, st));
            dev_axpy(st, -1.0, w.p, xc.p, len);
            ops.precond(xc.p, w.p);
            const double beta = dnorm(sc, st, w.p, len);
            const double cycle_start_res = true_res;
            if (beta == 0.0) break;
            dev_scal(st, 1.0 / beta, w.p, len);
            put_basis(0, w);
            givens_init_kernel<<<1, 1, 0, st>>>(WS.gst.p, restart, beta);
            CK_LAUNCH();
            auto issue = [&](int j) {
                double* stj = WS.stat.p + 4 * (j & 1);
                double* hj = hslot(j);
                ops.apply(B.dptr(j), w.p);
                ops.precond(w.p, tmp.p);
                std::swap(w, tmp);
                std::vector<const double*> vp(j + 1);
                for (int i = 0; i <= j; ++i) vp[i] = B.dptr(i);
                // h slot j & 1 is free once iteration j - 2's residual branch has read it
                if (two && j >= 2) CK(cudaStreamWaitEvent(st, WS.ev_stat[j & 1], 0));
                if (!dev_mgs_all(st, w.p, vp.data(), j + 1, hj, sc.partials.p, sc.ticket.p, sc.flag.p, sc.epoch,
                                 len)) {
                    for (int i = 0; i <= j; ++i) mgs_step_any(sc, B, w.p, i - 1, hj + (i - 1), i, hj + i);
                    mgs_step_any(sc, B, w.p, j, hj + j, -1, hj + j + 1);
                }
                if (two) {
                    CK(cudaEventRecord(WS.ev_mgs[j & 1], st));
                    CK(cudaStreamWaitEvent(sb, WS.ev_mgs[j & 1], 0));
                }
                const size_t gsm = (size_t(j + 1) * (restart + 2) + 4 * size_t(j) + 8) * sizeof(double);
                launch_pdl<kPdlVec>(givens_kernel, dim3(1), dim3(32), gsm, sb, hj, j, restart, WS.gst.p, ydev.p, stj);
                CK_LAUNCH();
                dev_multi_axpy(sb, xcb[j & 1]->p, x, vp.data(), ydev.p, j + 1, len);
                double* ax = two ? axb.p : tmp.p;
                if (two)
                    ops.apply_alt(xcb[j & 1]->p, ax, sb);
                else
                    ops.apply(xcb[j & 1]->p, ax);
                dev_sub_norm2(sb, b, ax, stj, scb.partials.p, scb.ticket.p, len);
                CK(cudaMemcpyAsync(WS.hstat + 4 * (j & 1), stj, 3 * sizeof(double), cudaMemcpyDeviceToHost, sb));
                CK(cudaEventRecord(WS.ev_stat[j & 1], sb));
            };
            bool happy = false;
            int jl = 0;
            issue(0);
            for (int j = 0;; ++j) {
                ++iter;
                const bool more = j + 1 < restart && iter < maxit;
                // iteration j + 1 is enqueued before j's residual is known unless j is predicted
                // to converge (the last residual times the last reduction factor within twice the
                // tolerance): a speculative iteration after convergence would cost a whole
                // iteration, the wait costs one host round trip
                const bool ahead = more && !(res_prev * rate <= 2.0 * tol);
                if (ahead) {  // v_{j+1} = w / ||w||, then iteration j + 1
                    dev_scal_rsqrt(st, hslot(j) + j + 1, w.p, len);
                    put_basis(j + 1, w);
                    issue(j + 1);
                }
                CK(cudaEventSynchronize(WS.ev_stat[j & 1]));
                const double* hs = WS.hstat + 4 * (j & 1);
                const double r2 = hs[0], wn = hs[1], prec_res = hs[2] / pbnorm;
                true_res = std::sqrt(r2) / bnorm;
                log.entries.push_back({iter, true_res, {}, prec_res, elapsed()});
                if (true_res < best_res) {
                    best_res = true_res;
                    copy_best(xcb[j & 1]->p);
                }
                jl = j;
                if (res_prev > 0.0) rate = std::min(1.0, true_res / res_prev);
                res_prev = true_res;
                if (true_res <= tol) log.converged = true;
                if (wn == 0.0) happy = true;
                if (log.converged || happy || !more) break;
                if (!ahead) {  // predicted convergence did not happen: continue synchronously
                    dev_scal_rsqrt(st, hslot(j) + j + 1, w.p, len);
                    put_basis(j + 1, w);
                    issue(j + 1);
                }
            }
            const bool stag = !log.converged && (true_res >= cycle_start_res * (1.0 - 1e-12) || happy);
            CK(cudaMemcpyAsync(x, xcb[jl & 1]->p, bytes, cudaMemcpyDeviceToDevice, sb));
            if (stag) {
                log.stagnated = true;
                CK(cudaMemcpyAsync(x, best.p, bytes, cudaMemcpyDeviceToDevice, sb));
            }
            if (two) {  // the next cycle (or the caller) reads x on the main stream
                CK(cudaEventRecord(WS.ev_x, sb));
                CK(cudaStreamWaitEvent(st, WS.ev_x, 0));
            }
            if (stag) break;
        }
        CK(cudaStreamSynchronize(st));
        if (two) CK(cudaStreamSynchronize(sb));
        return log;
    }

    while (iter < maxit && !log.converged && !stop_requested) {
        // r0 = M^{-1}(b - A x)
        ops.apply(x, w.p);
        CK(cudaMemcpyAsync(xc.p, b, bytes, cudaMemcpyDeviceToDevice, st));
        dev_axpy(st, -1.0, w.p, xc.p, len);
        ops.precond(xc.p, w.p);
        const double beta = dnorm(sc, st, w.p, len);
        const double cycle_start_res = true_res;
        if (beta == 0.0) break;
        dev_scal(st, 1.0 / beta, w.p, len);
        put_basis(0, w);

        std::vector<std::vector<double>> hcols;
        std::vector<double> gs_c, gs_s, g(1, beta);
        CK(cudaMemcpyAsync(xc.p, x, bytes, cudaMemcpyDeviceToDevice, st));
        bool happy = false;

        for (int j = 0; j < restart && iter < maxit; ++j) {
            ++iter;
            trace.mark(st);
            ops.apply(B.dptr(j), w.p);
            trace.mark(st);
            // host mode: x_cand of the previous iteration is dead (the best iterate is
            // recoverable from the basis)
            DevBuf<double>& spare = host_mode ? xc : tmp;
            ops.precond(w.p, spare.p);
            std::swap(w, spare);
            if (host_mode) {  // xc is free until x_cand: it caches streamed basis vectors
                B.cache = xc.p;
                B.cache_index = -1;
            }
            // the host slot of the next basis vector is mapped while the device works
            if (j + 1 < nbasis && B.on_host(j + 1)) B.ensure_host(j + 1);
            trace.mark(st);
            // MGS: h_i = <v_i, w>; w -= h_i v_i  (fused pairwise)
            bool fused = false;
            if (!host_mode && !std::getenv("FWI_GMRES_MGS_STEPS")) {
                std::vector<const double*> vp(j + 1);
                for (int i = 0; i <= j; ++i) vp[i] = B.dptr(i);
                fused = dev_mgs_all(st, w.p, vp.data(), j + 1, hdev.p, sc.partials.p, sc.ticket.p, sc.flag.p,
                                    sc.epoch, len);
            }
            if (!fused) {
                for (int i = 0; i <= j; ++i)
                    mgs_step_any(sc, B, w.p, i - 1, hdev.p + (i - 1), i, hdev.p + i);
                mgs_step_any(sc, B, w.p, j, hdev.p + j, -1, hdev.p + j + 1);
            }
            trace.mark(st);
            CK(cudaMemcpyAsync(hh.data(), hdev.p, (j + 2) * sizeof(double), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            std::vector<double> h(hh.begin(), hh.begin() + j + 2);
            const double wn = std::sqrt(h[j + 1]);
            h[j + 1] = wn;

            for (int i = 0; i < j; ++i) {
                const double t = gs_c[i] * h[i] + gs_s[i] * h[i + 1];
                h[i + 1] = -gs_s[i] * h[i] + gs_c[i] * h[i + 1];
                h[i] = t;
            }
            double c, s, rr;
            {
                const double an = std::abs(h[j]), bn = std::abs(h[j + 1]);
                const double t = std::sqrt(an * an + bn * bn);
                if (bn == 0.0) {
                    c = 1.0;
                    s = 0.0;
                    rr = h[j];
                } else if (an == 0.0) {
                    c = 0.0;
                    s = h[j + 1] / bn;
                    rr = bn;
                } else {
                    c = an / t;
                    s = (h[j] / an) * h[j + 1] / t;
                    rr = (h[j] / an) * t;
                }
            }
            gs_c.push_back(c);
            gs_s.push_back(s);
            h[j] = rr;
            h[j + 1] = 0.0;
            g.push_back(-s * g[j]);
            g[j] = c * g[j];
            hcols.push_back(h);
            const double prec_res = std::abs(g[j + 1]) / pbnorm;

            std::vector<double> y(j + 1);
            for (int i = j; i >= 0; --i) {
                double acc = g[i];
                for (int k2 = i + 1; k2 <= j; ++k2) acc -= hcols[k2][i] * y[k2];
                y[i] = acc / hcols[i][i];
            }
            CK(cudaMemcpyAsync(ydev.p, y.data(), (j + 1) * sizeof(double), cudaMemcpyHostToDevice, st));
            trace.mark(st);
            trace.mark(st);
            multi_axpy_any(B, xc.p, x, y, ydev.p, j + 1);
            last_j = j;
            trace.mark(st);

            // host mode: v_j's device copy is dead (its host copy is complete) and takes A x_cand
            DevBuf<double>& ax = host_mode ? B.vlast : tmp;
            if (host_mode) {
                CK(cudaStreamWaitEvent(st, B.ev_vlast, 0));
                B.vlast_index = -1;
            }
            ops.apply(xc.p, ax.p);
            dev_sub_norm2(st, b, ax.p, sc.out.p, sc.partials.p, sc.ticket.p, len);
            trace.mark(st);
            double r2 = 0;
            CK(cudaMemcpyAsync(&r2, sc.out.p, sizeof(double), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            trace.report(iter, j);
            true_res = std::sqrt(r2) / bnorm;
            log.entries.push_back({iter, true_res, {}, prec_res, elapsed()});
            if (true_res < best_res) {
                best_res = true_res;
                if (host_mode) {
                    best_kind = 2;
                    best_j = j;
                    best_y = y;
                } else {
                    save_best(xc.p);
                }
            }
            if (ops.observer) {
                const auto to0 = std::chrono::steady_clock::now();
                stop_requested = ops.observer(iter, xc.p);
                observer_time += seconds_since(to0);
            }
            if (true_res <= tol) log.converged = true;
            if (wn == 0.0) happy = true;
            if (log.converged || stop_requested || happy) break;
            if (j + 1 >= restart) break;  // the next basis vector would be discarded by the restart
            // v_{j+1} = w / ||w||
            dev_scal(st, 1.0 / wn, w.p, len);
            put_basis(j + 1, w);
        }
        // a full cycle without reducing the true residual (or a happy breakdown short of the
        // tolerance) returns the best iterate
        const bool fin = log.converged || stop_requested;
        const bool stag = !fin && (true_res >= cycle_start_res * (1.0 - 1e-12) || happy);
        if (!host_mode) {
            CK(cudaMemcpyAsync(x, xc.p, bytes, cudaMemcpyDeviceToDevice, st));
            if (stag) {
                log.stagnated = true;
                load_best(x);
                break;
            }
            continue;
        }
        if (stag) {
            if (best_kind == 2) {
                recompute_best(xc.p);
                CK(cudaMemcpyAsync(x, xc.p, bytes, cudaMemcpyDeviceToDevice, st));
            } else if (best_kind == 3) {
                CK(cudaMemcpyAsync(x, best_host, bytes, cudaMemcpyHostToDevice, st));
            }  // best_kind 1: x holds it
            log.stagnated = true;
            break;
        }
        if (!fin) {  // x moves on to x_cand: keep the best iterate recoverable
            if (best_kind == 2 && best_j != last_j) {
                recompute_best(w.p);
                materialise(w.p);
            } else if (best_kind == 2) {
                best_kind = 1;
            } else if (best_kind == 1) {
                materialise(x);
            }
        }
        CK(cudaMemcpyAsync(x, xc.p, bytes, cudaMemcpyDeviceToDevice, st));
    }
    CK(cudaStreamSynchronize(st));
    if (B.cs) CK(cudaStreamSynchronize(B.cs));
    return log;
}

void fill_log(const Log& lg, fwi_convergence_log* out) {
    if (!out) return;
    out->count = 0;
    for (const auto& e : lg.entries) {
        if (out->count >= out->capacity) break;
        fwi_log_entry& d = out->entries[out->count++];
        d.iteration = e.iteration;
        d.residual_norm = e.residual_norm;
        d.has_precond_residual = e.precond_residual.has_value();
        d.precond_residual = e.precond_residual.value_or(0.0);
        d.has_normal_residual = e.normal_residual.has_value();
        d.normal_residual = e.normal_residual.value_or(0.0);
        d.wall_time = e.wall_time;
        d.pad_ = 0;
    }
    out->converged = lg.converged;
    out->stagnated = lg.stagnated;
}

}  // namespace

void fsgn_gmres_step(Ctx& c, const fwi_fsgn_options& o, double* ds_host, fwi_convergence_log* log) {
    require(o.mode == FWI_PRECOND_EXACT || o.mode == FWI_PRECOND_ILU, "fsgn_gmres_step: unknown mode");
    if (o.mode == FWI_PRECOND_ILU) require(c.ilu != nullptr, "precond_apply: state has no ILU factorization");
    if (o.mode == FWI_PRECOND_EXACT)
        require(c.exact != nullptr, "precond_apply: state has no exact factorization");
    const int64_t len = c.vec_len;
    const int64_t n = c.n;
    cudaStream_t st = c.stream;
    // b = kkt_rhs
    if (!c.gmres_work) c.gmres_work = new GmresWork();
    GmresWork& ws = *c.gmres_work;
    const bool small = size_t(len) * sizeof(double) * size_t(o.restart + 8) < (size_t(8) << 30);
    Vec bv;
    bv.ctx = &c;
    bv.d = small ? ws.take(len) : DevBuf<double>(size_t(len));
    CK(cudaMemsetAsync(bv.d.p, 0, bv.d.bytes(), st));
    kkt_rhs(c, bv);
    DevBuf<double> xv = small ? ws.take(len) : DevBuf<double>(size_t(len));
    CK(cudaMemsetAsync(xv.p, 0, xv.bytes(), st));
    struct Back {
        GmresWork& ws;
        bool on;
        DevBuf<double>& a;
        DevBuf<double>& b;
        ~Back() {
            if (on) {
                ws.give(std::move(a));
                ws.give(std::move(b));
            }
        }
    } back{ws, small, bv.d, xv};
    // g = gradient(state): K adjoint solves (src/kkt.cpp:139-141). It only
    // normalises the E_cg metric; without the exact factorisation the metric
    // column is left unset.
    DevBuf<double> g(c.ds_stride), hds(c.ds_stride);
    CK(cudaMemsetAsync(g.p, 0, g.bytes(), st));
    CK(cudaMemsetAsync(hds.p, 0, hds.bytes(), st));
    double gnorm = 0.0;
    if (!c.gmres_work) c.gmres_work = new GmresWork();
    if (c.exact) {
        reduced_gradient(c, g.p);
        gnorm = dnorm(c.gmres_work->sc, st, g.p, c.ds_stride);
    }
    std::vector<std::pair<int, double>> metric;
    GmresOps ops;
    ops.len = len;
    ops.st = st;
    ops.apply = [&c](const double* in, double* out) { kkt_apply_raw(c, in, out); };
    ops.apply_alt = [&c](const double* in, double* out, cudaStream_t s) { kkt_apply_raw_on(c, in, out, s); };
    const int mode = o.mode;
    ops.precond = [&c, mode](const double* in, double* out) { precond_apply_raw(c, mode, in, out); };
    if (o.ecg_stride > 0) {
        require(c.exact != nullptr, "fsgn_gmres_step: the normal-equation metric needs the exact factorization");
        ops.observer = [&](int iter, const double* xi) {
            if (iter % o.ecg_stride != 0) return false;
            // normal_residual (src/reduced_space.cpp:154-161)
            reduced_hessian(c, c.ds_of(const_cast<double*>(xi)), hds.p);
            dev_axpy(st, -1.0, g.p, hds.p, c.ds_stride);
            Scratch sc;
            const double rn = dnorm(sc, st, hds.p, c.ds_stride);
            double e;
            if (gnorm == 0.0)
                e = rn == 0.0 ? 0.0 : INFINITY;
            else
                e = rn / gnorm;
            metric.emplace_back(iter, e);
            return o.ecg_stop_tol > 0.0 && e <= o.ecg_stop_tol;
        };
    }
    if (!c.gmres_work) c.gmres_work = new GmresWork();
    Log lg = gmres_core(ops, bv.d.p, xv.p, o.restart, o.tol, o.maxit, *c.gmres_work);
    if (!lg.entries.empty() && c.exact) lg.entries.front().normal_residual = gnorm > 0.0 ? 1.0 : 0.0;
    for (const auto& [it, e] : metric)
        for (auto& en : lg.entries)
            if (en.iteration == it) {
                en.normal_residual = e;
                break;
            }
    if (ds_host)
        CK(cudaMemcpyAsync(ds_host, c.ds_of(xv.p), n * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    fill_log(lg, log);
}

// rsgn_cg_step (src/reduced_space.cpp:163-170) over cg<RealVector>
// (include/fwi/krylov.hpp:79-120): CG on H ds = g, H = Re(J^H W^T W J) + eps I.
void rsgn_cg_step(Ctx& c, double tol, int maxit, double* ds_host, fwi_convergence_log* log) {
    require(c.exact != nullptr, "rsgn_cg_step: state has no exact factorization");
    const auto t0 = std::chrono::steady_clock::now();
    const int64_t len = c.ds_stride;
    cudaStream_t st = c.stream;
    Scratch sc;
    auto ddot = [&](const double* a, const double* b) {
        dev_dot_async(st, a, b, sc.out.p, sc.partials.p, sc.ticket.p, len);
        double h = 0;
        CK(cudaMemcpyAsync(&h, sc.out.p, sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        return h;
    };
    DevBuf<double> g(len), x(len), r(len), p(len), ap(len);
    for (auto* b : {&g, &x, &r, &p, &ap}) CK(cudaMemsetAsync(b->p, 0, b->bytes(), st));
    reduced_gradient(c, g.p);
    Log lg;
    const double bnorm = std::sqrt(ddot(g.p, g.p));
    if (bnorm == 0.0) {
        lg.entries.push_back({0, 0.0, {}, {}, seconds_since(t0)});
        lg.converged = true;
    } else {
        lg.entries.push_back({0, 1.0, {}, {}, seconds_since(t0)});
        CK(cudaMemcpyAsync(r.p, g.p, len * sizeof(double), cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(p.p, g.p, len * sizeof(double), cudaMemcpyDeviceToDevice, st));
        double rho = ddot(r.p, r.p);
        for (int it = 1; it <= maxit; ++it) {
            reduced_hessian(c, p.p, ap.p);
            const double pap = ddot(p.p, ap.p);
            if (!(pap > 0.0))
                throw FwiError(FWI_ERR_CG_BREAKDOWN, "cg: non-positive curvature, operator is not HPD");
            const double alpha = rho / pap;
            dev_axpy(st, alpha, p.p, x.p, len);
            dev_axpy(st, -alpha, ap.p, r.p, len);
            const double rn = std::sqrt(ddot(r.p, r.p)) / bnorm;
            lg.entries.push_back({it, rn, {}, {}, seconds_since(t0)});
            if (rn <= tol) {
                lg.converged = true;
                break;
            }
            const double rho_new = ddot(r.p, r.p);
            const double beta = rho_new / rho;
            rho = rho_new;
            dev_scal(st, beta, p.p, len);
            dev_axpy(st, 1.0, r.p, p.p, len);
        }
    }
    for (auto& e : lg.entries) e.normal_residual = e.residual_norm;  // src/reduced_space.cpp:166-168
    if (ds_host) CK(cudaMemcpyAsync(ds_host, x.p, c.n * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    fill_log(lg, log);
}

void gmres_generic(int64_t n, fwi_op_cb apply, fwi_op_cb precond, fwi_observer_cb observer, void* user,
                   const double* b, double* x, int restart, double tol, int maxit,
                   fwi_convergence_log* log) {
    require(n > 0 && n % 2 == 0, "gmres_generic: vector length must be positive and even");
    GmresOps ops;
    ops.len = n;
    ops.st = nullptr;  // legacy stream: callbacks may use any stream-ordered API
    ops.apply = [&](const double* in, double* out) {
        CK(cudaStreamSynchronize(nullptr));
        if (apply(user, in, out) != 0) throw FwiError(FWI_ERR_INVALID_ARGUMENT, "gmres: apply callback failed");
    };
    ops.precond = [&](const double* in, double* out) {
        CK(cudaStreamSynchronize(nullptr));
        if (precond(user, in, out) != 0)
            throw FwiError(FWI_ERR_INVALID_ARGUMENT, "gmres: precond callback failed");
    };
    if (observer)
        ops.observer = [&](int it, const double* xc) {
            CK(cudaStreamSynchronize(nullptr));
            return observer(user, it, xc) != 0;
        };
    GmresWork ws;
    Log lg = gmres_core(ops, b, x, restart, tol, maxit, ws);
    fill_log(lg, log);
}

}  // namespace fwi_b200
