// ctx.cuh — the device-resident GnState (fwi_dev_ctx) and KKT vectors.
//
// Reference counterpart: fwi::GnState (include/fwi/reduced_space.hpp:15-41)
// and fwi::KktVector (include/fwi/kkt.hpp:12-19).
//
// HBM layout (all fields stay resident; nothing is re-uploaded per call):
//   stencil   diag / east / south : 3 x n complex128  A(i,i), A(i,i+1), A(i,i+nx)
//             (A(i,i-1) = east[i-1] and A(i,i-nx) = south[i-nx] bitwise, the
//              assembled matrix being exactly complex-symmetric)
//   u         K x n complex128, source-major (u_k contiguous)  [+ complex64 copy]
//   receivers per-node table (node -> (k, w^2) sorted by k, then data index)
//   KKT vec   one flat buffer: [du: 2Kn doubles | ds: n (padded to ds_stride) | lambda: 2Kn]
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <vector>

#include "common.cuh"

namespace fwi_b200 {

struct ExactFactor;  // exact.cu
struct IluFactor;    // ilu.cu
struct GmresWork;    // gmres.cu
struct KktPlan;      // kkt_tma.cu
struct KktKmPlan;    // kkt_tma.cu

struct Ctx {
    // geometry / scalars
    int nx = 0, nz = 0, n = 0, K = 0, ndata = 0, n_pml = 0;
    double h = 0, freq_hz = 0, omega = 0, w2 = 0, eps = 0;
    double sigma_max = 0, power = 2;
    bool drop = false;
    int64_t ds_stride = 0;  // padded length of the ds block
    int64_t vec_len = 0;    // device doubles per KKT vector: 4Kn + ds_stride
    int precision_mask = 0;

    cudaStream_t stream = nullptr;

    // stencil (complex128)
    DevBuf<double2> diag, east, south;
    DevBuf<float2> diag32, east32, south32;
    DevBuf<double> s;
    // fields
    DevBuf<double2> u;
    DevBuf<float2> u32;
    DevBuf<double2> r, dpred;
    // survey
    std::vector<int> h_recv_offset, h_recv_node, h_src_node;
    std::vector<double> h_w, h_src_amp;
    DevBuf<int> recv_offset, recv_node;
    DevBuf<double> w;
    DevBuf<int> nrec_ptr, nrec_k;  // per-node receiver table
    DevBuf<double> nrec_w2;
    bool nrec_dup = false;  // some node has two entries of one source (co-located receivers)
    // factorisations
    ExactFactor* exact = nullptr;  // owned (exact_free)
    IluFactor* ilu = nullptr;      // owned (ilu_free)
    GmresWork* gmres_work = nullptr;  // owned (gmres_work_free): Krylov buffers reused across solves
    int64_t solve_count[2] = {0, 0};
    double t_ilu_factor = 0.0;  // host ILU(p) factorisation time of the current factors, s
    KktPlan* kplan[2] = {nullptr, nullptr};      // tile-TMA apply plans (c128, c64), built lazily
    KktPlan* kplan_alt[2] = {nullptr, nullptr};  // the same for applies on a second stream (GMRES)
    KktKmPlan* kmplan[2] = {nullptr, nullptr};   // source-major TMA apply plans (c128, c64), built lazily
    // 0: source-major TMA kernel (falling back to the tile-TMA kernel, then the plain kernel),
    // 1: plain kernel (FWI_KKT_KERNEL=plain), 2: tile-TMA kernel (FWI_KKT_KERNEL=tile)
    int kkt_variant = 0;
    const char* kkt_kernel[2] = {"", ""};  // K1 kernel of the last apply (c128, c64), fwi_dev_kkt_kernel
    // host copy of the stencil for the ILU factorisation (lazily)
    std::vector<double> h_s;

    // scratch
    DevBuf<double> red_partials;  // deterministic reductions
    DevBuf<unsigned int> red_ticket;
    DevBuf<double> red_out;       // scalar results
    DevBuf<double2> work_a, work_b, work_c;  // K*n complex scratch (precond)
    DevBuf<double> work_ds;
    // pipelined host-buffer apply (kkt_apply_host)
    static constexpr int kMaxChunks = 64;
    DevBuf<double> hx, hy, hpl;
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    cudaEvent_t ev_in[kMaxChunks] = {}, ev_out[kMaxChunks] = {};

    ~Ctx();
    double2* du_of(double* base) const { return reinterpret_cast<double2*>(base); }
    double* ds_of(double* base) const { return base + 2 * int64_t(K) * n; }
    double2* la_of(double* base) const {
        return reinterpret_cast<double2*>(base + 2 * int64_t(K) * n + ds_stride);
    }
    // K x n scratch, allocated on first use: kWorkA | kWorkB | kWorkC (+ ds scratch)
    static constexpr unsigned kWorkA = 1, kWorkB = 2, kWorkC = 4;
    void ensure_work(unsigned which = kWorkA | kWorkB | kWorkC);
};

struct Vec {
    Ctx* ctx = nullptr;
    int prec = FWI_C128;
    DevBuf<double> d;  // c128
    DevBuf<float> f;   // c64
    int64_t len() const { return ctx->vec_len; }
};

// ---- ctx.cu
Ctx* ctx_create(const fwi_state_desc& d);
void stencil_to_host(const Ctx& c, double* diag, double* east, double* south);

// ---- kkt.cu
void kkt_apply(Ctx& c, const Vec& xi, Vec& out);
void kkt_rhs(Ctx& c, Vec& out);
void kkt_apply_raw(Ctx& c, const double* xi, double* out);  // c128 flat device buffers
// the same on stream s, concurrently with applies on c.stream (its own tile-kernel plan)
void kkt_apply_raw_on(Ctx& c, const double* xi, double* out, cudaStream_t s);
bool kkt_apply_tma(Ctx& c, bool f32, const void* xi, void* out);
void kkt_apply_host(Ctx& c, const double* in, double* out);
void kkt_plan_free(KktPlan*);
void kkt_km_plan_free(KktKmPlan*);

// ---- vec.cu  (flat device arrays of len doubles; deterministic reductions)
double dev_dot(Ctx* c, cudaStream_t st, const double* x, const double* y, int64_t len);
void dev_axpy(cudaStream_t st, double a, const double* x, double* y, int64_t len);
void dev_scal(cudaStream_t st, double a, double* x, int64_t len);
void dev_scal_rsqrt(cudaStream_t st, const double* h2_dev, double* x, int64_t len);  // x /= sqrt(*h2)
// fused GMRES helpers
void dev_mgs_step(cudaStream_t st, double* w, const double* vprev, const double* hprev_dev,
                  const double* vnext, double* h_out_dev, double* partials, unsigned* ticket,
                  int64_t len);
// chunk version of dev_mgs_step: per-CTA partials (reduce_blocks() of them) to partials_out
void dev_mgs_step_parts(cudaStream_t st, double* w, const double* vprev, const double* hprev_dev,
                        const double* vnext, double* partials_out, int64_t len);
void dev_sum_ordered(cudaStream_t st, const double* partials, int count, double* out_dev);
// all m+1 fused MGS steps of one GMRES iteration in one launch (v: m device vectors,
// h_dev: m+1 outputs); false if it cannot run (caller falls back to dev_mgs_step)
bool dev_mgs_all(cudaStream_t st, double* w, const double* const* v, int m, double* h_dev, double* partials,
                 unsigned* ticket, unsigned* flag, unsigned& epoch, int64_t len);
void dev_multi_axpy(cudaStream_t st, double* out, const double* x, const double* const* v,
                    const double* y, int m, int64_t len);
void dev_sub_norm2(cudaStream_t st, const double* b, const double* ax, double* out_dev,
                   double* partials, unsigned* ticket, int64_t len);
void dev_dot_async(cudaStream_t st, const double* x, const double* y, double* out_dev,
                   double* partials, unsigned* ticket, int64_t len);
int reduce_blocks();

// ---- ilu.cu
void ilu_factor(Ctx& c, int level, double shift);
void ilu_solve_batch(Ctx& c, bool adjoint, const double2* b, double2* x, int nrhs);
void ilu_free(IluFactor*);
int64_t ilu_bytes(const IluFactor*);

// ---- exact.cu
void exact_factor(Ctx& c);
void exact_solve_batch(Ctx& c, bool adjoint, const double2* b, double2* x, int nrhs);
void exact_free(ExactFactor*);
void gmres_work_free(GmresWork*);
int64_t exact_bytes(const ExactFactor*);
double exact_probe_residual(const ExactFactor*);

// ---- bcr.cu (block cyclic reduction, used by exact.cu)
struct BcrFactor;
constexpr int kBcrMinLines = 256;  // lines from which cyclic reduction replaces the Schur sweeps
BcrFactor* bcr_factor(Ctx& c, bool col_lines, int nb, int L, const double2* coup, int* status);
void bcr_solve(Ctx& c, BcrFactor& f, const double2* coup, double2* W, int nrhs);
void bcr_free(BcrFactor*);
int64_t bcr_bytes(const BcrFactor*);

// ---- precond.cu
void precond_apply(Ctx& c, int mode, const Vec& v, Vec& out);
void precond_apply_raw(Ctx& c, int mode, const double* v, double* out);
void block_solve(Ctx& c, int mode, bool adjoint, const double2* b, double2* x, int nrhs);

// ---- gmres.cu
void fsgn_gmres_step(Ctx& c, const fwi_fsgn_options& o, double* ds_host, fwi_convergence_log* log);

}  // namespace fwi_b200
