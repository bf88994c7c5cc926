// ctx.cu — device GnState construction (make_gn_state, src/reduced_space.cpp:40-86):
// validation, 5-point PML stencil assembly on the device, survey tables,
// background fields (uploaded or computed by the device's exact block solver)
// and the data residual.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "ctx.cuh"

namespace fwi_b200 {

namespace {
constexpr double kPi = 3.141592653589793238462643383279502884;  // == std::numbers::pi

// fwi::stretch (src/grid.cpp:35-48), evaluated on the host with the same
// libm calls so the device stencil reproduces the reference coefficients.
void stretch_host(int n_axis, int n_pml, double sigma_max, double power, double pos, double omega,
                  double* out) {
    out[0] = 1.0;
    out[1] = 0.0;
    if (n_pml == 0) return;
    const double depth = std::max(n_pml - pos, pos - (n_axis - 1 - n_pml));
    if (depth <= 0.0) return;
    const double t = depth / n_pml;
    out[1] = sigma_max * std::pow(t, power) / omega;
}

// assemble_helmholtz (src/helmholtz.cpp:17-70) as coefficient planes.
// X/Z: stretch at integer nodes; XH/ZH: at i+0.5.
__global__ void assemble_kernel(int nx, int nz, double h2, double w2, const double* __restrict__ s,
                                const double2* __restrict__ X, const double2* __restrict__ XH,
                                const double2* __restrict__ Z, const double2* __restrict__ ZH,
                                double2* __restrict__ diag, double2* __restrict__ east,
                                double2* __restrict__ south) {
    const int ix = blockIdx.x * blockDim.x + threadIdx.x;
    const int iz = blockIdx.y * blockDim.y + threadIdx.y;
    if (ix >= nx || iz >= nz) return;
    const int64_t node = int64_t(iz) * nx + ix;
    if (on_boundary(ix, iz, nx, nz)) {
        diag[node] = make_double2(1.0, 0.0);
        east[node] = cz();
        south[node] = cz();
        return;
    }
    const double2 xi = X[ix], xp = XH[ix], xm = XH[ix - 1];
    const double2 zj = Z[iz], zp = ZH[iz], zm = ZH[iz - 1];
    const double2 cxp = cdiv(zj, rmul(h2, xp));
    const double2 cxm = cdiv(zj, rmul(h2, xm));
    const double2 czp = cdiv(xi, rmul(h2, zp));
    const double2 czm = cdiv(xi, rmul(h2, zm));
    const double t = __dmul_rn(w2, s[node]);
    const double2 mass = cmul(rmul(t, xi), zj);
    // SparseMatrixCSR::from_triplets stores 0 + value (src/sparse.cpp:45-50),
    // which normalises -0 to +0; do the same so the planes equal the CSR bitwise.
    diag[node] = cadd(cz(), csub(cadd(cadd(cadd(cxp, cxm), czp), czm), mass));
    east[node] = on_boundary(ix + 1, iz, nx, nz) ? cz() : cadd(cz(), make_double2(-cxp.x, -cxp.y));
    south[node] = on_boundary(ix, iz + 1, nx, nz) ? cz() : cadd(cz(), make_double2(-czp.x, -czp.y));
}

__global__ void to_c64_kernel(const double2* __restrict__ a, float2* __restrict__ b, int64_t m) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m;
         i += int64_t(gridDim.x) * blockDim.x)
        b[i] = make_float2(float(a[i].x), float(a[i].y));
}

// d_pred = observe(u) (src/forward.cpp:78-91); r = d_obs - d_pred.
__global__ void observe_kernel(int K, int64_t n, const int* __restrict__ off,
                               const int* __restrict__ node, const double2* __restrict__ u,
                               const double2* __restrict__ dobs, double2* __restrict__ dpred,
                               double2* __restrict__ r) {
    const int k = blockIdx.x;
    for (int j = off[k] + threadIdx.x; j < off[k + 1]; j += blockDim.x) {
        const double2 v = u[int64_t(k) * n + node[j]];
        dpred[j] = v;
        if (dobs) r[j] = csub(dobs[j], v);
    }
}

template <class T>
void upload(DevBuf<T>& b, const T* h, size_t n, cudaStream_t st) {
    b.alloc(n);
    if (n) CK(cudaMemcpyAsync(b.p, h, n * sizeof(T), cudaMemcpyHostToDevice, st));
}

}  // namespace

int sm_count() {
    static int v = [] {
        int dev = 0, c = 0;
        if (cudaGetDevice(&dev) != cudaSuccess) return 148;
        if (cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
        return c > 0 ? c : 148;
    }();
    return v;
}

Ctx::~Ctx() {
    if (gmres_work) gmres_work_free(gmres_work);
    if (exact) exact_free(exact);
    if (ilu) ilu_free(ilu);
    for (auto*& p : kplan)
        if (p) kkt_plan_free(p);
    for (auto*& p : kplan_alt)
        if (p) kkt_plan_free(p);
    for (auto*& p : kmplan)
        if (p) kkt_km_plan_free(p);
    for (auto& e : ev_in)
        if (e) cudaEventDestroy(e);
    for (auto& e : ev_out)
        if (e) cudaEventDestroy(e);
    if (s_h2d) cudaStreamDestroy(s_h2d);
    if (s_d2h) cudaStreamDestroy(s_d2h);
    if (stream) cudaStreamDestroy(stream);
}

void Ctx::ensure_work(unsigned which) {
    const size_t kn = size_t(K) * n;
    if ((which & kWorkA) && work_a.count < kn) work_a.alloc(kn);
    if ((which & kWorkB) && work_b.count < kn) work_b.alloc(kn);
    if ((which & kWorkC) && work_c.count < kn) work_c.alloc(kn);
    if (work_ds.count < size_t(ds_stride)) work_ds.alloc(ds_stride);
}

Ctx* ctx_create(const fwi_state_desc& d) {
    // ---- validation: build_grid (src/grid.cpp:9-19), SlownessModel::validate
    // (src/helmholtz.cpp:8-15), Survey::validate (src/forward.cpp:23-41),
    // make_gn_state (src/reduced_space.cpp:44-51).
    const fwi_grid_desc& g = d.grid;
    require(g.nx >= 3 && g.nz >= 3, "build_grid: need nx >= 3 and nz >= 3");
    require(g.h > 0.0, "build_grid: spacing h must be positive");
    require(g.n_pml >= 0, "build_grid: n_pml must be non-negative");
    require(2 * g.n_pml < std::min(g.nx, g.nz), "build_grid: PML frame consumes the whole domain");
    require(d.freq_hz > 0.0, "make_gn_state: frequency must be positive");
    require(d.epsilon > 0.0, "make_gn_state: epsilon must be positive");
    require(d.s != nullptr, "make_gn_state: slowness model is required");
    const fwi_survey_desc& sv = d.survey;
    require(sv.num_sources >= 1, "Survey: no sources");
    const int nx = g.nx, nz = g.nz;
    const int64_t n = int64_t(nx) * nz;
    require(n < (int64_t(1) << 31), "grid too large for int32 node indices");
    for (int64_t i = 0; i < n; ++i)
        require(d.s[i] > 0.0 && std::isfinite(d.s[i]),
                "SlownessModel: values must be positive and finite");
    auto usable = [&](int ix, int iz) {
        const bool core = ix >= g.n_pml && ix < nx - g.n_pml && iz >= g.n_pml && iz < nz - g.n_pml;
        return core && !on_boundary(ix, iz, nx, nz);
    };
    for (int k = 0; k < sv.num_sources; ++k) {
        require(usable(sv.src_ix[k], sv.src_iz[k]),
                "Survey: source " + std::to_string(k) + " is outside the core region");
        for (int j = sv.recv_offset[k]; j < sv.recv_offset[k + 1]; ++j)
            require(usable(sv.recv_ix[j], sv.recv_iz[j]),
                    "Survey: receiver of source " + std::to_string(k) + " is outside the core region");
    }

    auto c = std::make_unique<Ctx>();
    c->nx = nx;
    c->nz = nz;
    c->n = int(n);
    c->K = sv.num_sources;
    c->ndata = sv.recv_offset[sv.num_sources];
    c->n_pml = g.n_pml;
    c->h = g.h;
    c->sigma_max = g.pml_sigma_max;
    c->power = g.pml_power;
    c->freq_hz = d.freq_hz;
    c->omega = 2.0 * kPi * d.freq_hz;
    c->w2 = c->omega * c->omega;
    c->eps = d.epsilon;
    c->drop = d.drop_reg_term != 0;
    c->ds_stride = (n + 31) / 32 * 32;
    c->vec_len = 4 * int64_t(c->K) * n + c->ds_stride;
    c->precision_mask = d.precision_mask;
    if (const char* v = std::getenv("FWI_KKT_KERNEL")) c->kkt_variant = std::string(v) == "plain" ? 1 : std::string(v) == "tile" ? 2 : 0;
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    cudaStream_t st = c->stream;

    // ---- stencil
    std::vector<double> X(2 * nx), XH(2 * (nx - 1)), Z(2 * nz), ZH(2 * (nz - 1));
    for (int i = 0; i < nx; ++i) stretch_host(nx, g.n_pml, g.pml_sigma_max, g.pml_power, i, c->omega, &X[2 * i]);
    for (int i = 0; i + 1 < nx; ++i)
        stretch_host(nx, g.n_pml, g.pml_sigma_max, g.pml_power, i + 0.5, c->omega, &XH[2 * i]);
    for (int i = 0; i < nz; ++i) stretch_host(nz, g.n_pml, g.pml_sigma_max, g.pml_power, i, c->omega, &Z[2 * i]);
    for (int i = 0; i + 1 < nz; ++i)
        stretch_host(nz, g.n_pml, g.pml_sigma_max, g.pml_power, i + 0.5, c->omega, &ZH[2 * i]);
    DevBuf<double2> dX, dXH, dZ, dZH;
    upload(dX, reinterpret_cast<const double2*>(X.data()), nx, st);
    upload(dXH, reinterpret_cast<const double2*>(XH.data()), nx - 1, st);
    upload(dZ, reinterpret_cast<const double2*>(Z.data()), nz, st);
    upload(dZH, reinterpret_cast<const double2*>(ZH.data()), nz - 1, st);
    c->h_s.assign(d.s, d.s + n);
    upload(c->s, d.s, n, st);
    c->diag.alloc(n);
    c->east.alloc(n);
    c->south.alloc(n);
    {
        dim3 blk(32, 8), grd((nx + 31) / 32, (nz + 7) / 8);
        assemble_kernel<<<grd, blk, 0, st>>>(nx, nz, g.h * g.h, c->w2, c->s.p, dX.p, dXH.p, dZ.p,
                                             dZH.p, c->diag.p, c->east.p, c->south.p);
        CK_LAUNCH();
    }

    // ---- survey: weights (build_weights, src/forward.cpp:43-62) and node lists
    const int K = c->K, nd = c->ndata;
    c->h_recv_offset.assign(sv.recv_offset, sv.recv_offset + K + 1);
    c->h_recv_node.resize(nd);
    c->h_w.assign(nd, 1.0);
    c->h_src_node.resize(K);
    c->h_src_amp.resize(K);
    for (int k = 0; k < K; ++k) {
        c->h_src_node[k] = sv.src_iz[k] * nx + sv.src_ix[k];
        c->h_src_amp[k] = sv.src_amp ? sv.src_amp[k] : 1.0;
        for (int j = sv.recv_offset[k]; j < sv.recv_offset[k + 1]; ++j)
            c->h_recv_node[j] = sv.recv_iz[j] * nx + sv.recv_ix[j];
    }
    if (sv.weight_mode == FWI_WEIGHT_OFFSET) {
        double maxw = 0.0;
        for (int k = 0, i = 0; k < K; ++k)
            for (int j = sv.recv_offset[k]; j < sv.recv_offset[k + 1]; ++j, ++i) {
                const double dx = sv.recv_ix[j] - sv.src_ix[k], dz = sv.recv_iz[j] - sv.src_iz[k];
                c->h_w[i] = std::sqrt(dx * dx + dz * dz);
                maxw = std::max(maxw, c->h_w[i]);
            }
        if (maxw > 0.0)
            for (auto& v : c->h_w) v /= maxw;
    }
    upload(c->recv_offset, c->h_recv_offset.data(), K + 1, st);
    upload(c->recv_node, c->h_recv_node.data(), nd, st);
    upload(c->w, c->h_w.data(), nd, st);
    {
        // per-node table for the fused F block: entries sorted by (node, k, j)
        std::vector<int> cnt(n + 1, 0);
        for (int j = 0; j < nd; ++j) cnt[c->h_recv_node[j] + 1]++;
        for (int64_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
        std::vector<int> pos(cnt.begin(), cnt.end() - 1), ek(std::max(nd, 1));
        std::vector<double> ew(std::max(nd, 1));
        for (int k = 0; k < K; ++k)
            for (int j = c->h_recv_offset[k]; j < c->h_recv_offset[k + 1]; ++j) {
                const int p = pos[c->h_recv_node[j]]++;
                ek[p] = k;
                ew[p] = c->h_w[j] * c->h_w[j];
            }
        c->nrec_dup = false;
        for (int64_t i = 0; i < n && !c->nrec_dup; ++i)
            for (int q = cnt[i]; q + 1 < cnt[i + 1]; ++q)
                if (ek[q] == ek[q + 1]) {
                    c->nrec_dup = true;
                    break;
                }
        upload(c->nrec_ptr, cnt.data(), n + 1, st);
        upload(c->nrec_k, ek.data(), ek.size(), st);
        upload(c->nrec_w2, ew.data(), ew.size(), st);
    }

    // ---- reduction scratch
    c->red_partials.alloc(4096);
    c->red_ticket.alloc(64);
    CK(cudaMemsetAsync(c->red_ticket.p, 0, 64 * sizeof(unsigned), st));
    c->red_out.alloc(1024);

    // ---- factorisations and fields
    const bool need_exact = d.exact_factor || d.u == nullptr;
    if (need_exact) exact_factor(*c);
    c->u.alloc(size_t(K) * n);
    if (d.u) {
        CK(cudaMemcpyAsync(c->u.p, d.u, size_t(K) * n * sizeof(double2), cudaMemcpyHostToDevice, st));
    } else {
        // solve_forward (src/forward.cpp:64-76): f_k = amplitude/h^2 at the source node
        std::vector<double2> f(size_t(K) * n, make_double2(0.0, 0.0));
        const double load = 1.0 / (g.h * g.h);
        for (int k = 0; k < K; ++k) f[size_t(k) * n + c->h_src_node[k]].x = c->h_src_amp[k] * load;
        DevBuf<double2> df;
        upload(df, f.data(), f.size(), st);
        exact_solve_batch(*c, false, df.p, c->u.p, K);
        c->solve_count[FWI_PRECOND_EXACT] = 0;  // setup solves are not counted (as after make_gn_state)
        CK(cudaStreamSynchronize(st));
    }
    c->r.alloc(std::max(nd, 1));
    c->dpred.alloc(std::max(nd, 1));
    CK(cudaMemsetAsync(c->r.p, 0, std::max(nd, 1) * sizeof(double2), st));
    if (nd) {
        DevBuf<double2> dobs;
        if (d.d_obs && !d.r) upload(dobs, reinterpret_cast<const double2*>(d.d_obs), nd, st);
        observe_kernel<<<K, 128, 0, st>>>(K, n, c->recv_offset.p, c->recv_node.p, c->u.p, dobs.p,
                                          c->dpred.p, c->r.p);
        CK_LAUNCH();
        if (d.r) CK(cudaMemcpyAsync(c->r.p, d.r, nd * sizeof(double2), cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
    }
    if (d.ilu_level >= 0) ilu_factor(*c, d.ilu_level, d.ilu_diag_shift);

    if (c->precision_mask & (1 << FWI_C64)) {
        c->u32.alloc(size_t(K) * n);
        c->diag32.alloc(n);
        c->east32.alloc(n);
        c->south32.alloc(n);
        const int nb = grid_blocks(int64_t(K) * n, 256, 8 * sm_count());
        to_c64_kernel<<<nb, 256, 0, st>>>(c->u.p, c->u32.p, int64_t(K) * n);
        to_c64_kernel<<<grid_blocks(n, 256, 8 * sm_count()), 256, 0, st>>>(c->diag.p, c->diag32.p, n);
        to_c64_kernel<<<grid_blocks(n, 256, 8 * sm_count()), 256, 0, st>>>(c->east.p, c->east32.p, n);
        to_c64_kernel<<<grid_blocks(n, 256, 8 * sm_count()), 256, 0, st>>>(c->south.p, c->south32.p, n);
        CK_LAUNCH();
    }
    CK(cudaStreamSynchronize(st));
    return c.release();
}

void stencil_to_host(const Ctx& c, double* diag, double* east, double* south) {
    CK(cudaStreamSynchronize(c.stream));
    const size_t b = size_t(c.n) * sizeof(double2);
    if (diag) CK(cudaMemcpy(diag, c.diag.p, b, cudaMemcpyDeviceToHost));
    if (east) CK(cudaMemcpy(east, c.east.p, b, cudaMemcpyDeviceToHost));
    if (south) CK(cudaMemcpy(south, c.south.p, b, cudaMemcpyDeviceToHost));
}

bool pdl_enabled(int group) {
    static const bool on = !(std::getenv("FWI_PDL") && std::atoi(std::getenv("FWI_PDL")) == 0);
    // the fused MGS sweep (software grid barrier) runs slower as a dependent launch at config 3
    // (2.05 against 2.45 ms per GMRES iteration with it), so it is off by default
    static const int off = std::getenv("FWI_PDL_OFF") ? std::atoi(std::getenv("FWI_PDL_OFF")) : kPdlMgs;
    return on && !(group & off);
}

}  // namespace fwi_b200
