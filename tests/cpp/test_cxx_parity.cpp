// C++ parity test: the drop-in header fwi_b200/kkt.hpp (GPU) against the
// reference library (namespace fwi, compiled from /root/reference/proj/src
// into oracle/_ref) on the reference's own standard fixture
// (tests/support/fixtures.hpp:48-81 restated). Reads like the reference's
// tests/test_kkt.cpp. Exit code 0 = all checks passed.
#include <cmath>
#include <cstdio>
#include <algorithm>
#include <numbers>
#include <random>

#include "fwi/driver.hpp"
#include "fwi/ilu.hpp"
#include "fwi/kkt.hpp"
#include "fwi/krylov.hpp"
#include "fwi/lu.hpp"
#include "fwi/model_io.hpp"
#include "fwi_b200/kkt.hpp"

static int failures = 0;
#define CHECK(cond)                                                        \
    do {                                                                   \
        if (!(cond)) {                                                     \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);    \
            ++failures;                                                    \
        }                                                                  \
    } while (0)

using namespace fwi;

struct StandardInputs {  // the reference's standard fixture, as make_gn_state's arguments
    Grid2D grid;
    PmlProfile prof;
    SlownessModel initial;
    Survey sv;
    DataVector dobs;
    GnStateOptions o;
};

static StandardInputs standard_inputs(int ilu_level) {
    StandardInputs in;
    in.grid = build_grid(12, 12, 1.0, 2);
    in.prof = make_pml_profile(in.grid, 1.0);
    const SlownessModel truth = make_lens_model(in.grid, 1.0, 0.15, 5.5, 5.5, 2.0).to_slowness();
    in.initial.s.assign(in.grid.num_nodes(), 1.0);
    in.sv.frequencies_hz = {0.15};
    Survey::Source a, b;
    a.ix = 3, a.iz = 3, b.ix = 8, b.iz = 3;
    for (int ix = 3; ix <= 8; ++ix) {
        a.receivers.emplace_back(ix, 8);
        b.receivers.emplace_back(ix, 8);
    }
    in.sv.sources = {a, b};
    const double omega = 2.0 * 3.14159265358979323846 * 0.15;
    const LuFactors lu = LuFactors::factor(assemble_helmholtz(in.grid, in.prof, truth, omega).a);
    in.dobs = observe(in.grid, in.sv, solve_forward(lu, in.grid, in.sv));
    in.o.epsilon = 1e-2;
    if (ilu_level >= 0) in.o.ilu_level = ilu_level;
    return in;
}

static GnState standard_state(int ilu_level) {
    const StandardInputs in = standard_inputs(ilu_level);
    return make_gn_state(in.grid, in.prof, in.initial, in.sv, 0.15, in.dobs, in.o);
}

static double rel_c(const std::vector<std::complex<double>>& a, const std::vector<std::complex<double>>& b) {
    double num = 0, den = 0;
    for (size_t i = 0; i < a.size(); ++i) {
        num += std::norm(a[i] - b[i]);
        den += std::norm(b[i]);
    }
    return std::sqrt(num / den);
}

// squared slowness whose stencil diagonal 4/h^2 - w^2 s cancels exactly (h = 1, no PML):
// the exact-zero pivot of tests/test_ilu.cpp:107-120 and the zero row of
// tests/test_lu.cpp:44-47, built from a real Helmholtz instance
static double cancelling_slowness(double omega) {
    const double w2 = omega * omega;
    double s = 4.0 / w2;
    for (int t = 0; t < 64 && w2 * s != 4.0; ++t) s = std::nextafter(s, w2 * s > 4.0 ? 0.0 : 10.0);
    return s;
}

static KktVector random_kkt(const GnState& st, unsigned seed) {
    std::mt19937 rng(seed);
    std::normal_distribution<double> nd(0.0, 1.0);
    KktVector v = KktVector::zeros(st.num_sources(), st.model_size(), st.model_size());
    for (auto& b : v.du)
        for (auto& z : b) z = {nd(rng), nd(rng)};
    for (auto& z : v.ds) z = nd(rng);
    for (auto& b : v.lambda)
        for (auto& z : b) z = {nd(rng), nd(rng)};
    return v;
}

static bool same(const KktVector& a, const KktVector& b) {
    for (size_t k = 0; k < a.du.size(); ++k)
        if (a.du[k] != b.du[k] || a.lambda[k] != b.lambda[k]) return false;
    return a.ds == b.ds;
}

static double rel(const KktVector& a, const KktVector& b) {
    KktVector d = a;
    axpy(-1.0, b, d);
    return norm(d) / norm(b);
}

int main() {
    const GnState ref = standard_state(1000);
    // the reference's own linearisation point on the device (u, r uploaded as they are)
    gpu::GnState dev = gpu::gn_state_from_reference(ref, 1000);

    // kkt_apply, bit for bit (tests/test_kkt.cpp:71-79 asks 1e-10)
    for (unsigned s = 0; s < 5; ++s) {
        const KktVector xi = random_kkt(ref, 100 + 7 * s);
        gpu::KktVector gx(dev);
        gx.upload_from(xi);
        KktVector got = xi;
        gpu::kkt_apply(dev, gx).download_into(got);
        CHECK(same(got, kkt_apply(ref, xi)));
    }
    // kkt_rhs and the drop flag (tests/test_kkt.cpp:110-130)
    {
        KktVector got = KktVector::zeros(ref.num_sources(), ref.model_size(), ref.model_size());
        gpu::kkt_rhs(dev).download_into(got);
        CHECK(same(got, kkt_rhs(ref)));
    }
    // symmetry in the real inner product (tests/test_kkt.cpp:81-90)
    for (unsigned s = 0; s < 4; ++s) {
        gpu::KktVector a(dev), b(dev);
        a.upload_from(random_kkt(ref, 300 + s));
        b.upload_from(random_kkt(ref, 800 + s));
        const double lhs = gpu::dot(gpu::kkt_apply(dev, a), b), rhs = gpu::dot(gpu::kkt_apply(dev, b), a);
        CHECK(std::abs(lhs - rhs) <= 1e-12 * std::max(1.0, std::abs(lhs)));
    }
    // ILU at full fill equals exact (tests/test_kkt.cpp:142-151); ILU bit-exact to the reference
    {
        const KktVector v = random_kkt(ref, 55);
        gpu::KktVector gv(dev);
        gv.upload_from(v);
        KktVector ilu = v, ex = v;
        gpu::precond_apply(dev, gv, gpu::PrecondMode::ilu).download_into(ilu);
        gpu::precond_apply(dev, gv, gpu::PrecondMode::exact).download_into(ex);
        CHECK(same(ilu, precond_apply(ref, v, PrecondMode::ilu)));
        CHECK(rel(ex, precond_apply(ref, v, PrecondMode::exact)) < 1e-10);
        CHECK(rel(ilu, ex) < 1e-10);
    }
    // cost contract (tests/test_kkt.cpp:153-159)
    {
        gpu::KktVector gv(dev);
        gv.upload_from(random_kkt(ref, 7));
        dev.reset_solve_count();
        (void)gpu::precond_apply(dev, gv, gpu::PrecondMode::exact);
        CHECK(dev.solve_count() == 2 * ref.num_sources());
    }
    // fsgn: residual histories within 1e-8, the E_cg column populated (tests/test_kkt.cpp:161-177)
    {
        FsgnOptions fo;
        fo.mode = PrecondMode::exact;
        fo.tol = 1e-10;
        fo.maxit = 200;
        const StepResult want = fsgn_gmres_step(ref, fo);
        gpu::FsgnOptions go;
        go.tol = 1e-10;
        go.maxit = 200;
        const gpu::StepResult got = gpu::fsgn_gmres_step(dev, go);
        CHECK(got.log.converged == want.log.converged);
        CHECK(got.log.entries.size() == want.log.entries.size());
        // 1e-8 relative per iteration while the residual is above 1e-7; this 12x12 fixture
        // converges to 6e-11 in 11 iterations, and at that level both histories are rounding
        // noise, held to an absolute 1e-14 instead. (The north-star gate with no floor is
        // tests/test_gpu_history_gate.py on config 1, whose 50 iterations stay above 9e-7.)
        double worst = 0.0, worst_abs = 0.0;
        for (size_t i = 0; i < std::min(got.log.entries.size(), want.log.entries.size()); ++i) {
            const double a = got.log.entries[i].residual_norm, b = want.log.entries[i].residual_norm;
            const double d = std::abs(a - b) / b;
            std::printf("iter %2zu  ref %.6e  gpu %.6e  rel.dev %.2e\n", i, b, a, d);
            if (b >= 1e-7) worst = std::max(worst, d);
            else worst_abs = std::max(worst_abs, std::abs(a - b));
            CHECK(got.log.entries[i].normal_residual.has_value());
        }
        std::printf("max history deviation: %.3e relative (residual >= 1e-7), %.3e absolute below\n", worst,
                    worst_abs);
        CHECK(worst <= 1e-8);
        CHECK(worst_abs <= 1e-14);
        double num = 0, den = 0;
        for (size_t i = 0; i < want.delta_s.size(); ++i) {
            num += (got.delta_s[i] - want.delta_s[i]) * (got.delta_s[i] - want.delta_s[i]);
            den += want.delta_s[i] * want.delta_s[i];
        }
        CHECK(std::sqrt(num / den) < 1e-6);
    }
    // reduced-space gradient and Hessian action (src/reduced_space.cpp:120-152)
    {
        const std::vector<double> g = gpu::gradient(dev);
        const RealVector gr = gradient(ref);
        double num = 0, den = 0;
        for (size_t i = 0; i < g.size(); ++i) {
            num += (g[i] - gr[i]) * (g[i] - gr[i]);
            den += gr[i] * gr[i];
        }
        CHECK(std::sqrt(num / den) < 1e-10);
        RealVector v(gr.size());
        for (size_t i = 0; i < v.size(); ++i) v[i] = std::sin(0.37 * double(i));
        const std::vector<double> hv = gpu::hessian_apply(dev, std::vector<double>(v.begin(), v.end()));
        const RealVector hr = hessian_apply(ref, v);
        num = den = 0;
        for (size_t i = 0; i < hv.size(); ++i) {
            num += (hv[i] - hr[i]) * (hv[i] - hr[i]);
            den += hr[i] * hr[i];
        }
        CHECK(std::sqrt(num / den) < 1e-10);
    }
    // the reference's own gmres template (include/fwi/krylov.hpp:128-269) instantiated with the
    // device KktVector (its ADL plug point: copy, dot, norm, axpy, scal) over the device
    // operators, against the fused device GMRES and the reference on the CPU
    {
        auto apply = [&](const gpu::KktVector& v) { return gpu::kkt_apply(dev, v); };
        auto prec = [&](const gpu::KktVector& v) { return gpu::precond_apply(dev, v, gpu::PrecondMode::exact); };
        const gpu::KktVector b = gpu::kkt_rhs(dev);
        auto [x, log] = fwi::gmres(apply, prec, b, 30, 1e-9, 50);
        gpu::FsgnOptions go;
        go.tol = 1e-9;
        go.maxit = 50;
        go.ecg_stride = 0;
        const gpu::StepResult fused = gpu::fsgn_gmres_step(dev, go);
        FsgnOptions fo;
        fo.tol = 1e-9;
        fo.maxit = 50;
        fo.ecg_stride = 0;
        const StepResult want = fsgn_gmres_step(ref, fo);
        CHECK(log.converged && fused.log.converged && want.log.converged);
        CHECK(log.entries.size() == want.log.entries.size());
        CHECK(fused.log.entries.size() == want.log.entries.size());
        double w1 = 0, w2 = 0, a1 = 0, a2 = 0;  // relative above 1e-7, absolute below (as above)
        const size_t ne = std::min({log.entries.size(), fused.log.entries.size(), want.log.entries.size()});
        for (size_t i = 0; i < ne; ++i) {
            const double r = want.log.entries[i].residual_norm, g = log.entries[i].residual_norm;
            const double f = fused.log.entries[i].residual_norm;
            if (r >= 1e-7) {
                w1 = std::max(w1, std::abs(g - r) / r);
                w2 = std::max(w2, std::abs(f - g) / g);
            } else {
                a1 = std::max(a1, std::abs(g - r));
                a2 = std::max(a2, std::abs(f - g));
            }
        }
        std::printf("fwi::gmres<gpu::KktVector> (%zu entries): vs reference %.2e rel / %.2e abs, vs fused device "
                    "GMRES %.2e rel / %.2e abs\n", ne, w1, a1, w2, a2);
        CHECK(w1 <= 1e-8 && a1 <= 1e-14);
        CHECK(w2 <= 1e-8 && a2 <= 1e-14);
        const std::vector<double> xf = x.download();
        const size_t n = size_t(ref.model_size()), K = size_t(ref.num_sources());
        double num = 0, den = 0;
        for (size_t i = 0; i < n; ++i) {
            const double d = xf[2 * K * n + i] - fused.delta_s[i];
            num += d * d;
            den += fused.delta_s[i] * fused.delta_s[i];
        }
        CHECK(std::sqrt(num / den) < 1e-6);
    }
    // fwi::gpu::make_gn_state with the reference's make_gn_state arguments
    // (include/fwi/reduced_space.hpp:51-54): u and r computed on the device
    {
        const StandardInputs in = standard_inputs(1000);
        gpu::GnState dm = gpu::make_gn_state(in.grid, in.prof, in.initial, in.sv, 0.15, in.dobs, in.o);
        std::vector<std::complex<double>> uref;
        for (const auto& uk : ref.u.per_source) uref.insert(uref.end(), uk.begin(), uk.end());
        const double du = rel_c(dm.u(), uref), dr = rel_c(dm.residual(), ref.r);
        std::printf("make_gn_state on the device: u %.2e, r %.2e relative to the reference\n", du, dr);
        CHECK(du < 1e-10);
        CHECK(dr < 1e-8);
        CHECK(dm.info().has_ilu == 1 && dm.info().has_exact == 1);
        GnStateOptions bad = in.o;
        bad.epsilon = 0.0;
        bool threw = false;
        try {
            (void)gpu::make_gn_state(in.grid, in.prof, in.initial, in.sv, 0.15, in.dobs, bad);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
        threw = false;
        DataVector shortd(in.dobs.begin(), in.dobs.end() - 1);
        try {
            (void)gpu::make_gn_state(in.grid, in.prof, in.initial, in.sv, 0.15, shortd, in.o);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
    }
    // complex64 vectors keep their precision through copies and moves; sizes are checked
    {
        const size_t len = size_t(dev.info().vec_doubles);
        std::vector<double> flat(len);
        for (size_t i = 0; i < len; ++i) flat[i] = std::sin(0.1 * double(i));
        gpu::KktVector a(dev, FWI_C64);
        a.upload(flat);
        gpu::KktVector b = a;
        CHECK(b.precision() == FWI_C64);
        CHECK(b.download() == a.download());
        gpu::KktVector m = std::move(a);
        a = m;  // assignment to a moved-from vector
        CHECK(a.precision() == FWI_C64 && a.download() == m.download());
        gpu::KktVector c(dev);
        c = m;  // a complex128 target takes the source's precision
        CHECK(c.precision() == FWI_C64);
        bool threw = false;
        try {
            c.upload(std::vector<double>(len - 1));
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
        threw = false;
        try {
            (void)gpu::precond_apply(dev, c, gpu::PrecondMode::exact);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
    }
    // error conventions (tests/test_ilu.cpp:107-120, tests/test_lu.cpp:44-47) on Helmholtz
    // instances: the device raises the reference's exception types with the same index
    {
        bool threw = false;
        try {
            dev.factor_ilu(-1);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
        const double freq = 0.15, omega = 2.0 * std::numbers::pi * freq;
        const double sc = cancelling_slowness(omega);
        CHECK(omega * omega * sc == 4.0);
        // ZeroPivotError: one interior node whose diagonal cancels exactly (its earlier
        // neighbours are Dirichlet, so its ILU pivot is the bare diagonal)
        {
            const Grid2D g = build_grid(7, 6, 1.0, 0);
            PmlProfile prof;
            prof.sigma_max = 0.0;
            SlownessModel m;
            m.s.assign(g.num_nodes(), 1.0);
            m.s[g.index(1, 1)] = sc;
            int ref_index = -2, dev_index = -3;
            try {
                (void)IluFactors::factor(assemble_helmholtz(g, prof, m, omega).a, 2);
            } catch (const ZeroPivotError& e) {
                ref_index = e.index;
            }
            Survey sv;
            sv.frequencies_hz = {freq};
            Survey::Source src;
            src.ix = 3, src.iz = 3;
            src.receivers = {{4, 3}, {2, 4}};
            sv.sources = {src};
            GnStateOptions o;
            o.epsilon = 1.0;
            o.ilu_level = 2;
            const DataVector dobs(2, std::complex<double>(0.5, -0.25));
            try {
                (void)gpu::make_gn_state(g, prof, m, sv, freq, dobs, o);
            } catch (const gpu::ZeroPivotError& e) {
                dev_index = e.index;
            }
            std::printf("ZeroPivotError index: reference %d, device %d\n", ref_index, dev_index);
            CHECK(ref_index == g.index(1, 1) && dev_index == ref_index);
            o.ilu_diag_shift = 0.5;  // a shift rescues it, as in the reference
            bool ok = true;
            try {
                (void)gpu::make_gn_state(g, prof, m, sv, freq, dobs, o);
            } catch (const std::exception& e) {
                std::printf("unexpected: %s\n", e.what());
                ok = false;
            }
            CHECK(ok);
        }
        // SingularPivotError: the only interior node of a 3x3 grid, diagonal cancelled -> zero row
        {
            const Grid2D g = build_grid(3, 3, 1.0, 0);
            PmlProfile prof;
            prof.sigma_max = 0.0;
            SlownessModel m;
            m.s.assign(g.num_nodes(), 1.0);
            m.s[g.index(1, 1)] = sc;
            int ref_index = -2, dev_index = -3;
            try {
                (void)LuFactors::factor(assemble_helmholtz(g, prof, m, omega).a);
            } catch (const SingularPivotError& e) {
                ref_index = e.index;
            }
            Survey sv;
            sv.frequencies_hz = {freq};
            Survey::Source src;
            src.ix = 1, src.iz = 1;
            src.receivers = {{1, 1}};
            sv.sources = {src};
            GnStateOptions o;
            o.epsilon = 1.0;
            const DataVector dobs(1, std::complex<double>(1.0, 0.0));
            try {
                (void)gpu::make_gn_state(g, prof, m, sv, freq, dobs, o);
            } catch (const gpu::SingularPivotError& e) {
                dev_index = e.index;
            }
            std::printf("SingularPivotError index: reference %d, device %d\n", ref_index, dev_index);
            CHECK(ref_index == g.index(1, 1) && dev_index == ref_index);
        }
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "ok", failures);
    return failures ? 1 : 0;
}
