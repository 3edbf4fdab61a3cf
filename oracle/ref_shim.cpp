// oracle/_ref: the UNMODIFIED reference solver (/root/reference/proj/include/esp,
// header-only C++20) compiled into a shared library with a flat C ABI so the
// Python test-suite and bench.py's cpu_baseline leg can call it.
//
// TEST INFRASTRUCTURE ONLY.  Nothing in the product path
// (paper_2505_09727_b200/) links, loads or calls this library; it is the
// parity checker and the timed CPU reference arm.  The only substitution is
// FFTW3, which is absent from the image and is supplied by
// oracle/fftw_shim (see that header).  No reference source is copied: this
// file only includes the headers where they lie and forwards to them.
//
// Every wrapper returns 0 on success, 1 for std::invalid_argument,
// 2 for esp::NumericalError, 3 for esp::IoError, 4 for any other exception;
// ref_last_error() returns the message of the last failure (thread-local).

#include "esp/esp.hpp"

#include <cstring>
#include <string>

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const esp::NumericalError& e) {
        g_err = e.what();
        return 2;
    } catch (const esp::IoError& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

esp::ParticleSystem make_system(const double* box, long N, const double* pos, const double* q) {
    esp::ParticleSystem s;
    s.box = {box[0], box[1], box[2]};
    s.q.assign(q, q + N);
    s.pos.resize(N);
    for (long i = 0; i < N; ++i) s.pos[i] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
    return s;
}

void put_vec3(const std::vector<esp::Vec3>& v, double* out) {
    for (std::size_t i = 0; i < v.size(); ++i)
        for (int d = 0; d < 3; ++d) out[3 * i + d] = v[i][d];
}

void put_pc(const esp::detail::PiecewiseCheb& pc, double* coef, double* geom) {
    // coef: nseg x ncoef row-major; geom: lo, hi, inv_width, nseg, ncoef
    int k = 0;
    for (const auto& s : pc.segs)
        for (double c : s.coef) coef[k++] = c;
    if (geom) {
        geom[0] = pc.lo;
        geom[1] = pc.hi;
        geom[2] = pc.inv_width;
        geom[3] = static_cast<double>(pc.segs.size());
        geom[4] = pc.segs.empty() ? 0.0 : static_cast<double>(pc.segs[0].coef.size());
    }
}

}  // namespace

extern "C" {

struct ref_plan {
    esp::EwaldPlan plan;
};

// Flat mirror of the EwaldPlan scalars (ewald.hpp:67-94).
struct ref_plan_info {
    int family, window_family, force_method, P;
    int nf[3], base_nf[3];
    double eps, r_c, shape, c1, chi0, C0_split;
    double box[3], h[3], demand[3];
    double E_A, E_T, E_SI;
    int split_ncoef, split_nterms, win_nterms, pad;
};

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_threads(int n) { esp::thread_count() = n < 1 ? 1 : n; }
int ref_get_threads() { return esp::thread_count(); }

int ref_build_plan(const double* box, int family, double eps, double r_c, int ov_nf, int ov_P,
                   double ov_c1, int force_method, int allow_degraded, ref_plan** out) {
    return guarded([&] {
        esp::Overrides ov;
        ov.nf = ov_nf;
        ov.P = ov_P;
        ov.c1 = ov_c1;
        ov.force_method = force_method == 1 ? esp::ForceMethod::ad : esp::ForceMethod::ik;
        ov.allow_degraded = allow_degraded != 0;
        auto* h = new ref_plan;
        try {
            h->plan = esp::build_plan({box[0], box[1], box[2]},
                                      family == 1 ? esp::SplitFamily::gaussian
                                                  : esp::SplitFamily::pswf,
                                      eps, r_c, ov);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

void ref_plan_free(ref_plan* h) { delete h; }

int ref_plan_info_get(const ref_plan* h, ref_plan_info* o) {
    return guarded([&] {
        const esp::EwaldPlan& p = h->plan;
        std::memset(o, 0, sizeof(*o));
        o->family = p.family == esp::SplitFamily::gaussian ? 1 : 0;
        o->window_family = p.window_family == esp::WindowFamily::bspline ? 1 : 0;
        o->force_method = p.force_method == esp::ForceMethod::ad ? 1 : 0;
        o->P = p.P;
        for (int d = 0; d < 3; ++d) {
            o->nf[d] = p.nf[d];
            o->base_nf[d] = p.base_nf[d];
            o->box[d] = p.box[d];
            o->h[d] = p.h[d];
            o->demand[d] = p.demand[d];
        }
        o->eps = p.eps;
        o->r_c = p.r_c;
        o->shape = p.shape;
        o->c1 = p.c1;
        o->chi0 = p.split.chi0;
        o->C0_split = p.split.prolate.C0;
        o->E_A = p.stats.E_A;
        o->E_T = p.stats.E_T;
        o->E_SI = p.stats.E_SI;
        o->split_ncoef = p.split.Psi_pc.segs.empty()
                             ? 0
                             : static_cast<int>(p.split.Psi_pc.segs.size()
                                                * p.split.Psi_pc.segs[0].coef.size());
        o->split_nterms = static_cast<int>(p.split.prolate.coef.size());
        o->win_nterms = static_cast<int>(p.win[0].prolate.coef.size());
    });
}

int ref_plan_influence(const ref_plan* h, double* out) {
    return guarded([&] {
        const auto& v = h->plan.influence;
        std::memcpy(out, v.data(), sizeof(double) * v.size());
    });
}

// Psi / chi compiled tables (kernels.hpp:130-136): 16 x 13 each; geom = 5 doubles.
int ref_plan_split_tables(const ref_plan* h, double* psi, double* chi, double* geom) {
    return guarded([&] {
        put_pc(h->plan.split.Psi_pc, psi, geom);
        put_pc(h->plan.split.chi_pc, chi, nullptr);
    });
}

// Prolate Legendre coefficients of the split (a_k, psi(0)=1) and of window d.
int ref_plan_prolate_coef(const ref_plan* h, int which, double* out) {
    return guarded([&] {
        const auto& c = which < 0 ? h->plan.split.prolate.coef : h->plan.win[which].prolate.coef;
        std::memcpy(out, c.data(), sizeof(double) * c.size());
    });
}

// Window d: phi and dphi tables (4P x 13 each; kernels.hpp:234-244).
int ref_plan_window_tables(const ref_plan* h, int d, double* phi, double* dphi, double* geom) {
    return guarded([&] {
        put_pc(h->plan.win[d].phi_pc, phi, geom);
        put_pc(h->plan.win[d].dphi_pc, dphi, nullptr);
    });
}

// Point evaluators used to check restated kernels (kernels.hpp:76-95,188-229).
int ref_plan_eval_kernels(const ref_plan* h, int what, long n, const double* x, double* y) {
    return guarded([&] {
        const esp::EwaldPlan& p = h->plan;
        for (long i = 0; i < n; ++i) {
            switch (what) {
                case 0: y[i] = p.split.Psi(x[i]); break;
                case 1: y[i] = p.split.chi(x[i]); break;
                case 2: y[i] = p.split.chihat_n(x[i]); break;
                case 3: y[i] = p.win[0].phi(x[i]); break;
                case 4: y[i] = p.win[0].dphi(x[i]); break;
                case 5: y[i] = p.win[0].phi_hat(x[i]); break;
                case 6: y[i] = esp::local_kernel(p.split, x[i]).first; break;
                case 7: y[i] = esp::local_kernel(p.split, x[i]).second; break;
                default: throw std::invalid_argument("ref_plan_eval_kernels: bad selector");
            }
        }
    });
}

int ref_evaluate(const ref_plan* h, const double* box, long N, const double* pos,
                 const double* q, double* u, double* F, double* energy, double* timings) {
    return guarded([&] {
        esp::ParticleSystem s = make_system(box, N, pos, q);
        esp::EnergyForces ef = esp::evaluate(h->plan, s);
        std::memcpy(u, ef.u.data(), sizeof(double) * N);
        put_vec3(ef.F, F);
        *energy = ef.energy;
        if (timings) {
            const char* keys[6] = {"local", "spread", "fft", "scale", "ifft", "interpolate"};
            for (int k = 0; k < 6; ++k) timings[k] = ef.timings.at(keys[k]);
        }
    });
}

int ref_local_sum(const ref_plan* h, const double* box, long N, const double* pos,
                  const double* q, double* u, double* F) {
    return guarded([&] {
        esp::PartialField f = esp::local_sum(h->plan, make_system(box, N, pos, q));
        std::memcpy(u, f.u.data(), sizeof(double) * N);
        put_vec3(f.F, F);
    });
}

int ref_spectral_sum(const ref_plan* h, const double* box, long N, const double* pos,
                     const double* q, double* u, double* F) {
    return guarded([&] {
        esp::PartialField f = esp::spectral_sum(h->plan, make_system(box, N, pos, q));
        std::memcpy(u, f.u.data(), sizeof(double) * N);
        put_vec3(f.F, F);
    });
}

int ref_self_correction(const ref_plan* h, long N, const double* q, double* out) {
    return guarded([&] {
        std::vector<double> qq(q, q + N);
        auto s = esp::self_correction(h->plan, qq);
        std::memcpy(out, s.data(), sizeof(double) * N);
    });
}

// spread (gridder.hpp:215-241) on the positions as given; real part of the grid.
int ref_spread(const ref_plan* h, long N, const double* pos, const double* q, double* grid) {
    return guarded([&] {
        esp::GridArray g = esp::spread(make_system(h->plan.box.data(), N, pos, q), h->plan.win,
                                       h->plan.nf);
        for (std::size_t i = 0; i < g.v.size(); ++i) grid[i] = g.v[i].real();
    });
}

int ref_interpolate(const ref_plan* h, long N, const double* pos, const double* grid,
                    double* out) {
    return guarded([&] {
        esp::GridArray g = esp::GridArray::zeros(h->plan.nf);
        for (std::size_t i = 0; i < g.v.size(); ++i) g.v[i] = {grid[i], 0.0};
        std::vector<double> q(N, 0.0);
        auto u = esp::interpolate(g, h->plan.win, make_system(h->plan.box.data(), N, pos, q.data()));
        std::memcpy(out, u.data(), sizeof(double) * N);
    });
}

int ref_interpolate_gradient(const ref_plan* h, long N, const double* pos, const double* grid,
                             double* out) {
    return guarded([&] {
        esp::GridArray g = esp::GridArray::zeros(h->plan.nf);
        for (std::size_t i = 0; i < g.v.size(); ++i) g.v[i] = {grid[i], 0.0};
        std::vector<double> q(N, 0.0);
        auto gr = esp::interpolate_gradient(g, h->plan.win,
                                            make_system(h->plan.box.data(), N, pos, q.data()));
        put_vec3(gr, out);
    });
}

// In-place 3-D c2c on interleaved complex data through gridder.hpp's wrappers.
int ref_fft3(int n0, int n1, int n2, double* data, int sign) {
    return guarded([&] {
        esp::GridArray g = esp::GridArray::zeros({n0, n1, n2});
        for (std::size_t i = 0; i < g.v.size(); ++i) g.v[i] = {data[2 * i], data[2 * i + 1]};
        if (sign < 0) esp::fft_forward(g);
        else esp::fft_inverse(g);
        for (std::size_t i = 0; i < g.v.size(); ++i) {
            data[2 * i] = g.v[i].real();
            data[2 * i + 1] = g.v[i].imag();
        }
    });
}

// direct_ewald (reference.hpp:212-238); info = lambda, real_shells, recip_kmax, residual.
int ref_direct_ewald(const double* box, long N, const double* pos, const double* q, double tol,
                     double* u, double* F, double* energy, double* info) {
    return guarded([&] {
        esp::ReferenceResult r = esp::direct_ewald(make_system(box, N, pos, q), tol);
        std::memcpy(u, r.u.data(), sizeof(double) * N);
        put_vec3(r.F, F);
        *energy = r.energy;
        if (info) {
            info[0] = r.lambda;
            info[1] = r.real_shells;
            info[2] = r.recip_kmax;
            info[3] = r.residual;
        }
    });
}

int ref_relative_force_error(long N, const double* test, const double* ref, double* out) {
    return guarded([&] {
        std::vector<esp::Vec3> a(N), b(N);
        for (long i = 0; i < N; ++i)
            for (int d = 0; d < 3; ++d) {
                a[i][d] = test[3 * i + d];
                b[i][d] = ref[3 * i + d];
            }
        *out = esp::relative_force_error(a, b);
    });
}

// generate_system (io.hpp:82-148): kind 0 random, 1 rocksalt, 2 water-like lattice.
int ref_generate(int kind, long N, const double* box, unsigned long long seed, double* pos,
                 double* q) {
    return guarded([&] {
        esp::GeneratorSpec spec;
        spec.kind = kind == 1 ? esp::SystemKind::rocksalt
                              : kind == 2 ? esp::SystemKind::water_like : esp::SystemKind::random;
        spec.N = static_cast<std::size_t>(N);
        spec.box = {box[0], box[1], box[2]};
        spec.seed = seed;
        esp::ParticleSystem s = esp::generate_system(spec);
        std::memcpy(q, s.q.data(), sizeof(double) * N);
        put_vec3(s.pos, pos);
    });
}

int ref_solve_c(double eps, double* c) {
    return guarded([&] { *c = esp::solve_c(eps); });
}

int ref_next_even_5smooth(double x, int* out) {
    return guarded([&] { *out = esp::detail::next_even_5smooth(x); });
}

}  // extern "C"
