// Drop-in check: reference-style unit tests (test_ewald.cpp) written against
// include/esp/esp.hpp and run on the GPU through libesp_b200.so.  Plain main,
// one line per check, nonzero exit on failure (the reference's acceptance
// harness style).  Bitwise gates of the reference are tolerances here where
// GPU atomics reorder sums.
#include "esp/esp.hpp"

#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <stdexcept>
#include <vector>

static int failures = 0;
#define CHECK(cond)                                                                  \
    do {                                                                             \
        bool ok_ = (cond);                                                           \
        std::printf("%s  %s:%d  %s\n", ok_ ? "ok  " : "FAIL", __FILE__, __LINE__, #cond); \
        if (!ok_) ++failures;                                                        \
    } while (0)

template <class E, class F>
bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

// splitmix64 random +-1 system (io.hpp:33-44, 92-104)
static esp::ParticleSystem random_system(std::size_t N, esp::Vec3 box, std::uint64_t seed) {
    esp::ParticleSystem s;
    s.box = box;
    std::uint64_t st = seed;
    auto uni = [&st] {
        st += 0x9E3779B97F4A7C15ull;
        std::uint64_t z = st;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return static_cast<double>((z ^ (z >> 31)) >> 11) * 0x1.0p-53;
    };
    for (std::size_t i = 0; i < N; ++i) {
        esp::Vec3 p;
        for (int d = 0; d < 3; ++d) p[d] = box[d] * uni();
        s.pos.push_back(p);
        s.q.push_back(i % 2 == 0 ? 1.0 : -1.0);
    }
    return s;
}

int main() {
    const esp::Vec3 box{10.0, 10.0, 10.0};

    // parameter rows (test_ewald.cpp:26-43)
    {
        const double eps[5] = {1e-3, 5e-4, 1e-4, 5e-5, 1e-5};
        const int nf[5] = {32, 36, 40, 48, 48}, P[5] = {5, 5, 6, 7, 8};
        for (int r = 0; r < 5; ++r) {
            esp::EwaldPlan p = esp::build_plan(box, esp::SplitFamily::pswf, eps[r], 1.0);
            CHECK(p.nf[0] == nf[r] && p.nf[1] == nf[r] && p.nf[2] == nf[r] && p.P == P[r]);
            CHECK(p.stats.E_A <= eps[r]);
        }
    }
    // input rejection (test_ewald.cpp:151-190)
    CHECK(throws<std::invalid_argument>([&] { esp::build_plan(box, esp::SplitFamily::pswf, 1e-6, 1.0); }));
    CHECK(throws<std::invalid_argument>([&] { esp::build_plan(box, esp::SplitFamily::pswf, 1e-4, 5.0); }));
    {
        esp::Overrides odd;
        odd.nf = 15;
        CHECK(throws<std::invalid_argument>([&] { esp::build_plan(box, esp::SplitFamily::pswf, 1e-4, 1.0, odd); }));
        esp::Overrides low;
        low.nf = 20;
        CHECK(throws<esp::NumericalError>([&] { esp::build_plan(box, esp::SplitFamily::pswf, 1e-3, 1.0, low); }));
    }
    // isolated pair (test_ewald.cpp:192-227)
    {
        esp::EwaldPlan plan = esp::build_plan(box, esp::SplitFamily::pswf, 1e-3, 1.0);
        esp::ParticleSystem s;
        s.box = box;
        s.q = {1.0, -1.0};
        s.pos = {{1.0, 1.0, 1.0}, {1.3, 1.0, 1.0}};
        esp::PartialField f = esp::local_sum(plan, s);
        CHECK(f.u[0] == -f.u[1] && f.u[1] > 0.0);
        CHECK(f.F[0][0] == -f.F[1][0] && f.F[0][0] > 0.0 && f.F[0][1] == 0.0 && f.F[0][2] == 0.0);
        s.pos = {{1.0, 1.0, 1.0}, {3.5, 1.0, 1.0}};
        f = esp::local_sum(plan, s);
        CHECK(f.u[0] == 0.0 && f.u[1] == 0.0 && f.F[0][0] == 0.0);
        s.pos = {{0.1, 5.0, 5.0}, {9.8, 5.0, 5.0}};
        f = esp::local_sum(plan, s);
        CHECK(f.u[0] != 0.0 && f.F[0][0] < 0.0 && f.F[0][0] == -f.F[1][0]);
    }
    // contracts (test_ewald.cpp:364-381)
    {
        esp::EwaldPlan plan = esp::build_plan(box, esp::SplitFamily::pswf, 1e-3, 1.0);
        esp::ParticleSystem wrong = random_system(8, {8.0, 8.0, 8.0}, 1);
        CHECK(throws<std::invalid_argument>([&] { esp::evaluate(plan, wrong); }));
        esp::ParticleSystem charged = random_system(8, box, 1);
        charged.q[0] = 2.0;
        CHECK(throws<esp::NumericalError>([&] { esp::evaluate(plan, charged); }));
        esp::EnergyForces ef = esp::evaluate(plan, random_system(8, box, 1));
        CHECK(ef.timings.size() == 6);
        CHECK(ef.timings.at("local") > 0.0 && ef.timings.at("interpolate") > 0.0);
        CHECK(ef.device_timings.at("total") > 0.0);
        // spectral_sum fills the caller's map with the grid-pipeline stages
        std::map<std::string, double> sp;
        esp::spectral_sum(plan, random_system(8, box, 1), &sp);
        CHECK(sp.size() == 5 && sp.at("fft") > 0.0);
    }
    // translation invariance (test_ewald.cpp:383-409)
    {
        const double eps = 1e-4;
        esp::EwaldPlan plan = esp::build_plan(box, esp::SplitFamily::pswf, eps, 1.0);
        esp::ParticleSystem s = random_system(64, box, 21);
        esp::EnergyForces a = esp::evaluate(plan, s);
        esp::ParticleSystem t = s;
        for (auto& r : t.pos) {
            r[0] += 0.37;
            r[1] += -1.2;
            r[2] += 2.05;
        }
        esp::EnergyForces b = esp::evaluate(plan, t);
        double fs = 0, us = 0, df = 0, du = 0;
        for (std::size_t i = 0; i < s.size(); ++i) {
            us = std::max(us, std::fabs(a.u[i]));
            du = std::max(du, std::fabs(a.u[i] - b.u[i]));
            for (int d = 0; d < 3; ++d) {
                fs = std::max(fs, std::fabs(a.F[i][d]));
                df = std::max(df, std::fabs(a.F[i][d] - b.F[i][d]));
            }
        }
        CHECK(du <= 10 * eps * us && df <= 10 * eps * fs);
        CHECK(std::fabs(a.energy - b.energy) <= 10 * eps * std::fabs(a.energy));
    }
    // charge scaling (test_ewald.cpp:411-438), bitwise gate -> 1e-14
    {
        esp::EwaldPlan plan = esp::build_plan(box, esp::SplitFamily::pswf, 1e-3, 1.0);
        esp::ParticleSystem s = random_system(32, box, 29);
        esp::EnergyForces a = esp::evaluate(plan, s);
        for (auto& q : s.q) q *= 2.0;
        esp::EnergyForces b = esp::evaluate(plan, s);
        double worst = 0, scale = 0;
        for (std::size_t i = 0; i < s.size(); ++i) {
            scale = std::max(scale, std::fabs(a.u[i]));
            worst = std::max(worst, std::fabs(b.u[i] - 2.0 * a.u[i]));
        }
        CHECK(worst <= 1e-14 * 2.0 * scale);
        CHECK(std::fabs(b.energy - 4.0 * a.energy) <= 1e-13 * std::fabs(4.0 * a.energy));
    }
    // ik vs ad (test_ewald.cpp:340-351)
    {
        esp::ParticleSystem s = random_system(100, box, 23);
        esp::Overrides ik, ad;
        ad.force_method = esp::ForceMethod::ad;
        esp::EnergyForces a = esp::evaluate(esp::build_plan(box, esp::SplitFamily::pswf, 1e-3, 1.0, ik), s);
        esp::EnergyForces b = esp::evaluate(esp::build_plan(box, esp::SplitFamily::pswf, 1e-3, 1.0, ad), s);
        CHECK(esp::relative_force_error(b.F, a.F) <= 10 * 1e-3);
        CHECK(std::fabs(a.energy - b.energy) <= 1e-13 * std::fabs(a.energy));
    }
    // net force (test_ewald.cpp:463-476)
    {
        esp::EwaldPlan plan = esp::build_plan(box, esp::SplitFamily::pswf, 1e-4, 1.0);
        esp::EnergyForces ef = esp::evaluate(plan, random_system(128, box, 41));
        for (int d = 0; d < 3; ++d) {
            double net = 0, mag = 0;
            for (auto& F : ef.F) {
                net += F[d];
                mag += std::fabs(F[d]);
            }
            CHECK(std::fabs(net) <= 1e-8 * mag);
        }
    }
    // Madelung (test_ewald.cpp:493-508)
    {
        esp::ParticleSystem s;
        s.box = {2.0, 2.0, 2.0};
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j)
                for (int k = 0; k < 2; ++k) {
                    s.pos.push_back({1.0 * i, 1.0 * j, 1.0 * k});
                    s.q.push_back((i + j + k) % 2 == 0 ? 1.0 : -1.0);
                }
        esp::EnergyForces ef = esp::evaluate(esp::build_plan(s.box, esp::SplitFamily::pswf, 1e-5, 0.5), s);
        const double expect = -1.7475645946331822 / M_PI;
        CHECK(std::fabs(ef.energy - expect) <= 1e-4 * std::fabs(expect));
        double fs = 0;
        for (auto& F : ef.F)
            for (double c : F) fs = std::max(fs, std::fabs(c));
        CHECK(fs <= 1e-6);
    }
    // plan metadata (test_ewald.cpp:510-516)
    {
        esp::EwaldPlan plan = esp::build_plan(box, esp::SplitFamily::pswf, 1e-4, 1.0);
        CHECK(plan.total_modes() == 40ull * 40ull * 40ull);
        CHECK(std::fabs(plan.avg_neighbors(512) - 4.0 * M_PI / 3.0 * 512.0 / 1000.0) <= 1e-12);
        CHECK(plan.influence()[0] == 0.0);
    }
    // kernel objects, parameter selection, influence (kernels.hpp, ewald.hpp:338)
    {
        esp::EwaldPlan plan = esp::build_plan(box, esp::SplitFamily::pswf, 1e-4, 1.0);
        CHECK(std::fabs(plan.split.Psi(0.0)) <= 1e-14);
        CHECK(std::fabs(plan.split.Psi(1.0) - 1.0) <= 1e-12);
        CHECK(std::fabs(plan.split.chi(0.0) - plan.split.chi0) <= 1e-12 * plan.split.chi0);
        CHECK(plan.win[1].P == plan.P && plan.win[2].dim == 2);
        CHECK(plan.win[0].phi(0.0) > 0.0 && plan.win[0].phi(plan.win[0].half) == 0.0);
        esp::SelectResult sel = esp::select_parameters(esp::SplitFamily::pswf, 1e-4, box, 1.0);
        CHECK(sel.nf == plan.nf && sel.P == plan.P && sel.c1 == plan.c1);
        std::vector<double> a = plan.influence();
        std::vector<double> b = esp::influence_coefficients(plan.split, plan.win, plan.nf, box);
        CHECK(a == b);
        CHECK(throws<std::invalid_argument>(
            [&] { esp::influence_coefficients(plan.split, plan.win, {32, 32, 32}, box); }));
    }
    // spread / interpolate adjointness and the gradient (gridder.hpp:215-314,
    // test_gridder.cpp)
    {
        esp::EwaldPlan plan = esp::build_plan(box, esp::SplitFamily::pswf, 1e-4, 1.0);
        esp::ParticleSystem s = random_system(64, box, 5);
        esp::GridArray g = esp::spread(s, plan.win, plan.nf);
        esp::GridArray f = esp::GridArray::zeros(plan.nf);
        std::uint64_t st = 99;
        for (auto& c : f.v) {
            st = st * 6364136223846793005ull + 1442695040888963407ull;
            c = {static_cast<double>(st >> 11) * 0x1.0p-53 - 0.5, 0.0};
        }
        double lhs = 0.0, rhs = 0.0;
        for (std::size_t i = 0; i < g.v.size(); ++i) lhs += g.v[i].real() * f.v[i].real();
        std::vector<double> u = esp::interpolate(f, plan.win, s);
        for (std::size_t i = 0; i < u.size(); ++i) rhs += s.q[i] * u[i];
        CHECK(std::fabs(lhs - rhs) <= 1e-12 * std::fabs(lhs));
        std::vector<esp::Vec3> gr = esp::interpolate_gradient(f, plan.win, s);
        // central difference of interpolate along x for atom 0
        esp::ParticleSystem sp = s, sm = s;
        const double dx = 1e-5;
        sp.pos[0][0] += dx;
        sm.pos[0][0] -= dx;
        const double fd = (esp::interpolate(f, plan.win, sp)[0] - esp::interpolate(f, plan.win, sm)[0]) / (2 * dx);
        CHECK(std::fabs(fd - gr[0][0]) <= 1e-5 * (1.0 + std::fabs(gr[0][0])));
    }
    // FFT conventions (gridder.hpp:6-13, 85-100): inverse(forward(g)) = N g
    {
        esp::GridArray g = esp::GridArray::zeros({6, 10, 15});
        std::uint64_t st = 7;
        for (auto& c : g.v) {
            st = st * 6364136223846793005ull + 1442695040888963407ull;
            c = {static_cast<double>(st >> 11) * 0x1.0p-53, static_cast<double>(st >> 40) * 0x1.0p-24};
        }
        esp::GridArray h = g;
        esp::fft_forward(h);
        // mode (1, 0, 0) against a direct sum with e^{-i}
        std::complex<double> m{0.0, 0.0};
        for (int ix = 0; ix < 6; ++ix)
            for (int iy = 0; iy < 10; ++iy)
                for (int iz = 0; iz < 15; ++iz)
                    m += g.v[g.idx(ix, iy, iz)] * std::polar(1.0, -2.0 * M_PI * ix / 6.0);
        CHECK(std::abs(h.v[h.idx(1, 0, 0)] - m) <= 1e-12 * std::abs(m));
        esp::fft_inverse(h);
        double err = 0.0;
        for (std::size_t i = 0; i < g.v.size(); ++i)
            err = std::max(err, std::abs(h.v[i] / 900.0 - g.v[i]));
        CHECK(err <= 1e-13);
    }
    // direct Ewald (reference.hpp:212-238) against the ESP evaluation: Delta <= eps
    {
        esp::ParticleSystem s = random_system(200, box, 77);
        esp::ReferenceResult d = esp::direct_ewald(s, 1e-9);
        esp::EnergyForces ef = esp::evaluate(esp::build_plan(box, esp::SplitFamily::pswf, 1e-4, 1.0), s);
        CHECK(esp::relative_force_error(ef.F, d.F) <= 1e-4);
        CHECK(std::fabs(ef.energy - d.energy) <= 1e-4 * std::fabs(d.energy));
        CHECK(d.real_shells >= 1 && d.recip_kmax >= 1 && d.lambda > 0.0);
    }
    // evaluate() sharded over 2 and 3 ranks (esp::Shard, emulation members on
    // this GPU): each rank holds only its own atoms; equal to the
    // single-process evaluation up to summation order
    {
        const esp::Vec3 bx{24.0, 20.0, 22.0};
        esp::ParticleSystem s = random_system(4000, bx, 5);
        esp::EwaldPlan whole = esp::build_plan(bx, esp::SplitFamily::pswf, 1e-4, 2.0);
        esp::EnergyForces ref = esp::evaluate(whole, s, false);
        for (int G : {2, 3}) {
            std::vector<esp::EwaldPlan> plans;
            for (int r = 0; r < G; ++r) plans.push_back(esp::build_plan(bx, esp::SplitFamily::pswf, 1e-4, 2.0));
            const std::vector<int> own = esp::Shard::owner(plans[0], G, s.pos);
            std::vector<esp::ParticleSystem> parts(G);
            std::vector<std::vector<std::size_t>> idx(G);
            for (int r = 0; r < G; ++r) parts[r].box = bx;
            for (std::size_t i = 0; i < s.size(); ++i) {
                parts[own[i]].pos.push_back(s.pos[i]);
                parts[own[i]].q.push_back(s.q[i]);
                idx[own[i]].push_back(i);
            }
            long nmax = 0;
            for (auto& p : parts) nmax = std::max(nmax, static_cast<long>(p.size()));
            std::vector<std::unique_ptr<esp::Shard>> sh;
            std::vector<esp::Shard*> raw;
            for (int r = 0; r < G; ++r) {
                sh.emplace_back(new esp::Shard(plans[r], nullptr, r, G, nmax));
                raw.push_back(sh.back().get());
            }
            const std::vector<esp::EnergyForces> out = esp::Shard::evaluate_emulated(raw, parts);
            std::vector<esp::Vec3> F(s.size());
            double du = 0.0, umax = 0.0;
            for (int r = 0; r < G; ++r)
                for (std::size_t k = 0; k < idx[r].size(); ++k) {
                    F[idx[r][k]] = out[r].F[k];
                    du = std::max(du, std::fabs(out[r].u[k] - ref.u[idx[r][k]]));
                    umax = std::max(umax, std::fabs(ref.u[idx[r][k]]));
                }
            CHECK(std::fabs(out[0].energy - ref.energy) <= 1e-12 * std::fabs(ref.energy));
            CHECK(esp::relative_force_error(F, ref.F) <= 1e-12);
            CHECK(du <= 1e-12 * umax);
            CHECK(raw[0]->info().nranks == G && raw[0]->info().nccl == 0);
        }
        // an atom passed to the wrong rank is reported (esp_shard_check flags)
        esp::EwaldPlan p0 = esp::build_plan(bx, esp::SplitFamily::pswf, 1e-4, 2.0);
        esp::EwaldPlan p1 = esp::build_plan(bx, esp::SplitFamily::pswf, 1e-4, 2.0);
        esp::Shard a(p0, nullptr, 0, 2, 10), b(p1, nullptr, 1, 2, 10);
        esp::ParticleSystem s0, s1;
        s0.box = s1.box = bx;
        s0.pos = {{22.0, 1.0, 1.0}, {1.0, 2.0, 3.0}};   // the first atom is rank 1's
        s0.q = {1.0, -1.0};
        s1.pos = {{13.0, 5.0, 5.0}};
        s1.q = {0.0};
        CHECK(throws<std::invalid_argument>([&] { esp::Shard::evaluate_emulated({&a, &b}, {s0, s1}); }));
    }
    std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "PASSED", failures);
    return failures ? 1 : 0;
}
