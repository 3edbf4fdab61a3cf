// esp/esp.hpp -- drop-in C++ interface of the B200 ESP solver.
//
// Mirrors the reference's public API (namespace esp, header-only C++20 in
// /root/reference/proj/include/esp; README.md:58-64) for the force-evaluation
// path, implemented on the C ABI of libesp_b200.so (include/esp_b200.h):
//
//   EwaldPlan plan = esp::build_plan(box, esp::SplitFamily::pswf, eps, r_c);
//   EnergyForces ef = esp::evaluate(plan, system);        // runs on the GPU
//
// Same types, argument meanings and exceptions as the reference:
//   std::invalid_argument  where the reference throws it (bad eps/box/r_c,
//                          odd pinned n_f, P out of range, box mismatch);
//   esp::NumericalError    plans refused by the error model, non-neutral
//                          systems, window underflow;
//   esp::CudaError         (new) CUDA/cuFFT failure or no GPU -- there is no
//                          CPU fallback.
// Also mirrored: SplitKernel / WindowKernel (plan.split, plan.win with
// their evaluators), GridArray, spread / interpolate / interpolate_gradient,
// influence_coefficients, fft_forward / fft_inverse, select_parameters /
// SelectResult, direct_ewald / ReferenceResult -- all executed on the GPU.
// Differences (documented in INTEGRATION.md): results are not bitwise
// reproducible run to run (GPU atomics); EwaldPlan::influence is a method
// returning the full n_f^3 array on demand; thread_count() is accepted and
// ignored; set_device() picks the CUDA device for subsequent plans;
// direct_ewald has no N <= 1e4 cap.
//
// Link: -L<repo>/paper_2505_09727_b200 -lesp_b200 -Wl,-rpath,<that dir>
#pragma once

#include "../esp_b200.h"

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <complex>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace esp {

using Vec3 = std::array<double, 3>;

class NumericalError : public std::runtime_error {  // prolate.hpp:17-20
public:
    explicit NumericalError(const std::string& w) : std::runtime_error(w) {}
};
class CudaError : public std::runtime_error {
public:
    explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};

enum class SplitFamily { pswf, gaussian };   // kernels.hpp:19
enum class WindowFamily { pswf, bspline };
enum class ForceMethod { ik, ad };           // ewald.hpp:28

inline const char* to_string(SplitFamily f) { return f == SplitFamily::pswf ? "pswf" : "gaussian"; }
inline const char* to_string(ForceMethod m) { return m == ForceMethod::ik ? "ik" : "ad"; }

struct Overrides {  // ewald.hpp:38-47
    int nf = 0;
    int P = 0;
    double c1 = 0.0;
    ForceMethod force_method = ForceMethod::ik;
    bool allow_degraded = false;
};

struct PlanStats {  // ewald.hpp:61-65
    double E_A = 0.0, E_T = 0.0, E_SI = 0.0;
};

struct ParticleSystem {  // system.hpp:19-26
    Vec3 box{0.0, 0.0, 0.0};
    std::vector<double> q;
    std::vector<Vec3> pos;
    std::size_t size() const { return q.size(); }
    double volume() const { return box[0] * box[1] * box[2]; }
};

struct EnergyForces {  // system.hpp:49-55
    double energy = 0.0;
    std::vector<double> u;
    std::vector<Vec3> F;
    std::map<std::string, double> timings;
    // GPU-only stage times (not in the reference's struct): "bin", "total"
    std::map<std::string, double> device_timings;
};

struct PartialField {  // ewald.hpp:411-414
    std::vector<double> u;
    std::vector<Vec3> F;
};

namespace detail {

inline void check(int rc) {
    if (rc == ESP_OK) return;
    const std::string msg = esp_last_error();
    if (rc == ESP_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (rc == ESP_ERR_NUMERICAL) throw NumericalError(msg);
    if (rc == ESP_ERR_CUDA || rc == ESP_ERR_NO_DEVICE) throw CudaError(msg);
    throw std::runtime_error(msg);
}

inline int& device_slot() {
    static int d = 0;
    return d;
}

struct Handle {
    esp_plan* p = nullptr;
    std::mutex m;  // a C-ABI handle is not re-entrant
    ~Handle() { esp_plan_destroy(p); }
};

inline const double* flat(const std::vector<Vec3>& v) {
    return v.empty() ? nullptr : v[0].data();
}
inline double* flat(std::vector<Vec3>& v) { return v.empty() ? nullptr : v[0].data(); }

}  // namespace detail

// CUDA device for plans built afterwards (-1: host-only plans).
inline void set_device(int device) { detail::device_slot() = device; }
// Accepted for source compatibility (threads.hpp:14-17); the GPU path has no
// host thread pool.
inline int& thread_count() {
    static int n = 1;
    return n;
}

// Split and window kernels of a plan (kernels.hpp:63-229): the parameters of
// the reference's structs plus evaluators backed by the plan's tables.
struct SplitKernel {  // kernels.hpp:63-101
    SplitFamily family = SplitFamily::pswf;
    double eps = 0.0, shape = 0.0, r_c = 0.0, chi0 = 0.0;
    double Psi(double y) const { return eval(0, y); }
    double chi(double y) const { return eval(1, y); }
    double chihat_n(double k) const { return eval(2, k); }
    std::shared_ptr<detail::Handle> plan;

private:
    double eval(int what, double x) const {
        double y = 0.0;
        detail::check(esp_plan_eval_kernel(plan->p, what, 1, &x, &y));
        return y;
    }
};

struct WindowKernel {  // kernels.hpp:178-229
    WindowFamily family = WindowFamily::pswf;
    int P = 0;
    double h = 0.0;
    double c1 = std::numeric_limits<double>::quiet_NaN();
    double half = 0.0;  // P h / 2
    int dim = 0;        // which grid dimension of the plan
    double phi(double x) const { return eval(8 + dim, x); }
    double dphi(double x) const { return eval(11 + dim, x); }
    double phi_hat(double xi) const { return eval(14 + dim, xi); }
    std::shared_ptr<detail::Handle> plan;

private:
    double eval(int what, double x) const {
        double y = 0.0;
        detail::check(esp_plan_eval_kernel(plan->p, what, 1, &x, &y));
        return y;
    }
};

// gridder.hpp:59-72: complex128 row-major grid, z fastest
struct GridArray {
    std::array<int, 3> nf{0, 0, 0};
    std::vector<std::complex<double>> v;
    static GridArray zeros(std::array<int, 3> nf) {
        GridArray g;
        g.nf = nf;
        g.v.assign(static_cast<std::size_t>(nf[0]) * nf[1] * nf[2], {0.0, 0.0});
        return g;
    }
    std::size_t idx(int ix, int iy, int iz) const {
        return (static_cast<std::size_t>(ix) * nf[1] + iy) * nf[2] + iz;
    }
};

class EwaldPlan {  // ewald.hpp:67-94
public:
    SplitFamily family = SplitFamily::pswf;
    WindowFamily window_family = WindowFamily::pswf;
    double eps = 0.0;
    double r_c = 0.0;
    Vec3 box{};
    std::array<int, 3> nf{}, base_nf{};
    std::array<double, 3> demand{};
    std::array<double, 3> h{};
    int P = 0;
    double shape = 0.0;
    double c1 = std::numeric_limits<double>::quiet_NaN();
    ForceMethod force_method = ForceMethod::ik;
    SplitKernel split;
    std::array<WindowKernel, 3> win;
    PlanStats stats;

    std::size_t total_modes() const { return static_cast<std::size_t>(nf[0]) * nf[1] * nf[2]; }
    double avg_neighbors(std::size_t N) const {
        return (4.0 / 3.0) * M_PI * r_c * r_c * r_c * static_cast<double>(N) /
               (box[0] * box[1] * box[2]);
    }
    // influence coefficients p_k, full n_f^3 layout (gridder.hpp:162-210)
    std::vector<double> influence() const {
        std::vector<double> out(total_modes());
        detail::check(esp_plan_get_influence(h_->p, out.data()));
        return out;
    }
    esp_plan* handle() const { return h_->p; }
    std::mutex& mutex() const { return h_->m; }

private:
    std::shared_ptr<detail::Handle> h_;
    friend EwaldPlan build_plan(const Vec3&, SplitFamily, double, double, const Overrides&);
};

// ewald.hpp:355-405
inline EwaldPlan build_plan(const Vec3& box, SplitFamily family, double eps, double r_c,
                            const Overrides& ov = {}) {
    esp_overrides o{ov.nf, ov.P, ov.c1, ov.force_method == ForceMethod::ad ? ESP_FORCE_AD
                                                                           : ESP_FORCE_IK,
                    ov.allow_degraded ? 1 : 0};
    auto h = std::make_shared<detail::Handle>();
    detail::check(esp_plan_create(box.data(),
                                  family == SplitFamily::gaussian ? ESP_FAMILY_GAUSSIAN
                                                                  : ESP_FAMILY_PSWF,
                                  eps, r_c, &o, detail::device_slot(), &h->p));
    esp_plan_info info{};
    detail::check(esp_plan_get_info(h->p, &info));
    EwaldPlan plan;
    plan.h_ = h;
    plan.family = family;
    plan.window_family = family == SplitFamily::pswf ? WindowFamily::pswf : WindowFamily::bspline;
    plan.eps = info.eps;
    plan.r_c = info.r_c;
    for (int d = 0; d < 3; ++d) {
        plan.box[d] = info.box[d];
        plan.nf[d] = info.nf[d];
        plan.base_nf[d] = info.base_nf[d];
        plan.demand[d] = info.demand[d];
        plan.h[d] = info.h[d];
    }
    plan.P = info.P;
    plan.shape = info.shape;
    plan.c1 = info.c1;
    plan.force_method = ov.force_method;
    plan.stats = {info.E_A, info.E_T, info.E_SI};
    plan.split.family = family;
    plan.split.eps = info.eps;
    plan.split.shape = info.shape;
    plan.split.r_c = info.r_c;
    plan.split.chi0 = info.chi0;
    plan.split.plan = h;
    for (int d = 0; d < 3; ++d) {
        WindowKernel& w = plan.win[d];
        w.family = plan.window_family;
        w.P = info.P;
        w.h = info.h[d];
        w.c1 = info.c1;
        w.half = 0.5 * info.P * info.h[d];
        w.dim = d;
        w.plan = h;
    }
    return plan;
}

// ewald.hpp:49-59, 338-350: the parameter selection alone (a host-only plan)
struct SelectResult {
    SplitFamily family = SplitFamily::pswf;
    double shape = 0.0;
    int P = 0;
    double c1 = std::numeric_limits<double>::quiet_NaN();
    std::array<double, 3> demand{};
    std::array<int, 3> base_nf{};
    std::array<int, 3> nf{};
    double E_A = 0.0;
    double E_SI = 0.0;
};

inline SelectResult select_parameters(SplitFamily family, double eps, const Vec3& box,
                                      double r_c, const Overrides& ov = {}) {
    esp_overrides o{ov.nf, ov.P, ov.c1, ov.force_method == ForceMethod::ad ? ESP_FORCE_AD
                                                                           : ESP_FORCE_IK,
                    ov.allow_degraded ? 1 : 0};
    detail::Handle h;
    detail::check(esp_plan_create(box.data(),
                                  family == SplitFamily::gaussian ? ESP_FAMILY_GAUSSIAN
                                                                  : ESP_FAMILY_PSWF,
                                  eps, r_c, &o, -1, &h.p));
    esp_plan_info info{};
    detail::check(esp_plan_get_info(h.p, &info));
    SelectResult r;
    r.family = family;
    r.shape = info.shape;
    r.P = info.P;
    r.c1 = info.c1;
    for (int d = 0; d < 3; ++d) {
        r.demand[d] = info.demand[d];
        r.base_nf[d] = info.base_nf[d];
        r.nf[d] = info.nf[d];
    }
    r.E_A = info.E_A;
    r.E_SI = info.E_SI;
    return r;
}

// system.hpp:29-36
inline void fold(ParticleSystem& s) {
    for (auto& p : s.pos)
        for (int d = 0; d < 3; ++d) {
            const double L = s.box[d];
            p[d] -= L * std::floor(p[d] / L);
            if (p[d] >= L) p[d] = 0.0;
        }
}

// Deterministic mode of a plan (esp_plan_set_deterministic): bitwise
// reproducible evaluations, like the reference for any thread count
// (README.md:87-94); slower.
inline void set_deterministic(const EwaldPlan& plan, bool on) {
    std::lock_guard<std::mutex> lk(plan.mutex());
    detail::check(esp_plan_set_deterministic(plan.handle(), on ? 1 : 0));
}

// system.hpp:39-47
inline void require_neutral(const ParticleSystem& s) {
    detail::check(esp_check_neutral(static_cast<long>(s.size()), s.q.data()));
}

// ewald.hpp:619-649 (GPU).  Like the reference, `timings` holds the per-stage
// wall times (seconds) under exactly its keys {local, spread, fft, scale,
// ifft, interpolate}: CUDA events around each stage, the stages serialised on
// one stream as the reference runs them.  GPU-only times go to
// `device_timings` ("bin": fold, cell keys and sorts; "total": host wall time
// of the call).  stage_timings = false selects the overlapped CUDA-graph path
// (real-space sum concurrent with the grid pipeline); the six keys are then
// 0 and only device_timings["total"] is measured.
inline EnergyForces evaluate(const EwaldPlan& plan, const ParticleSystem& s,
                             bool stage_timings = true) {
    const long N = static_cast<long>(s.size());
    if (s.pos.size() != s.q.size()) throw std::invalid_argument("evaluate: pos/q length mismatch");
    EnergyForces out;
    out.u.resize(N);
    out.F.resize(N);
    esp_timings t{};
    const auto t0 = std::chrono::steady_clock::now();
    {
        std::lock_guard<std::mutex> lk(plan.mutex());
        detail::check(esp_evaluate(plan.handle(), s.box.data(), N, detail::flat(s.pos),
                                   s.q.data(), out.u.data(), detail::flat(out.F), &out.energy,
                                   stage_timings ? &t : nullptr));
    }
    out.timings["local"] = t.local;
    out.timings["spread"] = t.spread;
    out.timings["fft"] = t.fft;
    out.timings["scale"] = t.scale;
    out.timings["ifft"] = t.ifft;
    out.timings["interpolate"] = t.interpolate;
    out.device_timings["bin"] = t.bin;
    out.device_timings["total"] =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return out;
}

// ewald.hpp:419-515
inline PartialField local_sum(const EwaldPlan& plan, const ParticleSystem& s) {
    PartialField f;
    f.u.resize(s.size());
    f.F.resize(s.size());
    std::lock_guard<std::mutex> lk(plan.mutex());
    detail::check(esp_local_sum(plan.handle(), s.box.data(), static_cast<long>(s.size()),
                                detail::flat(s.pos), s.q.data(), f.u.data(), detail::flat(f.F)));
    return f;
}

// ewald.hpp:524-604
inline PartialField spectral_sum(const EwaldPlan& plan, const ParticleSystem& s,
                                 std::map<std::string, double>* timings = nullptr) {
    PartialField f;
    f.u.resize(s.size());
    f.F.resize(s.size());
    esp_timings t{};
    std::lock_guard<std::mutex> lk(plan.mutex());
    detail::check(esp_spectral_sum(plan.handle(), s.box.data(), static_cast<long>(s.size()),
                                   detail::flat(s.pos), s.q.data(), f.u.data(),
                                   detail::flat(f.F), timings ? &t : nullptr));
    if (timings) {  // the reference adds its tick() times into the caller's map
        (*timings)["spread"] += t.spread;
        (*timings)["fft"] += t.fft;
        (*timings)["scale"] += t.scale;
        (*timings)["ifft"] += t.ifft;
        (*timings)["interpolate"] += t.interpolate;
    }
    return f;
}

// ewald.hpp:609-615
inline std::vector<double> self_correction(const EwaldPlan& plan, const std::vector<double>& q) {
    std::vector<double> out(q.size());
    detail::check(esp_self_correction(plan.handle(), static_cast<long>(q.size()), q.data(),
                                      out.data()));
    return out;
}

namespace detail {
inline esp_plan* window_plan(const std::array<WindowKernel, 3>& win,
                             const std::array<int, 3>& nf) {
    if (!win[0].plan) throw std::invalid_argument("window kernels do not belong to a plan");
    esp_plan_info info{};
    check(esp_plan_get_info(win[0].plan->p, &info));
    for (int d = 0; d < 3; ++d)
        if (info.nf[d] != nf[d])  // gridder.hpp:141-148
            throw std::invalid_argument("grid size does not match the window kernels' plan");
    return win[0].plan->p;
}
inline std::vector<double> positions(const ParticleSystem& s) {
    std::vector<double> p(3 * s.size());
    for (std::size_t i = 0; i < s.size(); ++i)
        for (int d = 0; d < 3; ++d) p[3 * i + d] = s.pos[i][d];
    return p;
}
}  // namespace detail

// gridder.hpp:215-241 (GPU; the imaginary part is zero)
inline GridArray spread(const ParticleSystem& s, const std::array<WindowKernel, 3>& win,
                        const std::array<int, 3>& nf) {
    esp_plan* p = detail::window_plan(win, nf);
    std::vector<double> re(static_cast<std::size_t>(nf[0]) * nf[1] * nf[2]);
    const std::vector<double> pos = detail::positions(s);
    std::lock_guard<std::mutex> lk(win[0].plan->m);
    detail::check(esp_spread(p, static_cast<long>(s.size()), pos.data(), s.q.data(), re.data()));
    GridArray g = GridArray::zeros(nf);
    for (std::size_t i = 0; i < re.size(); ++i) g.v[i] = {re[i], 0.0};
    return g;
}

// gridder.hpp:244-277 (the real part of the grid)
inline std::vector<double> interpolate(const GridArray& g, const std::array<WindowKernel, 3>& win,
                                       const ParticleSystem& s) {
    esp_plan* p = detail::window_plan(win, g.nf);
    std::vector<double> re(g.v.size()), out(s.size());
    for (std::size_t i = 0; i < re.size(); ++i) re[i] = g.v[i].real();
    const std::vector<double> pos = detail::positions(s);
    std::lock_guard<std::mutex> lk(win[0].plan->m);
    detail::check(esp_interpolate(p, static_cast<long>(s.size()), pos.data(), re.data(),
                                  out.data()));
    return out;
}

// gridder.hpp:280-314
inline std::vector<Vec3> interpolate_gradient(const GridArray& g,
                                              const std::array<WindowKernel, 3>& win,
                                              const ParticleSystem& s) {
    esp_plan* p = detail::window_plan(win, g.nf);
    std::vector<double> re(g.v.size());
    std::vector<Vec3> out(s.size());
    for (std::size_t i = 0; i < re.size(); ++i) re[i] = g.v[i].real();
    const std::vector<double> pos = detail::positions(s);
    std::lock_guard<std::mutex> lk(win[0].plan->m);
    detail::check(esp_interpolate_gradient(p, static_cast<long>(s.size()), pos.data(), re.data(),
                                           detail::flat(out)));
    return out;
}

// gridder.hpp:162-210 (the plan's coefficients; full nf^3 layout)
inline std::vector<double> influence_coefficients(const SplitKernel& split,
                                                  const std::array<WindowKernel, 3>& win,
                                                  const std::array<int, 3>& nf, const Vec3& box) {
    esp_plan* p = detail::window_plan(win, nf);
    if (split.plan.get() != win[0].plan.get())
        throw std::invalid_argument("split and window kernels come from different plans");
    esp_plan_info info{};
    detail::check(esp_plan_get_info(p, &info));
    for (int d = 0; d < 3; ++d)
        if (info.box[d] != box[d]) throw std::invalid_argument("box does not match the plan");
    std::vector<double> out(static_cast<std::size_t>(nf[0]) * nf[1] * nf[2]);
    detail::check(esp_plan_get_influence(p, out.data()));
    return out;
}

// gridder.hpp:153-154: unnormalised forward (e^{-i}) / inverse (e^{+i}) on the GPU
inline void fft_forward(GridArray& g) {
    detail::check(esp_fft3(g.nf.data(), reinterpret_cast<double*>(g.v.data()), -1,
                           detail::device_slot()));
}
inline void fft_inverse(GridArray& g) {
    detail::check(esp_fft3(g.nf.data(), reinterpret_cast<double*>(g.v.data()), 1,
                           detail::device_slot()));
}

// reference.hpp:21-29
struct ReferenceResult {
    std::vector<double> u;
    std::vector<Vec3> F;
    double energy = 0.0;
    double lambda = 0.0;
    int real_shells = 0;
    int recip_kmax = 0;
    double residual = 0.0;
};

// reference.hpp:212-238 on the GPU: a pass at lambda = min(L)/6 plus the
// 1.3 lambda invariance pass.  Difference: no N <= 1e4 cap.
inline ReferenceResult direct_ewald(const ParticleSystem& system, double tol) {
    const long N = static_cast<long>(system.size());
    const std::vector<double> pos = detail::positions(system);
    ReferenceResult r;
    r.u.resize(N);
    r.F.resize(N);
    esp_direct_info i1{}, i2{};
    double e2 = 0.0;
    const double lam = std::min({system.box[0], system.box[1], system.box[2]}) / 6.0;
    detail::check(esp_direct_ewald(system.box.data(), N, pos.data(), system.q.data(), 0, nullptr,
                                   tol, lam, r.u.data(), detail::flat(r.F), &r.energy, &i1,
                                   detail::device_slot()));
    std::vector<double> u2(N), F2(3 * N);
    detail::check(esp_direct_ewald(system.box.data(), N, pos.data(), system.q.data(), 0, nullptr,
                                   tol, 1.3 * lam, u2.data(), F2.data(), &e2, &i2,
                                   detail::device_slot()));
    const double gap = std::fabs(r.energy - e2);
    if (gap > tol * std::max(1.0, std::fabs(r.energy)))
        throw NumericalError("direct_ewald: splitting-width invariance check failed");
    r.lambda = i1.lambda;
    r.real_shells = i1.real_shells;
    r.recip_kmax = i1.recip_kmax;
    r.residual = std::max(gap, i1.tail_bound);
    return r;
}

// ---- evaluate() sharded over the GPUs of one box (esp_shard_*) ------------
// One process per GPU; every rank builds its own plan (same arguments, its own
// device via set_device) and a Shard on it.  Rank 0's unique_id() is shared
// with the other ranks by the caller (MPI, a file, ...).  Each rank passes only
// the atoms it owns (owner(), the x-slab decomposition by grid plane) and gets
// back their u and F and the TOTAL energy; the ghost, halo, transpose and
// reduction traffic is NCCL inside the library.  Same results as
// evaluate(plan, whole system) up to summation order.
class Shard {
public:
    using Id = std::array<unsigned char, 128>;
    static Id unique_id() {
        Id id{};
        detail::check(esp_shard_unique_id(id.data()));
        return id;
    }
    // owner rank of every atom (any image)
    static std::vector<int> owner(const EwaldPlan& plan, int nranks, const std::vector<Vec3>& pos) {
        std::vector<int> o(pos.size());
        detail::check(esp_shard_owner(plan.handle(), nranks, static_cast<long>(pos.size()),
                                      detail::flat(pos), o.data()));
        return o;
    }
    // collective over nranks processes (id != nullptr), or an emulation
    // member (id == nullptr) for evaluate_emulated below
    Shard(const EwaldPlan& plan, const Id* id, int rank, int nranks, long max_own_atoms,
          long ghost_capacity = 0)
        : plan_(plan) {
        detail::check(esp_shard_create(plan.handle(), id ? id->data() : nullptr, rank, nranks,
                                       max_own_atoms, ghost_capacity, &h_));
    }
    ~Shard() { esp_shard_destroy(h_); }
    Shard(const Shard&) = delete;
    Shard& operator=(const Shard&) = delete;

    // this rank's atoms (host; collective: every rank calls it for the step)
    EnergyForces evaluate(const ParticleSystem& own) {
        EnergyForces out;
        const long n = static_cast<long>(own.size());
        if (own.pos.size() != own.q.size())
            throw std::invalid_argument("evaluate: pos/q length mismatch");
        out.u.resize(n);
        out.F.resize(n);
        std::lock_guard<std::mutex> lk(plan_.mutex());
        detail::check(esp_shard_evaluate_host(h_, own.box.data(), n, detail::flat(own.pos),
                                              own.q.data(), out.u.data(), detail::flat(out.F),
                                              &out.energy));
        return out;
    }
    // device pointers, asynchronous on `stream` (graph-capturable)
    void evaluate_device(const Vec3& box, long n_own, const double* pos, const double* q,
                         double* u, double* F, double* energy, void* stream) {
        detail::check(esp_shard_evaluate(h_, box.data(), n_own, pos, q, u, F, energy, stream));
    }
    void check() { detail::check(esp_shard_check(h_)); }
    esp_shard_info_t info() const {
        esp_shard_info_t i{};
        detail::check(esp_shard_info(h_, &i));
        return i;
    }
    esp_shard* handle() const { return h_; }

    // all ranks of one decomposition in this process on one GPU (emulation
    // members, messages moved by device copies): tests and single-GPU runs
    static std::vector<EnergyForces> evaluate_emulated(std::vector<Shard*> shards,
                                                       const std::vector<ParticleSystem>& own) {
        const int G = static_cast<int>(shards.size());
        if (static_cast<int>(own.size()) != G) throw std::invalid_argument("one system per shard");
        std::vector<esp_shard*> hs(G);
        std::vector<long> n(G);
        std::vector<const double*> P(G), Q(G);
        std::vector<double*> U(G), F(G);
        std::vector<EnergyForces> out(G);
        for (int r = 0; r < G; ++r) {
            hs[r] = shards[r]->h_;
            n[r] = static_cast<long>(own[r].size());
            out[r].u.resize(n[r]);
            out[r].F.resize(n[r]);
            P[r] = detail::flat(own[r].pos);
            Q[r] = own[r].q.data();
            U[r] = out[r].u.data();
            F[r] = detail::flat(out[r].F);
        }
        double e = 0.0;
        detail::check(esp_shard_evaluate_emulated_host(hs.data(), G, own[0].box.data(), n.data(),
                                                       P.data(), Q.data(), U.data(), F.data(),
                                                       &e));
        for (auto& o : out) o.energy = e;
        return out;
    }

private:
    const EwaldPlan& plan_;
    esp_shard* h_ = nullptr;
};

// reference.hpp:241-255
inline double relative_force_error(const std::vector<Vec3>& test, const std::vector<Vec3>& ref) {
    if (test.size() != ref.size())
        throw std::invalid_argument("relative_force_error: length mismatch");
    double num = 0.0, den = 0.0;
    for (std::size_t i = 0; i < ref.size(); ++i)
        for (int d = 0; d < 3; ++d) {
            const double e = test[i][d] - ref[i][d];
            num += e * e;
            den += ref[i][d] * ref[i][d];
        }
    if (den <= 0.0) throw std::invalid_argument("relative_force_error: zero reference norm");
    return std::sqrt(num / den);
}

}  // namespace esp
