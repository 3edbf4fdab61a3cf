// Host-side plan construction for the B200 ESP solver.
//
// A from-scratch restatement of the reference's plan-time mathematics
// (/root/reference/proj/include/esp: prolate.hpp, kernels.hpp, ewald.hpp
// :110-405, gridder.hpp:162-210).  It produces exactly the discretisation
// the reference selects (n_f, P, c1) and the coefficient tables the GPU
// kernels consume:
//   * split kernel Psi / chi on [0,1]: 16 uniform segments, degree-12
//     polynomials in the local coordinate t in [-1,1] (monomial form for
//     Horner on the device);
//   * spreading window phi / phi' per dimension: 4P uniform segments of
//     width h/4 on [-Ph/2, Ph/2], same representation;
//   * influence multipliers p_k on the D2Z half spectrum nx*ny*(nz/2+1).
// Nothing here touches the GPU.
#pragma once

#include <array>
#include <memory>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace espb {

// Error classes mirrored from the reference (std::invalid_argument,
// esp::NumericalError prolate.hpp:17-20).  They never cross the C ABI.
struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct NumericalError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// psi_0^c as an even-Legendre series, psi(0) = 1 (prolate.hpp:26-35).
struct Prolate {
    double c = 0.0;
    std::vector<double> a;  // psi(x) = sum_k a[k] P_{2k}(x)
    double C0 = 0.0;        // int_0^1 psi = a[0]
    double psi1 = 0.0;      // psi(1)
    double l2 = 0.0;        // ||psi||_{L2[-1,1]}
};

Prolate build_prolate(double c);
double solve_c(double eps);                                 // prolate.hpp:254-263
double prolate_cos(const std::vector<double>& a, double nu);  // prolate.hpp:77-87
int next_even_5smooth(double x);                            // numerics.hpp:289-293
int signed_mode(int i, int n);                              // gridder.hpp:76

// Degree-12 polynomial pieces on uniform segments; poly[s*13 + k] multiplies
// t^k with t = 2*(x - a_s)/(b_s - a_s) - 1.
struct PiecewisePoly {
    double lo = 0.0, hi = 1.0;
    int nseg = 0;
    std::vector<double> mono;  // nseg x 13 monomial coefficients in t
    std::vector<double> cheb;  // nseg x 13 Chebyshev-T coefficients (diagnostic)
    double eval(double x) const;
};

enum class Family : int { pswf = 0, gaussian = 1 };
enum class ForceMethod : int { ik = 0, ad = 1 };

struct Overrides {  // ewald.hpp:38-47
    int nf = 0;
    int P = 0;
    double c1 = 0.0;
    ForceMethod force_method = ForceMethod::ik;
    bool allow_degraded = false;
};

struct Plan {
    Family family = Family::pswf;
    ForceMethod force_method = ForceMethod::ik;
    double eps = 0.0, r_c = 0.0;
    std::array<double, 3> box{};
    std::array<int, 3> nf{}, base_nf{};
    std::array<double, 3> demand{}, h{};
    int P = 0;
    double shape = 0.0;  // split bandwidth c
    double c1 = 0.0;     // window bandwidth
    double chi0 = 0.0;   // chi(0) = 1/C0
    double self_coef = 0.0;  // chi0 / (4 pi r_c)
    double E_A = 0.0, E_T = 0.0, E_SI = 0.0;

    Prolate split;                       // bandwidth c
    Prolate window;                      // bandwidth c1
    PiecewisePoly Psi, chi;              // on [0,1], 16 segments
    std::array<PiecewisePoly, 3> phi, dphi;  // on [-half, half], 4P segments
    std::array<double, 3> half{};        // P h / 2
    std::vector<double> influence_half;  // nx * ny * (nz/2+1)
    // Pair-kernel form of the split (device K4): Psi(y) = y * H(z) with
    // z = 2 y^2 - 1 on y in [0,1], H a monomial polynomial in z, and
    // chi(y) = H + 2 (z+1) dH/dz (so one coefficient stream serves both).
    // For the PSWF split Psi(y)/y is an exact polynomial of degree
    // K = nterms-1 in y^2 (kernels.hpp:105-138); the degree is reduced to the
    // smallest meeting 2e-15 on Psi and 2e-14 (relative) on chi.  The
    // monomial form is well conditioned in z (sum |coef| ~ 3).
    std::vector<double> pair_G, pair_H;  // pair_G unused (kept empty)
    double pair_fit_err = 0.0;  // max deviation from the exact kernels

    // Host-side evaluators (used for validation and by the C ABI getters).
    double Psi_at(double y) const;     // kernels.hpp:76-81
    double chi_at(double y) const;     // kernels.hpp:90-95
    double chihat_n(double nu) const;  // kernels.hpp:97-100
    double phi_at(int d, double x) const;
    double dphi_at(int d, double x) const;
    double phi_hat(int d, double xi) const;  // kernels.hpp:219-229
    std::pair<double, double> local_kernel(double r) const;  // kernels.hpp:143-163
};

// Optional device backend for the O(n_f^3) plan tables (SURVEY 8(f) row 3:
// gridder.hpp:162-210, ewald.hpp:110-143): the chihat octant that feeds the
// aliasing estimate E_A of every grid-inflation step, and the influence half
// spectrum.  The E_A sums themselves stay on the host in long double so that
// the plan choices (n_f, c1) are those of the host path.
struct PlanDevice {
    virtual ~PlanDevice() = default;
    // val[(ax * h1 + ay) * h2 + az] = chihat_n(r_c |xi|), xi^2 = (f2[0][ax] +
    // f2[1][ay]) + f2[2][az], h_d = nf_d / 2 + 1 (0 at xi = 0)
    virtual void octant(const Plan& p, const std::array<std::vector<double>, 3>& f2,
                        std::vector<double>& val) = 0;
    // influence_half from the last octant: pref * chihat / xi^2 / (phihat_x^2
    // phihat_y^2 phihat_z^2) on the half spectrum (storage-index tables)
    virtual void influence(const Plan& p, const std::array<std::vector<double>, 3>& ph2,
                           const std::array<std::vector<double>, 3>& fr2, double pref,
                           std::vector<double>& out) = 0;
};

Plan build_plan(const std::array<double, 3>& box, Family family, double eps, double r_c,
                const Overrides& ov, PlanDevice* dev = nullptr);

// CUDA implementation of PlanDevice on one device (plan_device.cu).
std::unique_ptr<PlanDevice> make_plan_device(int device);

// Full nx*ny*nz influence array (reference layout), expanded from the half
// spectrum; used only for parity checks.
std::vector<double> influence_full(const Plan& p);

}  // namespace espb
