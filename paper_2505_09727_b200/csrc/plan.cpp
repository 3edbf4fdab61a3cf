// Host plan construction (see plan.hpp).  Every function names the reference
// routine whose mathematics it restates (file:line under
// /root/reference/proj/include/esp).  The algorithms are re-derived rather
// than transcribed: the ground state of the prolate operator is found by
// Sturm bisection + inverse iteration (the reference uses implicit QL), the
// bandwidth root by a bracketed secant/bisection hybrid polished to machine
// precision, and the spectral sums exploit the octant symmetry of the
// mode set.  Results agree with the reference to roundoff; the discrete
// choices (n_f, P, c1) are identical.

#include "plan.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <limits>
#include <thread>

namespace espb {

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr int kDeg = 12;          // polynomial degree of every table piece
constexpr int kNc = kDeg + 1;     // coefficients per piece
constexpr int kSplitSegs = 16;    // kernels.hpp:130-136

// ----------------------------------------------------------------------------
// Legendre sums
// ----------------------------------------------------------------------------

// sum_k a[k] P_{2k}(x) and its x-derivative (prolate.hpp:41-59 computes the
// same quantities).
void even_legendre(const std::vector<double>& a, double x, double* val, double* der) {
    double p_prev = 1.0, p = x;   // P_0, P_1
    double d_prev = 0.0, d = 1.0; // P'_0, P'_1
    double v = a[0], dv = 0.0;
    const int top = 2 * (static_cast<int>(a.size()) - 1);
    for (int n = 1; n < top; ++n) {
        double pn = ((2 * n + 1) * x * p - n * p_prev) / (n + 1);
        double dn = d_prev + (2 * n + 1) * p;
        p_prev = p;
        p = pn;
        d_prev = d;
        d = dn;
        if (((n + 1) & 1) == 0) {
            v += a[(n + 1) / 2] * p;
            dv += a[(n + 1) / 2] * d;
        }
    }
    *val = v;
    if (der) *der = dv;
}

// int_0^y sum_k a[k] P_{2k}(t) dt via int_0^y P_n = (P_{n+1} - P_{n-1})/(2n+1)
// (kernels.hpp:122-128).
double even_legendre_integral(const std::vector<double>& a, double y) {
    // walk P_0..P_{2K+1}
    const int K = static_cast<int>(a.size()) - 1;
    double acc = 0.0;
    double pm = 1.0, p = y;  // P_0, P_1
    // contribution of a[k] needs P_{2k-1} and P_{2k+1}
    std::vector<double> P(2 * K + 2);
    P[0] = 1.0;
    if (2 * K + 1 >= 1) P[1] = y;
    for (int n = 1; n + 1 < static_cast<int>(P.size()); ++n) {
        double pn = ((2 * n + 1) * y * p - n * pm) / (n + 1);
        pm = p;
        p = pn;
        P[n + 1] = pn;
    }
    for (int k = 0; k <= K; ++k) {
        int n = 2 * k;
        double lo = n >= 1 ? P[n - 1] : 0.0;
        acc += a[k] * (P[n + 1] - lo) / (2.0 * n + 1.0);
    }
    return acc;
}

// Extended-precision versions for the pair-kernel fit (the polynomial and its
// derivative must be accurate to ~1e-17 before rounding to double).
long double even_legendre_ld(const std::vector<double>& a, long double x) {
    long double pm = 1.0L, p = x, v = a[0];
    const int top = 2 * (static_cast<int>(a.size()) - 1);
    for (int n = 1; n < top; ++n) {
        long double pn = ((2 * n + 1) * x * p - n * pm) / (n + 1);
        pm = p;
        p = pn;
        if (((n + 1) & 1) == 0) v += a[(n + 1) / 2] * p;
    }
    return v;
}

long double even_legendre_integral_ld(const std::vector<double>& a, long double y) {
    const int K = static_cast<int>(a.size()) - 1;
    std::vector<long double> P(2 * K + 2);
    P[0] = 1.0L;
    P[1] = y;
    for (int n = 1; n + 1 < static_cast<int>(P.size()); ++n)
        P[n + 1] = ((2 * n + 1) * y * P[n] - n * P[n - 1]) / (n + 1);
    long double acc = 0.0L;
    for (int k = 0; k <= K; ++k) {
        const int n = 2 * k;
        acc += a[k] * (P[n + 1] - (n >= 1 ? P[n - 1] : 0.0L)) / (2.0L * n + 1.0L);
    }
    return acc;
}

// ----------------------------------------------------------------------------
// Spherical Bessel j_0..j_nmax by Miller's downward recurrence
// (restates numerics.hpp:174-203).
// ----------------------------------------------------------------------------
void sph_bessel_all(int nmax, double x, double* js) {
    x = std::fabs(x);
    for (int n = 0; n <= nmax; ++n) js[n] = 0.0;
    if (x < 1e-10) {
        js[0] = 1.0;
        if (nmax >= 1) js[1] = x / 3.0;
        return;
    }
    const double s = std::sin(x), c = std::cos(x);
    const double j0 = s / x;
    const double j1 = s / (x * x) - c / x;
    const int start = std::max(nmax, static_cast<int>(std::ceil(x))) + 40;
    double hi = 0.0, cur = 1e-300;
    for (int k = start; k >= 1; --k) {
        double lo = (2.0 * k + 1.0) / x * cur - hi;  // order k-1
        hi = cur;
        cur = lo;
        if (k - 1 <= nmax) js[k - 1] = cur;
        if (std::fabs(cur) > 1e250) {
            cur *= 1e-250;
            hi *= 1e-250;
            for (int n = 0; n <= nmax; ++n) js[n] *= 1e-250;
        }
    }
    double scale = (std::fabs(j0) >= std::fabs(j1) || nmax < 1) ? j0 / js[0] : j1 / js[1];
    for (int n = 0; n <= nmax; ++n) {
        js[n] *= scale;
        if (!std::isfinite(js[n])) js[n] = 0.0;
    }
}

// ----------------------------------------------------------------------------
// Lowest eigenpair of a symmetric tridiagonal matrix
// ----------------------------------------------------------------------------

// Number of eigenvalues < x (Sturm count from the LDL^T pivots).
int sturm_count(const std::vector<double>& d, const std::vector<double>& e, double x) {
    int cnt = 0;
    double q = d[0] - x;
    if (q < 0) ++cnt;
    for (std::size_t i = 1; i < d.size(); ++i) {
        if (q == 0.0) q = 1e-300;
        q = d[i] - x - e[i - 1] * e[i - 1] / q;
        if (q < 0) ++cnt;
    }
    return cnt;
}

// (T - s I) y = b with partial pivoting; T tridiagonal (diag d, off e).
std::vector<double> shifted_solve(const std::vector<double>& d, const std::vector<double>& e,
                                  double s, std::vector<double> b) {
    const int n = static_cast<int>(d.size());
    // Row k of the working band: u0 (diag), u1, u2 (fill-in); l (sub)
    std::vector<double> u0(n), u1(n, 0.0), u2(n, 0.0), sub(n, 0.0);
    for (int i = 0; i < n; ++i) {
        u0[i] = d[i] - s;
        if (i + 1 < n) u1[i] = e[i];
        if (i > 0) sub[i] = e[i - 1];
    }
    for (int k = 0; k + 1 < n; ++k) {
        // candidate pivots: u0[k] (row k) and sub[k+1] (row k+1)
        if (std::fabs(sub[k + 1]) > std::fabs(u0[k])) {
            // swap rows k and k+1 (row k+1 has entries sub[k+1], u0[k+1], u1[k+1])
            double r0 = sub[k + 1], r1 = u0[k + 1], r2 = u1[k + 1];
            sub[k + 1] = u0[k];
            u0[k + 1] = u1[k];
            u1[k + 1] = u2[k];
            u0[k] = r0;
            u1[k] = r1;
            u2[k] = r2;
            std::swap(b[k], b[k + 1]);
        }
        if (u0[k] == 0.0) u0[k] = 1e-300;
        double m = sub[k + 1] / u0[k];
        u0[k + 1] -= m * u1[k];
        u1[k + 1] -= m * u2[k];
        b[k + 1] -= m * b[k];
    }
    if (u0[n - 1] == 0.0) u0[n - 1] = 1e-300;
    for (int k = n - 1; k >= 0; --k) {
        double v = b[k];
        if (k + 1 < n) v -= u1[k] * b[k + 1];
        if (k + 2 < n) v -= u2[k] * b[k + 2];
        b[k] = v / u0[k];
    }
    return b;
}

double rayleigh(const std::vector<double>& d, const std::vector<double>& e,
                const std::vector<double>& v) {
    const std::size_t n = d.size();
    double num = 0.0;
    for (std::size_t i = 0; i < n; ++i) {
        double t = d[i] * v[i];
        if (i > 0) t += e[i - 1] * v[i - 1];
        if (i + 1 < n) t += e[i] * v[i + 1];
        num += v[i] * t;
    }
    return num;
}

void normalise(std::vector<double>& v) {
    double s = 0.0;
    for (double x : v) s += x * x;
    s = std::sqrt(s);
    for (double& x : v) x /= s;
}

std::vector<double> ground_state(const std::vector<double>& d, const std::vector<double>& e) {
    const int n = static_cast<int>(d.size());
    // Gershgorin bracket
    double lo = std::numeric_limits<double>::infinity(), hi = -lo;
    for (int i = 0; i < n; ++i) {
        double r = (i > 0 ? std::fabs(e[i - 1]) : 0.0) + (i + 1 < n ? std::fabs(e[i]) : 0.0);
        lo = std::min(lo, d[i] - r);
        hi = std::max(hi, d[i] + r);
    }
    for (int it = 0; it < 200; ++it) {
        double mid = 0.5 * (lo + hi);
        if (mid <= lo || mid >= hi) break;
        if (sturm_count(d, e, mid) >= 1) hi = mid;
        else lo = mid;
    }
    double theta = 0.5 * (lo + hi);
    std::vector<double> v(n, 1.0);
    normalise(v);
    for (int it = 0; it < 3; ++it) {
        v = shifted_solve(d, e, theta, v);
        normalise(v);
    }
    // Rayleigh-quotient-refined inverse iteration (as prolate.hpp:165-180)
    for (int it = 0; it < 2; ++it) {
        theta = rayleigh(d, e, v);
        v = shifted_solve(d, e, theta, v);
        normalise(v);
    }
    return v;
}

// ----------------------------------------------------------------------------
// Chebyshev fit on a segment -> monomial coefficients in t in [-1,1]
// (the fit restates numerics.hpp:235-253; the monomial form is ours).
// ----------------------------------------------------------------------------
void fit_piece(const std::function<double(double)>& f, double a, double b, double* cheb,
               double* mono) {
    double fv[kNc];
    for (int k = 0; k < kNc; ++k) {
        double t = std::cos(kPi * (k + 0.5) / kNc);
        fv[k] = f(0.5 * (a + b) + 0.5 * (b - a) * t);
    }
    for (int j = 0; j < kNc; ++j) {
        double s = 0.0;
        for (int k = 0; k < kNc; ++k) s += fv[k] * std::cos(kPi * j * (k + 0.5) / kNc);
        cheb[j] = 2.0 * s / kNc;
    }
    cheb[0] *= 0.5;
    // T_j(t) in the monomial basis, accumulated in extended precision
    long double Tm[kNc][kNc] = {};
    Tm[0][0] = 1.0L;
    Tm[1][1] = 1.0L;
    for (int j = 2; j < kNc; ++j)
        for (int p = 0; p < kNc; ++p) {
            long double v = -Tm[j - 2][p];
            if (p > 0) v += 2.0L * Tm[j - 1][p - 1];
            Tm[j][p] = v;
        }
    for (int p = 0; p < kNc; ++p) {
        long double s = 0.0L;
        for (int j = 0; j < kNc; ++j) s += static_cast<long double>(cheb[j]) * Tm[j][p];
        mono[p] = static_cast<double>(s);
    }
}

PiecewisePoly fit_uniform(const std::function<double(double)>& f, double lo, double hi,
                          int nseg) {
    PiecewisePoly pp;
    pp.lo = lo;
    pp.hi = hi;
    pp.nseg = nseg;
    pp.mono.assign(static_cast<std::size_t>(nseg) * kNc, 0.0);
    pp.cheb.assign(static_cast<std::size_t>(nseg) * kNc, 0.0);
    for (int s = 0; s < nseg; ++s) {
        double a = lo + (hi - lo) * s / nseg;
        double b = lo + (hi - lo) * (s + 1) / nseg;
        fit_piece(f, a, b, &pp.cheb[static_cast<std::size_t>(s) * kNc],
                  &pp.mono[static_cast<std::size_t>(s) * kNc]);
    }
    return pp;
}

// Cardinal B-spline M_P(v) on [0,P] (restates kernels.hpp:40-55).
double bspline(int P, double v) {
    if (v <= 0.0 || v >= P) return 0.0;
    double m[20] = {};
    int j0 = static_cast<int>(std::floor(v));
    if (j0 >= P) return 0.0;
    m[j0] = 1.0;
    for (int ord = 2; ord <= P; ++ord)
        for (int j = 0; j <= j0; ++j) {
            double u = v - j;
            m[j] = (u * m[j] + (ord - u) * m[j + 1]) / (ord - 1.0);
        }
    return m[0];
}


// Same fit with the samples, transform and basis change in long double.
std::vector<double> fit_z_poly_ld(const std::function<long double(long double)>& f, int deg) {
    const int n = deg + 1;
    const long double pi = 3.141592653589793238462643383279502884L;
    std::vector<long double> fv(n), cheb(n);
    for (int k = 0; k < n; ++k) fv[k] = f(std::cos(pi * (k + 0.5L) / n));
    for (int j = 0; j < n; ++j) {
        long double s = 0.0L;
        for (int k = 0; k < n; ++k) s += fv[k] * std::cos(pi * j * (k + 0.5L) / n);
        cheb[j] = 2.0L * s / n;
    }
    cheb[0] *= 0.5L;
    std::vector<std::vector<long double>> T(n, std::vector<long double>(n, 0.0L));
    T[0][0] = 1.0L;
    if (n > 1) T[1][1] = 1.0L;
    for (int j = 2; j < n; ++j)
        for (int p = 0; p < n; ++p) T[j][p] = (p > 0 ? 2.0L * T[j - 1][p - 1] : 0.0L) - T[j - 2][p];
    std::vector<double> mono(n);
    for (int p = 0; p < n; ++p) {
        long double s = 0.0L;
        for (int j = 0; j < n; ++j) s += cheb[j] * T[j][p];
        mono[p] = static_cast<double>(s);
    }
    return mono;
}

double horner(const std::vector<double>& m, double x) {
    double r = m.back();
    for (int k = static_cast<int>(m.size()) - 2; k >= 0; --k) r = r * x + m[k];
    return r;
}

bool is_5smooth(long n) {
    for (int p : {2, 3, 5})
        while (n % p == 0) n /= p;
    return n == 1;
}

// Default PSWF order by accuracy band (ewald.hpp:206-212).
int default_order(double eps) {
    const double s = 1.0 - 1e-9;
    if (eps >= 5e-4 * s) return 5;
    if (eps >= 1e-4 * s) return 6;
    if (eps >= 5e-5 * s) return 7;
    return 8;
}

// Parallel loop over [0, n) in contiguous chunks.
void par_for(int n, const std::function<void(int, int)>& body) {
    unsigned hw = std::thread::hardware_concurrency();
    int T = static_cast<int>(std::min<unsigned>(hw ? hw : 1, 32));
    if (T < 2 || n < 2 * T) {
        body(0, n);
        return;
    }
    std::vector<std::thread> pool;
    int chunk = (n + T - 1) / T;
    for (int t = 1; t < T; ++t) {
        int b = t * chunk, e = std::min(n, b + chunk);
        if (b < e) pool.emplace_back(body, b, e);
    }
    body(0, std::min(n, chunk));
    for (auto& th : pool) th.join();
}

// Octant cache of chihat_n(r_c |xi|) indexed by (|kx|, |ky|, |kz|).
struct Octant {
    std::array<int, 3> half{};  // nf/2 + 1
    std::vector<double> val;
    std::array<std::vector<double>, 3> f2;  // xi^2 per |k|
    double at(int ax, int ay, int az) const {
        return val[(static_cast<std::size_t>(ax) * half[1] + ay) * half[2] + az];
    }
};

}  // namespace

// ----------------------------------------------------------------------------
// public helpers
// ----------------------------------------------------------------------------

int signed_mode(int i, int n) { return i < (n + 1) / 2 ? i : i - n; }

int next_even_5smooth(double x) {
    long m = std::max<long>(2, static_cast<long>(std::ceil(x - 1e-9)));
    while (!(m % 2 == 0 && is_5smooth(m))) ++m;
    return static_cast<int>(m);
}

double prolate_cos(const std::vector<double>& a, double nu) {
    const int nmax = 2 * (static_cast<int>(a.size()) - 1);
    double js[1300];
    sph_bessel_all(nmax, nu, js);
    double s = 0.0;
    for (std::size_t k = 0; k < a.size(); ++k) s += (k & 1) ? -a[k] * js[2 * k] : a[k] * js[2 * k];
    return s;
}

double PiecewisePoly::eval(double x) const {
    double w = (hi - lo) / nseg;
    int s = static_cast<int>((x - lo) / w);
    s = std::clamp(s, 0, nseg - 1);
    double a = lo + (hi - lo) * s / nseg;
    double b = lo + (hi - lo) * (s + 1) / nseg;
    double t = (2.0 * x - a - b) / (b - a);
    const double* m = &mono[static_cast<std::size_t>(s) * kNc];
    double r = m[kDeg];
    for (int k = kDeg - 1; k >= 0; --k) r = r * t + m[k];
    return r;
}

// Ground state of the prolate operator in the even-Legendre basis
// (restates prolate.hpp:137-237: same matrix, same convergence and
// truncation rules, different eigen-solver).
Prolate build_prolate(double c) {
    if (!(c > 0.0)) throw InvalidArgument("build_prolate: c must be positive");
    const double tol = 1e-15;
    int n = 2 * static_cast<int>(std::ceil(c)) + 30;
    std::vector<double> a;
    for (;;) {
        std::vector<double> d(n), e(n - 1);
        const double c2 = c * c;
        for (int k = 0; k < n; ++k) {
            const double m = 2.0 * k;
            double x2 = (m + 1) * (m + 1) / ((2 * m + 1) * (2 * m + 3));
            if (k > 0) x2 += m * m / ((2 * m + 1) * (2 * m - 1));
            d[k] = m * (m + 1) + c2 * x2;
            if (k + 1 < n)
                e[k] = c2 * (2.0 * k + 1) * (2.0 * k + 2)
                       / ((4.0 * k + 3) * std::sqrt((4.0 * k + 1) * (4.0 * k + 5)));
        }
        std::vector<double> v = ground_state(d, e);
        a.assign(n, 0.0);
        double amax = 0.0;
        for (int k = 0; k < n; ++k) {
            a[k] = v[k] * std::sqrt((4.0 * k + 1) / 2.0);
            amax = std::max(amax, std::fabs(a[k]));
        }
        if (std::fabs(a[n - 1]) < tol * amax && std::fabs(a[n - 2]) < tol * amax) break;
        n += 16;
        if (n > 600)
            throw NumericalError("build_prolate: expansion order cap exceeded without "
                                 "trailing-coefficient convergence");
    }
    // psi(0) = sum a_k P_2k(0), P_2k(0) = (-1)^k (2k-1)!!/(2k)!!
    double v0 = 0.0, p0 = 1.0;
    for (std::size_t k = 0; k < a.size(); ++k) {
        if (k > 0) p0 *= -(2.0 * k - 1.0) / (2.0 * k);
        v0 += a[k] * p0;
    }
    for (double& x : a) x /= v0;
    if (a[0] < 0.0)
        for (double& x : a) x = -x;
    double amax = 0.0;
    for (double x : a) amax = std::max(amax, std::fabs(x));
    std::size_t keep = a.size();
    while (keep > 2 && std::fabs(a[keep - 2]) < tol * amax) --keep;
    a.resize(keep);

    Prolate p;
    p.c = c;
    p.a = a;
    p.C0 = a[0];
    double s1 = 0.0, l2 = 0.0;
    for (std::size_t k = 0; k < a.size(); ++k) {
        s1 += a[k];
        l2 += a[k] * a[k] * 2.0 / (4.0 * k + 1.0);
    }
    p.psi1 = s1;
    p.l2 = std::sqrt(l2);
    return p;
}

// Smallest c with psi(1)/||psi||_2 = eps (prolate.hpp:254-263).  Bracketed
// secant/bisection on [2, 28], then polished until the bracket is one ulp.
double solve_c(double eps) {
    if (!(eps >= 1e-8 && eps <= 1e-2))
        throw InvalidArgument("solve_c: eps must lie in [1e-8, 1e-2]");
    auto f = [eps](double c) {
        Prolate p = build_prolate(c);
        return std::log(std::max(p.psi1 / p.l2, 1e-300)) - std::log(eps);
    };
    double a = 2.0, b = 28.0, fa = f(a), fb = f(b);
    if (fa * fb > 0.0) throw NumericalError("solve_c: root not bracketed");
    for (int it = 0; it < 200; ++it) {
        double m;
        if (it % 3 == 2) m = 0.5 * (a + b);            // guarantee shrinkage
        else m = b - fb * (b - a) / (fb - fa);          // false position / secant
        if (!(m > std::min(a, b) && m < std::max(a, b))) m = 0.5 * (a + b);
        double fm = f(m);
        if (fm == 0.0) return m;
        if ((fm < 0) == (fa < 0)) {
            a = m;
            fa = fm;
        } else {
            b = m;
            fb = fm;
        }
        if (std::fabs(b - a) <= 4e-16 * std::fabs(b)) break;
    }
    return std::fabs(fa) < std::fabs(fb) ? a : b;
}

// ----------------------------------------------------------------------------
// Plan evaluators
// ----------------------------------------------------------------------------

double Plan::Psi_at(double y) const {
    if (y <= 0.0) return 0.0;
    if (y >= 1.0) return 1.0;
    return Psi.eval(y);
}
double Plan::chi_at(double y) const {
    if (family == Family::gaussian) return 2.0 * std::sqrt(shape / kPi) * std::exp(-shape * y * y);
    if (y < 0.0 || y > 1.0) return 0.0;
    return chi.eval(y);
}
double Plan::chihat_n(double nu) const {
    if (family == Family::gaussian) return std::exp(-nu * nu / (4.0 * shape));
    return prolate_cos(split.a, nu) / split.C0;
}
double Plan::phi_at(int d, double x) const {
    if (std::fabs(x) >= half[d]) return 0.0;
    return phi[d].eval(x);
}
double Plan::dphi_at(int d, double x) const {
    if (std::fabs(x) >= half[d]) return 0.0;
    return dphi[d].eval(x);
}
double Plan::phi_hat(int d, double xi) const {
    const double nu = std::fabs(xi);
    if (family == Family::gaussian) {
        double t = nu * h[d] / 2.0;
        double s = t == 0.0 ? 1.0 : std::sin(t) / t;
        double out = 1.0;
        for (int i = 0; i < P; ++i) out *= s;
        return out;
    }
    return prolate_cos(window.a, nu * half[d]) / window.C0;
}
std::pair<double, double> Plan::local_kernel(double r) const {
    if (r <= 0.0) throw InvalidArgument("local_kernel: r must be positive");
    if (r >= r_c) return {0.0, 0.0};
    const double inv4pi = 1.0 / (4.0 * kPi);
    double y = r / r_c;
    double one_minus;
    if (family == Family::gaussian) one_minus = std::erfc(std::sqrt(shape) * y);
    else one_minus = 1.0 - Psi_at(y);
    double pot = one_minus * inv4pi / r;
    double fr = pot / r + chi_at(y) * inv4pi / (r * r_c);
    return {pot, fr};
}

// ----------------------------------------------------------------------------
// Plan construction (restates ewald.hpp:236-405 and gridder.hpp:162-210)
// ----------------------------------------------------------------------------

namespace {

Octant build_octant(const Plan& p, const std::array<int, 3>& nf) {
    Octant o;
    for (int d = 0; d < 3; ++d) {
        o.half[d] = nf[d] / 2 + 1;
        o.f2[d].resize(o.half[d]);
        for (int k = 0; k < o.half[d]; ++k) {
            double xi = 2.0 * kPi * k / p.box[d];
            o.f2[d][k] = xi * xi;
        }
    }
    o.val.assign(static_cast<std::size_t>(o.half[0]) * o.half[1] * o.half[2], 0.0);
    par_for(o.half[0], [&](int b, int e) {
        for (int ax = b; ax < e; ++ax)
            for (int ay = 0; ay < o.half[1]; ++ay)
                for (int az = 0; az < o.half[2]; ++az) {
                    double xi2 = (o.f2[0][ax] + o.f2[1][ay]) + o.f2[2][az];
                    o.val[(static_cast<std::size_t>(ax) * o.half[1] + ay) * o.half[2] + az] =
                        xi2 == 0.0 ? 0.0 : p.chihat_n(p.r_c * std::sqrt(xi2));
                }
    });
    return o;
}

// Slab-marginalised spectral weights g = |chihat_n|/|xi|^2 (ewald.hpp:110-143),
// summed with the multiplicity of each |k| value.
struct Slabs {
    std::array<std::vector<double>, 3> slab;  // per storage index i
    double den = 0.0;
};

Slabs alias_slabs(const Octant& o, const std::array<int, 3>& nf) {
    std::array<std::vector<double>, 3> mult;
    for (int d = 0; d < 3; ++d) {
        mult[d].assign(o.half[d], 2.0);
        mult[d][0] = 1.0;
        if (nf[d] % 2 == 0) mult[d][nf[d] / 2] = 1.0;
        if (nf[d] == 1) mult[d][0] = 1.0;
    }
    // per-|k| marginals, long double; the ax range is split into fixed
    // chunks whose partial sums are combined in chunk order (deterministic)
    std::array<std::vector<long double>, 3> marg;
    for (int d = 0; d < 3; ++d) marg[d].assign(o.half[d], 0.0L);
    long double den = 0.0L;
    const int nchunk = std::min(o.half[0], 32);
    std::vector<std::array<std::vector<long double>, 3>> pm(nchunk);
    std::vector<long double> pden(nchunk, 0.0L);
    par_for(nchunk, [&](int cb, int ce) {
        for (int c = cb; c < ce; ++c) {
            auto& m = pm[c];
            for (int d = 0; d < 3; ++d) m[d].assign(o.half[d], 0.0L);
            const int ax0 = static_cast<int>(static_cast<long>(o.half[0]) * c / nchunk);
            const int ax1 = static_cast<int>(static_cast<long>(o.half[0]) * (c + 1) / nchunk);
            long double dsum = 0.0L;
            for (int ax = ax0; ax < ax1; ++ax)
                for (int ay = 0; ay < o.half[1]; ++ay)
                    for (int az = 0; az < o.half[2]; ++az) {
                        double xi2 = (o.f2[0][ax] + o.f2[1][ay]) + o.f2[2][az];
                        if (xi2 == 0.0) continue;
                        long double g = std::fabs(o.at(ax, ay, az)) / xi2;
                        dsum += g * mult[0][ax] * mult[1][ay] * mult[2][az];
                        m[0][ax] += g * mult[1][ay] * mult[2][az];
                        m[1][ay] += g * mult[0][ax] * mult[2][az];
                        m[2][az] += g * mult[0][ax] * mult[1][ay];
                    }
            pden[c] = dsum;
        }
    });
    for (int c = 0; c < nchunk; ++c) {
        den += pden[c];
        for (int d = 0; d < 3; ++d)
            for (int i = 0; i < o.half[d]; ++i) marg[d][i] += pm[c][d][i];
    }
    Slabs s;
    s.den = static_cast<double>(den);
    for (int d = 0; d < 3; ++d) {
        s.slab[d].resize(nf[d]);
        for (int i = 0; i < nf[d]; ++i)
            s.slab[d][i] = static_cast<double>(marg[d][std::abs(signed_mode(i, nf[d]))]);
    }
    return s;
}

// E_A for one window (ewald.hpp:152-158 with pswf_ratio :169-178 or
// bspline_ratio :160-165).
double aliasing(const Slabs& s, const std::array<int, 3>& nf,
                const std::function<double(int, int)>& ratio) {
    long double num = 0.0L;
    for (int d = 0; d < 3; ++d)
        for (int i = 0; i < nf[d]; ++i) num += 2.0L * s.slab[d][i] * ratio(d, i);
    return static_cast<double>(num / s.den);
}

}  // namespace

namespace {
// ESP_PLAN_TIMING=1: stage times of build_plan on stderr (diagnostics)
std::chrono::steady_clock::time_point g_plan_t0;
void plan_stage(const char* name) {
    static const bool on = std::getenv("ESP_PLAN_TIMING") != nullptr;
    if (!on) return;
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "plan %-14s %8.3f ms\n", name,
                 std::chrono::duration<double, std::milli>(t - g_plan_t0).count());
    g_plan_t0 = t;
}
}  // namespace

Plan build_plan(const std::array<double, 3>& box, Family family, double eps, double r_c,
                const Overrides& ov, PlanDevice* dev) {
    g_plan_t0 = std::chrono::steady_clock::now();
    if (!(eps >= 1e-5 && eps <= 1e-3))
        throw InvalidArgument("build_plan: eps out of supported range [1e-5, 1e-3]");
    const double Lmin = std::min({box[0], box[1], box[2]});
    if (!(Lmin > 0.0)) throw InvalidArgument("build_plan: invalid box");
    if (!(r_c > 0.0) || r_c >= Lmin / 2.0)
        throw InvalidArgument("build_plan: require 0 < r_c < min(L)/2");

    Plan p;
    p.family = family;
    p.force_method = ov.force_method;
    p.eps = eps;
    p.r_c = r_c;
    p.box = box;
    const bool gauss = family == Family::gaussian;

    // --- split kernel (kernels.hpp:105-138)
    if (gauss) {
        p.shape = std::log(1.0 / eps);
        p.chi0 = 2.0 * std::sqrt(p.shape / kPi);
        const double sa = std::sqrt(p.shape);
        p.Psi = fit_uniform([sa](double y) { return std::erf(sa * y); }, 0.0, 1.0, kSplitSegs);
        const double alpha = p.shape;
        p.chi = fit_uniform(
            [alpha](double y) { return 2.0 * std::sqrt(alpha / kPi) * std::exp(-alpha * y * y); },
            0.0, 1.0, kSplitSegs);
    } else {
        p.shape = solve_c(eps);
        p.split = build_prolate(p.shape);
        p.chi0 = 1.0 / p.split.C0;
        const Prolate& sp = p.split;
        p.Psi = fit_uniform([&sp](double y) { return even_legendre_integral(sp.a, y) / sp.C0; },
                            0.0, 1.0, kSplitSegs);
        p.chi = fit_uniform(
            [&sp](double y) {
                double v;
                even_legendre(sp.a, y, &v, nullptr);
                return v / sp.C0;
            },
            0.0, 1.0, kSplitSegs);
    }
    p.self_coef = p.chi0 / (4.0 * kPi * r_c);

    plan_stage("split");
    // --- pair-kernel polynomials in z = 2y^2 - 1 (device K4)
    {
        std::function<double(double)> G, H;  // exact chi(y) and Psi(y)/y
        if (gauss) {
            const double alpha = p.shape, sa = std::sqrt(alpha);
            G = [alpha](double y) { return 2.0 * std::sqrt(alpha / kPi) * std::exp(-alpha * y * y); };
            H = [sa, alpha](double y) {
                return y < 1e-8 ? 2.0 * std::sqrt(alpha / kPi) : std::erf(sa * y) / y;
            };
        } else {
            const Prolate& sp = p.split;
            G = [&sp](double y) {
                double v;
                even_legendre(sp.a, y, &v, nullptr);
                return v / sp.C0;
            };
            H = [&sp](double y) {
                if (y < 1e-8) return sp.a.empty() ? 0.0 : 1.0 / sp.C0 * [&] {
                    double v;
                    even_legendre(sp.a, 0.0, &v, nullptr);
                    return v;
                }();
                return even_legendre_integral(sp.a, y) / (sp.C0 * y);
            };
        }
        std::function<long double(long double)> Hld;  // Psi(y)/y in long double
        if (gauss) {
            const long double alpha = p.shape, sa = std::sqrt(alpha);
            Hld = [sa, alpha](long double y) {
                return y < 1e-10L ? 2.0L * std::sqrt(alpha / 3.141592653589793238462643383279502884L)
                                  : std::erf(sa * y) / y;
            };
        } else {
            const Prolate& sp = p.split;
            Hld = [&sp](long double y) {
                if (y < 1e-10L) return even_legendre_ld(sp.a, 0.0L) / sp.C0;
                return even_legendre_integral_ld(sp.a, y) / (sp.C0 * y);
            };
        }
        auto Hzl = [&Hld](long double z) {
            return Hld(std::sqrt(std::max(0.0L, 0.5L * (z + 1.0L))));
        };
        // Only H is tabulated; the kernel recovers chi = dPsi/dy from H and its
        // z-derivative: chi = H + 2 (z + 1) dH/dz (one coefficient stream).
        // Smallest degree meeting 2e-15 on Psi and 2e-14 * max|chi| on chi.
        double gmax = 0.0;
        for (int i = 0; i <= 400; ++i) gmax = std::max(gmax, std::fabs(G(i / 400.0)));
        double fit_psi = 2e-15, fit_chi = 2e-14;
        if (const char* e = std::getenv("ESP_PAIR_FIT")) {  // experiments: scale both targets
            const double f = std::atof(e);
            if (f > 0.0) {
                fit_psi *= f;
                fit_chi *= f;
            }
        }
        for (int deg = 6;; ++deg) {
            p.pair_H = fit_z_poly_ld(Hzl, deg);
            double epsi = 0.0, echi = 0.0;
            for (int i = 0; i <= 2000; ++i) {
                const double y = i / 2000.0, z = 2.0 * y * y - 1.0;
                double hv = p.pair_H.back(), dh = 0.0;
                for (int m = static_cast<int>(p.pair_H.size()) - 2; m >= 0; --m) {
                    dh = dh * z + hv;
                    hv = hv * z + p.pair_H[m];
                }
                epsi = std::max(epsi, std::fabs(y * hv - y * H(y)));
                echi = std::max(echi, std::fabs(hv + 2.0 * (z + 1.0) * dh - G(y)));
            }
            p.pair_fit_err = std::max(epsi, echi / std::max(1.0, gmax));
            if ((epsi <= fit_psi && echi <= fit_chi * std::max(1.0, gmax)) || deg >= 39) break;
        }
        p.pair_G.clear();
    }

    plan_stage("pairpoly");
    // --- parameter selection (ewald.hpp:236-330)
    p.P = ov.P > 0 ? ov.P : (gauss ? 5 : default_order(eps));
    if (p.P < 3 || p.P > 16) throw InvalidArgument("select_parameters: P out of range [3,16]");
    std::array<int, 3> nf{};
    for (int d = 0; d < 3; ++d) {
        if (gauss) {
            double trunc = 2.0 * p.shape * box[d] / (kPi * r_c);
            double si = box[d] * std::sqrt(p.shape) * std::pow(eps, -1.0 / p.P) / (2.0 * r_c);
            p.demand[d] = std::max(trunc, si);
        } else {
            p.demand[d] = p.shape * box[d] / (kPi * r_c);
        }
        if (ov.nf > 0) {
            if (ov.nf % 2 != 0)
                throw InvalidArgument("select_parameters: overridden n_f must be even");
            nf[d] = ov.nf;
        } else if (gauss) {
            nf[d] = next_even_5smooth(2.0 * std::ceil(p.shape * box[d] / (kPi * r_c)));
        } else {
            nf[d] = next_even_5smooth(std::ceil(p.shape * box[d] / (kPi * r_c)));
        }
    }
    p.base_nf = nf;

    std::vector<double> cand;
    std::vector<Prolate> cand_exp;
    if (!gauss) {
        if (ov.c1 > 0.0) cand.push_back(ov.c1);
        else
            for (int i = 0; i < 25; ++i) cand.push_back(p.shape * (1.0 + 0.5 * i / 24));
        cand_exp.resize(cand.size());
        par_for(static_cast<int>(cand.size()), [&](int b, int e) {
            for (int i = b; i < e; ++i) cand_exp[i] = build_prolate(cand[i]);
        });
    }

    plan_stage("prolate-cands");
    Octant oct;
    for (int step = 0;; ++step) {
        if (dev) {
            // the octant on the device: same |k| tables, chihat per point there
            oct.val.clear();
            for (int d = 0; d < 3; ++d) {
                oct.half[d] = nf[d] / 2 + 1;
                oct.f2[d].resize(oct.half[d]);
                for (int k = 0; k < oct.half[d]; ++k) {
                    const double xi = 2.0 * kPi * k / p.box[d];
                    oct.f2[d][k] = xi * xi;
                }
            }
            p.nf = nf;
            dev->octant(p, oct.f2, oct.val);
        } else {
            oct = build_octant(p, nf);
        }
        plan_stage("  octant");
        Slabs sl = alias_slabs(oct, nf);
        plan_stage("  slabs");
        double ea = std::numeric_limits<double>::infinity(), esi = 0.0;
        double c1best = std::numeric_limits<double>::quiet_NaN();
        if (gauss) {
            const int P = p.P;
            ea = aliasing(sl, nf, [&](int d, int i) {
                double k = signed_mode(i, nf[d]);
                return std::pow(std::fabs(k / (k + nf[d])), P);
            });
            double hmax = 0.0;
            for (int d = 0; d < 3; ++d) hmax = std::max(hmax, box[d] / nf[d]);
            esi = std::pow(std::sqrt(p.shape) * hmax / (2.0 * r_c), p.P);
        } else {
            // per-candidate ratio tables, then the scan (first strict minimum wins)
            std::vector<double> eas(cand.size());
            par_for(static_cast<int>(cand.size()), [&](int b, int e) {
                for (int ci = b; ci < e; ++ci) {
                    const Prolate& pe = cand_exp[ci];
                    eas[ci] = aliasing(sl, nf, [&](int d, int i) {
                        double k = signed_mode(i, nf[d]);
                        double lo = kPi * p.P * k / nf[d];
                        double hi = kPi * p.P * (k + nf[d]) / nf[d];
                        return std::fabs(prolate_cos(pe.a, hi) / prolate_cos(pe.a, lo));
                    });
                }
            });
            for (std::size_t ci = 0; ci < cand.size(); ++ci)
                if (eas[ci] < ea) {
                    ea = eas[ci];
                    c1best = cand[ci];
                }
        }
        p.nf = nf;
        p.E_A = ea;
        p.E_SI = esi;
        p.c1 = c1best;
        if (ov.nf > 0) break;
        if (std::max(ea, esi) <= eps) break;
        if (step >= 60)
            throw NumericalError("select_parameters: grid inflation did not reach the "
                                 "accuracy target");
        double hmax = 0.0;
        for (int d = 0; d < 3; ++d) hmax = std::max(hmax, box[d] / nf[d]);
        for (int d = 0; d < 3; ++d)
            if (box[d] / nf[d] >= hmax * (1.0 - 1e-12)) nf[d] = next_even_5smooth(nf[d] + 1.0);
    }

    plan_stage("octant+EA");
    // --- windows (kernels.hpp:234-273), 4P pieces on [-Ph/2, Ph/2]
    if (!gauss) p.window = build_prolate(p.c1);
    for (int d = 0; d < 3; ++d) {
        p.h[d] = box[d] / p.nf[d];
        if (!(p.h[d] > 0.0)) throw InvalidArgument("build_window: h must be positive");
        p.half[d] = p.P * p.h[d] / 2.0;
        const double half = p.half[d], hd = p.h[d];
        const int P = p.P;
        const Prolate& w = p.window;
        std::function<double(double)> f, df;
        if (gauss) {
            f = [P, hd](double x) { return bspline(P, x / hd + P / 2.0) / hd; };
            df = [P, hd](double x) {
                double u = x / hd + P / 2.0;
                return (bspline(P - 1, u) - bspline(P - 1, u - 1.0)) / (hd * hd);
            };
        } else {
            f = [&w, half](double x) {
                double t = x / half;
                if (std::fabs(t) > 1.0) return 0.0;
                double v;
                even_legendre(w.a, t, &v, nullptr);
                return v / (2.0 * half * w.C0);
            };
            df = [&w, half](double x) {
                double t = x / half;
                if (std::fabs(t) > 1.0) return 0.0;
                double v, dv;
                even_legendre(w.a, t, &v, &dv);
                return dv / (2.0 * half * half * w.C0);
            };
        }
        p.phi[d] = fit_uniform(f, -half, half, 4 * P);
        p.dphi[d] = fit_uniform(df, -half, half, 4 * P);
    }

    // --- footprint sanity (ewald.hpp:388-393)
    for (int d = 0; d < 3; ++d)
        if (p.P * p.h[d] / 2.0 > (r_c + p.h[d]) * (1.0 + 1e-9))
            throw NumericalError("build_plan: window footprint exceeds the split "
                                 "support by more than one cell");

    plan_stage("windows");
    // --- error stats (ewald.hpp:194-202, 395-401)
    p.E_T = 0.0;
    for (int d = 0; d < 3; ++d)
        p.E_T = std::max(p.E_T, std::fabs(p.chihat_n(r_c * kPi * p.nf[d] / box[d])));
    if (!ov.allow_degraded && (p.E_A > eps || p.E_T > eps || p.E_SI > eps))
        throw NumericalError("build_plan: grid pinned below the accuracy minimum "
                             "(predicted error exceeds eps)");

    plan_stage("errstats");
    // --- influence multipliers on the half spectrum (gridder.hpp:162-210)
    for (int d = 0; d < 3; ++d) {
        if (p.nf[d] < 2) throw InvalidArgument("grid: n_f must be at least 2");
        if (p.P > p.nf[d]) throw InvalidArgument("grid: window order P exceeds grid size n_f");
    }
    std::array<std::vector<double>, 3> ph2, fr2;  // phihat^2, xi^2 by storage index
    for (int d = 0; d < 3; ++d) {
        ph2[d].resize(p.nf[d]);
        fr2[d].resize(p.nf[d]);
        for (int i = 0; i < p.nf[d]; ++i) {
            int k = signed_mode(i, p.nf[d]);
            double xi = 2.0 * kPi * k / box[d];
            double ph = p.phi_hat(d, xi);
            if (std::fabs(ph) < 1e-30)
                throw NumericalError(
                    "influence: window transform underflow - window too narrow for grid");
            ph2[d][i] = ph * ph;
            fr2[d][i] = xi * xi;
        }
    }
    const double V = box[0] * box[1] * box[2];
    const double hx = p.h[0], hy = p.h[1], hz = p.h[2];
    const double pref = (hx * hy * hz) * (hx * hy * hz) / V;
    const int nx = p.nf[0], ny = p.nf[1], nzh = p.nf[2] / 2 + 1;
    if (dev) {
        dev->influence(p, ph2, fr2, pref, p.influence_half);
        plan_stage("influence(dev)");
        return p;
    }
    p.influence_half.assign(static_cast<std::size_t>(nx) * ny * nzh, 0.0);
    par_for(nx, [&](int b, int e) {
        for (int ix = b; ix < e; ++ix) {
            const int ax = std::abs(signed_mode(ix, nx));
            for (int iy = 0; iy < ny; ++iy) {
                const int ay = std::abs(signed_mode(iy, ny));
                const double xy = fr2[0][ix] + fr2[1][iy];
                const double wxy = ph2[0][ix] * ph2[1][iy];
                double* row = &p.influence_half[(static_cast<std::size_t>(ix) * ny + iy) * nzh];
                for (int iz = 0; iz < nzh; ++iz) {
                    const double xi2 = xy + fr2[2][iz];
                    if (xi2 == 0.0) {
                        row[iz] = 0.0;
                        continue;
                    }
                    const double G = oct.at(ax, ay, std::abs(signed_mode(iz, p.nf[2]))) / xi2;
                    row[iz] = pref * G / (wxy * ph2[2][iz]);
                }
            }
        }
    });
    plan_stage("influence");
    return p;
}

std::vector<double> influence_full(const Plan& p) {
    const int nx = p.nf[0], ny = p.nf[1], nz = p.nf[2], nzh = nz / 2 + 1;
    std::vector<double> out(static_cast<std::size_t>(nx) * ny * nz);
    for (int ix = 0; ix < nx; ++ix)
        for (int iy = 0; iy < ny; ++iy)
            for (int iz = 0; iz < nz; ++iz) {
                int jx = ix, jy = iy, jz = iz;
                if (iz >= nzh) {  // Hermitian partner (-k)
                    jx = (nx - ix) % nx;
                    jy = (ny - iy) % ny;
                    jz = (nz - iz) % nz;
                }
                out[(static_cast<std::size_t>(ix) * ny + iy) * nz + iz] =
                    p.influence_half[(static_cast<std::size_t>(jx) * ny + jy) * nzh + jz];
            }
    return out;
}

}  // namespace espb
