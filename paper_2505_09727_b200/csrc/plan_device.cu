// Device construction of the O(n_f^3) plan tables.
//
// The host plan (plan.cpp) spends its time in two grid-sized loops: the
// octant of chihat_n(r_c |xi|) over (|kx|, |ky|, |kz|), rebuilt at every
// grid-inflation step of the parameter selection (ewald.hpp:110-143, 293-328:
// the aliasing estimate E_A sums |chihat| / xi^2 over it), and the influence
// multipliers on the half spectrum (gridder.hpp:162-210).  Both are
// embarrassingly parallel; here they run as two kernels.  chihat_n restates
// the host path exactly: for the PSWF split the cosine transform of the
// prolate ground state, sum_k (-1)^k a_k j_2k(nu) / C0 with the spherical
// Bessel functions from Miller's downward recurrence (numerics.hpp:174-203,
// prolate.hpp:77-87) summed in the same order; for the Gaussian split
// exp(-nu^2 / (4 alpha)).  Results agree with the host tables to a few ulp
// (device sin / cos / exp), so the plan choices are unchanged
// (tests/test_gpu_plan_device.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "engine.hpp"  // CudaError
#include "plan.hpp"

namespace espb {
namespace {

#define PCK(x)                                                                          \
    do {                                                                                \
        cudaError_t e_ = (x);                                                           \
        if (e_ != cudaSuccess)                                                          \
            throw CudaError(std::string("CUDA error: ") + cudaGetErrorString(e_) +      \
                            " at " __FILE__ ":" + std::to_string(__LINE__));            \
    } while (0)

constexpr int kMaxTerms = 96;  // prolate expansion terms held per thread (j_0..j_2(K))

// prolate_cos(a, nu) of plan.cpp: sum_k (-1)^k a_k j_{2k}(nu) with j_n from
// sph_bessel_all (Miller's downward recurrence, rescaled against overflow,
// normalised by the exact j_0 or j_1).
__device__ double prolate_cos_dev(const double* __restrict__ a, int na, double nu) {
    double js[2 * kMaxTerms + 1];
    const int nmax = 2 * (na - 1);
    const double x = fabs(nu);
    for (int n = 0; n <= nmax; ++n) js[n] = 0.0;
    if (x < 1e-10) {
        js[0] = 1.0;
        if (nmax >= 1) js[1] = x / 3.0;
    } else {
        const double s = sin(x), c = cos(x);
        const double j0 = s / x;
        const double j1 = s / (x * x) - c / x;
        const int start = max(nmax, static_cast<int>(ceil(x))) + 40;
        double hi = 0.0, cur = 1e-300;
        for (int k = start; k >= 1; --k) {
            const double lo = (2.0 * k + 1.0) / x * cur - hi;
            hi = cur;
            cur = lo;
            if (k - 1 <= nmax) js[k - 1] = cur;
            if (fabs(cur) > 1e250) {
                cur *= 1e-250;
                hi *= 1e-250;
                for (int n = 0; n <= nmax; ++n) js[n] *= 1e-250;
            }
        }
        const double scale = (fabs(j0) >= fabs(j1) || nmax < 1) ? j0 / js[0] : j1 / js[1];
        for (int n = 0; n <= nmax; ++n) {
            js[n] *= scale;
            if (!isfinite(js[n])) js[n] = 0.0;
        }
    }
    double sum = 0.0;
    for (int k = 0; k < na; ++k) sum += (k & 1) ? -a[k] * js[2 * k] : a[k] * js[2 * k];
    return sum;
}

struct OctArgs {
    int h[3];
    const double* f2[3];
    const double* a;  // split prolate coefficients (PSWF)
    int na;
    double C0;
    double r_c;
    double alpha;  // Gaussian shape
    int gauss;
    double* val;
};

__global__ void __launch_bounds__(128) k_octant(OctArgs g) {
    const long n = static_cast<long>(g.h[0]) * g.h[1] * g.h[2];
    const long t = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
    if (t >= n) return;
    const int az = static_cast<int>(t % g.h[2]);
    const int ay = static_cast<int>((t / g.h[2]) % g.h[1]);
    const int ax = static_cast<int>(t / (static_cast<long>(g.h[1]) * g.h[2]));
    const double xi2 = (g.f2[0][ax] + g.f2[1][ay]) + g.f2[2][az];
    double v = 0.0;
    if (xi2 != 0.0) {
        const double nu = g.r_c * sqrt(xi2);
        v = g.gauss ? exp(-nu * nu / (4.0 * g.alpha)) : prolate_cos_dev(g.a, g.na, nu) / g.C0;
    }
    g.val[t] = v;
}

struct InflArgs {
    int nf[3];
    int h[3];  // octant extents
    const double* oct;
    const double* ph2[3];
    const double* fr2[3];
    double pref;
    double* out;  // nx * ny * (nz/2 + 1)
};

__device__ __forceinline__ int absmode(int i, int n) { return i < (n + 1) / 2 ? i : n - i; }

__global__ void __launch_bounds__(256) k_influence(InflArgs g) {
    const int nzh = g.nf[2] / 2 + 1;
    const long n = static_cast<long>(g.nf[0]) * g.nf[1] * nzh;
    const long t = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
    if (t >= n) return;
    const int iz = static_cast<int>(t % nzh);
    const int iy = static_cast<int>((t / nzh) % g.nf[1]);
    const int ix = static_cast<int>(t / (static_cast<long>(nzh) * g.nf[1]));
    // same operation order as plan.cpp (xy first, then the z term)
    const double xy = g.fr2[0][ix] + g.fr2[1][iy];
    const double wxy = g.ph2[0][ix] * g.ph2[1][iy];
    const double xi2 = xy + g.fr2[2][iz];
    double v = 0.0;
    if (xi2 != 0.0) {
        const int ax = absmode(ix, g.nf[0]), ay = absmode(iy, g.nf[1]), az = absmode(iz, g.nf[2]);
        const double G = g.oct[(static_cast<long>(ax) * g.h[1] + ay) * g.h[2] + az] / xi2;
        v = g.pref * G / (wxy * g.ph2[2][iz]);
    }
    g.out[t] = v;
}

class CudaPlanDevice final : public PlanDevice {
public:
    explicit CudaPlanDevice(int device) : device_(device) {}
    ~CudaPlanDevice() override {
        for (double* p : bufs_)
            if (p) cudaFree(p);
        if (d_oct_) cudaFree(d_oct_);
    }

    void octant(const Plan& p, const std::array<std::vector<double>, 3>& f2,
                std::vector<double>& val) override {
        PCK(cudaSetDevice(device_));
        OctArgs g{};
        long n = 1;
        for (int d = 0; d < 3; ++d) {
            g.h[d] = static_cast<int>(f2[d].size());
            n *= g.h[d];
            g.f2[d] = upload(d, f2[d]);
        }
        const bool gauss = p.family == Family::gaussian;
        g.gauss = gauss ? 1 : 0;
        g.alpha = p.shape;
        g.r_c = p.r_c;
        if (!gauss) {
            if (static_cast<int>(p.split.a.size()) > kMaxTerms)
                throw NumericalError("device plan: prolate expansion longer than supported");
            g.a = upload(3, p.split.a);
            g.na = static_cast<int>(p.split.a.size());
            g.C0 = p.split.C0;
        }
        if (n > oct_cap_) {
            if (d_oct_) cudaFree(d_oct_);
            d_oct_ = nullptr;
            PCK(cudaMalloc(&d_oct_, sizeof(double) * n));
            oct_cap_ = n;
        }
        g.val = d_oct_;
        for (int d = 0; d < 3; ++d) oct_h_[d] = g.h[d];
        k_octant<<<static_cast<unsigned>((n + 127) / 128), 128>>>(g);
        PCK(cudaGetLastError());
        val.resize(n);
        PCK(cudaMemcpy(val.data(), d_oct_, sizeof(double) * n, cudaMemcpyDeviceToHost));
    }

    void influence(const Plan& p, const std::array<std::vector<double>, 3>& ph2,
                   const std::array<std::vector<double>, 3>& fr2, double pref,
                   std::vector<double>& out) override {
        PCK(cudaSetDevice(device_));
        InflArgs g{};
        for (int d = 0; d < 3; ++d) {
            g.nf[d] = p.nf[d];
            g.h[d] = oct_h_[d];
            if (oct_h_[d] != p.nf[d] / 2 + 1)
                throw NumericalError("device plan: octant does not match the final grid");
            g.ph2[d] = upload(4 + d, ph2[d]);
            g.fr2[d] = upload(7 + d, fr2[d]);
        }
        g.oct = d_oct_;
        g.pref = pref;
        const long n = static_cast<long>(p.nf[0]) * p.nf[1] * (p.nf[2] / 2 + 1);
        double* d_out = nullptr;
        PCK(cudaMalloc(&d_out, sizeof(double) * n));
        g.out = d_out;
        k_influence<<<static_cast<unsigned>((n + 255) / 256), 256>>>(g);
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess) {
            out.resize(n);
            e = cudaMemcpy(out.data(), d_out, sizeof(double) * n, cudaMemcpyDeviceToHost);
        }
        cudaFree(d_out);
        PCK(e);
    }

private:
    // small per-slot device copies of the 1-D tables
    const double* upload(int slot, const std::vector<double>& v) {
        if (static_cast<long>(v.size()) > caps_[slot]) {
            if (bufs_[slot]) cudaFree(bufs_[slot]);
            bufs_[slot] = nullptr;
            PCK(cudaMalloc(&bufs_[slot], sizeof(double) * std::max<size_t>(v.size(), 1)));
            caps_[slot] = static_cast<long>(v.size());
        }
        PCK(cudaMemcpy(bufs_[slot], v.data(), sizeof(double) * v.size(), cudaMemcpyHostToDevice));
        return bufs_[slot];
    }

    int device_;
    double* bufs_[10] = {};
    long caps_[10] = {};
    double* d_oct_ = nullptr;
    long oct_cap_ = 0;
    int oct_h_[3] = {};
};

}  // namespace

std::unique_ptr<PlanDevice> make_plan_device(int device) {
    return std::make_unique<CudaPlanDevice>(device);
}

}  // namespace espb
