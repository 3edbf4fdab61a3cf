// Direct (mesh-free) Ewald summation on the GPU: the reference's ground-truth
// solver `direct_ewald_pass` (reference.hpp:42-206) restated for one B200,
// for all atoms or for a subset of target atoms (every atom is still a
// source).  It is the checker that certifies the ESP path against Ewald at
// the benchmark sizes, where the reference caps N at 1e4 (reference.hpp:213).
//
// Same mathematics and stopping rules as the reference:
//   real space   max-norm image shells m = 0, 1, ... until a whole shell
//                changes every target potential by < tol/10; pairs with
//                r/lambda > 27 skipped (erfc underflow); j == i skipped in m=0
//   reciprocal   all modes with max-norm 1..kmax, kmax the smallest m whose
//                per-mode bound (sum|q|/V) exp(-lambda^2 xi^2/4)/xi^2 < tol/10;
//                rho(xi) = sum_j q_j e^{-i xi.r_j}
//   self         u_i -= q_i / (2 pi^1.5 lambda)
// Summation order differs from the reference (block reductions, device
// atomics), so results agree to rounding, not bitwise.

#include "direct.hpp"
#include "engine.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

namespace espb {

namespace {

#define DK(x)                                                                         \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess)                                                        \
            throw CudaError(std::string("CUDA error: ") + cudaGetErrorString(e_) +    \
                            " at " __FILE__ ":" + std::to_string(__LINE__));          \
    } while (0)

constexpr double kPiD = 3.14159265358979323846;
constexpr int kDirThreads = 256;
constexpr int kMaxShellOffsets = 33 * 33 * 33;  // shell_cap 16
constexpr int kKzChunk = 16;                    // reciprocal modes per thread pass

template <class T>
struct DevBuf {
    T* p = nullptr;
    explicit DevBuf(size_t n) { DK(cudaMalloc(&p, sizeof(T) * std::max<size_t>(n, 1))); }
    ~DevBuf() { cudaFree(p); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

__device__ __forceinline__ void block_sum4(double v[4], double* red /* 4 x 32 */) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[c] += __shfl_xor_sync(0xffffffffu, v[c], o);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 0)
#pragma unroll
        for (int c = 0; c < 4; ++c) red[c * 32 + w] = v[c];
    __syncthreads();
    if (w == 0) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            double x = lane < nw ? red[c * 32 + lane] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            v[c] = x;
        }
    }
}

// One image shell of the real-space sum (reference.hpp:57-110) for the
// targets: blockIdx.y = target, threads over sources j; (du, F) partial sums
// are added into acc[t] = (du_shell, Fx, Fy, Fz).
__global__ void __launch_bounds__(kDirThreads) k_real_shell(long N, const double4* __restrict__ xyzq,
                                                            const long* __restrict__ tgt,
                                                            const double3* __restrict__ off,
                                                            int noff, int m0, double lambda,
                                                            double* __restrict__ acc) {
    __shared__ double red[4 * 32];
    const long i = tgt[blockIdx.y];
    const double4 pi = xyzq[i];
    const double inv4pi = 1.0 / (4.0 * kPiD);
    const double c2 = 2.0 / (lambda * sqrt(kPiD));
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (long j = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; j < N;
         j += static_cast<long>(gridDim.x) * blockDim.x) {
        const double4 pj = xyzq[j];
        const double dx = pi.x - pj.x, dy = pi.y - pj.y, dz = pi.z - pj.z;
        for (int o = 0; o < noff; ++o) {
            if (m0 && j == i) continue;
            const double3 n = off[o];
            const double rx = dx + n.x, ry = dy + n.y, rz = dz + n.z;
            const double r2 = rx * rx + ry * ry + rz * rz;
            const double r = sqrt(r2);
            const double a = r / lambda;
            if (a > 27.0) continue;
            const double er = erfc(a);
            v[0] += pj.w * er * inv4pi / r;
            const double fp = -(er / r2 + c2 * exp(-a * a) / r) * inv4pi;
            const double coef = -pi.w * pj.w * fp / r;
            v[1] += coef * rx;
            v[2] += coef * ry;
            v[3] += coef * rz;
        }
    }
    block_sum4(v, red);
    if (threadIdx.x == 0)
#pragma unroll
        for (int c = 0; c < 4; ++c) atomicAdd(&acc[4 * blockIdx.y + c], v[c]);
}

// Structure factors for one (kx, ky) row and a chunk of kz (reference.hpp:
// 168-175): rho = sum_j q_j e^{-i xi.r_j}.  e^{-i(kx tx + ky ty)} by sincos,
// the kz progression by recurrence from e^{-i kz0 tz}.
__global__ void __launch_bounds__(kDirThreads) k_rho(long N, const double4* __restrict__ xyzq,
                                                     int kmax, double bx, double by, double bz,
                                                     double2* __restrict__ rho) {
    __shared__ double red[2 * kKzChunk][32];
    const int W = 2 * kmax + 1;
    const int nch = (W + kKzChunk - 1) / kKzChunk;
    const int row = blockIdx.x / nch, ch = blockIdx.x - row * nch;
    const int kx = row / W - kmax, ky = row % W - kmax;
    const int kz0 = ch * kKzChunk - kmax;
    const int nk = min(kKzChunk, kmax - kz0 + 1);
    double re[kKzChunk], im[kKzChunk];
#pragma unroll
    for (int c = 0; c < kKzChunk; ++c) re[c] = im[c] = 0.0;
    for (long j = threadIdx.x; j < N; j += blockDim.x) {
        const double4 p = xyzq[j];
        const double txy = 2.0 * kPiD * (kx * p.x / bx + ky * p.y / by);
        const double tz = 2.0 * kPiD * p.z / bz;
        double s0, c0, ss, cs;
        sincos(-(txy + kz0 * tz), &s0, &c0);  // e^{-i(kx tx + ky ty + kz0 tz)}
        sincos(-tz, &ss, &cs);                // step e^{-i tz}
        double pr = c0, pim = s0;
#pragma unroll
        for (int c = 0; c < kKzChunk; ++c) {
            if (c < nk) {
                re[c] = fma(p.w, pr, re[c]);
                im[c] = fma(p.w, pim, im[c]);
            }
            const double nr = pr * cs - pim * ss, ni = pr * ss + pim * cs;
            pr = nr;
            pim = ni;
        }
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int c = 0; c < kKzChunk; ++c) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            re[c] += __shfl_xor_sync(0xffffffffu, re[c], o);
            im[c] += __shfl_xor_sync(0xffffffffu, im[c], o);
        }
        if (lane == 0) {
            red[2 * c][w] = re[c];
            red[2 * c + 1][w] = im[c];
        }
    }
    __syncthreads();
    if (threadIdx.x < 2 * kKzChunk) {
        const int c = threadIdx.x >> 1;
        double x = 0.0;
        for (int k = 0; k < nw; ++k) x += red[threadIdx.x][k];
        if (c < nk) {
            double* dst = reinterpret_cast<double*>(rho + (static_cast<long>(row) * W + (kz0 + kmax + c)));
            dst[threadIdx.x & 1] = x;
        }
    }
}

// Reciprocal part for the targets (reference.hpp:176-196): CTA per target,
// threads over all modes of the cube (k = 0 has weight 0).
__global__ void __launch_bounds__(kDirThreads) k_recip_targets(const double4* __restrict__ xyzq,
                                                               const long* __restrict__ tgt,
                                                               int kmax, double bx, double by,
                                                               double bz, double lambda, double V,
                                                               const double2* __restrict__ rho,
                                                               double* __restrict__ out) {
    __shared__ double red[4 * 32];
    const long i = tgt[blockIdx.x];
    const double4 p = xyzq[i];
    const int W = 2 * kmax + 1;
    const long nm = static_cast<long>(W) * W * W;
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (long m = threadIdx.x; m < nm; m += blockDim.x) {
        const int kz = static_cast<int>(m % W) - kmax;
        const int ky = static_cast<int>((m / W) % W) - kmax;
        const int kx = static_cast<int>(m / (static_cast<long>(W) * W)) - kmax;
        if (kx == 0 && ky == 0 && kz == 0) continue;
        const double xx = 2.0 * kPiD * kx / bx, xy = 2.0 * kPiD * ky / by, xz = 2.0 * kPiD * kz / bz;
        const double xi2 = xx * xx + xy * xy + xz * xz;
        const double w = exp(-lambda * lambda * xi2 / 4.0) / (xi2 * V);
        double s, c;
        sincos(2.0 * kPiD * (kx * p.x / bx + ky * p.y / by + kz * p.z / bz), &s, &c);
        const double2 r = rho[m];
        const double tr = c * r.x - s * r.y, ti = c * r.y + s * r.x;  // e^{+i xi.r_i} rho
        v[0] += w * tr;
        const double fc = p.w * w * ti;
        v[1] += fc * xx;
        v[2] += fc * xy;
        v[3] += fc * xz;
    }
    block_sum4(v, red);
    if (threadIdx.x == 0)
#pragma unroll
        for (int c = 0; c < 4; ++c) out[4 * blockIdx.x + c] = v[c];
}

double fold1h(double x, double L) {
    x -= L * std::floor(x / L);  // system.hpp:29-36
    if (x >= L) x = 0.0;
    return x;
}

}  // namespace

DirectPassResult direct_ewald_pass(int device, const double box[3], long N, const double* pos,
                                   const double* q, long ntarget, const long* targets, double tol,
                                   double lambda, double* u, double* F) {
    if (N <= 0) throw InvalidArgument("direct_ewald: empty system");
    if (!(tol >= 1e-12))
        throw InvalidArgument("direct_ewald: tol below double-precision trust (need >= 1e-12)");
    for (int d = 0; d < 3; ++d)
        if (!(box[d] > 0.0)) throw InvalidArgument("direct_ewald: invalid box");
    if (!(lambda > 0.0)) lambda = std::min({box[0], box[1], box[2]}) / 6.0;
    DK(cudaSetDevice(device));
    std::vector<long> tg;
    if (targets) {
        tg.assign(targets, targets + ntarget);
        for (long t : tg)
            if (t < 0 || t >= N) throw InvalidArgument("direct_ewald: target index out of range");
    } else {
        tg.resize(N);
        for (long i = 0; i < N; ++i) tg[i] = i;
    }
    const long nt = static_cast<long>(tg.size());
    DirectPassResult res;
    res.lambda = lambda;
    if (nt == 0) return res;
    if (nt > 65535L * 1024) throw InvalidArgument("direct_ewald: too many targets");

    std::vector<double> h(4 * N);
    double qabs = 0.0;
    for (long j = 0; j < N; ++j) {
        for (int d = 0; d < 3; ++d) h[4 * j + d] = fold1h(pos[3 * j + d], box[d]);
        h[4 * j + 3] = q[j];
        qabs += std::fabs(q[j]);
    }
    DevBuf<double4> d_xyzq(N);
    DevBuf<long> d_tg(nt);
    DevBuf<double> d_acc(4 * nt);
    DevBuf<double> d_real(4 * nt);
    DevBuf<double3> d_off(kMaxShellOffsets);
    DK(cudaMemcpy(d_xyzq.p, h.data(), sizeof(double) * 4 * N, cudaMemcpyHostToDevice));
    DK(cudaMemcpy(d_tg.p, tg.data(), sizeof(long) * nt, cudaMemcpyHostToDevice));
    DK(cudaMemset(d_real.p, 0, sizeof(double) * 4 * nt));

    // real space, shell by shell (reference.hpp:55-110)
    const int shell_cap = 16;
    std::vector<double> acc(4 * nt), real(4 * nt, 0.0);
    int sm_count = 148;
    DK(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, device));
    for (int m = 0; m <= shell_cap; ++m) {
        std::vector<double3> off;
        for (int nx = -m; nx <= m; ++nx)
            for (int ny = -m; ny <= m; ++ny)
                for (int nz = -m; nz <= m; ++nz)
                    if (std::max({std::abs(nx), std::abs(ny), std::abs(nz)}) == m)
                        off.push_back(make_double3(nx * box[0], ny * box[1], nz * box[2]));
        DK(cudaMemcpy(d_off.p, off.data(), sizeof(double3) * off.size(), cudaMemcpyHostToDevice));
        DK(cudaMemset(d_acc.p, 0, sizeof(double) * 4 * nt));
        // sources split over enough CTAs to fill the GPU for few targets
        const long want = std::max<long>(1, (4L * sm_count * 8) / std::max<long>(nt, 1));
        const unsigned gx = static_cast<unsigned>(
            std::min<long>(want, (N + kDirThreads - 1) / kDirThreads));
        for (long t0 = 0; t0 < nt; t0 += 65535) {
            const long tn = std::min<long>(65535, nt - t0);
            dim3 grid(gx, static_cast<unsigned>(tn));
            k_real_shell<<<grid, kDirThreads>>>(N, d_xyzq.p, d_tg.p + t0, d_off.p,
                                                static_cast<int>(off.size()), m == 0 ? 1 : 0,
                                                lambda, d_acc.p + 4 * t0);
            DK(cudaGetLastError());
        }
        DK(cudaMemcpy(acc.data(), d_acc.p, sizeof(double) * 4 * nt, cudaMemcpyDeviceToHost));
        double maxc = 0.0;
        for (long t = 0; t < nt; ++t) {
            for (int c = 0; c < 4; ++c) real[4 * t + c] += acc[4 * t + c];
            maxc = std::max(maxc, std::fabs(acc[4 * t]));
        }
        res.real_shells = m;
        if (m >= 1 && maxc < tol / 10.0) {
            res.tail_bound = std::max(res.tail_bound, maxc);
            break;
        }
        if (m == shell_cap) throw NumericalError("direct_ewald: real-space sum did not converge");
    }

    // reciprocal cutoff (reference.hpp:112-127)
    const double V = box[0] * box[1] * box[2];
    const double Lmax = std::max({box[0], box[1], box[2]});
    int kmax = 0;
    for (int m = 1;; ++m) {
        const double ximin = 2.0 * kPiD * m / Lmax;
        const double bound = (qabs / V) * std::exp(-lambda * lambda * ximin * ximin / 4.0) /
                             (ximin * ximin);
        if (bound < tol / 10.0) {
            kmax = m;
            res.tail_bound = std::max(res.tail_bound, bound);
            break;
        }
        if (m >= 512) throw NumericalError("direct_ewald: reciprocal sum did not converge");
    }
    res.recip_kmax = kmax;
    const int W = 2 * kmax + 1;
    const long nm = static_cast<long>(W) * W * W;
    DevBuf<double2> d_rho(nm);
    const int nch = (W + kKzChunk - 1) / kKzChunk;
    k_rho<<<static_cast<unsigned>(static_cast<long>(W) * W * nch), kDirThreads>>>(
        N, d_xyzq.p, kmax, box[0], box[1], box[2], d_rho.p);
    DK(cudaGetLastError());
    DevBuf<double> d_rec(4 * nt);
    for (long t0 = 0; t0 < nt; t0 += 1L << 30) {
        const long tn = std::min<long>(1L << 30, nt - t0);
        k_recip_targets<<<static_cast<unsigned>(tn), kDirThreads>>>(
            d_xyzq.p, d_tg.p + t0, kmax, box[0], box[1], box[2], lambda, V, d_rho.p,
            d_rec.p + 4 * t0);
        DK(cudaGetLastError());
    }
    std::vector<double> rec(4 * nt);
    DK(cudaMemcpy(rec.data(), d_rec.p, sizeof(double) * 4 * nt, cudaMemcpyDeviceToHost));
    const double self = 1.0 / (2.0 * std::pow(kPiD, 1.5) * lambda);
    for (long t = 0; t < nt; ++t) {
        const long i = tg[t];
        u[t] = real[4 * t] + rec[4 * t] - q[i] * self;
        for (int d = 0; d < 3; ++d) F[3 * t + d] = real[4 * t + 1 + d] + rec[4 * t + 1 + d];
    }
    return res;
}

}  // namespace espb
