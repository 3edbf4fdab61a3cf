// C ABI (include/esp_b200.h) over the host plan builder and the device engine.

#include "../../include/esp_b200.h"

#include "capi_internal.hpp"
#include "direct.hpp"

#include <cuda_runtime.h>
#include <cufft.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

namespace espc {
std::string& last_error() {
    static thread_local std::string e;
    return e;
}
}  // namespace espc

namespace {

using espc::cuda_ok;
using espc::engine;
using espc::guarded;

void check_box(const esp_plan* p, const double* box, const char* who) {
    // evaluate / spectral_sum require box == plan.box exactly (ewald.hpp:620-621)
    if (!box) return;
    for (int d = 0; d < 3; ++d)
        if (box[d] != p->plan.box[d])
            throw espb::InvalidArgument(std::string(who) + ": system box does not match plan box");
}

void require_neutral(long N, const double* q) {
    // system.hpp:39-47
    double total = 0.0, abssum = 0.0;
    for (long i = 0; i < N; ++i) {
        total += q[i];
        abssum += std::fabs(q[i]);
    }
    if (std::fabs(total) > 1e-12 * std::max(abssum, 1.0))
        throw espb::NumericalError("system is not charge neutral");
}

void stage(esp_plan* p, long N) {
    cuda_ok(cudaSetDevice(p->device), "cudaSetDevice");
    if (!p->stream) cuda_ok(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking), "stream");
    if (!p->d_e) cuda_ok(cudaMalloc(&p->d_e, 4 * sizeof(double)), "cudaMalloc");
    if (!p->h_e) cuda_ok(cudaMallocHost(&p->h_e, 4 * sizeof(double)), "cudaMallocHost");
    if (N <= p->cap) return;
    cudaFree(p->d_pos);
    cudaFree(p->d_q);
    cudaFree(p->d_u);
    cudaFree(p->d_F);
    long c = std::max<long>(N, 1);
    cuda_ok(cudaMalloc(&p->d_pos, 3 * c * sizeof(double)), "cudaMalloc");
    cuda_ok(cudaMalloc(&p->d_q, c * sizeof(double)), "cudaMalloc");
    cuda_ok(cudaMalloc(&p->d_u, 3 * c * sizeof(double)), "cudaMalloc");
    cuda_ok(cudaMalloc(&p->d_F, 3 * c * sizeof(double)), "cudaMalloc");
    p->cap = c;
}

constexpr long kZeroCopyMaxN = 1L << 17;

// Device address of a pinned host buffer (nullptr for pageable memory).
template <class T>
T* mapped(T* host) {
    if (!host) return nullptr;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, host) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (at.type != cudaMemoryTypeHost || !at.devicePointer) return nullptr;
    return static_cast<T*>(at.devicePointer);
}

void h2d(esp_plan* p, double* dst, const double* src, long n) {
    if (n > 0)
        cuda_ok(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyHostToDevice, p->stream),
                "H2D");
}
void d2h(esp_plan* p, double* dst, const double* src, long n) {
    if (n > 0)
        cuda_ok(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToHost, p->stream),
                "D2H");
}
void sync(esp_plan* p) { cuda_ok(cudaStreamSynchronize(p->stream), "synchronize"); }

void check_n(long N) {
    if (N < 0) throw espb::InvalidArgument("N must be non-negative");
    if (N > 0x7fffffffL) throw espb::InvalidArgument("N exceeds the 2^31-1 atom limit");
}

}  // namespace

extern "C" {

const char* esp_last_error(void) { return espc::last_error().c_str(); }
const char* esp_version(void) { return "esp-b200 0.1 (sm_100a)"; }

int esp_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int esp_plan_create(const double box[3], int family, double eps, double r_c,
                    const esp_overrides* ov, int device, esp_plan** out) {
    return guarded([&] {
        if (!out || !box) throw espb::InvalidArgument("null argument");
        *out = nullptr;
        espb::Overrides o;
        if (ov) {
            o.nf = ov->nf;
            o.P = ov->P;
            o.c1 = ov->c1;
            o.force_method = ov->force_method == ESP_FORCE_AD ? espb::ForceMethod::ad
                                                              : espb::ForceMethod::ik;
            o.allow_degraded = ov->allow_degraded != 0;
        }
        auto h = std::make_unique<esp_plan>();
        if (device >= 0) {
            int n = 0;
            if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
                cudaGetLastError();
                throw espb::CudaError("no CUDA device available");
            }
            if (device >= n) throw espb::InvalidArgument("device index out of range");
        }
        // the O(n_f^3) plan tables on the plan's device;
        // ESP_PLAN_DEVICE=0 keeps them on the host
        std::unique_ptr<espb::PlanDevice> pdev;
        const char* pd = std::getenv("ESP_PLAN_DEVICE");
        if (device >= 0 && !(pd && std::atoi(pd) == 0)) pdev = espb::make_plan_device(device);
        h->plan = espb::build_plan({box[0], box[1], box[2]},
                                   family == ESP_FAMILY_GAUSSIAN ? espb::Family::gaussian
                                                                 : espb::Family::pswf,
                                   eps, r_c, o, pdev.get());
        if (device >= 0) {
            h->device = device;
            h->eng = std::make_unique<espb::Engine>(h->plan, device);
        }
        *out = h.release();
    });
}

void esp_plan_destroy(esp_plan* plan) { delete plan; }

int esp_plan_get_info(const esp_plan* p, esp_plan_info* o) {
    return guarded([&] {
        if (!p || !o) throw espb::InvalidArgument("null argument");
        const espb::Plan& P = p->plan;
        std::memset(o, 0, sizeof(*o));
        o->family = static_cast<int>(P.family);
        o->force_method = static_cast<int>(P.force_method);
        o->P = P.P;
        for (int d = 0; d < 3; ++d) {
            o->nf[d] = P.nf[d];
            o->base_nf[d] = P.base_nf[d];
            o->box[d] = P.box[d];
            o->h[d] = P.h[d];
            o->demand[d] = P.demand[d];
            o->pair_cells[d] = std::max(1, static_cast<int>(std::floor(P.box[d] / P.r_c)));
        }
        o->eps = P.eps;
        o->r_c = P.r_c;
        o->shape = P.shape;
        o->c1 = P.c1;
        o->chi0 = P.chi0;
        o->E_A = P.E_A;
        o->E_T = P.E_T;
        o->E_SI = P.E_SI;
        o->self_coef = P.self_coef;
        o->n_split_coef = static_cast<int>(P.split.a.size());
        o->n_window_coef = static_cast<int>(P.window.a.size());
        o->pair_poly_degree = static_cast<int>(P.pair_H.size()) - 1;
        o->pencil_half = p->eng ? (p->eng->pencil_half() ? 1 : 0) : espb::Engine::pencil_half_env();
        o->fused_xpass = p->eng && p->eng->fused_xpass() ? 1 : 0;
        o->deterministic = p->eng && p->eng->deterministic() ? 1 : 0;
        o->pair_kernel = p->eng ? p->eng->pair_kernel() : -1;
        o->spread_kernel = p->eng ? p->eng->spread_kernel() : -1;
        o->pair_fit_err = P.pair_fit_err;
        o->device = p->device;
    });
}

int esp_plan_set_deterministic(esp_plan* p, int on) {
    return guarded([&] { engine(p).set_deterministic(on != 0); });
}

int esp_plan_get_influence(const esp_plan* p, double* out) {
    return guarded([&] {
        auto v = espb::influence_full(p->plan);
        std::memcpy(out, v.data(), v.size() * sizeof(double));
    });
}

int esp_plan_get_table(const esp_plan* p, int which, int dim, double* out, int* nseg) {
    return guarded([&] {
        const espb::PiecewisePoly* pp = nullptr;
        if (dim < 0 || dim > 2) throw espb::InvalidArgument("dim out of range");
        switch (which) {
            case 0: pp = &p->plan.Psi; break;
            case 1: pp = &p->plan.chi; break;
            case 2: pp = &p->plan.phi[dim]; break;
            case 3: pp = &p->plan.dphi[dim]; break;
            default: throw espb::InvalidArgument("table selector out of range");
        }
        if (nseg) *nseg = pp->nseg;
        if (out) std::memcpy(out, pp->cheb.data(), pp->cheb.size() * sizeof(double));
    });
}

int esp_plan_get_prolate(const esp_plan* p, int which, double* out, int* n) {
    return guarded([&] {
        const auto& a = which < 0 ? p->plan.split.a : p->plan.window.a;
        if (n) *n = static_cast<int>(a.size());
        if (out) std::memcpy(out, a.data(), a.size() * sizeof(double));
    });
}

int esp_plan_eval_kernel(const esp_plan* p, int what, long n, const double* x, double* y) {
    return guarded([&] {
        const espb::Plan& P = p->plan;
        for (long i = 0; i < n; ++i) {
            switch (what) {
                case 0: y[i] = P.Psi_at(x[i]); break;
                case 1: y[i] = P.chi_at(x[i]); break;
                case 2: y[i] = P.chihat_n(x[i]); break;
                case 3: y[i] = P.phi_at(0, x[i]); break;
                case 4: y[i] = P.dphi_at(0, x[i]); break;
                case 5: y[i] = P.phi_hat(0, x[i]); break;
                case 6: y[i] = P.local_kernel(x[i]).first; break;
                case 7: y[i] = P.local_kernel(x[i]).second; break;
                case 8: case 9: case 10: y[i] = P.phi_at(what - 8, x[i]); break;
                case 11: case 12: case 13: y[i] = P.dphi_at(what - 11, x[i]); break;
                case 14: case 15: case 16: y[i] = P.phi_hat(what - 14, x[i]); break;
                default: throw espb::InvalidArgument("kernel selector out of range");
            }
        }
    });
}

int esp_fft3(const int nf[3], double* data, int direction, int device) {
    return guarded([&] {
        if (!nf || !data) throw espb::InvalidArgument("null argument");
        if (nf[0] < 1 || nf[1] < 1 || nf[2] < 1) throw espb::InvalidArgument("fft: bad grid");
        if (direction != -1 && direction != 1)
            throw espb::InvalidArgument("fft: direction must be -1 (forward) or +1 (inverse)");
        cuda_ok(cudaSetDevice(device), "cudaSetDevice");
        const size_t n = static_cast<size_t>(nf[0]) * nf[1] * nf[2];
        void* d = nullptr;
        cuda_ok(cudaMalloc(&d, n * 2 * sizeof(double)), "cudaMalloc");
        struct Free {
            void* p;
            ~Free() { cudaFree(p); }
        } guard{d};
        cuda_ok(cudaMemcpy(d, data, n * 2 * sizeof(double), cudaMemcpyHostToDevice), "H2D");
        cufftHandle h = 0;
        if (cufftPlan3d(&h, nf[0], nf[1], nf[2], CUFFT_Z2Z) != CUFFT_SUCCESS)
            throw espb::CudaError("fft: cufftPlan3d failed");
        const cufftResult r = cufftExecZ2Z(h, static_cast<cufftDoubleComplex*>(d),
                                           static_cast<cufftDoubleComplex*>(d),
                                           direction < 0 ? CUFFT_FORWARD : CUFFT_INVERSE);
        cufftDestroy(h);
        if (r != CUFFT_SUCCESS) throw espb::CudaError("fft: cufftExecZ2Z failed");
        cuda_ok(cudaMemcpy(data, d, n * 2 * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    });
}

int esp_check_neutral(long N, const double* q) {
    return guarded([&] { require_neutral(N, q); });
}

int esp_self_correction(const esp_plan* p, long N, const double* q, double* out) {
    return guarded([&] {
        const double s0 = p->plan.self_coef;  // ewald.hpp:611
        for (long i = 0; i < N; ++i) out[i] = q[i] * s0;
    });
}

int esp_evaluate(esp_plan* p, const double box[3], long N, const double* pos, const double* q,
                 double* u, double* F, double* energy, esp_timings* timings) {
    return guarded([&] {
        espb::Engine& e = engine(p);
        check_box(p, box, "evaluate");
        check_n(N);
        stage(p, N);
        espb::StageTimes st;
        // pinned (page-locked) host buffers are device-accessible: for small
        // systems the fold kernel reads positions and charges over PCIe and
        // the combine kernel writes u and F back over PCIe -- no staging
        // copies (cfg2: -11 % end to end).  Large systems keep the bulk
        // copies, which move the bytes faster than the kernels' 8-byte
        // accesses do.
        const bool small = N > 0 && N <= kZeroCopyMaxN;
        const double *pos_m = small ? mapped(pos) : nullptr, *q_m = small ? mapped(q) : nullptr;
        double *u_m = small ? mapped(u) : nullptr, *F_m = small ? mapped(F) : nullptr;
        // require_neutral (system.hpp:39-47) before any output is written, as
        // the reference does (ewald.hpp:622): the caller's u / F stay
        // untouched when it throws.  The zero-copy path writes u / F from the
        // combine kernel, so it checks first (N <= 2^17: microseconds); the
        // bulk path runs the same host loop while the GPU evaluates, and only
        // copies the results out after it passed.
        if (pos_m && q_m && u_m && F_m) {
            require_neutral(N, q);
            e.evaluate(N, pos_m, q_m, p->d_u, p->d_F, p->d_e, p->d_e + 1, p->stream,
                       timings ? &st : nullptr, u_m, F_m);
        } else {
            h2d(p, p->d_pos, pos, 3 * N);
            h2d(p, p->d_q, q, N);
            e.evaluate(N, p->d_pos, p->d_q, p->d_u, p->d_F, p->d_e, p->d_e + 1, p->stream,
                       timings ? &st : nullptr);
            try {
                require_neutral(N, q);
            } catch (...) {
                sync(p);
                throw;
            }
            d2h(p, u, p->d_u, N);
            d2h(p, F, p->d_F, 3 * N);
        }
        double* hv = p->h_e;  // pinned: the small read stays on the async path
        cuda_ok(cudaMemcpyAsync(hv, p->d_e, 3 * sizeof(double), cudaMemcpyDeviceToHost, p->stream),
                "D2H");
        sync(p);
        *energy = hv[0];
        if (timings) {
            timings->local = st.local;
            timings->spread = st.spread;
            timings->fft = st.fft;
            timings->scale = st.scale;
            timings->ifft = st.ifft;
            timings->interpolate = st.interpolate;
            timings->bin = st.bin;
        }
    });
}

int esp_evaluate_device(esp_plan* p, const double box[3], long N, const double* pos_dev,
                        const double* q_dev, double* u_dev, double* F_dev, double* energy_dev,
                        void* stream) {
    return guarded([&] {
        espb::Engine& e = engine(p);
        check_box(p, box, "evaluate");
        check_n(N);
        cuda_ok(cudaSetDevice(p->device), "cudaSetDevice");
        e.evaluate(N, pos_dev, q_dev, u_dev, F_dev, energy_dev, nullptr,
                   static_cast<cudaStream_t>(stream), nullptr);
    });
}

int esp_eval_phase_a(esp_plan* p, const double box[3], long N, const double* pos_dev,
                     const double* q_dev, int rank, int nranks, double* grid_dev, void* stream) {
    return guarded([&] {
        espb::Engine& e = engine(p);
        check_box(p, box, "evaluate");
        check_n(N);
        e.phase_a(N, pos_dev, q_dev, rank, nranks, grid_dev, static_cast<cudaStream_t>(stream));
    });
}

int esp_eval_phase_b(esp_plan* p, int rank, int nranks, const double* grid_dev, double* u_dev,
                     double* F_dev, double* energy_dev, void* stream) {
    return guarded([&] {
        espb::Engine& e = engine(p);
        e.phase_b(rank, nranks, grid_dev, u_dev, F_dev, energy_dev,
                  static_cast<cudaStream_t>(stream));
    });
}

int esp_pencil_geometry(const esp_plan* p, int rank, int nranks, esp_pencil_info* out) {
    return guarded([&] {
        if (!p || !out) throw espb::InvalidArgument("null argument");
        const espb::PencilGeom G = espb::pencil_geometry(p->plan, rank, nranks);
        out->nranks = G.nranks;
        out->rank = G.rank;
        out->halo = G.halo;
        out->x0 = G.x0;
        out->x1 = G.x1;
        out->y0 = G.y0;
        out->y1 = G.y1;
        out->nfields = G.nfields;
        for (int d = 0; d < 3; ++d) out->nf[d] = p->plan.nf[d];
        out->hx = G.hx;
        out->S = G.S;
        out->nbx = G.nbx;
        out->bx0 = G.bx0;
        out->bx1 = G.bx1;
        out->slab_reals = G.slab_reals;
        out->spec_local = G.spec_local;
        out->spec_pencil = G.spec_pencil;
    });
}

int esp_pencil_phase_a(esp_plan* p, const double box[3], long N, const double* pos_dev,
                       const double* q_dev, int rank, int nranks, double* slab_dev, void* stream) {
    return guarded([&] {
        espb::Engine& e = engine(p);
        check_box(p, box, "evaluate");
        check_n(N);
        e.pencil_phase_a(N, pos_dev, q_dev, rank, nranks, slab_dev,
                         static_cast<cudaStream_t>(stream));
    });
}

int esp_pencil_forward(esp_plan* p, int rank, int nranks, const double* slab_dev,
                       double* send_dev, void* stream) {
    return guarded([&] {
        engine(p).pencil_forward(rank, nranks, slab_dev,
                                 reinterpret_cast<cufftDoubleComplex*>(send_dev),
                                 static_cast<cudaStream_t>(stream));
    });
}

int esp_pencil_solve(esp_plan* p, int rank, int nranks, double* recv_dev, double* A_dev,
                     double* B_dev, void* stream) {
    return guarded([&] {
        engine(p).pencil_solve(rank, nranks, reinterpret_cast<cufftDoubleComplex*>(recv_dev),
                               reinterpret_cast<cufftDoubleComplex*>(A_dev),
                               reinterpret_cast<cufftDoubleComplex*>(B_dev),
                               static_cast<cudaStream_t>(stream));
    });
}

int esp_pencil_backward(esp_plan* p, int rank, int nranks, const double* A_dev,
                        const double* B_dev, double* fslab_dev, void* stream) {
    return guarded([&] {
        engine(p).pencil_backward(rank, nranks, reinterpret_cast<const cufftDoubleComplex*>(A_dev),
                                  reinterpret_cast<const cufftDoubleComplex*>(B_dev), fslab_dev,
                                  static_cast<cudaStream_t>(stream));
    });
}

int esp_pencil_phase_b(esp_plan* p, int rank, int nranks, const double* fslab_dev, double* u_dev,
                       double* F_dev, double* energy_dev, void* stream) {
    return guarded([&] {
        engine(p).pencil_phase_b(rank, nranks, fslab_dev, u_dev, F_dev, energy_dev,
                                 static_cast<cudaStream_t>(stream));
    });
}

int esp_direct_ewald(const double box[3], long N, const double* pos, const double* q,
                     long ntarget, const long* targets, double tol, double lambda, double* u,
                     double* F, double* energy, esp_direct_info* info, int device) {
    return guarded([&] {
        if (!box || !pos || !q || !u || !F) throw espb::InvalidArgument("null argument");
        if (N <= 0) throw espb::InvalidArgument("direct_ewald: empty system");
        if (targets && ntarget < 0) throw espb::InvalidArgument("direct_ewald: bad target count");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
            cudaGetLastError();
            throw espb::CudaError("direct_ewald: no such CUDA device");
        }
        require_neutral(N, q);  // reference.hpp:218
        const espb::DirectPassResult r = espb::direct_ewald_pass(
            device, box, N, pos, q, targets ? ntarget : N, targets, tol, lambda, u, F);
        if (energy) {
            if (targets) {
                *energy = std::nan("");
            } else {
                double s = 0.0, c = 0.0;  // Kahan, as the reference
                for (long i = 0; i < N; ++i) {
                    const double y = q[i] * u[i] - c;
                    const double t = s + y;
                    c = (t - s) - y;
                    s = t;
                }
                *energy = 0.5 * s;
            }
        }
        if (info) {
            info->lambda = r.lambda;
            info->real_shells = r.real_shells;
            info->recip_kmax = r.recip_kmax;
            info->tail_bound = r.tail_bound;
        }
    });
}

long esp_grid_size(const esp_plan* p) {
    return p ? static_cast<long>(p->plan.nf[0]) * p->plan.nf[1] * p->plan.nf[2] : 0;
}

int esp_local_sum(esp_plan* p, const double box[3], long N, const double* pos, const double* q,
                  double* u, double* F) {
    return guarded([&] {
        espb::Engine& e = engine(p);
        // local_sum requires r_c < min(L)/2 of the system box (ewald.hpp:420-422)
        if (box) {
            double Lmin = std::min({box[0], box[1], box[2]});
            if (!(p->plan.r_c < Lmin / 2.0))
                throw espb::InvalidArgument("local_sum: require r_c < min(L)/2");
            check_box(p, box, "local_sum");
        }
        check_n(N);
        stage(p, N);
        h2d(p, p->d_pos, pos, 3 * N);
        h2d(p, p->d_q, q, N);
        e.local_sum(N, p->d_pos, p->d_q, p->d_u, p->d_F, p->stream);
        d2h(p, u, p->d_u, N);
        d2h(p, F, p->d_F, 3 * N);
        sync(p);
    });
}

int esp_spectral_sum(esp_plan* p, const double box[3], long N, const double* pos,
                     const double* q, double* u, double* F, esp_timings* timings) {
    return guarded([&] {
        espb::Engine& e = engine(p);
        check_box(p, box, "spectral_sum");
        check_n(N);
        stage(p, N);
        h2d(p, p->d_pos, pos, 3 * N);
        h2d(p, p->d_q, q, N);
        espb::StageTimes st;
        e.spectral_sum(N, p->d_pos, p->d_q, p->d_u, p->d_F, p->stream, timings ? &st : nullptr);
        d2h(p, u, p->d_u, N);
        d2h(p, F, p->d_F, 3 * N);
        sync(p);
        if (timings) {
            *timings = esp_timings{};
            timings->spread = st.spread;
            timings->fft = st.fft;
            timings->scale = st.scale;
            timings->ifft = st.ifft;
            timings->interpolate = st.interpolate;
        }
    });
}

int esp_spread(esp_plan* p, long N, const double* pos, const double* q, double* grid) {
    return guarded([&] {
        espb::Engine& e = engine(p);
        check_n(N);
        stage(p, N);
        const long M = static_cast<long>(p->plan.nf[0]) * p->plan.nf[1] * p->plan.nf[2];
        double* d_grid = nullptr;
        cuda_ok(cudaMalloc(&d_grid, M * sizeof(double)), "cudaMalloc");
        try {
            h2d(p, p->d_pos, pos, 3 * N);
            h2d(p, p->d_q, q, N);
            e.spread(N, p->d_pos, p->d_q, d_grid, p->stream);
            d2h(p, grid, d_grid, M);
            sync(p);
        } catch (...) {
            cudaFree(d_grid);
            throw;
        }
        cudaFree(d_grid);
    });
}

static int interp_common(esp_plan* p, long N, const double* pos, const double* grid, double* out,
                         bool gradient) {
    return guarded([&] {
        espb::Engine& e = engine(p);
        check_n(N);
        stage(p, N);
        const long M = static_cast<long>(p->plan.nf[0]) * p->plan.nf[1] * p->plan.nf[2];
        double* d_grid = nullptr;
        cuda_ok(cudaMalloc(&d_grid, M * sizeof(double)), "cudaMalloc");
        try {
            h2d(p, p->d_pos, pos, 3 * N);
            h2d(p, d_grid, grid, M);
            if (gradient) e.interpolate_gradient(N, p->d_pos, d_grid, p->d_u, p->stream);
            else e.interpolate(N, p->d_pos, d_grid, p->d_u, p->stream);
            d2h(p, out, p->d_u, gradient ? 3 * N : N);
            sync(p);
        } catch (...) {
            cudaFree(d_grid);
            throw;
        }
        cudaFree(d_grid);
    });
}

int esp_interpolate(esp_plan* p, long N, const double* pos, const double* grid, double* out) {
    return interp_common(p, N, pos, grid, out, false);
}

int esp_interpolate_gradient(esp_plan* p, long N, const double* pos, const double* grid,
                             double* out) {
    return interp_common(p, N, pos, grid, out, true);
}

int esp_last_launch_count(const esp_plan* p) { return p && p->eng ? p->eng->last_launches() : 0; }

int esp_last_pair_count(esp_plan* p, unsigned long long* ordered_pairs) {
    return guarded([&] {
        espb::Engine& e = engine(p);
        if (p->stream) cuda_ok(cudaStreamSynchronize(p->stream), "synchronize");
        cuda_ok(cudaDeviceSynchronize(), "synchronize");
        *ordered_pairs = e.last_pair_count();
    });
}

int esp_pair_eval_rate(esp_plan* p, double* pairs_per_s) {
    return guarded([&] {
        engine(p);
        *pairs_per_s = espb::pair_eval_rate(p->plan, p->device);
    });
}

int esp_fp64_peak(int device, double* tflops) {
    return guarded([&] { *tflops = espb::fp64_peak_tflops(device); });
}

}  // extern "C"
