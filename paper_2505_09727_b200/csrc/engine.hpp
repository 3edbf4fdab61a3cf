// Device engine for one ESP plan on one B200 (sm_100a).
//
// Owns the device copies of the plan tables, the cuFFT plans, the scratch
// buffers sized for the largest N seen, and two streams' worth of events.
// Every public method is asynchronous on the caller's stream unless noted;
// pointers are device pointers.  See DESIGN.md for the data layout and the
// kernel list (K1 spread, K2 influence/derivative multiply, K3 interpolation
// + combine, K4 real-space pair sum, plus the two counting sorts).
#pragma once

#include "plan.hpp"

#include <cuda_runtime.h>
#include <cufft.h>

#include <array>
#include <string>

namespace espb {

struct GridArgs;

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// Stage wall times in seconds (reference keys ewald.hpp:628-629 plus the
// GPU-only binning stage).
struct StageTimes {
    double local = 0, spread = 0, fft = 0, scale = 0, ifft = 0, interpolate = 0, bin = 0;
};

// Measured fp64 FMA throughput of the device (TFLOP/s), for the roofline.
double fp64_peak_tflops(int device);
// Ordered pairs per second of the K4 evaluation alone (operands in registers).
double pair_eval_rate(const Plan& p, int device);

class Engine {
public:
    Engine(const Plan& plan, int device);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    int device() const { return device_; }

    // Full evaluation (ewald.hpp:619-649): u = u_l + u_s - self, F = F_l + F_s,
    // energy_dev[0] = 1/2 sum q u.  qsum_dev (optional, 2 doubles) receives
    // (sum q, sum |q|) for the neutrality check.
    void evaluate(long N, const double* pos, const double* q, double* u, double* F,
                  double* energy_dev, double* qsum_dev, cudaStream_t s, StageTimes* t = nullptr);
    // Parts (ewald.hpp:419 local_sum, :524 spectral_sum).
    void local_sum(long N, const double* pos, const double* q, double* u, double* F,
                   cudaStream_t s);
    void spectral_sum(long N, const double* pos, const double* q, double* u, double* F,
                      cudaStream_t s);
    // Grid pipeline pieces (gridder.hpp:215, :244, :280); grid = nx*ny*nz reals.
    void spread(long N, const double* pos, const double* q, double* grid, cudaStream_t s);
    void interpolate(long N, const double* pos, const double* grid, double* out,
                     cudaStream_t s);
    void interpolate_gradient(long N, const double* pos, const double* grid, double* out,
                              cudaStream_t s);

    // Slab-decomposed evaluation over `nranks` GPUs (or emulated ranks).
    // Phase A (rank-local): bin/sort all atoms, real-space sum for the targets
    // in this rank's x-slab, spread this slab's atoms into grid_out (M reals).
    // The caller sums grid_out over ranks (NCCL all-reduce), then phase B: the
    // FFT pipeline on the summed grid, interpolation for this slab's atoms and
    // the combine; u/F/energy are this rank's partial sums (zero elsewhere) to
    // be summed over ranks.
    void phase_a(long N, const double* pos, const double* q, int rank, int nranks,
                 double* grid_out, cudaStream_t s);
    void phase_b(int rank, int nranks, const double* grid_in, double* u, double* F,
                 double* energy_dev, cudaStream_t s);

    // Launch count of the last evaluate() (our kernels only, excluding cuFFT).
    int last_launches() const { return launches_; }
    // Ordered in-range pairs (0 < r < r_c) evaluated by the last pair-kernel
    // launch, counted on the device (synchronous read).
    unsigned long long last_pair_count() const;

private:
    void enqueue(long N, const double* pos, const double* q, double* u, double* F,
                 double* energy_dev, double* qsum_dev, cudaStream_t s, StageTimes* t);
    void ensure_capacity(long N);
    void prepare(long N, const double* pos, const double* q, double* qsum_dev, cudaStream_t s);
    void run_pair(long N, cudaStream_t s, int rank, int nranks);
    void run_grid(long N, cudaStream_t s, StageTimes* t);
    void run_spread(long N, cudaStream_t s, int rank, int nranks, double* grid);
    void slab_bins(int rank, int nranks, int* b0, int* b1) const;
    long phase_n_ = 0;
    GridArgs grid_args() const;

    const Plan& plan_;
    int device_ = 0;
    int launches_ = 0;

    // geometry
    bool cells_ok_ = false;     // fine stencil fits the period (else all pairs)
    std::array<int, 3> F_{};    // fine cells per dim (sort key of the pair path)
    long ncellF_ = 0;
    int S_ = 8;                 // spread bin edge in grid cells
    std::array<int, 3> nb_{};   // spread bins per dim
    int nbin_ = 0;
    int W_ = 0;                 // spread tile edge (nodes)
    int RS_ = 0, PS_ = 0;       // padded tile strides
    long M_ = 0, Mh_ = 0;       // real grid size, half spectrum size
    int nfields_ = 4;           // 4 for ik, 1 for ad
    int pair_warps_ = 4;
    int pair_cap_ = 2048;
    int pM_ = 2, pMz_ = 4;      // fine stencil reach (columns, slices)

    // tables on device
    double* d_win_ = nullptr;        // 3 x 4P x 13 phi, then 3 x 4P x 13 dphi
    double* d_influence_ = nullptr;  // Mh
    double* d_xi_ = nullptr;         // nx + ny + nz derivative multipliers (Nyquist = 0)

    // scratch
    long cap_ = 0;
    double4* d_tmp_ = nullptr;   // folded xyzq, original order
    int* d_cellA_ = nullptr;
    int* d_rankA_ = nullptr;
    int* d_cellB_ = nullptr;
    int* d_rankB_ = nullptr;
    double4* d_xyzqA_ = nullptr;
    int* d_origA_ = nullptr;
    double4* d_xyzqB_ = nullptr;
    int* d_origB_ = nullptr;
    double4* d_loc_ = nullptr;   // (u_l, F_l) in original order
    double* d_epart_ = nullptr;  // energy partials
    int* d_countA_ = nullptr;    // ncell + 1
    int* d_startA_ = nullptr;
    int* d_countB_ = nullptr;    // nbin + 1
    int* d_startB_ = nullptr;
    void* d_scan_tmp_ = nullptr;
    size_t scan_tmp_bytes_ = 0;
    double* d_grid_ = nullptr;          // M reals
    cufftDoubleComplex* d_spec_ = nullptr;   // Mh
    cufftDoubleComplex* d_spec4_ = nullptr;  // nfields * Mh
    double* d_fields_ = nullptr;        // nfields * M
    double* d_qsum_ = nullptr;          // scratch for neutrality sums
    unsigned long long* d_npairs_ = nullptr;

    cufftHandle fwd_ = 0, inv_ = 0;
    void* d_cufft_work_ = nullptr;
    cudaStream_t aux_ = nullptr;
    cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
    cudaEvent_t ev_t_[8] = {};

    // CUDA graph of a full evaluation, keyed by its arguments
    struct GraphKey {
        long N;
        const void *pos, *q, *u, *F, *e, *qs;
        bool operator==(const GraphKey& o) const {
            return N == o.N && pos == o.pos && q == o.q && u == o.u && F == o.F && e == o.e &&
                   qs == o.qs;
        }
    };
    bool use_graph_ = true;
    bool warm_ = false;
    GraphKey gkey_{};
    cudaGraphExec_t gexec_ = nullptr;
    cudaStream_t gstream_ = nullptr;
    cudaEvent_t ev_gin_ = nullptr, ev_gout_ = nullptr;
    int graph_launches_ = 0;
};

}  // namespace espb
