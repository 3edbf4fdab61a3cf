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

#include <cstdlib>
#include <cuda_runtime.h>
#include <cufft.h>

#include <cstdio>
#include <array>
#include <vector>
#include <string>

// Device-side bounds checks of the checked build (build.py --checked,
// -DESP_DEVICE_CHECKS; loaded with ESP_B200_CHECKED=1): a failed check prints
// the condition and traps, failing the evaluation with a CUDA error.  The
// product build compiles them out.  (compute-sanitizer is not available on
// the GPU pool; these checks and the reference-parity tests stand in for it.)
#ifdef ESP_DEVICE_CHECKS
#define ESP_DCHECK(c)                                                                  \
    do {                                                                               \
        if (!(c)) {                                                                    \
            printf("ESP_DCHECK failed: %s at %s:%d (block %d thread %d)\n", #c,        \
                   __FILE__, __LINE__, static_cast<int>(blockIdx.x),                   \
                   static_cast<int>(threadIdx.x));                                     \
            __trap();                                                                  \
        }                                                                              \
    } while (0)
#else
#define ESP_DCHECK(c) \
    do {              \
    } while (0)
#endif

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

// Distributed-FFT decomposition over `nranks` GPUs:
// rank r owns the real-space x-planes [x0, x1) and the atoms in them (their
// footprints stay within `halo` planes) and, after the forward transpose, the
// spectral y-rows [y0, y1).  Host-only (no device).
struct PencilGeom {
    int nranks = 1, rank = 0;
    int halo = 0;           // planes exchanged with each x-neighbour
    int x0 = 0, x1 = 0;     // owned real-space planes
    int y0 = 0, y1 = 0;     // owned spectral rows after the transpose
    long slab_reals = 0;    // (x1 - x0 + 2 halo) * ny * nz: spread slab / one field slab
    long spec_local = 0;    // (x1 - x0) * ny * (nz/2+1): forward send size (complex)
    long spec_pencil = 0;   // nx * (y1 - y0) * (nz/2+1): forward receive size (complex)
    int nfields = 4;        // interleaved fields per node of the field slab
    // atom ownership: an atom belongs to the rank whose planes [x0, x1) hold
    // clamp(floor(fold(x) / hx), 0, nx - 1); the rank processes the spread
    // bins [bx0, bx1) (edge S) that intersect its planes
    double hx = 0.0;
    int S = 0, nbx = 0, bx0 = 0, bx1 = 0;
};
// Spread bin edge S (grid cells) the engine uses for a plan.
int spread_bin_edge(const Plan& p);
// Throws InvalidArgument when the decomposition is not possible (a rank
// with fewer planes than the halo, or nranks < 2).
PencilGeom pencil_geometry(const Plan& p, int rank, int nranks);

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
    // u_out / F_out (optional): final u and F written there (e.g. pinned host
    // memory, over PCIe) instead of into u / F, which are then device scratch.
    void evaluate(long N, const double* pos, const double* q, double* u, double* F,
                  double* energy_dev, double* qsum_dev, cudaStream_t s, StageTimes* t = nullptr,
                  double* u_out = nullptr, double* F_out = nullptr);
    // Parts (ewald.hpp:419 local_sum, :524 spectral_sum).
    void local_sum(long N, const double* pos, const double* q, double* u, double* F,
                   cudaStream_t s);
    void spectral_sum(long N, const double* pos, const double* q, double* u, double* F,
                      cudaStream_t s,
                      StageTimes* t = nullptr);
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

    // Distributed-FFT evaluation (pencil_geometry above).  Per rank, with the
    // caller moving data between the phases (NCCL send/recv, all-to-all):
    //   pencil_phase_a  bin/sort, real-space part of this rank's targets,
    //                   spread of its atoms into slab (slab_reals, with halos)
    //   [caller: add each halo into the neighbour's owned planes]
    //   pencil_forward  2-D FFT of the owned planes, packed per destination
    //                   rank into send (spec_local complex)
    //   [caller: all-to-all send -> recv (spec_pencil complex)]
    //   pencil_solve    x-FFT, influence (and x-derivative) multiply, inverse
    //                   x-FFT of the rank's y-rows -> A (and B for ik)
    //   [caller: all-to-all A, B back (same split sizes, reversed)]
    //   pencil_backward y/z-derivative spectra, inverse 2-D FFT into the
    //                   owned planes of fslab (nfields x slab_reals, interleaved)
    //   [caller: fill each halo of fslab from the neighbour's owned planes]
    //   pencil_phase_b  interpolation of the rank's atoms + combine: partial
    //                   u, F, energy (sum over ranks)
    void pencil_phase_a(long N, const double* pos, const double* q, int rank, int nranks,
                        double* slab, cudaStream_t s);
    void pencil_forward(int rank, int nranks, const double* slab, cufftDoubleComplex* send,
                        cudaStream_t s);
    void pencil_solve(int rank, int nranks, cufftDoubleComplex* recv, cufftDoubleComplex* A,
                      cufftDoubleComplex* B, cudaStream_t s);
    void pencil_backward(int rank, int nranks, const cufftDoubleComplex* A,
                         const cufftDoubleComplex* B, double* fslab, cudaStream_t s);
    void pencil_phase_b(int rank, int nranks, const double* fslab, double* u, double* F,
                        double* energy_dev, cudaStream_t s);

    // Distributed FFT with local inputs (esp_shard): the rank's atoms cover
    // only its slab, so N / box volume underestimates the density.  A hint
    // (atoms per unit volume of the whole system) replaces it in the cell-list
    // and staging-capacity choices, and the half-shell kernel then sizes its
    // staging without reading cell counts back (no host synchronisation:
    // the sharded evaluation can be captured in a CUDA graph).  0 = none.
    void set_density_hint(double rho) { density_hint_ = rho; }

    // Launch count of the last evaluate() (our kernels only, excluding cuFFT).
    int last_launches() const { return launches_; }
    // distributed-FFT K4 mode (fixed when the engine is built; see run_pair)
    bool pencil_half() const { return pencil_half_; }
    bool fused_xpass() const { return xpass_; }
    int pair_kernel() const { return pair_kernel_; }
    int spread_kernel() const { return spread_kernel_; }
    // Deterministic mode: bitwise-identical results run to run for the same
    // inputs (stable sorts instead of atomic ranks, full-list K4 without
    // partner REDs, K1 tiles flushed by bin colours with plain adds); the
    // reference's results are bit-identical for any thread count
    // (README.md:87-94).  Single-GPU evaluation paths.
    void set_deterministic(bool on);
    bool deterministic() const { return deterministic_; }
    static int pencil_half_env() {
        const char* e = std::getenv("ESP_PENCIL_HALF");
        return (e && std::atoi(e) == 0) ? 0 : 1;
    }
    // Ordered in-range pairs (0 < r < r_c) evaluated by the last pair-kernel
    // launch, counted on the device (synchronous read).
    unsigned long long last_pair_count() const;

private:
    void enqueue(long N, const double* pos, const double* q, double* u, double* F,
                 double* energy_dev, double* qsum_dev, cudaStream_t s, StageTimes* t,
                 double* u_out, double* F_out);
    void ensure_capacity(long N);
    void alloc_det(long n);
    void reconfigure(long N);
    void set_cells(int col_div);
    void alloc_cells();
    void alloc_bins(int sub);
    void prepare(long N, const double* pos, const double* q, double* qsum_dev, cudaStream_t s,
                 bool lean = false);
    void run_pair(long N, cudaStream_t s, int rank, int nranks, bool own_bins = false);
    bool run_pair_half(long N, cudaStream_t s, int rank = 0, int nranks = 1, bool own_bins = false);
    void run_grid(long N, cudaStream_t s, StageTimes* t);
    // n_k3 > 0: the K3 launch that follows is the enqueue's (N atoms), so the
    // tiled K3 may take the planar fields; -1 otherwise
    void spectral(const double* grid_in, cudaStream_t s, StageTimes* t, long n_k3);
    bool k3_planar_ = false;
    void run_spread(long N, cudaStream_t s, int rank, int nranks, double* grid,
                    const GridArgs* gslab = nullptr, long nreals = -1, int b0 = -1,
                    int b1 = -1);
    void finish(long N, int rank, int nranks, const double* fields, const GridArgs& g,
                double* u, double* F, double* energy_dev, cudaStream_t s, int b0 = -1,
                int b1 = -1);
    void pencil_plans(const PencilGeom& G);
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
    int sub_ = 2;               // sort sub-bins per spread-bin edge
    int nkeyB_ = 0;             // spread sort keys: nbin_ * sub_^3
    int W_ = 0;                 // spread tile edge (nodes)
    int RS_ = 0, PS_ = 0;       // padded tile strides
    long M_ = 0, Mh_ = 0;       // real grid size, half spectrum size
    int nfields_ = 4;           // 4 for ik, 1 for ad
    int pair_warps_ = 4;
    int pair_cap_ = 2048;
    int pair_lcap_ = 1024;      // per-warp candidate-list pieces
    int pM_ = 2, pMz_ = 4;      // fine stencil reach (columns, slices)
    int col_div_ = 2;           // column edge >= r_c / col_div_

    // tables on device
    double* d_win_ = nullptr;        // 3 x 4P x 13 phi, then 3 x 4P x 13 dphi
    double* d_influence_ = nullptr;  // Mh
    double* d_xi_ = nullptr;         // nx + ny + nz derivative multipliers (Nyquist = 0)
    bool xpass_ = false;             // 2-D cuFFT planes + k_xpass (x DFTs fused with K2)
    std::vector<int> xp_rad_;        // k_xpass Stockham radices (product n_x)
    double2* d_xtw_ = nullptr;       // n_x twiddles e^{-2 pi i t / n_x}
    double* d_fplanar_ = nullptr;    // k_xpass path: planar fields before interleaving

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
    double4* d_specres_ = nullptr;  // (u_s - q s0, F_s) in original order (K3 -> combine)
    bool deterministic_ = false;
    long det_cap_ = 0;              // deterministic mode: stable-sort scratch (atoms)
    int *d_det_keys_ = nullptr, *d_det_iota_ = nullptr, *d_det_perm_ = nullptr;
    void* d_det_tmp_ = nullptr;
    size_t det_tmp_bytes_ = 0;
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
    int* d_ovf_ = nullptr;
    double* d_acc_ = nullptr;           // half-shell K4: planar pair-sorted (u, F) sums, 4 x cap_              // half-shell K4: overflowed blocks (count, ids)
    long ovf_cap_ = 0;
    double density_hint_ = 0.0;        // set_density_hint
    bool pencil_half_ = true;           // distributed FFT with half-shell K4 (ESP_PENCIL_HALF=0: full
                                        // lists); local inputs return the ghost partner terms (dist.py)
    int tile_mode_ = -1;                // cluster-pair K4 (k_pair_tile) on one GPU: 1 always, otherwise never (ESP_PAIR_TILE)
    bool tmp_written_ = true;           // prepare() wrote the folded original-order copy d_tmp_
    const double* prep_q_ = nullptr;    // charges of the last prepare() (combine reads them when !tmp_written_)
    int spread_warp_mode_ = -1;         // warp-per-bin K1 (k_spread_warp): -1 auto (N >= 2^14), 0 never, 1 always (ESP_SPREAD_WARP)
    int phased_mode_ = 1;               // two-phase targets in k_pair_half (ESP_PAIR_PHASED=0: queue flushes inside the screening loop)
    int spread_kernel_ = -1;            // K1 kernel of the last launch (esp_plan_info.spread_kernel)
    int pair_kernel_ = -1;              // K4 kernel of the last launch (esp_plan_info.pair_kernel)
    int half_mode_ = 1;                 // half-shell K4: 0 never, 1 from kHalfMinN atoms, 2 always (ESP_PAIR_HALF)

    cufftHandle fwd_ = 0, inv_ = 0;
    // distributed-FFT plans, built for one (rank, nranks) at a time
    int pen_rank_ = -1, pen_nranks_ = 0;
    cufftHandle pen_f2d_ = 0, pen_x_ = 0, pen_i2d_ = 0;
    void* d_cufft_work_ = nullptr;
    cudaStream_t aux_ = nullptr, aux_hi_ = nullptr;
    cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
    cudaEvent_t ev_t_[8] = {};

    // CUDA graph of a full evaluation, keyed by its arguments
    struct GraphKey {
        long N;
        const void *pos, *q, *u, *F, *e, *qs, *uo, *Fo;
        bool operator==(const GraphKey& o) const {
            return N == o.N && pos == o.pos && q == o.q && u == o.u && F == o.F && e == o.e &&
                   qs == o.qs && uo == o.uo && Fo == o.Fo;
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
