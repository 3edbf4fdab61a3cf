/* esp_b200.h -- C ABI of the B200-native ESP (Ewald summation with prolates)
 * force evaluation.  This is the drop-in boundary: the reference solver is
 * the header-only C++ API in /root/reference/proj/include/esp (namespace
 * esp); include/esp/esp.hpp re-exposes that API on top of these entry
 * points, and INTEGRATION.md shows the ctypes binding.  Every entry point
 * below names the reference interface it replaces (file:line into
 * /root/reference/proj/include/esp).
 *
 * Conventions (kept from the reference, README.md:149-165):
 *   * positions are N x 3 doubles, row-major (the std::array<double,3>
 *     layout of ParticleSystem::pos, system.hpp:19-26); forces likewise;
 *   * Gaussian units, pair potential q_i q_j / (4 pi r); tinfoil boundary;
 *   * energy E = 1/2 sum_i q_i u_i;
 *   * fp64 throughout.
 * Results are not bitwise reproducible run to run (floating-point atomics
 * reorder sums on the GPU); they match the reference within the
 * tolerances stated in DESIGN.md.
 *
 * Errors: every function returns ESP_OK (0) or a positive status code and
 * sets a thread-local message readable with esp_last_error().  No C++
 * exception crosses this boundary.  The C++ header maps
 * ESP_ERR_INVALID_ARGUMENT -> std::invalid_argument and
 * ESP_ERR_NUMERICAL -> esp::NumericalError, as the reference throws them.
 *
 * Threading: a plan handle is not re-entrant; use one handle per host
 * thread.  There is no CPU fallback: device entry points fail with
 * ESP_ERR_CUDA when no GPU is usable.
 */
#ifndef ESP_B200_H
#define ESP_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ESP_OK 0
#define ESP_ERR_INVALID_ARGUMENT 1 /* std::invalid_argument in the reference */
#define ESP_ERR_NUMERICAL 2        /* esp::NumericalError (prolate.hpp:17-20) */
#define ESP_ERR_CUDA 3             /* CUDA / cuFFT runtime failure or no device */
#define ESP_ERR_NO_DEVICE 4        /* plan was created host-only (device < 0) */
#define ESP_ERR_INTERNAL 5

#define ESP_FAMILY_PSWF 0     /* SplitFamily::pswf (kernels.hpp:19) */
#define ESP_FAMILY_GAUSSIAN 1 /* SplitFamily::gaussian */
#define ESP_FORCE_IK 0        /* ForceMethod::ik (ewald.hpp:28), the default */
#define ESP_FORCE_AD 1        /* ForceMethod::ad */

typedef struct esp_plan esp_plan;

/* Overrides (ewald.hpp:38-47). Zero-initialise for the reference defaults. */
typedef struct {
    int nf;             /* 0 = auto; > 0 pins n_f in every dimension (even) */
    int P;              /* 0 = auto */
    double c1;          /* 0 = auto (PSWF window bandwidth) */
    int force_method;   /* ESP_FORCE_IK | ESP_FORCE_AD */
    int allow_degraded; /* build plans whose predicted error exceeds eps */
} esp_overrides;

/* Scalars of EwaldPlan (ewald.hpp:67-94) plus PlanStats (:61-65). */
typedef struct {
    int family, force_method, P;
    int nf[3], base_nf[3];
    double eps, r_c, shape, c1, chi0;
    double box[3], h[3], demand[3];
    double E_A, E_T, E_SI;
    double self_coef;       /* chi(0) / (4 pi r_c), ewald.hpp:609-615 */
    int n_split_coef;       /* prolate Legendre terms of the split */
    int n_window_coef;      /* prolate Legendre terms of the window */
    int pair_poly_degree;   /* degree of the device pair polynomials */
    double pair_fit_err;    /* their max deviation from the exact kernels */
    int device;             /* -1 for a host-only plan */
    int pair_cells[3];      /* GPU cell-list geometry */
    int pencil_half;        /* distributed FFT K4 mode, fixed at plan build
                             * (ESP_PENCIL_HALF, default 1): 1 = half-shell --
                             * ghost rows of esp_pencil_phase_b's output carry
                             * partner terms owed to their owners, which the
                             * caller must send back and add (see below);
                             * 0 = full lists, ghost rows are zero */
    int fused_xpass;        /* 1: the influence multiply and ik derivatives run
                             * inside the FFT's x pass (2-D cuFFT planes +
                             * k_xpass; even 5-smooth n_x <= 720, unless
                             * ESP_XPASS=0); 0: 3-D cuFFT + a multiply pass */
    int deterministic;      /* esp_plan_set_deterministic */
    int pair_kernel;        /* real-space kernel of the plan's last evaluation
                             * (selected per call from N and the density):
                             * -1 none yet, 0 full lists (k_pair), 1 half-shell
                             * (k_pair_half), 2 cluster pairs (k_pair_tile),
                             * 3 all pairs (box too small for the cell list) */
    int spread_kernel;      /* spreading kernel of the plan's last evaluation:
                             * -1 none yet, 0 k_spread (CTA per bin, thread per
                             * footprint node), 1 k_spread_warp (a warp per bin;
                             * single-GPU path, N >= 2^14, P in [5, 8];
                             * ESP_SPREAD_WARP=0/1 forces) */
} esp_plan_info;

/* Per-stage wall time in seconds (EnergyForces::timings keys,
 * ewald.hpp:628-634) plus the GPU binning stage.  Filled only by the
 * synchronous entry points when requested (stages are then serialised). */
typedef struct {
    double local, spread, fft, scale, ifft, interpolate, bin;
} esp_timings;

const char* esp_last_error(void);
const char* esp_version(void);
/* Number of visible CUDA devices (0 when none; never an error). */
int esp_device_count(void);

/* build_plan (ewald.hpp:355-405).  device >= 0 creates the device engine
 * on that CUDA device; device < 0 builds a host-only plan (parameter
 * selection and tables, no GPU needed).  *out owns all device state. */
int esp_plan_create(const double box[3], int family, double eps, double r_c,
                    const esp_overrides* ov, int device, esp_plan** out);
void esp_plan_destroy(esp_plan* plan);
int esp_plan_get_info(const esp_plan* plan, esp_plan_info* out);
/* Deterministic mode (default off): results bitwise identical run to run for
 * the same inputs on the same device, like the reference's results for any
 * thread count (README.md:87-94, test_cli.cpp:174-188).  Costs speed: stable
 * radix sorts instead of atomic counting-sort ranks, the full-list real-space
 * kernel (each atom's sum in a fixed order, no partner atomics), spreading
 * tiles flushed bin colour by colour with plain adds.  Single-GPU evaluation
 * entry points (esp_evaluate*, esp_local_sum, esp_spectral_sum, esp_spread);
 * the decompositions (phases, pencil, shard) keep their atomics.  Needs
 * n_f >= S + P + 2 (spread bin edge S, window P) in every dimension. */
int esp_plan_set_deterministic(esp_plan* plan, int on);

/* Plan tables (for parity checks).  influence: full nx*ny*nz reference
 * layout (gridder.hpp:162-210).  which: 0 Psi, 1 chi (16 x 13 Chebyshev-T
 * coefficients), 2 phi, 3 dphi of dimension dim (4P x 13).  prolate: which
 * -1 split, 0 window (Legendre coefficients a_k, psi(0) = 1). */
int esp_plan_get_influence(const esp_plan* plan, double* out);
int esp_plan_get_table(const esp_plan* plan, int which, int dim, double* out, int* nseg);
int esp_plan_get_prolate(const esp_plan* plan, int which, double* out, int* n);
/* Host evaluators of the plan kernels: what 0 Psi, 1 chi, 2 chihat_n,
 * 3 phi(dim 0), 4 dphi, 5 phi_hat, 6 local potential, 7 local radial force,
 * 8+d phi(dim d), 11+d dphi(dim d), 14+d phi_hat(dim d) (kernels.hpp:63-229). */
int esp_plan_eval_kernel(const esp_plan* plan, int what, long n, const double* x, double* y);

/* Unnormalised in-place 3-D DFT of nf[0]*nf[1]*nf[2] complex doubles
 * (interleaved re, im; row-major, z fastest) on the GPU: direction -1 forward
 * e^{-i}, +1 inverse e^{+i}; inverse(forward(g)) = N g (fft_forward /
 * fft_inverse, gridder.hpp:85-100, 153-154).  Host buffer, synchronous. */
int esp_fft3(const int nf[3], double* data, int direction, int device);

/* evaluate (ewald.hpp:619-649) on HOST buffers: copies in, evaluates on the
 * GPU, copies out, synchronises, checks charge neutrality.  Raises the
 * reference's errors: box mismatch -> INVALID_ARGUMENT, non-neutral ->
 * NUMERICAL.  timings may be NULL (then the stages overlap). */
int esp_evaluate(esp_plan* plan, const double box[3], long N, const double* pos,
                 const double* q, double* u, double* F, double* energy, esp_timings* timings);

/* Device-resident evaluate: all pointers are device pointers; energy_dev is
 * one device double; stream is a cudaStream_t (NULL = legacy default).
 * Asynchronous; charge neutrality is not checked here (see
 * esp_check_neutral). */
int esp_evaluate_device(esp_plan* plan, const double box[3], long N, const double* pos_dev,
                        const double* q_dev, double* u_dev, double* F_dev, double* energy_dev,
                        void* stream);

/* Slab-decomposed evaluation for nranks GPUs (one plan per rank; the ranks
 * may also be emulated sequentially on one GPU).  All pointers are device
 * pointers, asynchronous on `stream`.
 *   phase A: bins/sorts all N atoms (inputs replicated on every rank), sums
 *            the real-space part for the targets of this rank's x-slab and
 *            spreads this slab's atoms into grid_dev (nx*ny*nz reals).
 *   (caller: sum grid_dev over ranks, e.g. ncclAllReduce)
 *   phase B: FFT pipeline on the summed grid, interpolation and combine for
 *            this slab; u/F/energy receive this rank's PARTIAL sums (zero
 *            for atoms owned elsewhere).
 *   (caller: sum u, F, energy over ranks)
 * With nranks == 1 the two phases equal esp_evaluate_device. */
int esp_eval_phase_a(esp_plan* plan, const double box[3], long N, const double* pos_dev,
                     const double* q_dev, int rank, int nranks, double* grid_dev, void* stream);
int esp_eval_phase_b(esp_plan* plan, int rank, int nranks, const double* grid_dev, double* u_dev,
                     double* F_dev, double* energy_dev, void* stream);
/* Distributed-FFT evaluation: the charge grid and the
 * fields are distributed too -- rank r holds the x-planes [x0, x1) plus
 * `halo` planes on each side, and the spectrum's y-rows [y0, y1) between the
 * two transposes.  The caller moves data between the steps (NCCL over
 * NVLink on the GPU box); every pointer is a device pointer, complex buffers
 * are interleaved (re, im) doubles, all calls asynchronous on `stream`.
 *   esp_pencil_phase_a   bin/sort, real-space part of the rank's targets,
 *                        spread of its atoms into slab (slab_reals doubles,
 *                        planes x0-halo .. x1+halo-1)
 *   caller: send slab planes [0, halo) to rank r-1 and add them into its
 *           planes [x1-x0, x1-x0+halo); send planes [x1-x0+halo, x1-x0+2halo)
 *           to rank r+1 and add them into its planes [halo, 2halo) (periodic)
 *   esp_pencil_forward   2-D FFTs of the owned planes -> send (spec_local
 *                        complex; block for rank s = rows [y0(s), y1(s)))
 *   caller: all-to-all send -> recv (recv: spec_pencil complex; block from
 *           rank s = its planes [x0(s), x1(s)), in rank order)
 *   esp_pencil_solve     x-FFT, influence multiply, inverse x-FFT: recv
 *                        (clobbered) -> A, B (spec_pencil complex each; B
 *                        only for the ik force method, else may be NULL)
 *   caller: all-to-all A and B back (block for rank s = planes [x0(s), x1(s)))
 *   esp_pencil_backward  derivative spectra + inverse 2-D FFTs -> the owned
 *                        planes of fslab (nfields * slab_reals doubles, fields
 *                        interleaved per node)
 *   caller: fill fslab's halo planes from the neighbours' owned planes (the
 *           mirror of the first exchange, copying instead of adding)
 *   esp_pencil_phase_b   interpolation + combine for the rank's atoms:
 *                        partial u, F, energy (caller sums over ranks)
 * nranks >= 2; esp_pencil_geometry fails with INVALID_ARGUMENT when a rank
 * would own fewer x-planes than the halo.
 * Inputs: every rank passes either the whole system or only its own atoms
 * (ownership below) plus ghost atoms within r_c of its x-slab (the
 * neighbours' atoms, any order).  Outputs depend on esp_plan_info.pencil_half
 * (the same on every rank: it is fixed when the plan is built):
 *   pencil_half = 0: a rank computes u, F and the energy share of the atoms
 *     it owns, zero for the others.
 *   pencil_half = 1 (default): each unordered real-space pair is evaluated
 *     once, on the rank owning its base atom, and the partner's terms land in
 *     the partner's row -- also when the partner is another rank's atom.
 *     With replicated inputs, summing u and F over ranks (all-reduce) gives
 *     the result.  With local inputs, the ghost rows hold terms owed to the
 *     ghosts' owners: send each ghost row (u, Fx, Fy, Fz) back to the rank
 *     that sent the ghost and add it into that atom's row (the reverse of the
 *     ghost exchange); then E = 1/2 sum q_i u_i over the owned atoms
 *     (ewald.hpp:641-647) -- the energy output of phase_b does not include
 *     the returned terms. */
typedef struct esp_pencil_info {
    int nranks, rank;
    int halo;          /* planes exchanged with each x-neighbour */
    int x0, x1;        /* owned real-space x-planes */
    int y0, y1;        /* owned spectral y-rows */
    int nfields;       /* 4 (ik) or 1 (ad) */
    int nf[3];         /* grid size */
    /* atom ownership: an atom belongs to the rank whose planes [x0, x1)
     * hold clamp(floor(fold(x)/hx), 0, nf[0]-1) (fold as system.hpp:29-36)
     * -- the rank computes u and F of exactly those atoms; it processes the
     * spread bins [bx0, bx1) of edge S (of nbx) that intersect its planes */
    double hx;
    int S, nbx, bx0, bx1;
    long slab_reals;   /* (x1-x0+2 halo)*ny*nz */
    long spec_local;   /* (x1-x0)*ny*(nz/2+1) complex */
    long spec_pencil;  /* nx*(y1-y0)*(nz/2+1) complex */
} esp_pencil_info;
int esp_pencil_geometry(const esp_plan* plan, int rank, int nranks, esp_pencil_info* out);
int esp_pencil_phase_a(esp_plan* plan, const double box[3], long N, const double* pos_dev,
                       const double* q_dev, int rank, int nranks, double* slab_dev, void* stream);
int esp_pencil_forward(esp_plan* plan, int rank, int nranks, const double* slab_dev,
                       double* send_dev, void* stream);
int esp_pencil_solve(esp_plan* plan, int rank, int nranks, double* recv_dev, double* A_dev,
                     double* B_dev, void* stream);
int esp_pencil_backward(esp_plan* plan, int rank, int nranks, const double* A_dev,
                        const double* B_dev, double* fslab_dev, void* stream);
int esp_pencil_phase_b(esp_plan* plan, int rank, int nranks, const double* fslab_dev,
                       double* u_dev, double* F_dev, double* energy_dev, void* stream);

/* Direct (mesh-free) Ewald summation on the GPU: one pass of the reference's
 * ground-truth solver (direct_ewald_pass, reference.hpp:42-206) at splitting
 * width `lambda` (<= 0: min(L)/6, reference.hpp:222), same stopping rules
 * (tol/10 per image shell and per reciprocal mode).  Host pointers.  targets:
 * ntarget atom indices whose u and F are computed (every atom remains a
 * source), or NULL for all N atoms -- the subset form lifts the reference's
 * N <= 1e4 cap (reference.hpp:213) so the ESP path can be certified at the
 * benchmark sizes.  u: ntarget (or N), F: ntarget*3 (or N*3); energy (may be
 * NULL) = 1/2 sum q u when targets == NULL, NaN otherwise.  tol >= 1e-12,
 * neutral systems only (NUMERICAL otherwise). */
typedef struct esp_direct_info {
    double lambda;
    int real_shells;
    int recip_kmax;
    double tail_bound;
} esp_direct_info;
int esp_direct_ewald(const double box[3], long N, const double* pos, const double* q,
                     long ntarget, const long* targets, double tol, double lambda, double* u,
                     double* F, double* energy, esp_direct_info* info, int device);

/* Number of reals in the charge grid (nx*ny*nz) for sizing grid_dev. */
long esp_grid_size(const esp_plan* plan);

/* require_neutral (system.hpp:39-47) on host data. */
int esp_check_neutral(long N, const double* q);

/* Parts of the hot path on HOST buffers (synchronous). */
int esp_local_sum(esp_plan* plan, const double box[3], long N, const double* pos,
                  const double* q, double* u, double* F);          /* ewald.hpp:419-515 */
/* ewald.hpp:524-604; timings (may be NULL) receives the grid-pipeline stage
 * times (spread, fft, scale, ifft, interpolate; the stages then run
 * serialised on one stream), like the reference's optional timings map. */
int esp_spectral_sum(esp_plan* plan, const double box[3], long N, const double* pos,
                     const double* q, double* u, double* F, esp_timings* timings);
int esp_self_correction(const esp_plan* plan, long N, const double* q, double* out);
                                                                    /* ewald.hpp:609-615 */
int esp_spread(esp_plan* plan, long N, const double* pos, const double* q, double* grid);
                                                                    /* gridder.hpp:215-241 */
int esp_interpolate(esp_plan* plan, long N, const double* pos, const double* grid,
                    double* out);                                   /* gridder.hpp:244-277 */
int esp_interpolate_gradient(esp_plan* plan, long N, const double* pos, const double* grid,
                             double* out);                          /* gridder.hpp:280-314 */

/* Kernel launches issued by the last evaluate (our kernels, excluding
 * cuFFT and CUB scans). */
int esp_last_launch_count(const esp_plan* plan);

/* Ordered in-range pairs (0 < r < r_c) counted on the device by the last
 * pair-sum launch; the algorithmic work unit of the pair kernel
 * (96 flops per unordered pair).  Synchronises. */
int esp_last_pair_count(esp_plan* plan, unsigned long long* ordered_pairs);

/* Measured fp64 FMA-pipe throughput of a device in TFLOP/s (DFMA
 * microbenchmark; the fp64 roofline denominator). */
int esp_fp64_peak(int device, double* tflops);

/* Ordered pairs per second of the pair evaluation alone (operands in
 * registers, no neighbour search): the ceiling of K4's inner work. */
int esp_pair_eval_rate(esp_plan* plan, double* pairs_per_s);

/* ---- Sharded evaluation over the GPUs of one box -----------
 * One process per GPU, each with its own plan (same box / eps / r_c / family
 * / overrides on every rank, device = that process's GPU).  The system is
 * split into x-slabs by grid plane (the distributed-FFT decomposition of
 * esp_pencil_geometry): rank r passes ONLY the atoms it owns (partition with
 * esp_shard_owner) and gets back u and F of those atoms and the total energy.
 * Inside one esp_shard_evaluate call: ghost atoms within r_c of the slab
 * faces are exchanged with the two x-neighbours (fixed-capacity NCCL
 * send/recv), the pencil phases run, the spread halos and field halos go to
 * the neighbours, the half spectrum is transposed twice by grouped NCCL
 * send/recv (all-to-all), the half-shell real-space partner terms of the
 * ghosts go back to their owners, and the energy is all-reduced.  Everything
 * is asynchronous on `stream`, with no host synchronisation: the call can be
 * captured in a CUDA graph.  Replaces the single-process esp::evaluate
 * (ewald.hpp:619-649) for systems sharded over GPUs; API shape README.md:58-64.
 * The results equal esp_evaluate on the whole system up to summation order.
 *
 * NCCL is loaded at run time (libnccl.so.2). */
typedef struct esp_shard esp_shard;
typedef struct esp_shard_info_t {
    int rank, nranks;
    int x0, x1;             /* owned grid planes */
    double X0, X1;          /* owned slab in x (folded coordinates) */
    long max_own_atoms;     /* capacity for own atoms */
    long ghost_capacity;    /* ghost atoms per slab face (2x for two ranks) */
    long local_atoms;       /* own + ghost capacity: the rank's local system */
    int pencil_half;        /* real-space pairs once (ghost terms returned) */
    int nccl;               /* 1: NCCL communicator, 0: emulation member */
} esp_shard_info_t;

/* A new NCCL unique id (128 bytes) -- made on one rank and shared with the
 * others by the caller (e.g. a torch.distributed broadcast). */
int esp_shard_unique_id(void* id128);
/* Collective over nranks >= 2 processes when nccl_id != NULL
 * (ncclCommInitRank on the plan's device).  nccl_id == NULL makes an
 * emulation member for esp_shard_evaluate_emulated (all ranks' shards in one
 * process on one GPU, messages moved by device copies: tests).
 * max_own_atoms: upper bound of the atoms this rank will pass;
 * ghost_capacity: atoms per slab face (0 = from max_own_atoms and the slab
 * width, +30 %).  INVALID_ARGUMENT when a slab is narrower than r_c. */
int esp_shard_create(esp_plan* plan, const void* nccl_id, int rank, int nranks,
                     long max_own_atoms, long ghost_capacity, esp_shard** out);
void esp_shard_destroy(esp_shard* shard);
int esp_shard_info(const esp_shard* shard, esp_shard_info_t* info);
/* Owner rank of each atom (host positions N x 3, any image): the rank whose
 * planes hold clamp(floor(fold(x) / hx), 0, nx - 1). */
int esp_shard_owner(const esp_plan* plan, int nranks, long N, const double* pos, int* owner);
/* One sharded evaluation (collective: every rank calls it for the same step).
 * Device pointers: pos (n_own x 3), q (n_own) of this rank's atoms; out u
 * (n_own), F (n_own x 3), energy (1 double: the TOTAL energy, all-reduced).
 * A ghost-capacity overflow or a non-owned input atom is detected on the
 * device and reported by the next call (or esp_shard_check) as
 * ESP_ERR_NUMERICAL / ESP_ERR_INVALID_ARGUMENT. */
int esp_shard_evaluate(esp_shard* shard, const double box[3], long n_own, const double* pos_dev,
                       const double* q_dev, double* u_dev, double* F_dev, double* energy_dev,
                       void* stream);
/* All ranks of a decomposition in this process (emulation members, one GPU),
 * executed in lockstep; per-rank argument arrays. */
int esp_shard_evaluate_emulated(esp_shard* const* shards, int nranks, const double box[3],
                                const long* n_own, const double* const* pos_dev,
                                const double* const* q_dev, double* const* u_dev,
                                double* const* F_dev, double* const* energy_dev, void* stream);
/* Synchronises and reports the device-side error flags of the last call. */
int esp_shard_check(esp_shard* shard);
/* Host-buffer forms of the two above (synchronous): the own atoms are copied
 * into device buffers held by the shard (n_own <= max_own_atoms), the
 * evaluation runs, u / F / the total energy are copied back, and the device
 * flags are reported as by esp_shard_check.  The emulated form takes per-rank
 * host arrays and one energy. */
int esp_shard_evaluate_host(esp_shard* shard, const double box[3], long n_own, const double* pos,
                            const double* q, double* u, double* F, double* energy);
int esp_shard_evaluate_emulated_host(esp_shard* const* shards, int nranks, const double box[3],
                                     const long* n_own, const double* const* pos,
                                     const double* const* q, double* const* u,
                                     double* const* F, double* energy);

#ifdef __cplusplus
}
#endif

#endif /* ESP_B200_H */
