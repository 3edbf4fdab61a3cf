// Sharded ESP evaluation over the GPUs of one box, behind the C
// ABI: esp_shard_* in include/esp_b200.h.
//
// One process per GPU.  The system is split into x-slabs by grid plane (the
// distributed-FFT decomposition of engine.cu, pencil_geometry): every rank
// holds only the atoms it owns, and one esp_shard_evaluate call per rank and
// step runs, all on the caller's stream and without host synchronisation (so
// the whole call can be captured in a CUDA graph):
//   0  ghost pack      atoms within r_c of the slab faces -> fixed-capacity
//                      messages (count in the header; overflow flagged)
//      ghost exchange  NCCL send/recv with the two x-neighbours
//   1  ghost fill      own atoms + ghosts (+ q = 0 placeholders up to the
//                      capacity) -> the rank's local system; pencil_phase_a
//                      (bin/sort, half-shell K4 of the owned targets, K1 of the
//                      owned atoms into the slab + halos)
//      halo exchange   send/recv of the spread halos (added below)
//   2  halo add        + pencil_forward (2-D D2Z of the owned planes, packed)
//      all-to-all      grouped send/recv (forward transpose)
//   3  pencil_solve    x-FFT, influence multiply, x-derivative, inverse x-FFT
//      all-to-all      back (A, and B for ik)
//   4  pencil_backward y/z derivative spectra, inverse 2-D Z2D -> field slab
//      halo fill       send/recv of the field halos (copied)
//   5  pencil_phase_b  K3 + combine for the owned atoms
//      ghost return    (half-shell K4) the ghost rows' partner terms go back to
//                      the ranks that own those atoms
//   6  ghost add       returned terms into the owned rows; u, F out;
//                      E = 1/2 sum q u over the owned atoms
//      all-reduce      of E (one double)
// The same staged code runs in two transports: NCCL (one rank per process,
// the data plane over NVLink / NVSwitch) and an emulation that executes the
// ranks of one process in lockstep on one GPU, moving each message with a
// device copy (esp_shard_evaluate_emulated; what the single-GPU tests use --
// no rank ever waits on another rank's kernels).  Message pairing follows
// NCCL's rule: between two ranks, the k-th send matches the k-th receive.
//
// Reference: esp::evaluate (ewald.hpp:619-649) is the single-process
// computation this reproduces; API shape README.md:58-64.

#include "capi_internal.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

namespace {

using espc::cuda_ok;
using espc::engine;
using espc::guarded;

// ---- NCCL, resolved at run time (dlopen "libnccl.so.2": the copy a process
// already loaded, e.g. torch's, or the system one) -------------------------
struct Nccl {
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;

    static Nccl& get() {
        static Nccl n;
        static std::once_flag once;
        static std::string err;
        std::call_once(once, [] {
            void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
            if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
            if (!h) {
                err = std::string("NCCL not available: ") + dlerror();
                return;
            }
            auto sym = [&](const char* s) {
                void* p = dlsym(h, s);
                if (!p) err = std::string("NCCL symbol missing: ") + s;
                return p;
            };
            n.getUniqueId = reinterpret_cast<decltype(n.getUniqueId)>(sym("ncclGetUniqueId"));
            n.commInitRank = reinterpret_cast<decltype(n.commInitRank)>(sym("ncclCommInitRank"));
            n.commDestroy = reinterpret_cast<decltype(n.commDestroy)>(sym("ncclCommDestroy"));
            n.groupStart = reinterpret_cast<decltype(n.groupStart)>(sym("ncclGroupStart"));
            n.groupEnd = reinterpret_cast<decltype(n.groupEnd)>(sym("ncclGroupEnd"));
            n.send = reinterpret_cast<decltype(n.send)>(sym("ncclSend"));
            n.recv = reinterpret_cast<decltype(n.recv)>(sym("ncclRecv"));
            n.allReduce = reinterpret_cast<decltype(n.allReduce)>(sym("ncclAllReduce"));
            n.errorString = reinterpret_cast<decltype(n.errorString)>(sym("ncclGetErrorString"));
        });
        if (!err.empty()) throw espb::CudaError(err);
        return n;
    }
    void ok(ncclResult_t r, const char* what) const {
        if (r != ncclSuccess)
            throw espb::CudaError(std::string(what) + ": " + (errorString ? errorString(r) : "NCCL error"));
    }
};

// ---- kernels ----------------------------------------------------------------

__device__ __forceinline__ double fold_x(double x, double L) {
    // system.hpp:29-36
    x -= L * floor(x / L);
    if (x >= L) x = 0.0;
    return x;
}

struct PackArgs {
    long n;
    const double* pos;  // n x 3
    const double* q;
    double box[3];
    double X0, X1, reach;  // slab [X0, X1) in x, ghost reach
    double hx;
    int nx, x0, x1;        // owned planes (ownership check)
    int union_left;        // two ranks: one message (atoms near either face)
    double* sendL;         // [count | capL x (x, y, z, q)]
    double* sendR;
    int* idxL;
    int* idxR;
    int capL, capR;
    int* cnt;              // [2] counters (zero at entry)
    int* flags;            // bit 0 ghost overflow, bit 1 atom outside the rank's planes
};

__global__ void k_ghost_pack(PackArgs a) {
    const long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
    if (i >= a.n) return;
    const double x = fold_x(a.pos[3 * i], a.box[0]);
    const double y = fold_x(a.pos[3 * i + 1], a.box[1]);
    const double z = fold_x(a.pos[3 * i + 2], a.box[2]);
    const double qi = a.q[i];
    const int l = min(max(static_cast<int>(floor(x / a.hx)), 0), a.nx - 1);
    if (l < a.x0 || l >= a.x1) atomicOr(a.flags, 2);
    const bool toL = x - a.X0 <= a.reach, toR = a.X1 - x <= a.reach;
    auto put = [&](double* buf, int* idx, int* c, int cap) {
        const int k = atomicAdd(c, 1);
        if (k < cap) {
            double* r = buf + 1 + 4 * static_cast<long>(k);
            r[0] = x;
            r[1] = y;
            r[2] = z;
            r[3] = qi;
            idx[k] = static_cast<int>(i);
        } else {
            atomicOr(a.flags, 1);
        }
    };
    if (a.union_left) {
        if (toL || toR) put(a.sendL, a.idxL, a.cnt, a.capL);
    } else {
        if (toL) put(a.sendL, a.idxL, a.cnt, a.capL);
        if (toR) put(a.sendR, a.idxR, a.cnt + 1, a.capR);
    }
}

__global__ void k_ghost_count(double* sendL, double* sendR, const int* cnt, int capL, int capR) {
    if (threadIdx.x == 0) sendL[0] = static_cast<double>(min(cnt[0], capL));
    if (threadIdx.x == 1 && sendR) sendR[0] = static_cast<double>(min(cnt[1], capR));
}

// local system: [own atoms | ghosts from the right (capR) | from the left
// (capL)]; empty ghost slots are q = 0 copies of a received ghost (another
// rank's planes: neither spread nor interpolated here; every pair with them
// is zero) or, with no ghosts at all, of an own atom.
__global__ void k_ghost_fill(long n_own, const double* __restrict__ pos, const double* __restrict__ q,
                             const double* __restrict__ gR, int capR, const double* __restrict__ gL,
                             int capL, double* __restrict__ pos_l, double* __restrict__ q_l) {
    const long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
    const long n = n_own + capR + capL;
    if (i >= n) return;
    if (i < n_own) {
        pos_l[3 * i] = pos[3 * i];
        pos_l[3 * i + 1] = pos[3 * i + 1];
        pos_l[3 * i + 2] = pos[3 * i + 2];
        q_l[i] = q[i];
        return;
    }
    const int cR = capR > 0 ? static_cast<int>(gR[0]) : 0;
    const int cL = capL > 0 ? static_cast<int>(gL[0]) : 0;
    long k = i - n_own;
    const double* row = nullptr;
    bool real = false;
    if (k < capR) {
        if (k < cR) {
            row = gR + 1 + 4 * k;
            real = true;
        }
    } else {
        k -= capR;
        if (k < cL) {
            row = gL + 1 + 4 * k;
            real = true;
        }
    }
    if (!row) {
        if (cR > 0) row = gR + 1 + 4 * (k % cR);
        else if (cL > 0) row = gL + 1 + 4 * (k % cL);
    }
    if (row) {
        pos_l[3 * i] = row[0];
        pos_l[3 * i + 1] = row[1];
        pos_l[3 * i + 2] = row[2];
        q_l[i] = real ? row[3] : 0.0;
    } else {
        const long o = n_own > 0 ? k % n_own : 0;
        pos_l[3 * i] = n_own > 0 ? pos[3 * o] : 0.0;
        pos_l[3 * i + 1] = n_own > 0 ? pos[3 * o + 1] : 0.0;
        pos_l[3 * i + 2] = n_own > 0 ? pos[3 * o + 2] : 0.0;
        q_l[i] = 0.0;
    }
}

__global__ void k_add(long n, double* __restrict__ dst, const double* __restrict__ src) {
    const long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
    if (i < n) dst[i] += src[i];
}

// partner terms returned for the atoms this rank sent (idx[k], k < count)
__global__ void k_ghost_back(const double* __restrict__ sent, const int* __restrict__ idx, int cap,
                             const double* __restrict__ bu, const double* __restrict__ bF,
                             double* __restrict__ u, double* __restrict__ F) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int c = min(static_cast<int>(sent[0]), cap);
    if (k >= c) return;
    const int i = idx[k];
    u[i] += bu[k];
    F[3 * i] += bF[3 * k];
    F[3 * i + 1] += bF[3 * k + 1];
    F[3 * i + 2] += bF[3 * k + 2];
}

// owned rows out + E partial = 1/2 sum q u (ewald.hpp:641-647)
__global__ void __launch_bounds__(256) k_own_out(long n, const double* __restrict__ ul,
                                                 const double* __restrict__ Fl,
                                                 const double* __restrict__ q,
                                                 double* __restrict__ u, double* __restrict__ F,
                                                 double* __restrict__ e) {
    const long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
    double v = 0.0;
    if (i < n) {
        u[i] = ul[i];
        F[3 * i] = Fl[3 * i];
        F[3 * i + 1] = Fl[3 * i + 1];
        F[3 * i + 2] = Fl[3 * i + 2];
        v = 0.5 * q[i] * ul[i];
    }
    __shared__ double part[8];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < 8; ++w) s += part[w];
        if (s != 0.0) atomicAdd(e, s);
    }
}

unsigned blocks(long n, int b) { return static_cast<unsigned>(std::max<long>(1, (n + b - 1) / b)); }

struct Msg {
    int peer;
    void* buf;     // send: source, recv: destination
    size_t bytes;
};

double* dmalloc(long n) {
    double* p = nullptr;
    cuda_ok(cudaMalloc(&p, sizeof(double) * std::max<long>(n, 1)), "cudaMalloc (shard)");
    return p;
}

}  // namespace

struct esp_shard {
    esp_plan* plan = nullptr;
    int rank = 0, nranks = 1;
    ncclComm_t comm = nullptr;  // null: emulation member
    std::vector<espb::PencilGeom> geo;
    long n_own_cap = 0, gcap = 0;
    int capL = 0, capR = 0;      // my ghost messages (to left / to right)
    int regR = 0, regL = 0;      // ghost regions (from right / from left)
    long ncap = 0;               // local system size
    int left = 0, right = 0;
    double X0 = 0, X1 = 0, reach = 0;
    bool half = true;
    // buffers
    double *pos_l = nullptr, *q_l = nullptr, *sendL = nullptr, *sendR = nullptr;
    double *gR = nullptr, *gL = nullptr;
    int *idxL = nullptr, *idxR = nullptr, *cnt = nullptr, *flags = nullptr;
    int* h_flags = nullptr;  // pinned copy
    double *slab = nullptr, *hR = nullptr, *hL = nullptr, *send = nullptr, *recv = nullptr;
    double *A = nullptr, *B = nullptr, *A2 = nullptr, *B2 = nullptr, *fslab = nullptr;
    double *ul = nullptr, *Fl = nullptr, *e_part = nullptr;
    double *bRu = nullptr, *bRF = nullptr, *bLu = nullptr, *bLF = nullptr;
    // host-buffer entry points: device copies of the own atoms and outputs
    // (allocated on first use, n_own_cap atoms)
    double *hpos = nullptr, *hq = nullptr, *hu = nullptr, *hF = nullptr, *he = nullptr;
    void host_buffers() {
        if (hpos) return;
        hpos = dmalloc(3 * n_own_cap);
        hq = dmalloc(n_own_cap);
        hu = dmalloc(n_own_cap);
        hF = dmalloc(3 * n_own_cap);
        he = dmalloc(1);
    }
    // current call
    long n_own = 0;
    const double *pos = nullptr, *q = nullptr;
    double *u = nullptr, *F = nullptr, *energy = nullptr;

    ~esp_shard() {
        if (plan && plan->device >= 0) cudaSetDevice(plan->device);
        for (double* p : {pos_l, q_l, sendL, sendR, gR, gL, slab, hR, hL, send, recv, A, B, A2, B2,
                          fslab, ul, Fl, e_part, bRu, bRF, bLu, bLF, hpos, hq, hu, hF, he})
            cudaFree(p);
        for (int* p : {idxL, idxR, cnt, flags}) cudaFree(p);
        if (h_flags) cudaFreeHost(h_flags);
        if (comm) {
            try {
                Nccl::get().commDestroy(comm);
            } catch (...) {
            }
        }
    }

    const espb::PencilGeom& me() const { return geo[rank]; }
    long plane(int nfields = 1) const {
        return static_cast<long>(plan->plan.nf[1]) * plan->plan.nf[2] * nfields;
    }
    long nxl(int r) const { return geo[r].x1 - geo[r].x0; }
    long nyl(int r) const { return geo[r].y1 - geo[r].y0; }
    long nzh() const { return plan->plan.nf[2] / 2 + 1; }

    void setup() {
        const espb::Plan& P = plan->plan;
        geo.clear();
        for (int r = 0; r < nranks; ++r) geo.push_back(espb::pencil_geometry(P, r, nranks));
        left = (rank + nranks - 1) % nranks;
        right = (rank + 1) % nranks;
        const double hx = geo[0].hx;
        for (int r = 0; r < nranks; ++r) {
            const double a = geo[r].x0 * hx, b = geo[r].x1 >= P.nf[0] ? P.box[0] : geo[r].x1 * hx;
            if (b - a < P.r_c * (1.0 + 1e-9))
                throw espb::InvalidArgument("sharded evaluation: rank " + std::to_string(r) +
                                            " slab is narrower than r_c; use fewer ranks");
        }
        X0 = me().x0 * hx;
        X1 = me().x1 >= P.nf[0] ? P.box[0] : me().x1 * hx;
        reach = P.r_c * (1.0 + 1e-9) + 1e-12 * P.box[0];
        const bool two = nranks == 2;
        capL = static_cast<int>(two ? 2 * gcap : gcap);
        capR = static_cast<int>(two ? 0 : gcap);
        regR = capL;  // the right neighbour's capL
        regL = capR;
        ncap = n_own_cap + regR + regL;
        half = engine(plan).pencil_half();
        const espb::PencilGeom& g = me();
        const int nf = g.nfields;
        pos_l = dmalloc(3 * ncap);
        q_l = dmalloc(ncap);
        sendL = dmalloc(1 + 4L * capL);
        sendR = dmalloc(1 + 4L * capR);
        gR = dmalloc(1 + 4L * regR);
        gL = dmalloc(1 + 4L * regL);
        cuda_ok(cudaMemset(sendR, 0, sizeof(double)), "memset");
        cuda_ok(cudaMemset(gL, 0, sizeof(double)), "memset");
        cuda_ok(cudaMemset(gR, 0, sizeof(double)), "memset");
        cuda_ok(cudaMalloc(&idxL, sizeof(int) * std::max(capL, 1)), "cudaMalloc");
        cuda_ok(cudaMalloc(&idxR, sizeof(int) * std::max(capR, 1)), "cudaMalloc");
        cuda_ok(cudaMalloc(&cnt, sizeof(int) * 2), "cudaMalloc");
        cuda_ok(cudaMalloc(&flags, sizeof(int)), "cudaMalloc");
        cuda_ok(cudaMemset(flags, 0, sizeof(int)), "memset");
        cuda_ok(cudaMallocHost(&h_flags, sizeof(int)), "cudaMallocHost");
        *h_flags = 0;
        slab = dmalloc(g.slab_reals);
        hR = dmalloc(g.halo * plane());
        hL = dmalloc(g.halo * plane());
        send = dmalloc(2 * g.spec_local);
        recv = dmalloc(2 * g.spec_pencil);
        A = dmalloc(2 * g.spec_pencil);
        A2 = dmalloc(2 * g.spec_local);
        if (nf == 4) {
            B = dmalloc(2 * g.spec_pencil);
            B2 = dmalloc(2 * g.spec_local);
        }
        fslab = dmalloc(static_cast<long>(nf) * g.slab_reals);
        ul = dmalloc(ncap);
        Fl = dmalloc(3 * ncap);
        e_part = dmalloc(1);
        bRu = dmalloc(capR);
        bRF = dmalloc(3L * capR);
        bLu = dmalloc(capL);
        bLF = dmalloc(3L * capL);
        // the local inputs cover one slab: the engine takes the system's mean
        // density from the caller's bound instead (no read-backs)
        engine(plan).set_density_hint(static_cast<double>(n_own_cap) * nranks /
                                      (P.box[0] * P.box[1] * P.box[2]));
    }

    // ---- stages: compute on the stream, then the messages of the exchange
    // that follows (sends and receives in NCCL pairing order) ----
    void stage0(cudaStream_t s, std::vector<Msg>& snd, std::vector<Msg>& rcv) {
        const espb::Plan& P = plan->plan;
        cuda_ok(cudaMemsetAsync(cnt, 0, 2 * sizeof(int), s), "memset");
        cuda_ok(cudaMemsetAsync(flags, 0, sizeof(int), s), "memset");
        PackArgs a{};
        a.n = n_own;
        a.pos = pos;
        a.q = q;
        for (int d = 0; d < 3; ++d) a.box[d] = P.box[d];
        a.X0 = X0;
        a.X1 = X1;
        a.reach = reach;
        a.hx = geo[0].hx;
        a.nx = P.nf[0];
        a.x0 = me().x0;
        a.x1 = me().x1;
        a.union_left = nranks == 2;
        a.sendL = sendL;
        a.sendR = sendR;
        a.idxL = idxL;
        a.idxR = idxR;
        a.capL = capL;
        a.capR = capR;
        a.cnt = cnt;
        a.flags = flags;
        if (n_own > 0) k_ghost_pack<<<blocks(n_own, 256), 256, 0, s>>>(a);
        k_ghost_count<<<1, 32, 0, s>>>(sendL, capR > 0 ? sendR : nullptr, cnt, capL, capR);
        cuda_ok(cudaGetLastError(), "ghost pack");
        snd = {{left, sendL, sizeof(double) * (1 + 4L * capL)}};
        if (capR > 0) snd.push_back({right, sendR, sizeof(double) * (1 + 4L * capR)});
        rcv = {{right, gR, sizeof(double) * (1 + 4L * regR)}};
        if (regL > 0) rcv.push_back({left, gL, sizeof(double) * (1 + 4L * regL)});
    }
    void stage1(cudaStream_t s, std::vector<Msg>& snd, std::vector<Msg>& rcv) {
        k_ghost_fill<<<blocks(ncap, 256), 256, 0, s>>>(n_own, pos, q, gR, regR, gL, regL, pos_l, q_l);
        cuda_ok(cudaGetLastError(), "ghost fill");
        engine(plan).pencil_phase_a(n_own + regR + regL, pos_l, q_l, rank, nranks, slab, s);
        const long h = me().halo, n = nxl(rank), pl = plane();
        snd = {{left, slab, sizeof(double) * h * pl}, {right, slab + (n + h) * pl, sizeof(double) * h * pl}};
        rcv = {{right, hR, sizeof(double) * h * pl}, {left, hL, sizeof(double) * h * pl}};
    }
    void stage2(cudaStream_t s, std::vector<Msg>& snd, std::vector<Msg>& rcv) {
        const long h = me().halo, n = nxl(rank), pl = plane();
        k_add<<<blocks(h * pl, 256), 256, 0, s>>>(h * pl, slab + n * pl, hR);
        k_add<<<blocks(h * pl, 256), 256, 0, s>>>(h * pl, slab + h * pl, hL);
        cuda_ok(cudaGetLastError(), "halo add");
        engine(plan).pencil_forward(rank, nranks, slab, reinterpret_cast<cufftDoubleComplex*>(send), s);
        snd.clear();
        rcv.clear();
        long so = 0, ro = 0;
        for (int t = 0; t < nranks; ++t) {
            const long ns = 2 * nxl(rank) * nyl(t) * nzh(), nr = 2 * nxl(t) * nyl(rank) * nzh();
            snd.push_back({t, send + so, sizeof(double) * ns});
            rcv.push_back({t, recv + ro, sizeof(double) * nr});
            so += ns;
            ro += nr;
        }
    }
    void stage3(cudaStream_t s, std::vector<Msg>& snd, std::vector<Msg>& rcv) {
        engine(plan).pencil_solve(rank, nranks, reinterpret_cast<cufftDoubleComplex*>(recv),
                                  reinterpret_cast<cufftDoubleComplex*>(A),
                                  reinterpret_cast<cufftDoubleComplex*>(B), s);
        snd.clear();
        rcv.clear();
        for (double* buf : {A, B}) {
            if (!buf) continue;
            double* out = buf == A ? A2 : B2;
            long so = 0, ro = 0;
            for (int t = 0; t < nranks; ++t) {
                const long ns = 2 * nxl(t) * nyl(rank) * nzh(), nr = 2 * nxl(rank) * nyl(t) * nzh();
                snd.push_back({t, buf + so, sizeof(double) * ns});
                rcv.push_back({t, out + ro, sizeof(double) * nr});
                so += ns;
                ro += nr;
            }
        }
    }
    void stage4(cudaStream_t s, std::vector<Msg>& snd, std::vector<Msg>& rcv) {
        engine(plan).pencil_backward(rank, nranks, reinterpret_cast<const cufftDoubleComplex*>(A2),
                                     reinterpret_cast<const cufftDoubleComplex*>(B2), fslab, s);
        const long h = me().halo, n = nxl(rank), pl = plane(me().nfields);
        snd = {{left, fslab + h * pl, sizeof(double) * h * pl}, {right, fslab + n * pl, sizeof(double) * h * pl}};
        rcv = {{right, fslab + (n + h) * pl, sizeof(double) * h * pl}, {left, fslab, sizeof(double) * h * pl}};
    }
    void stage5(cudaStream_t s, std::vector<Msg>& snd, std::vector<Msg>& rcv) {
        engine(plan).pencil_phase_b(rank, nranks, fslab, ul, Fl, e_part, s);
        snd.clear();
        rcv.clear();
        if (!half) return;
        // ghost rows from the right go back right, from the left back left
        const long oR = n_own, oL = n_own + regR;
        if (regR > 0) {
            snd.push_back({right, ul + oR, sizeof(double) * regR});
            snd.push_back({right, Fl + 3 * oR, sizeof(double) * 3 * regR});
        }
        if (regL > 0) {
            snd.push_back({left, ul + oL, sizeof(double) * regL});
            snd.push_back({left, Fl + 3 * oL, sizeof(double) * 3 * regL});
        }
        if (capR > 0) {
            rcv.push_back({right, bRu, sizeof(double) * capR});
            rcv.push_back({right, bRF, sizeof(double) * 3 * capR});
        }
        if (capL > 0) {
            rcv.push_back({left, bLu, sizeof(double) * capL});
            rcv.push_back({left, bLF, sizeof(double) * 3 * capL});
        }
    }
    void stage6(cudaStream_t s) {
        if (half) {
            if (capL > 0) k_ghost_back<<<blocks(capL, 256), 256, 0, s>>>(sendL, idxL, capL, bLu, bLF, ul, Fl);
            if (capR > 0) k_ghost_back<<<blocks(capR, 256), 256, 0, s>>>(sendR, idxR, capR, bRu, bRF, ul, Fl);
        }
        cuda_ok(cudaMemsetAsync(energy, 0, sizeof(double), s), "memset");
        if (n_own > 0) k_own_out<<<blocks(n_own, 256), 256, 0, s>>>(n_own, ul, Fl, q, u, F, energy);
        cuda_ok(cudaGetLastError(), "shard output");
        // the previous call's flags (no synchronisation here)
        cuda_ok(cudaMemcpyAsync(h_flags, flags, sizeof(int), cudaMemcpyDeviceToHost, s), "flags");
    }
};

namespace {

using Stage = void (esp_shard::*)(cudaStream_t, std::vector<Msg>&, std::vector<Msg>&);
const Stage kStages[] = {&esp_shard::stage0, &esp_shard::stage1, &esp_shard::stage2,
                         &esp_shard::stage3, &esp_shard::stage4, &esp_shard::stage5};

void bind(esp_shard* sh, const double* box, long n_own, const double* pos, const double* q,
          double* u, double* F, double* energy) {
    if (!sh) throw espb::InvalidArgument("null shard");
    if (!box) throw espb::InvalidArgument("null box");
    for (int d = 0; d < 3; ++d)
        if (box[d] != sh->plan->plan.box[d])
            throw espb::InvalidArgument("sharded evaluate: system box does not match plan box");
    if (n_own < 0 || n_own > sh->n_own_cap)
        throw espb::InvalidArgument("sharded evaluate: n_own exceeds the shard's max_own_atoms");
    if (n_own > 0 && (!pos || !q || !u || !F)) throw espb::InvalidArgument("null argument");
    if (!energy) throw espb::InvalidArgument("null energy");
    if (*sh->h_flags & 1) throw espb::NumericalError("sharded evaluate: ghost capacity exceeded "
                                                     "on the previous call (raise ghost_capacity)");
    if (*sh->h_flags & 2)
        throw espb::InvalidArgument("sharded evaluate: an input atom is not owned by this rank "
                                    "(partition with esp_shard_owner)");
    sh->n_own = n_own;
    sh->pos = pos;
    sh->q = q;
    sh->u = u;
    sh->F = F;
    sh->energy = energy;
}

void nccl_exchange(esp_shard* sh, const std::vector<Msg>& snd, const std::vector<Msg>& rcv,
                   cudaStream_t s) {
    Nccl& n = Nccl::get();
    // messages to self are device copies (k-th send to self -> k-th receive)
    std::vector<const Msg*> ss, rs;
    for (const Msg& m : snd)
        if (m.peer == sh->rank) ss.push_back(&m);
    for (const Msg& m : rcv)
        if (m.peer == sh->rank) rs.push_back(&m);
    if (ss.size() != rs.size()) throw espb::CudaError("shard: unmatched self messages");
    for (size_t k = 0; k < ss.size(); ++k) {
        if (ss[k]->bytes != rs[k]->bytes) throw espb::CudaError("shard: self message size mismatch");
        if (ss[k]->bytes)
            cuda_ok(cudaMemcpyAsync(rs[k]->buf, ss[k]->buf, ss[k]->bytes, cudaMemcpyDeviceToDevice, s),
                    "self copy");
    }
    n.ok(n.groupStart(), "ncclGroupStart");
    for (const Msg& m : snd)
        if (m.peer != sh->rank && m.bytes)
            n.ok(n.send(m.buf, m.bytes, ncclChar, m.peer, sh->comm, s), "ncclSend");
    for (const Msg& m : rcv)
        if (m.peer != sh->rank && m.bytes)
            n.ok(n.recv(m.buf, m.bytes, ncclChar, m.peer, sh->comm, s), "ncclRecv");
    n.ok(n.groupEnd(), "ncclGroupEnd");
}

// lockstep emulation: the k-th send of rank r to rank p lands in the k-th
// receive of rank p from rank r
void emulated_exchange(const std::vector<std::vector<Msg>>& snd,
                       const std::vector<std::vector<Msg>>& rcv, cudaStream_t s) {
    const int G = static_cast<int>(snd.size());
    for (int r = 0; r < G; ++r)
        for (int p = 0; p < G; ++p) {
            std::vector<const Msg*> a, b;
            for (const Msg& m : snd[r])
                if (m.peer == p) a.push_back(&m);
            for (const Msg& m : rcv[p])
                if (m.peer == r) b.push_back(&m);
            if (a.size() != b.size())
                throw espb::CudaError("shard emulation: unmatched messages " + std::to_string(r) +
                                      " -> " + std::to_string(p));
            for (size_t k = 0; k < a.size(); ++k) {
                if (a[k]->bytes != b[k]->bytes)
                    throw espb::CudaError("shard emulation: message size mismatch " +
                                          std::to_string(r) + " -> " + std::to_string(p));
                if (a[k]->bytes)
                    cuda_ok(cudaMemcpyAsync(b[k]->buf, a[k]->buf, a[k]->bytes,
                                            cudaMemcpyDeviceToDevice, s),
                            "emulated copy");
            }
        }
}

esp_shard* make_shard(esp_plan* plan, int rank, int nranks, long max_own, long ghost_cap) {
    engine(plan);
    if (nranks < 2 || rank < 0 || rank >= nranks)
        throw espb::InvalidArgument("sharded evaluation: need nranks >= 2 and 0 <= rank < nranks");
    if (max_own < 0) throw espb::InvalidArgument("max_own_atoms must be non-negative");
    cuda_ok(cudaSetDevice(plan->device), "cudaSetDevice");
    auto sh = std::make_unique<esp_shard>();
    sh->plan = plan;
    sh->rank = rank;
    sh->nranks = nranks;
    sh->n_own_cap = max_own;
    if (ghost_cap <= 0) {
        // atoms within r_c of one face: max_own times reach / (narrowest slab
        // width), +30 % and a Poisson margin (the same on every rank that
        // passes the same max_own; NCCL ranks agree on the maximum below)
        const espb::Plan& P = plan->plan;
        double width = P.box[0];
        for (int r = 0; r < nranks; ++r) {
            const espb::PencilGeom g = espb::pencil_geometry(P, r, nranks);
            width = std::min(width, (g.x1 - g.x0) * g.hx);
        }
        const double e = static_cast<double>(max_own) * std::min(1.0, P.r_c / std::max(width, 1e-300));
        ghost_cap = static_cast<long>(1.3 * e + 6.0 * std::sqrt(e) + 256.0);
    }
    if (ghost_cap > (1L << 28)) throw espb::InvalidArgument("ghost capacity too large");
    sh->gcap = ghost_cap;
    return sh.release();
}

}  // namespace

extern "C" {

int esp_shard_unique_id(void* id) {
    return guarded([&] {
        if (!id) throw espb::InvalidArgument("null id");
        ncclUniqueId u;
        Nccl& n = Nccl::get();
        n.ok(n.getUniqueId(&u), "ncclGetUniqueId");
        std::memcpy(id, &u, sizeof(u));
    });
}

int esp_shard_create(esp_plan* plan, const void* nccl_id, int rank, int nranks,
                     long max_own_atoms, long ghost_capacity, esp_shard** out) {
    return guarded([&] {
        if (!out) throw espb::InvalidArgument("null out");
        std::unique_ptr<esp_shard> sh(make_shard(plan, rank, nranks, max_own_atoms, ghost_capacity));
        if (nccl_id) {
            Nccl& n = Nccl::get();
            ncclUniqueId u;
            std::memcpy(&u, nccl_id, sizeof(u));
            n.ok(n.commInitRank(&sh->comm, nranks, u, rank), "ncclCommInitRank");
            // message sizes must agree: every rank takes the largest ghost
            // capacity and own-atom bound (the local system's size)
            long* d = nullptr;
            cuda_ok(cudaMalloc(&d, 2 * sizeof(long)), "cudaMalloc");
            long h[2] = {sh->gcap, sh->n_own_cap};
            cuda_ok(cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice), "H2D");
            n.ok(n.allReduce(d, d, 2, ncclInt64, ncclMax, sh->comm, nullptr), "ncclAllReduce");
            cuda_ok(cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost), "D2H");
            cudaFree(d);
            sh->gcap = h[0];
        }
        sh->setup();
        *out = sh.release();
    });
}

void esp_shard_destroy(esp_shard* sh) { delete sh; }

int esp_shard_info(const esp_shard* sh, esp_shard_info_t* o) {
    return guarded([&] {
        if (!sh || !o) throw espb::InvalidArgument("null argument");
        std::memset(o, 0, sizeof(*o));
        o->rank = sh->rank;
        o->nranks = sh->nranks;
        o->x0 = sh->me().x0;
        o->x1 = sh->me().x1;
        o->X0 = sh->X0;
        o->X1 = sh->X1;
        o->max_own_atoms = sh->n_own_cap;
        o->ghost_capacity = sh->gcap;
        o->local_atoms = sh->ncap;
        o->pencil_half = sh->half ? 1 : 0;
        o->nccl = sh->comm ? 1 : 0;
    });
}

int esp_shard_owner(const esp_plan* plan, int nranks, long n, const double* pos, int* owner) {
    return guarded([&] {
        if (!plan || (n > 0 && (!pos || !owner))) throw espb::InvalidArgument("null argument");
        const espb::Plan& P = plan->plan;
        std::vector<int> x1;
        double hx = 0.0;
        for (int r = 0; r < nranks; ++r) {
            const espb::PencilGeom g = espb::pencil_geometry(P, r, nranks);
            x1.push_back(g.x1);
            hx = g.hx;
        }
        for (long i = 0; i < n; ++i) {
            double x = pos[3 * i];
            const double L = P.box[0];
            x -= L * std::floor(x / L);  // system.hpp:29-36
            if (x >= L) x = 0.0;
            const int l = std::min(std::max(static_cast<int>(std::floor(x / hx)), 0), P.nf[0] - 1);
            owner[i] = static_cast<int>(std::upper_bound(x1.begin(), x1.end(), l) - x1.begin());
        }
    });
}

int esp_shard_evaluate(esp_shard* sh, const double box[3], long n_own, const double* pos_dev,
                       const double* q_dev, double* u_dev, double* F_dev, double* energy_dev,
                       void* stream) {
    return guarded([&] {
        bind(sh, box, n_own, pos_dev, q_dev, u_dev, F_dev, energy_dev);
        if (!sh->comm)
            throw espb::InvalidArgument("shard has no NCCL communicator (use esp_shard_evaluate_emulated)");
        cuda_ok(cudaSetDevice(sh->plan->device), "cudaSetDevice");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        std::vector<Msg> snd, rcv;
        for (Stage st : kStages) {
            (sh->*st)(s, snd, rcv);
            nccl_exchange(sh, snd, rcv, s);
        }
        sh->stage6(s);
        Nccl& n = Nccl::get();
        n.ok(n.allReduce(energy_dev, energy_dev, 1, ncclFloat64, ncclSum, sh->comm, s), "ncclAllReduce");
    });
}

int esp_shard_evaluate_emulated(esp_shard* const* shards, int nranks, const double box[3],
                                const long* n_own, const double* const* pos_dev,
                                const double* const* q_dev, double* const* u_dev,
                                double* const* F_dev, double* const* energy_dev, void* stream) {
    return guarded([&] {
        if (!shards || nranks < 2) throw espb::InvalidArgument("emulation needs nranks >= 2 shards");
        for (int r = 0; r < nranks; ++r) {
            if (!shards[r] || shards[r]->rank != r || shards[r]->nranks != nranks)
                throw espb::InvalidArgument("emulation: shards must be ranks 0..nranks-1 of one decomposition");
            if (shards[r]->gcap != shards[0]->gcap)
                throw espb::InvalidArgument("emulation: shards disagree on the ghost capacity "
                                            "(create them with the same max_own_atoms / "
                                            "ghost_capacity)");
            bind(shards[r], box, n_own[r], pos_dev[r], q_dev[r], u_dev[r], F_dev[r], energy_dev[r]);
        }
        cuda_ok(cudaSetDevice(shards[0]->plan->device), "cudaSetDevice");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        std::vector<std::vector<Msg>> snd(nranks), rcv(nranks);
        for (Stage st : kStages) {
            for (int r = 0; r < nranks; ++r) (shards[r]->*st)(s, snd[r], rcv[r]);
            emulated_exchange(snd, rcv, s);
        }
        for (int r = 0; r < nranks; ++r) shards[r]->stage6(s);
        // all-reduce of the energy partials
        for (int r = 1; r < nranks; ++r)
            k_add<<<1, 32, 0, s>>>(1, energy_dev[0], energy_dev[r]);
        for (int r = 1; r < nranks; ++r)
            cuda_ok(cudaMemcpyAsync(energy_dev[r], energy_dev[0], sizeof(double),
                                    cudaMemcpyDeviceToDevice, s),
                    "energy copy");
        cuda_ok(cudaGetLastError(), "emulated all-reduce");
    });
}

// Host-buffer forms: copy the own atoms in, evaluate, copy u / F / energy out
// (synchronous), then report the device flags like esp_shard_check.
int esp_shard_evaluate_host(esp_shard* sh, const double box[3], long n_own, const double* pos,
                            const double* q, double* u, double* F, double* energy) {
    int rc = guarded([&] {
        if (!sh) throw espb::InvalidArgument("null shard");
        if (n_own < 0 || n_own > sh->n_own_cap)
            throw espb::InvalidArgument("n_own exceeds the shard's max_own_atoms");
        if (n_own > 0 && (!pos || !q || !u || !F)) throw espb::InvalidArgument("null argument");
        if (!energy) throw espb::InvalidArgument("null energy");
        cuda_ok(cudaSetDevice(sh->plan->device), "cudaSetDevice");
        sh->host_buffers();
        cuda_ok(cudaMemcpy(sh->hpos, pos, sizeof(double) * 3 * n_own, cudaMemcpyHostToDevice), "H2D");
        cuda_ok(cudaMemcpy(sh->hq, q, sizeof(double) * n_own, cudaMemcpyHostToDevice), "H2D");
    });
    if (rc) return rc;
    rc = esp_shard_evaluate(sh, box, n_own, sh->hpos, sh->hq, sh->hu, sh->hF, sh->he, nullptr);
    if (rc) return rc;
    rc = guarded([&] {
        cuda_ok(cudaMemcpy(u, sh->hu, sizeof(double) * n_own, cudaMemcpyDeviceToHost), "D2H");
        cuda_ok(cudaMemcpy(F, sh->hF, sizeof(double) * 3 * n_own, cudaMemcpyDeviceToHost), "D2H");
        cuda_ok(cudaMemcpy(energy, sh->he, sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    });
    return rc ? rc : esp_shard_check(sh);
}

int esp_shard_evaluate_emulated_host(esp_shard* const* shards, int nranks, const double box[3],
                                     const long* n_own, const double* const* pos,
                                     const double* const* q, double* const* u, double* const* F,
                                     double* energy) {
    std::vector<const double*> P(nranks > 0 ? nranks : 0), Q(P.size());
    std::vector<double*> U(P.size()), Fd(P.size()), Ed(P.size());
    int rc = guarded([&] {
        if (!shards || nranks < 2 || !n_own || !energy) throw espb::InvalidArgument("null argument");
        for (int r = 0; r < nranks; ++r) {
            esp_shard* sh = shards[r];
            if (!sh) throw espb::InvalidArgument("null shard");
            if (n_own[r] < 0 || n_own[r] > sh->n_own_cap)
                throw espb::InvalidArgument("n_own exceeds the shard's max_own_atoms");
            cuda_ok(cudaSetDevice(sh->plan->device), "cudaSetDevice");
            sh->host_buffers();
            cuda_ok(cudaMemcpy(sh->hpos, pos[r], sizeof(double) * 3 * n_own[r],
                               cudaMemcpyHostToDevice), "H2D");
            cuda_ok(cudaMemcpy(sh->hq, q[r], sizeof(double) * n_own[r], cudaMemcpyHostToDevice),
                    "H2D");
            P[r] = sh->hpos;
            Q[r] = sh->hq;
            U[r] = sh->hu;
            Fd[r] = sh->hF;
            Ed[r] = sh->he;
        }
    });
    if (rc) return rc;
    rc = esp_shard_evaluate_emulated(shards, nranks, box, n_own, P.data(), Q.data(), U.data(),
                                     Fd.data(), Ed.data(), nullptr);
    if (rc) return rc;
    rc = guarded([&] {
        for (int r = 0; r < nranks; ++r) {
            cuda_ok(cudaMemcpy(u[r], U[r], sizeof(double) * n_own[r], cudaMemcpyDeviceToHost), "D2H");
            cuda_ok(cudaMemcpy(F[r], Fd[r], sizeof(double) * 3 * n_own[r], cudaMemcpyDeviceToHost),
                    "D2H");
        }
        cuda_ok(cudaMemcpy(energy, Ed[0], sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    });
    for (int r = 0; r < nranks && !rc; ++r) rc = esp_shard_check(shards[r]);
    return rc;
}

int esp_shard_check(esp_shard* sh) {
    return guarded([&] {
        if (!sh) throw espb::InvalidArgument("null shard");
        cuda_ok(cudaSetDevice(sh->plan->device), "cudaSetDevice");
        int f = 0;
        cuda_ok(cudaMemcpy(&f, sh->flags, sizeof(int), cudaMemcpyDeviceToHost), "flags");
        *sh->h_flags = f;
        if (f & 1) throw espb::NumericalError("sharded evaluate: ghost capacity exceeded (raise ghost_capacity)");
        if (f & 2)
            throw espb::InvalidArgument("sharded evaluate: an input atom is not owned by this rank "
                                        "(partition with esp_shard_owner)");
    });
}

}  // extern "C"
