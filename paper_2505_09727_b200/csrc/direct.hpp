// Direct Ewald summation on the GPU (reference.hpp:42-206), all atoms or a
// subset of targets; see direct.cu.
#pragma once

namespace espb {

struct DirectPassResult {
    double lambda = 0.0;     // splitting width used
    int real_shells = 0;     // last max-norm image shell summed
    int recip_kmax = 0;      // reciprocal max-norm cutoff
    double tail_bound = 0.0; // max of the two stop-criterion bounds
};

// One pass at splitting width lambda (<= 0: min(L)/6, reference.hpp:222).
// pos: N x 3, q: N (host); targets: ntarget indices or nullptr for all atoms;
// u: ntarget (or N), F: ntarget x 3 (or N x 3), host.
DirectPassResult direct_ewald_pass(int device, const double box[3], long N, const double* pos,
                                   const double* q, long ntarget, const long* targets, double tol,
                                   double lambda, double* u, double* F);

}  // namespace espb
