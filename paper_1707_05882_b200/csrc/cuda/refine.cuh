// refine.cuh -- argument block of the eigenpair refinement (refine.cu).
#pragma once

#include "kernels.cuh"

namespace vrte {

struct RefineArgs {
    int d, batch;
    const double* wi;     // pair layout of the packed columns
    const double* mdiag;
    const int* flags;     // bit0 conservative (excluded, homogeneous.cpp:302)
    const double* wr;     // eigenvalues (gap classification)
    const double* femax;  // [batch] max |FE|
    double* shift;        // [batch][d] relative Newton shift
    double* nu;           // [batch][d][2]
    double* rho;          // [batch][d][2] 1/nu during refinement
    double* psi_p;        // packed d x d (p)
    double* psi_m;        // packed d x d (q' = psi-)
    double* ab_sum;       // d x d: M(p + q')
    double* ab_dif;       // d x d: M(q' - p)
    const double* G1;     // E ab_sum
    const double* G2;     // F ab_dif
    int* sidx;            // [batch][d] normalization index
    // d x 2d scratch (set A | set B)
    double* AL;
    double* BE;
    double* FB;           // F BE, then the RHS in place
    double* UT;           // solution u~
    double* EU;           // E u~
    double* sigma;        // [batch][2d][2]
    int* kind;            // [batch][2d]
    const int* slot_on;   // [batch] or null: slots whose modes are refined this step
};

void launch_refine_shift(const RefineArgs& a, cudaStream_t st);
void launch_refine_normalize(const RefineArgs& a, cudaStream_t st);
void launch_refine_setup(const RefineArgs& a, cudaStream_t st);
void launch_refine_rhs(const RefineArgs& a, cudaStream_t st);
void launch_refine_update(const RefineArgs& a, cudaStream_t st);
void launch_nu_rho(const RefineArgs& a, bool to_rho, cudaStream_t st);
// slot_on[b] &= (max_j residual[b][j] > target); count = number of slots left on.
// The refinement's extra steps are decided per (medium, order) slot, so a slot's
// result does not depend on which other slots share the plan (order shards).
void launch_compact_slots(const int* slot_on, int batch, int* list, int* n, cudaStream_t st);
void launch_refine_slots(int d, int batch, const double* residual, double target, int* slot_on, int* count,
                         cudaStream_t st);

}  // namespace vrte
