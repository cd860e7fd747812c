// particular.cuh -- argument block of the particular-solution kernels.
#pragma once

#include "kernels.cuh"

namespace vrte {

struct PartArgs {
    int d, batch, n_in;           // batch = (medium, order) pairs
    const double* mu_in;          // [n_in]
    const double* nu;             // [batch][d][2]
    const double* femax;          // [batch]
    const double* mdiag;          // [d]
    const int* order_index;       // [batch] -> m (messages)
    double* mu_eff;               // [batch][n_in]
    double* sigma;                // [batch][4 n_in][2]
    int* kind;                    // [batch][4 n_in]
    const double* fsp;            // F s+  [batch][R][d]
    const double* sp;             // s+
    const double* sm;             // s-
    double* rhs;                  // [batch][R][d]
    const double* g;              // solution g = Z y
    const double* eg;             // E g
    const double* feg;            // F E g
    double* zp;                   // Z+ [batch][R][d]
    double* zm;                   // Z-
    DeviceStatus* status;
    // per-slot adaptive refinement (null: every slot, no bookkeeping)
    int* part_on;                 // [batch] slot still refining
    double* part_slot;            // [batch] interim max balance residual
    double* part_prev;            // [batch] its value at the previous decision
};

void launch_dither(const PartArgs& a, cudaStream_t st);
void launch_part_rhs(const PartArgs& a, cudaStream_t st);
void launch_zpm(const PartArgs& a, cudaStream_t st);
// final = false: only the interim maximum of the balance residual (DeviceStatus::
// part_check) for the adaptive refinement; final = true: the reference's gates.
void launch_part_residual(const PartArgs& a, cudaStream_t st, bool final = true);
void launch_part_refine_residual(const PartArgs& a, double* W, cudaStream_t st);
// After an interim launch_part_residual: part_on[b] stays on while its balance
// residual exceeds `target` and (first decision, or) halved since the last one;
// count = slots still on.  Off slots get a zero correction (g unchanged).
void launch_part_decide(const PartArgs& a, double target, bool first, int* count, cudaStream_t st);

}  // namespace vrte
