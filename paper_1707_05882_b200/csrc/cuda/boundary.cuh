// boundary.cuh -- argument block of the boundary-system kernels.
#pragma once

#include "kernels.cuh"

namespace vrte {

struct BndArgs {
    ProblemDev p;
    int d;
    const double* psi_p;  // packed modes [om][d*d]
    const double* psi_m;
    const double* nu;     // [om][d][2]
    const double* wi;     // [om][d] (pair layout)
    const double* zp;     // [om][R][d]
    const double* zm;
    double* lhs;          // [mo][G*G]
    double* top0;         // [mo][d * 2d]
    double* rhs;          // [mo][R][G]
    double* up;           // [mo][R][d]
};

void launch_bnd_assemble(const BndArgs& a, cudaStream_t st);
void launch_bnd_rhs(const BndArgs& a, cudaStream_t st);
void launch_copy_zp0(const BndArgs& a, cudaStream_t st);
void lu_factor_batched(double* A, int G, int batch, int* ipiv, DeviceStatus* status,
                       const int* order_index, cudaStream_t st);
// kernels launched by lu_factor_batched + lu_solve_batched
int lu_launch_count(int G, int ncol);
void lu_solve_batched(const double* A, int G, int batch, const int* ipiv, double* B, int ncol,
                      cudaStream_t st);

}  // namespace vrte
