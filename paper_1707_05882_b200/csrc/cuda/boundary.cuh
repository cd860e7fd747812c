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
    double* lhs;          // [mo] row-major G x ldl (ldl = G + R: augmented with the right-hand sides)
    double* top0;         // [mo][d * 2d]
    double* rhs;          // [mo] row-major G x ldr (into the augmented lhs: lhs + G, ldr = ldl)
    int ldl, ldr;
    long long sl, sr;     // per-order strides of lhs and rhs
    double* up;           // [mo][R][d]
    // residual gate (boundary.cpp:233-257): an untouched copy of [A | B] (same
    // row-major layout as lhs, never factored) and per-order / per-column norms
    double* lhs0;         // [mo] G x ldl, or null (no gate)
    double* anorm;        // [mo][2]: max |A_ij|, ||A||_1
    double* bnorm;        // [mo][R][2]: max |b_i|, ||b||_1
    double* condm;        // [mo]: lower bound of cond_1(A), max over the right-hand sides
    double* colsum;       // [mo][G] scratch of the ||A||_1 reduction
    unsigned* colsum_ticket;  // [mo][G / 256 slabs]
    int* order_fail;      // [mo] a residual probe of this order failed (the fallback redoes only these)
    int* col_refine;      // [mo][R] right-hand sides taking the refinement step (full gate)
    double* resm;         // [mo] largest relative residual of the order (dumps)
    int K;                // residual probes (0: the full gate); their b_k in lhs0 columns G + R + k
};

// Residual probes (the default gate).  The BRDF needs only layer 0's unknowns,
// so the back substitution of the R right-hand sides stops there; the
// reference's per-right-hand-side residual check (boundary.cpp:236-254) is
// applied to K fixed pseudo-random right-hand sides instead, solved through
// every row: two combinations b_k = B v_k of the right-hand sides (their
// forward elimination is Y v_k, Y the eliminated columns of the augmented
// factorization; x_k = X v_k by linearity) and two random vectors of R^G
// (which also expose the matrix's small singular directions to the cond_1
// lower bound ||A||_1 ||x||_1 / ||b||_1).  A backward-stable solve gives every
// probe a residual ~eps scale; a probe above the reference's refinement
// threshold (1e-10 scale) or a non-finite solution entry sets
// DeviceStatus::bnd_fallback, and the host then runs the reference's exact gate
// on the full solution (launch_bnd_residual / launch_bnd_check).
constexpr int kBndProbes = 4;
constexpr int kBndCombProbes = 2;  // probes [0, 2): B v_k; [2, 4): random b
// After the factorization, before the back substitution overwrites Y: Xp
// [mo][G][K] (position order) <- Y v_k / the gathered random b; b_k into
// lhs0's columns G + R + k (storage rows; lhs0 row stride >= G + R + K).
void launch_bnd_probe_setup(const BndArgs& a, const int* perm, double* Xp, int G, int R, cudaStream_t st);
// Rp [mo][G][K] = A0 Xp (block-sparse), then the probe / finiteness check.
void launch_bnd_probe_check(const BndArgs& a, const double* Xp, double* Rp, const double* X, int row_lo, int G, int R,
                            DeviceStatus* status, cudaStream_t st);
// up[mo] <- saved[mo] for the orders whose probes passed (keep = order_fail == 0):
// the fallback's full solve replaces only the failed orders' stacks, so an
// order's result does not depend on the other orders of the plan.
void launch_bnd_keep_passed(const BndArgs& a, const double* saved, cudaStream_t st);
// Full-solution fallback: X [mo][G][R] <- rows of lhs0's B columns through the row map.
void launch_bnd_gather_b(const BndArgs& a, const int* perm, double* X, int G, int R, cudaStream_t st);

// The gate after the back substitution: the relative residual of every
// right-hand side, |A x - b|_max / (|A|_max |x|_max + |b|_max); residual = lhs0's
// B columns after bnd_residual_gemm.  stage 0: flags columns above 1e-10 for the
// one refinement step (DeviceStatus::bnd_refine) and fails on non-finite
// solutions; stage 1 (after refinement, or when nothing was refined): fails
// above 1e-9 (boundary.cpp:249-254).
void launch_bnd_norms(const BndArgs& a, int G, int R, cudaStream_t st);
void launch_bnd_residual(const BndArgs& a, const double* X, int G, int R, bool accumulate, cudaStream_t st);
void launch_bnd_check(const BndArgs& a, const double* X, int G, int R, int stage, DeviceStatus* status,
                      cudaStream_t st);
void launch_bnd_refine_rhs(const BndArgs& a, const int* perm, double* dX, int G, int R, cudaStream_t st);
void launch_bnd_add(const BndArgs& a, double* X, const double* dX, int G, int R, cudaStream_t st);

// zeroed: lhs already cleared by launch_bnd_zero (the pipeline clears it on the
// side stream under the eigen stage)
void launch_bnd_zero(const BndArgs& a, cudaStream_t st);
void launch_bnd_assemble(const BndArgs& a, cudaStream_t st, bool zeroed = false);
void launch_bnd_rhs(const BndArgs& a, cudaStream_t st);
void launch_copy_zp0(const BndArgs& a, cudaStream_t st);
// lu.cu: batched LU with partial pivoting on ROW-major G x G matrices.
// ipiv: [batch][G] absolute pivot rows (LAPACK order); perm: [batch][G] net
// row permutation (row i of P B = row perm[i] of B).
// prof_d / prof_P > 0: the matrix has the boundary-system staircase profile
// (bnd_row_end); rows past a column block's profile are skipped.
// lda: row stride (0 = G); ncols > G: the columns past G (right-hand sides of
// an augmented system [A | B]) are carried through the elimination.
// la (optional): look-ahead by one outer block -- the panels of block K+1 (and
// the update of block K+1's columns) on the high-priority stream la->hi while the
// rest of block K's trailing update runs on la->lo through a snapshot of the
// row map; both fork from and join back into st.
struct LuLookahead {
    cudaStream_t hi = nullptr, lo = nullptr;
    int* snap = nullptr;  // [batch][G]
    cudaEvent_t ev[4] = {};
};
// rd (optional): the right-hand sides are NOT carried through the factorization
// (ncols = G): the row map after each outer block's panels is saved in
// rd->snaps[K] and rd->ev[K] recorded, so lu_rhs_forward can apply each block's
// update to the right-hand-side columns later, on another stream, with exactly
// the arithmetic the augmented factorization would have used.
struct LuRhsDefer {
    int* snaps = nullptr;       // [nblocks][batch][G]
    cudaEvent_t* ev = nullptr;  // [nblocks]
    int nblocks = 0;
};
int lu_outer_blocks(int G);
void lu_factor_rm(double* A, int G, int batch, int* ipiv, int* perm, DeviceStatus* status,
                  const int* order_index, cudaStream_t st, int prof_d = 0, int prof_P = 0, int lda = 0,
                  int ncols = 0, cudaEvent_t cols_ready = nullptr, const LuLookahead* la = nullptr,
                  const LuRhsDefer* rd = nullptr);
// L^-1 P B in place in the columns [G, G + R) of a factorization run with rd:
// block K's update (fused block solve + GEMM over the staircase rows, through
// rd->snaps[K]) once rd->ev[K] has fired.
void lu_rhs_forward(double* A, int G, int lda, int R, int batch, const LuRhsDefer& rd, int prof_d, int prof_P,
                    cudaStream_t st);
int lu_rhs_forward_launch_count(int G);
// Back substitution of an augmented factorization (ncols = G + R) in place, down
// to row_lo (rounded down to a 64-row block); X [batch][G][R] receives rows >= that.
void lu_backsolve_aug(double* A, int G, int lda, int R, int batch, const int* perm, double* X, int row_lo,
                      cudaStream_t st);
// X = A^-1 B for row-major B, X ([batch][G][ncol]); B is not modified.  Only
// rows >= row_lo (rounded down to the 64-row block) of X are the solution.
void lu_solve_rm(const double* A, int G, int batch, const int* perm, const double* B, double* X,
                 int ncol, cudaStream_t st, int row_lo = 0, int prof_d = 0, int prof_P = 0);
// Column of the boundary system holding layer p's packed column j: layer 0
// (the only unknowns the tau = 0 field needs) is ordered LAST, so the back
// substitution stops after its 2d rows.
__host__ __device__ inline int bnd_col(int p, int j, int d, int G) { return (2 * d * p + j - 2 * d + G) % G; }
// Row of boundary equation r (boundary.cpp order: top d, interface p 2d each,
// bottom d): the top rows -- the only ones touching layer 0 besides interface 0
// -- are ordered LAST, so the system has a staircase profile: the columns of
// layer p >= 1 (ordered first) are nonzero only in rows < bnd_row_end.
__host__ __device__ inline int bnd_row(int r, int d, int G) { return (r - d + G) % G; }
// First row past the nonzero profile of (reordered) column `col`, P layers.
__host__ __device__ inline int bnd_row_end(int col, int d, int P) {
    const int G = 2 * d * P;
    if (P <= 1) return G;
    const int b = col / (2 * d);  // column block: b < P-1 is layer b+1, b = P-1 is layer 0
    if (b >= P - 1) return G;
    const int p = b + 1;
    return (p <= P - 2) ? 2 * d * (p + 1) : 2 * d * (P - 1) + d;
}
// Forward + backward substitution in place on right-hand sides already gathered
// through the row map (row i of X = row perm[i] of B): X <- A^-1 B, A factored
// by lu_factor_rm with row stride lda.  Columns < fwd_lo already hold L^-1 P B
// (forward-eliminated by an augmented factorization): back substitution only.
void lu_solve_gathered(const double* A, int G, int lda, int batch, const int* perm, double* X, int ncol,
                       cudaStream_t st, int fwd_lo = 0);
// X <- A^-1 X for K = 4 columns ([batch][G][K], position order) by one CTA per
// matrix (the boundary gate's residual probes); columns < fwd_lo already hold
// L^-1 P b.  G <= 4096 (the columns live in shared memory).
void lu_few_solve(const double* A, int G, int lda, int batch, const int* perm, double* X, int K, int fwd_lo,
                  cudaStream_t st);
int lu_rm_launch_count(int G);
int lu_aug_launch_count(int G, int R, int row_lo);
int lu_gathered_launch_count(int G, int ncol, int fwd_lo);

}  // namespace vrte
