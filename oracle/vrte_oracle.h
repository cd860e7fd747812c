/*
 * vrte_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference `vrte` BRDF path (arXiv 1707.05882
 * discrete-ordinate VRTE solver, /root/reference/proj/src) used as the
 * parity checker for the sm_100a product path and as the timed CPU
 * baseline (`bench.py --impl reference`).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / reference leg may load this library; the
 * product (libvrte.so) never links or calls it.
 *
 * Eigen (the reference's only numeric dependency, version unpinned,
 * proj/CMakeLists.txt:10) is absent from the image, so the dense algebra is
 * restated on LAPACK from scipy-openblas: dgeev for Eigen::EigenSolver,
 * dgetrf/dgetrs and zgetrf/zgetrs for PartialPivLU, zgecon for rcond,
 * dgesvd for JacobiSVD.  Parity is pinned by the reference's own golden
 * values (tests/test_oracle_golden.py).
 */
#ifndef VRTE_ORACLE_H
#define VRTE_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Plain-array material description (layers top first). coeffs holds
 * n_layers * order_count row-major 4x4 matrices B_l, already zero-padded to a
 * common order count (material.cpp:106-108). */
typedef struct oracle_material {
    int32_t n_layers;
    int32_t order_count;
    const double* omega;   /* [n_layers] */
    const double* tau;     /* [n_layers] */
    const double* coeffs;  /* [n_layers][order_count][16] */
    int32_t base_type;     /* 0 black, 1 lambertian, 2 mueller table */
    double rho;            /* lambertian albedo */
    int32_t table_n;       /* mueller table node count */
    const double* table;   /* [table_n*table_n][16] row-major, R(mu_i,-mu_j) at i*n+j */
} oracle_material;

typedef struct oracle_timings {
    double homogeneous, particular, boundary, reconstruction, total_wall;
    uint64_t homogeneous_solves, particular_solves, boundary_solves, reconstruction_items;
    uint64_t clamped_entries, dithered;
    double max_eigen_residual, max_boundary_condition;
} oracle_timings;

const char* oracle_last_error(void);
/* diagnostic: number of modes whose first recovery residual exceeded 5e-10 */
uint64_t oracle_polish_count(void);
/* 1: run the reference algorithm to its fp64 limit (polish every mode, refine
 * every linear solve once); 0: exactly the reference's thresholds (default). */
void oracle_set_accurate(int32_t on);
/* 1: factor each order's boundary matrix once per solver and reuse the LU for
 * every incident (the matrix has no incident or k dependence, boundary.cpp:219;
 * results are bit-identical to 0).  Tests only: the timed CPU baseline keeps
 * the reference's per-incident factorization (default 0). */
void oracle_set_cache_boundary(int32_t on);

/* types.cpp:27-68 */
int32_t oracle_quadrature(int32_t n, double* nodes, double* weights);
/* wigner.cpp:31-62 (out has lmax+1 entries) */
void oracle_wigner_d_sequence(int32_t m, int32_t n, int32_t lmax, double x, double* out);
/* wigner.cpp:64-81 */
void oracle_gsf_sequence(int32_t m, int32_t lmax, double x, double* p, double* r, double* t);
/* kernel.cpp:29-65: four arrays of N*N row-major 4x4 blocks (index i*N+j) */
int32_t oracle_kernel_blocks(const oracle_material* mat, int32_t layer, int32_t quad_n, int32_t m,
                             double* pp, double* pm, double* mp, double* mm);
/* kernel.cpp:89-109: up/down [N][16] at signed beam cosine mu_beam */
int32_t oracle_beam_column(const oracle_material* mat, int32_t layer, int32_t quad_n, int32_t m,
                           double mu_beam, double* up, double* down);
/* homogeneous.cpp:43-73: E, F column-major d x d, d = 4N */
int32_t oracle_reduced_ops(const oracle_material* mat, int32_t layer, int32_t quad_n, int32_t m,
                           double* e, double* f);
/* homogeneous.cpp:131-287: sorted modes. nu[2*d] (re,im), residual[d];
 * psi_plus/psi_minus: d modes x d entries, complex interleaved, mode-major
 * (may be NULL). Returns 0 or a vrte status code. */
int32_t oracle_homogeneous(const oracle_material* mat, int32_t layer, int32_t quad_n, int32_t m,
                           double* nu, double* residual, double* psi_plus, double* psi_minus);
/* particular.cpp:7-107 for one (m, k, mu0, I0). z_plus/z_minus [d]. */
int32_t oracle_particular(const oracle_material* mat, int32_t layer, int32_t quad_n, int32_t m,
                          int32_t k, double mu0, const double* stokes, double* z_plus,
                          double* z_minus, double* mu0_effective, double* residual);
/* brdf.cpp:43-125 through pipeline.cpp:57-220: the full BRDF table,
 * out[(ii*N + io)*n_dphi + ip][16] row-major Mueller entries. basis: 16
 * doubles (basis[4b+c]) or NULL for the default basis. threads 0 = hw.
 * up_components (optional, may be NULL): [n_in][4 basis][L][2 k][d] complex
 * interleaved tau=0 upward stacks, for stage-level debugging. */
int32_t oracle_brdf(const oracle_material* mat, int32_t quad_n, int32_t order_cap, int32_t threads,
                    const double* mu_in, size_t n_in, int32_t n_dphi, const double* basis,
                    double* out, oracle_timings* timings, double* up_components);

/* capi.cpp:138-174 vrte_solve_radiance: field at optical depths taus (n_tau = 0
 * -> {0}) on the signed zenith grid (2*zenith) x azimuth grid, from the beam
 * (mu0, phi0, stokes).  values [n_tau][2*zenith][azimuth][4]; reflectance [4]
 * (brdf.cpp:142-160); mus_out [2*zenith], phis_out [azimuth] may be NULL. */
int32_t oracle_radiance(const oracle_material* mat, int32_t quad_n, int32_t order_cap, int32_t threads, double mu0,
                        double phi0, const double* stokes, const double* taus, size_t n_tau, int32_t zenith,
                        int32_t azimuth, double* mus_out, double* phis_out, double* values, double* reflectance,
                        oracle_timings* timings);
/* Same with explicit signed directions / azimuths (NULL/0 -> grids); nodal = 1
 * returns the discrete-ordinate stacks at +nodes then -nodes (reconstruction.cpp:20-26)
 * instead of the source-function integration (values [n_tau][2N][n_phi][4]). */
int32_t oracle_radiance_at(const oracle_material* mat, int32_t quad_n, int32_t order_cap, int32_t threads,
                           double mu0, double phi0, const double* stokes, const double* taus, size_t n_tau,
                           int32_t zenith, int32_t azimuth, const double* mus_in, size_t n_mu_in,
                           const double* phis_in, size_t n_phi_in, int32_t nodal, double* mus_out,
                           double* phis_out, double* values, double* reflectance, oracle_timings* timings);

/* mc.cpp:1-315: raw Monte Carlo tallies (sum, sum_sq [2][zb][ab][4]; hits [2][zb][ab]). */
int32_t oracle_mc_trace(const oracle_material* mat, double mu0, double phi0, const double* stokes, uint64_t photons,
                        uint64_t seed, int32_t zenith_bins, int32_t azimuth_bins, int32_t threads, double* sum,
                        double* sum_sq, uint64_t* hits);

#ifdef __cplusplus
}
#endif

#endif
