/*
 * vrte_ext.h -- optional additions to the vrte C ABI (the reference ABI in
 * vrte.h is unchanged; these are new symbols, SURVEY.md §5 "add optional new
 * functions").
 */
#ifndef VRTE_EXT_H
#define VRTE_EXT_H

#include "vrte.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Device-side statistics of the last vrte_compute_brdf on this handle. */
typedef struct vrte_brdf_device_stats {
    double t_homogeneous, t_particular, t_boundary, t_synthesis; /* device seconds */
    uint64_t dithered, clamped, polished, kernel_launches;
    double max_eigen_residual, max_particular_residual;
    uint64_t material_hash; /* FNV-1a over the numeric content (brdf.cpp:11-41) */
    double max_balance_residual;    /* particular 8N balance residual (gate 1e-6) */
    double max_boundary_residual;   /* boundary system relative residual (gate 1e-9) */
    double max_boundary_condition;  /* lower bound of cond_1 of the boundary matrices */
    uint64_t boundary_refined;      /* boundary refinement step taken (boundary.cpp:245-248) */
    uint64_t boundary_cond_warnings;/* orders above the 1e14 warning level (boundary.cpp:259-263) */
    uint64_t boundary_fallback;     /* a residual probe failed: the full solution was checked */
    uint64_t eigen_slots;           /* (medium, order) slots through the eigen pipeline */
} vrte_brdf_device_stats;

VRTE_API vrte_status vrte_brdf_device_stats_get(const vrte_brdf* brdf, vrte_brdf_device_stats* out);

/* The table's grids (any pointer may be NULL): mu_in [n_in] as requested,
 * mu_out [n_out] the exit cosines (the quadrature nodes; with a Fresnel
 * interface the refraction cone's nodes mapped to the outside), dphi [n_dphi]. */
VRTE_API vrte_status vrte_brdf_grid(const vrte_brdf* brdf, double* mu_in, double* mu_out, double* dphi);

/* Build the device problem of a BRDF request without solving it (benchmark
 * plan creation; see vrte_cuda.h).  Returns an opaque plan. */
typedef struct vrte_cuda_plan vrte_cuda_plan;
VRTE_API vrte_status vrte_brdf_plan_create(const vrte_material* material, const vrte_options* options,
                                           const double* mu_in, size_t n_mu_in, int32_t n_dphi,
                                           const double* basis, int32_t device, int32_t m_begin,
                                           int32_t m_stride, int32_t n_orders, vrte_cuda_plan** out);

/* vrte_brdf_plan_create with the plan leased from the process pool (the
 * order-sharded multi-GPU calls of paper_1707_05882_b200/distributed.py: one
 * order shard solved per call, inputs uploaded, no allocation after the first
 * call of a shape); release it with vrte_cuda_plan_release (vrte_cuda.h). */
VRTE_API vrte_status vrte_brdf_plan_acquire(const vrte_material* material, const vrte_options* options,
                                            const double* mu_in, size_t n_mu_in, int32_t n_dphi,
                                            const double* basis, int32_t device, int32_t m_begin,
                                            int32_t m_stride, int32_t n_orders, vrte_cuda_plan** out);

/* Assemble a BRDF handle from the tau = 0 upward stacks of ALL orders,
 * up_all_orders [L][4 n_mu_in][4N] (host), gathered from order shards: the
 * Fourier synthesis runs on the device and the stacks are read, not kept. */
VRTE_API vrte_status vrte_brdf_from_stacks(const vrte_material* material, const vrte_options* options,
                                           const double* mu_in, size_t n_mu_in, int32_t n_dphi,
                                           const double* basis, const double* up_all_orders,
                                           vrte_brdf** out);

/* Solve `count` independent BRDF requests -- e.g. the 31 spectral bands of a
 * paint (BASELINE.json config 5, SURVEY.md §8(f) "spectral batch API") -- with
 * the same options, incident cosines, azimuth count and basis.  The requests
 * run concurrently (one device plan and CUDA stream each, `concurrency` host
 * threads; <= 0 picks 2).  out[i] receives request i's handle, or NULL when it
 * failed; the return value is the first failure (VRTE_OK if none), with its
 * message in vrte_last_error().  Each table is identical to the one
 * vrte_compute_brdf returns for that material alone. */
VRTE_API vrte_status vrte_compute_brdf_batch(const vrte_material* const* materials, size_t count,
                                             const vrte_options* options, const double* mu_in,
                                             size_t n_mu_in, int32_t n_dphi, const double* basis,
                                             int32_t concurrency, vrte_brdf** out);

/* Photon count of one tally bin (mc.hpp TallyGrid::hits; the reference keeps it
 * internal, its acceptance test skips bins with < 50 hits). */
VRTE_API vrte_status vrte_mc_tally_hits(const vrte_mc_tally* tally, int32_t hemisphere, int32_t zenith_bin,
                                        int32_t azimuth_bin, uint64_t* hits);

#ifdef __cplusplus
}
#endif

#endif
