/*
 * vrte_cuda.h -- internal C ABI between the host C++ of libvrte.so and its
 * sm_100a device pipeline ("the host C++ ... calls an
 * internal C ABI vrte_cuda_brdf(...) implemented in .cu").
 *
 * Plain pointers and sizes only.  All arrays are HOST arrays unless noted.
 * The public drop-in surface is vrte.h; these entry points are exported for
 * the benchmark (device-resident timing) and the multi-GPU order sharding.
 */
#ifndef VRTE_CUDA_H
#define VRTE_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#ifndef VRTE_API
#define VRTE_API __attribute__((visibility("default")))
#endif

/* One BRDF problem after host-side set-up (brdf.cpp:43-77, pipeline.cpp:27-55). */
typedef struct vrte_cuda_problem {
    int32_t N;            /* half-range quadrature nodes */
    int32_t L;            /* Fourier orders (after order_cap, pipeline.cpp:33-35) */
    int32_t L_coeffs;     /* expansion coefficients summed over l (kernel.cpp:30); 0 = L */
    int32_t n_layers;
    int32_t n_media;      /* distinct media after dedup (pipeline.cpp:37-54) */
    int32_t n_in;         /* incident cosines */
    int32_t n_dphi;       /* output azimuths */
    const double* nodes;    /* [N]  types.cpp:27-68 */
    const double* weights;  /* [N] */
    const double* omega;    /* [n_media] */
    const double* greek;    /* [n_media][L_coeffs][6]: beta alpha gamma delta eps zeta */
    const double* tau;      /* [n_layers] */
    const int32_t* medium;  /* [n_layers] -> medium index */
    const double* mu_in;    /* [n_in] */
    int32_t base_type;      /* 0 black, 1 lambertian, 2 mueller table */
    double rho;
    int32_t table_n;
    const double* table;      /* [table_n*table_n][16] row-major */
    const double* beam_rows;  /* [n_in][N][16]: base_row_at(node_i, mu0) */
    const double* post;       /* [n_in][16]: B (mu0 B)^+ (brdf.cpp:100-105) */
    const double* trig;       /* [L][n_dphi][2]: cos(m x), sin(m x), x = -dphi */
    /* order shard handled by this call: m = m_begin + k*m_stride, k < n_orders.
       n_orders = 0 means all L orders on this device. */
    int32_t m_begin, m_stride, n_orders;
    int32_t device;           /* CUDA ordinal; -1 = current device */
    /* vrte_cuda_brdf only: with n_devices > 1 the orders are sharded cyclically
       over these devices (m = k, k + D, ...), every shard runs the
       pipeline on its own device, the tau = 0 stacks are gathered to devices[0]
       (peer copies over NVLink) and synthesized there in order 0..L-1: the table
       is bitwise identical to the single-device one.  Repeated ordinals run
       several shards on one device. */
    const int32_t* devices;
    int32_t n_devices;
    /* Fresnel top interface (extension; NULL / 0 without one): refl_top [N][16]
       row-major Mueller reflection of the upward field at tau = 0 into the
       downward one (top boundary rows: down - R up = 0); pre [N][16] the
       left factor of the synthesized exit Mueller matrix per output node
       (T_out / n^2); the table keeps output nodes out_lo .. N-1 (the
       refraction cone). */
    const double* refl_top;
    const double* pre;
    int32_t out_lo;
    /* Debug dumps (vrte_options dump_*_path, pipeline.cpp:333-357,
       kernel.cpp:188-214): HOST buffers filled by the call when not NULL.
       dump_kernel [L][N][N][2][16]: A^m(+mu_i, +mu_j), A^m(+mu_i, -mu_j) of
       layer 0's medium; dump_nu [n_media][L][4N][2] and dump_residual
       [n_media][L][4N]: the modes' separation constants and 8N residuals;
       dump_boundary [L][2]: per order the cond_1 lower bound and the largest
       relative residual of the boundary system. */
    double* dump_kernel;
    double* dump_nu;
    double* dump_residual;
    double* dump_boundary;
    /* Scheduling hint: non-zero when this solve runs concurrently with others on
       the same device (spectral batch, pooled order shards): kernels pick their
       lower-register builds that let two CTAs share an SM. */
    int32_t concurrent;
} vrte_cuda_problem;

typedef struct vrte_cuda_result {
    double t_homogeneous;   /* device seconds per stage (CUDA events) */
    double t_particular;
    double t_boundary;
    double t_synthesis;
    double t_device;        /* whole device pipeline (first to last kernel) */
    double t_hessenberg;    /* per-kernel device seconds (CUDA events) */
    double t_hqr;
    double t_trevc;
    double t_refine;
    double t_lu_factor;
    double t_lu_solve;
    uint64_t dithered;
    uint64_t clamped;
    uint64_t polished;
    uint64_t kernel_launches;
    uint64_t qr_sweeps;     /* Francis sweeps / bulge-chase steps summed over matrices */
    uint64_t qr_steps;
    uint64_t qr_cycles[8];  /* debug: QR phase cycles / counters summed over matrices */
    double max_eigen_residual;
    double max_particular_residual;
    double max_balance_residual;    /* particular 8N balance (particular.cpp:86-105, gate 1e-6) */
    double max_boundary_residual;   /* |A x - b| / (|A||x| + |b|) (boundary.cpp:240-256, gate 1e-9) */
    double max_boundary_condition;  /* lower bound of cond_1 over the orders' boundary matrices */
    uint64_t boundary_refined;      /* 1 if the refinement step of boundary.cpp:245-248 ran */
    uint64_t boundary_cond_warnings;/* orders whose condition bound exceeds 1e14 (boundary.cpp:259-263) */
    uint64_t eigen_slots;   /* (medium, order) slots through the eigen pipeline (the rest are free-streaming) */
    uint64_t slots;         /* all (medium, order) slots of the call */
    uint64_t boundary_fallback; /* a residual probe failed (boundary.cuh): full solution + exact gate */
    uint64_t particular_extra_steps; /* refinement steps of the particular stage beyond the first */
    int32_t status;         /* 0 ok, 3 numerical, 5 argument */
    char message[512];
} vrte_cuda_result;

/* Radiance field (capi.cpp:138-174 / reconstruction.cpp:28-227):
 * the problem carries ONE incident (n_in = 1, mu_in[0] = the beam's mu0); the
 * field is evaluated at every (tau, signed mu, phi) of the grid. */
typedef struct vrte_cuda_radiance {
    int32_t n_tau, n_mu, n_phi;
    const double* taus;       /* [n_tau] optical depths */
    const double* mus;        /* [n_mu] signed output cosines (> 0 upward) */
    const double* phis;       /* [n_phi] azimuths */
    double phi0;              /* beam azimuth */
    double stokes[4];         /* beam I0 */
    const double* base_out;   /* [n_mu][N][16] base_row_at(|mu_o|, node_j) (m = 0, non-black base) */
    const double* base_beam;  /* [n_mu][16] base_row_at(|mu_o|, mu0) */
} vrte_cuda_radiance;

/* values [n_tau][n_mu][n_phi][4] (host), reflectance [4] (brdf.cpp:142-160). */
VRTE_API int32_t vrte_cuda_radiance_field(const vrte_cuda_problem* problem, const vrte_cuda_radiance* rad,
                                          double* values, double* reflectance, vrte_cuda_result* result);

/* Polarized Monte Carlo tracer (mc.cpp:1-315): raw tallies
 * sum / sum_sq [2][zb][ab][4] and hits [2][zb][ab] (host arrays).  Layers top
 * first; greek rows beta alpha gamma delta eps zeta. */
typedef struct vrte_cuda_mc {
    int32_t n_layers, Lc, base_type, table_n, zb, ab;
    uint64_t photons, seed;
    double mu0, phi0, rho, total;
    double stokes[4];
    const double* greek;        /* [n_layers][Lc][6] */
    const double* omega;        /* [n_layers] */
    const double* tops;         /* [n_layers] */
    const double* table;        /* [table_n^2][16] (base_type 2) */
    const double* table_nodes;  /* [table_n] */
    int32_t device;
} vrte_cuda_mc;
VRTE_API int32_t vrte_cuda_mc_trace(const vrte_cuda_mc* mc, double* sum, double* sum_sq, uint64_t* hits,
                                    vrte_cuda_result* result);

/* Recycled page-locked host buffers (per-size free list) for result tables;
 * falls back to the heap when pinning is unavailable. */
VRTE_API void* vrte_cuda_host_alloc(size_t bytes);
VRTE_API void vrte_cuda_host_free(void* p, size_t bytes);

/* Full solve: host inputs -> host table [n_in][N][n_dphi][16]. */
VRTE_API int32_t vrte_cuda_brdf(const vrte_cuda_problem* problem, double* table,
                                vrte_cuda_result* result);

/* Device-resident plan (benchmark / repeated solves of one shape). */
typedef struct vrte_cuda_plan vrte_cuda_plan;
VRTE_API int32_t vrte_cuda_plan_create(const vrte_cuda_problem* problem, vrte_cuda_plan** out,
                                       vrte_cuda_result* result);
/* Run the device pipeline `iters` times with inputs already resident; the
 * average device seconds per solve is returned in *seconds (CUDA events on the
 * plan's stream).  Table stays on the device. */
/* As vrte_cuda_plan_create, with the plan (device buffers, streams) leased from
 * the process-wide pool that vrte_cuda_brdf uses -- no allocation when a plan of
 * the same shape was released before; vrte_cuda_plan_release returns it. */
VRTE_API int32_t vrte_cuda_plan_acquire(const vrte_cuda_problem* problem, vrte_cuda_plan** out,
                                        vrte_cuda_result* result);
VRTE_API void vrte_cuda_plan_release(vrte_cuda_plan* plan);
VRTE_API int32_t vrte_cuda_plan_run(vrte_cuda_plan* plan, int32_t iters, double* seconds,
                                    vrte_cuda_result* result);
VRTE_API int32_t vrte_cuda_plan_fetch(vrte_cuda_plan* plan, double* table);
/* tau=0 upward stacks of the plan's orders: [n_orders][4 n_in][4N] (host). */
VRTE_API int32_t vrte_cuda_plan_fetch_up(vrte_cuda_plan* plan, double* up);
/* Device pointer to the same stacks ([n_orders][4 n_in][4N], on the plan's
 * device; valid until the plan's next run or destroy) and its element count:
 * the order-sharded paths exchange them with NCCL without host staging. */
VRTE_API int32_t vrte_cuda_plan_up_device(vrte_cuda_plan* plan, double** up, size_t* count);
/* Fourier synthesis + Mueller recovery of ALL L orders on the plan's device and
 * stream from device stacks up_all [L][4 n_in][4N] (order m at index m, e.g.
 * gathered from the order shards of every rank; reconstruction.cpp:201-227,
 * brdf.cpp:100-117), into the plan's table; copied to `table` (host
 * [n_in][N][n_dphi][16]) when not NULL.  The caller orders its own stream's
 * writes of up_all before the call (the call synchronizes the plan's stream). */
VRTE_API int32_t vrte_cuda_plan_synthesize_device(vrte_cuda_plan* plan, const double* up_all, double* table,
                                                  vrte_cuda_result* result);
/* Per-(medium, order) eigen data for debugging: wr, wi [n_media*n_orders][4N],
 * residual [n_media*n_orders][4N]. Any pointer may be NULL. */
VRTE_API int32_t vrte_cuda_plan_fetch_modes(vrte_cuda_plan* plan, double* wr, double* wi,
                                            double* residual, double* nu);
/* Reduced operators E, F [n_media*n_orders][4N*4N] column-major (debug/parity). */
VRTE_API int32_t vrte_cuda_plan_fetch_ef(vrte_cuda_plan* plan, double* E, double* F);
VRTE_API void vrte_cuda_plan_destroy(vrte_cuda_plan* plan);

/* Fourier synthesis from host-gathered stacks of ALL orders (multi-GPU root):
 * up [L][4 n_in][4N], host table out. */
VRTE_API int32_t vrte_cuda_synthesize(const vrte_cuda_problem* problem, const double* up,
                                      double* table, vrte_cuda_result* result);

VRTE_API int32_t vrte_cuda_device_count(void);
/* The calling thread's current CUDA device (0 when none is set). */
VRTE_API int32_t vrte_cuda_current_device(void);

/* Test hook: force (on != 0) the boundary stage's full-solution fallback -- the
 * path a failed residual probe takes (boundary.cuh) -- on every BRDF call of the
 * process, so the tests can compare it with the probe path. */
VRTE_API void vrte_cuda_debug_force_boundary_fallback(int32_t on);

/* Kernel-level check of the batched row-major LU (lu.cu) used by the boundary
 * stage: X[b] = A[b]^-1 B[b] for `batch` row-major G x G systems with `ncol`
 * right-hand sides (host arrays, row-major).  Returns 0, 3 (singular) or 5. */
VRTE_API int32_t vrte_cuda_lu_solve(const double* A, int32_t G, int32_t batch, const double* B,
                                    int32_t ncol, double* X, int32_t device);
/* Kernel-level check of the batched row-major LU factorization with partial
 * pivoting (lu.cu), in place: A [batch][G][ncols] row-major, the columns past G
 * eliminated along (augmented system); on return A holds L (unit lower, strictly
 * below the diagonal) and U at the physical rows, perm [batch][G] the row of each
 * position.  lookahead bit 0 runs the boundary stage's one-block look-ahead
 * schedule (two streams), else the serial one; bit 1 defers the columns past G:
 * the matrix is factored alone and they are eliminated afterwards on another
 * stream through the per-block row-map snapshots (the BRDF pipeline's path).
 * Returns 0, 3 (singular) or 5. */
VRTE_API int32_t vrte_cuda_lu_factor(double* A, int32_t G, int32_t ncols, int32_t batch, int32_t lookahead,
                                     int32_t* perm, int32_t device);
/* Kernel-level check of the blocked Hessenberg reduction (hessenberg.cu):
 * A[b] = Q[b] H[b] Q[b]^T for `batch` column-major d x d matrices (host arrays).
 * blocked = 0 selects the unblocked reference kernel. */
VRTE_API int32_t vrte_cuda_hessenberg(const double* A, int32_t d, int32_t batch, double* H, double* Q,
                                      int32_t blocked, int32_t device);
/* Kernel-level check of the eigen stage: real Schur form A[b] = Z T Z^T
 * (blocked Hessenberg + multishift QR with AED, eig.cu) and the eigenvalues
 * wr/wi [batch][d].  Returns 0, or 3 if the QR did not converge. */
VRTE_API int32_t vrte_cuda_schur(const double* A, int32_t d, int32_t batch, double* T, double* Z, double* wr,
                                 double* wi, int32_t device);
/* Same, with the QR kernel's per-matrix profile (debug): trace [batch][8] =
 * cycles, reflectors, sweeps, AED calls, AED cycles, chase cycles,
 * update-wait cycles, AED deflations (either pointer may be NULL; qr_ms: the
 * QR kernel's device time). */
VRTE_API int32_t vrte_cuda_schur_trace(const double* A, int32_t d, int32_t batch, double* T, double* Z, double* wr,
                                       double* wi, int32_t device, double* trace, double* qr_ms);

#ifdef __cplusplus
}
#endif

#endif
