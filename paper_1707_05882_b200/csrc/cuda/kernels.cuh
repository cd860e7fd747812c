// kernels.cuh -- device-side problem description and kernel launchers of the
// sm_100a BRDF path (orchestrated by brdf_device.cu).
#pragma once

#include "common.cuh"

namespace vrte {

// Device view of one BRDF solve (all pointers are device pointers).
// Orders handled on this device: m = m_begin + mo * m_stride, mo < n_orders.
struct ProblemDev {
    int N, L, n_media, n_layers, n_in, n_dphi;  // L: Fourier orders (after order_cap)
    int Lc;                                      // expansion-coefficient count (sum over l)
    int n_orders, m_begin, m_stride;
    const double* nodes;    // [N]
    const double* weights;  // [N]
    const double* omega;    // [n_media]
    const double* greek;    // [n_media][Lc][6] beta alpha gamma delta eps zeta
    const double* tau;      // [n_layers]
    const int* medium;      // [n_layers] -> medium index
    const double* mu_in;    // [n_in]
    int base_type;          // 0 black, 1 lambertian, 2 mueller table
    double rho;
    int table_n;
    const double* table;      // [table_n*table_n][16] row-major
    const double* beam_rows;  // [n_in][N][16] base_row_at(mu_i, mu0) (boundary.cpp:37-71)
    const double* refl_top;   // [N][16] Fresnel interface: down = R up at tau = 0 (null: none)
    __host__ __device__ int order_of(int mo) const { return m_begin + mo * m_stride; }
};

// phase.cu
void launch_gsf(const ProblemDev& p, const double* mus, int count, double sign, double* out,
                cudaStream_t st);
void launch_build_ef(const ProblemDev& p, const double* gsf, double* E, double* F,
                     cudaStream_t st);
void launch_kernel_dump(const ProblemDev& p, const double* gsf, int s, double* out, cudaStream_t st);
void launch_beam_source(const ProblemDev& p, const double* gsf_nodes, const double* gsf_beam,
                        double* sp, double* sm, cudaStream_t st);

// eig.cu
void launch_max_abs(const double* A, long long per, int batch, double* out, cudaStream_t st);
void launch_hessenberg(double* A, double* Z, int d, int batch, cudaStream_t st);
// hessenberg.cu: blocked reduction (panel kernel + DMMA trailing updates) and
// explicit Q in Z; `work` holds hessenberg_work_doubles(d) doubles per matrix.
int hessenberg_panel_width(int d);
size_t hessenberg_work_doubles(int d);
// (the two halves: the reduction of A, then Q from the reflectors left in work)
void launch_hessenberg_reduce(double* A, double* work, int d, int batch, cudaStream_t st);
void launch_hessenberg_formq(double* Z, double* work, int d, int batch, cudaStream_t st);
void launch_hessenberg_blocked(double* A, double* Z, double* work, int d, int batch,
                               cudaStream_t st);
int hessenberg_launch_count(int d);
// trace (debug, may be null): [batch][8] per matrix: cycles of rank 0,
// reflectors, sweeps, AED calls, AED cycles, chase cycles, update-wait cycles,
// AED deflations
void launch_hqr(double* H, double* Z, double* wr, double* wi, int d, int batch,
                DeviceStatus* status, cudaStream_t st, double* trace = nullptr, bool lean = false);
void launch_trevc(const double* T, const double* wr, const double* wi, double* Y, int d,
                  int batch, cudaStream_t st);
// Normalize packed eigenvector columns by their max complex modulus; returns
// the per-column scale applied in `scale` (may be null).
void launch_normalize_modes(double* X, const double* wi, int d, int batch, cudaStream_t st);
struct ModeArgs {
    int d, batch;
    const double* wr;
    const double* wi;
    const double* femax;   // [batch] max |FE| (lambda floor)
    const double* X;       // packed eigenvectors (normalized)
    const double* EX;      // E * X
    const double* mdiag;   // [d] node cosines repeated per Stokes row (device)
    double* nu;            // [batch][d][2] complex
    double* lam;           // [batch][d][2] current eigenvalue (for polish shifts)
    int* flags;            // [batch][d] bit0 conservative, bit1 polish-active
    double* psi_p;         // packed
    double* psi_m;         // packed
    double* ab_sum;        // M(psi+ + psi-)  (GEMM input for residual)
    double* ab_dif;        // M(psi- - psi+)
    DeviceStatus* status;
    const int* order_index;  // [batch] -> order m, for messages (may be null)
};
void launch_modes(const ModeArgs& a, cudaStream_t st);
struct ResidualArgs {
    int d, batch;
    const double* wi;
    const double* nu;
    const double* psi_p;
    const double* psi_m;
    const double* G1;  // E (a+b)
    const double* G2;  // F (b-a)
    const double* mdiag;
    double* residual;  // [batch][d]
};
void launch_residual(const ResidualArgs& a, cudaStream_t st);

// Shifted solves (F E - sigma_c I) y_c = r_c in the eigenbasis of F E: W must
// already hold V^-1 R; on return it holds (Lambda - sigma_c)^-1 V^-1 R.
// kind[c]: 0 real column, 1 complex pair (c: Re, c+1: Im), 2 skip;
// sigma: [batch][ncol][2].
void launch_eig_diag_solve(double* W, int d, int ncol, long long w_stride, const double* wr,
                           const double* wi, const double* sigma, const int* kind, int batch,
                           cudaStream_t st);
void launch_set_identity(double* Z, int d, int batch, cudaStream_t st);
void launch_fill_int(int* p, int n, int value, cudaStream_t st);
// Analytic modes / zero particular solution of free-streaming (kernel-free)
// slots [b0, b1) (eig.cu).
void launch_free_modes(int d, int b0, int b1, const double* mdiag, double* psi_p, double* psi_m,
                       double* nu, double* wr, double* wi, double* residual, double* zp, double* zm, int R,
                       cudaStream_t st);


// radiance.cu: source-function reconstruction of the radiance field
// (reconstruction.cpp:28-227) on one solve's device state.  All pointers are
// device pointers; p.n_in = 1 (the beam), R = 4 channels.
struct RadArgs {
    ProblemDev p;
    int R, n_tau, n_mu, n_phi, slot0;  // slot0: mo of order 0 (base term) when base_val != nullptr
    double mu0, phi0, tau_total;
    double stokes[4];
    const double* taus;       // [n_tau]
    const double* mus;        // [n_mu] signed output cosines
    const double* phis;       // [n_phi]
    const double* tau_top;    // [n_layers]
    const double* beam_top;   // [n_layers] exp(-tau_top / mu0)
    const double* gsf_n;      // [L][Lc][3][N]   (nodes)
    const double* gsf_b;      // [L][Lc][3][1]   (-mu0)
    double* gsf_o;            // [L][Lc][3][n_mu]
    double* wp;               // [B][4 n_mu][d] weighted kernel rows (col-major)
    double* wm;
    double* bb;               // [B][n_mu][16]  beam blocks A^m(mu_o, -mu0)
    double* acc_a;            // [B][4 n_mu][d] source-coefficient contractions
    double* acc_b;
    double* beam_src;         // [P][NO][n_mu][4 ch][4]
    const double* psi_p;      // [B][d][d] packed modes
    const double* psi_m;
    const double* nu;         // [B][d][2]
    const double* wi;         // [B][d]
    const double* zp;         // [B][R][d]
    const double* zm;
    const double* rhs_x;      // [NO][G][R] boundary solution (all layers)
    const double* base_out;   // [n_mu][N][16] base_row_at(|mu_o|, mu_j)
    const double* base_beam;  // [n_mu][16]    base_row_at(|mu_o|, mu0)
    double* down_bot;         // [4][d]
    double* base_val;         // [4][n_mu][4] (nullptr: no base term)
    double* comp;             // [NO][4][n_tau][n_mu][4]
    double* field;            // [n_tau][n_mu][n_phi][4]
    const double* up;         // [NO][R][d] tau = 0 stacks
    double* refl;             // [4]
};
int launch_radiance(RadArgs a, cudaStream_t st);


// mc.cu: polarized Monte Carlo tracer (mc.cpp).  Device pointers except the scalars.
struct McArgs {
    uint64_t photons, seed, ph0;  // ph0: first photon of this launch (chunked)
    int zb, ab, n_layers, Lc, base_type, table_n;
    double mu0, phi0, rho, total;
    double stokes[4];
    const double* greek;        // [n_layers][Lc][6] beta alpha gamma delta eps zeta
    const int* medium;          // [n_layers] -> greek/omega row
    const double* omega;        // [n_layers]
    const double* tops;         // [n_layers] optical depth of each layer top
    const double* table;        // [table_n^2][16] Mueller-table base
    const double* table_nodes;  // [table_n] Gauss nodes of the table
    double* cdf;                // [n_layers][2049]
    double* density;            // [n_layers][2048]
    int* fail;
    double* cta_grid;           // [n_cta][2 zb ab][9]
    double* out;                // [2 zb ab][9]: sum[4], sum_sq[4], hits
};
int mc_photons_per_cta();
// tabulates the phase functions, then traces photons [ph0, ph0 + n) into out (accumulated)
int launch_mc_tables(McArgs a, double* edge_scratch, cudaStream_t st);
int launch_mc_chunk(McArgs a, uint64_t n, cudaStream_t st);

}  // namespace vrte
