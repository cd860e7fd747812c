// boundary.cu -- global boundary system per Fourier order, boundary.cpp:142-265.
//
// The reference assembles and factors a complex (2dP)^2 system for every
// (incident, basis vector, order) although its matrix carries no incident
// dependence (boundary.cpp:219).  Here the matrix is assembled ONCE per order
// in a real basis (conjugate mode pairs -> Re/Im columns), LU-factored once,
// and every (incident, Stokes channel) is a right-hand side of one blocked
// triangular solve.  The tau = 0 upward stack (boundary.cpp:20-35) is then a
// single GEMM per order against [psi+ | att psi-] of the top layer.
#include <algorithm>
#include <vector>

#include "boundary.cuh"

namespace vrte {
namespace {

struct ModeView {
    const double* psi_p;
    const double* psi_m;
    const double* nu;
    const double* wi;
    int d;
    // complex psi(i) of the mode owning packed column jj
    __device__ void load(size_t om, int jj, int i, cplx& pp, cplx& pm, cplx& nuv, bool& im_col) const {
        const size_t vb = om * d;
        const double w = wi[vb + jj];
        const int j = (w < 0.0) ? jj - 1 : jj;
        im_col = w < 0.0;
        const bool pair = w != 0.0;
        const size_t cb = om * d * d + (size_t)j * d;
        pp = cmk(psi_p[cb + i], pair ? psi_p[cb + d + i] : 0.0);
        pm = cmk(psi_m[cb + i], pair ? psi_m[cb + d + i] : 0.0);
        nuv = cmk(nu[2 * (vb + j)], nu[2 * (vb + j) + 1]);
    }
};

__device__ inline cplx dflip(cplx v, int i) { return ((i & 3) >= 2) ? cmk(-v.re, -v.im) : v; }
__device__ inline cplx att_of(double tau, cplx nu) { return cexp_(cdiv(cmk(-tau, 0.0), nu)); }

// CTA per (order mo, layer p, 32 x 32 tile of (mode component i, packed column
// jj)); the system is stored ROW-major (lu.cu), lhs[mo][r * ldl + c].  The mode
// vectors are read along i (coalesced, column-major storage) into shared
// memory, the per-mode attenuation exp(-tau/nu) is computed once per column,
// and the system rows are written along jj (coalesced, row-major).
constexpr int AT = 32;  // tile edge
__global__ void __launch_bounds__(256) assemble_kernel(BndArgs a) {
    __shared__ double s_pr[AT][AT + 1], s_pi[AT][AT + 1], s_mr[AT][AT + 1], s_mi[AT][AT + 1];  // [jj][i]
    __shared__ double s_ar[AT], s_ai[AT];
    __shared__ int s_im[AT];
    const int d = a.d, P = a.p.n_layers, G = 2 * d * P;
    const int jj0 = blockIdx.x * AT, i0 = blockIdx.y * AT;
    const int p = blockIdx.z % P, mo = blockIdx.z / P;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    const size_t om = (size_t)a.p.medium[p] * a.p.n_orders + mo;
    const size_t vb = om * d;
    if (ty == 0) {
        const int jj = jj0 + tx;
        cplx att = cmk(0.0, 0.0);
        int imc = 0;
        if (jj < d) {
            const double w = a.wi[vb + jj];
            const int j = (w < 0.0) ? jj - 1 : jj;
            imc = w < 0.0;
            att = att_of(a.p.tau[p], cmk(a.nu[2 * (vb + j)], a.nu[2 * (vb + j) + 1]));
        }
        s_ar[tx] = att.re;
        s_ai[tx] = att.im;
        s_im[tx] = imc;
    }
    // read: lanes along i
    for (int q = ty; q < AT; q += 8) {
        const int jj = jj0 + q, i = i0 + tx;
        double pr = 0.0, pi = 0.0, mr = 0.0, mi = 0.0;
        if (jj < d && i < d) {
            const double w = a.wi[vb + jj];
            const int j = (w < 0.0) ? jj - 1 : jj;
            const size_t cb = om * d * d + (size_t)j * d;
            pr = a.psi_p[cb + i];
            mr = a.psi_m[cb + i];
            if (w != 0.0) {
                pi = a.psi_p[cb + d + i];
                mi = a.psi_m[cb + d + i];
            }
        }
        s_pr[q][tx] = pr;
        s_pi[q][tx] = pi;
        s_mr[q][tx] = mr;
        s_mi[q][tx] = mi;
    }
    __syncthreads();
    auto pk = [&](cplx v, int q) { return s_im[q] ? v.im : v.re; };
    // tau = 0 stacks of the top layer: T0[mo][jj][i] (column-major in jj), lanes along i
    if (p == 0) {
        double* T0 = a.top0 + (size_t)mo * d * 2 * d;
        for (int q = ty; q < AT; q += 8) {
            const int jj = jj0 + q, i = i0 + tx;
            if (jj >= d || i >= d) continue;
            const cplx pp = cmk(s_pr[q][tx], s_pi[q][tx]), pm = cmk(s_mr[q][tx], s_mi[q][tx]);
            const cplx att = cmk(s_ar[q], s_ai[q]);
            T0[(size_t)jj * d + i] = pk(pp, q);
            T0[(size_t)(d + jj) * d + i] = pk(att * pm, q);
        }
    }
    // write: lanes along jj (the system's columns)
    double* A = a.lhs + (size_t)mo * a.sl;
    double* A0 = a.lhs0 ? a.lhs0 + (size_t)mo * a.sl : nullptr;
    const int jj = jj0 + tx, q = tx;
    if (jj >= d) return;
    const int ca = bnd_col(p, jj, d, G);       // column A_p(jj)
    const int cbk = bnd_col(p, d + jj, d, G);  // column B_p(jj)
    const cplx att = cmk(s_ar[q], s_ai[q]);
    auto put = [&](int r, int c, double v) {
        const size_t o = (size_t)bnd_row(r, d, G) * a.ldl + c;
        A[o] = v;
        if (A0) A0[o] = v;
    };
    for (int ii = ty; ii < AT; ii += 8) {
        const int i = i0 + ii;
        if (i >= d) break;
        const cplx pp = cmk(s_pr[q][ii], s_pi[q][ii]), pm = cmk(s_mr[q][ii], s_mi[q][ii]);
        if (p == 0) {
            if (a.p.refl_top) {
                // Fresnel interface (extension): top rows are down - R up = 0, R the
                // interface reflection of node i/4 applied to the upward Stokes vector
                const double* Rm = a.p.refl_top + (size_t)(i >> 2) * 16 + 4 * (i & 3);
                const int g0 = ii & ~3;
                cplx ua = cmk(0.0, 0.0), ub = cmk(0.0, 0.0);
                for (int k = 0; k < 4; ++k) {
                    const cplx ppk = cmk(s_pr[q][g0 + k], s_pi[q][g0 + k]);
                    const cplx pmk = cmk(s_mr[q][g0 + k], s_mi[q][g0 + k]);
                    ua = ua + Rm[k] * ppk;
                    ub = ub + Rm[k] * (att * pmk);
                }
                put(i, ca, pk(dflip(pm, i) - ua, q));
                put(i, cbk, pk(att * dflip(pp, i) - ub, q));
            } else {
                put(i, ca, pk(dflip(pm, i), q));
                put(i, cbk, pk(att * dflip(pp, i), q));
            }
        }
        if (p < P - 1) {
            const int ru = d + 2 * d * p;
            put(ru + i, ca, pk(att * pp, q));
            put(ru + d + i, ca, pk(att * dflip(pm, i), q));
            put(ru + i, cbk, pk(pm, q));
            put(ru + d + i, cbk, pk(dflip(pp, i), q));
        }
        if (p > 0) {
            const int ru = d + 2 * d * (p - 1);
            put(ru + i, ca, -pk(pp, q));
            put(ru + d + i, ca, -pk(dflip(pm, i), q));
            put(ru + i, cbk, -pk(att * pm, q));
            put(ru + d + i, cbk, -pk(att * dflip(pp, i), q));
        }
        if (p == P - 1) {
            const int rb = d + 2 * d * (P - 1);
            put(rb + i, ca, pk(att * pp, q));
            put(rb + i, cbk, pk(pm, q));
        }
    }
}

// reflect_downward_field (boundary.cpp:73-97) of a real packed vector v.
__device__ void reflect_rows(const ProblemDev& p, const double* v, int d, int lane, double* out) {
    const int N = p.N;
    if (p.base_type == 1) {
        double f = 0.0;
        for (int n = lane; n < N; n += 32) f += p.weights[n] * p.nodes[n] * v[4 * n];
        // fixed-order reduction for determinism
        f = warp_sum(f);
        const double val = 2.0 * p.rho * f;
        for (int i = lane; i < d; i += 32) out[i] = ((i & 3) == 0) ? val : 0.0;
    } else {
        for (int i = lane; i < d; i += 32) {
            const int ni = i >> 2, r = i & 3;
            double acc = 0.0;
            for (int n = 0; n < N; ++n) {
                const double* t = p.table + ((size_t)ni * p.table_n + n) * 16 + 4 * r;
                const double s = t[0] * v[4 * n] + t[1] * v[4 * n + 1] + t[2] * v[4 * n + 2] +
                                 t[3] * v[4 * n + 3];
                acc += p.weights[n] * p.nodes[n] * s;
            }
            out[i] = acc;
        }
    }
}

// m = 0 base reflection of the bottom layer's columns (boundary.cpp:99-140,
// 229-233).  Warp per (packed column, A|B).
__global__ void base_kernel(BndArgs a, int mo) {
    extern __shared__ double sm[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gw = blockIdx.x * (blockDim.x >> 5) + w;
    const int d = a.d, P = a.p.n_layers, G = 2 * d * P;
    if (gw >= 2 * d) return;
    const int jj = gw % d, isb = gw / d;
    const int q = P - 1;
    const size_t om = (size_t)a.p.medium[q] * a.p.n_orders + mo;
    double* v = sm + (size_t)w * 2 * d;
    double* out = v + d;
    const ModeView mv{a.psi_p, a.psi_m, a.nu, a.wi, d};
    for (int i = lane; i < d; i += 32) {
        cplx pp, pm, nu;
        bool imc;
        mv.load(om, jj, i, pp, pm, nu, imc);
        const cplx att = att_of(a.p.tau[q], nu);
        const cplx val = isb ? dflip(pp, i) : att * dflip(pm, i);
        v[i] = imc ? val.im : val.re;
    }
    __syncwarp();
    reflect_rows(a.p, v, d, lane, out);
    __syncwarp();
    double* A = a.lhs + (size_t)mo * a.sl;
    double* A0 = a.lhs0 ? a.lhs0 + (size_t)mo * a.sl : nullptr;
    const int col = bnd_col(q, (isb ? d : 0) + jj, d, G);
    const int rb = d + 2 * d * (P - 1);
    for (int i = lane; i < d; i += 32) {
        const size_t o = (size_t)bnd_row(rb + i, d, G) * a.ldl + col;
        A[o] -= out[i];
        if (A0) A0[o] -= out[i];
    }
}

// Right-hand sides: warp per (order mo, column = incident*4 + channel).
// CTA per (order, RHS_TW consecutive columns), warp per column: the columns are
// built in a shared-memory tile [G][RHS_TW] and written to the augmented system
// and its untouched copy as whole row segments (a warp writing one column of
// the row-major system would touch one 32-byte sector per element).
template <int RHS_TW>
__device__ void rhs_column(const BndArgs& a, int mo, int col, double* tile, double* sm, int w, int lane);

template <int RHS_TW>
__global__ void rhs_kernel(BndArgs a) {
    extern __shared__ double shm[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int d = a.d, P = a.p.n_layers, G = 2 * d * P, R = 4 * a.p.n_in;
    const int mo = blockIdx.y, col0 = blockIdx.x * RHS_TW, col = col0 + w;
    double* tile = shm;                              // [G][RHS_TW]
    double* sm = shm + (size_t)G * RHS_TW;           // per-warp scratch [2d]
    if (col < R) rhs_column<RHS_TW>(a, mo, col, tile, sm, w, lane);
    __syncthreads();
    const int nc = min(RHS_TW, R - col0);
    double* A = a.lhs + (size_t)mo * a.sl + G + col0;
    double* A0 = a.lhs0 ? a.lhs0 + (size_t)mo * a.sl + G + col0 : nullptr;
    for (int e = threadIdx.x; e < G * RHS_TW; e += blockDim.x) {
        const int r = e / RHS_TW, cc = e % RHS_TW;
        if (cc >= nc) continue;
        const double v = tile[e];
        A[(size_t)r * a.ldl + cc] = v;
        if (A0) A0[(size_t)r * a.ldl + cc] = v;
    }
}

template <int RHS_TW>
__device__ void rhs_column(const BndArgs& a, int mo, int col, double* tile, double* sm, int w, int lane) {
    const int d = a.d, P = a.p.n_layers, G = 2 * d * P, R = 4 * a.p.n_in;
    const int ii = col / 4, c = col % 4;
    const int m = a.p.order_of(mo);
    const double mu0 = a.p.mu_in[ii];
    // row-major [G][R] per order (lu.cu); B(r) = rhs[mo][r * R + col]
    // writes B (and its untouched copy in lhs0), accumulating max|b| and ||b||_1
    double bmax = 0.0, b1 = 0.0;
    struct Ref {
        double* x;
        double* bmax;
        double* b1;
        __device__ void operator=(double v) const {
            *x = v;
            *bmax = fmax(*bmax, fabs(v));
            *b1 += fabs(v);
        }
    };
    struct RowView {  // storage row bnd_row(r) of this column in the tile
        double* base;
        int d, G;
        double* bmax;
        double* b1;
        __device__ Ref operator[](int r) const {
            return Ref{base + (size_t)bnd_row(r, d, G) * RHS_TW, bmax, b1};
        }
    } B{tile + w, d, G, &bmax, &b1};
    auto finish_norms = [&]() {
        if (!a.bnorm) return;
        const double mx = warp_max(bmax), s1 = warp_sum(b1);
        if (lane == 0) {
            a.bnorm[2 * ((size_t)mo * R + col)] = mx;
            a.bnorm[2 * ((size_t)mo * R + col) + 1] = s1;
        }
    };
    auto zp = [&](int p, int i) {
        const size_t om = (size_t)a.p.medium[p] * a.p.n_orders + mo;
        return a.zp[(om * R + col) * d + i];
    };
    auto zm = [&](int p, int i) {
        const size_t om = (size_t)a.p.medium[p] * a.p.n_orders + mo;
        return a.zm[(om * R + col) * d + i];
    };
    if (a.p.refl_top) {  // Fresnel interface: down - R up = -Z- + R Z+ at tau = 0
        for (int i = lane; i < d; i += 32) {
            const double* Rm = a.p.refl_top + (size_t)(i >> 2) * 16 + 4 * (i & 3);
            double r = -zm(0, i);
            for (int q = 0; q < 4; ++q) r += Rm[q] * zp(0, (i & ~3) + q);
            B[i] = r;
        }
    } else {
        for (int i = lane; i < d; i += 32) B[i] = -zm(0, i);
    }
    double tau_top = 0.0;
    for (int p = 0; p + 1 < P; ++p) {
        tau_top += a.p.tau[p];
        const double bn = exp(-tau_top / mu0);
        const int ru = d + 2 * d * p;
        for (int i = lane; i < d; i += 32) {
            B[ru + i] = bn * (zp(p + 1, i) - zp(p, i));
            B[ru + d + i] = bn * (zm(p + 1, i) - zm(p, i));
        }
    }
    const double tau_total = tau_top + a.p.tau[P - 1];
    const double bb = exp(-tau_total / mu0);
    const int rb = d + 2 * d * (P - 1), q = P - 1;
    const bool active = m == 0 && a.p.base_type != 0 && !(a.p.base_type == 1 && a.p.rho == 0.0);
    if (!active) {
        for (int i = lane; i < d; i += 32) B[rb + i] = -(bb * zp(q, i));
        finish_norms();
        return;
    }
    double* v = sm + (size_t)w * 2 * d;
    (void)R;
    double* out = v + d;
    for (int i = lane; i < d; i += 32) v[i] = bb * zm(q, i);
    __syncwarp();
    reflect_rows(a.p, v, d, lane, out);
    __syncwarp();
    const int kc = (c < 2) ? 1 : 2;
    for (int i = lane; i < d; i += 32) {
        const int n = i >> 2, r = i & 3;
        const double* R4 = a.p.beam_rows + ((size_t)ii * a.p.N + n) * 16;
        double s = (mu0 / kPi) * R4[4 * r + c] * bb;
        if ((kc == 1) != (r < 2)) s = 0.0;
        B[rb + i] = -(bb * zp(q, i)) + (out[i] + s);
    }
    finish_norms();
}

// up = Z+ of the top layer (then += Top0 * coefficients by GEMM).
__global__ void copy_zp0_kernel(BndArgs a) {
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const int d = a.d, R = 4 * a.p.n_in;
    const long long total = (long long)a.p.n_orders * R * d;
    if (idx >= total) return;
    const int mo = (int)(idx / ((long long)R * d));
    const size_t om = (size_t)a.p.medium[0] * a.p.n_orders + mo;
    const long long rest = idx % ((long long)R * d);
    a.up[idx] = a.zp[om * R * d + rest];
}

// Per order: max |A_ij| and ||A||_1 (max column sum) of the untouched copy.
// CTA per (order, 256-column slab); thread per column, rows looped (coalesced).
__global__ void bnd_anorm_kernel(BndArgs a, int G) {
    const int mo = blockIdx.y, c = blockIdx.x * blockDim.x + threadIdx.x;
    __shared__ double red[32];
    double mx = 0.0, cs = 0.0;
    if (c < G) {
        // rows split over blockIdx.z; 8 loads in flight per thread
        const int r0 = blockIdx.z * (G / gridDim.z), r1 = blockIdx.z + 1 == gridDim.z ? G : r0 + G / gridDim.z;
        const double* A0 = a.lhs0 + (size_t)mo * a.sl + c;
        int r = r0;
        for (; r + 8 <= r1; r += 8) {
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = fabs(A0[(size_t)(r + q) * a.ldl]);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                mx = fmax(mx, v[q]);
                cs += v[q];
            }
        }
        for (; r < r1; ++r) {
            const double v = fabs(A0[(size_t)r * a.ldl]);
            mx = fmax(mx, v);
            cs += v;
        }
    }
    // column sums of the row strips meet in colsum; the last strip's CTA of a
    // column slab (atomic ticket) reduces them into ||A||_1
    mx = block_max(mx, red);
    if (threadIdx.x == 0) atomic_max_double(&a.anorm[2 * mo], mx);
    if (c < G) atomicAdd(&a.colsum[(size_t)mo * G + c], cs);
    __threadfence();
    __shared__ unsigned ticket;
    if (threadIdx.x == 0) ticket = atomicAdd(&a.colsum_ticket[(size_t)mo * gridDim.x + blockIdx.x], 1u);
    __syncthreads();
    if (ticket + 1 != gridDim.z) return;
    __threadfence();
    double tot = c < G ? atomicAdd(&a.colsum[(size_t)mo * G + c], 0.0) : 0.0;
    tot = block_max(tot, red);
    if (threadIdx.x == 0) atomic_max_double(&a.anorm[2 * mo + 1], tot);
}

// Thread per (order, right-hand side): residual column of lhs0's B part after
// bnd_residual_gemm, solution X [mo][G][R] (row-major, unknown order).
__global__ void bnd_check_kernel(BndArgs a, const double* X, int G, int R, int stage, DeviceStatus* status) {
    const int mo = blockIdx.y, r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= R) return;
    const double* res = a.lhs0 + (size_t)mo * a.sl + G + r;
    const double* x = X + (size_t)mo * G * R + r;
    double rmax = 0.0, xmax = 0.0, x1 = 0.0;
    bool finite = true;
    for (int n = 0; n < G; ++n) {
        const double v = res[(size_t)n * a.ldl], xv = x[(size_t)n * R];
        finite = finite && isfinite(xv);
        rmax = fmax(rmax, fabs(v));
        xmax = fmax(xmax, fabs(xv));
        x1 += fabs(xv);
    }
    const double bmax = a.bnorm[2 * ((size_t)mo * R + r)], b1 = a.bnorm[2 * ((size_t)mo * R + r) + 1];
    const double amax = a.anorm[2 * mo], a1 = a.anorm[2 * mo + 1];
    const double scale = amax * fmax(xmax, 1e-300) + bmax;
    const double rel = bmax > 0.0 ? rmax / scale : 0.0;
    // lower bound of cond_1(A): ||A||_1 ||A^-1 b||_1 / ||b||_1
    const double cond = b1 > 0.0 ? a1 * x1 / b1 : 0.0;
    atomic_max_double(&a.condm[mo], cond);
    atomic_max_double(&status->max_boundary_residual, rel);
    atomic_max_double(&a.resm[mo], rel);
    const int m = a.p.order_of(mo);
    if (!finite || !(rmax == rmax)) {
        report_failure(status, kFailBoundary, 3, m, rmax, cond);
        return;
    }
    if (stage == 0) {  // per right-hand side, as the reference (boundary.cpp:244-248)
        const int refine = rmax > 1e-10 * scale;
        a.col_refine[(size_t)mo * R + r] = refine;
        if (refine) atomicExch(&status->bnd_refine, 1);
    }
    if (stage == 1 && bmax > 0.0 && rmax > 1e-9 * scale) report_failure(status, kFailBoundary, 3, m, rmax, cond);
}

// Refinement right-hand side: dX <- -(A x - b) gathered through the row map.
__global__ void bnd_refine_rhs_kernel(BndArgs a, const int* perm_all, double* dX, int G, int R) {
    const long long total = (long long)a.p.n_orders * G * R;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(e % R);
        const long long rb = e / R;
        const int i = (int)(rb % G), mo = (int)(rb / G);
        dX[e] = -a.lhs0[(size_t)mo * a.sl + (size_t)perm_all[(size_t)mo * G + i] * a.ldl + G + c];
    }
}

// X += dX on the right-hand sides flagged for refinement (X, dX [mo][G][R]).
__global__ void add_kernel(double* X, const double* dX, const int* col_refine, int G, int R, long long n) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
        if (col_refine[(e / ((long long)G * R)) * R + e % R]) X[e] += dX[e];
}

__device__ inline double probe_weight(int k, int c) {
    unsigned long long z = 0x9E3779B97F4A7C15ull * (unsigned long long)(k * 7919 + c + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return (double)(z >> 11) * 0x1.0p-52 - 1.0;  // uniform in [-1, 1)
}

// Warp per (order, row i): the forward-eliminated combination probes y_k(i) =
// sum_c v_k(c) Y(perm[i], c) and their b_k(i) = sum_c v_k(c) B0(i, c) (storage
// row i of the untouched copy), both read coalesced along the row; the random
// probes b_k(r) = w_k(r), gathered through the row map into Xp.
__global__ void bnd_probe_setup_kernel(BndArgs a, const int* perm_all, double* Xp, int G, int R) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long gw = blockIdx.x * (long long)(blockDim.x >> 5) + w;
    if (gw >= (long long)a.p.n_orders * G) return;
    const int mo = (int)(gw / G), i = (int)(gw % G);
    const int pi = perm_all[(size_t)mo * G + i];
    const double* y = a.lhs + (size_t)mo * a.sl + (size_t)pi * a.ldl + G;
    double* b0 = a.lhs0 + (size_t)mo * a.sl + (size_t)i * a.ldl + G;
    double ay[kBndCombProbes], ab[kBndCombProbes];
#pragma unroll
    for (int k = 0; k < kBndCombProbes; ++k) ay[k] = ab[k] = 0.0;
    for (int c = lane; c < R; c += 32) {
        const double yv = y[c], bv = b0[c];
#pragma unroll
        for (int k = 0; k < kBndCombProbes; ++k) {
            const double v = probe_weight(k, c);
            ay[k] = fma(v, yv, ay[k]);
            ab[k] = fma(v, bv, ab[k]);
        }
    }
#pragma unroll
    for (int k = 0; k < kBndCombProbes; ++k) {
        ay[k] = warp_sum(ay[k]);
        ab[k] = warp_sum(ab[k]);
    }
    double* xp = Xp + ((size_t)mo * G + i) * kBndProbes;
    if (lane < kBndProbes) {
        double xv, bv;
        if (lane < kBndCombProbes) {
            xv = lane == 0 ? ay[0] : ay[1];
            bv = lane == 0 ? ab[0] : ab[1];
        } else {
            xv = probe_weight(lane + 64, pi);
            bv = probe_weight(lane + 64, i);
        }
        xp[lane] = xv;
        b0[R + lane] = bv;
    }
}

// Warp per (order, probe): residual A0 x_k - b_k (Rp holds A0 x_k), the
// reference's relative measure and the cond_1 lower bound; plus, warp per
// (order, right-hand side), finiteness of the solved rows >= row_lo.
__global__ void bnd_probe_check_kernel(BndArgs a, const double* Xp, const double* Rp, const double* X, int row_lo,
                                       int G, int R, DeviceStatus* status) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long gw = blockIdx.x * (long long)(blockDim.x >> 5) + w;
    const int K = a.K, NO = a.p.n_orders;
    if (gw < (long long)NO * K) {
        const int mo = (int)(gw / K), k = (int)(gw % K);
        const double* b = a.lhs0 + (size_t)mo * a.sl + G + R + k;
        const double* x = Xp + (size_t)mo * G * K + k;
        const double* ax = Rp + (size_t)mo * G * K + k;
        double rmax = 0.0, bmax = 0.0, b1 = 0.0, xmax = 0.0, x1 = 0.0;
        bool finite = true;
        for (int n = lane; n < G; n += 32) {
            const double bv = b[(size_t)n * a.ldl], xv = x[(size_t)n * K];
            const double rv = ax[(size_t)n * K] - bv;
            finite = finite && isfinite(xv) && isfinite(rv);
            rmax = fmax(rmax, fabs(rv));
            bmax = fmax(bmax, fabs(bv));
            b1 += fabs(bv);
            xmax = fmax(xmax, fabs(xv));
            x1 += fabs(xv);
        }
        rmax = warp_max(rmax);
        bmax = warp_max(bmax);
        xmax = warp_max(xmax);
        b1 = warp_sum(b1);
        x1 = warp_sum(x1);
        finite = __all_sync(0xffffffffu, finite);
        if (lane == 0) {
            const double amax = a.anorm[2 * mo], a1 = a.anorm[2 * mo + 1];
            const double scale = amax * fmax(xmax, 1e-300) + bmax;
            const double rel = bmax > 0.0 ? rmax / scale : 0.0;
            const double cond = b1 > 0.0 ? a1 * x1 / b1 : 0.0;
            atomic_max_double(&a.condm[mo], cond);
            atomic_max_double(&status->max_boundary_residual, rel);
            atomic_max_double(&a.resm[mo], rel);
            if (!finite || !(rel <= 1e-10)) {
                atomicExch(&status->bnd_fallback, 1);
                atomicExch(&a.order_fail[mo], 1);
            }
        }
        return;
    }
    const long long q = gw - (long long)NO * K;
    if (q >= (long long)NO * R) return;
    const int mo = (int)(q / R), c = (int)(q % R);
    const double* x = X + (size_t)mo * G * R + c;
    bool finite = true;
    for (int n = row_lo + lane; n < G; n += 32) finite = finite && isfinite(x[(size_t)n * R]);
    finite = __all_sync(0xffffffffu, finite);
    if (lane == 0 && !finite) {
        atomicExch(&status->bnd_fallback, 1);
        atomicExch(&a.order_fail[mo], 1);
    }
}

__global__ void bnd_keep_kernel(BndArgs a, const double* saved) {
    const long long per = (long long)4 * a.p.n_in * a.d, total = (long long)a.p.n_orders * per;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x)
        if (!a.order_fail[e / per]) a.up[e] = saved[e];
}

__global__ void bnd_gather_b_kernel(BndArgs a, const int* perm_all, double* X, int G, int R) {
    const long long total = (long long)a.p.n_orders * G * R;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(e % R);
        const long long rb = e / R;
        const int i = (int)(rb % G), mo = (int)(rb / G);
        X[e] = a.lhs0[(size_t)mo * a.sl + (size_t)perm_all[(size_t)mo * G + i] * a.ldl + G + c];
    }
}

}  // namespace

void launch_bnd_norms(const BndArgs& a, int G, int R, cudaStream_t st) {
    (void)R;
    VRTE_CUDA_CHECK(cudaMemsetAsync(a.anorm, 0, sizeof(double) * 2 * (size_t)a.p.n_orders, st));
    VRTE_CUDA_CHECK(cudaMemsetAsync(a.colsum, 0, sizeof(double) * (size_t)a.p.n_orders * G, st));
    const int slabs = (G + 255) / 256;
    VRTE_CUDA_CHECK(cudaMemsetAsync(a.colsum_ticket, 0, sizeof(unsigned) * (size_t)a.p.n_orders * slabs, st));
    bnd_anorm_kernel<<<dim3(slabs, a.p.n_orders, 8), 256, 0, st>>>(a, G);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

// lhs0's B columns <- A x - b (or += A dx with accumulate): row-major
// Res (G x R) = A (G x G) X (G x R) - B, i.e. the column-major
// Res^T = X^T A^T - B^T with every operand read in place.
// The matrix is block sparse: each row block of equations touches the columns
// of at most two layers (bnd_row / bnd_col orders: interface p rows [2dp, 2dp+2d)
// hold layers p and p+1, the bottom rows layer P-1, the top rows layer 0), so
// the product runs per row block over its nonzero column range only.
namespace {
// C (row-major, ncol columns) = A0 X - (beta_first = -1: C's old value, i.e. b)
// over the nonzero column range of each row block.
void bnd_apply(const BndArgs& a, const double* X, long long ldx, long long sx, int ncol, double* C, long long ldc,
               long long sc, double beta_first, int G, cudaStream_t st) {
    const int d = a.d, P = a.p.n_layers;
    struct Seg {
        int r0, nr, c0, nc;
    };
    std::vector<Seg> segs;
    auto layer_cols = [&](int p) { return p == 0 ? G - 2 * d : 2 * d * (p - 1); };
    if (P == 1) {
        segs.push_back({0, G, 0, G});
    } else {
        for (int p = 0; p + 1 < P; ++p) {  // interface p: layers p, p+1
            const int c0 = layer_cols(p), c1 = layer_cols(p + 1);
            if (c1 == c0 + 2 * d)
                segs.push_back({2 * d * p, 2 * d, c0, 4 * d});
            else if (P == 2)
                segs.push_back({2 * d * p, 2 * d, 0, G});
            else {
                segs.push_back({2 * d * p, 2 * d, c0, 2 * d});
                segs.push_back({2 * d * p, 2 * d, c1, 2 * d});
            }
        }
        segs.push_back({2 * d * (P - 1), d, layer_cols(P - 1), 2 * d});  // bottom
        segs.push_back({G - d, d, layer_cols(0), 2 * d});                // top
    }
    std::vector<int> seen(G, 0);
    for (const Seg& q : segs) {
        GemmBatch g{};
        g.m = ncol;
        g.n = q.nr;
        g.k = q.nc;
        g.a = X + (size_t)q.c0 * ldx;
        g.lda = ldx;
        g.stride_a = sx;
        g.b = a.lhs0 + (size_t)q.r0 * a.ldl + q.c0;
        g.ldb = a.ldl;
        g.stride_b = a.sl;
        g.c = C + (size_t)q.r0 * ldc;
        g.ldc = ldc;
        g.stride_c = sc;
        g.batch = a.p.n_orders;
        g.alpha = 1.0;
        g.beta = seen[q.r0] ? 1.0 : beta_first;
        seen[q.r0] = 1;
        gemm_batched(g, st);
    }
}
}  // namespace

void launch_bnd_residual(const BndArgs& a, const double* X, int G, int R, bool accumulate, cudaStream_t st) {
    bnd_apply(a, X, R, (long long)G * R, R, a.lhs0 + G, a.ldl, a.sl, accumulate ? 1.0 : -1.0, G, st);
}

void launch_bnd_check(const BndArgs& a, const double* X, int G, int R, int stage, DeviceStatus* status,
                      cudaStream_t st) {
    bnd_check_kernel<<<dim3((R + 127) / 128, a.p.n_orders), 128, 0, st>>>(a, X, G, R, stage, status);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

void launch_bnd_refine_rhs(const BndArgs& a, const int* perm, double* dX, int G, int R, cudaStream_t st) {
    const long long total = (long long)a.p.n_orders * G * R;
    bnd_refine_rhs_kernel<<<(unsigned)std::min(16384LL, (total + 255) / 256), 256, 0, st>>>(a, perm, dX, G, R);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

void launch_bnd_add(const BndArgs& a, double* X, const double* dX, int G, int R, cudaStream_t st) {
    const long long n = (long long)a.p.n_orders * G * R;
    add_kernel<<<(unsigned)std::min(16384LL, (n + 255) / 256), 256, 0, st>>>(X, dX, a.col_refine, G, R, n);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

void launch_bnd_zero(const BndArgs& a, cudaStream_t st) {
    VRTE_CUDA_CHECK(cudaMemsetAsync(a.lhs, 0, sizeof(double) * (size_t)a.p.n_orders * a.sl, st));
}

void launch_bnd_assemble(const BndArgs& a, cudaStream_t st, bool zeroed) {
    const int d = a.d, P = a.p.n_layers, G = 2 * d * P;
    if (!zeroed) launch_bnd_zero(a, st);
    const dim3 grid((d + AT - 1) / AT, (d + AT - 1) / AT, (unsigned)(a.p.n_orders * P));
    assemble_kernel<<<grid, 256, 0, st>>>(a);
    VRTE_CUDA_CHECK(cudaGetLastError());
    const bool active = a.p.base_type != 0 && !(a.p.base_type == 1 && a.p.rho == 0.0);
    if (active) {
        for (int mo = 0; mo < a.p.n_orders; ++mo) {
            if (a.p.order_of(mo) != 0) continue;
            const int warps = 4;
            base_kernel<<<(2 * d + warps - 1) / warps, warps * 32, warps * 2 * d * sizeof(double),
                          st>>>(a, mo);
            VRTE_CUDA_CHECK(cudaGetLastError());
        }
    }
}

void launch_bnd_rhs(const BndArgs& a, cudaStream_t st) {
    // tile width 8 (64-byte row segments) while the tile fits, else 2
    const int R = 4 * a.p.n_in, G = 2 * a.d * a.p.n_layers;
    auto smem = [&](int tw) { return ((size_t)G * tw + (size_t)tw * 2 * a.d) * sizeof(double); };
    static unsigned long long attr8 = 0, attr2 = 0;
    if (smem(8) <= 200 * 1024) {
        smem_attr_once(rhs_kernel<8>, 200 * 1024, attr8);
        rhs_kernel<8><<<dim3((R + 7) / 8, a.p.n_orders), 8 * 32, smem(8), st>>>(a);
    } else {
        smem_attr_once(rhs_kernel<2>, 200 * 1024, attr2);
        rhs_kernel<2><<<dim3((R + 1) / 2, a.p.n_orders), 2 * 32, smem(2), st>>>(a);
    }
    VRTE_CUDA_CHECK(cudaGetLastError());
}

void launch_copy_zp0(const BndArgs& a, cudaStream_t st) {
    const long long total = (long long)a.p.n_orders * 4 * a.p.n_in * a.d;
    copy_zp0_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(a);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace vrte

namespace vrte {
void launch_bnd_probe_setup(const BndArgs& a, const int* perm, double* Xp, int G, int R, cudaStream_t st) {
    const long long warps = (long long)a.p.n_orders * G;
    bnd_probe_setup_kernel<<<(unsigned)((warps + 7) / 8), 256, 0, st>>>(a, perm, Xp, G, R);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

void launch_bnd_probe_check(const BndArgs& a, const double* Xp, double* Rp, const double* X, int row_lo, int G, int R,
                            DeviceStatus* status, cudaStream_t st) {
    const int K = a.K, NO = a.p.n_orders;
    bnd_apply(a, Xp, K, (long long)G * K, K, Rp, K, (long long)G * K, 0.0, G, st);
    const long long warps = (long long)NO * (K + R);
    bnd_probe_check_kernel<<<(unsigned)((warps + 7) / 8), 256, 0, st>>>(a, Xp, Rp, X, row_lo, G, R, status);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

void launch_bnd_gather_b(const BndArgs& a, const int* perm, double* X, int G, int R, cudaStream_t st) {
    const long long total = (long long)a.p.n_orders * G * R;
    bnd_gather_b_kernel<<<(unsigned)std::min(16384LL, (total + 255) / 256), 256, 0, st>>>(a, perm, X, G, R);
    VRTE_CUDA_CHECK(cudaGetLastError());
}
void launch_bnd_keep_passed(const BndArgs& a, const double* saved, cudaStream_t st) {
    const long long total = (long long)a.p.n_orders * 4 * a.p.n_in * a.d;
    bnd_keep_kernel<<<(unsigned)std::min(16384LL, (total + 255) / 256), 256, 0, st>>>(a, saved);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace vrte
