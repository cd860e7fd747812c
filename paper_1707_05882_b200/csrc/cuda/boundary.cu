// boundary.cu -- global boundary system per Fourier order, boundary.cpp:142-265.
//
// The reference assembles and factors a complex (2dP)^2 system for every
// (incident, basis vector, order) although its matrix carries no incident
// dependence (boundary.cpp:219).  Here the matrix is assembled ONCE per order
// in a real basis (conjugate mode pairs -> Re/Im columns), LU-factored once,
// and every (incident, Stokes channel) is a right-hand side of one blocked
// triangular solve.  The tau = 0 upward stack (boundary.cpp:20-35) is then a
// single GEMM per order against [psi+ | att psi-] of the top layer.
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

// Thread per (order mo, layer p, packed column jj, row i).
__global__ void assemble_kernel(BndArgs a) {
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const int d = a.d, P = a.p.n_layers, G = 2 * d * P;
    const long long total = (long long)a.p.n_orders * P * d * d;
    if (idx >= total) return;
    const int i = (int)(idx % d);
    const int jj = (int)((idx / d) % d);
    const int p = (int)((idx / ((long long)d * d)) % P);
    const int mo = (int)(idx / ((long long)d * d * P));
    const size_t om = (size_t)a.p.medium[p] * a.p.n_orders + mo;
    const ModeView mv{a.psi_p, a.psi_m, a.nu, a.wi, d};
    cplx pp, pm, nu;
    bool imc;
    mv.load(om, jj, i, pp, pm, nu, imc);
    const cplx att = att_of(a.p.tau[p], nu);
    auto pk = [&](cplx v) { return imc ? v.im : v.re; };
    double* A = a.lhs + (size_t)mo * G * G;
    const size_t ca = (size_t)(2 * d * p + jj) * G;      // column A_p(jj)
    const size_t cbk = (size_t)(2 * d * p + d + jj) * G;  // column B_p(jj)
    if (p == 0) {
        A[ca + i] = pk(dflip(pm, i));
        A[cbk + i] = pk(att * dflip(pp, i));
        double* T0 = a.top0 + (size_t)mo * d * 2 * d;
        T0[(size_t)jj * d + i] = pk(pp);
        T0[(size_t)(d + jj) * d + i] = pk(att * pm);
    }
    if (p < P - 1) {
        const int ru = d + 2 * d * p;
        A[ca + ru + i] = pk(att * pp);
        A[ca + ru + d + i] = pk(att * dflip(pm, i));
        A[cbk + ru + i] = pk(pm);
        A[cbk + ru + d + i] = pk(dflip(pp, i));
    }
    if (p > 0) {
        const int ru = d + 2 * d * (p - 1);
        A[ca + ru + i] = -pk(pp);
        A[ca + ru + d + i] = -pk(dflip(pm, i));
        A[cbk + ru + i] = -pk(att * pm);
        A[cbk + ru + d + i] = -pk(att * dflip(pp, i));
    }
    if (p == P - 1) {
        const int rb = d + 2 * d * (P - 1);
        A[ca + rb + i] = pk(att * pp);
        A[cbk + rb + i] = pk(pm);
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
    double* A = a.lhs + (size_t)mo * G * G;
    const size_t col = (size_t)(2 * d * q + (isb ? d : 0) + jj) * G;
    const int rb = d + 2 * d * (P - 1);
    for (int i = lane; i < d; i += 32) A[col + rb + i] -= out[i];
}

// Right-hand sides: warp per (order mo, column = incident*4 + channel).
__global__ void rhs_kernel(BndArgs a) {
    extern __shared__ double sm[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gw = blockIdx.x * (blockDim.x >> 5) + w;
    const int d = a.d, P = a.p.n_layers, G = 2 * d * P, R = 4 * a.p.n_in;
    if (gw >= a.p.n_orders * R) return;
    const int mo = gw / R, col = gw % R, ii = col / 4, c = col % 4;
    const int m = a.p.order_of(mo);
    const double mu0 = a.p.mu_in[ii];
    double* B = a.rhs + ((size_t)mo * R + col) * G;
    auto zp = [&](int p, int i) {
        const size_t om = (size_t)a.p.medium[p] * a.p.n_orders + mo;
        return a.zp[(om * R + col) * d + i];
    };
    auto zm = [&](int p, int i) {
        const size_t om = (size_t)a.p.medium[p] * a.p.n_orders + mo;
        return a.zm[(om * R + col) * d + i];
    };
    for (int i = lane; i < d; i += 32) B[i] = -zm(0, i);
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
        return;
    }
    double* v = sm + (size_t)w * 2 * d;
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
}

// ---------------------------------------------------------------- batched LU
// Panel factorization with partial pivoting, panel staged in shared memory.
__global__ void lu_panel_kernel(double* Aall, int G, int k0, int jb, int* ipiv_all,
                                DeviceStatus* status, const int* order_index) {
    extern __shared__ double P[];  // column-major np x jb
    __shared__ double rv[32];
    __shared__ int ri[32];
    __shared__ int s_piv;
    const int b = blockIdx.x, t = threadIdx.x, nt = blockDim.x;
    const int np = G - k0;
    double* A = Aall + (size_t)b * G * G;
    int* ipiv = ipiv_all + (size_t)b * G;
    for (int idx = t; idx < np * jb; idx += nt) {
        const int r = idx % np, c = idx / np;
        P[idx] = A[(size_t)(k0 + r) + (size_t)(k0 + c) * G];
    }
    __syncthreads();
    for (int j = 0; j < jb; ++j) {
        // argmax |P[r][j]|, r >= j (first index on ties)
        double best = -1.0;
        int bi = j;
        for (int r = j + t; r < np; r += nt) {
            const double v = fabs(P[(size_t)j * np + r]);
            if (v > best) {
                best = v;
                bi = r;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, best, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > best || (ov == best && oi < bi)) {
                best = ov;
                bi = oi;
            }
        }
        if ((t & 31) == 0) {
            rv[t >> 5] = best;
            ri[t >> 5] = bi;
        }
        __syncthreads();
        if (t == 0) {
            double bv = rv[0];
            int bidx = ri[0];
            for (int w = 1; w < (nt >> 5); ++w)
                if (rv[w] > bv || (rv[w] == bv && ri[w] < bidx)) {
                    bv = rv[w];
                    bidx = ri[w];
                }
            s_piv = bidx;
            ipiv[k0 + j] = k0 + bidx;
            if (bv == 0.0)
                report_failure(status, kFailLuSingular, 3, order_index ? order_index[b] : b,
                               (double)(k0 + j));
        }
        __syncthreads();
        const int pr = s_piv;
        if (pr != j)
            for (int c = t; c < jb; c += nt) {
                const double tmp = P[(size_t)c * np + j];
                P[(size_t)c * np + j] = P[(size_t)c * np + pr];
                P[(size_t)c * np + pr] = tmp;
            }
        __syncthreads();
        const double piv = P[(size_t)j * np + j];
        if (piv != 0.0) {
            const double rcp = 1.0 / piv;
            for (int r = j + 1 + t; r < np; r += nt) {
                const double l = P[(size_t)j * np + r] * rcp;
                P[(size_t)j * np + r] = l;
                for (int c = j + 1; c < jb; ++c) P[(size_t)c * np + r] -= l * P[(size_t)c * np + j];
            }
        }
        __syncthreads();
    }
    for (int idx = t; idx < np * jb; idx += nt) {
        const int r = idx % np, c = idx / np;
        A[(size_t)(k0 + r) + (size_t)(k0 + c) * G] = P[idx];
    }
}

// Row interchanges of the panel applied to every other column, then the
// unit-lower triangular solve for the U12 block row.  Thread per column.
__global__ void lu_swap_trsm_kernel(double* Aall, int G, int k0, int jb, const int* ipiv_all) {
    __shared__ double Lt[64 * 64];
    const int b = blockIdx.y;
    double* A = Aall + (size_t)b * G * G;
    const int* ipiv = ipiv_all + (size_t)b * G;
    for (int idx = threadIdx.x; idx < jb * jb; idx += blockDim.x) {
        const int r = idx % jb, c = idx / jb;
        Lt[r * 64 + c] = A[(size_t)(k0 + r) + (size_t)(k0 + c) * G];
    }
    __syncthreads();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= G || (c >= k0 && c < k0 + jb)) return;
    double* col = A + (size_t)c * G;
    for (int j = 0; j < jb; ++j) {
        const int pr = ipiv[k0 + j];
        if (pr != k0 + j) {
            const double tmp = col[k0 + j];
            col[k0 + j] = col[pr];
            col[pr] = tmp;
        }
    }
    if (c < k0) return;
    double x[64];
#pragma unroll 1
    for (int j = 0; j < jb; ++j) {
        double v = col[k0 + j];
        for (int i = 0; i < j; ++i) v -= Lt[j * 64 + i] * x[i];
        x[j] = v;
        col[k0 + j] = v;
    }
}

// getrs pieces: row interchanges on B, and the diagonal-block triangular
// solves of the blocked forward/backward substitution.  Thread per column.
__global__ void laswp_kernel(double* Ball, int G, int ncol, const int* ipiv_all) {
    const int b = blockIdx.y, c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncol) return;
    double* col = Ball + (size_t)b * G * ncol + (size_t)c * G;
    const int* ipiv = ipiv_all + (size_t)b * G;
    for (int i = 0; i < G; ++i) {
        const int pr = ipiv[i];
        if (pr != i) {
            const double tmp = col[i];
            col[i] = col[pr];
            col[pr] = tmp;
        }
    }
}

template <bool LOWER>
__global__ void trsm_diag_kernel(const double* Aall, double* Ball, int G, int ncol, int k0,
                                 int jb) {
    __shared__ double Tt[64 * 64];
    const int b = blockIdx.y;
    const double* A = Aall + (size_t)b * G * G;
    for (int idx = threadIdx.x; idx < jb * jb; idx += blockDim.x) {
        const int r = idx % jb, c = idx / jb;
        Tt[r * 64 + c] = A[(size_t)(k0 + r) + (size_t)(k0 + c) * G];
    }
    __syncthreads();
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncol) return;
    double* col = Ball + (size_t)b * G * ncol + (size_t)c * G + k0;
    double x[64];
    if (LOWER) {
#pragma unroll 1
        for (int j = 0; j < jb; ++j) {
            double v = col[j];
            for (int i = 0; i < j; ++i) v -= Tt[j * 64 + i] * x[i];
            x[j] = v;
        }
    } else {
#pragma unroll 1
        for (int j = jb - 1; j >= 0; --j) {
            double v = col[j];
            for (int i = j + 1; i < jb; ++i) v -= Tt[j * 64 + i] * x[i];
            x[j] = v / Tt[j * 64 + j];
        }
    }
    for (int j = 0; j < jb; ++j) col[j] = x[j];
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

}  // namespace

void launch_bnd_assemble(const BndArgs& a, cudaStream_t st) {
    const int d = a.d, P = a.p.n_layers, G = 2 * d * P;
    VRTE_CUDA_CHECK(cudaMemsetAsync(a.lhs, 0, sizeof(double) * (size_t)a.p.n_orders * G * G, st));
    const long long total = (long long)a.p.n_orders * P * d * d;
    assemble_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(a);
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
    const int warps = 4;
    const long long total = (long long)a.p.n_orders * 4 * a.p.n_in;
    rhs_kernel<<<(unsigned)((total + warps - 1) / warps), warps * 32,
                 warps * 2 * a.d * sizeof(double), st>>>(a);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

void lu_factor_batched(double* A, int G, int batch, int* ipiv, DeviceStatus* status,
                       const int* order_index, cudaStream_t st) {
    const int nb = 16;
    static bool attr = false;
    if (!attr) {
        VRTE_CUDA_CHECK(cudaFuncSetAttribute(lu_panel_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        attr = true;
    }
    for (int k0 = 0; k0 < G; k0 += nb) {
        const int jb = min(nb, G - k0);
        const size_t smem = (size_t)(G - k0) * jb * sizeof(double);
        lu_panel_kernel<<<batch, 256, smem, st>>>(A, G, k0, jb, ipiv, status, order_index);
        VRTE_CUDA_CHECK(cudaGetLastError());
        dim3 g2((G + 127) / 128, batch);
        lu_swap_trsm_kernel<<<g2, 128, 0, st>>>(A, G, k0, jb, ipiv);
        VRTE_CUDA_CHECK(cudaGetLastError());
        const int rest = G - k0 - jb;
        if (rest > 0) {
            GemmBatch g{};
            g.m = rest;
            g.n = rest;
            g.k = jb;
            g.a = A + (k0 + jb) + (size_t)k0 * G;
            g.lda = G;
            g.stride_a = (long long)G * G;
            g.b = A + k0 + (size_t)(k0 + jb) * G;
            g.ldb = G;
            g.stride_b = (long long)G * G;
            g.c = A + (k0 + jb) + (size_t)(k0 + jb) * G;
            g.ldc = G;
            g.stride_c = (long long)G * G;
            g.batch = batch;
            g.alpha = -1.0;
            g.beta = 1.0;
            gemm_batched(g, st);
        }
    }
}

void lu_solve_batched(const double* A, int G, int batch, const int* ipiv, double* B, int ncol,
                      cudaStream_t st) {
    const int nb = 64;
    dim3 gc((ncol + 127) / 128, batch);
    laswp_kernel<<<gc, 128, 0, st>>>(B, G, ncol, ipiv);
    VRTE_CUDA_CHECK(cudaGetLastError());
    for (int k0 = 0; k0 < G; k0 += nb) {
        const int jb = min(nb, G - k0);
        trsm_diag_kernel<true><<<gc, 128, 0, st>>>(A, B, G, ncol, k0, jb);
        VRTE_CUDA_CHECK(cudaGetLastError());
        const int rest = G - k0 - jb;
        if (rest > 0) {
            GemmBatch g{};
            g.m = rest;
            g.n = ncol;
            g.k = jb;
            g.a = A + (k0 + jb) + (size_t)k0 * G;
            g.lda = G;
            g.stride_a = (long long)G * G;
            g.b = B + k0;
            g.ldb = G;
            g.stride_b = (long long)G * ncol;
            g.c = B + k0 + jb;
            g.ldc = G;
            g.stride_c = (long long)G * ncol;
            g.batch = batch;
            g.alpha = -1.0;
            g.beta = 1.0;
            gemm_batched(g, st);
        }
    }
    const int nblk = (G + nb - 1) / nb;
    for (int bk = nblk - 1; bk >= 0; --bk) {
        const int k0 = bk * nb, jb = min(nb, G - k0);
        trsm_diag_kernel<false><<<gc, 128, 0, st>>>(A, B, G, ncol, k0, jb);
        VRTE_CUDA_CHECK(cudaGetLastError());
        if (k0 > 0) {
            GemmBatch g{};
            g.m = k0;
            g.n = ncol;
            g.k = jb;
            g.a = A + (size_t)k0 * G;
            g.lda = G;
            g.stride_a = (long long)G * G;
            g.b = B + k0;
            g.ldb = G;
            g.stride_b = (long long)G * ncol;
            g.c = B;
            g.ldc = G;
            g.stride_c = (long long)G * ncol;
            g.batch = batch;
            g.alpha = -1.0;
            g.beta = 1.0;
            gemm_batched(g, st);
        }
    }
}

int lu_launch_count(int G, int ncol) {
    const int nbf = 16, nbs = 64;
    const int panels = (G + nbf - 1) / nbf, blocks = (G + nbs - 1) / nbs;
    (void)ncol;
    return 3 * panels - 1 + 1 + 4 * blocks - 2;
}

void launch_copy_zp0(const BndArgs& a, cudaStream_t st) {
    const long long total = (long long)a.p.n_orders * 4 * a.p.n_in * a.d;
    copy_zp0_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(a);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace vrte
