// phase.cu -- generalized spherical function tables, the per-order phase-matrix
// Fourier kernels folded straight into the reduced operators E, F, and the
// beam-source columns.
//
// Reference: wigner.cpp:11-81 (recurrences), kernel.cpp:29-65 (A^m blocks),
// kernel.cpp:89-109 (beam column), homogeneous.cpp:43-73 (E, F),
// particular.cpp:7-25 (X+-).  The 4x4 products are written out with the
// 2+2 block sparsity of Pi_l and B_l (14 of 16 kernel entries are nonzero).
#include "kernels.cuh"

namespace vrte {
namespace {

// wigner.cpp:11-27: d^lmin_{m n}(x) = exp(lf) 2^-lmin (1-x)^{|m-n|/2} (1+x)^{|m+n|/2},
// lf = (1/2) log((2 lmin)! / (|m-n|! |m+n|!)) -- the x-independent part once per (m, n)
// (one warp: the lanes sum strided terms, then a butterfly)
__device__ double wigner_logfac(int m, int n) {
    const int lane = threadIdx.x & 31;
    const int lmin = max(abs(m), abs(n));
    const int a = abs(m - n), b = abs(m + n);
    double lf = 0.0;
    for (int k = 2 + lane; k <= 2 * lmin; k += 32) lf += log((double)k);
    for (int k = 2 + lane; k <= a; k += 32) lf -= log((double)k);
    for (int k = 2 + lane; k <= b; k += 32) lf -= log((double)k);
    lf = warp_sum(lf);
    return 0.5 * lf - lmin * log(2.0);
}
__device__ double wigner_start(int m, int n, double x, double lf) {
    const int a = abs(m - n), b = abs(m + n);
    double v = exp(lf);
    v *= pow(fmax(0.0, 1.0 - x), 0.5 * a) * pow(fmax(0.0, 1.0 + x), 0.5 * b);
    if (n < m && ((m - n) & 1)) v = -v;
    return v;
}

// CTA per order m, thread per mu: the three d^l_{m n} sequences (n = 0, 2, -2) by
// the upward recurrence (wigner.cpp:31-62), combined into P, R, T
// (wigner.cpp:64-81).  The recurrence coefficients depend on (l, m, n) only:
// tabulated once per CTA in shared memory as
//   d^{l}= (ca x + cb) d^{l-1} - cc d^{l-2},  ca = (2l-1)(l-1) l / c0,
//   cb = -(2l-1) m n / c0,  cc = l sqrt(((l-1)^2 - m^2)((l-1)^2 - n^2)) / c0,
//   c0 = (l-1) sqrt((l^2 - m^2)(l^2 - n^2)),
// so each step is three FMAs instead of two square roots and a division.
// Output layout: out[((m*Lc + l)*3 + {P,R,T})*ld + mu_index], l < Lc (coefficient count).
__global__ void gsf_kernel(int n_m, int L, int count, const double* __restrict__ mus,
                           double sign_mu, double* __restrict__ out, int ld) {
    extern __shared__ double coef[];  // [L][3][3]: ca, cb, cc per (l, q)
    __shared__ double s_lf[3];
    const int m = blockIdx.x;
    const int ns[3] = {0, 2, -2};
    for (int e = threadIdx.x; e < 3 * L; e += blockDim.x) {
        const int l = e / 3, q = e % 3, n = ns[q];
        const int lm = l - 1;
        double ca = 0.0, cb = 0.0, cc = 0.0;
        if (lm >= 1 && l > max(m, abs(n))) {
            const double lp = l;
            const double c0 = lm * sqrt((lp * lp - (double)m * m) * (lp * lp - (double)n * n));
            const double rc0 = 1.0 / c0;
            ca = (2.0 * lm + 1.0) * (lm * lp) * rc0;
            cb = -(2.0 * lm + 1.0) * ((double)m * n) * rc0;
            cc = lp * sqrt(((double)lm * lm - (double)m * m) * ((double)lm * lm - (double)n * n)) * rc0;
        }
        coef[e * 3 + 0] = ca;
        coef[e * 3 + 1] = cb;
        coef[e * 3 + 2] = cc;
    }
    if (threadIdx.x < 96) {  // warp q: the start value's factorial part for n = ns[q]
        const double lf = wigner_logfac(m, ns[threadIdx.x >> 5]);
        if ((threadIdx.x & 31) == 0) s_lf[threadIdx.x >> 5] = lf;
    }
    __syncthreads();
    const int lmax = L - 1;
    const double sgn = (m & 1) ? -1.0 : 1.0;
    for (int iu = threadIdx.x; iu < count; iu += blockDim.x) {
        const double x = sign_mu * mus[iu];
        // three independent recurrences advanced together
        double prev[3], cur[3];
        int lmin[3];
        for (int q = 0; q < 3; ++q) {
            lmin[q] = max(m, abs(ns[q]));
            prev[q] = 0.0;
            cur[q] = (lmin[q] <= lmax) ? wigner_start(m, ns[q], x, s_lf[q]) : 0.0;
        }
        for (int l = 0; l <= lmax; ++l) {
            double dv[3];
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                if (l < lmin[q]) {
                    dv[q] = 0.0;
                } else if (l == lmin[q]) {
                    dv[q] = cur[q];
                } else {
                    double next;
                    if (l == 1) {
                        next = x;
                    } else {
                        const double* c = coef + (l * 3 + q) * 3;
                        next = fma(fma(c[0], x, c[1]), cur[q], -c[2] * prev[q]);
                    }
                    prev[q] = cur[q];
                    cur[q] = next;
                    dv[q] = next;
                }
            }
            const size_t base = ((size_t)m * L + l) * 3;
            out[(base + 0) * ld + iu] = sgn * dv[0];
            out[(base + 1) * ld + iu] = 0.5 * sgn * (dv[1] + dv[2]);
            out[(base + 2) * ld + iu] = -0.5 * sgn * (dv[1] - dv[2]);
        }
    }
}

// A^m(+mu_i, +mu_j) and A^m(+mu_i, -mu_j) of medium s (kernel.cpp:45-63: the
// "phase-matrix Fourier coefficients Z^m" pp / pm blocks), accumulated over l
// in registers with the 2+2 sparsity of Pi B Pi.
__device__ __forceinline__ void kernel_blocks(const ProblemDev& p, const double* __restrict__ gsf, int s, int m,
                                              int i, int j, double app[4][4], double apm[4][4]) {
    const int N = p.N, L = p.Lc;
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) app[r][c] = apm[r][c] = 0.0;
    const double* gm = gsf + (size_t)m * L * 3 * N;
    const double* gk = p.greek + (size_t)s * L * 6;
    for (int l = m; l < L; ++l) {
        const double* gl = gm + (size_t)l * 3 * N;
        const double Pi = gl[i], Ri = gl[N + i], Ti = gl[2 * N + i];
        const double Pj = gl[j], Rj = gl[N + j], Tj = gl[2 * N + j];
        const double be = gk[6 * l + 0], al = gk[6 * l + 1], ga = gk[6 * l + 2];
        const double de = gk[6 * l + 3], ep = gk[6 * l + 4], ze = gk[6 * l + 5];
        // X = Pi_i B_l
        const double x00 = Pi * be, x01 = Pi * ga;
        const double x10 = Ri * ga, x11 = Ri * al, x12 = -Ti * ze, x13 = Ti * ep;
        const double x20 = -Ti * ga, x21 = -Ti * al, x22 = Ri * ze, x23 = -Ri * ep;
        const double x32 = Pi * ep, x33 = Pi * de;
        const double sl = ((l - m) & 1) ? -1.0 : 1.0;
        // A(+,+) += X Pi_j ; A(+,-) += s_l X (D Pi_j D)  (T_j -> -T_j)
        app[0][0] += x00 * Pj;
        app[0][1] += x01 * Rj;
        app[0][2] += -x01 * Tj;
        app[1][0] += x10 * Pj;
        app[1][1] += x11 * Rj - x12 * Tj;
        app[1][2] += -x11 * Tj + x12 * Rj;
        app[1][3] += x13 * Pj;
        app[2][0] += x20 * Pj;
        app[2][1] += x21 * Rj - x22 * Tj;
        app[2][2] += -x21 * Tj + x22 * Rj;
        app[2][3] += x23 * Pj;
        app[3][1] += -x32 * Tj;
        app[3][2] += x32 * Rj;
        app[3][3] += x33 * Pj;

        apm[0][0] += sl * (x00 * Pj);
        apm[0][1] += sl * (x01 * Rj);
        apm[0][2] += sl * (x01 * Tj);
        apm[1][0] += sl * (x10 * Pj);
        apm[1][1] += sl * (x11 * Rj + x12 * Tj);
        apm[1][2] += sl * (x11 * Tj + x12 * Rj);
        apm[1][3] += sl * (x13 * Pj);
        apm[2][0] += sl * (x20 * Pj);
        apm[2][1] += sl * (x21 * Rj + x22 * Tj);
        apm[2][2] += sl * (x21 * Tj + x22 * Rj);
        apm[2][3] += sl * (x23 * Pj);
        apm[3][1] += sl * (x32 * Tj);
        apm[3][2] += sl * (x32 * Rj);
        apm[3][3] += sl * (x33 * Pj);
    }
}

// E, F of every (medium s, order m) -- homogeneous.cpp:43-73 with A(+,+) and
// A(+,-) (kernel.cpp:45-63) accumulated per node pair (i, j) in registers.
// One thread per (s, m, i, j).
__global__ void build_ef_kernel(const ProblemDev p, const double* __restrict__ gsf,
                                double* __restrict__ E, double* __restrict__ F) {
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const int N = p.N, d = 4 * N;
    const long long total = (long long)p.n_media * p.n_orders * N * N;
    if (idx >= total) return;
    const int i = (int)(idx % N);
    const int j = (int)((idx / N) % N);
    const int om = (int)(idx / ((long long)N * N));  // s * n_orders + mo
    const int s = om / p.n_orders, m = p.order_of(om % p.n_orders);
    double app[4][4], apm[4][4];
    kernel_blocks(p, gsf, s, m, i, j, app, apm);
    const double half_omega = 0.5 * p.omega[s];
    const double sc = half_omega * p.weights[j];
    const double inv_mu = 1.0 / p.nodes[j];
    const double dsign[4] = {1.0, 1.0, -1.0, -1.0};
    double* Eo = E + (size_t)om * d * d;
    double* Fo = F + (size_t)om * d * d;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const size_t col = (size_t)(4 * j + c) * d;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const double k1 = sc * app[r][c];
            const double k2 = sc * apm[r][c] * dsign[c];
            const double id = (i == j && r == c) ? 1.0 : 0.0;
            Eo[col + 4 * i + r] = (id - k1 - k2) * inv_mu;
            Fo[col + 4 * i + r] = (id - k1 + k2) * inv_mu;
        }
    }
}

// Beam source per (s, m, incident ii, node i): the 4x4 blocks A^m(+-mu_i, -mu0)
// (kernel.cpp:89-109), scaled by omega/2pi (particular.cpp:17-24).  Column c of
// the block is the source for the unit Stokes vector e_c (D_k e_c = e_c for the
// k that owns channel c), so all four channels come out of one pass.
// Writes S+ = X+ + Delta X-, S- = X+ - Delta X- as [om][col = ii*4 + c][row].
__global__ void beam_source_kernel(const ProblemDev p, const double* __restrict__ gsf_nodes,
                                   const double* __restrict__ gsf_beam, double* __restrict__ sp,
                                   double* __restrict__ sm) {
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const int N = p.N, L = p.Lc, d = 4 * N, nin = p.n_in, R = 4 * nin;
    const long long total = (long long)p.n_media * p.n_orders * nin * N;
    if (idx >= total) return;
    const int i = (int)(idx % N);
    const int ii = (int)((idx / N) % nin);
    const int om = (int)(idx / ((long long)N * nin));
    const int s = om / p.n_orders, m = p.order_of(om % p.n_orders);
    double up[4][4], dn[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) up[r][c] = dn[r][c] = 0.0;
    const double* gk = p.greek + (size_t)s * L * 6;
    for (int l = m; l < L; ++l) {
        const double* gl = gsf_nodes + ((size_t)m * L + l) * 3 * N;
        const double* gb = gsf_beam + ((size_t)m * L + l) * 3 * nin;
        const double Pi = gl[i], Ri = gl[N + i], Ti = gl[2 * N + i];
        const double Pb = gb[ii], Rb = gb[nin + ii], Tb = gb[2 * nin + ii];
        const double be = gk[6 * l + 0], al = gk[6 * l + 1], ga = gk[6 * l + 2];
        const double de = gk[6 * l + 3], ep = gk[6 * l + 4], ze = gk[6 * l + 5];
        // Y = B_l Pi(mu_beam)
        double Y[4][4];
        Y[0][0] = be * Pb; Y[0][1] = ga * Rb; Y[0][2] = -ga * Tb; Y[0][3] = 0.0;
        Y[1][0] = ga * Pb; Y[1][1] = al * Rb; Y[1][2] = -al * Tb; Y[1][3] = 0.0;
        Y[2][0] = 0.0;     Y[2][1] = -ze * Tb; Y[2][2] = ze * Rb; Y[2][3] = -ep * Pb;
        Y[3][0] = 0.0;     Y[3][1] = -ep * Tb; Y[3][2] = ep * Rb; Y[3][3] = de * Pb;
        const double sl = ((l - m) & 1) ? -1.0 : 1.0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            up[0][c] += Pi * Y[0][c];
            up[1][c] += Ri * Y[1][c] - Ti * Y[2][c];
            up[2][c] += -Ti * Y[1][c] + Ri * Y[2][c];
            up[3][c] += Pi * Y[3][c];
            dn[0][c] += sl * (Pi * Y[0][c]);
            dn[1][c] += sl * (Ri * Y[1][c] + Ti * Y[2][c]);
            dn[2][c] += sl * (Ti * Y[1][c] + Ri * Y[2][c]);
            dn[3][c] += sl * (Pi * Y[3][c]);
        }
    }
    const double sc = p.omega[s] / (2.0 * kPi);
    const double dsign[4] = {1.0, 1.0, -1.0, -1.0};
    double* SP = sp + (size_t)om * d * R;
    double* SM = sm + (size_t)om * d * R;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const size_t col = (size_t)(ii * 4 + c) * d;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const double xp = sc * up[r][c], xm = sc * dn[r][c];
            SP[col + 4 * i + r] = xp + dsign[r] * xm;
            SM[col + 4 * i + r] = xp - dsign[r] * xm;
        }
    }
}

}  // namespace

void launch_gsf(const ProblemDev& p, const double* mus, int count, double sign, double* out,
                cudaStream_t st) {
    const size_t smem = (size_t)9 * p.Lc * sizeof(double);
    if (smem > 48 * 1024) {
        static unsigned long long attr = 0;
        smem_attr_once(gsf_kernel, 200 * 1024, attr);
    }
    gsf_kernel<<<p.L, 128, smem, st>>>(p.L, p.Lc, count, mus, sign, out, count);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

// Debug dump (kernel.cpp:188-214): the pp / pm blocks of medium s for the
// plan's orders, out [mo][i][j][2][16] row-major.  Thread per (mo, i, j).
__global__ void kernel_dump_kernel(const ProblemDev p, const double* __restrict__ gsf, int s, double* out) {
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const int N = p.N;
    if (idx >= (long long)p.n_orders * N * N) return;
    const int j = (int)(idx % N), i = (int)((idx / N) % N), mo = (int)(idx / ((long long)N * N));
    double app[4][4], apm[4][4];
    kernel_blocks(p, gsf, s, p.order_of(mo), i, j, app, apm);
    double* o = out + idx * 32;
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) {
            o[4 * r + c] = app[r][c];
            o[16 + 4 * r + c] = apm[r][c];
        }
}

void launch_kernel_dump(const ProblemDev& p, const double* gsf, int s, double* out, cudaStream_t st) {
    const long long total = (long long)p.n_orders * p.N * p.N;
    kernel_dump_kernel<<<(unsigned)((total + 127) / 128), 128, 0, st>>>(p, gsf, s, out);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

void launch_build_ef(const ProblemDev& p, const double* gsf, double* E, double* F,
                     cudaStream_t st) {
    const long long total = (long long)p.n_media * p.n_orders * p.N * p.N;
    build_ef_kernel<<<(unsigned)((total + 127) / 128), 128, 0, st>>>(p, gsf, E, F);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

void launch_beam_source(const ProblemDev& p, const double* gsf_nodes, const double* gsf_beam,
                        double* sp, double* sm, cudaStream_t st) {
    const long long total = (long long)p.n_media * p.n_orders * p.n_in * p.N;
    beam_source_kernel<<<(unsigned)((total + 127) / 128), 128, 0, st>>>(p, gsf_nodes, gsf_beam,
                                                                         sp, sm);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace vrte
