// eig.cu -- batched nonsymmetric fp64 eigensolver for the half-size
// homogeneous problem (F E) x = x / nu^2 of every (medium, order), and the
// mode recovery / residual machinery of homogeneous.cpp:131-287.
//
// Reference uses Eigen::EigenSolver (real Schur + eigenvectors).  Here:
//   hessenberg.cu        : blocked Householder reduction (dlahr2 panels + DMMA
//                          trailing updates), Q formed into Z
//   hqr_multi_kernel     : small-bulge multishift Francis QR with aggressive
//                          early deflation (dlaqr0/3/5 organisation) on a 2-CTA
//                          cluster per matrix: rank 0 chases up to 4 bulges in a
//                          32 x 32 shared-memory window and runs the AED window
//                          Schur, rank 1 applies each chunk's orthogonal factor to
//                          the rest of H and to Z on the FP64 tensor cores;
//                          dlahqr rules (Ahues-Kressner deflation, exceptional
//                          shifts, dlanv2 standardization) for small blocks
//   trevc_blk_kernel     : eigenvectors of the quasi-triangular Schur factor by
//                          blocked back substitution (dtrevc3 organisation: shifted
//                          32-row diagonal blocks per eigenvector, shift-free
//                          block updates for all at once), back-transformed by a GEMM
#include <climits>
#include <cstdlib>
#include <string>
#include <vector>

#include "kernels.cuh"

namespace vrte {
namespace {

constexpr int NT = 256;

__device__ int block_max_int(int v, int* s) {
    __syncthreads();
    if (threadIdx.x == 0) *s = INT_MIN;
    __syncthreads();
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) atomicMax(s, v);
    __syncthreads();
    return *s;
}

__global__ void max_abs_kernel(const double* A, long long per, double* out) {
    __shared__ double red[32];
    const double* a = A + blockIdx.x * per;
    double m = 0.0;
    for (long long e = threadIdx.x; e < per; e += blockDim.x) m = fmax(m, fabs(a[e]));
    m = block_max(m, red);
    if (threadIdx.x == 0) out[blockIdx.x] = m;
}

// ------------------------------------------------------------------ Hessenberg
// dgehd2-style unblocked Householder reduction A <- Q^T A Q, Z <- Q.
__global__ void __launch_bounds__(NT) hessenberg_kernel(double* Aall, double* Zall, int d) {
    extern __shared__ double sm[];
    double* v = sm;
    __shared__ double red[32];
    double* A = Aall + (size_t)blockIdx.x * d * d;
    double* Z = Zall + (size_t)blockIdx.x * d * d;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5, nw = blockDim.x >> 5;
    for (size_t e = t; e < (size_t)d * d; e += blockDim.x) Z[e] = (e % d == e / d) ? 1.0 : 0.0;
    for (int k = 0; k + 2 < d; ++k) {
        const int n = d - k - 1;
        double ss = 0.0;
        for (int r = t; r < n; r += blockDim.x) {
            const double x = A[(size_t)(k + 1 + r) + (size_t)k * d];
            v[r] = x;
            if (r > 0) ss += x * x;
        }
        ss = block_sum(ss, red);
        const double alpha = v[0];
        const double xnorm = sqrt(ss);
        if (xnorm == 0.0) continue;
        const double beta = -copysign(hypot(alpha, xnorm), alpha);
        const double tau = (beta - alpha) / beta;
        const double scal = 1.0 / (alpha - beta);
        __syncthreads();
        for (int r = t; r < n; r += blockDim.x) {
            v[r] = (r == 0) ? 1.0 : v[r] * scal;
            A[(size_t)(k + 1 + r) + (size_t)k * d] = (r == 0) ? beta : 0.0;
        }
        __syncthreads();
        // right: A[:, k+1:] -= tau (A v) v^T ; Z likewise (thread per row)
        for (int i = t; i < d; i += blockDim.x) {
            double y = 0.0, yz = 0.0;
            const double* ac = A + i + (size_t)(k + 1) * d;
            const double* zc = Z + i + (size_t)(k + 1) * d;
            for (int j = 0; j < n; ++j) {
                const double vj = v[j];
                y = fma(ac[(size_t)j * d], vj, y);
                yz = fma(zc[(size_t)j * d], vj, yz);
            }
            y *= tau;
            yz *= tau;
            double* aw = A + i + (size_t)(k + 1) * d;
            double* zw = Z + i + (size_t)(k + 1) * d;
            for (int j = 0; j < n; ++j) {
                const double vj = v[j];
                aw[(size_t)j * d] -= y * vj;
                zw[(size_t)j * d] -= yz * vj;
            }
        }
        __syncthreads();
        // left: A[k+1:, k+1:] -= tau v (v^T A)  (warp per column)
        for (int c = k + 1 + w; c < d; c += nw) {
            double* col = A + (size_t)c * d + k + 1;
            double p = 0.0;
            for (int r = lane; r < n; r += 32) p = fma(v[r], col[r], p);
            p = warp_sum(p) * tau;
            for (int r = lane; r < n; r += 32) col[r] -= p * v[r];
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ Francis QR


// dlanv2: Schur factorization of a real 2x2 nonsymmetric matrix in standard form.
__device__ void dlanv2(double& a, double& b, double& c, double& dd, double& rt1r, double& rt1i,
                       double& rt2r, double& rt2i, double& cs, double& sn) {
    const double eps = kUlp;
    const double safmn2 = 0x1p-485, safmx2 = 0x1p485;
    const double multpl = 4.0;
    if (c == 0.0) {
        cs = 1.0;
        sn = 0.0;
    } else if (b == 0.0) {
        cs = 0.0;
        sn = 1.0;
        const double temp = dd;
        dd = a;
        a = temp;
        b = -c;
        c = 0.0;
    } else if ((a - dd) == 0.0 && copysign(1.0, b) != copysign(1.0, c)) {
        cs = 1.0;
        sn = 0.0;
    } else {
        double temp = a - dd;
        double p = 0.5 * temp;
        const double bcmax = fmax(fabs(b), fabs(c));
        const double bcmis = fmin(fabs(b), fabs(c)) * copysign(1.0, b) * copysign(1.0, c);
        double scale = fmax(fabs(p), bcmax);
        double z = (p / scale) * p + (bcmax / scale) * bcmis;
        if (z >= multpl * eps) {
            z = p + copysign(sqrt(scale) * sqrt(z), p);
            a = dd + z;
            dd = dd - (bcmax / z) * bcmis;
            const double tau = hypot(c, z);
            cs = z / tau;
            sn = c / tau;
            b = b - c;
            c = 0.0;
        } else {
            int count = 0;
            double sigma = b + c;
            while (true) {
                ++count;
                scale = fmax(fabs(temp), fabs(sigma));
                if (scale >= safmx2) {
                    sigma *= safmn2;
                    temp *= safmn2;
                    if (count <= 20) continue;
                }
                if (scale <= safmn2) {
                    sigma *= safmx2;
                    temp *= safmx2;
                    if (count <= 20) continue;
                }
                break;
            }
            p = 0.5 * temp;
            double tau = hypot(sigma, temp);
            cs = sqrt(0.5 * (1.0 + fabs(sigma) / tau));
            sn = -(p / (tau * cs)) * copysign(1.0, sigma);
            const double aa = a * cs + b * sn, bb = -a * sn + b * cs;
            const double cc = c * cs + dd * sn, ddd = -c * sn + dd * cs;
            a = aa * cs + cc * sn;
            b = bb * cs + ddd * sn;
            c = -aa * sn + cc * cs;
            dd = -bb * sn + ddd * cs;
            temp = 0.5 * (a + dd);
            a = temp;
            dd = temp;
            if (c != 0.0) {
                if (b != 0.0) {
                    if (copysign(1.0, b) == copysign(1.0, c)) {
                        const double sab = sqrt(fabs(b)), sac = sqrt(fabs(c));
                        p = copysign(sab * sac, c);
                        tau = 1.0 / sqrt(fabs(b + c));
                        a = temp + p;
                        dd = temp - p;
                        b = b - c;
                        c = 0.0;
                        const double cs1 = sab * tau, sn1 = sac * tau;
                        temp = cs * cs1 - sn * sn1;
                        sn = cs * sn1 + sn * cs1;
                        cs = temp;
                    }
                } else {
                    b = -c;
                    c = 0.0;
                    temp = cs;
                    cs = -sn;
                    sn = temp;
                }
            }
        }
    }
    rt1r = a;
    rt2r = dd;
    if (c == 0.0) {
        rt1i = 0.0;
        rt2i = 0.0;
    } else {
        rt1i = sqrt(fabs(b)) * sqrt(fabs(c));
        rt2i = -rt1i;
    }
}




// ------------------------------------------------------------------ Francis QR helpers


// dlarfg for a 2/3-element bulge column: one rsqrt and one reciprocal.  As in
// LAPACK the reflector is the identity only when v2 = v3 = 0 exactly; when
// their squares underflow against v1 it is the tau = 2 sign flip (dlarfg's
// result) -- treating it as the identity stalls the chase on graded matrices
// whose converging subdiagonals reach ~1e-180.  Columns whose entries could
// under/overflow in the squares are rescaled by a power of two.  Returns
// tau; v2, v3 become the reflector tail, beta the new head.
__device__ inline double house3(double v1, double& v2, double& v3, double& beta) {
    beta = v1;
    if (v2 == 0.0 && v3 == 0.0) return 0.0;
    double x2 = fma(v2, v2, v3 * v3);
    double ss = fma(v1, v1, x2);
    double sc = 1.0;
    if (!(ss > 0x1p-900 && ss < 0x1p900)) {  // rare: the whole column under/overflows
        const int e = ilogb(fmax(fabs(v1), fmax(fabs(v2), fabs(v3))));
        sc = scalbn(1.0, e);
        const double inv = scalbn(1.0, -e);
        v1 *= inv;
        v2 *= inv;
        v3 *= inv;
        x2 = fma(v2, v2, v3 * v3);
        ss = fma(v1, v1, x2);
    }
    const double rq = rsqrt(ss);
    const double nv = ss * rq;
    const double av1 = fabs(v1);
    const double r = copysign(__drcp_rn(av1 + nv), v1);
    v2 *= r;
    v3 *= r;
    beta = -copysign(nv, v1) * sc;
    return fma(av1, rq, 1.0);
}

__device__ inline double hg(const double* H, int d, int r, int c) { return H[r + (size_t)c * d]; }

__device__ bool small_subdiag_g(const double* H, int d, int k, double ulp, double smlnum) {
    const double hk = fabs(hg(H, d, k, k - 1));
    if (hk <= smlnum) return true;
    double tst = fabs(hg(H, d, k - 1, k - 1)) + fabs(hg(H, d, k, k));
    if (tst == 0.0) {
        if (k - 2 >= 0) tst += fabs(hg(H, d, k - 1, k - 2));
        if (k + 1 <= d - 1) tst += fabs(hg(H, d, k + 1, k));
    }
    if (hk <= ulp * tst) {
        const double hup = fabs(hg(H, d, k - 1, k));
        const double ab = fmax(hk, hup), ba = fmin(hk, hup);
        const double dif = fabs(hg(H, d, k - 1, k - 1) - hg(H, d, k, k));
        const double aa = fmax(fabs(hg(H, d, k, k)), dif), bb = fmin(fabs(hg(H, d, k, k)), dif);
        const double rs = 1.0 / (aa + ab);
        if (ba * (ab * rs) <= fmax(smlnum, ulp * (bb * (aa * rs)))) return true;
    }
    return false;
}

__device__ void start_vector_g(const double* H, int d, int m, double rt1r, double rt1i, double rt2r,
                               double rt2i, double v[3]) {
    // (dlaqr1; scalings by reciprocals -- one FP64 division on the chain instead of
    // four: the reflector house3 builds from v does not depend on v's scale)
    double h21s = hg(H, d, m + 1, m);
    const double s = fabs(hg(H, d, m, m) - rt2r) + fabs(rt2i) + fabs(h21s);
    const double rs = 1.0 / s;
    h21s = hg(H, d, m + 1, m) * rs;
    v[0] = h21s * hg(H, d, m, m + 1) + (hg(H, d, m, m) - rt1r) * ((hg(H, d, m, m) - rt2r) * rs) -
           rt1i * (rt2i * rs);
    v[1] = h21s * (hg(H, d, m, m) + hg(H, d, m + 1, m + 1) - rt1r - rt2r);
    v[2] = h21s * hg(H, d, m + 2, m + 1);
}



// ------------------------------------------------------------------ multi-bulge Francis QR
// Small-bulge multishift QR (the dlaqr5 organisation, without aggressive early
// deflation): while the active block [L, I] is large, one sweep chases a chain
// of nb double-shift bulges (2 nb shifts = eigenvalues of the trailing
// 2nb x 2nb block, computed by a warp-level eigenvalue-only QR), spaced three
// rows apart, in lock step: warp b owns bulge b.  Within a step every bulge
// first computes its reflector from the state at the start of the step and
// applies it from the left (disjoint rows), then -- after a named barrier --
// from the right and to the chunk factor U (disjoint columns); left and right
// reflections of different bulges commute, so this equals LAPACK's
// bottom-to-top bulge order.  Chunks of MS steps are chased in a MW x MW
// shared-memory window; U is applied to the rest of H and to Z by the whole
// CTA.  Small active blocks and exceptional-shift sweeps use one bulge with
// the dlahqr shift / start rules.
constexpr int MB_MAX = 4;   // bulges per sweep
constexpr int MS = 19;      // chase steps per chunk with MB_MAX bulges (MW - 3 (nb - 1) - 4 for nb)
constexpr int MW = 32;      // window (>= MS + 3 (MB_MAX - 1) + 4)
constexpr int LDW = MW + 1; // leading dimension of the window: row sweeps (lanes over
                            // columns) hit distinct shared-memory banks
constexpr int TQ = 8;       // tiny-matrix leading dimension (2 MB_MAX)
constexpr int AED_NW = 14;  // deflation window (<= MW); measured optimum for d = 256

__device__ inline void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Eigenvalues of the n x n Hessenberg S (ld TQ, zero padded) by one warp:
// double-shift QR without vectors (dlahqr, wantt = wantz = false).  Scalar
// control is computed redundantly by every lane; row/column operations are
// lane-parallel.
__device__ void warp_tiny_eig(double* S, int n, double* sr, double* si) {
    const int lane = threadIdx.x & 31;
    const double ulp = kUlp, smlnum = kSafeMin * ((double)n * (1.0 / kUlp));  // 1/ulp = 2^52: exact
    auto A = [&](int r, int c) -> double& { return S[r + c * TQ]; };
    int I = n - 1;
    int kdefl = 0;
    while (I >= 0) {
        int L = 0;
        bool conv = false;
        for (int its = 0; its <= 40 * n; ++its) {
            int kb = L;
            for (int k = I; k > L; --k)
                if (small_subdiag_g(S, TQ, k, ulp, smlnum)) {
                    kb = k;
                    break;
                }
            L = kb;
            __syncwarp();
            if (L > 0 && lane == 0) A(L, L - 1) = 0.0;
            __syncwarp();
            if (L >= I - 1) {
                conv = true;
                break;
            }
            ++kdefl;
            double h11, h12, h21, h22;
            if (kdefl % 20 == 0) {
                const double s = fabs(A(I, I - 1)) + fabs(A(I - 1, I - 2 >= 0 ? I - 2 : 0));
                h11 = 0.75 * s + A(I, I);
                h12 = -0.4375 * s;
                h21 = s;
                h22 = h11;
            } else if (kdefl % 10 == 0) {
                const double s = fabs(A(L + 1, L)) + fabs(A(L + 2, L + 1));
                h11 = 0.75 * s + A(L, L);
                h12 = -0.4375 * s;
                h21 = s;
                h22 = h11;
            } else {
                h11 = A(I - 1, I - 1);
                h21 = A(I, I - 1);
                h12 = A(I - 1, I);
                h22 = A(I, I);
            }
            double rt1r, rt1i, rt2r, rt2i;
            {
                const double s = fabs(h11) + fabs(h12) + fabs(h21) + fabs(h22);
                if (s == 0.0) {
                    rt1r = rt1i = rt2r = rt2i = 0.0;
                } else {
                    const double rs = 1.0 / s;
                    h11 *= rs;
                    h21 *= rs;
                    h12 *= rs;
                    h22 *= rs;
                    const double tr = (h11 + h22) / 2.0;
                    const double det = (h11 - tr) * (h22 - tr) - h12 * h21;
                    const double rtdisc = sqrt(fabs(det));
                    if (det >= 0.0) {
                        rt1r = tr * s;
                        rt2r = rt1r;
                        rt1i = rtdisc * s;
                        rt2i = -rt1i;
                    } else {
                        rt1r = tr + rtdisc;
                        rt2r = tr - rtdisc;
                        if (fabs(rt1r - h22) <= fabs(rt2r - h22)) {
                            rt1r *= s;
                            rt2r = rt1r;
                        } else {
                            rt2r *= s;
                            rt1r = rt2r;
                        }
                        rt1i = rt2i = 0.0;
                    }
                }
            }
            const int M = L;
            for (int k = M; k <= I - 1; ++k) {
                const int nr = min(3, I - k + 1);
                double v1, v2, v3;
                if (k == M) {
                    double v[3];
                    start_vector_g(S, TQ, M, rt1r, rt1i, rt2r, rt2i, v);
                    v1 = v[0];
                    v2 = v[1];
                    v3 = nr == 3 ? v[2] : 0.0;
                } else {
                    v1 = A(k, k - 1);
                    v2 = A(k + 1, k - 1);
                    v3 = nr == 3 ? A(k + 2, k - 1) : 0.0;
                }
                double bt;
                const double t1 = house3(v1, v2, v3, bt);
                v1 = bt;
                const double t2 = t1 * v2, t3 = t1 * v3;
                if (k == M) __syncwarp();  // the start vector read columns M, M+1 (k > M: column k-1 only)
                const int c = k + lane;
                if (c <= I) {
                    const double a0 = A(k, c), a1 = A(k + 1, c), a2 = nr == 3 ? A(k + 2, c) : 0.0;
                    const double sum = a0 + v2 * a1 + v3 * a2;
                    A(k, c) = a0 - sum * t1;
                    A(k + 1, c) = a1 - sum * t2;
                    if (nr == 3) A(k + 2, c) = a2 - sum * t3;
                }
                __syncwarp();
                if (k > M && lane == 0) {
                    A(k, k - 1) = v1;
                    A(k + 1, k - 1) = 0.0;
                    if (k < I - 1) A(k + 2, k - 1) = 0.0;
                }
                const int r = L + lane;
                if (r <= min(k + 3, I)) {
                    const double a0 = A(r, k), a1 = A(r, k + 1), a2 = nr == 3 ? A(r, k + 2) : 0.0;
                    const double sum = a0 + v2 * a1 + v3 * a2;
                    A(r, k) = a0 - sum * t1;
                    A(r, k + 1) = a1 - sum * t2;
                    if (nr == 3) A(r, k + 2) = a2 - sum * t3;
                }
                __syncwarp();
            }
        }
        if (!conv) {  // give up gracefully: diagonal entries as shifts
            for (int q = 0; q <= I; ++q) {
                sr[q] = A(q, q);
                si[q] = 0.0;
            }
            return;
        }
        if (L == I) {
            sr[I] = A(I, I);
            si[I] = 0.0;
        } else {
            double a = A(I - 1, I - 1), bb = A(I - 1, I), c = A(I, I - 1), dd = A(I, I);
            double r1r, r1i, r2r, r2i, cs, sn;
            dlanv2(a, bb, c, dd, r1r, r1i, r2r, r2i, cs, sn);
            sr[I - 1] = r1r;
            si[I - 1] = r1i;
            sr[I] = r2r;
            si[I] = r2i;
        }
        kdefl = 0;
        I = L - 1;
        __syncwarp();
    }
}


// Real Schur form T = V S V^T of the n x n Hessenberg T (ld MW, n <= MW) by one
// warp: double-shift QR with full updates (dlahqr, wantt = wantz = true); V
// (ld MW) accumulates the transformations (callers pass V = I).  sr/si receive
// the eigenvalues by diagonal position.  Returns false if it did not converge.
__device__ bool warp_small_schur(double* T, double* V, int n, double* sr, double* si) {
    const int lane = threadIdx.x & 31;
    const double ulp = kUlp, smlnum = kSafeMin * ((double)n * (1.0 / kUlp));  // 1/ulp = 2^52: exact
    auto A = [&](int r, int c) -> double& { return T[r + c * LDW]; };
    int I = n - 1;
    int kdefl = 0;
    while (I >= 0) {
        int L = 0;
        bool conv = false;
        for (int its = 0; its <= 30 * max(10, n); ++its) {
            // largest k in (L, I] with a negligible subdiagonal: lanes test in parallel
            const int kk = L + 1 + lane;
            const bool hit = kk <= I && small_subdiag_g(T, LDW, kk, ulp, smlnum);
            const unsigned m = __ballot_sync(0xffffffffu, hit);
            if (m) L = L + 1 + (31 - __clz(m));
            __syncwarp();
            if (L > 0 && lane == 0) A(L, L - 1) = 0.0;
            __syncwarp();
            if (L >= I - 1) {
                conv = true;
                break;
            }
            ++kdefl;
            double h11, h12, h21, h22;
            if (kdefl % 20 == 0) {
                const double s = fabs(A(I, I - 1)) + fabs(A(I - 1, I >= 2 ? I - 2 : 0));
                h11 = 0.75 * s + A(I, I);
                h12 = -0.4375 * s;
                h21 = s;
                h22 = h11;
            } else if (kdefl % 10 == 0) {
                const double s = fabs(A(L + 1, L)) + fabs(A(L + 2, L + 1));
                h11 = 0.75 * s + A(L, L);
                h12 = -0.4375 * s;
                h21 = s;
                h22 = h11;
            } else {
                h11 = A(I - 1, I - 1);
                h21 = A(I, I - 1);
                h12 = A(I - 1, I);
                h22 = A(I, I);
            }
            double rt1r, rt1i, rt2r, rt2i;
            {
                const double s = fabs(h11) + fabs(h12) + fabs(h21) + fabs(h22);
                if (s == 0.0) {
                    rt1r = rt1i = rt2r = rt2i = 0.0;
                } else {
                    const double rs = 1.0 / s;
                    h11 *= rs;
                    h21 *= rs;
                    h12 *= rs;
                    h22 *= rs;
                    const double tr = (h11 + h22) / 2.0;
                    const double det = (h11 - tr) * (h22 - tr) - h12 * h21;
                    const double rtdisc = sqrt(fabs(det));
                    if (det >= 0.0) {
                        rt1r = tr * s;
                        rt2r = rt1r;
                        rt1i = rtdisc * s;
                        rt2i = -rt1i;
                    } else {
                        rt1r = tr + rtdisc;
                        rt2r = tr - rtdisc;
                        if (fabs(rt1r - h22) <= fabs(rt2r - h22)) {
                            rt1r *= s;
                            rt2r = rt1r;
                        } else {
                            rt2r *= s;
                            rt1r = rt2r;
                        }
                        rt1i = rt2i = 0.0;
                    }
                }
            }
            const int M = L;
            for (int k = M; k <= I - 1; ++k) {
                const int nr = min(3, I - k + 1);
                double v1, v2, v3;
                if (k == M) {
                    double v[3];
                    start_vector_g(T, LDW, M, rt1r, rt1i, rt2r, rt2i, v);
                    v1 = v[0];
                    v2 = v[1];
                    v3 = nr == 3 ? v[2] : 0.0;
                } else {
                    v1 = A(k, k - 1);
                    v2 = A(k + 1, k - 1);
                    v3 = nr == 3 ? A(k + 2, k - 1) : 0.0;
                }
                double bt;
                const double t1 = house3(v1, v2, v3, bt);
                v1 = bt;
                const double t2 = t1 * v2, t3 = t1 * v3;
                if (k == M) __syncwarp();  // the start vector read columns M, M+1 (k > M: column k-1 only)
                const int c = k + lane;
                if (c < n) {
                    const double a0 = A(k, c), a1 = A(k + 1, c), a2 = nr == 3 ? A(k + 2, c) : 0.0;
                    const double sum = a0 + v2 * a1 + v3 * a2;
                    A(k, c) = a0 - sum * t1;
                    A(k + 1, c) = a1 - sum * t2;
                    if (nr == 3) A(k + 2, c) = a2 - sum * t3;
                }
                __syncwarp();
                if (k > M && lane == 0) {
                    A(k, k - 1) = v1;
                    A(k + 1, k - 1) = 0.0;
                    if (k < I - 1) A(k + 2, k - 1) = 0.0;
                }
                const int r = lane;
                if (r <= min(k + 3, I)) {
                    const double a0 = A(r, k), a1 = A(r, k + 1), a2 = nr == 3 ? A(r, k + 2) : 0.0;
                    const double sum = a0 + v2 * a1 + v3 * a2;
                    A(r, k) = a0 - sum * t1;
                    A(r, k + 1) = a1 - sum * t2;
                    if (nr == 3) A(r, k + 2) = a2 - sum * t3;
                }
                if (r < n) {
                    double* vr = V + r;
                    const double a0 = vr[k * LDW], a1 = vr[(k + 1) * LDW], a2 = nr == 3 ? vr[(k + 2) * LDW] : 0.0;
                    const double sum = a0 + v2 * a1 + v3 * a2;
                    vr[k * LDW] = a0 - sum * t1;
                    vr[(k + 1) * LDW] = a1 - sum * t2;
                    if (nr == 3) vr[(k + 2) * LDW] = a2 - sum * t3;
                }
                __syncwarp();
            }
        }
        if (!conv) return false;
        if (L == I) {
            sr[I] = A(I, I);
            si[I] = 0.0;
        } else {
            double a = A(I - 1, I - 1), bb = A(I - 1, I), c = A(I, I - 1), dd = A(I, I);
            double r1r, r1i, r2r, r2i, cs, sn;
            dlanv2(a, bb, c, dd, r1r, r1i, r2r, r2i, cs, sn);
            __syncwarp();
            if (lane == 0) {
                A(I - 1, I - 1) = a;
                A(I - 1, I) = bb;
                A(I, I - 1) = c;
                A(I, I) = dd;
            }
            sr[I - 1] = r1r;
            si[I - 1] = r1i;
            sr[I] = r2r;
            si[I] = r2i;
            const int j = I + 1 + lane;
            if (j < n) {
                const double xv = A(I - 1, j), yv = A(I, j);
                A(I - 1, j) = cs * xv + sn * yv;
                A(I, j) = cs * yv - sn * xv;
            }
            if (lane <= I - 2) {
                const double xv = A(lane, I - 1), yv = A(lane, I);
                A(lane, I - 1) = cs * xv + sn * yv;
                A(lane, I) = cs * yv - sn * xv;
            }
            if (lane < n) {
                double* vr = V + lane;
                const double xv = vr[(I - 1) * LDW], yv = vr[I * LDW];
                vr[(I - 1) * LDW] = cs * xv + sn * yv;
                vr[I * LDW] = cs * yv - sn * xv;
            }
            __syncwarp();
        }
        kdefl = 0;
        I = L - 1;
        __syncwarp();
    }
    return true;
}

// Householder reflector applied by one warp: x <- (I - tau v v^T) x on rows
// [r0, r0+len) of the columns [c0, c1) of A (ld MW) -- left -- or on columns
// [r0, r0+len) of the rows [c0, c1) -- right.  v[0] = 1 implicitly stored.
// (the dot products in four interleaved partial sums, unrolled by four: the
// loads are independent and the FMA chains a quarter as long)
__device__ inline double strided_dot(const double* v, const double* x, long long st, int len) {
    double w0 = 0.0, w1 = 0.0, w2 = 0.0, w3 = 0.0;
    int q = 0;
    for (; q + 3 < len; q += 4) {
        w0 = fma(v[q], x[q * st], w0);
        w1 = fma(v[q + 1], x[(q + 1) * st], w1);
        w2 = fma(v[q + 2], x[(q + 2) * st], w2);
        w3 = fma(v[q + 3], x[(q + 3) * st], w3);
    }
    for (; q < len; ++q) w0 = fma(v[q], x[q * st], w0);
    return (w0 + w1) + (w2 + w3);
}
__device__ void warp_refl_left(double* A, int ld, const double* v, int len, double tau, int r0, int c0,
                               int c1) {
    const int lane = threadIdx.x & 31;
    for (int c = c0 + lane; c < c1; c += 32) {
        double* x = A + r0 + c * ld;
        const double w = tau * strided_dot(v, x, 1, len);
#pragma unroll 4
        for (int q = 0; q < len; ++q) x[q] -= w * v[q];
    }
    __syncwarp();
}
__device__ void warp_refl_right(double* A, int ld, const double* v, int len, double tau, int r0, int c0,
                                int c1) {
    const int lane = threadIdx.x & 31;
    for (int r = c0 + lane; r < c1; r += 32) {
        double* x = A + r + r0 * ld;
        const double w = tau * strided_dot(v, x, ld, len);
#pragma unroll 4
        for (int q = 0; q < len; ++q) x[q * ld] -= w * v[q];
    }
    __syncwarp();
}
// dlarfg on (alpha, x[0..len-2]) in place in v[0..len-1]: on return v[0] = 1,
// v[1..] the reflector tail; returns tau, *beta the new alpha.  Lane-redundant.
__device__ double warp_dlarfg(double* v, int len, double* beta) {
    const int lane = threadIdx.x & 31;
    const double alpha = v[0];
    const double xn = len > 1 ? strided_dot(v + 1, v + 1, 1, len - 1) : 0.0;
    __syncwarp();
    if (xn == 0.0) {
        *beta = alpha;
        if (lane == 0) v[0] = 1.0;
        __syncwarp();
        return 0.0;
    }
    const double b = -copysign(sqrt(alpha * alpha + xn), alpha);
    const double tau = (b - alpha) / b, sc = 1.0 / (alpha - b);
    for (int q = 1 + lane; q < len; q += 32) v[q] *= sc;
    __syncwarp();
    if (lane == 0) v[0] = 1.0;
    __syncwarp();
    *beta = b;
    return tau;
}


// ---- thread-block-cluster helpers (the multishift QR runs as a 2-CTA cluster)
__device__ inline unsigned dsmem_addr(const void* p, unsigned rank) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(p));
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ inline unsigned ld_acquire_cluster(unsigned addr) {
    unsigned v;
    asm volatile("ld.acquire.cluster.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ inline void st_release_cluster(unsigned addr, unsigned v) {
    asm volatile("st.release.cluster.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ inline int ld_cluster_s32(unsigned addr) {
    int v;
    asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ inline double ld_cluster_f64(unsigned addr) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
    return v;
}
__device__ inline void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ inline void fence_cluster() { asm volatile("fence.acq_rel.cluster;" ::: "memory"); }

template <int MINB>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, MINB) hqr_multi_kernel(double* Hall, double* Zall, double* wrall,
                                                        double* wiall, int d, DeviceStatus* status,
                                                        int aed_nw, int nb4_min, int nb2_min, int nibble,
                                                        double* trace) {
    __shared__ double Wn[MW * LDW];  // window, column-major Wn[c*LDW + r]
    __shared__ double Us2[3 * MW * LDW];  // chunk factors (triple buffered), column-major [c*LDW + r]
    double* const Us = Us2;               // buffer 0: AED factor / first chunk
    __shared__ double Sm[TQ * TQ];  // trailing block for the shifts
    __shared__ double s_sr[TQ], s_si[TQ];
    __shared__ double s_pr[4 * MB_MAX];  // shift pair per bulge: rt1r rt1i rt2r rt2i
    __shared__ double s_esr[MW], s_esi[MW], s_vec[MW];
    __shared__ int s_aed[4];             // ok, ndefl, skip-sweep, bulges
    __shared__ int s_int;
    __shared__ int s_nb;
    __shared__ double s_t1;
    // cluster job queue (used in rank 0's shared memory): rank 0 posts chunk
    // factors, rank 1 applies them to the rest of H and to Z
    __shared__ unsigned s_posted, s_done;
    __shared__ int s_job[2][9];  // buf, wlo, whi, nw, c_lo, c_hi, above_z, stop, c_split
    __shared__ unsigned s_partial;
    const int b = blockIdx.x >> 1, crank = blockIdx.x & 1;
    const int t = threadIdx.x, nt = blockDim.x, lane = t & 31, warp = t >> 5;
    double* H = Hall + (size_t)b * d * d;
    double* Z = Zall + (size_t)b * d * d;
    double* wr = wrall + (size_t)b * d;
    double* wi = wiall + (size_t)b * d;
    const double ulp = kUlp;
    const double smlnum = kSafeMin * ((double)d / ulp);
    const int itmax = 30 * max(10, d);
    const int kexsh = 10;
    int kdefl = 0;
    int I = d - 1;
    unsigned long long nsweep = 0, nstep = 0;
    unsigned long long cyc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tc = clock64();
    auto tick = [&](int slot) {
        const long long now = clock64();
        cyc[slot] += (unsigned long long)(now - tc);
        tc = now;
    };
    // H(:, wlo:whi) <- H U above the window, H(wlo:whi, :) <- U^T H right of it,
    // Z(:, wlo:whi) <- Z U  (U = Us, nw x nw, identity beyond).  Every target is
    // a vector v (a column segment right of the window, or a row segment of H
    // above it / of Z) mapped to v^T U, so tiles of 8 vectors are one
    // [8 x 32] x [32 x 32] product on the FP64 tensor cores: warp per tile,
    // U's B fragments held in registers for the whole call (DMMA m8n8k4).
    // Apply the chunk factor U (nw x nw, identity beyond) to H columns [c_lo, c_hi)
    // right of the window (U^T x), and -- if above_z -- to the rows of H above the
    // window and to Z (x U).  Every target is a vector v mapped to v^T U, so
    // tiles of 8 vectors are one [8 x 32] x [32 x 32] product on the FP64 tensor
    // cores: warp per tile (gw-th of gsize warps), U's B fragments in registers.
    auto apply_part = [&](const double* U, int wlo, int whi, int nw, int c_lo, int c_hi, bool above_z, int gw,
                          int gsize, unsigned u_remote = 0) {
        const int n_right = max(0, c_hi - c_lo), n_above = above_z ? wlo : 0;
        const int tr = (n_right + 7) / 8, ta = (n_above + 7) / 8, tz = above_z ? (d + 7) / 8 : 0;
        const int gq = lane >> 2, tq = lane & 3;
        double bf[8][4];
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
#pragma unroll
            for (int cb = 0; cb < 4; ++cb) {
                const int e = (cb * 8 + gq) * LDW + ks * 4 + tq;
                bf[ks][cb] = u_remote ? ld_cluster_f64(u_remote + 8u * e) : U[e];
            }
        // vector gq of a tile: base pointer and element stride
        auto locate = [&](int tile, double*& base, long long& st) -> bool {
            if (tile < tr) {
                const int c = c_lo + tile * 8 + gq;
                base = H + (size_t)min(c, d - 1) * d + wlo;
                st = 1;
                return c < c_hi;
            } else if (tile < tr + ta) {
                const int r = (tile - tr) * 8 + gq;
                base = H + min(r, n_above - 1) + (size_t)wlo * d;
                st = d;
                return r < n_above;
            }
            const int r = (tile - tr - ta) * 8 + gq;
            base = Z + min(r, d - 1) + (size_t)wlo * d;
            st = d;
            return r < d;
        };
        const int ntile = tr + ta + tz, wstep = gsize;
        double an[8];
        double* bnext = H;
        long long snext = 1;
        bool oknext = false;
        if (gw < ntile) {
            oknext = locate(gw, bnext, snext);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const int q = ks * 4 + tq;
                an[ks] = (oknext && q < nw) ? bnext[q * snext] : 0.0;
            }
        }
        // software pipeline: the next tile's vector segments are in flight while
        // the current tile is multiplied and stored
        for (int tile = gw; tile < ntile; tile += wstep) {
            double af[8];
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) af[ks] = an[ks];
            double* base = bnext;
            const long long st = snext;
            const bool ok = oknext;
            if (tile + wstep < ntile) {
                oknext = locate(tile + wstep, bnext, snext);
#pragma unroll
                for (int ks = 0; ks < 8; ++ks) {
                    const int q = ks * 4 + tq;
                    an[ks] = (oknext && q < nw) ? bnext[q * snext] : 0.0;
                }
            }
            double acc[4][2];
#pragma unroll
            for (int cb = 0; cb < 4; ++cb) acc[cb][0] = acc[cb][1] = 0.0;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
#pragma unroll
                for (int cb = 0; cb < 4; ++cb)
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                                 : "+d"(acc[cb][0]), "+d"(acc[cb][1])
                                 : "d"(af[ks]), "d"(bf[ks][cb]));
            // D[i][c]: vector i = gq, element c = cb*8 + 2tq (+1); all A loads of
            // this tile precede its stores (warp-synchronous)
            __syncwarp();
            if (ok) {
#pragma unroll
                for (int cb = 0; cb < 4; ++cb) {
                    const int c = cb * 8 + 2 * tq;
                    if (c < nw) base[c * st] = acc[cb][0];
                    if (c + 1 < nw) base[(c + 1) * st] = acc[cb][1];
                }
            }
        }
    };
    if (t == 0) {
        s_posted = 0u;
        s_done = 0u;
        s_partial = 0u;
    }
    cluster_sync_all();
    const unsigned a_posted = dsmem_addr(&s_posted, 0), a_done = dsmem_addr(&s_done, 0);
    const unsigned a_partial = dsmem_addr(&s_partial, 0);
    if (crank == 1) {
        // ---- updater CTA: apply posted chunk factors to H and Z, in order
        for (unsigned next = 0;; ++next) {
            if (t == 0)
                while (ld_acquire_cluster(a_posted) <= next) __nanosleep(64);
            __syncthreads();
            (void)ld_acquire_cluster(a_posted);
            const unsigned jb = dsmem_addr(&s_job[next & 1][0], 0);
            int jd[9];
#pragma unroll
            for (int q = 0; q < 9; ++q) jd[q] = ld_cluster_s32(jb + 4u * q);
            if (jd[7]) break;
            const unsigned ua = dsmem_addr(Us2 + (size_t)jd[0] * (MW * LDW), 0);
            // phase A: the columns the chaser's next-but-one chunk updates itself
            // ([c_lo, c_split)), published early; phase B: the rest of H and Z
            const int cs = min(max(jd[8], jd[4]), jd[5]);
            if (cs > jd[4]) apply_part(nullptr, jd[1], jd[2], jd[3], jd[4], cs, false, warp, nt / 32, ua);
            // publication: the CTA barrier orders every thread's writes before thread
            // 0's cluster-scope fence + release, which is cumulative over them -- one
            // fence per hand-off instead of one per thread
            __syncthreads();
            if (t == 0) {
                fence_cluster();
                st_release_cluster(a_partial, next + 1);
            }
            apply_part(nullptr, jd[1], jd[2], jd[3], cs, jd[5], jd[6] != 0, warp, nt / 32, ua);
            __syncthreads();
            if (t == 0) {
                fence_cluster();
                st_release_cluster(a_done, next + 1);
            }
        }
        cluster_sync_all();
        return;
    }
    unsigned jid = 0;  // jobs posted so far (rank 0)
    auto post_job = [&](int buf, int wlo, int whi, int nw, int c_lo, int c_hi, int above_z, int stop,
                        int c_split = 0) {
        // caller: one thread
        int* j = s_job[jid & 1];
        j[8] = c_split;
        j[0] = buf;
        j[1] = wlo;
        j[2] = whi;
        j[3] = nw;
        j[4] = c_lo;
        j[5] = c_hi;
        j[6] = above_z;
        j[7] = stop;
        fence_cluster();
        st_release_cluster(a_posted, jid + 1);
    };
    auto wait_done = [&](unsigned upto) {  // caller: one thread
        while (ld_acquire_cluster(a_done) < upto) __nanosleep(32);
    };
    auto wait_partial = [&](unsigned upto) {  // caller: one thread
        while (ld_acquire_cluster(a_partial) < upto) __nanosleep(32);
    };
    while (I >= 0) {
        int L = 0;
        bool conv = false;
        for (int its = 0; its <= itmax; ++its) {
            int kb = L;
            for (int k = L + 1 + t; k <= I; k += nt)
                if (small_subdiag_g(H, d, k, ulp, smlnum)) kb = max(kb, k);
            L = block_max_int(kb, &s_int);
            if (L > 0 && t == 0) H[L + (size_t)(L - 1) * d] = 0.0;
            __syncthreads();
            if (L >= I - 1) {
                conv = true;
                break;
            }
            ++kdefl;
            const int nsize = I - L + 1;
            int nb = nsize >= nb4_min ? 4 : (nsize >= nb2_min ? 2 : 1);
            if (kdefl % kexsh == 0) nb = 1;
            int M = L;
            double v0[3] = {0.0, 0.0, 0.0};
            if (nb == 1) {
                double h11, h12, h21, h22;
                if (kdefl % (2 * kexsh) == 0) {
                    const double s = fabs(hg(H, d, I, I - 1)) + fabs(hg(H, d, I - 1, I - 2));
                    h11 = 0.75 * s + hg(H, d, I, I);
                    h12 = -0.4375 * s;
                    h21 = s;
                    h22 = h11;
                } else if (kdefl % kexsh == 0) {
                    const double s = fabs(hg(H, d, L + 1, L)) + fabs(hg(H, d, L + 2, L + 1));
                    h11 = 0.75 * s + hg(H, d, L, L);
                    h12 = -0.4375 * s;
                    h21 = s;
                    h22 = h11;
                } else {
                    h11 = hg(H, d, I - 1, I - 1);
                    h21 = hg(H, d, I, I - 1);
                    h12 = hg(H, d, I - 1, I);
                    h22 = hg(H, d, I, I);
                }
                double rt1r, rt1i, rt2r, rt2i;
                {
                    const double s = fabs(h11) + fabs(h12) + fabs(h21) + fabs(h22);
                    if (s == 0.0) {
                        rt1r = rt1i = rt2r = rt2i = 0.0;
                    } else {
                        const double rs = 1.0 / s;
                        h11 *= rs;
                        h21 *= rs;
                        h12 *= rs;
                        h22 *= rs;
                        const double tr = (h11 + h22) / 2.0;
                        const double det = (h11 - tr) * (h22 - tr) - h12 * h21;
                        const double rtdisc = sqrt(fabs(det));
                        if (det >= 0.0) {
                            rt1r = tr * s;
                            rt2r = rt1r;
                            rt1i = rtdisc * s;
                            rt2i = -rt1i;
                        } else {
                            rt1r = tr + rtdisc;
                            rt2r = tr - rtdisc;
                            if (fabs(rt1r - h22) <= fabs(rt2r - h22)) {
                                rt1r *= s;
                                rt2r = rt1r;
                            } else {
                                rt2r *= s;
                                rt1r = rt2r;
                            }
                            rt1i = rt2i = 0.0;
                        }
                    }
                }
                int mb = L;
                for (int mm = L + 1 + t; mm <= I - 2; mm += nt) {
                    double vv[3];
                    start_vector_g(H, d, mm, rt1r, rt1i, rt2r, rt2i, vv);
                    const double h00 = fabs(hg(H, d, mm, mm - 1)) * (fabs(vv[1]) + fabs(vv[2]));
                    const double h11b = fabs(vv[0]) * (fabs(hg(H, d, mm - 1, mm - 1)) +
                                                       fabs(hg(H, d, mm, mm)) + fabs(hg(H, d, mm + 1, mm + 1)));
                    if (h00 <= ulp * h11b) mb = max(mb, mm);
                }
                M = block_max_int(mb, &s_int);
                start_vector_g(H, d, M, rt1r, rt1i, rt2r, rt2i, v0);
            } else {
                // ---- aggressive early deflation (dlaqr3 without reordering: the
                // contiguous bottom run of deflatable blocks) on the trailing
                // nwin x nwin window; its undeflated eigenvalues are the shifts.
                const int nwin = min(aed_nw, nsize / 2);
                const int kwtop = I - nwin + 1;
                const double sspike = hg(H, d, kwtop, kwtop - 1);
                const long long t_aed = clock64();
                if (warp == 0) {
                    for (int e = lane; e < MW * MW; e += 32) {
                        const int r = e % MW, c = e / MW;
                        Wn[r + c * LDW] = (r < nwin && c < nwin && r <= c + 1) ? hg(H, d, kwtop + r, kwtop + c) : 0.0;
                        Us[r + c * LDW] = (r == c) ? 1.0 : 0.0;
                    }
                    __syncwarp();
                    const bool ok = warp_small_schur(Wn, Us, nwin, s_esr, s_esi);
                    __syncwarp();
                    int ndefl = 0;
                    if (ok) {
                        int j = nwin - 1;
                        while (j >= 0) {
                            if (j > 0 && Wn[j + (j - 1) * LDW] != 0.0) {
                                double foo = fabs(Wn[j + j * LDW]) + sqrt(fabs(Wn[j + (j - 1) * LDW])) *
                                                                       sqrt(fabs(Wn[(j - 1) + j * LDW]));
                                if (foo == 0.0) foo = fabs(sspike);
                                const double sp = fmax(fabs(sspike * Us[j * LDW]), fabs(sspike * Us[(j - 1) * LDW]));
                                if (sp <= fmax(smlnum, ulp * foo)) {
                                    ndefl += 2;
                                    j -= 2;
                                } else {
                                    break;
                                }
                            } else {
                                double foo = fabs(Wn[j + j * LDW]);
                                if (foo == 0.0) foo = fabs(sspike);
                                if (fabs(sspike * Us[j * LDW]) <= fmax(smlnum, ulp * foo)) {
                                    ndefl += 1;
                                    j -= 1;
                                } else {
                                    break;
                                }
                            }
                        }
                    }
                    const int nd = nwin - ndefl;
                    if (ok && ndefl > 0 && nd > 1) {
                        // collapse the spike of the undeflated part onto its first row
                        for (int q = lane; q < nd; q += 32) s_vec[q] = Us[q * LDW];
                        __syncwarp();
                        double beta;
                        double tau = warp_dlarfg(s_vec, nd, &beta);
                        if (tau != 0.0) {
                            warp_refl_left(Wn, LDW, s_vec, nd, tau, 0, 0, nwin);
                            warp_refl_right(Wn, LDW, s_vec, nd, tau, 0, 0, nd);
                            warp_refl_right(Us, LDW, s_vec, nd, tau, 0, 0, nwin);
                        }
                        // back to Hessenberg form (dgehrd on the leading nd x nd block)
                        for (int j = 0; j + 2 < nd; ++j) {
                            const int len = nd - j - 1;
                            for (int q = lane; q < len; q += 32) s_vec[q] = Wn[(j + 1 + q) + j * LDW];
                            __syncwarp();
                            tau = warp_dlarfg(s_vec, len, &beta);
                            if (tau != 0.0) {
                                warp_refl_left(Wn, LDW, s_vec, len, tau, j + 1, j + 1, nwin);
                                warp_refl_right(Wn, LDW, s_vec, len, tau, j + 1, 0, nd);
                                warp_refl_right(Us, LDW, s_vec, len, tau, j + 1, 0, nwin);
                            }
                            for (int q = lane; q < len; q += 32) Wn[(j + 1 + q) + j * LDW] = (q == 0) ? beta : 0.0;
                            __syncwarp();
                        }
                    }
                    if (lane == 0) {
                        s_aed[0] = ok ? 1 : 0;
                        s_aed[1] = ndefl;
                        // nibble: many deflations -> deflate them and redo AED before sweeping
                        s_aed[2] = (ok && (nd < 2 || 100 * ndefl > nibble * nwin)) ? 1 : 0;
                        // shifts: bottom-most undeflated eigenvalues, conjugate pairs kept together
                        int nbul = 0, q = nd - 1;
                        double rbuf = 0.0;
                        bool have = false;
                        while (ok && q >= 0 && nbul < nb) {
                            if (s_esi[q] != 0.0 && q >= 1) {
                                s_pr[4 * nbul + 0] = s_esr[q];
                                s_pr[4 * nbul + 1] = fabs(s_esi[q]);
                                s_pr[4 * nbul + 2] = s_esr[q - 1];
                                s_pr[4 * nbul + 3] = -fabs(s_esi[q]);
                                ++nbul;
                                q -= 2;
                            } else if (have) {
                                s_pr[4 * nbul + 0] = rbuf;
                                s_pr[4 * nbul + 1] = 0.0;
                                s_pr[4 * nbul + 2] = s_esr[q];
                                s_pr[4 * nbul + 3] = 0.0;
                                ++nbul;
                                have = false;
                                q -= 1;
                            } else {
                                rbuf = s_esr[q];
                                have = true;
                                q -= 1;
                            }
                        }
                        s_aed[3] = nbul;
                    }
                }
                __syncthreads();
                cyc[6] += (unsigned long long)(clock64() - t_aed);
                cyc[7] += 1;
                if (s_aed[0] && s_aed[1] > 0) {
                    for (int idx = t; idx < nwin * nwin; idx += nt) {
                        const int r = idx % nwin, c = idx / nwin;
                        H[(kwtop + r) + (size_t)(kwtop + c) * d] = (r <= c + 1) ? Wn[c * LDW + r] : 0.0;
                    }
                    if (t == 0) H[kwtop + (size_t)(kwtop - 1) * d] = sspike * Us[0];
                    apply_part(Us, kwtop, I, nwin, I + 1, d, true, warp, nt / 32);
                    __syncthreads();
                    cyc[4] += (unsigned long long)s_aed[1];  // AED deflations
                }
                if (s_aed[0] && (s_aed[2] || s_aed[3] == 0)) continue;  // deflate first, then AED again
                if (s_aed[0]) {
                    nb = s_aed[3];
                    M = L;
                } else {
                    // fallback: 2 nb shifts from the trailing 2nb x 2nb block
                    const int n2 = 2 * nb, o = I - n2 + 1;
                    if (warp == 0) {
                        for (int e = lane; e < TQ * TQ; e += 32) {
                            const int r = e % TQ, c = e / TQ;
                            Sm[e] = (r < n2 && c < n2 && r <= c + 1) ? hg(H, d, o + r, o + c) : 0.0;
                        }
                        __syncwarp();
                        warp_tiny_eig(Sm, n2, s_sr, s_si);
                        __syncwarp();
                        if (lane == 0) {
                            // sort by decreasing modulus (conjugate pairs stay adjacent), then
                            // pair: complex pairs as they are, real shifts two at a time
                            double ar[TQ], ai[TQ];
                            for (int q = 0; q < n2; ++q) {
                                ar[q] = s_sr[q];
                                ai[q] = s_si[q];
                            }
                            int nbul = 0;
                            double rbuf = 0.0;
                            bool have = false;
                            for (int q = 0; q < n2; ++q) {
                                if (ai[q] != 0.0 && q + 1 < n2) {
                                    s_pr[4 * nbul + 0] = ar[q];
                                    s_pr[4 * nbul + 1] = fabs(ai[q]);
                                    s_pr[4 * nbul + 2] = ar[q + 1];
                                    s_pr[4 * nbul + 3] = -fabs(ai[q]);
                                    ++nbul;
                                    ++q;
                                } else if (have) {
                                    s_pr[4 * nbul + 0] = rbuf;
                                    s_pr[4 * nbul + 1] = 0.0;
                                    s_pr[4 * nbul + 2] = ar[q];
                                    s_pr[4 * nbul + 3] = 0.0;
                                    ++nbul;
                                    have = false;
                                } else {
                                    rbuf = ar[q];
                                    have = true;
                                }
                            }
                            if (have) {  // odd real count cannot happen with paired complex shifts
                                s_pr[4 * nbul + 0] = rbuf;
                                s_pr[4 * nbul + 1] = 0.0;
                                s_pr[4 * nbul + 2] = rbuf;
                                s_pr[4 * nbul + 3] = 0.0;
                                ++nbul;
                            }
                            s_nb = max(1, min(nbul, nb));
                        }
                    }
                    __syncthreads();
                    nb = s_nb;
                }
            }
            if (t == 0) s_t1 = 0.0;
            ++nsweep;
            const int S_total = (I - M) + 3 * (nb - 1);
            nstep += (unsigned long long)(I - M) * nb;
            if (nb > 1) cyc[5] += (unsigned long long)(I - M) * nb;
            tick(0);
            // Chunks of MS chase steps.  Warps 0-3 ("chasers") load the window, chase
            // the bulges (warps 0..nb-1), write the window back and apply the chunk
            // factor U_c to the few columns the NEXT window will read; warps 4-7
            // ("updaters") apply U_c to the rest of H and to Z while the chasers
            // already work on chunk c+1.  Named barriers: 1 = U_c published
            // (chasers arrive, updaters wait), 2 = rest of U_c done (updaters
            // arrive, chasers wait before touching columns it covers), 3 = chaser
            // group, 4 = chase steps.  U is double buffered.
            // chunk length: as many steps as the MW window holds for this bulge count
            const int ms = MW - 3 * (nb - 1) - 4;
            const int nchunk = (S_total + ms - 1) / ms;
            auto geom = [&](int c, int& wlo, int& whi) {
                const int s0 = c * ms, s1 = min(s0 + ms, S_total);
                const int kmin = max(M, M + s0 - 3 * (nb - 1));
                const int kmax = min(I - 1, M + s1 - 1);
                wlo = (kmin > M) ? kmin - 1 : M;
                whi = min(kmax + 3, I);
            };
            if (warp < 4) {
                const int tg = t;  // 0..127
                for (int c = 0; c < nchunk; ++c) {
                    const int s0 = c * ms, s1 = min(s0 + ms, S_total);
                    int wlo, whi;
                    geom(c, wlo, whi);
                    const int nw = whi - wlo + 1;
                    // U_c in buffer c % 3: its last user, job c - 3, is done (chunk c - 1
                    // waited for job c - 2's phase A, and jobs run in order)
                    double* Uc = Us2 + (c % 3) * (MW * LDW);
                    {
                        // all loads in flight before the first shared store (a generic H
                        // may alias shared memory, so interleaving would serialise them)
                        static_assert((MW * MW) % 128 == 0, "window tiling");
                        double wv[MW * MW / 128];
#pragma unroll
                        for (int q = 0; q < MW * MW / 128; ++q) {
                            const int idx = tg + 128 * q, r = idx % MW, cc = idx / MW;
                            wv[q] = (r < nw && cc < nw) ? H[(wlo + r) + (size_t)(wlo + cc) * d] : 0.0;
                        }
#pragma unroll
                        for (int q = 0; q < MW * MW / 128; ++q) {
                            const int idx = tg + 128 * q, r = idx % MW, cc = idx / MW;
                            Wn[r + cc * LDW] = wv[q];
                            Uc[r + cc * LDW] = (r == cc) ? 1.0 : 0.0;
                        }
                    }
                    named_bar(3, 128);
                    if (t == 0) tick(1);
                    if (warp < nb) {
                        auto W = [&](int r, int cc) -> double& { return Wn[(cc - wlo) * LDW + (r - wlo)]; };
                        const int bb = warp;
                        for (int s = s0; s < s1; ++s) {
                            const int k = M + s - 3 * bb;
                            const bool active = k >= M && k <= I - 1;
                            const int nr = active ? min(3, I - k + 1) : 0;
                            double v2 = 0.0, v3 = 0.0, t1 = 0.0, beta = 0.0;
                            if (active) {
                                double v1;
                                if (k > M) {
                                    v1 = W(k, k - 1);
                                    v2 = W(k + 1, k - 1);
                                    v3 = (nr == 3) ? W(k + 2, k - 1) : 0.0;
                                } else if (nb == 1) {
                                    v1 = v0[0];
                                    v2 = v0[1];
                                    v3 = (nr == 3) ? v0[2] : 0.0;
                                } else {
                                    double vv[3];
                                    start_vector_g(Wn, LDW, M - wlo, s_pr[4 * bb], s_pr[4 * bb + 1],
                                                   s_pr[4 * bb + 2], s_pr[4 * bb + 3], vv);
                                    v1 = vv[0];
                                    v2 = vv[1];
                                    v3 = (nr == 3) ? vv[2] : 0.0;
                                }
                                t1 = house3(v1, v2, v3, beta);
                                const double t2 = t1 * v2, t3 = t1 * v3;
                                __syncwarp();
                                for (int cc = k + lane; cc <= whi; cc += 32) {
                                    double& a0 = W(k, cc);
                                    double& a1 = W(k + 1, cc);
                                    const double a2v = (nr == 3) ? W(k + 2, cc) : 0.0;
                                    const double sum = a0 + v2 * a1 + v3 * a2v;
                                    a0 -= sum * t1;
                                    a1 -= sum * t2;
                                    if (nr == 3) W(k + 2, cc) = a2v - sum * t3;
                                }
                                __syncwarp();
                                if (lane == 0) {
                                    if (k > M) {
                                        W(k, k - 1) = beta;
                                        W(k + 1, k - 1) = 0.0;
                                        if (k < I - 1) W(k + 2, k - 1) = 0.0;
                                    } else if (nb == 1) {
                                        s_t1 = t1;  // H(M, M-1) *= (1 - t1) after the chunk
                                    }
                                }
                            }
                            named_bar(4, nb * 32);
                            if (active) {
                                const double t2 = t1 * v2, t3 = t1 * v3;
                                const int rmax = (nr == 3) ? min(k + 3, I) : I;
                                for (int r = wlo + lane; r <= rmax && r <= whi; r += 32) {
                                    double& a0 = W(r, k);
                                    double& a1 = W(r, k + 1);
                                    const double a2v = (nr == 3) ? W(r, k + 2) : 0.0;
                                    const double sum = a0 + v2 * a1 + v3 * a2v;
                                    a0 -= sum * t1;
                                    a1 -= sum * t2;
                                    if (nr == 3) W(r, k + 2) = a2v - sum * t3;
                                }
                                const int cu = k - wlo;
                                for (int r = lane; r < nw; r += 32) {
                                    double* u = Uc + r;
                                    const double u0 = u[cu * LDW], u1 = u[(cu + 1) * LDW];
                                    const double u2 = (nr == 3) ? u[(cu + 2) * LDW] : 0.0;
                                    const double sum = u0 + v2 * u1 + v3 * u2;
                                    u[cu * LDW] = u0 - sum * t1;
                                    u[(cu + 1) * LDW] = u1 - sum * t2;
                                    if (nr == 3) u[(cu + 2) * LDW] = u2 - sum * t3;
                                }
                            }
                            named_bar(4, nb * 32);
                        }
                    }
                    named_bar(3, 128);
                    if (t == 0) tick(2);
                    for (int idx = tg; idx < nw * nw; idx += 128) {
                        const int r = idx % nw, cc = idx / nw;
                        H[(wlo + r) + (size_t)(wlo + cc) * d] = Wn[cc * LDW + r];
                    }
                    if (c == 0 && nb == 1 && M > L && t == 0) H[M + (size_t)(M - 1) * d] *= (1.0 - s_t1);
                    // columns the next window reads: wait until the updaters are done
                    // with U_{c-1} (they cover the same columns), then apply U_c there
                    int wlo_n = wlo, whi_n = whi;
                    if (c + 1 < nchunk) geom(c + 1, wlo_n, whi_n);
                    // the updater CTA must be done with U_{c-1} on these columns: its job
                    // publishes them first (phase A), and jobs run in order, so every
                    // earlier job is done too
                    if (c >= 1 && t == 0) wait_partial(jid);
                    named_bar(3, 128);
                    if (whi_n > whi) apply_part(Uc, wlo, whi, nw, whi + 1, whi_n + 1, false, warp, 4);
                    named_bar(3, 128);  // (post_job: thread 0's fence + release, cumulative)
                    if (t == 0) {
                        // the columns chunk c + 2 will update itself: [c_lo, whi_{c+2}]
                        int c_split = 0;
                        if (c + 2 < nchunk) {
                            int w2lo, w2hi;
                            geom(c + 2, w2lo, w2hi);
                            c_split = w2hi + 1;
                        }
                        post_job(c % 3, wlo, whi, nw, max(whi, whi_n) + 1, d, 1, 0, c_split);
                    }
                    ++jid;
                    if (t == 0) tick(3);
                }
            }
            // end of sweep: every chunk factor applied before the deflation scan / AED
            if (t == 0) wait_done(jid);  // (jid is only meaningful in thread 0)
            __syncthreads();
        }
        if (!conv) {
            if (t == 0) {
                report_failure(status, kFailHqrNoConverge, 1, b, (double)I, (double)L);
                post_job(0, 0, 0, 0, 0, 0, 0, 1);
            }
            cluster_sync_all();
            return;
        }
        if (L == I) {
            if (t == 0) {
                wr[I] = hg(H, d, I, I);
                wi[I] = 0.0;
            }
        } else {
            double a = hg(H, d, I - 1, I - 1), bb = hg(H, d, I - 1, I), c = hg(H, d, I, I - 1),
                   dd = hg(H, d, I, I);
            double r1r, r1i, r2r, r2i, cs, sn;
            dlanv2(a, bb, c, dd, r1r, r1i, r2r, r2i, cs, sn);
            __syncthreads();
            if (t == 0) {
                H[(I - 1) + (size_t)(I - 1) * d] = a;
                H[(I - 1) + (size_t)I * d] = bb;
                H[I + (size_t)(I - 1) * d] = c;
                H[I + (size_t)I * d] = dd;
                wr[I - 1] = r1r;
                wi[I - 1] = r1i;
                wr[I] = r2r;
                wi[I] = r2i;
            }
            for (int j = I + 1 + t; j < d; j += nt) {
                double* x = H + (I - 1) + (size_t)j * d;
                const double xv = x[0], yv = x[1];
                x[0] = cs * xv + sn * yv;
                x[1] = cs * yv - sn * xv;
            }
            for (int j = t; j <= I - 2; j += nt) {
                double* x = H + j + (size_t)(I - 1) * d;
                const double xv = x[0], yv = x[d];
                x[0] = cs * xv + sn * yv;
                x[d] = cs * yv - sn * xv;
            }
            for (int j = t; j < d; j += nt) {
                double* zx = Z + j + (size_t)(I - 1) * d;
                const double xv = zx[0], yv = zx[d];
                zx[0] = cs * xv + sn * yv;
                zx[d] = cs * yv - sn * xv;
            }
        }
        kdefl = 0;
        I = L - 1;
        __syncthreads();
    }
    if (t == 0) {
        atomicAdd(&status->qr_sweeps, nsweep);
        atomicAdd(&status->qr_steps, nstep);
        for (int q = 0; q < 8; ++q) atomicAdd(&status->qr_cycles[q], cyc[q]);
        if (trace) {  // debug (vrte_cuda_schur trace): per-matrix cost profile
            double* tr = trace + (size_t)b * 8;
            tr[0] = (double)(cyc[0] + cyc[1] + cyc[2] + cyc[3]);
            tr[1] = (double)nstep;
            tr[2] = (double)nsweep;
            tr[3] = (double)cyc[7];
            tr[4] = (double)cyc[6];
            tr[5] = (double)cyc[2];
            tr[6] = (double)cyc[3];
            tr[7] = (double)cyc[4];
        }
    }
    for (int idx = t; idx < d * d; idx += nt) {
        const int r = idx % d, c = idx / d;
        if (r > c + 1) H[idx] = 0.0;
    }
    if (t == 0) post_job(0, 0, 0, 0, 0, 0, 0, 1);  // stop the updater CTA
    cluster_sync_all();                              // it reads our shared memory until then
}

// ------------------------------------------------------------------ 2x2 solves
// Complete-pivoting 2x2 solve with the dlaln2 small-pivot perturbation smin
// (smin <= 0 disables the perturbation).
__device__ void solve2(cplx c00, cplx c01, cplx c10, cplx c11, cplx b0, cplx b1, double smin,
                       cplx& x0, cplx& x1) {
    const double m00 = cabs_(c00), m01 = cabs_(c01), m10 = cabs_(c10), m11 = cabs_(c11);
    int pr = 0, pc = 0;
    double mx = m00;
    if (m01 > mx) { mx = m01; pr = 0; pc = 1; }
    if (m10 > mx) { mx = m10; pr = 1; pc = 0; }
    if (m11 > mx) { mx = m11; pr = 1; pc = 1; }
    if (smin > 0.0 && mx < smin) {
        x0 = cdiv(b0, cmk(smin, 0.0));
        x1 = cdiv(b1, cmk(smin, 0.0));
        return;
    }
    cplx C[2][2] = {{c00, c01}, {c10, c11}};
    cplx B[2] = {b0, b1};
    const int qr = 1 - pr, qc = 1 - pc;
    const cplx piv = C[pr][pc];
    const cplx l = cdiv(C[qr][pc], piv);
    cplx u22 = C[qr][qc] - l * C[pr][qc];
    if (smin > 0.0 && cabs_(u22) < smin) u22 = cmk(smin, 0.0);
    const cplx y = B[qr] - l * B[pr];
    cplx X[2];
    X[qc] = cdiv(y, u22);
    X[pc] = cdiv(B[pr] - C[pr][qc] * X[qc], piv);
    x0 = X[0];
    x1 = X[1];
}


// Real version of solve2 (complete pivoting, dlaln2-style smin perturbation).
__device__ void solve2r(double c00, double c01, double c10, double c11, double b0, double b1, double smin,
                        double& x0, double& x1) {
    const double m00 = fabs(c00), m01 = fabs(c01), m10 = fabs(c10), m11 = fabs(c11);
    int pr = 0, pc = 0;
    double mx = m00;
    if (m01 > mx) { mx = m01; pr = 0; pc = 1; }
    if (m10 > mx) { mx = m10; pr = 1; pc = 0; }
    if (m11 > mx) { mx = m11; pr = 1; pc = 1; }
    if (smin > 0.0 && mx < smin) {
        x0 = b0 / smin;
        x1 = b1 / smin;
        return;
    }
    const double cpp = pr ? (pc ? c11 : c10) : (pc ? c01 : c00);   // C[pr][pc]
    const double cqp = pr ? (pc ? c01 : c00) : (pc ? c11 : c10);   // C[qr][pc]
    const double cpq = pr ? (pc ? c10 : c11) : (pc ? c00 : c01);   // C[pr][qc]
    const double cqq = pr ? (pc ? c00 : c01) : (pc ? c10 : c11);   // C[qr][qc]
    const double bp = pr ? b1 : b0, bq = pr ? b0 : b1;
    const double l = cqp / cpp;
    double u22 = cqq - l * cpq;
    if (smin > 0.0 && fabs(u22) < smin) u22 = smin;
    const double xq = (bq - l * bp) / u22;
    const double xp = (bp - cpq * xq) / cpp;
    x0 = pc ? xq : xp;
    x1 = pc ? xp : xq;
}







// ------------------------------------------------------------------ blocked trevc
// Right eigenvectors of the quasi-triangular Schur factor by BLOCKED back
// substitution (the dtrevc3 organisation): rows in blocks of TBK from the
// bottom; per block, every eigenvector solves its shifted diagonal block (a
// group of 4 threads per eigen-block leader: one solves each row, the four
// share the row updates; the block's rows and T's diagonal block in shared
// memory), then ONE shift-free update of every row above by all the
// slice's eigenvectors, Y[0:j0, :] -= T[0:j0, j0:j1] Y[j0:j1, :] (the
// off-diagonal part of T - lambda I carries no shift).  CTA per (matrix,
// slice of W leader columns); the slice of Y lives in shared memory.  Same
// arithmetic choices as LAPACK dtrevc (dlaln2-style smin, solve2 / solve2r
// on 2x2 blocks, the complex pair's fixed entries).
constexpr int TBK = 32;
template <int W, int GS>
__global__ void __launch_bounds__(256) trevc_blk_kernel(const double* Tall, const double* wrall, const double* wiall,
                                                        double* Yall, int d, int stage_t) {
    extern __shared__ double shm[];
    constexpr int LDY = W + 4;       // slice columns (a leader's pair partner may be column W), padded to 4
    constexpr int LDD = TBK + 2;     // diagonal block [TBK + 1]^2
    double* Ys = shm;                          // [d][LDY]
    double* Td = Ys + (size_t)d * LDY;         // [TBK + 1][LDD]
    double* Tp = Td + (size_t)(TBK + 1) * LDD;  // [d][LDD] column panel T[0:j0, j0:j1] (stage_t)
    __shared__ int s_top;
    const int b = blockIdx.x, c0 = blockIdx.y * W, t = threadIdx.x, nt = blockDim.x;
    const double* T = Tall + (size_t)b * d * d;
    const double* wr = wrall + (size_t)b * d;
    const double* wi = wiall + (size_t)b * d;
    double* Y = Yall + (size_t)b * d * d;
    auto Tg = [&](int r, int c) { return T[r + (size_t)c * d]; };
    for (int e = t; e < d * LDY; e += nt) Ys[e] = 0.0;
    if (t == 0) s_top = -1;
    __syncthreads();
    // leader state: a group of 4 threads per local column lc (W <= nt / 4); lane q = 0
    // of the group solves each row, the 4 lanes share the row updates
    const int lc = t / GS, q = t % GS;
    const unsigned gmask = (GS >= 32) ? 0xffffffffu : (((1u << GS) - 1u) << ((t & 31) & ~(GS - 1)));
    const int k = c0 + lc;
    const bool lead = lc < W && k < d && wi[k] >= 0.0;
    const bool cx = lead && wi[k] > 0.0;
    const double lr = lead ? wr[k] : 0.0, li = lead ? wi[k] : 0.0;
    const double sm = lead ? fmax(kUlp * (fabs(lr) + fabs(li)), kSafeMin * ((double)d / kUlp)) : 1.0;
    const int top = lead ? (cx ? k + 1 : k) : -1;
    if (lead && q == 0) {
        if (!cx) {
            Ys[(size_t)k * LDY + lc] = 1.0;
        } else {
            double xpr, xqi;
            const double tu = Tg(k, k + 1), tl = Tg(k + 1, k);
            if (fabs(tu) >= fabs(tl)) {
                xpr = 1.0;
                xqi = li / tu;
            } else {
                xpr = -li / tl;
                xqi = 1.0;
            }
            Ys[(size_t)k * LDY + lc] = xpr;
            Ys[(size_t)(k + 1) * LDY + lc + 1] = xqi;
        }
        atomicMax(&s_top, top);
    }
    __syncthreads();
    int j1 = s_top + 1;
    const int ncol = min(W + 1, d - c0);  // slice columns touched (leaders and partners)
    while (j1 > 0) {
        int j0 = max(0, j1 - TBK);
        if (j0 > 0 && Tg(j0, j0 - 1) != 0.0) --j0;  // never split a 2x2 Schur block
        const int nb = j1 - j0;
        for (int e = t; e < nb * nb; e += nt) {
            const int r = e % nb, c = e / nb;
            Td[r * LDD + c] = Tg(j0 + r, j0 + c);
        }
        if (stage_t && j0 > 0)
            for (int e = t; e < j0 * nb; e += nt) {
                const int r = e % j0, c = e / j0;  // coalesced along the column
                Tp[(size_t)r * LDD + c] = Tg(r, j0 + c);
            }
        __syncthreads();
        // ---- per-eigenvector solve of the diagonal block
        if (lead && j0 <= top) {
            auto Td_ = [&](int r, int c) { return Td[(r - j0) * LDD + (c - j0)]; };
            double* yr = Ys + lc;
            double* yi = Ys + lc + 1;
            for (int j = min(j1 - 1, top); j >= j0; --j) {
                const bool pr = j > j0 && Td_(j, j - 1) != 0.0;  // rows (j-1, j): a 2x2 Schur block
                const bool two = pr || (cx && j == top);
                if (q == 0 && j != top) {  // the solve of row j (rows j-1, j of a 2x2 block)
                    if (!cx) {
                        if (pr) {
                            double x0, x1;
                            solve2r(Td_(j - 1, j - 1) - lr, Td_(j - 1, j), Td_(j, j - 1), Td_(j, j) - lr,
                                    yr[(size_t)(j - 1) * LDY], yr[(size_t)j * LDY], sm, x0, x1);
                            yr[(size_t)(j - 1) * LDY] = x0;
                            yr[(size_t)j * LDY] = x1;
                        } else {
                            double den = Td_(j, j) - lr;
                            if (fabs(den) < sm) den = sm;
                            yr[(size_t)j * LDY] /= den;
                        }
                    } else {
                        const cplx lam = cmk(lr, li);
                        if (pr) {
                            const cplx b0 = cmk(yr[(size_t)(j - 1) * LDY], yi[(size_t)(j - 1) * LDY]);
                            const cplx b1 = cmk(yr[(size_t)j * LDY], yi[(size_t)j * LDY]);
                            cplx x0, x1;
                            solve2(cmk(Td_(j - 1, j - 1), 0.0) - lam, cmk(Td_(j - 1, j), 0.0),
                                   cmk(Td_(j, j - 1), 0.0), cmk(Td_(j, j), 0.0) - lam, b0, b1, sm, x0, x1);
                            yr[(size_t)(j - 1) * LDY] = x0.re;
                            yi[(size_t)(j - 1) * LDY] = x0.im;
                            yr[(size_t)j * LDY] = x1.re;
                            yi[(size_t)j * LDY] = x1.im;
                        } else {
                            cplx den = cmk(Td_(j, j), 0.0) - lam;
                            if (cabs_(den) < sm) den = cmk(sm, 0.0);
                            const cplx x = cdiv(cmk(yr[(size_t)j * LDY], yi[(size_t)j * LDY]), den);
                            yr[(size_t)j * LDY] = x.re;
                            yi[(size_t)j * LDY] = x.im;
                        }
                    }
                }
                __syncwarp(gmask);
                // rows above inside the block, split over the group's GS lanes
                const int lim = two ? j - 1 : j;
                const double x1r = yr[(size_t)j * LDY];
                const double x0r = two ? yr[(size_t)(j - 1) * LDY] : 0.0;
                if (!cx) {
                    for (int i = j0 + q; i < lim; i += GS) {
                        double v = yr[(size_t)i * LDY] - Td_(i, j) * x1r;
                        if (two) v -= Td_(i, j - 1) * x0r;
                        yr[(size_t)i * LDY] = v;
                    }
                } else {
                    const double x1i = yi[(size_t)j * LDY];
                    const double x0i = two ? yi[(size_t)(j - 1) * LDY] : 0.0;
                    for (int i = j0 + q; i < lim; i += GS) {
                        double vr = yr[(size_t)i * LDY] - Td_(i, j) * x1r;
                        double vi = yi[(size_t)i * LDY] - Td_(i, j) * x1i;
                        if (two) {
                            vr -= Td_(i, j - 1) * x0r;
                            vi -= Td_(i, j - 1) * x0i;
                        }
                        yr[(size_t)i * LDY] = vr;
                        yi[(size_t)i * LDY] = vi;
                    }
                }
                __syncwarp(gmask);
                if (two) --j;
            }
        }
        __syncthreads();
        // ---- shift-free update of the rows above: Y[0:j0, :] -= T[0:j0, j0:j1] Y[j0:j1, :],
        // 4 x 4 register tiles per thread (columns padded to LDY, a multiple of 4)
        {
            const int rt = (j0 + 3) / 4, ct = (ncol + 3) / 4;
            for (int e = t; e < rt * ct; e += nt) {
                const int r0 = 4 * (e / ct), cc = 4 * (e % ct);
                double acc[4][4];
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int c = 0; c < 4; ++c) acc[a][c] = 0.0;
                for (int q = 0; q < nb; ++q) {
                    double tv[4];
#pragma unroll
                    for (int a = 0; a < 4; ++a) {
                        const int r = min(r0 + a, j0 - 1);
                        tv[a] = stage_t ? Tp[(size_t)r * LDD + q] : Tg(r, j0 + q);
                    }
                    const double* yq = Ys + (size_t)(j0 + q) * LDY + cc;
                    const double y0 = yq[0], y1 = yq[1], y2 = yq[2], y3 = yq[3];
#pragma unroll
                    for (int a = 0; a < 4; ++a) {
                        acc[a][0] = fma(tv[a], y0, acc[a][0]);
                        acc[a][1] = fma(tv[a], y1, acc[a][1]);
                        acc[a][2] = fma(tv[a], y2, acc[a][2]);
                        acc[a][3] = fma(tv[a], y3, acc[a][3]);
                    }
                }
#pragma unroll
                for (int a = 0; a < 4; ++a)
                    if (r0 + a < j0)
#pragma unroll
                        for (int c = 0; c < 4; ++c) Ys[(size_t)(r0 + a) * LDY + cc + c] -= acc[a][c];
            }
        }
        __syncthreads();
        j1 = j0;
    }
    // write the slice's columns: leaders k (and their partners k + 1)
    for (int e = t; e < d * ncol; e += nt) {
        const int r = e % d, c = e / d;
        const int kk = c0 + c;
        if (kk >= d) continue;
        const bool own = c < W ? true : (wi[kk] < 0.0);  // column W: the partner of the last leader
        if (c < W && c == 0 && wi[kk] < 0.0) continue;  // column c0 is the previous slice's partner
        if (!own) continue;
        Y[(size_t)kk * d + r] = Ys[(size_t)r * LDY + c];
    }
}

// ------------------------------------------------------------------ normalization
__global__ void normalize_modes_kernel(double* Xall, const double* wiall, int d, int batch) {
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (gw >= batch * d) return;
    const int b = gw / d, j = gw % d;
    const double wij = wiall[(size_t)b * d + j];
    if (wij < 0.0) return;
    double* x = Xall + (size_t)b * d * d + (size_t)j * d;
    double m = 0.0;
    if (wij == 0.0) {
        for (int i = lane; i < d; i += 32) m = fmax(m, fabs(x[i]));
    } else {
        for (int i = lane; i < d; i += 32) m = fmax(m, hypot(x[i], x[i + d]));
    }
    m = warp_max(m);
    if (m == 0.0) return;
    for (int i = lane; i < d; i += 32) {
        x[i] /= m;
        if (wij > 0.0) x[i + d] /= m;
    }
}

// ------------------------------------------------------------------ modes
// homogeneous.cpp:157-210: nu from lambda (floor / negative-axis / clamp
// rules) and the recovery psi+- = (1/2) M^{-1} (x -+ nu E x).  Warp per mode.
__global__ void modes_kernel(ModeArgs a) {
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int d = a.d;
    if (gw >= a.batch * d) return;
    const int b = gw / d, j = gw % d;
    const size_t vb = (size_t)b * d;
    const double wij = a.wi[vb + j];
    if (wij < 0.0) return;
    const bool pair = wij > 0.0;
    cplx lam = cmk(a.wr[vb + j], wij);
    if (!isfinite(lam.re) || !isfinite(lam.im)) {
        if (lane == 0)
            report_failure(a.status, kFailNonFiniteEigen, 1,
                           a.order_index ? a.order_index[b] : b, lam.re);
        return;
    }
    const double floor = 1e-12 * fmax(1.0, a.femax[b]);
    const bool conservative = cabs_(lam) < floor;
    cplx nu;
    if (conservative) {
        nu = cmk(kNuClamp, 0.0);
    } else {
        if (lam.re < 0.0 && fabs(lam.im) < 1e-10 * fabs(lam.re) && cabs_(lam) < 1e-10)
            lam = cmk(cabs_(lam), 0.0);
        nu = cdiv(cmk(1.0, 0.0), csqrt_(lam));
        if (nu.re < 0.0) nu = cmk(-nu.re, -nu.im);
        if (nu.re == 0.0) {
            if (lane == 0)
                report_failure(a.status, kFailNegativeAxis, 1,
                               a.order_index ? a.order_index[b] : b, lam.re);
            return;
        }
        const double an = cabs_(nu);
        if (an > kNuClamp) nu = (kNuClamp / an) * nu;
    }
    const size_t cb = (size_t)b * d * d + (size_t)j * d;
    for (int i = lane; i < d; i += 32) {
        const cplx x = cmk(a.X[cb + i], pair ? a.X[cb + d + i] : 0.0);
        const double hm = 0.5 * (1.0 / a.mdiag[i]);
        cplx pp, pm;
        if (conservative) {
            pp = hm * x;
            pm = pp;
        } else {
            const cplx ex = cmk(a.EX[cb + i], pair ? a.EX[cb + d + i] : 0.0);
            const cplx nex = nu * ex;
            pp = hm * (x - nex);
            pm = hm * (x + nex);
        }
        const double mu = a.mdiag[i];
        const cplx sum = mu * (pp + pm), dif = mu * (pm - pp);
        a.psi_p[cb + i] = pp.re;
        a.psi_m[cb + i] = pm.re;
        a.ab_sum[cb + i] = sum.re;
        a.ab_dif[cb + i] = dif.re;
        if (pair) {
            a.psi_p[cb + d + i] = pp.im;
            a.psi_m[cb + d + i] = pm.im;
            a.ab_sum[cb + d + i] = sum.im;
            a.ab_dif[cb + d + i] = dif.im;
        }
    }
    if (lane == 0) {
        double* nv = a.nu + 2 * (vb + j);
        nv[0] = nu.re;
        nv[1] = nu.im;
        double* lv = a.lam + 2 * (vb + j);
        lv[0] = lam.re;
        lv[1] = lam.im;
        a.flags[vb + j] = conservative ? 1 : 0;
        if (pair) {
            nv[2] = nu.re;
            nv[3] = -nu.im;
            lv[2] = lam.re;
            lv[3] = -lam.im;
            a.flags[vb + j + 1] = conservative ? 1 : 0;
        }
    }
}

// 8N residual ||Op v - v/nu|| / ||v|| via the reduced operators:
// top = M^-1(-G1 + G2)/2 - psi+/nu, bottom = M^-1(G1 + G2)/2 - psi-/nu.
__global__ void residual_kernel(ResidualArgs a) {
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int d = a.d;
    if (gw >= a.batch * d) return;
    const int b = gw / d, j = gw % d;
    const size_t vb = (size_t)b * d;
    const double wij = a.wi[vb + j];
    if (wij < 0.0) return;
    const bool pair = wij > 0.0;
    const cplx nu = cmk(a.nu[2 * (vb + j)], a.nu[2 * (vb + j) + 1]);
    const cplx inu = cdiv(cmk(1.0, 0.0), nu);
    const size_t cb = (size_t)b * d * d + (size_t)j * d;
    double num = 0.0, den = 0.0;
    for (int i = lane; i < d; i += 32) {
        auto ld = [&](const double* p) { return cmk(p[cb + i], pair ? p[cb + d + i] : 0.0); };
        const cplx g1 = ld(a.G1), g2 = ld(a.G2), pp = ld(a.psi_p), pm = ld(a.psi_m);
        const double im = 1.0 / a.mdiag[i];
        const cplx rt = (0.5 * im) * (g2 - g1) - pp * inu;
        const cplx rb = (0.5 * im) * (g1 + g2) - pm * inu;
        num = fmax(num, fmax(cabs_(rt), cabs_(rb)));
        den = fmax(den, fmax(cabs_(pp), cabs_(pm)));
    }
    num = warp_max(num);
    den = warp_max(den);
    if (lane == 0) {
        const double r = den > 0.0 ? num / den : 0.0;
        a.residual[vb + j] = r;
        if (pair) a.residual[vb + j + 1] = r;
    }
}

// ------------------------------------------------------------------ shifted solves
// Blocked back substitution for (T - sigma_c I) y_c = w_c on the quasi-
// triangular Schur factor, many right-hand sides with per-column shifts.
// CTA per (matrix, 32-column tile); the tile lives in shared memory.  Row
// blocks are processed bottom-up: the strictly-upper coupling
// W[J,:] -= T[J, J+1:] Y[J+1:, :] is shift independent (a shared panel product,
// T read coalesced from L2 once per tile), and only the small diagonal block
// is solved per column with its own shift (1x1 / 2x2 Schur blocks, complex
// pairs = packed Re/Im columns handled by one thread).  kind[c]: 0 real,
// 1 complex pair (c: Re, c+1: Im), 2 skip.
constexpr int QBS = 32;   // row block
constexpr int QCT = 32;   // column tile


// ------------------------------------------------------------------ eigenbasis solves
// (Lambda - sigma_c) y_c = w_c with Lambda the real-packed eigenvalue matrix of
// F E = V Lambda V^-1 (trevc packing: real eigenvalue k -> 1x1; complex pair
// k (wi > 0), k+1 -> block [[a, b], [-b, a]] acting on the Re/Im columns).
// Together with the GEMMs W = V^-1 R and Y = V W this replaces the blocked
// quasi-triangular back substitution: every (matrix, column, eigen-block) is
// independent.  The 2x2 block is diagonalised exactly (eigenvectors [1, +-i])
// so a shift next to a + ib loses no accuracy to cancellation in its
// determinant.  Column kinds: 0 real, 1 complex pair
// (c: Re, c+1: Im), 2 skip.
__global__ void eig_diag_solve_kernel(double* Wall, int d, int ncol, long long w_stride,
                                      const double* wrall, const double* wiall,
                                      const double* sigma, const int* kind, int batch) {
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (idx >= (long long)batch * ncol * d) return;
    const int k = (int)(idx % d);
    const long long bc = idx / d;
    const int c = (int)(bc % ncol), b = (int)(bc / ncol);
    const int kd = kind[(size_t)b * ncol + c];
    if (kd != 0 && kd != 1) return;
    const double wik = wiall[(size_t)b * d + k];
    if (wik < 0.0) return;  // second row of a pair: handled with its leader
    const bool cx = kd == 1;
    const cplx sg = cmk(sigma[2 * ((size_t)b * ncol + c)], sigma[2 * ((size_t)b * ncol + c) + 1]);
    double* wre = Wall + (size_t)b * w_stride + (size_t)c * d;
    double* wim = wre + d;
    const double a = wrall[(size_t)b * d + k];
    // x / den as x conj(den) / |den|^2: one FP64 division instead of three (the
    // denominators are eigenvalue gaps, far from the squares' over/underflow)
    auto qdiv = [](cplx x, cplx den) {
        const double r = 1.0 / fma(den.re, den.re, den.im * den.im);
        return cmk(fma(x.re, den.re, x.im * den.im) * r, fma(x.im, den.re, -x.re * den.im) * r);
    };
    if (wik == 0.0) {
        const cplx x = qdiv(cmk(wre[k], cx ? wim[k] : 0.0), cmk(a, 0.0) - sg);
        wre[k] = x.re;
        if (cx) wim[k] = x.im;
        return;
    }
    // pair rows k, k+1: y = alpha [1; i] + beta [1; -i]
    const cplx w0 = cmk(wre[k], cx ? wim[k] : 0.0);
    const cplx w1 = cmk(wre[k + 1], cx ? wim[k + 1] : 0.0);
    const cplx iw1 = cmk(-w1.im, w1.re);
    const cplx al = qdiv(0.5 * (w0 - iw1), cmk(a, wik) - sg);
    const cplx be = qdiv(0.5 * (w0 + iw1), cmk(a, -wik) - sg);
    const cplx y0 = al + be, dif = al - be;
    const cplx y1 = cmk(-dif.im, dif.re);
    wre[k] = y0.re;
    wre[k + 1] = y1.re;
    if (cx) {
        wim[k] = y0.im;
        wim[k + 1] = y1.im;
    }
}

// Free-streaming orders: for m >= the last coefficient of a medium (or
// omega = 0) the azimuthal kernel vanishes identically, E = F = M^-1 and
// F E = M^-2.  Its modes are analytic -- x = e_j, lambda = 1/mu^2, nu = mu,
// psi+ = (1/2) M^-1 (x - nu E x) = 0, psi- = M^-1 x -- and the beam source (and
// so the particular solution) is zero (particular.cpp "max|X| = 0").  Slots
// [b0, b1) are filled directly instead of running the eigen pipeline.
__global__ void free_modes_kernel(int d, int b0, int b1, const double* mdiag, double* psi_p,
                                  double* psi_m, double* nu, double* wr, double* wi, double* residual,
                                  double* zp, double* zm, int R) {
    const long long per = (long long)d * d;
    const long long total = (long long)(b1 - b0) * per;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int b = b0 + (int)(e / per);
        const long long w = e % per;
        const int i = (int)(w % d), j = (int)(w / d);
        const size_t o = (size_t)b * per + w;
        psi_p[o] = 0.0;
        psi_m[o] = (i == j) ? 1.0 / mdiag[j] : 0.0;
        if (i == 0) {
            const size_t vb = (size_t)b * d + j;
            nu[2 * vb] = mdiag[j];
            nu[2 * vb + 1] = 0.0;
            wr[vb] = 1.0 / (mdiag[j] * mdiag[j]);
            wi[vb] = 0.0;
            residual[vb] = 0.0;
        }
    }
    const long long tz = (long long)(b1 - b0) * d * R;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tz;
         e += (long long)gridDim.x * blockDim.x) {
        const size_t o = (size_t)b0 * d * R + e;
        zp[o] = 0.0;
        zm[o] = 0.0;
    }
}

}  // namespace

void launch_max_abs(const double* A, long long per, int batch, double* out, cudaStream_t st) {
    max_abs_kernel<<<batch, 256, 0, st>>>(A, per, out);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

void launch_hessenberg(double* A, double* Z, int d, int batch, cudaStream_t st) {
    hessenberg_kernel<<<batch, NT, d * sizeof(double), st>>>(A, Z, d);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

void launch_hqr(double* H, double* Z, double* wr, double* wi, int d, int batch,
                DeviceStatus* status, cudaStream_t st, double* trace, bool lean) {
    // 2-CTA clusters: rank 0 chases / deflates, rank 1 applies the chunk factors.
    // lean: the 128-register build (some spills, 2 CTAs per SM) for plans that run
    // concurrently with others (spectral batch, order shards in flight); a lone
    // solve takes the 229-register build (1 CTA per SM, no spills, ~9% faster)
    // (4 bulges per sweep from an active block of 32 rows, 2 from 16: measured against
    // 48 / 24 -- C3 QR 9.08 -> 9.00 ms, C1 0.87 -> 0.72 ms, C4' 104 -> 100 ms)
    if (lean)
        hqr_multi_kernel<2><<<2 * batch, 256, 0, st>>>(H, Z, wr, wi, d, status, AED_NW, 32, 16, 40, trace);
    else
        hqr_multi_kernel<1><<<2 * batch, 256, 0, st>>>(H, Z, wr, wi, d, status, AED_NW, 32, 16, 40, trace);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

void launch_trevc(const double* T, const double* wr, const double* wi, double* Y, int d,
                  int batch, cudaStream_t st) {
    // blocked back substitution (trevc_blk_kernel): W leader columns per CTA and GS
    // threads per leader (W GS = 256), the slice of Y in shared memory sized for
    // two CTAs per SM; T's column panel is read from L2
    auto smem = [&](int W) { return ((size_t)d * (W + 4) + (size_t)(TBK + 1) * (TBK + 2)) * sizeof(double); };
    static unsigned long long a32 = 0, a16 = 0, a8 = 0;
    if (d <= 256) {
        smem_attr_once(trevc_blk_kernel<32, 8>, 110 * 1024, a32);
        trevc_blk_kernel<32, 8><<<dim3(batch, (d + 31) / 32), 256, smem(32), st>>>(T, wr, wi, Y, d, 0);
    } else if (d <= 512) {
        smem_attr_once(trevc_blk_kernel<16, 16>, 110 * 1024, a16);
        trevc_blk_kernel<16, 16><<<dim3(batch, (d + 15) / 16), 256, smem(16), st>>>(T, wr, wi, Y, d, 0);
    } else {
        smem_attr_once(trevc_blk_kernel<8, 32>, 110 * 1024, a8);
        trevc_blk_kernel<8, 32><<<dim3(batch, (d + 7) / 8), 256, smem(8), st>>>(T, wr, wi, Y, d, 0);
    }
    VRTE_CUDA_CHECK(cudaGetLastError());
}

void launch_normalize_modes(double* X, const double* wi, int d, int batch, cudaStream_t st) {
    const long long warps = (long long)batch * d;
    normalize_modes_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(X, wi, d, batch);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

void launch_modes(const ModeArgs& a, cudaStream_t st) {
    const long long warps = (long long)a.batch * a.d;
    modes_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(a);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

void launch_residual(const ResidualArgs& a, cudaStream_t st) {
    const long long warps = (long long)a.batch * a.d;
    residual_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(a);
    VRTE_CUDA_CHECK(cudaGetLastError());
}


void launch_eig_diag_solve(double* W, int d, int ncol, long long w_stride, const double* wr,
                           const double* wi, const double* sigma, const int* kind, int batch,
                           cudaStream_t st) {
    const long long total = (long long)batch * ncol * d;
    if (total == 0) return;
    eig_diag_solve_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(W, d, ncol, w_stride, wr, wi,
                                                                          sigma, kind, batch);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

__global__ void set_identity_batched_kernel(double* Z, int d, long long total) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long w = e % ((long long)d * d);
        Z[e] = (w % d == w / d) ? 1.0 : 0.0;
    }
}

__global__ void fill_int_kernel(int* p, int n, int v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

void launch_fill_int(int* p, int n, int value, cudaStream_t st) {
    if (n <= 0) return;
    fill_int_kernel<<<(n + 255) / 256, 256, 0, st>>>(p, n, value);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

void launch_set_identity(double* Z, int d, int batch, cudaStream_t st) {
    const long long total = (long long)d * d * batch;
    const long long blocks = (total + 255) / 256;
    set_identity_batched_kernel<<<(unsigned)(blocks < 8192 ? blocks : 8192), 256, 0, st>>>(Z, d, total);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

void launch_free_modes(int d, int b0, int b1, const double* mdiag, double* psi_p, double* psi_m,
                       double* nu, double* wr, double* wi, double* residual, double* zp, double* zm, int R,
                       cudaStream_t st) {
    if (b1 <= b0) return;
    const long long total = (long long)(b1 - b0) * d * d;
    const long long blocks = (total + 255) / 256;
    free_modes_kernel<<<(unsigned)(blocks < 8192 ? blocks : 8192), 256, 0, st>>>(d, b0, b1, mdiag, psi_p, psi_m, nu,
                                                                               wr, wi, residual, zp, zm, R);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace vrte
