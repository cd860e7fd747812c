// hessenberg.cu -- blocked Householder reduction to upper Hessenberg form,
// A <- Q^T A Q, for every (medium, order) matrix F*E at once, and the explicit
// Q that seeds the Schur vectors of the Francis QR (eig.cu).
//
// Reference: Eigen::EigenSolver -> RealSchur -> HessenbergDecomposition
// (homogeneous.cpp:135); the algorithm here is the dgehrd / dlahr2 / dorghr
// organisation, restated for one SM per matrix:
//
//   hess_panel_kernel (CTA per matrix, nb columns): column j of the panel is
//     brought up to date with the deferred panel transformations
//       col = A[:,k] - Y_j V_j[k,:]^T,  col[c0+1:] <- (I - V_j T_j^T V_j^T) col
//     its reflector H_j = I - tau v v^T is generated (dlarfg), and the only
//     full-matrix pass of the step -- the matvec A v over the start-of-panel
//     matrix -- feeds Y = A V T:  Y[:,j] = tau (A v - Y_j (V_j^T v)),
//     T[0:j,j] = -tau T_j (V_j^T v).  Y, V, T stay in shared memory.
//   trailing update (batched DMMA GEMMs, all SMs):
//       A[:, c0+nb:]     -= Y V2^T                         (right)
//       A[c0+1:, c0+nb:] -= (V T^T) (V^T A[c0+1:, c0+nb:])  (left)
//   Q formation (dorghr order, backward over panels, trailing blocks only):
//       Q[c0+1:, c0+1:] -= (V T) (V^T Q[c0+1:, c0+1:])
//
// The reflectors V (unit leading entry, explicit zeros) and V T of every panel
// are kept in two d x d work matrices so Q is formed after the reduction and
// Z never enters the L2 working set of the panel matvecs.
#include "kernels.cuh"

namespace vrte {
namespace {

constexpr int HNT = 1024;

__device__ inline double block_sum_h(double v, double* red) { return block_sum(v, red); }

// Shared memory: Ys[d*nb] Vs[d*nb] Ts[nb*nb] col[d] part[max(HNT,d)] wv[nb] wt[nb] red[32]
__global__ void __launch_bounds__(HNT) hess_panel_kernel(double* Aall, double* Vall, double* VTall,
                                                         double* Yall, double* VTtall, int d, int c0,
                                                         int nb, int nbmax) {
    extern __shared__ double sm[];
    double* Ys = sm;
    double* Vs = Ys + (size_t)d * nb;
    double* Ts = Vs + (size_t)d * nb;
    double* col = Ts + nb * nb;
    double* part = col + d;
    double* wv = part + max(HNT, d);
    double* wt = wv + nb;
    double* red = wt + nb;
    const size_t dd = (size_t)d * d;
    double* A = Aall + blockIdx.x * dd;
    double* Vg = Vall + blockIdx.x * dd;
    double* VTg = VTall + blockIdx.x * dd;
    double* Yg = Yall + (size_t)blockIdx.x * d * nbmax;
    double* VTtg = VTtall + (size_t)blockIdx.x * d * nbmax;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nwarp = HNT / 32;
    // matvec decomposition: nsplit column slices per row when d < HNT
    const int nsplit = d < HNT ? HNT / d : 1;

    for (int e = t; e < nb * nb; e += HNT) Ts[e] = 0.0;
    for (int j = 0; j < nb; ++j) {
        const int k = c0 + j;
        // 1. column k with the panel's deferred right transformations
        for (int r = t; r < d; r += HNT) {
            double c = A[r + (size_t)k * d];
            for (int i = 0; i < j; ++i) c = fma(-Ys[r + (size_t)i * d], Vs[k + (size_t)i * d], c);
            col[r] = c;
        }
        __syncthreads();
        // 2. ... and the deferred left transformations (I - V T^T V^T) on rows c0+1..
        if (j > 0) {
            for (int i = warp; i < j; i += nwarp) {
                const double* vi = Vs + (size_t)i * d;
                double s = 0.0;
                for (int r = c0 + 1 + lane; r < d; r += 32) s = fma(vi[r], col[r], s);
                s = warp_sum(s);
                if (lane == 0) wv[i] = s;
            }
            __syncthreads();
            if (t < j) {
                double s = 0.0;
                for (int q = 0; q <= t; ++q) s = fma(Ts[q + t * nb], wv[q], s);
                wt[t] = s;
            }
            __syncthreads();
            for (int r = c0 + 1 + t; r < d; r += HNT) {
                double c = col[r];
                for (int i = 0; i < j; ++i) c = fma(-Vs[r + (size_t)i * d], wt[i], c);
                col[r] = c;
            }
            __syncthreads();
        }
        // 3. reflector (dlarfg) for col[k+1:]
        double ss = 0.0;
        for (int r = k + 2 + t; r < d; r += HNT) ss = fma(col[r], col[r], ss);
        ss = block_sum_h(ss, red);
        // the reflector's scalars only in the threads that use them (rows < d,
        // and the T column's t < j): 32 warps of redundant FP64 division /
        // square-root sequences would queue on the SM's FP64 pipe
        double tau = 0.0, beta = 0.0, scal = 0.0;
        if (t < d) {
            const double alpha = col[k + 1];
            const double xnorm = sqrt(ss);
            beta = alpha;
            if (xnorm != 0.0) {
                beta = -copysign(hypot(alpha, xnorm), alpha);
                tau = (beta - alpha) / beta;
                scal = 1.0 / (alpha - beta);
            }
        }
        double* vj = Vs + (size_t)j * d;
        for (int r = t; r < d; r += HNT) {
            double v, a;
            if (r <= k) {
                v = 0.0;
                a = col[r];
            } else if (r == k + 1) {
                v = 1.0;
                a = beta;
            } else {
                v = col[r] * scal;
                a = 0.0;
            }
            vj[r] = v;
            Vg[r + (size_t)k * d] = v;
            A[r + (size_t)k * d] = a;  // final Hessenberg column k
        }
        __syncthreads();
        // 4. y = A[:, k+1:] v[k+1:] over the start-of-panel matrix: nsplit column
        //    slices per row, 8 independent accumulators (8 loads in flight per thread)
        {
            const int cb = k + 1, ncols = d - cb;
            for (int rr = t; rr < d * nsplit; rr += HNT) {
                const int r = rr % d, s = rr / d;
                const int per = (ncols + nsplit - 1) / nsplit;
                const int ca = cb + s * per, ce = min(d, ca + per);
                double a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                const double* ap = A + r;
                int c = ca;
                for (; c + 15 < ce; c += 16) {  // 16 loads in flight per thread
                    double x[16];
#pragma unroll
                    for (int q = 0; q < 16; ++q) x[q] = ap[(size_t)(c + q) * d];
#pragma unroll
                    for (int q = 0; q < 16; ++q) a[q & 7] = fma(x[q], vj[c + q], a[q & 7]);
                }
                for (; c + 7 < ce; c += 8) {
#pragma unroll
                    for (int q = 0; q < 8; ++q) a[q] = fma(ap[(size_t)(c + q) * d], vj[c + q], a[q]);
                }
                for (; c < ce; ++c) a[0] = fma(ap[(size_t)c * d], vj[c], a[0]);
                part[s * d + r] = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
            }
        }
        // 5. u = V_j^T v (rows k+1..), T column, Y column
        for (int i = warp; i < j; i += nwarp) {
            const double* vi = Vs + (size_t)i * d;
            double s = 0.0;
            for (int r = k + 1 + lane; r < d; r += 32) s = fma(vi[r], vj[r], s);
            s = warp_sum(s);
            if (lane == 0) wv[i] = s;
        }
        __syncthreads();
        if (t < j) {
            double s = 0.0;
            for (int q = t; q < j; ++q) s = fma(Ts[t + q * nb], wv[q], s);
            wt[t] = -tau * s;
        }
        for (int r = t; r < d; r += HNT) {
            double y = part[r];
            for (int s = 1; s < nsplit; ++s) y += part[s * d + r];
            for (int i = 0; i < j; ++i) y = fma(-Ys[r + (size_t)i * d], wv[i], y);
            Ys[r + (size_t)j * d] = tau * y;
        }
        __syncthreads();
        if (t < j) Ts[t + j * nb] = wt[t];
        if (t == 0) Ts[j + j * nb] = tau;
        __syncthreads();
    }
    // Y, V T^T (left update) and V T (Q formation) to global
    for (int e = t; e < d * nb; e += HNT) {
        const int r = e % d, i = e / d;
        Yg[e] = Ys[e];
        double vt = 0.0, vtt = 0.0;
        for (int q = 0; q <= i; ++q) vt = fma(Vs[r + (size_t)q * d], Ts[q + i * nb], vt);
        for (int q = i; q < nb; ++q) vtt = fma(Vs[r + (size_t)q * d], Ts[i + q * nb], vtt);
        VTg[r + (size_t)(c0 + i) * d] = vt;
        VTtg[e] = vtt;
    }
}

__global__ void set_identity_kernel(double* Z, int d, long long total) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long w = e % ((long long)d * d);
        Z[e] = (w % d == w / d) ? 1.0 : 0.0;
    }
}

GemmBatch mk(int m, int n, int k, const double* a, long long lda, long long sa, bool ta,
             const double* b, long long ldb, long long sb, bool tb, double* c, long long ldc,
             long long sc, int batch, double alpha, double beta) {
    GemmBatch g{};
    g.m = m;
    g.n = n;
    g.k = k;
    g.a = a;
    g.lda = lda;
    g.stride_a = sa;
    g.trans_a = ta;
    g.b = b;
    g.ldb = ldb;
    g.stride_b = sb;
    g.trans_b = tb;
    g.c = c;
    g.ldc = ldc;
    g.stride_c = sc;
    g.batch = batch;
    g.alpha = alpha;
    g.beta = beta;
    return g;
}

}  // namespace

int hessenberg_panel_width(int d) {
    int nb = 8192 / (d > 0 ? d : 1);
    if (nb > 32) nb = 32;
    if (nb < 4) nb = 4;
    return nb;
}

size_t hessenberg_work_doubles(int d) {
    const int nb = hessenberg_panel_width(d);
    return 2 * (size_t)d * d + 3 * (size_t)d * nb;  // V, VT, Y, V T^T, W
}

void launch_hessenberg_reduce(double* A, double* work, int d, int batch, cudaStream_t st) {
    const int nbmax = hessenberg_panel_width(d);
    const long long dd = (long long)d * d, dn = (long long)d * nbmax;
    double* V = work;
    double* VT = V + dd * batch;
    double* Y = VT + dd * batch;
    double* VTt = Y + dn * batch;
    double* W = VTt + dn * batch;  // nbmax x d per matrix
    const size_t smem =
        (2 * (size_t)d * nbmax + nbmax * nbmax + d + (d > HNT ? d : HNT) + 2 * nbmax + 32) *
        sizeof(double);
    static unsigned long long attr = 0;
    smem_attr_once(hess_panel_kernel, 220 * 1024, attr);
    // (the panel kernel writes every row of each V / VT column it owns, zeros
    // included, so the Q-formation GEMMs need no cleared buffers)
    int npanel = 0;
    for (int c0 = 0; c0 < d - 2; c0 += nbmax) {
        const int nb = (d - 2 - c0) < nbmax ? (d - 2 - c0) : nbmax;
        hess_panel_kernel<<<batch, HNT, smem, st>>>(A, V, VT, Y, VTt, d, c0, nb, nbmax);
        VRTE_CUDA_CHECK(cudaGetLastError());
        ++npanel;
        const int n2 = d - c0 - nb;
        if (n2 <= 0) continue;
        double* Ar = A + (long long)(c0 + nb) * d;  // columns c0+nb..
        // right: A[:, c0+nb:] -= Y V[c0+nb:, panel]^T
        gemm_batched(mk(d, n2, nb, Y, d, dn, false, V + (c0 + nb) + (long long)c0 * d, d, dd, true, Ar,
                        d, dd, batch, -1.0, 1.0),
                     st);
        // left: W = V[c0+1:, panel]^T A[c0+1:, c0+nb:];  A[c0+1:, c0+nb:] -= (V T^T) W
        gemm_batched(mk(nb, n2, d - c0 - 1, V + (c0 + 1) + (long long)c0 * d, d, dd, true,
                        Ar + (c0 + 1), d, dd, false, W, nbmax, dn, batch, 1.0, 0.0),
                     st);
        gemm_batched(mk(d - c0 - 1, n2, nb, VTt + (c0 + 1), d, dn, false, W, nbmax, dn, false,
                        Ar + (c0 + 1), d, dd, batch, -1.0, 1.0),
                     st);
    }
}

// Q = Q_0 Q_1 ... Q_{P-1} of a finished reduction (its reflectors in `work`),
// accumulated backward on the trailing blocks.  Independent of the reduced
// matrix: the BRDF pipeline forms it on the side stream under the Francis QR.
void launch_hessenberg_formq(double* Z, double* work, int d, int batch, cudaStream_t st) {
    const int nbmax = hessenberg_panel_width(d);
    const long long dd = (long long)d * d, dn = (long long)d * nbmax;
    double* V = work;
    double* VT = V + dd * batch;
    double* Y = VT + dd * batch;
    double* VTt = Y + dn * batch;
    double* W = VTt + dn * batch;  // nbmax x d per matrix
    int npanel = 0;
    for (int c0 = 0; c0 < d - 2; c0 += nbmax) ++npanel;
    {
        const long long total = dd * batch;
        set_identity_kernel<<<(unsigned)((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096), 256, 0,
                              st>>>(Z, d, total);
        VRTE_CUDA_CHECK(cudaGetLastError());
    }
    for (int p = npanel - 1; p >= 0; --p) {
        const int c0 = p * nbmax;
        const int nb = (d - 2 - c0) < nbmax ? (d - 2 - c0) : nbmax;
        const int mq = d - c0 - 1;
        double* Qs = Z + (c0 + 1) + (long long)(c0 + 1) * d;
        gemm_batched(mk(nb, mq, mq, V + (c0 + 1) + (long long)c0 * d, d, dd, true, Qs, d, dd, false, W,
                        nbmax, dn, batch, 1.0, 0.0),
                     st);
        gemm_batched(mk(mq, mq, nb, VT + (c0 + 1) + (long long)c0 * d, d, dd, false, W, nbmax, dn,
                        false, Qs, d, dd, batch, -1.0, 1.0),
                     st);
    }
}

void launch_hessenberg_blocked(double* A, double* Z, double* work, int d, int batch, cudaStream_t st) {
    launch_hessenberg_reduce(A, work, d, batch, st);
    launch_hessenberg_formq(Z, work, d, batch, st);
}

int hessenberg_launch_count(int d) {
    const int nbmax = hessenberg_panel_width(d);
    int panels = 0;
    for (int c0 = 0; c0 < d - 2; c0 += nbmax) ++panels;
    return 1 + 4 * panels + 1 + 2 * panels;  // memset not counted as a kernel
}

}  // namespace vrte
