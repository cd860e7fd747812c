// lu.cu -- batched LU with partial pivoting on ROW-major matrices (dgetrf /
// dgetrs organisation), for the boundary systems of boundary.cpp:219-257 (one
// per Fourier order, every (incident, Stokes channel) a right-hand side) and
// for V^-1 of the eigenvector matrices (eig.cu).
//
// Row-major storage makes every row interchange a contiguous copy.  The
// factorization is blocked twice:
//   outer blocks of 64 columns: row interchanges of the whole block applied to
//     the other columns (staged in shared memory, one round trip), U12 by a
//     warp-parallel unit-lower triangular solve, and the trailing update as a
//     DMMA GEMM with k = 64;
//   inner panels of 16 (8, 4 for taller matrices) columns: register-resident
//     panel factorization (one row per thread, block-wide argmax pivoting with
//     LAPACK's first-index tie break), then the same swap / TRSM / GEMM steps
//     restricted to the outer block.
// The solve gathers the right-hand sides through the net row permutation,
// then runs blocked forward / backward substitution (TRSM on 64-row blocks +
// GEMM updates).
#include <cstdlib>
#include <stdexcept>

#include "boundary.cuh"

namespace vrte {
namespace {

constexpr int LU_NB = 64;  // outer block
constexpr int SW_TILE = 32;

// ------------------------------------------------------------------ panel
template <int NT, int RPT, int PB>
__global__ void __launch_bounds__(NT) lu_panel_rm_kernel(double* Aall, int G, long long strideA, int k0,
                                                         int jb, int rend, int* ipiv_all, DeviceStatus* status,
                                                         const int* order_index) {
    __shared__ double s_val[NT / 32];
    __shared__ int s_idx[NT / 32];
    __shared__ double prow[PB];
    __shared__ double srow[PB];
    __shared__ int s_piv;
    const int b = blockIdx.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
    double* A = Aall + (size_t)b * strideA;
    int* ipiv = ipiv_all + (size_t)b * G;
    const int np = rend - k0;  // rows past the profile end are zero in these columns
    double v[RPT][PB];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        const int r = t + i * NT;
        const double* src = A + (size_t)(k0 + r) * G + k0;
#pragma unroll
        for (int c = 0; c < PB; ++c) v[i][c] = (r < np && c < jb) ? src[c] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < PB; ++j) {
        if (j >= jb) break;
        // argmax |v[r][j]| over rows r >= j (first index on ties)
        double best = -1.0;
        int bi = 0x7fffffff;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const int r = t + i * NT;
            if (r >= j && r < np) {
                const double a = fabs(v[i][j]);
                if (a > best) {
                    best = a;
                    bi = r;
                }
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
        if (lane == 0) {
            s_val[w] = best;
            s_idx[w] = bi;
        }
        __syncthreads();
        if (w == 0) {
            best = lane < NT / 32 ? s_val[lane] : -1.0;
            bi = lane < NT / 32 ? s_idx[lane] : 0x7fffffff;
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, best, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ov > best || (ov == best && oi < bi)) {
                    best = ov;
                    bi = oi;
                }
            }
            if (lane == 0) {
                s_piv = bi;
                ipiv[k0 + j] = k0 + bi;
                if (!(best > 0.0))
                    report_failure(status, kFailLuSingular, 3, order_index ? order_index[b] : b,
                                   (double)(k0 + j));
            }
        }
        __syncthreads();
        const int pr = s_piv;
        // exchange rows j and pr through shared memory
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const int r = t + i * NT;
            if (r == pr) {
#pragma unroll
                for (int c = 0; c < PB; ++c) prow[c] = v[i][c];
            }
            if (r == j && pr != j) {
#pragma unroll
                for (int c = 0; c < PB; ++c) srow[c] = v[i][c];
            }
        }
        __syncthreads();
        const double piv = prow[j];
        const double rcp = piv != 0.0 ? 1.0 / piv : 0.0;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const int r = t + i * NT;
            if (pr != j) {
                if (r == j) {
#pragma unroll
                    for (int c = 0; c < PB; ++c) v[i][c] = prow[c];
                } else if (r == pr) {
#pragma unroll
                    for (int c = 0; c < PB; ++c) v[i][c] = srow[c];
                }
            }
            if (r > j && r < np && piv != 0.0) {
                const double l = v[i][j] * rcp;
                v[i][j] = l;
#pragma unroll
                for (int c = j + 1; c < PB; ++c) v[i][c] = fma(-l, prow[c], v[i][c]);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        const int r = t + i * NT;
        if (r < np) {
            double* dst = A + (size_t)(k0 + r) * G + k0;
#pragma unroll
            for (int c = 0; c < PB; ++c)
                if (c < jb) dst[c] = v[i][c];
        }
    }
}

// ------------------------------------------------------------------ row interchanges
// Pivots ipiv[k0 .. k0+npiv) (absolute rows, applied in order) on the columns
// [c_lo, c_hi) \ [s_lo, s_hi) of M (row-major, ld).  The npiv "top" rows and the
// distinct far rows of a 32-column tile are staged in shared memory, permuted
// there, and written back: one global round trip per tile.
__global__ void __launch_bounds__(256) lu_swap_rm_kernel(double* Mall, int ld, long long strideM,
                                                         const int* ipiv_all, int G, int k0, int npiv,
                                                         int c_lo, int c_hi, int s_lo, int s_hi) {
    __shared__ double top[LU_NB][SW_TILE + 1];
    __shared__ double far[LU_NB][SW_TILE + 1];
    __shared__ int prs[LU_NB];
    __shared__ int slot[LU_NB];
    const int b = blockIdx.y, t = threadIdx.x;
    const int col0 = c_lo + blockIdx.x * SW_TILE;
    if (col0 >= c_hi) return;
    if (col0 >= s_lo && col0 + SW_TILE <= s_hi) return;  // tile entirely inside the skipped panel
    double* M = Mall + (size_t)b * strideM;
    const int* ipiv = ipiv_all + (size_t)b * G;
    if (t < npiv) prs[t] = ipiv[k0 + t];
    __syncthreads();
    if (t < 32) {
        for (int j = t; j < npiv; j += 32) {
            const int pr = prs[j];
            int s = -1;
            if (pr >= k0 + npiv) {
                s = j;
                for (int q = 0; q < j; ++q)
                    if (prs[q] == pr) {
                        s = q;
                        break;
                    }
            }
            slot[j] = s;
        }
    }
    __syncthreads();
    const int c = t & 31;
    const int col = col0 + c;
    const bool live = col < c_hi && !(col >= s_lo && col < s_hi);
    for (int r = t >> 5; r < npiv; r += 8) {
        if (live) {
            top[r][c] = M[(size_t)(k0 + r) * ld + col];
            if (slot[r] == r) far[r][c] = M[(size_t)prs[r] * ld + col];
        }
    }
    __syncthreads();
    if (t < 32 && live) {
        for (int j = 0; j < npiv; ++j) {
            const int pr = prs[j];
            if (pr == k0 + j) continue;
            double* y = (pr < k0 + npiv) ? &top[pr - k0][c] : &far[slot[j]][c];
            const double tmp = top[j][c];
            top[j][c] = *y;
            *y = tmp;
        }
    }
    __syncthreads();
    for (int r = t >> 5; r < npiv; r += 8) {
        if (live) {
            M[(size_t)(k0 + r) * ld + col] = top[r][c];
            if (slot[r] == r) M[(size_t)prs[r] * ld + col] = far[r][c];
        }
    }
}

// ------------------------------------------------------------------ triangular block solves
// M[k0:k0+jb, c_lo:c_hi] <- T^-1 M[...] with T = A[k0:k0+jb, k0:k0+jb] (row-major
// ld G): unit lower (LOWER) or upper.  CTA per 32-column tile; warp per 4
// columns, lanes over rows (two rows per lane), the solved entry broadcast by
// shuffle -- substitution, not an explicit inverse.
template <bool LOWER>
__global__ void __launch_bounds__(256) lu_trsm_rm_kernel(const double* Aall, int G, long long strideA,
                                                         double* Mall, int ld, long long strideM, int k0,
                                                         int jb, int c_lo, int c_hi) {
    __shared__ double Ts[LU_NB][LU_NB + 1];
    const int b = blockIdx.y, t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int col0 = c_lo + blockIdx.x * SW_TILE;
    if (col0 >= c_hi) return;
    const double* A = Aall + (size_t)b * strideA;
    double* M = Mall + (size_t)b * strideM;
    for (int e = t; e < jb * jb; e += 256) {
        const int r = e / jb, cc = e % jb;
        Ts[r][cc] = A[(size_t)(k0 + r) * G + k0 + cc];
    }
    __syncthreads();
    // lane rows r0, r1; the warp's 4 consecutive columns (one 32-byte sector per row)
    const int r0 = lane, r1 = lane + 32, cw = col0 + w * 4;
    double x0[4], x1[4];
    bool lv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        lv[q] = cw + q < c_hi;
        x0[q] = (r0 < jb && lv[q]) ? M[(size_t)(k0 + r0) * ld + cw + q] : 0.0;
        x1[q] = (r1 < jb && lv[q]) ? M[(size_t)(k0 + r1) * ld + cw + q] : 0.0;
    }
    if (LOWER) {
        for (int j = 0; j < jb; ++j) {
            const int src = j & 31;
            const double l0 = (r0 > j && r0 < jb) ? Ts[r0][j] : 0.0;
            const double l1 = (r1 > j && r1 < jb) ? Ts[r1][j] : 0.0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double xj = __shfl_sync(0xffffffffu, j < 32 ? x0[q] : x1[q], src);
                x0[q] = fma(-l0, xj, x0[q]);
                x1[q] = fma(-l1, xj, x1[q]);
            }
        }
    } else {
        for (int j = jb - 1; j >= 0; --j) {
            const int src = j & 31;
            const double rd = 1.0 / Ts[j][j];
            const double u0 = (r0 < j) ? Ts[r0][j] : 0.0;
            const double u1 = (r1 < j) ? Ts[r1][j] : 0.0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double xj = __shfl_sync(0xffffffffu, j < 32 ? x0[q] : x1[q], src) * rd;
                if (r0 == j) x0[q] = xj;
                if (r1 == j) x1[q] = xj;
                x0[q] = fma(-u0, xj, x0[q]);
                x1[q] = fma(-u1, xj, x1[q]);
            }
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (r0 < jb && lv[q]) M[(size_t)(k0 + r0) * ld + cw + q] = x0[q];
        if (r1 < jb && lv[q]) M[(size_t)(k0 + r1) * ld + cw + q] = x1[q];
    }
}

// Net row permutation of the pivot sequence: out row i <- in row perm[i].
__global__ void lu_perm_kernel(const int* ipiv_all, int* perm_all, int G) {
    extern __shared__ int pm[];
    const int b = blockIdx.x;
    const int* ipiv = ipiv_all + (size_t)b * G;
    for (int i = threadIdx.x; i < G; i += blockDim.x) pm[i] = i;
    __syncthreads();
    if (threadIdx.x == 0)
        for (int j = 0; j < G; ++j) {
            const int p = ipiv[j];
            if (p != j) {
                const int tmp = pm[j];
                pm[j] = pm[p];
                pm[p] = tmp;
            }
        }
    __syncthreads();
    for (int i = threadIdx.x; i < G; i += blockDim.x) perm_all[(size_t)b * G + i] = pm[i];
}

__global__ void lu_gather_rows_kernel(const double* In, long long strideIn, double* Out,
                                      long long strideOut, const int* perm_all, int G, int ncol,
                                      int batch) {
    const long long total = (long long)batch * G * ncol;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(e % ncol);
        const long long rb = e / ncol;
        const int r = (int)(rb % G), b = (int)(rb / G);
        Out[(size_t)b * strideOut + (size_t)r * ncol + c] =
            In[(size_t)b * strideIn + (size_t)perm_all[(size_t)b * G + r] * ncol + c];
    }
}

// C (m x n) = alpha A (m x k) B (k x n) + beta C, all row-major: the col-major
// GEMM on the transposed views, C^T = B^T A^T.
void rm_gemm(int m, int n, int k, const double* A, long long lda, long long sa, const double* B,
             long long ldb, long long sb, double* C, long long ldc, long long sc, int batch,
             double alpha, double beta, cudaStream_t st) {
    GemmBatch g{};
    g.m = n;
    g.n = m;
    g.k = k;
    g.a = B;
    g.lda = ldb;
    g.stride_a = sb;
    g.trans_a = false;
    g.b = A;
    g.ldb = lda;
    g.stride_b = sa;
    g.trans_b = false;
    g.c = C;
    g.ldc = ldc;
    g.stride_c = sc;
    g.batch = batch;
    g.alpha = alpha;
    g.beta = beta;
    gemm_batched(g, st);
}

template <int NT, int RPT, int PB>
void panel_launch(double* A, int G, int k0, int jb, int rend, int* ipiv, DeviceStatus* status,
                  const int* order_index, int batch, cudaStream_t st) {
    lu_panel_rm_kernel<NT, RPT, PB><<<batch, NT, 0, st>>>(A, G, (long long)G * G, k0, jb, rend, ipiv, status,
                                                          order_index);
}

int panel_width(int G) { return G <= 1024 ? 16 : (G <= 2048 ? 8 : 4); }

void swap_launch(double* M, int ld, long long strideM, const int* ipiv, int G, int k0, int npiv,
                 int c_lo, int c_hi, int s_lo, int s_hi, int batch, cudaStream_t st) {
    if (npiv <= 0 || c_hi <= c_lo) return;
    dim3 grid((c_hi - c_lo + SW_TILE - 1) / SW_TILE, batch);
    lu_swap_rm_kernel<<<grid, 256, 0, st>>>(M, ld, strideM, ipiv, G, k0, npiv, c_lo, c_hi, s_lo, s_hi);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

template <bool LOWER>
void trsm_launch(const double* A, int G, double* M, int ld, long long strideM, int k0, int jb, int c_lo,
                 int c_hi, int batch, cudaStream_t st) {
    if (jb <= 0 || c_hi <= c_lo) return;
    dim3 grid((c_hi - c_lo + SW_TILE - 1) / SW_TILE, batch);
    lu_trsm_rm_kernel<LOWER><<<grid, 256, 0, st>>>(A, G, (long long)G * G, M, ld, strideM, k0, jb, c_lo,
                                                   c_hi);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace

void lu_factor_rm(double* A, int G, int batch, int* ipiv, int* perm, DeviceStatus* status,
                  const int* order_index, cudaStream_t st, int prof_d, int prof_P) {
    if (G > 4096) throw std::invalid_argument("vrte_cuda: boundary system larger than 4096 rows");
    const int PB = panel_width(G);
    // outer block: 128 columns (trailing GEMMs with k = 128), handled by the
    // 64-row swap / TRSM kernels in two halves; VRTE_LU_NB=64 for A/B runs
    static const int OB = std::getenv("VRTE_LU_NB") ? std::atoi(std::getenv("VRTE_LU_NB")) : 128;
    const long long gg = (long long)G * G;
    auto row_end = [&](int col) { return prof_d > 0 ? min(G, bnd_row_end(col, prof_d, prof_P)) : G; };
    for (int K0 = 0; K0 < G; K0 += OB) {
        const int NBk = min(OB, G - K0);
        const int rend = row_end(K0 + NBk - 1);  // profile is non-decreasing in the column
        for (int k0 = K0; k0 < K0 + NBk; k0 += PB) {
            const int jb = min(PB, K0 + NBk - k0);
            const int np = rend - k0;
            if (np <= 256)
                panel_launch<256, 1, 16>(A, G, k0, jb, rend, ipiv, status, order_index, batch, st);
            else if (np <= 512)
                panel_launch<512, 1, 16>(A, G, k0, jb, rend, ipiv, status, order_index, batch, st);
            else if (np <= 1024)
                panel_launch<1024, 1, 16>(A, G, k0, jb, rend, ipiv, status, order_index, batch, st);
            else if (np <= 2048)
                panel_launch<512, 4, 8>(A, G, k0, jb, rend, ipiv, status, order_index, batch, st);
            else
                panel_launch<512, 8, 4>(A, G, k0, jb, rend, ipiv, status, order_index, batch, st);
            VRTE_CUDA_CHECK(cudaGetLastError());
            const int c_end = K0 + NBk, rest_in = c_end - (k0 + jb);
            swap_launch(A, G, gg, ipiv, G, k0, jb, K0, c_end, k0, k0 + jb, batch, st);
            if (rest_in > 0) {
                trsm_launch<true>(A, G, A, G, gg, k0, jb, k0 + jb, c_end, batch, st);
                if (rend - k0 - jb > 0)
                    rm_gemm(rend - k0 - jb, rest_in, jb, A + (size_t)(k0 + jb) * G + k0, G, gg,
                            A + (size_t)k0 * G + k0 + jb, G, gg, A + (size_t)(k0 + jb) * G + k0 + jb, G, gg,
                            batch, -1.0, 1.0, st);
            }
        }
        // the block's interchanges on the other columns, in chunks of <= 64 pivots
        for (int p0 = K0; p0 < K0 + NBk; p0 += LU_NB)
            swap_launch(A, G, gg, ipiv, G, p0, min(LU_NB, K0 + NBk - p0), 0, G, K0, K0 + NBk, batch, st);
        const int rest = G - K0 - NBk;
        if (rest > 0) {
            // U12 = L11^-1 A12, blocked by 64 rows
            for (int r0 = K0; r0 < K0 + NBk; r0 += LU_NB) {
                const int rb = min(LU_NB, K0 + NBk - r0);
                trsm_launch<true>(A, G, A, G, gg, r0, rb, K0 + NBk, G, batch, st);
                const int below = K0 + NBk - (r0 + rb);
                if (below > 0)
                    rm_gemm(below, rest, rb, A + (size_t)(r0 + rb) * G + r0, G, gg, A + (size_t)r0 * G + K0 + NBk,
                            G, gg, A + (size_t)(r0 + rb) * G + K0 + NBk, G, gg, batch, -1.0, 1.0, st);
            }
            // trailing update: rows past the profile have zero multipliers
            if (rend - K0 - NBk > 0)
                rm_gemm(rend - K0 - NBk, rest, NBk, A + (size_t)(K0 + NBk) * G + K0, G, gg,
                        A + (size_t)K0 * G + K0 + NBk, G, gg, A + (size_t)(K0 + NBk) * G + K0 + NBk, G, gg,
                        batch, -1.0, 1.0, st);
        }
    }
    lu_perm_kernel<<<batch, 256, G * sizeof(int), st>>>(ipiv, perm, G);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

void lu_solve_rm(const double* A, int G, int batch, const int* perm, const double* Bin, double* X,
                 int ncol, cudaStream_t st, int row_lo, int prof_d, int prof_P) {
    const long long gg = (long long)G * G, gn = (long long)G * ncol;
    {
        const long long total = (long long)batch * gn;
        const long long blocks = (total + 255) / 256;
        lu_gather_rows_kernel<<<(unsigned)(blocks < 16384 ? blocks : 16384), 256, 0, st>>>(
            Bin, gn, X, gn, perm, G, ncol, batch);
        VRTE_CUDA_CHECK(cudaGetLastError());
    }
    for (int k0 = 0; k0 < G; k0 += LU_NB) {
        const int jb = min(LU_NB, G - k0);
        // (no profile here: later row interchanges move multipliers below the
        // staircase profile of earlier columns, so L itself is dense)
        (void)prof_d;
        (void)prof_P;
        trsm_launch<true>(A, G, X, ncol, gn, k0, jb, 0, ncol, batch, st);
        if (G - k0 - jb > 0)
            rm_gemm(G - k0 - jb, ncol, jb, A + (size_t)(k0 + jb) * G + k0, G, gg, X + (size_t)k0 * ncol,
                    ncol, gn, X + (size_t)(k0 + jb) * ncol, ncol, gn, batch, -1.0, 1.0, st);
    }
    // back substitution only down to row_lo: the unknowns above it are not
    // wanted (X rows < row_lo are left holding the forward solution)
    const int nblk = (G + LU_NB - 1) / LU_NB;
    const int blo = max(0, row_lo) / LU_NB, rl = blo * LU_NB;
    for (int bk = nblk - 1; bk >= blo; --bk) {
        const int k0 = bk * LU_NB, jb = min(LU_NB, G - k0);
        trsm_launch<false>(A, G, X, ncol, gn, k0, jb, 0, ncol, batch, st);
        if (k0 > rl)
            rm_gemm(k0 - rl, ncol, jb, A + (size_t)rl * G + k0, G, gg, X + (size_t)k0 * ncol, ncol, gn,
                    X + (size_t)rl * ncol, ncol, gn, batch, -1.0, 1.0, st);
    }
}

int lu_rm_launch_count(int G) {
    const int PB = panel_width(G);
    static const int OB = std::getenv("VRTE_LU_NB") ? std::atoi(std::getenv("VRTE_LU_NB")) : 128;
    int n = 0;
    for (int K0 = 0; K0 < G; K0 += OB) {
        const int NBk = min(OB, G - K0);
        for (int k0 = K0; k0 < K0 + NBk; k0 += PB) {
            const int jb = min(PB, K0 + NBk - k0);
            n += 2;  // panel + swap
            if (K0 + NBk - (k0 + jb) > 0) n += 1 + (G - k0 - jb > 0 ? 1 : 0);
        }
        n += (NBk + LU_NB - 1) / LU_NB;
        if (G - K0 - NBk > 0) n += 2 * ((NBk + LU_NB - 1) / LU_NB) - 1 + 1;
    }
    n += 1;                                          // perm
    const int nblk = (G + LU_NB - 1) / LU_NB;
    n += 1 + 2 * nblk - 1 + 2 * nblk - 1;            // gather + forward + backward (upper bound)
    return n;
}

}  // namespace vrte
