// lu.cu -- batched LU with partial pivoting on ROW-major matrices (dgetrf /
// dgetrs organisation), for the boundary systems of boundary.cpp:219-257 (one
// per Fourier order, every (incident, Stokes channel) a right-hand side) and
// for V^-1 of the eigenvector matrices (eig.cu).
//
// Lazy pivoting: rows are never moved.  A per-matrix row map (position ->
// physical row, returned as `perm`) is updated by the pivot search, and every
// later kernel addresses rows through it (the GEMMs through their index maps,
// common.cuh), so the row-interchange traffic of dlaswp -- a full HBM pass per
// pivot block -- disappears.  The factorization is blocked twice:
//   outer blocks of 128 columns, right-looking: U12 by the fused 128-row
//     block solve (lu_block_trsm_kernel) and the trailing update as one DMMA
//     GEMM with k = 128 over the rows inside the staircase profile; with a
//     one-block look-ahead on two streams for the boundary systems;
//   inner panels of 16 (8, 4 for taller matrices) columns, left-looking
//     (Crout) inside the outer block and fused into ONE kernel per panel: the
//     panel's U rows (unit-lower solve with the block's L, in shared memory),
//     the update of its column strip by the block's earlier panels (rows x 16 x
//     kk from registers), then register-resident factorization with
//     block-wide argmax pivoting (LAPACK's first-index tie break).
// The solve gathers the right-hand sides through the row map, then runs
// blocked forward / backward substitution (the fused solve on 128-row diagonal
// blocks + GEMM couplings), reading L and U rows through the map.
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "boundary.cuh"

namespace vrte {
namespace {

constexpr int LU_NB = 64;  // outer block

// ------------------------------------------------------------------ Crout panel (lazy pivoting)
constexpr int OB_MAX = 128;  // outer block width (bounds the panel kernel's shared memory)

// Panel [k0, k0+jb) of the outer block starting at K0 (kk = k0 - K0 earlier
// panel columns), positions [k0, rend) active, rows addressed through map.
// Shared memory: Us [KKMAX][PB] | (Ls [KKMAX][LDL] during the U solve, then
// Ps [NT*RPT][PSL], the updated strip, one padded row per position).
__device__ inline void cp_async8(double* smem, const double* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ inline void cp_async_wait_all() { asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::); }

template <int NT, int RPT, int PB>
struct PanelGeo {
    static constexpr int KKMAX = OB_MAX - PB, LDL = KKMAX + 1;
    static constexpr int PSL = PB + 2;  // 16-byte aligned rows, conflict-free LDS.128 per lane
    static constexpr int USL = PB <= 8 ? 8 : 24;  // 2*USL = 16 (mod 32): DMMA B-fragment reads 2 wavefronts
    static constexpr int US = KKMAX * USL;
    static constexpr int LS = KKMAX * LDL, PS = NT * RPT * PSL;
    static constexpr size_t bytes = (size_t)(US + (LS > PS ? LS : PS)) * sizeof(double);
};

template <int NT, int RPT, int PB>
__global__ void __launch_bounds__(NT) lu_panel_crout_kernel(double* Aall, int G, int lda, long long strideA, int* map_all,
                                                            int* ipiv_all, int K0, int k0, int jb, int rend,
                                                            DeviceStatus* status, const int* order_index) {
    using Geo = PanelGeo<NT, RPT, PB>;
    constexpr int KKMAX = Geo::KKMAX, LDL = Geo::LDL, PSL = Geo::PSL, USL = Geo::USL, KQ = (KKMAX + 3) / 4;
    constexpr int NTL = (PB + 7) / 8;  // 8-column DMMA tiles of the strip
    extern __shared__ double dsm[];
    double* Us = dsm;             // [kk][USL]: U rows of this panel's columns
    double* Ls = dsm + Geo::US;   // [kk][LDL]: strictly lower part of the block's L (positions K0..k0)
    double* Ps = dsm + Geo::US;   // [np][PSL]: the updated strip (after the U solve)
    __shared__ int s_map[NT * RPT];
    __shared__ int s_mapu[KKMAX];
    __shared__ unsigned s_kh[2][NT / 32], s_kl[2][NT / 32];
    __shared__ int s_kp[2][NT / 32];
    __shared__ __align__(16) double s_cand[2][NT / 32][PB];
    const int b = blockIdx.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int gq = lane >> 2, tq = lane & 3;
    constexpr int NW = NT / 32;
    double* A = Aall + (size_t)b * strideA;
    int* map = map_all + (size_t)b * G;
    int* ipiv = ipiv_all + (size_t)b * G;
    const int kk = k0 - K0, np = rend - k0;
#ifdef VRTE_LU_TRACE
    long long tr[6];
    tr[0] = clock64();
#define LU_STAMP(i) tr[i] = clock64()
#else
#define LU_STAMP(i)
#endif
    for (int r = t; r < np; r += NT) s_map[r] = map[k0 + r];
    for (int q = t; q < kk; q += NT) s_mapu[q] = map[K0 + q];
    __syncthreads();
    if (kk > 0) {
        // U(K0:k0, panel) = L11^-1 A(K0:k0, panel), L11 unit lower (the block's
        // earlier panels): async copies of L11 / the U rows, warp per column to solve
        for (int q = w; q < kk; q += NW) {
            const double* src = A + (size_t)s_mapu[q] * lda;
            for (int c = lane; c < q; c += 32) cp_async8(Ls + q * LDL + c, src + K0 + c);
            if (lane < jb) cp_async8(Us + q * USL + lane, src + k0 + lane);
            else if (lane < PB) Us[q * USL + lane] = 0.0;
        }
        cp_async_wait_all();
        __syncthreads();
        // blocked by the earlier panels (PB rows each): solve the PB x PB unit-lower
        // diagonal block (lane group of PB per column, shuffles within the group),
        // then update the rows below it from shared memory -- PB-step chains
        // instead of one kk-step shuffle chain per column
        constexpr int NG = NT / PB;
        const int grp = t / PB, gl = t % PB;
        for (int r0 = 0; r0 < kk; r0 += PB) {
            for (int cb = 0; cb < jb; cb += NG) {
                const int c = cb + grp;
                const bool act = c < jb;
                double x = act ? Us[(r0 + gl) * USL + c] : 0.0;
#pragma unroll
                for (int s2 = 0; s2 < PB - 1; ++s2) {
                    const double xs = __shfl_sync(0xffffffffu, x, s2, PB);
                    if (gl > s2) x = fma(-Ls[(r0 + gl) * LDL + r0 + s2], xs, x);
                }
                if (act) Us[(r0 + gl) * USL + c] = x;
            }
            __syncthreads();
            const int below = kk - r0 - PB;
            for (int e = t; e < below * jb; e += NT) {
                const int r = r0 + PB + e / jb, c = e - (e / jb) * jb;
                double acc = Us[r * USL + c];
#pragma unroll
                for (int s2 = 0; s2 < PB; ++s2) acc = fma(-Ls[r * LDL + r0 + s2], Us[(r0 + s2) * USL + c], acc);
                Us[r * USL + c] = acc;
            }
            __syncthreads();
        }
        for (int e = t; e < kk * jb; e += NT) {
            const int q = e / jb, c = e - q * jb;
            A[(size_t)s_mapu[q] * lda + k0 + c] = Us[q * USL + c];
        }
        __syncthreads();  // Ls is dead from here on (Ps aliases it)
    }
    LU_STAMP(1);
    // The panel strip, updated by the block's earlier panels, Ps = A - L(:, K0:k0) U,
    // on the FP64 tensor cores: warp per 8-row tile, the tile's whole L segment
    // (one 32-byte sector per row and k-step) requested before the first DMMA;
    // each fragment register is refilled with the next tile's value as soon as
    // its DMMA has issued, so the next tile's loads overlap this tile's math.
    {
        const int ntiles = (np + 7) / 8;
        auto row_of = [&](int tile) -> const double* {
            const int r = tile * 8 + gq;
            return (tile < ntiles && r < np) ? A + (size_t)s_map[r] * lda : nullptr;
        };
        double a[KQ];
        const double* row = row_of(w);
#pragma unroll
        for (int q = 0; q < KQ; ++q) a[q] = (row && 4 * q < kk) ? row[K0 + 4 * q + tq] : 0.0;
        for (int tile = w; tile < ntiles; tile += NW) {
            double c[NTL][2];
#pragma unroll
            for (int nt = 0; nt < NTL; ++nt) {
                const int cc = 8 * nt + 2 * tq;
                c[nt][0] = (row && cc < jb) ? row[k0 + cc] : 0.0;
                c[nt][1] = (row && cc + 1 < jb) ? row[k0 + cc + 1] : 0.0;
            }
            const double* nrow = row_of(tile + NW);
#pragma unroll
            for (int q = 0; q < KQ; ++q) {
                if (4 * q >= kk) break;
#pragma unroll
                for (int nt = 0; nt < NTL; ++nt) {
                    const int n = 8 * nt + gq;
                    const double bu = n < PB ? Us[(4 * q + tq) * USL + n] : 0.0;
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                                 : "+d"(c[nt][0]), "+d"(c[nt][1])
                                 : "d"(-a[q]), "d"(bu));
                }
                a[q] = nrow ? nrow[K0 + 4 * q + tq] : 0.0;
            }
            const int r = tile * 8 + gq;
            if (row) {
#pragma unroll
                for (int nt = 0; nt < NTL; ++nt) {
                    const int cc = 8 * nt + 2 * tq;
                    if (cc < PB) *reinterpret_cast<double2*>(Ps + r * PSL + cc) = make_double2(c[nt][0], c[nt][1]);
                }
            }
            row = nrow;
        }
    }
    __syncthreads();
    LU_STAMP(2);
    double v[RPT][PB];
    const double* src[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        const int r = t + i * NT;
        src[i] = r < np ? A + (size_t)s_map[r] * lda : nullptr;
#pragma unroll
        for (int c2 = 0; c2 < PB / 2; ++c2) {
            const double2 x = src[i] ? *reinterpret_cast<const double2*>(Ps + r * PSL + 2 * c2) : make_double2(0.0, 0.0);
            v[i][2 * c2] = x.x;
            v[i][2 * c2 + 1] = x.y;
        }
    }
    // Factor the strip.  Rows never move between threads: each row carries its
    // current position (LAPACK's interchange of positions j and pr is a swap of
    // two position labels).  One barrier per column: every warp publishes its
    // best candidate (key = |a| bits, then the smallest position) together with
    // the candidate's row, double buffered by column parity; after the barrier
    // every warp reduces the NW keys itself and reads the winner's row.
    int pos[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) pos[i] = src[i] ? t + i * NT : 0x7fffffff;
#pragma unroll
    for (int j = 0; j < PB; ++j) {
        if (j >= jb) break;
        const int buf = j & 1;
        // argmax |v| over positions >= j (first position on ties, idamax)
        unsigned long long kb = 0ull;
        int kp = 0x7fffffff;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const unsigned long long bits = (unsigned long long)__double_as_longlong(fabs(v[i][j]));
            if (pos[i] >= j && pos[i] != 0x7fffffff && (bits > kb || (bits == kb && pos[i] < kp))) {
                kb = bits;
                kp = pos[i];
            }
        }
        const unsigned hi = (unsigned)(kb >> 32), lo = (unsigned)kb;
        const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
        const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
        const int mp = __reduce_min_sync(0xffffffffu, (hi == mh && lo == ml) ? kp : 0x7fffffff);
        if (mp == 0x7fffffff) {
            if (lane == 0) {
                s_kh[buf][w] = 0u;
                s_kl[buf][w] = 0u;
                s_kp[buf][w] = 0x7fffffff;
            }
        } else {
#pragma unroll
            for (int i = 0; i < RPT; ++i)
                if (pos[i] == mp) {
                    s_kh[buf][w] = mh;
                    s_kl[buf][w] = ml;
                    s_kp[buf][w] = mp;
#pragma unroll
                    for (int c = j; c < PB; ++c) s_cand[buf][w][c] = v[i][c];
                }
        }
        __syncthreads();
        const unsigned h2 = lane < NW ? s_kh[buf][lane] : 0u;
        const unsigned l2 = lane < NW ? s_kl[buf][lane] : 0u;
        const int p2 = lane < NW ? s_kp[buf][lane] : 0x7fffffff;
        const unsigned gh = __reduce_max_sync(0xffffffffu, h2);
        const unsigned gl = __reduce_max_sync(0xffffffffu, h2 == gh ? l2 : 0u);
        const int pr = __reduce_min_sync(0xffffffffu, (h2 == gh && l2 == gl) ? p2 : 0x7fffffff);
        const int ww = __ffs(__ballot_sync(0xffffffffu, lane < NW && p2 == pr)) - 1;
        const double* prow = s_cand[buf][ww >= 0 ? ww : 0];
        if (t == 0) {
            ipiv[k0 + j] = ww >= 0 ? k0 + pr : k0 + j;
            if (!(gh != 0u || gl != 0u))
                report_failure(status, kFailLuSingular, 3, order_index ? order_index[b] : b, (double)(k0 + j));
        }
        const double piv = ww >= 0 ? prow[j] : 0.0;
        const double rcp = piv != 0.0 ? 1.0 / piv : 0.0;
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            if (pos[i] == pr)
                pos[i] = j;
            else if (pos[i] == j)
                pos[i] = pr;
            if (pos[i] > j && pos[i] != 0x7fffffff && piv != 0.0) {
                const double l = v[i][j] * rcp;
                v[i][j] = l;
#pragma unroll
                for (int c = j + 1; c < PB; ++c) v[i][c] = fma(-l, prow[c], v[i][c]);
            }
        }
    }
    LU_STAMP(3);
    // every row goes back to its own physical row (staged through Ps, then whole
    // rows per 16-byte lane group); the map records its position
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
        const int r = t + i * NT;
        if (src[i]) {
#pragma unroll
            for (int c2 = 0; c2 < PB / 2; ++c2)
                *reinterpret_cast<double2*>(Ps + r * PSL + 2 * c2) = make_double2(v[i][2 * c2], v[i][2 * c2 + 1]);
            map[k0 + pos[i]] = s_map[r];
        }
    }
    __syncthreads();
    if (jb == PB) {
        constexpr int LPR = PB / 2;  // lanes per row (16 bytes each)
        for (int e = t; e < np * LPR; e += NT) {
            const int r = e / LPR, c2 = e - r * LPR;
            *reinterpret_cast<double2*>(A + (size_t)s_map[r] * lda + k0 + 2 * c2) =
                *reinterpret_cast<const double2*>(Ps + r * PSL + 2 * c2);
        }
    } else {
        for (int e = t; e < np * jb; e += NT) {
            const int r = e / jb, c = e - r * jb;
            A[(size_t)s_map[r] * lda + k0 + c] = Ps[r * PSL + c];
        }
    }
#ifdef VRTE_LU_TRACE
    __syncthreads();
    LU_STAMP(4);
    if (t == 0 && b == 0)
        printf("panel NT=%d K0=%4d k0=%4d np=%4d kk=%3d | setup+U %6lld  strip %6lld  factor %6lld  store %6lld cycles\n", NT, K0,
               k0, np, kk, tr[1] - tr[0], tr[2] - tr[1], tr[3] - tr[2], tr[4] - tr[3]);
#endif
}

__global__ void lu_map_init_kernel(int* map, long long total, int G) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x)
        map[e] = (int)(e % G);
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
// GEMM on the transposed views, C^T = B^T A^T.  Optional row maps (per batch,
// stride map_stride): row i of A is A + arow[i]*lda, row k of B is B + brow[k]*ldb,
// row i of C is C + crow[i]*ldc (the pointers then carry only the column offset).
void rm_gemm(int m, int n, int k, const double* A, long long lda, long long sa, const double* B,
             long long ldb, long long sb, double* C, long long ldc, long long sc, int batch,
             double alpha, double beta, cudaStream_t st, const int* arow = nullptr, const int* brow = nullptr,
             const int* crow = nullptr, long long map_stride = 0) {
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
    g.amap = brow;
    g.bmap = arow;
    g.cmap = crow;
    g.map_stride = map_stride;
    gemm_batched(g, st);
}

template <int NT, int RPT, int PB>
void panel_launch(double* A, int G, int lda, int* map, int* ipiv, int K0, int k0, int jb, int rend,
                  DeviceStatus* status, const int* order_index, int batch, cudaStream_t st) {
    constexpr size_t smem = PanelGeo<NT, RPT, PB>::bytes;
    static unsigned long long attr = 0;
    smem_attr_once(lu_panel_crout_kernel<NT, RPT, PB>, (int)smem, attr);
    lu_panel_crout_kernel<NT, RPT, PB><<<batch, NT, smem, st>>>(A, G, lda, (long long)G * lda, map, ipiv, K0, k0,
                                                                jb, rend, status, order_index);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

// the kernel's PB must be the driver's panel width (it sizes the block's L in
// shared memory); rows per thread grow with the active height
template <int PB>
void panel_dispatch(int np, double* A, int G, int lda, int* map, int* ipiv, int K0, int k0, int jb, int rend,
                    DeviceStatus* status, const int* order_index, int batch, cudaStream_t st) {
    if (np <= 256)
        panel_launch<256, 1, PB>(A, G, lda, map, ipiv, K0, k0, jb, rend, status, order_index, batch, st);
    else if (np <= 512)
        panel_launch<512, 1, PB>(A, G, lda, map, ipiv, K0, k0, jb, rend, status, order_index, batch, st);
    else if (np <= 1024)
        panel_launch<512, 2, PB>(A, G, lda, map, ipiv, K0, k0, jb, rend, status, order_index, batch, st);
    else if constexpr (PB <= 8) {
        if (np <= 2048)
            panel_launch<512, 4, PB>(A, G, lda, map, ipiv, K0, k0, jb, rend, status, order_index, batch, st);
        else if constexpr (PB <= 4)
            panel_launch<512, 8, PB>(A, G, lda, map, ipiv, K0, k0, jb, rend, status, order_index, batch, st);
        else
            throw std::invalid_argument("lu: panel height exceeds the panel kernel");
    } else {
        throw std::invalid_argument("lu: panel height exceeds the panel kernel");
    }
}

int panel_width(int G) { return G <= 1024 ? 16 : (G <= 2048 ? 8 : 4); }

int outer_block() { return OB_MAX; }


// ------------------------------------------------------------------ few-column solve
// X <- A^-1 X for K columns (position order, [G][K] per matrix) by ONE CTA per
// matrix: the residual probes of the boundary gate (boundary.cuh), where the
// block-solve + GEMM launches of lu_solve_gathered cost tens of microseconds each
// for a handful of columns.  Columns < FL already hold L^-1 P b (back substitution
// only).  Per 64-row block: the coupling to the solved rows as a matvec (warp
// per row, L / U rows read coalesced through the row map), then the block's
// triangle from shared memory, one warp per column.
// x[k0 + r][c] -= sum_{j in [j0, j1)} A(perm[k0 + r], j) x[j][c] for rows r < jb,
// columns c >= c0: each warp takes 4 rows at once, 2 x 4 row loads in flight.
template <int K>
__device__ inline void few_matvec(const double* A, int lda, const int* perm, double* x, int k0, int jb, int j0,
                                  int j1, int c0, int warp, int nw, int lane) {
    for (int r0 = warp * 4; r0 < jb; r0 += nw * 4) {
        const double* row[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) row[q] = A + (size_t)perm[k0 + min(r0 + q, jb - 1)] * lda;
        double acc[4][K];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int c = 0; c < K; ++c) acc[q][c] = 0.0;
        int j = j0 + lane;
        for (; j + 96 < j1; j += 128) {  // 4 rows x 4 loads in flight per lane
            double a0[4], a1[4], a2[4], a3[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                a0[q] = row[q][j];
                a1[q] = row[q][j + 32];
                a2[q] = row[q][j + 64];
                a3[q] = row[q][j + 96];
            }
#pragma unroll
            for (int c = 0; c < K; ++c) {
                const double x0 = x[j * K + c], x1 = x[(j + 32) * K + c];
                const double x2 = x[(j + 64) * K + c], x3 = x[(j + 96) * K + c];
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    acc[q][c] = fma(a3[q], x3, fma(a2[q], x2, fma(a1[q], x1, fma(a0[q], x0, acc[q][c]))));
            }
        }
        for (; j + 32 < j1; j += 64) {
            double a0[4], a1[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                a0[q] = row[q][j];
                a1[q] = row[q][j + 32];
            }
#pragma unroll
            for (int c = 0; c < K; ++c) {
                const double x0 = x[j * K + c], x1 = x[(j + 32) * K + c];
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[q][c] = fma(a1[q], x1, fma(a0[q], x0, acc[q][c]));
            }
        }
        if (j < j1) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double a0 = row[q][j];
#pragma unroll
                for (int c = 0; c < K; ++c) acc[q][c] = fma(a0, x[j * K + c], acc[q][c]);
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int c = 0; c < K; ++c) {
                const double sv = warp_sum(acc[q][c]);
                if (lane == 0 && c >= c0 && r0 + q < jb) x[(k0 + r0 + q) * K + c] -= sv;
            }
    }
}

template <int K>
__global__ void __launch_bounds__(512) lu_few_solve_kernel(const double* Aall, int G, int lda, long long strideA,
                                                          const int* perm_all, double* Xall, int FL) {
    extern __shared__ double sm[];
    double* x = sm;                       // [G][K]
    double* T = sm + (size_t)G * K;       // [64][65] diagonal block
    const int b = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = blockDim.x >> 5;
    const double* A = Aall + (size_t)b * strideA;
    const int* perm = perm_all + (size_t)b * G;
    double* X = Xall + (size_t)b * G * K;
    for (int e = t; e < G * K; e += blockDim.x) x[e] = X[e];
    __syncthreads();
    const int nblk = (G + LU_NB - 1) / LU_NB;
    // ---- forward: unit lower L, columns [FL, K)
    if (FL < K)
        for (int bk = 0; bk < nblk; ++bk) {
            const int k0 = bk * LU_NB, jb = min(LU_NB, G - k0);
            for (int e = t; e < jb * LU_NB; e += blockDim.x) {
                const int r = e / LU_NB, c = e % LU_NB;
                T[r * (LU_NB + 1) + c] = c < jb ? A[(size_t)perm[k0 + r] * lda + k0 + c] : 0.0;
            }
            few_matvec<K>(A, lda, perm, x, k0, jb, 0, k0, FL, warp, nw, lane);
            __syncthreads();
            if (warp < K - FL) {
                const int c = FL + warp;
                double v0 = lane < jb ? x[(k0 + lane) * K + c] : 0.0;
                double v1 = lane + 32 < jb ? x[(k0 + lane + 32) * K + c] : 0.0;
                for (int j = 0; j < jb; ++j) {
                    const double xj = __shfl_sync(0xffffffffu, j < 32 ? v0 : v1, j & 31);
                    if (lane > j) v0 -= T[lane * (LU_NB + 1) + j] * xj;
                    if (lane + 32 > j && lane + 32 < jb) v1 -= T[(lane + 32) * (LU_NB + 1) + j] * xj;
                }
                if (lane < jb) x[(k0 + lane) * K + c] = v0;
                if (lane + 32 < jb) x[(k0 + lane + 32) * K + c] = v1;
            }
            __syncthreads();
        }
    // ---- backward: upper U (with its diagonal), every column
    for (int bk = nblk - 1; bk >= 0; --bk) {
        const int k0 = bk * LU_NB, jb = min(LU_NB, G - k0), k1 = k0 + jb;
        for (int e = t; e < jb * LU_NB; e += blockDim.x) {
            const int r = e / LU_NB, c = e % LU_NB;
            T[r * (LU_NB + 1) + c] = c < jb ? A[(size_t)perm[k0 + r] * lda + k0 + c] : 0.0;
        }
        few_matvec<K>(A, lda, perm, x, k0, jb, k1, G, 0, warp, nw, lane);
        __syncthreads();
        if (warp < K) {
            const int c = warp;
            double v0 = lane < jb ? x[(k0 + lane) * K + c] : 0.0;
            double v1 = lane + 32 < jb ? x[(k0 + lane + 32) * K + c] : 0.0;
            for (int j = jb - 1; j >= 0; --j) {
                const double piv = T[j * (LU_NB + 1) + j];
                double xj = __shfl_sync(0xffffffffu, j < 32 ? v0 : v1, j & 31) / piv;
                if (lane == j) v0 = xj;
                if (lane + 32 == j) v1 = xj;
                if (lane < j) v0 -= T[lane * (LU_NB + 1) + j] * xj;
                if (lane + 32 < j) v1 -= T[(lane + 32) * (LU_NB + 1) + j] * xj;
            }
            if (lane < jb) x[(k0 + lane) * K + c] = v0;
            if (lane + 32 < jb) x[(k0 + lane + 32) * K + c] = v1;
        }
        __syncthreads();
    }
    for (int e = t; e < G * K; e += blockDim.x) X[e] = x[e];
}
}  // namespace

namespace {
// U12 = L11^-1 A12 of an outer block (positions K0..K0+nb through the row map,
// nb <= OB_MAX) on a 32-column strip, one CTA per (strip, matrix), 2 CTAs per
// SM: L11's strict lower triangle packed in shared memory (row r at r(r-1)/2)
// and the strip in shared memory, both brought in by cp.async.  Rows in
// groups of 8: the group's coupling to every row above it,
//   X[g] -= L[g, 0:r0] X[0:r0],
// is an [8 x r0] x [r0 x 32] product on the FP64 tensor cores (warp per 8x8
// output tile, two accumulator chains), and the group's own 8 x 8 unit-lower
// triangle is applied as its explicit inverse (formed once per CTA: 16 tiny
// forward substitutions), x_i = sum_{j <= i} Li[i][j] y_j -- eight independent
// FMAs per row instead of a dependent chain.  The strips of one matrix are
// independent, so a split of the columns does not change any column's
// arithmetic.
constexpr int BT_W = 32;                            // strip width
constexpr int BT_L = OB_MAX * (OB_MAX + 1) / 2;     // packed triangle (upper: with its diagonal)
constexpr int BT_XL = BT_W + 4;                     // strip row stride (B fragments: 2-way at most)
constexpr int BT_G = OB_MAX / 8;                    // 8-row groups
constexpr size_t BT_SMEM = (size_t)(BT_L + OB_MAX * BT_XL + BT_G * 64) * sizeof(double);
// packed offsets: strict lower row r at r(r-1)/2 (entries j < r); upper row r at
// r nb - r(r-1)/2 (entries j = r .. nb-1, at offset j - r)
__device__ inline int bt_lo(int r) { return r * (r - 1) / 2; }
__device__ inline int bt_up(int r, int nb) { return r * nb - r * (r - 1) / 2; }

template <bool UPPER>
__global__ void __launch_bounds__(256, 2) lu_block_trsm_kernel(const double* Aall, int G, int lda, long long strideA,
                                                               const int* map_all, int K0, int nb, double* Mall,
                                                               int ldm, long long strideM, const int* mmap_all,
                                                               int c_lo, int c_hi) {
    extern __shared__ double btm[];
    double* Tp = btm;                      // packed triangle of the diagonal block
    double* Xs = btm + BT_L;               // [OB_MAX][BT_XL]
    double* Li = Xs + OB_MAX * BT_XL;      // [BT_G][8][8] inverses of the 8 x 8 diagonal blocks
    __shared__ int s_row[OB_MAX], s_mrow[OB_MAX];
    const int b = blockIdx.y, t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int gq = lane >> 2, tq = lane & 3;
    const int col0 = c_lo + blockIdx.x * BT_W;
    const double* A = Aall + (size_t)b * strideA;
    double* M = Mall + (size_t)b * strideM;
    const int* map = map_all + (size_t)b * G;
    const int* mmap = mmap_all ? mmap_all + (size_t)b * G : nullptr;
    if (t < nb) {
        s_row[t] = map[K0 + t];
        s_mrow[t] = mmap ? mmap[K0 + t] : K0 + t;
    }
    __syncthreads();
    const int c = col0 + lane;
    const bool live = c < c_hi;
    for (int r = w; r < OB_MAX; r += 8) {
        if (r < nb) {
            const double* src = A + (size_t)s_row[r] * lda;
            if (UPPER) {
                for (int j = r + lane; j < nb; j += 32) cp_async8(Tp + bt_up(r, nb) + (j - r), src + K0 + j);
            } else {
                for (int j = lane; j < r; j += 32) cp_async8(Tp + bt_lo(r) + j, src + K0 + j);
            }
            if (live) cp_async8(Xs + r * BT_XL + lane, M + (size_t)s_mrow[r] * ldm + c);
            else Xs[r * BT_XL + lane] = 0.0;
        } else {
            Xs[r * BT_XL + lane] = 0.0;
        }
    }
    cp_async_wait_all();
    __syncthreads();
    // T(r, j) for r, j inside the diagonal block (callers: the right triangle only)
    auto T = [&](int r, int j) -> double { return UPPER ? Tp[bt_up(r, nb) + (j - r)] : Tp[bt_lo(r) + j]; };
    // inverses of the diagonal 8 x 8 blocks: thread per (group, column jj)
    if (t < BT_G * 8) {
        const int g = t >> 3, jj = t & 7, r0 = 8 * g;
        double x[8];
        if (UPPER) {
#pragma unroll
            for (int i = 7; i >= 0; --i) {
                double v = (i == jj) ? 1.0 : 0.0;
                if (r0 + i < nb) {
                    if (i <= jj) {
#pragma unroll
                        for (int m = 0; m < 8; ++m)
                            if (m > i && m <= jj && r0 + m < nb) v = fma(-T(r0 + i, r0 + m), x[m], v);
                        v /= T(r0 + i, r0 + i);
                    } else {
                        v = 0.0;
                    }
                }
                x[i] = v;
            }
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                double v = (i == jj) ? 1.0 : 0.0;
                if (i > jj && r0 + i < nb) {
#pragma unroll
                    for (int m = 0; m < 8; ++m)
                        if (m >= jj && m < i) v = fma(-T(r0 + i, r0 + m), x[m], v);
                }
                x[i] = v;
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) Li[g * 64 + i * 8 + jj] = x[i];
    }
    __syncthreads();
    const int ngr = (nb + 7) / 8;
    for (int gi = 0; gi < ngr; ++gi) {
        const int g = UPPER ? ngr - 1 - gi : gi, r0 = 8 * g;
        // coupling to the solved rows (above for L, below for U) on the tensor
        // cores: warp w < 4 owns the columns 8w..8w+7, two accumulator chains
        const int k_lo = UPPER ? r0 + 8 : 0, k_hi = UPPER ? ngr * 8 : r0;
        if (k_hi > k_lo && w < 4) {
            const int ra = r0 + gq;
            const bool rok = ra < nb;
            const int rr = min(ra, nb - 1);
            double c0[2] = {0.0, 0.0}, c1[2] = {0.0, 0.0};
            for (int k = k_lo; k < k_hi; k += 8) {  // (k_hi - k_lo is a multiple of 8)
                const int ka = k + tq, kb = k + 4 + tq;
                const double a0 = (rok && ka < nb) ? T(rr, ka) : 0.0, a1 = (rok && kb < nb) ? T(rr, kb) : 0.0;
                const double b0 = Xs[ka * BT_XL + 8 * w + gq], b1 = Xs[kb * BT_XL + 8 * w + gq];
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(c0[0]), "+d"(c0[1]) : "d"(a0), "d"(b0));
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(c1[0]), "+d"(c1[1]) : "d"(a1), "d"(b1));
            }
            if (rok) {
                double* xr = Xs + ra * BT_XL + 8 * w + 2 * tq;
                xr[0] -= c0[0] + c1[0];
                xr[1] -= c0[1] + c1[1];
            }
        }
        __syncthreads();
        // the group's triangle by its inverse: warp w -> row r0 + w
        double x = 0.0;
        const double* lrow = Li + g * 64 + w * 8;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (UPPER ? j >= w : j <= w) x = fma(lrow[j], Xs[(r0 + j) * BT_XL + lane], x);
        __syncthreads();
        if (r0 + w < nb) Xs[(r0 + w) * BT_XL + lane] = x;
        __syncthreads();
    }
    if (live)
        for (int r = w; r < nb; r += 8) M[(size_t)s_mrow[r] * ldm + c] = Xs[r * BT_XL + lane];
}

// the diagonal block [K0, K0 + nb) (nb <= 128, rows through map) applied to the
// columns [c_lo, c_hi) of A: L^-1 (unit lower) or U^-1 (upper with its diagonal)
// (M: the strip's matrix, rows mmap[K0 + r] or K0 + r when mmap is null)
template <bool UPPER>
void block_trsm_launch(const double* A, int G, int lda, long long gg, const int* map, int K0, int nb, double* M,
                       int ldm, long long strideM, const int* mmap, int c_lo, int c_hi, int batch, cudaStream_t st) {
    if (c_hi <= c_lo || nb <= 0) return;
    constexpr int smem = (int)BT_SMEM;
    static unsigned long long attr = 0;
    smem_attr_once(lu_block_trsm_kernel<UPPER>, smem, attr);
    const dim3 grid((c_hi - c_lo + BT_W - 1) / BT_W, batch);
    lu_block_trsm_kernel<UPPER><<<grid, 256, smem, st>>>(A, G, lda, gg, map, K0, nb, M, ldm, strideM, mmap, c_lo,
                                                         c_hi);
    VRTE_CUDA_CHECK(cudaGetLastError());
}
template <bool UPPER>
void block_trsm_launch(double* A, int G, int lda, long long gg, const int* map, int K0, int nb, int c_lo, int c_hi,
                       int batch, cudaStream_t st) {
    block_trsm_launch<UPPER>(A, G, lda, gg, map, K0, nb, A, lda, gg, map, c_lo, c_hi, batch, st);
}

// Outer block [K0, K0 + NBk) (rows to rend) applied to columns [c_lo, c_hi):
// U12 = L11^-1 A12 on the block's pivot rows (the fused 128-row solve), then
// the trailing update A22 -= L21 U12 (rows past the profile have zero
// multipliers).
void block_update(double* A, int G, int lda, long long gg, const int* map, int K0, int NBk, int rend, int c_lo,
                  int c_hi, int batch, cudaStream_t st) {
    const int nc = c_hi - c_lo;
    if (nc <= 0) return;
    block_trsm_launch<false>(A, G, lda, gg, map, K0, NBk, c_lo, c_hi, batch, st);
    if (rend - K0 - NBk > 0)
        rm_gemm(rend - K0 - NBk, nc, NBk, A + K0, lda, gg, A + c_lo, lda, gg, A + c_lo, lda, gg, batch, -1.0, 1.0, st,
                map + K0 + NBk, map + K0, map + K0 + NBk, G);
}

void block_panels(double* A, int G, int lda, int* map, int* ipiv, int K0, int NBk, int rend, DeviceStatus* status,
                  const int* order_index, int batch, cudaStream_t st) {
    const int PB = panel_width(G);
    for (int k0 = K0; k0 < K0 + NBk; k0 += PB) {
        const int jb = min(PB, K0 + NBk - k0);
        const int np = rend - k0;
        if (PB == 16)
            panel_dispatch<16>(np, A, G, lda, map, ipiv, K0, k0, jb, rend, status, order_index, batch, st);
        else if (PB == 8)
            panel_dispatch<8>(np, A, G, lda, map, ipiv, K0, k0, jb, rend, status, order_index, batch, st);
        else
            panel_dispatch<4>(np, A, G, lda, map, ipiv, K0, k0, jb, rend, status, order_index, batch, st);
    }
}
}  // namespace

int lu_outer_blocks(int G) { return (G + OB_MAX - 1) / OB_MAX; }

void lu_factor_rm(double* A, int G, int batch, int* ipiv, int* perm, DeviceStatus* status,
                  const int* order_index, cudaStream_t st, int prof_d, int prof_P, int lda, int ncols,
                  cudaEvent_t cols_ready, const LuLookahead* la, const LuRhsDefer* rd) {
    if (G > 4096) throw std::invalid_argument("vrte_cuda: boundary system larger than 4096 rows");
    if (lda <= 0) lda = G;
    if (ncols <= 0) ncols = G;  // columns past G: right-hand sides eliminated along (augmented system)
    const int OB = outer_block();
    const long long gg = (long long)G * lda;
    int* map = perm;  // the row map IS the net permutation: row i of P A = row perm[i] of A
    auto row_end = [&](int col) { return prof_d > 0 ? min(G, bnd_row_end(col, prof_d, prof_P)) : G; };
    auto map_init = [&](cudaStream_t s) {
        const long long total = (long long)batch * G;
        lu_map_init_kernel<<<(unsigned)min(4096LL, (total + 255) / 256), 256, 0, s>>>(map, total, G);
        VRTE_CUDA_CHECK(cudaGetLastError());
    };
    // deferred right-hand sides: the row map as it stands after block K's panels
    auto rhs_snapshot = [&](int K0, cudaStream_t s) {
        if (!rd) return;
        const int kb = K0 / OB;
        VRTE_CUDA_CHECK(cudaMemcpyAsync(rd->snaps + (size_t)kb * batch * G, map, sizeof(int) * (size_t)batch * G,
                                        cudaMemcpyDeviceToDevice, s));
        VRTE_CUDA_CHECK(cudaEventRecord(rd->ev[kb], s));
    };
    if (!la || G <= OB) {
        map_init(st);
        for (int K0 = 0; K0 < G; K0 += OB) {
            const int NBk = min(OB, G - K0);
            const int rend = row_end(K0 + NBk - 1);  // profile is non-decreasing in the column
            block_panels(A, G, lda, map, ipiv, K0, NBk, rend, status, order_index, batch, st);
            rhs_snapshot(K0, st);
            if (cols_ready && ncols > K0 + NBk) {  // the columns past G (right-hand sides) come from another stream
                VRTE_CUDA_CHECK(cudaStreamWaitEvent(st, cols_ready, 0));
                cols_ready = nullptr;
            }
            block_update(A, G, lda, gg, map, K0, NBk, rend, K0 + NBk, ncols, batch, st);
        }
        return;
    }
    // Look-ahead by one block.  hi: panels(K), [wait rest(K-1)], map snapshot,
    // update of block K+1's columns, panels(K+1), ...; lo: the update of the
    // columns past block K+1 (the right-hand sides included) by block K, through
    // the snapshot -- the panels of block K+1 permute the positions past block K
    // while it runs, the snapshot keeps the set of rows block K's multipliers
    // live in.  Each row is updated by exactly the same operations as without
    // look-ahead, in the same order: the factors are bitwise identical.
    cudaStream_t hi = la->hi, lo = la->lo;
    VRTE_CUDA_CHECK(cudaEventRecord(la->ev[0], st));
    VRTE_CUDA_CHECK(cudaStreamWaitEvent(hi, la->ev[0], 0));
    VRTE_CUDA_CHECK(cudaStreamWaitEvent(lo, la->ev[0], 0));
    if (cols_ready) VRTE_CUDA_CHECK(cudaStreamWaitEvent(lo, cols_ready, 0));
    map_init(hi);
    block_panels(A, G, lda, map, ipiv, 0, min(OB, G), row_end(min(OB, G) - 1), status, order_index, batch, hi);
    rhs_snapshot(0, hi);
    bool rest_pending = false;
    for (int K0 = 0; K0 < G; K0 += OB) {
        const int NBk = min(OB, G - K0), c1 = K0 + NBk;
        const int rend = row_end(c1 - 1);
        const int nxt = min(OB, G - c1);  // block K+1's width (0: K is the last block)
        if (rest_pending) VRTE_CUDA_CHECK(cudaStreamWaitEvent(hi, la->ev[2], 0));
        rest_pending = false;
        if (nxt == 0) {  // last block: the right-hand sides only
            if (cols_ready) VRTE_CUDA_CHECK(cudaStreamWaitEvent(hi, cols_ready, 0));
            block_update(A, G, lda, gg, map, K0, NBk, rend, c1, ncols, batch, hi);
            break;
        }
        if (ncols > c1 + nxt) {
            VRTE_CUDA_CHECK(cudaMemcpyAsync(la->snap, map, sizeof(int) * (size_t)batch * G, cudaMemcpyDeviceToDevice, hi));
            VRTE_CUDA_CHECK(cudaEventRecord(la->ev[1], hi));
            VRTE_CUDA_CHECK(cudaStreamWaitEvent(lo, la->ev[1], 0));
            block_update(A, G, lda, gg, la->snap, K0, NBk, rend, c1 + nxt, ncols, batch, lo);
            VRTE_CUDA_CHECK(cudaEventRecord(la->ev[2], lo));
            rest_pending = true;
        }
        block_update(A, G, lda, gg, map, K0, NBk, rend, c1, c1 + nxt, batch, hi);
        block_panels(A, G, lda, map, ipiv, c1, nxt, row_end(c1 + nxt - 1), status, order_index, batch, hi);
        rhs_snapshot(c1, hi);
    }
    VRTE_CUDA_CHECK(cudaEventRecord(la->ev[3], lo));
    VRTE_CUDA_CHECK(cudaStreamWaitEvent(st, la->ev[3], 0));
    VRTE_CUDA_CHECK(cudaEventRecord(la->ev[3], hi));
    VRTE_CUDA_CHECK(cudaStreamWaitEvent(st, la->ev[3], 0));
}

void lu_rhs_forward(double* A, int G, int lda, int R, int batch, const LuRhsDefer& rd, int prof_d, int prof_P,
                    cudaStream_t st) {
    const int OB = outer_block();
    const long long gg = (long long)G * lda;
    for (int K0 = 0; K0 < G; K0 += OB) {
        const int NBk = min(OB, G - K0), kb = K0 / OB;
        const int rend = prof_d > 0 ? min(G, bnd_row_end(K0 + NBk - 1, prof_d, prof_P)) : G;
        VRTE_CUDA_CHECK(cudaStreamWaitEvent(st, rd.ev[kb], 0));
        block_update(A, G, lda, gg, rd.snaps + (size_t)kb * batch * G, K0, NBk, rend, G, G + R, batch, st);
    }
}

int lu_rhs_forward_launch_count(int G) {
    const int OB = outer_block();
    int n = 0;
    for (int K0 = 0; K0 < G; K0 += OB) n += 2;  // fused block solve + trailing GEMM (the last: rows below may be none)
    return n;
}

// Back substitution on an augmented factorization ([A | B] factored with
// ncols = G + R: the columns past G already hold L^-1 P B), in place through
// the row map, down to row_lo; then the solution rows [row_lo, G) are
// gathered in unknown order into X [batch][G][R].
__global__ void lu_gather_aug_kernel(const double* Aall, int G, int lda, int R, const int* perm_all, int row_lo,
                                     double* X, int batch, int c0) {
    const long long total = (long long)batch * (G - row_lo) * R;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(e % R);
        const long long rb = e / R;
        const int i = row_lo + (int)(rb % (G - row_lo)), b = (int)(rb / (G - row_lo));
        X[((size_t)b * G + i) * R + c] =
            Aall[(size_t)b * G * lda + (size_t)perm_all[(size_t)b * G + i] * lda + c0 + c];
    }
}

namespace {
// Back substitution of columns [c0, c0 + nc) of the augmented factorization in
// place, blocks bk_hi .. blo (64 rows each): outer steps of 2 x 64 rows, each
// the fused 128-row upper solve (lu_block_trsm_kernel<true>) and ONE update of
// the rows above down to blo's first row with k = 128 (the long-k GEMM runs
// near the DMMA rate; k = 64 does not).
void backsolve_blocks(double* A, int G, int lda, int c0, int nc, int batch, const int* perm, int bk_hi, int blo,
                      cudaStream_t st) {
    const long long gg = (long long)G * lda;
    const int rl = blo * LU_NB;
    for (int bk = bk_hi; bk >= blo; bk -= 2) {
        const int k1 = bk * LU_NB, jb1 = min(LU_NB, G - k1);
        const int k0 = (bk - 1 >= blo) ? k1 - LU_NB : k1, jb = k1 + jb1 - k0;
        block_trsm_launch<true>(A, G, lda, gg, perm, k0, jb, c0, c0 + nc, batch, st);
        if (k0 > rl)
            rm_gemm(k0 - rl, nc, jb, A + k0, lda, gg, A + c0, lda, gg, A + c0, lda, gg, batch, -1.0, 1.0, st,
                    perm + rl, perm + k0, perm + rl, G);
    }
}

int backsolve_launches(int bk_hi, int blo) {
    int n = 0;
    for (int bk = bk_hi; bk >= blo; bk -= 2) n += 1 + (bk - 1 > blo ? 1 : 0);
    return n;
}
}  // namespace

void lu_backsolve_aug(double* A, int G, int lda, int R, int batch, const int* perm, double* X, int row_lo,
                      cudaStream_t st) {
    const int nblk = (G + LU_NB - 1) / LU_NB;
    const int blo = max(0, row_lo) / LU_NB, rl = blo * LU_NB;
    backsolve_blocks(A, G, lda, G, R, batch, perm, nblk - 1, blo, st);
    const long long total = (long long)batch * (G - rl) * R;
    lu_gather_aug_kernel<<<(unsigned)min(16384LL, (total + 255) / 256), 256, 0, st>>>(A, G, lda, R, perm, rl, X,
                                                                                     batch, G);
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
    // L and U rows are read through the row map (perm); 128-row diagonal blocks
    // by the fused solve, the couplings as GEMMs
    (void)prof_d;
    (void)prof_P;
    for (int k0 = 0; k0 < G; k0 += OB_MAX) {
        const int jb = min(OB_MAX, G - k0);
        block_trsm_launch<false>(A, G, G, gg, perm, k0, jb, X, ncol, gn, nullptr, 0, ncol, batch, st);
        if (G - k0 - jb > 0)
            rm_gemm(G - k0 - jb, ncol, jb, A + k0, G, gg, X + (size_t)k0 * ncol, ncol, gn,
                    X + (size_t)(k0 + jb) * ncol, ncol, gn, batch, -1.0, 1.0, st, perm + k0 + jb, nullptr, nullptr, G);
    }
    // back substitution only down to row_lo's block: the unknowns above it are
    // not wanted (X rows there are left holding the forward solution)
    const int nblk = (G + OB_MAX - 1) / OB_MAX;
    const int blo = max(0, row_lo) / OB_MAX, rl = blo * OB_MAX;
    for (int bk = nblk - 1; bk >= blo; --bk) {
        const int k0 = bk * OB_MAX, jb = min(OB_MAX, G - k0);
        block_trsm_launch<true>(A, G, G, gg, perm, k0, jb, X, ncol, gn, nullptr, 0, ncol, batch, st);
        if (k0 > rl)
            rm_gemm(k0 - rl, ncol, jb, A + k0, G, gg, X + (size_t)k0 * ncol, ncol, gn, X + (size_t)rl * ncol, ncol,
                    gn, batch, -1.0, 1.0, st, perm + rl, nullptr, nullptr, G);
    }
}

void lu_solve_gathered(const double* A, int G, int lda, int batch, const int* perm, double* X, int ncol,
                       cudaStream_t st, int fwd_lo) {
    const long long gg = (long long)G * lda, gn = (long long)G * ncol;
    // forward substitution on columns [fwd_lo, ncol) (the others already hold L^-1 P b)
    if (fwd_lo < ncol)
        for (int k0 = 0; k0 < G; k0 += OB_MAX) {
            const int jb = min(OB_MAX, G - k0);
            block_trsm_launch<false>(A, G, lda, gg, perm, k0, jb, X, ncol, gn, nullptr, fwd_lo, ncol, batch, st);
            if (G - k0 - jb > 0)
                rm_gemm(G - k0 - jb, ncol - fwd_lo, jb, A + k0, lda, gg, X + (size_t)k0 * ncol + fwd_lo, ncol, gn,
                        X + (size_t)(k0 + jb) * ncol + fwd_lo, ncol, gn, batch, -1.0, 1.0, st, perm + k0 + jb, nullptr,
                        nullptr, G);
        }
    const int nblk = (G + OB_MAX - 1) / OB_MAX;
    for (int bk = nblk - 1; bk >= 0; --bk) {
        const int k0 = bk * OB_MAX, jb = min(OB_MAX, G - k0);
        block_trsm_launch<true>(A, G, lda, gg, perm, k0, jb, X, ncol, gn, nullptr, 0, ncol, batch, st);
        if (k0 > 0)
            rm_gemm(k0, ncol, jb, A + k0, lda, gg, X + (size_t)k0 * ncol, ncol, gn, X, ncol, gn, batch, -1.0, 1.0, st,
                    perm, nullptr, nullptr, G);
    }
}

int lu_gathered_launch_count(int G, int ncol, int fwd_lo) {
    const int nblk = (G + OB_MAX - 1) / OB_MAX;
    return (fwd_lo < ncol ? 2 * nblk - 1 : 0) + 2 * nblk - 1;
}

// the factorization with the look-ahead schedule (the boundary systems): per
// outer block its panels, then the update of the next block's columns (fused
// solve + GEMM) and of the rest (the same, on the other stream)
int lu_aug_launch_count(int G, int R, int row_lo) {
    const int PB = panel_width(G), OB = outer_block();
    int n = 1;  // row map init
    for (int K0 = 0; K0 < G; K0 += OB) {
        const int NBk = min(OB, G - K0), c1 = K0 + NBk, nxt = min(OB, G - c1);
        n += (NBk + PB - 1) / PB;
        if (nxt == 0)
            n += R > 0 ? 1 : 0;
        else
            n += 2 + (G + R > c1 + nxt ? 2 : 0);
    }
    const int nblk = (G + LU_NB - 1) / LU_NB, blo = max(0, row_lo) / LU_NB;
    n += backsolve_launches(nblk - 1, blo) + 1;  // + gather
    return n;
}

// serial factorization + gathered solve (the eigenvector inverse)
int lu_rm_launch_count(int G) {
    const int PB = panel_width(G), OB = outer_block();
    int n = 1;  // row map init
    for (int K0 = 0; K0 < G; K0 += OB) {
        const int NBk = min(OB, G - K0);
        n += (NBk + PB - 1) / PB;  // fused Crout panels
        if (G - K0 - NBk > 0) n += 2;  // fused block solve + trailing GEMM
    }
    const int nblk = (G + OB_MAX - 1) / OB_MAX;
    n += 1 + 2 * nblk - 1 + 2 * nblk - 1;  // gather + forward + backward
    return n;
}

}  // namespace vrte

namespace vrte {
void lu_few_solve(const double* A, int G, int lda, int batch, const int* perm, double* X, int K, int fwd_lo,
                  cudaStream_t st) {
    if (K != 4) throw std::invalid_argument("lu_few_solve: K = 4 only");
    if (G > 4096) throw std::invalid_argument("lu_few_solve: G > 4096");
    const size_t smem = ((size_t)G * K + (size_t)LU_NB * (LU_NB + 1)) * sizeof(double);
    constexpr int smem_max = (4096 * 4 + LU_NB * (LU_NB + 1)) * (int)sizeof(double);
    static unsigned long long attr = 0;
    smem_attr_once(lu_few_solve_kernel<4>, smem_max, attr);
    lu_few_solve_kernel<4><<<batch, 512, smem, st>>>(A, G, lda, (long long)G * lda, perm, X, fwd_lo);
    VRTE_CUDA_CHECK(cudaGetLastError());
}
}  // namespace vrte
