// gemm.cu -- batched fp64 GEMM for the dense contractions of the BRDF path
// (F*E, eigenvector back-transforms, 8N residual/refinement products,
// particular projections, boundary LU trailing updates, tau=0 field products).
//
// FP64 tensor cores: mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4; tcgen05 has no f64
// kind).  CTA tile 64 x 128 x 16, 8 warps as 2 x 4, each warp a 32 x 32 tile
// of 4 x 4 DMMA fragments (32 fp64 accumulators per thread).  Operands are
// streamed global -> shared with cp.async (2-stage double buffer, zero fill at
// the edges); the shared layout of each operand follows its transpose so the
// per-lane fragment loads are bank-conflict free:
//   A not transposed: As[k][m] (ld 72)     A transposed: As[m][k] (ld 20)
//   B not transposed: Bs[n][k] (ld 20)     B transposed: Bs[k][n] (ld 136)
// The epilogue stores the accumulator fragments directly; for the beta = 1
// trailing updates C is preloaded into the accumulators (overlapping the first
// operand tile) instead of being re-read in the epilogue.
#include <cstdlib>
#include <stdexcept>

#include "common.cuh"

namespace vrte {
namespace {

constexpr int BM = 64;

// shared-memory geometry of one pipeline stage for k-tile depth BK, tile width BN
template <int BK, int BN>
struct Geo {
    static constexpr int LDA_K = BM + 8;   // k-major A: As[k * LDA_K + m]
    static constexpr int LDA_M = BK + 4;   // m-major A: As[m * LDA_M + k]
    static constexpr int LDB_N = BK + 4;   // n-major B: Bs[n * LDB_N + k]
    static constexpr int LDB_K = BN + 8;   // k-major B: Bs[k * LDB_K + n]
    static constexpr int A_STAGE = (BK * LDA_K > BM * LDA_M) ? BK * LDA_K : BM * LDA_M;  // doubles
    static constexpr int B_STAGE = (BN * LDB_N > BK * LDB_K) ? BN * LDB_N : BK * LDB_K;
};

__device__ inline void cp_async8(double* smem, const double* gmem, bool valid) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int src_size = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_size));
}
__device__ inline void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ inline void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }
template <int N>
__device__ inline void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ inline void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// CTA tile BM x BN with NT = 2 BN threads: warps laid out (BM/32) x (BN/32),
// each a 32 x 32 tile of 4 x 4 DMMA fragments.
template <bool TA, bool TB, int BK, int ST, int MINB, int BN, bool MAP>
__global__ void __launch_bounds__(2 * BN, MINB) dmma_gemm_kernel(GemmBatch g) {
    constexpr int NT = 2 * BN, WN = BN / 32;
    using Gm = Geo<BK, BN>;
    constexpr int LDA_K = Gm::LDA_K, LDA_M = Gm::LDA_M, LDB_N = Gm::LDB_N, LDB_K = Gm::LDB_K;
    constexpr int A_STAGE = Gm::A_STAGE, B_STAGE = Gm::B_STAGE;
    extern __shared__ double smem[];
    double* As0 = smem;
    double* Bs0 = smem + ST * A_STAGE;
    int bz = blockIdx.z;
    if (g.zcount) {  // compacted batch (uniform per CTA: before any barrier)
        if (bz >= *g.zcount) return;
        bz = g.zmap[bz];
    }
    const double* A = g.a + bz * g.stride_a;
    const double* B = g.b + bz * g.stride_b;
    double* C = g.c + bz * g.stride_c;
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int wm = (warp / WN) * 32, wn = (warp % WN) * 32;  // warp tile origin in the CTA tile
    const int gq = lane >> 2, tq = lane & 3;                 // fragment coordinates
    // optional index maps (lazily pivoted LU, lu.cu): the k index of A, the n
    // index of B and the n index of C go through per-batch tables
    // (MAP = false: the plain kernel, no map state in registers)
    __shared__ int s_amap[MAP ? kMaxMapK : 1], s_bmap[MAP ? BN : 1], s_cmap[MAP ? BN : 1];
    const bool amapped = MAP && g.amap != nullptr, bmapped = MAP && g.bmap != nullptr,
               cmapped = MAP && g.cmap != nullptr;
    if (MAP) {
        const long long mo = (long long)bz * g.map_stride;
        if (amapped)
            for (int i = t; i < g.k; i += NT) s_amap[i] = g.amap[mo + i];
        for (int n = t; n < BN; n += NT) {
            const int gn = min(n0 + n, g.n - 1);
            if (bmapped) s_bmap[n] = g.bmap[mo + gn];
            if (cmapped) s_cmap[n] = g.cmap[mo + gn];
        }
        __syncthreads();
    }

    // mapped B rows: the per-thread row offsets are fixed over the k loop
    long long boff[MAP && !TB ? (BK * BN) / NT : 1];
    if (MAP && !TB) {
#pragma unroll
        for (int q = 0; q < (MAP && !TB ? (BK * BN) / NT : 1); ++q) {
            const int n = (t + q * NT) / BK;
            boff[q] = (long long)(bmapped ? s_bmap[n] : n0 + n) * g.ldb;
        }
    }
    auto load_stage = [&](int stage, int k0) {
        double* As = As0 + stage * A_STAGE;
        double* Bs = Bs0 + stage * B_STAGE;
        // A tile: BM x BK = 1024 doubles, 4 per thread
#pragma unroll
        for (int q = 0; q < (BM * BK) / NT; ++q) {
            const int e = t + q * NT;
            if (!TA) {  // contiguous along m: As[k][m]
                const int m = e % BM, k = e / BM;
                const int gm = m0 + m, gk = k0 + k;
                const bool ok = gm < g.m && gk < g.k;
                cp_async8(As + k * LDA_K + m, ok ? A + gm + (long long)(amapped ? s_amap[gk] : gk) * g.lda : A, ok);
            } else {    // contiguous along k: As[m][k]
                const int k = e % BK, m = e / BK;
                const int gm = m0 + m, gk = k0 + k;
                const bool ok = gm < g.m && gk < g.k;
                cp_async8(As + m * LDA_M + k, ok ? A + gk + (long long)gm * g.lda : A, ok);
            }
        }
        // B tile: BK x BN = 2048 doubles, 8 per thread
#pragma unroll
        for (int q = 0; q < (BK * BN) / NT; ++q) {
            const int e = t + q * NT;
            if (!TB) {  // contiguous along k: Bs[n][k]
                const int k = e % BK, n = e / BK;
                const int gn = n0 + n, gk = k0 + k;
                const bool ok = gn < g.n && gk < g.k;
                cp_async8(Bs + n * LDB_N + k, ok ? B + gk + (MAP ? boff[q] : (long long)gn * g.ldb) : B, ok);
            } else {    // contiguous along n: Bs[k][n]
                const int n = e % BN, k = e / BN;
                const int gn = n0 + n, gk = k0 + k;
                const bool ok = gn < g.n && gk < g.k;
                cp_async8(Bs + k * LDB_K + n, ok ? B + gn + (long long)gk * g.ldb : B, ok);
            }
        }
        cp_async_commit();
    };

    double acc[4][4][2];
    const int nk = (g.k + BK - 1) / BK;
    // prologue: ST-1 stages in flight (empty commit groups keep the count uniform)
#pragma unroll
    for (int s = 0; s < ST - 1; ++s) {
        if (s < nk)
            load_stage(s, s * BK);
        else
            cp_async_commit();
    }
    // beta = 1, alpha = +-1 (the trailing updates of LU / Hessenberg / refinement):
    // C is read into the accumulators while the first operand tile is in flight
    // (acc = alpha C, result = alpha acc), so no epilogue read round trip.
    const bool preload = g.beta == 1.0 && (g.alpha == 1.0 || g.alpha == -1.0);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            acc[i][j][0] = acc[i][j][1] = 0.0;
            if (preload) {
                const int gm = m0 + wm + 8 * i + gq, gn = n0 + wn + 8 * j + 2 * tq;
                if (gm < g.m) {
                    const int nl = wn + 8 * j + 2 * tq;
                    if (gn < g.n) acc[i][j][0] = g.alpha * C[gm + (long long)(cmapped ? s_cmap[nl] : gn) * g.ldc];
                    if (gn + 1 < g.n)
                        acc[i][j][1] = g.alpha * C[gm + (long long)(cmapped ? s_cmap[nl + 1] : gn + 1) * g.ldc];
                }
            }
        }

    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<ST - 2>();
        __syncthreads();
        {
            const int nx = kt + ST - 1;
            if (nx < nk)
                load_stage(nx % ST, nx * BK);
            else
                cp_async_commit();
        }
        const double* As = As0 + (kt % ST) * A_STAGE;
        const double* Bs = Bs0 + (kt % ST) * B_STAGE;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int m = wm + 8 * i + gq, k = kk + tq;
                af[i] = TA ? As[m * LDA_M + k] : As[k * LDA_K + m];
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int n = wn + 8 * j + gq, k = kk + tq;
                bf[j] = TB ? Bs[k * LDB_K + n] : Bs[n * LDB_N + k];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
    }
    // epilogue: fragments straight to global (each warp store covers 4 x 64-byte
    // column segments of the column-major C)
    const bool beta0 = g.beta == 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gm = m0 + wm + 8 * i + gq, gn = n0 + wn + 8 * j + 2 * tq;
            if (gm >= g.m) continue;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (gn + h >= g.n) continue;
                double* p = C + gm + (long long)(cmapped ? s_cmap[wn + 8 * j + 2 * tq + h] : gn + h) * g.ldc;
                const double v = g.alpha * acc[i][j][h];
                *p = preload ? v : (beta0 ? v : fma(g.beta, *p, v));
            }
        }
}

template <bool TA, bool TB, int BK, int ST, int MINB, int BN, bool MAP = false>
void launch(const GemmBatch& g, cudaStream_t stream) {
    static unsigned long long attr = 0;  // per-device bitmask (smem_attr_once)
    constexpr size_t smem = (size_t)ST * (Geo<BK, BN>::A_STAGE + Geo<BK, BN>::B_STAGE) * sizeof(double);
    int dev = 0;
    VRTE_CUDA_CHECK(cudaGetDevice(&dev));
    if (!(__atomic_load_n(&attr, __ATOMIC_ACQUIRE) & (1ull << (dev & 63)))) {
        VRTE_CUDA_CHECK(cudaFuncSetAttribute(dmma_gemm_kernel<TA, TB, BK, ST, MINB, BN, MAP>,
                                             cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        smem_attr_once(dmma_gemm_kernel<TA, TB, BK, ST, MINB, BN, MAP>, (int)smem, attr);
    }
    dim3 grid((g.m + BM - 1) / BM, (g.n + BN - 1) / BN, g.batch);
    dmma_gemm_kernel<TA, TB, BK, ST, MINB, BN, MAP><<<grid, 2 * BN, smem, stream>>>(g);
}

template <int BK, int ST, int MINB, int BN = 128>
void launch_cfg(const GemmBatch& g, cudaStream_t stream) {
    if (!g.trans_a && !g.trans_b && (g.amap || g.bmap || g.cmap))
        launch<false, false, BK, ST, MINB, BN, true>(g, stream);
    else if (!g.trans_a && !g.trans_b)
        launch<false, false, BK, ST, MINB, BN>(g, stream);
    else if (g.trans_a && !g.trans_b)
        launch<true, false, BK, ST, MINB, BN>(g, stream);
    else if (!g.trans_a && g.trans_b)
        launch<false, true, BK, ST, MINB, BN>(g, stream);
    else
        launch<true, true, BK, ST, MINB, BN>(g, stream);
}

}  // namespace

// Explicit pipeline configuration (k-tile depth, stages, CTAs per SM) --
// benchmarking hook; gemm_batched picks the measured best per shape class.
void gemm_batched_cfg(const GemmBatch& g, cudaStream_t stream, int bk, int stages, int minb) {
    if (g.m <= 0 || g.n <= 0 || g.batch <= 0) return;
    if (bk == 16 && stages == 2 && minb == 6) launch_cfg<16, 2, 6, 64>(g, stream);  // 64 x 64 tiles
    else if (bk == 16 && stages == 2 && minb == 3) launch_cfg<16, 2, 3>(g, stream);
    else if (bk == 16 && stages == 3) launch_cfg<16, 3, 2>(g, stream);
    else if (bk == 8 && stages == 4) launch_cfg<8, 4, 3>(g, stream);
    else launch_cfg<16, 2, 2>(g, stream);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

// Short contractions (k <= 96: LU / solve / Hessenberg trailing updates) are
// bound by per-CTA prologue/epilogue latency -> 3 CTAs per SM; long ones keep
// the register budget for a 3-stage pipeline (measured, profiles/r01_gemm_*).
void gemm_batched(const GemmBatch& g, cudaStream_t stream) {
    if ((g.amap && (g.trans_a || g.k > kMaxMapK)) || (g.bmap && g.trans_b))
        throw std::invalid_argument("gemm_batched: index maps need untransposed operands and k <= 256");
    const bool mapped = g.amap || g.bmap || g.cmap;
    constexpr int small_minb = 3;
    if (g.k <= 96)
        gemm_batched_cfg(g, stream, 16, 2, mapped ? 2 : small_minb);  // the mapped kernel needs the register budget
    else
        gemm_batched_cfg(g, stream, 16, 3, 2);
}

}  // namespace vrte
