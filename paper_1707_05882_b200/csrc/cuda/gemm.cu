// gemm.cu -- batched fp64 GEMM for the dense contractions of the BRDF path
// (F*E, eigenvector back-transforms, E*X recoveries, particular Z-projections,
// boundary trailing updates / triangular-solve updates, tau=0 field products).
//
// 64x64 CTA tile, BK=16 k-slab double-buffered in shared memory, 256 threads
// each owning a 4x4 register micro-tile (rows tx+16i, cols ty+16j so both smem
// operand reads are bank-conflict free).  DFMA pipe; B200's FP64 tensor rate
// equals its DFMA rate, so the tensor path buys nothing for fp64 here.
#include "common.cuh"

namespace vrte {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

template <bool TA, bool TB>
__global__ void __launch_bounds__(NT) gemm_kernel(GemmBatch g) {
    __shared__ double As[2][BK][BM + 1];
    __shared__ double Bs[2][BK][BN + 1];
    const int bz = blockIdx.z;
    const double* A = g.a + bz * g.stride_a;
    const double* B = g.b + bz * g.stride_b;
    double* C = g.c + bz * g.stride_c;
    const int r0 = blockIdx.x * BM, c0 = blockIdx.y * BN;
    const int t = threadIdx.x, tx = t & 15, ty = t >> 4;

    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;

    double ra[4], rb[4];
    auto load_regs = [&](int k0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            int i, kk;
            if (!TA) {
                i = t & 63;
                kk = (t >> 6) + 4 * q;
                const int gr = r0 + i, gk = k0 + kk;
                ra[q] = (gr < g.m && gk < g.k) ? A[gr + (long long)gk * g.lda] : 0.0;
            } else {
                kk = t & 15;
                i = (t >> 4) + 16 * q;
                const int gr = r0 + i, gk = k0 + kk;
                ra[q] = (gr < g.m && gk < g.k) ? A[gk + (long long)gr * g.lda] : 0.0;
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            int j, kk;
            if (!TB) {
                kk = t & 15;
                j = (t >> 4) + 16 * q;
                const int gc = c0 + j, gk = k0 + kk;
                rb[q] = (gc < g.n && gk < g.k) ? B[gk + (long long)gc * g.ldb] : 0.0;
            } else {
                j = t & 63;
                kk = (t >> 6) + 4 * q;
                const int gc = c0 + j, gk = k0 + kk;
                rb[q] = (gc < g.n && gk < g.k) ? B[gc + (long long)gk * g.ldb] : 0.0;
            }
        }
    };
    auto store_smem = [&](int buf) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (!TA)
                As[buf][(t >> 6) + 4 * q][t & 63] = ra[q];
            else
                As[buf][t & 15][(t >> 4) + 16 * q] = ra[q];
            if (!TB)
                Bs[buf][t & 15][(t >> 4) + 16 * q] = rb[q];
            else
                Bs[buf][(t >> 6) + 4 * q][t & 63] = rb[q];
        }
    };

    const int nk = (g.k + BK - 1) / BK;
    if (nk > 0) {
        load_regs(0);
        store_smem(0);
    }
    __syncthreads();
    for (int kt = 0; kt < nk; ++kt) {
        const int buf = kt & 1;
        if (kt + 1 < nk) load_regs((kt + 1) * BK);
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            double a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[buf][kk][tx + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[buf][kk][ty + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        if (kt + 1 < nk) store_smem(buf ^ 1);
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gr = r0 + tx + 16 * i, gc = c0 + ty + 16 * j;
            if (gr < g.m && gc < g.n) {
                double* p = C + gr + (long long)gc * g.ldc;
                const double v = g.alpha * acc[i][j];
                *p = (g.beta == 0.0) ? v : fma(g.beta, *p, v);
            }
        }
}

}  // namespace

void gemm_batched(const GemmBatch& g, cudaStream_t stream) {
    if (g.m <= 0 || g.n <= 0 || g.batch <= 0) return;
    dim3 grid((g.m + BM - 1) / BM, (g.n + BN - 1) / BN, g.batch);
    if (!g.trans_a && !g.trans_b)
        gemm_kernel<false, false><<<grid, NT, 0, stream>>>(g);
    else if (g.trans_a && !g.trans_b)
        gemm_kernel<true, false><<<grid, NT, 0, stream>>>(g);
    else if (!g.trans_a && g.trans_b)
        gemm_kernel<false, true><<<grid, NT, 0, stream>>>(g);
    else
        gemm_kernel<true, true><<<grid, NT, 0, stream>>>(g);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace vrte
