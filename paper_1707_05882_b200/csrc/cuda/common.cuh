// common.cuh -- shared device helpers for the sm_100a BRDF path.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#define VRTE_CUDA_CHECK(x)                                                                   \
    do {                                                                                     \
        cudaError_t err__ = (x);                                                             \
        if (err__ != cudaSuccess) vrte::cuda_fail(err__, #x, __FILE__, __LINE__);            \
    } while (0)

namespace vrte {

[[noreturn]] void cuda_fail(cudaError_t e, const char* what, const char* file, int line);

constexpr double kPi = 3.14159265358979323846;
constexpr double kNuClamp = 4e9;             // homogeneous.hpp:68
constexpr double kEigenResidualBound = 1e-9;  // homogeneous.hpp:71
constexpr double kUlp = 2.220446049250313e-16;      // dlamch('P')
constexpr double kSafeMin = 2.2250738585072014e-308; // dlamch('S')

// cudaFuncSetAttribute is per device: set a kernel's dynamic shared-memory
// limit once per (kernel, device) -- `mask` is the call site's static bitmask.
template <typename K>
inline void smem_attr_once(K kernel, int bytes, unsigned long long& mask) {
    int dev = 0;
    VRTE_CUDA_CHECK(cudaGetDevice(&dev));
    const unsigned long long bit = 1ull << (dev & 63);
    if (__atomic_load_n(&mask, __ATOMIC_ACQUIRE) & bit) return;
    VRTE_CUDA_CHECK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    __atomic_fetch_or(&mask, bit, __ATOMIC_ACQ_REL);
}

// Device-side failure record: the first failing (code, stage, index) wins
// and the host turns it into a NumericalError with the reference's wording.
struct DeviceStatus {
    int code;      // 0 ok, else failure kind (see FailKind)
    int stage;
    int index;     // (s*L + m) or m
    int aux;
    double value;  // offending residual / eigenvalue
    double value2;
    unsigned long long dithered;
    unsigned long long clamped;
    unsigned long long polished;
    double max_eigen_residual;
    double max_particular_residual;
    double max_boundary_residual;
    double max_boundary_condition;    // lower-bound estimate of cond_1 of the boundary matrices
    unsigned long long bnd_cond_warnings;  // orders above 1e14 (boundary.cpp:259-263 warns)
    int bnd_refine;                   // a right-hand side needs the refinement step
    int bnd_refined;                  // ... and it was taken
    int bnd_fallback;                 // a residual probe failed: full solve + reference gate
    double part_check;                // interim max balance residual (adaptive particular refinement)
    double max_balance_residual;      // particular 8N balance residual (particular.cpp:86-105)
    unsigned long long qr_sweeps;
    unsigned long long qr_steps;
    unsigned long long qr_cycles[8];  // debug phase timers (clock64 in thread 0)
    unsigned long long neg_key;       // ~(first negative-intensity table index) (atomicMax)
};

enum FailKind {
    kFailNone = 0,
    kFailHqrNoConverge = 1,
    kFailNonFiniteEigen = 2,
    kFailNegativeAxis = 3,
    kFailEigenResidual = 4,
    kFailParticular = 5,
    kFailBoundary = 6,
    kFailNegativeIntensity = 7,
    kFailLuSingular = 8,
    kFailBalance = 9,
    kFailNonFiniteTable = 10,
};

__device__ inline void report_failure(DeviceStatus* st, int code, int stage, int index, double v,
                                      double v2 = 0.0, int aux = 0) {
    if (atomicCAS(&st->code, 0, code) == 0) {
        st->stage = stage;
        st->index = index;
        st->aux = aux;
        st->value = v;
        st->value2 = v2;
    }
}

__device__ inline void atomic_max_double(double* addr, double v) {
    // valid for non-negative doubles: IEEE order == signed 64-bit integer order
    if (!(v >= 0.0)) return;
    atomicMax(reinterpret_cast<unsigned long long*>(addr), static_cast<unsigned long long>(__double_as_longlong(v)));
}

// ------------------------------------------------------------ complex helpers
struct cplx {
    double re, im;
};
__device__ __host__ inline cplx cmk(double r, double i) { return cplx{r, i}; }
__device__ __host__ inline cplx operator+(cplx a, cplx b) { return {a.re + b.re, a.im + b.im}; }
__device__ __host__ inline cplx operator-(cplx a, cplx b) { return {a.re - b.re, a.im - b.im}; }
__device__ __host__ inline cplx operator*(cplx a, cplx b) {
    return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
__device__ __host__ inline cplx operator*(double s, cplx a) { return {s * a.re, s * a.im}; }
__device__ __host__ inline cplx conjc(cplx a) { return {a.re, -a.im}; }
__device__ inline double cabs_(cplx a) { return hypot(a.re, a.im); }
// Smith's division (std::complex-like accuracy)
__device__ inline cplx cdiv(cplx a, cplx b) {
    if (fabs(b.re) >= fabs(b.im)) {
        const double r = b.im / b.re, den = b.re + b.im * r;
        return {(a.re + a.im * r) / den, (a.im - a.re * r) / den};
    }
    const double r = b.re / b.im, den = b.re * r + b.im;
    return {(a.re * r + a.im) / den, (a.im * r - a.re) / den};
}
// principal square root (std::sqrt(complex) semantics: Re >= 0, branch cut on negative axis)
__device__ inline cplx csqrt_(cplx z) {
    if (z.re == 0.0 && z.im == 0.0) return {0.0, z.im};
    const double t = sqrt((fabs(z.re) + hypot(z.re, z.im)) * 0.5);
    if (z.re >= 0.0) return {t, z.im / (2.0 * t)};
    return {fabs(z.im) / (2.0 * t), copysign(t, z.im)};
}
// exp(z)
__device__ inline cplx cexp_(cplx z) {
    const double e = exp(z.re);
    if (z.im == 0.0) return {e, 0.0};
    double s, c;
    sincos(z.im, &s, &c);
    return {e * c, e * s};
}

// ------------------------------------------------------------ reductions
__device__ inline double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ inline double warp_max(double v) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
// block-wide sum; `red` must hold >= 32 doubles; all threads get the result
__device__ inline double block_sum(double v, double* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double t = (threadIdx.x < nw) ? red[threadIdx.x] : 0.0;
    if (w == 0) t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
    __syncthreads();
    return red[0];
}
__device__ inline double block_max(double v, double* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double t = (threadIdx.x < nw) ? red[threadIdx.x] : 0.0;
    if (w == 0) t = warp_max(t);
    if (threadIdx.x == 0) red[0] = t;
    __syncthreads();
    return red[0];
}

// ------------------------------------------------------------ batched GEMM (gemm.cu)
// C[b] = alpha * op(A[b]) * op(B[b]) + beta * C[b], column-major, fp64.
struct GemmBatch {
    int m, n, k;
    const double* a;
    long long lda, stride_a;
    const double* b;
    long long ldb, stride_b;
    double* c;
    long long ldc, stride_c;
    int batch;
    double alpha, beta;
    bool trans_a, trans_b;
    // optional per-batch index maps (stride map_stride): A column k is A + amap[k]*lda,
    // B column n is B + bmap[n]*ldb, C column n is C + cmap[n]*ldc (null = identity)
    const int* amap;
    const int* bmap;
    const int* cmap;
    long long map_stride;
    // optional batch compaction: grid z < *zcount runs batch entry zmap[z] (the
    // refinement's extra steps on the slots still above target); null = all
    const int* zmap;
    const int* zcount;
};
constexpr int kMaxMapK = 256;
void gemm_batched(const GemmBatch& g, cudaStream_t stream);
void gemm_batched_cfg(const GemmBatch& g, cudaStream_t stream, int bk, int stages, int minb);

}  // namespace vrte
