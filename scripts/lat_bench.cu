// Latency microbenchmarks for the latency-bound kernels (LU panel, TRSM, QR
// chase): dependent-chain cycles per operation on one warp / one CTA.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, double a, double b, int n, long long* cyc) {
    double x = a;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, b, a);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = (t1 - t0);
}
__global__ void k_shfl(double* out, double a, int n, long long* cyc) {
    double x = a + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = (t1 - t0);
}
__global__ void k_redux(int* out, int n, long long* cyc) {
    unsigned x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __reduce_max_sync(0xffffffffu, x + threadIdx.x) - threadIdx.x;
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = (t1 - t0);
}
__global__ void k_bar(int* out, int n, long long* cyc) {
    __shared__ int s[1024];
    int x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        s[threadIdx.x] = x;
        __syncthreads();
        x = s[(threadIdx.x + 1) % blockDim.x] + 1;
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = (t1 - t0);
}
__global__ void k_rcp(double* out, double a, int n, long long* cyc) {
    double x = a + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = 1.0 / x + 1.0;
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = (t1 - t0);
}
__global__ void k_lds(double* out, int n, long long* cyc) {
    __shared__ double s[64];
    if (threadIdx.x < 64) s[threadIdx.x] = 0.0;
    __syncthreads();
    int idx = threadIdx.x & 31;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) idx = (int)s[idx] + (idx & 1);
    long long t1 = clock64();
    out[threadIdx.x] = idx;
    if (threadIdx.x == 0) *cyc = (t1 - t0);
}
__global__ void k_ldg(const long long* p, long long* out, int n, long long* cyc) {
    long long idx = 0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) idx = p[idx];
    long long t1 = clock64();
    out[threadIdx.x] = idx;
    if (threadIdx.x == 0) *cyc = (t1 - t0);
}

int main() {
    double* d;
    long long* c;
    int* di;
    cudaMalloc(&d, 1 << 20);
    cudaMalloc(&c, 64);
    cudaMalloc(&di, 1 << 16);
    long long h;
    const int n = 4096;
    auto rep = [&](const char* name, int ops) {
        cudaDeviceSynchronize();
        cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        printf("%-28s %7.1f cycles/op\n", name, (double)h / ops);
    };
    for (int rep2 = 0; rep2 < 2; ++rep2) {
        k_dfma<<<1, 32>>>(d, 1.0, 0.5, n, c); rep("DFMA chain", n);
        k_shfl<<<1, 32>>>(d, 1.0, n, c); rep("SHFL.64 chain", n);
        k_redux<<<1, 32>>>(di, n, c); rep("REDUX.MAX chain", n);
        k_rcp<<<1, 32>>>(d, 3.0, n, c); rep("1/x + 1 chain", n);
        k_lds<<<1, 32>>>(d, n, c); rep("LDS.64 chain", n);
        for (int nt : {32, 128, 256, 512, 1024}) {
            k_bar<<<1, nt>>>(di, n, c);
            char buf[64];
            snprintf(buf, sizeof buf, "STS+BAR+LDS (%d thr)", nt);
            rep(buf, n);
        }
    }
    // pointer chase in global memory: L2-resident (4 MB ring) and HBM (1 GB ring)
    for (size_t bytes : {(size_t)4 << 20, (size_t)1 << 30}) {
        long long* p;
        cudaMalloc(&p, bytes);
        const size_t nel = bytes / 8, stride = 4096 + 8;  // bytes per hop ~ 32 KB apart
        long long* hp = new long long[nel];
        for (size_t i = 0; i < nel; ++i) hp[i] = (long long)((i + stride) % nel);
        cudaMemcpy(p, hp, bytes, cudaMemcpyHostToDevice);
        delete[] hp;
        k_ldg<<<1, 1>>>(p, (long long*)d, 512, c);
        k_ldg<<<1, 1>>>(p, (long long*)d, 2048, c);
        char buf[64];
        snprintf(buf, sizeof buf, "LDG chase %zu MB", bytes >> 20);
        rep(buf, 2048);
        cudaFree(p);
    }
    return 0;
}
