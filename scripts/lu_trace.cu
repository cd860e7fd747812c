// Phase timing of the lazily pivoted LU (build with -DVRTE_LU_TRACE): batch of
// random G x G row-major systems, the panel kernel prints per-phase cycles of CTA 0.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "boundary.cuh"
namespace vrte {
[[noreturn]] void cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
    fprintf(stderr, "%s:%d %s: %s\n", file, line, what, cudaGetErrorString(e));
    exit(1);
}
}  // namespace vrte
int main(int argc, char** argv) {
    const int G = argc > 1 ? atoi(argv[1]) : 1024, batch = argc > 2 ? atoi(argv[2]) : 64;
    std::vector<double> h((size_t)G * G * batch);
    srand(1);
    for (auto& x : h) x = rand() / (double)RAND_MAX - 0.5;
    double *A, *A0;
    int *ipiv, *perm;
    vrte::DeviceStatus* st;
    cudaMalloc(&A, h.size() * 8);
    cudaMalloc(&A0, h.size() * 8);
    cudaMalloc(&ipiv, (size_t)G * batch * 4);
    cudaMalloc(&perm, (size_t)G * batch * 4);
    cudaMalloc(&st, sizeof(vrte::DeviceStatus));
    cudaMemcpy(A0, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int it = 0; it < 2; ++it) {
        cudaMemcpy(A, A0, h.size() * 8, cudaMemcpyDeviceToDevice);
        cudaMemset(st, 0, sizeof(vrte::DeviceStatus));
        cudaEventRecord(e0);
        vrte::lu_factor_rm(A, G, batch, ipiv, perm, st, nullptr, 0);
        cudaEventRecord(e1);
        cudaDeviceSynchronize();
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("iter %d: factor %.3f ms (G=%d batch=%d)\n", it, ms, G, batch);
        const int ncol = 256;
        double *B, *X;
        cudaMalloc(&B, (size_t)G * ncol * batch * 8);
        cudaMalloc(&X, (size_t)G * ncol * batch * 8);
        cudaMemset(B, 0, (size_t)G * ncol * batch * 8);
        cudaEventRecord(e0);
        vrte::lu_solve_rm(A, G, batch, perm, B, X, ncol, 0);
        cudaEventRecord(e1);
        cudaDeviceSynchronize();
        cudaEventElapsedTime(&ms, e0, e1);
        printf("iter %d: solve %.3f ms (ncol %d)\n", it, ms, ncol);
        cudaFree(B);
        cudaFree(X);
    }
    return 0;
}
