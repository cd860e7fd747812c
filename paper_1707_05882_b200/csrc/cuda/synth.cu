// synth.cu -- Fourier synthesis of the tau = 0 upward Stokes stacks and the
// Mueller recovery (reconstruction.cpp:201-227, kernel.cpp:111-122,
// brdf.cpp:100-117):
//   I_c(node, dphi) = 1/2 sum_m Phi_{k(c)}(m, -dphi) up_m(incident, c)[node]
//   F_r = [I_0 .. I_3] * T_ii,   T_ii = B (mu0 B)^+ computed on the host,
// then the F00 roundoff clamp.  Orders are summed in fixed order 0..L-1 so the
// table does not depend on how orders were sharded across devices.
#include "kernels.cuh"
#include "synth.cuh"

namespace vrte {
namespace {

// Thread per (incident ii, node io, azimuth ip).
__global__ void synth_kernel(SynthArgs a) {
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const int N = a.N, np = a.n_dphi, d = 4 * N, R = 4 * a.n_in;
    const int No = N - a.out_lo;
    const long long total = (long long)a.n_in * No * np;
    if (idx >= total) return;
    const int ip = (int)(idx % np);
    const int io = a.out_lo + (int)((idx / np) % No);
    const int ii = (int)(idx / ((long long)np * No));
    double e[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) e[r][c] = 0.0;
    for (int m = 0; m < a.L; ++m) {
        const double sc = (m == 0) ? 1.0 : 2.0;
        const double cs = a.trig[2 * ((size_t)m * np + ip)];
        const double sn = a.trig[2 * ((size_t)m * np + ip) + 1];
        const double p1[4] = {sc * cs, sc * cs, sc * sn, sc * sn};
        const double p2[4] = {sc * -sn, sc * -sn, sc * cs, sc * cs};
        const double* u = a.up + (size_t)a.slot_of_order[m] * R * d;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const double* col = u + (size_t)(ii * 4 + c) * d + 4 * io;
#pragma unroll
            for (int r = 0; r < 4; ++r) e[r][c] += 0.5 * ((c < 2 ? p1[r] : p2[r]) * col[r]);
        }
    }
    if (a.pre) {  // exit through the interface: e <- pre(node) e
        const double* P = a.pre + (size_t)io * 16;
        double t[4][4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) t[r][c] = P[4 * r] * e[0][c] + P[4 * r + 1] * e[1][c] + P[4 * r + 2] * e[2][c] +
                                                  P[4 * r + 3] * e[3][c];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 4; ++c) e[r][c] = t[r][c];
    }
    const double* Tm = a.post + (size_t)ii * 16;
    double f[16];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) s += e[r][k] * Tm[4 * k + c];
            f[4 * r + c] = s;
        }
    bool finite = true;
#pragma unroll
    for (int k = 0; k < 16; ++k) finite = finite && isfinite(f[k]);
    if (!finite) {
        // a non-finite entry never leaves with VRTE_OK (the boundary gate normally stops it first)
        report_failure(a.status, kFailNonFiniteTable, 4, (int)idx, f[0]);
    } else if (f[0] < -1e-9) {
        // brdf.cpp:108-112 throws at the FIRST such entry in (incident, exit,
        // azimuth) order: keep the value and record the smallest index
        atomicMax(&a.status->neg_key, ~(unsigned long long)idx);
        report_failure(a.status, kFailNegativeIntensity, 4, (int)idx, f[0]);
    } else if (f[0] < 0.0) {
        f[0] = 0.0;
        atomicAdd(&a.status->clamped, 1ull);
    }
    double* o = a.out + idx * 16;
#pragma unroll
    for (int k = 0; k < 16; ++k) o[k] = f[k];
}

}  // namespace

void launch_synth(const SynthArgs& a, cudaStream_t st) {
    const long long total = (long long)a.n_in * (a.N - a.out_lo) * a.n_dphi;
    synth_kernel<<<(unsigned)((total + 127) / 128), 128, 0, st>>>(a);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace vrte
