// particular.cu -- beam-response (particular) solutions for every
// (medium, order, incident, unit Stokes channel), particular.cpp:27-107.
//
// The reference factors F E - mu0^-2 I afresh for every incident; here the
// eigendecomposition F E = V Lambda V^-1 of the homogeneous stage is reused, so
// each right-hand side costs two GEMMs plus an independent 1x1 / 2x2 solve per
// entry (brdf_device.cu shifted_solve), followed by iterative refinement
// against the true operator F (E g).
#include "kernels.cuh"
#include "particular.cuh"

namespace vrte {
namespace {

// Resonance dither (particular.cpp:43-57): if 1/mu0^2 lies within 1e-8
// relative of any homogeneous eigenvalue 1/nu_j^2, mu0 <- mu0 (1 - 1e-7).
// Warp per (om, incident).  Also emits the per-column shift 1/mu0_eff^2.
__global__ void dither_kernel(PartArgs a) {
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (gw >= a.batch * a.n_in) return;
    const int om = gw / a.n_in, ii = gw % a.n_in;
    const int d = a.d;
    const double mu0 = a.mu_in[ii];
    const double target = 1.0 / (mu0 * mu0);
    bool hit = false;
    for (int j = lane; j < d; j += 32) {
        const cplx nu = cmk(a.nu[2 * ((size_t)om * d + j)], a.nu[2 * ((size_t)om * d + j) + 1]);
        const cplx lam = cdiv(cmk(1.0, 0.0), nu * nu);
        if (cabs_(lam - cmk(target, 0.0)) < 1e-8 * cabs_(lam)) hit = true;
    }
    hit = __any_sync(0xffffffffu, hit);
    const double mu_eff = hit ? mu0 * (1.0 - 1e-7) : mu0;
    if (lane < 4) {
        const size_t col = (size_t)om * 4 * a.n_in + 4 * ii + lane;
        a.sigma[2 * col] = 1.0 / (mu_eff * mu_eff);
        a.sigma[2 * col + 1] = 0.0;
        a.kind[col] = 0;
    }
    if (lane == 0) {
        a.mu_eff[(size_t)om * a.n_in + ii] = mu_eff;
        if (hit) atomicAdd(&a.status->dithered, 1ull);
    }
}

// rhs = F s+ - s- / mu0_eff ; W <- rhs (solved in place), R keeps rhs.
__global__ void rhs_kernel(PartArgs a) {
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const int d = a.d, R = 4 * a.n_in;
    const long long total = (long long)a.batch * R * d;
    if (idx >= total) return;
    const int om = (int)(idx / ((long long)R * d));
    const int col = (int)((idx / d) % R);
    const double mu = a.mu_eff[(size_t)om * a.n_in + col / 4];
    const double v = a.fsp[idx] - a.sm[idx] / mu;
    a.rhs[idx] = v;
}

// h = mu0 (s+ - E g), psi+- = (1/2) M^-1 (g +- h), Z+ = psi+, Z- = Delta psi-.
__global__ void zpm_kernel(PartArgs a) {
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const int d = a.d, R = 4 * a.n_in;
    const long long total = (long long)a.batch * R * d;
    if (idx >= total) return;
    const int i = (int)(idx % d);
    const int om = (int)(idx / ((long long)R * d));
    const int col = (int)((idx / d) % R);
    const double mu = a.mu_eff[(size_t)om * a.n_in + col / 4];
    const double g = a.g[idx];
    const double h = mu * (a.sp[idx] - a.eg[idx]);
    const double hm = 0.5 * (1.0 / a.mdiag[i]);
    const double pp = hm * (g + h), pm = hm * (g - h);
    a.zp[idx] = pp;
    a.zm[idx] = ((i & 3) >= 2) ? -pm : pm;
}

// System residual (particular.cpp:84-92): |(FE - sigma) g - rhs| against
// 1e-8 (|rhs| + |FE - sigma| |g|); |FE - sigma| bounded by max|FE| + sigma.
__global__ void part_residual_kernel(PartArgs a, bool final) {
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int d = a.d, R = 4 * a.n_in;
    if (gw >= a.batch * R) return;
    const int om = gw / R, col = gw % R;
    const double sg = a.sigma[2 * ((size_t)om * R + col)];
    const double mu = a.mu_eff[(size_t)om * a.n_in + col / 4];
    const size_t base = ((size_t)om * R + col) * d;
    double rmax = 0.0, bmax = 0.0, gmax = 0.0, balmax = 0.0, xmax = 0.0;
    bool finite = true;
    for (int i = lane; i < d; i += 32) {
        const double g = a.g[base + i], sp = a.sp[base + i], sm = a.sm[base + i];
        const double eg = a.eg[base + i], feg = a.feg[base + i], rhs = a.rhs[base + i];
        const double r = feg - sg * g - rhs;
        finite = finite && isfinite(g);
        rmax = fmax(rmax, fabs(r));
        bmax = fmax(bmax, fabs(rhs));
        gmax = fmax(gmax, fabs(g));
        // unreduced balance M^-1 x - z/mu0 + Op z (particular.cpp:86-99), the 8N
        // operator applied through E and F: with F h = mu0 (F s+ - F E g) and
        // F s+ = rhs + s-/mu0, its upper half and the D-flipped lower half are
        //   (x+ - (E g + F h)/2)/m - psi+/mu0,  (D x- - (E g - F h)/2)/m + psi-/mu0
        const double inv_m = 1.0 / a.mdiag[i];
        const double fh = mu * rhs + sm - mu * feg;
        const double xp = 0.5 * (sp + sm), dxm = 0.5 * (sp - sm);
        const double psip = a.zp[base + i];
        const double psim = ((i & 3) >= 2) ? -a.zm[base + i] : a.zm[base + i];
        const double up = (xp - 0.5 * (eg + fh)) * inv_m - psip / mu;
        const double lo = (dxm - 0.5 * (eg - fh)) * inv_m + psim / mu;
        balmax = fmax(balmax, fmax(fabs(up), fabs(lo)));
        xmax = fmax(xmax, fmax(fabs(xp), fabs(dxm)) * inv_m);
    }
    rmax = warp_max(rmax);
    bmax = warp_max(bmax);
    gmax = warp_max(gmax);
    balmax = warp_max(balmax);
    xmax = warp_max(xmax);
    finite = __all_sync(0xffffffffu, finite);
    if (lane == 0 && !final) {
        if (xmax > 0.0) {
            atomic_max_double(&a.status->part_check, balmax / xmax);
            if (a.part_slot) atomic_max_double(&a.part_slot[om], balmax / xmax);
        }
        return;
    }
    if (lane == 0) {
        const int m = a.order_index ? a.order_index[om] : om;
        const double scale = bmax + (a.femax[om] + sg) * gmax;
        const double rel = scale > 0.0 ? rmax / scale : 0.0;
        atomic_max_double(&a.status->max_particular_residual, rel);
        if (!finite || rmax > 1e-8 * fmax(scale, 1e-300))
            report_failure(a.status, kFailParticular, 2, m, a.mu_in[col / 4], rel);
        // a zero source skips the solve and its checks (particular.cpp:39-41)
        if (xmax > 0.0) {
            const double bal = balmax / xmax;
            atomic_max_double(&a.status->max_balance_residual, bal);
            if (!(bal <= 1e-6)) report_failure(a.status, kFailBalance, 2, m, bal);
        }
    }
}

// Iterative-refinement residual of the Schur-form solve, in place into W:
// W = rhs - ((F E) g - sigma g), with F E g = F (E g) from the GEMMs (true
// operator, not the Schur form).
__global__ void refine_residual_kernel(PartArgs a, double* W) {
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const int d = a.d, R = 4 * a.n_in;
    const long long total = (long long)a.batch * R * d;
    if (idx >= total) return;
    const int om = (int)(idx / ((long long)R * d));
    const int col = (int)((idx / d) % R);
    const double sg = a.sigma[2 * ((size_t)om * R + col)];
    W[idx] = (a.part_on && !a.part_on[om]) ? 0.0 : a.rhs[idx] - (a.feg[idx] - sg * a.g[idx]);
}

__global__ void part_decide_kernel(PartArgs a, double target, int first, int* count) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= a.batch) return;
    const double cur = a.part_slot[b];
    const int on = a.part_on[b] && cur > target && (first || cur < 0.5 * a.part_prev[b]);
    a.part_on[b] = on;
    a.part_prev[b] = cur;
    a.part_slot[b] = 0.0;  // ready for the next interim residual
    if (on) atomicAdd(count, 1);
}

}  // namespace

void launch_part_refine_residual(const PartArgs& a, double* W, cudaStream_t st) {
    const long long total = (long long)a.batch * 4 * a.n_in * a.d;
    refine_residual_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(a, W);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

void launch_dither(const PartArgs& a, cudaStream_t st) {
    const long long warps = (long long)a.batch * a.n_in;
    dither_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(a);
    VRTE_CUDA_CHECK(cudaGetLastError());
}
void launch_part_rhs(const PartArgs& a, cudaStream_t st) {
    const long long total = (long long)a.batch * 4 * a.n_in * a.d;
    rhs_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(a);
    VRTE_CUDA_CHECK(cudaGetLastError());
}
void launch_zpm(const PartArgs& a, cudaStream_t st) {
    const long long total = (long long)a.batch * 4 * a.n_in * a.d;
    zpm_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(a);
    VRTE_CUDA_CHECK(cudaGetLastError());
}
void launch_part_residual(const PartArgs& a, cudaStream_t st, bool final) {
    const long long warps = (long long)a.batch * 4 * a.n_in;
    part_residual_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(a, final);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

void launch_part_decide(const PartArgs& a, double target, bool first, int* count, cudaStream_t st) {
    VRTE_CUDA_CHECK(cudaMemsetAsync(count, 0, sizeof(int), st));
    part_decide_kernel<<<(a.batch + 127) / 128, 128, 0, st>>>(a, target, first ? 1 : 0, count);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace vrte
