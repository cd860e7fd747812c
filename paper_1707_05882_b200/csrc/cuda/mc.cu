// mc.cu -- polarized Monte Carlo tracer on the GPU (the
// statistical cross-check of the discrete-ordinate path): mc.cpp:1-315,
// kernel.cpp:147-186 (scatter matrix, intensity phase function),
// rotation.cpp:9-68 (meridian-frame Stokes rotations), boundary.cpp:37-71
// (Mueller-table base).
//
// One thread per photon with the reference's per-photon stream (splitmix64-
// seeded xoshiro256++, stream = photon index), so a photon's random sequence is
// the reference's; trajectories agree with it as long as libm and CUDA's
// transcendental functions round alike (they may differ in the last ulp, so
// agreement is statistical).  The intensity phase function is tabulated on the
// device (2048-cell inverse CDF, mc.cpp:47-88), the scattering matrix is summed
// per event by the Wigner-d recurrences (no tables).  Tallies are deterministic
// for a fixed (material, photons, seed, bins): each CTA reduces its photons'
// exit records per bin in photon order, then the CTA grids are summed in CTA
// order.
#include <cstdint>

#include "kernels.cuh"

namespace vrte {
namespace {

constexpr int kCells = 2048;
constexpr int kPhotonsPerCta = 128;

struct Rng {  // mc.cpp:11-45
    uint64_t s[4];
    __device__ static uint64_t splitmix(uint64_t& x) {
        x += 0x9e3779b97f4a7c15ull;
        uint64_t z = x;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    __device__ Rng(uint64_t seed, uint64_t stream) {
        uint64_t x = seed ^ (0x9e3779b97f4a7c15ull * (stream + 1));
        for (int i = 0; i < 4; ++i) s[i] = splitmix(x);
    }
    __device__ static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
    __device__ uint64_t next() {
        const uint64_t result = rotl(s[0] + s[3], 23) + s[0];
        const uint64_t t = s[1] << 17;
        s[2] ^= s[0];
        s[3] ^= s[1];
        s[1] ^= s[2];
        s[0] ^= s[3];
        s[2] ^= t;
        s[3] = rotl(s[3], 45);
        return result;
    }
    __device__ double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }
};

// wigner.cpp:11-27
__device__ double wigner_start_mc(int m, int n, double x) {
    const int lmin = max(abs(m), abs(n));
    const int a = abs(m - n), b = abs(m + n);
    double lf = 0.0;
    for (int k = 2; k <= 2 * lmin; ++k) lf += log((double)k);
    for (int k = 2; k <= a; ++k) lf -= log((double)k);
    for (int k = 2; k <= b; ++k) lf -= log((double)k);
    double v = exp(0.5 * lf - lmin * log(2.0));
    v *= pow(fmax(0.0, 1.0 - x), 0.5 * a) * pow(fmax(0.0, 1.0 + x), 0.5 * b);
    if (n < m && ((m - n) & 1)) v = -v;
    return v;
}

// Upward recurrence of d^l_{mn}(x) (wigner.cpp:31-62), one step at a time.
struct Wig {
    int m, n, lmin;
    double prev, cur;
    __device__ void init(int m_, int n_, int lmax, double x) {
        m = m_;
        n = n_;
        lmin = max(abs(m), abs(n));
        prev = 0.0;
        cur = lmin <= lmax ? wigner_start_mc(m, n, x) : 0.0;
    }
    // value at l (call with l = 0, 1, 2, ... in order)
    __device__ double at(int l, double x) {
        if (l < lmin) return 0.0;
        if (l == lmin) return cur;
        const int lm = l - 1;
        double next;
        if (lm == 0) {
            next = x;
        } else {
            const double lp = lm + 1.0;
            const double c0 = lm * sqrt((lp * lp - (double)m * m) * (lp * lp - (double)n * n));
            const double c1 = (2.0 * lm + 1.0) * (lm * lp * x - (double)m * n);
            const double c2 = lp * sqrt(((double)lm * lm - (double)m * m) * ((double)lm * lm - (double)n * n));
            next = (c1 * cur - c2 * prev) / c0;
        }
        prev = cur;
        cur = next;
        return next;
    }
};

// kernel.cpp:179-186 at the 2049 cell edges of every layer
__global__ void mc_phase_kernel(McArgs a, double* edge_val) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= a.n_layers * (kCells + 1)) return;
    const int i = idx % (kCells + 1), p = idx / (kCells + 1);
    const double x = i == 0 ? -1.0 : fmin(-1.0 + (2.0 / kCells) * i, 1.0);
    const double* gk = a.greek + (size_t)a.medium[p] * a.Lc * 6;
    Wig w;
    w.init(0, 0, a.Lc - 1, x);
    double a1 = 0.0;
    for (int l = 0; l < a.Lc; ++l) a1 += gk[6 * l] * w.at(l, x);
    edge_val[idx] = fmax(0.0, a1);
}
// trapezoid CDF, normalized (mc.cpp:52-70); thread per layer, sequential like the reference
__global__ void mc_cdf_kernel(McArgs a, const double* edge_val) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= a.n_layers) return;
    const double dx = 2.0 / kCells;
    const double* v = edge_val + (size_t)p * (kCells + 1);
    double* cdf = a.cdf + (size_t)p * (kCells + 1);
    double* den = a.density + (size_t)p * kCells;
    double total = 0.0;
    cdf[0] = 0.0;
    for (int i = 0; i < kCells; ++i) {
        total += 0.5 * (v[i] + v[i + 1]) * dx;
        cdf[i + 1] = total;
    }
    if (!(total > 0.0)) {
        atomicCAS(a.fail, 0, 1);
        return;
    }
    for (int i = 0; i <= kCells; ++i) cdf[i] /= total;
    for (int i = 0; i < kCells; ++i) den[i] = (cdf[i + 1] - cdf[i]) / dx;
}

struct V3 {
    double x, y, z;
};
__device__ inline V3 mk3(double x, double y, double z) { return {x, y, z}; }
__device__ inline double dot3(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ inline V3 cross3(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
__device__ inline V3 norm3(V3 a) {
    const double n = sqrt(dot3(a, a));
    return {a.x / n, a.y / n, a.z / n};
}
__device__ inline double reduce_az(double phi) {  // types.cpp:7-12
    double r = fmod(phi, 2.0 * kPi);
    if (r < 0.0) r += 2.0 * kPi;
    return r;
}
__device__ inline V3 unit_dir(double mu, double phi) {  // types.hpp:94-97 (phi reduced by the ctor)
    phi = reduce_az(phi);
    const double s = sqrt(fmax(0.0, 1.0 - mu * mu));
    return {s * cos(phi), s * sin(phi), mu};
}
__device__ V3 rotate_direction(V3 d, double ct, double psi) {  // mc.cpp:107-114
    const double st = sqrt(fmax(0.0, 1.0 - ct * ct));
    const V3 ax = fabs(d.z) < 0.99 ? mk3(0, 0, 1) : mk3(1, 0, 0);
    const V3 t1 = norm3(cross3(d, ax)), t2 = cross3(d, t1);
    const double c = cos(psi), s = sin(psi);
    return norm3(mk3(ct * d.x + st * (c * t1.x + s * t2.x), ct * d.y + st * (c * t1.y + s * t2.y),
                     ct * d.z + st * (c * t1.z + s * t2.z)));
}
__device__ inline V3 nudge_off_pole(V3 d) {  // rotation.cpp:9-15
    if (1.0 - fabs(d.z) < 1e-12) {
        d.x += 1e-9;
        d = norm3(d);
    }
    return d;
}
__device__ void meridian(V3 dir, V3& l, V3& r) {  // rotation.cpp:19-29
    const V3 d = nudge_off_pole(dir);
    const double s = sqrt(fmax(1e-300, d.x * d.x + d.y * d.y));
    const double cphi = d.x / s, sphi = d.y / s;
    l = mk3(d.z * cphi, d.z * sphi, -s);
    r = mk3(-sphi, cphi, 0.0);
}
__device__ void scatter_geometry(V3 din, V3 dout, double& c, double& eta_in, double& eta_out) {  // rotation.cpp:42-68
    din = nudge_off_pole(din);
    dout = nudge_off_pole(dout);
    c = fmin(fmax(dot3(din, dout), -1.0), 1.0);
    if (1.0 - fabs(c) < 1e-12) {
        const V3 pr = fabs(dout.z) < 0.9 ? mk3(0, 0, 1) : mk3(1, 0, 0);
        dout = norm3(mk3(dout.x + 1e-9 * pr.x, dout.y + 1e-9 * pr.y, dout.z + 1e-9 * pr.z));
        c = fmin(fmax(dot3(din, dout), -1.0), 1.0);
    }
    const V3 lin = norm3(mk3(dout.x - c * din.x, dout.y - c * din.y, dout.z - c * din.z));
    const V3 lout = norm3(mk3(c * dout.x - din.x, c * dout.y - din.y, c * dout.z - din.z));
    const V3 rout = cross3(dout, lout);
    V3 il, ir, ol, orr;
    meridian(din, il, ir);
    meridian(dout, ol, orr);
    eta_in = atan2(dot3(lin, ir), dot3(lin, il));
    eta_out = atan2(dot3(ol, rout), dot3(ol, lout));
}

// base_row_at (boundary.cpp:37-71) on the table's own Gauss nodes
__device__ void base_row(const McArgs& a, double mu_out, double mu_in, double R[16]) {
    for (int e = 0; e < 16; ++e) R[e] = 0.0;
    if (a.base_type == 1) {
        R[0] = 2.0 * a.rho;
        return;
    }
    const int n = a.table_n;
    const double* nd = a.table_nodes;
    auto interp = [&](double mu, int& lo, double& w) {
        if (mu <= nd[0]) {
            lo = 0;
            w = 0.0;
            return;
        }
        if (mu >= nd[n - 1]) {
            lo = n - 2 >= 0 ? n - 2 : 0;
            w = n >= 2 ? 1.0 : 0.0;
            return;
        }
        lo = 0;
        while (lo + 1 < n && nd[lo + 1] < mu) ++lo;
        w = (mu - nd[lo]) / (nd[lo + 1] - nd[lo]);
    };
    int li, lj;
    double wi, wj;
    interp(mu_out, li, wi);
    interp(mu_in, lj, wj);
    const int i1 = min(li + 1, n - 1), j1 = min(lj + 1, n - 1);
    const double* t00 = a.table + ((size_t)li * n + lj) * 16;
    const double* t01 = a.table + ((size_t)li * n + j1) * 16;
    const double* t10 = a.table + ((size_t)i1 * n + lj) * 16;
    const double* t11 = a.table + ((size_t)i1 * n + j1) * 16;
    for (int e = 0; e < 16; ++e)
        R[e] = (1 - wi) * (1 - wj) * t00[e] + (1 - wi) * wj * t01[e] + wi * (1 - wj) * t10[e] + wi * wj * t11[e];
}

// One photon (mc.cpp:140-231); writes its exit record (bin or -1, weight).
__global__ void __launch_bounds__(kPhotonsPerCta) mc_trace_kernel(McArgs a) {
    __shared__ int s_bin[kPhotonsPerCta];
    __shared__ double s_w[kPhotonsPerCta][4];
    const int t = threadIdx.x;
    const uint64_t ph = a.ph0 + (uint64_t)blockIdx.x * kPhotonsPerCta + t;
    int bin = -1;
    double w[4] = {0.0, 0.0, 0.0, 0.0};
    if (ph < a.photons) {
        Rng rng(a.seed, ph);
        double tau = 0.0;
        V3 dir = unit_dir(-a.mu0, a.phi0);
        for (int c = 0; c < 4; ++c) w[c] = a.stokes[c];
        int events = 0;
        bool done = false;
        for (int bounce = 0; bounce < 100000 && !done; ++bounce) {
            const double step = -log(fmax(1e-300, 1.0 - rng.uniform()));
            const double mu = dir.z;
            if (mu == 0.0) break;
            const double dtau = -mu * step;
            if (mu > 0.0 && tau + dtau < 0.0) {
                if (events > 0) bin = 0;  // top exit
                break;
            }
            if (mu < 0.0 && tau + dtau > a.total) {
                if (a.base_type == 0) {
                    if (events > 0) bin = 1;  // bottom exit
                    break;
                }
                tau = a.total;
                if (a.base_type == 1) {
                    const double refl = a.rho * w[0];
                    if (refl <= 0.0) break;
                    w[0] = refl;
                    w[1] = w[2] = w[3] = 0.0;
                } else {
                    const double mu_in = -dir.z;
                    const double mu_up = sqrt(fmax(rng.uniform(), 1e-300));
                    const double phi = 2.0 * kPi * rng.uniform();
                    double R[16], nw[4];
                    base_row(a, mu_up, mu_in, R);
                    for (int r = 0; r < 4; ++r)
                        nw[r] = 0.5 * (R[4 * r] * w[0] + R[4 * r + 1] * w[1] + R[4 * r + 2] * w[2] + R[4 * r + 3] * w[3]);
                    for (int r = 0; r < 4; ++r) w[r] = nw[r];
                    if (w[0] <= 0.0) break;
                    dir = unit_dir(fmax(mu_up, 1e-9), phi);
                    ++events;
                    continue;
                }
                const double mu_up = sqrt(fmax(rng.uniform(), 1e-300));
                const double phi = 2.0 * kPi * rng.uniform();
                dir = unit_dir(fmax(mu_up, 1e-9), phi);
                ++events;
                continue;
            }
            tau += dtau;
            int li = a.n_layers - 1;  // mc.cpp:100-105
            while (li > 0 && tau < a.tops[li]) --li;
            const double omega = a.omega[a.medium[li]];
            if (omega <= 0.0) break;  // absorbed
            // inverse-CDF sample (mc.cpp:72-87)
            const double u = rng.uniform();
            const double* cdf = a.cdf + (size_t)li * (kCells + 1);
            int lo = 0, hi = kCells;
            while (hi - lo > 1) {
                const int mid = (lo + hi) / 2;
                if (cdf[mid] <= u)
                    lo = mid;
                else
                    hi = mid;
            }
            const double mass = cdf[lo + 1] - cdf[lo];
            const double frac = mass > 0.0 ? (u - cdf[lo]) / mass : 0.5;
            const double ct = fmin(fmax(-1.0 + (2.0 / kCells) * (lo + frac), -1.0), 1.0);
            const double pdf = fmax(a.density[(size_t)li * kCells + lo], 1e-300);
            const double psi = 2.0 * kPi * rng.uniform();
            const V3 nd = rotate_direction(dir, ct, psi);
            double c2, ein, eout;
            scatter_geometry(dir, nd, c2, ein, eout);
            // scatter matrix at c2 (kernel.cpp:147-177)
            const double* gk = a.greek + (size_t)a.medium[li] * a.Lc * 6;
            Wig w00, w02, w22, w2m;
            w00.init(0, 0, a.Lc - 1, c2);
            w02.init(0, 2, a.Lc - 1, c2);
            w22.init(2, 2, a.Lc - 1, c2);
            w2m.init(2, -2, a.Lc - 1, c2);
            double a1 = 0, a4 = 0, b1 = 0, b2 = 0, apc = 0, amc = 0;
            for (int l = 0; l < a.Lc; ++l) {
                const double d00 = w00.at(l, c2), d02 = w02.at(l, c2), d22 = w22.at(l, c2), d2m = w2m.at(l, c2);
                const double* g = gk + 6 * l;  // beta alpha gamma delta eps zeta
                a1 += g[0] * d00;
                a4 += g[3] * d00;
                b1 += g[2] * d02;
                b2 -= g[4] * d02;
                apc += (g[1] + g[5]) * d22;
                amc += (g[1] - g[5]) * d2m;
            }
            const double a2 = 0.5 * (apc + amc), a3 = 0.5 * (apc - amc);
            // Z = L(eta_out) F L(eta_in), applied to w
            const double ci = cos(2.0 * ein), si = sin(2.0 * ein), co = cos(2.0 * eout), so = sin(2.0 * eout);
            const double q1 = ci * w[1] + si * w[2], u1 = -si * w[1] + ci * w[2];  // L(eta_in) w
            const double f0 = a1 * w[0] + b1 * q1, f1 = b1 * w[0] + a2 * q1;      // F
            const double f2 = a3 * u1 + b2 * w[3], f3 = -b2 * u1 + a4 * w[3];
            const double f = omega / (2.0 * pdf);
            w[0] = f * f0;
            w[1] = f * (co * f1 + so * f2);  // L(eta_out)
            w[2] = f * (-so * f1 + co * f2);
            w[3] = f * f3;
            dir = nd;
            ++events;
            if (w[0] <= 0.0) break;
            if (w[0] < 1e-4 * a.stokes[0]) {  // roulette (mc.cpp:116-117, 210-214)
                if (rng.uniform() * 10.0 > 1.0) break;
                for (int c = 0; c < 4; ++c) w[c] *= 10.0;
            }
        }
        if (bin >= 0) {  // tally bin (mc.cpp:124-138)
            const double mu = fabs(dir.z);
            if (mu <= 0.0) {
                bin = -1;
            } else {
                const double phi = reduce_az(atan2(dir.y, dir.x));
                const int iz = min((int)(mu * a.zb), a.zb - 1);
                const int ia = min((int)(phi / (2.0 * kPi) * a.ab), a.ab - 1);
                bin = (bin * a.zb + iz) * a.ab + ia;
            }
        }
    }
    s_bin[t] = bin;
    for (int c = 0; c < 4; ++c) s_w[t][c] = w[c];
    __syncthreads();
    // per-CTA grid, photons in order (deterministic)
    const int nbins = 2 * a.zb * a.ab;
    double* grid = a.cta_grid + (size_t)blockIdx.x * nbins * 9;
    for (int b = t; b < nbins; b += kPhotonsPerCta) {
        double s[4] = {0, 0, 0, 0}, q[4] = {0, 0, 0, 0};
        int h = 0;
        for (int p = 0; p < kPhotonsPerCta; ++p)
            if (s_bin[p] == b) {
                for (int c = 0; c < 4; ++c) {
                    s[c] += s_w[p][c];
                    q[c] += s_w[p][c] * s_w[p][c];
                }
                ++h;
            }
        for (int c = 0; c < 4; ++c) {
            grid[(size_t)b * 9 + c] = s[c];
            grid[(size_t)b * 9 + 4 + c] = q[c];
        }
        grid[(size_t)b * 9 + 8] = (double)h;
    }
}

// CTA grids summed in CTA order per (bin, quantity), added to the running total
__global__ void mc_reduce_kernel(McArgs a, int n_cta) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    const int nbins = 2 * a.zb * a.ab;
    if (idx >= nbins * 9) return;
    double acc = 0.0;
    for (int c = 0; c < n_cta; ++c) acc += a.cta_grid[(size_t)c * nbins * 9 + idx];
    a.out[idx] += acc;
}

}  // namespace

int mc_photons_per_cta() { return kPhotonsPerCta; }

int launch_mc_tables(McArgs a, double* edge_scratch, cudaStream_t st) {
    const int ne = a.n_layers * (kCells + 1);
    mc_phase_kernel<<<(ne + 127) / 128, 128, 0, st>>>(a, edge_scratch);
    mc_cdf_kernel<<<1, 32, 0, st>>>(a, edge_scratch);
    VRTE_CUDA_CHECK(cudaGetLastError());
    return 2;
}

int launch_mc_chunk(McArgs a, uint64_t n, cudaStream_t st) {
    const int n_cta = (int)((n + kPhotonsPerCta - 1) / kPhotonsPerCta);
    a.photons = a.ph0 + n;  // photons >= this index are idle in this launch
    mc_trace_kernel<<<n_cta, kPhotonsPerCta, 0, st>>>(a);
    const int nq = 2 * a.zb * a.ab * 9;
    mc_reduce_kernel<<<(nq + 127) / 128, 128, 0, st>>>(a, n_cta);
    VRTE_CUDA_CHECK(cudaGetLastError());
    return 2;
}

}  // namespace vrte

// ------------------------------------------------------------------ C ABI
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/vrte/vrte_cuda.h"

namespace vrte {
namespace {
struct DBuf {
    void* p = nullptr;
    ~DBuf() {
        if (p) cudaFree(p);
    }
    template <typename T>
    T* alloc(size_t n) {
        VRTE_CUDA_CHECK(cudaMalloc(&p, sizeof(T) * (n ? n : 1)));
        return static_cast<T*>(p);
    }
};
}  // namespace
}  // namespace vrte

extern "C" int32_t vrte_cuda_mc_trace(const vrte_cuda_mc* mc, double* sum, double* sum_sq, uint64_t* hits,
                                      vrte_cuda_result* result) {
    using namespace vrte;
    auto fill = [&](int code, const std::string& msg) {
        if (result) {
            result->status = code;
            std::snprintf(result->message, sizeof result->message, "%s", msg.c_str());
        }
        return code;
    };
    if (!mc || !sum || !sum_sq || !hits) return fill(5, "null argument");
    try {
        if (mc->device >= 0) VRTE_CUDA_CHECK(cudaSetDevice(mc->device));
        cudaStream_t st;
        VRTE_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        const int P = mc->n_layers, nbins = 2 * mc->zb * mc->ab;
        const uint64_t chunk = 1ull << 18;  // photons per launch (2048 CTAs: one wave)
        const uint64_t n_cta = (std::min<uint64_t>(chunk, mc->photons) + mc_photons_per_cta() - 1) / mc_photons_per_cta();
        DBuf bg, bm, bo, bt, btab, bnod, bcdf, bden, bfail, bgrid, bout, bedge;
        double* greek = bg.alloc<double>((size_t)P * mc->Lc * 6);
        int* med = bm.alloc<int>(P);
        double* om = bo.alloc<double>(P);
        double* tops = bt.alloc<double>(P);
        std::vector<int> mh(P);
        for (int p = 0; p < P; ++p) mh[p] = p;
        VRTE_CUDA_CHECK(cudaMemcpyAsync(greek, mc->greek, sizeof(double) * P * mc->Lc * 6, cudaMemcpyHostToDevice, st));
        VRTE_CUDA_CHECK(cudaMemcpyAsync(med, mh.data(), sizeof(int) * P, cudaMemcpyHostToDevice, st));
        VRTE_CUDA_CHECK(cudaMemcpyAsync(om, mc->omega, sizeof(double) * P, cudaMemcpyHostToDevice, st));
        VRTE_CUDA_CHECK(cudaMemcpyAsync(tops, mc->tops, sizeof(double) * P, cudaMemcpyHostToDevice, st));
        McArgs a{};
        a.photons = mc->photons;
        a.seed = mc->seed;
        a.zb = mc->zb;
        a.ab = mc->ab;
        a.n_layers = P;
        a.Lc = mc->Lc;
        a.base_type = mc->base_type;
        a.table_n = mc->table_n;
        a.mu0 = mc->mu0;
        a.phi0 = mc->phi0;
        a.rho = mc->rho;
        a.total = mc->total;
        for (int c = 0; c < 4; ++c) a.stokes[c] = mc->stokes[c];
        a.greek = greek;
        a.medium = med;
        a.omega = om;
        a.tops = tops;
        if (mc->base_type == 2) {
            double* tab = btab.alloc<double>((size_t)mc->table_n * mc->table_n * 16);
            double* nod = bnod.alloc<double>(mc->table_n);
            VRTE_CUDA_CHECK(cudaMemcpyAsync(tab, mc->table, sizeof(double) * mc->table_n * mc->table_n * 16,
                                            cudaMemcpyHostToDevice, st));
            VRTE_CUDA_CHECK(cudaMemcpyAsync(nod, mc->table_nodes, sizeof(double) * mc->table_n,
                                            cudaMemcpyHostToDevice, st));
            a.table = tab;
            a.table_nodes = nod;
        }
        a.cdf = bcdf.alloc<double>((size_t)P * (kCells + 1));
        a.density = bden.alloc<double>((size_t)P * kCells);
        a.fail = bfail.alloc<int>(1);
        a.cta_grid = bgrid.alloc<double>((size_t)n_cta * nbins * 9);
        a.out = bout.alloc<double>((size_t)nbins * 9);
        double* edge = bedge.alloc<double>((size_t)P * (kCells + 1));
        VRTE_CUDA_CHECK(cudaMemsetAsync(a.fail, 0, sizeof(int), st));
        VRTE_CUDA_CHECK(cudaMemsetAsync(a.out, 0, sizeof(double) * nbins * 9, st));
        uint64_t launches = launch_mc_tables(a, edge, st);
        int fail = 0;
        VRTE_CUDA_CHECK(cudaMemcpyAsync(&fail, a.fail, sizeof(int), cudaMemcpyDeviceToHost, st));
        VRTE_CUDA_CHECK(cudaStreamSynchronize(st));
        if (fail) {
            cudaStreamDestroy(st);
            throw std::domain_error("mc: intensity phase function has no positive mass");
        }
        for (uint64_t ph0 = 0; ph0 < mc->photons; ph0 += chunk) {
            a.ph0 = ph0;
            launches += launch_mc_chunk(a, std::min<uint64_t>(chunk, mc->photons - ph0), st);
        }
        std::vector<double> h((size_t)nbins * 9);
        VRTE_CUDA_CHECK(cudaMemcpyAsync(h.data(), a.out, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, st));
        VRTE_CUDA_CHECK(cudaStreamSynchronize(st));
        cudaStreamDestroy(st);
        for (int b = 0; b < nbins; ++b) {
            for (int c = 0; c < 4; ++c) {
                sum[(size_t)b * 4 + c] = h[(size_t)b * 9 + c];
                sum_sq[(size_t)b * 4 + c] = h[(size_t)b * 9 + 4 + c];
            }
            hits[b] = (uint64_t)h[(size_t)b * 9 + 8];
        }
        if (result) {
            result->kernel_launches = launches;
            result->status = 0;
            result->message[0] = 0;
        }
        return 0;
    } catch (const std::domain_error& e) {
        return fill(2, e.what());
    } catch (const std::exception& e) {
        return fill(3, e.what());
    }
}
