// refine.cu -- eigenpair refinement replacing the reference's polish loops
// (homogeneous.cpp:216-268).
//
// The reference re-factors a dense complex LU of F E - sigma (and of the 8N
// operator) for every marginal mode; at N = 64 that is most modes.  Inverse
// iteration through the Schur form cannot do the same job: the Schur form
// carries exactly the normwise QR backward error (~eps |FE| ~ 1e-9) that
// limits the raw eigenvectors.  Instead each mode is refined by Newton's
// method on the 8N eigenproblem  Op v = rho v,  rho = 1/nu  (bordered form,
// normalization v_s = 1 at the largest component):
//     (Op - rho) dv - drho v = -(Op v - rho v),   dv_s = 0,
// with the TRUE residual from the reduced operators (two GEMMs, accurate to
// eps |E| |v|) and the correction solved approximately through the Schur form
// via the 8N -> half-size folding
//     (FE - s^2) M u = s M(a + b') - F M(a - b'),  M t = -(E M u + M(a - b'))/s,
// (w = [p; Delta q'], u = p + q', t = p - q').  The approximate Jacobian
// makes the iteration converge linearly with rate ~ eps|FE|/gap, so 3 steps
// reach ~1e-12 residuals (the reference stops at 5e-10).  All modes of all
// (medium, order) pairs are refined in lock-step: every step is four batched
// GEMMs of width 2d, one of width d, and one warp-per-column back substitution.
#include "refine.cuh"

namespace vrte {
namespace {

// Per-mode relative offset of the Newton shift s = rho (1 + shift_j).
// Within a cluster of eigenvalues the approximate (Schur-form) Jacobian is
// accurate only to the QR backward error eps_j ~ eps |FE| / |lambda_j|.  With
// gap_j the relative distance to the nearest other eigenvalue:
//   gap_j > 100 eps_j (resolvable)   -> shift = 1e-3 gap_j: within-cluster
//                                       directions contract by ~1e-3 per step;
//   otherwise (unresolvable cluster) -> shift = 1e3 max(gap_j, eps_j): they
//                                       stagnate (factor 1 + 1e-3) instead of
//                                       being amplified by the Schur-form error.
// Every other direction contracts by ~shift/gap_other per step.  (A fixed
// shift always hits some cluster whose spread is comparable to it.)
__global__ void shift_kernel(RefineArgs a) {
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int d = a.d;
    if (gw >= a.batch * d) return;
    const int b = gw / d, j = gw % d;
    const size_t vb = (size_t)b * d;
    const cplx lj = cmk(a.wr[vb + j], a.wi[vb + j]);
    const double al = cabs_(lj);
    double g = 1e300;
    for (int k = lane; k < d; k += 32) {
        if (k == j) continue;
        g = fmin(g, cabs_(cmk(a.wr[vb + k], a.wi[vb + k]) - lj));
    }
    g = -warp_max(-g);
    if (lane == 0) {
        const double gap = al > 0.0 ? g / al : 1e300;
        const double epsq = al > 0.0 ? 2.220446049250313e-16 * a.femax[b] / al : 1e300;
        double sh = gap > 100.0 * epsq ? fmax(1e-3 * gap, 1e-14) : fmin(1e3 * fmax(gap, epsq), 1e-4);
        a.shift[vb + j] = 0.5 * sh;  // rho = lambda^-1/2 halves relative offsets
    }
}

struct MRef {
    int b, j, d;
    bool pair;
    size_t vb, cb;   // vector base (b*d), column base in a d x d packed matrix
    size_t cb2;      // column base in a d x 2d packed matrix (set A)
};

__device__ bool mref(int gw, const RefineArgs& a, MRef& m) {
    const int d = a.d;
    if (gw >= a.batch * d) return false;
    m.b = gw / d;
    m.j = gw % d;
    m.d = d;
    m.vb = (size_t)m.b * d;
    const double w = a.wi[m.vb + m.j];
    if (w < 0.0) return false;
    m.pair = w > 0.0;
    m.cb = (size_t)m.b * d * d + (size_t)m.j * d;
    m.cb2 = (size_t)m.b * 2 * d * d + (size_t)m.j * d;
    return true;
}
__device__ inline cplx ld(const double* p, size_t cb, int d, bool pair, int i) {
    return cmk(p[cb + i], pair ? p[cb + d + i] : 0.0);
}
__device__ inline void st(double* p, size_t cb, int d, bool pair, int i, cplx v) {
    p[cb + i] = v.re;
    if (pair) p[cb + d + i] = v.im;
}
// set B of a d x 2d buffer starts d columns after set A
__device__ inline size_t setb(const MRef& m) { return m.cb2 + (size_t)m.d * m.d; }

__device__ inline bool active(const RefineArgs& a, const MRef& m) {
    return (a.flags[m.vb + m.j] & 1) == 0;  // bit0: conservative (never refined)
}

// Normalize v = [p; q'] so that its largest component is exactly 1, then
// write the residual GEMM inputs ab_sum = M(p + q'), ab_dif = M(q' - p).
__global__ void normalize_kernel(RefineArgs a) {
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    MRef m;
    if (!mref(gw, a, m)) return;
    if (a.slot_on && !a.slot_on[m.b]) return;
    const int d = m.d;
    if (!active(a, m)) {
        // conservative modes: only refresh the residual inputs
        for (int i = lane; i < d; i += 32) {
            const cplx p = ld(a.psi_p, m.cb, d, m.pair, i), q = ld(a.psi_m, m.cb, d, m.pair, i);
            st(a.ab_sum, m.cb, d, m.pair, i, a.mdiag[i] * (p + q));
            st(a.ab_dif, m.cb, d, m.pair, i, a.mdiag[i] * (q - p));
        }
        return;
    }
    double best = -1.0;
    int bi = 0;
    for (int i = lane; i < 2 * d; i += 32) {
        const cplx v = i < d ? ld(a.psi_p, m.cb, d, m.pair, i) : ld(a.psi_m, m.cb, d, m.pair, i - d);
        const double av = cabs_(v);
        if (av > best) {
            best = av;
            bi = i;
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
    const cplx vs = bi < d ? ld(a.psi_p, m.cb, d, m.pair, bi) : ld(a.psi_m, m.cb, d, m.pair, bi - d);
    const cplx rvs = cdiv(cmk(1.0, 0.0), vs);  // one complex division per mode, not per element
    __syncwarp();
    for (int i = lane; i < d; i += 32) {
        cplx p = ld(a.psi_p, m.cb, d, m.pair, i) * rvs;
        cplx q = ld(a.psi_m, m.cb, d, m.pair, i) * rvs;
        if (i == bi) p = cmk(1.0, 0.0);  // the normalized component is exactly 1
        if (i + d == bi) q = cmk(1.0, 0.0);
        st(a.psi_p, m.cb, d, m.pair, i, p);
        st(a.psi_m, m.cb, d, m.pair, i, q);
        st(a.ab_sum, m.cb, d, m.pair, i, a.mdiag[i] * (p + q));
        st(a.ab_dif, m.cb, d, m.pair, i, a.mdiag[i] * (q - p));
    }
    if (lane == 0) a.sidx[m.vb + m.j] = bi;
}

// Residual r = Op v - rho v from G1 = E(a+b), G2 = F(b-a); set up the two
// shifted solves (set A: v, set B: r) as alpha = M(x + y'), beta = M(x - y');
// per-column shift s^2, s = rho (1 + shift_j).
__global__ void setup_kernel(RefineArgs a) {
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    MRef m;
    if (!mref(gw, a, m)) return;
    if (a.slot_on && !a.slot_on[m.b]) return;
    const int d = m.d;
    const bool act = active(a, m);
    const size_t kb = (size_t)m.b * 2 * d;
    if (lane == 0) {
        const int k = act ? (m.pair ? 1 : 0) : 2;
        a.kind[kb + m.j] = k;
        a.kind[kb + d + m.j] = k;
        if (m.pair) {
            a.kind[kb + m.j + 1] = 2;
            a.kind[kb + d + m.j + 1] = 2;
        }
        const cplx rho = cmk(a.rho[2 * (m.vb + m.j)], a.rho[2 * (m.vb + m.j) + 1]);
        const cplx s = (1.0 + a.shift[m.vb + m.j]) * rho;
        const cplx s2 = s * s;
        for (int set = 0; set < 2; ++set) {
            a.sigma[2 * (kb + set * d + m.j)] = s2.re;
            a.sigma[2 * (kb + set * d + m.j) + 1] = s2.im;
        }
    }
    if (!act) return;
    const cplx rho = cmk(a.rho[2 * (m.vb + m.j)], a.rho[2 * (m.vb + m.j) + 1]);
    for (int i = lane; i < d; i += 32) {
        const double mu = a.mdiag[i], im = 1.0 / mu;
        const cplx p = ld(a.psi_p, m.cb, d, m.pair, i), q = ld(a.psi_m, m.cb, d, m.pair, i);
        const cplx g1 = ld(a.G1, m.cb, d, m.pair, i), g2 = ld(a.G2, m.cb, d, m.pair, i);
        const cplx rt = (0.5 * im) * (g2 - g1) - rho * p;
        const cplx rb = (0.5 * im) * (g1 + g2) - rho * q;
        st(a.AL, m.cb2, d, m.pair, i, mu * (p + q));
        st(a.BE, m.cb2, d, m.pair, i, mu * (p - q));
        st(a.AL, setb(m), d, m.pair, i, mu * (rt + rb));
        st(a.BE, setb(m), d, m.pair, i, mu * (rt - rb));
    }
}

// RHS = s alpha - F beta (F beta in FB), in place into FB.
__global__ void rhs_kernel(RefineArgs a) {
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    MRef m;
    if (!mref(gw, a, m) || !active(a, m)) return;
    if (a.slot_on && !a.slot_on[m.b]) return;
    const int d = m.d;
    const cplx s = (1.0 + a.shift[m.vb + m.j]) * cmk(a.rho[2 * (m.vb + m.j)], a.rho[2 * (m.vb + m.j) + 1]);
    for (int set = 0; set < 2; ++set) {
        const size_t cb = set ? setb(m) : m.cb2;
        for (int i = lane; i < d; i += 32)
            st(a.FB, cb, d, m.pair, i, s * ld(a.AL, cb, d, m.pair, i) - ld(a.FB, cb, d, m.pair, i));
    }
}

// Unfold both solutions (u~ in UT, E u~ in EU) to (p, q') pairs and take the
// bordered Newton step: drho = b_s / a_s, v <- v - b + drho a, rho += drho.
__global__ void update_kernel(RefineArgs a) {
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    MRef m;
    if (!mref(gw, a, m) || !active(a, m)) return;
    if (a.slot_on && !a.slot_on[m.b]) return;
    const int d = m.d;
    const cplx s = (1.0 + a.shift[m.vb + m.j]) * cmk(a.rho[2 * (m.vb + m.j)], a.rho[2 * (m.vb + m.j) + 1]);
    const int si = a.sidx[m.vb + m.j];
    const cplx rs = cdiv(cmk(1.0, 0.0), s);  // one complex division per mode
    auto unfold = [&](size_t cb, int i, double im, cplx& p, cplx& q) {
        const cplx ut = ld(a.UT, cb, d, m.pair, i);
        const cplx tt = (ld(a.EU, cb, d, m.pair, i) + ld(a.BE, cb, d, m.pair, i)) * rs;
        const cplx u = im * ut, t = cmk(-im * tt.re, -im * tt.im);
        p = 0.5 * (u + t);
        q = 0.5 * (u - t);
    };
    cplx as, bs;
    {
        const int i = si < d ? si : si - d;
        const double im = 1.0 / a.mdiag[i];
        cplx ap, aq, bp, bq;
        unfold(m.cb2, i, im, ap, aq);
        unfold(setb(m), i, im, bp, bq);
        as = si < d ? ap : aq;
        bs = si < d ? bp : bq;
    }
    const cplx dr = cdiv(bs, as);
    bool fin = isfinite(dr.re) && isfinite(dr.im);
    if (!fin) return;  // keep the current pair (the reference's `break` on non-finite)
    // Safeguard: v is normalized to a largest component of 1 and the eigenpair is
    // already close (Schur-form accuracy), so a correction of half the vector (or
    // an eigenvalue move above 1e-3 relative) is the approximate Jacobian failing
    // -- an exactly repeated eigenvalue, whose eigenvectors span a plane the
    // bordered system does not fix -- not a better eigenpair: keep the current pair.
    double dmax = 0.0;
    for (int i = lane; i < d; i += 32) {
        const double im = 1.0 / a.mdiag[i];
        cplx ap, aq, bp, bq;
        unfold(m.cb2, i, im, ap, aq);
        unfold(setb(m), i, im, bp, bq);
        const cplx dp = dr * ap - bp, dq = dr * aq - bq;
        dmax = fmax(dmax, fmax(fmax(fabs(dp.re), fabs(dp.im)), fmax(fabs(dq.re), fabs(dq.im))));
    }
    dmax = warp_max(dmax);
    const cplx rho0 = cmk(a.rho[2 * (m.vb + m.j)], a.rho[2 * (m.vb + m.j) + 1]);
    if (!(dmax <= 0.5) || cabs_(dr) > 1e-3 * cabs_(rho0)) return;
    for (int i = lane; i < d; i += 32) {
        const double im = 1.0 / a.mdiag[i];
        cplx ap, aq, bp, bq;
        unfold(m.cb2, i, im, ap, aq);
        unfold(setb(m), i, im, bp, bq);
        const cplx p = ld(a.psi_p, m.cb, d, m.pair, i), q = ld(a.psi_m, m.cb, d, m.pair, i);
        st(a.psi_p, m.cb, d, m.pair, i, p - bp + dr * ap);
        st(a.psi_m, m.cb, d, m.pair, i, q - bq + dr * aq);
    }
    if (lane == 0) {
        const cplx rho = cmk(a.rho[2 * (m.vb + m.j)], a.rho[2 * (m.vb + m.j) + 1]) + dr;
        a.rho[2 * (m.vb + m.j)] = rho.re;
        a.rho[2 * (m.vb + m.j) + 1] = rho.im;
        if (m.pair) {
            a.rho[2 * (m.vb + m.j + 1)] = rho.re;
            a.rho[2 * (m.vb + m.j + 1) + 1] = -rho.im;
        }
    }
}

// rho <-> nu conversions around the refinement.
__global__ void nu_rho_kernel(RefineArgs a, int to_rho) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= a.batch * a.d) return;
    const cplx v = cmk(to_rho ? a.nu[2 * idx] : a.rho[2 * idx],
                       to_rho ? a.nu[2 * idx + 1] : a.rho[2 * idx + 1]);
    const cplx r = cdiv(cmk(1.0, 0.0), v);
    if (to_rho) {
        a.rho[2 * idx] = r.re;
        a.rho[2 * idx + 1] = r.im;
    } else if ((a.flags[idx] & 1) == 0) {
        a.nu[2 * idx] = r.re;
        a.nu[2 * idx + 1] = r.im;
    }
}

__global__ void refine_slots_kernel(int d, int batch, const double* residual, double target, int* slot_on,
                                    int* count) {
    const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (b >= batch) return;
    double mx = 0.0;
    for (int j = lane; j < d; j += 32) mx = fmax(mx, residual[(size_t)b * d + j]);
    mx = warp_max(mx);
    if (lane == 0) {
        const int on = slot_on[b] && mx > target;
        slot_on[b] = on;
        if (on) atomicAdd(count, 1);
    }
}

__global__ void compact_slots_kernel(const int* slot_on, int batch, int* list, int* n) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < batch; b += gridDim.x * blockDim.x)
        if (slot_on[b]) list[atomicAdd(n, 1)] = b;
}

inline unsigned warps_grid(int batch, int d) {
    return (unsigned)(((long long)batch * d * 32 + 255) / 256);
}

}  // namespace

void launch_refine_shift(const RefineArgs& a, cudaStream_t st) {
    shift_kernel<<<warps_grid(a.batch, a.d), 256, 0, st>>>(a);
    VRTE_CUDA_CHECK(cudaGetLastError());
}
void launch_refine_normalize(const RefineArgs& a, cudaStream_t st) {
    normalize_kernel<<<warps_grid(a.batch, a.d), 256, 0, st>>>(a);
    VRTE_CUDA_CHECK(cudaGetLastError());
}
void launch_refine_setup(const RefineArgs& a, cudaStream_t st) {
    setup_kernel<<<warps_grid(a.batch, a.d), 256, 0, st>>>(a);
    VRTE_CUDA_CHECK(cudaGetLastError());
}
void launch_refine_rhs(const RefineArgs& a, cudaStream_t st) {
    rhs_kernel<<<warps_grid(a.batch, a.d), 256, 0, st>>>(a);
    VRTE_CUDA_CHECK(cudaGetLastError());
}
void launch_refine_update(const RefineArgs& a, cudaStream_t st) {
    update_kernel<<<warps_grid(a.batch, a.d), 256, 0, st>>>(a);
    VRTE_CUDA_CHECK(cudaGetLastError());
}
void launch_nu_rho(const RefineArgs& a, bool to_rho, cudaStream_t st) {
    const int n = a.batch * a.d;
    nu_rho_kernel<<<(n + 255) / 256, 256, 0, st>>>(a, to_rho ? 1 : 0);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

void launch_refine_slots(int d, int batch, const double* residual, double target, int* slot_on, int* count,
                         cudaStream_t st) {
    VRTE_CUDA_CHECK(cudaMemsetAsync(count, 0, sizeof(int), st));
    refine_slots_kernel<<<(batch + 7) / 8, 256, 0, st>>>(d, batch, residual, target, slot_on, count);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

// the slots still refining as a list (any order: every slot's GEMMs are independent
// of which CTA runs them), for the compacted GEMMs of the extra steps
void launch_compact_slots(const int* slot_on, int batch, int* list, int* n, cudaStream_t st) {
    VRTE_CUDA_CHECK(cudaMemsetAsync(n, 0, sizeof(int), st));
    compact_slots_kernel<<<(batch + 255) / 256, 256, 0, st>>>(slot_on, batch, list, n);
    VRTE_CUDA_CHECK(cudaGetLastError());
}

}  // namespace vrte
