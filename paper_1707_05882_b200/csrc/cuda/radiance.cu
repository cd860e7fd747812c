// radiance.cu -- radiance field at arbitrary (tau, mu, phi) by source-function
// integration: reconstruction.cpp:28-227,
// pipeline.cpp:237-309, brdf.cpp:142-160, on the device state of one solve
// (modes, particular vectors, the FULL boundary solution of every layer).
//
// Per (medium, order) slot the kernel rows A^m(mu_o, +-mu_i) of every output
// direction, weighted by the quadrature, form [4 n_mu x d] matrices; the
// source coefficients of all modes (reconstruction.cpp:49-60) are then four
// batched DMMA GEMMs against the packed mode matrices (conjugate pairs as
// Re/Im columns, so the GEMM on real columns yields Re/Im of the complex
// contraction).  The closed-form layer integrals (reconstruction.cpp:87-149)
// run one thread per (order, Stokes channel, output direction, depth), in
// packed-real form: a conjugate pair with real boundary unknowns (x_j,
// x_{j+1}) contributes x_j Re T_j + x_{j+1} Im T_j, which is the reference's
// a_j T_j + conj(a_j T_j) with a_j = (x_j - i x_{j+1}) / 2 -- the field is real
// by construction.  Channels are the unit Stokes vectors (k = 1 for I, Q; k = 2
// for U, V, as in the BRDF path) combined with the beam's I0 in the azimuthal
// assembly (reconstruction.cpp:201-227).
#include "boundary.cuh"

namespace vrte {
namespace {

__device__ inline double dsgn(int c) { return (c & 2) ? -1.0 : 1.0; }  // D = diag(1,1,-1,-1)

// Weighted kernel rows per (slot om, output o, node i): WP = w_i A^m(mu_o, mu_i),
// WM = w_i A^m(mu_o, -mu_i) D (the D of Delta psi folded into the columns).
// Column-major [4 n_mu][d]: row o*4 + r, column 4 i + c.  kernel.cpp:67-87.
__global__ void rad_rows_kernel(RadArgs a) {
    const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const ProblemDev& p = a.p;
    const int N = p.N, L = p.Lc, nmu = a.n_mu, d = 4 * N, ld = 4 * nmu;
    const long long total = (long long)p.n_media * p.n_orders * nmu * N;
    if (idx >= total) return;
    const int i = (int)(idx % N);
    const int o = (int)((idx / N) % nmu);
    const int om = (int)(idx / ((long long)N * nmu));
    const int s = om / p.n_orders, m = p.order_of(om % p.n_orders);
    double app[4][4], apm[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) app[r][c] = apm[r][c] = 0.0;
    const double* gk = p.greek + (size_t)s * L * 6;
    for (int l = m; l < L; ++l) {
        const double* go = a.gsf_o + ((size_t)m * L + l) * 3 * nmu;
        const double* gn = a.gsf_n + ((size_t)m * L + l) * 3 * N;
        const double Pi = go[o], Ri = go[nmu + o], Ti = go[2 * nmu + o];
        const double Pj = gn[i], Rj = gn[N + i], Tj = gn[2 * N + i];
        const double be = gk[6 * l + 0], al = gk[6 * l + 1], ga = gk[6 * l + 2];
        const double de = gk[6 * l + 3], ep = gk[6 * l + 4], ze = gk[6 * l + 5];
        const double x00 = Pi * be, x01 = Pi * ga;
        const double x10 = Ri * ga, x11 = Ri * al, x12 = -Ti * ze, x13 = Ti * ep;
        const double x20 = -Ti * ga, x21 = -Ti * al, x22 = Ri * ze, x23 = -Ri * ep;
        const double x32 = Pi * ep, x33 = Pi * de;
        const double sl = ((l - m) & 1) ? -1.0 : 1.0;
        app[0][0] += x00 * Pj;
        app[0][1] += x01 * Rj;
        app[0][2] += -x01 * Tj;
        app[1][0] += x10 * Pj;
        app[1][1] += x11 * Rj - x12 * Tj;
        app[1][2] += -x11 * Tj + x12 * Rj;
        app[1][3] += x13 * Pj;
        app[2][0] += x20 * Pj;
        app[2][1] += x21 * Rj - x22 * Tj;
        app[2][2] += -x21 * Tj + x22 * Rj;
        app[2][3] += x23 * Pj;
        app[3][1] += -x32 * Tj;
        app[3][2] += x32 * Rj;
        app[3][3] += x33 * Pj;
        apm[0][0] += sl * (x00 * Pj);
        apm[0][1] += sl * (x01 * Rj);
        apm[0][2] += sl * (x01 * Tj);
        apm[1][0] += sl * (x10 * Pj);
        apm[1][1] += sl * (x11 * Rj + x12 * Tj);
        apm[1][2] += sl * (x11 * Tj + x12 * Rj);
        apm[1][3] += sl * (x13 * Pj);
        apm[2][0] += sl * (x20 * Pj);
        apm[2][1] += sl * (x21 * Rj + x22 * Tj);
        apm[2][2] += sl * (x21 * Tj + x22 * Rj);
        apm[2][3] += sl * (x23 * Pj);
        apm[3][1] += sl * (x32 * Tj);
        apm[3][2] += sl * (x32 * Rj);
        apm[3][3] += sl * (x33 * Pj);
    }
    const double w = p.weights[i];
    double* WP = a.wp + (size_t)om * ld * d;
    double* WM = a.wm + (size_t)om * ld * d;
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const size_t e = (size_t)(4 * i + c) * ld + 4 * o + r;
            WP[e] = w * app[r][c];
            WM[e] = w * apm[r][c] * dsgn(c);
        }
}

// Beam blocks A^m(mu_o, -mu0) per (slot, output): pipeline.cpp:244-256.
__global__ void rad_beam_block_kernel(RadArgs a) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    const ProblemDev& p = a.p;
    const int L = p.Lc, nmu = a.n_mu;
    if (idx >= p.n_media * p.n_orders * nmu) return;
    const int o = idx % nmu, om = idx / nmu;
    const int s = om / p.n_orders, m = p.order_of(om % p.n_orders);
    double bb[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) bb[r][c] = 0.0;
    const double* gk = p.greek + (size_t)s * L * 6;
    for (int l = m; l < L; ++l) {
        const double* go = a.gsf_o + ((size_t)m * L + l) * 3 * nmu;
        const double* gb = a.gsf_b + ((size_t)m * L + l) * 3;  // one incident (-mu0)
        const double Pi = go[o], Ri = go[nmu + o], Ti = go[2 * nmu + o];
        const double Pb = gb[0], Rb = gb[1], Tb = gb[2];
        const double be = gk[6 * l + 0], al = gk[6 * l + 1], ga = gk[6 * l + 2];
        const double de = gk[6 * l + 3], ep = gk[6 * l + 4], ze = gk[6 * l + 5];
        double Y[4][4];  // B_l Pi(-mu0)
        Y[0][0] = be * Pb; Y[0][1] = ga * Rb; Y[0][2] = -ga * Tb; Y[0][3] = 0.0;
        Y[1][0] = ga * Pb; Y[1][1] = al * Rb; Y[1][2] = -al * Tb; Y[1][3] = 0.0;
        Y[2][0] = 0.0;     Y[2][1] = -ze * Tb; Y[2][2] = ze * Rb; Y[2][3] = -ep * Pb;
        Y[3][0] = 0.0;     Y[3][1] = -ep * Tb; Y[3][2] = ep * Rb; Y[3][3] = de * Pb;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            bb[0][c] += Pi * Y[0][c];
            bb[1][c] += Ri * Y[1][c] - Ti * Y[2][c];
            bb[2][c] += -Ti * Y[1][c] + Ri * Y[2][c];
            bb[3][c] += Pi * Y[3][c];
        }
    }
    double* out = a.bb + (size_t)idx * 16;
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) out[4 * r + c] = bb[r][c];
}

// Beam source term per (layer p, order mo, output o, channel c), real
// (reconstruction.cpp:62-71): beam_top [ (w/2) sum_i (WP Z+ + WM Z-) + (w/2pi) B e_c ].
__global__ void rad_beam_src_kernel(RadArgs a) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    const ProblemDev& p = a.p;
    const int d = 4 * p.N, nmu = a.n_mu, ld = 4 * nmu, NO = p.n_orders;
    if (idx >= p.n_layers * NO * nmu * 4) return;
    const int c = idx & 3, o = (idx >> 2) % nmu, mo = (idx / (4 * nmu)) % NO, pl = idx / (4 * nmu * NO);
    const int s = p.medium[pl], om = s * NO + mo;
    const double* WP = a.wp + (size_t)om * ld * d;
    const double* WM = a.wm + (size_t)om * ld * d;
    const double* zp = a.zp + ((size_t)om * a.R + c) * d;
    const double* zm = a.zm + ((size_t)om * a.R + c) * d;
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k = 0; k < d; ++k) {
        const double zpk = zp[k], zmk = zm[k] * dsgn(k & 3);  // WM carries D
#pragma unroll
        for (int r = 0; r < 4; ++r) v[r] += WP[(size_t)k * ld + 4 * o + r] * zpk + WM[(size_t)k * ld + 4 * o + r] * zmk;
    }
    const double half_omega = 0.5 * p.omega[s];
    const double* B = a.bb + ((size_t)om * nmu + o) * 16;
    double* out = a.beam_src + (size_t)idx * 4;
#pragma unroll
    for (int r = 0; r < 4; ++r)
        out[r] = a.beam_top[pl] * (half_omega * v[r] + p.omega[s] / (2.0 * kPi) * B[4 * r + c]);
}

struct LayerCtx {
    const double* acc_a;  // [ld][d] column-major, rows o*4+r
    const double* acc_b;
    const double* nu;     // [d][2]
    const double* wi;     // [d]
    const double* x;      // boundary solution rows (stride R), channel column applied
    int colA, colB;       // bnd_col offsets of A_p(0), B_p(0) handled via bnd_col
    double thick, half_omega;
    const double* beam;   // [4]
};

__device__ inline cplx cexpd(cplx z) { return cexp_(z); }

// sum over the packed mode columns of the layer integrals (reconstruction.cpp:87-149)
// warp-cooperative: lanes split the mode columns, fixed-order butterfly sum
__device__ void layer_integral(const RadArgs& a, const LayerCtx& L, int o, int p, bool up, double mu, double t,
                               const double ib[4], double out[4], int lane) {
    const int d = 4 * a.p.N, ld = 4 * a.n_mu, G = 2 * d * a.p.n_layers;
    const double dth = L.thick;
    const double eb = up ? exp(-(dth - t) / mu) : exp(-t / mu);
    double ms[4] = {0.0, 0.0, 0.0, 0.0};
    const double emu_dt = exp(-(dth - t) / mu), emu_t = exp(-t / mu);
    for (int jj = lane; jj < d; jj += 32) {
        const double w = L.wi[jj];
        const int j = (w < 0.0) ? jj - 1 : jj;
        const bool pair = w != 0.0, imc = w < 0.0;
        const cplx nu = cmk(L.nu[2 * j], L.nu[2 * j + 1]);
        const double xa = L.x[(size_t)bnd_col(p, jj, d, G) * a.R];
        const double xb = L.x[(size_t)bnd_col(p, d + jj, d, G) * a.R];
        // complex factors of the from-top (rate nu, coefficient a) and from-bottom terms
        cplx ft, fb;
        const cplx inv_nu = cdiv(cmk(1.0, 0.0), nu);
        const cplx e_t = cexpd(cmk(-t * inv_nu.re, -t * inv_nu.im));                // e^{-t/nu}
        const cplx e_d = cexpd(cmk(-dth * inv_nu.re, -dth * inv_nu.im));            // e^{-d/nu}
        const cplx e_dt = cexpd(cmk(-(dth - t) * inv_nu.re, -(dth - t) * inv_nu.im));  // e^{-(d-t)/nu}
        const cplx mu_nu = cmk(mu * inv_nu.re, mu * inv_nu.im);
        const double dre = 1.0 / mu - inv_nu.re, dim = -inv_nu.im;
        const bool degen = hypot(dre, dim) < 1e-9;  // kDegenerateRate, reconstruction.cpp:85
        if (up) {
            // up_term_top(nu): (e^{-t/nu} - e^{-d/nu} e^{-(d-t)/mu}) / (1 + mu/nu)
            ft = cdiv(cmk(e_t.re - e_d.re * emu_dt, e_t.im - e_d.im * emu_dt), cmk(1.0 + mu_nu.re, mu_nu.im));
            // up_term_bottom(nu)
            if (degen)
                fb = cmk(emu_dt * ((dth - t) / mu), 0.0);
            else
                fb = cdiv(cmk(e_dt.re - emu_dt, e_dt.im), cmk(1.0 - mu_nu.re, -mu_nu.im));
        } else {
            // down_term_top(nu)
            if (degen)
                ft = cmk(emu_t * (t / mu), 0.0);
            else
                ft = cdiv(cmk(e_t.re - emu_t, e_t.im), cmk(1.0 - mu_nu.re, -mu_nu.im));
            // down_term_bottom(nu): (e^{-(d-t)/nu} - e^{-d/nu} e^{-t/mu}) / (1 + mu/nu)
            fb = cdiv(cmk(e_dt.re - e_d.re * emu_t, e_dt.im - e_d.im * emu_t), cmk(1.0 + mu_nu.re, mu_nu.im));
        }
        const double* ca = L.acc_a + (size_t)j * ld + 4 * o;
        const double* cb = L.acc_b + (size_t)j * ld + 4 * o;
        const double* ca2 = pair ? L.acc_a + (size_t)(j + 1) * ld + 4 * o : nullptr;
        const double* cb2 = pair ? L.acc_b + (size_t)(j + 1) * ld + 4 * o : nullptr;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const cplx va = cmk(L.half_omega * ca[r], pair ? L.half_omega * ca2[r] : 0.0);
            const cplx vb = cmk(L.half_omega * cb[r], pair ? L.half_omega * cb2[r] : 0.0);
            const cplx ta = ft * va, tb = fb * vb;
            ms[r] += xa * (imc ? ta.im : ta.re) + xb * (imc ? tb.im : tb.re);
        }
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) out[r] = ib[r] * eb + warp_sum(ms[r]);
    // beam term at the real rate mu0 (up_term_top / down_term_top with a = mu0)
    const double mu0 = a.mu0;
    double f;
    if (up) {
        f = (exp(-t / mu0) - exp(-dth / mu0) * emu_dt) / (1.0 + mu / mu0);
    } else {
        if (fabs(1.0 / mu - 1.0 / mu0) < 1e-9)
            f = emu_t * (t / mu);
        else
            f = (exp(-t / mu0) - emu_t) / (1.0 - mu / mu0);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) out[r] += f * L.beam[r];
}

// Components per (order mo, channel c, depth it, output o): reconstruction.cpp:151-199.
__global__ void rad_integrate_kernel(RadArgs a) {
    const int idx = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const ProblemDev& p = a.p;
    const int nmu = a.n_mu, NO = p.n_orders, P = p.n_layers, d = 4 * p.N, ld = 4 * nmu, G = 2 * d * P;
    if (idx >= NO * 4 * a.n_tau * nmu) return;
    const int o = idx % nmu, it = (idx / nmu) % a.n_tau, c = (idx / (nmu * a.n_tau)) % 4, mo = idx / (nmu * a.n_tau * 4);
    const int m = p.order_of(mo);
    const double mus = a.mus[o], mu = fabs(mus);
    const bool up = mus > 0.0;
    // locate_layer (reconstruction.cpp:12-19)
    const double tau = a.taus[it];
    int pt = 0;
    while (pt + 1 < P && tau >= a.tau_top[pt] + p.tau[pt]) ++pt;
    const double tl = fmin(fmax(tau - a.tau_top[pt], 0.0), p.tau[pt]);
    auto ctx = [&](int pl) {
        const int s = p.medium[pl], om = s * NO + mo;
        LayerCtx L;
        L.acc_a = a.acc_a + (size_t)om * ld * d;
        L.acc_b = a.acc_b + (size_t)om * ld * d;
        L.nu = a.nu + (size_t)om * d * 2;
        L.wi = a.wi + (size_t)om * d;
        L.x = a.rhs_x + (size_t)mo * G * a.R + c;
        L.thick = p.tau[pl];
        L.half_omega = 0.5 * p.omega[s];
        L.beam = a.beam_src + ((((size_t)pl * NO + mo) * nmu + o) * 4 + c) * 4;
        return L;
    };
    double bnd[4] = {0.0, 0.0, 0.0, 0.0}, val[4];
    if (up) {
        if (m == 0 && p.base_type != 0 && a.base_val) {
#pragma unroll
            for (int r = 0; r < 4; ++r) bnd[r] = a.base_val[((size_t)c * nmu + o) * 4 + r];
        }
        for (int pl = P - 1; pl > pt; --pl) {
            layer_integral(a, ctx(pl), o, pl, true, mu, 0.0, bnd, val, lane);
#pragma unroll
            for (int r = 0; r < 4; ++r) bnd[r] = val[r];
        }
        layer_integral(a, ctx(pt), o, pt, true, mu, tl, bnd, val, lane);
    } else {
        for (int pl = 0; pl < pt; ++pl) {
            layer_integral(a, ctx(pl), o, pl, false, mu, p.tau[pl], bnd, val, lane);
#pragma unroll
            for (int r = 0; r < 4; ++r) bnd[r] = val[r];
        }
        layer_integral(a, ctx(pt), o, pt, false, mu, tl, bnd, val, lane);
    }
    double* out = a.comp + ((((size_t)mo * 4 + c) * a.n_tau + it) * nmu + o) * 4;
    if (lane < 4) out[lane] = val[lane];
}

// m = 0 base reflection start value (reconstruction.cpp:176-192): the downward
// nodal stack at the bottom of the last layer per channel, then its reflection
// along every output direction plus the reflected attenuated beam.
__global__ void rad_base_down_kernel(RadArgs a, int mo) {
    const int idx = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const ProblemDev& p = a.p;
    const int d = 4 * p.N, NO = p.n_orders, P = p.n_layers, G = 2 * d * P;
    if (idx >= 4 * d) return;
    const int i = idx % d, c = idx / d;
    const int q = P - 1, s = p.medium[q], om = s * NO + mo;
    const double th = p.tau[q];
    const double* psp = a.psi_p + (size_t)om * d * d;
    const double* psm = a.psi_m + (size_t)om * d * d;
    const double* x = a.rhs_x + (size_t)mo * G * a.R + c;
    double v = 0.0;
    for (int jj = lane; jj < d; jj += 32) {
        const double w = a.wi[(size_t)om * d + jj];
        const int j = (w < 0.0) ? jj - 1 : jj;
        const bool pair = w != 0.0, imc = w < 0.0;
        const cplx nu = cmk(a.nu[2 * ((size_t)om * d + j)], a.nu[2 * ((size_t)om * d + j) + 1]);
        const cplx inv_nu = cdiv(cmk(1.0, 0.0), nu);
        const cplx ea = cexp_(cmk(-th * inv_nu.re, -th * inv_nu.im));  // e^{-t/nu}, t = thickness
        const cplx eb = cmk(1.0, 0.0);                                  // e^{-(d-t)/nu} = 1
        const cplx pm = cmk(psm[(size_t)j * d + i], pair ? psm[(size_t)(j + 1) * d + i] : 0.0);
        const cplx pp = cmk(psp[(size_t)j * d + i], pair ? psp[(size_t)(j + 1) * d + i] : 0.0);
        const double sg = dsgn(i & 3);
        const cplx ta = ea * cmk(sg * pm.re, sg * pm.im), tb = eb * cmk(sg * pp.re, sg * pp.im);
        v += x[(size_t)bnd_col(q, jj, d, G) * a.R] * (imc ? ta.im : ta.re) +
             x[(size_t)bnd_col(q, d + jj, d, G) * a.R] * (imc ? tb.im : tb.re);
    }
    v = warp_sum(v) + a.beam_top[q] * exp(-th / a.mu0) * a.zm[((size_t)om * a.R + c) * d + i];
    if (lane == 0) a.down_bot[(size_t)c * d + i] = v;
}

__global__ void rad_base_val_kernel(RadArgs a) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    const ProblemDev& p = a.p;
    const int N = p.N, d = 4 * N, nmu = a.n_mu;
    if (idx >= 4 * nmu * 4) return;
    const int r = idx & 3, o = (idx >> 2) % nmu, c = idx / (4 * nmu);
    double v = 0.0;
    for (int j = 0; j < N; ++j) {
        const double* R = a.base_out + ((size_t)o * N + j) * 16 + 4 * r;
        const double* dn = a.down_bot + (size_t)c * d + 4 * j;
        v += p.weights[j] * p.nodes[j] * (R[0] * dn[0] + R[1] * dn[1] + R[2] * dn[2] + R[3] * dn[3]);
    }
    // (mu0/pi) R(mu, mu0) e_c e^{-tau_tot/mu0}, kept by the selector of the channel's k
    if (((r < 2) == (c < 2)))
        v += (a.mu0 / kPi) * exp(-a.tau_total / a.mu0) * a.base_beam[(size_t)o * 16 + 4 * r + c];
    a.base_val[idx] = v;
}

// azimuthal assembly (reconstruction.cpp:201-227) with the beam's I0 per channel
__global__ void rad_assemble_kernel(RadArgs a) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    const int nmu = a.n_mu, nph = a.n_phi;
    if (idx >= a.n_tau * nmu * nph) return;
    const int ip = idx % nph, o = (idx / nph) % nmu, it = idx / (nph * nmu);
    const double x = -(a.phis[ip] - a.phi0);
    double tot[4] = {0.0, 0.0, 0.0, 0.0};
    for (int mo = 0; mo < a.p.n_orders; ++mo) {
        const int m = a.p.order_of(mo);
        const double sc = (m == 0) ? 1.0 : 2.0;
        double sn, cs;
        sincos(m * x, &sn, &cs);
        double k1[4] = {0, 0, 0, 0}, k2[4] = {0, 0, 0, 0};
        for (int c = 0; c < 4; ++c) {
            const double* v = a.comp + ((((size_t)mo * 4 + c) * a.n_tau + it) * nmu + o) * 4;
            double* k = c < 2 ? k1 : k2;
            for (int r = 0; r < 4; ++r) k[r] += a.stokes[c] * v[r];
        }
        tot[0] += 0.5 * sc * (cs * k1[0] - sn * k2[0]);
        tot[1] += 0.5 * sc * (cs * k1[1] - sn * k2[1]);
        tot[2] += 0.5 * sc * (sn * k1[2] + cs * k2[2]);
        tot[3] += 0.5 * sc * (sn * k1[3] + cs * k2[3]);
    }
    double* out = a.field + (size_t)idx * 4;
    for (int r = 0; r < 4; ++r) out[r] = tot[r];
}

// field reflectance (brdf.cpp:142-160): exiting nodal flux at tau = 0 over 19
// azimuths, divided by mu0 I0.  CTA (one warp) per node, then a fixed-order sum.
__global__ void rad_refl_node_kernel(RadArgs a, double* part) {
    const int i = blockIdx.x, j = threadIdx.x, N = a.p.N, d = 4 * N, nph = 19;
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    if (j < nph) {
        const double x = -(2.0 * kPi * j / nph);
        for (int mo = 0; mo < a.p.n_orders; ++mo) {
            const int m = a.p.order_of(mo);
            const double sc = (m == 0) ? 1.0 : 2.0;
            double sn, cs;
            sincos(m * x, &sn, &cs);
            double k1[4] = {0, 0, 0, 0}, k2[4] = {0, 0, 0, 0};
            for (int c = 0; c < 4; ++c) {
                const double* u = a.up + ((size_t)mo * a.R + c) * d + 4 * i;
                double* k = c < 2 ? k1 : k2;
                for (int r = 0; r < 4; ++r) k[r] += a.stokes[c] * u[r];
            }
            s[0] += 0.5 * sc * (cs * k1[0] - sn * k2[0]);
            s[1] += 0.5 * sc * (cs * k1[1] - sn * k2[1]);
            s[2] += 0.5 * sc * (sn * k1[2] + cs * k2[2]);
            s[3] += 0.5 * sc * (sn * k1[3] + cs * k2[3]);
        }
    }
    const double w = a.p.weights[i] * a.p.nodes[i] * (2.0 * kPi / nph);
    for (int r = 0; r < 4; ++r) {
        const double v = warp_sum(w * s[r]);
        if (j == 0) part[4 * i + r] = v;
    }
}
__global__ void rad_refl_sum_kernel(RadArgs a, const double* part) {
    const int r = threadIdx.x;
    if (r >= 4) return;
    double acc = 0.0;
    for (int i = 0; i < a.p.N; ++i) acc += part[4 * i + r];
    a.refl[r] = acc / fmax(a.mu0 * a.stokes[0], 1e-300);
}

}  // namespace

int launch_radiance(RadArgs a, cudaStream_t st) {
    const ProblemDev& p = a.p;
    const int N = p.N, d = 4 * N, nmu = a.n_mu, ld = 4 * nmu, B = p.n_media * p.n_orders;
    int nl = 0;
    launch_gsf(p, a.mus, nmu, 1.0, a.gsf_o, st);
    ++nl;
    {
        const long long total = (long long)B * nmu * N;
        rad_rows_kernel<<<(unsigned)((total + 127) / 128), 128, 0, st>>>(a);
        rad_beam_block_kernel<<<(B * nmu + 127) / 128, 128, 0, st>>>(a);
        VRTE_CUDA_CHECK(cudaGetLastError());
        nl += 2;
    }
    // source coefficients of every mode: acc_a = WP psi+ + WM psi-, acc_b = WP psi- + WM psi+
    auto g = [&](const double* A, const double* Bm, double* C, double beta) {
        GemmBatch gb{};
        gb.m = ld;
        gb.n = d;
        gb.k = d;
        gb.a = A;
        gb.lda = ld;
        gb.stride_a = (long long)ld * d;
        gb.b = Bm;
        gb.ldb = d;
        gb.stride_b = (long long)d * d;
        gb.c = C;
        gb.ldc = ld;
        gb.stride_c = (long long)ld * d;
        gb.batch = B;
        gb.alpha = 1.0;
        gb.beta = beta;
        gemm_batched(gb, st);
    };
    g(a.wp, a.psi_p, a.acc_a, 0.0);
    g(a.wm, a.psi_m, a.acc_a, 1.0);
    g(a.wp, a.psi_m, a.acc_b, 0.0);
    g(a.wm, a.psi_p, a.acc_b, 1.0);
    nl += 4;
    {
        const int total = p.n_layers * p.n_orders * nmu * 4;
        rad_beam_src_kernel<<<(total + 127) / 128, 128, 0, st>>>(a);
        VRTE_CUDA_CHECK(cudaGetLastError());
        ++nl;
    }
    if (a.base_val) {
        rad_base_down_kernel<<<(4 * d * 32 + 255) / 256, 256, 0, st>>>(a, a.slot0);
        rad_base_val_kernel<<<(16 * nmu + 127) / 128, 128, 0, st>>>(a);
        VRTE_CUDA_CHECK(cudaGetLastError());
        nl += 2;
    }
    {
        const long long total = (long long)p.n_orders * 4 * a.n_tau * nmu * 32;  // warp per item
        rad_integrate_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(a);
        const int tf = a.n_tau * nmu * a.n_phi;
        rad_assemble_kernel<<<(tf + 127) / 128, 128, 0, st>>>(a);
        rad_refl_node_kernel<<<N, 32, 0, st>>>(a, a.down_bot + 4 * (size_t)d);  // scratch after down_bot
        rad_refl_sum_kernel<<<1, 32, 0, st>>>(a, a.down_bot + 4 * (size_t)d);
        VRTE_CUDA_CHECK(cudaGetLastError());
        nl += 4;
    }
    return nl;
}

}  // namespace vrte
