// vrte_oracle.cpp -- TEST INFRASTRUCTURE ONLY (see vrte_oracle.h).
//
// A CPU restatement of the reference BRDF path that keeps the reference's
// algorithm and loop structure (serial incident x basis loops, parallel over
// orders; a fresh complex boundary LU per incident/basis/order; F*E and the
// 8N operator rebuilt for every particular solve) so that it is both the
// numerical oracle and a faithful CPU timing baseline.  Every routine cites
// the reference file:line it restates (paths under /root/reference/proj).
// Eigen is replaced by LAPACK from scipy-openblas.

#include "vrte_oracle.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

extern "C" {
void scipy_dgeev_(const char*, const char*, const int*, double*, const int*, double*, double*,
                  double*, const int*, double*, const int*, double*, const int*, int*, size_t,
                  size_t);
void scipy_dgetrf_(const int*, const int*, double*, const int*, int*, int*);
void scipy_dgetrs_(const char*, const int*, const int*, const double*, const int*, const int*,
                   double*, const int*, int*, size_t);
void scipy_zgetrf_(const int*, const int*, void*, const int*, int*, int*);
void scipy_zgetrs_(const char*, const int*, const int*, const void*, const int*, const int*, void*,
                   const int*, int*, size_t);
void scipy_zgecon_(const char*, const int*, const void*, const int*, const double*, double*, void*,
                   double*, int*, size_t);
void scipy_dgesvd_(const char*, const char*, const int*, const int*, double*, const int*, double*,
                   double*, const int*, double*, const int*, double*, const int*, int*, size_t,
                   size_t);
void scipy_dgemm_(const char*, const char*, const int*, const int*, const int*, const double*,
                  const double*, const int*, const double*, const int*, const double*, double*,
                  const int*, size_t, size_t);
void scipy_zgemm_(const char*, const char*, const int*, const int*, const int*, const void*,
                  const void*, const int*, const void*, const int*, const void*, void*, const int*,
                  size_t, size_t);
void scipy_openblas_set_num_threads(int);
}

namespace vo {

using cd = std::complex<double>;
constexpr double kPi = 3.14159265358979323846;
constexpr double kTwoPi = 2.0 * kPi;
constexpr double kNuClamp = 4e9;             // homogeneous.hpp:68
constexpr double kEigenResidualBound = 1e-9;  // homogeneous.hpp:71

struct ValidationError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NumericalError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------- small 4x4
struct M4 {
    double v[16] = {0};
    double& operator()(int r, int c) { return v[4 * r + c]; }
    double operator()(int r, int c) const { return v[4 * r + c]; }
};
static M4 mul(const M4& a, const M4& b) {
    M4 o;
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) {
            double s = 0;
            for (int k = 0; k < 4; ++k) s += a(r, k) * b(k, c);
            o(r, c) = s;
        }
    return o;
}
static void axpy4(M4& acc, double s, const M4& x) {
    for (int e = 0; e < 16; ++e) acc.v[e] += s * x.v[e];
}
static const double kParity[4] = {1.0, 1.0, -1.0, -1.0};  // kernel.hpp:10-13
static M4 parity_conjugate(const M4& x) {                  // kernel.cpp:20-27
    M4 o;
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) o(r, c) = kParity[r] * kParity[c] * x(r, c);
    return o;
}

// ---------------------------------------------------------------- inputs
struct Layer {
    double omega = 0, tau = 0;
    std::vector<M4> coeffs;
    int order_count() const { return (int)coeffs.size(); }
};
struct Base {
    int type = 0;  // 0 black, 1 lambertian, 2 table
    double rho = 0;
    int n = 0;
    std::vector<M4> table;
    const M4& at(int i, int j) const { return table[(size_t)i * n + j]; }
};
struct Material {
    std::vector<Layer> layers;
    Base base;
    int order_count() const { return layers.empty() ? 0 : layers.front().order_count(); }
};

static Material from_c(const oracle_material* m) {
    if (!m || m->n_layers < 1 || m->order_count < 1)
        throw ValidationError("oracle: empty material");
    Material out;
    for (int p = 0; p < m->n_layers; ++p) {
        Layer l;
        l.omega = m->omega[p];
        l.tau = m->tau[p];
        l.coeffs.resize(m->order_count);
        for (int k = 0; k < m->order_count; ++k)
            std::memcpy(l.coeffs[k].v, m->coeffs + ((size_t)p * m->order_count + k) * 16,
                        16 * sizeof(double));
        out.layers.push_back(std::move(l));
    }
    out.base.type = m->base_type;
    out.base.rho = m->rho;
    if (m->base_type == 2) {
        out.base.n = m->table_n;
        out.base.table.resize((size_t)m->table_n * m->table_n);
        for (size_t e = 0; e < out.base.table.size(); ++e)
            std::memcpy(out.base.table[e].v, m->table + e * 16, 16 * sizeof(double));
    }
    return out;
}

// ---------------------------------------------------------------- quadrature
struct Quad {
    int n = 0;
    std::vector<double> nodes, weights;
};
// types.cpp:27-68 -- Newton on P_n from cos(pi(k+0.75)/(n+0.5)), |dx|<1e-15.
static Quad build_quadrature(int n) {
    if (n < 1) throw ValidationError("quadrature: size must be at least 1");
    Quad q;
    q.n = n;
    q.nodes.assign(n, 0.0);
    q.weights.assign(n, 0.0);
    const int half = (n + 1) / 2;
    for (int k = 0; k < half; ++k) {
        double x = std::cos(kPi * (k + 0.75) / (n + 0.5));
        double dp = 0.0;
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = x;
            for (int l = 2; l <= n; ++l) {
                const double p2 = ((2.0 * l - 1.0) * x * p1 - (l - 1.0) * p0) / l;
                p0 = p1;
                p1 = p2;
            }
            dp = n * (x * p1 - p0) / (x * x - 1.0);
            const double dx = p1 / dp;
            x -= dx;
            if (std::abs(dx) < 1e-15) break;
        }
        const double w = 2.0 / ((1.0 - x * x) * dp * dp);
        q.nodes[n - 1 - k] = 0.5 * (1.0 + x);
        q.weights[n - 1 - k] = 0.5 * w;
        q.nodes[k] = 0.5 * (1.0 - x);
        q.weights[k] = 0.5 * w;
    }
    if (n == 1) {
        q.nodes[0] = 0.5;
        q.weights[0] = 1.0;
    }
    return q;
}

// ---------------------------------------------------------------- GSF
// wigner.cpp:11-27 closed-form start d^{lmin}_{mn}.
static double wigner_start(int m, int n, double x) {
    const int lmin = std::max(std::abs(m), std::abs(n));
    const int a = std::abs(m - n), b = std::abs(m + n);
    double lf = 0.0;
    for (int k = 2; k <= 2 * lmin; ++k) lf += std::log((double)k);
    for (int k = 2; k <= a; ++k) lf -= std::log((double)k);
    for (int k = 2; k <= b; ++k) lf -= std::log((double)k);
    double v = std::exp(0.5 * lf - lmin * std::log(2.0));
    v *= std::pow(std::max(0.0, 1.0 - x), 0.5 * a) * std::pow(std::max(0.0, 1.0 + x), 0.5 * b);
    if (n < m && ((m - n) & 1)) v = -v;
    return v;
}
// wigner.cpp:31-62 upward three-term recurrence in l.
static std::vector<double> wigner_seq(int m, int n, int lmax, double x) {
    std::vector<double> d((size_t)lmax + 1, 0.0);
    const int lmin = std::max(std::abs(m), std::abs(n));
    if (lmin > lmax) return d;
    d[lmin] = wigner_start(m, n, x);
    if (lmin == lmax) return d;
    const double mn = (double)m * n;
    double prev = 0.0, cur = d[lmin];
    for (int l = lmin; l < lmax; ++l) {
        double next;
        if (l == 0) {
            next = x;
        } else {
            const double lp = l + 1.0;
            const double c0 = l * std::sqrt((lp * lp - m * m) * (lp * lp - n * n));
            const double c1 = (2.0 * l + 1.0) * (l * lp * x - mn);
            const double c2 = lp * std::sqrt(((double)l * l - m * m) * ((double)l * l - n * n));
            next = (c1 * cur - c2 * prev) / c0;
        }
        prev = cur;
        cur = next;
        d[l + 1] = next;
    }
    return d;
}
struct Gsf {
    std::vector<double> p, r, t;
};
// wigner.cpp:64-81
static Gsf gsf_seq(int m, int lmax, double x) {
    Gsf g;
    const double sgn = (m & 1) ? -1.0 : 1.0;
    const auto d0 = wigner_seq(m, 0, lmax, x), d2p = wigner_seq(m, 2, lmax, x),
               d2m = wigner_seq(m, -2, lmax, x);
    g.p.resize(lmax + 1);
    g.r.resize(lmax + 1);
    g.t.resize(lmax + 1);
    for (int l = 0; l <= lmax; ++l) {
        g.p[l] = sgn * d0[l];
        g.r[l] = 0.5 * sgn * (d2p[l] + d2m[l]);
        g.t[l] = -0.5 * sgn * (d2p[l] - d2m[l]);
    }
    return g;
}
// wigner.cpp:83-93: diag(P,R,R,P), -T at (1,2),(2,1); flip_t gives D Pi D.
static M4 gsf_matrix(const Gsf& g, int l, bool flip_t) {
    M4 o;
    o(0, 0) = g.p[l];
    o(1, 1) = g.r[l];
    o(2, 2) = g.r[l];
    o(3, 3) = g.p[l];
    const double t = flip_t ? g.t[l] : -g.t[l];
    o(1, 2) = t;
    o(2, 1) = t;
    return o;
}

// ---------------------------------------------------------------- kernels
struct Kernel {
    int m = 0, n = 0;
    std::vector<M4> pp, pm, mp, mm;
    const M4& block(bool ru, bool cu, int i, int j) const {
        const auto& v = ru ? (cu ? pp : pm) : (cu ? mp : mm);
        return v[(size_t)i * n + j];
    }
};
// kernel.cpp:29-65
static Kernel assemble_kernel(int m, const Layer& layer, const Quad& q) {
    const int n = q.n, L = layer.order_count();
    Kernel k;
    k.m = m;
    k.n = n;
    const size_t nn = (size_t)n * n;
    k.pp.assign(nn, M4{});
    k.pm.assign(nn, M4{});
    k.mp.assign(nn, M4{});
    k.mm.assign(nn, M4{});
    if (m >= L) return k;
    std::vector<Gsf> tab(n);
    for (int i = 0; i < n; ++i) tab[i] = gsf_seq(m, L - 1, q.nodes[i]);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            M4 app, apm;
            for (int l = m; l < L; ++l) {
                const M4 left = mul(gsf_matrix(tab[i], l, false), layer.coeffs[l]);
                const M4 right = gsf_matrix(tab[j], l, false);
                const M4 right_neg = gsf_matrix(tab[j], l, true);
                const double s = ((l - m) & 1) ? -1.0 : 1.0;
                axpy4(app, 1.0, mul(left, right));
                axpy4(apm, s, mul(left, right_neg));
            }
            const size_t idx = (size_t)i * n + j;
            k.pp[idx] = app;
            k.pm[idx] = apm;
            k.mp[idx] = parity_conjugate(apm);
            k.mm[idx] = parity_conjugate(app);
        }
    return k;
}
struct KColumn {
    std::vector<M4> up, down;
};
// kernel.cpp:89-109
static KColumn beam_column(int m, const Layer& layer, const Quad& q, double mu_beam) {
    const int n = q.n, L = layer.order_count();
    KColumn c;
    c.up.assign(n, M4{});
    c.down.assign(n, M4{});
    if (m >= L) return c;
    const Gsf gb = gsf_seq(m, L - 1, mu_beam);
    std::vector<Gsf> tab(n);
    for (int i = 0; i < n; ++i) tab[i] = gsf_seq(m, L - 1, q.nodes[i]);
    for (int i = 0; i < n; ++i)
        for (int l = m; l < L; ++l) {
            const M4 right = mul(layer.coeffs[l], gsf_matrix(gb, l, false));
            const double s = ((l - m) & 1) ? -1.0 : 1.0;
            axpy4(c.up[i], 1.0, mul(gsf_matrix(tab[i], l, false), right));
            axpy4(c.down[i], s, mul(gsf_matrix(tab[i], l, true), right));
        }
    return c;
}

struct KRow {
    std::vector<M4> plus, minus;
};
// kernel.cpp:67-87: A^m(mu, +mu_j) and A^m(mu, -mu_j) for an arbitrary signed mu
static KRow kernel_row(int m, const Layer& layer, const Quad& q, double mu) {
    const int n = q.n, L = layer.order_count();
    KRow row;
    row.plus.assign(n, M4{});
    row.minus.assign(n, M4{});
    if (m >= L) return row;
    const Gsf g = gsf_seq(m, L - 1, mu);
    std::vector<Gsf> tab(n);
    for (int j = 0; j < n; ++j) tab[j] = gsf_seq(m, L - 1, q.nodes[j]);
    for (int j = 0; j < n; ++j)
        for (int l = m; l < L; ++l) {
            const M4 left = mul(gsf_matrix(g, l, false), layer.coeffs[l]);
            const double sgn = ((l - m) & 1) ? -1.0 : 1.0;
            axpy4(row.plus[j], 1.0, mul(left, gsf_matrix(tab[j], l, false)));
            axpy4(row.minus[j], sgn, mul(left, gsf_matrix(tab[j], l, true)));
        }
    return row;
}

// ---------------------------------------------------------------- dense helpers (col-major)
static void dgemm(char ta, char tb, int m, int n, int k, double alpha, const double* a, int lda,
                  const double* b, int ldb, double beta, double* c, int ldc) {
    scipy_dgemm_(&ta, &tb, &m, &n, &k, &alpha, a, &lda, b, &ldb, &beta, c, &ldc, 1, 1);
}
static double max_abs(const std::vector<double>& v) {
    double s = 0;
    for (double x : v) s = std::max(s, std::abs(x));
    return s;
}
static double max_abs(const std::vector<cd>& v) {
    double s = 0;
    for (const cd& x : v) s = std::max(s, std::abs(x));
    return s;
}
static bool all_finite(const std::vector<cd>& v) {
    for (const cd& x : v)
        if (!std::isfinite(x.real()) || !std::isfinite(x.imag())) return false;
    return true;
}
static bool all_finite(const std::vector<double>& v) {
    for (double x : v)
        if (!std::isfinite(x)) return false;
    return true;
}
// y = A x (A real col-major rows x cols)
static std::vector<cd> matvec(const std::vector<double>& a, int rows, int cols,
                              const std::vector<cd>& x) {
    std::vector<cd> y(rows, 0.0);
    for (int j = 0; j < cols; ++j) {
        const cd xj = x[j];
        const double* col = a.data() + (size_t)j * rows;
        for (int i = 0; i < rows; ++i) y[i] += col[i] * xj;
    }
    return y;
}
static std::vector<double> matvec(const std::vector<double>& a, int rows, int cols,
                                  const std::vector<double>& x) {
    std::vector<double> y(rows, 0.0);
    for (int j = 0; j < cols; ++j) {
        const double xj = x[j];
        const double* col = a.data() + (size_t)j * rows;
        for (int i = 0; i < rows; ++i) y[i] += col[i] * xj;
    }
    return y;
}
static std::vector<cd> matvec(const std::vector<cd>& a, int rows, int cols,
                              const std::vector<cd>& x) {
    std::vector<cd> y(rows, 0.0);
    for (int j = 0; j < cols; ++j) {
        const cd xj = x[j];
        const cd* col = a.data() + (size_t)j * rows;
        for (int i = 0; i < rows; ++i) y[i] += col[i] * xj;
    }
    return y;
}
// Complex LU (Eigen::PartialPivLU<MatrixXcd> stand-in).
struct ZLu {
    int n = 0;
    std::vector<cd> a;
    std::vector<int> piv;
    bool ok = true;
    explicit ZLu(std::vector<cd> m, int n_) : n(n_), a(std::move(m)), piv(n_) {
        int info = 0;
        scipy_zgetrf_(&n, &n, a.data(), &n, piv.data(), &info);
        ok = info >= 0;
    }
    std::vector<cd> solve(const std::vector<cd>& b) const {
        std::vector<cd> x = b;
        int info = 0, one = 1;
        const char t = 'N';
        scipy_zgetrs_(&t, &n, &one, a.data(), &n, piv.data(), x.data(), &n, &info, 1);
        return x;
    }
    double rcond(double anorm) const {
        std::vector<cd> work(2 * (size_t)n);
        std::vector<double> rwork(2 * (size_t)n);
        double rc = 0;
        int info = 0;
        const char nm = '1';
        scipy_zgecon_(&nm, &n, a.data(), &n, &anorm, &rc, work.data(), rwork.data(), &info, 1);
        return rc;
    }
};
struct DLu {
    int n = 0;
    std::vector<double> a;
    std::vector<int> piv;
    explicit DLu(std::vector<double> m, int n_) : n(n_), a(std::move(m)), piv(n_) {
        int info = 0;
        scipy_dgetrf_(&n, &n, a.data(), &n, piv.data(), &info);
    }
    std::vector<double> solve(const std::vector<double>& b) const {
        std::vector<double> x = b;
        int info = 0, one = 1;
        const char t = 'N';
        scipy_dgetrs_(&t, &n, &one, a.data(), &n, piv.data(), x.data(), &n, &info, 1);
        return x;
    }
};

// ---------------------------------------------------------------- reduced operators
struct Reduced {
    int m = 0, n = 0;
    double omega = 0;
    std::vector<double> e, f, mdiag, wdiag;  // d x d col-major; d
};
// homogeneous.cpp:43-73
static Reduced build_reduced(int m, const Layer& layer, const Quad& q, const Kernel& k) {
    const int n = q.n, d = 4 * n;
    Reduced r;
    r.m = m;
    r.n = n;
    r.omega = layer.omega;
    r.mdiag.resize(d);
    r.wdiag.resize(d);
    for (int i = 0; i < n; ++i)
        for (int c = 0; c < 4; ++c) {
            r.mdiag[4 * i + c] = q.nodes[i];
            r.wdiag[4 * i + c] = q.weights[i];
        }
    std::vector<double> k1((size_t)d * d, 0.0), k2((size_t)d * d, 0.0);
    const double ho = 0.5 * layer.omega;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            const double sc = ho * q.weights[j];
            const M4& app = k.block(true, true, i, j);
            const M4& apm = k.block(true, false, i, j);
            for (int rr = 0; rr < 4; ++rr)
                for (int cc = 0; cc < 4; ++cc) {
                    const size_t at = (size_t)(4 * j + cc) * d + (4 * i + rr);
                    k1[at] = sc * app(rr, cc);
                    k2[at] = sc * apm(rr, cc) * kParity[cc];
                }
        }
    r.e.assign((size_t)d * d, 0.0);
    r.f.assign((size_t)d * d, 0.0);
    for (int j = 0; j < d; ++j) {
        const double inv = 1.0 / r.mdiag[j];
        for (int i = 0; i < d; ++i) {
            const size_t at = (size_t)j * d + i;
            const double id = (i == j) ? 1.0 : 0.0;
            r.e[at] = (id - k1[at] - k2[at]) * inv;
            r.f[at] = (id - k1[at] + k2[at]) * inv;
        }
    }
    return r;
}
// homogeneous.cpp:109-129: M^{-1}((omega/2) A w - I), 8N x 8N col-major.
static std::vector<double> full_op(const Reduced& ops, const Kernel& k) {
    const int n = ops.n, d = 4 * n, D = 2 * d;
    std::vector<double> op((size_t)D * D, 0.0);
    const double ho = 0.5 * ops.omega;
    auto put = [&](int r0, int c0, double s, const M4& b) {
        for (int rr = 0; rr < 4; ++rr)
            for (int cc = 0; cc < 4; ++cc) op[(size_t)(c0 + cc) * D + r0 + rr] = s * b(rr, cc);
    };
    for (int i = 0; i < n; ++i) {
        const double inv_mu = 1.0 / ops.mdiag[4 * i];
        for (int j = 0; j < n; ++j) {
            const double w = ho * ops.wdiag[4 * j];
            put(4 * i, 4 * j, inv_mu * w, k.block(true, true, i, j));
            put(4 * i, d + 4 * j, inv_mu * w, k.block(true, false, i, j));
            put(d + 4 * i, 4 * j, -inv_mu * w, k.block(false, true, i, j));
            put(d + 4 * i, d + 4 * j, -inv_mu * w, k.block(false, false, i, j));
        }
        for (int c = 0; c < 4; ++c) {
            op[(size_t)(4 * i + c) * D + 4 * i + c] -= inv_mu;
            op[(size_t)(d + 4 * i + c) * D + d + 4 * i + c] += inv_mu;
        }
    }
    return op;
}
template <typename T>
static std::vector<T> block_parity(const std::vector<T>& v) {  // homogeneous.cpp:25-41
    std::vector<T> o = v;
    for (size_t i = 0; i + 3 < v.size(); i += 4) {
        o[i + 2] = -v[i + 2];
        o[i + 3] = -v[i + 3];
    }
    return o;
}

// ---------------------------------------------------------------- homogeneous
std::atomic<uint64_t> g_polish_modes{0};  // diagnostic: modes entering the polish loops
// VRTE_ORACLE_ACCURATE=1 (tests only): polish every mode, refine every linear
// solve once -- the same algorithm run to its fp64 accuracy limit, used to
// separate the reference's own rounding error from GPU-vs-reference deviations.
std::atomic<int> g_accurate{-1};
static bool accurate_mode() {
    int v = g_accurate.load();
    if (v < 0) {
        const char* e = std::getenv("VRTE_ORACLE_ACCURATE");
        v = (e && e[0] == '1') ? 1 : 0;
        g_accurate.store(v);
    }
    return v == 1;
}
static double polish_threshold() {
    static const double acc = std::getenv("VRTE_ORACLE_POLISH") ? std::atof(std::getenv("VRTE_ORACLE_POLISH")) : 0.0;
    return accurate_mode() ? acc : 0.5 * kEigenResidualBound;
}
struct Mode {
    cd nu;
    std::vector<cd> psi_plus, psi_minus;
    double residual = 0;
};
struct ModeSet {
    int m = 0, n = 0;
    std::vector<Mode> modes;
    double max_residual = 0;
};
// homogeneous.cpp:131-287 (Eigen::EigenSolver -> LAPACK dgeev).
static ModeSet solve_homogeneous(const Reduced& ops, const Kernel& kern) {
    const int d = 4 * ops.n;
    std::vector<double> fe((size_t)d * d);
    dgemm('N', 'N', d, d, d, 1.0, ops.f.data(), d, ops.e.data(), d, 0.0, fe.data(), d);

    std::vector<double> a = fe, wr(d), wi(d), vr((size_t)d * d);
    {
        int info = 0, lwork = -1, one = 1;
        double wq = 0;
        const char jl = 'N', jr = 'V';
        scipy_dgeev_(&jl, &jr, &d, a.data(), &d, wr.data(), wi.data(), nullptr, &one, vr.data(),
                     &d, &wq, &lwork, &info, 1, 1);
        lwork = (int)wq;
        std::vector<double> work(std::max(lwork, 1));
        scipy_dgeev_(&jl, &jr, &d, a.data(), &d, wr.data(), wi.data(), nullptr, &one, vr.data(),
                     &d, work.data(), &lwork, &info, 1, 1);
        if (info != 0)
            throw NumericalError("eigen decomposition failed at order m = " +
                                 std::to_string(ops.m));
    }
    std::vector<cd> lambdas(d);
    std::vector<std::vector<cd>> vecs(d, std::vector<cd>(d));
    for (int j = 0; j < d; ++j) {
        lambdas[j] = cd(wr[j], wi[j]);
        if (wi[j] == 0.0) {
            for (int i = 0; i < d; ++i) vecs[j][i] = vr[(size_t)j * d + i];
        } else if (wi[j] > 0.0 && j + 1 < d) {
            for (int i = 0; i < d; ++i) {
                vecs[j][i] = cd(vr[(size_t)j * d + i], vr[(size_t)(j + 1) * d + i]);
                vecs[j + 1][i] = std::conj(vecs[j][i]);
            }
        }
    }

    ModeSet set;
    set.m = ops.m;
    set.n = ops.n;
    set.modes.resize(d);
    std::vector<double> inv_m(d);
    for (int i = 0; i < d; ++i) inv_m[i] = 1.0 / ops.mdiag[i];
    const std::vector<double> fop = full_op(ops, kern);
    const int D = 2 * d;
    std::vector<cd> fop_c(fop.begin(), fop.end());
    std::vector<cd> fe_c(fe.begin(), fe.end());
    const double lambda_floor = 1e-12 * std::max(1.0, max_abs(fe));

    for (int j = 0; j < d; ++j) {
        cd lambda = lambdas[j];
        if (!std::isfinite(lambda.real()) || !std::isfinite(lambda.imag()))
            throw NumericalError("non-finite eigenvalue at order m = " + std::to_string(ops.m));
        const bool conservative = std::abs(lambda) < lambda_floor;
        cd nu;
        if (conservative) {
            nu = kNuClamp;
        } else {
            if (lambda.real() < 0.0 && std::abs(lambda.imag()) < 1e-10 * std::abs(lambda.real()) &&
                std::abs(lambda) < 1e-10)
                lambda = std::abs(lambda);
            nu = 1.0 / std::sqrt(lambda);
            if (nu.real() < 0.0) nu = -nu;
            if (nu.real() == 0.0)
                throw NumericalError("eigenvalue on the negative real axis at order m = " +
                                     std::to_string(ops.m));
            if (std::abs(nu) > kNuClamp) nu = kNuClamp * nu / std::abs(nu);
        }
        std::vector<cd> x = vecs[j];
        {
            const double s = max_abs(x);
            for (auto& v : x) v /= s;
        }
        auto recover = [&](const cd& nu_j, const std::vector<cd>& xv) {
            Mode mode;
            mode.nu = nu_j;
            mode.psi_plus.resize(d);
            mode.psi_minus.resize(d);
            if (conservative) {
                for (int i = 0; i < d; ++i) mode.psi_plus[i] = 0.5 * inv_m[i] * xv[i];
                mode.psi_minus = mode.psi_plus;
            } else {
                const std::vector<cd> ex = matvec(ops.e, d, d, xv);
                for (int i = 0; i < d; ++i) {
                    mode.psi_plus[i] = 0.5 * inv_m[i] * (xv[i] - nu_j * ex[i]);
                    mode.psi_minus[i] = 0.5 * inv_m[i] * (xv[i] + nu_j * ex[i]);
                }
            }
            std::vector<cd> v(D);
            const auto pm = block_parity(mode.psi_minus);
            for (int i = 0; i < d; ++i) {
                v[i] = mode.psi_plus[i];
                v[d + i] = pm[i];
            }
            const double vn = max_abs(v);
            std::vector<cd> r = matvec(fop, D, D, v);
            for (int i = 0; i < D; ++i) r[i] -= v[i] / nu_j;
            mode.residual = vn > 0.0 ? max_abs(r) / vn : 0.0;
            return mode;
        };
        Mode mode = recover(nu, x);
        if (!conservative && mode.residual > 0.5 * kEigenResidualBound) g_polish_modes.fetch_add(1);
        // homogeneous.cpp:216-240: half-size inverse-iteration polish.
        for (int pass = 0; pass < 2 && !conservative && mode.residual > polish_threshold();
             ++pass) {
            std::vector<cd> sh = fe_c;
            const cd shift = lambda * (1.0 + 1e-12);
            for (int i = 0; i < d; ++i) sh[(size_t)i * d + i] -= shift;
            ZLu lu(std::move(sh), d);
            std::vector<cd> xr = lu.solve(x);
            if (!all_finite(xr)) break;
            const double s = max_abs(xr);
            for (auto& v : xr) v /= s;
            const std::vector<cd> fx = matvec(fe_c, d, d, xr);
            cd num = 0.0;
            double den = 0.0;
            for (int i = 0; i < d; ++i) {
                num += std::conj(xr[i]) * fx[i];
                den += std::norm(xr[i]);
            }
            const cd lam_r = num / den;
            cd nu_r = 1.0 / std::sqrt(lam_r);
            if (nu_r.real() < 0.0) nu_r = -nu_r;
            if (!(nu_r.real() > 0.0)) break;
            Mode refined = recover(nu_r, xr);
            if (refined.residual < mode.residual) {
                mode = std::move(refined);
                x = xr;
                lambda = lam_r;
            } else {
                break;
            }
        }
        // homogeneous.cpp:241-268: polish on the full 8N operator.
        for (int pass = 0; pass < 2 && !conservative && mode.residual > polish_threshold();
             ++pass) {
            std::vector<cd> v(D);
            const auto pm = block_parity(mode.psi_minus);
            for (int i = 0; i < d; ++i) {
                v[i] = mode.psi_plus[i];
                v[d + i] = pm[i];
            }
            const cd shift = (1.0 / mode.nu) * (1.0 + 1e-12);
            std::vector<cd> sh = fop_c;
            for (int i = 0; i < D; ++i) sh[(size_t)i * D + i] -= shift;
            ZLu lu(std::move(sh), D);
            std::vector<cd> w = lu.solve(v);
            if (!all_finite(w)) break;
            const double s = max_abs(w);
            for (auto& z : w) z /= s;
            const std::vector<cd> ow = matvec(fop_c, D, D, w);
            cd num = 0.0;
            double den = 0.0;
            for (int i = 0; i < D; ++i) {
                num += std::conj(w[i]) * ow[i];
                den += std::norm(w[i]);
            }
            const cd inv_nu = num / den;
            if (!(inv_nu.real() > 0.0)) break;
            Mode refined;
            refined.nu = 1.0 / inv_nu;
            refined.psi_plus.assign(w.begin(), w.begin() + d);
            refined.psi_minus = block_parity(std::vector<cd>(w.begin() + d, w.end()));
            std::vector<cd> r = ow;
            for (int i = 0; i < D; ++i) r[i] -= inv_nu * w[i];
            refined.residual = max_abs(r) / max_abs(w);
            if (refined.residual < mode.residual)
                mode = std::move(refined);
            else
                break;
        }
        set.modes[j] = std::move(mode);
    }
    std::sort(set.modes.begin(), set.modes.end(), [](const Mode& a, const Mode& b) {
        if (a.nu.real() != b.nu.real()) return a.nu.real() > b.nu.real();
        return a.nu.imag() < b.nu.imag();
    });
    for (const auto& md : set.modes) set.max_residual = std::max(set.max_residual, md.residual);
    if (set.max_residual > kEigenResidualBound) {
        char buf[256];
        std::snprintf(buf, sizeof buf,
                      "homogeneous mode residual %g exceeds %g at order m = %d (|FE| ~ %g)",
                      set.max_residual, kEigenResidualBound, ops.m, max_abs(fe));
        throw NumericalError(buf);
    }
    return set;
}

// ---------------------------------------------------------------- particular
struct Source {
    std::vector<double> xp, xm;
    double mu0 = 1.0;
};
// particular.cpp:7-25. `stokes` is I0; k in {1,2} selects D_k.
static Source build_source(int m, int k, const Layer& layer, double mu0, const double* stokes,
                           const Quad& q) {
    const int n = q.n;
    Source s;
    s.mu0 = mu0;
    s.xp.assign(4 * n, 0.0);
    s.xm.assign(4 * n, 0.0);
    if (layer.omega == 0.0) return s;
    const KColumn col = beam_column(m, layer, q, -mu0);
    double sel[4];
    for (int c = 0; c < 4; ++c) sel[c] = ((k == 1) == (c < 2)) ? stokes[c] : 0.0;
    const double sc = layer.omega / (2.0 * kPi);
    for (int i = 0; i < n; ++i)
        for (int r = 0; r < 4; ++r) {
            double u = 0, dn = 0;
            for (int c = 0; c < 4; ++c) {
                u += col.up[i](r, c) * sel[c];
                dn += col.down[i](r, c) * sel[c];
            }
            s.xp[4 * i + r] = sc * u;
            s.xm[4 * i + r] = sc * dn;
        }
    return s;
}
struct Part {
    std::vector<double> zp, zm, g;
    double mu0_eff = 1.0, residual = 0;
    bool dithered = false;
};
// particular.cpp:27-107
static Part solve_particular(const Reduced& ops, const Source& src, const ModeSet& modes,
                             const Kernel& kern) {
    const int d = 4 * ops.n;
    Part out;
    out.mu0_eff = src.mu0;
    out.zp.assign(d, 0.0);
    out.zm.assign(d, 0.0);
    out.g.assign(d, 0.0);
    if (std::max(max_abs(src.xp), max_abs(src.xm)) == 0.0) return out;
    double mu0 = src.mu0;
    for (const auto& md : modes.modes) {
        const cd lam = 1.0 / (md.nu * md.nu);
        if (std::abs(lam - 1.0 / (mu0 * mu0)) < 1e-8 * std::abs(lam)) {
            mu0 *= (1.0 - 1e-7);
            out.dithered = true;
            break;
        }
    }
    out.mu0_eff = mu0;
    const auto pxm = block_parity(src.xm);
    std::vector<double> sp(d), sm(d);
    for (int i = 0; i < d; ++i) {
        sp[i] = src.xp[i] + pxm[i];
        sm[i] = src.xp[i] - pxm[i];
    }
    std::vector<double> lhs((size_t)d * d);
    dgemm('N', 'N', d, d, d, 1.0, ops.f.data(), d, ops.e.data(), d, 0.0, lhs.data(), d);
    for (int i = 0; i < d; ++i) lhs[(size_t)i * d + i] -= 1.0 / (mu0 * mu0);
    std::vector<double> rhs = matvec(ops.f, d, d, sp);
    for (int i = 0; i < d; ++i) rhs[i] -= sm[i] / mu0;
    DLu lu(lhs, d);
    std::vector<double> g = lu.solve(rhs);
    if (accurate_mode()) {
        std::vector<double> r = matvec(lhs, d, d, g);
        for (int i = 0; i < d; ++i) r[i] = rhs[i] - r[i];
        const std::vector<double> dg = lu.solve(r);
        for (int i = 0; i < d; ++i) g[i] += dg[i];
    }
    {
        std::vector<double> r = matvec(lhs, d, d, g);
        for (int i = 0; i < d; ++i) r[i] -= rhs[i];
        const double sys_res = max_abs(r);
        const double scale = max_abs(rhs) + max_abs(lhs) * max_abs(g);
        if (!all_finite(g) || sys_res > 1e-8 * std::max(scale, 1e-300)) {
            char buf[160];
            std::snprintf(buf, sizeof buf, "singular beam-response system at order m = %d, mu0 = %g",
                          ops.m, src.mu0);
            throw NumericalError(buf);
        }
    }
    const std::vector<double> eg = matvec(ops.e, d, d, g);
    std::vector<double> psip(d), psim(d);
    for (int i = 0; i < d; ++i) {
        const double h = mu0 * (sp[i] - eg[i]);
        psip[i] = 0.5 / ops.mdiag[i] * (g[i] + h);
        psim[i] = 0.5 / ops.mdiag[i] * (g[i] - h);
    }
    out.g = g;
    out.zp = psip;
    out.zm = block_parity(psim);
    // particular.cpp:86-105: unreduced balance residual.
    const std::vector<double> fop = full_op(ops, kern);
    const int D = 2 * d;
    std::vector<double> z(D), minvx(D);
    for (int i = 0; i < d; ++i) {
        z[i] = out.zp[i];
        z[d + i] = out.zm[i];
        minvx[i] = src.xp[i] / ops.mdiag[i];
        minvx[d + i] = -src.xm[i] / ops.mdiag[i];
    }
    std::vector<double> rv = matvec(fop, D, D, z);
    for (int i = 0; i < D; ++i) rv[i] += minvx[i] - z[i] / mu0;
    out.residual = max_abs(rv) / std::max(max_abs(minvx), 1e-300);
    if (out.residual > 1e-6) {
        char buf[160];
        std::snprintf(buf, sizeof buf, "beam-response residual %g at order m = %d", out.residual,
                      ops.m);
        throw NumericalError(buf);
    }
    return out;
}

// ---------------------------------------------------------------- boundary
static std::vector<cd> mode_exp_at(const ModeSet& ms, double t) {  // boundary.cpp:11-16
    std::vector<cd> e(ms.modes.size());
    for (size_t j = 0; j < ms.modes.size(); ++j) e[j] = std::exp(-t / ms.modes[j].nu);
    return e;
}
// boundary.cpp:37-71 bilinear table rows (Lambertian: 2 rho in (0,0)).
static M4 base_row_at(const Base& base, const Quad& q, double mu_out, double mu_in) {
    M4 r;
    if (base.type == 0) return r;
    if (base.type == 1) {
        r(0, 0) = 2.0 * base.rho;
        return r;
    }
    auto interp = [&](double mu, int& lo, double& w) {
        const auto& nd = q.nodes;
        if (mu <= nd.front()) {
            lo = 0;
            w = 0.0;
            return;
        }
        if (mu >= nd.back()) {
            lo = q.n - 2 >= 0 ? q.n - 2 : 0;
            w = q.n >= 2 ? 1.0 : 0.0;
            return;
        }
        lo = 0;
        while (lo + 1 < q.n && nd[lo + 1] < mu) ++lo;
        w = (mu - nd[lo]) / (nd[lo + 1] - nd[lo]);
    };
    int li, lj;
    double wi, wj;
    interp(mu_out, li, wi);
    interp(mu_in, lj, wj);
    const int i1 = std::min(li + 1, q.n - 1), j1 = std::min(lj + 1, q.n - 1);
    for (int e = 0; e < 16; ++e)
        r.v[e] = (1 - wi) * (1 - wj) * base.at(li, lj).v[e] + (1 - wi) * wj * base.at(li, j1).v[e] +
                 wi * (1 - wj) * base.at(i1, lj).v[e] + wi * wj * base.at(i1, j1).v[e];
    return r;
}
// boundary.cpp:73-97
static std::vector<cd> reflect_down(const Base& base, const Quad& q, const std::vector<cd>& down) {
    const int n = q.n;
    std::vector<cd> out(4 * n, 0.0);
    if (base.type == 0) return out;
    if (base.type == 1) {
        cd flux = 0.0;
        for (int j = 0; j < n; ++j) flux += q.weights[j] * q.nodes[j] * down[4 * j];
        const cd val = 2.0 * base.rho * flux;
        for (int i = 0; i < n; ++i) out[4 * i] = val;
        return out;
    }
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            const M4& t = base.at(i, j);
            const double wm = q.weights[j] * q.nodes[j];
            for (int r = 0; r < 4; ++r) {
                cd s = 0.0;
                for (int c = 0; c < 4; ++c) s += t(r, c) * down[4 * j + c];
                out[4 * i + r] += wm * s;
            }
        }
    return out;
}
struct BaseRefl {
    bool active = false;
    std::vector<cd> lref_h;  // d x 2d col-major
    std::vector<double> lref_p, lref_s;
};
// boundary.cpp:99-140
static BaseRefl build_base_reflection(const Base& base, const Quad& q, int m, int k, double mu0,
                                      const double* stokes, const ModeSet& bm, const Part& bp,
                                      double bottom_tau, double beam_at_base) {
    BaseRefl rf;
    const int n = q.n, d = 4 * n, nm = (int)bm.modes.size();
    if (base.type == 0 || m > 0) return rf;
    if (base.type == 1 && base.rho == 0.0) return rf;
    rf.active = true;
    rf.lref_h.assign((size_t)d * 2 * nm, 0.0);
    const std::vector<cd> ea = mode_exp_at(bm, bottom_tau);
    for (int j = 0; j < nm; ++j) {
        std::vector<cd> a = block_parity(bm.modes[j].psi_minus);
        for (auto& v : a) v *= ea[j];
        const auto ra = reflect_down(base, q, a);
        const auto rb = reflect_down(base, q, block_parity(bm.modes[j].psi_plus));
        std::copy(ra.begin(), ra.end(), rf.lref_h.begin() + (size_t)j * d);
        std::copy(rb.begin(), rb.end(), rf.lref_h.begin() + (size_t)(nm + j) * d);
    }
    {
        std::vector<cd> zm(d);
        for (int i = 0; i < d; ++i) zm[i] = beam_at_base * bp.zm[i];
        const auto rp = reflect_down(base, q, zm);
        rf.lref_p.resize(d);
        for (int i = 0; i < d; ++i) rf.lref_p[i] = rp[i].real();
    }
    auto beam_row = [&](const M4& r) {
        double s[4];
        for (int a = 0; a < 4; ++a) {
            double acc = 0;
            for (int c = 0; c < 4; ++c) acc += r(a, c) * stokes[c];
            s[a] = (mu0 / kPi) * acc * beam_at_base;
        }
        for (int a = 0; a < 4; ++a)
            if ((k == 1) != (a < 2)) s[a] = 0.0;
        return std::vector<double>(s, s + 4);
    };
    rf.lref_s.assign(d, 0.0);
    if (base.type == 1) {
        const auto s = beam_row(base_row_at(base, q, q.nodes[0], mu0));
        for (int i = 0; i < n; ++i)
            for (int a = 0; a < 4; ++a) rf.lref_s[4 * i + a] = s[a];
    } else {
        for (int i = 0; i < n; ++i) {
            const auto s = beam_row(base_row_at(base, q, q.nodes[i], mu0));
            for (int a = 0; a < 4; ++a) rf.lref_s[4 * i + a] = s[a];
        }
    }
    return rf;
}
struct LayerCoef {
    std::vector<cd> a, b;
};
struct OrderBoundary {
    std::vector<LayerCoef> coef[2];
    double condition = 0, residual = 0;
};
// Memo of one order's boundary left-hand side and its LU (tests only, see
// oracle_set_cache_boundary): the LHS carries no incident or k dependence
// (boundary.cpp:219), so reusing the factors of the identical matrix leaves
// every solution bit for bit unchanged and only skips the rebuild.
std::atomic<int> g_cache_boundary{0};
struct BoundaryLhs {
    std::vector<cd> lhs;
    double anorm1 = 0.0, lhs_norm = 0.0, condition = 0.0;
    std::unique_ptr<ZLu> lu;
    std::mutex mu;
};
// boundary.cpp:142-265: complex global block system, LU, 2 RHS, refinement.
static OrderBoundary solve_boundary(const Material& spec, double mu0, const double* stokes,
                                    const Quad& q, int m, const std::vector<const ModeSet*>& modes,
                                    const std::vector<const Part*> parts[2], BoundaryLhs* memo = nullptr) {
    const int n = q.n, d = 4 * n, P = (int)spec.layers.size(), blk = 2 * d, G = blk * P;
    std::vector<double> tau_top(P, 0.0);
    for (int p = 1; p < P; ++p) tau_top[p] = tau_top[p - 1] + spec.layers[p - 1].tau;
    const double tau_total = tau_top[P - 1] + spec.layers[P - 1].tau;
    std::vector<std::vector<cd>> att(P);
    for (int p = 0; p < P; ++p) att[p] = mode_exp_at(*modes[p], spec.layers[p].tau);

    std::unique_lock<std::mutex> memo_lock;
    if (memo) memo_lock = std::unique_lock<std::mutex>(memo->mu);
    const bool have_lhs = memo && memo->lu;
    std::vector<cd> lhs_own(have_lhs ? 0 : (size_t)G * G, 0.0);
    std::vector<cd>& lhs = have_lhs ? memo->lhs : lhs_own;
    std::vector<cd> rhs[2] = {std::vector<cd>(G, 0.0), std::vector<cd>(G, 0.0)};
    auto put = [&](int col, int row0, const std::vector<cd>& v, cd s) {
        if (have_lhs) return;
        cd* c = lhs.data() + (size_t)col * G + row0;
        for (int i = 0; i < d; ++i) c[i] = s * v[i];
    };
    auto ca = [&](int p, int j) { return blk * p + j; };
    auto cb = [&](int p, int j) { return blk * p + d + j; };
    for (int j = 0; j < d; ++j) {
        const Mode& md = modes[0]->modes[j];
        put(ca(0, j), 0, block_parity(md.psi_minus), 1.0);
        put(cb(0, j), 0, block_parity(md.psi_plus), att[0][j]);
    }
    for (int k = 0; k < 2; ++k)
        for (int i = 0; i < d; ++i) rhs[k][i] = -parts[k][0]->zm[i];
    for (int p = 0; p + 1 < P; ++p) {
        const int ru = d + 2 * d * p, rd = ru + d;
        for (int j = 0; j < d; ++j) {
            const Mode& mp = modes[p]->modes[j];
            put(ca(p, j), ru, mp.psi_plus, att[p][j]);
            put(cb(p, j), ru, mp.psi_minus, 1.0);
            put(ca(p, j), rd, block_parity(mp.psi_minus), att[p][j]);
            put(cb(p, j), rd, block_parity(mp.psi_plus), 1.0);
            const Mode& mq = modes[p + 1]->modes[j];
            put(ca(p + 1, j), ru, mq.psi_plus, -1.0);
            put(cb(p + 1, j), ru, mq.psi_minus, -att[p + 1][j]);
            put(ca(p + 1, j), rd, block_parity(mq.psi_minus), -1.0);
            put(cb(p + 1, j), rd, block_parity(mq.psi_plus), -att[p + 1][j]);
        }
        const double bn = std::exp(-tau_top[p + 1] / mu0);
        for (int k = 0; k < 2; ++k)
            for (int i = 0; i < d; ++i) {
                rhs[k][ru + i] = bn * (parts[k][p + 1]->zp[i] - parts[k][p]->zp[i]);
                rhs[k][rd + i] = bn * (parts[k][p + 1]->zm[i] - parts[k][p]->zm[i]);
            }
    }
    const int rb = d + 2 * d * (P - 1), qq = P - 1;
    const double beam_base = std::exp(-tau_total / mu0);
    BaseRefl refl[2];
    for (int k = 0; k < 2; ++k)
        refl[k] = build_base_reflection(spec.base, q, m, k + 1, mu0, stokes, *modes[qq],
                                        *parts[k][qq], spec.layers[qq].tau, beam_base);
    for (int j = 0; j < d; ++j) {
        const Mode& md = modes[qq]->modes[j];
        put(ca(qq, j), rb, md.psi_plus, att[qq][j]);
        put(cb(qq, j), rb, md.psi_minus, 1.0);
        if (refl[0].active && !have_lhs) {
            cd* c1 = lhs.data() + (size_t)ca(qq, j) * G + rb;
            cd* c2 = lhs.data() + (size_t)cb(qq, j) * G + rb;
            for (int i = 0; i < d; ++i) {
                c1[i] -= refl[0].lref_h[(size_t)j * d + i];
                c2[i] -= refl[0].lref_h[(size_t)(d + j) * d + i];
            }
        }
    }
    for (int k = 0; k < 2; ++k)
        for (int i = 0; i < d; ++i) {
            rhs[k][rb + i] = -(beam_base * parts[k][qq]->zp[i]);
            if (refl[k].active) rhs[k][rb + i] += refl[k].lref_p[i] + refl[k].lref_s[i];
        }

    double anorm1 = 0.0, lhs_norm = 0.0;
    std::unique_ptr<ZLu> lu_own;
    OrderBoundary out;
    if (have_lhs) {
        anorm1 = memo->anorm1;
        lhs_norm = memo->lhs_norm;
        out.condition = memo->condition;
    } else {
        for (int j = 0; j < G; ++j) {
            double cs = 0;
            for (int i = 0; i < G; ++i) {
                const double a = std::abs(lhs[(size_t)j * G + i]);
                cs += a;
                lhs_norm = std::max(lhs_norm, a);
            }
            anorm1 = std::max(anorm1, cs);
        }
        lu_own = std::make_unique<ZLu>(lhs, G);
        out.condition = 1.0 / std::max(lu_own->rcond(anorm1), 1e-300);
        if (memo) {
            memo->anorm1 = anorm1;
            memo->lhs_norm = lhs_norm;
            memo->condition = out.condition;
            memo->lhs = std::move(lhs_own);
            memo->lu = std::move(lu_own);
        }
    }
    const ZLu& lu = memo ? *memo->lu : *lu_own;
    const std::vector<cd>& A = memo ? memo->lhs : lhs_own;
    for (int k = 0; k < 2; ++k) {
        std::vector<cd> c = lu.solve(rhs[k]);
        const double rn = max_abs(rhs[k]);
        auto resid_of = [&](const std::vector<cd>& x) {
            std::vector<cd> r = matvec(A, G, G, x);
            for (int i = 0; i < G; ++i) r[i] -= rhs[k][i];
            return r;
        };
        double scale = lhs_norm * std::max(max_abs(c), 1e-300) + rn;
        double resid = max_abs(resid_of(c));
        // accurate mode: VRTE_ORACLE_BND_STEPS refinement steps (default 1)
        static const int acc_steps =
            std::getenv("VRTE_ORACLE_BND_STEPS") ? std::atoi(std::getenv("VRTE_ORACLE_BND_STEPS")) : 1;
        const int steps = accurate_mode() ? acc_steps : (resid > 1e-10 * scale ? 1 : 0);
        for (int it = 0; it < steps; ++it) {
            std::vector<cd> r = resid_of(c);
            for (auto& v : r) v = -v;
            const std::vector<cd> dc = lu.solve(r);
            for (int i = 0; i < G; ++i) c[i] += dc[i];
            resid = max_abs(resid_of(c));
            scale = lhs_norm * std::max(max_abs(c), 1e-300) + rn;
        }
        if (!all_finite(c) || (rn > 0.0 && resid > 1e-9 * scale)) {
            char buf[200];
            std::snprintf(buf, sizeof buf,
                          "boundary system ill-conditioned at order m = %d (condition ~ %g, "
                          "residual %g)",
                          m, out.condition, resid);
            throw NumericalError(buf);
        }
        out.residual = std::max(out.residual, rn > 0 ? resid / scale : 0.0);
        out.coef[k].resize(P);
        for (int p = 0; p < P; ++p) {
            out.coef[k][p].a.assign(c.begin() + blk * p, c.begin() + blk * p + d);
            out.coef[k][p].b.assign(c.begin() + blk * p + d, c.begin() + blk * p + 2 * d);
        }
    }
    return out;
}

// ---------------------------------------------------------------- pipeline
template <typename Fn>
static void parallel_for(int threads, size_t count, Fn&& fn) {
    if (threads <= 1 || count <= 1) {
        for (size_t i = 0; i < count; ++i) fn(i);
        return;
    }
    std::atomic<size_t> next{0};
    std::vector<std::thread> pool;
    const int nt = (int)std::min<size_t>(threads, count);
    for (int t = 0; t < nt; ++t)
        pool.emplace_back([&] {
            for (size_t i = next.fetch_add(1); i < count; i = next.fetch_add(1)) fn(i);
        });
    for (auto& th : pool) th.join();
}
static double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

// ---------------------------------------------------------------- radiance reconstruction
// reconstruction.cpp:28-199: source-function integration along an arbitrary
// direction, per (order, k) chain of layers.
using V4c = std::array<cd, 4>;
struct SrcCoeffs {
    std::vector<std::pair<cd, V4c>> from_top, from_bottom;
    V4c beam{};
    double mu0 = 1.0, thickness = 0.0;
};
static void add4(V4c& a, cd s, const V4c& x) {
    for (int c = 0; c < 4; ++c) a[c] += s * x[c];
}
static V4c mat4v(const M4& a, const cd* x) {  // A (real 4x4) * complex 4-vector
    V4c o{};
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) o[r] += a(r, c) * x[c];
    return o;
}
struct ChainEntry {
    const Layer* layer;
    const ModeSet* modes;
    const Part* part;
    std::vector<cd> coef_a, coef_b;
    double tau_top, thickness, beam_top;
};
// reconstruction.cpp:28-72
static SrcCoeffs source_coefficients(const ChainEntry& e, const Quad& q, int k, double mu0, const double* stokes,
                                     const KRow& row, const M4& beam_block) {
    const int n = q.n;
    const double half_omega = 0.5 * e.layer->omega;
    SrcCoeffs out;
    out.mu0 = mu0;
    out.thickness = e.thickness;
    std::vector<M4> wp(n), wm(n);
    for (int i = 0; i < n; ++i) {
        axpy4(wp[i], q.weights[i], row.plus[i]);
        axpy4(wm[i], q.weights[i], row.minus[i]);
    }
    for (size_t j = 0; j < e.modes->modes.size(); ++j) {
        const Mode& md = e.modes->modes[j];
        const auto down_a = block_parity(md.psi_minus), down_b = block_parity(md.psi_plus);
        V4c aa{}, ab{};
        for (int i = 0; i < n; ++i) {
            const V4c t1 = mat4v(wp[i], &md.psi_plus[4 * i]), t2 = mat4v(wm[i], &down_a[4 * i]);
            const V4c t3 = mat4v(wp[i], &md.psi_minus[4 * i]), t4 = mat4v(wm[i], &down_b[4 * i]);
            for (int c = 0; c < 4; ++c) {
                aa[c] += t1[c] + t2[c];
                ab[c] += t3[c] + t4[c];
            }
        }
        V4c ta{}, tb{};
        add4(ta, half_omega * e.coef_a[j], aa);
        add4(tb, half_omega * e.coef_b[j], ab);
        out.from_top.emplace_back(md.nu, ta);
        out.from_bottom.emplace_back(md.nu, tb);
    }
    V4c beam{};
    for (int i = 0; i < n; ++i) {
        cd zp[4], zm[4];
        for (int c = 0; c < 4; ++c) {
            zp[c] = e.part->zp[4 * i + c];
            zm[c] = e.part->zm[4 * i + c];
        }
        const V4c t1 = mat4v(wp[i], zp), t2 = mat4v(wm[i], zm);
        for (int c = 0; c < 4; ++c) beam[c] += t1[c] + t2[c];
    }
    for (auto& b : beam) b *= half_omega;
    cd sel[4];
    for (int c = 0; c < 4; ++c) sel[c] = ((k == 1) == (c < 2)) ? stokes[c] : 0.0;  // kernel.cpp:124-128
    const V4c bb = mat4v(beam_block, sel);
    add4(beam, e.layer->omega / (2.0 * kPi), bb);
    for (int c = 0; c < 4; ++c) out.beam[c] = e.beam_top * beam[c];
    return out;
}
constexpr double kDegenerateRate = 1e-9;  // reconstruction.cpp:85
// reconstruction.cpp:87-121
static V4c up_top(cd a, const V4c& c, double mu, double t, double d) {
    const cd f = (std::exp(-t / a) - std::exp(-d / a) * std::exp(-(d - t) / mu)) / (1.0 + mu / a);
    V4c o;
    for (int q = 0; q < 4; ++q) o[q] = c[q] * f;
    return o;
}
static V4c up_bottom(cd b, const V4c& c, double mu, double t, double d) {
    cd f;
    if (std::abs(1.0 / mu - 1.0 / b) < kDegenerateRate)
        f = std::exp(-(d - t) / mu) * ((d - t) / mu);
    else
        f = (std::exp(-(d - t) / b) - std::exp(-(d - t) / mu)) / (1.0 - mu / b);
    V4c o;
    for (int q = 0; q < 4; ++q) o[q] = c[q] * f;
    return o;
}
static V4c down_top(cd a, const V4c& c, double mu, double t) {
    cd f;
    if (std::abs(1.0 / mu - 1.0 / a) < kDegenerateRate)
        f = std::exp(-t / mu) * (t / mu);
    else
        f = (std::exp(-t / a) - std::exp(-t / mu)) / (1.0 - mu / a);
    V4c o;
    for (int q = 0; q < 4; ++q) o[q] = c[q] * f;
    return o;
}
static V4c down_bottom(cd b, const V4c& c, double mu, double t, double d) {
    const cd f = (std::exp(-(d - t) / b) - std::exp(-d / b) * std::exp(-t / mu)) / (1.0 + mu / b);
    V4c o;
    for (int q = 0; q < 4; ++q) o[q] = c[q] * f;
    return o;
}
// reconstruction.cpp:123-149
static V4c integrate_up(const SrcCoeffs& s, double mu, double t, const V4c& ib) {
    const double d = s.thickness;
    V4c v;
    for (int q = 0; q < 4; ++q) v[q] = ib[q] * std::exp(-(d - t) / mu);
    for (const auto& [a, c] : s.from_top) add4(v, 1.0, up_top(a, c, mu, t, d));
    for (const auto& [b, c] : s.from_bottom) add4(v, 1.0, up_bottom(b, c, mu, t, d));
    add4(v, 1.0, up_top(cd(s.mu0, 0.0), s.beam, mu, t, d));
    return v;
}
static V4c integrate_down(const SrcCoeffs& s, double mu, double t, const V4c& it) {
    const double d = s.thickness;
    V4c v;
    for (int q = 0; q < 4; ++q) v[q] = it[q] * std::exp(-t / mu);
    for (const auto& [a, c] : s.from_top) add4(v, 1.0, down_top(a, c, mu, t));
    for (const auto& [b, c] : s.from_bottom) add4(v, 1.0, down_bottom(b, c, mu, t, d));
    add4(v, 1.0, down_top(cd(s.mu0, 0.0), s.beam, mu, t));
    return v;
}
// boundary.cpp:20-35 (chain_stacks): up/down nodal stacks of one chain entry at local depth t
static void chain_stacks(const ChainEntry& e, double mu0, double t, std::vector<cd>& up, std::vector<cd>& down) {
    const int d = (int)e.part->zp.size();
    up.assign(d, 0.0);
    down.assign(d, 0.0);
    for (size_t j = 0; j < e.modes->modes.size(); ++j) {
        const Mode& md = e.modes->modes[j];
        const cd ea = e.coef_a[j] * std::exp(-t / md.nu);
        const cd eb = e.coef_b[j] * std::exp(-(e.thickness - t) / md.nu);
        const auto dm = block_parity(md.psi_minus), dp = block_parity(md.psi_plus);
        for (int i = 0; i < d; ++i) {
            up[i] += ea * md.psi_plus[i] + eb * md.psi_minus[i];
            down[i] += ea * dm[i] + eb * dp[i];
        }
    }
    const double beam = e.beam_top * std::exp(-t / mu0);
    for (int i = 0; i < d; ++i) {
        up[i] += beam * e.part->zp[i];
        down[i] += beam * e.part->zm[i];
    }
}
// reconstruction.cpp:151-199
static std::vector<V4c> reconstruct_component(const std::vector<ChainEntry>& chain, const Quad& q, int m, int k,
                                              double mu0, const double* stokes, const Base& base, double mu_signed,
                                              const std::vector<double>& taus, const std::vector<KRow>& rows,
                                              const std::vector<M4>& beam_blocks) {
    const int P = (int)chain.size();
    const double mu = std::abs(mu_signed);
    std::vector<SrcCoeffs> co(P);
    for (int p = 0; p < P; ++p) co[p] = source_coefficients(chain[p], q, k, mu0, stokes, rows[p], beam_blocks[p]);
    std::vector<std::pair<int, double>> tg(taus.size());
    for (size_t it = 0; it < taus.size(); ++it) {  // reconstruction.cpp:12-19 locate_layer
        int p = 0;
        while (p + 1 < P && taus[it] >= chain[p].tau_top + chain[p].thickness) ++p;
        tg[it] = {p, std::clamp(taus[it] - chain[p].tau_top, 0.0, chain[p].thickness)};
    }
    std::vector<V4c> out(taus.size(), V4c{});
    V4c bnd{};
    if (mu_signed <= 0.0) {
        for (int p = 0; p < P; ++p) {
            for (size_t it = 0; it < taus.size(); ++it)
                if (tg[it].first == p) out[it] = integrate_down(co[p], mu, tg[it].second, bnd);
            bnd = integrate_down(co[p], mu, chain[p].thickness, bnd);
        }
        return out;
    }
    if (m == 0 && base.type != 0) {
        const ChainEntry& last = chain.back();
        const double tau_total = last.tau_top + last.thickness;
        std::vector<cd> upn, dnn;
        chain_stacks(last, mu0, last.thickness, upn, dnn);
        for (int j = 0; j < q.n; ++j) {
            const M4 r = base_row_at(base, q, mu, q.nodes[j]);
            const V4c v = mat4v(r, &dnn[4 * j]);
            add4(bnd, q.weights[j] * q.nodes[j], v);
        }
        const M4 rb = base_row_at(base, q, mu, mu0);
        double sv[4] = {0, 0, 0, 0};
        for (int r = 0; r < 4; ++r)
            for (int c = 0; c < 4; ++c) sv[r] += rb(r, c) * stokes[c];
        const double f = (mu0 / kPi) * std::exp(-tau_total / mu0);
        for (int c = 0; c < 4; ++c)
            if ((k == 1) == (c < 2)) bnd[c] += f * sv[c];
    }
    for (int p = P - 1; p >= 0; --p) {
        for (size_t it = 0; it < taus.size(); ++it)
            if (tg[it].first == p) out[it] = integrate_up(co[p], mu, tg[it].second, bnd);
        bnd = integrate_up(co[p], mu, 0.0, bnd);
    }
    return out;
}
// reconstruction.cpp:201-227
static void assemble_field(const std::vector<std::array<V4c, 2>>& comps, double dphi, double out[4]) {
    const double x = -dphi;
    cd tot[4] = {0, 0, 0, 0};
    double scale = 0.0, imag = 0.0;
    for (size_t m = 0; m < comps.size(); ++m) {
        const double sc = (m == 0) ? 1.0 : 2.0, c = std::cos(m * x), s = std::sin(m * x);
        const double p1[4] = {sc * c, sc * c, sc * s, sc * s}, p2[4] = {-sc * s, -sc * s, sc * c, sc * c};
        for (int q = 0; q < 4; ++q) {
            tot[q] += 0.5 * (p1[q] * comps[m][0][q] + p2[q] * comps[m][1][q]);
            scale = std::max({scale, std::abs(comps[m][0][q]), std::abs(comps[m][1][q])});
        }
    }
    for (int q = 0; q < 4; ++q) imag = std::max(imag, std::abs(tot[q].imag()));
    if (imag > 1e-9 * scale + 1e-300) {
        char buf[200];
        std::snprintf(buf, sizeof buf,
                      "imaginary residue %g exceeds tolerance (scale %g); conjugate mode pairing is broken", imag,
                      scale);
        throw NumericalError(buf);
    }
    for (int q = 0; q < 4; ++q) out[q] = tot[q].real();
}
static double reduce_azimuth(double phi) {  // types.cpp:7-12
    double r = std::fmod(phi, kTwoPi);
    if (r < 0.0) r += kTwoPi;
    return r;
}

// ---------------------------------------------------------------- Monte Carlo (mc.cpp:1-315)
// Polarized photon tracer restated for the statistical cross-checks of
// SURVEY §8(f) rank 4.  Per-photon xoshiro256++ streams, tabulated inverse CDF
// of the intensity phase function, meridian-frame Stokes rotations, fixed
// 16384-photon blocks merged in order (thread-count independent).
struct McRng {  // mc.cpp:11-45
    uint64_t s[4];
    static uint64_t splitmix(uint64_t& x) {
        x += 0x9e3779b97f4a7c15ull;
        uint64_t z = x;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    McRng(uint64_t seed, uint64_t stream) {
        uint64_t x = seed ^ (0x9e3779b97f4a7c15ull * (stream + 1));
        for (auto& w : s) w = splitmix(x);
    }
    static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
    uint64_t next() {
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
    double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};
static double scalar_phase(const Layer& layer, double x) {  // kernel.cpp:179-186
    const int lmax = layer.order_count() - 1;
    const auto d00 = wigner_seq(0, 0, lmax, x);
    double a1 = 0.0;
    for (int l = 0; l <= lmax; ++l) a1 += layer.coeffs[l](0, 0) * d00[l];
    return a1;
}
struct McPdf {  // mc.cpp:47-88
    static constexpr int kCells = 2048;
    std::vector<double> cdf, density;
    explicit McPdf(const Layer& layer) {
        cdf.assign(kCells + 1, 0.0);
        density.assign(kCells, 0.0);
        const double dx = 2.0 / kCells;
        double prev = std::max(0.0, scalar_phase(layer, -1.0)), total = 0.0;
        for (int i = 0; i < kCells; ++i) {
            const double x1 = std::min(-1.0 + dx * (i + 1), 1.0);
            const double cur = std::max(0.0, scalar_phase(layer, x1));
            total += 0.5 * (prev + cur) * dx;
            cdf[i + 1] = total;
            prev = cur;
        }
        if (total <= 0.0) throw ValidationError("mc: intensity phase function has no positive mass");
        for (auto& c : cdf) c /= total;
        for (int i = 0; i < kCells; ++i) density[i] = (cdf[i + 1] - cdf[i]) / dx;
    }
    std::pair<double, double> sample(double u) const {
        int lo = 0, hi = kCells;
        while (hi - lo > 1) {
            const int mid = (lo + hi) / 2;
            (cdf[mid] <= u ? lo : hi) = mid;
        }
        const double mass = cdf[lo + 1] - cdf[lo];
        const double frac = mass > 0.0 ? (u - cdf[lo]) / mass : 0.5;
        const double dx = 2.0 / kCells;
        const double x = std::clamp(-1.0 + dx * (lo + frac), -1.0, 1.0);
        return {x, std::max(density[lo], 1e-300)};
    }
};
using V3 = std::array<double, 3>;
static V3 v3norm(V3 a) {
    const double n = std::sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
    return {a[0] / n, a[1] / n, a[2] / n};
}
static V3 cross(const V3& a, const V3& b) {
    return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}
static double dot(const V3& a, const V3& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
static V3 unit_dir(double mu, double phi) {  // types.hpp:94-97
    const double sn = std::sqrt(std::max(0.0, 1.0 - mu * mu));
    return {sn * std::cos(phi), sn * std::sin(phi), mu};
}
static V3 rotate_direction(const V3& d, double ct, double psi) {  // mc.cpp:107-114
    const double st = std::sqrt(std::max(0.0, 1.0 - ct * ct));
    const V3 a = std::abs(d[2]) < 0.99 ? V3{0, 0, 1} : V3{1, 0, 0};
    const V3 t1 = v3norm(cross(d, a)), t2 = cross(d, t1);
    const double c = std::cos(psi), sn = std::sin(psi);
    return v3norm({ct * d[0] + st * (c * t1[0] + sn * t2[0]), ct * d[1] + st * (c * t1[1] + sn * t2[1]),
                   ct * d[2] + st * (c * t1[2] + sn * t2[2])});
}
static V3 nudge_off_pole(V3 d) {  // rotation.cpp:9-15
    if (1.0 - std::abs(d[2]) < 1e-12) {
        d[0] += 1e-9;
        d = v3norm(d);
    }
    return d;
}
static void meridian_basis(const V3& dir, V3& l, V3& r) {  // rotation.cpp:19-29
    const V3 d = nudge_off_pole(dir);
    const double sxy = std::sqrt(std::max(1e-300, d[0] * d[0] + d[1] * d[1]));
    const double cphi = d[0] / sxy, sphi = d[1] / sxy;
    l = {d[2] * cphi, d[2] * sphi, -sxy};
    r = {-sphi, cphi, 0.0};
}
static void scatter_geometry(const V3& din_raw, const V3& dout_raw, double& ct, double& eta_in, double& eta_out) {
    V3 din = nudge_off_pole(din_raw), dout = nudge_off_pole(dout_raw);  // rotation.cpp:42-68
    double c = std::clamp(dot(din, dout), -1.0, 1.0);
    if (1.0 - std::abs(c) < 1e-12) {
        const V3 probe = std::abs(dout[2]) < 0.9 ? V3{0, 0, 1} : V3{1, 0, 0};
        dout = v3norm({dout[0] + 1e-9 * probe[0], dout[1] + 1e-9 * probe[1], dout[2] + 1e-9 * probe[2]});
        c = std::clamp(dot(din, dout), -1.0, 1.0);
    }
    const V3 lin = v3norm({dout[0] - c * din[0], dout[1] - c * din[1], dout[2] - c * din[2]});
    const V3 lout = v3norm({c * dout[0] - din[0], c * dout[1] - din[1], c * dout[2] - din[2]});
    const V3 rout = cross(dout, lout);
    V3 il, ir, ol, orr;
    meridian_basis(din, il, ir);
    meridian_basis(dout, ol, orr);
    ct = c;
    eta_in = std::atan2(dot(lin, ir), dot(lin, il));
    eta_out = std::atan2(dot(ol, rout), dot(ol, lout));
}
static M4 stokes_rot(double eta) {  // rotation.cpp:31-40
    M4 l;
    l(0, 0) = l(3, 3) = 1.0;
    const double c = std::cos(2.0 * eta), sn = std::sin(2.0 * eta);
    l(1, 1) = c;
    l(1, 2) = sn;
    l(2, 1) = -sn;
    l(2, 2) = c;
    return l;
}
static M4 scatter_matrix(const Layer& layer, double ct) {  // kernel.cpp:147-177
    const int lmax = layer.order_count() - 1;
    const auto d00 = wigner_seq(0, 0, lmax, ct), d02 = wigner_seq(0, 2, lmax, ct), d22 = wigner_seq(2, 2, lmax, ct),
               d2m2 = wigner_seq(2, -2, lmax, ct);
    double a1 = 0, a4 = 0, b1 = 0, b2 = 0, apc = 0, amc = 0;
    for (int l = 0; l <= lmax; ++l) {
        const M4& b = layer.coeffs[l];  // greek_of: beta, alpha, gamma, delta, eps, zeta
        a1 += b(0, 0) * d00[l];
        a4 += b(3, 3) * d00[l];
        b1 += b(0, 1) * d02[l];
        b2 -= b(3, 2) * d02[l];
        apc += (b(1, 1) + b(2, 2)) * d22[l];
        amc += (b(1, 1) - b(2, 2)) * d2m2[l];
    }
    M4 f;
    f(0, 0) = a1;
    f(0, 1) = f(1, 0) = b1;
    f(1, 1) = 0.5 * (apc + amc);
    f(2, 2) = 0.5 * (apc - amc);
    f(2, 3) = b2;
    f(3, 2) = -b2;
    f(3, 3) = a4;
    return f;
}
struct McGrid {
    int zb = 0, ab = 0;
    std::vector<double> sum, sum_sq;  // [2][zb][ab][4]
    std::vector<uint64_t> hits;
};
struct McTracer {  // mc.cpp:119-231
    const Material& spec;
    double mu0, phi0;
    const double* stokes;
    const std::vector<double>& tops;
    double total;
    const std::vector<McPdf>& pdfs;
    const Quad* base_quad;
    McGrid& g;
    int layer_at(double tau) const {  // mc.cpp:100-105
        int p = (int)tops.size() - 1;
        while (p > 0 && tau < tops[p]) --p;
        return p;
    }
    void tally(const V3& dir, const double w[4], bool top) {
        const double mu = std::abs(dir[2]);
        if (mu <= 0.0) return;
        const double phi = reduce_azimuth(std::atan2(dir[1], dir[0]));
        const int iz = std::min((int)(mu * g.zb), g.zb - 1);
        const int ia = std::min((int)(phi / kTwoPi * g.ab), g.ab - 1);
        const size_t idx = ((size_t)(top ? 0 : 1) * g.zb + iz) * g.ab + ia;
        for (int c = 0; c < 4; ++c) {
            g.sum[idx * 4 + c] += w[c];
            g.sum_sq[idx * 4 + c] += w[c] * w[c];
        }
        g.hits[idx] += 1;
    }
    void trace(McRng& rng) {
        double tau = 0.0;
        V3 dir = unit_dir(-mu0, phi0);
        double w[4] = {stokes[0], stokes[1], stokes[2], stokes[3]};
        int events = 0;
        for (int bounce = 0; bounce < 100000; ++bounce) {
            const double step = -std::log(std::max(1e-300, 1.0 - rng.uniform()));
            const double mu = dir[2];
            if (mu == 0.0) return;
            const double dtau = -mu * step;
            if (mu > 0.0 && tau + dtau < 0.0) {
                if (events > 0) tally(dir, w, true);
                return;
            }
            if (mu < 0.0 && tau + dtau > total) {
                if (spec.base.type == 0) {
                    if (events > 0) tally(dir, w, false);
                    return;
                }
                tau = total;
                if (spec.base.type == 1) {
                    const double refl = spec.base.rho * w[0];
                    if (refl <= 0.0) return;
                    w[0] = refl;
                    w[1] = w[2] = w[3] = 0.0;
                } else {
                    const double mu_in = -dir[2];
                    const double mu_up = std::sqrt(std::max(rng.uniform(), 1e-300));
                    const double phi = kTwoPi * rng.uniform();
                    const M4 r = base_row_at(spec.base, *base_quad, mu_up, mu_in);
                    double nw[4];
                    for (int a = 0; a < 4; ++a) {
                        nw[a] = 0.0;
                        for (int b = 0; b < 4; ++b) nw[a] += r(a, b) * w[b];
                        nw[a] *= 0.5;
                    }
                    std::copy(nw, nw + 4, w);
                    if (w[0] <= 0.0) return;
                    dir = unit_dir(std::max(mu_up, 1e-9), reduce_azimuth(phi));
                    ++events;
                    continue;
                }
                const double mu_up = std::sqrt(std::max(rng.uniform(), 1e-300));
                const double phi = kTwoPi * rng.uniform();
                dir = unit_dir(std::max(mu_up, 1e-9), reduce_azimuth(phi));
                ++events;
                continue;
            }
            tau += dtau;
            const int li = layer_at(tau);
            const Layer& layer = spec.layers[li];
            if (layer.omega <= 0.0) return;
            const auto [ct, pdf] = pdfs[li].sample(rng.uniform());
            const double psi = kTwoPi * rng.uniform();
            const V3 nd = rotate_direction(dir, ct, psi);
            double c2, ein, eout;
            scatter_geometry(dir, nd, c2, ein, eout);
            const M4 z = mul(mul(stokes_rot(eout), scatter_matrix(layer, c2)), stokes_rot(ein));
            double nw[4];
            const double f = layer.omega / (2.0 * pdf);
            for (int a = 0; a < 4; ++a) {
                nw[a] = 0.0;
                for (int b = 0; b < 4; ++b) nw[a] += z(a, b) * w[b];
                nw[a] *= f;
            }
            std::copy(nw, nw + 4, w);
            dir = nd;
            ++events;
            if (w[0] <= 0.0) return;
            if (w[0] < 1e-4 * stokes[0]) {  // kRouletteThreshold, kRouletteBoost (mc.cpp:116-117)
                if (rng.uniform() * 10.0 > 1.0) return;
                for (auto& x : w) x *= 10.0;
            }
        }
    }
};
// mc.cpp:256-312
static McGrid mc_trace(const Material& spec, double mu0, double phi0, const double* stokes, uint64_t photons,
                       uint64_t seed, int zb, int ab, int threads) {
    if (photons < 1) throw ValidationError("mc: photon count must be positive");
    if (zb < 1 || ab < 1) throw ValidationError("mc: bin counts must be positive");
    const int P = (int)spec.layers.size();
    std::vector<double> tops(P, 0.0);
    for (int p = 1; p < P; ++p) tops[p] = tops[p - 1] + spec.layers[p - 1].tau;
    const double total = tops.back() + spec.layers.back().tau;
    std::vector<McPdf> pdfs;
    for (const auto& l : spec.layers) pdfs.emplace_back(l);
    Quad bq;
    if (spec.base.type == 2) bq = build_quadrature(spec.base.n);
    auto make = [&] {
        McGrid g;
        g.zb = zb;
        g.ab = ab;
        g.sum.assign((size_t)2 * zb * ab * 4, 0.0);
        g.sum_sq.assign((size_t)2 * zb * ab * 4, 0.0);
        g.hits.assign((size_t)2 * zb * ab, 0);
        return g;
    };
    McGrid tot = make();
    const uint64_t kBlock = 16384, nblk = (photons + kBlock - 1) / kBlock, kChunk = 256;
    for (uint64_t c0 = 0; c0 < nblk; c0 += kChunk) {
        const uint64_t chunk = std::min(kChunk, nblk - c0);
        std::vector<McGrid> gs(chunk, make());
        parallel_for(threads, chunk, [&](size_t b) {
            const uint64_t blk = c0 + b, begin = blk * kBlock, end = std::min(begin + kBlock, photons);
            McTracer tr{spec, mu0, phi0, stokes, tops, total, pdfs, spec.base.type == 2 ? &bq : nullptr, gs[b]};
            for (uint64_t ph = begin; ph < end; ++ph) {
                McRng rng(seed, ph);
                tr.trace(rng);
            }
        });
        for (uint64_t b = 0; b < chunk; ++b)
            for (size_t i = 0; i < tot.sum.size(); ++i) {
                tot.sum[i] += gs[b].sum[i];
                tot.sum_sq[i] += gs[b].sum_sq[i];
                if (i % 4 == 0) tot.hits[i / 4] += gs[b].hits[i / 4];
            }
    }
    return tot;
}

struct OrderState {
    Kernel kernel;
    Reduced ops;
    ModeSet modes;
};

// pipeline.cpp:27-220 restated for the BRDF path.
class Solver {
  public:
    Solver(Material spec, int quad_n, int order_cap, int threads)
        : spec_(std::move(spec)), threads_(threads) {
        quad_ = build_quadrature(quad_n);
        L_ = spec_.order_count();
        if (order_cap > 0) L_ = std::min(L_, order_cap);
        // pipeline.cpp:37-54 medium dedup (omega + coefficients, not tau)
        sig_.resize(spec_.layers.size());
        for (size_t p = 0; p < spec_.layers.size(); ++p) {
            int s = -1;
            for (size_t qq = 0; qq < p; ++qq) {
                const auto& a = spec_.layers[p];
                const auto& b = spec_.layers[qq];
                bool same = a.omega == b.omega && a.coeffs.size() == b.coeffs.size();
                for (size_t l = 0; same && l < a.coeffs.size(); ++l)
                    for (int e = 0; e < 16; ++e)
                        if (a.coeffs[l].v[e] != b.coeffs[l].v[e]) same = false;
                if (same) {
                    s = sig_[qq];
                    break;
                }
            }
            if (s < 0) {
                s = (int)rep_.size();
                rep_.push_back((int)p);
            }
            sig_[p] = s;
        }
        states_.assign(rep_.size(), std::vector<OrderState>(L_));
        for (int m = 0; m < L_; ++m) bmemo_.push_back(std::make_unique<BoundaryLhs>());
    }
    const Quad& quad() const { return quad_; }
    int order_count() const { return L_; }
    oracle_timings t{};

    // pipeline.cpp:57-93
    void prepare_homogeneous() {
        if (ready_) return;
        const double t0 = now_s();
        const size_t items = rep_.size() * (size_t)L_;
        std::vector<std::string> fail(items);
        parallel_for(threads_, items, [&](size_t idx) {
            const int s = (int)(idx / L_), m = (int)(idx % L_);
            try {
                const Layer& layer = spec_.layers[rep_[s]];
                OrderState st;
                st.kernel = assemble_kernel(m, layer, quad_);
                st.ops = build_reduced(m, layer, quad_, st.kernel);
                st.modes = solve_homogeneous(st.ops, st.kernel);
                states_[s][m] = std::move(st);
            } catch (const std::exception& e) {
                fail[idx] = e.what();
            }
        });
        for (const auto& f : fail)
            if (!f.empty()) throw NumericalError(f);
        for (const auto& per : states_)
            for (const auto& st : per) t.max_eigen_residual = std::max(t.max_eigen_residual, st.modes.max_residual);
        t.homogeneous_solves += items;
        t.homogeneous += now_s() - t0;
        ready_ = true;
    }

    // pipeline.cpp:95-199 + nodal_components at tau = 0 (pipeline.cpp:201-209,
    // reconstruction.cpp:11-26, boundary.cpp:20-35).  Returns up[m][k] (d).
    std::vector<std::vector<std::vector<cd>>> solve_incident_top(double mu0, const double* stokes) {
        prepare_homogeneous();
        if (!(mu0 > 0.0 && mu0 <= 1.0)) throw ValidationError("incident mu0 must lie in (0,1]");
        const int P = (int)spec_.layers.size(), S = (int)rep_.size(), d = 4 * quad_.n;
        std::vector<Part> parts((size_t)L_ * 2 * S);
        {
            const double t0 = now_s();
            std::vector<std::string> fail(parts.size());
            parallel_for(threads_, parts.size(), [&](size_t idx) {
                const int m = (int)(idx / (2 * S)), k = (int)((idx / S) % 2) + 1,
                          s = (int)(idx % S);
                try {
                    const Layer& layer = spec_.layers[rep_[s]];
                    const auto& st = states_[s][m];
                    const Source src = build_source(m, k, layer, mu0, stokes, quad_);
                    parts[idx] = solve_particular(st.ops, src, st.modes, st.kernel);
                } catch (const std::exception& e) {
                    fail[idx] = e.what();
                }
            });
            for (const auto& f : fail)
                if (!f.empty()) throw NumericalError(f);
            t.particular_solves += parts.size();
            for (const auto& pp : parts) t.dithered += pp.dithered ? 1 : 0;
            t.particular += now_s() - t0;
        }
        std::vector<std::vector<std::vector<cd>>> up(L_, std::vector<std::vector<cd>>(2));
        {
            const double t0 = now_s();
            std::vector<std::string> fail(L_);
            std::vector<double> conds(L_, 0.0);
            parallel_for(threads_, (size_t)L_, [&](size_t mi) {
                const int m = (int)mi;
                try {
                    std::vector<const ModeSet*> ms(P);
                    std::vector<const Part*> pk[2];
                    pk[0].resize(P);
                    pk[1].resize(P);
                    for (int p = 0; p < P; ++p) {
                        ms[p] = &states_[sig_[p]][m].modes;
                        pk[0][p] = &parts[((size_t)m * 2 + 0) * S + sig_[p]];
                        pk[1][p] = &parts[((size_t)m * 2 + 1) * S + sig_[p]];
                    }
                    const OrderBoundary ob = solve_boundary(spec_, mu0, stokes, quad_, m, ms, pk, boundary_memo(m));
                    conds[m] = ob.condition;
                    // tau = 0 upward stack of layer 0 (t_local = 0, beam_top = 1)
                    const ModeSet& m0 = *ms[0];
                    const double th = spec_.layers[0].tau;
                    for (int k = 0; k < 2; ++k) {
                        std::vector<cd> u(d, 0.0);
                        for (size_t j = 0; j < m0.modes.size(); ++j) {
                            const cd ea = ob.coef[k][0].a[j] * std::exp(-0.0 / m0.modes[j].nu);
                            const cd eb = ob.coef[k][0].b[j] * std::exp(-(th - 0.0) / m0.modes[j].nu);
                            for (int i = 0; i < d; ++i)
                                u[i] += ea * m0.modes[j].psi_plus[i] + eb * m0.modes[j].psi_minus[i];
                        }
                        const double beam = 1.0 * std::exp(-0.0 / mu0);
                        for (int i = 0; i < d; ++i) u[i] += beam * pk[k][0]->zp[i];
                        up[m][k] = std::move(u);
                    }
                } catch (const std::exception& e) {
                    fail[m] = e.what();
                }
            });
            for (const auto& f : fail)
                if (!f.empty()) throw NumericalError(f);
            for (double c : conds) t.max_boundary_condition = std::max(t.max_boundary_condition, c);
            t.boundary_solves += L_;
            t.boundary += now_s() - t0;
        }
        return up;
    }

    // pipeline.cpp:253-309 (radiance_field) on the solve_incident chains
    // (pipeline.cpp:95-199), brdf.cpp:142-160 (field reflectance).
    // values [n_tau][n_mu][n_phi][4]
    void radiance(double mu0, double phi0, const double* stokes, const std::vector<double>& taus,
                  const std::vector<double>& mus, const std::vector<double>& phis, double* values,
                  double* reflectance, bool nodal = false) {
        prepare_homogeneous();
        if (!(mu0 > 0.0 && mu0 <= 1.0)) throw ValidationError("incident mu0 must lie in (0,1]");
        const int P = (int)spec_.layers.size(), S = (int)rep_.size();
        const double t0 = now_s();
        std::vector<Part> parts((size_t)L_ * 2 * S);
        std::vector<std::string> fail(std::max(parts.size(), (size_t)L_));
        parallel_for(threads_, parts.size(), [&](size_t idx) {
            const int m = (int)(idx / (2 * S)), k = (int)((idx / S) % 2) + 1, s = (int)(idx % S);
            try {
                const Layer& layer = spec_.layers[rep_[s]];
                const auto& st = states_[s][m];
                parts[idx] = solve_particular(st.ops, build_source(m, k, layer, mu0, stokes, quad_), st.modes,
                                              st.kernel);
            } catch (const std::exception& e) {
                fail[idx] = e.what();
            }
        });
        for (const auto& f : fail)
            if (!f.empty()) throw NumericalError(f);
        std::vector<double> tau_top(P, 0.0);
        for (int p = 1; p < P; ++p) tau_top[p] = tau_top[p - 1] + spec_.layers[p - 1].tau;
        // chains[m][k][p]
        std::vector<std::array<std::vector<ChainEntry>, 2>> chains(L_);
        parallel_for(threads_, (size_t)L_, [&](size_t mi) {
            const int m = (int)mi;
            try {
                std::vector<const ModeSet*> ms(P);
                std::vector<const Part*> pk[2];
                pk[0].resize(P);
                pk[1].resize(P);
                for (int p = 0; p < P; ++p) {
                    ms[p] = &states_[sig_[p]][m].modes;
                    pk[0][p] = &parts[((size_t)m * 2 + 0) * S + sig_[p]];
                    pk[1][p] = &parts[((size_t)m * 2 + 1) * S + sig_[p]];
                }
                const OrderBoundary ob = solve_boundary(spec_, mu0, stokes, quad_, m, ms, pk, boundary_memo(m));
                for (int k = 0; k < 2; ++k) {
                    auto& ch = chains[m][k];
                    ch.resize(P);
                    for (int p = 0; p < P; ++p) {
                        ch[p].layer = &spec_.layers[p];
                        ch[p].modes = ms[p];
                        ch[p].part = pk[k][p];
                        ch[p].coef_a = ob.coef[k][p].a;
                        ch[p].coef_b = ob.coef[k][p].b;
                        ch[p].tau_top = tau_top[p];
                        ch[p].thickness = spec_.layers[p].tau;
                        ch[p].beam_top = std::exp(-tau_top[p] / mu0);
                    }
                }
            } catch (const std::exception& e) {
                fail[m] = e.what();
            }
        });
        for (const auto& f : fail)
            if (!f.empty()) throw NumericalError(f);
        t.boundary_solves += L_;
        const size_t nt = taus.size(), nm = mus.size(), nph = phis.size();
        if (nodal) {
            // discrete-ordinate stacks at the nodes (reconstruction.cpp:20-26 nodal_stacks):
            // mus = +nodes then -nodes
            const int N = quad_.n;
            for (size_t it = 0; it < nt; ++it) {
                std::vector<std::array<std::vector<cd>, 2>> up(L_), dn(L_);
                for (int m = 0; m < L_; ++m)
                    for (int k = 0; k < 2; ++k) {
                        const auto& ch = chains[m][k];
                        int p = 0;
                        while (p + 1 < P && taus[it] >= ch[p].tau_top + ch[p].thickness) ++p;
                        const double tl = std::clamp(taus[it] - ch[p].tau_top, 0.0, ch[p].thickness);
                        chain_stacks(ch[p], mu0, tl, up[m][k], dn[m][k]);
                    }
                for (int sgn = 0; sgn < 2; ++sgn)
                    for (int i = 0; i < N; ++i) {
                        std::vector<std::array<V4c, 2>> comps(L_);
                        for (int m = 0; m < L_; ++m)
                            for (int k = 0; k < 2; ++k)
                                for (int c = 0; c < 4; ++c)
                                    comps[m][k][c] = (sgn == 0 ? up : dn)[m][k][4 * i + c];
                        for (size_t ip = 0; ip < nph; ++ip)
                            assemble_field(comps, phis[ip] - phi0,
                                           values + ((it * (2 * N) + sgn * N + i) * nph + ip) * 4);
                    }
            }
            return;
        }
        std::vector<std::string> fail2(nm);
        parallel_for(threads_, nm, [&](size_t imu) {
            try {
                const double mu = mus[imu];
                std::vector<std::vector<std::array<V4c, 2>>> per_tau(nt, std::vector<std::array<V4c, 2>>(L_));
                for (int m = 0; m < L_; ++m) {
                    std::vector<KRow> rows(P);
                    std::vector<M4> bb(P);
                    for (int p = 0; p < P; ++p) {  // pipeline.cpp:237-258 direction_kernels
                        const Layer& layer = spec_.layers[p];
                        rows[p] = kernel_row(m, layer, quad_, mu);
                        if (m < layer.order_count()) {
                            const Gsf go = gsf_seq(m, layer.order_count() - 1, mu),
                                      gi = gsf_seq(m, layer.order_count() - 1, -mu0);
                            for (int l = m; l < layer.order_count(); ++l)
                                axpy4(bb[p], 1.0,
                                      mul(mul(gsf_matrix(go, l, false), layer.coeffs[l]), gsf_matrix(gi, l, false)));
                        }
                    }
                    for (int k = 0; k < 2; ++k) {
                        const auto v = reconstruct_component(chains[m][k], quad_, m, k + 1, mu0, stokes, spec_.base, mu,
                                                             taus, rows, bb);
                        for (size_t it = 0; it < nt; ++it) per_tau[it][m][k] = v[it];
                    }
                }
                for (size_t it = 0; it < nt; ++it)
                    for (size_t ip = 0; ip < nph; ++ip)
                        assemble_field(per_tau[it], phis[ip] - phi0, values + ((it * nm + imu) * nph + ip) * 4);
            } catch (const std::exception& e) {
                fail2[imu] = e.what();
            }
        });
        for (const auto& f : fail2)
            if (!f.empty()) throw NumericalError(f);
        t.reconstruction_items += nm * nt;
        if (reflectance) {
            // nodal components at tau = 0 (layer 0, t = 0), 19 azimuths (brdf.hpp:46-48)
            const int n_phi = 19, N = quad_.n;
            std::vector<std::array<std::vector<cd>, 2>> up(L_);
            for (int m = 0; m < L_; ++m)
                for (int k = 0; k < 2; ++k) {
                    std::vector<cd> dn;
                    chain_stacks(chains[m][k][0], mu0, 0.0, up[m][k], dn);
                }
            double flux[4] = {0, 0, 0, 0};
            for (int i = 0; i < N; ++i)
                for (int j = 0; j < n_phi; ++j) {
                    std::vector<std::array<V4c, 2>> comps(L_);
                    for (int m = 0; m < L_; ++m)
                        for (int k = 0; k < 2; ++k)
                            for (int c = 0; c < 4; ++c) comps[m][k][c] = up[m][k][4 * i + c];
                    double sv[4];
                    assemble_field(comps, kTwoPi * j / n_phi, sv);
                    const double w = quad_.weights[i] * quad_.nodes[i] * (kTwoPi / n_phi);
                    for (int c = 0; c < 4; ++c) flux[c] += w * sv[c];
                }
            const double inc = std::max(mu0 * stokes[0], 1e-300);
            for (int c = 0; c < 4; ++c) reflectance[c] = flux[c] / inc;
        }
        t.reconstruction += now_s() - t0;
    }

  private:
    Material spec_;
    int threads_;
    Quad quad_;
    int L_ = 0;
    std::vector<int> sig_, rep_;
    std::vector<std::vector<OrderState>> states_;
    std::vector<std::unique_ptr<BoundaryLhs>> bmemo_;
    bool ready_ = false;
    BoundaryLhs* boundary_memo(int m) { return g_cache_boundary.load() ? bmemo_[m].get() : nullptr; }
};

// reconstruction.cpp:201-227 (FourierBasis::phi, kernel.cpp:111-122).
static void azimuthal_assemble(const std::vector<std::vector<std::vector<cd>>>& up, int node,
                               double dphi, double out[4]) {
    const double x = -dphi;
    cd tot[4] = {0, 0, 0, 0};
    double scale = 0.0;
    for (size_t m = 0; m < up.size(); ++m) {
        const double sc = (m == 0) ? 1.0 : 2.0;
        const double c = std::cos((double)m * x), s = std::sin((double)m * x);
        const double p1[4] = {sc * c, sc * c, sc * s, sc * s};
        const double p2[4] = {-sc * s, -sc * s, sc * c, sc * c};
        for (int r = 0; r < 4; ++r)
            tot[r] += 0.5 * (p1[r] * up[m][0][4 * node + r] + p2[r] * up[m][1][4 * node + r]);
        for (int k = 0; k < 2; ++k)
            for (int r = 0; r < 4; ++r) scale = std::max(scale, std::abs(up[m][k][4 * node + r]));
    }
    double imag = 0;
    for (int r = 0; r < 4; ++r) imag = std::max(imag, std::abs(tot[r].imag()));
    if (imag > 1e-9 * scale + 1e-300) {
        char buf[200];
        std::snprintf(buf, sizeof buf,
                      "imaginary residue %g exceeds tolerance (scale %g); conjugate mode pairing "
                      "is broken",
                      imag, scale);
        throw NumericalError(buf);
    }
    for (int r = 0; r < 4; ++r) out[r] = tot[r].real();
}

// 4x4 inverse by Gauss-Jordan with partial pivoting (Eigen inverse() stand-in).
static void inv4(const double a_in[16], double out[16]) {
    double a[4][8];
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 8; ++c) a[r][c] = c < 4 ? a_in[4 * r + c] : (c - 4 == r ? 1.0 : 0.0);
    for (int c = 0; c < 4; ++c) {
        int p = c;
        for (int r = c + 1; r < 4; ++r)
            if (std::abs(a[r][c]) > std::abs(a[p][c])) p = r;
        for (int k = 0; k < 8; ++k) std::swap(a[c][k], a[p][k]);
        const double dv = a[c][c];
        for (int k = 0; k < 8; ++k) a[c][k] /= dv;
        for (int r = 0; r < 4; ++r)
            if (r != c) {
                const double f = a[r][c];
                for (int k = 0; k < 8; ++k) a[r][k] -= f * a[c][k];
            }
    }
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) out[4 * r + c] = a[r][c + 4];
}

// brdf.cpp:43-125
static void compute_brdf(const Material& mat, int quad_n, int order_cap, int threads,
                         const double* mu_in, size_t n_in, int n_dphi, const double* basis_in,
                         double* out, oracle_timings* tm, double* comps) {
    const double tw = now_s();
    double basis[16] = {1, 0, 0, 0, 1, 1, 0, 0, 1, 0, 1, 0, 1, 0, 0, 1};  // brdf.cpp:7-9
    if (basis_in) std::memcpy(basis, basis_in, sizeof basis);
    const int nb = 4;
    {  // JacobiSVD condition check (brdf.cpp:45-52); basis_mat(4 x nb) col b = basis[b]
        double bm[16];
        for (int b = 0; b < nb; ++b)
            for (int c = 0; c < 4; ++c) bm[b * 4 + c] = basis[4 * b + c];
        double s[4], work[64];
        int info = 0, four = 4, lw = 64, one = 1;
        const char jn = 'N';
        double dummy = 0;
        scipy_dgesvd_(&jn, &jn, &four, &four, bm, &four, s, &dummy, &one, &dummy, &one, work, &lw,
                      &info, 1, 1);
        const double cond = s[0] / std::max(s[3], 1e-300);
        if (cond > 1e3)
            throw ValidationError("brdf: incident Stokes basis is ill-conditioned (condition " +
                                  std::to_string(cond) + ")");
    }
    if (n_dphi < 1) throw ValidationError("brdf: dphi grid must have at least one point");
    for (size_t i = 0; i < n_in; ++i)
        if (!(mu_in[i] > 0.0 && mu_in[i] <= 1.0))
            throw ValidationError("brdf: incident cosines must lie in (0,1]");

    Solver solver(mat, quad_n, order_cap, threads);
    solver.prepare_homogeneous();
    const Quad& q = solver.quad();
    const int N = q.n, L = solver.order_count(), d = 4 * N;
    std::vector<double> dphi(n_dphi);
    for (int j = 0; j < n_dphi; ++j) dphi[j] = kTwoPi * j / n_dphi;

    uint64_t clamped = 0;
    for (size_t ii = 0; ii < n_in; ++ii) {
        const double mu0 = mu_in[ii];
        std::vector<double> exits((size_t)nb * N * n_dphi * 4);
        for (int b = 0; b < nb; ++b) {
            const auto up = solver.solve_incident_top(mu0, basis + 4 * b);
            if (comps) {
                for (int m = 0; m < L; ++m)
                    for (int k = 0; k < 2; ++k)
                        for (int i = 0; i < d; ++i) {
                            const size_t at =
                                ((((ii * nb + b) * (size_t)L + m) * 2 + k) * d + i) * 2;
                            comps[at] = up[m][k][i].real();
                            comps[at + 1] = up[m][k][i].imag();
                        }
            }
            for (int io = 0; io < N; ++io)
                for (int ip = 0; ip < n_dphi; ++ip)
                    azimuthal_assemble(up, io, dphi[ip],
                                       &exits[(((size_t)b * N + io) * n_dphi + ip) * 4]);
        }
        // pinv = I^T (I I^T)^{-1}, I = mu0 * basis_mat (4 x nb)
        double I[16], IIt[16], inv[16], pinv[16];
        for (int c = 0; c < 4; ++c)
            for (int b = 0; b < nb; ++b) I[c * 4 + b] = mu0 * basis[4 * b + c];
        for (int r = 0; r < 4; ++r)
            for (int c = 0; c < 4; ++c) {
                double s = 0;
                for (int b = 0; b < nb; ++b) s += I[r * 4 + b] * I[c * 4 + b];
                IIt[4 * r + c] = s;
            }
        inv4(IIt, inv);
        for (int b = 0; b < nb; ++b)
            for (int c = 0; c < 4; ++c) {
                double s = 0;
                for (int k = 0; k < 4; ++k) s += I[k * 4 + b] * inv[4 * k + c];
                pinv[b * 4 + c] = s;  // (nb x 4) row-major
            }
        for (int io = 0; io < N; ++io)
            for (int ip = 0; ip < n_dphi; ++ip) {
                double fr[16];
                for (int r = 0; r < 4; ++r)
                    for (int c = 0; c < 4; ++c) {
                        double s = 0;
                        for (int b = 0; b < nb; ++b)
                            s += exits[(((size_t)b * N + io) * n_dphi + ip) * 4 + r] * pinv[b * 4 + c];
                        fr[4 * r + c] = s;
                    }
                if (fr[0] < 0.0) {
                    if (fr[0] < -1e-9)
                        throw NumericalError("brdf: negative intensity entry " + std::to_string(fr[0]));
                    fr[0] = 0.0;
                    ++clamped;
                }
                std::memcpy(out + ((ii * N + io) * (size_t)n_dphi + ip) * 16, fr, sizeof fr);
            }
    }
    if (tm) {
        *tm = solver.t;
        tm->clamped_entries = clamped;
        tm->total_wall = now_s() - tw;
    }
}

}  // namespace vo

// ---------------------------------------------------------------- C API
namespace {
thread_local std::string g_err;
template <typename Fn>
int32_t guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const vo::ValidationError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}
struct OneThreadBlas {
    OneThreadBlas() { scipy_openblas_set_num_threads(1); }
};
const OneThreadBlas kBlasInit;
}  // namespace

extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }

uint64_t oracle_polish_count(void) { return vo::g_polish_modes.load(); }

void oracle_set_accurate(int32_t on) { vo::g_accurate.store(on ? 1 : 0); }
void oracle_set_cache_boundary(int32_t on) { vo::g_cache_boundary.store(on ? 1 : 0); }

int32_t oracle_quadrature(int32_t n, double* nodes, double* weights) {
    return guarded([&] {
        const auto q = vo::build_quadrature(n);
        std::copy(q.nodes.begin(), q.nodes.end(), nodes);
        std::copy(q.weights.begin(), q.weights.end(), weights);
    });
}

void oracle_wigner_d_sequence(int32_t m, int32_t n, int32_t lmax, double x, double* out) {
    const auto d = vo::wigner_seq(m, n, lmax, x);
    std::copy(d.begin(), d.end(), out);
}

void oracle_gsf_sequence(int32_t m, int32_t lmax, double x, double* p, double* r, double* t) {
    const auto g = vo::gsf_seq(m, lmax, x);
    std::copy(g.p.begin(), g.p.end(), p);
    std::copy(g.r.begin(), g.r.end(), r);
    std::copy(g.t.begin(), g.t.end(), t);
}

int32_t oracle_kernel_blocks(const oracle_material* cm, int32_t layer, int32_t quad_n, int32_t m,
                             double* pp, double* pm, double* mp, double* mm) {
    return guarded([&] {
        const auto mat = vo::from_c(cm);
        const auto q = vo::build_quadrature(quad_n);
        const auto k = vo::assemble_kernel(m, mat.layers.at(layer), q);
        for (size_t e = 0; e < k.pp.size(); ++e) {
            std::memcpy(pp + 16 * e, k.pp[e].v, 128);
            std::memcpy(pm + 16 * e, k.pm[e].v, 128);
            std::memcpy(mp + 16 * e, k.mp[e].v, 128);
            std::memcpy(mm + 16 * e, k.mm[e].v, 128);
        }
    });
}

int32_t oracle_beam_column(const oracle_material* cm, int32_t layer, int32_t quad_n, int32_t m,
                           double mu_beam, double* up, double* down) {
    return guarded([&] {
        const auto mat = vo::from_c(cm);
        const auto q = vo::build_quadrature(quad_n);
        const auto c = vo::beam_column(m, mat.layers.at(layer), q, mu_beam);
        for (int i = 0; i < q.n; ++i) {
            std::memcpy(up + 16 * i, c.up[i].v, 128);
            std::memcpy(down + 16 * i, c.down[i].v, 128);
        }
    });
}

int32_t oracle_reduced_ops(const oracle_material* cm, int32_t layer, int32_t quad_n, int32_t m,
                           double* e, double* f) {
    return guarded([&] {
        const auto mat = vo::from_c(cm);
        const auto q = vo::build_quadrature(quad_n);
        const auto k = vo::assemble_kernel(m, mat.layers.at(layer), q);
        const auto r = vo::build_reduced(m, mat.layers.at(layer), q, k);
        std::copy(r.e.begin(), r.e.end(), e);
        std::copy(r.f.begin(), r.f.end(), f);
    });
}

int32_t oracle_homogeneous(const oracle_material* cm, int32_t layer, int32_t quad_n, int32_t m,
                           double* nu, double* residual, double* psi_plus, double* psi_minus) {
    return guarded([&] {
        const auto mat = vo::from_c(cm);
        const auto q = vo::build_quadrature(quad_n);
        const auto k = vo::assemble_kernel(m, mat.layers.at(layer), q);
        const auto r = vo::build_reduced(m, mat.layers.at(layer), q, k);
        const auto ms = vo::solve_homogeneous(r, k);
        const int d = 4 * q.n;
        for (int j = 0; j < d; ++j) {
            nu[2 * j] = ms.modes[j].nu.real();
            nu[2 * j + 1] = ms.modes[j].nu.imag();
            residual[j] = ms.modes[j].residual;
            for (int i = 0; i < d; ++i) {
                if (psi_plus) {
                    psi_plus[2 * ((size_t)j * d + i)] = ms.modes[j].psi_plus[i].real();
                    psi_plus[2 * ((size_t)j * d + i) + 1] = ms.modes[j].psi_plus[i].imag();
                }
                if (psi_minus) {
                    psi_minus[2 * ((size_t)j * d + i)] = ms.modes[j].psi_minus[i].real();
                    psi_minus[2 * ((size_t)j * d + i) + 1] = ms.modes[j].psi_minus[i].imag();
                }
            }
        }
    });
}

int32_t oracle_particular(const oracle_material* cm, int32_t layer, int32_t quad_n, int32_t m,
                          int32_t k, double mu0, const double* stokes, double* z_plus,
                          double* z_minus, double* mu0_effective, double* residual) {
    return guarded([&] {
        const auto mat = vo::from_c(cm);
        const auto q = vo::build_quadrature(quad_n);
        const auto& ly = mat.layers.at(layer);
        const auto kern = vo::assemble_kernel(m, ly, q);
        const auto r = vo::build_reduced(m, ly, q, kern);
        const auto ms = vo::solve_homogeneous(r, kern);
        const auto src = vo::build_source(m, k, ly, mu0, stokes, q);
        const auto pt = vo::solve_particular(r, src, ms, kern);
        std::copy(pt.zp.begin(), pt.zp.end(), z_plus);
        std::copy(pt.zm.begin(), pt.zm.end(), z_minus);
        if (mu0_effective) *mu0_effective = pt.mu0_eff;
        if (residual) *residual = pt.residual;
    });
}

int32_t oracle_brdf(const oracle_material* cm, int32_t quad_n, int32_t order_cap, int32_t threads,
                    const double* mu_in, size_t n_in, int32_t n_dphi, const double* basis,
                    double* out, oracle_timings* timings, double* up_components) {
    if (!cm || !mu_in || n_in == 0 || !out) {
        g_err = "null argument";
        return 5;
    }
    return guarded([&] {
        int th = threads;
        if (th <= 0) th = (int)std::max(1u, std::thread::hardware_concurrency());
        const auto mat = vo::from_c(cm);
        vo::compute_brdf(mat, quad_n, order_cap, th, mu_in, n_in, n_dphi > 0 ? n_dphi : 19, basis,
                         out, timings, up_components);
    });
}


// capi.cpp:138-174 (vrte_solve_radiance) restated: grids from pipeline.cpp:358-390.
int32_t oracle_radiance_at(const oracle_material* cm, int32_t quad_n, int32_t order_cap, int32_t threads,
                           double mu0, double phi0, const double* stokes, const double* taus, size_t n_tau,
                           int32_t zenith, int32_t azimuth, const double* mus_in, size_t n_mu_in,
                           const double* phis_in, size_t n_phi_in, int32_t nodal, double* mus_out,
                           double* phis_out, double* values, double* reflectance, oracle_timings* timings);
int32_t oracle_radiance(const oracle_material* cm, int32_t quad_n, int32_t order_cap, int32_t threads, double mu0,
                        double phi0, const double* stokes, const double* taus, size_t n_tau, int32_t zenith,
                        int32_t azimuth, double* mus_out, double* phis_out, double* values, double* reflectance,
                        oracle_timings* timings) {
    return oracle_radiance_at(cm, quad_n, order_cap, threads, mu0, phi0, stokes, taus, n_tau, zenith, azimuth,
                              nullptr, 0, nullptr, 0, 0, mus_out, phis_out, values, reflectance, timings);
}

int32_t oracle_radiance_at(const oracle_material* cm, int32_t quad_n, int32_t order_cap, int32_t threads,
                           double mu0, double phi0, const double* stokes, const double* taus, size_t n_tau,
                           int32_t zenith, int32_t azimuth, const double* mus_in, size_t n_mu_in,
                           const double* phis_in, size_t n_phi_in, int32_t nodal, double* mus_out,
                           double* phis_out, double* values, double* reflectance, oracle_timings* timings) {
    if (!cm || !stokes || !values || (n_tau > 0 && !taus) || zenith < 1 || azimuth < 1) {
        g_err = "null argument";
        return 5;
    }
    return guarded([&] {
        int th = threads;
        if (th <= 0) th = (int)std::max(1u, std::thread::hardware_concurrency());
        const auto mat = vo::from_c(cm);
        vo::Solver solver(mat, quad_n, order_cap, th);
        std::vector<double> tv(taus, taus + n_tau);
        if (tv.empty()) tv.push_back(0.0);
        std::vector<double> up(zenith);
        for (int i = 0; i < zenith; ++i)
            up[i] = zenith == 1 ? 1.0 : std::clamp((double)i / (zenith - 1), 1e-6, 1.0);  // clamp_mu, kMinMu
        std::vector<double> mus;
        for (double m : up) mus.push_back(m);
        for (double m : up) mus.push_back(-m);
        std::vector<double> phis(azimuth);
        const double p0 = vo::reduce_azimuth(phi0);
        for (int j = 0; j < azimuth; ++j)
            phis[j] = azimuth == 1 ? p0 : vo::reduce_azimuth(p0 + vo::kPi * j / (azimuth - 1));
        if (mus_in && n_mu_in) mus.assign(mus_in, mus_in + n_mu_in);
        if (phis_in && n_phi_in) phis.assign(phis_in, phis_in + n_phi_in);
        if (nodal) {  // +nodes then -nodes
            const auto& q = solver.quad();
            mus.clear();
            for (int i = 0; i < q.n; ++i) mus.push_back(q.nodes[i]);
            for (int i = 0; i < q.n; ++i) mus.push_back(-q.nodes[i]);
        }
        solver.radiance(mu0, p0, stokes, tv, mus, phis, values, reflectance, nodal != 0);
        if (mus_out) std::copy(mus.begin(), mus.end(), mus_out);
        if (phis_out) std::copy(phis.begin(), phis.end(), phis_out);
        if (timings) *timings = solver.t;
    });
}


// mc.cpp:256-312 (vrte_mc_trace, capi.cpp:328-346): raw tallies sum/sum_sq [2][zb][ab][4], hits [2][zb][ab]
int32_t oracle_mc_trace(const oracle_material* cm, double mu0, double phi0, const double* stokes, uint64_t photons,
                        uint64_t seed, int32_t zenith_bins, int32_t azimuth_bins, int32_t threads, double* sum,
                        double* sum_sq, uint64_t* hits) {
    if (!cm || !stokes || !sum || !sum_sq || !hits) {
        g_err = "null argument";
        return 5;
    }
    return guarded([&] {
        int th = threads;
        if (th <= 0) th = (int)std::max(1u, std::thread::hardware_concurrency());
        const auto mat = vo::from_c(cm);
        const auto g = vo::mc_trace(mat, mu0, vo::reduce_azimuth(phi0), stokes, photons, seed, zenith_bins,
                                    azimuth_bins, th);
        std::copy(g.sum.begin(), g.sum.end(), sum);
        std::copy(g.sum_sq.begin(), g.sum_sq.end(), sum_sq);
        std::copy(g.hits.begin(), g.hits.end(), hits);
    });
}

}  // extern "C"
