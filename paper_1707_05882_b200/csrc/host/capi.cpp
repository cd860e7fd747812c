// capi.cpp -- the drop-in C ABI (reference src/capi.cpp:1-378).
//
// vrte_compute_brdf keeps the reference's argument checks, validation order,
// error mapping (guarded(): ValidationError -> 2, NumericalError/other -> 3,
// null arguments -> 5) and handle ownership.  Instead of the VrteSolver
// thread pool it hands a flat problem to the sm_100a pipeline (vrte_cuda.h).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <complex>
#include <cstring>
#include <stdexcept>
#include <fstream>
#include <atomic>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "host.hpp"
#include "vrte/vrte.h"
#include "vrte/vrte_cuda.h"
#include "vrte/vrte_ext.h"

using namespace vrte::host;

namespace {

// Every plan drives several CUDA streams (main, side, right-hand sides, factorization
// look-ahead); with plans in flight together (batch API, order shards) the default
// 8 hardware work queues would alias streams onto one queue.  Ask for the maximum
// when the library is loaded -- effective if the process has not created its CUDA
// context yet, never overriding a value the application set.
const bool g_connections = [] {
    setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 0);
    return true;
}();

thread_local std::string g_last_error;

vrte_status set_error(vrte_status code, const std::string& message) {
    g_last_error = message;
    return code;
}

template <typename Fn>
vrte_status guarded(Fn&& fn) {  // capi.cpp:21-32
    try {
        return fn();
    } catch (const ValidationError& e) {
        return set_error(VRTE_E_VALIDATION, e.what());
    } catch (const NumericalError& e) {
        return set_error(VRTE_E_NUMERICAL, e.what());
    } catch (const std::exception& e) {
        return set_error(VRTE_E_NUMERICAL, e.what());
    }
}

double wall_now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Singular values of the 4 x nb basis matrix by one-sided Jacobi
// (Eigen::JacobiSVD stand-in for brdf.cpp:45-52).
void singular_values4(const double basis[16], double sv[4]) {
    double a[4][4];  // columns = basis vectors
    for (int b = 0; b < 4; ++b)
        for (int c = 0; c < 4; ++c) a[b][c] = basis[4 * b + c];
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0.0;
        for (int p = 0; p < 3; ++p)
            for (int q = p + 1; q < 4; ++q) {
                double alpha = 0, beta = 0, gamma = 0;
                for (int k = 0; k < 4; ++k) {
                    alpha += a[p][k] * a[p][k];
                    beta += a[q][k] * a[q][k];
                    gamma += a[p][k] * a[q][k];
                }
                if (gamma == 0.0) continue;
                off = std::max(off, std::abs(gamma) / std::sqrt(alpha * beta));
                const double zeta = (beta - alpha) / (2.0 * gamma);
                const double t = std::copysign(1.0, zeta) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
                for (int k = 0; k < 4; ++k) {
                    const double x = a[p][k], y = a[q][k];
                    a[p][k] = c * x - s * y;
                    a[q][k] = s * x + c * y;
                }
            }
        if (off < 1e-15) break;
    }
    for (int b = 0; b < 4; ++b) {
        double s = 0;
        for (int k = 0; k < 4; ++k) s += a[b][k] * a[b][k];
        sv[b] = std::sqrt(s);
    }
    std::sort(sv, sv + 4, [](double x, double y) { return x > y; });
}

void inv4(const double in[16], double out[16]) {
    double a[4][8];
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 8; ++c) a[r][c] = c < 4 ? in[4 * r + c] : (c - 4 == r ? 1.0 : 0.0);
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

// VRTE_DEVICE: CUDA ordinal of single-device calls (-1 = the caller's current device).
int env_device() {
    const char* dev = std::getenv("VRTE_DEVICE");
    return dev ? std::atoi(dev) : -1;
}

// VRTE_DEVICES: comma-separated ordinals, or "all" visible devices.
std::vector<int> env_devices() {
    std::vector<int> out;
    const char* e = std::getenv("VRTE_DEVICES");
    if (!e || !*e) return out;
    if (std::string(e) == "all") {
        for (int k = 0; k < vrte_cuda_device_count(); ++k) out.push_back(k);
        return out;
    }
    std::string cur;
    for (const char* c = e;; ++c) {
        if (*c == ',' || *c == 0) {
            if (!cur.empty()) {
                char* end = nullptr;
                const long v = std::strtol(cur.c_str(), &end, 10);
                if (!end || *end || v < 0) throw ValidationError("VRTE_DEVICES: bad device ordinal '" + cur + "'");
                out.push_back((int)v);
            }
            cur.clear();
            if (*c == 0) break;
        } else if (*c != ' ') {
            cur += *c;
        }
    }
    return out;
}

// Host-side set-up of one BRDF request (brdf.cpp:43-77, pipeline.cpp:27-55):
// validated inputs flattened into the device problem description.
struct BrdfSetup {
    MaterialSpec spec;
    Quadrature quad;
    int L = 0;
    std::vector<int> medium, rep, devices;
    std::vector<int> sig_to_medium;  // reference signature k (first appearance) -> device medium index
    std::vector<double> omega, greek, tau, mu_in, beam_rows, post, trig, table_flat, dphi;
    std::vector<double> mu_in_user, refl_top, pre;  // Fresnel interface (mu_in = refracted cosines)
    Quadrature quad_out;  // output nodes / weights of the table (= quad without an interface)
    double basis[16];
    vrte_cuda_problem prob{};
};

void build_setup(BrdfSetup& s, const MaterialSpec& mat, const vrte_options* options,
                 const double* mu_in, size_t n_in, int32_t n_dphi_arg, const double* basis_in) {
    const double defb[16] = {1, 0, 0, 0, 1, 1, 0, 0, 1, 0, 1, 0, 1, 0, 0, 1};  // brdf.cpp:7-9
    std::memcpy(s.basis, basis_in ? basis_in : defb, sizeof s.basis);
    const int n_dphi = n_dphi_arg > 0 ? n_dphi_arg : 19;
    // VrteSolver ctor (pipeline.cpp:27-36)
    s.spec = mat;
    validate_material(s.spec);
    const int qn = options ? options->quadrature_n : 40;
    if (qn < 1) throw ValidationError("solver: quadrature size must be at least 1");
    // compute_brdf validation order (brdf.cpp:45-62)
    {
        double sv[4];
        singular_values4(s.basis, sv);
        const double cond = sv[0] / std::max(sv[3], 1e-300);
        if (cond > 1e3)
            throw ValidationError("brdf: incident Stokes basis is ill-conditioned (condition " +
                                  std::to_string(cond) + ")");
    }
    if (n_dphi < 1) throw ValidationError("brdf: dphi grid must have at least one point");
    for (size_t i = 0; i < n_in; ++i)
        if (!(mu_in[i] > 0.0 && mu_in[i] <= 1.0))
            throw ValidationError("brdf: incident cosines must lie in (0,1]");
    const double nif = s.spec.interface_n;
    const bool fresnel = nif > 1.0;
    int n_hi = qn;
    if (fresnel) {
        // the refraction cone mu > mu_c and the total-internal-reflection range each
        // get a Gauss rule; the cone's nodes are the table's output directions
        n_hi = (qn + 1) / 2;
        s.quad = build_split_gauss_quadrature(qn, std::sqrt(1.0 - 1.0 / (nif * nif)), n_hi);
    } else {
        s.quad = build_double_gauss_quadrature(qn);
    }
    s.L = s.spec.order_count();
    if (options && options->order_cap > 0) s.L = std::min(s.L, options->order_cap);
    const int N = s.quad.n, L = s.L, P = (int)s.spec.layers.size();
    const int Lc = s.spec.order_count();  // the l-sum always spans every coefficient
    // medium dedup: identical omega + coefficients share one solve (pipeline.cpp:37-54)
    s.medium.assign(P, -1);
    s.rep.clear();
    for (int p = 0; p < P; ++p) {
        int sig = -1;
        for (int q = 0; q < p && sig < 0; ++q) {
            const auto& a = s.spec.layers[p];
            const auto& b = s.spec.layers[q];
            if (a.omega == b.omega && a.coeffs == b.coeffs) sig = s.medium[q];
        }
        if (sig < 0) {
            sig = (int)s.rep.size();
            s.rep.push_back(p);
        }
        s.medium[p] = sig;
    }
    const int S = (int)s.rep.size();
    {
        // media ordered by decreasing expansion length: the orders m >= a medium's last
        // nonzero coefficient are free-streaming (zero kernel, analytic modes) and the
        // device skips them when they are the trailing slots of the LAST medium
        // (brdf_device.cu setup_plan), whatever the layer order
        auto lc_of = [&](int k) {
            const auto& layer = s.spec.layers[s.rep[k]];
            if (layer.omega == 0.0) return 0;
            int lc = 0;
            for (int l = 0; l < (int)layer.coeffs.size(); ++l)
                for (int r = 0; r < 4; ++r)
                    for (int c = 0; c < 4; ++c)
                        if (at(layer.coeffs[l], r, c) != 0.0) lc = l + 1;
            return lc;
        };
        std::vector<int> order(S), lcs(S), rank(S);
        for (int k = 0; k < S; ++k) {
            order[k] = k;
            lcs[k] = lc_of(k);
        }
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return lcs[a] > lcs[b]; });
        std::vector<int> rep2(S);
        for (int k = 0; k < S; ++k) {
            rank[order[k]] = k;
            rep2[k] = s.rep[order[k]];
        }
        s.rep = rep2;
        for (int p = 0; p < P; ++p) s.medium[p] = rank[s.medium[p]];
        s.sig_to_medium = rank;
    }
    s.omega.resize(S);
    s.greek.assign((size_t)S * Lc * 6, 0.0);
    for (int k = 0; k < S; ++k) {
        const auto& layer = s.spec.layers[s.rep[k]];
        s.omega[k] = layer.omega;
        for (int l = 0; l < Lc; ++l) {
            const Mat4& b = layer.coeffs[l];  // greek_of, kernel.cpp:15-17
            double* g = &s.greek[((size_t)k * Lc + l) * 6];
            g[0] = at(b, 0, 0);
            g[1] = at(b, 1, 1);
            g[2] = at(b, 0, 1);
            g[3] = at(b, 3, 3);
            g[4] = at(b, 3, 2);
            g[5] = at(b, 2, 2);
        }
    }
    s.tau.resize(P);
    for (int p = 0; p < P; ++p) s.tau[p] = s.spec.layers[p].tau;
    s.mu_in_user.assign(mu_in, mu_in + n_in);
    s.mu_in.assign(mu_in, mu_in + n_in);
    if (fresnel)
        for (auto& m : s.mu_in) m = refract_in(nif, m);  // the beam inside the medium
    // base rows at the beam (boundary.cpp:125-139): Lambertian uses node 0's row
    s.beam_rows.assign(n_in * (size_t)N * 16, 0.0);
    const bool lam = std::holds_alternative<LambertianBase>(s.spec.base);
    for (size_t ii = 0; ii < n_in; ++ii)
        for (int i = 0; i < N; ++i) {
            const Mat4 r = base_row_at(s.spec.base, s.quad, s.quad.nodes[lam ? 0 : i], mu_in[ii]);
            std::memcpy(&s.beam_rows[(ii * N + i) * 16], r.data(), 128);
        }
    if (const auto* tab = std::get_if<MuellerTableBase>(&s.spec.base)) {
        if (tab->n < N)
            throw ValidationError("base: mueller table has fewer nodes than the quadrature");
        s.table_flat.resize((size_t)tab->n * tab->n * 16);
        for (size_t e = 0; e < tab->table.size(); ++e)
            std::memcpy(&s.table_flat[e * 16], tab->table[e].data(), 128);
    }
    // Mueller recovery operator per incident: B (mu0 B)^+ (brdf.cpp:100-105)
    s.post.resize(n_in * 16);
    for (size_t ii = 0; ii < n_in; ++ii) {
        const double mu0 = mu_in[ii];
        double I[16], IIt[16], inv[16], pinv[16];
        for (int c = 0; c < 4; ++c)
            for (int b = 0; b < 4; ++b) I[c * 4 + b] = mu0 * s.basis[4 * b + c];
        for (int r = 0; r < 4; ++r)
            for (int c = 0; c < 4; ++c) {
                double acc = 0;
                for (int b = 0; b < 4; ++b) acc += I[r * 4 + b] * I[c * 4 + b];
                IIt[4 * r + c] = acc;
            }
        inv4(IIt, inv);
        for (int b = 0; b < 4; ++b)
            for (int c = 0; c < 4; ++c) {
                double acc = 0;
                for (int k = 0; k < 4; ++k) acc += I[k * 4 + b] * inv[4 * k + c];
                pinv[b * 4 + c] = acc;
            }
        for (int c = 0; c < 4; ++c)  // post[c][col] = sum_b basis_b[c] pinv[b][col]
            for (int col = 0; col < 4; ++col) {
                double acc = 0;
                for (int b = 0; b < 4; ++b) acc += s.basis[4 * b + c] * pinv[b * 4 + col];
                s.post[ii * 16 + 4 * c + col] = acc;
            }
    }
    s.quad_out = s.quad;
    s.refl_top.clear();
    s.pre.clear();
    if (fresnel) {
        // beam: inside Stokes = (mu0 / mu0') T_in(mu0) I0 (power through the surface);
        // post' = that factor times B (mu0 B)^+; exits: T_out(mu) / n^2 (radiance theorem)
        for (size_t ii = 0; ii < n_in; ++ii) {
            const Mat4 T = fresnel_transmit_in(nif, mu_in[ii]);
            const double f = mu_in[ii] / s.mu_in[ii];
            double np[16];
            for (int c = 0; c < 4; ++c)
                for (int col = 0; col < 4; ++col) {
                    double acc = 0.0;
                    for (int k = 0; k < 4; ++k) acc += f * at(T, c, k) * s.post[ii * 16 + 4 * k + col];
                    np[4 * c + col] = acc;
                }
            std::memcpy(&s.post[ii * 16], np, sizeof np);
        }
        s.refl_top.resize((size_t)N * 16);
        s.pre.assign((size_t)N * 16, 0.0);
        for (int i = 0; i < N; ++i) {
            const Mat4 Rm = fresnel_reflect_inside(nif, s.quad.nodes[i]);
            std::memcpy(&s.refl_top[(size_t)i * 16], Rm.data(), 128);
            if (i >= N - n_hi) {
                const Mat4 To = fresnel_transmit_out(nif, s.quad.nodes[i]);
                for (int e = 0; e < 16; ++e) s.pre[(size_t)i * 16 + e] = To[e] / (nif * nif);
            }
        }
        // output directions outside and their weights: mu' dmu' = n^2 mu dmu
        s.quad_out.n = n_hi;
        s.quad_out.nodes.clear();
        s.quad_out.weights.clear();
        for (int i = N - n_hi; i < N; ++i) {
            const double mo = refract_out(nif, s.quad.nodes[i]);
            s.quad_out.nodes.push_back(mo);
            s.quad_out.weights.push_back(nif * nif * s.quad.weights[i] * s.quad.nodes[i] / mo);
        }
    }
    s.dphi.resize(n_dphi);
    for (int j = 0; j < n_dphi; ++j) s.dphi[j] = kTwoPi * j / n_dphi;
    s.trig.resize((size_t)L * n_dphi * 2);
    for (int m = 0; m < L; ++m)
        for (int j = 0; j < n_dphi; ++j) {
            const double x = -s.dphi[j];
            s.trig[2 * ((size_t)m * n_dphi + j)] = std::cos(m * x);
            s.trig[2 * ((size_t)m * n_dphi + j) + 1] = std::sin(m * x);
        }
    vrte_cuda_problem& p = s.prob;
    p.N = N;
    p.L = L;
    p.L_coeffs = Lc;
    p.n_layers = P;
    p.n_media = S;
    p.n_in = (int32_t)n_in;
    p.n_dphi = n_dphi;
    p.nodes = s.quad.nodes.data();
    p.weights = s.quad.weights.data();
    p.omega = s.omega.data();
    p.greek = s.greek.data();
    p.tau = s.tau.data();
    p.medium = s.medium.data();
    p.mu_in = s.mu_in.data();
    p.base_type = lam ? 1 : (std::holds_alternative<MuellerTableBase>(s.spec.base) ? 2 : 0);
    p.rho = lam ? std::get<LambertianBase>(s.spec.base).rho : 0.0;
    p.table_n = p.base_type == 2 ? std::get<MuellerTableBase>(s.spec.base).n : 0;
    p.table = s.table_flat.empty() ? nullptr : s.table_flat.data();
    p.beam_rows = s.beam_rows.data();
    p.post = s.post.data();
    p.trig = s.trig.data();
    p.m_begin = 0;
    p.m_stride = 1;
    p.n_orders = 0;
    p.refl_top = fresnel ? s.refl_top.data() : nullptr;
    p.pre = fresnel ? s.pre.data() : nullptr;
    p.out_lo = fresnel ? N - n_hi : 0;
    p.device = env_device();
    // VRTE_DEVICES="0,1,..." (or "all"): shard the orders of one solve over these
    // devices (vrte_options is caller-allocated ABI and keeps its layout)
    s.devices = env_devices();
    if (s.devices.size() > 1) {
        p.devices = s.devices.data();
        p.n_devices = (int32_t)s.devices.size();
    }
}

}  // namespace

struct vrte_material {
    MaterialSpec spec;
};

struct vrte_mc_tally {  // capi.cpp:83-86 (mc.hpp TallyGrid)
    std::vector<double> sum, sum_sq;  // [2][zb][ab][4]
    std::vector<uint64_t> hits;       // [2][zb][ab]
    int zb = 0, ab = 0;
    uint64_t photons = 0;
    double mu0 = 1.0, tau_bottom = 0.0;
};

struct vrte_field {  // capi.cpp:69-74
    RadianceField field;
    vrte_timings timings{};
    double reflectance[4] = {0, 0, 0, 0};
};

struct vrte_brdf {
    BrdfTable table;
    Quadrature quadrature;
    vrte_timings timings{};
    vrte_brdf_device_stats stats{};
};

extern "C" {

const char* vrte_last_error(void) { return g_last_error.c_str(); }

const char* vrte_version(void) { return "1.0.0"; }

vrte_status vrte_material_load(const char* path, vrte_material** out) {
    if (!path || !out) return set_error(VRTE_E_ARGUMENT, "null argument");
    return guarded([&] {
        auto h = std::make_unique<vrte_material>();
        h->spec = load_material_file(path);
        *out = h.release();
        return VRTE_OK;
    });
}

vrte_status vrte_material_parse(const char* json_text, const char* base_dir, vrte_material** out) {
    if (!json_text || !out) return set_error(VRTE_E_ARGUMENT, "null argument");
    return guarded([&] {
        auto h = std::make_unique<vrte_material>();
        h->spec = parse_material_json(json_text, base_dir ? base_dir : "");
        *out = h.release();
        return VRTE_OK;
    });
}

void vrte_material_free(vrte_material* material) { delete material; }

vrte_status vrte_material_info(const vrte_material* material, int32_t* order_count,
                               int32_t* layer_count) {
    if (!material) return set_error(VRTE_E_ARGUMENT, "null material");
    if (order_count) *order_count = material->spec.order_count();
    if (layer_count) *layer_count = (int32_t)material->spec.layers.size();
    return VRTE_OK;
}

void vrte_options_init(vrte_options* options) {
    if (!options) return;
    std::memset(options, 0, sizeof *options);
    options->quadrature_n = 40;
    options->out_zenith = 11;
    options->out_azimuth = 19;
}

// ---------------------------------------------------------------- radiance
// capi.cpp:138-232: solve one beam (the material's source, or the options'
// override), reconstruct the field on the signed zenith x azimuth grid at the
// requested depths on the device (radiance.cu), field reflectance brdf.cpp:142-160.
vrte_status vrte_solve_radiance(const vrte_material* material, const vrte_options* options,
                                const double* tau_levels, size_t n_tau, vrte_field** out) {
    if (!material || !out || (n_tau > 0 && !tau_levels)) return set_error(VRTE_E_ARGUMENT, "null argument");
    return guarded([&] {
        const double t0 = wall_now();
        auto h = std::make_unique<vrte_field>();
        BeamSource beam = material->spec.source;
        if (options && options->incident_override) {
            beam.mu0 = options->incident_mu0;
            beam.phi0 = options->incident_phi0;
        }
        // the reference's order: VrteSolver ctor (material, quadrature size), then the
        // incident check of solve_incident (pipeline.cpp:27-36, 97-98)
        {
            MaterialSpec check = material->spec;
            validate_material(check);
            if (options && options->quadrature_n < 1)
                throw ValidationError("solver: quadrature size must be at least 1");
            if (check.interface_n != 1.0)
                throw ValidationError("radiance: the Fresnel interface extension is BRDF-only");
        }
        if (!(beam.mu0 > 0.0 && beam.mu0 <= 1.0))
            throw ValidationError("incident mu0 must lie in (0,1]");
        BrdfSetup s;
        const double mu0 = beam.mu0;
        build_setup(s, material->spec, options, &mu0, 1, 1, nullptr);
        // grids (pipeline.cpp:358-390): a negative count is std::vector's length_error
        // (status 3); an empty grid gives an empty field (the solve and the
        // reflectance still run, here on a one-point grid that is then dropped)
        const int zen_req = options ? options->out_zenith : 11, azi_req = options ? options->out_azimuth : 19;
        if (zen_req < 0 || azi_req < 0) throw std::length_error("cannot create std::vector larger than max_size()");
        const bool empty_grid = zen_req == 0 || azi_req == 0;
        const int zen = zen_req == 0 ? 1 : zen_req, azi = azi_req == 0 ? 1 : azi_req;
        std::vector<double> up(zen);
        for (int i = 0; i < zen; ++i) {
            const double m = zen == 1 ? 1.0 : (double)i / (zen - 1);
            up[i] = std::fabs(m) >= 1e-6 ? m : (m < 0.0 ? -1e-6 : 1e-6);  // clamp_mu, kMinMu
        }
        RadianceField& f = h->field;
        f.taus.assign(tau_levels, tau_levels + n_tau);
        if (f.taus.empty()) f.taus.push_back(0.0);
        for (double m : up) f.mus.push_back(m);
        for (double m : up) f.mus.push_back(-m);
        const double p0 = reduce_azimuth(beam.phi0);
        f.phis.resize(azi);
        for (int j = 0; j < azi; ++j) f.phis[j] = azi == 1 ? p0 : reduce_azimuth(p0 + kPi * j / (azi - 1));
        const int N = s.quad.n, nmu = (int)f.mus.size();
        std::vector<double> base_out((size_t)nmu * N * 16), base_beam((size_t)nmu * 16);
        for (int o = 0; o < nmu; ++o) {
            const double mu = std::fabs(f.mus[o]);
            for (int j = 0; j < N; ++j) {
                const Mat4 r = base_row_at(s.spec.base, s.quad, mu, s.quad.nodes[j]);
                std::memcpy(&base_out[((size_t)o * N + j) * 16], r.data(), 128);
            }
            const Mat4 rb = base_row_at(s.spec.base, s.quad, mu, mu0);
            std::memcpy(&base_beam[(size_t)o * 16], rb.data(), 128);
        }
        vrte_cuda_radiance rad{};
        rad.n_tau = (int32_t)f.taus.size();
        rad.n_mu = nmu;
        rad.n_phi = azi;
        rad.taus = f.taus.data();
        rad.mus = f.mus.data();
        rad.phis = f.phis.data();
        rad.phi0 = p0;
        for (int c = 0; c < 4; ++c) rad.stokes[c] = beam.stokes[c];
        rad.base_out = base_out.data();
        rad.base_beam = base_beam.data();
        f.values.assign((size_t)rad.n_tau * nmu * azi * 4, 0.0);
        vrte_cuda_result r{};
        const int32_t rc = vrte_cuda_radiance_field(&s.prob, &rad, f.values.data(), h->reflectance, &r);
        if (rc == 5) throw std::invalid_argument(r.message);
        if (rc != 0) throw NumericalError(r.message);
        if (empty_grid) {
            if (zen_req == 0) f.mus.clear();
            if (azi_req == 0) f.phis.clear();
            f.values.clear();
        }
        const uint64_t S = s.rep.size(), L = s.L;
        h->timings.homogeneous = r.t_homogeneous;
        h->timings.particular = r.t_particular;
        h->timings.boundary = r.t_boundary;
        h->timings.homogeneous_solves = S * L;
        h->timings.particular_solves = 2 * L * S;
        h->timings.boundary_solves = L;
        h->timings.reconstruction_items = (uint64_t)f.mus.size() * f.taus.size();
        h->timings.total_wall = wall_now() - t0;
        h->timings.reconstruction = h->timings.total_wall - r.t_device;
        *out = h.release();
        return VRTE_OK;
    });
}
vrte_status vrte_field_size(const vrte_field* field, size_t* n_tau, size_t* n_mu, size_t* n_phi) {
    if (!field) return set_error(VRTE_E_ARGUMENT, "null field");
    if (n_tau) *n_tau = field->field.taus.size();
    if (n_mu) *n_mu = field->field.mus.size();
    if (n_phi) *n_phi = field->field.phis.size();
    return VRTE_OK;
}
vrte_status vrte_field_row(const vrte_field* field, size_t tau_index, size_t mu_index, size_t phi_index,
                           double row[7]) {
    if (!field || !row) return set_error(VRTE_E_ARGUMENT, "null argument");
    const RadianceField& f = field->field;
    if (tau_index >= f.taus.size() || mu_index >= f.mus.size() || phi_index >= f.phis.size())
        return set_error(VRTE_E_ARGUMENT, "field index out of range");
    const double* s = &f.values[((tau_index * f.mus.size() + mu_index) * f.phis.size() + phi_index) * 4];
    row[0] = f.taus[tau_index];
    row[1] = f.mus[mu_index];
    row[2] = f.phis[phi_index];
    for (int c = 0; c < 4; ++c) row[3 + c] = s[c];
    return VRTE_OK;
}
vrte_status vrte_field_write_csv(const vrte_field* field, const char* path) {
    if (!field || !path) return set_error(VRTE_E_ARGUMENT, "null argument");
    return guarded([&] {
        write_radiance_csv(path, field->field);
        return VRTE_OK;
    });
}
vrte_status vrte_field_timings(const vrte_field* field, vrte_timings* out) {
    if (!field || !out) return set_error(VRTE_E_ARGUMENT, "null argument");
    *out = field->timings;
    return VRTE_OK;
}
vrte_status vrte_field_reflectance(const vrte_field* field, double out[4]) {
    if (!field || !out) return set_error(VRTE_E_ARGUMENT, "null argument");
    for (int c = 0; c < 4; ++c) out[c] = field->reflectance[c];
    return VRTE_OK;
}
void vrte_field_free(vrte_field* field) { delete field; }

// ---------------------------------------------------------------- Monte Carlo
// capi.cpp:328-378 / mc.cpp: the tracer runs on the GPU (mc.cu), photon per thread.
vrte_status vrte_mc_trace(const vrte_material* material, const vrte_options* options, uint64_t photons,
                          uint64_t seed, int32_t zenith_bins, int32_t azimuth_bins, vrte_mc_tally** out) {
    if (!material || !out) return set_error(VRTE_E_ARGUMENT, "null argument");
    return guarded([&] {
        auto h = std::make_unique<vrte_mc_tally>();
        MaterialSpec spec = material->spec;
        if (options && options->incident_override) {
            spec.source.mu0 = options->incident_mu0;
            spec.source.phi0 = options->incident_phi0;
        }
        if (photons < 1) throw ValidationError("mc: photon count must be positive");
        if (zenith_bins < 1 || azimuth_bins < 1) throw ValidationError("mc: bin counts must be positive");
        const int P = (int)spec.layers.size(), Lc = spec.order_count();
        std::vector<double> greek((size_t)P * Lc * 6, 0.0), omega(P), tops(P, 0.0);
        for (int p = 0; p < P; ++p) {
            const auto& layer = spec.layers[p];
            omega[p] = layer.omega;
            if (p > 0) tops[p] = tops[p - 1] + spec.layers[p - 1].tau;
            for (int l = 0; l < layer.order_count() && l < Lc; ++l) {
                const Mat4& bm = layer.coeffs[l];  // greek_of, kernel.cpp:14-16
                double* g = &greek[((size_t)p * Lc + l) * 6];
                g[0] = at(bm, 0, 0);
                g[1] = at(bm, 1, 1);
                g[2] = at(bm, 0, 1);
                g[3] = at(bm, 3, 3);
                g[4] = at(bm, 3, 2);
                g[5] = at(bm, 2, 2);
            }
        }
        if (spec.interface_n != 1.0)
            throw ValidationError("mc: the Fresnel interface extension is BRDF-only");
        vrte_cuda_mc mc{};
        mc.n_layers = P;
        mc.Lc = Lc;
        mc.zb = zenith_bins;
        mc.ab = azimuth_bins;
        mc.photons = photons;
        mc.seed = seed;
        mc.mu0 = spec.source.mu0;
        mc.phi0 = reduce_azimuth(spec.source.phi0);
        for (int c = 0; c < 4; ++c) mc.stokes[c] = spec.source.stokes[c];
        mc.total = tops[P - 1] + spec.layers[P - 1].tau;
        mc.greek = greek.data();
        mc.omega = omega.data();
        mc.tops = tops.data();
        std::vector<double> table_flat, table_nodes;
        if (const auto* lam = std::get_if<LambertianBase>(&spec.base)) {
            mc.base_type = 1;
            mc.rho = lam->rho;
        } else if (const auto* tab = std::get_if<MuellerTableBase>(&spec.base)) {
            mc.base_type = 2;
            mc.table_n = tab->n;
            table_flat.resize((size_t)tab->n * tab->n * 16);
            for (size_t e = 0; e < tab->table.size(); ++e) std::memcpy(&table_flat[e * 16], tab->table[e].data(), 128);
            table_nodes = build_double_gauss_quadrature(tab->n).nodes;  // mc.cpp:274-276
            mc.table = table_flat.data();
            mc.table_nodes = table_nodes.data();
        }
        mc.device = env_device();
        const size_t bins = 2 * (size_t)zenith_bins * azimuth_bins;
        h->sum.assign(bins * 4, 0.0);
        h->sum_sq.assign(bins * 4, 0.0);
        h->hits.assign(bins, 0);
        vrte_cuda_result r{};
        const int32_t rc = vrte_cuda_mc_trace(&mc, h->sum.data(), h->sum_sq.data(), h->hits.data(), &r);
        if (rc == 2) throw ValidationError(r.message);
        if (rc == 5) throw std::invalid_argument(r.message);
        if (rc != 0) throw NumericalError(r.message);
        h->zb = zenith_bins;
        h->ab = azimuth_bins;
        h->photons = photons;
        h->mu0 = spec.source.mu0;
        h->tau_bottom = mc.total;
        *out = h.release();
        return VRTE_OK;
    });
}

namespace {
// mc.cpp:235-253: flux-weighted bin average and its standard error
double mc_bin_flux_measure(const vrte_mc_tally& t, int iz) {
    const double lo = (double)iz / t.zb, hi = (double)(iz + 1) / t.zb;
    return 0.5 * (hi * hi - lo * lo) * (kTwoPi / t.ab);
}
void mc_radiance(const vrte_mc_tally& t, int hemi, int iz, int ia, double s[4], double se[4]) {
    const size_t idx = ((size_t)hemi * t.zb + iz) * t.ab + ia;
    const double n = (double)t.photons, meas = mc_bin_flux_measure(t, iz);
    for (int c = 0; c < 4; ++c) {
        s[c] = t.sum[idx * 4 + c] * (t.mu0 / (n * meas));
        const double mean = t.sum[idx * 4 + c] / n;
        const double var = std::max(0.0, t.sum_sq[idx * 4 + c] / n - mean * mean);
        se[c] = (t.mu0 / meas) * std::sqrt(var / std::max(1.0, n - 1.0));
    }
}
}  // namespace

vrte_status vrte_mc_tally_row(const vrte_mc_tally* tally, int32_t hemisphere, int32_t zenith_bin,
                              int32_t azimuth_bin, double row[10]) {
    if (!tally || !row) return set_error(VRTE_E_ARGUMENT, "null argument");
    const auto& t = *tally;
    if (hemisphere < 0 || hemisphere > 1 || zenith_bin < 0 || zenith_bin >= t.zb || azimuth_bin < 0 ||
        azimuth_bin >= t.ab)
        return set_error(VRTE_E_ARGUMENT, "tally index out of range");
    double s[4], se[4];
    mc_radiance(t, hemisphere, zenith_bin, azimuth_bin, s, se);
    row[0] = (zenith_bin + 0.5) / t.zb;
    row[1] = kTwoPi * (azimuth_bin + 0.5) / t.ab;
    for (int c = 0; c < 4; ++c) {
        row[2 + c] = s[c];
        row[6 + c] = se[c];
    }
    return VRTE_OK;
}
vrte_status vrte_mc_tally_write_csv(const vrte_mc_tally* tally, const char* path) {
    if (!tally || !path) return set_error(VRTE_E_ARGUMENT, "null argument");
    return guarded([&] {  // csv.cpp:90-109
        std::ofstream out(path);
        if (!out) throw ValidationError("cannot open output file: " + std::string(path));
        auto f17 = [](double v) {
            char buf[40];
            std::snprintf(buf, sizeof buf, "%.17g", v);
            return std::string(buf);
        };
        out << "tau,mu,phi,I,Q,U,V,se_i,se_q,se_u,se_v\n";
        const auto& t = *tally;
        for (int hemi = 0; hemi < 2; ++hemi) {
            const double tau = hemi == 0 ? 0.0 : t.tau_bottom, sign = hemi == 0 ? 1.0 : -1.0;
            for (int iz = 0; iz < t.zb; ++iz)
                for (int ia = 0; ia < t.ab; ++ia) {
                    double s[4], se[4];
                    mc_radiance(t, hemi, iz, ia, s, se);
                    out << f17(tau) << ',' << f17(sign * (iz + 0.5) / t.zb) << ',' << f17(kTwoPi * (ia + 0.5) / t.ab);
                    for (int c = 0; c < 4; ++c) out << ',' << f17(s[c]);
                    for (int c = 0; c < 4; ++c) out << ',' << f17(se[c]);
                    out << '\n';
                }
        }
        return VRTE_OK;
    });
}
void vrte_mc_tally_free(vrte_mc_tally* tally) { delete tally; }

vrte_status vrte_mc_tally_hits(const vrte_mc_tally* tally, int32_t hemisphere, int32_t zenith_bin,
                               int32_t azimuth_bin, uint64_t* hits) {
    if (!tally || !hits) return set_error(VRTE_E_ARGUMENT, "null argument");
    const auto& t = *tally;
    if (hemisphere < 0 || hemisphere > 1 || zenith_bin < 0 || zenith_bin >= t.zb || azimuth_bin < 0 ||
        azimuth_bin >= t.ab)
        return set_error(VRTE_E_ARGUMENT, "tally index out of range");
    *hits = t.hits[((size_t)hemisphere * t.zb + zenith_bin) * t.ab + azimuth_bin];
    return VRTE_OK;
}

// ---------------------------------------------------------------- BRDF
}  // extern "C"

namespace {
// vrte_compute_brdf with an explicit device (>= -1; -2 = from the environment,
// order-sharded over VRTE_DEVICES when it lists several).
// Debug dumps of vrte_options (pipeline.cpp:333-357, kernel.cpp:188-214): the
// same files and formats as the reference.  Differences: one boundary line per
// order (the boundary matrix is factored once per order for every incident),
// its residual the largest over the order's right-hand sides / residual probes.
struct Dumps {
    std::string eigen, boundary, kernel;
    std::vector<double> nu, residual, bnd, kern;
    bool any() const { return !eigen.empty() || !boundary.empty() || !kernel.empty(); }
};

Dumps prepare_dumps(const vrte_options* options, BrdfSetup& s) {
    Dumps d;
    if (!options) return d;
    if (options->dump_eigen_path) d.eigen = options->dump_eigen_path;
    if (options->dump_boundary_path) d.boundary = options->dump_boundary_path;
    if (options->dump_kernel_path) d.kernel = options->dump_kernel_path;
    if (!d.any()) return d;
    const size_t S = s.rep.size(), L = s.L, dd = 4 * (size_t)s.quad.n, N = s.quad.n;
    if (!d.eigen.empty()) {
        d.nu.resize(S * L * dd * 2);
        d.residual.resize(S * L * dd);
        s.prob.dump_nu = d.nu.data();
        s.prob.dump_residual = d.residual.data();
    }
    if (!d.boundary.empty()) {
        d.bnd.resize(L * 2);
        s.prob.dump_boundary = d.bnd.data();
    }
    if (!d.kernel.empty()) {
        d.kern.resize(L * N * N * 32);
        s.prob.dump_kernel = d.kern.data();
    }
    s.prob.devices = nullptr;  // dumps come from the single-device path
    s.prob.n_devices = 0;
    return d;
}

void write_dumps(const Dumps& d, const BrdfSetup& s) {
    const int L = s.L, N = s.quad.n, dd = 4 * N;
    char buf[200];
    if (!d.kernel.empty()) {
        std::ofstream out(d.kernel);
        if (!out) throw ValidationError("cannot open kernel dump file: " + d.kernel);
        out << "m,i,j,sign_i,sign_j";
        for (int e = 0; e < 16; ++e) out << ",a" << (e / 4) << (e % 4);
        out << "\n";
        const double ds[4] = {1.0, 1.0, -1.0, -1.0};  // parity_conjugate (kernel.cpp:20-27)
        for (int m = 0; m < L; ++m)
            for (int si = 0; si < 2; ++si)
                for (int sj = 0; sj < 2; ++sj)
                    for (int i = 0; i < N; ++i)
                        for (int j = 0; j < N; ++j) {
                            // pp, pm from the device; mp = D pm D, mm = D pp D
                            const double* blk = &d.kern[(((size_t)m * N + i) * N + j) * 32 + (si == sj ? 0 : 16)];
                            out << m << ',' << i << ',' << j << ',' << (si == 0 ? 1 : -1) << ',' << (sj == 0 ? 1 : -1);
                            for (int r = 0; r < 4; ++r)
                                for (int c = 0; c < 4; ++c) {
                                    const double v = si == 0 ? blk[4 * r + c] : ds[r] * ds[c] * blk[4 * r + c];
                                    std::snprintf(buf, sizeof buf, "%.17g", v);
                                    out << ',' << buf;
                                }
                            out << "\n";
                        }
    }
    if (!d.eigen.empty()) {
        std::ofstream out(d.eigen);
        out << "m,lambda_re,lambda_im,nu_re,nu_im,residual\n";
        for (size_t sig = 0; sig < s.sig_to_medium.size(); ++sig) {
            const int med = s.sig_to_medium[sig];
            for (int m = 0; m < L; ++m) {
                const size_t base = ((size_t)med * L + m) * dd;
                std::vector<int> idx(dd);
                for (int j = 0; j < dd; ++j) idx[j] = j;
                // the reference's mode order (homogeneous.cpp:272-276)
                std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) {
                    const double ar = d.nu[2 * (base + a)], br = d.nu[2 * (base + b)];
                    if (ar != br) return ar > br;
                    return d.nu[2 * (base + a) + 1] < d.nu[2 * (base + b) + 1];
                });
                for (int j : idx) {
                    const std::complex<double> nu(d.nu[2 * (base + j)], d.nu[2 * (base + j) + 1]);
                    const std::complex<double> lambda = 1.0 / (nu * nu);
                    std::snprintf(buf, sizeof buf, "%d,%.17g,%.17g,%.17g,%.17g,%.3g\n", m, lambda.real(), lambda.imag(),
                                  nu.real(), nu.imag(), d.residual[base + j]);
                    out << buf;
                }
            }
        }
    }
    if (!d.boundary.empty()) {
        std::ofstream out(d.boundary);
        out << "m,condition_estimate,residual\n";
        for (int m = 0; m < L; ++m) {
            std::snprintf(buf, sizeof buf, "%d,%.6g,%.3g\n", m, d.bnd[2 * m], d.bnd[2 * m + 1]);
            out << buf;
        }
    }
}

vrte_status compute_brdf_on(const vrte_material* material, const vrte_options* options, const double* mu_in,
                            size_t n_mu_in, int32_t n_dphi, const double* basis, int device, vrte_brdf** out,
                            bool concurrent = false) {
    if (!material || !out || !mu_in || n_mu_in == 0) return set_error(VRTE_E_ARGUMENT, "null argument");
    return guarded([&] {
        const double t0 = wall_now();
        auto h = std::make_unique<vrte_brdf>();
        BrdfSetup s;
        build_setup(s, material->spec, options, mu_in, n_mu_in, n_dphi, basis);
        if (device >= -1) {
            s.prob.device = device;
            s.prob.devices = nullptr;
            s.prob.n_devices = 0;
        }
        const Dumps dumps = prepare_dumps(options, s);
        s.prob.concurrent = concurrent ? 1 : 0;
        const int N = s.quad.n, np = s.prob.n_dphi;
        BrdfTable& t = h->table;
        t.mu_in = s.mu_in_user;
        t.mu_out = s.quad_out.nodes;
        t.dphi = s.dphi;
        t.quadrature_n = N;
        t.order_count = s.L;
        t.material_hash = material_hash(s.spec);
        t.entries.resize(n_mu_in * (size_t)s.quad_out.n * np * 16);  // overwritten by the device result
        vrte_cuda_result r{};
        const int32_t rc = vrte_cuda_brdf(&s.prob, t.entries.data(), &r);
        if (rc == 5) throw std::invalid_argument(r.message);
        if (rc != 0) throw NumericalError(r.message);
        if (dumps.any()) write_dumps(dumps, s);
        h->quadrature = s.quad_out;
        const uint64_t S = s.rep.size(), L = s.L, nb = 4;
        h->timings.homogeneous = r.t_homogeneous;
        h->timings.particular = r.t_particular;
        h->timings.boundary = r.t_boundary;
        h->timings.reconstruction = 0.0;  // BRDF path leaves it 0
        h->timings.homogeneous_solves = S * L;
        h->timings.particular_solves = n_mu_in * nb * 2 * L * S;
        h->timings.boundary_solves = n_mu_in * nb * L;
        h->timings.reconstruction_items = 0;
        h->stats.t_homogeneous = r.t_homogeneous;
        h->stats.t_particular = r.t_particular;
        h->stats.t_boundary = r.t_boundary;
        h->stats.t_synthesis = r.t_synthesis;
        h->stats.dithered = r.dithered;
        h->stats.clamped = r.clamped;
        h->stats.polished = r.polished;
        h->stats.kernel_launches = r.kernel_launches;
        h->stats.max_eigen_residual = r.max_eigen_residual;
        h->stats.max_particular_residual = r.max_particular_residual;
        h->stats.max_balance_residual = r.max_balance_residual;
        h->stats.max_boundary_residual = r.max_boundary_residual;
        h->stats.max_boundary_condition = r.max_boundary_condition;
        h->stats.boundary_refined = r.boundary_refined;
        h->stats.boundary_fallback = r.boundary_fallback;
        h->stats.eigen_slots = r.eigen_slots;
        h->stats.boundary_cond_warnings = r.boundary_cond_warnings;
        h->stats.material_hash = t.material_hash;
        h->timings.total_wall = wall_now() - t0;
        *out = h.release();
        return VRTE_OK;
    });
}
}  // namespace

extern "C" {

vrte_status vrte_compute_brdf(const vrte_material* material, const vrte_options* options,
                              const double* mu_in, size_t n_mu_in, int32_t n_dphi,
                              const double* basis, vrte_brdf** out) {
    return compute_brdf_on(material, options, mu_in, n_mu_in, n_dphi, basis, -2, out);
}

vrte_status vrte_compute_brdf_batch(const vrte_material* const* materials, size_t count,
                                    const vrte_options* options, const double* mu_in, size_t n_mu_in,
                                    int32_t n_dphi, const double* basis, int32_t concurrency,
                                    vrte_brdf** out) {
    if (!materials || !out || !mu_in || n_mu_in == 0) return set_error(VRTE_E_ARGUMENT, "null argument");
    for (size_t i = 0; i < count; ++i) out[i] = nullptr;
    // Band sharding: request i runs on devices[i % D] of
    // VRTE_DEVICES (whole bands, no order sharding inside a band); without it,
    // every request runs on the caller's device, resolved here on the calling
    // thread (the workers are fresh threads whose current device is 0).
    std::vector<int> devs;
    try {
        devs = env_devices();
    } catch (const std::exception& e) {
        return set_error(VRTE_E_VALIDATION, e.what());
    }
    if (devs.empty()) {
        int d = env_device();
        if (d < 0 && vrte_cuda_device_count() > 0) d = vrte_cuda_current_device();
        devs.push_back(d);
    }
    const size_t per_dev = concurrency > 0 ? (size_t)concurrency : 2;
    const size_t nthreads = std::min<size_t>(count, per_dev * devs.size());
    std::atomic<size_t> next{0};
    std::mutex mtx;
    vrte_status first = VRTE_OK;
    size_t first_index = count;
    std::string first_msg;
    auto worker = [&] {
        for (size_t i = next++; i < count; i = next++) {
            vrte_brdf* h = nullptr;
            const vrte_status rc = materials[i] ? compute_brdf_on(materials[i], options, mu_in, n_mu_in, n_dphi,
                                                                  basis, devs[i % devs.size()], &h, nthreads > 1)
                                                : set_error(VRTE_E_ARGUMENT, "null material");
            if (rc == VRTE_OK) {
                out[i] = h;
            } else {
                std::lock_guard<std::mutex> lk(mtx);
                if (i < first_index) {
                    first_index = i;
                    first = rc;
                    first_msg = g_last_error;
                }
            }
        }
    };
    std::vector<std::thread> pool;
    for (size_t k = 1; k < nthreads; ++k) pool.emplace_back(worker);
    worker();
    for (auto& th : pool) th.join();
    if (first != VRTE_OK) return set_error(first, first_msg);
    return VRTE_OK;
}

vrte_status vrte_brdf_size(const vrte_brdf* brdf, size_t* n_in, size_t* n_out, size_t* n_dphi) {
    if (!brdf) return set_error(VRTE_E_ARGUMENT, "null brdf");
    if (n_in) *n_in = brdf->table.mu_in.size();
    if (n_out) *n_out = brdf->table.mu_out.size();
    if (n_dphi) *n_dphi = brdf->table.dphi.size();
    return VRTE_OK;
}

vrte_status vrte_brdf_entry(const vrte_brdf* brdf, size_t in_index, size_t out_index,
                            size_t dphi_index, double entry[16]) {
    if (!brdf || !entry) return set_error(VRTE_E_ARGUMENT, "null argument");
    const auto& t = brdf->table;
    if (in_index >= t.mu_in.size() || out_index >= t.mu_out.size() || dphi_index >= t.dphi.size())
        return set_error(VRTE_E_ARGUMENT, "brdf index out of range");
    const double* m =
        &t.entries[((in_index * t.mu_out.size() + out_index) * t.dphi.size() + dphi_index) * 16];
    std::memcpy(entry, m, 16 * sizeof(double));
    return VRTE_OK;
}

vrte_status vrte_brdf_write_csv(const vrte_brdf* brdf, const char* path) {
    if (!brdf || !path) return set_error(VRTE_E_ARGUMENT, "null argument");
    return guarded([&] {
        write_brdf_csv(path, brdf->table);
        return VRTE_OK;
    });
}

vrte_status vrte_brdf_write_binary(const vrte_brdf* brdf, const char* path) {
    if (!brdf || !path) return set_error(VRTE_E_ARGUMENT, "null argument");
    return guarded([&] {
        write_brdf_binary(path, brdf->table);
        return VRTE_OK;
    });
}

vrte_status vrte_brdf_reflectance(const vrte_brdf* brdf, size_t in_index, double out[4]) {
    if (!brdf || !out) return set_error(VRTE_E_ARGUMENT, "null argument");
    const auto& t = brdf->table;
    if (in_index >= t.mu_in.size()) return set_error(VRTE_E_ARGUMENT, "brdf index out of range");
    // brdf.cpp:127-140
    double acc[4] = {0, 0, 0, 0};
    const double w_phi = kTwoPi / (double)t.dphi.size();
    for (size_t io = 0; io < t.mu_out.size(); ++io)
        for (size_t ip = 0; ip < t.dphi.size(); ++ip) {
            const double* m = &t.entries[((in_index * t.mu_out.size() + io) * t.dphi.size() + ip) * 16];
            const double w = brdf->quadrature.weights[io] * brdf->quadrature.nodes[io] * w_phi;
            for (int c = 0; c < 4; ++c) acc[c] += w * m[c];
        }
    for (int c = 0; c < 4; ++c) out[c] = acc[c];
    return VRTE_OK;
}

vrte_status vrte_brdf_timings(const vrte_brdf* brdf, vrte_timings* out) {
    if (!brdf || !out) return set_error(VRTE_E_ARGUMENT, "null argument");
    *out = brdf->timings;
    return VRTE_OK;
}

void vrte_brdf_free(vrte_brdf* brdf) { delete brdf; }

// ---------------------------------------------------------------- extensions
vrte_status vrte_brdf_grid(const vrte_brdf* brdf, double* mu_in, double* mu_out, double* dphi) {
    if (!brdf) return set_error(VRTE_E_ARGUMENT, "null brdf");
    const auto& t = brdf->table;
    if (mu_in) std::memcpy(mu_in, t.mu_in.data(), sizeof(double) * t.mu_in.size());
    if (mu_out) std::memcpy(mu_out, t.mu_out.data(), sizeof(double) * t.mu_out.size());
    if (dphi) std::memcpy(dphi, t.dphi.data(), sizeof(double) * t.dphi.size());
    return VRTE_OK;
}

vrte_status vrte_brdf_device_stats_get(const vrte_brdf* brdf, vrte_brdf_device_stats* out) {
    if (!brdf || !out) return set_error(VRTE_E_ARGUMENT, "null argument");
    *out = brdf->stats;
    return VRTE_OK;
}

vrte_status vrte_brdf_plan_create(const vrte_material* material, const vrte_options* options,
                                  const double* mu_in, size_t n_mu_in, int32_t n_dphi,
                                  const double* basis, int32_t device, int32_t m_begin,
                                  int32_t m_stride, int32_t n_orders, vrte_cuda_plan** out) {
    if (!material || !out || !mu_in || n_mu_in == 0) return set_error(VRTE_E_ARGUMENT, "null argument");
    return guarded([&] {
        BrdfSetup s;
        build_setup(s, material->spec, options, mu_in, n_mu_in, n_dphi, basis);
        s.prob.device = device;
        s.prob.m_begin = m_begin;
        s.prob.m_stride = m_stride > 0 ? m_stride : 1;
        s.prob.n_orders = n_orders;
        vrte_cuda_result r{};
        const int32_t rc = vrte_cuda_plan_create(&s.prob, out, &r);
        if (rc == 5) throw std::invalid_argument(r.message);
        if (rc != 0) throw NumericalError(r.message);
        return VRTE_OK;
    });
}

vrte_status vrte_brdf_plan_acquire(const vrte_material* material, const vrte_options* options,
                                   const double* mu_in, size_t n_mu_in, int32_t n_dphi,
                                   const double* basis, int32_t device, int32_t m_begin,
                                   int32_t m_stride, int32_t n_orders, vrte_cuda_plan** out) {
    if (!material || !out || !mu_in || n_mu_in == 0) return set_error(VRTE_E_ARGUMENT, "null argument");
    return guarded([&] {
        BrdfSetup s;
        build_setup(s, material->spec, options, mu_in, n_mu_in, n_dphi, basis);
        s.prob.device = device;
        s.prob.m_begin = m_begin;
        s.prob.m_stride = m_stride > 0 ? m_stride : 1;
        s.prob.n_orders = n_orders;
        s.prob.devices = nullptr;
        s.prob.n_devices = 0;
        s.prob.concurrent = 1;  // pooled order shards run several plans per device
        vrte_cuda_result r{};
        const int32_t rc = vrte_cuda_plan_acquire(&s.prob, out, &r);
        if (rc == 5) throw std::invalid_argument(r.message);
        if (rc != 0) throw NumericalError(r.message);
        return VRTE_OK;
    });
}

vrte_status vrte_brdf_from_stacks(const vrte_material* material, const vrte_options* options,
                                  const double* mu_in, size_t n_mu_in, int32_t n_dphi,
                                  const double* basis, const double* up_all_orders, vrte_brdf** out) {
    if (!material || !out || !mu_in || n_mu_in == 0 || !up_all_orders)
        return set_error(VRTE_E_ARGUMENT, "null argument");
    return guarded([&] {
        const double t0 = wall_now();
        auto h = std::make_unique<vrte_brdf>();
        BrdfSetup s;
        build_setup(s, material->spec, options, mu_in, n_mu_in, n_dphi, basis);
        const int N = s.quad.n, np = s.prob.n_dphi;
        BrdfTable& t = h->table;
        t.mu_in = s.mu_in_user;
        t.mu_out = s.quad_out.nodes;
        t.dphi = s.dphi;
        t.quadrature_n = N;
        t.order_count = s.L;
        t.material_hash = material_hash(s.spec);
        t.entries.resize(n_mu_in * (size_t)s.quad_out.n * np * 16);
        vrte_cuda_result r{};
        const int32_t rc = vrte_cuda_synthesize(&s.prob, up_all_orders, t.entries.data(), &r);
        if (rc == 5) throw std::invalid_argument(r.message);
        if (rc != 0) throw NumericalError(r.message);
        h->quadrature = s.quad_out;
        h->stats.clamped = r.clamped;
        h->stats.material_hash = t.material_hash;
        h->timings.total_wall = wall_now() - t0;
        *out = h.release();
        return VRTE_OK;
    });
}

}  // extern "C"
