// host.hpp -- host-side types of libvrte.so: material model, quadrature,
// validation and the BRDF table.  Restates the reference's input plumbing
// (core/types.*, core/material.*, brdf/brdf.hpp) without Eigen.
#pragma once

#include "vrte/vrte_cuda.h"
#include <array>
#include <new>
#include <utility>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

namespace vrte::host {

constexpr double kPi = 3.14159265358979323846;
constexpr double kTwoPi = 2.0 * kPi;

struct ValidationError : std::runtime_error {  // types.hpp:20-24 -> VRTE_E_VALIDATION
    using std::runtime_error::runtime_error;
};
struct NumericalError : std::runtime_error {  // types.hpp:28-32 -> VRTE_E_NUMERICAL
    using std::runtime_error::runtime_error;
};

using Mat4 = std::array<double, 16>;  // row-major
inline double& at(Mat4& m, int r, int c) { return m[4 * r + c]; }
inline double at(const Mat4& m, int r, int c) { return m[4 * r + c]; }

struct LayerSpec {  // material.hpp:21-27
    double omega = 0.0;
    double tau = 0.0;
    std::vector<Mat4> coeffs;
    int order_count() const { return (int)coeffs.size(); }
};
struct BlackBase {};
struct LambertianBase {
    double rho = 0.0;
};
struct MuellerTableBase {
    int n = 0;
    std::vector<Mat4> table;  // row-major n*n, R(mu_i, -mu_j) at i*n + j
    const Mat4& at(int i, int j) const { return table[(size_t)i * n + j]; }
};
using BaseReflector = std::variant<BlackBase, LambertianBase, MuellerTableBase>;
struct BeamSource {
    double mu0 = 1.0, phi0 = 0.0;
    std::array<double, 4> stokes{1.0, 0.0, 0.0, 0.0};
};
struct MaterialSpec {  // material.hpp:59-71
    std::vector<LayerSpec> layers;
    BaseReflector base = BlackBase{};
    BeamSource source;
    // Extension (absent from the reference): a smooth
    // dielectric interface on top of the stack, refractive index of the medium
    // relative to the outside; 1 = no interface (the reference's model).
    double interface_n = 1.0;
    int order_count() const { return layers.empty() ? 0 : layers.front().order_count(); }
};

struct Quadrature {
    int n = 0;
    std::vector<double> nodes, weights;
};

Quadrature build_double_gauss_quadrature(int n);  // types.cpp:27-68
// Gauss-Legendre on (0, mu_c) with n - n_hi nodes and on (mu_c, 1) with n_hi
// nodes (the Fresnel interface's refraction cone and total-internal-reflection
// range each get a full Gauss rule); ascending nodes.
Quadrature build_split_gauss_quadrature(int n, double mu_c, int n_hi);
// Fresnel Mueller matrices of a smooth interface between the medium (relative
// index n > 1 against the outside) and the outside, row-major, Stokes
// (I, Q = I_par - I_perp, U, V) in the meridian frame (= plane of incidence):
//   reflection for light inside the medium hitting the interface at cosine mu
//   (total internal reflection below the critical cosine), power
//   transmittance outside -> inside at outside cosine mu, and inside -> outside
//   at inside cosine mu; 0 / identity at n = 1.
Mat4 fresnel_reflect_inside(double n, double mu);
Mat4 fresnel_transmit_in(double n, double mu_out);
Mat4 fresnel_transmit_out(double n, double mu_in);
double refract_in(double n, double mu_out);   // outside cosine -> inside cosine
double refract_out(double n, double mu_in);   // inside cosine -> outside (0 beyond the critical angle)
void validate_material(MaterialSpec& spec);       // material.cpp:43-109
std::vector<Mat4> load_coefficient_file(const std::string& path);
MaterialSpec parse_material_json(const std::string& text, const std::string& base_dir);
MaterialSpec load_material_file(const std::string& path);
double reduce_azimuth(double phi);
Mat4 base_row_at(const BaseReflector& base, const Quadrature& quad, double mu_out, double mu_in);
uint64_t material_hash(const MaterialSpec& spec);  // brdf.cpp:11-41

// Page-locked, recycled host storage for the BRDF table: the device result lands
// by DMA at full PCIe/C2C speed, and elements are default-initialized (no
// zero-fill pass over 10 MB before the copy overwrites it).  vrte_cuda_host_*
// (brdf_device.cu) keep a per-size free list; plain heap memory if pinning fails.
template <typename T>
struct PinnedAlloc {
    using value_type = T;
    PinnedAlloc() = default;
    template <typename U>
    PinnedAlloc(const PinnedAlloc<U>&) {}
    T* allocate(size_t n) { return static_cast<T*>(vrte_cuda_host_alloc(n * sizeof(T))); }
    void deallocate(T* p, size_t n) { vrte_cuda_host_free(p, n * sizeof(T)); }
    template <typename U>
    void construct(U* p) {
        ::new (static_cast<void*>(p)) U;  // default-init
    }
    template <typename U, typename... A>
    void construct(U* p, A&&... a) {
        ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
    }
    template <typename U>
    bool operator==(const PinnedAlloc<U>&) const { return true; }
    template <typename U>
    bool operator!=(const PinnedAlloc<U>&) const { return false; }
};

struct BrdfTable {  // brdf.hpp:9-24
    std::vector<double> mu_in, mu_out, dphi;
    std::vector<double, PinnedAlloc<double>> entries;  // [in][out][dphi][16] row-major Mueller
    int quadrature_n = 0, order_count = 0;
    uint64_t material_hash = 0;
};

void write_brdf_csv(const std::string& path, const BrdfTable& t);     // csv.cpp:111-129
// pipeline.hpp RadianceField: values [tau][mu][phi][4]
struct RadianceField {
    std::vector<double> taus, mus, phis, values;
};
void write_radiance_csv(const std::string& path, const RadianceField& f);  // csv.cpp:28-40
void write_brdf_binary(const std::string& path, const BrdfTable& t);  // csv.cpp:147-168

}  // namespace vrte::host
