// gen_random_materials.cpp -- test infrastructure: reproduces the reference's
// randomized test materials (tests/support/materials.hpp:66-84 random_layer,
// acceptance_main.cpp:232-252 random_material, test_boundary.cpp:206-214 and
// acceptance_main.cpp:270-283 layer splitting) with libstdc++'s mt19937_64 and
// uniform_*_distribution (implementation-defined, hence the committed output).
// Build: g++ -O2 -std=c++17 gen_random_materials.cpp -o gen && ./gen > random_materials.json
#include <array>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

struct Layer {
    double omega, tau;
    std::vector<std::array<double, 6>> coeffs;  // beta alpha gamma delta eps zeta
};

static Layer random_layer(std::mt19937_64& rng, int order_count) {
    std::uniform_real_distribution<double> uni(0.0, 1.0);
    Layer layer;
    layer.omega = 0.2 + 0.75 * uni(rng);
    layer.tau = 0.1 + 2.9 * uni(rng);
    layer.coeffs.assign(order_count, {0, 0, 0, 0, 0, 0});
    layer.coeffs[0] = {1, 0, 0, 0.5 * (uni(rng) - 0.5), 0, 0};
    double scale = 1.0;
    for (int l = 1; l < order_count; ++l) {
        scale *= 0.4 + 0.35 * uni(rng);
        // argument evaluation order of greek(...) in the reference: the
        // compiler's (GCC: right to left) -- reproduced explicitly
        const double beta = scale * (2 * l + 1) * (uni(rng) - 0.2);
        const double zeta = scale * (2 * l + 1) * (uni(rng) - 0.3);
        const double eps = scale * (2 * l + 1) * 0.3 * (uni(rng) - 0.5);
        const double delta = scale * (2 * l + 1) * 0.5 * (uni(rng) - 0.5);
        const double gamma = scale * (2 * l + 1) * 0.5 * (uni(rng) - 0.5);
        const double alpha = scale * (2 * l + 1) * (uni(rng) - 0.3);
        layer.coeffs[l] = {beta, alpha, gamma, delta, eps, zeta};
    }
    return layer;
}

static void print_layer(const Layer& L, bool last) {
    std::printf("      {\"omega\": %.17g, \"tau\": %.17g, \"coeffs\": [", L.omega, L.tau);
    for (size_t l = 0; l < L.coeffs.size(); ++l) {
        std::printf("%s[", l ? ", " : "");
        for (int q = 0; q < 6; ++q) std::printf("%s%.17g", q ? ", " : "", L.coeffs[l][q]);
        std::printf("]");
    }
    std::printf("]}%s\n", last ? "" : ",");
}

int main() {
    std::printf("{\n  \"generator\": \"tests/golden/gen_random_materials.cpp (libstdc++ mt19937_64)\",\n");
    // acceptance criterion 5 (seed 20240914): 5 random materials
    std::printf("  \"random_materials_20240914\": [\n");
    {
        std::mt19937_64 rng(20240914);
        for (int trial = 0; trial < 5; ++trial) {
            std::uniform_int_distribution<int> layer_count(1, 3);
            std::uniform_int_distribution<int> orders(2, 5);
            std::uniform_real_distribution<double> uni(0.0, 1.0);
            const int layers = layer_count(rng);
            const int order_count = orders(rng);
            std::vector<Layer> ls;
            for (int p = 0; p < layers; ++p) ls.push_back(random_layer(rng, order_count));
            const double base_pick = uni(rng);
            std::string base = "black";
            double albedo = 0.0;
            if (base_pick >= 0.4) {
                base = "lambertian";
                albedo = uni(rng);
            }
            std::printf("    {\"base\": \"%s\", \"albedo\": %.17g, \"layers\": [\n", base.c_str(), albedo);
            for (int p = 0; p < layers; ++p) print_layer(ls[p], p + 1 == layers);
            std::printf("    ]}%s\n", trial < 4 ? "," : "");
            (void)uni(rng);  // source mu0
            (void)uni(rng);  // stokes q
            (void)uni(rng);  // stokes u
            (void)uni(rng);  // stokes v
        }
    }
    std::printf("  ],\n");
    // test_boundary.cpp:206 (seed 2024): 3 layers split into 2,3,4 identical sublayers
    std::printf("  \"split_2024\": [\n");
    {
        std::mt19937_64 rng(2024);
        for (int trial = 0; trial < 3; ++trial) {
            const Layer layer = random_layer(rng, 3);
            std::printf("    {\"pieces\": %d, \"albedo\": 0.2, \"layer\":\n", 2 + trial);
            print_layer(layer, true);
            std::printf("    }%s\n", trial < 2 ? "," : "");
        }
    }
    std::printf("  ]\n}\n");
    return 0;
}
