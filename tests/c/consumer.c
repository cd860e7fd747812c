/* A plain C consumer of the drop-in library, written against the reference
 * header's API only (include/vrte/vrte.h), as an application linked with
 * -lvrte would be (proj/README.md:142-162, tests/test_capi.cpp:85-119).
 *
 *   consumer <material.json> [N] [--solve]
 *
 * Loads the material, prints L and the layer count; with --solve it computes
 * the BRDF at mu_in = {0.6, 1.0} with 5 azimuths and prints F00 of the first
 * entry, the reflectance and the timings' solve counters. Exit code = the
 * first non-OK vrte_status (its text on stderr). */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "vrte/vrte.h"

static int fail(vrte_status s) {
    fprintf(stderr, "vrte status %d: %s\n", (int)s, vrte_last_error());
    return (int)s;
}

int main(int argc, char** argv) {
    if (argc < 2) return 64;
    vrte_material* mat = NULL;
    vrte_status s = vrte_material_load(argv[1], &mat);
    if (s != VRTE_OK) return fail(s);
    int32_t L = 0, layers = 0;
    if ((s = vrte_material_info(mat, &L, &layers)) != VRTE_OK) return fail(s);
    printf("version %s L %d layers %d\n", vrte_version(), (int)L, (int)layers);
    if (argc > 3 && strcmp(argv[3], "--solve") == 0) {
        vrte_options opt;
        vrte_options_init(&opt);
        opt.quadrature_n = atoi(argv[2]);
        const double mu[2] = {0.6, 1.0};
        vrte_brdf* b = NULL;
        if ((s = vrte_compute_brdf(mat, &opt, mu, 2, 5, NULL, &b)) != VRTE_OK) return fail(s);
        size_t n_in = 0, n_out = 0, n_dphi = 0;
        vrte_brdf_size(b, &n_in, &n_out, &n_dphi);
        double e[16], r[4];
        vrte_brdf_entry(b, 0, 0, 0, e);
        vrte_brdf_reflectance(b, 0, r);
        vrte_timings t;
        vrte_brdf_timings(b, &t);
        printf("size %zu %zu %zu F00 %.17g R %.17g solves %llu %llu %llu\n", n_in, n_out, n_dphi, e[0], r[0],
               (unsigned long long)t.homogeneous_solves, (unsigned long long)t.particular_solves,
               (unsigned long long)t.boundary_solves);
        /* out-of-range index: VRTE_E_ARGUMENT, as the reference (capi.cpp:280-281) */
        if (vrte_brdf_entry(b, 2, 0, 0, e) != VRTE_E_ARGUMENT) return 99;
        vrte_brdf_free(b);
    }
    vrte_material_free(mat);
    vrte_material_free(NULL);
    return 0;
}
