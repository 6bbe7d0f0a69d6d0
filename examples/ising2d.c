/* ising2d.c -- the C ABI used directly from C (no Python): a 2D Ising adsorption/desorption
 * lattice (eq.(Arrhenius), the target workload's parameters at a smaller size), Bernoulli(1/2)
 * start uploaded bit-packed, Lie macro-steps, observables after each.
 *
 *   gcc -O2 -I include examples/ising2d.c -L paper_1105_4673_b200 -lkmc_b200 \
 *       -Wl,-rpath,$PWD/paper_1105_4673_b200 -o ising2d && ./ising2d [side] [steps]
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "kmc.h"

#define CHECK(call)                                                                      \
    do {                                                                                 \
        kmc_status st_ = (call);                                                         \
        if (st_ != KMC_OK && st_ != KMC_WTRUNCATED) {                                    \
            fprintf(stderr, "%s failed (%d): %s\n", #call, (int)st_,                     \
                    ctx ? kmc_last_error(ctx) : kmc_create_error());                     \
            return 1;                                                                    \
        }                                                                                \
    } while (0)

static uint64_t splitmix64(uint64_t* s) {   /* input generator only (not the method's RNG) */
    uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

int main(int argc, char** argv) {
    const int64_t side = argc > 1 ? atoll(argv[1]) : 4096;
    const int steps = argc > 2 ? atoi(argv[2]) : 5;
    kmc_ctx* ctx = NULL;
    kmc_geometry geom = {0};
    geom.ndim = 2;
    geom.dims[0] = side;
    geom.dims[1] = side;
    geom.cell[0] = 8;
    geom.cell[1] = 8;
    geom.colours = 0;        /* auto: 2 for spin flip */
    geom.replicas = 1;
    geom.seed = 0xB200;
    kmc_model model = {0};
    model.kind = KMC_ADSDES;
    model.ca = 1.0; model.cd = 1.0; model.beta = 1.5; model.K = 1.0; model.h = -2.0;
    CHECK(kmc_create(&geom, &model, NULL, &ctx));

    /* bit-packed Bernoulli(1/2) start: one u64 word per 8x8 cell, uniform random bits */
    const int64_t nwords = (side / 8) * (side / 8);
    uint64_t* words = (uint64_t*)malloc((size_t)nwords * 8);
    uint64_t s = 12345;
    for (int64_t i = 0; i < nwords; ++i) words[i] = splitmix64(&s);
    CHECK(kmc_set_config_packed(ctx, words, nwords));
    free(words);

    for (int k = 0; k < steps; ++k) {
        CHECK(kmc_run(ctx, 1.0, 1.0, KMC_LIE));
        kmc_obs o;
        CHECK(kmc_observables(ctx, &o, NULL));
        printf("t=%.1f events=%llu coverage=%.6f energy=%.1f\n", o.time, (unsigned long long)o.events,
               o.coverage[1], o.energy);
    }
    kmc_destroy(ctx);
    return 0;
}
