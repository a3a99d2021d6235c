/*
 * c_api_demo.c -- the C-ABI of libnbody.so used from plain C (no Python, no torch).
 *
 *   gcc -O2 -I include -o c_api_demo examples/c_api_demo.c \
 *       -L paper_2509_19294_b200 -lnbody -Wl,-rpath,$PWD/paper_2509_19294_b200 -lm
 *   ./c_api_demo [n]          # needs a GPU for everything after nbody_plan
 *
 * Builds a seeded uniform-cube system in host memory, lets nbody_init copy it to the GPU,
 * evaluates forces into host arrays (nbody_compute_forces), advances 10 Hermite steps
 * (nbody_step) and prints the energy before and after (nbody_energy); then checkpoints
 * (nbody_get_state + nbody_get_derivs), resumes in a second context (nbody_init +
 * nbody_set_derivs) and checks that 5 more steps in both contexts agree bit for bit.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "nbody.h"

static double urand(uint64_t* s) {   /* xorshift64*, seeded: inputs only */
    *s ^= *s >> 12;
    *s ^= *s << 25;
    *s ^= *s >> 27;
    return (double)((*s * 2685821657736338717ULL) >> 11) * (1.0 / 9007199254740992.0);
}

int main(int argc, char** argv) {
    const int64_t n = argc > 1 ? atoll(argv[1]) : 4096;
    int64_t i0, i1, slot, chunk, n_chunks;
    if (nbody_plan(n, 1, 0, 0, &i0, &i1, &slot, &chunk, &n_chunks) != NBODY_OK) {
        fprintf(stderr, "plan: %s\n", nbody_last_error(NULL));
        return 1;
    }
    printf("plan: n=%lld chunk=%lld n_chunks=%lld\n", (long long)n, (long long)chunk,
           (long long)n_chunks);
    if (argc > 2) return 0;   /* plan only (CPU check) */

    double* m = malloc(sizeof(double) * n);
    double* x = malloc(sizeof(double) * 3 * n);
    double* v = malloc(sizeof(double) * 3 * n);
    double* acc = malloc(sizeof(double) * 3 * n);
    double* jerk = malloc(sizeof(double) * 3 * n);
    uint64_t s = 12345;
    for (int64_t i = 0; i < n; ++i) {
        m[i] = 1.0 / (double)n;
        for (int c = 0; c < 3; ++c) {
            x[c * n + i] = 2.0 * urand(&s) - 1.0;
            v[c * n + i] = 0.1 * (2.0 * urand(&s) - 1.0);
        }
    }
    nbody_config cfg = {0};
    cfg.n = n;
    cfg.G = 1.0;
    cfg.eps = 1e-2;
    cfg.dt = 1.0 / 1024;
    cfg.integrator = NBODY_HERMITE4;
    cfg.world = 1;
    nbody_ctx* ctx = NULL;
    if (nbody_init(&cfg, m, x, v, &ctx) != NBODY_OK) {
        fprintf(stderr, "init: %s\n", nbody_last_error(NULL));
        return 1;
    }
    double ke0, pe0, ke1, pe1;
    int rc = nbody_compute_forces(ctx, acc, jerk);
    if (!rc) rc = nbody_energy(ctx, &ke0, &pe0);
    if (!rc) rc = nbody_step(ctx, 10);
    if (!rc) rc = nbody_energy(ctx, &ke1, &pe1);
    if (!rc) rc = nbody_get_state(ctx, x, v);
    if (rc) {
        fprintf(stderr, "error %d: %s\n", rc, nbody_last_error(ctx));
        nbody_destroy(ctx);
        return 1;
    }
    double px = 0, py = 0, pz = 0;
    for (int64_t i = 0; i < n; ++i) {
        px += m[i] * acc[i];
        py += m[i] * acc[n + i];
        pz += m[i] * acc[2 * n + i];
    }
    printf("a[0] = (%.6e, %.6e, %.6e)  sum m a = (%.1e, %.1e, %.1e)\n", acc[0], acc[n], acc[2 * n], px,
           py, pz);
    printf("E0 = %.12f  E(10 dt) = %.12f  rel. change %.2e\n", ke0 + pe0, ke1 + pe1,
           fabs((ke1 + pe1) - (ke0 + pe0)) / fabs(ke0 + pe0));
    /* checkpoint at this call boundary, resume in a fresh context, 5 more steps in both */
    double* x2 = malloc(sizeof(double) * 3 * n);
    double* v2 = malloc(sizeof(double) * 3 * n);
    nbody_ctx* ctx2 = NULL;
    rc = nbody_get_derivs(ctx, acc, jerk);
    if (!rc) rc = nbody_init(&cfg, m, x, v, &ctx2);
    if (!rc) rc = nbody_set_derivs(ctx2, acc, jerk);
    if (!rc) rc = nbody_step(ctx, 5);
    if (!rc) rc = nbody_step(ctx2, 5);
    if (!rc) rc = nbody_get_state(ctx, x, v);
    if (!rc) rc = nbody_get_state(ctx2, x2, v2);
    if (rc) {
        fprintf(stderr, "resume error %d: %s\n", rc, nbody_last_error(ctx2 ? ctx2 : ctx));
        nbody_destroy(ctx2);
        nbody_destroy(ctx);
        return 1;
    }
    int same = 1;
    for (int64_t k = 0; k < 3 * n; ++k) same &= x[k] == x2[k] && v[k] == v2[k];
    printf("resume: %s\n", same ? "bit-identical" : "DIFFERS");
    nbody_destroy(ctx2);
    nbody_destroy(ctx);
    free(m); free(x); free(v); free(acc); free(jerk); free(x2); free(v2);
    return same ? 0 : 1;
}
