/*
 * oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for the
 * direct-summation N-body hot path of arXiv 2509.19294.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, helper or constant with the CUDA product path
 * (paper_2509_19294_b200/csrc); the product never links or imports it.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (section in brackets),
 * "R#n" = reading #n listed in DESIGN.md section 3 (taken from SURVEY.md
 * section 8(c)).
 *
 * Every function below is the plain definition written out:
 *   - forces: P:134-138 [Sec. 3, force equation]: F_i = sum_{j != i}
 *     G m_i m_j (r_j - r_i) / r_ij^3, here as acceleration a_i = F_i / m_i,
 *     with Plummer softening r^2 -> r^2 + eps^2 (R#1) and the jerk
 *     ("its first time derivative") as the exact time derivative of
 *     the softened acceleration (R#2).  fp64 throughout ("naive,
 *     double-precision brute-force implementation of the O(N^2) algorithm").
 *   - hermite: the fp64 "remaining calculations" of P:158 [Sec. 3], read
 *     as the 4th-order Hermite predictor-corrector P(EC)^1 with shared dt
 *     and the Makino-Aarseth a2/a3 corrector (R#3).
 *   - leapfrog: kick-drift-kick (velocity Verlet) with shared dt on the
 *     accelerations alone -- SURVEY 8(f) row f1 (the "kick-drift update"
 *     alternative BASELINE.json names).
 *   - energy: KE = 1/2 sum m |v|^2, PE = -G sum_{i<j} m_i m_j /
 *     sqrt(r^2 + eps^2) (R#1, R#14), fp64.
 *
 * Layout: SoA, x[c*n + i] is component c (0..2) of particle i.
 * The softening enters as eps2 (the squared softening) exactly as given;
 * parity runs pass eps2 = fp32(eps*eps) (R#18).
 *
 * Threads split the i loop only; each i is a sequential ascending-j sum, so
 * values do not depend on the thread count.  Build: gcc -O2
 * -ffp-contract=off -fopenmp (no fast-math, no FMA contraction).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int oracle_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}

/*
 * Acceleration and jerk of particle i due to all j != i.
 * P:136 [Sec. 3, equation]; jerk per R#2:
 *   d = r_j - r_i, w = v_j - v_i, s = |d|^2 + eps2,
 *   a_i += G m_j d / s^{3/2}
 *   j_i += G m_j ( w / s^{3/2} - 3 (d.w) d / s^{5/2} )
 * Returns 0, or 1 if eps2 == 0 and a distinct pair coincides (s == 0); then
 * *bad_j is set to that j.
 */
static int force_on_i(int64_t n, double G, double eps2, const double* m,
                      const double* x, const double* v, int64_t i,
                      double a_out[3], double j_out[3], int64_t* bad_j) {
    double ax = 0.0, ay = 0.0, az = 0.0;
    double jx = 0.0, jy = 0.0, jz = 0.0;
    const double xi = x[0 * n + i], yi = x[1 * n + i], zi = x[2 * n + i];
    const double vxi = v[0 * n + i], vyi = v[1 * n + i], vzi = v[2 * n + i];
    for (int64_t j = 0; j < n; ++j) {
        if (j == i) continue; /* the sum runs over j != i */
        const double dx = x[0 * n + j] - xi;
        const double dy = x[1 * n + j] - yi;
        const double dz = x[2 * n + j] - zi;
        const double wx = v[0 * n + j] - vxi;
        const double wy = v[1 * n + j] - vyi;
        const double wz = v[2 * n + j] - vzi;
        const double s = dx * dx + dy * dy + dz * dz + eps2;
        if (s == 0.0) { *bad_j = j; return 1; }
        const double ri = 1.0 / sqrt(s);   /* 1/r, correctly rounded ops */
        const double ri2 = ri * ri;        /* 1/r^2 */
        const double ri3 = ri * ri * ri;   /* 1/r^3 */
        const double gm = G * m[j];
        const double dw = dx * wx + dy * wy + dz * wz; /* d . w */
        ax += gm * dx * ri3;
        ay += gm * dy * ri3;
        az += gm * dz * ri3;
        jx += gm * (wx * ri3 - 3.0 * dw * dx * ri3 * ri2);
        jy += gm * (wy * ri3 - 3.0 * dw * dy * ri3 * ri2);
        jz += gm * (wz * ri3 - 3.0 * dw * dz * ri3 * ri2);
    }
    a_out[0] = ax; a_out[1] = ay; a_out[2] = az;
    j_out[0] = jx; j_out[1] = jy; j_out[2] = jz;
    return 0;
}

/*
 * oracle_forces: accelerations and jerks for the particles listed in idx
 * (idx == NULL means all n, in order).  acc, jerk are [3][n_idx] SoA (either
 * may be NULL).  Returns 0; 1 on a coincident pair with eps2 == 0, with
 * bad_pair[0..1] = (i, j) when bad_pair != NULL.
 */
int oracle_forces(int64_t n, double G, double eps2, const double* m,
                  const double* x, const double* v, const int64_t* idx,
                  int64_t n_idx, double* acc, double* jerk, int64_t* bad_pair) {
    if (idx == NULL) n_idx = n;
    int status = 0;
    int64_t bi = -1, bj = -1;
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t k = 0; k < n_idx; ++k) {
        const int64_t i = idx ? idx[k] : k;
        double a[3], jk[3];
        int64_t badj = -1;
        if (force_on_i(n, G, eps2, m, x, v, i, a, jk, &badj)) {
#pragma omp critical
            {
                if (!status || i < bi) { status = 1; bi = i; bj = badj; }
            }
            continue;
        }
        for (int c = 0; c < 3; ++c) {
            if (acc) acc[c * n_idx + k] = a[c];
            if (jerk) jerk[c * n_idx + k] = jk[c];
        }
    }
    if (status && bad_pair) { bad_pair[0] = bi; bad_pair[1] = bj; }
    return status;
}

/*
 * oracle_energy: KE = 1/2 sum_i m_i |v_i|^2 ;
 * PE = -G sum_{i<j} m_i m_j / sqrt(|r_j - r_i|^2 + eps2)  (R#1, R#14).
 * PE is accumulated per i over j > i, then the per-i sums are added in
 * ascending i (independent of the thread count).  Returns 1 on a coincident
 * pair with eps2 == 0.
 */
int oracle_energy(int64_t n, double G, double eps2, const double* m,
                  const double* x, const double* v, double* ke_out,
                  double* pe_out) {
    double* pe_i = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    if (!pe_i) return 2;
    int status = 0;
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 0; i < n; ++i) {
        double s_i = 0.0;
        for (int64_t j = i + 1; j < n; ++j) {
            const double dx = x[0 * n + j] - x[0 * n + i];
            const double dy = x[1 * n + j] - x[1 * n + i];
            const double dz = x[2 * n + j] - x[2 * n + i];
            const double s = dx * dx + dy * dy + dz * dz + eps2;
            if (s == 0.0) {
#pragma omp atomic write
                status = 1;
                continue;
            }
            s_i += m[i] * m[j] / sqrt(s);
        }
        pe_i[i] = s_i;
    }
    double ke = 0.0, pe = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double v2 = v[0 * n + i] * v[0 * n + i] +
                          v[1 * n + i] * v[1 * n + i] +
                          v[2 * n + i] * v[2 * n + i];
        ke += 0.5 * m[i] * v2;
        pe += pe_i[i];
    }
    free(pe_i);
    *ke_out = ke;
    *pe_out = -G * pe;
    return status;
}

/*
 * oracle_hermite: nsteps shared-dt 4th-order Hermite steps, P(EC)^1 (R#3).
 * State x, v [3][n] in/out; acc, jerk [3][n] in/out hold a0, j0 at the
 * current state (computed here first when init_aj != 0) and on return the
 * forces evaluated at the last predicted state, which is what the next step
 * uses as a0, j0.
 *
 * Per step, per particle and component (textbook Taylor predictor, then the
 * Makino-Aarseth corrector):
 *   xp = x + v dt + a0 dt^2/2 + j0 dt^3/6
 *   vp = v + a0 dt + j0 dt^2/2
 *   (a1, j1) = forces at (xp, vp)
 *   a2 = (-6 (a0 - a1) - dt (4 j0 + 2 j1)) / dt^2
 *   a3 = (12 (a0 - a1) + 6 dt (j0 + j1)) / dt^3
 *   x  = xp + a2 dt^4/24 + a3 dt^5/120
 *   v  = vp + a2 dt^3/6 + a3 dt^4/24
 *   a0 <- a1, j0 <- j1
 * Returns 0, 1 on a coincident pair, 2 on allocation failure, 3 on a
 * non-finite state.
 */
int oracle_hermite(int64_t n, double G, double eps2, double dt, int64_t nsteps,
                   const double* m, double* x, double* v, double* acc,
                   double* jerk, int init_aj) {
    const size_t sz = sizeof(double) * 3 * (size_t)n;
    double* xp = (double*)malloc(sz);
    double* vp = (double*)malloc(sz);
    double* a1 = (double*)malloc(sz);
    double* j1 = (double*)malloc(sz);
    int rc = 0;
    if (!xp || !vp || !a1 || !j1) { rc = 2; goto done; }
    if (init_aj && oracle_forces(n, G, eps2, m, x, v, NULL, n, acc, jerk, NULL)) {
        rc = 1; goto done;
    }
    const double dt2 = dt * dt, dt3 = dt2 * dt, dt4 = dt3 * dt, dt5 = dt4 * dt;
    for (int64_t s = 0; s < nsteps; ++s) {
        for (int64_t k = 0; k < 3 * n; ++k) {
            xp[k] = x[k] + v[k] * dt + acc[k] * dt2 / 2.0 + jerk[k] * dt3 / 6.0;
            vp[k] = v[k] + acc[k] * dt + jerk[k] * dt2 / 2.0;
        }
        if (oracle_forces(n, G, eps2, m, xp, vp, NULL, n, a1, j1, NULL)) {
            rc = 1; goto done;
        }
        for (int64_t k = 0; k < 3 * n; ++k) {
            const double a2 = (-6.0 * (acc[k] - a1[k]) - dt * (4.0 * jerk[k] + 2.0 * j1[k])) / dt2;
            const double a3 = (12.0 * (acc[k] - a1[k]) + 6.0 * dt * (jerk[k] + j1[k])) / dt3;
            x[k] = xp[k] + a2 * dt4 / 24.0 + a3 * dt5 / 120.0;
            v[k] = vp[k] + a2 * dt3 / 6.0 + a3 * dt4 / 24.0;
            acc[k] = a1[k];
            jerk[k] = j1[k];
            if (!isfinite(x[k]) || !isfinite(v[k])) rc = 3;
        }
        if (rc) goto done;
    }
done:
    free(xp); free(vp); free(a1); free(j1);
    return rc;
}

/*
 * oracle_leapfrog: nsteps kick-drift-kick steps (velocity Verlet), shared dt.
 * acc [3][n] in/out holds a(x) at the current state (computed first when
 * init_a != 0).  Per step, per particle and component:
 *   v_half = v + a dt/2 ;  x = x + v_half dt ;  a = a(x) ;  v = v_half + a dt/2
 * Returns 0, 1 on a coincident pair, 2 on allocation failure, 3 non-finite.
 */
int oracle_leapfrog(int64_t n, double G, double eps2, double dt, int64_t nsteps,
                    const double* m, double* x, double* v, double* acc, int init_a) {
    double* jerk = (double*)malloc(sizeof(double) * 3 * (size_t)n);
    int rc = 0;
    if (!jerk) return 2;
    if (init_a && oracle_forces(n, G, eps2, m, x, v, NULL, n, acc, jerk, NULL)) {
        rc = 1; goto done;
    }
    for (int64_t s = 0; s < nsteps; ++s) {
        for (int64_t k = 0; k < 3 * n; ++k) {
            v[k] = v[k] + acc[k] * dt / 2.0;   /* kick */
            x[k] = x[k] + v[k] * dt;           /* drift */
        }
        if (oracle_forces(n, G, eps2, m, x, v, NULL, n, acc, jerk, NULL)) { rc = 1; goto done; }
        for (int64_t k = 0; k < 3 * n; ++k) {
            v[k] = v[k] + acc[k] * dt / 2.0;   /* kick */
            if (!isfinite(x[k]) || !isfinite(v[k])) rc = 3;
        }
        if (rc) goto done;
    }
done:
    free(jerk);
    return rc;
}

/*
 * ---------------------------------------------------------------------------
 * Block (individual) time steps -- SURVEY 8(f) row f4, "then block
 * (individual) time steps": the production form of the 4th-order Hermite
 * scheme of R#3 (reading R#28).  Every particle carries its own
 * step dt_i = dt_max / 2^k_i (level k_i, 0 <= k_i <= kmax) and its own time
 * t_i; times are held exactly as integer ticks of dt_max / 2^kmax.  One block
 * step, in this order:
 *   1. t_next = min_i (t_i + dt_i); the active set A = {i : t_i + dt_i == t_next}
 *   2. predict every particle j to t_next with its own Taylor polynomial,
 *      D = t_next - t_j:  xp = x + v D + a D^2/2 + j D^3/6,  vp = v + a D + j D^2/2
 *      (the predictor of oracle_hermite with dt -> D)
 *   3. (a1, j1) for i in A from all predicted j != i (oracle_forces)
 *   4. correct i in A with the corrector of oracle_hermite and dt = dt_i
 *   5. new step from the Aarseth criterion at t_next with the interpolated
 *      derivatives a^(2)(t_next) = a2 + dt_i a3, a^(3) = a3:
 *        dt_c = sqrt(eta (|a1| |a^(2)| + |j1|^2) / (|j1| |a^(3)| + |a^(2)|^2))
 *      and the block rules: if dt_c < dt_i halve until dt_i <= dt_c (or
 *      k == kmax); else if dt_c >= 2 dt_i and t_next is a multiple of 2 dt_i,
 *      double once; otherwise keep.  t_i <- t_next, a0 <- a1, j0 <- j1.
 * Initial levels (init != 0): the largest dt_max / 2^k <= eta_s |a| / |j|
 * (k = 0 when j = 0).  One call advances ncycles * dt_max; every particle is
 * synchronised at the end.  level [n] in/out, stats[0] += block steps,
 * stats[1] += sum over block steps of |A|.  crit [n] (may be NULL) receives
 * the last criterion value dt_c of every particle (eta_s |a|/|j| after init);
 * d2_out, d3_out [3][n] (may be NULL) the a^(2)(t_next), a^(3) it used.
 * Returns 0, 1 coincident pair, 2 allocation failure, 3 non-finite state,
 * 4 invalid arguments.
 */
static double block_dt(double dt_max, int k) { return ldexp(dt_max, -k); }

static double norm3(const double* p, int64_t n, int64_t i) {
    return sqrt(p[0 * n + i] * p[0 * n + i] + p[1 * n + i] * p[1 * n + i] + p[2 * n + i] * p[2 * n + i]);
}

int oracle_block_init_levels(int64_t n, double dt_max, int kmax, double eta_s, const double* acc,
                             const double* jerk, int32_t* level, double* crit) {
    for (int64_t i = 0; i < n; ++i) {
        const double an = norm3(acc, n, i), jn = norm3(jerk, n, i);
        const double dts = jn > 0.0 ? eta_s * an / jn : INFINITY;
        int k = 0;
        while (k < kmax && block_dt(dt_max, k) > dts) ++k;
        level[i] = k;
        if (crit) crit[i] = dts;
    }
    return 0;
}

int oracle_hermite_block(int64_t n, double G, double eps2, double dt_max, int kmax, double eta,
                         double eta_s, int64_t ncycles, const double* m, double* x, double* v,
                         double* acc, double* jerk, int32_t* level, int init, int64_t* stats,
                         double* crit, double* d2_out, double* d3_out) {
    if (n < 1 || kmax < 0 || kmax > 50 || ncycles < 0 || !(dt_max > 0.0) || !(eta > 0.0)) return 4;
    const size_t sz = sizeof(double) * 3 * (size_t)n;
    double* xp = (double*)malloc(sz);
    double* vp = (double*)malloc(sz);
    int64_t* T = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    int64_t* act = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    double* a1 = (double*)malloc(sz);
    double* j1 = (double*)malloc(sz);
    int rc = 0;
    if (!xp || !vp || !T || !act || !a1 || !j1) { rc = 2; goto done; }
    if (init) {
        if (oracle_forces(n, G, eps2, m, x, v, NULL, n, acc, jerk, NULL)) { rc = 1; goto done; }
        oracle_block_init_levels(n, dt_max, kmax, eta_s, acc, jerk, level, crit);
    }
    const double tick = ldexp(dt_max, -kmax);
    const int64_t T_end = ncycles << kmax;
    for (int64_t i = 0; i < n; ++i) {
        if (level[i] < 0 || level[i] > kmax) { rc = 4; goto done; }
        T[i] = 0;
    }
    for (;;) {
        /* 1. next block time and the active set */
        int64_t T_next = INT64_MAX;
        for (int64_t i = 0; i < n; ++i) {
            const int64_t Ti = T[i] + ((int64_t)1 << (kmax - level[i]));
            if (Ti < T_next) T_next = Ti;
        }
        if (T_next > T_end) break;
        int64_t na = 0;
        for (int64_t i = 0; i < n; ++i)
            if (T[i] + ((int64_t)1 << (kmax - level[i])) == T_next) act[na++] = i;
        /* 2. predict everyone to t_next */
        for (int64_t j = 0; j < n; ++j) {
            const double D = (double)(T_next - T[j]) * tick, D2 = D * D, D3 = D2 * D;
            for (int c = 0; c < 3; ++c) {
                const int64_t k = c * n + j;
                xp[k] = x[k] + v[k] * D + acc[k] * D2 / 2.0 + jerk[k] * D3 / 6.0;
                vp[k] = v[k] + acc[k] * D + jerk[k] * D2 / 2.0;
            }
        }
        /* 3. forces on the active particles from all predicted particles */
        if (oracle_forces(n, G, eps2, m, xp, vp, act, na, a1, j1, NULL)) { rc = 1; goto done; }
        /* 4.-5. correct, new step */
        for (int64_t q = 0; q < na; ++q) {
            const int64_t i = act[q];
            const int ki = level[i];
            const double dt = block_dt(dt_max, ki);
            const double dt2 = dt * dt, dt3 = dt2 * dt, dt4 = dt3 * dt, dt5 = dt4 * dt;
            double s_a1 = 0, s_j1 = 0, s_a2 = 0, s_a3 = 0;
            for (int c = 0; c < 3; ++c) {
                const int64_t k = c * n + i;
                const double A1 = a1[c * na + q], J1 = j1[c * na + q];
                const double a2 = (-6.0 * (acc[k] - A1) - dt * (4.0 * jerk[k] + 2.0 * J1)) / dt2;
                const double a3 = (12.0 * (acc[k] - A1) + 6.0 * dt * (jerk[k] + J1)) / dt3;
                x[k] = xp[k] + a2 * dt4 / 24.0 + a3 * dt5 / 120.0;
                v[k] = vp[k] + a2 * dt3 / 6.0 + a3 * dt4 / 24.0;
                acc[k] = A1;
                jerk[k] = J1;
                const double a2t = a2 + dt * a3;     /* a^(2) at t_next */
                if (d2_out) d2_out[k] = a2t;
                if (d3_out) d3_out[k] = a3;
                s_a1 += A1 * A1; s_j1 += J1 * J1; s_a2 += a2t * a2t; s_a3 += a3 * a3;
                if (!isfinite(x[k]) || !isfinite(v[k])) rc = 3;
            }
            const double na1 = sqrt(s_a1), nj1 = sqrt(s_j1), na2 = sqrt(s_a2), na3 = sqrt(s_a3);
            const double den = nj1 * na3 + na2 * na2;
            const double dtc = den > 0.0 ? sqrt(eta * (na1 * na2 + nj1 * nj1) / den) : INFINITY;
            int kn = ki;
            if (dtc < dt) {
                while (kn < kmax && block_dt(dt_max, kn) > dtc) ++kn;
            } else if (ki > 0 && dtc >= 2.0 * dt && T_next % ((int64_t)2 << (kmax - ki)) == 0) {
                kn = ki - 1;
            }
            level[i] = kn;
            T[i] = T_next;
            if (crit) crit[i] = dtc;
        }
        if (rc) goto done;
        if (stats) { stats[0] += 1; stats[1] += na; }
    }
done:
    free(xp); free(vp); free(T); free(act); free(a1); free(j1);
    return rc;
}
