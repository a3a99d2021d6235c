/*
 * nbody.h -- C-ABI of libnbody.so, the B200-native (sm_100a) hot path of
 * direct-summation gravitational N-body simulation (arXiv 2509.19294).
 *
 * The library computes what the paper offloads to its accelerator -- the
 * O(N^2) pairwise acceleration and its time derivative (jerk) for every
 * particle, P:134-138 [Sec. 3, force equation and "the acceleration and its
 * first time derivative (jerk) for each particle in all three spatial
 * dimensions"] -- in FP32 (P:158 [Sec. 3] "acceleration, jerk, and other
 * intermediate values within the force calculation are computed in single
 * precision"), and the fp64 "remaining calculations" of P:158 (the particle
 * update of a 4th-order Hermite integrator, reading R#3) on the
 * GPU instead of the host.  i-particles are sharded over ranks (P:140
 * [Sec. 3] "the outer for-loop ... is distributed"; P:251 future work "MPI
 * with multiple accelerators") and the j-set is all-gathered every step
 * with NCCL ("each core requires access to the complete set of
 * particle data").
 *
 * Conventions for every function below:
 *  - Return value: an nbody_status; 0 == NBODY_OK.  A message naming the
 *    offending index where there is one is available from
 *    nbody_last_error().  After an asynchronous failure (CUDA, NCCL,
 *    non-finite state) the context is sticky: every later call returns
 *    NBODY_ESTATE until nbody_destroy().
 *  - Array layout: structure-of-arrays fp64.  A "[3][k]" array holds
 *    component c of particle i at index c*k + i.
 *  - Pointers may be device pointers or host pointers (pageable or pinned);
 *    the library resolves them through unified addressing and copies with
 *    cudaMemcpy*Async on the context's stream.  Caller-owned memory stays
 *    caller-owned; the context owns every internal buffer, event, stream and
 *    communicator and nbody_destroy() releases them.
 *  - Ordering: all device work is stream-ordered on cfg->stream (or a
 *    library-created stream when NULL).  Functions that return host values
 *    (nbody_energy, nbody_sync, nbody_get_state into host memory,
 *    nbody_prof_read) block until the work they depend on is done.
 *  - Collectives: with world > 1 (and loopback == 0) nbody_init,
 *    nbody_compute_forces, nbody_step, nbody_energy and nbody_destroy are
 *    collective: every rank calls them in the same order, as in MPI.
 *  - Threading: one host thread per context at a time.
 *  - Determinism: for fixed (n, eps, dt, jchunks) results are bit-identical
 *    across world sizes, loopback and repeated runs (DESIGN.md section 6,
 *    canonical reduction order).
 */
#ifndef NBODY_H
#define NBODY_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nbody_ctx nbody_ctx; /* opaque; owns all device state */

enum nbody_status {
    NBODY_OK = 0,
    NBODY_EINVAL = 1,     /* invalid argument or configuration (names index)   */
    NBODY_ENONFINITE = 2, /* non-finite particle state (names the particle)    */
    NBODY_ECUDA = 3,      /* CUDA runtime / launch failure                     */
    NBODY_ENCCL = 4,      /* NCCL failure or library not loadable              */
    NBODY_ENOMEM = 5,     /* device allocation failed                          */
    NBODY_ESTATE = 6      /* context is in a failed (sticky) state             */
};

enum nbody_integrator {
    NBODY_HERMITE4 = 0,       /* 4th-order Hermite P(EC)^1, shared dt (R#3)     */
    NBODY_LEAPFROG_KDK = 1,   /* kick-drift-kick leapfrog, accel only (NEXT f1) */
    NBODY_HERMITE4_BLOCK = 2  /* Hermite-4 with block (individual) time steps
                                 dt_i = dt / 2^k_i (NEXT f4, R#28)    */
};

typedef struct {
    int64_t n;            /* total particles over all ranks, >= 2; at most      
                             2^31 - 1 per shard (n / world, rounded up)        */
    double G;             /* gravitational constant, finite, > 0               */
    double eps;           /* Plummer softening, finite, >= 0 (R#1).  The force
                             kernel uses eps2 = fp32(eps*eps) (R#18).  eps == 0
                             is accepted; coincident distinct particles then
                             give a non-finite force -> NBODY_ENONFINITE.      */
    double dt;            /* shared time step, finite, > 0                     */
    int32_t integrator;   /* enum nbody_integrator                             */
    int32_t device;       /* CUDA device ordinal of this rank                  */
    int32_t rank;         /* i-shard index, 0 <= rank < world (ignored when
                             loopback != 0)                                    */
    int32_t world;        /* number of i-shards, 1 <= world <= n               */
    int32_t loopback;     /* != 0: emulate all `world` shards inside this one
                             context on one GPU, shard by shard (test mode; no
                             NCCL).  Every shard packs into its own exchange
                             buffer; the all-gather is emulated by one device
                             copy per remote slice into it, issued between the
                             same local-chunk and remote-chunk force launches
                             an NCCL rank issues (environment
                             NBODY_LOOPBACK_CONCURRENT=1: in the rank's stream
                             form instead -- copies and remote launch on a
                             second stream, concurrent with the local launch).
                             Outputs cover all n.                              */
    int32_t jchunks;      /* max number of j-chunks of the canonical reduction
                             (0 -> 128).  Must be equal on every rank.          */
    int32_t hilo;         /* != 0: two-float positions (NEXT f2): packets also
                             carry lo = fp32(x - fp32(x)) and the force kernel
                             forms d = (xj_hi - xi_hi) + (xj_lo - xi_lo), so
                             fp64 states off the fp32 grid keep ~1e-6 relative
                             force error (+6 FADD per interaction).            */
    const uint8_t* nccl_id; /* 128-byte ncclUniqueId from nbody_nccl_unique_id
                             on rank 0, broadcast by the caller; required when
                             world > 1 and loopback == 0; optional with
                             world == 1 (then a 1-rank NCCL communicator is
                             used for the exchange).  The communicator is
                             non-blocking: every NCCL call waits at most
                             NBODY_NCCL_TIMEOUT_S seconds (environment,
                             default 600) to make progress, else NBODY_ENCCL
                             (a missing or dead peer rank).                    */
    void* stream;         /* cudaStream_t to order work on; NULL -> the library
                             creates a non-blocking stream; pass
                             cudaStreamLegacy ((void*)1) for the legacy
                             default stream                                    */
    /* NBODY_HERMITE4_BLOCK only (ignored otherwise); dt above is the largest
     * step dt_max, and every particle steps with dt_max / 2^k, 0 <= k <= kmax. */
    double eta;           /* Aarseth accuracy parameter, finite, > 0 (0.01-0.02
                             typical): dt_c = sqrt(eta (|a||a2| + |j|^2) /
                             (|j||a3| + |a2|^2))                               */
    double eta_s;         /* startup parameter, finite, > 0: first level from
                             eta_s |a| / |j|                                   */
    int32_t kmax;         /* deepest level, 0 <= kmax <= 50 (0 -> 20)           */
} nbody_config;

/* Partition and reduction plan (pure host function, no GPU needed).
 * Rank r owns the contiguous global range [i0, i1) with
 * i0 = r * slot, i1 = min(n, (r + 1) * slot), slot = B * ceil(n / (B world)) with
 * B = 1024, the force kernel's i-block,
 * so all ranks but the last own `slot` particles (SPEC S:96 partition,
 * read with padding at the tail only so the j order never depends on world).
 * chunk = 256 * ceil(n / (256 * jchunks)) j-particles per canonical
 * reduction chunk, n_chunks = ceil(n / chunk).  Any output pointer may be
 * NULL.  Returns NBODY_EINVAL for n < 2, world < 1, world > n, rank outside
 * [0, world), jchunks < 0 or slot > 2^31 - 1. */
int nbody_plan(int64_t n, int32_t world, int32_t rank, int32_t jchunks,
               int64_t* i0, int64_t* i1, int64_t* slot, int64_t* chunk,
               int64_t* n_chunks);

/* Writes a fresh 128-byte ncclUniqueId to out (call on rank 0 only, then
 * broadcast it).  Returns NBODY_ENCCL if libnccl cannot be loaded. */
int nbody_nccl_unique_id(uint8_t out[128]);

/* Creates a context for this rank.  m [n], x [3][n], v [3][n] describe the
 * FULL system (P:136 masses and position vectors; velocities for the jerk,
 * P:138); each rank copies its own shard (all shards when loopback != 0) and
 * blocks until the copy is done, so the caller may free the inputs on
 * return.  Validation, returning NBODY_EINVAL with the
 * first bad index in the message: n >= 2; m finite and > 0; x and v finite;
 * G > 0; eps >= 0; dt > 0; 0 <= rank < world <= n; integrator known; with
 * eps > 0, G max(m) / eps^3 <= 1e30 (the fp32 range of the pair terms,
 * G m_j / s^{3/2} <= G m_j / eps^3).  fp32(eps^2) below FLT_MIN (eps = 0, or
 * subnormal, which the FTZ force pass flushes to 0) selects the guarded pass
 * that excludes s == 0 (R#17).  On error *out is NULL. */
int nbody_init(const nbody_config* cfg, const double* m, const double* x,
               const double* v, nbody_ctx** out);

/* This context's particle range [i0, i1) in global order ([0, n) in
 * loopback mode). */
int nbody_local_range(const nbody_ctx* ctx, int64_t* i0, int64_t* i1);

/* Evaluates acceleration and jerk of every local particle at the current
 * state (jerk R#2), caches them as the Hermite a0, j0 and writes
 * them, stream-ordered, to acc / jerk ([3][i1 - i0] each; either may be
 * NULL).  With NBODY_LEAPFROG_KDK only the acceleration is evaluated (the
 * 18-flop acceleration-only kernel) and a non-NULL jerk is zero-filled.  G m_j (r_j - r_i) / (r^2 + eps^2)^{3/2} summed over all j in FP32
 * per 256-j tile, tiles and chunks folded in fp64 in a fixed order.
 * With eps > 0 the j == i term is exactly zero.  Collective. */
int nbody_compute_forces(nbody_ctx* ctx, double* acc, double* jerk);

/* Advances the state by nsteps >= 1 steps of dt of the configured
 * integrator.  Hermite: evaluates a0, j0 first if not cached, then per step
 * predict (fp64) -> exchange -> force (FP32) -> correct (fp64): exactly one
 * force evaluation per step (P(EC)^1, R#3).  Leapfrog (NEXT f1): kick
 * v += a dt/2, drift x += v dt -> exchange -> acceleration-only force pass ->
 * kick v += a dt/2, one evaluation per step.  Non-blocking; a non-finite
 * state is reported by the next blocking call.
 * Block time steps (NBODY_HERMITE4_BLOCK, R#28): advances nsteps * dt with
 * individual steps dt_i = dt / 2^k_i; each block step predicts every
 * particle to t_next = min_i(t_i + dt_i) (fp64), exchanges the packets,
 * evaluates forces on the active set {i : t_i + dt_i == t_next} only,
 * corrects it with its own dt_i and picks its next level from the Aarseth
 * criterion (halve as often as needed, double at most once and only when
 * t_next is a multiple of 2 dt_i).  Levels start from eta_s |a| / |j| at the
 * first step after init or nbody_set_state(keep_forces = 0).  Every
 * particle is synchronised at the end of the call.  With world = 1 or
 * loopback shards the whole call is one CUDA-graph launch that sizes every
 * force pass on the device (non-blocking, except the first call, which builds
 * the graph); with NCCL ranks or kernel timing on it blocks once per block
 * step.  Collective. */
int nbody_step(nbody_ctx* ctx, int32_t nsteps);

/* Checkpoint / exact resume.  The state between steps is (x, v) plus the
 * derivatives the next step starts from: a0, j0 of the last P(EC)^1 step,
 * evaluated at the predicted positions, so re-evaluating them at the
 * corrected state (what a fresh nbody_init does) changes the next step in
 * the last bits.  nbody_get_derivs copies them ([3][i1 - i0] each, host or
 * device; evaluated first if no step or force call has produced them; jerk
 * ignored for the leapfrog integrator, may be NULL), blocking for host
 * pointers.  nbody_set_derivs restores them into a context holding the
 * same (x, v) (after nbody_init or nbody_set_state): the next nbody_step
 * then continues bit for bit as the saved run would have (checks
 * finiteness: NBODY_EINVAL naming the index; jerk required for the Hermite
 * integrators).  nbody_set_levels (block time steps only) restores every
 * local particle's level k_i (int32 [i1 - i0], host or device; NBODY_EINVAL
 * naming a level outside [0, kmax]) so the next nbody_step keeps them instead
 * of restarting from eta_s.  A saved block run is (x, v, a0, j0, levels) at
 * a call boundary, where every particle is synchronised.  Blocks. */
int nbody_get_derivs(nbody_ctx* ctx, double* acc, double* jerk);
int nbody_set_derivs(nbody_ctx* ctx, const double* acc, const double* jerk);
int nbody_set_levels(nbody_ctx* ctx, const int32_t* level);

/* Block time steps only: block steps taken and sum over them of the active
 * count since init (either may be NULL), and the current level k_i of every
 * local particle (level: int32 [i1 - i0], host or device, may be NULL; all
 * zero before the first step).  Blocks.  NBODY_EINVAL for other integrators. */
int nbody_block_stats(nbody_ctx* ctx, int64_t* block_steps, int64_t* active_sum,
                      int32_t* level);

/* Total kinetic and potential energy of the whole system (all ranks) in
 * fp64: KE = 1/2 sum m |v|^2, PE = -G sum_{i<j} m_i m_j / sqrt(r^2 + eps^2)
 * with eps^2 = fp32(eps*eps) (R#14, R#18).  Host scalars; blocks.
 * Collective. */
int nbody_energy(nbody_ctx* ctx, double* kinetic, double* potential);

/* Copies the current local state x, v ([3][i1 - i0] each, either may be
 * NULL) to the given pointers; blocks when a pointer is host memory. */
int nbody_get_state(nbody_ctx* ctx, double* x, double* v);

/* Replaces the local state with x, v ([3][i1 - i0], host or device).  With
 * keep_forces != 0 the caller asserts the state is the one nbody_get_state
 * returned (round trip through the host, as the paper's host-side
 * integrator does), so the cached a0, j0 stay valid; otherwise they
 * are invalidated and re-evaluated by the next step.  Checks finiteness
 * (NBODY_EINVAL naming the index).  Collective only through later calls. */
int nbody_set_state(nbody_ctx* ctx, const double* x, const double* v,
                    int32_t keep_forces);

/* Blocks until all enqueued work is done and surfaces asynchronous errors
 * (NBODY_ENONFINITE naming the first non-finite particle, NBODY_ECUDA,
 * NBODY_ENCCL). */
int nbody_sync(nbody_ctx* ctx);

/* Kernel timing for measurement.  nbody_prof_enable(ctx, 1) makes the
 * context bracket every force-kernel launch with CUDA events on the stream
 * that launches it; nbody_prof_read blocks, then returns the summed event
 * time of those launches (ms), their count, and the count of all kernels
 * this context launched since the last reset (reset != 0 clears all three
 * after reading; kernels a block-step CUDA graph launches on the device are
 * counted from the device's block-step counter).  Any output may be NULL. */
int nbody_prof_enable(nbody_ctx* ctx, int32_t on);
int nbody_prof_read(nbody_ctx* ctx, double* force_ms, int64_t* force_launches,
                    int64_t* kernel_launches, int32_t reset);

/* Per-launch force-kernel times (ms, launch order) recorded since the last
 * reset while profiling was on: writes min(count, cap) values to ms and the
 * total number recorded to *count.  Blocks.  In loopback mode the launches of
 * shard s follow those of shard s - 1 within each evaluation, so per-shard
 * (per-emulated-GPU) times can be read off (scripts/project_scaling.py). */
int nbody_prof_launch_times(nbody_ctx* ctx, double* ms, int64_t cap, int64_t* count);

/* Sizes of the same launches: i particles (the active count for block time
 * steps, read on the host loop that profiling selects) and real (unpadded) j
 * particles, so n_i[k] * n_j[k] is launch k's interaction count.  Host-only,
 * does not block; writes min(count, cap) entries of each non-NULL array. */
int nbody_prof_launch_sizes(nbody_ctx* ctx, int64_t* n_i, int64_t* n_j, int64_t cap,
                            int64_t* count);

/* How steps were executed since init: shared-step CUDA-graph replays (one
 * per step; block time steps: one per nbody_step call) and steps launched
 * eagerly kernel by kernel (any output may be NULL).  Host-only. */
int nbody_exec_stats(const nbody_ctx* ctx, int64_t* graph_launches, int64_t* eager_steps);

/* Message for the last failure on ctx (or of the last failed nbody_init /
 * plan call when ctx is NULL).  Never NULL; valid until the next call. */
const char* nbody_last_error(const nbody_ctx* ctx);

/* Releases everything the context owns.  NULL is a no-op.  Collective for a
 * healthy context (ncclCommFinalize, bounded by NBODY_NCCL_TIMEOUT_S); a
 * context in the sticky failed state, or whose finalize times out, aborts its
 * communicator (ncclCommAbort) and returns without waiting for peers. */
void nbody_destroy(nbody_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* NBODY_H */
