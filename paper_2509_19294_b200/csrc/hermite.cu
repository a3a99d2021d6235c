// hermite.cu -- fp64 particle update kernels around the force pass.
//
// The paper keeps "all remaining calculations ... in double precision on
// the CPU cores" (P:158 [Sec. 3]); here they stay fp64 but run on the GPU,
// fused so that each step touches the per-particle state once:
//   predict_pack          x, v, a0, j0 -> xp, vp (fp64) and fp32 packets
//   correct_predict_pack  fold chunk partials -> a1, j1; Hermite corrector;
//                         a0 <- a1, j0 <- j1; predictor for the next step;
//                         packets -> the exchange buffer
// With integrator == NBODY_LEAPFROG_KDK (NEXT f1) the same two kernels do the
// kick-drift and the closing kick of kick-drift-kick on accelerations only.
// Block time steps (NEXT f4, R#28) add block_* kernels: next block time,
// active set, predictor of every particle to it, corrector + new level of
// the active ones.
// Integrator reading R#3: 4th-order Hermite P(EC)^1 with shared dt and the
// Makino-Aarseth a2/a3 corrector:
//   xp = x + v dt + a0 dt^2/2 + j0 dt^3/6,  vp = v + a0 dt + j0 dt^2/2
//   a2 = (-6 (a0 - a1) - dt (4 j0 + 2 j1)) / dt^2
//   a3 = (12 (a0 - a1) + 6 dt (j0 + j1)) / dt^3
//   x  = xp + a2 dt^4/24 + a3 dt^5/120,  v = vp + a2 dt^3/6 + a3 dt^4/24
// All kernels are HBM-bound grid-stride loops over the local particles;
// SoA fp64 rows give coalesced 8-byte accesses, packets are 2 x 16-byte
// stores per particle.
#include "internal.h"

#include <algorithm>

#include <math.h>



namespace nb {

namespace {

constexpr int kBlock = 256;

__device__ __forceinline__ void flag_bad(unsigned long long* bad, int64_t ig) {
    atomicMin(bad, (unsigned long long)ig);
}

__device__ __forceinline__ int64_t ticks_of(const StateArgs& a, int k) {
    return (int64_t)1 << (a.kmax - k);
}

__device__ __forceinline__ double dt_of(const StateArgs& a, int k) { return ldexp(a.dt, -k); }

// state of active particle i the corrector reads (loaded before the fold's partials)
struct CorrIn {
    double a0[3], j0[3], xp[3], vp[3];
};
__device__ __forceinline__ void load_corr_in(const StateArgs& a, int i, CorrIn& in) {
    for (int c = 0; c < 3; ++c) {
        const int64_t o = c * a.n_loc_pad + i;
        in.a0[c] = a.a0[o]; in.j0[c] = a.j0[o]; in.xp[c] = a.xp[o]; in.vp[c] = a.vp[o];
    }
}

// One component c of the block corrector for active particle i after the fold: Hermite
// corrector with dt_i (R#3), a0 <- a1, j0 <- j1; returns the four squares the Aarseth
// criterion sums.  Products and sums of the criterion are explicitly rounded (no FMA
// contraction), so the serial form (correct_slot) and the warp form (one lane per
// component, block_correct_kernel) give the same bits.
__device__ __forceinline__ bool correct_comp(const StateArgs& a, int i, int c, double dt, double a0, double j0,
                                             double xp, double vp, double a1, double j1, double sq[4]) {
    const double dt2 = dt * dt, dt3 = dt2 * dt, dt4 = dt3 * dt, dt5 = dt4 * dt;
    const int64_t o = c * a.n_loc_pad + i;
    const double a2 = (-6.0 * (a0 - a1) - dt * (4.0 * j0 + 2.0 * j1)) / dt2;
    const double a3 = (12.0 * (a0 - a1) + 6.0 * dt * (j0 + j1)) / dt3;
    const double x = xp + a2 * dt4 / 24.0 + a3 * dt5 / 120.0;
    const double v = vp + a2 * dt3 / 6.0 + a3 * dt4 / 24.0;
    a.x[o] = x;
    a.v[o] = v;
    a.a0[o] = a1;
    a.j0[o] = j1;
    const double a2t = a2 + dt * a3;   // a^(2) at t_next
    sq[0] = __dmul_rn(a1, a1); sq[1] = __dmul_rn(j1, j1);
    sq[2] = __dmul_rn(a2t, a2t); sq[3] = __dmul_rn(a3, a3);
    return isfinite(x) && isfinite(v) && isfinite(a1) && isfinite(j1);
}

// the Aarseth criterion from the summed squares and the new level (R#28)
__device__ __forceinline__ void correct_finish(const StateArgs& a, int i, int k, double dt, const double s[4],
                                               bool ok, unsigned long long tn) {
    if (!ok) flag_bad(a.bad, a.i_base + i);
    const double na1 = sqrt(s[0]), nj1 = sqrt(s[1]), na2 = sqrt(s[2]), na3 = sqrt(s[3]);
    const double den = nj1 * na3 + na2 * na2;
    const double dtc = den > 0.0 ? sqrt(a.eta * (na1 * na2 + nj1 * nj1) / den) : INFINITY;
    int kn = k;
    if (dtc < dt) {
        while (kn < a.kmax && dt_of(a, kn) > dtc) ++kn;
    } else if (k > 0 && dtc >= 2.0 * dt && tn % (2ull * (unsigned long long)ticks_of(a, k)) == 0) {
        kn = k - 1;
    }
    if (kn != k) {
        atomicSub(a.lvl_cnt + k, 1);
        atomicAdd(a.lvl_cnt + kn, 1);
    }
    a.lev[i] = kn;
    a.T[i] = (int64_t)tn;
}

// one active slot of the corrector after the fold, serially over the components
__device__ __forceinline__ void correct_slot(const StateArgs& a, int i, const CorrIn& in, const double f[6],
                                             unsigned long long tn) {
    const int k = a.lev[i];
    NB_CHECK(k >= 0 && k <= a.kmax && a.T[i] >= 0);
    const double dt = dt_of(a, k);
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    bool ok = true;
    for (int c = 0; c < 3; ++c) {
        double sq[4];
        ok = correct_comp(a, i, c, dt, in.a0[c], in.j0[c], in.xp[c], in.vp[c], f[c], f[3 + c], sq) && ok;
        for (int q = 0; q < 4; ++q) s[q] = __dadd_rn(s[q], sq[q]);
    }
    correct_finish(a, i, k, dt, s, ok, tn);
}

// fp64 -> fp32 RNE packet (R#18); with hi/lo (NEXT f2) also the fp32 tail
// lo = RNE(x - hi), so hi + lo carries ~48 bits of the fp64 position.
__device__ __forceinline__ void store_packet(const StateArgs& a, int64_t k, const double x[3],
                                             const double v[3], double gm) {
    const float px = __double2float_rn(x[0]), py = __double2float_rn(x[1]);
    const float pz = __double2float_rn(x[2]), pm = __double2float_rn(gm);
    const float qx = __double2float_rn(v[0]), qy = __double2float_rn(v[1]);
    const float qz = __double2float_rn(v[2]);
    a.pkt[k] = make_jpkt(px, py, pz, pm, qx, qy, qz, a.eps2);
    if (a.pklo)
        a.pklo[k] = make_float4(__double2float_rn(x[0] - (double)px),
                                __double2float_rn(x[1] - (double)py),
                                __double2float_rn(x[2] - (double)pz), 0.f);
}

__global__ void pack_state_kernel(StateArgs a) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n_loc; i += gridDim.x * blockDim.x) {
        double x[3], v[3];
        for (int c = 0; c < 3; ++c) {
            x[c] = a.x[c * a.n_loc_pad + i];
            v[c] = a.v[c * a.n_loc_pad + i];
        }
        store_packet(a, a.i_base + i, x, v, a.G * a.m[i]);
    }
}

// Hermite (R#3): Taylor predictor.  Leapfrog (NEXT f1): the kick + drift half
// of kick-drift-kick, vp = v + a dt/2 (the half-step velocity), xp = x + vp dt.
__device__ __forceinline__ void predict(const StateArgs& a, int i, const double x[3],
                                        const double v[3], const double ac[3],
                                        const double jk[3], double m) {
    const double dt = a.dt, dt2 = dt * dt, dt3 = dt2 * dt;
    double xp[3], vp[3];
    bool ok = true;
    for (int c = 0; c < 3; ++c) {
        if (a.integrator == 0) {
            xp[c] = x[c] + v[c] * dt + ac[c] * dt2 / 2.0 + jk[c] * dt3 / 6.0;
            vp[c] = v[c] + ac[c] * dt + jk[c] * dt2 / 2.0;
        } else {
            vp[c] = v[c] + ac[c] * dt / 2.0;
            xp[c] = x[c] + vp[c] * dt;
        }
        a.xp[c * a.n_loc_pad + i] = xp[c];
        a.vp[c * a.n_loc_pad + i] = vp[c];
        ok = ok && isfinite(xp[c]) && isfinite(vp[c]);
    }
    if (!ok) flag_bad(a.bad, a.i_base + i);
    store_packet(a, a.i_base + i, xp, vp, a.G * m);
}

__global__ void predict_pack_kernel(StateArgs a) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n_loc; i += gridDim.x * blockDim.x) {
        double x[3], v[3], ac[3], jk[3];
        for (int c = 0; c < 3; ++c) {
            x[c] = a.x[c * a.n_loc_pad + i];
            v[c] = a.v[c * a.n_loc_pad + i];
            ac[c] = a.a0[c * a.n_loc_pad + i];
            jk[c] = a.j0[c * a.n_loc_pad + i];
        }
        predict(a, i, x, v, ac, jk, a.m[i]);
    }
}


// canonical fold of column i of the chunk partials: per component an ascending-chunk fp64
// left fold from +0 (the order every path shares), all ncomp components at once with the components' loads interleaved so that 4 chunks x ncomp
// independent loads are in flight (the fold is load-latency bound when few columns are
// folded, e.g. a small block-step active set)
__device__ __forceinline__ void fold_all(const StateArgs& a, int i, double out[6]) {
    const double* p = a.partial + i;
    const int64_t row = a.n_loc_pad, stride = (int64_t)a.ncomp * a.n_loc_pad;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0, s4 = 0.0, s5 = 0.0;
    if (a.ncomp == 6) {
#pragma unroll 4
        for (int c = 0; c < a.n_chunks; ++c) {
            const double* q = p + c * stride;
            s0 += q[0]; s1 += q[row]; s2 += q[2 * row];
            s3 += q[3 * row]; s4 += q[4 * row]; s5 += q[5 * row];
        }
    } else {
#pragma unroll 4
        for (int c = 0; c < a.n_chunks; ++c) {
            const double* q = p + c * stride;
            s0 += q[0]; s1 += q[row]; s2 += q[2 * row];
        }
    }
    out[0] = s0; out[1] = s1; out[2] = s2; out[3] = s3; out[4] = s4; out[5] = s5;
}

__global__ void fold_forces_kernel(StateArgs a) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n_loc; i += gridDim.x * blockDim.x) {
        bool ok = true;
        double f[6];
        fold_all(a, i, f);
        for (int c = 0; c < 3; ++c) {
            const double ac = f[c], jk = f[3 + c];
            a.a0[c * a.n_loc_pad + i] = ac;
            a.j0[c * a.n_loc_pad + i] = jk;
            ok = ok && isfinite(ac) && isfinite(jk);
        }
        if (!ok) flag_bad(a.bad, a.i_base + i);
    }
}

// kEarly: all state loads before the fold -- best when the pass is latency-bound (small
// n); with many particles the extra live registers cost the fold's memory parallelism,
// so large passes load the state after the fold (both before any store)
template <bool kEarly>
__global__ void correct_predict_pack_kernel(StateArgs a) {
    const double dt = a.dt, dt2 = dt * dt, dt3 = dt2 * dt, dt4 = dt3 * dt, dt5 = dt4 * dt;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n_loc; i += gridDim.x * blockDim.x) {
        double x[3], v[3], a1[3], j1[3], f[6], a0[3], j0[3], xp[3], vp[3];
        bool ok = true;
        // state loads before any store: at small N this pass is bound by dependent load
        // round trips, and the stores below would keep the compiler from hoisting them
        if (!kEarly) fold_all(a, i, f);
        for (int c = 0; c < 3; ++c) {
            const int64_t o = c * a.n_loc_pad + i;
            a0[c] = a.a0[o]; j0[c] = a.j0[o]; xp[c] = a.xp[o]; vp[c] = a.vp[o];
        }
        const double mi = a.m[i];
        if (kEarly) fold_all(a, i, f);
        for (int c = 0; c < 3; ++c) {
            const int64_t o = c * a.n_loc_pad + i;
            a1[c] = f[c];
            j1[c] = f[3 + c];
            if (a.integrator == 0) {   // Hermite corrector (R#3)
                const double a2 = (-6.0 * (a0[c] - a1[c]) - dt * (4.0 * j0[c] + 2.0 * j1[c])) / dt2;
                const double a3 = (12.0 * (a0[c] - a1[c]) + 6.0 * dt * (j0[c] + j1[c])) / dt3;
                x[c] = xp[c] + a2 * dt4 / 24.0 + a3 * dt5 / 120.0;
                v[c] = vp[c] + a2 * dt3 / 6.0 + a3 * dt4 / 24.0;
            } else {                   // leapfrog: closing kick
                x[c] = xp[c];
                v[c] = vp[c] + a1[c] * dt / 2.0;
            }
            a.x[o] = x[c];
            a.v[o] = v[c];
            a.a0[o] = a1[c];
            a.j0[o] = j1[c];
            ok = ok && isfinite(x[c]) && isfinite(v[c]) && isfinite(a1[c]) && isfinite(j1[c]);
        }
        if (!ok) flag_bad(a.bad, a.i_base + i);
        predict(a, i, x, v, a1, j1, mi);
    }
}

__global__ void fill_padding_kernel(JPkt* pkt, float4* pklo, int64_t from, int64_t to, float eps2) {
    for (int64_t k = from + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < to;
         k += (int64_t)gridDim.x * blockDim.x) {
        // zero mass far away: contributes exactly 0 (padding)
        pkt[k] = make_jpkt(1e18f, 1e18f, 1e18f, 0.f, 0.f, 0.f, 0.f, eps2);
        if (pklo) pklo[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

__global__ void validate_kernel(StateArgs a, unsigned long long* bad2) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n_loc; i += gridDim.x * blockDim.x) {
        const double mi = a.m[i];
        if (!(isfinite(mi) && mi > 0.0)) flag_bad(&bad2[0], a.i_base + i);
        else atomicMax(&bad2[2], (unsigned long long)__double_as_longlong(mi));   // max mass (> 0: bits order)
        bool ok = true;
        for (int c = 0; c < 3; ++c)
            ok = ok && isfinite(a.x[c * a.n_loc_pad + i]) && isfinite(a.v[c * a.n_loc_pad + i]);
        if (!ok) flag_bad(&bad2[1], a.i_base + i);
    }
}

__global__ void validate_derivs_kernel(StateArgs a, unsigned long long* bad2) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n_loc; i += gridDim.x * blockDim.x) {
        bool ok = true;
        for (int c = 0; c < 3; ++c)
            ok = ok && isfinite(a.a0[c * a.n_loc_pad + i]) && (a.ncomp != 6 || isfinite(a.j0[c * a.n_loc_pad + i]));
        if (!ok) flag_bad(&bad2[1], a.i_base + i);
    }
}
__global__ void validate_levels_kernel(StateArgs a, unsigned long long* bad2) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n_loc; i += gridDim.x * blockDim.x)
        if (a.lev[i] < 0 || a.lev[i] > a.kmax) flag_bad(&bad2[1], a.i_base + i);
}

// ---------------------------------------------------------------- block time steps
// NBODY_HERMITE4_BLOCK (NEXT f4, R#28): individual steps
// dt_i = dt_max / 2^k_i; times are integer ticks of dt_max / 2^kmax, so the
// block schedule (which particles are due, commensurability for doubling)
// is exact integer arithmetic.  Only the level choice is floating point
// (the Aarseth criterion, fp64 here as in the oracle).

// Level histogram: one atomic per distinct level in the warp.
__device__ __forceinline__ void count_level(int32_t* cnt, int k) {
    const unsigned act = __activemask();
    const unsigned peers = __match_any_sync(act, k);
    if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(cnt + k, __popc(peers));
}

// t_next after block time t (ticks) = the next multiple of the finest occupied level's
// step.  Equal to min_i (T_i + dt_i) because every particle at level k was last active
// at the last multiple of its dt_k (levels start at T = 0, halve at any of their own
// step times, and double only at multiples of the doubled step, R#28), and the steps
// are nested powers of two.  ~0 when no particle is counted (an empty rank).
// Called by a whole warp: each lane loads two counters (kmax <= 50), so the finest
// occupied level costs one L2 round trip.
__device__ __forceinline__ unsigned long long next_block_time(const int32_t* cnt, int kmax,
                                                              unsigned long long t) {
    const int lane = threadIdx.x & 31;
    const bool o0 = lane <= kmax && __ldcg(cnt + lane) > 0;
    const bool o1 = lane + 32 <= kmax && __ldcg(cnt + lane + 32) > 0;
    const unsigned b0 = __ballot_sync(0xffffffffu, o0), b1 = __ballot_sync(0xffffffffu, o1);
    const int kf = b1 ? 63 - __clz(b1) : (b0 ? 31 - __clz(b0) : -1);
    if (kf < 0) return ~0ull;
    const unsigned long long d = 1ull << (kmax - kf);
    return (t / d + 1) * d;
}

__device__ __forceinline__ double norm3(const double* p, int64_t stride, int i) {
    const double x = p[i], y = p[stride + i], z = p[2 * stride + i];
    return sqrt(x * x + y * y + z * z);
}

// startup level: largest dt_max / 2^k <= eta_s |a| / |j| (k = 0 when j = 0)
__global__ void block_init_levels_kernel(StateArgs a) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n_loc; i += gridDim.x * blockDim.x) {
        const double an = norm3(a.a0, a.n_loc_pad, i), jn = norm3(a.j0, a.n_loc_pad, i);
        const double dts = jn > 0.0 ? a.eta_s * an / jn : INFINITY;
        int k = 0;
        while (k < a.kmax && dt_of(a, k) > dts) ++k;
        a.lev[i] = k;
        a.T[i] = 0;
        count_level(a.lvl_cnt, k);
    }
}

__global__ void block_reset_time_kernel(StateArgs a) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n_loc; i += gridDim.x * blockDim.x) {
        a.T[i] = 0;
        count_level(a.lvl_cnt, a.lev[i]);
    }
}

// t_next = min_i (t_i + dt_i): exact integer minimum, so order-independent;
// one atomic per warp after a shuffle reduction

__global__ void block_begin_kernel(unsigned long long* tcur, int32_t* nact, int nshards) {
    if (threadIdx.x == 0) *tcur = 0;
    for (int q = threadIdx.x; q < nshards; q += blockDim.x) nact[q] = 0;
}

// NCCL ranks: the rank's own t_next (one warp), reduced with MIN over ranks afterwards
__global__ void block_tnext_kernel(StateArgs a) {
    const unsigned long long tn = next_block_time(a.lvl_cnt, a.kmax, *a.tcur);
    if (threadIdx.x == 0) *a.tnext = tn;
}

__global__ void block_set_tend_kernel(long long* ctl, unsigned long long t_end) {
    ctl[0] = (long long)t_end;
    ctl[3] = 0;
}

// the force node of shard q for force kind k (0 list, 1 packed tile-split, 2 scalar
// tile-split, 3 list in 1024-i CTAs)
__device__ __forceinline__ cudaGraphDeviceNode_t force_node(const BlockGraphNodes* nodes, int q, int k) {
    return k == 0 ? nodes->force[q] : k == 1 ? nodes->force_ts[q] : k == 2 ? nodes->force_ts1[q]
                                                                           : nodes->force_big[q];
}

__device__ void block_decide(long long* ctl, const unsigned long long* tnext, unsigned long long* tcur,
                             int32_t* append, int32_t* nact, int nshards, cudaGraphConditionalHandle cond,
                             BlockGraphNodes* nodes) {
    const bool done = *tnext > (unsigned long long)ctl[0];
    // freeze this block step's active counts (force passes and corrector read them) and
    // reset the selection pass's append counters for the next block step
    long long na = 0;
    for (int q = 0; q < nshards; ++q) {
        nact[q] = done ? 0 : append[q];
        append[q] = 0;
        na += nact[q];
    }
    if (!done) {
        ctl[1] += 1;
        ctl[2] += na;
    }
    ctl[3] = done ? 1 : 0;
    *tcur = *tnext;   // the clock the next selection pass starts from
    if (nodes) {   // inside the block-step graph
        for (int q = 0; q < nshards; ++q) {
            if (!nodes->force[q]) continue;   // shard without particles: no force node
            // few active particles: a tile-split kernel (same partials), else the list kernel
            // (the rule of nbody.cu block_force_kind)
            const int kind = nact[q] <= nodes->ts1_max                      ? 2
                             : (nodes->ts_ok[q] && nact[q] <= nodes->ts_max) ? 1
                             : nact[q] >= nodes->big_min[q]                  ? 3
                                                                              : 0;
            const int ipb = kind == 2   ? nodes->ts1_i_per_block
                            : kind == 1 ? nodes->ts_i_per_block
                            : kind == 3 ? nodes->big_i_per_block
                                        : nodes->i_per_block;
            const int nb = (nact[q] + ipb - 1) / ipb;
            const int want = nb > 0 ? kind : -1;
            const int cur = nodes->cur[q];
            if (cur == -2) {   // first decision after capture: every captured node is enabled
                for (int k = 0; k < 4; ++k) {
                    const cudaGraphDeviceNode_t nd = force_node(nodes, q, k);
                    if (nd) cudaGraphKernelNodeSetEnabled(nd, k == want);   // null: not captured
                }
            } else if (cur != want) {   // switch nodes only when the kind changes
                if (cur >= 0) cudaGraphKernelNodeSetEnabled(force_node(nodes, q, cur), false);
                if (want >= 0) cudaGraphKernelNodeSetEnabled(force_node(nodes, q, want), true);
            }
            // the grid only when it changes (a kind switch resets it: the other node's grid
            // may be stale)
            if (want >= 0 && (cur != want || nodes->nb[q] != nb))
                cudaGraphKernelNodeSetGridDim(force_node(nodes, q, want),
                                              dim3((unsigned)nb, (unsigned)nodes->chunks[q], 1));
            nodes->nb[q] = want >= 0 ? nb : -1;
            nodes->cur[q] = want;
        }
        cudaGraphSetConditional(cond, done ? 0u : 1u);
    }
}

__global__ void block_decide_kernel(long long* ctl, const unsigned long long* tnext,
                                    unsigned long long* tcur, int32_t* append, int32_t* nact,
                                    int nshards, cudaGraphConditionalHandle cond,
                                    BlockGraphNodes* nodes) {
    block_decide(ctl, tnext, tcur, append, nact, nshards, cond, nodes);
}

// active set {i : t_i + dt_i == t_next} (atomic append: slot order is irrelevant to the
// results, every slot's force is the same j loop) and every local particle predicted to t_next with
// its own polynomial (the predictor of predict() with dt -> D = t_next - t_i), packed for
// the exchange.  In the block step past t_end the prediction is scratch nobody reads.
// one particle of the active-set selection + prediction pass (append to *nact / ilist)
// the state one particle's selection + prediction reads, loaded ahead of t_next
struct SelIn {
    double x[3], v[3], ac[3], jk[3], m;
    int64_t T;
    int32_t lev;
};
__device__ __forceinline__ void load_sel_in(const StateArgs& a, int i, SelIn& in) {
    for (int c = 0; c < 3; ++c) {
        const int64_t o = c * a.n_loc_pad + i;
        in.x[c] = a.x[o]; in.v[c] = a.v[o]; in.ac[c] = a.a0[o]; in.jk[c] = a.j0[o];
    }
    in.m = a.m[i];
    in.T = a.T[i];
    in.lev = a.lev[i];
}
__device__ __forceinline__ void select_predict_one(const StateArgs& a, int i, const SelIn& in,
                                                   unsigned long long tn, double tick, int32_t* nact) {
    NB_CHECK((unsigned long long)(in.T + ticks_of(a, in.lev)) >= tn);   // none left behind
    const bool active = (unsigned long long)(in.T + ticks_of(a, in.lev)) == tn;
    if (active) {
        const int slot = atomicAdd(nact, 1);
        NB_CHECK(slot >= 0 && slot < a.n_loc);
        a.ilist[slot] = i;
    }
    const double D = (double)(int64_t)(tn - (unsigned long long)in.T) * tick;
    const double D2 = D * D, D3 = D2 * D;
    double xp[3], vp[3];
    const double *xs = in.x, *vs = in.v, *as = in.ac, *js = in.jk;
    bool ok = true;
    for (int c = 0; c < 3; ++c) {
        const int64_t o = c * a.n_loc_pad + i;
        const double x = xs[c], v = vs[c], ac = as[c], jk = js[c];
        xp[c] = x + v * D + ac * D2 / 2.0 + jk * D3 / 6.0;
        vp[c] = v + ac * D + jk * D2 / 2.0;
        if (active) {   // only the corrector reads xp, vp, and only for active particles
            a.xp[o] = xp[c];
            a.vp[o] = vp[c];
        }
        ok = ok && isfinite(xp[c]) && isfinite(vp[c]);
    }
    if (!ok) flag_bad(a.bad, a.i_base + i);
    store_packet(a, a.i_base + i, xp, vp, a.G * in.m);
}

__global__ void block_select_predict_kernel(StateArgs a) {
    // the first particle's state is loaded before t_next (its L2 round trip overlaps them)
    const int i_first = blockIdx.x * blockDim.x + threadIdx.x;
    SelIn first;
    if (i_first < a.n_loc) load_sel_in(a, i_first, first);
    // t_next: from the level counts the previous corrector left (every CTA derives the same
    // value; CTA 0 publishes it for decide / force / corrector), or given (NCCL ranks)
    __shared__ unsigned long long tn_s;
    if (a.self_tnext) {
        if (threadIdx.x < 32) {
            const unsigned long long t = next_block_time(a.lvl_cnt, a.kmax, *a.tcur);
            if (threadIdx.x == 0) {
                tn_s = t;
                if (blockIdx.x == 0) *a.tnext = t;
            }
        }
    } else if (threadIdx.x == 0) {
        tn_s = *a.tnext;
    }
    __syncthreads();
    const unsigned long long tn = tn_s;
    const double tick = ldexp(a.dt, -a.kmax);
    if (i_first < a.n_loc) select_predict_one(a, i_first, first, tn, tick, a.nact);
    for (int i = i_first + gridDim.x * blockDim.x; i < a.n_loc; i += gridDim.x * blockDim.x) {
        SelIn in;
        load_sel_in(a, i, in);
        select_predict_one(a, i, in, tn, tick, a.nact);
    }
    if (!a.sel_done) return;
    // one shard: the last CTA to finish runs the decide step (block_decide_kernel's body)
    // -- every CTA's appends are complete and visible once it has taken its ticket
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(a.sel_done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        *a.sel_done = 0;
        block_decide(a.ctl, a.tnext, a.tcur, a.nact, a.nact_cur, 1, a.cond, a.gnodes);
    }
}

// fold of slot q's chunk partials by one warp: lane l loads chunk c0 + l of every
// component (32 chunks in flight per load round instead of one thread's serial walk) --
// the same additions, in the same order, as fold_all.  The 32 values of a round go through
// the warp's shared-memory slab red[32][6]: lane k < 6
// then adds component k's 32 values in ascending chunk order (6 active lanes, 32 LDS + 32
// DADD each, instead of 192 64-bit shuffles + 192 DADD in every lane), and the next
// round's loads are issued before this round's adds (C2 block steps 5.00 -> 4.68 ms per
// dt_max, C3 76.0 -> 74.1, interleaved A/B against the shuffle form, profiles/r02_fold_ab.jsonl).
// lane's values of the fold round starting at chunk c0 (0 past the last chunk)
__device__ __forceinline__ void fold_load(const StateArgs& a, int q, int lane, int c0, double v[6]) {
    const double* p = a.partial + q;
    const int64_t row = a.n_loc_pad, stride = (int64_t)a.ncomp * a.n_loc_pad;
    const int c = c0 + lane;
#pragma unroll
    for (int k = 0; k < 6; ++k) v[k] = c < a.n_chunks ? p[c * stride + k * row] : 0.0;
}
// v: round 0 already loaded by the caller (fold_load(a, q, lane, 0, v))
__device__ __forceinline__ void fold_warp(const StateArgs& a, int q, int lane, double v[6], double out[6],
                                          double (*red)[6]) {
    double s = 0.0;   // lane k < 6: component k
    auto load = [&](int c0) { fold_load(a, q, lane, c0, v); };
    for (int c0 = 0; c0 < a.n_chunks; c0 += 32) {
        const int cnt = min(32, a.n_chunks - c0);
#pragma unroll
        for (int k = 0; k < 6; ++k) red[lane][k] = v[k];
        __syncwarp();
        if (c0 + 32 < a.n_chunks) load(c0 + 32);   // next round in flight during the adds
        if (lane < 6)
            for (int u = 0; u < cnt; ++u) s += red[u][lane];
        __syncwarp();
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) out[k] = __shfl_sync(0xffffffffu, s, k);
}

// Active sets up to this size (and at most one slot per warp of the launch) fold one
// slot per warp (latency-bound regime), larger ones one slot per thread
// (bandwidth-bound); the results are identical.
constexpr int kWarpFoldMax = 4096;

__global__ void block_correct_kernel(StateArgs a) {
    const int32_t n_act = *a.nact_cur;
    const unsigned long long tn = *a.tnext;
    const int nw = (int)((gridDim.x * blockDim.x) >> 5);
    if (n_act <= min(kWarpFoldMax, nw) && a.ncomp == 6) {   // at most one slot per warp
        __shared__ double red[kBlock / 32][32][6];   // one fold slab per warp
        const int lane = threadIdx.x & 31;
        for (int q = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); q < n_act; q += nw) {
            // the fold's first round does not depend on the slot's particle: its loads are
            // issued with the active-list read, the state loads after it
            double v[6];
            fold_load(a, q, lane, 0, v);
            const int i = a.ilist[q];
            NB_CHECK(q < a.n_loc && i >= 0 && i < a.n_loc);
            const int cc = lane < 3 ? lane : 0;
            const int64_t o = cc * a.n_loc_pad + i;
            const double a0 = a.a0[o], j0 = a.j0[o], xp = a.xp[o], vp = a.vp[o];
            const int k = a.lev[i];
            double f[6];
            fold_warp(a, q, lane, v, f, red[threadIdx.x >> 5]);
            // corrector: one lane per component, lane 0 sums the criterion's squares in
            // component order and sets the level (the arithmetic of correct_slot)
            const double dt = dt_of(a, k);
            double sq[4] = {0.0, 0.0, 0.0, 0.0};
            bool ok = true;
            if (lane < 3) ok = correct_comp(a, i, lane, dt, a0, j0, xp, vp, f[lane], f[3 + lane], sq);
            const bool all_ok = __all_sync(0xffffffffu, ok);
            double s4[4] = {0.0, 0.0, 0.0, 0.0};
            for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int r = 0; r < 4; ++r) s4[r] = __dadd_rn(s4[r], __shfl_sync(0xffffffffu, sq[r], c));
            if (lane == 0) {
                NB_CHECK(k >= 0 && k <= a.kmax && a.T[i] >= 0);
                correct_finish(a, i, k, dt, s4, all_ok, tn);
            }
        }
    } else {
        for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n_act; q += gridDim.x * blockDim.x) {
            const int i = a.ilist[q];
            NB_CHECK(q < a.n_loc && i >= 0 && i < a.n_loc);
            CorrIn in;
            load_corr_in(a, i, in);   // loads first (see correct_predict_pack_kernel)
            double f[6];
            fold_all(a, q, f);
            correct_slot(a, i, in, f, tn);
        }
    }
}


// launch shape of an O(n) grid-stride pass: 256-thread CTAs, or for small n fewer
// threads per CTA (a multiple of 32) so that the pass still spreads over ~148 SMs --
// at N ~ 1 000 these passes are bound by dependent load latency, not bandwidth
struct Dims {
    unsigned grid, block;
};
Dims dims_for(int64_t n) {
    if (n < 1) n = 1;
    int64_t block = kBlock;
    if (n < 148LL * kBlock) block = std::max<int64_t>(32, (n + 148 * 32 - 1) / (148 * 32) * 32);
    int64_t g = (n + block - 1) / block;
    if (g > 148 * 16) g = 148 * 16;
    return Dims{(unsigned)g, (unsigned)block};
}

}  // namespace

cudaError_t launch_validate(const StateArgs& a, unsigned long long* bad2, cudaStream_t s) {
    if (a.n_loc <= 0) return cudaSuccess;
    validate_kernel<<<dims_for(a.n_loc).grid, dims_for(a.n_loc).block, 0, s>>>(a, bad2);
    return cudaGetLastError();
}
cudaError_t launch_validate_derivs(const StateArgs& a, unsigned long long* bad2, cudaStream_t s) {
    if (a.n_loc <= 0) return cudaSuccess;
    validate_derivs_kernel<<<dims_for(a.n_loc).grid, dims_for(a.n_loc).block, 0, s>>>(a, bad2);
    return cudaGetLastError();
}
cudaError_t launch_validate_levels(const StateArgs& a, unsigned long long* bad2, cudaStream_t s) {
    if (a.n_loc <= 0) return cudaSuccess;
    validate_levels_kernel<<<dims_for(a.n_loc).grid, dims_for(a.n_loc).block, 0, s>>>(a, bad2);
    return cudaGetLastError();
}
cudaError_t launch_pack_state(const StateArgs& a, cudaStream_t s) {
    if (a.n_loc <= 0) return cudaSuccess;
    pack_state_kernel<<<dims_for(a.n_loc).grid, dims_for(a.n_loc).block, 0, s>>>(a);
    return cudaGetLastError();
}
cudaError_t launch_predict_pack(const StateArgs& a, cudaStream_t s) {
    if (a.n_loc <= 0) return cudaSuccess;
    predict_pack_kernel<<<dims_for(a.n_loc).grid, dims_for(a.n_loc).block, 0, s>>>(a);
    return cudaGetLastError();
}
cudaError_t launch_fold_forces(const StateArgs& a, cudaStream_t s) {
    if (a.n_loc <= 0) return cudaSuccess;
    fold_forces_kernel<<<dims_for(a.n_loc).grid, dims_for(a.n_loc).block, 0, s>>>(a);
    return cudaGetLastError();
}
cudaError_t launch_correct_predict_pack(const StateArgs& a, cudaStream_t s) {
    if (a.n_loc <= 0) return cudaSuccess;
    if (a.n_loc < 148 * kBlock)
        correct_predict_pack_kernel<true><<<dims_for(a.n_loc).grid, dims_for(a.n_loc).block, 0, s>>>(a);
    else
        correct_predict_pack_kernel<false><<<dims_for(a.n_loc).grid, dims_for(a.n_loc).block, 0, s>>>(a);
    return cudaGetLastError();
}
cudaError_t launch_block_init_levels(const StateArgs& a, cudaStream_t s) {
    if (a.n_loc <= 0) return cudaSuccess;
    block_init_levels_kernel<<<dims_for(a.n_loc).grid, dims_for(a.n_loc).block, 0, s>>>(a);
    return cudaGetLastError();
}
cudaError_t launch_block_reset_time(const StateArgs& a, cudaStream_t s) {
    if (a.n_loc <= 0) return cudaSuccess;
    block_reset_time_kernel<<<dims_for(a.n_loc).grid, dims_for(a.n_loc).block, 0, s>>>(a);
    return cudaGetLastError();
}
cudaError_t launch_block_select_predict(const StateArgs& a, cudaStream_t s) {
    // a rank that owns no particles still runs the fused decide step (one CTA, no particles)
    if (a.n_loc <= 0 && !a.sel_done) return cudaSuccess;
    const Dims d = dims_for(a.n_loc > 0 ? a.n_loc : 1);
    block_select_predict_kernel<<<d.grid, d.block, 0, s>>>(a);
    return cudaGetLastError();
}
cudaError_t launch_block_correct(const StateArgs& a, cudaStream_t s) {
    block_correct_kernel<<<dims_for(a.n_loc > 0 ? a.n_loc : 1).grid, dims_for(a.n_loc > 0 ? a.n_loc : 1).block, 0,
                           s>>>(a);
    return cudaGetLastError();
}
cudaError_t launch_block_begin(unsigned long long* tcur, int32_t* nact, int nshards, cudaStream_t s) {
    block_begin_kernel<<<1, 32, 0, s>>>(tcur, nact, nshards);
    return cudaGetLastError();
}
cudaError_t launch_block_tnext(const StateArgs& a, cudaStream_t s) {
    block_tnext_kernel<<<1, 32, 0, s>>>(a);
    return cudaGetLastError();
}
cudaError_t launch_block_set_tend(long long* ctl, unsigned long long t_end, cudaStream_t s) {
    block_set_tend_kernel<<<1, 1, 0, s>>>(ctl, t_end);
    return cudaGetLastError();
}
cudaError_t launch_block_decide(long long* ctl, const unsigned long long* tnext, unsigned long long* tcur,
                                int32_t* nact, int32_t* nact_cur, int nshards,
                                cudaGraphConditionalHandle cond, BlockGraphNodes* nodes, cudaStream_t s) {
    block_decide_kernel<<<1, 1, 0, s>>>(ctl, tnext, tcur, nact, nact_cur, nshards, cond, nodes);
    return cudaGetLastError();
}
cudaError_t launch_fill_padding(JPkt* pkt, float4* pklo, int64_t from, int64_t to, float eps2, cudaStream_t s) {
    if (to <= from) return cudaSuccess;
    fill_padding_kernel<<<dims_for(to - from).grid, dims_for(to - from).block, 0, s>>>(pkt, pklo, from, to, eps2);
    return cudaGetLastError();
}

}  // namespace nb
