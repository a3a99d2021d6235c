// internal.h -- shared declarations of the libnbody kernels and runtime.
// Product code only; nothing here is shared with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// NB_DEBUG_CHECKS=1 (debug builds only; tests/test_gpu_debug_checks.py): device-side bounds
// asserts on every index the block-step and force kernels derive from device data.  The
// pool this was built on has no compute-sanitizer, so these stand in for memcheck.
#ifndef NB_DEBUG_CHECKS
#define NB_DEBUG_CHECKS 0
#endif
#if NB_DEBUG_CHECKS
#include <cassert>
#define NB_CHECK(cond) assert(cond)
#else
#define NB_CHECK(cond) ((void)0)
#endif

namespace nb {

// j-particle packet, the B200 replacement of the paper's replicated 32x32
// tiles.  Two layouts (compile-time NB_PKT_DUP):
//  1: 64 B, every scalar stored twice so the force loop reads each j operand
//     as a {lo, hi} register pair (FFMA2/FADD2/FMUL2 with a broadcast .F32
//     scalar operand run ~30% slower in isolation, scripts/ubench_fp32.cu);
//  0: 32 B, (x, y, z, G m) (vx, vy, vz, eps2); j operands broadcast.
// The spare lane carries the softening eps2 = fp32(eps^2).
#ifndef NB_PKT_DUP
#define NB_PKT_DUP 0
#endif
#if NB_PKT_DUP
struct __align__(16) JPkt {
    float4 a;  // x, x, y, y        (fp32, RNE from fp64 state)
    float4 b;  // z, z, Gm, Gm
    float4 c;  // vx, vx, vy, vy
    float4 d;  // vz, vz, eps2, eps2
};
__device__ __forceinline__ JPkt make_jpkt(float x, float y, float z, float gm, float vx, float vy,
                                          float vz, float eps2) {
    JPkt k;
    k.a = make_float4(x, x, y, y);
    k.b = make_float4(z, z, gm, gm);
    k.c = make_float4(vx, vx, vy, vy);
    k.d = make_float4(vz, vz, eps2, eps2);
    return k;
}
__device__ __forceinline__ float4 jpkt_pos(const JPkt& k) { return make_float4(k.a.x, k.a.z, k.b.x, k.b.z); }
__device__ __forceinline__ float4 jpkt_vel(const JPkt& k) { return make_float4(k.c.x, k.c.z, k.d.x, k.d.z); }
#else
struct __align__(16) JPkt {
    float4 p;  // x, y, z, G m      (fp32, RNE from fp64 state)
    float4 v;  // vx, vy, vz, eps2
};
__device__ __forceinline__ JPkt make_jpkt(float x, float y, float z, float gm, float vx, float vy,
                                          float vz, float eps2) {
    JPkt k;
    k.p = make_float4(x, y, z, gm);
    k.v = make_float4(vx, vy, vz, eps2);
    return k;
}
__device__ __forceinline__ float4 jpkt_pos(const JPkt& k) { return k.p; }   // w = G m
__device__ __forceinline__ float4 jpkt_vel(const JPkt& k) { return k.v; }   // w = eps2
#endif

constexpr int kTile = 256;  // j per fp32 partial-sum tile (R#10)

// Force pass arguments.  One CTA = (i-block, chunk); see force.cu.
struct ForceArgs {
    const JPkt* pkt;     // all-gathered j packets [L]
    const float4* pklo;  // NEXT f2 hi/lo: fp32(x - fp32(x)) tails [L], or nullptr
    int64_t i_base;      // global index of local particle 0
    int32_t n_loc;       // local particles
    int64_t n_loc_pad;   // row stride of `partial`
    int32_t chunk;       // j per chunk (multiple of kTile)
    int32_t n_chunks;    // chunks in the canonical order
    int32_t c_first;     // first chunk of this launch
    int32_t c_count;     // chunks in this launch (grid.y)
    float eps2;          // fp32(eps^2)
    double* partial;     // [n_chunks][ncomp][n_loc_pad] (acc x,y,z [, jerk x,y,z])
    unsigned long long* coincident;  // eps == 0 only: min global i of a coincident pair
    const int32_t* ilist;  // block steps: local index of the particle in i-slot il, or nullptr
                           // (slot il is particle il); partial rows are indexed by slot
    const int32_t* n_dev;  // with ilist: the active count on the device; n_loc then only sizes
                           // the grid (host count, or a placeholder the decide kernel rewrites)
};

// Launches the force pass for chunks c_first .. c_first + c_count - 1 (mod
// n_chunks) over all local i; jerk == false is the acceleration-only kernel
// (leapfrog, NEXT f1; partial has 3 components).  Returns the launch error.
cudaError_t launch_force(const ForceArgs& a, bool guard_self, bool jerk, cudaStream_t s);
// The same pass pinned to the 1024-i CTA shape (the exchange-overlap launch, sized in
// whole waves of that shape by the runtime).
cudaError_t launch_force_big(const ForceArgs& a, bool guard_self, bool jerk, cudaStream_t s);
int force_i_per_block();
int force_list_i_per_block(bool big);   // i per CTA of the active-list (block-step) force launches
// Active-list force pass in the 256-i (big = false) or the 1024-i CTA shape (large active
// sets: the big shape is ~2.5 % faster per interaction once it fills >= 2 waves).
cudaError_t launch_force_list(const ForceArgs& a, bool guard_self, bool big, cudaStream_t s);
// Tile-split force pass (few i: block steps with small active sets, N ~ 1 000): same
// partials, bit for bit, as launch_force; CTA = (64 i packed or 32 i scalar, chunk), one
// warp per j-tile.  With ilist (needs n_dev, jerk) packed or scalar; plain launches
// scalar only (launch_force picks it for latency-bound sizes).
cudaError_t launch_force_tsplit(const ForceArgs& a, bool guard_self, bool jerk, bool scalar, cudaStream_t s);
int force_tsplit_i_per_block(bool scalar);
int force_tsplit_threads(int chunk);
int force_tsplit_max();         // block steps: largest active count for the packed tile-split kernel
int force_tsplit1_max();        // ... and for the scalar one
// resident force CTAs per SM for the kernel variant (occupancy calculator)
int force_ctas_per_sm(bool jerk, bool hilo);

struct BlockGraphNodes;

// fp64 particle-update kernels (hermite.cu).
struct StateArgs {
    int32_t n_loc;
    int64_t n_loc_pad;   // row stride of x, v, a0, j0, xp, vp, partial
    int64_t i_base;      // global index of local particle 0
    double G, dt;
    float eps2;          // fp32(eps^2), written into the packets' spare lanes
    const double* m;     // [n_loc]
    double *x, *v, *a0, *j0, *xp, *vp;  // [3][n_loc_pad]
    const double* partial;  // [n_chunks][ncomp][n_loc_pad]
    int32_t n_chunks;
    int32_t ncomp;       // 6 (Hermite: acc + jerk) or 3 (leapfrog: acc)
    int32_t integrator;  // NBODY_HERMITE4 (0) or NBODY_LEAPFROG_KDK (1)
    JPkt* pkt;           // all packets; local particle i goes to pkt[i_base + i]
    float4* pklo;        // hi/lo position tails (nullptr unless hilo)
    unsigned long long* bad;  // min global index of a non-finite particle
    // block time steps (NBODY_HERMITE4_BLOCK, R#28); dt above is dt_max
    int64_t* T;          // [n_loc] particle time in ticks of dt_max / 2^kmax
    int32_t* lev;        // [n_loc] level k: dt_i = dt_max / 2^k
    int32_t* ilist;      // [n_loc] active particles (local indices), slot order
    int32_t* nact;       // active-set append counter of the selection pass (device)
    int32_t* nact_cur;   // this block step's active count, frozen by the decide kernel
    unsigned long long* tnext;  // this block step's time in ticks (device, shared by shards)
    unsigned long long* tcur;   // the previous block step's time (the clock the levels refer to)
    int32_t self_tnext;  // 1: the selection pass derives t_next from the level counts itself;
                         // 0: t_next is already in *tnext (NCCL ranks: a min over ranks)
    int32_t* lvl_cnt;    // [64] particles per level, all shards (device); t_next derives from it
    long long* ctl;      // block-run control [t_end ticks, block steps, sum of active, done]
    int32_t kmax;
    double eta, eta_s;
    // one shard: the selection pass's last CTA also runs the decide step (no separate
    // decide launch); sel_done is its CTA counter (device, zero between launches), cond /
    // gnodes the block-step graph's conditional handle and force-node table (graph only)
    unsigned* sel_done;
    cudaGraphConditionalHandle cond;
    BlockGraphNodes* gnodes;
};
cudaError_t launch_pack_state(const StateArgs& a, cudaStream_t s);     // x, v -> pkt
cudaError_t launch_predict_pack(const StateArgs& a, cudaStream_t s);   // x,v,a0,j0 -> xp,vp,pkt
cudaError_t launch_fold_forces(const StateArgs& a, cudaStream_t s);    // partial -> a0, j0
cudaError_t launch_correct_predict_pack(const StateArgs& a, cudaStream_t s);
cudaError_t launch_fill_padding(JPkt* pkt, float4* pklo, int64_t from, int64_t to, float eps2,
                                cudaStream_t s);
// bad2[0]: min global index with m not finite or <= 0; bad2[1]: x or v not finite;
// bad2[2]: atomicMax of the valid masses' bit patterns (caller zeroes it first)
cudaError_t launch_validate(const StateArgs& a, unsigned long long* bad2, cudaStream_t s);
// checkpoint restore: a0, j0 finite (bad2[1] = first bad global index); levels in [0, kmax]
cudaError_t launch_validate_derivs(const StateArgs& a, unsigned long long* bad2, cudaStream_t s);
cudaError_t launch_validate_levels(const StateArgs& a, unsigned long long* bad2, cudaStream_t s);

// fp64 energy (energy.cu).  eall: [L] (x, y, z, m) of every particle.
cudaError_t launch_energy_pack(const StateArgs& a, double4* eall, cudaStream_t s);
cudaError_t launch_energy(const double4* eall, int64_t n, int64_t i_base,
                          int32_t n_loc, const double* v, int64_t n_loc_pad,
                          const double* m, double eps2, double* block_sums,
                          int nblocks_max, double* out2, cudaStream_t s);
int energy_blocks(int32_t n_loc);

// block time steps (hermite.cu, R#28)
// Both add every local particle's level to lvl_cnt (zeroed by the caller first).
cudaError_t launch_block_init_levels(const StateArgs& a, cudaStream_t s);  // lev from eta_s, T = 0
cudaError_t launch_block_reset_time(const StateArgs& a, cudaStream_t s);   // T = 0 (call start)
// start of a call: clock at 0 (tcur), append counters of all nshards shards reset
cudaError_t launch_block_begin(unsigned long long* tcur, int32_t* nact, int nshards, cudaStream_t s);
// NCCL ranks: this rank's t_next from its level counts into *tnext (then a min over ranks)
cudaError_t launch_block_tnext(const StateArgs& a, cudaStream_t s);
// ctl[0] = t_end (start of a call)
cudaError_t launch_block_set_tend(long long* ctl, unsigned long long t_end, cudaStream_t s);
// after t_next and the active sets: done = t_next > t_end (then the active counts are zeroed so
// the rest of the block step is a no-op), statistics, and -- inside the block-step CUDA graph
// -- the WHILE-loop condition and the grid (ceil(nact / i_per_block), chunks[q]) of every
// shard's device-updatable force node (disabled when its active set is empty)
struct BlockGraphNodes {
    cudaGraphDeviceNode_t force[8];      // per shard (loopback shards <= 8 use the graph)
    cudaGraphDeviceNode_t force_big[8];  // the same list pass in the 1024-i CTA shape
    int32_t big_min[8];                  // active counts >= big_min take force_big
    cudaGraphDeviceNode_t force_ts[8];   // packed tile-split launch of the same shard (if ts_ok)
    cudaGraphDeviceNode_t force_ts1[8];  // scalar tile-split launch (if ts1_max > 0)
    int32_t chunks[8];
    int32_t ts_ok[8];                    // chunk has >= 2 tiles: packed tile-split usable
    int32_t i_per_block, big_i_per_block, ts_i_per_block, ts1_i_per_block;
    int32_t ts_max, ts1_max;             // active counts <= ts1_max: scalar; <= ts_max: packed
    int32_t cur[8];                      // enabled force node per shard (kind, -1 none, -2 unknown)
    int32_t nb[8];                       // ... and the grid x it was last given (-1 unknown)
};
cudaError_t launch_block_decide(long long* ctl, const unsigned long long* tnext, unsigned long long* tcur,
                                int32_t* nact, int32_t* nact_cur, int nshards,
                                cudaGraphConditionalHandle cond, BlockGraphNodes* nodes, cudaStream_t s);

// active set + every particle predicted to t_next and packed (one pass)
cudaError_t launch_block_select_predict(const StateArgs& a, cudaStream_t s);
// correct the active particles (count nact_cur, read on the device), new levels and level
// counts, T = t_next.  No grid-wide tail: the next selection pass derives its t_next from
// the level counts and the decide kernel resets the append counters.
cudaError_t launch_block_correct(const StateArgs& a, cudaStream_t s);

}  // namespace nb
