// force.cu -- the hot loop: softened acceleration + jerk, all i x all j,
// FP32 pair arithmetic on sm_100a packed FP32x2 (FFMA2/FADD2/FMUL2) plus
// MUFU.RSQ, j-tiles staged in shared memory by bulk TMA (cp.async.bulk)
// into an mbarrier ring.
//
// What it computes (P:134-138 [Sec. 3, force equation]; softening R#1; jerk
// R#2): for every local i and every j of the chunk
//     d = x_j - x_i, w = v_j - v_i, s = |d|^2 + eps^2
//     a_i += G m_j d / s^{3/2}
//     j_i += G m_j (w - 3 (d.w) d / s) / s^{3/2}
// in FP32 ("acceleration, jerk, and other intermediate values ... in
// single precision"), summed sequentially over the 256 j of a tile, the
// tile sums added in fp64 in ascending tile order; the fp64 chunk sum is
// written to partial[chunk][6][i].  Chunks are folded in ascending order by
// the fp64 particle-update kernels (hermite.cu), so the grouping of every
// floating-point operation is fixed by (n, chunk) alone (R#10).
//
// Mapping (B200 redesign of the paper's core/tile mapping):
//   CTA  = (i-block of kI = 2 * kPairs * kThreads particles, j-chunk)
//   thread = kPairs packed i-pairs in registers (x_i, v_i negated so every
//            difference is one FADD2 with the broadcast j operand)
//   j      = broadcast from shared memory (LDS.128 x 2 per j per thread)
//   producer = thread 0 issues cp.async.bulk of 8 KiB tiles (the paper's
//            `read` kernel + circular buffers, as TMA + mbarriers)
//   block time steps: i-slot il holds local particle ilist[il] (the active
//            set, R#28); only the i prologue and the eps = 0 report see it
#include "internal.h"

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cstdlib>
#include <cstring>
#include <cstdio>
#include <type_traits>

namespace nb {

namespace {

// Tuning knobs (defaults chosen by the sweep in scripts/sweep_force.py;
// profiles/ holds the measurements).
#ifndef FK_THREADS
#define FK_THREADS 128
#endif
#ifndef FK_PAIRS
#define FK_PAIRS 4
#endif
#ifndef FK_STAGES
#define FK_STAGES 2
#endif
#ifndef FK_MINB
#define FK_MINB 2
#endif
#ifndef FK_MINB_ACC
#define FK_MINB_ACC 2    // acceleration-only kernel (leapfrog)
#endif
#ifndef FK_UNROLL
#define FK_UNROLL 2
#endif
#ifndef FK_SMALL_UNROLL
#define FK_SMALL_UNROLL 2   // j unroll of the 256-i CTA shape
#endif
#ifndef FK_SMALL_LIST_UNROLL
#define FK_SMALL_LIST_UNROLL 4   // ... in its active-list form (profiles/r01_small_unroll.txt)
#endif
#ifndef FK_TS_UNROLL
#define FK_TS_UNROLL 4   // j unroll of the packed tile-split form (sweep: profiles/r01_tsplit_unroll.txt)
#endif
#ifndef FK_TS1_UNROLL
#define FK_TS1_UNROLL 8  // j unroll of the scalar tile-split form (sweep: profiles/r01_tsplit_unroll.txt)
#endif
#ifndef FK_ACC_SMEM
#define FK_ACC_SMEM 1
#endif

constexpr int kStages = FK_STAGES;        // smem ring depth (tiles)
constexpr int kUnroll = FK_UNROLL;
constexpr int kTsUnroll = FK_TS_UNROLL, kTs1Unroll = FK_TS1_UNROLL;
constexpr int kTileBytes = kTile * (int)sizeof(JPkt);
constexpr int kLoTileBytes = kTile * (int)sizeof(float4);   // hi/lo position tails (NEXT f2)
static_assert(kStages * 8 <= 64, "mbarrier area");

// CTA shape: P packed i-pairs per thread, T threads, MINB resident CTAs per SM
// (launch bounds).  Two shapes are instantiated: the
// default (1024 i per CTA) and a small one (256 i per CTA) for launches with
// few i -- block-step active sets and small N -- where 1024-i CTAs would leave
// most SMs idle.  Every i's j loop is identical in both, so results are too.
template <int P, int T, int MINB, int MINB_ACC, int U = FK_UNROLL, int UL = U>
struct FkCfg {
    static constexpr int kPairs = P, kThreads = T, kMinB = MINB, kMinBAcc = MINB_ACC;
    static constexpr int kUnrollJ = U, kUnrollList = UL;   // j-loop unroll: plain / active-list
    static constexpr int kIPerBlock = 2 * P * T;
    static constexpr int kAccSmemBytes = FK_ACC_SMEM ? 6 * 2 * P * T * 8 : 0;
    // shared memory: [ring: kStages j-tiles][ring_lo: kStages lo-tiles][64 B mbarriers][fp64 acc]
    static constexpr int kOffLo = kStages * kTileBytes;
    static constexpr int kOffBar = kOffLo + kStages * kLoTileBytes;
    static constexpr int kOffAcc = kOffBar + 64;
    static constexpr int kSmemBytes = kOffAcc + kAccSmemBytes;
};
using CfgBig = FkCfg<FK_PAIRS, FK_THREADS, FK_MINB, FK_MINB_ACC>;
#ifndef FK_SMALL_PAIRS
#define FK_SMALL_PAIRS 1
#endif
#ifndef FK_SMALL_THREADS
#define FK_SMALL_THREADS 128
#endif
#ifndef FK_SMALL_MINB
#define FK_SMALL_MINB 6
#endif
using CfgSmall = FkCfg<FK_SMALL_PAIRS, FK_SMALL_THREADS, FK_SMALL_MINB, FK_SMALL_MINB, FK_SMALL_UNROLL,
                       FK_SMALL_LIST_UNROLL>;
constexpr int kIPerBlock = CfgBig::kIPerBlock;

typedef unsigned long long f2;  // packed {lo, hi} fp32 pair in one 64-bit register

__device__ __forceinline__ f2 f2make(float lo, float hi) {
    f2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ f2 f2bc(float a) { return f2make(a, a); }
__device__ __forceinline__ void f2split(f2 a, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a));
}
__device__ __forceinline__ f2 fadd2(f2 a, f2 b) {
    f2 d;
    asm("add.rn.ftz.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2 fmul2(f2 a, f2 b) {
    f2 d;
    asm("mul.rn.ftz.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2 ffma2(f2 a, f2 b, f2 c) {
    f2 d;
    asm("fma.rn.ftz.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ float rsqrt_ftz(float s) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(s));
    return r;
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
    }
}
// 1-D bulk TMA global -> shared, completion counted on `bar` (UBLKCP in SASS)
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

// j operands of one interaction, broadcast to both lanes of a pair
struct JOps {
    f2 x, y, z, m, eps2, vx, vy, vz, lx, ly, lz;
    float mass;   // G m_j (eps = 0 report: padding j has mass 0)
};
// negated i state of one packed i-pair
struct IPair {
    f2 nx, ny, nz, nvx, nvy, nvz, nlx, nly, nlz;
};

// j operands of tile entry jj (shared memory), broadcast to both pair lanes
template <bool kJerk, bool kHiLo>
__device__ __forceinline__ JOps load_jops(const JPkt* tile, const float4* tile_lo, int jj) {
    JOps jo;
#if NB_PKT_DUP
    // j operands arrive as {v, v} register pairs (packet layout, internal.h)
    const ulonglong2 A = *reinterpret_cast<const ulonglong2*>(&tile[jj].a);
    const ulonglong2 B = *reinterpret_cast<const ulonglong2*>(&tile[jj].b);
    const ulonglong2 D = *reinterpret_cast<const ulonglong2*>(&tile[jj].d);
    jo.x = A.x; jo.y = A.y; jo.z = B.x; jo.m = B.y; jo.eps2 = D.y;
    jo.vx = jo.vy = jo.vz = 0ull;
    if (kJerk) {
        const ulonglong2 Cc = *reinterpret_cast<const ulonglong2*>(&tile[jj].c);
        jo.vx = Cc.x; jo.vy = Cc.y; jo.vz = D.x;
    }
    jo.mass = tile[jj].b.z;
#else
    const float4 P = tile[jj].p;
    const float4 V = tile[jj].v;
    jo.x = f2bc(P.x); jo.y = f2bc(P.y); jo.z = f2bc(P.z); jo.m = f2bc(P.w);
    jo.eps2 = f2bc(V.w);
    jo.vx = f2bc(V.x); jo.vy = f2bc(V.y); jo.vz = f2bc(V.z);
    jo.mass = P.w;
#endif
    jo.lx = jo.ly = jo.lz = 0ull;
    if (kHiLo) {
        const float4 L = tile_lo[jj];
        jo.lx = f2bc(L.x); jo.ly = f2bc(L.y); jo.lz = f2bc(L.z);
    }
    return jo;
}

struct JOps1 {
    float x, y, z, m, eps2, vx, vy, vz, lx, ly, lz;
};
struct IOne {
    float nx, ny, nz, nvx, nvy, nvz, nlx, nly, nlz;
};
template <bool kJerk, bool kHiLo>
__device__ __forceinline__ JOps1 load_jops1(const JPkt* tile, const float4* tile_lo, int jj) {
    const float4 P = jpkt_pos(tile[jj]), V = jpkt_vel(tile[jj]);
    JOps1 j{P.x, P.y, P.z, P.w, V.w, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (kJerk) { j.vx = V.x; j.vy = V.y; j.vz = V.z; }
    if (kHiLo) {
        const float4 L = tile_lo[jj];
        j.lx = L.x; j.ly = L.y; j.lz = L.z;
    }
    return j;
}

// negated i state of the particle in packet src (0 for a padding slot)
template <bool kHiLo>
__device__ __forceinline__ void load_i(const ForceArgs& a, bool valid, int64_t src, float (&q)[9]) {
    if (valid) {
        const JPkt pk = a.pkt[src];
        const float4 P = jpkt_pos(pk), V = jpkt_vel(pk);
        q[0] = -P.x; q[1] = -P.y; q[2] = -P.z;
        q[3] = -V.x; q[4] = -V.y; q[5] = -V.z;
        if (kHiLo) {
            const float4 Lo = a.pklo[src];
            q[6] = -Lo.x; q[7] = -Lo.y; q[8] = -Lo.z;
        } else {
            q[6] = q[7] = q[8] = 0.f;
        }
    } else {
#pragma unroll
        for (int k = 0; k < 9; ++k) q[k] = 0.f;
    }
}

// eps = 0, s == 0 in i-slot sl: a coincident pair unless it is the self term
// (same global index) or padding (slot past n_loc, or a massless padding j)
struct GuardCtx {   // what the eps = 0 report needs (kernel parameters, passed by value)
    const int32_t* ilist;
    int64_t i_base;
    unsigned long long* coincident;
    int n_loc;
};
template <bool kList>
__device__ __forceinline__ void report_coincident(const GuardCtx& g, int sl, int64_t jg, float jmass) {
    if (sl >= g.n_loc || jmass == 0.f) return;
    const int64_t ig = g.i_base + (kList ? g.ilist[sl] : sl);
    if (ig != jg) atomicMin(g.coincident, (unsigned long long)ig);
}

// One j against one packed i-pair: the FP32 interaction of the file header, in two
// halves.  front(): d = x_j - x_i (hi/lo: + the tails), s = |d|^2 + eps^2, ri = 1/sqrt(s)
// (MUFU.RSQ); back(): mr3 = G m_j ri^3, a += mr3 d, jerk += mr3 (w - 3 (d.w) ri^2 d).
// interact() runs both.  (A software-pipelined j loop running front() of j + 1 before
// back() of j measured 3-17 % slower, profiles/r02_sweep_force.txt.)  Every force kernel
// (all CTA shapes, the tile-split kernels) runs exactly this instruction sequence per
// lane, so their tile sums are bit-identical.  m3 = {-3, -3}.  kGuard (eps = 0): s == 0 gives ri = 0 and reports a
// coincident pair of distinct particles; sl_lo / sl_hi are the lanes' i-slots.
struct Front {
    f2 dx, dy, dz, ri;
};
template <bool kGuard, bool kHiLo, bool kList>
__device__ __forceinline__ Front front(const JOps& j, const IPair& i, int sl_lo, int sl_hi, int64_t jg,
                                       const GuardCtx& g) {
    Front f;
    f.dx = fadd2(j.x, i.nx);
    f.dy = fadd2(j.y, i.ny);
    f.dz = fadd2(j.z, i.nz);
    if (kHiLo) {   // d = (x_j^hi - x_i^hi) + (x_j^lo - x_i^lo)   (NEXT f2)
        f.dx = fadd2(f.dx, fadd2(j.lx, i.nlx));
        f.dy = fadd2(f.dy, fadd2(j.ly, i.nly));
        f.dz = fadd2(f.dz, fadd2(j.lz, i.nlz));
    }
    f2 s2 = ffma2(f.dx, f.dx, j.eps2);
    s2 = ffma2(f.dy, f.dy, s2);
    s2 = ffma2(f.dz, f.dz, s2);
    float s_lo, s_hi;
    f2split(s2, s_lo, s_hi);
    float r_lo = rsqrt_ftz(s_lo), r_hi = rsqrt_ftz(s_hi);
    if (kGuard) {  // eps == 0: exclude j == i (s == 0), R#17
        if (s_lo == 0.f) {
            r_lo = 0.f;
            report_coincident<kList>(g, sl_lo, jg, j.mass);
        }
        if (s_hi == 0.f) {
            r_hi = 0.f;
            report_coincident<kList>(g, sl_hi, jg, j.mass);
        }
    }
    f.ri = f2make(r_lo, r_hi);
    return f;
}
template <bool kJerk, int kNC, int kP>
__device__ __forceinline__ void back(const JOps& j, const IPair& i, const Front& f, f2 (&acc)[kNC][kP], int p,
                                     f2 m3) {
    const f2 ri2 = fmul2(f.ri, f.ri);
    const f2 mr3 = fmul2(fmul2(j.m, f.ri), ri2);   // G m_j / s^{3/2}
    acc[0][p] = ffma2(mr3, f.dx, acc[0][p]);
    acc[1][p] = ffma2(mr3, f.dy, acc[1][p]);
    acc[2][p] = ffma2(mr3, f.dz, acc[2][p]);
    if (kJerk) {
        const f2 wx = fadd2(j.vx, i.nvx);
        const f2 wy = fadd2(j.vy, i.nvy);
        const f2 wz = fadd2(j.vz, i.nvz);
        f2 rv = fmul2(f.dx, wx);
        rv = ffma2(f.dy, wy, rv);
        rv = ffma2(f.dz, wz, rv);                   // d . w
        const f2 q3 = fmul2(fmul2(rv, ri2), m3);    // -3 (d.w) / s
        acc[3 % kNC][p] = ffma2(mr3, ffma2(q3, f.dx, wx), acc[3 % kNC][p]);
        acc[4 % kNC][p] = ffma2(mr3, ffma2(q3, f.dy, wy), acc[4 % kNC][p]);
        acc[5 % kNC][p] = ffma2(mr3, ffma2(q3, f.dz, wz), acc[5 % kNC][p]);
    }
}
template <bool kGuard, bool kJerk, bool kHiLo, bool kList, int kNC, int kP>
__device__ __forceinline__ void interact(const JOps& j, const IPair& i, f2 (&acc)[kNC][kP], int p,
                                         f2 m3, int sl_lo, int sl_hi, int64_t jg, const GuardCtx& g) {
    const Front f = front<kGuard, kHiLo, kList>(j, i, sl_lo, sl_hi, jg, g);
    back<kJerk>(j, i, f, acc, p, m3);
}

template <bool kGuard, bool kJerk, bool kHiLo, class C, bool kList = false>
__global__ void __launch_bounds__(C::kThreads, kJerk ? C::kMinB : C::kMinBAcc) force_kernel(ForceArgs a) {
    constexpr int kPairs = C::kPairs, kThreads = C::kThreads;
    constexpr int kIPerBlock = C::kIPerBlock;
    constexpr int kOffLo = C::kOffLo, kOffBar = C::kOffBar, kOffAcc = C::kOffAcc;
    constexpr int kNC = kJerk ? 6 : 3;   // accumulated components: a (+ jerk)
    constexpr uint32_t kStageTx = kTileBytes + (kHiLo ? kLoTileBytes : 0);
    extern __shared__ __align__(128) unsigned char smem[];
    JPkt* ring = reinterpret_cast<JPkt*>(smem);
    float4* ring_lo = reinterpret_cast<float4*>(smem + kOffLo);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kOffBar);

    const int tid = threadIdx.x;
    int n_loc = a.n_loc;
    if constexpr (kList) n_loc = *a.n_dev;   // block steps: active count read on the device
    // Active-list launches (block time steps) read the active count on the device; their
    // grid (ceil(count / kIPerBlock), chunks) is set by the host or, inside the block-step
    // CUDA graph, by the decide kernel (device-updatable node).  One CTA = one work item.
    if constexpr (kList)
        if ((int)blockIdx.x * kIPerBlock >= n_loc) return;

    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const int c = (a.c_first + (int)blockIdx.y) % a.n_chunks;
    const int64_t jc0 = (int64_t)c * a.chunk;
    const int ntile = a.chunk / kTile;
    const int ib = (int)blockIdx.x * kIPerBlock;

    // ---- i-particles: kPairs packed pairs, stored negated (d = x_j + (-x_i))
    f2 nx[kPairs], ny[kPairs], nz[kPairs], nvx[kPairs], nvy[kPairs], nvz[kPairs];
    f2 nlx[kPairs], nly[kPairs], nlz[kPairs];   // hi/lo: negated low parts
#pragma unroll
    for (int p = 0; p < kPairs; ++p) {
        float q[2][9];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int il = ib + (2 * p + h) * kThreads + tid;
            if (il < n_loc) {
                int64_t src = a.i_base + il;
                if constexpr (kList) {   // block steps: active slot
                    NB_CHECK(a.ilist[il] >= 0 && a.ilist[il] < a.n_loc_pad);   // a.n_loc may be the active count
                    src = a.i_base + a.ilist[il];
                }
                const JPkt pk = a.pkt[src];
                const float4 P = jpkt_pos(pk), V = jpkt_vel(pk);
                q[h][0] = -P.x; q[h][1] = -P.y; q[h][2] = -P.z;
                q[h][3] = -V.x; q[h][4] = -V.y; q[h][5] = -V.z;
                if (kHiLo) {
                    const float4 Lo = a.pklo[src];
                    q[h][6] = -Lo.x; q[h][7] = -Lo.y; q[h][8] = -Lo.z;
                }
            } else {  // padding i: computed, never stored
#pragma unroll
                for (int k = 0; k < 9; ++k) q[h][k] = 0.f;
            }
        }
        nx[p] = f2make(q[0][0], q[1][0]);
        ny[p] = f2make(q[0][1], q[1][1]);
        nz[p] = f2make(q[0][2], q[1][2]);
        nvx[p] = f2make(q[0][3], q[1][3]);
        nvy[p] = f2make(q[0][4], q[1][4]);
        nvz[p] = f2make(q[0][5], q[1][5]);
        if (kHiLo) {
            nlx[p] = f2make(q[0][6], q[1][6]);
            nly[p] = f2make(q[0][7], q[1][7]);
            nlz[p] = f2make(q[0][8], q[1][8]);
        } else {
            nlx[p] = nly[p] = nlz[p] = 0ull;
        }
    }

#if FK_ACC_SMEM
    // fp64 chunk accumulators in shared memory: [k][l][tid], conflict-free
    double* acc_s = reinterpret_cast<double*>(smem + kOffAcc);
#define ACC64(k, l) acc_s[((k) * 2 * kPairs + (l)) * kThreads + tid]
#else
    double acc64[kNC][2 * kPairs];
#define ACC64(k, l) acc64[k][l]
#endif
#pragma unroll
    for (int k = 0; k < kNC; ++k)
#pragma unroll
        for (int l = 0; l < 2 * kPairs; ++l) ACC64(k, l) = 0.0;

    if (tid == 0) {
        for (int s = 0; s < kStages && s < ntile; ++s) {
            mbar_expect_tx(&full[s], kStageTx);
            tma_load_1d(ring + s * kTile, a.pkt + jc0 + (int64_t)s * kTile, kTileBytes, &full[s]);
            if (kHiLo)
                tma_load_1d(ring_lo + s * kTile, a.pklo + jc0 + (int64_t)s * kTile, kLoTileBytes,
                            &full[s]);
        }
    }

    const GuardCtx gc{a.ilist, a.i_base, a.coincident, n_loc};
    const f2 m3 = f2bc(-3.0f);
    IPair ip[kPairs];
#pragma unroll
    for (int p = 0; p < kPairs; ++p)
        ip[p] = IPair{nx[p], ny[p], nz[p], nvx[p], nvy[p], nvz[p], nlx[p], nly[p], nlz[p]};

    for (int t = 0; t < ntile; ++t) {
        const int s = t % kStages;
        mbar_wait(&full[s], (uint32_t)((t / kStages) & 1));
        const JPkt* tile = ring + s * kTile;
        const float4* tile_lo = ring_lo + s * kTile;

        f2 acc[kNC][kPairs];
#pragma unroll
        for (int k = 0; k < kNC; ++k)
#pragma unroll
            for (int p = 0; p < kPairs; ++p) acc[k][p] = 0ull;

        const int64_t jt0 = jc0 + (int64_t)t * kTile;   // global index of the tile's first j
#pragma unroll(kList ? C::kUnrollList : C::kUnrollJ)
        for (int jj = 0; jj < kTile; ++jj) {
            const JOps jo = load_jops<kJerk, kHiLo>(tile, tile_lo, jj);
            const int64_t jg = kGuard ? jt0 + jj : 0;
#pragma unroll
            for (int p = 0; p < kPairs; ++p)
                interact<kGuard, kJerk, kHiLo, kList>(jo, ip[p], acc, p, m3, ib + 2 * p * kThreads + tid,
                                                      ib + (2 * p + 1) * kThreads + tid, jg, gc);
        }
        // tile sum -> fp64, ascending tile order
#pragma unroll
        for (int k = 0; k < kNC; ++k)
#pragma unroll
            for (int p = 0; p < kPairs; ++p) {
                float lo, hi;
                f2split(acc[k][p], lo, hi);
                ACC64(k, 2 * p) += (double)lo;
                ACC64(k, 2 * p + 1) += (double)hi;
            }
        __syncthreads();  // every warp is done reading stage s
        if (tid == 0 && t + kStages < ntile) {
            mbar_expect_tx(&full[s], kStageTx);
            tma_load_1d(ring + s * kTile, a.pkt + jc0 + (int64_t)(t + kStages) * kTile, kTileBytes,
                        &full[s]);
            if (kHiLo)
                tma_load_1d(ring_lo + s * kTile, a.pklo + jc0 + (int64_t)(t + kStages) * kTile,
                            kLoTileBytes, &full[s]);
        }
    }

    // chunk partial [chunk][kNC][n_loc_pad], coalesced fp64 stores
    NB_CHECK(c >= 0 && c < a.n_chunks && jc0 + a.chunk <= (int64_t)a.n_chunks * a.chunk);
    NB_CHECK(ib + kIPerBlock <= a.n_loc_pad || n_loc <= ib);
    double* out = a.partial + (int64_t)c * kNC * a.n_loc_pad;
#pragma unroll
    for (int l = 0; l < 2 * kPairs; ++l) {
        const int il = ib + l * kThreads + tid;
        if (il < n_loc) {
#pragma unroll
            for (int k = 0; k < kNC; ++k) out[(int64_t)k * a.n_loc_pad + il] = ACC64(k, l);
        }
    }
#undef ACC64
}

// ---- tile-split kernel: few i, one warp per j-tile.
// The list kernel gives each CTA a whole chunk (chunk / 256 tiles) of j for
// its i: with a few active particles (block time steps) or a small N the
// launch has too few CTAs, each one serial j loop, and leaves most of the GPU
// idle (scripts/block_launch_sizes.py).  Here CTA = (kI i, chunk) with one
// warp per tile: warp w stages tile r0 + w into its own shared-memory buffer
// and computes that tile's fp32 sums, and after each round of W tiles the CTA
// adds the round's tile sums to the fp64 chunk sums in ascending tile order --
// the same additions, in the same order, as force_kernel, so the partials are
// bit-identical to every other shape's.
//   packed (kScalar = false): lane = one i-pair (slots ib + lane, ib + 32 + lane),
//            interact() as in force_kernel; 64 i per CTA.
//   scalar (kScalar = true): lane = one i (slot ib + lane), interact1(), the
//            same operations on one lane; 32 i per CTA.  A warp's j loop is
//            issue-bound (~26 FP32 instructions per j), and a packed instruction
//            holds the FMA pipe for two cycles, so the scalar form runs a tile in
//            about half the time for half the i: it is the faster one when the
//            launch is latency-bound (tiny active sets, N ~ 1 000).
constexpr int kTsWarpsMax = 8;
constexpr int kTsplitMaxDefault = 1024;   // packed tile-split up to this many active i
constexpr int kTsplit1MaxDefault = 256;   // scalar tile-split up to this many active i
// shared memory of a W-warp CTA (sized by W, so short chunks get more CTAs per SM):
// [W tile buffers][W x <=6 x <=64 fp32 tile sums][<=6 x <=64 fp64 chunk sums][W mbarriers]
template <bool kHiLo>
struct TsCfg {
    static constexpr int kTileB = kTileBytes + (kHiLo ? kLoTileBytes : 0);
    __host__ __device__ static constexpr int off_sum(int W) { return W * kTileB; }
    __host__ __device__ static constexpr int off_acc(int W) { return off_sum(W) + W * 6 * 64 * 4; }
    __host__ __device__ static constexpr int off_bar(int W) { return off_acc(W) + 6 * 64 * 8; }
    __host__ __device__ static constexpr int smem_bytes(int W) { return off_bar(W) + W * 8; }
    static constexpr int kSmemMax = smem_bytes(kTsWarpsMax);
};

__device__ __forceinline__ float fadd1(float a, float b) {
    float d;
    asm("add.rn.ftz.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}
__device__ __forceinline__ float fmul1(float a, float b) {
    float d;
    asm("mul.rn.ftz.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}
__device__ __forceinline__ float ffma1(float a, float b, float c) {
    float d;
    asm("fma.rn.ftz.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

// interact() on one lane: the same operations in the same order (FTZ, RN), so
// each lane's tile sum equals the corresponding lane of the packed form
template <bool kGuard, bool kJerk, bool kHiLo, bool kList, int kNC>
__device__ __forceinline__ void interact1(const JOps1& j, const IOne& i, float (&acc)[kNC], int sl,
                                          int64_t jg, const GuardCtx& g) {
    float dx = fadd1(j.x, i.nx);
    float dy = fadd1(j.y, i.ny);
    float dz = fadd1(j.z, i.nz);
    if (kHiLo) {
        dx = fadd1(dx, fadd1(j.lx, i.nlx));
        dy = fadd1(dy, fadd1(j.ly, i.nly));
        dz = fadd1(dz, fadd1(j.lz, i.nlz));
    }
    float s2 = ffma1(dx, dx, j.eps2);
    s2 = ffma1(dy, dy, s2);
    s2 = ffma1(dz, dz, s2);
    float ri = rsqrt_ftz(s2);
    if (kGuard && s2 == 0.f) {
        ri = 0.f;
        report_coincident<kList>(g, sl, jg, j.m);
    }
    const float ri2 = fmul1(ri, ri);
    const float mr3 = fmul1(fmul1(j.m, ri), ri2);
    acc[0] = ffma1(mr3, dx, acc[0]);
    acc[1] = ffma1(mr3, dy, acc[1]);
    acc[2] = ffma1(mr3, dz, acc[2]);
    if (kJerk) {
        const float wx = fadd1(j.vx, i.nvx);
        const float wy = fadd1(j.vy, i.nvy);
        const float wz = fadd1(j.vz, i.nvz);
        float rv = fmul1(dx, wx);
        rv = ffma1(dy, wy, rv);
        rv = ffma1(dz, wz, rv);
        const float q3 = fmul1(fmul1(rv, ri2), -3.0f);
        acc[3 % kNC] = ffma1(mr3, ffma1(q3, dx, wx), acc[3 % kNC]);
        acc[4 % kNC] = ffma1(mr3, ffma1(q3, dy, wy), acc[4 % kNC]);
        acc[5 % kNC] = ffma1(mr3, ffma1(q3, dz, wz), acc[5 % kNC]);
    }
}

template <bool kGuard, bool kJerk, bool kHiLo, bool kScalar, bool kList>
__global__ void __launch_bounds__(kTsWarpsMax * 32, 2) force_tsplit_kernel(ForceArgs a) {
    using C = TsCfg<kHiLo>;
    constexpr int kI = kScalar ? 32 : 64, kNC = kJerk ? 6 : 3, kH = kScalar ? 1 : 2;
    int n_loc = a.n_loc;
    if constexpr (kList) n_loc = *a.n_dev;   // block steps: active count read on the device
    const int ib = (int)blockIdx.x * kI;
    if (ib >= n_loc) return;
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, W = (int)blockDim.x >> 5;
    JPkt* tile = reinterpret_cast<JPkt*>(smem + w * C::kTileB);
    float4* tile_lo = reinterpret_cast<float4*>(smem + w * C::kTileB + kTileBytes);
    float* tsum = reinterpret_cast<float*>(smem + C::off_sum(W));
    double* acc64 = reinterpret_cast<double*>(smem + C::off_acc(W));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::off_bar(W)) + w;
    const int c = (a.c_first + (int)blockIdx.y) % a.n_chunks;
    const int64_t jc0 = (int64_t)c * a.chunk;
    const int ntile = a.chunk / kTile;
    // stage tile t with one bulk TMA copy (+ the hi/lo tails) on the warp's mbarrier
    auto stage = [&](int t) {
        mbar_expect_tx(bar, kTileBytes + (kHiLo ? kLoTileBytes : 0));
        tma_load_1d(tile, a.pkt + jc0 + (int64_t)t * kTile, kTileBytes, bar);
        if (kHiLo) tma_load_1d(tile_lo, a.pklo + jc0 + (int64_t)t * kTile, kLoTileBytes, bar);
    };
    if (lane == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (w < ntile) stage(w);   // first tile in flight while the i-particles load
    }
    __syncwarp();

    float q[kH][9];
#pragma unroll
    for (int h = 0; h < kH; ++h) {
        const int il = ib + h * 32 + lane;
        const bool valid = il < n_loc;
        int64_t src = 0;
        if (valid) {
            if constexpr (kList) {
                NB_CHECK(a.ilist[il] >= 0 && a.ilist[il] < a.n_loc_pad);   // a.n_loc may be the active count
                src = a.i_base + a.ilist[il];
            } else {
                src = a.i_base + il;
            }
        }
        load_i<kHiLo>(a, valid, src, q[h]);
    }
    const GuardCtx gc{a.ilist, a.i_base, a.coincident, n_loc};
    const f2 m3 = f2bc(-3.0f);
    IPair ip;
    IOne i1;
    if constexpr (kScalar) {
        i1 = IOne{q[0][0], q[0][1], q[0][2], q[0][3], q[0][4], q[0][5], q[0][6], q[0][7], q[0][8]};
    } else {
        ip = IPair{f2make(q[0][0], q[kH - 1][0]), f2make(q[0][1], q[kH - 1][1]), f2make(q[0][2], q[kH - 1][2]),
                   f2make(q[0][3], q[kH - 1][3]), f2make(q[0][4], q[kH - 1][4]), f2make(q[0][5], q[kH - 1][5]),
                   f2make(q[0][6], q[kH - 1][6]), f2make(q[0][7], q[kH - 1][7]), f2make(q[0][8], q[kH - 1][8])};
    }
    for (int k = tid; k < kNC * kI; k += blockDim.x) acc64[k] = 0.0;

    uint32_t phase = 0;
    for (int r0 = 0; r0 < ntile; r0 += W) {
        const int t = r0 + w;
        if (t < ntile) {
            if (lane == 0 && r0 > 0) stage(t);   // round 0 was issued in the prologue
            mbar_wait(bar, phase);
            phase ^= 1;
            float* ts = tsum + w * kNC * kI;
            if constexpr (kScalar) {
                float acc[kNC];
#pragma unroll
                for (int k = 0; k < kNC; ++k) acc[k] = 0.f;
#pragma unroll kTs1Unroll
                for (int jj = 0; jj < kTile; ++jj) {
                    const JOps1 jo = load_jops1<kJerk, kHiLo>(tile, tile_lo, jj);
                    const int64_t jg = kGuard ? jc0 + (int64_t)t * kTile + jj : 0;
                    interact1<kGuard, kJerk, kHiLo, kList>(jo, i1, acc, ib + lane, jg, gc);
                }
#pragma unroll
                for (int k = 0; k < kNC; ++k) ts[k * kI + lane] = acc[k];
            } else {
                f2 acc[kNC][1];
#pragma unroll
                for (int k = 0; k < kNC; ++k) acc[k][0] = 0ull;
#pragma unroll kTsUnroll
                for (int jj = 0; jj < kTile; ++jj) {
                    const JOps jo = load_jops<kJerk, kHiLo>(tile, tile_lo, jj);
                    const int64_t jg = kGuard ? jc0 + (int64_t)t * kTile + jj : 0;
                    interact<kGuard, kJerk, kHiLo, kList>(jo, ip, acc, 0, m3, ib + lane, ib + 32 + lane, jg, gc);
                }
#pragma unroll
                for (int k = 0; k < kNC; ++k) {
                    float lo, hi;
                    f2split(acc[k][0], lo, hi);
                    ts[k * kI + lane] = lo;
                    ts[k * kI + 32 + lane] = hi;
                }
            }
        }
        __syncthreads();   // this round's tile sums are in shared memory
        const int nr = min(W, ntile - r0);
        for (int k = tid; k < kNC * kI; k += blockDim.x) {
            double sum = acc64[k];
            for (int u = 0; u < nr; ++u) sum += (double)tsum[u * kNC * kI + k];   // ascending tiles
            acc64[k] = sum;
        }
        __syncthreads();   // tile buffers and tile sums are free for the next round
    }
    NB_CHECK(c >= 0 && c < a.n_chunks);
    NB_CHECK(ib + kI <= a.n_loc_pad || n_loc <= ib);
    double* out = a.partial + (int64_t)c * kNC * a.n_loc_pad;
    for (int k = tid; k < kNC * kI; k += blockDim.x) {
        const int il = ib + k % kI;
        if (il < n_loc) out[(int64_t)(k / kI) * a.n_loc_pad + il] = acc64[k];
    }
}

}  // namespace

int force_i_per_block() { return kIPerBlock; }
int force_tsplit_i_per_block(bool scalar) { return scalar ? 32 : 64; }
int force_tsplit_threads(int chunk) { return 32 * std::max(1, std::min(kTsWarpsMax, chunk / kTile)); }
int force_list_i_per_block(bool big) { return big ? CfgBig::kIPerBlock : CfgSmall::kIPerBlock; }

int sm_count();

template <bool G, bool J, bool H, class C>
cudaError_t set_attr() {
    cudaError_t e = cudaFuncSetAttribute(force_kernel<G, J, H, C>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if constexpr (J)   // active-list variant (block steps)
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(force_kernel<G, J, H, C, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    return e;
}

template <class C>
cudaError_t set_attrs() {
    cudaError_t e = cudaSuccess, r;
    if ((r = set_attr<false, false, false, C>()) != cudaSuccess) e = r;
    if ((r = set_attr<false, false, true, C>()) != cudaSuccess) e = r;
    if ((r = set_attr<false, true, false, C>()) != cudaSuccess) e = r;
    if ((r = set_attr<false, true, true, C>()) != cudaSuccess) e = r;
    if ((r = set_attr<true, false, false, C>()) != cudaSuccess) e = r;
    if ((r = set_attr<true, false, true, C>()) != cudaSuccess) e = r;
    if ((r = set_attr<true, true, false, C>()) != cudaSuccess) e = r;
    if ((r = set_attr<true, true, true, C>()) != cudaSuccess) e = r;
    return e;
}

template <bool G, bool J, bool H, bool S, bool L>
cudaError_t set_ts_attr() {
    return cudaFuncSetAttribute(force_tsplit_kernel<G, J, H, S, L>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                TsCfg<H>::kSmemMax);
}
// instantiated: list (block steps, jerk) packed + scalar; plain (small launches) scalar
template <bool G, bool H>
cudaError_t set_ts_attrs_gh() {
    cudaError_t e = set_ts_attr<G, true, H, false, true>();
    if (e == cudaSuccess) e = set_ts_attr<G, true, H, true, true>();
    if (e == cudaSuccess) e = set_ts_attr<G, true, H, true, false>();
    if (e == cudaSuccess) e = set_ts_attr<G, false, H, true, false>();
    return e;
}
cudaError_t set_tsplit_attrs() {
    cudaError_t e = set_ts_attrs_gh<false, false>();
    if (e == cudaSuccess) e = set_ts_attrs_gh<false, true>();
    if (e == cudaSuccess) e = set_ts_attrs_gh<true, false>();
    if (e == cudaSuccess) e = set_ts_attrs_gh<true, true>();
    return e;
}

// dynamic shared memory above 48 KiB must be opted into once per instantiation
// (a function attribute belongs to the current device's context: once per device)
cudaError_t ensure_attrs() {
    static std::mutex mu;
    static std::atomic<uint64_t> done_mask{0};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = 1ull << (dev & 63);
    if (done_mask.load(std::memory_order_acquire) & bit) return cudaSuccess;
    std::lock_guard<std::mutex> lock(mu);
    if (done_mask.load(std::memory_order_relaxed) & bit) return cudaSuccess;
    e = set_attrs<CfgBig>();
    if (e == cudaSuccess) e = set_attrs<CfgSmall>();
    if (e == cudaSuccess) e = set_tsplit_attrs();
    if (e == cudaSuccess) done_mask.fetch_or(bit, std::memory_order_release);
    return e;
}

template <bool G, bool J, bool H, class C>
cudaError_t launch_one(const ForceArgs& a, unsigned c_count, cudaStream_t s) {
    cudaError_t e = ensure_attrs();
    if (e != cudaSuccess) return e;
    // the active-list indirection is a separate instantiation so that the plain
    // kernels' register allocation (and speed) is untouched by it
    const dim3 grid((unsigned)std::max<int64_t>(1, (a.n_loc + C::kIPerBlock - 1) / C::kIPerBlock), c_count);
    if (a.ilist) {
        if constexpr (J) {
            if (!a.n_dev) return cudaErrorInvalidValue;
            force_kernel<G, J, H, C, true><<<grid, C::kThreads, C::kSmemBytes, s>>>(a);
        } else {
            return cudaErrorInvalidValue;   // block time steps: jerk kernel
        }
    } else {
        force_kernel<G, J, H, C><<<grid, C::kThreads, C::kSmemBytes, s>>>(a);
    }
    return cudaGetLastError();
}

template <bool G, bool J, class C>
cudaError_t launch_gj(const ForceArgs& a, cudaStream_t s) {
    return a.pklo ? launch_one<G, J, true, C>(a, (unsigned)a.c_count, s)
                  : launch_one<G, J, false, C>(a, (unsigned)a.c_count, s);
}

template <class C>
cudaError_t launch_cfg(const ForceArgs& a, bool guard_self, bool jerk, cudaStream_t s) {
    if (jerk) return guard_self ? launch_gj<true, true, C>(a, s) : launch_gj<false, true, C>(a, s);
    return guard_self ? launch_gj<true, false, C>(a, s) : launch_gj<false, false, C>(a, s);
}

int sm_count() {
    static int n = [] {
        int dev = 0, v = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
            cudaGetLastError();
            return 148;
        }
        return v;
    }();
    return n;
}

// The small CTA shape when the default one would fill fewer than two waves of
// the GPU (its per-CTA efficiency is within ~10 % of the default's,
// profiles/r01_sweep_force.txt p1b6, and it quarters the idle i-slots).
bool use_small_cta(const ForceArgs& a) {
    const char* ov = getenv("NBODY_FORCE_CTA");   // tests: small | big (default: by size)
    if (ov && !strcmp(ov, "small")) return true;
    if (ov && (!strcmp(ov, "big") || !strcmp(ov, "tiny"))) return false;
    const int64_t ctas = (int64_t)((a.n_loc + kIPerBlock - 1) / kIPerBlock) * a.c_count;
    return ctas < 2LL * FK_MINB * sm_count();
}

// Launches whose 256-i CTAs would not give every SM one CTA (N ~ 1 000) are
// latency-bound: the scalar tile-split kernel runs them with 32 i per warp.
bool use_tiny(const ForceArgs& a) {
    const char* ov = getenv("NBODY_FORCE_CTA");
    if (ov && *ov) return !strcmp(ov, "tiny");
    const int64_t ctas = (int64_t)((a.n_loc + CfgSmall::kIPerBlock - 1) / CfgSmall::kIPerBlock) * a.c_count;
    return ctas < sm_count();
}

cudaError_t launch_force_list(const ForceArgs& a, bool guard_self, bool big, cudaStream_t s) {
    if (a.c_count <= 0 || a.n_loc <= 0) return cudaSuccess;
    if (!a.ilist) return cudaErrorInvalidValue;
    return big ? launch_cfg<CfgBig>(a, guard_self, true, s) : launch_cfg<CfgSmall>(a, guard_self, true, s);
}

cudaError_t launch_force_big(const ForceArgs& a, bool guard_self, bool jerk, cudaStream_t s) {
    if (a.c_count <= 0 || a.n_loc <= 0) return cudaSuccess;
    if (a.ilist) return cudaErrorInvalidValue;
    return launch_cfg<CfgBig>(a, guard_self, jerk, s);
}

cudaError_t launch_force(const ForceArgs& a, bool guard_self, bool jerk, cudaStream_t s) {
    if (a.c_count <= 0 || a.n_loc <= 0) return cudaSuccess;
    if (a.ilist) return launch_cfg<CfgSmall>(a, guard_self, jerk, s);   // active-list kernel
#ifndef FK_NO_SMALL
    if (use_tiny(a)) return launch_force_tsplit(a, guard_self, jerk, true, s);
    if (use_small_cta(a)) return launch_cfg<CfgSmall>(a, guard_self, jerk, s);
#endif
    return launch_cfg<CfgBig>(a, guard_self, jerk, s);
}

template <bool G, bool J, bool H, bool S, bool L>
cudaError_t launch_ts(const ForceArgs& a, cudaStream_t s) {
    const int ipb = S ? 32 : 64;
    const dim3 grid((unsigned)std::max<int64_t>(1, (a.n_loc + ipb - 1) / ipb), (unsigned)a.c_count);
    const int threads = force_tsplit_threads(a.chunk);
    force_tsplit_kernel<G, J, H, S, L><<<grid, threads, TsCfg<H>::smem_bytes(threads / 32), s>>>(a);
    return cudaGetLastError();
}
template <bool G, bool H>
cudaError_t launch_ts_gh(const ForceArgs& a, bool jerk, bool scalar, cudaStream_t s) {
    if (a.ilist) {   // block steps (jerk)
        if (!a.n_dev || !jerk) return cudaErrorInvalidValue;
        return scalar ? launch_ts<G, true, H, true, true>(a, s) : launch_ts<G, true, H, false, true>(a, s);
    }
    if (!scalar) return cudaErrorInvalidValue;   // plain launches use the scalar form only
    return jerk ? launch_ts<G, true, H, true, false>(a, s) : launch_ts<G, false, H, true, false>(a, s);
}

cudaError_t launch_force_tsplit(const ForceArgs& a, bool guard_self, bool jerk, bool scalar, cudaStream_t s) {
    if (a.c_count <= 0 || a.n_loc <= 0) return cudaSuccess;
    cudaError_t e = ensure_attrs();
    if (e != cudaSuccess) return e;
    if (guard_self)
        return a.pklo ? launch_ts_gh<true, true>(a, jerk, scalar, s) : launch_ts_gh<true, false>(a, jerk, scalar, s);
    return a.pklo ? launch_ts_gh<false, true>(a, jerk, scalar, s) : launch_ts_gh<false, false>(a, jerk, scalar, s);
}

// Block steps: active counts up to force_tsplit1_max() use the scalar tile-split
// kernel, up to force_tsplit_max() the packed one when a chunk has >= 2 tiles, larger
// ones the list kernel.  NBODY_TSPLIT1_MAX / NBODY_TSPLIT_MAX override (0 disables;
// read per call: tests switch them per context).  Chosen by scripts/tsplit_sweep.sh.
int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e && *e ? std::max(0, atoi(e)) : dflt;
}
int force_tsplit_max() { return env_int("NBODY_TSPLIT_MAX", kTsplitMaxDefault); }
int force_tsplit1_max() { return env_int("NBODY_TSPLIT1_MAX", kTsplit1MaxDefault); }

int force_ctas_per_sm(bool jerk, bool hilo) {
    int n = 0;
    cudaError_t e = ensure_attrs();
    if (e != cudaSuccess) {
        cudaGetLastError();
        return FK_MINB;
    }
    constexpr int kT = CfgBig::kThreads, kS = CfgBig::kSmemBytes;
    if (jerk)
        e = hilo ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, force_kernel<false, true, true, CfgBig>, kT, kS)
                 : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, force_kernel<false, true, false, CfgBig>, kT, kS);
    else
        e = hilo ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, force_kernel<false, false, true, CfgBig>, kT, kS)
                 : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, force_kernel<false, false, false, CfgBig>, kT, kS);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return FK_MINB;
    }
    return n > 0 ? n : 1;
}

}  // namespace nb
