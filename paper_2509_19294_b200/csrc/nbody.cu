// nbody.cu -- the C-ABI runtime of libnbody.so (declared in include/nbody.h).
//
// Owns the device state of one rank (or of all ranks in loopback mode),
// the exchange buffer, the CUDA events/streams and the NCCL communicator,
// and sequences the per-step kernels:
//
//   predict+pack (fp64 -> fp32 packets)            hermite.cu
//   exchange: ncclAllGather of 32-B packets         (P > 1; comm stream)
//   force pass over the local j-chunks              force.cu   -- overlaps the
//   force pass over the remote j-chunks             force.cu      all-gather
//   fold chunks + correct + predict + pack (fp64)   hermite.cu
//
// NCCL is resolved with dlopen at first use (the libnccl.so.2 the process
// already loaded, i.e. torch's, unless NBODY_NCCL_LIB names another), so the
// library never links a second NCCL and never needs one for world == 1.  The
// communicator is non-blocking: every NCCL call is followed by a bounded wait
// (NBODY_NCCL_TIMEOUT_S) for it to leave ncclInProgress, so a rank that never
// arrives or dies turns into NBODY_ENCCL instead of a hang, and a failed
// context is torn down with ncclCommAbort.
//
// Loopback mode (cfg.loopback, tests and the scaling projection) runs `world`
// shards in one context on one GPU.  Each shard owns its exchange buffer, and
// the all-gather is emulated by one cudaMemcpyAsync per remote slice into it,
// between the same local-first / remote-second force launches an NCCL rank
// issues -- so a wrong slice offset or a local launch that reads a remote
// chunk changes the result (tests/test_gpu_exchange.py).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges cost nothing unless a tool is attached

#include <sched.h>

#include <cfloat>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"
#include "nbody.h"

using nb::JPkt;

namespace {

thread_local std::string g_last_error = "";

// NVTX range for profilers (nsys / ncu --nvtx): every C-ABI entry point and, on the eager
// path, every phase of a step is a named range (inside a CUDA graph only its launch is)
struct Nvtx {
    explicit Nvtx(const char* name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
    Nvtx(const Nvtx&) = delete;
    Nvtx& operator=(const Nvtx&) = delete;
};

// ------------------------------------------------------------------ NCCL

struct NcclApi {
    bool tried = false, ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRankConfig)(ncclComm_t*, int, ncclUniqueId, int, ncclConfig_t*) = nullptr;
    ncclResult_t (*CommFinalize)(ncclComm_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi load_nccl() {
    NcclApi api;
    api.tried = true;
    const char* path = getenv("NBODY_NCCL_LIB");
    void* h = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        api.why = std::string("cannot load NCCL: ") + dlerror();
        return api;
    }
#define NB_SYM(field, name)                                         \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name)); \
    if (!api.field) {                                                \
        api.why = std::string("NCCL symbol missing: ") + name;       \
        return api;                                                  \
    }
    NB_SYM(GetUniqueId, "ncclGetUniqueId");
    NB_SYM(CommInitRankConfig, "ncclCommInitRankConfig");
    NB_SYM(CommFinalize, "ncclCommFinalize");
    NB_SYM(CommDestroy, "ncclCommDestroy");
    NB_SYM(CommAbort, "ncclCommAbort");
    NB_SYM(CommGetAsyncError, "ncclCommGetAsyncError");
    NB_SYM(AllGather, "ncclAllGather");
    NB_SYM(AllReduce, "ncclAllReduce");
    NB_SYM(GetErrorString, "ncclGetErrorString");
#undef NB_SYM
    api.ok = true;
    return api;
}

// resolved once per process; the function-local static makes concurrent first
// calls from several threads safe
NcclApi& nccl() {
    static NcclApi api = load_nccl();
    return api;
}

// ------------------------------------------------------------------ plan

struct Plan {
    int64_t i0, i1, slot, chunk, n_chunks;
};

int make_plan(int64_t n, int32_t world, int32_t rank, int32_t jchunks, Plan* p, std::string* why) {
    if (n < 2) { *why = "n must be >= 2"; return NBODY_EINVAL; }
    if (world < 1 || world > n) { *why = "world must satisfy 1 <= world <= n"; return NBODY_EINVAL; }
    if (rank < 0 || rank >= world) { *why = "rank must satisfy 0 <= rank < world"; return NBODY_EINVAL; }
    if (jchunks < 0) { *why = "jchunks must be >= 0"; return NBODY_EINVAL; }
    const int64_t jc = jchunks == 0 ? 128 : jchunks;
    const int64_t T = nb::kTile;
    // slot: multiple of the force i-block, so which arithmetic (FP32 pair lane or
    // FP64 slot) a particle gets depends on its global index only (P-invariant)
    const int64_t B = nb::force_i_per_block();
    p->slot = B * ((n + B * world - 1) / (B * world));
    p->i0 = std::min<int64_t>(n, rank * p->slot);
    p->i1 = std::min<int64_t>(n, (int64_t)(rank + 1) * p->slot);
    if (p->slot > INT32_MAX) {   // per-shard counts are int32 on the device
        *why = "n / world must not exceed 2^31 - 1 particles per shard";
        return NBODY_EINVAL;
    }
    p->chunk = T * ((n + T * jc - 1) / (T * jc));
    p->n_chunks = (n + p->chunk - 1) / p->chunk;
    return NBODY_OK;
}

// ------------------------------------------------------------------ context

struct Shard {
    Plan plan;
    JPkt* pkt = nullptr;      // exchange buffer this shard packs into and reads j from: the
    float4* pklo = nullptr;   // context's (NCCL / world 1), or its own (loopback shards >= 1)
    bool own_pkt = false;
    int32_t n_loc = 0;
    int64_t n_loc_pad = 0;
    double *m = nullptr, *x = nullptr, *v = nullptr, *a0 = nullptr, *j0 = nullptr;
    double *xp = nullptr, *vp = nullptr, *partial = nullptr;
    int32_t c_lo = 0, c_hi = 0;  // local chunks [c_lo, c_hi)
    int64_t* T = nullptr;        // block time steps: particle times (ticks), levels,
    int32_t* lev = nullptr;      // active list (R#28)
    int32_t* ilist = nullptr;
};

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

}  // namespace

struct nbody_ctx {
    nbody_config cfg{};
    int64_t n = 0, L = 0;
    int sm_count = 148;
    float eps2f = 0.f;
    int nshards = 1;
    std::vector<Shard> sh;
    JPkt* pkt = nullptr;
    float4* pklo = nullptr;   // hi/lo position tails (cfg.hilo)
    bool guard = false;       // eps2f < FLT_MIN (0 or subnormal, flushed to 0 on the device):
                              // the force pass excludes s == 0 explicitly (R#17)
    double4* eall = nullptr;
    double* eblk = nullptr;
    int eblk_cap = 0;
    double* eout = nullptr;  // [nshards][2]
    unsigned long long* flags = nullptr;  // [0] non-finite, [1] coincident, [2..4] validate
    // block time steps (R#28): t_next (ticks, shared by all shards), per-shard
    // active counts, pinned read-back of both, run statistics
    unsigned long long* tnext = nullptr;   // this block step's time (ticks)
    unsigned long long* tcur = nullptr;    // the previous block step's time
    int32_t* nact = nullptr;               // per shard: selection append counters
    int32_t* nact_cur = nullptr;           // per shard: this block step's active counts
    int32_t* lvl_cnt = nullptr;   // [64] particles per level, all shards
    unsigned* sel_done = nullptr;  // selection-pass CTA counter (decide fused, one shard)
    nb::BlockGraphNodes* gnodes = nullptr;   // device copy of the graph's force-node handles
    long long* ctl = nullptr;            // [t_end, block steps, active sum, done] (device)
    void* hbuf = nullptr;
    bool levels_ok = false;
    cudaGraphExec_t block_graph = nullptr;   // WHILE-loop graph of block steps (R#28)
    bool block_graph_failed = false;         // NCCL ranks: the capture was refused -> host loop
    cudaStream_t stream = nullptr, comm_stream = nullptr;
    bool own_stream = false;
    cudaEvent_t ev_packed = nullptr, ev_gathered = nullptr;
    ncclComm_t comm = nullptr;
    double nccl_timeout_s = 600.0;
    bool loop_concurrent = false;   // loopback shards in the NCCL rank's stream form (NBODY_LOOPBACK_CONCURRENT)
    bool have_a0 = false, predicted = false;
    bool use_graph = true;
    cudaGraphExec_t step_graph = nullptr;
    int64_t graph_kernels = 0, graph_force = 0;
    bool prof = false;
    std::vector<cudaEvent_t> prof_ev;  // pairs
    std::vector<int64_t> prof_ni, prof_nj;   // i and j particles of each timed launch
    size_t prof_used = 0;
    int64_t n_force = 0, n_kernels = 0;
    int64_t graph_launches = 0, eager_steps = 0;   // nbody_exec_stats
    // block-step graph runs launch their kernels on the device: counted at prof_read time
    // from the block-step counter ctl[1] (minus the host-driven block steps since the reset)
    int64_t block_graph_calls = 0, block_host_steps = 0, block_steps_at_reset = 0;
    std::string err;
    int sticky = 0;
};

namespace {

int fail(nbody_ctx* c, int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) {
        c->err = buf;
        if (code == NBODY_ECUDA || code == NBODY_ENCCL || code == NBODY_ENONFINITE) c->sticky = code;
    }
    g_last_error = buf;
    return code;
}

#define CK(ctx, call)                                                                      \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            return fail(ctx, NBODY_ECUDA, "%s failed: %s (%s:%d)", #call,                  \
                        cudaGetErrorString(e_), __FILE__, __LINE__);                       \
    } while (0)

// Non-blocking communicator: a call returns ncclSuccess or ncclInProgress, and the next
// call may only be issued once the communicator has left ncclInProgress.  Wait for
// that, at most c->nccl_timeout_s seconds (then NBODY_ENCCL, and the context is torn
// down with ncclCommAbort).
int nccl_settle(nbody_ctx* c, ncclResult_t r, const char* what) {
    if (r != ncclSuccess && r != ncclInProgress)
        return fail(c, NBODY_ENCCL, "%s failed: %s", what, nccl().GetErrorString(r));
    const auto t0 = std::chrono::steady_clock::now();
    for (int spin = 0;; ++spin) {
        ncclResult_t st = ncclSuccess;
        ncclResult_t q = nccl().CommGetAsyncError(c->comm, &st);
        if (q != ncclSuccess) return fail(c, NBODY_ENCCL, "%s: ncclCommGetAsyncError: %s", what, nccl().GetErrorString(q));
        if (st == ncclSuccess) return NBODY_OK;
        if (st != ncclInProgress) return fail(c, NBODY_ENCCL, "%s: %s", what, nccl().GetErrorString(st));
        const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (el > c->nccl_timeout_s)
            return fail(c, NBODY_ENCCL, "%s: no progress after %.1f s (NBODY_NCCL_TIMEOUT_S); a peer rank "
                        "is missing or dead", what, el);
        if (spin > 64) sched_yield();
    }
}

#define CKNCCL(ctx, call)                                                                  \
    do {                                                                                   \
        int rc_ = nccl_settle(ctx, (call), #call);                                         \
        if (rc_) return rc_;                                                               \
    } while (0)

#define GUARD(ctx)                                                                          \
    do {                                                                                    \
        if (!(ctx)) return fail(nullptr, NBODY_EINVAL, "null context");                     \
        if ((ctx)->sticky)                                                                  \
            return fail(ctx, NBODY_ESTATE, "context failed earlier: %s", (ctx)->err.c_str()); \
        CK(ctx, cudaSetDevice((ctx)->cfg.device));                                          \
    } while (0)

int ncomp(const nbody_ctx* c) { return c->cfg.integrator == NBODY_LEAPFROG_KDK ? 3 : 6; }
bool is_block(const nbody_ctx* c) { return c->cfg.integrator == NBODY_HERMITE4_BLOCK; }

nb::StateArgs state_args(nbody_ctx* c, Shard& s) {
    nb::StateArgs a;
    a.n_loc = s.n_loc;
    a.n_loc_pad = s.n_loc_pad;
    a.i_base = s.plan.i0;
    a.G = c->cfg.G;
    a.dt = c->cfg.dt;
    a.eps2 = c->eps2f;
    a.m = s.m;
    a.x = s.x; a.v = s.v; a.a0 = s.a0; a.j0 = s.j0; a.xp = s.xp; a.vp = s.vp;
    a.partial = s.partial;
    a.n_chunks = (int32_t)s.plan.n_chunks;
    a.ncomp = ncomp(c);
    a.integrator = c->cfg.integrator == NBODY_LEAPFROG_KDK ? 1 : 0;   // predictor/corrector family
    a.pkt = s.pkt;
    a.pklo = s.pklo;
    a.bad = c->flags;
    a.T = s.T;
    a.lev = s.lev;
    a.ilist = s.ilist;
    a.nact = c->nact ? c->nact + (&s - c->sh.data()) : nullptr;
    a.nact_cur = c->nact_cur ? c->nact_cur + (&s - c->sh.data()) : nullptr;
    a.tnext = c->tnext;
    a.tcur = c->tcur;
    a.self_tnext = c->comm ? 0 : 1;   // NCCL ranks reduce t_next over ranks first
    a.lvl_cnt = c->lvl_cnt;
    a.sel_done = nullptr;   // block_step_body enables the fused decide step
    a.cond = 0;
    a.gnodes = nullptr;
    a.ctl = c->ctl;
    a.kmax = c->cfg.kmax;
    a.eta = c->cfg.eta;
    a.eta_s = c->cfg.eta_s;
    return a;
}

bool use_nccl(const nbody_ctx* c) { return c->comm != nullptr; }
// block steps with one shard per context fold the decide step into the selection pass
bool decide_fused(const nbody_ctx* c) { return c->nshards == 1; }

// force pass over chunks [c_first, c_first + c_count) for the shard's local
// particles, or (block steps) for the n_i active particles listed in ilist
// tsplit (block steps): 0 = list kernel (256-i CTAs), 1 = packed tile-split, 2 = scalar
// tile-split, 3 = list kernel (1024-i CTAs); plain launches: 0 (CTA shape by size) or
// kForceBig (1024-i CTAs: the exchange-overlap launch, sized in whole waves of that shape)
constexpr int kForceBig = 4;
int launch_force_range(nbody_ctx* c, Shard& s, int32_t c_first, int32_t c_count, int32_t n_i = -1,
                       const int32_t* ilist = nullptr, const int32_t* n_dev = nullptr, int tsplit = 0,
                       cudaStream_t st = nullptr) {
    if (!st) st = c->stream;
    if (n_i < 0) n_i = s.n_loc;
    if (c_count <= 0 || n_i <= 0) return NBODY_OK;
    nb::ForceArgs f;
    f.pkt = s.pkt;
    f.pklo = s.pklo;
    f.i_base = s.plan.i0;
    f.n_loc = n_i;
    f.ilist = ilist;
    f.n_dev = n_dev;
    f.n_loc_pad = s.n_loc_pad;
    f.chunk = (int32_t)s.plan.chunk;
    f.n_chunks = (int32_t)s.plan.n_chunks;
    f.c_first = c_first;
    f.c_count = c_count;
    f.eps2 = c->eps2f;
    f.partial = s.partial;
    f.coincident = c->flags + 1;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->prof) {
        if (c->prof_used + 2 > c->prof_ev.size()) {
            for (int k = 0; k < 2; ++k) {
                cudaEvent_t e;
                CK(c, cudaEventCreate(&e));
                c->prof_ev.push_back(e);
            }
        }
        e0 = c->prof_ev[c->prof_used];
        e1 = c->prof_ev[c->prof_used + 1];
        c->prof_used += 2;
        int64_t nj = 0;   // real j particles in chunks c_first .. c_first + c_count - 1 (mod n_chunks)
        for (int32_t q = 0; q < c_count; ++q) {
            const int64_t ch = (c_first + q) % s.plan.n_chunks;
            nj += std::min<int64_t>(c->n, (ch + 1) * s.plan.chunk) - ch * s.plan.chunk;
        }
        c->prof_ni.resize(c->prof_used / 2);
        c->prof_nj.resize(c->prof_used / 2);
        c->prof_ni.back() = n_i;
        c->prof_nj.back() = nj;
        CK(c, cudaEventRecord(e0, st));
    }
    if (tsplit == 1 || tsplit == 2)
        CK(c, nb::launch_force_tsplit(f, c->guard, ncomp(c) == 6, tsplit == 2, st));
    else if (ilist)
        CK(c, nb::launch_force_list(f, c->guard, tsplit == 3, st));
    else if (tsplit == kForceBig)
        CK(c, nb::launch_force_big(f, c->guard, ncomp(c) == 6, st));
    else
        CK(c, nb::launch_force(f, c->guard, ncomp(c) == 6, st));
    if (e1) CK(c, cudaEventRecord(e1, st));
    c->n_force++;
    c->n_kernels++;
    return NBODY_OK;
}

// ---- exchange (a2).  Rank r's slice of the exchange buffer holds particles
// [r * slot, (r + 1) * slot) (R#22); both back ends address slices through these two.
// NB_TEST_MUTATE (never set in the product build): deliberately wrong variants that
// tests/test_gpu_exchange.py builds to show the exchange tests detect them --
// 1: slices permuted (rank r addressed at (r + 1) mod world), 2: the local-first launch
// starts at chunk 0 instead of the rank's first local chunk.
#ifndef NB_TEST_MUTATE
#define NB_TEST_MUTATE 0
#endif
size_t slice_begin(const nbody_ctx* c, int r) {
    if (NB_TEST_MUTATE == 1) r = (r + 1) % c->cfg.world;
    return (size_t)r * (size_t)c->sh[0].plan.slot;
}
size_t slice_len(const nbody_ctx* c) { return (size_t)c->sh[0].plan.slot; }

// NCCL: in-place all-gather of every rank's packet slice (and hi/lo tails) on stream st
int gather_packets(nbody_ctx* c, cudaStream_t st) {
    const size_t off = slice_begin(c, c->cfg.rank), len = slice_len(c);
    constexpr size_t kPf = sizeof(JPkt) / sizeof(float), kLf = sizeof(float4) / sizeof(float);
    float* base = reinterpret_cast<float*>(c->pkt);
    CKNCCL(c, nccl().AllGather(base + off * kPf, base, len * kPf, ncclFloat32, c->comm, st));
    if (c->pklo) {
        float* lo = reinterpret_cast<float*>(c->pklo);
        CKNCCL(c, nccl().AllGather(lo + off * kLf, lo, len * kLf, ncclFloat32, c->comm, st));
    }
    return NBODY_OK;
}

// loopback: what the all-gather delivers to shard q -- every other shard's slice, copied
// from that shard's own buffer into q's, one cudaMemcpyAsync per slice
int gather_into(nbody_ctx* c, int q, cudaStream_t st) {
    const size_t len = slice_len(c);
    Shard& d = c->sh[q];
    for (int r = 0; r < c->nshards; ++r) {
        if (r == q) continue;
        const size_t off = slice_begin(c, r);
        CK(c, cudaMemcpyAsync(d.pkt + off, c->sh[r].pkt + off, len * sizeof(JPkt), cudaMemcpyDeviceToDevice, st));
        if (d.pklo)
            CK(c, cudaMemcpyAsync(d.pklo + off, c->sh[r].pklo + off, len * sizeof(float4),
                                  cudaMemcpyDeviceToDevice, st));
    }
    return NBODY_OK;
}

// Chunks of the local-first force launch that overlaps the exchange: one wave of
// (i-block x chunk) work items in the 1024-i CTA shape the launch is pinned to (a
// partial wave would idle SMs until it drains, costing more than the ~10 us gather);
// fewer when the rank has fewer local chunks.  Results do not depend on it.
int32_t overlap_chunks(const nbody_ctx* c, const Shard& s) {
    const int32_t nl = s.c_hi - s.c_lo;
    const int64_t n_ib = (s.n_loc + nb::force_i_per_block() - 1) / nb::force_i_per_block();
    if (nl <= 0 || n_ib <= 0) return 0;
    const int64_t slots = (int64_t)c->sm_count * nb::force_ctas_per_sm(ncomp(c) == 6, s.pklo != nullptr);
    return (int32_t)std::min<int64_t>(nl, std::max<int64_t>(1, slots / n_ib));
}

// exchange the packets every shard's pack kernel wrote and run every shard's force pass:
// local chunks first on the compute stream, overlapping the exchange on the comm stream;
// the remaining chunks on the comm stream right behind the exchange, so that launch is
// ordered after the data it reads but not after the local launch -- its CTAs take SM
// slots as the local launch's CTAs drain instead of waiting for its last wave (two
// stream-ordered launches would pay a partial wave each: C3 at P = 8 ran 8 waves of work
// items for 6.9 waves of work); then the compute stream joins the comm stream.
int exchange_and_force(nbody_ctx* c) {
    Nvtx r("nbody: exchange + force");
    int rc;
    if (use_nccl(c)) {
        Shard& s = c->sh[0];
        CK(c, cudaEventRecord(c->ev_packed, c->stream));
        CK(c, cudaStreamWaitEvent(c->comm_stream, c->ev_packed, 0));
        if ((rc = gather_packets(c, c->comm_stream))) return rc;
        const int32_t f = overlap_chunks(c, s), nch = (int32_t)s.plan.n_chunks;
        if ((rc = launch_force_range(c, s, s.c_lo, f, -1, nullptr, nullptr, kForceBig))) return rc;
        if ((rc = launch_force_range(c, s, (s.c_lo + f) % nch, nch - f, -1, nullptr, nullptr, 0, c->comm_stream)))
            return rc;
        CK(c, cudaEventRecord(c->ev_gathered, c->comm_stream));
        CK(c, cudaStreamWaitEvent(c->stream, c->ev_gathered, 0));
    } else if (c->nshards > 1 && c->loop_concurrent) {
        // loopback, timing form (scripts/project_scaling.py): per shard the rank's streams --
        // the emulated gather (one copy per slice) and the remote launch on the comm stream,
        // concurrent with the local-first launch; shards joined one after another
        for (int q = 0; q < c->nshards; ++q) {
            Shard& s = c->sh[q];
            const int32_t f = overlap_chunks(c, s), nch = (int32_t)s.plan.n_chunks;
            CK(c, cudaEventRecord(c->ev_packed, c->stream));
            CK(c, cudaStreamWaitEvent(c->comm_stream, c->ev_packed, 0));
            if ((rc = gather_into(c, q, c->comm_stream))) return rc;
            if ((rc = launch_force_range(c, s, s.c_lo, f, -1, nullptr, nullptr, kForceBig))) return rc;
            if ((rc = launch_force_range(c, s, (s.c_lo + f) % nch, nch - f, -1, nullptr, nullptr, 0,
                                         c->comm_stream)))
                return rc;
            CK(c, cudaEventRecord(c->ev_gathered, c->comm_stream));
            CK(c, cudaStreamWaitEvent(c->stream, c->ev_gathered, 0));
        }
    } else if (c->nshards > 1) {
        // loopback, checking form (default): per shard the same two launches with the emulated
        // gather strictly between them on one stream, so a local-first launch that reads a
        // remote chunk always reads the previous step's data and a wrong slice offset always
        // lands in the remote launch's input (tests/test_gpu_exchange.py)
        for (int q = 0; q < c->nshards; ++q) {
            Shard& s = c->sh[q];
            const int32_t f = overlap_chunks(c, s), nch = (int32_t)s.plan.n_chunks;
            const int32_t c0 = NB_TEST_MUTATE == 2 ? 0 : s.c_lo;
            if ((rc = launch_force_range(c, s, c0, f, -1, nullptr, nullptr, kForceBig))) return rc;
            if ((rc = gather_into(c, q, c->stream))) return rc;
            if ((rc = launch_force_range(c, s, (c0 + f) % nch, nch - f))) return rc;
        }
    } else {
        Shard& s = c->sh[0];   // world == 1: every packet already sits in the buffer
        if ((rc = launch_force_range(c, s, 0, (int32_t)s.plan.n_chunks))) return rc;
    }
    return NBODY_OK;
}

int ensure_forces(nbody_ctx* c) {
    if (c->have_a0) return NBODY_OK;
    int rc;
    for (auto& s : c->sh) {
        CK(c, nb::launch_pack_state(state_args(c, s), c->stream));
        c->n_kernels++;
    }
    if ((rc = exchange_and_force(c))) return rc;
    for (auto& s : c->sh) {
        CK(c, nb::launch_fold_forces(state_args(c, s), c->stream));
        c->n_kernels++;
    }
    c->have_a0 = true;
    c->predicted = false;
    return NBODY_OK;
}

int check_flags(nbody_ctx* c) {
    unsigned long long h[2];
    CK(c, cudaMemcpyAsync(h, c->flags, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    if (h[1] != ULLONG_MAX)
        return fail(c, NBODY_ENONFINITE, "coincident pair involving particle %llu with eps = 0", h[1]);
    if (h[0] != ULLONG_MAX)
        return fail(c, NBODY_ENONFINITE, "non-finite state at particle %llu", h[0]);
    if (use_nccl(c)) {
        ncclResult_t ar;
        CKNCCL(c, nccl().CommGetAsyncError(c->comm, &ar));
        if (ar != ncclSuccess && ar != ncclInProgress)
            return fail(c, NBODY_ENCCL, "NCCL async error: %s", nccl().GetErrorString(ar));
    }
    return NBODY_OK;
}

// copy the local [3][n_loc_pad] rows of every shard to/from a user
// [3][k] array (k = local count, or n in loopback mode)
enum Rows { ROWS_X, ROWS_V, ROWS_A0, ROWS_J0 };
int copy_rows(nbody_ctx* c, double* user, bool to_user, Rows which, bool* host) {
    int64_t k0 = c->sh.front().plan.i0;
    int64_t k = c->sh.back().plan.i1 - k0;
    *host = !is_device_ptr(user);
    for (auto& s : c->sh) {
        if (s.n_loc <= 0) continue;
        double* dev = which == ROWS_X ? s.x : which == ROWS_V ? s.v : which == ROWS_A0 ? s.a0 : s.j0;
        double* u = user + (s.plan.i0 - k0);
        if (to_user)
            CK(c, cudaMemcpy2DAsync(u, k * 8, dev, s.n_loc_pad * 8, s.n_loc * 8, 3, cudaMemcpyDefault,
                                    c->stream));
        else
            CK(c, cudaMemcpy2DAsync(dev, s.n_loc_pad * 8, u, k * 8, s.n_loc * 8, 3, cudaMemcpyDefault,
                                    c->stream));
    }
    return NBODY_OK;
}

void free_ctx(nbody_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->cfg.device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->step_graph) cudaGraphExecDestroy(c->step_graph);
    if (c->comm && nccl().ok) {
        // a failed context (or a peer that never arrives) must not block here: abort it;
        // a healthy one is finalized (bounded wait) and destroyed
        bool abort = c->sticky != 0;
        if (!abort) {
            const std::string err = c->err;
            abort = nccl_settle(c, nccl().CommFinalize(c->comm), "ncclCommFinalize") != NBODY_OK;
            if (!abort) c->err = err;
        }
        if (abort) nccl().CommAbort(c->comm);
        else nccl().CommDestroy(c->comm);
        c->comm = nullptr;
    }
    for (auto& s : c->sh) {
        if (s.own_pkt) { cudaFree(s.pkt); cudaFree(s.pklo); }
        cudaFree(s.m); cudaFree(s.x); cudaFree(s.v); cudaFree(s.a0); cudaFree(s.j0);
        cudaFree(s.xp); cudaFree(s.vp); cudaFree(s.partial);
        cudaFree(s.T); cudaFree(s.lev); cudaFree(s.ilist);
    }
    cudaFree(c->tnext);
    cudaFree(c->tcur);
    cudaFree(c->nact_cur);
    cudaFree(c->nact);
    cudaFree(c->lvl_cnt);
    cudaFree(c->sel_done);
    cudaFree(c->ctl);
    cudaFree(c->gnodes);
    if (c->block_graph) cudaGraphExecDestroy(c->block_graph);
    if (c->hbuf) cudaFreeHost(c->hbuf);
    cudaFree(c->pkt);
    cudaFree(c->pklo);
    cudaFree(c->eall);
    cudaFree(c->eblk);
    cudaFree(c->eout);
    cudaFree(c->flags);
    for (auto e : c->prof_ev) cudaEventDestroy(e);
    if (c->ev_packed) cudaEventDestroy(c->ev_packed);
    if (c->ev_gathered) cudaEventDestroy(c->ev_gathered);
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

template <class T>
int dalloc(nbody_ctx* c, T** p, size_t count) {
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(c, NBODY_ENOMEM, "cudaMalloc of %zu bytes failed: %s", count * sizeof(T),
                    cudaGetErrorString(e));
    }
    return NBODY_OK;
}

int init_impl(const nbody_config* cfg, const double* m, const double* x, const double* v,
              nbody_ctx* c) {
    int rc;
    const nbody_config& k = *cfg;
    if (!(std::isfinite(k.G) && k.G > 0)) return fail(c, NBODY_EINVAL, "G must be finite and > 0");
    if (!(std::isfinite(k.eps) && k.eps >= 0)) return fail(c, NBODY_EINVAL, "eps must be finite and >= 0");
    if (!(std::isfinite(k.dt) && k.dt > 0)) return fail(c, NBODY_EINVAL, "dt must be finite and > 0");
    if (k.integrator != NBODY_HERMITE4 && k.integrator != NBODY_LEAPFROG_KDK &&
        k.integrator != NBODY_HERMITE4_BLOCK)
        return fail(c, NBODY_EINVAL, "integrator %d not supported", k.integrator);
    if (k.integrator == NBODY_HERMITE4_BLOCK) {
        if (!(std::isfinite(k.eta) && k.eta > 0))
            return fail(c, NBODY_EINVAL, "eta must be finite and > 0 for block time steps");
        if (!(std::isfinite(k.eta_s) && k.eta_s > 0))
            return fail(c, NBODY_EINVAL, "eta_s must be finite and > 0 for block time steps");
        if (k.kmax < 0 || k.kmax > 50) return fail(c, NBODY_EINVAL, "kmax must be in [0, 50]");
    }
    if (!m || !x || !v) return fail(c, NBODY_EINVAL, "m, x and v must be non-NULL");
    if (k.world > 1 && !k.loopback && !k.nccl_id)
        return fail(c, NBODY_EINVAL, "world > 1 needs nccl_id (or loopback)");
    c->cfg = k;
    if (k.integrator == NBODY_HERMITE4_BLOCK && k.kmax == 0) c->cfg.kmax = 20;
    c->n = k.n;
    const char* ng = getenv("NBODY_NO_GRAPH");
    c->use_graph = !(ng && *ng && *ng != '0');
    c->eps2f = (float)(k.eps * k.eps);
    c->guard = c->eps2f < FLT_MIN;   // 0, or subnormal (flushed to 0 by the FTZ force pass)
    if (const char* t = getenv("NBODY_NCCL_TIMEOUT_S"); t && *t && atof(t) > 0) c->nccl_timeout_s = atof(t);
    if (const char* t = getenv("NBODY_LOOPBACK_CONCURRENT"); t && *t && *t != '0') c->loop_concurrent = true;
    c->nshards = k.loopback ? k.world : 1;
    c->sh.resize(c->nshards);
    std::string why;
    for (int s = 0; s < c->nshards; ++s) {
        const int32_t r = k.loopback ? s : k.rank;
        if ((rc = make_plan(k.n, k.world, r, k.jchunks, &c->sh[s].plan, &why)))
            return fail(c, rc, "%s", why.c_str());
    }
    const Plan& p0 = c->sh[0].plan;
    c->L = std::max<int64_t>((int64_t)k.world * p0.slot, p0.n_chunks * p0.chunk);

    CK(c, cudaSetDevice(k.device));
    CK(c, cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, k.device));
    if (k.stream) {
        c->stream = (cudaStream_t)k.stream;
    } else {
        CK(c, cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->own_stream = true;
    }
    CK(c, cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
    CK(c, cudaEventCreateWithFlags(&c->ev_packed, cudaEventDisableTiming));
    CK(c, cudaEventCreateWithFlags(&c->ev_gathered, cudaEventDisableTiming));

    if ((rc = dalloc(c, &c->pkt, (size_t)c->L))) return rc;
    if (k.hilo && (rc = dalloc(c, &c->pklo, (size_t)c->L))) return rc;
    for (int q = 0; q < c->nshards; ++q) {
        Shard& s = c->sh[q];
        if (q == 0) {
            s.pkt = c->pkt;
            s.pklo = c->pklo;
            continue;
        }
        s.own_pkt = true;   // loopback: every shard packs into and reads from its own buffer
        if ((rc = dalloc(c, &s.pkt, (size_t)c->L))) return rc;
        if (k.hilo && (rc = dalloc(c, &s.pklo, (size_t)c->L))) return rc;
    }
    if ((rc = dalloc(c, &c->flags, 5))) return rc;
    if (is_block(c)) {
        if ((rc = dalloc(c, &c->tnext, 1)) || (rc = dalloc(c, &c->tcur, 1)) ||
            (rc = dalloc(c, &c->nact, (size_t)c->nshards)) || (rc = dalloc(c, &c->nact_cur, (size_t)c->nshards)) ||
            (rc = dalloc(c, &c->lvl_cnt, 64)) || (rc = dalloc(c, &c->sel_done, 1)) ||
            (rc = dalloc(c, &c->ctl, 4)) || (rc = dalloc(c, &c->gnodes, 1)))
            return rc;
        CK(c, cudaMemsetAsync(c->ctl, 0, 4 * sizeof(long long), c->stream));
        CK(c, cudaMemsetAsync(c->sel_done, 0, sizeof(unsigned), c->stream));
        CK(c, cudaMallocHost(&c->hbuf, 8 + 4 * (size_t)c->nshards));
    }
    CK(c, cudaMemsetAsync(c->flags, 0xff, 4 * sizeof(unsigned long long), c->stream));
    CK(c, cudaMemsetAsync(c->flags + 4, 0, sizeof(unsigned long long), c->stream));
    for (auto& s : c->sh) {
        CK(c, nb::launch_fill_padding(s.pkt, s.pklo, 0, c->L, c->eps2f, c->stream));
        c->n_kernels++;
    }

    const int64_t ib = nb::force_i_per_block();
    for (auto& s : c->sh) {
        s.n_loc = (int32_t)(s.plan.i1 - s.plan.i0);
        s.n_loc_pad = std::max<int64_t>(ib, ib * ((s.n_loc + ib - 1) / ib));
        const size_t v3 = 3 * (size_t)s.n_loc_pad;
        if ((rc = dalloc(c, &s.m, (size_t)s.n_loc_pad))) return rc;
        if ((rc = dalloc(c, &s.x, v3)) || (rc = dalloc(c, &s.v, v3)) || (rc = dalloc(c, &s.a0, v3)) ||
            (rc = dalloc(c, &s.j0, v3)) || (rc = dalloc(c, &s.xp, v3)) || (rc = dalloc(c, &s.vp, v3)))
            return rc;
        if ((rc = dalloc(c, &s.partial, (size_t)s.plan.n_chunks * ncomp(c) * s.n_loc_pad))) return rc;
        if (is_block(c)) {
            if ((rc = dalloc(c, &s.T, (size_t)s.n_loc_pad)) || (rc = dalloc(c, &s.lev, (size_t)s.n_loc_pad)) ||
                (rc = dalloc(c, &s.ilist, (size_t)s.n_loc_pad)))
                return rc;
            CK(c, cudaMemsetAsync(s.T, 0, (size_t)s.n_loc_pad * sizeof(int64_t), c->stream));
            CK(c, cudaMemsetAsync(s.lev, 0, (size_t)s.n_loc_pad * sizeof(int32_t), c->stream));
        }
        // local chunks: those inside [i0, i0 + slot) of this rank's exchange slice
        const int64_t lo = s.plan.i0 == s.plan.i1 ? 0 : s.plan.i0;
        const int64_t hi = s.plan.i0 == s.plan.i1 ? 0 : s.plan.i0 + s.plan.slot;
        s.c_lo = (int32_t)((lo + s.plan.chunk - 1) / s.plan.chunk);
        s.c_hi = (int32_t)std::min<int64_t>(s.plan.n_chunks, hi / s.plan.chunk);
        if (s.c_hi < s.c_lo) s.c_hi = s.c_lo;
        if (s.n_loc <= 0) continue;
        CK(c, cudaMemcpyAsync(s.m, m + s.plan.i0, s.n_loc * 8, cudaMemcpyDefault, c->stream));
        CK(c, cudaMemcpy2DAsync(s.x, s.n_loc_pad * 8, x + s.plan.i0, k.n * 8, s.n_loc * 8, 3,
                                cudaMemcpyDefault, c->stream));
        CK(c, cudaMemcpy2DAsync(s.v, s.n_loc_pad * 8, v + s.plan.i0, k.n * 8, s.n_loc * 8, 3,
                                cudaMemcpyDefault, c->stream));
        CK(c, nb::launch_validate(state_args(c, s), c->flags + 2, c->stream));
        c->n_kernels++;
    }
    unsigned long long bad[3];
    CK(c, cudaMemcpyAsync(bad, c->flags + 2, sizeof bad, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    if (bad[0] != ULLONG_MAX) return fail(c, NBODY_EINVAL, "mass of particle %llu is not finite and > 0", bad[0]);
    if (bad[1] != ULLONG_MAX) return fail(c, NBODY_EINVAL, "position or velocity of particle %llu is not finite", bad[1]);
    // fp32 range of the pair terms: G m_j / s^{3/2} <= G max(m) / eps^3 must stay far below
    // FLT_MAX (1e30 leaves 8 decades for |v|, the jerk terms and the tile sums); with
    // eps = 0 a pair closer than that range allows is reported as non-finite instead
    double mmax = 0;
    memcpy(&mmax, &bad[2], sizeof mmax);
    if (k.eps > 0 && k.G * mmax / (k.eps * k.eps * k.eps) > 1e30)
        return fail(c, NBODY_EINVAL, "G max(m) / eps^3 = %.3g exceeds the fp32 range of the force pass "
                    "(limit 1e30): increase eps", k.G * mmax / (k.eps * k.eps * k.eps));

    if (k.nccl_id && !k.loopback) {
        NcclApi& api = nccl();
        if (!api.ok) return fail(c, NBODY_ENCCL, "%s", api.why.c_str());
        ncclUniqueId id;
        memcpy(id.internal, k.nccl_id, NCCL_UNIQUE_ID_BYTES);
        ncclConfig_t nc = NCCL_CONFIG_INITIALIZER;
        nc.blocking = 0;   // bounded waits (nccl_settle), abortable
        ncclResult_t r = api.CommInitRankConfig(&c->comm, k.world, id, k.rank, &nc);
        if (r != ncclSuccess && r != ncclInProgress) c->comm = nullptr;   // nothing to abort
        CKNCCL(c, r);
    }
    return NBODY_OK;
}

}  // namespace

// ======================================================================= C-ABI

extern "C" {

int nbody_plan(int64_t n, int32_t world, int32_t rank, int32_t jchunks, int64_t* i0, int64_t* i1,
               int64_t* slot, int64_t* chunk, int64_t* n_chunks) {
    Plan p;
    std::string why;
    int rc = make_plan(n, world, rank, jchunks, &p, &why);
    if (rc) return fail(nullptr, rc, "%s", why.c_str());
    if (i0) *i0 = p.i0;
    if (i1) *i1 = p.i1;
    if (slot) *slot = p.slot;
    if (chunk) *chunk = p.chunk;
    if (n_chunks) *n_chunks = p.n_chunks;
    return NBODY_OK;
}

int nbody_nccl_unique_id(uint8_t out[128]) {
    NcclApi& api = nccl();
    if (!api.ok) return fail(nullptr, NBODY_ENCCL, "%s", api.why.c_str());
    ncclUniqueId id;
    ncclResult_t r = api.GetUniqueId(&id);
    if (r != ncclSuccess) return fail(nullptr, NBODY_ENCCL, "ncclGetUniqueId: %s", api.GetErrorString(r));
    memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
    return NBODY_OK;
}

int nbody_init(const nbody_config* cfg, const double* m, const double* x, const double* v,
               nbody_ctx** out) {
    Nvtx r("nbody_init");
    if (!out) return fail(nullptr, NBODY_EINVAL, "out is NULL");
    *out = nullptr;
    if (!cfg) return fail(nullptr, NBODY_EINVAL, "cfg is NULL");
    nbody_ctx* c = new nbody_ctx();
    int rc = init_impl(cfg, m, x, v, c);
    if (rc) {
        g_last_error = c->err;
        free_ctx(c);
        return rc;
    }
    *out = c;
    return NBODY_OK;
}

int nbody_local_range(const nbody_ctx* c, int64_t* i0, int64_t* i1) {
    if (!c) return fail(nullptr, NBODY_EINVAL, "null context");
    if (i0) *i0 = c->sh.front().plan.i0;
    if (i1) *i1 = c->sh.back().plan.i1;
    return NBODY_OK;
}

int nbody_compute_forces(nbody_ctx* c, double* acc, double* jerk) {
    Nvtx r("nbody_compute_forces");
    GUARD(c);
    int rc;
    c->have_a0 = false;
    if ((rc = ensure_forces(c))) return rc;
    const int64_t k0 = c->sh.front().plan.i0;
    const int64_t k = c->sh.back().plan.i1 - k0;
    bool host = false;
    for (auto& s : c->sh) {
        if (s.n_loc <= 0) continue;
        if (acc) {
            host |= !is_device_ptr(acc);
            CK(c, cudaMemcpy2DAsync(acc + (s.plan.i0 - k0), k * 8, s.a0, s.n_loc_pad * 8, s.n_loc * 8, 3,
                                    cudaMemcpyDefault, c->stream));
        }
        if (jerk) {
            host |= !is_device_ptr(jerk);
            CK(c, cudaMemcpy2DAsync(jerk + (s.plan.i0 - k0), k * 8, s.j0, s.n_loc_pad * 8, s.n_loc * 8,
                                    3, cudaMemcpyDefault, c->stream));
        }
    }
    if (host) return check_flags(c);
    return NBODY_OK;
}

namespace {
// one steady-state step: exchange + force (+ overlap) then fold/correct/predict/pack
int one_step(nbody_ctx* c) {
    int rc;
    if ((rc = exchange_and_force(c))) return rc;
    Nvtx r("nbody: fold + correct + predict + pack");
    for (auto& s : c->sh) {
        CK(c, nb::launch_correct_predict_pack(state_args(c, s), c->stream));
        c->n_kernels++;
    }
    return NBODY_OK;
}
}  // namespace

namespace {
// Block time steps (R#28): nsteps * dt_max of individual Hermite steps.  One block
// step: reset counters, t_next = min(t_i + dt_i) (device reduction, NCCL min over
// ranks), active lists, decide (done = t_next > t_end; statistics), predict + pack
// everything, exchange, force pass over the active slots (count read on the device),
// correct + new levels.  No launch needs a host-side count, so without NCCL the whole
// loop is one CUDA graph with a WHILE node whose condition the decide kernel sets;
// with NCCL (or kernel timing on) the host drives the loop and reads `done`.
// t_next and the active counts start reset (block_begin before the first block step, then
// the last CTA of each block step's corrector)
int block_step_body(nbody_ctx* c, cudaGraphConditionalHandle cond, nb::BlockGraphNodes* nodes) {
    int rc;
    // t_next from the level counts the previous corrector left: derived by the selection
    // pass itself, except with NCCL ranks, where it is each rank's value reduced with MIN
    if (use_nccl(c)) {
        CK(c, nb::launch_block_tnext(state_args(c, c->sh[0]), c->stream));
        CKNCCL(c, nccl().AllReduce(c->tnext, c->tnext, 1, ncclUint64, ncclMin, c->comm, c->stream));
    }
    for (auto& s : c->sh) {
        nb::StateArgs a = state_args(c, s);
        if (decide_fused(c)) {   // the selection pass's last CTA runs the decide step
            a.sel_done = c->sel_done;
            a.cond = cond;
            a.gnodes = nodes;
        }
        CK(c, nb::launch_block_select_predict(a, c->stream));
    }
    if (!decide_fused(c))
        CK(c, nb::launch_block_decide(c->ctl, c->tnext, c->tcur, c->nact, c->nact_cur, c->nshards, cond, nodes,
                                      c->stream));
    return NBODY_OK;
}

// force kernel for a block step with n_i active particles: 2 = scalar tile-split,
// 1 = packed tile-split (needs >= 2 tiles per chunk), 3 = list kernel in 1024-i CTAs
// (from big_min on), 0 = list kernel in 256-i CTAs
bool packed_tsplit_ok(const Shard& s) { return s.plan.chunk >= 2 * nb::kTile && nb::force_tsplit_max() > 0; }
// smallest active count whose 1024-i CTAs fill four waves of the GPU (NBODY_LISTBIG_MIN
// overrides; read per call like the tile-split thresholds).  Swept on C3 and C4 block
// steps: 2 waves (5 120 active at 128 chunks) and 20 000 active (4.3 waves) within
// 0.5 %, from 2 000 active on slower (profiles/r01_listbig_sweep.jsonl).
int32_t list_big_min(const nbody_ctx* c, const Shard& s) {
    const char* e = getenv("NBODY_LISTBIG_MIN");
    if (e && *e) return std::max(1, atoi(e));
    static const int per_sm[2] = {nb::force_ctas_per_sm(true, false), nb::force_ctas_per_sm(true, true)};
    const int64_t waves4 = 4LL * c->sm_count * per_sm[c->pklo != nullptr];
    const int64_t ib = (waves4 + s.plan.n_chunks - 1) / s.plan.n_chunks;   // i-blocks needed
    return (int32_t)std::min<int64_t>(INT32_MAX, ib * nb::force_list_i_per_block(true));
}
int block_force_kind(const nbody_ctx* c, const Shard& s, int64_t n_i) {
    if (n_i <= nb::force_tsplit1_max()) return 2;
    if (packed_tsplit_ok(s) && n_i <= nb::force_tsplit_max()) return 1;
    if (n_i >= list_big_min(c, s)) return 3;
    return 0;
}

// make the force launch just captured on c->stream device-updatable; its handle
int capture_force_node(nbody_ctx* c, cudaGraphDeviceNode_t* out) {
    cudaStreamCaptureStatus st;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    CK(c, cudaStreamGetCaptureInfo(c->stream, &st, nullptr, nullptr, &deps, &nd));
    if (st != cudaStreamCaptureStatusActive || nd != 1)
        return fail(c, NBODY_ECUDA, "block graph: force node not found in the capture");
    cudaLaunchAttributeValue av = {};
    av.deviceUpdatableKernelNode.deviceUpdatable = 1;
    CK(c, cudaGraphKernelNodeSetAttribute(deps[0], cudaLaunchAttributeDeviceUpdatableKernelNode, &av));
    cudaLaunchAttributeValue got = {};
    CK(c, cudaGraphKernelNodeGetAttribute(deps[0], cudaLaunchAttributeDeviceUpdatableKernelNode, &got));
    *out = got.deviceUpdatableKernelNode.devNode;
    return NBODY_OK;
}

// predict, exchange, force on the active sets, correct.  Host loop: n_act[q] are the
// active counts read back, and each shard launches the list or the tile-split force
// kernel by its count.  Graph capture (n_act == nullptr): both launches are captured,
// device-updatable, and the decide kernel enables one of them per block step.
int block_step_rest(nbody_ctx* c, const int32_t* n_act, nb::BlockGraphNodes* nodes) {
    int rc;
    if (use_nccl(c) && (rc = gather_packets(c, c->stream))) return rc;
    for (int q = 0; c->nshards > 1 && q < c->nshards; ++q)
        if ((rc = gather_into(c, q, c->stream))) return rc;
    for (int q = 0; q < c->nshards; ++q) {
        Shard& s = c->sh[q];
        const int32_t n_i = n_act ? n_act[q] : std::max<int32_t>(1, s.n_loc);
        if (n_i <= 0 || s.n_loc <= 0) continue;
        const int32_t nch = (int32_t)s.plan.n_chunks;
        if (nodes) {
            if ((rc = launch_force_range(c, s, 0, nch, n_i, s.ilist, c->nact_cur + q)) ||
                (rc = capture_force_node(c, &nodes->force[q])))
                return rc;
            // the 1024-i list node only where an active set can reach big_min (a disabled
            // node still costs the graph a little every block step)
            nodes->big_min[q] = list_big_min(c, s);
            if (nodes->big_min[q] <= s.n_loc) {
                if ((rc = launch_force_range(c, s, 0, nch, n_i, s.ilist, c->nact_cur + q, 3)) ||
                    (rc = capture_force_node(c, &nodes->force_big[q])))
                    return rc;
            } else {
                nodes->big_min[q] = INT32_MAX;
            }
            nodes->chunks[q] = nch;
            nodes->ts_ok[q] = packed_tsplit_ok(s) ? 1 : 0;
            if (nodes->ts_ok[q] &&
                ((rc = launch_force_range(c, s, 0, nch, n_i, s.ilist, c->nact_cur + q, 1)) ||
                 (rc = capture_force_node(c, &nodes->force_ts[q]))))
                return rc;
            if (nodes->ts1_max > 0 &&
                ((rc = launch_force_range(c, s, 0, nch, n_i, s.ilist, c->nact_cur + q, 2)) ||
                 (rc = capture_force_node(c, &nodes->force_ts1[q]))))
                return rc;
        } else if ((rc = launch_force_range(c, s, 0, nch, n_i, s.ilist, c->nact_cur + q, block_force_kind(c, s, n_i)))) {
            return rc;
        }
    }
    for (int q = 0; q < c->nshards; ++q) CK(c, nb::launch_block_correct(state_args(c, c->sh[q]), c->stream));
    c->n_kernels += (decide_fused(c) ? 0 : 1) + 3 * (int64_t)c->nshards;   // select, force, correct; decide
    return NBODY_OK;
}

int block_run_host(nbody_ctx* c);
int block_run(nbody_ctx* c, int32_t nsteps) {
    int rc;
    const int kmax = c->cfg.kmax;
    if ((int64_t)nsteps > (INT64_MAX >> (kmax + 1)))
        return fail(c, NBODY_EINVAL, "nsteps * 2^kmax overflows the block clock");
    if ((rc = ensure_forces(c))) return rc;
    CK(c, cudaMemsetAsync(c->lvl_cnt, 0, 64 * sizeof(int32_t), c->stream));
    for (auto& s : c->sh) {
        if (c->levels_ok)
            CK(c, nb::launch_block_reset_time(state_args(c, s), c->stream));   // all synchronised
        else
            CK(c, nb::launch_block_init_levels(state_args(c, s), c->stream));
        c->n_kernels++;
    }
    c->levels_ok = true;
    CK(c, nb::launch_block_set_tend(c->ctl, (unsigned long long)nsteps << kmax, c->stream));
    CK(c, nb::launch_block_begin(c->tcur, c->nact, c->nshards, c->stream));
    // NCCL ranks capture the t_next all-reduce and the packet all-gather into the WHILE body
    // too (every rank runs the same number of iterations: done derives from the reduced
    // t_next); if the runtime refuses that capture the host-driven loop is used instead
    const bool graph_ok = !c->block_graph_failed && !c->prof && c->use_graph && c->nshards <= 8 &&
                          c->stream != cudaStreamLegacy && c->stream != cudaStreamPerThread &&
                          c->stream != nullptr;
    if (graph_ok) {
        if (!c->block_graph) {
            cudaGraph_t g = nullptr;
            CK(c, cudaGraphCreate(&g, 0));
            cudaGraphConditionalHandle cond;
            cudaGraphNodeParams cp = {};
            cudaGraphNode_t node;
            cudaError_t e = cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault);
            if (e == cudaSuccess) {
                cp.type = cudaGraphNodeTypeConditional;
                cp.conditional.handle = cond;
                cp.conditional.type = cudaGraphCondTypeWhile;
                cp.conditional.size = 1;
                e = cudaGraphAddNode(&node, g, nullptr, 0, &cp);
            }
            if (e == cudaSuccess)
                e = cudaStreamBeginCaptureToGraph(c->stream, cp.conditional.phGraph_out[0], nullptr, nullptr,
                                                  0, cudaStreamCaptureModeThreadLocal);
            if (e != cudaSuccess) {
                cudaGraphDestroy(g);
                CK(c, e);
            }
            const int64_t nk0 = c->n_kernels, nf0 = c->n_force;
            nb::BlockGraphNodes hn = {};
            hn.i_per_block = nb::force_list_i_per_block(false);
            hn.big_i_per_block = nb::force_list_i_per_block(true);
            hn.ts_i_per_block = nb::force_tsplit_i_per_block(false);
            hn.ts1_i_per_block = nb::force_tsplit_i_per_block(true);
            hn.ts_max = nb::force_tsplit_max();
            hn.ts1_max = nb::force_tsplit1_max();
            for (int q = 0; q < 8; ++q) hn.cur[q] = -2, hn.nb[q] = -1;
            rc = block_step_body(c, cond, c->gnodes);
            if (!rc) rc = block_step_rest(c, nullptr, &hn);
            cudaGraph_t body = nullptr;
            e = cudaStreamEndCapture(c->stream, &body);
            c->n_kernels = nk0;
            c->n_force = nf0;
            if (!rc && e == cudaSuccess) e = cudaGraphInstantiate(&c->block_graph, g, 0);
            cudaGraphDestroy(g);
            if (rc) return rc;
            if (e != cudaSuccess && use_nccl(c)) {
                cudaGetLastError();
                c->block_graph = nullptr;
                c->block_graph_failed = true;   // fall through to the host-driven loop
                return block_run_host(c);
            }
            CK(c, e);
            CK(c, cudaMemcpyAsync(c->gnodes, &hn, sizeof hn, cudaMemcpyHostToDevice, c->stream));
            CK(c, cudaStreamSynchronize(c->stream));   // hn is a stack object
        }
        CK(c, cudaGraphLaunch(c->block_graph, c->stream));
        c->block_graph_calls++;
        c->graph_launches++;
        return NBODY_OK;
    }
    return block_run_host(c);
}

// host-driven block-step loop (kernel timing, no capturable stream, or an NCCL capture the
// runtime refused): one host round trip per block step
int block_run_host(nbody_ctx* c) {
    int rc;
    long long* h_done = reinterpret_cast<long long*>(c->hbuf);
    int32_t* h_nact = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(c->hbuf) + 8);
    for (;;) {
        if ((rc = block_step_body(c, cudaGraphConditionalHandle{}, nullptr))) return rc;
        CK(c, cudaMemcpyAsync(h_done, c->ctl + 3, sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
        CK(c, cudaMemcpyAsync(h_nact, c->nact_cur, 4 * (size_t)c->nshards, cudaMemcpyDeviceToHost, c->stream));
        CK(c, cudaStreamSynchronize(c->stream));
        if (*h_done) break;
        if ((rc = block_step_rest(c, h_nact, nullptr))) return rc;
        c->block_host_steps++;
        c->eager_steps++;
    }
    return NBODY_OK;
}
}  // namespace

int nbody_step(nbody_ctx* c, int32_t nsteps) {
    Nvtx r("nbody_step");
    GUARD(c);
    if (nsteps < 1) return fail(c, NBODY_EINVAL, "nsteps must be >= 1");
    int rc;
    if (is_block(c)) return block_run(c, nsteps);
    if ((rc = ensure_forces(c))) return rc;
    if (!c->predicted) {
        for (auto& s : c->sh) {
            CK(c, nb::launch_predict_pack(state_args(c, s), c->stream));
            c->n_kernels++;
        }
        c->predicted = true;
    }
    // Steady-state steps replay one captured CUDA graph (fork/join over the comm
    // stream included) unless kernel timing is on or the stream cannot capture.
    const bool graph_ok = !c->prof && c->use_graph && c->stream != cudaStreamLegacy &&
                          c->stream != cudaStreamPerThread && c->stream != nullptr;
    if (graph_ok && !c->step_graph) {
        const int64_t nk0 = c->n_kernels, nf0 = c->n_force;
        CK(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
        rc = one_step(c);
        cudaGraph_t g = nullptr;
        cudaError_t e = cudaStreamEndCapture(c->stream, &g);
        if (rc) { if (g) cudaGraphDestroy(g); return rc; }
        CK(c, e);
        e = cudaGraphInstantiate(&c->step_graph, g, 0);
        cudaGraphDestroy(g);
        CK(c, e);
        c->graph_kernels = c->n_kernels - nk0;
        c->graph_force = c->n_force - nf0;
        c->n_kernels = nk0;
        c->n_force = nf0;
    }
    for (int32_t t = 0; t < nsteps; ++t) {
        if (graph_ok) {
            CK(c, cudaGraphLaunch(c->step_graph, c->stream));
            c->n_kernels += c->graph_kernels;
            c->n_force += c->graph_force;
            c->graph_launches++;
        } else {
            if ((rc = one_step(c))) return rc;
            c->eager_steps++;
        }
    }
    return NBODY_OK;
}

int nbody_energy(nbody_ctx* c, double* kinetic, double* potential) {
    Nvtx r("nbody_energy");
    GUARD(c);
    int rc;
    if (!c->eall) {
        if ((rc = dalloc(c, &c->eall, (size_t)c->L))) return rc;
        CK(c, cudaMemsetAsync(c->eall, 0, (size_t)c->L * sizeof(double4), c->stream));
        int mb = 1;
        for (auto& s : c->sh) mb = std::max(mb, nb::energy_blocks(s.n_loc));
        if ((rc = dalloc(c, &c->eblk, 2 * (size_t)mb))) return rc;
        c->eblk_cap = mb;
        if ((rc = dalloc(c, &c->eout, 2 * (size_t)std::max(c->nshards, (int)c->cfg.world)))) return rc;
    }
    for (auto& s : c->sh) {
        CK(c, nb::launch_energy_pack(state_args(c, s), c->eall, c->stream));
        c->n_kernels++;
    }
    if (use_nccl(c)) {
        const size_t cnt = (size_t)c->sh[0].plan.slot * 4;
        double* base = reinterpret_cast<double*>(c->eall);
        CKNCCL(c, nccl().AllGather(base + (size_t)c->cfg.rank * cnt, base, cnt, ncclFloat64, c->comm,
                                   c->stream));
    }
    const double eps2 = (double)c->eps2f;
    for (int q = 0; q < c->nshards; ++q) {
        Shard& s = c->sh[q];
        const int slot = use_nccl(c) ? c->cfg.rank : q;
        CK(c, nb::launch_energy(c->eall, c->n, s.plan.i0, s.n_loc, s.v, s.n_loc_pad, s.m, eps2, c->eblk,
                                c->eblk_cap, c->eout + 2 * slot, c->stream));
        c->n_kernels += 2;
    }
    const int nsum = use_nccl(c) ? c->cfg.world : c->nshards;
    if (use_nccl(c)) {
        // gather every rank's (KE, PE) pair (in place); summed on the host in rank order
        CKNCCL(c, nccl().AllGather(c->eout + 2 * c->cfg.rank, c->eout, 2, ncclFloat64, c->comm,
                                   c->stream));
    }
    std::vector<double> h(2 * (size_t)nsum);
    CK(c, cudaMemcpyAsync(h.data(), c->eout, h.size() * 8, cudaMemcpyDeviceToHost, c->stream));
    if ((rc = check_flags(c))) return rc;
    double ke = 0, pe = 0;
    for (int q = 0; q < nsum; ++q) {
        ke += h[2 * q];
        pe += h[2 * q + 1];
    }
    if (kinetic) *kinetic = ke;
    if (potential) *potential = -0.5 * c->cfg.G * pe;
    return NBODY_OK;
}

int nbody_get_state(nbody_ctx* c, double* x, double* v) {
    GUARD(c);
    int rc;
    bool hx = false, hv = false;
    if (x && (rc = copy_rows(c, x, true, ROWS_X, &hx))) return rc;
    if (v && (rc = copy_rows(c, v, true, ROWS_V, &hv))) return rc;
    if (hx || hv) return check_flags(c);
    return NBODY_OK;
}

int nbody_set_state(nbody_ctx* c, const double* x, const double* v, int32_t keep_forces) {
    GUARD(c);
    int rc;
    bool hx = false, hv = false;
    if (x && (rc = copy_rows(c, const_cast<double*>(x), false, ROWS_X, &hx))) return rc;
    if (v && (rc = copy_rows(c, const_cast<double*>(v), false, ROWS_V, &hv))) return rc;
    CK(c, cudaMemsetAsync(c->flags + 2, 0xff, 2 * sizeof(unsigned long long), c->stream));
    for (auto& s : c->sh) {
        CK(c, nb::launch_validate(state_args(c, s), c->flags + 2, c->stream));
        c->n_kernels++;
    }
    unsigned long long bad[2];
    CK(c, cudaMemcpyAsync(bad, c->flags + 2, sizeof bad, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    if (bad[1] != ULLONG_MAX) {
        c->have_a0 = false;
        c->predicted = false;
        return fail(c, NBODY_EINVAL, "position or velocity of particle %llu is not finite", bad[1]);
    }
    if (!keep_forces) {
        c->have_a0 = false;
        c->levels_ok = false;   // block steps: levels restart from eta_s
    }
    c->predicted = false;
    return NBODY_OK;
}

int nbody_get_derivs(nbody_ctx* c, double* acc, double* jerk) {
    GUARD(c);
    int rc;
    if ((rc = ensure_forces(c))) return rc;
    bool ha = false, hj = false;
    if (acc && (rc = copy_rows(c, acc, true, ROWS_A0, &ha))) return rc;
    if (jerk && ncomp(c) == 6 && (rc = copy_rows(c, jerk, true, ROWS_J0, &hj))) return rc;
    if (ha || hj) return check_flags(c);
    return NBODY_OK;
}

int nbody_set_derivs(nbody_ctx* c, const double* acc, const double* jerk) {
    GUARD(c);
    int rc;
    if (!acc || (ncomp(c) == 6 && !jerk))
        return fail(c, NBODY_EINVAL, "acc (and jerk for the Hermite integrators) must be non-NULL");
    bool ha = false, hj = false;
    if ((rc = copy_rows(c, const_cast<double*>(acc), false, ROWS_A0, &ha))) return rc;
    if (ncomp(c) == 6 && (rc = copy_rows(c, const_cast<double*>(jerk), false, ROWS_J0, &hj))) return rc;
    CK(c, cudaMemsetAsync(c->flags + 2, 0xff, 2 * sizeof(unsigned long long), c->stream));
    for (auto& s : c->sh) {
        CK(c, nb::launch_validate_derivs(state_args(c, s), c->flags + 2, c->stream));
        c->n_kernels++;
    }
    unsigned long long bad[2];
    CK(c, cudaMemcpyAsync(bad, c->flags + 2, sizeof bad, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    if (bad[1] != ULLONG_MAX) {
        c->have_a0 = false;
        c->predicted = false;
        return fail(c, NBODY_EINVAL, "acceleration or jerk of particle %llu is not finite", bad[1]);
    }
    c->have_a0 = true;      // the next step starts from these derivatives
    c->predicted = false;
    return NBODY_OK;
}

int nbody_set_levels(nbody_ctx* c, const int32_t* level) {
    GUARD(c);
    if (!is_block(c)) return fail(c, NBODY_EINVAL, "nbody_set_levels needs NBODY_HERMITE4_BLOCK");
    if (!level) return fail(c, NBODY_EINVAL, "level must be non-NULL");
    const int64_t k0 = c->sh.front().plan.i0;
    for (auto& s : c->sh)
        if (s.n_loc > 0)
            CK(c, cudaMemcpyAsync(s.lev, level + (s.plan.i0 - k0), 4 * (size_t)s.n_loc, cudaMemcpyDefault,
                                  c->stream));
    CK(c, cudaMemsetAsync(c->flags + 2, 0xff, 2 * sizeof(unsigned long long), c->stream));
    for (auto& s : c->sh) {
        CK(c, nb::launch_validate_levels(state_args(c, s), c->flags + 2, c->stream));
        c->n_kernels++;
    }
    unsigned long long bad[2];
    CK(c, cudaMemcpyAsync(bad, c->flags + 2, sizeof bad, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    if (bad[1] != ULLONG_MAX) {
        c->levels_ok = false;
        return fail(c, NBODY_EINVAL, "level of particle %llu is outside [0, kmax = %d]", bad[1], c->cfg.kmax);
    }
    c->levels_ok = true;    // the next nbody_step keeps them (no eta_s restart)
    return NBODY_OK;
}

int nbody_block_stats(nbody_ctx* c, int64_t* block_steps, int64_t* active_sum, int32_t* level) {
    GUARD(c);
    if (!is_block(c)) return fail(c, NBODY_EINVAL, "nbody_block_stats needs NBODY_HERMITE4_BLOCK");
    if (level) {
        const int64_t k0 = c->sh.front().plan.i0;
        for (auto& s : c->sh)
            if (s.n_loc > 0)
                CK(c, cudaMemcpyAsync(level + (s.plan.i0 - k0), s.lev, 4 * (size_t)s.n_loc, cudaMemcpyDefault,
                                      c->stream));
    }
    long long h[4];
    CK(c, cudaMemcpyAsync(h, c->ctl, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    if (block_steps) *block_steps = h[1];
    if (active_sum) *active_sum = h[2];
    return NBODY_OK;
}

int nbody_sync(nbody_ctx* c) {
    GUARD(c);
    CK(c, cudaStreamSynchronize(c->comm_stream));
    return check_flags(c);
}

int nbody_prof_enable(nbody_ctx* c, int32_t on) {
    if (!c) return fail(nullptr, NBODY_EINVAL, "null context");
    c->prof = on != 0;
    return NBODY_OK;
}

int nbody_prof_read(nbody_ctx* c, double* force_ms, int64_t* force_launches, int64_t* kernel_launches,
                    int32_t reset) {
    GUARD(c);
    CK(c, cudaStreamSynchronize(c->stream));
    double ms = 0;
    for (size_t q = 0; q + 1 < c->prof_used; q += 2) {
        float t = 0;
        CK(c, cudaEventElapsedTime(&t, c->prof_ev[q], c->prof_ev[q + 1]));
        ms += t;
    }
    if (force_ms) *force_ms = ms;
    int64_t graph_kernels = 0;
    if (is_block(c)) {
        long long steps = 0;
        CK(c, cudaMemcpy(&steps, c->ctl + 1, sizeof steps, cudaMemcpyDeviceToHost));
        const int64_t graph_steps = steps - c->block_steps_at_reset - c->block_host_steps;
        // per block step select, force, correct per shard and decide; per call one last
        // iteration (select, decide, correct) that finds the run done
        const int64_t dk = decide_fused(c) ? 0 : 1;   // a separate decide launch
        graph_kernels = (3 * (int64_t)c->nshards + dk) * graph_steps +
                        (2 * (int64_t)c->nshards + dk) * c->block_graph_calls;
        if (reset) {
            c->block_steps_at_reset = steps;
            c->block_host_steps = 0;
            c->block_graph_calls = 0;
        }
    }
    if (force_launches) *force_launches = c->n_force;
    if (kernel_launches) *kernel_launches = c->n_kernels + graph_kernels;
    if (reset) {
        c->prof_used = 0;
        c->n_force = 0;
        c->n_kernels = 0;
    }
    return NBODY_OK;
}

int nbody_prof_launch_times(nbody_ctx* c, double* ms, int64_t cap, int64_t* count) {
    GUARD(c);
    CK(c, cudaStreamSynchronize(c->stream));
    const int64_t nrec = (int64_t)(c->prof_used / 2);
    for (int64_t q = 0; q < nrec && q < cap && ms; ++q) {
        float t = 0;
        CK(c, cudaEventElapsedTime(&t, c->prof_ev[2 * q], c->prof_ev[2 * q + 1]));
        ms[q] = t;
    }
    if (count) *count = nrec;
    return NBODY_OK;
}

int nbody_prof_launch_sizes(nbody_ctx* c, int64_t* n_i, int64_t* n_j, int64_t cap, int64_t* count) {
    if (!c) return fail(nullptr, NBODY_EINVAL, "null context");
    const int64_t nrec = (int64_t)(c->prof_used / 2);
    for (int64_t q = 0; q < nrec && q < cap; ++q) {
        if (n_i) n_i[q] = c->prof_ni[q];
        if (n_j) n_j[q] = c->prof_nj[q];
    }
    if (count) *count = nrec;
    return NBODY_OK;
}

int nbody_exec_stats(const nbody_ctx* c, int64_t* graph_launches, int64_t* eager_steps) {
    if (!c) return fail(nullptr, NBODY_EINVAL, "null context");
    if (graph_launches) *graph_launches = c->graph_launches;
    if (eager_steps) *eager_steps = c->eager_steps;
    return NBODY_OK;
}

const char* nbody_last_error(const nbody_ctx* c) {
    if (c) return c->err.c_str();
    return g_last_error.c_str();
}

void nbody_destroy(nbody_ctx* c) {
    Nvtx r("nbody_destroy");
    free_ctx(c);
}

}  // extern "C"
