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

#include <math.h>

namespace nb {

namespace {

constexpr int kBlock = 256;

__device__ __forceinline__ void flag_bad(unsigned long long* bad, int64_t ig) {
    atomicMin(bad, (unsigned long long)ig);
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
    if (a.pk64) {   // exact fp64 copy for the force kernel's FP64-pipe i-particles
        JPkt64 q;
        q.p = make_double4(x[0], x[1], x[2], gm);
        q.v = make_double4(v[0], v[1], v[2], (double)a.eps2);
        a.pk64[k] = q;
    }
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
                                        const double jk[3]) {
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
    store_packet(a, a.i_base + i, xp, vp, a.G * a.m[i]);
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
        predict(a, i, x, v, ac, jk);
    }
}

// canonical fold: ascending chunk order, fp64 left fold from +0
__device__ __forceinline__ double fold(const StateArgs& a, int k, int i) {
    if (k >= a.ncomp) return 0.0;   // leapfrog: no jerk
    double s = 0.0;
    const double* p = a.partial + (int64_t)k * a.n_loc_pad + i;
    const int64_t stride = (int64_t)a.ncomp * a.n_loc_pad;
    for (int c = 0; c < a.n_chunks; ++c) s += p[c * stride];
    return s;
}

__global__ void fold_forces_kernel(StateArgs a) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n_loc; i += gridDim.x * blockDim.x) {
        bool ok = true;
        for (int c = 0; c < 3; ++c) {
            const double ac = fold(a, c, i), jk = fold(a, 3 + c, i);
            a.a0[c * a.n_loc_pad + i] = ac;
            a.j0[c * a.n_loc_pad + i] = jk;
            ok = ok && isfinite(ac) && isfinite(jk);
        }
        if (!ok) flag_bad(a.bad, a.i_base + i);
    }
}

__global__ void correct_predict_pack_kernel(StateArgs a) {
    const double dt = a.dt, dt2 = dt * dt, dt3 = dt2 * dt, dt4 = dt3 * dt, dt5 = dt4 * dt;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n_loc; i += gridDim.x * blockDim.x) {
        double x[3], v[3], a1[3], j1[3];
        bool ok = true;
        for (int c = 0; c < 3; ++c) {
            const int64_t o = c * a.n_loc_pad + i;
            a1[c] = fold(a, c, i);
            j1[c] = fold(a, 3 + c, i);
            if (a.integrator == 0) {   // Hermite corrector (R#3)
                const double a0 = a.a0[o], j0 = a.j0[o];
                const double a2 = (-6.0 * (a0 - a1[c]) - dt * (4.0 * j0 + 2.0 * j1[c])) / dt2;
                const double a3 = (12.0 * (a0 - a1[c]) + 6.0 * dt * (j0 + j1[c])) / dt3;
                x[c] = a.xp[o] + a2 * dt4 / 24.0 + a3 * dt5 / 120.0;
                v[c] = a.vp[o] + a2 * dt3 / 6.0 + a3 * dt4 / 24.0;
            } else {                   // leapfrog: closing kick
                x[c] = a.xp[o];
                v[c] = a.vp[o] + a1[c] * dt / 2.0;
            }
            a.x[o] = x[c];
            a.v[o] = v[c];
            a.a0[o] = a1[c];
            a.j0[o] = j1[c];
            ok = ok && isfinite(x[c]) && isfinite(v[c]) && isfinite(a1[c]) && isfinite(j1[c]);
        }
        if (!ok) flag_bad(a.bad, a.i_base + i);
        predict(a, i, x, v, a1, j1);
    }
}

__global__ void fill_padding_kernel(JPkt* pkt, float4* pklo, JPkt64* pk64, int64_t from, int64_t to,
                                    float eps2) {
    for (int64_t k = from + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < to;
         k += (int64_t)gridDim.x * blockDim.x) {
        // zero mass far away: contributes exactly 0 (padding)
        pkt[k] = make_jpkt(1e18f, 1e18f, 1e18f, 0.f, 0.f, 0.f, 0.f, eps2);
        if (pklo) pklo[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (pk64) {
            JPkt64 q;
            q.p = make_double4(1e18, 1e18, 1e18, 0.0);
            q.v = make_double4(0.0, 0.0, 0.0, (double)eps2);
            pk64[k] = q;
        }
    }
}

__global__ void validate_kernel(StateArgs a, unsigned long long* bad2) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n_loc; i += gridDim.x * blockDim.x) {
        const double mi = a.m[i];
        if (!(isfinite(mi) && mi > 0.0)) flag_bad(&bad2[0], a.i_base + i);
        bool ok = true;
        for (int c = 0; c < 3; ++c)
            ok = ok && isfinite(a.x[c * a.n_loc_pad + i]) && isfinite(a.v[c * a.n_loc_pad + i]);
        if (!ok) flag_bad(&bad2[1], a.i_base + i);
    }
}

unsigned grid_for(int64_t n) {
    int64_t g = (n + kBlock - 1) / kBlock;
    if (g > 148 * 16) g = 148 * 16;
    return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace

cudaError_t launch_validate(const StateArgs& a, unsigned long long* bad2, cudaStream_t s) {
    if (a.n_loc <= 0) return cudaSuccess;
    validate_kernel<<<grid_for(a.n_loc), kBlock, 0, s>>>(a, bad2);
    return cudaGetLastError();
}
cudaError_t launch_pack_state(const StateArgs& a, cudaStream_t s) {
    if (a.n_loc <= 0) return cudaSuccess;
    pack_state_kernel<<<grid_for(a.n_loc), kBlock, 0, s>>>(a);
    return cudaGetLastError();
}
cudaError_t launch_predict_pack(const StateArgs& a, cudaStream_t s) {
    if (a.n_loc <= 0) return cudaSuccess;
    predict_pack_kernel<<<grid_for(a.n_loc), kBlock, 0, s>>>(a);
    return cudaGetLastError();
}
cudaError_t launch_fold_forces(const StateArgs& a, cudaStream_t s) {
    if (a.n_loc <= 0) return cudaSuccess;
    fold_forces_kernel<<<grid_for(a.n_loc), kBlock, 0, s>>>(a);
    return cudaGetLastError();
}
cudaError_t launch_correct_predict_pack(const StateArgs& a, cudaStream_t s) {
    if (a.n_loc <= 0) return cudaSuccess;
    correct_predict_pack_kernel<<<grid_for(a.n_loc), kBlock, 0, s>>>(a);
    return cudaGetLastError();
}
cudaError_t launch_fill_padding(JPkt* pkt, float4* pklo, JPkt64* pk64, int64_t from, int64_t to,
                                float eps2, cudaStream_t s) {
    if (to <= from) return cudaSuccess;
    fill_padding_kernel<<<grid_for(to - from), kBlock, 0, s>>>(pkt, pklo, pk64, from, to, eps2);
    return cudaGetLastError();
}

}  // namespace nb
