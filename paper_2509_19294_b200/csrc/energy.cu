// energy.cu -- fp64 total-energy diagnostic (off the per-step path).
//
// KE = 1/2 sum_i m_i |v_i|^2 and PE = -G/2 sum_i m_i sum_{j != i} m_j /
// sqrt(|x_j - x_i|^2 + eps^2), computed over the local i against all j
// (readings R#14, R#18; BASELINE.json asks for energy drift, which needs
// fp64 pair terms: C1's drift is ~1e-10).  The per-i sums are reduced per
// block in a fixed tree, then by one block in fixed order, so the result is
// deterministic.
#include "internal.h"

namespace nb {

namespace {

constexpr int kEBlock = 256;
constexpr int kETile = 256;

__global__ void energy_pack_kernel(StateArgs a, double4* eall) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n_loc; i += gridDim.x * blockDim.x) {
        eall[a.i_base + i] = make_double4(a.x[i], a.x[a.n_loc_pad + i], a.x[2 * a.n_loc_pad + i], a.m[i]);
    }
}

__device__ double block_sum(double v, double* sh) {
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    const double r = sh[0];
    __syncthreads();
    return r;
}

// one thread per local i; j streamed through shared memory
__global__ void __launch_bounds__(kEBlock) energy_kernel(const double4* __restrict__ eall, int64_t n,
                                                         int64_t i_base, int n_loc,
                                                         const double* __restrict__ v,
                                                         int64_t n_loc_pad,
                                                         const double* __restrict__ m, double eps2,
                                                         double* block_sums) {
    __shared__ double4 tile[kETile];
    __shared__ double red[kEBlock];
    const int il = blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = il < n_loc;
    const int64_t ig = i_base + il;
    double4 me = make_double4(0, 0, 0, 0);
    if (live) me = eall[ig];
    double pe = 0.0;
    for (int64_t j0 = 0; j0 < n; j0 += kETile) {
        const int64_t jl = j0 + threadIdx.x;
        tile[threadIdx.x] = jl < n ? eall[jl] : make_double4(0, 0, 0, 0);
        __syncthreads();
        const int nj = (int)((n - j0) < kETile ? (n - j0) : kETile);
        for (int k = 0; k < nj; ++k) {
            const double4 q = tile[k];
            const double dx = q.x - me.x, dy = q.y - me.y, dz = q.z - me.z;
            const double s = dx * dx + dy * dy + dz * dz + eps2;
            const double t = q.w * rsqrt(s);
            pe += (j0 + k == ig) ? 0.0 : t;
        }
        __syncthreads();
    }
    double ke = 0.0;
    if (live) {
        const double vx = v[il], vy = v[n_loc_pad + il], vz = v[2 * n_loc_pad + il];
        ke = 0.5 * m[il] * (vx * vx + vy * vy + vz * vz);
        pe = me.w * pe;
    } else {
        pe = 0.0;
    }
    const double bke = block_sum(ke, red);
    const double bpe = block_sum(pe, red);
    if (threadIdx.x == 0) {
        block_sums[2 * blockIdx.x] = bke;
        block_sums[2 * blockIdx.x + 1] = bpe;
    }
}

__global__ void energy_final_kernel(const double* block_sums, int nblocks, double* out2) {
    __shared__ double red[kEBlock];
    double ke = 0.0, pe = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x) {
        ke += block_sums[2 * b];
        pe += block_sums[2 * b + 1];
    }
    const double k = block_sum(ke, red);
    const double p = block_sum(pe, red);
    if (threadIdx.x == 0) {
        out2[0] = k;
        out2[1] = p;  // sum_i m_i sum_{j != i} m_j / r_ij (caller applies -G/2)
    }
}

}  // namespace

int energy_blocks(int32_t n_loc) { return (n_loc + kEBlock - 1) / kEBlock; }

cudaError_t launch_energy_pack(const StateArgs& a, double4* eall, cudaStream_t s) {
    if (a.n_loc <= 0) return cudaSuccess;
    energy_pack_kernel<<<(a.n_loc + 255) / 256, 256, 0, s>>>(a, eall);
    return cudaGetLastError();
}

cudaError_t launch_energy(const double4* eall, int64_t n, int64_t i_base, int32_t n_loc,
                          const double* v, int64_t n_loc_pad, const double* m, double eps2,
                          double* block_sums, int nblocks_max, double* out2, cudaStream_t s) {
    const int nb = energy_blocks(n_loc);
    if (nb > nblocks_max) return cudaErrorInvalidValue;
    if (nb > 0)
        energy_kernel<<<nb, kEBlock, 0, s>>>(eall, n, i_base, n_loc, v, n_loc_pad, m, eps2, block_sums);
    energy_final_kernel<<<1, kEBlock, 0, s>>>(block_sums, nb, out2);
    return cudaGetLastError();
}

}  // namespace nb
