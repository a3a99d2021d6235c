// ubench_operands.cu -- FP32x2 operand-form microbenchmark: does a packed
// FADD2/FFMA2/FMUL2 with a scalar broadcast (.F32) operand run at the full
// packed rate?  (The force loop issues 8 of its 13 packed instructions per
// i-pair and j with the j value as a broadcast operand.)
// Independent chains, full chip, CUDA events, SM clock measured in-kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_operands ubench_operands.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CHAINS 8
constexpr int kIters = 1 << 14;

typedef unsigned long long f2;

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ f2 bc(float a) {
    f2 r;
    asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(a));
    return r;
}

template <int MODE>
__global__ void __launch_bounds__(256) kern(float* out, float b, float c, unsigned long long* clk) {
    f2 p[CHAINS], q[CHAINS], r[CHAINS];
    float s[CHAINS];
    for (int k = 0; k < CHAINS; ++k) {
        const float a = threadIdx.x * 1e-3f + k;
        asm("mov.b64 %0, {%1, %2};" : "=l"(p[k]) : "f"(a), "f"(a + 1.f));
        // per-thread values (not uniform registers), as j data from shared memory are
        const float tq = threadIdx.x * 1e-9f;
        asm("mov.b64 %0, {%1, %2};" : "=l"(q[k]) : "f"(0.999f - k * 1e-4f + tq), "f"(0.998f - tq));
        asm("mov.b64 %0, {%1, %2};" : "=l"(r[k]) : "f"(1e-3f * k + tq), "f"(2e-3f - tq));
        s[k] = b + k * 1e-6f + tq;
    }
    const f2 qs = q[0];
    const float ss = c + threadIdx.x * 1e-9f;
    long long t0 = clock64();
    unsigned long long g0 = gtimer();
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int k = 0; k < CHAINS; ++k) {
            if (MODE == 0) {  // FADD2 pair + pair (shared second operand)
                asm volatile("add.rn.ftz.f32x2 %0, %0, %1;" : "+l"(p[k]) : "l"(qs));
            } else if (MODE == 1) {  // FADD2 broadcast (shared) + pair: the force loop's d = x_j - x_i
                asm volatile("add.rn.ftz.f32x2 %0, %1, %0;" : "+l"(p[k]) : "l"(bc(ss)));
            } else if (MODE == 2) {  // FADD2 broadcast (distinct per chain) + pair
                asm volatile("add.rn.ftz.f32x2 %0, %1, %0;" : "+l"(p[k]) : "l"(bc(s[k])));
            } else if (MODE == 3) {  // FFMA2 pair*pair + broadcast: s = dx*dx + eps2
                asm volatile("fma.rn.ftz.f32x2 %0, %0, %1, %2;" : "+l"(p[k]) : "l"(q[k]), "l"(bc(ss)));
            } else if (MODE == 4) {  // FMUL2 broadcast * pair: m_j * ri
                asm volatile("mul.rn.ftz.f32x2 %0, %1, %0;" : "+l"(p[k]) : "l"(bc(ss)));
            } else if (MODE == 5) {  // FFMA2 three distinct pairs
                asm volatile("fma.rn.ftz.f32x2 %0, %1, %2, %0;" : "+l"(p[k]) : "l"(q[k]), "l"(r[k]));
            } else if (MODE == 6) {  // FFMA2 pair * broadcast (shared) + pair
                asm volatile("fma.rn.ftz.f32x2 %0, %1, %2, %0;" : "+l"(p[k]) : "l"(q[k]), "l"(bc(ss)));
            } else if (MODE == 7) {  // FFMA2 pair * broadcast (distinct) + pair
                asm volatile("fma.rn.ftz.f32x2 %0, %1, %2, %0;" : "+l"(p[k]) : "l"(q[k]), "l"(bc(s[k])));
            } else if (MODE == 8) {  // FFMA2 pair * pair + broadcast (distinct)
                asm volatile("fma.rn.ftz.f32x2 %0, %0, %1, %2;" : "+l"(p[k]) : "l"(q[k]), "l"(bc(s[k])));
            } else if (MODE == 9) {  // FFMA2 p*p + pair (shared addend): s = dy*dy + s
                asm volatile("fma.rn.ftz.f32x2 %0, %1, %1, %0;" : "+l"(p[k]) : "l"(q[k]));
            }
        }
    }
    long long t1 = clock64();
    unsigned long long g1 = gtimer();
    float acc = 0;
    for (int k = 0; k < CHAINS; ++k) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(p[k]));
        acc += lo + hi + s[k];
    }
    if (acc == 12345.f) out[0] = acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        clk[0] = (unsigned long long)(t1 - t0);
        clk[1] = g1 - g0;
    }
}

template <int MODE>
void run(const char* name, int sms, int bps) {
    float* out;
    unsigned long long* clk;
    cudaMalloc(&out, 4);
    cudaMalloc(&clk, 16);
    const int blocks = sms * bps, threads = 256;
    kern<MODE><<<blocks, threads>>>(out, 0.999f, 1e-3f, clk);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<MODE><<<blocks, threads>>>(out, 0.999f, 1e-3f, clk);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[2];
    cudaMemcpy(h, clk, 16, cudaMemcpyDeviceToHost);
    const double ghz = (double)h[0] / (double)h[1];
    const double lane_ops = (double)blocks * threads * kIters * CHAINS * 2.0;
    const double per_sm_clk = lane_ops / (ms * 1e-3) / sms / (ghz * 1e9);
    printf("%-40s warps/SMSP=%2d %8.3f ms  clock %.3f GHz  %7.2f lane-ops/clk/SM\n", name, bps * 2, ms,
           ghz, per_sm_clk);
    cudaFree(out);
    cudaFree(clk);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("SMs %d (peak 128 FP32 lane-ops/clk/SM)\n", sms);
    for (int bps : {8, 1}) {
        run<0>("FADD2 pair + pair(shared)", sms, bps);
        run<1>("FADD2 bcast(shared) + pair", sms, bps);
        run<2>("FADD2 bcast(distinct) + pair", sms, bps);
        run<3>("FFMA2 pair*pair + bcast(shared)", sms, bps);
        run<4>("FMUL2 bcast(shared) * pair", sms, bps);
        run<5>("FFMA2 pair*pair + pair (distinct)", sms, bps);
        run<6>("FFMA2 pair*bcast(shared) + pair", sms, bps);
        run<7>("FFMA2 pair*bcast(distinct) + pair", sms, bps);
        run<8>("FFMA2 pair*pair + bcast(distinct)", sms, bps);
        run<9>("FFMA2 q*q + p", sms, bps);
    }
    return 0;
}
