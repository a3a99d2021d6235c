// ubench_fp32.cu -- FP32 pipe microbenchmark that fixes the roofline peak
// denominator ("microbenchmark FFMA vs FFMA2 throughput before
// reporting any %").  Independent dependency chains, full chip, CUDA events,
// SM clock measured in-kernel (clock64 vs %globaltimer).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_fp32 ubench_fp32.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CHAINS 8
constexpr int kIters = 1 << 14;

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <int MODE>
__global__ void __launch_bounds__(256) kern(float* out, float b, float c, unsigned long long* clk) {
    __shared__ float4 sm[256];
    sm[threadIdx.x] = make_float4(threadIdx.x, 1.f, 2.f, 3.f);
    __syncthreads();
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sm);
    float a[CHAINS];
    unsigned long long p[CHAINS];
    for (int k = 0; k < CHAINS; ++k) {
        a[k] = threadIdx.x * 1e-3f + k;
        asm("mov.b64 %0, {%1, %2};" : "=l"(p[k]) : "f"(a[k]), "f"(a[k] + 1.f));
    }
    double dd[CHAINS];
    const double db = 0.999999;
    for (int k = 0; k < CHAINS; ++k) dd[k] = k + threadIdx.x * 1e-3;
    unsigned long long q[CHAINS], r[CHAINS];
    float qs[CHAINS], rs[CHAINS];
    for (int k = 0; k < CHAINS; ++k) {
        qs[k] = 0.999f - k * 1e-4f + threadIdx.x * 1e-7f;
        rs[k] = 1e-3f * k;
        asm("mov.b64 %0, {%1, %2};" : "=l"(q[k]) : "f"(qs[k]), "f"(qs[k] - 1e-5f));
        asm("mov.b64 %0, {%1, %2};" : "=l"(r[k]) : "f"(rs[k]), "f"(rs[k] + 1e-5f));
    }
    unsigned long long bb, cc;
    asm("mov.b64 %0, {%1, %2};" : "=l"(bb) : "f"(b), "f"(b));
    asm("mov.b64 %0, {%1, %2};" : "=l"(cc) : "f"(c), "f"(c));
    long long t0 = clock64();
    unsigned long long g0 = gtimer();
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int k = 0; k < CHAINS; ++k) {
            if (MODE == 0) {  // scalar FFMA
                asm volatile("fma.rn.ftz.f32 %0, %0, %1, %2;" : "+f"(a[k]) : "f"(b), "f"(c));
            } else if (MODE == 1) {  // packed FFMA2, all operands packed
                asm volatile("fma.rn.ftz.f32x2 %0, %0, %1, %2;" : "+l"(p[k]) : "l"(bb), "l"(cc));
            } else if (MODE == 2) {  // FFMA2 + scalar FFMA interleaved 1:1
                asm volatile("fma.rn.ftz.f32x2 %0, %0, %1, %2;" : "+l"(p[k]) : "l"(bb), "l"(cc));
                asm volatile("fma.rn.ftz.f32 %0, %0, %1, %2;" : "+f"(a[k]) : "f"(b), "f"(c));
            } else if (MODE == 3) {  // MUFU.RSQ
                asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(a[k]));
            } else if (MODE == 4) {  // FFMA2 with 4 FFMA2 : 1 MUFU (the force-loop mix)
                asm volatile("fma.rn.ftz.f32x2 %0, %0, %1, %2;" : "+l"(p[k]) : "l"(bb), "l"(cc));
                if ((k & 3) == 0) asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(a[k]));
            } else if (MODE == 5) {  // FADD2
                asm volatile("add.rn.ftz.f32x2 %0, %0, %1;" : "+l"(p[k]) : "l"(cc));
            } else if (MODE == 6) {  // FFMA2, three distinct 64-bit operands every instruction
                asm volatile("fma.rn.ftz.f32x2 %0, %1, %2, %0;" : "+l"(p[k]) : "l"(q[k]), "l"(r[k]));
            } else if (MODE == 7) {  // FFMA2, one operand (q[0]) shared by consecutive instructions
                asm volatile("fma.rn.ftz.f32x2 %0, %1, %2, %0;" : "+l"(p[k]) : "l"(q[0]), "l"(r[k]));
            } else if (MODE == 8) {  // FFMA2 with a broadcast scalar operand (distinct per k)
                unsigned long long sb;
                asm("mov.b64 %0, {%1, %1};" : "=l"(sb) : "f"(a[k]));
                asm volatile("fma.rn.ftz.f32x2 %0, %1, %2, %0;" : "+l"(p[k]) : "l"(q[k]), "l"(sb));
            } else if (MODE == 10) {  // FMUL2 with an immediate operand
                asm volatile("mul.rn.ftz.f32x2 %0, %0, %1;" : "+l"(p[k]) : "l"(0x3f7ff972bf7ff972ull));
            } else if (MODE == 11) {  // FMUL2 with a register pair operand
                asm volatile("mul.rn.ftz.f32x2 %0, %0, %1;" : "+l"(p[k]) : "l"(q[k]));
            } else if (MODE >= 12 && MODE <= 15) {  // FFMA2 + broadcast LDS (128/64/32-bit)
                asm volatile("fma.rn.ftz.f32x2 %0, %0, %1, %2;" : "+l"(p[k]) : "l"(bb), "l"(cc));
                const int every = (MODE == 12 || MODE == 15) ? 8 : 4;
                if (k % every == 0) {
                    const uint32_t addr = sbase + ((it * 16 + k * 16) & 4095);
                    if (MODE == 12 || MODE == 13) {
                        float4 t;
                        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(t.x), "=f"(t.y), "=f"(t.z), "=f"(t.w) : "r"(addr));
                        a[k] += t.x + t.w;
                    } else if (MODE == 14) {
                        float2 t;
                        asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(t.x), "=f"(t.y) : "r"(addr));
                        a[k] += t.x;
                    } else {
                        float4 t;
                        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(t.x), "=f"(t.y), "=f"(t.z), "=f"(t.w) : "r"(addr));
                        a[k] = t.x;   // consume without FMA-pipe work (MODE 15)
                    }
                }
            } else if (MODE == 16) {  // DFMA only
                asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(dd[k]) : "d"(db));
            } else if (MODE == 17) {  // FFMA2 + DFMA 1:1 (independent chains)
                asm volatile("fma.rn.ftz.f32x2 %0, %0, %1, %2;" : "+l"(p[k]) : "l"(bb), "l"(cc));
                asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(dd[k]) : "d"(db));
            } else if (MODE == 18) {  // FFMA2 + DFMA 2:1
                asm volatile("fma.rn.ftz.f32x2 %0, %0, %1, %2;" : "+l"(p[k]) : "l"(bb), "l"(cc));
                if (k & 1) asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(dd[k]) : "d"(db));
            } else if (MODE == 19) {  // FFMA2 / FMUL2 / FADD2 round robin (independent chains)
                if (k % 3 == 0) asm volatile("fma.rn.ftz.f32x2 %0, %0, %1, %2;" : "+l"(p[k]) : "l"(bb), "l"(cc));
                if (k % 3 == 1) asm volatile("mul.rn.ftz.f32x2 %0, %0, %1;" : "+l"(p[k]) : "l"(bb));
                if (k % 3 == 2) asm volatile("add.rn.ftz.f32x2 %0, %0, %1;" : "+l"(p[k]) : "l"(cc));
            } else if (MODE == 20) {  // the force loop's dependency shape: 3-deep FFMA2 chains x 8, + MUFU per 13
                unsigned long long t1, t2;
                asm volatile("add.rn.ftz.f32x2 %0, %1, %2;" : "=l"(t1) : "l"(p[k]), "l"(q[k]));
                asm volatile("fma.rn.ftz.f32x2 %0, %1, %1, %2;" : "=l"(t2) : "l"(t1), "l"(cc));
                asm volatile("fma.rn.ftz.f32x2 %0, %1, %2, %0;" : "+l"(p[k]) : "l"(t2), "l"(bb));
            } else if (MODE == 21) {  // 4 FFMA2 : 3 DFMA (hybrid force-loop ratio), independent
                asm volatile("fma.rn.ftz.f32x2 %0, %0, %1, %2;" : "+l"(p[k]) : "l"(bb), "l"(cc));
                if (k % 4 != 3) asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(dd[k]) : "d"(db));
            } else if (MODE == 22) {  // same FP32 work alone
                asm volatile("fma.rn.ftz.f32x2 %0, %0, %1, %2;" : "+l"(p[k]) : "l"(bb), "l"(cc));
            } else if (MODE == 9) {  // scalar FFMA, three distinct registers
                asm volatile("fma.rn.ftz.f32 %0, %1, %2, %0;" : "+f"(a[k]) : "f"(qs[k]), "f"(rs[k]));
            }
        }
    }
    long long t1 = clock64();
    unsigned long long g1 = gtimer();
    float s = 0;
    for (int k = 0; k < CHAINS; ++k) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(p[k]));
        s += a[k] + lo + hi + (float)dd[k];
    }
    if (s == 12345.f) out[0] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        clk[0] = (unsigned long long)(t1 - t0);
        clk[1] = g1 - g0;
    }
}

template <int MODE>
void run(const char* name, double lane_ops_per_inst, int sms, int bps = 8) {
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
    // lane_ops_per_inst = FP32 lane-ops per chain per iteration (MUFU counted only in mode 3)
    const double lane_ops = (double)blocks * threads * kIters * CHAINS * lane_ops_per_inst;
    const double per_sm_clk = lane_ops / (ms * 1e-3) / sms / (ghz * 1e9);
    printf("%-28s bps=%d %8.3f ms  clock %.3f GHz  %7.2f lane-ops/clk/SM  (%.2f T lane-ops/s)\n", name, ms,
           bps, ghz, per_sm_clk, lane_ops / (ms * 1e-3) / 1e12);
    cudaFree(out);
    cudaFree(clk);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("SMs %d\n", sms);
    run<0>("FFMA (scalar)", 1.0, sms);
    run<1>("FFMA2 (packed)", 2.0, sms);
    run<2>("FFMA2+FFMA 1:1", 3.0, sms);
    run<3>("MUFU.RSQ", 1.0, sms);
    run<4>("FFMA2 + MUFU 4:1 (FFMA2 lanes)", 2.0, sms);
    run<5>("FADD2 (packed)", 2.0, sms);
    run<6>("FFMA2 3 distinct pairs", 2.0, sms);
    run<7>("FFMA2 shared A operand", 2.0, sms);
    run<8>("FFMA2 pair x bcast + pair", 2.0, sms);
    run<9>("FFMA 3 distinct regs", 1.0, sms);
    run<10>("FMUL2 immediate", 2.0, sms);
    run<11>("FMUL2 register pair", 2.0, sms);
    run<12>("FFMA2 8 : 1 LDS.128 (+2 FADD)", 2.0, sms);
    run<13>("FFMA2 4 : 1 LDS.128 (+2 FADD)", 2.0, sms);
    run<14>("FFMA2 4 : 1 LDS.64 (+1 FADD)", 2.0, sms);
    run<15>("FFMA2 8 : 1 LDS.128 (no use)", 2.0, sms);
    run<16>("DFMA (fp64 lanes)", 1.0, sms);
    run<17>("FFMA2 + DFMA 1:1 (fp32 lanes)", 2.0, sms);
    run<18>("FFMA2 + DFMA 2:1 (fp32 lanes)", 2.0, sms);
    run<19>("FFMA2/FMUL2/FADD2 mix", 2.0, sms);
    run<20>("FADD2->FFMA2->FFMA2 chains", 6.0, sms);
    for (int b : {1, 2, 8}) {
        run<21>("4 FFMA2 : 3 DFMA (fp32 lanes)", 2.0, sms, b);
        run<22>("FFMA2 alone (fp32 lanes)", 2.0, sms, b);
    }
    for (int b : {1}) {
        run<1>("FFMA2 (packed)", 2.0, sms, b);
        run<20>("FADD2->FFMA2->FFMA2 chains", 6.0, sms, b);
        run<4>("FFMA2 + MUFU 4:1 (FFMA2 lanes)", 2.0, sms, b);
    }
    return 0;
}
