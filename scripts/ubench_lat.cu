// ubench_lat.cu -- dependent-chain latency (cycles) of FFMA, FFMA2, MUFU.RSQ, LDS.128 on sm_100a
// (one warp, clock64).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_lat ubench_lat.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int N = 4096;
template <int M>
__global__ void lat(float* out, long long* cyc, float b) {
    __shared__ float4 sm[64];
    if (threadIdx.x < 64) sm[threadIdx.x] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();
    float a = threadIdx.x * 1e-3f + 1.f;
    unsigned long long p;
    asm("mov.b64 %0, {%1, %1};" : "=l"(p) : "f"(a));
    unsigned long long bb;
    asm("mov.b64 %0, {%1, %1};" : "=l"(bb) : "f"(b));
    uint32_t addr = (uint32_t)__cvta_generic_to_shared(sm);
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) {
        if (M == 0) asm volatile("fma.rn.ftz.f32 %0, %0, %1, %1;" : "+f"(a) : "f"(b));
        if (M == 1) asm volatile("fma.rn.ftz.f32x2 %0, %0, %1, %1;" : "+l"(p) : "l"(bb));
        if (M == 2) asm volatile("rsqrt.approx.ftz.f32 %0, %0;" : "+f"(a));
        if (M == 3) {
            float4 t;
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(t.x), "=f"(t.y), "=f"(t.z), "=f"(t.w) : "r"(addr));
            addr += __float_as_uint(t.x);  // dependent address (t.x == 0)
        }
        if (M == 4) asm volatile("add.rn.ftz.f32x2 %0, %0, %1;" : "+l"(p) : "l"(bb));
    }
    long long t1 = clock64();
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(p));
    if (a + lo + hi == 1234.5f) out[0] = a + addr;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int M>
void run(const char* name) {
    float* o; long long* c; long long h;
    cudaMalloc(&o, 4); cudaMalloc(&c, 8);
    lat<M><<<1, 32>>>(o, c, 0.999f);
    lat<M><<<1, 32>>>(o, c, 0.999f);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-12s %6.2f cycles per dependent op\n", name, (double)h / N);
}
int main() { run<0>("FFMA"); run<1>("FFMA2"); run<4>("FADD2"); run<2>("MUFU.RSQ"); run<3>("LDS.128"); return 0; }
