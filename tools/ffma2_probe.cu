// Microbenchmark: FP32 FFMA vs packed FFMA2 (fma.rn.f32x2) throughput per SM on sm_100a.
// Each thread runs 8 independent chains; reports FMA/clk/SM for both forms.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kIter = 4096;
__global__ void ffma1(float* out, float a, float b) {
    float x[8];
    for (int k = 0; k < 8; k++) x[k] = threadIdx.x * 1e-3f + k;
    for (int i = 0; i < kIter; i++)
#pragma unroll
        for (int k = 0; k < 8; k++) x[k] = fmaf(x[k], a, b);
    float s = 0; for (int k = 0; k < 8; k++) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void ffma2(float* out, float a, float b) {
    unsigned long long x[4];
    for (int k = 0; k < 4; k++) { float2 f = make_float2(threadIdx.x * 1e-3f + k, k + 0.5f); x[k] = *reinterpret_cast<unsigned long long*>(&f); }
    float2 af = make_float2(a, a), bf = make_float2(b, b);
    unsigned long long A = *reinterpret_cast<unsigned long long*>(&af), B = *reinterpret_cast<unsigned long long*>(&bf);
    for (int i = 0; i < kIter; i++)
#pragma unroll
        for (int k = 0; k < 4; k++) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[k]) : "l"(A), "l"(B));
    float s = 0; for (int k = 0; k < 4; k++) { float2 f = *reinterpret_cast<float2*>(&x[k]); s += f.x + f.y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* out; cudaMalloc(&out, 1 << 26);
    const int blocks = nsm * 8, threads = 256;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int form = 0; form < 2; form++) {
        for (int rep = 0; rep < 3; rep++) {
            cudaEventRecord(e0);
            if (form == 0) ffma1<<<blocks, threads>>>(out, 0.999f, 1e-3f);
            else ffma2<<<blocks, threads>>>(out, 0.999f, 1e-3f);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            const double fmas = (double)blocks * threads * kIter * 8;
            if (rep == 2) printf("%s: %.3f ms, %.1f TFMA/s, %.1f FMA/clk/SM at %d MHz (attr)\n", form ? "FFMA2" : "FFMA ", ms,
                   fmas / ms / 1e9, fmas / (ms * 1e-3) / nsm / (clk * 1e3), clk / 1000);
        }
    }
    return 0;
}
