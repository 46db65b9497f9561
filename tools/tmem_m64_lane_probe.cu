// Probe: can tcgen05.mma.cta_group::1.kind::f16 with M = 64 write D at TMEM lane offset 16, and
// where do its rows land?  A[m][k] = (k == 0) ? (m + 1) : 0, B[n][k] = (k == 0) ? 1 : 0, N = 16:
// D[m][n] = m + 1.  Two MMAs: lane offset 0 with +0, lane offset 16 with A scaled by 100.
#include <cuda_fp16.h>
#include <stdint.h>
#include <stdio.h>

__device__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

__global__ void probe(float* out) {
    __shared__ __align__(1024) __half A[2][64 * 16];
    __shared__ __align__(1024) __half B[16 * 16];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tm;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int LBO = 128, SBO = 256;
    for (int s = 0; s < 2; s++) {
        char* a = (char*)A[s];
        for (int e = t; e < 64 * 16; e += blockDim.x) {
            const int mn = e / 16, k = e % 16;
            __half v = __float2half(k == 0 ? (float)(mn + 1) * (s ? 100.f : 1.f) : 0.f);
            *(__half*)(a + (mn / 8) * SBO + (k / 8) * LBO + (k % 8) * 16 + (mn % 8) * 2) = v;
        }
    }
    char* b = (char*)B;
    for (int e = t; e < 16 * 16; e += blockDim.x) {
        const int mn = e / 16, k = e % 16;
        *(__half*)(b + (mn / 8) * SBO + (k / 8) * LBO + (k % 8) * 16 + (mn % 8) * 2) = __float2half(k == 0 ? 1.f : 0.f);
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(su32(&tm)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tm;
    if (t == 0) {
        const uint32_t idesc = (1u << 4) | (1u << 15) | (1u << 16) | ((16u >> 3) << 17) | ((64u >> 4) << 24);
        for (int s = 0; s < 2; s++)
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, 0, 0;\n"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + ((uint32_t)(16 * s) << 16)),
                         "l"(desc(su32(A[s]), LBO, SBO)), "l"(desc(su32(B), LBO, SBO)), "r"(idesc));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    }
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int c = 0; c < 16; c++) out[(warp * 32 + lane) * 16 + c] = __uint_as_float(r[c]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

int main() {
    float* d;
    cudaMalloc(&d, 128 * 16 * 4);
    cudaMemset(d, 0, 128 * 16 * 4);
    float h[128 * 16];
    probe<<<1, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("err=%s\n", cudaGetErrorString(e));
    for (int l = 0; l < 128; l += 1) printf("lane %3d: col0 %8.1f col15 %8.1f\n", l, h[l * 16], h[l * 16 + 15]);
    return 0;
}
