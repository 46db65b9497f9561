// Micro-benchmark: back-to-back tcgen05.mma kind::f16 (M=128, N, K=16, SS operands in
// shared memory) from one thread into one TMEM accumulator; cycles per MMA vs N, layout,
// and CTAs per SM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo, uint32_t lay) {
    return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) |
           (1ull << 46) | ((uint64_t)lay << 61);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(smem_u32(bar)), "r"(ph) : "memory");
}

template <int N, int LAY>
__global__ void probe(int iters, int per_commit, long long* out) {
    extern __shared__ __align__(1024) char sm[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tm;
    const uint32_t base = (smem_u32(sm) + 1023) & ~1023u;
    for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) ((uint32_t*)(sm + (base - smem_u32(sm))))[i] = 0;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tm)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x == 0) {
        const uint32_t idesc = (1u << 4) | (1u << 15) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint64_t ad = LAY ? desc(base, 4096, 1024, 2) : desc(base, 128, 512, 0);
        const uint64_t bd = desc(base + 8192, 128, 512, 0);
        long long t0 = clock64();
        uint32_t ph = 0;
        for (int i = 0; i < iters; i++) {
            for (int k = 0; k < per_commit; k++) mma(tm, ad + ((k & 1) * (LAY ? 128 : 16)), bd + (k & 1) * 16, idesc, 1u);
            commit(&bar);
            wait(&bar, ph);
            ph ^= 1;
        }
        long long t1 = clock64();
        atomicAdd((unsigned long long*)out, (unsigned long long)(t1 - t0));
    }
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256));
}

// no wait between commits: pure issue stream (the ring is assumed deep)
template <int N, int LAY>
__global__ void probe_stream(int iters, long long* out) {
    extern __shared__ __align__(1024) char sm[];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tm;
    const uint32_t base = (smem_u32(sm) + 1023) & ~1023u;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tm)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x == 0) {
        const uint32_t idesc = (1u << 4) | (1u << 15) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint64_t ad = LAY ? desc(base, 4096, 1024, 2) : desc(base, 128, 512, 0);
        const uint64_t bd = desc(base + 8192, 128, 512, 0);
        long long t0 = clock64();
        for (int i = 0; i < iters; i++) mma(tm, ad + ((i & 1) * (LAY ? 128 : 16)), bd + (i & 1) * 16, idesc, 1u);
        commit(&bar);
        wait(&bar, 0);
        long long t1 = clock64();
        atomicAdd((unsigned long long*)out, (unsigned long long)(t1 - t0));
    }
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256));
}

template <int N, int LAY>
void run(int ctas_per_sm) {
    long long* d;
    cudaMalloc(&d, 8);
    const int smem = 32768;
    cudaFuncSetAttribute(probe_stream<N, LAY>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe<N, LAY>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int grid = 148 * ctas_per_sm, iters = 4096;
    for (int rep = 0; rep < 2; rep++) {
        cudaMemset(d, 0, 8);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        probe_stream<N, LAY><<<grid, 128, smem>>>(iters, d);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        if (rep) printf("stream N=%3d lay=%d cps=%d: %.1f cyc/MMA/stream, wall %.3f ms -> %.1f ns per MMA per SM\n", N, LAY, ctas_per_sm,
                        (double)h / grid / iters, ms, ms * 1e6 / (iters * (double)ctas_per_sm));
    }
    for (int pc : {2, 4, 8}) {
        cudaMemset(d, 0, 8);
        probe<N, LAY><<<grid, 128, smem>>>(iters / pc, pc, d);
        cudaDeviceSynchronize();
        long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("   commit+wait every %d MMAs: %.1f cyc/MMA/stream\n", pc, (double)h / grid / (iters / pc * pc));
    }
    cudaError_t e = cudaGetLastError();
    if (e) printf("err %s\n", cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    run<48, 0>(1); run<48, 2>(1); run<48, 2>(2); run<48, 2>(4);
    run<64, 2>(1); run<128, 2>(1); run<256, 2>(1);
    return 0;
}
