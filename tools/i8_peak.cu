// Dense tcgen05 tensor-pipe peak probe (sm_100a): one CTA per SM, one thread
// issues R back-to-back tcgen05.mma (M=128, N=256, operands from smem
// descriptors, accumulating in TMEM) of the given kind; CUDA-event time over
// the whole grid -> dense TOPS.  kind::i8 (s8 x s8 -> s32, K=32) is the
// "integer tensor-pipe peak" the prefill roofline divides by (bench.py reads
// profiles/i8_peak.json); kind::f16 (bf16, K=16) and kind::f8f6f4 (e4m3,
// K=32) for comparison.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/i8_peak tools/i8_peak.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {  // K-major, no swizzle
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((128 >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((256 >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

template <int KIND>  // 0 i8, 1 bf16, 2 e4m3
__global__ void __launch_bounds__(128, 1) peak(int R, unsigned long long* clk) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) unsigned long long bar;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t d = s_tmem;
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);
    // idesc: D format (bits 4-5: 1 = f32, 2 = s32), A/B format bits 7-9 / 10-12,
    // N >> 3 at bit 17, M >> 4 at bit 24
    constexpr uint32_t N = 256, M = 128;
    constexpr uint32_t idesc = KIND == 0 ? ((2u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24))
                               : KIND == 1 ? ((1u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24))
                                           : ((1u << 4) | ((N >> 3) << 17) | ((M >> 4) << 24));
    const unsigned long long t0 = clock64();
    if (threadIdx.x == 0) {
        const uint64_t a = sdesc(sb), b = sdesc(sb + 16384);
        for (int r = 0; r < R; ++r) {
            if (KIND == 0)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                             "l"(a), "l"(b), "r"(idesc), "r"(r));
            else if (KIND == 1)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                             "l"(a), "l"(b), "r"(idesc), "r"(r));
            else
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                             "l"(a), "l"(b), "r"(idesc), "r"(r));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
        asm volatile("{\n\t.reg .pred P;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W;\n\t}" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
        clk[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem));
    }
}

template <int KIND>
static double run(const char* name, int K, unsigned long long* clk, int sms) {
    const int R = 20000;
    cudaFuncSetAttribute(peak<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    peak<KIND><<<sms, 128, 64 * 1024>>>(R, clk);  // warm-up
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int t = 0; t < 5; ++t) {
        cudaEventRecord(e0);
        peak<KIND><<<sms, 128, 64 * 1024>>>(R, clk);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    unsigned long long c = 0;
    cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
    const double ops = 2.0 * 128 * 256 * K * (double)R * sms;
    const double tops = ops / (best * 1e-3) / 1e12;
    printf("{\"kind\": \"%s\", \"tops\": %.1f, \"mac_per_clk_per_sm\": %.0f, \"ms\": %.3f, \"err\": \"%s\"}\n", name, tops,
           128.0 * 256 * K * R / (double)c, best, cudaGetErrorString(cudaGetLastError()));
    return tops;
}

int main() {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* clk;
    cudaMalloc(&clk, 8 * 1024);
    run<0>("i8", 32, clk, sms);
    run<1>("bf16", 16, clk, sms);
    run<2>("e4m3", 32, clk, sms);
    return 0;
}
