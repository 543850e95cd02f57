// tcgen05.mma kind::f16 / kind::i8 throughput probe (sm_100a): one thread issues
// R back-to-back MMAs (M=128, N in {64,128,144,256}, K step 16 bf16 / 32 i8)
// into one TMEM accumulator, A from TMEM ("ts") or from SMEM ("ss"); B from
// SMEM (K-major, no swizzle).  Prints clk per MMA and MAC/clk/SM.
#include <cstdio>
#include <cstdint>
#include "../paper_2603_07904_b200/csrc/dyq_ptx.cuh"
using namespace dyq;
__device__ __forceinline__ void mma_i8_ta(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc));
}
__global__ void bench(int N, int mode, int R, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t s_tmem;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) { tc::alloc(ptx::smem_u32(&s_tmem), 512); tc::relinquish(); }
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f803f80u;
    tc::fence_before(); __syncthreads(); tc::fence_after();
    const uint32_t tmem = s_tmem;
    long long t0 = 0, t1 = 0;
    if (threadIdx.x == 0) {
        const uint32_t sb = ptx::smem_u32(sm);
        const uint64_t bd = tc::smem_desc(sb, 128, 256);
        const uint64_t ad = tc::smem_desc(sb + 32768, 128, 256);
        const bool i8 = mode >= 2;
        const uint32_t idesc = i8 ? tc::idesc_i8_s8s8(128, N) : tc::idesc_bf16(128, N);
        t0 = clock64();
        for (int r = 0; r < R; ++r) {
            if (mode == 0) tc::mma_f16_ta(tmem, tmem + 256, bd, idesc, r > 0);
            else if (mode == 1) tc::mma_f16(tmem, ad, bd, idesc, r > 0);
            else if (mode == 2) mma_i8_ta(tmem, tmem + 256, bd, idesc, r > 0);
            else tc::mma_i8(tmem, ad, bd, idesc, r > 0);
        }
        tc::commit(ptx::smem_u32(&bar));
        ptx::mbar_wait(&bar, 0);
        t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    tc::fence_before(); __syncthreads();
    if (warp == 0) { tc::fence_after(); tc::dealloc(tmem, 512); }
}
int main() {
    long long* d; cudaMalloc(&d, 8 * 256);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    const char* names[4] = {"f16 A=tmem", "f16 A=smem", "i8 A=tmem", "i8 A=smem"};
    for (int mode = 0; mode < 4; ++mode)
        for (int N : {64, 128, 144, 256}) {
            const int R = 2000;
            bench<<<148, 128, 64 * 1024>>>(N, mode, R, d);
            cudaError_t e = cudaDeviceSynchronize();
            long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
            const double clk = (double)h[0] / R;
            const double kk = mode >= 2 ? 32 : 16;
            printf("%-11s N=%3d: %7.1f clk/MMA  %7.0f MAC/clk/SM  %s\n", names[mode], N, clk, 128.0 * N * kk / clk,
                   cudaGetErrorString(e));
        }
}
