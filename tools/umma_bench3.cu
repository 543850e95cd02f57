// tcgen05.mma issue-rate probe (sm_100a), M=128, N=144, A from TMEM, B SMEM.
// Variants (template V):
//  0: thread 0 only, constant descriptors, one D, K-steps unrolled in pairs
//  1: whole warp loops, MMA inside elect.sync, constant descriptors, one D
//  2: as 1, B descriptor walks a 4-stage ring (runtime, warp-uniform)
//  3: as 2, D cycles over 3 buffers (runtime), 3 MMAs per unit chained
//  4: as 3 with the 3 units' MMAs interleaved (distance 3)
#include <cstdio>
#include <cstdint>
#include "../paper_2603_07904_b200/csrc/dyq_ptx.cuh"
using namespace dyq;
__device__ __forceinline__ uint32_t elect_one() {
    uint32_t p;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(p));
    return p;
}
template <int KIND>
__device__ __forceinline__ void mma(uint32_t d, uint32_t a, uint64_t b, uint32_t acc) {
    if (KIND == 0) tc::mma_f16_ta(d, a, b, tc::idesc_bf16(128, 144), acc);
    else tc::mma_f8_ta(d, a, b, tc::idesc_e4m3(128, 144), acc);
}
template <int KIND, int V>
__global__ void bench(int R, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t s_tmem;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) { tc::alloc(ptx::smem_u32(&s_tmem), 512); tc::relinquish(); }
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = KIND ? 0x38383838u : 0x3f803f80u;
    tc::fence_proxy_async_smem();
    tc::fence_before(); __syncthreads(); tc::fence_after();
    const uint32_t tmem = s_tmem;
    const uint32_t sb = ptx::smem_u32(sm);
    long long t0 = clock64();
    if (V == 0) {
        if (threadIdx.x == 0) {
            const uint64_t b0 = tc::smem_desc(sb, 128, 256), b1 = tc::smem_desc(sb + 8192, 128, 256);
            for (int r = 0; r < R; r += 2) {
                mma<KIND>(tmem, tmem + 480, b0, 1);
                mma<KIND>(tmem, tmem + 488, b1, 1);
            }
            tc::commit(ptx::smem_u32(&bar));
        }
    } else if (warp == 0) {
        const uint32_t e = elect_one();
        if (V == 1) {
            const uint64_t b0 = tc::smem_desc(sb, 128, 256), b1 = tc::smem_desc(sb + 8192, 128, 256);
            for (int r = 0; r < R; r += 2) {
                if (e) mma<KIND>(tmem, tmem + 480, b0, 1);
                if (e) mma<KIND>(tmem, tmem + 488, b1, 1);
                __syncwarp();
            }
        } else if (V == 2) {
            for (int r = 0; r < R; r += 2) {
                const uint32_t st = sb + (r & 3) * 16384;
                if (e) mma<KIND>(tmem, tmem + 480, tc::smem_desc(st, 128, 256), 1);
                if (e) mma<KIND>(tmem, tmem + 488, tc::smem_desc(st + 8192, 128, 256), 1);
                __syncwarp();
            }
        } else if (V == 3) {
            int b = 0;
            for (int r = 0; r < R; r += 3) {
                const uint32_t st = sb + (r & 3) * 16384, d = tmem + b * 144;
                if (e) {
                    mma<KIND>(d, tmem + 464, tc::smem_desc(st, 128, 256), 0);
                    mma<KIND>(d, tmem + 472, tc::smem_desc(st + 8192, 128, 256), 1);
                    mma<KIND>(d, tmem + 480, tc::smem_desc(st + 4096, 128, 256), 1);
                }
                __syncwarp();
                b = b == 2 ? 0 : b + 1;
            }
        } else {
            for (int r = 0; r < R; r += 9) {
                const uint32_t st = sb + (r & 3) * 16384;
                if (e) {
#pragma unroll
                    for (int ks = 0; ks < 3; ++ks)
#pragma unroll
                        for (int u = 0; u < 3; ++u)
                            mma<KIND>(tmem + u * 144, tmem + 464 + ks * 8, tc::smem_desc(st + ks * 4096, 128, 256), ks > 0);
                }
                __syncwarp();
            }
        }
        if (e) tc::commit(ptx::smem_u32(&bar));
        __syncwarp();
    }
    if (threadIdx.x == 0) {
        ptx::mbar_wait(&bar, 0);
        out[blockIdx.x] = clock64() - t0;
    }
    tc::fence_before(); __syncthreads();
    if (warp == 0) { tc::fence_after(); tc::dealloc(tmem, 512); }
}
int main() {
    long long* d; cudaMalloc(&d, 8 * 256);
    auto go = [&](auto kern, const char* nm, int R) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        kern<<<148, 128, 96 * 1024>>>(R, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        printf("%-40s %6.1f clk/MMA (floor 72)  %s\n", nm, (double)h[0] / R, cudaGetErrorString(e));
    };
    go(bench<0, 0>, "bf16 V0 thread0 const", 3600);
    go(bench<0, 1>, "bf16 V1 warp+elect const", 3600);
    go(bench<0, 2>, "bf16 V2 warp+elect ring", 3600);
    go(bench<0, 3>, "bf16 V3 ring, 3 D, chained", 3600);
    go(bench<0, 4>, "bf16 V4 ring, 3 D, interleaved", 3600);
    go(bench<1, 0>, "e4m3 V0 thread0 const", 3600);
    go(bench<1, 1>, "e4m3 V1 warp+elect const", 3600);
    go(bench<1, 2>, "e4m3 V2 warp+elect ring", 3600);
    go(bench<1, 3>, "e4m3 V3 ring, 3 D, chained", 3600);
    go(bench<1, 4>, "e4m3 V4 ring, 3 D, interleaved", 3600);
}
