// Probe: (1) tcgen05.st 16x256b register -> (lane, column) mapping, read back
// with 32x32b; (2) tcgen05.mma kind::f16 with the A operand in TMEM: which half
// of a 32-bit column holds the even k.  Build: nvcc -gencode
// arch=compute_100a,code=sm_100a -std=c++17 -I paper_2603_07904_b200/csrc
// tools/tmem_probe.cu -o /tmp/tmem_probe
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include "dyq_ptx.cuh"
using namespace dyq;

__device__ __forceinline__ void st16x256(uint32_t taddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("tcgen05.st.sync.aligned.16x256b.x1.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(a), "r"(b),
                 "r"(c), "r"(d));
}
__device__ __forceinline__ void st32(uint32_t taddr, const uint32_t* r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
}
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void mma_f16_ta(uint32_t d, uint32_t a_tmem, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a_tmem), "l"(bd), "r"(idesc), "r"(acc));
}

// out1[32 lanes][8 cols]: values read back after a 16x256b store at lane 0 / col 0
// out2[128][8]: D = A (TMEM, 128x16) x B^T (smem, 8x16), N = 8
__global__ void probe(uint32_t* out1, float* out2, const uint16_t* A, const uint16_t* B) {
    __shared__ uint32_t s_tmem;
    __shared__ __align__(128) uint8_t sB[8 * 32];
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) { tc::alloc(ptx::smem_u32(&s_tmem), 64); tc::relinquish(); }
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
    // B canonical K-major no-swizzle: (n>>3)*256 + (k>>3)*128 + (n&7)*16 + (k&7)*2, n < 8
    for (int i = threadIdx.x; i < 8 * 16; i += blockDim.x) {
        const int n = i / 16, k = i % 16;
        *reinterpret_cast<uint16_t*>(sB + (k >> 3) * 128 + (n & 7) * 16 + (k & 7) * 2) = B[n * 16 + k];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tm = s_tmem;
    // (1) 16x256b store from warp 0: value = thread*16 + reg
    if (warp == 0) {
        st16x256(tm + 0, lane * 16 + 0, lane * 16 + 1, lane * 16 + 2, lane * 16 + 3);
        wait_st();
        uint32_t r[8];
        tc::ld8(tm + 0, r);
        tc::wait_ld();
        for (int j = 0; j < 8; ++j) out1[lane * 8 + j] = r[j];
    }
    // (2) A into TMEM columns 16..23 with 32x32b: thread = row m (lane), column j = (A[m][2j], A[m][2j+1])
    {
        const int m = warp * 32 + lane;
        uint32_t r[8];
        for (int j = 0; j < 8; ++j) r[j] = (uint32_t)A[m * 16 + 2 * j] | ((uint32_t)A[m * 16 + 2 * j + 1] << 16);
        st32(tm + ((uint32_t)(warp * 32) << 16) + 16, r);
        wait_st();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mma_f16_ta(tm + 32, tm + 16, tc::smem_desc(ptx::smem_u32(sB), 128, 256), tc::idesc_bf16(128, 8), 0);
        tc::commit(ptx::smem_u32(&bar));
    }
    __syncwarp();
    ptx::mbar_wait(&bar, 0);
    tc::fence_after();
    {
        uint32_t r[8];
        tc::ld8(tm + ((uint32_t)(warp * 32) << 16) + 32, r);
        tc::wait_ld();
        const int m = warp * 32 + lane;
        for (int j = 0; j < 8; ++j) out2[m * 8 + j] = __uint_as_float(r[j]);
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) { tc::fence_after(); tc::dealloc(tm, 64); }
}

static uint16_t f2bf(float f) { uint32_t u; memcpy(&u, &f, 4); return (uint16_t)(u >> 16); }

int main() {
    uint32_t* d1; float* d2; uint16_t *dA, *dB;
    cudaMalloc(&d1, 32 * 8 * 4); cudaMalloc(&d2, 128 * 8 * 4);
    cudaMalloc(&dA, 128 * 16 * 2); cudaMalloc(&dB, 8 * 16 * 2);
    uint16_t hA[128 * 16], hB[8 * 16];
    for (int m = 0; m < 128; ++m) for (int k = 0; k < 16; ++k) hA[m * 16 + k] = f2bf((float)((m * 3 + k * 7) % 11 - 5));
    for (int n = 0; n < 8; ++n) for (int k = 0; k < 16; ++k) hB[n * 16 + k] = f2bf((float)(k == n ? 1 : 0) + (k == 8 + n ? 100 : 0));
    cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
    cudaMemset(d1, 0xff, 32 * 8 * 4);
    probe<<<1, 128>>>(d1, d2, dA, dB);
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    uint32_t h1[256]; float h2[1024];
    cudaMemcpy(h1, d1, sizeof h1, cudaMemcpyDeviceToHost); cudaMemcpy(h2, d2, sizeof h2, cudaMemcpyDeviceToHost);
    printf("(1) 16x256b store: lane: col0..7 = thread*16+reg\n");
    for (int l = 0; l < 16; ++l) {
        printf("lane %2d:", l);
        for (int j = 0; j < 8; ++j) printf(" T%02d.r%d", h1[l * 8 + j] / 16, h1[l * 8 + j] % 16);
        printf("\n");
    }
    // (2) expected with packing low half = even k: D[m][n] = A[m][n] + 100*A[m][8+n]
    int ok_lo = 1, ok_hi = 1;
    for (int m = 0; m < 128; ++m) for (int n = 0; n < 8; ++n) {
        auto a = [&](int k) { return (float)((m * 3 + k * 7) % 11 - 5); };
        float lo = a(n) + 100 * a(8 + n);
        // if the halves were swapped, element k would read A[k^1]
        float hi = a(n ^ 1) + 100 * a((8 + n) ^ 1);
        if (h2[m * 8 + n] != lo) ok_lo = 0;
        if (h2[m * 8 + n] != hi) ok_hi = 0;
    }
    printf("(2) A-in-TMEM mma: even-k-in-low-half %s, swapped %s; D[0][0..3] = %g %g %g %g\n", ok_lo ? "MATCH" : "no",
           ok_hi ? "MATCH" : "no", h2[0], h2[1], h2[2], h2[3]);
    return 0;
}
