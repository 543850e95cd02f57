// kind::f8f6f4 (e4m3 x e4m3 -> f32) probe: (1) clk per MMA at M=128, N=144/256,
// A from SMEM; (2) exactness of integer group sums: A, B hold e4m3 encodings of
// random integers in [-15, 15] (the centred W4 / A2 / A4 codes), K = 64 (two
// MMAs of K = 32); D must equal the exact integer sum (|sum| <= 64 * 225).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include "../paper_2603_07904_b200/csrc/dyq_ptx.cuh"
using namespace dyq;
__host__ __device__ uint8_t e4m3_of_int(int v) {  // exact for |v| <= 15
    if (v == 0) return 0;
    const uint8_t sgn = v < 0 ? 0x80 : 0;
    int a = v < 0 ? -v : v;
    int e = 0;
    while ((a >> e) > 1) ++e;                 // a in [2^e, 2^(e+1))
    const int man = (a - (1 << e)) << (3 - e);  // 3 mantissa bits (e <= 3)
    return sgn | (uint8_t)(((e + 7) << 3) | man);
}
__device__ __forceinline__ void mma_f8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// canonical K-major no-swizzle, 32 B per row per K=32 step: [ks][row>>3][khalf][row&7][16]
__host__ __device__ int koff(int row, int k, int rows) {
    const int ks = k >> 5, kk = k & 31;
    return ks * rows * 32 + (row >> 3) * 256 + (kk >> 4) * 128 + (row & 7) * 16 + (kk & 15);
}
__host__ __device__ constexpr uint32_t idesc_f8(int M, int N) {  // D f32, A e4m3 (0), B e4m3 (0), K-major
    return (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__global__ void probe(const uint8_t* A, const uint8_t* B, int N, int R, float* D, long long* clk) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t s_tmem;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) { tc::alloc(ptx::smem_u32(&s_tmem), 512); tc::relinquish(); }
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
    for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) sm[i] = A[i];
    for (int i = threadIdx.x; i < N * 64; i += blockDim.x) sm[16384 + i] = B[i];
    tc::fence_proxy_async_smem();
    tc::fence_before(); __syncthreads(); tc::fence_after();
    const uint32_t tmem = s_tmem;
    if (threadIdx.x == 0) {
        const uint32_t sa = ptx::smem_u32(sm), sb = sa + 16384;
        const uint32_t id = idesc_f8(128, N);
        long long t0 = clock64();
        for (int r = 0; r < R; ++r)
            for (int ks = 0; ks < 2; ++ks)
                mma_f8(tmem, tc::smem_desc(sa + ks * 128 * 32, 128, 256), tc::smem_desc(sb + ks * N * 32, 128, 256), id,
                       ks > 0 || (r > 0 && R > 1 ? 0 : 0));
        tc::commit(ptx::smem_u32(&bar));
        ptx::mbar_wait(&bar, 0);
        clk[0] = (clock64() - t0) / (2 * R);
    }
    tc::fence_before(); __syncthreads(); tc::fence_after();
    // read D: warp w -> lanes 32w.., 32x32b.x1 per column
    for (int c = 0; c < N; ++c) {
        uint32_t v;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        D[(warp * 32 + (threadIdx.x & 31)) * N + c] = __uint_as_float(v);
    }
    tc::fence_before(); __syncthreads();
    if (warp == 0) { tc::fence_after(); tc::dealloc(tmem, 512); }
}
int main() {
    for (int N : {144, 256}) {
        int* a = new int[128 * 64]; int* b = new int[N * 64];
        uint8_t* ha = new uint8_t[128 * 64]; uint8_t* hb = new uint8_t[N * 64];
        srand(N);
        for (int r = 0; r < 128; ++r) for (int k = 0; k < 64; ++k) {
            a[r * 64 + k] = (r < 8) ? (k % 2 ? 15 : -15) : rand() % 31 - 15;
            ha[koff(r, k, 128)] = e4m3_of_int(a[r * 64 + k]);
        }
        for (int n = 0; n < N; ++n) for (int k = 0; k < 64; ++k) {
            b[n * 64 + k] = (n < 8) ? (k % 2 ? 15 : -15) : rand() % 31 - 15;
            hb[koff(n, k, N)] = e4m3_of_int(b[n * 64 + k]);
        }
        uint8_t *dA, *dB; float* dD; long long* dc;
        cudaMalloc(&dA, 128 * 64); cudaMalloc(&dB, N * 64); cudaMalloc(&dD, 128 * N * 4); cudaMalloc(&dc, 8);
        cudaMemcpy(dA, ha, 128 * 64, cudaMemcpyHostToDevice); cudaMemcpy(dB, hb, N * 64, cudaMemcpyHostToDevice);
        cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        probe<<<1, 128, 48 * 1024>>>(dA, dB, N, 1, dD, dc);
        cudaError_t e = cudaDeviceSynchronize();
        float* D = new float[128 * N]; cudaMemcpy(D, dD, 128 * N * 4, cudaMemcpyDeviceToHost);
        int bad = 0; double maxerr = 0;
        for (int r = 0; r < 128; ++r) for (int n = 0; n < N; ++n) {
            long s = 0; for (int k = 0; k < 64; ++k) s += (long)a[r * 64 + k] * b[n * 64 + k];
            const double err = fabs(D[r * N + n] - (double)s);
            if (err != 0) ++bad;
            if (err > maxerr) maxerr = err;
        }
        printf("N=%d exactness: %d / %d mismatches, max |err| %.1f, D[0]=%.1f (exact %d)  %s\n", N, bad, 128 * N, maxerr,
               D[0], 64 * 225, cudaGetErrorString(e));
        probe<<<148, 128, 48 * 1024>>>(dA, dB, N, 1000, dD, dc);
        cudaDeviceSynchronize();
        long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
        printf("N=%d f8f6f4 K=32: %lld clk/MMA  %.0f MAC/clk/SM\n", N, c, 128.0 * N * 32 / c);
    }
}
