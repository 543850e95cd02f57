// Per-SM L2 -> shared-memory ingest rate: each CTA (one per SM) streams a small
// L2-resident buffer into an smem ring with cp.async.bulk (1 producer thread,
// S stages of C bytes), or with LDG.128 by all warps.  Prints B/clk/SM.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void bulk(const uint8_t* src, int chunk, int S, int iters, int nsplit, long long* out) {
    // producer p = warp (lane 0 of each warp), own S-stage ring of chunk bytes
    extern __shared__ __align__(128) uint8_t smem[];
    const int lanes = nsplit;  // nsplit reused: producers are lanes 0..lanes-1 of each warp
    const int P = (blockDim.x / 32) * lanes, p = (threadIdx.x / 32) * lanes + (threadIdx.x & 31);
    uint64_t* full = (uint64_t*)smem + p * 8;
    uint8_t* ring = smem + 1024 + (size_t)p * S * chunk;
    if ((threadIdx.x & 31) < lanes) {
        for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if ((threadIdx.x & 31) >= lanes) return;
    iters /= P;
    const uint8_t* base = src + (size_t)(blockIdx.x % 8) * (1 << 20);
    long long t0 = clock64();
    uint32_t ph = 0;
    int s = 0;
    for (int i = 0; i < iters + S; ++i) {
        if (i >= S) {  // wait for the copy issued S iterations ago
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                             : "=r"(ok) : "r"(smem_u32(&full[s])), "r"(ph ^ 1));
        }
        if (i < iters) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(chunk));
            const int part = chunk;
            for (int k = 0; k < 1; ++k)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(smem_u32(ring + (size_t)s * chunk + k * part)), "l"(base + ((size_t)i * chunk) % (1 << 20) + k * part),
                             "r"(part), "r"(smem_u32(&full[s])) : "memory");
        }
        if (++s == S) { s = 0; ph ^= 1; }
    }
    if (p == 0) out[blockIdx.x] = clock64() - t0;
}
__global__ void ldg(const uint4* src, int iters, long long* out, int* sink) {
    const uint4* base = src + (size_t)(blockIdx.x % 8) * (1 << 16);
    long long t0 = clock64();
    uint32_t acc = 0;
    for (int i = 0; i < iters; ++i) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(base + ((i * 8 + u) * blockDim.x + threadIdx.x) % (1 << 16));
#pragma unroll
        for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
    if (acc == 0x12345) sink[0] = acc;
}
int main() {
    uint8_t* src; cudaMalloc(&src, 16 << 20); cudaMemset(src, 1, 16 << 20);
    long long* out; cudaMalloc(&out, 8 * 1024); int* sink; cudaMalloc(&sink, 4);
    cudaFuncSetAttribute(bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    long long h[1024];
    for (int W : {1, 2})
        for (int lanes : {1, 2, 4, 8})
            for (int chunk : {4096, 16384}) {
                const int S = 2, grid = 148;
                if ((size_t)chunk * S * W * lanes > 200 * 1024) continue;
                const int iters = 800;
                bulk<<<grid, 32 * W, 1024 + chunk * S * W * lanes>>>(src, chunk, S, iters, lanes, out);
                cudaDeviceSynchronize();
                cudaMemcpy(h, out, 8 * grid, cudaMemcpyDeviceToHost);
                long long mx = 0; for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
                printf("bulk warps=%d lanes/warp=%d chunk=%5d S=%d: %6.1f B/clk/SM  %s\n", W, lanes, chunk, S,
                       (double)iters * chunk / mx, cudaGetErrorString(cudaGetLastError()));
            }
    for (int grid : {16, 148})
        for (int bs : {256, 512, 1024}) {
            const int iters = 200;
            ldg<<<grid, bs>>>((const uint4*)src, iters, out, sink);
            cudaDeviceSynchronize();
            cudaMemcpy(h, out, 8 * grid, cudaMemcpyDeviceToHost);
            long long mx = 0; for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
            printf("ldg  grid=%3d block=%4d U=8: %6.1f B/clk/SM\n", grid, bs, (double)iters * 8 * 16 * bs / mx);
        }
}
