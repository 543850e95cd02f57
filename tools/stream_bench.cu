// stream_bench.cu -- HBM read-streaming microbenchmark for the decode design.
// Variants: (1) cp.async.bulk into an smem ring (1 producer thread, S stages,
// chunk bytes C), consumers only release; (2) LDG.128 streaming by every warp
// with U independent loads in flight per lane.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_bench tools/stream_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cstdlib>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void bulk_stream(const uint8_t* __restrict__ src, size_t bytes, int chunk, int S, int hint,
                            unsigned long long* sink) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* full = (uint64_t*)smem;
    uint64_t* empty = full + S;
    uint8_t* ring = smem + 128 * ((16 * S + 127) / 128);
    const size_t nchunks = bytes / chunk;
    const size_t per = (nchunks + gridDim.x - 1) / gridDim.x;
    const size_t c0 = blockIdx.x * per, c1 = min(nchunks, c0 + per);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[s])), "r"(blockDim.x / 32 - 1));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    if (warp == 0) {
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (size_t c = c0, i = 0; c < c1; ++c, ++i) {
                if (i >= (size_t)S) {
                    uint32_t ok = 0;
                    while (!ok)
                        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                                     : "=r"(ok) : "r"(smem_u32(&empty[s])), "r"(ph ^ 1) : "memory");
                }
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(chunk));
                if (hint)
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                                 ::"r"(smem_u32(ring + (size_t)s * chunk)), "l"(src + c * chunk), "r"(chunk), "r"(smem_u32(&full[s])), "l"(pol) : "memory");
                else
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                 ::"r"(smem_u32(ring + (size_t)s * chunk)), "l"(src + c * chunk), "r"(chunk), "r"(smem_u32(&full[s])) : "memory");
                if (++s == S) { s = 0; ph ^= 1; }
            }
        }
        return;
    }
    unsigned long long acc = 0;
    int s = 0;
    uint32_t ph = 0;
    for (size_t c = c0; c < c1; ++c) {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                         : "=r"(ok) : "r"(smem_u32(&full[s])), "r"(ph) : "memory");
        acc += ring[(size_t)s * chunk + (warp * 32 + lane) % chunk];
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
        if (++s == S) { s = 0; ph ^= 1; }
    }
    if (acc == 0x1234567) *sink = acc;
}

template <int U>
__global__ void ldg_stream(const uint4* __restrict__ src, size_t n16, unsigned long long* sink) {
    const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t nth = (size_t)gridDim.x * blockDim.x;
    uint32_t acc = 0;
    size_t i = tid;
    for (; i + (U - 1) * nth < n16; i += U * nth) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src + i + u * nth));
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
    for (; i < n16; i += nth) acc ^= src[i].x;
    if (acc == 0x1234567) *sink = acc;
}

// back-to-back launches of a `bytes`-sized stream (decode-layer sized), optional PDL
static void b2b(const uint8_t* buf, size_t bytes, int chunk, int S, int pdl, int sms, unsigned long long* sink) {
    const size_t smem = 128 * ((16 * S + 127) / 128) + (size_t)S * chunk;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms);
    cfg.blockDim = dim3(288);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int R = 40;
    for (int r = 0; r < 3; ++r) cudaLaunchKernelEx(&cfg, bulk_stream, buf + (r % 8) * bytes, bytes, chunk, S, 1, sink);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < R; ++r) cudaLaunchKernelEx(&cfg, bulk_stream, buf + (r % 8) * bytes, bytes, chunk, S, 1, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("b2b bytes=%6.1fMB chunk=%5d S=%2d pdl=%d: %7.2f us/launch %8.1f GB/s\n", bytes / 1e6, chunk, S, pdl,
           ms * 1e3 / R, bytes / (ms / R * 1e-3) / 1e9);
}

int main() {
    const size_t bytes = 1ull << 30;
    uint8_t* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(bulk_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](auto launch, const char* name) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-48s %8.1f GB/s\n", name, 5.0 * bytes / (ms * 1e-3) / 1e9);
    };
    for (size_t mb : {8, 26, 52, 104})
        for (int pdl = 0; pdl < 2; ++pdl)
            b2b(buf, mb * 1000000 / 16384 * 16384, 16384, 6, pdl, sms, sink);
    if (getenv("B2B_ONLY")) return 0;
    char name[128];
    for (int hint = 0; hint < 2; ++hint)
        for (int chunk : {4096, 8192, 16384, 32768})
            for (int ctas : {1, 2, 3, 4})
                for (int kb : {64, 100, 200}) {
                    if (ctas * kb > 224) continue;
                    const int S = (kb * 1024 - 256) / chunk;
                    if (S < 2) continue;
                    const size_t smem = 128 * ((16 * S + 127) / 128) + (size_t)S * chunk;
                    snprintf(name, sizeof name, "bulk hint=%d chunk=%5d ctas/SM=%d S=%2d", hint, chunk, ctas, S);
                    timeit([&] { bulk_stream<<<sms * ctas, 288, smem>>>(buf, bytes, chunk, S, hint, sink); }, name);
                }
    for (int bs : {256, 512}) {
        for (int occ : {2, 4, 8}) {
            snprintf(name, sizeof name, "ldg U=4 block=%d blocks/SM=%d", bs, occ);
            timeit([&] { ldg_stream<4><<<sms * occ, bs>>>((const uint4*)buf, bytes / 16, sink); }, name);
            snprintf(name, sizeof name, "ldg U=8 block=%d blocks/SM=%d", bs, occ);
            timeit([&] { ldg_stream<8><<<sms * occ, bs>>>((const uint4*)buf, bytes / 16, sink); }, name);
        }
    }
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
