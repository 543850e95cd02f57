// Promotion-loop probe (sm_100a): the prefill kernel's per-group CUDA-core work
// in isolation -- W warps per CTA (one CTA per SM), each warp owns TMEM lane
// quadrant warp % 4 and NC of the 144 accumulator columns; per iteration
// (= one K-group): tcgen05.ld.32x32b of its NC columns, one wait, then
// acc += D * s_x[col] * s_w[row] (FMUL2 + FFMA2) with s_x broadcast from smem.
// Prints clk per iteration; the FMA-pipe floor is 128 * 144 * 2 / 128 = 288.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pb tools/promo_bench.cu
#include <cstdint>
#include <cstdio>

#define LDX(N) "tcgen05.ld.sync.aligned.32x32b.x" #N ".b32 "

template <int N>
__device__ __forceinline__ void tld(uint32_t t, uint32_t* r);
template <>
__device__ __forceinline__ void tld<4>(uint32_t t, uint32_t* r) {
    asm volatile(LDX(4) "{%0,%1,%2,%3}, [%4];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(t));
}
template <>
__device__ __forceinline__ void tld<8>(uint32_t t, uint32_t* r) {
    asm volatile(LDX(8) "{%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(t));
}
template <>
__device__ __forceinline__ void tld<16>(uint32_t t, uint32_t* r) {
    asm volatile(LDX(16) "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(t));
}
template <int N>
__device__ __forceinline__ void tld_n(uint32_t t, uint32_t* r) {  // N multiple of 4
    if constexpr (N >= 16) {
        tld<16>(t, r);
        tld_n<N - 16>(t + 16, r + 16);
    } else if constexpr (N >= 8) {
        tld<8>(t, r);
        tld_n<N - 8>(t + 8, r + 8);
    } else if constexpr (N >= 4) {
        tld<4>(t, r);
    }
}

__device__ __forceinline__ void fma2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
    uint64_t d = ((uint64_t)__float_as_uint(d1) << 32) | __float_as_uint(d0);
    const uint64_t a = ((uint64_t)__float_as_uint(a1) << 32) | __float_as_uint(a0);
    const uint64_t b = ((uint64_t)__float_as_uint(b1) << 32) | __float_as_uint(b0);
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
    d0 = __uint_as_float((uint32_t)d);
    d1 = __uint_as_float((uint32_t)(d >> 32));
}
__device__ __forceinline__ void mul2(float& r0, float& r1, float a0, float a1, float b0, float b1) {
    uint64_t d;
    const uint64_t a = ((uint64_t)__float_as_uint(a1) << 32) | __float_as_uint(a0);
    const uint64_t b = ((uint64_t)__float_as_uint(b1) << 32) | __float_as_uint(b0);
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    r0 = __uint_as_float((uint32_t)d);
    r1 = __uint_as_float((uint32_t)(d >> 32));
}

// MODE 0: packed FMUL2 + FFMA2; 1: scalar FMUL + FFMA; 2: no TMEM load (math only); 3: load only
template <int W, int NC, int MODE, int SPLIT>
__global__ void __launch_bounds__(W * 32, 1) probe(int iters, unsigned long long* out, float* sink) {
    __shared__ uint32_t s_tmem;
    __shared__ __align__(16) float s_x[8][144];
    __shared__ float s_w[8][128];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 8 * 144; i += blockDim.x) (&s_x[0][0])[i] = 1.f + i * 1e-3f;
    for (int i = threadIdx.x; i < 8 * 128; i += blockDim.x) (&s_w[0][0])[i] = 1.f - i * 1e-4f;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int q = warp & 3, c = warp >> 2;
    const int col0 = c * NC;
    const uint32_t tb = s_tmem + ((uint32_t)(q * 32) << 16) + col0;
    float acc[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) acc[i] = 0.f;
    uint32_t v[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) v[i] = __float_as_uint(1.0f + i);
    __syncthreads();
    const long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int s = it & 7;
        const uint32_t tt = tb + (it & 1) * 144 * 0;
        constexpr int CH = NC / SPLIT;
#pragma unroll
        for (int sp = 0; sp < SPLIT; ++sp) {
            if (MODE != 2) {
                tld_n<CH>(tt + sp * CH, v + sp * CH);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            }
            if (MODE != 3) {
                const float sw = s_w[s][q * 32 + lane];
                const float* sx = &s_x[s][col0 + sp * CH];
#pragma unroll
                for (int j = 0; j < CH; j += 4) {
                    const float4 x4 = *reinterpret_cast<const float4*>(sx + j);
                    float* a = acc + sp * CH + j;
                    const uint32_t* d = v + sp * CH + j;
                    if (MODE == 1) {
                        a[0] = fmaf(__uint_as_float(d[0]) * x4.x, sw, a[0]);
                        a[1] = fmaf(__uint_as_float(d[1]) * x4.y, sw, a[1]);
                        a[2] = fmaf(__uint_as_float(d[2]) * x4.z, sw, a[2]);
                        a[3] = fmaf(__uint_as_float(d[3]) * x4.w, sw, a[3]);
                    } else {
                        float t0, t1, t2, t3;
                        mul2(t0, t1, __uint_as_float(d[0]), __uint_as_float(d[1]), x4.x, x4.y);
                        mul2(t2, t3, __uint_as_float(d[2]), __uint_as_float(d[3]), x4.z, x4.w);
                        fma2(a[0], a[1], t0, t1, sw, sw);
                        fma2(a[2], a[3], t2, t3, sw, sw);
                    }
                }
            } else {
                acc[sp] += __uint_as_float(v[sp * CH]);
            }
        }
    }
    const long long c1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(c1 - c0);
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < NC; ++i) t += acc[i];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = t;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem));
}

template <int W, int NC, int MODE, int SPLIT>
void run(const char* name, unsigned long long* d, float* sink) {
    const int iters = 4000;
    probe<W, NC, MODE, SPLIT><<<148, W * 32>>>(iters, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long c[148];
    cudaMemcpy(c, d, sizeof c, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
    printf("%-34s W=%2d NC=%2d split=%d  %.1f clk/group (floor 288)  %s\n", name, W, NC, SPLIT, (double)mx / iters,
           cudaGetErrorString(e));
}

int main1() {
    unsigned long long* d;
    float* sink;
    cudaMalloc(&d, 8 * 2048);
    cudaMalloc(&sink, 4 * 148 * 1024);
    run<8, 72, 0, 1>("packed, 8 warps", d, sink);
    run<8, 72, 0, 2>("packed, 8 warps", d, sink);
    run<8, 72, 1, 1>("scalar, 8 warps", d, sink);
    run<8, 72, 2, 1>("math only, 8 warps", d, sink);
    run<8, 72, 3, 1>("load only, 8 warps", d, sink);
    run<16, 36, 0, 1>("packed, 16 warps", d, sink);
    run<16, 36, 1, 1>("scalar, 16 warps", d, sink);
    run<16, 36, 2, 1>("math only, 16 warps", d, sink);
    run<16, 36, 3, 1>("load only, 16 warps", d, sink);
    run<12, 48, 0, 1>("packed, 12 warps", d, sink);
    run<12, 48, 0, 2>("packed, 12 warps", d, sink);
    run<24, 24, 0, 1>("packed, 24 warps", d, sink);
    run<32, 36, 0, 1>("packed, 32 warps (2 col sets)", d, sink);
    return 0;
}

// ---- 16x256b layout (the prefill kernel's): thread (gid, t) holds rows gid,
// gid + 8 of each 16-row sub-tile and columns 2t, 2t + 1 of each 8-column
// block; one LDS.64 of s_x per block serves 8 elements.
__device__ __forceinline__ void l16_x1(uint32_t t, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(t));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((128 >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((256 >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
// MMAK: 0 none, 1 = one extra warp issues chained kind::f16 128x144x16 MMAs
// (A from TMEM, B from smem) into TMEM columns [160, 304) while the
// promotion warps run; 2 = kind::f8f6f4 (e4m3, K = 32)
template <int W, int NB, int SUBS, int MMAK = 0>
__global__ void __launch_bounds__(W * 32 + (MMAK ? 32 : 0), 1) probe16(int iters, unsigned long long* out, float* sink) {
    __shared__ uint32_t s_tmem;
    __shared__ __align__(1024) uint8_t s_b[16384];
    __shared__ volatile int s_done;
    __shared__ unsigned long long s_nmma;
    __shared__ __align__(8) unsigned long long s_bar;
    __shared__ __align__(16) float s_x[8][144];
    __shared__ __align__(16) float s_w[8][128];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 8 * 144; i += blockDim.x) (&s_x[0][0])[i] = 1.f + i * 1e-3f;
    for (int i = threadIdx.x; i < 8 * 128; i += blockDim.x) (&s_w[0][0])[i] = 1.f - i * 1e-4f;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&s_tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) reinterpret_cast<uint32_t*>(s_b)[i] = 0;
    if (threadIdx.x == 0) {
        s_done = 0;
        s_nmma = 0;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&s_bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (MMAK && warp == W) {
        // MMA issuer: chained 4-step groups until the promotion warps finish
        const uint32_t d = s_tmem + 160, a = s_tmem + 400;
        const uint64_t bd = sdesc((uint32_t)__cvta_generic_to_shared(s_b));
        const uint32_t idesc = MMAK == 1 ? ((1u << 4) | (1u << 7) | (1u << 10) | ((144u >> 3) << 17) | ((128u >> 4) << 24))
                                         : ((1u << 4) | ((144u >> 3) << 17) | ((128u >> 4) << 24));
        unsigned long long n = 0;
        while (!s_done) {
            if (lane == 0) {
                for (int k = 0; k < 4; ++k) {
                    if (MMAK == 1)
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a + 8 * k), "l"(bd), "r"(idesc), "r"(k));
                    else
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a + 8 * k), "l"(bd), "r"(idesc), "r"(k));
                }
                n += 4;
            }
            __syncwarp();
        }
        if (lane == 0) {
            s_nmma = n;
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                (uint32_t)__cvta_generic_to_shared(&s_bar)) : "memory");
            asm volatile("{\n\t.reg .pred P;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra W;\n\t}" ::"r"(
                (uint32_t)__cvta_generic_to_shared(&s_bar)) : "memory");
        }
        __syncwarp();
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        __syncthreads();
        if (warp == 0) {}
        return;
    }
    const int q = warp & 3, c = warp >> 2;
    const int gid = lane >> 2, t = lane & 3;
    const int col0 = (c * NB * 8) % 144;
    const uint32_t tb = s_tmem + ((uint32_t)(q * 32) << 16) + col0;
    float acc[SUBS][NB][4];
#pragma unroll
    for (int s = 0; s < SUBS; ++s)
#pragma unroll
        for (int i = 0; i < NB; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[s][i][j] = 0.f;
    if (MMAK) asm volatile("bar.sync 1, %0;" ::"r"(W * 32)); else __syncthreads();
    
    const long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int s = it & 7;
        uint32_t v[SUBS][NB][4];
#pragma unroll
        for (int si = 0; si < SUBS; ++si)
#pragma unroll
            for (int b = 0; b < NB; ++b) l16_x1(tb + ((uint32_t)(16 * si) << 16) + b * 8, v[si][b]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        float2 sw[SUBS];
#pragma unroll
        for (int si = 0; si < SUBS; ++si)
            sw[si] = *reinterpret_cast<const float2*>(&s_w[s][(2 * q + si) * 16 + 2 * gid]);
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            const float2 sx = *reinterpret_cast<const float2*>(&s_x[s][col0 + b * 8 + 2 * t]);
#pragma unroll
            for (int si = 0; si < SUBS; ++si) {
                float t0, t1, t2, t3;
                float* a = acc[si][b];
                mul2(t0, t1, __uint_as_float(v[si][b][0]), __uint_as_float(v[si][b][1]), sx.x, sx.y);
                mul2(t2, t3, __uint_as_float(v[si][b][2]), __uint_as_float(v[si][b][3]), sx.x, sx.y);
                fma2(a[0], a[1], t0, t1, sw[si].x, sw[si].x);
                fma2(a[2], a[3], t2, t3, sw[si].y, sw[si].y);
            }
        }
    }
    const long long c1 = clock64();
    if (MMAK) {
        asm volatile("bar.sync 1, %0;" ::"r"(W * 32));
        if (threadIdx.x == 0) s_done = 1;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(c1 - c0);
    if (threadIdx.x == 0 && MMAK) out[200 + blockIdx.x] = s_nmma;
    float tt = 0.f;
#pragma unroll
    for (int s = 0; s < SUBS; ++s)
#pragma unroll
        for (int i = 0; i < NB; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) tt += acc[s][i][j];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = tt;
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tmem));
    }
}
template <int W, int NB, int SUBS, int MMAK = 0>
void run16(unsigned long long* d, float* sink) {
    const int iters = 4000;
    probe16<W, NB, SUBS, MMAK><<<148, W * 32 + (MMAK ? 32 : 0)>>>(iters, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long c[148];
    cudaMemcpy(c, d, sizeof c, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
    const double elems = (double)W * 32 * NB * 4 * SUBS;  // per iteration per CTA
    unsigned long long nm = 0;
    if (MMAK) cudaMemcpy(&nm, d + 200, 8, cudaMemcpyDeviceToHost);
    printf("mma=%d (%llu MMAs, %.1f clk each) ", MMAK, nm, nm ? (double)mx / nm : 0.0);
    printf("16x256b W=%2d NB=%d subs=%d: %.1f clk/iter, %.1f clk per 18432 elements (floor 288)  %s\n", W, NB, SUBS,
           (double)mx / iters, (double)mx / iters * 18432.0 / elems, cudaGetErrorString(e));
}
int main2() {
    unsigned long long* d;
    float* sink;
    cudaMalloc(&d, 8 * 2048);
    cudaMalloc(&sink, 4 * 148 * 1024);
    run16<8, 9, 2>(d, sink);
    run16<16, 4, 2>(d, sink);
    run16<16, 5, 2>(d, sink);
    run16<12, 6, 2>(d, sink);
    run16<24, 3, 2>(d, sink);
    run16<16, 9, 1>(d, sink);
    run16<8, 9, 2, 1>(d, sink);
    run16<12, 6, 2, 1>(d, sink);
    run16<16, 4, 2, 1>(d, sink);
    run16<8, 9, 2, 2>(d, sink);
    run16<12, 6, 2, 2>(d, sink);
    return 0;
}
int main() {
    setvbuf(stdout, NULL, _IONBF, 0);
    main1();
    main2();
    return 0;
}
