// kind::f8f6f4 probe for the round-2 prefill design (A from TMEM, e4m3):
//  (1) exactness of UNCENTRED weight codes e4m3(q), q in [0, 15], against
//      centred activation codes Bc in [-15, 15] (K = 64: two MMAs), plus a
//      third MMA carrying the zero-point correction -z_w * SXc as base-16
//      digits (A: -z, -16 z, -16 z at the group's window slots; B: d0, d1,
//      16 d2; every other A entry 0, the rest of B arbitrary finite bytes):
//      D must equal Sum_k (q - z) * Bc exactly, incl. |partial sums| ~ 2^15.
//  (2) clk per (group, token tile) of the promotion loop at N = 144 with 8
//      warps (32x32b TMEM loads, s_x broadcast LDS, FMUL2 + FFMA2), with the
//      MMAs of the next units in flight.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include "../paper_2603_07904_b200/csrc/dyq_ptx.cuh"
using namespace dyq;
__host__ __device__ uint8_t e4m3_of_int(int v) {  // exact for the integers used here
    if (v == 0) return 0;
    const uint8_t sgn = v < 0 ? 0x80 : 0;
    int a = v < 0 ? -v : v;
    int e = 0;
    while ((a >> e) > 1) ++e;
    int man = e <= 3 ? (a - (1 << e)) << (3 - e) : (a - (1 << e)) >> (e - 3);
    if (e > 3 && ((a - (1 << e)) & ((1 << (e - 3)) - 1))) return 0x7F;  // not exact -> NaN (flags a bug)
    return sgn | (uint8_t)(((e + 7) << 3) | man);
}
__host__ __device__ constexpr uint32_t idesc_f8(int M, int N) {
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void st32x32_x8(uint32_t t, const uint32_t* r) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(t), "r"(r[0]), "r"(r[1]),
                 "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
// B canonical K-major no-swizzle, one K=32 step: [row>>3][khalf][row&7][16 B]
__host__ __device__ int boff(int row, int kk) { return (row >> 3) * 256 + (kk >> 4) * 128 + (row & 7) * 16 + (kk & 15); }

// A: [128][96] bytes (3 K steps: k 0..63 main, 64..95 corr), B: [3][N][32] canonical
__global__ void exact_probe(const uint8_t* A, const uint8_t* B, int N, float* D) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t s_tmem;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) { tc::alloc(ptx::smem_u32(&s_tmem), 512); tc::relinquish(); }
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
    for (int i = threadIdx.x; i < 3 * N * 32; i += blockDim.x) sm[i] = B[i];
    tc::fence_proxy_async_smem();
    tc::fence_before(); __syncthreads(); tc::fence_after();
    const uint32_t tmem = s_tmem, at = tmem + 256;
    {   // A rows -> TMEM columns 256.. (lane = row, column j = k 4j..4j+3)
        const int row = warp * 32 + lane;
        for (int ks = 0; ks < 3; ++ks) {
            uint32_t r[8];
            for (int j = 0; j < 8; ++j) r[j] = *reinterpret_cast<const uint32_t*>(A + row * 96 + ks * 32 + 4 * j);
            st32x32_x8(at + ((uint32_t)(warp * 32) << 16) + ks * 8, r);
        }
        tc::wait_st();
    }
    tc::fence_before(); __syncthreads(); tc::fence_after();
    if (threadIdx.x == 0) {
        const uint32_t sb = ptx::smem_u32(sm);
        for (int ks = 0; ks < 3; ++ks)
            tc::mma_f8_ta(tmem, at + ks * 8, tc::smem_desc(sb + ks * N * 32, 128, 256), idesc_f8(128, N), ks > 0);
        tc::commit(ptx::smem_u32(&bar));
        ptx::mbar_wait(&bar, 0);
    }
    tc::fence_before(); __syncthreads(); tc::fence_after();
    for (int c = 0; c < N; ++c) {
        uint32_t v;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        D[(warp * 32 + lane) * N + c] = __uint_as_float(v);
    }
    tc::fence_before(); __syncthreads();
    if (warp == 0) { tc::fence_after(); tc::dealloc(tmem, 512); }
}

// promotion-loop timing: 8 promotion warps, 3 accumulator buffers of 144
// columns, one MMA thread keeping them full (A in TMEM, B smem, e4m3, 3 MMAs
// per unit); per unit each promotion thread does 72 columns of its lane.
template <int NW, int MODE>
__global__ void __launch_bounds__(NW * 32 + 64, 1) promo_probe(int units, float* out, long long* clk) {
    constexpr int NCOL = 144 / (NW / 4);  // columns per warp per unit
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t s_tmem;
    __shared__ uint64_t full[3], empty[3];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 3 * 144 * 32; i += blockDim.x) sm[i] = 0x38;  // e4m3 1.0
    float* sx = reinterpret_cast<float*>(sm + 16384);
    for (int i = threadIdx.x; i < 144; i += blockDim.x) sx[i] = 1.0f + i * 1e-3f;
    if (warp == 0) { tc::alloc(ptx::smem_u32(&s_tmem), 512); tc::relinquish(); }
    if (threadIdx.x == 0) {
        for (int b = 0; b < 3; ++b) { ptx::mbar_init(&full[b], 1); ptx::mbar_init(&empty[b], NW); }
        ptx::fence_mbar_init();
    }
    tc::fence_proxy_async_smem();
    tc::fence_before(); __syncthreads(); tc::fence_after();
    const uint32_t tmem = s_tmem;
    long long t0 = clock64();
    if (warp == NW) {
        if (lane == 0 && !(MODE & 4)) {
            const uint32_t sb = ptx::smem_u32(sm);
            for (int u = 0; u < units; ++u) {
                const int b = u % 3;
                if (u >= 3) ptx::mbar_wait(&empty[b], ((u / 3) - 1) & 1);
                tc::fence_after();
                for (int ks = 0; ks < 3; ++ks)
                    tc::mma_f8_ta(tmem + b * 144, tmem + 448 + ks * 8, tc::smem_desc(sb + ks * 144 * 32, 128, 256),
                                  idesc_f8(128, 144), ks > 0);
                tc::commit(ptx::smem_u32(&full[b]));
            }
        }
    } else if (warp < NW) {
        const int q = warp & 3, h = warp >> 2;
        const uint32_t sxa = ptx::smem_u32(sx) + h * NCOL * 4;
        float acc[NCOL];
        for (int i = 0; i < NCOL; ++i) acc[i] = 0.f;
        const float sw = 1.0f + lane * 1e-4f;
        uint32_t v[NCOL];
        for (int i = 0; i < NCOL; ++i) v[i] = __float_as_uint(1.0f + i);
        for (int u = 0; u < units; ++u) {
            const int b = u % 3;
            if (!(MODE & 4)) ptx::mbar_wait(&full[b], (u / 3) & 1);
            tc::fence_after();
            const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16) + b * 144 + h * NCOL;
            if (!(MODE & 2)) {
#pragma unroll
                for (int c = 0; c + 16 <= NCOL; c += 16) tc::ld16(tb + c, *reinterpret_cast<uint32_t(*)[16]>(v + c));
                if (NCOL % 16) tc::ld8(tb + (NCOL / 16) * 16, v + (NCOL / 16) * 16);
                tc::wait_ld();
            }
            tc::fence_before();
            __syncwarp();
            if (lane == 0 && !(MODE & 4)) ptx::mbar_arrive(&empty[b]);
            if (!(MODE & 1))
#pragma unroll
            for (int c = 0; c < NCOL; c += 4) {
                const uint4 s4 = ptx::lds128(sxa + c * 4);
                float t0_, t1_, t2_, t3_;
                ptx::mul2f(t0_, t1_, __uint_as_float(v[c]), __uint_as_float(v[c + 1]), __uint_as_float(s4.x), __uint_as_float(s4.y));
                ptx::mul2f(t2_, t3_, __uint_as_float(v[c + 2]), __uint_as_float(v[c + 3]), __uint_as_float(s4.z), __uint_as_float(s4.w));
                ptx::fma2f(acc[c], acc[c + 1], t0_, t1_, sw, sw);
                ptx::fma2f(acc[c + 2], acc[c + 3], t2_, t3_, sw, sw);
            }
        }
        float s = 0.f;
        for (int i = 0; i < NCOL; ++i) s += acc[i] + __uint_as_float(v[i]);
        out[blockIdx.x * 256 + threadIdx.x] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) clk[blockIdx.x] = clock64() - t0;
    tc::fence_before(); __syncthreads();
    if (warp == 0) { tc::fence_after(); tc::dealloc(tmem, 512); }
}

int main() {
    srand(7);
    const int N = 144;
    int bad_total = 0;
    for (int trial = 0; trial < 6; ++trial) {
        static int q[128][64], z[128], Bc[144][64];
        static uint8_t hA[128 * 96], hB[3 * 144 * 32];
        const int slot = trial % 5;  // the group's window slot: k = 64 + 3 slot + {0, 1, 2}
        for (int r = 0; r < 128; ++r) {
            z[r] = (trial == 1) ? 15 : (trial == 2 ? 0 : rand() % 16);
            for (int k = 0; k < 64; ++k) q[r][k] = (trial <= 2 && r < 16) ? 15 : rand() % 16;
        }
        for (int m = 0; m < N; ++m)
            for (int k = 0; k < 64; ++k)
                Bc[m][k] = (trial <= 2 && m < 16) ? ((m & 1) ? 15 : -15) : rand() % 31 - 15;
        for (int r = 0; r < 128; ++r) {
            for (int k = 0; k < 64; ++k) hA[r * 96 + k] = e4m3_of_int(q[r][k]);
            for (int k = 64; k < 96; ++k) hA[r * 96 + k] = 0;
            hA[r * 96 + 64 + 3 * slot + 0] = e4m3_of_int(-z[r]);
            hA[r * 96 + 64 + 3 * slot + 1] = e4m3_of_int(-16 * z[r]);
            hA[r * 96 + 64 + 3 * slot + 2] = e4m3_of_int(-16 * z[r]);
        }
        for (int m = 0; m < N; ++m) {
            int S = 0;
            for (int k = 0; k < 64; ++k) S += Bc[m][k];
            const int sg = S < 0 ? -1 : 1, a = S < 0 ? -S : S;
            const int d0 = a & 15, d1 = (a >> 4) & 15, d2 = a >> 8;
            for (int k = 0; k < 64; ++k) hB[(k >> 5) * N * 32 + boff(m, k & 31)] = e4m3_of_int(Bc[m][k]);
            for (int kk = 0; kk < 32; ++kk)  // junk (finite) everywhere A is 0
                hB[2 * N * 32 + boff(m, kk)] = e4m3_of_int(rand() % 31 - 15);
            hB[2 * N * 32 + boff(m, 3 * slot + 0)] = e4m3_of_int(sg * d0);
            hB[2 * N * 32 + boff(m, 3 * slot + 1)] = e4m3_of_int(sg * d1);
            hB[2 * N * 32 + boff(m, 3 * slot + 2)] = e4m3_of_int(sg * 16 * d2);
        }
        uint8_t *dA, *dB;
        float* dD;
        cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dD, 128 * N * 4);
        cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
        cudaFuncSetAttribute(exact_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        exact_probe<<<1, 128, 32 * 1024>>>(dA, dB, N, dD);
        const cudaError_t e = cudaDeviceSynchronize();
        static float D[128 * 144];
        cudaMemcpy(D, dD, sizeof D, cudaMemcpyDeviceToHost);
        int bad = 0;
        double maxerr = 0, maxabs = 0;
        for (int r = 0; r < 128; ++r)
            for (int m = 0; m < N; ++m) {
                long s = 0;
                for (int k = 0; k < 64; ++k) s += (long)(q[r][k] - z[r]) * Bc[m][k];
                const double err = fabs(D[r * N + m] - (double)s);
                bad += err != 0;
                maxerr = fmax(maxerr, err);
                maxabs = fmax(maxabs, fabs((double)s));
            }
        bad_total += bad;
        printf("trial %d slot %d: %d / %d mismatches, max err %.1f, max |I| %.0f  %s\n", trial, slot, bad, 128 * N,
               maxerr, maxabs, cudaGetErrorString(e));
        cudaFree(dA); cudaFree(dB); cudaFree(dD);
    }
    printf("EXACT %s\n", bad_total ? "FAIL" : "OK");
    // promotion loop timing
    float* dout;
    long long* dclk;
    cudaMalloc(&dout, 148 * 1024 * 4);
    cudaMalloc(&dclk, 148 * 8);
    auto run = [&](auto kern, int nw, int mode, const char* what) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        const int units = 512;
        kern<<<148, nw * 32 + 64, 20 * 1024>>>(units, dout, dclk);
        const cudaError_t e = cudaDeviceSynchronize();
        long long c[148];
        cudaMemcpy(c, dclk, sizeof c, cudaMemcpyDeviceToHost);
        printf("promotion NW=%2d mode=%d (%s): %.1f clk per 128x144 unit (FMA floor 288)  %s\n", nw, mode, what,
               (double)c[0] / units, cudaGetErrorString(e));
    };
    run(promo_probe<8, 0>, 8, 0, "full");
    run(promo_probe<8, 1>, 8, 1, "no math");
    run(promo_probe<8, 2>, 8, 2, "no TMEM loads");
    run(promo_probe<8, 6>, 8, 6, "math only, no MMA");
    run(promo_probe<8, 4>, 8, 4, "loads+math, no MMA");
    run(promo_probe<16, 0>, 16, 0, "full");
    run(promo_probe<16, 1>, 16, 1, "no math");
    run(promo_probe<16, 6>, 16, 6, "math only, no MMA");
    run(promo_probe<16, 4>, 16, 4, "loads+math, no MMA");
    return 0;
}
