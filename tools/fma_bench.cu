// FP32 FMA-pipe throughput (sm_100a): scalar FFMA (3-register form) vs packed
// FFMA2 / FMUL2 (fma.rn.f32x2), 8 independent chains per thread, W warps per SM.
#include <cstdio>
#include <cstdint>
template <int MODE>
__global__ void k(int iters, float* out, long long* clk) {
    float a[16], b = 1.0001f + threadIdx.x * 1e-7f, c = 0.9999f;
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = i * 0.001f + threadIdx.x * 1e-6f;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {
#pragma unroll
            for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], b, c);
        } else {
#pragma unroll
            for (int i = 0; i < 16; i += 2) {
                uint64_t d = ((uint64_t)__float_as_uint(a[i + 1]) << 32) | __float_as_uint(a[i]);
                const uint64_t bb = ((uint64_t)__float_as_uint(b) << 32) | __float_as_uint(b);
                const uint64_t cc = ((uint64_t)__float_as_uint(c) << 32) | __float_as_uint(c);
                if (MODE == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(d) : "l"(bb), "l"(cc));
                else asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(d) : "l"(bb));
                a[i] = __uint_as_float((uint32_t)d);
                a[i + 1] = __uint_as_float((uint32_t)(d >> 32));
            }
        }
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
int main() {
    float* o; long long* c; cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 148 * 8);
    const char* nm[3] = {"FFMA (scalar)", "FFMA2 (f32x2)", "FMUL2 (f32x2)"};
    for (int mode = 0; mode < 3; ++mode)
        for (int W : {4, 8, 16, 32}) {
            const int iters = 4096;
            if (mode == 0) k<0><<<148, 32 * W>>>(iters, o, c);
            else if (mode == 1) k<1><<<148, 32 * W>>>(iters, o, c);
            else k<2><<<148, 32 * W>>>(iters, o, c);
            cudaDeviceSynchronize();
            long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            const double lane_ops = (double)iters * 16 * 32 * W;  // element-ops per SM
            printf("%-14s warps=%2d: %6.1f element-ops/clk/SM\n", nm[mode], W, lane_ops / h);
        }
}
