// dyq_actquant.cu -- dynamic activation quantization (PAPER.md P:220, P:223:
// the step-wise activation switches between BF16 and X in {2,4,8}; Eq. (2) per
// (token, group), reading 6).  Decode layout (see dyq_internal.cuh).
#include "dyq_internal.cuh"

namespace dyq {

// One warp per (token m, group g); M <= DEC_MPAD tokens starting at row m0.
// Rows of the padded tile beyond M and A16 rows get zero codes / params.
__global__ void actquant_dec_kernel(WLayout L, const uint16_t* __restrict__ x, int M, int m0,
                                    const int32_t* __restrict__ row_bits, int bits, uint8_t* __restrict__ xq,
                                    uint2* __restrict__ par, int64_t* err) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= DEC_MPAD * L.NG) return;
    const int m = warp / L.NG, g = warp % L.NG;
    uint8_t* dst = xq + (size_t)m * L.K + (size_t)g * L.G;
    uint2* pdst = par + (size_t)g * DEC_MPAD + m;
    const int b = (m < M) ? (row_bits ? row_bits[m0 + m] : bits) : 0;
    if (b != 2 && b != 4 && b != 8) {
        // padding row or BF16 bypass row: zero codes
        if (b == 16) {  // still report non-finite inputs of bypass rows
            const uint16_t* src = x + (size_t)(m0 + m) * L.K + (size_t)g * L.G;
            for (int k = lane; k < L.G; k += 32)
                if (!finite_f(bf16_bits_to_float(src[k])))
                    report_nonfinite(err, (int64_t)(m0 + m) * L.K + (int64_t)g * L.G + k);
        }
        for (int k = lane; k < L.G; k += 32) dst[k] = 0;
        if (lane == 0) *pdst = make_uint2(0u, 0u);
        return;
    }
    const uint16_t* src = x + (size_t)(m0 + m) * L.K + (size_t)g * L.G;
    constexpr int MAXV = 4;  // G <= 128
    float v[MAXV];
    float vmin = 0.f, vmax = 0.f;
    int bad = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
        const int k = lane + 32 * i;
        v[i] = 0.f;
        if (k < L.G) {
            v[i] = bf16_bits_to_float(src[k]);
            if (!finite_f(v[i])) bad = min(bad, k);
            vmin = fminf(vmin, v[i]);
            vmax = fmaxf(vmax, v[i]);
        }
    }
    vmin = warp_min(vmin);
    vmax = warp_max(vmax);
#pragma unroll
    for (int o = 16; o; o >>= 1) bad = min(bad, __shfl_xor_sync(0xffffffffu, bad, o));
    if (bad != 0x7fffffff && lane == 0)
        report_nonfinite(err, (int64_t)(m0 + m) * L.K + (int64_t)g * L.G + bad);
    float s;
    int z;
    fit_params(vmin, vmax, b, &s, &z);
    int sum = 0;
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
        const int k = lane + 32 * i;
        if (k < L.G) {
            const int q = quantize_one(v[i], s, z, b, L.round_mode);
            sum += q;
            // 64-k sub-block permutation of the decode layout
            const int pos = (k & ~63) + dec_perm(k & 63);
            dst[pos] = (uint8_t)q;
        }
    }
    sum = warp_sum_i(sum);
    if (lane == 0) *pdst = make_uint2(__float_as_uint(s), ((uint32_t)z << 16) | (uint32_t)sum);
}

dyq_status_t launch_actquant_dec(const WLayout& L, const uint16_t* x, int M, int m0, const int32_t* row_bits,
                                 int bits, void* ws, int64_t* err, cudaStream_t st) {
    // rows m0 .. m0+M-1 (M <= DEC_MPAD) of x / row_bits (base pointers)
    const ActLayoutDec A = act_layout_dec(L);
    uint8_t* xq = reinterpret_cast<uint8_t*>(ws) + A.xq_off;
    uint2* par = reinterpret_cast<uint2*>(reinterpret_cast<uint8_t*>(ws) + A.par_off);
    const int warps = DEC_MPAD * L.NG;
    actquant_dec_kernel<<<(warps * 32 + 255) / 256, 256, 0, st>>>(L, x, M, m0, row_bits, bits, xq, par, err);
    return check_launch("actquant_dec_kernel");
}

// Test hook: export the decode-layout activation codes in logical layout.
__global__ void actquant_export_kernel(WLayout L, int M, int m0, const uint8_t* __restrict__ xq,
                                       const uint2* __restrict__ par, uint8_t* oq, float* os, uint8_t* oz,
                                       int32_t* oSX) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)M * L.K) return;
    const int m = (int)(idx / L.K), k = (int)(idx % L.K);
    const int pos = (k & ~63) + dec_perm(k & 63);
    oq[(size_t)(m0 + m) * L.K + k] = xq[(size_t)m * L.K + pos];
    if (k % L.G == 0) {
        const int g = k / L.G;
        const uint2 p = par[(size_t)g * DEC_MPAD + m];
        os[(size_t)(m0 + m) * L.NG + g] = __uint_as_float(p.x);
        oz[(size_t)(m0 + m) * L.NG + g] = (uint8_t)(p.y >> 16);
        oSX[(size_t)(m0 + m) * L.NG + g] = (int32_t)(p.y & 0xffffu);
    }
}

dyq_status_t launch_actquant_export(const WLayout& L, int M, const void* ws, uint8_t* xq, float* sx,
                                    uint8_t* zx, int32_t* SX, int m0, cudaStream_t st) {
    const ActLayoutDec A = act_layout_dec(L);
    const size_t total = (size_t)M * L.K;
    actquant_export_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
        L, M, m0, reinterpret_cast<const uint8_t*>(ws) + A.xq_off,
        reinterpret_cast<const uint2*>(reinterpret_cast<const uint8_t*>(ws) + A.par_off), xq, sx, zx, SX);
    return check_launch("actquant_export_kernel");
}

}  // namespace dyq
