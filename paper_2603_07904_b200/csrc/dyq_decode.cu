// dyq_decode.cu -- the decode-regime quantized linear layer (M <= 16 tokens).
//
// the INT4-pinned weights stay densely packed in GMEM and
// are "decompressed on the fly ... within registers"; the activation
// codes of the step's width feed the integer MMA.  At M <= 16 this layer is
// HBM-bound (~0.58 B per weight at W4/G=64), so the design goal is streaming
// the packed weights once at full bandwidth:
//   * one CTA = one 16-row sub-tile, 8 warps split K by groups (split-K inside
//     the CTA, fixed-order smem reduction -> deterministic);
//   * each lane streams 16 B per (16 rows x 64 k) chunk with a 128-bit
//     non-allocating load; chunks are pre-permuted by dyq_pack_weights into the
//     exact register order of the mma.m16n8k32 A fragment;
//   * nibbles are widened with two LOP3s per 8 weights (no table, no shuffle);
//   * integer rows run IMMA.16832.U8.U8 (tokens = the n8 dimension) and the
//     per-group zero-point algebra
//         I = P - z_w*SX - z_x*(Sum q - G*z_w),  P = Sum Xq*q   (exact int32)
//     is applied in the group epilogue; Sum q comes from IDP.4A on the
//     widened registers (no extra bytes);
//   * A16 rows (BF16 bypass) convert the same registers to bf16
//     (q - z_w is exact in bf16) and run HMMA.16816 against x.
//   * y = Sum_g s_x s_w I (fp32), reduced across warps in a fixed order.
#include "dyq_internal.cuh"

namespace dyq {

struct DecArgs {
    WLayout L;
    const uint8_t* codes;
    const float* scales;
    const uint8_t* zeros;
    const uint16_t* x;      // base [Mtotal, K] bf16
    const int32_t* row_bits;
    int bits;
    int M, m0;              // this call handles rows m0 .. m0+M-1 (M <= 16)
    void* y;                // base [Mtotal, N]
    int y_dtype;
    int32_t* I_out;         // base [Mtotal, N, NG] (partials mode)
    const uint8_t* xq;      // [16][K] decode layout
    const uint2* par;       // [NG][16]
};

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

__device__ __forceinline__ void mma_u8(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void mma_bf16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// bytes (lo pair or hi pair) of a u8x4 register -> bf16x2 of (q - z).
template <int WBITS>
__device__ __forceinline__ uint32_t u8pair_to_bf16(uint32_t v, int hi_pair, uint32_t zz) {
    if (WBITS == 4) {
        // 0x43 00 | q = bf16(128 + q) exactly for q <= 127; subtract bf16(128 + z)
        const uint32_t t = __byte_perm(v, 0x4343u, hi_pair ? 0x5342u : 0x5140u);
        __nv_bfloat162 r = __hsub2(*reinterpret_cast<const __nv_bfloat162*>(&t),
                                   *reinterpret_cast<const __nv_bfloat162*>(&zz));
        return *reinterpret_cast<uint32_t*>(&r);
    } else {
        // fp32 magic 2^23 + q (exact), minus (2^23 + z), then pack to bf16 (|q-z| <= 255: exact)
        const uint32_t f0 = __byte_perm(v, 0x4B000000u, hi_pair ? 0x7542u : 0x7540u);
        const uint32_t f1 = __byte_perm(v, 0x4B000000u, hi_pair ? 0x7543u : 0x7541u);
        const float zf = __uint_as_float(zz);
        const float a = __uint_as_float(f0) - zf, b = __uint_as_float(f1) - zf;
        __nv_bfloat162 r = __floats2bfloat162_rn(a, b);
        return *reinterpret_cast<uint32_t*>(&r);
    }
}

template <int WBITS, int NT8, bool PARTIALS>
__global__ void __launch_bounds__(256) qlinear_decode_kernel(const DecArgs a) {
    constexpr int NW = 8;
    const WLayout& L = a.L;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gid = lane >> 2, t = lane & 3;
    const int st = blockIdx.x;            // 16-row sub-tile
    const int tile = st >> 3, sub = st & 7;
    const int n0 = st * 16;
    const int SPG = L.G >> 6;             // slab pairs per group
    const int gb = (warp * L.NG) / NW, ge = ((warp + 1) * L.NG) / NW;

    // token flags (B-fragment token = j*8+gid; C-fragment tokens = j*8+2t+q)
    bool any_int = false, any16 = false;
    uint32_t is16_mask = 0;  // bit (j*2+q) for C tokens
#pragma unroll
    for (int j = 0; j < NT8; ++j) {
        const int tb = j * 8 + gid;
        if (tb < a.M) {
            const int b = a.row_bits ? a.row_bits[a.m0 + tb] : a.bits;
            any16 |= (b == 16);
            any_int |= (b != 16);
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int tc = j * 8 + 2 * t + q;
            if (tc < a.M) {
                const int b = a.row_bits ? a.row_bits[a.m0 + tc] : a.bits;
                if (b == 16) is16_mask |= 1u << (j * 2 + q);
            }
        }
    }
    any16 = __any_sync(0xffffffffu, any16);
    any_int = __any_sync(0xffffffffu, any_int);

    float facc[NT8][4];
#pragma unroll
    for (int j = 0; j < NT8; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i) facc[j][i] = 0.f;

    for (int g = gb; g < ge; ++g) {
        // group metadata (rows gid, gid+8 adjacent by construction)
        const size_t mi = meta_index(L, tile, g, sub, gid);
        const float2 sw = *reinterpret_cast<const float2*>(a.scales + mi);
        const uchar2 zw = *reinterpret_cast<const uchar2*>(a.zeros + mi);
        uint32_t zz_g, zz_g8;
        if (WBITS == 4) {
            zz_g = 0x43004300u | ((uint32_t)zw.x << 16) | zw.x;
            zz_g8 = 0x43004300u | ((uint32_t)zw.y << 16) | zw.y;
        } else {
            zz_g = __float_as_uint(8388608.f + (float)zw.x);
            zz_g8 = __float_as_uint(8388608.f + (float)zw.y);
        }
        int iacc[NT8][4];
        float hacc[NT8][4];
#pragma unroll
        for (int j = 0; j < NT8; ++j)
#pragma unroll
            for (int i = 0; i < 4; ++i) { iacc[j][i] = 0; hacc[j][i] = 0.f; }
        uint32_t sq_g = 0, sq_g8 = 0;

        for (int spi = 0; spi < SPG; ++spi) {
            const int sp = g * SPG + spi;
            const uint8_t* ch = a.codes + chunk_offset(L, tile, sp, sub);
            uint32_t A[2][4];  // per slab: lo_g, lo_g8, hi_g, hi_g8 (u8x4)
            if (WBITS == 4) {
                const uint4 w = ldg_stream(ch + lane * 16);
                const uint32_t wg[2] = {w.x, w.z}, wg8[2] = {w.y, w.w};
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    A[s][0] = wg[s] & 0x0F0F0F0Fu;
                    A[s][1] = wg8[s] & 0x0F0F0F0Fu;
                    A[s][2] = (wg[s] >> 4) & 0x0F0F0F0Fu;
                    A[s][3] = (wg8[s] >> 4) & 0x0F0F0F0Fu;
                }
                sq_g = __dp4a(A[0][0] + A[0][2] + A[1][0] + A[1][2], 0x01010101u, sq_g);
                sq_g8 = __dp4a(A[0][1] + A[0][3] + A[1][1] + A[1][3], 0x01010101u, sq_g8);
            } else {
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    const uint4 w = ldg_stream(ch + s * 512 + lane * 16);
                    A[s][0] = w.x; A[s][1] = w.y; A[s][2] = w.z; A[s][3] = w.w;
                    sq_g = __dp4a(w.x, 0x01010101u, sq_g);
                    sq_g = __dp4a(w.z, 0x01010101u, sq_g);
                    sq_g8 = __dp4a(w.y, 0x01010101u, sq_g8);
                    sq_g8 = __dp4a(w.w, 0x01010101u, sq_g8);
                }
            }
            if (any_int) {
#pragma unroll
                for (int j = 0; j < NT8; ++j) {
                    const uint4 xb = *reinterpret_cast<const uint4*>(a.xq + (size_t)(j * 8 + gid) * L.K +
                                                                      (size_t)sp * 64 + t * 16);
                    mma_u8(iacc[j], A[0], xb.x, xb.y);
                    mma_u8(iacc[j], A[1], xb.z, xb.w);
                }
            }
            if (any16) {
#pragma unroll
                for (int s = 0; s < 2; ++s) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {  // h=0: lo regs (k 4t..), h=1: hi regs (k 16+4t..)
                        const uint32_t rg = A[s][h * 2 + 0], rg8 = A[s][h * 2 + 1];
                        uint32_t A16[4];
                        A16[0] = u8pair_to_bf16<WBITS>(rg, 0, zz_g);
                        A16[1] = u8pair_to_bf16<WBITS>(rg8, 0, zz_g8);
                        A16[2] = u8pair_to_bf16<WBITS>(rg, 1, zz_g);
                        A16[3] = u8pair_to_bf16<WBITS>(rg8, 1, zz_g8);
#pragma unroll
                        for (int j = 0; j < NT8; ++j) {
                            const int tb = j * 8 + gid;
                            uint2 xb = make_uint2(0u, 0u);
                            if (tb < a.M)
                                xb = *reinterpret_cast<const uint2*>(
                                    a.x + (size_t)(a.m0 + tb) * L.K + (size_t)sp * 64 + s * 32 + h * 16 + 4 * t);
                            mma_bf16(hacc[j], A16, xb.x, xb.y);
                        }
                    }
                }
            }
        }
        // ---- group epilogue: exact integer correction, then fp32 dequant
        sq_g += __shfl_xor_sync(0xffffffffu, sq_g, 1);
        sq_g += __shfl_xor_sync(0xffffffffu, sq_g, 2);
        sq_g8 += __shfl_xor_sync(0xffffffffu, sq_g8, 1);
        sq_g8 += __shfl_xor_sync(0xffffffffu, sq_g8, 2);
        const int T_g = (int)sq_g - L.G * (int)zw.x;
        const int T_g8 = (int)sq_g8 - L.G * (int)zw.y;
#pragma unroll
        for (int j = 0; j < NT8; ++j) {
            const uint4 pp = *reinterpret_cast<const uint4*>(a.par + (size_t)g * DEC_MPAD + j * 8 + 2 * t);
            const float sx[2] = {__uint_as_float(pp.x), __uint_as_float(pp.z)};
            const int zx[2] = {(int)(pp.y >> 16), (int)(pp.w >> 16)};
            const int SX[2] = {(int)(pp.y & 0xffffu), (int)(pp.w & 0xffffu)};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int q = i & 1, hi = i >> 1;
                const int zwr = hi ? zw.y : zw.x;
                const int Tr = hi ? T_g8 : T_g;
                const float swr = hi ? sw.y : sw.x;
                const int I = iacc[j][i] - zwr * SX[q] - zx[q] * Tr;
                const bool a16 = (is16_mask >> (j * 2 + q)) & 1u;
                if constexpr (PARTIALS) {
                    const int tc = j * 8 + 2 * t + q;
                    if (tc < a.M) {
                        const int n = n0 + gid + 8 * hi;
                        a.I_out[((size_t)(a.m0 + tc) * L.N + n) * L.NG + g] = a16 ? 0 : I;
                    }
                } else {
                    facc[j][i] += a16 ? hacc[j][i] * swr : (float)I * (swr * sx[q]);
                }
            }
        }
    }
    if constexpr (PARTIALS) return;
    else {
    // ---- fixed-order cross-warp reduction and store
    __shared__ float red[NW][NT8 * 8][17];
#pragma unroll
    for (int j = 0; j < NT8; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i) red[warp][j * 8 + 2 * t + (i & 1)][gid + 8 * (i >> 1)] = facc[j][i];
    __syncthreads();
    for (int idx = threadIdx.x; idx < NT8 * 8 * 16; idx += blockDim.x) {
        const int tok = idx >> 4, r = idx & 15;
        if (tok < a.M) {
            float s = 0.f;
#pragma unroll
            for (int w = 0; w < NW; ++w) s += red[w][tok][r];
            const size_t o = (size_t)(a.m0 + tok) * L.N + n0 + r;
            if (a.y_dtype == 0)
                reinterpret_cast<float*>(a.y)[o] = s;
            else
                reinterpret_cast<__nv_bfloat16*>(a.y)[o] = __float2bfloat16_rn(s);
        }
    }
    }
}

template <int WBITS, bool PARTIALS>
static void launch_t(const DecArgs& a, int nt8, cudaStream_t st) {
    const dim3 grid(a.L.N / 16), block(256);
    if (nt8 == 1)
        qlinear_decode_kernel<WBITS, 1, PARTIALS><<<grid, block, 0, st>>>(a);
    else
        qlinear_decode_kernel<WBITS, 2, PARTIALS><<<grid, block, 0, st>>>(a);
}

dyq_status_t launch_decode(const WLayout& L, const void* codes, const void* meta, const uint16_t* x, int M,
                           int m0, int /*Mtotal*/, const int32_t* row_bits, int bits, void* y, int y_dtype,
                           int32_t* I_out, const void* ws, cudaStream_t st) {
    const ActLayoutDec A = act_layout_dec(L);
    DecArgs a;
    a.L = L;
    a.codes = reinterpret_cast<const uint8_t*>(codes);
    a.scales = reinterpret_cast<const float*>(meta);
    a.zeros = reinterpret_cast<const uint8_t*>(meta) + L.zeros_off;
    a.x = x;
    a.row_bits = row_bits;
    a.bits = bits;
    a.M = M;
    a.m0 = m0;
    a.y = y;
    a.y_dtype = y_dtype;
    a.I_out = I_out;
    a.xq = reinterpret_cast<const uint8_t*>(ws) + A.xq_off;
    a.par = reinterpret_cast<const uint2*>(reinterpret_cast<const uint8_t*>(ws) + A.par_off);
    const int nt8 = M <= 8 ? 1 : 2;
    const bool partials = I_out != nullptr;
    if (L.wbits == 4) {
        if (partials) launch_t<4, true>(a, nt8, st); else launch_t<4, false>(a, nt8, st);
    } else {
        if (partials) launch_t<8, true>(a, nt8, st); else launch_t<8, false>(a, nt8, st);
    }
    return check_launch("qlinear_decode_kernel");
}

}  // namespace dyq
