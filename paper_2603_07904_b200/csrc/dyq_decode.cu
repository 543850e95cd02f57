// dyq_decode.cu -- the decode-regime quantized linear layer (M <= 16 tokens).
//
// the INT4-pinned weights stay densely packed in GMEM and
// are "decompressed on the fly ... within registers"; the activation
// codes of the step's width feed the integer MMA.  At M <= 16 this layer is
// HBM-bound (~0.58 B per weight at W4/G=64), so everything is organised around
// streaming the packed weights exactly once at full HBM bandwidth
// (measured B200 read-stream ceiling ~7.2 TB/s, tools/stream_bench.cu):
//
//  * work unit = (128-row tile, K-group); a pipeline STAGE = up to GPS
//    consecutive units of one tile (~16 KB of codes: one bulk copy) + their
//    metadata (one copy) + the activation slices (one copy per array) -- big
//    copies keep the TMA engine's per-copy cost off the critical path;
//  * one CTA per SM (stream-K: contiguous unit ranges, tile-major); the
//    producer issues the first stages' WEIGHT copies before griddepcontrol.wait,
//    so weight streaming starts under programmatic dependent launch (PDL);
//  * one producer thread runs an S-stage mbarrier ring (cp.async.bulk);
//  * 16 consumer warps, warp w = 16-row sub-tile w & 7, working on every group
//    of the stages of parity w >> 3: one LDS.128 per lane is the
//    exact register image of two mma.m16n8k32 A fragments (pre-permuted by
//    dyq_pack_weights); nibbles widen with LOP3s; integer tokens run
//    IMMA.16832.U8.U8 (tokens = the n8 dimension) with the exact per-group
//    zero-point algebra
//        I = P - z_w*SX - z_x*(Sum q - G*z_w),   P = Sum Xq*q   (int32)
//    where Sum q comes from one more IMMA against an all-ones B (no shuffles);
//    A16 tokens (the BF16 bypass) convert the same registers to bf16
//    (q - z_w is exact) and run HMMA.16816 against x;
//  * y = Sum_g s_x s_w I in fp32 (packed FMUL2/FFMA2); a tile split across
//    CTAs is reduced deterministically: each contributor writes a private
//    slot, the last to arrive (per-tile counter) sums slots in slot order.
#include <stdlib.h>

#include "dyq_internal.cuh"
#include "dyq_ptx.cuh"

namespace dyq {

struct DecArgs {
    WLayout L;
    const uint8_t* codes;
    const uint8_t* meta;    // 640-B block per (tile, group)
    const uint16_t* x;      // base [Mtotal, K] bf16
    const int32_t* row_bits;
    int bits;
    int M, m0;              // rows m0 .. m0+M-1 (M <= 16)
    void* y;                // base [Mtotal, N]
    int y_dtype;
    int32_t* I_out;         // base [Mtotal, N, NG] (partials mode)
    const uint8_t* ws;      // activation workspace (ActLayoutDec)
    ActLayoutDec A;
    float* part;            // split-K slots [(grid + T128)][16 tok][128 rows]
    int* counters;          // [T128]
    int upc;                // units per CTA
    int gps;                // groups (units) per stage
    int stages, stage_bytes;
    int off_meta, off_par, off_xq, off_x16;  // offsets inside a stage
    int debug_skip;         // DYQ_DEBUG_SKIP=1: consumers skip the math (copy-path timing only; debug)
};

__device__ __forceinline__ void mma_u8(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void mma_u8s8(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
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

// packed fp32x2 arithmetic (FMUL2 / FFMA2 on sm_100)
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

constexpr int DEC_CWARPS = 16;  // consumer warps: (sub-tile w & 7) x (stage parity w >> 3)
constexpr int DEC_THREADS = 32 * (DEC_CWARPS + 1);  // + 1 producer warp
constexpr int DEC_CONSUMERS = 32 * DEC_CWARPS;

enum { MODE_INT = 0, MODE_A16 = 1, MODE_MIXED = 2, MODE_INTC = 3 };  // INTC: centred s8 activation codes

// Split-K tile flush: direct store when the CTA owns the whole tile, otherwise
// private slot + last-arriver deterministic reduction.
template <int NT8>
__device__ __forceinline__ void dec_flush(const DecArgs& a, int tile, const float (&facc)[NT8][4], int warp,
                                          int gid, int t, int* s_flag) {
    const WLayout& L = a.L;
    const int NG = L.NG;
    const int nsub = (tile == L.T128 - 1) ? L.nsub_last : 8;
    const int nrows = nsub * 16;
    const int c_first = (tile * NG) / a.upc;
    const int c_last = (tile * NG + NG - 1) / a.upc;
    const int nc = c_last - c_first + 1;
    if (nc == 1) {
        if (warp < nsub) {
#pragma unroll
            for (int j = 0; j < NT8; ++j)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int tok = j * 8 + 2 * t + (i & 1);
                    if (tok < a.M) {
                        const size_t o = (size_t)(a.m0 + tok) * L.N + tile * 128 + warp * 16 + gid + 8 * (i >> 1);
                        if (a.y_dtype == 0)
                            reinterpret_cast<float*>(a.y)[o] = facc[j][i];
                        else
                            reinterpret_cast<__nv_bfloat16*>(a.y)[o] = __float2bfloat16_rn(facc[j][i]);
                    }
                }
        }
        return;
    }
    const int base = c_first + tile;  // slot range of this tile
    float* P = a.part + (size_t)(base + ((int)blockIdx.x - c_first)) * 16 * 128;
    if (warp < nsub) {
#pragma unroll
        for (int j = 0; j < NT8; ++j)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int tok = j * 8 + 2 * t + (i & 1);
                P[tok * 128 + warp * 16 + gid + 8 * (i >> 1)] = facc[j][i];
            }
    }
    ptx::named_bar_sync(1, DEC_CONSUMERS);
    if (threadIdx.x == 0) *s_flag = (ptx::atom_add_acq_rel_gpu(&a.counters[tile], 1) == nc - 1);
    ptx::named_bar_sync(1, DEC_CONSUMERS);
    if (*s_flag) {
        for (int idx = threadIdx.x; idx < a.M * nrows; idx += DEC_CONSUMERS) {
            const int tok = idx / nrows, r = idx - tok * nrows;
            // all slot loads in flight before the (slot-ordered, deterministic) sum
            const float* src = a.part + (size_t)base * 16 * 128 + tok * 128 + r;
            float sum = 0.f;
            for (int k0 = 0; k0 < nc; k0 += 16) {
                float v[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) v[k] = (k0 + k < nc) ? __ldcg(src + (size_t)(k0 + k) * 16 * 128) : 0.f;
#pragma unroll
                for (int k = 0; k < 16; ++k) sum += v[k];
            }
            const size_t o = (size_t)(a.m0 + tok) * L.N + tile * 128 + r;
            if (a.y_dtype == 0)
                reinterpret_cast<float*>(a.y)[o] = sum;
            else
                reinterpret_cast<__nv_bfloat16*>(a.y)[o] = __float2bfloat16_rn(sum);
        }
        if (threadIdx.x == 0) a.counters[tile] = 0;  // self-cleaning for the next call
    }
    ptx::named_bar_sync(1, DEC_CONSUMERS);
}

// One group (unit) of one 16-row sub-tile for this warp.  `st` = stage base
// (shared address), gi = index of the group inside the stage.
template <int WBITS, int NT8, int SPG, int MODE, bool PARTIALS>
__device__ __forceinline__ void dec_group(const DecArgs& a, uint32_t st, int gi, int g, int tile, int nsub,
                                          float (&facc)[NT8][4], uint32_t is16_mask) {
    constexpr int G = SPG * 64;
    const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) & 7;  // warp = sub-tile
    const int gid = lane >> 2, t = lane & 3;
    const WLayout& L = a.L;
    const uint32_t ONES = 0x01010101u;
    const int gps = a.gps;
    const uint32_t mb = st + a.off_meta + gi * META_BLOCK;
    const uint2 swr2 = ptx::lds64(mb + meta_slot(warp, gid) * 4);
    const float sw0 = __uint_as_float(swr2.x), sw1 = __uint_as_float(swr2.y);
    const uint32_t zw2 = ptx::lds16(mb + 512 + meta_slot(warp, gid));
    const int zw0 = zw2 & 0xff, zw1 = zw2 >> 8;
    uint32_t zz_g = 0, zz_g8 = 0;
    if (MODE != MODE_INT) {
        if (WBITS == 4) {
            zz_g = 0x43004300u | ((uint32_t)zw0 << 16) | (uint32_t)zw0;
            zz_g8 = 0x43004300u | ((uint32_t)zw1 << 16) | (uint32_t)zw1;
        } else {
            zz_g = __float_as_uint(8388608.f + (float)zw0);
            zz_g8 = __float_as_uint(8388608.f + (float)zw1);
        }
    }
    int iacc[NT8][4];
    float hacc[NT8][4];
    int sq[4] = {0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < NT8; ++j)
#pragma unroll
        for (int k = 0; k < 4; ++k) { iacc[j][k] = 0; hacc[j][k] = 0.f; }
#pragma unroll
    for (int spi = 0; spi < SPG; ++spi) {
        uint32_t A[2][4];  // per slab: lo_g, lo_g8, hi_g, hi_g8 (u8x4)
        const uint32_t cb = st + ((gi * SPG + spi) * nsub + warp) * (WBITS * 128) + lane * 16;
        if (WBITS == 4) {
            const uint4 w = ptx::lds128(cb);
            A[0][0] = w.x & 0x0F0F0F0Fu;
            A[0][1] = w.y & 0x0F0F0F0Fu;
            A[0][2] = (w.x >> 4) & 0x0F0F0F0Fu;
            A[0][3] = (w.y >> 4) & 0x0F0F0F0Fu;
            A[1][0] = w.z & 0x0F0F0F0Fu;
            A[1][1] = w.w & 0x0F0F0F0Fu;
            A[1][2] = (w.z >> 4) & 0x0F0F0F0Fu;
            A[1][3] = (w.w >> 4) & 0x0F0F0F0Fu;
        } else {
            const uint4 w0 = ptx::lds128(cb);
            const uint4 w1 = ptx::lds128(cb + 512);
            A[0][0] = w0.x; A[0][1] = w0.y; A[0][2] = w0.z; A[0][3] = w0.w;
            A[1][0] = w1.x; A[1][1] = w1.y; A[1][2] = w1.z; A[1][3] = w1.w;
        }
        if (MODE == MODE_INTC) {
            // centred s8 activations: P' = Sum q (Xq - z_x) directly
#pragma unroll
            for (int j = 0; j < NT8; ++j) {
                const uint4 xb = ptx::lds128(st + a.off_xq + ((j * gps + gi) * 8 + gid) * G + spi * 64 + t * 16);
                mma_u8s8(iacc[j], A[0], xb.x, xb.y);
                mma_u8s8(iacc[j], A[1], xb.z, xb.w);
            }
        } else if (MODE != MODE_A16) {
            // Sum q for rows gid, gid+8 from an all-ones B (no shuffles)
            mma_u8(sq, A[0], ONES, ONES);
            mma_u8(sq, A[1], ONES, ONES);
#pragma unroll
            for (int j = 0; j < NT8; ++j) {
                const uint4 xb = ptx::lds128(st + a.off_xq + ((j * gps + gi) * 8 + gid) * G + spi * 64 + t * 16);
                mma_u8(iacc[j], A[0], xb.x, xb.y);
                mma_u8(iacc[j], A[1], xb.z, xb.w);
            }
        }
        if (MODE == MODE_A16 || MODE == MODE_MIXED) {
#pragma unroll
            for (int j = 0; j < NT8; ++j) {
                const uint32_t xr = st + a.off_x16 + (((j * gps + gi) * 8 + gid) * G + spi * 64 + t * 16) * 2;
                const uint4 xa = ptx::lds128(xr);       // slab 0: h0 (x,y), h1 (z,w)
                const uint4 xc = ptx::lds128(xr + 16);  // slab 1
#pragma unroll
                for (int s2 = 0; s2 < 2; ++s2) {
                    const uint4 xx = s2 ? xc : xa;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const uint32_t rg = A[s2][h * 2 + 0], rg8 = A[s2][h * 2 + 1];
                        uint32_t A16[4];
                        A16[0] = u8pair_to_bf16<WBITS>(rg, 0, zz_g);
                        A16[1] = u8pair_to_bf16<WBITS>(rg8, 0, zz_g8);
                        A16[2] = u8pair_to_bf16<WBITS>(rg, 1, zz_g);
                        A16[3] = u8pair_to_bf16<WBITS>(rg8, 1, zz_g8);
                        mma_bf16(hacc[j], A16, h ? xx.z : xx.x, h ? xx.w : xx.y);
                    }
                }
            }
        }
    }
    // ---- group epilogue: exact integer correction, then fp32 dequant
    const int T_g = sq[0] - G * zw0;
    const int T_g8 = sq[2] - G * zw1;
#pragma unroll
    for (int j = 0; j < NT8; ++j) {
        uint4 pp = make_uint4(0u, 0u, 0u, 0u);
        if (MODE != MODE_A16) pp = ptx::lds128(st + a.off_par + gi * 128 + (j * 8 + 2 * t) * 8);
        const float sx0 = __uint_as_float(pp.x), sx1 = __uint_as_float(pp.z);
        const int zx0 = (int)(pp.y >> 16), zx1 = (int)(pp.w >> 16);
        const int SX0 = (int)(pp.y & 0xffffu), SX1 = (int)(pp.w & 0xffffu);
        int I[4];
        if (MODE == MODE_INTC) {  // par = {s_x, SXc = Sum (Xq - z_x)}
            const int SXc0 = (int)pp.y, SXc1 = (int)pp.w;
            I[0] = iacc[j][0] - zw0 * SXc0;
            I[1] = iacc[j][1] - zw0 * SXc1;
            I[2] = iacc[j][2] - zw1 * SXc0;
            I[3] = iacc[j][3] - zw1 * SXc1;
        } else {
            I[0] = iacc[j][0] - zw0 * SX0 - zx0 * T_g;
            I[1] = iacc[j][1] - zw0 * SX1 - zx1 * T_g;
            I[2] = iacc[j][2] - zw1 * SX0 - zx0 * T_g8;
            I[3] = iacc[j][3] - zw1 * SX1 - zx1 * T_g8;
        }
        if constexpr (PARTIALS) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int q = k & 1, hi = k >> 1;
                const int tc = j * 8 + 2 * t + q;
                if (tc < a.M) {
                    const bool a16 = (is16_mask >> (j * 2 + q)) & 1u;
                    const int n = tile * 128 + warp * 16 + gid + 8 * hi;
                    a.I_out[((size_t)(a.m0 + tc) * L.N + n) * L.NG + g] = a16 ? 0 : I[k];
                }
            }
        } else if (MODE == MODE_INT || MODE == MODE_INTC) {
            // (I0, I1) * (sx0, sx1) * sw_row  with packed fp32x2
            float t0, t1, t2, t3;
            mul2(t0, t1, (float)I[0], (float)I[1], sx0, sx1);
            mul2(t2, t3, (float)I[2], (float)I[3], sx0, sx1);
            fma2(facc[j][0], facc[j][1], t0, t1, sw0, sw0);
            fma2(facc[j][2], facc[j][3], t2, t3, sw1, sw1);
        } else if (MODE == MODE_A16) {
            fma2(facc[j][0], facc[j][1], hacc[j][0], hacc[j][1], sw0, sw0);
            fma2(facc[j][2], facc[j][3], hacc[j][2], hacc[j][3], sw1, sw1);
        } else {
            const float sxv[2] = {sx0, sx1};
            const float swv[2] = {sw0, sw1};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int q = k & 1, hi = k >> 1;
                const bool a16 = (is16_mask >> (j * 2 + q)) & 1u;
                facc[j][k] += a16 ? hacc[j][k] * swv[hi] : (float)I[k] * (swv[hi] * sxv[q]);
            }
        }
    }
}

// Consumer loop over the CTA's stages (must enumerate stages exactly like the
// producer).  Consumer warp w works on sub-tile w & 7 for every group of the
// stages of parity w >> 3; the two parities' partial sums are combined through
// shared memory only when a tile is flushed.
template <int NT8>
__device__ __forceinline__ void combine_parities(float (&facc)[NT8][4], float* scr, int par, int sub, int lane) {
    float* p = scr + (sub * 32 + lane) * (NT8 * 4);
    if (par == 1) {
#pragma unroll
        for (int j = 0; j < NT8; ++j)
#pragma unroll
            for (int k = 0; k < 4; ++k) p[j * 4 + k] = facc[j][k];
    }
    ptx::named_bar_sync(2, DEC_CONSUMERS);
    if (par == 0) {
#pragma unroll
        for (int j = 0; j < NT8; ++j)
#pragma unroll
            for (int k = 0; k < 4; ++k) facc[j][k] += p[j * 4 + k];
    }
    ptx::named_bar_sync(2, DEC_CONSUMERS);
}

template <int WBITS, int NT8, int SPG, int MODE, bool PARTIALS>
__device__ __forceinline__ void dec_consume(const DecArgs& a, uint32_t bar_full, uint32_t bar_empty,
                                            uint32_t stage0, int* s_flag, float* scr, int u0, int u1,
                                            uint32_t is16_mask) {
    const WLayout& L = a.L;
    const int NG = L.NG;
    const int S = a.stages;
    const int lane = threadIdx.x & 31, cw = threadIdx.x >> 5;
    const int sub = cw & 7, par = cw >> 3;
    const int gid = lane >> 2, t = lane & 3;
    const uint32_t stage_bytes = (uint32_t)a.stage_bytes;
    int s = 0, i = 0;
    uint32_t ph = 0;
    int cur_tile = -1;
    float facc[NT8][4];
#pragma unroll
    for (int j = 0; j < NT8; ++j)
#pragma unroll
        for (int k = 0; k < 4; ++k) facc[j][k] = 0.f;
    const int gps = a.gps;
    int tile = u0 / NG, g0 = u0 - (u0 / NG) * NG;  // one division per CTA, then incremental
    for (int u = u0; u < u1; ++i) {
        if (g0 == NG) { g0 = 0; ++tile; }
        int n = NG - g0;
        n = n < gps ? n : gps;
        n = n < u1 - u ? n : u1 - u;
        if (!PARTIALS && tile != cur_tile) {
            if (cur_tile >= 0) {
                combine_parities<NT8>(facc, scr, par, sub, lane);
                dec_flush<NT8>(a, cur_tile, facc, par ? 8 : sub, gid, t, s_flag);
            }
            cur_tile = tile;
#pragma unroll
            for (int j = 0; j < NT8; ++j)
#pragma unroll
                for (int k = 0; k < 4; ++k) facc[j][k] = 0.f;
        }
        if ((i & 1) == par) {
            const int nsub = (tile == L.T128 - 1) ? L.nsub_last : 8;
            ptx::mbar_wait_u32(bar_full + 8 * s, ph);
            if (sub < nsub && a.debug_skip == 0) {
                const uint32_t st = stage0 + s * stage_bytes;
#pragma unroll 2
                for (int gi = 0; gi < n; ++gi)
                    dec_group<WBITS, NT8, SPG, MODE, PARTIALS>(a, st, gi, g0 + gi, tile, nsub, facc, is16_mask);
            }
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_u32(bar_empty + 8 * s);
        }
        if (++s == S) { s = 0; ph ^= 1; }
        u += n;
        g0 += n;
    }
    if constexpr (!PARTIALS) {
        if (cur_tile >= 0) {
            combine_parities<NT8>(facc, scr, par, sub, lane);
            dec_flush<NT8>(a, cur_tile, facc, par ? 8 : sub, gid, t, s_flag);
        }
    }
}

template <int WBITS, int NT8, int SPG, bool PARTIALS>
__global__ void __launch_bounds__(DEC_THREADS) qlinear_decode_kernel(const DecArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    const WLayout& L = a.L;
    const int S = a.stages;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + S;
    int* s_flag = reinterpret_cast<int*>(empty + S);
    uint8_t* stage0 = smem + 128 * ((16 * S + 4 + 127) / 128);
    const int NG = L.NG;
    constexpr int G = SPG * 64;
    const int U = L.T128 * NG;
    const int u0 = blockIdx.x * a.upc;
    const int u1 = min(U, u0 + a.upc);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int stage_bytes = a.stage_bytes;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], DEC_CWARPS / 2);  // the 8 warps of the stage's parity
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    if (u0 >= u1) {
        ptx::pdl_launch_dependents();
        return;
    }

    if (warp == DEC_CWARPS) {  // ------------------------------------ producer
        if (lane == 0) {
            const uint64_t pol = ptx::policy_evict_first();
            const int chunk = L.chunk;
            auto issue_w = [&](int s, int tile, int g0, int n) {
                const int nsub = (tile == L.T128 - 1) ? L.nsub_last : 8;
                const uint32_t cbytes = (uint32_t)(n * SPG * nsub * chunk);
                uint8_t* st = stage0 + (size_t)s * stage_bytes;
                ptx::mbar_expect_tx(&full[s], cbytes + n * META_BLOCK);
                ptx::bulk_g2s_evict_first(st, a.codes + chunk_offset(L, tile, g0 * SPG, 0), cbytes, &full[s], pol);
                ptx::bulk_g2s(st + a.off_meta, a.meta + meta_block(L, tile, g0), n * META_BLOCK, &full[s]);
            };
            // (1) weights of the first S stages: independent of the preceding kernels
            int u = u0, i = 0;
            for (; i < S && u < u1; ++i) {
                const int tile = u / NG, g0 = u - tile * NG;
                const int n = min(a.gps, min(NG - g0, u1 - u));
                issue_w(i, tile, g0, n);
                u += n;
            }
            const int npre = i;
            // (2) activations: produced by the preceding kernels
            ptx::pdl_wait();
            bool any16 = false;
            for (int m = 0; m < a.M; ++m) any16 |= ((a.row_bits ? a.row_bits[a.m0 + m] : a.bits) == 16);
            auto issue_a = [&](int s, int g0, int n) {
                uint8_t* st = stage0 + (size_t)s * stage_bytes;
                const uint32_t xb = (uint32_t)(n * 8 * G);
                ptx::mbar_arrive_expect_tx(&full[s], n * 128 + NT8 * xb + (any16 ? NT8 * xb * 2 : 0));
                ptx::bulk_g2s(st + a.off_par, a.ws + a.A.par_off + (size_t)g0 * 128, n * 128, &full[s]);
#pragma unroll
                for (int h = 0; h < NT8; ++h)
                    ptx::bulk_g2s(st + a.off_xq + h * a.gps * 8 * G,
                                  a.ws + a.A.xq_off + ((size_t)h * NG + g0) * 8 * G, xb, &full[s]);
                if (any16) {
#pragma unroll
                    for (int h = 0; h < NT8; ++h)
                        ptx::bulk_g2s(st + a.off_x16 + h * a.gps * 8 * G * 2,
                                      a.ws + a.A.x16_off + ((size_t)h * NG + g0) * 8 * G * 2, xb * 2, &full[s]);
                }
            };
            u = u0;
            for (int k = 0; k < npre; ++k) {
                const int tile = u / NG, g0 = u - tile * NG;
                const int n = min(a.gps, min(NG - g0, u1 - u));
                issue_a(k, g0, n);
                u += n;
            }
            // (3) steady state
            int s = npre % S;
            uint32_t ph = 0;
            while (u < u1) {
                const int tile = u / NG, g0 = u - tile * NG;
                const int n = min(a.gps, min(NG - g0, u1 - u));
                ptx::mbar_wait(&empty[s], ph);
                issue_w(s, tile, g0, n);
                issue_a(s, g0, n);
                if (++s == S) { s = 0; ph ^= 1; }
                u += n;
            }
            // every weight byte of this CTA is in flight: let the next kernel's
            // CTAs launch (PDL trigger, one per CTA) so its producer can start
            ptx::pdl_launch_dependents();
        }
        return;
    }

    // ---------------------------------------------------------- consumers
    const int gid = lane >> 2, t = lane & 3;
    ptx::pdl_wait();  // row_bits come from the preceding kernels
    bool any_int = false, any16 = false;
    uint32_t is16_mask = 0;  // bit (j*2+q) for the C-fragment tokens j*8+2t+q
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
    const uint32_t bar_full = ptx::smem_u32(full), bar_empty = ptx::smem_u32(empty);
    const uint32_t st0 = ptx::smem_u32(stage0);
    float* scr = reinterpret_cast<float*>(stage0 + (size_t)S * stage_bytes);
    if (!any16 && dec_call_centred(a.M, a.m0, a.row_bits, a.bits))
        dec_consume<WBITS, NT8, SPG, MODE_INTC, PARTIALS>(a, bar_full, bar_empty, st0, s_flag, scr, u0, u1, is16_mask);
    else if (PARTIALS || (any_int && any16))
        dec_consume<WBITS, NT8, SPG, MODE_MIXED, PARTIALS>(a, bar_full, bar_empty, st0, s_flag, scr, u0, u1, is16_mask);
    else if (any16)
        dec_consume<WBITS, NT8, SPG, MODE_A16, PARTIALS>(a, bar_full, bar_empty, st0, s_flag, scr, u0, u1, is16_mask);
    else
        dec_consume<WBITS, NT8, SPG, MODE_INT, PARTIALS>(a, bar_full, bar_empty, st0, s_flag, scr, u0, u1, is16_mask);
}

// ------------------------------------------------------------------ host
struct DecPlan {
    int upc, grid, gps, stages, stage_bytes;
    int off_meta, off_par, off_xq, off_x16;
    size_t smem;
};

static int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) {
            cudaGetLastError();
            sms = 148;
        }
    }
    return sms;
}

static int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return v ? atoi(v) : dflt;
}

// NT8 = 2 when M > 8 (two halves of 8 tokens)
static DecPlan dec_plan(const WLayout& L, int nt8) {
    DecPlan p;
    const int unit_codes = (L.G / 64) * 8 * L.chunk;  // full tile
    static const int stage_code_kb = env_int("DYQ_DEC_STAGE_KB", 32);
    p.gps = (stage_code_kb * 1024) / unit_codes;
    if (p.gps < 1) p.gps = 1;
    if (p.gps > L.NG) p.gps = L.NG;
    p.off_meta = p.gps * unit_codes;
    p.off_par = p.off_meta + p.gps * META_BLOCK;
    p.off_xq = p.off_par + p.gps * 128;
    p.off_x16 = p.off_xq + nt8 * p.gps * 8 * L.G;
    p.stage_bytes = p.off_x16 + nt8 * p.gps * 8 * L.G * 2;
    static const int smem_kb = env_int("DYQ_DEC_SMEM_KB", 200);
    p.stages = (smem_kb * 1024 - 256) / p.stage_bytes;
    p.stages = p.stages < 2 ? 2 : (p.stages > 32 ? 32 : p.stages);
    p.smem = 128 * ((16 * p.stages + 4 + 127) / 128) + (size_t)p.stages * p.stage_bytes +
             (size_t)8 * 32 * 8 * 4;  // + parity-combine scratch
    const int U = L.T128 * L.NG;
    static const int ctas = env_int("DYQ_DEC_CTAS", 1);
    const int target = num_sms() * ctas;
    p.upc = (U + target - 1) / target;
    if (p.upc < 1) p.upc = 1;
    p.grid = (U + p.upc - 1) / p.upc;
    return p;
}

// split-K slot storage: (grid + T128) slots of 16 x 128 floats, then T128 counters
size_t decode_ws_bytes(const WLayout& L) {
    const DecPlan p = dec_plan(L, 2);
    return (size_t)(p.grid + L.T128) * 16 * 128 * 4 + (((size_t)L.T128 * 4 + 255) & ~(size_t)255);
}

template <int WBITS, int NT8, int SPG, bool PARTIALS>
static cudaError_t launch_k2(const DecArgs& a, const DecPlan& p, cudaStream_t st) {
    auto kern = qlinear_decode_kernel<WBITS, NT8, SPG, PARTIALS>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr_set = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.grid);
    cfg.blockDim = dim3(DEC_THREADS);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

template <int WBITS, int NT8, bool PARTIALS>
static cudaError_t launch_k(const DecArgs& a, const DecPlan& p, cudaStream_t st) {
    return a.L.G == 64 ? launch_k2<WBITS, NT8, 1, PARTIALS>(a, p, st) : launch_k2<WBITS, NT8, 2, PARTIALS>(a, p, st);
}

// ws layout: [split-K slots + tile counters (decode_ws_bytes, zeroed once,
// self-cleaning)] [activation area written by the quantizer kernel].
dyq_status_t launch_decode(const WLayout& L, const void* codes, const void* meta, const uint16_t* x, int M,
                           int m0, const int32_t* row_bits, int bits, void* y, int y_dtype, int32_t* I_out,
                           void* ws, int64_t* /*err*/, cudaStream_t st) {
    const int nt8 = M <= 8 ? 1 : 2;
    const ActLayoutDec A = act_layout_dec(L);
    const DecPlan p = dec_plan(L, nt8);
    const DecPlan p2 = dec_plan(L, 2);  // workspace is sized with the NT8 = 2 plan (same grid)
    DecArgs a;
    a.L = L;
    a.codes = reinterpret_cast<const uint8_t*>(codes);
    a.meta = reinterpret_cast<const uint8_t*>(meta);
    a.x = x;
    a.row_bits = row_bits;
    a.bits = bits;
    a.M = M;
    a.m0 = m0;
    a.y = y;
    a.y_dtype = y_dtype;
    a.I_out = I_out;
    uint8_t* wsb = reinterpret_cast<uint8_t*>(ws);
    a.ws = wsb + ((decode_ws_bytes(L) + 255) & ~(size_t)255);
    a.A = A;
    a.part = reinterpret_cast<float*>(wsb);
    a.counters = reinterpret_cast<int*>(wsb + (size_t)(p2.grid + L.T128) * 16 * 128 * 4);
    a.upc = p.upc;
    a.gps = p.gps;
    a.stages = p.stages;
    a.stage_bytes = p.stage_bytes;
    a.off_meta = p.off_meta;
    a.off_par = p.off_par;
    a.off_xq = p.off_xq;
    a.off_x16 = p.off_x16;
    static const int dbg = env_int("DYQ_DEBUG_SKIP", 0);
    a.debug_skip = dbg;
    const bool partials = I_out != nullptr;
    cudaError_t e;
#define DYQ_DISPATCH(WB)                                                                      \
    if (partials) e = nt8 == 1 ? launch_k<WB, 1, true>(a, p, st) : launch_k<WB, 2, true>(a, p, st); \
    else e = nt8 == 1 ? launch_k<WB, 1, false>(a, p, st) : launch_k<WB, 2, false>(a, p, st);
    if (L.wbits == 4) {
        DYQ_DISPATCH(4)
    } else {
        DYQ_DISPATCH(8)
    }
#undef DYQ_DISPATCH
    if (e != cudaSuccess) return set_error(DYQ_ECUDA, "qlinear_decode_kernel launch: %s", cudaGetErrorString(e));
    return check_launch("qlinear_decode_kernel");
}

}  // namespace dyq
