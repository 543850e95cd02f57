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
//    metadata (one copy) + the activation records of those K-groups (one copy,
//    plus one for the bf16 rows of BF16-bypass tokens) -- big copies keep the
//    TMA engine's per-copy cost off the critical path;
//  * stream-K: contiguous unit ranges, tile-major, ONE CTA per SM (544
//    threads: 16 consumer warps + 1 producer warp, up to 56 KB of codes per
//    stage).  Under programmatic dependent launch (PDL) the producer issues
//    its first stages' weight copies BEFORE griddepcontrol.wait -- weights
//    never depend on the previous kernel -- so weight streaming overlaps the
//    tail of the preceding kernel (act-quant or the previous linear);
//  * consumer warp w owns 16-row sub-tile w & 7 and the even / odd groups
//    (w >> 3) of every stage; one LDS.128 per lane is the exact register
//    image of two mma.m16n8k32 A fragments (pre-permuted by
//    dyq_pack_weights); nibbles widen with LOP3s; integer tokens run
//    IMMA.16832.U8.U8 (tokens = the n8 dimension) with the exact per-group
//    zero-point algebra
//        I = P - z_w*SX - z_x*(Sum q - G*z_w),   P = Sum Xq*q   (int32)
//    where Sum q comes from one more IMMA against an all-ones B (no shuffles);
//    A2/A4-only calls use centred s8 codes (I = P' - z_w*SXc, one IMMA);
//    A16 tokens (the BF16 bypass) convert the same registers to bf16
//    (q - z_w is exact) and run HMMA.16816 against x; the two parity warps of
//    a sub-tile combine through shared memory (64-thread named barrier);
//  * y = Sum_g s_x s_w I in fp32 (packed FMUL2/FFMA2).  A tile split across
//    CTAs is reduced by a DESIGNATED reducer: the contributors of a tile are
//    CTAs c_first..c_last, c_first holds the tile's first groups at the END of
//    its range, so it reduces; the others publish a private slot (smem ->
//    cp.async.bulk -> completion wait -> counter increment) and never wait;
//    c_first acquires the counter, sums the slots in contributor order
//    (deterministic) and writes y.
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
    const uint8_t* ws;      // activation area (ActLayoutDec)
    ActLayoutDec A;
    float* part;            // split-K slots [(grid + T128)][16 tok][128 rows]
    int* counters;          // [T128][8 sub-tiles]
    int upc;                // units per CTA
    int gps;                // groups (units) per stage
    int stages, stage_bytes;
    int off_meta, off_cp, off_x16;  // offsets inside a stage
    uint64_t* trace;                // dyq_trace_enable buffer or null
    const int32_t* gate;            // dyq_qlinear_masked gate or null
    uint32_t serial;
    TpPeers tp;                     // fused TP epilogue (tp.n = 0: off)
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

#ifndef DYQ_DEC_CWARPS
#define DYQ_DEC_CWARPS 16
#endif
#ifndef DYQ_DEC_UNROLL
#define DYQ_DEC_UNROLL 2
#endif
// consumer warps: warp w = sub-tile w & 7; with 16 warps, warp w >> 3 takes the
// odd / even groups of every stage and the pair combines through shared memory
constexpr int DEC_CWARPS = DYQ_DEC_CWARPS;
constexpr int DEC_THREADS = 32 * (DEC_CWARPS + 1);  // + 1 producer warp
constexpr int DEC_UNROLL = DYQ_DEC_UNROLL;
constexpr int DEC_MINB = DEC_CWARPS == 8 ? 2 : 1;   // CTAs per SM (register budget)

enum { MODE_INT = 0, MODE_A16 = 1, MODE_MIXED = 2, MODE_INTC = 3 };  // INTC: centred s8 activation codes

// Per-warp scratch for split-K slot publication (after the stages and the
// 16-warp combine area).
__device__ __forceinline__ float* dec_slot_scratch(const DecArgs& a, int sub) {
    extern __shared__ __align__(128) uint8_t smem[];
    return reinterpret_cast<float*>(smem + 256 + (size_t)a.stages * a.stage_bytes + 8 * 32 * 8 * 4) + sub * 256;
}
// Lane 0 of a contributor warp: once its bulk slot store completed, count it.
// The slot was written by the async proxy (cp.async.bulk shared->global) and
// is read by the reducer through the generic proxy after its ld.acquire of
// the counter.  The writer has already waited for the bulk store to COMPLETE
// (cp.async.bulk.wait_group 0, i.e. the bytes are in L2, the gpu-scope
// coherence point) before it increments, so a relaxed increment is ordered
// after the data on this hardware; the PTX-model-strict form (async->generic
// proxy fence + red.release.gpu) costs ~1.2 us per gate|up call (B200 A/B:
// 12.65 -> 13.9 us, 35a9e9e) and is kept as a build switch
// (DYQ_DEC_RELAXED_PUBLISH=0).  DESIGN.md §5 records the trade.
#ifndef DYQ_DEC_RELAXED_PUBLISH
#define DYQ_DEC_RELAXED_PUBLISH 1
#endif
__device__ __forceinline__ void dec_count_slot(int* p) {
#if DYQ_DEC_RELAXED_PUBLISH
    ptx::red_add_relaxed_gpu(p, 1);
#else
    asm volatile("fence.proxy.async.global;" ::: "memory");
    ptx::red_add_release_gpu(p, 1);
#endif
}
__device__ __forceinline__ void dec_publish(int*& pend, int lane) {
    if (lane == 0 && pend) {
        ptx::bulk_wait_all();
        dec_count_slot(pend);
        pend = nullptr;
    }
}

// Split-K flush of one sub-tile by its warp.  When the CTA owns the whole
// tile: direct store.  Otherwise the contributors of a tile are the CTAs
// c_first..c_last of the stream-K order; CTA c_first holds the tile's FIRST
// groups at the END of its range, every other contributor holds its part at
// the START of its range.  So c_first is the designated reducer: the others
// write a private slot and release-increment the (tile, sub-tile) counter
// without waiting (fire and forget, long before c_first gets there); c_first
// acquires the counter, adds the slots in contributor order (deterministic)
// to its own partial sums and writes y.  All CTAs of the grid are co-resident
// (grid <= #SMs, one CTA per SM), so the reducer's wait always ends.
__shared__ int s_tp_subtiles;  // fused TP: sub-tiles of y this CTA wrote

template <int NT8, bool TP>
__device__ __forceinline__ void dec_flush_warp(const DecArgs& a, int tile, const float (&facc)[NT8][4], int sub,
                                               int lane, int*& pend) {
    const WLayout& L = a.L;
    const int NG = L.NG;
    const int nsub = (tile == L.T128 - 1) ? L.nsub_last : 8;
    if (sub >= nsub) return;  // warp-uniform
    const int gid = lane >> 2, t = lane & 3;
    const int c_first = (tile * NG) / a.upc;
    const int c_last = (tile * NG + NG - 1) / a.upc;
    const int nc = c_last - c_first + 1;
    const int c = (int)blockIdx.x - c_first;
    auto store = [&](int tok, int r, float v) {
        if (a.row_bits && a.row_bits[a.m0 + tok] == 0) return;  // masked row: y untouched
        if constexpr (TP) {  // every rank's full y, this rank's columns
            const size_t o = (size_t)(a.m0 + tok) * a.tp.ldy + a.tp.col0 + tile * 128 + sub * 16 + r;
            const __nv_bfloat16 h = __float2bfloat16_rn(v);
            for (int p = 0; p < a.tp.n; ++p) reinterpret_cast<__nv_bfloat16*>(a.tp.y[p])[o] = h;
            return;
        }
        const size_t o = (size_t)(a.m0 + tok) * L.N + tile * 128 + sub * 16 + r;
        if (a.y_dtype == 0)
            reinterpret_cast<float*>(a.y)[o] = v;
        else
            reinterpret_cast<__nv_bfloat16*>(a.y)[o] = __float2bfloat16_rn(v);
    };
    int* cnt = &a.counters[tile * 8 + sub];
    const int base = c_first + tile;  // slot range of this tile
    if (nc > 1 && c != 0) {
        // slot = [sub][16 tok][16 rows] fp32, published through the async proxy
        // (bulk store): the relaxed counter increment follows the completion of
        // the copy (cp.async.bulk.wait_group), deferred to the next stage
        // boundary (dec_publish) so this warp never stalls on it.  No
        // gpu-scope release fence (MEMBAR.ALL.GPU would wait for the CTA's
        // in-flight weight copies).
        float* scr = dec_slot_scratch(a, sub);
#pragma unroll
        for (int j = 0; j < NT8; ++j)
#pragma unroll
            for (int i = 0; i < 4; ++i) scr[(j * 8 + 2 * t + (i & 1)) * 16 + gid + 8 * (i >> 1)] = facc[j][i];
        ptx::fence_proxy_async_cta();
        __syncwarp();
        if (lane == 0) {
            ptx::bulk_wait_all();  // previous publication of this warp (scratch reuse)
            if (pend) dec_count_slot(pend);
            float* P = a.part + ((size_t)(base + c) * 8 + sub) * 16 * 16;
            ptx::bulk_s2g(P, ptx::smem_u32(scr), NT8 * 8 * 16 * 4);
            pend = cnt;
        }
        return;
    }
    float v[NT8][4];
#pragma unroll
    for (int j = 0; j < NT8; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i) v[j][i] = facc[j][i];
    if (nc > 1) {
        if (lane == 0) {
            if (threadIdx.x == 0) trace_ev(a.trace, a.serial, 1, 5);
            while (ptx::ld_acquire_gpu(cnt) < nc - 1) __nanosleep(64);
            if (threadIdx.x == 0) trace_ev(a.trace, a.serial, 1, 6);
            *cnt = 0;  // self-cleaning: the next call's contributors start after this kernel
        }
        __syncwarp();
        const float* src = a.part + ((size_t)base * 8 + sub) * 16 * 16;
        constexpr int SL = 8 * 16 * 16;  // floats per slot
        // all slots' loads in flight at once (one L2 round trip per 8 contributors),
        // then the sums in contributor order
        for (int c0 = 1; c0 < nc; c0 += 8) {
            float w[8][NT8][4];
#pragma unroll
            for (int k = 0; k < 8; ++k)
#pragma unroll
                for (int j = 0; j < NT8; ++j)
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        w[k][j][i] = (c0 + k < nc) ? __ldcg(src + (c0 + k) * SL + (j * 8 + 2 * t + (i & 1)) * 16 +
                                                            gid + 8 * (i >> 1))
                                                   : 0.f;
#pragma unroll
            for (int k = 0; k < 8; ++k)
#pragma unroll
                for (int j = 0; j < NT8; ++j)
#pragma unroll
                    for (int i = 0; i < 4; ++i) v[j][i] += w[k][j][i];
        }
    }
#pragma unroll
    for (int j = 0; j < NT8; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int tok = j * 8 + 2 * t + (i & 1);
            if (tok < a.M) store(tok, gid + 8 * (i >> 1), v[j][i]);
        }
    if constexpr (TP) {  // counted here, announced once per CTA (dec_tp_announce)
        __syncwarp();
        if (lane == 0) atomicAdd_block(&s_tp_subtiles, 1);
    }
}

// Fused TP: after every consumer warp is done, one thread fences at system
// scope (the CTA barrier orders all warps' peer stores before it) and adds
// the CTA's sub-tile count to every rank's flag -- one fence and tp.n atomics
// per CTA instead of per 16-column sub-tile.
__device__ __forceinline__ void dec_tp_announce(const DecArgs& a) {
    ptx::named_bar_sync(9, DEC_CWARPS * 32);
    if (threadIdx.x == 0) {
        const int n = s_tp_subtiles;
        if (n) {
            __threadfence_system();  // fence.acq_rel.sys / red.release.sys / gpu scope: no faster
            for (int p = 0; p < a.tp.n; ++p) atomicAdd_system(a.tp.flag[p], (unsigned long long)n);
        }
    }
}

// One group (unit) of one 16-row sub-tile for this warp.  `st` = stage base
// (shared address), gi = index of the group inside the stage.
template <int WBITS, int NT8, int SPG, int MODE, bool PARTIALS>
__device__ __forceinline__ void dec_group(const DecArgs& a, uint32_t st, int gi, int g, int tile, int nsub,
                                          float (&facc)[NT8][4], uint32_t is16_mask) {
    constexpr int G = SPG * 64;
    constexpr int CPS = NT8 * 8 * G + NT8 * 64;  // activation record bytes per group (ActLayoutDec::cp_stride)
    constexpr int X16S = NT8 * 8 * G * 2;        // bf16 rows per group (ActLayoutDec::x16_stride)
    const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) & 7;  // warp = sub-tile
    const int gid = lane >> 2, t = lane & 3;
    const WLayout& L = a.L;
    const uint32_t ONES = 0x01010101u;
    const uint32_t rec = st + a.off_cp + gi * CPS;
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
                const uint4 xb = ptx::lds128(rec + (j * 8 + gid) * G + spi * 64 + t * 16);
                mma_u8s8(iacc[j], A[0], xb.x, xb.y);
                mma_u8s8(iacc[j], A[1], xb.z, xb.w);
            }
        } else if (MODE != MODE_A16) {
            // Sum q for rows gid, gid+8 from an all-ones B (no shuffles)
            mma_u8(sq, A[0], ONES, ONES);
            mma_u8(sq, A[1], ONES, ONES);
#pragma unroll
            for (int j = 0; j < NT8; ++j) {
                const uint4 xb = ptx::lds128(rec + (j * 8 + gid) * G + spi * 64 + t * 16);
                mma_u8(iacc[j], A[0], xb.x, xb.y);
                mma_u8(iacc[j], A[1], xb.z, xb.w);
            }
        }
        if (MODE == MODE_A16 || MODE == MODE_MIXED) {
#pragma unroll
            for (int j = 0; j < NT8; ++j) {
                const uint32_t xr = st + a.off_x16 + gi * X16S + ((j * 8 + gid) * G + spi * 64 + t * 16) * 2;
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
        if (MODE != MODE_A16) pp = ptx::lds128(rec + NT8 * 8 * G + (j * 8 + 2 * t) * 8);
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

// End of this CTA's part of a tile: with 16 consumer warps the odd-group warp
// of each sub-tile hands its partial sums to the even-group warp (shared
// memory + a 64-thread named barrier per sub-tile), which flushes.
template <int NT8, bool TP>
__device__ __forceinline__ void dec_tile_done(const DecArgs& a, int tile, float (&facc)[NT8][4], int sub, int par,
                                              int lane, int*& pend) {
    if constexpr (DEC_CWARPS == 16) {
        extern __shared__ __align__(128) uint8_t smem[];
        float* p = reinterpret_cast<float*>(smem + 256 + (size_t)a.stages * a.stage_bytes) + (sub * 32 + lane) * 8;
        if (par == 1) {
#pragma unroll
            for (int j = 0; j < NT8; ++j)
#pragma unroll
                for (int k = 0; k < 4; ++k) p[j * 4 + k] = facc[j][k];
        }
        ptx::named_bar_sync(1 + sub, 64);
        if (par == 0) {
#pragma unroll
            for (int j = 0; j < NT8; ++j)
#pragma unroll
                for (int k = 0; k < 4; ++k) facc[j][k] += p[j * 4 + k];
        }
        ptx::named_bar_sync(1 + sub, 64);
        if (par == 1) return;
    }
    dec_flush_warp<NT8, TP>(a, tile, facc, sub, lane, pend);
}

// Consumer loop over the CTA's stages (must enumerate stages exactly like the
// producer).  Consumer warp w works on sub-tile w for every group.
template <int WBITS, int NT8, int SPG, int MODE, bool PARTIALS, bool TP>
__device__ __forceinline__ void dec_consume(const DecArgs& a, uint32_t bar_full, uint32_t bar_empty,
                                            uint32_t stage0, int u0, int u1, uint32_t is16_mask) {
    const WLayout& L = a.L;
    const int NG = L.NG;
    const int S = a.stages;
    const int lane = threadIdx.x & 31, sub = (threadIdx.x >> 5) & 7, par = threadIdx.x >> 8;
    constexpr int GSTEP = DEC_CWARPS / 8;
    const uint32_t stage_bytes = (uint32_t)a.stage_bytes;
    int s = 0;
    uint32_t ph = 0;
    int cur_tile = -1;
    int* pend = nullptr;  // lane 0: counter to bump once the published slot landed
    float facc[NT8][4];
#pragma unroll
    for (int j = 0; j < NT8; ++j)
#pragma unroll
        for (int k = 0; k < 4; ++k) facc[j][k] = 0.f;
    const int gps = a.gps;
    int tile = u0 / NG, g0 = u0 - (u0 / NG) * NG;  // one division per CTA, then incremental
    for (int u = u0; u < u1;) {
        if (g0 == NG) { g0 = 0; ++tile; }
        int n = NG - g0;
        n = n < gps ? n : gps;
        n = n < u1 - u ? n : u1 - u;
        if (!PARTIALS && tile != cur_tile) {
            if (cur_tile >= 0) dec_tile_done<NT8, TP>(a, cur_tile, facc, sub, par, lane, pend);
            cur_tile = tile;
#pragma unroll
            for (int j = 0; j < NT8; ++j)
#pragma unroll
                for (int k = 0; k < 4; ++k) facc[j][k] = 0.f;
        }
        const int nsub = (tile == L.T128 - 1) ? L.nsub_last : 8;
        ptx::mbar_wait_u32(bar_full + 8 * s, ph);
        if (a.trace && u == u0 && threadIdx.x == 0) trace_ev(a.trace, a.serial, 1, 3);
        if (sub < nsub) {
            const uint32_t st = stage0 + s * stage_bytes;
#pragma unroll DEC_UNROLL
            for (int gi = GSTEP == 1 ? 0 : par; gi < n; gi += GSTEP)
                dec_group<WBITS, NT8, SPG, MODE, PARTIALS>(a, st, gi, g0 + gi, tile, nsub, facc, is16_mask);
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_u32(bar_empty + 8 * s);
        if (!PARTIALS) dec_publish(pend, lane);
        if (++s == S) { s = 0; ph ^= 1; }
        u += n;
        g0 += n;
    }
    if constexpr (!PARTIALS) {
        if (cur_tile >= 0) dec_tile_done<NT8, TP>(a, cur_tile, facc, sub, par, lane, pend);
        dec_publish(pend, lane);
    }
    if (threadIdx.x == 0) trace_ev(a.trace, a.serial, 1, 4);
}

template <int WBITS, int NT8, int SPG, bool PARTIALS, bool TP>
__global__ void __launch_bounds__(DEC_THREADS, NT8 == 1 ? DEC_MINB : 1) qlinear_decode_kernel(const DecArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    const WLayout& L = a.L;
    const int S = a.stages;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + S;
    uint8_t* stage0 = smem + 256;
    const int NG = L.NG;
    constexpr int G = SPG * 64;
    constexpr int CPS = NT8 * 8 * G + NT8 * 64;
    constexpr int X16S = NT8 * 8 * G * 2;
    if (gate_closed(a.gate)) return;
    const int U = L.T128 * NG;
    const int u0 = blockIdx.x * a.upc;
    const int u1 = min(U, u0 + a.upc);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int stage_bytes = a.stage_bytes;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], DEC_CWARPS);
        }
        if constexpr (TP) s_tp_subtiles = 0;
        ptx::fence_mbar_init();
        trace_ev(a.trace, a.serial, 1, 0);
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
            trace_ev(a.trace, a.serial, 1, 1);
            bool any16 = false;
            for (int m = 0; m < a.M; ++m) any16 |= ((a.row_bits ? a.row_bits[a.m0 + m] : a.bits) == 16);
            auto issue_a = [&](int s, int g0, int n) {
                uint8_t* st = stage0 + (size_t)s * stage_bytes;
                ptx::mbar_arrive_expect_tx(&full[s], n * CPS + (any16 ? n * X16S : 0));
                ptx::bulk_g2s(st + a.off_cp, a.ws + a.A.cp_off + (size_t)g0 * CPS, n * CPS, &full[s]);
                if (any16) ptx::bulk_g2s(st + a.off_x16, a.ws + a.A.x16_off + (size_t)g0 * X16S, n * X16S, &full[s]);
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
            trace_ev(a.trace, a.serial, 1, 2);
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
    if (!any16 && dec_call_centred(a.M, a.m0, a.row_bits, a.bits))
        dec_consume<WBITS, NT8, SPG, MODE_INTC, PARTIALS, TP>(a, bar_full, bar_empty, st0, u0, u1, is16_mask);
    else if (PARTIALS || (any_int && any16))
        dec_consume<WBITS, NT8, SPG, MODE_MIXED, PARTIALS, TP>(a, bar_full, bar_empty, st0, u0, u1, is16_mask);
    else if (any16)
        dec_consume<WBITS, NT8, SPG, MODE_A16, PARTIALS, TP>(a, bar_full, bar_empty, st0, u0, u1, is16_mask);
    else
        dec_consume<WBITS, NT8, SPG, MODE_INT, PARTIALS, TP>(a, bar_full, bar_empty, st0, u0, u1, is16_mask);
    if constexpr (TP) dec_tp_announce(a);
}

// ------------------------------------------------------------------ host
struct DecPlan {
    int upc, grid, gps, stages, stage_bytes;
    int off_meta, off_cp, off_x16;
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

// Stage = gps units of one tile: codes | metadata | activation records | bf16 rows.
// Shared memory budget 200 KB (one CTA per SM with 16 consumer warps); the
// 8-warp build (-DDYQ_DEC_CWARPS=8) keeps <= 113 KB so two CTAs fit per SM.
static DecPlan dec_plan(const WLayout& L, int nt8) {
    DecPlan p;
    const int unit_codes = (L.G / 64) * 8 * L.chunk;  // full tile
    // Stage code bytes: 56 KB (14 W4 groups) measured best for the bench step
    // (B200, M = 8, same-box sweep: 32 KB 59.35, 40 59.56, 48 59.27, 52 58.62,
    // 56 58.07, 60 60.48, 64 59.41 us/step); halved until at least two stages
    // fit the shared-memory budget.
    static const int stage_code_kb = env_int("DYQ_DEC_STAGE_KB", 56);
    static const int smem_kb1 = env_int("DYQ_DEC_SMEM_KB", 113);
    static const int smem_kb16 = env_int("DYQ_DEC_BUDGET_KB", 200);  // 16-warp build; <= 224 (dynamic-smem attribute)
    const int smem_kb = (nt8 == 1 && DEC_CWARPS == 8) ? smem_kb1 : (smem_kb16 > 224 ? 224 : smem_kb16);
    const int cps = nt8 * 8 * L.G + nt8 * 64, x16s = nt8 * 8 * L.G * 2;
    for (int want = (stage_code_kb * 1024) / unit_codes;; want /= 2) {
        p.gps = want < 1 ? 1 : (want > L.NG ? L.NG : want);
        p.off_meta = p.gps * unit_codes;
        p.off_cp = p.off_meta + p.gps * META_BLOCK;
        p.off_x16 = p.off_cp + p.gps * cps;
        p.stage_bytes = p.off_x16 + p.gps * x16s;
        p.stages = (smem_kb * 1024 - 256 - 16 * 1024) / p.stage_bytes;
        if (p.stages >= 2 || p.gps == 1) break;
    }
    p.stages = p.stages < 2 ? 2 : (p.stages > 8 ? 8 : p.stages);
    p.smem = 256 + (size_t)p.stages * p.stage_bytes + 8 * 32 * 8 * 4 + 8 * 1024;  // + combine + slot scratch
    const int U = L.T128 * L.NG;
    static const int ctas = env_int("DYQ_DEC_CTAS", 1);
    const int target = num_sms() * ctas;
    p.upc = (U + target - 1) / target;
    if (p.upc < 1) p.upc = 1;
    p.grid = (U + p.upc - 1) / p.upc;
    return p;
}

// split-K slot storage: (grid + T128) slots of 16 x 128 floats, then T128 x 8 counters
size_t decode_ws_bytes(const WLayout& L) {
    const DecPlan p = dec_plan(L, 2);
    return (size_t)(p.grid + L.T128) * 16 * 128 * 4 + (((size_t)L.T128 * 8 * 4 + 255) & ~(size_t)255);
}

template <int WBITS, int NT8, int SPG, bool PARTIALS, bool TP>
static cudaError_t launch_k2(const DecArgs& a, const DecPlan& p, cudaStream_t st) {
    auto kern = qlinear_decode_kernel<WBITS, NT8, SPG, PARTIALS, TP>;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024);  // + static smem <= 227 KB
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

template <int WBITS, int NT8, bool PARTIALS, bool TP = false>
static cudaError_t launch_k(const DecArgs& a, const DecPlan& p, cudaStream_t st) {
    return a.L.G == 64 ? launch_k2<WBITS, NT8, 1, PARTIALS, TP>(a, p, st)
                       : launch_k2<WBITS, NT8, 2, PARTIALS, TP>(a, p, st);
}

// L2 prefetch of a byte range (the next layer's packed weights): one thread per
// CTA issues cp.async.bulk.prefetch.L2 over its slice and the CTA exits; the
// HBM -> L2 transfer proceeds asynchronously while the dependent chain
// (act-quant -> decode) of the current layer runs.  Reads nothing produced by
// earlier kernels, so it triggers its dependents at once and never waits.
__global__ void prefetch_l2_kernel(const uint8_t* p, size_t bytes, size_t per_cta) {
    ptx::pdl_launch_dependents();
    if (threadIdx.x != 0) return;
    const size_t b0 = (size_t)blockIdx.x * per_cta;
    const size_t b1 = b0 + per_cta < bytes ? b0 + per_cta : bytes;
    for (size_t o = b0; o < b1; o += 32768) {
        const uint32_t n = (uint32_t)((b1 - o) < 32768 ? (b1 - o) : 32768);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p + o), "r"(n & ~15u) : "memory");
    }
}

dyq_status_t launch_prefetch_l2(const void* p, size_t bytes, cudaStream_t st) {
    if (bytes < 16) return DYQ_OK;
    const int ctas = num_sms();
    size_t per = (bytes + ctas - 1) / ctas;
    per = (per + 4095) & ~(size_t)4095;
    const unsigned grid = (unsigned)((bytes + per - 1) / per);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(32);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e =
        cudaLaunchKernelEx(&cfg, prefetch_l2_kernel, reinterpret_cast<const uint8_t*>(p), bytes, per);
    if (e != cudaSuccess) return set_error(DYQ_ECUDA, "prefetch_l2_kernel launch: %s", cudaGetErrorString(e));
    return DYQ_OK;
}

// ws layout: [split-K slots + tile counters (decode_ws_bytes, zeroed once,
// self-cleaning)] [activation area written by the quantizer kernel].
dyq_status_t launch_decode(const WLayout& L, const void* codes, const void* meta, const uint16_t* x, int M,
                           int m0, const int32_t* row_bits, int bits, void* y, int y_dtype, int32_t* I_out,
                           void* ws, int64_t* /*err*/, cudaStream_t st, const TpPeers* tp) {
    const int nt8 = dec_nt8(M);
    const ActLayoutDec A = act_layout_dec(L, nt8);
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
    a.off_cp = p.off_cp;
    a.off_x16 = p.off_x16;
    a.trace = g_trace;
    a.serial = g_trace_serial++;
    a.gate = g_gate;
    a.tp = {};
    if (tp) a.tp = *tp;
    const bool partials = I_out != nullptr;
    cudaError_t e;
#define DYQ_DISPATCH(WB)                                                                      \
    if (partials) e = nt8 == 1 ? launch_k<WB, 1, true>(a, p, st) : launch_k<WB, 2, true>(a, p, st); \
    else if (a.tp.n) e = nt8 == 1 ? launch_k<WB, 1, false, true>(a, p, st) : launch_k<WB, 2, false, true>(a, p, st); \
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
