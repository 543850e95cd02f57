// dyq_decode_ldg.cu -- decode-regime quantized linear layer, register-streaming
// variant (M <= 16 tokens).  Same math as dyq_decode.cu; different data path:
//
//  * no producer warp, no shared-memory ring: every warp streams its OWN
//    contiguous range of (16-row sub-tile, K-group) units (warp-granular
//    stream-K over N/16 x K/G units), keeping D = 4 units of packed weights
//    + metadata in flight in registers (128-bit non-allocating loads);
//  * the weight prefetch for the first D units is issued BEFORE
//    griddepcontrol.wait, so under programmatic dependent launch it overlaps
//    the activation quantizer that precedes this kernel;
//  * a sub-tile split across warps is reduced with fp32 atomics into a
//    [16][N] workspace block; the last contributor (per-sub-tile counter)
//    converts to the output dtype and clears the block (self-cleaning).
// Measured B200 read-stream ceiling for this access pattern: ~7.2-7.4 TB/s
// (tools/stream_bench.cu, ldg variant).
#include <stdlib.h>

#include "dyq_internal.cuh"
#include "dyq_ptx.cuh"

namespace dyq {

struct LdgArgs {
    WLayout L;
    const uint8_t* codes;
    const uint8_t* meta;
    const uint16_t* x;
    const int32_t* row_bits;
    int bits;
    int M, m0;
    void* y;
    int y_dtype;
    int32_t* I_out;
    const uint8_t* act;     // activation area (ActLayoutDec)
    ActLayoutDec A;
    float* acc;             // [16][N] fp32 (self-cleaning)
    int* counters;          // [N/16]
    int upw;                // units per warp
};

__device__ __forceinline__ uint4 ldg_nc128(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ uint2 ldg_nc64(const void* p) {
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t ldg_nc16(const void* p) {
    unsigned short r;
    asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(r) : "l"(p));
    return r;
}

__device__ __forceinline__ void mma_u8_l(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_bf16_l(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void fma2_l(float& d0, float& d1, float a0, float a1, float b0, float b1) {
    uint64_t d = ((uint64_t)__float_as_uint(d1) << 32) | __float_as_uint(d0);
    const uint64_t a = ((uint64_t)__float_as_uint(a1) << 32) | __float_as_uint(a0);
    const uint64_t b = ((uint64_t)__float_as_uint(b1) << 32) | __float_as_uint(b0);
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
    d0 = __uint_as_float((uint32_t)d);
    d1 = __uint_as_float((uint32_t)(d >> 32));
}
__device__ __forceinline__ void mul2_l(float& r0, float& r1, float a0, float a1, float b0, float b1) {
    uint64_t d;
    const uint64_t a = ((uint64_t)__float_as_uint(a1) << 32) | __float_as_uint(a0);
    const uint64_t b = ((uint64_t)__float_as_uint(b1) << 32) | __float_as_uint(b0);
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    r0 = __uint_as_float((uint32_t)d);
    r1 = __uint_as_float((uint32_t)(d >> 32));
}
template <int WBITS>
__device__ __forceinline__ uint32_t pair_bf16(uint32_t v, int hi_pair, uint32_t zz) {
    if (WBITS == 4) {
        const uint32_t t = __byte_perm(v, 0x4343u, hi_pair ? 0x5342u : 0x5140u);
        __nv_bfloat162 r = __hsub2(*reinterpret_cast<const __nv_bfloat162*>(&t),
                                   *reinterpret_cast<const __nv_bfloat162*>(&zz));
        return *reinterpret_cast<uint32_t*>(&r);
    } else {
        const uint32_t f0 = __byte_perm(v, 0x4B000000u, hi_pair ? 0x7542u : 0x7540u);
        const uint32_t f1 = __byte_perm(v, 0x4B000000u, hi_pair ? 0x7543u : 0x7541u);
        const float zf = __uint_as_float(zz);
        __nv_bfloat162 r = __floats2bfloat162_rn(__uint_as_float(f0) - zf, __uint_as_float(f1) - zf);
        return *reinterpret_cast<uint32_t*>(&r);
    }
}

enum { LM_INT = 0, LM_A16 = 1, LM_MIXED = 2 };
constexpr int LDG_D = 4;  // units in flight per warp

// Per-unit register payload: codes (W4: 1 x 16 B per slab pair; W8: 2 x 16 B), metadata.
template <int WBITS, int SPG>
struct UnitRegs {
    uint4 w[SPG * (WBITS / 4)];
    uint2 sw;
    uint32_t zw;
};

template <int WBITS, int SPG>
__device__ __forceinline__ void load_unit(const LdgArgs& a, int st, int g, int lane, int gid,
                                          UnitRegs<WBITS, SPG>& r) {
    const WLayout& L = a.L;
    const int tile = st >> 3, sub = st & 7;
#pragma unroll
    for (int spi = 0; spi < SPG; ++spi) {
        const uint8_t* ch = a.codes + chunk_offset(L, tile, g * SPG + spi, sub) + lane * 16;
#pragma unroll
        for (int h = 0; h < WBITS / 4; ++h) r.w[spi * (WBITS / 4) + h] = ldg_nc128(ch + h * 512);
    }
    const uint8_t* mb = a.meta + meta_block(L, tile, g);
    r.sw = ldg_nc64(mb + meta_slot(sub, gid) * 4);
    r.zw = ldg_nc16(mb + 512 + meta_slot(sub, gid));
}

template <int WBITS, int NT8, int SPG, int MODE, bool PARTIALS>
__device__ __forceinline__ void compute_unit(const LdgArgs& a, const UnitRegs<WBITS, SPG>& r, int st, int g,
                                             float (&facc)[NT8][4], uint32_t is16_mask, int lane) {
    constexpr int G = SPG * 64;
    const WLayout& L = a.L;
    const int gid = lane >> 2, t = lane & 3;
    const uint32_t ONES = 0x01010101u;
    const float sw0 = __uint_as_float(r.sw.x), sw1 = __uint_as_float(r.sw.y);
    const int zw0 = r.zw & 0xff, zw1 = r.zw >> 8;
    uint32_t zz_g = 0, zz_g8 = 0;
    if (MODE != LM_INT) {
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
        uint32_t A[2][4];
        if (WBITS == 4) {
            const uint4 w = r.w[spi];
            A[0][0] = w.x & 0x0F0F0F0Fu;
            A[0][1] = w.y & 0x0F0F0F0Fu;
            A[0][2] = (w.x >> 4) & 0x0F0F0F0Fu;
            A[0][3] = (w.y >> 4) & 0x0F0F0F0Fu;
            A[1][0] = w.z & 0x0F0F0F0Fu;
            A[1][1] = w.w & 0x0F0F0F0Fu;
            A[1][2] = (w.z >> 4) & 0x0F0F0F0Fu;
            A[1][3] = (w.w >> 4) & 0x0F0F0F0Fu;
        } else {
            const uint4 w0 = r.w[spi * 2], w1 = r.w[spi * 2 + 1];
            A[0][0] = w0.x; A[0][1] = w0.y; A[0][2] = w0.z; A[0][3] = w0.w;
            A[1][0] = w1.x; A[1][1] = w1.y; A[1][2] = w1.z; A[1][3] = w1.w;
        }
        if (MODE != LM_A16) {
            mma_u8_l(sq, A[0], ONES, ONES);
            mma_u8_l(sq, A[1], ONES, ONES);
#pragma unroll
            for (int j = 0; j < NT8; ++j) {
                const uint4 xb = __ldg(reinterpret_cast<const uint4*>(
                    a.act + a.A.xq_off + act_xq_index(L.NG, G, j * 8 + gid, g, spi * 64 + t * 16)));
                mma_u8_l(iacc[j], A[0], xb.x, xb.y);
                mma_u8_l(iacc[j], A[1], xb.z, xb.w);
            }
        }
        if (MODE != LM_INT) {
#pragma unroll
            for (int j = 0; j < NT8; ++j) {
                const uint8_t* xr =
                    a.act + a.A.x16_off + act_xq_index(L.NG, G, j * 8 + gid, g, spi * 64 + t * 16) * 2;
                const uint4 xa = __ldg(reinterpret_cast<const uint4*>(xr));
                const uint4 xc = __ldg(reinterpret_cast<const uint4*>(xr + 16));
#pragma unroll
                for (int s2 = 0; s2 < 2; ++s2) {
                    const uint4 xx = s2 ? xc : xa;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const uint32_t rg = A[s2][h * 2 + 0], rg8 = A[s2][h * 2 + 1];
                        uint32_t A16[4];
                        A16[0] = pair_bf16<WBITS>(rg, 0, zz_g);
                        A16[1] = pair_bf16<WBITS>(rg8, 0, zz_g8);
                        A16[2] = pair_bf16<WBITS>(rg, 1, zz_g);
                        A16[3] = pair_bf16<WBITS>(rg8, 1, zz_g8);
                        mma_bf16_l(hacc[j], A16, h ? xx.z : xx.x, h ? xx.w : xx.y);
                    }
                }
            }
        }
    }
    const int T_g = sq[0] - G * zw0;
    const int T_g8 = sq[2] - G * zw1;
#pragma unroll
    for (int j = 0; j < NT8; ++j) {
        uint4 pp = make_uint4(0u, 0u, 0u, 0u);
        if (MODE != LM_A16)
            pp = __ldg(reinterpret_cast<const uint4*>(a.act + a.A.par_off + ((size_t)g * DEC_MPAD + j * 8 + 2 * t) * 8));
        const float sx0 = __uint_as_float(pp.x), sx1 = __uint_as_float(pp.z);
        const int zx0 = (int)(pp.y >> 16), zx1 = (int)(pp.w >> 16);
        const int SX0 = (int)(pp.y & 0xffffu), SX1 = (int)(pp.w & 0xffffu);
        int I[4];
        I[0] = iacc[j][0] - zw0 * SX0 - zx0 * T_g;
        I[1] = iacc[j][1] - zw0 * SX1 - zx1 * T_g;
        I[2] = iacc[j][2] - zw1 * SX0 - zx0 * T_g8;
        I[3] = iacc[j][3] - zw1 * SX1 - zx1 * T_g8;
        if constexpr (PARTIALS) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int q = k & 1, hi = k >> 1;
                const int tc = j * 8 + 2 * t + q;
                if (tc < a.M) {
                    const bool a16 = (is16_mask >> (j * 2 + q)) & 1u;
                    const int n = st * 16 + gid + 8 * hi;
                    a.I_out[((size_t)(a.m0 + tc) * L.N + n) * L.NG + g] = a16 ? 0 : I[k];
                }
            }
        } else if (MODE == LM_INT) {
            float t0, t1, t2, t3;
            mul2_l(t0, t1, (float)I[0], (float)I[1], sx0, sx1);
            mul2_l(t2, t3, (float)I[2], (float)I[3], sx0, sx1);
            fma2_l(facc[j][0], facc[j][1], t0, t1, sw0, sw0);
            fma2_l(facc[j][2], facc[j][3], t2, t3, sw1, sw1);
        } else if (MODE == LM_A16) {
            fma2_l(facc[j][0], facc[j][1], hacc[j][0], hacc[j][1], sw0, sw0);
            fma2_l(facc[j][2], facc[j][3], hacc[j][2], hacc[j][3], sw1, sw1);
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

// flush a sub-tile's partial: direct store if this warp owns all of it,
// else fp32 atomics + last-arriver conversion.
template <int NT8>
__device__ __forceinline__ void ldg_flush(const LdgArgs& a, int st, const float (&facc)[NT8][4], int lane) {
    const WLayout& L = a.L;
    const int gid = lane >> 2, t = lane & 3;
    const int NG = L.NG;
    const int nc = ((st + 1) * NG - 1) / a.upw - (st * NG) / a.upw + 1;
    auto store = [&](size_t o, float v) {
        if (a.y_dtype == 0)
            reinterpret_cast<float*>(a.y)[o] = v;
        else
            reinterpret_cast<__nv_bfloat16*>(a.y)[o] = __float2bfloat16_rn(v);
    };
    if (nc == 1) {
#pragma unroll
        for (int j = 0; j < NT8; ++j)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int tok = j * 8 + 2 * t + (i & 1);
                if (tok < a.M) store((size_t)(a.m0 + tok) * L.N + st * 16 + gid + 8 * (i >> 1), facc[j][i]);
            }
        return;
    }
#pragma unroll
    for (int j = 0; j < NT8; ++j)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int tok = j * 8 + 2 * t + (i & 1);
            if (tok < a.M) atomicAdd(&a.acc[(size_t)tok * L.N + st * 16 + gid + 8 * (i >> 1)], facc[j][i]);
        }
    __threadfence();
    __syncwarp();
    int last = 0;
    if (lane == 0) last = (atomicAdd(&a.counters[st], 1) == nc - 1);
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
        __threadfence();
        for (int idx = lane; idx < a.M * 16; idx += 32) {
            const int tok = idx >> 4, r = idx & 15;
            float* p = &a.acc[(size_t)tok * L.N + st * 16 + r];
            const float v = __ldcg(p);
            __stcg(p, 0.f);
            store((size_t)(a.m0 + tok) * L.N + st * 16 + r, v);
        }
        if (lane == 0) a.counters[st] = 0;
    }
}

template <int WBITS, int NT8, int SPG, int MODE, bool PARTIALS>
__device__ __forceinline__ void ldg_run(const LdgArgs& a, int u0, int u1, UnitRegs<WBITS, SPG> (&ring)[LDG_D],
                                        uint32_t is16_mask, int lane) {
    const int NG = a.L.NG;
    float facc[NT8][4];
#pragma unroll
    for (int j = 0; j < NT8; ++j)
#pragma unroll
        for (int k = 0; k < 4; ++k) facc[j][k] = 0.f;
    int st = u0 / NG, g = u0 - st * NG;          // unit being computed
    int lst = st, lg = g;                         // unit being loaded (ahead by D)
#pragma unroll
    for (int d = 0; d < LDG_D; ++d)
        if (++lg == NG) { lg = 0; ++lst; }
    for (int u = u0; u < u1; u += LDG_D) {
#pragma unroll
        for (int d = 0; d < LDG_D; ++d) {
            if (u + d < u1) {
                compute_unit<WBITS, NT8, SPG, MODE, PARTIALS>(a, ring[d], st, g, facc, is16_mask, lane);
                if (u + d + LDG_D < u1) load_unit<WBITS, SPG>(a, lst, lg, lane, lane >> 2, ring[d]);
                if (++lg == NG) { lg = 0; ++lst; }
                if (++g == NG || u + d + 1 == u1) {
                    if constexpr (!PARTIALS) {
                        ldg_flush<NT8>(a, st, facc, lane);
#pragma unroll
                        for (int j = 0; j < NT8; ++j)
#pragma unroll
                            for (int k = 0; k < 4; ++k) facc[j][k] = 0.f;
                    }
                    if (g == NG) { g = 0; ++st; }
                }
            }
        }
    }
}

template <int WBITS, int NT8, int SPG, bool PARTIALS>
__global__ void __launch_bounds__(256) qlinear_decode_ldg_kernel(const LdgArgs a) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int U = (a.L.N / 16) * a.L.NG;
    const int u0 = gw * a.upw, u1 = min(U, u0 + a.upw);
    UnitRegs<WBITS, SPG> ring[LDG_D];
    // weights first: independent of the preceding kernels
    {
        int st = u0 / a.L.NG, g = u0 - (u0 / a.L.NG) * a.L.NG;
#pragma unroll
        for (int d = 0; d < LDG_D; ++d) {
            if (u0 + d < u1) load_unit<WBITS, SPG>(a, st, g, lane, lane >> 2, ring[d]);
            if (++g == a.L.NG) { g = 0; ++st; }
        }
    }
    ptx::pdl_launch_dependents();
    ptx::pdl_wait();  // activations / row_bits come from the preceding kernels
    if (u0 >= u1) return;
    const int gid = lane >> 2, t = lane & 3;
    bool any_int = false, any16 = false;
    uint32_t is16_mask = 0;
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
    if (PARTIALS || (any_int && any16))
        ldg_run<WBITS, NT8, SPG, LM_MIXED, PARTIALS>(a, u0, u1, ring, is16_mask, lane);
    else if (any16)
        ldg_run<WBITS, NT8, SPG, LM_A16, PARTIALS>(a, u0, u1, ring, is16_mask, lane);
    else
        ldg_run<WBITS, NT8, SPG, LM_INT, PARTIALS>(a, u0, u1, ring, is16_mask, lane);
}

static int ldg_env(const char* n, int d) {
    const char* v = getenv(n);
    return v ? atoi(v) : d;
}

static int ldg_num_sms() {
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

// workspace for this path: fp32 [16][N] + counters [N/16]
size_t decode_ldg_ws_bytes(const WLayout& L) {
    return (size_t)DEC_MPAD * L.N * 4 + (((size_t)(L.N / 16) * 4 + 255) & ~(size_t)255);
}

template <int WBITS, int NT8, int SPG, bool PARTIALS>
static cudaError_t ldg_launch(const LdgArgs& a, int grid, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, qlinear_decode_ldg_kernel<WBITS, NT8, SPG, PARTIALS>, a);
}

dyq_status_t launch_decode_ldg(const WLayout& L, const void* codes, const void* meta, const uint16_t* x, int M,
                               int m0, const int32_t* row_bits, int bits, void* y, int y_dtype, int32_t* I_out,
                               void* ws_dec, const void* act, cudaStream_t st) {
    const int nt8 = M <= 8 ? 1 : 2;
    LdgArgs a;
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
    a.act = reinterpret_cast<const uint8_t*>(act);
    a.A = act_layout_dec(L);
    a.acc = reinterpret_cast<float*>(ws_dec);
    a.counters = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(ws_dec) + (size_t)DEC_MPAD * L.N * 4);
    static const int wpsm = ldg_env("DYQ_LDG_WARPS_PER_SM", 32);
    const int U = (L.N / 16) * L.NG;
    const int target = ldg_num_sms() * wpsm;
    a.upw = (U + target - 1) / target;
    if (a.upw < 1) a.upw = 1;
    const int warps = (U + a.upw - 1) / a.upw;
    const int grid = (warps + 7) / 8;
    const bool partials = I_out != nullptr;
    cudaError_t e;
#define DYQ_LDG(WB, SPG)                                                                                \
    if (partials) e = nt8 == 1 ? ldg_launch<WB, 1, SPG, true>(a, grid, st) : ldg_launch<WB, 2, SPG, true>(a, grid, st); \
    else e = nt8 == 1 ? ldg_launch<WB, 1, SPG, false>(a, grid, st) : ldg_launch<WB, 2, SPG, false>(a, grid, st);
    if (L.wbits == 4) {
        if (L.G == 64) { DYQ_LDG(4, 1) } else { DYQ_LDG(4, 2) }
    } else {
        if (L.G == 64) { DYQ_LDG(8, 1) } else { DYQ_LDG(8, 2) }
    }
#undef DYQ_LDG
    if (e != cudaSuccess) return set_error(DYQ_ECUDA, "qlinear_decode_ldg_kernel launch: %s", cudaGetErrorString(e));
    return check_launch("qlinear_decode_ldg_kernel");
}

}  // namespace dyq
