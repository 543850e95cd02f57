// dyq_prefill.cu -- the prefill-regime quantized linear layer (M > 16 tokens):
// a warp-specialised tcgen05 GEMM with TMEM accumulators (sm_100a).
//
// "the packed activations ... utilize native INT4 and INT8
// Tensor Cores"; "the computationally intensive visual prefill".  On
// sm_100a there is no int4 MMA (tcgen05 .kind::i4 does not exist), so every
// integer width runs on the 8-bit tensor pipe (tcgen05.mma .kind::i8 -> s32);
// the BF16 bypass runs .kind::f16 (bf16 x bf16 -> f32).
//
// CTA = one 128-row weight tile x one 144-token tile (288 = 2 x 144: the
// OpenVLA prefill of 256 vision + 32 text tokens tiles exactly), whole K:
//   warp 0      producer: per K-group, bulk copies (TMA engine) of the packed
//               codes, the 640-B metadata block, the activation operand (already
//               in the UMMA canonical K-major layout, written by the prefill
//               activation quantizer) and the token scales;
//   warp 1      MMA issuer (one thread): tcgen05.mma per 32-B K step into a
//               double-buffered TMEM accumulator (one buffer per group);
//   warps 2-3   transform: packed int4 -> 8-bit (or bf16 (q - z_w)) operand in
//               the canonical no-swizzle K-major layout;
//   warps 4-11  promotion: tcgen05.ld the group's sums, scale by s_x s_w and
//               accumulate fp32 in registers; store y at the end.
//
// Zero points: when the weights are W4 and no token of the
// tile runs at 8 bits, BOTH operands are centred -- A = q - z_w (transform) and
// B = Xq - z_x (quantizer), each in [-15, 15] -- so the s8 x s8 MMA yields the
// exact group sum I = Sum (Xq - z_x)(q - z_w) directly and the promotion is only
// acc += float(I) * s_x * s_w (INTC mode).  Otherwise (A8 or W8 operands do not
// fit s8) u8 x u8 codes are multiplied and the promotion applies
//     I = P - z_w SX - z_x (Sum q - G z_w)
// with Sum q taken from an all-ones token column of the MMA (INTU mode).
// The per-group promotion is intrinsic to per-group scales on both operands: it
// bounds the tensor pipe to roughly G / (64 c) of peak for c CUDA-core
// instructions per accumulator element (c ~ 2.25 in INTC mode).
#include <stdlib.h>

#include "dyq_internal.cuh"
#include "dyq_ptx.cuh"

namespace dyq {

constexpr int PT = 144;   // real tokens per token tile
constexpr int PTE = 160;  // operand rows in the code layout (row 144 = all-ones column)
constexpr int PRE_WARPS = 12;
constexpr int PRE_THREADS = PRE_WARPS * 32;
constexpr int PAR_BYTES = PT * 8;  // per (tile, group): float s_x[144] then uint32 (z_x<<16|SX)[144]

struct PreArgs {
    WLayout L;
    const uint8_t* codes;
    const uint8_t* meta;
    const int32_t* row_bits;
    int bits;
    int M;
    void* y;
    int y_dtype;
    int32_t* I_out;
    const uint8_t* act;  // prefill activation area
    PreActLayout P;
    int stages, stage_bytes;
    int off_meta, off_b, off_par, off_a;
};

enum { PMODE_INTC = 0, PMODE_INTU = 1, PMODE_BF16 = 2 };

__device__ __forceinline__ int token_bits(const PreArgs& a, int m) { return a.row_bits ? a.row_bits[m] : a.bits; }

// tile flags: bit0 int tokens, bit1 A16 tokens, bit2 A8 tokens
__device__ __forceinline__ int tile_flags_from_bits(int b) { return b == 16 ? 2 : (b == 8 ? 5 : 1); }

template <int WBITS, int SPG, int MODE, bool PARTIALS>
__global__ void __launch_bounds__(PRE_THREADS, 1) qlinear_prefill_kernel(const PreArgs a) {
    constexpr int G = SPG * 64;
    constexpr bool INT = MODE != PMODE_BF16;
    constexpr int KSTEPS = INT ? G / 32 : G / 16;                     // MMA K steps per group
    constexpr int NMMA = MODE == PMODE_INTU ? PTE : PT;               // MMA N
    constexpr uint32_t BSTEP = INT ? PTE * 32 : PT * 32;              // bytes per K step of B in smem
    const WLayout& L = a.L;
    const int tile = blockIdx.x, tt = blockIdx.y;
    const int NG = L.NG;
    const int S = a.stages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nsub = (tile == L.T128 - 1) ? L.nsub_last : 8;

    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* xformed = full + S;
    uint64_t* empty = xformed + S;
    uint64_t* tfull = empty + S;   // [2]
    uint64_t* tempty = tfull + 2;  // [2]
    uint32_t* s_tmem = reinterpret_cast<uint32_t*>(tempty + 2);
    int* s_flags = reinterpret_cast<int*>(s_tmem + 1);
    uint8_t* stage0 = smem + 1024;

    // which kinds of tokens live in this token tile? (same rule as the quantizer)
    if (threadIdx.x == 0) *s_flags = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < PT; i += PRE_THREADS) {
        const int m = tt * PT + i;
        if (m < a.M) atomicOr(s_flags, tile_flags_from_bits(token_bits(a, m)));
    }
    __syncthreads();
    const int flags = *s_flags;
    const bool centred = (L.wbits == 4) && !(flags & 4);
    bool run;
    if (PARTIALS) run = flags != 0 && (MODE == PMODE_INTC ? centred : !centred);
    else if (MODE == PMODE_BF16) run = (flags & 2) != 0;
    else run = (flags & 1) && (MODE == PMODE_INTC ? centred : !centred);
    if (!run) return;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&xformed[s], 2);    // 2 transform warps
            ptx::mbar_init(&empty[s], 1 + 8);  // MMA commit + 8 promotion warps
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&tfull[b], 1);
            ptx::mbar_init(&tempty[b], 8);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 1) {
        tc::alloc(ptx::smem_u32(s_tmem), 512);
        tc::relinquish();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = *s_tmem;
    const uint32_t sbase = ptx::smem_u32(stage0);

    if (warp == 0) {
        // ------------------------------------------------------ producer
        if (lane == 0) {
            const uint32_t cbytes = (uint32_t)(SPG * nsub * L.chunk);
            const uint32_t bbytes = KSTEPS * BSTEP;
            for (int g = 0; g < NG; ++g) {
                const int s = g % S;
                if (g >= S) ptx::mbar_wait(&empty[s], ((g / S) - 1) & 1);
                uint8_t* st = stage0 + (size_t)s * a.stage_bytes;
                ptx::mbar_arrive_expect_tx(&full[s], cbytes + META_BLOCK + bbytes + PAR_BYTES);
                ptx::bulk_g2s(st, a.codes + chunk_offset(L, tile, g * SPG, 0), cbytes, &full[s]);
                ptx::bulk_g2s(st + a.off_meta, a.meta + meta_block(L, tile, g), META_BLOCK, &full[s]);
                const size_t tg = (size_t)tt * NG + g;
                if (INT)
                    ptx::bulk_g2s(st + a.off_b, a.act + a.P.codes_off + tg * a.P.codes_group, bbytes, &full[s]);
                else
                    ptx::bulk_g2s(st + a.off_b, a.act + a.P.x16_off + tg * a.P.x16_group, bbytes, &full[s]);
                ptx::bulk_g2s(st + a.off_par, a.act + a.P.par_off + tg * PAR_BYTES, PAR_BYTES, &full[s]);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------ MMA issuer
        const uint32_t idesc = MODE == PMODE_INTC   ? tc::idesc_i8_s8s8(128, NMMA)
                               : MODE == PMODE_INTU ? tc::idesc_i8_u8u8(128, NMMA)
                                                    : tc::idesc_bf16(128, NMMA);
        for (int g = 0; g < NG; ++g) {
            const int s = g % S, b = g & 1;
            ptx::mbar_wait(&xformed[s], (g / S) & 1);
            if (g >= 2) ptx::mbar_wait(&tempty[b], ((g >> 1) - 1) & 1);
            tc::fence_after();
            if (lane == 0) {
                const uint32_t st = sbase + s * a.stage_bytes;
                const uint32_t d = tmem + b * 256;
#pragma unroll
                for (int ks = 0; ks < KSTEPS; ++ks) {
                    const uint64_t ad = tc::smem_desc(st + a.off_a + ks * 4096, 128, 256);
                    const uint64_t bd = tc::smem_desc(st + a.off_b + ks * BSTEP, 128, 256);
                    if (INT)
                        tc::mma_i8(d, ad, bd, idesc, ks > 0);
                    else
                        tc::mma_f16(d, ad, bd, idesc, ks > 0);
                }
                tc::commit(ptx::smem_u32(&tfull[b]));
                tc::commit(ptx::smem_u32(&empty[s]));
            }
            __syncwarp();
        }
    } else if (warp < 4) {
        // ------------------------------------------------------ transform
        const int tid = threadIdx.x - 64;  // 0..63
        for (int g = 0; g < NG; ++g) {
            const int s = g % S;
            ptx::mbar_wait(&full[s], (g / S) & 1);
            uint8_t* st = stage0 + (size_t)s * a.stage_bytes;
            uint8_t* A = st + a.off_a;
            const uint8_t* zrow = st + a.off_meta + 512;
            if (WBITS == 4) {
                // SPG * nsub * 32 lane-chunks of 16 B: [spi][sub][lane]
                for (int c = tid; c < SPG * nsub * 32; c += 64) {
                    const int spi = c / (nsub * 32), cc = c - spi * nsub * 32;
                    const int sub = cc >> 5, ln = cc & 31;
                    const int gid = ln >> 2, t = ln & 3;
                    const uint4 w = *reinterpret_cast<const uint4*>(st + c * 16);
                    const uint32_t ws4[4] = {w.x, w.y, w.z, w.w};  // (slab0,r0) (slab0,r1) (slab1,r0) (slab1,r1)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int slab = j >> 1, r = sub * 16 + gid + 8 * (j & 1);
                        uint32_t lo = ws4[j] & 0x0F0F0F0Fu, hi = (ws4[j] >> 4) & 0x0F0F0F0Fu;
                        if (MODE == PMODE_INTC) {
                            // s8 (q - z_w): (128 + q - z) per byte never borrows, then flip the sign bit
                            const uint32_t zz = (uint32_t)zrow[meta_slot(sub, r & 15)] * 0x01010101u;
                            lo = ((lo | 0x80808080u) - zz) ^ 0x80808080u;
                            hi = ((hi | 0x80808080u) - zz) ^ 0x80808080u;
                        }
                        if (INT) {
                            uint8_t* p = A + (spi * 2 + slab) * 4096 + (r >> 3) * 256 + (r & 7) * 16 + 4 * t;
                            *reinterpret_cast<uint32_t*>(p) = lo;
                            *reinterpret_cast<uint32_t*>(p + 128) = hi;
                        } else {
                            const uint32_t zw = zrow[meta_slot(sub, r & 15)];
                            const uint32_t zz = 0x43004300u | (zw << 16) | zw;
                            const __nv_bfloat162 z2 = *reinterpret_cast<const __nv_bfloat162*>(&zz);
                            const uint32_t plo0 = __byte_perm(lo, 0x4343u, 0x5140u), plo1 = __byte_perm(lo, 0x4343u, 0x5342u);
                            const uint32_t phi0 = __byte_perm(hi, 0x4343u, 0x5140u), phi1 = __byte_perm(hi, 0x4343u, 0x5342u);
                            __nv_bfloat162 t0 = __hsub2(*reinterpret_cast<const __nv_bfloat162*>(&plo0), z2);
                            __nv_bfloat162 t1 = __hsub2(*reinterpret_cast<const __nv_bfloat162*>(&plo1), z2);
                            __nv_bfloat162 t2 = __hsub2(*reinterpret_cast<const __nv_bfloat162*>(&phi0), z2);
                            __nv_bfloat162 t3 = __hsub2(*reinterpret_cast<const __nv_bfloat162*>(&phi1), z2);
                            // lo nibbles: k = 32*slab + 4t + b -> K step 4*spi + 2*slab, hi: +1
                            const int ks = spi * 4 + slab * 2;
                            const int off = (r >> 3) * 256 + (t >> 1) * 128 + (r & 7) * 16 + (t & 1) * 8;
                            *reinterpret_cast<uint2*>(A + ks * 4096 + off) =
                                make_uint2(*reinterpret_cast<uint32_t*>(&t0), *reinterpret_cast<uint32_t*>(&t1));
                            *reinterpret_cast<uint2*>(A + (ks + 1) * 4096 + off) =
                                make_uint2(*reinterpret_cast<uint32_t*>(&t2), *reinterpret_cast<uint32_t*>(&t3));
                        }
                    }
                }
            } else {
                // W8: [spi][sub][slab][lane][16 B = R0 R1 R2 R3]
                for (int c = tid; c < SPG * nsub * 64; c += 64) {
                    const int spi = c / (nsub * 64), cc = c - spi * nsub * 64;
                    const int sub = cc >> 6, slab = (cc >> 5) & 1, ln = cc & 31;
                    const int gid = ln >> 2, t = ln & 3;
                    const uint4 w = *reinterpret_cast<const uint4*>(st + c * 16);
                    const uint32_t R[4] = {w.x, w.y, w.z, w.w};  // (r0,h0) (r1,h0) (r0,h1) (r1,h1)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int r = sub * 16 + gid + 8 * (j & 1), h = j >> 1;
                        if (INT) {
                            uint8_t* p = A + (spi * 2 + slab) * 4096 + (r >> 3) * 256 + h * 128 + (r & 7) * 16 + 4 * t;
                            *reinterpret_cast<uint32_t*>(p) = R[j];
                        } else {
                            const float zf = 8388608.f + (float)zrow[meta_slot(sub, r & 15)];
                            float f[4];
#pragma unroll
                            for (int bb = 0; bb < 4; ++bb)
                                f[bb] = __uint_as_float(__byte_perm(R[j], 0x4B000000u, 0x7540u + bb)) - zf;
                            __nv_bfloat162 p0 = __floats2bfloat162_rn(f[0], f[1]);
                            __nv_bfloat162 p1 = __floats2bfloat162_rn(f[2], f[3]);
                            const int ks = spi * 4 + slab * 2 + h;
                            const int off = (r >> 3) * 256 + (t >> 1) * 128 + (r & 7) * 16 + (t & 1) * 8;
                            *reinterpret_cast<uint2*>(A + ks * 4096 + off) =
                                make_uint2(*reinterpret_cast<uint32_t*>(&p0), *reinterpret_cast<uint32_t*>(&p1));
                        }
                    }
                }
            }
            tc::fence_proxy_async_smem();  // generic smem writes -> async proxy (MMA operand)
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&xformed[s]);
        }
    } else {
        // ------------------------------------------------------ promotion
        const int e = warp - 4;      // 0..7
        const int q = warp & 3;      // TMEM lane quadrant (hardware: warp id % 4)
        const int h = e >> 2;        // column half: tokens [72h, 72h + 72)
        const int r = q * 32 + lane;  // weight row in the tile = TMEM lane
        const int sub = r >> 4, rr = r & 15;
        constexpr int NC = PT / 2;   // 72 columns per thread
        float facc[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) facc[c] = 0.f;
        for (int g = 0; g < NG; ++g) {
            const int s = g % S, b = g & 1;
            ptx::mbar_wait(&tfull[b], (g >> 1) & 1);
            tc::fence_after();
            const uint8_t* st = stage0 + (size_t)s * a.stage_bytes;
            const float sw = reinterpret_cast<const float*>(st + a.off_meta)[meta_slot(sub, rr)];
            const int zw = st[a.off_meta + 512 + meta_slot(sub, rr)];
            const float* sxp = reinterpret_cast<const float*>(st + a.off_par) + h * NC;
            const uint32_t* cxp = reinterpret_cast<const uint32_t*>(st + a.off_par + PT * 4) + h * NC;
            const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16) + b * 256;
            int T = 0;
            if (MODE == PMODE_INTU) {
                uint32_t sq;
                tc::ld1(tb + PT, sq);
                tc::wait_ld();
                T = (int)sq - G * zw;
            }
#pragma unroll
            for (int c0 = 0; c0 < NC; c0 += 24) {
                uint32_t v[24];
                tc::ld8(tb + h * NC + c0, &v[0]);
                tc::ld8(tb + h * NC + c0 + 8, &v[8]);
                tc::ld8(tb + h * NC + c0 + 16, &v[16]);
                tc::wait_ld();
                if (c0 + 24 == NC) {  // all columns of this buffer are in registers
                    tc::fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&tempty[b]);
                }
#pragma unroll
                for (int c = 0; c < 24; c += 4) {
                    const float4 sx4 = *reinterpret_cast<const float4*>(sxp + c0 + c);
                    const float sxv[4] = {sx4.x, sx4.y, sx4.z, sx4.w};
                    int I[4];
                    if (MODE == PMODE_INTU) {
                        const uint4 cx4 = *reinterpret_cast<const uint4*>(cxp + c0 + c);
                        const uint32_t cxv[4] = {cx4.x, cx4.y, cx4.z, cx4.w};
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            I[k] = (int)v[c + k] - zw * (int)(cxv[k] & 0xffffu) - (int)(cxv[k] >> 16) * T;
                    } else if (INT) {
#pragma unroll
                        for (int k = 0; k < 4; ++k) I[k] = (int)v[c + k];
                    }
                    if constexpr (PARTIALS) {
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const int m = tt * PT + h * NC + c0 + c + k;
                            if (m < a.M && r < nsub * 16)
                                a.I_out[((size_t)m * L.N + tile * 128 + r) * NG + g] =
                                    token_bits(a, m) == 16 ? 0 : I[k];
                        }
                    } else if (INT) {
#pragma unroll
                        for (int k = 0; k < 4; k += 2) {
                            float t0, t1;
                            ptx::mul2f(t0, t1, (float)I[k], (float)I[k + 1], sxv[k], sxv[k + 1]);
                            ptx::fma2f(facc[c0 + c + k], facc[c0 + c + k + 1], t0, t1, sw, sw);
                        }
                    } else {
#pragma unroll
                        for (int k = 0; k < 4; k += 2)
                            ptx::fma2f(facc[c0 + c + k], facc[c0 + c + k + 1], __uint_as_float(v[c + k]),
                                     __uint_as_float(v[c + k + 1]), sw, sw);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&empty[s]);
        }
        if constexpr (!PARTIALS) {
            if (r < nsub * 16) {
                const int n = tile * 128 + r;
#pragma unroll 4
                for (int c = 0; c < NC; ++c) {
                    const int m = tt * PT + h * NC + c;
                    if (m >= a.M) break;
                    const bool is16 = token_bits(a, m) == 16;
                    if (is16 != (MODE == PMODE_BF16)) continue;
                    const size_t o = (size_t)m * L.N + n;
                    if (a.y_dtype == 0)
                        reinterpret_cast<float*>(a.y)[o] = facc[c];
                    else
                        reinterpret_cast<__nv_bfloat16*>(a.y)[o] = __float2bfloat16_rn(facc[c]);
                }
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 1) {
        tc::fence_after();
        tc::dealloc(tmem, 512);
    }
}

// -------------------------------------------- prefill activation quantizer
// One warp per (token tile tt, operand row 0..PTE-1, group g).  Rows < 144 are
// tokens: integer rows get Eq. (2) codes -- centred (Xq - z_x, s8) when the tile
// runs in INTC mode, raw u8 otherwise -- and their scales; A16 rows get a bf16
// copy for the bypass path; padding rows are zero.  Row 144 is the all-ones
// column (INTU mode), rows 145.. are zero.
__global__ void actquant_pre_kernel(WLayout L, const uint16_t* __restrict__ x, int M,
                                    const int32_t* __restrict__ row_bits, int bits, uint8_t* __restrict__ act,
                                    PreActLayout P, int64_t* err) {
    const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int NG = L.NG, G = L.G;
    const int TT = (M + PT - 1) / PT;
    if (wid >= TT * PTE * NG) return;
    const int g = wid % NG;
    const int row = (wid / NG) % PTE;
    const int tt = wid / (NG * PTE);
    const size_t tg = (size_t)tt * NG + g;
    uint8_t* cg = act + P.codes_off + tg * P.codes_group;
    auto code_at = [&](int k) -> uint8_t* {
        const int ks = k >> 5, kb = k & 31;
        return cg + ks * (PTE * 32) + (row >> 3) * 256 + (kb >> 4) * 128 + (row & 7) * 16 + (kb & 15);
    };
    // tile mode (identical rule in the GEMM kernel): centred iff W4 and no A8 token
    int fl = 0;
    for (int i = lane; i < PT; i += 32) {
        const int mm = tt * PT + i;
        if (mm < M) fl |= tile_flags_from_bits(row_bits ? row_bits[mm] : bits);
    }
    fl = __reduce_or_sync(0xffffffffu, fl);
    const bool centred = (L.wbits == 4) && !(fl & 4);
    if (row >= PT) {  // ones column (uncentred tiles) / padding
        const uint8_t val = (row == PT && !centred) ? 1 : 0;
        for (int k = lane; k < G; k += 32) *code_at(k) = val;
        return;
    }
    const int m = tt * PT + row;
    const int b = m < M ? (row_bits ? row_bits[m] : bits) : 0;
    uint8_t* xg = act + P.x16_off + tg * P.x16_group;
    auto x16_at = [&](int k) -> uint16_t* {
        const int ks = k >> 4, kk = k & 15;
        return reinterpret_cast<uint16_t*>(xg + ks * (PT * 32) + (row >> 3) * 256 + (kk >> 3) * 128 + (row & 7) * 16 +
                                           (kk & 7) * 2);
    };
    float* sxo = reinterpret_cast<float*>(act + P.par_off + tg * PAR_BYTES) + row;
    uint32_t* cxo = reinterpret_cast<uint32_t*>(act + P.par_off + tg * PAR_BYTES + PT * 4) + row;
    const uint16_t* src = x + (size_t)m * L.K + (size_t)g * G;
    constexpr int MAXV = 4;
    float v[MAXV];
    uint16_t raw[MAXV];
    float vmin = 0.f, vmax = 0.f;
    int bad = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
        const int k = lane + 32 * i;
        raw[i] = 0;
        v[i] = 0.f;
        if (k < G && b != 0) {
            raw[i] = src[k];
            v[i] = bf16_bits_to_float(raw[i]);
            if (!finite_f(v[i])) bad = min(bad, k);
            vmin = fminf(vmin, v[i]);
            vmax = fmaxf(vmax, v[i]);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) bad = min(bad, __shfl_xor_sync(0xffffffffu, bad, o));
    if (bad != 0x7fffffff && lane == 0) report_nonfinite(err, (int64_t)m * L.K + (int64_t)g * G + bad);
    if (b != 2 && b != 4 && b != 8) {
#pragma unroll
        for (int i = 0; i < MAXV; ++i) {
            const int k = lane + 32 * i;
            if (k < G) {
                *code_at(k) = 0;
                *x16_at(k) = (b == 16) ? raw[i] : (uint16_t)0;
            }
        }
        if (lane == 0) {
            *sxo = 0.f;
            *cxo = 0u;
        }
        return;
    }
    vmin = warp_min(vmin);
    vmax = warp_max(vmax);
    float s;
    int z;
    fit_params(vmin, vmax, b, &s, &z);
    int sum = 0;
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
        const int k = lane + 32 * i;
        if (k < G) {
            const int qv = quantize_one(v[i], s, z, b, L.round_mode);
            sum += qv;
            *code_at(k) = centred ? (uint8_t)(int8_t)(qv - z) : (uint8_t)qv;
            *x16_at(k) = 0;
        }
    }
    sum = warp_sum_i(sum);
    if (lane == 0) {
        *sxo = s;
        *cxo = ((uint32_t)z << 16) | (uint32_t)sum;
    }
}

// ------------------------------------------------------------------ host
PreActLayout pre_act_layout(const WLayout& L, int M) {
    PreActLayout P;
    const int TT = (M + PT - 1) / PT;
    P.codes_group = (size_t)(L.G / 32) * PTE * 32;
    P.x16_group = (size_t)(L.G / 16) * PT * 32;
    P.codes_off = 0;
    P.x16_off = ((size_t)TT * L.NG * P.codes_group + 255) & ~(size_t)255;
    P.par_off = P.x16_off + (((size_t)TT * L.NG * P.x16_group + 255) & ~(size_t)255);
    P.bytes = P.par_off + (((size_t)TT * L.NG * PAR_BYTES + 255) & ~(size_t)255);
    return P;
}

dyq_status_t launch_actquant_pre(const WLayout& L, const uint16_t* x, int M, const int32_t* row_bits, int bits,
                                 void* act, int64_t* err, cudaStream_t st) {
    const PreActLayout P = pre_act_layout(L, M);
    const int TT = (M + PT - 1) / PT;
    const long long warps = (long long)TT * PTE * L.NG;
    actquant_pre_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(
        L, x, M, row_bits, bits, reinterpret_cast<uint8_t*>(act), P, err);
    return check_launch("actquant_pre_kernel");
}

template <int WBITS, int SPG, int MODE, bool PARTIALS>
static cudaError_t pre_launch(const PreArgs& a0, dim3 grid, cudaStream_t st) {
    PreArgs a = a0;
    constexpr int G = SPG * 64;
    constexpr bool INT = MODE != PMODE_BF16;
    const int raw = SPG * 8 * 512 * (WBITS / 4);
    const int bbytes = INT ? (G / 32) * PTE * 32 : (G / 16) * PT * 32;
    const int abytes = INT ? (G / 32) * 4096 : (G / 16) * 4096;
    a.off_meta = raw;
    a.off_b = (a.off_meta + META_BLOCK + 127) & ~127;
    a.off_par = a.off_b + bbytes;
    a.off_a = (a.off_par + PAR_BYTES + 127) & ~127;
    a.stage_bytes = (a.off_a + abytes + 127) & ~127;
    a.stages = (200 * 1024) / a.stage_bytes;
    if (a.stages > 8) a.stages = 8;
    if (a.stages < 2) a.stages = 2;
    const size_t smem = 1024 + (size_t)a.stages * a.stage_bytes;
    auto kern = qlinear_prefill_kernel<WBITS, SPG, MODE, PARTIALS>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr = true;
    }
    kern<<<grid, PRE_THREADS, smem, st>>>(a);
    return cudaGetLastError();
}

template <int MODE, bool PARTIALS>
static cudaError_t pre_dispatch(const PreArgs& a, dim3 grid, cudaStream_t st) {
    if (a.L.wbits == 4)
        return a.L.G == 64 ? pre_launch<4, 1, MODE, PARTIALS>(a, grid, st) : pre_launch<4, 2, MODE, PARTIALS>(a, grid, st);
    if (MODE == PMODE_INTC) return cudaSuccess;  // W8 codes never fit the centred s8 operand
    return a.L.G == 64 ? pre_launch<8, 1, MODE, PARTIALS>(a, grid, st) : pre_launch<8, 2, MODE, PARTIALS>(a, grid, st);
}

dyq_status_t launch_prefill(const WLayout& L, const void* codes, const void* meta, int M, const int32_t* row_bits,
                            int bits, void* y, int y_dtype, int32_t* I_out, const void* act, cudaStream_t st) {
    PreArgs a;
    a.L = L;
    a.codes = reinterpret_cast<const uint8_t*>(codes);
    a.meta = reinterpret_cast<const uint8_t*>(meta);
    a.row_bits = row_bits;
    a.bits = bits;
    a.M = M;
    a.y = y;
    a.y_dtype = y_dtype;
    a.I_out = I_out;
    a.act = reinterpret_cast<const uint8_t*>(act);
    a.P = pre_act_layout(L, M);
    const dim3 grid(L.T128, (M + PT - 1) / PT);
    // three kernel variants; each CTA runs only if its token tile needs it
    cudaError_t e;
    if (I_out) {
        e = pre_dispatch<PMODE_INTC, true>(a, grid, st);
        if (e == cudaSuccess) e = pre_dispatch<PMODE_INTU, true>(a, grid, st);
    } else {
        e = pre_dispatch<PMODE_INTC, false>(a, grid, st);
        if (e == cudaSuccess) e = pre_dispatch<PMODE_INTU, false>(a, grid, st);
        if (e == cudaSuccess) e = pre_dispatch<PMODE_BF16, false>(a, grid, st);
    }
    if (e != cudaSuccess) return set_error(DYQ_ECUDA, "qlinear_prefill_kernel launch: %s", cudaGetErrorString(e));
    return DYQ_OK;
}

}  // namespace dyq
