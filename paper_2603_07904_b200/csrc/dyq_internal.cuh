// dyq_internal.cuh -- layouts, launch-plan structs and small device helpers
// shared by the libdyq.so translation units.  Product code: never includes
// anything under oracle/.
#pragma once
#include <cuda_fp8.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/dyq.h"

namespace dyq {

// ------------------------------------------------------------------ layout
// Packed weights (DESIGN.md §"Data layout in HBM").
//   rows are grouped in 128-row tiles; a tile holds up to 8 sub-tiles of 16
//   rows (the last tile may be ragged: N % 16 == 0 is required);
//   K is walked in "slab pairs" of 64 input channels (two 32-wide MMA k-steps).
//   One chunk = (tile, slab pair, sub-tile) = 16 rows x 64 k:
//     W4: 512 B = 32 lanes x 16 B, lane L = 4*gid + t (gid = row % 8, t = 0..3)
//         holds [slab0 word(row gid)][slab0 word(row gid+8)]
//               [slab1 word(row gid)][slab1 word(row gid+8)],
//         word byte b: lo nibble = q[k = 32*slab + 4t + b],
//                      hi nibble = q[k = 32*slab + 16 + 4t + b].
//     W8: 1024 B = [slab (2)][lane (32)][16 B = R0 R1 R2 R3], the u8 A-fragment
//         registers of mma.m16n8k32: R0 = q[gid][4t..4t+3], R1 = q[gid+8][4t..],
//         R2 = q[gid][16+4t..], R3 = q[gid+8][16+4t..] (k relative to the slab).
//   Chunks are ordered (tile, slab pair, sub-tile) so that one (tile, slab pair)
//   is 8 contiguous chunks (4 KB for W4) -- one bulk copy for the prefill kernel.
// Metadata: one 640-byte block per (tile, group) -- 128 fp32 scales then 128
//   u8 zero-points -- so a decode unit's metadata is one bulk copy.  Inside a
//   block, row r of sub-tile `sub` sits at slot sub * 16 + p, p = 2 * (r % 8) +
//   r / 8: the decode lane of group gid reads the (row gid, row gid+8) pair with
//   one 8-byte (scales) / 2-byte (zeros) load.

struct WLayout {
    int N, K, G, wbits, round_mode;
    int NG;       // K / G
    int NSP;      // K / 64 slab pairs
    int T128;     // ceil(N / 128)
    int nsub_last;
    int chunk;    // bytes per (tile, sp, sub) chunk
    size_t codes_bytes, meta_bytes;
};

__host__ __device__ inline size_t chunk_offset(const WLayout& L, int tile, int sp, int sub) {
    const int nsub = (tile == L.T128 - 1) ? L.nsub_last : 8;
    return ((size_t)tile * L.NSP * 8 + (size_t)sp * nsub + sub) * (size_t)L.chunk;
}
constexpr int META_BLOCK = 640;  // bytes of metadata per (tile, group)
__host__ __device__ inline size_t meta_block(const WLayout& L, int tile, int g) {
    return ((size_t)tile * L.NG + g) * META_BLOCK;
}
__host__ __device__ inline int meta_slot(int sub, int r) { return sub * 16 + 2 * (r & 7) + (r >> 3); }

// Activations for the decode kernel (M <= 16 tokens per call, nt8 = M <= 8 ? 1 : 2
// halves of 8 tokens).  Per K-group g one contiguous record of cp_stride bytes
//   codes [nt8 halves][8 tok][G] u8 Eq. (2) codes (or centred s8, see below)
//   par   [8 * nt8 tok] {float s_x; uint32 (z_x << 16) | SX  or  SXc}
// so a run of consecutive K-groups is ONE bulk copy per pipeline stage; then
//   x16 [NG][nt8 * 8 tok][G] bf16 copy of x for A16 (BF16-bypass) rows, else 0
//   zx  [NG][16] u8 z_x (test hook only).
// Inside each 64-k block the k order is permuted so that decode lane t reads
// all of its B-fragment words with 16-byte loads:
//   position t*16 + s*8 + h*4 + b  <->  k = 32*s + 16*h + 4*t + b
// (u8 codes: one 16-B load; bf16: two 16-B loads), and the lane owning C-tokens
// (2t, 2t+1) reads both tokens' parameters with one 16-B load.
constexpr int DEC_MPAD = 16;
__host__ __device__ inline int dec_nt8(int M) { return M <= 8 ? 1 : 2; }
__host__ __device__ inline int dec_perm(int kk) {  // kk in [0,64) -> position
    const int s = kk >> 5, h = (kk >> 4) & 1, t = (kk >> 2) & 3, b = kk & 3;
    return t * 16 + s * 8 + h * 4 + b;
}

// Fused tensor-parallel epilogue: the decode kernel
// stores its column shard straight into every rank's full output y[p]
// ([M, ldy] bf16, column offset col0) -- peer memory over NVLink, mapped with
// CUDA IPC -- then release-increments every rank's flag once per 16-column
// sub-tile.  n = 0: ordinary single-output epilogue.
constexpr int TP_MAX = 8;
constexpr int PRE_PT = 144;  // prefill token tile (dyq_prefill.cu PT): flag increments per call
struct TpPeers {
    void* y[TP_MAX];
    unsigned long long* flag[TP_MAX];
    int n, ldy, col0;
};

struct ActLayoutDec {
    size_t cp_off, x16_off, zx_off, bytes;
    int nt8, cp_stride, x16_stride;
};
__host__ __device__ inline ActLayoutDec act_layout_dec(const WLayout& L, int nt8) {
    ActLayoutDec A;
    A.nt8 = nt8;
    A.cp_stride = nt8 * 8 * L.G + nt8 * 8 * 8;
    A.x16_stride = nt8 * 8 * L.G * 2;
    A.cp_off = 0;
    A.x16_off = ((size_t)L.NG * A.cp_stride + 255) & ~(size_t)255;
    A.zx_off = A.x16_off + (((size_t)L.NG * A.x16_stride + 255) & ~(size_t)255);
    A.bytes = A.zx_off + (((size_t)L.NG * DEC_MPAD + 255) & ~(size_t)255);
    return A;
}
// Decode activation format of a call: CENTRED when every token of the call runs
// at 2 or 4 bits -- codes stored as s8 (Xq - z_x) and par = {s_x, SXc = Sum (Xq - z_x)},
// so the kernel needs one u8 x s8 IMMA and I = P' - z_w * SXc; otherwise RAW u8
// codes with par = {s_x, z_x << 16 | SX}.
__device__ __forceinline__ bool dec_call_centred(int M, int m0, const int32_t* row_bits, int bits) {
    bool c = true;
    for (int m = 0; m < M; ++m) {
        const int b = row_bits ? row_bits[m0 + m] : bits;
        c &= (b == 2 || b == 4);
    }
    return c;
}

// Prefill activation operand (M > 16): per (144-token tile, K-group) one
// record [s_x | B] (one bulk copy per group) holding the UMMA canonical
// K-major no-swizzle B operand of the tcgen05 kernel,
//   x16 [TT][NG][G/16 K-steps][144 rows] bf16: centred codes Xq - z_x (exact),
//       x for A16 rows, 0 for absent rows
//   par [TT][NG][144] f32 s_x (1 for A16 rows, 0 for absent rows)
//   mode [TT] u8: 1 = the tile's operands are e4m3 (dyq_pre_tile_e4m3)
// (codes_off / codes_group are unused, kept 0).
constexpr size_t PRE_CNT_BYTES = 1024;  // prefill stream-K counters, just before the prefill area
struct PreActLayout {
    size_t codes_off, x16_off, par_off, mode_off, bytes;
    size_t codes_group, x16_group, rec;
};

// ---------------------------------------------------------------- tracing
// Optional %globaltimer event trace (dyq_trace_enable; debugging / profiling
// only): buffer = [count][capacity][records of 2 x u64 {tag, ns}],
// tag = serial << 32 | kernel << 24 | event << 16 | blockIdx.x.
extern uint64_t* g_trace;   // host-side copy of the enabled buffer (or null)
extern uint32_t g_trace_serial;
__device__ __forceinline__ void trace_ev(uint64_t* tr, uint32_t serial, uint32_t kernel, uint32_t ev) {
    if (!tr) return;
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned long long i = atomicAdd(reinterpret_cast<unsigned long long*>(tr), 1ull);
    if (i < tr[1]) {
        tr[2 + 2 * i] = ((uint64_t)serial << 32) | (kernel << 24) | (ev << 16) | (blockIdx.x & 0xffffu);
        tr[3 + 2 * i] = t;
    }
}

// ------------------------------------------------------------ error words
__device__ inline void report_nonfinite(int64_t* err, int64_t idx) {
    if (err) atomicMin(reinterpret_cast<unsigned long long*>(err), (unsigned long long)idx);
}

__device__ inline float bf16_bits_to_float(uint16_t h) {
    return __uint_as_float(((uint32_t)h) << 16);
}

// ------------------------------------------------- exact quantizer pieces
// Fit of DESIGN.md readings 2-4 (restated from PAPER.md Eq. 2, P:100-106 and
// SPEC S:43-51): lo = min(0, min v), hi = max(0, max v) (exact), R = max(hi-lo,
// 1e-8) in fp64, s64 = R / (2^b-1), stored s = fp32(s64), z = clamp(half-up(-lo/s64)).
// Explicit _rn intrinsics: no contraction, IEEE rounding.
__device__ inline void fit_params(float vmin, float vmax, int bits, float* s_out, int* z_out) {
    double lo = vmin < 0.f ? (double)vmin : 0.0;
    double hi = vmax > 0.f ? (double)vmax : 0.0;
    const double levels = (double)((1 << bits) - 1);
    double R = __dadd_rn(hi, -lo);
    if (R < 1e-8) R = 1e-8;
    const double s64 = __ddiv_rn(R, levels);
    const double zr = __ddiv_rn(-lo, s64);
    const double fl = floor(zr);
    double zq = fl + ((__dadd_rn(zr, -fl) >= 0.5) ? 1.0 : 0.0);
    if (zq < 0.0) zq = 0.0;
    if (zq > levels) zq = levels;
    *s_out = __double2float_rn(s64);
    *z_out = (int)zq;
}

// Exact floor(v / s) of the real quotient of two fp32 values (s > 0), in fp32:
// an estimate from the correctly rounded reciprocal is off by at most one for
// |v / s| < 2^20; the sign of each FMA remainder v - q s is exact (the FMA
// rounds the exact value once, and a non-zero difference of these operands is
// >= 2^-149, never flushed: no -ftz), so two checks make the floor exact.
// Equal to the oracle's floor(fp64(v) / fp64(s)) (reading 4).
__device__ __forceinline__ float floor_div_exact(float v, float s) {
    float q = floorf(__fmul_rn(v, __frcp_rn(s)));
    if (fmaf(-q, s, v) < 0.f) {
        q -= 1.f;
    } else if (fmaf(-(q + 1.f), s, v) >= 0.f) {
        q += 1.f;
    }
    return q;
}

// Eq. (2): q = clamp(floor(v / s) + z, 0, 2^b - 1) with the exact floor;
// round_mode 1: floor(v / s + 1/2), decided exactly from the sign of 2v - (2t+1)s.
__device__ inline int quantize_one(float v, float s, int z, int bits, int round_mode) {
    float f = floor_div_exact(v, s);
    if (round_mode == 1 && fmaf(-(2.f * f + 1.f), s, 2.f * v) >= 0.f) f += 1.f;
    float c = f + (float)z;
    const float levels = (float)((1 << bits) - 1);
    c = c < 0.f ? 0.f : (c > levels ? levels : c);
    return (int)c;
}

__device__ inline bool finite_f(float v) { return isfinite(v); }

// SwiGLU activation of one element, bf16(silu(g) * u) with fp32 math -- the
// exact float ops of silu_mul_kernel (dyq_model.cu), so the fused and the
// separate path give identical bits.
__device__ __forceinline__ uint16_t silu_mul_bf16(uint16_t gb, uint16_t ub) {
    const float g = bf16_bits_to_float(gb), u = bf16_bits_to_float(ub);
    return __bfloat16_as_ushort(__float2bfloat16_rn(g / (1.f + __expf(-g)) * u));
}

// -------------------------------------------------------------- warp ops
// Warp reductions with one REDUX instruction each (sm_80+).  Floats go through
// an order-preserving int map (exact: min / max return an input value; the
// callers' values are finite or already reported as non-finite).
__device__ __forceinline__ int f2ord(float f) {
    const int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float ord2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }
__device__ inline float warp_min(float v) { return ord2f(__reduce_min_sync(0xffffffffu, f2ord(v))); }
__device__ inline float warp_max(float v) { return ord2f(__reduce_max_sync(0xffffffffu, f2ord(v))); }
__device__ inline int warp_sum_i(int v) { return __reduce_add_sync(0xffffffffu, v); }
__device__ inline int warp_min_i(int v) { return __reduce_min_sync(0xffffffffu, v); }

// One decode-quantizer job (a whole warp): token row m (of rows m0 ..) and
// K-group g of x at the row's bits into the decode activation layout (records
// codes at dec_perm positions + {s_x, z_x << 16 | SX} or, centred, {s_x,
// SXc}; bf16 copies of BF16-bypass rows in x16; z_x bytes).  m >= M: padding
// row (zeros).  Used by actquant_dec_kernel and by the decode attention
// kernel's epilogue (the o projection's input, dyq_model.cu).
__device__ inline void aq_dec_job(const WLayout& L, const uint16_t* __restrict__ x, int M, int m0,
                                  const int32_t* __restrict__ row_bits, int bits, uint8_t* __restrict__ ws,
                                  const ActLayoutDec& A, int64_t* err, int gated, int g, int m, bool centred) {
    const int lane = threadIdx.x & 31;
    const int MP = 8 * A.nt8;
    uint8_t* rec = ws + A.cp_off + (size_t)g * A.cp_stride;
    uint8_t* dq = rec + (size_t)m * L.G;
    uint16_t* d16 = reinterpret_cast<uint16_t*>(ws + A.x16_off + (size_t)g * A.x16_stride) + (size_t)m * L.G;
    uint2* pdst = reinterpret_cast<uint2*>(rec + MP * L.G) + m;
    uint8_t* zdst = ws + A.zx_off + (size_t)g * DEC_MPAD + m;
    const int b = (m < M) ? (row_bits ? row_bits[m0 + m] : bits) : 0;
    // gated: x = [g | u] rows of width 2K (SwiGLU input); the activation is
    // bf16(silu(g) * u), the same float ops as silu_mul_kernel (dyq_model.cu)
    const uint16_t* src = x + (size_t)(m0 + m) * L.K * (gated ? 2 : 1) + (size_t)g * L.G;
    constexpr int MAXV = 4;  // G <= 128
    float v[MAXV];
    uint16_t raw[MAXV];
    float vmin = 0.f, vmax = 0.f;
    int bad = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < MAXV; ++i) {
        const int k = lane + 32 * i;
        v[i] = 0.f;
        raw[i] = 0;
        if (k < L.G && b != 0) {
            raw[i] = gated ? silu_mul_bf16(src[k], src[k + L.K]) : src[k];
            v[i] = bf16_bits_to_float(raw[i]);
            if (!finite_f(v[i])) bad = min(bad, k);
            vmin = fminf(vmin, v[i]);
            vmax = fmaxf(vmax, v[i]);
        }
    }
    bad = warp_min_i(bad);
    if (bad != 0x7fffffff && lane == 0)
        report_nonfinite(err, (int64_t)(m0 + m) * L.K + (int64_t)g * L.G + bad);
    if (b != 2 && b != 4 && b != 8) {  // padding row or BF16 bypass row
#pragma unroll
        for (int i = 0; i < MAXV; ++i) {
            const int k = lane + 32 * i;
            if (k < L.G) {
                const int pos = (k & ~63) + dec_perm(k & 63);
                dq[pos] = 0;
                d16[pos] = (b == 16) ? raw[i] : (uint16_t)0;
            }
        }
        if (lane == 0) {
            *pdst = make_uint2(0u, 0u);
            *zdst = 0;
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
        if (k < L.G) {
            const int q = quantize_one(v[i], s, z, b, L.round_mode);
            sum += q;
            const int pos = (k & ~63) + dec_perm(k & 63);
            dq[pos] = centred ? (uint8_t)(int8_t)(q - z) : (uint8_t)q;
            d16[pos] = 0;
        }
    }
    sum = warp_sum_i(sum);
    if (lane == 0) {
        *pdst = make_uint2(__float_as_uint(s), centred ? (uint32_t)(sum - L.G * z) : ((uint32_t)z << 16) | (uint32_t)sum);
        *zdst = (uint8_t)z;
    }
}


// ------------------------------------------- prefill activation quantizer job
constexpr int PRE_PAR_BYTES = PRE_PT * 4;  // record head: float s_x[144]
constexpr int AQP_TPR = 4;                 // threads per token row
// Physical byte position, inside one 32-k e4m3 K step, of logical k (0..31):
// the packed W4 fragment puts k = 4t + i (low nibbles) in TMEM column 2t and
// k = 16 + 4t + i (high nibbles) in column 2t + 1, so B follows that order.
__host__ __device__ inline int e4m3_kpos(int kl) { return 8 * ((kl >> 2) & 3) + 4 * ((kl >> 4) & 1) + (kl & 3); }
__device__ __forceinline__ uint8_t e4m3_of(float v) {  // exact for integers |v| <= 15
    return (uint8_t)__nv_cvt_float_to_fp8(v, __NV_SATFINITE, __NV_E4M3);
}
// One job of the prefill quantizer: quarter `half` (G/4 = KH inputs) of token
// row `row` of record (token tile tt, K-group g) -- the AQP_TPR jobs of a row
// are adjacent lanes of one warp (quad shuffles), every lane of the warp runs
// a job.  Used by actquant_pre_kernel (one CTA per record, dyq_prefill.cu) and
// by the policy step's add + RMSNorm epilogue (dyq_model.cu).
template <int KH>
__device__ __forceinline__ void aqp_job(const WLayout& L, const uint16_t* __restrict__ x, int M,
                                        const int32_t* __restrict__ row_bits, int bits, uint8_t* __restrict__ act,
                                        const PreActLayout& P, int64_t* err, bool f8, int gated, int tt, int g,
                                        int row, int half) {
    constexpr int PT = PRE_PT;
    constexpr int PAR_BYTES = PRE_PAR_BYTES;
    const int NG = L.NG, G = L.G;
    const int m = tt * PT + row;
    const int b = m < M ? (row_bits ? row_bits[m] : bits) : 0;
    const size_t tg = (size_t)tt * NG + g;
    uint8_t* xg = act + tg * P.rec + PAR_BYTES;  // record [s_x | B]
    const int k0 = half * KH;  // inputs k0 .. k0 + KH - 1
    const uint16_t* src = x + (size_t)(m < M ? m : 0) * L.K * (gated ? 2 : 1) + (size_t)g * G + k0;  // gated: [g | u]
    constexpr int NW = KH / 2;  // 32-bit words per thread
    uint32_t raw[NW];
    float vmin = 0.f, vmax = 0.f;
    int bad = 0x7fffffff;
    if (b != 0) {
#pragma unroll
        for (int i = 0; i < NW; i += 4) {
            uint4 w4 = *reinterpret_cast<const uint4*>(src + 2 * i);
            if (gated) {
                const uint4 u4 = *reinterpret_cast<const uint4*>(src + L.K + 2 * i);
                const uint32_t gw[4] = {w4.x, w4.y, w4.z, w4.w}, uw[4] = {u4.x, u4.y, u4.z, u4.w};
                uint32_t o[4];
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    o[e] = (uint32_t)silu_mul_bf16(gw[e] & 0xffffu, uw[e] & 0xffffu) |
                           ((uint32_t)silu_mul_bf16(gw[e] >> 16, uw[e] >> 16) << 16);
                w4 = make_uint4(o[0], o[1], o[2], o[3]);
            }
            raw[i] = w4.x;
            raw[i + 1] = w4.y;
            raw[i + 2] = w4.z;
            raw[i + 3] = w4.w;
        }
#pragma unroll
        for (int i = 0; i < NW; ++i)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const float v = bf16_bits_to_float((uint16_t)(raw[i] >> (16 * hh)));
                if (!finite_f(v)) bad = min(bad, k0 + 2 * i + hh);
                vmin = fminf(vmin, v);
                vmax = fmaxf(vmax, v);
            }
    }
    // quad combine (the row's four threads are adjacent lanes)
    vmin = fminf(vmin, __shfl_xor_sync(0xffffffffu, vmin, 1));
    vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, 1));
    bad = min(bad, __shfl_xor_sync(0xffffffffu, bad, 1));
    vmin = fminf(vmin, __shfl_xor_sync(0xffffffffu, vmin, 2));
    vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, 2));
    bad = min(bad, __shfl_xor_sync(0xffffffffu, bad, 2));
    if (bad != 0x7fffffff && half == 0) report_nonfinite(err, (int64_t)m * L.K + (int64_t)g * G + bad);
    float* sxo = reinterpret_cast<float*>(act + tg * P.rec) + row;
    const bool quant = b == 2 || b == 4 || b == 8;
    float s = 1.f;
    int z = 0;
    if (quant) fit_params(vmin, vmax, b, &s, &z);
    if (half == 0) *sxo = quant ? s : (b == 16 ? 1.f : 0.f);
    // codes of this thread's inputs (as exact centred integers), then the
    // layout-ordered 16-B stores
    auto val = [&](int i, int hh) -> float {  // input k0 + 2i + hh
        const uint16_t r = (uint16_t)(raw[i] >> (16 * hh));
        if (quant) return (float)(quantize_one(bf16_bits_to_float(r), s, z, b, L.round_mode) - z);
        return 0.f;
    };
    uint8_t* rowb = xg + (row >> 3) * 256 + (row & 7) * 16;
    if (!f8) {
        // bf16: this thread covers K steps ks = k0/16 .. (k0 + KH)/16 - 1
#pragma unroll
        for (int ks = 0; ks < KH / 16; ++ks) {
#pragma unroll
            for (int kh = 0; kh < 2; ++kh) {  // kk >> 3
                uint32_t o[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int i = ks * 8 + kh * 4 + e;  // word index: k = k0 + 2i, 2i + 1
                    if (b == 16) {
                        o[e] = raw[i];
                    } else if (quant) {
                        const __nv_bfloat162 p2 = __floats2bfloat162_rn(val(i, 0), val(i, 1));  // |q - z| <= 255: exact
                        o[e] = *reinterpret_cast<const uint32_t*>(&p2);
                    } else {
                        o[e] = 0;
                    }
                }
                const int KS = (k0 >> 4) + ks;
                *reinterpret_cast<uint4*>(rowb + KS * (PT * 32) + kh * 128) = make_uint4(o[0], o[1], o[2], o[3]);
            }
        }
    } else if constexpr (KH == 16) {
        // e4m3, G = 64: a 32-k K step spans thread pair (A: k 0-15, B: 16-31);
        // chunk 0 = [A0 B0 A1 B1], chunk 1 = [A2 B2 A3 B3] (4-byte runs of k)
        uint32_t w[4];
#pragma unroll
        for (int r4 = 0; r4 < 4; ++r4) {
            w[r4] = 0u;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int kt = 4 * r4 + e;
                const uint32_t q8 = quant ? (uint32_t)e4m3_of(val(kt >> 1, kt & 1)) : 0u;  // |q - z| <= 15
                w[r4] |= q8 << (8 * e);
            }
        }
        const bool isA = (half & 1) == 0;
        const uint32_t x0 = __shfl_xor_sync(0xffffffffu, isA ? w[2] : w[0], 1);
        const uint32_t x1 = __shfl_xor_sync(0xffffffffu, isA ? w[3] : w[1], 1);
        const int KS = half >> 1;
        const uint4 o = isA ? make_uint4(w[0], x0, w[1], x1) : make_uint4(x0, w[2], x1, w[3]);
        *reinterpret_cast<uint4*>(rowb + KS * (PT * 32) + (isA ? 0 : 128)) = o;
    } else {
        // e4m3: one 32-k K step per thread (G = 128)
#pragma unroll
        for (int ks = 0; ks < KH / 32; ++ks) {
#pragma unroll
            for (int c = 0; c < 2; ++c) {  // p >> 4
                uint32_t o[4] = {0, 0, 0, 0};
#pragma unroll
                for (int pp = 0; pp < 16; ++pp) {
                    const int p = 16 * c + pp;
                    const int kl = (((p >> 2) & 1) << 4) | (((p >> 3) & 3) << 2) | (p & 3);  // e4m3_kpos^-1
                    const int kt = ks * 32 + kl;  // input index within this thread
                    const uint32_t q8 = quant ? (uint32_t)e4m3_of(val(kt >> 1, kt & 1)) : 0u;  // |q - z| <= 15
                    o[pp >> 2] |= q8 << (8 * (pp & 3));
                }
                const int KS = (k0 >> 5) + ks;
                *reinterpret_cast<uint4*>(rowb + KS * (PT * 32) + c * 128) = make_uint4(o[0], o[1], o[2], o[3]);
            }
        }
    }
}


size_t decode_ws_bytes(const WLayout& L);
// the decode activation area (actquant_dec_kernel's output) of a qlinear workspace
uint8_t* dec_act_area(const WLayout& L, void* ws);
// the prefill activation area (actquant_pre_kernel's output) of a qlinear workspace
uint8_t* pre_act_area(const WLayout& L, void* ws);
// DYQ_PRE_E4M3: the prefill quantizer picks e4m3 operand tiles (dyq_prefill.cu)
bool prefill_e4m3(const WLayout& L);
dyq_status_t launch_prefetch_l2(const void* p, size_t bytes, cudaStream_t st);
PreActLayout pre_act_layout(const WLayout& L, int M);
// prefill stream-K: the largest number of CTAs sharing one output tile (1 =
// none split) and the fp32 partial-tile bytes the workspace reserves after the
// prefill activation area
int prefill_ksplit(const WLayout& L, int M);
size_t prefill_part_bytes(const WLayout& L, int M);
dyq_status_t launch_actquant_pre(const WLayout& L, const uint16_t* x, int M, const int32_t* row_bits, int bits,
                                 void* act, int64_t* err, cudaStream_t st, int gated = 0);
dyq_status_t launch_prefill(const WLayout& L, const void* codes, const void* meta, int M, const int32_t* row_bits,
                            int bits, void* y, int y_dtype, int32_t* I_out, const void* act, cudaStream_t st, const TpPeers* tp = nullptr);
extern int g_path;
// Device gate of the current masked qlinear call (dyq_qlinear_masked): when
// non-null every kernel of the call waits for its predecessors, reads *gate and
// returns at once if it is 0 (no row of this call is live), before any copy.
extern thread_local const int32_t* g_gate;
__device__ __forceinline__ bool gate_closed(const int32_t* gate) {
    if (!gate) return false;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    return *reinterpret_cast<const volatile int32_t*>(gate) == 0;
}
// dyq_select.cu
size_t sel_state_bytes(int32_t E, const dyq_calib_t& c);
dyq_status_t launch_sel_init(int32_t E, const dyq_calib_t& c, void* state, cudaStream_t st);
dyq_status_t launch_sel_reset(void* state, int32_t E, const uint8_t* mask, cudaStream_t st);
dyq_status_t launch_select(void* state, int32_t E, const dyq_calib_t* cal_or_null, const float* prev_action,
                           int32_t* bits, double* S_out, int32_t* target_out, int32_t tpe, const int32_t* tab4,
                           int32_t* row_bits, cudaStream_t st);
dyq_status_t launch_route(const int32_t* bits, int32_t E, int32_t tpe, const int32_t* tab4, int32_t* row_bits,
                          cudaStream_t st);
}  // namespace dyq

// host-side helpers (dyq_host.cu)
namespace dyq {
bool pdl_enabled();  // DYQ_NO_PDL=1 disables programmatic dependent launch (A/B timing)
dyq_status_t set_error(dyq_status_t st, const char* fmt, ...);
dyq_status_t check_launch(const char* what);
bool make_layout(const dyq_wdesc_t* wd, WLayout* L);

// kernel launchers (one per TU)
dyq_status_t launch_pack(const WLayout& L, const uint16_t* w, void* codes, void* meta,
                         int64_t* err, cudaStream_t st);
dyq_status_t launch_unpack(const WLayout& L, const void* codes, const void* meta, uint8_t* q,
                           float* s, uint8_t* z, cudaStream_t st);
dyq_status_t launch_actquant_dec(const WLayout& L, const uint16_t* x, int M, int m0, const int32_t* row_bits,
                                 int bits, void* ws, int64_t* err, cudaStream_t st, int gated = 0);
// dyq_qlinear on the SwiGLU of gu = [g | u] (rows of 2K): the activation
// quantizers form bf16(silu(g) * u) on the fly (policy step, not exported).
dyq_status_t qlinear_gated(const dyq_wdesc_t* wd, const void* codes, const void* meta, const uint16_t* gu, int32_t M,
                           const int32_t* row_bits, int32_t bits, void* y, int32_t y_dtype, void* ws, size_t ws_bytes,
                           int64_t* err, cudaStream_t st);
dyq_status_t launch_actquant_export(const WLayout& L, int M, const int32_t* row_bits, int bits, const void* ws,
                                    uint8_t* xq, float* sx, uint8_t* zx, int32_t* SX, int m0, cudaStream_t st);
// rows m0 .. m0+M-1 (M <= DEC_MPAD); x, row_bits, y, I_out are base pointers;
// ws = zero-initialised split-K accumulator area (decode_ws_bytes)
dyq_status_t launch_decode(const WLayout& L, const void* codes, const void* meta, const uint16_t* x, int M,
                           int m0, const int32_t* row_bits, int bits, void* y, int y_dtype, int32_t* I_out,
                           void* ws, int64_t* err, cudaStream_t st, const TpPeers* tp = nullptr);
}  // namespace dyq
