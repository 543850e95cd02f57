// dyq_prefill.cu -- the prefill-regime quantized linear layer (M > 16 tokens):
// a warp-specialised tcgen05 GEMM with TMEM accumulators (sm_100a).
//
// "the packed activations ... utilize native INT4 and INT8
// Tensor Cores"; "the computationally intensive visual prefill".
//
// Exact integer group sums on the bf16 tensor pipe.  Both operands are fed
// CENTRED, as integers held in bf16:
//     A[n][k] = q_w[n,k] - z_w[n,g]        |A| <= 255 (W8), <= 15 (W4)
//     B[m][k] = Xq[m,k]  - z_x[m,g]        |B| <= 255 (A8), <= 15 (A4), <= 3 (A2)
// Every integer of magnitude <= 256 is exact in bf16, every product is exact in
// fp32 (16 significant bits), and a group sum is bounded by G * 255^2 <= 8.3e6
// < 2^24, so tcgen05.mma .kind::f16 with an fp32 accumulator returns the exact
// integer I[m,n,g] = Sum_k (Xq - z_x)(q - z_w) of Eq. (2)'s codes -- the value
// the paper's INT4/INT8 tensor cores produce -- already as a float.  (The parity
// tests check I bit-exactly, extreme A8 x W8 codes included.)  Why not
// .kind::i8: with per-group scales on BOTH operands every group sum must be
// promoted on the CUDA cores (acc += I * s_x * s_w per element and group); with
// the s32 accumulator that costs an I2F per element plus a zero-point correction
// for u8 operands, and those CUDA-core instructions -- not the tensor pipe --
// bound the kernel.  The fp32 accumulator halves the promotion, and the bf16
// pipe's rate (half of i8) stays above what the promotion can consume.
// BF16-bypass tokens (A16) use the same MMA with B = x and s_x = 1, so
// one pass serves any mix of activation widths in a token tile.
// E4M3 mode (W4 tiles whose tokens all run A2 / A4): every centred code
// (|q - z_w| <= 15, |Xq - z_x| <= 15) is exact in e4m3 and the fp32 sums are
// exact (tools/f8_probe.cu), so the same integer group sums come from
// tcgen05.mma .kind::f8f6f4 with K = 32 per instruction -- half the MMAs and
// half the B bytes of the bf16 path.  Decided per 144-token tile, identically
// in the quantizer and here (dyq_pre_tile_e4m3).
//
// CTA = one 128-row weight tile x one 144-token tile (288 = 2 x 144: the OpenVLA
// prefill of 256 vision + 32 text tokens tiles exactly), whole K, 14 warps:
//   warp 0      producer: per K-group, bulk copies (TMA engine) of the packed
//               codes, the 640-B metadata block, the B operand (already in the
//               UMMA canonical K-major layout, written by the prefill quantizer)
//               and the token scales into an smem ring;
//   warp 1      MMA issuer (one thread): G/16 tcgen05.mma per group, A from
//               TMEM, B from smem, into a double-buffered TMEM accumulator;
//   warps 2-5   transform: packed codes -> bf16 (q - z_w), written straight to
//               TMEM with tcgen05.st.16x256b (the packed lane-fragment order IS
//               the 16x256b register fragment), so the A operand never touches
//               shared memory;
//   warps 6-13  promotion: tcgen05.ld.16x256b the group's sums, acc += D s_x s_w
//               (FMUL2 + FFMA2) in registers; transposed 16-B stores at the end.
// TMEM columns: [0,144) [144,288) accumulators, then NA A-operand buffers.
#include <stdlib.h>
#include <cuda_fp8.h>
#include <type_traits>

#include "dyq_internal.cuh"
#include "dyq_ptx.cuh"


namespace dyq {

#ifndef DYQ_PRE_MAX_STAGES
// ring depth cap (smem fits 7 stages): round-2 same-box A/B at M = 288, W4A4
// G64, block: 4 stages 275.0, 5 stages 274.0, 7 stages 280.6 us (gate|up
// 107.9 / 108.0 / 109.5) -- the depth is not the bound, a shallower ring is
// slightly faster
#define DYQ_PRE_MAX_STAGES 5
#endif
constexpr int PT = 144;  // tokens per token tile (MMA N)
static_assert(PT == PRE_PT, "dyq_tp_flag_delta counts prefill token tiles");
// warps: 0 weight producer, 1 MMA issuer, 2 activation producer, 3-6
// transform, 7-14 promotion.  A warp may only touch TMEM lanes of quadrant
// (warp id % 4): the transform warps cover quadrants 3, 0, 1, 2 and each
// column half of the promotion warps covers all four.  (Registers: each SM
// sub-partition holds 16 K, so > 12 warps per CTA cap a thread at 128.)
constexpr int PRE_WARPS = 15;
constexpr int PRE_THREADS = PRE_WARPS * 32;
constexpr int PAR_BYTES = PRE_PAR_BYTES;  // per (tile, group): float s_x[144] (1 for A16 tokens, 0 for absent)
constexpr int XF_WARP0 = 3, XF_WARPS = 4;
constexpr int PR_WARP0 = 7, PR_WARPS = 8;  // promotion warps
constexpr int STG_ROW = 128 * 2 + 16;  // epilogue staging: bytes per token (128 bf16 rows + pad)
#ifndef DYQ_PRE_EXP
// timing-only experiments (tools/build_variant.py; results are wrong): bit 0
// promotion without its math, 1 transform without its work, 2 no MMAs (commit
// only), 3 promotion without TMEM loads.  0 in product builds.
#define DYQ_PRE_EXP 0
#endif
#ifndef DYQ_PRE_GTRACE
// per-group %globaltimer stamps of CTA 0 into the trace buffer (timing-only
// builds, tools/trace_prefill_groups.py): slot 16 + 512 * event + group
#define DYQ_PRE_GTRACE 0
#endif
#ifndef DYQ_PRE_MIN_GROUPS
#define DYQ_PRE_MIN_GROUPS 32  // stream-K: at least this many K-groups per CTA (16 / 32 / 64: o 41.9 / 38.9 / 51.4 us)
#endif
constexpr uint32_t ACC_COLS = 2 * PT;   // TMEM: two 144-column accumulators, then the A buffers

__device__ __forceinline__ void gstamp(uint64_t* tr, int ev, int i) {
#if DYQ_PRE_GTRACE
    if (tr && blockIdx.x == 0 && i < 512) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        tr[16 + 512 * ev + i] = t;
    }
#endif
}

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
    const uint8_t* act;  // prefill activation area (B operand, s_x, per-tile mode bytes)
    PreActLayout P;
    int stages, stage_bytes;
    int off_meta, off_b, off_par;
    int off_stage;       // epilogue staging area (bytes from the dynamic smem base)
    int TT;              // 144-token tiles
    long long W;         // work groups = T128 * TT * NG, split contiguously over gridDim.x CTAs
    TpPeers tp;          // fused TP epilogue (TP instantiation only; one whole unit per CTA)
    float* part;         // stream-K partial tiles [2 * gridDim.x][144 tokens][128 rows] fp32
    int* cnt;            // [gridDim.x] per-reducer arrival counters (zeroed once, self-resetting)
    const int32_t* gate; // dyq_qlinear_masked gate or null
    uint64_t* trace;     // dyq_trace_enable buffer or null (kernel id 4; events below)
    uint32_t serial;
};
// trace events (tools/trace_prefill.py): 0 CTA entry, 1 promotion past
// griddepcontrol.wait, 2 first accumulator ready, 3 segment's last group
// promoted, 4 segment epilogue done (reducer: after its wait), 5 CTA exit

// Physical byte position, inside one 32-k e4m3 K step, of logical k (0..31):
// the packed W4 fragment puts k = 4t + i (low nibbles) in TMEM column 2t and
// k = 16 + 4t + i (high nibbles) in column 2t + 1, so B follows that order.



// Stream-K partition: CTA c owns work groups [sk_begin(c), sk_begin(c + 1)) of
// the flat order w = ((tile * TT + tt) * NG + g) -- tile-major, so the token
// tiles of one weight tile run back to back (its codes stay in L2).
__host__ __device__ inline long long sk_begin(long long W, int P, int c) { return (W * c) / P; }

template <int WBITS, int SPG, bool PARTIALS, bool TP>
__global__ void __launch_bounds__(PRE_THREADS, 1) qlinear_prefill_kernel(const PreArgs a) {
    constexpr int G = SPG * 64;
    constexpr int KSTEPS = G / 16;         // bf16 MMA K steps per group
    constexpr uint32_t BSTEP = PT * 32;    // B bytes per K step
    constexpr int NA = SPG == 1 ? 6 : 3;   // A-operand buffers in TMEM
    constexpr uint32_t A_COLS = 8 * KSTEPS;
    const WLayout& L = a.L;
    const int NG = L.NG, TT = a.TT;
    const long long w0 = sk_begin(a.W, gridDim.x, blockIdx.x), w1 = sk_begin(a.W, gridDim.x, blockIdx.x + 1);
    const int nw = (int)(w1 - w0);
    const int S = a.stages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint8_t* mode = a.act + a.P.mode_off;  // per token tile: 1 = e4m3 operands (written by the quantizer)

    extern __shared__ __align__(1024) uint8_t smem[];
    if (gate_closed(a.gate)) return;
    if (threadIdx.x == 0) trace_ev(a.trace, a.serial, 4, 0);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;   // [2]
    uint64_t* tempty = tfull + 2;  // [2]
    uint64_t* afull = tempty + 2;  // [NA]
    uint64_t* aempty = afull + NA; // [NA]
    uint32_t* s_tmem = reinterpret_cast<uint32_t*>(aempty + NA);
    uint8_t* stage0 = smem + 1024;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            ptx::mbar_init(&full[s], 2);  // weight producer + activation producer
            ptx::mbar_init(&empty[s], 1 + XF_WARPS + PR_WARPS);  // MMA commit + transform + promotion warps
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&tfull[b], 1);
            ptx::mbar_init(&tempty[b], PR_WARPS);
        }
        for (int i = 0; i < NA; ++i) {
            ptx::mbar_init(&afull[i], XF_WARPS);
            ptx::mbar_init(&aempty[i], 1);
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
    // walk of this CTA's groups: (unit u = tile * TT + tt, group g)
    struct Walk {
        int tile, tt, g;
    };
    auto walk0 = [&]() {
        const int u = (int)(w0 / NG);
        return Walk{u / TT, u % TT, (int)(w0 - (long long)u * NG)};
    };
    auto next = [&](Walk& k) {
        if (++k.g == NG) {
            k.g = 0;
            if (++k.tt == TT) {
                k.tt = 0;
                ++k.tile;
            }
        }
    };

    if (warp == 0) {
        // ------------------------------------------------ weight producer
        // Weights never depend on the preceding kernel: the first stages are
        // issued before griddepcontrol.wait, overlapping its tail under PDL.
        if (lane == 0) {
            Walk k = walk0();
            int s = 0;
            uint32_t ph = 0;
            for (int i = 0; i < nw; ++i, next(k)) {
                if (i >= S) ptx::mbar_wait(&empty[s], ph ^ 1);
                const int nsub = (k.tile == L.T128 - 1) ? L.nsub_last : 8;
                const uint32_t cbytes = (uint32_t)(SPG * nsub * L.chunk);
                uint8_t* st = stage0 + (size_t)s * a.stage_bytes;
                ptx::mbar_arrive_expect_tx(&full[s], cbytes + META_BLOCK);
                ptx::bulk_g2s(st, a.codes + chunk_offset(L, k.tile, k.g * SPG, 0), cbytes, &full[s]);
                ptx::bulk_g2s(st + a.off_meta, a.meta + meta_block(L, k.tile, k.g), META_BLOCK, &full[s]);
                if (++s == S) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp == 2) {
        // -------------------------------------------- activation producer
        ptx::pdl_wait();  // the B operand, s_x and the mode bytes come from the quantizer
        if (lane == 0) ptx::pdl_launch_dependents();
        if (lane == 0) {
            Walk k = walk0();
            int s = 0;
            uint32_t ph = 0;
            for (int i = 0; i < nw; ++i, next(k)) {
                if (i >= S) ptx::mbar_wait(&empty[s], ph ^ 1);
                const uint32_t bbytes = mode[k.tt] ? KSTEPS * BSTEP / 2 : KSTEPS * BSTEP;  // e4m3: K = 32 per step
                uint8_t* st = stage0 + (size_t)s * a.stage_bytes;
                const size_t tg = (size_t)k.tt * NG + k.g;
                // one copy per group: the record is [s_x | B operand] (stage: off_b = off_par + PAR_BYTES)
                gstamp(a.trace, 6, i);
                ptx::mbar_arrive_expect_tx(&full[s], PAR_BYTES + bbytes);
                ptx::bulk_g2s(st + a.off_par, a.act + tg * a.P.rec, PAR_BYTES + bbytes, &full[s]);
                if (++s == S) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------ MMA issuer
        ptx::pdl_wait();
        constexpr uint32_t idesc = tc::idesc_bf16(128, PT);
        constexpr uint32_t idesc8 = tc::idesc_e4m3(128, PT);
        Walk k = walk0();
        int s = 0, ai = 0;
        uint32_t ph = 0, aph = 0;
        for (int i = 0; i < nw; ++i, next(k)) {
            const int b = i & 1;
            const bool f8 = WBITS == 4 && mode[k.tt];
            ptx::mbar_wait(&full[s], ph);      // B operand landed
            if (lane == 0) gstamp(a.trace, 0, i);
            ptx::mbar_wait(&afull[ai], aph);   // A operand written to TMEM
            if (lane == 0) gstamp(a.trace, 1, i);
            if (i >= 2) ptx::mbar_wait(&tempty[b], ((i >> 1) - 1) & 1);
            if (lane == 0) gstamp(a.trace, 2, i);
            tc::fence_after();
            if (lane == 0 && !(DYQ_PRE_EXP & 4)) {
                const uint32_t st = sbase + s * a.stage_bytes;
                const uint32_t d = tmem + b * PT;
                const uint32_t at = tmem + ACC_COLS + ai * A_COLS;
                if (f8) {
#pragma unroll
                    for (int ks = 0; ks < KSTEPS / 2; ++ks) {
                        const uint64_t bd = tc::smem_desc(st + a.off_b + ks * BSTEP, 128, 256);
                        tc::mma_f8_ta(d, at + ks * 8, bd, idesc8, ks > 0);
                    }
                } else {
#pragma unroll
                    for (int ks = 0; ks < KSTEPS; ++ks) {
                        const uint64_t bd = tc::smem_desc(st + a.off_b + ks * BSTEP, 128, 256);
                        tc::mma_f16_ta(d, at + ks * 8, bd, idesc, ks > 0);
                    }
                }
                tc::commit(ptx::smem_u32(&tfull[b]));
                tc::commit(ptx::smem_u32(&empty[s]));
                tc::commit(ptx::smem_u32(&aempty[ai]));
            } else if (lane == 0) {
                tc::commit(ptx::smem_u32(&tfull[b]));
                tc::commit(ptx::smem_u32(&empty[s]));
                tc::commit(ptx::smem_u32(&aempty[ai]));
            }
            __syncwarp();
            if (++s == S) { s = 0; ph ^= 1; }
            if (++ai == NA) { ai = 0; aph ^= 1; }
        }
    } else if (warp >= XF_WARP0 && warp < XF_WARP0 + XF_WARPS) {
        // ------------------------------------------------------ transform
        // Warp with TMEM quadrant q writes the A rows of sub-tiles 2q and 2q+1
        // (TMEM lanes 32q.. and 32q+16..).  Lane (gid, t) owns lane-chunk
        // (gid, t) of each sub-tile: rows gid and gid+8, k = 4t..4t+3 of every K
        // step -- exactly the 16x256b register fragment, so each sub-tile and
        // slab pair is one LDS.128 and one tcgen05.st.16x256b.x4.
        ptx::pdl_wait();
        const int q = warp & 3;
        Walk k = walk0();
        int s = 0, ai = 0;
        uint32_t ph = 0, aph = 0;
        for (int i = 0; i < nw; ++i, next(k)) {
            const bool f8 = WBITS == 4 && mode[k.tt];
            const int nsub = (k.tile == L.T128 - 1) ? L.nsub_last : 8;
            ptx::mbar_wait(&full[s], ph);
            if (i >= NA) ptx::mbar_wait(&aempty[ai], aph ^ 1);
            tc::fence_after();
            const uint8_t* st = stage0 + (size_t)s * a.stage_bytes;
            const uint8_t* zrow = st + a.off_meta + 512;
            const uint32_t at = tmem + ACC_COLS + ai * A_COLS;
#pragma unroll
            for (int si = 0; si < 2; ++si) {
                const int sub = 2 * q + si;
                if (sub >= nsub || (DYQ_PRE_EXP & 2)) break;
                const uint32_t tl = at + ((uint32_t)(32 * q + 16 * si) << 16);
                // zero points of rows gid and gid+8 are adjacent metadata slots
                const uint32_t z01 = *reinterpret_cast<const uint16_t*>(zrow + sub * 16 + 2 * (lane >> 2));
                if (WBITS == 4 && f8) {
                    // e4m3 (q - z_w): K step = slab; TMEM column 2t <- low nibbles,
                    // 2t + 1 <- high nibbles (e4m3_kpos), rows gid / gid + 8
                    // fp16 (1024 + q) pairs by byte permutes (0x64XX is exactly 1024 + XX),
                    // minus fp16 (1024 + z): exact (q - z), then one cvt to e4m3x2 per pair
                    const uint32_t zh0 = 0x64006400u | ((z01 & 0xffu) * 0x00010001u);
                    const uint32_t zh1 = 0x64006400u | ((z01 >> 8) * 0x00010001u);
#pragma unroll
                    for (int spi = 0; spi < SPG; ++spi) {
                        const uint4 wv = *reinterpret_cast<const uint4*>(st + ((spi * nsub + sub) * 32 + lane) * 16);
                        const uint32_t ws4[4] = {wv.x, wv.y, wv.z, wv.w};
                        uint32_t r[8];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int slab = j >> 1, rs = j & 1;
                            const uint32_t zz = rs ? zh1 : zh0;
#pragma unroll
                            for (int hn = 0; hn < 2; ++hn) {
                                const uint32_t x = hn ? (ws4[j] >> 4) & 0x0F0F0F0Fu : ws4[j] & 0x0F0F0F0Fu;
                                const uint32_t h01 = __byte_perm(x, 0x6464u, 0x5140u), h23 = __byte_perm(x, 0x6464u, 0x5342u);
                                const __half2 d01 = __hsub2(*reinterpret_cast<const __half2*>(&h01), *reinterpret_cast<const __half2*>(&zz));
                                const __half2 d23 = __hsub2(*reinterpret_cast<const __half2*>(&h23), *reinterpret_cast<const __half2*>(&zz));
                                const uint32_t p01 = __nv_cvt_halfraw2_to_fp8x2(*reinterpret_cast<const __half2_raw*>(&d01), __NV_SATFINITE, __NV_E4M3);
                                const uint32_t p23 = __nv_cvt_halfraw2_to_fp8x2(*reinterpret_cast<const __half2_raw*>(&d23), __NV_SATFINITE, __NV_E4M3);
                                r[slab * 4 + rs * 2 + hn] = (p01 & 0xffffu) | (p23 << 16);
                            }
                        }
                        tc::st16x256_x2(tl + spi * 16, r);
                    }
                } else if (WBITS == 4) {
                    // bf16 (128 + z) pairs; 0x43XX is exactly 128 + XX for XX < 128
                    const uint32_t zz0 = 0x43004300u | ((z01 & 0xffu) * 0x00010001u);
                    const uint32_t zz1 = 0x43004300u | ((z01 >> 8) * 0x00010001u);
#pragma unroll
                    for (int spi = 0; spi < SPG; ++spi) {
                        // W4 chunk words: (slab0,r0) (slab0,r1) (slab1,r0) (slab1,r1);
                        // byte i: k = 32 slab + 4t + i (low nibble), +16 (high nibble)
                        const uint4 wv = *reinterpret_cast<const uint4*>(st + ((spi * nsub + sub) * 32 + lane) * 16);
                        const uint32_t ws4[4] = {wv.x, wv.y, wv.z, wv.w};
                        uint32_t r[16];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int slab = j >> 1, rs = j & 1;
                            const uint32_t zz = rs ? zz1 : zz0;
                            const __nv_bfloat162 z2 = *reinterpret_cast<const __nv_bfloat162*>(&zz);
                            const uint32_t lo = ws4[j] & 0x0F0F0F0Fu, hi = (ws4[j] >> 4) & 0x0F0F0F0Fu;
                            const uint32_t p[4] = {__byte_perm(lo, 0x4343u, 0x5140u), __byte_perm(lo, 0x4343u, 0x5342u),
                                                   __byte_perm(hi, 0x4343u, 0x5140u), __byte_perm(hi, 0x4343u, 0x5342u)};
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const __nv_bfloat162 d2 = __hsub2(*reinterpret_cast<const __nv_bfloat162*>(&p[u]), z2);
                                // K step 2 slab + (u>>1) (high nibbles: +1), register (rows gid / gid+8, pair u&1)
                                r[(2 * slab + (u >> 1)) * 4 + rs * 2 + (u & 1)] = *reinterpret_cast<const uint32_t*>(&d2);
                            }
                        }
                        tc::st16x256_x4(tl + spi * 32, r);
                    }
                } else {
                    const float zf0 = 8388608.f + (float)(z01 & 0xffu), zf1 = 8388608.f + (float)(z01 >> 8);
#pragma unroll
                    for (int spi = 0; spi < SPG; ++spi) {
                        uint32_t r[16];
#pragma unroll
                        for (int slab = 0; slab < 2; ++slab) {
                            // W8 chunk words: (r0,h0) (r1,h0) (r0,h1) (r1,h1); byte i: k = 32 slab + 16 h + 4t + i
                            const uint4 wq = *reinterpret_cast<const uint4*>(
                                st + (((spi * nsub + sub) * 2 + slab) * 32 + lane) * 16);
                            const uint32_t R[4] = {wq.x, wq.y, wq.z, wq.w};
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                const int rs = j & 1, hh = j >> 1;
                                const float zf = rs ? zf1 : zf0;
                                float f[4];
#pragma unroll
                                for (int bb = 0; bb < 4; ++bb)  // (2^23 + byte) - (2^23 + z): exact q - z
                                    f[bb] = __uint_as_float(__byte_perm(R[j], 0x4B000000u, 0x7540u + bb)) - zf;
                                __nv_bfloat162 p0 = __floats2bfloat162_rn(f[0], f[1]);
                                __nv_bfloat162 p1 = __floats2bfloat162_rn(f[2], f[3]);
                                const int ks = 2 * slab + hh;
                                r[ks * 4 + rs * 2 + 0] = *reinterpret_cast<uint32_t*>(&p0);
                                r[ks * 4 + rs * 2 + 1] = *reinterpret_cast<uint32_t*>(&p1);
                            }
                        }
                        tc::st16x256_x4(tl + spi * 32, r);
                    }
                }
            }
            tc::wait_st();
            tc::fence_before();
            __syncwarp();
            if (lane == 0) {
                ptx::mbar_arrive(&afull[ai]);
                ptx::mbar_arrive(&empty[s]);
                if (warp == XF_WARP0) gstamp(a.trace, 5, i);
                if (warp == XF_WARP0 + 1) gstamp(a.trace, 7, i);
            }
            if (++s == S) { s = 0; ph ^= 1; }
            if (++ai == NA) { ai = 0; aph ^= 1; }
        }
    } else if (warp >= PR_WARP0) {
        // ------------------------------------------------------ promotion
        // 16x256b loads: thread (gid, t) holds rows 32q + 16 si + gid (+8) and
        // columns 8 blk + 2t, 2t+1 -- each thread needs only 18 of the 72 s_x.
        // Outer loop: this CTA's segments (one unit each); inner loop: the
        // segment's K-groups; the epilogue runs once per segment.
        ptx::pdl_wait();
        const bool tr0 = a.trace && threadIdx.x == PR_WARP0 * 32;
        if (tr0) trace_ev(a.trace, a.serial, 4, 1);
        const int e = warp - PR_WARP0;  // 0..7
        const int q = warp & 3;         // TMEM lane quadrant (hardware: warp id % 4)
        const int h = e >> 2;           // column half: tokens [72h, 72h + 72)
        const int gid = lane >> 2, t = lane & 3;
        constexpr int NC = PT / 2;      // 72 columns per warp
        constexpr int NB = NC / 8;      // 9 column blocks
        const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16) + h * NC;
        const int swo = (2 * q) * 16 + 2 * gid;  // s_w slot of rows gid / gid + 8 of sub-tile 2q (+16: 2q+1)
        const int sxo = h * NC + 2 * t;          // first s_x of this thread
        float facc[NB * 8];             // [blk][si][j]
#pragma unroll
        for (int c = 0; c < NB * 8; ++c) facc[c] = 0.f;
        int s = 0, i = 0;
        long long w = w0;
        while (w < w1) {
            const int u = (int)(w / NG);
            const int g0 = (int)(w - (long long)u * NG);
            const int g1 = (w1 - (long long)u * NG) < NG ? (int)(w1 - (long long)u * NG) : NG;  // exclusive
            const int tile = u / TT, tt = u - tile * TT;
            const int nsub = (tile == L.T128 - 1) ? L.nsub_last : 8;
            for (int g = g0; g < g1; ++g, ++i) {
                const int b = i & 1;
                ptx::mbar_wait(&tfull[b], (i >> 1) & 1);
                if (tr0 && i == 0) trace_ev(a.trace, a.serial, 4, 2);
                if (threadIdx.x == PR_WARP0 * 32) gstamp(a.trace, 3, i);
                tc::fence_after();
                const uint8_t* st = stage0 + (size_t)s * a.stage_bytes;
                const float* swp = reinterpret_cast<const float*>(st + a.off_meta) + swo;
                const float2 sw0 = *reinterpret_cast<const float2*>(swp);       // sub 2q
                const float2 sw1 = *reinterpret_cast<const float2*>(swp + 16);  // sub 2q+1
                const float* sxp = reinterpret_cast<const float*>(st + a.off_par) + sxo;
                const uint32_t tb = tq + b * PT;
                auto promote = [&](const uint32_t* v, int nblk, int blk0) {
#pragma unroll
                    for (int bi = 0; bi < nblk; ++bi) {
                        const float2 sx = *reinterpret_cast<const float2*>(sxp + (blk0 + bi) * 8);
#pragma unroll
                        for (int si = 0; si < 2; ++si) {
                            const uint32_t* vv = v + si * 4 * nblk + bi * 4;
                            const float2 sw = si ? sw1 : sw0;
                            float* fa = facc + ((blk0 + bi) * 2 + si) * 4;
                            float t0, t1, t2, t3;
                            ptx::mul2f(t0, t1, __uint_as_float(vv[0]), __uint_as_float(vv[1]), sx.x, sx.y);
                            ptx::mul2f(t2, t3, __uint_as_float(vv[2]), __uint_as_float(vv[3]), sx.x, sx.y);
                            ptx::fma2f(fa[0], fa[1], t0, t1, sw.x, sw.x);
                            ptx::fma2f(fa[2], fa[3], t2, t3, sw.y, sw.y);
                        }
                    }
                };
                auto partials = [&](const uint32_t* v, int nblk, int blk0) {
#pragma unroll
                    for (int bi = 0; bi < nblk; ++bi)
#pragma unroll
                        for (int si = 0; si < 2; ++si)
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                const int r = 32 * q + 16 * si + gid + 8 * (j >> 1);
                                const int m = tt * PT + sxo + (blk0 + bi) * 8 + (j & 1);
                                if (m < a.M && r < nsub * 16) {
                                    const int bm = a.row_bits ? a.row_bits[m] : a.bits;
                                    a.I_out[((size_t)m * L.N + tile * 128 + r) * NG + g] =
                                        bm == 16 ? 0 : __float2int_rn(__uint_as_float(v[si * 4 * nblk + bi * 4 + j]));
                                }
                            }
                };
                if (DYQ_PRE_EXP & 8) {
                    tc::fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&tempty[b]);
                } else {
#pragma unroll
                for (int c = 0; c < 2; ++c) {  // blocks 0-3, 4-7
                    uint32_t v[32];
                    tc::ld16x256_x4(tb + c * 32, v);
                    tc::ld16x256_x4(tb + (16u << 16) + c * 32, v + 16);
                    tc::wait_ld();
                    if (PARTIALS) partials(v, 4, c * 4);
                    else if (!(DYQ_PRE_EXP & 1)) promote(v, 4, c * 4);
                    else facc[c] += __uint_as_float(v[c]);
                }
                {  // block 8
                    uint32_t v[8];
                    tc::ld16x256_x1(tb + 64, v);
                    tc::ld16x256_x1(tb + (16u << 16) + 64, v + 4);
                    tc::wait_ld();
                    tc::fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&tempty[b]);
                    if (PARTIALS) partials(v, 1, 8);
                    else if (!(DYQ_PRE_EXP & 1)) promote(v, 1, 8);
                    else facc[2] += __uint_as_float(v[2]);
                }
                }
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&empty[s]);
                if (threadIdx.x == PR_WARP0 * 32) gstamp(a.trace, 4, i);
                if (++s == S) s = 0;
            }
            if (tr0) trace_ev(a.trace, a.serial, 4, 3);
            if constexpr (!PARTIALS) {
                // ---- segment end.  whole unit: y directly; otherwise an fp32
                // partial tile [144 tokens][128 rows] for prefill_fixup_kernel
                // (slot 2c: the CTA's first segment started mid-unit, else 2c+1)
                const bool whole = g0 == 0 && g1 == NG;
                const int rb = 32 * q + gid;  // row of element (si 0, j 0)
                const int mb = tt * PT + sxo;  // token of element (blk 0, j 0)
                // y for one finished tile: bf16 outputs are transposed through
                // the staging area ([token][row], 272-B rows) and leave as
                // coalesced 16-B stores of each token's 128-row segment;
                // fp32 outputs (tests) are stored directly.
                auto write_out = [&]() {
                    if (!TP && a.y_dtype == 0) {
                        const size_t n0 = (size_t)tile * 128 + rb;
#pragma unroll
                        for (int ii = 0; ii < NB * 8; ++ii) {
                            const int blk = ii >> 3, si = (ii >> 2) & 1, j = ii & 3;
                            const int dr = 16 * si + 8 * (j >> 1), dm = blk * 8 + (j & 1);
                            if (rb + dr < nsub * 16 && mb + dm < a.M && !(a.row_bits && a.row_bits[mb + dm] == 0))
                                reinterpret_cast<float*>(a.y)[(size_t)(mb + dm) * L.N + n0 + dr] = facc[ii];
                            facc[ii] = 0.f;
                        }
                        return;
                    }
                    uint8_t* stg = smem + a.off_stage;
#pragma unroll
                    for (int ii = 0; ii < NB * 8; ++ii) {
                        const int blk = ii >> 3, si = (ii >> 2) & 1, j = ii & 3;
                        *reinterpret_cast<__nv_bfloat16*>(stg + (sxo + blk * 8 + (j & 1)) * STG_ROW +
                                                          (rb + 16 * si + 8 * (j >> 1)) * 2) =
                            __float2bfloat16_rn(facc[ii]);
                        facc[ii] = 0.f;
                    }
                    ptx::named_bar_sync(1, PR_WARPS * 32);
                    const int tid = threadIdx.x - PR_WARP0 * 32;
                    for (int k = tid; k < PT * 16; k += PR_WARPS * 32) {
                        const int c = k >> 4, part = k & 15;
                        const int m = tt * PT + c;
                        if (part >= 2 * nsub || m >= a.M) continue;
                        if (a.row_bits && a.row_bits[m] == 0) continue;  // masked row: y untouched
                        const uint4 v = *reinterpret_cast<const uint4*>(stg + c * STG_ROW + part * 16);
                        if constexpr (TP) {  // bf16 into every rank's full y, this rank's columns
                            const size_t o = ((size_t)m * a.tp.ldy + a.tp.col0 + (size_t)tile * 128) * 2 + part * 16;
                            for (int p = 0; p < a.tp.n; ++p)
                                *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(a.tp.y[p]) + o) = v;
                        } else {
                            *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(a.y) +
                                                      ((size_t)m * L.N + (size_t)tile * 128) * 2 + part * 16) = v;
                        }
                    }
                    ptx::named_bar_sync(1, PR_WARPS * 32);  // staging free for the next tile
                };
                if (whole) {
                    write_out();
                    if constexpr (TP) {  // announce this unit's nsub sub-tiles (see dec_tp_announce)
                        if (threadIdx.x == PR_WARP0 * 32) {
                            __threadfence_system();
                            for (int p = 0; p < a.tp.n; ++p) atomicAdd_system(a.tp.flag[p], (unsigned long long)nsub);
                        }
                    }
                } else if (g0 != 0) {
                    // HEAD part of a unit split across CTAs (this CTA's first
                    // segment): an fp32 partial tile [144 tokens][128 rows] in
                    // slot c, then one arrival on the reducer's counter.  The
                    // reducer is the CTA holding the unit's first groups, which
                    // reaches them at the END of its range, so it rarely waits.
                    float* slot = a.part + (size_t)blockIdx.x * (PT * 128) + sxo * 128 + rb;
#pragma unroll
                    for (int ii = 0; ii < NB * 8; ++ii) {
                        const int blk = ii >> 3, si = (ii >> 2) & 1, j = ii & 3;
                        __stcg(slot + (blk * 8 + (j & 1)) * 128 + 16 * si + 8 * (j >> 1), facc[ii]);
                        facc[ii] = 0.f;
                    }
                    ptx::named_bar_sync(1, PR_WARPS * 32);
                    if (threadIdx.x == PR_WARP0 * 32) {
                        const long long ub = (long long)u * NG;
                        const int c_lo = (int)(((ub + 1) * gridDim.x - 1) / a.W);  // CTA holding group ub
                        __threadfence();
                        atomicAdd(a.cnt + c_lo, 1);
                    }
                } else {
                    // REDUCER: this CTA holds the unit's first groups (its last
                    // segment); the other contributors c + 1 .. c_hi each
                    // published a head slot.  Sum in CTA order (deterministic).
                    const long long ue = (long long)(u + 1) * NG;
                    const int c_hi = (int)((ue * gridDim.x - 1) / a.W);  // CTA holding group ue - 1
                    if (threadIdx.x == PR_WARP0 * 32) {
                        const int need = c_hi - (int)blockIdx.x;
                        while (ptx::ld_acquire_gpu(a.cnt + blockIdx.x) < need) __nanosleep(64);
                        a.cnt[blockIdx.x] = 0;  // self-reset (no other arrival targets this CTA this call)
                    }
                    ptx::named_bar_sync(1, PR_WARPS * 32);
                    for (int cc = (int)blockIdx.x + 1; cc <= c_hi; ++cc) {
                        const float* slot = a.part + (size_t)cc * (PT * 128) + sxo * 128 + rb;
#pragma unroll
                        for (int ii = 0; ii < NB * 8; ++ii) {
                            const int blk = ii >> 3, si = (ii >> 2) & 1, j = ii & 3;
                            facc[ii] += __ldcg(slot + (blk * 8 + (j & 1)) * 128 + 16 * si + 8 * (j >> 1));
                        }
                    }
                    write_out();
                }
            }
            if (tr0) trace_ev(a.trace, a.serial, 4, 4);
            w += g1 - g0;
        }
    }
    tc::fence_before();
    __syncthreads();
    if (threadIdx.x == 0) trace_ev(a.trace, a.serial, 4, 5);
    if (warp == 1) {
        tc::fence_after();
        tc::dealloc(tmem, 512);
    }
}

// -------------------------------------------- prefill activation quantizer
// One CTA per (token tile tt, K-group g); four threads per token row of the
// tile (576 threads): each holds G/4 of the group's inputs (16-B loads), the
// quad combines min / max and the non-finite index with two shuffles, and
// each thread writes its part of the B operand in the UMMA canonical K-major
// layout
//   bf16: [tt][g][K step ks][row>>3][kk>>3][row&7][kk&7]   (16 k per K step)
//   e4m3: [tt][g][K step ks][row>>3][p>>4][row&7][p&15]    (32 k per K step,
//         p = e4m3_kpos(k); at G = 64 a K step spans a thread pair, which
//         swaps two words to form whole 16-B chunks)
// holding the centred codes Xq - z_x of Eq. (2) for integer tokens (exact in
// bf16 / e4m3), x itself for A16 tokens and 0 for absent rows; and s_x per
// token (1 for A16 tokens, 0 for absent rows) at the head of the record.
template <int KH>  // inputs per thread = G / AQP_TPR
__global__ void __launch_bounds__(AQP_TPR * PT) actquant_pre_kernel(WLayout L, const uint16_t* __restrict__ x, int M,
                                                          const int32_t* __restrict__ row_bits, int bits,
                                                          uint8_t* __restrict__ act, PreActLayout P, int64_t* err,
                                                          int e4m3_ok, int gated, const int32_t* gate) {
    if (gate_closed(gate)) return;
    ptx::pdl_wait();  // x / row_bits come from the preceding kernels
    ptx::pdl_launch_dependents();
    const int NG = L.NG;
    const int g = blockIdx.x % NG, tt = blockIdx.x / NG;
    const int row = threadIdx.x / AQP_TPR, half = threadIdx.x % AQP_TPR;  // half: quarter of the group
    const int m = tt * PT + row;
    const int b = m < M ? (row_bits ? row_bits[m] : bits) : 0;
    // tile mode (dyq_pre_tile_e4m3): every present token of tile tt at A2 / A4
    const bool f8 = e4m3_ok && __syncthreads_and(m >= M || b == 2 || b == 4);
    if (threadIdx.x == 0 && g == 0) act[P.mode_off + tt] = f8 ? 1 : 0;  // read by the MMA kernel
    aqp_job<KH>(L, x, M, row_bits, bits, act, P, err, f8, gated, tt, g, row, half);
}

// ------------------------------------------------------------------ host
// e4m3 mode: W4 weights only (W8 centred codes reach +-255).  Off by default:
// bit-exact, but its A-operand transform (cvt to e4m3) outweighs the halved MMA
// count with 4 transform warps (B200: gate|up 137 vs 130 us);
// DYQ_PRE_E4M3=1 enables it (read per call, so tests can exercise it).  Both
// kernels of a call see the same value.
static bool pre_e4m3_enabled(const WLayout& L) {
    const char* v = getenv("DYQ_PRE_E4M3");
    return v && atoi(v) != 0 && L.wbits == 4;
}

bool prefill_e4m3(const WLayout& L) { return pre_e4m3_enabled(L); }

PreActLayout pre_act_layout(const WLayout& L, int M) {
    PreActLayout P;
    const int TT = (M + PT - 1) / PT;
    P.codes_group = 0;
    P.codes_off = 0;
    P.x16_group = (size_t)(L.G / 16) * PT * 32;  // B operand bytes per (tile, group)
    P.rec = PAR_BYTES + P.x16_group;             // record [s_x (144 f32) | B]
    P.x16_off = PAR_BYTES;
    P.par_off = 0;
    P.mode_off = ((size_t)TT * L.NG * P.rec + 255) & ~(size_t)255;
    P.bytes = P.mode_off + (((size_t)TT + 255) & ~(size_t)255);
    return P;
}

dyq_status_t launch_actquant_pre(const WLayout& L, const uint16_t* x, int M, const int32_t* row_bits, int bits,
                                 void* act, int64_t* err, cudaStream_t st, int gated) {
    const PreActLayout P = pre_act_layout(L, M);
    const int TT = (M + PT - 1) / PT;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(TT * L.NG));
    cfg.blockDim = dim3(AQP_TPR * PT);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, L.G == 64 ? actquant_pre_kernel<16> : actquant_pre_kernel<32>, L, x, M, row_bits, bits,
                                             reinterpret_cast<uint8_t*>(act), P, err, pre_e4m3_enabled(L) ? 1 : 0, gated, g_gate);
    if (e != cudaSuccess) return set_error(DYQ_ECUDA, "actquant_pre_kernel launch: %s", cudaGetErrorString(e));
    return check_launch("actquant_pre_kernel");
}

static int sm_count() {
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

// Persistent stream-K grid: one CTA per SM (at most), each with a contiguous
// range of >= DYQ_PRE_MIN_GROUPS K-groups of the flat (tile, token tile, group)
// order.  DYQ_PRE_CTAS=n overrides the CTA count (experiments, tools/).
static int prefill_grid(const WLayout& L, int M) {
    static const int force = [] {
        const char* v = getenv("DYQ_PRE_CTAS");
        return v ? atoi(v) : 0;
    }();
    const long long W = (long long)L.T128 * ((M + PT - 1) / PT) * L.NG;
    long long P = force > 0 ? force : W / DYQ_PRE_MIN_GROUPS;
    if (P > sm_count()) P = sm_count();  // all CTAs co-resident: a reducer may wait on any other CTA
    if (P > W) P = W;
    return (int)(P < 1 ? 1 : P);
}

size_t prefill_part_bytes(const WLayout& L, int M) {
    return M > 0 ? (size_t)prefill_grid(L, M) * PT * 128 * sizeof(float) : 0;
}

// Largest number of CTAs sharing one (tile, token tile) unit (1 = no unit is
// split across CTAs; dyq_qlinear_plan).
int prefill_ksplit(const WLayout& L, int M) {
    if (M <= 0) return 1;
    const int P = prefill_grid(L, M);
    const long long W = (long long)L.T128 * ((M + PT - 1) / PT) * L.NG;
    int best = 1, run = 1;
    long long prev_unit = -1;
    for (int c = 1; c < P; ++c) {
        const long long b = sk_begin(W, P, c);  // boundary between CTAs c-1 and c
        if (b % L.NG == 0) continue;
        run = (b / L.NG == prev_unit) ? run + 1 : 2;  // each mid-unit boundary adds a contributor
        prev_unit = b / L.NG;
        best = run > best ? run : best;
    }
    return best;
}

template <int WBITS, int SPG, bool PARTIALS, bool TP = false>
static cudaError_t pre_launch(const PreArgs& a0, int grid, cudaStream_t st) {
    PreArgs a = a0;
    constexpr int G = SPG * 64;
    const int raw = SPG * 8 * 512 * (WBITS / 4);
    const int bbytes = (G / 16) * PT * 32;
    a.off_meta = raw;
    a.off_par = (a.off_meta + META_BLOCK + 127) & ~127;
    a.off_b = a.off_par + PAR_BYTES;  // 16-B aligned (canonical no-swizzle layout)
    a.stage_bytes = (a.off_b + bbytes + 127) & ~127;
    constexpr int stg_bytes = PT * STG_ROW;
    a.stages = (226 * 1024 - 1024 - stg_bytes) / a.stage_bytes;
    if (a.stages > DYQ_PRE_MAX_STAGES) a.stages = DYQ_PRE_MAX_STAGES;
    if (a.stages < 2) a.stages = 2;
    a.off_stage = 1024 + a.stages * a.stage_bytes;
    const size_t smem = (size_t)a.off_stage + stg_bytes;
    auto kern = qlinear_prefill_kernel<WBITS, SPG, PARTIALS, TP>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(PRE_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr1[1];
    attr1[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr1[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr1;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

template <bool PARTIALS, bool TP = false>
static cudaError_t pre_dispatch(const PreArgs& a, int grid, cudaStream_t st) {
    if (a.L.wbits == 4)
        return a.L.G == 64 ? pre_launch<4, 1, PARTIALS, TP>(a, grid, st) : pre_launch<4, 2, PARTIALS, TP>(a, grid, st);
    return a.L.G == 64 ? pre_launch<8, 1, PARTIALS, TP>(a, grid, st) : pre_launch<8, 2, PARTIALS, TP>(a, grid, st);
}

dyq_status_t launch_prefill(const WLayout& L, const void* codes, const void* meta, int M, const int32_t* row_bits,
                            int bits, void* y, int y_dtype, int32_t* I_out, const void* act, cudaStream_t st,
                            const TpPeers* tp) {
    if (M <= 0) return DYQ_OK;
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
    a.TT = (M + PT - 1) / PT;
    a.W = (long long)L.T128 * a.TT * L.NG;
    a.tp = {};
    if (tp) a.tp = *tp;
    // the fused TP epilogue announces whole units: one unit per CTA
    const int grid = tp ? L.T128 * a.TT : prefill_grid(L, M);
    a.part = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(const_cast<void*>(act)) +
                                      ((a.P.bytes + 255) & ~(size_t)255));
    a.cnt = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(const_cast<void*>(act)) - PRE_CNT_BYTES);
    a.trace = g_trace;
    a.serial = g_trace_serial++;
    a.gate = g_gate;
    const cudaError_t e = I_out ? pre_dispatch<true>(a, grid, st)
                          : tp  ? pre_dispatch<false, true>(a, grid, st)
                                : pre_dispatch<false>(a, grid, st);
    if (e != cudaSuccess) return set_error(DYQ_ECUDA, "qlinear_prefill_kernel launch: %s", cudaGetErrorString(e));
    return DYQ_OK;
}

}  // namespace dyq
