// dyq_model.cu -- the policy step around the quantized linears (SURVEY.md §8(a)
// A9): Llama-2 / OpenVLA block glue and the step orchestration
// select_bits -> route -> prefill -> action head -> decode passes -> detok
// (P:300-321).  The glue is not the paper's method: plain,
// memory-bound kernels (RMSNorm, RoPE, SiLU*mul) and CUDA-core attention over
// at most n_vis + n_text + n_act = 295 positions; every FLOP that matters
// runs in the qlinear kernels (dyq_decode.cu / dyq_prefill.cu).
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "dyq_internal.cuh"
#include "dyq_ptx.cuh"

namespace dyq {

constexpr int HD = 128;  // head dim (Llama-2-7B: 4096 / 32)

__device__ __forceinline__ float bf2f(uint16_t h) { return __uint_as_float((uint32_t)h << 16); }
__device__ __forceinline__ uint16_t f2bf(float f) { return __bfloat16_as_ushort(__float2bfloat16_rn(f)); }

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    float s = 0.f;
    for (int i = 0; i < nw; ++i) s += red[i];
    return s;
}

// h (+)= delta; y = RMSNorm(h) * w  (fp32 statistics over the bf16 h values)
__global__ void add_rmsnorm_kernel(uint16_t* __restrict__ h, const uint16_t* __restrict__ delta,
                                   const uint16_t* __restrict__ w, int d, float eps, uint16_t* __restrict__ y) {
    __shared__ float red[32];
    const size_t row = blockIdx.x;
    uint16_t* hr = h + row * d;
    float ss = 0.f;
    for (int i = threadIdx.x * 2; i < d; i += blockDim.x * 2) {
        float a = bf2f(hr[i]), b = bf2f(hr[i + 1]);
        if (delta) {
            a = bf2f(f2bf(a + bf2f(delta[row * d + i])));
            b = bf2f(f2bf(b + bf2f(delta[row * d + i + 1])));
            hr[i] = f2bf(a);
            hr[i + 1] = f2bf(b);
        }
        ss += a * a + b * b;
    }
    const float inv = rsqrtf(block_sum(ss, red) / (float)d + eps);
    for (int i = threadIdx.x * 2; i < d; i += blockDim.x * 2) {
        y[row * d + i] = f2bf(bf2f(hr[i]) * inv * bf2f(w[i]));
        y[row * d + i + 1] = f2bf(bf2f(hr[i + 1]) * inv * bf2f(w[i + 1]));
    }
}

// Same op, one 16-B vector of 8 elements per thread (d = 8 * blockDim.x), h
// kept in registers between the statistics and the output pass; PDL-launched.
// Prefill activation records of the next linear written by add_rmsnorm8's
// epilogue (policy step prefill pass): act = the linear's prefill activation
// area (null: off), rows 0 .. M-1.
struct PQuant {
    uint8_t* act;
    PreActLayout P;
    WLayout L;
    const int32_t* row_bits;
    int bits, M;
    int64_t* err;
};

__global__ void __launch_bounds__(1024) add_rmsnorm8_kernel(uint16_t* __restrict__ h,
                                                            const uint16_t* __restrict__ delta,
                                                            const uint16_t* __restrict__ w, int d, float eps,
                                                            uint16_t* __restrict__ y, PQuant pq) {
    __shared__ float red[32];
    ptx::pdl_wait();
    ptx::pdl_launch_dependents();
    const size_t o = (size_t)blockIdx.x * d + threadIdx.x * 8;
    const uint4 hv = *reinterpret_cast<const uint4*>(h + o);
    const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w};
    float a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = bf2f((uint16_t)(hw[k >> 1] >> (16 * (k & 1))));
    if (delta) {
        const uint4 dv = *reinterpret_cast<const uint4*>(delta + o);
        const uint32_t dw[4] = {dv.x, dv.y, dv.z, dv.w};
        uint32_t nh[4];
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
            const uint16_t lo = f2bf(a[k] + bf2f((uint16_t)(dw[k >> 1] & 0xffffu)));
            const uint16_t hi = f2bf(a[k + 1] + bf2f((uint16_t)(dw[k >> 1] >> 16)));
            a[k] = bf2f(lo);
            a[k + 1] = bf2f(hi);
            nh[k >> 1] = (uint32_t)lo | ((uint32_t)hi << 16);
        }
        *reinterpret_cast<uint4*>(h + o) = make_uint4(nh[0], nh[1], nh[2], nh[3]);
    }
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < 8; k += 2) ss += a[k] * a[k] + a[k + 1] * a[k + 1];
    const float inv = rsqrtf(block_sum(ss, red) / (float)d + eps);
    const uint4 wv = *reinterpret_cast<const uint4*>(w + threadIdx.x * 8);
    const uint32_t ww[4] = {wv.x, wv.y, wv.z, wv.w};
    uint32_t yo[4];
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
        const uint16_t lo = f2bf(a[k] * inv * bf2f((uint16_t)(ww[k >> 1] & 0xffffu)));
        const uint16_t hi = f2bf(a[k + 1] * inv * bf2f((uint16_t)(ww[k >> 1] >> 16)));
        yo[k >> 1] = (uint32_t)lo | ((uint32_t)hi << 16);
    }
    *reinterpret_cast<uint4*>(y + o) = make_uint4(yo[0], yo[1], yo[2], yo[3]);
    if (!pq.act) return;
    // the row's records: thread (g, quarter) = one aqp_job (NG * 4 threads,
    // whole warps; bf16 operand mode), and the token tile's mode byte
    __syncthreads();  // the row of y is written (CTA-visible)
    const int row = blockIdx.x, tt = row / PRE_PT;
    const int t = (int)threadIdx.x;
    if (t < pq.L.NG * AQP_TPR) {
        if (pq.L.G == 64)
            aqp_job<16>(pq.L, y, pq.M, pq.row_bits, pq.bits, pq.act, pq.P, pq.err, false, 0, tt, t / AQP_TPR,
                        row - tt * PRE_PT, t % AQP_TPR);
        else
            aqp_job<32>(pq.L, y, pq.M, pq.row_bits, pq.bits, pq.act, pq.P, pq.err, false, 0, tt, t / AQP_TPR,
                        row - tt * PRE_PT, t % AQP_TPR);
    }
    if (t == 0 && row == tt * PRE_PT) pq.act[pq.P.mode_off + tt] = 0;  // bf16 operands
}

// Launch with programmatic dependent launch (every kernel launched this way
// calls griddepcontrol.wait before reading anything a previous kernel wrote).
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// rotate_half RoPE of one pair (i, i + HD/2) at position pos: the one
// definition rope_kernel and the fused decode attention (attn_decode2_kernel
// with theta > 0) share, with explicit roundings (no contraction), so the two
// paths give the same bits
__device__ __forceinline__ void rope_pair(float x1, float x2, float pos, int i, float theta, uint16_t& o1,
                                          uint16_t& o2) {
    const float inv_freq = powf(theta, -2.f * (float)i / (float)HD);
    float sn, cs;
    sincosf(__fmul_rn(pos, inv_freq), &sn, &cs);
    o1 = f2bf(__fsub_rn(__fmul_rn(x1, cs), __fmul_rn(x2, sn)));
    o2 = f2bf(__fadd_rn(__fmul_rn(x2, cs), __fmul_rn(x1, sn)));
}

// rotate_half RoPE on the q and k parts: pairs (i, i + HD/2) of every head
__global__ void rope_kernel(uint16_t* __restrict__ qkv, int M, int S, int pos0, int d, int H, float theta) {
    ptx::pdl_wait();
    ptx::pdl_launch_dependents();
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int half = HD / 2;
    const size_t per_row = (size_t)2 * H * half;
    if (idx >= (size_t)M * per_row) return;
    const int m = (int)(idx / per_row);
    const int r = (int)(idx % per_row);
    const int which = r / (H * half);  // 0 = q, 1 = k
    const int hh = (r / half) % H, i = r % half;
    uint16_t* p = qkv + (size_t)m * 3 * d + (size_t)which * d + hh * HD;
    rope_pair(bf2f(p[i]), bf2f(p[i + half]), (float)(m % S + pos0), i, theta, p[i], p[i + half]);
}

__device__ __forceinline__ size_t kv_off(int e, int l, int kv, int pos, int L, int T, int d) {
    return ((((size_t)e * L + l) * 2 + kv) * T + pos) * d;
}

// Causal attention, prefill.  CTA = (32-query block, head, episode), 8 warps x
// 4 queries.  K (rows padded to 130 bf16: conflict-free lane-per-key dot
// products) and V of keys [0, qend) staged in shared memory.
constexpr int AQB = 32;
constexpr int AKP = HD + 2;
__host__ __device__ inline size_t attn_ks_bytes(int S) { return ((size_t)S * AKP * 2 + 15) & ~(size_t)15; }
__global__ void __launch_bounds__(256) attn_prefill_kernel(const uint16_t* __restrict__ qkv, int S, int d, int H,
                                                           uint16_t* __restrict__ kv, int layer, int L, int T,
                                                           uint16_t* __restrict__ out) {
    extern __shared__ __align__(16) uint8_t sm[];
    const int q0 = blockIdx.x * AQB, hh = blockIdx.y, e = blockIdx.z;
    const int qend = min(q0 + AQB, S);
    uint16_t* Ks = reinterpret_cast<uint16_t*>(sm);
    uint16_t* Vs = reinterpret_cast<uint16_t*>(sm + attn_ks_bytes(S));
    float* qs = reinterpret_cast<float*>(sm + attn_ks_bytes(S) + (size_t)S * HD * 2);  // [8][HD]
    float* ps = qs + 8 * HD;                                                          // [8][S]
    const size_t rs = (size_t)3 * d;
    const uint16_t* base = qkv + (size_t)e * S * rs;
    // generic path (any 2-byte alignment of qkv / kv): element-wise global
    // accesses, 32-bit only in shared memory
    for (int idx = threadIdx.x; idx < qend * (HD / 2); idx += blockDim.x) {
        const int j = idx / (HD / 2), c = (idx % (HD / 2)) * 2;
        const uint16_t* kp = base + j * rs + d + hh * HD + c;
        const uint16_t* vp = base + j * rs + 2 * d + hh * HD + c;
        const uint16_t k0 = kp[0], k1 = kp[1], v0 = vp[0], v1 = vp[1];
        *reinterpret_cast<uint32_t*>(Ks + j * AKP + c) = (uint32_t)k0 | ((uint32_t)k1 << 16);
        *reinterpret_cast<uint32_t*>(Vs + j * HD + c) = (uint32_t)v0 | ((uint32_t)v1 << 16);
        if (j >= q0) {  // this block's rows go to the KV cache
            uint16_t* kc = kv + kv_off(e, layer, 0, j, L, T, d) + hh * HD + c;
            uint16_t* vc = kv + kv_off(e, layer, 1, j, L, T, d) + hh * HD + c;
            kc[0] = k0; kc[1] = k1;
            vc[0] = v0; vc[1] = v1;
        }
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float scale = rsqrtf((float)HD);
    float* qw = qs + warp * HD;
    float* pw = ps + warp * S;
    for (int qi = 0; qi < AQB / 8; ++qi) {
        const int q = q0 + warp * (AQB / 8) + qi;
        if (q >= qend) break;
        for (int c = lane; c < HD; c += 32) qw[c] = bf2f(base[q * rs + hh * HD + c]) * scale;
        __syncwarp();
        float mx = -INFINITY;
        for (int j = lane; j <= q; j += 32) {
            const uint16_t* kr = Ks + j * AKP;
            float s = 0.f;
#pragma unroll 8
            for (int c = 0; c < HD; c += 2) {
                const uint32_t k2 = *reinterpret_cast<const uint32_t*>(kr + c);
                s = fmaf(qw[c], __uint_as_float(k2 << 16), s);
                s = fmaf(qw[c + 1], __uint_as_float(k2 & 0xffff0000u), s);
            }
            pw[j] = s;
            mx = fmaxf(mx, s);
        }
        mx = warp_max(mx);
        float sum = 0.f;
        for (int j = lane; j <= q; j += 32) {
            const float p = __expf(pw[j] - mx);
            pw[j] = p;
            sum += p;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        __syncwarp();
        float o0 = 0.f, o1 = 0.f, o2 = 0.f, o3 = 0.f;
        for (int j = 0; j <= q; ++j) {
            const float p = pw[j];
            const uint2 v = *reinterpret_cast<const uint2*>(Vs + j * HD + lane * 4);
            o0 = fmaf(p, __uint_as_float(v.x << 16), o0);
            o1 = fmaf(p, __uint_as_float(v.x & 0xffff0000u), o1);
            o2 = fmaf(p, __uint_as_float(v.y << 16), o2);
            o3 = fmaf(p, __uint_as_float(v.y & 0xffff0000u), o3);
        }
        const float inv = 1.f / sum;
        uint16_t* orow = out + ((size_t)e * S + q) * d + hh * HD + lane * 4;
        orow[0] = f2bf(o0 * inv);
        orow[1] = f2bf(o1 * inv);
        orow[2] = f2bf(o2 * inv);
        orow[3] = f2bf(o3 * inv);
        __syncwarp();
    }
}

// Causal prefill attention on the tensor cores (mma.sync m16n8k16 bf16 -> fp32,
// FlashAttention-2 style online softmax).  CTA = (64-query block, head,
// episode), 4 warps x 16 queries; Q fragments stay in registers, K / V blocks of
// 64 keys are staged in shared memory (row stride 136 bf16: conflict-free
// ldmatrix), S = Q K^T and O += P V with P re-packed from the S accumulators.
// The CTA also writes its own 64 keys' K / V rows into the KV cache.
constexpr int FQ = 64, FK = 64, FST = HD + 8;  // query / key block, smem row stride (bf16)
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf2(float lo, float hi) {
    return (uint32_t)f2bf(lo) | ((uint32_t)f2bf(hi) << 16);
}
__global__ void __launch_bounds__(128) attn_prefill_tc_kernel(const uint16_t* __restrict__ qkv, int S, int d, int H,
                                                              uint16_t* __restrict__ kv, int layer, int L, int T,
                                                              uint16_t* __restrict__ out) {
    extern __shared__ __align__(16) uint16_t fs[];
    uint16_t* Qs = fs;              // [FQ][FST]
    uint16_t* Ks = Qs + FQ * FST;   // [FK][FST]
    uint16_t* Vs = Ks + FK * FST;   // [FK][FST]
    ptx::pdl_wait();
    ptx::pdl_launch_dependents();
    const int q0 = blockIdx.x * FQ, hh = blockIdx.y, e = blockIdx.z;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, t = lane & 3;
    const size_t rs = (size_t)3 * d;
    const uint16_t* base = qkv + (size_t)e * S * rs + hh * HD;
    // ---- Q tile -> smem -> fragments (8 k-steps of 16 dims)
    for (int i = tid; i < FQ * (HD / 8); i += 128) {
        const int r = i / (HD / 8), c = (i % (HD / 8)) * 8;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (q0 + r < S) v = *reinterpret_cast<const uint4*>(base + (size_t)(q0 + r) * rs + c);
        *reinterpret_cast<uint4*>(Qs + r * FST + c) = v;
    }
    __syncthreads();
    uint32_t qf[HD / 16][4];
    {
        const uint32_t qb = ptx::smem_u32(Qs + (warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8) * FST + (lane >> 4) * 8);
#pragma unroll
        for (int ks = 0; ks < HD / 16; ++ks) ldsm_x4(qb + ks * 32, qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3]);
    }
    float o[HD / 8][4];
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;  // rows g and g + 8 of this warp
    const float sl2 = rsqrtf((float)HD) * 1.4426950408889634f;  // scale * log2(e)
    const int qr0 = q0 + warp * 16 + g, qr1 = qr0 + 8;
    const int kb_last = min(q0 + FQ - 1, S - 1) / FK;
    for (int kb = 0; kb <= kb_last; ++kb) {
        const int k0 = kb * FK;
        __syncthreads();  // previous block's K / V reads done
        for (int i = tid; i < FK * (HD / 8); i += 128) {
            const int r = i / (HD / 8), c = (i % (HD / 8)) * 8;
            uint4 kk = make_uint4(0u, 0u, 0u, 0u), vv = kk;
            if (k0 + r < S) {
                kk = *reinterpret_cast<const uint4*>(base + (size_t)(k0 + r) * rs + d + c);
                vv = *reinterpret_cast<const uint4*>(base + (size_t)(k0 + r) * rs + 2 * d + c);
                if (k0 + r >= q0 && k0 + r < q0 + FQ) {  // this CTA's keys go to the KV cache
                    *reinterpret_cast<uint4*>(kv + kv_off(e, layer, 0, k0 + r, L, T, d) + hh * HD + c) = kk;
                    *reinterpret_cast<uint4*>(kv + kv_off(e, layer, 1, k0 + r, L, T, d) + hh * HD + c) = vv;
                }
            }
            *reinterpret_cast<uint4*>(Ks + r * FST + c) = kk;
            *reinterpret_cast<uint4*>(Vs + r * FST + c) = vv;
        }
        __syncthreads();
        // ---- S = Q K^T: 8 n-tiles of 8 keys
        float sacc[FK / 8][4];
#pragma unroll
        for (int j = 0; j < FK / 8; ++j) sacc[j][0] = sacc[j][1] = sacc[j][2] = sacc[j][3] = 0.f;
        const uint32_t kbse = ptx::smem_u32(Ks + ((lane & 7) + (lane >> 4) * 8) * FST + ((lane >> 3) & 1) * 8);
#pragma unroll
        for (int jp = 0; jp < FK / 16; ++jp) {  // pairs of n-tiles
#pragma unroll
            for (int ks = 0; ks < HD / 16; ++ks) {
                uint32_t b0, b1, b2, b3;
                ldsm_x4(kbse + (jp * 16 * FST + ks * 16) * 2, b0, b1, b2, b3);
                mma16816(sacc[2 * jp], qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3], b0, b1);
                mma16816(sacc[2 * jp + 1], qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3], b2, b3);
            }
        }
        // ---- causal mask, online softmax (base 2)
        float bm0 = -INFINITY, bm1 = -INFINITY;
#pragma unroll
        for (int j = 0; j < FK / 8; ++j) {
            const int kc = k0 + j * 8 + 2 * t;
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                sacc[j][u] = (kc + u <= qr0 && kc + u < S) ? sacc[j][u] * sl2 : -INFINITY;
                sacc[j][2 + u] = (kc + u <= qr1 && kc + u < S) ? sacc[j][2 + u] * sl2 : -INFINITY;
                bm0 = fmaxf(bm0, sacc[j][u]);
                bm1 = fmaxf(bm1, sacc[j][2 + u]);
            }
        }
#pragma unroll
        for (int off = 1; off < 4; off <<= 1) {
            bm0 = fmaxf(bm0, __shfl_xor_sync(0xffffffffu, bm0, off));
            bm1 = fmaxf(bm1, __shfl_xor_sync(0xffffffffu, bm1, off));
        }
        const float nm0 = fmaxf(m0, bm0), nm1 = fmaxf(m1, bm1);
        // rows with no visible key yet keep m = -inf: use 0 as the exponent base there
        const float b0e = nm0 == -INFINITY ? 0.f : nm0, b1e = nm1 == -INFINITY ? 0.f : nm1;
        const float c0 = exp2f(m0 - b0e), c1 = exp2f(m1 - b1e);
        m0 = nm0;
        m1 = nm1;
        float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
        for (int j = 0; j < FK / 8; ++j) {
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                sacc[j][u] = exp2f(sacc[j][u] - b0e);
                sacc[j][2 + u] = exp2f(sacc[j][2 + u] - b1e);
                rs0 += sacc[j][u];
                rs1 += sacc[j][2 + u];
            }
        }
        l0 = l0 * c0 + rs0;
        l1 = l1 * c1 + rs1;
#pragma unroll
        for (int i = 0; i < HD / 8; ++i) {
            o[i][0] *= c0;
            o[i][1] *= c0;
            o[i][2] *= c1;
            o[i][3] *= c1;
        }
        // ---- O += P V: 4 k-steps of 16 keys, 16 dim-tiles of 8
        const uint32_t vbse = ptx::smem_u32(Vs + ((lane & 7) + ((lane >> 3) & 1) * 8) * FST + (lane >> 4) * 8);
#pragma unroll
        for (int kk = 0; kk < FK / 16; ++kk) {
            // P = P_hi + P_lo, both bf16 (the fp32 probabilities to ~2^-16
            // relative): two MMAs per V fragment instead of one bf16-rounded P
            uint32_t ah[4], al[4];
            const float* pv[4] = {&sacc[2 * kk][0], &sacc[2 * kk][2], &sacc[2 * kk + 1][0], &sacc[2 * kk + 1][2]};
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const uint16_t h0 = f2bf(pv[r][0]), h1 = f2bf(pv[r][1]);
                ah[r] = (uint32_t)h0 | ((uint32_t)h1 << 16);
                al[r] = pack_bf2(pv[r][0] - bf2f(h0), pv[r][1] - bf2f(h1));
            }
#pragma unroll
            for (int np = 0; np < HD / 16; ++np) {
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(vbse + (kk * 16 * FST + np * 16) * 2, b0, b1, b2, b3);
                mma16816(o[2 * np], ah[0], ah[1], ah[2], ah[3], b0, b1);
                mma16816(o[2 * np + 1], ah[0], ah[1], ah[2], ah[3], b2, b3);
                mma16816(o[2 * np], al[0], al[1], al[2], al[3], b0, b1);
                mma16816(o[2 * np + 1], al[0], al[1], al[2], al[3], b2, b3);
            }
        }
    }
    // ---- normalise and store (rows qr0, qr1)
#pragma unroll
    for (int off = 1; off < 4; off <<= 1) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, off);
        l1 += __shfl_xor_sync(0xffffffffu, l1, off);
    }
    const float i0 = 1.f / l0, i1 = 1.f / l1;
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
        const int c = hh * HD + i * 8 + 2 * t;
        if (qr0 < S)
            *reinterpret_cast<uint32_t*>(out + ((size_t)e * S + qr0) * d + c) = pack_bf2(o[i][0] * i0, o[i][1] * i0);
        if (qr1 < S)
            *reinterpret_cast<uint32_t*>(out + ((size_t)e * S + qr1) * d + c) = pack_bf2(o[i][2] * i1, o[i][3] * i1);
    }
}

// Decode attention: CTA = (head, episode); the new token's K, V are written to
// the cache at `pos`, then softmax(q K^T) V over positions 0..pos.
__global__ void __launch_bounds__(256) attn_decode_kernel(const uint16_t* __restrict__ qkv, int pos, int d, int H,
                                                          uint16_t* __restrict__ kv, int layer, int L, int T,
                                                          uint16_t* __restrict__ out) {
    extern __shared__ __align__(16) uint8_t sm[];
    float* qsh = reinterpret_cast<float*>(sm);  // [HD]
    float* ps = qsh + HD;                        // [pos + 1]
    float* red = ps + (pos + 1);                 // [32]
    float* part = red + 32;                      // [4][HD]
    const int hh = blockIdx.x, e = blockIdx.y;
    const size_t rs = (size_t)3 * d;
    const uint16_t* row = qkv + (size_t)e * rs;
    uint16_t* Kc = kv + kv_off(e, layer, 0, 0, L, T, d) + hh * HD;
    uint16_t* Vc = kv + kv_off(e, layer, 1, 0, L, T, d) + hh * HD;
    const float scale = rsqrtf((float)HD);
    for (int c = threadIdx.x; c < HD; c += blockDim.x) {
        Kc[(size_t)pos * d + c] = row[d + hh * HD + c];
        Vc[(size_t)pos * d + c] = row[2 * d + hh * HD + c];
        qsh[c] = bf2f(row[hh * HD + c]) * scale;
    }
    __syncthreads();
    float mx = -INFINITY;
    for (int j = threadIdx.x; j <= pos; j += blockDim.x) {
        const uint16_t* kr = Kc + (size_t)j * d;
        float s = 0.f;
#pragma unroll 4
        for (int c = 0; c < HD; c += 8) {
            const uint4 k8 = *reinterpret_cast<const uint4*>(kr + c);
            const uint32_t kk[4] = {k8.x, k8.y, k8.z, k8.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                s = fmaf(qsh[c + 2 * u], __uint_as_float(kk[u] << 16), s);
                s = fmaf(qsh[c + 2 * u + 1], __uint_as_float(kk[u] & 0xffff0000u), s);
            }
        }
        ps[j] = s;
        mx = fmaxf(mx, s);
    }
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    mx = red[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) mx = fmaxf(mx, red[i]);
    __syncthreads();
    float sum = 0.f;
    for (int j = threadIdx.x; j <= pos; j += blockDim.x) {
        const float p = __expf(ps[j] - mx);
        ps[j] = p;
        sum += p;
    }
    sum = block_sum(sum, red);  // (contains the barrier that publishes ps)
    // o[c] over keys: thread = (dim pair, key quarter)
    const int c2 = (threadIdx.x & 63) * 2, qt = threadIdx.x >> 6;
    float o0 = 0.f, o1 = 0.f;
    for (int j = qt; j <= pos; j += 4) {
        const uint32_t v = *reinterpret_cast<const uint32_t*>(Vc + (size_t)j * d + c2);
        o0 = fmaf(ps[j], __uint_as_float(v << 16), o0);
        o1 = fmaf(ps[j], __uint_as_float(v & 0xffff0000u), o1);
    }
    part[qt * HD + c2] = o0;
    part[qt * HD + c2 + 1] = o1;
    __syncthreads();
    if (threadIdx.x < HD) {
        const float o = part[threadIdx.x] + part[HD + threadIdx.x] + part[2 * HD + threadIdx.x] +
                        part[3 * HD + threadIdx.x];
        out[(size_t)e * d + hh * HD + threadIdx.x] = f2bf(o / sum);
    }
}

// Decode attention, latency-optimised: CTA = (head, episode), 512 threads.
// Scores: one thread per key with the whole 256-B key row in flight (16
// independent 16-B loads) before the dot product; P V: thread = (8-dim chunk,
// key slice of 32), 16-B value loads, partial sums reduced through shared
// memory.  PDL-launched.
constexpr int ADT = 512;
// Quantization of the attention output for the o projection inside the
// attention kernel (policy step): ws = the o linear's decode activation area
// (null: off), rows 0 .. M-1 = episodes.
struct OQuant {
    uint8_t* ws;
    ActLayoutDec A;
    WLayout L;
    const int32_t* row_bits;
    int bits, M;
    int64_t* err;
};

// theta > 0: RoPE of this head's q and new k applied here (rope_pair, the
// rope_kernel arithmetic) instead of by a separate rope_kernel launch.
// oq.ws != null: the CTA then quantizes its head's output groups with
// aq_dec_job -- the o projection's act-quant kernel is not launched.
__global__ void __launch_bounds__(ADT) attn_decode2_kernel(const uint16_t* __restrict__ qkv, int pos, int d, int H,
                                                           uint16_t* __restrict__ kv, int layer, int L, int T,
                                                           uint16_t* __restrict__ out, float theta, OQuant oq) {
    extern __shared__ __align__(16) float smf[];
    float* qsh = smf;            // [HD]
    float* red = qsh + HD;       // [32]
    float* part = red + 32;      // [32 slices][HD]
    float* ps = part + 32 * HD;  // [pos + 1]
    ptx::pdl_wait();
    ptx::pdl_launch_dependents();
    const int hh = blockIdx.x, e = blockIdx.y;
    const size_t rs = (size_t)3 * d;
    const uint16_t* row = qkv + (size_t)e * rs;
    uint16_t* Kc = kv + kv_off(e, layer, 0, 0, L, T, d) + hh * HD;
    uint16_t* Vc = kv + kv_off(e, layer, 1, 0, L, T, d) + hh * HD;
    const float scale = rsqrtf((float)HD);
    const int tid = threadIdx.x;
    if (theta > 0.f) {
        if (tid < HD / 8)
            *reinterpret_cast<uint4*>(Vc + (size_t)pos * d + tid * 8) =
                *reinterpret_cast<const uint4*>(row + 2 * d + hh * HD + tid * 8);
        if (tid < HD) {  // threads [0, HD/2): q pairs, [HD/2, HD): k pairs
            const int i = tid & (HD / 2 - 1);
            const uint16_t* src = row + (tid < HD / 2 ? 0 : d) + hh * HD;
            uint16_t o1, o2;
            rope_pair(bf2f(src[i]), bf2f(src[i + HD / 2]), (float)pos, i, theta, o1, o2);
            if (tid < HD / 2) {
                qsh[i] = bf2f(o1) * scale;
                qsh[i + HD / 2] = bf2f(o2) * scale;
            } else {
                Kc[(size_t)pos * d + i] = o1;
                Kc[(size_t)pos * d + i + HD / 2] = o2;
            }
        }
    } else {
        if (tid < HD / 8) {
            *reinterpret_cast<uint4*>(Kc + (size_t)pos * d + tid * 8) =
                *reinterpret_cast<const uint4*>(row + d + hh * HD + tid * 8);
            *reinterpret_cast<uint4*>(Vc + (size_t)pos * d + tid * 8) =
                *reinterpret_cast<const uint4*>(row + 2 * d + hh * HD + tid * 8);
        }
        if (tid < HD) qsh[tid] = bf2f(row[hh * HD + tid]) * scale;
    }
    __syncthreads();
    float mx = -INFINITY;
    for (int j = tid; j <= pos; j += ADT) {
        const uint4* kr = reinterpret_cast<const uint4*>(Kc + (size_t)j * d);
        float s = 0.f;
#pragma unroll
        for (int hlf = 0; hlf < 2; ++hlf) {  // 8 x 16-B loads in flight, then 64 FMAs
            uint4 k8[HD / 16];
#pragma unroll
            for (int c = 0; c < HD / 16; ++c) k8[c] = kr[hlf * (HD / 16) + c];
#pragma unroll
            for (int c = 0; c < HD / 16; ++c) {
                const uint32_t kk[4] = {k8[c].x, k8[c].y, k8[c].z, k8[c].w};
                const int cb = (hlf * (HD / 16) + c) * 8;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    s = fmaf(qsh[cb + 2 * u], __uint_as_float(kk[u] << 16), s);
                    s = fmaf(qsh[cb + 2 * u + 1], __uint_as_float(kk[u] & 0xffff0000u), s);
                }
            }
        }
        ps[j] = s;
        mx = fmaxf(mx, s);
    }
    mx = warp_max(mx);
    if ((tid & 31) == 0) red[tid >> 5] = mx;
    __syncthreads();
    mx = red[0];
    for (int i = 1; i < ADT / 32; ++i) mx = fmaxf(mx, red[i]);
    __syncthreads();
    float sum = 0.f;
    for (int j = tid; j <= pos; j += ADT) {
        const float p = __expf(ps[j] - mx);
        ps[j] = p;
        sum += p;
    }
    sum = block_sum(sum, red);  // (contains the barrier that publishes ps)
    const int c8 = tid & 15, sl = tid >> 4;  // 16 chunks of 8 dims x 32 key slices
    float o[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    int j = sl;
    for (; j + 96 <= pos; j += 128) {  // 4 keys per iteration, loads first
        uint4 v4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v4[u] = *reinterpret_cast<const uint4*>(Vc + (size_t)(j + 32 * u) * d + c8 * 8);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float p = ps[j + 32 * u];
            const uint32_t vv[4] = {v4[u].x, v4[u].y, v4[u].z, v4[u].w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                o[2 * k] = fmaf(p, __uint_as_float(vv[k] << 16), o[2 * k]);
                o[2 * k + 1] = fmaf(p, __uint_as_float(vv[k] & 0xffff0000u), o[2 * k + 1]);
            }
        }
    }
    for (; j <= pos; j += 32) {
        const uint4 v = *reinterpret_cast<const uint4*>(Vc + (size_t)j * d + c8 * 8);
        const float p = ps[j];
        const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            o[2 * k] = fmaf(p, __uint_as_float(vv[k] << 16), o[2 * k]);
            o[2 * k + 1] = fmaf(p, __uint_as_float(vv[k] & 0xffff0000u), o[2 * k + 1]);
        }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) part[sl * HD + c8 * 8 + k] = o[k];
    __syncthreads();
    if (tid < HD) {
        float acc = 0.f;
#pragma unroll 8
        for (int q = 0; q < 32; ++q) acc += part[q * HD + tid];
        out[(size_t)e * d + hh * HD + tid] = f2bf(acc / sum);
    }
    if (oq.ws) {
        __syncthreads();  // this CTA's HD outputs of row e are written (CTA-visible)
        // (padding rows M .. 8 nt8 - 1 of the records are left as they are: the
        // decode kernel's token columns are independent, padding columns never stored)
        const int gph = HD / oq.L.G;
        const bool centred = dec_call_centred(oq.M, 0, oq.row_bits, oq.bits);
        for (int gi = tid >> 5; gi < gph; gi += ADT / 32)
            aq_dec_job(oq.L, out, oq.M, 0, oq.row_bits, oq.bits, oq.ws, oq.A, oq.err, 0, hh * gph + gi, e, centred);
    }
}

// Decode-pass form of add_rmsnorm8_kernel with the next linear's activation
// quantization in its epilogue.  CTA (row, slice): every CTA of a row reads
// the whole row of h_in (+ delta) and forms the row's sum of squares exactly
// as add_rmsnorm8_kernel does (same thread mapping, same reduction, so the
// same bits), then writes only its d/NS slice of h_out (= h_in + delta, or a
// copy) and y, and quantizes that slice's K-groups with aq_dec_job.  h_in is never written (the policy step
// alternates two h buffers), so no CTA reads a value another CTA updated.
__global__ void __launch_bounds__(1024) add_rmsnorm_q_kernel(const uint16_t* __restrict__ h_in,
                                                             const uint16_t* __restrict__ delta,
                                                             const uint16_t* __restrict__ w, int d, float eps,
                                                             uint16_t* __restrict__ y, uint16_t* __restrict__ h_out,
                                                             OQuant q) {
    __shared__ float red[32];
    ptx::pdl_wait();
    ptx::pdl_launch_dependents();
    const int row = blockIdx.x, slice = blockIdx.y, NS = gridDim.y;
    const int tps = (int)blockDim.x / NS;  // threads per slice
    const bool mine = (int)threadIdx.x / tps == slice;
    const size_t o = (size_t)row * d + threadIdx.x * 8;
    const uint4 hv = *reinterpret_cast<const uint4*>(h_in + o);
    const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w};
    float a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = bf2f((uint16_t)(hw[k >> 1] >> (16 * (k & 1))));
    uint32_t nh[4] = {hw[0], hw[1], hw[2], hw[3]};
    if (delta) {
        const uint4 dv = *reinterpret_cast<const uint4*>(delta + o);
        const uint32_t dw[4] = {dv.x, dv.y, dv.z, dv.w};
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
            const uint16_t lo = f2bf(a[k] + bf2f((uint16_t)(dw[k >> 1] & 0xffffu)));
            const uint16_t hi = f2bf(a[k + 1] + bf2f((uint16_t)(dw[k >> 1] >> 16)));
            a[k] = bf2f(lo);
            a[k + 1] = bf2f(hi);
            nh[k >> 1] = (uint32_t)lo | ((uint32_t)hi << 16);
        }
    }
    if (mine && h_out) *reinterpret_cast<uint4*>(h_out + o) = make_uint4(nh[0], nh[1], nh[2], nh[3]);
    float ss = 0.f;
#pragma unroll
    for (int k = 0; k < 8; k += 2) ss += a[k] * a[k] + a[k + 1] * a[k + 1];
    const float inv = rsqrtf(block_sum(ss, red) / (float)d + eps);
    if (mine) {
        const uint4 wv = *reinterpret_cast<const uint4*>(w + threadIdx.x * 8);
        const uint32_t ww[4] = {wv.x, wv.y, wv.z, wv.w};
        uint32_t yo[4];
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
            const uint16_t lo = f2bf(a[k] * inv * bf2f((uint16_t)(ww[k >> 1] & 0xffffu)));
            const uint16_t hi = f2bf(a[k + 1] * inv * bf2f((uint16_t)(ww[k >> 1] >> 16)));
            yo[k >> 1] = (uint32_t)lo | ((uint32_t)hi << 16);
        }
        *reinterpret_cast<uint4*>(y + o) = make_uint4(yo[0], yo[1], yo[2], yo[3]);
    }
    if (!q.ws) return;
    __syncthreads();  // this CTA's slice of y is written (CTA-visible)
    // (the padding rows M .. 8 nt8 - 1 of the records are left as they are:
    // the decode kernel's token columns are independent, padding columns are
    // never stored)
    const int G = q.L.G, gps = d / NS / G;
    const bool centred = dec_call_centred(q.M, 0, q.row_bits, q.bits);
    for (int gi = (int)threadIdx.x >> 5; gi < gps; gi += (int)blockDim.x >> 5)
        aq_dec_job(q.L, y, q.M, 0, q.row_bits, q.bits, q.ws, q.A, q.err, 0, slice * gps + gi, row, centred);
}

__global__ void silu_mul_kernel(const uint16_t* __restrict__ gu, int M, int ffn, uint16_t* __restrict__ act) {
    ptx::pdl_wait();
    ptx::pdl_launch_dependents();
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)M * ffn) return;
    const size_t m = idx / ffn, j = idx % ffn;
    const float g = bf2f(gu[m * 2 * ffn + j]), u = bf2f(gu[m * 2 * ffn + ffn + j]);
    act[idx] = f2bf(g / (1.f + __expf(-g)) * u);
}

// One CTA per episode: fp32 logits over the n_bins action-bin rows, argmax.
__global__ void head_argmax_kernel(const uint16_t* __restrict__ x, int row_stride, int d,
                                   const uint16_t* __restrict__ W, int n_bins, float* __restrict__ logits,
                                   int32_t* __restrict__ tok, int tok_stride) {
    ptx::pdl_wait();
    ptx::pdl_launch_dependents();
    extern __shared__ __align__(16) float xs[];  // [d]
    __shared__ float bv[32];
    __shared__ int bi[32];
    const int e = blockIdx.x;
    const uint16_t* xr = x + (size_t)e * row_stride * d;
    for (int i = threadIdx.x; i < d; i += blockDim.x) xs[i] = bf2f(xr[i]);
    __syncthreads();
    float best = -INFINITY;
    int bidx = 0x7fffffff;
    for (int b = threadIdx.x; b < n_bins; b += blockDim.x) {
        const uint16_t* wr = W + (size_t)b * d;
        float s = 0.f;
        for (int i = 0; i < d; i += 8) {
            const uint4 w8 = *reinterpret_cast<const uint4*>(wr + i);
            const uint32_t ww[4] = {w8.x, w8.y, w8.z, w8.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                s = fmaf(xs[i + 2 * u], __uint_as_float(ww[u] << 16), s);
                s = fmaf(xs[i + 2 * u + 1], __uint_as_float(ww[u] & 0xffff0000u), s);
            }
        }
        if (logits) logits[(size_t)e * n_bins + b] = s;
        if (s > best || (s == best && b < bidx)) { best = s; bidx = b; }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const float ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
        if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; }
    }
    if ((threadIdx.x & 31) == 0) { bv[threadIdx.x >> 5] = best; bi[threadIdx.x >> 5] = bidx; }
    __syncthreads();
    if (threadIdx.x == 0) {
        best = bv[0];
        bidx = bi[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            if (bv[w] > best || (bv[w] == best && bi[w] < bidx)) { best = bv[w]; bidx = bi[w]; }
        tok[(size_t)e * tok_stride] = bidx;
    }
}

// h rows of the prefill sequence: vision embeddings, then text-token embeddings
__global__ void embed_prefill_kernel(const uint16_t* __restrict__ vis, const int32_t* __restrict__ text,
                                     const uint16_t* __restrict__ embed, int n_vis, int n_text, int d,
                                     uint16_t* __restrict__ h, int src_E) {
    ptx::pdl_wait();
    ptx::pdl_launch_dependents();
    const int S = n_vis + n_text;
    const int row = blockIdx.x;  // e * S + i
    const int e = (row / S) % src_E, i = row % S;  // replicas e, e + src_E, ... share an observation
    const uint16_t* src = i < n_vis ? vis + ((size_t)e * n_vis + i) * d
                                    : embed + (size_t)text[(size_t)e * n_text + (i - n_vis)] * d;
    for (int c = threadIdx.x * 8; c < d; c += blockDim.x * 8)
        *reinterpret_cast<uint4*>(h + (size_t)row * d + c) = *reinterpret_cast<const uint4*>(src + c);
}

// Action head, spread over many CTAs: CTA (e, bin block) computes 32 bins'
// logits with one warp per bin (coalesced 16-B loads of W rows, warp-shuffle
// sums); the argmax over the logits row is a second tiny kernel (lowest index
// among equal maxima, as head_argmax_kernel).
constexpr int HB = 32;  // bins per CTA
__global__ void __launch_bounds__(256) head_logits_kernel(const uint16_t* __restrict__ x, int row_stride, int d,
                                                          const uint16_t* __restrict__ W, int n_bins,
                                                          float* __restrict__ logits) {
    extern __shared__ __align__(16) float xsh[];  // [d]
    ptx::pdl_wait();
    ptx::pdl_launch_dependents();
    const int e = blockIdx.x, b0 = blockIdx.y * HB;
    const uint16_t* xr = x + (size_t)e * row_stride * d;
    for (int i = threadIdx.x * 8; i < d; i += blockDim.x * 8) {
        const uint4 v = *reinterpret_cast<const uint4*>(xr + i);
        const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            xsh[i + 2 * u] = __uint_as_float(vv[u] << 16);
            xsh[i + 2 * u + 1] = __uint_as_float(vv[u] & 0xffff0000u);
        }
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int bb = warp; bb < HB; bb += 8) {
        const int b = b0 + bb;
        if (b >= n_bins) break;
        const uint16_t* wr = W + (size_t)b * d;
        float s = 0.f;
        for (int i = lane * 8; i < d; i += 256) {
            const uint4 w8 = *reinterpret_cast<const uint4*>(wr + i);
            const float4 xa = *reinterpret_cast<const float4*>(xsh + i);
            const float4 xb = *reinterpret_cast<const float4*>(xsh + i + 4);
            s = fmaf(xa.x, __uint_as_float(w8.x << 16), s);
            s = fmaf(xa.y, __uint_as_float(w8.x & 0xffff0000u), s);
            s = fmaf(xa.z, __uint_as_float(w8.y << 16), s);
            s = fmaf(xa.w, __uint_as_float(w8.y & 0xffff0000u), s);
            s = fmaf(xb.x, __uint_as_float(w8.z << 16), s);
            s = fmaf(xb.y, __uint_as_float(w8.z & 0xffff0000u), s);
            s = fmaf(xb.z, __uint_as_float(w8.w << 16), s);
            s = fmaf(xb.w, __uint_as_float(w8.w & 0xffff0000u), s);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) logits[(size_t)e * n_bins + b] = s;
    }
}
__global__ void __launch_bounds__(256) argmax_rows_kernel(const float* __restrict__ logits, int n_bins,
                                                          int32_t* __restrict__ tok, int tok_stride) {
    __shared__ float bv[32];
    __shared__ int bi[32];
    ptx::pdl_wait();
    ptx::pdl_launch_dependents();
    const int e = blockIdx.x;
    float best = -INFINITY;
    int bidx = 0x7fffffff;
    for (int b = threadIdx.x; b < n_bins; b += blockDim.x) {
        const float s = logits[(size_t)e * n_bins + b];
        if (s > best || (s == best && b < bidx)) { best = s; bidx = b; }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const float ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
        if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; }
    }
    if ((threadIdx.x & 31) == 0) { bv[threadIdx.x >> 5] = best; bi[threadIdx.x >> 5] = bidx; }
    __syncthreads();
    if (threadIdx.x == 0) {
        best = bv[0];
        bidx = bi[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            if (bv[w] > best || (bv[w] == best && bi[w] < bidx)) { best = bv[w]; bidx = bi[w]; }
        tok[(size_t)e * tok_stride] = bidx;
    }
}

// decode input: embedding of the previous action token (vocab id vocab - n_bins + bin)
__global__ void embed_action_kernel(const int32_t* __restrict__ tok, int n_act, int t, const uint16_t* __restrict__ embed,
                                    int vocab, int n_bins, int d, uint16_t* __restrict__ h) {
    ptx::pdl_wait();
    ptx::pdl_launch_dependents();
    const int e = blockIdx.x;
    const int id = vocab - n_bins + tok[(size_t)e * n_act + t];
    for (int c = threadIdx.x * 8; c < d; c += blockDim.x * 8)
        *reinterpret_cast<uint4*>(h + (size_t)e * d + c) = *reinterpret_cast<const uint4*>(embed + (size_t)id * d + c);
}

__global__ void detok_kernel(const int32_t* __restrict__ tok, int E, int n_act, int n_bins, float* __restrict__ act,
                             float* __restrict__ prev, const int32_t* __restrict__ bits, int32_t* __restrict__ bits_out) {
    ptx::pdl_wait();
    ptx::pdl_launch_dependents();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < E * n_act) {
        const float v = -1.f + (2.f * (float)tok[i] + 1.f) / (float)n_bins;
        act[i] = v;
        // the kinematic proxies read a_{t-1} as [E, 7] (x,y,z, rx,ry,rz, grip)
        const int e = i / n_act, k = i % n_act;
        if (k < 7) prev[e * 7 + k] = v;
    }
    if (bits_out && i < E) bits_out[i] = bits[i];
}

// Variant-table routing (dyq_model_desc_t wbits_of / abits_of): per row of
// episode e = r / tpe, b*_e -> (weight copy, activation bits); rows of the
// other copy get 0 (masked), and gates[c] = 1 iff copy c (0: W4, 1: W8) has a
// live row.  One CTA.
__global__ void variant_route_kernel(const int32_t* __restrict__ bits, int E, int tpe, int4 wtab, int4 atab,
                                     int32_t* __restrict__ rb4, int32_t* __restrict__ rb8, int32_t* __restrict__ gates) {
    ptx::pdl_wait();
    ptx::pdl_launch_dependents();
    __shared__ int any4, any8;
    if (threadIdx.x == 0) any4 = any8 = 0;
    __syncthreads();
    const int wt[4] = {wtab.x, wtab.y, wtab.z, wtab.w}, at[4] = {atab.x, atab.y, atab.z, atab.w};
    int a4 = 0, a8 = 0;
    for (int r = threadIdx.x; r < E * tpe; r += blockDim.x) {
        const int b = bits[r / tpe];
        const int i = b == 2 ? 0 : b == 4 ? 1 : b == 8 ? 2 : 3;
        const bool w8 = wt[i] == 8;
        rb4[r] = w8 ? 0 : at[i];
        rb8[r] = w8 ? at[i] : 0;
        a4 |= !w8;
        a8 |= w8;
    }
    if (a4) any4 = 1;
    if (a8) any8 = 1;
    __syncthreads();
    if (threadIdx.x == 0) {
        gates[0] = any4;
        gates[1] = any8;
    }
}

__global__ void fill_i32_kernel(int32_t* __restrict__ p, int n, int v) {
    ptx::pdl_wait();
    ptx::pdl_launch_dependents();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = v;
}

// ------------------------------------------------------------------ host
static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

struct ModelLayout {
    int S, T, MP;
    size_t h, h2, xn, delta, att, qkv, gu, act, ws[8], rbp, rbd, bits, tok, prev, logits, err, total;
    size_t rb8p, rb8d, gates;      // variant table: W8 rows (prefill / decode), gates [W4p, W8p, W4d, W8d]
    size_t ws_bytes[8], kv_bytes;  // one qlinear workspace per linear shape (split-K counters are per shape); 4-7: W8
    bool w8;
};

static dyq_wdesc_t wdesc_of(const dyq_model_desc_t& m, int which) {
    dyq_wdesc_t w{};
    w.group = m.group;
    w.wbits = which >= 4 ? 8 : m.wbits;
    which &= 3;
    w.round_mode = 0;
    switch (which) {
        case 0: w.N = 3 * m.d; w.K = m.d; break;
        case 1: w.N = m.d; w.K = m.d; break;
        case 2: w.N = 2 * m.ffn; w.K = m.d; break;
        default: w.N = m.d; w.K = m.ffn; break;
    }
    return w;
}

static dyq_status_t model_layout(const dyq_model_desc_t* m, ModelLayout* L) {
    if (!m) return set_error(DYQ_EINVAL, "null model descriptor");
    if (m->n_layers <= 0 || m->d <= 0 || m->ffn <= 0 || m->n_heads <= 0 || m->E <= 0 || m->vocab <= 0)
        return set_error(DYQ_EINVAL, "model dimensions must be positive");
    if (m->d != m->n_heads * HD) return set_error(DYQ_EUNSUPPORTED, "head dim must be %d (d = n_heads * %d)", HD, HD);
    if (m->d % 16 || m->ffn % 16) return set_error(DYQ_ESHAPE, "d and ffn must be multiples of 16");
    if (m->n_vis < 0 || m->n_text < 1 || m->n_act < 1 || m->n_act > 7 + 64 || m->n_bins < 1 || m->n_bins > m->vocab)
        return set_error(DYQ_EINVAL, "bad token counts");
    if (m->n_act < 7) return set_error(DYQ_EINVAL, "n_act must be >= 7 (the kinematic proxies read a 7-dof action)");
    L->S = m->n_vis + m->n_text;
    L->T = L->S + m->n_act;
    L->MP = m->E * L->S;
    if (L->MP > 65536) return set_error(DYQ_ESHAPE, "E * (n_vis + n_text) must be <= 65536");
    const size_t MP = L->MP, d = m->d, ffn = m->ffn;
    L->w8 = m->codes_w8 != nullptr;
    if (L->w8 && (!m->meta_w8 || m->wbits != 4)) return set_error(DYQ_EINVAL, "W8 table needs meta_w8 and W4 codes");
    for (int i = 0; i < 4; ++i) {
        if (m->wbits_of[i] != 0 && m->wbits_of[i] != 4 && m->wbits_of[i] != 8)
            return set_error(DYQ_EINVAL, "wbits_of[%d] must be 4 or 8", i);
        if (m->wbits_of[i] == 8 && !L->w8) return set_error(DYQ_EINVAL, "wbits_of[%d] = 8 without W8 copies", i);
        const int a = m->abits_of[i];
        if (a != 0 && a != 2 && a != 4 && a != 8 && a != 16) return set_error(DYQ_EINVAL, "abits_of[%d] = %d", i, a);
    }
    if (m->prefill_bits != 0 && m->prefill_bits != 2 && m->prefill_bits != 4 && m->prefill_bits != 8 &&
        m->prefill_bits != 16)
        return set_error(DYQ_EINVAL, "prefill_bits must be 0, 2, 4, 8 or 16");
    const int nshapes = L->w8 ? 8 : 4;
    for (int which = 4; which < 8; ++which) L->ws_bytes[which] = 0;
    for (int which = 0; which < nshapes; ++which) {
        const dyq_wdesc_t w = wdesc_of(*m, which);
        // a step may run any e <= desc.E episodes (prefill M = e * S, decode
        // M = e) and the prefill split factor is not monotone in M, so the
        // workspace is the maximum over every M the step can issue
        size_t wsb = 0;
        for (int e = 1; e <= m->E; ++e)
            for (int M : {e * L->S, e}) {
                size_t b = 0;
                dyq_status_t rc = dyq_qlinear_workspace(&w, M, &b);
                if (rc) return rc;
                wsb = b > wsb ? b : wsb;
            }
        L->ws_bytes[which] = wsb;
    }
    size_t o = 0;
    auto take = [&](size_t bytes) { const size_t r = o; o += al256(bytes); return r; };
    L->h = take(MP * d * 2);
    L->h2 = take(MP * d * 2);  // the decode passes' second h buffer (add_rmsnorm_q ping-pong)
    L->xn = take(MP * d * 2);
    L->delta = take(MP * d * 2);
    L->att = take(MP * d * 2);
    L->qkv = take(MP * 3 * d * 2);
    L->gu = take(MP * 2 * ffn * 2);
    L->act = take(MP * ffn * 2);
    for (int which = 0; which < 8; ++which) L->ws[which] = take(L->ws_bytes[which]);
    L->rbp = take(MP * 4);
    L->rbd = take((size_t)m->E * 4);
    L->rb8p = take(MP * 4);
    L->rb8d = take((size_t)m->E * 4);
    L->gates = take(16);
    L->bits = take((size_t)m->E * 4);
    L->tok = take((size_t)m->E * m->n_act * 4);
    L->prev = take((size_t)m->E * 7 * 4);
    L->logits = take((size_t)m->E * m->n_bins * 4);
    L->err = take(8);
    L->total = o;
    L->kv_bytes = (size_t)m->E * m->n_layers * 2 * L->T * d * 2;
    return DYQ_OK;
}

struct Model {
    dyq_model_desc_t d;
    std::vector<const void*> codes, meta, codes8, meta8;
    cudaStream_t side = nullptr;  // paper mode: the selector's stream
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    ModelLayout L;
    int t = 0;
    uint8_t* sb() const { return reinterpret_cast<uint8_t*>(d.scratch); }
    template <class T>
    T* at(size_t off) const { return reinterpret_cast<T*>(sb() + off); }
};

}  // namespace dyq

using namespace dyq;

extern "C" {

dyq_status_t dyq_add_rmsnorm(uint16_t* h, const uint16_t* delta, const uint16_t* w, int32_t M, int32_t d, float eps,
                             uint16_t* y, dyq_stream_t stream) {
    if (M < 0 || d <= 0 || d % 2) return set_error(DYQ_ESHAPE, "bad rmsnorm shape");
    if (M == 0) return DYQ_OK;
    if (!h || !w || !y) return set_error(DYQ_EINVAL, "null pointer");
    const bool al = ((uintptr_t)h | (uintptr_t)w | (uintptr_t)y | (uintptr_t)delta) % 16 == 0;
    if (d % 256 == 0 && d / 8 <= 1024 && al) {
        const cudaError_t e = launch_pdl(add_rmsnorm8_kernel, dim3(M), dim3(d / 8), 0, (cudaStream_t)stream, h, delta,
                                         w, d, eps, y, PQuant{});
        if (e != cudaSuccess) return set_error(DYQ_ECUDA, "add_rmsnorm8_kernel: %s", cudaGetErrorString(e));
        return check_launch("add_rmsnorm8_kernel");
    }
    add_rmsnorm_kernel<<<M, 256, 0, (cudaStream_t)stream>>>(h, delta, w, d, eps, y);
    return check_launch("add_rmsnorm_kernel");
}

dyq_status_t dyq_rope(uint16_t* qkv, int32_t M, int32_t S, int32_t pos0, int32_t d, int32_t H, float theta,
                      dyq_stream_t stream) {
    if (M < 0 || S <= 0 || d != H * HD) return set_error(DYQ_ESHAPE, "bad rope shape (head dim %d)", HD);
    if (M == 0) return DYQ_OK;
    const size_t n = (size_t)M * 2 * H * (HD / 2);
    const cudaError_t e = launch_pdl(rope_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0,
                                     (cudaStream_t)stream, qkv, M, S, pos0, d, H, theta);
    if (e != cudaSuccess) return set_error(DYQ_ECUDA, "rope_kernel: %s", cudaGetErrorString(e));
    return check_launch("rope_kernel");
}

dyq_status_t dyq_attention_prefill(const uint16_t* qkv, int32_t E, int32_t S, int32_t d, int32_t H, uint16_t* kv,
                                   int32_t layer, int32_t L, int32_t T, uint16_t* out, dyq_stream_t stream) {
    if (E <= 0 || S <= 0 || S > T || d != H * HD || layer < 0 || layer >= L)
        return set_error(DYQ_ESHAPE, "bad attention shape");
    if (d % 8 == 0 && ((uintptr_t)qkv | (uintptr_t)kv | (uintptr_t)out) % 16 == 0) {
        const size_t smem_tc = (size_t)(FQ + 2 * FK) * FST * 2;
        static bool attr_tc = false;
        if (!attr_tc) {
            cudaFuncSetAttribute(attn_prefill_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_tc);
            attr_tc = true;
        }
        const cudaError_t e = launch_pdl(attn_prefill_tc_kernel, dim3((S + FQ - 1) / FQ, H, E), dim3(128), smem_tc,
                                         (cudaStream_t)stream, qkv, S, d, H, kv, layer, L, T, out);
        if (e != cudaSuccess) return set_error(DYQ_ECUDA, "attn_prefill_tc_kernel: %s", cudaGetErrorString(e));
        return check_launch("attn_prefill_tc_kernel");
    }
    const size_t smem = attn_ks_bytes(S) + (size_t)S * HD * 2 + 8 * HD * 4 + (size_t)8 * S * 4;
    if (smem > 227 * 1024) return set_error(DYQ_EUNSUPPORTED, "attention prefill: S = %d too long", S);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(attn_prefill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr = true;
    }
    const dim3 grid((S + AQB - 1) / AQB, H, E);
    attn_prefill_kernel<<<grid, 256, smem, (cudaStream_t)stream>>>(qkv, S, d, H, kv, layer, L, T, out);
    return check_launch("attn_prefill_kernel");
}

}  // extern "C"

namespace dyq {
// Decode attention; theta > 0 also applies RoPE to the step's q and new k
// (the policy step's fused path).  The fused form needs the aligned kernel:
// on a misaligned buffer the caller falls back to dyq_rope + the generic
// kernel (returns DYQ_EUNSUPPORTED without launching).
static dyq_status_t attention_decode(const uint16_t* qkv, int32_t E, int32_t pos, int32_t d, int32_t H, uint16_t* kv,
                                     int32_t layer, int32_t L, int32_t T, uint16_t* out, float theta,
                                     cudaStream_t stream, const OQuant& oq = OQuant{}) {
    if (E <= 0 || pos < 0 || pos >= T || d != H * HD || layer < 0 || layer >= L)
        return set_error(DYQ_ESHAPE, "bad attention shape");
    if (d % 8 == 0 && ((uintptr_t)qkv | (uintptr_t)kv) % 16 == 0) {
        const size_t smem2 = (HD + 32 + 32 * HD + (size_t)(pos + 1)) * 4;
        if (smem2 > 48 * 1024) {
            static bool attr = false;
            if (!attr) {
                cudaFuncSetAttribute(attn_decode2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
                attr = true;
            }
        }
        const cudaError_t e = launch_pdl(attn_decode2_kernel, dim3(H, E), dim3(ADT), smem2, stream, qkv, pos, d, H, kv,
                                         layer, L, T, out, theta, oq);
        if (e != cudaSuccess) return set_error(DYQ_ECUDA, "attn_decode2_kernel: %s", cudaGetErrorString(e));
        return check_launch("attn_decode2_kernel");
    }
    if (theta > 0.f || oq.ws) return DYQ_EUNSUPPORTED;
    const size_t smem = (HD + (size_t)(pos + 1) + 32 + 4 * HD) * 4;
    attn_decode_kernel<<<dim3(H, E), 256, smem, stream>>>(qkv, pos, d, H, kv, layer, L, T, out);
    return check_launch("attn_decode_kernel");
}

// add_rmsnorm_q_kernel launcher: DYQ_EUNSUPPORTED (nothing launched) when the
// shape does not split into 256-wide slices of whole K-groups.
static dyq_status_t add_rmsnorm_q(const uint16_t* h_in, const uint16_t* delta, const uint16_t* w, int M, int d,
                                  float eps, uint16_t* y, uint16_t* h_out, const OQuant& q, cudaStream_t st) {
    if (M <= 0 || d % 256 || d / 8 > 1024 || (q.ws && (256 % q.L.G || q.L.K != d))) return DYQ_EUNSUPPORTED;
    if (((uintptr_t)h_in | (uintptr_t)delta | (uintptr_t)w | (uintptr_t)y | (uintptr_t)h_out) % 16)
        return DYQ_EUNSUPPORTED;
    const cudaError_t e = launch_pdl(add_rmsnorm_q_kernel, dim3(M, d / 256), dim3(d / 8), 0, st, h_in, delta, w, d,
                                     eps, y, h_out, q);
    if (e != cudaSuccess) return set_error(DYQ_ECUDA, "add_rmsnorm_q_kernel: %s", cudaGetErrorString(e));
    return check_launch("add_rmsnorm_q_kernel");
}

// add_rmsnorm8_kernel with the next linear's prefill records in its epilogue;
// DYQ_EUNSUPPORTED (nothing launched) when a row's K-groups are not whole
// warps of quarter jobs or the shape / alignment does not fit the kernel.
static dyq_status_t add_rmsnorm_pq(uint16_t* h, const uint16_t* delta, const uint16_t* w, int M, int d, float eps,
                                   uint16_t* y, const PQuant& pq, cudaStream_t st) {
    const int jobs = pq.L.NG * AQP_TPR;
    if (M <= 0 || d % 256 || d / 8 > 1024 || pq.L.K != d || (pq.L.G != 64 && pq.L.G != 128) || jobs > d / 8 ||
        jobs % 32)
        return DYQ_EUNSUPPORTED;
    if (((uintptr_t)h | (uintptr_t)delta | (uintptr_t)w | (uintptr_t)y) % 16) return DYQ_EUNSUPPORTED;
    const cudaError_t e = launch_pdl(add_rmsnorm8_kernel, dim3(M), dim3(d / 8), 0, st, h, delta, w, d, eps, y, pq);
    if (e != cudaSuccess) return set_error(DYQ_ECUDA, "add_rmsnorm8_kernel: %s", cudaGetErrorString(e));
    return check_launch("add_rmsnorm8_kernel");
}
}  // namespace dyq

extern "C" {
dyq_status_t dyq_attention_decode(const uint16_t* qkv, int32_t E, int32_t pos, int32_t d, int32_t H, uint16_t* kv,
                                  int32_t layer, int32_t L, int32_t T, uint16_t* out, dyq_stream_t stream) {
    return attention_decode(qkv, E, pos, d, H, kv, layer, L, T, out, 0.f, (cudaStream_t)stream);
}

dyq_status_t dyq_attention_decode_rope(const uint16_t* qkv, int32_t E, int32_t pos, int32_t d, int32_t H, float theta,
                                       uint16_t* kv, int32_t layer, int32_t L, int32_t T, uint16_t* out,
                                       dyq_stream_t stream) {
    if (!(theta > 0.f)) return set_error(DYQ_EINVAL, "rope theta must be positive");
    const dyq_status_t rc = attention_decode(qkv, E, pos, d, H, kv, layer, L, T, out, theta, (cudaStream_t)stream);
    if (rc == DYQ_EUNSUPPORTED) return set_error(DYQ_EUNSUPPORTED, "fused rope + attention needs 16-B aligned qkv / kv");
    return rc;
}

dyq_status_t dyq_silu_mul(const uint16_t* gu, int32_t M, int32_t ffn, uint16_t* act, dyq_stream_t stream) {
    if (M < 0 || ffn <= 0) return set_error(DYQ_ESHAPE, "bad silu_mul shape");
    if (M == 0) return DYQ_OK;
    const size_t n = (size_t)M * ffn;
    const cudaError_t e = launch_pdl(silu_mul_kernel, dim3((unsigned)((n + 255) / 256)), dim3(256), 0,
                                     (cudaStream_t)stream, gu, M, ffn, act);
    if (e != cudaSuccess) return set_error(DYQ_ECUDA, "silu_mul_kernel: %s", cudaGetErrorString(e));
    return check_launch("silu_mul_kernel");
}

dyq_status_t dyq_head_argmax(const uint16_t* x, int32_t E, int32_t row_stride, int32_t d, const uint16_t* W,
                             int32_t n_bins, float* logits, int32_t* tok, int32_t tok_stride, dyq_stream_t stream) {
    if (E <= 0 || d <= 0 || d % 8 || n_bins <= 0) return set_error(DYQ_ESHAPE, "bad head shape");
    if (logits && d % 256 == 0 && ((uintptr_t)x | (uintptr_t)W) % 16 == 0 && (size_t)d * 4 <= 48 * 1024) {
        cudaError_t e = launch_pdl(head_logits_kernel, dim3(E, (n_bins + HB - 1) / HB), dim3(256), (size_t)d * 4,
                                   (cudaStream_t)stream, x, row_stride, d, W, n_bins, logits);
        if (e == cudaSuccess)
            e = launch_pdl(argmax_rows_kernel, dim3(E), dim3(256), 0, (cudaStream_t)stream, (const float*)logits, n_bins,
                           tok, tok_stride);
        if (e != cudaSuccess) return set_error(DYQ_ECUDA, "head_logits/argmax: %s", cudaGetErrorString(e));
        return check_launch("head_logits_kernel");
    }
    const cudaError_t e = launch_pdl(head_argmax_kernel, dim3(E), dim3(256), (size_t)d * 4, (cudaStream_t)stream, x,
                                     row_stride, d, W, n_bins, logits, tok, tok_stride);
    if (e != cudaSuccess) return set_error(DYQ_ECUDA, "head_argmax_kernel: %s", cudaGetErrorString(e));
    return check_launch("head_argmax_kernel");
}

dyq_status_t dyq_model_size(const dyq_model_desc_t* desc, size_t* kv_bytes, size_t* scratch_bytes) {
    ModelLayout L;
    dyq_status_t rc = model_layout(desc, &L);
    if (rc) return rc;
    if (kv_bytes) *kv_bytes = L.kv_bytes;
    if (scratch_bytes) *scratch_bytes = L.total;
    return DYQ_OK;
}

dyq_status_t dyq_model_bind(const dyq_model_desc_t* desc, void** model) {
    if (!model) return set_error(DYQ_EINVAL, "null output handle");
    ModelLayout L;
    dyq_status_t rc = model_layout(desc, &L);
    if (rc) return rc;
    if (!desc->codes || !desc->meta || !desc->attn_norm || !desc->mlp_norm || !desc->final_norm || !desc->embed ||
        !desc->head_bins || !desc->kv || !desc->scratch)
        return set_error(DYQ_EINVAL, "null pointer in model descriptor");
    Model* m = new Model();
    m->d = *desc;
    m->codes.assign(desc->codes, desc->codes + 4 * desc->n_layers);
    m->meta.assign(desc->meta, desc->meta + 4 * desc->n_layers);
    for (int i = 0; i < 4 * desc->n_layers; ++i)
        if (!m->codes[i] || !m->meta[i]) {
            delete m;
            return set_error(DYQ_EINVAL, "null packed-weight pointer for linear %d", i);
        }
    if (L.w8) {
        m->codes8.assign(desc->codes_w8, desc->codes_w8 + 4 * desc->n_layers);
        m->meta8.assign(desc->meta_w8, desc->meta_w8 + 4 * desc->n_layers);
        for (int i = 0; i < 4 * desc->n_layers; ++i)
            if (!m->codes8[i] || !m->meta8[i]) {
                delete m;
                return set_error(DYQ_EINVAL, "null W8 packed-weight pointer for linear %d", i);
            }
    }
    if (desc->paper_mode &&
        (cudaStreamCreateWithFlags(&m->side, cudaStreamNonBlocking) != cudaSuccess ||
         cudaEventCreateWithFlags(&m->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
         cudaEventCreateWithFlags(&m->ev_join, cudaEventDisableTiming) != cudaSuccess)) {
        delete m;
        return check_launch("dyq_model_bind (paper-mode stream)");
    }
    m->d.codes = nullptr;
    m->d.meta = nullptr;
    m->d.codes_w8 = nullptr;
    m->d.meta_w8 = nullptr;
    m->L = L;
    *model = m;
    return DYQ_OK;
}

dyq_status_t dyq_model_init(void* model, dyq_stream_t stream) {
    Model* m = reinterpret_cast<Model*>(model);
    if (!m) return set_error(DYQ_EINVAL, "null model");
    m->t = 0;
    if (cudaMemsetAsync(m->d.scratch, 0, m->L.total, (cudaStream_t)stream) != cudaSuccess)
        return check_launch("dyq_model_init");
    return DYQ_OK;
}

dyq_status_t dyq_model_free(void* model) {
    Model* m = reinterpret_cast<Model*>(model);
    if (m && m->side) {
        cudaStreamDestroy(m->side);
        cudaEventDestroy(m->ev_fork);
        cudaEventDestroy(m->ev_join);
    }
    delete m;
    return DYQ_OK;
}

// One control step.  forced == nullptr: b*_t from the selection state (the
// product path); else per-episode bits forced[E] (device) and no selection.
// Episode e reads observation e % src_E (calibration replicas).
static dyq_status_t policy_step_impl(void* model, void* state, const int32_t* forced, int32_t src_E, int32_t E,
                                     const uint16_t* vis, const int32_t* text, float* action_out, int32_t* bits_out,
                                     dyq_stream_t stream) {
    Model* m = reinterpret_cast<Model*>(model);
    if (!m || (!state && !forced) || !vis || !text || !action_out) return set_error(DYQ_EINVAL, "null pointer");
    const dyq_model_desc_t& D = m->d;
    const ModelLayout& L = m->L;
    if (E <= 0 || E > D.E) return set_error(DYQ_EINVAL, "E = %d outside [1, %d]", E, D.E);
    const int S = L.S, d = D.d, H = D.n_heads, NL = D.n_layers;
    const int MP = E * S;
    uint16_t* h = m->at<uint16_t>(L.h);
    uint16_t* xn = m->at<uint16_t>(L.xn);
    uint16_t* delta = m->at<uint16_t>(L.delta);
    uint16_t* att = m->at<uint16_t>(L.att);
    uint16_t* qkv = m->at<uint16_t>(L.qkv);
    uint16_t* gu = m->at<uint16_t>(L.gu);
    uint16_t* act = m->at<uint16_t>(L.act);
    void* ws[4];
    for (int i = 0; i < 4; ++i) ws[i] = m->at<uint8_t>(L.ws[i]);
    int32_t* rbp = m->at<int32_t>(L.rbp);
    int32_t* rbd = m->at<int32_t>(L.rbd);
    int32_t* bits = m->at<int32_t>(L.bits);
    int32_t* tok = m->at<int32_t>(L.tok);
    float* prev = m->at<float>(L.prev);
    float* logits = m->at<float>(L.logits);
    int64_t* err = m->at<int64_t>(L.err);
    uint16_t* kv = reinterpret_cast<uint16_t*>(D.kv);
    const cudaStream_t st = (cudaStream_t)stream;
    dyq_status_t rc;
#define DYQ_TRY(x)        \
    do {                  \
        rc = (x);         \
        if (rc) return rc; \
    } while (0)
    dyq_wdesc_t wd[8];
    for (int i = 0; i < 8; ++i) wd[i] = wdesc_of(D, i);
    void* ws8[4];
    for (int i = 0; i < 4; ++i) ws8[i] = m->at<uint8_t>(L.ws[4 + i]);
    int32_t* rb8p = m->at<int32_t>(L.rb8p);
    int32_t* rb8d = m->at<int32_t>(L.rb8d);
    int32_t* gates = m->at<int32_t>(L.gates);  // [W4 prefill, W8 prefill, W4 decode, W8 decode]
    const bool w8 = L.w8 && !forced;           // forced-bits steps (calibration) stay on the W4 table
    const char* fo = getenv("DYQ_FUSE_OQ");     // 0: the o projection's separate act-quant kernel (A/B, tests)
    const bool fuse_oq = !(fo && atoi(fo) == 0);
    const bool paper = D.paper_mode && !forced && m->side;
    const int pre_bits = D.prefill_bits ? D.prefill_bits : 16;
    int4 wtab = make_int4(4, 4, 4, 4), atab = make_int4(2, 4, 8, 16);
    if (D.wbits_of[0] | D.wbits_of[1] | D.wbits_of[2] | D.wbits_of[3])
        wtab = make_int4(D.wbits_of[0] ? D.wbits_of[0] : 4, D.wbits_of[1] ? D.wbits_of[1] : 4,
                         D.wbits_of[2] ? D.wbits_of[2] : 4, D.wbits_of[3] ? D.wbits_of[3] : 4);
    const bool atab_set = D.abits_of[0] | D.abits_of[1] | D.abits_of[2] | D.abits_of[3];
    if (atab_set)
        atab = make_int4(D.abits_of[0] ? D.abits_of[0] : 2, D.abits_of[1] ? D.abits_of[1] : 4,
                         D.abits_of[2] ? D.abits_of[2] : 8, D.abits_of[3] ? D.abits_of[3] : 16);
    const int32_t atab_h[4] = {atab.x, atab.y, atab.z, atab.w};

    // b*_t from a_{t-1}, then per-row activation bits (variant table)
    auto select = [&](cudaStream_t s_sel, bool prefill_rows) -> dyq_status_t {
        const dyq_stream_t ss = (dyq_stream_t)s_sel;
        if (w8) {
            DYQ_TRY(dyq_select_bits(state, E, m->t == 0 ? nullptr : prev, bits, nullptr, nullptr, ss));
            if (prefill_rows &&
                launch_pdl(variant_route_kernel, dim3(1), dim3(256), 0, s_sel, (const int32_t*)bits, E, S, wtab, atab,
                           rbp, rb8p, gates) != cudaSuccess)
                return set_error(DYQ_ECUDA, "variant_route_kernel launch");
            if (launch_pdl(variant_route_kernel, dim3(1), dim3(32), 0, s_sel, (const int32_t*)bits, E, 1, wtab, atab,
                           rbd, rb8d, gates + 2) != cudaSuccess)
                return set_error(DYQ_ECUDA, "variant_route_kernel launch");
            return check_launch("variant_route_kernel");
        }
        if (prefill_rows)
            DYQ_TRY(dyq_select_route(state, E, m->t == 0 ? nullptr : prev, bits, S, atab_set ? atab_h : nullptr, rbp,
                                     nullptr, nullptr, ss));
        else
            DYQ_TRY(dyq_select_bits(state, E, m->t == 0 ? nullptr : prev, bits, nullptr, nullptr, ss));
        return dyq_route_bits(bits, E, 1, atab_set ? atab_h : nullptr, rbd, ss);
    };
    if (forced) {
        DYQ_TRY(dyq_route_bits(forced, E, S, nullptr, rbp, stream));
        DYQ_TRY(dyq_route_bits(forced, E, 1, nullptr, rbd, stream));
        bits = const_cast<int32_t*>(forced);  // detok copies it to bits_out
    } else if (paper) {
        // the selector overlaps the visual prefill on a side stream
        // (fork / join by events: one graph with two branches under capture);
        // the prefill runs at the fixed prefill width on the W4 copy
        if (cudaEventRecord(m->ev_fork, st) != cudaSuccess || cudaStreamWaitEvent(m->side, m->ev_fork, 0) != cudaSuccess)
            return check_launch("paper-mode fork");
        DYQ_TRY(select(m->side, false));
        if (cudaEventRecord(m->ev_join, m->side) != cudaSuccess) return check_launch("paper-mode join record");
        if (launch_pdl(fill_i32_kernel, dim3((MP + 255) / 256), dim3(256), 0, st, rbp, MP, pre_bits) != cudaSuccess)
            return set_error(DYQ_ECUDA, "fill_i32_kernel launch");
        DYQ_TRY(check_launch("fill_i32_kernel"));
    } else {
        DYQ_TRY(select(st, true));
    }

    // one qlinear of the block: on the W4 copy with rows rb, and (variant
    // table) on the W8 copy with rows rb8, each gated on having live rows
    auto qlin = [&](int which, size_t li, const uint16_t* x, int M, int32_t* rb, int32_t* rb8, const int32_t* g,
                    uint16_t* y, bool gated_in) -> dyq_status_t {
        const bool two = w8 && rb8 != nullptr;
        if (two) g_gate = g;
        rc = gated_in ? qlinear_gated(&wd[which], m->codes[li + which], m->meta[li + which], x, M, rb, 0, y, 1,
                                      ws[which], L.ws_bytes[which], err, st)
                      : dyq_qlinear(&wd[which], m->codes[li + which], m->meta[li + which], x, M, rb, 0, y, 1,
                                    ws[which], L.ws_bytes[which], err, stream);
        if (two && !rc) {
            g_gate = g + 1;
            rc = gated_in ? qlinear_gated(&wd[4 + which], m->codes8[li + which], m->meta8[li + which], x, M, rb8, 0, y,
                                          1, ws8[which], L.ws_bytes[4 + which], err, st)
                          : dyq_qlinear(&wd[4 + which], m->codes8[li + which], m->meta8[li + which], x, M, rb8, 0, y,
                                        1, ws8[which], L.ws_bytes[4 + which], err, stream);
        }
        g_gate = nullptr;
        return rc;
    };

    // Decode passes, W4-pinned table, M <= 16: the activation quantization of
    // the o, gate|up and next-layer qkv projections runs in the epilogue of
    // the kernel producing their input (attention, add + RMSNorm), each
    // linear then runs dyq_qlinear_q on those records.  add_rmsnorm_q reads
    // h from hc and writes h + delta to ho (then swapped), two per layer, so
    // hc is h again at the end of every pass.
    uint16_t* hc = h;
    uint16_t* ho = m->at<uint16_t>(L.h2);
    bool qkv_ready = false;  // xn's qkv records already in ws[0]
    auto oquant = [&](int which, int M, int32_t* rb) {
        OQuant q{};
        WLayout Lw;
        if (make_layout(&wd[which], &Lw)) {
            q.ws = dec_act_area(Lw, ws[which]);
            q.A = act_layout_dec(Lw, dec_nt8(M));
            q.L = Lw;
            q.row_bits = rb;
            q.bits = 0;
            q.M = M;
            q.err = err;
        }
        return q;
    };
    auto pquant = [&](int which, int M, int32_t* rb) {
        PQuant q{};
        WLayout Lw;
        if (make_layout(&wd[which], &Lw) && !prefill_e4m3(Lw)) {
            q.act = pre_act_area(Lw, ws[which]);
            q.P = pre_act_layout(Lw, M);
            q.L = Lw;
            q.row_bits = rb;
            q.bits = 0;
            q.M = M;
            q.err = err;
        }
        return q;
    };
    // add + RMSNorm into xn; with mode 1 (decode path) / 2 (prefill path) it
    // also writes linear `which`'s activation records (-1: none); *quantized
    // tells whether it did
    auto norm = [&](const uint16_t* dl, const uint16_t* nwt, int M, int32_t* rb, int which, int mode,
                    bool* quantized) -> dyq_status_t {
        *quantized = false;
        if (mode == 2 && which >= 0) {
            const PQuant q = pquant(which, M, rb);
            const dyq_status_t r = q.act ? add_rmsnorm_pq(hc, dl, nwt, M, d, D.rms_eps, xn, q, st) : DYQ_EUNSUPPORTED;
            if (r == DYQ_OK) {
                *quantized = true;
                return DYQ_OK;
            }
            if (r != DYQ_EUNSUPPORTED) return r;
        }
        if (mode == 1) {
            const OQuant q = which >= 0 ? oquant(which, M, rb) : OQuant{};
            const dyq_status_t r = add_rmsnorm_q(hc, dl, nwt, M, d, D.rms_eps, xn, dl ? ho : nullptr, q, st);
            if (r == DYQ_OK) {
                if (dl) std::swap(hc, ho);
                *quantized = q.ws != nullptr;
                return DYQ_OK;
            }
            if (r != DYQ_EUNSUPPORTED) return r;
        }
        return dyq_add_rmsnorm(hc, dl, nwt, M, d, D.rms_eps, xn, stream);
    };
    // the fused records' mode for an M-row call: 1 = decode kernels (M <= 16),
    // 2 = prefill kernels, as dyq_qlinear would route it; 0 = separate kernels
    auto fuse_mode = [&](int M, int32_t* rb8) {
        if (!fuse_oq || (w8 && rb8 != nullptr) || g_path != 0) return 0;
        return M <= DEC_MPAD ? 1 : 2;
    };
    // linear `which` on the records its producer wrote (mode 1 / 2)
    auto run_ready = [&](int which, size_t li, const uint16_t* x, int M, int32_t* rb, uint16_t* y,
                         int mode) -> dyq_status_t {
        if (mode == 1)
            return dyq_qlinear_q(&wd[which], m->codes[li + which], m->meta[li + which], x, M, rb, 0, y, 1, ws[which],
                                 L.ws_bytes[which], stream);
        WLayout Lw;
        if (!make_layout(&wd[which], &Lw)) return set_error(DYQ_EINVAL, "bad weight descriptor");
        return launch_prefill(Lw, m->codes[li + which], m->meta[li + which], M, rb, 0, y, 1, nullptr,
                              pre_act_area(Lw, ws[which]), st);
    };
    auto layer = [&](int l, int M, int32_t* rb, int32_t* rb8, const int32_t* g, bool prefill, int pos)
        -> dyq_status_t {
        const size_t li = (size_t)4 * l;
        const int fmode = fuse_mode(M, rb8);
        if (qkv_ready && fmode)
            DYQ_TRY(run_ready(0, li, xn, M, rb, qkv, fmode));
        else
            DYQ_TRY(qlin(0, li, xn, M, rb, rb8, g, qkv, false));
        qkv_ready = false;
        bool o_done = false;
        if (prefill) {
            DYQ_TRY(dyq_rope(qkv, M, S, 0, d, H, D.rope_theta, stream));
            DYQ_TRY(dyq_attention_prefill(qkv, E, S, d, H, kv, l, NL, L.T, att, stream));
        } else {
            // RoPE inside the decode attention kernel (one launch less per layer
            // and decode pass), and -- W4-pinned table, M <= 16 -- the o
            // projection's activation quantization in its epilogue (one more);
            // the separate kernels where the fused ones cannot run
            OQuant oq{};
            WLayout Lo;
            const bool fuse_o = fmode == 1 && make_layout(&wd[1], &Lo);  // dyq_qlinear would take the decode path
            if (fuse_o) {
                oq.ws = dec_act_area(Lo, ws[1]);
                oq.A = act_layout_dec(Lo, dec_nt8(M));
                oq.L = Lo;
                oq.row_bits = rb;
                oq.bits = 0;
                oq.M = M;
                oq.err = err;
            }
            rc = attention_decode(qkv, E, pos, d, H, kv, l, NL, L.T, att, D.rope_theta, st, oq);
            if (rc == DYQ_EUNSUPPORTED) {
                DYQ_TRY(dyq_rope(qkv, M, 1, pos, d, H, D.rope_theta, stream));
                DYQ_TRY(dyq_attention_decode(qkv, E, pos, d, H, kv, l, NL, L.T, att, stream));
            } else if (rc) {
                return rc;
            } else {
                o_done = fuse_o;
            }
        }
        if (o_done)  // o projection on the records the attention kernel wrote
            DYQ_TRY(dyq_qlinear_q(&wd[1], m->codes[li + 1], m->meta[li + 1], att, M, rb, 0, delta, 1, ws[1],
                                  L.ws_bytes[1], stream));
        else
            DYQ_TRY(qlin(1, li, att, M, rb, rb8, g, delta, false));
        bool gu_ready = false;
        DYQ_TRY(norm(delta, D.mlp_norm + (size_t)l * d, M, rb, 2, fmode, &gu_ready));
        if (gu_ready)
            DYQ_TRY(run_ready(2, li, xn, M, rb, gu, fmode));
        else
            DYQ_TRY(qlin(2, li, xn, M, rb, rb8, g, gu, false));
        // SwiGLU fused into the down projection's activation quantization
        // (bit-identical to dyq_silu_mul + dyq_qlinear; one launch less per layer)
        DYQ_TRY(qlin(3, li, gu, M, rb, rb8, g, delta, true));
        const uint16_t* nw = l + 1 < NL ? D.attn_norm + (size_t)(l + 1) * d : D.final_norm;
        DYQ_TRY(norm(delta, nw, M, rb, l + 1 < NL ? 0 : -1, fmode, &qkv_ready));
        return DYQ_OK;
    };
    auto bring_h_home = [&]() -> dyq_status_t {  // after an odd number of in-place fallbacks
        if (hc != h) {
            if (cudaMemcpyAsync(h, hc, (size_t)L.MP * d * 2, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
                return check_launch("h copy");
            std::swap(hc, ho);
        }
        return DYQ_OK;
    };

    // ---- prefill: vision + text tokens
    if (launch_pdl(embed_prefill_kernel, dim3(MP), dim3(128), 0, st, vis, text, D.embed, D.n_vis, D.n_text, d, h,
                   src_E) !=
        cudaSuccess)
        return set_error(DYQ_ECUDA, "embed_prefill_kernel launch");
    DYQ_TRY(check_launch("embed_prefill_kernel"));
    DYQ_TRY(norm(nullptr, D.attn_norm, MP, rbp, 0, fuse_mode(MP, paper ? nullptr : rb8p), &qkv_ready));
    for (int l = 0; l < NL; ++l) DYQ_TRY(layer(l, MP, rbp, paper ? nullptr : rb8p, gates, true, 0));
    DYQ_TRY(bring_h_home());
    if (paper && cudaStreamWaitEvent(st, m->ev_join, 0) != cudaSuccess) return check_launch("paper-mode join");
    DYQ_TRY(dyq_head_argmax(xn + (size_t)(S - 1) * d, E, S, d, D.head_bins, D.n_bins, logits, tok, D.n_act, stream));
    // ---- decode passes: one action token per pass
    for (int t = 1; t < D.n_act; ++t) {
        if (launch_pdl(embed_action_kernel, dim3(E), dim3(128), 0, st, tok, D.n_act, t - 1, D.embed, D.vocab, D.n_bins,
                       d, h) != cudaSuccess)
            return set_error(DYQ_ECUDA, "embed_action_kernel launch");
        DYQ_TRY(check_launch("embed_action_kernel"));
        DYQ_TRY(norm(nullptr, D.attn_norm, E, rbd, 0, fuse_mode(E, rb8d), &qkv_ready));
        for (int l = 0; l < NL; ++l) DYQ_TRY(layer(l, E, rbd, rb8d, gates + 2, false, S + t - 1));
        DYQ_TRY(bring_h_home());
        DYQ_TRY(dyq_head_argmax(xn, E, 1, d, D.head_bins, D.n_bins, logits, tok + t, D.n_act, stream));
    }
    if (launch_pdl(detok_kernel, dim3((E * D.n_act + 127) / 128), dim3(128), 0, st, tok, E, D.n_act, D.n_bins,
                   action_out, prev, bits, bits_out) != cudaSuccess)
        return set_error(DYQ_ECUDA, "detok_kernel launch");
    DYQ_TRY(check_launch("detok_kernel"));
#undef DYQ_TRY
    m->t += 1;
    return DYQ_OK;
}

dyq_status_t dyq_policy_step(void* model, void* state, int32_t E, const uint16_t* vis, const int32_t* text,
                             float* action_out, int32_t* bits_out, dyq_stream_t stream) {
    if (!state) return set_error(DYQ_EINVAL, "null state");
    return policy_step_impl(model, state, nullptr, E, E, vis, text, action_out, bits_out, stream);
}

dyq_status_t dyq_policy_step_bits(void* model, int32_t E, const int32_t* bits, const uint16_t* vis,
                                  const int32_t* text, float* action_out, dyq_stream_t stream) {
    if (!bits) return set_error(DYQ_EINVAL, "null bits");
    return policy_step_impl(model, nullptr, bits, E, E, vis, text, action_out, nullptr, stream);
}

// e[e, j] = || a[(j+1) Ec + e, :] - a[e, :] ||_2 in fp64, j = 0..2 (b = 2, 4, 8)
__global__ void calib_errors_kernel(const float* __restrict__ a, int Ec, int n_act, double* __restrict__ e_out) {
    ptx::pdl_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 3 * Ec) return;
    const int e = i / 3, j = i % 3;
    const float* ref = a + (size_t)e * n_act;
    const float* q = a + ((size_t)(j + 1) * Ec + e) * n_act;
    double acc = 0.0;
    for (int k = 0; k < n_act; ++k) {
        const double d = (double)q[k] - (double)ref[k];
        acc = __dadd_rn(acc, __dmul_rn(d, d));
    }
    e_out[i] = __dsqrt_rn(acc);
}

__global__ void calib_bits_kernel(int Ec, int32_t* __restrict__ bits) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < 4 * Ec) bits[i] = (i < Ec) ? 16 : (2 << (i / Ec - 1));  // 16 | 2 | 4 | 8
}

dyq_status_t dyq_calib_errors(const float* actions, int32_t Ec, int32_t n_act, double* err_out, dyq_stream_t stream) {
    if (!actions || !err_out) return set_error(DYQ_EINVAL, "null pointer");
    if (Ec <= 0 || n_act <= 0) return set_error(DYQ_ESHAPE, "Ec = %d, n_act = %d", Ec, n_act);
    if (launch_pdl(calib_errors_kernel, dim3((3 * Ec + 127) / 128), dim3(128), 0, (cudaStream_t)stream, actions, Ec,
                   n_act, err_out) != cudaSuccess)
        return set_error(DYQ_ECUDA, "calib_errors_kernel launch");
    return check_launch("calib_errors_kernel");
}

dyq_status_t dyq_calib_collect(void* model, void* state, int32_t Ec, const uint16_t* vis, const int32_t* text,
                               float* actions_out, double* S_out, double* err_out, dyq_stream_t stream) {
    Model* m = reinterpret_cast<Model*>(model);
    if (!m || !state || !vis || !text || !actions_out || !S_out || !err_out)
        return set_error(DYQ_EINVAL, "null pointer");
    if (Ec <= 0 || 4 * Ec > m->d.E) return set_error(DYQ_EINVAL, "4 * Ec = %d outside [4, E = %d]", 4 * Ec, m->d.E);
    const ModelLayout& L = m->L;
    int32_t* bits = m->at<int32_t>(L.bits);
    float* prev = m->at<float>(L.prev);       // a*_{t-1} of stream e at prev[e * 7] (FP replicas first)
    const cudaStream_t st = (cudaStream_t)stream;
    dyq_status_t rc = dyq_select_bits(state, Ec, m->t == 0 ? nullptr : prev, bits, S_out, nullptr, stream);
    if (rc) return rc;
    int32_t* fb = bits;  // [desc.E >= 4 Ec]: b*_t of the selection above is not used
    calib_bits_kernel<<<(4 * Ec + 127) / 128, 128, 0, st>>>(Ec, fb);
    if ((rc = check_launch("calib_bits_kernel"))) return rc;
    if ((rc = policy_step_impl(model, nullptr, fb, Ec, 4 * Ec, vis, text, actions_out, nullptr, stream))) return rc;
    return dyq_calib_errors(actions_out, Ec, m->d.n_act, err_out, stream);
}

}  // extern "C"
