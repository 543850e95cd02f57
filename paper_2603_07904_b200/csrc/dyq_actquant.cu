// dyq_actquant.cu -- dynamic activation quantization (PAPER.md P:220, P:223:
// the step-wise activation switches between BF16 and X in {2,4,8}; Eq. (2) per
// (token, group), reading 6).  Writes the decode layout described in
// dyq_internal.cuh (one codes+params record per K-group, x16, zx).
#include "dyq_internal.cuh"
#include "dyq_ptx.cuh"

#ifndef DYQ_AQ_THREADS
#define DYQ_AQ_THREADS 512  // threads per act-quant CTA (one warp per (group, token)); 512 measured best
#endif

namespace dyq {

// One warp per (group g, token m); M <= DEC_MPAD tokens starting at row m0,
// padded to 8 * nt8 rows.  A16 rows: zero codes / params and a bf16 copy of x
// in x16; padding rows (m >= M): all zero.
__global__ void actquant_dec_kernel(WLayout L, const uint16_t* __restrict__ x, int M, int m0,
                                    const int32_t* __restrict__ row_bits, int bits, uint8_t* __restrict__ ws,
                                    ActLayoutDec A, int64_t* err, uint64_t* trace, uint32_t serial, int gated,
                                    const int32_t* gate) {
    if (gate_closed(gate)) return;
    ptx::pdl_launch_dependents();
    if (threadIdx.x == 0) trace_ev(trace, serial, 2, 0);
    ptx::pdl_wait();  // x may be produced by the preceding kernel
    if (threadIdx.x == 0) trace_ev(trace, serial, 2, 1);
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int MP = 8 * A.nt8;
    if (warp >= MP * L.NG) return;
    const int g = warp / MP, m = warp % MP;
    aq_dec_job(L, x, M, m0, row_bits, bits, ws, A, err, gated, g, m, dec_call_centred(M, m0, row_bits, bits));
    if (threadIdx.x == 0) trace_ev(trace, serial, 2, 2);
}

dyq_status_t launch_actquant_dec(const WLayout& L, const uint16_t* x, int M, int m0, const int32_t* row_bits,
                                 int bits, void* ws, int64_t* err, cudaStream_t st, int gated) {
    // rows m0 .. m0+M-1 (M <= DEC_MPAD) of x / row_bits (base pointers)
    const ActLayoutDec A = act_layout_dec(L, dec_nt8(M));
    const int warps = 8 * A.nt8 * L.NG;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((warps * 32 + DYQ_AQ_THREADS - 1) / DYQ_AQ_THREADS);
    cfg.blockDim = dim3(DYQ_AQ_THREADS);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, actquant_dec_kernel, L, x, M, m0, row_bits, bits,
                                             reinterpret_cast<uint8_t*>(ws), A, err, g_trace, g_trace_serial++, gated, g_gate);
    if (e != cudaSuccess) return set_error(DYQ_ECUDA, "actquant_dec_kernel launch: %s", cudaGetErrorString(e));
    return check_launch("actquant_dec_kernel");
}

// Test hook: export the decode-layout activation codes in logical layout.
__global__ void actquant_export_kernel(WLayout L, int M, int m0, const int32_t* __restrict__ row_bits, int bits,
                                       const uint8_t* __restrict__ ws, ActLayoutDec A, uint8_t* oq, float* os,
                                       uint8_t* oz, int32_t* oSX) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)M * L.K) return;
    const int m = (int)(idx / L.K), k = (int)(idx % L.K);
    const int g = k / L.G, kk = k % L.G;
    const int pos = (kk & ~63) + dec_perm(kk & 63);
    const bool centred = dec_call_centred(M, m0, row_bits, bits);
    const int z = ws[A.zx_off + (size_t)g * DEC_MPAD + m];
    const uint8_t* rec = ws + A.cp_off + (size_t)g * A.cp_stride;
    const uint8_t c = rec[(size_t)m * L.G + pos];
    const int b = row_bits ? row_bits[m0 + m] : bits;
    oq[(size_t)(m0 + m) * L.K + k] = (centred && b != 16) ? (uint8_t)((int)(int8_t)c + z) : c;
    if (kk == 0) {
        const uint2 p = reinterpret_cast<const uint2*>(rec + 8 * A.nt8 * L.G)[m];
        os[(size_t)(m0 + m) * L.NG + g] = __uint_as_float(p.x);
        oz[(size_t)(m0 + m) * L.NG + g] = (uint8_t)z;
        oSX[(size_t)(m0 + m) * L.NG + g] = centred ? (int32_t)p.y + L.G * z : (int32_t)(p.y & 0xffffu);
    }
}

dyq_status_t launch_actquant_export(const WLayout& L, int M, const int32_t* row_bits, int bits, const void* ws,
                                    uint8_t* xq, float* sx, uint8_t* zx, int32_t* SX, int m0, cudaStream_t st) {
    const ActLayoutDec A = act_layout_dec(L, dec_nt8(M));
    const size_t total = (size_t)M * L.K;
    actquant_export_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
        L, M, m0, row_bits, bits, reinterpret_cast<const uint8_t*>(ws), A, xq, sx, zx, SX);
    return check_launch("actquant_export_kernel");
}

}  // namespace dyq
