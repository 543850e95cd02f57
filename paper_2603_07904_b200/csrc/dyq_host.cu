#include <mutex>
#include <unordered_map>
// dyq_host.cu -- the C ABI of include/dyq.h: argument validation, sizing, plans
// and kernel routing.  No allocation, no host synchronization on the hot path.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <climits>
#include <stdlib.h>

#include "dyq_internal.cuh"

namespace dyq {

static thread_local char g_err[512] = "";
int g_path = 0;
thread_local const int32_t* g_gate = nullptr;
uint64_t* g_trace = nullptr;
uint32_t g_trace_serial = 0;  // 0 auto, 1 decode, 2 prefill (read by the router)

dyq_status_t set_error(dyq_status_t st, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return st;
}

dyq_status_t check_launch(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(DYQ_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return DYQ_OK;
}

bool pdl_enabled() {
    static const int off = getenv("DYQ_NO_PDL") ? atoi(getenv("DYQ_NO_PDL")) : 0;
    return off == 0;
}

bool make_layout(const dyq_wdesc_t* wd, WLayout* L) {
    if (!wd) return false;
    L->N = wd->N;
    L->K = wd->K;
    L->G = wd->group;
    L->wbits = wd->wbits;
    L->round_mode = wd->round_mode;
    if (L->N <= 0 || L->K <= 0 || L->G <= 0) return false;
    L->NG = L->K / L->G;
    L->NSP = L->K / 64;
    L->T128 = (L->N + 127) / 128;
    L->nsub_last = (L->N - 128 * (L->T128 - 1)) / 16;
    L->chunk = 512 * (L->wbits / 4);
    L->codes_bytes = (size_t)L->N * L->K * L->wbits / 8;
    L->meta_bytes = (size_t)L->T128 * L->NG * META_BLOCK;
    return true;
}

static dyq_status_t validate_wdesc(const dyq_wdesc_t* wd, WLayout* L) {
    if (!wd) return set_error(DYQ_EINVAL, "null weight descriptor");
    if (wd->wbits != 4 && wd->wbits != 8)
        return set_error(DYQ_EINVAL, "wbits must be 4 or 8 (got %d)", wd->wbits);
    if (wd->group != 64 && wd->group != 128)
        return set_error(DYQ_ESHAPE, "group must be 64 or 128 (got %d)", wd->group);
    if (wd->N <= 0 || wd->K <= 0) return set_error(DYQ_ESHAPE, "N, K must be positive");
    if (wd->N % 16) return set_error(DYQ_ESHAPE, "N %% 16 != 0 (N=%d)", wd->N);
    if (wd->K % wd->group) return set_error(DYQ_ESHAPE, "K %% group != 0 (K=%d, G=%d)", wd->K, wd->group);
    if (wd->round_mode != 0 && wd->round_mode != 1) return set_error(DYQ_EINVAL, "round_mode must be 0 or 1");
    if (!make_layout(wd, L)) return set_error(DYQ_ESHAPE, "bad layout");
    return DYQ_OK;
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }

}  // namespace dyq

using namespace dyq;

extern "C" {

const char* dyq_last_error(void) { return g_err; }
const char* dyq_version(void) { return "dyq 0.1 sm_100a"; }

// Debug trace of kernel timestamps (caller-owned device buffer; null disables).
dyq_status_t dyq_trace_enable(void* dev_buf, int64_t bytes, dyq_stream_t stream) {
    if (!dev_buf) {
        g_trace = nullptr;
        return DYQ_OK;
    }
    if (bytes < 64) return set_error(DYQ_EINVAL, "trace buffer too small");
    const uint64_t hdr[2] = {0ull, (uint64_t)((bytes - 16) / 16)};
    if (cudaMemcpyAsync(dev_buf, hdr, sizeof(hdr), cudaMemcpyHostToDevice, (cudaStream_t)stream) != cudaSuccess)
        return check_launch("dyq_trace_enable");
    g_trace = reinterpret_cast<uint64_t*>(dev_buf);
    return DYQ_OK;
}

dyq_status_t dyq_set_path(int32_t path) {
    if (path < 0 || path > 2) return set_error(DYQ_EINVAL, "path must be 0, 1 or 2");
    g_path = path;
    return DYQ_OK;
}

dyq_status_t dyq_error_reset(int64_t* err, dyq_stream_t stream) {
    if (!err) return set_error(DYQ_EINVAL, "null err");
    static const int64_t none = INT64_MAX;
    // 8-byte pageable source: staged by the driver before return
    if (cudaMemcpyAsync(err, &none, sizeof none, cudaMemcpyHostToDevice, (cudaStream_t)stream) != cudaSuccess)
        return check_launch("dyq_error_reset");
    return DYQ_OK;
}

dyq_status_t dyq_error_read(const int64_t* err, int64_t* host_index, dyq_stream_t stream) {
    if (!err || !host_index) return set_error(DYQ_EINVAL, "null pointer");
    int64_t v = INT64_MAX;
    if (cudaMemcpyAsync(&v, err, sizeof v, cudaMemcpyDeviceToHost, (cudaStream_t)stream) != cudaSuccess ||
        cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess)
        return check_launch("dyq_error_read");
    *host_index = v;
    if (v != INT64_MAX) return set_error(DYQ_ENONFINITE, "non-finite input at linear index %lld", (long long)v);
    return DYQ_OK;
}

dyq_status_t dyq_check_error(const int64_t* err, int64_t* host_index, dyq_stream_t stream) {
    if (!err || !host_index) return set_error(DYQ_EINVAL, "null pointer");
    struct Poll {
        int64_t* slot = nullptr;  // pinned host
        cudaEvent_t ev = nullptr;
        bool pending = false;
    };
    static std::mutex mu;
    static std::unordered_map<const int64_t*, Poll> polls;
    std::lock_guard<std::mutex> lock(mu);
    Poll& p = polls[err];
    if (!p.slot) {
        if (cudaHostAlloc(reinterpret_cast<void**>(&p.slot), sizeof(int64_t), cudaHostAllocDefault) != cudaSuccess ||
            cudaEventCreateWithFlags(&p.ev, cudaEventDisableTiming) != cudaSuccess) {
            polls.erase(err);
            return check_launch("dyq_check_error (pinned slot)");
        }
    }
    if (!p.pending) {
        if (cudaMemcpyAsync(p.slot, err, sizeof(int64_t), cudaMemcpyDeviceToHost, (cudaStream_t)stream) != cudaSuccess ||
            cudaEventRecord(p.ev, (cudaStream_t)stream) != cudaSuccess)
            return check_launch("dyq_check_error");
        p.pending = true;
    }
    const cudaError_t q = cudaEventQuery(p.ev);
    if (q == cudaErrorNotReady) {
        *host_index = -1;
        return DYQ_OK;
    }
    if (q != cudaSuccess) return check_launch("dyq_check_error (event)");
    p.pending = false;
    const int64_t v = *reinterpret_cast<volatile int64_t*>(p.slot);
    *host_index = v;
    if (v != INT64_MAX) return set_error(DYQ_ENONFINITE, "non-finite input at linear index %lld", (long long)v);
    return DYQ_OK;
}

dyq_status_t dyq_pack_weights_size(const dyq_wdesc_t* wd, size_t* codes_bytes, size_t* meta_bytes) {
    WLayout L;
    dyq_status_t rc = validate_wdesc(wd, &L);
    if (rc) return rc;
    if (!codes_bytes || !meta_bytes) return set_error(DYQ_EINVAL, "null size pointer");
    *codes_bytes = L.codes_bytes;
    *meta_bytes = L.meta_bytes;
    return DYQ_OK;
}

dyq_status_t dyq_pack_weights(const dyq_wdesc_t* wd, const uint16_t* w_bf16, void* codes, void* meta,
                              int64_t* err, dyq_stream_t stream) {
    WLayout L;
    dyq_status_t rc = validate_wdesc(wd, &L);
    if (rc) return rc;
    if (!w_bf16 || !codes || !meta) return set_error(DYQ_EINVAL, "null pointer");
    if (!aligned16(codes) || !aligned16(meta)) return set_error(DYQ_EINVAL, "codes/meta must be 16-byte aligned");
    return launch_pack(L, w_bf16, codes, meta, err, (cudaStream_t)stream);
}

dyq_status_t dyq_unpack_for_check(const dyq_wdesc_t* wd, const void* codes, const void* meta, uint8_t* q,
                                  float* s, uint8_t* z, dyq_stream_t stream) {
    WLayout L;
    dyq_status_t rc = validate_wdesc(wd, &L);
    if (rc) return rc;
    if (!codes || !meta || !q || !s || !z) return set_error(DYQ_EINVAL, "null pointer");
    return launch_unpack(L, codes, meta, q, s, z, (cudaStream_t)stream);
}

static dyq_status_t validate_calib(const dyq_calib_t* c) {
    if (!c) return set_error(DYQ_EINVAL, "null calibration table");
    if (!(0.0 <= c->theta_24 && c->theta_24 <= c->theta_48 && c->theta_48 <= c->theta_fp))
        return set_error(DYQ_EINVAL, "thresholds must satisfy 0 <= theta_24 <= theta_48 <= theta_fp (S:198)");
    if (!(c->lambda >= 0.0 && c->lambda <= 1.0)) return set_error(DYQ_EINVAL, "lambda must be in [0,1]");
    if (!(c->D_acc > 0.0) || !(c->eta > 0.0)) return set_error(DYQ_EINVAL, "D_acc and eta must be > 0 (S:199)");
    if (!(c->J_cap > 0.0)) return set_error(DYQ_EINVAL, "J_cap must be > 0");
    if (c->K < 1) return set_error(DYQ_EINVAL, "K must be >= 1 (S:199)");
    if (c->W_macro < 1 || c->W_macro > 64 || c->W_micro < 1 || c->W_micro > 64)
        return set_error(DYQ_EINVAL, "windows must be in [1,64]");
    if (c->H < 1 || c->H > 1024) return set_error(DYQ_EINVAL, "H must be in [1,1024]");
    return DYQ_OK;
}

dyq_status_t dyq_state_size(int32_t E, const dyq_calib_t* calib, size_t* bytes) {
    dyq_status_t rc = validate_calib(calib);
    if (rc) return rc;
    if (E <= 0 || E > (1 << 20)) return set_error(DYQ_ESHAPE, "E out of range");
    if (!bytes) return set_error(DYQ_EINVAL, "null bytes");
    *bytes = sel_state_bytes(E, *calib);
    return DYQ_OK;
}

dyq_status_t dyq_state_init(int32_t E, const dyq_calib_t* calib, void* state, dyq_stream_t stream) {
    dyq_status_t rc = validate_calib(calib);
    if (rc) return rc;
    if (E <= 0 || E > (1 << 20)) return set_error(DYQ_ESHAPE, "E out of range");
    if (!state || !aligned16(state)) return set_error(DYQ_EINVAL, "state must be a 16-byte aligned device buffer");
    return launch_sel_init(E, *calib, state, (cudaStream_t)stream);
}

// E is needed for the grid; the reset kernel reads it from the device header,
// so launch for the maximum and let threads beyond E exit.
dyq_status_t dyq_state_reset_episode(void* state, const uint8_t* mask, dyq_stream_t stream) {
    if (!state) return set_error(DYQ_EINVAL, "null state");
    return launch_sel_reset(state, 1 << 16, mask, (cudaStream_t)stream);
}

dyq_status_t dyq_select_bits(void* state, int32_t E, const float* prev_action, int32_t* bits, double* S_out,
                             int32_t* target_out, dyq_stream_t stream) {
    if (!state || !bits) return set_error(DYQ_EINVAL, "null pointer");
    if (E <= 0 || E > (1 << 20)) return set_error(DYQ_ESHAPE, "E out of range");
    return launch_select(state, E, nullptr, prev_action, bits, S_out, target_out, 0, nullptr, nullptr,
                         (cudaStream_t)stream);
}

dyq_status_t dyq_select_route(void* state, int32_t E, const float* prev_action, int32_t* bits,
                              int32_t tokens_per_episode, const int32_t* abits_of_host, int32_t* row_bits,
                              double* S_out, int32_t* target_out, dyq_stream_t stream) {
    if (!state || !bits || !row_bits) return set_error(DYQ_EINVAL, "null pointer");
    if (E <= 0 || E > (1 << 20)) return set_error(DYQ_ESHAPE, "E out of range");
    if (tokens_per_episode <= 0) return set_error(DYQ_ESHAPE, "tokens_per_episode must be positive");
    if (abits_of_host)
        for (int i = 0; i < 4; ++i) {
            const int b = abits_of_host[i];
            if (b != 2 && b != 4 && b != 8 && b != 16)
                return set_error(DYQ_EINVAL, "abits_of[%d] = %d not in {2,4,8,16}", i, b);
        }
    return launch_select(state, E, nullptr, prev_action, bits, S_out, target_out, tokens_per_episode, abits_of_host,
                         row_bits, (cudaStream_t)stream);
}

dyq_status_t dyq_route_bits(const int32_t* bits, int32_t E, int32_t tpe, const int32_t* abits_of_host,
                            int32_t* row_bits, dyq_stream_t stream) {
    if (!bits || !row_bits) return set_error(DYQ_EINVAL, "null pointer");
    if (E <= 0 || tpe <= 0) return set_error(DYQ_ESHAPE, "E and tokens_per_episode must be positive");
    if (abits_of_host)
        for (int i = 0; i < 4; ++i) {
            const int b = abits_of_host[i];
            if (b != 2 && b != 4 && b != 8 && b != 16) return set_error(DYQ_EINVAL, "abits_of entries must be 2/4/8/16");
        }
    return launch_route(bits, E, tpe, abits_of_host, row_bits, (cudaStream_t)stream);
}

// Workspace = [decode split-K accumulator + tile counters (must start zeroed;
// self-cleaning)] [standalone activation-quantizer output (dyq_act_quant)].
static size_t act_area_offset(const WLayout& L) { return (decode_ws_bytes(L) + 255) & ~(size_t)255; }
}  // extern "C"
namespace dyq {
uint8_t* dec_act_area(const WLayout& L, void* ws) { return reinterpret_cast<uint8_t*>(ws) + act_area_offset(L); }
}  // namespace dyq
extern "C" {
// The 1 KB before the prefill area holds the prefill stream-K unit counters
// (fixed position per shape, so they stay zeroed for every M; self-resetting).
static size_t prefill_area_offset(const WLayout& L) {
    return ((act_area_offset(L) + act_layout_dec(L, 2).bytes + 1023) & ~(size_t)1023) + PRE_CNT_BYTES;
}
}  // extern "C"
namespace dyq {
uint8_t* pre_act_area(const WLayout& L, void* ws) { return reinterpret_cast<uint8_t*>(ws) + prefill_area_offset(L); }
}  // namespace dyq
extern "C" {

dyq_status_t dyq_qlinear_workspace(const dyq_wdesc_t* wd, int32_t M, size_t* bytes) {
    WLayout L;
    dyq_status_t rc = validate_wdesc(wd, &L);
    if (rc) return rc;
    if (M < 0 || M > 65536) return set_error(DYQ_ESHAPE, "M out of range [0, 65536]");
    if (!bytes) return set_error(DYQ_EINVAL, "null bytes");
    // the prefill activation area is reserved for every M > 0: dyq_set_path(2)
    // routes even M <= 16 through the prefill kernels (split-K only for M > 16)
    size_t pre = 0;
    if (M > 0) pre = ((pre_act_layout(L, M).bytes + 255) & ~(size_t)255) + prefill_part_bytes(L, M);
    *bytes = prefill_area_offset(L) + pre;
    return DYQ_OK;
}

dyq_status_t dyq_qlinear_masked(const dyq_wdesc_t* wd, const void* codes, const void* meta, const uint16_t* x,
                                int32_t M, const int32_t* row_bits, const int32_t* gate, void* y, int32_t y_dtype,
                                void* workspace, size_t ws_bytes, int64_t* err, dyq_stream_t stream) {
    if (!row_bits) return set_error(DYQ_EINVAL, "dyq_qlinear_masked needs row_bits");
    g_gate = gate;
    const dyq_status_t rc = dyq_qlinear(wd, codes, meta, x, M, row_bits, 0, y, y_dtype, workspace, ws_bytes, err, stream);
    g_gate = nullptr;
    return rc;
}

dyq_status_t dyq_qlinear_plan(const dyq_wdesc_t* wd, int32_t M, int32_t* path, int32_t* ksplit) {
    WLayout L;
    dyq_status_t rc = validate_wdesc(wd, &L);
    if (rc) return rc;
    if (M < 0 || M > 65536) return set_error(DYQ_ESHAPE, "M out of range [0, 65536]");
    const bool pre = g_path == 2 || (g_path == 0 && M > DEC_MPAD);
    if (path) *path = pre ? 2 : 1;
    if (ksplit) *ksplit = pre ? prefill_ksplit(L, M) : 1;
    return DYQ_OK;
}

dyq_status_t dyq_workspace_init(void* ws, size_t bytes, dyq_stream_t stream) {
    if (!ws && bytes) return set_error(DYQ_EINVAL, "null workspace");
    if (bytes && cudaMemsetAsync(ws, 0, bytes, (cudaStream_t)stream) != cudaSuccess)
        return check_launch("dyq_workspace_init");
    return DYQ_OK;
}

static dyq_status_t validate_ql(const dyq_wdesc_t* wd, WLayout* L, const void* codes, const void* meta,
                                const uint16_t* x, int32_t M, const int32_t* row_bits, int32_t bits, bool has_out,
                                int32_t y_dtype, bool check_ydt, void* ws, size_t ws_bytes) {
    dyq_status_t rc = validate_wdesc(wd, L);
    if (rc) return rc;
    if (M < 0 || M > 65536) return set_error(DYQ_ESHAPE, "M out of range [0, 65536]");
    if (M == 0) return DYQ_OK;
    if (!codes || !meta || !x || !ws || !has_out) return set_error(DYQ_EINVAL, "null pointer");
    if (!aligned16(codes) || !aligned16(meta) || !aligned16(ws) || !aligned16(x))
        return set_error(DYQ_EINVAL, "codes/meta/x/workspace must be 16-byte aligned");
    if (!row_bits && bits != 2 && bits != 4 && bits != 8 && bits != 16)
        return set_error(DYQ_EINVAL, "bits must be 2, 4, 8 or 16 (got %d)", bits);
    if (check_ydt && y_dtype != 0 && y_dtype != 1) return set_error(DYQ_EINVAL, "y_dtype must be 0 (fp32) or 1 (bf16)");
    size_t need = 0;
    dyq_qlinear_workspace(wd, M, &need);
    if (ws_bytes < need) return set_error(DYQ_EINVAL, "workspace too small (%zu < %zu)", ws_bytes, need);
    return DYQ_OK;
}

// Decode path: per 16-token tile, the activation quantizer writes the
// workspace's activation area, then the decode kernel streams the weights
// (programmatic dependent launch lets it start before the quantizer ends).
static dyq_status_t run_decode(const WLayout& L, const void* codes, const void* meta, const uint16_t* x, int32_t M,
                               const int32_t* row_bits, int32_t bits, void* y, int32_t y_dtype, int32_t* I, void* ws,
                               int64_t* err, cudaStream_t st, int gated = 0) {
    if (g_path == 2 || (g_path == 0 && M > DEC_MPAD)) {
        // prefill: tcgen05 kernels over 128-token tiles
        uint8_t* pa = reinterpret_cast<uint8_t*>(ws) + prefill_area_offset(L);
        dyq_status_t rc = launch_actquant_pre(L, x, M, row_bits, bits, pa, err, st, gated);
        if (rc) return rc;
        return launch_prefill(L, codes, meta, M, row_bits, bits, y, y_dtype, I, pa, st);
    }
    uint8_t* area = reinterpret_cast<uint8_t*>(ws) + act_area_offset(L);
    for (int m0 = 0; m0 < M; m0 += DEC_MPAD) {
        const int mt = (M - m0) < DEC_MPAD ? (M - m0) : DEC_MPAD;
        dyq_status_t rc = launch_actquant_dec(L, x, mt, m0, row_bits, bits, area, err, st, gated);
        if (rc) return rc;
        rc = launch_decode(L, codes, meta, x, mt, m0, row_bits, bits, y, y_dtype, I, ws, err, st);
        if (rc) return rc;
    }
    return DYQ_OK;
}

}  // extern "C"

namespace dyq {
// Policy-step internal (not exported): dyq_qlinear on the SwiGLU activation of
// gu = [g | u] (rows of 2K); the quantizers form bf16(silu(g) u) on the fly,
// bit-identical to dyq_silu_mul followed by dyq_qlinear.
dyq_status_t qlinear_gated(const dyq_wdesc_t* wd, const void* codes, const void* meta, const uint16_t* gu, int32_t M,
                           const int32_t* row_bits, int32_t bits, void* y, int32_t y_dtype, void* ws, size_t ws_bytes,
                           int64_t* err, cudaStream_t st) {
    WLayout L;
    dyq_status_t rc = validate_ql(wd, &L, codes, meta, gu, M, row_bits, bits, y != nullptr, y_dtype, true, ws,
                                  ws_bytes);
    if (rc || M == 0) return rc;
    return run_decode(L, codes, meta, gu, M, row_bits, bits, y, y_dtype, nullptr, ws, err, st, 1);
}
}  // namespace dyq

extern "C" {

dyq_status_t dyq_qlinear(const dyq_wdesc_t* wd, const void* codes, const void* meta, const uint16_t* x, int32_t M,
                         const int32_t* row_bits, int32_t bits, void* y, int32_t y_dtype, void* workspace,
                         size_t ws_bytes, int64_t* err, dyq_stream_t stream) {
    WLayout L;
    dyq_status_t rc = validate_ql(wd, &L, codes, meta, x, M, row_bits, bits, y != nullptr, y_dtype, true, workspace,
                                  ws_bytes);
    if (rc || M == 0) return rc;
    if (!aligned16(y)) return set_error(DYQ_EINVAL, "y must be 16-byte aligned");
    return run_decode(L, codes, meta, x, M, row_bits, bits, y, y_dtype, nullptr, workspace, err, (cudaStream_t)stream);
}

// Fused TP decode: this rank's column shard of y is
// stored by the decode kernel's epilogue into every rank's full y (peer
// memory), each 16-column sub-tile announced on every rank's flag.
dyq_status_t dyq_qlinear_tp(const dyq_wdesc_t* wd, const void* codes, const void* meta, const uint16_t* x,
                            int32_t M, const int32_t* row_bits, int32_t bits, const dyq_tp_peers_t* peers,
                            void* workspace, size_t ws_bytes, int64_t* err, dyq_stream_t stream) {
    if (!peers) return set_error(DYQ_EINVAL, "null peers");
    if (peers->world < 1 || peers->world > DYQ_TP_MAX || peers->rank < 0 || peers->rank >= peers->world)
        return set_error(DYQ_EINVAL, "bad rank %d / world %d", peers->rank, peers->world);
    for (int p = 0; p < peers->world; ++p) {
        if (!peers->y[p] || !peers->flag[p]) return set_error(DYQ_EINVAL, "null y / flag of rank %d", p);
        if (!aligned16(peers->y[p])) return set_error(DYQ_EINVAL, "y of rank %d must be 16-byte aligned", p);
    }
    WLayout L;
    dyq_status_t rc = validate_ql(wd, &L, codes, meta, x, M, row_bits, bits, true, 1, true, workspace, ws_bytes);
    if (rc || M == 0) return rc;
    TpPeers tp{};
    tp.n = peers->world;
    for (int p = 0; p < tp.n; ++p) {
        tp.y[p] = peers->y[p];
        tp.flag[p] = reinterpret_cast<unsigned long long*>(peers->flag[p]);
    }
    tp.ldy = peers->world * wd->N;
    tp.col0 = peers->rank * wd->N;
    const cudaStream_t st = (cudaStream_t)stream;
    const bool prefill = g_path == 2 || (g_path == 0 && M > DEC_MPAD);  // as run_decode
    if (!prefill && M > DEC_MPAD)
        return set_error(DYQ_EUNSUPPORTED, "fused TP decode handles M <= %d per call (M = %d)", DEC_MPAD, M);
    if (prefill) {  // tcgen05 kernel, TP epilogue per (tile, token tile) CTA
        uint8_t* pa = reinterpret_cast<uint8_t*>(workspace) + prefill_area_offset(L);
        rc = launch_actquant_pre(L, x, M, row_bits, bits, pa, err, st);
        if (rc) return rc;
        return launch_prefill(L, codes, meta, M, row_bits, bits, nullptr, 1, nullptr, pa, st, &tp);
    }
    uint8_t* area = reinterpret_cast<uint8_t*>(workspace) + act_area_offset(L);
    rc = launch_actquant_dec(L, x, M, 0, row_bits, bits, area, err, st);
    if (rc) return rc;
    return launch_decode(L, codes, meta, x, M, 0, row_bits, bits, nullptr, 1, nullptr, workspace, err, st, &tp);
}

dyq_status_t dyq_tp_flag_delta(int32_t N, int32_t M, uint64_t* delta) {
    if (!delta) return set_error(DYQ_EINVAL, "null delta");
    if (N <= 0 || N % 16 || M < 0) return set_error(DYQ_ESHAPE, "N = %d, M = %d", N, M);
    const bool prefill = g_path == 2 || (g_path == 0 && M > DEC_MPAD);
    const int tiles = (M == 0) ? 0 : (prefill ? (M + PRE_PT - 1) / PRE_PT : 1);
    *delta = (uint64_t)(N / 16) * (uint64_t)tiles;
    return DYQ_OK;
}

dyq_status_t dyq_qlinear_i32_partials(const dyq_wdesc_t* wd, const void* codes, const void* meta, const uint16_t* x,
                                      int32_t M, const int32_t* row_bits, int32_t bits, int32_t* I, void* workspace,
                                      size_t ws_bytes, int64_t* err, dyq_stream_t stream) {
    WLayout L;
    dyq_status_t rc = validate_ql(wd, &L, codes, meta, x, M, row_bits, bits, I != nullptr, 0, false, workspace,
                                  ws_bytes);
    if (rc || M == 0) return rc;
    return run_decode(L, codes, meta, x, M, row_bits, bits, nullptr, 0, I, workspace, err, (cudaStream_t)stream);
}

// Asynchronous HBM -> L2 prefetch of packed weights (e.g. the next layer's
// codes and metadata while the current layer's dependent chain runs).
dyq_status_t dyq_prefetch_l2(const void* p, size_t bytes, dyq_stream_t stream) {
    if (!p && bytes) return set_error(DYQ_EINVAL, "null pointer");
    if (((uintptr_t)p & 15) != 0) return set_error(DYQ_EINVAL, "prefetch address must be 16-byte aligned");
    return launch_prefetch_l2(p, bytes, (cudaStream_t)stream);
}

// Standalone quantizer into the workspace's activation area (inspection / reuse).
dyq_status_t dyq_act_quant(const dyq_wdesc_t* wd, const uint16_t* x, int32_t M, const int32_t* row_bits,
                           int32_t bits, void* ws, size_t ws_bytes, int64_t* err, dyq_stream_t stream) {
    WLayout L;
    dyq_status_t rc = validate_wdesc(wd, &L);
    if (rc) return rc;
    if (M < 0 || M > DEC_MPAD) return set_error(DYQ_EUNSUPPORTED, "dyq_act_quant supports M <= %d", DEC_MPAD);
    if (M == 0) return DYQ_OK;
    if (!x || !ws) return set_error(DYQ_EINVAL, "null pointer");
    if (!aligned16(ws) || !aligned16(x)) return set_error(DYQ_EINVAL, "x/workspace must be 16-byte aligned");
    if (!row_bits && bits != 2 && bits != 4 && bits != 8 && bits != 16)
        return set_error(DYQ_EINVAL, "bits must be 2, 4, 8 or 16 (got %d)", bits);
    size_t need = 0;
    dyq_qlinear_workspace(wd, M, &need);
    if (ws_bytes < need) return set_error(DYQ_EINVAL, "workspace too small (%zu < %zu)", ws_bytes, need);
    return launch_actquant_dec(L, x, M, 0, row_bits, bits, reinterpret_cast<uint8_t*>(ws) + act_area_offset(L), err,
                               (cudaStream_t)stream);
}

// Linear layer on activations already quantized into `ws` by dyq_act_quant.
dyq_status_t dyq_qlinear_q(const dyq_wdesc_t* wd, const void* codes, const void* meta, const uint16_t* x,
                           int32_t M, const int32_t* row_bits, int32_t bits, void* y, int32_t y_dtype, void* ws,
                           size_t ws_bytes, dyq_stream_t stream) {
    WLayout L;
    dyq_status_t rc = validate_ql(wd, &L, codes, meta, x, M, row_bits, bits, y != nullptr, y_dtype, true, ws,
                                  ws_bytes);
    if (rc || M == 0) return rc;
    if (M > DEC_MPAD) return set_error(DYQ_EUNSUPPORTED, "dyq_qlinear_q supports M <= %d", DEC_MPAD);
    return launch_decode(L, codes, meta, x, M, 0, row_bits, bits, y, y_dtype, nullptr, ws, nullptr,
                         (cudaStream_t)stream);
}

dyq_status_t dyq_act_quant_for_check(const dyq_wdesc_t* wd, const uint16_t* x, int32_t M, const int32_t* row_bits,
                                     int32_t bits, uint8_t* xq, float* sx, uint8_t* zx, int32_t* SX, void* ws,
                                     size_t ws_bytes, int64_t* err, dyq_stream_t stream) {
    WLayout L;
    dyq_status_t rc = validate_wdesc(wd, &L);
    if (rc) return rc;
    if (M < 0 || M > 65536) return set_error(DYQ_ESHAPE, "M out of range");
    if (!x || !xq || !sx || !zx || !SX || !ws) return set_error(DYQ_EINVAL, "null pointer");
    if (!row_bits && bits != 2 && bits != 4 && bits != 8 && bits != 16)
        return set_error(DYQ_EINVAL, "bits must be 2, 4, 8 or 16");
    size_t need = 0;
    dyq_qlinear_workspace(wd, M, &need);
    if (ws_bytes < need) return set_error(DYQ_EINVAL, "workspace too small");
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t* area = reinterpret_cast<uint8_t*>(ws) + act_area_offset(L);
    for (int m0 = 0; m0 < M; m0 += DEC_MPAD) {
        const int mt = (M - m0) < DEC_MPAD ? (M - m0) : DEC_MPAD;
        rc = launch_actquant_dec(L, x, mt, m0, row_bits, bits, area, err, st);
        if (rc) return rc;
        rc = launch_actquant_export(L, mt, row_bits, bits, area, xq, sx, zx, SX, m0, st);
        if (rc) return rc;
    }
    return DYQ_OK;
}

}  // extern "C"
