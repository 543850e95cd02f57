/*
 * dyq.h -- C ABI of the B200-native DyQ-VLA qlinear hot path (libdyq.so).
 *
 * The method (arXiv 2603.07904, /root/reference/PAPER.md = "P:line"): weights
 * are frozen at INT4 ("INT4-pinned weights across all precision settings",
 * P:332-333), activations are re-quantized every control step at a width
 * b*_t in {2,4,8} or bypassed at BF16 (16), and b*_t is chosen
 * from two kinematic proxies by the Eq. (6) lookup and the Alg. 1 hysteresis
 * dispatcher.  This header exposes that hot path:
 *
 *   dyq_pack_weights   - offline weight quantization at wbits (Eq. 2)
 *   dyq_select_bits    - kinematic proxies -> S_t -> bhat_t -> b*_t (Alg. 1)
 *   dyq_act_quant      - dynamic activation quantization at the step's width
 *   dyq_qlinear        - quantized linear layer  y = dequant(I)
 *
 * Conventions (all functions):
 *  - Pointers are DEVICE pointers unless the parameter says "host".
 *  - Every call is stream-ordered on `stream` and non-blocking: no host
 *    synchronization, no device allocation.  The caller owns every buffer and
 *    sizes them with the *_size / *_workspace queries.
 *  - Returns dyq_status_t.  Argument / shape errors are detected synchronously
 *    (DYQ_EINVAL / DYQ_ESHAPE / DYQ_EUNSUPPORTED) before anything is enqueued;
 *    dyq_last_error() returns a thread-local message.  CUDA launch failures
 *    return DYQ_ECUDA.  No C++ exception crosses this ABI.
 *  - Non-finite inputs ("rejects input with a diagnostic identifying the
 *    offending index") cannot be detected synchronously on a stream: kernels
 *    atomicMin the smallest offending linear element index into the caller's
 *    device int64 `err` (initialise it with dyq_error_reset; INT64_MAX = none)
 *    and the caller polls it (dyq_check_error, non-blocking; dyq_error_read
 *    synchronizes).  Outputs derived from
 *    non-finite inputs are unspecified.  `err` may be NULL (no reporting).
 *  - Packed weights are immutable after packing and may be shared by any
 *    number of streams.  Selection state is single-owner and mutated in step
 *    order.
 *
 * Layouts: see DESIGN.md §"Data layout in HBM".  Tensors are row-major.
 * bf16 is passed as raw 16-bit patterns (uint16_t).
 */
#ifndef DYQ_H
#define DYQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define DYQ_API __attribute__((visibility("default")))
#else
#define DYQ_API
#endif

typedef struct CUstream_st* dyq_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
    DYQ_OK = 0,
    DYQ_EINVAL = 1,       /* bad argument value (bits, null pointer, table ordering) */
    DYQ_ESHAPE = 2,       /* inconsistent / unsupported shape (K % G, N % 16, ...)   */
    DYQ_EUNSUPPORTED = 3, /* valid but not implemented on this build                */
    DYQ_ENONFINITE = 4,   /* non-finite input (reported through err)               */
    DYQ_ECUDA = 5,        /* CUDA runtime error                                     */
    DYQ_ENCCL = 6         /* collective error                                       */
} dyq_status_t;

/* Thread-local description of the last error on this thread ("" if none). */
DYQ_API const char* dyq_last_error(void);
/* Library version string, e.g. "dyq 0.1 sm_100a". */
DYQ_API const char* dyq_version(void);
/* Debug/profiling only: record %globaltimer events of the decode-path kernels
 * into a caller-owned DEVICE buffer laid out as [u64 count][u64 capacity]
 * [capacity x {u64 tag, u64 ns}], tag = serial << 32 | kernel << 24 |
 * event << 16 | blockIdx.x.  dev_buf = NULL disables (the default).  The header
 * words are written with an async copy on `stream`.  DYQ_EINVAL if bytes < 64. */
DYQ_API dyq_status_t dyq_trace_enable(void* dev_buf, int64_t bytes, dyq_stream_t stream);

/* ---------------------------------------------------------------- errors */
/* err: device int64; reset to INT64_MAX (= no error). */
DYQ_API dyq_status_t dyq_error_reset(int64_t* err, dyq_stream_t stream);
/* Synchronizes `stream` and copies *err to *host_index (INT64_MAX = none).
 * Returns DYQ_ENONFINITE if an index was recorded.  (Debug / test path.) */
DYQ_API dyq_status_t dyq_error_read(const int64_t* err, int64_t* host_index, dyq_stream_t stream);
/* Non-blocking poll of *err (SURVEY §8(b) dyq_check_error): the first call
 * for `err` enqueues an async device->host copy into a library-owned pinned
 * slot plus an event on `stream` and returns at once; every call queries the
 * event without waiting.  While the copy is in flight: DYQ_OK with
 * *host_index = -1.  Once it has landed: *host_index = the recorded value
 * (INT64_MAX = none), DYQ_ENONFINITE if an index was recorded, else DYQ_OK;
 * the next call re-arms a fresh copy.  Never synchronizes the stream. */
DYQ_API dyq_status_t dyq_check_error(const int64_t* err, int64_t* host_index, dyq_stream_t stream);

/* ------------------------------------------------------------ weight pack */
/* Weight descriptor.  One (scale, zero-point) per output row n and per group
 * of `group` consecutive input channels (reading 5).
 *   N          output features (rows of W), N % 16 == 0
 *   K          input features, K % group == 0
 *   group      G in {64, 128}
 *   wbits      4 (the paper's INT4-pinned weights) or 8 (optional table)
 *   round_mode 0 = floor exactly as Eq. (2) (default), 1 = round-to-nearest  */
typedef struct {
    int32_t N, K, group, wbits, round_mode;
} dyq_wdesc_t;

/* Bytes of the packed code buffer and of the metadata buffer (scales fp32 +
 * zero-points u8, 5 B per (row, group), padded to whole 128-row tiles). */
DYQ_API dyq_status_t dyq_pack_weights_size(const dyq_wdesc_t* wd, size_t* codes_bytes,
                                   size_t* meta_bytes);

/* Quantize W [N,K] bf16 (device) per (row, group) with the fit of DESIGN.md
 * readings 2-4 (zero-inclusive min-max in fp64, fp32 stored scale, half-up
 * zero point) and Eq. (2); write codes in the kernel layout and
 * the metadata.  codes / meta: device buffers of the sizes above (16-byte
 * aligned).  Offline: not on the per-step path ("we freeze the weights"). */
DYQ_API dyq_status_t dyq_pack_weights(const dyq_wdesc_t* wd, const uint16_t* w_bf16,
                              void* codes, void* meta, int64_t* err,
                              dyq_stream_t stream);

/* Test hook: decode the kernel layout back to logical q [N,K] u8,
 * s [N,K/G] fp32, z [N,K/G] u8 (device buffers). */
DYQ_API dyq_status_t dyq_unpack_for_check(const dyq_wdesc_t* wd, const void* codes,
                                  const void* meta, uint8_t* q, float* s,
                                  uint8_t* z, dyq_stream_t stream);

/* -------------------------------------------------------- bit selection */
/* Calibration table; field names follow SPEC S:261 (CalibrationTable JSON).
 *   theta_24, theta_48, theta_fp  Eq. (6) thresholds and the fallback
 *                                 threshold, 0<=t24<=t48<=tfp
 *   lambda                        fusion weight in [0,1]
 *   D_acc, eta                    error-bound parameters, > 0
 *                                 (calibration only; validated, unused here)
 *   J_cap                         jerk cap (> 0; use 1e300 for none)
 *   K                             Alg. 1 delay window, >= 1
 *   W_macro, W_micro              window lengths, 1..64
 *   H                             p95 history length, 1..1024
 *   clamp_M                       1 = clamp M to [0,1], 0 = literal */
typedef struct {
    double theta_24, theta_48, theta_fp, lambda, D_acc, eta, J_cap;
    int32_t K, W_macro, W_micro, H, clamp_M;
} dyq_calib_t;

/* Device bytes of the selection state for E control streams. */
DYQ_API dyq_status_t dyq_state_size(int32_t E, const dyq_calib_t* calib, size_t* bytes);
/* Initialise the state (all histories empty, dispatcher (16,0,16)). */
DYQ_API dyq_status_t dyq_state_init(int32_t E, const dyq_calib_t* calib, void* state,
                            dyq_stream_t stream);
/* Episode reset for streams with mask[e] != 0 (mask: device u8 [E] or NULL =
 * all): clears windows, prev_rot, warm-up and the dispatcher; keeps the p95
 * history buffers (reading 23).  The stream's next dyq_select_bits
 * (or dyq_policy_step) does not observe its prev_action row: that action
 * belongs to the previous episode (the decision at t uses the actions
 * <= t-1 of the same episode), so the new episode starts like t = 0. */
DYQ_API dyq_status_t dyq_state_reset_episode(void* state, const uint8_t* mask,
                                     dyq_stream_t stream);
/* One control step for every stream: observe a_{t-1} (prev_action, device
 * float [E,7] = [x,y,z, rx,ry,rz, gripper], or NULL at t = 0), update the
 * kinematic proxies M_t and J_t, the windowed means
 * (P:229-231), S_t, bhat_t (Alg. 1 line 2) and b*_t (Alg. 1
 * lines 3-9).  Writes bits[E] (int32 in {2,4,8,16}) and,
 * optionally, S_out[E] (fp64) and target_out[E] (bhat_t).  Bit-exact with the
 * CPU oracle (fp64, fixed evaluation order, no FMA contraction). */
DYQ_API dyq_status_t dyq_select_bits(void* state, int32_t E, const float* prev_action,
                             int32_t* bits, double* S_out, int32_t* target_out,
                             dyq_stream_t stream);
/* dyq_select_bits fused with dyq_route_bits (one kernel per control step):
 * also writes row_bits[e * tokens_per_episode + i] = abits_of(bits[e]) for
 * i < tokens_per_episode.  Same state / outputs / errors as the two calls. */
DYQ_API dyq_status_t dyq_select_route(void* state, int32_t E, const float* prev_action,
                              int32_t* bits, int32_t tokens_per_episode,
                              const int32_t* abits_of_host /* [4] or NULL */, int32_t* row_bits,
                              double* S_out, int32_t* target_out, dyq_stream_t stream);
/* Expand per-episode bits to per-token activation bits through the variant
 * table (DESIGN.md conflict C1): row_bits[m] = abits_of(bits[m / tokens_per_episode]).
 * abits_of maps b* in {2,4,8,16} -> activation bits; pass NULL for identity
 * (the paper's W4-pinned table: W4A2 / W4A4 / W4A8 / W4A16). */
DYQ_API dyq_status_t dyq_route_bits(const int32_t* bits, int32_t E, int32_t tokens_per_episode,
                            const int32_t* abits_of_host /* [4] or NULL */,
                            int32_t* row_bits, dyq_stream_t stream);

/* -------------------------------------------------- activation quantizer */
/* Workspace bytes for dyq_qlinear with M tokens against descriptor wd (holds
 * the quantized activations, their per-group parameters and the split-K
 * partials).  Must be zeroed once before first use (dyq_workspace_init).  A
 * workspace belongs to one weight SHAPE (N, K, group, wbits): it may be reused
 * for every M and every layer of that shape (its split-K tile counters reset
 * themselves), but not shared with another shape, whose layout would overwrite
 * the counters. */
DYQ_API dyq_status_t dyq_qlinear_workspace(const dyq_wdesc_t* wd, int32_t M, size_t* bytes);
DYQ_API dyq_status_t dyq_workspace_init(void* workspace, size_t bytes, dyq_stream_t stream);

/* The launch plan dyq_qlinear / dyq_qlinear_i32_partials use for M rows of
 * this shape (host only, no device work): *path = 1 decode kernel (M <= 16),
 * 2 tcgen05 prefill kernel; *ksplit = K-group split factor of the prefill
 * grid (1 = none; > 1: each split writes fp32 partial tiles reduced in split
 * order, or its own groups of the integer partials).  Either pointer may be
 * NULL.  Lets tests assert which code path a parity case exercised. */
DYQ_API dyq_status_t dyq_qlinear_plan(const dyq_wdesc_t* wd, int32_t M, int32_t* path, int32_t* ksplit);

/* ------------------------------------------------------------- qlinear */
/* y[m,n] = Sum_g s_x[m,g] s_w[n,g] Sum_{k in g} (Xq[m,k]-z_x[m,g]) (q[n,k]-z_w[n,g])
 * for integer rows (row_bits[m] in {2,4,8}); the codes Xq are the dynamic
 * quantization of x[m,:] at row_bits[m] bits (Eq. 2 per (token, group)).
 * For A16 rows (row_bits[m] == 16, the BF16 bypass):
 * y[m,n] = Sum_g s_w[n,g] Sum_{k in g} x[m,k] (q[n,k]-z_w[n,g]).
 *   x         device bf16 [M,K]
 *   row_bits  device int32 [M] (activation bits per token) or NULL -> `bits`
 *   y         device [M,N] (16-byte aligned), y_dtype 0 = fp32, 1 = bf16
 *   workspace device buffer of dyq_qlinear_workspace() bytes (zeroed once)
 * One call reads the packed weights once for any mix of activation widths.
 * M in [0, 65536]; M <= 16 runs the bandwidth-bound decode kernel, larger M
 * the tcgen05 prefill kernel.  Integer group sums are exact (int32); the fp32
 * epilogue order is unspecified (tolerance in DESIGN.md). */
DYQ_API dyq_status_t dyq_qlinear(const dyq_wdesc_t* wd, const void* codes, const void* meta,
                         const uint16_t* x, int32_t M, const int32_t* row_bits,
                         int32_t bits, void* y, int32_t y_dtype, void* workspace,
                         size_t ws_bytes, int64_t* err, dyq_stream_t stream);

/* Split form of dyq_qlinear for callers that reuse one quantized activation
 * for several linears with the same K (e.g. Q/K/V, gate/up: P:334 quantizes
 * once per activation, not per GEMM):
 *   dyq_act_quant  quantizes x [M,K] at row_bits into `workspace` (Eq. 2 per
 *                  (token, group)); the workspace then holds the codes, s_x,
 *                  z_x and SX of this activation;
 *   dyq_qlinear_q  runs the linear layer on those codes (x is still read for
 *                  A16 rows).  Same arguments / semantics as dyq_qlinear.
 * Currently M <= 16 (the decode regime); larger M returns DYQ_EUNSUPPORTED. */
DYQ_API dyq_status_t dyq_act_quant(const dyq_wdesc_t* wd, const uint16_t* x, int32_t M,
                                   const int32_t* row_bits, int32_t bits, void* workspace,
                                   size_t ws_bytes, int64_t* err, dyq_stream_t stream);
DYQ_API dyq_status_t dyq_qlinear_q(const dyq_wdesc_t* wd, const void* codes, const void* meta,
                                   const uint16_t* x, int32_t M, const int32_t* row_bits,
                                   int32_t bits, void* y, int32_t y_dtype, void* workspace,
                                   size_t ws_bytes, dyq_stream_t stream);

/* Asynchronous HBM -> L2 prefetch of `bytes` bytes at device address p
 * (16-byte aligned), e.g. the next layer's packed codes and metadata, issued
 * while the current layer's dependent chain (act-quant -> qlinear) runs.  The
 * packed weights never depend on earlier kernels (weights are frozen),
 * so the transfer overlaps that chain; stream-ordered, no host sync.  A hint
 * only: results never depend on it.  Bytes beyond the L2 capacity (126 MB on
 * B200) evict earlier prefetched lines.  DYQ_EINVAL on a null / misaligned p. */
DYQ_API dyq_status_t dyq_prefetch_l2(const void* p, size_t bytes, dyq_stream_t stream);

/* Test hook: same main loop, writes the exact integer group sums
 * I[m,n,g] (int32 [M,N,K/G]; 0 for A16 rows) instead of y. */
DYQ_API dyq_status_t dyq_qlinear_i32_partials(const dyq_wdesc_t* wd, const void* codes,
                                      const void* meta, const uint16_t* x, int32_t M,
                                      const int32_t* row_bits, int32_t bits,
                                      int32_t* I, void* workspace, size_t ws_bytes,
                                      int64_t* err, dyq_stream_t stream);

/* Test hook: run only the activation quantizer of dyq_qlinear and export its
 * result in logical layout: xq [M,K] u8, sx [M,K/G] fp32, zx [M,K/G] u8,
 * SX [M,K/G] int32 (A16 rows zeroed).  Same kernel as the qlinear path. */
DYQ_API dyq_status_t dyq_act_quant_for_check(const dyq_wdesc_t* wd, const uint16_t* x, int32_t M,
                                     const int32_t* row_bits, int32_t bits, uint8_t* xq,
                                     float* sx, uint8_t* zx, int32_t* SX, void* workspace,
                                     size_t ws_bytes, int64_t* err, dyq_stream_t stream);

/* Force the kernel family (testing / benchmarking): 0 = auto (default),
 * 1 = decode (M <= 64 only), 2 = prefill.  Process-wide. */
DYQ_API dyq_status_t dyq_set_path(int32_t path);

/* dyq_qlinear with device-side masking (the variant table's building block):
 * rows m with row_bits[m] == 0 are not computed into y (y rows left as they
 * were), and if gate != NULL and *gate == 0 at execution time every kernel of
 * the call returns immediately (no weight bytes are read).  row_bits must be
 * non-NULL.  Lets two calls on different weight copies (W4 / W8) share one
 * output, each owning its rows, with the choice made on the device. */
DYQ_API dyq_status_t dyq_qlinear_masked(const dyq_wdesc_t* wd, const void* codes, const void* meta,
                                        const uint16_t* x, int32_t M, const int32_t* row_bits,
                                        const int32_t* gate, void* y, int32_t y_dtype, void* workspace,
                                        size_t ws_bytes, int64_t* err, dyq_stream_t stream);

/* ============================================================ policy step
 * one VLA control step around the quantized linears.  The
 * backbone is OpenVLA's Llama-2: n_vis vision embeddings (synthetic
 * in this repo; the vision encoder is out of scope) + n_text text tokens are
 * prefilled through n_layers blocks
 *   x = RMSNorm(h); qkv = qlinear(x); RoPE(q, k); a = causal attention (KV cache);
 *   h += qlinear_o(a); x = RMSNorm(h); h += qlinear_down(SiLU(g) * u),
 *   [g | u] = qlinear_gate_up(x)
 * then the action head (the LM-head rows of the n_bins action-bin tokens, the
 * last n_bins ids of the vocabulary) + argmax gives the first action token,
 * and n_act - 1 decode passes give the rest (one b* for all tokens of the step,
 * P:346); action value of bin b = -1 + (2b + 1) / n_bins.  Every
 * qlinear runs at the activation bits of the episode's b*_t from
 * dyq_select_bits through the W4-pinned variant table.
 * All buffers are caller-owned (sizes from dyq_model_size); dyq_model_bind
 * makes a host-side handle only (no device allocation). */
typedef struct {
    int32_t n_layers, d, ffn, n_heads, vocab, E; /* E = max episodes per step          */
    int32_t n_vis, n_text, n_act, n_bins;        /* 256, 32, 7, 256 (OpenVLA)           */
    int32_t group, wbits;                        /* packing of every linear             */
    float rms_eps, rope_theta;                   /* 1e-5 (Llama-2: 1e-5), 10000         */
    const void* const* codes;   /* host array [n_layers * 4] of device pointers: qkv, o, gate_up, down */
    const void* const* meta;    /* same order                                           */
    const uint16_t* attn_norm;  /* device bf16 [n_layers, d]                            */
    const uint16_t* mlp_norm;   /* device bf16 [n_layers, d]                            */
    const uint16_t* final_norm; /* device bf16 [d]                                      */
    const uint16_t* embed;      /* device bf16 [vocab, d]                               */
    const uint16_t* head_bins;  /* device bf16 [n_bins, d]: LM-head rows of the bin tokens */
    void* kv;                   /* device, kv_bytes: [E][n_layers][2][T][d] bf16, T = n_vis+n_text+n_act */
    void* scratch;              /* device, scratch_bytes (activations, qlinear workspace, ...)  */
    /* ---- optional (all-zero = the paper's defaults) ----
     * Variant table (P:221 pins the default to INT4): b*_t in
     * {2, 4, 8, 16} (index 0..3) selects a weight copy wbits_of[i] in {4, 8}
     * and activation bits abits_of[i].  A step's rows are routed per episode
     * to the W4 or the W8 copy (codes_w8 / meta_w8: same order as codes,
     * packed with wbits = 8 and the same group); each linear runs once per
     * copy with the other copy's rows masked, and a copy with no live row is
     * skipped on the device (dyq_qlinear_masked) -- a precision switch is a
     * pointer + kernel-variant choice made on the GPU, with no host round trip.
     * wbits_of all 0 -> {4,4,4,4}; abits_of all 0 -> {2,4,8,16}. */
    const void* const* codes_w8; /* host array [n_layers * 4] or NULL (W4 only)        */
    const void* const* meta_w8;
    int32_t wbits_of[4];
    int32_t abits_of[4];
    /* Paper mode (§V-B): 1 = b*_t is selected on a side stream that
     * overlaps the visual prefill (joined by an event before the decode
     * passes); the prefill runs at prefill_bits on the W4 copy, the decode
     * passes at b*_t.  0 (default): b*_t also switches the prefill. */
    int32_t paper_mode;
    int32_t prefill_bits;        /* paper_mode prefill activation bits; 0 -> 16 (BF16) */
} dyq_model_desc_t;
DYQ_API dyq_status_t dyq_model_size(const dyq_model_desc_t* desc, size_t* kv_bytes, size_t* scratch_bytes);
DYQ_API dyq_status_t dyq_model_bind(const dyq_model_desc_t* desc, void** model);
/* zero the scratch (split-K counters) and start new episodes (no prev action) */
DYQ_API dyq_status_t dyq_model_init(void* model, dyq_stream_t stream);
DYQ_API dyq_status_t dyq_model_free(void* model);
/* vis_emb device bf16 [E, n_vis, d]; text_ids device int32 [E, n_text];
 * action_out device f32 [E, n_act]; bits_out device int32 [E] (b*_t) or NULL.
 * state = dyq_select_bits state for >= E streams.  E <= desc.E. */
DYQ_API dyq_status_t dyq_policy_step(void* model, void* state, int32_t E, const uint16_t* vis_emb,
                                     const int32_t* text_ids, float* action_out, int32_t* bits_out,
                                     dyq_stream_t stream);

/* Glue kernels of the policy step, exported for tests (device pointers, bf16 = uint16).
 * h (+)= delta (if delta != NULL, h updated in place); y = RMSNorm(h) * w, rows of d. */
DYQ_API dyq_status_t dyq_add_rmsnorm(uint16_t* h, const uint16_t* delta, const uint16_t* w, int32_t M,
                                     int32_t d, float eps, uint16_t* y, dyq_stream_t stream);
/* in-place rotary embedding of the q and k parts of qkv [M, 3d]; position of
 * row m = (m % rows_per_episode) + pos0 */
DYQ_API dyq_status_t dyq_rope(uint16_t* qkv, int32_t M, int32_t rows_per_episode, int32_t pos0, int32_t d,
                              int32_t n_heads, float theta, dyq_stream_t stream);
/* causal self-attention of E episodes of S tokens (rows e*S + i of qkv / out);
 * also writes K, V rows 0..S-1 of layer `layer` into the cache */
DYQ_API dyq_status_t dyq_attention_prefill(const uint16_t* qkv, int32_t E, int32_t S, int32_t d,
                                           int32_t n_heads, uint16_t* kv, int32_t layer, int32_t n_layers,
                                           int32_t T, uint16_t* out, dyq_stream_t stream);
/* one new token per episode at position pos: writes its K, V into the cache,
 * attends over cache positions 0..pos */
DYQ_API dyq_status_t dyq_attention_decode(const uint16_t* qkv, int32_t E, int32_t pos, int32_t d,
                                          int32_t n_heads, uint16_t* kv, int32_t layer, int32_t n_layers,
                                          int32_t T, uint16_t* out, dyq_stream_t stream);
/* dyq_rope (rows_per_episode = 1, pos0 = pos) of the q and k parts followed by
 * dyq_attention_decode, in one kernel: the rotated k goes into the cache, qkv
 * is left unrotated; bit-identical to the two calls.  qkv and kv 16-B aligned
 * and d % 8 == 0, else DYQ_EUNSUPPORTED (nothing launched). */
DYQ_API dyq_status_t dyq_attention_decode_rope(const uint16_t* qkv, int32_t E, int32_t pos, int32_t d,
                                               int32_t n_heads, float theta, uint16_t* kv, int32_t layer,
                                               int32_t n_layers, int32_t T, uint16_t* out, dyq_stream_t stream);
/* act[m, j] = SiLU(gu[m, j]) * gu[m, ffn + j] */
DYQ_API dyq_status_t dyq_silu_mul(const uint16_t* gu, int32_t M, int32_t ffn, uint16_t* act,
                                  dyq_stream_t stream);
/* logits[e, b] = x[e*row_stride] . head_bins[b] (fp32); tok[e*tok_stride] = argmax_b (lowest b on ties) */
DYQ_API dyq_status_t dyq_head_argmax(const uint16_t* x, int32_t E, int32_t row_stride, int32_t d,
                                     const uint16_t* head_bins, int32_t n_bins, float* logits, int32_t* tok,
                                     int32_t tok_stride, dyq_stream_t stream);

/* ====================================================== tensor parallelism
 * SURVEY.md §8(a) A8 / BASELINE config 5 (not in the paper): column (N)
 * sharding of every quantized linear across the GPUs of one node.  Rank r packs
 * rows [n0, n1) = dyq_tp_shard(N, P, r) of the weight (K-groups never span
 * ranks, so the shard's pack equals the row slice of the full pack), runs
 * dyq_qlinear into y_shard [M, N/P] bf16, and dyq_tp_allgather joins the shards
 * with an NCCL all-gather over NVLink (NCCL is dlopen'ed: libnccl.so.2, or the
 * path in $DYQ_NCCL_LIB) plus a column interleave. */
DYQ_API dyq_status_t dyq_tp_shard(int32_t N, int32_t world, int32_t rank, int32_t* n0, int32_t* n1);
/* id_host: host buffer of 128 bytes (ncclUniqueId), created on one rank and
 * broadcast by the caller (e.g. over the torch process group). */
DYQ_API dyq_status_t dyq_comm_unique_id(void* id_host);
DYQ_API dyq_status_t dyq_comm_init(const void* id_host, int32_t rank, int32_t world, void** comm);
DYQ_API dyq_status_t dyq_comm_destroy(void* comm);
/* y [M, N] bf16 (every rank) <- concat_r y_shard_r [M, N/P]; gather_buf device
 * [P, M, N/P] bf16 (unused, may be NULL, when M == 1).  N % (16 P) == 0. */
DYQ_API dyq_status_t dyq_tp_allgather(void* comm, const uint16_t* y_shard, int32_t M, int32_t N,
                                      uint16_t* gather_buf, uint16_t* y, dyq_stream_t stream);
/* the interleave step alone: y[m, r Ns + j] = buf[r, m, j] (Ns % 8 == 0) */
DYQ_API dyq_status_t dyq_tp_interleave(const uint16_t* buf, int32_t P, int32_t M, int32_t Ns, uint16_t* y,
                                       dyq_stream_t stream);

/* -------------------------- fused tensor-parallel decode epilogue (NEXT-1) */
/* The all-gather of the column shards folded into the decode kernel: rank r's
 * epilogue stores y[:, r Ns + j] (bf16) straight into EVERY rank's full output
 * y[p] ([M, world * Ns], peer memory over NVLink / NVSwitch, mapped with
 * dyq_ipc_open); each CTA then fences at system scope and adds the number of
 * 16-column sub-tiles it wrote to every rank's flag[p].  One call adds
 * dyq_tp_flag_delta(N, M) to every flag once all ranks' parts have landed
 * (N / 16 for decode, M <= 16; N / 16 per 144-token tile for the tcgen05
 * prefill path); dyq_tp_wait orders a rank's stream after the running total.
 * Consecutive calls must alternate between two y buffers (a peer may start
 * call c+1 while this rank still reads call c's output).  Both regimes:
 * decode (M <= 16, one launch) and prefill (M > 16).
 * wd = this rank's shard descriptor (N = Ns, dyq_tp_shard rows). */
#define DYQ_TP_MAX 8
typedef struct {
    int32_t world, rank;
    void* y[DYQ_TP_MAX];        /* rank p's full y as mapped in this process   */
    uint64_t* flag[DYQ_TP_MAX]; /* rank p's arrival counter (u64, zeroed once) */
} dyq_tp_peers_t;
DYQ_API dyq_status_t dyq_qlinear_tp(const dyq_wdesc_t* wd, const void* codes, const void* meta,
                                    const uint16_t* x, int32_t M, const int32_t* row_bits, int32_t bits,
                                    const dyq_tp_peers_t* peers, void* workspace, size_t ws_bytes,
                                    int64_t* err, dyq_stream_t stream);
/* Per-call flag increment of dyq_qlinear_tp for full width N and M tokens. */
DYQ_API dyq_status_t dyq_tp_flag_delta(int32_t N, int32_t M, uint64_t* delta);
/* Stream-ordered wait until *flag >= target (device u64, ld.acquire.sys).
 * Bounded: after 10 s the kernel sets *timed_out = 1 (device int32, may be
 * NULL) and returns rather than hang the GPU. */
DYQ_API dyq_status_t dyq_tp_wait(const uint64_t* flag, uint64_t target, int32_t* timed_out,
                                 dyq_stream_t stream);
/* CUDA IPC of device buffers, for peer y / flag buffers of other processes.
 * A handle (64 B) names the whole allocation holding dev_ptr (e.g. a caching
 * allocator segment); offset_out = dev_ptr - allocation base.  The caller
 * exchanges (handle, offset) (e.g. over the torch process group); dyq_ipc_open
 * returns the peer's dev_ptr in this process.  One open per peer allocation
 * (CUDA refuses to map the same allocation twice): keep a rank's y buffers and
 * flag in one allocation.  dyq_ipc_close(ptr, offset) unmaps. */
DYQ_API dyq_status_t dyq_ipc_handle(void* dev_ptr, void* handle_out, uint64_t* offset_out);
DYQ_API dyq_status_t dyq_ipc_open(const void* handle, uint64_t offset, void** dev_ptr);
DYQ_API dyq_status_t dyq_ipc_close(void* dev_ptr, uint64_t offset);

/* ------------------------------------------- offline threshold calibration */
/* PAPER.md §IV-B: eps_a(S) = D_acc / (S + eta); Eq. (5)
 * minimal bits under the bound; Theta = {theta_24, theta_48} from
 * calibration trajectories, in SPEC's binned isotonic reading
 * with DESIGN.md readings C1-C6.
 *
 * Forced-bits policy step: like dyq_policy_step, but episode e runs at the
 * given b*_t = bits[e] (device int32 [E], values in {2,4,8,16}) and no
 * selection state is read or updated. */
DYQ_API dyq_status_t dyq_policy_step_bits(void* model, int32_t E, const int32_t* bits, const uint16_t* vis_emb,
                                          const int32_t* text_ids, float* action_out, dyq_stream_t stream);
/* One calibration step for Ec control streams ("executing the
 * full-precision model on a representative calibration subset"):
 *   1. S_t of every stream from a*_{t-1} (dyq_select_bits on `state`, >= Ec
 *      streams; NULL action at the model's first step) -> S_out (device f64 [Ec]);
 *   2. ONE batched policy step over 4 Ec replicas of the observations
 *      (vis_emb [Ec, n_vis, d], text_ids [Ec, n_text]) at b = 16 | 2 | 4 | 8:
 *      actions_out (device f32 [4 Ec, n_act]) rows [0, Ec) = a*_t (BF16 path,
 *      which the next step's S observes), rows [(j+1) Ec, (j+2) Ec) = a^(b_j);
 *   3. err_out (device f64 [Ec, 3]) = || a^(b) - a* ||_2, b = 2, 4, 8.
 * Requires 4 Ec <= desc.E.  The counterfactual actions never drive the
 * trajectory (the environment steps with a*). */
DYQ_API dyq_status_t dyq_calib_collect(void* model, void* state, int32_t Ec, const uint16_t* vis_emb,
                                       const int32_t* text_ids, float* actions_out, double* S_out,
                                       double* err_out, dyq_stream_t stream);
/* err_out[e, j] = || a[(j+1) Ec + e, :] - a[e, :] ||_2 (fp64, j = 0..2), a
 * device f32 [4 Ec, n_act]: step 3 of dyq_calib_collect on its own. */
DYQ_API dyq_status_t dyq_calib_errors(const float* actions, int32_t Ec, int32_t n_act, double* err_out,
                                      dyq_stream_t stream);
/* Derive Theta (HOST pointers; offline).  S host f64 [n], err host f64 [n, 3]
 * = (e^(2), e^(4), e^(8)) per step.  calib: reads theta_fp, D_acc, eta (> 0),
 * writes theta_24 <= theta_48 <= theta_fp; other fields untouched.
 *   - samples with S outside [0, theta_fp] are ignored (BF16 steps);
 *   - n_bins uniform bins on [0, theta_fp] (SPEC: 32); mean e^(2), e^(4) per
 *     bin; bins with >= n_min samples (SPEC: 50) get a count-weighted
 *     isotonic (non-decreasing) fit, the others are interpolated between
 *     covered neighbours (coverage warning: *n_undercovered);
 *   - theta_24 = lower edge of the first bin whose smoothed e^(2) exceeds
 *     eps_a at the bin's upper edge, else theta_fp; theta_48 likewise with
 *     e^(4), raised to theta_24 if below.
 * Optional outputs (NULL to skip): smoothed [2, n_bins], counts [n_bins].
 * Errors: DYQ_EINVAL for n <= 0, bad parameters, or no bin with n_min samples.
 * Deterministic: sequential fp64 sums in sample order. */
DYQ_API dyq_status_t dyq_calib_derive(const double* S, const double* err, int64_t n, int32_t n_bins,
                                      int32_t n_min, dyq_calib_t* calib, double* smoothed,
                                      int64_t* counts, int32_t* n_undercovered);
/* Audit a table on (held-out) samples (HOST pointers): a sample
 * with S in [0, theta_fp] runs b = Phi(S) (Eq. (6)) and is satisfied iff
 * e^(b) <= eps_a(S); others run BF16 and are satisfied.  n_quant = samples in
 * the quantized domain, n_ok = satisfied samples (of n), worst [n_bins]
 * (or NULL) = per-bin max e^(b) / eps_a(S), 0 for empty bins.  n = 0 is
 * valid (zero counts).  DYQ_EINVAL if the thresholds are not ordered. */
DYQ_API dyq_status_t dyq_calib_validate(const dyq_calib_t* calib, const double* S, const double* err,
                                        int64_t n, int32_t n_bins, int64_t* n_quant, int64_t* n_ok,
                                        double* worst);

#ifdef __cplusplus
}
#endif
#endif /* DYQ_H */
