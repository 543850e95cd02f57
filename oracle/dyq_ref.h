/*
 * dyq_ref.h -- CPU ORACLE for the DyQ-VLA qlinear hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library.  The product path (paper_2603_07904_b200)
 * never includes, links or calls it; it shares no code, header, table or helper
 * with the CUDA library (include/dyq.h).
 *
 * Every function restates a passage of /root/reference/PAPER.md (P:line) or of
 * SPEC.md (S:line); readings where the paper is silent are the §8(c) readings
 * listed in DESIGN.md §"Readings".  Host pointers, synchronous errors.
 *
 * Return codes: 0 ok, 1 invalid argument, 2 shape error, 4 non-finite input
 * (index written to *bad_index).
 */
#ifndef DYQ_REF_H
#define DYQ_REF_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* O1 fit (S:43-51 + readings 2,3): zero-inclusive min-max, fp64 fit, fp32 stored
 * scale, half-up zero point computed from the fp64 scale. */
int dyq_ref_quant_fit(const double* v, int64_t n, int bits, float* s_out,
                      uint8_t* z_out, int64_t* bad_index);

/* O2 quantize, Eq. (2): q = clamp(floor(v/s) + z, 0, 2^b-1),
 * floor of the fp64 quotient of the fp32 operands; round_mode 1 = nearest. */
void dyq_ref_quantize(const double* v, int64_t n, float s, uint8_t z, int bits,
                      int round_mode, uint8_t* q);

/* O3 dequantize: xhat = s*(q-z), fp64. */
void dyq_ref_dequantize(const uint8_t* q, int64_t n, float s, uint8_t z,
                        double* xhat);

/* O4 pack (reading 5): per (row n, group g of G consecutive k).
 * w_bf16: [N,K] bf16 bit patterns.  Outputs in LOGICAL layout:
 * q [N*K] codes, s [N*K/G], z [N*K/G], sumq [N*K/G] (Sum_k q, for checks). */
int dyq_ref_pack_weights(int32_t N, int32_t K, int32_t G, int32_t wbits,
                         int32_t round_mode, const uint16_t* w_bf16, uint8_t* q,
                         float* s, uint8_t* z, int32_t* sumq, int64_t* bad_index);

/* O5 act-quant (reading 6): per (token m, group g) at abits[m] in
 * {2,4,8}; abits[m]==16 leaves the row unquantized (q,s,z,SX rows zeroed).
 * SX[m,g] = Sum_{k in g} Xq. */
int dyq_ref_act_quant(int32_t M, int32_t K, int32_t G, const int32_t* abits,
                      int32_t round_mode, const uint16_t* x_bf16, uint8_t* xq,
                      float* sx, uint8_t* zx, int32_t* SX, int64_t* bad_index);

/* O6 qlinear: for integer rows
 *   I[m,n,g] = Sum_{k in g} (Xq[m,k]-zx[m,g]) * (q[n,k]-zw[n,g])   (int64, exact)
 *   y[m,n]   = Sum_g (double)sx[m,g] * (double)sw[n,g] * I[m,n,g]  (fp64)
 * for A16 rows (reading 9):
 *   y[m,n]   = Sum_g (double)sw[n,g] * Sum_k (double)x[m,k] * (q[n,k]-zw[n,g]).
 * I (may be NULL) is [M,N,K/G] int32 (A16 rows: 0).  y is [M,N] fp64. */
int dyq_ref_qlinear(int32_t M, int32_t N, int32_t K, int32_t G,
                    const int32_t* abits, const uint16_t* x_bf16,
                    const uint8_t* xq, const float* sx, const uint8_t* zx,
                    const uint8_t* q, const float* sw, const uint8_t* zw,
                    double* y, int32_t* I);

/* O7 kinematic bit selection (P:175-177, P:228-234, P:236-250, P:288-296,
 * Alg. 1).  Opaque per-stream state. */
typedef struct {
    double theta_24, theta_48, theta_fp, lambda, D_acc, eta, J_cap;
    int32_t K, W_macro, W_micro, H, clamp_M;
} dyq_ref_calib_t;

void* dyq_ref_state_new(int32_t E, const dyq_ref_calib_t* calib);
void  dyq_ref_state_free(void* st);
/* episode reset (reading 23): clears windows, prev_rot, warm-up counter and the
 * dispatcher (16,0,16); keeps the p95 history buffers; the stream's next
 * select_bits does not observe its prev_action row (the previous episode's
 * last action).  mask may be NULL (all). */
void  dyq_ref_state_reset_episode(void* st, const uint8_t* mask);
/* One control step for all E streams.  prev_action [E,7] = a_{t-1} (NULL at
 * t = 0: nothing observed).  Outputs (each may be NULL): bits [E] = b*_t,
 * target [E] = bhat_t, S [E], Mbar [E], Jbar [E]. */
int dyq_ref_select_bits(void* st, const float* prev_action, int32_t* bits,
                        int32_t* target, double* S, double* Mbar, double* Jbar);
/* O8: Eq. (4) literal over a target sequence. */
void dyq_ref_eq4(const int32_t* targets, int32_t T, int32_t K, int32_t init,
                 int32_t* out);
/* Alg. 1 alone over a target sequence from state (b*,c,bbar) = init. */
void dyq_ref_alg1(const int32_t* targets, int32_t T, int32_t K, int32_t init_b,
                  int32_t init_c, int32_t init_bbar, int32_t* out,
                  int32_t* counter_out);
/* Eq. (6) lookup and Alg. 1 line 2. */
int32_t dyq_ref_phi(double S, double theta_24, double theta_48);
int32_t dyq_ref_target_bits(double S, int warmup, double theta_24,
                            double theta_48, double theta_fp);
/* nearest-rank percentile (reading 14): sorted[(pct*n + 99)/100 - 1] */
double dyq_ref_percentile(const double* v, int32_t n, int32_t pct);
/* bytes of per-stream state (Table IV analogue) */
int64_t dyq_ref_state_bytes_per_stream(const dyq_ref_calib_t* calib);

#ifdef __cplusplus
}
#endif
#endif
