/*
 * dyq_ref.c -- plain, slow, obviously-correct CPU ORACLE for DyQ-VLA's qlinear
 * hot path.  TEST INFRASTRUCTURE ONLY (see dyq_ref.h): not part of the product.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC (no FMA
 * contraction: reading 24 requires the kinematic arithmetic to be evaluated
 * exactly in the written order).
 *
 * Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n.
 */
#include "dyq_ref.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static double bf16_to_double(uint16_t h) {
    uint32_t u = ((uint32_t)h) << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return (double)f;
}

static int is_finite_d(double v) { return !isnan(v) && !isinf(v); }

/* ------------------------------------------------------------------------- */
/* O1: fit.  SPEC S:46 gives scale = max(max-min, eps)/(2^b-1) and
 * z = clamp(round(-min/scale)).  Readings: the range is made
 * zero-inclusive (lo = min(min,0), hi = max(max,0)) so the S:81 bound holds and
 * 0 maps to an exact code; the fit runs in fp64 (reproduces S:51's z = 128);
 * the scale is stored as fp32; z rounds half-up from the fp64 scale.          */
int dyq_ref_quant_fit(const double* v, int64_t n, int bits, float* s_out,
                      uint8_t* z_out, int64_t* bad_index) {
    if (bits != 2 && bits != 4 && bits != 8) return 1;
    if (n <= 0) return 2;
    double lo = 0.0, hi = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        if (!is_finite_d(v[i])) {
            if (bad_index) *bad_index = i;
            return 4;
        }
        if (v[i] < lo) lo = v[i];
        if (v[i] > hi) hi = v[i];
    }
    const double levels = (double)((1 << bits) - 1);
    double R = hi - lo;
    if (R < 1e-8) R = 1e-8; /* eps_range */
    const double s64 = R / levels;
    const double zr = -lo / s64;
    const double fl = floor(zr);
    double zq = fl + ((zr - fl) >= 0.5 ? 1.0 : 0.0); /* round half up */
    if (zq < 0.0) zq = 0.0;
    if (zq > levels) zq = levels;
    *s_out = (float)s64;
    *z_out = (uint8_t)zq;
    return 0;
}

/* O2: Eq. (2): Q(X) = clamp(floor(X/s) + z, 0, 2^b - 1). */
void dyq_ref_quantize(const double* v, int64_t n, float s, uint8_t z, int bits,
                      int round_mode, uint8_t* q) {
    const double levels = (double)((1 << bits) - 1);
    for (int64_t i = 0; i < n; ++i) {
        double r = v[i] / (double)s;
        double f = round_mode == 1 ? floor(r + 0.5) : floor(r);
        double c = f + (double)z;
        if (c < 0.0) c = 0.0;
        if (c > levels) c = levels;
        q[i] = (uint8_t)c;
    }
}

/* O3: P:106, Xhat = s (Q(X) - z). */
void dyq_ref_dequantize(const uint8_t* q, int64_t n, float s, uint8_t z,
                        double* xhat) {
    for (int64_t i = 0; i < n; ++i) xhat[i] = (double)s * ((double)q[i] - (double)z);
}

/* O4: weights frozen at wbits, one (s,z) per row and per group
 * of G consecutive input channels (reading 5). */
int dyq_ref_pack_weights(int32_t N, int32_t K, int32_t G, int32_t wbits,
                         int32_t round_mode, const uint16_t* w_bf16, uint8_t* q,
                         float* s, uint8_t* z, int32_t* sumq, int64_t* bad_index) {
    if (wbits != 4 && wbits != 8) return 1;
    if (N <= 0 || K <= 0 || G <= 0 || K % G) return 2;
    const int32_t NG = K / G;
    double* buf = (double*)malloc(sizeof(double) * (size_t)G);
    if (!buf) return 1;
    for (int32_t n = 0; n < N; ++n) {
        for (int32_t g = 0; g < NG; ++g) {
            const int64_t base = (int64_t)n * K + (int64_t)g * G;
            for (int32_t k = 0; k < G; ++k) buf[k] = bf16_to_double(w_bf16[base + k]);
            int64_t bi = -1;
            int rc = dyq_ref_quant_fit(buf, G, wbits, &s[(int64_t)n * NG + g],
                                       &z[(int64_t)n * NG + g], &bi);
            if (rc) {
                if (bad_index) *bad_index = base + bi;
                free(buf);
                return rc;
            }
            dyq_ref_quantize(buf, G, s[(int64_t)n * NG + g], z[(int64_t)n * NG + g],
                             wbits, round_mode, &q[base]);
            if (sumq) {
                int32_t acc = 0;
                for (int32_t k = 0; k < G; ++k) acc += q[base + k];
                sumq[(int64_t)n * NG + g] = acc;
            }
        }
    }
    free(buf);
    return 0;
}

/* O5: dynamic activation quantization at the step's width,
 * per (token, group) (reading 6); abits == 16 is the BF16 bypass. */
int dyq_ref_act_quant(int32_t M, int32_t K, int32_t G, const int32_t* abits,
                      int32_t round_mode, const uint16_t* x_bf16, uint8_t* xq,
                      float* sx, uint8_t* zx, int32_t* SX, int64_t* bad_index) {
    if (M < 0 || K <= 0 || G <= 0 || K % G) return 2;
    const int32_t NG = K / G;
    double* buf = (double*)malloc(sizeof(double) * (size_t)G);
    if (!buf) return 1;
    for (int32_t m = 0; m < M; ++m) {
        const int32_t b = abits[m];
        if (b != 2 && b != 4 && b != 8 && b != 16) {
            free(buf);
            return 1;
        }
        for (int32_t g = 0; g < NG; ++g) {
            const int64_t base = (int64_t)m * K + (int64_t)g * G;
            const int64_t mg = (int64_t)m * NG + g;
            for (int32_t k = 0; k < G; ++k) buf[k] = bf16_to_double(x_bf16[base + k]);
            if (b == 16) {
                for (int32_t k = 0; k < G; ++k) {
                    if (!is_finite_d(buf[k])) {
                        if (bad_index) *bad_index = base + k;
                        free(buf);
                        return 4;
                    }
                    xq[base + k] = 0;
                }
                sx[mg] = 0.0f;
                zx[mg] = 0;
                SX[mg] = 0;
                continue;
            }
            int64_t bi = -1;
            int rc = dyq_ref_quant_fit(buf, G, b, &sx[mg], &zx[mg], &bi);
            if (rc) {
                if (bad_index) *bad_index = base + bi;
                free(buf);
                return rc;
            }
            dyq_ref_quantize(buf, G, sx[mg], zx[mg], b, round_mode, &xq[base]);
            int32_t acc = 0;
            for (int32_t k = 0; k < G; ++k) acc += xq[base + k];
            SX[mg] = acc;
        }
    }
    free(buf);
    return 0;
}

/* O6: the quantized linear layer.  Per group the integer product of the
 * zero-point-centred codes (Xhat = s (Q - z), on both operands) is
 * accumulated exactly, then dequantized by s_x * s_w in fp64.                */
int dyq_ref_qlinear(int32_t M, int32_t N, int32_t K, int32_t G,
                    const int32_t* abits, const uint16_t* x_bf16,
                    const uint8_t* xq, const float* sx, const uint8_t* zx,
                    const uint8_t* q, const float* sw, const uint8_t* zw,
                    double* y, int32_t* I) {
    if (M < 0 || N <= 0 || K <= 0 || G <= 0 || K % G) return 2;
    const int32_t NG = K / G;
    for (int32_t m = 0; m < M; ++m) {
        const int a16 = abits[m] == 16;
        for (int32_t n = 0; n < N; ++n) {
            double acc = 0.0;
            for (int32_t g = 0; g < NG; ++g) {
                const int64_t wg = (int64_t)n * NG + g;
                const int64_t ag = (int64_t)m * NG + g;
                const int64_t wk = (int64_t)n * K + (int64_t)g * G;
                const int64_t xk = (int64_t)m * K + (int64_t)g * G;
                if (a16) {
                    double d = 0.0;
                    for (int32_t k = 0; k < G; ++k)
                        d += bf16_to_double(x_bf16[xk + k]) *
                             ((double)q[wk + k] - (double)zw[wg]);
                    acc += (double)sw[wg] * d;
                    if (I) I[((int64_t)m * N + n) * NG + g] = 0;
                } else {
                    int64_t s = 0;
                    for (int32_t k = 0; k < G; ++k)
                        s += ((int64_t)xq[xk + k] - (int64_t)zx[ag]) *
                             ((int64_t)q[wk + k] - (int64_t)zw[wg]);
                    acc += (double)sx[ag] * (double)sw[wg] * (double)s;
                    if (I) I[((int64_t)m * N + n) * NG + g] = (int32_t)s;
                }
            }
            y[(int64_t)m * N + n] = acc;
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* O7: kinematic proxies -> S_t -> bhat_t -> Alg. 1.                           */

typedef struct {
    double* mag;   /* ring of ||a^xyz||, capacity H ("historical magnitudes") */
    double* jerk;  /* ring of ||a^rot_t - a^rot_{t-1}||                     */
    int32_t hist_n, hist_pos;
    double* Mwin;  /* last W_macro values of M_i */
    double* Jwin;  /* last W_micro values of J_i */
    int32_t Mwin_n, Mwin_pos, Jwin_n, Jwin_pos;
    double prev_rot[3];
    int32_t steps_seen; /* observations since (re)start; warm-up while < W_macro */
    int32_t skip_next;  /* set by an episode reset: the next a_{t-1} is the previous
                         * episode's last action and is not observed (reading 23;
                         * the decision at t uses actions <= t-1 of THIS episode) */
    int32_t bstar, c, bbar; /* Alg. 1 state */
} ref_stream_t;

typedef struct {
    int32_t E;
    dyq_ref_calib_t cal;
    ref_stream_t* s;
} ref_state_t;

static void stream_reset_episode(ref_stream_t* s) {
    s->Mwin_n = s->Mwin_pos = s->Jwin_n = s->Jwin_pos = 0;
    s->prev_rot[0] = s->prev_rot[1] = s->prev_rot[2] = 0.0;
    s->steps_seen = 0;
    s->bstar = 16; s->c = 0; s->bbar = 16; /* S:254 safe cold start */
}

static void stream_new_episode(ref_stream_t* s) {
    stream_reset_episode(s);
    s->skip_next = 1;
}

void* dyq_ref_state_new(int32_t E, const dyq_ref_calib_t* cal) {
    if (E <= 0 || !cal || cal->H <= 0 || cal->W_macro <= 0 || cal->W_micro <= 0 ||
        cal->K < 1)
        return NULL;
    ref_state_t* st = (ref_state_t*)calloc(1, sizeof *st);
    st->E = E;
    st->cal = *cal;
    st->s = (ref_stream_t*)calloc((size_t)E, sizeof(ref_stream_t));
    for (int32_t e = 0; e < E; ++e) {
        ref_stream_t* s = &st->s[e];
        s->mag = (double*)calloc((size_t)cal->H, sizeof(double));
        s->jerk = (double*)calloc((size_t)cal->H, sizeof(double));
        s->Mwin = (double*)calloc((size_t)cal->W_macro, sizeof(double));
        s->Jwin = (double*)calloc((size_t)cal->W_micro, sizeof(double));
        s->hist_n = s->hist_pos = 0;
        stream_reset_episode(s);
    }
    return st;
}

void dyq_ref_state_free(void* p) {
    ref_state_t* st = (ref_state_t*)p;
    if (!st) return;
    for (int32_t e = 0; e < st->E; ++e) {
        free(st->s[e].mag); free(st->s[e].jerk);
        free(st->s[e].Mwin); free(st->s[e].Jwin);
    }
    free(st->s);
    free(st);
}

void dyq_ref_state_reset_episode(void* p, const uint8_t* mask) {
    ref_state_t* st = (ref_state_t*)p;
    for (int32_t e = 0; e < st->E; ++e)
        if (!mask || mask[e]) stream_new_episode(&st->s[e]);
}

static int cmp_double(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

/* Nearest-rank percentile: k = ceil(pct*n/100) = (pct*n+99)/100,
 * value = k-th smallest.  The oracle sorts a copy (qsort is the library step). */
double dyq_ref_percentile(const double* v, int32_t n, int32_t pct) {
    if (n <= 0) return 0.0;
    double* tmp = (double*)malloc(sizeof(double) * (size_t)n);
    memcpy(tmp, v, sizeof(double) * (size_t)n);
    qsort(tmp, (size_t)n, sizeof(double), cmp_double);
    int32_t k = (pct * n + 99) / 100;
    if (k < 1) k = 1;
    double r = tmp[k - 1];
    free(tmp);
    return r;
}

/* Eq. (6): boundaries belong to the lower-bit interval. */
int32_t dyq_ref_phi(double S, double t24, double t48) {
    if (S <= t24) return 2;
    if (S <= t48) return 4;
    return 8;
}

/* Alg. 1 line 2 with the warm-up rule. */
int32_t dyq_ref_target_bits(double S, int warmup, double t24, double t48, double tfp) {
    if (warmup) return 16;
    if (S > tfp) return 16;
    return dyq_ref_phi(S, t24, t48);
}

/* Alg. 1 lines 3-9, one step; indicator products written out. */
static int32_t alg1_step(int32_t bhat, int32_t K, int32_t* bstar, int32_t* c,
                         int32_t* bbar) {
    if (bhat >= *bstar) { /* line 3-4 */
        *bstar = bhat; *c = 0; *bbar = bhat;
    } else {
        const int32_t bbar_prev = *bbar, c_prev = *c;
        /* line 6: bbar_t = max(bhat, bbar_{t-1} * I(c_{t-1} > 0)) */
        int32_t carried = c_prev > 0 ? bbar_prev : 0;
        int32_t nb = bhat > carried ? bhat : carried;
        /* line 7: c_t = c_{t-1} * I(bbar_t = bbar_{t-1}) + 1 */
        int32_t nc = c_prev * (nb == bbar_prev ? 1 : 0) + 1;
        /* line 8: b*_t = bbar_t I(c_t = K) + b*_{t-1} I(c_t < K); c_t mod K */
        int32_t ns = nc == K ? nb : *bstar;
        *bstar = ns; *c = nc % K; *bbar = nb;
    }
    return *bstar;
}

void dyq_ref_alg1(const int32_t* targets, int32_t T, int32_t K, int32_t init_b,
                  int32_t init_c, int32_t init_bbar, int32_t* out,
                  int32_t* counter_out) {
    int32_t b = init_b, c = init_c, bb = init_bbar;
    for (int32_t t = 0; t < T; ++t) {
        out[t] = alg1_step(targets[t], K, &b, &c, &bb);
        if (counter_out) counter_out[t] = c;
    }
}

/* O8: Eq. (4) literally; fewer than K targets -> hold. */
void dyq_ref_eq4(const int32_t* targets, int32_t T, int32_t K, int32_t init,
                 int32_t* out) {
    int32_t prev = init;
    for (int32_t t = 0; t < T; ++t) {
        int32_t bh = targets[t];
        int32_t b;
        if (bh >= prev) {
            b = bh;
        } else if (t + 1 >= K) {
            int32_t mx = targets[t];
            for (int32_t i = t - K + 1; i <= t; ++i) if (targets[i] > mx) mx = targets[i];
            b = mx <= bh ? bh : prev;
        } else {
            b = prev;
        }
        out[t] = b;
        prev = b;
    }
}

static double window_mean(const double* w, int32_t cap, int32_t n, int32_t pos) {
    /* arithmetic mean over the window contents, summed oldest -> newest
     * ("partial windows average over what exists") */
    if (n == 0) return 0.0;
    int32_t start = (pos - n + cap) % cap;
    double sum = 0.0;
    for (int32_t i = 0; i < n; ++i) sum = sum + w[(start + i) % cap];
    return sum / (double)n;
}

int dyq_ref_select_bits(void* p, const float* prev_action, int32_t* bits,
                        int32_t* target, double* S_out, double* Mbar_out,
                        double* Jbar_out) {
    ref_state_t* st = (ref_state_t*)p;
    const dyq_ref_calib_t* c = &st->cal;
    for (int32_t e = 0; e < st->E; ++e) {
        ref_stream_t* s = &st->s[e];
        const int skip = s->skip_next;
        s->skip_next = 0;
        if (prev_action && !skip) {
            const float* a = prev_action + (int64_t)e * 7;
            const double x = a[0], y = a[1], z = a[2];
            const double r0 = a[3], r1 = a[4], r2 = a[5];
            for (int i = 0; i < 6; ++i)
                if (!is_finite_d((double)a[i])) return 4;
            /* ||a^xyz||_2, evaluated left to right, no contraction */
            const double mag = sqrt(x * x + y * y + z * z);
            /* ||a^rot_t - a^rot_{t-1}||_2; first observation: 0 (reading 16) */
            double jerk = 0.0;
            if (s->steps_seen > 0) {
                const double d0 = r0 - s->prev_rot[0];
                const double d1 = r1 - s->prev_rot[1];
                const double d2 = r2 - s->prev_rot[2];
                jerk = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
            }
            s->prev_rot[0] = r0; s->prev_rot[1] = r1; s->prev_rot[2] = r2;
            s->mag[s->hist_pos] = mag;
            s->jerk[s->hist_pos] = jerk;
            s->hist_pos = (s->hist_pos + 1) % c->H;
            if (s->hist_n < c->H) s->hist_n++;
            /* mu_max, nu_max: 95th percentiles of the history,
             * eps-floored at 1e-6 */
            double mu = dyq_ref_percentile(s->mag, s->hist_n, 95);
            double nu = dyq_ref_percentile(s->jerk, s->hist_n, 95);
            if (mu < 1e-6) mu = 1e-6;
            if (nu < 1e-6) nu = 1e-6;
            /* M_t = 1 - ||a^xyz||/mu_max, clamped to [0,1] */
            double M = 1.0 - mag / mu;
            if (c->clamp_M) {
                if (M < 0.0) M = 0.0;
                if (M > 1.0) M = 1.0;
            }
            /* J_t = ||drot||/nu_max, capped at J_cap */
            double J = jerk / nu;
            if (J > c->J_cap) J = c->J_cap;
            s->Mwin[s->Mwin_pos] = M;
            s->Mwin_pos = (s->Mwin_pos + 1) % c->W_macro;
            if (s->Mwin_n < c->W_macro) s->Mwin_n++;
            s->Jwin[s->Jwin_pos] = J;
            s->Jwin_pos = (s->Jwin_pos + 1) % c->W_micro;
            if (s->Jwin_n < c->W_micro) s->Jwin_n++;
            s->steps_seen++;
        }
        /* windowed means and the fused sensitivity */
        const double Mbar = window_mean(s->Mwin, c->W_macro, s->Mwin_n, s->Mwin_pos);
        const double Jbar = window_mean(s->Jwin, c->W_micro, s->Jwin_n, s->Jwin_pos);
        const double lam_term = c->lambda * Mbar;
        const double one_minus = 1.0 - c->lambda;
        const double jer_term = one_minus * Jbar;
        double S = lam_term + jer_term;
        if (S < 0.0) S = 0.0;
        const int warm = s->steps_seen < c->W_macro;
        const int32_t bhat = dyq_ref_target_bits(S, warm, c->theta_24, c->theta_48, c->theta_fp);
        const int32_t b = alg1_step(bhat, c->K, &s->bstar, &s->c, &s->bbar);
        if (bits) bits[e] = b;
        if (target) target[e] = bhat;
        if (S_out) S_out[e] = S;
        if (Mbar_out) Mbar_out[e] = Mbar;
        if (Jbar_out) Jbar_out[e] = Jbar;
    }
    return 0;
}

int64_t dyq_ref_state_bytes_per_stream(const dyq_ref_calib_t* c) {
    /* history rings + windows + prev_rot (fp64) + counters (int32) */
    return (int64_t)(2 * c->H + c->W_macro + c->W_micro + 3) * 8 + 10 * 4;
}
