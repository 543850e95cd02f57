// dyq_select.cu -- kinematic proxies -> S_t -> bhat_t -> Alg. 1 (b*_t), on device.
//
// PAPER.md: Motion Fineness M_t = 1 - ||a^xyz||/mu_max and Angular Jerk
// J_t = ||a^rot_t - a^rot_{t-1}||/nu_max with 95th-percentile normalizers
// (P:175-177); window means over W_macro / W_micro; fused
// S_t = max(0, lambda*M~ + (1-lambda)*J~); bhat_t = 16 if S_t > theta_fp
// else Phi(S_t) (Alg. 1 line 2; Eq. 6); the saturating
// counter dispatcher (Alg. 1 lines 3-9).  The paper runs this on the
// CPU and writes b* into zero-copy memory; here it is one tiny
// in-stream kernel that writes bits[] in device memory, so the qlinear kernels
// route on it without a host round trip (DESIGN.md conflict C3).
//
// Bit-exactness with the oracle: fp64 everywhere, explicit _rn intrinsics (no
// FMA contraction), the oracle's evaluation order.  The nearest-rank 95th
// percentile (reading 14) is read off a SORTED copy of each history
// ring kept in the state: a step deletes the overwritten value and inserts the
// new one (O(1) parallel time instead of re-sorting); the k-th smallest of a
// multiset is unique, so this equals the oracle's sort-then-index exactly.
// Latency: one CTA per stream stages its whole state block in shared memory
// with one coalesced load, and writes it back with one coalesced store.
#include "dyq_internal.cuh"
#include "dyq_ptx.cuh"

namespace dyq {

struct SelHeader {
    dyq_calib_t cal;
    int32_t E;
    int32_t stride;  // bytes per stream
    int32_t off_jerk, off_Mwin, off_Jwin, off_prev, off_int, off_smag, off_sjerk;
};
constexpr size_t SEL_HDR = 256;
static_assert(sizeof(SelHeader) <= SEL_HDR, "header");

// I_SKIP: set by an episode reset -- the stream's next a_{t-1} belongs to the
// previous episode and is not observed (reading 23, S:259 causality)
enum { I_HIST_N = 0, I_HIST_POS, I_MW_N, I_MW_POS, I_JW_N, I_JW_POS, I_STEPS, I_BSTAR, I_C, I_BBAR, I_SKIP, I_COUNT };

__host__ inline SelHeader make_sel_header(int32_t E, const dyq_calib_t& c) {
    SelHeader h{};
    h.cal = c;
    h.E = E;
    int off = c.H * 8;  // mag
    h.off_jerk = off;
    off += c.H * 8;
    h.off_Mwin = off;
    off += c.W_macro * 8;
    h.off_Jwin = off;
    off += c.W_micro * 8;
    h.off_prev = off;
    off += 3 * 8;
    h.off_int = off;
    off += I_COUNT * 4;
    off = (off + 7) & ~7;
    h.off_smag = off;  // sorted copies of the two rings (first HIST_N entries valid)
    off += c.H * 8;
    h.off_sjerk = off;
    off += c.H * 8;
    h.stride = (off + 15) & ~15;
    return h;
}

size_t sel_state_bytes(int32_t E, const dyq_calib_t& c) {
    return SEL_HDR + (size_t)E * make_sel_header(E, c).stride;
}

__device__ inline void reset_episode_dev(const SelHeader& h, uint8_t* base) {
    int32_t* I = reinterpret_cast<int32_t*>(base + h.off_int);
    double* prev = reinterpret_cast<double*>(base + h.off_prev);
    I[I_MW_N] = I[I_MW_POS] = I[I_JW_N] = I[I_JW_POS] = 0;
    I[I_STEPS] = 0;
    I[I_BSTAR] = 16; I[I_C] = 0; I[I_BBAR] = 16;
    prev[0] = prev[1] = prev[2] = 0.0;
}

__global__ void sel_init_kernel(uint8_t* state) {
    const SelHeader h = *reinterpret_cast<const SelHeader*>(state);
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= h.E) return;
    uint8_t* base = state + SEL_HDR + (size_t)e * h.stride;
    int32_t* I = reinterpret_cast<int32_t*>(base + h.off_int);
    I[I_HIST_N] = I[I_HIST_POS] = 0;
    reset_episode_dev(h, base);
    I[I_SKIP] = 0;
}

__global__ void sel_reset_kernel(uint8_t* state, const uint8_t* mask) {
    const SelHeader h = *reinterpret_cast<const SelHeader*>(state);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < h.E; e += gridDim.x * blockDim.x) {
        if (mask && !mask[e]) continue;
        uint8_t* base = state + SEL_HDR + (size_t)e * h.stride;
        reset_episode_dev(h, base);
        reinterpret_cast<int32_t*>(base + h.off_int)[I_SKIP] = 1;
    }
}

__device__ inline double window_mean(const double* w, int cap, int n, int pos) {
    if (n == 0) return 0.0;
    const int start = (pos - n + cap) % cap;
    double sum = 0.0;
    for (int i = 0; i < n; ++i) sum = __dadd_rn(sum, w[(start + i) % cap]);
    return __ddiv_rn(sum, (double)n);
}

__device__ inline int phi_dev(double S, double t24, double t48) {
    if (S <= t24) return 2;
    if (S <= t48) return 4;
    return 8;
}

#ifndef DYQ_SEL_THREADS
#define DYQ_SEL_THREADS 1024  // one history slot per thread (H <= 1024); step A/B: 256 60.0, 512 59.5, 1024 59.3 us
#endif
constexpr int SEL_THREADS = DYQ_SEL_THREADS;
constexpr int SEL_PER = 1024 / SEL_THREADS;  // H <= 1024 = SEL_THREADS * SEL_PER

// Sorted-multiset update of srt[0..n): delete one copy of `old` (when full),
// insert x.  All threads of the CTA call it; srt lives in shared memory.
__device__ void sorted_replace(double* srt, int n, bool full, double old, double x, int* s_r, int* s_cnt) {
    double v[SEL_PER];
    int le = 0;
#pragma unroll
    for (int r = 0; r < SEL_PER; ++r) {
        const int i = threadIdx.x + SEL_THREADS * r;
        v[r] = i < n ? srt[i] : 0.0;
        if (i < n) {
            le += (v[r] <= x);
            if (full && v[r] == old && (i == 0 || srt[i - 1] != old)) *s_r = i;  // first copy of old
        }
    }
    if (le) atomicAdd(s_cnt, le);
    __syncthreads();
    const int rm = full ? *s_r : n;                       // index removed (n: none)
    const int p = *s_cnt - ((full && old <= x) ? 1 : 0);  // insertion index of x
#pragma unroll
    for (int r = 0; r < SEL_PER; ++r) {
        const int i = threadIdx.x + SEL_THREADS * r;
        if (i < n && i != rm) {
            const int b = i - (i > rm ? 1 : 0);
            srt[b + (b >= p ? 1 : 0)] = v[r];
        }
    }
    if (threadIdx.x == 0) srt[p] = x;
    __syncthreads();
}

// One CTA per stream e: observe a_{t-1}, update the proxies, decide b*_t
// (Alg. 1), write bits[e] and, when row_bits != NULL, the routed activation
// bits of the stream's tpe tokens (fused dyq_route_bits).
__global__ void __launch_bounds__(SEL_THREADS) select_bits_kernel(uint8_t* state, const float* __restrict__ prev_action,
                                                                  int32_t* bits, double* S_out, int32_t* target_out,
                                                                  int tpe, int4 tab, int32_t* row_bits) {
    extern __shared__ __align__(16) uint8_t ssm[];  // [header 256 B][episode block stride B]
    __shared__ double s_x[2], s_old[2];
    __shared__ int s_n, s_full, s_r[2], s_cnt[2];
    const int e = blockIdx.x;
    ptx::pdl_wait();  // state and a_{t-1} come from the preceding kernels
    ptx::pdl_launch_dependents();
    const bool observe = prev_action != nullptr;
    float act[6];
    if (observe && threadIdx.x == 0) {  // issued first: its latency overlaps the state copy
#pragma unroll
        for (int i = 0; i < 6; ++i) act[i] = prev_action[(size_t)e * 7 + i];
    }
    {
        const uint4* src = reinterpret_cast<const uint4*>(state);
        uint4* dst = reinterpret_cast<uint4*>(ssm);
        for (int i = threadIdx.x; i < (int)(SEL_HDR / 16); i += SEL_THREADS) dst[i] = src[i];
    }
    __syncthreads();
    const SelHeader& h = *reinterpret_cast<const SelHeader*>(ssm);
    if (e >= h.E) return;  // block-uniform: more CTAs than initialised streams
    const dyq_calib_t& c = h.cal;
    uint8_t* gbase = state + SEL_HDR + (size_t)e * h.stride;
    uint8_t* base = ssm + SEL_HDR;
    for (int i = threadIdx.x; i < h.stride / 16; i += SEL_THREADS)
        reinterpret_cast<uint4*>(base)[i] = reinterpret_cast<const uint4*>(gbase)[i];
    double* mag = reinterpret_cast<double*>(base);
    double* jerk = reinterpret_cast<double*>(base + h.off_jerk);
    double* Mwin = reinterpret_cast<double*>(base + h.off_Mwin);
    double* Jwin = reinterpret_cast<double*>(base + h.off_Jwin);
    double* prev = reinterpret_cast<double*>(base + h.off_prev);
    double* smag = reinterpret_cast<double*>(base + h.off_smag);
    double* sjerk = reinterpret_cast<double*>(base + h.off_sjerk);
    int32_t* I = reinterpret_cast<int32_t*>(base + h.off_int);
    __syncthreads();

    const bool skip = I[I_SKIP] != 0;  // first step after an episode reset: a_{t-1} is stale
    __syncthreads();
    if (skip && threadIdx.x == 0) I[I_SKIP] = 0;
    if (observe && !skip) {
        if (threadIdx.x == 0) {
            const double x = act[0], y = act[1], z = act[2];
            const double r0 = act[3], r1 = act[4], r2 = act[5];
            // ||a^xyz||_2 left to right, no contraction
            const double mv = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
            double jv = 0.0;  // first observation: J = 0 (reading 16)
            if (I[I_STEPS] > 0) {
                const double d0 = __dadd_rn(r0, -prev[0]);
                const double d1 = __dadd_rn(r1, -prev[1]);
                const double d2 = __dadd_rn(r2, -prev[2]);
                jv = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2)));
            }
            prev[0] = r0; prev[1] = r1; prev[2] = r2;
            const int pos = I[I_HIST_POS];
            const int n = I[I_HIST_N];
            s_full = n == c.H;
            s_old[0] = mag[pos];
            s_old[1] = jerk[pos];
            mag[pos] = mv;
            jerk[pos] = jv;
            I[I_HIST_POS] = (pos + 1) % c.H;
            s_n = n;
            if (n < c.H) I[I_HIST_N] = n + 1;
            s_x[0] = mv;
            s_x[1] = jv;
            s_r[0] = s_r[1] = 0;
            s_cnt[0] = s_cnt[1] = 0;
        }
        __syncthreads();
        const int n = s_n;
        const bool full = s_full != 0;
        sorted_replace(smag, n, full, s_old[0], s_x[0], &s_r[0], &s_cnt[0]);
        sorted_replace(sjerk, n, full, s_old[1], s_x[1], &s_r[1], &s_cnt[1]);
        if (threadIdx.x == 0) {
            const int n1 = full ? n : n + 1;
            const int k = (95 * n1 + 99) / 100;  // nearest rank, ceil(0.95 n)
            double mu = smag[k - 1], nu = sjerk[k - 1];
            if (mu < 1e-6) mu = 1e-6;
            if (nu < 1e-6) nu = 1e-6;
            double M = __dadd_rn(1.0, -__ddiv_rn(s_x[0], mu));
            if (c.clamp_M) {
                if (M < 0.0) M = 0.0;
                if (M > 1.0) M = 1.0;
            }
            double J = __ddiv_rn(s_x[1], nu);
            if (J > c.J_cap) J = c.J_cap;
            int p = I[I_MW_POS];
            Mwin[p] = M;
            I[I_MW_POS] = (p + 1) % c.W_macro;
            if (I[I_MW_N] < c.W_macro) I[I_MW_N] += 1;
            p = I[I_JW_POS];
            Jwin[p] = J;
            I[I_JW_POS] = (p + 1) % c.W_micro;
            if (I[I_JW_N] < c.W_micro) I[I_JW_N] += 1;
            I[I_STEPS] += 1;
        }
    }
    __shared__ int s_bstar;
    if (threadIdx.x == 0) {
        const double Mbar = window_mean(Mwin, c.W_macro, I[I_MW_N], I[I_MW_POS]);
        const double Jbar = window_mean(Jwin, c.W_micro, I[I_JW_N], I[I_JW_POS]);
        const double lam_term = __dmul_rn(c.lambda, Mbar);
        const double one_minus = __dadd_rn(1.0, -c.lambda);
        const double jer_term = __dmul_rn(one_minus, Jbar);
        double S = __dadd_rn(lam_term, jer_term);
        if (S < 0.0) S = 0.0;
        const bool warm = I[I_STEPS] < c.W_macro;
        int bhat;
        if (warm || S > c.theta_fp) bhat = 16;
        else bhat = phi_dev(S, c.theta_24, c.theta_48);
        // Alg. 1 lines 3-9
        int bstar = I[I_BSTAR], cnt = I[I_C], bbar = I[I_BBAR];
        if (bhat >= bstar) {
            bstar = bhat; cnt = 0; bbar = bhat;
        } else {
            const int carried = cnt > 0 ? bbar : 0;
            const int nb = bhat > carried ? bhat : carried;
            const int nc = cnt * (nb == bbar ? 1 : 0) + 1;
            bstar = nc == c.K ? nb : bstar;
            cnt = nc % c.K;
            bbar = nb;
        }
        I[I_BSTAR] = bstar; I[I_C] = cnt; I[I_BBAR] = bbar;
        bits[e] = bstar;
        if (S_out) S_out[e] = S;
        if (target_out) target_out[e] = bhat;
        s_bstar = bstar;
    }
    __syncthreads();
    if (row_bits) {
        const int b = s_bstar;
        const int ab = b == 2 ? tab.x : b == 4 ? tab.y : b == 8 ? tab.z : tab.w;
        for (int i = threadIdx.x; i < tpe; i += SEL_THREADS) row_bits[(size_t)e * tpe + i] = ab;
    }
    for (int i = threadIdx.x; i < h.stride / 16; i += SEL_THREADS)
        reinterpret_cast<uint4*>(gbase)[i] = reinterpret_cast<const uint4*>(base)[i];
}

__global__ void route_bits_kernel(const int32_t* bits, int E, int tpe, int4 tab, int32_t* row_bits) {
    const int m = blockIdx.x * blockDim.x + threadIdx.x;
    if (m >= E * tpe) return;
    const int b = bits[m / tpe];
    row_bits[m] = b == 2 ? tab.x : b == 4 ? tab.y : b == 8 ? tab.z : tab.w;
}

dyq_status_t launch_sel_init(int32_t E, const dyq_calib_t& c, void* state, cudaStream_t st) {
    const SelHeader h = make_sel_header(E, c);
    cudaMemsetAsync(state, 0, sel_state_bytes(E, c), st);
    cudaMemcpyAsync(state, &h, sizeof h, cudaMemcpyHostToDevice, st);  // pageable: staged synchronously
    sel_init_kernel<<<(E + 127) / 128, 128, 0, st>>>(reinterpret_cast<uint8_t*>(state));
    return check_launch("sel_init_kernel");
}

dyq_status_t launch_sel_reset(void* state, int32_t E, const uint8_t* mask, cudaStream_t st) {
    (void)E;  // E lives in the device header; the kernel strides over it
    sel_reset_kernel<<<8, 256, 0, st>>>(reinterpret_cast<uint8_t*>(state), mask);
    return check_launch("sel_reset_kernel");
}

dyq_status_t launch_select(void* state, int32_t E, const dyq_calib_t* cal_or_null, const float* prev_action,
                           int32_t* bits, double* S_out, int32_t* target_out, int32_t tpe, const int32_t* tab4,
                           int32_t* row_bits, cudaStream_t st) {
    // the calibration (hence the state block size) lives on the device; size
    // shared memory for the maximum (H = 1024, windows 64) unless known
    dyq_calib_t cmax{};
    cmax.H = 1024;
    cmax.W_macro = 64;
    cmax.W_micro = 64;
    const SelHeader hmax = make_sel_header(1, cal_or_null ? *cal_or_null : cmax);
    const size_t smem = SEL_HDR + (size_t)hmax.stride;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(select_bits_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        attr = true;
    }
    const int4 tab = tab4 ? make_int4(tab4[0], tab4[1], tab4[2], tab4[3]) : make_int4(2, 4, 8, 16);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(E);
    cfg.blockDim = dim3(SEL_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr1[1];
    attr1[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr1[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr1;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, select_bits_kernel, reinterpret_cast<uint8_t*>(state), prev_action,
                                             bits, S_out, target_out, tpe, tab, row_bits);
    if (e != cudaSuccess) return set_error(DYQ_ECUDA, "select_bits_kernel launch: %s", cudaGetErrorString(e));
    return check_launch("select_bits_kernel");
}

dyq_status_t launch_route(const int32_t* bits, int32_t E, int32_t tpe, const int32_t* tab4, int32_t* row_bits,
                          cudaStream_t st) {
    const int4 tab = tab4 ? make_int4(tab4[0], tab4[1], tab4[2], tab4[3]) : make_int4(2, 4, 8, 16);
    const int total = E * tpe;
    route_bits_kernel<<<(total + 255) / 256, 256, 0, st>>>(bits, E, tpe, tab, row_bits);
    return check_launch("route_bits_kernel");
}

}  // namespace dyq
