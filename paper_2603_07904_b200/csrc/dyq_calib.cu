// dyq_calib.cu -- offline threshold calibration (§IV-B, P:262-285;
// SPEC's binned isotonic reading S:289-306; readings C1-C6).
//
// Host code: the derivation is O(n) over at most ~1e6 calibration steps plus a
// 32-bin isotonic fit, run once offline.  The GPU-heavy part of calibration --
// evaluating the policy counterfactually at 16 / 2 / 4 / 8 bits every step --
// is dyq_calib_collect (dyq_model.cu), one batched policy step per control
// step.  Evaluation order (sequential fp64 sums in sample order, PAV merges
// left to right) is fixed so a table is a deterministic function of its
// samples.
#include <cmath>
#include <vector>

#include "dyq_internal.cuh"

namespace {

// Reading C1: bin i = floor(S / w), w = theta_fp / n_bins, S = theta_fp in
// the last bin; -1 outside [0, theta_fp] (those steps run BF16).
int bin_of(double S, double tfp, double w, int n_bins) {
    if (!(S >= 0.0 && S <= tfp)) return -1;
    const int i = (int)std::floor(S / w);
    return i < n_bins ? i : n_bins - 1;
}

// Weighted pool-adjacent-violators over y[0..n) (reading C3).
void pav(const double* y, const double* wt, int n, double* out) {
    struct Block {
        double mean, weight;
        int len;
    };
    std::vector<Block> b;
    for (int i = 0; i < n; ++i) {
        b.push_back({y[i], wt[i], 1});
        while (b.size() > 1 && b[b.size() - 2].mean > b.back().mean) {
            const Block r = b.back();
            b.pop_back();
            const Block l = b.back();
            b.pop_back();
            b.push_back({(l.mean * l.weight + r.mean * r.weight) / (l.weight + r.weight), l.weight + r.weight,
                         l.len + r.len});
        }
    }
    int k = 0;
    for (const Block& x : b)
        for (int j = 0; j < x.len; ++j) out[k++] = x.mean;
}

dyq_status_t check_params(const dyq_calib_t* c, int n_bins) {
    if (!c) return dyq::set_error(DYQ_EINVAL, "null calib");
    if (!(c->theta_fp > 0.0) || !(c->D_acc > 0.0) || !(c->eta > 0.0))
        return dyq::set_error(DYQ_EINVAL, "theta_fp, D_acc, eta must be > 0");
    if (n_bins < 1 || n_bins > 4096) return dyq::set_error(DYQ_EINVAL, "n_bins = %d outside [1, 4096]", n_bins);
    return DYQ_OK;
}

}  // namespace

extern "C" {

dyq_status_t dyq_calib_derive(const double* S, const double* err, int64_t n, int32_t n_bins, int32_t n_min,
                              dyq_calib_t* calib, double* smoothed, int64_t* counts_out, int32_t* n_undercovered) {
    dyq_status_t rc = check_params(calib, n_bins);
    if (rc) return rc;
    if (n <= 0 || !S || !err) return dyq::set_error(DYQ_EINVAL, "empty calibration set");
    if (n_min < 1) return dyq::set_error(DYQ_EINVAL, "n_min = %d < 1", n_min);
    const double tfp = calib->theta_fp, w = tfp / n_bins;
    std::vector<int64_t> cnt(n_bins, 0);
    std::vector<double> sum(2 * (size_t)n_bins, 0.0);
    for (int64_t t = 0; t < n; ++t) {
        const int i = bin_of(S[t], tfp, w, n_bins);
        if (i < 0) continue;
        cnt[i] += 1;
        sum[i] += err[3 * t + 0];
        sum[n_bins + i] += err[3 * t + 1];
    }
    std::vector<int> cov;
    int under = 0;
    for (int i = 0; i < n_bins; ++i) {
        if (cnt[i] >= n_min)
            cov.push_back(i);
        else
            ++under;
    }
    if (cov.empty()) return dyq::set_error(DYQ_EINVAL, "no bin reaches n_min = %d samples", n_min);
    const int nc = (int)cov.size();
    std::vector<double> sm(2 * (size_t)n_bins), y(nc), wt(nc), fit(nc);
    for (int j = 0; j < 2; ++j) {
        for (int c = 0; c < nc; ++c) {
            y[c] = sum[(size_t)j * n_bins + cov[c]] / (double)cnt[cov[c]];
            wt[c] = (double)cnt[cov[c]];
        }
        pav(y.data(), wt.data(), nc, fit.data());
        double* row = sm.data() + (size_t)j * n_bins;
        // reading C2: interpolate under-covered bins between covered neighbours
        int c = 0;
        for (int i = 0; i < n_bins; ++i) {
            while (c < nc && cov[c] < i) ++c;
            if (c < nc && cov[c] == i) {
                row[i] = fit[c];
            } else if (c == 0) {
                row[i] = fit[0];
            } else if (c == nc) {
                row[i] = fit[nc - 1];
            } else {
                const int a = cov[c - 1], b = cov[c];
                const double t = (double)(i - a) / (double)(b - a);
                row[i] = fit[c - 1] + t * (fit[c] - fit[c - 1]);
            }
        }
    }
    double th[2];
    for (int j = 0; j < 2; ++j) {
        th[j] = tfp;
        for (int i = 0; i < n_bins; ++i) {
            const double eps = calib->D_acc / ((double)(i + 1) * w + calib->eta);
            if (sm[(size_t)j * n_bins + i] > eps) {
                th[j] = (double)i * w;
                break;
            }
        }
    }
    calib->theta_24 = th[0];
    calib->theta_48 = th[1] < th[0] ? th[0] : th[1];
    if (smoothed)
        for (size_t k = 0; k < sm.size(); ++k) smoothed[k] = sm[k];
    if (counts_out)
        for (int i = 0; i < n_bins; ++i) counts_out[i] = cnt[i];
    if (n_undercovered) *n_undercovered = under;
    return DYQ_OK;
}

dyq_status_t dyq_calib_validate(const dyq_calib_t* calib, const double* S, const double* err, int64_t n,
                                int32_t n_bins, int64_t* n_quant, int64_t* n_ok, double* worst) {
    dyq_status_t rc = check_params(calib, n_bins);
    if (rc) return rc;
    if (n < 0 || (n > 0 && (!S || !err))) return dyq::set_error(DYQ_EINVAL, "null samples");
    if (!(0.0 <= calib->theta_24 && calib->theta_24 <= calib->theta_48 && calib->theta_48 <= calib->theta_fp))
        return dyq::set_error(DYQ_EINVAL, "thresholds not ordered 0 <= t24 <= t48 <= tfp");
    const double tfp = calib->theta_fp, w = tfp / n_bins;
    int64_t q = 0, ok = 0;
    if (worst)
        for (int i = 0; i < n_bins; ++i) worst[i] = 0.0;
    for (int64_t t = 0; t < n; ++t) {
        const int i = bin_of(S[t], tfp, w, n_bins);
        if (i < 0) {
            ++ok;  // BF16 step: no quantization error
            continue;
        }
        ++q;
        const double eps = calib->D_acc / (S[t] + calib->eta);
        // Eq. (6), boundaries in the lower-bit interval (as dyq_select_bits)
        const int col = S[t] <= calib->theta_24 ? 0 : (S[t] <= calib->theta_48 ? 1 : 2);
        const double e = err[3 * t + col];
        if (e <= eps) ++ok;
        if (worst && e / eps > worst[i]) worst[i] = e / eps;
    }
    if (n_quant) *n_quant = q;
    if (n_ok) *n_ok = ok;
    return DYQ_OK;
}

}  // extern "C"
