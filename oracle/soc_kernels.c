/* CPU oracle kernels for second-order-cone runs — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's numba loops so that the oracle
 * reproduces the reference's rounding exactly (sequential sums of squares,
 * glibc exp, no FMA contraction: build with -ffp-contract=off):
 *   orc_soc_lambda_max  <- cones.py:216-234 (_soc_lambda_bounds, max half)
 *   orc_soc_exp_run     <- cones.py:252-274 (_soc_exp_run)
 *   orc_soc_inf_norm    <- cones.py:237-249 (_soc_inf_norm)
 * X is a run of k blocks stored row-major with w = d+1 coordinates per block
 * (vector part first, scalar last), exactly the reference's Element layout.
 */
#include <math.h>
#include <stdint.h>

static const double kSqrt2 = 1.4142135623730951;

static double block_sq(const double *row, int64_t d) {
    double s = 0.0;
    for (int64_t j = 0; j < d; ++j) s += row[j] * row[j];
    return s;
}

double orc_soc_lambda_max(const double *X, int64_t k, int64_t w) {
    const int64_t d = w - 1;
    double hi = -INFINITY;
    for (int64_t i = 0; i < k; ++i) {
        const double *row = X + i * w;
        double lam = (row[d] + sqrt(block_sq(row, d))) / kSqrt2;
        if (lam > hi) hi = lam;
    }
    return hi;
}

double orc_soc_exp_run(const double *X, double *out, int64_t k, int64_t w, double shift) {
    const int64_t d = w - 1;
    double tr = 0.0;
    for (int64_t i = 0; i < k; ++i) {
        const double *row = X + i * w;
        double *o = out + i * w;
        double nrm = sqrt(block_sq(row, d));
        double a = exp((row[d] + nrm) / kSqrt2 - shift);
        double b = exp((row[d] - nrm) / kSqrt2 - shift);
        double c = nrm > 0.0 ? (a - b) / (kSqrt2 * nrm) : 0.0;
        for (int64_t j = 0; j < d; ++j) o[j] = c * row[j];
        o[d] = (a + b) / kSqrt2;
        tr += a + b;
    }
    return tr;
}

double orc_soc_inf_norm(const double *X, int64_t k, int64_t w) {
    const int64_t d = w - 1;
    double hi = 0.0;
    for (int64_t i = 0; i < k; ++i) {
        const double *row = X + i * w;
        double v = (fabs(row[d]) + sqrt(block_sq(row, d))) / kSqrt2;
        if (v > hi) hi = v;
    }
    return hi;
}
