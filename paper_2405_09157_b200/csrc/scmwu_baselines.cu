// scmwu_baselines.cu — the reference's independent verification solvers on the GPU
// (SURVEY §8(f) row 3): sc_meb_baseline, sc_gilbert_baseline (include/scmwu.h).
#include <algorithm>
#include <vector>

#include "scmwu_handle.h"

namespace scmwu {
// -------------------------------------------------------------------------------------
// GPU verification baselines: the reference's independent solvers
// meb_baseline (Badoiu-Clarkson, R/baselines.py:34-85) and gilbert_baseline (Frank-Wolfe
// on the polytope distance, R/baselines.py:88-161) over a resident instance.  One
// cooperative persistent launch each; every iteration is one streaming argmax/argmin
// pass (warp per row, butterfly sums) + ONE grid barrier: CTAs write (value, row) pairs
// to a parity double buffer and every CTA folds all of them (max / min value, lowest row
// on ties = the reference's first-index rule) and applies the identical update to its
// own copy of the iterate, so no second barrier or broadcast is needed.

// deterministic block sum (warp butterflies, then the warps in index order)
__device__ double block_sum(double v, double* red8) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) red8[warp] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red8[w];
    return s;
}

// better (value, row) under a max (sign = 1) or min (sign = -1) rule, lowest row on ties
__device__ __forceinline__ void arg_better(double& bv, int64_t& bi, double v, int64_t i,
                                           double sign) {
    const double a = sign * v, b = sign * bv;
    if (a > b || (a == b && i < bi)) { bv = v; bi = i; }
}

__device__ void block_arg(double& bv, int64_t& bi, double sign, double* sv, int64_t* si) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const double v = __shfl_xor_sync(0xffffffffu, bv, o);
        const int64_t i = __shfl_xor_sync(0xffffffffu, bi, o);
        arg_better(bv, bi, v, i, sign);
    }
    __syncthreads();
    if (lane == 0) { sv[warp] = bv; si[warp] = bi; }
    __syncthreads();
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) arg_better(bv, bi, sv[w], si[w], sign);
}

// one pass: argmax over rows [a, b) of (|x_i - c| + r_i) (mode 0, c = iterate) or
// argmin / argmax of x_i . z (mode 1 / 2); warp per row, rows dealt cyclically to the
// grid's warps
__device__ void arg_pass(const double* X, int ld, int d, const double* radii, int64_t a,
                         int64_t b, const double* c, int mode, double& bv, int64_t& bi) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const double sign = mode == 1 ? -1.0 : 1.0;
    for (int64_t i = a + gw; i < b; i += nw) {
        const double* xr = X + i * ld;
        double s = 0.0;
        for (int j = lane; j < d; j += 32) {
            if (mode == 0) { const double t = c[j] - xr[j]; s = fma(t, t, s); }
            else s = fma(xr[j], c[j], s);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const double v = mode == 0 ? sqrt(s) + radii[i] : s;
        arg_better(bv, bi, v, i, sign);
    }
}

__global__ void __launch_bounds__(256) meb_kernel(const double* X, int ld, int d,
                                                  const double* radii, int64_t n,
                                                  int64_t iters, double* part,
                                                  unsigned long long* bar, double* c_out) {
    extern __shared__ double bsm[];
    double* c = bsm;                         // iterate (every CTA keeps its own copy)
    double* xf = bsm + ld;                   // the farthest row
    double* sv = xf + ld;                    // 8 warp values
    int64_t* si = reinterpret_cast<int64_t*>(sv + 8);
    double* red8 = sv + 16;
    const int G = gridDim.x;
    for (int j = threadIdx.x; j < d; j += blockDim.x) c[j] = X[j];
    __syncthreads();
    for (int64_t t = 1; t <= iters; ++t) {
        double bv = -1.0;                    // R/baselines.py:40-41
        int64_t bi = 0;
        arg_pass(X, ld, d, radii, 0, n, c, 0, bv, bi);
        block_arg(bv, bi, 1.0, sv, si);
        double* pb = part + (size_t)(t & 1) * 2 * G;
        if (threadIdx.x == 0) {
            pb[2 * blockIdx.x] = bv;
            pb[2 * blockIdx.x + 1] = __longlong_as_double((long long)bi);
        }
        grid_barrier(bar, (unsigned long long)t * G);
        bv = -1.0; bi = 0;
        for (int q = 0; q < G; ++q)
            arg_better(bv, bi, __ldcg(pb + 2 * q),
                       (int64_t)__double_as_longlong(__ldcg(pb + 2 * q + 1)), 1.0);
        const double* xr = X + bi * ld;
        double s = 0.0;
        for (int j = threadIdx.x; j < d; j += blockDim.x) {
            xf[j] = xr[j];
            const double df = xr[j] - c[j];
            s = fma(df, df, s);
        }
        const double dist = sqrt(block_sum(s, red8));
        const double step = 1.0 / ((double)t + 1.0);
        if (dist > 0.0) {
            const double scale = 1.0 + radii[bi] / dist;
            for (int j = threadIdx.x; j < d; j += blockDim.x)
                c[j] += step * scale * (xf[j] - c[j]);
        }
        __syncthreads();
    }
    if (blockIdx.x == 0)
        for (int j = threadIdx.x; j < d; j += blockDim.x) c_out[j] = c[j];
}

// log[it] = {best P row, best Q row, lambda} of every update (host rebuilds mu, gamma)
__global__ void __launch_bounds__(256) gilbert_kernel(const double* X, int ld, int d,
                                                      int64_t n1, int64_t n, double gap_tol,
                                                      int64_t max_iters, double* part,
                                                      unsigned long long* bar, double* z_out,
                                                      double* log, double* info) {
    extern __shared__ double bsm[];
    double* z = bsm;
    double* dk = bsm + ld;
    double* sv = dk + ld;
    int64_t* si = reinterpret_cast<int64_t*>(sv + 8);
    double* red8 = sv + 16;
    const int G = gridDim.x;
    for (int j = threadIdx.x; j < d; j += blockDim.x) z[j] = X[j] - X[n1 * ld + j];
    __syncthreads();
    double gap = INFINITY;
    int64_t it = 0, updates = 0;
    for (int64_t k = 1; k <= max_iters; ++k) {
        it = k;
        double pv = INFINITY, qv = -INFINITY;   // R/baselines.py:107-122
        int64_t pi = 0, qi = 0;
        arg_pass(X, ld, d, nullptr, 0, n1, z, 1, pv, pi);
        arg_pass(X, ld, d, nullptr, n1, n, z, 2, qv, qi);
        block_arg(pv, pi, -1.0, sv, si);
        block_arg(qv, qi, 1.0, sv, si);
        double* pb = part + (size_t)(k & 1) * 4 * G;
        if (threadIdx.x == 0) {
            pb[4 * blockIdx.x] = pv;
            pb[4 * blockIdx.x + 1] = __longlong_as_double((long long)pi);
            pb[4 * blockIdx.x + 2] = qv;
            pb[4 * blockIdx.x + 3] = __longlong_as_double((long long)qi);
        }
        grid_barrier(bar, (unsigned long long)k * G);
        pv = INFINITY; qv = -INFINITY; pi = 0; qi = n1;
        for (int q = 0; q < G; ++q) {
            arg_better(pv, pi, __ldcg(pb + 4 * q),
                       (int64_t)__double_as_longlong(__ldcg(pb + 4 * q + 1)), -1.0);
            arg_better(qv, qi, __ldcg(pb + 4 * q + 2),
                       (int64_t)__double_as_longlong(__ldcg(pb + 4 * q + 3)), 1.0);
        }
        const double* xp = X + pi * ld;
        const double* xq = X + qi * ld;
        double zd = 0.0, dn = 0.0;
        for (int j = threadIdx.x; j < d; j += blockDim.x) {
            const double v = (xp[j] - xq[j]) - z[j];
            dk[j] = v;
            zd = fma(z[j], v, zd);
            dn = fma(v, v, dn);
        }
        const double zdiff = block_sum(zd, red8);
        const double denom = block_sum(dn, red8);
        gap = -2.0 * zdiff;
        if (gap < gap_tol || denom == 0.0) break;
        double lam = -zdiff / denom;
        if (lam > 1.0) lam = 1.0;
        if (lam <= 0.0) break;
        for (int j = threadIdx.x; j < d; j += blockDim.x) z[j] += lam * dk[j];
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            log[3 * updates] = (double)pi;
            log[3 * updates + 1] = (double)(qi - n1);
            log[3 * updates + 2] = lam;
        }
        ++updates;
        __syncthreads();
    }
    if (blockIdx.x == 0) {
        for (int j = threadIdx.x; j < d; j += blockDim.x) z_out[j] = z[j];
        if (threadIdx.x == 0) { info[0] = gap; info[1] = (double)it; info[2] = (double)updates; }
    }
}

}  // namespace scmwu

extern "C" {

// cooperative grid for the baseline kernels: at most one CTA per 8 rows, co-resident
static int baseline_grid(sc_handle* h, const void* fn, size_t smem, int64_t rows) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, smem) != cudaSuccess ||
        per_sm < 1)
        return 0;
    const int64_t want = std::max<int64_t>(1, (rows + 7) / 8);
    return (int)std::min<int64_t>(want, (int64_t)h->sms * std::min(per_sm, 2));
}

int sc_meb_baseline(sc_handle* h, int64_t iters, double* center, double* value) {
    if (!h || !center || iters < 0) return SC_EARG;
    if (h->prob.kind != SC_SES || h->prob.world > 1) {
        h->err = "meb_baseline needs a single-GPU SES handle";
        return SC_EARG;
    }
    CK(cudaSetDevice(h->prob.device), "set device");
    const int64_t n = h->prob.n_local;
    const int d = h->prob.d, ld = h->ld;
    const size_t smem = (size_t)(2 * ld + 32) * 8;
    const int G = baseline_grid(h, (const void*)meb_kernel, smem, n);
    if (G < 1) { h->err = "baseline kernel does not fit"; return SC_ECUDA; }
    double *part = nullptr, *cout = nullptr;
    unsigned long long* bar = nullptr;
    CK(pool_alloc((void**)&part, 4 * (size_t)G * 8, h->prob.device, h->stream), "alloc baseline");
    CK(pool_alloc((void**)&cout, (size_t)d * 8, h->prob.device, h->stream), "alloc baseline");
    CK(pool_alloc((void**)&bar, 8, h->prob.device, h->stream), "alloc baseline");
    CK(cudaMemsetAsync(bar, 0, 8, h->stream), "zero barrier");
    const double* X = h->X;
    const double* radii = h->radii;
    double* pp = part;
    double* co = cout;
    unsigned long long* bb = bar;
    int64_t nn = n, it = iters;
    int ldv = ld, dv = d;
    void* args[] = {(void*)&X, &ldv, &dv, (void*)&radii, &nn, &it, &pp, &bb, &co};
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)meb_kernel, G, 256, args, smem,
                                                h->stream);
    ++h->launches;
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e == cudaSuccess) e = h_get(h, center, cout, (size_t)d * 8);
    pool_free(part, h->stream);
    pool_free(cout, h->stream);
    pool_free(bar, h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "meb baseline");
    if (value) return sc_progress(h, center, value);   // max_i |v_i - c| + r_i
    return SC_OK;
}

int sc_gilbert_baseline(sc_handle* h, double gap_tol, int64_t max_iters, double* value,
                        double* gap, int64_t* iterations, double* mu, double* gam) {
    if (!h || !value || !(gap_tol > 0.0) || max_iters < 0) return SC_EARG;
    if (h->prob.kind != SC_SVM || h->prob.world > 1) {
        h->err = "gilbert_baseline needs a single-GPU SVM handle";
        return SC_EARG;
    }
    CK(cudaSetDevice(h->prob.device), "set device");
    const int64_t n = h->prob.n_local, n1 = h->prob.n1_local;
    const int d = h->prob.d, ld = h->ld;
    const size_t smem = (size_t)(2 * ld + 32) * 8;
    const int G = baseline_grid(h, (const void*)gilbert_kernel, smem, n);
    if (G < 1) { h->err = "baseline kernel does not fit"; return SC_ECUDA; }
    double *part = nullptr, *zout = nullptr, *logb = nullptr, *info = nullptr;
    unsigned long long* bar = nullptr;
    CK(pool_alloc((void**)&part, 8 * (size_t)G * 8, h->prob.device, h->stream), "alloc baseline");
    CK(pool_alloc((void**)&zout, (size_t)d * 8, h->prob.device, h->stream), "alloc baseline");
    CK(pool_alloc((void**)&logb, 3 * (size_t)std::max<int64_t>(1, max_iters) * 8, h->prob.device, h->stream), "alloc baseline log");
    CK(pool_alloc((void**)&info, 4 * 8, h->prob.device, h->stream), "alloc baseline");
    CK(pool_alloc((void**)&bar, 8, h->prob.device, h->stream), "alloc baseline");
    CK(cudaMemsetAsync(bar, 0, 8, h->stream), "zero barrier");
    const double* X = h->X;
    double *pp = part, *zo = zout, *lg = logb, *inf = info;
    unsigned long long* bb = bar;
    int64_t a1 = n1, an = n, mi = max_iters;
    double tol = gap_tol;
    int ldv = ld, dv = d;
    void* args[] = {(void*)&X, &ldv, &dv, &a1, &an, &tol, &mi, &pp, &bb, &zo, &lg, &inf};
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)gilbert_kernel, G, 256, args,
                                                smem, h->stream);
    ++h->launches;
    double hi[3] = {INFINITY, 0.0, 0.0};
    std::vector<double> z(d);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e == cudaSuccess) e = h_get(h, hi, info, 3 * 8);
    if (e == cudaSuccess) e = h_get(h, z.data(), zout, (size_t)d * 8);
    const int64_t updates = (int64_t)hi[2];
    std::vector<double> lg_h(3 * (size_t)updates);
    if (e == cudaSuccess && updates > 0)
        e = h_get(h, lg_h.data(), logb, lg_h.size() * 8);
    pool_free(part, h->stream);
    pool_free(zout, h->stream);
    pool_free(logb, h->stream);
    pool_free(info, h->stream);
    pool_free(bar, h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "gilbert baseline");
    if (max_iters == 0) { hi[1] = 0.0; }
    double nz = 0.0;
    for (int j = 0; j < d; ++j) nz += z[j] * z[j];
    *value = sqrt(nz);
    if (gap) *gap = hi[0];
    if (iterations) *iterations = (int64_t)hi[1];
    // mu, gamma from the update log: every update scales by (1 - lam) and adds lam to the
    // chosen vertex; the starting vertex is row 0 of each side
    if (mu || gam) {
        if (mu) for (int64_t i = 0; i < n1; ++i) mu[i] = 0.0;
        if (gam) for (int64_t i = 0; i < n - n1; ++i) gam[i] = 0.0;
        double suffix = 1.0;   // prod_{l > k} (1 - lam_l)
        for (int64_t k = updates - 1; k >= 0; --k) {
            const double lam = lg_h[3 * k + 2];
            if (mu) mu[(int64_t)lg_h[3 * k]] += lam * suffix;
            if (gam) gam[(int64_t)lg_h[3 * k + 1]] += lam * suffix;
            suffix *= 1.0 - lam;
        }
        if (mu) mu[0] += suffix;
        if (gam) gam[0] += suffix;
    }
    return SC_OK;
}

}  // extern "C"
