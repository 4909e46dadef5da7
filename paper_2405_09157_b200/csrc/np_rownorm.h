// np_rownorm.h — the row norms of np.linalg.norm(A, axis=1) with numpy's exact operation
// order, for the range D the solvers derive every width and logit scale from
// (R/ses.py:65-72: max_i |v_1 - v_i| + g_1 + g_i; R/svm.py:62-66: max_i |x_i|).
//
// np.linalg.norm(A, axis=1) of a real C-contiguous A is sqrt(add.reduce(A * A, axis=1));
// the reduction along a contiguous row is numpy's pairwise summation (DOUBLE_pairwise_sum,
// numpy/_core/src/umath/loops_utils.h.src): n < 8 sequential from 0.0; n <= 128 eight
// interleaved accumulators combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the
// n % 8 tail in order; n > 128 split at n/2 rounded down to a multiple of 8.  Products
// and sums are separately rounded (no fused multiply-add).  Checked bit for bit against
// numpy in tests/test_range.py (CPU, through the emulator) and tests/test_gpu_range.py.
#pragma once

#ifdef __CUDACC__
#define SC_NP_HD __host__ __device__ __forceinline__
#else
#define SC_NP_HD inline
#endif

namespace scmwu {

SC_NP_HD double np_add(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dadd_rn(a, b);
#else
    return a + b;
#endif
}
SC_NP_HD double np_sq(double x, const double* anchor, int j) {
#ifdef __CUDA_ARCH__
    const double v = anchor ? __dsub_rn(x, anchor[j]) : x;
    return __dmul_rn(v, v);
#else
    const double v = anchor ? x - anchor[j] : x;
    return v * v;
#endif
}

// sum of (x_j - anchor_j)^2 (anchor NULL: x_j^2) over j < n, numpy's pairwise order, for
// one block of n <= 128 elements
SC_NP_HD double np_block_sumsq(const double* x, const double* anchor, int n) {
    if (n < 8) {
        double res = 0.0;
        for (int i = 0; i < n; ++i) res = np_add(res, np_sq(x[i], anchor, i));
        return res;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = np_sq(x[j], anchor, j);
    int i = 8;
    for (; i < n - n % 8; i += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = np_add(r[j], np_sq(x[i + j], anchor, i + j));
    }
    double res = np_add(np_add(np_add(r[0], r[1]), np_add(r[2], r[3])),
                        np_add(np_add(r[4], r[5]), np_add(r[6], r[7])));
    for (; i < n; ++i) res = np_add(res, np_sq(x[i], anchor, i));
    return res;
}

// the recursive split for n > 128 (DEPTH levels: n <= 128 * 2^DEPTH; d <= 512 needs 2)
template <int DEPTH>
SC_NP_HD double np_sumsq(const double* x, const double* anchor, int n) {
    if constexpr (DEPTH > 0) {
        if (n > 128) {
            int n2 = n / 2;
            n2 -= n2 % 8;
            return np_add(np_sumsq<DEPTH - 1>(x, anchor, n2),
                          np_sumsq<DEPTH - 1>(x + n2, anchor ? anchor + n2 : nullptr, n - n2));
        }
    }
    return np_block_sumsq(x, anchor, n);
}

constexpr int kNpDepth = 4;   // rows up to 2048 elements

// the per-row term of the range: SES (|x - v1| + g1) + g_i (R/ses.py:70-71), SVM |x|
SC_NP_HD double np_range_term(const double* x, const double* anchor, int d, double g1,
                              double gi, bool ses) {
    const double nrm = sqrt(np_sumsq<kNpDepth>(x, anchor, d));
    return ses ? np_add(np_add(nrm, g1), gi) : nrm;
}

}  // namespace scmwu
