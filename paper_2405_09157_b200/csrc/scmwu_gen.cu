// scmwu_gen.cu — on-device instance generation (sc_create_generated):
// rows drawn in HBM with a counter-based Philox keyed by (seed, global row), and the
// range D computed on the way.
#include <string.h>

#include <algorithm>

#include "np_rownorm.h"
#include "scmwu_handle.h"

namespace scmwu {
// -------------------------------------------------------------------------------------
// On-device instance generation (sc_create_generated).  Counter-based Philox4x32-10
// keyed by the seed; the counter is (column pair, global row, stream), so a row's values
// do not depend on which rank generates it or in which order.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

// uniform in (0, 1) from 53 random bits
__device__ __forceinline__ double unit_open(uint32_t a, uint32_t b) {
    const uint64_t m = ((uint64_t)a << 21) ^ (uint64_t)(b >> 11);
    return ((double)m + 0.5) * 0x1p-53;
}

// two standard normals (Box-Muller) for columns 2c, 2c+1 of generator row `row`
__device__ __forceinline__ void normal_pair(uint64_t seed, uint64_t row, uint32_t c,
                                            uint32_t stream, double& z0, double& z1) {
    const uint4 r = philox4x32_10(make_uint4(c, (uint32_t)row, (uint32_t)(row >> 32), stream),
                                  make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
    const double rad = sqrt(-2.0 * log(unit_open(r.x, r.y)));
    double s, co;
    sincospi(2.0 * unit_open(r.z, r.w), &s, &co);
    z0 = rad * co;
    z1 = rad * s;
}

// One warp per row.  Rows [grow0, grow0 + rows) of the global instance are written to
// X (row stride ld; the padding column, if any, is zeroed).  dist: sc_gen_dist.  For
// SC_GEN_SVM_CLUSTERS rows g < n1 are P (+shift * dir), the rest Q (-shift * dir).
// dmax (optional) receives the max over the rows of |x_g - anchor| (anchor NULL: |x_g|)
// as the bit pattern of a non-negative double.
__global__ void gen_kernel(double* X, int ld, int d, int64_t rows, int64_t grow0, int dist,
                           uint64_t seed, int64_t n_global, int64_t n1, double shift,
                           const double* dir, const double* anchor,
                           unsigned long long* dmax) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int pairs = (d + 1) >> 1;
    double best = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < rows;
         i += warps) {
        const int64_t g = grow0 + i;
        // sphere surface: antipodal pairs (row k+j = -row j), the odd last row its own
        int64_t src = g;
        double sign = 1.0;
        if (dist == 2) {
            const int64_t k = n_global / 2;
            if (g >= k) src = g - k;
            if (g >= k && g < 2 * k) sign = -1.0;
        }
        double nrm2 = 0.0;
        for (int c = lane; c < pairs; c += 32) {
            double z0, z1;
            normal_pair(seed, (uint64_t)src, (uint32_t)c, 0u, z0, z1);
            nrm2 += z0 * z0;
            if (2 * c + 1 < d) nrm2 += z1 * z1;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) nrm2 += __shfl_xor_sync(0xffffffffu, nrm2, o);
        double scale = 1.0, off = 0.0;
        if (dist != 0) {
            scale = sign / sqrt(nrm2);
            if (dist == 1 || dist == 3) {
                const uint4 r = philox4x32_10(
                    make_uint4(0xFFFFFFFFu, (uint32_t)src, (uint32_t)(src >> 32), 1u),
                    make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
                scale *= pow(unit_open(r.x, r.y), 1.0 / (double)d);
            }
            if (dist == 3) off = g < n1 ? shift : -shift;
        }
        double* row = X + i * (int64_t)ld;
        double acc = 0.0;
        for (int c = lane; c < pairs; c += 32) {
            double z0, z1;
            normal_pair(seed, (uint64_t)src, (uint32_t)c, 0u, z0, z1);
            const int j = 2 * c;
            double x0 = z0 * scale, x1 = z1 * scale;
            if (dist == 3) {
                x0 += off * dir[j];
                if (j + 1 < d) x1 += off * dir[j + 1];
            }
            const double a0 = anchor ? x0 - anchor[j] : x0;
            acc += a0 * a0;
            row[j] = x0;
            if (j + 1 < d) {
                const double a1 = anchor ? x1 - anchor[j + 1] : x1;
                acc += a1 * a1;
                row[j + 1] = x1;
            } else if (j + 1 < ld) {
                row[j + 1] = 0.0;
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        best = fmax(best, sqrt(acc));
    }
    if (dmax && lane == 0 && best > 0.0) atomicMax(dmax, (unsigned long long)__double_as_longlong(best));
}

// order-preserving integer image of a double (atomicMax over the images = max over the
// values, independent of the order the rows are visited in)
__device__ __forceinline__ unsigned long long ord_key(double v) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ inline double ord_value(unsigned long long k) {
    const unsigned long long b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
    double v;
    memcpy(&v, &b, 8);
    return v;
}

// The range term of rows [first, rows) with numpy's operation order (np_rownorm.h): one
// thread per row (a one-off pass; the row's sectors are reused from L1 by the thread's
// next loads).  SES: (|x_i - v1| + g1) + g_i, SVM: |x_i|.
__global__ void range_kernel(const double* X, int ld, int d, int64_t first, int64_t rows,
                             const double* radii, const double* anchor, double g1, int ses,
                             unsigned long long* kmax) {
    double best = -INFINITY;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = first + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows;
         i += stride) {
        const double v = np_range_term(X + i * (int64_t)ld, anchor, d, g1,
                                       ses ? radii[i] : 0.0, ses != 0);
        best = v > best || v != v ? v : best;   // NaN propagates, as in numpy's max
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const double u = __shfl_xor_sync(0xffffffffu, best, o);
        best = u > best || u != u ? u : best;
    }
    if ((threadIdx.x & 31) == 0 && best != -INFINITY) atomicMax(kmax, ord_key(best));
}

}  // namespace scmwu

// D of the resident rows, numpy-exact (R/ses.py:65-72 over global rows >= 1 with the
// anchor v1 and g1 of the handle; R/svm.py:62-66); -inf when this shard has no such row
int sc_row_range(sc_handle* h, double* D_out) {
    if (!h || !D_out) return SC_EARG;
    const sc_problem& P = h->prob;
    const bool ses = P.kind == SC_SES;
    const int64_t first = ses && P.row0 == 0 ? 1 : 0;
    const int64_t rows = P.n_local;
    CK(cudaSetDevice(P.device), "set device");
    unsigned long long* kmax = reinterpret_cast<unsigned long long*>(h->scratch);
    CK(cudaMemsetAsync(kmax, 0, 8, h->stream), "zero range");   // key 0 < key(-inf)
    if (rows > first) {
        const int64_t per = 256;
        const int blocks = (int)std::max<int64_t>(
            1, std::min<int64_t>((int64_t)h->sms * 8, (rows - first + per - 1) / per));
        range_kernel<<<blocks, (int)per, 0, h->stream>>>(h->X, h->ld, P.d, first, rows,
                                                         h->radii, ses ? h->v1 : nullptr,
                                                         h->g1, ses ? 1 : 0, kmax);
        ++h->launches;
        CK(cudaGetLastError(), "range kernel");
    }
    unsigned long long k = 0;
    CK(h_get(h, &k, kmax, 8), "read range");
    *D_out = k == 0 ? -INFINITY : ord_value(k);
    return SC_OK;
}

// Draw this handle's rows (and, SES, the anchor row 0) into HBM; *D_out receives the range
// over this shard's rows (SES max_i |v_1 - v_i|, SVM max_i |x_i|).
int generate_rows(sc_handle* h, const sc_gen* gen, double* D_out) {
    const sc_problem& P = h->prob;
    const sc_problem* prob = &h->prob;
    const int d = P.d;
    const int64_t n = P.n_local;
    // every rank draws the global anchor row 0 itself (SES), then its own rows
    // the handle's scratch (2 x 4096 doubles): the range word, then the SVM direction
    unsigned long long* dmax = reinterpret_cast<unsigned long long*>(h->scratch);
    double* dir = nullptr;
    CK(cudaMemsetAsync(dmax, 0, 8, h->stream), "zero range");
    double shift = 0.0;
    if (prob->kind == SC_SVM) {
        dir = h->scratch + 8;
        CK(h_put(h, dir, gen->direction, (size_t)d * 8), "copy direction");
        shift = 1.0 + gen->gap / 2.0;
    } else {
        gen_kernel<<<1, 32, 0, h->stream>>>(h->v1, d, d, 1, 0, gen->dist, gen->seed, P.n,
                                            0, 0.0, nullptr, nullptr, nullptr);
    }
    const int blocks = (int)std::min<int64_t>((int64_t)h->sms * 8, (n + 7) / 8);
    gen_kernel<<<blocks, 256, 0, h->stream>>>(
        h->X, h->ld, d, n, P.row0, gen->dist, gen->seed, P.n, P.n1, shift, dir,
        prob->kind == SC_SES ? h->v1 : nullptr, dmax);
    h->launches += prob->kind == SC_SES ? 2 : 1;
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    unsigned long long bits = 0;
    if (e == cudaSuccess) e = h_get(h, &bits, dmax, 8);
    if (e != cudaSuccess) return cuda_fail(h, e, "generate rows");
    memcpy(D_out, &bits, 8);
    return SC_OK;
}
