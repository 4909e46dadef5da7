// scmwu_kernel.cuh — the persistent SCMWU kernel of the B200 engine (include/scmwu.h).
//
// One sc_ftp call = one cooperative launch of a persistent kernel with one CTA
// per SM (grid G <= 148).  Every MWU iteration is ONE streaming pass over the
// point matrix X (n x d fp64, row-sharded across CTAs):
//
//   producer warp   cp.async.bulk (1-D TMA) of X tiles (+ radii) into an
//                   S-stage shared-memory ring, mbarrier full/empty handshake;
//                   it keeps prefetching the next pass while the consumers sit
//                   in the grid reduction and the control tail, so HBM never idles.
//   consumer warps  lane groups of LPR lanes own one row each; CPL columns per
//                   lane live in registers.  Per row: the closed-form cone
//                   exponential (2 exp for SES, 1 for SVM), the oracle sums and
//                   every deferred check.  Partials are reduced
//                   warp -> CTA -> global (fixed order, deterministic).
//   grid reduction  partials[G][RW] in HBM/L2, barrier, column-distributed fold,
//                   barrier, every CTA reads the RW reduced values.
//   control tail    warp 0 of every CTA runs scmwu_control.h redundantly (same
//                   inputs -> same decisions, no broadcast needed).
//
// Reference hot path replaced (R = /root/reference/pkg/src/symcone/):
//   Scmwu.current/observe  R/mwu.py:57-70 -> cones.normalized_exp R/cones.py:399-420,
//   inf_norm R/cones.py:349-361, ses_oracle R/ses.py:90-132, ses_progress
//   R/ses.py:82-87, svm_oracle R/svm.py:97-127, svm_progress R/svm.py:87-94,
//   pd_counter R/svm.py:173-181, the loops of solve_ftp R/meta.py:313-364 and
//   refine_run R/meta.py:499-568.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "scmwu_control.h"

#pragma once

namespace scmwu {

constexpr int kNW = 7;                      // consumer warps (8 warps total: 255 regs)
constexpr int kThreads = (kNW + 1) * 32;    // + 1 producer warp
constexpr int kNumSlots = 5;                // pending, callmin, sep, best, last
constexpr double kInvSqrt2 = 0.7071067811865476;
constexpr int kMaxSmem = 232448;            // 227 KB opt-in per CTA on sm_100

struct WarpLanes {
    __host__ __device__ static int lane() {
#ifdef __CUDA_ARCH__
        return threadIdx.x & 31;
#else
        return 0;
#endif
    }
    __host__ __device__ static int nl() {
#ifdef __CUDA_ARCH__
        return 32;
#else
        return 1;
#endif
    }
    __host__ __device__ static double sum(double x) {
#ifdef __CUDA_ARCH__
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
#endif
        return x;
    }
    __host__ __device__ static void sync() {
#ifdef __CUDA_ARCH__
        __syncwarp();
#endif
    }
    __host__ __device__ static double ldcg(const double* p) {
#ifdef __CUDA_ARCH__
        return __ldcg(p);
#else
        return *p;
#endif
    }
};

// --------------------------------------------------------------------------------------
// kernel parameters
struct KParams {
    int kind, d, ld, dd, rw, pw;
    int G, gP;                 // grid; SVM: CTAs [0, gP) hold P rows
    int tile_rows, stages, resident;
    int64_t n, n1;
    const double* X;           // n x ld (ld even, padded with zeros)
    const double* radii;       // SES: n rounded up to even (zero padded)
    const int64_t* row_begin;  // G + 1
    double rho, inv_rho, R, ln_r, D, g1;
    const double* red0;        // reduced vector of iterate 1 (all logits 0)
    double* partials;          // G x rw
    double* redg;              // rw
    unsigned long long* bar;   // grid barrier counter (zeroed per launch)
    double* ring;
    int64_t ring_cap;
    double* slots;             // kNumSlots x slot_len
    int slot_len;
    sc_ftp_args args;
    sc_ftp_result* res;
    double* y_tilde;
    double* best_y;
    int* status;
    uint32_t stage_stride;     // bytes per ring stage
    uint32_t rad_off;          // byte offset of the radii inside a stage
};

// --------------------------------------------------------------------------------------
// PTX helpers: mbarrier + 1-D bulk async copy (TMA)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* b, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    while (!mbar_try_wait(b, parity)) {
    }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* b) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
        "[%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(b))
        : "memory");
}
__device__ __forceinline__ void consumer_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(kNW * 32) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// grid barrier among the consumer warps of all CTAs (co-residency guaranteed by the
// cooperative launch); `target` = (barrier ordinal) * G.
__device__ __forceinline__ void grid_barrier(unsigned long long* bar, unsigned long long target) {
    consumer_sync();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1ull);
        while (ld_acquire(bar) < target) {
        }
        __threadfence();
    }
    consumer_sync();
}

// --------------------------------------------------------------------------------------
// combine operators of the reduced layout
enum Op { kSum = 0, kMax = 1, kMin = 2 };
__host__ __device__ __forceinline__ int red_op(int kind, int j) {
    if (kind == SC_SES) {
        if (j == kS_M || j == kS_F || j == kS_Wd || j == kS_Fw) return kMax;
        return kSum;
    }
    switch (j) {
        case kV_M: case kV_Wd: case kV_maxQW: case kV_maxQy: case kV_maxQz: return kMax;
        case kV_minresP: case kV_minresQ: case kV_minPW: case kV_minPy: case kV_minPz:
            return kMin;
        default: return kSum;
    }
}
__host__ __device__ __forceinline__ double op_identity(int op) {
    return op == kSum ? 0.0 : (op == kMax ? -INFINITY : INFINITY);
}
__device__ __forceinline__ double op_apply(int op, double a, double b) {
    return op == kSum ? a + b : (op == kMax ? fmax(a, b) : fmin(a, b));
}
// SVM: the partial column (one side) feeding reduced column j, and which side owns it
// (0 = both, 1 = P, 2 = Q)
__device__ __forceinline__ void svm_src(int d, int j, int& pc, int& side) {
    switch (j) {
        case kV_TP: pc = kP_T; side = 1; return;
        case kV_TQ: pc = kP_T; side = 2; return;
        case kV_M: pc = kP_M; side = 0; return;
        case kV_minresP: pc = kP_minres; side = 1; return;
        case kV_minresQ: pc = kP_minres; side = 2; return;
        case kV_Wd: pc = kP_Wd; side = 0; return;
        case kV_minPW: pc = kP_extW; side = 1; return;
        case kV_maxQW: pc = kP_extW; side = 2; return;
        case kV_minPy: pc = kP_extY; side = 1; return;
        case kV_maxQy: pc = kP_extY; side = 2; return;
        case kV_minPz: pc = kP_extZ; side = 1; return;
        case kV_maxQz: pc = kP_extZ; side = 2; return;
        default:
            if (j < kV_Vec + d) { pc = kP_Vec + (j - kV_Vec); side = 1; }
            else { pc = kP_Vec + (j - kV_Vec - d); side = 2; }
            return;
    }
}
// in-CTA (warp-partials) combine op of a one-sided SVM partial column
__device__ __forceinline__ int svm_part_op(int j, bool isP) {
    switch (j) {
        case kP_M: case kP_Wd: return kMax;
        case kP_minres: return kMin;
        case kP_extW: case kP_extY: case kP_extZ: return isP ? kMin : kMax;
        default: return kSum;
    }
}

template <int LPR>
__device__ __forceinline__ double group_sum(double x) {
#pragma unroll
    for (int o = LPR / 2; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}
template <int LPR>
__device__ __forceinline__ double across_sum(double x) {
#pragma unroll
    for (int o = LPR; o < 32; o <<= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}
template <int LPR>
__device__ __forceinline__ double across_max(double x) {
#pragma unroll
    for (int o = LPR; o < 32; o <<= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
    return x;
}
template <int LPR>
__device__ __forceinline__ double across_min(double x) {
#pragma unroll
    for (int o = LPR; o < 32; o <<= 1) x = fmin(x, __shfl_xor_sync(0xffffffffu, x, o));
    return x;
}

// --------------------------------------------------------------------------------------
// shared-memory map
struct SmemMap {
    uint64_t* full;
    uint64_t* empty;
    double* vec;       // 10 control vectors of dd8
    double* ytd;       // y_tilde dummy for CTAs != 0
    double* red;       // rw
    double* wpart;     // kNW x pw
    PassParams* pp;
    sc_ftp_result* resd;
    volatile int* flags;  // [0] done, [1] consumed tiles
    unsigned char* ring;
};

__host__ __device__ inline int dd8_of(int dd) { return (dd + 1) & ~1; }

__host__ __device__ inline size_t smem_fixed_bytes(int dd, int rw, int pw, int stages) {
    size_t b = 0;
    b += 2 * (size_t)stages * 8;                       // mbarriers
    b += 11 * (size_t)dd8_of(dd) * 8;                  // control vectors + y_tilde dummy
    b += (size_t)((rw + 1) & ~1) * 8;                  // red
    b += (size_t)kNW * ((pw + 1) & ~1) * 8;            // warp partials
    b += sizeof(PassParams) + sizeof(sc_ftp_result) + 64;
    return (b + 127) & ~(size_t)127;
}

__device__ inline SmemMap carve(unsigned char* base, const KParams& p) {
    SmemMap m;
    m.ring = base;
    size_t off = (size_t)p.stages * p.stage_stride;
    m.full = reinterpret_cast<uint64_t*>(base + off);
    m.empty = m.full + p.stages;
    off += 2 * (size_t)p.stages * 8;
    const int dd8 = dd8_of(p.dd);
    m.vec = reinterpret_cast<double*>(base + off);
    off += 10 * (size_t)dd8 * 8;
    m.ytd = reinterpret_cast<double*>(base + off);
    off += (size_t)dd8 * 8;
    m.red = reinterpret_cast<double*>(base + off);
    off += (size_t)((p.rw + 1) & ~1) * 8;
    m.wpart = reinterpret_cast<double*>(base + off);
    off += (size_t)kNW * ((p.pw + 1) & ~1) * 8;
    m.pp = reinterpret_cast<PassParams*>(base + off);
    off += sizeof(PassParams);
    m.resd = reinterpret_cast<sc_ftp_result*>(base + off);
    off += sizeof(sc_ftp_result);
    m.flags = reinterpret_cast<volatile int*>(base + off);
    return m;
}

// --------------------------------------------------------------------------------------
// producer: stream this CTA's tiles through the ring, pass after pass
static __device__ void producer(const KParams& p, const SmemMap& m, int64_t r0, int64_t r1,
                         int ntiles) {
    if ((threadIdx.x & 31) != 0) return;
    const int S = p.stages;
    int64_t issued = 0;
    auto issue = [&](int64_t seq) {
        const int stage = (int)(seq % S);
        const int tile = (int)(seq % ntiles);
        const int64_t a = r0 + (int64_t)tile * p.tile_rows;
        const int64_t b = min(r1, a + (int64_t)p.tile_rows);
        unsigned char* dst = m.ring + (size_t)stage * p.stage_stride;
        const uint32_t xb = (uint32_t)((b - a) * p.ld * 8);
        uint32_t bytes = xb;
        int64_t ra = 0, rb = 0;
        if (p.kind == SC_SES) {
            ra = a & ~(int64_t)1;
            rb = (b + 1) & ~(int64_t)1;
            bytes += (uint32_t)((rb - ra) * 8);
        }
        mbar_arrive_tx(&m.full[stage], bytes);
        bulk_g2s(dst, p.X + a * p.ld, xb, &m.full[stage]);
        if (p.kind == SC_SES)
            bulk_g2s(dst + p.rad_off, p.radii + ra, (uint32_t)((rb - ra) * 8), &m.full[stage]);
    };
    if (p.resident) {
        for (int64_t s = 0; s < ntiles; ++s) issue(s);
        issued = ntiles;
    } else {
        for (;;) {
            const int stage = (int)(issued % S);
            const int64_t k = issued / S;
            bool quit = false;
            if (k > 0) {
                const uint32_t par = (uint32_t)((k - 1) & 1);
                while (!mbar_try_wait(&m.empty[stage], par)) {
                    if (m.flags[0]) { quit = true; break; }
                }
            }
            if (quit || m.flags[0]) break;
            issue(issued);
            ++issued;
        }
    }
    // wait for the completion of every copy still in flight before the CTA exits
    while (!m.flags[0]) {
    }
    __threadfence_block();
    const int64_t consumed = p.resident ? 0 : (int64_t)m.flags[1];
    for (int64_t s = consumed; s < issued; ++s) {
        const int stage = (int)(s % S);
        mbar_wait(&m.full[stage], (uint32_t)((s / S) & 1));
    }
}

// --------------------------------------------------------------------------------------
// consumer pass over this CTA's rows: SES
template <int LPR, int CPL, bool CHECK>
__device__ void ses_pass(const KParams& p, const SmemMap& m, const PassParams& pp,
                         int64_t r0, int64_t r1, int ntiles, int64_t& consumed, int pass_idx) {
    constexpr int RPW = 32 / LPR;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grp = lane / LPR, l = lane % LPR;
    const int d = p.d, ld = p.ld, dd8 = dd8_of(p.dd);
    const double* ysum = m.vec;
    const double* yprev = m.vec + dd8;
    const double* ywin = m.vec + 5 * dd8;
    double U[CPL], up[CPL], Sd[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        const int j = l + LPR * c;
        U[c] = j < d ? ysum[j] : 0.0;
        up[c] = j < d ? yprev[j] : 0.0;
        Sd[c] = 0.0;
    }
    const double t = pp.t, er = pp.eta_rho, al = pp.alpha, sh = pp.shift;
    const double er_t = er * t;
    double T = 0, Lin = 0, Rad = 0, M = -INFINITY, F = -INFINITY, Wd = 0, Fw = -INFINITY;
    const double inv_t = 1.0 / t;
    for (int tile = 0; tile < ntiles; ++tile, ++consumed) {
        const int stage = p.resident ? tile : (int)(consumed % p.stages);
        if (!p.resident || pass_idx == 0)
            mbar_wait(&m.full[stage], p.resident ? 0u : (uint32_t)((consumed / p.stages) & 1));
        const int64_t a = r0 + (int64_t)tile * p.tile_rows;
        const int nr = (int)(min(r1, a + (int64_t)p.tile_rows) - a);
        const double* xs = reinterpret_cast<const double*>(m.ring + (size_t)stage * p.stage_stride);
        const double* rs = reinterpret_cast<const double*>(m.ring + (size_t)stage * p.stage_stride +
                                                           p.rad_off) +
                           (a & 1);
        for (int base = warp * RPW; base < nr; base += kNW * RPW) {
            const int r = base + grp;
            const bool valid = r < nr;
            const double* xr = xs + (size_t)(valid ? r : 0) * ld;
            double df[CPL];
            double aa = 0, ll = 0, w2 = 0, f2 = 0;
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                const int j = l + LPR * c;
                if (j < d) {
                    const double v = xr[j];
                    const double x = fma(-t, v, U[c]);
                    df[c] = x;
                    aa = fma(x, x, aa);
                    ll = fma(v, x, ll);
                    const double w = up[c] - v;
                    w2 = fma(w, w, w2);
                    if (CHECK) {
                        const double y = ywin[j] - v;
                        f2 = fma(y, y, f2);
                    }
                } else {
                    df[c] = 0.0;
                }
            }
            aa = group_sum<LPR>(aa);
            ll = group_sum<LPR>(ll);
            w2 = group_sum<LPR>(w2);
            if (CHECK) f2 = group_sum<LPR>(f2);
            double cc = 0.0;
            if (valid) {
                const double g = rs[r];
                const double ra = sqrt(aa);
                F = fmax(F, ra * inv_t + g);
                if (CHECK) Fw = fmax(Fw, sqrt(f2) + g);
                if (a + r > 0) {
                    const double nrm = er * ra;
                    const double x0 = -er_t * (al - g);
                    const double lp = (x0 + nrm) * kInvSqrt2, lm = (x0 - nrm) * kInvSqrt2;
                    const double A = exp(lp - sh), B = exp(lm - sh);
                    cc = nrm > 0.0 ? (A - B) / (kSqrt2 * nrm) : 0.0;
                    T += A + B;
                    Lin = fma(cc, ll, Lin);
                    Rad = fma(g, A + B, Rad);
                    M = fmax(M, lp);
                    Wd = fmax(Wd, (fabs(al - g) + sqrt(w2)) * kInvSqrt2);
                }
            }
#pragma unroll
            for (int c = 0; c < CPL; ++c) Sd[c] = fma(cc, df[c], Sd[c]);
        }
        if (!p.resident) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&m.empty[stage]);
        }
    }
    // warp reduction across lane groups (scalars identical inside a group)
    T = across_sum<LPR>(T);
    Lin = across_sum<LPR>(Lin);
    Rad = across_sum<LPR>(Rad);
    M = across_max<LPR>(M);
    F = across_max<LPR>(F);
    Wd = across_max<LPR>(Wd);
    Fw = across_max<LPR>(Fw);
    double* wp = m.wpart + (size_t)warp * ((p.pw + 1) & ~1);
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        const double s = across_sum<LPR>(Sd[c]);
        const int j = l + LPR * c;
        if (grp == 0 && j < d) wp[kS_Vec + j] = s;
    }
    if (lane == 0) {
        wp[kS_T] = T; wp[kS_Lin] = Lin; wp[kS_Rad] = Rad; wp[kS_M] = M;
        wp[kS_F] = F; wp[kS_Wd] = Wd; wp[kS_Fw] = Fw;
    }
}

// consumer pass: SVM (this CTA holds one side)
template <int LPR, int CPL, bool CHECK>
__device__ void svm_pass(const KParams& p, const SmemMap& m, const PassParams& pp,
                         int64_t r0, int64_t r1, int ntiles, int64_t& consumed, int pass_idx,
                         bool isP) {
    constexpr int RPW = 32 / LPR;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grp = lane / LPR, l = lane % LPR;
    const int d = p.d, ld = p.ld, dd8 = dd8_of(p.dd);
    const double* ysum = m.vec;
    const double* yprev = m.vec + dd8;
    const double* ywin = m.vec + 5 * dd8;
    const double* zv = m.vec + 6 * dd8;
    double W[CPL], wp_[CPL], G[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        const int j = l + LPR * c;
        W[c] = j < d ? ysum[j] : 0.0;
        wp_[c] = j < d ? yprev[j] : 0.0;
        G[c] = 0.0;
    }
    const double sg = isP ? 1.0 : -1.0;
    const double S = isP ? pp.S1 : pp.S2;
    const double sp = isP ? pp.s1p : pp.s2p;
    const double er = pp.eta_rho, sh = pp.shift;
    double T = 0, M = -INFINITY, mres = INFINITY, Wd = 0;
    double eW = isP ? INFINITY : -INFINITY, eY = eW, eZ = eW;
    for (int tile = 0; tile < ntiles; ++tile, ++consumed) {
        const int stage = p.resident ? tile : (int)(consumed % p.stages);
        if (!p.resident || pass_idx == 0)
            mbar_wait(&m.full[stage], p.resident ? 0u : (uint32_t)((consumed / p.stages) & 1));
        const int64_t a = r0 + (int64_t)tile * p.tile_rows;
        const int nr = (int)(min(r1, a + (int64_t)p.tile_rows) - a);
        const double* xs = reinterpret_cast<const double*>(m.ring + (size_t)stage * p.stage_stride);
        for (int base = warp * RPW; base < nr; base += kNW * RPW) {
            const int r = base + grp;
            const bool valid = r < nr;
            const double* xr = xs + (size_t)(valid ? r : 0) * ld;
            double xv[CPL];
            double dW = 0, dw = 0, dy = 0, dz = 0;
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                const int j = l + LPR * c;
                const double x = j < d ? xr[j] : 0.0;
                xv[c] = x;
                dW = fma(x, W[c], dW);
                dw = fma(x, wp_[c], dw);
                if (CHECK && j < d) {
                    dy = fma(x, ywin[j], dy);
                    dz = fma(x, zv[j], dz);
                }
            }
            dW = group_sum<LPR>(dW);
            dw = group_sum<LPR>(dw);
            if (CHECK) {
                dy = group_sum<LPR>(dy);
                dz = group_sum<LPR>(dz);
            }
            double e = 0.0;
            if (valid) {
                const double lg = -er * (sg * dW - S);
                e = exp(lg - sh);
                T += e;
                M = fmax(M, lg);
                const double res = sg * dw - sp;
                Wd = fmax(Wd, fabs(res));
                mres = fmin(mres, res);
                if (isP) {
                    eW = fmin(eW, dW);
                    if (CHECK) { eY = fmin(eY, dy); eZ = fmin(eZ, dz); }
                } else {
                    eW = fmax(eW, dW);
                    if (CHECK) { eY = fmax(eY, dy); eZ = fmax(eZ, dz); }
                }
            }
#pragma unroll
            for (int c = 0; c < CPL; ++c) G[c] = fma(e, xv[c], G[c]);
        }
        if (!p.resident) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&m.empty[stage]);
        }
    }
    T = across_sum<LPR>(T);
    M = across_max<LPR>(M);
    mres = across_min<LPR>(mres);
    Wd = across_max<LPR>(Wd);
    if (isP) {
        eW = across_min<LPR>(eW); eY = across_min<LPR>(eY); eZ = across_min<LPR>(eZ);
    } else {
        eW = across_max<LPR>(eW); eY = across_max<LPR>(eY); eZ = across_max<LPR>(eZ);
    }
    double* wpp = m.wpart + (size_t)warp * ((p.pw + 1) & ~1);
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        const double s = across_sum<LPR>(G[c]);
        const int j = l + LPR * c;
        if (grp == 0 && j < d) wpp[kP_Vec + j] = s;
    }
    if (lane == 0) {
        wpp[kP_T] = T; wpp[kP_M] = M; wpp[kP_minres] = mres; wpp[kP_Wd] = Wd;
        wpp[kP_extW] = eW; wpp[kP_extY] = eY; wpp[kP_extZ] = eZ;
    }
}

// --------------------------------------------------------------------------------------
// the persistent kernel
template <int KIND, int LPR, int CPL>
__global__ void __launch_bounds__(kThreads, 1) scmwu_kernel(const KParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    const SmemMap m = carve(smem, p);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x;
    const int64_t r0 = p.row_begin[b], r1 = p.row_begin[b + 1];
    const int ntiles = (int)((r1 - r0 + p.tile_rows - 1) / p.tile_rows);
    const bool isP = KIND == SC_SVM && b < p.gP;
    if (threadIdx.x == 0) {
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(&m.full[s], 1);
            mbar_init(&m.empty[s], kNW);
        }
        m.flags[0] = 0;
        m.flags[1] = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == kNW) {
        if (ntiles > 0) producer(p, m, r0, r1, ntiles);
        else if (lane == 0) { while (!m.flags[0]) { } }
        __syncthreads();
        return;
    }

    // ------------------------------------------------------------ consumers
    const int dd8 = dd8_of(p.dd);
    const int tid = threadIdx.x;
    Control<WarpLanes> ctl;
    PassParams* pp = m.pp;
    double* y_tilde = b == 0 ? p.y_tilde : m.ytd;
    if (warp == 0) {
        ctl.kind = KIND; ctl.d = p.d; ctl.dd = p.dd; ctl.is_max = KIND == SC_SES;
        ctl.rho = p.rho; ctl.inv_rho = p.inv_rho; ctl.R = p.R; ctl.ln_r = p.ln_r;
        ctl.D = p.D; ctl.g1 = p.g1;
        ctl.res = b == 0 ? p.res : m.resd;
        ctl.writer = b == 0;
        double* V = m.vec;
        ctl.v = CtlVecs{V, V + dd8, V + 2 * dd8, V + 3 * dd8, V + 4 * dd8, V + 5 * dd8,
                        V + 6 * dd8, V + 7 * dd8, V + 8 * dd8, V + 9 * dd8};
        const int sl = p.slot_len;
        ctl.s = CtlSlots{p.ring, p.ring_cap, p.slots, p.slots + sl, p.slots + 2 * sl,
                         p.slots + 4 * sl};
        for (int j = lane; j < dd8; j += 32) {
            for (int q = 0; q < 10; ++q) V[q * dd8 + j] = 0.0;
            if (KIND == SC_SES && j < p.d) V[9 * dd8 + j] = p.X[j];   // anchor v1
        }
        __syncwarp();
        int act = ctl.begin(p.args, p.red0, y_tilde, nullptr, pp);
        if (lane == 0) pp->action = act;
    }
    consumer_sync();

    int64_t consumed = 0;
    int pass_idx = 0;
    unsigned long long nbar = 0;
    // columns of the reduced vector folded by this CTA
    const int c0 = (int)((int64_t)b * p.rw / p.G), c1 = (int)((int64_t)(b + 1) * p.rw / p.G);
    while (pp->action == kPass) {
        const PassParams ps = *pp;
        if (ntiles > 0) {
            if (KIND == SC_SES) {
                if (ps.check) ses_pass<LPR, CPL, true>(p, m, ps, r0, r1, ntiles, consumed, pass_idx);
                else ses_pass<LPR, CPL, false>(p, m, ps, r0, r1, ntiles, consumed, pass_idx);
            } else {
                if (ps.check)
                    svm_pass<LPR, CPL, true>(p, m, ps, r0, r1, ntiles, consumed, pass_idx, isP);
                else
                    svm_pass<LPR, CPL, false>(p, m, ps, r0, r1, ntiles, consumed, pass_idx, isP);
            }
        }
        consumer_sync();
        // CTA partial, fixed warp order, written in the reduced layout
        const int pws = (p.pw + 1) & ~1;
        for (int j = tid; j < p.rw; j += kNW * 32) {
            double v;
            if (KIND == SC_SES) {
                const int op = red_op(KIND, j);
                v = op_identity(op);
                if (ntiles > 0)
                    for (int w = 0; w < kNW; ++w) v = op_apply(op, v, m.wpart[w * pws + j]);
            } else {
                int pc, side;
                svm_src(p.d, j, pc, side);
                const int op = red_op(KIND, j);
                v = op_identity(op);
                const bool mine = side == 0 || (side == 1) == isP;
                if (mine && ntiles > 0) {
                    const int pop = svm_part_op(pc, isP);
                    double acc = op_identity(pop);
                    for (int w = 0; w < kNW; ++w) acc = op_apply(pop, acc, m.wpart[w * pws + pc]);
                    v = acc;
                }
            }
            p.partials[(size_t)b * p.rw + j] = v;
        }
        grid_barrier(p.bar, (++nbar) * (unsigned long long)p.G);
        // column-distributed fold over the G partials: warp per column, fixed tree
        for (int j = c0 + warp; j < c1; j += kNW) {
            const int op = red_op(KIND, j);
            double acc = op_identity(op);
            for (int q = lane; q < p.G; q += 32)
                acc = op_apply(op, acc, __ldcg(p.partials + (size_t)q * p.rw + j));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
                acc = op_apply(op, acc, __shfl_xor_sync(0xffffffffu, acc, o));
            if (lane == 0) p.redg[j] = acc;
        }
        grid_barrier(p.bar, (++nbar) * (unsigned long long)p.G);
        for (int j = tid; j < p.rw; j += kNW * 32) m.red[j] = __ldcg(p.redg + j);
        consumer_sync();
        if (warp == 0) {
            int act = ctl.after_pass(m.red, p.red0, y_tilde, pp);
            if (lane == 0) pp->action = act;
        }
        consumer_sync();
        ++pass_idx;
    }
    // stop the producer, then publish the result (CTA 0)
    if (tid == 0) {
        m.flags[1] = (int)consumed;
        __threadfence_block();
        m.flags[0] = 1;
    }
    if (b == 0 && warp == 0) {
        for (int j = lane; j < p.dd; j += 32) p.best_y[j] = ctl.v.besty[j];
        if (lane == 0) {
            *p.status = ctl.status;
            p.res->passes = pass_idx;
        }
    }
    __syncthreads();
}

typedef void (*KernelFn)(const KParams);

}  // namespace scmwu

// explicit instantiation + lookup, used by the scmwu_inst_*.cu translation units
#define SCMWU_INST(K, L, C)                                                            \
    template __global__ void scmwu::scmwu_kernel<K, L, C>(const scmwu::KParams);
#define SCMWU_MATCH(K, L, C) \
    if (kind == K && lpr == L && cpl == C) return scmwu::scmwu_kernel<K, L, C>;
