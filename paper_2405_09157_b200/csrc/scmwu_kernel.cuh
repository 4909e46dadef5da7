// scmwu_kernel.cuh — the persistent SCMWU kernel of the B200 engine (include/scmwu.h).
//
// One sc_ftp call = one cooperative launch of a persistent kernel with one CTA
// per SM (grid G <= 148).  Every MWU iteration is ONE streaming pass over the
// point matrix X (n x d fp64, row-sharded across CTAs):
//
//   streaming       every warp owns every 8th warp tile (TRW rows + radii) of its
//                   CTA's rows and keeps SW of them in flight in its own shared-
//                   memory ring: lane 0 issues cp.async.bulk (1-D TMA) copies that
//                   complete on per-stage mbarriers; the stream wraps into the next
//                   pass, so those copies land during the grid reduction and tail.
//   compute         lane groups of LPR lanes own one row, CPL columns per lane in
//                   registers; NB row-groups are reduced together by a shuffle
//                   reduce-scatter so every lane then runs the per-row scalar math
//                   (closed-form cone exponential: 2 exp for SES, 1 for SVM) for its
//                   own row; a second sweep over the staged rows accumulates the
//                   weighted d-vector.  Every deferred check rides along
//                   (DESIGN.md §3-4).  Partials: warp -> CTA -> global, fixed order.
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

// Index invariants of the streaming and reduction code, checked in -DSCMWU_CHECKED builds
// (build.py --checked -> libscmwu_checked.so, tests/test_gpu_checked.py): a failed check
// prints the condition and traps, which aborts the whole cooperative launch (no CTA is
// left spinning in a grid barrier).  Compiled out of the product library.
#ifdef SCMWU_CHECKED
#define SC_DCHECK(c)                                                                       \
    do {                                                                                   \
        if (!(c)) {                                                                        \
            printf("SC_DCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, \
                   #c, (int)blockIdx.x, (int)threadIdx.x);                                 \
            __trap();                                                                      \
        }                                                                                  \
    } while (0)
#else
#define SC_DCHECK(c) \
    do {             \
    } while (0)
#endif

#pragma once

namespace scmwu {

constexpr int kNW = 8;                      // warps per CTA; each streams its own tiles
constexpr int kThreads = kNW * 32;          // 256 threads: up to 255 registers
constexpr int kNumSlots = 5;                // pending, callmin, sep, best, last
constexpr double kInvSqrt2 = 0.7071067811865476;
constexpr int kMaxSmem = 232448;            // 227 KB opt-in per CTA on sm_100
constexpr int kMaxWorld = 8;                // GPUs of one NVLink/NVSwitch node
// build variants for A/B measurements (-DSCMWU_LEAN drops the experimental fold modes
// and the multi-GPU exchange from the kernel body)
#ifdef SCMWU_LEAN
constexpr bool kFoldVariants = false, kMultiGpu = false;
#else
constexpr bool kFoldVariants = true, kMultiGpu = true;
#endif

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
    // three independent butterfly sums interleaved (ILP)
    __host__ __device__ static void sum3(double& a, double& b, double& c) {
#ifdef __CUDA_ARCH__
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double x = __shfl_xor_sync(0xffffffffu, a, o);
            const double y = __shfl_xor_sync(0xffffffffu, b, o);
            const double z = __shfl_xor_sync(0xffffffffu, c, o);
            a += x;
            b += y;
            c += z;
        }
#endif
    }
    // two independent butterfly sums interleaved (ILP)
    __host__ __device__ static void sum2(double& a, double& b) {
#ifdef __CUDA_ARCH__
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double x = __shfl_xor_sync(0xffffffffu, a, o);
            const double y = __shfl_xor_sync(0xffffffffu, b, o);
            a += x;
            b += y;
        }
#endif
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
    // asynchronous global -> shared copy of n (even) doubles, 16 bytes per lane-chunk,
    // L2 only (.cg): the ring is rewritten by CTA 0, so L1 must not serve stale lines
    __host__ __device__ static void prefetch(double* dst, const double* src, int n) {
#ifdef __CUDA_ARCH__
        for (int c = (int)(threadIdx.x & 31); c < n / 2; c += 32) {
            const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst + 2 * c);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + 2 * c)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
#else
        for (int j = 0; j < n; ++j) dst[j] = src[j];
#endif
    }
    __host__ __device__ static void prefetch_wait() {
#ifdef __CUDA_ARCH__
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
#endif
    }
};

// --------------------------------------------------------------------------------------
// kernel parameters
struct KParams {
    int kind, d, ld, dd, rw, pw;
    int G, gP;                 // grid; SVM: CTAs [0, gP) hold P rows
    int tile_rows, stages, resident;   // rows per warp tile, stages per warp ring
    int fold_mode;                     // kFoldTwoBarriers / kFoldRedundant / kFoldLast
    int wrap_prefetch;                 // 1: prefetch the next pass during the reduction
    int flush_after_tail;              // 1: issue the next pass's copies after the tail
    int by_smid;                       // 1: work slot = SM id (G == #SMs, balanced rows)
    long long* slot_cycles;            // optional: per slot {streaming cycles, SM id}
    double l2_frac;                    // fraction of every CTA's tiles kept in L2 (0: off)
    int vworld;                        // > 1: emulate that many ranks on this GPU (tests)
    int64_t n, n1;
    const double* X;           // n x ld (ld even, padded with zeros)
    const double* radii;       // SES: n rounded up to even (zero padded)
    const int64_t* row_begin;  // per slot {first row, end row, tile stride, SVM P side}
    double rho, inv_rho, R, ln_r, D, g1;
    const double* red0;        // reduced vector of iterate 1 (all logits 0)
    double* partials;          // 2 (pass parity) x G x rw
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
    long long* timing;         // optional: per-phase clock64 sums of CTA 0 / thread 0
    const double* v1;          // SES anchor row (d values)
    // row sharding across GPUs (world > 1): mailboxes in every rank's HBM, mapped here
    int world, shard;
    int64_t row0;              // global index of this rank's first row
    int64_t pass_base;         // passes run by earlier calls (mailbox parity / flag epochs)
    double* mbox[kMaxWorld];   // rank r's mailbox data [2][world][rw] (peer pointers)
    unsigned long long* mflag[kMaxWorld];   // rank r's arrival flags [world]
    long long xtimeout;        // cycles a rank waits for a peer's exchange flag
    int drop_rank;             // tests only (SCMWU_FAULT_DROP_RANK): this rank never arrives
    // whole-solve residency (sc_solve): the adaptive search runs between the passes
    int solve;
    sc_solve_args sargs;
    const double* seed;        // the seed point (d values)
    sc_solve_result* sres;
    sc_search_step* steps;
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
// the same copy with an L2 eviction-priority hint (createpolicy): rows kept in L2 across
// passes use evict_last, the streamed remainder evict_first
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* b, bool keep) {
    uint64_t pol;
    if (keep)
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    else
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(b)), "l"(pol)
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
// The CTA's writes are ordered before thread 0's release by bar.sync (release is
// cumulative); the other threads' reads are ordered after its acquire by the second
// bar.sync.  No full fences: one L2 reduction plus the acquire polling.
// `abort` (optional): a launch-wide abort word; a CTA that finds it set stops waiting, sets
// sflag[1] and leaves the pass loop, so no CTA is left spinning in a barrier that the
// aborting CTAs never reach (multi-GPU exchange failure).
__device__ __forceinline__ void grid_barrier(unsigned long long* bar, unsigned long long target,
                                             const unsigned long long* abort = nullptr,
                                             volatile int* sflag = nullptr) {
    consumer_sync();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(bar) : "memory");
        while (ld_acquire(bar) < target) {
            if (abort != nullptr && *(volatile const unsigned long long*)abort != 0) {
                sflag[1] = 1;
                break;
            }
#if defined(SCMWU_POLL_NS) && SCMWU_POLL_NS > 0
            __nanosleep(SCMWU_POLL_NS);   // A/B: back off instead of hammering the L2 line
#endif
        }
    }
    consumer_sync();
}
// word of the (zeroed per launch) barrier buffer that carries the abort decision; the
// emulated-rank counters use words 8 .. 8 * (kMaxWorld + 1)
constexpr int kAbortWord = 96;

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
__host__ __device__ __forceinline__ double op_apply(int op, double a, double b) {
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
//
// ring: kNW per-warp rings of SW stages; stage (w, s) holds TRW rows of X (+ radii).
struct SmemMap {
    uint64_t* full;    // [kNW * SW]
    uint64_t* empty;   // [kNW * SW]
    double* vec;       // 10 control vectors of dd8
    double* ytd;       // y_tilde dummy for CTAs != 0
    double* evict;     // prefetched window entry (dd8)
    double* pend;      // pending pd_counter state (dd8 + IterState)
    double* red;       // rw
    double* wpart;     // kNW x pw
    PassParams* pp;
    sc_ftp_result* resd;
    void* ctl;         // the control state between tails (warp 0 holds it in registers
                       // only while the tail runs, so the passes get those registers)
    void* srch;        // the adaptive-search state (sc_solve)
    double* sbest;     // the search's best_y (dd8)
    volatile int* flags;  // spare
    unsigned char* ring;
};

__host__ __device__ inline int dd8_of(int dd) { return (dd + 1) & ~1; }

__host__ __device__ inline size_t smem_fixed_bytes(int dd, int rw, int pw, int nstages) {
    size_t b = 0;
    b += 2 * (size_t)nstages * 8;                      // mbarriers
    b += 12 * (size_t)dd8_of(dd) * 8;                  // control vectors, y_tilde dummy, evict
    b += ((size_t)dd8_of(dd) + sizeof(IterState) / 8) * 8;   // pending state
    b += (size_t)((rw + 1) & ~1) * 8;                  // red
    b += (size_t)kNW * ((pw + 1) & ~1) * 8;            // warp partials
    b += sizeof(PassParams) + sizeof(sc_ftp_result) + 16 * 4 + 64;
    b += sizeof(Control<WarpLanes>) + 16;
    b += sizeof(Search<WarpLanes>) + 16 + (size_t)dd8_of(dd) * 8;   // sc_solve state
    return (b + 127) & ~(size_t)127;
}

__device__ inline SmemMap carve(unsigned char* base, const KParams& p) {
    SmemMap m;
    m.ring = base;
    const int ns = kNW * p.stages;
    size_t off = (size_t)ns * p.stage_stride;
    m.full = reinterpret_cast<uint64_t*>(base + off);
    m.empty = m.full + ns;
    off += 2 * (size_t)ns * 8;
    const int dd8 = dd8_of(p.dd);
    m.vec = reinterpret_cast<double*>(base + off);
    off += 10 * (size_t)dd8 * 8;
    m.ytd = reinterpret_cast<double*>(base + off);
    off += (size_t)dd8 * 8;
    m.evict = reinterpret_cast<double*>(base + off);
    off += (size_t)dd8 * 8;
    m.pend = reinterpret_cast<double*>(base + off);
    off += ((size_t)dd8 + sizeof(IterState) / 8) * 8;
    m.red = reinterpret_cast<double*>(base + off);
    off += (size_t)((p.rw + 1) & ~1) * 8;
    m.wpart = reinterpret_cast<double*>(base + off);
    off += (size_t)kNW * ((p.pw + 1) & ~1) * 8;
    m.pp = reinterpret_cast<PassParams*>(base + off);
    off += sizeof(PassParams);
    m.resd = reinterpret_cast<sc_ftp_result*>(base + off);
    off += sizeof(sc_ftp_result);
    off = (off + 15) & ~(size_t)15;
    m.ctl = base + off;
    off += sizeof(Control<WarpLanes>);
    off = (off + 15) & ~(size_t)15;
    m.srch = base + off;
    off += sizeof(Search<WarpLanes>);
    off = (off + 15) & ~(size_t)15;
    m.sbest = reinterpret_cast<double*>(base + off);
    off += (size_t)dd8 * 8;
    m.flags = reinterpret_cast<volatile int*>(base + off);
    return m;
}

// tiles of one pass: warp tile j (rows [r0 + j*TRW, ...)) belongs to consumer warp j % kNW
__host__ __device__ inline int warp_tile_count(int nwt, int w) {
    return nwt > w ? (nwt - w + kNW - 1) / kNW : 0;
}

// --------------------------------------------------------------------------------------
// per-warp streaming: every warp owns warp tiles j = w, w + kNW, ... of its CTA's rows and
// keeps SW of them in flight in its own ring (lane 0 issues the bulk copies), so there
// is no producer bottleneck and no cross-warp coupling.  The stream wraps from pass to
// pass, so the first SW tiles of the next pass load while the grid reduction and the
// control tail run.
struct WarpStream {
    int cnt;          // warp tiles per pass
    int issued;       // tiles of the current pass issued so far
    int deferred;     // copies for the NEXT pass held back until after the reduction
    int s;            // stage of the next tile to consume
    uint32_t phase;   // parity of that stage's full barrier
    int s_issue;      // stage the next copy goes to (tiles fill stages cyclically)
    int inflight;     // issued and not yet consumed
    int64_t tstride;  // rows between this CTA's consecutive warp tiles
    int keep;         // tiles [0, keep) of this CTA are loaded with an L2 evict_last hint
};

__device__ __forceinline__ void issue_tile(const KParams& p, const SmemMap& m, int64_t r0,
                                           int64_t r1, const WarpStream& ws, int w, int q,
                                           int stage) {
    const int slot = w * p.stages + stage;
    const int j = w + q * kNW;                    // this CTA's tile index
    const int64_t a = r0 + (int64_t)j * ws.tstride;
    const int64_t b = min(r1, a + (int64_t)p.tile_rows);
    unsigned char* dst = m.ring + (size_t)slot * p.stage_stride;
    const uint32_t xb = (uint32_t)((b - a) * p.ld * 8);
    uint32_t bytes = xb;
    int64_t ra = 0, rb = 0;
    if (p.kind == SC_SES) {
        ra = a & ~(int64_t)1;
        rb = (b + 1) & ~(int64_t)1;
        bytes += (uint32_t)((rb - ra) * 8);
    }
    SC_DCHECK(stage >= 0 && stage < p.stages && w >= 0 && w < kNW);
    SC_DCHECK(a >= r0 && a < b && b <= r1 && r1 <= p.n && b - a <= p.tile_rows);
    SC_DCHECK(xb <= p.rad_off && (p.kind != SC_SES || p.rad_off + (rb - ra) * 8 <= p.stage_stride));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive_tx(&m.full[slot], bytes);
    if (ws.keep > 0) {   // the CTA's first `keep` tiles stay in L2 across passes
        const bool keep = j < ws.keep;
        bulk_g2s_hint(dst, p.X + a * p.ld, xb, &m.full[slot], keep);
        if (p.kind == SC_SES)
            bulk_g2s_hint(dst + p.rad_off, p.radii + ra, (uint32_t)((rb - ra) * 8),
                          &m.full[slot], keep);
        return;
    }
    bulk_g2s(dst, p.X + a * p.ld, xb, &m.full[slot]);
    if (p.kind == SC_SES)
        bulk_g2s(dst + p.rad_off, p.radii + ra, (uint32_t)((rb - ra) * 8), &m.full[slot]);
}

__device__ __forceinline__ void stream_start(const KParams& p, const SmemMap& m, int64_t r0,
                                             int64_t r1, int w, WarpStream& ws, int nwt) {
    ws.cnt = warp_tile_count(nwt, w);
    ws.s = 0;
    ws.phase = 0;
    const int first = ws.cnt < p.stages ? ws.cnt : p.stages;
    if ((threadIdx.x & 31) == 0)
        for (int q = 0; q < first; ++q) issue_tile(p, m, r0, r1, ws, w,q, q);
    ws.issued = first;
    ws.deferred = 0;
    ws.inflight = first;
    ws.s_issue = first % p.stages;
}

// Copies of the next pass are held back while the grid reduction runs: ~30 MB of
// prefetches in flight make the barrier's L2 atomics and polls queue behind them
// (measured: barrier 1 grew to ~23k cycles, profiles/r01_overhead.md).  They are
// issued here, after the reduction, and overlap the control tail instead.
__device__ __forceinline__ void stream_flush(const KParams& p, const SmemMap& m, int64_t r0,
                                             int64_t r1, int w, WarpStream& ws) {
    if (p.resident || ws.deferred == 0) return;
    if (p.wrap_prefetch) {               // already issued at the end of the pass
        ws.issued = ws.deferred;
        ws.deferred = 0;
        return;
    }
    if ((threadIdx.x & 31) == 0)
        for (int q = 0; q < ws.deferred; ++q) {
            issue_tile(p, m, r0, r1, ws, w,q, ws.s_issue);
            ws.s_issue = ws.s_issue + 1 == p.stages ? 0 : ws.s_issue + 1;
        }
    else
        ws.s_issue = (ws.s_issue + ws.deferred) % p.stages;
    ws.issued = ws.deferred;
    ws.inflight += ws.deferred;
    ws.deferred = 0;
}

__device__ __forceinline__ const unsigned char* acquire_stage(const KParams& p,
                                                              const SmemMap& m, int w,
                                                              const WarpStream& ws,
                                                              int pass_idx) {
    const int slot = w * p.stages + ws.s;
    SC_DCHECK(ws.s >= 0 && ws.s < p.stages);
    if (!p.resident || pass_idx == 0) mbar_wait(&m.full[slot], ws.phase);
    return m.ring + (size_t)slot * p.stage_stride;
}

// after the warp finished reading the stage: refill it with the tile SW ahead
__device__ __forceinline__ void release_stage(const KParams& p, const SmemMap& m, int64_t r0,
                                              int64_t r1, int w, WarpStream& ws) {
    if (p.resident) {
        ws.s = ws.s + 1 == ws.cnt ? 0 : ws.s + 1;
        return;
    }
    __syncwarp();
    --ws.inflight;
    if (ws.issued < ws.cnt) {            // the next tile of this pass
        if ((threadIdx.x & 31) == 0) issue_tile(p, m, r0, r1, ws, w,ws.issued, ws.s_issue);
        ++ws.issued;
        ++ws.inflight;
        ws.s_issue = ws.s_issue + 1 == p.stages ? 0 : ws.s_issue + 1;
    } else if (p.wrap_prefetch) {        // (A/B) prefetch the next pass right away
        if ((threadIdx.x & 31) == 0) issue_tile(p, m, r0, r1, ws, w,ws.deferred, ws.s_issue);
        ++ws.deferred;
        ++ws.inflight;
        ws.s_issue = ws.s_issue + 1 == p.stages ? 0 : ws.s_issue + 1;
    } else {
        ++ws.deferred;                   // a tile of the next pass: see stream_flush
    }
    if (++ws.s == p.stages) { ws.s = 0; ws.phase ^= 1u; }
}

// before exit: wait for every copy still in flight
__device__ __forceinline__ void stream_drain(const KParams& p, const SmemMap& m, int w,
                                             WarpStream& ws) {
    if (p.resident) return;
    for (int i = 0; i < ws.inflight; ++i) {
        mbar_wait(&m.full[w * p.stages + ws.s], ws.phase);
        if (++ws.s == p.stages) { ws.s = 0; ws.phase ^= 1u; }
    }
}

// --------------------------------------------------------------------------------------
// Which row of a 4-row group a lane group reads.  A 64-bit shared load serves 16 lanes per
// wavefront: lane groups 0 and 1 (and 2, 3) share one.  With 800-byte rows (d = 100)
// adjacent rows start 8 banks apart, so groups reading rows r and r + 1 collide on 8 banks
// (round-1 ncu: 4.2 wavefronts per load instead of 2); rows r and r + 2 start 16 banks
// apart and do not.  Groups therefore take rows {0, 2, 1, 3}.
template <int RPW>
__host__ __device__ __forceinline__ int row_of_group(int grp) {
    if (RPW != 4) return grp;
    return grp == 1 ? 2 : (grp == 2 ? 1 : grp);
}

// --------------------------------------------------------------------------------------
// batched row math: NB row-groups of RPW rows are reduced by a shuffle reduce-scatter,
// after which lane (grp, l) holds the complete sums of row (l / DUP) * RPW + grp
// (DUP = LPR / NB identical copies), so the per-row scalar math (sqrt, exp, div) runs
// once per lane for NB * RPW rows instead of once per lane group.
// Select-free: the caller stores row-group k ^ (l / DUP) in slot k (an XOR permutation
// per lane), so at every level ALL lanes keep slot i and send slot i + half — the
// partner's slot i + half then holds the same row-group as my slot i — and slot 0 ends
// with row-group l / DUP.  Same pairs, same operand order as the select form: the sums
// are bit-identical, without 2 selects per value per level.
template <int LPR, int NB, int V>
__device__ __forceinline__ void reduce_scatter(double (&v)[V][NB], int l) {
    (void)l;
#pragma unroll
    for (int lev = 0, o = LPR / 2, half = NB / 2; half >= 1; ++lev, o >>= 1, half >>= 1) {
#pragma unroll
        for (int s = 0; s < V; ++s) {
#pragma unroll
            for (int i = 0; i < half; ++i)
                v[s][i] = v[s][i] + __shfl_xor_sync(0xffffffffu, v[s][i + half], o);
        }
    }
#pragma unroll
    for (int o = LPR / (2 * NB); o >= 1; o >>= 1) {
#pragma unroll
        for (int s = 0; s < V; ++s) v[s][0] += __shfl_xor_sync(0xffffffffu, v[s][0], o);
    }
}

// --------------------------------------------------------------------------------------
// consumer pass over this warp's tiles: SES.  MODE 0: iterate only (the control tail
// certified the width check of iteration k-1 by a bound); 1: + the exact
// width residuals; 2: + the window-average progress (check iterations).
template <int LPR, int CPL, int NB, bool FULL, int MODE>
__device__ void ses_pass(const KParams& p, const SmemMap& m, const PassParams& pp,
                         int64_t r0, int64_t r1, WarpStream& ws, int pass_idx) {
    constexpr bool CHECK = MODE == 2;
    constexpr bool WIDTH = MODE >= 1;
    constexpr int RPW = 32 / LPR;
    constexpr int DUP = LPR / NB;
    // per-row sums: |df|^2, then |y_prev - v|^2 (WIDTH), |y_win - v|^2 (CHECK)
    constexpr int NV = 1 + (WIDTH ? 1 : 0) + (CHECK ? 1 : 0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grp = lane / LPR, l = lane % LPR;
    const int rg = row_of_group<RPW>(grp);
    const int d = p.d, ld = p.ld, dd8 = dd8_of(p.dd);
    const double* ysum = m.vec;
    const double* yprev = m.vec + dd8;
    const double* ywin = m.vec + 5 * dd8;
    bool ok[CPL];
    double U[CPL], up[WIDTH ? CPL : 1], Sd[CPL];   // the window average (CHECK) stays in smem
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        const int j = l + LPR * c;
        // FULL: d > LPR * (CPL - 1), so only the last column slot can be short; the other
        // guards fold away at compile time (-4% on the C2 pass, profiles/r01_overhead.md)
        ok[c] = (FULL && c < CPL - 1) || j < d;
        U[c] = ok[c] ? ysum[j] : 0.0;
        if (WIDTH) up[WIDTH ? c : 0] = ok[c] ? yprev[j] : 0.0;
        Sd[c] = 0.0;
    }
    const double t = pp.t, er = pp.eta_rho, al = pp.alpha, sh = pp.shift;
    const double er_t = er * t;
    const double inv_t = 1.0 / t;
    const int myk = l / DUP;                 // row-group whose sums this lane ends up with
    const bool primary = (l % DUP) == 0;
    // K = sum_i c_i |df_i|^2 (the tail forms Lin = (U . Sd - K) / t from it)
    double T = 0, K = 0, Rad = 0, M = -INFINITY, F = -INFINITY, Wd = 0, Fw = -INFINITY;
    for (int q = 0; q < ws.cnt; ++q) {
        const int j = warp + q * kNW;
        const unsigned char* st = acquire_stage(p, m, warp, ws, pass_idx);
        const int64_t a = r0 + (int64_t)j * ws.tstride;
        const int nr = (int)(min(r1, a + (int64_t)p.tile_rows) - a);
        const double* xs = reinterpret_cast<const double*>(st);
        const double* rs = reinterpret_cast<const double*>(st + p.rad_off) + (a & 1);
        const int r = myk * RPW + rg;               // the row this lane finishes (phase B)
        const double g = r < nr ? rs[r] : 0.0;
        // phase A: per-lane partial sums of NB rows; the differences stay in registers
        // for phase C (one shared-memory read and one DFMA less per element)
        double v[NV][NB];
        double dfk[NB][CPL];
#pragma unroll
        for (int k = 0; k < NB; ++k) {
            const int r = (k ^ myk) * RPW + rg;    // slot k: row-group k ^ myk
            const double* xr = xs + (size_t)(r < nr ? r : 0) * ld + l;
            double sa = 0, sw = 0, sf = 0;
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                dfk[k][c] = 0.0;
                if (ok[c]) {
                    const double x = xr[LPR * c];
                    const double df = fma(-t, x, U[c]);
                    dfk[k][c] = df;
                    sa = fma(df, df, sa);
                    if (WIDTH) {
                        const double wv = up[WIDTH ? c : 0] - x;
                        sw = fma(wv, wv, sw);
                    }
                    if (CHECK) {
                        const double yv = ywin[l + LPR * c] - x;
                        sf = fma(yv, yv, sf);
                    }
                }
            }
            v[0][k] = sa;
            if (WIDTH) v[WIDTH ? 1 : 0][k] = sw;
            if (CHECK) v[NV - 1][k] = sf;
        }
        reduce_scatter<LPR, NB, NV>(v, l);
        // phase B: per-row scalar math, one row per lane (DUP copies)
        double cc = 0.0;
        if (r < nr) {
            const double ra = sqrt(v[0][0]);
            if (primary) {
                F = fmax(F, fma(ra, inv_t, g));
                if (CHECK) Fw = fmax(Fw, sqrt(v[NV - 1][0]) + g);
            }
            if (p.row0 + a + r > 0) {   // global row 0 is the anchor, not a block
                const double nrm = er * ra;
                const double x0 = -er_t * (al - g);
                const double lp = (x0 + nrm) * kInvSqrt2, lm = (x0 - nrm) * kInvSqrt2;
                const double A = sc_exp(lp - sh), B = sc_exp(lm - sh);
                cc = nrm > 0.0 ? (A - B) / (kSqrt2 * nrm) : 0.0;
                if (primary) {
                    T += A + B;
                    K = fma(cc, v[0][0], K);
                    Rad = fma(g, A + B, Rad);
                    M = fmax(M, lp);
                    if (WIDTH) Wd = fmax(Wd, (fabs(al - g) + sqrt(v[WIDTH ? 1 : 0][0])) * kInvSqrt2);
                }
            }
        }
        // phase C: S_d += c_i (U - t v_i) from the differences kept in registers
        // (zero in the unused column slots)
#pragma unroll
        for (int k = 0; k < NB; ++k) {
            const double ck = __shfl_sync(0xffffffffu, cc, grp * LPR + (k ^ myk) * DUP);
#pragma unroll
            for (int c = 0; c < CPL; ++c) Sd[c] = fma(ck, dfk[k][c], Sd[c]);
        }
        // (releasing the stage right after phase A instead: SES C2 134 -> 137 us/pass, C4
        // unchanged, profiles/r02_kernel_ab.md; SVM keeps the early release)
        release_stage(p, m, r0, r1, warp, ws);
    }
    // warp reduction (all 32 lanes; non-primary lanes hold identities)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        T += __shfl_xor_sync(0xffffffffu, T, o);
        K += __shfl_xor_sync(0xffffffffu, K, o);
        Rad += __shfl_xor_sync(0xffffffffu, Rad, o);
        M = fmax(M, __shfl_xor_sync(0xffffffffu, M, o));
        F = fmax(F, __shfl_xor_sync(0xffffffffu, F, o));
        Wd = fmax(Wd, __shfl_xor_sync(0xffffffffu, Wd, o));
        Fw = fmax(Fw, __shfl_xor_sync(0xffffffffu, Fw, o));
    }
    double* wp = m.wpart + (size_t)warp * ((p.pw + 1) & ~1);
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        const double s = across_sum<LPR>(Sd[c]);
        const int j = l + LPR * c;
        if (grp == 0 && j < d) wp[kS_Vec + j] = s;
    }
    if (lane == 0) {
        wp[kS_T] = T; wp[kS_Lin] = K; wp[kS_Rad] = Rad; wp[kS_M] = M;
        wp[kS_F] = F; wp[kS_Wd] = Wd; wp[kS_Fw] = Fw;
    }
}

// consumer pass: SVM (this CTA holds one side)
template <int LPR, int CPL, int NB, bool FULL, bool CHECK>
__device__ void svm_pass(const KParams& p, const SmemMap& m, const PassParams& pp,
                         int64_t r0, int64_t r1, WarpStream& ws, int pass_idx, bool isP) {
    constexpr int RPW = 32 / LPR;
    constexpr int DUP = LPR / NB;
    constexpr int NV = CHECK ? 4 : 2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grp = lane / LPR, l = lane % LPR;
    const int rg = row_of_group<RPW>(grp);
    const int d = p.d, ld = p.ld, dd8 = dd8_of(p.dd);
    const double* ysum = m.vec;
    const double* yprev = m.vec + dd8;
    const double* ywin = m.vec + 5 * dd8;
    const double* zv = m.vec + 6 * dd8;
    bool ok[CPL];
    double W[CPL], wq[CPL], G[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        const int j = l + LPR * c;
        ok[c] = (FULL && c < CPL - 1) || j < d;
        W[c] = ok[c] ? ysum[j] : 0.0;
        wq[c] = ok[c] ? yprev[j] : 0.0;
        G[c] = 0.0;
    }
    const double sg = isP ? 1.0 : -1.0;
    const double S = isP ? pp.S1 : pp.S2;
    const double sp = isP ? pp.s1p : pp.s2p;
    const double er = pp.eta_rho, sh = pp.shift;
    const int myk = l / DUP;
    const bool primary = (l % DUP) == 0;
    double T = 0, M = -INFINITY, mres = INFINITY, Wd = 0;
    double eW = isP ? INFINITY : -INFINITY, eY = eW, eZ = eW;
    for (int q = 0; q < ws.cnt; ++q) {
        const int j = warp + q * kNW;
        const unsigned char* st = acquire_stage(p, m, warp, ws, pass_idx);
        const int64_t a = r0 + (int64_t)j * ws.tstride;
        const int nr = (int)(min(r1, a + (int64_t)p.tile_rows) - a);
        const double* xs = reinterpret_cast<const double*>(st);
        double v[NV][NB];
        double xk[NB][CPL];   // the staged rows, kept in registers for the G update
#pragma unroll
        for (int k = 0; k < NB; ++k) {
            const int r = (k ^ myk) * RPW + rg;    // slot k: row-group k ^ myk
            const double* xr = xs + (size_t)(r < nr ? r : 0) * ld + l;
            double dW = 0, dw = 0, dy = 0, dz = 0;
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                xk[k][c] = 0.0;
                if (ok[c]) {
                    const double x = xr[LPR * c];
                    xk[k][c] = x;
                    dW = fma(x, W[c], dW);
                    dw = fma(x, wq[c], dw);
                    if (CHECK) {
                        const int jj = l + LPR * c;
                        dy = fma(x, ywin[jj], dy);
                        dz = fma(x, zv[jj], dz);
                    }
                }
            }
            v[0][k] = dW; v[1][k] = dw;
            if (CHECK) { v[2][k] = dy; v[3][k] = dz; }
        }
        // the tile is in registers: hand the stage back before the row math, so its refill
        // is in flight during phases B and C (C3 shape 126.0 -> 125.5 us/pass)
        release_stage(p, m, r0, r1, warp, ws);
        reduce_scatter<LPR, NB, NV>(v, l);
        const int r = myk * RPW + rg;
        double e = 0.0;
        if (r < nr) {
            const double dW = v[0][0];
            const double lg = -er * (sg * dW - S);
            e = sc_exp(lg - sh);
            if (primary) {
                T += e;
                M = fmax(M, lg);
                const double res = sg * v[1][0] - sp;
                Wd = fmax(Wd, fabs(res));
                mres = fmin(mres, res);
                if (isP) {
                    eW = fmin(eW, dW);
                    if (CHECK) { eY = fmin(eY, v[2][0]); eZ = fmin(eZ, v[3][0]); }
                } else {
                    eW = fmax(eW, dW);
                    if (CHECK) { eY = fmax(eY, v[2][0]); eZ = fmax(eZ, v[3][0]); }
                }
            }
        }
#pragma unroll
        for (int k = 0; k < NB; ++k) {
            const double ek = __shfl_sync(0xffffffffu, e, grp * LPR + (k ^ myk) * DUP);
#pragma unroll
            for (int c = 0; c < CPL; ++c) G[c] = fma(ek, xk[k][c], G[c]);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        T += __shfl_xor_sync(0xffffffffu, T, o);
        M = fmax(M, __shfl_xor_sync(0xffffffffu, M, o));
        mres = fmin(mres, __shfl_xor_sync(0xffffffffu, mres, o));
        Wd = fmax(Wd, __shfl_xor_sync(0xffffffffu, Wd, o));
        if (isP) {
            eW = fmin(eW, __shfl_xor_sync(0xffffffffu, eW, o));
            eY = fmin(eY, __shfl_xor_sync(0xffffffffu, eY, o));
            eZ = fmin(eZ, __shfl_xor_sync(0xffffffffu, eZ, o));
        } else {
            eW = fmax(eW, __shfl_xor_sync(0xffffffffu, eW, o));
            eY = fmax(eY, __shfl_xor_sync(0xffffffffu, eY, o));
            eZ = fmax(eZ, __shfl_xor_sync(0xffffffffu, eZ, o));
        }
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
// fold of all G CTA partials by one CTA: warp per FC-column chunk, lanes stride over the
// partials, then a butterfly per column (fixed order: bitwise reproducible)
enum FoldMode { kFoldTwoBarriers = 0, kFoldRedundant = 1, kFoldLast = 2 };

// Multi-GPU exchange (after this rank's columns went out to every mailbox and the
// local grid barrier): raise our flag on every rank, wait for every rank's flag, fold
// the rank vectors in rank order into `red`.  Flags are monotone pass counters across
// calls (no reset race).  A peer missing for p.xtimeout cycles sets the launch-wide abort
// word: every CTA of this launch then leaves its barrier or poll and the pass loop, and the
// call returns SC_ENCCL (the handle is marked unusable: the flag epochs of the ranks no
// longer agree).
// Out of line: it must not cost the streaming loop registers.
// The rank a CTA belongs to.  Real multi-GPU (world > 1): every CTA of this GPU is rank
// `shard`.  Emulated ranks on one GPU (vworld > 1, tests): the grid is split into vworld
// groups of G / vworld CTAs, each group a rank with its own rows, barrier counter and
// mailbox, all running the same exchange code as real ranks do.
struct RankGroup {
    int W;                       // ranks (1: single GPU)
    int rank;
    int G;                       // CTAs of this rank
    int first;                   // its first CTA index
    unsigned long long* bar;     // its grid-barrier counter
};

__device__ __forceinline__ RankGroup rank_group(const KParams& p, int b) {
    RankGroup g;
    if (p.vworld > 1) {
        g.W = p.vworld;
        g.G = p.G / p.vworld;
        g.rank = b / g.G;
        g.first = g.rank * g.G;
        g.bar = p.bar + 8 * (g.rank + 1);
    } else {
        g.W = p.world > 1 ? p.world : 1;
        g.rank = p.world > 1 ? p.shard : 0;
        g.G = p.G;
        g.first = 0;
        g.bar = p.bar;
    }
    return g;
}

template <int KIND>
static __device__ __noinline__ void rank_exchange(const KParams& p, const RankGroup g,
                                                  double* red, volatile int* flags,
                                                  int pass_idx) {
    const int tid = threadIdx.x;
    const unsigned long long want = (unsigned long long)(p.pass_base + pass_idx + 1);
    // thread r raises this rank's flag in rank r's mailbox and then waits for rank r's
    // flag in ours, so the W release stores and the W acquire polls run in parallel
    // (one thread doing them in sequence cost one system-scope round trip per rank).
    // Ordering: the mailbox stores of every folding warp precede the grid barrier this
    // CTA passed (thread 0's acquire + bar.sync), so thread r's release covers them.
    // (fault injection for the failure-path test: rank p.drop_rank never raises its flags)
    if (tid < g.W && (int)blockIdx.x == g.first && g.rank != p.drop_rank)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p.mflag[tid] + g.rank),
                     "l"(want)
                     : "memory");
    if (tid < g.W) {
        const long long t0 = clock64();
        unsigned long long v;
        volatile unsigned long long* abort = p.bar + kAbortWord;
        do {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];"
                         : "=l"(v) : "l"(p.mflag[g.rank] + tid) : "memory");
            if (v >= want) break;
            if (*abort != 0) { flags[1] = 1; break; }
            if (clock64() - t0 > p.xtimeout) {
                flags[1] = 1;
                *abort = 1;
                __threadfence();
                break;
            }
        } while (true);
    }
    consumer_sync();
    if (flags[1]) return;
    const double* mb = p.mbox[g.rank] + (size_t)((p.pass_base + pass_idx) & 1) * g.W * p.rw;
    for (int j = tid; j < p.rw; j += kNW * 32) {
        const int op = red_op(KIND, j);
        double acc = op_identity(op);
        for (int r = 0; r < g.W; ++r) acc = op_apply(op, acc, __ldcg(mb + (size_t)r * p.rw + j));
        red[j] = acc;
    }
}

// Every CTA folds all G partials itself (one grid barrier per pass instead of two): warp w
// sums the contiguous partial range [w*G/8, (w+1)*G/8) lane-per-column (its loads issue
// ahead of the adds), then the 8 range sums are combined in warp order.  Columns go in
// chunks of the warp-partial scratch (pws doubles per warp).  The order is fixed and the
// same in every CTA, so all CTAs hold identical reduced vectors.
template <int KIND>
static __device__ __noinline__ void fold_redundant(const KParams& p, double* wpart,
                                                   double* red, const double* part, int pws) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q0 = warp * p.G / kNW, q1 = (warp + 1) * p.G / kNW;
    for (int c0 = 0; c0 < p.rw; c0 += pws) {
        const int c1 = min(p.rw, c0 + pws);
        for (int j = c0 + lane; j < c1; j += 32) {
            const int op = red_op(KIND, j);
            double acc = op_identity(op);
#pragma unroll 8
            for (int q = q0; q < q1; ++q)
                acc = op_apply(op, acc, __ldcg(part + (size_t)q * p.rw + j));
            wpart[warp * pws + (j - c0)] = acc;
        }
        consumer_sync();
        for (int j = c0 + (int)threadIdx.x; j < c1; j += kNW * 32) {
            const int op = red_op(KIND, j);
            double acc = op_identity(op);
            for (int w = 0; w < kNW; ++w) acc = op_apply(op, acc, wpart[w * pws + (j - c0)]);
            red[j] = acc;
        }
        consumer_sync();
    }
}

template <int KIND>
static __device__ __noinline__ void fold_all(const KParams& p, const double* part, double* red,
                                            bool publish) {
    constexpr int FC = 8;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int j0 = warp * FC; j0 < p.rw; j0 += kNW * FC) {
        double acc[FC];
        int op[FC];
#pragma unroll
        for (int k = 0; k < FC; ++k) {
            op[k] = red_op(KIND, min(j0 + k, p.rw - 1));
            acc[k] = op_identity(op[k]);
        }
        for (int q = lane; q < p.G; q += 32) {
            const double* row = part + (size_t)q * p.rw;
#pragma unroll
            for (int k = 0; k < FC; ++k)
                if (j0 + k < p.rw) acc[k] = op_apply(op[k], acc[k], __ldcg(row + j0 + k));
        }
#pragma unroll
        for (int k = 0; k < FC; ++k) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
                acc[k] = op_apply(op[k], acc[k], __shfl_xor_sync(0xffffffffu, acc[k], o));
            if (lane == 0 && j0 + k < p.rw) {
                red[j0 + k] = acc[k];
                if (publish) p.redg[j0 + k] = acc[k];
            }
        }
    }
}

// --------------------------------------------------------------------------------------
// control tails (warp 0 of every CTA, between passes).  Out of line: the control state is
// loaded from and stored back to shared memory here, so none of it is live in the
// streaming loop's register allocation.  They take plain pointers, not the SmemMap: a
// reference would force the map into local memory, and the streaming loop's shared
// loads would lose their address space (generic LD/ST instead of LDS/STS).
template <int KIND>
static __device__ __noinline__ int ctl_tail(const KParams& p, void* ctl_mem, const double* red,
                                            double* y_tilde, PassParams* pp) {
    Control<WarpLanes>* const sm = reinterpret_cast<Control<WarpLanes>*>(ctl_mem);
    Control<WarpLanes> ctl = *sm;
    const int act = ctl.after_pass(red, p.red0, y_tilde, pp);
    __syncwarp();
    if ((threadIdx.x & 31) == 0) *sm = ctl;
    __syncwarp();
    return act;
}
template <int KIND>
static __device__ __noinline__ int solve_tail(const KParams& p, void* ctl_mem, void* srch_mem,
                                              const double* red, double* y_tilde,
                                              PassParams* pp) {
    Control<WarpLanes>* const csm = reinterpret_cast<Control<WarpLanes>*>(ctl_mem);
    Search<WarpLanes>* const ssm = reinterpret_cast<Search<WarpLanes>*>(srch_mem);
    Control<WarpLanes> ctl = *csm;
    const int phase = ssm->phase;
    if (phase == kBracket || phase == kRefine) {
        // inside a feasibility test (almost every pass): only the test's control state is
        // needed; the search state is loaded when the test ends
        int act = ctl.after_pass(red, p.red0, y_tilde, pp);
        if (act == kPass) {
            __syncwarp();
            if ((threadIdx.x & 31) == 0) *csm = ctl;
            __syncwarp();
            return act;
        }
        Search<WarpLanes> srch = *ssm;
        act = srch.test_done(ctl, p.red0, y_tilde, pp);
        __syncwarp();
        if ((threadIdx.x & 31) == 0) {
            *csm = ctl;
            *ssm = srch;
        }
        __syncwarp();
        return act;
    }
    Search<WarpLanes> srch = *ssm;
    const int act = srch.after_pass(ctl, red, p.red0, y_tilde, pp);
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
        *csm = ctl;
        *ssm = srch;
    }
    __syncwarp();
    return act;
}

// --------------------------------------------------------------------------------------
// the persistent kernel
template <int KIND, int LPR, int CPL, int NB, bool FULL>
__global__ void __launch_bounds__(kThreads, 1) scmwu_kernel(const __grid_constant__ KParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
#ifdef SCMWU_PHASE_TIMING
    __shared__ long long tt_sh[8];
#endif
    const SmemMap m = carve(smem, p);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x;
    // work slot: the CTA index, or (one CTA per SM, rows balanced by the measured
    // per-SM streaming rates) the SM id, so a slot's rows and its place in the fixed-order
    // fold do not depend on how this launch mapped CTAs to SMs
    int slot = b;
    if (p.by_smid) {
        unsigned s;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
        slot = (int)s;
    }
    // this slot's warp tiles: tile j covers rows [r0 + j * tstride, + tile_rows) below r1
    SC_DCHECK(slot >= 0 && slot < p.G);
    const int64_t r0 = p.row_begin[4 * slot], r1 = p.row_begin[4 * slot + 1];
    const int64_t tstride = p.row_begin[4 * slot + 2];
    SC_DCHECK(r0 >= 0 && r1 <= p.n && (r1 <= r0 || tstride >= p.tile_rows));
    const int nwt = r1 > r0 ? (int)((r1 - r0 + tstride - 1) / tstride) : 0;
    const bool isP = KIND == SC_SVM && p.row_begin[4 * slot + 3] != 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kNW * p.stages; ++s) mbar_init(&m.full[s], 1);
        m.flags[0] = 0;
        m.flags[1] = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    WarpStream ws;
    ws.tstride = tstride;
    ws.keep = (int)((double)nwt * p.l2_frac);
    stream_start(p, m, r0, r1, warp, ws, nwt);

    // ------------------------------------------------------------ consumers
    const int dd8 = dd8_of(p.dd);
    const int tid = threadIdx.x;
    // The control state lives in shared memory between tails: warp 0 loads it into
    // registers for the tail and stores it back, so it is dead (no registers) during the
    // streaming passes.  Every lane holds identical scalars; lane 0 stores them.
    using Ctl = Control<WarpLanes>;
    using Srch = Search<WarpLanes>;
    Ctl* const ctl_sm = reinterpret_cast<Ctl*>(m.ctl);
    PassParams* pp = m.pp;
    double* y_tilde = b == 0 && !p.solve ? p.y_tilde : m.ytd;
    if (warp == 0) {
        Ctl ctl;
        ctl.kind = KIND; ctl.d = p.d; ctl.dd = p.dd; ctl.is_max = KIND == SC_SES;
        ctl.rho = p.rho; ctl.inv_rho = p.inv_rho; ctl.R = p.R; ctl.ln_r = p.ln_r;
        ctl.D = p.D; ctl.g1 = p.g1;
        ctl.res = b == 0 && !p.solve ? p.res : m.resd;
        ctl.writer = b == 0;
        double* V = m.vec;
        ctl.v = CtlVecs{V, V + dd8, V + 2 * dd8, V + 3 * dd8, V + 4 * dd8, V + 5 * dd8,
                        V + 6 * dd8, V + 7 * dd8, V + 8 * dd8, V + 9 * dd8};
        const int sl = p.slot_len;
        ctl.evict_buf = m.evict;
        ctl.pend_buf = m.pend;
#ifdef SCMWU_PHASE_TIMING
        // tail-section sums in shared memory (a global read-modify-write per mark cost
        // ~1k cycles each and inflated the measured tail)
        if (p.timing != nullptr && b == 0 && lane == 0) {
            for (int i = 0; i < 8; ++i) tt_sh[i] = 0;
            ctl.tt = tt_sh;
        }
#endif
        ctl.s = CtlSlots{p.ring, p.ring_cap, dd8, p.slots, p.slots + sl, p.slots + 2 * sl,
                         p.slots + 4 * sl, p.slots + 3 * sl};
        for (int j = lane; j < dd8; j += 32) {
            for (int q = 0; q < 10; ++q) V[q * dd8 + j] = 0.0;
            if (KIND == SC_SES && j < p.d) V[9 * dd8 + j] = p.v1[j];   // anchor v1
        }
        __syncwarp();
        int act;
        if (p.solve) {
            Srch srch;
            srch.R = p.R; srch.rho = p.rho; srch.ln_r = p.ln_r;
            srch.kind = KIND; srch.d = p.d; srch.dd = p.dd;
            srch.sbest = m.sbest; srch.yprog = ctl.v.ywin; srch.log = p.steps;
            srch.writer = b == 0;
            act = srch.begin(ctl, p.sargs, p.seed, pp);
            if (lane == 0) *reinterpret_cast<Srch*>(m.srch) = srch;
        } else {
            act = ctl.begin(p.args, p.red0, y_tilde, nullptr, pp);
        }
        if (lane == 0) {
            pp->action = act;
            *ctl_sm = ctl;
        }
    }
    consumer_sync();

    int pass_idx = 0;
    unsigned long long nbar = 0;
    // multi-GPU (real or emulated ranks): barriers also watch the launch-wide abort word
    const unsigned long long* abort_w =
        kMultiGpu && (p.world > 1 || p.vworld > 1) ? p.bar + kAbortWord : nullptr;
    // columns of the reduced vector folded by this CTA
    const RankGroup grp = rank_group(p, b);
    const int lb = b - grp.first;                 // index of this CTA within its rank
    const int c0 = (int)((int64_t)lb * p.rw / grp.G), c1 = (int)((int64_t)(lb + 1) * p.rw / grp.G);
    const int pws = (p.pw + 1) & ~1;
    // per-phase timing only in -DSCMWU_PHASE_TIMING builds: the nine live counters
    // would otherwise cost registers in the streaming loop of every build
#ifdef SCMWU_PHASE_TIMING
    const bool timed = p.timing != nullptr && b == 0 && tid == 0;
#else
    constexpr bool timed = false;
#endif
    long long tacc[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    long long tprev = timed ? clock64() : 0;
#define SCMWU_TMARK(i)                               \
    if (timed) {                                     \
        const long long tnow = clock64();            \
        tacc[i] += tnow - tprev;                     \
        tprev = tnow;                                \
    }
#ifdef SCMWU_PHASE_TIMING
    long long tcta = 0, tcta0 = 0;
    unsigned long long g_start = 0, g_end = 0, g_arr = 0, g_rel = 0;
#endif
    int64_t width_passes = 0;
    // partition calibration (p.slot_cycles set): this slot's streaming cycles over all
    // passes (thread 0; pass start to the CTA join)
    long long scyc = 0, scyc0 = 0;
    while (pp->action == kPass) {
        const PassParams ps = *pp;
        if (p.slot_cycles != nullptr && tid == 0) scyc0 = clock64();
#ifdef SCMWU_PHASE_TIMING
        if (tid == 0) {
            tcta0 = clock64();
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_start));
        }
#endif
        if (KIND == SC_SES) {
            width_passes += (ps.check || ps.width) ? 1 : 0;
            if (ps.check) ses_pass<LPR, CPL, NB, FULL, 2>(p, m, ps, r0, r1, ws, pass_idx);
            else if (ps.width) ses_pass<LPR, CPL, NB, FULL, 1>(p, m, ps, r0, r1, ws, pass_idx);
            else ses_pass<LPR, CPL, NB, FULL, 0>(p, m, ps, r0, r1, ws, pass_idx);
        } else {
            if (ps.check) svm_pass<LPR, CPL, NB, FULL, true>(p, m, ps, r0, r1, ws, pass_idx, isP);
            else svm_pass<LPR, CPL, NB, FULL, false>(p, m, ps, r0, r1, ws, pass_idx, isP);
        }
        SCMWU_TMARK(0)
        consumer_sync();
        if (p.slot_cycles != nullptr && tid == 0) scyc += clock64() - scyc0;
#ifdef SCMWU_PHASE_TIMING
        // per-CTA streaming time (all CTAs): the skew the first grid barrier absorbs
        if (tid == 0 && p.timing != nullptr) {
            const long long tnow = clock64();
            tcta += tnow - tcta0;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_end));
        }
#endif
        SCMWU_TMARK(1)
        // CTA partial, fixed warp order, written in the reduced layout (partials are
        // double-buffered by pass parity for the single-barrier redundant fold)
        double* const part = p.partials + (size_t)(pass_idx & 1) * p.G * p.rw;
        const int nw_act = nwt < kNW ? nwt : kNW;   // warps that own at least one tile
        SC_DCHECK(KIND != SC_SES || p.rw <= pws);
        for (int j = tid; j < p.rw; j += kNW * 32) {
            double v;
            if (KIND == SC_SES) {
                const int op = red_op(KIND, j);
                v = op_identity(op);
                for (int w = 0; w < nw_act; ++w) v = op_apply(op, v, m.wpart[w * pws + j]);
            } else {
                int pc, side;
                svm_src(p.d, j, pc, side);
                const int op = red_op(KIND, j);
                v = op_identity(op);
                const bool mine = side == 0 || (side == 1) == isP;
                if (mine && nw_act > 0) {
                    const int pop = svm_part_op(pc, isP);
                    double acc = op_identity(pop);
                    for (int w = 0; w < nw_act; ++w)
                        acc = op_apply(pop, acc, m.wpart[w * pws + pc]);
                    v = acc;
                }
            }
            part[(size_t)slot * p.rw + j] = v;
        }
        SCMWU_TMARK(2)
        if (kFoldVariants && p.fold_mode == kFoldLast && grp.W <= 1) {
            // one global synchronisation: the CTA whose arrival completes the pass
            // folds all partials (fixed tree) and publishes them with a release epoch
            consumer_sync();
            if (tid == 0) {
                unsigned long long old;
                asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;"
                             : "=l"(old) : "l"(p.bar) : "memory");
                m.flags[0] = old + 1 == (unsigned long long)(pass_idx + 1) * p.G ? 1 : 0;
            }
            consumer_sync();
            SCMWU_TMARK(3)
            if (m.flags[0]) {
                fold_all<KIND>(p, part, m.red, true);
                SCMWU_TMARK(4)
                consumer_sync();
                if (tid == 0)
                    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p.bar + 1),
                                 "l"((unsigned long long)(pass_idx + 1))
                                 : "memory");
                SCMWU_TMARK(5)
            } else {
                SCMWU_TMARK(4)
                if (tid == 0)
                    while (ld_acquire(p.bar + 1) < (unsigned long long)(pass_idx + 1)) {
                    }
                consumer_sync();
                SCMWU_TMARK(5)
                for (int j = tid; j < p.rw; j += kNW * 32) m.red[j] = __ldcg(p.redg + j);
            }
            consumer_sync();
            SCMWU_TMARK(6)
        } else if (p.fold_mode == kFoldRedundant && grp.W <= 1) {
            // every CTA folds all G partials itself with the same fixed tree
            // one barrier: the partials are double-buffered by pass parity, and a CTA can
            // run at most one pass ahead of the slowest reader
            grid_barrier(grp.bar, (++nbar) * (unsigned long long)grp.G);
            SCMWU_TMARK(3)
            fold_redundant<KIND>(p, m.wpart, m.red, part, pws);
            SCMWU_TMARK(4)
            SCMWU_TMARK(6)
        } else {
#ifdef SCMWU_PHASE_TIMING
            consumer_sync();
            if (tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_arr));
#endif
            grid_barrier(grp.bar, (++nbar) * (unsigned long long)grp.G, abort_w, m.flags);
#ifdef SCMWU_PHASE_TIMING
            if (tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_rel));
#endif
            if (m.flags[1]) {   // another CTA gave up on a peer: leave without folding
                if (b == 0 && tid == 0) *p.status = SC_ENCCL;
                break;
            }
            SCMWU_TMARK(3)
            // column-distributed fold over this rank's G partials: warp per column, fixed
            // tree
            const double* gpart = part + (size_t)grp.first * p.rw;
            SC_DCHECK(grp.G <= 160 && grp.first + grp.G <= p.G && c1 <= p.rw);
            for (int j = c0 + warp; j < c1; j += kNW) {
                const int op = red_op(KIND, j);
                double acc = op_identity(op);
                // all loads first (G <= 160: at most 5 per lane), then the fixed-order fold
                double ld[5];
#pragma unroll
                for (int i = 0; i < 5; ++i) {
                    const int q = lane + 32 * i;
                    ld[i] = q < grp.G ? __ldcg(gpart + (size_t)q * p.rw + j) : 0.0;
                }
#pragma unroll
                for (int i = 0; i < 5; ++i)
                    if (lane + 32 * i < grp.G) acc = op_apply(op, acc, ld[i]);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1)
                    acc = op_apply(op, acc, __shfl_xor_sync(0xffffffffu, acc, o));
                if (lane == 0) {
                    if (kMultiGpu && grp.W > 1) {
                        // this rank's folded column -> slot [parity][rank] of EVERY rank's
                        // mailbox (NVLink stores to the peers' HBM)
                        const size_t off =
                            ((size_t)((p.pass_base + pass_idx) & 1) * grp.W + grp.rank) * p.rw + j;
                        SC_DCHECK(grp.W <= kMaxWorld && grp.rank < grp.W);
                        for (int r = 0; r < grp.W; ++r) p.mbox[r][off] = acc;
                    } else {
                        p.redg[j] = acc;
                    }
                }
            }
            // one system-scope fence per warp after all its mailbox stores (a fence per
            // column cost ~7 us per pass with 8 emulated ranks at d = 512,
            // tools/exchange_bench.py)
            if (kMultiGpu && grp.W > 1 && lane == 0 && c0 + warp < c1) __threadfence_system();
            SCMWU_TMARK(4)
            grid_barrier(grp.bar, (++nbar) * (unsigned long long)grp.G, abort_w, m.flags);
            SCMWU_TMARK(5)
            if (kMultiGpu && grp.W > 1) {
                if (!m.flags[1]) rank_exchange<KIND>(p, grp, m.red, m.flags, pass_idx);
            } else {
                for (int j = tid; j < p.rw; j += kNW * 32) m.red[j] = __ldcg(p.redg + j);
            }
            consumer_sync();
            SCMWU_TMARK(6)
        }
        // the reduction is done: release the next pass's copies (they overlap the tail);
        // warp 0 runs the tail, so it issues its own copies after it (issuing right
        // before the tail slowed the tail's first section 3k -> 7k cycles)
        if (warp != 0 && !p.flush_after_tail) stream_flush(p, m, r0, r1, warp, ws);
        if (m.flags[1]) {   // a peer never arrived: give up with an exchange error
            if (b == 0 && tid == 0) *p.status = SC_ENCCL;
            break;
        }
        if (warp == 0) {
            const int act = p.solve ? solve_tail<KIND>(p, m.ctl, m.srch, m.red, y_tilde, pp)
                                    : ctl_tail<KIND>(p, m.ctl, m.red, y_tilde, pp);
            if (lane == 0) pp->action = act;
            stream_flush(p, m, r0, r1, warp, ws);
        }
        SCMWU_TMARK(7)
        consumer_sync();
        if (warp != 0 && p.flush_after_tail) stream_flush(p, m, r0, r1, warp, ws);
        SCMWU_TMARK(8)
        ++pass_idx;
    }
#undef SCMWU_TMARK
    if (timed)
        for (int i = 0; i < 9; ++i) p.timing[i] = tacc[i];
#ifdef SCMWU_PHASE_TIMING
    if (tid == 0 && p.timing != nullptr) {
        p.timing[16 + b] = tcta;
        int smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        p.timing[16 + 160 + b] = smid;
        p.timing[16 + 320 + b] = (long long)g_start;   // last pass, global ns clock
        p.timing[16 + 480 + b] = (long long)g_end;
        p.timing[16 + 640 + b] = (long long)g_arr;     // last pass: first grid barrier
        p.timing[16 + 800 + b] = (long long)g_rel;
    }
    if (p.timing != nullptr && b == 0 && tid == 0)
        for (int i = 0; i < 8; ++i) p.timing[16 + 960 + i] = tt_sh[i];
#endif
    if (p.slot_cycles != nullptr && tid == 0) {
        unsigned s;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
        p.slot_cycles[2 * slot] = scyc;
        p.slot_cycles[2 * slot + 1] = (long long)s;
    }
    // wait for the prefetched copies of the (never run) next pass, then publish (CTA 0)
    stream_drain(p, m, warp, ws);
    if (b == 0 && warp == 0 && p.solve) {
        __syncwarp();
        const Srch* sr = reinterpret_cast<const Srch*>(m.srch);
        for (int j = lane; j < p.dd; j += 32) p.best_y[j] = m.sbest[j];
        if (lane == 0) {
            sc_solve_result& o = *p.sres;
            o.lower = sr->Lb; o.upper = sr->Ub; o.best_value = sr->best_f;
            o.has_best = sr->has_best; o.termination = sr->termination();
            o.total_iterations = sr->total; o.search_steps = sr->nsteps;
            o.has_pd = sr->has_pd; o.pd_dist = sr->pd_best;
            o.seed_f = sr->seed_f; o.final_f = sr->final_f;
            o.width_alpha = sr->w_alpha; o.width_iteration = sr->w_iter;
            o.width_norm = sr->w_norm;
            o.passes = pass_idx;
            o.width_passes = width_passes;
            if (!m.flags[1]) *p.status = sr->status;
        }
    } else if (b == 0 && warp == 0) {
        __syncwarp();
        for (int j = lane; j < p.dd; j += 32) p.best_y[j] = ctl_sm->v.besty[j];
        if (lane == 0) {
            if (!m.flags[1]) *p.status = ctl_sm->status;
            p.res->passes = pass_idx;
            p.res->width_passes = width_passes;
        }
    }
    __syncthreads();
}

typedef void (*KernelFn)(const KParams);

}  // namespace scmwu

// explicit instantiation + lookup, used by the scmwu_inst_*.cu translation units
#define SCMWU_INST(K, L, C, B, F)                                                       \
    template __global__ void scmwu::scmwu_kernel<K, L, C, B, F>(                         \
        const __grid_constant__ scmwu::KParams);
#define SCMWU_MATCH(K, L, C, B, F)                                        \
    if (kind == K && lpr == L && cpl == C && nb == B && full == F) \
        return scmwu::scmwu_kernel<K, L, C, B, F>;
