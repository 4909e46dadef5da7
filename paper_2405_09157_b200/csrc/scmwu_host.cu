// scmwu_host.cu — host side of the B200 engine: the C ABI of include/scmwu.h,
// launch configuration and the one-off kernels (progress, iterate, column sums).
#include <stdlib.h>

#include <cmath>
#include <map>
#include <mutex>

#include "scmwu_handle.h"

namespace scmwu {
// --------------------------------------------------------------------------------------
// one-off kernels
__global__ void progress_kernel(const double* X, const double* radii, int64_t n, int64_t n1,
                                int d, int ld, int kind, const double* y, double* out) {
    // out[block*3 + {0,1,2}]: SES {max dist+r}, SVM {min P.y, max Q.y}
    const int lane = threadIdx.x & 31;
    const int warps = blockDim.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5);
    const int64_t nw = (int64_t)gridDim.x * warps;
    double a0 = kind == SC_SES ? -INFINITY : INFINITY, a1 = -INFINITY;
    for (int64_t i = gw; i < n; i += nw) {
        const double* xr = X + i * ld;
        double s = 0.0;
        for (int j = lane; j < d; j += 32) {
            if (kind == SC_SES) { double t = xr[j] - y[j]; s = fma(t, t, s); }
            else s = fma(xr[j], y[j], s);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (kind == SC_SES) a0 = fmax(a0, sqrt(s) + radii[i]);
        else if (i < n1) a0 = fmin(a0, s);
        else a1 = fmax(a1, s);
    }
    __shared__ double sh[2][32];
    if (lane == 0) { sh[0][threadIdx.x >> 5] = a0; sh[1][threadIdx.x >> 5] = a1; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < warps; ++w) {
            a0 = kind == SC_SES ? fmax(a0, sh[0][w]) : fmin(a0, sh[0][w]);
            a1 = fmax(a1, sh[1][w]);
        }
        out[blockIdx.x * 2] = a0;
        out[blockIdx.x * 2 + 1] = a1;
    }
}

// iterate materialisation: p for SES blocks / SVM coordinates, from an IterState slot.
__global__ void iterate_kernel(const double* X, const double* radii, int64_t n, int64_t n1,
                               int d, int ld, int kind, const double* slot, int dd, double rho,
                               double alpha, double* out, int64_t first) {
    const IterState st = *reinterpret_cast<const IterState*>(slot + dd + (dd & 1));
    const double er = st.eta / rho;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (kind == SC_SES) {
        if (i < first || i >= n) return;   // local rows; global row 0 is the anchor
        const double* v = X + i * ld;
        const double g = radii[i];
        double a = 0.0;
        for (int j = 0; j < d; ++j) { double x = fma(-st.t, v[j], slot[j]); a = fma(x, x, a); }
        const double ra = sqrt(a);
        const double nrm = er * ra;
        const double x0 = -(er * st.t) * (alpha - g);
        const double A = sc_exp((x0 + nrm) * kInvSqrt2 - st.shift);
        const double B = sc_exp((x0 - nrm) * kInvSqrt2 - st.shift);
        const double cc = nrm > 0.0 ? (A - B) / (kSqrt2 * nrm) : 0.0;
        double* o = out + (i - first) * (d + 1);
        for (int j = 0; j < d; ++j) {
            const double x = fma(-st.t, v[j], slot[j]);
            o[j] = (cc * (-er * x)) / st.T;
        }
        o[d] = ((A + B) / kSqrt2) / st.T;
    } else {
        if (i >= n) return;
        const double* x = X + i * ld;
        double s = 0.0;
        for (int j = 0; j < d; ++j) s = fma(x[j], slot[j], s);
        const bool P = i < n1;
        const double lg = -er * ((P ? 1.0 : -1.0) * s - (P ? slot[d] : slot[d + 1]));
        out[i] = sc_exp(lg - st.shift) / st.T;
    }
}

// column sums of P and Q rows (SVM iterate 1: all weights equal).  Fixed order, independent
// of the grid: rows [a, b) are cut into `chunks` equal ranges; block (column tile, chunk)
// sums its range with warp w taking rows w, w + 8, ... (lane = column, coalesced row reads)
// and folds the 8 warp sums in warp order; colsum_fold_kernel then adds the chunk partials
// in chunk order.  (One thread per column walking all rows took ~90 ms at C3.)
__global__ void colsum_chunk_kernel(const double* X, int64_t a, int64_t b, int d, int ld,
                                    int chunks, double* part) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int j = blockIdx.x * 32 + lane;
    const int64_t rows = b - a;
    const int64_t r0 = a + rows * blockIdx.y / chunks, r1 = a + rows * (blockIdx.y + 1) / chunks;
    double s = 0.0;
    if (j < d)
        for (int64_t i = r0 + w; i < r1; i += 8) s += X[i * ld + j];
    __shared__ double sh[8][32];
    sh[w][lane] = s;
    __syncthreads();
    if (w == 0 && j < d) {
        double t = 0.0;
        for (int k = 0; k < 8; ++k) t += sh[k][lane];
        part[(size_t)blockIdx.y * d + j] = t;
    }
}

__global__ void colsum_fold_kernel(const double* part, int chunks, int d, double* out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= d) return;
    double s = 0.0;
    for (int c = 0; c < chunks; ++c) s += part[(size_t)c * d + j];
    out[j] = s;
}

}  // namespace scmwu

// ======================================================================================
// host side
using namespace scmwu;

static bool pick_cfg(int d, LaunchCfg& c) {
    // {max d, lanes per row, columns per lane, row-groups per batch}
    static const int tab[][4] = {{4, 2, 2, 2},     {8, 2, 4, 2},     {12, 4, 3, 4},
                                 {16, 4, 4, 4},    {24, 4, 6, 4},    {32, 4, 8, 4},
                                 {48, 8, 6, 4},    {64, 8, 8, 4},    {80, 8, 10, 4},
                                 {104, 8, 13, 4},  {128, 8, 16, 2},  {192, 16, 12, 2},
                                 {256, 16, 16, 2}, {384, 32, 12, 2}, {512, 32, 16, 2}};
    for (auto& r : tab)
        if (d <= r[0]) { c.lpr = r[1]; c.cpl = r[2]; c.nb = r[3]; return true; }
    return false;
}

// out[0, d) = column sums of rows [a, b) of X (device), on the handle's stream
static cudaError_t column_sums(sc_handle* h, int64_t a, int64_t b, double* out) {
    const int d = h->prob.d;
    const int chunks = (int)std::max<int64_t>(1, std::min<int64_t>(1024, (b - a) / 256));
    double* part = nullptr;
    cudaError_t e = pool_alloc((void**)&part, (size_t)chunks * d * 8, h->prob.device, h->stream);
    if (e != cudaSuccess) return e;
    colsum_chunk_kernel<<<dim3((d + 31) / 32, chunks), 256, 0, h->stream>>>(h->X, a, b, d, h->ld,
                                                                          chunks, part);
    colsum_fold_kernel<<<(d + 127) / 128, 128, 0, h->stream>>>(part, chunks, d, out);
    e = cudaStreamSynchronize(h->stream);
    pool_free(part, h->stream);
    return e;
}

// kernels are instantiated in scmwu_inst_*.cu (compiled in parallel)
namespace scmwu {
KernelFn scmwu_lookup_0(int kind, int lpr, int cpl, int nb, bool full);
KernelFn scmwu_lookup_1(int kind, int lpr, int cpl, int nb, bool full);
KernelFn scmwu_lookup_2(int kind, int lpr, int cpl, int nb, bool full);
KernelFn scmwu_lookup_3(int kind, int lpr, int cpl, int nb, bool full);
KernelFn scmwu_lookup_4(int kind, int lpr, int cpl, int nb, bool full);
KernelFn scmwu_lookup_5(int kind, int lpr, int cpl, int nb, bool full);
KernelFn scmwu_lookup_6(int kind, int lpr, int cpl, int nb, bool full);
KernelFn scmwu_lookup_7(int kind, int lpr, int cpl, int nb, bool full);
KernelFn scmwu_lookup_8(int kind, int lpr, int cpl, int nb, bool full);
}  // namespace scmwu

// full: every column slot but the last is in range (d > lpr * (cpl - 1)), so only the last
// slot needs a runtime guard.  Instantiated for every SES config and for the SVM configs of
// the BASELINE dimensions; a full request falls back to the guarded kernel (correct for
// any d).
static KernelFn kernel_lookup(int kind, int lpr, int cpl, int nb, bool full) {
    KernelFn (*fns[])(int, int, int, int, bool) = {scmwu_lookup_0, scmwu_lookup_1,
                                                   scmwu_lookup_2, scmwu_lookup_3,
                                                   scmwu_lookup_4, scmwu_lookup_5,
                                                   scmwu_lookup_6, scmwu_lookup_7,
                                                   scmwu_lookup_8};
    for (auto f : fns)
        if (KernelFn k = f(kind, lpr, cpl, nb, full)) return k;
    if (full) return kernel_lookup(kind, lpr, cpl, nb, false);
    return nullptr;
}

// Row partition balanced per SM (one CTA per SM).  B200 SMs do not stream at the same
// rate: per-SM pass times of the persistent kernel spread by ~15 % and repeat run to run
// to < 1 % (tools/die_probe.cu, profiles/r01_overhead.md), so with an equal partition the
// first grid barrier absorbs the slowest SM's excess every pass.  The kernel itself is the
// calibration: the first sc_ftp of a large single-GPU handle runs a short refine probe
// with the equal cyclic partition, reads every SM's streaming cycles for its tiles and
// derives per-SM throughput weights (quantised to 1/1024 of the fastest).  They are cached
// per (device, kernel) for the process, so every later handle of that kernel partitions
// identically (bitwise-reproducible results within a process).  SCMWU_BALANCE=0 disables.
// (A pure streaming probe, tools/die_probe.cu, overshoots: it measures bandwidth shares, while
// the SES pass is partly compute bound: SES C2 136 -> 149 us/pass.)
static std::mutex g_calib_mu;
static std::map<std::pair<int, const void*>, std::vector<double>> g_calib;

// The per-handle device buffers (X, radii, window ring, partials, control slots, ...) come
// from the device's stream-ordered pool, which keeps up to SCMWU_POOL_GB (default 4) of freed memory mapped:
// a solve through the public API creates and destroys a handle per call, and plain
// cudaFree / cudaMalloc of ~1 GB cost 0.01-0.3 s each on B200 (C2: close 0.16-0.29 s,
// ring growth up to 0.37 s, tools/solve_gaps.py).  Allocation and free are synchronised
// on the handle's stream, so the memory is usable from any stream afterwards.  IPC-shared
// mailboxes stay on cudaMalloc (pool memory cannot be exported with cudaIpcGetMemHandle).
// Buffers larger than the retained size use plain cudaMalloc: the pool would release them
// anyway, and growing it by 82 GB (C5 shape) took the e2e step (generate + 64 passes +
// destroy) from 0.11 s to 0.40 s.
static std::mutex g_pool_mu;
struct DevPool {
    cudaMemPool_t pool = nullptr;   // private to the engine (not the device's default pool)
    uint64_t thr = 0;               // retained bytes
    int handles = 0;                // live handles on the device
};
static std::map<int, DevPool> g_pools;
static std::map<void*, bool> g_pool_ptrs;    // live pointers that came from the pool

static DevPool& dev_pool(int device) {   // g_pool_mu held
    auto it = g_pools.find(device);
    if (it != g_pools.end()) return it->second;
    DevPool& dp = g_pools[device];
    double gb = 12.0;   // >= the C4 matrix (10^7 x 100 fp64 = 8 GB) plus its ring
    if (const char* e = getenv("SCMWU_POOL_GB")) gb = std::max(0.0, atof(e));
    dp.thr = (uint64_t)(gb * 1073741824.0);
    cudaMemPoolProps props;
    memset(&props, 0, sizeof(props));
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    if (dp.thr == 0 || cudaMemPoolCreate(&dp.pool, &props) != cudaSuccess ||
        cudaMemPoolSetAttribute(dp.pool, cudaMemPoolAttrReleaseThreshold, &dp.thr) !=
            cudaSuccess) {
        dp.pool = nullptr;
        dp.thr = 0;
    }
    cudaGetLastError();
    return dp;
}

cudaError_t pool_alloc(void** p, size_t bytes, int device, cudaStream_t s) {
    cudaMemPool_t pool;
    {
        std::lock_guard<std::mutex> lock(g_pool_mu);
        DevPool& dp = dev_pool(device);
        pool = bytes <= dp.thr ? dp.pool : nullptr;
    }
    if (pool == nullptr) return cudaMalloc(p, std::max<size_t>(bytes, 8));
    cudaError_t e = cudaMallocFromPoolAsync(p, std::max<size_t>(bytes, 8), pool, s);
    if (e != cudaSuccess) return e;
    {
        std::lock_guard<std::mutex> lock(g_pool_mu);
        g_pool_ptrs[*p] = true;
    }
    return cudaStreamSynchronize(s);
}

void pool_free(void* p, cudaStream_t s) {
    if (p == nullptr) return;
    bool pooled;
    {
        std::lock_guard<std::mutex> lock(g_pool_mu);
        pooled = g_pool_ptrs.erase(p) > 0;
    }
    if (!pooled) {
        cudaFree(p);
        return;
    }
    cudaFreeAsync(p, s);
    cudaStreamSynchronize(s);
}

// live handles per device.  The pool keeps freed memory mapped after the last handle
// closes (a public-API solve creates and destroys a handle per call); sc_pool_trim returns
// it to the driver.  The pool is private to the engine, so no other cudaMallocAsync user of
// the process (torch, NCCL) inherits the retention threshold.
static void pool_handle_open(int device) {
    std::lock_guard<std::mutex> lock(g_pool_mu);
    dev_pool(device).handles += 1;
}
static void pool_handle_close(int device) {
    std::lock_guard<std::mutex> lock(g_pool_mu);
    DevPool& dp = dev_pool(device);
    if (dp.handles > 0) dp.handles -= 1;
}

// Off by default: the equal cyclic partition by CTA index makes the fixed-order fold, and
// with it every result, bitwise reproducible across processes and boxes (the calibrated
// weights are re-measured per process).  Measured on B200 (profiles/r02_kernel_ab.md): at
// configs[3] (SES n = 10^7, d = 100) the calibrated partition does not help (per-CTA pass
// times spread 1.82M-2.00M cycles with it, 1.91M-1.99M without; 1252-1311 vs 1250-1290
// us/pass); at n = 10^6 it saved 2-3 % (round 1).  SCMWU_BALANCE=1 opts in.
static bool balance_enabled() {
    const char* e = getenv("SCMWU_BALANCE");
    return e != nullptr && atoi(e) != 0;
}

static const std::vector<double>* sm_weights(sc_handle* h) {
    std::lock_guard<std::mutex> lock(g_calib_mu);
    auto it = g_calib.find({h->prob.device, (const void*)h->fn});
    return it == g_calib.end() ? nullptr : &it->second;
}

// tiles [0, T) of one side split over `slots` contiguous blocks in proportion to the
// weights (largest remainder, ties to the lower slot)
static std::vector<int64_t> weighted_split(int64_t T, const std::vector<double>& w) {
    const int k = (int)w.size();
    double W = 0.0;
    for (double x : w) W += x;
    std::vector<int64_t> cnt(k);
    std::vector<std::pair<double, int>> rem(k);
    int64_t used = 0;
    for (int i = 0; i < k; ++i) {
        const double ideal = (double)T * w[i] / W;
        cnt[i] = (int64_t)std::floor(ideal);
        used += cnt[i];
        rem[i] = {-(ideal - (double)cnt[i]), i};
    }
    std::sort(rem.begin(), rem.end());
    for (int64_t r = 0; r < T - used; ++r) ++cnt[rem[(size_t)(r % k)].second];
    return cnt;
}

static int configure(sc_handle* h, int grid_req) {
    const int d = h->prob.d;
    const int RPW = 32 / h->cfg.lpr;
    const int64_t n = h->prob.n_local;
    // grid: one CTA per SM, at most one CTA per warp-step of rows
    int G = grid_req > 0 ? grid_req : h->sms;
    const int64_t step = (int64_t)kNW * RPW;
    if (grid_req <= 0) G = (int)std::min<int64_t>(G, std::max<int64_t>(1, (n + step - 1) / step));
    const int64_t n1 = h->prob.kind == SC_SVM ? h->prob.n1_local : 0, n2 = n - n1;
    (void)d;
    const bool two_sided = h->prob.kind == SC_SVM && n1 > 0 && n2 > 0;
    // emulated ranks (tests, SCMWU_VWORLD): W groups of G / W CTAs, one per rank
    const int W = h->vworld > 1 ? h->vworld : 1;
    if (two_sided) G = std::max(G, 2);
    G = std::min(G, h->sms);
    G = std::min(G, 160);   // the column fold loads at most 5 partials per lane
    if (W > 1) G = std::max(2 * W, G / W * W);
    if (G < 1) G = 1;
    if (two_sided && G < 2) { h->err = "SVM needs >= 2 SMs"; return SC_EARG; }
    // warp tiles: NB row-groups of RPW rows; one SW-stage ring per consumer warp
    const int64_t rowb = (int64_t)h->ld * 8;
    const int tr = h->cfg.nb * RPW;
    h->tile_rows = tr;
    const uint32_t xb = (uint32_t)((int64_t)tr * rowb);
    h->rad_off = (xb + 15) & ~15u;
    const uint32_t radb = h->prob.kind == SC_SES ? (uint32_t)((tr + 2) * 8) : 0u;
    h->stage_stride = (h->rad_off + radb + 127) & ~127u;
    // Partition: per slot {first row, end row, row stride between its warp tiles, SVM P}.
    // Within a side (SVM: P rows then Q rows, every CTA single-sided) the tiles are dealt
    // cyclically: slot c of a side with g slots takes tiles c, c+g, ... (every CTA streams
    // from the whole address range).  Large single-GPU handles switch to contiguous blocks
    // per SM id sized by the calibrated per-SM rates (see sm_weights).
    std::vector<int64_t> cta(4 * (size_t)G, 0);
    h->by_smid = false;
    h->grid_req = grid_req;
    const bool big = n / tr >= (int64_t)64 * G;   // >= 64 tiles per SM: worth balancing
    h->balance_ok = G == h->sms && big && h->prob.world <= 1 && W == 1 && balance_enabled();
    const std::vector<double>* wp = h->balance_ok ? sm_weights(h) : nullptr;
    if (wp != nullptr && (int)wp->size() == G) h->by_smid = true;
    auto deal = [&](int s0, int s1, int64_t rs, int64_t re, bool P) {
        if (s1 <= s0) return;
        if (h->by_smid) {
            const int64_t T = (re - rs + tr - 1) / tr;
            // whole groups of kNW tiles per SM, so its 8 warps get equal tile counts; the
            // < kNW leftover tiles go to the slots one each, from the first
            std::vector<int64_t> cnt = weighted_split(
                T / kNW, std::vector<double>(wp->begin() + s0, wp->begin() + s1));
            for (auto& c : cnt) c *= kNW;
            for (int64_t r = 0; r < T % kNW; ++r) ++cnt[(size_t)(r % cnt.size())];
            int64_t t0 = 0;
            for (int i = 0; i < s1 - s0; ++i) {
                const int sl = s0 + i;
                cta[4 * sl] = rs + t0 * tr;
                cta[4 * sl + 1] = std::min(re, rs + (t0 + cnt[i]) * tr);
                cta[4 * sl + 2] = tr;
                cta[4 * sl + 3] = P ? 1 : 0;
                t0 += cnt[i];
            }
            return;
        }
        const int g = s1 - s0;
        for (int i = 0; i < g; ++i) {
            const int sl = s0 + i;
            cta[4 * sl] = rs + (int64_t)i * tr;
            cta[4 * sl + 1] = re;
            cta[4 * sl + 2] = (int64_t)g * tr;
            cta[4 * sl + 3] = P ? 1 : 0;
        }
    };
    const int Gv = G / W;
    h->gP = 0;
    for (int r = 0; r < W; ++r) {
        // rank r's rows: the np.array_split rule of the real sharding (shard.row_ranges)
        const int64_t q = n / W, m = n % W;
        const int64_t R0 = r * q + std::min<int64_t>(r, m), R1 = R0 + q + (r < m ? 1 : 0);
        const int s0 = r * Gv, s1 = s0 + Gv;
        if (h->prob.kind == SC_SES) { deal(s0, s1, R0, R1, false); continue; }
        const int64_t p0 = R0, p1 = std::min(R1, std::max(R0, n1));   // P rows of the rank
        if (p1 > p0 && R1 > p1) {
            int gp = (int)llround((double)Gv * (double)(p1 - p0) / (double)(R1 - R0));
            gp = std::max(1, std::min(Gv - 1, gp));
            deal(s0, s0 + gp, p0, p1, true);
            deal(s0 + gp, s1, p1, R1, false);
            if (r == 0) h->gP = gp;
        } else {
            deal(s0, s1, R0, R1, p1 > p0);
            if (r == 0 && p1 > p0) h->gP = Gv;
        }
    }
    int nwt = 0;
    int64_t covered = 0;   // rows over all slots' tiles: must be n exactly (no gap, no overlap)
    for (int sl = 0; sl < G; ++sl) {
        const int64_t c0 = cta[4 * sl], c1 = cta[4 * sl + 1], st = cta[4 * sl + 2];
        const int t = c1 > c0 && st > 0 ? (int)((c1 - c0 + st - 1) / st) : 0;
        nwt = std::max(nwt, t);
        if (t > 0) {
            if (c0 < 0 || c1 > n || st < tr) { h->err = "partition: bad slot range"; return SC_EARG; }
            covered += (int64_t)(t - 1) * tr + std::min<int64_t>(tr, c1 - (c0 + (int64_t)(t - 1) * st));
        }
    }
    if (covered != n) { h->err = "partition does not cover the rows exactly once"; return SC_EARG; }
    const int per_warp = (nwt + kNW - 1) / kNW;
    auto need = [&](int sw) {
        return (size_t)kNW * sw * h->stage_stride + smem_fixed_bytes(h->dd, h->rw, h->pw, kNW * sw);
    };
    int S = 1;
    while (S < 64 && need(S + 1) <= (size_t)kMaxSmem) ++S;
    h->resident = per_warp <= S ? 1 : 0;
    if (h->resident) S = std::max(per_warp, 1);
    else if (S < 2) { h->err = "shared memory too small for a double-buffered ring"; return SC_EARG; }
    h->stages = S;
    h->smem = need(S);
    if (h->smem > (size_t)kMaxSmem) { h->err = "shared memory budget exceeded"; return SC_EARG; }
    h->grid = G;
    h->cta_h = cta;
    pool_free(h->row_begin, h->stream);
    pool_free(h->partials, h->stream);
    CK(pool_alloc((void**)&h->row_begin, cta.size() * sizeof(int64_t), h->prob.device, h->stream), "alloc rows");
    CK(h_put(h, h->row_begin, cta.data(), cta.size() * sizeof(int64_t)),
       "copy rows");
    CK(pool_alloc((void**)&h->partials, 2 * (size_t)G * h->rw * sizeof(double), h->prob.device, h->stream), "alloc partials");
    CK(cudaFuncSetAttribute(h->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)h->smem),
       "smem attribute");
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, h->fn, kThreads, h->smem),
       "occupancy");
    if (per_sm < 1) { h->err = "kernel does not fit on an SM"; return SC_ECUDA; }
    return SC_OK;
}

// Host rows (pitch d) -> device rows (pitch ld).  Pinned (page-locked / registered)
// input is copied directly; pageable input goes through two pinned 32 MB staging
// buffers so the host memcpy of one chunk overlaps the DMA of the other.
static int upload_rows(sc_handle* h, double* dst, const double* src, int64_t rows, int d) {
    if (rows <= 0) return SC_OK;
    const size_t rowb = (size_t)d * 8, dpitch = (size_t)h->ld * 8;
    cudaPointerAttributes at;
    // equal pitches (even d): one linear copy.  A 2-D copy of 800-byte rows runs at ~7 GB/s
    // against ~55 GB/s linear (C2: 117 ms vs 15 ms for 808 MB).
    auto copy = [&](double* dd, const double* ss, int64_t m) {
        return rowb == dpitch
                   ? cudaMemcpyAsync(dd, ss, (size_t)m * rowb, cudaMemcpyHostToDevice, h->stream)
                   : cudaMemcpy2DAsync(dd, dpitch, ss, rowb, rowb, m, cudaMemcpyHostToDevice,
                                       h->stream);
    };
    if (cudaPointerGetAttributes(&at, src) == cudaSuccess && at.type == cudaMemoryTypeHost) {
        CK(copy(dst, src, rows), "copy X (pinned)");
        CK(cudaStreamSynchronize(h->stream), "copy X");
        return SC_OK;
    }
    cudaGetLastError();   // clear the lookup error on pageable memory
    const int64_t chunk = std::max<int64_t>(1, (int64_t)(32u << 20) / (int64_t)rowb);
    void* stage[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    int status = SC_OK;
    for (int i = 0; i < 2 && status == SC_OK; ++i) {
        if (cudaMallocHost(&stage[i], (size_t)chunk * rowb) != cudaSuccess ||
            cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming) != cudaSuccess)
            status = SC_EOOM;
    }
    for (int64_t a = 0, k = 0; status == SC_OK && a < rows; a += chunk, ++k) {
        const int64_t m = std::min(chunk, rows - a);
        const int i = (int)(k & 1);
        if (k >= 2 && cudaEventSynchronize(done[i]) != cudaSuccess) { status = SC_ECUDA; break; }
        memcpy(stage[i], src + a * d, (size_t)m * rowb);
        if (copy(dst + a * h->ld, static_cast<const double*>(stage[i]), m) != cudaSuccess ||
            cudaEventRecord(done[i], h->stream) != cudaSuccess)
            status = SC_ECUDA;
    }
    if (cudaStreamSynchronize(h->stream) != cudaSuccess && status == SC_OK) status = SC_ECUDA;
    for (int i = 0; i < 2; ++i) {
        if (stage[i]) cudaFreeHost(stage[i]);
        if (done[i]) cudaEventDestroy(done[i]);
    }
    if (status != SC_OK) h->err = "staged upload of X failed";
    return status;
}

extern "C" {

int sc_version(void) { return 1000; }

int sc_pool_trim(int32_t device) {
    std::lock_guard<std::mutex> lock(g_pool_mu);
    auto it = g_pools.find(device);
    if (it == g_pools.end() || it->second.pool == nullptr) return SC_OK;
    return cudaMemPoolTrimTo(it->second.pool, 0) == cudaSuccess ? SC_OK : SC_ECUDA;
}

// sc_create (host rows X / X_tail / radii) and sc_create_generated (gen != NULL: rows drawn
// on the device, zero radii; *D_out receives this shard's range D)
static int create_impl(const sc_problem* prob, const double* X, const double* X_tail,
                       const double* radii, const sc_gen* gen, double* D_out,
                       sc_handle** out) {
    if (!out) return SC_EARG;
    *out = nullptr;
    if (!prob || (!X && !gen) || prob->d < 1 || prob->n < 2) return SC_EARG;
    if (prob->kind != SC_SES && prob->kind != SC_SVM) return SC_EARG;
    if (prob->kind == SC_SES && !radii && !gen) return SC_EARG;
    if (prob->kind == SC_SVM && (prob->n1 < 1 || prob->n1 >= prob->n || radii)) return SC_EARG;
    sc_handle* h = new sc_handle();
    *out = h;
    h->prob = *prob;
    // row sharding: normalise the single-GPU case, validate the shard
    sc_problem& P = h->prob;
    if (P.world <= 1) {
        P.world = 1; P.shard = 0; P.row0 = 0; P.n_local = P.n;
        P.n1_local = P.kind == SC_SVM ? P.n1 : 0;
    } else {
        if (P.world > kMaxWorld || P.shard < 0 || P.shard >= P.world || P.n_local < 1 ||
            P.row0 < 0 || P.row0 + P.n_local > P.n || X_tail) {
            h->err = "bad row shard";
            return SC_EARG;
        }
        P.n1_local = P.kind == SC_SVM
                         ? std::max<int64_t>(0, std::min<int64_t>(P.n_local, P.n1 - P.row0))
                         : 0;
    }
    const int d = prob->d;
    const int64_t n = P.n_local;   // rows resident on this GPU
    if (!pick_cfg(d, h->cfg)) { h->err = "d > 512 is not supported yet"; return SC_EARG; }
    if (const char* cfg = getenv("SCMWU_CFG")) {   // A/B: "lanes,cols,groups"
        LaunchCfg c{};
        if (sscanf(cfg, "%d,%d,%d", &c.lpr, &c.cpl, &c.nb) == 3 && c.lpr * c.cpl >= d)
            h->cfg = c;
    }
    const bool full = d > h->cfg.lpr * (h->cfg.cpl - 1);
    h->fn = kernel_lookup(prob->kind, h->cfg.lpr, h->cfg.cpl, h->cfg.nb, full);
    if (!h->fn) { h->err = "no kernel instantiated for this d"; return SC_EARG; }
    h->dd = prob->kind == SC_SES ? d + 1 : d + 2;
    h->ld = (d + 1) & ~1;
    h->rw = red_width(prob->kind, d);
    h->pw = part_width(prob->kind, d);
    h->slot_len = h->dd + (h->dd & 1) + (int)(sizeof(IterState) / sizeof(double));
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev), "device count");
    if (prob->device < 0 || prob->device >= ndev) { h->err = "no such CUDA device"; return SC_ECUDA; }
    CK(cudaSetDevice(prob->device), "set device");
    cudaDeviceProp dp;
    CK(cudaGetDeviceProperties(&dp, prob->device), "device properties");
    if (dp.major < 10) { h->err = "needs an sm_100 (B200) device"; return SC_ECUDA; }
    if (!dp.cooperativeLaunch) { h->err = "cooperative launch unsupported"; return SC_ECUDA; }
    h->sms = dp.multiProcessorCount;
    CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking), "stream");
    pool_handle_open(prob->device);
    h->pool_open = true;
    CK(cudaEventCreate(&h->ev0), "event");
    CK(cudaEventCreate(&h->ev1), "event");
    CK(cudaEventCreate(&h->mk0), "event");
    CK(cudaEventCreate(&h->mk1), "event");
    // X: n x ld, rows padded to an even length (16-byte rows for the bulk copies)
    const size_t xbytes = (size_t)n * h->ld * sizeof(double);
    CK(pool_alloc((void**)&h->X, xbytes, prob->device, h->stream), "alloc X");
    CK(pool_alloc((void**)&h->scratch, 2 * 4096 * 8, h->prob.device, h->stream), "alloc scratch");
    const int64_t n_head = X_tail ? prob->n1 : n;
    CK(pool_alloc((void**)&h->v1, (size_t)d * 8, h->prob.device, h->stream), "alloc anchor");
    CK(h_zero(h, h->v1, (size_t)d * 8), "zero anchor");
    if (gen) {
        const int st = generate_rows(h, gen, D_out);   // scmwu_gen.cu
        if (st != SC_OK) return st;
    } else {
        if (h->ld != d) CK(h_zero(h, h->X, xbytes), "zero X");   // ordered before the upload
        int up = upload_rows(h, h->X, X, n_head, d);
        if (up == SC_OK && X_tail) up = upload_rows(h, h->X + n_head * h->ld, X_tail, n - n_head, d);
        if (up != SC_OK) return up;
        // SES anchor row (global row 0; sharded: sc_set_globals provides it)
        if (P.row0 == 0) CK(h_put(h, h->v1, X, (size_t)d * 8), "anchor");
    }
    if (prob->kind == SC_SES) {
        const int64_t nr = (n + 1) & ~(int64_t)1;
        CK(pool_alloc((void**)&h->radii, (size_t)(nr + 2) * 8, prob->device, h->stream), "alloc radii");
        CK(h_zero(h, h->radii, (size_t)(nr + 2) * 8), "zero radii");
        if (radii) {
            CK(h_put(h, h->radii, radii, (size_t)n * 8), "copy radii");
            h->g1 = P.row0 == 0 ? radii[0] : 0.0;   // sharded: sc_set_globals provides it
        }
    }
    // reduced vector of iterate 1 (cum = 0: every exponent 0) over the LOCAL rows;
    // sharded handles get the rank-ordered fold through sc_set_globals
    h->red0_h.assign(h->rw, 0.0);
    if (prob->kind == SC_SES) {
        double rad = 0.0;
        const int64_t first = P.row0 == 0 ? 1 : 0;   // global row 0 is not a block
        if (radii)
            for (int64_t i = first; i < n; ++i) rad += 2.0 * radii[i];
        h->red0_h[kS_T] = 2.0 * (double)(n - first);
        h->red0_h[kS_Rad] = rad;
    } else {
        const int64_t n1l = P.n1_local;
        h->red0_h[kV_TP] = (double)n1l;
        h->red0_h[kV_TQ] = (double)(n - n1l);
        double* cs = h->scratch;   // 2 x 4096 doubles >= 2 d
        CK(column_sums(h, 0, n1l, cs), "colsum P");
        CK(column_sums(h, n1l, n, cs + d), "colsum Q");
        h->launches += 4;
        CK(h_get(h, h->red0_h.data() + kV_Vec, cs, 2 * (size_t)d * 8),
           "copy colsum");
    }
    // Emulated ranks on one GPU (tests only, SCMWU_VWORLD = 2..8 with world <= 1): the
    // iterate-1 vector is the rank-ordered fold of the ranks' local vectors, exactly as a
    // sharded solve builds it (shard.fold_ranks), and every rank gets a mailbox in this
    // GPU's memory; the kernel then runs the real exchange code between CTA groups.
    if (const char* e = getenv("SCMWU_VWORLD")) {
        const int W = atoi(e);
        if (W > 1 && W <= kMaxWorld && P.world <= 1 && n >= 2 * W) {
            h->vworld = W;
            std::vector<double> acc(h->rw);
            for (int j = 0; j < h->rw; ++j) {
                const int op = red_op(prob->kind, j);
                acc[j] = op_identity(op);
            }
            double* cs = h->scratch;
            for (int r = 0; r < W; ++r) {
                const int64_t q = n / W, m = n % W;
                const int64_t R0 = r * q + std::min<int64_t>(r, m), R1 = R0 + q + (r < m ? 1 : 0);
                std::vector<double> loc(h->rw, 0.0);
                if (prob->kind == SC_SES) {
                    double rad = 0.0;
                    const int64_t first = R0 == 0 ? 1 : 0;
                    if (radii)
                        for (int64_t i = R0 + first; i < R1; ++i) rad += 2.0 * radii[i];
                    loc[kS_T] = 2.0 * (double)(R1 - R0 - first);
                    loc[kS_Rad] = rad;
                } else {
                    const int64_t p1 = std::min(R1, std::max(R0, P.n1_local));
                    loc[kV_TP] = (double)(p1 - R0);
                    loc[kV_TQ] = (double)(R1 - p1);
                    CK(column_sums(h, R0, p1, cs), "colsum P");
                    CK(column_sums(h, p1, R1, cs + d), "colsum Q");
                    CK(h_get(h, loc.data() + kV_Vec, cs, 2 * (size_t)d * 8), "copy colsum");
                }
                for (int j = 0; j < h->rw; ++j) acc[j] = op_apply(red_op(prob->kind, j), acc[j], loc[j]);
            }
            h->red0_h = acc;
            // mailboxes of all emulated ranks: [flags 64 | data 2 x W x rw] each
            const size_t mb = 64 * 8 + 2 * (size_t)W * h->rw * 8;
            CK(cudaMalloc(&h->mbox_base, mb * W), "alloc mailboxes");
            CK(h_zero(h, h->mbox_base, mb * W), "zero mailboxes");
            CK(cudaStreamSynchronize(h->stream), "zero mailboxes");
            for (int r = 0; r < W; ++r) h->peer_base[r] = static_cast<char*>(h->mbox_base) + mb * r;
        }
    }
    CK(pool_alloc((void**)&h->red0, h->rw * 8, h->prob.device, h->stream), "alloc red0");
    CK(h_put(h, h->red0, h->red0_h.data(), h->rw * 8), "copy red0");
    CK(pool_alloc((void**)&h->redg, h->rw * 8, h->prob.device, h->stream), "alloc redg");
    CK(pool_alloc((void**)&h->bar, 1024, h->prob.device, h->stream), "alloc barrier");   // + one counter per emulated rank
    CK(pool_alloc((void**)&h->slots, (size_t)kNumSlots * h->slot_len * 8, h->prob.device, h->stream), "alloc slots");
    CK(h_zero(h, h->slots, (size_t)kNumSlots * h->slot_len * 8), "zero slots");
    CK(pool_alloc((void**)&h->res, sizeof(sc_ftp_result), h->prob.device, h->stream), "alloc result");
    CK(pool_alloc((void**)&h->y_tilde, h->dd * 8, h->prob.device, h->stream), "alloc y");
    CK(pool_alloc((void**)&h->best_y, h->dd * 8, h->prob.device, h->stream), "alloc y");
    CK(pool_alloc((void**)&h->yvec, (size_t)(d + 2) * 8, h->prob.device, h->stream), "alloc y");
    CK(pool_alloc((void**)&h->status, sizeof(int), h->prob.device, h->stream), "alloc status");
    int st = configure(h, prob->grid);
    if (st != SC_OK) return st;
    h->err.clear();
    return SC_OK;
}

int sc_create(const sc_problem* prob, const double* X, const double* X_tail, const double* radii,
              sc_handle** out) {
    return create_impl(prob, X, X_tail, radii, nullptr, nullptr, out);
}

// width / trace bound / rank as the solvers derive them (R/ses.py:161,169, R/svm.py:168,186)
static void derive_constants(sc_problem* p) {
    if (p->kind == SC_SES) {
        p->rho = 3.0 * p->D / sqrt(2.0);
        p->R = sqrt(2.0);
        p->rank = 2 * (p->n - 1);
    } else {
        p->rho = 2.0 * p->D;
        p->R = 2.0;
        p->rank = p->n;
    }
    p->ln_r = log((double)p->rank);
}

int sc_create_generated(sc_problem* prob, const sc_gen* gen, double* v1_out, sc_handle** out) {
    if (!out) return SC_EARG;
    *out = nullptr;
    if (!prob || !gen) return SC_EARG;
    const bool ses_dist = gen->dist >= SC_GEN_GAUSSIAN && gen->dist <= SC_GEN_SPHERE_SURFACE;
    if (prob->kind == SC_SES && !ses_dist) return SC_EARG;
    if (prob->kind == SC_SVM &&
        (gen->dist != SC_GEN_SVM_CLUSTERS || !gen->direction || !(gen->gap > 0.0)))
        return SC_EARG;
    prob->D = 1.0;   // placeholder until the device range is known
    derive_constants(prob);
    double D = 0.0;
    const int st = create_impl(prob, nullptr, nullptr, nullptr, gen, &D, out);
    if (st != SC_OK) return st;
    sc_handle* h = *out;
    prob->D = D;
    derive_constants(prob);
    h->prob.D = prob->D;
    h->prob.rho = prob->rho;
    h->prob.R = prob->R;
    h->prob.rank = prob->rank;
    h->prob.ln_r = prob->ln_r;
    if (v1_out && prob->kind == SC_SES)
        CK(h_get(h, v1_out, h->v1, (size_t)prob->d * 8), "copy anchor");
    return SC_OK;
}

int sc_set_range(sc_handle* h, double D) {
    if (!h || !(D >= 0.0)) return SC_EARG;
    h->prob.D = D;
    derive_constants(&h->prob);
    return SC_OK;
}

int sc_read_rows(sc_handle* h, int64_t first, int64_t count, double* out) {
    if (!h || !out || first < 0 || count < 0 || first + count > h->prob.n_local) return SC_EARG;
    if (count == 0) return SC_OK;
    CK(cudaMemcpy2D(out, (size_t)h->prob.d * 8, h->X + first * h->ld, (size_t)h->ld * 8,
                    (size_t)h->prob.d * 8, (size_t)count, cudaMemcpyDeviceToHost),
       "read rows");
    return SC_OK;
}

int sc_set_grid(sc_handle* h, int32_t grid) {
    if (!h) return SC_EARG;
    CK(cudaSetDevice(h->prob.device), "set device");
    return configure(h, grid);
}

// window history for runs of up to T iterations: max(64, T/2) + 2 entries, capped at
// SCMWU_RING_GB (default 2 GiB: 2.6M entries at d = 100, 0.5M at d = 512); a run whose
// window outgrows the ring stops with SC_EOOM instead of overwriting live entries
static int ensure_ring(sc_handle* h, int64_t T) {
    int64_t need = std::max<int64_t>(kLadderBase, T / 2) + 2;
    const int dd8 = (h->dd + 1) & ~1;                             // 16-byte ring entries
    double ring_gb = 2.0;
    if (const char* e = getenv("SCMWU_RING_GB")) ring_gb = std::max(1e-6, atof(e));
    const int64_t cap_lim = std::max<int64_t>(kLadderBase + 2, (int64_t)(ring_gb * 1073741824.0) / (dd8 * 8));
    if (need > cap_lim) need = cap_lim;
    if (need > h->ring_cap) {
        pool_free(h->ring, h->stream);
        h->ring = nullptr;
        CK(pool_alloc((void**)&h->ring, (size_t)need * dd8 * 8, h->prob.device, h->stream),
           "alloc window ring");
        h->ring_cap = need;
    }
    return SC_OK;
}

// kernel parameters common to sc_ftp and sc_solve
static int fill_params(sc_handle* h, KParams& p, long long* slot_cycles) {
    memset(&p, 0, sizeof(p));
    p.kind = h->prob.kind; p.d = h->prob.d; p.ld = h->ld; p.dd = h->dd; p.rw = h->rw; p.pw = h->pw;
    p.G = h->grid; p.gP = h->gP; p.tile_rows = h->tile_rows; p.stages = h->stages;
    p.resident = h->resident; p.n = h->prob.n; p.n1 = h->prob.n1;
    // grid reduction scheme (SCMWU_FOLD=0 two barriers, 1 redundant, 2 last arriver)
    // measured on B200 (profiles/r01_overhead.md): two barriers 8.3 us/pass at C1,
    // last-arriver 16.9 us (147 CTAs poll one line while one CTA folds), redundant worse
    p.fold_mode = kFoldTwoBarriers;
    if (const char* f = getenv("SCMWU_FOLD")) p.fold_mode = atoi(f);
    // next-pass prefetch placement (A/B, profiles/r01_overhead.md): during the reduction
    // (default, best by ~1%), after the reduction (SCMWU_DEFER_PREFETCH) or after the tail
    // (SCMWU_DEFER_PREFETCH + SCMWU_FLUSH_AFTER_TAIL)
    p.wrap_prefetch = getenv("SCMWU_DEFER_PREFETCH") ? 0 : 1;
    p.flush_after_tail = getenv("SCMWU_FLUSH_AFTER_TAIL") ? 1 : 0;
    p.by_smid = h->by_smid ? 1 : 0;
    p.slot_cycles = slot_cycles;
    // L2 residency of part of X across passes: every CTA loads its first tiles with an
    // evict_last hint, the rest evict_first, so ~40 MB of X are served from L2 every pass
    // (same box, us/pass, keep 0 / 40 / 80 / 110 MB: SES C2 136.1 / 131.7 / 133.0 / 135.1,
    // SVM C3 128.0 / 124.7 / 125.3 / 125.7).  SCMWU_L2_KEEP_MB overrides (0 = no hints).
    double keep_mb = 40.0;
    if (const char* e = getenv("SCMWU_L2_KEEP_MB")) keep_mb = atof(e);
    const double xbytes = (double)h->prob.n_local * h->ld * 8.0;
    p.l2_frac = xbytes > 0.0 ? std::min(1.0, std::max(0.0, keep_mb * 1e6 / xbytes)) : 0.0;
    p.X = h->X; p.radii = h->radii; p.row_begin = h->row_begin;
    p.rho = h->prob.rho; p.inv_rho = 1.0 / h->prob.rho; p.R = h->prob.R; p.ln_r = h->prob.ln_r;
    p.D = h->prob.D; p.g1 = h->g1;
    p.red0 = h->red0; p.partials = h->partials; p.redg = h->redg; p.bar = h->bar;
    p.ring = h->ring; p.ring_cap = h->ring_cap; p.slots = h->slots; p.slot_len = h->slot_len;
    p.res = h->res; p.y_tilde = h->y_tilde; p.best_y = h->best_y;
    p.status = h->status; p.stage_stride = h->stage_stride; p.rad_off = h->rad_off;
    if (!h->timing && getenv("SCMWU_TIMING")) {
        CK(cudaMalloc(&h->timing, (16 + 6 * 160 + 16) * 8), "alloc timing");
    }
    if (h->timing) CK(cudaMemsetAsync(h->timing, 0, (16 + 6 * 160 + 16) * 8, h->stream), "timing");
    p.timing = h->timing;
    p.v1 = h->v1;
    p.world = h->prob.world;
    p.shard = h->prob.shard;
    p.row0 = h->prob.row0;
    p.pass_base = h->pass_total;
    p.vworld = h->vworld;
    {   // peer timeout of the in-kernel exchange: SCMWU_EXCHANGE_TIMEOUT_S (default 30 s)
        double secs = 30.0;
        if (const char* e = getenv("SCMWU_EXCHANGE_TIMEOUT_S")) secs = std::max(1e-3, atof(e));
        int khz = 0;
        cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, h->prob.device);
        p.xtimeout = (long long)(secs * 1e3 * (double)(khz > 0 ? khz : 2000000));
    }
    p.drop_rank = -1;
    if (const char* e = getenv("SCMWU_FAULT_DROP_RANK")) p.drop_rank = atoi(e);
    if (h->vworld > 1) {
        for (int r = 0; r < h->vworld; ++r) {
            p.mflag[r] = reinterpret_cast<unsigned long long*>(h->peer_base[r]);
            p.mbox[r] = reinterpret_cast<double*>(static_cast<char*>(h->peer_base[r]) + 64 * 8);
        }
    }
    if (p.world > 1) {
        if (!h->connected) { h->err = "sharded handle is not connected (sc_connect)"; return SC_EARG; }
        for (int r = 0; r < p.world; ++r) {
            p.mflag[r] = reinterpret_cast<unsigned long long*>(h->peer_base[r]);
            p.mbox[r] = reinterpret_cast<double*>(static_cast<char*>(h->peer_base[r]) + 64 * 8);
        }
    }
    return SC_OK;
}

// one cooperative launch of the persistent kernel; returns the kernel's status word
static int launch(sc_handle* h, KParams& p, int* status, float* ms) {
    CK(cudaMemsetAsync(h->bar, 0, 1024, h->stream), "reset barrier");
    CK(cudaMemsetAsync(h->res, 0, sizeof(sc_ftp_result), h->stream), "reset result");
    CK(cudaMemsetAsync(h->status, 0xff, sizeof(int), h->stream), "reset status");
    void* kargs[] = {&p};
    CK(cudaEventRecord(h->ev0, h->stream), "event");
    CK(cudaLaunchCooperativeKernel((const void*)h->fn, dim3(h->grid), dim3(kThreads), kargs,
                                   h->smem, h->stream),
       "persistent kernel launch");
    h->launches += 1;
    CK(cudaEventRecord(h->ev1, h->stream), "event");
    CK(cudaStreamSynchronize(h->stream), "persistent kernel");
    *status = -1;
    CK(h_get(h, status, h->status, sizeof(int)), "copy status");
    *ms = 0.f;
    cudaEventElapsedTime(ms, h->ev0, h->ev1);
    return SC_OK;
}

static int kernel_status(sc_handle* h, int status) {
    if (status == SC_EWIDTH) { h->err = "width violation"; return SC_EWIDTH; }
    if (status == SC_EOOM) {
        h->err = "the suffix window outgrew the window ring (raise SCMWU_RING_GB)";
        return SC_EOOM;
    }
    if (status == SC_ENCCL) {
        h->broken = true;
        h->err = "a peer rank did not arrive at the in-kernel exchange (timeout)";
        return SC_ENCCL;
    }
    if (status != SC_OK) { h->err = "kernel did not complete"; return SC_ECUDA; }
    return SC_OK;
}

static int ftp_impl(sc_handle* h, const sc_ftp_args* args, sc_ftp_result* res,
                    double* y_tilde, double* best_y, long long* slot_cycles) {
    if (!h || !args || !res || !y_tilde || !best_y) return SC_EARG;
    memset(res, 0, sizeof(*res));
    if (h->broken) {
        h->err = "handle unusable after a multi-GPU exchange failure";
        return SC_ENCCL;
    }
    if (args->mode != SC_MODE_FTP && args->mode != SC_MODE_REFINE) return SC_EARG;
    if (!(args->alpha > 0.0)) { h->err = "alpha must be positive"; return SC_EARG; }
    const int64_t T = args->mode == SC_MODE_FTP ? args->budget : args->horizon;
    if (T < 0 || (args->mode == SC_MODE_REFINE && T < 1)) {
        h->err = "budget/horizon out of range";
        return SC_EARG;
    }
    CK(cudaSetDevice(h->prob.device), "set device");
    int st = ensure_ring(h, T);
    if (st != SC_OK) return st;
    KParams p;
    st = fill_params(h, p, slot_cycles);
    if (st != SC_OK) return st;
    h->last_alpha = args->alpha;
    p.args = *args;
    int status = -1;
    float ms = 0.f;
    st = launch(h, p, &status, &ms);
    if (st != SC_OK) return st;
    CK(h_get(h, res, h->res, sizeof(sc_ftp_result)), "copy result");
    CK(h_get(h, y_tilde, h->y_tilde, h->dd * 8), "copy y");
    CK(h_get(h, best_y, h->best_y, h->dd * 8), "copy y");
    res->kernel_ms = ms;
    h->pass_total += res->passes;
    h->has_callmin = res->has_counter_min != 0;
    h->has_sep = res->kind == SC_PRIMAL;
    return kernel_status(h, status);
}

// Balanced-partition calibration (see sm_weights): refine runs at the feasible end of the
// range (they never separate) report every SM's streaming cycles for its tiles.  Round 1
// runs with the equal cyclic partition; rounds 2-4 re-measure under the weighted partition
// (loading an SM's GPC changes its rate) and replace the weights (same box, us/pass:
// 1 round SES 135.4 SVM 131.4, 2 rounds 133.7 / 128.9, 4 rounds SVM another -0.6 %).  The handle's call
// state is restored afterwards (slots, pass counter, pd flags).
static bool probe_throughput(sc_handle* h, std::vector<double>& thr) {
    const int G = h->grid;
    sc_ftp_args a;
    memset(&a, 0, sizeof(a));
    a.mode = SC_MODE_REFINE;
    a.has_progress = 1;
    a.alpha = h->prob.kind == SC_SES ? h->prob.D : 1e-3 * h->prob.D;
    a.ceil_ln_r = (int64_t)ceil(h->prob.ln_r);
    a.horizon = std::max<int64_t>(24, a.ceil_ln_r);
    a.delta = 1e-4;
    a.patience = 10;
    a.enabled = 0;
    a.gain_rel = 1e-4;
    a.lo = -INFINITY;
    a.hi = INFINITY;
    a.target = NAN;
    long long* dc = nullptr;
    if (!(a.alpha > 0.0) || cudaMalloc(&dc, 2 * (size_t)G * sizeof(long long)) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    sc_ftp_result r;
    std::vector<double> yt(h->dd), by(h->dd);
    const int st = ftp_impl(h, &a, &r, yt.data(), by.data(), dc);
    std::vector<long long> hc(2 * (size_t)G);
    const bool ok = st == SC_OK && r.passes >= 16 &&
                    h_get(h, hc.data(), dc, hc.size() * 8) ==
                        cudaSuccess;
    cudaFree(dc);
    // restore the call state the probe touched
    h_zero(h, h->slots, (size_t)kNumSlots * h->slot_len * 8);
    h->has_sep = h->has_callmin = false;
    h->pass_total = 0;
    h->err.clear();
    if (!ok) { cudaGetLastError(); return false; }
    thr.assign(G, 0.0);
    for (int b = 0; b < G; ++b) {
        const int64_t c0 = h->cta_h[4 * b], c1 = h->cta_h[4 * b + 1], sd = h->cta_h[4 * b + 2];
        const int64_t tiles = c1 > c0 ? (c1 - c0 + sd - 1) / sd : 0;
        const long long cyc = hc[2 * b], sm = hc[2 * b + 1];
        if (sm < 0 || sm >= G || cyc <= 0 || tiles <= 0 || thr[sm] != 0.0) return false;
        thr[sm] = (double)tiles / (double)cyc;
    }
    return true;
}

static void calibrate_partition(sc_handle* h) {
    h->calib_tried = true;
    const int G = h->grid;
    const auto key = std::make_pair(h->prob.device, (const void*)h->fn);
    std::vector<double> thr;
    for (int round = 0; round < 4; ++round) {
        if (!probe_throughput(h, thr)) break;
        const double mx = *std::max_element(thr.begin(), thr.end());
        std::vector<double> w(G);
        for (int s = 0; s < G; ++s)
            w[s] = std::max(1.0, std::round(1024.0 * thr[s] / mx)) / 1024.0;
        {
            std::lock_guard<std::mutex> lock(g_calib_mu);
            g_calib[key] = w;
        }
        configure(h, h->grid_req);
        if (!h->by_smid) break;
    }
}

int sc_ftp(sc_handle* h, const sc_ftp_args* args, sc_ftp_result* res, double* y_tilde,
           double* best_y) {
    if (!h || !args || !res || !y_tilde || !best_y) return SC_EARG;
    if (h->balance_ok && !h->by_smid && !h->calib_tried) {
        CK(cudaSetDevice(h->prob.device), "set device");
        if (sm_weights(h) != nullptr) {   // another handle of this kernel calibrated
            h->calib_tried = true;
            configure(h, h->grid_req);
        } else {
            calibrate_partition(h);
        }
    }
    return ftp_impl(h, args, res, y_tilde, best_y, nullptr);
}

int sc_solve(sc_handle* h, const sc_solve_args* args, const double* seed_y,
             sc_solve_result* res, double* best_y, sc_search_step* steps) {
    if (!h || !args || !seed_y || !res || !best_y || (!steps && args->max_steps > 0))
        return SC_EARG;
    memset(res, 0, sizeof(*res));
    if (h->broken) {
        h->err = "handle unusable after a multi-GPU exchange failure";
        return SC_ENCCL;
    }
    if (!(args->eps > 0.0 && args->eps < 1.0) || !(args->L0 >= 0.0 && args->L0 < args->U0) ||
        args->max_steps < 0 || args->refine_horizon < 1) {
        h->err = "bad search arguments";
        return SC_EARG;
    }
    CK(cudaSetDevice(h->prob.device), "set device");
    if (h->balance_ok && !h->by_smid && !h->calib_tried) {   // opt-in (SCMWU_BALANCE=1)
        if (sm_weights(h) != nullptr) {
            h->calib_tried = true;
            configure(h, h->grid_req);
        } else {
            calibrate_partition(h);
        }
    }
    // the longest feasibility test of a search: a bracketing test (<= 2048) or a refine
    // round (<= refine_horizon)
    int st = ensure_ring(h, std::max<int64_t>(args->refine_horizon, kBracketTestCap));
    if (st != SC_OK) return st;
    const int nsteps = std::max(1, args->max_steps);
    if (h->steps_cap < nsteps) {
        pool_free(h->steps_dev, h->stream);
        h->steps_dev = nullptr;
        CK(pool_alloc((void**)&h->steps_dev, (size_t)nsteps * sizeof(sc_search_step),
                      h->prob.device, h->stream), "alloc step log");
        h->steps_cap = nsteps;
    }
    if (!h->sres_dev)
        CK(pool_alloc((void**)&h->sres_dev, sizeof(sc_solve_result), h->prob.device, h->stream),
           "alloc solve result");
    KParams p;
    st = fill_params(h, p, nullptr);
    if (st != SC_OK) return st;
    CK(h_put(h, h->yvec, seed_y, (size_t)h->prob.d * 8), "copy seed");
    CK(h_zero(h, h->slots + 3 * h->slot_len, h->slot_len * 8), "reset best_pd");  // per solve
    CK(h_zero(h, h->sres_dev, sizeof(sc_solve_result)), "reset solve result");
    p.solve = 1;
    p.sargs = *args;
    p.seed = h->yvec;
    p.sres = h->sres_dev;
    p.steps = h->steps_dev;
    p.args.mode = SC_MODE_FTP;   // unused: every test's arguments come from the search
    int status = -1;
    float ms = 0.f;
    st = launch(h, p, &status, &ms);
    if (st != SC_OK) return st;
    CK(h_get(h, res, h->sres_dev, sizeof(sc_solve_result)), "copy solve result");
    CK(h_get(h, best_y, h->best_y, h->dd * 8), "copy y");
    const int ns = std::min(res->search_steps, args->max_steps);
    if (ns > 0) CK(h_get(h, steps, h->steps_dev, (size_t)ns * sizeof(sc_search_step)), "copy steps");
    res->kernel_ms = ms;
    h->pass_total += res->passes;
    h->has_callmin = false;
    h->has_sep = false;
    return kernel_status(h, status);
}

int sc_progress_parts(sc_handle* h, const double* y, double* out) {
    if (!h || !y || !out) return SC_EARG;
    CK(cudaSetDevice(h->prob.device), "set device");
    const int d = h->prob.d;
    CK(cudaMemcpyAsync(h->yvec, y, d * 8, cudaMemcpyHostToDevice, h->stream), "copy y");
    const int blocks = std::min(h->sms * 4, 2048);
    progress_kernel<<<blocks, 256, 0, h->stream>>>(h->X, h->radii, h->prob.n_local,
                                                   h->prob.n1_local, d, h->ld, h->prob.kind,
                                                   h->yvec, h->scratch);
    h->launches += 1;
    CK(cudaGetLastError(), "progress kernel");
    std::vector<double> part(2 * blocks);
    CK(cudaMemcpyAsync(part.data(), h->scratch, part.size() * 8, cudaMemcpyDeviceToHost,
                       h->stream), "copy progress");
    CK(cudaStreamSynchronize(h->stream), "progress");
    if (h->prob.kind == SC_SES) {
        double m = -INFINITY;
        for (int b = 0; b < blocks; ++b) m = std::max(m, part[2 * b]);
        out[0] = m;
        out[1] = 0.0;
    } else {
        double mp = INFINITY, mq = -INFINITY;
        for (int b = 0; b < blocks; ++b) {
            mp = std::min(mp, part[2 * b]);
            mq = std::max(mq, part[2 * b + 1]);
        }
        out[0] = mp;
        out[1] = mq;
    }
    return SC_OK;
}

int sc_progress(sc_handle* h, const double* y, double* f) {
    if (!h || !y || !f) return SC_EARG;
    if (h->prob.world > 1) { h->err = "sharded handle: use sc_progress_parts"; return SC_EARG; }
    double parts[2];
    int st = sc_progress_parts(h, y, parts);
    if (st != SC_OK) return st;
    if (h->prob.kind == SC_SES) {
        *f = parts[0];
    } else {
        double nrm = 0.0;
        for (int j = 0; j < h->prob.d; ++j) nrm += y[j] * y[j];
        *f = Control<WarpLanes>::svm_margin(parts[0], parts[1], sqrt(nrm));
    }
    return SC_OK;
}

int sc_local_red0(sc_handle* h, double* out) {
    if (!h || !out) return SC_EARG;
    for (int j = 0; j < h->rw; ++j) out[j] = h->red0_h[j];
    return SC_OK;
}

int sc_set_globals(sc_handle* h, const double* red0, const double* v1, double g1) {
    if (!h || !red0) return SC_EARG;
    CK(cudaSetDevice(h->prob.device), "set device");
    for (int j = 0; j < h->rw; ++j) h->red0_h[j] = red0[j];
    CK(h_put(h, h->red0, red0, h->rw * 8), "copy red0");
    if (v1) CK(h_put(h, h->v1, v1, h->prob.d * 8), "copy anchor");
    h->g1 = g1;
    return SC_OK;
}

static size_t mbox_bytes(const sc_handle* h) {
    return 64 * 8 + 2 * (size_t)h->prob.world * h->rw * 8;
}

int sc_ipc_handle(sc_handle* h, void* out64) {
    if (!h || !out64 || h->prob.world <= 1) return SC_EARG;
    CK(cudaSetDevice(h->prob.device), "set device");
    if (!h->mbox_base) {
        CK(cudaMalloc(&h->mbox_base, mbox_bytes(h)), "alloc mailbox");
        CK(h_zero(h, h->mbox_base, mbox_bytes(h)), "zero mailbox");
        CK(cudaStreamSynchronize(h->stream), "zero mailbox");   // peers read it next
    }
    cudaIpcMemHandle_t ih;
    CK(cudaIpcGetMemHandle(&ih, h->mbox_base), "ipc handle");
    static_assert(sizeof(ih) == 64, "CUDA IPC handles are 64 bytes");
    memcpy(out64, &ih, 64);
    return SC_OK;
}

int sc_connect(sc_handle* h, const void* handles) {
    if (!h || !handles || h->prob.world <= 1 || !h->mbox_base) return SC_EARG;
    CK(cudaSetDevice(h->prob.device), "set device");
    for (int r = 0; r < h->prob.world; ++r) {
        if (r == h->prob.shard) { h->peer_base[r] = h->mbox_base; continue; }
        cudaIpcMemHandle_t ih;
        memcpy(&ih, static_cast<const char*>(handles) + 64 * r, 64);
        CK(cudaIpcOpenMemHandle(&h->peer_base[r], ih, cudaIpcMemLazyEnablePeerAccess),
           "open peer mailbox");
    }
    h->connected = true;
    return SC_OK;
}

int sc_iterate(sc_handle* h, double* out) {
    if (!h || !out) return SC_EARG;
    CK(cudaSetDevice(h->prob.device), "set device");
    const int64_t n = h->prob.n_local;
    const int64_t first = h->prob.kind == SC_SES && h->prob.row0 == 0 ? 1 : 0;
    const int64_t size = h->prob.kind == SC_SES ? (n - first) * (h->prob.d + 1) : n;
    double* buf = nullptr;
    CK(pool_alloc((void**)&buf, (size_t)std::max<int64_t>(size, 1) * 8, h->prob.device, h->stream),
       "alloc iterate");
    // the `last` slot holds the latest iterate's state (written by the last sc_ftp)
    iterate_kernel<<<(unsigned)((n + 255) / 256), 256, 0, h->stream>>>(
        h->X, h->radii, n, h->prob.n1_local, h->prob.d, h->ld, h->prob.kind,
        h->slots + 4 * h->slot_len, h->dd, h->prob.rho, h->last_alpha, buf, first);
    h->launches += 1;
    cudaError_t e = cudaStreamSynchronize(h->stream);
    if (e == cudaSuccess) e = h_get(h, out, buf, (size_t)size * 8);
    pool_free(buf, h->stream);
    if (e != cudaSuccess) return cuda_fail(h, e, "iterate");
    return SC_OK;
}

int sc_pd_commit(sc_handle* h, int32_t which) {
    if (!h || h->prob.kind != SC_SVM) return SC_EARG;
    if (which != 0 && which != 1 && which != 2) return SC_EARG;
    CK(cudaSetDevice(h->prob.device), "set device");
    if (which == 2) {   // back to the t = 0 state (uniform pair)
        CK(h_zero(h, h->slots + 3 * h->slot_len, h->slot_len * 8), "reset pair");
        return SC_OK;
    }
    const double* src = h->slots + (which == 0 ? 1 : 2) * h->slot_len;
    CK(h_copy(h, h->slots + 3 * h->slot_len, src, h->slot_len * 8, cudaMemcpyDeviceToDevice),
       "commit");
    return SC_OK;
}

int sc_pd_pair(sc_handle* h, double* mu, double* gam, double* dist) {
    if (!h || h->prob.kind != SC_SVM || !mu || !gam || !dist) return SC_EARG;
    CK(cudaSetDevice(h->prob.device), "set device");
    const int64_t n = h->prob.n_local, n1 = h->prob.n1_local;
    const int d = h->prob.d;
    double* buf = nullptr;
    CK(pool_alloc((void**)&buf, (size_t)n * 8, h->prob.device, h->stream), "alloc pair");
    // e_i * T from the committed state (T cancels in the normalisation below)
    std::vector<double> slot(h->slot_len);
    CK(h_get(h, slot.data(), h->slots + 3 * h->slot_len, h->slot_len * 8), "copy slot");
    IterState* st = reinterpret_cast<IterState*>(slot.data() + h->dd + (h->dd & 1));
    if (st->T == 0.0) {   // never committed: uniform weights (t = 0 state)
        st->T = 1.0; st->eta = 1.0; st->t = 0.0; st->shift = 0.0;
        CK(h_put(h, h->slots + 3 * h->slot_len, slot.data(), h->slot_len * 8), "init slot");
    }
    iterate_kernel<<<(unsigned)((n + 255) / 256), 256, 0, h->stream>>>(
        h->X, h->radii, n, n1, d, h->ld, SC_SVM, h->slots + 3 * h->slot_len, h->dd, h->prob.rho,
        0.0, buf, 0);
    h->launches += 1;
    std::vector<double> e(n);
    cudaError_t ce = cudaStreamSynchronize(h->stream);
    if (ce == cudaSuccess) ce = h_get(h, e.data(), buf, (size_t)n * 8);
    pool_free(buf, h->stream);
    if (ce != cudaSuccess) return cuda_fail(h, ce, "pd pair");
    if (h->prob.world > 1) {   // sharded: raw local weights, the host normalises globally
        for (int64_t i = 0; i < n1; ++i) mu[i] = e[i];
        for (int64_t i = n1; i < n; ++i) gam[i - n1] = e[i];
        *dist = NAN;
        return SC_OK;
    }
    double sP = 0.0, sQ = 0.0;
    for (int64_t i = 0; i < n1; ++i) sP += e[i];
    for (int64_t i = n1; i < n; ++i) sQ += e[i];
    for (int64_t i = 0; i < n1; ++i) mu[i] = e[i] / sP;
    for (int64_t i = n1; i < n; ++i) gam[i - n1] = e[i] / sQ;
    // distance of the uniform pair from the column sums; callers keep the committed one
    const int64_t N1 = h->prob.n1, N = h->prob.n;
    double s = 0.0;
    for (int j = 0; j < d; ++j) {
        double z = h->red0_h[kV_Vec + j] / (double)N1 - h->red0_h[kV_Vec + d + j] / (double)(N - N1);
        s += z * z;
    }
    *dist = sqrt(s);
    return SC_OK;
}

int sc_info(const sc_handle* h, int64_t* out) {
    if (!h || !out) return SC_EARG;
    out[0] = h->grid; out[1] = kThreads; out[2] = h->cfg.lpr; out[3] = h->cfg.cpl;
    out[4] = h->tile_rows; out[5] = h->stages; out[6] = h->resident; out[7] = (int64_t)h->smem;
    (void)h->cfg.nb;
    return SC_OK;
}

int sc_mark(sc_handle* h, int32_t which) {
    if (!h || (which != 0 && which != 1)) return SC_EARG;
    CK(cudaSetDevice(h->prob.device), "set device");
    CK(cudaEventRecord(which == 0 ? h->mk0 : h->mk1, h->stream), "mark");
    if (which == 1) CK(cudaEventSynchronize(h->mk1), "mark");
    return SC_OK;
}

int sc_elapsed(sc_handle* h, float* ms) {
    if (!h || !ms) return SC_EARG;
    CK(cudaEventElapsedTime(ms, h->mk0, h->mk1), "elapsed");
    return SC_OK;
}

int64_t sc_launches(const sc_handle* h) { return h ? h->launches : 0; }

int sc_debug_timing(sc_handle* h, double* out) {
    if (!h || !out) return SC_EARG;
    if (!h->timing) { for (int i = 0; i < 9 + 6 * 160 + 7; ++i) out[i] = 0.0; return SC_OK; }
    long long t[16 + 6 * 160 + 16];
    CK(h_get(h, t, h->timing, sizeof(t)), "copy timing");
    for (int i = 0; i < 9; ++i) out[i] = (double)t[i];
    for (int i = 0; i < 6 * 160; ++i) out[9 + i] = (double)t[16 + i];
    for (int i = 0; i < 7; ++i) out[9 + 6 * 160 + i] = (double)t[16 + 6 * 160 + i];
    return SC_OK;
}

const char* sc_last_error(const sc_handle* h) { return h ? h->err.c_str() : "null handle"; }

void sc_destroy(sc_handle* h) {
    if (!h) return;
    cudaSetDevice(h->prob.device);
    void* bufs[] = {h->X, h->radii, h->red0, h->partials, h->redg, h->row_begin, h->bar, h->timing,
                    h->ring, h->slots, h->res, h->y_tilde, h->best_y, h->scratch, h->yvec,
                    h->status, h->v1, h->mbox_base, h->steps_dev, h->sres_dev};
    for (int r = 0; r < kMaxWorld && h->vworld <= 1; ++r)   // emulated ranks: own memory
        if (h->peer_base[r] && h->peer_base[r] != h->mbox_base) cudaIpcCloseMemHandle(h->peer_base[r]);
    for (void* b : bufs)   // pool or cudaMalloc memory (pool_free tells them apart)
        if (b) { if (h->stream) pool_free(b, h->stream); else cudaFree(b); }
    if (h->ev0) cudaEventDestroy(h->ev0);
    if (h->ev1) cudaEventDestroy(h->ev1);
    if (h->mk0) cudaEventDestroy(h->mk0);
    if (h->mk1) cudaEventDestroy(h->mk1);
    if (h->stream) cudaStreamDestroy(h->stream);
    if (h->pool_open) pool_handle_close(h->prob.device);
    delete h;
}

}  // extern "C"
