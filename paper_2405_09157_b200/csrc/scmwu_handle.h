// scmwu_handle.h — the engine handle shared by the host translation units
// (scmwu_host.cu: lifecycle, partition, feasibility tests; scmwu_baselines.cu: the
// verification baselines).  Private: not part of the C ABI.
#pragma once

#include "scmwu_kernel.cuh"

using namespace scmwu;

struct LaunchCfg {
    int lpr, cpl, nb;
};

struct sc_handle {
    sc_problem prob;
    int dd, ld, rw, pw, slot_len;
    LaunchCfg cfg;
    int sms = 0, grid = 0, gP = 0, tile_rows = 0, stages = 0, resident = 0;
    uint32_t stage_stride = 0, rad_off = 0;
    size_t smem = 0;
    KernelFn fn = nullptr;
    double g1 = 0.0;
    double last_alpha = 0.0;
    // device buffers
    double *X = nullptr, *radii = nullptr, *red0 = nullptr, *partials = nullptr, *redg = nullptr;
    int64_t* row_begin = nullptr;
    unsigned long long* bar = nullptr;
    double* ring = nullptr;
    int64_t ring_cap = 0;
    double* slots = nullptr;
    sc_ftp_result* res = nullptr;
    double *y_tilde = nullptr, *best_y = nullptr, *scratch = nullptr, *yvec = nullptr;
    int* status = nullptr;
    long long* timing = nullptr;     // SCMWU_TIMING=1: per-phase cycle sums of the last call
    double* v1 = nullptr;            // SES anchor row
    sc_search_step* steps_dev = nullptr;   // sc_solve: the search log
    int steps_cap = 0;
    sc_solve_result* sres_dev = nullptr;
    // sharding: this rank's mailbox (flags + 2 x world x rw doubles) and the peers'
    void* mbox_base = nullptr;
    void* peer_base[kMaxWorld] = {};
    bool connected = false;
    bool pool_open = false;          // counted in the device pool's live handles
    bool broken = false;             // a multi-GPU exchange failed: the handle is unusable
    int64_t pass_total = 0;          // passes of all previous calls (identical on all ranks)
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, mk0 = nullptr, mk1 = nullptr;
    int64_t launches = 0;
    // host state
    std::vector<double> red0_h;
    bool has_sep = false, has_callmin = false;
    bool by_smid = false;            // rows balanced per SM (configure)
    int vworld = 0;                  // tests: emulated ranks on this GPU (SCMWU_VWORLD)
    bool balance_ok = false;         // eligible for the balanced partition (configure)
    bool calib_tried = false;        // the calibration probe ran for this handle
    int grid_req = 0;
    std::vector<int64_t> cta_h;      // host copy of the partition {r0, r1, stride} per slot
    std::string err;
};

inline int cuda_fail(sc_handle* h, cudaError_t e, const char* what) {
    if (h) h->err = std::string(what) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? SC_EOOM : SC_ECUDA;
}
#define CK(call, what)                                   \
    do {                                                 \
        cudaError_t _e = (call);                         \
        if (_e != cudaSuccess) return cuda_fail(h, _e, what); \
    } while (0)

// Every copy and memset of a handle's buffers is ordered on the handle's stream (plain
// cudaMemset / cudaMemcpy would run on the legacy stream, which the handle's stream does
// not wait for); the synchronous forms wait for the stream before returning.
inline cudaError_t h_zero(sc_handle* h, void* p, size_t bytes) {
    return cudaMemsetAsync(p, 0, bytes, h->stream);
}
inline cudaError_t h_copy(sc_handle* h, void* dst, const void* src, size_t bytes,
                          cudaMemcpyKind kind) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, kind, h->stream);
    return e != cudaSuccess ? e : cudaStreamSynchronize(h->stream);
}
inline cudaError_t h_put(sc_handle* h, void* dst, const void* src, size_t bytes) {
    return h_copy(h, dst, src, bytes, cudaMemcpyHostToDevice);
}
inline cudaError_t h_get(sc_handle* h, void* dst, const void* src, size_t bytes) {
    return h_copy(h, dst, src, bytes, cudaMemcpyDeviceToHost);
}

// scmwu_host.cu: the engine's private stream-ordered pool (freed memory up to SCMWU_POOL_GB
// stays mapped while a handle of the device is alive); larger buffers use cudaMalloc
cudaError_t pool_alloc(void** p, size_t bytes, int device, cudaStream_t s);
void pool_free(void* p, cudaStream_t s);

// scmwu_gen.cu: draw a generated instance into the handle's X (and v1); *D_out = range
int generate_rows(sc_handle* h, const sc_gen* gen, double* D_out);
