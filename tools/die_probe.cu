// die_probe.cu — is the per-SM streaming rate set by the SM's die? (dev tool)
//
// 1) every CTA (one per SM) times dependent L2-hit loads of ONE fixed line: SMs on the
//    line's home die see a shorter latency than SMs on the other die (B300 notes:
//    234 vs 262 cycles), which splits the SMs into the two dies.
// 2) every CTA streams an equal contiguous share of a large buffer through per-warp bulk
//    copy rings (the engine's pattern) and records its own streaming time.
// Prints per-SM (die class, latency, streaming time) and the per-class means.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o die_probe tools/die_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void latency_kernel(const uint64_t* line, long long* out, int* smid_out) {
    if (threadIdx.x != 0) return;
    uint64_t idx = 0;
    long long best = 1LL << 60;
    for (int rep = 0; rep < 64; ++rep) {
        const long long t0 = clock64();
        for (int i = 0; i < 32; ++i) idx = __ldcg(line + (idx & 7));   // dependent chain
        const long long t = clock64() - t0;
        best = t < best ? t : best;
    }
    int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    out[blockIdx.x] = best / 32 + (long long)(idx & 0);
    smid_out[blockIdx.x] = smid;
}

__global__ void __launch_bounds__(256, 1)
stream_kernel(const char* X, size_t bytes, int tile, int S, int reps, long long* tout) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int W = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    unsigned char* ring = smem + 1024;
    const size_t per = bytes / gridDim.x / tile * tile;
    const char* base = X + (size_t)blockIdx.x * per;
    const int ntiles = (int)(per / tile);
    if (lane == 0)
        for (int s = 0; s < S; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[w * S + s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const long long t0 = clock64();
    uint32_t phase = 0;
    int s = 0;
    double acc = 0;
    for (int r = 0; r < reps; ++r) {
        int issued = 0, s_issue = 0;
        auto issue = [&](int q, int st) {
            uint64_t* b = &bars[w * S + st];
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)),
                         "r"(tile) : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], "
                "%2, [%3];" ::"r"(su32(ring + (size_t)(w * S + st) * tile)),
                "l"(base + (size_t)(w + q * W) * tile), "r"(tile), "r"(su32(b)) : "memory");
        };
        const int mine = (ntiles - w + W - 1) / W;
        if (lane == 0)
            for (; issued < S && issued < mine; ++issued) issue(issued, (s + issued) % S);
        issued = S < mine ? S : mine;
        s_issue = (s + issued) % S;
        for (int q = 0; q < mine; ++q) {
            uint64_t* b = &bars[w * S + s];
            uint32_t ok = 0;
            while (!ok)
                asm volatile(
                    "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
                    "selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(su32(b)), "r"(phase) : "memory");
            acc += reinterpret_cast<const double*>(ring + (size_t)(w * S + s) * tile)[lane];
            __syncwarp();
            if (issued < mine) {
                if (lane == 0) issue(issued, s_issue);
                ++issued;
                s_issue = s_issue + 1 == S ? 0 : s_issue + 1;
            }
            if (++s == S) { s = 0; phase ^= 1u; }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) tout[blockIdx.x] = clock64() - t0 + (acc == 1.2345 ? 1 : 0);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint64_t* line;
    cudaMalloc(&line, 4096);
    cudaMemset(line, 0, 4096);
    long long *lat, *tst;
    int* smid;
    cudaMalloc(&lat, sms * 8);
    cudaMalloc(&tst, sms * 8);
    cudaMalloc(&smid, sms * 4);
    const size_t bytes = (size_t)8e9;
    char* X;
    cudaMalloc(&X, bytes);
    cudaMemset(X, 0, bytes);
    latency_kernel<<<sms, 32>>>(line, lat, smid);
    const int tile = 13056, S = 2;
    const size_t sm = 1024 + (size_t)8 * S * tile;
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    stream_kernel<<<sms, 256, sm>>>(X, bytes, tile, S, 1, tst);   // warm-up
    stream_kernel<<<sms, 256, sm>>>(X, bytes, tile, S, 3, tst);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<long long> hl(sms), ht(sms);
    std::vector<int> hs(sms);
    cudaMemcpy(hl.data(), lat, sms * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(ht.data(), tst, sms * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hs.data(), smid, sms * 4, cudaMemcpyDeviceToHost);
    // split the latencies at the largest gap
    std::vector<long long> sl = hl;
    std::sort(sl.begin(), sl.end());
    long long cut = sl[0];
    long long gap = -1;
    for (int i = 1; i < sms; ++i)
        if (sl[i] - sl[i - 1] > gap) { gap = sl[i] - sl[i - 1]; cut = sl[i]; }
    double tn = 0, tf = 0;
    int nn = 0, nf = 0;
    for (int b = 0; b < sms; ++b) {
        const bool near = hl[b] < cut;
        printf("cta %3d sm %3d lat %4lld %s stream %lld\n", b, hs[b], hl[b], near ? "near" : "far ",
               ht[b]);
        if (near) { tn += ht[b]; ++nn; } else { tf += ht[b]; ++nf; }
    }
    printf("latency split at %lld (gap %lld): near %d SMs mean stream %.0f, far %d SMs mean "
           "stream %.0f\n", cut, gap, nn, nn ? tn / nn : 0.0, nf, nf ? tf / nf : 0.0);
    return 0;
}
