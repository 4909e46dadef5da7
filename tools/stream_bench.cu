// stream_bench.cu — read-streaming ceiling of the engine's memory pattern (dev tool).
//
// 148 CTAs x W warps; each CTA owns a contiguous slice of a large buffer and each warp
// streams every W-th tile of it through its own ring of S shared-memory stages with
// 1-D bulk copies (cp.async.bulk + mbarrier complete_tx), exactly like the persistent
// kernel's per-warp rings.  After a stage lands the warp optionally spins `delay` cycles
// (a stand-in for the row math) and sums a few words, then refills the stage.  Also a
// plain LDG.128 streaming kernel for comparison.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o stream_bench tools/stream_bench.cu
//   ./stream_bench [GB]
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t su32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void __launch_bounds__(512, 1)
ring_kernel(const char* X, size_t bytes, int tile, int S, int delay, int reps, double* sink) {
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
    __syncwarp();
    double acc = 0.0;
    uint32_t phase = 0;
    int s = 0;                        // consumer position carries over between reps
    for (int r = 0; r < reps; ++r) {
        int issued = 0, s_issue = 0;
        auto issue = [&](int q, int st) {
            const int t = w + q * W;
            uint64_t* b = &bars[w * S + st];
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)),
                         "r"(tile)
                         : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], "
                "%2, [%3];" ::"r"(su32(ring + (size_t)(w * S + st) * tile)),
                "l"(base + (size_t)t * tile), "r"(tile), "r"(su32(b))
                : "memory");
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
                    "selp.u32 %0, 1, 0, p; }"
                    : "=r"(ok)
                    : "r"(su32(b)), "r"(phase)
                    : "memory");
            const double* st = reinterpret_cast<const double*>(ring + (size_t)(w * S + s) * tile);
            acc += st[lane];
            if (delay) {
                const long long t0 = clock64();
                while (clock64() - t0 < delay) {
                }
            }
            __syncwarp();
            if (issued < mine) {
                if (lane == 0) issue(issued, s_issue);
                ++issued;
                s_issue = s_issue + 1 == S ? 0 : s_issue + 1;
            }
            if (++s == S) { s = 0; phase ^= 1u; }
        }
    }
    if (acc == 12345.678) sink[0] = acc;
}

__global__ void ldg_kernel(const double2* X, size_t n2, int reps, double* sink) {
    double acc = 0.0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r) {
        size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
        for (; i + 7 * stride < n2; i += 8 * stride) {
            double2 v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = __ldcs(X + i + k * stride);
#pragma unroll
            for (int k = 0; k < 8; ++k) acc += v[k].x + v[k].y;
        }
    }
    if (acc == 12345.678) sink[0] = acc;
}

int main(int argc, char** argv) {
    const double gb = argc > 1 ? atof(argv[1]) : 8.0;
    const size_t bytes = (size_t)(gb * 1e9) & ~(size_t)0xFFFF;
    char* X;
    double* sink;
    cudaMalloc(&X, bytes);
    cudaMalloc(&sink, 8);
    cudaMemset(X, 1, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int reps = 3;
    {
        cudaError_t e = cudaDeviceSynchronize();
        printf("setup: %s (X=%p, %zu bytes)\n", cudaGetErrorString(e), (void*)X, bytes);
    }
    auto run_ring = [&](int W, int tile, int S, int delay) {
        const size_t sm = 1024 + (size_t)W * S * tile;
        if (sm > 227 * 1024) return;
        ring_kernel<<<sms, W * 32, sm>>>(X, bytes, tile, S, delay, 1, sink);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("ring W=%d tile=%d S=%d: %s\n", W, tile, S, cudaGetErrorString(e));
            exit(1);
        }
        cudaEventRecord(e0);
        ring_kernel<<<sms, W * 32, sm>>>(X, bytes, tile, S, delay, reps, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const size_t moved = bytes / sms / tile * tile * sms * reps;
        printf("ring W=%2d tile=%6d S=%2d inflight/SM=%4zu KB delay=%5d: %7.1f GB/s  %s\n", W,
               tile, S, (size_t)W * S * tile / 1024, delay, moved / (ms * 1e6),
               cudaGetErrorString(cudaGetLastError()));
    };
    for (int delay : {0, 1000, 3000})
        for (int W : {8, 16})
            for (int tile : {4096, 8192, 13056, 16384})
                for (int S : {2, 3, 4, 6})
                    run_ring(W, tile, S, delay);
    {
        ldg_kernel<<<sms * 4, 512>>>((const double2*)X, bytes / 16, 1, sink);
        cudaEventRecord(e0);
        ldg_kernel<<<sms * 4, 512>>>((const double2*)X, bytes / 16, reps, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("ldg.128 x8 unrolled: %.1f GB/s\n", (double)bytes * reps / (ms * 1e6));
    }
    return 0;
}
