// bulk_bench.cu -- per-SM global -> shared copy throughput from an L2-resident source, the way
// k_gala_kf streams its digit blocks: one CTA per SM, a ring of S slots of C bytes, one producer lane
// issuing cp.async.bulk (1-D TMA) with mbarrier complete_tx, one consumer lane releasing slots.
// Variants: spinning warps polling an mbarrier with all 32 lanes (k_gala_kf's expander/epilogue waits),
// and cp.async (LDGSTS, 16 B per thread) by W loader warps instead of the TMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bulk_bench tools/bulk_bench.cu && tools/bulk_bench
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool try_wait(uint64_t* b, uint32_t ph)
{
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(smem_u32(b)), "r"(ph) : "memory");
    return ok;
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) { while (!try_wait(b, ph)) {} }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory"); }

// MODE 0: TMA bulk, 1 producer lane.  MODE 1: cp.async 16 B by LW loader warps (ring slot split over them).
template <int MODE, int LW>
__global__ void __launch_bounds__(512, 1) k_copy(const uint8_t* __restrict__ src, long long span, int C, int S, int iters,
                                                  int spin_warps, unsigned long long* out, int nprod, int odd_idle)
{
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ uint64_t full[16], empty[16], never;
    __shared__ volatile int done;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; i++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[i])), "r"(MODE == 0 ? 1 : LW * 32));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[i])));
        }
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&never)));
        asm volatile("fence.mbarrier_init.release.cluster;");
        done = 0;
    }
    __syncthreads();
    // each CTA walks its own window of the (L2-resident) source
    const long long base = ((long long)blockIdx.x * 1315423911LL) % (span - (long long)C * iters % span - C + 1);
    long long t0 = 0;
    if (odd_idle && (blockIdx.x & 1)) {
        // idle partner CTA (same TPC when the launch uses clusters of 2)
    } else if (MODE == 0 && warp >= 2 + spin_warps && warp < 2 + spin_warps + nprod) {
        if (lane == 0) {
            const int me = warp - 2 - spin_warps;
            uint32_t ph = 0;
            int s = 0;
            t0 = clock64();
            for (int it = 0; it < iters; it++) {
                if (it % nprod != me) { if (++s == S) { s = 0; ph ^= 1; } continue; }
                wait(&empty[s], ph ^ 1);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(C) : "memory");
                const long long off = (base + (long long)it * C) % (span - C);
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(smem_u32(sm + (size_t)s * C)), "l"(src + (off & ~15LL)), "r"(C), "r"(smem_u32(&full[s])) : "memory");
                if (++s == S) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {   // consumer: releases each slot as soon as it lands
            uint32_t ph = 0;
            int s = 0;
            long long ts = clock64();
            for (int it = 0; it < iters; it++) {
                wait(&full[s], ph);
                arrive(&empty[s]);
                if (++s == S) { s = 0; ph ^= 1; }
            }
            const long long te = clock64();
            if (blockIdx.x == 0) { out[0] = (unsigned long long)(te - ts); }
            done = 1;
        }
    } else if (warp == 0) {
    } else if (MODE == 1 && warp >= 2 && warp < 2 + LW) {
        const int lt = (warp - 2) * 32 + lane;
        uint32_t ph = 0;
        int s = 0;
        for (int it = 0; it < iters; it++) {
            wait(&empty[s], ph ^ 1);
            const long long off = ((base + (long long)it * C) % (span - C)) & ~15LL;
            for (int b = lt * 16; b < C; b += LW * 32 * 16)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sm + (size_t)s * C + b)), "l"(src + off + b) : "memory");
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[s])) : "memory");
            if (++s == S) { s = 0; ph ^= 1; }
        }
    } else if (warp >= 2 + (MODE == 1 ? LW : 0) && warp < 2 + (MODE == 1 ? LW : 0) + spin_warps) {
        // spinning waiters (all lanes poll a barrier that completes only at the end)
        while (!done) try_wait(&never, 0);
    }
    __syncthreads();
    (void)t0;
}

__global__ void k_set(int* p) { *p = 1; }

int main()
{
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const long long span = 32ll << 20;   // 32 MB: L2-resident
    uint8_t* src;
    CK(cudaMalloc(&src, span + (1 << 20)));
    CK(cudaMemset(src, 1, span + (1 << 20)));
    unsigned long long* out;
    CK(cudaMalloc(&out, 4096));
    CK(cudaFuncSetAttribute(k_copy<0, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));

    CK(cudaFuncSetAttribute(k_copy<1, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    struct V { int mode, lw, C, S, spin, nprod, odd_idle; } vs[] = {
        {0, 1, 4096, 8, 0, 1, 0}, {0, 1, 16384, 6, 0, 1, 0}, {0, 1, 32768, 6, 0, 1, 0}, {0, 1, 65536, 3, 0, 1, 0},
        {0, 1, 4096, 8, 0, 1, 1}, {0, 1, 16384, 6, 0, 1, 1}, {0, 1, 32768, 6, 0, 1, 1},
        {0, 1, 4096, 8, 0, 4, 0}, {0, 1, 16384, 8, 0, 2, 0}, {0, 1, 16384, 8, 0, 4, 0}, {0, 1, 4096, 16, 0, 8, 0},
        {0, 1, 16384, 6, 12, 1, 0},
        {1, 8, 16384, 6, 0, 1, 0}, {1, 8, 16384, 6, 0, 1, 1},
    };
    for (auto v : vs) {
        const int iters = (int)((64ll << 20) / v.C);   // 64 MB per SM
        unsigned long long h = 0;
        CK(cudaMemset(out, 0, 4096));
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        const int threads = 64 + 32 * ((v.mode == 1 ? v.lw : 0) + v.spin + v.nprod);
        const size_t smem = (size_t)v.C * v.S;
        cudaEventRecord(e0);
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(sms); cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = smem; cfg.attrs = at; cfg.numAttrs = 1;
        if (v.mode == 0) CK(cudaLaunchKernelEx(&cfg, k_copy<0, 1>, (const uint8_t*)src, span, v.C, v.S, iters, v.spin, out, v.nprod, v.odd_idle));
        else CK(cudaLaunchKernelEx(&cfg, k_copy<1, 8>, (const uint8_t*)src, span, v.C, v.S, iters, v.spin, out, v.nprod, v.odd_idle));
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        CK(cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost));
        const double bytes = (double)iters * v.C;
        const int copiers = v.odd_idle ? sms / 2 : sms;
        printf("%s LW=%d C=%6d S=%2d spin=%2d prod=%d %s: %7.1f B/clk/CTA (CTA 0 clocks)  chip %.2f TB/s (events)\n",
               v.mode == 0 ? "bulk   " : "cp.async", v.lw, v.C, v.S, v.spin, v.nprod, v.odd_idle ? "1 of 2 per pair" : "every CTA     ",
               bytes / (double)h, bytes * copiers / (ms * 1e-3) / 1e12);
    }
    return 0;
}
