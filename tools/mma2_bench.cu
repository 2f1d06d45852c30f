// mma2_bench.cu -- issue rate of tcgen05.mma.cta_group::2.kind::i8 (the k_gala_kf MMA: M 256 across a CTA
// pair, N 256, K 32, SWIZZLE_NONE K-major) with zero operands, committing every CMT MMAs (multicast to both
// CTAs), and before each group waiting for the commit of the group DEP back:
//   MODE 0: one issuing thread that waits on the mbarrier itself;
//   MODE 1: two issuing threads (warps 0 and 1) taking alternate groups, each waiting on the mbarrier;
//   MODE 2: one issuing thread polling a shared-memory flag that a helper thread sets after its own
//           mbarrier wait (the issuer never touches an mbarrier).
// Reports SM clocks per MMA (each SM computes 128 x 256 x 32 per MMA: 128 clocks at the tensor peak).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma2_bench tools/mma2_bench.cu && tools/mma2_bench
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}
__device__ __forceinline__ void wait_cl(uint64_t* b, uint32_t ph)
{
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(b)), "r"(ph) : "memory");
}

template <int CMT, int DEP, int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_mma2(int iters, unsigned long long* out)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar[64], fin;
    __shared__ uint32_t tbase;
    __shared__ volatile int flag;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 2 * 4096 / 16; i += blockDim.x) ((uint4*)sm)[i] = make_uint4(0, 0, 0, 0);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < 64; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&fin)), "r"(MODE == 1 ? 2 : 1));
        asm volatile("fence.mbarrier_init.release.cluster;");
        flag = 0;
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tbase;
    const uint16_t mask = 3;
    const bool issuer = rank == 0 && lane == 0 && (warp == 0 || (MODE == 1 && warp == 1));
    if (issuer) {
        const int me = MODE == 1 ? warp : 0, nis = MODE == 1 ? 2 : 1;
        const uint32_t idesc = (2u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
        const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 4096);
        const long long t0 = clock64();
        for (int r = 0; r < iters; r++) {
            const int gi = r / CMT;
            if (gi % nis != me) continue;
            if (r % CMT == 0 && DEP) {   // before a group: wait for the commit DEP groups back
                const int w = gi - DEP;
                if (w >= 0) {
                    if (MODE == 2) {
                        while (flag < w + 1) {
                        }
                    } else {
                        wait_cl(&bar[w & 63], (uint32_t)((w >> 6) & 1));
                    }
                }
            }
            const uint64_t ad = desc(a0, 2048, 128), bd = desc(b0, 2048, 128);
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(1u));
            if (r % CMT == CMT - 1)
                asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                             ::"r"(smem_u32(&bar[gi & 63])), "h"(mask) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                     ::"r"(smem_u32(&fin)), "h"(mask) : "memory");
        if (me == 0) {
            wait_cl(&fin, 0);
            out[blockIdx.x >> 1] = (unsigned long long)(clock64() - t0);
        }
    } else if (MODE == 2 && rank == 0 && warp == 2 && lane == 0) {   // helper: barrier completions -> flag
        for (int g = 0; g < iters / CMT; g++) {
            wait_cl(&bar[g & 63], (uint32_t)((g >> 6) & 1));
            flag = g + 1;
        }
    } else if (rank == 1 && threadIdx.x == 0) {
        wait_cl(&fin, 0);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

template <int CMT, int DEP, int MODE>
static int run(const char* name, int sms)
{
    const int smem = 2 * 4096 + 1024;
    CK(cudaFuncSetAttribute(k_mma2<CMT, DEP, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    unsigned long long* d;
    CK(cudaMalloc(&d, sms * 8));
    const int iters = 20480;
    k_mma2<CMT, DEP, MODE><<<sms, 128, smem>>>(128, d);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_mma2<CMT, DEP, MODE><<<sms, 128, smem>>>(iters, d);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    CK(cudaGetLastError());
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long h[1024];
    CK(cudaMemcpy(h, d, sms / 2 * 8, cudaMemcpyDeviceToHost));
    double mx = 0;
    for (int i = 0; i < sms / 2; i++) mx = h[i] > mx ? h[i] : mx;
    printf("cta_group::2 i8 M256 N256 K32 %-28s %7.1f clk/MMA per SM (%.3f ms)\n", name, mx / iters, ms);
    cudaFree(d);
    return 0;
}

int main()
{
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    sms &= ~1;
    run<8, 0, 0>("commit/8, no waits", sms);
    run<8, 2, 0>("commit/8 wait-2", sms);
    run<8, 3, 0>("commit/8 wait-3", sms);
    run<8, 2, 1>("2 issuers commit/8 wait-2", sms);
    run<8, 3, 1>("2 issuers commit/8 wait-3", sms);
    run<8, 4, 1>("2 issuers commit/8 wait-4", sms);
    run<8, 2, 2>("flag-poll commit/8 wait-2", sms);
    run<8, 3, 2>("flag-poll commit/8 wait-3", sms);
    return 0;
}
