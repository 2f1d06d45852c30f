// mma_bench.cu -- tcgen05.mma issue-rate microbenchmark (one CTA per SM, one lane issuing back-to-back
// MMAs on zero operands into one TMEM accumulator; no other traffic).  Reports SM clocks per MMA and
// MACs per SM per clock for the int8 (kind::i8), fp8 (kind::f8f6f4) and bf16 (kind::f16) forms at
// M = 128, N = 128 / 256, K = 32 bytes, SWIZZLE_NONE (two core-matrix orders) and SWIZZLE_128B.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_bench tools/mma_bench.cu && tools/mma_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout)
{
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}

// KIND 0: i8 (s32 acc), 1: f16 bf16 (f32 acc), 2: f8f6f4 e4m3 (f32 acc).  LAY 0: none, kc-major
// (LBO = K-chunk stride, SBO 128); 1: none, row-group-major (LBO 128, SBO 256); 2: SWIZZLE_128B (SBO 1024)
template <int KIND, int N, int LAY, int CMT = 0, int BAR = 0, int ISS = 1>
__global__ void __launch_bounds__(128, 1) k_mma(int iters, unsigned long long* out)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar, dummy[64];
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (128 + 256) * 128 / 16; i += blockDim.x) ((uint4*)sm)[i] = make_uint4(0, 0, 0, 0);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        for (int i = 0; i < 64; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&dummy[i])));
        if (BAR < 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&dummy[31])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tbase;
    if ((threadIdx.x & 31) == 0 && warp < ISS) {   // ISS issuing warps, accumulator per warp
        const uint32_t tmem_w = tmem + (uint32_t)(warp * (256 / ISS) * 0);
        uint32_t idesc;
        if (KIND == 0) idesc = (2u << 4);
        else if (KIND == 1) idesc = (1u << 4) | (1u << 7) | (1u << 10);
        else idesc = (1u << 4);
        idesc |= ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 128 * 128);
        long long t0 = clock64();
        for (int r = 0; r < iters / ISS; r++) {
            uint64_t ad, bd;
            const int ks = r & 3;
            if (LAY == 0) { ad = desc(a0, 2048, 128, 0); bd = desc(b0, N * 16, 128, 0); }
            else if (LAY == 1) { ad = desc(a0, 128, 256, 0); bd = desc(b0, 128, 256, 0); }
            else { ad = desc(a0 + ks * 32, 16, 1024, 2); bd = desc(b0 + ks * 32, 16, 1024, 2); }
            const uint32_t acc = r ? 1u : 0u;
            if (KIND == 0)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_w), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
            else if (KIND == 1)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
            else
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
            if (BAR < 0 && (r & 1)) {   // -1: try_wait on a completed barrier every 2 MMAs; -2: test_wait
                uint32_t ok = 0;
                while (!ok) {
                    if (BAR == -1)
                        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                                     : "=r"(ok) : "r"(smem_u32(&dummy[31])) : "memory");
                    else
                        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                                     : "=r"(ok) : "r"(smem_u32(&dummy[31])) : "memory");
                }
            }
            if (CMT && (r % CMT) == CMT - 1) {
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&dummy[warp * 32 + ((r / (CMT ? CMT : 1)) & 31)])) : "memory");
                if (BAR) {   // wait for the commit of CMT MMAs before (BAR = 1: the previous one)
                    const int w = r / (CMT ? CMT : 1) - BAR;
                    if (w >= 0) {
                        uint32_t ok = 0;
                        const uint32_t ph = (uint32_t)((w >> 5) & 1);
                        while (!ok)
                            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                                         : "=r"(ok) : "r"(smem_u32(&dummy[warp * 32 + (w & 31)])), "r"(ph) : "memory");
                    }
                }
            }
        }
        if (warp == 0) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
        if (warp == 0) out[blockIdx.x] = (unsigned long long)(clock64() - t0);
    }
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

template <int KIND, int N, int LAY, int CMT = 0, int BAR = 0, int ISS = 1>
static int run(const char* name, int sms)
{
    const int smem = (128 + 256) * 128 + 1024;
    CK(cudaFuncSetAttribute(k_mma<KIND, N, LAY, CMT, BAR, ISS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    unsigned long long* d;
    CK(cudaMalloc(&d, sms * 8));
    const int iters = 20000;
    k_mma<KIND, N, LAY, CMT, BAR, ISS><<<sms, 128, smem>>>(100, d);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_mma<KIND, N, LAY, CMT, BAR, ISS><<<sms, 128, smem>>>(iters, d);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long h[1024];
    CK(cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost));
    double mx = 0;
    for (int i = 0; i < sms; i++) mx = h[i] > mx ? h[i] : mx;
    const double cpm = mx / iters;
    const double macs = 128.0 * N * 32 / (KIND == 1 ? 2 : 1);
    printf("%-28s %7.1f clk/MMA  %7.0f MAC/clk/SM  (%.3f ms, %.1f TMAC/s chip)\n", name, cpm, macs / cpm, ms,
           macs * iters * sms / (ms * 1e-3) / 1e12);
    cudaFree(d);
    return 0;
}

int main_ring();
int main(int argc, char** argv)
{
    if (argc > 1) return main_ring();
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0, 256, 0, 1>("i8   N256 commit/1", sms);
    run<0, 256, 0, 2>("i8   N256 commit/2", sms);
    run<0, 256, 0, 8>("i8   N256 commit/8", sms);
    run<0, 256, 0, 2, 1>("i8   N256 commit/2 wait-1", sms);
    run<0, 256, 0, 0, -1>("i8   N256 try_wait(done)/2", sms);
    run<0, 256, 0, 0, -2>("i8   N256 test_wait(done)/2", sms);
    run<0, 256, 0, 0, -1, 2>("i8   N256 try_wait/2 2 issuers", sms);
    run<0, 256, 0, 0, 0, 2>("i8   N256 2 issuers", sms);
    run<0, 256, 0, 8, 2>("i8   N256 commit/8 wait-2", sms);
    run<0, 256, 0, 8, 4>("i8   N256 commit/8 wait-4", sms);
    run<0, 256, 0, 2, 4, 2>("i8   N256 2iss commit/2 wait-4", sms);
    run<0, 256, 0, 2, 8, 2>("i8   N256 2iss commit/2 wait-8", sms);
    run<0, 256, 0, 4, 4, 2>("i8   N256 2iss commit/4 wait-4", sms);
    run<0, 256, 0, 2, 4>("i8   N256 commit/2 wait-4", sms);
    run<0, 256, 0, 2, 8>("i8   N256 commit/2 wait-8", sms);
    run<0, 256, 0, 2, 16>("i8   N256 commit/2 wait-16", sms);
    run<0, 256, 0, 2, 24>("i8   N256 commit/2 wait-24", sms);
    run<0, 256, 0, 8, 1>("i8   N256 commit/8 wait-1", sms);
    run<0, 128, 0>("i8   N128 none(kc)", sms);
    run<0, 256, 0>("i8   N256 none(kc)", sms);
    run<0, 256, 1>("i8   N256 none(rg)", sms);
    run<0, 256, 2>("i8   N256 sw128", sms);
    run<2, 256, 0>("f8   N256 none(kc)", sms);
    run<2, 256, 2>("f8   N256 sw128", sms);
    run<1, 256, 0>("bf16 N256 none(kc)", sms);
    run<1, 256, 2>("bf16 N256 sw128", sms);
    return 0;
}

// ---------------------------------------------------------------------------
// Ring round trip: issuer warp(s) wait full[s], issue K MMAs, commit empty[s]; a producer warp waits
// empty[s] and arrives full[s] (no data).  S slots; ISS issuers take alternate stages.
template <int K, int S, int ISS, int SPIN = 0, int RND = 0, int KFL = 0>
__global__ void __launch_bounds__(512, 1) k_ring(int stages, unsigned long long* out)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full[S], empty[S], done[2], never;
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < (128 + 256) * 128 / 16; i += blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u + blockIdx.x;
        uint4 v;
        v.x = h = h * 1664525u + 1013904223u; v.y = h = h * 1664525u + 1013904223u;
        v.z = h = h * 1664525u + 1013904223u; v.w = h * 1664525u + 1013904223u;
        ((uint4*)sm)[i] = RND ? v : make_uint4(0, 0, 0, 0);
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(KFL ? 512 : 256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; i++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[i])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[i])));
        }
        for (int i = 0; i < 2; i++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done[i])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&never)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tbase;
    volatile int* flag = (volatile int*)&tbase + 1;
    auto wait = [](uint64_t* b, uint32_t ph) {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(ok) : "r"(smem_u32(b)), "r"(ph) : "memory");
    };
    long long t0 = clock64();
    if (warp < ISS && lane == 0) {
        const uint32_t idesc = (2u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
        const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 128 * 128);
        for (int gs = warp; gs < stages; gs += ISS) {
            const int s = gs % S;
            wait(&full[s], (uint32_t)((gs / S) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;");
            for (int r = 0; r < K; r++) {
                uint64_t ad = desc(a0, 2048, 128, 0), bd = desc(b0, 4096, 128, 0);
                uint32_t dd = tmem;
                if (KFL) {   // k_gala_kf's addressing: rotating stage buffers, accumulator per 32 stages
                    ad = desc(a0 + s * K * 4096 + r * 4096, 2048, 128, 0);
                    bd = desc(a0 + S * K * 4096 + s * K * 8192 + r * 8192, 4096, 128, 0);
                    dd = tmem + (uint32_t)(((gs >> 5) & 1) * 256);
                }
                asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 1;" ::"r"(dd), "l"(ad), "l"(bd), "r"(idesc));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&done[warp])) : "memory");
        wait(&done[warp], 0);
        if (warp == 0) {
            out[blockIdx.x] = (unsigned long long)(clock64() - t0);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&never)) : "memory");
        }
    } else if (warp >= 4 && warp < 4 + SPIN) {   // SPIN warps, all lanes polling a barrier until the end
        wait(&never, 0);
    } else if (warp == 3 && lane == 0) {
        for (int gs = 0; gs < stages; gs++) {
            const int s = gs % S;
            wait(&empty[s], (uint32_t)(((gs / S) & 1) ^ 1));
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
        }
    }
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(KFL ? 512 : 256));
}

template <int K, int S, int ISS, int SPIN = 0, int RND = 0, int KFL = 0>
static int ring(int sms)
{
    const int smem = KFL ? S * K * 12288 + 1024 : (128 + 256) * 128 + 1024;
    CK(cudaFuncSetAttribute(k_ring<K, S, ISS, SPIN, RND, KFL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    unsigned long long* d;
    CK(cudaMalloc(&d, sms * 8));
    const int stages = 20000 / K;
    k_ring<K, S, ISS, SPIN, RND, KFL><<<sms, 512, smem>>>(64, d);
    CK(cudaDeviceSynchronize());
    k_ring<K, S, ISS, SPIN, RND, KFL><<<sms, 512, smem>>>(stages, d);
    CK(cudaDeviceSynchronize());
    unsigned long long h[1024];
    CK(cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost));
    double mx = 0;
    for (int i = 0; i < sms; i++) mx = h[i] > mx ? h[i] : mx;
    printf("ring K=%d MMAs/stage, S=%d slots, %d issuer(s), %2d spinning warps, %s data, kf layout %d: %6.1f clk/MMA\n", K, S, ISS, SPIN, RND ? "random" : "zero", KFL, mx / (stages * K));
    cudaFree(d);
    return 0;
}

int main_ring()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    ring<2, 8, 2>(sms); ring<2, 8, 2, 0, 1, 1>(sms); ring<2, 8, 2, 0, 0, 1>(sms); ring<8, 2, 1, 0, 1, 1>(sms); ring<8, 2, 2, 0, 1, 1>(sms);
    return 0;
}
