// mma2sm_check.cu -- semantics check of tcgen05.mma.cta_group::2.kind::i8 (M 256, N 256, K 32):
// each CTA of the pair stages its half of A (rows 128 r ..) and of B (rows 128 r ..) in the SWIZZLE_NONE
// K-major layout the key-folded kernel uses; rank 0 issues one MMA; both CTAs read their TMEM rows.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma2sm_check tools/mma2sm_check.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_check(const uint8_t* A, const uint8_t* B, int* D)
{
    __shared__ __align__(1024) uint8_t sa[128 * 32], sb[128 * 32];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // K-major no swizzle: chunk (row r, kc) at kc * 2048 + (r / 8) * 128 + (r % 8) * 16
    for (int i = tid; i < 128 * 2; i += blockDim.x) {
        const int r = i >> 1, kc = i & 1;
        for (int b = 0; b < 16; b++) {
            sa[kc * 2048 + (r >> 3) * 128 + (r & 7) * 16 + b] = A[(rank * 128 + r) * 32 + kc * 16 + b];
            sb[kc * 2048 + (r >> 3) * 128 + (r & 7) * 16 + b] = B[(rank * 128 + r) * 32 + kc * 16 + b];
        }
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tbase;
    if (rank == 0 && tid == 0) {
        const uint32_t idesc = (2u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
        const uint64_t ad = desc(smem_u32(sa), 2048, 128), bd = desc(smem_u32(sb), 2048, 128);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(0));
        const uint16_t mask = 3;
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                     ::"r"(smem_u32(&bar)), "h"(mask) : "memory");
    }
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int c0 = 0; c0 < 256; c0 += 8) {
        uint32_t x[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]), "=r"(x[7])
                     : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int i = 0; i < 8; i++) D[(rank * 128 + warp * 32 + lane) * 256 + c0 + i] = (int)x[i];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

int main()
{
    std::vector<uint8_t> A(256 * 32), B(256 * 32);
    srand(1);
    for (auto& v : A) v = (uint8_t)(rand() & 255);
    for (auto& v : B) v = (uint8_t)(rand() & 255);
    uint8_t *dA, *dB;
    int* dD;
    cudaMalloc(&dA, A.size());
    cudaMalloc(&dB, B.size());
    cudaMalloc(&dD, 256 * 256 * 4);
    cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, 256 * 256 * 4);
    k_check<<<2, 128>>>(dA, dB, dD);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    std::vector<int> D(256 * 256);
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0, shown = 0;
    for (int m = 0; m < 256; m++)
        for (int n = 0; n < 256; n++) {
            int ref = 0;
            for (int k = 0; k < 32; k++) ref += (int)A[m * 32 + k] * (int)B[n * 32 + k];
            if (ref != D[m * 256 + n]) {
                if (shown++ < 5) printf("m %d n %d got %d want %d\n", m, n, D[m * 256 + n], ref);
                bad++;
            }
        }
    printf("mismatches %d of %d\n", bad, 256 * 256);
    // which layout matches? try B halves swapped / interleaved
    return 0;
}
