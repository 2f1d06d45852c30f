// imad_bench.cu -- issue-rate microbenchmark of the integer multiply flavours the modmul roof rests on
// (IMAD, IMAD.WIDE.U32, IMAD.HI.U32) and of the library's special-form Shoup modmul itself.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/imad_bench tools/imad_bench.cu && tools/imad_bench
//
// Each thread runs 8 independent chains (enough ILP to cover the 4-cycle latency) of one
// instruction flavour; 148 x 16 CTAs of 256 threads; the rate is instructions (or modmuls) per SM
// per clock at the measured SM clock.  Check the SASS with cuobjdump -sass: every chain body must
// be exactly one instruction of the flavour.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int KIND>
__global__ void __launch_bounds__(256) k_rate(uint32_t a, uint32_t b, int iters, uint64_t* sink)
{
    uint32_t x[8];
    uint64_t y[8];
#pragma unroll
    for (int i = 0; i < 8; i++) {
        x[i] = threadIdx.x * 8 + i + blockIdx.x;
        y[i] = x[i];
    }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            if (KIND == 0) {          // IMAD: x = x * a + b (32-bit)
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(a), "r"(b));
            } else if (KIND == 1) {   // IMAD.WIDE.U32: y = x * a + y (32 x 32 -> 64, accumulate)
                asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(y[i]) : "r"(x[i]), "r"(a));
                x[i] ^= (uint32_t)y[i];
            } else if (KIND == 2) {   // IMAD.HI.U32: x = hi(x * a) + b
                asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(a), "r"(b));
            } else {                  // IMAD.WIDE.U32 alone: y = x * a, x = hi(y) (a register alias, no extra op)
                asm volatile("{\n\t.reg .u64 t;\n\tmul.wide.u32 t, %0, %1;\n\tmov.b64 {%2, %0}, t;\n\t}"
                             : "+r"(x[i]) : "r"(a), "r"(b));
            }
        }
    }
    uint64_t acc = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) acc ^= x[i] ^ y[i];
    sink[blockIdx.x * 256 + threadIdx.x] = acc;
}

int main()
{
    int dev = 0, sms = 0, clk_khz = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
    const int blocks = sms * 16, iters = 1 << 14;
    uint64_t* sink;
    CK(cudaMalloc(&sink, (size_t)blocks * 256 * 8));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[4] = {"IMAD (mad.lo.u32)", "IMAD.WIDE.U32 (mad.wide.u32 acc) + LOP3", "IMAD.HI.U32 (mad.hi.u32)",
                             "IMAD.WIDE.U32 (mul.wide.u32, hi half fed back)"};
    for (int kind = 0; kind < 4; kind++) {
        for (int rep = 0; rep < 2; rep++) {
            CK(cudaEventRecord(e0));
            if (kind == 0) k_rate<0><<<blocks, 256>>>(3, 7, iters, sink);
            else if (kind == 1) k_rate<1><<<blocks, 256>>>(3, 7, iters, sink);
            else if (kind == 2) k_rate<2><<<blocks, 256>>>(3, 7, iters, sink);
            else k_rate<3><<<blocks, 256>>>(3, 7, iters, sink);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep == 0) continue;   // warm-up
            const double ops = (double)blocks * 256 * iters * 8;
            const double per_s = ops / (ms * 1e-3);
            printf("{\"flavour\": \"%s\", \"ms\": %.3f, \"Gops_per_s\": %.1f, \"ops_per_sm_per_clk_at_max\": %.2f}\n",
                   names[kind], ms, per_s / 1e9, per_s / sms / (clk_khz * 1e3));
        }
    }
    return 0;
}
