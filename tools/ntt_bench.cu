// ntt_bench.cu -- standalone microbenchmark of forward-NTT kernel variants
// (N = 8192, one 60-bit prime).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I paper_2105_01827_b200/csrc tools/ntt_bench.cu -o tools/ntt_bench
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "gala_device.cuh"

typedef unsigned __int128 u128;
static u64 h_mulmod(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
static u64 h_pow(u64 b, u64 e, u64 q)
{
    u64 r = 1;
    b %= q;
    while (e) {
        if (e & 1) r = h_mulmod(r, b, q);
        b = h_mulmod(b, b, q);
        e >>= 1;
    }
    return r;
}
static int h_brv(int x, int logN)
{
    int r = 0;
    for (int i = 0; i < logN; i++) r |= ((x >> i) & 1) << (logN - 1 - i);
    return r;
}

#define CKE(x)                                                                      \
    do {                                                                            \
        cudaError_t e = (x);                                                        \
        if (e != cudaSuccess) {                                                     \
            printf("CUDA error %s at %d\n", cudaGetErrorString(e), __LINE__);       \
            exit(1);                                                                \
        }                                                                           \
    } while (0)

// A/C: one CTA per polynomial, twiddles from global
template <int RMAX, int THREADS>
__global__ void __launch_bounds__(THREADS, 1) v_percta(const u64* in, u64* out, const ulonglong2* tw, u64 q, int logN)
{
    extern __shared__ u64 sm[];
    const int N = 1 << logN;
    const u64* src = in + (long long)blockIdx.x * N;
    for (int i = threadIdx.x; i < N; i += blockDim.x) sm[pad(i)] = src[i];
    __syncthreads();
    ntt_fwd_smem<false, RMAX>(sm, tw, q, logN);
    u64* dst = out + (long long)blockIdx.x * N;
    for (int i = threadIdx.x; i < N; i += blockDim.x) dst[i] = csub(csub(sm[pad(i)], 2 * q), q);
}

// B: persistent CTA, twiddle table staged once in shared memory
template <int RMAX, int THREADS>
__global__ void __launch_bounds__(THREADS, 1) v_persist(const u64* in, u64* out, const ulonglong2* tw, u64 q, int logN,
                                                       int polys)
{
    extern __shared__ u64 sm[];
    const int N = 1 << logN;
    ulonglong2* stw = (ulonglong2*)(sm + padded_words(N));
    for (int i = threadIdx.x; i < N; i += blockDim.x) stw[i] = tw[i];
    for (int p = blockIdx.x; p < polys; p += gridDim.x) {
        const u64* src = in + (long long)p * N;
        for (int i = threadIdx.x; i < N; i += blockDim.x) sm[pad(i)] = src[i];
        __syncthreads();
        ntt_fwd_smem<true, RMAX>(sm, stw, q, logN);
        u64* dst = out + (long long)p * N;
        for (int i = threadIdx.x; i < N; i += blockDim.x) dst[i] = csub(csub(sm[pad(i)], 2 * q), q);
        __syncthreads();
    }
}

// H: 2 CTAs/SM (512 threads, 64 regs), each thread owns two radix-8 groups per pass
template <int RMAX, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) v_percta2(const u64* in, u64* out, const ulonglong2* tw, u64 q, int logN)
{
    extern __shared__ u64 sm[];
    const int N = 1 << logN;
    const u64* src = in + (long long)blockIdx.x * N;
    for (int i = threadIdx.x; i < N; i += blockDim.x) sm[pad(i)] = src[i];
    __syncthreads();
    ntt_fwd_smem<false, RMAX>(sm, tw, q, logN);
    u64* dst = out + (long long)blockIdx.x * N;
    for (int i = threadIdx.x; i < N; i += blockDim.x) dst[i] = csub(csub(sm[pad(i)], 2 * q), q);
}

// I: persistent, double-buffered: cp.async prefetch of the next polynomial while transforming the current
template <int RMAX, int THREADS>
__global__ void __launch_bounds__(THREADS, 1) v_pipe(const u64* in, u64* out, const ulonglong2* tw, u64 q, int logN, int polys)
{
    extern __shared__ u64 sm[];
    const int N = 1 << logN;
    u64* buf[2] = {sm, sm + padded_words(N)};
    int p = blockIdx.x, cur = 0;
    auto prefetch = [&](int pp, u64* b) {
        const u64* src = in + (long long)pp * N;
        for (int i = threadIdx.x; i < N; i += blockDim.x) {
            unsigned sa = (unsigned)__cvta_generic_to_shared(b + pad(i));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(src + i));
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    if (p < polys) prefetch(p, buf[0]);
    for (; p < polys; p += gridDim.x) {
        int nxt = p + gridDim.x;
        if (nxt < polys) prefetch(nxt, buf[cur ^ 1]);
        if (nxt < polys) asm volatile("cp.async.wait_group 1;\n" ::);
        else asm volatile("cp.async.wait_group 0;\n" ::);
        __syncthreads();
        ntt_fwd_smem<false, RMAX>(buf[cur], tw, q, logN);
        u64* dst = out + (long long)p * N;
        for (int i = threadIdx.x; i < N; i += blockDim.x) dst[i] = csub(csub(buf[cur][pad(i)], 2 * q), q);
        __syncthreads();
        cur ^= 1;
    }
}

// J: explicit pass plan; the first pass loads straight from global into registers
template <int R>
__device__ __forceinline__ void fwd_pass_from_global(const u64* __restrict__ g, u64* s, const ulonglong2* __restrict__ tw,
                                                     u64 q, int logN)
{
    const int N = 1 << logN;
    const int G = N >> R;
    const int lt = logN - R;
    const u64 q2 = 2 * q;
    for (int gi = threadIdx.x; gi < G; gi += blockDim.x) {
        const int off = gi;   // s0 = 0: blk = 0
        u64 x[1 << R];
#pragma unroll
        for (int k = 0; k < (1 << R); k++) x[k] = g[off + (k << lt)];
#pragma unroll
        for (int l = 0; l < R; l++) {
            const int m = 1 << l;
            const int half = 1 << (R - 1 - l);
#pragma unroll
            for (int k = 0; k < (1 << R); k++) {
                if (k & half) continue;
                const ulonglong2 w = __ldg(&tw[m + (k >> (R - l))]);
                u64 U = x[k];
                U = U >= q2 ? U - q2 : U;
                u64 V = shoup_lazy(x[k + half], w.x, w.y, q);
                x[k] = U + V;
                x[k + half] = U - V + q2;
            }
        }
#pragma unroll
        for (int k = 0; k < (1 << R); k++) s[pad(off + (k << lt))] = x[k];
    }
}

template <int R0, int R1, int R2, int R3, int R4, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) v_plan(const u64* in, u64* out, const ulonglong2* tw, u64 q, int logN)
{
    extern __shared__ u64 sm[];
    const int N = 1 << logN;
    const u64* src = in + (long long)blockIdx.x * N;
    fwd_pass_from_global<R0>(src, sm, tw, q, logN);
    __syncthreads();
    int s0 = R0;
    if (R1) { fwd_pass<(R1 ? R1 : 1)>(sm, tw, q, logN, s0); __syncthreads(); s0 += R1; }
    if (R2) { fwd_pass<(R2 ? R2 : 1)>(sm, tw, q, logN, s0); __syncthreads(); s0 += R2; }
    if (R3) { fwd_pass<(R3 ? R3 : 1)>(sm, tw, q, logN, s0); __syncthreads(); s0 += R3; }
    if (R4) { fwd_pass<(R4 ? R4 : 1)>(sm, tw, q, logN, s0); __syncthreads(); s0 += R4; }
    u64* dst = out + (long long)blockIdx.x * N;
    for (int i = threadIdx.x; i < N; i += blockDim.x) dst[i] = csub(csub(sm[pad(i)], 2 * q), q);
}

// K: special-form prime + reduced lazy reductions for q < 2^60 (16q < 2^64): the U fold to [0,2q)
// happens only at the first stage of each radix-8 pass; bounds grow by 2q per stage within the pass.
template <int R, bool SF>
__device__ __forceinline__ void fwd_pass_k(u64* s, const ulonglong2* __restrict__ tw, u64 q, int logN, int s0)
{
    const int N = 1 << logN;
    const int G = N >> R;
    const int lt = logN - s0 - R;
    const int t_end = 1 << lt;
    const u64 q2 = 2 * q, q4 = 4 * q, q8 = 8 * q;
    for (int g = threadIdx.x; g < G; g += blockDim.x) {
        const int blk = g >> lt, off = g & (t_end - 1);
        const int base = (blk << (logN - s0)) + off;
        u64 x[1 << R];
#pragma unroll
        for (int k = 0; k < (1 << R); k++) {
            u64 v = s[pad(base + (k << lt))];     // input < 8q: fold to [0, 2q)
            v = v >= q4 ? v - q4 : v;
            x[k] = v >= q2 ? v - q2 : v;
        }
#pragma unroll
        for (int l = 0; l < R; l++) {
            const int m = 1 << (s0 + l);
            const int half = 1 << (R - 1 - l);
#pragma unroll
            for (int k = 0; k < (1 << R); k++) {
                if (k & half) continue;
                const ulonglong2 w = __ldg(&tw[m + (blk << l) + (k >> (R - l))]);
                u64 U = x[k];
                u64 V = shoup_lz<SF>(x[k + half], w.x, w.y, q);
                x[k] = U + V;
                x[k + half] = U - V + q2;   // bounds: [0, (2 + 2(l+1)) q)
            }
        }
#pragma unroll
        for (int k = 0; k < (1 << R); k++) s[pad(base + (k << lt))] = x[k];   // < 8q
    }
    (void)q8;
}

template <bool SF>
__global__ void __launch_bounds__(512, 2) v_k(const u64* in, u64* out, const ulonglong2* tw, u64 q, int logN)
{
    extern __shared__ u64 sm[];
    const int N = 1 << logN;
    const u64* src = in + (long long)blockIdx.x * N;
    fwd_first_pass<1, SF>([=](int i) { return src[i]; }, sm, tw, q, logN);
    __syncthreads();
    for (int s0 = 1; s0 < logN; s0 += 3) {
        fwd_pass_k<3, SF>(sm, tw, q, logN, s0);
        __syncthreads();
    }
    u64* dst = out + (long long)blockIdx.x * N;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        u64 v = sm[pad(i)];
        v = v >= 4 * q ? v - 4 * q : v;
        v = v >= 2 * q ? v - 2 * q : v;
        dst[i] = v >= q ? v - q : v;
    }
}

template <bool SF>
__global__ void __launch_bounds__(512, 2) v_g(const u64* in, u64* out, const ulonglong2* tw, u64 q, int logN)
{
    extern __shared__ u64 sm[];
    const int N = 1 << logN;
    const u64* src = in + (long long)blockIdx.x * N;
    ntt_fwd_g<SF>([=](int i) { return src[i]; }, sm, tw, q, logN);
    u64* dst = out + (long long)blockIdx.x * N;
    for (int i = threadIdx.x; i < N; i += blockDim.x) dst[i] = csub(csub(sm[pad(i)], 2 * q), q);
}

// M: Montgomery-form twiddles (8 B each; w 2^64 mod q) and the special-form REDC: the product from four
// 32x32 partials, then redc_sf_lazy; same [0, 2q) lazy bound as Shoup
__device__ __forceinline__ u64 mont_lazy_pp(u64 x, u64 wm, u64 q)
{
    AccPP<> a;
    a.set(x, wm);
    u64 hi, lo;
    a.value(hi, lo);
    return redc_sf_lazy(hi, lo, q);
}
template <int R>
__device__ __forceinline__ void fwd_pass_m(u64* s, const u64* __restrict__ tw, u64 q, int logN, int s0)
{
    const int N = 1 << logN;
    const int G = N >> R;
    const int lt = logN - s0 - R;
    const int t_end = 1 << lt;
    const u64 q2 = 2 * q;
    for (int g = threadIdx.x; g < G; g += blockDim.x) {
        const int blk = g >> lt, off = g & (t_end - 1);
        const int base = (blk << (logN - s0)) + off;
        u64 x[1 << R];
#pragma unroll
        for (int k = 0; k < (1 << R); k++) x[k] = s[pad(base + (k << lt))];
#pragma unroll
        for (int l = 0; l < R; l++) {
            const int m = 1 << (s0 + l);
            const int half = 1 << (R - 1 - l);
#pragma unroll
            for (int k = 0; k < (1 << R); k++) {
                if (k & half) continue;
                const u64 w = __ldg(&tw[m + (blk << l) + (k >> (R - l))]);
                u64 U = x[k];
                U = U >= q2 ? U - q2 : U;
                u64 V = mont_lazy_pp(x[k + half], w, q);
                x[k] = U + V;
                x[k + half] = U - V + q2;
            }
        }
#pragma unroll
        for (int k = 0; k < (1 << R); k++) s[pad(base + (k << lt))] = x[k];
    }
}
__global__ void __launch_bounds__(512, 2) v_m(const u64* in, u64* out, const u64* tw, u64 q, int logN)
{
    extern __shared__ u64 sm[];
    const int N = 1 << logN;
    const u64* src = in + (long long)blockIdx.x * N;
    for (int i = threadIdx.x; i < N; i += blockDim.x) sm[pad(i)] = src[i];
    __syncthreads();
    fwd_pass_m<1>(sm, tw, q, logN, 0);
    __syncthreads();
    for (int s0 = 1; s0 < logN; s0 += 3) {
        fwd_pass_m<3>(sm, tw, q, logN, s0);
        __syncthreads();
    }
    u64* dst = out + (long long)blockIdx.x * N;
    for (int i = threadIdx.x; i < N; i += blockDim.x) dst[i] = csub(csub(sm[pad(i)], 2 * q), q);
}

// A: approximate Shoup quotient (three of the four 32x32 partials of x w'; the quotient is at most 2
// short, so the product lands in [0, 4q)) with q < 2^60 and 6q lazy bounds through the pass
__device__ __forceinline__ u64 shoup_approx_sf(u64 x, u64 w, u64 wsh, u64 q)
{
    const uint32_t x0 = (uint32_t)x, x1 = (uint32_t)(x >> 32), s0 = (uint32_t)wsh, s1 = (uint32_t)(wsh >> 32);
    const u64 qh = (u64)x1 * s1 + (((u64)x0 * s1) >> 32) + (((u64)x1 * s0) >> 32);
    const uint32_t a = (uint32_t)(q >> 32);
    const u64 hq = qh + ((u64)((uint32_t)qh * a) << 32);
    return x * w - hq;
}
template <int R>
__device__ __forceinline__ void fwd_pass_a(u64* s, const ulonglong2* __restrict__ tw, u64 q, int logN, int s0)
{
    const int N = 1 << logN;
    const int G = N >> R;
    const int lt = logN - s0 - R;
    const int t_end = 1 << lt;
    const u64 q2 = 2 * q, q4 = 4 * q;
    for (int g = threadIdx.x; g < G; g += blockDim.x) {
        const int blk = g >> lt, off = g & (t_end - 1);
        const int base = (blk << (logN - s0)) + off;
        u64 x[1 << R];
#pragma unroll
        for (int k = 0; k < (1 << R); k++) x[k] = s[pad(base + (k << lt))];
#pragma unroll
        for (int l = 0; l < R; l++) {
            const int m = 1 << (s0 + l);
            const int half = 1 << (R - 1 - l);
#pragma unroll
            for (int k = 0; k < (1 << R); k++) {
                if (k & half) continue;
                const ulonglong2 w = __ldg(&tw[m + (blk << l) + (k >> (R - l))]);
                u64 U = x[k];                       // < 6q
                U = U >= q4 ? U - q4 : U;
                U = U >= q2 ? U - q2 : U;           // [0, 2q)
                u64 V = shoup_approx_sf(x[k + half], w.x, w.y, q);   // [0, 4q)
                x[k] = U + V;                       // [0, 6q)
                x[k + half] = U - V + q4;           // (0, 6q)
            }
        }
#pragma unroll
        for (int k = 0; k < (1 << R); k++) s[pad(base + (k << lt))] = x[k];
    }
}
__global__ void __launch_bounds__(512, 2) v_a(const u64* in, u64* out, const ulonglong2* tw, u64 q, int logN)
{
    extern __shared__ u64 sm[];
    const int N = 1 << logN;
    const u64* src = in + (long long)blockIdx.x * N;
    fwd_first_pass<1, true>([=](int i) { return src[i]; }, sm, tw, q, logN);
    __syncthreads();
    for (int s0 = 1; s0 < logN; s0 += 3) {
        fwd_pass_a<3>(sm, tw, q, logN, s0);
        __syncthreads();
    }
    u64* dst = out + (long long)blockIdx.x * N;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        u64 v = sm[pad(i)];
        v = v >= 4 * q ? v - 4 * q : v;
        v = v >= 2 * q ? v - 2 * q : v;
        dst[i] = v >= q ? v - q : v;
    }
}

int main()
{
    const int logN = 13, N = 1 << logN;
    const u64 q = 1152921092289986561ull; // 60-bit special form a*2^32+1
    // primitive 2N-th root: g^((q-1)/2N), g least non-residue
    u64 g = 2;
    while (h_pow(g, (q - 1) / 2, q) == 1) g++;
    u64 psi = h_pow(g, (q - 1) / (2 * N), q);
    std::vector<ulonglong2> tw(N);
    for (int k = 0; k < N; k++) {
        u64 w = h_pow(psi, (u64)h_brv(k, logN), q);
        tw[k] = make_ulonglong2(w, (u64)(((u128)w << 64) / q));
    }
    const int P = 4096;
    std::vector<u64> h(P * (size_t)N);
    srand(1);
    for (auto& x : h) x = (((u64)rand() << 40) ^ ((u64)rand() << 20) ^ (u64)rand()) % q;
    u64 *din, *dref, *dout;
    ulonglong2* dtw;
    CKE(cudaMalloc(&din, h.size() * 8));
    CKE(cudaMalloc(&dref, h.size() * 8));
    CKE(cudaMalloc(&dout, h.size() * 8));
    CKE(cudaMalloc(&dtw, N * 16));
    CKE(cudaMemcpy(din, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
    CKE(cudaMemcpy(dtw, tw.data(), N * 16, cudaMemcpyHostToDevice));
    const int smem = padded_words(N) * 8;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double bfly = (double)P * (N / 2) * logN;
    std::vector<u64> ref(h.size()), got(h.size());

    auto run = [&](const char* name, auto launch, bool is_ref) {
        launch();
        CKE(cudaDeviceSynchronize());
        cudaEventRecord(a);
        for (int it = 0; it < 5; it++) launch();
        cudaEventRecord(b);
        CKE(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 5;
        CKE(cudaMemcpy(got.data(), is_ref ? dref : dout, got.size() * 8, cudaMemcpyDeviceToHost));
        if (is_ref) ref = got;
        bool ok = got == ref;
        printf("%-28s %8.3f ms  %7.1f Gbfly/s  %s\n", name, ms, bfly / (ms * 1e-3) / 1e9, ok ? "ok" : "MISMATCH");
    };

    CKE(cudaFuncSetAttribute(v_percta<3, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    run("A percta R3 T1024", [&] { v_percta<3, 1024><<<P, 1024, smem>>>(din, dref, dtw, q, logN); }, true);
    CKE(cudaFuncSetAttribute(v_percta<4, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    run("C percta R4 T512", [&] { v_percta<4, 512><<<P, 512, smem>>>(din, dout, dtw, q, logN); }, false);
    CKE(cudaFuncSetAttribute(v_percta<5, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    run("F percta R5 T256", [&] { v_percta<5, 256><<<P, 256, smem>>>(din, dout, dtw, q, logN); }, false);
    CKE(cudaFuncSetAttribute(v_percta<2, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    run("G percta R2 T1024", [&] { v_percta<2, 1024><<<P, 1024, smem>>>(din, dout, dtw, q, logN); }, false);
    const int smemB = smem + N * 16;
    CKE(cudaFuncSetAttribute(v_persist<3, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, smemB));
    run("B persist R3 T1024", [&] { v_persist<3, 1024><<<148, 1024, smemB>>>(din, dout, dtw, q, logN, P); }, false);
    CKE(cudaFuncSetAttribute(v_persist<4, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, smemB));
    run("E persist R4 T512", [&] { v_persist<4, 512><<<148, 512, smemB>>>(din, dout, dtw, q, logN, P); }, false);
    CKE(cudaFuncSetAttribute(v_percta2<3, 512, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    run("H percta R3 T512 x2", [&] { v_percta2<3, 512, 2><<<P, 512, smem>>>(din, dout, dtw, q, logN); }, false);
    CKE(cudaFuncSetAttribute(v_percta2<2, 512, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    run("H2 percta R2 T512 x2", [&] { v_percta2<2, 512, 2><<<P, 512, smem>>>(din, dout, dtw, q, logN); }, false);
    CKE(cudaFuncSetAttribute(v_percta2<3, 256, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    run("H3 percta R3 T256 x3", [&] { v_percta2<3, 256, 3><<<P, 256, smem>>>(din, dout, dtw, q, logN); }, false);
#define PLAN(name, a, b, c, d, e, T, MB)                                                                      \
    CKE(cudaFuncSetAttribute(v_plan<a, b, c, d, e, T, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));      \
    run(name, [&] { v_plan<a, b, c, d, e, T, MB><<<P, T, smem>>>(din, dout, dtw, q, logN); }, false);
    PLAN("J 3,3,3,3,1 T512x2 gl", 3, 3, 3, 3, 1, 512, 2)
    PLAN("J 4,3,3,3 T512x2 gl", 4, 3, 3, 3, 0, 512, 2)
    PLAN("J 3,3,3,4 T512x2 gl", 3, 3, 3, 4, 0, 512, 2)
    PLAN("J 1,3,3,3,3 T512x2 gl", 1, 3, 3, 3, 3, 512, 2)
    PLAN("J 4,4,4,1 T512x2 gl", 4, 4, 4, 1, 0, 512, 2)
    PLAN("J 3,3,3,3,1 T256x3 gl", 3, 3, 3, 3, 1, 256, 3)
    PLAN("J 3,3,3,3,1 T1024x1 gl", 3, 3, 3, 3, 1, 1024, 1)
    CKE(cudaFuncSetAttribute(v_g<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    run("G prod plan generic", [&] { v_g<false><<<P, 512, smem>>>(din, dout, dtw, q, logN); }, false);
    CKE(cudaFuncSetAttribute(v_g<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    run("G prod plan SF", [&] { v_g<true><<<P, 512, smem>>>(din, dout, dtw, q, logN); }, false);
    {
        std::vector<u64> twm(N);
        for (int k = 0; k < N; k++) twm[k] = (u64)((((u128)tw[k].x) << 64) % q);
        u64* dtwm;
        CKE(cudaMalloc(&dtwm, N * 8));
        CKE(cudaMemcpy(dtwm, twm.data(), N * 8, cudaMemcpyHostToDevice));
        CKE(cudaFuncSetAttribute(v_m, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        run("M montgomery tw + sf REDC", [&] { v_m<<<P, 512, smem>>>(din, dout, dtwm, q, logN); }, false);
        CKE(cudaFuncSetAttribute(v_g<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        run("G prod plan SF (again)", [&] { v_g<true><<<P, 512, smem>>>(din, dout, dtw, q, logN); }, false);
    }
    CKE(cudaFuncSetAttribute(v_a, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    run("A approx Shoup, 6q bounds", [&] { v_a<<<P, 512, smem>>>(din, dout, dtw, q, logN); }, false);
    run("A approx Shoup, 6q bounds", [&] { v_a<<<P, 512, smem>>>(din, dout, dtw, q, logN); }, false);
    CKE(cudaFuncSetAttribute(v_k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    run("K SF + pass-level folds", [&] { v_k<true><<<P, 512, smem>>>(din, dout, dtw, q, logN); }, false);
    CKE(cudaFuncSetAttribute(v_k<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    run("K generic + pass-level folds", [&] { v_k<false><<<P, 512, smem>>>(din, dout, dtw, q, logN); }, false);
    const int smemI = 2 * smem;
    CKE(cudaFuncSetAttribute(v_pipe<3, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, smemI));
    run("I pipe R3 T1024", [&] { v_pipe<3, 1024><<<148, 1024, smemI>>>(din, dout, dtw, q, logN, P); }, false);
    CKE(cudaFuncSetAttribute(v_pipe<4, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, smemI));
    run("I2 pipe R4 T512", [&] { v_pipe<4, 512><<<148, 512, smemI>>>(din, dout, dtw, q, logN, P); }, false);
    return 0;
}
