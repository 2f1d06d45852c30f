// gala_device.cuh -- sm_100a device primitives for 60-bit-class RNS arithmetic.
//
// Modular multiply flavours (all on the 32-bit IMAD pipe via mul.lo/mul.hi.u64):
//   * Shoup   (fixed operand w with companion w' = floor(w 2^64 / q)): NTT twiddles
//   * Montgomery REDC (R = 2^64): plaintext and key operands stored pre-scaled by R,
//     so products and 128-bit lazy sums reduce with one REDC
// Harvey lazy butterflies keep NTT values in [0, 4q); all primes are < 2^62.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

typedef uint64_t u64;
typedef int64_t i64;

#define GALA_MAXM 8   // ciphertext primes + special prime + plaintext modulus

struct ModC {
    u64 q;        // modulus
    u64 qinv_neg; // -q^-1 mod 2^64
    u64 r2;       // 2^128 mod q (to Montgomery form via REDC(x * r2))
};

// Everything a kernel needs about one BFV context, passed by value.
struct DevCtx {
    int N, logN, L, M;          // M = L + 1 (special prime at index L); plaintext at index M
    ModC mod[GALA_MAXM];
    const ulonglong2* twf[GALA_MAXM]; // psi^brv(k), Shoup companion
    const ulonglong2* twi[GALA_MAXM]; // psi^-brv(k), Shoup companion
    u64 ninv[GALA_MAXM], ninv_sh[GALA_MAXM];
    u64 delta[GALA_MAXM];       // floor(Q/p) mod q_j
    u64 delta_sh[GALA_MAXM];
    u64 pinv_mont[GALA_MAXM];   // P^-1 * R mod q_j (Montgomery operand)
    u64 qhat_inv[GALA_MAXM];    // [(Q/q_i)^-1]_{q_i}
    u64 qhat_inv_sh[GALA_MAXM];
    int lazy[GALA_MAXM];        // products a 128-bit accumulator may take before REDC: k q^2 < q 2^64
    u64 p;                      // plaintext modulus
    const u64* S;               // secret, NTT (bit-reversed), Montgomery form, [M][N]
    const int* slot_pos;        // slot index -> bit-reversed NTT_p position
};

// ---------------------------------------------------------------------------
// scalar arithmetic
__device__ __forceinline__ u64 csub(u64 x, u64 q) { return x >= q ? x - q : x; }
__device__ __forceinline__ u64 add_mod(u64 a, u64 b, u64 q) { return csub(a + b, q); }
__device__ __forceinline__ u64 sub_mod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }

// Shoup: x * w mod q, result in [0, 2q) for any x < 2^64 (w < q)
__device__ __forceinline__ u64 shoup_lazy(u64 x, u64 w, u64 wsh, u64 q)
{
    u64 hi = __umul64hi(x, wsh);
    return x * w - hi * q;
}
__device__ __forceinline__ u64 shoup(u64 x, u64 w, u64 wsh, u64 q) { return csub(shoup_lazy(x, w, wsh, q), q); }

// Shoup for special-form primes q = a 2^32 + 1: hi * q mod 2^64 = hi + ((lo32(hi) a mod 2^32) << 32),
// one 32-bit IMAD instead of a 64x64 low product.  Same result as shoup_lazy.
__device__ __forceinline__ u64 shoup_lazy_sf(u64 x, u64 w, u64 wsh, u64 q)
{
    const u64 hi = __umul64hi(x, wsh);
    const uint32_t a = (uint32_t)(q >> 32);
    const u64 hq = hi + ((u64)((uint32_t)hi * a) << 32);
    return x * w - hq;
}
template <bool SF>
__device__ __forceinline__ u64 shoup_lz(u64 x, u64 w, u64 wsh, u64 q)
{
    if (SF) return shoup_lazy_sf(x, w, wsh, q);
    return shoup_lazy(x, w, wsh, q);
}

// Montgomery REDC of hi:lo < q 2^64 for a special-form q = a 2^32 + 1 (every prime REDC sees;
// gala_create rejects others): returns (hi:lo) 2^-64 mod q in [0, 2q).  -q^-1 = a 2^32 - 1 mod 2^64,
// so m = lo (-q^-1) is one 32-bit multiply, and hi64(m q) = m1 a + ((m0 a + m1) >> 32) is two
// 32x32 wide products; the carry of lo + lo64(m q) is (lo != 0).
__device__ __forceinline__ u64 redc_sf_lazy(u64 hi, u64 lo, u64 q)
{
    u64 r;
    asm("{\n\t.reg .u32 lo0, lo1, h0, h1, t, m0, m1, th, u0, u1, nz, a;\n\t.reg .pred p;\n\t"
        "mov.b64 {lo0, lo1}, %1;\n\t"
        "mov.b64 {h0, h1}, %2;\n\t"
        "mov.b64 {t, a}, %3;\n\t"
        "mul.lo.u32 t, lo0, a;\n\t"
        "sub.cc.u32 m0, 0, lo0;\n\t"
        "subc.u32 m1, t, lo1;\n\t"
        "mad.lo.cc.u32 t, m0, a, m1;\n\t"
        "madc.hi.u32 th, m0, a, 0;\n\t"
        "mad.lo.cc.u32 u0, m1, a, th;\n\t"
        "madc.hi.u32 u1, m1, a, 0;\n\t"
        "or.b32 t, lo0, lo1;\n\t"
        "setp.ne.u32 p, t, 0;\n\t"
        "selp.u32 nz, 1, 0, p;\n\t"
        "add.cc.u32 h0, h0, u0;\n\t"
        "addc.u32 h1, h1, u1;\n\t"
        "add.cc.u32 h0, h0, nz;\n\t"
        "addc.u32 h1, h1, 0;\n\t"
        "mov.b64 %0, {h0, h1};\n\t"
        "}"
        : "=l"(r)
        : "l"(lo), "l"(hi), "l"(q));
    return r;
}
__device__ __forceinline__ u64 redc_lazy(u64 hi, u64 lo, const ModC& m) { return redc_sf_lazy(hi, lo, m.q); }
__device__ __forceinline__ u64 mont_mul(u64 a, u64 b, const ModC& m)
{
    return csub(redc_lazy(__umul64hi(a, b), a * b, m), m.q);
}
struct Acc128 {
    u64 lo, hi;
    __device__ __forceinline__ Acc128() : lo(0), hi(0) {}
    __device__ __forceinline__ void mac(u64 a, u64 b)
    {
        u64 l = a * b, h = __umul64hi(a, b);
        lo += l;
        hi += h + (lo < l ? 1ull : 0ull);
    }
    __device__ __forceinline__ u64 reduce(const ModC& m) const { return csub(redc_lazy(hi, lo, m), m.q); }
};

// 128-bit sum of products built from 32x32 -> 64 partial products, each accumulated in its own
// register by one IMAD.WIDE.U32 (the a0 b0 partials through a carry chain).  Valid wherever Acc128
// is: for k products of operands below A, B (both >= q) with k A B < q 2^64, the cross sums stay
// below k B < 2^64 and k A < 2^64.  set() starts the sum with its first product.  MERGE keeps the
// two cross sums in one register: only for 2 k max(A, B) < 2^64 (e.g. up to 4 canonical products
// with q < 2^60, or 1 with q < 2^62).
template <bool MERGE = false>
struct AccPP {
    u64 s00, s01, s10, s11;
    uint32_t c00;
    __device__ __forceinline__ AccPP() {}
    __device__ __forceinline__ void clear() { s00 = s01 = s10 = s11 = 0; c00 = 0; }
    __device__ __forceinline__ void set(u64 a, u64 b)
    {
        const uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32), b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
        s00 = (u64)a0 * b0;
        c00 = 0;
        s01 = (u64)a0 * b1;
        if (MERGE) s01 += (u64)a1 * b0;
        else s10 = (u64)a1 * b0;
        s11 = (u64)a1 * b1;
    }
    __device__ __forceinline__ void mac(u64 a, u64 b)
    {
        const uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32), b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
        asm("{\n\t.reg .u64 t;\n\tmul.wide.u32 t, %2, %3;\n\tadd.cc.u64 %0, %0, t;\n\taddc.u32 %1, %1, 0;\n\t}"
            : "+l"(s00), "+r"(c00)
            : "r"(a0), "r"(b0));
        s01 += (u64)a0 * b1;
        if (MERGE) s01 += (u64)a1 * b0;
        else s10 += (u64)a1 * b0;
        s11 += (u64)a1 * b1;
    }
    // the 128-bit sum as hi:lo
    __device__ __forceinline__ void value(u64& hi, u64& lo) const
    {
        if (MERGE) {
            asm("{\n\t.reg .u32 x0, x1, l0, l1, h0, h1;\n\t"
                "mov.b64 {x0, x1}, %3;\n\t"
                "mov.b64 {l0, l1}, %2;\n\t"
                "mov.b64 {h0, h1}, %4;\n\t"
                "add.cc.u32 l1, l1, x0;\n\t"
                "addc.cc.u32 h0, h0, x1;\n\t"
                "addc.u32 h1, h1, 0;\n\t"
                "add.cc.u32 h0, h0, %5;\n\t"
                "addc.u32 h1, h1, 0;\n\t"
                "mov.b64 %0, {h0, h1};\n\t"
                "mov.b64 %1, {l0, l1};\n\t"
                "}"
                : "=l"(hi), "=l"(lo)
                : "l"(s00), "l"(s01), "l"(s11), "r"(c00));
            return;
        }
        asm("{\n\t.reg .u32 x0, x1, y0, y1, m0, m1, m2, l0, l1, h0, h1;\n\t"
            "mov.b64 {x0, x1}, %3;\n\t"
            "mov.b64 {y0, y1}, %4;\n\t"
            "add.cc.u32 m0, x0, y0;\n\t"            // mid = s01 + s10 (65 bits)
            "addc.cc.u32 m1, x1, y1;\n\t"
            "addc.u32 m2, 0, 0;\n\t"
            "mov.b64 {l0, l1}, %2;\n\t"
            "mov.b64 {h0, h1}, %5;\n\t"
            "add.cc.u32 l1, l1, m0;\n\t"            // lo = s00 + (mid << 32)
            "addc.cc.u32 h0, h0, m1;\n\t"           // hi = s11 + (mid >> 32) + carries + c00
            "addc.u32 h1, h1, m2;\n\t"
            "add.cc.u32 h0, h0, %6;\n\t"
            "addc.u32 h1, h1, 0;\n\t"
            "mov.b64 %0, {h0, h1};\n\t"
            "mov.b64 %1, {l0, l1};\n\t"
            "}"
            : "=l"(hi), "=l"(lo)
            : "l"(s00), "l"(s01), "l"(s10), "l"(s11), "r"(c00));
    }
    __device__ __forceinline__ u64 reduce_sf(u64 q) const
    {
        u64 hi, lo;
        value(hi, lo);
        return csub(redc_sf_lazy(hi, lo, q), q);
    }
};

// streaming (evict-first) global accesses for polynomial data, so the twiddle
// tables keep their L1 residency
__device__ __forceinline__ u64 ld_cs(const u64* p) { return (u64)__ldcs((const unsigned long long*)p); }
__device__ __forceinline__ void st_cs(u64* p, u64 v) { __stcs((unsigned long long*)p, (unsigned long long)v); }

__device__ __forceinline__ int brv(int x, int logN) { return (int)(__brev((unsigned)x) >> (32 - logN)); }

// Galois automorphism X -> X^g on the bit-reversed NTT domain:
// out[i] = in[ auto_src(i) ]
__device__ __forceinline__ int auto_src(int i, u64 g, int logN)
{
    unsigned two_n_mask = (2u << logN) - 1u;
    unsigned nat = (unsigned)brv(i, logN);
    unsigned e = ((2u * nat + 1u) * (unsigned)g) & two_n_mask;
    return brv((int)((e - 1u) >> 1), logN);
}

// shared-memory index padding: one 8-byte word per 32 (bank-conflict relief
// for the small-stride NTT passes)
__device__ __forceinline__ int pad(int i) { return i + (i >> 5); }
__host__ __device__ constexpr int padded_words(int n) { return n + (n >> 5); }

// ---------------------------------------------------------------------------
// In-shared-memory negacyclic NTT.  Forward: Cooley-Tukey, natural -> bit-reversed,
// merged psi powers; inverse: Gentleman-Sande, bit-reversed -> natural (without the
// N^-1 scale).  A pass processes R consecutive stages in registers: each thread owns
// groups of 2^R elements spaced t_end apart.
template <bool TW_SMEM>
__device__ __forceinline__ ulonglong2 tw_load(const ulonglong2* p)
{
    if (TW_SMEM) return *p;
    return __ldg(p);
}

template <int R, bool TW_SMEM = false, bool SF = false>
__device__ __forceinline__ void fwd_pass(u64* s, const ulonglong2* __restrict__ tw, u64 q, int logN, int s0)
{
    const int N = 1 << logN;
    const int G = N >> R;
    const int lt = logN - s0 - R;      // log2(t_end)
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
                const ulonglong2 w = tw_load<TW_SMEM>(&tw[m + (blk << l) + (k >> (R - l))]);
                u64 U = x[k];
                U = U >= q2 ? U - q2 : U;
                u64 V = shoup_lz<SF>(x[k + half], w.x, w.y, q);
                x[k] = U + V;
                x[k + half] = U - V + q2;
            }
        }
#pragma unroll
        for (int k = 0; k < (1 << R); k++) s[pad(base + (k << lt))] = x[k];
    }
}

template <int R, bool TW_SMEM = false, bool SF = false>
__device__ __forceinline__ void inv_pass(u64* s, const ulonglong2* __restrict__ tw, u64 q, int logN, int s0)
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
        for (int l = R - 1; l >= 0; l--) {
            const int m = 1 << (s0 + l);
            const int half = 1 << (R - 1 - l);
#pragma unroll
            for (int k = 0; k < (1 << R); k++) {
                if (k & half) continue;
                const ulonglong2 w = tw_load<TW_SMEM>(&tw[m + (blk << l) + (k >> (R - l))]);
                u64 U = x[k], V = x[k + half];
                u64 a = U + V;
                x[k] = a >= q2 ? a - q2 : a;
                x[k + half] = shoup_lz<SF>(U - V + q2, w.x, w.y, q);
            }
        }
#pragma unroll
        for (int k = 0; k < (1 << R); k++) s[pad(base + (k << lt))] = x[k];
    }
}

#define GALA_NTT_R 3

template <int RMAX, bool TW_SMEM>
__device__ __forceinline__ void fwd_dispatch(u64* s, const ulonglong2* tw, u64 q, int logN, int s0, int r)
{
    if (RMAX >= 5 && r == 5) fwd_pass<(RMAX >= 5 ? 5 : 1), TW_SMEM>(s, tw, q, logN, s0);
    else if (RMAX >= 4 && r == 4) fwd_pass<(RMAX >= 4 ? 4 : 1), TW_SMEM>(s, tw, q, logN, s0);
    else if (r == 3) fwd_pass<3, TW_SMEM>(s, tw, q, logN, s0);
    else if (r == 2) fwd_pass<2, TW_SMEM>(s, tw, q, logN, s0);
    else fwd_pass<1, TW_SMEM>(s, tw, q, logN, s0);
}
template <int RMAX, bool TW_SMEM>
__device__ __forceinline__ void inv_dispatch(u64* s, const ulonglong2* tw, u64 q, int logN, int s0, int r)
{
    if (RMAX >= 5 && r == 5) inv_pass<(RMAX >= 5 ? 5 : 1), TW_SMEM>(s, tw, q, logN, s0);
    else if (RMAX >= 4 && r == 4) inv_pass<(RMAX >= 4 ? 4 : 1), TW_SMEM>(s, tw, q, logN, s0);
    else if (r == 3) inv_pass<3, TW_SMEM>(s, tw, q, logN, s0);
    else if (r == 2) inv_pass<2, TW_SMEM>(s, tw, q, logN, s0);
    else inv_pass<1, TW_SMEM>(s, tw, q, logN, s0);
}

// input: s[pad(i)] in [0, 4q); output in [0, 4q) (bit-reversed order)
template <bool TW_SMEM = false, int RMAX = GALA_NTT_R>
__device__ __forceinline__ void ntt_fwd_smem(u64* s, const ulonglong2* tw, u64 q, int logN)
{
    int s0 = 0;
    while (s0 < logN) {
        int r = logN - s0 < RMAX ? logN - s0 : RMAX;
        fwd_dispatch<RMAX, TW_SMEM>(s, tw, q, logN, s0, r);
        __syncthreads();
        s0 += r;
    }
}

// input: s[pad(i)] in [0, 2q) bit-reversed; output in [0, 2q) natural, *not* scaled by N^-1
template <bool TW_SMEM = false, int RMAX = GALA_NTT_R>
__device__ __forceinline__ void ntt_inv_smem(u64* s, const ulonglong2* tw, u64 q, int logN)
{
    // passes mirror the forward split, executed from the last stage group down
    int first = logN % RMAX;
    int s0 = logN - (first ? first : RMAX);
    while (s0 >= 0) {
        int r = logN - s0 < RMAX ? logN - s0 : RMAX;
        inv_dispatch<RMAX, TW_SMEM>(s, tw, q, logN, s0, r);
        __syncthreads();
        s0 -= RMAX;
    }
}

// 512 threads for N = 8192 (two radix-8 groups per thread per pass) so that two
// CTAs (2 x 66 KB smem, <= 64 registers) share an SM and overlap their memory phases
// ---------------------------------------------------------------------------
// Production NTT plans (radix-8 passes, the odd remainder pass at the global
// edge): forward = [first pass fed straight from global memory through a loader
// functor] + radix-8 smem passes; inverse = radix-8 smem passes + [last pass
// written straight to global memory through a storer functor].  For log N = 13
// the split is 1,3,3,3,3 (forward) and 3,3,3,3,1 (inverse).
__host__ __device__ constexpr int edge_r(int logN) { return logN % 3 == 0 ? 3 : logN % 3; }

template <int R, bool SF, class Loader>
__device__ __forceinline__ void fwd_first_pass(Loader ld, u64* s, const ulonglong2* __restrict__ tw, u64 q, int logN)
{
    const int N = 1 << logN;
    const int G = N >> R;
    const int lt = logN - R;
    const u64 q2 = 2 * q;
    for (int g = threadIdx.x; g < G; g += blockDim.x) {
        u64 x[1 << R];
#pragma unroll
        for (int k = 0; k < (1 << R); k++) x[k] = ld(g + (k << lt));
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
                u64 V = shoup_lz<SF>(x[k + half], w.x, w.y, q);
                x[k] = U + V;
                x[k + half] = U - V + q2;
            }
        }
#pragma unroll
        for (int k = 0; k < (1 << R); k++) s[pad(g + (k << lt))] = x[k];
    }
}

template <int R, bool SF, class Storer>
__device__ __forceinline__ void inv_last_pass(const u64* s, const ulonglong2* __restrict__ tw, u64 q, int logN, Storer st)
{
    const int N = 1 << logN;
    const int G = N >> R;
    const int lt = logN - R;
    const u64 q2 = 2 * q;
    for (int g = threadIdx.x; g < G; g += blockDim.x) {
        u64 x[1 << R];
#pragma unroll
        for (int k = 0; k < (1 << R); k++) x[k] = s[pad(g + (k << lt))];
#pragma unroll
        for (int l = R - 1; l >= 0; l--) {
            const int m = 1 << l;
            const int half = 1 << (R - 1 - l);
#pragma unroll
            for (int k = 0; k < (1 << R); k++) {
                if (k & half) continue;
                const ulonglong2 w = __ldg(&tw[m + (k >> (R - l))]);
                u64 U = x[k], V = x[k + half];
                u64 a = U + V;
                x[k] = a >= q2 ? a - q2 : a;
                x[k + half] = shoup_lz<SF>(U - V + q2, w.x, w.y, q);
            }
        }
#pragma unroll
        for (int k = 0; k < (1 << R); k++) st(g + (k << lt), x[k]);
    }
}

// forward: ld(i) -> natural-order input in [0, 4q); result in s (bit-reversed, [0, 4q)); ends synced
template <bool SF = true, class Loader>
__device__ __forceinline__ void ntt_fwd_g(Loader ld, u64* s, const ulonglong2* tw, u64 q, int logN)
{
    const int r0 = edge_r(logN);
    if (r0 == 1) fwd_first_pass<1, SF>(ld, s, tw, q, logN);
    else if (r0 == 2) fwd_first_pass<2, SF>(ld, s, tw, q, logN);
    else fwd_first_pass<3, SF>(ld, s, tw, q, logN);
    __syncthreads();
    for (int s0 = r0; s0 < logN; s0 += 3) {
        fwd_pass<3, false, SF>(s, tw, q, logN, s0);
        __syncthreads();
    }
}

// inverse: s holds bit-reversed input in [0, 2q) (synced); st(i, v) receives the natural-order
// output v in [0, 2q) *before* the N^-1 scaling
template <bool SF = true, class Storer>
__device__ __forceinline__ void ntt_inv_g(u64* s, const ulonglong2* tw, u64 q, int logN, Storer st)
{
    const int rl = edge_r(logN);
    for (int s0 = logN - 3; s0 >= rl; s0 -= 3) {
        inv_pass<3, false, SF>(s, tw, q, logN, s0);
        __syncthreads();
    }
    if (rl == 1) inv_last_pass<1, SF>(s, tw, q, logN, st);
    else if (rl == 2) inv_last_pass<2, SF>(s, tw, q, logN, st);
    else inv_last_pass<3, SF>(s, tw, q, logN, st);
}

__host__ __device__ inline int ntt_threads(int N)
{
    int t = N >> (GALA_NTT_R + 1);
    return t < 32 ? 32 : t;
}
