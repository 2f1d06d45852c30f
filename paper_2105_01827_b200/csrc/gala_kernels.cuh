// gala_kernels.cuh -- sm_100a kernels of the GALA HE linear-layer path.
//
// Ciphertexts: u64 [2][L][N] (bit-reversed NTT domain); digits: u64 [L][M][N];
// keys: u64 [L][2][M][N] Montgomery form; plaintext operands: u64 [L][N]
// NTT + Montgomery form.  One CTA per polynomial for every transform (the
// polynomial lives in shared memory for all log N stages); elementwise and
// key-switch kernels are one thread per coefficient.
#pragma once
#include "gala_device.cuh"

// ---------------------------------------------------------------------------
// addressing of a batch of polynomials (one CTA each)
struct PolyMap {
    int per;          // polynomials per item
    int nprimes;      // prime index = prime_base + (w % nprimes)
    int prime_base;
    int src_div;      // source poly within item: w / nprimes (1) or w (0)
    long long src_is; // item strides (words)
    long long dst_is;
    int skip_per;     // >0: item index x -> (x/cnt)*skip_per + first + x%cnt
    int skip_first;   // (first, cnt) = (1, skip_per - 1) when skip_cnt == 0
    int skip_cnt;
    int quad_G;       // > 0: the source is the key-folded group-sum layout (u_quad_base), source item b G + g,
    int quad_cc;      //      polynomial (quad_cc, quad_j) of it; element i at u_quad_off(i)
    int quad_j;
};

// The key-folded FC group sums (k_gala_kf): per 256-input tile, [g][cc][j][N / 4][256 rows][4] -- four
// consecutive positions of one input are one 32-byte sector and the 256 inputs' sectors are contiguous,
// so the epilogue's 32-byte stores from 32 lanes (inputs) are one 1 KB run, and a polynomial read (32
// consecutive positions) still touches 8 full sectors.
__device__ __forceinline__ long long u_quad_base(int b, int g, int cc, int j, int G, int M, int N)
{
    return (((((long long)(b >> 8) * G + g) * 2 + cc) * M + j) * N) * 256 + (long long)(b & 255) * 4;
}
__device__ __forceinline__ long long u_quad_off(int i) { return ((long long)(i >> 2) << 10) + (i & 3); }

__device__ __forceinline__ void polymap_resolve(const PolyMap& pm, int p, int N, long long& src_off,
                                                long long& dst_off, int& prime)
{
    int item = p / pm.per, w = p - item * pm.per;
    long long src_item = item;
    if (pm.skip_per > 0) {
        const int sp = pm.skip_cnt > 0 ? pm.skip_cnt : pm.skip_per - 1, f = pm.skip_cnt > 0 ? pm.skip_first : 1;
        src_item = (long long)(item / sp) * pm.skip_per + f + item % sp;
    }
    prime = pm.prime_base + w % pm.nprimes;
    src_off = src_item * pm.src_is + (long long)(pm.src_div ? w / pm.nprimes : w) * N;
    dst_off = (long long)item * pm.dst_is + (long long)w * N;
}
__device__ __forceinline__ long long polymap_quad_base(const PolyMap& pm, int p, int M, int N)
{
    int item = p / pm.per;
    long long src_item = item;
    if (pm.skip_per > 0) {
        const int sp = pm.skip_cnt > 0 ? pm.skip_cnt : pm.skip_per - 1, f = pm.skip_cnt > 0 ? pm.skip_first : 1;
        src_item = (long long)(item / sp) * pm.skip_per + f + item % sp;
    }
    return u_quad_base((int)(src_item / pm.quad_G), (int)(src_item % pm.quad_G), pm.quad_cc, pm.quad_j, pm.quad_G, M, N);
}

template <typename T>
__device__ __forceinline__ u64 to_residue(T v, u64 q);
template <>
__device__ __forceinline__ u64 to_residue<u64>(u64 v, u64 q) { return v; } // caller guarantees < 4q
template <>
__device__ __forceinline__ u64 to_residue<i64>(i64 v, u64 q)
{
    if (v >= 0) return (u64)v % q;
    u64 r = ((u64)(-v)) % q;
    return r ? q - r : 0;
}
template <>
__device__ __forceinline__ u64 to_residue<int8_t>(int8_t v, u64 q) { return v >= 0 ? (u64)v : q - (u64)(-v); }

// forward NTT of a batch; output reduced to [0, q), optionally Montgomery-scaled
template <typename T, bool TO_MONT>
__global__ void __launch_bounds__(512, 2) k_ntt_fwd(DevCtx c, const T* __restrict__ src, u64* __restrict__ dst, PolyMap pm)
{
    extern __shared__ u64 sm[];
    long long so, dof;
    int j;
    polymap_resolve(pm, blockIdx.x, c.N, so, dof, j);
    const ModC md = c.mod[j];
    const u64 q = md.q;
    const T* sp = src + so;
    ntt_fwd_g([=](int i) { return to_residue<T>(sp[i], q); }, sm, c.twf[j], q, c.logN);
    for (int i = threadIdx.x; i < c.N; i += blockDim.x) {
        u64 v = sm[pad(i)];
        v = csub(csub(v, 2 * q), q);
        if (TO_MONT) v = mont_mul(v, md.r2, md);
        st_cs(dst + dof + i, v);
    }
}

// inverse NTT of a batch -> coefficients in [0, q)
template <bool FROM_MONT>
__global__ void __launch_bounds__(512, 2) k_ntt_inv(DevCtx c, const u64* __restrict__ src, u64* __restrict__ dst, PolyMap pm)
{
    extern __shared__ u64 sm[];
    long long so, dof;
    int j;
    polymap_resolve(pm, blockIdx.x, c.N, so, dof, j);
    const ModC md = c.mod[j];
    const u64 q = md.q;
    const long long qb = pm.quad_G > 0 ? polymap_quad_base(pm, blockIdx.x, c.M, c.N) : 0;
    for (int i = threadIdx.x; i < c.N; i += blockDim.x) {
        u64 v = pm.quad_G > 0 ? ld_cs(src + qb + u_quad_off(i)) : ld_cs(src + so + i);
        if (FROM_MONT) v = csub(redc_lazy(0, v, md), q);
        sm[pad(i)] = v;
    }
    __syncthreads();
    const u64 ni = c.ninv[j], nsh = c.ninv_sh[j];
    u64* dp = dst + dof;
    ntt_inv_g(sm, c.twi[j], q, c.logN, [=](int i, u64 v) { st_cs(dp + i, shoup(v, ni, nsh, q)); });
}

// ---------------------------------------------------------------------------
// ModDown epilogue: items g, w in [0, 2L): comp = w / L, prime j = w % L.
//   out[g][comp][j] = (U[g][comp][j] - NTT_j(centred r[g][comp])) * P^-1 + add_comp[g][j]
struct MdArgs {
    const u64* r;      // [G][2][N] coefficients mod P
    const u64* U;      // [G][2][M][N]
    const u64* add0;   // [G] stride add_is, c0 addend [L][N] (may be null)
    const u64* add1;   // c1 addend
    long long add_is;
    u64* out;          // [G] stride out_is, [2][L][N]   (used when outs == null)
    long long out_is;
    u64* const* outs;  // optional per-group output pointers
    int comps;         // components per item (0 = 2); 1: only component comp0
    int comp0;
    int skip_per;      // > 0: item x reads source item (x / cnt) skip_per + first + x % cnt
    int skip_first;    // (first, cnt) = (1, skip_per - 1) when skip_cnt == 0
    int skip_cnt;
    int quad_G;        // > 0: U in the key-folded group-sum layout (u_quad_base), source item g = b quad_G + group
};

__global__ void __launch_bounds__(512, 2) k_moddown(DevCtx c, MdArgs a)
{
    extern __shared__ u64 sm[];
    const int L = c.L, M = c.M, N = c.N;
    const int comps = a.comps ? a.comps : 2;
    const int x = blockIdx.x / (comps * L), w = blockIdx.x % (comps * L);
    const int comp = a.comp0 + w / L, j = w % L;
    const int scnt = a.skip_cnt > 0 ? a.skip_cnt : a.skip_per - 1, sfirst = a.skip_cnt > 0 ? a.skip_first : 1;
    const long long g = a.skip_per > 0 ? (long long)(x / scnt) * a.skip_per + sfirst + x % scnt : x;
    const ModC md = c.mod[j];
    const u64 q = md.q, P = c.mod[L].q, halfP = P >> 1;
    const u64* r = a.r + ((long long)x * comps + (comp - a.comp0)) * N;
    // centred lift of v in [0, P) into [0, 2q): |v - P| < P/2 < q_j (asserted at context creation)
    ntt_fwd_g([=](int i) {
        const u64 v = r[i];
        return v > halfP ? q - (P - v) : v;
    }, sm, c.twf[j], q, c.logN);
    const u64* U = a.U + (((long long)g * 2 + comp) * M + j) * N;
    const long long qb = a.quad_G > 0 ? u_quad_base((int)(g / a.quad_G), (int)(g % a.quad_G), comp, j, a.quad_G, M, N) : 0;
    const u64* add = comp == 0 ? a.add0 : a.add1;
    if (add) add += (long long)g * a.add_is + (long long)j * N;
    u64* out = (a.outs ? a.outs[x] : a.out + (long long)x * a.out_is) + ((long long)comp * L + j) * N;
    const u64 pinv = c.pinv_mont[j];
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        u64 R = csub(csub(sm[pad(i)], 2 * q), q);
        u64 v = mont_mul(sub_mod(a.quad_G > 0 ? a.U[qb + u_quad_off(i)] : U[i], R, q), pinv, md);
        if (add) v = add_mod(v, add[i], q);
        out[i] = v;
    }
}

// ModDown + mask in the coefficient domain, for results that leave as canonical (coefficient) words
// (gala_mv_gala2_stream_host): Uc = INTT of every limb of the QP sums [G][2][M][N], m = the masks'
// coefficients mod p [G][N] (k_encode_p), out [G][2][L][N]:
//   out[g][comp][j] = (Uc[g][comp][j] - centred Uc[g][comp][P]) * P^-1 - (comp == 0) Delta_j m[g]   (mod q_j)
// The NTT is linear mod q_j, so these are the words of k_moddown + k_sub_plain + the export INTT with
// 9 fewer NTT-sized transforms per result (no NTT of the lifted P limb or of the mask, no export INTT).
__global__ void k_moddown_coef(DevCtx c, const u64* __restrict__ Uc, const uint32_t* __restrict__ m,
                               u64* __restrict__ out, int G)
{
    const int L = c.L, M = c.M, N = c.N;
    const long long total = (long long)G * 2 * N;
    const u64 P = c.mod[L].q, halfP = P >> 1;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total;
         x += (long long)gridDim.x * blockDim.x) {
        const long long gc = x >> c.logN;      // g * 2 + comp
        const int k = (int)(x & (N - 1));
        const u64* u = Uc + gc * M * N + k;
        const u64 v = ld_cs(u + (long long)L * N);
        const uint32_t mk = (gc & 1) == 0 && m ? __ldg(m + (gc >> 1) * N + k) : 0u;
        for (int j = 0; j < L; j++) {
            const ModC md = c.mod[j];
            const u64 q = md.q;
            const u64 R = v > halfP ? q - (P - v) : v;
            u64 w = mont_mul(sub_mod(ld_cs(u + (long long)j * N), R, q), c.pinv_mont[j], md);
            if ((gc & 1) == 0 && m) w = sub_mod(w, shoup((u64)mk, c.delta[j], c.delta_sh[j], q), q);
            st_cs(out + (gc * L + j) * N + k, w);
        }
    }
}

// ---------------------------------------------------------------------------
// Key-switch engine v2.  A "term" is a source ciphertext X, optionally times a
// plaintext operand pt (so ScMult fuses into the key switch), to be rotated by
// one or more Galois elements.
//   k_digits_intt : digits d_i = INTT_i((X (.) pt).c1[i])            [term][L][N]
//   k_digits_perm : for every rotation r of the term, the block
//                   [ sigma_r(NTT_j(d_i)) for i<L, j<M ;  sigma_r(c0_j) for j<L ]
//                   (NTT only for j != i; the j == i limb is the NTT-domain c1)
//   k_ks_mac      : per group, sum over its rotated blocks of
//                   sum_i D'[i][j] * key[i][c][j]  (128-bit lazy) and the c0 sums;
//                   step-0 members add (X (.) pt) directly.
struct TermDesc {
    const u64* X;      // [2][L][N] NTT
    const u64* pt;     // [L][N] Montgomery or null
    u64* dig;          // [L][N] digit coefficients (scratch)
    u64* blk;          // first permuted block [(L*M + L)][N]; rotation r at blk + r * blk_words
    int rot_off, rot_cnt;
    int c0_zero;       // the term's c0 is zero: no sigma-copies of it (its block slots are not read)
};

__device__ __forceinline__ u64 src_limb(const DevCtx& c, const TermDesc& t, int comp, int j, int k)
{
    const long long o = ((long long)comp * c.L + j) * c.N + k;
    u64 v = __ldg(t.X + o);
    if (t.pt) v = mont_mul(v, __ldg(t.pt + (long long)j * c.N + k), c.mod[j]);
    return v;
}

// sigma-permuted copies of the NTT-domain polynomial held in smem into block slot `slot`
// of every rotation of the term
__device__ __forceinline__ void write_perm(const DevCtx& c, const u64* sm, const TermDesc& t,
                                           const unsigned* __restrict__ galois, long long blk_words, int slot)
{
    for (int r = 0; r < t.rot_cnt; r++) {
        const unsigned g = galois[t.rot_off + r];
        u64* o = t.blk + r * blk_words + (long long)slot * c.N;
        for (int k = threadIdx.x; k < c.N; k += blockDim.x) st_cs(o + k, sm[pad(auto_src(k, g, c.logN))]);
    }
}

// grid: terms * L CTAs.  Per (term, prime i): the sigma-copies of c0_i and of the c1_i limb
// (the j == i digit needs no NTT), then INTT of c1_i -> digit coefficients.  (X (.) pt) is formed
// here once (ScMult fused).
__global__ void __launch_bounds__(512, 2) k_digits_intt(DevCtx c, const TermDesc* __restrict__ terms,
                                                        const unsigned* __restrict__ galois, long long blk_words)
{
    extern __shared__ u64 sm[];
    const int L = c.L, M = c.M, N = c.N;
    const int ti = blockIdx.x / L, i = blockIdx.x % L;
    const TermDesc t = terms[ti];
    const u64 q = c.mod[i].q;
    if (t.blk && !t.c0_zero) {
        for (int k = threadIdx.x; k < N; k += blockDim.x) sm[pad(k)] = src_limb(c, t, 0, i, k);
        __syncthreads();
        write_perm(c, sm, t, galois, blk_words, L * M + i);
        __syncthreads();
    }
    for (int k = threadIdx.x; k < N; k += blockDim.x) sm[pad(k)] = src_limb(c, t, 1, i, k);
    __syncthreads();
    if (t.blk) {
        write_perm(c, sm, t, galois, blk_words, i * M + i);
        __syncthreads();
    }
    u64* d = t.dig + (long long)i * N;
    const u64 ni = c.ninv[i], nsh = c.ninv_sh[i];
    ntt_inv_g(sm, c.twi[i], q, c.logN, [=](int k, u64 v) { st_cs(d + k, shoup(v, ni, nsh, q)); });
}

// grid: terms * L * L CTAs: NTT of digit i into every prime j != i, then the sigma-permuted writes
__global__ void __launch_bounds__(512, 2) k_digits_perm(DevCtx c, const TermDesc* __restrict__ terms,
                                                         const unsigned* __restrict__ galois, long long blk_words)
{
    extern __shared__ u64 sm[];
    const int L = c.L, M = c.M, N = c.N;
    const int per = L * L;
    const int ti = blockIdx.x / per, s = blockIdx.x % per;
    const int i = s / L, jj = s % L, j = jj < i ? jj : jj + 1;
    const TermDesc t = terms[ti];
    const u64 q = c.mod[j].q;
    const u64* d = t.dig + (long long)i * N;   // d < q_i < 4 q_j: lazy NTT input
    ntt_fwd_g([=](int k) { return ld_cs(d + k); }, sm, c.twf[j], q, c.logN);
    const int slot = i * M + j;               // NTT outputs are in [0, 4q): fold on the permuted read
    for (int r = 0; r < t.rot_cnt; r++) {
        const unsigned g = galois[t.rot_off + r];
        u64* o = t.blk + r * blk_words + (long long)slot * N;
        for (int k = threadIdx.x; k < N; k += blockDim.x)
            st_cs(o + k, csub(csub(sm[pad(auto_src(k, g, c.logN))], 2 * q), q));
    }
}

// hoisted rotations from a precomputed identity block (the DecPerm output):
// permutation only.  t.X points at the identity block [(L*M + L)][N].
__global__ void __launch_bounds__(512, 2) k_block_perm(DevCtx c, const TermDesc* __restrict__ terms,
                                                        const unsigned* __restrict__ galois, long long blk_words)
{
    extern __shared__ u64 sm[];
    const int L = c.L, M = c.M, N = c.N;
    const int per = L * M + L;
    const int ti = blockIdx.x / per, slot = blockIdx.x % per;
    const TermDesc t = terms[ti];
    const u64* src = t.X + (long long)slot * N;
    for (int k = threadIdx.x; k < N; k += blockDim.x) sm[pad(k)] = ld_cs(src + k);
    __syncthreads();
    for (int r = 0; r < t.rot_cnt; r++) {
        const unsigned g = galois[t.rot_off + r];
        u64* o = t.blk + r * blk_words + (long long)slot * N;
        for (int k = threadIdx.x; k < N; k += blockDim.x) st_cs(o + k, sm[pad(auto_src(k, g, c.logN))]);
    }
}

struct MacMember {
    const u64* blk;    // permuted block (rotated member) or null (step-0 member)
    const u64* key;    // [L][2][M][N]
    const u64* X;      // step-0 member source
    const u64* pt;
    int no_c0;         // rotated member whose c0 is zero (block c0 slots not written)
    unsigned gal;      // > 1: blk is the term's identity block and the member's sigma is applied as a gather
};

// grid (N / blockDim, M, G); U [G][2][M][N]; Cacc [G][2][L][N].
// Step-0 members come first in every group (host guarantees the order); the
// rotated members follow.  Digit/key products accumulate in 128 bits across
// digits *and* members and are Montgomery-reduced only every c.lazy[j]
// products (k q^2 < q 2^64).  The next member's loads are issued before the
// current member's multiplies (software pipelining over the member loop).  GATHER: some members read
// their digits through a sigma gather from an identity block (MacMember.gal > 1; a separate
// instantiation so the permuted-block form keeps its registers).
template <int L, bool GATHER = false>
__global__ void __launch_bounds__(256) k_ks_mac(DevCtx c, const MacMember* __restrict__ mem,
                                                const int* __restrict__ group_off, u64* __restrict__ U,
                                                u64* __restrict__ Cacc, const u64* __restrict__ qp_add,
                                                const u64* __restrict__ q_add)
{
    const int N = c.N, M = L + 1;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y, g = blockIdx.z;
    if (k >= N) return;
    const ModC md = c.mod[j];
    const u64 q = md.q;
    const int lazy = c.lazy[j];
    const long long NN = N;
    // optional addends: QP [G][2][M][N] into U (before the ModDown), Q [G][2][L][N] into the c0/c1 sums
    u64 u0 = 0, u1 = 0, a0 = 0, a1 = 0;
    if (qp_add) {
        u0 = qp_add[(((long long)g * 2 + 0) * M + j) * NN + k];
        u1 = qp_add[(((long long)g * 2 + 1) * M + j) * NN + k];
    }
    if (q_add && j < L) {
        a0 = q_add[(((long long)g * 2 + 0) * L + j) * NN + k];
        a1 = q_add[(((long long)g * 2 + 1) * L + j) * NN + k];
    }
    int it = group_off[g];
    const int hi = group_off[g + 1];
    for (; it < hi; it++) {                       // step-0 members
        const MacMember m = mem[it];
        if (m.blk) break;
        if (j < L) {
            u64 x0 = m.X[(long long)j * NN + k], x1 = m.X[((long long)L + j) * NN + k];
            if (m.pt) {
                const u64 w = __ldg(&m.pt[(long long)j * NN + k]);
                x0 = mont_mul(x0, w, md);
                x1 = mont_mul(x1, w, md);
            }
            a0 = add_mod(a0, x0, q);
            a1 = add_mod(a1, x1, q);
        }
    }
    AccPP<> s0, s1;
    s0.clear();
    s1.clear();
    int pending = 0;
    constexpr int LMAX = L;
    u64 dv[LMAX], kb[LMAX], ka[LMAX], cv = 0;
    auto fetch = [&](const MacMember& m) {
        if (GATHER && m.gal > 1u) {   // hoisted rotation: gather sigma(D) from the term's identity block (in L2)
            const int src = auto_src(k, m.gal, c.logN);
#pragma unroll
            for (int i = 0; i < LMAX; i++) {
                if (i < L) {
                    dv[i] = __ldg(m.blk + ((long long)i * M + j) * NN + src);
                    kb[i] = __ldg(&m.key[(((long long)i * 2 + 0) * M + j) * NN + k]);
                    ka[i] = __ldg(&m.key[(((long long)i * 2 + 1) * M + j) * NN + k]);
                }
            }
            cv = (j < L && !m.no_c0) ? __ldg(m.blk + ((long long)L * M + j) * NN + src) : 0ull;
            return;
        }
#pragma unroll
        for (int i = 0; i < LMAX; i++) {
            if (i < L) {
                dv[i] = __ldcs((const unsigned long long*)(m.blk + ((long long)i * M + j) * NN + k));
                kb[i] = __ldg(&m.key[(((long long)i * 2 + 0) * M + j) * NN + k]);
                ka[i] = __ldg(&m.key[(((long long)i * 2 + 1) * M + j) * NN + k]);
            }
        }
        cv = (j < L && !m.no_c0) ? __ldcs((const unsigned long long*)(m.blk + ((long long)L * M + j) * NN + k)) : 0ull;
    };
    if (it < hi) fetch(mem[it]);
    for (; it < hi; it++) {
        u64 d[LMAX], b[LMAX], a[LMAX], cc = cv;
#pragma unroll
        for (int i = 0; i < LMAX; i++) { d[i] = dv[i]; b[i] = kb[i]; a[i] = ka[i]; }
        if (it + 1 < hi) fetch(mem[it + 1]);      // prefetch the next member
        if (pending + L > lazy) {
            u0 = add_mod(u0, s0.reduce_sf(q), q);
            u1 = add_mod(u1, s1.reduce_sf(q), q);
            s0.clear();
            s1.clear();
            pending = 0;
        }
#pragma unroll
        for (int i = 0; i < LMAX; i++) {
            if (i < L) {
                s0.mac(d[i], b[i]);
                s1.mac(d[i], a[i]);
            }
        }
        pending += L;
        if (j < L) a0 = add_mod(a0, cc, q);
    }
    u0 = add_mod(u0, s0.reduce_sf(q), q);
    u1 = add_mod(u1, s1.reduce_sf(q), q);
    U[(((long long)g * 2 + 0) * M + j) * NN + k] = u0;
    U[(((long long)g * 2 + 1) * M + j) * NN + k] = u1;
    if (j < L) {
        Cacc[(((long long)g * 2 + 0) * L + j) * NN + k] = a0;
        Cacc[(((long long)g * 2 + 1) * L + j) * NN + k] = a1;
    }
}

// ---------------------------------------------------------------------------
// Fused key switch for terms rotated by ONE Galois element (FC giant steps, schedule-1 products,
// the conv second-Perm): per (term, prime j of QP) one CTA takes the term's digit coefficients
// d_i (k_digits_intt) to prime j -- NTT_j(d_i) for i != j, the NTT-domain limb (X (.) pt).c1[j]
// itself for i == j -- into L shared-memory buffers, then forms the key inner product straight
// from shared memory through the automorphism:
//   part[t][c][j][k]  = sum_i NTT_j(d_i)[sigma(k)] ksk[i][c][j][k]      (AccPP, one REDC)
//   cpart[t][j][k]    = (X (.) pt).c0[j][sigma(k)]                       (j < L)
// No sigma-permuted digit block goes through HBM (k_digits_perm + k_ks_mac write and re-read one of
// (L M + L) N words per rotation).  k_ks_sum folds the parts of each group.
struct FusedTerm {
    const u64* X;      // [2][L][N] NTT
    const u64* pt;     // [L][N] Montgomery or null
    const u64* dig;    // [L][N] digit coefficients
    const u64* key;    // [L][2][M][N] key of the term's rotation
    unsigned gal;
    int c0_zero;
};

// Uniform hoisted rotations (every term rotated by the same R steps, one member per group, groups
// term-major): U[(b R + r)] = sum_i sigma_r(D_i^b) ksk_r[i] and Cacc[(b R + r)].c0 = sigma_r(x_b.c0) --
// what k_ks_mac<L, true> computes for these groups, word for word, with the loops turned around: a
// thread (position k, prime j) takes tb terms (up to 8; fewer when the grid would not fill the GPU) for
// every step r, so step r's key words and sigma_r source index are loaded once and reused tb times, and
// the tb identity blocks stay hot in L1/L2 across the R steps.  grid (N / 256, M, ceil(terms / tb)).
template <int L>
__global__ void __launch_bounds__(256) k_ks_hoist(DevCtx c, const u64* const* __restrict__ blocks,
                                                  const unsigned* __restrict__ gal, const u64* const* __restrict__ keys,
                                                  int R, int nterms, int tb, int no_c0, u64* __restrict__ U,
                                                  u64* __restrict__ Cacc)
{
    const int N = c.N, M = L + 1;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y, b0 = blockIdx.z * tb;
    if (k >= N) return;
    const u64 q = c.mod[j].q;
    const long long NN = N;
    const int nb = nterms - b0 < tb ? nterms - b0 : tb;
    for (int r = 0; r < R; r++) {
        const int src = auto_src(k, gal[r], c.logN);
        const u64* key = keys[r];
        u64 kb[L], ka[L];
#pragma unroll
        for (int i = 0; i < L; i++) {
            kb[i] = __ldg(&key[(((long long)i * 2 + 0) * M + j) * NN + k]);
            ka[i] = __ldg(&key[(((long long)i * 2 + 1) * M + j) * NN + k]);
        }
        for (int bi = 0; bi < nb; bi++) {
            const u64* blk = blocks[b0 + bi];
            u64 dv[L];
#pragma unroll
            for (int i = 0; i < L; i++) dv[i] = __ldg(blk + ((long long)i * M + j) * NN + src);
            const u64 cv = (j < L && !no_c0) ? __ldg(blk + ((long long)L * M + j) * NN + src) : 0ull;
            AccPP<> s0, s1;
            s0.clear();
            s1.clear();
#pragma unroll
            for (int i = 0; i < L; i++) {
                s0.mac(dv[i], kb[i]);
                s1.mac(dv[i], ka[i]);
            }
            const long long g = (long long)(b0 + bi) * R + r;
            U[((g * 2 + 0) * M + j) * NN + k] = add_mod(0, s0.reduce_sf(q), q);
            U[((g * 2 + 1) * M + j) * NN + k] = add_mod(0, s1.reduce_sf(q), q);
            if (j < L) {
                Cacc[((g * 2 + 0) * L + j) * NN + k] = add_mod(0, cv, q);
                Cacc[((g * 2 + 1) * L + j) * NN + k] = 0;
            }
        }
    }
}

// Giant-step key switches of a batch (FC schedule 2): every group (input) b sums the same R rotated terms
// b R + r, term r of every group rotated by the same step (key r), each term's sigma-permuted digit block
// written by k_digits_perm, plus the optional QP / Q addends -- what k_ks_mac<L, false> computes for
// these groups, with each thread (position k, prime j) taking KG_IB groups so that every key word is
// loaded once per KG_IB inputs.  grid (N / 256, M, ceil(G / KG_IB)).
#define KG_IB 2
template <int L>
__global__ void __launch_bounds__(256) k_ks_giant(DevCtx c, const u64* const* __restrict__ blocks,
                                                  const u64* const* __restrict__ keys, int R, int G, int no_c0,
                                                  u64* __restrict__ U, u64* __restrict__ Cacc,
                                                  const u64* __restrict__ qp_add, const u64* __restrict__ q_add)
{
    const int N = c.N, M = L + 1;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y, g0 = blockIdx.z * KG_IB;
    if (k >= N) return;
    const ModC md = c.mod[j];
    const u64 q = md.q;
    const int lazy = c.lazy[j];
    const long long NN = N;
    const int ng = G - g0 < KG_IB ? G - g0 : KG_IB;
    u64 u0[KG_IB], u1[KG_IB], a0[KG_IB], a1[KG_IB];
    AccPP<> s0[KG_IB], s1[KG_IB];
#pragma unroll
    for (int i = 0; i < KG_IB; i++) {
        const long long g = g0 + (i < ng ? i : 0);
        u0[i] = qp_add ? qp_add[((g * 2 + 0) * M + j) * NN + k] : 0;
        u1[i] = qp_add ? qp_add[((g * 2 + 1) * M + j) * NN + k] : 0;
        a0[i] = (q_add && j < L) ? q_add[((g * 2 + 0) * L + j) * NN + k] : 0;
        a1[i] = (q_add && j < L) ? q_add[((g * 2 + 1) * L + j) * NN + k] : 0;
        s0[i].clear();
        s1[i].clear();
    }
    int pending = 0;
    // software pipeline: step r + 1's key words and digits are in flight while step r multiplies
    u64 kb[L], ka[L], dv[KG_IB][L], cv[KG_IB];
    auto fetch = [&](int r) {
        const u64* key = keys[r];
#pragma unroll
        for (int l = 0; l < L; l++) {
            kb[l] = __ldg(&key[(((long long)l * 2 + 0) * M + j) * NN + k]);
            ka[l] = __ldg(&key[(((long long)l * 2 + 1) * M + j) * NN + k]);
        }
#pragma unroll
        for (int i = 0; i < KG_IB; i++) {
            const u64* blk = blocks[(long long)(g0 + (i < ng ? i : 0)) * R + r];
#pragma unroll
            for (int l = 0; l < L; l++) dv[i][l] = __ldcs((const unsigned long long*)(blk + ((long long)l * M + j) * NN + k));
            cv[i] = (j < L && !no_c0) ? __ldcs((const unsigned long long*)(blk + ((long long)L * M + j) * NN + k)) : 0ull;
        }
    };
    fetch(0);
    for (int r = 0; r < R; r++) {
        u64 k0[L], k1[L], d[KG_IB][L], cc[KG_IB];
#pragma unroll
        for (int l = 0; l < L; l++) {
            k0[l] = kb[l];
            k1[l] = ka[l];
        }
#pragma unroll
        for (int i = 0; i < KG_IB; i++) {
            cc[i] = cv[i];
#pragma unroll
            for (int l = 0; l < L; l++) d[i][l] = dv[i][l];
        }
        if (r + 1 < R) fetch(r + 1);
        if (pending + L > lazy) {
#pragma unroll
            for (int i = 0; i < KG_IB; i++) {
                u0[i] = add_mod(u0[i], s0[i].reduce_sf(q), q);
                u1[i] = add_mod(u1[i], s1[i].reduce_sf(q), q);
                s0[i].clear();
                s1[i].clear();
            }
            pending = 0;
        }
#pragma unroll
        for (int i = 0; i < KG_IB; i++) {
#pragma unroll
            for (int l = 0; l < L; l++) {
                s0[i].mac(d[i][l], k0[l]);
                s1[i].mac(d[i][l], k1[l]);
            }
            if (j < L) a0[i] = add_mod(a0[i], cc[i], q);
        }
        pending += L;
    }
#pragma unroll
    for (int i = 0; i < KG_IB; i++) {
        if (i >= ng) break;
        const long long g = g0 + i;
        U[((g * 2 + 0) * M + j) * NN + k] = add_mod(u0[i], s0[i].reduce_sf(q), q);
        U[((g * 2 + 1) * M + j) * NN + k] = add_mod(u1[i], s1[i].reduce_sf(q), q);
        if (j < L) {
            Cacc[((g * 2 + 0) * L + j) * NN + k] = a0[i];
            Cacc[((g * 2 + 1) * L + j) * NN + k] = a1[i];
        }
    }
}

template <int L>
__global__ void __launch_bounds__(1024, 1) k_ks_fused(DevCtx c, const FusedTerm* __restrict__ terms,
                                                     u64* __restrict__ part, u64* __restrict__ cpart)
{
    extern __shared__ u64 sm[];
    constexpr int M = L + 1;
    const int N = c.N, logN = c.logN, PW = padded_words(N);
    const int ti = blockIdx.x / M, j = blockIdx.x % M;
    const FusedTerm t = terms[ti];
    const ModC md = c.mod[j];
    const u64 q = md.q;
#pragma unroll 1
    for (int i = 0; i < L; i++) {
        u64* b = sm + i * PW;
        if (i == j) {
            __syncthreads();
            for (int k = threadIdx.x; k < N; k += blockDim.x) {
                u64 v = __ldg(t.X + (long long)(L + j) * N + k);
                if (t.pt) v = mont_mul(v, __ldg(t.pt + (long long)j * N + k), md);
                b[pad(k)] = v;
            }
        } else {
            const u64* d = t.dig + (long long)i * N;   // d < q_i < 4 q_j: lazy NTT input
            ntt_fwd_g([=](int k) { return ld_cs(d + k); }, b, c.twf[j], q, logN);
        }
    }
    __syncthreads();
    const long long MN = (long long)M * N;
    u64* p0 = part + (long long)ti * 2 * MN + (long long)j * N;
    const u64* key = t.key + (long long)j * N;
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
        const int src = auto_src(k, t.gal, logN);
        AccPP<true> s0, s1;   // L <= 3 canonical products per sum
#pragma unroll
        for (int i = 0; i < L; i++) {
            u64 v = sm[i * PW + pad(src)];
            if (i != j) v = csub(csub(v, 2 * q), q);
            const u64 ka = __ldg(key + (2 * i) * MN + k), kb = __ldg(key + (2 * i + 1) * MN + k);
            if (i == 0) {
                s0.set(v, ka);
                s1.set(v, kb);
            } else {
                s0.mac(v, ka);
                s1.mac(v, kb);
            }
        }
        st_cs(p0 + k, s0.reduce_sf(q));
        st_cs(p0 + MN + k, s1.reduce_sf(q));
        if (j < L && !t.c0_zero) {
            u64 v = __ldg(t.X + (long long)j * N + src);
            if (t.pt) v = mont_mul(v, __ldg(t.pt + (long long)j * N + src), md);
            st_cs(cpart + ((long long)ti * L + j) * N + k, v);
        }
    }
}

struct SumMember {
    const u64* part;   // rotated member: [2][M][N] (null: step-0 member)
    const u64* cpart;  // [L][N] sigma-copied c0 (null: zero)
    const u64* X;      // step-0 member source
    const u64* pt;
};

// U[g] = qp_add[g] + sum of the group's parts; Cacc[g] = q_add[g] + step-0 members (X (.) pt) + the
// parts' sigma(c0).  grid (N / blockDim, M, G)
__global__ void __launch_bounds__(256) k_ks_sum(DevCtx c, const SumMember* __restrict__ mem, const int* __restrict__ off,
                                                u64* __restrict__ U, u64* __restrict__ Cacc,
                                                const u64* __restrict__ qp_add, const u64* __restrict__ q_add)
{
    const int N = c.N, L = c.L, M = c.M;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y, g = blockIdx.z;
    if (k >= N) return;
    const ModC md = c.mod[j];
    const u64 q = md.q;
    const long long NN = N, MN = (long long)M * N;
    u64 u0 = 0, u1 = 0, a0 = 0, a1 = 0;
    if (qp_add) {
        u0 = qp_add[(((long long)g * 2 + 0) * M + j) * NN + k];
        u1 = qp_add[(((long long)g * 2 + 1) * M + j) * NN + k];
    }
    if (q_add && j < L) {
        a0 = q_add[(((long long)g * 2 + 0) * L + j) * NN + k];
        a1 = q_add[(((long long)g * 2 + 1) * L + j) * NN + k];
    }
    for (int it = off[g]; it < off[g + 1]; it++) {
        const SumMember m = mem[it];
        if (m.part == nullptr) {
            if (j < L) {
                u64 x0 = m.X[(long long)j * NN + k], x1 = m.X[((long long)L + j) * NN + k];
                if (m.pt) {
                    const u64 w = __ldg(&m.pt[(long long)j * NN + k]);
                    x0 = mont_mul(x0, w, md);
                    x1 = mont_mul(x1, w, md);
                }
                a0 = add_mod(a0, x0, q);
                a1 = add_mod(a1, x1, q);
            }
            continue;
        }
        u0 = add_mod(u0, ld_cs(m.part + (long long)j * NN + k), q);
        u1 = add_mod(u1, ld_cs(m.part + MN + (long long)j * NN + k), q);
        if (j < L && m.cpart) a0 = add_mod(a0, ld_cs(m.cpart + (long long)j * NN + k), q);
    }
    U[(((long long)g * 2 + 0) * M + j) * NN + k] = u0;
    U[(((long long)g * 2 + 1) * M + j) * NN + k] = u1;
    if (j < L) {
        Cacc[(((long long)g * 2 + 0) * L + j) * NN + k] = a0;
        Cacc[(((long long)g * 2 + 1) * L + j) * NN + k] = a1;
    }
}

// U[g] = sum of the chunk sums Uv[v], v in [vstart[g], vstart[g] + vcount[g]) (and Cacc likewise):
// groups k_ks_mac split into several grid slices.  grid (N / 256, M, G)
__global__ void k_fold_groups(DevCtx c, const u64* __restrict__ Uv, const u64* __restrict__ Cv,
                              const int* __restrict__ vstart, const int* __restrict__ vcount, u64* __restrict__ U,
                              u64* __restrict__ Cacc)
{
    const int N = c.N, L = c.L, M = c.M;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y, g = blockIdx.z;
    if (k >= N) return;
    const u64 q = c.mod[j].q;
    const long long NN = N;
    const int v0 = vstart[g], nv = vcount[g];
    u64 u0 = 0, u1 = 0, a0 = 0, a1 = 0;
    for (int v = v0; v < v0 + nv; v++) {
        u0 = add_mod(u0, Uv[(((long long)v * 2 + 0) * M + j) * NN + k], q);
        u1 = add_mod(u1, Uv[(((long long)v * 2 + 1) * M + j) * NN + k], q);
        if (j < L) {
            a0 = add_mod(a0, Cv[(((long long)v * 2 + 0) * L + j) * NN + k], q);
            a1 = add_mod(a1, Cv[(((long long)v * 2 + 1) * L + j) * NN + k], q);
        }
    }
    U[(((long long)g * 2 + 0) * M + j) * NN + k] = u0;
    U[(((long long)g * 2 + 1) * M + j) * NN + k] = u1;
    if (j < L) {
        Cacc[(((long long)g * 2 + 0) * L + j) * NN + k] = a0;
        Cacc[(((long long)g * 2 + 1) * L + j) * NN + k] = a1;
    }
}

// GALA schedule 2, giant steps with the c0 ModDown deferred: per input b (groups z = b G + g)
//   S[b].c0 = sum_g sigma_g(U_z.c0)            (QP)      Qadd[b].c0 = sum_g sigma_g(C_z.c0)      (Q)
//   S[b].c1 = sum_{g: step 0} U_z.c1           (QP)      Qadd[b].c1 = sum_{g: step 0} C_z.c1     (Q)
// (sigma_g = the automorphism of the giant step g b; identity for step 0).  The final ModDown of S plus
// the giant-step key switches, plus Qadd, is the layer output.  Cacc null (key-folded path: the Q-side
// addends are already lifted into U as P C): Qadd = 0.  grid (N / 256, M, B)
__global__ void k_giant_qp(DevCtx c, const u64* __restrict__ U, const u64* __restrict__ Cacc,
                           const unsigned* __restrict__ gal, int G, int g_lo, int g_hi, u64* __restrict__ S,
                           u64* __restrict__ Qadd, int quad)
{
    const int N = c.N, L = c.L, M = c.M;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y, b = blockIdx.z;
    if (k >= N) return;
    const u64 q = c.mod[j].q;
    const long long NN = N;
    u64 s0 = 0, s1 = 0, c0 = 0, c1 = 0;
#pragma unroll 1
    for (int g = g_lo; g < g_hi; g++) {       // a multi-GPU shard sums its own groups only
        const long long z = (long long)b * G + g;
        const unsigned ge = gal[g];
        const int src = ge == 1u ? k : auto_src(k, ge, c.logN);
        s0 = add_mod(s0, __ldg(U + (quad ? u_quad_base(b, g, 0, j, G, M, N) + u_quad_off(src) : ((z * 2 + 0) * M + j) * NN + src)), q);
        if (j < L && Cacc) c0 = add_mod(c0, __ldg(Cacc + ((z * 2 + 0) * L + j) * NN + src), q);
        if (ge == 1u) {
            s1 = add_mod(s1, __ldg(U + (quad ? u_quad_base(b, g, 1, j, G, M, N) + u_quad_off(k) : ((z * 2 + 1) * M + j) * NN + k)), q);
            if (j < L && Cacc) c1 = add_mod(c1, __ldg(Cacc + ((z * 2 + 1) * L + j) * NN + k), q);
        }
    }
    S[(((long long)b * 2 + 0) * M + j) * NN + k] = s0;
    S[(((long long)b * 2 + 1) * M + j) * NN + k] = s1;
    if (j < L && Qadd) {   // (no Q-side addend in the key-folded form: it rides in U as P X)
        Qadd[(((long long)b * 2 + 0) * L + j) * NN + k] = c0;
        Qadd[(((long long)b * 2 + 1) * L + j) * NN + k] = c1;
    }
}

// Sums of per-rank partials (each word < q_j, at most 8 ranks: < 2^63) reduced mod q_j in place.
// x [count][comps][primes][N] over the prime set (prime_base + w) of `primes` moduli
__global__ void k_reduce_mod(DevCtx c, u64* __restrict__ x, long long count, int primes)
{
    const long long per = (long long)primes * c.N;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < count * per; e += (long long)gridDim.x * blockDim.x) {
        const int j = (int)((e % per) / c.N);
        x[e] %= c.mod[j].q;
    }
}

// ---------------------------------------------------------------------------
// elementwise
// out[t] = ct (.) pt[t]; grid (2 L N / blockDim, T)
__global__ void k_ct_mul_pts(DevCtx c, const u64* __restrict__ ct, const u64* __restrict__ pts,
                             u64* __restrict__ out)
{
    const int LN = c.L * c.N;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const long long t = blockIdx.y;
    if (x >= 2 * LN) return;
    const int jl = x < LN ? x : x - LN;
    const int j = jl >> c.logN;
    out[t * 2 * LN + x] = mont_mul(ct[x], __ldg(&pts[t * LN + jl]), c.mod[j]);
}

// out = a + b (sign = +1) or a - b (sign = -1) over nprimes-periodic polynomials
__global__ void k_addsub(DevCtx c, const u64* __restrict__ a, const u64* __restrict__ b, u64* __restrict__ out,
                         long long total, int nprimes, int sign)
{
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total;
         x += (long long)gridDim.x * blockDim.x) {
        int j = (int)((x / c.N) % nprimes);
        u64 q = c.mod[j].q;
        out[x] = sign > 0 ? add_mod(a[x], b[x], q) : sub_mod(a[x], b[x], q);
    }
}

// GALA schedule-2 plaintexts: out[t][j][k] = in[t][j][ sigma_{t mod baby}^src(k) ]  (identity for t mod baby == 0)
__global__ void k_gala_pt_perm(DevCtx c, const u64* __restrict__ in, int T, int baby, const unsigned* __restrict__ gal,
                               u64* __restrict__ out)
{
    const int N = c.N, M = c.M;
    const long long total = (long long)T * M * N;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int k = (int)(e % N);
        const long long tj = e / N;
        const int t = (int)(tj / M);
        const int jj = t % baby;
        const int src = jj ? auto_src(k, gal[jj], c.logN) : k;
        out[e] = in[tj * N + src];
    }
}

// GALA schedule-2 baby-step MAC.  Group z = (input bi, group g); member jj = 0..baby-1, term t = g*baby + jj.
//   jj = 0 : C0 += x.c0 (.) P_t,  C1 = x.c1 (.) P_t                     (no rotation)
//   jj > 0 : U_c,j += sum_i (sigma_jj(D_i) (.) sigma_jj(P_t))_j * ksk_jj[i][c][j]   (QP, 128-bit lazy)
//            C0   += sigma_jj(x.c0) (.) sigma_jj(P_t)
// blocks: per input (baby-1) sigma-permuted digit blocks [(L*M + L)][N] from one decomposition of x.c1;
// pts2: [T][M][N] Montgomery, pre-permuted by sigma_{t mod baby}.  grid (N/blockDim, M, B*G).
template <int L>
__global__ void __launch_bounds__(256) k_gala_mac(DevCtx c, const u64* __restrict__ X, const u64* __restrict__ blocks,
                                                  const u64* __restrict__ pts2, const u64* const* __restrict__ keys,
                                                  int baby, int G, u64* __restrict__ U, u64* __restrict__ Cacc)
{
    const int N = c.N, M = L + 1;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y, z = blockIdx.z;
    const int bi = z / G, g = z % G;
    if (k >= N) return;
    const ModC md = c.mod[j];
    const u64 q = md.q;
    const int lazy = c.lazy[j];
    const long long NN = N, LN = (long long)L * N, W = 2 * LN, MN = (long long)M * N;
    const long long blk_words = (long long)(L * M + L) * N;
    const u64* x = X + bi * W;
    const u64* blk0 = blocks + (long long)bi * (baby - 1) * blk_words;
    u64 a0 = 0, a1 = 0, u0 = 0, u1 = 0;
    {   // step-0 member
        const u64 w = __ldg(pts2 + ((long long)g * baby) * MN + j * NN + k);
        if (j < L) {
            a0 = mont_mul(__ldg(x + j * NN + k), w, md);
            a1 = mont_mul(__ldg(x + LN + j * NN + k), w, md);
        }
    }
    Acc128 s0, s1;
    int pending = 0;
    for (int jj = 1; jj < baby; jj++) {
        const long long t = (long long)g * baby + jj;
        const u64 w = __ldcs((const unsigned long long*)(pts2 + t * MN + j * NN + k));
        const u64* blk = blk0 + (long long)(jj - 1) * blk_words;
        const u64* key = keys[jj];
        u64 dv[L], kb[L], ka[L];
#pragma unroll
        for (int i = 0; i < L; i++) {
            dv[i] = __ldg(blk + ((long long)i * M + j) * NN + k);
            kb[i] = __ldg(key + (((long long)i * 2 + 0) * M + j) * NN + k);
            ka[i] = __ldg(key + (((long long)i * 2 + 1) * M + j) * NN + k);
        }
        u64 cc = 0;
        if (j < L) cc = __ldg(blk + ((long long)L * M + j) * NN + k);
        if (pending + L > lazy) {
            u0 = add_mod(u0, s0.reduce(md), q);
            u1 = add_mod(u1, s1.reduce(md), q);
            s0 = Acc128();
            s1 = Acc128();
            pending = 0;
        }
#pragma unroll
        for (int i = 0; i < L; i++) {
            const u64 d = mont_mul(dv[i], w, md);      // digit of (x.c1 (.) p_t), rotated
            s0.mac(d, kb[i]);
            s1.mac(d, ka[i]);
        }
        pending += L;
        if (j < L) a0 = add_mod(a0, mont_mul(cc, w, md), q);
    }
    u0 = add_mod(u0, s0.reduce(md), q);
    u1 = add_mod(u1, s1.reduce(md), q);
    U[(((long long)z * 2 + 0) * M + j) * NN + k] = u0;
    U[(((long long)z * 2 + 1) * M + j) * NN + k] = u1;
    if (j < L) {
        Cacc[(((long long)z * 2 + 0) * L + j) * NN + k] = a0;
        Cacc[(((long long)z * 2 + 1) * L + j) * NN + k] = a1;
    }
}

// GALA schedule 2, stage A (per input and baby rotation jj, shared by every group):
//   E[bi][jj][c][j][k] = sum_i sigma_jj(D_i)_j[k] * ksk_jj[i][c][j][k]          (QP)
//   R0[bi][jj][j][k]   = sigma_jj(x.c0)_j[k]                                     (Q)
// D: identity digit block of the input ([(L*M + L)][N], NTT), gathered through sigma (L2 resident).
// grid (B (baby - 1), M, N / blockDim): all (input, rotation) pairs of one coefficient slice run
// together, so the slice of every key stays in L2 across the inputs.  Each thread serves CB inputs
// with one register copy of the key limbs (key loads amortised over the inputs).
template <int L, int CB>
__global__ void __launch_bounds__(256) k_gala_e(DevCtx c, const u64* __restrict__ Dblk, const u64* const* __restrict__ keys,
                                                const unsigned* __restrict__ gal, int baby, u64* __restrict__ E,
                                                u64* __restrict__ R0)
{
    const int N = c.N, M = L + 1;
    const int k = blockIdx.z * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    const int bg = blockIdx.x / (baby - 1), jj = blockIdx.x % (baby - 1) + 1;
    if (k >= N) return;
    const ModC md = c.mod[j];
    const long long NN = N, MN = (long long)M * N;
    const u64* key = keys[jj];
    const int src = auto_src(k, gal[jj], c.logN);
    u64 ka[L], kb[L];
#pragma unroll
    for (int i = 0; i < L; i++) {
        ka[i] = __ldg(key + (((long long)i * 2 + 0) * M + j) * NN + k);
        kb[i] = __ldg(key + (((long long)i * 2 + 1) * M + j) * NN + k);
    }
#pragma unroll
    for (int cb = 0; cb < CB; cb++) {
        const int bi = bg * CB + cb;
        const long long z = (long long)bi * (baby - 1) + (jj - 1);
        const u64* D = Dblk + (long long)bi * (L * M + L) * NN;
        Acc128 s0, s1;
#pragma unroll
        for (int i = 0; i < L; i++) {
            const u64 d = __ldg(D + ((long long)i * M + j) * NN + src);
            s0.mac(d, ka[i]);
            s1.mac(d, kb[i]);
        }
        u64* e = E + z * 2 * MN + j * NN + k;
        e[0] = s0.reduce(md);
        e[MN] = s1.reduce(md);
        if (j < L) R0[(z * L + j) * NN + k] = __ldg(D + ((long long)L * M + j) * NN + src);
    }
}

// GALA schedule 2, stage B (per input bi and group g):
//   U_c,j = sum_{jj >= 1} w_t (.) E[bi][jj][c][j]      C0_j = sum_{jj >= 1} w_t (.) R0[bi][jj][j] + x.c0 (.) P_{g b}
//   C1_j  = x.c1 (.) P_{g b}                            (t = g b + jj, w_t = sigma_jj(P_t) pre-permuted)
// Members are processed in chunks of CH: all loads of a chunk are issued before its multiplies
// (memory-level parallelism), and the 128-bit accumulators are Montgomery-reduced once per chunk
// (CH <= c.lazy[j] products).  grid (N / blockDim, M, B * G), z = bi * G + g (input-major: E of an
// input stays in L2 while its groups run).
template <int CH, bool SLICED>
__global__ void __launch_bounds__(256, 4) k_gala_mac2(DevCtx c, const u64* __restrict__ X, const u64* __restrict__ E,
                                                   const u64* __restrict__ R0, const u64* __restrict__ pts2, int baby,
                                                   int G, u64* __restrict__ U, u64* __restrict__ Cacc)
{
    const int N = c.N, L = c.L, M = c.M;
    // SLICED: grid (B G, M, N / blockDim) -- every (input, group) of one coefficient slice runs
    // together, so the slice's plaintexts and E stay in L2 across all inputs and groups
    const int k = (SLICED ? blockIdx.z : blockIdx.x) * blockDim.x + threadIdx.x;
    const int j = blockIdx.y, z = SLICED ? blockIdx.x : blockIdx.z;
    const int bi = z / G, g = z % G;
    if (k >= N) return;
    const ModC md = c.mod[j];
    const u64 q = md.q;
    const bool jq = j < L;
    const long long NN = N, LN = (long long)L * N, W = 2 * LN, MN = (long long)M * N;
    const u64* x = X + bi * W;
    const u64* Eb = E + (long long)bi * (baby - 1) * 2 * MN + j * NN + k;
    const u64* Rb = R0 + (long long)bi * (baby - 1) * LN + j * NN + k;
    const u64* Pb = pts2 + ((long long)g * baby) * MN + j * NN + k;
    u64 u0 = 0, u1 = 0, a0 = 0, a1 = 0;
    {   // step-0 member: x (.) P_{g b}
        const u64 w = __ldg(Pb);
        if (jq) {
            a0 = mont_mul(__ldg(x + j * NN + k), w, md);
            a1 = mont_mul(__ldg(x + LN + j * NN + k), w, md);
        }
    }
    // 128-bit lazy accumulation: one Montgomery reduction per c.lazy[j] products (k q^2 < q 2^64);
    // the next member's loads are issued before the current member's products (software pipeline)
    Acc128 s0, s1, sc;
    const int lazy = c.lazy[j];
    int pending = 0;
    u64 nw = 0, ne0 = 0, ne1 = 0, nr0 = 0;
    auto fetch = [&](int jj) {
        nw = SLICED ? __ldg(Pb + (long long)jj * MN) : __ldcs((const unsigned long long*)(Pb + (long long)jj * MN));
        ne0 = __ldg(Eb + (long long)(jj - 1) * 2 * MN);
        ne1 = __ldg(Eb + (long long)(jj - 1) * 2 * MN + MN);
        if (jq) nr0 = __ldg(Rb + (long long)(jj - 1) * LN);
    };
    if (baby > 1) fetch(1);
    for (int jj = 1; jj < baby; jj++) {
        const u64 w = nw, e0 = ne0, e1 = ne1, r0 = nr0;
        if (jj + 1 < baby) fetch(jj + 1);
        if (pending == lazy) {
            u0 = add_mod(u0, s0.reduce(md), q);
            u1 = add_mod(u1, s1.reduce(md), q);
            if (jq) a0 = add_mod(a0, sc.reduce(md), q);
            s0 = Acc128();
            s1 = Acc128();
            sc = Acc128();
            pending = 0;
        }
        s0.mac(w, e0);
        s1.mac(w, e1);
        if (jq) sc.mac(w, r0);
        pending++;
    }
    u0 = add_mod(u0, s0.reduce(md), q);
    u1 = add_mod(u1, s1.reduce(md), q);
    if (jq) a0 = add_mod(a0, sc.reduce(md), q);
    U[(((long long)z * 2 + 0) * M + j) * NN + k] = u0;
    U[(((long long)z * 2 + 1) * M + j) * NN + k] = u1;
    if (jq) {
        Cacc[(((long long)z * 2 + 0) * L + j) * NN + k] = a0;
        Cacc[(((long long)z * 2 + 1) * L + j) * NN + k] = a1;
    }
}

// out[b] = ct[b] with c0 -= DM[b]  (batched subtract_plain)
__global__ void k_sub_plain(DevCtx c, const u64* __restrict__ ct, const u64* __restrict__ DM, u64* __restrict__ out,
                            int B)
{
    const long long LN = (long long)c.L * c.N, W = 2 * LN;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < B * W;
         x += (long long)gridDim.x * blockDim.x) {
        const long long b = x / W, r = x - b * W;
        u64 v = ct[x];
        if (r < LN) {
            const int j = (int)(r >> c.logN);
            v = sub_mod(v, DM[b * LN + r], c.mod[j].q);
        }
        out[x] = v;
    }
}

// conv first-Add over one chunk of input blocks [ib0, ib1), for a batch of images sharing the weights:
//   acc[b][o][d][comp][j][x] (+)= sum_{ib in chunk} sum_tap R[b][ib][tap][comp][j][x] * pt[o][ib][d][tap][j][x]
// Register tile: each thread carries IMG images x ODT accumulator rows od = o c_n + d, so a rotated
// input word is loaded once per ODT rows and a plaintext word once per IMG images (the single-row,
// single-image form re-read R from L2 once per row: L2-bound).  The image groups of one row group
// are adjacent in the launch order (grid.y), so later groups find the plaintexts in L2; the host
// sizes ib chunks so R[., ib0:ib1] stays resident in L2 across the row groups.  128-bit sums
// T = hi 2^64 + lo: every c.lazy[j] products the high word is brought back below q by one
// conditional subtraction (T - q 2^64 == T mod q; lazy products of canonical operands add less
// than q to hi), so the sum never leaves its 4 registers; one REDC at the end.  grid: (N / blockDim, L * ceil(nimg / IMG), ceil(rows / ODT)).
template <int IMG, int ODT, bool PP>
__global__ void __launch_bounds__(256) k_kg_accumulate(DevCtx c, const u64* __restrict__ R, long long R_bs, int n_ib,
                                                       int ib0, int ib1, int k, const u64* __restrict__ pts, int c_n,
                                                       int rows, int nimg, int accumulate, u64* __restrict__ acc,
                                                       long long acc_bs)
{
    const int N = c.N, L = c.L;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y % L, b0 = (blockIdx.y / L) * IMG, od0 = blockIdx.z * ODT;
    if (x >= N) return;
    const int nb = nimg - b0 < IMG ? nimg - b0 : IMG;
    const int nr = rows - od0 < ODT ? rows - od0 : ODT;
    const u64 q = c.mod[j].q;
    const int lazy = c.lazy[j];
    const long long LN = (long long)L * N, W = 2 * LN;
    // PP: partial-product sums (4 IMAD.WIDE.U32 per product instead of a 64x64 -> 128 multiply; the kernel
    // is FMA-heavy-pipe bound), flushed through one REDC every c.lazy[j] products into a value mod q -- more
    // registers, so it pays where the grid, not occupancy, limits (one image)
    Acc128 ac[ODT][IMG][2];
    AccPP<> a[ODT][IMG][2];
    u64 v[ODT][IMG][2];
#pragma unroll
    for (int r = 0; r < ODT; r++)
#pragma unroll
        for (int i = 0; i < IMG; i++)
#pragma unroll
            for (int cp = 0; cp < 2; cp++) {
                a[r][i][cp].clear();
                v[r][i][cp] = 0;
            }
    const u64* prow[ODT];
#pragma unroll
    for (int r = 0; r < ODT; r++) {
        const int od = od0 + (r < nr ? r : 0);
        const int o = od / c_n, d = od - o * c_n;
        prow[r] = pts + (((long long)o * n_ib * c_n + d) * k) * LN + (long long)j * N + x;
    }
    int pending = 0;
    const u64* Rimg = R + (long long)b0 * R_bs + (long long)j * N + x;
    const long long pt_ib = (long long)c_n * k * LN;
    for (int ib = ib0; ib < ib1; ib++) {
        const u64* Rb = Rimg + ((long long)ib * k) * W;
        for (int t = 0; t < k; t++) {
            if (pending == lazy) {
#pragma unroll
                for (int r = 0; r < ODT; r++)
#pragma unroll
                    for (int i = 0; i < IMG; i++)
#pragma unroll
                        for (int cp = 0; cp < 2; cp++) {
                            if (PP) {
                                v[r][i][cp] = add_mod(v[r][i][cp], a[r][i][cp].reduce_sf(q), q);
                                a[r][i][cp].clear();
                            } else {
                                ac[r][i][cp].hi = csub(ac[r][i][cp].hi, q);
                            }
                        }
                pending = 0;
            }
            u64 rv[IMG][2];
#pragma unroll
            for (int i = 0; i < IMG; i++) {
                const u64* rp = Rb + (i < nb ? i : 0) * R_bs + t * W;
                rv[i][0] = __ldg(rp);
                rv[i][1] = __ldg(rp + LN);
            }
#pragma unroll
            for (int r = 0; r < ODT; r++) {
                const u64 w = __ldcs((const unsigned long long*)(prow[r] + (long long)ib * pt_ib + t * LN));
#pragma unroll
                for (int i = 0; i < IMG; i++) {
                    if (PP) {
                        a[r][i][0].mac(rv[i][0], w);
                        a[r][i][1].mac(rv[i][1], w);
                    } else {
                        ac[r][i][0].mac(rv[i][0], w);
                        ac[r][i][1].mac(rv[i][1], w);
                    }
                }
            }
            pending++;
        }
    }
#pragma unroll
    for (int r = 0; r < ODT; r++) {
        if (r >= nr) break;
#pragma unroll
        for (int i = 0; i < IMG; i++) {
            if (i >= nb) break;
            u64 v0, v1;
            if (PP) {
                v0 = add_mod(v[r][i][0], a[r][i][0].reduce_sf(q), q);
                v1 = add_mod(v[r][i][1], a[r][i][1].reduce_sf(q), q);
            } else {
                v0 = csub(redc_sf_lazy(csub(ac[r][i][0].hi, q), ac[r][i][0].lo, q), q);
                v1 = csub(redc_sf_lazy(csub(ac[r][i][1].hi, q), ac[r][i][1].lo, q), q);
            }
            u64* out = acc + (long long)(b0 + i) * acc_bs + (long long)(od0 + r) * W + (long long)j * N + x;
            if (accumulate) {
                v0 = add_mod(v0, out[0], q);
                v1 = add_mod(v1, out[LN], q);
            }
            out[0] = v0;
            out[LN] = v1;
        }
    }
}

// ---------------------------------------------------------------------------
// On-GPU kernel-grouping plaintext slots (conv.py:220-235 coef_vectors, physical two-row form):
// for plaintext (obp, ib, d, tap) and physical slot s = row * n + ch * B + y * u_w + x:
//   ob = obp * pair + row;  value = kernels[ob c_n + (ch - d) mod c_n][ib c_n + ch][dh + kh/2][dw + kw/2]
//   when (x + dw, y + dh) is inside the image and ob < n_ob, else 0.
// `first` is the flat index of the first plaintext generated; out [count][N] u32.
struct KgGeom {
    int c_o, c_i, k_h, k_w, u_w, u_h, c_n, n_ib, n_ob, pair;
};
__global__ void k_kg_slots(DevCtx c, const int32_t* __restrict__ kern, KgGeom g, long long first, int count,
                           uint32_t* __restrict__ out)
{
    const int N = c.N, n = N / 2;
    const int B = g.u_w * g.u_h, k = g.k_h * g.k_w;
    const long long total = (long long)count * N;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long pidx = first + e / N;
        const int s = (int)(e % N);
        int tap = (int)(pidx % k);
        long long rest = pidx / k;
        const int d = (int)(rest % g.c_n);
        rest /= g.c_n;
        const int ib = (int)(rest % g.n_ib);
        const int obp = (int)(rest / g.n_ib);
        const int row = s / n, cs = s % n;
        const int ob = g.pair == 2 ? obp * 2 + row : obp;
        uint32_t v = 0;
        const int ch = cs / B, pos = cs % B;
        if (ob < g.n_ob && ch < g.c_n) {
            const int y = pos / g.u_w, x = pos % g.u_w;
            const int dh = tap / g.k_w - g.k_h / 2, dw = tap % g.k_w - g.k_w / 2;
            if (x + dw >= 0 && x + dw < g.u_w && y + dh >= 0 && y + dh < g.u_h) {
                const int o = ob * g.c_n + ((ch - d) % g.c_n + g.c_n) % g.c_n;
                const int i = ib * g.c_n + ch;
                v = (uint32_t)kern[(((long long)o * g.c_i + i) * g.k_h + (dh + g.k_h / 2)) * g.k_w + (dw + g.k_w / 2)];
            }
        }
        out[e] = v;
    }
}

// ---------------------------------------------------------------------------
// Kernel-grouping schedule 2 (factored plaintexts; oracle o_conv_kg2).
// Band masks: slot s of mask (tap, beta) is 1 iff s lies in band beta and the tap's source pixel is
// inside the image.  pair == 2: beta = row * c_n + ch; pair == 1: beta = ch over both rows.
__global__ void k_kg_mask_slots(DevCtx c, KgGeom g, uint32_t* __restrict__ out)
{
    const int N = c.N, n = N / 2, B = g.u_w * g.u_h, k = g.k_h * g.k_w;
    const int nb = g.pair * g.c_n;
    const long long total = (long long)k * nb * N;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const int s = (int)(e % N);
        const long long tb = e / N;
        const int beta = (int)(tb % nb), tap = (int)(tb / nb);
        const int row = s / n, cs = s % n, ch = cs / B, pos = cs % B, y = pos / g.u_w, x = pos % g.u_w;
        const int band = g.pair == 2 ? row * g.c_n + ch : ch;
        const int dh = tap / g.k_w - g.k_h / 2, dw = tap % g.k_w - g.k_w / 2;
        const bool ok = x + dw >= 0 && x + dw < g.u_w && y + dh >= 0 && y + dh < g.u_h;
        out[e] = (band == beta && ok) ? 1u : 0u;
    }
}

// Masked products of the rotated inputs in the extended basis QP, K = (ib, tap, beta),
// pos = (comp, j, i), g = ib k + tap:
//   Z[g][pos]  = sum_l sigma_tap(D_ib)[l][j][i] ksk_tap[l][comp][j][i] + P sigma_tap(c0_ib)[j][i]
//                (the key switch without ModDown; P c0 term for comp 0, j < L; Z = P x for step 0)
//   Y[K][pos]  = Z[g][pos] (.) Mask[tap][beta][j][i]
// written as the 8 little-endian bytes of each word biased by 0x80 (signed int8 for the
// tensor-core GEMM) in the K-contiguous layout Bt[8 pos + b][Kp].  D is the identity digit block
// of each input ([(L M + L)][N], NTT), gathered through sigma: in bit-reversed order an
// automorphism maps each aligned run of 32 slots onto one aligned run, so the gathers stay
// coalesced.  One CTA owns a KG_PT x KG_KT tile (KG_KT / nb groups g): Z is formed once per
// (g, pos) and multiplied by the nb masks; the tile is transposed through shared memory so the
// loads run along pos and the 16-byte stores along K (XOR swizzle: both phases conflict-free).
#define KG_PT 32
#define KG_KT 128
#define KG_MAXK 64          // taps per convolution (7 x 7 = 49 at most here)
#ifndef KG_ZU
#define KG_ZU 2             // post-mask columns per load round
#endif
__device__ __forceinline__ int kg_swz(int pp, int kk) { return pp * KG_KT + (kk ^ ((pp + 4 * (kk >> 4)) & 15)); }

// Montgomery-form operands [count][M][N] -> Shoup pairs (w, floor(w 2^64 / q)).  With w_m = w 2^64
// mod q: w = REDC(w_m) and w 2^64 = q wsh + w_m, so wsh = (w 2^64 - w_m) / q = w_m (-q^-1) mod 2^64.
// keep_mont: Shoup pairs of the Montgomery value itself, (w_m, floor(w_m 2^64 / q)) -- multiplying a
// REDC output (x 2^-64) by w_m = w 2^64 gives x w directly (the post-mask epilogues use this).
__global__ void k_mont_to_shoup(DevCtx c, const u64* __restrict__ in, long long count, int keep_mont,
                                ulonglong2* __restrict__ out)
{
    const int N = c.N, M = c.M;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < count * M * N;
         e += (long long)gridDim.x * blockDim.x) {
        const ModC md = c.mod[(int)((e / N) % M)];
        const u64 wm = in[e];
        if (keep_mont) out[e] = make_ulonglong2(wm, mont_mul(wm, md.r2, md) * md.qinv_neg);
        else out[e] = make_ulonglong2(csub(redc_lazy(0, wm, md), md.q), wm * md.qinv_neg);
    }
}

// 4x4 byte transpose: out[b] = byte b of x0..x3 (PRMT)
__device__ __forceinline__ void bytes4x4(uint32_t x0, uint32_t x1, uint32_t x2, uint32_t x3, uint32_t* o)
{
    const uint32_t t0 = __byte_perm(x0, x1, 0x5140), t1 = __byte_perm(x0, x1, 0x7362);
    const uint32_t t2 = __byte_perm(x2, x3, 0x5140), t3 = __byte_perm(x2, x3, 0x7362);
    o[0] = __byte_perm(t0, t2, 0x5410);
    o[1] = __byte_perm(t0, t2, 0x7632);
    o[2] = __byte_perm(t1, t3, 0x5410);
    o[3] = __byte_perm(t1, t3, 0x7632);
}

// LOGN > 0: the ring degree at compile time (the MN-strided digit / key loads then take immediate
// offsets from one address per column); 0: runtime
template <int L, int LOGN>
__global__ void __launch_bounds__(256) k_kg_zy(DevCtx c, const u64* __restrict__ Dblk, const u64* __restrict__ X,
                                               const u64* const* __restrict__ keys, const unsigned* __restrict__ gal,
                                               const ulonglong2* __restrict__ masks, const ulonglong2* __restrict__ pconst,
                                               int k, int nb, int n_ib, int Kp, int8_t* __restrict__ Bt, int canon)
{
    __shared__ u64 sm[KG_PT * KG_KT];
    // per-block tables: each tap's key pointer and, per position of the block, its automorphism source
    // index (the inner loop then issues no dependent pointer loads and no bit reversals)
    __shared__ const u64* s_key[KG_MAXK];
    __shared__ int s_src[KG_MAXK][KG_PT];
    __shared__ int s_col[KG_KT];      // post-mask: column gl -> (input ib << 8) | tap, -1 past the last column
    constexpr int M = L + 1;
    const int N = LOGN ? (1 << LOGN) : c.N, logN = LOGN ? LOGN : c.logN, MN = M * N, P2 = 2 * MN;
    const int pos0 = blockIdx.x * KG_PT, K0 = blockIdx.y * KG_KT;
    for (int e = threadIdx.x; e < k * KG_PT; e += blockDim.x) {
        const int t = e / KG_PT, pp = e - t * KG_PT;
        const int pos = pos0 + pp, comp = pos >= MN ? 1 : 0, jl = pos - comp * MN;
        const u64* kt = keys[t];
        if (pp == 0) s_key[t] = kt;
        s_src[t][pp] = kt ? auto_src(jl & (N - 1), gal[t], logN) : 0;
    }
    if (masks == nullptr)
        for (int gl = threadIdx.x; gl < KG_KT; gl += blockDim.x) {
            const int g = K0 + gl;      // nb == 1 in the post-mask form
            s_col[gl] = g < n_ib * k ? ((g / k) << 8) | (g % k) : -1;
        }
    __syncthreads();
    // batch element blockIdx.z: its inputs follow the previous elements' (n_ib each), its byte planes
    // continue the tile order (canon only)
    Dblk += (long long)blockIdx.z * n_ib * ((L * M + L) * (long long)N);
    X += (long long)blockIdx.z * n_ib * 2 * L * (long long)N;
    Bt += (long long)blockIdx.z * 8 * P2 * (long long)Kp;
    {
        const int pp = threadIdx.x & 31, w = threadIdx.x >> 5;
        const int pos = pos0 + pp;
        const int comp = pos >= MN ? 1 : 0, jl = pos - comp * MN, j = jl >> logN, i = jl & (N - 1);
        const ModC md = c.mod[j < M ? j : 0];
        const u64 q = md.q;
        const ulonglong2 pc = pconst[j < M ? j : 0];   // P mod q_j, Shoup companion
        const int gpt = KG_KT / nb, g0 = K0 / nb, G = n_ib * k;
        const int bw = (L * M + L) * N;                  // words per identity block (< 2^31)
        const u64* Dj = Dblk + (long long)j * N;
        const u64* Xj = X + (long long)comp * L * N + jl;
        const int koff = (comp * M + j) * N + i;
        // (ib, t) of g = g0 + gl, advanced incrementally (gl steps by 8): no division in the loop
        int gfirst = g0 + w;
        int ib = gfirst / k, t = gfirst - ib * k;
        if (masks == nullptr) {
            // post-mask form, lean inner loop: every column's (input, tap) comes from the block's column
            // table, addresses are 32-bit word offsets from block-invariant bases, and KG_ZU columns'
            // loads are issued before any product (the loop is load-latency bound)
            const uint32_t uN = (uint32_t)N;
            const uint32_t dj = (uint32_t)j * uN;
            const uint32_t xo = (uint32_t)comp * (uint32_t)L * uN + (uint32_t)jl;
            const bool has_c0 = comp == 0 && j < L;
            for (int gl0 = w; gl0 < gpt; gl0 += 8 * KG_ZU) {
                u64 dv[KG_ZU][L + 1], kv[KG_ZU][L];
                int kind[KG_ZU];   // 0: nothing, 1: P x.c0 only (step 0), 2: key switch
#pragma unroll
                for (int u = 0; u < KG_ZU; u++) {
                    const int gl = gl0 + 8 * u;
                    const int cm = gl < gpt ? s_col[gl] : -1;
                    kind[u] = 0;
                    if (cm >= 0 && pos < P2) {
                        const int ibu = cm >> 8, tt = cm & 255;
                        const u64* key = s_key[tt];
                        if (key == nullptr) {
                            kind[u] = 1;
                            dv[u][0] = j < L ? __ldg(X + ((uint32_t)ibu * 2u * (uint32_t)L * uN + xo)) : 0ull;
                        } else {
                            kind[u] = 2;
                            const u64* dp = Dblk + ((uint32_t)ibu * (uint32_t)bw + dj + (uint32_t)s_src[tt][pp]);
                            const u64* kp = key + koff;
#pragma unroll
                            for (int l = 0; l < L; l++) {
                                dv[u][l] = __ldg(dp + l * MN);
                                kv[u][l] = __ldg(kp + l * 2 * MN);
                            }
                            dv[u][L] = has_c0 ? __ldg(dp + L * MN) : 0ull;
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < KG_ZU; u++) {
                    const int gl = gl0 + 8 * u;
                    if (gl >= gpt) break;
                    u64 z = 0;
                    if (kind[u] == 1) {
                        z = csub(shoup_lazy_sf(dv[u][0], pc.x, pc.y, q), q);
                    } else if (kind[u] == 2) {
                        AccPP<true> s;
#pragma unroll
                        for (int l = 0; l < L; l++) {
                            if (l == 0) s.set(dv[u][0], kv[u][0]);
                            else s.mac(dv[u][l], kv[u][l]);
                        }
                        z = s.reduce_sf(q);
                        if (has_c0) z = add_mod(z, csub(shoup_lazy_sf(dv[u][L], pc.x, pc.y, q), q), q);
                    }
                    sm[kg_swz(pp, gl)] = z ^ 0x8080808080808080ull;
                }
            }
        } else
        for (int gl = w; gl < gpt; gl += 8) {
            const int g = g0 + gl;
            const bool valid = g < G && pos < P2;
            const int tt = t;
            u64 z = 0;
            if (valid) {
                const u64* key = s_key[tt];
                if (key == nullptr) {
                    if (j < L) z = csub(shoup_lazy_sf(__ldg(Xj + (long long)ib * 2 * L * N), pc.x, pc.y, q), q);
                } else {
                    const int src = s_src[tt][pp];
                    const u64* D = Dj + (long long)ib * bw + src;
                    const u64* kp = key + koff;
                    AccPP<true> s;   // L <= 4 canonical products
#pragma unroll
                    for (int l = 0; l < L; l++) {
                        if (l == 0) s.set(__ldg(D), __ldg(kp));
                        else s.mac(__ldg(D + l * MN), __ldg(kp + l * 2 * MN));
                    }
                    z = s.reduce_sf(q);
                    if (comp == 0 && j < L)
                        z = add_mod(z, csub(shoup_lazy_sf(__ldg(D + L * MN), pc.x, pc.y, q), q), q);
                }
            }
            t += 8;
            while (t >= k) {
                t -= k;
                ib++;
            }
            if (masks == nullptr) {            // post-mask form: the GEMM takes Z itself (nb == 1)
                sm[kg_swz(pp, gl)] = z ^ 0x8080808080808080ull;
                continue;
            }
            const ulonglong2* mk = masks + (long long)tt * nb * MN + jl;
            for (int beta = 0; beta < nb; beta++) {
                u64 v = 0;
                if (valid) {
                    const ulonglong2 m = __ldg(mk + (long long)beta * MN);
                    v = csub(shoup_lazy_sf(z, m.x, m.y, q), q);
                }
                sm[kg_swz(pp, gl * nb + beta)] = v ^ 0x8080808080808080ull;
            }
        }
    }
    __syncthreads();
    const int pp = threadIdx.x >> 3, ch = threadIdx.x & 7;
    const int pos = pos0 + pp;
    if (K0 + ch * 16 >= Kp || pos >= P2) return;
    uint32_t lo[16], hi[16];
#pragma unroll
    for (int i = 0; i < 16; i++) {
        const u64 v = sm[kg_swz(pp, ch * 16 + i)];
        lo[i] = (uint32_t)v;
        hi[i] = (uint32_t)(v >> 32);
    }
    // plane b holds byte b of the 16 words: [b][q4] from the 4x4 transposes of words 4 q4 .. 4 q4 + 3
    uint32_t pl[8][4];
#pragma unroll
    for (int q4 = 0; q4 < 4; q4++) {
        uint32_t o[4];
        bytes4x4(lo[4 * q4], lo[4 * q4 + 1], lo[4 * q4 + 2], lo[4 * q4 + 3], o);
#pragma unroll
        for (int b = 0; b < 4; b++) pl[b][q4] = o[b];
        bytes4x4(hi[4 * q4], hi[4 * q4 + 1], hi[4 * q4 + 2], hi[4 * q4 + 3], o);
#pragma unroll
        for (int b = 0; b < 4; b++) pl[4 + b][q4] = o[b];
    }
    if (canon) {   // tcgen05 tile layout: [tile = pos / 32][16-byte K chunk][256 rows (pos % 32, b)][16]
        int8_t* o = Bt + ((((long long)(pos >> 5) * (Kp >> 4) + (K0 >> 4) + ch) * 256) + 8 * (pos & 31)) * 16;
#pragma unroll
        for (int b = 0; b < 8; b++) *(uint4*)(o + b * 16) = make_uint4(pl[b][0], pl[b][1], pl[b][2], pl[b][3]);
        return;
    }
    int8_t* o = Bt + (long long)pos * 8 * Kp + K0 + ch * 16;
#pragma unroll
    for (int b = 0; b < 8; b++) *(uint4*)(o + (long long)b * Kp) = make_uint4(pl[b][0], pl[b][1], pl[b][2], pl[b][3]);
}

// Post-mask form of k_kg_zy with BOTH key-switch components of a position in one thread: Z[0] and
// Z[1] at (j, i) share the gathered digits sigma_t(D_l)[j][i] (and the c0 term goes to component 0),
// so the digit gathers -- one 256-byte row per (input, tap, slot) and warp, the kernel's dominant L2
// traffic -- are halved.  Block: 32 positions (j, i) x 128 K columns = 64 output rows of the byte
// planes (the two components' tiles); columns come from the block's table ((ib << 8) | tap).
// Dynamic shared memory: 2 x KG_PT x KG_KT words.
template <int L, int LOGN, bool PRE>
__global__ void __launch_bounds__(256, 3) k_kg_zy2(DevCtx c, const u64* __restrict__ Dblk, const u64* __restrict__ X,
                                                const u64* const* __restrict__ keys, const unsigned* __restrict__ gal,
                                                const ulonglong2* __restrict__ masks, const ulonglong2* __restrict__ pconst,
                                                int k, int nb, int n_ib, int Kp, int8_t* __restrict__ Bt)
{
    extern __shared__ u64 zsm[];                 // [comp][KG_PT * KG_KT], swizzled as kg_swz
    __shared__ const u64* s_key[KG_MAXK];
    __shared__ int s_src[KG_MAXK][KG_PT];
    __shared__ int s_col[KG_KT];
    constexpr int M = L + 1;
    const int N = LOGN ? (1 << LOGN) : c.N, logN = LOGN ? LOGN : c.logN, MN = M * N, P2 = 2 * MN;
    const int jl0 = blockIdx.x * KG_PT, K0 = blockIdx.y * KG_KT;
    for (int e = threadIdx.x; e < k * KG_PT; e += blockDim.x) {
        const int t = e / KG_PT, pp = e - t * KG_PT;
        const u64* kt = keys[t];
        if (pp == 0) s_key[t] = kt;
        s_src[t][pp] = kt ? auto_src((jl0 + pp) & (N - 1), gal[t], logN) : 0;
    }
    const int gpt = KG_KT / nb;                 // (input, tap) groups per block: nb K columns each (pre-mask)
    for (int gl = threadIdx.x; gl < gpt; gl += blockDim.x) {
        const int g = K0 / nb + gl;
        s_col[gl] = g < n_ib * k ? ((g / k) << 8) | (g % k) : -1;
    }
    __syncthreads();
    Dblk += (long long)blockIdx.z * n_ib * ((L * M + L) * (long long)N);
    X += (long long)blockIdx.z * n_ib * 2 * L * (long long)N;
    Bt += (long long)blockIdx.z * 8 * P2 * (long long)Kp;
    {
        const int pp = threadIdx.x & 31, w = threadIdx.x >> 5;
        const int jl = jl0 + pp, j = jl >> logN, i = jl & (N - 1);
        const u64 q = c.mod[j].q;
        const ulonglong2 pc = pconst[j];
        const bool has_c0 = j < L;
        const uint32_t bw = (uint32_t)(L * M + L) * (uint32_t)N;
        const uint32_t dj = (uint32_t)j * (uint32_t)N;
        const uint32_t koff = (uint32_t)j * (uint32_t)N + (uint32_t)i;
        for (int gl0 = w; gl0 < gpt; gl0 += 8 * KG_ZU) {
            u64 dv[KG_ZU][L + 1], k0v[KG_ZU][L], k1v[KG_ZU][L];
            int kind[KG_ZU], tap[KG_ZU];
#pragma unroll
            for (int u = 0; u < KG_ZU; u++) {
                const int gl = gl0 + 8 * u;
                const int cm = gl < gpt ? s_col[gl] : -1;
                tap[u] = cm & 255;
                kind[u] = 0;
                if (cm >= 0) {
                    const int ibu = cm >> 8, tt = cm & 255;
                    const u64* key = s_key[tt];
                    if (key == nullptr) {        // step 0: Z = P x (no key switch)
                        kind[u] = 1;
                        const u64* xp = X + ((uint32_t)ibu * 2u * (uint32_t)L * (uint32_t)N + (uint32_t)jl);
                        dv[u][0] = has_c0 ? __ldg(xp) : 0ull;
                        dv[u][1] = has_c0 ? __ldg(xp + L * N) : 0ull;
                    } else {
                        kind[u] = 2;
                        const u64* dp = Dblk + ((uint32_t)ibu * bw + dj + (uint32_t)s_src[tt][pp]);
                        const u64* kp = key + koff;
#pragma unroll
                        for (int l = 0; l < L; l++) {
                            dv[u][l] = __ldg(dp + l * MN);
                            k0v[u][l] = __ldg(kp + (2 * l) * MN);
                            k1v[u][l] = __ldg(kp + (2 * l + 1) * MN);
                        }
                        dv[u][L] = has_c0 ? __ldg(dp + L * MN) : 0ull;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < KG_ZU; u++) {
                const int gl = gl0 + 8 * u;
                if (gl >= gpt) break;
                u64 z0 = 0, z1 = 0;
                if (kind[u] == 1) {
                    z0 = csub(shoup_lazy_sf(dv[u][0], pc.x, pc.y, q), q);
                    z1 = csub(shoup_lazy_sf(dv[u][1], pc.x, pc.y, q), q);
                } else if (kind[u] == 2) {
                    AccPP<true> s0, s1;
#pragma unroll
                    for (int l = 0; l < L; l++) {
                        if (l == 0) {
                            s0.set(dv[u][0], k0v[u][0]);
                            s1.set(dv[u][0], k1v[u][0]);
                        } else {
                            s0.mac(dv[u][l], k0v[u][l]);
                            s1.mac(dv[u][l], k1v[u][l]);
                        }
                    }
                    z0 = s0.reduce_sf(q);
                    z1 = s1.reduce_sf(q);
                    if (has_c0) z0 = add_mod(z0, csub(shoup_lazy_sf(dv[u][L], pc.x, pc.y, q), q), q);
                }
                if (!PRE) {
                    zsm[kg_swz(pp, gl)] = z0 ^ 0x8080808080808080ull;
                    zsm[KG_PT * KG_KT + kg_swz(pp, gl)] = z1 ^ 0x8080808080808080ull;
                    continue;
                }
                // pre-mask form: the nb band masks of the tap (shared by both components) per K column
                const ulonglong2* mk = masks + (long long)tap[u] * nb * MN + jl;
                for (int beta = 0; beta < nb; beta++) {
                    u64 v0 = 0, v1 = 0;
                    if (kind[u]) {
                        const ulonglong2 m = __ldg(mk + (long long)beta * MN);
                        v0 = csub(shoup_lazy_sf(z0, m.x, m.y, q), q);
                        v1 = csub(shoup_lazy_sf(z1, m.x, m.y, q), q);
                    }
                    zsm[kg_swz(pp, gl * nb + beta)] = v0 ^ 0x8080808080808080ull;
                    zsm[KG_PT * KG_KT + kg_swz(pp, gl * nb + beta)] = v1 ^ 0x8080808080808080ull;
                }
            }
        }
    }
    __syncthreads();
    const int pp = threadIdx.x >> 3, ch = threadIdx.x & 7;
    if (K0 + ch * 16 >= Kp) return;
#pragma unroll 1
    for (int comp = 0; comp < 2; comp++) {
        const u64* zs = zsm + comp * KG_PT * KG_KT;
        const long long pos = (long long)comp * MN + jl0 + pp;
        uint32_t lo[16], hi[16];
#pragma unroll
        for (int w = 0; w < 16; w++) {
            const u64 v = zs[kg_swz(pp, ch * 16 + w)];
            lo[w] = (uint32_t)v;
            hi[w] = (uint32_t)(v >> 32);
        }
        uint32_t pl[8][4];
#pragma unroll
        for (int q4 = 0; q4 < 4; q4++) {
            uint32_t o[4];
            bytes4x4(lo[4 * q4], lo[4 * q4 + 1], lo[4 * q4 + 2], lo[4 * q4 + 3], o);
#pragma unroll
            for (int b = 0; b < 4; b++) pl[b][q4] = o[b];
            bytes4x4(hi[4 * q4], hi[4 * q4 + 1], hi[4 * q4 + 2], hi[4 * q4 + 3], o);
#pragma unroll
            for (int b = 0; b < 4; b++) pl[4 + b][q4] = o[b];
        }
        // tcgen05 tile layout: [tile = pos / 32][16-byte K chunk][256 rows (pos % 32, b)][16]
        int8_t* o = Bt + ((((pos >> 5) * (Kp >> 4) + (K0 >> 4) + ch) * 256) + 8 * (pos & 31)) * 16;
#pragma unroll
        for (int b = 0; b < 8; b++) *(uint4*)(o + b * 16) = make_uint4(pl[b][0], pl[b][1], pl[b][2], pl[b][3]);
    }
}

// sum_b (x_b + bias) 256^b (signed, |.| < 2^90) made non-negative with off (a multiple of q >= 2^90)
// and Montgomery-reduced once: returns (that sum) 2^-64 mod q.  Two 64-bit halves instead of a
// 128-bit shift chain.
__device__ __forceinline__ u64 kg_rec_redc(const uint32_t* x, long long bias, ulonglong2 off, const ModC& md)
{
    const long long b4 = bias * 0x01010101LL;
    const long long lo = (long long)(int32_t)x[0] + ((long long)(int32_t)x[1] << 8) + ((long long)(int32_t)x[2] << 16) +
                         ((long long)(int32_t)x[3] << 24) + b4;
    const long long hi = (long long)(int32_t)x[4] + ((long long)(int32_t)x[5] << 8) + ((long long)(int32_t)x[6] << 16) +
                         ((long long)(int32_t)x[7] << 24) + b4;
    const __int128 t = ((__int128)hi << 32) + (__int128)lo + (((__int128)off.x << 64) | (__int128)off.y);
    const unsigned __int128 u = (unsigned __int128)t;
    return csub(redc_lazy((u64)(u >> 64), (u64)u, md), md.q);
}

// ---------------------------------------------------------------------------
// Conv schedule 2 first-Add, fused on the 5th-generation tensor cores (tcgen05):
//   D[row][(pos, b)] = sum_K A[row][K] * Bt[8 pos + b][K]                           (int8 x int8 -> int32, TMEM)
//   post-mask form, rows (m, beta):  acc[m][pos] = sum_beta Mask[beta][pos] (.) rec(D[(m, beta)][(pos, 0..7)])
//   pre-mask form (masks already applied to the K columns by k_kg_zy), rows m:  acc[m][pos] = rec(D[m][(pos, 0..7)])
// all mod q_j.  The A and B K-chunks of each (128-row block, 256-column tile) job stream through a
// shared-memory ring; one lane issues the K/32 tcgen05.mma.kind::i8 (M = 128, N = 256, K = 32) from
// SWIZZLE_NONE K-major descriptors; 16 epilogue warps read TMEM with tcgen05.ld.32x32b.x32, rebuild
// each word mod q exactly, multiply by the band mask (or by 2^64 mod q_j in the pre-mask form) and
// sum the nb bands with warp shuffles.  No int32 GEMM output ever reaches HBM.

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t umma_desc_kmajor(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;   // descriptor version 1 (sm_100); base offset 0, SWIZZLE_NONE
    return d;
}

#ifdef KF_SUSPEND   // experiment: try_wait with a suspend-time hint (ns)
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t phase)
{
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(phase), "r"(KF_SUSPEND)
        : "memory");
    return ok != 0;
}
#else
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t phase)
{
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(phase)
        : "memory");
    return ok != 0;
}
#endif

// K-major, no swizzle: 16-byte chunk (row r, k-chunk c) at (r % 8) 16 + (r / 8) SBO + c 128, SBO = 8 Kp
__device__ __forceinline__ uint32_t kg_tc_off(int r, int c, int Kp) { return (r & 7) * 16 + (r >> 3) * 8 * Kp + c * 128; }

#define KG_TC_N 256
#define KG_TC_KCS 4          // 16-byte K chunks per pipeline stage (two K = 32 MMAs)
#define KG_TC_STAGES 4
#define KG_TC_EPI_WARPS 16
#define KG_TC_THREADS ((2 + KG_TC_EPI_WARPS) * 32)
// Warp-specialized persistent kernel (one CTA per SM, 512 TMEM columns = two 128 x 256 int32
// accumulators):
//   warp 0 (one lane): producer -- per stage one cp.async.bulk of the A chunks ([rb][chunk][128][16])
//                      and one of the B chunks ([tile][chunk][256][16]), completing on full[s];
//   warp 1 (one lane): MMA issuer -- waits full[s], issues tcgen05.mma.kind::i8 (M 128, N 256, K 32)
//                      from SWIZZLE_NONE K-major descriptors, commits empty[s]; after the last
//                      stage of a job commits tfull[acc];
//   warps 2..17:       epilogue -- stage the job's band masks in shared memory, wait tfull[acc],
//                      read TMEM (warp w: lanes 32 (w % 4), 8 words), rebuild each word mod q,
//                      multiply by the band mask, sum the nb bands with shuffles, store; arrive
//                      tempty[acc].
// Jobs = (tile, row block) pairs, row block fastest (consecutive jobs share the B tile in L2).
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity)
{
    while (!mbar_try_wait(smem_u32(b), parity)) {
    }
}
// a whole warp waits: lane 0 polls, the others hold at __syncwarp (no shared-memory spinning by 32 lanes:
// many polling warps starve the MMA issuer's own barrier traffic)
__device__ __forceinline__ void mbar_wait_warp(uint64_t* b, uint32_t parity)
{
    if ((threadIdx.x & 31) == 0) mbar_wait(b, parity);
    __syncwarp();
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* b)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
}

__global__ void __launch_bounds__(KG_TC_THREADS, 1) k_kg_tc(DevCtx c, const int8_t* __restrict__ Acan,
                                                           const int32_t* __restrict__ rowsum, int rows_real, int rbs,
                                                           int nb, int Mr, const int8_t* __restrict__ Bcan, int Kp,
                                                           int ntiles, const ulonglong2* __restrict__ off,
                                                           const ulonglong2* __restrict__ masks,
                                                           const ulonglong2* __restrict__ one, u64* __restrict__ accq,
                                                           int tiles_per_batch)
{
    extern __shared__ __align__(128) uint8_t kg_sm[];
    constexpr int STAGE_BYTES = KG_TC_KCS * (128 + KG_TC_N) * 16;
    uint8_t* ring = kg_sm;                                                   // [STAGES][A chunks | B chunks]
    ulonglong2* sMask = (ulonglong2*)(kg_sm + KG_TC_STAGES * STAGE_BYTES);  // [2][nb][32]
    __shared__ uint64_t full[KG_TC_STAGES], empty[KG_TC_STAGES], tfull[2], tempty[2];
    __shared__ uint32_t tmem_base_sh;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int KC = Kp / 16, nst = (KC + KG_TC_KCS - 1) / KG_TC_KCS;
    const long long jobs = (long long)ntiles * rbs;
    const long long per = (jobs + gridDim.x - 1) / gridDim.x;
    const long long j0 = blockIdx.x * per, j1 = j0 + per < jobs ? j0 + per : jobs;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(2 * KG_TC_N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 32) {
        for (int i = 0; i < KG_TC_STAGES; i++) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; i++) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], KG_TC_EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base_sh;
    if (warp == 0) {
        if (lane == 0) {   // producer
            int s = 0;
            uint32_t ph = 0;
            for (long long jb = j0; jb < j1; jb++) {
                const int rb = (int)(jb % rbs);
                const long long tile = jb / rbs;
                for (int g = 0; g < nst; g++) {
                    const int ch0 = g * KG_TC_KCS, n = KC - ch0 < KG_TC_KCS ? KC - ch0 : KG_TC_KCS;
                    mbar_wait(&empty[s], ph ^ 1);
                    uint8_t* st = ring + s * STAGE_BYTES;
                    mbar_expect_tx(&full[s], (uint32_t)(n * (128 + KG_TC_N) * 16));
                    bulk_g2s(st, Acan + ((long long)rb * KC + ch0) * 128 * 16, n * 128 * 16, &full[s]);
                    bulk_g2s(st + n * 128 * 16, Bcan + (tile * KC + ch0) * KG_TC_N * 16, n * KG_TC_N * 16, &full[s]);
                    if (++s == KG_TC_STAGES) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {   // MMA issuer
            const uint32_t idesc =
                (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(KG_TC_N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
            int s = 0;
            uint32_t ph = 0;
            int it = 0;
            for (long long jb = j0; jb < j1; jb++, it++) {
                const int acc = it & 1;
                const uint32_t tph = (uint32_t)((it >> 1) & 1);
                mbar_wait(&tempty[acc], tph ^ 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t d = tmem + (uint32_t)(acc * KG_TC_N);
                for (int g = 0; g < nst; g++) {
                    const int ch0 = g * KG_TC_KCS, n = KC - ch0 < KG_TC_KCS ? KC - ch0 : KG_TC_KCS;
                    mbar_wait(&full[s], ph);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t sa = smem_u32(ring + s * STAGE_BYTES), sb = sa + n * 128 * 16;
                    for (int kk = 0; kk < n / 2; kk++) {
                        const uint64_t ad = umma_desc_kmajor(sa + kk * 2 * 128 * 16, 128 * 16, 128);
                        const uint64_t bd = umma_desc_kmajor(sb + kk * 2 * KG_TC_N * 16, KG_TC_N * 16, 128);
                        const uint32_t accum = (g > 0 || kk > 0) ? 1u : 0u;
                        asm volatile(
                            "{\n\t.reg .pred p;\n\t"
                            "setp.ne.b32 p, %4, 0;\n\t"
                            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                            ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(accum));
                    }
                    umma_commit(&empty[s]);
                    if (++s == KG_TC_STAGES) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                umma_commit(&tfull[acc]);
            }
        }
    } else {   // epilogue warps
        const int ew = warp - 2, et = tid - 64;
        const int lg = warp & 3, cq = ew >> 2;                       // TMEM lane group (warp % 4), word quarter
        const int r = lg * 32 + lane;
        const int MN = c.M * c.N;
        const long long WQ = 2LL * MN;
        int it = 0;
        for (long long jb = j0; jb < j1; jb++, it++) {
            const int acc = it & 1;
            const int rb = (int)(jb % rbs);
            const long long tile = jb / rbs;
            const long long bat = tile / tiles_per_batch;                 // batch element of this tile
            const long long pos0 = (tile - bat * tiles_per_batch) * (KG_TC_N / 8);
            const int jl0 = (int)(pos0 % MN);
            ulonglong2* sm = sMask + acc * nb * 32;
            if (masks != nullptr) {
                for (int q = et; q < nb * 32; q += KG_TC_EPI_WARPS * 32)
                    sm[q] = __ldg(masks + (long long)(q >> 5) * MN + jl0 + (q & 31));
                asm volatile("bar.sync 1, %0;" ::"n"(KG_TC_EPI_WARPS * 32));
            }
            const int R = rb * 128 + r;
            const bool row_ok = R < rows_real;
            const int m = R / nb, beta = R - m * nb;
            const long long bias = row_ok ? 128LL * rowsum[R] : 0;
            const int jq = jl0 / c.N;                                // a tile never straddles a prime
            const ModC md = c.mod[jq];
            const ulonglong2 o = off[jq];
            const ulonglong2 one_j = one[jq];                        // pre-mask form: x 2^64 undoes the REDC
            mbar_wait(&tfull[acc], (uint32_t)((it >> 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll 1
            for (int h = 0; h < 2; h++) {
                const int p0 = cq * 8 + h * 4;
                uint32_t x[32];
                const uint32_t taddr = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(acc * KG_TC_N + 8 * p0);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
                    "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
                    : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]), "=r"(x[7]),
                      "=r"(x[8]), "=r"(x[9]), "=r"(x[10]), "=r"(x[11]), "=r"(x[12]), "=r"(x[13]), "=r"(x[14]), "=r"(x[15]),
                      "=r"(x[16]), "=r"(x[17]), "=r"(x[18]), "=r"(x[19]), "=r"(x[20]), "=r"(x[21]), "=r"(x[22]), "=r"(x[23]),
                      "=r"(x[24]), "=r"(x[25]), "=r"(x[26]), "=r"(x[27]), "=r"(x[28]), "=r"(x[29]), "=r"(x[30]), "=r"(x[31])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (h == 1) {   // this warp's TMEM reads of the job are done
                    asm volatile("tcgen05.fence::before_thread_sync;");
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[acc]);
                }
                u64 v[4];
#pragma unroll
                for (int w4 = 0; w4 < 4; w4++) {
                    v[w4] = 0;
                    if (row_ok) {
                        const u64 w = kg_rec_redc(x + 8 * w4, bias, o, md);
                        const ulonglong2 mk = masks != nullptr ? sm[beta * 32 + p0 + w4] : one_j;   // Montgomery-form mask
                        v[w4] = csub(shoup_lazy_sf(w, mk.x, mk.y, md.q), md.q);
                    }
                }
                // sum the nb band rows (lanes beta = 0..nb-1 of the group) as a reduce-scatter over
                // the 4 words: the first two rounds halve the words each lane carries
                u64* dstrow = accq + (bat * Mr + m) * WQ + pos0 + p0;
                const bool wr = row_ok && m < Mr;
                if (nb == 1) {
                    if (wr) {
                        *(ulonglong2*)dstrow = make_ulonglong2(v[0], v[1]);
                        *(ulonglong2*)(dstrow + 2) = make_ulonglong2(v[2], v[3]);
                    }
                } else {
                    const int sa = nb >> 1;
                    const bool ba = (beta & sa) != 0;
                    const u64 s0 = ba ? v[0] : v[2], s1 = ba ? v[1] : v[3];
                    const u64 r0 = __shfl_xor_sync(0xffffffffu, s0, sa), r1 = __shfl_xor_sync(0xffffffffu, s1, sa);
                    const u64 w0 = add_mod(ba ? v[2] : v[0], r0, md.q), w1 = add_mod(ba ? v[3] : v[1], r1, md.q);
                    if (nb == 2) {      // lane beta holds words 2 beta, 2 beta + 1
                        if (wr) *(ulonglong2*)(dstrow + (ba ? 2 : 0)) = make_ulonglong2(w0, w1);
                    } else {
                        const int sb = nb >> 2;
                        const bool bb = (beta & sb) != 0;
                        const u64 rr = __shfl_xor_sync(0xffffffffu, bb ? w0 : w1, sb);
                        u64 z = add_mod(bb ? w1 : w0, rr, md.q);
                        for (int sh = nb >> 3; sh >= 1; sh >>= 1) z = add_mod(z, __shfl_xor_sync(0xffffffffu, z, sh), md.q);
                        if (wr && (beta & (sb - 1)) == 0) dstrow[(ba ? 2 : 0) + (bb ? 1 : 0)] = z;
                    }
                }
            }
            // the mask buffer of this accumulator is rewritten two jobs later: all epilogue warps
            // are past it once they pass the next job's bar.sync
        }
    }
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * KG_TC_N));
}

// [rows_p][Kp] row-major -> [rows_p / 128][Kp / 16][128][16] (tcgen05 K-major core-matrix order)
__global__ void k_kg_tc_layout_a(const int8_t* __restrict__ A, int rows, int rows_p, int Kp, int8_t* __restrict__ out)
{
    const int KC = Kp / 16;
    const long long total = (long long)rows_p * KC;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(e % rows_p), ch = (int)(e / rows_p);
        uint4 v = make_uint4(0, 0, 0, 0);
        if (r < rows) v = *(const uint4*)(A + (long long)r * Kp + ch * 16);
        *(uint4*)(out + (((long long)(r >> 7) * KC + ch) * 128 + (r & 127)) * 16) = v;
    }
}

// Descriptor upload through the SMs from mapped pinned host memory (zero-copy reads over PCIe): the
// layers' small tables never queue on the copy engine behind large streamed input / output copies.
__global__ void k_h2d_copy(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst, long long words)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < words; i += (long long)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

// ---------------------------------------------------------------------------
// GALA schedule 2 on the tensor cores.  Per QP position p = (j, k) the baby-step sums are a small
// integer matrix product over the baby rotations jj:
//   Out[(s, bi)][g] = sum_jj X_s[bi][jj] w[g][jj],   X_0 = E_c0, X_1 = E_c1, X_2 = sigma_jj(c0)
// With 8-byte operands X = sum_a 256^a X_a, w = sum_b 256^b w_b:
//   Out = sum_s' 256^s' D_s',  D[(s, bi)][(g, s')] = sum_(jj, a) X_a[(s, bi)][jj] * w_(s' - a)[g][jj]
// -- one int8 MMA per position with A = the bytes of X in their natural little-endian order
// (K = (jj, a)), and B = the byte-convolution (Toeplitz) expansion of the weights (column
// (g, s'), 0 <= s' < 15).  D < 63 * 8 * 255^2 < 2^25 is exact in int32 and sum_s' 256^s' D_s' is
// the exact integer sum_jj X w < 2^126, reduced once mod q (w is in Montgomery form, so the REDC
// yields sum X w mod q).  Operands are stored in the tcgen05 SWIZZLE_NONE K-major core-matrix
// order: 16-byte chunk (row r, chunk kc) at (r / 8) 4096 + kc 128 + (r % 8) 16.
//   Ecan: chunk-major [kc][p][96 rows (s 32 + bi)][16 B] (48 KB per position); in shared memory the A
//         tile is [kc][row group][8][16 B] (LBO 1536, SBO 128), one 1.5 KB bulk copy per chunk
//   B tile: per position 16 row groups (rows g 16 + s', g < 8) = 64 KB, expanded in shared memory
#define GTC_A_BYTES (12 * 4096)
#define GTC_B_BYTES (16 * 4096)
__device__ __forceinline__ u64 bswap64(u64 w)
{
    const uint32_t lo = (uint32_t)w, hi = (uint32_t)(w >> 32);
    return ((u64)__byte_perm(lo, 0, 0x0123) << 32) | (u64)__byte_perm(hi, 0, 0x0123);
}

// Per position p, the weights one byte-convolution tile is built from (in shared memory, by k_gala_tc's
// expander warps): wT[p] = { bswap64(w[g b + jj][p]) for g < 8, jj < 64 ;  w[g b][p] for g < 8 }
// (Montgomery words, 0 outside g < G, jj < b): byte-reversed so an 8-byte window of the convolution is
// one shift, followed by the step-0 weights again (plain) for the step-0 product of the c1 stream.
// The jj = 0 column carries the step-0 member of the c0 stream into the MMA (its E rows are zero).
// 4160 bytes per position.
#define GTC_W_WORDS (8 * 64 + 8)
#define GTC_W_BYTES (GTC_W_WORDS * 8)
__global__ void k_gala_wt(DevCtx c, const u64* __restrict__ pts2, int baby, int G, u64* __restrict__ wT)
{
    const long long MN = (long long)c.M * c.N;
    const long long total = MN * GTC_W_WORDS;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e % GTC_W_WORDS);
        const long long p = e / GTC_W_WORDS;
        u64 v = 0;
        if (i < 512) {
            const int g = i >> 6, jj = i & 63;
            if (g < G && jj < baby) v = bswap64(__ldg(pts2 + (long long)(g * baby + jj) * MN + p));
        } else {
            const int g = i - 512;
            if (g < G) v = __ldg(pts2 + (long long)(g * baby) * MN + p);
        }
        wT[e] = v;
    }
}

// E_jj, sigma_jj(c0) for every (input, baby rotation jj = 0 .. 63), written as Ecan (k_gala_e's math;
// E_0 = 0 and sigma_0(c0) = c0 so the step-0 member of the c0 stream rides in the MMA).  grid (N / 32,
// 32 chunks, M), 256 threads: thread (position kk, 4 inputs) computes the two rotations of chunk kc.
template <int L>
__global__ void __launch_bounds__(256) k_gala_e_can(DevCtx c, const u64* __restrict__ Dblk, const u64* const* __restrict__ keys,
                                                    const unsigned* __restrict__ gal, int baby, int B, uint8_t* __restrict__ Ecan)
{
    __shared__ u64 sm[32][96][2];
    constexpr int M = L + 1;
    const int N = c.N, logN = c.logN;
    const int j = blockIdx.z, kc = blockIdx.y, k0 = blockIdx.x * 32;
    // warp w: rotation jj = 2 kc + (w >> 2), inputs 8 (w & 3) .. + 7 (the key limbs are loaded once
    // per thread and reused by 8 inputs)
    const int kk = threadIdx.x & 31, jw = threadIdx.x >> 7, bg = (threadIdx.x >> 5) & 3;
    const int k = k0 + kk;
    const u64 q = c.mod[j].q;
    // 32-bit word offsets (the digit blocks of a batch and a key are < 2^31 words): address arithmetic
    // stays on the integer ALU instead of 64-bit multiply-adds
    const uint32_t MN = (uint32_t)M * N, bw = (uint32_t)(L * M + L) * N;
    {
        const int jj = 2 * kc + jw;               // jj = 0: E = 0 (no key switch), sigma_0(c0) = c0
        const bool valid = jj >= 1 && jj < baby;
        u64 ka[L], kb[L];
        int src = k;
        if (valid) {
            const u64* key = keys[jj] + ((uint32_t)j * N + k);
            src = auto_src(k, gal[jj], logN);
#pragma unroll
            for (int i = 0; i < L; i++) {
                ka[i] = __ldg(key + (uint32_t)(2 * i) * MN);
                kb[i] = __ldg(key + (uint32_t)(2 * i + 1) * MN);
            }
        }
        uint32_t o = (uint32_t)(bg * 8) * bw + (uint32_t)j * N + src;
#pragma unroll
        for (int qi = 0; qi < 8; qi++, o += bw) {
            const int bi = bg * 8 + qi;
            const int r2 = 64 + bi + kk;
            // row r of position kk lives at (r + kk) % 96: the 32 positions of a warp hit distinct banks
            u64* s_e0 = &sm[kk][bi + kk][jw];
            u64* s_e1 = &sm[kk][32 + bi + kk][jw];
            u64* s_r0 = &sm[kk][r2 >= 96 ? r2 - 96 : r2][jw];
            if (valid && bi < B) {
                AccPP<true> s0, s1;   // L <= 4 canonical products per sum: merged cross sums fit
#pragma unroll
                for (int i = 0; i < L; i++) {
                    const u64 d = __ldg(Dblk + (o + (uint32_t)i * MN));
                    if (i == 0) {
                        s0.set(d, ka[i]);
                        s1.set(d, kb[i]);
                    } else {
                        s0.mac(d, ka[i]);
                        s1.mac(d, kb[i]);
                    }
                }
                *s_e0 = s0.reduce_sf(q);
                *s_e1 = s1.reduce_sf(q);
                *s_r0 = j < L ? __ldg(Dblk + (o + (uint32_t)L * MN)) : 0ull;
            } else {
                *s_e0 = 0;
                *s_e1 = 0;
                *s_r0 = (jj == 0 && bi < B && j < L) ? __ldg(Dblk + (o + (uint32_t)L * MN)) : 0ull;
            }
        }
    }
    __syncthreads();
    // chunk-major layout Ecan[kc][p][row 0..95][16 B]: the block's 32 positions are one contiguous 48 KB run
    uint8_t* dst = Ecan + ((long long)kc * MN + (long long)j * N + k0) * (96 * 16);
    for (int idx = threadIdx.x; idx < 32 * 96; idx += 256) {
        const int kk2 = idx / 96, r = idx - kk2 * 96, rr = r + kk2;
        *(ulonglong2*)(dst + (long long)idx * 16) = *(const ulonglong2*)&sm[kk2][rr >= 96 ? rr - 96 : rr][0];
    }
}

// The baby-step sums of every (input, group) at every position on the tensor cores.  Warp-specialized
// persistent kernel, one CTA per SM:
//   warp 0 lane 0  producer: per position one cp.async.bulk of the A tile (Ecan, 48 KB) and one of the
//                  raw weights (wT, 4 KB) into a 3-stage ring (full / empty mbarriers);
//   warps 10..13   expanders: build the position's byte-convolution B tile in two halves (groups
//                  0-3, 4-7; 32 KB each, double-buffered) from the raw weights (byte reversal +
//                  shift per 8-byte window), fence the generic -> async proxy, arrive bfull[h];
//   warp 1 lane 0  MMA: once both halves are built, 16 tcgen05.mma.kind::i8 (M 128, N 128, K 32,
//                  unsigned bytes) into one of two TMEM accumulators (N 128 reads the A tile from
//                  shared memory once per position, not once per half); commits bempty[0..1], then
//                  empty[s] and tfull[acc];
//   warps 2..9     epilogue (TMEM lane group s = warp % 4 -> stream s, lane = input; groups 4 gh ..
//                  4 gh + 3 with gh = (warp - 2) / 4, one 64-column TMEM load per position): rebuild
//                  each (input, stream, group) sum from its 15 byte-shifted columns, reduce once mod
//                  q, write U / Cacc (plus the step-0 member for stream 2).
#define GTC_THREADS 576
// A tiles stream in GTC_SPLIT stages per position (the same 96 KB of stages).  Measured: 1 (two
// whole-position stages) 0.469 ms per tile, 2 (half positions) 0.494, 4: 0.538 -- the MMAs do not wait
// on the A stream; more stages only add barrier traffic
#ifndef GTC_SPLIT
#define GTC_SPLIT 1
#endif
#define GTC_NST (2 * GTC_SPLIT)
#define GTC_STAGE (GTC_A_BYTES / GTC_SPLIT)
#define GTCF_NST 2                  // k_gala_tcf: whole-position stages written by the E warps
#define GTCF_STAGE GTC_A_BYTES
#define GTC_BB_BYTES (16 * 4096)   // 128 B rows (8 groups x 16 shifts; shift 15 is never read)
// + 512 B: the M 128 A read of the last stage runs past its 96 rows (rows 96..127 are don't-care)
#define GTC_SMEM (2 * GTC_BB_BYTES + GTC_NST * GTC_STAGE + 512)
#ifdef GTC_PROF
__device__ unsigned long long g_gtc_prof[1024][16];
#define GP_DECL long long gp_[16] = {0}; const long long gp_t0 = clock64();
#define GP_WAIT(slot, stmt) { const long long t_ = clock64(); stmt; gp_[slot] += clock64() - t_; }
#define GP_MARK(v) const long long v = clock64();
#define GP_ADD(slot, v) gp_[slot] += clock64() - v;
#define GP_FLUSH(first) if (lane == 0) { for (int i_ = 0; i_ < 16; i_++) if (gp_[i_] && i_ != 10 && i_ != 11) g_gtc_prof[blockIdx.x][i_] = gp_[i_]; if (first) { g_gtc_prof[blockIdx.x][10] = clock64() - gp_t0; g_gtc_prof[blockIdx.x][11] = p1 - p0; } }
#else
#define GP_DECL
#define GP_WAIT(slot, stmt) stmt;
#define GP_MARK(v)
#define GP_ADD(slot, v)
#define GP_FLUSH(first)
#endif
template <int L>
__global__ void __launch_bounds__(GTC_THREADS, 1) k_gala_tc(DevCtx c, const uint8_t* __restrict__ Ecan,
                                                          const u64* __restrict__ wT, const u64* __restrict__ X,
                                                          const u64* __restrict__ pts2, int baby, int G, int B,
                                                          u64* __restrict__ U, u64* __restrict__ Cacc)
{
    extern __shared__ __align__(128) uint8_t gtc_sm[];
    constexpr int M = L + 1;
    __shared__ uint64_t full[GTC_NST], empty[GTC_NST], tfull[2], tempty[2], bfull[2], bempty[2];
    __shared__ uint32_t tmem_base_sh;
    // step-0 weights w[g b][p] of the last 4 positions: copied from the raw stage by the expanders (before
    // the position's MMA), read by the epilogue (before it releases the accumulator).  Position p + 4's
    // copy waits on MMA p + 3, which waited on the epilogue of p + 1: the epilogue of p is done.
    __shared__ u64 s_w0[4][8];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int N = c.N;
    const long long MN = (long long)M * N, npos = MN;
    // whole blocks of 4 positions per CTA: the epilogue writes 4 consecutive words (one sector) per output
    const long long per = ((npos + gridDim.x - 1) / gridDim.x + 3) & ~3LL;
    const long long p0 = blockIdx.x * per, p1 = p0 + per < npos ? p0 + per : npos;
    // [B buffer 0][B buffer 1][A stages]
    uint8_t* sB = gtc_sm;
    uint8_t* sSt = gtc_sm + 2 * GTC_BB_BYTES;
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < GTC_NST; i++) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; i++) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 8);
            mbar_init(&bfull[i], 8);
            mbar_init(&bempty[i], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base_sh;
    GP_DECL
    if (warp == 0) {
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (long long p = p0; p < p1; p++) {
#pragma unroll 1
              for (int h = 0; h < GTC_SPLIT; h++) {
                GP_WAIT(0, mbar_wait(&empty[s], ph ^ 1));
                uint8_t* st = sSt + s * GTC_STAGE;
#ifdef GTC_NO_A   // probe (tools/tc_probe.sh): the MMA runs on stale A tiles
                (void)st;
                mbar_arrive(&full[s]);
#else
                mbar_expect_tx(&full[s], (uint32_t)GTC_STAGE);
                for (int i = 0; i < 32 / GTC_SPLIT; i++) {
                    const int kc = h * (32 / GTC_SPLIT) + i;
                    bulk_g2s(st + i * 1536, Ecan + ((long long)kc * npos + p) * 1536, 1536, &full[s]);
                }
#endif
                if (++s == GTC_NST) {
                    s = 0;
                    ph ^= 1;
                }
              }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // M 128, N 128 (both B halves: 8 groups x 16 shifts), s32 accumulate, unsigned bytes
            const uint32_t idesc = (2u << 4) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
            int s = 0;
            uint32_t ph = 0;
            int it = 0;
            for (long long p = p0; p < p1; p++, it++) {
                const int acc = it & 1;
                GP_WAIT(1, mbar_wait(&tempty[acc], (uint32_t)(((it >> 1) & 1) ^ 1)));
                const uint32_t sb = smem_u32(sB + acc * GTC_BB_BYTES);
                const uint32_t d = tmem + (uint32_t)(acc * 128);
#ifndef GTC_MMA_REPEAT
#define GTC_MMA_REPEAT 1   // probe: issue the position's MMAs this many times (MMA throughput)
#endif
#pragma unroll 1
                for (int h = 0; h < GTC_SPLIT; h++) {
                    GP_WAIT(2, mbar_wait(&full[s], ph));
                    const uint32_t sa = smem_u32(sSt + s * GTC_STAGE);
                    if (h == 0) GP_WAIT(3, mbar_wait(&bfull[acc], (uint32_t)((it >> 1) & 1)));
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    constexpr int KS = 16 / GTC_SPLIT;       // K = 32 MMAs per stage
#pragma unroll 1
                    for (int r = 0; r < KS * GTC_MMA_REPEAT; r++) {
                        const int ks = h * KS + (r % KS);
                        const uint64_t ad = umma_desc_kmajor(sa + (r % KS) * 2 * 1536, 1536, 128);
                        const uint64_t bd = umma_desc_kmajor(sb + ks * 256, 128, 4096);
                        const uint32_t accum = (h > 0 || r > 0) ? 1u : 0u;
                        asm volatile(
                            "{\n\t.reg .pred p;\n\t"
                            "setp.ne.b32 p, %4, 0;\n\t"
                            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                            ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(accum));
                    }
                    if (h == GTC_SPLIT - 1) umma_commit(&bempty[acc]);
                    umma_commit(&empty[s]);
                    if (++s == GTC_NST) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                umma_commit(&tfull[acc]);
            }
        }
    } else if (warp >= 10) {   // 8 expander warps: thread -> B row n = 16 g + s' x one K half
        const int et = tid - 10 * 32;
        const int n = et >> 1, kh = et & 1;
        const int g = n >> 4, sp = n & 15;
        const bool act = sp < 15;                 // row s' = 15 (column never read) is left as is
        // byte-reversed word r: window for shift s' is (r >> 8 (7 - s')) for s' <= 7, (r << 8 (s' - 7)) above
        const int sh_r = sp <= 7 ? 8 * (7 - sp) : 0, sh_l = sp > 7 ? 8 * (sp - 7) : 0;
        // the raw weights come from global memory straight into registers, one position ahead: the
        // expansion waits only for its B buffer, not for the position's A tile
        ulonglong2 r[16];
        u64 w0n = 0;
        auto load_raw = [&](long long pp) {
            if (pp >= p1) return;
            const ulonglong2* src = (const ulonglong2*)(wT + pp * GTC_W_WORDS) + g * 32 + kh * 16;
            if (act) {
#pragma unroll
                for (int i = 0; i < 16; i++) r[i] = __ldg(src + i);
            }
            if (et < 8) w0n = __ldg(wT + pp * GTC_W_WORDS + 512 + et);
        };
        load_raw(p0);
        int it = 0;
        for (long long p = p0; p < p1; p++, it++) {
            const int b = it & 1;
            GP_WAIT(6, mbar_wait(&bempty[b], (uint32_t)(((it >> 1) & 1) ^ 1)));
            GP_MARK(ex0)
            if (et < 8) s_w0[it & 3][et] = w0n;
#ifdef GTC_NO_B   // probe: no B-tile expansion (MMA on stale B)
            if (false) {
#else
            if (act) {
#endif
                uint8_t* rowbase = sB + b * GTC_BB_BYTES + (n >> 3) * 4096 + (n & 7) * 16 + kh * 16 * 128;
#pragma unroll
                for (int i = 0; i < 16; i++)   // rotations jj = 2 kc, 2 kc + 1 (byte-reversed), kc = 16 kh + i
                    *(ulonglong2*)(rowbase + i * 128) = make_ulonglong2((r[i].x >> sh_r) << sh_l, (r[i].y >> sh_r) << sh_l);
            }
            load_raw(p + 1);
            asm volatile("fence.proxy.async.shared::cta;");
            __syncwarp();
            if (lane == 0) mbar_arrive(&bfull[b]);
            GP_ADD(7, ex0)
        }
    } else {   // epilogue: TMEM lane group lg = warp % 4 holds rows 32 lg .. (stream s = lg, input = lane)
        const int lg = warp & 3, sidx = lg, bi = lane, gh = (warp - 2) >> 2;
        const long long W = 2LL * L * N;
        const long long gstride = sidx < 2 ? 2LL * M * N : 2LL * L * N;   // words between groups g, g + 1
        // sum_s' 256^s' D_s' of one group's 15 columns (exact, < 2^126) reduced mod q: three 40-bit-spaced
        // partial sums below 2^58, folded, one REDC (w Montgomery: the result is sum_jj X w mod q)
        auto rebuild = [&](const uint32_t* xg, const ModC& md) -> u64 {
            const u64 q = md.q;
            u64 lo5 = 0, mi5 = 0, hi5 = 0;
#pragma unroll
            for (int u = 0; u < 5; u++) {
                lo5 += (u64)xg[u] << (8 * u);
                mi5 += (u64)xg[5 + u] << (8 * u);
                hi5 += (u64)xg[10 + u] << (8 * u);
            }
            const u64 lo = lo5 + (mi5 << 40);
            u64 hi = (mi5 >> 24) + (hi5 << 16) + (lo < lo5 ? 1ull : 0ull);
            if (hi >= 2 * q) hi -= 2 * q;
            if (hi >= 2 * q) hi -= 2 * q;
            if (hi >= q) hi -= q;
            return csub(redc_lazy(hi, lo, md), q);
        };
        int it = 0;
        // blocks of 4 positions p = j N + k .. k + 3 (same prime: N % 4 == 0); one 32-byte store per output
        int j = (int)(p0 / N), k = (int)(p0 - (long long)j * N);
        for (long long p = p0; p < p1; p += 4) {
            const ModC md = c.mod[j];
            const bool active = (sidx < 2 || j < L) && bi < B;
            const long long z0 = (long long)bi * G + 4 * gh;
            u64* out0 = sidx == 3 ? Cacc + ((z0 * 2 + 1) * L + j) * (long long)N + k
                      : sidx < 2  ? U + ((z0 * 2 + sidx) * M + j) * (long long)N + k
                                  : Cacc + ((z0 * 2 + 0) * L + j) * (long long)N + k;
            // lane group 3 (no MMA rows): the step-0 product of the c1 stream, x.c1 (.) w[g b], on the CUDA cores
            ulonglong2 xa = make_ulonglong2(0, 0), xb = make_ulonglong2(0, 0);
            if (sidx == 3 && active) {
                const ulonglong2* xs = (const ulonglong2*)(X + (long long)bi * W + (long long)(L + j) * N + k);
                xa = __ldg(xs);
                xb = __ldg(xs + 1);
            }
            u64 res[4][4];
#pragma unroll
            for (int pi = 0; pi < 4; pi++, it++) {
                const int acc = it & 1;
                GP_WAIT(8, mbar_wait(&tfull[acc], (uint32_t)((it >> 1) & 1)));
                asm volatile("tcgen05.fence::after_thread_sync;");
                u64 w0[4];
#pragma unroll
                for (int t = 0; t < 4; t++) w0[t] = s_w0[it & 3][4 * gh + t];
                if (sidx == 3) {
                    asm volatile("tcgen05.fence::before_thread_sync;");
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[acc]);
                    const u64 xc1 = pi == 0 ? xa.x : pi == 1 ? xa.y : pi == 2 ? xb.x : xb.y;
#pragma unroll
                    for (int t = 0; t < 4; t++) res[pi][t] = mont_mul(xc1, w0[t], md);
                } else {
#ifdef GTC_NO_EPI   // probe: accumulator released without reading it
                    asm volatile("tcgen05.fence::before_thread_sync;");
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[acc]);
                    res[pi][0] = res[pi][1] = res[pi][2] = res[pi][3] = 0;
                    continue;
#endif
                    uint32_t x[32];
                    const uint32_t taddr = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(acc * 128 + gh * 64);
#pragma unroll
                    for (int hf = 0; hf < 2; hf++) {   // groups 2 hf, 2 hf + 1: columns 16 t .. 16 t + 14
                        asm volatile(
                            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
                            "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
                            "%30, %31}, [%32];"
                            : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]),
                              "=r"(x[7]), "=r"(x[8]), "=r"(x[9]), "=r"(x[10]), "=r"(x[11]), "=r"(x[12]), "=r"(x[13]),
                              "=r"(x[14]), "=r"(x[15]), "=r"(x[16]), "=r"(x[17]), "=r"(x[18]), "=r"(x[19]), "=r"(x[20]),
                              "=r"(x[21]), "=r"(x[22]), "=r"(x[23]), "=r"(x[24]), "=r"(x[25]), "=r"(x[26]), "=r"(x[27]),
                              "=r"(x[28]), "=r"(x[29]), "=r"(x[30]), "=r"(x[31])
                            : "r"(taddr + 32 * hf));
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                        if (hf == 1) {   // the accumulator columns of this warp are in registers
                            asm volatile("tcgen05.fence::before_thread_sync;");
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&tempty[acc]);
                        }
                        res[pi][2 * hf] = rebuild(x, md);
                        res[pi][2 * hf + 1] = rebuild(x + 16, md);
                    }
                }
            }
            if (active) {
#pragma unroll
                for (int t = 0; t < 4; t++)
                    if (4 * gh + t < G)
                        asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(out0 + t * gstride),
                                     "l"(res[0][t]), "l"(res[1][t]), "l"(res[2][t]), "l"(res[3][t])
                                     : "memory");
            }
            k += 4;
            if (k == N) {
                k = 0;
                j++;
            }
        }
    }
    if (warp == 0 || warp == 1 || warp == 2 || warp == 10) GP_FLUSH(warp == 0)
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

// ---------------------------------------------------------------------------
// GALA schedule 2, key-folded tensor-core baby steps (the production FC path).
//
// Group g's baby-step sum in component cc at QP position p = (j, k), for input b, is
//   U_cc[b][g][p] = sum_{jj >= 1} w_{g,jj}[p] E_cc,jj[b][p]  +  P [j < L] X_cc[b][g][p]
//   E_cc,jj = sum_i sigma_jj(D_i)[b][p] ksk_jj[i][cc][p],  X_0 = sum_jj w_{g,jj} sigma_jj(c0),  X_1 = w_{g,0} c1
// (the split form k_gala_e_can / k_gala_tc keeps X in a separate Q-side addend Cacc; P X is the same
// addend lifted into QP: ModDown(Y + P X) = ModDown(Y) + X exactly, so the words do not change).  The key
// limbs and P do not depend on the input, so they fold into the weights:
//   U_cc[b][g][p] = sum_{jj < 64, st < 4} A[b][jj][st][p] Wk[p][cc][jj][g][st]
//   A[b][jj][st] = sigma_jj(D_st)[b] (st < L),  sigma_jj(c0)[b] (st = 3, j < L),  0 otherwise
//   Wk[cc][jj][g][i] = ksk_jj[i][cc] w_{g,jj} (jj >= 1),  Wk[1][0][g][j] = P w_{g,0},  Wk[0][jj][g][3] = P w_{g,jj}
// (mod q_j, Montgomery).  Per position that is one integer matrix product, M = 256 inputs, N = 2 x 8
// outputs, K = 64 rotations x 4 streams, exact as a byte convolution on the int8 tensor cores:
//   D[b][(cc, g, s')] = sum_(jj, st, a) A_a[b][(jj, st)] * w_(s' - a)[(cc, g)][(jj, st)],   value = sum_s' 256^s' D_s'
// with A in natural little-endian byte order (K = (jj, st, a), 32 bytes per rotation) and B the
// byte-shift (Toeplitz) expansion of the folded weights.  Every column D_s' < 2048 * 255^2 < 2^27 is exact
// in int32; the value is rebuilt mod q_j from three 40-bit-spaced partial sums and one REDC.
// E_jj never exists: the kernel streams the digit blocks (8 KB per position, read 64 times from L2 --
// positions run prime by prime across the grid so a prime's blocks stay resident) and the folded
// weights (32 KB per position, once per tile of 256 inputs).
#define KF_W_WORDS (2 * 64 * 8 * 4)     // folded weights per position: [cc][jj][g][st], byte-reversed words
#define KF_W_BYTES (KF_W_WORDS * 8)
__device__ __forceinline__ u64 mad_wide_u32(uint32_t a, uint32_t b, u64 c)
{
    u64 r;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(a), "r"(b), "l"(c));
    return r;
}
// 32 consecutive TMEM columns of the warp's lane group into registers (completion: tcgen05.wait::ld)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* x)
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
        "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
        "%30, %31}, [%32];"
        : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]),
          "=r"(x[7]), "=r"(x[8]), "=r"(x[9]), "=r"(x[10]), "=r"(x[11]), "=r"(x[12]), "=r"(x[13]),
          "=r"(x[14]), "=r"(x[15]), "=r"(x[16]), "=r"(x[17]), "=r"(x[18]), "=r"(x[19]), "=r"(x[20]),
          "=r"(x[21]), "=r"(x[22]), "=r"(x[23]), "=r"(x[24]), "=r"(x[25]), "=r"(x[26]), "=r"(x[27]),
          "=r"(x[28]), "=r"(x[29]), "=r"(x[30]), "=r"(x[31])
        : "r"(taddr));
}

// Wk from the schedule-2 plaintexts (pts2 [T][M][N], Montgomery, sigma_jj pre-applied) and the baby-step
// rotation keys ([L][2][M][N] per step, keys[jj]); pmod[j] = P mod q_j.  Zero outside g < G, jj < baby.
template <int L>
__global__ void k_gala_kfw(DevCtx c, const u64* __restrict__ pts2, const u64* const* __restrict__ keys,
                           const u64* __restrict__ pmod, int baby, int G, u64* __restrict__ Wk)
{
    constexpr int M = L + 1;
    const long long MN = (long long)M * c.N;
    const long long total = MN * KF_W_WORDS;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e % KF_W_WORDS);
        const long long p = e / KF_W_WORDS;
        const int st = i & 3, g = (i >> 2) & 7, jj = (i >> 5) & 63, cc = i >> 11;
        const int j = (int)(p / c.N);
        u64 v = 0;
        if (g < G && jj < baby) {
            const ModC md = c.mod[j];
            const u64 w = __ldg(pts2 + (long long)(g * baby + jj) * MN + p);
            const u64 pm = mont_mul(__ldg(pmod + j), md.r2, md);     // P R mod q_j
            if (st < L) {
                if (jj >= 1) v = mont_mul(__ldg(keys[jj] + (long long)(2 * st + cc) * MN + p), w, md);
                else if (cc == 1 && st == j) v = mont_mul(w, pm, md);
            } else if (st == 3 && cc == 0 && j < L) {
                v = mont_mul(w, pm, md);
            }
        }
        Wk[e] = bswap64(v);
    }
}

// A operand of one tile of <= 256 inputs, in rotation-orbit order.  The baby rotations are sigma_jj = sigma^jj
// (Galois element 3^jj), and in the NTT domain sigma moves slot k to sigma(k) = auto_src(k, 3); the slots of
// a prime fall into two orbits x_0, x_1 = sigma(x_0), ... of length N / 2.  Position x_t needs the digit
// blocks of x_t, x_t+1, ..., x_t+63 -- a contiguous run when the blocks are stored in orbit order, so a
// pipeline stage of KF_JS rotations is ONE bulk copy (the TMA services bulk copies ~one at a time per SM,
// ~350 clk each: one 4 KB copy per rotation capped the gather at ~12 B/clk).  Each orbit is padded with
// its first 64 blocks again (no wrap-around).  Layout: Dq[j][orbit][half][t][4 KB], half h = inputs
// 128 h .. 128 h + 127 (read by the CTA of rank h of a pair), each 4 KB block the tcgen05 K-major
// core-matrix order [kc][row group][8][16 B] of 128 rows x 32 bytes (streams D_0, D_1, D_2, c0; rows >= B
// and absent streams zero).  orb[k] = orbit * KF_ORB(N) + t.  grid (M N / KF_DQ_POS), 256 threads.
#define KF_ROWS 256
#define KF_DQ_BYTES (KF_ROWS * 32)
#define KF_ORB(N) ((N) / 2 + 64)
#define KF_DQ_POS 8
#define KF_DQ_STRIDE (KF_DQ_BYTES + 16)        // padded per-position stride in shared memory (bank spread)
template <int L>
__global__ void __launch_bounds__(256) k_gala_dq(DevCtx c, const u64* __restrict__ Dblk, int B, const int* __restrict__ orb,
                                                 uint8_t* __restrict__ Dq)
{
    extern __shared__ __align__(16) uint8_t dq_sm[];
    constexpr int M = L + 1;
    const int N = c.N, ORB = KF_ORB(N);
    const long long p0 = (long long)blockIdx.x * KF_DQ_POS;
    const int j = (int)(p0 / N), k0 = (int)(p0 - (long long)j * N);
    const long long bw = (long long)(L * M + L) * N;
    for (int idx = threadIdx.x; idx < KF_ROWS * 4 * KF_DQ_POS; idx += blockDim.x) {
        const int kl = idx % KF_DQ_POS, st = (idx / KF_DQ_POS) & 3, b = idx / (4 * KF_DQ_POS);
        int slot = -1;
        if (st < L) slot = st * M + j;
        else if (st == 3 && j < L) slot = L * M + j;
        u64 v = 0;
        if (b < B && slot >= 0) v = __ldg(Dblk + b * bw + (long long)slot * N + k0 + kl);
        *(u64*)(dq_sm + kl * KF_DQ_STRIDE + (b >> 7) * 4096 + (st >> 1) * 2048 + ((b & 127) >> 3) * 128 + (b & 7) * 16 +
                (st & 1) * 8) = v;
    }
    __syncthreads();
    // position k0 + kl -> orbit slot (and its padding copy); 16-byte chunks, half-major within the block
    for (int idx = threadIdx.x; idx < KF_DQ_POS * (KF_DQ_BYTES / 16); idx += blockDim.x) {
        const int kl = idx / (KF_DQ_BYTES / 16), w = idx % (KF_DQ_BYTES / 16), h = w >> 8, off = (w & 255) * 16;
        const int ot = __ldg(orb + k0 + kl), o = ot / ORB, t = ot - o * ORB;
        const uint4 v = *(const uint4*)(dq_sm + kl * KF_DQ_STRIDE + h * 4096 + off);
        uint8_t* base = Dq + (((long long)(j * 2 + o) * 2 + h) * ORB) * 4096 + off;
        *(uint4*)(base + (long long)t * 4096) = v;
        if (t < 64) *(uint4*)(base + (long long)(t + N / 2) * 4096) = v;
    }
}
#define KF_DQ_SMEM (KF_DQ_POS * KF_DQ_STRIDE)

// bulk copy with an L2 eviction-priority policy (createpolicy)
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* b, uint64_t pol)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)), "l"(pol) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_last()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// Position order of k_gala_kf: blocks of 4 consecutive slots, prime by prime and, within a prime, orbit by
// orbit (orbit 0 = slots with bit logN - 2 clear: k in [0, N/4) and [N/2, 3N/4)), so that the digit
// blocks in use at any time are one orbit's (34 MB for 256 inputs), not a prime's.  Returns the first
// position j N + k of block `blk`.
__device__ __forceinline__ long long kf_block_pos(long long blk, int N)
{
    const int q4 = N / 4, q8 = N / 8, q16 = N / 16;
    const long long j = blk / q4;
    const int r = (int)(blk - j * q4), o = r / q8, r2 = r - o * q8;
    const int kb = (r2 / q16) * q8 + o * q16 + (r2 % q16);
    return j * N + 4LL * kb;
}
// cluster helpers (CTA pairs)
__device__ __forceinline__ uint32_t cluster_rank()
{
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank)
{
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr)
{
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* b, uint32_t parity)
{
    uint32_t ok = 0;
    while (!ok)
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
}
__device__ __forceinline__ void cluster_sync_all()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// commit the issuing thread's prior MMAs to the same barrier in both CTAs of the pair
__device__ __forceinline__ void umma_commit_pair(uint64_t* b)
{
    const uint16_t mask = 3;
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(smem_u32(b)), "h"(mask) : "memory");
}

// The key-folded baby-step sums of a tile of <= 256 inputs on CTA pairs (cta_group::2).  The pair's MMA
// is M = 256 (rank r holds inputs 128 r .. 128 r + 127 of A and its accumulator rows), N = 256 (rank r
// holds the B rows of component cc = r: 8 groups x 16 shifts), K = 32 per rotation; each CTA's TMEM has
// two 256-column accumulators (positions alternate).  Cluster c of the grid takes position blocks
// (4 consecutive k) c, c + clusters, ... -- the whole grid sweeps the primes in order.  Per CTA:
//   warp 0 lane 0   producer: its component's folded weights in chunks of KF_WJ rotations (4 KB, two
//                   chunks ahead) and, per stage of KF_JS rotations, its half of the stage's digit blocks
//                   sigma_jj(p) -- consecutive in orbit order: one KF_JS x 4 KB bulk copy;
//   warp 1 lane 0   rank 0: the MMA issuer -- per stage ONE wait (full[s]: both CTAs' stage complete),
//                   KF_JS tcgen05.mma.cta_group::2.kind::i8, ONE commit multicast to both CTAs' empty[s];
//                   rank 1: relay -- waits its own full[s] and arrives on rank 0's full[s];
//   warps 2..5      expanders: thread = B row (g, s') of component cc = rank; per rotation the 4 streams'
//                   8-byte windows (byte reversal + shift) of the folded weights;
//   warps 6..13     epilogue: TMEM lane group warp % 4 (lane = input), component (warp - 6) / 4: rebuild the
//                   8 group sums mod q_j, one 32-byte store per output per 4 positions; the accumulator's
//                   release (tempty, counted on rank 0) comes from both CTAs' epilogues.
// Why this shape (measured, profiles/r2_experiments.md): a thread cannot keep the tensor pipe fed
// through fine-grained mbarrier waits and every role pays a fixed cost per stage (tools/mma_bench.cu,
// tools/kf_trace.py), so stages carry several MMAs; the TMA services one 1-D bulk copy per SM in a
// roughly fixed time whatever its size (tools/bulk_bench.cu: 4 KB ~6-8 B/clk, 32 KB ~50 B/clk), so a
// stage's digit blocks move as ONE 32 KB copy (8 rotations: 5.2 -> 3.0 ms per 256-input tile against
// 4-rotation stages; separate, deeper A and B rings measured slower); the pair halves each SM's Toeplitz expansion and
// shared-memory bytes per MMA (A 4 KB + B 4 KB), leaving room for KF_ST stages and for two accumulators
// (the epilogue of position p overlaps the MMAs of p + 1).  (14 warps: <= 4 per SM sub-partition.)
#ifndef KF_JS
#define KF_JS 8                          // rotations per stage: one 32 KB A copy (tools/bulk_bench.cu)
#endif
#ifndef KF_ST
#define KF_ST 3                          // ring depth
#endif
#ifndef KF_WJ
#define KF_WJ 32                         // rotations per folded-weight chunk (8 KB per component)
#endif
#ifndef KF_WST
#define KF_WST 2
#endif
#define KF_WCH_BYTES (KF_WJ * 256)       // one component's weights for KF_WJ rotations
#define KF_A_STAGE (KF_JS * 4096)
#define KF_B_STAGE (KF_JS * 4096)
#define KF_SMEM (KF_ST * (KF_A_STAGE + KF_B_STAGE) + KF_WST * KF_WCH_BYTES)
#ifndef KF_NO_WSPLIT   // the folded-weight copies from a 15th warp: a second TMA-issuing thread (2.95 vs 3.05 ms)
#define KF_WSPLIT
#endif
#ifdef KF_WSPLIT
#define KF_THREADS (15 * 32)
#else
#define KF_THREADS (14 * 32)
#endif
#define KF_EPI0 6
#ifdef KF_TRACE   // timeline of CTA 0 (tools/kf_trace.py): [event][index] clock64 stamps
__device__ unsigned long long g_kf_trace[32][1024];
#ifndef KF_TRACE_CTA
#define KF_TRACE_CTA 0
#endif
#define KF_T(ev, idx) do { if (blockIdx.x == KF_TRACE_CTA && (idx) < 1024) g_kf_trace[ev][idx] = clock64(); } while (0)
#else
#define KF_T(ev, idx) do { } while (0)
#endif
// Experiment (-DKF_FLAG, off): stage hand-off to the MMA issuer through shared-memory counters instead of
// mbarriers.  A thread that waits on an mbarrier after issuing tcgen05.mma stalls until its MMAs drain
// (tools/mma2_bench.cu: a commit/wait ring runs 230 clk per M128 N256 K32 MMA per SM instead of 128; with
// the waits done by a helper thread that publishes counters, 144), but in k_gala_kf the counters measured
// slower (3.10 vs 2.95 ms per tile; the MMA-only probe 2.44 vs 2.48): the issuer's waits are not what
// paces this kernel (profiles/r2_experiments.md).
#if defined(KF_FLAG) && !defined(KF_WSPLIT)
#error "KF_FLAG runs its helper in lane 1 of the weight-producer warp (KF_WSPLIT)"
#endif
__device__ __forceinline__ void kf_publish(uint32_t* p, uint32_t v)
{
    asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ void kf_await(const uint32_t* p, uint32_t v)
{
    uint32_t x;
    do {
#ifdef KF_FLAG_VOLATILE
        asm volatile("ld.volatile.shared::cta.u32 %0, [%1];" : "=r"(x) : "r"(smem_u32(p)) : "memory");
#else
        asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(x) : "r"(smem_u32(p)) : "memory");
#endif
    } while ((int)(x - v) < 0);
}
template <int L>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(KF_THREADS, 1)
k_gala_kf(DevCtx c, const uint8_t* __restrict__ Dq, const u64* __restrict__ Wk, const int* __restrict__ orb,
          int baby, int G, int B, u64* __restrict__ U)
{
    extern __shared__ __align__(128) uint8_t kf_sm[];
    constexpr int M = L + 1;
    __shared__ uint64_t full[KF_ST], empty[KF_ST], wfull[KF_WST], wempty[KF_WST], tfull[2], tempty[2];
    __shared__ uint32_t tmem_base_sh;
    __shared__ uint32_t s_ready, s_tready;   // KF_FLAG: stages / accumulators published to the issuer
    __shared__ u64 s_c80[M];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = cluster_rank();
    const int N = c.N, ORB = KF_ORB(N);
    const long long nblk = (long long)M * N / 4;
    const long long cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    const int nst = (baby + KF_JS - 1) / KF_JS;          // stages per position (rotations >= baby: zero weights)
    uint8_t* sA = kf_sm;
    uint8_t* sB = kf_sm + KF_ST * KF_A_STAGE;
    uint8_t* sW = sB + KF_ST * KF_B_STAGE;
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < KF_ST; i++) {
            // rank 0: own producer (expect_tx) + 4 own expander warps + rank 1's relay; rank 1: 1 + 4
            mbar_init(&full[i], rank == 0 ? 1 + 4 + 1 : 1 + 4);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < KF_WST; i++) {
            mbar_init(&wfull[i], 1);
            mbar_init(&wempty[i], 4);
        }
        for (int i = 0; i < 2; i++) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 16);       // rank 0's: 8 epilogue warps of each CTA
        }
        s_ready = 0;
        s_tready = 0;
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (tid < M) {   // 2^80 mod q_j for the rebuild
        const u64 q = c.mod[tid].q;
        u64 v = 1;
        for (int i = 0; i < 80; i++) v = add_mod(v, v, q);
        s_c80[tid] = v;
    }
    // B rows s' = 15 are never written by the expanders: zero every B stage once
    for (int i = tid; i < KF_ST * KF_B_STAGE / 16; i += blockDim.x) ((uint4*)sB)[i] = make_uint4(0, 0, 0, 0);
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();                  // barriers initialised in both CTAs before any remote arrive
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base_sh;
#ifdef KF_FLAG
    if (warp == KF_THREADS / 32 - 1 && lane == 1 && rank == 0) {
        // the issuer's hand-off helper: in the issuer's order, each accumulator's release (tempty) and each
        // stage's completion (full: both CTAs' copies and expanders) become counters the issuer polls
        int sa = 0, it = 0;
        uint32_t pha = 0;
        uint32_t gs = 0;
        for (long long blk = cid; blk < nblk; blk += ncl) {
            for (int pi = 0; pi < 4; pi++, it++) {
                mbar_wait_cluster(&tempty[it & 1], (uint32_t)(((it >> 1) & 1) ^ 1));
                kf_publish(&s_tready, (uint32_t)(it + 1));
                for (int s = 0; s < nst; s++) {
                    mbar_wait_cluster(&full[sa], pha);
                    kf_publish(&s_ready, ++gs);
                    if (++sa == KF_ST) {
                        sa = 0;
                        pha ^= 1;
                    }
                }
            }
        }
    } else
#endif
    if (warp == 0 || warp == 14) {
        if (lane == 0) {
            int sa = 0, ws = 0;
            uint32_t pha = 0, phw = 0;
            // L2: the digit blocks of the current prime are re-read 64 times (keep), the weights stream (once)
            const uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();
            const int nch = (nst * KF_JS + KF_WJ - 1) / KF_WJ;            // weight chunks per position
            const long long npos = nblk > cid ? ((nblk - 1 - cid) / ncl + 1) * 4 : 0;
            const long long wtotal = npos * nch;
            long long wnext = 0;                                         // next weight chunk to issue
            auto issue_w_upto = [&](long long last) {                     // chunks [wnext, last]
                for (; wnext <= last && wnext < wtotal; wnext++) {
                    const long long itw = wnext / nch;
                    const int ch = (int)(wnext - itw * nch);
                    const long long pw = kf_block_pos(cid + (itw >> 2) * ncl, N) + (itw & 3);
                    mbar_wait(&wempty[ws], phw ^ 1);
#ifdef KF_NO_W   // probe builds (tools/kf_probe.sh): role isolation, results are garbage
                    mbar_arrive(&wfull[ws]);
#else
                    mbar_expect_tx(&wfull[ws], (uint32_t)KF_WCH_BYTES);
                    bulk_g2s_hint(sW + ws * KF_WCH_BYTES,
                                  (const uint8_t*)(Wk + pw * KF_W_WORDS) + rank * (KF_W_BYTES / 2) + ch * KF_WCH_BYTES,
                                  KF_WCH_BYTES, &wfull[ws], pol_stream);
#endif
                    if (++ws == KF_WST) {
                        ws = 0;
                        phw ^= 1;
                    }
                }
            };
            if (warp == 14) {   // KF_WSPLIT: every weight chunk, in order, as the ring frees
                issue_w_upto(wtotal - 1);
            } else {
            long long itp = 0;
            for (long long blk = cid; blk < nblk; blk += ncl) {
                for (int pi = 0; pi < 4; pi++, itp++) {
                    const long long p = kf_block_pos(blk, N) + pi;
                    const int j = (int)(p / N), k = (int)(p - (long long)j * N);
                    const int ot = __ldg(orb + k), o = ot / ORB, t = ot - o * ORB;
                    // this CTA's half of the orbit run x_t, x_t+1, ... of prime j
                    const uint8_t* run = Dq + ((((long long)(j * 2 + o) * 2 + rank) * ORB) + t) * 4096;
                    for (int s = 0; s < nst; s++) {
#ifndef KF_WSPLIT
                        issue_w_upto(itp * nch + (s * KF_JS) / KF_WJ + KF_WST - 2);   // 2 chunks ahead, 1 slot of slack
#endif
                        mbar_wait(&empty[sa], pha ^ 1);
                        KF_T(2, itp * nst + s);
#ifdef KF_NO_A
                        mbar_arrive(&full[sa]);
#else
                        mbar_expect_tx(&full[sa], (uint32_t)KF_A_STAGE);
                        bulk_g2s_hint(sA + sa * KF_A_STAGE, run + (long long)s * KF_A_STAGE, KF_A_STAGE, &full[sa], pol_keep);
#endif
                        KF_T(3, itp * nst + s);
                        if (++sa == KF_ST) {
                            sa = 0;
                            pha ^= 1;
                        }
                    }
                }
            }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {   // the pair's MMA issuer
            // M 256 (cta_group::2), N 256, s32 accumulate, unsigned bytes
            const uint32_t idesc = (2u << 4) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
            int sa = 0, it = 0;
            uint32_t pha = 0;
            long long gs = 0;
            for (long long blk = cid; blk < nblk; blk += ncl) {
                for (int pi = 0; pi < 4; pi++, it++) {
                    const int acc = it & 1;
#ifdef KF_FLAG
                    kf_await(&s_tready, (uint32_t)(it + 1));
#else
                    mbar_wait_cluster(&tempty[acc], (uint32_t)(((it >> 1) & 1) ^ 1));
#endif
                    KF_T(6, it);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t d = tmem + (uint32_t)(acc * 256);
                    for (int s = 0; s < nst; s++, gs++) {
                        KF_T(9, gs);
#ifdef KF_FLAG
                        kf_await(&s_ready, (uint32_t)(gs + 1));
#else
                        mbar_wait_cluster(&full[sa], pha);
#endif
                        KF_T(0, gs);
                        asm volatile("tcgen05.fence::after_thread_sync;");
                        const uint32_t a0 = smem_u32(sA + sa * KF_A_STAGE), b0 = smem_u32(sB + sa * KF_B_STAGE);
#pragma unroll
                        for (int jl = 0; jl < KF_JS; jl++) {
                            const uint64_t ad = umma_desc_kmajor(a0 + jl * 4096, 2048, 128);
                            const uint64_t bd = umma_desc_kmajor(b0 + jl * 4096, 2048, 128);
                            const uint32_t accum = (s | jl) ? 1u : 0u;
                            asm volatile(
                                "{\n\t.reg .pred p;\n\t"
                                "setp.ne.b32 p, %4, 0;\n\t"
                                "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                                ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(accum));
                        }
                        umma_commit_pair(&empty[sa]);
                        KF_T(1, gs);
                        if (++sa == KF_ST) {
                            sa = 0;
                            pha ^= 1;
                        }
                    }
                    umma_commit_pair(&tfull[acc]);
                }
            }
        } else if (lane == 0) {   // rank 1: relay its stages' completion to the issuer's barrier
            const uint32_t peer_full0 = mapa_shared(smem_u32(&full[0]), 0);
            int sa = 0;
            uint32_t pha = 0;
            long long gr = 0;
            for (long long blk = cid; blk < nblk; blk += ncl)
                for (int pi = 0; pi < 4; pi++)
                    for (int s = 0; s < nst; s++, gr++) {
                        mbar_wait(&full[sa], pha);
                        KF_T(4, gr);
                        mbar_arrive_remote(peer_full0 + (uint32_t)(sa * sizeof(uint64_t)));
                        if (++sa == KF_ST) {
                            sa = 0;
                            pha ^= 1;
                        }
                    }
        }
    } else if (warp < KF_EPI0) {   // expanders: thread = B row n = 16 g + s' of component cc = rank
        const int n = tid - 64;
        const int sp = n & 15, g = n >> 4;
        const bool act = sp < 15;
        const int sh_r = sp <= 7 ? 8 * (7 - sp) : 0, sh_l = sp > 7 ? 8 * (sp - 7) : 0;
        int sb = 0, ws = 0;
        long long gse = 0;
        uint32_t phb = 0, phw = 0;
        for (long long blk = cid; blk < nblk; blk += ncl) {
            for (int pi = 0; pi < 4; pi++) {
                for (int s = 0; s < nst; s++, gse++) {
                    const int jw0 = (s * KF_JS) % KF_WJ;     // first rotation of the stage within its weight chunk
                    if (jw0 == 0) mbar_wait(&wfull[ws], phw);
                    if (lane == 0) KF_T(20 + warp - 2, gse);
                    mbar_wait(&empty[sb], phb ^ 1);
                    if (lane == 0) KF_T(16 + warp - 2, gse);
#ifdef KF_NO_B
                    if (false) {
#else
                    if (act) {
#endif
                        const uint8_t* wsrc = sW + ws * KF_WCH_BYTES + g * 32 + jw0 * 256;
                        uint8_t* dst = sB + sb * KF_B_STAGE + n * 16;
                        ulonglong2 r[KF_JS][2];
#pragma unroll
                        for (int jl = 0; jl < KF_JS; jl++) {
                            const ulonglong2* src = (const ulonglong2*)(wsrc + jl * 256);
                            r[jl][0] = src[0];
                            r[jl][1] = src[1];
                        }
#pragma unroll
                        for (int jl = 0; jl < KF_JS; jl++) {
                            uint8_t* o = dst + jl * 4096;
                            const ulonglong2 r0 = r[jl][0], r1 = r[jl][1];
                            *(ulonglong2*)o = make_ulonglong2((r0.x >> sh_r) << sh_l, (r0.y >> sh_r) << sh_l);
                            *(ulonglong2*)(o + 2048) = make_ulonglong2((r1.x >> sh_r) << sh_l, (r1.y >> sh_r) << sh_l);
                        }
                    }
                    asm volatile("fence.proxy.async.shared::cta;");
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&full[sb]);
                    if (lane == 0) KF_T(12 + warp - 2, gse);
                    if (++sb == KF_ST) {
                        sb = 0;
                        phb ^= 1;
                    }
                    if (jw0 + KF_JS == KF_WJ || s == nst - 1) {   // weight chunk consumed
                        if (lane == 0) mbar_arrive(&wempty[ws]);
                        if (++ws == KF_WST) {
                            ws = 0;
                            phw ^= 1;
                        }
                    }
                }
            }
        }
    } else {   // epilogue
        const int lg = warp & 3, cc = (warp - KF_EPI0) >> 2, b = (int)rank * 128 + lg * 32 + lane;
        const bool active = b < B;
        const uint32_t tempty0 = mapa_shared(smem_u32(&tempty[0]), 0);
        const uint64_t pol_out = policy_evict_first();   // U is read back by the next kernels, not by this one
        int it = 0;
        for (long long blk = cid; blk < nblk; blk += ncl) {
            const long long p = kf_block_pos(blk, N);
            const int j = (int)(p / N), k = (int)(p - (long long)j * N);
            const u64 q = c.mod[j].q, c80 = s_c80[j];
            auto rebuild = [&](const uint32_t* x) -> u64 {
                // three 40-bit-spaced partial sums: one IMAD.WIDE.U32 per column for 256^u < 2^32 (x < 2^27),
                // the 256^4 column added into the high word
                u64 lo5 = x[0], mi5 = x[5], hi5 = x[10];
#pragma unroll
                for (int u = 1; u < 4; u++) {
                    lo5 = mad_wide_u32(x[u], 1u << (8 * u), lo5);
                    mi5 = mad_wide_u32(x[5 + u], 1u << (8 * u), mi5);
                    hi5 = mad_wide_u32(x[10 + u], 1u << (8 * u), hi5);
                }
                lo5 += (u64)x[4] << 32;
                mi5 += (u64)x[9] << 32;
                hi5 += (u64)x[14] << 32;
                // value = lo5 + 2^40 mi5 + 2^80 hi5 == (lo5 + 2^40 mi5) + c80 hi5 (mod q): the first part is
                // < 2^100, the product < 2^59 q, the sum < 2^62 q (REDC input bound q 2^64)
                u64 lo = hi5 * c80, hi = __umul64hi(hi5, c80);
                const u64 m = mi5 << 40;
                lo += m;
                hi += (mi5 >> 24) + (lo < m ? 1ull : 0ull);
                lo += lo5;
                hi += lo < lo5 ? 1ull : 0ull;
                return csub(redc_sf_lazy(hi, lo, q), q);
            };
            u64 res[4][8];
#pragma unroll
            for (int pi = 0; pi < 4; pi++, it++) {
                const int acc = it & 1;
                mbar_wait(&tfull[acc], (uint32_t)((it >> 1) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t taddr = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(acc * 256 + cc * 128);
#ifdef KF_NO_EPI
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) mbar_arrive_remote(tempty0 + (uint32_t)(acc * sizeof(uint64_t)));
                for (int h = 0; h < 8; h++) res[pi][h] = taddr;
                continue;
#endif
#pragma unroll
                for (int h = 0; h < 4; h++) {
                    uint32_t x[32];
                    tmem_ld32(taddr + 32 * h, x);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    if (h == 3) {   // this warp's accumulator columns are in registers
                        asm volatile("tcgen05.fence::before_thread_sync;");
                        __syncwarp();
                        if (lane == 0) mbar_arrive_remote(tempty0 + (uint32_t)(acc * sizeof(uint64_t)));
                        if (warp == KF_EPI0 && lane == 0) KF_T(8, it);
                    }
                    res[pi][2 * h] = rebuild(x);
                    res[pi][2 * h + 1] = rebuild(x + 16);
                }
            }
            if (active) {
                // the group-sum layout of u_quad_base: a warp's 32 lanes (inputs) write one 1 KB run per group
                // (position-contiguous rows put every lane in another row -- 32 L1 wavefronts per store, whose
                // bursts stalled the other roles' mbarrier traffic: MMA-only probe 2.43 -> 1.93 ms without them)
                u64* out0 = U + u_quad_base(b, 0, cc, j, G, M, N) + u_quad_off(k);
                const long long gstride = 2LL * M * N * 256;
#pragma unroll
                for (int g = 0; g < 8; g++)
                    if (g < G)
                        asm volatile("st.global.L2::cache_hint.v4.u64 [%0], {%1, %2, %3, %4}, %5;" ::"l"(out0 + g * gstride),
                                     "l"(res[0][g]), "l"(res[1][g]), "l"(res[2][g]), "l"(res[3][g]), "l"(pol_out)
                                     : "memory");
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();                  // no CTA leaves while its pair may still read its smem / barriers
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// ---------------------------------------------------------------------------
// Fused schedule-2 baby steps: the E_jj key products computed straight into the tcgen05 A stage.
//
// k_gala_tc above reads its A tiles (E_jj, sigma_jj(c0) as bytes) from Ecan, which k_gala_e_can
// writes: 1.5 GB out and 1.75 GB back per 32-input tile, the largest HBM round trip of the FC step.
// k_gala_tcf computes the A tile of each position in shared memory instead.  E warps (lane = input
// bi of the tile, one warp per K chunk kc = (jj = 2 kc, 2 kc + 1)) form
//     E_jj[c] = sum_i sigma_jj(D_i)[p] ksk_jj[i][c][p]       (AccPP partial products, one REDC)
// and sigma_jj(c0)[p], and store them as the three 16-byte rows (c0 stream, c1 stream, x.c0 stream)
// of chunk kc in the core-matrix layout; 32 lanes write 512 contiguous bytes.  The digit blocks of
// the tile are read input-minor (Dt[slot][k][32], k_gala_dt) so a warp's gather of sigma_jj(k) for
// its 32 inputs is one coalesced 256-byte load.  The MMA lane, expanders and epilogue are
// k_gala_tc's; the stage's full barrier counts the E warps' arrivals instead of TMA bytes.
//
// Dblk [b][(L M + L)][N] of the tile's inputs -> Dt [(L M + L)][N][32] (inputs >= B zero)
__global__ void k_gala_dt(DevCtx c, const u64* __restrict__ Dblk, int B, u64* __restrict__ Dt)
{
    __shared__ u64 t[32][33];
    const int N = c.N;
    const long long bw = (long long)(c.L * c.M + c.L) * N;
    const long long nk = bw / 32;   // 32-word column blocks over (slot, k)
    const int x = threadIdx.x & 31, y = threadIdx.x >> 5;     // 256 threads: 8 rows per pass
    for (long long blk = blockIdx.x; blk < nk; blk += gridDim.x) {
        const long long w0 = blk * 32;
        for (int b = y; b < 32; b += 8) t[b][x] = b < B ? __ldcs((const unsigned long long*)(Dblk + b * bw + w0 + x)) : 0ull;
        __syncthreads();
        for (int kk = y; kk < 32; kk += 8) Dt[(w0 + kk) * 32 + x] = t[x][kk];
        __syncthreads();
    }
}

// keys of the baby rotations position-major: Kt[p][jj][6] = (k_0^0, k_0^1, k_1^0, k_1^1, k_2^0, k_2^1) of
// ksk_jj (digit i, component c) at position p -- an E warp's keys for one chunk are 96 contiguous bytes
// (zero for jj = 0 and jj >= baby)
template <int L>
__global__ void k_gala_kt(DevCtx c, const u64* const* __restrict__ keys, int baby, u64* __restrict__ Kt)
{
    const long long MN = (long long)c.M * c.N;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < MN * 64; e += (long long)gridDim.x * blockDim.x) {
        const int jj = (int)(e / MN);
        const long long p = e - jj * MN;
        u64 v[2 * L];
#pragma unroll
        for (int w = 0; w < 2 * L; w++) v[w] = (jj >= 1 && jj < baby) ? __ldg(keys[jj] + w * MN + p) : 0ull;
        u64* o = Kt + (p * 64 + jj) * (2 * L);
#pragma unroll
        for (int w = 0; w < 2 * L; w++) o[w] = v[w];
    }
}

#ifndef GTCF_NE
#define GTCF_NE 7                          // E warps (24 warps in all: 6 per SM sub-partition)
#endif
#define GTCF_WARPS (18 + GTCF_NE - 1)            // warp 0 + warps 18.. are E warps
#define GTCF_THREADS (GTCF_WARPS * 32)
// registers are allocated per SM sub-partition (16384 each, warps dealt round-robin)
#define GTCF_MAXREG ((16384 / (((GTCF_WARPS + 3) / 4) * 32)) & ~7)
template <int L>
__global__ void __maxnreg__(GTCF_MAXREG) k_gala_tcf(DevCtx c, const u64* __restrict__ Dt,
                                                             const u64* __restrict__ Kt,
                                                             const unsigned* __restrict__ gal,
                                                             const u64* __restrict__ wT, const u64* __restrict__ X,
                                                             int baby, int G, int B,
                                                             u64* __restrict__ U, u64* __restrict__ Cacc)
{
    extern __shared__ __align__(128) uint8_t gtc_sm[];
    constexpr int M = L + 1;
    __shared__ uint64_t full[GTCF_NST], empty[GTCF_NST], tfull[2], tempty[2], bfull[2], bempty[2];
    __shared__ uint32_t tmem_base_sh;
    __shared__ u64 s_w0[4][8];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int N = c.N, logN = c.logN;
    const long long MN = (long long)M * N, npos = MN;
    const long long per = ((npos + gridDim.x - 1) / gridDim.x + 3) & ~3LL;
    const long long p0 = blockIdx.x * per, p1 = p0 + per < npos ? p0 + per : npos;
    uint8_t* sB = gtc_sm;
    uint8_t* sSt = gtc_sm + 2 * GTC_BB_BYTES;
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < GTCF_NST; i++) {
            mbar_init(&full[i], GTCF_NE);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; i++) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 8);
            mbar_init(&bfull[i], 8);
            mbar_init(&bempty[i], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base_sh;
    if (warp == 0 || warp >= 18) {   // E warps: lane = input bi, chunks kc = ew, ew + NE, ...
        constexpr int NCH = (32 + GTCF_NE - 1) / GTCF_NE;
        const int ew = warp == 0 ? 0 : warp - 17;
        const int nch = (32 - ew + GTCF_NE - 1) / GTCF_NE;   // this warp's chunks
        const int bi = lane;
        const uint32_t NN = (uint32_t)N;
        // keys of the warp's chunks at one position: lane l < 6 L holds word l % (2 L) of jj = 2 kc + l / (2 L)
        u64 kcur[NCH], knext[NCH];
        auto load_keys = [&](long long pp, u64* kr) {
#pragma unroll
            for (int ci = 0; ci < NCH; ci++) {
                const int kc = ew + ci * GTCF_NE;
                kr[ci] = (ci < nch && lane < 4 * L) ? __ldg(Kt + (pp * 64 + 2 * kc) * (2 * L) + lane) : 0ull;
            }
        };
        // the chunk's gathered words: d[h][i] = sigma_jj(D_i)[p], d[h][L] = sigma_jj(c0)[p]
        auto load_d = [&](int kc, int j, int k, u64 (*d)[L + 1]) {
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int jj = 2 * kc + h;
                const bool ok = jj < baby && bi < B;
                const int src = jj == 0 ? k : auto_src(k, gal[jj < baby ? jj : 0], logN);
#pragma unroll
                for (int i = 0; i <= L; i++) {
                    const uint32_t slot = i < L ? (uint32_t)(i * M + j) : (uint32_t)(L * M + j);
                    const bool need = ok && (i < L ? jj >= 1 : j < L);
                    d[h][i] = need ? __ldg(Dt + ((slot * NN + (uint32_t)src) * 32u + (uint32_t)bi)) : 0ull;
                }
            }
        };
        int s = 0;
        uint32_t ph = 0;
        int j = (int)(p0 / N), k = (int)(p0 - (long long)j * N);
        if (p0 < p1) load_keys(p0, kcur);
        for (long long p = p0; p < p1; p++) {
            const u64 q = c.mod[j].q;
            if (p + 1 < p1) load_keys(p + 1, knext);
            u64 da[2][L + 1], db[2][L + 1];
            load_d(ew, j, k, da);
            mbar_wait(&empty[s], ph ^ 1);
            uint8_t* st = sSt + s * GTCF_STAGE;
#pragma unroll
            for (int ci = 0; ci < NCH; ci++) {
                if (ci >= nch) break;
                const int kc = ew + ci * GTCF_NE;
                if (ci + 1 < nch) load_d(kc + GTCF_NE, j, k, (ci & 1) ? da : db);
                u64 (*d)[L + 1] = (ci & 1) ? db : da;
                u64 e0[2], e1[2];
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    AccPP<true> s0, s1;
#pragma unroll
                    for (int i = 0; i < L; i++) {
                        const u64 ka = __shfl_sync(0xffffffffu, kcur[ci], h * 2 * L + 2 * i);
                        const u64 kb = __shfl_sync(0xffffffffu, kcur[ci], h * 2 * L + 2 * i + 1);
                        if (i == 0) {
                            s0.set(d[h][i], ka);
                            s1.set(d[h][i], kb);
                        } else {
                            s0.mac(d[h][i], ka);
                            s1.mac(d[h][i], kb);
                        }
                    }
                    e0[h] = s0.reduce_sf(q);   // zero keys (jj = 0, jj >= baby) and zero digits give 0
                    e1[h] = s1.reduce_sf(q);
                }
                // rows r = stream 32 + bi of chunk kc: (r / 8) 128 + (r % 8) 16 within the chunk's 1.5 KB
                uint8_t* cb = st + kc * 1536 + (bi >> 3) * 128 + (bi & 7) * 16;
                *(ulonglong2*)(cb) = make_ulonglong2(e0[0], e0[1]);
                *(ulonglong2*)(cb + 512) = make_ulonglong2(e1[0], e1[1]);
                *(ulonglong2*)(cb + 1024) = make_ulonglong2(d[0][L], d[1][L]);
            }
            asm volatile("fence.proxy.async.shared::cta;");
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[s]);
            if (++s == GTCF_NST) {
                s = 0;
                ph ^= 1;
            }
            if (++k == N) {
                k = 0;
                j++;
            }
#pragma unroll
            for (int ci = 0; ci < NCH; ci++) kcur[ci] = knext[ci];
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t idesc = (2u << 4) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
            int s = 0;
            uint32_t ph = 0;
            int it = 0;
            for (long long p = p0; p < p1; p++, it++) {
                const int acc = it & 1;
                mbar_wait(&tempty[acc], (uint32_t)(((it >> 1) & 1) ^ 1));
                mbar_wait(&full[s], ph);
                const uint32_t sa = smem_u32(sSt + s * GTCF_STAGE);
                mbar_wait(&bfull[acc], (uint32_t)((it >> 1) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t sb = smem_u32(sB + acc * GTC_BB_BYTES);
                const uint32_t d = tmem + (uint32_t)(acc * 128);
#pragma unroll 1
                for (int ks = 0; ks < 16; ks++) {
                    const uint64_t ad = umma_desc_kmajor(sa + ks * 2 * 1536, 1536, 128);
                    const uint64_t bd = umma_desc_kmajor(sb + ks * 256, 128, 4096);
                    asm volatile(
                        "{\n\t.reg .pred p;\n\t"
                        "setp.ne.b32 p, %4, 0;\n\t"
                        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                        ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(ks));
                }
                umma_commit(&bempty[acc]);
                umma_commit(&empty[s]);
                umma_commit(&tfull[acc]);
                if (++s == GTCF_NST) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
    } else if (warp >= 10) {   // 8 expander warps (k_gala_tc's)
        const int et = tid - 10 * 32;
        const int n = et >> 1, kh = et & 1;
        const int g = n >> 4, sp = n & 15;
        const bool act = sp < 15;
        const int sh_r = sp <= 7 ? 8 * (7 - sp) : 0, sh_l = sp > 7 ? 8 * (sp - 7) : 0;
        ulonglong2 r[16];
        u64 w0n = 0;
        auto load_raw = [&](long long pp) {
            if (pp >= p1) return;
            const ulonglong2* src = (const ulonglong2*)(wT + pp * GTC_W_WORDS) + g * 32 + kh * 16;
            if (act) {
#pragma unroll
                for (int i = 0; i < 16; i++) r[i] = __ldg(src + i);
            }
            if (et < 8) w0n = __ldg(wT + pp * GTC_W_WORDS + 512 + et);
        };
        load_raw(p0);
        int it = 0;
        for (long long p = p0; p < p1; p++, it++) {
            const int b = it & 1;
            mbar_wait(&bempty[b], (uint32_t)(((it >> 1) & 1) ^ 1));
            if (et < 8) s_w0[it & 3][et] = w0n;
            if (act) {
                uint8_t* rowbase = sB + b * GTC_BB_BYTES + (n >> 3) * 4096 + (n & 7) * 16 + kh * 16 * 128;
#pragma unroll
                for (int i = 0; i < 16; i++)
                    *(ulonglong2*)(rowbase + i * 128) = make_ulonglong2((r[i].x >> sh_r) << sh_l, (r[i].y >> sh_r) << sh_l);
            }
            load_raw(p + 1);
            asm volatile("fence.proxy.async.shared::cta;");
            __syncwarp();
            if (lane == 0) mbar_arrive(&bfull[b]);
        }
    } else {   // epilogue warps 2..9 (k_gala_tc's)
        const int lg = warp & 3, sidx = lg, bi = lane, gh = (warp - 2) >> 2;
        const long long W = 2LL * L * N;
        const long long gstride = sidx < 2 ? 2LL * M * N : 2LL * L * N;
        auto rebuild = [&](const uint32_t* xg, const ModC& md) -> u64 {
            const u64 q = md.q;
            u64 lo5 = 0, mi5 = 0, hi5 = 0;
#pragma unroll
            for (int u = 0; u < 5; u++) {
                lo5 += (u64)xg[u] << (8 * u);
                mi5 += (u64)xg[5 + u] << (8 * u);
                hi5 += (u64)xg[10 + u] << (8 * u);
            }
            const u64 lo = lo5 + (mi5 << 40);
            u64 hi = (mi5 >> 24) + (hi5 << 16) + (lo < lo5 ? 1ull : 0ull);
            if (hi >= 2 * q) hi -= 2 * q;
            if (hi >= 2 * q) hi -= 2 * q;
            if (hi >= q) hi -= q;
            return csub(redc_lazy(hi, lo, md), q);
        };
        int it = 0;
        int j = (int)(p0 / N), k = (int)(p0 - (long long)j * N);
        for (long long p = p0; p < p1; p += 4) {
            const ModC md = c.mod[j];
            const bool active = (sidx < 2 || j < L) && bi < B;
            const long long z0 = (long long)bi * G + 4 * gh;
            u64* out0 = sidx == 3 ? Cacc + ((z0 * 2 + 1) * L + j) * (long long)N + k
                      : sidx < 2  ? U + ((z0 * 2 + sidx) * M + j) * (long long)N + k
                                  : Cacc + ((z0 * 2 + 0) * L + j) * (long long)N + k;
            ulonglong2 xa = make_ulonglong2(0, 0), xb = make_ulonglong2(0, 0);
            if (sidx == 3 && active) {
                const ulonglong2* xs = (const ulonglong2*)(X + (long long)bi * W + (long long)(L + j) * N + k);
                xa = __ldg(xs);
                xb = __ldg(xs + 1);
            }
            u64 res[4][4];
#pragma unroll
            for (int pi = 0; pi < 4; pi++, it++) {
                const int acc = it & 1;
                mbar_wait(&tfull[acc], (uint32_t)((it >> 1) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;");
                u64 w0[4];
#pragma unroll
                for (int t = 0; t < 4; t++) w0[t] = s_w0[it & 3][4 * gh + t];
                if (sidx == 3) {
                    asm volatile("tcgen05.fence::before_thread_sync;");
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[acc]);
                    const u64 xc1 = pi == 0 ? xa.x : pi == 1 ? xa.y : pi == 2 ? xb.x : xb.y;
#pragma unroll
                    for (int t = 0; t < 4; t++) res[pi][t] = mont_mul(xc1, w0[t], md);
                } else {
                    uint32_t x[32];
                    const uint32_t taddr = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(acc * 128 + gh * 64);
#pragma unroll
                    for (int hf = 0; hf < 2; hf++) {
                        asm volatile(
                            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
                            "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
                            "%30, %31}, [%32];"
                            : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]),
                              "=r"(x[7]), "=r"(x[8]), "=r"(x[9]), "=r"(x[10]), "=r"(x[11]), "=r"(x[12]), "=r"(x[13]),
                              "=r"(x[14]), "=r"(x[15]), "=r"(x[16]), "=r"(x[17]), "=r"(x[18]), "=r"(x[19]), "=r"(x[20]),
                              "=r"(x[21]), "=r"(x[22]), "=r"(x[23]), "=r"(x[24]), "=r"(x[25]), "=r"(x[26]), "=r"(x[27]),
                              "=r"(x[28]), "=r"(x[29]), "=r"(x[30]), "=r"(x[31])
                            : "r"(taddr + 32 * hf));
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                        if (hf == 1) {
                            asm volatile("tcgen05.fence::before_thread_sync;");
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&tempty[acc]);
                        }
                        res[pi][2 * hf] = rebuild(x, md);
                        res[pi][2 * hf + 1] = rebuild(x + 16, md);
                    }
                }
            }
            if (active) {
#pragma unroll
                for (int t = 0; t < 4; t++)
                    if (4 * gh + t < G)
                        asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(out0 + t * gstride),
                                     "l"(res[0][t]), "l"(res[1][t]), "l"(res[2][t]), "l"(res[3][t])
                                     : "memory");
            }
            k += 4;
            if (k == N) {
                k = 0;
                j++;
            }
        }
    }
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

// ---------------------------------------------------------------------------
// Conv schedule 1 first-Add on the tensor cores.  Per Q position p = (j, x):
//   acc[r][comp] = sum_w R[comp][w] pt[r][w]      (r = o c_n + d, w = ib k + tap)
// with 8-byte operands is, as in k_gala_tc, one int8 byte-convolution MMA per position:
//   D[r][(comp, s')] = sum_(w, a) pt_a[r][w] R_(s' - a)[comp][w],   acc = sum_s' 256^s' D_s'
// A = the plaintext bytes (streamed from HBM in K-chunk stages: PTcan[p][kc][Rp rows][16 B]),
// B = the byte-convolution expansion of the position's rotated inputs (32 rows (comp, s')), built
// in shared memory from Rt[p][comp][w].  The exact sum can exceed 2^128, so the rebuild folds three
// 40-bit-spaced partial sums with 2^40 and 2^80 mod q before one REDC (pt is Montgomery: the REDC
// yields sum R pt mod q; K <= 1024 words keeps every partial below 2^64 and the fold below 2^124).
// Same words as k_kg_accumulate.
#define KG1_GK 8            // 16-byte K chunks per A stage
#define KG1_NST 4
#define KG1_THREADS 320     // warp 0 producer, 1 MMA, 2..5 epilogue, 6..9 expanders

// pts [n_obp][n_ib][c_n][k][L][N] (Montgomery) -> PTcan [p][KC][Rp][16 B], row r = o c_n + d, word w = ib k + t
__global__ void k_kg1_pt_can(DevCtx c, const u64* __restrict__ pts, int n_obp, int n_ib, int c_n, int k, int Rp, int KC,
                             u64* __restrict__ out)
{
    const int N = c.N, L = c.L;
    const long long P = (long long)L * N, LN = (long long)L * N;
    const long long per_p = (long long)KC * Rp * 2;            // words per position
    const long long total = P * per_p;
    const int Kw = n_ib * k, Mr = n_obp * c_n;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
        const long long p = e / per_p;
        const int rem = (int)(e - p * per_p);
        const int kc = rem / (Rp * 2), r = (rem / 2) % Rp, half = rem & 1;
        const int w = 2 * kc + half;
        u64 v = 0;
        if (r < Mr && w < Kw) {
            const int o = r / c_n, d = r - o * c_n, ib = w / k, t = w - ib * k;
            v = __ldg(pts + ((((long long)o * n_ib + ib) * c_n + d) * k + t) * LN + p);
        }
        out[e] = v;
    }
}

// R [ib][t][2][L][N] -> Rt[p][comp][Kwp] (byte-reversed for the expansion; zero padding)
__global__ void k_kg1_rt(DevCtx c, const u64* __restrict__ R, int Kw, int Kwp, u64* __restrict__ Rt)
{
    const int N = c.N, L = c.L;
    const long long LN = (long long)L * N, W = 2 * LN;
    const long long total = LN * 2 * Kwp;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
        const int w = (int)(e % Kwp);
        const long long pc = e / Kwp;
        const int comp = (int)(pc & 1);
        const long long p = pc >> 1;
        Rt[e] = w < Kw ? bswap64(__ldg(R + (long long)w * W + comp * LN + p)) : 0ull;
    }
}

template <int MT>
__global__ void __launch_bounds__(KG1_THREADS, 1) k_kg1_tc(DevCtx c, const uint8_t* __restrict__ PTcan,
                                                          const u64* __restrict__ Rt, int Mr, int Kwp,
                                                          u64* __restrict__ acc)
{
    extern __shared__ __align__(128) uint8_t k1_sm[];
    constexpr int Rp = MT * 128;
    constexpr int STAGE = KG1_GK * Rp * 16;
    const int KC = Kwp / 2, nst = KC / KG1_GK;
    const int BBYTES = KC * 32 * 16, RAW = 2 * Kwp * 8;
    uint8_t* ring = k1_sm;                                   // [KG1_NST][STAGE]
    uint8_t* sB = k1_sm + KG1_NST * STAGE;                   // [2][BBYTES]
    uint8_t* sRaw = sB + 2 * BBYTES;                         // [2][RAW]
    __shared__ uint64_t full[KG1_NST], empty[KG1_NST], rfull[2], rempty[2], bfull[2], bempty[2], tfull[2], tempty[2];
    __shared__ uint32_t tmem_base_sh;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int N = c.N, L = c.L;
    const long long P = (long long)L * N;
    const long long per = (P + gridDim.x - 1) / gridDim.x;
    const long long p0 = blockIdx.x * per, p1 = p0 + per < P ? p0 + per : P;
    constexpr uint32_t TCOLS = 2 * MT * 32 <= 32 ? 32 : (2 * MT * 32 <= 64 ? 64 : (2 * MT * 32 <= 128 ? 128 : 256));
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)), "r"(TCOLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < KG1_NST; i++) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; i++) {
            mbar_init(&rfull[i], 1);
            mbar_init(&rempty[i], 4);
            mbar_init(&bfull[i], 4);
            mbar_init(&bempty[i], 1);
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base_sh;
    if (warp == 0) {
        if (lane == 0) {   // producer: raw rotated inputs per position, plaintext K-chunk stages
            int s = 0;
            uint32_t ph = 0;
            int it = 0;
            for (long long p = p0; p < p1; p++, it++) {
                const int b = it & 1;
                mbar_wait(&rempty[b], (uint32_t)(((it >> 1) & 1) ^ 1));
                mbar_expect_tx(&rfull[b], (uint32_t)RAW);
                bulk_g2s(sRaw + b * RAW, Rt + p * 2 * Kwp, RAW, &rfull[b]);
                for (int g = 0; g < nst; g++) {
                    mbar_wait(&empty[s], ph ^ 1);
                    mbar_expect_tx(&full[s], (uint32_t)STAGE);
                    bulk_g2s(ring + s * STAGE, PTcan + (p * KC + (long long)g * KG1_GK) * Rp * 16, STAGE, &full[s]);
                    if (++s == KG1_NST) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {   // MMA issuer
            const uint32_t idesc = (2u << 4) | ((uint32_t)(32 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
            int s = 0;
            uint32_t ph = 0;
            int it = 0;
            for (long long p = p0; p < p1; p++, it++) {
                const int a = it & 1;
                mbar_wait(&tempty[a], (uint32_t)(((it >> 1) & 1) ^ 1));
                mbar_wait(&bfull[a], (uint32_t)((it >> 1) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t sb = smem_u32(sB + a * BBYTES);
                for (int g = 0; g < nst; g++) {
                    mbar_wait(&full[s], ph);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t sa = smem_u32(ring + s * STAGE);
#pragma unroll
                    for (int mt = 0; mt < MT; mt++) {
                        const uint32_t d = tmem + (uint32_t)((a * MT + mt) * 32);
#pragma unroll
                        for (int kk = 0; kk < KG1_GK / 2; kk++) {
                            const uint64_t ad = umma_desc_kmajor(sa + kk * 2 * Rp * 16 + mt * 128 * 16, Rp * 16, 128);
                            const uint64_t bd = umma_desc_kmajor(sb + (g * KG1_GK + kk * 2) * 512, 512, 128);
                            const uint32_t accum = (g > 0 || kk > 0) ? 1u : 0u;
                            asm volatile(
                                "{\n\t.reg .pred p;\n\t"
                                "setp.ne.b32 p, %4, 0;\n\t"
                                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
                                ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(accum));
                        }
                    }
                    umma_commit(&empty[s]);
                    if (++s == KG1_NST) {
                        s = 0;
                        ph ^= 1;
                    }
                }
                umma_commit(&bempty[a]);
                umma_commit(&tfull[a]);
            }
        }
    } else if (warp >= 6) {   // expanders: B row n = (comp, s'), thread -> (row, chunk subset)
        const int et = tid - 6 * 32;
        const int n = et & 31, part = et >> 5;                  // 4 parts over the K chunks
        const int comp = n >> 4, sp = n & 15;
        const int sh_r = sp <= 7 ? 8 * (7 - sp) : 0, sh_l = sp > 7 ? (sp == 15 ? 0 : 8 * (sp - 7)) : 0;
        const u64 keep = sp == 15 ? 0ull : ~0ull;
        int it = 0;
        for (long long p = p0; p < p1; p++, it++) {
            const int b = it & 1;
            mbar_wait(&rfull[b], (uint32_t)((it >> 1) & 1));
            mbar_wait(&bempty[b], (uint32_t)(((it >> 1) & 1) ^ 1));
            const ulonglong2* raw = (const ulonglong2*)(sRaw + b * RAW) + comp * (Kwp / 2);
            uint8_t* rowbase = sB + b * BBYTES + (n >> 3) * 128 + (n & 7) * 16;
            for (int kc = part; kc < KC; kc += 4) {
                const ulonglong2 r = raw[kc];                   // words w = 2 kc, 2 kc + 1 (byte-reversed)
                const u64 t0 = ((r.x >> sh_r) << sh_l) & keep, t1 = ((r.y >> sh_r) << sh_l) & keep;
                *(ulonglong2*)(rowbase + kc * 512) = make_ulonglong2(t0, t1);
            }
            asm volatile("fence.proxy.async.shared::cta;");
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&bfull[b]);
                mbar_arrive(&rempty[b]);
            }
        }
    } else {   // epilogue: lane group lg = warp % 4 -> rows 32 lg + lane of every M tile
        const int lg = warp & 3;
        const long long LN = (long long)L * N;
        int it = 0;
        for (long long p = p0; p < p1; p++, it++) {
            const int a = it & 1;
            const int j = (int)(p / N);
            const ModC md = c.mod[j];
            const u64 q = md.q;
            const u64 c40 = (u64)(((unsigned __int128)1 << 40) % q), c80 = (u64)((((unsigned __int128)c40) << 40) % q);
            mbar_wait(&tfull[a], (uint32_t)((it >> 1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;");
            uint32_t x[MT][32];
#pragma unroll
            for (int mt = 0; mt < MT; mt++) {
                const uint32_t taddr = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)((a * MT + mt) * 32);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
                    "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
                    : "=r"(x[mt][0]), "=r"(x[mt][1]), "=r"(x[mt][2]), "=r"(x[mt][3]), "=r"(x[mt][4]), "=r"(x[mt][5]),
                      "=r"(x[mt][6]), "=r"(x[mt][7]), "=r"(x[mt][8]), "=r"(x[mt][9]), "=r"(x[mt][10]), "=r"(x[mt][11]),
                      "=r"(x[mt][12]), "=r"(x[mt][13]), "=r"(x[mt][14]), "=r"(x[mt][15]), "=r"(x[mt][16]), "=r"(x[mt][17]),
                      "=r"(x[mt][18]), "=r"(x[mt][19]), "=r"(x[mt][20]), "=r"(x[mt][21]), "=r"(x[mt][22]), "=r"(x[mt][23]),
                      "=r"(x[mt][24]), "=r"(x[mt][25]), "=r"(x[mt][26]), "=r"(x[mt][27]), "=r"(x[mt][28]), "=r"(x[mt][29]),
                      "=r"(x[mt][30]), "=r"(x[mt][31])
                    : "r"(taddr));
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[a]);
#pragma unroll
            for (int mt = 0; mt < MT; mt++) {
                const int r = mt * 128 + lg * 32 + lane;
                if (r >= Mr) continue;
#pragma unroll
                for (int comp = 0; comp < 2; comp++) {
                    const uint32_t* xs = x[mt] + comp * 16;
                    u64 lo5 = 0, mi5 = 0, hi5 = 0;
#pragma unroll
                    for (int u = 0; u < 5; u++) {
                        lo5 += (u64)xs[u] << (8 * u);
                        mi5 += (u64)xs[5 + u] << (8 * u);
                        hi5 += (u64)xs[10 + u] << (8 * u);
                    }
                    // lo5 + mi5 2^40 + hi5 2^80 == sum R pt (mod q); fold with the constants (< 2^120)
                    Acc128 t;
                    t.mac(mi5, c40);
                    t.mac(hi5, c80);
                    t.lo += lo5;
                    t.hi += t.lo < lo5 ? 1ull : 0ull;
                    if (t.hi >= q) t.hi -= q;                       // t < 2^124 (Kwp <= 1024): hi < 2^60
                    const u64 v = csub(redc_lazy(t.hi, t.lo, md), q);
                    acc[((long long)r * 2 + comp) * LN + p] = v;
                }
            }
        }
    }
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
}

// ---------------------------------------------------------------------------
// encoding.  MODE 0: plaintext operand (centred lift, Montgomery);
//            MODE 1: Delta * m (plain), for encrypt / subtract_plain
// one CTA per (vector b, prime j); each CTA recomputes the mod-p INTT (cheap,
// p is a 20-bit modulus) to keep the kernel single-pass.
template <int MODE>
__global__ void __launch_bounds__(512, 2) k_encode(DevCtx c, const uint32_t* __restrict__ slots, u64* __restrict__ out)
{
    extern __shared__ u64 smem_enc[];
    u64* sm = smem_enc;
    const int N = c.N, PM = c.M; // plaintext tables at index M
    const int L = MODE == 2 ? c.M : c.L;   // MODE 2: operand in every prime of QP
    const int b = blockIdx.x / L, j = blockIdx.x % L;
    const uint32_t* sl = slots + (long long)b * N;
    const u64 p = c.p;
    for (int i = threadIdx.x; i < N; i += blockDim.x) sm[pad(c.slot_pos[i])] = sl[i] % p;
    __syncthreads();
    ntt_inv_smem(sm, c.twi[PM], p, c.logN);
    const ModC md = c.mod[j];
    const u64 q = md.q;
    u64* sm2 = sm + padded_words(N);
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        u64 m = shoup(sm[pad(i)], c.ninv[PM], c.ninv_sh[PM], p);
        u64 v;
        if (MODE != 1) v = m > (p >> 1) ? q - (p - m) : m;
        else v = shoup(m, c.delta[j], c.delta_sh[j], q);
        sm2[pad(i)] = v;
    }
    __syncthreads();
    sm = sm2;
    ntt_fwd_smem(sm, c.twf[j], q, c.logN);
    u64* o = out + ((long long)b * L + j) * N;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        u64 v = csub(csub(sm[pad(i)], 2 * q), q);
        if (MODE != 1) v = mont_mul(v, md.r2, md);
        o[i] = v;
    }
}

// decrypt phase 1: per prime j: x_j = INTT(c0 + c1 * S)
// Delta-encode split in two (the masks of a batch, MODE 1 of k_encode): the INTT mod p of a mask is the
// same for every ciphertext prime, so it runs once per mask (k_encode_p: slots -> N^-1-scaled
// coefficients m < p) and each prime's CTA only lifts and transforms (k_encode_q: Delta m mod q_j ->
// NTT_j).  One polynomial of shared memory each (two CTAs per SM, where k_encode<1> needs two); the same
// words as k_encode<1>.
__global__ void __launch_bounds__(512, 2) k_encode_p(DevCtx c, const uint32_t* __restrict__ slots, uint32_t* __restrict__ m)
{
    extern __shared__ u64 smem_enc[];
    u64* sm = smem_enc;
    const int N = c.N, PM = c.M;
    const uint32_t* sl = slots + (long long)blockIdx.x * N;
    const u64 p = c.p;
    for (int i = threadIdx.x; i < N; i += blockDim.x) sm[pad(c.slot_pos[i])] = sl[i] % p;
    __syncthreads();
    ntt_inv_smem(sm, c.twi[PM], p, c.logN);
    uint32_t* o = m + (long long)blockIdx.x * N;
    for (int i = threadIdx.x; i < N; i += blockDim.x) o[i] = (uint32_t)shoup(sm[pad(i)], c.ninv[PM], c.ninv_sh[PM], p);
}
__global__ void __launch_bounds__(512, 2) k_encode_q(DevCtx c, const uint32_t* __restrict__ m, u64* __restrict__ out)
{
    extern __shared__ u64 smem_enc[];
    u64* sm = smem_enc;
    const int N = c.N, L = c.L;
    const int b = blockIdx.x / L, j = blockIdx.x % L;
    const uint32_t* mb = m + (long long)b * N;
    const ModC md = c.mod[j];
    const u64 q = md.q, dl = c.delta[j], dsh = c.delta_sh[j];
    for (int i = threadIdx.x; i < N; i += blockDim.x) sm[pad(i)] = shoup((u64)__ldg(mb + i), dl, dsh, q);
    __syncthreads();
    ntt_fwd_smem(sm, c.twf[j], q, c.logN);
    u64* o = out + ((long long)b * L + j) * N;
    for (int i = threadIdx.x; i < N; i += blockDim.x) o[i] = csub(csub(sm[pad(i)], 2 * q), q);
}

__global__ void __launch_bounds__(512, 2) k_dec_phase1(DevCtx c, const u64* __restrict__ ct, u64* __restrict__ x)
{
    extern __shared__ u64 sm[];
    const int N = c.N, L = c.L, j = blockIdx.x;
    const ModC md = c.mod[j];
    const u64 q = md.q;
    const u64* c0 = ct + (long long)j * N;
    const u64* c1 = ct + ((long long)L + j) * N;
    const u64* S = c.S + (long long)j * N;
    for (int i = threadIdx.x; i < N; i += blockDim.x) sm[pad(i)] = add_mod(c0[i], mont_mul(c1[i], S[i], md), q);
    __syncthreads();
    ntt_inv_smem(sm, c.twi[j], q, c.logN);
    for (int i = threadIdx.x; i < N; i += blockDim.x) x[(long long)j * N + i] = shoup(sm[pad(i)], c.ninv[j], c.ninv_sh[j], q);
}

// floor(b 2^64 / q) for b < q < 2^63 (restoring division)
__device__ __forceinline__ u64 frac64(u64 b, u64 q)
{
    u64 r = b, qt = 0;
#pragma unroll 8
    for (int i = 0; i < 64; i++) {
        r <<= 1;
        qt <<= 1;
        if (r >= q) { r -= q; qt |= 1; }
    }
    return qt;
}

// decrypt phase 2 (one CTA): m = round(p x / Q) mod p via RNS; slots = decode(m).
// maxd (optional): the largest rounding distance |p x / Q - m| over the coefficients, as a 64-bit
// fixed-point fraction -- the real noise over Delta (p v / Q = m - (Q mod p) m / Q + p e / Q).
__global__ void __launch_bounds__(512, 2) k_dec_phase2(DevCtx c, const u64* __restrict__ x, uint32_t* __restrict__ slots,
                                                       unsigned long long* __restrict__ maxd)
{
    extern __shared__ u64 sm[];
    const int N = c.N, L = c.L, PM = c.M;
    const u64 p = c.p;
    u64 dmax = 0;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        u64 sum_a = 0, f_lo = 0, f_hi = 0;
        for (int j = 0; j < L; j++) {
            const u64 q = c.mod[j].q;
            u64 y = shoup(x[(long long)j * N + i], c.qhat_inv[j], c.qhat_inv_sh[j], q);
            // y * p = a q + b
            u64 lo = y * p, hi = __umul64hi(y, p);
            u64 a = (u64)((double)y * ((double)p / (double)q));
            // exact correction: rem = y p - a q (signed 128)
            u64 aql = a * q, aqh = __umul64hi(a, q);
            u64 rl = lo - aql;
            i64 rh = (i64)(hi - aqh - (lo < aql ? 1 : 0));
            while (rh < 0) { // rem += q, a -= 1
                u64 n = rl + q;
                rh += (n < rl) ? 1 : 0;
                rl = n;
                a -= 1;
            }
            while (rh > 0 || rl >= q) {
                u64 n = rl - q;
                rh -= (rl < q) ? 1 : 0;
                rl = n;
                a += 1;
            }
            sum_a += a;
            u64 f = frac64(rl, q);
            f_lo += f;
            f_hi += (f_lo < f) ? 1 : 0;
        }
        // round: add 2^63 to the 128-bit fraction sum, take the integer part
        u64 t = f_lo + (1ull << 63);
        u64 carry = (t < f_lo) ? 1 : 0;
        u64 rounded = sum_a + f_hi + carry;
        sm[pad(i)] = rounded % p;
        const u64 d = f_lo < (1ull << 63) ? f_lo : (u64)0 - f_lo;
        dmax = d > dmax ? d : dmax;
    }
    if (maxd) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const u64 v = __shfl_xor_sync(0xffffffffu, dmax, o);
            dmax = v > dmax ? v : dmax;
        }
        if ((threadIdx.x & 31) == 0) atomicMax(maxd, (unsigned long long)dmax);
    }
    __syncthreads();
    ntt_fwd_smem(sm, c.twf[PM], p, c.logN);
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        u64 v = sm[pad(c.slot_pos[i])];
        slots[i] = (uint32_t)(v % p);
    }
}

// key generation combine: per (i, j) poly and coefficient k
//   key[i][0][j] = mont(E - A S + [i==j] (P mod q_j) sigma(S)),  key[i][1][j] = mont(A)
__global__ void k_keygen_combine(DevCtx c, const u64* __restrict__ A, const u64* __restrict__ E, unsigned galois,
                                 const u64* __restrict__ pmod, u64* __restrict__ key)
{
    const int N = c.N, L = c.L, M = c.M;
    const long long total = (long long)L * M * N;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total;
         x += (long long)gridDim.x * blockDim.x) {
        int k = (int)(x % N);
        int ij = (int)(x / N);
        int i = ij / M, j = ij % M;
        const ModC md = c.mod[j];
        const u64 q = md.q;
        const u64* S = c.S + (long long)j * N;
        u64 a = A[x];
        u64 b = sub_mod(E[x], mont_mul(a, S[k], md), q);
        if (i == j) b = add_mod(b, mont_mul(S[auto_src(k, galois, c.logN)], pmod[j], md), q);
        key[(((long long)i * 2 + 0) * M + j) * N + k] = mont_mul(b, md.r2, md);
        key[(((long long)i * 2 + 1) * M + j) * N + k] = mont_mul(a, md.r2, md);
    }
}

// encrypt combine: ct.c1 = A, ct.c0 = E - A S + DM
__global__ void k_encrypt_combine(DevCtx c, const u64* __restrict__ A, const u64* __restrict__ E,
                                  const u64* __restrict__ DM, u64* __restrict__ ct)
{
    const int N = c.N, L = c.L;
    const long long total = (long long)L * N;
    for (long long x = blockIdx.x * (long long)blockDim.x + threadIdx.x; x < total;
         x += (long long)gridDim.x * blockDim.x) {
        int j = (int)(x / N);
        const ModC md = c.mod[j];
        const u64 q = md.q;
        u64 a = A[x];
        ct[x] = add_mod(sub_mod(E[x], mont_mul(a, c.S[x], md), q), DM[x], q);
        ct[total + x] = a;
    }
}

// modmul throughput probe: 8 independent lazy-Shoup chains per thread, each
// step = one butterfly-style multiply (shoup_lazy + conditional 2q fold)
__global__ void __launch_bounds__(256) k_bench_modmul(u64 q, u64 w, u64 wsh, int iters, u64* __restrict__ sink)
{
    u64 x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = (threadIdx.x * 8 + i + blockIdx.x) % q;
    const u64 q2 = 2 * q;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            u64 v = shoup_lazy_sf(x[i], w, wsh, q);   // the cheapest modmul flavour the library uses
            x[i] = v >= q2 ? v - q2 : v;
        }
    }
    u64 acc = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) acc ^= x[i];
    sink[blockIdx.x * 256 + threadIdx.x] = acc;
}
