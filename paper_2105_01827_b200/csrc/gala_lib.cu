// gala_lib.cu -- host side of the B200-native GALA library: context, keys,
// op seam, fused GALA dot product and kernel-grouping convolution, C-ABI.
//
// Every schedule here mirrors the CPU oracle (oracle/bfv_oracle.c) operation
// for operation, so ciphertext words agree exactly.  See include/gala_b200.h.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "gala_kernels.cuh"
#include "../../include/gala_b200.h"

typedef unsigned __int128 u128;

static thread_local std::string g_err;
static std::atomic<unsigned long long> g_launches{0};

static int set_err(int code, const char* fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            return set_err(GALA_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                           __FILE__, __LINE__);                                                    \
    } while (0)

#define LAUNCHED()                                                                                 \
    do {                                                                                           \
        g_launches++;                                                                              \
        cudaError_t e_ = cudaGetLastError();                                                       \
        if (e_ != cudaSuccess)                                                                     \
            return set_err(GALA_ERR_CUDA, "kernel launch failed: %s (%s:%d)", cudaGetErrorString(e_), \
                           __FILE__, __LINE__);                                                    \
    } while (0)

#define RET(...)                      \
    do {                              \
        int r_ = (__VA_ARGS__);       \
        if (r_ != GALA_OK) return r_; \
    } while (0)

// ---------------------------------------------------------------------------
// host modular helpers
static u64 h_mulmod(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
static u64 h_pow(u64 b, u64 e, u64 q)
{
    u64 r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = h_mulmod(r, b, q);
        b = h_mulmod(b, b, q);
        e >>= 1;
    }
    return r;
}
static u64 h_inv(u64 a, u64 q) { return h_pow(a, q - 2, q); }
static u64 h_shoup(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }
static int h_brv(int x, int logN)
{
    int r = 0;
    for (int i = 0; i < logN; i++) r |= ((x >> i) & 1) << (logN - 1 - i);
    return r;
}

// pinned staging buffer for small per-call descriptor tables
struct Staging {
    void* host = nullptr;
    size_t cap = 0;
    cudaEvent_t done = nullptr;
};

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
};

struct gala_ctx {
    DevCtx dc;
    int device = 0;
    cudaStream_t stream = 0;
    std::vector<u64> primes;  // L + 1 (special last)
    u64 p = 0;
    void* d_tables = nullptr; // twiddles for M + 1 moduli
    u64* d_S = nullptr;
    int* d_slot_pos = nullptr;
    u64* d_pmod = nullptr;    // P mod q_j (plain)
    bool has_secret = false;
    std::map<int, u64*> keys; // step -> [L][2][M][N]
    size_t key_bytes = 0;
    Staging stage;
    int smem_ntt = 0;         // bytes of one padded polynomial
    std::mutex mu;
};

static inline int norm_step(const gala_ctx* c, int step)
{
    int n = c->dc.N / 2;
    return ((step % n) + n) % n;
}
static inline unsigned galois_of(const gala_ctx* c, int step)
{
    return (unsigned)h_pow(3, (u64)norm_step(c, step), 2 * (u64)c->dc.N);
}

// stream-ordered scratch
template <typename T>
static int scratch(gala_ctx* c, T** p, size_t count)
{
    size_t bytes = count * sizeof(T);
    if (bytes == 0) bytes = 8;
    CK(cudaMallocAsync((void**)p, bytes, c->stream));
    return GALA_OK;
}
static void release(gala_ctx* c, void* p)
{
    if (p) cudaFreeAsync(p, c->stream);
}

// copy a small host table to device via the pinned staging buffer
static int upload(gala_ctx* c, const void* src, size_t bytes, void** dst)
{
    Staging& s = c->stage;
    if (s.done) CK(cudaEventSynchronize(s.done)); // previous upload consumed
    if (bytes > s.cap) {
        if (s.host) cudaFreeHost(s.host);
        s.cap = bytes < (1 << 16) ? (1 << 16) : bytes;
        CK(cudaMallocHost(&s.host, s.cap));
    }
    if (!s.done) CK(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
    memcpy(s.host, src, bytes);
    CK(cudaMallocAsync(dst, bytes, c->stream));
    CK(cudaMemcpyAsync(*dst, s.host, bytes, cudaMemcpyHostToDevice, c->stream));
    CK(cudaEventRecord(s.done, c->stream));
    return GALA_OK;
}

// ---------------------------------------------------------------------------
// launch helpers
static PolyMap pm_make(int per, int nprimes, int prime_base, int src_div, long long src_is, long long dst_is,
                       int skip_per = 0)
{
    PolyMap pm;
    pm.per = per;
    pm.nprimes = nprimes;
    pm.prime_base = prime_base;
    pm.src_div = src_div;
    pm.src_is = src_is;
    pm.dst_is = dst_is;
    pm.skip_per = skip_per;
    return pm;
}

template <typename T, bool MONT>
static int launch_fwd(gala_ctx* c, const T* src, u64* dst, int polys, PolyMap pm)
{
    if (polys <= 0) return GALA_OK;
    k_ntt_fwd<T, MONT><<<polys, ntt_threads(c->dc.N), c->smem_ntt, c->stream>>>(c->dc, src, dst, pm);
    LAUNCHED();
    return GALA_OK;
}
template <bool MONT>
static int launch_inv(gala_ctx* c, const u64* src, u64* dst, int polys, PolyMap pm)
{
    if (polys <= 0) return GALA_OK;
    k_ntt_inv<MONT><<<polys, ntt_threads(c->dc.N), c->smem_ntt, c->stream>>>(c->dc, src, dst, pm);
    LAUNCHED();
    return GALA_OK;
}
static int grid_for(long long total, int threads)
{
    long long b = (total + threads - 1) / threads;
    if (b > 148 * 32) b = 148 * 32;
    return (int)(b < 1 ? 1 : b);
}

// ---------------------------------------------------------------------------
// key switching building blocks

// digits of `count` items' c1 (items at X + x * x_stride, with optional skip
// remap), D [count][L][M][N]
static int decompose_items(gala_ctx* c, const u64* X, long long x_stride, int count, int skip_per, u64* D)
{
    const int N = c->dc.N, L = c->dc.L, M = c->dc.M;
    if (count <= 0) return GALA_OK;
    u64* dig;
    RET(scratch(c, &dig, (size_t)count * L * N));
    // INTT of c1 limbs -> digits in [0, q_i)
    RET(launch_inv<false>(c, X + (long long)L * N, dig, count * L,
                          pm_make(L, L, 0, 0, x_stride, (long long)L * N, skip_per)));
    // NTT of digit i into every prime j (digit < q_i < 4 q_j)
    RET(launch_fwd<u64, false>(c, dig, D, count * L * M,
                               pm_make(L * M, M, 0, 1, (long long)L * N, (long long)L * M * N)));
    release(c, dig);
    return GALA_OK;
}

// U[G] (QP) and Cacc[G] from item descriptors; then ModDown into out[g]
static int ks_groups(gala_ctx* c, const std::vector<KsItem>& items, const std::vector<int>& off, u64* out,
                     long long out_is)
{
    const int N = c->dc.N, L = c->dc.L, M = c->dc.M;
    const int G = (int)off.size() - 1;
    if (G <= 0) return GALA_OK;
    // descriptor upload (items then offsets, one staging copy)
    size_t ib = items.size() * sizeof(KsItem), ob = off.size() * sizeof(int);
    std::vector<char> blob(ib + ob);
    memcpy(blob.data(), items.data(), ib);
    memcpy(blob.data() + ib, off.data(), ob);
    void* d_blob;
    RET(upload(c, blob.data(), blob.size(), &d_blob));
    u64 *U, *Cacc, *r;
    RET(scratch(c, &U, (size_t)G * 2 * M * N));
    RET(scratch(c, &Cacc, (size_t)G * 2 * L * N));
    RET(scratch(c, &r, (size_t)G * 2 * N));
    const int th = N < 256 ? N : 256;
    dim3 grid((N + th - 1) / th, M, G);
    k_ks_accum<<<grid, th, 0, c->stream>>>(c->dc, (const KsItem*)d_blob, (const int*)((char*)d_blob + ib), U,
                                           Cacc);
    LAUNCHED();
    // r = INTT_P(U[g][comp][P])
    RET(launch_inv<false>(c, U + (long long)L * N, r, G * 2, pm_make(1, 1, L, 0, (long long)M * N, N)));
    MdArgs a;
    a.r = r;
    a.U = U;
    a.add0 = Cacc;
    a.add1 = Cacc + (long long)L * N;
    a.add_is = 2LL * L * N;
    a.out = out;
    a.out_is = out_is;
    k_moddown<<<G * 2 * L, ntt_threads(N), c->smem_ntt, c->stream>>>(c->dc, a);
    LAUNCHED();
    release(c, U);
    release(c, Cacc);
    release(c, r);
    release(c, d_blob);
    return GALA_OK;
}

static const u64* key_for(gala_ctx* c, int step)
{
    auto it = c->keys.find(norm_step(c, step));
    return it == c->keys.end() ? nullptr : it->second;
}

// out[g] = sum_{j < per} rot_{j * unit}(X[g * per + j]), one lazy ModDown per g
static int rotate_sum_regular(gala_ctx* c, const u64* X, int G, int per, int unit, u64* out)
{
    const int N = c->dc.N, L = c->dc.L, M = c->dc.M;
    const long long W = 2LL * L * N, DW = (long long)L * M * N;
    if (per == 1) {
        CK(cudaMemcpyAsync(out, X, sizeof(u64) * W * G, cudaMemcpyDeviceToDevice, c->stream));
        return GALA_OK;
    }
    // key check first
    for (int j = 1; j < per; j++)
        if (norm_step(c, j * unit) != 0 && !key_for(c, j * unit))
            return set_err(GALA_ERR_NOKEY, "missing rotation key for step %d", norm_step(c, j * unit));
    u64* D;
    const int nrot = G * (per - 1);
    RET(scratch(c, &D, (size_t)nrot * DW));
    RET(decompose_items(c, X, W, nrot, per, D));
    std::vector<KsItem> items;
    std::vector<int> off;
    items.reserve((size_t)G * per);
    for (int g = 0; g < G; g++) {
        off.push_back((int)items.size());
        for (int j = 0; j < per; j++) {
            KsItem it;
            it.X = X + (long long)(g * per + j) * W;
            int s = norm_step(c, j * unit);
            if (s == 0) {
                it.D = nullptr;
                it.key = nullptr;
                it.galois = 1;
                it.step0 = 1;
            } else {
                it.D = D + (long long)(g * (per - 1) + (j - 1)) * DW;
                it.key = key_for(c, s);
                it.galois = galois_of(c, s);
                it.step0 = 0;
            }
            items.push_back(it);
        }
    }
    off.push_back((int)items.size());
    RET(ks_groups(c, items, off, out, W));
    release(c, D);
    return GALA_OK;
}

// ---------------------------------------------------------------------------
// C-ABI
extern "C" {

const char* gala_last_error(void) { return g_err.c_str(); }
int gala_version(void) { return 1; }
uint64_t gala_launch_count(void) { return g_launches.load(); }

static void free_ctx(gala_ctx* c)
{
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    for (auto& kv : c->keys) cudaFree(kv.second);
    if (c->d_tables) cudaFree(c->d_tables);
    if (c->d_S) cudaFree(c->d_S);
    if (c->d_slot_pos) cudaFree(c->d_slot_pos);
    if (c->d_pmod) cudaFree(c->d_pmod);
    if (c->stage.host) cudaFreeHost(c->stage.host);
    if (c->stage.done) cudaEventDestroy(c->stage.done);
    delete c;
}

int gala_ctx_create(gala_ctx** out, int N, int L, const uint64_t* primes, const uint64_t* psis, uint64_t p,
                    uint64_t psi_p, int device)
{
    *out = nullptr;
    if (N < 8 || N > 8192 || (N & (N - 1))) return set_err(GALA_ERR_PARAM, "N=%d must be a power of two in [8, 8192]", N);
    if (L < 1 || L + 2 > GALA_MAXM) return set_err(GALA_ERR_PARAM, "L=%d out of range", L);
    const int M = L + 1;
    for (int j = 0; j < M; j++) {
        if (primes[j] >= (1ull << 62)) return set_err(GALA_ERR_PARAM, "prime %d exceeds 2^62", j);
        if ((primes[j] - 1) % (2ull * N)) return set_err(GALA_ERR_PARAM, "prime %d not 1 mod 2N", j);
    }
    for (int i = 0; i < M; i++)
        for (int j = 0; j < M; j++) {
            if (primes[i] >= 4 * (u128)primes[j]) return set_err(GALA_ERR_PARAM, "prime spread too wide for lazy lifts");
            if (i == L && j < L && primes[L] / 2 >= primes[j])
                return set_err(GALA_ERR_PARAM, "special prime must be < 2 q_j");
        }
    if ((p - 1) % (2ull * N)) return set_err(GALA_ERR_PARAM, "p=%llu is not 1 mod 2N", (unsigned long long)p);
    gala_ctx* c = new gala_ctx();
    c->device = device;
    c->p = p;
    c->primes.assign(primes, primes + M);
    if (cudaSetDevice(device) != cudaSuccess) {
        delete c;
        return set_err(GALA_ERR_CUDA, "cudaSetDevice(%d) failed", device);
    }
    DevCtx& d = c->dc;
    memset(&d, 0, sizeof(d));
    d.N = N;
    d.L = L;
    d.M = M;
    while ((1 << d.logN) < N) d.logN++;
    d.p = p;
    // moduli: 0..L-1 ciphertext, L special, M plaintext
    std::vector<u64> mods(primes, primes + M);
    mods.push_back(p);
    std::vector<u64> roots(psis, psis + M);
    roots.push_back(psi_p);
    const int NM = M + 1;
    // twiddle tables: [NM][2][N] ulonglong2
    std::vector<ulonglong2> tw((size_t)NM * 2 * N);
    for (int j = 0; j < NM; j++) {
        u64 q = mods[j], psi = roots[j] % q, ipsi = h_inv(psi, q);
        if (h_pow(psi, (u64)N, q) != q - 1) {
            delete c;
            return set_err(GALA_ERR_PARAM, "psi for modulus %d is not a primitive 2N-th root", j);
        }
        for (int k = 0; k < N; k++) {
            int e = h_brv(k, d.logN);
            u64 w = h_pow(psi, (u64)e, q), iw = h_pow(ipsi, (u64)e, q);
            tw[((size_t)j * 2 + 0) * N + k] = make_ulonglong2(w, h_shoup(w, q));
            tw[((size_t)j * 2 + 1) * N + k] = make_ulonglong2(iw, h_shoup(iw, q));
        }
        d.mod[j].q = q;
        u64 inv = 1; // q^-1 mod 2^64 (Newton)
        for (int it = 0; it < 7; it++) inv *= 2 - q * inv;
        d.mod[j].qinv_neg = (u64)0 - inv;
        u64 r1 = (u64)(((u128)1 << 64) % q);
        d.mod[j].r2 = h_mulmod(r1, r1, q);
        d.ninv[j] = h_inv((u64)N % q, q);
        d.ninv_sh[j] = h_shoup(d.ninv[j], q);
    }
    // Delta = floor(Q / p) mod q_j, through multi-limb Q
    std::vector<u64> Q(1, 1);
    for (int i = 0; i < L; i++) {
        u128 carry = 0;
        for (auto& limb : Q) {
            u128 v = (u128)limb * primes[i] + carry;
            limb = (u64)v;
            carry = v >> 64;
        }
        if (carry) Q.push_back((u64)carry);
    }
    std::vector<u64> Dq(Q.size());
    u128 rem = 0;
    for (int k = (int)Q.size() - 1; k >= 0; k--) {
        u128 cur = (rem << 64) | Q[k];
        Dq[k] = (u64)(cur / p);
        rem = cur % p;
    }
    std::vector<u64> pmod(M);
    for (int j = 0; j < M; j++) {
        u64 q = primes[j];
        u128 acc = 0;
        for (int k = (int)Dq.size() - 1; k >= 0; k--) acc = ((acc << 64) | Dq[k]) % q;
        d.delta[j] = (u64)acc;
        d.delta_sh[j] = h_shoup(d.delta[j], q);
        pmod[j] = primes[L] % q;
        if (j < L) {
            u64 pinv = h_inv(primes[L] % q, q);
            d.pinv_mont[j] = h_mulmod(pinv, (u64)(((u128)1 << 64) % q), q);
        }
    }
    for (int i = 0; i < L; i++) {
        u64 qh = 1;
        for (int k = 0; k < L; k++)
            if (k != i) qh = h_mulmod(qh, primes[k] % primes[i], primes[i]);
        d.qhat_inv[i] = h_inv(qh, primes[i]);
        d.qhat_inv_sh[i] = h_shoup(d.qhat_inv[i], primes[i]);
    }
    // slot positions: slot (r, col) -> evaluation at zeta^(+-3^col) -> NTT_p bit-reversed index
    std::vector<int> slot_pos(N);
    {
        int n = N / 2;
        u64 e = 1, two_n = 2 * (u64)N;
        for (int col = 0; col < n; col++) {
            slot_pos[col] = h_brv((int)((e - 1) / 2), d.logN);
            slot_pos[n + col] = h_brv((int)((two_n - e - 1) / 2), d.logN);
            e = (e * 3) % two_n;
        }
    }
    int rc = GALA_OK;
#define CKC(call)                                                                                 \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess) {                                                                  \
            rc = set_err(GALA_ERR_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_));          \
            free_ctx(c);                                                                          \
            return rc;                                                                            \
        }                                                                                         \
    } while (0)
    CKC(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CKC(cudaMalloc(&c->d_tables, tw.size() * sizeof(ulonglong2)));
    CKC(cudaMemcpy(c->d_tables, tw.data(), tw.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice));
    for (int j = 0; j < NM; j++) {
        d.twf[j] = (const ulonglong2*)c->d_tables + ((size_t)j * 2 + 0) * N;
        d.twi[j] = (const ulonglong2*)c->d_tables + ((size_t)j * 2 + 1) * N;
    }
    CKC(cudaMalloc(&c->d_slot_pos, sizeof(int) * N));
    CKC(cudaMemcpy(c->d_slot_pos, slot_pos.data(), sizeof(int) * N, cudaMemcpyHostToDevice));
    d.slot_pos = c->d_slot_pos;
    CKC(cudaMalloc(&c->d_pmod, sizeof(u64) * M));
    CKC(cudaMemcpy(c->d_pmod, pmod.data(), sizeof(u64) * M, cudaMemcpyHostToDevice));
    CKC(cudaMalloc(&c->d_S, sizeof(u64) * (size_t)M * N));
    d.S = c->d_S;
    c->smem_ntt = padded_words(N) * (int)sizeof(u64);
    // opt in to large dynamic shared memory for every NTT-carrying kernel
    CKC(cudaFuncSetAttribute(k_ntt_fwd<u64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, c->smem_ntt));
    CKC(cudaFuncSetAttribute(k_ntt_fwd<u64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, c->smem_ntt));
    CKC(cudaFuncSetAttribute(k_ntt_fwd<i64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, c->smem_ntt));
    CKC(cudaFuncSetAttribute(k_ntt_fwd<int8_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, c->smem_ntt));
    CKC(cudaFuncSetAttribute(k_ntt_inv<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, c->smem_ntt));
    CKC(cudaFuncSetAttribute(k_ntt_inv<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, c->smem_ntt));
    CKC(cudaFuncSetAttribute(k_moddown, cudaFuncAttributeMaxDynamicSharedMemorySize, c->smem_ntt));
    CKC(cudaFuncSetAttribute(k_encode<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * c->smem_ntt));
    CKC(cudaFuncSetAttribute(k_encode<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * c->smem_ntt));
    CKC(cudaFuncSetAttribute(k_dec_phase1, cudaFuncAttributeMaxDynamicSharedMemorySize, c->smem_ntt));
    CKC(cudaFuncSetAttribute(k_dec_phase2, cudaFuncAttributeMaxDynamicSharedMemorySize, c->smem_ntt));
    // keep freed scratch in the pool (stream-ordered allocator as a caching pool)
    cudaMemPool_t pool;
    CKC(cudaDeviceGetDefaultMemPool(&pool, device));
    u64 thresh = ~0ull;
    CKC(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh));
#undef CKC
    *out = c;
    return GALA_OK;
}

void gala_ctx_destroy(gala_ctx* c) { free_ctx(c); }

int gala_set_stream(gala_ctx* c, void* s)
{
    if (!c) return set_err(GALA_ERR_STATE, "null context");
    c->stream = (cudaStream_t)s;
    return GALA_OK;
}

int gala_sync(gala_ctx* c)
{
    CK(cudaStreamSynchronize(c->stream));
    return GALA_OK;
}

int gala_set_secret(gala_ctx* c, const int8_t* s_host)
{
    const int N = c->dc.N, M = c->dc.M;
    int8_t* ds;
    RET(scratch(c, &ds, N));
    CK(cudaMemcpyAsync(ds, s_host, N, cudaMemcpyHostToDevice, c->stream));
    RET(launch_fwd<int8_t, true>(c, ds, c->d_S, M, pm_make(M, M, 0, 1, 0, (long long)M * N)));
    release(c, ds);
    CK(cudaStreamSynchronize(c->stream));
    c->has_secret = true;
    return GALA_OK;
}

int gala_gen_rotation_key(gala_ctx* c, int step, const uint64_t* a_host, const int64_t* e_host)
{
    if (!c->has_secret) return set_err(GALA_ERR_STATE, "secret key not set");
    const int N = c->dc.N, L = c->dc.L, M = c->dc.M;
    int s = norm_step(c, step);
    if (s == 0) return GALA_OK;
    const size_t kw = (size_t)L * 2 * M * N;
    u64 *da, *A, *E;
    i64* de;
    RET(scratch(c, &da, (size_t)L * M * N));
    RET(scratch(c, &A, (size_t)L * M * N));
    RET(scratch(c, &E, (size_t)L * M * N));
    RET(scratch(c, &de, (size_t)L * N));
    CK(cudaMemcpyAsync(da, a_host, sizeof(u64) * L * M * N, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(de, e_host, sizeof(i64) * L * N, cudaMemcpyHostToDevice, c->stream));
    RET(launch_fwd<u64, false>(c, da, A, L * M, pm_make(L * M, M, 0, 0, 0, 0)));
    RET(launch_fwd<i64, false>(c, de, E, L * M, pm_make(L * M, M, 0, 1, 0, 0)));
    u64* key = nullptr;
    auto it = c->keys.find(s);
    if (it != c->keys.end()) key = it->second;
    else {
        CK(cudaMalloc(&key, sizeof(u64) * kw));
        c->keys[s] = key;
        c->key_bytes += sizeof(u64) * kw;
    }
    k_keygen_combine<<<grid_for((long long)L * M * N, 256), 256, 0, c->stream>>>(c->dc, A, E, galois_of(c, s),
                                                                                 c->d_pmod, key);
    LAUNCHED();
    release(c, da);
    release(c, A);
    release(c, E);
    release(c, de);
    CK(cudaStreamSynchronize(c->stream));
    return GALA_OK;
}

int gala_has_rotation_key(gala_ctx* c, int step)
{
    return norm_step(c, step) == 0 || key_for(c, step) != nullptr;
}

size_t gala_key_bytes(gala_ctx* c) { return c->key_bytes; }

int gala_encode_plain(gala_ctx* c, const uint32_t* slots, int B, uint64_t* pt)
{
    if (B <= 0) return GALA_OK;
    k_encode<0><<<B * c->dc.L, ntt_threads(c->dc.N), 2 * c->smem_ntt, c->stream>>>(c->dc, slots, pt);
    LAUNCHED();
    return GALA_OK;
}

int gala_encrypt(gala_ctx* c, const uint32_t* slots, const uint64_t* a, const int64_t* e, uint64_t* ct)
{
    if (!c->has_secret) return set_err(GALA_ERR_STATE, "secret key not set");
    const int N = c->dc.N, L = c->dc.L;
    u64 *A, *E, *DM;
    RET(scratch(c, &A, (size_t)L * N));
    RET(scratch(c, &E, (size_t)L * N));
    RET(scratch(c, &DM, (size_t)L * N));
    RET(launch_fwd<u64, false>(c, a, A, L, pm_make(L, L, 0, 0, 0, 0)));
    RET(launch_fwd<i64, false>(c, e, E, L, pm_make(L, L, 0, 1, 0, 0)));
    k_encode<1><<<L, ntt_threads(N), 2 * c->smem_ntt, c->stream>>>(c->dc, slots, DM);
    LAUNCHED();
    k_encrypt_combine<<<grid_for((long long)L * N, 256), 256, 0, c->stream>>>(c->dc, A, E, DM, ct);
    LAUNCHED();
    release(c, A);
    release(c, E);
    release(c, DM);
    return GALA_OK;
}

int gala_decrypt(gala_ctx* c, const uint64_t* ct, uint32_t* slots)
{
    if (!c->has_secret) return set_err(GALA_ERR_STATE, "secret key not set");
    const int N = c->dc.N, L = c->dc.L;
    u64* x;
    RET(scratch(c, &x, (size_t)L * N));
    k_dec_phase1<<<L, ntt_threads(N), c->smem_ntt, c->stream>>>(c->dc, ct, x);
    LAUNCHED();
    k_dec_phase2<<<1, ntt_threads(N), c->smem_ntt, c->stream>>>(c->dc, x, slots);
    LAUNCHED();
    release(c, x);
    return GALA_OK;
}

int gala_add(gala_ctx* c, const uint64_t* a, const uint64_t* b, uint64_t* out)
{
    long long total = 2LL * c->dc.L * c->dc.N;
    k_addsub<<<grid_for(total, 256), 256, 0, c->stream>>>(c->dc, a, b, out, total, c->dc.L, 1);
    LAUNCHED();
    return GALA_OK;
}

int gala_scmult(gala_ctx* c, const uint64_t* ct, const uint64_t* pt, uint64_t* out)
{
    const int N = c->dc.N, L = c->dc.L;
    dim3 grid((2 * L * N + 255) / 256, 1);
    k_ct_mul_pts<<<grid, 256, 0, c->stream>>>(c->dc, ct, pt, out);
    LAUNCHED();
    return GALA_OK;
}

int gala_sub_plain(gala_ctx* c, const uint64_t* ct, const uint32_t* r, uint64_t* out)
{
    const int N = c->dc.N, L = c->dc.L;
    u64* DM;
    RET(scratch(c, &DM, (size_t)L * N));
    k_encode<1><<<L, ntt_threads(N), 2 * c->smem_ntt, c->stream>>>(c->dc, r, DM);
    LAUNCHED();
    if (out != ct) CK(cudaMemcpyAsync(out + (long long)L * N, ct + (long long)L * N, sizeof(u64) * L * N,
                                      cudaMemcpyDeviceToDevice, c->stream));
    long long total = (long long)L * N;
    k_addsub<<<grid_for(total, 256), 256, 0, c->stream>>>(c->dc, ct, DM, out, total, L, -1);
    LAUNCHED();
    release(c, DM);
    return GALA_OK;
}

size_t gala_digits_words(gala_ctx* c) { return (size_t)c->dc.L * c->dc.M * c->dc.N; }

int gala_decompose(gala_ctx* c, const uint64_t* ct, uint64_t* digits)
{
    return decompose_items(c, ct, 0, 1, 0, digits);
}

int gala_rotate_hoisted(gala_ctx* c, const uint64_t* ct, const uint64_t* digits, int step, uint64_t* out)
{
    const int N = c->dc.N, L = c->dc.L;
    int s = norm_step(c, step);
    if (s == 0) {
        if (out != ct) CK(cudaMemcpyAsync(out, ct, sizeof(u64) * 2 * L * N, cudaMemcpyDeviceToDevice, c->stream));
        return GALA_OK;
    }
    const u64* key = key_for(c, s);
    if (!key) return set_err(GALA_ERR_NOKEY, "missing rotation key for step %d", s);
    std::vector<KsItem> items(1);
    items[0].D = digits;
    items[0].X = ct;
    items[0].key = key;
    items[0].galois = galois_of(c, s);
    items[0].step0 = 0;
    std::vector<int> off = {0, 1};
    return ks_groups(c, items, off, out, 2LL * L * N);
}

int gala_rotate(gala_ctx* c, const uint64_t* ct, int step, uint64_t* out)
{
    const int N = c->dc.N, L = c->dc.L, M = c->dc.M;
    int s = norm_step(c, step);
    if (s == 0) {
        if (out != ct) CK(cudaMemcpyAsync(out, ct, sizeof(u64) * 2 * L * N, cudaMemcpyDeviceToDevice, c->stream));
        return GALA_OK;
    }
    if (!key_for(c, s)) return set_err(GALA_ERR_NOKEY, "missing rotation key for step %d", s);
    u64* D;
    RET(scratch(c, &D, (size_t)L * M * N));
    RET(gala_decompose(c, ct, D));
    RET(gala_rotate_hoisted(c, ct, D, s, out));
    release(c, D);
    return GALA_OK;
}

int gala_bsgs_baby(int T)
{
    int lg = 0;
    while ((1 << lg) < T) lg++;
    return 1 << ((lg + 1) / 2);
}

int gala_mv_gala(gala_ctx* c, const uint64_t* ct, const uint64_t* pts, int T, int baby, const uint32_t* r,
                 uint64_t* out, uint64_t* masked)
{
    const int N = c->dc.N, L = c->dc.L;
    if (T <= 0) return set_err(GALA_ERR_DIM, "T must be positive");
    if (baby <= 0) baby = gala_bsgs_baby(T);
    if (T % baby) return set_err(GALA_ERR_PARAM, "baby step %d does not divide T=%d", baby, T);
    const int G = T / baby;
    const long long W = 2LL * L * N;
    for (int j = 1; j < baby; j++)
        if (!gala_has_rotation_key(c, j)) return set_err(GALA_ERR_NOKEY, "missing rotation key for step %d", j);
    for (int g = 1; g < G; g++)
        if (!gala_has_rotation_key(c, g * baby))
            return set_err(GALA_ERR_NOKEY, "missing rotation key for step %d", norm_step(c, g * baby));
    u64* U;
    RET(scratch(c, &U, (size_t)T * W));
    dim3 grid((unsigned)((2 * L * N + 255) / 256), (unsigned)T);
    k_ct_mul_pts<<<grid, 256, 0, c->stream>>>(c->dc, ct, pts, U);
    LAUNCHED();
    if (G == 1) {
        RET(rotate_sum_regular(c, U, 1, baby, 1, out));
    } else {
        u64* inner;
        RET(scratch(c, &inner, (size_t)G * W));
        RET(rotate_sum_regular(c, U, G, baby, 1, inner));
        RET(rotate_sum_regular(c, inner, 1, G, baby, out));
        release(c, inner);
    }
    release(c, U);
    if (r && masked) RET(gala_sub_plain(c, out, r, masked));
    return GALA_OK;
}

int gala_mv_gala_host(gala_ctx* c, const uint64_t* ct_host, const uint64_t* pts, int T, int baby,
                      const uint32_t* r_host, uint64_t* masked_host)
{
    const int N = c->dc.N, L = c->dc.L;
    const long long W = 2LL * L * N;
    u64 *coef, *ct, *out, *masked;
    uint32_t* r;
    RET(scratch(c, &coef, (size_t)W));
    RET(scratch(c, &ct, (size_t)W));
    RET(scratch(c, &out, (size_t)W));
    RET(scratch(c, &masked, (size_t)W));
    RET(scratch(c, &r, (size_t)N));
    CK(cudaMemcpyAsync(coef, ct_host, sizeof(u64) * W, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(r, r_host, sizeof(uint32_t) * N, cudaMemcpyHostToDevice, c->stream));
    RET(gala_ct_import(c, coef, ct, 1));
    RET(gala_mv_gala(c, ct, pts, T, baby, r, out, masked));
    RET(gala_ct_export(c, masked, coef, 1));
    CK(cudaMemcpyAsync(masked_host, coef, sizeof(u64) * W, cudaMemcpyDeviceToHost, c->stream));
    release(c, coef);
    release(c, ct);
    release(c, out);
    release(c, masked);
    release(c, r);
    CK(cudaStreamSynchronize(c->stream));
    return GALA_OK;
}

int gala_conv_kg(gala_ctx* c, const uint64_t* cts, int n_ib, const uint64_t* pts, int n_obp, int c_n, int k,
                 const int* tap_steps, int band_step, uint64_t* outs)
{
    const int N = c->dc.N, L = c->dc.L, M = c->dc.M;
    const long long W = 2LL * L * N, DW = (long long)L * M * N;
    if (n_ib <= 0 || n_obp <= 0 || c_n <= 0 || k <= 0) return set_err(GALA_ERR_DIM, "empty convolution");
    std::vector<int> rot_taps;
    for (int t = 0; t < k; t++) {
        int s = norm_step(c, tap_steps[t]);
        if (s != 0) {
            if (!key_for(c, s)) return set_err(GALA_ERR_NOKEY, "missing rotation key for step %d", s);
            rot_taps.push_back(t);
        }
    }
    for (int d = 1; d < c_n; d++)
        if (!gala_has_rotation_key(c, d * band_step))
            return set_err(GALA_ERR_NOKEY, "missing rotation key for step %d", norm_step(c, d * band_step));
    // input rotations R[ib][tap]: one DecPerm per input, HstPerm per nonzero tap
    u64* R;
    RET(scratch(c, &R, (size_t)n_ib * k * W));
    for (int ib = 0; ib < n_ib; ib++)
        for (int t = 0; t < k; t++)
            if (norm_step(c, tap_steps[t]) == 0)
                CK(cudaMemcpyAsync(R + ((long long)ib * k + t) * W, cts + (long long)ib * W, sizeof(u64) * W,
                                   cudaMemcpyDeviceToDevice, c->stream));
    if (!rot_taps.empty()) {
        u64* D;
        RET(scratch(c, &D, (size_t)n_ib * DW));
        RET(decompose_items(c, cts, W, n_ib, 0, D));
        // one group per (ib, rotated tap), each its own ModDown; outputs land
        // directly in R via per-group output stride: process tap by tap so the
        // output stride is regular (k * W per ib)
        for (int t : rot_taps) {
            std::vector<KsItem> items;
            std::vector<int> off;
            int s = norm_step(c, tap_steps[t]);
            for (int ib = 0; ib < n_ib; ib++) {
                off.push_back((int)items.size());
                KsItem it;
                it.D = D + (long long)ib * DW;
                it.X = cts + (long long)ib * W;
                it.key = key_for(c, s);
                it.galois = galois_of(c, s);
                it.step0 = 0;
                items.push_back(it);
            }
            off.push_back((int)items.size());
            RET(ks_groups(c, items, off, R + (long long)t * W, (long long)k * W));
        }
        release(c, D);
    }
    // first-Add: acc[o][d] over all input blocks and taps
    u64* acc;
    RET(scratch(c, &acc, (size_t)n_obp * c_n * W));
    const int th = N < 256 ? N : 256;
    dim3 grid((N + th - 1) / th, L, n_obp * c_n);
    k_kg_accumulate<<<grid, th, 0, c->stream>>>(c->dc, R, n_ib, k, pts, c_n, acc);
    LAUNCHED();
    release(c, R);
    // second-Perm: out[o] = sum_d rot_{d * band}(acc[o][d]), one lazy ModDown per o
    RET(rotate_sum_regular(c, acc, n_obp, c_n, band_step, outs));
    release(c, acc);
    return GALA_OK;
}

int gala_ct_export(gala_ctx* c, const uint64_t* ct, uint64_t* coef, int count)
{
    const int N = c->dc.N, L = c->dc.L;
    return launch_inv<false>(c, ct, coef, count * 2 * L, pm_make(2 * L, L, 0, 0, 2LL * L * N, 2LL * L * N));
}

int gala_ct_import(gala_ctx* c, const uint64_t* coef, uint64_t* ct, int count)
{
    const int N = c->dc.N, L = c->dc.L;
    return launch_fwd<u64, false>(c, coef, ct, count * 2 * L, pm_make(2 * L, L, 0, 0, 2LL * L * N, 2LL * L * N));
}

int gala_pt_export(gala_ctx* c, const uint64_t* pt, uint64_t* coef, int count)
{
    const int N = c->dc.N, L = c->dc.L;
    return launch_inv<true>(c, pt, coef, count * L, pm_make(L, L, 0, 0, (long long)L * N, (long long)L * N));
}

} // extern "C"
