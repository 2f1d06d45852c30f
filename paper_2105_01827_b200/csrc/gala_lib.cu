// gala_lib.cu -- host side of the B200-native GALA library: context, keys,
// op seam, fused GALA dot product and kernel-grouping convolution, C-ABI.
//
// Every schedule here mirrors the CPU oracle (oracle/bfv_oracle.c) operation
// for operation, so ciphertext words agree exactly.  See include/gala_b200.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
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

// launch with optional per-kernel CUDA-event timing (gala_profile_*)
#define KLAUNCH(ctx, name, ...)                                                                    \
    do {                                                                                           \
        cudaEvent_t ev0_ = nullptr, ev1_ = nullptr;                                                \
        if ((ctx)->prof_on) prof_begin((ctx), &ev0_, &ev1_);                                       \
        __VA_ARGS__;                                                                               \
        if ((ctx)->prof_on) prof_end((ctx), name, ev0_, ev1_);                                     \
        LAUNCHED();                                                                                \
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
    // ring of descriptor staging buffers: an upload waits only for the one GALA_STAGES uploads back, so
    // the host can enqueue a whole layer (several engine calls) ahead of the GPU
    static constexpr int GALA_STAGES = 16;
    Staging stage[GALA_STAGES];
    int stage_next = 0;
    int smem_ntt = 0;         // bytes of one padded polynomial
    cudaStream_t side = nullptr;              // independent work (mask encoding) overlapped with the layer
    // coefficient-domain finish (gala_mv_gala2_stream_host): when set, the final ModDown of the fused FC layer writes
    // masked canonical words here (k_moddown_coef) instead of NTT-form outputs; coef_m = the masks' coefficients mod p
    u64* coef_out = nullptr;
    uint32_t* coef_m = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // streamed host entry points: copy-in / copy-out streams and per-slot events (created on first use)
    cudaStream_t cs_in = nullptr, cs_out = nullptr;
    cudaEvent_t ev_h2d[2] = {}, ev_used[2] = {}, ev_done[2] = {}, ev_d2h[2] = {}, ev_alloc = nullptr;
    std::mutex mu;
    // per-kernel CUDA-event profiling
    bool prof_on = false;
    struct Rec {
        const char* name;
        cudaEvent_t a, b;
    };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
    u64* d_kg_off = nullptr;                  // per prime: multiple of q >= 2^90 (128-bit, hi/lo)
    int num_sms = 148;
    // tensor-core FC weights: key-folded (k_gala_kf, default) or the split E / MMA pair (GALA_FC_KF=0)
    bool fc_kf = true;
    int fc_tc_min_T = 128;                    // smallest T on the key-folded tensor-core tiles (gala_set_fc_tc_min_terms)
    int* d_kf_orb = nullptr;                  // NTT slot -> orbit * KF_ORB(N) + t (k_gala_dq / k_gala_kf)
};

static void prof_begin(gala_ctx* c, cudaEvent_t* a, cudaEvent_t* b)
{
    for (cudaEvent_t* e : {a, b}) {
        if (!c->pool.empty()) {
            *e = c->pool.back();
            c->pool.pop_back();
        } else {
            cudaEventCreate(e);
        }
    }
    cudaEventRecord(*a, c->stream);
}
static void prof_end(gala_ctx* c, const char* name, cudaEvent_t a, cudaEvent_t b)
{
    cudaEventRecord(b, c->stream);
    c->recs.push_back({name, a, b});
}

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
    Staging& s = c->stage[c->stage_next];
    c->stage_next = (c->stage_next + 1) % gala_ctx::GALA_STAGES;
    if (s.done) CK(cudaEventSynchronize(s.done)); // previous upload consumed
    if (bytes > s.cap) {
        if (s.host) cudaFreeHost(s.host);
        s.cap = bytes < (1 << 16) ? (1 << 16) : (bytes + 3) / 4 * 4;
        CK(cudaHostAlloc(&s.host, s.cap, cudaHostAllocMapped));
    }
    if (!s.done) CK(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
    memcpy(s.host, src, bytes);
    const size_t words = (bytes + 3) / 4;
    CK(cudaMallocAsync(dst, words * 4, c->stream));
    // read by the SMs straight from the mapped staging buffer, not by the copy engine: a layer's tables
    // must not wait behind a streamed batch's 13 MB input copy (gala_mv_gala2_stream_host)
    void* src_dev = nullptr;
    CK(cudaHostGetDevicePointer(&src_dev, s.host, 0));
    const int blocks = (int)((words + 255) / 256 < 32 ? (words + 255) / 256 : 32);
    k_h2d_copy<<<blocks, 256, 0, c->stream>>>((const uint32_t*)src_dev, (uint32_t*)*dst, (long long)words);
    CK(cudaGetLastError());
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
    pm.skip_first = 0;
    pm.skip_cnt = 0;
    pm.quad_G = 0;
    pm.quad_cc = 0;
    pm.quad_j = 0;
    return pm;
}

template <typename T, bool MONT>
static int launch_fwd(gala_ctx* c, const T* src, u64* dst, int polys, PolyMap pm, const char* tag = "k_ntt_fwd")
{
    if (polys <= 0) return GALA_OK;
    KLAUNCH(c, tag, k_ntt_fwd<T, MONT><<<polys, ntt_threads(c->dc.N), c->smem_ntt, c->stream>>>(c->dc, src, dst, pm));
    return GALA_OK;
}
template <bool MONT>
static int launch_inv(gala_ctx* c, const u64* src, u64* dst, int polys, PolyMap pm, const char* tag = "k_ntt_inv")
{
    if (polys <= 0) return GALA_OK;
    KLAUNCH(c, tag, k_ntt_inv<MONT><<<polys, ntt_threads(c->dc.N), c->smem_ntt, c->stream>>>(c->dc, src, dst, pm));
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

// ---------------------------------------------------------------------------
// Key-switch engine: any set of "terms" (X or X (.) pt), each rotated by one
// or more steps, summed into groups with one lazy ModDown per group.
//   group output = sum over members of rot_step(member)
// A member is either a rotation (term, r) or a step-0 term added directly.
struct EngTerm {
    const u64* X;
    const u64* pt;
    std::vector<int> steps;   // nonzero rotation steps of this term
    const u64* ntt_block;     // optional: precomputed identity block (hoisted DecPerm)
    bool c0_zero = false;     // X.c0 is zero: skip its sigma-copies and sums
};
struct EngMember {
    int term;
    int rot;                  // index into term.steps, or -1 for a step-0 member
};

static const u64* key_for(gala_ctx* c, int step);
// experiments: GALA_DEBUG_DUMP=prefix writes a device buffer to prefix_<tag>.bin (synchronous)
static void debug_dump(gala_ctx* c, const char* tag, const u64* d, size_t words)
{
    const char* pre = getenv("GALA_DEBUG_DUMP");
    if (!pre || !d) return;
    std::vector<u64> h(words);
    cudaStreamSynchronize(c->stream);
    cudaMemcpy(h.data(), d, words * 8, cudaMemcpyDeviceToHost);
    std::string fn = std::string(pre) + "_" + tag + ".bin";
    FILE* f = fopen(fn.c_str(), "wb");
    if (f) {
        fwrite(h.data(), 8, words, f);
        fclose(f);
    }
}
// key-folded tensor-core FC weights (k_gala_kf) for this context
static bool fc_kf_on(const gala_ctx* c) { return c->fc_kf && c->dc.L <= 3 && c->dc.N % 16 == 0 && c->dc.N >= 128; }

// The rotation orbits of the NTT slots (k_gala_dq): slot k has evaluation exponent e = 2 brv(k) + 1 mod 2N;
// the baby rotation sigma^jj multiplies it by 3^jj, so e = +-3^t splits the slots into orbit 0 (+) and
// orbit 1 (-) of length N / 2 each, and x_t (orbit o, index t) needs the blocks x_t .. x_t+63.
static int kf_orbit_table(gala_ctx* c, const int** out)
{
    if (!c->d_kf_orb) {
        const int N = c->dc.N, logN = c->dc.logN;
        const u64 twoN = 2 * (u64)N;
        std::vector<int> orb(N, -1);
        for (int o = 0; o < 2; o++) {
            u64 e = o == 0 ? 1 : twoN - 1;
            for (int t = 0; t < N / 2; t++) {
                const int k = h_brv((int)((e - 1) / 2), logN);
                orb[k] = o * KF_ORB(N) + t;
                e = (e * 3) % twoN;
            }
        }
        for (int k = 0; k < N; k++)
            if (orb[k] < 0) return set_err(GALA_ERR_PARAM, "internal: NTT slot %d outside the rotation orbits", k);
        CK(cudaMalloc(&c->d_kf_orb, sizeof(int) * N));
        CK(cudaMemcpy(c->d_kf_orb, orb.data(), sizeof(int) * N, cudaMemcpyHostToDevice));
    }
    *out = c->d_kf_orb;
    return GALA_OK;
}

static int moddown_groups(gala_ctx* c, u64* U, u64* Cacc, int G, u64* const* d_outs)
{
    const int N = c->dc.N, L = c->dc.L, M = c->dc.M;
    u64* r;
    RET(scratch(c, &r, (size_t)G * 2 * N));
    RET(launch_inv<false>(c, U + (long long)L * N, r, G * 2, pm_make(1, 1, L, 0, (long long)M * N, N),
                          "k_ntt_inv[moddown]"));
    MdArgs a{};
    a.r = r;
    a.U = U;
    a.add0 = Cacc;
    a.add1 = Cacc + (long long)L * N;
    a.add_is = 2LL * L * N;
    a.out = nullptr;
    a.out_is = 0;
    a.outs = d_outs;
    KLAUNCH(c, "k_moddown", k_moddown<<<G * 2 * L, ntt_threads(N), c->smem_ntt, c->stream>>>(c->dc, a));
    release(c, r);
    return GALA_OK;
}

// The fused form of rotate_engine (every rotated term has one rotation): k_digits_intt (digit
// coefficients only), k_ks_fused (digit NTTs + key inner product per (term, prime)), k_ks_sum (group
// sums with the step-0 members and addends), one lazy ModDown per group.  Same words.
static int rotate_engine_fused(gala_ctx* c, const std::vector<EngTerm>& terms,
                               const std::vector<std::vector<EngMember>>& groups, const std::vector<u64*>& outs,
                               const u64* qp_add, const u64* q_add)
{
    const int N = c->dc.N, L = c->dc.L, M = c->dc.M;
    const int G = (int)groups.size();
    std::vector<int> rot_idx(terms.size(), -1);
    int n_rot = 0;
    for (size_t t = 0; t < terms.size(); t++) {
        if (terms[t].steps.empty()) continue;
        if (!key_for(c, terms[t].steps[0])) return set_err(GALA_ERR_NOKEY, "missing rotation key for step %d", norm_step(c, terms[t].steps[0]));
        rot_idx[t] = n_rot++;
    }
    u64 *dig = nullptr, *part = nullptr, *cpart = nullptr;
    if (n_rot) {
        RET(scratch(c, &dig, (size_t)n_rot * L * N));
        RET(scratch(c, &part, (size_t)n_rot * 2 * M * N));
        RET(scratch(c, &cpart, (size_t)n_rot * L * N));
    }
    std::vector<TermDesc> td;
    std::vector<FusedTerm> ft;
    for (size_t t = 0; t < terms.size(); t++) {
        if (rot_idx[t] < 0) continue;
        TermDesc d{};
        d.X = terms[t].X;
        d.pt = terms[t].pt;
        d.dig = dig + (long long)rot_idx[t] * L * N;
        d.blk = nullptr;               // no sigma-copies: k_ks_fused reads the limbs itself
        d.rot_off = 0;
        d.rot_cnt = 0;
        td.push_back(d);
        FusedTerm f{};
        f.X = terms[t].X;
        f.pt = terms[t].pt;
        f.dig = d.dig;
        f.key = key_for(c, terms[t].steps[0]);
        f.gal = galois_of(c, terms[t].steps[0]);
        f.c0_zero = terms[t].c0_zero ? 1 : 0;
        ft.push_back(f);
    }
    std::vector<SumMember> mem;
    std::vector<int> off;
    for (const auto& g : groups) {
        off.push_back((int)mem.size());
        for (const auto& m : g) {
            const EngTerm& T = terms[m.term];
            SumMember sm{};
            if (m.rot < 0) {
                sm.X = T.X;
                sm.pt = T.pt;
            } else {
                const int r = rot_idx[m.term];
                sm.part = part + (long long)r * 2 * M * N;
                sm.cpart = T.c0_zero ? nullptr : cpart + (long long)r * L * N;
            }
            mem.push_back(sm);
        }
    }
    off.push_back((int)mem.size());
    auto align = [](size_t x) { return (x + 15) & ~(size_t)15; };
    const size_t o_td = 0, o_ft = align(td.size() * sizeof(TermDesc));
    const size_t o_mem = align(o_ft + ft.size() * sizeof(FusedTerm));
    const size_t o_off = align(o_mem + mem.size() * sizeof(SumMember));
    const size_t o_out = align(o_off + off.size() * sizeof(int));
    std::vector<char> blob(o_out + outs.size() * sizeof(u64*));
    if (!td.empty()) memcpy(blob.data() + o_td, td.data(), td.size() * sizeof(TermDesc));
    if (!ft.empty()) memcpy(blob.data() + o_ft, ft.data(), ft.size() * sizeof(FusedTerm));
    memcpy(blob.data() + o_mem, mem.data(), mem.size() * sizeof(SumMember));
    memcpy(blob.data() + o_off, off.data(), off.size() * sizeof(int));
    memcpy(blob.data() + o_out, outs.data(), outs.size() * sizeof(u64*));
    char* d_blob;
    RET(upload(c, blob.data(), blob.size(), (void**)&d_blob));
    if (n_rot) {
        const int nt = ntt_threads(N);
        KLAUNCH(c, "k_digits_intt", k_digits_intt<<<(unsigned)(n_rot * L), nt, c->smem_ntt, c->stream>>>(
                                        c->dc, (const TermDesc*)(d_blob + o_td), nullptr, 0));
        const size_t smem = (size_t)L * padded_words(N) * 8;
        const FusedTerm* dft = (const FusedTerm*)(d_blob + o_ft);
        // one CTA per SM (L smem polynomials): twice the NTT kernels' threads, so the SM keeps 32 warps
        const int ntf = N >= 1024 ? 2 * nt : nt;
        switch (L) {
            case 1: KLAUNCH(c, "k_ks_fused", (k_ks_fused<1><<<(unsigned)(n_rot * M), ntf, smem, c->stream>>>(c->dc, dft, part, cpart))); break;
            case 2: KLAUNCH(c, "k_ks_fused", (k_ks_fused<2><<<(unsigned)(n_rot * M), ntf, smem, c->stream>>>(c->dc, dft, part, cpart))); break;
            default: KLAUNCH(c, "k_ks_fused", (k_ks_fused<3><<<(unsigned)(n_rot * M), ntf, smem, c->stream>>>(c->dc, dft, part, cpart))); break;
        }
    }
    u64 *U, *Cacc;
    RET(scratch(c, &U, (size_t)G * 2 * M * N));
    RET(scratch(c, &Cacc, (size_t)G * 2 * L * N));
    const int th = N < 256 ? N : 256;
    KLAUNCH(c, "k_ks_sum", k_ks_sum<<<dim3((unsigned)((N + th - 1) / th), (unsigned)M, (unsigned)G), th, 0, c->stream>>>(
                               c->dc, (const SumMember*)(d_blob + o_mem), (const int*)(d_blob + o_off), U, Cacc, qp_add, q_add));
    release(c, dig);
    release(c, part);
    release(c, cpart);
    RET(moddown_groups(c, U, Cacc, G, (u64* const*)(d_blob + o_out)));
    release(c, U);
    release(c, Cacc);
    release(c, d_blob);
    return GALA_OK;
}

// qp_add [G][2][M][N] (optional) is added to each group's key-switch sum before its ModDown, q_add
// [G][2][L][N] (optional) after it.
static int rotate_engine(gala_ctx* c, const std::vector<EngTerm>& terms,
                         const std::vector<std::vector<EngMember>>& groups, const std::vector<u64*>& outs,
                         const u64* qp_add = nullptr, const u64* q_add = nullptr, u64* raw_U = nullptr,
                         u64* raw_C = nullptr)
{
    const int N = c->dc.N, L = c->dc.L, M = c->dc.M;
    const int G = (int)groups.size();
    if (G == 0) return GALA_OK;
    // every rotated term rotated by exactly one element, no hoisted identity block: the fused key
    // switch (digit NTTs + key inner product in one kernel, no permuted block in HBM)
    bool fusable = L <= 3 && getenv("GALA_KS_FUSED") != nullptr;
    for (const auto& t : terms)
        if (!t.steps.empty() && (t.steps.size() != 1 || t.ntt_block)) fusable = false;
    if (fusable && !raw_U) return rotate_engine_fused(c, terms, groups, outs, qp_add, q_add);
    const long long blk_words = (long long)(L * M + L) * N;
    // hoisted terms (several rotations of one decomposition): ONE identity block per term, and k_ks_mac
    // applies each member's sigma as a gather from it (the block stays in L2 while the term's rotations
    // run) instead of one sigma-permuted block per rotation in HBM.  GALA_KS_GATHER=0: permuted blocks.
    const bool gather = !(getenv("GALA_KS_GATHER") && getenv("GALA_KS_GATHER")[0] == '0');
    auto gathered = [&](const EngTerm& T) { return gather && T.steps.size() > 1; };
    // rotated terms and their rotation slices
    std::vector<int> term_rot_base(terms.size(), -1);
    int n_rot = 0, n_dig = 0;
    for (size_t t = 0; t < terms.size(); t++) {
        for (int s : terms[t].steps)
            if (!key_for(c, s)) return set_err(GALA_ERR_NOKEY, "missing rotation key for step %d", norm_step(c, s));
        if (!terms[t].steps.empty()) {
            if (gathered(terms[t]) && terms[t].ntt_block) continue;   // reads the caller's identity block
            term_rot_base[t] = n_rot;
            n_rot += gathered(terms[t]) ? 1 : (int)terms[t].steps.size();
            if (!terms[t].ntt_block) n_dig++;
        }
    }
    u64 *dig = nullptr, *blk = nullptr;
    if (n_dig) RET(scratch(c, &dig, (size_t)n_dig * L * N));
    if (n_rot) RET(scratch(c, &blk, (size_t)n_rot * blk_words));
    std::vector<TermDesc> td, td_hoisted;
    std::vector<unsigned> gal;
    int di = 0;
    for (size_t t = 0; t < terms.size(); t++) {
        if (terms[t].steps.empty()) continue;
        if (gathered(terms[t]) && terms[t].ntt_block) continue;
        TermDesc d{};
        d.X = terms[t].X;
        d.pt = terms[t].pt;
        d.c0_zero = terms[t].c0_zero ? 1 : 0;
        d.dig = terms[t].ntt_block ? nullptr : dig + (long long)(di++) * L * N;
        d.blk = blk + (long long)term_rot_base[t] * blk_words;
        d.rot_off = (int)gal.size();
        if (gathered(terms[t])) {   // the identity block only
            d.rot_cnt = 1;
            gal.push_back(1u);
        } else {
            d.rot_cnt = (int)terms[t].steps.size();
            for (int s : terms[t].steps) gal.push_back(galois_of(c, s));
        }
        if (terms[t].ntt_block) {
            d.X = terms[t].ntt_block;   // identity block as the permutation source
            td_hoisted.push_back(d);
        } else {
            td.push_back(d);
        }
    }
    std::vector<MacMember> mem;
    std::vector<int> off;
    // long groups (the conv second-Perm sums c_n - 1 rotations) are split into chunks of at most
    // kChunk rotated members, one k_ks_mac grid slice each, and the chunk sums folded afterwards:
    // each thread's serial member loop stays short
    const int kChunk = 16;
    const bool can_split = qp_add == nullptr && q_add == nullptr;
    std::vector<int> vstart, vcount;   // real group -> its virtual groups
    for (auto& g0 : groups) {
        std::vector<EngMember> g(g0);   // k_ks_mac expects the step-0 members first
        std::stable_partition(g.begin(), g.end(), [](const EngMember& m) { return m.rot < 0; });
        int n0 = 0;
        while (n0 < (int)g.size() && g[n0].rot < 0) n0++;
        const int nrot = (int)g.size() - n0;
        const int S = can_split && nrot > 2 * kChunk ? (nrot + kChunk - 1) / kChunk : 1;
        vstart.push_back((int)off.size());
        vcount.push_back(S);
        int mi = 0;
        for (int sidx = 0; sidx < S; sidx++) {
            off.push_back((int)mem.size());
            // chunk 0 takes the step-0 members; rotated members are dealt evenly
            const int r_lo = (int)((long long)nrot * sidx / S), r_hi = (int)((long long)nrot * (sidx + 1) / S);
            const int hi = n0 + r_hi;
            if (sidx == 0) mi = 0;
            else mi = n0 + r_lo;
            for (; mi < hi; mi++) {
                const EngMember& m = g[mi];
                MacMember mm{};
            const EngTerm& T = terms[m.term];
            if (m.rot < 0) {
                mm.blk = nullptr;
                mm.key = nullptr;
                mm.X = T.X;
                mm.pt = T.pt;
            } else {
                if (gathered(T)) {
                    mm.blk = T.ntt_block ? T.ntt_block : blk + (long long)term_rot_base[m.term] * blk_words;
                    mm.gal = galois_of(c, T.steps[m.rot]);
                } else {
                    mm.blk = blk + (long long)(term_rot_base[m.term] + m.rot) * blk_words;
                }
                mm.key = key_for(c, T.steps[m.rot]);
                mm.X = nullptr;
                mm.pt = nullptr;
                mm.no_c0 = T.c0_zero ? 1 : 0;
            }
            mem.push_back(mm);
            }
        }
    }
    off.push_back((int)mem.size());
    const int V = (int)off.size() - 1;   // virtual groups
    // one descriptor blob
    auto align = [](size_t x) { return (x + 15) & ~(size_t)15; };
    size_t o_td = 0, o_th = align(o_td + td.size() * sizeof(TermDesc));
    size_t o_gal = align(o_th + td_hoisted.size() * sizeof(TermDesc));
    size_t o_mem = align(o_gal + gal.size() * sizeof(unsigned));
    size_t o_off = align(o_mem + mem.size() * sizeof(MacMember));
    size_t o_out = align(o_off + off.size() * sizeof(int));
    size_t total = o_out + outs.size() * sizeof(u64*);
    std::vector<char> blob(total);
    if (!td.empty()) memcpy(blob.data() + o_td, td.data(), td.size() * sizeof(TermDesc));
    if (!td_hoisted.empty()) memcpy(blob.data() + o_th, td_hoisted.data(), td_hoisted.size() * sizeof(TermDesc));
    if (!gal.empty()) memcpy(blob.data() + o_gal, gal.data(), gal.size() * sizeof(unsigned));
    memcpy(blob.data() + o_mem, mem.data(), mem.size() * sizeof(MacMember));
    memcpy(blob.data() + o_off, off.data(), off.size() * sizeof(int));
    memcpy(blob.data() + o_out, outs.data(), outs.size() * sizeof(u64*));
    char* d_blob;
    RET(upload(c, blob.data(), total, (void**)&d_blob));
    const int nt = ntt_threads(N);
    if (!td.empty()) {
        KLAUNCH(c, "k_digits_intt", k_digits_intt<<<(unsigned)(td.size() * L), nt, c->smem_ntt, c->stream>>>(
                                        c->dc, (const TermDesc*)(d_blob + o_td), (const unsigned*)(d_blob + o_gal),
                                        blk_words));
        KLAUNCH(c, "k_digits_perm", k_digits_perm<<<(unsigned)(td.size() * L * L), nt, c->smem_ntt,
                                                    c->stream>>>(c->dc, (const TermDesc*)(d_blob + o_td),
                                                                 (const unsigned*)(d_blob + o_gal), blk_words));
    }
    if (!td_hoisted.empty()) {
        KLAUNCH(c, "k_block_perm", k_block_perm<<<(unsigned)(td_hoisted.size() * (L * M + L)), nt, c->smem_ntt,
                                                  c->stream>>>(c->dc, (const TermDesc*)(d_blob + o_th),
                                                               (const unsigned*)(d_blob + o_gal), blk_words));
    }
    u64 *U, *Cacc, *r, *Uv = nullptr, *Cv = nullptr;
    RET(scratch(c, &U, (size_t)G * 2 * M * N));
    RET(scratch(c, &Cacc, (size_t)G * 2 * L * N));
    RET(scratch(c, &r, (size_t)G * 2 * N));
    if (V > G) {
        RET(scratch(c, &Uv, (size_t)V * 2 * M * N));
        RET(scratch(c, &Cv, (size_t)V * 2 * L * N));
    }
    const int th = N < 256 ? N : 256;
    dim3 grid((N + th - 1) / th, M, V);
    {
        u64* const Uo = V > G ? Uv : U;
        u64* const Co = V > G ? Cv : Cacc;
        const MacMember* dm = (const MacMember*)(d_blob + o_mem);
        const int* doff = (const int*)(d_blob + o_off);
        bool any_gather = false;
        for (const auto& m : mem) any_gather = any_gather || m.gal > 1u;
        // uniform hoisted rotations (every term rotated by the same steps, gathered, one member per group,
        // groups term-major, no addends): k_ks_hoist reuses each step's key words across up to 8 terms
        const int R = terms.empty() ? 0 : (int)terms[0].steps.size();
        bool hoist = any_gather && V == G && qp_add == nullptr && q_add == nullptr && !raw_U && R > 1 &&
                     (long long)terms.size() * R == G && getenv("GALA_KS_HOIST") == nullptr;
        for (size_t t = 0; hoist && t < terms.size(); t++)
            hoist = gathered(terms[t]) && terms[t].steps == terms[0].steps && terms[t].c0_zero == terms[0].c0_zero;
        for (int g = 0; hoist && g < G; g++)
            hoist = groups[g].size() == 1 && groups[g][0].term == g / R && groups[g][0].rot == g % R;
        // giant steps of a batch (every group sums the same R single-step terms, term-major, no gather, no
        // step-0 members): k_ks_giant reuses each key word across KG_IB groups
        const int Rg = G > 0 ? (int)groups[0].size() : 0;
        // GALA_KS_GIANT: unset -> when the grid fills the GPU; "force" -> always (tests); anything else -> never
        const char* ge = getenv("GALA_KS_GIANT");
        const bool g_force = ge && strcmp(ge, "force") == 0;
        bool giant = !any_gather && V == G && Rg >= 1 && (long long)Rg * G == (long long)terms.size() && !raw_U &&
                     (ge == nullptr || g_force) &&
                     (g_force || (long long)((N + th - 1) / th) * M * ((G + KG_IB - 1) / KG_IB) >= 2LL * c->num_sms);
        for (size_t t = 0; giant && t < terms.size(); t++)
            giant = terms[t].steps.size() == 1 && !terms[t].ntt_block && terms[t].steps[0] == terms[t % Rg].steps[0] &&
                    terms[t].c0_zero == terms[0].c0_zero;
        for (int g = 0; giant && g < G; g++) {
            giant = (int)groups[g].size() == Rg;
            for (int r = 0; giant && r < Rg; r++) giant = groups[g][r].term == g * Rg + r && groups[g][r].rot == 0;
        }
        if (giant) {
            std::vector<const u64*> gb(terms.size()), gk(Rg);
            for (size_t t = 0; t < terms.size(); t++) gb[t] = blk + (long long)term_rot_base[t] * blk_words;
            for (int r = 0; r < Rg; r++) gk[r] = key_for(c, terms[r].steps[0]);
            std::vector<const u64*> gall(gb);
            gall.insert(gall.end(), gk.begin(), gk.end());
            char* d_g;
            RET(upload(c, gall.data(), gall.size() * sizeof(u64*), (void**)&d_g));
            const u64* const* d_gb = (const u64* const*)d_g;
            const u64* const* d_gk = d_gb + gb.size();
            const dim3 gg((unsigned)((N + th - 1) / th), (unsigned)M, (unsigned)((G + KG_IB - 1) / KG_IB));
            const int nc0 = terms[0].c0_zero ? 1 : 0;
#define KSG(LL) KLAUNCH(c, "k_ks_mac", (k_ks_giant<LL><<<gg, th, 0, c->stream>>>(c->dc, d_gb, d_gk, Rg, G, nc0, U, Cacc, qp_add, q_add)))
            switch (L) {
                case 1: KSG(1); break;
                case 2: KSG(2); break;
                case 3: KSG(3); break;
                default: KSG(4); break;
            }
#undef KSG
            release(c, d_g);
        } else if (hoist) {
            std::vector<const u64*> hb(terms.size()), hk(R);
            std::vector<unsigned> hg(R);
            for (size_t t = 0; t < terms.size(); t++)
                hb[t] = terms[t].ntt_block ? terms[t].ntt_block : blk + (long long)term_rot_base[t] * blk_words;
            for (int r = 0; r < R; r++) {
                hk[r] = key_for(c, terms[0].steps[r]);
                hg[r] = galois_of(c, terms[0].steps[r]);
            }
            std::vector<char> hbl(sizeof(u64*) * (hb.size() + R) + sizeof(unsigned) * R);
            memcpy(hbl.data(), hb.data(), sizeof(u64*) * hb.size());
            memcpy(hbl.data() + sizeof(u64*) * hb.size(), hk.data(), sizeof(u64*) * R);
            memcpy(hbl.data() + sizeof(u64*) * (hb.size() + R), hg.data(), sizeof(unsigned) * R);
            char* d_h;
            RET(upload(c, hbl.data(), hbl.size(), (void**)&d_h));
            const u64* const* d_hb = (const u64* const*)d_h;
            const u64* const* d_hk = d_hb + hb.size();
            const unsigned* d_hg = (const unsigned*)(d_hk + R);
            const int nterms = (int)terms.size(), nc0 = terms[0].c0_zero ? 1 : 0;
            const long long xy = (long long)((N + th - 1) / th) * M;
            int tb = 8;   // terms per thread: key reuse, unless the grid would then underfill the GPU
            while (tb > 1 && xy * ((nterms + tb - 1) / tb) < 2LL * c->num_sms) tb /= 2;
            const dim3 gh((unsigned)((N + th - 1) / th), (unsigned)M, (unsigned)((nterms + tb - 1) / tb));
#define KSH(LL) KLAUNCH(c, "k_ks_mac", (k_ks_hoist<LL><<<gh, th, 0, c->stream>>>(c->dc, d_hb, d_hg, d_hk, R, nterms, tb, nc0, U, Cacc)))
            switch (L) {
                case 1: KSH(1); break;
                case 2: KSH(2); break;
                case 3: KSH(3); break;
                default: KSH(4); break;
            }
#undef KSH
            release(c, d_h);
        } else {
#define KSMAC(LL)                                                                                                   \
    do {                                                                                                            \
        if (any_gather)                                                                                             \
            KLAUNCH(c, "k_ks_mac", (k_ks_mac<LL, true><<<grid, th, 0, c->stream>>>(c->dc, dm, doff, Uo, Co, qp_add, q_add))); \
        else                                                                                                        \
            KLAUNCH(c, "k_ks_mac", (k_ks_mac<LL, false><<<grid, th, 0, c->stream>>>(c->dc, dm, doff, Uo, Co, qp_add, q_add))); \
    } while (0)
        switch (L) {
            case 1: KSMAC(1); break;
            case 2: KSMAC(2); break;
            case 3: KSMAC(3); break;
            default: KSMAC(4); break;
        }
#undef KSMAC
        }
    }
    if (V > G) {   // fold the chunk sums of every split group
        int* d_vsc;
        std::vector<int> vsc(vstart);
        vsc.insert(vsc.end(), vcount.begin(), vcount.end());
        RET(upload(c, vsc.data(), vsc.size() * sizeof(int), (void**)&d_vsc));
        KLAUNCH(c, "k_fold_groups", k_fold_groups<<<dim3((unsigned)((N + th - 1) / th), (unsigned)M, (unsigned)G), th, 0,
                                                    c->stream>>>(c->dc, Uv, Cv, d_vsc, d_vsc + G, U, Cacc));
        release(c, d_vsc);
        release(c, Uv);
        release(c, Cv);
    }
    if (raw_U) {   // multi-GPU partial: the groups' QP sums and Q addends before any ModDown
        CK(cudaMemcpyAsync(raw_U, U, sizeof(u64) * (size_t)G * 2 * M * N, cudaMemcpyDeviceToDevice, c->stream));
        CK(cudaMemcpyAsync(raw_C, Cacc, sizeof(u64) * (size_t)G * 2 * L * N, cudaMemcpyDeviceToDevice, c->stream));
    } else if (c->coef_out) {
        // results leave as canonical words: INTT every limb of the QP sums, then ModDown and the mask pointwise
        // in the coefficient domain (same words; no NTT of the lifted P limb, no export INTT)
        if (q_add) return set_err(GALA_ERR_PARAM, "internal: coefficient-domain finish with a Q-side addend");
        for (const EngTerm& t : terms)
            if (!t.c0_zero || t.steps.empty())
                return set_err(GALA_ERR_PARAM, "internal: coefficient-domain finish needs rotated terms without c0");
        u64* Uc;
        RET(scratch(c, &Uc, (size_t)G * 2 * M * N));
        RET(launch_inv<false>(c, U, Uc, G * 2 * M, pm_make(2 * M, M, 0, 0, 2LL * M * N, 2LL * M * N), "k_ntt_inv[moddown]"));
        if (c->coef_m) CK(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
        KLAUNCH(c, "k_moddown", k_moddown_coef<<<grid_for((long long)G * 2 * N, 256), 256, 0, c->stream>>>(
                                    c->dc, Uc, c->coef_m, c->coef_out, G));
        release(c, Uc);
    } else {
    RET(launch_inv<false>(c, U + (long long)L * N, r, G * 2, pm_make(1, 1, L, 0, (long long)M * N, N),
                          "k_ntt_inv[moddown]"));
    MdArgs a{};
    a.r = r;
    a.U = U;
    a.add0 = Cacc;
    a.add1 = Cacc + (long long)L * N;
    a.add_is = 2LL * L * N;
    a.out = nullptr;
    a.out_is = 0;
    a.outs = (u64* const*)(d_blob + o_out);
    KLAUNCH(c, "k_moddown", k_moddown<<<G * 2 * L, nt, c->smem_ntt, c->stream>>>(c->dc, a));
    }
    release(c, U);
    release(c, Cacc);
    release(c, r);
    release(c, dig);
    release(c, blk);
    release(c, d_blob);
    return GALA_OK;
}

static const u64* key_for(gala_ctx* c, int step)
{
    auto it = c->keys.find(norm_step(c, step));
    return it == c->keys.end() ? nullptr : it->second;
}

// For each batch element b and group g:
//   out_b[g] = sum_{j < per} rot_{j * unit}(X_b[g * per + j] (.) pt[g * per + j]),
// one lazy ModDown per (b, g); all batch elements share the launches.
static int rotate_sum_regular(gala_ctx* c, const u64* X, long long x_stride, long long x_bstride, const u64* pts,
                              int B, int G, int per, int unit, u64* out, long long out_bstride)
{
    const int N = c->dc.N, L = c->dc.L;
    const long long W = 2LL * L * N, PW = (long long)L * N;
    std::vector<EngTerm> terms;
    std::vector<std::vector<EngMember>> groups((size_t)B * G);
    std::vector<u64*> outs;
    terms.reserve((size_t)B * G * per);
    for (int b = 0; b < B; b++)
        for (int g = 0; g < G; g++) {
            auto& grp = groups[(size_t)b * G + g];
            for (int j = 0; j < per; j++) {
                const int idx = g * per + j;
                EngTerm t;
                t.X = X + b * x_bstride + (long long)idx * x_stride;
                t.pt = pts ? pts + (long long)idx * PW : nullptr;
                t.ntt_block = nullptr;
                int s = norm_step(c, j * unit);
                if (s) t.steps.push_back(s);
                terms.push_back(t);
                grp.push_back({(int)terms.size() - 1, s ? 0 : -1});
            }
            outs.push_back(out + b * out_bstride + (long long)g * W);
        }
    return rotate_engine(c, terms, groups, outs);
}

// Delta encode(r[b]) for a batch, issued on the side stream so it overlaps the layer; the main
// stream joins before the subtraction (mask_finish).  DM is allocated on the main stream first.
static int mask_begin(gala_ctx* c, const uint32_t* r, int B, u64** DM)
{
    const int N = c->dc.N, L = c->dc.L;
    RET(scratch(c, DM, (size_t)B * L * N));
    CK(cudaEventRecord(c->ev_fork, c->stream));
    CK(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    cudaStream_t main = c->stream;
    cudaEvent_t a = nullptr, b = nullptr;
    c->stream = c->side;   // profiling events belong on the side stream
    uint32_t* mcoef;
    int rs = scratch(c, &mcoef, (size_t)B * N);   // B x N u32 coefficients
    if (rs != GALA_OK) {
        c->stream = main;
        return rs;
    }
    if (c->prof_on) prof_begin(c, &a, &b);
    k_encode_p<<<B, ntt_threads(N), c->smem_ntt, c->side>>>(c->dc, r, mcoef);
    k_encode_q<<<B * L, ntt_threads(N), c->smem_ntt, c->side>>>(c->dc, mcoef, *DM);
    if (c->prof_on) prof_end(c, "k_encode", a, b);
    release(c, mcoef);
    c->stream = main;
    g_launches += 2;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(GALA_ERR_CUDA, "kernel launch failed: %s", cudaGetErrorString(e));
    CK(cudaEventRecord(c->ev_join, c->side));
    return GALA_OK;
}
static int mask_finish(gala_ctx* c, const u64* ct, u64* DM, int B, u64* out)
{
    const int N = c->dc.N, L = c->dc.L;
    const long long W = 2LL * L * N;
    CK(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
    KLAUNCH(c, "k_sub_plain", k_sub_plain<<<grid_for((long long)B * W, 256), 256, 0, c->stream>>>(c->dc, ct, DM, out, B));
    release(c, DM);
    return GALA_OK;
}

// The coefficient-domain finish needs only the masks' coefficients mod p (k_encode_p), on the side stream
static int mask_begin_coef(gala_ctx* c, const uint32_t* r, int B, uint32_t** mcoef)
{
    const int N = c->dc.N;
    RET(scratch(c, mcoef, (size_t)B * N));
    CK(cudaEventRecord(c->ev_fork, c->stream));
    CK(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
    cudaStream_t main = c->stream;
    cudaEvent_t a = nullptr, b = nullptr;
    c->stream = c->side;
    if (c->prof_on) prof_begin(c, &a, &b);
    k_encode_p<<<B, ntt_threads(N), c->smem_ntt, c->side>>>(c->dc, r, *mcoef);
    if (c->prof_on) prof_end(c, "k_encode", a, b);
    c->stream = main;
    g_launches += 1;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_err(GALA_ERR_CUDA, "kernel launch failed: %s", cudaGetErrorString(e));
    CK(cudaEventRecord(c->ev_join, c->side));
    return GALA_OK;
}

// masked[b] = ct[b] - Delta encode(r[b]) for a batch (one encode launch for all b)
static int sub_plain_batch(gala_ctx* c, const u64* ct, const uint32_t* r, int B, u64* out)
{
    const int N = c->dc.N, L = c->dc.L;
    const long long W = 2LL * L * N, LN = (long long)L * N;
    u64* DM;
    RET(scratch(c, &DM, (size_t)B * LN));
    uint32_t* mcoef;
    RET(scratch(c, &mcoef, (size_t)B * N));
    KLAUNCH(c, "k_encode", k_encode_p<<<B, ntt_threads(N), c->smem_ntt, c->stream>>>(c->dc, r, mcoef));
    KLAUNCH(c, "k_encode", k_encode_q<<<B * L, ntt_threads(N), c->smem_ntt, c->stream>>>(c->dc, mcoef, DM));
    release(c, mcoef);
    KLAUNCH(c, "k_sub_plain", k_sub_plain<<<grid_for((long long)B * W, 256), 256, 0, c->stream>>>(c->dc, ct, DM, out, B));
    release(c, DM);
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
    if (c->d_kf_orb) cudaFree(c->d_kf_orb);
    for (Staging& st : c->stage) {
        if (st.host) cudaFreeHost(st.host);
        if (st.done) cudaEventDestroy(st.done);
    }
    if (c->side) {
        cudaStreamSynchronize(c->side);
        cudaStreamDestroy(c->side);
    }
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    for (cudaStream_t st : {c->cs_in, c->cs_out})
        if (st) {
            cudaStreamSynchronize(st);
            cudaStreamDestroy(st);
        }
    for (int i = 0; i < 2; i++)
        for (cudaEvent_t e : {c->ev_h2d[i], c->ev_used[i], c->ev_done[i], c->ev_d2h[i]})
            if (e) cudaEventDestroy(e);
    if (c->ev_alloc) cudaEventDestroy(c->ev_alloc);
    for (auto& r : c->recs) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto e : c->pool) cudaEventDestroy(e);
    if (c->d_kg_off) cudaFree(c->d_kg_off);
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
        if ((primes[j] & 0xffffffffull) != 1)
            return set_err(GALA_ERR_PARAM, "prime %d is not of the special form a*2^32 + 1 required by the NTT", j);
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
        {
            u128 kmax = (((u128)1) << 64) / q; // k q < 2^64  =>  k products of (< q) x (< q) stay below q 2^64
            d.lazy[j] = (int)(kmax > 64 ? 64 : kmax) - 1;
            if (d.lazy[j] < 1) d.lazy[j] = 1;
        }
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
    CKC(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    CKC(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    CKC(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
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
    // opt in to large dynamic shared memory for every NTT-carrying kernel.  The attribute is
    // process-global per function, so always request the largest ring (N = 8192): contexts of
    // different N coexist.
    const int kMaxSmem = padded_words(8192) * (int)sizeof(u64);
    CKC(cudaFuncSetAttribute(k_ntt_fwd<u64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    CKC(cudaFuncSetAttribute(k_ntt_fwd<u64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    CKC(cudaFuncSetAttribute(k_ntt_fwd<i64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    CKC(cudaFuncSetAttribute(k_ntt_fwd<int8_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    CKC(cudaFuncSetAttribute(k_ntt_inv<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    CKC(cudaFuncSetAttribute(k_ntt_inv<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    CKC(cudaFuncSetAttribute(k_moddown, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    CKC(cudaFuncSetAttribute(k_gala_tc<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, GTC_SMEM));
    CKC(cudaFuncSetAttribute(k_gala_tc<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, GTC_SMEM));
    CKC(cudaFuncSetAttribute(k_gala_tc<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, GTC_SMEM));
#define ZY2_ATTR1(LL, LN, PR) CKC(cudaFuncSetAttribute(k_kg_zy2<LL, LN, PR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * KG_PT * KG_KT * 8))
#define ZY2_ATTR(LL, LN) ZY2_ATTR1(LL, LN, false); ZY2_ATTR1(LL, LN, true)
    ZY2_ATTR(1, 0); ZY2_ATTR(1, 12); ZY2_ATTR(1, 13);
    ZY2_ATTR(2, 0); ZY2_ATTR(2, 12); ZY2_ATTR(2, 13);
    ZY2_ATTR(3, 0); ZY2_ATTR(3, 12); ZY2_ATTR(3, 13);
    ZY2_ATTR(4, 0); ZY2_ATTR(4, 12); ZY2_ATTR(4, 13);
#undef ZY2_ATTR
#undef ZY2_ATTR1
    CKC(cudaFuncSetAttribute(k_ks_fused<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    CKC(cudaFuncSetAttribute(k_ks_fused<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kMaxSmem));
    CKC(cudaFuncSetAttribute(k_ks_fused<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * kMaxSmem));
    CKC(cudaFuncSetAttribute(k_gala_tcf<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, GTC_SMEM));
    CKC(cudaFuncSetAttribute(k_gala_tcf<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, GTC_SMEM));
    CKC(cudaFuncSetAttribute(k_gala_tcf<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, GTC_SMEM));
    CKC(cudaFuncSetAttribute(k_gala_tcf<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, GTC_SMEM));
    CKC(cudaFuncSetAttribute(k_gala_tc<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, GTC_SMEM));
    CKC(cudaFuncSetAttribute(k_gala_kf<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, KF_SMEM));
    CKC(cudaFuncSetAttribute(k_gala_kf<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, KF_SMEM));
    CKC(cudaFuncSetAttribute(k_gala_kf<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, KF_SMEM));
    CKC(cudaFuncSetAttribute(k_gala_dq<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, KF_DQ_SMEM));  // 64 KB
    CKC(cudaFuncSetAttribute(k_gala_dq<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, KF_DQ_SMEM));
    CKC(cudaFuncSetAttribute(k_gala_dq<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, KF_DQ_SMEM));
    {
        const char* e = getenv("GALA_FC_KF");
        c->fc_kf = !(e && e[0] == '0');
    }
    CKC(cudaFuncSetAttribute(k_kg1_tc<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CKC(cudaFuncSetAttribute(k_kg1_tc<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CKC(cudaFuncSetAttribute(k_kg1_tc<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    CKC(cudaFuncSetAttribute(k_kg_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             KG_TC_STAGES * KG_TC_KCS * (128 + KG_TC_N) * 16 + 2 * 512 * 32));
    {
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        c->num_sms = sms > 0 ? sms : 148;
    }
    CKC(cudaFuncSetAttribute(k_digits_intt, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    CKC(cudaFuncSetAttribute(k_digits_perm, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    CKC(cudaFuncSetAttribute(k_block_perm, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    CKC(cudaFuncSetAttribute(k_encode<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kMaxSmem));
    CKC(cudaFuncSetAttribute(k_encode<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kMaxSmem));
    CKC(cudaFuncSetAttribute(k_encode_p, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    CKC(cudaFuncSetAttribute(k_encode_q, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    CKC(cudaFuncSetAttribute(k_encode<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kMaxSmem));
    CKC(cudaFuncSetAttribute(k_dec_phase1, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
    CKC(cudaFuncSetAttribute(k_dec_phase2, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
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
    KLAUNCH(c, "k_keygen_combine", k_keygen_combine<<<grid_for((long long)L * M * N, 256), 256, 0, c->stream>>>(c->dc, A, E, galois_of(c, s),
                                                                                 c->d_pmod, key));
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
    KLAUNCH(c, "k_encode", k_encode<0><<<B * c->dc.L, ntt_threads(c->dc.N), 2 * c->smem_ntt, c->stream>>>(c->dc, slots, pt));
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
    KLAUNCH(c, "k_encode", k_encode<1><<<L, ntt_threads(N), 2 * c->smem_ntt, c->stream>>>(c->dc, slots, DM));
    KLAUNCH(c, "k_encrypt_combine", k_encrypt_combine<<<grid_for((long long)L * N, 256), 256, 0, c->stream>>>(c->dc, A, E, DM, ct));
    release(c, A);
    release(c, E);
    release(c, DM);
    return GALA_OK;
}

static int decrypt_run(gala_ctx* c, const uint64_t* ct, uint32_t* slots, double* noise_frac)
{
    if (!c->has_secret) return set_err(GALA_ERR_STATE, "secret key not set");
    const int N = c->dc.N, L = c->dc.L;
    u64* x;
    unsigned long long* maxd = nullptr;
    RET(scratch(c, &x, (size_t)L * N));
    if (noise_frac) {
        RET(scratch(c, &maxd, 1));
        CK(cudaMemsetAsync(maxd, 0, sizeof(unsigned long long), c->stream));
    }
    KLAUNCH(c, "k_dec_phase1", k_dec_phase1<<<L, ntt_threads(N), c->smem_ntt, c->stream>>>(c->dc, ct, x));
    KLAUNCH(c, "k_dec_phase2", k_dec_phase2<<<1, ntt_threads(N), c->smem_ntt, c->stream>>>(c->dc, x, slots, maxd));
    release(c, x);
    if (noise_frac) {
        unsigned long long h = 0;
        CK(cudaMemcpyAsync(&h, maxd, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
        release(c, maxd);
        CK(cudaStreamSynchronize(c->stream));
        *noise_frac = (double)h / 18446744073709551616.0;
    }
    return GALA_OK;
}

int gala_decrypt(gala_ctx* c, const uint64_t* ct, uint32_t* slots) { return decrypt_run(c, ct, slots, nullptr); }

int gala_decrypt_noise(gala_ctx* c, const uint64_t* ct, uint32_t* slots, double* noise_frac)
{
    if (!noise_frac) return set_err(GALA_ERR_PARAM, "noise_frac must not be null");
    return decrypt_run(c, ct, slots, noise_frac);
}

int gala_add(gala_ctx* c, const uint64_t* a, const uint64_t* b, uint64_t* out)
{
    long long total = 2LL * c->dc.L * c->dc.N;
    KLAUNCH(c, "k_addsub", k_addsub<<<grid_for(total, 256), 256, 0, c->stream>>>(c->dc, a, b, out, total, c->dc.L, 1));
    return GALA_OK;
}

int gala_scmult(gala_ctx* c, const uint64_t* ct, const uint64_t* pt, uint64_t* out)
{
    const int N = c->dc.N, L = c->dc.L;
    dim3 grid((2 * L * N + 255) / 256, 1);
    KLAUNCH(c, "k_ct_mul_pts", k_ct_mul_pts<<<grid, 256, 0, c->stream>>>(c->dc, ct, pt, out));
    return GALA_OK;
}

int gala_sub_plain(gala_ctx* c, const uint64_t* ct, const uint32_t* r, uint64_t* out)
{
    const int N = c->dc.N, L = c->dc.L;
    u64* DM;
    RET(scratch(c, &DM, (size_t)L * N));
    KLAUNCH(c, "k_encode", k_encode<1><<<L, ntt_threads(N), 2 * c->smem_ntt, c->stream>>>(c->dc, r, DM));
    if (out != ct) CK(cudaMemcpyAsync(out + (long long)L * N, ct + (long long)L * N, sizeof(u64) * L * N,
                                      cudaMemcpyDeviceToDevice, c->stream));
    long long total = (long long)L * N;
    KLAUNCH(c, "k_addsub", k_addsub<<<grid_for(total, 256), 256, 0, c->stream>>>(c->dc, ct, DM, out, total, L, -1));
    release(c, DM);
    return GALA_OK;
}

size_t gala_digits_words(gala_ctx* c) { return (size_t)(c->dc.L * c->dc.M + c->dc.L) * c->dc.N; }

// DecPerm: the identity-permuted digit block [(L*M + L)][N] (NTT digits of c1, then c0)
int gala_decompose(gala_ctx* c, const uint64_t* ct, uint64_t* digits)
{
    const int N = c->dc.N, L = c->dc.L, M = c->dc.M;
    u64* dig;
    RET(scratch(c, &dig, (size_t)L * N));
    TermDesc d{};
    d.X = ct;
    d.pt = nullptr;
    d.dig = dig;
    d.blk = digits;
    d.rot_off = 0;
    d.rot_cnt = 1;
    struct {
        TermDesc t{};
        unsigned g;
    } b = {d, 1u};
    char* d_blob;
    RET(upload(c, &b, sizeof(b), (void**)&d_blob));
    const int nt = ntt_threads(N);
    const unsigned* dg = (const unsigned*)(d_blob + offsetof(decltype(b), g));
    const long long bw = (long long)(L * M + L) * N;
    KLAUNCH(c, "k_digits_intt", k_digits_intt<<<L, nt, c->smem_ntt, c->stream>>>(c->dc, (const TermDesc*)d_blob, dg, bw));
    KLAUNCH(c, "k_digits_perm", k_digits_perm<<<L * L, nt, c->smem_ntt, c->stream>>>(c->dc, (const TermDesc*)d_blob,
                                                                                     dg, bw));
    release(c, dig);
    release(c, d_blob);
    return GALA_OK;
}

// HstPerm: rotation of the group's source from its DecPerm block
int gala_rotate_hoisted(gala_ctx* c, const uint64_t* ct, const uint64_t* digits, int step, uint64_t* out)
{
    const int N = c->dc.N, L = c->dc.L;
    int s = norm_step(c, step);
    if (s == 0) {
        if (out != ct) CK(cudaMemcpyAsync(out, ct, sizeof(u64) * 2 * L * N, cudaMemcpyDeviceToDevice, c->stream));
        return GALA_OK;
    }
    EngTerm t;
    t.X = ct;
    t.pt = nullptr;
    t.steps = {s};
    t.ntt_block = digits;
    return rotate_engine(c, {t}, {{{0, 0}}}, {out});
}

// Batched hoisted rotations: every input decomposed once, rotated by every step (one full key switch
// with its own ModDown per output).  outs [B][S][2][L][N].  Same words as gala_rotate per (input, step).
int gala_rotate_batch(gala_ctx* c, const uint64_t* cts, int B, const int* steps_host, int S, uint64_t* outs)
{
    const int N = c->dc.N, L = c->dc.L;
    const long long W = 2LL * L * N;
    if (B <= 0 || S <= 0) return set_err(GALA_ERR_DIM, "empty rotation batch");
    std::vector<int> st(S);
    for (int i = 0; i < S; i++) {
        st[i] = norm_step(c, steps_host[i]);
        if (st[i] == 0) return set_err(GALA_ERR_PARAM, "step %d is the identity", steps_host[i]);
        if (!key_for(c, st[i])) return set_err(GALA_ERR_NOKEY, "missing rotation key for step %d", st[i]);
    }
    std::vector<EngTerm> terms(B);
    std::vector<std::vector<EngMember>> groups;
    std::vector<u64*> o;
    for (int b = 0; b < B; b++) {
        terms[b].X = cts + b * W;
        terms[b].pt = nullptr;
        terms[b].ntt_block = nullptr;
        terms[b].steps = st;
        for (int i = 0; i < S; i++) {
            groups.push_back({{b, i}});
            o.push_back(outs + ((long long)b * S + i) * W);
        }
    }
    return rotate_engine(c, terms, groups, o);
}

int gala_rotate(gala_ctx* c, const uint64_t* ct, int step, uint64_t* out)
{
    const int N = c->dc.N, L = c->dc.L;
    int s = norm_step(c, step);
    if (s == 0) {
        if (out != ct) CK(cudaMemcpyAsync(out, ct, sizeof(u64) * 2 * L * N, cudaMemcpyDeviceToDevice, c->stream));
        return GALA_OK;
    }
    EngTerm t;
    t.X = ct;
    t.pt = nullptr;
    t.steps = {s};
    t.ntt_block = nullptr;
    return rotate_engine(c, {t}, {{{0, 0}}}, {out});
}

int gala_bsgs_baby(int T)
{
    int lg = 0;
    while ((1 << lg) < T) lg++;
    return 1 << ((lg + 1) / 2);
}

int gala_mv_gala_batch(gala_ctx* c, const uint64_t* cts, int B, const uint64_t* pts, int T, int baby,
                       const uint32_t* r, uint64_t* outs, uint64_t* masked)
{
    const int N = c->dc.N, L = c->dc.L;
    if (T <= 0 || B <= 0) return set_err(GALA_ERR_DIM, "T and B must be positive");
    if (baby <= 0) baby = gala_bsgs_baby(T);
    if (T % baby) return set_err(GALA_ERR_PARAM, "baby step %d does not divide T=%d", baby, T);
    const int G = T / baby;
    const long long W = 2LL * L * N;
    for (int j = 1; j < baby; j++)
        if (!gala_has_rotation_key(c, j)) return set_err(GALA_ERR_NOKEY, "missing rotation key for step %d", j);
    for (int g = 1; g < G; g++)
        if (!gala_has_rotation_key(c, g * baby))
            return set_err(GALA_ERR_NOKEY, "missing rotation key for step %d", norm_step(c, g * baby));
    u64* DM = nullptr;
    if (r && masked) RET(mask_begin(c, r, B, &DM));   // overlaps the layer on the side stream
    if (T == 1) {
        for (int b = 0; b < B; b++) {
            dim3 grid((unsigned)((2 * L * N + 255) / 256), 1);
            KLAUNCH(c, "k_ct_mul_pts", k_ct_mul_pts<<<grid, 256, 0, c->stream>>>(c->dc, cts + b * W, pts, outs + b * W));
        }
    } else if (G == 1) {
        RET(rotate_sum_regular(c, cts, 0, W, pts, B, 1, baby, 1, outs, W));
    } else {
        u64* inner;
        RET(scratch(c, &inner, (size_t)B * G * W));
        // baby steps with ScMult fused, then giant steps; each over the whole batch
        RET(rotate_sum_regular(c, cts, 0, W, pts, B, G, baby, 1, inner, (long long)G * W));
        RET(rotate_sum_regular(c, inner, W, (long long)G * W, nullptr, B, 1, G, baby, outs, W));
        release(c, inner);
    }
    if (DM) RET(mask_finish(c, outs, DM, B, masked));
    return GALA_OK;
}

int gala_mv_gala(gala_ctx* c, const uint64_t* ct, const uint64_t* pts, int T, int baby, const uint32_t* r,
                 uint64_t* out, uint64_t* masked)
{
    return gala_mv_gala_batch(c, ct, 1, pts, T, baby, r, out, masked);
}

// ---------------------------------------------------------------------------
// GALA schedule 2: one decomposition of x.c1 per input, digits hoisted across the
// plaintext product (oracle o_mv_gala2).  Plaintexts in every prime of QP, pre-permuted.
int gala_encode_gala_weights(gala_ctx* c, const uint32_t* slots, int T, int baby, uint64_t* pts2)
{
    const int N = c->dc.N, M = c->dc.M;
    if (T <= 0 || baby <= 0 || T % baby) return set_err(GALA_ERR_PARAM, "baby %d must divide T=%d", baby, T);
    u64* tmp;
    RET(scratch(c, &tmp, (size_t)T * M * N));
    KLAUNCH(c, "k_encode", k_encode<2><<<T * M, ntt_threads(N), 2 * c->smem_ntt, c->stream>>>(c->dc, slots, tmp));
    std::vector<unsigned> gal(baby, 1u);
    for (int jj = 1; jj < baby; jj++) gal[jj] = galois_of(c, jj);
    void* d_gal;
    RET(upload(c, gal.data(), gal.size() * sizeof(unsigned), &d_gal));
    KLAUNCH(c, "k_gala_pt_perm", k_gala_pt_perm<<<grid_for((long long)T * M * N, 256), 256, 0, c->stream>>>(
                                     c->dc, tmp, T, baby, (const unsigned*)d_gal, pts2));
    release(c, tmp);
    release(c, d_gal);
    return GALA_OK;
}

// g_lo / g_hi: only the giant groups [g_lo, g_hi) (a multi-GPU shard; the baby-step sums of every group
// are computed, the giant-step key switches and inner ModDowns of the shard's groups only).  raw_U /
// raw_Q: return, per input, the QP sum before the final ModDown [B][2][M][N] and the Q addend
// [B][2][L][N] instead of outs / masked (gala_mv_gala2_finish completes the layer from the sums of
// every shard's raw outputs).
static int mv2_run(gala_ctx* c, const uint64_t* cts, int B, const uint64_t* pts2, const uint8_t* wcan, int T, int baby,
                   const uint32_t* r, uint64_t* outs, uint64_t* masked, int g_lo = 0, int g_hi = -1,
                   uint64_t* raw_U = nullptr, uint64_t* raw_Q = nullptr)
{
    const int N = c->dc.N, L = c->dc.L, M = c->dc.M;
    if (T <= 0 || B <= 0) return set_err(GALA_ERR_DIM, "T and B must be positive");
    if (baby <= 0) baby = gala_bsgs_baby(T);
    if (T % baby) return set_err(GALA_ERR_PARAM, "baby step %d does not divide T=%d", baby, T);
    const int G = T / baby;
    if ((long long)T > N / 2) return set_err(GALA_ERR_DIM, "T=%d exceeds the %d slots of a row", T, N / 2);
    if (g_hi < 0) g_hi = G;
    if (g_lo < 0 || g_lo >= g_hi || g_hi > G) return set_err(GALA_ERR_PARAM, "bad giant-group range [%d, %d) of %d", g_lo, g_hi, G);
    if ((g_lo != 0 || g_hi != G) && !raw_U) return set_err(GALA_ERR_PARAM, "a giant-group shard returns raw sums");
    const long long W = 2LL * L * N, MN = (long long)M * N;
    const long long blk_words = (long long)(L * M + L) * N;
    for (int j = 1; j < baby; j++)
        if (!gala_has_rotation_key(c, j)) return set_err(GALA_ERR_NOKEY, "missing rotation key for step %d", j);
    for (int g = 1; g < G; g++)
        if (!gala_has_rotation_key(c, g * baby))
            return set_err(GALA_ERR_NOKEY, "missing rotation key for step %d", norm_step(c, g * baby));
    if (baby == 1 && raw_U) return set_err(GALA_ERR_PARAM, "sharded trees need a baby step > 1");
    if (baby == 1) {   // T == 1 (a single group with one member) or degenerate trees: plain products + giant sum
        u64* prods;
        RET(scratch(c, &prods, (size_t)B * T * W));
        for (int b = 0; b < B; b++)
            for (int t = 0; t < T; t++) {
                dim3 grid((unsigned)((2 * L * N + 255) / 256), 1);
                KLAUNCH(c, "k_ct_mul_pts", k_ct_mul_pts<<<grid, 256, 0, c->stream>>>(
                                               c->dc, cts + b * W, pts2 + t * MN, prods + ((long long)b * T + t) * W));
            }
        RET(rotate_sum_regular(c, prods, W, (long long)T * W, nullptr, B, 1, T, 1, outs, W));
        release(c, prods);
        if (r && masked) RET(sub_plain_batch(c, outs, r, B, masked));
        return GALA_OK;
    }
    u64* DM = nullptr;
    if (c->coef_out && r && !raw_U) RET(mask_begin_coef(c, r, B, &c->coef_m));
    else if (r && masked && !raw_U) RET(mask_begin(c, r, B, &DM));   // overlaps the layer on the side stream
    // 1. one decomposition per input: identity digit block [(L*M + L)][N] (digits of x.c1 in every
    //    prime of QP, then x.c0)
    u64 *dig, *Dblk;
    RET(scratch(c, &dig, (size_t)B * L * N));
    RET(scratch(c, &Dblk, (size_t)B * blk_words));
    std::vector<TermDesc> td(B);
    for (int b = 0; b < B; b++) {
        td[b].X = cts + b * W;
        td[b].pt = nullptr;
        td[b].dig = dig + (long long)b * L * N;
        td[b].blk = Dblk + (long long)b * blk_words;
        td[b].rot_off = 0;
        td[b].rot_cnt = 1;
    }
    std::vector<unsigned> gal(baby, 1u);          // gal[0] = identity (the decomposition block)
    std::vector<const u64*> keys(baby, nullptr);
    for (int jj = 1; jj < baby; jj++) {
        gal[jj] = galois_of(c, jj);
        keys[jj] = key_for(c, jj);
    }
    size_t o_gal = (td.size() * sizeof(TermDesc) + 15) & ~(size_t)15;
    size_t o_keys = (o_gal + gal.size() * sizeof(unsigned) + 15) & ~(size_t)15;
    std::vector<char> blob(o_keys + keys.size() * sizeof(u64*));
    memcpy(blob.data(), td.data(), td.size() * sizeof(TermDesc));
    memcpy(blob.data() + o_gal, gal.data(), gal.size() * sizeof(unsigned));
    memcpy(blob.data() + o_keys, keys.data(), keys.size() * sizeof(u64*));
    char* d_blob;
    RET(upload(c, blob.data(), blob.size(), (void**)&d_blob));
    const int nt = ntt_threads(N);
    const unsigned* d_gal = (const unsigned*)(d_blob + o_gal);
    KLAUNCH(c, "k_digits_intt", k_digits_intt<<<(unsigned)(B * L), nt, c->smem_ntt, c->stream>>>(
                                    c->dc, (const TermDesc*)d_blob, d_gal, blk_words));
    KLAUNCH(c, "k_digits_perm", k_digits_perm<<<(unsigned)(B * L * L), nt, c->smem_ntt, c->stream>>>(
                                    c->dc, (const TermDesc*)d_blob, d_gal, blk_words));
    // 2. stage A: E_jj = sum_i sigma_jj(D_i) ksk_jj[i] per input and baby rotation (shared by all groups);
    //    stage B: per (input, group) U = sum_jj w_t E_jj, C0 = sum_jj w_t sigma_jj(c0) (+ step-0 member)
    const int Z = B * G;
    // key-folded tiles (k_gala_kf) for layers large enough for a tile's fixed per-position cost (64 rotations x
    // 8 groups of MMA columns whatever T is): T >= 128 (config 2); config 1 (T = 8) stays on the CUDA cores,
    // 1.6 vs 2.2 us per layer at 1024 inputs
    const bool kf = wcan != nullptr && fc_kf_on(c) && B >= 16 && T >= c->fc_tc_min_T && G <= 8 && baby <= 64 &&
                    getenv("GALA_FC_NO_TC") == nullptr;
    u64 *E = nullptr, *R0 = nullptr, *U, *Cacc, *rr;
    // (key-folded: the u_quad_base layout, whole 256-input tiles)
    RET(scratch(c, &U, (size_t)(kf ? (B + KF_ROWS - 1) / KF_ROWS * KF_ROWS * G : Z) * 2 * M * N));
    RET(scratch(c, &Cacc, (size_t)Z * 2 * L * N));
    RET(scratch(c, &rr, (size_t)Z * 2 * N));
    // the tensor-core tile always spans 32 input rows: it pays off from about half a tile of inputs
    // (config 2 at B = 8: 0.139 ms/layer vs 0.097 on the CUDA cores; B = 32: 0.044 vs 0.088)
    // larger batches run the tensor-core pair per tile of 32 inputs (every tile >= 16) when the layer is
    // large enough for a tile's fixed per-position cost (K = 64 rotations x 8 bytes whatever T is) to pay:
    // T >= 128 (config 2: 17.5k -> 19.3k layers/s at 96 inputs; config 1, T = 8, stays on the CUDA cores,
    // 0.0016 vs 0.0066 ms per layer at 1024 inputs); the rest of the layer stays batched over all B
    const bool tc = !kf && wcan != nullptr && !fc_kf_on(c) && B >= 16 &&
                    (B <= 32 || (T >= 128 && (B % 32 == 0 || B % 32 >= 16))) &&
                    G <= 8 && baby <= 64 && (N % 32) == 0 && getenv("GALA_FC_NO_TC") == nullptr;
    // fused E + MMA kernel (k_gala_tcf): experiment, slower than the k_gala_e_can / k_gala_tc pair so far
    // (the E warps are load-latency bound at 7-11 warps per SM; profiles/r2_experiments.md)
    const bool fused = tc && getenv("GALA_FC_FUSED") != nullptr;
    if (kf) {
        // key-folded tensor-core baby steps: per tile of <= 256 inputs the A blocks in rotation-orbit order
        // (k_gala_dq), then one persistent kernel on CTA pairs; U carries the Q-side addends lifted into QP
        // (P C), so Cacc is not formed
        release(c, Cacc);
        Cacc = nullptr;
        const int* orb;
        RET(kf_orbit_table(c, &orb));
        uint8_t* Dq;
        RET(scratch(c, &Dq, (size_t)M * 4 * KF_ORB(N) * 4096));
        // CTA pairs (cta_group::2): an even grid of at most one CTA per SM
        const long long nblk = MN / 4;
        int grid = (int)(2 * nblk < c->num_sms ? 2 * nblk : c->num_sms) & ~1;
        if (grid < 2) grid = 2;
        for (int b0 = 0; b0 < B; b0 += KF_ROWS) {
            const int bt = B - b0 < KF_ROWS ? B - b0 : KF_ROWS;
            const u64* Dt = Dblk + (long long)b0 * blk_words;
            u64* Ut = U + (long long)b0 * G * 2 * M * N;
#define GALA_KF(LL)                                                                                               \
    do {                                                                                                          \
        KLAUNCH(c, "k_gala_dq", (k_gala_dq<LL><<<(unsigned)(MN / KF_DQ_POS), 256, KF_DQ_SMEM, c->stream>>>(c->dc, Dt, bt, orb, Dq))); \
        KLAUNCH(c, "k_gala_kf", (k_gala_kf<LL><<<grid, KF_THREADS, KF_SMEM, c->stream>>>(c->dc, Dq, (const u64*)wcan,   \
                                                                                     orb, baby, G, bt, Ut)));      \
    } while (0)
            switch (L) {
                case 1: GALA_KF(1); break;
                case 2: GALA_KF(2); break;
                default: GALA_KF(3); break;
            }
#undef GALA_KF
        }
        release(c, Dq);
        debug_dump(c, "U", U, (size_t)Z * 2 * M * N);
    } else if (fused) {
        // tensor-core baby-step sums with the E_jj key products computed in the kernel (k_gala_tcf):
        // per tile of 32 inputs, the digit blocks input-minor (k_gala_dt), then one persistent kernel
        u64 *Dt, *Kt;
        RET(scratch(c, &Dt, (size_t)blk_words * 32));
        RET(scratch(c, &Kt, (size_t)MN * 64 * 2 * L));
        const u64* const* dk = (const u64* const*)(d_blob + o_keys);
        switch (L) {
            case 1: KLAUNCH(c, "k_gala_kt", (k_gala_kt<1><<<grid_for(MN * 64, 256), 256, 0, c->stream>>>(c->dc, dk, baby, Kt))); break;
            case 2: KLAUNCH(c, "k_gala_kt", (k_gala_kt<2><<<grid_for(MN * 64, 256), 256, 0, c->stream>>>(c->dc, dk, baby, Kt))); break;
            case 3: KLAUNCH(c, "k_gala_kt", (k_gala_kt<3><<<grid_for(MN * 64, 256), 256, 0, c->stream>>>(c->dc, dk, baby, Kt))); break;
            default: KLAUNCH(c, "k_gala_kt", (k_gala_kt<4><<<grid_for(MN * 64, 256), 256, 0, c->stream>>>(c->dc, dk, baby, Kt))); break;
        }
        for (int b0 = 0; b0 < B; b0 += 32) {
            const int bt = B - b0 < 32 ? B - b0 : 32;
            KLAUNCH(c, "k_gala_dt", k_gala_dt<<<c->num_sms * 8, 256, 0, c->stream>>>(c->dc, Dblk + (long long)b0 * blk_words, bt, Dt));
            const u64* Xt = cts + (long long)b0 * 2 * L * N;
            u64* Ut = U + (long long)b0 * G * 2 * M * N;
            u64* Ct = Cacc + (long long)b0 * G * 2 * L * N;
#define GALA_TCF(LL)                                                                                       \
    KLAUNCH(c, "k_gala_tc", (k_gala_tcf<LL><<<c->num_sms, GTCF_THREADS, GTC_SMEM, c->stream>>>(               \
                                c->dc, Dt, Kt, d_gal, (const u64*)wcan, Xt, baby, G, bt, Ut, Ct)))
            switch (L) {
                case 1: GALA_TCF(1); break;
                case 2: GALA_TCF(2); break;
                case 3: GALA_TCF(3); break;
                default: GALA_TCF(4); break;
            }
#undef GALA_TCF
        }
        release(c, Dt);
        release(c, Kt);
    } else if (tc) {
        // tensor-core baby-step sums: E packed as int8 MMA operands, weights as their byte-convolution
        uint8_t* Ecan;
        RET(scratch(c, &Ecan, (size_t)MN * GTC_A_BYTES));
        const u64* const* dk = (const u64* const*)(d_blob + o_keys);
        dim3 ge((unsigned)(N / 32), 32, (unsigned)M);
        for (int b0 = 0; b0 < B; b0 += 32) {
            const int bt = B - b0 < 32 ? B - b0 : 32;
            const u64* Dt = Dblk + (long long)b0 * blk_words;
            const u64* Xt = cts + (long long)b0 * 2 * L * N;
            u64* Ut = U + (long long)b0 * G * 2 * M * N;
            u64* Ct = Cacc + (long long)b0 * G * 2 * L * N;
#define GALA_ECAN(LL) KLAUNCH(c, "k_gala_e", (k_gala_e_can<LL><<<ge, 256, 0, c->stream>>>(c->dc, Dt, dk, d_gal, baby, bt, Ecan)))
#define GALA_TC(LL)                                                                                        \
    KLAUNCH(c, "k_gala_tc", (k_gala_tc<LL><<<c->num_sms, GTC_THREADS, GTC_SMEM, c->stream>>>(                   \
                                c->dc, Ecan, (const u64*)wcan, Xt, pts2, baby, G, bt, Ut, Ct)))
            switch (L) {
                case 1: GALA_ECAN(1); GALA_TC(1); break;
                case 2: GALA_ECAN(2); GALA_TC(2); break;
                case 3: GALA_ECAN(3); GALA_TC(3); break;
                default: GALA_ECAN(4); GALA_TC(4); break;
            }
#undef GALA_ECAN
#undef GALA_TC
        }
        release(c, Ecan);
        debug_dump(c, "U", U, (size_t)Z * 2 * M * N);
        debug_dump(c, "C", Cacc, (size_t)Z * 2 * L * N);
    } else {
    RET(scratch(c, &E, (size_t)B * (baby - 1) * 2 * MN));
    RET(scratch(c, &R0, (size_t)B * (baby - 1) * L * N));
    {
        const int th = N < 256 ? N : 256;
        const u64* const* dk = (const u64* const*)(d_blob + o_keys);
        const int cb = B % 4 == 0 ? 4 : (B % 2 == 0 ? 2 : 1);   // inputs per thread (key reuse)
        dim3 ga((B / cb) * (baby - 1), M, (N + th - 1) / th);
#define GALA_E(LL)                                                                                              \
    do {                                                                                                        \
        if (cb == 4) KLAUNCH(c, "k_gala_e", (k_gala_e<LL, 4><<<ga, th, 0, c->stream>>>(c->dc, Dblk, dk, d_gal, baby, E, R0))); \
        else if (cb == 2) KLAUNCH(c, "k_gala_e", (k_gala_e<LL, 2><<<ga, th, 0, c->stream>>>(c->dc, Dblk, dk, d_gal, baby, E, R0))); \
        else KLAUNCH(c, "k_gala_e", (k_gala_e<LL, 1><<<ga, th, 0, c->stream>>>(c->dc, Dblk, dk, d_gal, baby, E, R0)));     \
    } while (0)
        switch (L) {
            case 1: GALA_E(1); break;
            case 2: GALA_E(2); break;
            case 3: GALA_E(3); break;
            default: GALA_E(4); break;
        }
#undef GALA_E
        // one (input, group) per thread (measured best: sharing plaintext loads across inputs, or an
        // smem-tiled modular GEMM, costs occupancy / Montgomery products and runs slower)
        // one member's loads in flight at a time (larger load chunks or sharing plaintext loads across
        // inputs raise register pressure and lose to occupancy), 128-bit lazy accumulation with one
        // REDC per c.lazy[j] members, coefficient-slice-major grid (measured best on B200)
        dim3 gb(G * B, M, (N + th - 1) / th);
        KLAUNCH(c, "k_gala_mac2", (k_gala_mac2<1, true><<<gb, th, 0, c->stream>>>(c->dc, cts, E, R0, pts2, baby, G, U, Cacc)));
    }
    release(c, E);
    release(c, R0);
    }
    release(c, dig);
    release(c, Dblk);
    // 3. giant steps with the c0 ModDown deferred.  Group g's sum (U_z in QP, C_z in Q; z = b G + g) is
    //    rotated by g b.  Only its c1 needs a ModDown (to be decomposed for the key switch); its c0 is
    //    rotated in QP and summed: S.c0 = sum_g sigma_g(U_z.c0), S.c1 = U_{b,0}.c1, and one final
    //    ModDown of S + the key-switch sums gives the layer (oracle: o_mv_gala2).
    std::vector<unsigned> ggal(G, 1u);
    for (int g = 1; g < G; g++) ggal[g] = galois_of(c, g * baby);
    unsigned* d_ggal;
    RET(upload(c, ggal.data(), ggal.size() * sizeof(unsigned), (void**)&d_ggal));
    u64 *S, *Qadd = nullptr;
    RET(scratch(c, &S, (size_t)B * 2 * M * N));
    if (Cacc) RET(scratch(c, &Qadd, (size_t)B * 2 * L * N));   // key-folded form: no Q-side addend
    {
        const int th = N < 256 ? N : 256;
        dim3 gq((unsigned)((N + th - 1) / th), (unsigned)M, (unsigned)B);
        KLAUNCH(c, "k_giant_qp", k_giant_qp<<<gq, th, 0, c->stream>>>(c->dc, U, Cacc, d_ggal, G, g_lo, g_hi, S, Qadd,
                                                                       kf ? 1 : 0));
    }
    const int ga = g_lo > 1 ? g_lo : 1;                 // the shard's giant groups g >= 1
    const int Gs = g_hi > ga ? g_hi - ga : 0;
    const int Zi = B * Gs;
    u64* inner = nullptr;
    if (Zi > 0) {
        // inner ModDown of c1 for the groups g >= 1 (item x -> z = (x / (G-1)) G + 1 + x % (G-1))
        RET(scratch(c, &inner, (size_t)Zi * W));
        PolyMap pmi = pm_make(1, 1, L, 0, 2LL * M * N, N, G);
        pmi.skip_first = ga;
        pmi.skip_cnt = Gs;
        if (kf) {   // the P limb of c1 straight from the key-folded group-sum layout
            pmi.quad_G = G;
            pmi.quad_cc = 1;
            pmi.quad_j = L;
        }
        RET(launch_inv<false>(c, kf ? U : U + (long long)(M + L) * N, rr, Zi, pmi, "k_ntt_inv[moddown]"));
        MdArgs a{};
        a.quad_G = kf ? G : 0;
        a.r = rr;
        a.U = U;
        a.add0 = Cacc;
        a.add1 = Cacc ? Cacc + (long long)L * N : nullptr;
        a.add_is = 2LL * L * N;
        a.out = inner;
        a.out_is = W;
        a.outs = nullptr;
        a.comps = 1;
        a.comp0 = 1;
        a.skip_per = G;
        a.skip_first = ga;
        a.skip_cnt = Gs;
        KLAUNCH(c, "k_moddown", k_moddown<<<Zi * L, nt, c->smem_ntt, c->stream>>>(c->dc, a));
    }
    release(c, U);
    release(c, Cacc);
    release(c, rr);
    release(c, d_blob);
    // 4. per input: the G-1 giant-step key switches of (0, c1') plus S before one lazy ModDown, plus Qadd
    {
        std::vector<EngTerm> terms;
        std::vector<std::vector<EngMember>> groups((size_t)B);
        std::vector<u64*> eouts;
        terms.reserve((size_t)Zi);
        for (int b = 0; b < B; b++) {
            for (int g = ga; g < g_hi; g++) {
                EngTerm t;
                t.X = inner + ((long long)b * Gs + (g - ga)) * W;
                t.pt = nullptr;
                t.ntt_block = nullptr;
                t.c0_zero = true;
                t.steps.push_back(norm_step(c, g * baby));
                terms.push_back(t);
                groups[(size_t)b].push_back({(int)terms.size() - 1, 0});
            }
            eouts.push_back(outs + (long long)b * W);
        }
        RET(rotate_engine(c, terms, groups, eouts, S, Qadd, raw_U, raw_Q));
    }
    release(c, inner);
    release(c, S);
    release(c, Qadd);
    release(c, d_ggal);
    if (c->coef_m) {
        release(c, c->coef_m);
        c->coef_m = nullptr;
    }
    if (DM) RET(mask_finish(c, outs, DM, B, masked));
    return GALA_OK;
}

int gala_mv_gala2_batch(gala_ctx* c, const uint64_t* cts, int B, const uint64_t* pts2, int T, int baby,
                        const uint32_t* r, uint64_t* outs, uint64_t* masked)
{
    return mv2_run(c, cts, B, pts2, nullptr, T, baby, r, outs, masked);
}

int gala_mv_gala2_batch_tc(gala_ctx* c, const uint64_t* cts, int B, const uint64_t* pts2, const uint8_t* wcan, int T,
                           int baby, const uint32_t* r, uint64_t* outs, uint64_t* masked)
{
    return mv2_run(c, cts, B, pts2, wcan, T, baby, r, outs, masked);
}

int gala_mv_gala2_partial(gala_ctx* c, const uint64_t* cts, int B, const uint64_t* pts2, const uint8_t* wcan, int T,
                          int baby, int g_lo, int g_hi, uint64_t* qp_sum, uint64_t* q_add)
{
    if (!qp_sum || !q_add) return set_err(GALA_ERR_PARAM, "partial sums need output buffers");
    return mv2_run(c, cts, B, pts2, wcan, T, baby, nullptr, nullptr, nullptr, g_lo, g_hi, qp_sum, q_add);
}

int gala_mv_gala2_finish(gala_ctx* c, uint64_t* qp_sum, uint64_t* q_add, int B, const uint32_t* r, uint64_t* outs,
                         uint64_t* masked)
{
    const int N = c->dc.N, L = c->dc.L, M = c->dc.M;
    if (B <= 0) return set_err(GALA_ERR_DIM, "empty batch");
    // the words are sums over the shards of values below q_j: exact reduction first
    KLAUNCH(c, "k_reduce_mod", k_reduce_mod<<<grid_for((long long)B * 2 * M * N, 256), 256, 0, c->stream>>>(c->dc, qp_sum, 2LL * B, M));
    KLAUNCH(c, "k_reduce_mod", k_reduce_mod<<<grid_for((long long)B * 2 * L * N, 256), 256, 0, c->stream>>>(c->dc, q_add, 2LL * B, L));
    u64* rr;
    RET(scratch(c, &rr, (size_t)B * 2 * N));
    RET(launch_inv<false>(c, qp_sum + (long long)L * N, rr, B * 2, pm_make(1, 1, L, 0, (long long)M * N, N),
                          "k_ntt_inv[moddown]"));
    MdArgs a{};
    a.r = rr;
    a.U = qp_sum;
    a.add0 = q_add;
    a.add1 = q_add + (long long)L * N;
    a.add_is = 2LL * L * N;
    a.out = outs;
    a.out_is = 2LL * L * N;
    a.outs = nullptr;
    KLAUNCH(c, "k_moddown", k_moddown<<<B * 2 * L, ntt_threads(N), c->smem_ntt, c->stream>>>(c->dc, a));
    release(c, rr);
    if (r && masked) RET(sub_plain_batch(c, outs, r, B, masked));
    return GALA_OK;
}

size_t gala_fc_tc_weight_bytes(gala_ctx* c)
{
    return (size_t)c->dc.M * c->dc.N * (fc_kf_on(c) ? (size_t)KF_W_BYTES : (size_t)GTC_W_BYTES);
}

int gala_fc_tc_weights(gala_ctx* c, const uint64_t* pts2, int T, int baby, uint8_t* wcan)
{
    if (baby <= 0 || T % baby) return set_err(GALA_ERR_PARAM, "baby %d must divide T=%d", baby, T);
    const int G = T / baby;
    if (G > 8 || baby > 64) return set_err(GALA_ERR_PARAM, "tensor-core FC path needs T/baby <= 8 and baby <= 64");
    if (fc_kf_on(c)) {
        // key-folded weights: the baby-step rotation keys and P multiplied into the plaintexts (k_gala_kfw)
        std::vector<const u64*> keys(64, nullptr);
        for (int jj = 1; jj < baby; jj++) {
            keys[jj] = key_for(c, jj);
            if (!keys[jj]) return set_err(GALA_ERR_NOKEY, "missing rotation key for step %d (generate the baby-step keys "
                                                          "before the tensor-core weights)", jj);
        }
        const u64** dk;
        RET(upload(c, keys.data(), keys.size() * sizeof(u64*), (void**)&dk));
        const long long total = (long long)c->dc.M * c->dc.N * KF_W_WORDS;
        const int gr = grid_for(total, 256);
        switch (c->dc.L) {
            case 1: KLAUNCH(c, "k_gala_kfw", (k_gala_kfw<1><<<gr, 256, 0, c->stream>>>(c->dc, pts2, dk, c->d_pmod, baby, G, (u64*)wcan))); break;
            case 2: KLAUNCH(c, "k_gala_kfw", (k_gala_kfw<2><<<gr, 256, 0, c->stream>>>(c->dc, pts2, dk, c->d_pmod, baby, G, (u64*)wcan))); break;
            default: KLAUNCH(c, "k_gala_kfw", (k_gala_kfw<3><<<gr, 256, 0, c->stream>>>(c->dc, pts2, dk, c->d_pmod, baby, G, (u64*)wcan))); break;
        }
        release(c, (void*)dk);
        return GALA_OK;
    }
    const long long total = (long long)c->dc.M * c->dc.N * GTC_W_WORDS;
    KLAUNCH(c, "k_gala_wt", k_gala_wt<<<grid_for(total, 256), 256, 0, c->stream>>>(c->dc, pts2, baby, G, (u64*)wcan));
    return GALA_OK;
}

static int mv_batch_host(gala_ctx* c, int schedule, const uint64_t* cts_host, int B, const uint64_t* pts, int T,
                         int baby, const uint32_t* r_host, uint64_t* masked_host, const uint8_t* wcan = nullptr)
{
    const int N = c->dc.N, L = c->dc.L;
    const long long W = 2LL * L * N;
    u64 *coef, *ct, *out, *masked;
    uint32_t* r;
    RET(scratch(c, &coef, (size_t)B * W));
    RET(scratch(c, &ct, (size_t)B * W));
    RET(scratch(c, &out, (size_t)B * W));
    RET(scratch(c, &masked, (size_t)B * W));
    RET(scratch(c, &r, (size_t)B * N));
    CK(cudaMemcpyAsync(coef, cts_host, sizeof(u64) * B * W, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(r, r_host, sizeof(uint32_t) * B * N, cudaMemcpyHostToDevice, c->stream));
    RET(gala_ct_import(c, coef, ct, B));
    if (schedule == 2) RET(mv2_run(c, ct, B, pts, wcan, T, baby, r, out, masked));
    else RET(gala_mv_gala_batch(c, ct, B, pts, T, baby, r, out, masked));
    RET(gala_ct_export(c, masked, coef, B));
    CK(cudaMemcpyAsync(masked_host, coef, sizeof(u64) * B * W, cudaMemcpyDeviceToHost, c->stream));
    release(c, coef);
    release(c, ct);
    release(c, out);
    release(c, masked);
    release(c, r);
    CK(cudaStreamSynchronize(c->stream));
    return GALA_OK;
}

int gala_mv_gala_batch_host(gala_ctx* c, const uint64_t* cts_host, int B, const uint64_t* pts, int T, int baby,
                            const uint32_t* r_host, uint64_t* masked_host)
{
    return mv_batch_host(c, 1, cts_host, B, pts, T, baby, r_host, masked_host);
}

int gala_mv_gala2_batch_host(gala_ctx* c, const uint64_t* cts_host, int B, const uint64_t* pts2, int T, int baby,
                             const uint32_t* r_host, uint64_t* masked_host)
{
    return mv_batch_host(c, 2, cts_host, B, pts2, T, baby, r_host, masked_host);
}

int gala_mv_gala2_batch_tc_host(gala_ctx* c, const uint64_t* cts_host, int B, const uint64_t* pts2, const uint8_t* wcan,
                                int T, int baby, const uint32_t* r_host, uint64_t* masked_host)
{
    return mv_batch_host(c, 2, cts_host, B, pts2, T, baby, r_host, masked_host, wcan);
}

// S consecutive batches of B inputs from host memory, the transfers overlapped with the layers: the
// inputs of batch s + 1 are copied in (cs_in) while batch s computes, and batch s - 1's masked words are
// copied out (cs_out) -- PCIe is full duplex.  Two staging slots per direction; every batch's H2D and
// D2H happen inside the call, which returns when the last batch's words are in masked_host.
// cts_host [S][B][2][L][N] canonical words, r_host [S][B][N], masked_host [S][B][2][L][N].
static int mv_stream_host(gala_ctx* c, int schedule, const uint64_t* cts_host, int S, int B, const uint64_t* pts,
                          const uint8_t* wcan, int T, int baby, const uint32_t* r_host, uint64_t* masked_host)
{
    if (S <= 0 || B <= 0) return set_err(GALA_ERR_DIM, "empty stream (S=%d, B=%d)", S, B);
    const int N = c->dc.N, L = c->dc.L;
    const long long W = 2LL * L * N;
    if (!c->cs_in) {
        CK(cudaStreamCreateWithFlags(&c->cs_in, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&c->cs_out, cudaStreamNonBlocking));
        for (int i = 0; i < 2; i++)
            for (cudaEvent_t* e : {&c->ev_h2d[i], &c->ev_used[i], &c->ev_done[i], &c->ev_d2h[i]})
                CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_alloc, cudaEventDisableTiming));
    }
    u64 *hin[2], *hout[2], *ct, *out, *masked;
    uint32_t* rr[2];
    for (int i = 0; i < 2; i++) {
        RET(scratch(c, &hin[i], (size_t)B * W));
        RET(scratch(c, &hout[i], (size_t)B * W));
        RET(scratch(c, &rr[i], (size_t)B * N));
    }
    RET(scratch(c, &ct, (size_t)B * W));
    RET(scratch(c, &out, (size_t)B * W));
    RET(scratch(c, &masked, (size_t)B * W));
    CK(cudaEventRecord(c->ev_alloc, c->stream));
    CK(cudaStreamWaitEvent(c->cs_in, c->ev_alloc, 0));
    CK(cudaStreamWaitEvent(c->cs_out, c->ev_alloc, 0));
    // the coefficient-domain finish applies where mv2_run takes the key-folded form (its predicate, restated)
    bool coef = false;
    if (schedule == 2 && r_host && masked_host) {
        const int bb = baby > 0 ? baby : gala_bsgs_baby(T);
        const char* ce = getenv("GALA_STREAM_COEF");
        coef = wcan != nullptr && fc_kf_on(c) && B >= 16 && T >= c->fc_tc_min_T && bb > 1 && T % bb == 0 && T / bb <= 8 &&
               bb <= 64 && getenv("GALA_FC_NO_TC") == nullptr && !(ce && ce[0] == '0');
    }
    const char* nc = getenv("GALA_STREAM_NOCOPY");   // experiment: "in", "out" or both skipped
    const bool noin = nc && strcmp(nc, "out") != 0, noout = nc && strcmp(nc, "in") != 0;
    // large copies go in 1 MB pieces: the layers' own small descriptor uploads share the copy engine and
    // would otherwise queue behind a whole 13 MB batch (measured: +0.18 ms per step)
    auto chunked = [&](void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t st) -> int {
        const size_t piece = (size_t)1 << 20;
        for (size_t o = 0; o < bytes; o += piece)
            CK(cudaMemcpyAsync((char*)dst + o, (const char*)src + o, bytes - o < piece ? bytes - o : piece, kind, st));
        return GALA_OK;
    };
    auto copy_in = [&](int b) -> int {
        const int sl = b & 1;
        if (noin) {
            CK(cudaEventRecord(c->ev_h2d[sl], c->cs_in));
            return GALA_OK;
        }
        if (b >= 2) CK(cudaStreamWaitEvent(c->cs_in, c->ev_used[sl], 0));   // batch b - 2 consumed the slot
        RET(chunked(hin[sl], cts_host + (long long)b * B * W, sizeof(u64) * B * W, cudaMemcpyHostToDevice, c->cs_in));
        CK(cudaMemcpyAsync(rr[sl], r_host + (long long)b * B * N, sizeof(uint32_t) * B * N, cudaMemcpyHostToDevice,
                           c->cs_in));
        CK(cudaEventRecord(c->ev_h2d[sl], c->cs_in));
        return GALA_OK;
    };
    RET(copy_in(0));
    for (int b = 0; b < S; b++) {
        const int sl = b & 1;
        if (b + 1 < S) RET(copy_in(b + 1));   // enqueued ahead: overlaps this batch's layers
        CK(cudaStreamWaitEvent(c->stream, c->ev_h2d[sl], 0));
        RET(gala_ct_import(c, hin[sl], ct, B));
        if (coef) {
            // key-folded layers finish in the coefficient domain: the final ModDown writes the masked canonical
            // words straight into the staging slot (k_moddown_coef), no mask NTT and no export INTT
            if (b >= 2) CK(cudaStreamWaitEvent(c->stream, c->ev_d2h[sl], 0));   // batch b - 2's words copied out
            c->coef_out = hout[sl];
            const int rc = mv2_run(c, ct, B, pts, wcan, T, baby, rr[sl], out, masked);
            c->coef_out = nullptr;
            if (c->coef_m) {
                release(c, c->coef_m);
                c->coef_m = nullptr;
            }
            RET(rc);
            CK(cudaEventRecord(c->ev_used[sl], c->stream));
        } else {
        if (schedule == 2) RET(mv2_run(c, ct, B, pts, wcan, T, baby, rr[sl], out, masked));
        else RET(gala_mv_gala_batch(c, ct, B, pts, T, baby, rr[sl], out, masked));
        CK(cudaEventRecord(c->ev_used[sl], c->stream));
        if (b >= 2) CK(cudaStreamWaitEvent(c->stream, c->ev_d2h[sl], 0));   // batch b - 2's words copied out
        RET(gala_ct_export(c, masked, hout[sl], B));
        }
        CK(cudaEventRecord(c->ev_done[sl], c->stream));
        CK(cudaStreamWaitEvent(c->cs_out, c->ev_done[sl], 0));
        if (!noout)
            RET(chunked(masked_host + (long long)b * B * W, hout[sl], sizeof(u64) * B * W, cudaMemcpyDeviceToHost,
                        c->cs_out));
        CK(cudaEventRecord(c->ev_d2h[sl], c->cs_out));
    }
    CK(cudaStreamSynchronize(c->cs_out));
    CK(cudaStreamSynchronize(c->cs_in));
    for (int i = 0; i < 2; i++) {
        release(c, hin[i]);
        release(c, hout[i]);
        release(c, rr[i]);
    }
    release(c, ct);
    release(c, out);
    release(c, masked);
    CK(cudaStreamSynchronize(c->stream));
    return GALA_OK;
}

int gala_mv_gala2_stream_host(gala_ctx* c, const uint64_t* cts_host, int S, int B, const uint64_t* pts2,
                              const uint8_t* wcan, int T, int baby, const uint32_t* r_host, uint64_t* masked_host)
{
    return mv_stream_host(c, 2, cts_host, S, B, pts2, wcan, T, baby, r_host, masked_host);
}

int gala_mv_gala_host(gala_ctx* c, const uint64_t* ct_host, const uint64_t* pts, int T, int baby,
                      const uint32_t* r_host, uint64_t* masked_host)
{
    return gala_mv_gala_batch_host(c, ct_host, 1, pts, T, baby, r_host, masked_host);
}

// schedule-1 plaintexts on the tensor cores: tile geometry
static void kg1_geom(int n_ib, int n_obp, int c_n, int k, int* Rp, int* Kwp, int* MT)
{
    const int Mr = n_obp * c_n, Kw = n_ib * k;
    *MT = (Mr + 127) / 128;
    *Rp = *MT * 128;
    *Kwp = (Kw + 15) / 16 * 16;
}

static size_t kg1_smem(int MT, int Kwp)
{
    return (size_t)KG1_NST * KG1_GK * MT * 128 * 16 + 2 * (size_t)(Kwp / 2) * 512 + 2 * (size_t)Kwp * 16;
}

size_t gala_kg1_tc_bytes(gala_ctx* c, int n_ib, int n_obp, int c_n, int k)
{
    int Rp, Kwp, MT;
    kg1_geom(n_ib, n_obp, c_n, k, &Rp, &Kwp, &MT);
    if ((MT != 1 && MT != 2 && MT != 4) || Kwp > 1024 || kg1_smem(MT, Kwp) > 220 * 1024 || c->dc.N % 32) return 0;
    return (size_t)c->dc.L * c->dc.N * Kwp * Rp * 8;
}

int gala_kg1_tc_weights(gala_ctx* c, const uint64_t* pts, int n_obp, int n_ib, int c_n, int k, uint64_t* ptcan)
{
    int Rp, Kwp, MT;
    kg1_geom(n_ib, n_obp, c_n, k, &Rp, &Kwp, &MT);
    if (gala_kg1_tc_bytes(c, n_ib, n_obp, c_n, k) == 0) return set_err(GALA_ERR_PARAM, "layer shape not supported on the tensor-core path");
    const long long total = (long long)c->dc.L * c->dc.N * (Kwp / 2) * Rp * 2;
    KLAUNCH(c, "k_kg1_pt_can", k_kg1_pt_can<<<grid_for(total, 256), 256, 0, c->stream>>>(c->dc, pts, n_obp, n_ib, c_n, k, Rp,
                                                                                     Kwp / 2, ptcan));
    return GALA_OK;
}

static int conv_kg_run(gala_ctx* c, const uint64_t* cts, int n_ib, const uint64_t* pts, const uint64_t* ptcan, int n_obp,
                       int c_n, int k, const int* tap_steps, int band_step, uint64_t* outs, int B = 1);

int gala_conv_kg(gala_ctx* c, const uint64_t* cts, int n_ib, const uint64_t* pts, int n_obp, int c_n, int k,
                 const int* tap_steps, int band_step, uint64_t* outs)
{
    return conv_kg_run(c, cts, n_ib, pts, nullptr, n_obp, c_n, k, tap_steps, band_step, outs);
}

int gala_conv_kg_tc(gala_ctx* c, const uint64_t* cts, int n_ib, const uint64_t* ptcan, int n_obp, int c_n, int k,
                    const int* tap_steps, int band_step, uint64_t* outs)
{
    return conv_kg_run(c, cts, n_ib, nullptr, ptcan, n_obp, c_n, k, tap_steps, band_step, outs);
}

int gala_conv_kg_batch(gala_ctx* c, const uint64_t* cts, int B, int n_ib, const uint64_t* pts, int n_obp, int c_n, int k,
                       const int* tap_steps, int band_step, uint64_t* outs)
{
    if (B <= 0) return set_err(GALA_ERR_DIM, "empty image batch");
    return conv_kg_run(c, cts, n_ib, pts, nullptr, n_obp, c_n, k, tap_steps, band_step, outs, B);
}

// B images sharing the weights: cts [B][n_ib][W] -> outs [B][n_obp][W]; every stage runs once for the batch
static int conv_kg_run(gala_ctx* c, const uint64_t* cts, int n_ib, const uint64_t* pts, const uint64_t* ptcan, int n_obp,
                       int c_n, int k, const int* tap_steps, int band_step, uint64_t* outs, int B)
{
    const int N = c->dc.N, L = c->dc.L;
    const long long W = 2LL * L * N;
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
    // input rotations R[ib][tap]: one DecPerm per input (digit NTTs once), HstPerm per nonzero tap
    u64* R;
    if (ptcan && B > 1) {   // the tensor-core first-Add takes one image per call
        for (int b = 0; b < B; b++)
            RET(conv_kg_run(c, cts + (long long)b * n_ib * W, n_ib, pts, ptcan, n_obp, c_n, k, tap_steps, band_step,
                            outs + (long long)b * n_obp * W, 1));
        return GALA_OK;
    }
    const int nin = B * n_ib;   // inputs of every image, image-major
    RET(scratch(c, &R, (size_t)nin * k * W));
    for (int t = 0; t < k; t++)   // unrotated taps: one strided copy over every input
        if (norm_step(c, tap_steps[t]) == 0)
            CK(cudaMemcpy2DAsync(R + (long long)t * W, sizeof(u64) * k * W, cts, sizeof(u64) * W, sizeof(u64) * W,
                                 (size_t)nin, cudaMemcpyDeviceToDevice, c->stream));
    if (!rot_taps.empty()) {
        std::vector<EngTerm> terms;
        std::vector<std::vector<EngMember>> groups;
        std::vector<u64*> outs;
        for (int ib = 0; ib < nin; ib++) {
            EngTerm t;
            t.X = cts + (long long)ib * W;
            t.pt = nullptr;
            t.ntt_block = nullptr;
            for (int tap : rot_taps) t.steps.push_back(norm_step(c, tap_steps[tap]));
            terms.push_back(t);
            for (size_t r = 0; r < rot_taps.size(); r++) {
                groups.push_back({{ib, (int)r}});
                outs.push_back(R + ((long long)ib * k + rot_taps[r]) * W);
            }
        }
        RET(rotate_engine(c, terms, groups, outs));
    }
    // first-Add: acc[o][d] over all input blocks and taps
    u64* acc;
    RET(scratch(c, &acc, (size_t)B * n_obp * c_n * W));
    if (ptcan) {   // on the tensor cores: position-major plaintext bytes x byte-convolution of R
        int Rp, Kwp, MT;
        kg1_geom(n_ib, n_obp, c_n, k, &Rp, &Kwp, &MT);
        if (gala_kg1_tc_bytes(c, n_ib, n_obp, c_n, k) == 0) return set_err(GALA_ERR_PARAM, "layer shape not supported on the tensor-core path");
        u64* Rt;
        RET(scratch(c, &Rt, (size_t)L * N * 2 * Kwp));
        KLAUNCH(c, "k_kg1_rt", k_kg1_rt<<<grid_for((long long)L * N * 2 * Kwp, 256), 256, 0, c->stream>>>(c->dc, R, n_ib * k, Kwp, Rt));
        release(c, R);
        const size_t smem = kg1_smem(MT, Kwp);
        const int grid1 = c->num_sms;
#define KG1(MTV) KLAUNCH(c, "k_kg1_tc", (k_kg1_tc<MTV><<<grid1, KG1_THREADS, smem, c->stream>>>(c->dc, (const uint8_t*)ptcan, Rt, n_obp * c_n, Kwp, acc)))
        if (MT == 1) KG1(1);
        else if (MT == 2) KG1(2);
        else KG1(4);
#undef KG1
        release(c, Rt);
        RET(rotate_sum_regular(c, acc, W, 0, nullptr, 1, n_obp, c_n, band_step, outs, 0));
        release(c, acc);
        return GALA_OK;
    }
    const int th = N < 256 ? N : 256;
    const int rows = n_obp * c_n;
    // register tile (images x rows per thread), measured at config 3 x 16 images: 2 x 2 0.030,
    // 1 x 4 0.032, 2 x 4 0.036 (170 registers), 2 x 1 0.036, 1 x 1 0.050 ms per image
    int img = B >= 2 ? 2 : 1;
    int odt = rows >= 2 ? 2 : 1;
    if (const char* e = getenv("GALA_KGACC")) {   // A/B experiments: "img,odt"
        int a = 0, b2 = 0;
        if (sscanf(e, "%d,%d", &a, &b2) == 2 && (a == 1 || a == 2) && (b2 == 1 || b2 == 2 || b2 == 4)) {
            img = a;
            odt = b2;
        }
    }
    // partial-product accumulators: one image (config 3: 84 -> 60 us; grid-limited), not the 2-image tile
    // (30 -> 33 us per image at 16 images: register-limited)
    bool pp = img == 1;
    if (const char* e = getenv("GALA_KGACC_PP")) pp = atoi(e) != 0;
    dim3 grid((N + th - 1) / th, L * ((B + img - 1) / img), (rows + odt - 1) / odt);
    // input-block chunks whose rotated inputs (k * W words each, every image) fit comfortably in L2 (~48 MB)
    const long long chunk_bytes = 48ll << 20;
    int per_chunk = (int)(chunk_bytes / ((long long)B * k * W * 8));
    if (per_chunk < 1) per_chunk = 1;
    const long long R_bs = (long long)n_ib * k * W, acc_bs = (long long)rows * W;
    for (int ib0 = 0; ib0 < n_ib; ib0 += per_chunk) {
        const int ib1 = ib0 + per_chunk < n_ib ? ib0 + per_chunk : n_ib;
#define KGACC(IM, OD)                                                                                              \
    do {                                                                                                           \
        if (pp)                                                                                                    \
            KLAUNCH(c, "k_kg_accumulate", (k_kg_accumulate<IM, OD, true><<<grid, th, 0, c->stream>>>(              \
                                              c->dc, R, R_bs, n_ib, ib0, ib1, k, pts, c_n, rows, B, ib0 > 0, acc, acc_bs))); \
        else                                                                                                       \
            KLAUNCH(c, "k_kg_accumulate", (k_kg_accumulate<IM, OD, false><<<grid, th, 0, c->stream>>>(             \
                                              c->dc, R, R_bs, n_ib, ib0, ib1, k, pts, c_n, rows, B, ib0 > 0, acc, acc_bs))); \
    } while (0)
        if (img == 2) {
            if (odt == 4) KGACC(2, 4);
            else if (odt == 2) KGACC(2, 2);
            else KGACC(2, 1);
        } else {
            if (odt == 4) KGACC(1, 4);
            else if (odt == 2) KGACC(1, 2);
            else KGACC(1, 1);
        }
#undef KGACC
    }
    release(c, R);
    // second-Perm: out[b][o] = sum_d rot_{d * band}(acc[b][o][d]), one lazy ModDown per (b, o)
    RET(rotate_sum_regular(c, acc, W, 0, nullptr, 1, B * n_obp, c_n, band_step, outs, 0));
    release(c, acc);
    return GALA_OK;
}

int gala_kg_encode_weights(gala_ctx* c, const int32_t* kern, int c_o, int c_i, int k_h, int k_w, int u_w, int u_h,
                           int pair, uint64_t* pts)
{
    const int N = c->dc.N, L = c->dc.L, n = N / 2;
    const int B = u_w * u_h;
    if (B <= 0 || n % B || (k_h % 2) == 0 || (k_w % 2) == 0 || (pair != 1 && pair != 2))
        return set_err(GALA_ERR_PARAM, "bad kernel-grouping geometry");
    KgGeom g;
    g.c_o = c_o;
    g.c_i = c_i;
    g.k_h = k_h;
    g.k_w = k_w;
    g.u_w = u_w;
    g.u_h = u_h;
    g.c_n = n / B;
    if (c_i % g.c_n || c_o % g.c_n) return set_err(GALA_ERR_PARAM, "channels must be multiples of c_n=%d", g.c_n);
    g.n_ib = c_i / g.c_n;
    g.n_ob = c_o / g.c_n;
    g.pair = pair;
    const int n_obp = (g.n_ob + pair - 1) / pair;
    const long long total = (long long)n_obp * g.n_ib * g.c_n * k_h * k_w;
    const int chunk = 4096;   // plaintexts per generate+encode round (32 MB of slots at N = 8192)
    uint32_t* slots;
    RET(scratch(c, &slots, (size_t)chunk * N));
    for (long long first = 0; first < total; first += chunk) {
        const int cnt = (int)(total - first < chunk ? total - first : chunk);
        KLAUNCH(c, "k_kg_slots", k_kg_slots<<<grid_for((long long)cnt * N, 256), 256, 0, c->stream>>>(c->dc, kern, g, first,
                                                                                                  cnt, slots));
        RET(gala_encode_plain(c, slots, cnt, pts + first * L * N));
    }
    release(c, slots);
    return GALA_OK;
}

// ---------------------------------------------------------------------------
// Kernel grouping, schedule 2 (factored plaintexts).  Every KG plaintext is a sum over the c_n
// bands of a 0/1 band mask times one kernel coefficient, so
//   acc[o][d] = sum_{ib, tap, beta} A[(o, d)][(ib, tap, beta)] * (Z[ib][tap] (.) Mask[tap][beta])
// with small signed integer A (Z: the rotated inputs, kept in the extended basis QP).  The masked
// products are split into bytes and the contraction over K = (ib, tap, beta) runs as an int8
// tensor-core GEMM (cuBLASLt, exact int32 accumulation); a recombination kernel rebuilds each word
// mod q exactly, then one ModDown per accumulator.  Post-mask form (frame-embedded inputs): the band
// masks move behind the GEMM (rows (m, beta), K = (ib, tap)).  K stays input-major: a K tile then
// touches the digit blocks of few inputs (tap-major was measured 20% slower, L2 misses).
// Oracle: o_conv_kg2.

int gala_kg2_encode_masks(gala_ctx* c, int k_h, int k_w, int u_w, int u_h, int pair, int band_only, uint64_t* masks)
{
    const int N = c->dc.N, L = c->dc.L, n = N / 2;
    const int B = u_w * u_h;
    if (B <= 0 || n % B || (k_h % 2) == 0 || (k_w % 2) == 0 || (pair != 1 && pair != 2))
        return set_err(GALA_ERR_PARAM, "bad kernel-grouping geometry");
    KgGeom g{};
    g.k_h = band_only ? 1 : k_h;   // band-only masks: no tap dimension
    g.k_w = band_only ? 1 : k_w;
    g.u_w = u_w;
    g.u_h = u_h;
    g.c_n = n / B;
    g.pair = pair;
    const int count = g.k_h * g.k_w * pair * g.c_n;
    uint32_t* slots;
    RET(scratch(c, &slots, (size_t)count * N));
    KLAUNCH(c, "k_kg_mask_slots", k_kg_mask_slots<<<grid_for((long long)count * N, 256), 256, 0, c->stream>>>(c->dc, g, slots));
    const int M = c->dc.M;
    u64* mont;
    RET(scratch(c, &mont, (size_t)count * M * N));
    for (int first = 0; first < count; first += 4096) {
        const int cnt = count - first < 4096 ? count - first : 4096;
        KLAUNCH(c, "k_encode", k_encode<2><<<cnt * M, ntt_threads(N), 2 * c->smem_ntt, c->stream>>>(
                                   c->dc, slots + (long long)first * N, mont + (long long)first * M * N));
    }
    KLAUNCH(c, "k_mont_to_shoup", k_mont_to_shoup<<<grid_for((long long)count * M * N, 256), 256, 0, c->stream>>>(
                                      c->dc, mont, count, band_only ? 1 : 0, (ulonglong2*)masks));
    release(c, slots);
    release(c, mont);
    (void)L;
    return GALA_OK;
}

static unsigned __int128 kg_offset(u64 q)
{
    const unsigned __int128 two90 = (unsigned __int128)1 << 90;
    return (two90 / q + 1) * q;
}

// nbatch independent images (e.g. the halo tiles of one layer) share the weights and every launch:
// cts [nbatch][n_ib][2][L][N] -> outs [nbatch][Mr / c_n][2][L][N] (fused tcgen05 path only for nbatch > 1)
static int conv_kg2_run(gala_ctx* c, bool post, const uint64_t* cts, int n_ib, const uint64_t* masks, int k, int nb,
                        const int8_t* coef, const int32_t* rowsum, int Mr, int Kp, const int* tap_steps, int band_step,
                        int c_n, uint64_t* outs, int nbatch = 1)
{
    const int N = c->dc.N, L = c->dc.L, M = c->dc.M;
    const long long W = 2LL * L * N, WQ = 2LL * M * N;
    if (n_ib <= 0 || k <= 0 || nb <= 0 || c_n <= 0 || Mr <= 0 || Mr % c_n) return set_err(GALA_ERR_DIM, "bad schedule-2 dims");
    if (k > KG_MAXK) return set_err(GALA_ERR_DIM, "at most %d kernel taps", KG_MAXK);
    const int Kreal = n_ib * k * (post ? 1 : nb);
    const int rows = post ? Mr * nb : Mr;     // GEMM rows
    if (Kp % 32 || Kp < Kreal) return set_err(GALA_ERR_DIM, "Kp=%d must be a multiple of 32 covering K=%d", Kp, Kreal);
    if (post && (nb > 32 || 32 % nb)) return set_err(GALA_ERR_DIM, "post-mask form needs nb | 32 (got %d)", nb);
    if (N % 32) return set_err(GALA_ERR_DIM, "ring degree below 32");
    // every int8 x int8 product has |a b| <= 128 * 128 = 2^14 (both operands may be -128: coefficients
    // and 0x80-biased bytes), so the int32 GEMM sums stay exact while Kp * 2^14 <= INT32_MAX (Kp < 2^17)
    if ((long long)Kp * 16384 > 2147483647LL) return set_err(GALA_ERR_DIM, "K too large for exact int32 accumulation");
    std::vector<int> tsteps(k);
    bool any_rot = false;
    for (int t = 0; t < k; t++) {
        tsteps[t] = norm_step(c, tap_steps[t]);
        if (tsteps[t] != 0) {
            if (!key_for(c, tsteps[t])) return set_err(GALA_ERR_NOKEY, "missing rotation key for step %d", tsteps[t]);
            any_rot = true;
        }
    }
    for (int d = 1; d < c_n; d++)
        if (!gala_has_rotation_key(c, d * band_step))
            return set_err(GALA_ERR_NOKEY, "missing rotation key for step %d", norm_step(c, d * band_step));
    if (!c->d_kg_off) {
        // [0, 2 GALA_MAXM): 128-bit offsets (hi, lo) per prime; [2 GALA_MAXM, 4 GALA_MAXM): (P mod q_j, Shoup);
        // [4 GALA_MAXM, 6 GALA_MAXM): (2^64 mod q_j, Shoup) -- the "mask" of the pre-mask epilogue
        std::vector<u64> off(6 * GALA_MAXM, 0);
        const u64 P = c->primes[L];
        for (int j = 0; j < M; j++) {
            unsigned __int128 o = kg_offset(c->primes[j]);
            off[2 * j] = (u64)(o >> 64);
            off[2 * j + 1] = (u64)o;
            const u64 pj = P % c->primes[j];
            off[2 * GALA_MAXM + 2 * j] = pj;
            off[2 * GALA_MAXM + 2 * j + 1] = (u64)((((unsigned __int128)pj) << 64) / c->primes[j]);
            const u64 rj = (u64)((((unsigned __int128)1) << 64) % c->primes[j]);
            off[4 * GALA_MAXM + 2 * j] = rj;
            off[4 * GALA_MAXM + 2 * j + 1] = (u64)((((unsigned __int128)rj) << 64) / c->primes[j]);
        }
        CK(cudaMalloc(&c->d_kg_off, sizeof(u64) * off.size()));
        CK(cudaMemcpy(c->d_kg_off, off.data(), sizeof(u64) * off.size(), cudaMemcpyHostToDevice));
    }
    const int nb_y = post ? 1 : nb;          // masks applied per K column (pre) or per GEMM row group (post)
    if (KG_KT % nb_y) return set_err(GALA_ERR_DIM, "band count %d must divide %d", nb, KG_KT);
    // 1. one decomposition per input: identity digit block [(L M + L)][N]
    const long long blk_words = (long long)(L * M + L) * N;
    const int n_in = nbatch * n_ib;          // decomposed inputs over the whole batch
    u64 *dig, *Dblk;
    RET(scratch(c, &dig, (size_t)n_in * L * N));
    RET(scratch(c, &Dblk, (size_t)n_in * blk_words));
    std::vector<TermDesc> td(n_in);
    for (int b = 0; b < n_in; b++) {
        td[b].X = cts + b * W;
        td[b].pt = nullptr;
        td[b].dig = dig + (long long)b * L * N;
        td[b].blk = Dblk + (long long)b * blk_words;
        td[b].rot_off = 0;
        td[b].rot_cnt = 1;
    }
    std::vector<unsigned> gal(k + 1, 1u);     // gal[0] = identity (the decomposition); gal[1 + t] per tap
    std::vector<const u64*> keys(k, nullptr);
    for (int t = 0; t < k; t++) {
        if (tsteps[t]) {
            gal[1 + t] = galois_of(c, tsteps[t]);
            keys[t] = key_for(c, tsteps[t]);
        }
    }
    size_t o_gal = (td.size() * sizeof(TermDesc) + 15) & ~(size_t)15;
    size_t o_keys = (o_gal + gal.size() * sizeof(unsigned) + 15) & ~(size_t)15;
    std::vector<char> blob(o_keys + keys.size() * sizeof(u64*));
    memcpy(blob.data(), td.data(), td.size() * sizeof(TermDesc));
    memcpy(blob.data() + o_gal, gal.data(), gal.size() * sizeof(unsigned));
    memcpy(blob.data() + o_keys, keys.data(), keys.size() * sizeof(u64*));
    char* d_blob;
    RET(upload(c, blob.data(), blob.size(), (void**)&d_blob));
    const int nt = ntt_threads(N);
    const unsigned* d_gal = (const unsigned*)(d_blob + o_gal);
    if (any_rot) {
        KLAUNCH(c, "k_digits_intt", k_digits_intt<<<(unsigned)(n_in * L), nt, c->smem_ntt, c->stream>>>(
                                        c->dc, (const TermDesc*)d_blob, d_gal, blk_words));
        KLAUNCH(c, "k_digits_perm", k_digits_perm<<<(unsigned)(n_in * L * L), nt, c->smem_ntt, c->stream>>>(
                                        c->dc, (const TermDesc*)d_blob, d_gal, blk_words));
    }
    // the byte planes are written in the tensor-core tile order so every k_kg_tc pipeline stage is one
    // bulk copy
    // 2. fused key switch (no ModDown) + band masks -> biased bytes, K-contiguous: Bt[8 WQ][Kp]
    int8_t* Bt;
    RET(scratch(c, &Bt, (size_t)8 * WQ * Kp * nbatch));
    {
        dim3 grid((unsigned)((WQ + KG_PT - 1) / KG_PT), (unsigned)((Kp + KG_KT - 1) / KG_KT), (unsigned)nbatch);
        const u64* const* dk = (const u64* const*)(d_blob + o_keys);
        const ulonglong2* pm = (const ulonglong2*)(c->d_kg_off + 2 * GALA_MAXM);
#define KG_ZYN(LL, LN)                                                                                              \
    KLAUNCH(c, "k_kg_zy", (k_kg_zy<LL, LN><<<grid, 256, 0, c->stream>>>(c->dc, Dblk, cts, dk, d_gal + 1,           \
                                                                   post ? nullptr : (const ulonglong2*)masks, pm, k,  \
                                                                   nb_y, n_ib, Kp, Bt, 1)))
#define KG_ZY(LL)                                                                                                  \
    do {                                                                                                           \
        if (c->dc.logN == 13) KG_ZYN(LL, 13);                                                                      \
        else if (c->dc.logN == 12) KG_ZYN(LL, 12);                                                                 \
        else KG_ZYN(LL, 0);                                                                                        \
    } while (0)
#define KG_ZY2P(LL, LN, PRE)                                                                                        \
    KLAUNCH(c, "k_kg_zy", (k_kg_zy2<LL, LN, PRE><<<grid2, 256, 2 * KG_PT * KG_KT * 8, c->stream>>>(                  \
                              c->dc, Dblk, cts, dk, d_gal + 1, post ? nullptr : (const ulonglong2*)masks, pm, k, nb_y, \
                              n_ib, Kp, Bt)))
#define KG_ZY2N(LL, LN)                                                                                             \
    do {                                                                                                           \
        if (post) KG_ZY2P(LL, LN, false);                                                                          \
        else KG_ZY2P(LL, LN, true);                                                                                \
    } while (0)
#define KG_ZY2(LL)                                                                                                 \
    do {                                                                                                           \
        if (c->dc.logN == 13) KG_ZY2N(LL, 13);                                                                     \
        else if (c->dc.logN == 12) KG_ZY2N(LL, 12);                                                                \
        else KG_ZY2N(LL, 0);                                                                                       \
    } while (0)
        // both key-switch components per thread (k_kg_zy2; N >= 32, so a block of 32 positions never
        // straddles a prime); GALA_KG_ZY1 selects the one-component kernel (A/B experiments)
        const dim3 grid2((unsigned)((WQ / 2 + KG_PT - 1) / KG_PT), (unsigned)((Kp + KG_KT - 1) / KG_KT), (unsigned)nbatch);
        if (getenv("GALA_KG_ZY1") == nullptr) {
            switch (L) {
                case 1: KG_ZY2(1); break;
                case 2: KG_ZY2(2); break;
                case 3: KG_ZY2(3); break;
                default: KG_ZY2(4); break;
            }
        } else {
            switch (L) {
                case 1: KG_ZY(1); break;
                case 2: KG_ZY(2); break;
                case 3: KG_ZY(3); break;
                default: KG_ZY(4); break;
            }
        }
#undef KG_ZY
#undef KG_ZYN
#undef KG_ZY2
#undef KG_ZY2N
#undef KG_ZY2P
    }
    release(c, dig);
    release(c, Dblk);
    release(c, d_blob);
    u64* accq;
    RET(scratch(c, &accq, (size_t)nbatch * Mr * WQ));
    {
        // 3+4. first-Add on the tensor cores (k_kg_tc) with the byte recombination in the epilogue: post-mask,
        // GEMM rows (m, beta) times their band masks and summed over the nb bands; pre-mask (masks already
        // in the K columns), one GEMM row per accumulator and no mask (the 2^64 mod q_j constant instead)
        const int nb_e = post ? nb : 1;
        const int rows_p = (rows + 127) / 128 * 128;
        int8_t* Acan;
        RET(scratch(c, &Acan, (size_t)rows_p * Kp));
        KLAUNCH(c, "k_kg_tc_layout_a", k_kg_tc_layout_a<<<grid_for((long long)rows_p * Kp / 16, 256), 256, 0, c->stream>>>(
                                           coef, rows, rows_p, Kp, Acan));
        const int ntiles = (int)(8 * WQ / KG_TC_N) * nbatch;
        const int rbs = rows_p / 128;
        long long jobs = (long long)ntiles * rbs;
        const int grid = (int)(jobs < c->num_sms ? jobs : c->num_sms);
        const size_t smem = (size_t)KG_TC_STAGES * KG_TC_KCS * (128 + KG_TC_N) * 16 + 2 * 512 * (size_t)nb_e;
        KLAUNCH(c, "k_kg_tc", k_kg_tc<<<grid, KG_TC_THREADS, smem, c->stream>>>(
                                  c->dc, Acan, rowsum, rows, rbs, nb_e, Mr, Bt, Kp, ntiles, (const ulonglong2*)c->d_kg_off,
                                  post ? (const ulonglong2*)masks : nullptr, (const ulonglong2*)c->d_kg_off + 2 * GALA_MAXM,
                                  accq, (int)(8 * WQ / KG_TC_N)));
        release(c, Acan);
        release(c, Bt);
    }
    // 5. one ModDown per accumulator (straight into outs when there is no second-Perm)
    const int Mb = Mr * nbatch;              // accumulators over the batch
    u64 *acc = outs, *rr;
    if (c_n > 1) RET(scratch(c, &acc, (size_t)Mb * W));
    RET(scratch(c, &rr, (size_t)Mb * 2 * N));
    RET(launch_inv<false>(c, accq + (long long)L * N, rr, Mb * 2, pm_make(1, 1, L, 0, (long long)M * N, N),
                          "k_ntt_inv[moddown]"));
    MdArgs a{};
    a.r = rr;
    a.U = accq;
    a.add0 = nullptr;
    a.add1 = nullptr;
    a.add_is = 0;
    a.out = acc;
    a.out_is = W;
    a.outs = nullptr;
    KLAUNCH(c, "k_moddown", k_moddown<<<Mb * 2 * L, ntt_threads(N), c->smem_ntt, c->stream>>>(c->dc, a));
    release(c, rr);
    release(c, accq);
    // 6. second-Perm: out[o] = sum_d rot_{d * band}(acc[o][d]), one lazy ModDown per o
    if (c_n > 1) {
        RET(rotate_sum_regular(c, acc, W, (long long)Mr * W, nullptr, nbatch, Mr / c_n, c_n, band_step, outs,
                               (long long)(Mr / c_n) * W));
        release(c, acc);
    }
    return GALA_OK;
}

int gala_conv_kg2(gala_ctx* c, const uint64_t* cts, int n_ib, const uint64_t* masks, int k, int nb,
                  const int8_t* coef, const int32_t* rowsum, int Mr, int Kp, const int* tap_steps, int band_step,
                  int c_n, uint64_t* outs)
{
    return conv_kg2_run(c, false, cts, n_ib, masks, k, nb, coef, rowsum, Mr, Kp, tap_steps, band_step, c_n, outs);
}

int gala_conv_kg2_post(gala_ctx* c, const uint64_t* cts, int n_ib, const uint64_t* masks, int k, int nb,
                       const int8_t* coef, const int32_t* rowsum, int Mr, int Kp, const int* tap_steps, int band_step,
                       int c_n, uint64_t* outs)
{
    return conv_kg2_run(c, true, cts, n_ib, masks, k, nb, coef, rowsum, Mr, Kp, tap_steps, band_step, c_n, outs);
}

int gala_conv_kg2_post_batch(gala_ctx* c, const uint64_t* cts, int nbatch, int n_ib, const uint64_t* masks, int k, int nb,
                             const int8_t* coef, const int32_t* rowsum, int Mr, int Kp, const int* tap_steps,
                             int band_step, int c_n, uint64_t* outs)
{
    if (nbatch <= 0) return set_err(GALA_ERR_DIM, "empty batch");
    return conv_kg2_run(c, true, cts, n_ib, masks, k, nb, coef, rowsum, Mr, Kp, tap_steps, band_step, c_n, outs, nbatch);
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

int gala_set_fc_tc_min_terms(gala_ctx* c, int min_terms)
{
    if (min_terms < 1) return set_err(GALA_ERR_PARAM, "min_terms must be >= 1");
    c->fc_tc_min_T = min_terms;
    return GALA_OK;
}

int gala_profile_enable(gala_ctx* c, int on)
{
    c->prof_on = on != 0;
    return GALA_OK;
}

// aggregate recorded launches by kernel name into JSON {"name": [count, total_ms], ...};
// synchronises the stream and clears the records
int gala_profile_json(gala_ctx* c, char* buf, size_t cap)
{
    CK(cudaStreamSynchronize(c->stream));
    std::map<std::string, std::pair<long, double>> agg;
    for (auto& r : c->recs) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        auto& e = agg[r.name];
        e.first += 1;
        e.second += ms;
        c->pool.push_back(r.a);
        c->pool.push_back(r.b);
    }
    c->recs.clear();
    std::string out = "{";
    bool first = true;
    for (auto& kv : agg) {
        char tmp[256];
        snprintf(tmp, sizeof(tmp), "%s\"%s\": [%ld, %.6f]", first ? "" : ", ", kv.first.c_str(), kv.second.first,
                 kv.second.second);
        out += tmp;
        first = false;
    }
    out += "}";
    if (out.size() + 1 > cap) return set_err(GALA_ERR_DIM, "profile buffer too small (%zu)", out.size() + 1);
    memcpy(buf, out.c_str(), out.size() + 1);
    return GALA_OK;
}

// Throughput of the library's own 60-bit Shoup modmul (the NTT butterfly
// multiply) in modmul/s: every thread runs 8 independent dependency chains.
int gala_bench_modmul(gala_ctx* c, int blocks, int iters, double* modmul_per_s)
{
    u64* sink;
    RET(scratch(c, &sink, (size_t)blocks * 256));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const u64 q = c->primes[0];
    const u64 w = (q >> 3) | 1, wsh = h_shoup(w % q, q);
    k_bench_modmul<<<blocks, 256, 0, c->stream>>>(q, w % q, wsh, iters, sink); // warm-up
    CK(cudaEventRecord(a, c->stream));
    KLAUNCH(c, "k_bench_modmul", k_bench_modmul<<<blocks, 256, 0, c->stream>>>(q, w % q, wsh, iters, sink));
    CK(cudaEventRecord(b, c->stream));
    CK(cudaEventSynchronize(b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    *modmul_per_s = (double)blocks * 256.0 * 8.0 * iters / (ms * 1e-3);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    release(c, sink);
    return GALA_OK;
}

} // extern "C"

#ifdef GTC_PROF
extern "C" int gala_debug_gtc_prof(unsigned long long* out, int rows)
{
    return (int)cudaMemcpyFromSymbol(out, g_gtc_prof, (size_t)rows * 16 * sizeof(unsigned long long));
}
#endif


// k_gala_kf timeline of CTA 0 (experiment builds with -DKF_TRACE; tools/kf_trace.py)
extern "C" int gala_debug_kf_trace(unsigned long long* out)
{
#ifdef KF_TRACE
    return (int)cudaMemcpyFromSymbol(out, g_kf_trace, sizeof(unsigned long long) * 32 * 1024);
#else
    (void)out;
    return -1;
#endif
}
