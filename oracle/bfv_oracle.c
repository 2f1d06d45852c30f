/*
 * bfv_oracle.c -- CPU RNS-BFV oracle.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or
 * the timed CPU baseline.  The product path (paper_2105_01827_b200) never
 * links or calls it.
 *
 * What it restates.  The reference package (arxiv 2105.01827, GALA) ships a
 * *mock* HE backend whose ciphertexts are plaintext slot vectors
 * (pkg/src/gala/backend.py:1-17).  The slot semantics this oracle must
 * reproduce after decryption are:
 *   encrypt/decrypt  backend.py:228-243      rotate_left   ring.py:86-91
 *   he_add           backend.py:246-254      he_scmult     backend.py:257-265
 *   he_perm          backend.py:268-276      he_decperm/he_hstperm 279-294
 *   subtract_plain   backend.py:297-311
 *   mv_gala          matvec.py:305-320 (sum_t perm(scmult(x, p_t), t))
 *   mimo_kernel_grouping conv.py:268-293 (first-Add, second-Perm)
 * The reference has no ciphertext words; this file *defines* them (SURVEY.md
 * section 8(c)): every algorithmic choice below (digit decomposition, key
 * layout, ModDown rounding, BSGS tree, lazy ModDown points) is the contract
 * the CUDA library must match word for word.
 *
 * Representation: ring Z_q[X]/(X^N+1); every ciphertext / key polynomial is
 * kept in the *natural-order* NTT domain, A[k] = a(psi^(2k+1)).  All public
 * entry points exchange canonical coefficient-domain words (natural order,
 * values in [0, q_j)), so internal layouts never leak into the contract.
 *
 * Scheme (one special prime P, hybrid key switching with one digit per
 * ciphertext prime):
 *   encode(slots)  slot (r,c) <-> m(zeta^(e)), e = 3^c (row 0) / -3^c (row 1)
 *   encrypt        c1 = a, c0 = -a s + e + Delta m,   Delta = floor(Q/p)
 *   decrypt        m = round(p [c0 + c1 s]_Q / Q) mod p (RNS, exact rounding
 *                  through a 2^-64 fixed-point fraction sum)
 *   plain operand  centred lift of encode(slots) into every q_j
 *   ksk_g[i]       b = -a_i s + e_i + [j==i] (P mod q_i) sigma_g(s)  (mod q_j)
 *                  b = -a_i s + e_i                                 (mod P)
 *   decompose      d_i = [c1]_{q_i} in [0,q_i), D_ij = NTT_j(d_i mod q_j)
 *   KSraw(g)       U_c,j = sum_i sigma_g(D_ij) * ksk_g[i].(b|a)_j  (over QP)
 *   ModDown(U)     r = centred INTT_P(U_P); out_j = (U_j - NTT_j(r)) P^-1
 *   rotate(g)      (sigma_g(c0) + MD(U_0), MD(U_1))
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef uint64_t u64;
typedef int64_t i64;
typedef unsigned __int128 u128;

#define MAXM 6 /* L <= 4 ciphertext primes + 1 special + spare */

typedef struct {
    u64 q;
    u64 *psi_pow, *psi_pow_sh;   /* psi^i and Shoup companions      */
    u64 *ipsi_pow, *ipsi_pow_sh; /* psi^-i * N^-1 and companions    */
    u64 *w, *w_sh;               /* omega^k (k < N/2), omega = psi^2 */
    u64 *iw, *iw_sh;             /* omega^-k                        */
} modtab;

typedef struct {
    int N, logN, L, M;           /* M = L + 1 (with the special prime) */
    modtab t[MAXM];              /* t[0..L-1] = q_j, t[L] = P           */
    modtab tp;                   /* plaintext modulus p                 */
    u64 p;
    u64 delta_mod[MAXM];         /* floor(Q/p) mod q_j                  */
    u64 P_mod[MAXM], Pinv[MAXM]; /* P mod q_j, P^-1 mod q_j             */
    u64 qhat_inv[MAXM];          /* [(Q/q_i)^-1]_{q_i}                  */
    int *slot_ntt;               /* slot index -> NTT_p natural index   */
    u64 *S;                      /* secret, NTT, [M][N]                 */
    i64 *s;                      /* secret coefficients                 */
    u64 **ksk;                   /* by step: [L][2][M][N] NTT           */
    int nsteps;
} octx;

/* ------------------------------------------------------------------ */
/* scalar modular arithmetic                                           */
static inline u64 mulmod(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
static inline u64 addmod(u64 a, u64 b, u64 q) { u64 s = a + b; return s >= q ? s - q : s; }
static inline u64 submod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }
static inline u64 shoup(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }
static inline u64 mulshoup(u64 a, u64 w, u64 wsh, u64 q)
{
    u64 hi = (u64)(((u128)a * wsh) >> 64);
    u64 r = a * w - hi * q;
    return r >= q ? r - q : r;
}
static u64 powmod(u64 b, u64 e, u64 q)
{
    u64 r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = mulmod(r, b, q);
        b = mulmod(b, b, q);
        e >>= 1;
    }
    return r;
}
static u64 invmod(u64 a, u64 q) { return powmod(a, q - 2, q); } /* q prime */
static inline u64 from_signed(i64 v, u64 q)
{
    if (v >= 0) return (u64)v % q;
    u64 m = (u64)(-(v + 1)) % q; /* -(v+1) >= 0 */
    return q - 1 - m;
}

/* ------------------------------------------------------------------ */
/* NTT: natural order in, natural order out: A[k] = a(psi^(2k+1)).      */
static void tab_init(modtab *t, u64 q, u64 psi, int N)
{
    t->q = q;
    size_t sz = (size_t)N * sizeof(u64);
    t->psi_pow = malloc(sz); t->psi_pow_sh = malloc(sz);
    t->ipsi_pow = malloc(sz); t->ipsi_pow_sh = malloc(sz);
    t->w = malloc(sz / 2 + 8); t->w_sh = malloc(sz / 2 + 8);
    t->iw = malloc(sz / 2 + 8); t->iw_sh = malloc(sz / 2 + 8);
    u64 ipsi = invmod(psi, q), ninv = invmod((u64)N % q, q);
    u64 x = 1, y = ninv;
    for (int i = 0; i < N; i++) {
        t->psi_pow[i] = x; t->psi_pow_sh[i] = shoup(x, q);
        t->ipsi_pow[i] = y; t->ipsi_pow_sh[i] = shoup(y, q);
        x = mulmod(x, psi, q); y = mulmod(y, ipsi, q);
    }
    u64 om = mulmod(psi, psi, q), iom = invmod(om, q);
    x = 1; y = 1;
    for (int i = 0; i < N / 2; i++) {
        t->w[i] = x; t->w_sh[i] = shoup(x, q);
        t->iw[i] = y; t->iw_sh[i] = shoup(y, q);
        x = mulmod(x, om, q); y = mulmod(y, iom, q);
    }
}
static void tab_free(modtab *t)
{
    free(t->psi_pow); free(t->psi_pow_sh); free(t->ipsi_pow); free(t->ipsi_pow_sh);
    free(t->w); free(t->w_sh); free(t->iw); free(t->iw_sh);
}

static void bitrev_perm(u64 *a, int N)
{
    for (int i = 1, j = 0; i < N; i++) {
        int bit = N >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) { u64 t = a[i]; a[i] = a[j]; a[j] = t; }
    }
}

static void cyclic_ntt(u64 *a, int N, const u64 *w, const u64 *wsh, u64 q)
{
    bitrev_perm(a, N);
    for (int len = 2; len <= N; len <<= 1) {
        int half = len >> 1, stride = N / len;
        for (int i = 0; i < N; i += len)
            for (int k = 0; k < half; k++) {
                u64 u = a[i + k];
                u64 v = mulshoup(a[i + k + half], w[k * stride], wsh[k * stride], q);
                a[i + k] = addmod(u, v, q);
                a[i + k + half] = submod(u, v, q);
            }
    }
}

static void ntt_fwd(const modtab *t, u64 *a, int N)
{
    for (int i = 0; i < N; i++) a[i] = mulshoup(a[i], t->psi_pow[i], t->psi_pow_sh[i], t->q);
    cyclic_ntt(a, N, t->w, t->w_sh, t->q);
}
static void ntt_inv(const modtab *t, u64 *a, int N)
{
    cyclic_ntt(a, N, t->iw, t->iw_sh, t->q);
    for (int i = 0; i < N; i++) a[i] = mulshoup(a[i], t->ipsi_pow[i], t->ipsi_pow_sh[i], t->q);
}

/* sigma_g in the natural NTT domain: out[k] = in[((2k+1) g mod 2N - 1)/2] */
static void automorph_ntt(const u64 *in, u64 *out, int N, u64 g)
{
    u64 two_n = 2 * (u64)N;
    for (int k = 0; k < N; k++) {
        u64 e = ((2 * (u64)k + 1) * g) % two_n;
        out[k] = in[(e - 1) / 2];
    }
}
/* sigma_g on signed coefficients: X^i -> X^(i g mod 2N), wrap negates */
static void automorph_coef_signed(const i64 *in, i64 *out, int N, u64 g)
{
    u64 two_n = 2 * (u64)N;
    for (int i = 0; i < N; i++) {
        u64 e = ((u64)i * g) % two_n;
        if (e < (u64)N) out[e] = in[i];
        else out[e - N] = -in[i];
    }
}

static u64 galois(int step, int N)
{
    int n = N / 2;
    int s = ((step % n) + n) % n;
    return powmod(3, (u64)s, 2 * (u64)N);
}

/* ------------------------------------------------------------------ */
/* context                                                             */
void *o_create(int N, int L, const u64 *primes, const u64 *psis, u64 p, u64 psi_p)
{
    if (L < 1 || L + 1 > MAXM || N < 8 || (N & (N - 1))) return NULL;
    octx *c = calloc(1, sizeof(octx));
    c->N = N; c->L = L; c->M = L + 1; c->p = p;
    while ((1 << c->logN) < N) c->logN++;
    for (int j = 0; j < c->M; j++) tab_init(&c->t[j], primes[j], psis[j], N);
    tab_init(&c->tp, p, psi_p, N);
    /* Delta = floor(Q/p) mod q_j via multi-limb Q */
    u64 Qlimb[MAXM + 1];
    int nl = 1;
    memset(Qlimb, 0, sizeof(Qlimb));
    Qlimb[0] = 1;
    for (int i = 0; i < L; i++) {
        u128 carry = 0;
        for (int k = 0; k < nl; k++) {
            u128 v = (u128)Qlimb[k] * primes[i] + carry;
            Qlimb[k] = (u64)v; carry = v >> 64;
        }
        if (carry) Qlimb[nl++] = (u64)carry;
    }
    u64 D[MAXM + 1];
    u128 rem = 0;
    for (int k = nl - 1; k >= 0; k--) {
        u128 cur = (rem << 64) | Qlimb[k];
        D[k] = (u64)(cur / p); rem = cur % p;
    }
    for (int j = 0; j < c->M; j++) {
        u64 q = primes[j];
        u128 acc = 0;
        for (int k = nl - 1; k >= 0; k--) acc = ((acc << 64) | D[k]) % q;
        c->delta_mod[j] = (u64)acc;
        c->P_mod[j] = primes[L] % q;
        c->Pinv[j] = (j < L) ? invmod(primes[L] % q, q) : 0;
    }
    for (int i = 0; i < L; i++) {
        u64 qh = 1;
        for (int k = 0; k < L; k++) if (k != i) qh = mulmod(qh, primes[k] % primes[i], primes[i]);
        c->qhat_inv[i] = invmod(qh, primes[i]);
    }
    /* slot map */
    int n = N / 2;
    c->slot_ntt = malloc(sizeof(int) * N);
    u64 e = 1, two_n = 2 * (u64)N;
    for (int col = 0; col < n; col++) {
        c->slot_ntt[col] = (int)((e - 1) / 2);
        c->slot_ntt[n + col] = (int)((two_n - e - 1) / 2);
        e = (e * 3) % two_n;
    }
    c->nsteps = n;
    c->ksk = calloc((size_t)n, sizeof(u64 *));
    return c;
}

void o_destroy(void *h)
{
    octx *c = h;
    if (!c) return;
    for (int j = 0; j < c->M; j++) tab_free(&c->t[j]);
    tab_free(&c->tp);
    free(c->slot_ntt); free(c->S); free(c->s);
    for (int i = 0; i < c->nsteps; i++) free(c->ksk[i]);
    free(c->ksk);
    free(c);
}

int o_set_secret(void *h, const int8_t *s)
{
    octx *c = h;
    int N = c->N;
    free(c->S); free(c->s);
    c->S = malloc(sizeof(u64) * (size_t)c->M * N);
    c->s = malloc(sizeof(i64) * N);
    for (int i = 0; i < N; i++) c->s[i] = s[i];
    for (int j = 0; j < c->M; j++) {
        u64 *Sj = c->S + (size_t)j * N;
        for (int i = 0; i < N; i++) Sj[i] = from_signed(s[i], c->t[j].q);
        ntt_fwd(&c->t[j], Sj, N);
    }
    return 0;
}

/* a: [L][M][N] uniform coefficients (mod each prime), e: [L][N] signed */
int o_gen_rotkey(void *h, int step, const u64 *a, const i64 *e)
{
    octx *c = h;
    int N = c->N, L = c->L, M = c->M, n = N / 2;
    if (!c->S) return -3;
    int s = ((step % n) + n) % n;
    if (s == 0) return 0;
    u64 g = galois(s, N);
    i64 *sr = malloc(sizeof(i64) * N);
    automorph_coef_signed(c->s, sr, N, g);
    u64 *key = malloc(sizeof(u64) * (size_t)L * 2 * M * N);
    u64 *tmp = malloc(sizeof(u64) * N), *sp = malloc(sizeof(u64) * N);
    for (int i = 0; i < L; i++)
        for (int j = 0; j < M; j++) {
            const modtab *t = &c->t[j];
            u64 q = t->q;
            u64 *b = key + (((size_t)i * 2 + 0) * M + j) * N;
            u64 *ak = key + (((size_t)i * 2 + 1) * M + j) * N;
            for (int k = 0; k < N; k++) ak[k] = a[((size_t)i * M + j) * N + k] % q;
            ntt_fwd(t, ak, N);
            for (int k = 0; k < N; k++) tmp[k] = from_signed(e[(size_t)i * N + k], q);
            ntt_fwd(t, tmp, N);
            const u64 *Sj = c->S + (size_t)j * N;
            for (int k = 0; k < N; k++) b[k] = submod(tmp[k], mulmod(ak[k], Sj[k], q), q);
            if (j == i) {
                for (int k = 0; k < N; k++) sp[k] = from_signed(sr[k], q);
                ntt_fwd(t, sp, N);
                for (int k = 0; k < N; k++) b[k] = addmod(b[k], mulmod(c->P_mod[j], sp[k], q), q);
            }
        }
    free(c->ksk[s]);
    c->ksk[s] = key;
    free(sr); free(tmp); free(sp);
    return 0;
}

/* ------------------------------------------------------------------ */
/* encoding                                                            */
void o_encode_p(void *h, const uint32_t *slots, u64 *m)
{
    octx *c = h;
    int N = c->N;
    for (int i = 0; i < N; i++) m[c->slot_ntt[i]] = slots[i] % c->p;
    ntt_inv(&c->tp, m, N);
}
void o_decode_p(void *h, const u64 *m, uint32_t *slots)
{
    octx *c = h;
    int N = c->N;
    u64 *A = malloc(sizeof(u64) * N);
    memcpy(A, m, sizeof(u64) * N);
    ntt_fwd(&c->tp, A, N);
    for (int i = 0; i < N; i++) slots[i] = (uint32_t)A[c->slot_ntt[i]];
    free(A);
}

/* plaintext operand, NTT domain [L][N] (centred lift of the mod-p poly) */
static void encode_pt_ntt(const octx *c, const uint32_t *slots, u64 *pt)
{
    int N = c->N;
    u64 *m = malloc(sizeof(u64) * N);
    o_encode_p((void *)c, slots, m);
    u64 half = c->p >> 1;
    for (int j = 0; j < c->L; j++) {
        u64 q = c->t[j].q;
        u64 *d = pt + (size_t)j * N;
        for (int i = 0; i < N; i++) d[i] = m[i] > half ? q - (c->p - m[i]) : m[i];
        ntt_fwd(&c->t[j], d, N);
    }
    free(m);
}
/* canonical plaintext words (coefficient domain) for cross-checking */
void o_encode(void *h, const uint32_t *slots, u64 *pt)
{
    octx *c = h;
    encode_pt_ntt(c, slots, pt);
    for (int j = 0; j < c->L; j++) ntt_inv(&c->t[j], pt + (size_t)j * c->N, c->N);
}

/* Delta * encode(slots), NTT domain, [L][N] */
static void encode_scaled_ntt(const octx *c, const uint32_t *slots, u64 *out)
{
    int N = c->N;
    u64 *m = malloc(sizeof(u64) * N);
    o_encode_p((void *)c, slots, m);
    for (int j = 0; j < c->L; j++) {
        u64 q = c->t[j].q;
        u64 *d = out + (size_t)j * N;
        for (int i = 0; i < N; i++) d[i] = mulmod(c->delta_mod[j], m[i], q);
        ntt_fwd(&c->t[j], d, N);
    }
    free(m);
}

/* ciphertext layout helpers: [2][L][N] */
static void ct_to_ntt(const octx *c, const u64 *in, u64 *out)
{
    int N = c->N, L = c->L;
    memcpy(out, in, sizeof(u64) * 2 * (size_t)L * N);
    for (int k = 0; k < 2; k++)
        for (int j = 0; j < L; j++) ntt_fwd(&c->t[j], out + ((size_t)k * L + j) * N, N);
}
static void ct_from_ntt(const octx *c, const u64 *in, u64 *out)
{
    int N = c->N, L = c->L;
    memcpy(out, in, sizeof(u64) * 2 * (size_t)L * N);
    for (int k = 0; k < 2; k++)
        for (int j = 0; j < L; j++) ntt_inv(&c->t[j], out + ((size_t)k * L + j) * N, N);
}

void o_encrypt(void *h, const uint32_t *slots, const u64 *a, const i64 *e, u64 *ct)
{
    octx *c = h;
    int N = c->N, L = c->L;
    u64 *dm = malloc(sizeof(u64) * (size_t)L * N);
    u64 *A = malloc(sizeof(u64) * N), *E = malloc(sizeof(u64) * N);
    u64 *out = malloc(sizeof(u64) * 2 * (size_t)L * N);
    encode_scaled_ntt(c, slots, dm);
    for (int j = 0; j < L; j++) {
        u64 q = c->t[j].q;
        for (int i = 0; i < N; i++) { A[i] = a[(size_t)j * N + i] % q; E[i] = from_signed(e[i], q); }
        ntt_fwd(&c->t[j], A, N);
        ntt_fwd(&c->t[j], E, N);
        const u64 *Sj = c->S + (size_t)j * N;
        u64 *c0 = out + (size_t)j * N, *c1 = out + ((size_t)L + j) * N;
        for (int i = 0; i < N; i++) {
            c1[i] = A[i];
            c0[i] = addmod(submod(E[i], mulmod(A[i], Sj[i], q), q), dm[(size_t)j * N + i], q);
        }
    }
    ct_from_ntt(c, out, ct);
    free(dm); free(A); free(E); free(out);
}

/* exact-rounding RNS decryption; see header */
void o_decrypt(void *h, const u64 *ct, uint32_t *slots)
{
    octx *c = h;
    int N = c->N, L = c->L;
    u64 *X = malloc(sizeof(u64) * (size_t)L * N);
    u64 *m = malloc(sizeof(u64) * N);
    u64 *tmp = malloc(sizeof(u64) * N);
    for (int j = 0; j < L; j++) {
        u64 q = c->t[j].q;
        u64 *x = X + (size_t)j * N;
        memcpy(x, ct + (size_t)j * N, sizeof(u64) * N);
        memcpy(tmp, ct + ((size_t)L + j) * N, sizeof(u64) * N);
        ntt_fwd(&c->t[j], x, N);
        ntt_fwd(&c->t[j], tmp, N);
        const u64 *Sj = c->S + (size_t)j * N;
        for (int i = 0; i < N; i++) x[i] = addmod(x[i], mulmod(tmp[i], Sj[i], q), q);
        ntt_inv(&c->t[j], x, N);
    }
    for (int i = 0; i < N; i++) {
        u64 sum_a = 0;
        u128 frac = 0;
        for (int j = 0; j < L; j++) {
            u64 q = c->t[j].q;
            u64 y = mulmod(X[(size_t)j * N + i], c->qhat_inv[j], q);
            u128 yp = (u128)y * c->p;
            u64 aq = (u64)(yp / q), b = (u64)(yp % q);
            sum_a += aq;
            frac += (u128)((((u128)b) << 64) / q);
        }
        u64 rounded = sum_a + (u64)((frac + ((u128)1 << 63)) >> 64);
        m[i] = rounded % c->p;
    }
    o_decode_p(c, m, slots);
    free(X); free(m); free(tmp);
}

/* ------------------------------------------------------------------ */
/* elementwise ops on canonical words                                  */
void o_add(void *h, const u64 *a, const u64 *b, u64 *out)
{
    octx *c = h;
    int N = c->N, L = c->L;
    for (int k = 0; k < 2; k++)
        for (int j = 0; j < L; j++) {
            u64 q = c->t[j].q;
            size_t o = ((size_t)k * L + j) * N;
            for (int i = 0; i < N; i++) out[o + i] = addmod(a[o + i], b[o + i], q);
        }
}

void o_sub_plain(void *h, const u64 *ct, const uint32_t *r, u64 *out)
{
    octx *c = h;
    int N = c->N, L = c->L;
    u64 *dm = malloc(sizeof(u64) * (size_t)L * N);
    encode_scaled_ntt(c, r, dm);
    for (int j = 0; j < L; j++) ntt_inv(&c->t[j], dm + (size_t)j * N, N);
    memcpy(out, ct, sizeof(u64) * 2 * (size_t)L * N);
    for (int j = 0; j < L; j++) {
        u64 q = c->t[j].q;
        for (int i = 0; i < N; i++) out[(size_t)j * N + i] = submod(ct[(size_t)j * N + i], dm[(size_t)j * N + i], q);
    }
    free(dm);
}

static void scmult_ntt(const octx *c, const u64 *ctn, const u64 *pt, u64 *out)
{
    int N = c->N, L = c->L;
    for (int k = 0; k < 2; k++)
        for (int j = 0; j < L; j++) {
            u64 q = c->t[j].q;
            size_t o = ((size_t)k * L + j) * N;
            for (int i = 0; i < N; i++) out[o + i] = mulmod(ctn[o + i], pt[(size_t)j * N + i], q);
        }
}

void o_scmult(void *h, const u64 *ct, const uint32_t *slots, u64 *out)
{
    octx *c = h;
    size_t W = 2 * (size_t)c->L * c->N;
    u64 *ctn = malloc(sizeof(u64) * W), *res = malloc(sizeof(u64) * W);
    u64 *pt = malloc(sizeof(u64) * (size_t)c->L * c->N);
    ct_to_ntt(c, ct, ctn);
    encode_pt_ntt(c, slots, pt);
    scmult_ntt(c, ctn, pt, res);
    ct_from_ntt(c, res, out);
    free(ctn); free(res); free(pt);
}

/* ------------------------------------------------------------------ */
/* key switching                                                       */
/* D: [L][M][N] NTT digits of c1 (NTT, [L][N]) */
static void decompose(const octx *c, const u64 *c1, u64 *D)
{
    int N = c->N, L = c->L, M = c->M;
    u64 *d = malloc(sizeof(u64) * N);
    for (int i = 0; i < L; i++) {
        memcpy(d, c1 + (size_t)i * N, sizeof(u64) * N);
        ntt_inv(&c->t[i], d, N);
        for (int j = 0; j < M; j++) {
            u64 *Dij = D + ((size_t)i * M + j) * N;
            if (j == i) { memcpy(Dij, c1 + (size_t)i * N, sizeof(u64) * N); continue; }
            u64 q = c->t[j].q;
            for (int k = 0; k < N; k++) Dij[k] = d[k] % q;
            ntt_fwd(&c->t[j], Dij, N);
        }
    }
    free(d);
}

/* U[2][M][N] += KSraw(step, D) */
static int ks_accumulate(const octx *c, int step, const u64 *D, u64 *U)
{
    int N = c->N, L = c->L, M = c->M, n = N / 2;
    int s = ((step % n) + n) % n;
    const u64 *key = c->ksk[s];
    if (!key) return -2;
    u64 g = galois(s, N);
    u64 *perm = malloc(sizeof(u64) * N);
    for (int i = 0; i < L; i++)
        for (int j = 0; j < M; j++) {
            u64 q = c->t[j].q;
            automorph_ntt(D + ((size_t)i * M + j) * N, perm, N, g);
            for (int comp = 0; comp < 2; comp++) {
                const u64 *kk = key + (((size_t)i * 2 + comp) * M + j) * N;
                u64 *u = U + ((size_t)comp * M + j) * N;
                for (int k = 0; k < N; k++) u[k] = addmod(u[k], mulmod(perm[k], kk[k], q), q);
            }
        }
    free(perm);
    return 0;
}

/* out[L][N] NTT = ModDown(U[M][N]) (one component) */
static void moddown(const octx *c, const u64 *U, u64 *out)
{
    int N = c->N, L = c->L;
    const modtab *tP = &c->t[L];
    u64 P = tP->q, halfP = P >> 1;
    u64 *r = malloc(sizeof(u64) * N), *R = malloc(sizeof(u64) * N);
    memcpy(r, U + (size_t)L * N, sizeof(u64) * N);
    ntt_inv(tP, r, N);
    for (int j = 0; j < L; j++) {
        u64 q = c->t[j].q;
        for (int k = 0; k < N; k++) {
            u64 v = r[k];
            R[k] = v > halfP ? from_signed(-(i64)(P - v), q) : v % q;
        }
        ntt_fwd(&c->t[j], R, N);
        const u64 *Uj = U + (size_t)j * N;
        for (int k = 0; k < N; k++) out[(size_t)j * N + k] = mulmod(submod(Uj[k], R[k], q), c->Pinv[j], q);
    }
    free(r); free(R);
}

static void automorph_ct(const octx *c, const u64 *in, u64 *out, int nprimes_comp, u64 g)
{
    for (int k = 0; k < nprimes_comp; k++) automorph_ntt(in + (size_t)k * c->N, out + (size_t)k * c->N, c->N, g);
}

/* NTT-domain hoisted rotation of ctn (NTT [2][L][N]) by each step; D precomputed */
static int rotate_from_digits(const octx *c, const u64 *ctn, const u64 *D, int step, u64 *outn)
{
    int N = c->N, L = c->L, M = c->M, n = N / 2;
    int s = ((step % n) + n) % n;
    size_t W = 2 * (size_t)L * N;
    if (s == 0) { memcpy(outn, ctn, sizeof(u64) * W); return 0; }
    u64 *U = calloc(2 * (size_t)M * N, sizeof(u64));
    u64 *md = malloc(sizeof(u64) * (size_t)L * N);
    int rc = ks_accumulate(c, s, D, U);
    if (rc) { free(U); free(md); return rc; }
    u64 g = galois(s, N);
    automorph_ct(c, ctn, outn, L, g); /* c0 */
    moddown(c, U, md);
    for (int j = 0; j < L; j++) {
        u64 q = c->t[j].q;
        for (int k = 0; k < N; k++) outn[(size_t)j * N + k] = addmod(outn[(size_t)j * N + k], md[(size_t)j * N + k], q);
    }
    moddown(c, U + (size_t)M * N, outn + (size_t)L * N);
    free(U); free(md);
    return 0;
}

/* DecPerm once, HstPerm per step.  outs: [nsteps][2][L][N] canonical */
int o_rotate_hoisted(void *h, const u64 *ct, const int *steps, int nsteps, u64 *outs)
{
    octx *c = h;
    int N = c->N, L = c->L, M = c->M;
    size_t W = 2 * (size_t)L * N;
    u64 *ctn = malloc(sizeof(u64) * W), *tmp = malloc(sizeof(u64) * W);
    u64 *D = malloc(sizeof(u64) * (size_t)L * M * N);
    ct_to_ntt(c, ct, ctn);
    decompose(c, ctn + (size_t)L * N, D);
    int rc = 0;
    for (int t = 0; t < nsteps && !rc; t++) {
        rc = rotate_from_digits(c, ctn, D, steps[t], tmp);
        if (!rc) ct_from_ntt(c, tmp, outs + (size_t)t * W);
    }
    free(ctn); free(tmp); free(D);
    return rc;
}

/* ------------------------------------------------------------------ */
/* sum_k rot_{steps[k]}(X_k) with one lazy ModDown:                     */
/*   c0 = sum_k sigma_k(X_k.c0) + MD(sum_{k: step!=0} KSraw_0)           */
/*   c1 = sum_{k: step==0} X_k.c1 + MD(sum KSraw_1)                      */
/* X: NTT [cnt][2][L][N]; out NTT [2][L][N].                             */
static int rotate_sum_lazy(const octx *c, const u64 *X, const int *steps, int cnt, u64 *out)
{
    int N = c->N, L = c->L, M = c->M, n = N / 2;
    size_t W = 2 * (size_t)L * N, UW = 2 * (size_t)M * N;
    memset(out, 0, sizeof(u64) * W);
    u64 *U = calloc(UW, sizeof(u64));
    u64 *Ut = malloc(sizeof(u64) * UW * (size_t)cnt);
    int *rcs = calloc((size_t)cnt, sizeof(int));
    u64 *perm = malloc(sizeof(u64) * (size_t)L * N);
#pragma omp parallel for schedule(dynamic)
    for (int k = 0; k < cnt; k++) {
        int s = ((steps[k] % n) + n) % n;
        u64 *Uk = Ut + (size_t)k * UW;
        memset(Uk, 0, sizeof(u64) * UW);
        if (s == 0) continue;
        u64 *D = malloc(sizeof(u64) * (size_t)L * M * N);
        decompose(c, X + (size_t)k * W + (size_t)L * N, D);
        rcs[k] = ks_accumulate(c, s, D, Uk);
        free(D);
    }
    int rc = 0;
    for (int k = 0; k < cnt; k++) {
        if (rcs[k]) rc = rcs[k];
        int s = ((steps[k] % n) + n) % n;
        const u64 *Xk = X + (size_t)k * W;
        for (int j = 0; j < M; j++) {
            u64 q = c->t[j].q;
            for (int comp = 0; comp < 2; comp++) {
                u64 *u = U + ((size_t)comp * M + j) * N;
                const u64 *v = Ut + (size_t)k * UW + ((size_t)comp * M + j) * N;
                for (int i = 0; i < N; i++) u[i] = addmod(u[i], v[i], q);
            }
        }
        if (s == 0) {
            for (size_t i = 0; i < W; i++) {
                u64 q = c->t[(i / N) % L].q;
                out[i] = addmod(out[i], Xk[i], q);
            }
        } else {
            automorph_ct(c, Xk, perm, L, galois(s, N));
            for (size_t i = 0; i < (size_t)L * N; i++) {
                u64 q = c->t[i / N].q;
                out[i] = addmod(out[i], perm[i], q);
            }
        }
    }
    u64 *md = malloc(sizeof(u64) * (size_t)L * N);
    for (int comp = 0; comp < 2; comp++) {
        moddown(c, U + (size_t)comp * M * N, md);
        for (size_t i = 0; i < (size_t)L * N; i++) {
            u64 q = c->t[i / N].q;
            out[(size_t)comp * L * N + i] = addmod(out[(size_t)comp * L * N + i], md[i], q);
        }
    }
    free(U); free(Ut); free(rcs); free(perm); free(md);
    return rc;
}

int o_bsgs_baby(int T)
{
    int lg = 0;
    while ((1 << lg) < T) lg++;
    return 1 << ((lg + 1) / 2);
}

/*
 * GALA dot product (matvec.py:305-320), BSGS tree with lazy ModDown:
 *   u_t = x (.) pt_t
 *   inner_g = sum_{j<b} rot_j(u_{g b + j})          (one ModDown per g)
 *   out     = sum_{g<G} rot_{g b}(inner_g)           (one ModDown)
 *   masked  = out - Delta encode(r)                  (sharing.py:34-45)
 * Logical counts stay T ScMult, T-1 Perm, T-1 Add (+1 mask add).
 * pts: [T][N] slot values; r may be NULL (masked not produced).
 */
int o_mv_gala(void *h, const u64 *ct, const uint32_t *pts, int T, int baby,
              const uint32_t *r, u64 *out, u64 *masked)
{
    octx *c = h;
    int N = c->N, L = c->L;
    if (baby <= 0) baby = o_bsgs_baby(T);
    if (T % baby) return -4;
    int G = T / baby;
    size_t W = 2 * (size_t)L * N;
    u64 *ctn = malloc(sizeof(u64) * W);
    ct_to_ntt(c, ct, ctn);
    u64 *U = malloc(sizeof(u64) * W * (size_t)T);
#pragma omp parallel for schedule(static)
    for (int t = 0; t < T; t++) {
        u64 *pt = malloc(sizeof(u64) * (size_t)L * N);
        encode_pt_ntt(c, pts + (size_t)t * N, pt);
        scmult_ntt(c, ctn, pt, U + (size_t)t * W);
        free(pt);
    }
    u64 *inner = malloc(sizeof(u64) * W * (size_t)G);
    int *steps = malloc(sizeof(int) * (size_t)(baby > G ? baby : G));
    int rc = 0;
    for (int j = 0; j < baby; j++) steps[j] = j;
    for (int g = 0; g < G && !rc; g++)
        rc = rotate_sum_lazy(c, U + (size_t)g * baby * W, steps, baby, inner + (size_t)g * W);
    u64 *res = malloc(sizeof(u64) * W);
    for (int g = 0; g < G; g++) steps[g] = g * baby;
    if (!rc) rc = rotate_sum_lazy(c, inner, steps, G, res);
    if (!rc) {
        ct_from_ntt(c, res, out);
        if (r && masked) o_sub_plain(c, out, r, masked);
    }
    free(ctn); free(U); free(inner); free(steps); free(res);
    return rc;
}

/* plaintext operand in all L+1 primes (centred lift), NTT domain [M][N] */
static void encode_pt_ntt_qp(const octx *c, const uint32_t *slots, u64 *pt)
{
    int N = c->N;
    u64 *m = malloc(sizeof(u64) * N);
    o_encode_p((void *)c, slots, m);
    u64 half = c->p >> 1;
    for (int j = 0; j < c->M; j++) {
        u64 q = c->t[j].q;
        u64 *d = pt + (size_t)j * N;
        for (int i = 0; i < N; i++) d[i] = m[i] > half ? q - (c->p - m[i]) : m[i];
        ntt_fwd(&c->t[j], d, N);
    }
    free(m);
}

/*
 * GALA dot product, schedule v2 ("digits hoisted across the plaintext product").
 * Same logical tree as o_mv_gala (T ScMult, T-1 Perm, T-1 Add), but every
 * baby-step key switch reuses ONE decomposition of the input: for term t,
 *   d'_i = d_i * p_t   (integer polynomials; sum_i d'_i g_i = c1 p_t mod Q)
 * so  KSraw(sigma_j, x (.) p_t) = sum_i sigma_j(D_i (.) P_t) * ksk_j[i]  over QP,
 * with P_t the centred lift of p_t in every prime of QP.  Giant steps rotate
 * the group sums with their own decompositions; only the c1 of a group sum is
 * brought down to Q (it must be decomposed), its c0 is rotated in QP and summed,
 * and one final ModDown covers those sums and the giant-step key switches.
 */
int o_mv_gala2(void *h, const u64 *ct, const uint32_t *pts, int T, int baby, const uint32_t *r, u64 *out,
               u64 *masked)
{
    octx *c = h;
    int N = c->N, L = c->L, M = c->M, n = N / 2;
    if (baby <= 0) baby = o_bsgs_baby(T);
    if (T % baby) return -4;
    if (T > n) return -4;
    int G = T / baby;
    size_t W = 2 * (size_t)L * N, UW = 2 * (size_t)M * N, LN = (size_t)L * N;
    u64 *ctn = malloc(sizeof(u64) * W);
    ct_to_ntt(c, ct, ctn);
    u64 *D = malloc(sizeof(u64) * (size_t)L * M * N);
    decompose(c, ctn + LN, D);
    /* per group g: U_g (QP, both components), C0_g (Q: c0 rotation sums), C1_g (Q: step-0 c1 product) */
    u64 *Ug = calloc(UW * (size_t)G, sizeof(u64));
    u64 *C0g = calloc(LN * (size_t)G, sizeof(u64));
    u64 *C1g = calloc(LN * (size_t)G, sizeof(u64));
    int rc = 0;
    for (int j = 1; j < baby; j++) if (!c->ksk[j % n]) rc = -2;
    for (int g = 1; g < G; g++) if (!c->ksk[(g * baby) % n]) rc = -2;
    if (rc) { free(ctn); free(D); free(Ug); free(C0g); free(C1g); return rc; }
#pragma omp parallel for schedule(dynamic)
    for (int g = 0; g < G; g++) {
        u64 *U = Ug + (size_t)g * UW, *C0 = C0g + (size_t)g * LN, *C1 = C1g + (size_t)g * LN;
        u64 *P = malloc(sizeof(u64) * (size_t)M * N);
        u64 *X = malloc(sizeof(u64) * N), *Y = malloc(sizeof(u64) * N);
        for (int jj = 0; jj < baby; jj++) {
            int t = g * baby + jj;
            encode_pt_ntt_qp(c, pts + (size_t)t * N, P);
            if (jj == 0) {
                for (int j = 0; j < L; j++) {
                    u64 q = c->t[j].q;
                    for (int k = 0; k < N; k++) {
                        C0[(size_t)j * N + k] = addmod(C0[(size_t)j * N + k],
                                                       mulmod(ctn[(size_t)j * N + k], P[(size_t)j * N + k], q), q);
                        C1[(size_t)j * N + k] = mulmod(ctn[((size_t)L + j) * N + k], P[(size_t)j * N + k], q);
                    }
                }
                continue;
            }
            u64 gal = galois(jj, N);
            const u64 *key = c->ksk[jj % n];
            for (int i = 0; i < L; i++)
                for (int j = 0; j < M; j++) {
                    u64 q = c->t[j].q;
                    const u64 *Dij = D + ((size_t)i * M + j) * N;
                    for (int k = 0; k < N; k++) X[k] = mulmod(Dij[k], P[(size_t)j * N + k], q);
                    automorph_ntt(X, Y, N, gal);
                    for (int comp = 0; comp < 2; comp++) {
                        const u64 *kk = key + (((size_t)i * 2 + comp) * M + j) * N;
                        u64 *u = U + ((size_t)comp * M + j) * N;
                        for (int k = 0; k < N; k++) u[k] = addmod(u[k], mulmod(Y[k], kk[k], q), q);
                    }
                }
            for (int j = 0; j < L; j++) {
                u64 q = c->t[j].q;
                for (int k = 0; k < N; k++) X[k] = mulmod(ctn[(size_t)j * N + k], P[(size_t)j * N + k], q);
                automorph_ntt(X, Y, N, gal);
                for (int k = 0; k < N; k++) C0[(size_t)j * N + k] = addmod(C0[(size_t)j * N + k], Y[k], q);
            }
        }
        free(P); free(X); free(Y);
    }
    /* giant steps, c0 ModDown deferred: S.c0 = sum_g sigma_g(U_g.c0), S.c1 = U_0.c1 (QP);
     * Qadd.c0 = sum_g sigma_g(C0_g), Qadd.c1 = C1_0 (Q); group g >= 1: c1' = C1_g + ModDown(U_g.c1)
     * is key-switched for the rotation by g b into Uks (QP).  out = ModDown(S + Uks) + Qadd. */
    u64 *S = calloc(UW, sizeof(u64)), *Uks = calloc(UW, sizeof(u64)), *Qadd = calloc(W, sizeof(u64));
    u64 *perm = malloc(sizeof(u64) * N);
    for (int g = 0; g < G; g++) {
        const u64 *U = Ug + (size_t)g * UW;
        u64 ge = g ? galois((g * baby) % n, N) : 1;
        for (int j = 0; j < M; j++) {
            u64 q = c->t[j].q;
            if (g) automorph_ntt(U + (size_t)j * N, perm, N, ge);
            else memcpy(perm, U + (size_t)j * N, sizeof(u64) * N);
            for (int k = 0; k < N; k++) S[(size_t)j * N + k] = addmod(S[(size_t)j * N + k], perm[k], q);
        }
        for (int j = 0; j < L; j++) {
            u64 q = c->t[j].q;
            const u64 *C0 = C0g + (size_t)g * LN + (size_t)j * N;
            if (g) automorph_ntt(C0, perm, N, ge);
            else memcpy(perm, C0, sizeof(u64) * N);
            for (int k = 0; k < N; k++) Qadd[(size_t)j * N + k] = addmod(Qadd[(size_t)j * N + k], perm[k], q);
        }
    }
    memcpy(S + (size_t)M * N, Ug + (size_t)M * N, sizeof(u64) * (size_t)M * N);
    memcpy(Qadd + LN, C1g, sizeof(u64) * LN);
    int *rcs = calloc((size_t)G, sizeof(int));
    u64 *Ut = calloc(UW * (size_t)G, sizeof(u64));
#pragma omp parallel for schedule(dynamic)
    for (int g = 1; g < G; g++) {
        u64 *c1p = malloc(sizeof(u64) * LN), *Dg = malloc(sizeof(u64) * (size_t)L * M * N);
        moddown(c, Ug + (size_t)g * UW + (size_t)M * N, c1p);
        for (size_t i = 0; i < LN; i++) {
            u64 q = c->t[i / N].q;
            c1p[i] = addmod(c1p[i], C1g[(size_t)g * LN + i], q);
        }
        decompose(c, c1p, Dg);
        rcs[g] = ks_accumulate(c, g * baby, Dg, Ut + (size_t)g * UW);
        free(c1p); free(Dg);
    }
    for (int g = 1; g < G; g++) {
        if (rcs[g]) rc = rcs[g];
        for (int j = 0; j < M; j++) {
            u64 q = c->t[j].q;
            for (int comp = 0; comp < 2; comp++) {
                u64 *u = Uks + ((size_t)comp * M + j) * N;
                const u64 *v = Ut + (size_t)g * UW + ((size_t)comp * M + j) * N;
                for (int k = 0; k < N; k++) u[k] = addmod(u[k], v[k], q);
            }
        }
    }
    if (!rc) {
        u64 *resn = malloc(sizeof(u64) * W), *md = malloc(sizeof(u64) * LN);
        for (size_t i = 0; i < UW; i++) {
            u64 q = c->t[(i / N) % M].q;
            S[i] = addmod(S[i], Uks[i], q);
        }
        for (int comp = 0; comp < 2; comp++) {
            moddown(c, S + (size_t)comp * M * N, md);
            for (size_t i = 0; i < LN; i++) {
                u64 q = c->t[i / N].q;
                resn[(size_t)comp * LN + i] = addmod(md[i], Qadd[(size_t)comp * LN + i], q);
            }
        }
        ct_from_ntt(c, resn, out);
        if (r && masked) o_sub_plain(c, out, r, masked);
        free(resn); free(md);
    }
    free(ctn); free(D); free(Ug); free(C0g); free(C1g); free(S); free(Uks); free(Qadd); free(perm); free(rcs); free(Ut);
    return rc;
}

/*
 * Kernel-grouping convolution (conv.py:268-293), physical form:
 *   R[ib][tap] = HstPerm(DecPerm(x_ib), tap_steps[tap])   (tap step 0 -> x)
 *   acc[o][d]  = sum_ib sum_tap R[ib][tap] (.) pt[o][ib][d][tap]   (first-Add)
 *   out[o]     = sum_d rot_{d*band_step}(acc[o][d])  (one lazy ModDown)
 * cts: [n_ib][2][L][N]; pts: [n_obp][n_ib][c_n][k][N] slot values.
 */
int o_conv_kg(void *h, const u64 *cts, int n_ib, const uint32_t *pts, int n_obp,
              int c_n, int k, const int *tap_steps, int band_step, u64 *outs)
{
    octx *c = h;
    int N = c->N, L = c->L, M = c->M;
    size_t W = 2 * (size_t)L * N;
    u64 *R = malloc(sizeof(u64) * W * (size_t)n_ib * k);
    int rc = 0;
    int *rcs = calloc((size_t)n_ib, sizeof(int));
#pragma omp parallel for schedule(dynamic)
    for (int ib = 0; ib < n_ib; ib++) {
        u64 *ctn = malloc(sizeof(u64) * W);
        u64 *D = malloc(sizeof(u64) * (size_t)L * M * N);
        ct_to_ntt(c, cts + (size_t)ib * W, ctn);
        int need = 0;
        for (int t = 0; t < k; t++) need |= (tap_steps[t] % (N / 2)) != 0;
        if (need) decompose(c, ctn + (size_t)L * N, D);
        for (int t = 0; t < k && !rcs[ib]; t++)
            rcs[ib] = rotate_from_digits(c, ctn, D, tap_steps[t], R + ((size_t)ib * k + t) * W);
        free(ctn); free(D);
    }
    for (int ib = 0; ib < n_ib; ib++) if (rcs[ib]) rc = rcs[ib];
    free(rcs);
    if (rc) { free(R); return rc; }
    u64 *acc = calloc(W * (size_t)n_obp * c_n, sizeof(u64));
#pragma omp parallel for collapse(2) schedule(dynamic)
    for (int o = 0; o < n_obp; o++)
        for (int d = 0; d < c_n; d++) {
            u64 *A = acc + ((size_t)o * c_n + d) * W;
            u64 *pt = malloc(sizeof(u64) * (size_t)L * N);
            u64 *prod = malloc(sizeof(u64) * W);
            for (int ib = 0; ib < n_ib; ib++)
                for (int t = 0; t < k; t++) {
                    const uint32_t *sl = pts + ((((size_t)o * n_ib + ib) * c_n + d) * k + t) * N;
                    encode_pt_ntt(c, sl, pt);
                    scmult_ntt(c, R + ((size_t)ib * k + t) * W, pt, prod);
                    for (size_t i = 0; i < W; i++) {
                        u64 q = c->t[(i / N) % L].q;
                        A[i] = addmod(A[i], prod[i], q);
                    }
                }
            free(pt); free(prod);
        }
    int *steps = malloc(sizeof(int) * (size_t)c_n);
    for (int d = 0; d < c_n; d++) steps[d] = d * band_step;
    u64 *res = malloc(sizeof(u64) * W);
    for (int o = 0; o < n_obp && !rc; o++) {
        rc = rotate_sum_lazy(c, acc + (size_t)o * c_n * W, steps, c_n, res);
        if (!rc) ct_from_ntt(c, res, outs + (size_t)o * W);
    }
    free(R); free(acc); free(steps); free(res);
    return rc;
}

/*
 * Kernel-grouping convolution, schedule 2 (factored plaintexts; used for L >= 2 and int8 kernels).
 * Every KG plaintext is sum over bands beta of coef * M_{tap,beta}, with M_{tap,beta} the 0/1 mask of
 * band beta's valid pixels for the tap (conv.py:220-235).  So
 *   Y[ib][tap][beta] = R[ib][tap] (.) encode(M_{tap,beta})
 *   acc[o][d]        = sum_{ib,tap,beta} c(o,d,ib,tap,beta) * Y[ib][tap][beta]   (integer scalars, mod q)
 *   out[o]           = sum_d rot_{d B}(acc[o][d])                                (lazy ModDown, as o_conv_kg)
 * c = kern[ob c_n + (ch - d) mod c_n][ib c_n + ch][tap] (centred integers), ob = pair*o + row.
 * Bands: pair == 2 -> beta = row * c_n + ch (rows hold output blocks 2o, 2o+1); pair == 1 -> beta = ch
 * over both rows.  kern: int32 [c_o][c_i][k_h][k_w] centred.
 */
/*
 * Kernel grouping, schedule 2 ("factored plaintexts", GPU gala_conv_kg2).  Every KG plaintext
 * pt[ob][ib][d][tap] of o_conv_kg is a sum over bands beta of a 0/1 band mask Mask[tap][beta]
 * times one kernel coefficient, so the first-Add becomes
 *   acc[o][d] = sum_{ib, tap, beta} kern[(o, d), (ib, tap, beta)] * (Z[ib][tap] (.) Mask[tap][beta])
 * with small signed integer coefficients (the GPU evaluates it as an int8 GEMM over byte limbs).
 * The rotated inputs stay in the extended basis QP:  Z = KSraw(step, D) + P * sigma(c0)
 * (Z = P * X for tap step 0), masks are encoded in all L+1 primes, and one ModDown per acc[o][d]
 * replaces one per rotated input (ModDown(U + P V) = ModDown(U) + V exactly).  The second-Perm is
 * the lazy rotate-and-sum of o_conv_kg.  pair == 2: band beta = row * c_n + ch (output block
 * pair * o + row on hypercube row `row`); pair == 1: beta = ch over both rows.
 * band_only != 0 drops the tap-validity factor of the masks (the taps read the cyclic neighbours
 * inside each band): exact for every output pixel whose receptive field stays inside the zero
 * margin or halo of a frame embedding, which is how the GPU's post-mask form is used.
 * kern: centred int32 [c_o][c_i][k_h][k_w] (reference kernels, conv.py:220-235).
 */
int o_conv_kg2(void *h, const u64 *cts, int n_ib, const int32_t *kern, int c_o, int c_i, int k_h, int k_w,
               int u_w, int u_h, int pair, int band_only, u64 *outs)
{
    octx *c = h;
    int N = c->N, L = c->L, M = c->M, n = N / 2;
    size_t W = 2 * (size_t)L * N, WQ = 2 * (size_t)M * N, MN = (size_t)M * N;
    int B = u_w * u_h;
    if (B <= 0 || n % B || (pair != 1 && pair != 2)) return -4;
    int c_n = n / B, n_ob = c_o / c_n, n_obp = (n_ob + pair - 1) / pair, k = k_h * k_w;
    int nb = pair * c_n;
    u64 P = c->t[L].q;
    int *tap_steps = malloc(sizeof(int) * (size_t)k);
    for (int t = 0; t < k; t++) {
        int dh = t / k_w - k_h / 2, dw = t % k_w - k_w / 2;
        tap_steps[t] = (((dh * u_w + dw) % n) + n) % n;
    }
    /* 1. rotated inputs in QP: Z[ib][tap] [2][M][N] (DecPerm once per input, HstPerm per tap) */
    u64 *Z = calloc(WQ * (size_t)n_ib * k, sizeof(u64));
    int rc = 0;
    int *rcs = calloc((size_t)n_ib, sizeof(int));
#pragma omp parallel for schedule(dynamic)
    for (int ib = 0; ib < n_ib; ib++) {
        u64 *ctn = malloc(sizeof(u64) * W), *sc0 = malloc(sizeof(u64) * (size_t)L * N);
        u64 *D = malloc(sizeof(u64) * (size_t)L * M * N);
        ct_to_ntt(c, cts + (size_t)ib * W, ctn);
        decompose(c, ctn + (size_t)L * N, D);
        for (int t = 0; t < k && !rcs[ib]; t++) {
            u64 *z = Z + ((size_t)ib * k + t) * WQ;
            int s = tap_steps[t];
            if (s == 0) {
                for (int comp = 0; comp < 2; comp++)
                    for (int j = 0; j < L; j++) {
                        u64 q = c->t[j].q, Pq = P % q;
                        for (int i = 0; i < N; i++)
                            z[(comp * MN) + (size_t)j * N + i] = mulmod(ctn[((size_t)comp * L + j) * N + i], Pq, q);
                    }
                continue;
            }
            rcs[ib] = ks_accumulate(c, s, D, z);
            automorph_ct(c, ctn, sc0, L, galois(s, N));
            for (int j = 0; j < L; j++) {
                u64 q = c->t[j].q, Pq = P % q;
                for (int i = 0; i < N; i++)
                    z[(size_t)j * N + i] = addmod(z[(size_t)j * N + i], mulmod(sc0[(size_t)j * N + i], Pq, q), q);
            }
        }
        free(ctn); free(sc0); free(D);
    }
    for (int ib = 0; ib < n_ib; ib++) if (rcs[ib]) rc = rcs[ib];
    free(rcs);
    if (rc) { free(Z); free(tap_steps); return rc; }
    /* 2. band masks in all L+1 primes: Mk[tap][beta] NTT [M][N] */
    u64 *Mk = malloc(sizeof(u64) * MN * (size_t)k * nb);
#pragma omp parallel for collapse(2)
    for (int t = 0; t < k; t++)
        for (int beta = 0; beta < nb; beta++) {
            uint32_t *sl = malloc(sizeof(uint32_t) * N);
            int dh = t / k_w - k_h / 2, dw = t % k_w - k_w / 2;
            for (int s = 0; s < N; s++) {
                int row = s / n, cs = s % n, ch = cs / B, pos = cs % B, y = pos / u_w, x = pos % u_w;
                int band = pair == 2 ? row * c_n + ch : ch;
                int ok = band_only || (x + dw >= 0 && x + dw < u_w && y + dh >= 0 && y + dh < u_h);
                sl[s] = (uint32_t)(band == beta && ok);
            }
            encode_pt_ntt_qp(c, sl, Mk + ((size_t)t * nb + beta) * MN);
            free(sl);
        }
    /* 3. Y = Z (.) Mask and the integer-coefficient first-Add, in QP */
    u64 *Y = malloc(sizeof(u64) * WQ * (size_t)n_ib * k * nb);
#pragma omp parallel for collapse(3)
    for (int ib = 0; ib < n_ib; ib++)
        for (int t = 0; t < k; t++)
            for (int beta = 0; beta < nb; beta++) {
                const u64 *z = Z + ((size_t)ib * k + t) * WQ, *mk = Mk + ((size_t)t * nb + beta) * MN;
                u64 *y = Y + (((size_t)ib * k + t) * nb + beta) * WQ;
                for (size_t i2 = 0; i2 < WQ; i2++) y[i2] = mulmod(z[i2], mk[i2 % MN], c->t[(i2 / N) % M].q);
            }
    u64 *acc = malloc(sizeof(u64) * W * (size_t)n_obp * c_n);
#pragma omp parallel for collapse(2) schedule(dynamic)
    for (int o = 0; o < n_obp; o++)
        for (int d = 0; d < c_n; d++) {
            u64 *A = calloc(WQ, sizeof(u64));
            for (int ib = 0; ib < n_ib; ib++)
                for (int t = 0; t < k; t++)
                    for (int beta = 0; beta < nb; beta++) {
                        int row = pair == 2 ? beta / c_n : 0, ch = beta % c_n;
                        int ob = pair * o + row;
                        if (ob >= n_ob) continue;
                        int oo = ob * c_n + ((ch - d) % c_n + c_n) % c_n, ii = ib * c_n + ch;
                        int32_t cf = kern[(((size_t)oo * c_i + ii) * k_h + t / k_w) * k_w + t % k_w];
                        if (!cf) continue;
                        const u64 *Yv = Y + (((size_t)ib * k + t) * nb + beta) * WQ;
                        for (size_t i2 = 0; i2 < WQ; i2++) {
                            u64 q = c->t[(i2 / N) % M].q;
                            A[i2] = addmod(A[i2], mulmod(from_signed(cf, q), Yv[i2], q), q);
                        }
                    }
            /* one ModDown per accumulator */
            u64 *dst = acc + ((size_t)o * c_n + d) * W;
            moddown(c, A, dst);
            moddown(c, A + MN, dst + (size_t)L * N);
            free(A);
        }
    /* 4. second-Perm with one lazy ModDown per output */
    int *steps = malloc(sizeof(int) * (size_t)c_n);
    for (int d = 0; d < c_n; d++) steps[d] = d * B;
    u64 *res = malloc(sizeof(u64) * W);
    for (int o = 0; o < n_obp && !rc; o++) {
        rc = rotate_sum_lazy(c, acc + (size_t)o * c_n * W, steps, c_n, res);
        if (!rc) ct_from_ntt(c, res, outs + (size_t)o * W);
    }
    free(Z); free(Mk); free(acc); free(Y); free(steps); free(res); free(tap_steps);
    return rc;
}

/* test hooks: raw NTT on a single modulus (idx < 0: plaintext modulus) */
void o_ntt(void *h, int idx, u64 *a, int inverse)
{
    octx *c = h;
    const modtab *t = idx < 0 ? &c->tp : &c->t[idx];
    if (inverse) ntt_inv(t, a, c->N);
    else ntt_fwd(t, a, c->N);
}

int o_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
