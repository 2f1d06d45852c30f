/*
 * gala_b200.h -- C-ABI of the B200-native GALA HE linear-layer library.
 *
 * The reference (arxiv 2105.01827, package `gala`) has no native code: its
 * drop-in seam is the Python module `gala.backend` ("Swapping in a real
 * lattice backend means re-implementing the functions in this module",
 * pkg/src/gala/backend.py:12-16) plus the two scheme entry points on the hot
 * path, `mv_gala` (pkg/src/gala/matvec.py:305-320) and
 * `mimo_kernel_grouping` (pkg/src/gala/conv.py:268-293).  Each entry point
 * below names the reference function it replaces.  The Python package
 * paper_2105_01827_b200 binds these with ctypes.
 *
 * Conventions
 *  - Plain pointers and sizes only.  "dev" pointers are CUDA device memory,
 *    "host" pointers are host memory.  All device work is enqueued on the
 *    context's stream (gala_set_stream); calls return after enqueueing
 *    unless stated otherwise.
 *  - Ciphertext (device): uint64 [2][L][N], RNS limbs, NTT domain in the
 *    library's internal (bit-reversed) order.  Canonical words (coefficient
 *    domain, natural order, values in [0, q_j)) are produced by
 *    gala_ct_export / consumed by gala_ct_import.
 *  - Plaintext operand (device): uint64 [L][N], internal form (NTT,
 *    Montgomery-scaled).  Produced only by gala_encode_plain.
 *  - Slot vectors: uint32 [N]; slots [0, N/2) are hypercube row 0 and
 *    [N/2, N) row 1.  A rotation by `step` rotates both rows left by step
 *    (Galois element 3^step mod 2N), i.e. ring.py:86-91 on each row.
 *  - Return value: GALA_OK or a negative status; gala_last_error() has text.
 */
#ifndef GALA_B200_H
#define GALA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GALA_OK 0
#define GALA_ERR_PARAM (-1)   /* -> gala.errors.ParameterError */
#define GALA_ERR_DIM (-2)     /* -> gala.errors.DimensionError */
#define GALA_ERR_NOKEY (-3)   /* -> ParameterError: rotation key missing */
#define GALA_ERR_CUDA (-4)    /* -> gala.errors.GalaError */
#define GALA_ERR_STATE (-5)   /* -> GalaError: e.g. secret not set */

typedef struct gala_ctx gala_ctx;

const char *gala_last_error(void);
int gala_version(void);

/* Context: HEParams (backend.py:80-114) + the BFV instance derived from it.
 * primes: L ciphertext primes followed by the special prime (L+1 values);
 * psis: a primitive 2N-th root for each of them; psi_p: same for p. */
int gala_ctx_create(gala_ctx **out, int N, int L, const uint64_t *primes, const uint64_t *psis,
                    uint64_t p, uint64_t psi_p, int device);
void gala_ctx_destroy(gala_ctx *ctx);
int gala_set_stream(gala_ctx *ctx, void *cuda_stream);
int gala_sync(gala_ctx *ctx);

/* Keys (client side, from host-supplied randomness). */
int gala_set_secret(gala_ctx *ctx, const int8_t *s_host /* [N] ternary */);
/* a_host: [L][L+1][N] uniform coefficients; e_host: [L][N] signed errors */
int gala_gen_rotation_key(gala_ctx *ctx, int step, const uint64_t *a_host, const int64_t *e_host);
int gala_has_rotation_key(gala_ctx *ctx, int step);
size_t gala_key_bytes(gala_ctx *ctx);

/* encrypt (backend.py:228-234): a_dev [L][N] uniform coefficients, e_dev [N] */
int gala_encrypt(gala_ctx *ctx, const uint32_t *slots_dev, const uint64_t *a_dev, const int64_t *e_dev,
                 uint64_t *ct_dev);
/* decrypt (backend.py:237-243); slots_dev [N] */
int gala_decrypt(gala_ctx *ctx, const uint64_t *ct_dev, uint32_t *slots_dev);
/* Decrypt and measure the real noise: *noise_frac = max over coefficients of |p v / Q - m|, i.e. the
 * noise as a fraction of Delta (decryption is exact below 1/2).  The Python decrypt raises
 * NoiseOverflowError from 1/4 on -- past 1/2 the noise wraps and the slots are silently wrong, so the
 * check keeps two bits of margin (the reference's mock raises on its own noise recurrence). */
int gala_decrypt_noise(gala_ctx *ctx, const uint64_t *ct_dev, uint32_t *slots_dev, double *noise_frac);
/* batch encode of B slot vectors into plaintext operands [B][L][N] */
int gala_encode_plain(gala_ctx *ctx, const uint32_t *slots_dev, int B, uint64_t *pt_dev);

/* op seam (backend.py:246-311) */
int gala_add(gala_ctx *ctx, const uint64_t *a_dev, const uint64_t *b_dev, uint64_t *out_dev);   /* he_add */
int gala_scmult(gala_ctx *ctx, const uint64_t *ct_dev, const uint64_t *pt_dev, uint64_t *out_dev); /* he_scmult */
int gala_sub_plain(gala_ctx *ctx, const uint64_t *ct_dev, const uint32_t *r_slots_dev,
                   uint64_t *out_dev);                                                            /* subtract_plain */
int gala_rotate(gala_ctx *ctx, const uint64_t *ct_dev, int step, uint64_t *out_dev);             /* he_perm */
/* he_decperm: digits [L][L+1][N] */
int gala_decompose(gala_ctx *ctx, const uint64_t *ct_dev, uint64_t *digits_dev);
size_t gala_digits_words(gala_ctx *ctx);
/* he_hstperm: ct_dev is the group's source (its c0 is rotated directly) */
int gala_rotate_hoisted(gala_ctx *ctx, const uint64_t *ct_dev, const uint64_t *digits_dev, int step,
                        uint64_t *out_dev);

/* Fused GALA dot product (mv_gala + gen_additive_share, matvec.py:305-320,
 * sharing.py:34-45): out = sum_t rot_t(ct (.) pts[t]) over a BSGS tree
 * (baby <= 0: automatic), masked = out - Delta encode(r).  r_slots_dev
 * and masked_dev may be NULL. */
int gala_mv_gala(gala_ctx *ctx, const uint64_t *ct_dev, const uint64_t *pts_dev, int T, int baby,
                 const uint32_t *r_slots_dev, uint64_t *out_dev, uint64_t *masked_dev);
/* Batched form: B independent inputs cts_dev [B][2][L][N] against the same
 * plaintexts; r_slots_dev [B][N]; outs/masked [B][2][L][N].  All inputs share
 * every launch (grids scale with B). */
int gala_mv_gala_batch(gala_ctx *ctx, const uint64_t *cts_dev, int B, const uint64_t *pts_dev, int T, int baby,
                       const uint32_t *r_slots_dev, uint64_t *outs_dev, uint64_t *masked_dev);
int gala_bsgs_baby(int T);

/* GALA schedule 2 (the production schedule when the noise budget allows; see
 * DESIGN.md): one gadget decomposition of each input's c1, digits hoisted
 * across the plaintext product (sum_i (d_i p_t) g_i = c1 p_t mod Q), so the
 * T-1 baby-step key switches need no NTTs.  The giant steps bring only the c1
 * of a group sum down to Q; the c0 parts are rotated in QP and share the final
 * ModDown.  Plaintexts come from gala_encode_gala_weights: slots [T][N] -> pts2
 * [T][L+1][N] (every prime of QP, pre-permuted by sigma_{t mod baby}).
 * T <= N/2.  Matches oracle o_mv_gala2. */
int gala_encode_gala_weights(gala_ctx *ctx, const uint32_t *slots_dev, int T, int baby, uint64_t *pts2_dev);
int gala_mv_gala2_batch(gala_ctx *ctx, const uint64_t *cts_dev, int B, const uint64_t *pts2_dev, int T, int baby,
                        const uint32_t *r_slots_dev, uint64_t *outs_dev, uint64_t *masked_dev);
/* host-buffer form of gala_mv_gala2_batch (canonical words in/out, blocks until done) */
int gala_mv_gala2_batch_host(gala_ctx *ctx, const uint64_t *cts_host, int B, const uint64_t *pts2_dev, int T,
                             int baby, const uint32_t *r_slots_host, uint64_t *masked_host);
/* Same with host buffers (canonical words in/out), copies on the context
 * stream; blocks until the result is in host memory. */
int gala_mv_gala_host(gala_ctx *ctx, const uint64_t *ct_host, const uint64_t *pts_dev, int T, int baby,
                      const uint32_t *r_slots_host, uint64_t *masked_host);
/* Batched host-buffer form: cts_host [B][2][L][N] canonical words, r [B][N]. */
int gala_mv_gala_batch_host(gala_ctx *ctx, const uint64_t *cts_host, int B, const uint64_t *pts_dev, int T,
                            int baby, const uint32_t *r_slots_host, uint64_t *masked_host);

/* GALA schedule 2 with the baby-step sums on the int8 tensor cores (tcgen05): per QP position the
 * weights' byte-convolution (Toeplitz) expansion is the MMA B operand (built in shared memory from
 * the position-major weights gala_fc_tc_weights writes to wcan_dev, gala_fc_tc_weight_bytes bytes =
 * 4 KB per position) and E_jj, packed per position, the A operand.  Same words as gala_mv_gala2_batch (exact modular arithmetic).
 * Used for T/baby <= 8, baby <= 64 and 16 <= B <= 32 -- or, for T >= 128, any B whose 32-input
 * tiles all hold >= 16 inputs (one E / MMA kernel pair per tile, everything else batched over B);
 * otherwise the CUDA-core path runs. */
/* Multi-GPU split of one schedule-2 layer across its giant groups (
 * reference: "independent output blocks may be computed in parallel with per-block
 * meters merged", backend.py:134-139 CostMeter.merge).  Each rank runs gala_mv_gala2_partial on its
 * group range [g_lo, g_hi) (every rank the same inputs and weights), returning per input the QP sum
 * before the final ModDown, qp_sum [B][2][L+1][N], and the Q addend q_add [B][2][L][N] (wcan may be
 * null: CUDA-core baby-step sums).  The element-wise u64 sums of all ranks' buffers (an NCCL
 * reduce: every word < q_j, at most 8 ranks, so < 2^63 and exact) go to gala_mv_gala2_finish on
 * the root, which reduces them mod q_j, applies the final ModDown, adds q_add and masks: the same
 * words as gala_mv_gala2_batch(_tc) on one GPU. */
int gala_mv_gala2_partial(gala_ctx *ctx, const uint64_t *cts_dev, int B, const uint64_t *pts2_dev,
                          const uint8_t *wcan_dev, int T, int baby, int g_lo, int g_hi, uint64_t *qp_sum_dev,
                          uint64_t *q_add_dev);
int gala_mv_gala2_finish(gala_ctx *ctx, uint64_t *qp_sum_dev, uint64_t *q_add_dev, int B, const uint32_t *r_dev,
                         uint64_t *outs_dev, uint64_t *masked_dev);
size_t gala_fc_tc_weight_bytes(gala_ctx *ctx);
int gala_fc_tc_weights(gala_ctx *ctx, const uint64_t *pts2_dev, int T, int baby, uint8_t *wcan_dev);
int gala_mv_gala2_batch_tc(gala_ctx *ctx, const uint64_t *cts_dev, int B, const uint64_t *pts2_dev,
                           const uint8_t *wcan_dev, int T, int baby, const uint32_t *r_slots_dev,
                           uint64_t *outs_dev, uint64_t *masked_dev);
int gala_mv_gala2_batch_tc_host(gala_ctx *ctx, const uint64_t *cts_host, int B, const uint64_t *pts2_dev,
                                const uint8_t *wcan_dev, int T, int baby, const uint32_t *r_slots_host,
                                uint64_t *masked_host);

/* Streamed form for serving: S consecutive batches of B inputs from (pinned) host memory, each
 * batch through the fused layer as gala_mv_gala2_batch_tc_host (wcan_dev may be NULL: CUDA-core
 * schedule 2), with the host<->device copies overlapped with the layers -- batch s + 1 is copied in
 * and batch s - 1 copied out while batch s computes.  Returns when all S batches' masked words are in
 * masked_host.  cts_host [S][B][2][L][N], r_slots_host [S][B][N], masked_host [S][B][2][L][N];
 * same words as S separate host calls. */
int gala_mv_gala2_stream_host(gala_ctx *ctx, const uint64_t *cts_host, int S, int B, const uint64_t *pts2_dev,
                              const uint8_t *wcan_dev, int T, int baby, const uint32_t *r_slots_host,
                              uint64_t *masked_host);

/* Batched hoisted rotations (the raw key-switch throughput probe; he_decperm + he_hstperm,
 * backend.py:279-294, for many inputs at once): cts_dev [B][2][L][N], steps_host [S] (non-zero),
 * outs_dev [B][S][2][L][N]; each output equals gala_rotate(input, step). */
int gala_rotate_batch(gala_ctx *ctx, const uint64_t *cts_dev, int B, const int *steps_host, int S, uint64_t *outs_dev);

/* Fused kernel-grouping convolution (mimo_kernel_grouping, conv.py:268-293):
 * cts_dev [n_ib][2][L][N]; pts_dev [n_obp][n_ib][c_n][k][L][N];
 * tap_steps_host [k] (rotation per tap, conv.py:84-91); out [n_obp][2][L][N] */
int gala_conv_kg(gala_ctx *ctx, const uint64_t *cts_dev, int n_ib, const uint64_t *pts_dev, int n_obp,
                 int c_n, int k, const int *tap_steps_host, int band_step, uint64_t *outs_dev);

/* Batch of B images sharing one layer's weights (same words as B gala_conv_kg calls):
 * cts_dev [B][n_ib][2][L][N] -> outs_dev [B][n_obp][2][L][N].  Every stage (input rotations,
 * first-Add, second-Perm) runs once for the batch; the first-Add loads each plaintext word once
 * per 4 images. */
int gala_conv_kg_batch(gala_ctx *ctx, const uint64_t *cts_dev, int B, int n_ib, const uint64_t *pts_dev, int n_obp,
                       int c_n, int k, const int *tap_steps_host, int band_step, uint64_t *outs_dev);

/* Schedule-1 first-Add on the int8 tensor cores: per Q position one byte-convolution MMA of the
 * plaintext bytes (A, position-major ptcan_dev written once by gala_kg1_tc_weights from the
 * gala_kg_encode_weights plaintexts; gala_kg1_tc_bytes bytes, 0 if the shape is unsupported:
 * n_obp c_n <= 512 rows, n_ib k <= 1024 words) with the rotated inputs' byte-shift expansion (B).
 * Same words as gala_conv_kg. */
size_t gala_kg1_tc_bytes(gala_ctx *ctx, int n_ib, int n_obp, int c_n, int k);
int gala_kg1_tc_weights(gala_ctx *ctx, const uint64_t *pts_dev, int n_obp, int n_ib, int c_n, int k, uint64_t *ptcan_dev);
int gala_conv_kg_tc(gala_ctx *ctx, const uint64_t *cts_dev, int n_ib, const uint64_t *ptcan_dev, int n_obp, int c_n, int k,
                    const int *tap_steps_host, int band_step, uint64_t *outs_dev);

/* On-GPU kernel-grouping weight encoding (coef_vectors, conv.py:220-235, in the physical
 * two-row form): kernels_dev int32 [c_o][c_i][k_h][k_w] (values mod p) -> pts_dev
 * [n_obp][n_ib][c_n][k_h k_w][L][N] ready for gala_conv_kg.  pair = 2 puts output blocks
 * 2o and 2o+1 on hypercube rows 0 and 1; pair = 1 replicates. */
int gala_kg_encode_weights(gala_ctx *ctx, const int32_t *kernels_dev, int c_o, int c_i, int k_h, int k_w, int u_w,
                           int u_h, int pair, uint64_t *pts_dev);

/* Kernel grouping, schedule 2 (factored plaintexts; same outputs as gala_conv_kg up to the
 * exact integer evaluation order -- oracle o_conv_kg2).  The KG plaintexts of
 * coef_vectors (conv.py:220-235) factor into 0/1 band masks times one kernel coefficient each.
 * The rotated inputs stay in the extended basis QP (no ModDown per rotation); one ModDown per
 * accumulator.  gala_kg2_encode_masks: masks_dev [k_h k_w][pair c_n][L+1][N][2] (NTT, Shoup pairs
 * (w, floor(w 2^64 / q))).
 * gala_conv_kg2: coef_dev int8 [Mr][Kp] (Mr = n_obp c_n rows (o, d); K = (ib, tap, beta)
 * columns, zero-padded to Kp % 16 == 0; entry = centred kernel coefficient
 * kern[pair o + row][ib c_n + ch][tap] of band beta = row c_n + ch at rotation offset d),
 * rowsum_dev int32 [Mr] = row sums of coef; outs_dev [n_obp][2][L][N]. */
int gala_kg2_encode_masks(gala_ctx *ctx, int k_h, int k_w, int u_w, int u_h, int pair, int band_only,
                          uint64_t *masks_dev);
int gala_conv_kg2(gala_ctx *ctx, const uint64_t *cts_dev, int n_ib, const uint64_t *masks_dev, int k, int nb,
                  const int8_t *coef_dev, const int32_t *rowsum_dev, int Mr, int Kp, const int *tap_steps_host,
                  int band_step, int c_n, uint64_t *outs_dev);
/* Post-mask form for frame-embedded inputs (band_only masks [pair c_n][L+1][N][2], no tap
 * factor: exact on every output pixel whose receptive field stays inside the frame's zero margin
 * or halo).  The masks leave the K columns: acc[m] = sum_beta Mask_beta (.) (A_(m, beta) . Z), so the
 * GEMM runs on the bytes of the rotated inputs Z (K = (ib, tap)) with rows (m, beta):
 * coef_dev int8 [Mr nb][Kp], rowsum_dev int32 [Mr nb]. */
int gala_conv_kg2_post(gala_ctx *ctx, const uint64_t *cts_dev, int n_ib, const uint64_t *masks_dev, int k, int nb,
                       const int8_t *coef_dev, const int32_t *rowsum_dev, int Mr, int Kp, const int *tap_steps_host,
                       int band_step, int c_n, uint64_t *outs_dev);

/* The same for nbatch independent images sharing the weights (e.g. a layer's halo tiles):
 * cts_dev [nbatch][n_ib][2][L][N] -> outs_dev [nbatch][Mr / c_n][2][L][N]; one pass of launches. */
int gala_conv_kg2_post_batch(gala_ctx *ctx, const uint64_t *cts_dev, int nbatch, int n_ib, const uint64_t *masks_dev,
                             int k, int nb, const int8_t *coef_dev, const int32_t *rowsum_dev, int Mr, int Kp,
                             const int *tap_steps_host, int band_step, int c_n, uint64_t *outs_dev);

/* canonical word import/export of `count` ciphertexts */
int gala_ct_export(gala_ctx *ctx, const uint64_t *ct_dev, uint64_t *coef_dev, int count);
int gala_ct_import(gala_ctx *ctx, const uint64_t *coef_dev, uint64_t *ct_dev, int count);
/* canonical plaintext-operand words (coefficients of the centred lift) */
int gala_pt_export(gala_ctx *ctx, const uint64_t *pt_dev, uint64_t *coef_dev, int count);

/* Tensor-core FC policy: the smallest tree (T terms) that runs the baby-step sums on the tensor cores
 * (default 128: a key-folded tile's cost per QP position does not shrink with T; smaller trees use the
 * CUDA cores).  Words are identical either way; parity tests lower it to exercise the tiles on small
 * rings.  (No reference counterpart: a scheduling knob of this backend.) */
int gala_set_fc_tc_min_terms(gala_ctx *ctx, int min_terms);

/* kernel launches issued by this process so far (for bench accounting) */
uint64_t gala_launch_count(void);

/* Tracing: per-kernel CUDA-event timing of every launch while enabled.
 * gala_profile_json synchronises, writes {"kernel": [launches, total_ms], ...}
 * and clears the records. */
int gala_profile_enable(gala_ctx *ctx, int on);
int gala_profile_json(gala_ctx *ctx, char *buf, size_t cap);

/* Throughput probe of the library's 60-bit Shoup modmul (modmul/s); the
 * integer-roofline denominator used by bench.py. */
int gala_bench_modmul(gala_ctx *ctx, int blocks, int iters, double *modmul_per_s);

#ifdef __cplusplus
}
#endif
#endif
