/*
 * lf_b200.h — C ABI of the B200-native CKKS core (libcerium_b200.so).
 *
 * This is the drop-in boundary under the reference's Python operator API
 * (`limbforge.ckks`, /root/reference/pkg/src/limbforge/ckks.py:59-225, re-exported at
 * __init__.py:10-34).  The Python host layer `paper_2512_11269_b200` mirrors that API
 * function for function and calls the entry points below through ctypes; a foreign host
 * (cgo, JNI, N-API) would bind the same symbols.
 *
 * Conventions
 *  - Every function returns 0 on success, non-zero on failure; lf_last_error() describes
 *    the last failure of the calling thread.
 *  - Residues are uint32 (primes < 2^28, reference params.py:14-16), stored limb-major:
 *    a polynomial over n basis primes is n contiguous rows of N words.
 *  - All data pointers are DEVICE pointers owned by the caller; `stream` is a
 *    cudaStream_t passed as void*.  Calls are asynchronous on that stream, never
 *    synchronise the host, and never allocate (workspace is passed in), except
 *    lf_ctx_create / lf_ctx_destroy.
 *  - Metadata arrays (prime indices, scalars) are HOST arrays; `prime_idx[r]` indexes the
 *    context's prime list (main primes 0..L, then special primes L+1..L+alpha).
 *  - Canonical residues in, canonical residues out; `out` may alias inputs unless noted.
 */
#ifndef LF_B200_H
#define LF_B200_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct LfCtx lf_ctx;

#define LF_ABI_VERSION 1

/* element-wise op codes (reference poly.py:85-117) */
#define LF_OP_ADD 0            /* a + b                 row_add      poly.py:85   */
#define LF_OP_SUB 1            /* a - b                 row_sub      poly.py:89   */
#define LF_OP_MUL 2            /* a * b                 row_mul      poly.py:94   */
#define LF_OP_NEG 3            /* -a                    row_neg      poly.py:104  */
#define LF_OP_SCALAR_MUL 4     /* a * s_r               row_scalar_mul poly.py:108 */
#define LF_OP_MULACC 5         /* c + a * b             row_mulacc   poly.py:98   */
#define LF_OP_MODSTEP 6        /* (a - b) * s_r         row_modstep  poly.py:112  */
#define LF_OP_MUL_SCALAR_ADD 7 /* a * s_r + b           (fused helper)            */
#define LF_OP_ADD_SCALAR 8     /* a + s_r               (constant add, bootstrap)  */

int lf_abi_version(void);
const char* lf_last_error(void);

/* Base-conversion engine of every fused pipeline (no reference counterpart: an execution
 * choice, results are bit-identical): 1 = tcgen05 kind::i8 tensor cores with byte-split
 * weights (default; env LF_BC_TC=0 starts with 0), 0 = IMAD.WIDE kernel.  Process-wide. */
int lf_set_bconv_engine(int engine);
int lf_get_bconv_engine(void);

/* Context: per-prime constants and twiddle tables for ring dimension N = 2^logN.
 * psis[i] is the primitive 2N-th root used by the reference (modmath.py:61-68: smallest
 * generator g, psi = g^((q-1)/2N)); tables follow ntt.py:22-67.  Replaces the reference's
 * ntt_tables() cache (ntt.py:44-67). */
int lf_ctx_create(int logN, int nprimes, const uint32_t* primes, const uint32_t* psis,
                  lf_ctx** out);
int lf_ctx_destroy(lf_ctx* ctx);

/* Batched negacyclic NTT, in place.  Replaces ntt_forward / ntt_inverse (ntt.py:70-105)
 * and poly_ntt / poly_intt (poly.py:212-225).  Output of lf_ntt_fwd is in the reference's
 * bit-reversed evaluation order. */
int lf_ntt_fwd(const lf_ctx* ctx, uint32_t* rows, int nrows, const int32_t* prime_idx,
               void* stream);
int lf_ntt_inv(const lf_ctx* ctx, uint32_t* rows, int nrows, const int32_t* prime_idx,
               void* stream);

/* Element-wise row primitives (poly.py:85-117, 183-209).  b, c may be NULL when the op does
 * not read them; scalars (host, one per row, reduced mod the row's prime) may be NULL. */
int lf_ewise(const lf_ctx* ctx, int op, uint32_t* out, const uint32_t* a, const uint32_t* b,
             const uint32_t* c, int nrows, const int32_t* prime_idx, const uint32_t* scalars,
             void* stream);

/* Evaluation-domain automorphism X -> X^g on nrows rows: out[i] = in[perm_g(i)]
 * (ntt.py:108-126, poly.py:120-121, 228-231).  g odd.  out must not alias in. */
int lf_automorph(const lf_ctx* ctx, uint32_t* out, const uint32_t* in, uint32_t g, int nrows,
                 void* stream);

/* Exact base conversion of coefficient-domain rows (poly.py:150-178): src holds k rows,
 * out receives m rows.  `table` is a device blob laid out as described in DESIGN.md
 * ("BConv table") and built by the host (paper_2512_11269_b200/plan.py). */
int lf_bconv(const lf_ctx* ctx, uint32_t* out, const uint32_t* src, const uint32_t* table,
             int k, int m, int W, void* stream);

/* ---- fused hybrid keyswitch pipeline ---------------------------------------------------
 * lf_ctx_enable_keyswitch builds, once, every constant of the keyswitch / rescale path for a
 * context whose first n_main primes are the main basis q_0..q_L and the rest the special
 * basis (reference params.py:117-131), with d round-robin digits (params.py:23-41).
 *
 * Layouts (uint32 words, rows of N):
 *   x            level+1 rows                       (one polynomial, eval domain)
 *   ciphertext   2 x (level+1) rows: b rows then a rows      (ckks.py:40-50)
 *   evk          d x 2 x (L+1+alpha) rows: digit j, (b, a), extended-basis row (keys.py:40-49)
 *   out          2 x (level+1) rows (ks_b then ks_a, or b' then a')
 * Batched calls process `batch` independent instances; *_bstride are the word strides
 * between instances (0 = shared, e.g. one relinearisation key for the whole batch).
 * workspace: lf_ks_workspace_bytes(ctx, level, batch) bytes of device memory. */
int lf_ctx_enable_keyswitch(lf_ctx* ctx, int n_main, int d);
size_t lf_ks_workspace_bytes(const lf_ctx* ctx, int level, int batch);

/* keyswitch(x, evk) -> (ks_b, ks_a) over the main ids of x's level.
 * Replaces ckks.keyswitch (ckks.py:134-140) = keyswitch_decompose (ckks.py:95-117) +
 * keyswitch_inner_product (ckks.py:120-131) + mod_down x2 (poly.py:251-281). */
int lf_keyswitch(const lf_ctx* ctx, int level, const uint32_t* x, size_t x_bstride,
                 const uint32_t* evk, size_t evk_bstride, uint32_t* out, size_t out_bstride,
                 int batch, void* workspace, void* stream);

/* Measurement helper: lf_keyswitch with CUDA events recorded on `stream` around each of the
 * five fused kernels; synchronises on the last event and writes their durations (ms) to
 * stage_ms[0..4] = {modup_in, modup_bconv, ks_inner, moddown_bconv, moddown_out}. */
int lf_keyswitch_profiled(const lf_ctx* ctx, int level, const uint32_t* x, size_t x_bstride,
                          const uint32_t* evk, size_t evk_bstride, uint32_t* out,
                          size_t out_bstride, int batch, void* workspace, void* stream,
                          float* stage_ms);

/* hom_mul (ckks.py:182-194): tensor product + relinearisation, no rescale. */
int lf_hom_mul(const lf_ctx* ctx, int level, const uint32_t* ct1, const uint32_t* ct2,
               size_t ct_bstride, const uint32_t* rlk, uint32_t* out, size_t out_bstride,
               int batch, void* workspace, void* stream);

/* hom_mul followed by ndrop in {1, 2} rescales (ckks.py:182-194, then ckks.py:220-225 ndrop
 * times), bit for bit, with the rescale folded into the relinearisation's ModDown: one exact
 * floor division by P q_level [q_level-1] instead of a division by P and a second pass.
 * out = 2 x (level + 1 - ndrop) rows; workspace as lf_keyswitch. */
int lf_hom_mul_rescale(const lf_ctx* ctx, int level, int ndrop, const uint32_t* ct1,
                       const uint32_t* ct2, size_t ct_bstride, const uint32_t* rlk, uint32_t* out,
                       size_t out_bstride, int batch, void* workspace, void* stream);

/* lf_hom_mul_rescale over ciphertexts whose polynomials are ct*_pitch >= level + 1 rows apart
 * (the a rows of instance i of ct1 start at ct1 + i * ct1_bstride + ct1_pitch * N; ct2 has its
 * own stride and pitch): level-dropped row-prefix views of higher-level ciphertext blocks are
 * used in place, without a copy. */
int lf_hom_mul_rescale_p(const lf_ctx* ctx, int level, int ndrop, const uint32_t* ct1,
                         size_t ct1_bstride, int ct1_pitch, const uint32_t* ct2, size_t ct2_bstride,
                         int ct2_pitch, const uint32_t* rlk, uint32_t* out, size_t out_bstride,
                         int batch, void* workspace, void* stream);

/* lf_hom_mul_rescale over a LIST of independent operand pairs at one level (instance b: ct1s[b]
 * with pitch1[b] rows per polynomial, ct2s[b] with pitch2[b]), as one batch: the independent
 * products of a polynomial evaluation's dependency wave run in one pipeline without gathering
 * their operands.  add_b (NULL: none): an integer K_b added to every b residue of product b,
 * i.e. ckks add_const (ckks.py:152-161 with an encoded constant) folded into the epilogue.
 * out = batch x 2 x (level + 1 - ndrop) rows, instance stride out_bstride. */
int lf_hom_mul_rescale_list(const lf_ctx* ctx, int level, int ndrop, const uint32_t* const* ct1s,
                            const int* pitch1, const uint32_t* const* ct2s, const int* pitch2,
                            const int64_t* add_b, const uint32_t* rlk, uint32_t* out,
                            size_t out_bstride, int batch, void* workspace, void* stream);

/* Galois automorphism g with keyswitch (hom_rotate, ckks.py:197-217: decompose, permute the
 * pieces, inner product, mod_down; b' = sigma_g(b) + ks_b).  g = 5^steps mod 2N for a
 * rotation, 2N-1 for conjugation. */
int lf_rotate(const lf_ctx* ctx, int level, const uint32_t* ct, size_t ct_bstride, uint32_t g,
              const uint32_t* key, size_t key_bstride, uint32_t* out, size_t out_bstride,
              int batch, void* workspace, void* stream);

/* Hoisted rotations (the reference's hoisting semantics, ckks.py:1-7, 197-203 and
 * polyir.py:435-469): ONE ModUp of ct.a shared by n_rot Galois automorphisms gs[r] with keys
 * keys[r] (host array of device pointers).  out: n_rot ciphertexts, out_bstride words apart.
 * Bit-identical to n_rot separate lf_rotate calls. */
size_t lf_rotate_hoisted_workspace_bytes(const lf_ctx* ctx, int level, int n_rot);
int lf_rotate_hoisted(const lf_ctx* ctx, int level, const uint32_t* ct, int n_rot,
                      const uint32_t* gs, const uint32_t* const* keys, uint32_t* out,
                      size_t out_bstride, void* workspace, void* stream);

/* n independent rotations, each with its own ciphertext (ct_bstride words apart), Galois
 * element gs[r] and key keys[r] (host array of device pointers): n separate lf_rotate calls in
 * one pipeline (the giant steps of a BSGS linear transform).  Workspace:
 * lf_ks_workspace_bytes(ctx, level, min(n, 64)). */
int lf_rotate_batch(const lf_ctx* ctx, int level, const uint32_t* cts, size_t ct_bstride, int n,
                    const uint32_t* gs, const uint32_t* const* keys, uint32_t* out,
                    size_t out_bstride, void* workspace, void* stream);

/* Permuted-key forms of lf_rotate_hoisted_ext and lf_rotate_batch, bit-identical results.
 * keys[r] holds the rotation key for gs[r] with every row permuted by the inverse
 * automorphism: lf_automorph(ctx, pk, key, gs[r]^-1 mod 2N, d * 2 * (L+1+alpha), s).  The
 * inner product then runs on unpermuted lines (sum_j piece_j * K_j o sigma^-1) and applies
 * sigma_g once to the two accumulators instead of to every digit's piece. */
int lf_rotate_hoisted_ext_pk(const lf_ctx* ctx, int level, const uint32_t* ct, int n_rot,
                             const uint32_t* gs, const uint32_t* const* keys, uint32_t* out_ext,
                             size_t out_bstride, void* workspace, void* stream);
int lf_rotate_batch_pk(const lf_ctx* ctx, int level, const uint32_t* cts, size_t ct_bstride, int n,
                       const uint32_t* gs, const uint32_t* const* keys, uint32_t* out,
                       size_t out_bstride, void* workspace, void* stream);

/* One BSGS linear-transform inner sum over the extended basis (hoisted ModDown):
 *   out[k] = P ct * pts[k][0] + sum_r (P sigma_r(ct.b) + <pieces, K_r>, <pieces, K_r>)_sigma * pts[k][1+r]
 * i.e. lf_rotate_hoisted_ext_pk of the n_rot rotations (gs, permuted keys) followed by
 * lf_ptmac_rows for each of the n_giant giant steps, without materialising the rotated
 * ciphertexts.  pts: HOST array [n_giant][n_rot + 1] of device pointers to extended-basis
 * plaintexts (level+1+alpha rows, eval domain); NULL where a giant step has no diagonal.
 * out: n_giant x 2 x (level+1+alpha) rows.  Limits: n_rot <= 32, n_giant <= 4.
 * Workspace: lf_rotate_hoisted_workspace_bytes(ctx, level, 1). */
int lf_bsgs_ext(const lf_ctx* ctx, int level, const uint32_t* ct, int n_rot, const uint32_t* gs,
                const uint32_t* const* keys, int n_giant, const uint32_t* const* pts, uint32_t* out,
                void* workspace, void* stream);

/* ---- kernel-plan interpreter (the reference's KernelRunner boundary, codegen.py:346-443) ----
 * One step of a compiled kernel plan: op i of every lane, one launch.  ops is a DEVICE array of
 * nops lf_plan_op records; each reads its sources at coefficient n, writes the canonical
 * result to dst (a register row) and, when store != NULL, to the operand row (the lane op's
 * store_slot).  Opcodes follow limbir.py:46-56; COPY stages a row (for the NTT/INTT steps,
 * which run through lf_ntt_fwd / lf_ntt_inv on the step's contiguous register rows). */
#define LF_POP_ADD 0        /* row_add      poly.py:85   */
#define LF_POP_SUB 1        /* row_sub      poly.py:89   */
#define LF_POP_MUL 2        /* row_mul      poly.py:94   */
#define LF_POP_MULACC 3     /* src0 + src1 * src2 (codegen.py:389-391) */
#define LF_POP_NEG 4        /* row_neg      poly.py:104  */
#define LF_POP_SCALARMUL 5  /* row_scalar_mul poly.py:108 */
#define LF_POP_MODSTEP 6    /* row_modstep  poly.py:112  */
#define LF_POP_AUTOMORPH 7  /* out[i] = src[perm_g(i)] (ntt.py:108-126) */
#define LF_POP_BCONV 8      /* exact conversion of k source rows to the lane prime (poly.py:150-178) */
#define LF_POP_COPY 9
typedef struct lf_plan_op {
  int32_t opcode, pidx;          /* LF_POP_*, prime index of the lane */
  uint32_t scalar, galois;       /* scalar reduced mod the lane prime; galois element (odd) */
  int32_t nsrc, k, W, pad;       /* sources; BConv: k sources and table words */
  const uint32_t* const* src;    /* device array of nsrc device row pointers */
  uint32_t* dst;                 /* register row (may be NULL) */
  uint32_t* store;               /* operand row to store into, or NULL */
  const uint32_t* table;         /* BConv table blob (k sources -> 1 target), else NULL */
} lf_plan_op;
int lf_plan_step(const lf_ctx* ctx, const lf_plan_op* ops, int nops, void* stream);

/* rescale (ckks.py:220-225, poly.py:284-287): out = 2 x level rows. */
size_t lf_rescale_workspace_bytes(const lf_ctx* ctx, int level, int batch);
int lf_rescale(const lf_ctx* ctx, int level, const uint32_t* ct, size_t ct_bstride,
               uint32_t* out, size_t out_bstride, int batch, void* workspace, void* stream);

/* rescale by the top ndrop in {1, 2} primes: ndrop = 2 equals two successive lf_rescale calls
 * (ckks.py:220-225 twice) bit for bit, in one pass.  out = 2 x (level + 1 - ndrop) rows;
 * workspace as lf_rescale. */
int lf_rescale_multi(const lf_ctx* ctx, int level, int ndrop, const uint32_t* ct,
                     size_t ct_bstride, uint32_t* out, size_t out_bstride, int batch,
                     void* workspace, void* stream);

/* lf_rescale_multi over ciphertexts whose polynomials are ct_pitch >= level + 1 rows apart
 * (row-prefix views of higher-level blocks, as lf_hom_mul_rescale_p). */
int lf_rescale_multi_p(const lf_ctx* ctx, int level, int ndrop, const uint32_t* ct, size_t ct_bstride,
                       int ct_pitch, uint32_t* out, size_t out_bstride, int batch, void* workspace,
                       void* stream);

/* keyswitch_decompose (ckks.py:95-117) materialised: pieces = beta x (level+1+alpha) rows,
 * eval domain, digit-major; beta = min(d, level+1).  Workspace as lf_keyswitch (batch 1). */
int lf_ks_decompose(const lf_ctx* ctx, int level, const uint32_t* x, uint32_t* pieces,
                    void* workspace, void* stream);

/* ---- bootstrap helpers (no reference counterpart: the reference has no bootstrap,
 * SPEC.md:8,136; built from the reference's row primitives, poly.py:85-121) ------------- */

/* ModRaise: `in` holds nin coefficient-domain rows mod q_0 (prime index 0); out receives
 * nin x nout rows, row i*nout + r = centred lift of in[i] (in (-q0/2, q0/2]) mod prime r. */
int lf_modraise(const lf_ctx* ctx, uint32_t* out, const uint32_t* in, int nin, int nout,
                void* stream);

/* Plaintext multiply-accumulate of a linear transform: out (2 x nrows rows: b then a) =
 * sum_i (b_i, a_i) * pt_i over nterm <= 32 terms; b, a, pt are HOST arrays of device row
 * pointers (nrows rows each, main primes 0..nrows-1).  Equals mul_plain + hom_add
 * (ckks.py:152-179) term by term. */
int lf_ptmac(const lf_ctx* ctx, uint32_t* out, int nrows, int nterm, const uint32_t* const* b,
             const uint32_t* const* a, const uint32_t* const* pt, void* stream);

/* Linear combination with constants: out (2 x nrows rows) = sum_i k_i * (b_i, a_i) over
 * nterm <= 8 terms; k is a HOST array [nterm][nrows] of per-row constants (any uint32, reduced
 * mod the row's prime).  Equals poly_scalar_mul + poly_add (poly.py:183-209) term by term. */
int lf_lincomb(const lf_ctx* ctx, uint32_t* out, int nrows, int nterm, const uint32_t* const* b,
               const uint32_t* const* a, const uint32_t* k, void* stream);
/* lf_lincomb plus a per-row constant cb[r] (HOST array, any uint32) added to the b rows:
 * sum_i k_i * ct_i + (cb, 0), i.e. then an add of a constant plaintext (ckks.py:152-179). */
int lf_lincomb_c(const lf_ctx* ctx, uint32_t* out, int nrows, int nterm, const uint32_t* const* b,
                 const uint32_t* const* a, const uint32_t* k, const uint32_t* cb, void* stream);

/* LFHE wire rows (little-endian uint64, reference serial.py:1-14, 63-69) <-> device uint32
 * residues, n words, both pointers on the device. */
int lf_rows_from_u64(uint32_t* out, const uint64_t* in, size_t n, void* stream);
int lf_rows_to_u64(uint64_t* out, const uint32_t* in, size_t n, void* stream);

/* Hoisted-ModDown building blocks for BSGS linear transforms: the same key switch as
 * lf_rotate_hoisted, stopped before ModDown.  out_ext receives, per rotation r,
 * 2 x (level+1+alpha) rows (extended basis, eval domain): (P*sigma_g(b) + acc_b, acc_a), the
 * inner product of keyswitch_inner_product (ckks.py:120-131) over permuted pieces.
 * lf_moddown_ext applies mod_down (poly.py:251-281) to both polynomials of such blocks. */
int lf_rotate_hoisted_ext(const lf_ctx* ctx, int level, const uint32_t* ct, int n_rot,
                          const uint32_t* gs, const uint32_t* const* keys, uint32_t* out_ext,
                          size_t out_bstride, void* workspace, void* stream);
size_t lf_moddown_workspace_bytes(const lf_ctx* ctx, int level, int batch);
int lf_moddown_ext(const lf_ctx* ctx, int level, const uint32_t* in_ext, size_t in_bstride,
                   uint32_t* out, size_t out_bstride, int batch, void* workspace, void* stream);

/* lf_moddown_ext followed by ndrop in {1, 2} rescales (ckks.py:220-225), bit for bit, as ONE
 * exact floor division by P q_level [q_level-1] (the tables of lf_hom_mul_rescale): out =
 * batch x 2 x (level + 1 - ndrop) rows; workspace as lf_moddown_ext. */
int lf_moddown_ext_rescale(const lf_ctx* ctx, int level, int ndrop, const uint32_t* in_ext,
                           size_t in_bstride, uint32_t* out, size_t out_bstride, int batch,
                           void* workspace, void* stream);
/* lf_ptmac over rows with arbitrary primes (prime_idx: HOST array, nrows entries). */
int lf_ptmac_rows(const lf_ctx* ctx, uint32_t* out, int nrows, const int32_t* prime_idx, int nterm,
                  const uint32_t* const* b, const uint32_t* const* a, const uint32_t* const* pt,
                  void* stream);

/* mul_plain by a compressed plaintext (reference compress.py:163-176): unique holds nrows x
 * unique_count values (eval domain); position i of row r reads unique[r][i / (N/unique_count)].
 * ct / out: 2 x nrows rows (b then a).  Bit-equal to mul_plain with the expanded plaintext. */
int lf_mul_compressed(const lf_ctx* ctx, uint32_t* out, const uint32_t* ct, const uint32_t* unique,
                      int nrows, int unique_count, void* stream);

/* ---------------------------------------------------------------------------------------
 * Limb-sharded keyswitch over k GPUs (reference multidev.py).  Placement as the
 * reference's partitioner (multidev.py:55-56): main row i on rank i % k, special row j on
 * rank j % k.  Each rank holds only its rows of the ciphertexts AND of the evaluation keys
 * (key rows: main_loc(L) ascending, then special_loc: lf_shard_info n_key_rows), and runs the
 * fused pipeline on them; the InputBroadcast exchange (multidev.py:172-185, 291-412) is two
 * all-gathers per keyswitch: the (l+1) row-INTT'd digit rows before the ModUp conversion and
 * the 2 alpha row-INTT'd special rows before ModDown.  Results are bit-identical to
 * lf_keyswitch / lf_hom_mul / lf_rotate restricted to the rank's rows.
 *   op 0 keyswitch(x):  x = local rows of x, out = (ks_b, ks_a) local rows (keyswitch, ckks.py:134-140)
 *   op 1 hom_mul:       x = local a1 rows, x2 = local a2 rows, e0/e1 = local ct1/ct2 blocks (ckks.py:182-194)
 *   op 2 hom_rotate:    x = local ct.a rows, e0 = local ct block, galois[b] (ckks.py:197-217)
 * Blocks are (2, n_main, N) (b rows then a rows); strides are in words. */
typedef struct lf_shard lf_shard;
typedef struct lf_comm lf_comm;
typedef struct lf_shard_call {
  int level, op, batch;                 /* batch <= 64 */
  const uint32_t* x;
  const uint32_t* x2;
  size_t x_bstride;
  const uint32_t* const* keys;          /* per instance: the rank's key rows (d, 2, n_key_rows, N) */
  const uint32_t* galois;               /* per instance (op 2), host array */
  uint32_t* out;
  size_t out_bstride;
  const uint32_t* e0;
  const uint32_t* e1;
  size_t e_bstride;
} lf_shard_call;
int lf_shard_create(const lf_ctx* ctx, int k, int rank, lf_shard** out);
int lf_shard_destroy(lf_shard* sh);
int lf_shard_info(const lf_shard* sh, int level, int* n_main, int* n_ext, int* n_key_rows, int* n_special);
size_t lf_shard_ws_bytes(const lf_shard* sh, int level, int batch);
/* byte offsets inside the workspace and per-rank byte counts of the two gathers:
 * {ModUp send, ModUp bytes, ModUp recv, ModDown send, ModDown bytes, ModDown recv};
 * recv holds the k ranks' send buffers back to back (an all-gather). */
int lf_shard_gather_layout(const lf_shard* sh, int level, int batch, size_t* out6);
/* one phase (0: before the ModUp gather, 1: between the gathers, 2: after the ModDown gather),
 * for callers that perform the all-gathers themselves */
int lf_shard_ks_phase(const lf_shard* sh, int phase, const lf_shard_call* call, void* workspace, void* stream);
/* NCCL communicator owned by the library (libnccl.so.2 resolved at run time): rank 0 creates
 * the 128-byte unique id, the caller broadcasts it, every rank calls lf_comm_create. */
int lf_comm_unique_id(void* out128);
int lf_comm_create(int nranks, int rank, const void* id128, lf_comm** out);
int lf_comm_destroy(lf_comm* comm);
int lf_shard_attach_comm(lf_shard* sh, lf_comm* comm);
/* the whole sharded keyswitch on `stream`, both all-gathers through the attached communicator
 * (ncclAllGather on the same stream: asynchronous, graph-capturable, no host synchronisation) */
int lf_shard_keyswitch(const lf_shard* sh, const lf_shard_call* call, void* workspace, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LF_B200_H */
