// C ABI entry points (include/lf_b200.h): context management and the unfused primitives.
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "lf_ops.h"
#include "lf_plan.h"

static thread_local char g_err[512] = "";

void lf_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

#define LF_CUDA(call)                                                                \
  do {                                                                               \
    cudaError_t e__ = (call);                                                        \
    if (e__ != cudaSuccess) {                                                        \
      lf_set_error("%s:%d: %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e__)); \
      return 3;                                                                      \
    }                                                                                \
  } while (0)

static u32 powmod(u64 b, u64 e, u64 q) {
  u64 r = 1;
  b %= q;
  while (e) {
    if (e & 1) r = r * b % q;
    b = b * b % q;
    e >>= 1;
  }
  return (u32)r;
}
static u32 shoup(u32 w, u32 q) { return (u32)(((u64)w << 32) / q); }
static u32 brev(u32 x, int bits) {
  u32 r = 0;
  for (int b = 0; b < bits; ++b) r |= ((x >> b) & 1u) << (bits - 1 - b);
  return r;
}

extern "C" {

int lf_abi_version(void) { return LF_ABI_VERSION; }
const char* lf_last_error(void) { return g_err; }

int lf_ctx_create(int logN, int nprimes, const uint32_t* primes, const uint32_t* psis,
                  lf_ctx** out) {
  if (!out || !primes || !psis) { lf_set_error("lf_ctx_create: null argument"); return 1; }
  if (logN < 4 || logN > 16) { lf_set_error("lf_ctx_create: logN %d outside [4,16]", logN); return 2; }
  if (nprimes < 1 || nprimes > 255) { lf_set_error("lf_ctx_create: nprimes %d", nprimes); return 2; }
  const u32 N = 1u << logN;
  std::vector<PrimeK> pk(nprimes);
  std::vector<uint2> twf((size_t)nprimes * N), twi((size_t)nprimes * N);
  for (int i = 0; i < nprimes; ++i) {
    const u32 q = primes[i], psi = psis[i];
    if (q >= (1u << 28) || q % (2 * N) != 1) {
      lf_set_error("lf_ctx_create: prime %u not < 2^28 and 1 mod 2N", q);
      return 2;
    }
    if (powmod(psi, N, q) != q - 1) {
      lf_set_error("lf_ctx_create: psi %u is not a primitive 2N-th root mod %u", psi, q);
      return 2;
    }
    PrimeK k{};
    k.q = q;
    k.qbar = (u32)((((u64)1) << 32) / q);
    k.r32 = (u32)((((u64)1) << 32) % q);
    k.r32p = shoup(k.r32, q);
    k.ninv = powmod(N, q - 2, q);
    k.ninvp = shoup(k.ninv, q);
    pk[i] = k;
    const u32 ipsi = powmod(psi, q - 2, q);
    std::vector<u32> pw(N), ipw(N);
    u64 a = 1, b = 1;
    for (u32 j = 0; j < N; ++j) {
      pw[j] = (u32)a;
      ipw[j] = (u32)b;
      a = a * psi % q;
      b = b * ipsi % q;
    }
    for (u32 j = 0; j < N; ++j) {
      const u32 w = pw[brev(j, logN)], iw = ipw[brev(j, logN)];
      twf[(size_t)i * N + j] = make_uint2(w, shoup(w, q));
      twi[(size_t)i * N + j] = make_uint2(iw, shoup(iw, q));
    }
  }
  // Row-pass twiddle subtrees, transposed per CTA line block for the depths the second phase of
  // a line transform reads (thread-varying roots): see TwTree<LP> in lf_line.cuh.
  std::vector<uint2> twfT(twf), twiT(twi);
  {
    int L1, L2;
    lf_split(logN, L1, L2);
    const int DS = (L2 + 1) / 2;
    int lpc = 256 / (1 << (L2 / 2));
    if (lpc < 1) lpc = 1;
    const int span = lpc < (1 << L1) ? lpc : (1 << L1);
    // column tree (root 1, the first L1 levels; read through TwGlobalT<L1>{.., 1, 1} by the
    // BConv column passes): its second-phase depths transposed the same way, span 1
    const int DSc = (L1 + 1) / 2;
    for (int i = 0; i < nprimes; ++i)
      for (int d = DSc; d < L1; ++d) {
        const int kk = d - DSc;
        const size_t c0 = (size_t)i * N + ((size_t)1 << d);
        for (int off = 0; off < (1 << d); ++off) {
          const size_t dst = c0 + (size_t)(off & ((1 << kk) - 1)) * (1u << DSc) + (off >> kk);
          twfT[dst] = twf[c0 + off];
          twiT[dst] = twi[c0 + off];
        }
      }
    for (int i = 0; i < nprimes; ++i)
      for (int d = DS; d < L2; ++d) {
        const int kk = d - DS, cnt = span << d;
        for (int b = 0; b < (1 << L1) / span; ++b) {
          const size_t c0 = (size_t)i * N + ((size_t)((1u << L1) + (u32)(b * span)) << d);
          for (int off = 0; off < cnt; ++off) {
            const size_t dst = c0 + (size_t)(off & ((1 << kk) - 1)) * (span << DS) + (off >> kk);
            twfT[dst] = twf[c0 + off];
            twiT[dst] = twi[c0 + off];
          }
        }
      }
  }
  LfCtx* c = new LfCtx();
  c->logN = logN;
  c->N = (int)N;
  c->nprimes = nprimes;
  c->h_pk = new PrimeK[nprimes];
  memcpy(c->h_pk, pk.data(), sizeof(PrimeK) * nprimes);
  LF_CUDA(cudaMalloc(&c->d_pk, sizeof(PrimeK) * nprimes));
  LF_CUDA(cudaMalloc(&c->d_twf, sizeof(uint2) * twf.size()));
  LF_CUDA(cudaMalloc(&c->d_twi, sizeof(uint2) * twi.size()));
  LF_CUDA(cudaMemcpy(c->d_pk, pk.data(), sizeof(PrimeK) * nprimes, cudaMemcpyHostToDevice));
  LF_CUDA(cudaMemcpy(c->d_twf, twf.data(), sizeof(uint2) * twf.size(), cudaMemcpyHostToDevice));
  LF_CUDA(cudaMemcpy(c->d_twi, twi.data(), sizeof(uint2) * twi.size(), cudaMemcpyHostToDevice));
  LF_CUDA(cudaMalloc(&c->d_twfT, sizeof(uint2) * twfT.size()));
  LF_CUDA(cudaMalloc(&c->d_twiT, sizeof(uint2) * twiT.size()));
  LF_CUDA(cudaMemcpy(c->d_twfT, twfT.data(), sizeof(uint2) * twfT.size(), cudaMemcpyHostToDevice));
  LF_CUDA(cudaMemcpy(c->d_twiT, twiT.data(), sizeof(uint2) * twiT.size(), cudaMemcpyHostToDevice));
  *out = c;
  return 0;
}

int lf_ctx_destroy(lf_ctx* ctx) {
  if (!ctx) return 0;
  lf_free_ks_plan(ctx->ks);
  cudaFree(ctx->d_pk);
  cudaFree(ctx->d_twf);
  cudaFree(ctx->d_twi);
  cudaFree(ctx->d_twfT);
  cudaFree(ctx->d_twiT);
  delete[] ctx->h_pk;
  delete ctx;
  return 0;
}

static int fill_rowmap(const lf_ctx* ctx, RowMap& rm, const int32_t* pidx, int r0, int n) {
  rm.n = n;
  for (int r = 0; r < n; ++r) {
    const int p = pidx[r0 + r];
    if (p < 0 || p >= ctx->nprimes) { lf_set_error("prime index %d out of range", p); return 2; }
    rm.p[r] = (unsigned char)p;
  }
  return 0;
}

static int ntt_common(const lf_ctx* ctx, uint32_t* rows, int nrows, const int32_t* pidx,
                      void* stream, bool inv) {
  if (!ctx || (!rows && nrows) || (!pidx && nrows)) { lf_set_error("lf_ntt: null argument"); return 1; }
  for (int r0 = 0; r0 < nrows; r0 += LF_MAX_ROWS) {
    RowMap rm;
    const int n = nrows - r0 < LF_MAX_ROWS ? nrows - r0 : LF_MAX_ROWS;
    if (int e = fill_rowmap(ctx, rm, pidx, r0, n)) return e;
    if (int e = lf_launch_ntt(ctx, rows + (size_t)r0 * ctx->N, rm, inv, (cudaStream_t)stream))
      return e;
  }
  return 0;
}

int lf_ntt_fwd(const lf_ctx* ctx, uint32_t* rows, int nrows, const int32_t* pidx, void* stream) {
  return ntt_common(ctx, rows, nrows, pidx, stream, false);
}
int lf_ntt_inv(const lf_ctx* ctx, uint32_t* rows, int nrows, const int32_t* pidx, void* stream) {
  return ntt_common(ctx, rows, nrows, pidx, stream, true);
}

int lf_ewise(const lf_ctx* ctx, int op, uint32_t* out, const uint32_t* a, const uint32_t* b,
             const uint32_t* c, int nrows, const int32_t* pidx, const uint32_t* scalars,
             void* stream) {
  if (!ctx || !out || !a || (!pidx && nrows)) { lf_set_error("lf_ewise: null argument"); return 1; }
  if (op < LF_OP_ADD || op > LF_OP_ADD_SCALAR) { lf_set_error("lf_ewise: bad op %d", op); return 2; }
  const bool needs_b = op == LF_OP_ADD || op == LF_OP_SUB || op == LF_OP_MUL || op == LF_OP_MULACC ||
                       op == LF_OP_MODSTEP || op == LF_OP_MUL_SCALAR_ADD;
  if (needs_b && !b) { lf_set_error("lf_ewise: op %d needs b", op); return 1; }
  if (op == LF_OP_MULACC && !c) { lf_set_error("lf_ewise: MULACC needs c"); return 1; }
  const size_t N = ctx->N;
  for (int r0 = 0; r0 < nrows; r0 += LF_MAX_ROWS) {
    RowMap rm;
    const int n = nrows - r0 < LF_MAX_ROWS ? nrows - r0 : LF_MAX_ROWS;
    if (int e = fill_rowmap(ctx, rm, pidx, r0, n)) return e;
    const size_t off = (size_t)r0 * N;
    if (int e = lf_launch_ewise(ctx, op, out + off, a + off, b ? b + off : nullptr,
                                c ? c + off : nullptr, rm, scalars ? scalars + r0 : nullptr,
                                (cudaStream_t)stream))
      return e;
  }
  return 0;
}

int lf_automorph(const lf_ctx* ctx, uint32_t* out, const uint32_t* in, uint32_t g, int nrows,
                 void* stream) {
  if (!ctx || !out || !in) { lf_set_error("lf_automorph: null argument"); return 1; }
  if (!(g & 1)) { lf_set_error("lf_automorph: automorphism index must be odd"); return 2; }
  if (out == in) { lf_set_error("lf_automorph: out must not alias in"); return 2; }
  return lf_launch_automorph(ctx, out, in, g, nrows, (cudaStream_t)stream);
}

int lf_bconv(const lf_ctx* ctx, uint32_t* out, const uint32_t* src, const uint32_t* table,
             int k, int m, int W, void* stream) {
  if (!ctx || !out || !src || !table) { lf_set_error("lf_bconv: null argument"); return 1; }
  return lf_launch_bconv(ctx, out, src, table, k, m, W, (cudaStream_t)stream);
}

int lf_modraise(const lf_ctx* ctx, uint32_t* out, const uint32_t* in, int nin, int nout,
                void* stream) {
  if (!ctx || !out || !in) { lf_set_error("lf_modraise: null argument"); return 1; }
  if (nout < 1 || nout > ctx->nprimes || nin < 1) { lf_set_error("lf_modraise: bad row counts"); return 2; }
  return lf_launch_modraise(ctx, out, in, nin, nout, (cudaStream_t)stream);
}

int lf_ptmac(const lf_ctx* ctx, uint32_t* out, int nrows, int nterm, const uint32_t* const* b,
             const uint32_t* const* a, const uint32_t* const* pt, void* stream) {
  if (!ctx || !out || !b || !a || !pt) { lf_set_error("lf_ptmac: null argument"); return 1; }
  if (nterm < 1 || nterm > LF_PTMAC_MAX) { lf_set_error("lf_ptmac: nterm %d outside [1, %d]", nterm, LF_PTMAC_MAX); return 2; }
  if (nrows < 1 || nrows > ctx->nprimes) { lf_set_error("lf_ptmac: bad nrows %d", nrows); return 2; }
  for (int i = 0; i < nterm; ++i)
    if (!b[i] || !a[i] || !pt[i]) { lf_set_error("lf_ptmac: null term %d", i); return 1; }
  return lf_launch_ptmac(ctx, out, nrows, nterm, b, a, pt, nullptr, (cudaStream_t)stream);
}

int lf_ptmac_rows(const lf_ctx* ctx, uint32_t* out, int nrows, const int32_t* prime_idx, int nterm,
                  const uint32_t* const* b, const uint32_t* const* a, const uint32_t* const* pt,
                  void* stream) {
  if (!ctx || !out || !b || !a || !pt || !prime_idx) { lf_set_error("lf_ptmac_rows: null argument"); return 1; }
  if (nterm < 1 || nterm > LF_PTMAC_MAX) { lf_set_error("lf_ptmac_rows: nterm %d outside [1, %d]", nterm, LF_PTMAC_MAX); return 2; }
  if (nrows < 1 || nrows > LF_MAX_ROWS) { lf_set_error("lf_ptmac_rows: bad nrows %d", nrows); return 2; }
  for (int r = 0; r < nrows; ++r)
    if (prime_idx[r] < 0 || prime_idx[r] >= ctx->nprimes) { lf_set_error("lf_ptmac_rows: bad prime index"); return 2; }
  for (int i = 0; i < nterm; ++i)
    if (!b[i] || !a[i] || !pt[i]) { lf_set_error("lf_ptmac_rows: null term %d", i); return 1; }
  return lf_launch_ptmac(ctx, out, nrows, nterm, b, a, pt, prime_idx, (cudaStream_t)stream);
}

int lf_lincomb(const lf_ctx* ctx, uint32_t* out, int nrows, int nterm, const uint32_t* const* b,
               const uint32_t* const* a, const uint32_t* k, void* stream) {
  if (!ctx || !out || !b || !a || !k) { lf_set_error("lf_lincomb: null argument"); return 1; }
  if (nterm < 1 || nterm > LF_LINCOMB_MAX) { lf_set_error("lf_lincomb: nterm %d outside [1, %d]", nterm, LF_LINCOMB_MAX); return 2; }
  if (nrows < 1 || nrows > ctx->nprimes || nrows > LF_LINCOMB_ROWS) { lf_set_error("lf_lincomb: bad nrows %d", nrows); return 2; }
  for (int i = 0; i < nterm; ++i)
    if (!b[i] || !a[i]) { lf_set_error("lf_lincomb: null term %d", i); return 1; }
  return lf_launch_lincomb(ctx, out, nrows, nterm, b, a, k, nullptr, (cudaStream_t)stream);
}

int lf_lincomb_c(const lf_ctx* ctx, uint32_t* out, int nrows, int nterm, const uint32_t* const* b,
                 const uint32_t* const* a, const uint32_t* k, const uint32_t* cb, void* stream) {
  if (!ctx || !out || !b || !a || !k || !cb) { lf_set_error("lf_lincomb_c: null argument"); return 1; }
  if (nterm < 1 || nterm > LF_LINCOMB_MAX) { lf_set_error("lf_lincomb_c: nterm %d outside [1, %d]", nterm, LF_LINCOMB_MAX); return 2; }
  if (nrows < 1 || nrows > ctx->nprimes || nrows > LF_LINCOMB_ROWS) { lf_set_error("lf_lincomb_c: bad nrows %d", nrows); return 2; }
  for (int i = 0; i < nterm; ++i)
    if (!b[i] || !a[i]) { lf_set_error("lf_lincomb_c: null term %d", i); return 1; }
  return lf_launch_lincomb(ctx, out, nrows, nterm, b, a, k, cb, (cudaStream_t)stream);
}

int lf_rows_from_u64(uint32_t* out, const uint64_t* in, size_t n, void* stream) {
  if (!out || !in) { lf_set_error("lf_rows_from_u64: null argument"); return 1; }
  return lf_launch_convert(out, in, n, true, (cudaStream_t)stream);
}

int lf_rows_to_u64(uint64_t* out, const uint32_t* in, size_t n, void* stream) {
  if (!out || !in) { lf_set_error("lf_rows_to_u64: null argument"); return 1; }
  return lf_launch_convert(out, in, n, false, (cudaStream_t)stream);
}

int lf_mul_compressed(const lf_ctx* ctx, uint32_t* out, const uint32_t* ct, const uint32_t* unique,
                      int nrows, int unique_count, void* stream) {
  if (!ctx || !out || !ct || !unique) { lf_set_error("lf_mul_compressed: null argument"); return 1; }
  if (nrows < 1 || nrows > ctx->nprimes) { lf_set_error("lf_mul_compressed: bad nrows %d", nrows); return 2; }
  if (unique_count < 1 || unique_count > ctx->N || (unique_count & (unique_count - 1)) || ctx->N % unique_count) {
    lf_set_error("lf_mul_compressed: unique_count %d must be a power of two dividing N", unique_count);
    return 2;
  }
  int lb = 0;
  while ((unique_count << lb) < ctx->N) ++lb;
  return lf_launch_mul_compressed(ctx, out, ct, unique, nrows, unique_count, lb, (cudaStream_t)stream);
}

int lf_plan_step(const lf_ctx* ctx, const lf_plan_op* ops, int nops, void* stream) {
  if (!ctx || (!ops && nops > 0)) { lf_set_error("lf_plan_step: null argument"); return 1; }
  return lf_launch_plan_step(ctx, ops, nops, (cudaStream_t)stream);
}

}  // extern "C"
