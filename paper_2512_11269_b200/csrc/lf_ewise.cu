// Row primitives (reference poly.py:85-121) and the coefficient-domain exact base conversion
// (poly.py:150-178, 234-248) on row batches.  Rows are N contiguous uint32 words; row r uses
// prime rm.p[r].  All outputs are canonical residues; `out` may alias any input.
#include "lf_ntt.cuh"
#include "lf_bconv.cuh"
#include "lf_ops.h"

#define LF_LAUNCH_CHECK_EW(call)                                               \
  do {                                                                         \
    cudaError_t e__ = (call);                                                  \
    if (e__ != cudaSuccess) {                                                  \
      lf_set_error("%s:%d: launch: %s", __FILE__, __LINE__, cudaGetErrorString(e__)); \
      return 3;                                                                \
    }                                                                          \
  } while (0)

struct EwArgs {
  u32* out;
  const u32* a;
  const u32* b;
  const u32* c;
  int op;
  RowMap rm;
  u32 s[LF_MAX_ROWS];
  u32 sp[LF_MAX_ROWS];
};

LF_DEV u32 ew_one(int op, u32 a, u32 b, u32 c, u32 s, u32 sp, const PrimeK& k) {
  const u32 q = k.q;
  switch (op) {
    case LF_OP_ADD: return addmod(a, b, q);
    case LF_OP_SUB: return submod(a, b, q);
    case LF_OP_MUL: return mulmod(a, b, k);
    case LF_OP_NEG: return a ? q - a : 0u;
    case LF_OP_SCALAR_MUL: return mul_shoup(a, s, sp, q);
    case LF_OP_MULACC: return reduce64((u64)a * b + c, k);
    case LF_OP_MODSTEP: return mul_shoup(submod(a, b, q), s, sp, q);
    case LF_OP_MUL_SCALAR_ADD: return addmod(mul_shoup(a, s, sp, q), b, q);   // a*s + b
    case LF_OP_ADD_SCALAR: return addmod(a, s, q);                              // a + s
    default: return 0u;
  }
}

__global__ void __launch_bounds__(256) k_ewise(EwArgs A, LfDev dv, int logN) {
  lf_pdl_trigger();
  lf_pdl_wait();
  const int row = blockIdx.y;
  const PrimeK k = dv.pk[A.rm.p[row]];
  const u32 s = A.s[row], sp = A.sp[row];
  const size_t N = (size_t)1 << logN;
  const size_t nv = N / 4;
  const size_t off = row * N;
  const uint4* a4 = reinterpret_cast<const uint4*>(A.a + off);
  const uint4* b4 = A.b ? reinterpret_cast<const uint4*>(A.b + off) : nullptr;
  const uint4* c4 = A.c ? reinterpret_cast<const uint4*>(A.c + off) : nullptr;
  uint4* o4 = reinterpret_cast<uint4*>(A.out + off);
  for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < nv;
       v += (size_t)gridDim.x * blockDim.x) {
    const uint4 a = a4[v];
    const uint4 b = b4 ? b4[v] : make_uint4(0, 0, 0, 0);
    const uint4 c = c4 ? c4[v] : make_uint4(0, 0, 0, 0);
    uint4 o;
    o.x = ew_one(A.op, a.x, b.x, c.x, s, sp, k);
    o.y = ew_one(A.op, a.y, b.y, c.y, s, sp, k);
    o.z = ew_one(A.op, a.z, b.z, c.z, s, sp, k);
    o.w = ew_one(A.op, a.w, b.w, c.w, s, sp, k);
    o4[v] = o;
  }
}

// out[r][i] = in[r][perm_g(i)]   (out must not alias in)
__global__ void __launch_bounds__(256) k_automorph(u32* out, const u32* in, u32 g, int logN,
                                                   int nrows) {
  lf_pdl_trigger();
  lf_pdl_wait();
  const size_t N = (size_t)1 << logN;
  const size_t total = N * nrows;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
       idx += (size_t)gridDim.x * blockDim.x) {
    const size_t row = idx >> logN;
    const u32 i = (u32)(idx & (N - 1));
    out[idx] = in[(row << logN) + auto_src_index(i, g, logN)];
  }
}

// Coefficient-domain exact conversion: src (k rows) -> out (m rows), one thread per coeff.
__global__ void __launch_bounds__(128) k_bconv(u32* out, const u32* src, BconvDev B, LfDev dv) {
  lf_pdl_trigger();
  lf_pdl_wait();
  const size_t N = (size_t)1 << dv.logN;
  const size_t n = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (n >= N) return;
  u32 y[64];
  for (int i = 0; i < B.k; ++i) {
    const PrimeK ks = dv.pk[B.src_pi[i]];
    y[i] = mul_shoup(src[i * N + n] % ks.q, B.c[i], B.cp[i], ks.q);
  }
  const u32 u = bconv_u(y, B);
  for (int t = 0; t < B.m; ++t) {
    const PrimeK kt = dv.pk[B.tgt_pi[t]];
    u64 acc = (u64)u * B.negS[t];
    for (int i = 0; i < B.k; ++i) acc += (u64)y[i] * B.w[(size_t)t * B.k + i];
    out[t * N + n] = reduce64(acc, kt);
  }
}

// ModRaise (bootstrap): coefficient rows mod q0 -> centred lift in (-q0/2, q0/2] reduced into
// the primes of nout rows: out[i*nout + r] = lift(in[i]) mod q_r.
__global__ void __launch_bounds__(256) k_modraise(u32* out, const u32* in, int nin, int nout,
                                                  LfDev dv) {
  lf_pdl_trigger();
  lf_pdl_wait();
  const size_t N = (size_t)1 << dv.logN;
  const u32 q0 = dv.pk[0].q;
  const size_t total = N * nin * nout;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
       idx += (size_t)gridDim.x * blockDim.x) {
    const size_t pos = idx & (N - 1);
    const size_t rr = idx >> dv.logN;            // i * nout + r
    const int r = (int)(rr % nout), i = (int)(rr / nout);
    const PrimeK k = dv.pk[r];
    const u32 c = in[(size_t)i * N + pos];
    u32 v;
    if (c > q0 / 2) {
      const u32 m = reduce32(q0 - c, k);        // (c - q0) mod q_r = -( (q0 - c) mod q_r )
      v = m ? k.q - m : 0u;
    } else {
      v = reduce32(c, k);
    }
    out[idx] = v;
  }
}

// Plaintext multiply-accumulate over terms (bootstrap linear transforms):
// out[p][r] = sum_i ct_i[p][r] * pt_i[r]  (p in {b, a}, r < nrows), 64-bit lazy sums.
struct PtMacArgs {
  u32* out;                 // 2 x nrows rows
  int nterm, nrows;
  RowMap rm;                // prime index of each row
  const u32* b[LF_PTMAC_MAX];
  const u32* a[LF_PTMAC_MAX];
  const u32* pt[LF_PTMAC_MAX];
};

__global__ void __launch_bounds__(256) k_ptmac(PtMacArgs A, LfDev dv) {
  lf_pdl_trigger();
  lf_pdl_wait();
  const int row = blockIdx.y;                   // 0 .. 2*nrows-1
  const int p = row / A.nrows, r = row % A.nrows;
  const PrimeK k = dv.pk[A.rm.p[r]];
  const size_t N = (size_t)1 << dv.logN;
  const size_t off = (size_t)r * N;
  for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < N / 4;
       v += (size_t)gridDim.x * blockDim.x) {
    u64 acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    for (int i = 0; i < A.nterm; ++i) {
      const u32* src = p ? A.a[i] : A.b[i];
      const uint4 x = reinterpret_cast<const uint4*>(src + off)[v];
      const uint4 y = reinterpret_cast<const uint4*>(A.pt[i] + off)[v];
      acc0 += (u64)x.x * y.x;
      acc1 += (u64)x.y * y.y;
      acc2 += (u64)x.z * y.z;
      acc3 += (u64)x.w * y.w;
    }
    reinterpret_cast<uint4*>(A.out + (size_t)row * N)[v] =
        make_uint4(reduce64(acc0, k), reduce64(acc1, k), reduce64(acc2, k), reduce64(acc3, k));
  }
}

// Linear combination with per-term, per-row constants (bootstrap polynomial leaves):
// out[p][r] = sum_i k_i[r] * ct_i[p][r]  (p in {b, a}), 64-bit lazy sums.
struct LinCombArgs {
  u32* out;
  int nterm, nrows;
  const u32* b[LF_LINCOMB_MAX];
  const u32* a[LF_LINCOMB_MAX];
  u32 k[LF_LINCOMB_MAX][LF_LINCOMB_ROWS];
  u32 c0[LF_LINCOMB_ROWS];   // constant added to the b rows (0 when none)
};

__global__ void __launch_bounds__(256) k_lincomb(LinCombArgs A, LfDev dv) {
  lf_pdl_trigger();
  lf_pdl_wait();
  const int row = blockIdx.y;
  const int p = row / A.nrows, r = row % A.nrows;
  const PrimeK k = dv.pk[r];
  const size_t N = (size_t)1 << dv.logN;
  const size_t off = (size_t)r * N;
  for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < N / 4;
       v += (size_t)gridDim.x * blockDim.x) {
    const u64 c0 = p ? 0u : A.c0[r];
    u64 acc0 = c0, acc1 = c0, acc2 = c0, acc3 = c0;
    for (int i = 0; i < A.nterm; ++i) {
      const u32* src = p ? A.a[i] : A.b[i];
      const uint4 x = reinterpret_cast<const uint4*>(src + off)[v];
      const u32 c = A.k[i][r];
      acc0 += (u64)x.x * c;
      acc1 += (u64)x.y * c;
      acc2 += (u64)x.z * c;
      acc3 += (u64)x.w * c;
    }
    reinterpret_cast<uint4*>(A.out + (size_t)row * N)[v] =
        make_uint4(reduce64(acc0, k), reduce64(acc1, k), reduce64(acc2, k), reduce64(acc3, k));
  }
}

int lf_launch_lincomb(const LfCtx* ctx, u32* out, int nrows, int nterm, const u32* const* b,
                      const u32* const* a, const u32* k, const u32* cb, cudaStream_t s) {
  LinCombArgs A;
  A.out = out; A.nterm = nterm; A.nrows = nrows;
  for (int r = 0; r < nrows; ++r) A.c0[r] = cb ? cb[r] % ctx->h_pk[r].q : 0u;
  for (int i = 0; i < nterm; ++i) {
    A.b[i] = b[i]; A.a[i] = a[i];
    for (int r = 0; r < nrows; ++r) A.k[i][r] = k[(size_t)i * nrows + r] % ctx->h_pk[r].q;
  }
  const int nv = ctx->N / 4;
  const int bx = (nv + 255) / 256 < 16 ? (nv + 255) / 256 : 16;
  dim3 grid(bx, 2 * nrows);
  LF_LAUNCH_CHECK_EW(lf_launch(k_lincomb, dim3(grid), dim3(256), 0, s, 1, A, ctx->dev()));
  LF_CHECK_LAUNCH();
  return 0;
}

// Wire-format conversion (LFHE rows are little-endian uint64, serial.py:1-14): narrow to the
// device's uint32 residues (values < 2^28) or widen back.
__global__ void __launch_bounds__(256) k_narrow(u32* out, const unsigned long long* in, size_t n) {
  lf_pdl_trigger();
  lf_pdl_wait();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = (u32)in[i];
}
__global__ void __launch_bounds__(256) k_widen(unsigned long long* out, const u32* in, size_t n) {
  lf_pdl_trigger();
  lf_pdl_wait();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

int lf_launch_convert(void* out, const void* in, size_t n, bool narrow, cudaStream_t s) {
  size_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks == 0) return 0;
  if (narrow) LF_LAUNCH_CHECK_EW(lf_launch(k_narrow, dim3((unsigned)blocks), dim3(256), 0, s, 1, (u32*)out, (const unsigned long long*)in, n));
  else LF_LAUNCH_CHECK_EW(lf_launch(k_widen, dim3((unsigned)blocks), dim3(256), 0, s, 1, (unsigned long long*)out, (const u32*)in, n));
  LF_CHECK_LAUNCH();
  return 0;
}

// Compressed-plaintext multiply (reference compress.py:163-176): the plaintext row stores one
// value per block of `1 << lb` consecutive evaluation positions; out = ct * unique[pos >> lb].
__global__ void __launch_bounds__(256) k_mul_compressed(u32* out, const u32* ct, const u32* uq,
                                                        int nrows, int ucount, int lb, LfDev dv) {
  lf_pdl_trigger();
  lf_pdl_wait();
  const size_t N = (size_t)1 << dv.logN;
  const size_t total = N * 2 * nrows;
  for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total;
       idx += (size_t)gridDim.x * blockDim.x) {
    const size_t rr = idx >> dv.logN;           // p * nrows + row
    const int row = (int)(rr % nrows);
    const u32 pos = (u32)(idx & (N - 1));
    const PrimeK k = dv.pk[row];
    out[idx] = mulmod(ct[idx], uq[(size_t)row * ucount + (pos >> lb)], k);
  }
}

int lf_launch_mul_compressed(const LfCtx* ctx, u32* out, const u32* ct, const u32* uq, int nrows,
                             int ucount, int lb, cudaStream_t s) {
  const size_t total = (size_t)ctx->N * 2 * nrows;
  size_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  LF_LAUNCH_CHECK_EW(lf_launch(k_mul_compressed, dim3((unsigned)blocks), dim3(256), 0, s, 1, out, ct, uq, nrows, ucount, lb, ctx->dev()));
  LF_CHECK_LAUNCH();
  return 0;
}

int lf_launch_modraise(const LfCtx* ctx, u32* out, const u32* in, int nin, int nout,
                       cudaStream_t s) {
  const size_t total = (size_t)ctx->N * nin * nout;
  size_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  LF_LAUNCH_CHECK_EW(lf_launch(k_modraise, dim3((unsigned)blocks), dim3(256), 0, s, 1, out, in, nin, nout, ctx->dev()));
  LF_CHECK_LAUNCH();
  return 0;
}

int lf_launch_ptmac(const LfCtx* ctx, u32* out, int nrows, int nterm, const u32* const* b,
                    const u32* const* a, const u32* const* pt, const int32_t* pidx, cudaStream_t s) {
  PtMacArgs A;
  A.out = out; A.nterm = nterm; A.nrows = nrows;
  A.rm.n = nrows;
  for (int r = 0; r < nrows; ++r) A.rm.p[r] = (unsigned char)(pidx ? pidx[r] : r);
  for (int i = 0; i < nterm; ++i) { A.b[i] = b[i]; A.a[i] = a[i]; A.pt[i] = pt[i]; }
  const int nv = ctx->N / 4;
  const int bx = (nv + 255) / 256 < 16 ? (nv + 255) / 256 : 16;
  dim3 grid(bx, 2 * nrows);
  LF_LAUNCH_CHECK_EW(lf_launch(k_ptmac, dim3(grid), dim3(256), 0, s, 1, A, ctx->dev()));
  LF_CHECK_LAUNCH();
  return 0;
}

int lf_launch_ewise(const LfCtx* ctx, int op, u32* out, const u32* a, const u32* b,
                    const u32* c, const RowMap& rm, const u32* scalars, cudaStream_t s) {
  EwArgs A;
  A.out = out; A.a = a; A.b = b; A.c = c; A.op = op; A.rm = rm;
  for (int r = 0; r < rm.n; ++r) {
    const u32 q = ctx->h_pk[rm.p[r]].q;
    const u32 v = scalars ? scalars[r] % q : 0u;
    A.s[r] = v;
    A.sp[r] = (u32)(((u64)v << 32) / q);
  }
  const int nv = ctx->N / 4;
  const int bx = (nv + 255) / 256 < 64 ? (nv + 255) / 256 : 64;
  dim3 grid(bx, rm.n);
  LF_LAUNCH_CHECK_EW(lf_launch(k_ewise, dim3(grid), dim3(256), 0, s, 1, A, ctx->dev(), ctx->logN));
  LF_CHECK_LAUNCH();
  return 0;
}

int lf_launch_automorph(const LfCtx* ctx, u32* out, const u32* in, u32 g, int nrows,
                        cudaStream_t s) {
  const size_t total = (size_t)ctx->N * nrows;
  size_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  LF_LAUNCH_CHECK_EW(lf_launch(k_automorph, dim3((unsigned)blocks), dim3(256), 0, s, 1, out, in, g, ctx->logN, nrows));
  LF_CHECK_LAUNCH();
  return 0;
}

int lf_launch_bconv(const LfCtx* ctx, u32* out, const u32* src, const u32* tab, int k, int m,
                    int W, cudaStream_t s) {
  if (k > 64 || W > LF_BC_MAXW) {
    lf_set_error("bconv: k=%d W=%d exceeds limits", k, W);
    return 2;
  }
  const BconvDev B = lf_bconv_view(tab, k, m, W);
  const int blocks = (ctx->N + 127) / 128;
  LF_LAUNCH_CHECK_EW(lf_launch(k_bconv, dim3(blocks), dim3(128), 0, s, 1, out, src, B, ctx->dev()));
  LF_CHECK_LAUNCH();
  return 0;
}
