// Standalone batched forward / inverse negacyclic NTT (reference ntt.py:70-105).
// Two kernels per direction: a column pass (first L1 CT stages / last L1 GS stages) and a
// row pass.  Each row of the batch may use a different prime (RowMap).
#include "lf_ntt.cuh"

template <int L1, int L2>
__global__ void __launch_bounds__(NttShape<L1, L2>::TC)
k_ntt_fwd_C(u32* rows, RowMap rm, LfDev dv) {
  using S = NttShape<L1, L2>;
  using C = LineCfg<L1>;
  constexpr int TILES = S::NCOL / S::CW;
  extern __shared__ u32 sm[];
  const int row = blockIdx.x / TILES, col0 = (blockIdx.x % TILES) * S::CW;
  const int c = threadIdx.x % S::CW, tl = threadIdx.x / S::CW;
  const int pi = rm.p[row];
  const u32 q = dv.pk[pi].q;
  const uint2* tw = dv.twf + ((size_t)pi << (L1 + L2));
  u32* base = rows + ((size_t)row << (L1 + L2)) + col0 + c;
  u32 x[C::E];
  load_col_step1<L1, L2>(x, base, tl);
  fwd_line<L1, 1>(x, 1u, tw, q, sm, tl, AddrC<L1, S::CW>{c}, SyncBlock{});
  store_col_step2<L1, L2>(x, base, tl);
}

template <int L1, int L2>
__global__ void __launch_bounds__(NttShape<L1, L2>::TR)
k_ntt_fwd_R(u32* rows, RowMap rm, LfDev dv, int nlines) {
  using S = NttShape<L1, L2>;
  using C = LineCfg<L2>;
  extern __shared__ u32 sm[];
  const int tl = threadIdx.x % C::T, ln = threadIdx.x / C::T;
  int line = blockIdx.x * S::LPC + ln;
  const bool valid = line < nlines;
  if (!valid) line = nlines - 1;
  const int row = line >> L1, hi = line & ((1 << L1) - 1);
  const int pi = rm.p[row];
  const PrimeK pk = dv.pk[pi];
  const uint2* tw = dv.twf + ((size_t)pi << (L1 + L2));
  u32* base = rows + ((size_t)line << L2);
  u32 x[C::E];
  load_row_step1<L2>(x, base, tl);
  fwd_line<L2, S::FWD_C_OUT>(x, (1u << L1) + hi, tw, pk.q, sm, tl,
                             AddrR<L2>{ln * pitchR<L2>()}, SyncWarp{});
#pragma unroll
  for (int e = 0; e < C::E; ++e) x[e] = reduce32(x[e], pk);
  if (valid) store_row_step2<L2>(x, base, tl);
}

template <int L1, int L2>
__global__ void __launch_bounds__(NttShape<L1, L2>::TR)
k_ntt_inv_R(u32* rows, RowMap rm, LfDev dv, int nlines) {
  using S = NttShape<L1, L2>;
  using C = LineCfg<L2>;
  extern __shared__ u32 sm[];
  const int tl = threadIdx.x % C::T, ln = threadIdx.x / C::T;
  int line = blockIdx.x * S::LPC + ln;
  const bool valid = line < nlines;
  if (!valid) line = nlines - 1;
  const int row = line >> L1, hi = line & ((1 << L1) - 1);
  const int pi = rm.p[row];
  const u32 q = dv.pk[pi].q;
  const uint2* tw = dv.twi + ((size_t)pi << (L1 + L2));
  u32* base = rows + ((size_t)line << L2);
  u32 x[C::E];
  load_row_step2<L2>(x, base, tl);
  inv_line<L2>(x, (1u << L1) + hi, tw, q, sm, tl, AddrR<L2>{ln * pitchR<L2>()}, SyncWarp{});
  if (valid) store_row_step1<L2>(x, base, tl);
}

template <int L1, int L2>
__global__ void __launch_bounds__(NttShape<L1, L2>::TC)
k_ntt_inv_C(u32* rows, RowMap rm, LfDev dv) {
  using S = NttShape<L1, L2>;
  using C = LineCfg<L1>;
  constexpr int TILES = S::NCOL / S::CW;
  extern __shared__ u32 sm[];
  const int row = blockIdx.x / TILES, col0 = (blockIdx.x % TILES) * S::CW;
  const int c = threadIdx.x % S::CW, tl = threadIdx.x / S::CW;
  const int pi = rm.p[row];
  const PrimeK pk = dv.pk[pi];
  const uint2* tw = dv.twi + ((size_t)pi << (L1 + L2));
  u32* base = rows + ((size_t)row << (L1 + L2)) + col0 + c;
  u32 x[C::E];
  load_col_step2<L1, L2>(x, base, tl);
  inv_line<L1>(x, 1u, tw, pk.q, sm, tl, AddrC<L1, S::CW>{c}, SyncBlock{});
#pragma unroll
  for (int j = 0; j < C::E; ++j) x[j] = mul_shoup(x[j], pk.ninv, pk.ninvp, pk.q);
  store_col_step1<L1, L2>(x, base, tl);
}

int lf_launch_ntt(const LfCtx* ctx, u32* rows, const RowMap& rm, bool inverse, cudaStream_t s) {
  const LfDev dv = ctx->dev();
  const int nrows = rm.n;
  if (nrows <= 0) return 0;
#define LF_NTT_LAUNCH(A, B)                                                                 \
  {                                                                                         \
    using S = NttShape<A, B>;                                                               \
    const int nlines = nrows << A;                                                          \
    const int gridR = (nlines + S::LPC - 1) / S::LPC;                                       \
    const int gridC = nrows * (S::NCOL / S::CW);                                            \
    const size_t smC = smemC_words<A, S::CW>() * 4;                                         \
    const size_t smR = (size_t)S::LPC * pitchR<B>() * 4;                                    \
    if (!inverse) {                                                                         \
      k_ntt_fwd_C<A, B><<<gridC, S::TC, smC, s>>>(rows, rm, dv);                            \
      k_ntt_fwd_R<A, B><<<gridR, S::TR, smR, s>>>(rows, rm, dv, nlines);                    \
    } else {                                                                                \
      k_ntt_inv_R<A, B><<<gridR, S::TR, smR, s>>>(rows, rm, dv, nlines);                    \
      k_ntt_inv_C<A, B><<<gridC, S::TC, smC, s>>>(rows, rm, dv);                            \
    }                                                                                       \
  }
  LF_DISPATCH_LOGN(ctx->logN, LF_NTT_LAUNCH)
#undef LF_NTT_LAUNCH
  LF_CHECK_LAUNCH();
  return 0;
}
