// Standalone batched forward / inverse negacyclic NTT (reference ntt.py:70-105).
// Two kernels per direction: a column pass (first L1 CT stages / last L1 GS stages) and a
// row pass.  Each row of the batch may use a different prime (RowMap).  Every CTA stages the
// twiddles its lines need in shared memory first (coalesced 16-byte loads): the column pass
// uses the 2^L1 nodes under root 1, the row pass the subtrees under its LPCR line roots.
#include "lf_ntt.cuh"

template <int L1, int L2>
__global__ void __launch_bounds__(NttShape<L1, L2>::TC)
k_ntt_fwd_C(u32* rows, RowMap rm, LfDev dv) {
  using S = NttShape<L1, L2>;
  using C = LineCfg<L1>;
  constexpr int TILES = S::NCOL / S::CW;
  extern __shared__ __align__(16) u32 sm[];
  uint2* tws = reinterpret_cast<uint2*>(sm);
  u32* xs = sm + 2 * C::M;
  const int row = blockIdx.x / TILES, col0 = (blockIdx.x % TILES) * S::CW;
  const int c = threadIdx.x % S::CW, tl = threadIdx.x / S::CW;
  const int pi = rm.p[row];
  const u32 q = dv.pk[pi].q;
  stage_flat<C::M>(tws, dv.twf + ((size_t)pi << (L1 + L2)), threadIdx.x, blockDim.x);
  u32* base = rows + ((size_t)row << (L1 + L2)) + col0 + c;
  u32 x[C::E];
  load_col_step1<L1, L2>(x, base, tl);
  __syncthreads();
  fwd_line<L1, 1>(x, 1u, TwFlat{tws}, q, xs, tl, AddrC<L1, S::CW>{c}, SyncBlock{});
  store_col_step2<L1, L2>(x, base, tl);
}

template <int L1, int L2>
__global__ void __launch_bounds__(NttShape<L1, L2>::TRR)
k_ntt_fwd_R(u32* rows, RowMap rm, LfDev dv) {
  using S = NttShape<L1, L2>;
  using C = LineCfg<L2>;
  constexpr int GROUPS = (1 << L1) / S::LPCR;
  extern __shared__ __align__(16) u32 sm[];
  uint2* tws = reinterpret_cast<uint2*>(sm);
  u32* xs = sm + 2 * S::LPCR * (C::M - 1) + 2;
  const int tl = threadIdx.x % C::T, ln = threadIdx.x / C::T;
  const int row = blockIdx.x / GROUPS, hi0 = (blockIdx.x % GROUPS) * S::LPCR, hi = hi0 + ln;
  const int pi = rm.p[row];
  const PrimeK pk = dv.pk[pi];
  __shared__ unsigned long long twbar;
  tw_bulk_begin<L2>(tws, dv.twfT + ((size_t)pi << (L1 + L2)), (1u << L1) + hi0, S::LPCR, &twbar);
  u32* base = rows + ((size_t)row << (L1 + L2)) + ((size_t)hi << L2);
  u32 x[C::E];
  load_row_step1<L2>(x, base, tl);
  tw_bulk_wait(&twbar);
  fwd_line<L2, S::FWD_C_OUT>(x, (1u << L1) + hi, TwTree<L2>{tws, (1u << L1) + hi0, S::LPCR}, pk.q, xs,
                             tl, AddrR<L2>{ln * pitchR<L2>()}, SyncWarp{});
#pragma unroll
  for (int e = 0; e < C::E; ++e) x[e] = reduce32(x[e], pk);
  store_row_step2<L2>(x, base, tl);
}

template <int L1, int L2>
__global__ void __launch_bounds__(NttShape<L1, L2>::TRR)
k_ntt_inv_R(u32* rows, RowMap rm, LfDev dv) {
  using S = NttShape<L1, L2>;
  using C = LineCfg<L2>;
  constexpr int GROUPS = (1 << L1) / S::LPCR;
  extern __shared__ __align__(16) u32 sm[];
  uint2* tws = reinterpret_cast<uint2*>(sm);
  u32* xs = sm + 2 * S::LPCR * (C::M - 1) + 2;
  const int tl = threadIdx.x % C::T, ln = threadIdx.x / C::T;
  const int row = blockIdx.x / GROUPS, hi0 = (blockIdx.x % GROUPS) * S::LPCR, hi = hi0 + ln;
  const int pi = rm.p[row];
  const u32 q = dv.pk[pi].q;
  __shared__ unsigned long long twbar;
  tw_bulk_begin<L2>(tws, dv.twiT + ((size_t)pi << (L1 + L2)), (1u << L1) + hi0, S::LPCR, &twbar);
  u32* base = rows + ((size_t)row << (L1 + L2)) + ((size_t)hi << L2);
  u32 x[C::E];
  load_row_step2<L2>(x, base, tl);
  tw_bulk_wait(&twbar);
  inv_line<L2>(x, (1u << L1) + hi, TwTree<L2>{tws, (1u << L1) + hi0, S::LPCR}, q, xs, tl,
               AddrR<L2>{ln * pitchR<L2>()}, SyncWarp{});
  store_row_step1<L2>(x, base, tl);
}

template <int L1, int L2>
__global__ void __launch_bounds__(NttShape<L1, L2>::TC)
k_ntt_inv_C(u32* rows, RowMap rm, LfDev dv) {
  using S = NttShape<L1, L2>;
  using C = LineCfg<L1>;
  constexpr int TILES = S::NCOL / S::CW;
  extern __shared__ __align__(16) u32 sm[];
  uint2* tws = reinterpret_cast<uint2*>(sm);
  u32* xs = sm + 2 * C::M;
  const int row = blockIdx.x / TILES, col0 = (blockIdx.x % TILES) * S::CW;
  const int c = threadIdx.x % S::CW, tl = threadIdx.x / S::CW;
  const int pi = rm.p[row];
  const PrimeK pk = dv.pk[pi];
  stage_flat<C::M>(tws, dv.twi + ((size_t)pi << (L1 + L2)), threadIdx.x, blockDim.x);
  u32* base = rows + ((size_t)row << (L1 + L2)) + col0 + c;
  u32 x[C::E];
  load_col_step2<L1, L2>(x, base, tl);
  __syncthreads();
  inv_line<L1>(x, 1u, TwFlat{tws}, pk.q, xs, tl, AddrC<L1, S::CW>{c}, SyncBlock{});
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
    const int gridR = nrows * ((1 << A) / S::LPCR);                                         \
    const int gridC = nrows * (S::NCOL / S::CW);                                            \
    const size_t smC = (smemC_words<A, S::CW>() + 2 * LineCfg<A>::M) * 4;                   \
    const size_t smR = rowpass_smem_bytes<A, B>(0);                                         \
    lf_smem_optin(k_ntt_fwd_R<A, B>, smR);                                                  \
    lf_smem_optin(k_ntt_inv_R<A, B>, smR);                                                  \
    if (!inverse) {                                                                         \
      k_ntt_fwd_C<A, B><<<gridC, S::TC, smC, s>>>(rows, rm, dv);                            \
      k_ntt_fwd_R<A, B><<<gridR, S::TRR, smR, s>>>(rows, rm, dv);                           \
    } else {                                                                                \
      k_ntt_inv_R<A, B><<<gridR, S::TRR, smR, s>>>(rows, rm, dv);                           \
      k_ntt_inv_C<A, B><<<gridC, S::TC, smC, s>>>(rows, rm, dv);                            \
    }                                                                                       \
  }
  LF_DISPATCH_LOGN(ctx->logN, LF_NTT_LAUNCH)
#undef LF_NTT_LAUNCH
  LF_CHECK_LAUNCH();
  return 0;
}
