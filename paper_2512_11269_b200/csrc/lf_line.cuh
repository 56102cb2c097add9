// Register-resident NTT line transforms.
//
// A row of N = 2^L residues is viewed as a 2^L1 x 2^L2 matrix, element e = hi*2^L2 + lo.
// The reference's forward transform (ntt.py:70-86) is a Cooley-Tukey network whose stage s
// pairs elements at distance N/2^(s+1) with twiddle psi_brv[2^s + (e >> (L-s))].  The first
// L1 stages only mix `hi` (one independent 2^L1-point "column line" per lo) and the last L2
// stages only mix `lo` (one "row line" per hi).  In both cases stage k of a line uses twiddle
// index (R << k) + (p >> (LP - k)) where p is the position inside the line and R the line's
// root in the heap-ordered twiddle table: R = 1 for column lines, R = 2^L1 + hi for row lines.
// The inverse (ntt.py:89-105) is the Gentleman-Sande network with the same indexing.
//
// A line of LP stages (M = 2^LP points) is processed by T = 2^floor(LP/2) threads each
// holding E = 2^ceil(LP/2) registers:
//   step 1: thread tl holds positions p = tl + T*j (j < E); runs the first LA = ceil(LP/2)
//           stages entirely in registers (root R).
//   exchange through shared memory.
//   step 2: thread tl holds positions p = tl*E + e (e < E), i.e. G = E/T contiguous groups of
//           T points, each an independent LB = floor(LP/2)-stage sub-transform with root
//           (R << LA) + tl*G + gi.
// Forward: step1 -> exchange -> step2.  Inverse: step2^-1 -> exchange -> step1^-1.
//
// Lazy reduction (forward): a butterfly outputs X + T and X - T + 2q with T = Shoup(Y) in
// [0, 2q), so the bound grows by 2q per stage and only X needs an occasional csub(8q) to stay
// below 16q < 2^32.  The bound is tracked at compile time (units of q).  The inverse uses
// Harvey's butterfly with inputs/outputs in [0, 2q).
#pragma once
#include <type_traits>
#include "lf_arith.cuh"

template <int LP>
struct LineCfg {
  static constexpr int LA = (LP + 1) / 2;
  static constexpr int LB = LP / 2;
  static constexpr int T = 1 << LB;
  static constexpr int E = 1 << LA;
  static constexpr int G = E / T;
  static constexpr int M = 1 << LP;
};

// ---- compile-time bound tracking for the lazy forward butterflies ------------------------
__host__ __device__ constexpr bool fwd_needs_corr(int b) { return b + 2 > 16; }
__host__ __device__ constexpr int fwd_next_bound(int b) { return (fwd_needs_corr(b) ? 8 : b) + 2; }
__host__ __device__ constexpr int fwd_bound_at(int b, int stages) {
  return stages == 0 ? b : fwd_bound_at(fwd_next_bound(b), stages - 1);
}
// bit k set <=> stage k (starting from bound b) must correct X first.  Used through a
// constexpr variable so the per-stage decision folds away after unrolling.
__host__ __device__ constexpr unsigned fwd_corr_mask(int b, int stages) {
  unsigned m = 0;
  for (int k = 0; k < stages; ++k) {
    if (fwd_needs_corr(b)) m |= 1u << k;
    b = fwd_next_bound(b);
  }
  return m;
}

// ---- twiddle sources --------------------------------------------------------------------
// get(depth, node): twiddle {w, w'} of heap node `node`, which sits `depth` levels below the
// line root.  TwGlobal reads the per-prime table in HBM/L2; TwTree reads a CTA's staged copy of
// the subtrees under roots R0 .. R0+span-1 (row passes); TwFlat reads a staged copy of the
// first 2^L1 nodes (column passes, root 1).
struct TwGlobal {
  const uint2* p;
  LF_DEV uint2 get(int, u32 n) const { return __ldg(&p[n]); }
};
// Depths d >= LineCfg<LP>::LA are read in the second phase of a line transform, where the
// threads of a line hold consecutive roots r (at depth LA) and read node (r << k) + blk: the
// staged copy (from LfDev::twfT / twiT) holds them transposed, [blk][r], so a warp's reads hit
// consecutive words instead of 2^k-strided ones (bank conflicts).
template <int LP>
struct TwTree {
  const uint2* s;
  u32 R0;
  int span;
  LF_DEV uint2 get(int d, u32 n) const {
    constexpr int DS = LineCfg<LP>::LA;
    const u32 off = n - (R0 << d);
    const int base = span * ((1 << d) - 1);
    if (d < DS) return s[base + off];
    const int kk = d - DS;
    return s[base + (int)(off & ((1u << kk) - 1)) * (span << DS) + (int)(off >> kk)];
  }
};
// TwTree's transposed layout read straight from the global copy (LfDev::twfT / twiT): the
// CTA's line block starts at root R0 (a multiple of span); consecutive threads of the second
// phase read consecutive entries (fewer L1 sectors than the natural table).
template <int LP>
struct TwGlobalT {
  const uint2* p;
  u32 R0;
  int span;
  LF_DEV uint2 get(int d, u32 n) const {
    constexpr int DS = LineCfg<LP>::LA;
    if (d < DS) return __ldg(&p[n]);
    const u32 off = n - (R0 << d);
    const int kk = d - DS;
    return __ldg(&p[((size_t)R0 << d) + (off & ((1u << kk) - 1)) * (u32)(span << DS) + (off >> kk)]);
  }
};
struct TwFlat {
  const uint2* s;
  LF_DEV uint2 get(int, u32 n) const { return s[n]; }
};

// Stage the subtrees (LP levels) under roots R0..R0+span-1 of table `tab` into smem `dst`
// (span * (2^LP - 1) entries), cooperatively and coalesced.  Caller syncs afterwards.
// Asynchronous variant (cp.async, no register round trip): the copies land while the thread
// goes on issuing its data loads; call cp_async_wait_all() + a barrier before reading.
LF_DEV void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
LF_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <int LP>
LF_DEV void stage_tree_async(uint2* dst, const uint2* __restrict__ tab, u32 R0, int span, int tid,
                             int nthr) {
#pragma unroll
  for (int d = 0; d < LP; ++d) {
    const uint2* src = tab + ((size_t)R0 << d);
    uint2* o = dst + span * ((1 << d) - 1);
    const int n = span << d;
    if ((n & 1) == 0 && (((size_t)R0 << d) & 1) == 0 && ((span * ((1 << d) - 1)) & 1) == 0) {
      for (int i = tid; i < n / 2; i += nthr) cp_async16(o + 2 * i, src + 2 * i);
    } else {
      for (int i = tid; i < n; i += nthr) o[i] = __ldg(&src[i]);
    }
  }
}

// TMA bulk-copy variant (cp.async.bulk, completion on an mbarrier): ONE thread issues one
// bulk copy per tree depth; the other threads keep issuing their data loads.  Call
// tw_bulk_begin from all threads (it contains the barrier that publishes the mbarrier init)
// and tw_bulk_wait from all threads before the first twiddle read.  Depths whose extent is not
// 16-byte aligned (tiny rings only) are copied by the issuing thread directly.
LF_DEV void mbar_wait(unsigned long long* bar, unsigned phase) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  while (!done) {
    asm volatile("{\n\t.reg .pred p;\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(a), "r"(phase) : "memory");
  }
}

template <int LP>
LF_DEV void tw_bulk_begin(uint2* dst, const uint2* __restrict__ tab, u32 R0, int span,
                          unsigned long long* bar) {
  if (threadIdx.x == 0) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    unsigned tx = 0;
#pragma unroll
    for (int d = 0; d < LP; ++d) {
      const uint2* src = tab + ((size_t)R0 << d);
      uint2* o = dst + span * ((1 << d) - 1);
      const unsigned bytes = (unsigned)(span << d) * 8u;
      if ((bytes & 15u) == 0 && ((size_t)src & 15u) == 0 && ((size_t)o & 15u) == 0) tx += bytes;
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(tx) : "memory");
#pragma unroll
    for (int d = 0; d < LP; ++d) {
      const uint2* src = tab + ((size_t)R0 << d);
      uint2* o = dst + span * ((1 << d) - 1);
      const unsigned bytes = (unsigned)(span << d) * 8u;
      if ((bytes & 15u) == 0 && ((size_t)src & 15u) == 0 && ((size_t)o & 15u) == 0) {
        const unsigned so = (unsigned)__cvta_generic_to_shared(o);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(so), "l"(src), "r"(bytes), "r"(a) : "memory");
      } else {
        for (int i = 0; i < (span << d); ++i) o[i] = __ldg(&src[i]);
      }
    }
  }
  __syncthreads();
}
LF_DEV void tw_bulk_wait(unsigned long long* bar) { mbar_wait(bar, 0); }

template <int M>
LF_DEV void stage_flat(uint2* dst, const uint2* __restrict__ tab, int tid, int nthr) {
  for (int i = tid; i < M; i += nthr) dst[i] = __ldg(&tab[i]);
}

// Forward CT sub-transform of 2^K registers.  Input bound BIN (units of q).  DOFF = depth of
// `root` below the line root.  Stages are instantiated one by one (template recursion) so every
// register index is a compile-time constant: a runtime-bounded inner loop would make nvcc demote
// the register array to local memory.
template <int K, int k, int BIN, int DOFF, class TW>
LF_DEV void ct_stage(u32* x, u32 root, const TW& tw, u32 q) {
  constexpr int h = 1 << (K - 1 - k);
  constexpr bool corr = (fwd_corr_mask(BIN, K) >> k) & 1u;
#pragma unroll
  for (int blk = 0; blk < (1 << k); ++blk) {
    const uint2 w = tw.get(DOFF + k, (root << k) + blk);
#pragma unroll
    for (int j = 0; j < h; ++j) {
      u32 X = x[blk * 2 * h + j];
      const u32 Y = x[blk * 2 * h + h + j];
      if (corr) X = csub(X, 8 * q);
      const u32 t = mul_shoup_lazy(Y, w.x, w.y, q);
      x[blk * 2 * h + j] = X + t;
      x[blk * 2 * h + h + j] = X - t + 2 * q;
    }
  }
  if constexpr (k + 1 < K) ct_stage<K, k + 1, BIN, DOFF>(x, root, tw, q);
}

template <int K, int BIN, int DOFF = 0, class TW>
LF_DEV void ct_sub(u32* x, u32 root, const TW& tw, u32 q) {
  static_assert(BIN <= 16, "input bound too large");
  if constexpr (K > 0) ct_stage<K, 0, BIN, DOFF>(x, root, tw, q);
}

// Inverse GS sub-transform of 2^K registers, Harvey butterflies, [0,2q) in and out.
template <int K, int k, int DOFF, class TW>
LF_DEV void gs_stage(u32* x, u32 root, const TW& tw, u32 q) {
  constexpr int h = 1 << (K - 1 - k);
#pragma unroll
  for (int blk = 0; blk < (1 << k); ++blk) {
    const uint2 w = tw.get(DOFF + k, (root << k) + blk);
#pragma unroll
    for (int j = 0; j < h; ++j) {
      const u32 X = x[blk * 2 * h + j];
      const u32 Y = x[blk * 2 * h + h + j];
      x[blk * 2 * h + j] = csub(X + Y, 2 * q);
      x[blk * 2 * h + h + j] = mul_shoup_lazy(X - Y + 2 * q, w.x, w.y, q);
    }
  }
  if constexpr (k > 0) gs_stage<K, k - 1, DOFF>(x, root, tw, q);
}

template <int K, int DOFF = 0, class TW>
LF_DEV void gs_sub(u32* x, u32 root, const TW& tw, u32 q) {
  if constexpr (K > 0) gs_stage<K, K - 1, DOFF>(x, root, tw, q);
}

// Output bound (units of q) of a full forward line with input bound BIN.
template <int LP, int BIN>
struct FwdLineBound {
  static constexpr int step1 = fwd_bound_at(BIN, LineCfg<LP>::LA);
  static constexpr int value = fwd_bound_at(step1, LineCfg<LP>::LB);
};

// Exchange helpers.  `Addr` maps a line position to a shared-memory word index for the
// calling thread's line.  Sync is the barrier covering all threads of a line.
// A warp-synchronous exchange buffer is reused by the next line transform of the same warp, so
// the writes must not overtake the previous reads of other lanes: sync first (the CUDA model
// does not guarantee lockstep; compute-sanitizer racecheck flags the WAR otherwise).  Block /
// group barriers are placed by the calling kernels.
struct SyncBlock {
  LF_DEV void operator()() const { __syncthreads(); }
};
struct SyncWarp {
  LF_DEV void operator()() const { __syncwarp(__activemask()); }
};

template <class Sync>
LF_DEV void xchg_pre(Sync sync) {
  if constexpr (std::is_same<Sync, SyncWarp>::value) sync();
}

template <int LP, class Addr, class Sync>
LF_DEV void xchg_12(u32* x, u32* sm, int tl, Addr addr, Sync sync) {
  using C = LineCfg<LP>;
  xchg_pre(sync);
#pragma unroll
  for (int j = 0; j < C::E; ++j) sm[addr(tl + C::T * j)] = x[j];
  sync();
#pragma unroll
  for (int e = 0; e < C::E; ++e) x[e] = sm[addr(tl * C::E + e)];
}

template <int LP, class Addr, class Sync>
LF_DEV void xchg_21(u32* x, u32* sm, int tl, Addr addr, Sync sync) {
  using C = LineCfg<LP>;
  xchg_pre(sync);
#pragma unroll
  for (int e = 0; e < C::E; ++e) sm[addr(tl * C::E + e)] = x[e];
  sync();
#pragma unroll
  for (int j = 0; j < C::E; ++j) x[j] = sm[addr(tl + C::T * j)];
}

// Forward line: x in step-1 layout (bound BIN) -> step-2 layout (bound FwdLineBound).
// The caller must make sure `sm` is free to overwrite (pre-sync) when needed.
template <int LP, int BIN, class TW, class Addr, class Sync>
LF_DEV void fwd_line(u32* x, u32 root, const TW& tw, u32 q, u32* sm, int tl, Addr addr,
                     Sync sync) {
  using C = LineCfg<LP>;
  ct_sub<C::LA, BIN, 0>(x, root, tw, q);
  xchg_12<LP>(x, sm, tl, addr, sync);
  constexpr int B1 = FwdLineBound<LP, BIN>::step1;
#pragma unroll
  for (int gi = 0; gi < C::G; ++gi)
    ct_sub<C::LB, B1, C::LA>(x + gi * C::T, (root << C::LA) + tl * C::G + gi, tw, q);
}
template <int LP, int BIN, class Addr, class Sync>
LF_DEV void fwd_line(u32* x, u32 root, const uint2* tw, u32 q, u32* sm, int tl, Addr addr,
                     Sync sync) {
  fwd_line<LP, BIN>(x, root, TwGlobal{tw}, q, sm, tl, addr, sync);
}

// Inverse line: x in step-2 layout ([0,2q)) -> step-1 layout ([0,2q)), no N^-1 scaling.
template <int LP, class TW, class Addr, class Sync>
LF_DEV void inv_line(u32* x, u32 root, const TW& tw, u32 q, u32* sm, int tl, Addr addr,
                     Sync sync) {
  using C = LineCfg<LP>;
#pragma unroll
  for (int gi = 0; gi < C::G; ++gi)
    gs_sub<C::LB, C::LA>(x + gi * C::T, (root << C::LA) + tl * C::G + gi, tw, q);
  xchg_21<LP>(x, sm, tl, addr, sync);
  gs_sub<C::LA, 0>(x, root, tw, q);
}
template <int LP, class Addr, class Sync>
LF_DEV void inv_line(u32* x, u32 root, const uint2* tw, u32 q, u32* sm, int tl, Addr addr,
                     Sync sync) {
  inv_line<LP>(x, root, TwGlobal{tw}, q, sm, tl, addr, sync);
}
