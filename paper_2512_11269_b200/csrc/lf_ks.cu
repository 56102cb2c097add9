// Fused hybrid keyswitch pipeline (reference ckks.py:95-140, poly.py:251-287) and the ops
// built on it: hom_mul (ckks.py:182-194), hom_rotate (ckks.py:197-217), rescale
// (ckks.py:220-225).
//
// With N = 2^L1 * 2^L2 (see lf_line.cuh) one keyswitch of x at level l is five kernels:
//   K_A  modup_in     row pass of INTT(x)            x (l+1 rows)           -> T0 (l+1)
//                     [hom_mul: x = a1*a2 formed on load]
//   K_BC bconv_colpass column pass of INTT, exact BConv of each digit onto ext \ G_j,
//                     column pass of the NTT          T0                     -> T1 (beta x ext)
//   K_C  ks_inner     row pass of the NTT of every piece row, automorphism (rotate),
//                     inner product with the key over all digits (64-bit lazy sums);
//                     main rows -> ACC, special rows -> row pass of their INTT -> T2
//   K_BC bconv_colpass (ModDown) column pass of INTT(special rows), BConv onto main primes,
//                     column pass of the NTT          T2 (2 alpha)           -> T3 (2 (l+1))
//   K_E  moddown_out  row pass of the NTT, (acc - conv) * P^-1, epilogue
//                     [hom_mul: + d0/d1; rotate: + sigma_g(b)]            -> out (2 (l+1))
// Every pass works on whole lines held in registers, so each intermediate row crosses HBM
// (or L2) once per kernel boundary.  All kernels take a batch dimension (grid.z).
// Intermediates T0..T3 are stored LINE-TRANSPOSED: inside each 2^L2-word line, element
// p = tl + T*j (the row pass's step-1 order) lives at word tl*E + j, so the row kernels move
// them with contiguous 16-byte accesses; the column kernels are layout-agnostic (every column
// is transformed identically), they only see a permuted column order.
#include "lf_ntt.cuh"
#include "lf_bconv.cuh"
#include "lf_plan.h"
#include "lf_ops.h"
#include "lf_umma.cuh"

#define LF_BC_MAXG 16
#define LF_LAUNCH_CHECK(call)                                                  \
  do {                                                                         \
    cudaError_t e__ = (call);                                                  \
    if (e__ != cudaSuccess) {                                                  \
      lf_set_error("%s:%d: launch: %s", __FILE__, __LINE__, cudaGetErrorString(e__)); \
      return 3;                                                                \
    }                                                                          \
  } while (0)
#define LF_MAXB 64     // batch instances per launch (per-instance key / galois element)

// hom_mul over a list of independent operand pairs (instance b: ct1 at c1[b] with p1[b] rows per
// polynomial, ct2 at c2[b] with p2[b]): products of different ciphertexts at one level run as ONE
// batch without gathering them into a contiguous block first.
struct MulList {
  const u32* c1[LF_MAXB];
  const u32* c2[LF_MAXB];
  int p1[LF_MAXB], p2[LF_MAXB];
  long long addb[LF_MAXB];   // integer added to every b residue of the product (0: none)
  int on;
};

LF_DEV void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

struct BcGroupDev;
LF_DEV int bc_src_row(int row0, int sr, int rstride) { return row0 + (sr & 0xFFFF) + (sr >> 16) * rstride; }

struct BcArgs {
  const u32* src;
  u32* dst;
  size_t src_bs, dst_bs;     // batch strides (words)
  int ngroups, tsplit;
  // limb-sharded pipeline: source rows gathered from k ranks; src_rows[i] = (rank << 16) | slot
  // and the row is slot + rank * src_rstride (0: plain row indices)
  int src_rstride;
  BcGroupDev g[LF_BC_MAXG];
};

// ---------------------------------------------------------------------------------------
// K_A: row pass of the inverse NTT.  MODE 0: rows of x; MODE 1: rows of a1*a2 (tensor d2).
template <int L1, int L2, int MODE>
__global__ void __launch_bounds__(NttShape<L1, L2>::TRR)
k_modup_in(const u32* __restrict__ x, const u32* __restrict__ x2, u32* __restrict__ T0,
           size_t x_bs, size_t t_bs, int nrows, LfDev dv, int rpp, int src_rs, int src_r0, int pbase,
           int nbatch, int bpc, int pstep, size_t x2_bs, int src_rs2, MulList ml) {
  using S = NttShape<L1, L2>;
  using C = LineCfg<L2>;
  constexpr int GROUPS = (1 << L1) / S::LPCR;
  extern __shared__ __align__(16) u32 sm[];
  const int tl = threadIdx.x % C::T, ln = threadIdx.x / C::T;
  const int row = blockIdx.x / GROUPS, hi0 = (blockIdx.x % GROUPS) * S::LPCR, hi = hi0 + ln;
  // row r: source row (r / rpp) * src_rs + src_r0 + r % rpp, prime pbase + pstep * (r % rpp)
  const int pi = pbase + pstep * (row % rpp);
  const PrimeK pk = dv.pk[pi];
  uint2* tws = reinterpret_cast<uint2*>(sm);
  __shared__ unsigned long long twbar;
  lf_pdl_trigger();
  tw_bulk_begin<L2>(tws, dv.twiT + ((size_t)pi << (L1 + L2)), (1u << L1) + hi0, S::LPCR, &twbar);
  lf_pdl_wait();
  // instances blockIdx.z*bpc .. +bpc-1 share the staged twiddles
  const size_t roff = ((size_t)((row / rpp) * src_rs + src_r0 + row % rpp) << (L1 + L2)) + ((size_t)hi << L2);
  const int b0 = blockIdx.z * bpc, b1 = min(nbatch, b0 + bpc);
#pragma unroll 1
  for (int b = b0; b < b1; ++b) {
    const size_t off = (size_t)b * x_bs + roff;
    u32 v[C::E];
    if (MODE == 1 && ml.on)          // a1 rows of instance b (row < level + 1: roff = row's offset)
      load_row_step2<L2>(v, ml.c1[b] + ((size_t)ml.p1[b] << (L1 + L2)) + roff, tl);
    else
      load_row_step2<L2>(v, x + off, tl);
    if (MODE == 1) {
      u32 w[C::E];
      if (ml.on)
        load_row_step2<L2>(w, ml.c2[b] + ((size_t)ml.p2[b] << (L1 + L2)) + roff, tl);
      else
        load_row_step2<L2>(w, x2 + (size_t)b * x2_bs + (((size_t)((row / rpp) * src_rs2 + src_r0 + row % rpp) << (L1 + L2)) + ((size_t)hi << L2)), tl);
#pragma unroll
      for (int e = 0; e < C::E; ++e) v[e] = mulmod(v[e], w[e], pk);
    }
    if (b + 1 < b1 && !(MODE == 1 && ml.on)) prefetch_l1(x + off + x_bs + (size_t)tl * C::E);
    if (b == b0) {
      tw_bulk_wait(&twbar);
    } else {
      __syncwarp();
    }
    inv_line<L2>(v, (1u << L1) + hi, TwTree<L2>{tws, (1u << L1) + hi0, S::LPCR}, pk.q,
                 rowpass_xs<L1, L2>(sm), tl, AddrR<L2>{ln * pitchR<L2>()}, SyncWarp{});
    store_row_step2<L2>(v, T0 + (size_t)b * t_bs + ((size_t)row << (L1 + L2)) + ((size_t)hi << L2), tl);
  }
}

// ---------------------------------------------------------------------------------------
// K_BC: column pass of INTT on k source rows, exact BConv, column pass of NTT per target.
LF_DEV u32 bconv_u_smem(const u32* Yp, int ystride, const BconvDev& B) {
  double v = 0.0;
  for (int i = 0; i < B.k; ++i) v = fma((double)Yp[i * ystride], B.inv_s[i], v);
  const double r = rint(v);
  if (fabs(v - r) >= 0x1p-40) return (u32)floor(v);
  u32 y[64];
  bool z = true;
  for (int i = 0; i < B.k; ++i) {
    y[i] = Yp[i * ystride];
    z &= y[i] == 0;
  }
  if (z) return 0;
  return bconv_u_exact(y, B, (u32)r);
}

// Shared-memory tile of the converted sources: Y[i][tl][c][E].  A thread's E values are
// contiguous (LDS.128/STS.128); the four 16-byte chunks of each 16-word block are rotated by
// (c >> 1) so the 8 threads of a quarter-warp (consecutive c) hit 8 disjoint bank quads.
template <int L1>
struct YTile {
  static constexpr int E = LineCfg<L1>::E;
  static constexpr int T = LineCfg<L1>::T;
};

// Barrier over one thread group (named barrier when the group is whole warps; otherwise the
// CTA has a single group and __syncthreads is used).
template <bool NAMED>
struct SyncGroup {
  int id, n;
  LF_DEV void operator()() const {
    if (NAMED) asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
    else __syncthreads();
  }
};

// physical word offset of logical 4-word chunk lq of a thread slot
LF_DEV int ychunk(int lq, int rot) { return 4 * ((lq + rot) & 3) + 16 * (lq >> 2); }

template <int E>
LF_DEV void y_load(u32* v, const u32* slot, int rot) {
  if constexpr (E % 16 == 0) {
#pragma unroll
    for (int q = 0; q < E / 4; ++q) {
      const uint4 t = *reinterpret_cast<const uint4*>(slot + ychunk(q, rot));
      v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < E; ++q) v[q] = slot[q];
  }
}
template <int E>
LF_DEV void y_store(u32* slot, const u32* v, int rot) {
  if constexpr (E % 16 == 0) {
#pragma unroll
    for (int q = 0; q < E / 4; ++q)
      *reinterpret_cast<uint4*>(slot + ychunk(q, rot)) =
          make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  } else {
#pragma unroll
    for (int q = 0; q < E; ++q) slot[q] = v[q];
  }
}

// x < 2^64 -> [0, 4q) (lazy; the forward NTT accepts it with input bound 4)
LF_DEV u32 reduce64_lazy4(u64 x, const PrimeK& k) {
  const u32 hi = (u32)(x >> 32), lo = (u32)x;
  return mul_shoup_lazy(hi, k.r32, k.r32p, k.q) + reduce32_lazy(lo, k);
}

// Multiply-accumulate of one target over the K source tiles of this thread, for the EH
// positions [h*EH, (h+1)*EH) of its E: acc[j] += y_i[j] * w[i] (64-bit lazy sums, exact:
// K * 2^56 < 2^64).  KEX > 0: K known at compile time (fully unrolled, weights in registers);
// KEX == 0: runtime K, one source per iteration with the next weight prefetched.
template <int E, int EH, int KEX, int YI>
LF_DEV void bconv_mac(u64* acc, const u32* const* yq, const u32* wrow, int k, const u32* slot0,
                      int h) {
  if constexpr (E % 16 == 0) {
    constexpr int KK = KEX > 0 ? KEX : 1;
#pragma unroll (KEX > 0 ? KK : 1)
    for (int i = 0; i < (KEX > 0 ? KEX : k); ++i) {
      const u32 wv = wrow[i];                      // shared memory, warp-uniform address
#pragma unroll
      for (int q = 0; q < EH / 4; ++q) {
        const int lq = h * (EH / 4) + q;
        const uint4 tv = *reinterpret_cast<const uint4*>(yq[lq & 3] + i * YI + 16 * (lq >> 2));
        acc[4 * q + 0] += (u64)tv.x * wv;
        acc[4 * q + 1] += (u64)tv.y * wv;
        acc[4 * q + 2] += (u64)tv.z * wv;
        acc[4 * q + 3] += (u64)tv.w * wv;
      }
    }
  } else {
#pragma unroll 1
    for (int i = 0; i < k; ++i) {
      const u32 wv = wrow[i];
      const u32* slot = slot0 + (size_t)i * YI + h * EH;
#pragma unroll
      for (int j = 0; j < EH; ++j) acc[j] += (u64)slot[j] * wv;
    }
  }
}

#ifndef LF_BC_MINB
#define LF_BC_MINB 2
#endif
template <int L1, int L2, int CW, int KMAX, int TG, int KEX>
__global__ void __launch_bounds__(TG * CW * LineCfg<L1>::T, (TG * CW * LineCfg<L1>::T) >= 512 ? LF_BC_MINB : 1)
k_bconv_colpass(BcArgs A, LfDev dv, int kmax, int nbatch) {
  using C = LineCfg<L1>;
  constexpr int E = C::E, T = C::T;
  constexpr int GT = CW * T;
  constexpr int NCT = (1 << L2) / CW;
  constexpr int logN = L1 + L2;
  constexpr int YI = T * CW * E;                               // words per source
  extern __shared__ __align__(16) u32 sm[];
  const int grp = threadIdx.x / GT, lt = threadIdx.x % GT;
  const int c = lt % CW, tl = lt / CW;
  const int rot = c >> 1;
  // blockIdx.x = ((group * NCT + ct) * nbatch + b) * tsplit + ts: the tsplit CTAs that share one
  // (group, column tile, instance) are consecutive and form a thread-block cluster.
  int bid = blockIdx.x;
  const int ts = bid % A.tsplit;
  bid /= A.tsplit;
  const int b = bid % nbatch;
  bid /= nbatch;
  const int ct = bid % NCT;
  const BcGroupDev& G = A.g[bid / NCT];
  const BconvDev& B = G.B;
  // k: this group's sources; kw: sources the MAC loop runs over (KEX pads smaller groups of
  // a non-uniform launch with zero tiles and zero weights)
  const int k = B.k;
  const int kw = KEX > 0 ? KEX : k;
  const int col = ct * CW + c;
  u32* Ybase = sm + (size_t)(tl * CW + c) * E;
  u32* X = sm + (size_t)kmax * YI + grp * smemC_words<L1, CW>();
  u32* Wsm = sm + (size_t)kmax * YI + TG * smemC_words<L1, CW>();    // weights of [t0, t1)
  const u32* src = A.src + (size_t)b * A.src_bs;
  u32* dst = A.dst + (size_t)b * A.dst_bs;
  const AddrC<L1, CW> addr{c};
  static_assert(TG == 1 || GT % 32 == 0, "thread groups must be whole warps");
  const SyncGroup<GT % 32 == 0> gsync{1 + grp, GT};

  const int chunk = (B.m + A.tsplit - 1) / A.tsplit;
  const int t0 = ts * chunk, t1 = min(B.m, t0 + chunk);
  lf_pdl_trigger();
  if (kw == k) {
    for (int w = threadIdx.x; w < (t1 - t0) * k; w += blockDim.x) Wsm[w] = __ldg(&B.w[(size_t)t0 * k + w]);
  } else {
    for (int w = threadIdx.x; w < (t1 - t0) * kw; w += blockDim.x) {
      const int tt = w / kw, i = w - tt * kw;
      Wsm[w] = i < k ? __ldg(&B.w[(size_t)(t0 + tt) * k + i]) : 0u;
    }
  }
  lf_pdl_wait();

  // phase 1: INTT column pass of each source row, sources split over the groups and (when the
  // target range is split over a cluster) over the cluster's CTAs; the other CTAs' converted
  // source tiles are then pulled through distributed shared memory instead of recomputed.
  const int cl = A.tsplit;
  for (int i = ts + cl * grp; i < kw; i += cl * TG) {
    if (i >= k) {                                      // padding tile (block-uniform branch)
      u32 z[E];
#pragma unroll
      for (int j = 0; j < E; ++j) z[j] = 0;
      y_store<E>(Ybase + (size_t)i * YI, z, rot);
      continue;
    }
    const int pi = B.src_pi[i];
    const PrimeK pk = dv.pk[pi];
    u32 x[E];
    load_col_step2<L1, L2>(x, src + ((size_t)bc_src_row(G.src_row0, G.src_rows[i], A.src_rstride) << logN) + col, tl);
    inv_line<L1>(x, 1u, TwGlobalT<L1>{dv.twiT + ((size_t)pi << logN), 1u, 1}, pk.q, X, tl, addr, gsync);
    const u32 ci = B.c[i], cpi = B.cp[i];
#pragma unroll
    for (int j = 0; j < E; ++j) x[j] = mul_shoup(x[j], ci, cpi, pk.q);
    y_store<E>(Ybase + (size_t)i * YI, x, rot);
    gsync();
  }
  if (cl > 1) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    for (int i = 0; i < kw; ++i) {
      const int r = i % cl;
      if (r == ts) continue;
      for (int v = threadIdx.x; v < YI / 4; v += blockDim.x) {
        u32* loc = sm + (size_t)i * YI + 4 * v;
        const unsigned la = (unsigned)__cvta_generic_to_shared(loc);
        unsigned ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(r));
        uint4 q;
        asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w) : "r"(ra) : "memory");
        *reinterpret_cast<uint4*>(loc) = q;
      }
    }
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");   // done reading peers
  }
  __syncthreads();

  // phase 2: exact overflow counts u (< 64) for this thread's E positions, packed 4 per word
  u32 up[(E + 3) / 4];
  {
    double v[E];
#pragma unroll
    for (int j = 0; j < E; ++j) v[j] = 0.0;
#pragma unroll 1
    for (int i = 0; i < k; ++i) {
      u32 y[E];
      y_load<E>(y, Ybase + (size_t)i * YI, rot);
      const double is = B.inv_s[i];
#pragma unroll
      for (int j = 0; j < E; ++j) v[j] = fma((double)y[j], is, v[j]);
    }
#pragma unroll
    for (int w = 0; w < (E + 3) / 4; ++w) up[w] = 0;
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const double r = rint(v[j]);
      u32 uj;
      if (fabs(v[j] - r) >= 0x1p-40) {
        uj = (u32)floor(v[j]);
      } else {
        u32 yy[64];
        bool z = true;
        for (int i = 0; i < k; ++i) {
          const u32* slot = Ybase + (size_t)i * YI;
          yy[i] = (E % 16 == 0) ? slot[ychunk(j / 4, rot) + (j % 4)] : slot[j];
          z &= yy[i] == 0;
        }
        uj = z ? 0u : bconv_u_exact(yy, B, (u32)r);
      }
      up[j / 4] |= uj << (8 * (j % 4));
    }
  }

  // phase 3: targets of this split, round-robin over the groups: BConv -> NTT column pass
  const u32* yq[4];                                    // rotated chunk bases (no per-load math)
#pragma unroll
  for (int q = 0; q < 4; ++q) yq[q] = Ybase + 4 * ((q + rot) & 3);
#pragma unroll 1
  for (int t = t0 + grp; t < t1; t += TG) {
    const int pi = B.tgt_pi[t];
    const PrimeK pk = dv.pk[pi];
    const u32 ns = B.negS[t];
    const u32* wrow = Wsm + (t - t0) * kw;
    constexpr int EH = E >= 16 ? E / 2 : E;
    u32 x[E];
#pragma unroll
    for (int h = 0; h < E / EH; ++h) {
      u64 acc[EH];
#pragma unroll
      for (int j = 0; j < EH; ++j)
        acc[j] = (u64)((up[(h * EH + j) / 4] >> (8 * ((h * EH + j) % 4))) & 0xFFu) * ns;
      bconv_mac<E, EH, KEX, YI>(acc, yq, wrow, kw, Ybase, h);
#pragma unroll
      for (int j = 0; j < EH; ++j) x[h * EH + j] = reduce64_lazy4(acc[j], pk);
    }
    fwd_line<L1, 4>(x, 1u, TwGlobalT<L1>{dv.twfT + ((size_t)pi << logN), 1u, 1}, pk.q, X, tl, addr, gsync);
    store_col_step2<L1, L2>(x, dst + ((size_t)(G.dst_row0 + G.dst_rows[t]) << logN) + col, tl);
    gsync();
  }
  if (cl > 1) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");   // peers done with my tile
}

// ---------------------------------------------------------------------------------------
// K_BC on the 5th-generation tensor cores (tcgen05.mma kind::i8, accumulators in TMEM).
//
// The base-conversion MAC of a target t over the k converted sources, Σ_i y_i·w_ti − u·S, is
// computed mod t as a u8 x u8 -> s32 GEMM: with y_i = Σ_a y_ia 2^(8a) (bytes) and the weights
// pre-multiplied and split on the host, w'_tiab = byte b of 2^(8a) w_ti mod t,
//     S_tb = Σ_(i,a) y_ia w'_tiab  (+ u · byte b of negS_t),     X_t = Σ_b S_tb 2^(8b)
// and X_t ≡ Σ_i y_i w_ti + u·negS_t (mod t), X_t < 2^46.  The A operand (one row per
// coefficient, K = 4k+1 bytes: the k sources as little-endian u32 and u) IS the source tile:
// phase 1 writes the converted sources straight into the UMMA canonical layout.  M-tile e
// (128 rows) holds element e of every thread of a 128-thread group, so TMEM lane lt is the
// coefficient thread lt of every group needs: each group reads 4 columns per element for its
// own target.  One CTA per SM: 8 groups (1024 threads) x 8 targets per round, 16 M-tiles x
// (8 targets x 4 bytes) = 512 TMEM columns; the MMAs of round r+1 run during the NTT column
// passes of round r.  Replaces 10 IMAD.WIDE per target element (the fmaheavy-bound part of
// k_bconv_colpass) with ~6 ALU ops and a quarter of a tcgen05.ld.
#ifdef LF_BC_TRACE
// Phase timestamps of two CTAs (experiment builds only: -DLF_BC_TRACE): recorded into shared
// memory by thread 0 of each group, printed after the kernel's work.
#define LF_TR_ON (blockIdx.x == 0 || blockIdx.x == 2000)
#define LF_TR(slot) do { if (LF_TR_ON && (threadIdx.x % 128) == 0 && tr_n < 48) { \
    tr_t[threadIdx.x / 128][tr_n] = clock64(); tr_c[threadIdx.x / 128][tr_n++] = slot; } } while (0)
#else
#define LF_TR(slot) do {} while (0)
#endif
template <int L1, int L2, int KB, bool UEPI>
__global__ void __launch_bounds__(1024, 1)
k_bconv_tc(BcArgs A, LfDev dv, int nbatch, int wbytes) {
  using C = LineCfg<L1>;
  constexpr int E = C::E, T = C::T;
  constexpr int CW = 8, TG = 8, GT = CW * T;
  static_assert(GT == 128 && E == 16, "k_bconv_tc expects 16 x 16 column lines");
  constexpr int NCT = (1 << L2) / CW;
  constexpr int logN = L1 + L2;
  constexpr int SBO = KB / 16 * 128;            // bytes per 8-row group of the A operand
  constexpr int MT = 16 * SBO;                  // bytes per M-tile (128 rows)
  constexpr int ABYTES = E * MT + 128;          // + tail met by the aliased 4th K-chunk (KB = 48)
  extern __shared__ __align__(1024) unsigned char smb[];
  __shared__ uint64_t mbar;                     // MMA completion of the current round
  __shared__ uint32_t tbase_s;
  __shared__ double invs_sm[16];                // 1 / s_i of the sources (phase 2)
  __shared__ unsigned char u_sm[UEPI ? 16 * 128 : 1];   // overflow counts when 4k = KB (epilogue term)
#ifdef LF_BC_TRACE
  __shared__ long long tr_t[8][48];
  __shared__ char tr_c[8][48];
  int tr_n = 0;
#endif
  unsigned char* As = smb;
  unsigned char* Ws = smb + ABYTES;
  const int grp = threadIdx.x / GT, lt = threadIdx.x % GT;
  const int c = lt % CW, tl = lt / CW;
  u32* X = reinterpret_cast<u32*>(Ws + wbytes) + grp * smemC_words<L1, CW>();
  int bid = blockIdx.x;
  const int ts = bid % A.tsplit;
  bid /= A.tsplit;
  const int b = bid % nbatch;
  bid /= nbatch;
  const int ct = bid % NCT;
  const BcGroupDev& G = A.g[bid / NCT];
  const BconvDev& B = G.B;
  const int k = B.k;
  const int col = ct * CW + c;
  const u32* src = A.src + (size_t)b * A.src_bs;
  u32* dst = A.dst + (size_t)b * A.dst_bs;
  const AddrC<L1, CW> addr{c};
  const SyncGroup<true> gsync{1 + grp, GT};
  // this thread's row inside an M-tile: byte offset of 16-byte K-chunk 0
  const int rowoff = (lt / 8) * SBO + (lt % 8) * 16;
  auto yword = [&](int e, int i) -> u32* {
    return reinterpret_cast<u32*>(As + e * MT + rowoff + (i / 4) * 128 + (i % 4) * 4);
  };

  // targets of this CTA: an even-aligned chunk (target pairs are 512-byte operand blocks)
  const int chunk = ((B.m + A.tsplit - 1) / A.tsplit + 1) & ~1;
  const int t0 = min(B.m, ts * chunk), t1 = min(B.m, t0 + chunk);
  const int nrounds = (t1 - t0 + TG - 1) / TG;
  lf_pdl_trigger();
  {   // weights of [t0, t1) -> Ws (zero beyond), TMEM, mbarrier
    const uint4* wsrc = reinterpret_cast<const uint4*>(B.w8 + (size_t)t0 * 256);
    const int nw = (t1 - t0 + 1) / 2 * 32, nz = nrounds * TG / 2 * 32;
    uint4* wd = reinterpret_cast<uint4*>(Ws);
    for (int v = threadIdx.x; v < nz; v += blockDim.x) wd[v] = v < nw ? __ldg(wsrc + v) : make_uint4(0, 0, 0, 0);
    if (threadIdx.x < 32) tmem_alloc(&tbase_s, 512);
    if (threadIdx.x == 0) {
      mbar_init(&mbar, 1);
    }
    if (threadIdx.x < k) invs_sm[threadIdx.x] = B.inv_s[threadIdx.x];
  }
  lf_pdl_wait();

  // phase 1: INTT column pass of each source, times c_i, into the A operand (rows = lanes).
  // (A remainder of k % 8 sources run with all 1024 threads per source, one butterfly per
  // thread and stage through shared memory, measured slower than one group per source.)
  LF_TR('1');
  const int cl = A.tsplit;
  for (int i = ts + cl * grp; i < k; i += cl * TG) {
    const int pi = B.src_pi[i];
    const PrimeK pk = dv.pk[pi];
    u32 x[E];
    load_col_step2<L1, L2>(x, src + ((size_t)bc_src_row(G.src_row0, G.src_rows[i], A.src_rstride) << logN) + col, tl);
    LF_TR('l');
    inv_line<L1>(x, 1u, TwGlobalT<L1>{dv.twiT + ((size_t)pi << logN), 1u, 1}, pk.q, X, tl, addr, gsync);
    LF_TR('i');
    const u32 ci = B.c[i], cpi = B.cp[i];
#pragma unroll
    for (int e = 0; e < E; ++e) *yword(e, i) = mul_shoup(x[e], ci, cpi, pk.q);
    gsync();
  }
  LF_TR('E');
  if (cl > 1) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    for (int i = 0; i < k; ++i) {
      const int r = i % cl;
      if (r == ts) continue;
      for (int v = threadIdx.x; v < E * GT; v += blockDim.x) {
        const int e = v / GT, l2 = v % GT;
        u32* loc = reinterpret_cast<u32*>(As + e * MT + (l2 / 8) * SBO + (l2 % 8) * 16 + (i / 4) * 128 + (i % 4) * 4);
        const unsigned la = (unsigned)__cvta_generic_to_shared(loc);
        unsigned ra, q;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(r));
        asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(q) : "r"(ra) : "memory");
        *loc = q;
      }
    }
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");   // done reading peers
  }
  __syncthreads();

  // phase 2: exact overflow count u of each element (only group 0's 128 threads hold distinct
  // rows; the 8 groups split the 16 M-tiles, two per thread) -> K-row 4k of the A operand.
  // The two elements' fp64 sums run as independent chains over 16-byte source chunks (a
  // quarter-warp reads 128 contiguous bytes: conflict-free); any summation order is exact here
  // (the 2^-40 risk window dwarfs the rounding of k <= 11 terms).
  static_assert(E == 2 * TG, "two M-tiles per thread in phase 2");
  const bool u_epi = UEPI && 4 * k + 1 > KB;       // k = KB / 4 sources fill every K-byte
  {
    double v[2] = {0.0, 0.0};
    const uint4* yc[2] = {reinterpret_cast<const uint4*>(yword(grp, 0)),
                          reinterpret_cast<const uint4*>(yword(grp + TG, 0))};
#pragma unroll 1
    for (int j = 0; 4 * j < k; ++j) {
      const uint4 a = yc[0][8 * j], b = yc[1][8 * j];
      const u32 av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (4 * j + q < k) {
          const double is = invs_sm[4 * j + q];
          v[0] = fma((double)av[q], is, v[0]);
          v[1] = fma((double)bv[q], is, v[1]);
        }
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = grp + h * TG;
      const double r = rint(v[h]);
      u32 uj;
      if (fabs(v[h] - r) >= 0x1p-40) {
        uj = (u32)floor(v[h]);
      } else {
        u32 yy[64];
        bool z = true;
        for (int i = 0; i < k; ++i) { yy[i] = *yword(e, i); z &= yy[i] == 0; }
        uj = z ? 0u : bconv_u_exact(yy, B, (u32)r);
      }
      if (u_epi) u_sm[e * 128 + lt] = (unsigned char)uj;
      else *yword(e, k) = uj;
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase_s;
  const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(As), w0 = (uint32_t)__cvta_generic_to_shared(Ws);
  // One MMA set per round: 8 targets x 4 byte columns (N = 32) over the 16 M-tiles.  (Two
  // independent N = 16 sets measured slower: the tensor core re-streams the whole A operand
  // from shared memory per MMA, so halving N doubles the operand traffic.)
  constexpr uint32_t IDESC = umma_idesc_u8(128, 32);
  auto issue = [&](int r) {
#pragma unroll 1
    for (int e = 0; e < E; ++e)
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2)
        umma_i8(tmem + 32 * e, umma_sdesc(a0 + e * MT + 256 * s2, 128, SBO),
                umma_sdesc(w0 + r * 2048 + 256 * s2, 128, 512), IDESC, s2 > 0);
    umma_commit(&mbar);
  };
  LF_TR('U');
  if (threadIdx.x == 0 && nrounds > 0) issue(0);

  // phase 3: per round, group g takes target t0 + 8 r + g: S_b from TMEM -> X mod t (lazy) ->
  // NTT column pass -> destination row.  A CTA barrier after the TMEM reads frees the
  // accumulators for round r + 1's MMAs.  (Letting the last warp to arrive on an acq_rel
  // shared counter issue them instead, without a barrier, gave no speed-up and produced wrong
  // accumulators in rare launches: the tcgen05 ordering needs the full barrier.)
  const uint32_t tlane = tmem + ((uint32_t)(32 * ((threadIdx.x / 32) % 4)) << 16) + 4 * grp;
#pragma unroll 1
  for (int r = 0; r < nrounds; ++r) {
    const int t = t0 + TG * r + grp;
    const bool active = t < t1;                          // uniform over the group's 4 warps
    PrimeK pk;
    if (active) pk = dv.pk[B.tgt_pi[t]];
    LF_TR('r');
    mbar_wait(&mbar, r & 1);
    tc_fence_after();
    LF_TR('m');
    u32 x[E];
    if (active) {
      const u32 nsu = u_epi ? B.negS[t] : 0u;
#pragma unroll
      for (int h = 0; h < E / 4; ++h) {
        u32 s[4][4];
#pragma unroll
        for (int j = 0; j < 4; ++j) tmem_ld4(tlane + 32 * (4 * h + j), s[j][0], s[j][1], s[j][2], s[j][3]);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const u32 lo = s[j][0] + (s[j][1] << 8), z = s[j][2] + (s[j][3] << 8);
          u64 X = (u64)lo + ((u64)z << 16);
          if (u_epi) X += (u64)u_sm[(4 * h + j) * 128 + lt] * nsu;
          x[4 * h + j] = reduce64_lazy4(X, pk);
        }
      }
    }
    tc_fence_before();
    __syncthreads();                                     // TMEM free for the next round
    if (threadIdx.x == 0 && r + 1 < nrounds) {
      tc_fence_after();
      issue(r + 1);
    }
    LF_TR('d');
    if (active) {
      fwd_line<L1, 4>(x, 1u, TwGlobalT<L1>{dv.twfT + ((size_t)B.tgt_pi[t] << logN), 1u, 1}, pk.q, X, tl, addr, gsync);
      LF_TR('n');
      store_col_step2<L1, L2>(x, dst + ((size_t)(G.dst_row0 + G.dst_rows[t]) << logN) + col, tl);
    }
  }
  LF_TR('z');
#ifdef LF_BC_TRACE
  if (LF_TR_ON && (threadIdx.x % 128) == 0)
    for (int i = 0; i < tr_n; ++i)
      printf("TR b%d g%d %c %lld\n", blockIdx.x, threadIdx.x / 128, tr_c[threadIdx.x / 128][i],
             tr_t[threadIdx.x / 128][i] - tr_t[threadIdx.x / 128][0]);
#endif
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
  if (cl > 1) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");   // peers done with my tile
}

// ---------------------------------------------------------------------------------------
// K_C: inner product over digits (+ automorphism), ACC / T2 outputs.
struct KsInnerArgs {
  const u32* T1;       // beta x ext rows
  const u32* x;        // own rows source (x, or a1 for the tensor mode)
  const u32* x2;       // a2 (tensor mode)
  u32* acc;            // 2 x (l+1) rows
  u32* T2;             // 2 x alpha rows
  size_t t1_bs, x_bs, acc_bs, t2_bs;
  const u32* rowk;     // plan: per main row {s, s', pinv, pinv'}
  int level, d, beta, L, alpha, R;
  int nbatch;          // grid.x = batch (fastest, so a key line is reused from L2) x lines
  int pre;             // 1: T1 holds finished eval-domain pieces (natural layout, k_pieces ran once
                       //    for a hoisted batch): no row NTT here, only the permuted load + MAC
  int ext_out;         // 1: write (P*sigma_g(b) + acc_b, acc_a) over the extended basis, eval domain,
                       //    into acc (2 x ext rows per instance) and skip ModDown (hoisted-ModDown BSGS)
  const u32* eb;       // ext_out: ct.b rows (shared by all instances), P mod q_t table
  const u32* pmod;
  int fuse_nd;         // tensor mode fused with a rescale by fuse_nd primes: the top fuse_nd main
                       // rows get + P*(d0, d1) and join the special rows in T2 (t2_rows per poly)
  int t2_rows;
  const u32 *c1, *c2;  // fuse_nd: ct1, ct2 (b rows then a rows, c_ne rows per poly)
  size_t c_bs, c2_bs;  // instance strides of ct1 / ct2
  int c_ne, c2_ne;     // rows per polynomial of ct1 / ct2
  size_t x2_bs;        // instance stride of x2
  MulList ml;          // XMODE 1 with ml.on: per-instance operands (x, x2, c1, c2 derived)
  const u32* keyp[LF_MAXB];   // per instance: (d, 2, R, N) key
  u32 gs[LF_MAXB];            // per instance: galois element (GALOIS mode)
  // limb-sharded pipeline (null tmap: one device holds every row): CTA row r of this rank's
  // extended rows is ext position tmap[r] and key row kmap[r]; storage holds n_main_st main
  // rows then the special rows, ext_st rows per digit in T1
  const int* tmap;
  const int* kmap;
  int n_main_st, ext_st;
};

#ifndef LF_KSI_MINB
#define LF_KSI_MINB 2
#endif
#ifndef LF_KSI_PF
// L1 prefetch one digit ahead: 1 the piece line, 2 the key lines.  Keys are read by every
// instance of the batch (L2-resident); prefetching them into L1 as well evicts the pieces:
// 30.9 us (1) against 31.7 (3), 32.1 (0), 32.4 (2) per C2 keyswitch at batch 32.
#define LF_KSI_PF 1
#endif
// GMODE 0: no automorphism; 1: sigma_g applied to every digit's piece line before the MAC;
// 2: permuted keys (keys stored as K o sigma_g^-1, lf_permute_rotation_key): the MAC runs in
//    the source frame on unpermuted lines, and only the two accumulators are permuted at the end.
template <int L1, int L2, int GMODE, int XMODE>
__global__ void __launch_bounds__(NttShape<L1, L2>::TRR, LF_KSI_MINB)
k_ks_inner(KsInnerArgs A, LfDev dv) {
  constexpr bool GALOIS = GMODE != 0;
  constexpr bool KP = GMODE == 2;
  using S = NttShape<L1, L2>;
  using C = LineCfg<L2>;
  constexpr int M2 = C::M;
  constexpr int logN = L1 + L2;
  constexpr int BIN = S::FWD_C_OUT;
  extern __shared__ u32 sm[];
  const int tl = threadIdx.x % C::T, ln = threadIdx.x / C::T;
  const int groups = (1 << L1) / S::LPCR;
  const size_t b = blockIdx.x % A.nbatch;
  const int bl = blockIdx.x / A.nbatch;
  const int r = bl / groups;                                 // storage row
  const int t = A.tmap ? A.tmap[r] : r;                      // ext position
  const int hi = (bl % groups) * S::LPCR + ln;
  const int l = A.level;
  const bool is_main = t <= l;
  const int pi = is_main ? t : A.L + 1 + (t - l - 1);       // prime index
  const int kr = A.kmap ? A.kmap[r] : pi;                    // key row
  const PrimeK pk = dv.pk[pi];
  const int ext = A.tmap ? A.ext_st : l + 1 + A.alpha;      // T1 rows per digit
  const int nms = A.tmap ? A.n_main_st : l + 1;             // main rows in storage
  const int rs = is_main ? r : r - nms;                      // storage index within main / special
  u32* xs = rowpass_xs<L1, L2>(sm) + ln * (pitchR<L2>() + M2);
  u32* perm_buf = xs + pitchR<L2>();
  const AddrR<L2> addr{0};

  int hs = hi;
  const u32 gal = A.gs[b];
  const u32* keyb = A.keyp[b];
  if (GALOIS) hs = (int)(auto_src_index((u32)hi << L2, gal, logN) >> L2);
  // twiddle subtrees of this CTA's source lines.  The automorphism maps an aligned block of
  // LPCR lines onto an aligned block of LPCR lines, so one staged block serves all of them.
  uint2* tws = reinterpret_cast<uint2*>(sm);
  int hi0s = (bl % groups) * S::LPCR;
  if (GALOIS)
    hi0s = (int)((auto_src_index((u32)hi0s << L2, gal, logN) >> L2) / S::LPCR) * S::LPCR;
  // L1 prefetch of one digit's data for this thread (its 64-byte slices of the piece row and of
  // the two key rows): issued one digit ahead so the loads at the top of the next iteration hit
  // L1 instead of exposing the full HBM/L2 latency to the first butterfly.
  const int own_j = is_main ? t % A.d : -1;
  const int hk = KP ? hs : hi;                                // line of the key rows
  auto prefetch_digit = [&](int j) {
    if (j >= A.beta) return;
    const size_t lo = ((size_t)hk << L2) + (size_t)tl * C::E;
    if ((LF_KSI_PF & 1) && (j != own_j || A.pre))
      prefetch_l1(A.T1 + b * A.t1_bs + ((size_t)(j * ext + r) << logN) + ((size_t)hs << L2) + (size_t)tl * C::E);
    if (LF_KSI_PF & 2) {
      prefetch_l1(keyb + (((size_t)(j * 2 + 0) * A.R + kr) << logN) + lo);
      prefetch_l1(keyb + (((size_t)(j * 2 + 1) * A.R + kr) << logN) + lo);
    }
  };
  __shared__ unsigned long long twbar;
  lf_pdl_trigger();
  if (!A.pre)           // finished pieces need no row NTT here
    tw_bulk_begin<L2>(tws, dv.twfT + ((size_t)pi << logN), (1u << L1) + hi0s, S::LPCR, &twbar);
  lf_pdl_wait();
  prefetch_digit(0);
  if (!A.pre) tw_bulk_wait(&twbar);

  u64 accb[C::E], acca[C::E];
#pragma unroll
  for (int e = 0; e < C::E; ++e) { accb[e] = 0; acca[e] = 0; }

  for (int j = 0; j < A.beta; ++j) {
    prefetch_digit(j + 1);
    u32 pc[C::E];
    if (A.pre) {
      // finished piece: load the source line, permute inside it (sigma_g) through smem
      load_row_step2<L2>(pc, A.T1 + b * A.t1_bs + ((size_t)(j * ext + r) << logN) + ((size_t)hs << L2), tl);
      if (GALOIS && !KP) {
        __syncwarp();                  // previous digit's gathers from perm_buf are done
#pragma unroll
        for (int e = 0; e < C::E; ++e) perm_buf[brev_bits(tl * C::E + e, L2)] = pc[e];
        __syncwarp();
#pragma unroll
        for (int e = 0; e < C::E; ++e) {
          const u32 pos = ((u32)hi << L2) + tl * C::E + e;
          pc[e] = perm_buf[auto_src_slot_brev(pos, gal, logN, L2)];
        }
      }
    } else if (j == own_j) {
      // own row of digit j: (x_t * s_t), permuted by sigma_g for rotations
      const u32 s = A.rowk[4 * t], sp = A.rowk[4 * t + 1];
      const u32* xr = (XMODE == 1 && A.ml.on ? A.ml.c1[b] + ((size_t)A.ml.p1[b] << logN) : A.x + b * A.x_bs) +
                      ((size_t)r << logN);
      if (GALOIS) {
        // the source line, coalesced; sigma_g through the line's slot buffer (GMODE 1)
        load_row_step2<L2>(pc, xr + ((size_t)hs << L2), tl);
#pragma unroll
        for (int e = 0; e < C::E; ++e) pc[e] = mul_shoup_lazy(pc[e], s, sp, pk.q);
        if (!KP) {
          __syncwarp();
#pragma unroll
          for (int e = 0; e < C::E; ++e) perm_buf[brev_bits(tl * C::E + e, L2)] = pc[e];
          __syncwarp();
#pragma unroll
          for (int e = 0; e < C::E; ++e) {
            const u32 pos = ((u32)hi << L2) + tl * C::E + e;
            pc[e] = perm_buf[auto_src_slot_brev(pos, gal, logN, L2)];
          }
        }
      } else {
        const u32* xr2 = (XMODE == 1 && A.ml.on ? A.ml.c2[b] + ((size_t)A.ml.p2[b] << logN) : A.x2 + b * A.x2_bs) +
                         ((size_t)r << logN);
        load_row_step2<L2>(pc, xr + ((size_t)hi << L2), tl);
        if (XMODE == 1) {
          u32 w[C::E];
          load_row_step2<L2>(w, xr2 + ((size_t)hi << L2), tl);
#pragma unroll
          for (int e = 0; e < C::E; ++e) pc[e] = mulmod(pc[e], w[e], pk);
        }
#pragma unroll
        for (int e = 0; e < C::E; ++e) pc[e] = mul_shoup_lazy(pc[e], s, sp, pk.q);
      }
    } else {
      const u32* tr = A.T1 + b * A.t1_bs + ((size_t)(j * ext + r) << logN) + ((size_t)hs << L2);
      load_row_step2<L2>(pc, tr, tl);
      fwd_line<L2, BIN>(pc, (1u << L1) + hs, TwTree<L2>{tws, (1u << L1) + hi0s, S::LPCR}, pk.q, xs,
                        tl, addr, SyncWarp{});
      if (GALOIS && !KP) {
        __syncwarp();                  // previous digit's gathers from perm_buf are done
#pragma unroll
        for (int e = 0; e < C::E; ++e) perm_buf[brev_bits(tl * C::E + e, L2)] = pc[e];
        __syncwarp();
#pragma unroll
        for (int e = 0; e < C::E; ++e) {
          const u32 pos = ((u32)hi << L2) + tl * C::E + e;
          pc[e] = perm_buf[auto_src_slot_brev(pos, gal, logN, L2)];
        }
      }
    }
    if (A.beta > 15) {
#pragma unroll
      for (int e = 0; e < C::E; ++e) pc[e] = reduce32_lazy(pc[e], pk);
    }
    {
      // key rows are loaded only now (L1-prefetched one digit ahead): keeping them live across
      // the row NTT would push the kernel past 128 registers and spill the twiddle addresses
      u32 kv[C::E];
      load_row_step2<L2>(kv, keyb + (((size_t)(j * 2 + 0) * A.R + kr) << logN) + ((size_t)hk << L2), tl);
#pragma unroll
      for (int e = 0; e < C::E; ++e) accb[e] += (u64)pc[e] * kv[e];
      load_row_step2<L2>(kv, keyb + (((size_t)(j * 2 + 1) * A.R + kr) << logN) + ((size_t)hk << L2), tl);
#pragma unroll
      for (int e = 0; e < C::E; ++e) acca[e] += (u64)pc[e] * kv[e];
    }
  }
  u32 rb[C::E], ra[C::E];
#pragma unroll
  for (int e = 0; e < C::E; ++e) { rb[e] = reduce64(accb[e], pk); ra[e] = reduce64(acca[e], pk); }
  if (KP) {
    // source frame -> output line: + P * b (unpermuted) first, then sigma_g on both accumulators
    if (A.ext_out && is_main) {
      const u32 pm = A.pmod[2 * t], pmp = A.pmod[2 * t + 1];
      u32 bv[C::E];
      load_row_step2<L2>(bv, A.eb + ((size_t)t << logN) + ((size_t)hs << L2), tl);
#pragma unroll
      for (int e = 0; e < C::E; ++e) rb[e] = addmod(rb[e], mul_shoup(bv[e], pm, pmp, pk.q), pk.q);
    }
#pragma unroll
    for (int e = 0; e < C::E; ++e) perm_buf[brev_bits(tl * C::E + e, L2)] = rb[e];
    __syncwarp();
#pragma unroll
    for (int e = 0; e < C::E; ++e)
      rb[e] = perm_buf[auto_src_slot_brev(((u32)hi << L2) + tl * C::E + e, gal, logN, L2)];
    __syncwarp();
#pragma unroll
    for (int e = 0; e < C::E; ++e) perm_buf[brev_bits(tl * C::E + e, L2)] = ra[e];
    __syncwarp();
#pragma unroll
    for (int e = 0; e < C::E; ++e)
      ra[e] = perm_buf[auto_src_slot_brev(((u32)hi << L2) + tl * C::E + e, gal, logN, L2)];
    __syncwarp();
  }
  if (A.ext_out) {
    if (is_main && !KP) {   // + P * sigma_g(b): the b part of the rotation before the division by P
      const u32 pm = A.pmod[2 * t], pmp = A.pmod[2 * t + 1];
      const u32* br = A.eb + ((size_t)t << logN);
#pragma unroll
      for (int e = 0; e < C::E; ++e) {
        const u32 pos = ((u32)hi << L2) + tl * C::E + e;
        const u32 v = br[GALOIS ? auto_src_index(pos, gal, logN) : pos];
        rb[e] = addmod(rb[e], mul_shoup(v, pm, pmp, pk.q), pk.q);
      }
    }
    store_row_step2<L2>(rb, A.acc + b * A.acc_bs + ((size_t)t << logN) + ((size_t)hi << L2), tl);
    store_row_step2<L2>(ra, A.acc + b * A.acc_bs + ((size_t)(ext + t) << logN) + ((size_t)hi << L2), tl);
  } else if (is_main && t <= l - A.fuse_nd) {
    store_row_step2<L2>(rb, A.acc + b * A.acc_bs + ((size_t)rs << logN) + ((size_t)hi << L2), tl);
    store_row_step2<L2>(ra, A.acc + b * A.acc_bs + ((size_t)(nms + rs) << logN) + ((size_t)hi << L2), tl);
  } else {
    // special row, or (fused rescale) one of the top main rows: T2 holds the rows the division
    // by P q_l [q_{l-1}] converts, in coefficient form after the row pass of the INTT
    const int s = is_main ? A.alpha + (t - (l + 1 - A.fuse_nd)) : rs;
    if (XMODE == 1 && is_main) {
      // + P * (d0, d1) (ckks.py:189-193: d0 = b1 b2, d1 = b1 a2 + a1 b2) before the division
      const u32 pm = A.pmod[2 * t], pmp = A.pmod[2 * t + 1];
      const u32* c1 = A.ml.on ? A.ml.c1[b] : A.c1 + b * A.c_bs;
      const u32* c2 = A.ml.on ? A.ml.c2[b] : A.c2 + b * A.c2_bs;
      const int ne1 = A.ml.on ? A.ml.p1[b] : A.c_ne, ne2 = A.ml.on ? A.ml.p2[b] : A.c2_ne;
      const size_t lo = (size_t)hi << L2;
      u32 b1[C::E], b2[C::E], o[C::E];
      load_row_step2<L2>(b1, c1 + ((size_t)t << logN) + lo, tl);
      load_row_step2<L2>(b2, c2 + ((size_t)t << logN) + lo, tl);
#pragma unroll
      for (int e = 0; e < C::E; ++e)
        rb[e] = addmod(rb[e], mul_shoup(mulmod(b1[e], b2[e], pk), pm, pmp, pk.q), pk.q);
      load_row_step2<L2>(o, c2 + ((size_t)(ne2 + t) << logN) + lo, tl);         // a2
#pragma unroll
      for (int e = 0; e < C::E; ++e) b1[e] = mulmod(b1[e], o[e], pk);          // b1 a2
      load_row_step2<L2>(o, c1 + ((size_t)(ne1 + t) << logN) + lo, tl);         // a1
#pragma unroll
      for (int e = 0; e < C::E; ++e) {
        const u32 d1 = addmod(b1[e], mulmod(o[e], b2[e], pk), pk.q);
        ra[e] = addmod(ra[e], mul_shoup(d1, pm, pmp, pk.q), pk.q);
      }
    }
    const TwGlobalT<L2> tw{dv.twiT + ((size_t)pi << logN), (1u << L1) + (u32)((bl % groups) * S::LPCR), S::LPCR};
    __syncwarp();
    inv_line<L2>(rb, (1u << L1) + hi, tw, pk.q, xs, tl, addr, SyncWarp{});
    store_row_step2<L2>(rb, A.T2 + b * A.t2_bs + ((size_t)s << logN) + ((size_t)hi << L2), tl);
    __syncwarp();
    inv_line<L2>(ra, (1u << L1) + hi, tw, pk.q, xs, tl, addr, SyncWarp{});
    store_row_step2<L2>(ra, A.T2 + b * A.t2_bs + ((size_t)(A.t2_rows + s) << logN) + ((size_t)hi << L2), tl);
  }
}

// ---------------------------------------------------------------------------------------
// K_C fused with the giant-step plaintext sums of a BSGS linear transform (hoisted ModDown):
// one CTA owns a few lines of one extended-basis row and runs EVERY baby rotation for them,
//   rot_r = sigma_r(P b + sum_j piece_j * K'_rj)  (permuted keys K' = K o sigma^-1, source frame)
// and accumulates out_k += rot_r * pt_{k,r} for every giant k in registers.  The rotated
// extended ciphertexts never reach memory; only the giant sums (ngiant x 2 x ext rows) do.
// Bit-identical to lf_rotate_hoisted_ext + lf_ptmac_rows (exact modular sums, any order).
#define LF_BSGS_GMAX 4
#define LF_BSGS_RMAX 32
struct BsgsExtArgs {
  const u32* T1;                 // beta x ext finished eval-domain pieces (k_pieces, natural)
  const u32* ct;                 // b rows then a rows (level+1 each)
  const u32* pmod;               // [n_main][2]: P mod q_t, Shoup companion
  u32* out;                      // ngiant x 2 x ext rows
  int level, L, alpha, beta, R, ext, nrot, ngiant;
  const u32* keyp[LF_BSGS_RMAX];                 // permuted key of rotation r
  u32 gs[LF_BSGS_RMAX];
  const u32* pt[LF_BSGS_GMAX][LF_BSGS_RMAX + 1]; // [giant][0: identity baby, 1 + r: rotation r]
};

template <int L1, int L2>
struct BsgsShape {
  static constexpr int M2 = 1 << L2;              // line length
  static constexpr int TPL = M2 / 4;              // threads per line (4 consecutive words each)
  static constexpr int LINES0 = 256 / TPL;
  static constexpr int LINES = LINES0 < (1 << L1) ? LINES0 : (1 << L1);
  static constexpr int THREADS = LINES * TPL;
};

template <int L1, int L2, int G>
__global__ void __launch_bounds__(BsgsShape<L1, L2>::THREADS)
k_bsgs_ext(BsgsExtArgs A, LfDev dv) {
  using S = BsgsShape<L1, L2>;
  constexpr int logN = L1 + L2;
  constexpr int M2 = S::M2;
  __shared__ u32 buf[S::LINES * M2];
  const int ln = threadIdx.x / S::TPL, tid = threadIdx.x % S::TPL;
  constexpr int CPR = (1 << L1) / S::LINES;       // CTAs per row
  const int t = blockIdx.x / CPR;
  const int hi = (blockIdx.x % CPR) * S::LINES + ln;
  const int l = A.level;
  const bool is_main = t <= l;
  const int pi = is_main ? t : A.L + 1 + (t - l - 1);
  const PrimeK pk = dv.pk[pi];
  const int ext = A.ext;
  u32* lb = buf + ln * M2;
  const int e0 = tid * 4;
  u32 pm = 0, pmp = 0;
  if (is_main) { pm = A.pmod[2 * t]; pmp = A.pmod[2 * t + 1]; }
  lf_pdl_trigger();
  lf_pdl_wait();

  u32 ob[G][4], oa[G][4];
#pragma unroll
  for (int k = 0; k < G; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e) { ob[k][e] = 0; oa[k][e] = 0; }

  // identity baby: P * ct on the main rows (its special rows are zero)
  if (is_main) {
    const uint4 vb = *reinterpret_cast<const uint4*>(A.ct + ((size_t)t << logN) + ((size_t)hi << L2) + e0);
    const uint4 va = *reinterpret_cast<const uint4*>(A.ct + ((size_t)(l + 1 + t) << logN) + ((size_t)hi << L2) + e0);
    const u32 xb[4] = {vb.x, vb.y, vb.z, vb.w}, xa[4] = {va.x, va.y, va.z, va.w};
#pragma unroll
    for (int k = 0; k < G; ++k) {
      const u32* p = A.pt[k][0];
      if (!p) continue;
      const uint4 pv = *reinterpret_cast<const uint4*>(p + ((size_t)t << logN) + ((size_t)hi << L2) + e0);
      const u32 pw[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const u32 w = mul_shoup(pw[e], pm, pmp, pk.q);           // P * pt
        ob[k][e] = addmod(ob[k][e], mulmod(xb[e], w, pk), pk.q);
        oa[k][e] = addmod(oa[k][e], mulmod(xa[e], w, pk), pk.q);
      }
    }
  }

#pragma unroll 1
  for (int r = 0; r < A.nrot; ++r) {
    const u32 g = A.gs[r];
    const int hs = (int)(auto_src_index((u32)hi << L2, g, logN) >> L2);
    const size_t src = ((size_t)hs << L2) + e0;
    const u32* key = A.keyp[r];
    u64 ab[4] = {0, 0, 0, 0}, aa[4] = {0, 0, 0, 0};
#pragma unroll 1
    for (int j = 0; j < A.beta; ++j) {
      const uint4 pc = *reinterpret_cast<const uint4*>(A.T1 + ((size_t)(j * ext + t) << logN) + src);
      const uint4 kb = *reinterpret_cast<const uint4*>(key + (((size_t)(j * 2 + 0) * A.R + pi) << logN) + src);
      const uint4 ka = *reinterpret_cast<const uint4*>(key + (((size_t)(j * 2 + 1) * A.R + pi) << logN) + src);
      ab[0] += (u64)pc.x * kb.x; ab[1] += (u64)pc.y * kb.y; ab[2] += (u64)pc.z * kb.z; ab[3] += (u64)pc.w * kb.w;
      aa[0] += (u64)pc.x * ka.x; aa[1] += (u64)pc.y * ka.y; aa[2] += (u64)pc.z * ka.z; aa[3] += (u64)pc.w * ka.w;
      if (A.beta > 15 && (j & 15) == 15) {
#pragma unroll
        for (int e = 0; e < 4; ++e) { ab[e] = reduce64(ab[e], pk); aa[e] = reduce64(aa[e], pk); }
      }
    }
    u32 rb[4], ra[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) { rb[e] = reduce64(ab[e], pk); ra[e] = reduce64(aa[e], pk); }
    if (is_main) {          // + P * b, then sigma_r (source frame -> output line)
      const uint4 bv = *reinterpret_cast<const uint4*>(A.ct + ((size_t)t << logN) + src);
      const u32 bw[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) rb[e] = addmod(rb[e], mul_shoup(bw[e], pm, pmp, pk.q), pk.q);
    }
    u32 sl[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) sl[e] = auto_src_slot_brev(((u32)hi << L2) + e0 + e, g, logN, L2);
    __syncthreads();                       // previous rotation's reads of buf are done
#pragma unroll
    for (int e = 0; e < 4; ++e) lb[brev_bits(e0 + e, L2)] = rb[e];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 4; ++e) rb[e] = lb[sl[e]];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 4; ++e) lb[brev_bits(e0 + e, L2)] = ra[e];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 4; ++e) ra[e] = lb[sl[e]];
#pragma unroll
    for (int k = 0; k < G; ++k) {
      const u32* p = A.pt[k][1 + r];
      if (!p) continue;
      const uint4 pv = *reinterpret_cast<const uint4*>(p + ((size_t)t << logN) + ((size_t)hi << L2) + e0);
      const u32 pw[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        ob[k][e] = addmod(ob[k][e], mulmod(rb[e], pw[e], pk), pk.q);
        oa[k][e] = addmod(oa[k][e], mulmod(ra[e], pw[e], pk), pk.q);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < G; ++k) {
    if (k >= A.ngiant) break;
    u32* ob_ = A.out + ((size_t)((k * 2 + 0) * ext + t) << logN) + ((size_t)hi << L2) + e0;
    u32* oa_ = A.out + ((size_t)((k * 2 + 1) * ext + t) << logN) + ((size_t)hi << L2) + e0;
    *reinterpret_cast<uint4*>(ob_) = make_uint4(ob[k][0], ob[k][1], ob[k][2], ob[k][3]);
    *reinterpret_cast<uint4*>(oa_) = make_uint4(oa[k][0], oa[k][1], oa[k][2], oa[k][3]);
  }
}

// ---------------------------------------------------------------------------------------
// k_bsgs_ext for beta = BETA known at compile time, software-pipelined in registers: the
// operands of baby rotation r + 1 (BETA pieces, 2 BETA key rows, ct.b, G diagonals: 16 B each
// per thread) are loaded while rotation r is multiplied, permuted and accumulated, so every
// thread keeps a whole rotation of loads (~240 B) in flight instead of one digit (48 B).
// Same arithmetic as k_bsgs_ext, bit for bit.
#ifndef LF_BSGS_MINB
#define LF_BSGS_MINB 2
#endif
template <int BETA, int G>
struct BsOps {
  uint4 pc[BETA], kb[BETA], ka[BETA], b, d[G];
};

template <int L1, int L2, int G, int BETA>
__global__ void __launch_bounds__(BsgsShape<L1, L2>::THREADS, LF_BSGS_MINB)
k_bsgs_pipe(BsgsExtArgs A, LfDev dv) {
  using S = BsgsShape<L1, L2>;
  constexpr int logN = L1 + L2;
  constexpr int M2 = S::M2;
  __shared__ u32 buf[S::LINES * M2];
  const int ln = threadIdx.x / S::TPL, tid = threadIdx.x % S::TPL;
  constexpr int CPR = (1 << L1) / S::LINES;
  const int t = blockIdx.x / CPR;
  const int hi = (blockIdx.x % CPR) * S::LINES + ln;
  const int l = A.level;
  const bool is_main = t <= l;
  const int pi = is_main ? t : A.L + 1 + (t - l - 1);
  const PrimeK pk = dv.pk[pi];
  const int ext = A.ext;
  u32* lb = buf + ln * M2;
  const int e0 = tid * 4;
  u32 pm = 0, pmp = 0;
  if (is_main) { pm = A.pmod[2 * t]; pmp = A.pmod[2 * t + 1]; }
  const size_t dst = ((size_t)t << logN) + ((size_t)hi << L2) + e0;
  auto load = [&](int r, BsOps<BETA, G>& o) {
    const int hs = (int)(auto_src_index((u32)hi << L2, A.gs[r], logN) >> L2);
    const size_t src = ((size_t)hs << L2) + e0;
    const u32* key = A.keyp[r];
#pragma unroll
    for (int j = 0; j < BETA; ++j) {
      o.pc[j] = __ldg(reinterpret_cast<const uint4*>(A.T1 + ((size_t)(j * ext + t) << logN) + src));
      o.kb[j] = __ldg(reinterpret_cast<const uint4*>(key + (((size_t)(j * 2 + 0) * A.R + pi) << logN) + src));
      o.ka[j] = __ldg(reinterpret_cast<const uint4*>(key + (((size_t)(j * 2 + 1) * A.R + pi) << logN) + src));
    }
    o.b = is_main ? __ldg(reinterpret_cast<const uint4*>(A.ct + ((size_t)t << logN) + src)) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int k = 0; k < G; ++k) {
      const u32* p = k < A.ngiant ? A.pt[k][1 + r] : nullptr;
      o.d[k] = p ? __ldg(reinterpret_cast<const uint4*>(p + dst)) : make_uint4(0, 0, 0, 0);
    }
  };
  lf_pdl_trigger();
  lf_pdl_wait();
  BsOps<BETA, G> cur;
  if (A.nrot > 0) load(0, cur);

  u32 ob[G][4], oa[G][4];
#pragma unroll
  for (int k = 0; k < G; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e) { ob[k][e] = 0; oa[k][e] = 0; }
  if (is_main) {            // identity baby: P * ct on the main rows (its special rows are zero)
    const uint4 vb = *reinterpret_cast<const uint4*>(A.ct + dst);
    const uint4 va = *reinterpret_cast<const uint4*>(A.ct + ((size_t)(l + 1 + t) << logN) + ((size_t)hi << L2) + e0);
    const u32 xb[4] = {vb.x, vb.y, vb.z, vb.w}, xa[4] = {va.x, va.y, va.z, va.w};
#pragma unroll
    for (int k = 0; k < G; ++k) {
      const u32* p = A.pt[k][0];
      if (!p) continue;
      const uint4 pv = *reinterpret_cast<const uint4*>(p + dst);
      const u32 pw[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const u32 w = mul_shoup(pw[e], pm, pmp, pk.q);
        ob[k][e] = addmod(ob[k][e], mulmod(xb[e], w, pk), pk.q);
        oa[k][e] = addmod(oa[k][e], mulmod(xa[e], w, pk), pk.q);
      }
    }
  }

#pragma unroll 1
  for (int r = 0; r < A.nrot; ++r) {
    const u32 g = A.gs[r];
    u64 ab[4] = {0, 0, 0, 0}, aa[4] = {0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < BETA; ++j) {
      const uint4 pc = cur.pc[j], kb = cur.kb[j], ka = cur.ka[j];
      ab[0] += (u64)pc.x * kb.x; ab[1] += (u64)pc.y * kb.y; ab[2] += (u64)pc.z * kb.z; ab[3] += (u64)pc.w * kb.w;
      aa[0] += (u64)pc.x * ka.x; aa[1] += (u64)pc.y * ka.y; aa[2] += (u64)pc.z * ka.z; aa[3] += (u64)pc.w * ka.w;
    }
    // rotation r + 1's operands are requested once this rotation's pieces and keys are
    // consumed (their registers are free), and land during the reduction, sigma and the
    // diagonal MACs below
    BsOps<BETA, G> nxt;
    const uint4 bcur = cur.b;
    uint4 dcur[G];
#pragma unroll
    for (int k = 0; k < G; ++k) dcur[k] = cur.d[k];
    if (r + 1 < A.nrot) load(r + 1, nxt);
    u32 rb[4], ra[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) { rb[e] = reduce64(ab[e], pk); ra[e] = reduce64(aa[e], pk); }
    if (is_main) {          // + P * b, then sigma_r (source frame -> output line)
      const u32 bw[4] = {bcur.x, bcur.y, bcur.z, bcur.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) rb[e] = addmod(rb[e], mul_shoup(bw[e], pm, pmp, pk.q), pk.q);
    }
    u32 sl[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) sl[e] = auto_src_slot_brev(((u32)hi << L2) + e0 + e, g, logN, L2);
    __syncthreads();                       // previous rotation's reads of buf are done
#pragma unroll
    for (int e = 0; e < 4; ++e) lb[brev_bits(e0 + e, L2)] = rb[e];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 4; ++e) rb[e] = lb[sl[e]];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 4; ++e) lb[brev_bits(e0 + e, L2)] = ra[e];
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 4; ++e) ra[e] = lb[sl[e]];
#pragma unroll
    for (int k = 0; k < G; ++k) {
      if (k >= A.ngiant || !A.pt[k][1 + r]) continue;
      const u32 pw[4] = {dcur[k].x, dcur[k].y, dcur[k].z, dcur[k].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        ob[k][e] = addmod(ob[k][e], mulmod(rb[e], pw[e], pk), pk.q);
        oa[k][e] = addmod(oa[k][e], mulmod(ra[e], pw[e], pk), pk.q);
      }
    }
    cur = nxt;
  }
#pragma unroll
  for (int k = 0; k < G; ++k) {
    if (k >= A.ngiant) break;
    u32* ob_ = A.out + ((size_t)((k * 2 + 0) * ext + t) << logN) + ((size_t)hi << L2) + e0;
    u32* oa_ = A.out + ((size_t)((k * 2 + 1) * ext + t) << logN) + ((size_t)hi << L2) + e0;
    *reinterpret_cast<uint4*>(ob_) = make_uint4(ob[k][0], ob[k][1], ob[k][2], ob[k][3]);
    *reinterpret_cast<uint4*>(oa_) = make_uint4(oa[k][0], oa[k][1], oa[k][2], oa[k][3]);
  }
}

// ---------------------------------------------------------------------------------------
// K_E: row pass of the NTT of the converted rows, (acc - conv) * scalar, epilogue.
enum { EPI_KS = 0, EPI_MUL = 1, EPI_ROT = 2 };
struct ModDownArgs {
  const u32* T3;       // 2 x nt rows (pass-C output)
  const u32* acc;      // 2 x nacc rows (canonical, eval); row t of poly p at p*nacc + t
  u32* out;            // 2 x nt rows
  const u32* e0;       // epilogue inputs (ct1 for MUL: b1 | a1 ; ct for ROT)
  const u32* e1;       // ct2 for MUL
  size_t t3_bs, acc_bs, out_bs, e_bs, e1_bs;
  const u32* scal;     // per target t: scalar, Shoup companion at scal[t*sstride], +1
  int sstride;
  const u32* dscal;    // EPI_MUL fused with a rescale: (q_l [q_{l-1}])^-1 for the d terms, stride 2
  int nt, nacc, ne;    // targets, acc rows per poly, epilogue rows per poly
  int ne1;             // rows per poly of e1 (EPI_MUL)
  int nbatch, bpc;     // instances; instances per CTA (sharing the staged twiddles)
  u32 gs[LF_MAXB];     // per instance galois element (EPI_ROT)
  const int* tmap;     // limb-sharded: storage row r is main prime tmap[r] (null: r)
  MulList ml;          // EPI_MUL with ml.on: per-instance epilogue operands
};

template <int L1, int L2, int EPI>
__global__ void __launch_bounds__(NttShape<L1, L2>::TRR)
k_moddown_out(ModDownArgs A, LfDev dv) {
  using S = NttShape<L1, L2>;
  using C = LineCfg<L2>;
  constexpr int logN = L1 + L2;
  constexpr int BIN = S::FWD_C_OUT;
  extern __shared__ u32 sm[];
  const int tl = threadIdx.x % C::T, ln = threadIdx.x / C::T;
  const int groups = (1 << L1) / S::LPCR;
  const int t = blockIdx.x / groups;                   // storage row
  const int pi = A.tmap ? A.tmap[t] : t;               // main prime index
  const int hi = (blockIdx.x % groups) * S::LPCR + ln;
  const PrimeK pk = dv.pk[pi];
  const u32 sc = A.scal[pi * A.sstride], scp = A.scal[pi * A.sstride + 1];
  uint2* tws = reinterpret_cast<uint2*>(sm);
  const u32 R0 = (1u << L1) + (blockIdx.x % groups) * S::LPCR;
  __shared__ unsigned long long twbar;
  lf_pdl_trigger();
  tw_bulk_begin<L2>(tws, dv.twfT + ((size_t)pi << logN), R0, S::LPCR, &twbar);
  lf_pdl_wait();
  const TwTree<L2> tw{tws, R0, S::LPCR};
  u32* xs = rowpass_xs<L1, L2>(sm);
  const AddrR<L2> addr{ln * pitchR<L2>()};
  const size_t lo0 = ((size_t)hi << L2);
  const int b0 = blockIdx.z * A.bpc, b1 = min(A.nbatch, b0 + A.bpc);
#pragma unroll 1
  for (int bb = b0; bb < b1; ++bb) {
  const size_t b = bb;
#pragma unroll 1
  for (int p = 0; p < 2; ++p) {
    u32 cv[C::E], av[C::E];
    load_row_step2<L2>(cv, A.T3 + b * A.t3_bs + ((size_t)(p * A.nt + t) << logN) + lo0, tl);
    if (p == 0) {     // the a-polynomial's rows arrive in L1 while the b-polynomial is processed
      prefetch_l1(A.T3 + b * A.t3_bs + ((size_t)(A.nt + t) << logN) + lo0 + (size_t)tl * C::E);
      prefetch_l1(A.acc + b * A.acc_bs + ((size_t)t << logN) + lo0 + (size_t)tl * C::E);
      prefetch_l1(A.acc + b * A.acc_bs + ((size_t)(A.nacc + t) << logN) + lo0 + (size_t)tl * C::E);
    }
    if (p || bb != b0) {
      __syncwarp();
    } else {
      tw_bulk_wait(&twbar);
    }
    fwd_line<L2, BIN>(cv, (1u << L1) + hi, tw, pk.q, xs, tl, addr, SyncWarp{});
    load_row_step2<L2>(av, A.acc + b * A.acc_bs + ((size_t)(p * A.nacc + t) << logN) + lo0, tl);
#pragma unroll
    for (int e = 0; e < C::E; ++e) {
      const u32 v = av[e] + 8 * pk.q - csub(cv[e], 8 * pk.q);     // (0, 9q)
      av[e] = mul_shoup(v, sc, scp, pk.q);
    }
    if (EPI == EPI_MUL) {
      // d0 = b1*b2 ; d1 = b1*a2 + a1*b2  (ckks.py:189-193)
      const u32* c1 = A.ml.on ? A.ml.c1[b] : A.e0 + b * A.e_bs;
      const u32* c2 = A.ml.on ? A.ml.c2[b] : A.e1 + b * A.e1_bs;
      const int ne1 = A.ml.on ? A.ml.p1[b] : A.ne, ne2 = A.ml.on ? A.ml.p2[b] : A.ne1;
      u32 b1[C::E], b2[C::E], o1[C::E], o2[C::E];
      load_row_step2<L2>(b1, c1 + ((size_t)t << logN) + lo0, tl);
      load_row_step2<L2>(b2, c2 + ((size_t)t << logN) + lo0, tl);
      const u32 ds = A.dscal ? A.dscal[2 * pi] : 0u, dsp = A.dscal ? A.dscal[2 * pi + 1] : 0u;
      if (p == 0) {
#pragma unroll
        for (int e = 0; e < C::E; ++e) {
          u32 d0 = mulmod(b1[e], b2[e], pk);
          if (A.dscal) d0 = mul_shoup(d0, ds, dsp, pk.q);
          av[e] = addmod(av[e], d0, pk.q);
        }
        if (A.ml.on && A.ml.addb[b]) {       // + K (mod q): a constant folded into the product
          const long long K = A.ml.addb[b];
          u32 kv = reduce64((u64)(K < 0 ? -K : K), pk);
          if (K < 0 && kv) kv = pk.q - kv;
#pragma unroll
          for (int e = 0; e < C::E; ++e) av[e] = addmod(av[e], kv, pk.q);
        }
      } else {
        load_row_step2<L2>(o1, c1 + ((size_t)(ne1 + t) << logN) + lo0, tl);
        load_row_step2<L2>(o2, c2 + ((size_t)(ne2 + t) << logN) + lo0, tl);
#pragma unroll
        for (int e = 0; e < C::E; ++e) {
          u32 d1 = reduce64((u64)b1[e] * o2[e] + (u64)o1[e] * b2[e], pk);
          if (A.dscal) d1 = mul_shoup(d1, ds, dsp, pk.q);
          av[e] = addmod(av[e], d1, pk.q);
        }
      }
    } else if (EPI == EPI_ROT) {
      if (p == 0) {
        // + sigma_g(b): load the source line coalesced, permute it through the line's exchange
        // buffer (bit-reversed slots: conflict-free), instead of a per-element global gather
        const u32 g = A.gs[b];
        const int hs = (int)(auto_src_index((u32)hi << L2, g, logN) >> L2);
        u32 bv[C::E];
        load_row_step2<L2>(bv, A.e0 + b * A.e_bs + ((size_t)t << logN) + ((size_t)hs << L2), tl);
        u32* pb = xs + ln * pitchR<L2>();
        __syncwarp();                       // the line transform's reads of xs are done
#pragma unroll
        for (int e = 0; e < C::E; ++e) pb[brev_bits(tl * C::E + e, L2)] = bv[e];
        __syncwarp();
#pragma unroll
        for (int e = 0; e < C::E; ++e)
          av[e] = addmod(av[e], pb[auto_src_slot_brev(((u32)hi << L2) + tl * C::E + e, g, logN, L2)], pk.q);
        __syncwarp();                       // before the next line transform reuses xs
      }
    }
    store_row_step2<L2>(av, A.out + b * A.out_bs + ((size_t)(p * A.nt + t) << logN) + lo0, tl);
  }
  }
}

// ---------------------------------------------------------------------------------------
// Materialised pieces (keyswitch_decompose API): finish the NTT of T1 rows, own rows x*s.
template <int L1, int L2>
__global__ void __launch_bounds__(NttShape<L1, L2>::TRR)
k_pieces(const u32* T1, const u32* __restrict__ x, u32* out,
         const u32* rowk, int level, int d, int L, int alpha, LfDev dv) {
  using S = NttShape<L1, L2>;
  using C = LineCfg<L2>;
  constexpr int logN = L1 + L2;
  extern __shared__ u32 sm[];
  const int tl = threadIdx.x % C::T, ln = threadIdx.x / C::T;
  const int groups = (1 << L1) / S::LPCR;
  const int ext = level + 1 + alpha;
  const int r = blockIdx.x / groups;          // j * ext + t
  const int j = r / ext, t = r % ext;
  const int hi = (blockIdx.x % groups) * S::LPCR + ln;
  const bool is_main = t <= level;
  const int pi = is_main ? t : L + 1 + (t - level - 1);
  const PrimeK pk = dv.pk[pi];
  const size_t lo0 = (size_t)hi << L2;
  lf_pdl_trigger();
  lf_pdl_wait();
  u32 v[C::E];
  if (is_main && t % d == j) {
    load_row_step2<L2>(v, x + ((size_t)t << logN) + lo0, tl);
#pragma unroll
    for (int e = 0; e < C::E; ++e) v[e] = mul_shoup(v[e], rowk[4 * t], rowk[4 * t + 1], pk.q);
  } else {
    load_row_step2<L2>(v, T1 + ((size_t)r << logN) + lo0, tl);
    fwd_line<L2, S::FWD_C_OUT>(v, (1u << L1) + hi,
                               TwGlobalT<L2>{dv.twfT + ((size_t)pi << logN),
                                             (1u << L1) + (u32)((blockIdx.x % groups) * S::LPCR), S::LPCR}, pk.q,
                               rowpass_xs<L1, L2>(sm), tl, AddrR<L2>{ln * pitchR<L2>()}, SyncWarp{});
#pragma unroll
    for (int e = 0; e < C::E; ++e) v[e] = reduce32(v[e], pk);
  }
  store_row_step2<L2>(v, out + ((size_t)r << logN) + lo0, tl);
}

// =======================================================================================
// host side
struct KsWs {
  u32 *T0, *T1, *acc, *T2, *T3;
  size_t per_sh;   // words per instance of the shared part (ModUp output), 0 when hoisted
  size_t per;      // words per instance of the per-key part
};

static size_t ks_ws_rows_shared(const LfKsPlan* P, int level) {
  const int l1 = level + 1, ext = l1 + P->n_special;
  const int beta = P->d < l1 ? P->d : l1;
  return (size_t)l1 + (size_t)beta * ext;
}
static size_t ks_ws_rows_inst(const LfKsPlan* P, int level) {
  const int l1 = level + 1;
  return 4 * (size_t)l1 + 2 * (size_t)P->n_special;
}
static size_t ks_ws_rows(const LfKsPlan* P, int level) {
  return ks_ws_rows_shared(P, level) + ks_ws_rows_inst(P, level);
}

// Layout: nsh x [T0 | T1] then batch x [acc | T2 | T3].
static KsWs carve(const LfCtx* ctx, int level, void* ws, int nsh = 1, bool hoisted = false,
                  int nd = 0) {
  const LfKsPlan* P = ctx->ks;
  const int l1 = level + 1;
  const size_t N = ctx->N;
  const size_t sh = ks_ws_rows_shared(P, level) * N, in = ks_ws_rows_inst(P, level) * N;
  KsWs w;
  u32* p = (u32*)ws;
  w.T0 = p;
  w.T1 = p + (size_t)l1 * N;
  p += (size_t)nsh * sh;
  w.acc = p;
  w.T2 = p + 2 * (size_t)l1 * N;
  w.T3 = w.T2 + 2 * (size_t)(P->n_special + nd) * N;     // T3 has 2 nd rows fewer
  w.per_sh = hoisted ? 0 : sh;
  w.per = in;
  return w;
}

template <int L1, int L2, int CW, int KMAX, int TG, int KEX>
static int launch_bc(const LfCtx* ctx, const BcArgs& A, int batch, int kmax, cudaStream_t s) {
  using Y_ = YTile<L1>;
  int mmax = 0;
  for (int g = 0; g < A.ngroups; ++g) mmax = A.g[g].B.m > mmax ? A.g[g].B.m : mmax;
  const int wwords = ((mmax + A.tsplit - 1) / A.tsplit) * kmax;
  const size_t sm = ((size_t)kmax * Y_::T * CW * Y_::E + (size_t)TG * smemC_words<L1, CW>() + wwords) * 4;
  if (sm > 227 * 1024) { lf_set_error("bconv: shared memory %zu too large", sm); return 2; }
  auto kern = k_bconv_colpass<L1, L2, CW, KMAX, TG, KEX>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const long nblocks = (long)batch * ((1 << L2) / CW) * A.ngroups * A.tsplit;
  LfDev dv = ctx->dev();
  LF_LAUNCH_CHECK(lf_launch(kern, dim3((unsigned)nblocks), dim3(TG * CW * LineCfg<L1>::T), sm, s,
                            A.tsplit, A, dv, kmax, batch));
  return 0;
}

static int env_int(const char* name, int dflt);

template <int L1, int L2, int KB, bool UEPI = false>
static int launch_bc_tc(const LfCtx* ctx, const BcArgs& A, int batch, cudaStream_t s) {
  constexpr int SBO = KB / 16 * 128;
  constexpr size_t ABYTES = (size_t)16 * 16 * SBO + 128;
  int mmax = 0;
  for (int g = 0; g < A.ngroups; ++g) mmax = A.g[g].B.m > mmax ? A.g[g].B.m : mmax;
  const int chunk = ((mmax + A.tsplit - 1) / A.tsplit + 1) & ~1;
  const int wbytes = (chunk + 7) / 8 * 8 * 256;
  const size_t sm = ABYTES + wbytes + (size_t)8 * smemC_words<L1, 8>() * 4;
  if (sm > 227 * 1024) { lf_set_error("bconv_tc: shared memory %zu too large", sm); return 2; }
  auto kern = k_bconv_tc<L1, L2, KB, UEPI>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const long nblocks = (long)batch * ((1 << L2) / 8) * A.ngroups * A.tsplit;
  LfDev dv = ctx->dev();
  LF_LAUNCH_CHECK(lf_launch(kern, dim3((unsigned)nblocks), dim3(1024), sm, s, A.tsplit, A, dv, batch, wbytes));
  return 0;
}

// Column tile width and group count: CW = 8 columns (32-byte row segments) and four thread
// groups sharing the source tile for the production sizes; narrower tiles for large digit
// counts (d = 1 style parameter sets) or tiny rings.  At N = 2^16, launches with at most 12
// sources per group use the compile-time-K kernel.  With byte-split weight tables (k <= 16)
// the conversion runs on the tensor cores (k_bconv_tc; LF_BC_TC=0 selects the IMAD kernel);
// k = 16 fills the 64 K-bytes and takes the overflow term in the epilogue (UEPI).
static int g_bc_engine = -1;     // -1: not read yet; 1: tensor cores when tables allow; 0: IMAD
static int bc_engine() {
  if (g_bc_engine < 0) g_bc_engine = env_int("LF_BC_TC", 1) ? 1 : 0;
  return g_bc_engine;
}

template <int L1, int L2>
static int launch_bc_auto(const LfCtx* ctx, const BcArgs& A, int batch, int kmax, cudaStream_t s) {
  if constexpr (L1 == 8 && L2 == 8) {
    bool tc = bc_engine() != 0, uepi = false;
    int kb = 0;
    for (int g = 0; g < A.ngroups && tc; ++g) {
      tc = A.g[g].B.w8 != nullptr;
      kb = A.g[g].B.kb > kb ? A.g[g].B.kb : kb;
      uepi |= 4 * A.g[g].B.k + 1 > 64;
    }
    if (tc && kb == 48) return launch_bc_tc<L1, L2, 48>(ctx, A, batch, s);
    if (tc && kb == 64 && !uepi) return launch_bc_tc<L1, L2, 64>(ctx, A, batch, s);
    if (tc && kb == 64) return launch_bc_tc<L1, L2, 64, true>(ctx, A, batch, s);
  }
  constexpr int NCOL = 1 << L2;
  constexpr int CW8 = NCOL >= 8 ? 8 : NCOL;
  constexpr int TG = (CW8 * LineCfg<L1>::T) % 32 == 0 ? 4 : 1;
  if (kmax > 16) return launch_bc<L1, L2, (NCOL >= 2 ? 2 : 1), 64, 1, 0>(ctx, A, batch, kmax, s);
  if constexpr (L1 == 8 && L2 == 8) {
    // groups with fewer sources than kmax (uneven digits) run padded with zero tiles
    switch (kmax) {
#define LF_BC_K(K) case K: return launch_bc<L1, L2, CW8, 16, TG, K>(ctx, A, batch, kmax, s);
      LF_BC_K(1) LF_BC_K(2) LF_BC_K(3) LF_BC_K(4) LF_BC_K(5) LF_BC_K(6) LF_BC_K(7) LF_BC_K(8) LF_BC_K(9)
      LF_BC_K(10) LF_BC_K(11) LF_BC_K(12)
#undef LF_BC_K
      default: break;
    }
  }
  return launch_bc<L1, L2, CW8, 16, TG, 0>(ctx, A, batch, kmax, s);
}

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

static int bc_tsplit(int ngroups, int batch, int ncoltiles, int mmax, int limit = 96) {
  // Split the target range over a cluster only while the launch has fewer CTAs than ~2/3 of
  // the 148 SMs: each CTA then converts all its targets from one source tile (no DSMEM
  // exchange), which measured fastest whenever the grid already covers the GPU (C2 batch 1:
  // ModUp 75 -> 63 us unsplit; ModDown with 2 groups needs the split: 64 -> 43 us).
  int ts = 1;
  while (ts < 8 && (long)ngroups * batch * ncoltiles * ts < limit && mmax / (ts * 2) >= 4) ts *= 2;
  return ts;
}

enum { OP_KS = 0, OP_MUL = 1, OP_ROT = 2 };

struct KsCall {
  int level, batch, op;
  bool hoisted;             // one ModUp shared by all instances (x_bs = e_bs = 0)
  const u32 *x, *x2;        // K_A/K_C inputs: x (op KS: the poly; MUL: a1, a2; ROT: ct.a)
  size_t x_bs;
  const u32* key;           // instance b uses keylist[b0+b] if given, else key + (b0+b)*key_bs
  size_t key_bs;
  const u32* const* keylist;
  u32* out;                 // batch x 2 x (l+1)
  size_t out_bs;
  const u32 *e0, *e1;       // epilogue (MUL: ct1, ct2; ROT: ct)
  size_t e_bs;
  u32 g;                    // galois element (ROT): glist[b0+b] if given, else g
  const u32* glist;
  int b0;                   // first instance of this chunk
  bool ext_out;             // stop after the inner product: out = 2 x ext rows per instance
  int rescale_nd;           // MUL: fuse a rescale by this many primes into the ModDown (0: none)
  bool kperm;               // ROT: keys in permuted form (lf_permute_rotation_key)
  const BsgsExtArgs* bsgs;  // hoisted ROT: K_C fused with the giant-step sums (k_bsgs_ext)
  size_t x2s() const { return sep2 ? x2_bs : x_bs; }
  size_t e1s() const { return sep2 ? e1_bs : e_bs; }
  int pitch, pitch2;        // MUL: rows per polynomial of ct1 / ct2 (>= level + 1; 0: level + 1)
  size_t x2_bs, e1_bs;      // MUL: instance strides of a2 / ct2 (used when sep2)
  const u32* const* c1l;    // MUL over an operand list (instance b0 + b): ct1 / ct2 bases and
  const u32* const* c2l;    // rows per polynomial (null: strided operands)
  const int *p1l, *p2l;
  const int64_t* addl;      // MUL list: per-instance constant added to b (null: none)
  bool sep2;                // ct2 has its own stride and pitch (else those of ct1)
  const u32* keyp_of(int b) const { return keylist ? keylist[b0 + b] : key + (size_t)(b0 + b) * key_bs; }
  u32 g_of(int b) const { return glist ? glist[b0 + b] : g; }
};

template <int L1, int L2>
static int ks_pipeline(const LfCtx* ctx, const KsCall& c, void* ws, cudaStream_t s,
                       cudaEvent_t* ev = nullptr) {
  using S = NttShape<L1, L2>;
  const LfKsPlan* P = ctx->ks;
  const KsLevelPlan& K = P->lv[c.level];
  const int l1 = c.level + 1, alpha = P->n_special;
  const size_t N = ctx->N;
  const int nsh = c.hoisted ? 1 : c.batch;
  const int nd = c.op == OP_MUL ? c.rescale_nd : 0;
  const KsWs w = carve(ctx, c.level, ws, nsh, c.hoisted, nd);
  const int nt = l1 - nd;                  // output rows per polynomial
  const LfDev dv = ctx->dev();
  const size_t smR = rowpass_smem_bytes<L1, L2>(0);
  const int groups = (1 << L1) / S::LPCR;

#define LF_MARK(i) do { if (ev) cudaEventRecord(ev[i], s); } while (0)
  MulList ml{};
  if (c.op == OP_MUL && c.c1l) {
    ml.on = 1;
    for (int b = 0; b < c.batch; ++b) {
      ml.c1[b] = c.c1l[c.b0 + b]; ml.c2[b] = c.c2l[c.b0 + b];
      ml.p1[b] = c.p1l[c.b0 + b]; ml.p2[b] = c.p2l[c.b0 + b];
      ml.addb[b] = c.addl ? (long long)c.addl[c.b0 + b] : 0;
    }
  }
  LF_MARK(0);
  // K_A
  {
#ifndef LF_BPC
#define LF_BPC 4
#endif
    const int bpc_in = nsh >= 2 * LF_BPC ? LF_BPC : 1;      // instances per CTA (shared twiddles)
    dim3 grid(l1 * groups, 1, (nsh + bpc_in - 1) / bpc_in);
    if (c.op == OP_MUL)
      { lf_smem_optin(k_modup_in<L1, L2, 1>, smR); LF_LAUNCH_CHECK(lf_launch(k_modup_in<L1, L2, 1>, dim3(grid), dim3(S::TRR), smR, s, 1, c.x, c.x2, w.T0, c.x_bs, w.per_sh, l1, dv, l1, 0, 0, 0, nsh, bpc_in, 1, c.x2s(), l1, ml)); }
    else
      { lf_smem_optin(k_modup_in<L1, L2, 0>, smR); LF_LAUNCH_CHECK(lf_launch(k_modup_in<L1, L2, 0>, dim3(grid), dim3(S::TRR), smR, s, 1, c.x, nullptr, w.T0, c.x_bs, w.per_sh, l1, dv, l1, 0, 0, 0, nsh, bpc_in, 1, (size_t)0, 0, MulList{})); }
    LF_CHECK_LAUNCH();
  }
  LF_MARK(1);
  // K_BC (ModUp)
  {
    BcArgs A{};
    A.src = w.T0; A.dst = w.T1; A.src_bs = w.per_sh; A.dst_bs = w.per_sh;
    A.ngroups = K.beta;
    int kmax = 0, mmax = 0;
    for (int j = 0; j < K.beta; ++j) {
      A.g[j] = K.up[j];
      kmax = K.up[j].B.k > kmax ? K.up[j].B.k : kmax;
      mmax = K.up[j].B.m > mmax ? K.up[j].B.m : mmax;
    }
    A.tsplit = bc_tsplit(K.beta, nsh, (1 << L2) / 8, mmax, env_int("LF_TSPLIT_UP", 96));
    if (int e = launch_bc_auto<L1, L2>(ctx, A, nsh, kmax, s)) return e;
  }
  // hoisted batch: finish the NTT of every piece ONCE (in place, natural layout); each rotation's
  // inner product then only permutes and multiplies (no per-rotation row NTT)
  const bool pre = c.hoisted && (c.batch > 1 || c.bsgs);
  if (pre) {
    dim3 grid(K.beta * K.ext * groups);
    lf_smem_optin(k_pieces<L1, L2>, smR);
    LF_LAUNCH_CHECK(lf_launch(k_pieces<L1, L2>, dim3(grid), dim3(S::TRR), smR, s, 1, w.T1, c.x, w.T1, P->rowk, c.level, P->d, P->L,
                                              P->n_special, dv));
    LF_CHECK_LAUNCH();
  }
  LF_MARK(2);
  if (c.bsgs) {
    using SB = BsgsShape<L1, L2>;
    BsgsExtArgs A = *c.bsgs;
    A.T1 = w.T1; A.pmod = P->pmod; A.level = c.level; A.L = P->L; A.alpha = alpha;
    A.beta = K.beta; A.R = P->L + 1 + alpha; A.ext = K.ext;
    dim3 grid(K.ext * ((1 << L1) / SB::LINES));
    static int pipe = -1;
    if (pipe < 0) pipe = env_int("LF_BSGS_PIPE", 1);
    if (pipe && A.beta == 4) {
      switch (A.ngiant) {
#define LF_BP(GG) case GG: LF_LAUNCH_CHECK(lf_launch(k_bsgs_pipe<L1, L2, GG, 4>, grid, dim3(SB::THREADS), 0, s, 1, A, dv)); break;
        LF_BP(1) LF_BP(2) LF_BP(3) LF_BP(4)
#undef LF_BP
        default: lf_set_error("bsgs: %d giant steps (max %d)", A.ngiant, LF_BSGS_GMAX); return 2;
      }
      LF_CHECK_LAUNCH();
      return 0;
    }
    switch (A.ngiant) {
#define LF_BG(GG) case GG: LF_LAUNCH_CHECK(lf_launch(k_bsgs_ext<L1, L2, GG>, grid, dim3(SB::THREADS), 0, s, 1, A, dv)); break;
      LF_BG(1) LF_BG(2) LF_BG(3) LF_BG(4)
#undef LF_BG
      default: lf_set_error("bsgs: %d giant steps (max %d)", A.ngiant, LF_BSGS_GMAX); return 2;
    }
    LF_CHECK_LAUNCH();
    return 0;
  }
  // K_C
  {
    KsInnerArgs A{};
    A.T1 = w.T1; A.x = c.x; A.x2 = c.x2; A.acc = w.acc; A.T2 = w.T2;
    A.t1_bs = w.per_sh; A.x_bs = c.x_bs; A.acc_bs = w.per; A.t2_bs = w.per;
    A.rowk = P->rowk; A.level = c.level; A.d = P->d; A.beta = K.beta; A.L = P->L; A.alpha = alpha;
    A.R = P->L + 1 + alpha; A.nbatch = c.batch;
    A.ext_out = c.ext_out ? 1 : 0;
    A.pre = pre ? 1 : 0;
    A.fuse_nd = nd; A.t2_rows = alpha + nd;
    A.c1 = c.e0; A.c2 = c.e1; A.c_bs = c.e_bs; A.c_ne = c.pitch > 0 ? c.pitch : l1;
    A.c2_bs = c.e1s(); A.c2_ne = c.sep2 ? (c.pitch2 > 0 ? c.pitch2 : l1) : A.c_ne; A.x2_bs = c.x2s();
    A.ml = ml;
    A.pmod = P->pmod;
    if (c.ext_out) { A.acc = c.out; A.acc_bs = c.out_bs; A.eb = c.e0; A.pmod = P->pmod; }
    for (int b = 0; b < c.batch; ++b) { A.keyp[b] = c.keyp_of(b); A.gs[b] = c.g_of(b); }
    const size_t smC = rowpass_smem_bytes<L1, L2>(LineCfg<L2>::M);
    dim3 grid(K.ext * groups * c.batch);
    if (c.op == OP_ROT && c.kperm) { lf_smem_optin(k_ks_inner<L1, L2, 2, 0>, smC); LF_LAUNCH_CHECK(lf_launch(k_ks_inner<L1, L2, 2, 0>, dim3(grid), dim3(S::TRR), smC, s, 1, A, dv)); }
    else if (c.op == OP_ROT) { lf_smem_optin(k_ks_inner<L1, L2, 1, 0>, smC); LF_LAUNCH_CHECK(lf_launch(k_ks_inner<L1, L2, 1, 0>, dim3(grid), dim3(S::TRR), smC, s, 1, A, dv)); }
    else if (c.op == OP_MUL) { lf_smem_optin(k_ks_inner<L1, L2, 0, 1>, smC); LF_LAUNCH_CHECK(lf_launch(k_ks_inner<L1, L2, 0, 1>, dim3(grid), dim3(S::TRR), smC, s, 1, A, dv)); }
    else { lf_smem_optin(k_ks_inner<L1, L2, 0, 0>, smC); LF_LAUNCH_CHECK(lf_launch(k_ks_inner<L1, L2, 0, 0>, dim3(grid), dim3(S::TRR), smC, s, 1, A, dv)); }
    LF_CHECK_LAUNCH();
  }
  LF_MARK(3);
  if (c.ext_out) return 0;
  // K_BC (ModDown)
  {
    BcArgs A{};
    A.src = w.T2; A.dst = w.T3; A.src_bs = w.per; A.dst_bs = w.per;
    A.ngroups = 2;
    for (int p = 0; p < 2; ++p) {
      if (nd) {
        A.g[p] = K.dr[nd - 1][p];
        continue;
      }
      A.g[p].B = P->down;
      A.g[p].B.m = l1;                     // prefix of the level-L table
      A.g[p].src_rows = P->iota;
      A.g[p].dst_rows = P->iota;
      A.g[p].src_row0 = p * alpha;
      A.g[p].dst_row0 = p * l1;
    }
    A.tsplit = bc_tsplit(2, c.batch, (1 << L2) / 8, nt, env_int("LF_TSPLIT_DOWN", 96));
    if (int e = launch_bc_auto<L1, L2>(ctx, A, c.batch, alpha + nd, s)) return e;
  }
  LF_MARK(4);
  // K_E
  {
    ModDownArgs A{};
    A.T3 = w.T3; A.acc = w.acc; A.out = c.out; A.e0 = c.e0; A.e1 = c.e1;
    A.t3_bs = w.per; A.acc_bs = w.per; A.out_bs = c.out_bs; A.e_bs = c.e_bs; A.e1_bs = c.e1s();
    A.scal = P->rowk + 2; A.sstride = 4; A.nt = nt; A.nacc = l1; A.ne = c.pitch > 0 ? c.pitch : l1;
    A.ne1 = c.sep2 ? (c.pitch2 > 0 ? c.pitch2 : l1) : A.ne;
    A.ml = ml;
    if (nd) {
      A.scal = P->pqinv[nd - 1] + (size_t)c.level * P->n_main * 2; A.sstride = 2;
      A.dscal = (nd == 1 ? P->qinv : P->qinv2) + (size_t)c.level * P->n_main * 2;
    }
    for (int b = 0; b < c.batch; ++b) A.gs[b] = c.g_of(b);
    A.nbatch = c.batch;
    A.bpc = c.batch >= 2 * LF_BPC ? LF_BPC : 1;
    dim3 grid(nt * groups, 1, (c.batch + A.bpc - 1) / A.bpc);
    if (c.op == OP_MUL) { lf_smem_optin(k_moddown_out<L1, L2, EPI_MUL>, smR); LF_LAUNCH_CHECK(lf_launch(k_moddown_out<L1, L2, EPI_MUL>, dim3(grid), dim3(S::TRR), smR, s, 1, A, dv)); }
    else if (c.op == OP_ROT) { lf_smem_optin(k_moddown_out<L1, L2, EPI_ROT>, smR); LF_LAUNCH_CHECK(lf_launch(k_moddown_out<L1, L2, EPI_ROT>, dim3(grid), dim3(S::TRR), smR, s, 1, A, dv)); }
    else { lf_smem_optin(k_moddown_out<L1, L2, EPI_KS>, smR); LF_LAUNCH_CHECK(lf_launch(k_moddown_out<L1, L2, EPI_KS>, dim3(grid), dim3(S::TRR), smR, s, 1, A, dv)); }
    LF_CHECK_LAUNCH();
  }
  LF_MARK(5);
#undef LF_MARK
  (void)N;
  return 0;
}

// rescale by the top `nd` primes (1: ckks.rescale, ckks.py:220-225 / poly.py:284-287; 2: two
// successive rescales fused into one floor division by q_l q_{l-1}, bit-identical since
// floor(floor(X/a)/b) = floor(X/(ab)) for the exact representative X >= 0).
template <int L1, int L2>
static int rescale_pipeline(const LfCtx* ctx, int level, int nd, const u32* ct, size_t ct_bs,
                            u32* out, size_t out_bs, int batch, void* ws, cudaStream_t s, int pitch = 0) {
  if (pitch <= 0) pitch = level + 1;           // rows per polynomial of ct
  using S = NttShape<L1, L2>;
  const LfKsPlan* P = ctx->ks;
  const KsLevelPlan& K = P->lv[level];
  const int l = level;
  const int nt = l + 1 - nd;                    // kept rows
  const size_t N = ctx->N;
  const LfDev dv = ctx->dev();
  const size_t smR = rowpass_smem_bytes<L1, L2>(0);
  const int groups = (1 << L1) / S::LPCR;
  u32* T2 = (u32*)ws;                      // per instance: 2 nd rows, then T3: 2 nt rows
  const size_t per = (2 * (size_t)nd + 2 * (size_t)nt) * N;
  u32* T3 = T2 + 2 * (size_t)nd * N;
  {  // row pass of INTT of the dropped rows of b and a
    dim3 grid(2 * nd * groups, 1, batch);
    { lf_smem_optin(k_modup_in<L1, L2, 0>, smR); LF_LAUNCH_CHECK(lf_launch(k_modup_in<L1, L2, 0>, dim3(grid), dim3(S::TRR), smR, s, 1, ct, nullptr, T2, ct_bs, per, 2 * nd, dv, nd, pitch, nt, nt, batch, 1, 1, (size_t)0, 0, MulList{})); }
    LF_CHECK_LAUNCH();
  }
  {
    BcArgs A{};
    A.src = T2; A.dst = T3; A.src_bs = per; A.dst_bs = per;
    A.ngroups = 2;
    A.g[0] = nd == 1 ? K.resc[0] : K.resc2[0];
    A.g[1] = nd == 1 ? K.resc[1] : K.resc2[1];
    A.tsplit = bc_tsplit(2, batch, (1 << L2) / 8, nt);
    if (int e = launch_bc_auto<L1, L2>(ctx, A, batch, nd, s)) return e;
  }
  {
    ModDownArgs A{};
    A.T3 = T3; A.acc = ct; A.out = out; A.e0 = nullptr; A.e1 = nullptr;
    A.t3_bs = per; A.acc_bs = ct_bs; A.out_bs = out_bs; A.e_bs = 0;
    A.scal = (nd == 1 ? P->qinv : P->qinv2) + (size_t)l * P->n_main * 2; A.sstride = 2;
    A.nt = nt; A.nacc = pitch; A.ne = 0;
    A.nbatch = batch;
    A.bpc = 1;
    dim3 grid(nt * groups, 1, batch);
    { lf_smem_optin(k_moddown_out<L1, L2, EPI_KS>, smR); LF_LAUNCH_CHECK(lf_launch(k_moddown_out<L1, L2, EPI_KS>, dim3(grid), dim3(S::TRR), smR, s, 1, A, dv)); }
    LF_CHECK_LAUNCH();
  }
  return 0;
}

// ModDown of both polynomials of an extended-basis ciphertext (poly.py:251-281 twice): row
// INTT of the 2 alpha special rows, BConv onto the main primes, row NTT + (x - conv) P^-1.
template <int L1, int L2>
static int moddown_pipeline(const LfCtx* ctx, int level, const u32* in, size_t in_bs, u32* out,
                            size_t out_bs, int batch, void* ws, cudaStream_t s) {
  using S = NttShape<L1, L2>;
  const LfKsPlan* P = ctx->ks;
  const int l1 = level + 1, alpha = P->n_special, ext = l1 + alpha;
  const size_t N = ctx->N;
  const LfDev dv = ctx->dev();
  const size_t smR = rowpass_smem_bytes<L1, L2>(0);
  const int groups = (1 << L1) / S::LPCR;
  u32* T2 = (u32*)ws;                              // per instance: 2 alpha rows, then T3: 2 (l+1)
  const size_t per = (2 * (size_t)alpha + 2 * (size_t)l1) * N;
  u32* T3 = T2 + 2 * (size_t)alpha * N;
  {
    dim3 grid(2 * alpha * groups, 1, batch);
    { lf_smem_optin(k_modup_in<L1, L2, 0>, smR); LF_LAUNCH_CHECK(lf_launch(k_modup_in<L1, L2, 0>, dim3(grid), dim3(S::TRR), smR, s, 1, in, nullptr, T2, in_bs, per, 2 * alpha, dv, alpha, ext, l1, P->L + 1, batch, 1, 1, (size_t)0, 0, MulList{})); }
    LF_CHECK_LAUNCH();
  }
  {
    BcArgs A{};
    A.src = T2; A.dst = T3; A.src_bs = per; A.dst_bs = per;
    A.ngroups = 2;
    for (int p = 0; p < 2; ++p) {
      A.g[p].B = P->down;
      A.g[p].B.m = l1;
      A.g[p].src_rows = P->iota;
      A.g[p].dst_rows = P->iota;
      A.g[p].src_row0 = p * alpha;
      A.g[p].dst_row0 = p * l1;
    }
    A.tsplit = bc_tsplit(2, batch, (1 << L2) / 8, l1);
    if (int e = launch_bc_auto<L1, L2>(ctx, A, batch, alpha, s)) return e;
  }
  {
    ModDownArgs A{};
    A.T3 = T3; A.acc = in; A.out = out; A.e0 = nullptr; A.e1 = nullptr;
    A.t3_bs = per; A.acc_bs = in_bs; A.out_bs = out_bs; A.e_bs = 0;
    A.scal = P->rowk + 2; A.sstride = 4; A.nt = l1; A.nacc = ext; A.ne = 0;
    A.nbatch = batch;
    A.bpc = 1;
    dim3 grid(l1 * groups, 1, batch);
    { lf_smem_optin(k_moddown_out<L1, L2, EPI_KS>, smR); LF_LAUNCH_CHECK(lf_launch(k_moddown_out<L1, L2, EPI_KS>, dim3(grid), dim3(S::TRR), smR, s, 1, A, dv)); }
    LF_CHECK_LAUNCH();
  }
  return 0;
}

template <int L1, int L2>
static int decompose_pipeline(const LfCtx* ctx, int level, const u32* x, u32* pieces, void* ws,
                              cudaStream_t s) {
  using S = NttShape<L1, L2>;
  const LfKsPlan* P = ctx->ks;
  const KsLevelPlan& K = P->lv[level];
  const int l1 = level + 1;
  const KsWs w = carve(ctx, level, ws);
  const LfDev dv = ctx->dev();
  const size_t smR = rowpass_smem_bytes<L1, L2>(0);
  const int groups = (1 << L1) / S::LPCR;
  {
    dim3 grid(l1 * groups, 1, 1);
    { lf_smem_optin(k_modup_in<L1, L2, 0>, smR); LF_LAUNCH_CHECK(lf_launch(k_modup_in<L1, L2, 0>, dim3(grid), dim3(S::TRR), smR, s, 1, x, nullptr, w.T0, 0, 0, l1, dv, l1, 0, 0, 0, 1, 1, 1, (size_t)0, 0, MulList{})); }
    LF_CHECK_LAUNCH();
  }
  {
    BcArgs A{};
    A.src = w.T0; A.dst = w.T1; A.ngroups = K.beta;
    int kmax = 0, mmax = 0;
    for (int j = 0; j < K.beta; ++j) {
      A.g[j] = K.up[j];
      kmax = K.up[j].B.k > kmax ? K.up[j].B.k : kmax;
      mmax = K.up[j].B.m > mmax ? K.up[j].B.m : mmax;
    }
    A.tsplit = bc_tsplit(K.beta, 1, (1 << L2) / 8, mmax);
    if (int e = launch_bc_auto<L1, L2>(ctx, A, 1, kmax, s)) return e;
  }
  {
    dim3 grid(K.beta * K.ext * groups);
    lf_smem_optin(k_pieces<L1, L2>, smR);
    LF_LAUNCH_CHECK(lf_launch(k_pieces<L1, L2>, dim3(grid), dim3(S::TRR), smR, s, 1, w.T1, x, pieces, P->rowk, level, P->d, P->L,
                                              P->n_special, dv));
    LF_CHECK_LAUNCH();
  }
  return 0;
}

// =======================================================================================
// C ABI
static int ks_check(const lf_ctx* ctx, int level) {
  if (!ctx) { lf_set_error("null context"); return 1; }
  if (!ctx->ks) { lf_set_error("keyswitch plans not built (call lf_ctx_enable_keyswitch)"); return 2; }
  if (level < 0 || level > ctx->ks->L) { lf_set_error("level %d outside [0, %d]", level, ctx->ks->L); return 2; }
  return 0;
}

static int run_ks_chunk(const lf_ctx* ctx, const KsCall& c, void* ws, cudaStream_t s,
                        cudaEvent_t* ev) {
#define LF_KS(A, B) { if (int e = ks_pipeline<A, B>(ctx, c, ws, s, ev)) return e; }
  LF_DISPATCH_LOGN(ctx->logN, LF_KS)
#undef LF_KS
  return 0;
}

// Instances are processed LF_MAXB at a time (the per-instance key / galois tables live in the
// kernel parameters); the workspace of a chunk is reused by the next one on the same stream.
static int run_ks(const lf_ctx* ctx, const KsCall& c, void* ws, cudaStream_t s,
                  cudaEvent_t* ev = nullptr) {
  if (c.batch <= LF_MAXB) return run_ks_chunk(ctx, c, ws, s, ev);
  if (ev) { lf_set_error("profiled keyswitch: batch > %d", LF_MAXB); return 2; }
  for (int b0 = 0; b0 < c.batch; b0 += LF_MAXB) {
    KsCall k = c;
    k.batch = c.batch - b0 < LF_MAXB ? c.batch - b0 : LF_MAXB;
    k.x = c.x + (c.hoisted ? 0 : b0 * c.x_bs);
    if (c.x2) k.x2 = c.x2 + (c.hoisted ? 0 : b0 * c.x2s());
    k.out = c.out + b0 * c.out_bs;
    if (c.e0) k.e0 = c.e0 + (c.hoisted ? 0 : b0 * c.e_bs);
    if (c.e1) k.e1 = c.e1 + (c.hoisted ? 0 : b0 * c.e1s());
    k.b0 = b0;
    if (int e = run_ks_chunk(ctx, k, ws, s, nullptr)) return e;
  }
  return 0;
}

// ModDown of extended-basis ciphertexts fused with a rescale by nd in {1, 2} primes: ONE exact
// floor division by P q_level [q_level-1] (the K.dr tables of lf_hom_mul_rescale), bit-identical
// to lf_moddown_ext followed by nd rescales.  The INTT row pass puts each polynomial's alpha
// special rows and its nd top main rows into T2 in the tables' source order.
template <int L1, int L2>
static int moddown_rescale_pipeline(const LfCtx* ctx, int level, int nd, const u32* in, size_t in_bs,
                                    u32* out, size_t out_bs, int batch, void* ws, cudaStream_t s) {
  using S = NttShape<L1, L2>;
  const LfKsPlan* P = ctx->ks;
  const KsLevelPlan& K = P->lv[level];
  const int l1 = level + 1, alpha = P->n_special, ext = l1 + alpha, nt = l1 - nd;
  const size_t N = ctx->N;
  const LfDev dv = ctx->dev();
  const size_t smR = rowpass_smem_bytes<L1, L2>(0);
  const int groups = (1 << L1) / S::LPCR;
  u32* T2 = (u32*)ws;                              // per instance: 2 (alpha + nd) rows, then T3: 2 nt
  const size_t per = (2 * (size_t)(alpha + nd) + 2 * (size_t)nt) * N;
  u32* T3 = T2 + 2 * (size_t)(alpha + nd) * N;
  lf_smem_optin(k_modup_in<L1, L2, 0>, smR);
  for (int p = 0; p < 2; ++p) {
    const u32* src = in + (size_t)p * ext * N;
    u32* t2p = T2 + (size_t)p * (alpha + nd) * N;
    {   // specials: input rows l+1 .. l+alpha, primes L+1 ..
      dim3 grid(alpha * groups, 1, batch);
      LF_LAUNCH_CHECK(lf_launch(k_modup_in<L1, L2, 0>, dim3(grid), dim3(S::TRR), smR, s, 1, src, nullptr, t2p, in_bs, per,
                                alpha, dv, alpha, 0, l1, P->L + 1, batch, 1, 1, (size_t)0, 0, MulList{}));
    }
    {   // the nd top main rows l-nd+1 .. l
      dim3 grid(nd * groups, 1, batch);
      LF_LAUNCH_CHECK(lf_launch(k_modup_in<L1, L2, 0>, dim3(grid), dim3(S::TRR), smR, s, 1, src, nullptr,
                                t2p + (size_t)alpha * N, in_bs, per, nd, dv, nd, 0, l1 - nd, l1 - nd, batch, 1, 1,
                                (size_t)0, 0, MulList{}));
    }
    LF_CHECK_LAUNCH();
  }
  {
    BcArgs A{};
    A.src = T2; A.dst = T3; A.src_bs = per; A.dst_bs = per;
    A.ngroups = 2;
    A.g[0] = K.dr[nd - 1][0];
    A.g[1] = K.dr[nd - 1][1];
    A.tsplit = bc_tsplit(2, batch, (1 << L2) / 8, nt);
    if (int e = launch_bc_auto<L1, L2>(ctx, A, batch, alpha + nd, s)) return e;
  }
  {
    ModDownArgs A{};
    A.T3 = T3; A.acc = in; A.out = out; A.e0 = nullptr; A.e1 = nullptr;
    A.t3_bs = per; A.acc_bs = in_bs; A.out_bs = out_bs; A.e_bs = 0;
    A.scal = P->pqinv[nd - 1] + (size_t)level * P->n_main * 2; A.sstride = 2;
    A.nt = nt; A.nacc = ext; A.ne = 0;
    A.nbatch = batch;
    A.bpc = 1;
    dim3 grid(nt * groups, 1, batch);
    { lf_smem_optin(k_moddown_out<L1, L2, EPI_KS>, smR); LF_LAUNCH_CHECK(lf_launch(k_moddown_out<L1, L2, EPI_KS>, dim3(grid), dim3(S::TRR), smR, s, 1, A, dv)); }
    LF_CHECK_LAUNCH();
  }
  return 0;
}

extern "C" {

int lf_set_bconv_engine(int engine) {
  if (engine != 0 && engine != 1) { lf_set_error("bconv engine %d (0: IMAD, 1: tensor cores)", engine); return 2; }
  g_bc_engine = engine;
  return 0;
}
int lf_get_bconv_engine(void) { return bc_engine(); }

int lf_ctx_enable_keyswitch(lf_ctx* ctx, int n_main, int d) {
  if (!ctx) { lf_set_error("null context"); return 1; }
  return lf_build_ks_plan(ctx, n_main, d);
}

size_t lf_ks_workspace_bytes(const lf_ctx* ctx, int level, int batch) {
  if (ks_check(ctx, level)) return 0;
  return ks_ws_rows(ctx->ks, level) * (size_t)ctx->N * 4 * (size_t)(batch < 1 ? 1 : batch);
}

int lf_keyswitch(const lf_ctx* ctx, int level, const uint32_t* x, size_t x_bstride,
                 const uint32_t* evk, size_t evk_bstride, uint32_t* out, size_t out_bstride,
                 int batch, void* workspace, void* stream) {
  if (int e = ks_check(ctx, level)) return e;
  if (!x || !evk || !out || !workspace) { lf_set_error("lf_keyswitch: null argument"); return 1; }
  KsCall c{};
  c.level = level; c.batch = batch; c.op = OP_KS;
  c.x = x; c.x2 = x; c.x_bs = x_bstride; c.key = evk; c.key_bs = evk_bstride;
  c.out = out; c.out_bs = out_bstride;
  return run_ks(ctx, c, workspace, (cudaStream_t)stream);
}

int lf_hom_mul(const lf_ctx* ctx, int level, const uint32_t* ct1, const uint32_t* ct2,
               size_t ct_bstride, const uint32_t* rlk, uint32_t* out, size_t out_bstride,
               int batch, void* workspace, void* stream) {
  if (int e = ks_check(ctx, level)) return e;
  if (!ct1 || !ct2 || !rlk || !out || !workspace) { lf_set_error("lf_hom_mul: null argument"); return 1; }
  const size_t arow = (size_t)(level + 1) * ctx->N;
  KsCall c{};
  c.level = level; c.batch = batch; c.op = OP_MUL;
  c.x = ct1 + arow; c.x2 = ct2 + arow; c.x_bs = ct_bstride; c.key = rlk; c.key_bs = 0;
  c.out = out; c.out_bs = out_bstride; c.e0 = ct1; c.e1 = ct2; c.e_bs = ct_bstride;
  return run_ks(ctx, c, workspace, (cudaStream_t)stream);
}

int lf_hom_mul_rescale(const lf_ctx* ctx, int level, int ndrop, const uint32_t* ct1,
                       const uint32_t* ct2, size_t ct_bstride, const uint32_t* rlk, uint32_t* out,
                       size_t out_bstride, int batch, void* workspace, void* stream) {
  return lf_hom_mul_rescale_p(ctx, level, ndrop, ct1, ct_bstride, level + 1, ct2, ct_bstride, level + 1, rlk,
                              out, out_bstride, batch, workspace, stream);
}

int lf_hom_mul_rescale_p(const lf_ctx* ctx, int level, int ndrop, const uint32_t* ct1, size_t ct1_bstride,
                         int ct1_pitch, const uint32_t* ct2, size_t ct2_bstride, int ct2_pitch,
                         const uint32_t* rlk, uint32_t* out, size_t out_bstride, int batch, void* workspace,
                         void* stream) {
  if (int e = ks_check(ctx, level)) return e;
  if (!ct1 || !ct2 || !rlk || !out || !workspace) { lf_set_error("lf_hom_mul_rescale: null argument"); return 1; }
  if (ndrop < 1 || ndrop > 2 || level < ndrop) {
    lf_set_error("lf_hom_mul_rescale: cannot drop %d primes at level %d", ndrop, level);
    return 2;
  }
  if (ct1_pitch < level + 1 || ct2_pitch < level + 1) {
    lf_set_error("lf_hom_mul_rescale_p: row pitch %d / %d < level + 1", ct1_pitch, ct2_pitch);
    return 2;
  }
  KsCall c{};
  c.level = level; c.batch = batch; c.op = OP_MUL; c.rescale_nd = ndrop;
  c.pitch = ct1_pitch; c.pitch2 = ct2_pitch; c.sep2 = true;
  c.x = ct1 + (size_t)ct1_pitch * ctx->N; c.x2 = ct2 + (size_t)ct2_pitch * ctx->N;
  c.x_bs = ct1_bstride; c.x2_bs = ct2_bstride; c.key = rlk; c.key_bs = 0;
  c.out = out; c.out_bs = out_bstride; c.e0 = ct1; c.e1 = ct2; c.e_bs = ct1_bstride; c.e1_bs = ct2_bstride;
  return run_ks(ctx, c, workspace, (cudaStream_t)stream);
}

int lf_hom_mul_rescale_list(const lf_ctx* ctx, int level, int ndrop, const uint32_t* const* ct1s,
                            const int* pitch1, const uint32_t* const* ct2s, const int* pitch2,
                            const int64_t* add_b, const uint32_t* rlk, uint32_t* out, size_t out_bstride,
                            int batch, void* workspace, void* stream) {
  if (int e = ks_check(ctx, level)) return e;
  if (!ct1s || !ct2s || !pitch1 || !pitch2 || !rlk || !out || !workspace || batch < 1) {
    lf_set_error("lf_hom_mul_rescale_list: bad argument");
    return 1;
  }
  if (ndrop < 1 || ndrop > 2 || level < ndrop) {
    lf_set_error("lf_hom_mul_rescale_list: cannot drop %d primes at level %d", ndrop, level);
    return 2;
  }
  for (int b = 0; b < batch; ++b)
    if (!ct1s[b] || !ct2s[b] || pitch1[b] < level + 1 || pitch2[b] < level + 1) {
      lf_set_error("lf_hom_mul_rescale_list: instance %d: null operand or row pitch < level + 1", b);
      return 2;
    }
  KsCall c{};
  c.level = level; c.batch = batch; c.op = OP_MUL; c.rescale_nd = ndrop;
  c.c1l = ct1s; c.c2l = ct2s; c.p1l = pitch1; c.p2l = pitch2; c.addl = add_b;
  c.x = ct1s[0] + (size_t)pitch1[0] * ctx->N; c.x2 = ct2s[0] + (size_t)pitch2[0] * ctx->N; c.x_bs = 0;
  c.key = rlk; c.key_bs = 0;
  c.out = out; c.out_bs = out_bstride; c.e0 = ct1s[0]; c.e1 = ct2s[0]; c.e_bs = 0;
  return run_ks(ctx, c, workspace, (cudaStream_t)stream);
}

int lf_rotate(const lf_ctx* ctx, int level, const uint32_t* ct, size_t ct_bstride, uint32_t g,
              const uint32_t* key, size_t key_bstride, uint32_t* out, size_t out_bstride,
              int batch, void* workspace, void* stream) {
  if (int e = ks_check(ctx, level)) return e;
  if (!ct || !key || !out || !workspace) { lf_set_error("lf_rotate: null argument"); return 1; }
  if (!(g & 1)) { lf_set_error("lf_rotate: galois element must be odd"); return 2; }
  const size_t arow = (size_t)(level + 1) * ctx->N;
  KsCall c{};
  c.level = level; c.batch = batch; c.op = OP_ROT;
  c.x = ct + arow; c.x2 = c.x; c.x_bs = ct_bstride; c.key = key; c.key_bs = key_bstride;
  c.out = out; c.out_bs = out_bstride; c.e0 = ct; c.e1 = nullptr; c.e_bs = ct_bstride;
  c.g = g & ((2u << ctx->logN) - 1);
  return run_ks(ctx, c, workspace, (cudaStream_t)stream);
}

int lf_keyswitch_profiled(const lf_ctx* ctx, int level, const uint32_t* x, size_t x_bstride,
                          const uint32_t* evk, size_t evk_bstride, uint32_t* out,
                          size_t out_bstride, int batch, void* workspace, void* stream,
                          float* stage_ms) {
  if (int e = ks_check(ctx, level)) return e;
  if (!x || !evk || !out || !workspace || !stage_ms) { lf_set_error("lf_keyswitch_profiled: null argument"); return 1; }
  KsCall c{};
  c.level = level; c.batch = batch; c.op = OP_KS;
  c.x = x; c.x2 = x; c.x_bs = x_bstride; c.key = evk; c.key_bs = evk_bstride;
  c.out = out; c.out_bs = out_bstride;
  cudaEvent_t ev[6];
  for (auto& e : ev) cudaEventCreate(&e);
  int rc = run_ks(ctx, c, workspace, (cudaStream_t)stream, ev);
  if (!rc) {
    cudaEventSynchronize(ev[5]);
    for (int i = 0; i < 5; ++i) cudaEventElapsedTime(&stage_ms[i], ev[i], ev[i + 1]);
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return rc;
}

size_t lf_rotate_hoisted_workspace_bytes(const lf_ctx* ctx, int level, int n_rot) {
  if (ks_check(ctx, level)) return 0;
  const int n = n_rot < LF_MAXB ? (n_rot < 1 ? 1 : n_rot) : LF_MAXB;
  return (ks_ws_rows_shared(ctx->ks, level) + (size_t)n * ks_ws_rows_inst(ctx->ks, level)) *
         (size_t)ctx->N * 4;
}

int lf_rotate_hoisted(const lf_ctx* ctx, int level, const uint32_t* ct, int n_rot,
                      const uint32_t* gs, const uint32_t* const* keys, uint32_t* out,
                      size_t out_bstride, void* workspace, void* stream) {
  if (int e = ks_check(ctx, level)) return e;
  if (!ct || !gs || !keys || !out || !workspace || n_rot < 1) {
    lf_set_error("lf_rotate_hoisted: bad argument");
    return 1;
  }
  for (int r = 0; r < n_rot; ++r)
    if (!(gs[r] & 1) || !keys[r]) { lf_set_error("lf_rotate_hoisted: rotation %d: bad key or even galois element", r); return 2; }
  const size_t arow = (size_t)(level + 1) * ctx->N;
  KsCall c{};
  c.level = level; c.batch = n_rot; c.op = OP_ROT; c.hoisted = true;
  c.x = ct + arow; c.x2 = c.x; c.x_bs = 0; c.keylist = keys;
  c.out = out; c.out_bs = out_bstride; c.e0 = ct; c.e1 = nullptr; c.e_bs = 0;
  c.glist = gs;
  return run_ks(ctx, c, workspace, (cudaStream_t)stream);
}

static int rotate_batch_impl(const lf_ctx* ctx, int level, const uint32_t* cts, size_t ct_bstride,
                             int n, const uint32_t* gs, const uint32_t* const* keys, uint32_t* out,
                             size_t out_bstride, void* workspace, void* stream, bool kperm) {
  if (int e = ks_check(ctx, level)) return e;
  if (!cts || !gs || !keys || !out || !workspace || n < 1) {
    lf_set_error("lf_rotate_batch: bad argument");
    return 1;
  }
  for (int r = 0; r < n; ++r)
    if (!(gs[r] & 1) || !keys[r]) { lf_set_error("lf_rotate_batch: instance %d: bad key or even galois element", r); return 2; }
  const size_t arow = (size_t)(level + 1) * ctx->N;
  KsCall c{};
  c.level = level; c.batch = n; c.op = OP_ROT; c.hoisted = false;
  c.x = cts + arow; c.x2 = c.x; c.x_bs = ct_bstride; c.keylist = keys;
  c.out = out; c.out_bs = out_bstride; c.e0 = cts; c.e1 = nullptr; c.e_bs = ct_bstride;
  c.glist = gs; c.kperm = kperm;
  return run_ks(ctx, c, workspace, (cudaStream_t)stream);
}

int lf_rotate_batch(const lf_ctx* ctx, int level, const uint32_t* cts, size_t ct_bstride, int n,
                    const uint32_t* gs, const uint32_t* const* keys, uint32_t* out,
                    size_t out_bstride, void* workspace, void* stream) {
  return rotate_batch_impl(ctx, level, cts, ct_bstride, n, gs, keys, out, out_bstride, workspace,
                           stream, false);
}

int lf_rotate_batch_pk(const lf_ctx* ctx, int level, const uint32_t* cts, size_t ct_bstride, int n,
                       const uint32_t* gs, const uint32_t* const* keys, uint32_t* out,
                       size_t out_bstride, void* workspace, void* stream) {
  return rotate_batch_impl(ctx, level, cts, ct_bstride, n, gs, keys, out, out_bstride, workspace,
                           stream, true);
}

size_t lf_rescale_workspace_bytes(const lf_ctx* ctx, int level, int batch) {
  if (!ctx) return 0;
  return (2 + 2 * (size_t)level) * ctx->N * 4 * (size_t)(batch < 1 ? 1 : batch);
}

int lf_rescale(const lf_ctx* ctx, int level, const uint32_t* ct, size_t ct_bstride,
               uint32_t* out, size_t out_bstride, int batch, void* workspace, void* stream) {
  if (int e = ks_check(ctx, level)) return e;
  if (level < 1) { lf_set_error("rescale at level 0"); return 2; }
  if (!ct || !out || !workspace) { lf_set_error("lf_rescale: null argument"); return 1; }
#define LF_RS(A, B) { if (int e = rescale_pipeline<A, B>(ctx, level, 1, ct, ct_bstride, out, out_bstride, batch, workspace, (cudaStream_t)stream)) return e; }
  LF_DISPATCH_LOGN(ctx->logN, LF_RS)
#undef LF_RS
  return 0;
}

int lf_rescale_multi(const lf_ctx* ctx, int level, int ndrop, const uint32_t* ct, size_t ct_bstride,
                     uint32_t* out, size_t out_bstride, int batch, void* workspace, void* stream) {
  return lf_rescale_multi_p(ctx, level, ndrop, ct, ct_bstride, level + 1, out, out_bstride, batch, workspace, stream);
}

int lf_rescale_multi_p(const lf_ctx* ctx, int level, int ndrop, const uint32_t* ct, size_t ct_bstride, int ct_pitch,
                       uint32_t* out, size_t out_bstride, int batch, void* workspace, void* stream) {
  if (int e = ks_check(ctx, level)) return e;
  if (ct_pitch < level + 1) { lf_set_error("lf_rescale_multi_p: row pitch %d < level + 1", ct_pitch); return 2; }
  if (ndrop < 1 || ndrop > 2) { lf_set_error("lf_rescale_multi: ndrop %d not in {1, 2}", ndrop); return 2; }
  if (level < ndrop) { lf_set_error("rescale by %d primes at level %d", ndrop, level); return 2; }
  if (!ct || !out || !workspace) { lf_set_error("lf_rescale_multi: null argument"); return 1; }
#define LF_RS(A, B) { if (int e = rescale_pipeline<A, B>(ctx, level, ndrop, ct, ct_bstride, out, out_bstride, batch, workspace, (cudaStream_t)stream, ct_pitch)) return e; }
  LF_DISPATCH_LOGN(ctx->logN, LF_RS)
#undef LF_RS
  return 0;
}

static int rotate_hoisted_ext_impl(const lf_ctx* ctx, int level, const uint32_t* ct, int n_rot,
                                   const uint32_t* gs, const uint32_t* const* keys, uint32_t* out_ext,
                                   size_t out_bstride, void* workspace, void* stream, bool kperm) {
  if (int e = ks_check(ctx, level)) return e;
  if (!ct || !gs || !keys || !out_ext || !workspace || n_rot < 1) {
    lf_set_error("lf_rotate_hoisted_ext: bad argument");
    return 1;
  }
  for (int r = 0; r < n_rot; ++r)
    if (!(gs[r] & 1) || !keys[r]) { lf_set_error("lf_rotate_hoisted_ext: rotation %d: bad key or even galois element", r); return 2; }
  const size_t arow = (size_t)(level + 1) * ctx->N;
  KsCall c{};
  c.level = level; c.batch = n_rot; c.op = OP_ROT; c.hoisted = true; c.ext_out = true;
  c.x = ct + arow; c.x2 = c.x; c.x_bs = 0; c.keylist = keys;
  c.out = out_ext; c.out_bs = out_bstride; c.e0 = ct; c.e1 = nullptr; c.e_bs = 0;
  c.glist = gs; c.kperm = kperm;
  return run_ks(ctx, c, workspace, (cudaStream_t)stream);
}

int lf_rotate_hoisted_ext(const lf_ctx* ctx, int level, const uint32_t* ct, int n_rot,
                          const uint32_t* gs, const uint32_t* const* keys, uint32_t* out_ext,
                          size_t out_bstride, void* workspace, void* stream) {
  return rotate_hoisted_ext_impl(ctx, level, ct, n_rot, gs, keys, out_ext, out_bstride, workspace,
                                 stream, false);
}

int lf_rotate_hoisted_ext_pk(const lf_ctx* ctx, int level, const uint32_t* ct, int n_rot,
                             const uint32_t* gs, const uint32_t* const* keys, uint32_t* out_ext,
                             size_t out_bstride, void* workspace, void* stream) {
  return rotate_hoisted_ext_impl(ctx, level, ct, n_rot, gs, keys, out_ext, out_bstride, workspace,
                                 stream, true);
}

int lf_bsgs_ext(const lf_ctx* ctx, int level, const uint32_t* ct, int n_rot, const uint32_t* gs,
                const uint32_t* const* keys, int n_giant, const uint32_t* const* pts, uint32_t* out,
                void* workspace, void* stream) {
  if (int e = ks_check(ctx, level)) return e;
  if (!ct || !gs || !keys || !pts || !out || !workspace || n_rot < 1 || n_rot > LF_BSGS_RMAX ||
      n_giant < 1 || n_giant > LF_BSGS_GMAX) {
    lf_set_error("lf_bsgs_ext: bad argument (n_rot %d <= %d, n_giant %d <= %d)", n_rot, LF_BSGS_RMAX,
                 n_giant, LF_BSGS_GMAX);
    return 1;
  }
  for (int r = 0; r < n_rot; ++r)
    if (!(gs[r] & 1) || !keys[r]) { lf_set_error("lf_bsgs_ext: rotation %d: bad key or even galois element", r); return 2; }
  BsgsExtArgs B{};
  B.ct = ct; B.out = out; B.nrot = n_rot; B.ngiant = n_giant;
  for (int r = 0; r < n_rot; ++r) { B.keyp[r] = keys[r]; B.gs[r] = gs[r] & ((2u << ctx->logN) - 1); }
  for (int k = 0; k < n_giant; ++k)
    for (int r = 0; r <= n_rot; ++r) B.pt[k][r] = pts[(size_t)k * (n_rot + 1) + r];
  const size_t arow = (size_t)(level + 1) * ctx->N;
  KsCall c{};
  c.level = level; c.batch = n_rot; c.op = OP_ROT; c.hoisted = true; c.ext_out = true; c.kperm = true;
  c.x = ct + arow; c.x2 = c.x; c.x_bs = 0; c.keylist = keys;
  c.out = out; c.out_bs = 0; c.e0 = ct; c.e1 = nullptr; c.e_bs = 0;
  c.glist = gs; c.bsgs = &B;
  return run_ks_chunk(ctx, c, workspace, (cudaStream_t)stream, nullptr);
}

size_t lf_moddown_workspace_bytes(const lf_ctx* ctx, int level, int batch) {
  if (ks_check(ctx, level)) return 0;
  return (2 * (size_t)ctx->ks->n_special + 2 * (size_t)(level + 1)) * ctx->N * 4 *
         (size_t)(batch < 1 ? 1 : batch);
}

int lf_moddown_ext_rescale(const lf_ctx* ctx, int level, int ndrop, const uint32_t* in_ext, size_t in_bstride,
                           uint32_t* out, size_t out_bstride, int batch, void* workspace, void* stream) {
  if (int e = ks_check(ctx, level)) return e;
  if (!in_ext || !out || !workspace || batch < 1) { lf_set_error("lf_moddown_ext_rescale: bad argument"); return 1; }
  if (ndrop < 1 || ndrop > 2 || level < ndrop) {
    lf_set_error("lf_moddown_ext_rescale: cannot drop %d primes at level %d", ndrop, level);
    return 2;
  }
#define LF_MDR(A, B) { if (int e = moddown_rescale_pipeline<A, B>(ctx, level, ndrop, in_ext, in_bstride, out, out_bstride, batch, workspace, (cudaStream_t)stream)) return e; }
  LF_DISPATCH_LOGN(ctx->logN, LF_MDR)
#undef LF_MDR
  return 0;
}

int lf_moddown_ext(const lf_ctx* ctx, int level, const uint32_t* in_ext, size_t in_bstride,
                   uint32_t* out, size_t out_bstride, int batch, void* workspace, void* stream) {
  if (int e = ks_check(ctx, level)) return e;
  if (!in_ext || !out || !workspace || batch < 1) { lf_set_error("lf_moddown_ext: bad argument"); return 1; }
#define LF_MD(A, B) { if (int e = moddown_pipeline<A, B>(ctx, level, in_ext, in_bstride, out, out_bstride, batch, workspace, (cudaStream_t)stream)) return e; }
  LF_DISPATCH_LOGN(ctx->logN, LF_MD)
#undef LF_MD
  return 0;
}

int lf_ks_decompose(const lf_ctx* ctx, int level, const uint32_t* x, uint32_t* pieces,
                    void* workspace, void* stream) {
  if (int e = ks_check(ctx, level)) return e;
  if (!x || !pieces || !workspace) { lf_set_error("lf_ks_decompose: null argument"); return 1; }
#define LF_DC(A, B) { if (int e = decompose_pipeline<A, B>(ctx, level, x, pieces, workspace, (cudaStream_t)stream)) return e; }
  LF_DISPATCH_LOGN(ctx->logN, LF_DC)
#undef LF_DC
  return 0;
}

}  // extern "C"

// =======================================================================================
// Limb-sharded keyswitch (reference multidev.py:55-56 placement, InputBroadcast
// pattern multidev.py:172-185, 291-412).  The five fused kernels run on this rank's rows only;
// the two cross-limb stages read all-gathered buffers:
//   phase 0  K_A  row INTT of the local main rows of x            -> T0s (m_slots rows)
//   gather   T0s of every rank                                    -> T0g
//   phase 1  K_BC ModUp: every digit's sources from T0g, targets = local extended rows;
//            K_C  row NTT + key inner product with the LOCAL key rows; local special rows'
//            row INTT                                             -> acc, T2s (2 s_slots rows)
//   gather   T2s of every rank                                    -> T2g
//   phase 2  K_BC ModDown from T2g onto the local main rows; K_E (acc - conv) P^-1 + epilogue
// Modular sums are associative and the gathers move exact residues, so every output residue
// equals the single-device pipeline's.
#include <dlfcn.h>
#include <nccl.h>

struct lf_comm {
  ncclComm_t comm;
  int nranks, rank;
};

namespace {
struct NcclApi {
  ncclResult_t (*get_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  const char* (*err)(ncclResult_t) = nullptr;
  bool ok = false;
};
// NCCL is resolved at run time from the libnccl already loaded by the process (torch's), so
// the library never carries a second NCCL.
const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.get_id = (decltype(a.get_id))dlsym(h, "ncclGetUniqueId");
    a.init_rank = (decltype(a.init_rank))dlsym(h, "ncclCommInitRank");
    a.all_gather = (decltype(a.all_gather))dlsym(h, "ncclAllGather");
    a.destroy = (decltype(a.destroy))dlsym(h, "ncclCommDestroy");
    a.err = (decltype(a.err))dlsym(h, "ncclGetErrorString");
    a.ok = a.get_id && a.init_rank && a.all_gather && a.destroy && a.err;
    return a;
  }();
  return api;
}
}  // namespace

struct ShardWs {
  u32 *T0s, *T0g, *T1, *acc, *T2s, *T2g, *T3;
  size_t t0_rows, t2_rows;       // rows each rank sends per gather (whole batch)
};

static ShardWs shard_carve(const LfCtx* ctx, const LfShardPlan* P, int level, int batch, void* ws) {
  const ShardLevel& S = P->lv[level];
  const size_t N = ctx->N, B = batch;
  ShardWs w;
  u32* p = (u32*)ws;
  w.t0_rows = B * S.m_slots;
  w.t2_rows = B * 2 * P->s_slots;
  w.T0s = p; p += w.t0_rows * N;
  w.T0g = p; p += P->k * w.t0_rows * N;
  w.T1 = p;  p += B * S.beta * S.ext * N;
  w.acc = p; p += B * 2 * S.n_main * N;
  w.T2s = p; p += w.t2_rows * N;
  w.T2g = p; p += P->k * w.t2_rows * N;
  w.T3 = p;  p += B * 2 * S.n_main * N;
  return w;
}
static size_t shard_ws_words(const LfCtx* ctx, const LfShardPlan* P, int level, int batch) {
  ShardWs w = shard_carve(ctx, P, level, batch, nullptr);
  return (size_t)(w.T3 - (u32*)nullptr) + (size_t)batch * 2 * P->lv[level].n_main * ctx->N;
}

template <int L1, int L2>
static int shard_phase(const LfCtx* ctx, const LfShardPlan* P, int phase, const lf_shard_call* c, void* ws,
                       cudaStream_t s) {
  using S_ = NttShape<L1, L2>;
  const LfKsPlan* K = ctx->ks;
  const int level = c->level, B = c->batch;
  const ShardLevel& S = P->lv[level];
  const ShardWs w = shard_carve(ctx, P, level, B, ws);
  const size_t N = ctx->N;
  const LfDev dv = ctx->dev();
  const size_t smR = rowpass_smem_bytes<L1, L2>(0);
  const int groups = (1 << L1) / S_::LPCR;
  const int nm = S.n_main;
  if (phase == 0) {
    if (nm == 0) return 0;
    const int bpc = B >= 2 * LF_BPC ? LF_BPC : 1;
    dim3 grid(nm * groups, 1, (B + bpc - 1) / bpc);
    const size_t tbs = (size_t)S.m_slots * N;
    if (c->op == OP_MUL) { lf_smem_optin(k_modup_in<L1, L2, 1>, smR); LF_LAUNCH_CHECK(lf_launch(k_modup_in<L1, L2, 1>, grid, dim3(S_::TRR), smR, s, 1, c->x, c->x2, w.T0s, c->x_bstride, tbs, nm, dv, nm, 0, 0, P->rank, B, bpc, P->k, c->x_bstride, 0, MulList{})); }
    else { lf_smem_optin(k_modup_in<L1, L2, 0>, smR); LF_LAUNCH_CHECK(lf_launch(k_modup_in<L1, L2, 0>, grid, dim3(S_::TRR), smR, s, 1, c->x, (const u32*)nullptr, w.T0s, c->x_bstride, tbs, nm, dv, nm, 0, 0, P->rank, B, bpc, P->k, (size_t)0, 0, MulList{})); }
    LF_CHECK_LAUNCH();
    return 0;
  }
  if (phase == 1) {
    {   // K_BC ModUp
      BcArgs A{};
      A.src = w.T0g; A.dst = w.T1; A.src_bs = (size_t)S.m_slots * N; A.dst_bs = (size_t)S.beta * S.ext * N;
      A.src_rstride = (int)w.t0_rows;
      int kmax = 0, mmax = 0, ng = 0;
      for (int j = 0; j < S.beta; ++j) {
        if (!S.up_m[j]) continue;
        A.g[ng] = S.up[j];
        kmax = S.up[j].B.k > kmax ? S.up[j].B.k : kmax;
        mmax = S.up[j].B.m > mmax ? S.up[j].B.m : mmax;
        ++ng;
      }
      A.ngroups = ng;
      if (ng) {
        A.tsplit = bc_tsplit(ng, B, (1 << L2) / 8, mmax, env_int("LF_TSPLIT_UP", 96));
        if (int e = launch_bc_auto<L1, L2>(ctx, A, B, kmax, s)) return e;
      }
    }
    {   // K_C
      KsInnerArgs A{};
      A.T1 = w.T1; A.x = c->x; A.x2 = c->x2 ? c->x2 : c->x; A.acc = w.acc; A.T2 = w.T2s;
      A.t1_bs = (size_t)S.beta * S.ext * N; A.x_bs = c->x_bstride; A.x2_bs = c->x_bstride; A.acc_bs = (size_t)2 * nm * N;
      A.t2_bs = (size_t)2 * P->s_slots * N;
      A.rowk = K->rowk; A.level = level; A.d = K->d; A.beta = S.beta; A.L = K->L; A.alpha = K->n_special;
      A.R = P->n_key_rows; A.nbatch = B; A.pre = 0; A.ext_out = 0; A.fuse_nd = 0; A.t2_rows = P->s_slots;
      A.pmod = K->pmod;
      A.tmap = S.tmap; A.kmap = S.kmap; A.n_main_st = nm; A.ext_st = S.ext;
      for (int b = 0; b < B; ++b) { A.keyp[b] = c->keys[b]; A.gs[b] = c->galois ? c->galois[b] : 1u; }
      const size_t smC = rowpass_smem_bytes<L1, L2>(LineCfg<L2>::M);
      dim3 grid(S.ext * groups * B);
      if (S.ext) {
        if (c->op == OP_ROT) { lf_smem_optin(k_ks_inner<L1, L2, 1, 0>, smC); LF_LAUNCH_CHECK(lf_launch(k_ks_inner<L1, L2, 1, 0>, grid, dim3(S_::TRR), smC, s, 1, A, dv)); }
        else if (c->op == OP_MUL) { lf_smem_optin(k_ks_inner<L1, L2, 0, 1>, smC); LF_LAUNCH_CHECK(lf_launch(k_ks_inner<L1, L2, 0, 1>, grid, dim3(S_::TRR), smC, s, 1, A, dv)); }
        else { lf_smem_optin(k_ks_inner<L1, L2, 0, 0>, smC); LF_LAUNCH_CHECK(lf_launch(k_ks_inner<L1, L2, 0, 0>, grid, dim3(S_::TRR), smC, s, 1, A, dv)); }
        LF_CHECK_LAUNCH();
      }
    }
    return 0;
  }
  if (nm == 0) return 0;
  {   // K_BC ModDown
    BcArgs A{};
    A.src = w.T2g; A.dst = w.T3; A.src_bs = (size_t)2 * P->s_slots * N; A.dst_bs = (size_t)2 * nm * N;
    A.src_rstride = (int)w.t2_rows;
    A.ngroups = 2;
    for (int p = 0; p < 2; ++p) {
      A.g[p] = P->down[p];
      A.g[p].B.m = nm;                     // prefix of the level-L local table
      A.g[p].dst_row0 = p * nm;
    }
    A.tsplit = bc_tsplit(2, B, (1 << L2) / 8, nm, env_int("LF_TSPLIT_DOWN", 96));
    if (int e = launch_bc_auto<L1, L2>(ctx, A, B, K->n_special, s)) return e;
  }
  {   // K_E
    ModDownArgs A{};
    A.T3 = w.T3; A.acc = w.acc; A.out = c->out; A.e0 = c->e0; A.e1 = c->e1;
    A.t3_bs = (size_t)2 * nm * N; A.acc_bs = A.t3_bs; A.out_bs = c->out_bstride; A.e_bs = c->e_bstride;
    A.e1_bs = c->e_bstride;
    A.scal = K->rowk + 2; A.sstride = 4; A.nt = nm; A.nacc = nm; A.ne = nm; A.ne1 = nm;
    A.tmap = S.tmap;
    for (int b = 0; b < B; ++b) A.gs[b] = c->galois ? c->galois[b] : 1u;
    A.nbatch = B;
    A.bpc = B >= 2 * LF_BPC ? LF_BPC : 1;
    dim3 grid(nm * groups, 1, (B + A.bpc - 1) / A.bpc);
    if (c->op == OP_MUL) { lf_smem_optin(k_moddown_out<L1, L2, EPI_MUL>, smR); LF_LAUNCH_CHECK(lf_launch(k_moddown_out<L1, L2, EPI_MUL>, grid, dim3(S_::TRR), smR, s, 1, A, dv)); }
    else if (c->op == OP_ROT) { lf_smem_optin(k_moddown_out<L1, L2, EPI_ROT>, smR); LF_LAUNCH_CHECK(lf_launch(k_moddown_out<L1, L2, EPI_ROT>, grid, dim3(S_::TRR), smR, s, 1, A, dv)); }
    else { lf_smem_optin(k_moddown_out<L1, L2, EPI_KS>, smR); LF_LAUNCH_CHECK(lf_launch(k_moddown_out<L1, L2, EPI_KS>, grid, dim3(S_::TRR), smR, s, 1, A, dv)); }
    LF_CHECK_LAUNCH();
  }
  return 0;
}

static int run_shard_phase(const LfCtx* ctx, const LfShardPlan* P, int phase, const lf_shard_call* c, void* ws,
                           cudaStream_t s) {
#define LF_SH(A, B_) { if (int e = shard_phase<A, B_>(ctx, P, phase, c, ws, s)) return e; }
  LF_DISPATCH_LOGN(ctx->logN, LF_SH)
#undef LF_SH
  return 0;
}

extern "C" {

struct lf_shard {
  const LfCtx* ctx;
  LfShardPlan* plan;
  cudaStream_t comm_stream;     // the all-gathers of an overlapped (two half-batch) keyswitch
  cudaEvent_t ev[8];
};

int lf_shard_create(const lf_ctx* ctx, int k, int rank, lf_shard** out) {
  if (!ctx || !out) { lf_set_error("lf_shard_create: null argument"); return 1; }
  LfShardPlan* P = nullptr;
  if (int e = lf_build_shard_plan(ctx, k, rank, &P)) return e;
  lf_shard* sh = new lf_shard{ctx, P, nullptr, {}};
  if (cudaStreamCreateWithFlags(&sh->comm_stream, cudaStreamNonBlocking) != cudaSuccess) sh->comm_stream = nullptr;
  for (int i = 0; i < 8 && sh->comm_stream; ++i)
    if (cudaEventCreateWithFlags(&sh->ev[i], cudaEventDisableTiming) != cudaSuccess) {
      for (int j = 0; j < i; ++j) cudaEventDestroy(sh->ev[j]);
      cudaStreamDestroy(sh->comm_stream);
      sh->comm_stream = nullptr;
    }
  *out = sh;
  return 0;
}

int lf_shard_destroy(lf_shard* sh) {
  if (!sh) return 0;
  if (sh->comm_stream) {
    for (int i = 0; i < 8; ++i) cudaEventDestroy(sh->ev[i]);
    cudaStreamDestroy(sh->comm_stream);
  }
  lf_free_shard_plan(sh->plan);
  delete sh;
  return 0;
}

int lf_shard_info(const lf_shard* sh, int level, int* n_main, int* n_ext, int* n_key_rows, int* n_special) {
  if (!sh || level < 0 || level > sh->plan->L) { lf_set_error("lf_shard_info: bad shard or level"); return 1; }
  const ShardLevel& S = sh->plan->lv[level];
  if (n_main) *n_main = S.n_main;
  if (n_ext) *n_ext = S.ext;
  if (n_key_rows) *n_key_rows = sh->plan->n_key_rows;
  if (n_special) *n_special = sh->plan->n_sp;
  return 0;
}

size_t lf_shard_ws_bytes(const lf_shard* sh, int level, int batch) {
  if (!sh || level < 0 || level > sh->plan->L || batch < 1) return 0;
  size_t w = shard_ws_words(sh->ctx, sh->plan, level, batch);
  if (batch >= 2) {            // two half-batch workspaces of the overlapped schedule
    const int h0 = (batch + 1) / 2;
    const size_t w2 = shard_ws_words(sh->ctx, sh->plan, level, h0) + shard_ws_words(sh->ctx, sh->plan, level, batch - h0);
    w = w2 > w ? w2 : w;
  }
  return w * 4;
}

int lf_shard_gather_layout(const lf_shard* sh, int level, int batch, size_t* out6) {
  if (!sh || !out6 || level < 0 || level > sh->plan->L || batch < 1) { lf_set_error("lf_shard_gather_layout: bad argument"); return 1; }
  const ShardWs w = shard_carve(sh->ctx, sh->plan, level, batch, nullptr);
  const size_t rb = (size_t)sh->ctx->N * 4;
  out6[0] = (size_t)((char*)w.T0s - (char*)nullptr); out6[1] = w.t0_rows * rb; out6[2] = (size_t)((char*)w.T0g - (char*)nullptr);
  out6[3] = (size_t)((char*)w.T2s - (char*)nullptr); out6[4] = w.t2_rows * rb; out6[5] = (size_t)((char*)w.T2g - (char*)nullptr);
  return 0;
}

static int shard_check(const lf_shard* sh, const lf_shard_call* c, void* ws) {
  if (!sh || !c || !ws) { lf_set_error("sharded keyswitch: null argument"); return 1; }
  if (c->level < 0 || c->level > sh->plan->L) { lf_set_error("sharded keyswitch: level %d", c->level); return 2; }
  if (c->batch < 1 || c->batch > LF_MAXB) { lf_set_error("sharded keyswitch: batch %d outside [1, %d]", c->batch, LF_MAXB); return 2; }
  if (c->op != OP_KS && c->op != OP_MUL && c->op != OP_ROT) { lf_set_error("sharded keyswitch: op %d", c->op); return 2; }
  if (!c->keys || (sh->plan->lv[c->level].n_main && (!c->x || !c->out))) { lf_set_error("sharded keyswitch: null argument"); return 1; }
  if ((c->op == OP_MUL && (!c->x2 || !c->e0 || !c->e1)) || (c->op == OP_ROT && (!c->e0 || !c->galois))) {
    lf_set_error("sharded keyswitch: op %d needs its epilogue operands", c->op);
    return 1;
  }
  return 0;
}

int lf_shard_ks_phase(const lf_shard* sh, int phase, const lf_shard_call* call, void* ws, void* stream) {
  if (int e = shard_check(sh, call, ws)) return e;
  if (phase < 0 || phase > 2) { lf_set_error("lf_shard_ks_phase: phase %d", phase); return 2; }
  return run_shard_phase(sh->ctx, sh->plan, phase, call, ws, (cudaStream_t)stream);
}

int lf_comm_unique_id(void* out128) {
  const NcclApi& a = nccl();
  if (!a.ok) { lf_set_error("NCCL not available (libnccl.so.2)"); return 3; }
  ncclUniqueId id;
  ncclResult_t r = a.get_id(&id);
  if (r != ncclSuccess) { lf_set_error("ncclGetUniqueId: %s", a.err(r)); return 3; }
  memcpy(out128, &id, sizeof(id));
  return 0;
}

int lf_comm_create(int nranks, int rank, const void* id128, lf_comm** out) {
  const NcclApi& a = nccl();
  if (!a.ok) { lf_set_error("NCCL not available (libnccl.so.2)"); return 3; }
  if (!id128 || !out || nranks < 1 || rank < 0 || rank >= nranks) { lf_set_error("lf_comm_create: bad argument"); return 1; }
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  lf_comm* c = new lf_comm{nullptr, nranks, rank};
  ncclResult_t r = a.init_rank(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) { delete c; lf_set_error("ncclCommInitRank: %s", a.err(r)); return 3; }
  *out = c;
  return 0;
}

int lf_comm_destroy(lf_comm* c) {
  if (!c) return 0;
  if (c->comm) nccl().destroy(c->comm);
  delete c;
  return 0;
}

int lf_shard_attach_comm(lf_shard* sh, lf_comm* comm) {
  if (!sh) { lf_set_error("lf_shard_attach_comm: null shard"); return 1; }
  if (comm && (comm->nranks != sh->plan->k || comm->rank != sh->plan->rank)) {
    lf_set_error("lf_shard_attach_comm: communicator rank %d/%d, shard %d/%d", comm->rank, comm->nranks,
                 sh->plan->rank, sh->plan->k);
    return 2;
  }
  sh->plan->comm = comm;
  return 0;
}

static int shard_gather(const lf_shard* sh, const ShardWs& w, bool modup, cudaStream_t s) {
  lf_comm* cm = (lf_comm*)sh->plan->comm;
  const size_t rb = (size_t)sh->ctx->N * 4;
  const void* src = modup ? w.T0s : w.T2s;
  void* dst = modup ? w.T0g : w.T2g;
  const size_t bytes = (modup ? w.t0_rows : w.t2_rows) * rb;
  if (cm) {
    ncclResult_t r = nccl().all_gather(src, dst, bytes, ncclUint8, cm->comm, s);
    if (r != ncclSuccess) { lf_set_error("ncclAllGather (%s): %s", modup ? "ModUp" : "ModDown", nccl().err(r)); return 3; }
  } else if (cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess) {
    lf_set_error("sharded keyswitch: copy failed"); return 3;
  }
  return 0;
}

// One limb-sharded keyswitch / hom_mul / rotation batch.  Batches of two or more run as two
// half-batches whose all-gathers go on the shard's comm stream, so each half's exchange overlaps
// the other half's kernels (phase 0 h0 | gather h0 + phase 0 h1 | phase 1 h0 + gather h1 | ...);
// the NCCL calls are issued in the same order on every rank.
int lf_shard_keyswitch(const lf_shard* sh, const lf_shard_call* call, void* ws, void* stream) {
  if (int e = shard_check(sh, call, ws)) return e;
  lf_comm* cm = (lf_comm*)sh->plan->comm;
  if (!cm && sh->plan->k > 1) { lf_set_error("lf_shard_keyswitch: no communicator attached (lf_shard_attach_comm)"); return 2; }
  cudaStream_t s = (cudaStream_t)stream;
  if (call->batch < 2 || !sh->comm_stream) {
    const ShardWs w = shard_carve(sh->ctx, sh->plan, call->level, call->batch, ws);
    if (int e = run_shard_phase(sh->ctx, sh->plan, 0, call, ws, s)) return e;
    if (int e = shard_gather(sh, w, true, s)) return e;
    if (int e = run_shard_phase(sh->ctx, sh->plan, 1, call, ws, s)) return e;
    if (int e = shard_gather(sh, w, false, s)) return e;
    return run_shard_phase(sh->ctx, sh->plan, 2, call, ws, s);
  }
  const int h0 = (call->batch + 1) / 2;
  lf_shard_call c[2] = {*call, *call};
  c[0].batch = h0;
  c[1].batch = call->batch - h0;
  if (call->x) c[1].x = call->x + (size_t)h0 * call->x_bstride;
  if (call->x2) c[1].x2 = call->x2 + (size_t)h0 * call->x_bstride;
  if (call->out) c[1].out = call->out + (size_t)h0 * call->out_bstride;
  if (call->e0) c[1].e0 = call->e0 + (size_t)h0 * call->e_bstride;
  if (call->e1) c[1].e1 = call->e1 + (size_t)h0 * call->e_bstride;
  c[1].keys = call->keys + h0;
  if (call->galois) c[1].galois = call->galois + h0;
  void* wsp[2] = {ws, (u32*)ws + shard_ws_words(sh->ctx, sh->plan, call->level, h0)};
  ShardWs w[2];
  for (int h = 0; h < 2; ++h) w[h] = shard_carve(sh->ctx, sh->plan, call->level, c[h].batch, wsp[h]);
  cudaStream_t cs = sh->comm_stream;
  cudaEvent_t* ev = const_cast<cudaEvent_t*>(sh->ev);
#define LF_SH(x) do { if (int e__ = (x)) return e__; } while (0)
#define LF_CU(x) do { if ((x) != cudaSuccess) { lf_set_error("sharded keyswitch: stream sync failed"); return 3; } } while (0)
  LF_SH(run_shard_phase(sh->ctx, sh->plan, 0, &c[0], wsp[0], s));
  LF_CU(cudaEventRecord(ev[0], s)); LF_CU(cudaStreamWaitEvent(cs, ev[0], 0));
  LF_SH(shard_gather(sh, w[0], true, cs));                                   // gather 1 of h0
  LF_CU(cudaEventRecord(ev[1], cs));
  LF_SH(run_shard_phase(sh->ctx, sh->plan, 0, &c[1], wsp[1], s));
  LF_CU(cudaEventRecord(ev[2], s));
  LF_CU(cudaStreamWaitEvent(s, ev[1], 0));
  LF_SH(run_shard_phase(sh->ctx, sh->plan, 1, &c[0], wsp[0], s));
  LF_CU(cudaEventRecord(ev[3], s));
  LF_CU(cudaStreamWaitEvent(cs, ev[2], 0));
  LF_SH(shard_gather(sh, w[1], true, cs));                                   // gather 1 of h1
  LF_CU(cudaEventRecord(ev[4], cs));
  LF_CU(cudaStreamWaitEvent(cs, ev[3], 0));
  LF_SH(shard_gather(sh, w[0], false, cs));                                  // gather 2 of h0
  LF_CU(cudaEventRecord(ev[5], cs));
  LF_CU(cudaStreamWaitEvent(s, ev[4], 0));
  LF_SH(run_shard_phase(sh->ctx, sh->plan, 1, &c[1], wsp[1], s));
  LF_CU(cudaEventRecord(ev[6], s));
  LF_CU(cudaStreamWaitEvent(s, ev[5], 0));
  LF_SH(run_shard_phase(sh->ctx, sh->plan, 2, &c[0], wsp[0], s));
  LF_CU(cudaStreamWaitEvent(cs, ev[6], 0));
  LF_SH(shard_gather(sh, w[1], false, cs));                                  // gather 2 of h1
  LF_CU(cudaEventRecord(ev[7], cs));
  LF_CU(cudaStreamWaitEvent(s, ev[7], 0));
  LF_SH(run_shard_phase(sh->ctx, sh->plan, 2, &c[1], wsp[1], s));
#undef LF_SH
#undef LF_CU
  return 0;
}

}  // extern "C"
