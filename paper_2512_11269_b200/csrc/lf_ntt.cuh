// Column-pass / row-pass building blocks of the two-pass negacyclic NTT.
#pragma once
#include "lf_common.cuh"

// Shared-memory addressing of a column tile: [p][c] with one pad row every E rows.
template <int LP, int CW>
struct AddrC {
  int c;
  LF_DEV int operator()(int p) const { return (p + (p >> LineCfg<LP>::LA)) * CW + c; }
};
// Row lines: [line][p] with one pad word every E words.
template <int LP>
struct AddrR {
  int base;
  LF_DEV int operator()(int p) const { return base + p + (p >> LineCfg<LP>::LA); }
};

template <int LP, int CW>
__host__ __device__ constexpr int smemC_words() {
  return (LineCfg<LP>::M + LineCfg<LP>::M / LineCfg<LP>::E) * CW;
}
template <int LP>
__host__ __device__ constexpr int pitchR() {
  return LineCfg<LP>::M + LineCfg<LP>::M / LineCfg<LP>::E;
}

// Default tile shapes.
template <int L1, int L2>
struct NttShape {
  static constexpr int NCOL = 1 << L2;
  static constexpr int CW = NCOL < 32 ? NCOL : 32;          // columns per pass-C CTA
  static constexpr int TC = LineCfg<L1>::T * CW;             // threads per pass-C CTA
  static constexpr int TR_LINE = LineCfg<L2>::T;
  static constexpr int LPC = (256 / TR_LINE) > 0 ? (256 / TR_LINE) : 1;   // lines per pass-R CTA
  static constexpr int TR = TR_LINE * LPC;
  // kernels whose CTA works on lines of ONE row (all lines share a prime): at most 2^L1 lines
  static constexpr int LPCR = LPC < (1 << L1) ? LPC : (1 << L1);
  static constexpr int TRR = TR_LINE * LPCR;
  // bound after any column pass (the BConv kernels feed it lazily reduced inputs < 4q)
  static constexpr int FWD_C_OUT = FwdLineBound<L1, 4>::value;
};

// ---- column pass loads/stores (thread (tl, c) of a CW-column tile) ----------------------
template <int L1, int L2>
LF_DEV void load_col_step1(u32* x, const u32* __restrict__ base, int tl) {
  using C = LineCfg<L1>;
#pragma unroll
  for (int j = 0; j < C::E; ++j) x[j] = base[(size_t)(tl + C::T * j) << L2];
}
template <int L1, int L2>
LF_DEV void load_col_step2(u32* x, const u32* __restrict__ base, int tl) {
  using C = LineCfg<L1>;
#pragma unroll
  for (int e = 0; e < C::E; ++e) x[e] = base[(size_t)(tl * C::E + e) << L2];
}
template <int L1, int L2>
LF_DEV void store_col_step1(const u32* x, u32* base, int tl) {
  using C = LineCfg<L1>;
#pragma unroll
  for (int j = 0; j < C::E; ++j) base[(size_t)(tl + C::T * j) << L2] = x[j];
}
template <int L1, int L2>
LF_DEV void store_col_step2(const u32* x, u32* base, int tl) {
  using C = LineCfg<L1>;
#pragma unroll
  for (int e = 0; e < C::E; ++e) base[(size_t)(tl * C::E + e) << L2] = x[e];
}

// ---- row pass loads/stores (thread tl of a line; base = start of the line) --------------
template <int L2>
LF_DEV void load_row_step1(u32* x, const u32* __restrict__ base, int tl) {
  using C = LineCfg<L2>;
#pragma unroll
  for (int j = 0; j < C::E; ++j) x[j] = base[tl + C::T * j];
}
template <int L2>
LF_DEV void load_row_step2(u32* x, const u32* __restrict__ base, int tl) {
  using C = LineCfg<L2>;
  if constexpr (C::E % 4 == 0) {
    const uint4* b4 = reinterpret_cast<const uint4*>(base + tl * C::E);
#pragma unroll
    for (int v = 0; v < C::E / 4; ++v) {
      uint4 t = b4[v];
      x[4 * v] = t.x; x[4 * v + 1] = t.y; x[4 * v + 2] = t.z; x[4 * v + 3] = t.w;
    }
  } else {
#pragma unroll
    for (int e = 0; e < C::E; ++e) x[e] = base[tl * C::E + e];
  }
}
template <int L2>
LF_DEV void store_row_step1(const u32* x, u32* base, int tl) {
  using C = LineCfg<L2>;
#pragma unroll
  for (int j = 0; j < C::E; ++j) base[tl + C::T * j] = x[j];
}
template <int L2>
LF_DEV void store_row_step2(const u32* x, u32* base, int tl) {
  using C = LineCfg<L2>;
  if constexpr (C::E % 4 == 0) {
    uint4* b4 = reinterpret_cast<uint4*>(base + tl * C::E);
#pragma unroll
    for (int v = 0; v < C::E / 4; ++v)
      b4[v] = make_uint4(x[4 * v], x[4 * v + 1], x[4 * v + 2], x[4 * v + 3]);
  } else {
#pragma unroll
    for (int e = 0; e < C::E; ++e) base[tl * C::E + e] = x[e];
  }
}

// Dispatch a functor templated on (L1, L2) for logN in [4, 16].
#define LF_DISPATCH_LOGN(logN, FN)                 \
  switch (logN) {                                  \
    case 4: FN(2, 2); break;                       \
    case 5: FN(2, 3); break;                       \
    case 6: FN(3, 3); break;                       \
    case 7: FN(3, 4); break;                       \
    case 8: FN(4, 4); break;                       \
    case 9: FN(4, 5); break;                       \
    case 10: FN(5, 5); break;                      \
    case 11: FN(5, 6); break;                      \
    case 12: FN(6, 6); break;                      \
    case 13: FN(6, 7); break;                      \
    case 14: FN(7, 7); break;                      \
    case 15: FN(7, 8); break;                      \
    case 16: FN(8, 8); break;                      \
    default: lf_set_error("unsupported logN %d", logN); return 2; \
  }

// Shared memory of a row-pass CTA (LPCR lines of one row): staged twiddle subtrees
// (LPCR * (2^L2 - 1) uint2), then per line the exchange buffer plus `extra` words.
template <int L1, int L2>
inline size_t rowpass_smem_bytes(int extra) {
  using S = NttShape<L1, L2>;
  return ((size_t)2 * S::LPCR * (LineCfg<L2>::M - 1) + 2 + (size_t)S::LPCR * (pitchR<L2>() + extra)) * 4;
}
template <int L1, int L2>
LF_DEV u32* rowpass_xs(u32* sm) {
  return sm + 2 * NttShape<L1, L2>::LPCR * (LineCfg<L2>::M - 1) + 2;
}
