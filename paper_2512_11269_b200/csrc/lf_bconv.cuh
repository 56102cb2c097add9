// Exact RNS base conversion (reference poly.py:140-178).
//
// For source primes s_1..s_k (product S) and a target prime t:
//   y_i = r_i * c_i mod s_i            (c_i = (S/s_i)^-1 mod s_i, optionally times extra factors)
//   u   = floor(sum_i y_i / s_i)       exact: float64 fast path, multiword decision when
//                                      |v - rint(v)| < 2^-40 (the reference's threshold)
//   out = sum_i y_i * ((S/s_i) mod t) + u * ((t - S mod t) mod t)   (mod t)
// which equals (exact CRT lift in [0, S)) mod t, bit for bit with the reference.
// Tables are target-major so that a prefix of the targets is itself a valid table
// (ModDown at level l uses the first l+1 targets of the level-L table).
#pragma once
#include "lf_common.cuh"

// Device view of a conversion table blob built by the host (see lf_bconv_layout below).
struct BconvDev {
  int k, m, W;
  const double* inv_s;   // [k]   1/s_i
  const u32* src_pi;     // [k]   prime index of source i
  const u32* c;          // [k]   y multiplier
  const u32* cp;         // [k]   Shoup companion of c
  const u32* tgt_pi;     // [m]   prime index of target t
  const u32* negS;       // [m]   (t - S mod t) mod t
  const u32* w;          // [m*k] (S/s_i) mod t, target-major: w[t*k + i]
  const u32* shat;       // [k*W] S/s_i as W little-endian 32-bit words
  const u32* S;          // [W]   S as W words
  // tensor-core form (k_bconv_tc), or null: per target t, 4 rows b = 0..3 of K bytes with
  // B[t][b][4i+a] = byte b of (2^(8a) (S/s_i) mod t) and B[t][b][4k] = byte b of negS[t], stored
  // as the UMMA canonical K-major operand (pairs of targets = 8-row core-matrix groups, 512 B)
  const unsigned char* w8;
  int kb;                // A-operand bytes per row the table was built for (48 or 64)
};

// Word offsets inside the blob (u32 units; inv_s first so the doubles are 8-byte aligned).
__host__ __device__ inline size_t lf_bconv_words(int k, int m, int W) {
  return (size_t)5 * k + 2 * (size_t)m + (size_t)k * m + (size_t)k * W + W;
}
__host__ __device__ inline BconvDev lf_bconv_view(const u32* base, int k, int m, int W) {
  BconvDev b;
  b.k = k; b.m = m; b.W = W;
  b.inv_s = reinterpret_cast<const double*>(base);
  b.src_pi = base + 2 * k;
  b.c = base + 3 * k;
  b.cp = base + 4 * k;
  b.tgt_pi = base + 5 * k;
  b.negS = base + 5 * k + m;
  b.w = base + 5 * k + 2 * m;
  b.shat = base + 5 * k + 2 * m + (size_t)k * m;
  b.S = b.shat + (size_t)k * W;
  b.w8 = nullptr;
  b.kb = 0;
  return b;
}

#define LF_BC_MAXW 64

// Exact decision for the risky case: returns r if sum y_i*Shat_i >= r*S else r-1.
LF_DEV u32 bconv_u_exact(const u32* y, const BconvDev& B, u32 r) {
  u32 a[LF_BC_MAXW + 2], b[LF_BC_MAXW + 2];
  const int W = B.W;
  for (int w = 0; w < W + 2; ++w) { a[w] = 0; b[w] = 0; }
  for (int i = 0; i < B.k; ++i) {
    u64 carry = 0;
    const u32* sh = B.shat + (size_t)i * W;
    for (int w = 0; w < W; ++w) {
      u64 t = (u64)y[i] * sh[w] + a[w] + carry;
      a[w] = (u32)t;
      carry = t >> 32;
    }
    for (int w = W; w < W + 2 && carry; ++w) {
      u64 t = (u64)a[w] + carry;
      a[w] = (u32)t;
      carry = t >> 32;
    }
  }
  u64 carry = 0;
  for (int w = 0; w < W; ++w) {
    u64 t = (u64)r * B.S[w] + carry;
    b[w] = (u32)t;
    carry = t >> 32;
  }
  b[W] = (u32)carry;
  for (int w = W + 1; w >= 0; --w) {
    if (a[w] != b[w]) return a[w] > b[w] ? r : r - 1;
  }
  return r;   // equal
}

// y[0..k) canonical residues -> exact overflow count u.
LF_DEV u32 bconv_u(const u32* y, const BconvDev& B) {
  double v = 0.0;
  for (int i = 0; i < B.k; ++i) v = fma((double)y[i], B.inv_s[i], v);
  const double r = rint(v);
  if (fabs(v - r) >= 0x1p-40) return (u32)floor(v);
  if (r == 0.0) {
    bool z = true;
    for (int i = 0; i < B.k; ++i) z &= (y[i] == 0);
    if (z) return 0;
  }
  return bconv_u_exact(y, B, (u32)r);
}
