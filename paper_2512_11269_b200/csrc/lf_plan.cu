// Host construction of the keyswitch / rescale plans (constants of reference ckks.py:85-140,
// poly.py:140-178, 251-287, keys.py:85-97), uploaded to HBM in one allocation.
#include <cmath>
#include <cstring>
#include <vector>

#include "lf_plan.h"

namespace {

typedef std::vector<u32> Big;   // little-endian 32-bit words

u32 mulm(u32 a, u32 b, u32 q) { return (u32)((u64)a * b % q); }
u32 powm(u32 b, u64 e, u32 q) {
  u64 r = 1, x = b % q;
  while (e) {
    if (e & 1) r = r * x % q;
    x = x * x % q;
    e >>= 1;
  }
  return (u32)r;
}
u32 invm(u32 a, u32 q) { return powm(a, q - 2, q); }
u32 shoupc(u32 w, u32 q) { return (u32)(((u64)w << 32) / q); }

void big_mul(Big& a, u32 m) {
  u64 carry = 0;
  for (auto& w : a) {
    u64 t = (u64)w * m + carry;
    w = (u32)t;
    carry = t >> 32;
  }
  if (carry) a.push_back((u32)carry);
}

struct Blob {
  std::vector<u32> w;
  size_t align2() {            // keep doubles 8-byte aligned
    if (w.size() & 1) w.push_back(0);
    return w.size();
  }
  size_t push(const std::vector<u32>& v) {
    size_t o = w.size();
    w.insert(w.end(), v.begin(), v.end());
    return o;
  }
};

struct TabRec {
  size_t off;
  int k, m, W;
  size_t w8off;            // word offset of the tensor-core byte table (0: none)
  int kb;
};

// Byte-split weights of the tensor-core base conversion (BconvDev::w8): for target t and
// output byte b, K-row [4i+a] = byte b of 2^(8a) (S/s_i) mod t, [4k] = byte b of negS[t].
// Layout: target pair p = t/2 is one 512-byte block of four 16-byte K-chunks x 8 rows
// (row (t%2)*4 + b), the canonical no-swizzle K-major UMMA operand (lf_umma.cuh).
size_t build_w8(Blob& b, const std::vector<u32>& primes, const std::vector<int>& tgt, int k,
                const std::vector<u32>& w, const std::vector<u32>& negS, int& kb) {
  const int m = (int)tgt.size();
  kb = 4 * k + 1 <= 48 ? 48 : 64;
  // k = 16 fills all 64 K-bytes with sources: the overflow term u * negS is then added in the
  // kernel's epilogue instead of riding along as K-row 4k
  const int krows = 4 * k + 1 <= 64 ? 4 * k + 1 : 4 * k;
  const int mp = (m + 1) & ~1;
  std::vector<unsigned char> bytes((size_t)mp * 256, 0);
  for (int t = 0; t < m; ++t) {
    const u32 q = primes[tgt[t]];
    for (int K = 0; K < krows; ++K) {
      u32 v;
      if (K == 4 * k) v = negS[t];
      else v = (u32)(((u64)w[(size_t)t * k + K / 4] << (8 * (K % 4))) % q);
      for (int bb = 0; bb < 4; ++bb)
        bytes[(size_t)(t / 2) * 512 + (K / 16) * 128 + ((t % 2) * 4 + bb) * 16 + K % 16] = (v >> (8 * bb)) & 255;
    }
  }
  while (b.w.size() % 4) b.w.push_back(0);        // 16-byte aligned
  const size_t off = b.w.size();
  std::vector<u32> words(bytes.size() / 4);
  memcpy(words.data(), bytes.data(), bytes.size());
  b.push(words);
  return off;
}

// Exact base-conversion table (layout lf_bconv_view).  `mult[i]` is folded into c_i.
TabRec build_table(Blob& b, const std::vector<u32>& primes, const std::vector<int>& src,
                   const std::vector<int>& tgt, const std::vector<u32>& mult) {
  const int k = (int)src.size(), m = (int)tgt.size();
  Big S{1};
  for (int i : src) big_mul(S, primes[i]);
  while (S.size() > 1 && S.back() == 0) S.pop_back();
  const int W = (int)S.size() + 1;
  TabRec r{b.align2(), k, m, W, 0, 0};
  std::vector<u32> v;
  for (int i = 0; i < k; ++i) {
    double inv = 1.0 / (double)primes[src[i]];
    u32 two[2];
    memcpy(two, &inv, 8);
    v.push_back(two[0]);
    v.push_back(two[1]);
  }
  for (int i = 0; i < k; ++i) v.push_back((u32)src[i]);
  std::vector<u32> c(k), negS(m), wts((size_t)m * k);
  for (int i = 0; i < k; ++i) {
    const u32 s = primes[src[i]];
    u32 hat = 1;                                   // (S/s_i) mod s_i
    for (int j = 0; j < k; ++j)
      if (j != i) hat = mulm(hat, primes[src[j]] % s, s);
    c[i] = mulm(invm(hat, s), mult[i] % s, s);
  }
  for (int i = 0; i < k; ++i) v.push_back(c[i]);
  for (int i = 0; i < k; ++i) v.push_back(shoupc(c[i], primes[src[i]]));
  for (int t = 0; t < m; ++t) v.push_back((u32)tgt[t]);
  for (int t = 0; t < m; ++t) {
    const u32 q = primes[tgt[t]];
    u32 sm = 1;
    for (int i = 0; i < k; ++i) sm = mulm(sm, primes[src[i]] % q, q);
    negS[t] = (q - sm) % q;
    v.push_back(negS[t]);
  }
  for (int t = 0; t < m; ++t) {
    const u32 q = primes[tgt[t]];
    for (int i = 0; i < k; ++i) {
      u32 h = 1;
      for (int j = 0; j < k; ++j)
        if (j != i) h = mulm(h, primes[src[j]] % q, q);
      wts[(size_t)t * k + i] = h;
      v.push_back(h);
    }
  }
  for (int i = 0; i < k; ++i) {
    Big h{1};
    for (int j = 0; j < k; ++j)
      if (j != i) big_mul(h, primes[src[j]]);
    h.resize(W, 0);
    v.insert(v.end(), h.begin(), h.end());
  }
  Big Sw = S;
  Sw.resize(W, 0);
  v.insert(v.end(), Sw.begin(), Sw.end());
  b.push(v);
  if (4 * k <= 64) r.w8off = build_w8(b, primes, tgt, k, wts, negS, r.kb);
  return r;
}

}  // namespace

int lf_build_ks_plan(LfCtx* ctx, int n_main, int d) {
  const int n_sp = ctx->nprimes - n_main;
  if (n_main < 2 || n_main > LF_MAXMAIN || n_sp < 1 || d < 1 || d > LF_MAXD) {
    lf_set_error("keyswitch plan: n_main=%d n_special=%d d=%d outside limits", n_main, n_sp, d);
    return 2;
  }
  if (n_sp > 64) { lf_set_error("keyswitch plan: too many special primes"); return 2; }
  const int L = n_main - 1;
  std::vector<u32> primes(ctx->nprimes), ninv(ctx->nprimes);
  for (int i = 0; i < ctx->nprimes; ++i) {
    primes[i] = ctx->h_pk[i].q;
    ninv[i] = ctx->h_pk[i].ninv;
  }
  Blob blob;
  // identity row list
  std::vector<u32> iota(n_main > n_sp + 2 ? n_main : n_sp + 2);
  for (size_t i = 0; i < iota.size(); ++i) iota[i] = (u32)i;
  const size_t off_iota = blob.push(iota);

  // decomposition scalars s_i for the own digit of limb i: (Q_L/Q_Dj mod q_i)^-1, j = i % d
  // (ckks.py:85-92, keys.py:85-92), and P^-1 mod q_i (poly.py:280)
  auto dec_scalar = [&](int j, int i) {
    const u32 q = primes[i];
    u32 f = 1;
    for (int t = 0; t <= L; ++t)
      if (t % d != j) f = mulm(f, primes[t] % q, q);
    return invm(f, q);
  };
  std::vector<u32> rowk, pmodv;
  for (int t = 0; t <= L; ++t) {
    const u32 q = primes[t];
    const u32 s = dec_scalar(t % d, t);
    u32 P = 1;
    for (int j = 0; j < n_sp; ++j) P = mulm(P, primes[n_main + j] % q, q);
    const u32 pinv = invm(P, q);
    rowk.insert(rowk.end(), {s, shoupc(s, q), pinv, shoupc(pinv, q)});
    pmodv.insert(pmodv.end(), {P, shoupc(P, q)});
  }
  const size_t off_rowk = blob.push(rowk);
  const size_t off_pmod = blob.push(pmodv);
  std::vector<u32> qinv((size_t)n_main * n_main * 2, 0);
  for (int l = 1; l <= L; ++l)
    for (int t = 0; t < l; ++t) {
      const u32 q = primes[t], v = invm(primes[l] % q, q);
      qinv[((size_t)l * n_main + t) * 2] = v;
      qinv[((size_t)l * n_main + t) * 2 + 1] = shoupc(v, q);
    }
  const size_t off_qinv = blob.push(qinv);
  // (q_l q_{l-1})^-1 mod q_t for the fused double rescale (two successive rescales,
  // ckks.py:220-225, equal one floor division by q_l q_{l-1})
  std::vector<u32> qinv2((size_t)n_main * n_main * 2, 0);
  for (int l = 2; l <= L; ++l)
    for (int t = 0; t < l - 1; ++t) {
      const u32 q = primes[t], v = invm(mulm(primes[l] % q, primes[l - 1] % q, q), q);
      qinv2[((size_t)l * n_main + t) * 2] = v;
      qinv2[((size_t)l * n_main + t) * 2 + 1] = shoupc(v, q);
    }
  const size_t off_qinv2 = blob.push(qinv2);
  // (P q_l)^-1 and (P q_l q_{l-1})^-1 mod q_t: relinearisation fused with one / two rescales
  // (mod_down then rescale, poly.py:251-287, as one floor division by P q_l [q_{l-1}])
  size_t off_pqinv[2];
  for (int nd = 1; nd <= 2; ++nd) {
    std::vector<u32> tab((size_t)n_main * n_main * 2, 0);
    for (int l = nd; l <= L; ++l)
      for (int t = 0; t <= l - nd; ++t) {
        const u32 q = primes[t];
        u32 f = 1;
        for (int j = 0; j < n_sp; ++j) f = mulm(f, primes[n_main + j] % q, q);
        for (int u = l - nd + 1; u <= l; ++u) f = mulm(f, primes[u] % q, q);
        const u32 v = invm(f, q);
        tab[((size_t)l * n_main + t) * 2] = v;
        tab[((size_t)l * n_main + t) * 2 + 1] = shoupc(v, q);
      }
    off_pqinv[nd - 1] = blob.push(tab);
  }

  // ModDown table: specials -> main 0..L, y-multiplier folds the INTT's N^-1.
  std::vector<int> sp_src, main_all;
  std::vector<u32> sp_mult;
  for (int j = 0; j < n_sp; ++j) { sp_src.push_back(n_main + j); sp_mult.push_back(ninv[n_main + j]); }
  for (int t = 0; t <= L; ++t) main_all.push_back(t);
  const TabRec down = build_table(blob, primes, sp_src, main_all, sp_mult);

  // per level
  struct LvRec {
    int beta, ext;
    TabRec up[LF_MAXD];
    size_t src_off[LF_MAXD], dst_off[LF_MAXD];
    TabRec resc, resc2, dr[2];
  };
  std::vector<LvRec> lvr(L + 1);
  for (int l = 0; l <= L; ++l) {
    LvRec& R = lvr[l];
    const int ext = l + 1 + n_sp;
    R.ext = ext;
    R.beta = d < l + 1 ? d : l + 1;
    for (int j = 0; j < R.beta; ++j) {
      std::vector<int> src, tgt;
      std::vector<u32> mult, srows, drows;
      for (int i = j; i <= l; i += d) {
        src.push_back(i);
        mult.push_back(mulm(ninv[i], dec_scalar(j, i), primes[i]));
        srows.push_back((u32)i);
      }
      for (int pos = 0; pos < ext; ++pos) {
        const int pi = pos <= l ? pos : n_main + (pos - l - 1);
        if (pos <= l && pos % d == j) continue;
        tgt.push_back(pi);
        drows.push_back((u32)pos);
      }
      R.up[j] = build_table(blob, primes, src, tgt, mult);
      R.src_off[j] = blob.push(srows);
      R.dst_off[j] = blob.push(drows);
    }
    if (l >= 1) {
      std::vector<int> src{l}, tgt;
      for (int t = 0; t < l; ++t) tgt.push_back(t);
      R.resc = build_table(blob, primes, src, tgt, {ninv[l]});
    }
    if (l >= 2) {
      std::vector<int> src{l - 1, l}, tgt;
      for (int t = 0; t < l - 1; ++t) tgt.push_back(t);
      R.resc2 = build_table(blob, primes, src, tgt, {ninv[l - 1], ninv[l]});
    }
    for (int nd = 1; nd <= 2 && nd <= l; ++nd) {     // sources in T2 order: specials, then mains
      std::vector<int> src(sp_src), tgt;
      std::vector<u32> mult(sp_mult);
      for (int u = l - nd + 1; u <= l; ++u) { src.push_back(u); mult.push_back(ninv[u]); }
      for (int t = 0; t <= l - nd; ++t) tgt.push_back(t);
      R.dr[nd - 1] = build_table(blob, primes, src, tgt, mult);
    }
  }

  void* dmem = nullptr;
  if (cudaMalloc(&dmem, blob.w.size() * 4) != cudaSuccess ||
      cudaMemcpy(dmem, blob.w.data(), blob.w.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
    lf_set_error("keyswitch plan: device allocation failed");
    return 3;
  }
  const u32* base = (const u32*)dmem;
  auto view = [&](const TabRec& r) {
    BconvDev v = lf_bconv_view(base + r.off, r.k, r.m, r.W);
    if (r.w8off) { v.w8 = (const unsigned char*)(base + r.w8off); v.kb = r.kb; }
    return v;
  };

  LfKsPlan* P = new LfKsPlan();
  P->n_main = n_main;
  P->n_special = n_sp;
  P->d = d;
  P->L = L;
  P->dmem = dmem;
  P->iota = (const int*)(base + off_iota);
  P->rowk = base + off_rowk;
  P->pmod = base + off_pmod;
  P->qinv = base + off_qinv;
  P->qinv2 = base + off_qinv2;
  P->pqinv[0] = base + off_pqinv[0];
  P->pqinv[1] = base + off_pqinv[1];
  P->down = view(down);
  P->lv.resize(L + 1);
  for (int l = 0; l <= L; ++l) {
    KsLevelPlan& K = P->lv[l];
    const LvRec& R = lvr[l];
    K.level = l;
    K.beta = R.beta;
    K.ext = R.ext;
    for (int j = 0; j < R.beta; ++j) {
      K.up[j].B = view(R.up[j]);
      K.up[j].src_rows = (const int*)(base + R.src_off[j]);
      K.up[j].dst_rows = (const int*)(base + R.dst_off[j]);
      K.up[j].src_row0 = 0;
      K.up[j].dst_row0 = j * R.ext;
    }
    if (l >= 1) {
      for (int p = 0; p < 2; ++p) {
        K.resc[p].B = view(R.resc);
        K.resc[p].src_rows = P->iota;
        K.resc[p].dst_rows = P->iota;
        K.resc[p].src_row0 = p;
        K.resc[p].dst_row0 = p * l;
      }
    }
    for (int nd = 1; nd <= 2 && nd <= l; ++nd)
      for (int p = 0; p < 2; ++p) {
        K.dr[nd - 1][p].B = view(R.dr[nd - 1]);
        K.dr[nd - 1][p].src_rows = P->iota;
        K.dr[nd - 1][p].dst_rows = P->iota;
        K.dr[nd - 1][p].src_row0 = p * (n_sp + nd);
        K.dr[nd - 1][p].dst_row0 = p * (l + 1 - nd);
      }
    if (l >= 2) {
      for (int p = 0; p < 2; ++p) {
        K.resc2[p].B = view(R.resc2);
        K.resc2[p].src_rows = P->iota;
        K.resc2[p].dst_rows = P->iota;
        K.resc2[p].src_row0 = 2 * p;
        K.resc2[p].dst_row0 = p * (l - 1);
      }
    }
  }
  if (ctx->ks) lf_free_ks_plan(ctx->ks);
  ctx->ks = P;
  return 0;
}

int lf_build_shard_plan(const LfCtx* ctx, int k, int rank, LfShardPlan** out) {
  const LfKsPlan* K = ctx->ks;
  if (!K) { lf_set_error("shard plan: keyswitch plans not built"); return 2; }
  if (k < 1 || k > 64 || rank < 0 || rank >= k) { lf_set_error("shard plan: rank %d of %d", rank, k); return 2; }
  const int n_main = K->n_main, n_sp = K->n_special, d = K->d, L = K->L;
  std::vector<u32> primes(ctx->nprimes), ninv(ctx->nprimes);
  for (int i = 0; i < ctx->nprimes; ++i) { primes[i] = ctx->h_pk[i].q; ninv[i] = ctx->h_pk[i].ninv; }
  auto dec_scalar = [&](int j, int i) {
    const u32 q = primes[i];
    u32 f = 1;
    for (int t = 0; t <= L; ++t)
      if (t % d != j) f = mulm(f, primes[t] % q, q);
    return invm(f, q);
  };
  std::vector<int> sp_loc;
  for (int j = rank; j < n_sp; j += k) sp_loc.push_back(j);
  const int s_slots = (n_sp + k - 1) / k;
  int n_main_L = 0;
  for (int i = rank; i <= L; i += k) ++n_main_L;
  Blob blob;
  blob.w.push_back(0);                      // offset 0 means "none" for the w8 tables
  struct LvRec {
    int n_main, ext, beta, m_slots;
    size_t tmap, kmap;
    TabRec up[LF_MAXD];
    size_t src_off[LF_MAXD], dst_off[LF_MAXD];
    int up_m[LF_MAXD];
  };
  std::vector<LvRec> lvr(L + 1);
  for (int l = 0; l <= L; ++l) {
    LvRec& R = lvr[l];
    std::vector<int> pos, krow;               // local rows: main (ascending), then special
    for (int i = rank; i <= l; i += k) { pos.push_back(i); krow.push_back(i / k); }
    R.n_main = (int)pos.size();
    for (int j : sp_loc) { pos.push_back(l + 1 + j); krow.push_back(n_main_L + j / k); }
    R.ext = (int)pos.size();
    R.beta = d < l + 1 ? d : l + 1;
    R.m_slots = (l + 1 + k - 1) / k;
    R.tmap = blob.push(std::vector<u32>(pos.begin(), pos.end()));
    R.kmap = blob.push(std::vector<u32>(krow.begin(), krow.end()));
    for (int j = 0; j < R.beta; ++j) {
      std::vector<int> src, tgt;
      std::vector<u32> mult, srows, drows;
      for (int i = j; i <= l; i += d) {
        src.push_back(i);
        mult.push_back(mulm(ninv[i], dec_scalar(j, i), primes[i]));
        srows.push_back(((u32)(i % k) << 16) | (u32)(i / k));
      }
      for (int r = 0; r < R.ext; ++r) {
        const int t = pos[r];
        if (t <= l && t % d == j) continue;
        tgt.push_back(t <= l ? t : n_main + (t - l - 1));
        drows.push_back((u32)(j * R.ext + r));
      }
      R.up_m[j] = (int)tgt.size();
      if (tgt.empty()) { tgt.push_back(0); drows.push_back(0); }     // idle group: never launched
      R.up[j] = build_table(blob, primes, src, tgt, mult);
      R.src_off[j] = blob.push(srows);
      R.dst_off[j] = blob.push(drows);
    }
  }
  // ModDown: all specials -> local main rows at L (a prefix serves every level)
  std::vector<int> sp_src, main_loc_L;
  std::vector<u32> sp_mult, dsrc[2], iota;
  for (int j = 0; j < n_sp; ++j) {
    sp_src.push_back(n_main + j);
    sp_mult.push_back(ninv[n_main + j]);
    for (int p = 0; p < 2; ++p) dsrc[p].push_back(((u32)(j % k) << 16) | (u32)(p * s_slots + j / k));
  }
  for (int i = rank; i <= L; i += k) main_loc_L.push_back(i);
  if (main_loc_L.empty()) main_loc_L.push_back(0);      // a rank without main rows (k > L+1)
  for (size_t i = 0; i < main_loc_L.size(); ++i) iota.push_back((u32)i);
  const TabRec down = build_table(blob, primes, sp_src, main_loc_L, sp_mult);
  const size_t off_dsrc0 = blob.push(dsrc[0]), off_dsrc1 = blob.push(dsrc[1]), off_iota = blob.push(iota);

  void* dmem = nullptr;
  if (cudaMalloc(&dmem, blob.w.size() * 4) != cudaSuccess ||
      cudaMemcpy(dmem, blob.w.data(), blob.w.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
    lf_set_error("shard plan: device allocation failed");
    return 3;
  }
  const u32* base = (const u32*)dmem;
  auto view = [&](const TabRec& r) {
    BconvDev v = lf_bconv_view(base + r.off, r.k, r.m, r.W);
    if (r.w8off) { v.w8 = (const unsigned char*)(base + r.w8off); v.kb = r.kb; }
    return v;
  };
  LfShardPlan* P = new LfShardPlan();
  P->k = k; P->rank = rank; P->L = L; P->alpha = n_sp; P->d = d;
  P->n_sp = (int)sp_loc.size(); P->s_slots = s_slots; P->n_key_rows = n_main_L + (int)sp_loc.size();
  P->dmem = dmem; P->comm = nullptr;
  P->lv.resize(L + 1);
  for (int l = 0; l <= L; ++l) {
    ShardLevel& S = P->lv[l];
    const LvRec& R = lvr[l];
    S.n_main = R.n_main; S.ext = R.ext; S.beta = R.beta; S.m_slots = R.m_slots;
    S.tmap = (const int*)(base + R.tmap);
    S.kmap = (const int*)(base + R.kmap);
    for (int j = 0; j < R.beta; ++j) {
      S.up_m[j] = R.up_m[j];
      S.up[j].B = view(R.up[j]);
      S.up[j].src_rows = (const int*)(base + R.src_off[j]);
      S.up[j].dst_rows = (const int*)(base + R.dst_off[j]);
      S.up[j].src_row0 = 0;
      S.up[j].dst_row0 = 0;
    }
  }
  for (int p = 0; p < 2; ++p) {
    P->down[p].B = view(down);
    P->down[p].src_rows = (const int*)(base + (p ? off_dsrc1 : off_dsrc0));
    P->down[p].dst_rows = (const int*)(base + off_iota);
    P->down[p].src_row0 = 0;
    P->down[p].dst_row0 = 0;          // set per call: p * n_main(level)
  }
  *out = P;
  return 0;
}

void lf_free_shard_plan(LfShardPlan* p) {
  if (!p) return;
  cudaFree(p->dmem);
  delete p;
}

void lf_free_ks_plan(LfKsPlan* p) {
  if (!p) return;
  cudaFree(p->dmem);
  delete p;
}
