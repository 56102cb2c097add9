// Keyswitch / rescale plans: every constant the fused kernels need, built once per context on
// the host from the prime list (no big-integer library: products are formed word by word) and
// kept resident in HBM.
#pragma once
#include <vector>

#include "lf_bconv.cuh"

#define LF_MAXD 16        // max digits d
#define LF_MAXMAIN 64     // max main primes L+1

// One base-conversion group of a K_BC launch: source rows src_row0 + src_rows[i] of the
// source buffer, target rows dst_row0 + dst_rows[t] of the destination buffer.
struct BcGroupDev {
  BconvDev B;
  const int* src_rows;
  const int* dst_rows;
  int src_row0, dst_row0;
};

struct KsLevelPlan {
  int level, beta, ext;
  BcGroupDev up[LF_MAXD];      // ModUp conversion of digit j (sources G_j, targets ext \ G_j)
  BcGroupDev resc[2];          // rescale at this level: q_level -> q_0..q_{level-1} (b and a)
  BcGroupDev resc2[2];         // double rescale: {q_{level-1}, q_level} -> q_0..q_{level-2}
  BcGroupDev dr[2][2];         // [nd-1][poly]: ModDown fused with a rescale by nd primes:
                               // {specials, q_{level-nd+1}..q_level} -> q_0..q_{level-nd}
};

struct LfKsPlan {
  int n_main, n_special, d, L;
  std::vector<KsLevelPlan> lv;     // index = level
  BconvDev down;                   // ModDown: specials -> main 0..L (prefix per level)
  const int* iota;                 // device 0..max(n_main, n_special) identity row list
  const u32* rowk;                 // [n_main][4]: s_t, s_t' (own-digit decomposition scalar), P^-1, P^-1'
  const u32* pmod;                 // [n_main][2]: P mod q_t and Shoup companion (extended rotations)
  const u32* qinv;                 // [n_main][n_main][2]: q_l^-1 mod q_t and Shoup companion
  const u32* qinv2;                // [n_main][n_main][2]: (q_l q_{l-1})^-1 mod q_t, companion
  const u32* pqinv[2];             // [n_main][n_main][2]: (P q_l)^-1, (P q_l q_{l-1})^-1 mod q_t
  void* dmem;
};

int lf_build_ks_plan(struct LfCtx* ctx, int n_main, int d);
void lf_free_ks_plan(LfKsPlan* p);

// Limb-sharded keyswitch plan of ONE rank out of k (reference multidev.py:55-56 placement:
// main row i on rank i % k, special j on rank j % k).  Local rows are stored main-first in
// ascending prime order; cross-rank sources come from the all-gathered buffers, whose rows
// are addressed as (rank << 16) | slot (BcArgs::src_rstride).
struct ShardLevel {
  int n_main, ext, beta;         // local main rows at this level, local extended rows, digits
  int m_slots;                   // T0 rows each rank contributes to the ModUp all-gather
  int up_m[LF_MAXD];             // real targets of digit group j on this rank (0: group idle)
  const int* tmap;               // [ext] extended-basis position of local row r
  const int* kmap;               // [ext] row of the rank's local key (main_loc(L) ++ special_loc)
  BcGroupDev up[LF_MAXD];        // digit j: all sources G_j (gathered) -> local ext rows not in G_j
};
struct LfShardPlan {
  int k, rank, L, alpha, d;
  int n_sp, s_slots;             // local special rows; special rows each rank contributes (per poly)
  int n_key_rows;                // rows of the rank's local key: |main_loc(L)| + n_sp
  std::vector<ShardLevel> lv;
  BcGroupDev down[2];            // ModDown of poly p: all alpha specials (gathered) -> local main rows
  void* dmem;
  void* comm;                    // lf_comm* (NCCL) or null (the host performs the gathers)
};
int lf_build_shard_plan(const struct LfCtx* ctx, int k, int rank, LfShardPlan** out);
void lf_free_shard_plan(LfShardPlan* p);
