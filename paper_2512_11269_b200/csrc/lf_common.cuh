// Shared host/device declarations of the B200 CKKS core.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "lf_arith.cuh"
#include "lf_line.cuh"

// Device view of one parameter context (all tables resident in HBM).
struct LfDev {
  const PrimeK* pk;      // [nprimes]  per-prime constants
  const uint2* twf;      // [nprimes << logN]  {psi^brv(i), Shoup companion}
  const uint2* twi;      // [nprimes << logN]  {psi^-brv(i), Shoup companion}
  const uint2* twfT;     // twf / twi with the row-pass subtrees of depth >= LineCfg<L2>::LA
  const uint2* twiT;     //   stored transposed per CTA line block (TwTree<LP>, tw_bulk_begin)
  int logN;
  int nprimes;
};

// Prime index of each row of a row batch (rows are N contiguous words each).
#define LF_MAX_ROWS 256
struct RowMap {
  int n;
  unsigned char p[LF_MAX_ROWS];
};

struct LfKsPlan;
struct LfCtx {
  int logN, N, nprimes;
  LfKsPlan* ks;          // keyswitch plans (lf_ctx_enable_keyswitch), or null
  PrimeK* d_pk;
  uint2* d_twf;
  uint2* d_twi;
  uint2* d_twfT;
  uint2* d_twiT;
  PrimeK* h_pk;
  LfDev dev() const { return LfDev{d_pk, d_twf, d_twi, d_twfT, d_twiT, logN, nprimes}; }
};

// error plumbing (lf_api.cu)
void lf_set_error(const char* fmt, ...);
#define LF_CHECK_LAUNCH()                                                  \
  do {                                                                     \
    cudaError_t e__ = cudaGetLastError();                                  \
    if (e__ != cudaSuccess) {                                              \
      lf_set_error("%s:%d: %s", __FILE__, __LINE__, cudaGetErrorString(e__)); \
      return 3;                                                            \
    }                                                                      \
  } while (0)

// split of logN into column-pass (L1) and row-pass (L2) stage counts
inline void lf_split(int logN, int& L1, int& L2) {
  L1 = logN / 2;
  L2 = logN - L1;
}

// Opt a kernel into more than 48 KB of dynamic shared memory.
template <class K>
inline void lf_smem_optin(K kern, size_t bytes) {
  if (bytes > 48 * 1024)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// Programmatic dependent launch (sm_90+).  Every kernel launched through lf_launch() calls
// lf_pdl_trigger() first (the next kernel of the stream may be scheduled as soon as all CTAs of
// this one are resident) and lf_pdl_wait() before its first access to data written by the
// previous kernel, so its independent prologue (twiddle / weight staging) overlaps the
// previous kernel's tail.  Kernels launched the ordinary way simply see full serialisation.
// Measured on B200 (C2 keyswitch batch 1: 211 -> 257 us; bootstrap 18.5 -> 18.9 ms): the early
// CTAs hold shared memory while they wait and slow the previous kernel's tail, so programmatic
// serialisation is OFF by default (LF_PDL=1 turns it on); the wait/trigger instructions are
// no-ops without it.
LF_DEV void lf_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
LF_DEV void lf_pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

#ifndef LF_PDL
#define LF_PDL 0
#endif
template <typename... KArgs, typename... Args>
inline cudaError_t lf_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                             cudaStream_t s, int cluster, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int n = 0;
  if (LF_PDL) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = cluster;
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

// host launchers (lf_ntt.cu)
int lf_launch_ntt(const LfCtx* ctx, u32* rows, const RowMap& rm, bool inverse, cudaStream_t s);
