// Kernel-plan interpreter: the B200 side of the reference's KernelRunner boundary
// (codegen.py:346-443; plans from plan_kernels, codegen.py:445+).  A plan's lanes are
// independent per-prime op chains over limb rows; op i of every lane writes register i
// (codegen.py:160-172), so the host runs a plan as a sequence of STEPS: step i executes op i of
// all lanes in ONE launch (grid.y = lane op, grid.x = coefficient blocks).  Registers are rows
// of a device scratch laid out [step][lane][N], which makes the rows an NTT/INTT step writes
// contiguous, so those go through the batched lf_ntt path (the host stages them with COPY).
// Every op writes canonical residues; stored rows therefore equal the reference's lazily
// reduced ones (it only defers reductions that cannot change a value mod q).
#include "lf_ntt.cuh"
#include "lf_bconv.cuh"
#include "lf_ops.h"

struct LfPlanOpDev {        // mirrors lf_plan_op in lf_b200.h
  int32_t opcode, pidx;
  uint32_t scalar, galois;
  int32_t nsrc, k, W, pad;
  const u32* const* src;    // nsrc row pointers (device array)
  u32* dst;
  u32* store;
  const u32* table;         // BConv: k sources -> 1 target blob
};
static_assert(sizeof(LfPlanOpDev) == sizeof(lf_plan_op), "lf_plan_op layout");

__global__ void __launch_bounds__(256) k_plan_step(const LfPlanOpDev* ops, LfDev dv) {
  lf_pdl_trigger();
  lf_pdl_wait();
  const LfPlanOpDev o = ops[blockIdx.y];
  const size_t N = (size_t)1 << dv.logN;
  const size_t n = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (n >= N) return;
  const PrimeK pk = dv.pk[o.pidx];
  const u32 q = pk.q;
  u32 v = 0;
  switch (o.opcode) {
    case LF_POP_ADD: v = addmod(o.src[0][n], o.src[1][n], q); break;
    case LF_POP_SUB: v = submod(o.src[0][n], o.src[1][n], q); break;
    case LF_POP_MUL: v = mulmod(o.src[0][n], o.src[1][n], pk); break;
    case LF_POP_MULACC: v = reduce64((u64)o.src[1][n] * o.src[2][n] + o.src[0][n], pk); break;
    case LF_POP_NEG: { const u32 a = o.src[0][n]; v = a ? q - a : 0u; break; }
    case LF_POP_SCALARMUL: v = mulmod(o.src[0][n], o.scalar, pk); break;
    case LF_POP_MODSTEP: v = mulmod(submod(o.src[0][n], o.src[1][n], q), o.scalar, pk); break;
    case LF_POP_AUTOMORPH: v = o.src[0][auto_src_index((u32)n, o.galois, dv.logN)]; break;
    case LF_POP_COPY: v = o.src[0][n]; break;
    case LF_POP_BCONV: {
      const BconvDev B = lf_bconv_view(o.table, o.k, 1, o.W);
      u32 y[64];
      for (int i = 0; i < B.k; ++i) {
        const PrimeK ks = dv.pk[B.src_pi[i]];
        y[i] = mul_shoup(o.src[i][n] % ks.q, B.c[i], B.cp[i], ks.q);
      }
      const u32 u = bconv_u(y, B);
      u64 acc = (u64)u * B.negS[0];
      for (int i = 0; i < B.k; ++i) acc += (u64)y[i] * B.w[i];
      v = reduce64(acc, pk);
      break;
    }
    default: return;
  }
  if (o.dst) o.dst[n] = v;
  if (o.store) o.store[n] = v;
}

int lf_launch_plan_step(const LfCtx* ctx, const void* ops, int nops, cudaStream_t s) {
  if (nops < 1) return 0;
  if (nops > 65535) { lf_set_error("lf_plan_step: %d ops in one step (max 65535)", nops); return 2; }
  const unsigned bx = (unsigned)((ctx->N + 255) / 256);
  cudaError_t e = lf_launch(k_plan_step, dim3(bx, (unsigned)nops), dim3(256), 0, s, 1,
                            (const LfPlanOpDev*)ops, ctx->dev());
  if (e != cudaSuccess) { lf_set_error("lf_plan_step: launch: %s", cudaGetErrorString(e)); return 3; }
  LF_CHECK_LAUNCH();
  return 0;
}
