// tcgen05 (5th-generation tensor core) helpers for sm_100a: TMEM allocation, the u8 x u8 -> s32
// MMA (kind::i8) with operands in shared memory, completion through an mbarrier, and the
// TMEM -> register load of the epilogue.  Used by the byte-split base conversion
// (k_bconv_tc, lf_ks.cu).
//
// Operand layout ("canonical K-major, no swizzle"): an operand of R rows x K bytes is a grid of
// 8-row x 16-byte core matrices, each 128 contiguous bytes (row r of the core matrix at byte
// 16 r).  Core matrices adjacent in K are LBO bytes apart, adjacent 8-row groups SBO bytes apart.
// One kind::i8 MMA consumes K = 32 bytes (two core matrices along K).
#pragma once
#include <cstdint>

#define LF_UMMA_DEV __device__ __forceinline__

// Shared-memory matrix descriptor (version 1, SWIZZLE_NONE, base offset 0).
LF_UMMA_DEV uint64_t umma_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;                       // descriptor version (sm_100)
  return d;                                     // layout type 0 = SWIZZLE_NONE
}

// Instruction descriptor: A, B unsigned 8-bit, both K-major, D signed 32-bit, M x N.
__host__ __device__ constexpr uint32_t umma_idesc_u8(int M, int N) {
  return (2u << 4)                              // D format S32
         | (0u << 7) | (0u << 10)               // A, B: u8
         | ((uint32_t)(N >> 3) << 17)
         | ((uint32_t)(M >> 4) << 24);
}

LF_UMMA_DEV void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, bool accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
      :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"((uint32_t)accum));
}

// Arrive on an mbarrier once every previously issued tcgen05.mma of this thread completed.
LF_UMMA_DEV void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               :: "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}

LF_UMMA_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;"
               :: "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count) : "memory");
}

LF_UMMA_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "LF_MBW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra LF_MBW_%=;\n\t}\n"
      :: "r"(a), "r"(parity) : "memory");
}

// Generic-proxy shared-memory writes -> visible to the tensor core (async proxy).
LF_UMMA_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
LF_UMMA_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
LF_UMMA_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// TMEM allocation (one warp; `cols` a power of two >= 32); the base address lands in *dst.
LF_UMMA_DEV void tmem_alloc(uint32_t* dst, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
               :: "r"((uint32_t)__cvta_generic_to_shared(dst)), "r"(cols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
LF_UMMA_DEV void tmem_dealloc(uint32_t base, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(base), "r"(cols) : "memory");
}

// 4 consecutive 32-bit TMEM columns of this thread's lane (warp w reads lanes 32 (w % 4) ..).
LF_UMMA_DEV void tmem_ld4(uint32_t taddr, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(taddr));
}
LF_UMMA_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
