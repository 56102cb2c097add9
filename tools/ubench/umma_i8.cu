// Correctness probe for the tcgen05 kind::i8 operand layout used by k_bconv_tc:
// A = 128 rows x 48 bytes (3 K-chunks per 8-row group, SBO = 384, the 4th chunk of a K-step
// aliases the next group and meets zero B bytes), B = 32 rows x 64 bytes (4th chunk zero),
// D[m][n] = sum_k A[m][k] * B[n][k] in TMEM, read back with tcgen05.ld 32x32b.
// nvcc -gencode arch=compute_100a,code=sm_100a -I paper_2512_11269_b200/csrc tools/ubench/umma_i8.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include "lf_umma.cuh"

__global__ void k_probe(const uint8_t* A, const uint8_t* B, int* D) {
  __shared__ __align__(1024) uint8_t sa[16 * 384 + 128];
  __shared__ __align__(1024) uint8_t sb[4 * 512];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, w = t / 32;
  // A row t: chunk c (16 bytes) at (t/8)*384 + c*128 + (t%8)*16
  for (int c = 0; c < 3; ++c)
    for (int j = 0; j < 16; ++j) sa[(t / 8) * 384 + c * 128 + (t % 8) * 16 + j] = A[t * 48 + c * 16 + j];
  for (int j = 0; j < 128; ++j) if (t == 0) sa[16 * 384 + j] = 0xAB;   // tail garbage
  if (t < 32)
    for (int c = 0; c < 4; ++c)
      for (int j = 0; j < 16; ++j) sb[(t / 8) * 512 + c * 128 + (t % 8) * 16 + j] = c < 3 ? B[t * 48 + c * 16 + j] : 0;
  if (w == 0) tmem_alloc(&tbase, 32);
  if (t == 0) mbar_init(&bar, 1);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (t == 0) {
    const uint32_t a0 = (uint32_t)__cvta_generic_to_shared(sa), b0 = (uint32_t)__cvta_generic_to_shared(sb);
    const uint32_t id = umma_idesc_u8(128, 32);
    umma_i8(tm, umma_sdesc(a0, 128, 384), umma_sdesc(b0, 128, 512), id, false);
    umma_i8(tm, umma_sdesc(a0 + 256, 128, 384), umma_sdesc(b0 + 256, 128, 512), id, true);
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t v[32];
  for (int c = 0; c < 8; ++c)
    tmem_ld4(tm + ((uint32_t)(32 * (w % 4)) << 16) + 4 * c, v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  tmem_ld_wait();
  for (int n = 0; n < 32; ++n) D[t * 32 + n] = (int)v[n];
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc(tm, 32);
}

int main() {
  uint8_t hA[128 * 48], hB[32 * 48];
  srand(1);
  for (auto& x : hA) x = rand() & 255;
  for (auto& x : hB) x = rand() & 255;
  uint8_t *dA, *dB;
  int* dD;
  cudaMalloc(&dA, sizeof hA);
  cudaMalloc(&dB, sizeof hB);
  cudaMalloc(&dD, 128 * 32 * 4);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  k_probe<<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("FAIL launch: %s\n", cudaGetErrorString(e)); return 1; }
  static int hD[128 * 32];
  cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 32; ++n) {
      int s = 0;
      for (int k = 0; k < 48; ++k) s += hA[m * 48 + k] * hB[n * 48 + k];
      if (s != hD[m * 32 + n] && bad++ < 8) printf("m=%d n=%d got %d want %d\n", m, n, hD[m * 32 + n], s);
    }
  printf(bad ? "FAIL %d mismatches\n" : "PASS umma i8 layout\n", bad);
  return bad != 0;
}
