// Throughput of the integer multiply-accumulate formulations used by the BConv MAC on sm_100a.
// Each thread runs R independent accumulator chains for ITER iterations; time with events.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef uint32_t u32; typedef uint64_t u64;
#define ITER 4096
#define R 8

__global__ void k_wide(u64* out, u32 a0, u32 b0) {
  u64 acc[R]; u32 a[R];
  for (int r = 0; r < R; ++r) { acc[r] = r; a[r] = a0 + threadIdx.x + r; }
  u32 b = b0;
  for (int i = 0; i < ITER; ++i) {
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] += (u64)a[r] * b;
    b += 3;
  }
  u64 s = 0; for (int r = 0; r < R; ++r) s += acc[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_hi(u64* out, u32 a0, u32 b0) {
  u32 acc[R]; u32 a[R];
  for (int r = 0; r < R; ++r) { acc[r] = r; a[r] = a0 + threadIdx.x + r; }
  u32 b = b0;
  for (int i = 0; i < ITER; ++i) {
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] += __umulhi(a[r], b);
    b += 3;
  }
  u64 s = 0; for (int r = 0; r < R; ++r) s += acc[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_lo(u64* out, u32 a0, u32 b0) {
  u32 acc[R]; u32 a[R];
  for (int r = 0; r < R; ++r) { acc[r] = r; a[r] = a0 + threadIdx.x + r; }
  u32 b = b0;
  for (int i = 0; i < ITER; ++i) {
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] += a[r] * b;
    b += 3;
  }
  u64 s = 0; for (int r = 0; r < R; ++r) s += acc[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// Shoup MAC: acc += y*w - umulhi(y, w')*q  (lazy, [0, 2q) per term)
__global__ void k_shoup(u64* out, u32 a0, u32 b0) {
  u32 acc[R]; u32 a[R];
  const u32 q = 268369921u;
  for (int r = 0; r < R; ++r) { acc[r] = r; a[r] = a0 + threadIdx.x + r; }
  u32 w = b0, wp = b0 * 7;
  for (int i = 0; i < ITER; ++i) {
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] += a[r] * w - __umulhi(a[r], wp) * q;
    w += 3; wp += 5;
  }
  u64 s = 0; for (int r = 0; r < R; ++r) s += acc[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dfma(u64* out, u32 a0, u32 b0) {
  double acc[R]; double a[R];
  for (int r = 0; r < R; ++r) { acc[r] = r; a[r] = (double)(a0 + threadIdx.x + r); }
  double b = b0;
  for (int i = 0; i < ITER; ++i) {
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = fma(a[r], b, acc[r]);
    b += 3.0;
  }
  double s = 0; for (int r = 0; r < R; ++r) s += acc[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (u64)s;
}
// mixed: half the chains IMAD.WIDE, half DFMA (pipe overlap)
__global__ void k_mix(u64* out, u32 a0, u32 b0) {
  u64 acc[R / 2]; u32 a[R / 2]; double dacc[R / 2]; double da[R / 2];
  for (int r = 0; r < R / 2; ++r) { acc[r] = r; a[r] = a0 + threadIdx.x + r; dacc[r] = r; da[r] = a[r]; }
  u32 b = b0; double db = b0;
  for (int i = 0; i < ITER; ++i) {
#pragma unroll
    for (int r = 0; r < R / 2; ++r) { acc[r] += (u64)a[r] * b; dacc[r] = fma(da[r], db, dacc[r]); }
    b += 3; db += 3.0;
  }
  u64 s = 0; for (int r = 0; r < R / 2; ++r) s += acc[r] + (u64)dacc[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class K>
void run(const char* name, K k, u64* d, double ops_per_thread_iter) {
  dim3 grid(148 * 8), block(256);
  k<<<grid, block>>>(d, 12345, 678);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) k<<<grid, block>>>(d, 12345 + i, 678);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = 5.0 * grid.x * block.x * ITER * ops_per_thread_iter;
  printf("%-8s %8.3f ms  %8.1f Gop/s  %6.1f op/clk/SM (at 1965 MHz)\n", name, ms, ops / ms / 1e6,
         ops / (ms * 1e-3) / 148 / 1.965e9);
}

int main() {
  u64* d; cudaMalloc(&d, 148 * 8 * 256 * 8);
  run("wide", k_wide, d, R);
  run("hi", k_hi, d, R);
  run("lo", k_lo, d, R);
  run("shoup", k_shoup, d, R);
  run("dfma", k_dfma, d, R);
  run("mix", k_mix, d, R);
  return 0;
}
