// Throughput of the register-resident 256-point line transform (lf_line.cuh) with the data
// and twiddles on chip: no global memory in the loop.  Reports butterflies/clk/SM for
//   row   : 16 threads per line, lines = consecutive lanes, warp-synchronous exchange
//   col   : 8-column tile, 16 threads per column (AddrC), named barrier over a 128-thread group
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2512_11269_b200/csrc tools/ubench/ntt_line.cu -o tools/ubench/ntt_line
#include <cstdio>
#include "lf_ntt.cuh"

#define ITER 64

template <bool NAMED>
struct SyncG {
  int id, n;
  LF_DEV void operator()() const {
    if (NAMED) asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
    else __syncwarp();
  }
};

// MODE 0: row lines (warp sync), MODE 1: column tiles (named barrier per 128 threads)
template <int MODE, int NT>
__global__ void __launch_bounds__(NT) k_line(u32* out, const uint2* tw_g, u32 q) {
  using C = LineCfg<8>;
  __shared__ uint2 tws[256];
  extern __shared__ u32 xs[];
  for (int i = threadIdx.x; i < 256; i += NT) tws[i] = tw_g[i];
  __syncthreads();
  u32 x[C::E];
#pragma unroll
  for (int e = 0; e < C::E; ++e) x[e] = (threadIdx.x * 7 + e * 13) % q;
  u32 acc = 0;
  if (MODE == 0) {
    const int tl = threadIdx.x % 16, ln = threadIdx.x / 16;
    const AddrR<8> addr{ln * pitchR<8>()};
    for (int it = 0; it < ITER; ++it) {
      fwd_line<8, 4>(x, 1u, TwFlat{tws}, q, xs, tl, addr, SyncWarp{});
#pragma unroll
      for (int e = 0; e < C::E; ++e) x[e] = csub(csub(x[e], 8 * q), 4 * q) & 0x3FFFFFF;
    }
  } else {
    const int g = threadIdx.x / 128, lt = threadIdx.x % 128, c = lt % 8, tl = lt / 8;
    const AddrC<8, 8> addr{c};
    u32* X = xs + g * smemC_words<8, 8>();
    const SyncG<true> gs{1 + g, 128};
    for (int it = 0; it < ITER; ++it) {
      fwd_line<8, 4>(x, 1u, TwFlat{tws}, q, X, tl, addr, gs);
      gs();
#pragma unroll
      for (int e = 0; e < C::E; ++e) x[e] = csub(csub(x[e], 8 * q), 4 * q) & 0x3FFFFFF;
    }
  }
#pragma unroll
  for (int e = 0; e < C::E; ++e) acc += x[e];
  out[blockIdx.x * NT + threadIdx.x] = acc;
}

template <int MODE, int NT>
void run(const char* name, int ctas_per_sm, u32* out, const uint2* tw, u32 q, size_t smem) {
  int sms = 148;
  auto kern = k_line<MODE, NT>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = sms * ctas_per_sm * 8;
  kern<<<grid, NT, smem>>>(out, tw, q);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<<<grid, NT, smem>>>(out, tw, q);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double bf = (double)grid * NT * ITER * 64;     // 16 elements x 8 stages / 2 per thread
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("%-28s %8.3f ms  %6.2f T bfly/s  %5.2f bfly/clk/SM  (err %s)\n", name, ms, bf / ms / 1e9,
         bf / (ms * 1e-3) / (sms * (double)clk * 1e3), cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const u32 q = 268369921u;
  uint2 h[256];
  for (int i = 0; i < 256; ++i) { h[i].x = (u32)((i * 2654435761u) % q); h[i].y = (u32)(((unsigned long long)h[i].x << 32) / q); }
  uint2* tw; u32* out;
  cudaMalloc(&tw, sizeof(h)); cudaMemcpy(tw, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMalloc(&out, 148 * 64 * 1024 * 4);
  run<0, 256>("row 256thr x 8 CTA/SM", 8, out, tw, q, 16 * pitchR<8>() * 4);
  run<0, 256>("row 256thr x 4 CTA/SM", 4, out, tw, q, 16 * pitchR<8>() * 4);
  run<1, 1024>("col 1024thr x 2 CTA/SM", 2, out, tw, q, 8 * smemC_words<8, 8>() * 4);
  run<1, 512>("col 512thr x 4 CTA/SM", 4, out, tw, q, 4 * smemC_words<8, 8>() * 4);
  return 0;
}
