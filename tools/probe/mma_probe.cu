// mma_probe.cu — measured tcgen05.mma issue-to-completion throughput per (M, N, operand source),
// one CTA per SM, a single thread issuing back-to-back kind::f16 MMAs (K = 16) on zeroed SMEM
// operands into TMEM, clock64 around ITERS MMAs + commit + wait.  Prints cycles per MMA and the
// fraction of the dense bf16 peak (8192 flop / clk / SM) it corresponds to.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include tools/probe/mma_probe.cu -o mma_probe -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2505_20600_b200/csrc/tc_common.cuh"
using namespace ig;

constexpr int ITERS = 4096;

__global__ void __launch_bounds__(128, 1) probe(int M, int N, int ts, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  tc::fence_proxy_async_smem();
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc<512>(&tslot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = tc::idesc_bf16(M, N, 0);
    const uint32_t a = tc::smem_u32(smem), b = tc::smem_u32(smem + 32 * 1024);
    // warm-up
    for (int i = 0; i < 64; ++i) {
      if (ts) tc::mma_bf16_ts(tmem, tmem + 256, tc::sdesc_sw128(b, 16, 1024), idesc, 1);
      else tc::mma_bf16_ss(tmem, tc::sdesc_sw128(a, 16, 1024), tc::sdesc_sw128(b, 16, 1024), idesc, 1);
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 0);
    const long long t0 = clock64();
    for (int i = 0; i < ITERS; ++i) {
      if (ts) tc::mma_bf16_ts(tmem, tmem + 256, tc::sdesc_sw128(b + (i & 3) * 32, 16, 1024), idesc, 1);
      else tc::mma_bf16_ss(tmem, tc::sdesc_sw128(a + (i & 3) * 32, 16, 1024), tc::sdesc_sw128(b + (i & 3) * 32, 16, 1024), idesc, 1);
    }
    tc::mma_commit(&bar);
    tc::mbar_wait(&bar, 1);
    const long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc<512>(tmem);
}

__device__ __forceinline__ void mma2_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
      :
      : "r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// cta_group::2: a cluster of two CTAs, M = 256 (128 rows per CTA), B split across the pair
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe2(int N, int ts, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t rank = tc::cluster_ctarank();
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  tc::fence_proxy_async_smem();
  if (threadIdx.x == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
  if (threadIdx.x < 32) tc::tmem_alloc2<512>(&tslot);
  tc::tc_fence_before();
  tc::cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0 && rank == 0) {
    const uint32_t idesc = tc::idesc_bf16(256, N, 0);
    const uint32_t a = tc::smem_u32(smem), b = tc::smem_u32(smem + 32 * 1024);
    for (int i = 0; i < 64; ++i) {
      if (ts) mma2_bf16_ts(tmem, tmem + 256, tc::sdesc_sw128(b, 16, 1024), idesc, 1);
      else tc::mma2_bf16_ss(tmem, tc::sdesc_sw128(a, 16, 1024), tc::sdesc_sw128(b, 16, 1024), idesc, 1);
    }
    tc::mma2_commit_mc(&bar, 0x3);
    tc::mbar_wait(&bar, 0);
    const long long t0 = clock64();
    for (int i = 0; i < ITERS; ++i) {
      if (ts) mma2_bf16_ts(tmem, tmem + 256, tc::sdesc_sw128(b + (i & 3) * 32, 16, 1024), idesc, 1);
      else tc::mma2_bf16_ss(tmem, tc::sdesc_sw128(a + (i & 3) * 32, 16, 1024), tc::sdesc_sw128(b + (i & 3) * 32, 16, 1024), idesc, 1);
    }
    tc::mma2_commit_mc(&bar, 0x3);
    tc::mbar_wait(&bar, 1);
    out[blockIdx.x / 2] = clock64() - t0;
  } else if (threadIdx.x == 0) {
    tc::mbar_wait(&bar, 0);
    tc::mbar_wait(&bar, 1);
  }
  tc::tc_fence_before();
  tc::cluster_sync();
  if (threadIdx.x < 32) tc::tmem_dealloc2<512>(tmem);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d;
  cudaMalloc(&d, sms * sizeof(long long));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  struct Cfg { int M, N, ts; } cfgs[] = {{128, 256, 0}, {128, 128, 0}, {128, 64, 0}, {128, 32, 0}, {64, 256, 0},
                                          {64, 128, 0}, {128, 256, 1}, {128, 128, 1}, {128, 64, 1}};
  printf("{\"probe\": \"tcgen05.mma kind::f16 K=16, one thread per SM issuing %d back-to-back MMAs, %d SMs\", \"rows\": [\n", ITERS, sms);
  bool first = true;
  for (auto c : cfgs) {
    for (int grid : {1, sms}) {
      probe<<<grid, 128, 100 * 1024>>>(c.M, c.N, c.ts, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      long long h[1024];
      cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
      const double cyc = (double)mx / ITERS;
      const double ideal = (double)c.M * c.N * 16 * 2 / 8192.0;
      printf("%s  {\"M\": %d, \"N\": %d, \"A\": \"%s\", \"ctas\": %d, \"cycles_per_mma\": %.1f, \"ideal_cycles\": %.1f, \"frac_of_peak\": %.3f}",
             first ? "" : ",\n", c.M, c.N, c.ts ? "tmem" : "smem", grid, cyc, ideal, ideal / cyc);
      first = false;
    }
  }
  cudaFuncSetAttribute(probe2, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  struct Cfg2 { int N, ts; } cfgs2[] = {{256, 0}, {128, 0}, {64, 0}, {256, 1}, {128, 1}, {64, 1}};
  for (auto c : cfgs2) {
    for (int grid : {2, 2 * (sms / 2)}) {
      probe2<<<grid, 128, 100 * 1024>>>(c.N, c.ts, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      long long h[1024];
      cudaMemcpy(h, d, grid / 2 * sizeof(long long), cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int i = 0; i < grid / 2; ++i) mx = h[i] > mx ? h[i] : mx;
      const double cyc = (double)mx / ITERS;
      const double ideal = 128.0 * c.N * 16 * 2 / 8192.0;  // per SM: its 128 rows
      printf(",\n  {\"M\": 256, \"cta_group\": 2, \"N\": %d, \"A\": \"%s\", \"ctas\": %d, \"cycles_per_mma\": %.1f, \"ideal_cycles\": %.1f, \"frac_of_peak\": %.3f}",
             c.N, c.ts ? "tmem" : "smem", grid, cyc, ideal, ideal / cyc);
    }
  }
  printf("\n]}\n");
  return 0;
}
