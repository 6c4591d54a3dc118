// k_gemm_simt.cu — CUDA-core GEMM C = A B^T (+ fused epilogues) for the fp32 PARITY mode
// (SURVEY §8(c) C-TOL: TF32 tensor cores cannot meet rtol 1e-4, so fp32 uses true FFMA).
// A [M,K] row-major, B [N,K] row-major (weights [out, in]).  64x64x16 tiles, 256 threads,
// 4x4 outputs per thread, fixed K order (batch-invariant: no split-K).
#include "kernels.h"

namespace ig {

template <typename T>
__device__ __forceinline__ void gemm_epilogue_store(const GemmArgs& g, int r, int c, float acc) {
  const T* bias = reinterpret_cast<const T*>(g.bias);
  float y = acc + (bias ? to_f<T>(bias[c]) : 0.f);
  switch (g.epi) {
    case EPI_STORE:
    case EPI_GELU: {
      if (g.epi == EPI_GELU) y = gelu_tanh(y);
      if (g.out_f32) reinterpret_cast<float*>(g.C)[(long long)r * g.ldc + c] = y;
      else reinterpret_cast<T*>(g.C)[(long long)r * g.ldc + c] = from_f<T>(y);
      break;
    }
    case EPI_GATED_RES: {
      const RowInfo info = g.ri[g.ri_off + r];
      float* X = reinterpret_cast<float*>(g.C) + (long long)r * g.ldc + c;
      *X = *X + g.gate[(long long)info.req * g.gate_ld + c] * y;
      break;
    }
    case EPI_POS: {
      const RowInfo info = g.ri[g.ri_off + r];
      if (g.pos) y += to_f<T>(reinterpret_cast<const T*>(g.pos)[(long long)info.tok * g.pos_ld + c]);
      reinterpret_cast<float*>(g.C)[(long long)r * g.ldc + c] = y;
      break;
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) gemm_simt_kernel(GemmArgs g) {
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const T* A = reinterpret_cast<const T*>(g.A);
  const T* B = reinterpret_cast<const T*>(g.B);
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < g.K; k0 += BK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = tid + i * 256;        // 0..1023
      const int row = e / BK, kk = e % BK;
      const int ga = m0 + row, gb = n0 + row, gk = k0 + kk;
      As[kk][row] = (ga < g.M && gk < g.K) ? to_f<T>(A[(long long)ga * g.lda + gk]) : 0.f;
      Bs[kk][row] = (gb < g.N && gk < g.K) ? to_f<T>(B[(long long)gb * g.ldb + gk]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = As[kk][ty * 4 + i]; b[i] = Bs[kk][tx * 4 + i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = m0 + ty * 4 + i;
    if (r >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = n0 + tx * 4 + j;
      if (c < g.N) gemm_epilogue_store<T>(g, r, c, acc[i][j]);
    }
  }
}

template <typename T>
void launch_gemm_simt(const GemmArgs& g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0) return;
  dim3 grid((g.N + 63) / 64, (g.M + 63) / 64);
  gemm_simt_kernel<T><<<grid, 256, 0, st>>>(g);
}
template void launch_gemm_simt<float>(const GemmArgs&, cudaStream_t);
template void launch_gemm_simt<bf16>(const GemmArgs&, cudaStream_t);

}  // namespace ig
