// common.cuh — shared device/host helpers for libig (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libig is written for sm_100a (B200) only"
#endif

namespace ig {

typedef __nv_bfloat16 bf16;

// Per-row metadata of the packed batch (a2 batch assembly).
// req: index of the request in the ig_edit_step call; slot: its K/V ring slot;
// kvpos: row of this token in the request's merged positional K/V buffer
//        (text t -> t, image token i -> L_txt + i; C-AMB 8);
// tok: image token index i (>= 0) or -1 for a text row (RoPE position source, C-AMB 7).
struct RowInfo {
  int req, slot, kvpos, tok;
};

// Per-segment descriptor for ragged attention: query rows [q_start, q_start + q_len) of the
// packed Q attend to the K/V buffer at kv_base (+ per-launch offset).
struct AttnSeg {
  int q_start, q_len;
  long long kv_base;  // element offset of the slot's ring base in the K/V arena
};

template <typename T> __device__ __forceinline__ float to_f(T x);
template <> __device__ __forceinline__ float to_f<float>(float x) { return x; }
template <> __device__ __forceinline__ float to_f<bf16>(bf16 x) { return __bfloat162float(x); }

template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ bf16 from_f<bf16>(float x) { return __float2bfloat16_rn(x); }

__device__ __forceinline__ float gelu_tanh(float x) {
  // 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3)))  (C-AMB 6)
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  float u = k0 * (x + k1 * x * x * x);
  return 0.5f * x * (1.0f + tanhf(u));
}

__device__ __forceinline__ float silu(float x) { return x / (1.0f + expf(-x)); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace ig
