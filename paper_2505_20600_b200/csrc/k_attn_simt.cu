// k_attn_simt.cu — CUDA-core varlen attention for the fp32 PARITY mode (C-TOL 1e-4).
// O = softmax(Q K^T / sqrt(d)) V per (segment, head): each ragged query
// segment of the packed batch attends to its request's full merged K/V buffer (L rows).
// CTA = 8 warps = 8 query rows of one (segment, head); K/V tiles of 32 keys staged in
// shared memory and shared by the 8 warps; online softmax with a per-row running max
// (rescale decisions per row: batch-invariant, SURVEY §8(c) bitwise requirement 3).
#include <math.h>
#include "kernels.h"

namespace ig {

constexpr int AS_ROWS = 8, AS_KT = 32, AS_MAXD = 128;

template <typename T>
__global__ void __launch_bounds__(AS_ROWS * 32) attn_simt_kernel(AttnArgs a) {
  __shared__ float Ks[AS_KT][AS_MAXD + 1];
  __shared__ float Vs[AS_KT][AS_MAXD + 1];
  __shared__ float qs[AS_ROWS][AS_MAXD];
  const AttnSeg seg = a.segs[blockIdx.z];
  const int h = blockIdx.y;
  const int d = a.head_dim;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qi = blockIdx.x * AS_ROWS + warp;  // row inside the segment
  if (blockIdx.x * AS_ROWS >= seg.q_len) return;  // whole CTA idle (uniform)
  const bool active = qi < seg.q_len;
  const long long H = (long long)a.heads * d;
  const T* Q = reinterpret_cast<const T*>(a.Q);
  const T* Kb = reinterpret_cast<const T*>(a.kv_arena) + seg.kv_base + a.kv_off;
  const T* Vb = Kb + (long long)a.L * H;
  if (active)
    for (int t = lane; t < d; t += 32)
      qs[warp][t] = to_f<T>(Q[(long long)(seg.q_start + qi) * a.ldq + h * d + t]);
  float m = -INFINITY, l = 0.f;
  float o[AS_MAXD / 32] = {};
  for (int k0 = 0; k0 < a.L; k0 += AS_KT) {
    __syncthreads();
    for (int i = threadIdx.x; i < AS_KT * d; i += blockDim.x) {
      const int j = i / d, t = i % d;
      const int key = k0 + j;
      float kv = 0.f, vv = 0.f;
      if (key < a.L) {
        kv = to_f<T>(Kb[(long long)key * H + h * d + t]);
        vv = to_f<T>(Vb[(long long)key * H + h * d + t]);
      }
      Ks[j][t] = kv;
      Vs[j][t] = vv;
    }
    __syncthreads();
    if (!active) continue;
    float s = 0.f;
    for (int t = 0; t < d; ++t) s = fmaf(qs[warp][t], Ks[lane][t], s);
    s *= a.scale;
    if (k0 + lane >= a.L) s = -INFINITY;
    const float mt = warp_max(s);
    const float m_new = fmaxf(m, mt);
    const float alpha = expf(m - m_new);  // m = -inf on the first tile -> 0
    const float p = expf(s - m_new);
    l = l * alpha + warp_sum(p);
#pragma unroll
    for (int e = 0; e < AS_MAXD / 32; ++e) o[e] *= alpha;
    for (int j = 0; j < AS_KT; ++j) {
      const float pj = __shfl_sync(0xffffffffu, p, j);
#pragma unroll
      for (int e = 0; e < AS_MAXD / 32; ++e) {
        const int t = lane + 32 * e;
        if (t < d) o[e] = fmaf(pj, Vs[j][t], o[e]);
      }
    }
    m = m_new;
  }
  if (!active) return;
  T* O = reinterpret_cast<T*>(a.O) + (long long)(seg.q_start + qi) * a.ldo + h * d;
  const float inv = 1.0f / l;
#pragma unroll
  for (int e = 0; e < AS_MAXD / 32; ++e) {
    const int t = lane + 32 * e;
    if (t < d) O[t] = from_f<T>(o[e] * inv);
  }
}

template <typename T>
void launch_attn_simt(const AttnArgs& a, cudaStream_t st) {
  if (a.nseg <= 0 || a.max_qlen <= 0) return;
  dim3 grid((a.max_qlen + AS_ROWS - 1) / AS_ROWS, a.heads, a.nseg);
  attn_simt_kernel<T><<<grid, AS_ROWS * 32, 0, st>>>(a);
}
template void launch_attn_simt<float>(const AttnArgs&, cudaStream_t);
template void launch_attn_simt<bf16>(const AttnArgs&, cudaStream_t);

}  // namespace ig
