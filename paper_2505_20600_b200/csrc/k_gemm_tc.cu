// k_gemm_tc.cu — kernel (c): persistent tcgen05/TMEM/TMA tensor-core GEMM, bf16 in, fp32
// accumulate, with the step's fused epilogues (bias, GELU-tanh, gated residual into the fp32
// residual stream, positional-embedding add).  C[M,N] = A[M,K] B[N,K]^T: the masked-row
// projections / MLP of the mask-aware step (P:384-386 token-wise ops on masked rows only;
// Table 1 rows XW and (XW1)W2).
//
// Structure (one CTA per SM, persistent over output tiles, static round-robin schedule):
//   warp 0      TMA producer: A tile [128 x 64] and B tile [BN x 64] per stage, SWIZZLE_128B
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=16)
//   warps 4..7  epilogue: tcgen05.ld (thread = output row) -> epilogue math -> global stores
// Pipelines: smem full/empty mbarriers (TMA <-> MMA), TMEM full/empty (MMA <-> epilogue) with
// a double-buffered accumulator so tile i's epilogue overlaps tile i+1's mainloop.
// Fixed tile shape and K order independent of M: batch-invariant (SURVEY §8(c) bitwise
// requirement 1).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <mutex>
#include <unordered_map>
#include <cstdlib>
#include "kernels.h"
#include "ig_internal.h"
#include "tc_common.cuh"

namespace ig {

namespace {
constexpr int BM = 128, BK = 64;
constexpr int NUM_THREADS = 256;

// EPI_GATED_RES staging (gated_reduce_chunk): per epilogue warp two [32 rows][32 fp32] tiles
constexpr int EPI_RED_BYTES = 4 * 2 * 32 * 32 * 4;
template <int BN>
struct Cfg {
  static constexpr int STAGES = BN == 256 ? 4 : (BN == 128 ? 6 : 8);
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;  // double-buffered fp32 accumulator
  static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_RED_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

// GELU-tanh with the MUFU tanh (rel. error ~2^-11, below the bf16 output rounding 2^-8)
// the same GELU on a pair with packed f32x2 FMA-pipe ops (half the FP instructions)
__device__ __forceinline__ float2 gelu_tanh_fast2(float2 x) {
  const float2 xx = __fmul2_rn(x, x);
  const float2 inner = __ffma2_rn(__fmul2_rn(xx, make_float2(0.044715f, 0.044715f)), x, x);
  const float2 u = __fmul2_rn(inner, make_float2(0.7978845608028654f, 0.7978845608028654f));
  float2 t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t.x) : "f"(u.x));
  asm("tanh.approx.f32 %0, %1;" : "=f"(t.y) : "f"(u.y));
  const float2 hx = __fmul2_rn(x, make_float2(0.5f, 0.5f));
  return __ffma2_rn(hx, t, hx);
}

__device__ __forceinline__ float gelu_tanh_fast(float x) {
  const float u = 0.7978845608028654f * fmaf(0.044715f * x, x * x, x);
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
  return 0.5f * x * (1.0f + t);
}

// Grouped raster (L2 reuse): consecutive tiles walk G m-blocks first, then n, so the tiles in
// flight share a small band of A rows (G blocks) and of B rows; G is sized on the host so the
// A band stays well inside L2 (measured: n-fastest order re-read B up to 6.5x).
__device__ __forceinline__ void tile_coords(int t, int num_m, int num_n, int G, int& mb, int& nb) {
  const int group_size = G * num_n;
  const int group = t / group_size;
  const int first_m = group * G;
  const int gm = min(G, num_m - first_m);
  const int local = t - group * group_size;
  mb = first_m + local % gm;
  nb = local / gm;
}

// EPI_GEGLU: 32 hidden columns (ra) and their 32 gate columns (rg, 128 columns later in the
// interleaved tile) -> 32 outputs at column n0/2 + c: (a + b_a) * gelu_erf(g + b_g)
__device__ __forceinline__ void epilogue_geglu(const GemmArgs& g, int row, int ocol, const uint32_t (&ra)[32],
                                               const uint32_t (&rg)[32], const bf16* ba, const bf16* bg) {
  bf16* c = reinterpret_cast<bf16*>(g.C) + (long long)row * g.ldc + ocol;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 u;
    uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float y[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = q * 8 + 2 * e + h;
        float a = __uint_as_float(ra[i]), gt = __uint_as_float(rg[i]);
        if (ba) { a += __bfloat162float(ba[i]); gt += __bfloat162float(bg[i]); }
        y[h] = a * (0.5f * gt * (1.f + erff(gt * 0.70710678118654752f)));
      }
      __nv_bfloat162 p = __floats2bfloat162_rn(y[0], y[1]);
      w[e] = *reinterpret_cast<uint32_t*>(&p);
    }
    reinterpret_cast<uint4*>(c)[q] = u;
  }
}

// epilogue math of one 32-column chunk of one row, in registers: bias, then GELU / positional or
// per-image term (EPI_POS) / residual (EPI_ADDRES).  bchunk: this chunk's 32 bias values (global
// memory, or the tile's bias slice staged in shared memory by the 2-CTA kernel), nullptr
// without bias.  Row-dependent loads only for rows < M.
__device__ __forceinline__ void chunk_math(const GemmArgs& g, int row, int col0, float (&v)[32], const RowInfo& info,
                                           const bf16* bchunk) {
  const bool full = col0 + 32 <= g.N;
  if (bchunk) {
    if (full) {
      const uint4* b4 = reinterpret_cast<const uint4*>(bchunk);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 u = b4[q];
        const __nv_bfloat162* hb = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 y = __fadd2_rn(make_float2(v[q * 8 + 2 * e], v[q * 8 + 2 * e + 1]), __bfloat1622float2(hb[e]));
          v[q * 8 + 2 * e] = y.x;
          v[q * 8 + 2 * e + 1] = y.y;
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col0 + i < g.N) v[i] += __bfloat162float(bchunk[i]);
    }
  }
  if (g.epi == EPI_GELU) {
    if (g.precise_gelu) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = gelu_tanh(v[i]);
    } else {
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        const float2 y = gelu_tanh_fast2(make_float2(v[i], v[i + 1]));
        v[i] = y.x;
        v[i + 1] = y.y;
      }
    }
  } else if (g.epi == EPI_POS && row < g.M && g.pos) {
    const long long prow = g.pos_div > 0 ? (long long)(g.ri_off + row) / g.pos_div : (long long)info.tok;
    const bf16* pos = reinterpret_cast<const bf16*>(g.pos) + prow * g.pos_ld + col0;
    if (full && (reinterpret_cast<uintptr_t>(pos) & 15) == 0) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(pos) + q);
        const __nv_bfloat162* hb = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 p = __bfloat1622float2(hb[e]);
          v[8 * q + 2 * e] += p.x;
          v[8 * q + 2 * e + 1] += p.y;
        }
      }
    } else {
      for (int i = 0; i < 32; ++i)
        if (col0 + i < g.N) v[i] += __bfloat162float(pos[i]);
    }
  } else if (g.epi == EPI_ADDRES && row < g.M) {
    const float* rs = g.res + (long long)row * g.ldc + col0;
    if (full) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(rs) + q);
        v[4 * q] += a.x; v[4 * q + 1] += a.y; v[4 * q + 2] += a.z; v[4 * q + 3] += a.w;
      }
    } else {
      for (int i = 0; i < 32; ++i)
        if (col0 + i < g.N) v[i] += rs[i];
    }
  }
}

// thread-per-row stores of one chunk (bf16 outputs: a TMA-store variant measured 0-4% slower on
// the GELU / store GEMMs; fp32 outputs go through tma_store_f32)
template <int BN>
__device__ __forceinline__ void epilogue_chunk(const GemmArgs& g, int row, int col0, const uint32_t (&r)[32],
                                               const RowInfo* info, const bf16* bchunk) {
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
  const bool full = col0 + 32 <= g.N;
  chunk_math(g, row, col0, v, *info, bchunk);
  if (g.out_f32 || g.epi == EPI_POS || g.epi == EPI_ADDRES) {
    float* c = reinterpret_cast<float*>(g.C) + (long long)row * g.ldc + col0;
    if (full) {
#pragma unroll
      for (int q = 0; q < 8; ++q)
        reinterpret_cast<float4*>(c)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else {
      for (int i = 0; i < 32; ++i)
        if (col0 + i < g.N) c[i] = v[i];
    }
  } else {
    bf16* c = reinterpret_cast<bf16*>(g.C) + (long long)row * g.ldc + col0;
    if (full) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 u;
        uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          __nv_bfloat162 p = __floats2bfloat162_rn(v[q * 8 + 2 * e], v[q * 8 + 2 * e + 1]);
          w[e] = *reinterpret_cast<uint32_t*>(&p);
        }
        reinterpret_cast<uint4*>(c)[q] = u;
      }
    } else {
      for (int i = 0; i < 32; ++i)
        if (col0 + i < g.N) c[i] = __float2bfloat16_rn(v[i]);
    }
  }
}

__device__ __forceinline__ bool tma_out_f32(const GemmArgs& g) {
  return ((g.epi == EPI_STORE || g.epi == EPI_GELU) && g.out_f32) || g.epi == EPI_POS || g.epi == EPI_ADDRES;
}
// Stores through the TMA unit: a warp's 32 rows x 128 bytes (32 fp32 columns) are
// staged in shared memory in the SWIZZLE_128B layout of the output map (16-byte chunk q of row
// r at slot q ^ (r & 7)) and written by one cp.async.bulk.tensor store — full 128-byte rows per
// transaction instead of 32 scattered 16-byte pieces per warp instruction; rows >= M and
// columns >= N fall outside the map.  Two staging buffers per warp alternate (`cnt`), reused
// after the bulk group issued from them has been read.
__device__ __forceinline__ void tma_stage_wait(int lane, int& cnt, int& k) {
  k = cnt++;
  if (k >= 2) {
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
  }
}
__device__ __forceinline__ void tma_stage_issue(const CUtensorMap* tm, int lane, float4* buf, int col0, int row0,
                                                bool reduce_add) {
  tc::fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    if (reduce_add)
      asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];"
                   ::"l"(reinterpret_cast<uint64_t>(tm)), "r"(tc::smem_u32(buf)), "r"(col0), "r"(row0)
                   : "memory");
    else
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
                   ::"l"(reinterpret_cast<uint64_t>(tm)), "r"(tc::smem_u32(buf)), "r"(col0), "r"(row0)
                   : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
}
// fp32 output (EPI_STORE / EPI_GELU with out_f32, EPI_POS, EPI_ADDRES): 32 columns
__device__ __forceinline__ void tma_store_f32(const GemmArgs& g, const CUtensorMap* tm, int lane, int row0, int col0,
                                              const uint32_t (&r)[32], const RowInfo& info, const bf16* bchunk,
                                              float4* wbuf, int& cnt) {
  int k;
  tma_stage_wait(lane, cnt, k);
  tc::tmem_ld_wait();
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
  chunk_math(g, row0 + lane, col0, v, info, bchunk);
  float4* buf = wbuf + (k & 1) * 256;
#pragma unroll
  for (int q = 0; q < 8; ++q)
    buf[lane * 8 + (q ^ (lane & 7))] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  tma_stage_issue(tm, lane, buf, col0, row0, false);
}

// EPI_GATED_RES through the TMA unit: t = rn(gate * (acc + bias)) per element goes into this
// warp's [32 rows x 32 cols] staging tile (16-byte chunk q of row r at slot q ^ (r & 7): the
// SWIZZLE_128B pattern of the map) and one cp.reduce.async.bulk .add.f32 adds the tile into the
// fp32 residual in L2 — coalesced, and no residual loads on the SMs (rows >= M / cols >= N fall
// outside the map).  Both GEMM kernels use it, so every tile path rounds x + t identically (batch
// invariance).  The caller has issued tcgen05.ld of r; two staging buffers alternate per warp
// (`cnt` counts the warp's chunks), and a buffer is rewritten only after the reduce issued from
// it two chunks earlier has read it.
__device__ __forceinline__ void gated_reduce_chunk(const GemmArgs& g, const CUtensorMap* tmX, int lane, int row0,
                                                   int col0, uint32_t (&r)[32], int req, const bf16* bchunk,
                                                   float4* wbuf, int& cnt) {
  const int k = cnt++;
  if (k >= 2) {
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    __syncwarp();
  }
  tc::tmem_ld_wait();
  const bool full = col0 + 32 <= g.N;
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
  if (bchunk) {
    if (full) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 u = reinterpret_cast<const uint4*>(bchunk)[q];
        const __nv_bfloat162* hb = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 y = __fadd2_rn(make_float2(v[q * 8 + 2 * e], v[q * 8 + 2 * e + 1]), __bfloat1622float2(hb[e]));
          v[q * 8 + 2 * e] = y.x;
          v[q * 8 + 2 * e + 1] = y.y;
        }
      }
    } else {
      for (int i = 0; i < 32; ++i)
        if (col0 + i < g.N) v[i] = __fadd_rn(v[i], __bfloat162float(bchunk[i]));
    }
  }
  const float* grow = g.gate + (long long)req * g.gate_ld + col0;
  float4* buf = wbuf + (k & 1) * 256;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    float4 gv = make_float4(0.f, 0.f, 0.f, 0.f);
    if (full) {
      gv = __ldg(reinterpret_cast<const float4*>(grow) + q);
    } else {
      float* gp = reinterpret_cast<float*>(&gv);
      for (int e = 0; e < 4; ++e)
        if (col0 + 4 * q + e < g.N) gp[e] = grow[4 * q + e];
    }
    const float2 lo = __fmul2_rn(make_float2(gv.x, gv.y), make_float2(v[4 * q], v[4 * q + 1]));
    const float2 hi = __fmul2_rn(make_float2(gv.z, gv.w), make_float2(v[4 * q + 2], v[4 * q + 3]));
    buf[lane * 8 + (q ^ (lane & 7))] = make_float4(lo.x, lo.y, hi.x, hi.y);
  }
  tc::fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];"
                 ::"l"(reinterpret_cast<uint64_t>(tmX)), "r"(tc::smem_u32(buf)), "r"(col0), "r"(row0)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
}

// Fused a6 epilogue for one head (d columns starting at absolute column col0 of the [q|k|v]
// output) of one row: bias, per-head RMSNorm with gain (q, k), RoPE at the row's ORIGINAL
// token position (C-AMB 7), then q -> packed Q row, k/v -> the request's positional K/V
// buffer row (the fresh half of the merge by mask index, C-AMB 8).
template <int DH>
__device__ __forceinline__ void epilogue_qkv_head(const GemmArgs& g, int row, int col0, const uint32_t (&r)[DH],
                                                  const RowInfo& info, const bf16* bchunk) {
  const QkvEpi& e = g.qkv;
  // packed f32x2 FMA-pipe arithmetic throughout (the epilogue is issue-bound, like GELU's)
  float2 v[DH / 2];
#pragma unroll
  for (int i = 0; i < DH / 2; ++i) v[i] = make_float2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
  if (bchunk) {
#pragma unroll
    for (int q = 0; q < DH / 8; ++q) {
      uint4 u = reinterpret_cast<const uint4*>(bchunk)[q];
      const __nv_bfloat162* hb = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int t = 0; t < 4; ++t) v[q * 4 + t] = __fadd2_rn(v[q * 4 + t], __bfloat1622float2(hb[t]));
    }
  }
  const int cq = col0 + e.col_base;             // column in [q|k|v] (col_base = H: K/V only)
  const int which = (int)(cq / e.H);            // 0 q, 1 k, 2 v
  const int hcol = (int)(cq - which * e.H);     // column inside the hidden dim
  bf16* dst;
  if (which == 0) {
    dst = reinterpret_cast<bf16*>(e.Q) + (long long)(g.ri_off + row) * e.H + hcol;
  } else {
    dst = reinterpret_cast<bf16*>(e.kv_arena) + info.slot * e.slot_stride + e.buf_off +
          (which == 2 ? e.L * e.H : 0) + (long long)info.kvpos * e.H + hcol;
  }
  if (which < 2) {
    if (e.qk_norm) {
      float2 ss2 = make_float2(0.f, 0.f);
#pragma unroll
      for (int i = 0; i < DH / 2; ++i) ss2 = __ffma2_rn(v[i], v[i], ss2);
      const float rinv = rsqrtf((ss2.x + ss2.y) / DH + 1e-6f);
      const float2 rinv2 = make_float2(rinv, rinv);
      const bf16* gn = reinterpret_cast<const bf16*>(which == 0 ? e.qg : e.kg);
#pragma unroll
      for (int q = 0; q < DH / 8; ++q) {
        uint4 u = reinterpret_cast<const uint4*>(gn)[q];
        const __nv_bfloat162* hg = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int t = 0; t < 4; ++t) v[q * 4 + t] = __fmul2_rn(v[q * 4 + t], __fmul2_rn(rinv2, __bfloat1622float2(hg[t])));
      }
    }
    if (e.rope) {
      int p1 = 0, p2 = 0;
      if (info.tok >= 0) { p1 = info.tok / e.grid_w; p2 = info.tok - p1 * e.grid_w; }
#pragma unroll
      for (int j = 0; j < DH / 2; ++j) {
        const int pos = j < e.ax1_pair ? 0 : (j < e.ax2_pair ? p1 : p2);
        const float2 cs = __ldg(e.rope_tab + (long long)j * e.rope_maxpos + pos);
        // (x0, x1) -> (x0 c - x1 s, x0 s + x1 c) as x0 * (c, s) + x1 * (-s, c)
        const float2 t = __fmul2_rn(make_float2(v[j].y, v[j].y), make_float2(-cs.y, cs.x));
        v[j] = __ffma2_rn(make_float2(v[j].x, v[j].x), cs, t);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < DH / 8; ++q) {
    uint4 u;
    uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      __nv_bfloat162 p = __float22bfloat162_rn(v[q * 4 + t]);
      w[t] = *reinterpret_cast<uint32_t*>(&p);
    }
    reinterpret_cast<uint4*>(dst)[q] = u;
  }
}

template <int BN, bool CONV = false>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmX, const GemmArgs g, int num_m, int num_n, int G) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint8_t* sred = smem + C::STAGES * C::STAGE_BYTES;  // [4 warps][2][32][32] fp32, 1024-aligned
  uint64_t* full = reinterpret_cast<uint64_t*>(sred + EPI_RED_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_tiles = num_m * num_n;
  const int num_k = (g.K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch_desc(&tmA);
    tc::tma_prefetch_desc(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 4);
    }
    tc::fence_barrier_init();
  }
  asm volatile("griddepcontrol.launch_dependents;");
  if (warp == 1) tc::tmem_alloc<C::TMEM_COLS>(tmem_slot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: inputs of the previous kernel visible

  if (warp == 0) {
    if (lane == 0) {  // ===== TMA producer =====
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int mb, nb;
        tile_coords(t, num_m, num_n, G, mb, nb);
        const int m0 = mb * BM, n0 = nb * BN;
        // implicit conv: the tile's 128 output pixels are 128 / min(W, 128) whole image rows (or
        // one 128-pixel run of a wider row) of one image: (image, row, column) of its first pixel,
        // once per tile
        int cn = 0, cy = 0, cx = 0;
        if constexpr (CONV) {
          const long long HW = (long long)g.conv_H * g.conv_W;
          cn = (int)(m0 / HW);
          const int rem = (int)(m0 - cn * HW);
          cy = rem / g.conv_W;
          cx = rem - cy * g.conv_W;
        }
        int tap = 0, cb = 0;
        for (int kb = 0; kb < num_k; ++kb) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          tc::mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
          if constexpr (CONV) {
            // k-block kb = (tap, 64-channel chunk): ONE 4-D box {64 channels, run, rows, 1} of the
            // zero-padded input at the tap's offset (padded (y + dy, x + dx) = output (y, x) tap)
            const int dy = tap / 3, dx = tap - dy * 3;
            tc::tma_load_4d(sA + stage * C::A_BYTES, &tmA, &full[stage], cb * BK, cx + dx, cy + dy, cn);
            if (++cb == (g.conv_cin >> 6)) { cb = 0; ++tap; }
          } else {
            tc::tma_load_2d(sA + stage * C::A_BYTES, &tmA, &full[stage], kb * BK, m0);
          }
          tc::tma_load_2d(sB + stage * C::B_BYTES, &tmB, &full[stage], kb * BK, n0);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ===== MMA issuer =====
      constexpr uint32_t idesc = tc::idesc_bf16(BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        tc::mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_k; ++kb) {
          tc::mbar_wait(&full[stage], phase);
          tc::tc_fence_after();
          const uint32_t a_addr = tc::smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_addr = tc::smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = tc::sdesc_sw128(a_addr + k * 32, 16, 1024);
            const uint64_t bd = tc::sdesc_sw128(b_addr + k * 32, 16, 1024);
            tc::mma_bf16_ss(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          tc::mma_commit(&empty[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        tc::mma_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {  // ===== epilogue =====
    const int quad = warp & 3;
    int red_cnt = 0;  // EPI_GATED_RES chunks reduced so far (staging buffer parity)
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      int mb, nb;
      tile_coords(t, num_m, num_n, G, mb, nb);
      const int m0 = mb * BM, n0 = nb * BN;
      tc::mbar_wait(&tfull[acc], acc_phase);
      tc::tc_fence_after();
      const int row = m0 + quad * 32 + lane;
      RowInfo info{0, 0, 0, 0};
      if (row < g.M && g.ri && (g.epi == EPI_GATED_RES || g.epi == EPI_POS || g.epi == EPI_QKV))
        info = g.ri[g.ri_off + row];
      const uint32_t tbase = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN;
      const bf16* gbias = reinterpret_cast<const bf16*>(g.bias);
#define BIAS_AT(c) (gbias ? gbias + n0 + (c) : nullptr)
      if (g.epi == EPI_QKV) {
        if (g.qkv.head_dim == 128) {
#pragma unroll 1
          for (int c = 0; c < BN; c += 128) {
            uint32_t v[128];
#pragma unroll
            for (int s = 0; s < 4; ++s) tc::tmem_ld32(tbase + c + 32 * s, *reinterpret_cast<uint32_t(*)[32]>(&v[32 * s]));
            tc::tmem_ld_wait();
            if (row < g.M && n0 + c < g.N) epilogue_qkv_head<128>(g, row, n0 + c, v, info, BIAS_AT(c));
          }
        } else {
#pragma unroll 1
          for (int c = 0; c < BN; c += 64) {
            uint32_t v[64];
#pragma unroll
            for (int s = 0; s < 2; ++s) tc::tmem_ld32(tbase + c + 32 * s, *reinterpret_cast<uint32_t(*)[32]>(&v[32 * s]));
            tc::tmem_ld_wait();
            if (row < g.M && n0 + c < g.N) epilogue_qkv_head<64>(g, row, n0 + c, v, info, BIAS_AT(c));
          }
        }
      } else if (BN == 256 && g.epi == EPI_GEGLU) {
#pragma unroll 1
        for (int c = 0; c < 128; c += 32) {
          uint32_t ra[32], rg[32];
          tc::tmem_ld32(tbase + c, ra);
          tc::tmem_ld32(tbase + 128 + c, rg);
          tc::tmem_ld_wait();
          if (row < g.M && n0 + c < g.N) epilogue_geglu(g, row, n0 / 2 + c, ra, rg, BIAS_AT(c), BIAS_AT(128 + c));
        }
      } else if (g.epi == EPI_GATED_RES) {
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          if (n0 + c >= g.N) break;  // warp-uniform
          uint32_t r[32];
          tc::tmem_ld32(tbase + c, r);
          gated_reduce_chunk(g, &tmX, lane, m0 + quad * 32, n0 + c, r, info.req, BIAS_AT(c),
                             reinterpret_cast<float4*>(sred) + quad * 2 * 256, red_cnt);
        }
      } else if (tma_out_f32(g)) {
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          if (n0 + c >= g.N) break;  // warp-uniform
          uint32_t r[32];
          tc::tmem_ld32(tbase + c, r);
          tma_store_f32(g, &tmX, lane, m0 + quad * 32, n0 + c, r, info, BIAS_AT(c),
                        reinterpret_cast<float4*>(sred) + quad * 2 * 256, red_cnt);
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          uint32_t r[32];
          tc::tmem_ld32(tbase + c, r);
          tc::tmem_ld_wait();
          if (row < g.M && n0 + c < g.N) epilogue_chunk<BN>(g, row, n0 + c, r, &info, BIAS_AT(c));
        }
      }
#undef BIAS_AT
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  if (warp >= 4 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // TMA stores / reduces
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<C::TMEM_COLS>(tmem_base);
}


// ---- 2-CTA variant: a cluster of two CTAs (one TPC) computes a 256 x 256 tile with
// tcgen05.mma.cta_group::2 (M = 256, N = 256, K = 16).  Each CTA loads its own 128 rows of A
// and 128 rows (half) of B; both halves of B feed the pair's MMA, halving per-SM operand
// traffic versus the 1-CTA 128 x 256 tile.  Only the leader CTA issues MMAs; commits are
// multicast to both CTAs; each CTA's epilogue warps drain their own TMEM (rows 128r..128r+127)
// and release the accumulator to the leader with a cluster-scope mbarrier arrive.
// BN: tile width (256; a 256 x 160 variant measured no faster than 256 even where it needs fewer
// wave-cycles — its N = 160 MMAs cost about as much as N = 256 — and was removed)
template <int BN>
struct Cfg2 {
  static constexpr int STAGES = BN == 256 ? 6 : 7;
  static constexpr int A_BYTES = 128 * BK * 2;
  static constexpr int B_BYTES = (BN / 2) * BK * 2;  // this CTA's half of the B tile
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 512;
  static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_RED_BYTES + 1024 + 256 + 2 * 256 * 2 /*bias slices*/;
};

template <bool CONV = false, int BN = 256>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmX, const GemmArgs g, int num_m, int num_n, int G) {
  static_assert(BN % 32 == 0 && (BN / 2) % 8 == 0 && BN <= 256, "2-CTA tile width");
  using C = Cfg2<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint8_t* sred = smem + C::STAGES * C::STAGE_BYTES;  // [4 warps][2][32][32] fp32, 1024-aligned
  uint64_t* full = reinterpret_cast<uint64_t*>(sred + EPI_RED_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  bf16* sbias = reinterpret_cast<bf16*>(sred + EPI_RED_BYTES + 256);  // [2][256]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = tc::cluster_ctarank();
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  const int num_tiles = num_m * num_n;
  const int num_k = (g.K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch_desc(&tmA);
    tc::tma_prefetch_desc(&tmB);
    if (g.epi != EPI_QKV && g.epi != EPI_GEGLU) tc::tma_prefetch_desc(&tmX);
    for (int s = 0; s < C::STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is used)
    }
    tc::fence_barrier_init();
  }
  asm volatile("griddepcontrol.launch_dependents;");
  if (warp == 1) tc::tmem_alloc2<C::TMEM_COLS>(tmem_slot);
  tc::tc_fence_before();
  tc::cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: inputs of the previous kernel visible

  if (warp == 0) {
    if (lane == 0) {  // ===== TMA producer (both CTAs) =====
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cluster; t < num_tiles; t += nclusters) {
        int mb, nb;
        tile_coords(t, num_m, num_n, G, mb, nb);
        const int m0 = mb * 256 + rank * 128, n0 = nb * BN + rank * (BN / 2);
        int cn = 0, cy = 0, cx = 0;  // implicit conv: first output pixel of this CTA's 128 (see gemm_tc_kernel)
        if constexpr (CONV) {
          const long long HW = (long long)g.conv_H * g.conv_W;
          cn = (int)(m0 / HW);
          const int rem = (int)(m0 - cn * HW);
          cy = rem / g.conv_W;
          cx = rem - cy * g.conv_W;
        }
        int tap = 0, cb = 0;
        for (int kb = 0; kb < num_k; ++kb) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          if (rank == 0) tc::mbar_arrive_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
          if constexpr (CONV) {
            const int dy = tap / 3, dx = tap - dy * 3;
            tc::tma_load_4d_2sm(sA + stage * C::A_BYTES, &tmA, &full[stage], cb * BK, cx + dx, cy + dy, cn);
            if (++cb == (g.conv_cin >> 6)) { cb = 0; ++tap; }
          } else {
            tc::tma_load_2d_2sm(sA + stage * C::A_BYTES, &tmA, &full[stage], kb * BK, m0);
          }
          tc::tma_load_2d_2sm(sB + stage * C::B_BYTES, &tmB, &full[stage], kb * BK, n0);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // ===== MMA issuer (leader CTA) =====
      constexpr uint32_t idesc = tc::idesc_bf16(256, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = cluster; t < num_tiles; t += nclusters) {
        tc::mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < num_k; ++kb) {
          tc::mbar_wait(&full[stage], phase);
          tc::tc_fence_after();
          const uint32_t a_addr = tc::smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_addr = tc::smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            tc::mma2_bf16_ss(d_tmem, tc::sdesc_sw128(a_addr + k * 32, 16, 1024),
                             tc::sdesc_sw128(b_addr + k * 32, 16, 1024), idesc, (kb | k) != 0);
          tc::mma2_commit_mc(&empty[stage], 0x3);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        tc::mma2_commit_mc(&tfull[acc], 0x3);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {  // ===== epilogue (both CTAs, own TMEM rows) =====
    const int quad = warp & 3;
    int red_cnt = 0;  // EPI_GATED_RES chunks reduced so far (staging buffer parity)
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = cluster; t < num_tiles; t += nclusters) {
      int mb, nb;
      tile_coords(t, num_m, num_n, G, mb, nb);
      const int m0 = mb * 256 + rank * 128, n0 = nb * BN;
      // the tile's bias slice -> shared memory (one 4-byte load per epilogue thread), so the
      // chunks below read it at shared-memory latency instead of one global round trip each;
      // double-buffered by accumulator, and the per-tile barrier keeps warps within one tile
      bf16* sb = sbias + acc * 256;  // slice stride 256 whatever BN: every thread writes 2 of 256 entries
      const bf16* gbias = reinterpret_cast<const bf16*>(g.bias);
      if (gbias) {
        const int i = 2 * ((warp - 4) * 32 + lane);
        sb[i] = n0 + i < g.N ? gbias[n0 + i] : __float2bfloat16_rn(0.f);
        sb[i + 1] = n0 + i + 1 < g.N ? gbias[n0 + i + 1] : __float2bfloat16_rn(0.f);
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
#define BIAS_AT(c) (gbias ? sb + (c) : nullptr)
      tc::mbar_wait(&tfull[acc], acc_phase);
      tc::tc_fence_after();
      const int row = m0 + quad * 32 + lane;
      RowInfo info{0, 0, 0, 0};
      if (row < g.M && g.ri && (g.epi == EPI_GATED_RES || g.epi == EPI_POS || g.epi == EPI_QKV))
        info = g.ri[g.ri_off + row];
      const uint32_t tbase = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN;
      if (BN == 256 && g.epi == EPI_QKV) {
        if (g.qkv.head_dim == 128) {
#pragma unroll 1
          for (int c = 0; c < BN; c += 128) {
            uint32_t v[128];
#pragma unroll
            for (int s = 0; s < 4; ++s) tc::tmem_ld32(tbase + c + 32 * s, *reinterpret_cast<uint32_t(*)[32]>(&v[32 * s]));
            tc::tmem_ld_wait();
            if (row < g.M && n0 + c < g.N) epilogue_qkv_head<128>(g, row, n0 + c, v, info, BIAS_AT(c));
          }
        } else {
#pragma unroll 1
          for (int c = 0; c < BN; c += 64) {
            uint32_t v[64];
#pragma unroll
            for (int s = 0; s < 2; ++s) tc::tmem_ld32(tbase + c + 32 * s, *reinterpret_cast<uint32_t(*)[32]>(&v[32 * s]));
            tc::tmem_ld_wait();
            if (row < g.M && n0 + c < g.N) epilogue_qkv_head<64>(g, row, n0 + c, v, info, BIAS_AT(c));
          }
        }
      } else if (BN == 256 && g.epi == EPI_GEGLU) {
#pragma unroll 1
        for (int c = 0; c < 128; c += 32) {
          uint32_t ra[32], rg[32];
          tc::tmem_ld32(tbase + c, ra);
          tc::tmem_ld32(tbase + 128 + c, rg);
          tc::tmem_ld_wait();
          if (row < g.M && n0 + c < g.N) epilogue_geglu(g, row, n0 / 2 + c, ra, rg, BIAS_AT(c), BIAS_AT(128 + c));
        }
      } else if (g.epi == EPI_GATED_RES) {
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          if (n0 + c >= g.N) break;  // warp-uniform
          uint32_t r[32];
          tc::tmem_ld32(tbase + c, r);
          gated_reduce_chunk(g, &tmX, lane, m0 + quad * 32, n0 + c, r, info.req, gbias ? sb + c : nullptr,
                             reinterpret_cast<float4*>(sred) + quad * 2 * 256, red_cnt);
        }
      } else if (tma_out_f32(g)) {
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          if (n0 + c >= g.N) break;  // warp-uniform
          uint32_t r[32];
          tc::tmem_ld32(tbase + c, r);
          tma_store_f32(g, &tmX, lane, m0 + quad * 32, n0 + c, r, info, BIAS_AT(c),
                        reinterpret_cast<float4*>(sred) + quad * 2 * 256, red_cnt);
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          uint32_t r[32];
          tc::tmem_ld32(tbase + c, r);
          tc::tmem_ld_wait();
          if (row < g.M && n0 + c < g.N) epilogue_chunk<BN>(g, row, n0 + c, r, &info, BIAS_AT(c));
        }
      }
#undef BIAS_AT
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0) tc::mbar_arrive(&tempty[acc]);
        else tc::mbar_arrive_cluster(&tempty[acc], 0);
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  if (warp >= 4 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // TMA stores / reduces
  tc::tc_fence_before();
  tc::cluster_sync();
  if (warp == 1) tc::tmem_dealloc2<C::TMEM_COLS>(tmem_base);
}

// ---- host side -----------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;
int g_num_sms = 0;

void init_driver() {
  std::call_once(g_encode_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(gemm_tc_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<256>::SMEM);
    cudaFuncSetAttribute(gemm_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<128>::SMEM);
    cudaFuncSetAttribute(gemm_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<64>::SMEM);
    cudaFuncSetAttribute(gemm_tc_kernel<256, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<256>::SMEM);
    cudaFuncSetAttribute(gemm_tc_kernel<128, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<128>::SMEM);
    cudaFuncSetAttribute(gemm_tc2_kernel<false, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg2<256>::SMEM);
    cudaFuncSetAttribute(gemm_tc2_kernel<true, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg2<256>::SMEM);
  });
}

// 2-D bf16 tensor map over a row-major [rows, cols] matrix with leading dimension ld, box
// [box_rows, 64 cols], 128-byte swizzle; out-of-bounds reads fill zeros.
// Encoded maps are cached per (pointer, shape, box): the weights' maps never change and the
// workspaces' recur every step, so the driver encode runs once instead of twice per launch
// (host enqueue cost matters for small single-request steps).
struct TmapKey {
  const void* ptr; long long rows, cols, ld; int box;
  bool operator==(const TmapKey& o) const {
    return ptr == o.ptr && rows == o.rows && cols == o.cols && ld == o.ld && box == o.box;
  }
};
struct TmapHash {
  size_t operator()(const TmapKey& k) const {
    size_t h = std::hash<const void*>()(k.ptr);
    for (long long v : {k.rows, k.cols, k.ld, (long long)k.box}) h = h * 1000003u ^ std::hash<long long>()(v);
    return h;
  }
};
bool encode_tmap(CUtensorMap* m, const void* ptr, long long rows, long long cols, long long ld, int box_rows);
bool make_tmap(CUtensorMap* m, const void* ptr, long long rows, long long cols, long long ld, int box_rows) {
  thread_local std::unordered_map<TmapKey, CUtensorMap, TmapHash> cache;
  const TmapKey k{ptr, rows, cols, ld, box_rows};
  auto it = cache.find(k);
  if (it != cache.end()) { *m = it->second; return true; }
  if (!encode_tmap(m, ptr, rows, cols, ld, box_rows)) return false;
  if (cache.size() > 8192) cache.clear();
  cache.emplace(k, *m);
  return true;
}
bool encode_tmap(CUtensorMap* m, const void* ptr, long long rows, long long cols, long long ld, int box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}
// fp32 [rows, cols] (ld floats) map with a 32 x 32 box, 128-byte swizzle: the target of the gated
// residual's TMA reduce-add
bool make_tmap_f32(CUtensorMap* m, const void* ptr, long long rows, long long cols, long long ld) {
  thread_local std::unordered_map<TmapKey, CUtensorMap, TmapHash> cache;
  const TmapKey k{ptr, rows, cols, ld, -32};
  auto it = cache.find(k);
  if (it != cache.end()) { *m = it->second; return true; }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  if (cache.size() > 8192) cache.clear();
  cache.emplace(k, *m);
  return true;
}
// implicit-conv A operand: the zero-padded NHWC input as a 4-D map {C_in, W + 2, H + 2, N} with a
// {64, min(W, 128), 128 / min(W, 128), 1} box: a tile's 128 output pixels at one tap and one
// 64-channel chunk in ONE TMA load (rows of the box skip the 2 padding pixels between image rows)
bool make_tmap_conv(CUtensorMap* m, const void* ptr, long long n, int H, int W, int cin) {
  thread_local std::unordered_map<TmapKey, CUtensorMap, TmapHash> cache;
  const TmapKey k{ptr, n * (H + 2), (long long)(W + 2), cin, -4};
  auto it = cache.find(k);
  if (it != cache.end()) { *m = it->second; return true; }
  const int bw = W < BM ? W : BM;
  cuuint64_t dims[4] = {(cuuint64_t)cin, (cuuint64_t)(W + 2), (cuuint64_t)(H + 2), (cuuint64_t)n};
  cuuint64_t strides[3] = {(cuuint64_t)cin * 2, (cuuint64_t)cin * 2 * (W + 2), (cuuint64_t)cin * 2 * (W + 2) * (H + 2)};
  cuuint32_t box[4] = {64, (cuuint32_t)bw, (cuuint32_t)(BM / bw), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  if (cache.size() > 8192) cache.clear();
  cache.emplace(k, *m);
  return true;
}

// the output map of the TMA epilogues: fp32 32 x 32 boxes (gated residual reduce-add, fp32
// stores); `fallback` (any valid map) otherwise
CUtensorMap out_map(const GemmArgs& g, const CUtensorMap& fallback) {
  CUtensorMap m = fallback;
  const bool f32 = g.epi == EPI_GATED_RES || g.epi == EPI_POS || g.epi == EPI_ADDRES ||
                   ((g.epi == EPI_STORE || g.epi == EPI_GELU) && g.out_f32);
  if (f32) make_tmap_f32(&m, g.C, g.M, g.N, g.ldc);
  return m;
}
}  // namespace

// m-blocks per raster group: keep the group's A band (G * rows * K * 2 bytes) around 32 MB
int raster_group(int num_m, int rows, int K) {
  const long long band = 32ll << 20;
  long long G = band / ((long long)rows * K * 2);
  if (G < 1) G = 1;
  if (G > num_m) G = num_m;
  return (int)G;
}

bool gemm_tc_supported(const GemmArgs& g) {
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!al16(g.A) || !al16(g.B) || (g.lda & 7) || (g.ldb & 7) || (g.K & 7)) return false;
  if (g.epi == EPI_GEGLU) {
    if (!al16(g.C) || (g.ldc & 7) || g.out_f32 || (g.N % 256)) return false;
  } else if (g.epi == EPI_STORE || g.epi == EPI_GELU) {
    if (!al16(g.C) || (g.ldc & (g.out_f32 ? 3 : 7))) return false;
  } else if (g.epi != EPI_QKV) {
    if (!al16(g.C) || (g.ldc & 3)) return false;
    if (g.epi == EPI_GATED_RES && (!al16(g.gate) || (g.gate_ld & 3))) return false;
    if (g.epi == EPI_ADDRES && !al16(g.res)) return false;
  }
  if (g.bias && !al16(g.bias)) return false;
  if (g.epi == EPI_QKV && ((g.qkv.head_dim != 128 && g.qkv.head_dim != 64) || (g.qkv.H % 64) || g.N + g.qkv.col_base != 3 * g.qkv.H))
    return false;
  return true;
}

void gemm_tc_init() { init_driver(); }

void launch_gemm_tc(const GemmArgs& g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0) return;
  init_driver();
  bool wide = g.N > 128 || g.epi == EPI_QKV || g.epi == EPI_GEGLU;
  // Small problems (fewer 256 x 256 tiles than a quarter of the SMs, e.g. the single-request
  // or low-mask-ratio GEMMs): 128 x 128 one-CTA tiles put 4x as many SMs to work.  Only the
  // tile shape changes — every output is still one full-K accumulation in the same K order —
  // so results do not depend on the choice (batch invariance holds).
  const ig_tuning& tun = ig_tuning_ref();
  const bool no_small = !tun.gemm_small_tiles;
  const long long tiles2 = (long long)((g.M + 255) / 256) * ((g.N + 255) / 256);
  if (!no_small && wide && g.epi != EPI_GEGLU && tiles2 * 4 < g_num_sms) wide = false;
  if (wide && tun.gemm_two_cta && g.M > 128) {  // 2-CTA 256 x BN tiles
    constexpr int BN2 = 256;
    CUtensorMap ta, tb;
    make_tmap(&ta, g.A, g.M, g.K, g.lda, 128);
    make_tmap(&tb, g.B, g.N, g.K, g.ldb, BN2 / 2);
    const int num_m = (g.M + 255) / 256, num_n = (g.N + BN2 - 1) / BN2;
    const int tiles = num_m * num_n;
    const int clusters = tiles < g_num_sms / 2 ? tiles : g_num_sms / 2;
    const int G2 = raster_group(num_m, 256, g.K);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * clusters); cfg.blockDim = dim3(NUM_THREADS); cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at; cfg.numAttrs = g.pdl ? 1 : 0;
    const CUtensorMap tx = out_map(g, tb);
    cfg.dynamicSmemBytes = Cfg2<256>::SMEM;
    cudaLaunchKernelEx(&cfg, gemm_tc2_kernel<false, 256>, ta, tb, tx, g, num_m, num_n, G2);
    return;
  }
  // Still fewer 128 x 128 tiles than half the SMs (single-request SD3 out-projections / fc2:
  // 36-48 tiles of K = 1536-6144, one long k-loop each on a third of the GPU): 128 x 64 tiles
  // double the CTAs.  Tile shape only (same full-K order per output), so batch invariance holds;
  // the QKV / GEGLU epilogues need whole heads / paired halves (>= 128 columns).
  const bool no_bn64 = !tun.gemm_bn64;
  const long long tiles1 = (long long)((g.M + BM - 1) / BM) * ((g.N + 127) / 128);
  const bool narrow = !wide && !no_bn64 && !no_small && g.epi != EPI_QKV && g.epi != EPI_GEGLU &&
                      tiles1 * 2 <= g_num_sms;
  const int BN = wide ? 256 : (narrow ? 64 : 128);
  CUtensorMap ta, tb;
  make_tmap(&ta, g.A, g.M, g.K, g.lda, BM);
  make_tmap(&tb, g.B, g.N, g.K, g.ldb, BN);
  const int num_m = (g.M + BM - 1) / BM, num_n = (g.N + BN - 1) / BN;
  const int tiles = num_m * num_n;
  const int grid = tiles < g_num_sms ? tiles : g_num_sms;
  const int G = raster_group(num_m, BM, g.K);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid); cfg.blockDim = dim3(NUM_THREADS); cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at; cfg.numAttrs = g.pdl ? 1 : 0;
  const CUtensorMap tx = out_map(g, tb);
  if (wide) {
    cfg.dynamicSmemBytes = Cfg<256>::SMEM;
    cudaLaunchKernelEx(&cfg, gemm_tc_kernel<256>, ta, tb, tx, g, num_m, num_n, G);
  } else if (narrow) {
    cfg.dynamicSmemBytes = Cfg<64>::SMEM;
    cudaLaunchKernelEx(&cfg, gemm_tc_kernel<64>, ta, tb, tx, g, num_m, num_n, G);
  } else {
    cfg.dynamicSmemBytes = Cfg<128>::SMEM;
    cudaLaunchKernelEx(&cfg, gemm_tc_kernel<128>, ta, tb, tx, g, num_m, num_n, G);
  }
}

bool conv3x3_tc_supported(int H, int W, int cin) {
  if (cin % 64 || H <= 0 || W <= 0) return false;
  const bool wok = (W == 8 || W == 16 || W == 32 || W == 64 || W == 128 || W % 128 == 0);
  return wok && ((long long)H * W) % BM == 0;
}

void launch_conv3x3_tc(const GemmArgs& g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0) return;
  init_driver();
  const long long images = g.M / ((long long)g.conv_H * g.conv_W);
  CUtensorMap ta, tb;
  make_tmap_conv(&ta, g.A, images, g.conv_H, g.conv_W, g.conv_cin);  // padded input, 4-D box per tile
  // C_out a multiple of 256 (1280): 2-CTA 256 x 256 tiles (half the B operand per SM), like the
  // projections; else 128 x 128 one-CTA tiles (C_out 320 / 640: no half-empty 256-column tile)
  const ig_tuning& tun = ig_tuning_ref();
  const bool conv_1cta = !tun.conv_two_cta;
  // C_out >= 256: 2-CTA 256 x 256 tiles, the last one partial for C_out = 320 / 640 (measured:
  // as fast as or faster than 256 x 160 tiles, whose N = 160 MMAs cost about as much as N = 256
  // — ncu cycles in profiles/r02_bn160_ab_cycles.txt — and than 128 x 128 one-CTA tiles)
  if (!conv_1cta && tun.gemm_two_cta && g.N >= 256 && g.M > 128) {
    constexpr int BN2 = 256;
    CUtensorMap tb2;
    make_tmap(&tb2, g.B, g.N, g.K, g.ldb, BN2 / 2);
    const int num_m = (g.M + 255) / 256, num_n = (g.N + BN2 - 1) / BN2;
    const int tiles = num_m * num_n;
    const int clusters = tiles < g_num_sms / 2 ? tiles : g_num_sms / 2;
    gemm_tc2_kernel<true, 256><<<2 * clusters, NUM_THREADS, Cfg2<256>::SMEM, st>>>(ta, tb2, out_map(g, tb2), g, num_m, num_n,
                                                                                raster_group(num_m, 256, g.K));
    return;
  }
  const bool wide = g.N >= 256 && g.N % 256 == 0;
  const int BN = wide ? 256 : 128;
  make_tmap(&tb, g.B, g.N, g.K, g.ldb, BN);
  const int num_m = (g.M + BM - 1) / BM, num_n = (g.N + BN - 1) / BN;
  const int tiles = num_m * num_n;
  const int grid = tiles < g_num_sms ? tiles : g_num_sms;
  const int G = raster_group(num_m, BM, g.K);
  if (wide)
    gemm_tc_kernel<256, true><<<grid, NUM_THREADS, Cfg<256>::SMEM, st>>>(ta, tb, out_map(g, tb), g, num_m, num_n, G);
  else
    gemm_tc_kernel<128, true><<<grid, NUM_THREADS, Cfg<128>::SMEM, st>>>(ta, tb, out_map(g, tb), g, num_m, num_n, G);
}

}  // namespace ig
