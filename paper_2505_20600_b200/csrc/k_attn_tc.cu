// k_attn_tc.cu — kernel (d): varlen flash attention on tcgen05 tensor cores (bf16, d = 128).
// Masked queries x merged full K/V ("Q ... of only the newly generated token
// along with the K and V matrices of all present tokens"): each ragged query segment of the
// packed continuous batch attends to its own request's positional K/V buffer of L rows.
//
// One CTA per (pair of 128-row query tiles A/B, head, segment); 384 threads:
//   warp 0       TMA producer: Q_A, Q_B once, then K/V tiles of 128 keys (2-stage ring,
//                shared by both query tiles)
//   warp 1       TMEM allocator + single-thread MMA issuer, ping-pong over the two tiles:
//                  S_t = Q_t K_j^T      (SS, M=128 N=128 K=128, fp32 in TMEM)
//                  O_t += P_t V_j       (TS: P read from TMEM where it overwrote S_t, V an
//                                        MN-major smem operand; fp32 O_t in TMEM)
//                while softmax group A works on S_A(j) the tensor core runs S_B(j) / PV_B(j-1)
//   warps 4..7   softmax of tile A, warps 8..11 softmax of tile B; thread = query row (TMEM
//                lane): row max, exp2, row sum in fp32, P packed to bf16 and stored back to
//                TMEM (tcgen05.st).  Lazy O correction with a threshold: a row keeps its stale
//                max unless the new max exceeds it by more than 8 (log2 units, P <= 2^8), and
//                only rescales O then — decisions per row, so a row's result never depends on
//                its tile-mates (batch invariance).
// TMEM (512 columns): [S_A|P_A 128][O_A 128][S_B|P_B 128][O_B 128].
// Ordering: tcgen05.mma execute in issue order, and S_t(j+1) is issued after PV_t(j), so when
// softmax t sees S_t(j+1) complete (its commit covers every earlier MMA) PV_t(j) has finished
// reading P_t(j) and writing O_t: O_t is stable for the correction, the P region is free.
// Keys >= L (ragged last tile) are zero-filled by TMA and masked to -inf.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <mutex>
#include <vector>
#include <cstdlib>
#include "kernels.h"
#include "tc_common.cuh"

namespace ig {
namespace {

constexpr int BQ = 128, BKV = 128;
constexpr int CHUNK = 128 * 64 * 2;             // one [128 rows x 64 cols] bf16 SW128 box
constexpr int KSTAGES = 3;   // K ring (needed first: S = Q K^T), fetched two tiles ahead
constexpr int VSTAGES = 2;   // V ring (needed one softmax later: O += P V)
constexpr int NTHREADS = 384;
template <int D>
struct AC {                                     // per-head-dim configuration (d = 64 or 128)
  static constexpr int NCH = D / 64;            // 64-column SW128 boxes per row
  static constexpr int Q_BYTES = NCH * CHUNK;   // per query tile
  static constexpr int KV_BYTES = NCH * CHUNK;  // each for K and V
  static constexpr int TSTRIDE = 128 + D;       // TMEM columns per tile: S/P 128, O D
  static constexpr int SMEM_BYTES = 2 * Q_BYTES + (KSTAGES + VSTAGES) * KV_BYTES + 1024 + 256;
};
constexpr float RESCALE_THRESHOLD = 8.0f;       // log2 units
// exp2 on the FMA pipe (ex2_poly2) for one pair in 16, interleaved with the MUFU pairs
// (ncu A/B, batch-8 shape: 0.939 vs 0.954 ms; 8 or 16 pairs in 64 are slower)
#ifndef POLY_AT
#define POLY_AT(i) (((i) & 15) == 15)
#endif
// d = 64 does half the MMA work per score, so the MUFU exp2 rate (16 / clk / SM) bounds the
// softmax at about twice the MMA time: move a larger share of the pairs to the FMA pipe
// (round 2, without the register split every share 1/4 .. 5/8 was slower — it spilled; with
// setmaxnreg 1 in 4 pairs is 5% fewer cycles at the UNet / SD3 shapes, 3 in 8 and 1 in 2 less
// good: profiles/r02_attn_restructure_ab.md)
#ifndef POLY64_AT
#define POLY64_AT(i) (((i) & 3) == 3)
#endif
#ifndef ATTN_MAX3
#define ATTN_MAX3 0       // row max with 3-input FMNMX3 (half the max-phase instructions)
#endif
#ifndef ATTN_SETMAXNREG
#define ATTN_SETMAXNREG 1  // per-warpgroup register split (producer/MMA low, softmax high)
#endif
#ifndef ATTN_REGS_PRODUCER
#define ATTN_REGS_PRODUCER 56
#endif
#ifndef ATTN_REGS_SOFTMAX
#define ATTN_REGS_SOFTMAX 224
#endif
#ifndef ATTN_SPLIT_S
#define ATTN_SPLIT_S 0  // 1: S_t(j+1) in two N = 64 halves, the first issued once S_t(j) is loaded (measured slower)
#endif
#ifndef ATTN_ST_CHUNKS
#define ATTN_ST_CHUNKS 1  // P stored to TMEM in 1, 2 or 4 pieces as the exps complete
#endif

struct Bars {
  uint64_t q_full;
  uint64_t k_full[KSTAGES], k_empty[KSTAGES], v_full[VSTAGES], v_empty[VSTAGES];
  uint64_t s_full[2], p_full[2], o_done[2], s_used[2];
  uint32_t tmem;
};

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 p = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&p);
}

#ifdef IG_ATTN_TRACE
__device__ long long g_trace[5][2][40];
#define TRACE(ev, t, j)                                                                              \
  do {                                                                                               \
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (j) < 40)                           \
      g_trace[ev][t][j] = (long long)clock64();                                                      \
  } while (0)
#else
#define TRACE(ev, t, j) do { } while (0)
#endif

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

__device__ __forceinline__ float ex2_fast(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe for a pair (relieves the MUFU unit, which would otherwise bound the
// softmax at the tensor-core rate): round-to-nearest split x = j + f, |f| <= 1/2, a degree-3
// polynomial for 2^f (relative error < 1e-5, far below the bf16 rounding of P), and j added
// into the exponent field.  x is clamped at -127 (2^-127 ~ 0).
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  x.x = fmaxf(x.x, -127.f);
  x.y = fmaxf(x.y, -127.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);  // 1.5 * 2^23
  const float2 t = __fadd2_rn(x, magic);
  const float2 j = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __ffma2_rn(j, make_float2(-1.f, -1.f), x);
  float2 p = __ffma2_rn(f, make_float2(0.05550411f, 0.05550411f), make_float2(0.24022651f, 0.24022651f));
  p = __ffma2_rn(p, f, make_float2(0.69314718f, 0.69314718f));
  p = __ffma2_rn(p, f, make_float2(1.f, 1.f));
  const int ex = __float_as_int(t.x) << 23, ey = __float_as_int(t.y) << 23;
  return make_float2(__int_as_float(__float_as_int(p.x) + ex), __int_as_float(__float_as_int(p.y) + ey));
}

__device__ __forceinline__ void tma_load_3d(void* smem, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
      ::"r"(tc::smem_u32(smem)), "l"(reinterpret_cast<uint64_t>(m)), "r"(tc::smem_u32(bar)), "r"(c0), "r"(c1),
      "r"(c2) : "memory");
}

template <int D>
__global__ void __launch_bounds__(NTHREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKV,
                   const AttnArgs a, float scale_log2) {
  asm volatile("griddepcontrol.launch_dependents;");  // let a PDL GEMM (out-projection) stage its prologue
  using C = AC<D>;
  constexpr int Q_BYTES = C::Q_BYTES, KV_BYTES = C::KV_BYTES, TS = C::TSTRIDE;
  // compact grid: blockIdx.x enumerates the (segment, query-tile pair) work items, decoded
  // from the per-segment pair counts (no idle CTAs for short segments)
  int z = blockIdx.z, pair = blockIdx.x;
  if (a.n_pairs > 0) {
    for (z = 0; z < a.nseg; ++z) {
      const int np = (a.segs[z].q_len + 2 * BQ - 1) / (2 * BQ);
      if (pair < np) break;
      pair -= np;
    }
  }
  const AttnSeg seg = a.segs[z];
  const int h = blockIdx.y;
  const int q0 = pair * 2 * BQ;
  if (q0 >= seg.q_len) return;
  const bool has_b = q0 + BQ < seg.q_len;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                              // [2 tiles][Q_BYTES]
  uint8_t* sK = sQ + 2 * Q_BYTES;                  // [KSTAGES][KV_BYTES]
  uint8_t* sV = sK + KSTAGES * KV_BYTES;           // [VSTAGES][KV_BYTES]
  Bars* bar = reinterpret_cast<Bars*>(sV + VSTAGES * KV_BYTES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkv = (a.L + BKV - 1) / BKV;
  const long long H = (long long)a.heads * D;
  const long long plane_elems = (long long)a.L * H;
  const int planeK = (int)((seg.kv_base + a.kv_off) / plane_elems);

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch_desc(&tmQ);
    tc::tma_prefetch_desc(&tmKV);
    tc::mbar_init(&bar->q_full, 1);
    for (int s = 0; s < KSTAGES; ++s) { tc::mbar_init(&bar->k_full[s], 1); tc::mbar_init(&bar->k_empty[s], 1); }
    for (int s = 0; s < VSTAGES; ++s) { tc::mbar_init(&bar->v_full[s], 1); tc::mbar_init(&bar->v_empty[s], 1); }
    for (int t = 0; t < 2; ++t) {
      tc::mbar_init(&bar->s_full[t], 1);
      tc::mbar_init(&bar->p_full[t], 4);
      tc::mbar_init(&bar->o_done[t], 1);
      tc::mbar_init(&bar->s_used[t], 4);
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<512>(&bar->tmem);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = bar->tmem;
  // register split per warpgroup (setmaxnreg, ATTN_SETMAXNREG): the TMA / MMA warpgroup needs few
  // registers, the two softmax warpgroups hold a 128-column row of S each.  Each role executes its
  // own setmaxnreg inside its branch (a dec / inc before a merge point makes ptxas compile the
  // merged code for the smaller count)
#if ATTN_SETMAXNREG
#define REG_DEC() asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(ATTN_REGS_PRODUCER))
#define REG_INC() asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(ATTN_REGS_SOFTMAX))
#else
#define REG_DEC() do { } while (0)
#define REG_INC() do { } while (0)
#endif

  if (warp == 0) {
    REG_DEC();
    if (lane == 0) {  // ===== TMA producer =====
      const int qrow = seg.q_start + q0;
      tc::mbar_arrive_expect_tx(&bar->q_full, (has_b ? 2 : 1) * Q_BYTES);
#pragma unroll
      for (int c = 0; c < C::NCH; ++c) {
        tc::tma_load_2d(sQ + c * CHUNK, &tmQ, &bar->q_full, h * D + 64 * c, qrow);
        if (has_b) tc::tma_load_2d(sQ + Q_BYTES + c * CHUNK, &tmQ, &bar->q_full, h * D + 64 * c, qrow + BQ);
      }
      for (int j = 0; j < nkv; ++j) {  // K ring
        const int s = j % KSTAGES;
        tc::mbar_wait(&bar->k_empty[s], ((j / KSTAGES) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&bar->k_full[s], KV_BYTES);
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
          tma_load_3d(sK + s * KV_BYTES + c * CHUNK, &tmKV, &bar->k_full[s], h * D + 64 * c, j * BKV, planeK);
      }
    }
  } else if (warp == 2) {
    REG_DEC();
    if (lane == 0) {  // ===== TMA producer, V ring =====
      for (int j = 0; j < nkv; ++j) {
        const int s = j % VSTAGES;
        tc::mbar_wait(&bar->v_empty[s], ((j / VSTAGES) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&bar->v_full[s], KV_BYTES);
#pragma unroll
        for (int c = 0; c < C::NCH; ++c)
          tma_load_3d(sV + s * KV_BYTES + c * CHUNK, &tmKV, &bar->v_full[s], h * D + 64 * c, j * BKV, planeK + 1);
      }
    }
  } else if (warp == 1) {
    REG_DEC();
    if (lane == 0) {  // ===== MMA issuer =====
      constexpr uint32_t idS = tc::idesc_bf16(BQ, BKV, 0);
      constexpr uint32_t idO = tc::idesc_bf16(BQ, D, 1);  // B = V is MN-major
      const int ntiles = has_b ? 2 : 1;
      tc::mbar_wait(&bar->q_full, 0);
      auto issue_S = [&](int t, int j) {
        const uint32_t q_addr = tc::smem_u32(sQ + t * Q_BYTES);
        const uint32_t k_addr = tc::smem_u32(sK + (j % KSTAGES) * KV_BYTES);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k >> 2) * CHUNK + (k & 3) * 32;
          tc::mma_bf16_ss(tmem + t * TS, tc::sdesc_sw128(q_addr + off, 16, 1024),
                          tc::sdesc_sw128(k_addr + off, 16, 1024), idS, k != 0);
        }
        tc::mma_commit(&bar->s_full[t]);
      };
      // P_t(j) lives in the upper 64 columns of the S_t region (bf16 pairs), so the lower half
      // of S_t(j+1) (keys 0..63 of the next tile) can be computed while softmax t still works on
      // S_t(j) (as soon as it has loaded it); only the upper half waits behind PV_t(j)
      constexpr uint32_t POFF = ATTN_SPLIT_S ? 64 : 0;
      auto issue_PV = [&](int t, int j) {
        TRACE(0, t, j);  // MMA warp starts waiting for P_t(j)
        tc::mbar_wait(&bar->p_full[t], j & 1);
        TRACE(1, t, j);  // P_t(j) ready
        tc::tc_fence_after();
        const uint32_t v_addr = tc::smem_u32(sV + (j % VSTAGES) * KV_BYTES);
#pragma unroll
        for (int k = 0; k < BKV / 16; ++k)
          tc::mma_bf16_ts(tmem + t * TS + 128, tmem + t * TS + POFF + k * 8,
                          tc::sdesc_sw128(v_addr + k * 2048, CHUNK, 1024), idO, (j | k) != 0);
      };
#if ATTN_SPLIT_S
      constexpr uint32_t idS64 = tc::idesc_bf16(BQ, 64, 0);
      auto issue_S_half = [&](int t, int j, int half) {  // keys [64 half, 64 half + 64) of tile j
        const uint32_t q_addr = tc::smem_u32(sQ + t * Q_BYTES);
        const uint32_t k_addr = tc::smem_u32(sK + (j % KSTAGES) * KV_BYTES) + half * 8192;
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k >> 2) * CHUNK + (k & 3) * 32;
          tc::mma_bf16_ss(tmem + t * TS + half * 64, tc::sdesc_sw128(q_addr + off, 16, 1024),
                          tc::sdesc_sw128(k_addr + off, 16, 1024), idS64, k != 0);
        }
      };
#endif
      tc::mbar_wait(&bar->k_full[0], 0);
      tc::tc_fence_after();
      for (int t = 0; t < ntiles; ++t) issue_S(t, 0);
      tc::mma_commit(&bar->k_empty[0]);
      for (int j = 0; j < nkv; ++j) {
        const bool more = j + 1 < nkv;
        tc::mbar_wait(&bar->v_full[j % VSTAGES], (j / VSTAGES) & 1);
        tc::tc_fence_after();
        for (int t = 0; t < ntiles; ++t) {
#if ATTN_SPLIT_S
          if (more) {
            if (t == 0) tc::mbar_wait(&bar->k_full[(j + 1) % KSTAGES], ((j + 1) / KSTAGES) & 1);
            tc::mbar_wait(&bar->s_used[t], j & 1);  // softmax t has S_t(j) in registers
            tc::tc_fence_after();
            issue_S_half(t, j + 1, 0);
          }
          issue_PV(t, j);
          if (more) {
            issue_S_half(t, j + 1, 1);
            tc::mma_commit(&bar->s_full[t]);
          } else {
            tc::mma_commit(&bar->o_done[t]);
          }
#else
          issue_PV(t, j);
          if (more) {
            if (t == 0) {
              tc::mbar_wait(&bar->k_full[(j + 1) % KSTAGES], ((j + 1) / KSTAGES) & 1);
              tc::tc_fence_after();
            }
            issue_S(t, j + 1);
          } else {
            tc::mma_commit(&bar->o_done[t]);
          }
#endif
        }
        tc::mma_commit(&bar->v_empty[j % VSTAGES]);
        if (more) tc::mma_commit(&bar->k_empty[(j + 1) % KSTAGES]);
      }
    }
  } else if (warp >= 4) {  // ===== softmax / correction / epilogue, tile t =====
    REG_INC();
    const int t = (warp - 4) >> 2;
    if (t == 0 || has_b) {
      const int quad = warp & 3;
      const int row = quad * 32 + lane;  // query row inside the tile == TMEM lane
      const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
      const uint32_t tS = tmem + t * TS + lane_off, tO = tS + 128;
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < nkv; ++j) {
        if (lane == 0 && quad == 0) TRACE(2, t, j);  // softmax starts waiting for S_t(j)
        tc::mbar_wait(&bar->s_full[t], j & 1);
        if (lane == 0 && quad == 0) TRACE(3, t, j);  // S_t(j) seen
        tc::tc_fence_after();
        uint32_t r[128];
        tc::tmem_ld32(tS + 0, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
        tc::tmem_ld32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
        tc::tmem_ld32(tS + 64, *reinterpret_cast<uint32_t(*)[32]>(&r[64]));
        tc::tmem_ld32(tS + 96, *reinterpret_cast<uint32_t(*)[32]>(&r[96]));
        tc::tmem_ld_wait();
#if ATTN_SPLIT_S
        tc::tc_fence_before();  // S_t(j) is in registers: the MMA warp may overwrite its lower half
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&bar->s_used[t]);
#endif
        const int valid = a.L - j * BKV;  // keys >= L are masked (ragged last tile only)
        // row max as 8 independent partial chains (latency, one warp per SMSP in this phase)
        float pm[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) pm[u] = -INFINITY;
        if (valid < BKV) {
#pragma unroll
          for (int i = 0; i < 128; ++i)
            if (i >= valid) r[i] = __float_as_uint(-INFINITY);
        }
#if ATTN_MAX3
#pragma unroll
        for (int i = 0; i < 128; i += 16)
#pragma unroll
          for (int u = 0; u < 8; ++u) pm[u] = fmax3(pm[u], __uint_as_float(r[i + u]), __uint_as_float(r[i + 8 + u]));
        const float mx = fmax3(fmax3(pm[0], pm[1], pm[2]), fmax3(pm[3], pm[4], pm[5]), fmaxf(pm[6], pm[7]));
#else
#pragma unroll
        for (int i = 0; i < 128; i += 8)
#pragma unroll
          for (int u = 0; u < 8; ++u) pm[u] = fmaxf(pm[u], __uint_as_float(r[i + u]));
        const float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])),
                               fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
#endif
        // scores in log2 units: s * scale * log2(e).  Keep the stale max unless it grew by
        // more than the threshold (per row).
        const float mxs = mx * scale_log2;
        const float m_use = (mxs > m + RESCALE_THRESHOLD) ? mxs : m;
        const float alpha = exp2f(m - m_use);  // 1 when kept, 0 on the first tile
        const float2 sc2 = make_float2(scale_log2, scale_log2);
        const float2 nm2 = make_float2(-m_use, -m_use);
        float2 acc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] = make_float2(0.f, 0.f);
        // P_t(j) goes back to TMEM in ATTN_ST_CHUNKS pieces, each stored as soon as its exps are
        // done, so the stores overlap the remaining exps
        constexpr int PCH = 64 / ATTN_ST_CHUNKS;  // packed bf16x2 words per chunk
#pragma unroll
        for (int c = 0; c < ATTN_ST_CHUNKS; ++c) {
#pragma unroll
          for (int i = c * PCH; i < (c + 1) * PCH; ++i) {  // in-place pack: r[i] <- bf16x2(p[2i], p[2i+1])
            const float2 x = __ffma2_rn(make_float2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1])), sc2, nm2);
            const bool poly = D == 64 ? POLY64_AT(i) : POLY_AT(i);
            const float2 pp = poly ? ex2_poly2(x) : make_float2(ex2_fast(x.x), ex2_fast(x.y));
            acc[i & 3] = __fadd2_rn(acc[i & 3], pp);
            r[i] = pack_bf16(pp.x, pp.y);
          }
          const uint32_t tP = tS + (ATTN_SPLIT_S ? 64 : 0);  // P_t(j): bf16 pairs, 64 columns
          if (PCH == 64) {
            tc::tmem_st32(tP + 0, &r[0]);
            tc::tmem_st32(tP + 32, &r[32]);
          } else if (PCH == 32) {
            tc::tmem_st32(tP + c * 32, &r[c * 32]);
          } else {
            tc::tmem_st16(tP + c * 16, *reinterpret_cast<const uint32_t(*)[16]>(&r[c * 16]));
          }
        }
        const float2 s01 = __fadd2_rn(acc[0], acc[1]), s23 = __fadd2_rn(acc[2], acc[3]);
        const float2 s4 = __fadd2_rn(s01, s23);
        const float sum = s4.x + s4.y;
        if (j > 0 && __any_sync(0xffffffffu, m_use > m)) {
#pragma unroll 1
          for (int c = 0; c < D; c += 32) {
            uint32_t o[32];
            tc::tmem_ld32(tO + c, o);
            tc::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tc::tmem_st32(tO + c, o);
          }
        }
        l = l * alpha + sum;
        m = m_use;
        tc::tmem_st_wait();
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&bar->p_full[t]);
        if (lane == 0 && quad == 0) TRACE(4, t, j);  // softmax done
      }
      // epilogue: O / l -> bf16 -> global
      tc::mbar_wait(&bar->o_done[t], 0);
      tc::tc_fence_after();
      const int qi = q0 + t * BQ + row;
      const float inv = 1.0f / l;
      bf16* out = reinterpret_cast<bf16*>(a.O) + (long long)(seg.q_start + qi) * a.ldo + h * D;
#pragma unroll 1
      for (int c = 0; c < D; c += 32) {
        uint32_t o[32];
        tc::tmem_ld32(tO + c, o);
        tc::tmem_ld_wait();
        if (qi < seg.q_len) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 v;
            v.x = pack_bf16(__uint_as_float(o[8 * q + 0]) * inv, __uint_as_float(o[8 * q + 1]) * inv);
            v.y = pack_bf16(__uint_as_float(o[8 * q + 2]) * inv, __uint_as_float(o[8 * q + 3]) * inv);
            v.z = pack_bf16(__uint_as_float(o[8 * q + 4]) * inv, __uint_as_float(o[8 * q + 5]) * inv);
            v.w = pack_bf16(__uint_as_float(o[8 * q + 6]) * inv, __uint_as_float(o[8 * q + 7]) * inv);
            *reinterpret_cast<uint4*>(out + c + 8 * q) = v;
          }
        }
      }
    }
  } else {
    REG_DEC();  // warp 3: idle
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<512>(tmem);
#ifdef IG_ATTN_TRACE
  if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) {
    __threadfence();
    for (int j = 0; j < 40 && j < nkv; ++j)
      for (int t = 0; t < 2; ++t)
        printf("TR %d %d %lld %lld %lld %lld %lld\n", t, j, g_trace[0][t][j], g_trace[1][t][j], g_trace[2][t][j],
               g_trace[3][t][j], g_trace[4][t][j]);
  }
#endif
}

PFN_cuTensorMapEncodeTiled_v12000 g_enc = nullptr;
std::once_flag g_once;

void init_attn() {
  std::call_once(g_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    g_enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    cudaFuncSetAttribute(attn_tc_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, AC<128>::SMEM_BYTES);
    cudaFuncSetAttribute(attn_tc_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, AC<64>::SMEM_BYTES);
  });
}
}  // namespace

void attn_tc_init() { init_attn(); }

bool attn_tc_supported(const AttnArgs& a) {
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const long long H = (long long)a.heads * a.head_dim;
  return (a.head_dim == 128 || a.head_dim == 64) && al16(a.Q) && al16(a.O) && al16(a.kv_arena) && (a.ldq % 8) == 0 &&
         (a.ldo % 8) == 0 && ((a.kv_off % ((long long)a.L * H)) == 0);
}

void launch_attn_tc(const AttnArgs& a, cudaStream_t st) {
  if (a.nseg <= 0 || a.max_qlen <= 0) return;
  init_attn();
  const long long H = (long long)a.heads * a.head_dim;
  CUtensorMap tq, tkv;
  // encoded maps cached per (pointer, shape) like the GEMM's (host enqueue cost)
  struct Ent { const void* p; long long x, y, z; CUtensorMap m; };
  thread_local std::vector<Ent> cache;
  auto lookup = [&](const void* p, long long x, long long y, long long z, CUtensorMap* out) {
    for (auto& e : cache)
      if (e.p == p && e.x == x && e.y == y && e.z == z) { *out = e.m; return true; }
    return false;
  };
  auto remember = [&](const void* p, long long x, long long y, long long z, const CUtensorMap& m) {
    if (cache.size() > 256) cache.clear();
    cache.push_back(Ent{p, x, y, z, m});
  };
  if (!lookup(a.Q, H, a.q_rows, a.ldq, &tq)) {
    cuuint64_t dims[2] = {(cuuint64_t)H, (cuuint64_t)a.q_rows};
    cuuint64_t strides[1] = {(cuuint64_t)(a.ldq * 2)};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    g_enc(&tq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(a.Q), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    remember(a.Q, H, a.q_rows, a.ldq, tq);
  }
  if (!lookup(a.kv_arena, H, a.L, -1, &tkv)) {
    // K/V arena as 3-D [planes][L][H]: plane p = K or V of one (slot, ring buffer); rows >= L
    // are out of bounds (zero fill) for the ragged last key tile.
    cuuint64_t dims[3] = {(cuuint64_t)H, (cuuint64_t)a.L, (cuuint64_t)(1u << 20)};
    cuuint64_t strides[2] = {(cuuint64_t)(H * 2), (cuuint64_t)(a.L * H * 2)};
    cuuint32_t box[3] = {64, 128, 1};
    cuuint32_t es[3] = {1, 1, 1};
    g_enc(&tkv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(a.kv_arena), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    remember(a.kv_arena, H, a.L, -1, tkv);
  }
  dim3 grid = a.n_pairs > 0 ? dim3(a.n_pairs, a.heads, 1)
                            : dim3((a.max_qlen + 2 * BQ - 1) / (2 * BQ), a.heads, a.nseg);
  const float scale_log2 = a.scale * 1.4426950408889634f;
  if (a.head_dim == 128) attn_tc_kernel<128><<<grid, NTHREADS, AC<128>::SMEM_BYTES, st>>>(tq, tkv, a, scale_log2);
  else attn_tc_kernel<64><<<grid, NTHREADS, AC<64>::SMEM_BYTES, st>>>(tq, tkv, a, scale_log2);
}

}  // namespace ig
