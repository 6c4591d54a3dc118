// k_attn_tc.cu — kernel (d): varlen flash attention on tcgen05 tensor cores (bf16, d = 128).
// Masked queries x merged full K/V ("Q ... of only the newly generated token
// along with the K and V matrices of all present tokens"): each ragged query segment of the
// packed continuous batch attends to its own request's positional K/V buffer of L rows.
//
// One CTA per (query tile of 128 rows, head, segment):
//   warp 0      TMA producer: Q tile once, then K/V tiles of 128 keys into a 2-stage ring
//   warp 1      TMEM allocator + single-thread MMA issuer:
//                 S_j = Q K_j^T   (SS, M=128 N=128 K=128, fp32 in TMEM, double-buffered)
//                 O  += P_j V_j   (SS, P from shared memory, V MN-major, fp32 O in TMEM)
//               S_{j+1} is issued before waiting for softmax j, so QK^T overlaps softmax.
//   warps 4..7  softmax, thread = query row (TMEM lane): row max / exp2 / row sum in fp32,
//               P (bf16) written to shared memory in the SW128 K-major layout; the O row is
//               rescaled in TMEM only when that row's running max grows — a per-row decision,
//               so a row's result never depends on its tile-mates (batch invariance).
// Keys >= L (ragged last tile) are zero-filled by TMA and masked to -inf.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <mutex>
#include "kernels.h"
#include "tc_common.cuh"

namespace ig {
namespace {

constexpr int BQ = 128, BKV = 128, D = 128;
constexpr int CHUNK = 128 * 64 * 2;             // one [128 rows x 64 cols] bf16 SW128 box
constexpr int Q_BYTES = 2 * CHUNK;              // 32 KB
constexpr int KV_BYTES = 2 * CHUNK;             // 32 KB each for K and V
constexpr int STAGES = 2;
constexpr int SMEM_BYTES = Q_BYTES + STAGES * 2 * KV_BYTES + 2 * CHUNK /*P*/ + 1024 + 256;
constexpr int NTHREADS = 256;

struct Bars {
  uint64_t q_full;
  uint64_t kv_full[STAGES], kv_empty[STAGES];
  uint64_t s_full[2], s_empty[2];
  uint64_t p_full, pv_done;
  uint32_t tmem;
};

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 p = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&p);
}

__global__ void __launch_bounds__(NTHREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKV,
                   const AttnArgs a, float scale_log2) {
  const AttnSeg seg = a.segs[blockIdx.z];
  const int h = blockIdx.y;
  const int q0 = blockIdx.x * BQ;
  if (q0 >= seg.q_len) return;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + Q_BYTES;                      // [STAGES][KV_BYTES]
  uint8_t* sV = sK + STAGES * KV_BYTES;            // [STAGES][KV_BYTES]
  uint8_t* sP = sV + STAGES * KV_BYTES;            // [2 chunks][128 rows][128 B]
  Bars* bar = reinterpret_cast<Bars*>(sP + 2 * CHUNK);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkv = (a.L + BKV - 1) / BKV;
  const long long H = (long long)a.heads * D;
  // plane index of this segment's K (and V = K + 1) in the 3-D K/V tensor map
  const long long plane_elems = (long long)a.L * H;
  const int planeK = (int)((seg.kv_base + a.kv_off) / plane_elems);

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch_desc(&tmQ);
    tc::tma_prefetch_desc(&tmKV);
    tc::mbar_init(&bar->q_full, 1);
    for (int s = 0; s < STAGES; ++s) { tc::mbar_init(&bar->kv_full[s], 1); tc::mbar_init(&bar->kv_empty[s], 1); }
    for (int s = 0; s < 2; ++s) { tc::mbar_init(&bar->s_full[s], 1); tc::mbar_init(&bar->s_empty[s], 4); }
    tc::mbar_init(&bar->p_full, 4);
    tc::mbar_init(&bar->pv_done, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<512>(&bar->tmem);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = bar->tmem;
  const uint32_t tS[2] = {tmem, tmem + 128};
  const uint32_t tO = tmem + 256;

  if (warp == 0) {
    if (lane == 0) {  // ===== TMA producer =====
      const int qrow = seg.q_start + q0;
      tc::mbar_arrive_expect_tx(&bar->q_full, Q_BYTES);
      tc::tma_load_2d(sQ, &tmQ, &bar->q_full, h * D, qrow);
      tc::tma_load_2d(sQ + CHUNK, &tmQ, &bar->q_full, h * D + 64, qrow);
      for (int j = 0; j < nkv; ++j) {
        const int s = j % STAGES;
        tc::mbar_wait(&bar->kv_empty[s], ((j / STAGES) & 1) ^ 1);
        tc::mbar_arrive_expect_tx(&bar->kv_full[s], 2 * KV_BYTES);
        uint8_t* k = sK + s * KV_BYTES;
        uint8_t* v = sV + s * KV_BYTES;
        const int kvrow = j * BKV;
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
            ::"r"(tc::smem_u32(k)), "l"(reinterpret_cast<uint64_t>(&tmKV)), "r"(tc::smem_u32(&bar->kv_full[s])),
            "r"(h * D), "r"(kvrow), "r"(planeK) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
            ::"r"(tc::smem_u32(k + CHUNK)), "l"(reinterpret_cast<uint64_t>(&tmKV)), "r"(tc::smem_u32(&bar->kv_full[s])),
            "r"(h * D + 64), "r"(kvrow), "r"(planeK) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
            ::"r"(tc::smem_u32(v)), "l"(reinterpret_cast<uint64_t>(&tmKV)), "r"(tc::smem_u32(&bar->kv_full[s])),
            "r"(h * D), "r"(kvrow), "r"(planeK + 1) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
            ::"r"(tc::smem_u32(v + CHUNK)), "l"(reinterpret_cast<uint64_t>(&tmKV)), "r"(tc::smem_u32(&bar->kv_full[s])),
            "r"(h * D + 64), "r"(kvrow), "r"(planeK + 1) : "memory");
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ===== MMA issuer =====
      constexpr uint32_t idS = tc::idesc_bf16(BQ, BKV, 0);
      constexpr uint32_t idO = tc::idesc_bf16(BQ, D, 1);  // B = V is MN-major
      const uint32_t q_addr = tc::smem_u32(sQ);
      const uint32_t p_addr = tc::smem_u32(sP);
      tc::mbar_wait(&bar->q_full, 0);
      auto issue_S = [&](int j) {
        const int s = j % STAGES, b = j & 1;
        tc::mbar_wait(&bar->kv_full[s], (j / STAGES) & 1);
        tc::mbar_wait(&bar->s_empty[b], ((j >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        const uint32_t k_addr = tc::smem_u32(sK + s * KV_BYTES);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k >> 2) * CHUNK + (k & 3) * 32;
          tc::mma_bf16_ss(tS[b], tc::sdesc_sw128(q_addr + off, 16, 1024), tc::sdesc_sw128(k_addr + off, 16, 1024),
                          idS, k != 0);
        }
        tc::mma_commit(&bar->s_full[b]);
      };
      auto issue_PV = [&](int j) {
        const int s = j % STAGES;
        tc::mbar_wait(&bar->p_full, j & 1);
        tc::tc_fence_after();
        const uint32_t v_addr = tc::smem_u32(sV + s * KV_BYTES);
#pragma unroll
        for (int k = 0; k < BKV / 16; ++k) {
          const uint32_t poff = (k >> 2) * CHUNK + (k & 3) * 32;
          tc::mma_bf16_ss(tO, tc::sdesc_sw128(p_addr + poff, 16, 1024),
                          tc::sdesc_sw128(v_addr + k * 2048, CHUNK, 1024), idO, (j | k) != 0);
        }
        tc::mma_commit(&bar->pv_done);
        tc::mma_commit(&bar->kv_empty[s]);
      };
      issue_S(0);
      for (int j = 1; j < nkv; ++j) {
        issue_S(j);
        issue_PV(j - 1);
      }
      issue_PV(nkv - 1);
    }
  } else if (warp >= 4) {  // ===== softmax / correction / epilogue =====
    const int quad = warp & 3;
    const int row = quad * 32 + lane;  // query row inside the tile == TMEM lane
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    float m = -INFINITY, l = 0.f;
    uint8_t* prow = sP + row * 128;
    const int swz = row & 7;
    for (int j = 0; j < nkv; ++j) {
      const int b = j & 1;
#ifdef IG_HANG_CHECK
      if (threadIdx.x == 128 && blockIdx.x == 0 && blockIdx.y == 0) printf("sm j=%d wait s_full\n", j);
#endif
      tc::mbar_wait(&bar->s_full[b], (j >> 1) & 1);
      tc::tc_fence_after();
      uint32_t r[128];
      tc::tmem_ld32(tS[b] + lane_off + 0, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
      tc::tmem_ld32(tS[b] + lane_off + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
      tc::tmem_ld32(tS[b] + lane_off + 64, *reinterpret_cast<uint32_t(*)[32]>(&r[64]));
      tc::tmem_ld32(tS[b] + lane_off + 96, *reinterpret_cast<uint32_t(*)[32]>(&r[96]));
      tc::tmem_ld_wait();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&bar->s_empty[b]);  // S buffer may be overwritten by S_{j+2}
      const int valid = a.L - j * BKV;                    // keys >= L are masked
      float mx = -INFINITY;
#pragma unroll
      for (int i = 0; i < 128; ++i) {
        float s = __uint_as_float(r[i]) * scale_log2;
        if (i >= valid) s = -INFINITY;
        r[i] = __float_as_uint(s);
        mx = fmaxf(mx, s);
      }
      const float m_new = fmaxf(m, mx);
      const float alpha = exp2f(m - m_new);  // 0 on the first tile
      float sum = 0.f;
      uint32_t pk[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        const float p0 = exp2f(__uint_as_float(r[2 * i]) - m_new);
        const float p1 = exp2f(__uint_as_float(r[2 * i + 1]) - m_new);
        sum += p0 + p1;
        pk[i] = pack_bf16(p0, p1);
      }
      l = l * alpha + sum;
      // P_j may only overwrite shared memory / O may only be rescaled once PV_{j-1} is done
#ifdef IG_HANG_CHECK
      if (threadIdx.x == 128 && blockIdx.x == 0 && blockIdx.y == 0) printf("sm j=%d m=%f mnew=%f l=%f wait pv\n", j, m, m_new, l);
#endif
      if (j > 0) {
        tc::mbar_wait(&bar->pv_done, (j - 1) & 1);
        tc::tc_fence_after();
      }
#ifdef IG_HANG_CHECK
      if (threadIdx.x == 128 && blockIdx.x == 0 && blockIdx.y == 0) printf("sm j=%d pv ok\n", j);
#endif
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int base = c * 32 + u * 4;
          uint4 v = make_uint4(pk[base], pk[base + 1], pk[base + 2], pk[base + 3]);
          *reinterpret_cast<uint4*>(prow + c * CHUNK + ((u ^ swz) << 4)) = v;
        }
      // Lazy correction of the O accumulator.  tcgen05.ld/st are warp-collective, so the warp
      // runs the pass if any of its rows needs it; rows whose max did not grow use alpha = 1
      // (an exact multiply), keeping each row's result independent of its tile-mates.
      if (j > 0 && __any_sync(0xffffffffu, m_new > m)) {
#pragma unroll 1
        for (int c = 0; c < D; c += 16) {
          uint32_t o[16];
          tc::tmem_ld16(tO + lane_off + c, o);
          tc::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tc::tmem_st16(tO + lane_off + c, o);
        }
        tc::tmem_st_wait();
      }
#ifdef IG_HANG_CHECK
      if (threadIdx.x == 128 && blockIdx.x == 0 && blockIdx.y == 0) printf("sm j=%d rescale done\n", j);
#endif
      m = m_new;
      tc::fence_proxy_async_smem();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&bar->p_full);
    }
    // epilogue: O / l -> bf16 -> global
    tc::mbar_wait(&bar->pv_done, (nkv - 1) & 1);
    tc::tc_fence_after();
    const int qi = q0 + row;
    const float inv = 1.0f / l;
    bf16* out = reinterpret_cast<bf16*>(a.O) + (long long)(seg.q_start + qi) * a.ldo + h * D;
#pragma unroll 1
    for (int c = 0; c < D; c += 32) {
      uint32_t o[32];
      tc::tmem_ld32(tO + lane_off + c, o);
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
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<512>(tmem);
}

PFN_cuTensorMapEncodeTiled_v12000 g_enc = nullptr;
std::once_flag g_once;

void init_attn() {
  std::call_once(g_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    g_enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  });
}
}  // namespace

bool attn_tc_supported(const AttnArgs& a) {
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const long long H = (long long)a.heads * a.head_dim;
  return a.head_dim == D && al16(a.Q) && al16(a.O) && al16(a.kv_arena) && (a.ldq % 8) == 0 &&
         (a.ldo % 8) == 0 && ((a.kv_off % ((long long)a.L * H)) == 0);
}

void launch_attn_tc(const AttnArgs& a, cudaStream_t st) {
  if (a.nseg <= 0 || a.max_qlen <= 0) return;
  init_attn();
  const long long H = (long long)a.heads * a.head_dim;
  // Q: 2-D [rows, H] with leading dimension ldq.  Rows: enough to cover every segment.
  CUtensorMap tq, tkv;
  {
    cuuint64_t dims[2] = {(cuuint64_t)H, (cuuint64_t)a.q_rows};
    cuuint64_t strides[1] = {(cuuint64_t)(a.ldq * 2)};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    g_enc(&tq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(a.Q), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  {
    // K/V arena as 3-D [planes][L][H]: plane p = K or V of one (slot, ring buffer); rows >= L
    // are out of bounds (zero fill) for the ragged last key tile.
    cuuint64_t dims[3] = {(cuuint64_t)H, (cuuint64_t)a.L, (cuuint64_t)(1u << 20)};
    cuuint64_t strides[2] = {(cuuint64_t)(H * 2), (cuuint64_t)(a.L * H * 2)};
    cuuint32_t box[3] = {64, 128, 1};
    cuuint32_t es[3] = {1, 1, 1};
    g_enc(&tkv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(a.kv_arena), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  dim3 grid((a.max_qlen + BQ - 1) / BQ, a.heads, a.nseg);
  const float scale_log2 = a.scale * 1.4426950408889634f;
  attn_tc_kernel<<<grid, NTHREADS, SMEM_BYTES, st>>>(tq, tkv, a, scale_log2);
}

}  // namespace ig
