// kernels.h — host-side launchers of libig's CUDA kernels (internal; not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "common.cuh"

namespace ig {

// ---- a1 index build (k_rows.cu) --------------------------------------------------------
void launch_mask_index(const uint8_t* mask, int L, int32_t* idx_m, int32_t* idx_u,
                       int32_t* n_m_dev, cudaStream_t st);

// ---- a2/a4 batch assembly + entry gather (k_rows.cu) -------------------------------------
struct ReqDev {
  int slot, n_m, txt_row0, img_row0;  // packed-row offsets of this request's segments
  const int32_t* idx_m;
  const int32_t* idx_u;
  float* latent;
  const void* txt;
  const float* cond;
  float sigma, dsig;                  // dsig = sigma_next - sigma
  int has_cache;
  int n_ui;                           // unmasked rows included (Algorithm-1 dense prefix)
  int uimg_row0;                      // packed row of the first included unmasked row
  int pad;
  const float* tlatent;               // template input latent of this step [L_img, C]
};
// Fills row_info[M] and gathers: X[txt rows] = txt (fp32), Ain[img rows - M_txt] = latent
// rows at idx_m (as T).  M_txt = n * L_txt.
// Rows [M, M_full) are the included unmasked image rows (dense prefix): latent rows of the
// template's input latent at idx_u.
// img_to_x (UNet models, C == H): the masked image rows are copied into X (fp32, exact)
// instead of Ain.
template <typename T>
void launch_build_rows(const ReqDev* reqs, int n, int L_txt, int C, int H, int M_txt, int M,
                       RowInfo* row_info, float* X, T* Ain, cudaStream_t st, int M_full = -1,
                       int img_to_x = 0);
// UNet exit: latent_req[idx_m[j]][:] = X[img_row][:] (fp32 copy of the stack's output rows)
void launch_scatter_rows(const ReqDev* reqs, int M, const RowInfo* ri, int H, const float* X, cudaStream_t st);
// UNet cross-attention context: dst[q * Lc + j][:] = reqs[q].txt[j][:] (T, width Dc)
template <typename T>
void launch_pack_ctx(const ReqDev* reqs, int n, int Lc, int Dc, T* dst, cudaStream_t st);
// GEGLU on an unfused projection u [M, 2F] (ld ldu): out[r][j] = u[r][j] * gelu_erf(u[r][F + j])
template <typename T>
void launch_geglu(const T* u, long long ldu, int M, int F, T* out, long long ldo, cudaStream_t st);
// EPI_GEGLU weight layout: dst row (256 t + i) = src row (128 t + i) for i < 128 (hidden) and
// src row (F + 128 t + i - 128) otherwise (gate); rows of K elements (bf16); F % 128 == 0
void launch_permute_geglu_rows(const bf16* src, bf16* dst, int F, int K, cudaStream_t st);

// ---- a3 conditioning (k_norm.cu) --------------------------------------------------------
// temb[r][0:256] = [cos(1000 sigma_r f_k) | sin(...)], computed in double, stored as float.
void launch_timestep_embed(const ReqDev* reqs, int n, float* temb, cudaStream_t st);

struct GemvProb {
  const void* W;      // [N, K] row-major (T)
  const void* b;      // [N] (T) or null
  const float* x;     // [n, K] fp32 input rows (already activated)
  float* y;           // [n, ldy] fp32 output
  const float* addv;  // optional [n, ldadd] added after bias (cond_vec)
  int N, K, ldx, ldy, ldadd, act_out;  // act_out: 0 none, 1 silu
  int row_group0;     // prefix of row groups (filled by the launcher)
};
template <typename T>
void launch_gemv(const GemvProb* probs_dev, int nprob, int total_groups, int n, int maxK,
                 cudaStream_t st);
// y = silu(x) elementwise (fp32), n*H elements; optionally also a bf16 copy (GEMM operand)
void launch_silu(const float* x, float* y, long long count, cudaStream_t st, bf16* yb = nullptr);
// vec[r] += addv per request pointer (cond vectors live in caller buffers)
void launch_add_cond(const ReqDev* reqs, int n, int H, float* vec, cudaStream_t st);

// ---- a5 LN + modulate (k_norm.cu) -------------------------------------------------------
// h[r] = LN(X[r]) * (1 + mod[req][scale_off + c]) + mod[req][shift_off + c], rows [r0, r1)
template <typename T>
void launch_ln_mod(const float* X, int H, int r0, int r1, const RowInfo* ri, const float* mod,
                   int mod_ld, int shift_off, int scale_off, float eps, T* h, int ldh,
                   cudaStream_t st);

// ---- a6 epilogue: QK-norm, RoPE, Q pack, positional K/V merge (k_rows.cu) ---------------
struct QkvPost {
  const void* qkv;  int ld_qkv;     // [M, >=3H] rows r0..r1 (T)
  void* Q;                          // [M, H] packed (T)
  void* kv_arena;                   // ring arena (T)
  long long slot_stride, buf_off;   // elements
  long long L, H;                   // merged length, hidden
  const void* qg; const void* kg;   // [d] gains (T) or null
  const float2* rope_tab;           // [d/2 pairs][max_pos] (cos, sin), or null
  int rope_maxpos, ax1_pair, ax2_pair;  // pair index where axis 1 / axis 2 start
  int heads, head_dim, grid_w, qk_norm, rope;
  int r0, r1;
};
template <typename T>
void launch_qkv_post(const QkvPost& p, const RowInfo* ri, cudaStream_t st);

// ---- a7 compacted cache gather (zero-copy, copy lane) (k_rows.cu) -----------------------
// for each of n requests with cache: rows idx_u of src K and V (host-mapped or device)
// -> ring rows L_txt + idx_u.
struct KvGatherReq {
  const void* srcK; const void* srcV;  // [L_img, H] (compute dtype, or e4m3 bytes for q8)
  const int32_t* idx_u; int n_u;
  void* dstK; void* dstV;              // [L, H] positional ring buffer
  const float* sclK; const float* sclV;  // q8 only: [L_img, heads] dequantization scales
};
// FP8 (e4m3) K/V cache: per (token, head) scale = amax / 448, q = e4m3_rn(x / scale)
// (saturating), x' = bf16(q * scale).  Quantize rows [0, rows) of src (bf16 [rows, H]) to
// dst (u8 [rows, H]) + scl ([rows, heads]); one warp per (row, K|V plane).
void launch_kv_quant(const bf16* srcK, const bf16* srcV, long long rows, int H, int heads, uint8_t* dstK,
                     uint8_t* dstV, float* sclK, float* sclV, cudaStream_t st);
// gather + dequantize unmasked rows of an e4m3 source into the bf16 ring buffer
void launch_kv_gather_q8(const KvGatherReq* reqs_dev, int n, int max_nu, int L_txt, int H, int heads,
                         cudaStream_t st);
void launch_kv_gather(const KvGatherReq* reqs_dev, int n, int max_nu, int L_txt, int H,
                      int elem_bytes, cudaStream_t st);

// dst[0, n) = src[0, n) by SM loads (src may be mapped pinned host memory), 16-byte vectors
void launch_copy_bytes(void* dst, const void* src, size_t n, cudaStream_t st);
// debug / fault injection (ig_debug_set): a one-thread spin of `ns` nanoseconds on a stream,
// and +add on the K and V rows of the token idx_u[0] of one positional K/V buffer
void launch_spin(unsigned long long ns, cudaStream_t st);
void launch_corrupt_row(void* plane_k, long long vplane_elems, const int32_t* idx_u, int Lt, int H, int es,
                        float add, cudaStream_t st);

// ---- Y variant (k_rows.cu) ------------------------------------------------------
// LN-modulation of rows [r0, r1) read from the staged Y rows (V plane, position ri[r].kvpos of
// slot ri[r].slot) instead of the fp32 residual (exact widening: same bits as via the residual)
template <typename T>
void launch_ln_mod_staged(const void* arena, long long slot_stride, long long buf_off, long long L, int H, int r0,
                          int r1, const RowInfo* ri, const float* mod, int mod_ld, int shift_off, int scale_off,
                          float eps, T* h, int ldh, cudaStream_t st);
// dst[i] = T(src[i]), n a multiple of 4
template <typename T>
void launch_rows_to(const float* src, void* dst, long long n, cudaStream_t st);

// ---- load deduplication (k_rows.cu): requests on the same (template, step) ------
// Member e of a dedupe group reuses the rows its source request (slot0) already loaded: for
// every unmasked token of the member that is also unmasked in the source (bits0[tok] == 0),
// copy the staged K and V rows (V only for Y blocks) of ring buffer buf_off from slot0 to slot.
struct DedupeEnt {
  const int32_t* idx_u; int n_u;
  const uint8_t* bits0;  // source request's mask bitmap (1 = masked)
  int slot0, slot;
  int v_only;            // per block, from the entry's own cache: 1 = Y block (V landing plane only)
  int skip;              // per block: 1 = nothing staged for this entry (Y block inside the prefix)
};
constexpr int MAX_DEDUPE = 16;
struct DedupeArgs {
  DedupeEnt e[MAX_DEDUPE];
  int n, max_nu;
  void* arena; long long slot_stride, buf_off, L;
  int Lt, H, es;
};
void launch_kv_dedupe(const DedupeArgs& a, cudaStream_t st);

// ---- a11 exit: Euler scatter (k_rows.cu) ------------------------------------------------
// latent_req[idx_m[j]][c] += dsig_req * v[img_row][c]
void launch_scatter_euler(const ReqDev* reqs, int n, int M_img, const RowInfo* ri, int M_txt,
                          int C, const float* v, cudaStream_t st);

// ---- GEMM (k_gemm_simt.cu / k_gemm_tc.cu) -----------------------------------------------
enum Epi : int {
  EPI_STORE = 0,      // C = acc + b (TOut)
  EPI_GELU = 1,       // C = gelu_tanh(acc + b) (TOut)
  EPI_GATED_RES = 2,  // X[r, c] += gate[req(r)][c] * (acc + b)  (C is fp32 X)
  EPI_POS = 3,        // X[r, c] = acc + b + pos[tok(r)][c]      (C is fp32 X)
  EPI_QKV = 4,        // q,k: per-head RMSNorm + RoPE; q -> packed Q, k,v -> positional K/V
  EPI_GEGLU = 5,      // tcgen05 only, B/bias rows tile-interleaved (permute_geglu_rows): every
                      // 256-column tile holds 128 hidden columns then their 128 gate columns;
                      // C[r, n0/2 + j] = (acc_j + b_j) * gelu_erf(acc_{128+j} + b_{128+j}) (TOut)
  EPI_ADDRES = 6,     // C[r, c] = acc + b + res[r, c]  (C and res fp32, leading dimension ldc)
};
// Extra arguments of the fused QKV epilogue (a6: norm, RoPE and the positional merge done
// on the fp32 accumulators, one bf16 rounding per output).
struct QkvEpi {
  void* Q;                          // [M, H] packed (bf16)
  void* kv_arena;                   // ring arena (bf16)
  long long slot_stride, buf_off;   // elements
  long long L, H;
  const void* qg; const void* kg;   // [d] gains (bf16) or null
  const float2* rope_tab;           // [d/2][rope_maxpos] (cos, sin) or null
  int rope_maxpos, ax1_pair, ax2_pair;
  int head_dim, grid_w, qk_norm, rope;
  int col_base;                     // first output column's offset in [q|k|v] (H: K/V only)
};
struct GemmArgs {
  const void* A; long long lda;   // [M, K] row-major
  const void* B; long long ldb;   // [N, K] row-major (weights [out, in])
  const void* bias;               // [N] (same dtype as B) or null
  void* C; long long ldc;         // output (TOut) or fp32 residual
  int M, N, K;
  int epi;
  const float* gate; long long gate_ld;  // EPI_GATED_RES: mod + gate offset, row stride
  const RowInfo* ri;                     // row metadata (rows are A-rows offset by ri_off)
  int ri_off;
  const void* pos; long long pos_ld;     // EPI_POS table (T)
  int out_f32;                           // EPI_STORE/GELU: 1 => C is fp32
  int precise_gelu;                      // 1 => tanhf instead of MUFU tanh.approx (debug)
  QkvEpi qkv;                            // EPI_QKV only
  int pos_div;                           // EPI_POS: > 0 => table row (ri_off + row) / pos_div
                                         // (a per-image vector, e.g. a ResBlock's timestep term)
  const float* res;                      // EPI_ADDRES residual source
  int conv_H, conv_W, conv_cin;          // implicit 3x3 conv (launch_conv3x3_tc), else 0
  int pdl;                               // 1: programmatic dependent launch (the prologue — barrier
                                         // init, TMEM alloc, descriptor prefetch — overlaps the
                                         // previous kernel's tail; griddepcontrol.wait before any
                                         // global read); only right after another kernel
};
template <typename T>
void launch_gemm_simt(const GemmArgs& g, cudaStream_t st);
// tcgen05/TMEM/TMA bf16 GEMM (returns false if the shape is unsupported)
bool gemm_tc_supported(const GemmArgs& g);
void launch_gemm_tc(const GemmArgs& g, cudaStream_t st);
// Implicit-GEMM 3x3 convolution (stride 1, zero padding 1) on tcgen05: output pixels m of
// N images [H, W] (NHWC rows, M = N*H*W) x C_out = sum over the 9 taps and C_in of the
// zero-PADDED input A [N][H+2][W+2][C_in] (bf16) times B [C_out][9*C_in] (k = tap*C_in + c).
// The A tile of 128 output pixels at tap (dy, dx) is 128/W contiguous runs of the padded
// buffer, each one TMA box.  Needs C_in % 64 == 0, W in {8,16,32,64,128} or W % 128 == 0,
// (H*W) % 128 == 0 (conv3x3_tc_supported).  g.A = padded buffer, g.K = 9*C_in.
bool conv3x3_tc_supported(int H, int W, int cin);
void launch_conv3x3_tc(const GemmArgs& g, cudaStream_t st);

// ---- a8 attention (k_attn_simt.cu / k_attn_tc.cu) ---------------------------------------
struct AttnArgs {
  const void* Q; long long ldq;   // packed [M, H]
  void* O; long long ldo;         // packed [M, H] (may alias a column block of a wider buf)
  const void* kv_arena; long long kv_off;  // K at kv_base + kv_off, V at + L*H
  const AttnSeg* segs; int nseg; int max_qlen;
  int n_pairs;                    // sum over segments of ceil(q_len / 256): the tcgen05 grid's x
                                  // (0: the kernel falls back to max_qlen x nseg with idle CTAs)
  int q_rows;                     // rows of Q / O (bounds for the TMA tensor map)
  int L, heads, head_dim;
  float scale;                    // 1/sqrt(d)
};
template <typename T>
void launch_attn_simt(const AttnArgs& a, cudaStream_t st);
bool attn_tc_supported(const AttnArgs& a);
// one-time driver setup (function attributes, entry points) outside any stream capture
void attn_tc_init();
void gemm_tc_init();
void launch_attn_tc(const AttnArgs& a, cudaStream_t st);

}  // namespace ig
