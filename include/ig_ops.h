/* ig_ops.h — per-kernel entry points of libig, exported for parity tests and benchmarks.
 * Same conventions as ig.h (status codes, host-side validation before enqueue, void*
 * streams, caller-owned device buffers).  These call exactly the kernels ig_edit_step uses.
 */
#ifndef IG_OPS_H_
#define IG_OPS_H_
#include "ig.h"

#ifdef __cplusplus
extern "C" {
#endif

/* a6/a9/a10 — C[M,N] = epi(A[M,K] B[N,K]^T + bias[N]) (kernel c).  dtype IG_BF16 runs the
 * tcgen05/TMEM/TMA tensor-core GEMM (fp32 accumulate), IG_F32 the CUDA-core FFMA GEMM.
 * A, B, bias have the given dtype; C is fp32 when out_f32 else dtype.  epi: 0 = store,
 * 1 = GELU-tanh (C-AMB 6), 5 = GEGLU (IG_BF16 only; UNet feed-forward, C-AMB 32): B and bias
 * rows tile-interleaved — every group of 256 rows holds 128 "hidden" rows then their 128 "gate"
 * rows — and C[M, N/2] (bf16) = hidden * GELU_erf(gate), N % 256 == 0.  Row-major with leading
 * dimensions in elements.  IG_BF16 requires K % 8 == 0 (TMA zero-fills the K tail of the last
 * 64-wide slice), lda/ldb multiples of 8, ldc a multiple of 8 (bf16 C) or 4 (fp32 C), and
 * 16-byte aligned pointers (IG_EUNSUPPORTED otherwise); M and N are arbitrary. */
ig_status ig_op_gemm(int dtype, const void* A, long long lda, const void* B, long long ldb,
                     const void* bias, void* C, long long ldc, int M, int N, int K, int epi,
                     int out_f32, void* stream);

/* a9/a10 gated-residual epilogue variant (kernel c): X[M,N] (fp32, leading dimension ldx) +=
 * gate[N] (fp32, one request) * (A B^T + bias).  Same dtype rules as ig_op_gemm. */
ig_status ig_op_gemm_gated(int dtype, const void* A, long long lda, const void* B, long long ldb,
                           const void* bias, float* X, long long ldx, const float* gate, int M, int N,
                           int K, void* stream);

/* a8 — ragged attention (kernel d): for each segment s (host array
 * segs[s] = {q_start, q_len, kv_index}) and head j: O[q rows, j] = softmax(Q K^T * scale) V
 * where K = kv + kv_index*2*L*H ([L, H]) and V = K + L*H.  Q, O: [M, H] packed rows with
 * leading dimensions ldq/ldo (elements); H = heads*head_dim.  scale = 1/sqrt(head_dim). */
ig_status ig_op_attention(int dtype, const void* Q, long long ldq, void* O, long long ldo,
                          const void* kv, const int32_t* segs, int nseg, int L, int heads,
                          int head_dim, void* stream);

/* Test/bench I/O helper: cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault) on `stream`
 * followed by a stream synchronisation (any host/device combination, UVA pointers). */
ig_status ig_copy(void* dst, const void* src, size_t bytes, void* stream);

/* Whole-UNet 3x3 convolution (stride 1, zero padding 1; include/ig_unet.h): y [N*H*W][C_out] fp32
 * (NHWC rows) = conv(x) + bias, x_padded = bf16 [N][H+2][W+2][C_in] with zero borders, w = bf16
 * [C_out][9*C_in] (k = (ky*3 + kx)*C_in + c), bias bf16 [C_out] or NULL.  Implicit-GEMM tcgen05
 * kernel when C_in % 64 == 0, W in {8,16,32,64,128} or W % 128 == 0 and (H*W) % 128 == 0
 * (2-CTA 256x256 tiles when C_out % 256 == 0, else 128x128); otherwise im2col + the tcgen05
 * GEMM.  C_in % 8 == 0, C_out % 4 == 0 (IG_EINVAL / IG_EUNSUPPORTED otherwise). */
ig_status ig_op_conv3x3(const void* x_padded, int n_img, int H, int W, int cin, const void* w, const void* bias,
                        int cout, float* y, void* stream);

/* Per-request input staging for the host-buffer path (e.g. a request's text tokens at
 * admission): an SM-driven copy of `bytes` from PINNED host memory `src` (cudaHostAlloc /
 * cudaHostRegister'ed, device-mapped) into device memory `dst`, enqueued on `stream`.  Unlike a
 * cudaMemcpyAsync it does not queue on the copy engines behind the cache prefetch.  IG_EINVAL
 * if src is not pinned host memory. */
ig_status ig_stage_input(void* dst, const void* src, size_t bytes, void* stream);

/* Process-wide tuning knobs of libig (one struct instead of scattered switches).  Every field is
 * a 0/1 flag unless stated; defaults are the measured-best settings (profiles/).
 * The first ig_tuning_get / ig_tuning_set or libig launch seeds the struct from the environment
 * (the variable named per field, for A/B tools that cannot call the ABI); ig_tuning_set replaces
 * it.  Changes apply to launches enqueued after the call; CUDA graphs of steps captured earlier
 * keep the configuration they were captured with.  No field changes results except precise_gelu
 * (a different GELU approximation) — tile shapes and launch mechanics are batch-invariant. */
typedef struct ig_tuning {
  int pdl;              /* programmatic dependent launch of GEMMs after a kernel (1; env IG_NO_PDL) */
  int copy_thread;      /* copy-lane enqueues on their own host thread (1; env IG_NO_COPY_THREAD) */
  int load_dedupe;      /* host-tier load dedupe across requests on one (template, step) (1; IG_NO_DEDUPE) */
  int cross_kv_overlap; /* UNet: next block's cross-attention K/V GEMM on a side stream (1; IG_NO_XOVERLAP) */
  int gemm_two_cta;     /* 2-CTA 256x256 tiles for large GEMMs and convs (1; IG_GEMM_1CTA) */
  int gemm_small_tiles; /* 128x128 one-CTA tiles below SMs/4 2-CTA tiles (1; IG_GEMM_NO_SMALL) */
  int gemm_bn64;        /* 128x64 tiles below SMs/2 128x128 tiles (1; IG_GEMM_NO_BN64) */
  int conv_two_cta;     /* implicit conv: 2-CTA tiles for C_out >= 256 (1; IG_CONV_1CTA) */
  int precise_gelu;     /* debug: libm erf / tanh GELU instead of the MUFU forms (0; IG_PRECISE_GELU) */
  int op_repeat;        /* ig_op_attention: launches per call, benchmarking aid (1; IG_OP_REPEAT=n) */
  int txt_overlap;      /* double blocks: text-stream ops on a side stream, concurrent with the image
                           stream's, for steps of <= 4096 rows outside profiling (1; IG_NO_TXT_OVERLAP) */
} ig_tuning;
ig_status ig_tuning_get(ig_tuning* out);       /* IG_EINVAL if out is NULL */
ig_status ig_tuning_set(const ig_tuning* t);   /* IG_EINVAL if t is NULL or op_repeat < 1 */

#ifdef __cplusplus
}
#endif
#endif
