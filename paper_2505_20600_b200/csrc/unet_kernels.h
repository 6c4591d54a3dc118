// unet_kernels.h — launchers of the whole-UNet step's dense-part kernels (k_conv.cu; internal).
#pragma once
#include "kernels.h"

namespace ig {

struct UReq {            // per request of a UNet step (device descriptor)
  float* latent;         // [P0][lat_ch] fp32 (caller's)
  const float* cond;     // [temb_dim] fp32 or null
  float sigma, dsig;     // t = 1000 sigma; Euler step sigma' - sigma
  float c_in;            // input scaling 1 / sqrt(sigma^2 + 1)
  int pad;
};
struct URows {           // a request's row list at one level
  const int32_t* idx;    // token indices (ascending), or null = all tokens 0..n-1
  int n;                 // number of rows
  int row0;              // first packed row
  const float* y;        // t2d_out unmasked list: the cache plane [P][C] of this Transformer2D
};

void launch_gn_stats(const float* x1, int C1, const float* x2, int C2, int N, int P, int G, float eps,
                     float2* partial, float2* stats, cudaStream_t st);
// coef: scratch [N][C1 + C2] float2 (per image and channel GroupNorm affine)
void launch_gn_apply_padded(const float* x1, int C1, const float* x2, int C2, const float2* stats, const bf16* gamma,
                            const bf16* beta, int G, int do_silu, int N, int H, int W, bf16* dst, float2* coef,
                            cudaStream_t st);
void launch_upsample_padded(const float* x, int C, int N, int H, int W, bf16* dst, cudaStream_t st);
void launch_im2col(const float* x, int C, int N, int H, int W, int stride, const float* scale, int Kp, bf16* dst,
                   cudaStream_t st);
void launch_im2col_padded(const bf16* pad, int C, int N, int H, int W, int Kp, bf16* dst, cudaStream_t st);
void launch_gather_latents(const UReq* rq, int n, int P, int C, float* dst, cudaStream_t st);
void launch_unet_sinusoid(const UReq* rq, int n, int dim, float* out, cudaStream_t st);
void launch_temb_finish(const UReq* rq, int n, int E, float* v, bf16* out, cudaStream_t st);
void launch_silu_inplace(float* x, long long n, cudaStream_t st);
void launch_t2d_in_rows(const URows* rl, int n, int max_rows, const float* x, int P, int C, const float2* stats,
                        const bf16* gamma, const bf16* beta, int G, bf16* dst, cudaStream_t st);
void launch_rows_move(const URows* rl, int n, int max_rows, float* T, int P, int C, const float* src, bf16* dstp,
                      int to_packed, cudaStream_t st);
void launch_t2d_out(const URows* rl, const URows* rlu, int n, int max_rows, const float* x, const float* po, int P, int C,
                    float* out, cudaStream_t st);
void launch_unet_euler(const UReq* rq, const URows* rl, int n, int max_rows, int P, int C, const float* eps,
                       cudaStream_t st);
void launch_cat_bf16(const float* x1, int C1, const float* x2, int C2, long long rows, bf16* dst, cudaStream_t st);

}  // namespace ig
