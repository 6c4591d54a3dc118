/* ig_unet.h — C ABI of libig's whole-UNet mask-aware step (BASELINE config 5, "SDXL-UNet-shaped
 * attention/ResBlock stack at 1024x1024 ... mask-ratio sweep 1-100% vs dense step").
 *
 * The paper: a UNet reshapes its latent (B, C, H, W) to (B, H x W, C) for its transformer
 * blocks, which are 82% of SDXL's compute (P:213 footnote); InstGenIE computes
 * them for the masked tokens only with the template's cached activations for the
 * rest (fig:transformer_alter / fig:transformer-Bottom).  The ResBlocks, resamplers,
 * GroupNorms and the in/out convolutions mix neighbouring pixels and run DENSE on the full
 * latent (implicit-GEMM tcgen05 convolutions).  Each Transformer2D (GroupNorm -> proj_in ->
 * BasicTransformerBlocks -> proj_out -> residual) runs on its level's masked tokens; its
 * blocks read the unmasked tokens' K/V from the cache (one ig_ctx attention stack per
 * Transformer2D, include/ig.h), and its output rows of the unmasked tokens are the template's
 * (cached per step, fp32).  Level masks: 2x2 any-pool of the latent mask (C-AMB 13).  Sampler:
 * eps = UNet(latent / sqrt(sigma^2 + 1), t = 1000 sigma), latent += (sigma' - sigma) eps on
 * the masked latent rows (C-AMB 34).  Architecture: public SDXL layout (C-AMB 34): oracle in
 * oracle/unet_full.py.  bf16 tensor-core arithmetic, fp32 hidden states.
 *
 * Conventions as in ig.h (ig_status, host-side validation before enqueue, caller-owned buffers).
 */
#ifndef IG_UNET_H_
#define IG_UNET_H_

#include "ig.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int lat_ch;        /* latent channels (4)                                                  */
  int grid;          /* latent H = W (128 at 1024^2); levels grid, grid/2, grid/4             */
  int ch[3];         /* channels per level (320, 640, 1280); multiples of 64                  */
  int depth[3];      /* transformer blocks per Transformer2D per level (0, 2, 10)             */
  int head_dim;      /* 64                                                                    */
  int ctx_len, ctx_dim;  /* cross-attention text context (77, 2048)                           */
  int n_res;         /* ResBlocks per down level (2); up levels n_res + 1                     */
  int gn_groups;     /* 32                                                                    */
  float gn_eps, t2d_gn_eps, ln_eps;  /* 1e-5, 1e-6, 1e-5                                      */
} ig_unet_desc;

typedef struct ig_unet ig_unet;              /* model: weights view, per-Transformer2D stacks,
                                                workspaces for max_batch requests             */
typedef struct ig_unet_cache ig_unet_cache;  /* one template: per Transformer2D the blocks' K/V
                                                (ig_cache) + the Transformer2D outputs, per step */
typedef struct ig_unet_mask ig_unet_mask;    /* one request's masks at the three levels        */

/* Length of the weight table (synth.unet_full_weight_table order: time MLP, conv_in, then the
 * down / mid / up parts in execution order — each ResBlock gn1, conv1, temb, gn2, conv2
 * (+ skip), each Transformer2D gn, proj_in, blocks (17 tensors each, ig.h UNet block order),
 * proj_out, each resampler conv — then out.gn and conv_out).  Convolutions [C_out][9*C_in]
 * with k = (ky*3 + kx)*C_in + c; all tensors bf16. */
int ig_unet_weight_count(const ig_unet_desc* desc);

/* weights: device pointers in table order (caller-owned).  max_batch requests per step;
 * prefetch_depth: the Transformer2D stacks' copy-lane ring depth.  IG_EINVAL /
 * IG_EUNSUPPORTED on bad shapes (channels not multiples of 64, grid not divisible by 4). */
ig_status ig_unet_create(const ig_unet_desc* desc, const void* const* weights, int n_weights, int device,
                         int max_batch, int prefetch_depth, ig_unet** out);
void ig_unet_destroy(ig_unet* u);

/* Masks at admission: mask = host uint8 [grid*grid] (nonzero = masked latent token); the
 * level-1/2 masks are its 2x2 any-pools.  Enqueued on `stream` (no device sync). */
ig_status ig_unet_mask_build(ig_unet* u, const uint8_t* mask, void* stream, ig_unet_mask** out, int* n_masked);
void ig_unet_mask_free(ig_unet_mask* m);

/* Template pass: n_steps dense steps from `latent` (dev [grid*grid][lat_ch] fp32, updated in
 * place along the trajectory) recording every Transformer2D's block K/V and outputs into a new
 * cache in `tier` (IG_CACHE_HOST pinned / IG_CACHE_DEVICE HBM).  ctx: dev [ctx_len][ctx_dim]
 * bf16; cond: dev [4*ch[0]] fp32 added to the timestep embedding, or NULL.  sigmas: host
 * [n_steps + 1].  Synchronises `stream`. */
ig_status ig_unet_template(ig_unet* u, float* latent, const void* ctx, const float* cond, const float* sigmas,
                           int n_steps, int tier, void* stream, ig_unet_cache** out);
void ig_unet_cache_free(ig_unet_cache* c);

typedef struct {
  float* latent;                /* dev [grid*grid][lat_ch] fp32; masked rows updated          */
  const ig_unet_mask* mask;
  const ig_unet_cache* cache;   /* may be NULL only for an all-ones mask                       */
  int step;                     /* index into the cache's schedule                             */
  float sigma, sigma_next;
  const void* ctx;              /* dev [ctx_len][ctx_dim] bf16                                 */
  const float* cond;            /* dev [4*ch[0]] fp32 or NULL                                  */
} ig_unet_req;

/* One mask-aware denoising step for a batch of n <= max_batch requests (dense parts batched
 * over the requests; each Transformer2D on the masked rows of every request).  Requests with
 * n_m == 0 are skipped (latent bit-identical).  Enqueues on `stream`.
 * Errors: IG_EINVAL, IG_ECACHE_MISS, IG_ECACHE_INCOMPAT, IG_ENOMEM, IG_ECUDA. */
ig_status ig_unet_step(ig_unet* u, const ig_unet_req* reqs, int n, void* stream);

/* Counters of the last ig_unet_step (kernel launches of the dense parts + every stack's). */
ig_status ig_unet_last_stats(const ig_unet* u, ig_stats* out);

#ifdef __cplusplus
}
#endif
#endif /* IG_UNET_H_ */
