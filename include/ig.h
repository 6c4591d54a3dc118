/* ig.h — C ABI of libig, the B200-native mask-aware denoising step of InstGenIE
 * (arXiv 2505.20600), K/V-caching variant (fig:transformer_alter).
 *
 * Citations: P:n = PAPER.md line n; S:n = SPEC.md line n; C-AMB k / §8(x) = the numbered
 * readings in DESIGN.md (taken from SURVEY.md §8(c)).
 *
 * Conventions for every entry point
 *  - Every call returns ig_status; IG_OK == 0.  No C++ exception crosses the ABI.
 *    ig_last_error() returns a thread-local message for the last non-OK status.
 *  - All argument, shape and compatibility checks run on the host BEFORE anything is
 *    enqueued: a non-OK status means nothing was enqueued (no partial enqueue).
 *  - "dev" pointers are CUDA device pointers on the context's device, "host" pointers are
 *    host memory.  `stream` arguments are cudaStream_t passed as void* (NULL = the legacy
 *    default stream).  Calls return after enqueue unless documented otherwise.
 *  - Ownership: the caller owns every buffer it passes in (weights, latents, masks, text,
 *    cond vectors, streams) and must keep them alive until the enqueued work completes.
 *    The library owns ig_ctx workspaces, per-slot K/V staging rings, ig_mask index lists
 *    and ig_cache storage (pinned host or device memory), freed by the *_free/_destroy calls.
 *  - One host thread per ig_ctx.  Contexts on different devices are independent.
 */
#ifndef IG_H_
#define IG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  IG_OK = 0,
  IG_EINVAL = 1,          /* invalid argument / shape mismatch        */
  IG_ECACHE_INCOMPAT = 2, /* cache built for another model/schedule, or step out of range */
  IG_ECACHE_MISS = 3,     /* 0 < n_m < L_img but no cache supplied                 */
  IG_ENUMERIC = 4,        /* non-finite output (debug checks only)                  */
  IG_ENOMEM = 5,          /* allocation failed or a step exceeds max_batch / max_rows      */
  IG_ECUDA = 6,           /* CUDA runtime/driver error (message has cudaGetErrorString)    */
  IG_EUNSUPPORTED = 7     /* shape the kernels do not support (see ig_ctx_create)          */
} ig_status;

typedef enum { IG_F32 = 0, IG_BF16 = 1 } ig_dtype;

/* Model shape (Flux-/SD3-shaped DiT; the paper's X in R^{B x L x H}).
 * L_img = grid_h*grid_w image tokens (latent (B,C,H,W) reshaped to (B, H*W, C)),
 * L = txt_len + L_img.  Validated by ig_ctx_create.
 * Constraints: hidden = heads*head_dim; head_dim in {16, 64, 128}; hidden % 64 == 0;
 * mlp_hidden % 64 == 0; lat_ch % 4 == 0; rope_axes sum to head_dim when rope != 0. */
typedef struct {
  int n_double, n_single;   /* double-stream (img/txt weights) and single-stream blocks */
  int hidden, heads, head_dim, mlp_hidden;
  int lat_ch, grid_h, grid_w, txt_len;
  int qk_norm;              /* per-head RMSNorm on q,k with gains (C-AMB 6)              */
  int rope;                 /* 3-axis RoPE at ORIGINAL token positions (C-AMB 7)         */
  int rope_axes[3];
  float rope_theta, ln_eps;
  int pos_embed_2d;         /* SD3: add pos_embed[token] at img_in                       */
  int context_pre_only_last;/* SD3: last double block's text stream only feeds K/V      */
  ig_dtype dtype;           /* IG_F32 = parity mode (fp32 SIMT), IG_BF16 = perf mode    */
  /* SDXL-UNet attention stack (BASELINE config 5; "a latent of shape
   * (B, C, H, W) is reshaped to (B, H x W, C) to pass through transformer blocks"): n_unet > 0
   * selects a model of n_unet BasicTransformerBlocks (C-AMB 31-33): x += SelfAttn(LN1(x)),
   * x += CrossAttn(LN2(x), context [ctx_len, ctx_dim]), x += GEGLU-FF(LN3(x)); LayerNorms with
   * affine (eps = ln_eps), no conditioning, no text rows.  Requires n_double = n_single = 0,
   * txt_len = 0, qk_norm = rope = pos_embed_2d = 0, lat_ch = hidden (the request's "latent"
   * is the level's hidden state [L_img, hidden] fp32; a step runs the stack on its masked rows
   * and writes the block stack's output rows back in place), mlp_hidden = GEGLU inner width. */
  int n_unet, ctx_len, ctx_dim;
} ig_model_desc;

/* UNet weight table (n_unet > 0), per block i:
 *   ln1.g [H], ln1.b [H], attn1.qkv.w [3H,H] (to_q|to_k|to_v, no bias), attn1.out.w [H,H],
 *   attn1.out.b, ln2.g, ln2.b, attn2.q.w [H,H] (no bias), attn2.kv.w [2H,ctx_dim] (to_k|to_v,
 *   no bias), attn2.out.w [H,H], attn2.out.b, ln3.g, ln3.b, ff.geglu.w [2F,H] ([hidden|gate]
 *   rows), ff.geglu.b [2F], ff.out.w [H,F], ff.out.b — 17 entries per block.
 *
 * Weight table (device pointers, caller-owned, dtype = desc.dtype except where noted),
 * in this fixed order; matrices are [out, in] row-major (nn.Linear), each followed by its
 * bias [out]:
 *   img_in.w [H,C], img_in.b, t_mlp1.w [H,256], t_mlp1.b, t_mlp2.w [H,H], t_mlp2.b,
 *   final_mod.w [2H,H], final_mod.b, proj_out.w [C,H], proj_out.b,
 *   (pos_embed_2d) pos_embed [L_img,H],
 *   for each double block i, for s in (img, txt):
 *       mod.w [6H,H] (2H for a context-pre-only text stream), mod.b, qkv.w [3H,H], qkv.b,
 *       (qk_norm) q_norm_g [d], k_norm_g [d],
 *       (unless context-pre-only) proj.w [H,H], proj.b, fc1.w [F,H], fc1.b, fc2.w [H,F], fc2.b
 *   for each single block i:
 *       mod.w [3H,H], mod.b, lin1.w [3H+F,H], lin1.b, (qk_norm) q_norm_g, k_norm_g,
 *       lin2.w [H,H+F], lin2.b
 * Modulation chunk order: double (shift1, scale1, gate1, shift2, scale2, gate2); single
 * (shift, scale, gate); final and context-pre-only (scale, shift).  ig_weight_count()
 * returns the table length for a descriptor. */
int ig_weight_count(const ig_model_desc* desc);

typedef struct {
  int max_batch;       /* continuous-batching slots (default 8)                    */
  int max_rows;        /* max packed query rows per step, sum_r (L_txt + n_m,r) (default  */
                       /* max_batch * L)                                                  */
  int prefetch_depth;  /* D: layers the copy lane runs ahead of compute (default 2)       */
  int copy_mode;       /* 0 = full-L per-layer cudaMemcpyAsync (all L_img rows),          */
                       /* 1 = compacted: only unmasked rows — host-tier caches by the copy */
                       /*     engines, one cudaMemcpyAsync / cudaMemcpy2DAsync per strided */
                       /*     group of unmasked runs (a group may also cover a few masked  */
                       /*     rows; the step then waits for the copy before the fresh K/V  */
                       /*     merge); HBM-tier caches via the SM gather                    */
                       /* 2 = compacted: zero-copy SM gather kernel on the copy stream     */
  int debug_checks;    /* 1 = check the latent for non-finite values after each step     */
  int cache_fp8;       /* 1 = caches created by this ctx store K/V as e4m3 with a fp32   */
                       /*     scale per (token, head): scale = amax/448, x' = bf16(q*scale)*/
                       /*     (halves host-link bytes; bf16 mode only)          */
  int cache_y;         /* 1 = caches created by this ctx hold Y, the template's block     */
                       /*     OUTPUT rows of the image tokens [steps][blocks][L_img][H]    */
                       /*     (fig:transformer-Bottom): half the     */
                       /*     bytes of K/V; a step recomputes the unmasked tokens' K/V     */
                       /*     from them (LN-mod + K/V projection).  With cache_fp8 every   */
                       /*     plane (K, V, Y) is e4m3 + per (token, head) scales, scale     */
                       /*     planes in the same plane order after all data planes         */
  int cache_kv_blocks; /* with cache_y: hybrid cache — this many blocks keep K/V, the     */
                       /*     other N - cache_kv_blocks are Y blocks (0 = pure Y): the     */
                       /*     first N - kv_blocks entries of the bit-reversal order over   */
                       /*     the next power of two >= N (entries >= N skipped), i.e. Y    */
                       /*     blocks spread evenly over the step.  Per step, block b       */
                       /*     stores [K_b, V_b] if it is a K/V block, then [Y_b] if block  */
                       /*     b or b + 1 is a Y block (ig_cache_write takes that order)    */
  int use_graphs;      /* 1 = capture each distinct step shape (row counts, plan, cache    */
                       /*     kinds, descriptor slot) as a CUDA graph and replay it: one   */
                       /*     launch per step instead of ~10 per block.  Applies to steps  */
                       /*     whose caches are HBM-resident (or absent) with copy_mode != 0,*/
                       /*     on a non-default stream, profiling off; others run eagerly   */
} ig_ctx_opts;

typedef struct ig_ctx ig_ctx;
typedef struct ig_cache ig_cache;
typedef struct ig_mask ig_mask;

/* Create a context on `device`.  weights: n_weights device pointers in table order.
 * opts may be NULL (defaults).  Allocates workspaces and per-slot K/V rings
 * (max_batch x (D+1) x 2 x L x H elements).  Errors: IG_EINVAL, IG_EUNSUPPORTED, IG_ENOMEM,
 * IG_ECUDA. */
ig_status ig_ctx_create(const ig_model_desc* desc, const void* const* weights, int n_weights,
                        int device, const ig_ctx_opts* opts, ig_ctx** out);
void ig_ctx_destroy(ig_ctx* ctx);

typedef enum { IG_CACHE_HOST = 0, IG_CACHE_DEVICE = 1 } ig_cache_tier;

/* Template cache: for every (step s, block b) the image-token K and V exactly as consumed
 * by attention (post-bias, post-RMSNorm, post-RoPE; C-AMB 2), layout
 * [n_steps][n_blocks][2 (K,V)][L_img][H] — or, for a ctx created with cache_y, the block
 * output Y [n_steps][n_blocks][L_img][H] — dtype = desc.dtype, in pinned host memory
 * (IG_CACHE_HOST, "host memory ... for cached activations") or in HBM
 * (IG_CACHE_DEVICE), followed by the template's input latent of every step
 * [n_steps][L_img][lat_ch] fp32 (used by the Algorithm-1 dense prefix, ig_set_plan).  Bytes = n_steps*n_blocks*2*L_img*H*sizeof(dtype): twice the
 * Y-cache size ("doubles the sizes of the cached activations"). */
ig_status ig_cache_create(ig_ctx* ctx, int n_steps, int tier, ig_cache** out);

/* Dense sampler over the template's own schedule (C-AMB 10; "pre-computed
 * activations from previous requests"): runs n_steps full-token steps from `latent`
 * (dev [L_img, lat_ch] fp32, updated in place along the trajectory), recording every
 * (step, block) K/V into a new cache.  sigmas: host [n_steps+1].  txt: dev [txt_len, H]
 * (desc.dtype), cond_vec: dev [H] fp32.  Uses slot 0's staging; must not run concurrently
 * with ig_edit_step on the same ctx.  Synchronises `stream` before returning. */
ig_status ig_cache_template(ig_ctx* ctx, float* latent, const void* txt, const float* cond_vec,
                            const float* sigmas, int n_steps, int tier, void* stream,
                            ig_cache** out);

/* Record the template into an EXISTING cache (e.g. one attached to a shared-memory segment by
 * ig_cache_attach: one host copy per box, written once, read by every GPU's
 * process).  Same semantics as ig_cache_template; the cache must have this ctx's cache kind
 * (K/V, Y or hybrid split; bf16 or fp8) and at least n_steps steps, and no enqueued step may
 * read it.  Synchronises `stream`. */
ig_status ig_cache_template_into(ig_ctx* ctx, float* latent, const void* txt, const float* cond_vec,
                                 const float* sigmas, int n_steps, ig_cache* cache, void* stream);

/* Bytes of a cache of this ctx's cache kind for n_steps steps (planes + per-step template
 * latents; the size to give a shared segment for ig_cache_attach). */
ig_status ig_cache_bytes(const ig_ctx* ctx, int n_steps, size_t* bytes);

/* A host-tier cache on CALLER-OWNED host memory (SURVEY §8(e) "template caches live once in host
 * shared memory; each process maps them with cudaHostRegister"): host_mem (>= ig_cache_bytes,
 * e.g. a POSIX shared-memory mapping that several processes map) is page-locked and mapped with
 * cudaHostRegister; the layout is exactly ig_cache_create's.  ig_cache_free unregisters it and
 * never frees it.  Contents are whatever the memory holds (record it with
 * ig_cache_template_into in one process, attach in the others after that finished). */
ig_status ig_cache_attach(ig_ctx* ctx, int n_steps, void* host_mem, size_t bytes, ig_cache** out);

/* Peer-HBM template pool (P:622-634 cache hierarchy, template reuse P:263-267): an
 * HBM-tier cache (IG_CACHE_DEVICE) of one process is exported as an opaque handle of
 * IG_CACHE_HANDLE_BYTES bytes (CUDA IPC); another process imports it on its own ctx — on another
 * GPU the copy lane then reads the cached rows from the owner's HBM over NVLink (peer access)
 * instead of streaming them from host memory over PCIe.  The importer's ctx must have the same
 * cache kind (ig_cache_bytes must match: IG_ECACHE_INCOMPAT otherwise); ig_cache_free of an
 * imported cache closes the mapping (the owner keeps the storage, and must outlive importers).
 * IG_EUNSUPPORTED when the two devices cannot access each other. */
#define IG_CACHE_HANDLE_BYTES 128
ig_status ig_cache_export(const ig_cache* cache, void* handle, size_t handle_bytes);
ig_status ig_cache_import(ig_ctx* ctx, const void* handle, ig_cache** out);


/* Copy of a cache into another tier (e.g. an HBM-resident hot template) in the
 * cache format of `ctx` (a bf16 cache cloned by a cache_fp8 ctx is quantized per (token,
 * head) on the device).  Same schedule.  Synchronous. */
ig_status ig_cache_clone(ig_ctx* ctx, const ig_cache* src, int tier, ig_cache** out);

/* Write a whole cache from caller K/V in the compute dtype (dev or host pointer,
 * [n_steps][n_blocks][2][L_img][H]); FP8 caches are quantized on the device (per (token, head)
 * scale = amax/448, e4m3 round-to-nearest-even, saturating).  latents (optional, fp32
 * [n_steps][L_img][lat_ch]): the template's input latent of every step (Algorithm-1 dense
 * prefix).  Synchronous on `stream`. */
ig_status ig_cache_write(ig_ctx* ctx, ig_cache* cache, const void* kv, const float* latents, void* stream);

/* Raw storage of a cache: host or device pointer (per tier) and its size in bytes, for
 * test I/O and for filling a synthetic cache.  The pointer stays owned by the cache. */
ig_status ig_cache_storage(ig_cache* cache, void** ptr, size_t* bytes, int* tier);
/* Deferred until no enqueued step references the cache (pin count). */
void ig_cache_free(ig_cache* cache);

/* a1 — index build (kernel a, C-AMB 13-16).  mask: dev uint8 [L_img], nonzero =
 * masked.  Builds idx_m (ascending masked token indices) and idx_u (ascending complement)
 * on the device and returns n_m to the host (one stream sync at admission, never on the
 * step path).  n_masked may be NULL. */
ig_status ig_mask_build(ig_ctx* ctx, const uint8_t* mask, void* stream, ig_mask** out,
                        int* n_masked);
/* a1 from a HOST bitmap (the serving path's admission, no device sync): mask = host uint8
 * [L_img] (nonzero = masked), read before the call returns.  n_m, the unmasked runs and the
 * bitmap are derived on the host; the bitmap goes up with one small async copy and kernel (a)
 * builds idx_m / idx_u on the device, all enqueued on `stream` (stream-ordered allocation).
 * Steps that use the mask must run on `stream` or be ordered after it.  ig_mask_free of such a
 * mask is stream-ordered after the last step that read it (the stream must still exist). */
ig_status ig_mask_build_host(ig_ctx* ctx, const uint8_t* mask, void* stream, ig_mask** out,
                             int* n_masked);
/* Device pointers to idx_m [n_m] and idx_u [L_img - n_m] (int32) and n_m. */
ig_status ig_mask_indices(const ig_mask* mask, const int32_t** idx_m, const int32_t** idx_u,
                          int* n_m);
void ig_mask_free(ig_mask* mask);

typedef struct {
  int slot;                /* continuous-batching slot 0..max_batch-1, stable for the       */
                           /* request's life; distinct within one call                      */
  float* latent;           /* [L_img, lat_ch] fp32, in/out: masked rows updated, unmasked    */
                           /* rows untouched (C-AMB 11).  Device memory, or pinned host memory */
                           /* (cudaHostAlloc / cudaHostRegister; the host-buffer path of the   */
                           /* public API): the gather and Euler-scatter kernels then read and  */
                           /* write only the masked rows in place over the host link           */
  const ig_mask* mask;
  const ig_cache* cache;   /* NULL allowed only when n_m == L_img (ignored then, C-AMB 27)   */
  int step;                /* index into the cache's schedule (C-AMB 9)                      */
  float sigma, sigma_next; /* flow-matching Euler step; t = 1000*sigma (C-AMB 12)            */
  const void* txt;         /* dev [txt_len, H] (desc.dtype); UNet models: the cross-attention */
                           /* context [ctx_len, ctx_dim] (desc.dtype)                        */
  const float* cond_vec;   /* dev [H] fp32 (unused, may be NULL, for UNet models)            */
} ig_edit_req;

/* Y-cache requests (cache created by a cache_y ctx; any ctx can consume them, and a batch may
 * mix both kinds): block b's unmasked input rows are the template's Y_{b-1} rows (block 0:
 * img_in of the template's input latent; a block after a dense-prefix block: the computed
 * rows), they go through LN-modulation and the K/V projection only (Q, attention output and
 * the MLP stay on the masked rows), and the copy lane moves one plane per block instead of two.
 *
 * One mask-aware denoising step for a ragged continuous batch (P:642-659 step-level
 * continuous batching): for every block, only the [txt | masked image] rows of each
 * request go through the GEMMs, their fresh K/V are merged by mask index
 * with the template's cached unmasked-token K/V (fig:transformer_alter), masked-Q x full-KV
 * attention runs ragged across the batch, and the final velocity is scattered into
 * the masked latent rows.  The cache is prefetched layer by layer on the ctx copy stream,
 * D layers ahead, with event hand-off.  Requests with n_m == 0 are skipped
 * (no copies, latent bit-identical).  Enqueues on `stream`; returns after enqueue.
 * Errors: IG_EINVAL, IG_ECACHE_MISS, IG_ECACHE_INCOMPAT, IG_ENOMEM, IG_ECUDA. */
ig_status ig_edit_step(ig_ctx* ctx, const ig_edit_req* reqs, int n, void* stream);

/* Explicit warm-up: enqueue on the ctx copy stream the cached K/V of (req->cache,
 * req->step, layer) into req->slot's staging buffer for that layer and record the slot's
 * layer event.  ig_edit_step consumes a layer that was prefetched this way instead of
 * copying it again (only for layers < prefetch_depth of the next step). */
ig_status ig_prefetch_layer(ig_ctx* ctx, const ig_edit_req* req, int layer);

/* One step of a template recording (ig_cache_template's loop body, for callers that drive their
 * own sampler — e.g. the whole-UNet runtime recording each Transformer2D's K/V): the dense step
 * of req->latent (every token; req->mask / req->cache ignored) with every block's K/V (or Y)
 * written to entry `step` of `cache`, and req->latent copied in as the step's template input.
 * Enqueued on `stream`. */
ig_status ig_record_step(ig_ctx* ctx, const ig_edit_req* req, ig_cache* cache, int step, void* stream);

const char* ig_last_error(void);

/* Algorithm 1 block plan ("bubble-free pipeline"): the first k blocks of
 * a step run without cached activations over ALL tokens of each cache-using request (the
 * unmasked image tokens entering from the template's input latent of that step, recorded in
 * the cache), the remaining blocks use the cache (C-AMB 23: dense blocks must form a prefix
 * under K/V caching).  mode 0: k = 0 (always cache); mode 1: fixed k; mode 2: k chosen per
 * step by minimising the two-lane pipeline latency of the batch under the linear latency
 * models comp = comp_s_per_flop * FLOPs + comp_s and load = load_s_per_byte * bytes + load_s
 * (P:701-726), with the ring depth as the copy lane's look-ahead.  Use a prefetch_depth at
 * least as large as the expected prefix. */
ig_status ig_set_plan(ig_ctx* ctx, int mode, int k, double comp_s_per_flop, double comp_s,
                      double load_s_per_byte, double load_s);
/* Prefix length chosen by the last ig_edit_step. */
int ig_last_plan(const ig_ctx* ctx);

/* Host-only helper (no device, no ctx): the copy-engine calls the copy lane issues for a
 * host-tier cache under copy_mode 1 (a7; P:546-552 block-wise loading of the cached rows).
 * mask: L bytes, nonzero = masked token (raster order over a grid W tokens wide; W = 0 if
 * unknown).  row_bytes: one K (or V) row.  groups: cap x 4 ints per group {start, len, stride,
 * count} in token rows — one call moves rows [start + i*stride, start + i*stride + len) for
 * i < count, of the K and the V plane.  Every unmasked token is covered exactly once; masked
 * rows are covered only where that is cheaper than another call (a call costs the link time of
 * ~275 KB, so the plan minimises calls x 275 KB / (2 row_bytes) + masked rows copied).
 * *n_groups is always set; IG_EINVAL when it exceeds cap (nothing written) or on a bad
 * argument. */
ig_status ig_plan_copy_groups(const uint8_t* mask, int L, int W, int row_bytes, int* groups, int cap, int* n_groups);

/* Counters of the last ig_edit_step / ig_cache_template call on this ctx. */
typedef struct {
  long long kernel_launches;  /* libig kernels enqueued                      */
  long long h2d_bytes;        /* cache bytes copied host->device            */
  long long d2d_bytes;        /* cache bytes copied device->device          */
  long long d2h_bytes;        /* cache bytes recorded device->host          */
  long long rows;             /* packed query rows M                         */
  long long host_ns;          /* host time spent enqueueing the call, not counting the wait for
                                 a free descriptor slot (back-pressure from the GPU)            */
  long long dma_calls;        /* copy-engine calls the copy lane issued (copy_mode 1 groups)  */
} ig_stats;
ig_status ig_last_stats(const ig_ctx* ctx, ig_stats* out);

/* Live per-kernel-class timing for the roofline report: while enabled, every libig launch
 * on the compute stream is bracketed by CUDA events (recorded on the launching stream) and
 * tagged with its ALGORITHMIC work (flops for GEMM/attention = 2*M*N*K and 4*sum(q)*L*H;
 * bytes for the HBM-bound kernels).  ig_profile_read synchronises those events, returns the
 * per-class totals accumulated since the last read, and resets them. */
typedef enum {
  IG_K_GEMM = 0, IG_K_ATTN = 1, IG_K_LNMOD = 2, IG_K_QKVPOST = 3, IG_K_COND = 4,
  IG_K_ROWS = 5,
  IG_K_COPY = 6,  /* copy lane (a7): one entry per block's cache copy, timed on the copy stream */
  IG_K_NCLASS = 7
} ig_kernel_class;
typedef struct {
  long long launches;
  double ms;     /* sum of event-timed launch durations                       */
  double flops;  /* algorithmic flops of those launches (GEMM, attention)      */
  double bytes;  /* algorithmic HBM bytes of those launches (other classes)    */
} ig_prof_entry;
ig_status ig_profile_enable(ig_ctx* ctx, int enable);
ig_status ig_profile_read(ig_ctx* ctx, ig_prof_entry out[IG_K_NCLASS]);

/* Teacher-forced single block (debug/parity export): runs block `block` of the
 * step for ONE request on caller-given packed input rows and writes the packed output rows.
 * X_in, X_out: dev fp32 [txt_len + n_m, H], rows ordered [text 0..L_txt-1 | masked image
 * tokens ascending] (C-AMB 15).  The block's cached K/V come from (req->cache, req->step) and
 * the modulation from (req->sigma, req->cond_vec) exactly as in ig_edit_step.  The latent is
 * not touched.  Synchronous on `stream`. */
ig_status ig_debug_block(ig_ctx* ctx, const ig_edit_req* req, int block, const float* X_in,
                         float* X_out, void* stream);

/* Merged positional K/V buffer of (slot, block) as the last step left it (SURVEY §8(b) debug
 * export, T3/T4): the ring buffer block % (prefetch_depth + 1) of the slot, rows [text 0..L_txt-1
 * | image 0..L_img-1] (C-AMB 8), each plane [L][H] in desc.dtype.  Valid for the last
 * prefetch_depth + 1 blocks of the last step of that slot (earlier blocks' buffers were reused).
 * k_out, v_out: dev or host pointers of L*H elements.  Synchronises `stream` and the copy lane. */
ig_status ig_debug_dump_kv(ig_ctx* ctx, int slot, int block, void* k_out, void* v_out, void* stream);

/* Race tests and fault injection (SPEC S:615 negative control).  Debug only —
 * every key is 0 in normal operation:
 *   IG_DBG_SPIN_COPY_NS     the copy lane spins this many ns before each block's cache copy
 *                           (a slow copy lane: exposes a missing RAW wait)
 *   IG_DBG_SPIN_COMPUTE_NS  the compute lane spins before each attention (a slow compute lane:
 *                           exposes a missing WAR wait before a ring buffer is overwritten)
 *   IG_DBG_DROP_RAW         1 = compute does NOT wait for the copy of a block (negative control)
 *   IG_DBG_DROP_WAR         1 = the copy lane does NOT wait for the buffer's previous reader
 *   IG_DBG_CORRUPT_ROW      v > 0: after each block's copy add v to every element of the K and
 *                           V rows of the first unmasked token of the batch's first cache user
 *                           (a corrupted cache row: must turn parity red)
 *   IG_DBG_POISON_RING      immediate (value ignored): synchronise the device and fill every
 *                           slot's K/V ring with NaN; a correct step re-stages every row it
 *                           reads, so its result is unchanged
 *   IG_DBG_SEQUENTIAL       1 = sequential loading (the ablation of P:299-300 / fig:pipeline_load):
 *                           block b's cache copy starts only after block b-1 finished computing
 *                           and block b waits for it — no copy/compute overlap
 * IG_EINVAL on an unknown key or a negative value. */
typedef enum {
  IG_DBG_SPIN_COPY_NS = 1, IG_DBG_SPIN_COMPUTE_NS = 2, IG_DBG_DROP_RAW = 3, IG_DBG_DROP_WAR = 4,
  IG_DBG_CORRUPT_ROW = 5, IG_DBG_POISON_RING = 6, IG_DBG_SEQUENTIAL = 7
} ig_debug_key;
ig_status ig_debug_set(ig_ctx* ctx, int key, long long value);

#ifdef __cplusplus
}
#endif
#endif /* IG_H_ */
