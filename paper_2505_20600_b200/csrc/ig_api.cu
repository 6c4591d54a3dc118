// ig_api.cu — libig host runtime: contexts, masks, template caches, the mask-aware step
// (ig_edit_step) and its layer-wise cache prefetch pipeline.  C ABI in include/ig.h.
//
// Step structure: batch assembly -> conditioning GEMVs -> entry gather +
// img_in -> per block [LN+mod -> QKV GEMM -> (wait cache copy) -> QK-norm/RoPE/positional
// K/V merge -> ragged attention -> (free buffer) -> out-proj (+MLP) with gated residual] ->
// final layer -> Euler scatter.  The copy stream moves the template's cached K/V of block
// b + R into ring buffer (b % R) while block b computes ("while loading the i-th
// block, the computation stream can concurrently execute the computation of the (i-1)-th").
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <cstdint>
#include <condition_variable>
#include <deque>
#include <functional>
#include <mutex>
#include <thread>
#include <chrono>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/ig.h"
#include "../../include/ig_ops.h"
#include "kernels.h"
#include "ig_internal.h"
#include "unet_kernels.h"

using namespace ig;

#include <execinfo.h>
#include <signal.h>
#include <unistd.h>
// IG_SEGV_TRACE=1: print a native backtrace of libig on SIGSEGV (debug aid)
static void ig_segv_handler(int sig) {
  void* buf[64];
  int n = backtrace(buf, 64);
  backtrace_symbols_fd(buf, n, 2);
  _exit(128 + sig);
}
__attribute__((constructor)) static void ig_install_trace() {
  if (getenv("IG_SEGV_TRACE")) signal(SIGSEGV, ig_segv_handler);
}

// ----------------------------------------------------------------------------------------
// errors
// ----------------------------------------------------------------------------------------
static thread_local std::string g_err;

static ig_status set_err(ig_status s, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define CUDA_TRY(expr)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return set_err(IG_ECUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_),   \
                     __FILE__, __LINE__);                                                  \
  } while (0)

extern "C" const char* ig_last_error(void) { return g_err.c_str(); }

ig_status ig_internal_err(ig_status s, const char* msg) {
  g_err = msg;
  return s;
}

// ----------------------------------------------------------------------------------------
// structures
// ----------------------------------------------------------------------------------------
namespace {
struct LinW {
  const void* w = nullptr;
  const void* b = nullptr;
  int out = 0, in = 0;
};
struct StreamW {
  LinW mod, qkv, proj, fc1, fc2;
  const void* qg = nullptr;
  const void* kg = nullptr;
  bool pre_only = false;
  int mod_t = -1;  // index into ctx->mods
};
struct SingleW {
  LinW mod, lin1, lin2;
  const void* qg = nullptr;
  const void* kg = nullptr;
  int mod_t = -1;
};
// UNet BasicTransformerBlock (config 5; ig.h weight table): LayerNorm affines live in
// ctx->unet_ln as (shift = beta, scale = gamma - 1) rows for the LN-modulation kernel
struct UnetW {
  const void* qkv = nullptr;            // [3H, H], no bias
  LinW out1, q2, kv2, out2, geglu, ff2; // q2 / kv2 without bias
  const void* geglu_w_tc = nullptr;     // tile-interleaved copy for EPI_GEGLU (bf16 + tcgen05)
  const void* geglu_b_tc = nullptr;
};
struct ModT {
  const LinW* w;
  int k;
  long long off;  // float offset inside one request's modulation row
};
constexpr int NSTAGE = 4;
constexpr int MAXR = 32;  // max ring depth R = D + 1

// a7 host tier, copy_mode 1: the unmasked runs of a mask (raster order over the token grid)
// are covered by groups, ONE copy-engine call each: group g moves token rows
// [start + i * stride, start + i * stride + len) for i < count (a 1-D span when count == 1,
// cudaMemcpy2DAsync rows otherwise; the K and V planes of a group together in one
// cudaMemcpy3DAsync when the plane strides allow).  A copy-engine call costs ~5 us whatever its
// size (tools/dma_probe.py on this pool: 6 KB copies run at 1.2 GB/s, a 2-D copy of 64 rows of
// 24 KB at 48 GB/s, the link peaks at 55.5 GB/s), i.e. as much link time as ~275 KB of
// payload, so the grouping is a shortest path over the runs: cost = calls x call_rows + masked
// rows copied (also planned with masked gaps < call_rows / 3 pre-merged; the cheaper plan wins).  Candidate groups over runs i..j: the contiguous span [s_i, e_j), or strided
// rows with stride s_{i+1} - s_i or the grid width W (a rectangle's runs, or the rows around a
// blob).  Masked rows a group also covers carry template values that the block's fresh K/V
// overwrite: the compute lane waits for the copy before the QKV epilogue's positional merge
// (early wait).
struct CopyGroup {
  int start, len, stride, count;
};
struct CopyOp {  // one copy-engine call: `height` rows of `width` bytes, `pitch` apart, on
  void* dst;     // `planes` planes (src_plane / dst_plane bytes apart)
  const void* src;
  size_t width, height, pitch;
  int planes;
  size_t src_plane, dst_plane;
};
constexpr double DMA_CALL_BYTES = 275e3;  // link payload equivalent of one call's fixed cost
int copy_call_rows(size_t row_bytes, int planes) {
  return std::max(1, (int)std::lround(DMA_CALL_BYTES / ((double)row_bytes * std::max(planes, 1))));
}
// shortest path over `runs`; returns calls x call_rows + rows copied beyond the runs
long long copy_groups_dp(const std::vector<std::pair<int, int>>& runs, int L, int W, int call_rows,
                         std::vector<CopyGroup>& out) {
  out.clear();
  const int n = (int)runs.size();
  if (n == 0) return 0;
  const long long INF = (long long)1 << 60;
  std::vector<long long> best(n + 1, INF);
  std::vector<CopyGroup> pick(n + 1);
  std::vector<int> from(n + 1, 0);
  best[0] = 0;
  auto S = [&](int k) { return runs[k].first; };
  auto E = [&](int k) { return runs[k].first + runs[k].second; };
  for (int i = 0; i < n; ++i) {
    if (best[i] >= INF) continue;
    long long exact = 0;
    for (int j = i; j < n; ++j) {  // contiguous span over runs i..j
      exact += runs[j].second;
      const long long c = best[i] + call_rows + (E(j) - S(i) - exact);
      if (c < best[j + 1]) {
        best[j + 1] = c;
        pick[j + 1] = CopyGroup{S(i), E(j) - S(i), 0, 1};
        from[j + 1] = i;
      }
    }
    if (i + 1 >= n) continue;
    const int cand[2] = {S(i + 1) - S(i), W};
    for (int ci = 0; ci < 2; ++ci) {
      const int stride = cand[ci];
      if (stride <= 0 || (ci == 1 && stride == cand[0])) continue;
      const int lo_lim = i > 0 ? E(i - 1) : 0;  // row 0 must not reach the previous run
      int base = S(i), top = E(i);
      exact = runs[i].second;
      for (int j = i + 1; j < n; ++j) {
        const int k = j - i;
        base = std::min(base, S(j) - k * stride);
        top = std::max(top, E(j) - k * stride);
        if (top - base > stride || base < lo_lim) break;  // rows would overlap / reach run i-1
        exact += runs[j].second;
        const long long last_end = (long long)top + (long long)k * stride;
        if (last_end > (j + 1 < n ? S(j + 1) : L)) continue;  // last row reaches the next run
        const long long c = best[i] + call_rows + ((long long)(top - base) * (k + 1) - exact);
        if (c < best[j + 1]) {
          best[j + 1] = c;
          pick[j + 1] = CopyGroup{base, top - base, stride, k + 1};
          from[j + 1] = i;
        }
      }
    }
  }
  for (int j = n; j > 0; j = from[j]) out.push_back(pick[j]);
  std::reverse(out.begin(), out.end());
  return best[n];
}
// returns the plan's link-time rows: rows moved + calls x call_rows
long long make_copy_groups(const std::vector<std::pair<int, int>>& runs, int L, int W, int call_rows,
                           std::vector<CopyGroup>& out) {
  long long exact = 0;
  for (const auto& r : runs) exact += r.second;
  const long long c0 = copy_groups_dp(runs, L, W, call_rows, out);
  // a noisy mask edge leaves many short runs that the strided candidates cannot follow: also
  // plan over the runs with masked gaps < call_rows / 3 merged (copying such a gap is cheaper
  // than a call) and keep the cheaper plan, both costed against the exact runs
  std::vector<std::pair<int, int>> merged;
  long long gap_rows = 0;
  for (const auto& r : runs) {
    const int gap = merged.empty() ? 0 : r.first - (merged.back().first + merged.back().second);
    if (!merged.empty() && 3 * gap < call_rows) {
      merged.back().second = r.first + r.second - merged.back().first;
      gap_rows += gap;
    } else {
      merged.push_back(r);
    }
  }
  if (merged.size() == runs.size()) return exact + c0;
  std::vector<CopyGroup> alt;
  const long long c1 = copy_groups_dp(merged, L, W, call_rows, alt) + gap_rows;
  if (c1 < c0) out.swap(alt);
  return exact + std::min(c0, c1);
}
// copy-engine calls for `planes` planes of token rows of `row` bytes between positional buffers
void push_group_copies(std::vector<CopyOp>& v, char* dst, const char* src, size_t row,
                       const std::vector<CopyGroup>& groups, int planes = 1, size_t src_plane = 0,
                       size_t dst_plane = 0) {
  for (const CopyGroup& g : groups)
    v.push_back(CopyOp{dst + (size_t)g.start * row, src + (size_t)g.start * row, (size_t)g.len * row,
                       (size_t)g.count, (size_t)(g.count > 1 ? g.stride : g.len) * row, planes, src_plane,
                       dst_plane});
}
cudaError_t issue_copy_op(const CopyOp& c, cudaStream_t st) {
  if (c.planes == 2) {
    // both planes in one 3-D copy when each plane stride is a whole number of row pitches
    // (1-D spans: pitch = the plane stride itself)
    const bool span = c.height == 1;
    const size_t sp = span ? c.src_plane : c.pitch, dp = span ? c.dst_plane : c.pitch;
    if (c.src_plane % sp == 0 && c.dst_plane % dp == 0) {
      cudaMemcpy3DParms p{};
      p.srcPtr = make_cudaPitchedPtr(const_cast<void*>(c.src), sp, c.width, c.src_plane / sp);
      p.dstPtr = make_cudaPitchedPtr(c.dst, dp, c.width, c.dst_plane / dp);
      p.extent = make_cudaExtent(c.width, c.height, 2);
      p.kind = cudaMemcpyDefault;
      return cudaMemcpy3DAsync(&p, st);
    }
  }
  cudaError_t e = cudaSuccess;
  for (int w = 0; w < c.planes && e == cudaSuccess; ++w) {
    char* d = (char*)c.dst + w * c.dst_plane;
    const char* s = (const char*)c.src + w * c.src_plane;
    e = c.height == 1 ? cudaMemcpyAsync(d, s, c.width, cudaMemcpyDefault, st)
                      : cudaMemcpy2DAsync(d, c.pitch, s, c.pitch, c.width, c.height, cudaMemcpyDefault, st);
  }
  return e;
}
}  // namespace

struct ig_mask {
  int L_img = 0, n_m = 0;
  std::vector<std::pair<int, int>> runs;  // host: maximal runs (start, len) of unmasked tokens
  std::vector<CopyGroup> groups;          // host: strided DMA groups covering `runs` (copy_mode 1)
  long long dma_rows = 0;                 // rows the groups move + calls x call_rows (link-time rows)
  std::vector<uint8_t> bits;              // host: 1 = masked (load deduplication)
  uint8_t* bits_dev = nullptr;            // device copy of bits
  int32_t* idx = nullptr;  // device: idx_m at [0, L_img), idx_u at [L_img, 2 L_img), n_m at [2 L_img]
  bool async_alloc = false;                 // ig_mask_build_host: idx + bits_dev are ONE stream-ordered allocation
  cudaStream_t build_st = nullptr;          // stream of the build
  mutable cudaStream_t last_st = nullptr;   // compute stream of the last step that read the mask
  mutable bool used = false;
};

struct ig_cache {
  ig_model_desc desc{};
  int n_steps = 0, tier = 0;
  int fp8 = 0;              // 1: e4m3 data [steps][blocks][2][L_img][H] + fp32 scales [..][heads]
  int y = 0;                // 1: Y variant (block outputs of the image tokens), see ymode
  int kv_blocks = 0;        // hybrid: number of blocks that keep K/V (0 = pure Y)
  std::vector<uint8_t> ymode;  // per block: 1 = Y block (interleaved order, ig.h cache_kv_blocks)
  int step_planes = 0;      // planes per step: [K_b, V_b] for K/V blocks, then [Y_b] when block b
                            // or b + 1 is a Y block (Y_b feeds block b + 1)
  size_t scale_off = 0;     // byte offset of the scale region (fp8 only)
  size_t lat_off = 0;       // template input latent per step [steps][L_img][C] fp32 (Algorithm-1
                            // dense prefix: unmasked rows enter from the template's trajectory)
  void* ptr = nullptr;     // pinned host (mapped) or device
  void* dptr = nullptr;    // device-visible pointer (== ptr with UVA)
  bool registered = false; // caller-provided host memory (ig_cache_attach): unregistered, never freed
  bool imported = false;   // another process's HBM cache opened by IPC (ig_cache_import): closed, never freed
  int owner_device = -1;   // device that holds the storage (peer tier: != device)
  size_t bytes = 0;
  mutable std::atomic<int> pins{0};
  std::atomic<bool> zombie{false};
  int device = 0;
};

struct ig_ctx {
  ig_model_desc d{};
  ig_ctx_opts o{};
  int device = 0;
  size_t esz = 4;
  int H = 0, F = 0, C = 0, L = 0, Limg = 0, Lt = 0, nb = 0, R = 2;
  std::vector<const void*> w;
  LinW img_in, t1, t2, fmod, pout;
  const void* pos_embed = nullptr;
  std::vector<StreamW> dimg, dtxt;
  std::vector<SingleW> sgl;
  std::vector<UnetW> unet;
  // UNet-only buffers: LN constants fp32 [nb][3][2H]; ones [H] (ungated residual); cross K/V
  // arena [max_batch][2][ctx_len][H]; packed contexts [max_batch * ctx_len][ctx_dim]; the
  // context rows' RowInfo (static: slot = request index, kvpos = context token); unfused GEGLU
  // input [max_rows][2F]; interleaved GEGLU weights (bf16)
  float* unet_ln = nullptr;
  float* ones = nullptr;
  void* xkv = nullptr;
  void* ctxp = nullptr;
  RowInfo* ri_c = nullptr;
  void* u2 = nullptr;
  void* geglu_tc = nullptr;
  // bf16: the next block's cross K/V GEMM runs on a side stream while the current block's
  // self-attention chain (small-M GEMMs that leave SMs idle) runs on the compute stream; the
  // cross arena is double-buffered by block parity
  cudaStream_t xs = nullptr;
  // double blocks: the text stream's ops run on ts concurrently with the image stream's (disjoint
  // rows of X / h / Q / cat; ig_tuning.txt_overlap)
  cudaStream_t ts = nullptr;
  cudaEvent_t ev_tfork[2] = {}, ev_tjoin[2] = {};
  cudaEvent_t ev_xfork = nullptr, ev_xkv[2] = {}, ev_xuse[2] = {};
  std::vector<ModT> mods;
  long long mod_ld = 0;
  int fmod_t = -1;
  // device buffers
  float *X = nullptr, *vel = nullptr, *temb = nullptr, *tmp = nullptr, *vec = nullptr,
        *svec = nullptr, *modbuf = nullptr;
  void *h = nullptr, *qkv = nullptr, *Q = nullptr, *cat = nullptr, *Ain = nullptr;
  void* kv_arena = nullptr;
  long long slot_stride = 0, buf_elems = 0;
  float2* rope_tab = nullptr;
  int rope_maxpos = 1;
  GemvProb *gv_t1 = nullptr, *gv_t2 = nullptr, *gv_mod = nullptr;
  // bf16 mode: every block's modulation weight packed into one [mod_ld, H] matrix (+ bias) so
  // the whole a3 modulation is ONE tensor-core GEMM [n, H] x [mod_ld, H]^T (HBM-bound on the
  // 6.5 GB of weights) instead of a CUDA-core GEMV
  void* modw = nullptr;
  void* modb = nullptr;
  bf16* svec_bf = nullptr;
  int gv_mod_groups = 0;
  std::vector<GemvProb> gv_mod_host;
  // per-step descriptors: device ring + pinned host staging
  size_t stage_bytes = 0;
  char* h_stage[NSTAGE] = {};
  char* d_stage[NSTAGE] = {};
  char* m_stage[NSTAGE] = {};  // device (UVA) view of the mapped pinned h_stage
  char* d_gstage = nullptr;    // graph-mode steps: one fixed device descriptor slot (see run_step)
  cudaEvent_t ev_stage[NSTAGE] = {};
  int stage_i = 0;
  RowInfo* ri = nullptr;
  // streams / events
  cudaStream_t copy_st = nullptr;
  cudaEvent_t ev_copy[MAXR] = {}, ev_comp[MAXR] = {}, ev_desc = nullptr;
  // explicit prefetch bookkeeping: (slot, layer) -> (cache, step) already in the ring
  struct Pref { const ig_cache* c = nullptr; int step = -1; };
  std::vector<Pref> pref;  // [max_batch * R]
  ig_mask* ones_mask = nullptr;
  std::vector<CopyOp> b_copies;      // copy-lane scratch (copy_mode 1): one copy-engine call each
  // FP8 cache staging (cache_fp8): per (slot, ring buffer) e4m3 rows + scales landed by the DMA
  // lane before the dequantizing gather into the bf16 ring; per ring buffer for recording
  uint8_t* q8in = nullptr;  float* q8in_scl = nullptr;
  uint8_t* q8rec = nullptr; float* q8rec_scl = nullptr;
  // Y recording staging (cache_y): per ring buffer the block output's image rows in the
  // compute dtype, read by the D2H on the copy stream; ev_yrec guards its reuse (WAR)
  void* yrec = nullptr;
  cudaEvent_t ev_yrec[MAXR] = {};
  uint8_t* q8yrec = nullptr; float* q8yrec_scl = nullptr;  // FP8 Y recording: [R][2][plane] (+ scales)
  ig_stats stats{};
  // first enqueue failure of the copy lane inside the current step (checked at the step's end:
  // a rejected DMA leaves ring rows stale, so the step must not report success)
  cudaError_t copy_err = cudaSuccess;
  size_t copy_err_idx = 0;
  // ig_debug_set keys (race tests and fault injection; all 0 in normal operation)
  long long dbg[9] = {};
  // Copy-lane host thread: the cache-prefetch enqueues (strided DMA copies of the unmasked
  // runs, gathers, dedupe) run on their own host thread, so the compute launches are never
  // stuck behind the copy engines' queue back-pressure.  Jobs run in order; the compute thread
  // waits (host side) only for the job that recorded the ring event it is about to wait on.
  struct CopyLane {
    std::thread thr;
    std::mutex mu;
    std::condition_variable cv, cv_done;
    std::deque<std::function<void()>> q;
    long long pushed = 0, done = 0;
    bool stop = false;
  } lane;
  bool lane_on = false;        // this step issues copies through the thread
  ig_stats cstats{};           // copy-lane counters of the current step (merged after the drain)
  std::vector<long long> job_of_block;  // per block: lane job that issued its copy (-1: inline / none)
  // CUDA graphs of whole steps (ig_ctx_opts.use_graphs): keyed by everything that shapes the
  // launches (row counts, plan, staging slot, cache kinds); the per-step data (sigmas, step
  // indices, cache plane pointers, latents) live in the descriptors the graph itself pulls
  // from the staging slot, so a replay needs no re-enqueue
  struct GraphEnt { cudaGraphExec_t exec; ig_stats stats; unsigned long long last_used; };
  unsigned long long step_no = 0;  // steps run on this ctx (graph LRU / in-flight test)
  std::unordered_map<std::string, GraphEnt> graphs;
  bool capturing = false;
  unsigned cap_mask = 0;  // ring buffers whose ev_comp was recorded inside the capture
  // a graph ran last: the ring events' latest records are capture nodes (not waitable
  // eagerly), so the next eager step first re-records them after the graph on its stream
  bool graph_tail = false;
  cudaStream_t graph_st = nullptr;
  // PDL: the next GEMM may overlap its prologue with the previous kernel only if nothing but a
  // kernel precedes it on the stream (no event wait, memcpy or step boundary in between)
  bool pdl_block = true;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // Algorithm-1 block plan (ig_set_plan): 0 off, 1 forced dense-prefix length, 2 model
  int plan_mode = 0, plan_k = 0, last_plan_k = 0;
  double pm_cs = 0, pm_cb = 0, pm_ls = 0, pm_lb = 0;  // s/FLOP, s, s/byte, s
  // live profiling (ig_profile_enable)
  bool prof = false;
  cudaEvent_t prof_t0 = nullptr;
  struct ProfRec { int kind; cudaEvent_t a, b; double flops, bytes; int M, N, K, epi; };
  std::vector<ProfRec> prof_recs;
  std::vector<cudaEvent_t> ev_pool;
  ig_prof_entry prof_acc[IG_K_NCLASS] = {};
};

static cudaEvent_t pool_event(ig_ctx* ctx) {
  if (!ctx->ev_pool.empty()) {
    cudaEvent_t e = ctx->ev_pool.back();
    ctx->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// RAII bracket around one launch when profiling is enabled
struct ProfScope {
  ig_ctx* ctx; cudaStream_t st; int kind; double flops, bytes; cudaEvent_t a = nullptr;
  int M = 0, N = 0, K = 0, epi = -1;
  ProfScope(ig_ctx* c, cudaStream_t s, int k, double f, double b, int m = 0, int n = 0, int kk = 0, int e = -1)
      : ctx(c), st(s), kind(k), flops(f), bytes(b), M(m), N(n), K(kk), epi(e) {
    if (ctx->prof) { a = pool_event(ctx); cudaEventRecord(a, st); }
  }
  ~ProfScope() {
    if (!a) return;
    cudaEvent_t b = pool_event(ctx);
    cudaEventRecord(b, st);
    ctx->prof_recs.push_back({kind, a, b, flops, bytes, M, N, K, epi});
  }
};

// ----------------------------------------------------------------------------------------
// helpers
// ----------------------------------------------------------------------------------------
static bool desc_equal(const ig_model_desc& a, const ig_model_desc& b) {
  return memcmp(&a, &b, sizeof(a)) == 0;
}

extern "C" int ig_weight_count(const ig_model_desc* d) {
  if (!d) return -1;
  if (d->n_unet > 0) return 17 * d->n_unet;
  int n = 10 + (d->pos_embed_2d ? 1 : 0);
  for (int i = 0; i < d->n_double; ++i)
    for (int s = 0; s < 2; ++s) {
      bool pre = d->context_pre_only_last && s == 1 && i == d->n_double - 1;
      n += 4 + (d->qk_norm ? 2 : 0) + (pre ? 0 : 6);
    }
  n += d->n_single * (6 + (d->qk_norm ? 2 : 0));
  return n;
}

static void free_cache_now(ig_cache* c) {
  if (!c) return;
  if (c->ptr) {
    if (c->registered) cudaHostUnregister(c->ptr);
    else if (c->imported) cudaIpcCloseMemHandle(c->ptr);
    else if (c->tier == IG_CACHE_HOST) cudaFreeHost(c->ptr);
    else cudaFree(c->ptr);
  }
  delete c;
}

// caches freed while a step still pinned them (ig_cache_free is deferred); reaped
// by later ig_cache_free / ig_edit_step / ig_ctx_destroy calls once their pins dropped
static std::mutex g_zombie_mu;
static std::vector<ig_cache*> g_zombies;

static void reap_zombies_locked(int device) {
  for (size_t i = 0; i < g_zombies.size();) {
    ig_cache* z = g_zombies[i];
    if ((device < 0 || z->device == device) && z->pins.load() == 0) {
      int cur = 0;
      cudaGetDevice(&cur);
      const int dev = z->device;
      if (dev != cur) cudaSetDevice(dev);
      free_cache_now(z);
      if (dev != cur) cudaSetDevice(cur);
      g_zombies.erase(g_zombies.begin() + i);
    } else {
      ++i;
    }
  }
}

static void reap_zombies(ig_ctx* ctx) {
  std::lock_guard<std::mutex> lk(g_zombie_mu);
  reap_zombies_locked(ctx->device);
}

static void CUDART_CB unpin_cb(void* p) {
  ig_cache* c = (ig_cache*)p;
  c->pins.fetch_sub(1);
}

// ----------------------------------------------------------------------------------------
// kernel dispatch by dtype (fp32 parity mode -> CUDA cores; bf16 -> tensor cores)
// ----------------------------------------------------------------------------------------
static bool g_tc_gemm = true;   // tcgen05 GEMM for bf16 (set false only by IG_TEST_SIMT)
static bool g_tc_attn = true;


static void gemm(ig_ctx* ctx, const GemmArgs& g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0) return;
  ctx->stats.kernel_launches++;
  ProfScope ps(ctx, st, IG_K_GEMM, 2.0 * g.M * g.N * g.K, 0.0, g.M, g.N, g.K, g.epi);
  GemmArgs g2 = g;
  g2.pdl = ig_tuning_ref().pdl && !ctx->pdl_block && !ctx->prof;  // (profiling brackets launches with events)
  ctx->pdl_block = false;
  if (ctx->d.dtype == IG_F32) launch_gemm_simt<float>(g, st);
  else if (g_tc_gemm && gemm_tc_supported(g)) launch_gemm_tc(g2, st);
  else launch_gemm_simt<bf16>(g, st);
}

// a launch on a side stream: never programmatic, leaves the compute stream's PDL state alone
static void gemm_side(ig_ctx* ctx, const GemmArgs& g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0) return;
  ctx->stats.kernel_launches++;
  ProfScope ps(ctx, st, IG_K_GEMM, 2.0 * g.M * g.N * g.K, 0.0, g.M, g.N, g.K, g.epi);
  if (g_tc_gemm && gemm_tc_supported(g)) launch_gemm_tc(g, st);
  else launch_gemm_simt<bf16>(g, st);
}

// every event wait on the compute stream goes through here: the kernel after it must not be a
// programmatic (PDL) launch
static void stream_wait(ig_ctx* ctx, cudaStream_t st, cudaEvent_t ev) {
  cudaStreamWaitEvent(st, ev, 0);
  ctx->pdl_block = true;
}

static void attention(ig_ctx* ctx, const AttnArgs& a, cudaStream_t st, double flops) {
  ctx->stats.kernel_launches++;
  ProfScope ps(ctx, st, IG_K_ATTN, flops, 0.0);
  if (ctx->d.dtype == IG_F32) launch_attn_simt<float>(a, st);
  else if (g_tc_attn && attn_tc_supported(a)) launch_attn_tc(a, st);
  else launch_attn_simt<bf16>(a, st);
}

// ----------------------------------------------------------------------------------------
// context
// ----------------------------------------------------------------------------------------
static ig_status validate_desc(const ig_model_desc* d) {
  if (!d) return set_err(IG_EINVAL, "desc is NULL");
  if (d->hidden <= 0 || d->heads <= 0 || d->head_dim <= 0 || d->hidden != d->heads * d->head_dim)
    return set_err(IG_EINVAL, "hidden (%d) must equal heads (%d) * head_dim (%d)", d->hidden,
                   d->heads, d->head_dim);
  if (d->n_double < 0 || d->n_single < 0 || d->n_unet < 0 || d->n_double + d->n_single + d->n_unet <= 0)
    return set_err(IG_EINVAL, "need at least one block");
  if (d->n_unet > 0) {
    if (d->n_double || d->n_single || d->txt_len || d->qk_norm || d->rope || d->pos_embed_2d ||
        d->context_pre_only_last || d->lat_ch != d->hidden)
      return set_err(IG_EINVAL, "UNet models: no double/single blocks, txt_len = qk_norm = rope = "
                                "pos_embed_2d = 0 and lat_ch = hidden");
    if (d->ctx_len <= 0 || d->ctx_dim <= 0 || d->ctx_dim % 8)
      return set_err(IG_EINVAL, "UNet models need ctx_len > 0 and ctx_dim a positive multiple of 8");
  } else if (d->ctx_len || d->ctx_dim) {
    return set_err(IG_EINVAL, "ctx_len / ctx_dim are for UNet models only");
  }
  if (d->grid_h <= 0 || d->grid_w <= 0 || d->lat_ch <= 0 || d->txt_len < 0 || d->mlp_hidden <= 0)
    return set_err(IG_EINVAL, "bad grid/lat_ch/txt_len/mlp_hidden");
  if (d->head_dim != 16 && d->head_dim != 64 && d->head_dim != 128)
    return set_err(IG_EUNSUPPORTED, "head_dim %d not in {16, 64, 128}", d->head_dim);
  if (d->hidden % 64 || d->mlp_hidden % 64 || d->lat_ch % 4)
    return set_err(IG_EUNSUPPORTED, "hidden and mlp_hidden must be multiples of 64, lat_ch of 4");
  if (d->hidden > 4096) return set_err(IG_EUNSUPPORTED, "hidden > 4096");
  if (d->rope && d->rope_axes[0] + d->rope_axes[1] + d->rope_axes[2] != d->head_dim)
    return set_err(IG_EINVAL, "rope axes must sum to head_dim");
  if (d->rope && ((d->rope_axes[0] | d->rope_axes[1] | d->rope_axes[2]) & 1))
    return set_err(IG_EINVAL, "rope axes must be even");
  if (d->dtype != IG_F32 && d->dtype != IG_BF16) return set_err(IG_EINVAL, "bad dtype");
  if (d->context_pre_only_last && d->n_double <= 0)
    return set_err(IG_EINVAL, "context_pre_only_last needs a double block");
  return IG_OK;
}

static ig_status build_rope_table(ig_ctx* ctx) {
  const ig_model_desc& d = ctx->d;
  if (!d.rope) return IG_OK;
  const int P = std::max(1, std::max(d.grid_h, d.grid_w));
  const int pairs = d.head_dim / 2;
  std::vector<float2> tab((size_t)pairs * P);
  int e = 0;
  for (int a = 0; a < 3; ++a) {
    const int da = d.rope_axes[a];
    for (int j = 0; j < da / 2; ++j, ++e) {
      const double w = std::pow((double)d.rope_theta, -2.0 * j / da);
      for (int p = 0; p < P; ++p) {
        const double phi = p * w;
        tab[(size_t)e * P + p] = make_float2((float)std::cos(phi), (float)std::sin(phi));
      }
    }
  }
  ctx->rope_maxpos = P;
  CUDA_TRY(cudaMalloc(&ctx->rope_tab, tab.size() * sizeof(float2)));
  CUDA_TRY(cudaMemcpy(ctx->rope_tab, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice));
  return IG_OK;
}

extern "C" void ig_ctx_destroy(ig_ctx* ctx);
static void lane_stop(ig_ctx* ctx);

extern "C" ig_status ig_ctx_create(const ig_model_desc* desc, const void* const* weights,
                                   int n_weights, int device, const ig_ctx_opts* opts,
                                   ig_ctx** out) {
  if (!out) return set_err(IG_EINVAL, "out is NULL");
  *out = nullptr;
  ig_status s = validate_desc(desc);
  if (s != IG_OK) return s;
  const int nw = ig_weight_count(desc);
  if (!weights || n_weights != nw)
    return set_err(IG_EINVAL, "expected %d weight pointers, got %d", nw, n_weights);
  for (int i = 0; i < nw; ++i)
    if (!weights[i]) return set_err(IG_EINVAL, "weight %d is NULL", i);
  ig_ctx_opts o{8, 0, 2, 0, 0, 0, 0, 0, 0};
  if (opts) o = *opts;
  if (o.max_batch <= 0) o.max_batch = 8;
  if (o.max_batch > 16) return set_err(IG_EUNSUPPORTED, "max_batch > 16");
  if (o.prefetch_depth <= 0) o.prefetch_depth = 2;
  if (o.prefetch_depth + 1 > MAXR) return set_err(IG_EUNSUPPORTED, "prefetch_depth > %d", MAXR - 1);
  if (o.copy_mode < 0 || o.copy_mode > 2) return set_err(IG_EINVAL, "copy_mode must be 0, 1 or 2");
  if (o.cache_fp8 && desc->dtype != IG_BF16) return set_err(IG_EUNSUPPORTED, "FP8 caches need the bf16 mode");
  const int Lall = desc->txt_len + desc->grid_h * desc->grid_w;
  if (o.max_rows <= 0) o.max_rows = o.max_batch * Lall;
  if (desc->n_unet > 0) {
    o.max_rows = std::max(o.max_rows, o.max_batch * desc->ctx_len);  // the context rows' K/V projection
  }

  CUDA_TRY(cudaSetDevice(device));
  ig_ctx* ctx = new ig_ctx();
  ctx->d = *desc;
  ctx->o = o;
  ctx->device = device;
  ctx->esz = desc->dtype == IG_F32 ? 4 : 2;
  ctx->H = desc->hidden; ctx->F = desc->mlp_hidden; ctx->C = desc->lat_ch;
  ctx->Limg = desc->grid_h * desc->grid_w; ctx->Lt = desc->txt_len; ctx->L = Lall;
  ctx->nb = desc->n_double + desc->n_single + desc->n_unet;
  ctx->R = o.prefetch_depth + 1;
  ctx->w.assign(weights, weights + nw);
  const int H = ctx->H, F = ctx->F, C = ctx->C;

  // resolve the weight table (order documented in ig.h)
  int k = 0;
  auto lin = [&](LinW& l, int outd, int ind) { l.w = weights[k++]; l.b = weights[k++]; l.out = outd; l.in = ind; };
  std::vector<const void*> ln_ptrs;  // UNet: [nb][3][gamma, beta]
  ctx->unet.resize(desc->n_unet);
  for (int i = 0; i < desc->n_unet; ++i) {
    UnetW& u = ctx->unet[i];
    auto nobias = [&](LinW& l, int outd, int ind) { l.w = weights[k++]; l.out = outd; l.in = ind; };
    ln_ptrs.push_back(weights[k++]); ln_ptrs.push_back(weights[k++]);
    u.qkv = weights[k++];
    lin(u.out1, H, H);
    ln_ptrs.push_back(weights[k++]); ln_ptrs.push_back(weights[k++]);
    nobias(u.q2, H, H);
    nobias(u.kv2, 2 * H, desc->ctx_dim);
    lin(u.out2, H, H);
    ln_ptrs.push_back(weights[k++]); ln_ptrs.push_back(weights[k++]);
    lin(u.geglu, 2 * F, H);
    lin(u.ff2, H, F);
  }
  if (desc->n_unet == 0) {
  lin(ctx->img_in, H, C);
  lin(ctx->t1, H, 256);
  lin(ctx->t2, H, H);
  lin(ctx->fmod, 2 * H, H);
  lin(ctx->pout, C, H);
  if (desc->pos_embed_2d) ctx->pos_embed = weights[k++];
  ctx->dimg.resize(desc->n_double);
  ctx->dtxt.resize(desc->n_double);
  for (int i = 0; i < desc->n_double; ++i)
    for (int sidx = 0; sidx < 2; ++sidx) {
      StreamW& sw = sidx == 0 ? ctx->dimg[i] : ctx->dtxt[i];
      sw.pre_only = desc->context_pre_only_last && sidx == 1 && i == desc->n_double - 1;
      lin(sw.mod, (sw.pre_only ? 2 : 6) * H, H);
      lin(sw.qkv, 3 * H, H);
      if (desc->qk_norm) { sw.qg = weights[k++]; sw.kg = weights[k++]; }
      if (!sw.pre_only) { lin(sw.proj, H, H); lin(sw.fc1, F, H); lin(sw.fc2, H, F); }
    }
  ctx->sgl.resize(desc->n_single);
  for (int i = 0; i < desc->n_single; ++i) {
    SingleW& sw = ctx->sgl[i];
    lin(sw.mod, 3 * H, H);
    lin(sw.lin1, 3 * H + F, H);
    if (desc->qk_norm) { sw.qg = weights[k++]; sw.kg = weights[k++]; }
    lin(sw.lin2, H, H + F);
  }
  }  // n_unet == 0
  // modulation tensors and their offsets inside one request's modulation row
  auto add_mod = [&](const LinW* l, int kk) {
    ctx->mods.push_back({l, kk, ctx->mod_ld});
    ctx->mod_ld += (long long)kk * H;
    return (int)ctx->mods.size() - 1;
  };
  for (int i = 0; i < desc->n_double; ++i) {
    ctx->dimg[i].mod_t = add_mod(&ctx->dimg[i].mod, 6);
    if (ctx->Lt > 0) ctx->dtxt[i].mod_t = add_mod(&ctx->dtxt[i].mod, ctx->dtxt[i].pre_only ? 2 : 6);
  }
  for (int i = 0; i < desc->n_single; ++i) ctx->sgl[i].mod_t = add_mod(&ctx->sgl[i].mod, 3);
  if (desc->n_unet == 0) ctx->fmod_t = add_mod(&ctx->fmod, 2);

  // workspaces
  const long long Mx = o.max_rows, B = o.max_batch, es = (long long)ctx->esz;
  auto dmalloc = [&](void** p, size_t bytes) -> bool { return cudaMalloc(p, std::max<size_t>(bytes, 256)) == cudaSuccess; };
  bool okm = true;
  okm &= dmalloc((void**)&ctx->X, Mx * H * 4);
  okm &= dmalloc((void**)&ctx->vel, Mx * C * 4);
  okm &= dmalloc((void**)&ctx->temb, B * 256 * 4);
  okm &= dmalloc((void**)&ctx->tmp, B * H * 4);
  okm &= dmalloc((void**)&ctx->vec, B * H * 4);
  okm &= dmalloc((void**)&ctx->svec, B * H * 4);
  okm &= dmalloc((void**)&ctx->modbuf, B * ctx->mod_ld * 4);
  okm &= dmalloc(&ctx->h, Mx * H * es);
  okm &= dmalloc(&ctx->qkv, Mx * 3 * H * es);
  okm &= dmalloc(&ctx->Q, Mx * H * es);
  okm &= dmalloc(&ctx->cat, Mx * (H + F) * es);
  okm &= dmalloc(&ctx->Ain, Mx * C * es);
  okm &= dmalloc((void**)&ctx->ri, Mx * sizeof(RowInfo));
  ctx->buf_elems = 2LL * ctx->L * H;
  ctx->slot_stride = ctx->buf_elems * (ctx->R + 1);  // R ring buffers + 1 for dense-prefix blocks
  okm &= dmalloc(&ctx->kv_arena, (size_t)(B * ctx->slot_stride * es));
  if (!okm) { ig_ctx_destroy(ctx); return set_err(IG_ENOMEM, "workspace allocation failed"); }
  cudaMemset(ctx->kv_arena, 0, (size_t)(B * ctx->slot_stride * es));
  cudaMemset(ctx->X, 0, Mx * H * 4);
  if ((s = build_rope_table(ctx)) != IG_OK) { ig_ctx_destroy(ctx); return s; }
  if (desc->n_unet > 0) {  // UNet constants and buffers
    const int nbu = desc->n_unet, Lc = desc->ctx_len, Dc = desc->ctx_dim;
    okm &= dmalloc((void**)&ctx->unet_ln, (size_t)nbu * 3 * 2 * H * 4);
    okm &= dmalloc((void**)&ctx->ones, (size_t)H * 4);
    okm &= dmalloc(&ctx->xkv, (size_t)2 * B * 2 * Lc * H * es);  // two block-parity halves
    okm &= dmalloc(&ctx->ctxp, (size_t)B * Lc * Dc * es);
    okm &= dmalloc((void**)&ctx->ri_c, (size_t)B * Lc * sizeof(RowInfo));
    okm &= dmalloc(&ctx->u2, (size_t)Mx * 2 * F * es);
    const bool tc_geglu = desc->dtype == IG_BF16 && F % 128 == 0;
    if (tc_geglu) okm &= dmalloc(&ctx->geglu_tc, (size_t)nbu * 2 * F * (H + 1) * 2);
    if (!okm) { ig_ctx_destroy(ctx); return set_err(IG_ENOMEM, "UNet workspace allocation failed"); }
    // LN affine -> (shift = beta, scale = gamma - 1): LN(x) * (1 + scale) + shift == LN(x) * gamma + beta
    // (gamma - 1 is exact in fp32 for gamma in [0.5, 2], and 1 + (gamma - 1) == gamma there)
    std::vector<float> lnh((size_t)nbu * 3 * 2 * H), ones(H, 1.f);
    std::vector<char> tmp((size_t)H * es);
    for (int i = 0; i < nbu * 3; ++i) {
      for (int w = 0; w < 2; ++w) {
        CUDA_TRY(cudaMemcpy(tmp.data(), ln_ptrs[2 * i + w], (size_t)H * es, cudaMemcpyDeviceToHost));
        for (int c = 0; c < H; ++c) {
          float v;
          if (es == 4) v = reinterpret_cast<const float*>(tmp.data())[c];
          else { uint32_t b = (uint32_t)reinterpret_cast<const uint16_t*>(tmp.data())[c] << 16; memcpy(&v, &b, 4); }
          if (w == 0) lnh[(size_t)i * 2 * H + H + c] = v - 1.f;  // scale
          else lnh[(size_t)i * 2 * H + c] = v;                   // shift
        }
      }
    }
    CUDA_TRY(cudaMemcpy(ctx->unet_ln, lnh.data(), lnh.size() * 4, cudaMemcpyHostToDevice));
    cudaStreamCreateWithFlags(&ctx->xs, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&ctx->ev_xfork, cudaEventDisableTiming);
    for (int i = 0; i < 2; ++i) {
      cudaEventCreateWithFlags(&ctx->ev_xkv[i], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&ctx->ev_xuse[i], cudaEventDisableTiming);
    }
    CUDA_TRY(cudaMemcpy(ctx->ones, ones.data(), (size_t)H * 4, cudaMemcpyHostToDevice));
    std::vector<RowInfo> ric((size_t)B * Lc);
    for (int q = 0; q < B; ++q)
      for (int j = 0; j < Lc; ++j) ric[(size_t)q * Lc + j] = RowInfo{q, q, j, -1};
    CUDA_TRY(cudaMemcpy(ctx->ri_c, ric.data(), ric.size() * sizeof(RowInfo), cudaMemcpyHostToDevice));
    if (tc_geglu)
      for (int i = 0; i < nbu; ++i) {
        bf16* wd = (bf16*)ctx->geglu_tc + (size_t)i * 2 * F * (H + 1);
        bf16* bd = wd + (size_t)2 * F * H;
        launch_permute_geglu_rows((const bf16*)ctx->unet[i].geglu.w, wd, F, H, 0);
        launch_permute_geglu_rows((const bf16*)ctx->unet[i].geglu.b, bd, F, 1, 0);
        ctx->unet[i].geglu_w_tc = wd;
        ctx->unet[i].geglu_b_tc = bd;
      }
  }

  // static GEMV problem lists (a3)
  std::vector<GemvProb> p1(1), p2(1);
  p1[0] = GemvProb{ctx->t1.w, ctx->t1.b, ctx->temb, ctx->tmp, nullptr, H, 256, 256, H, 0, 1, 0};
  p2[0] = GemvProb{ctx->t2.w, ctx->t2.b, ctx->tmp, ctx->vec, nullptr, H, H, H, H, 0, 0, 0};
  constexpr int ROWS_PER_GROUP = 32;
  int groups = 0;
  for (auto& m : ctx->mods) {
    GemvProb g{m.w->w, m.w->b, ctx->svec, ctx->modbuf + m.off, nullptr, m.k * H, H, H,
               (int)ctx->mod_ld, 0, 0, groups};
    groups += (g.N + ROWS_PER_GROUP - 1) / ROWS_PER_GROUP;
    ctx->gv_mod_host.push_back(g);
  }
  ctx->gv_mod_groups = groups;
  if (desc->dtype == IG_BF16) {
    okm &= dmalloc(&ctx->modw, (size_t)ctx->mod_ld * H * 2);
    okm &= dmalloc(&ctx->modb, (size_t)ctx->mod_ld * 2);
    okm &= dmalloc((void**)&ctx->svec_bf, (size_t)B * H * 2);
    if (!okm) { ig_ctx_destroy(ctx); return set_err(IG_ENOMEM, "modulation pack allocation failed"); }
    for (auto& m : ctx->mods) {
      cudaMemcpy((char*)ctx->modw + (size_t)m.off * H * 2, m.w->w, (size_t)m.k * H * H * 2, cudaMemcpyDeviceToDevice);
      cudaMemcpy((char*)ctx->modb + (size_t)m.off * 2, m.w->b, (size_t)m.k * H * 2, cudaMemcpyDeviceToDevice);
    }
  }
  okm &= dmalloc((void**)&ctx->gv_t1, sizeof(GemvProb));
  okm &= dmalloc((void**)&ctx->gv_t2, sizeof(GemvProb));
  okm &= dmalloc((void**)&ctx->gv_mod, ctx->gv_mod_host.size() * sizeof(GemvProb));
  if (!okm) { ig_ctx_destroy(ctx); return set_err(IG_ENOMEM, "workspace allocation failed"); }
  cudaMemcpy(ctx->gv_t1, p1.data(), sizeof(GemvProb), cudaMemcpyHostToDevice);
  cudaMemcpy(ctx->gv_t2, p2.data(), sizeof(GemvProb), cudaMemcpyHostToDevice);
  cudaMemcpy(ctx->gv_mod, ctx->gv_mod_host.data(), ctx->gv_mod_host.size() * sizeof(GemvProb),
             cudaMemcpyHostToDevice);

  if (o.cache_fp8) {
    const size_t pl = (size_t)ctx->Limg * H, spl = (size_t)ctx->Limg * desc->heads;
    okm &= dmalloc((void**)&ctx->q8in, (size_t)B * ctx->R * 2 * pl);
    okm &= dmalloc((void**)&ctx->q8in_scl, (size_t)B * ctx->R * 2 * spl * 4);
    okm &= dmalloc((void**)&ctx->q8rec, (size_t)ctx->R * 2 * pl);
    okm &= dmalloc((void**)&ctx->q8rec_scl, (size_t)ctx->R * 2 * spl * 4);
    if (!okm) { ig_ctx_destroy(ctx); return set_err(IG_ENOMEM, "fp8 staging allocation failed"); }
  }
  if (o.cache_y && o.cache_fp8) {
    okm &= dmalloc((void**)&ctx->q8yrec, (size_t)ctx->R * 2 * ctx->Limg * H);
    okm &= dmalloc((void**)&ctx->q8yrec_scl, (size_t)ctx->R * 2 * ctx->Limg * desc->heads * 4);
  }
  if (o.cache_y) {
    okm &= dmalloc(&ctx->yrec, (size_t)ctx->R * ctx->Limg * H * es);
    if (!okm) { ig_ctx_destroy(ctx); return set_err(IG_ENOMEM, "Y recording staging allocation failed"); }
  }
  // per-step descriptor staging: ReqDev[B] + AttnSeg[2B] + 2 x KvGatherReq[nb * B]
  ctx->stage_bytes = B * sizeof(ReqDev) + 8 * B * sizeof(AttnSeg) + 2 * (size_t)ctx->nb * B * sizeof(KvGatherReq) + 1024;
  for (int i = 0; i < NSTAGE; ++i) {
    if (cudaHostAlloc((void**)&ctx->h_stage[i], ctx->stage_bytes, cudaHostAllocMapped | cudaHostAllocPortable) !=
            cudaSuccess ||
        cudaHostGetDevicePointer((void**)&ctx->m_stage[i], ctx->h_stage[i], 0) != cudaSuccess ||
        cudaMalloc((void**)&ctx->d_stage[i], ctx->stage_bytes) != cudaSuccess) {
      ig_ctx_destroy(ctx);
      return set_err(IG_ENOMEM, "staging allocation failed");
    }
    cudaEventCreateWithFlags(&ctx->ev_stage[i], cudaEventDisableTiming);
  }
  if (cudaMalloc((void**)&ctx->d_gstage, ctx->stage_bytes) != cudaSuccess) {
    ig_ctx_destroy(ctx);
    return set_err(IG_ENOMEM, "staging allocation failed");
  }
  cudaStreamCreateWithFlags(&ctx->copy_st, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&ctx->ts, cudaStreamNonBlocking);
  for (int i = 0; i < 2; ++i) {
    cudaEventCreateWithFlags(&ctx->ev_tfork[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->ev_tjoin[i], cudaEventDisableTiming);
  }
  for (int i = 0; i < MAXR; ++i) {
    cudaEventCreateWithFlags(&ctx->ev_copy[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->ev_comp[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->ev_yrec[i], cudaEventDisableTiming);
  }
  cudaEventCreateWithFlags(&ctx->ev_desc, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming);
  ctx->pref.assign((size_t)B * ctx->R, ig_ctx::Pref{});
  if (desc->dtype == IG_BF16) { gemm_tc_init(); attn_tc_init(); }  // before any graph capture
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { ig_ctx_destroy(ctx); return set_err(IG_ECUDA, "ctx init: %s", cudaGetErrorString(e)); }
  *out = ctx;
  return IG_OK;
}

extern "C" void ig_ctx_destroy(ig_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  lane_stop(ctx);
  cudaDeviceSynchronize();  // every enqueued step (and its unpin callback) has finished
  reap_zombies(ctx);
  void* bufs[] = {ctx->X, ctx->vel, ctx->temb, ctx->tmp, ctx->vec, ctx->svec, ctx->modbuf, ctx->h,
                  ctx->qkv, ctx->Q, ctx->cat, ctx->Ain, ctx->ri, ctx->kv_arena, ctx->rope_tab,
                  ctx->gv_t1, ctx->gv_t2, ctx->gv_mod, ctx->modw, ctx->modb, ctx->svec_bf,
                  ctx->q8in, ctx->q8in_scl, ctx->q8rec, ctx->q8rec_scl, ctx->yrec, ctx->unet_ln,
                  ctx->ones, ctx->xkv, ctx->ctxp, ctx->ri_c, ctx->u2, ctx->geglu_tc,
                  ctx->q8yrec, ctx->q8yrec_scl};
  for (void* b : bufs) if (b) cudaFree(b);
  for (int i = 0; i < NSTAGE; ++i) {
    if (ctx->h_stage[i]) cudaFreeHost(ctx->h_stage[i]);
    if (ctx->d_stage[i]) cudaFree(ctx->d_stage[i]);
    if (ctx->ev_stage[i]) cudaEventDestroy(ctx->ev_stage[i]);
  }
  if (ctx->d_gstage) cudaFree(ctx->d_gstage);
  for (int i = 0; i < MAXR; ++i) {
    if (ctx->ev_copy[i]) cudaEventDestroy(ctx->ev_copy[i]);
    if (ctx->ev_comp[i]) cudaEventDestroy(ctx->ev_comp[i]);
    if (ctx->ev_yrec[i]) cudaEventDestroy(ctx->ev_yrec[i]);
  }
  if (ctx->ev_desc) cudaEventDestroy(ctx->ev_desc);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->xs) cudaStreamDestroy(ctx->xs);
  if (ctx->ts) cudaStreamDestroy(ctx->ts);
  for (int i = 0; i < 2; ++i) {
    if (ctx->ev_tfork[i]) cudaEventDestroy(ctx->ev_tfork[i]);
    if (ctx->ev_tjoin[i]) cudaEventDestroy(ctx->ev_tjoin[i]);
  }
  if (ctx->ev_xfork) cudaEventDestroy(ctx->ev_xfork);
  for (int i = 0; i < 2; ++i) {
    if (ctx->ev_xkv[i]) cudaEventDestroy(ctx->ev_xkv[i]);
    if (ctx->ev_xuse[i]) cudaEventDestroy(ctx->ev_xuse[i]);
  }
  for (auto& g : ctx->graphs) cudaGraphExecDestroy(g.second.exec);
  for (auto& r : ctx->prof_recs) { ctx->ev_pool.push_back(r.a); ctx->ev_pool.push_back(r.b); }
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->copy_st) cudaStreamDestroy(ctx->copy_st);
  if (ctx->ones_mask) ig_mask_free(ctx->ones_mask);
  delete ctx;
}

extern "C" ig_status ig_profile_enable(ig_ctx* ctx, int enable) {
  if (!ctx) return set_err(IG_EINVAL, "ctx is NULL");
  ctx->prof = enable != 0;
  if (ctx->prof) {  // time origin of the IG_PROFILE_DUMP timeline
    if (!ctx->prof_t0) cudaEventCreate(&ctx->prof_t0);
    cudaEventRecord(ctx->prof_t0, ctx->copy_st);
  }
  return IG_OK;
}

extern "C" ig_status ig_profile_read(ig_ctx* ctx, ig_prof_entry out[IG_K_NCLASS]) {
  if (!ctx || !out) return set_err(IG_EINVAL, "NULL argument");
  CUDA_TRY(cudaSetDevice(ctx->device));
  const char* dump = getenv("IG_PROFILE_DUMP");
  FILE* fd = dump ? fopen(dump, "a") : nullptr;
  for (auto& r : ctx->prof_recs) {
    CUDA_TRY(cudaEventSynchronize(r.b));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, r.a, r.b));
    if (fd) {
      float t0 = 0.f;
      if (ctx->prof_t0) cudaEventElapsedTime(&t0, ctx->prof_t0, r.a);
      fprintf(fd, "%d,%d,%d,%d,%d,%.6f,%.6g,%.6g,%.4f\n", r.kind, r.M, r.N, r.K, r.epi, ms, r.flops, r.bytes, t0);
    }
    ig_prof_entry& e = ctx->prof_acc[r.kind];
    e.launches++;
    e.ms += ms;
    e.flops += r.flops;
    e.bytes += r.bytes;
    ctx->ev_pool.push_back(r.a);
    ctx->ev_pool.push_back(r.b);
  }
  if (fd) fclose(fd);
  ctx->prof_recs.clear();
  for (int k = 0; k < IG_K_NCLASS; ++k) out[k] = ctx->prof_acc[k];
  for (int k = 0; k < IG_K_NCLASS; ++k) ctx->prof_acc[k] = ig_prof_entry{};
  return IG_OK;
}

extern "C" ig_status ig_plan_copy_groups(const uint8_t* mask, int L, int W, int row_bytes, int* groups, int cap,
                                         int* n_groups) {
  if (!mask || !n_groups || L <= 0 || W < 0 || row_bytes <= 0 || cap < 0 || (cap > 0 && !groups))
    return set_err(IG_EINVAL, "bad argument");
  std::vector<std::pair<int, int>> runs;
  for (int i = 0; i < L;) {
    if (mask[i]) { ++i; continue; }
    int j = i;
    while (j < L && !mask[j]) ++j;
    runs.push_back({i, j - i});
    i = j;
  }
  std::vector<CopyGroup> g;
  make_copy_groups(runs, L, W, copy_call_rows((size_t)row_bytes, 2), g);
  *n_groups = (int)g.size();
  if ((int)g.size() > cap) return set_err(IG_EINVAL, "%d groups exceed cap %d", (int)g.size(), cap);
  for (size_t k = 0; k < g.size(); ++k) {
    groups[4 * k + 0] = g[k].start;
    groups[4 * k + 1] = g[k].len;
    groups[4 * k + 2] = g[k].stride;
    groups[4 * k + 3] = g[k].count;
  }
  return IG_OK;
}

extern "C" ig_status ig_last_stats(const ig_ctx* ctx, ig_stats* out) {
  if (!ctx || !out) return set_err(IG_EINVAL, "NULL argument");
  *out = ctx->stats;
  return IG_OK;
}

// ----------------------------------------------------------------------------------------
// masks (a1): kernel (a) builds idx_m / idx_u on the device; n_m comes back with one sync
// at admission (CS5), never on the step path.
// ----------------------------------------------------------------------------------------
extern "C" ig_status ig_mask_build(ig_ctx* ctx, const uint8_t* mask, void* stream, ig_mask** out,
                                   int* n_masked) {
  if (!ctx || !mask || !out) return set_err(IG_EINVAL, "NULL argument");
  *out = nullptr;
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = (cudaStream_t)stream;
  ig_mask* m = new ig_mask();
  m->L_img = ctx->Limg;
  if (cudaMalloc(&m->idx, (2 * ctx->Limg + 1) * sizeof(int32_t)) != cudaSuccess) {
    delete m;
    return set_err(IG_ENOMEM, "mask index allocation failed");
  }
  launch_mask_index(mask, ctx->Limg, m->idx, m->idx + ctx->Limg, m->idx + 2 * ctx->Limg, st);
  int32_t n = 0;
  std::vector<uint8_t> hm(ctx->Limg);
  cudaError_t e = cudaMemcpyAsync(&n, m->idx + 2 * ctx->Limg, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(hm.data(), mask, ctx->Limg, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  for (auto& v : hm) v = v != 0;
  m->bits = hm;
  if (e == cudaSuccess) e = cudaMalloc(&m->bits_dev, ctx->Limg);
  if (e == cudaSuccess) e = cudaMemcpy(m->bits_dev, hm.data(), ctx->Limg, cudaMemcpyHostToDevice);
  for (int i = 0; i < ctx->Limg;) {  // unmasked runs for the compacted DMA copy (copy_mode 1)
    if (hm[i]) { ++i; continue; }
    int j = i;
    while (j < ctx->Limg && !hm[j]) ++j;
    m->runs.push_back({i, j - i});
    i = j;
  }
  m->dma_rows = make_copy_groups(m->runs, ctx->Limg, ctx->d.grid_w, copy_call_rows((size_t)ctx->H * ctx->esz, 2),
                                 m->groups);
  if (e != cudaSuccess) {
    cudaFree(m->idx);
    if (m->bits_dev) cudaFree(m->bits_dev);
    delete m;
    return set_err(IG_ECUDA, "mask build: %s", cudaGetErrorString(e));
  }
  m->n_m = n;
  if (n_masked) *n_masked = n;
  *out = m;
  return IG_OK;
}

extern "C" ig_status ig_mask_indices(const ig_mask* m, const int32_t** idx_m, const int32_t** idx_u,
                                     int* n_m) {
  if (!m) return set_err(IG_EINVAL, "mask is NULL");
  if (idx_m) *idx_m = m->idx;
  if (idx_u) *idx_u = m->idx + m->L_img;
  if (n_m) *n_m = m->n_m;
  return IG_OK;
}

// host-bitmap mask build for a token grid of L tokens (also used by the whole-UNet runtime for
// its per-level masks, ig_internal.h)
ig_status ig_mask_build_host_L(int device, int L, const uint8_t* mask, void* stream, ig_mask** out, int* n_masked,
                               int W, int row_bytes) {
  if (!mask || !out || L <= 0) return set_err(IG_EINVAL, "NULL argument");
  *out = nullptr;
  CUDA_TRY(cudaSetDevice(device));
  cudaStream_t st = (cudaStream_t)stream;
  ig_mask* m = new ig_mask();
  m->L_img = L;
  m->bits.resize(L);
  int n = 0;
  for (int i = 0; i < L; ++i) { m->bits[i] = mask[i] != 0; n += m->bits[i]; }
  for (int i = 0; i < L;) {  // unmasked runs for the compacted DMA copy (copy_mode 1)
    if (m->bits[i]) { ++i; continue; }
    int j = i;
    while (j < L && !m->bits[j]) ++j;
    m->runs.push_back({i, j - i});
    i = j;
  }
  m->dma_rows = make_copy_groups(m->runs, L, W, copy_call_rows(row_bytes > 0 ? (size_t)row_bytes : 6144, 2), m->groups);
  // one stream-ordered allocation: idx_m | idx_u | n_m (int32), then the bitmap (u8)
  const size_t idx_bytes = ((size_t)(2 * L + 1) * sizeof(int32_t) + 15) & ~(size_t)15;
  void* base = nullptr;
  cudaError_t e = cudaMallocAsync(&base, idx_bytes + L, st);
  if (e == cudaSuccess) {
    m->idx = (int32_t*)base;
    m->bits_dev = (uint8_t*)base + idx_bytes;
    // pageable source: the call returns once the bytes are staged (no device sync)
    e = cudaMemcpyAsync(m->bits_dev, m->bits.data(), L, cudaMemcpyHostToDevice, st);
  }
  if (e != cudaSuccess) {
    if (base) cudaFreeAsync(base, st);
    delete m;
    return set_err(IG_ECUDA, "mask build: %s", cudaGetErrorString(e));
  }
  launch_mask_index(m->bits_dev, L, m->idx, m->idx + L, m->idx + 2 * L, st);
  m->async_alloc = true;
  m->build_st = st;
  m->n_m = n;
  if (n_masked) *n_masked = n;
  *out = m;
  return IG_OK;
}

extern "C" ig_status ig_mask_build_host(ig_ctx* ctx, const uint8_t* mask, void* stream, ig_mask** out,
                                        int* n_masked) {
  if (!ctx) return set_err(IG_EINVAL, "NULL argument");
  return ig_mask_build_host_L(ctx->device, ctx->Limg, mask, stream, out, n_masked, ctx->d.grid_w,
                              (int)(ctx->H * ctx->esz));
}

extern "C" void ig_mask_free(ig_mask* m) {
  if (!m) return;
  if (m->async_alloc) {  // stream-ordered: after the last step that read the mask (no device sync)
    cudaFreeAsync(m->idx, m->used ? m->last_st : m->build_st);
  } else {
    cudaFree(m->idx);
    if (m->bits_dev) cudaFree(m->bits_dev);
  }
  delete m;
}

static ig_status get_ones_mask(ig_ctx* ctx, ig_mask** out) {
  if (!ctx->ones_mask) {
    uint8_t* ones = nullptr;
    CUDA_TRY(cudaMalloc(&ones, ctx->Limg));
    CUDA_TRY(cudaMemset(ones, 1, ctx->Limg));
    ig_status s = ig_mask_build(ctx, ones, nullptr, &ctx->ones_mask, nullptr);
    cudaFree(ones);
    if (s != IG_OK) return s;
  }
  *out = ctx->ones_mask;
  return IG_OK;
}

// ----------------------------------------------------------------------------------------
// caches
// ----------------------------------------------------------------------------------------
// Which blocks of a hybrid cache are Y blocks (ig.h cache_kv_blocks): the first N - kv_blocks
// blocks of the bit-reversal order over the next power of two >= N (values >= N skipped), so
// Y blocks are spread evenly over the step (the copy lane sees a locally balanced mix) and the
// Y-block sets of different splits are nested.
static std::vector<uint8_t> y_modes(int N, int y, int kv_blocks) {
  std::vector<uint8_t> m(N, 0);
  if (!y) return m;
  int bits = 0;
  while ((1 << bits) < N) ++bits;
  int taken = 0;
  const int ny = N - std::max(0, std::min(kv_blocks, N));
  for (int k = 0; k < (1 << bits) && taken < ny; ++k) {
    int v = 0;
    for (int i = 0; i < bits; ++i) v |= ((k >> i) & 1) << (bits - 1 - i);
    if (v < N) { m[v] = 1; ++taken; }
  }
  return m;
}
static inline bool blk_kv(const std::vector<uint8_t>& m, int b) { return !m[b]; }
static inline bool blk_yrec(const std::vector<uint8_t>& m, int b) {
  return m[b] || (b + 1 < (int)m.size() && m[b + 1]);
}
static int planes_of(const std::vector<uint8_t>& m, int b) { return (blk_kv(m, b) ? 2 : 0) + (blk_yrec(m, b) ? 1 : 0); }
static int step_planes(const std::vector<uint8_t>& m) {
  int n = 0;
  for (int b = 0; b < (int)m.size(); ++b) n += planes_of(m, b);
  return n;
}
static size_t cache_kv_bytes(const ig_ctx* ctx, int n_steps, int fp8, const std::vector<uint8_t>& m) {
  if (fp8) return (size_t)n_steps * step_planes(m) * ctx->Limg * ((size_t)ctx->H + 4 * ctx->d.heads);
  return (size_t)n_steps * step_planes(m) * ctx->Limg * ctx->H * ctx->esz;
}
static size_t cache_bytes(const ig_ctx* ctx, int n_steps, int fp8, const std::vector<uint8_t>& m) {
  return cache_kv_bytes(ctx, n_steps, fp8, m) + (size_t)n_steps * ctx->Limg * ctx->C * 4;
}
static float* cache_latent(const ig_ctx* ctx, const ig_cache* c, int step) {
  return (float*)((char*)c->ptr + c->lat_off + (size_t)step * ctx->Limg * ctx->C * 4);
}
static const float* cache_latent_dev(const ig_ctx* ctx, const ig_cache* c, int step) {
  return (const float*)((const char*)c->dptr + ((char*)cache_latent(ctx, c, step) - (char*)c->ptr));
}
// data plane (which = 0 K, 1 V, 2 Y) of (step, block) and its scale plane (fp8 caches)
static size_t plane_index(const ig_ctx* ctx, const ig_cache* c, int step, int b, int which) {
  if (!c->y) return ((size_t)step * ctx->nb + b) * 2 + which;
  size_t idx = (size_t)step * c->step_planes;
  for (int bb = 0; bb < b; ++bb) idx += planes_of(c->ymode, bb);
  if (which == 2) idx += blk_kv(c->ymode, b) ? 2 : 0;
  else idx += which;
  return idx;
}
static char* cache_plane(const ig_ctx* ctx, const ig_cache* c, int step, int b, int which) {
  const size_t row = c->fp8 ? (size_t)ctx->H : (size_t)ctx->H * ctx->esz;
  return (char*)c->ptr + plane_index(ctx, c, step, b, which) * ctx->Limg * row;
}
// block b of a request on cache c runs as a Y block (unmasked rows replenished, K/V recomputed)
static inline bool y_block(const ig_cache* c, int b) { return c && c->y && c->ymode[b]; }
static float* cache_scales(const ig_ctx* ctx, const ig_cache* c, int step, int b, int which) {
  return (float*)((char*)c->ptr + c->scale_off + plane_index(ctx, c, step, b, which) * ctx->Limg * ctx->d.heads * 4);
}
static const char* cache_plane_dev(const ig_ctx* ctx, const ig_cache* c, int step, int b, int which) {
  return (const char*)c->dptr + (cache_plane(ctx, c, step, b, which) - (char*)c->ptr);
}
static const float* cache_scales_dev(const ig_ctx* ctx, const ig_cache* c, int step, int b, int which) {
  return (const float*)((const char*)c->dptr + ((char*)cache_scales(ctx, c, step, b, which) - (char*)c->ptr));
}

static ig_status cache_create_kind(ig_ctx* ctx, int n_steps, int tier, int fp8, int y, int kv_blocks, ig_cache** out);
extern "C" ig_status ig_cache_create(ig_ctx* ctx, int n_steps, int tier, ig_cache** out) {
  if (!ctx || !out) return set_err(IG_EINVAL, "NULL argument");
  return cache_create_kind(ctx, n_steps, tier, ctx->o.cache_fp8, ctx->o.cache_y, ctx->o.cache_kv_blocks, out);
}

static ig_status cache_create_kind(ig_ctx* ctx, int n_steps, int tier, int fp8, int y, int kv_blocks, ig_cache** out) {
  *out = nullptr;
  if (n_steps <= 0) return set_err(IG_EINVAL, "n_steps must be positive");
  if (tier != IG_CACHE_HOST && tier != IG_CACHE_DEVICE) return set_err(IG_EINVAL, "bad tier");
  CUDA_TRY(cudaSetDevice(ctx->device));
  ig_cache* c = new ig_cache();
  c->desc = ctx->d;
  c->n_steps = n_steps;
  c->tier = tier;
  c->device = ctx->device;
  c->fp8 = fp8;
  c->y = y;
  c->kv_blocks = y ? std::max(0, std::min(kv_blocks, ctx->nb)) : ctx->nb;
  c->ymode = y_modes(ctx->nb, y, c->kv_blocks);
  c->step_planes = step_planes(c->ymode);
  c->bytes = cache_bytes(ctx, n_steps, c->fp8, c->ymode);
  if (c->fp8) c->scale_off = (size_t)n_steps * c->step_planes * ctx->Limg * ctx->H;
  c->lat_off = cache_kv_bytes(ctx, n_steps, c->fp8, c->ymode);
  cudaError_t e;
  if (tier == IG_CACHE_HOST) {
    e = cudaHostAlloc(&c->ptr, c->bytes, cudaHostAllocMapped | cudaHostAllocPortable);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer(&c->dptr, c->ptr, 0);
  } else {
    e = cudaMalloc(&c->ptr, c->bytes);
    c->dptr = c->ptr;
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    if (c->ptr) { if (tier == IG_CACHE_HOST) cudaFreeHost(c->ptr); else cudaFree(c->ptr); }
    const size_t bytes = c->bytes;
    delete c;
    return set_err(IG_ENOMEM, "cache allocation of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
  }
  *out = c;
  return IG_OK;
}

extern "C" ig_status ig_cache_bytes(const ig_ctx* ctx, int n_steps, size_t* bytes) {
  if (!ctx || !bytes) return set_err(IG_EINVAL, "NULL argument");
  if (n_steps <= 0) return set_err(IG_EINVAL, "n_steps must be positive");
  const std::vector<uint8_t> m = y_modes(ctx->nb, ctx->o.cache_y, ctx->o.cache_y ? ctx->o.cache_kv_blocks : ctx->nb);
  *bytes = cache_bytes(ctx, n_steps, ctx->o.cache_fp8, m);
  return IG_OK;
}

extern "C" ig_status ig_cache_attach(ig_ctx* ctx, int n_steps, void* host_mem, size_t bytes, ig_cache** out) {
  if (!ctx || !host_mem || !out) return set_err(IG_EINVAL, "NULL argument");
  *out = nullptr;
  if (n_steps <= 0) return set_err(IG_EINVAL, "n_steps must be positive");
  size_t need = 0;
  ig_status s = ig_cache_bytes(ctx, n_steps, &need);
  if (s != IG_OK) return s;
  if (bytes < need) return set_err(IG_EINVAL, "host_mem holds %zu bytes, the cache needs %zu", bytes, need);
  CUDA_TRY(cudaSetDevice(ctx->device));
  ig_cache* c = new ig_cache();
  c->desc = ctx->d;
  c->n_steps = n_steps;
  c->tier = IG_CACHE_HOST;
  c->device = ctx->device;
  c->fp8 = ctx->o.cache_fp8;
  c->y = ctx->o.cache_y;
  c->kv_blocks = c->y ? std::max(0, std::min(ctx->o.cache_kv_blocks, ctx->nb)) : ctx->nb;
  c->ymode = y_modes(ctx->nb, c->y, c->kv_blocks);
  c->step_planes = step_planes(c->ymode);
  c->bytes = need;
  if (c->fp8) c->scale_off = (size_t)n_steps * c->step_planes * ctx->Limg * ctx->H;
  c->lat_off = cache_kv_bytes(ctx, n_steps, c->fp8, c->ymode);
  cudaError_t e = cudaHostRegister(host_mem, need, cudaHostRegisterMapped | cudaHostRegisterPortable);
  if (e == cudaSuccess) e = cudaHostGetDevicePointer(&c->dptr, host_mem, 0);
  if (e != cudaSuccess) {
    cudaGetLastError();
    delete c;
    return set_err(IG_ECUDA, "cudaHostRegister of %zu bytes failed: %s", need, cudaGetErrorString(e));
  }
  c->ptr = host_mem;
  c->registered = true;
  *out = c;
  return IG_OK;
}

// ---- peer-HBM template pool: a device-tier cache held in one GPU's HBM, opened by
// the processes of the other GPUs through CUDA IPC and read over NVLink (peer access) by the
// copy lane's gather kernel instead of crossing the host link
typedef struct { char bytes[64]; } ig_ipc_raw;
static_assert(sizeof(cudaIpcMemHandle_t) <= 64, "IPC handle size");

extern "C" ig_status ig_cache_export(const ig_cache* c, void* handle, size_t handle_bytes) {
  if (!c || !handle) return set_err(IG_EINVAL, "NULL argument");
  if (handle_bytes < IG_CACHE_HANDLE_BYTES) return set_err(IG_EINVAL, "handle buffer < %d bytes", IG_CACHE_HANDLE_BYTES);
  if (c->tier != IG_CACHE_DEVICE || c->imported || c->registered)
    return set_err(IG_EINVAL, "only an HBM-tier cache allocated by this process can be exported");
  CUDA_TRY(cudaSetDevice(c->device));
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, c->ptr));
  // layout: IPC handle, then the schedule length, the storage device and the byte count
  memset(handle, 0, IG_CACHE_HANDLE_BYTES);
  memcpy(handle, &h, sizeof(h));
  int32_t meta[2] = {c->n_steps, c->device};
  memcpy((char*)handle + 64, meta, sizeof(meta));
  uint64_t by = c->bytes;
  memcpy((char*)handle + 72, &by, sizeof(by));
  return IG_OK;
}

extern "C" ig_status ig_cache_import(ig_ctx* ctx, const void* handle, ig_cache** out) {
  if (!ctx || !handle || !out) return set_err(IG_EINVAL, "NULL argument");
  *out = nullptr;
  int32_t meta[2];
  memcpy(meta, (const char*)handle + 64, sizeof(meta));
  uint64_t by = 0;
  memcpy(&by, (const char*)handle + 72, sizeof(by));
  const int n_steps = meta[0], owner = meta[1];
  if (n_steps <= 0) return set_err(IG_EINVAL, "bad cache handle");
  size_t need = 0;
  ig_status s = ig_cache_bytes(ctx, n_steps, &need);
  if (s != IG_OK) return s;
  if ((size_t)by != need)
    return set_err(IG_ECACHE_INCOMPAT, "exported cache holds %llu bytes, this ctx's cache kind needs %zu",
                   (unsigned long long)by, need);
  CUDA_TRY(cudaSetDevice(ctx->device));
  if (owner != ctx->device) {  // read the peer's HBM over NVLink: enable peer access (idempotent)
    int can = 0;
    CUDA_TRY(cudaDeviceCanAccessPeer(&can, ctx->device, owner));
    if (!can) return set_err(IG_EUNSUPPORTED, "device %d cannot access peer %d", ctx->device, owner);
    cudaError_t pe = cudaDeviceEnablePeerAccess(owner, 0);
    if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) return set_err(IG_ECUDA, "peer access: %s", cudaGetErrorString(pe));
    cudaGetLastError();
  }
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* p = nullptr;
  CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  ig_cache* c = new ig_cache();
  c->desc = ctx->d;
  c->n_steps = n_steps;
  c->tier = IG_CACHE_DEVICE;
  c->device = ctx->device;
  c->owner_device = owner;
  c->fp8 = ctx->o.cache_fp8;
  c->y = ctx->o.cache_y;
  c->kv_blocks = c->y ? std::max(0, std::min(ctx->o.cache_kv_blocks, ctx->nb)) : ctx->nb;
  c->ymode = y_modes(ctx->nb, c->y, c->kv_blocks);
  c->step_planes = step_planes(c->ymode);
  c->bytes = need;
  if (c->fp8) c->scale_off = (size_t)n_steps * c->step_planes * ctx->Limg * ctx->H;
  c->lat_off = cache_kv_bytes(ctx, n_steps, c->fp8, c->ymode);
  c->ptr = c->dptr = p;
  c->imported = true;
  *out = c;
  return IG_OK;
}

extern "C" ig_status ig_cache_clone(ig_ctx* ctx, const ig_cache* src, int tier, ig_cache** out) {
  if (!ctx || !src || !out) return set_err(IG_EINVAL, "NULL argument");
  *out = nullptr;
  if (!desc_equal(src->desc, ctx->d)) return set_err(IG_ECACHE_INCOMPAT, "cache built for another model");
  const bool quantize = ctx->o.cache_fp8 && !src->fp8;  // bf16 -> fp8 conversion
  if (!ctx->o.cache_fp8 && src->fp8) return set_err(IG_EUNSUPPORTED, "cannot clone an fp8 cache into bf16");
  CUDA_TRY(cudaSetDevice(ctx->device));
  ig_cache* c = nullptr;
  ig_status s = cache_create_kind(ctx, src->n_steps, tier, quantize ? 1 : src->fp8, src->y, src->kv_blocks, &c);
  if (s != IG_OK) return s;
  cudaError_t e = cudaSuccess;
  if (!quantize) {
    e = cudaMemcpy(c->ptr, src->ptr, src->bytes, cudaMemcpyDefault);
  } else if (src->y) {  // Y / hybrid: every plane in storage order -> quantize -> destination
    const size_t pl = (size_t)ctx->Limg * ctx->H, spl = (size_t)ctx->Limg * ctx->d.heads;
    void* tmp = nullptr;
    e = cudaMalloc(&tmp, pl * 2);
    const size_t np = (size_t)src->n_steps * src->step_planes;
    for (size_t i = 0; i < np && e == cudaSuccess; ++i) {
      e = cudaMemcpy(tmp, (const char*)src->ptr + i * pl * 2, pl * 2, cudaMemcpyDefault);
      if (e != cudaSuccess) break;
      launch_kv_quant((const bf16*)tmp, (const bf16*)tmp, ctx->Limg, ctx->H, ctx->d.heads, ctx->q8rec, ctx->q8rec + pl,
                      ctx->q8rec_scl, ctx->q8rec_scl + spl, 0);
      e = cudaMemcpy((char*)c->ptr + i * pl, ctx->q8rec, pl, cudaMemcpyDefault);
      if (e == cudaSuccess)
        e = cudaMemcpy((char*)c->ptr + c->scale_off + i * spl * 4, ctx->q8rec_scl, spl * 4, cudaMemcpyDefault);
    }
    if (tmp) cudaFree(tmp);
    if (e == cudaSuccess)
      e = cudaMemcpy(cache_latent(ctx, c, 0), cache_latent(ctx, src, 0), (size_t)src->n_steps * ctx->Limg * ctx->C * 4,
                     cudaMemcpyDefault);
  } else {  // per (step, block): bf16 planes -> device temp -> quantize -> destination
    const size_t pl = (size_t)ctx->Limg * ctx->H, spl = (size_t)ctx->Limg * ctx->d.heads;
    void* tmp = nullptr;
    e = cudaMalloc(&tmp, 2 * pl * 2);
    for (int st = 0; st < src->n_steps && e == cudaSuccess; ++st)
      for (int b = 0; b < ctx->nb && e == cudaSuccess; ++b) {
        e = cudaMemcpy(tmp, cache_plane(ctx, src, st, b, 0), 2 * pl * 2, cudaMemcpyDefault);
        if (e != cudaSuccess) break;
        launch_kv_quant((const bf16*)tmp, (const bf16*)tmp + pl, ctx->Limg, ctx->H, ctx->d.heads, ctx->q8rec,
                        ctx->q8rec + pl, ctx->q8rec_scl, ctx->q8rec_scl + spl, 0);
        for (int w = 0; w < 2 && e == cudaSuccess; ++w) {
          e = cudaMemcpy(cache_plane(ctx, c, st, b, w), ctx->q8rec + w * pl, pl, cudaMemcpyDefault);
          if (e == cudaSuccess)
            e = cudaMemcpy(cache_scales(ctx, c, st, b, w), ctx->q8rec_scl + w * spl, spl * 4, cudaMemcpyDefault);
        }
      }
    if (tmp) cudaFree(tmp);
    if (e == cudaSuccess)
      e = cudaMemcpy(cache_latent(ctx, c, 0), cache_latent(ctx, src, 0), (size_t)src->n_steps * ctx->Limg * ctx->C * 4,
                     cudaMemcpyDefault);
  }
  if (e != cudaSuccess) { free_cache_now(c); return set_err(IG_ECUDA, "cache clone: %s", cudaGetErrorString(e)); }
  *out = c;
  return IG_OK;
}

extern "C" ig_status ig_cache_write(ig_ctx* ctx, ig_cache* c, const void* kv, const float* latents, void* stream) {
  if (!ctx || !c || !kv) return set_err(IG_EINVAL, "NULL argument");
  if (!desc_equal(c->desc, ctx->d)) return set_err(IG_ECACHE_INCOMPAT, "cache built for another model");
  if (c->fp8 && !ctx->q8rec) return set_err(IG_EUNSUPPORTED, "fp8 cache needs a ctx created with cache_fp8");
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = (cudaStream_t)stream;
  const size_t pl = (size_t)ctx->Limg * ctx->H, spl = (size_t)ctx->Limg * ctx->d.heads;
  if (!c->fp8) {  // the caller's buffer is the storage layout of every step: one copy
    CUDA_TRY(cudaMemcpyAsync(c->ptr, kv, c->lat_off, cudaMemcpyDefault, st));
  }
  if (c->fp8 && c->y) {  // Y / hybrid: the caller's planes in storage order, one by one
    const size_t np = (size_t)c->n_steps * c->step_planes;
    for (size_t i = 0; i < np; ++i) {
      const bf16* src = (const bf16*)((const char*)kv + i * pl * ctx->esz);
      launch_kv_quant(src, src, ctx->Limg, ctx->H, ctx->d.heads, ctx->q8rec, ctx->q8rec + pl, ctx->q8rec_scl,
                      ctx->q8rec_scl + spl, st);
      CUDA_TRY(cudaMemcpyAsync((char*)c->ptr + i * pl, ctx->q8rec, pl, cudaMemcpyDefault, st));
      CUDA_TRY(cudaMemcpyAsync((char*)c->ptr + c->scale_off + i * spl * 4, ctx->q8rec_scl, spl * 4, cudaMemcpyDefault, st));
      CUDA_TRY(cudaStreamSynchronize(st));
    }
  }
  for (int s = 0; s < c->n_steps && c->fp8 && !c->y; ++s)
    for (int b = 0; b < ctx->nb; ++b) {
      const char* src = (const char*)kv + (((size_t)s * ctx->nb + b) * 2) * pl * ctx->esz;
      {
        launch_kv_quant((const bf16*)src, (const bf16*)(src + pl * ctx->esz), ctx->Limg, ctx->H, ctx->d.heads,
                        ctx->q8rec, ctx->q8rec + pl, ctx->q8rec_scl, ctx->q8rec_scl + spl, st);
        for (int w = 0; w < 2; ++w) {
          CUDA_TRY(cudaMemcpyAsync(cache_plane(ctx, c, s, b, w), ctx->q8rec + w * pl, pl, cudaMemcpyDefault, st));
          CUDA_TRY(cudaMemcpyAsync(cache_scales(ctx, c, s, b, w), ctx->q8rec_scl + w * spl, spl * 4, cudaMemcpyDefault, st));
        }
        CUDA_TRY(cudaStreamSynchronize(st));
      }
    }
  if (latents)
    CUDA_TRY(cudaMemcpyAsync(cache_latent(ctx, c, 0), latents, (size_t)c->n_steps * ctx->Limg * ctx->C * 4,
                             cudaMemcpyDefault, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return IG_OK;
}

extern "C" ig_status ig_cache_storage(ig_cache* c, void** ptr, size_t* bytes, int* tier) {
  if (!c) return set_err(IG_EINVAL, "cache is NULL");
  if (ptr) *ptr = c->ptr;
  if (bytes) *bytes = c->bytes;
  if (tier) *tier = c->tier;
  return IG_OK;
}

extern "C" void ig_cache_free(ig_cache* c) {
  if (!c) return;
  std::lock_guard<std::mutex> lk(g_zombie_mu);
  reap_zombies_locked(-1);  // earlier zombies whose pins dropped
  if (c->pins.load() == 0) free_cache_now(c);
  else { c->zombie = true; g_zombies.push_back(c); }
}

// ----------------------------------------------------------------------------------------
// the step
// ----------------------------------------------------------------------------------------
struct StepReq {
  const ig_edit_req* r;
  const ig_mask* m;
  bool use_cache;
};

// Enqueue the cached K/V of block b for every cache-using request into ring buffer b % R.
// Per request, by cache kind:
//   bf16, host tier : copy_mode 0 -> two full-L memcpys; else DMA runs of unmasked rows
//   bf16, HBM tier  : copy_mode 0 -> two full-L memcpys; else the SM gather kernel
//   fp8 (any tier)  : host tier first lands e4m3 runs + scale planes in a staging buffer by DMA;
//                     then the dequantizing gather writes bf16 unmasked rows into the ring
// kvg_dev/kvq_dev: per (block, request) gather descriptors (n_u = 0 when not applicable).
struct CopyPlan {
  bool any = false, gather = false, gather_q8 = false;
  int max_nu = 0;
  int kplan = 0;  // Algorithm-1 dense prefix: Y caches load Y_{b-1} for blocks b > kplan only
  // load deduplication: requests on the same (host-tier cache, step) as an earlier
  // request of the batch DMA only the rows that request did not load; the rest are copied
  // HBM -> HBM from its ring buffer (kv_dedupe_kernel)
  std::vector<int> dsrc;                                // per request: source index or -1
  std::vector<std::vector<std::pair<int, int>>> druns;  // per member: runs of U_r \ U_src
  std::vector<std::vector<CopyGroup>> dgroups;          // per member: DMA groups covering druns
  std::vector<int> dshared;                             // per member: |U_r ∩ U_src|
  std::vector<const ig_cache*> dcache;                  // per dedupe entry: the cache its pair shares
  DedupeArgs dd{};
};

static void lane_main(ig_ctx* ctx) {
  cudaSetDevice(ctx->device);
  auto& L = ctx->lane;
  for (;;) {
    std::function<void()> job;
    {
      std::unique_lock<std::mutex> lk(L.mu);
      L.cv.wait(lk, [&] { return L.stop || !L.q.empty(); });
      if (L.q.empty()) return;  // stop requested and drained
      job = std::move(L.q.front());
      L.q.pop_front();
    }
    job();
    {
      std::lock_guard<std::mutex> lk(L.mu);
      ++L.done;
    }
    L.cv_done.notify_all();
  }
}

static long long lane_push(ig_ctx* ctx, std::function<void()> fn) {
  auto& L = ctx->lane;
  if (!L.thr.joinable()) L.thr = std::thread(lane_main, ctx);
  long long seq;
  {
    std::lock_guard<std::mutex> lk(L.mu);
    L.q.push_back(std::move(fn));
    seq = ++L.pushed;
  }
  L.cv.notify_one();
  return seq;
}

static void lane_wait(ig_ctx* ctx, long long seq) {  // until job `seq` (1-based) has run
  auto& L = ctx->lane;
  std::unique_lock<std::mutex> lk(L.mu);
  L.cv_done.wait(lk, [&] { return L.done >= seq; });
}

static void lane_drain(ig_ctx* ctx) {
  long long seq;
  {
    std::lock_guard<std::mutex> lk(ctx->lane.mu);
    seq = ctx->lane.pushed;
  }
  lane_wait(ctx, seq);
}

static void lane_stop(ig_ctx* ctx) {
  auto& L = ctx->lane;
  if (!L.thr.joinable()) return;
  {
    std::lock_guard<std::mutex> lk(L.mu);
    L.stop = true;
  }
  L.cv.notify_all();
  L.thr.join();
}

static inline void note_copy(ig_ctx* ctx, cudaError_t e) {
  if (e != cudaSuccess && ctx->copy_err == cudaSuccess) ctx->copy_err = e;
}

static void issue_copy_now(ig_ctx* ctx, const std::vector<StepReq>& sr, const KvGatherReq* kvg_dev,
                           const KvGatherReq* kvq_dev, int b, const CopyPlan& plan, ig_stats& cs) {
  const int buf = b % ctx->R;
  // inside a graph capture only this step's records are visible; earlier steps completed
  // before the graph starts (same stream)
  if ((!ctx->capturing || (ctx->cap_mask >> buf & 1u)) && !ctx->dbg[IG_DBG_DROP_WAR])
    cudaStreamWaitEvent(ctx->copy_st, ctx->ev_comp[buf], 0);
  if (ctx->dbg[IG_DBG_SPIN_COPY_NS]) launch_spin((unsigned long long)ctx->dbg[IG_DBG_SPIN_COPY_NS], ctx->copy_st);
  const long long by0 = cs.h2d_bytes + cs.d2d_bytes;
  ProfScope ps(ctx, ctx->copy_st, IG_K_COPY, 0.0, 0.0, b);
  const int n = (int)sr.size();
  const size_t row = (size_t)ctx->H * ctx->esz;
  const size_t txt_off = (size_t)ctx->Lt * row, vplane = (size_t)ctx->L * row;
  std::vector<CopyOp>& cps = ctx->b_copies;
  cps.clear();
  for (int q = 0; q < n; ++q) {
    if (!sr[q].use_cache) continue;
    const ig_edit_req* r = sr[q].r;
    const ig_cache* c = r->cache;
    const bool host = c->tier == IG_CACHE_HOST;
    const int slot = r->slot;
    const int n_u = ctx->Limg - sr[q].m->n_m;
    long long by = 0;
    if (y_block(c, b) && c->fp8) {  // FP8 Y block: Y_{b-1} e4m3 runs + scales -> staging V half
      if (b <= plan.kplan) continue;
      if (host) {
        const size_t pl = (size_t)ctx->Limg * ctx->H, spl = (size_t)ctx->Limg * ctx->d.heads * 4;
        uint8_t* sd = ctx->q8in + ((size_t)slot * ctx->R + buf) * 2 * pl + pl;
        char* ss = (char*)ctx->q8in_scl + ((size_t)slot * ctx->R + buf) * 2 * spl + spl;
        const char* src = cache_plane(ctx, c, r->step, b - 1, 2);
        push_group_copies(cps, (char*)sd, src, (size_t)ctx->H, sr[q].m->groups);
        cps.push_back(CopyOp{ss, cache_scales(ctx, c, r->step, b - 1, 2), spl, 1, spl, 1, 0, 0});
        cs.h2d_bytes += (long long)n_u * ctx->H + (long long)spl;
      } else {
        cs.d2d_bytes += (long long)n_u * (ctx->H + 4 * ctx->d.heads);
      }
      continue;
    }
    if (y_block(c, b)) {  // Y block: the template's Y_{b-1} rows of the unmasked tokens -> V plane
      if (b <= plan.kplan) continue;  // block 0 / first block after the prefix: computed rows
      const char* src = cache_plane(ctx, c, r->step, b - 1, 2);
      char* dst = (char*)ctx->kv_arena + ((size_t)slot * ctx->slot_stride + (size_t)buf * ctx->buf_elems) * ctx->esz +
                  vplane + txt_off;
      const bool gathered = host ? ctx->o.copy_mode == 2 : ctx->o.copy_mode != 0;
      if (gathered) {
        by = (long long)n_u * row;  // SM gather kernel below
      } else if (ctx->o.copy_mode == 0) {
        note_copy(ctx, cudaMemcpyAsync(dst, src, (size_t)ctx->Limg * row, cudaMemcpyDefault, ctx->copy_st));
        by = (long long)ctx->Limg * row;
      } else {
        const bool dd = !plan.dsrc.empty() && plan.dsrc[q] >= 0;
        push_group_copies(cps, dst, src, row, dd ? plan.dgroups[q] : sr[q].m->groups);
        by = (long long)(dd ? n_u - plan.dshared[q] : n_u) * row;
        if (dd) cs.d2d_bytes += (long long)plan.dshared[q] * row;
      }
      if (host) cs.h2d_bytes += by; else cs.d2d_bytes += by;
      continue;
    }
    if (c->fp8) {
      by = 2LL * n_u * (ctx->H + 4 * ctx->d.heads);
      if (host) {  // e4m3 runs + whole scale planes -> staging (slot, buf)
        const size_t pl = (size_t)ctx->Limg * ctx->H, spl = (size_t)ctx->Limg * ctx->d.heads * 4;
        uint8_t* sd = ctx->q8in + ((size_t)slot * ctx->R + buf) * 2 * pl;
        char* ss = (char*)ctx->q8in_scl + ((size_t)slot * ctx->R + buf) * 2 * spl;
        for (int w = 0; w < 2; ++w) {
          const char* src = cache_plane(ctx, c, r->step, b, w);
          push_group_copies(cps, (char*)(sd + w * pl), src, (size_t)ctx->H, sr[q].m->groups);
          cps.push_back(CopyOp{ss + w * spl, cache_scales(ctx, c, r->step, b, w), spl, 1, spl, 1, 0, 0});
        }
        by = 2LL * n_u * ctx->H + 2LL * ctx->Limg * ctx->d.heads * 4;
      }
    } else if (ctx->o.copy_mode == 0) {
      const size_t plane = (size_t)ctx->Limg * row;
      auto& pf = ctx->pref[(size_t)slot * ctx->R + buf];
      const bool prefetched = (pf.c == c && pf.step == r->step && b < ctx->R);
      pf = ig_ctx::Pref{};
      if (!prefetched) {
        char* dst = (char*)ctx->kv_arena + ((size_t)slot * ctx->slot_stride + (size_t)buf * ctx->buf_elems) * ctx->esz;
        note_copy(ctx, cudaMemcpyAsync(dst + txt_off, cache_plane(ctx, c, r->step, b, 0), plane, cudaMemcpyDefault,
                                       ctx->copy_st));
        note_copy(ctx, cudaMemcpyAsync(dst + vplane + txt_off, cache_plane(ctx, c, r->step, b, 1), plane,
                                       cudaMemcpyDefault, ctx->copy_st));
        by = 2 * (long long)plane;
      }
    } else if (host && ctx->o.copy_mode == 1) {  // DMA runs straight into the ring
      char* dst = (char*)ctx->kv_arena + ((size_t)slot * ctx->slot_stride + (size_t)buf * ctx->buf_elems) * ctx->esz;
      const bool dd = !plan.dsrc.empty() && plan.dsrc[q] >= 0;
      const char* srcK = cache_plane(ctx, c, r->step, b, 0);
      const size_t splane = (size_t)(cache_plane(ctx, c, r->step, b, 1) - srcK);  // V plane after K
      push_group_copies(cps, dst + txt_off, srcK, row, dd ? plan.dgroups[q] : sr[q].m->groups, 2, splane, vplane);
      by = 2LL * (dd ? n_u - plan.dshared[q] : n_u) * row;
      if (dd) cs.d2d_bytes += 2LL * plan.dshared[q] * row;
    } else {
      by = 2LL * n_u * row;  // SM gather kernel below
    }
    if (host) cs.h2d_bytes += by; else cs.d2d_bytes += by;
  }
  for (size_t i = 0; i < cps.size(); ++i) {  // one DMA call per group (copy engines)
    const cudaError_t ce = issue_copy_op(cps[i], ctx->copy_st);
    if (ce != cudaSuccess && ctx->copy_err == cudaSuccess) {
      ctx->copy_err = ce;
      ctx->copy_err_idx = i;
    }
  }
  cs.dma_calls += (long long)cps.size();
  if (plan.dd.n > 0) {  // rows shared with an earlier same-(cache, step) request: HBM -> HBM
    // per entry from ITS cache (entries of one batch may sit on caches of different kinds)
    DedupeArgs dd = plan.dd;
    dd.buf_off = (long long)buf * ctx->buf_elems;
    int live = 0;
    for (int i = 0; i < dd.n; ++i) {
      const ig_cache* ce = plan.dcache[i];
      dd.e[i].v_only = y_block(ce, b) ? 1 : 0;
      dd.e[i].skip = (y_block(ce, b) && b <= plan.kplan) ? 1 : 0;
      live += !dd.e[i].skip;
    }
    if (live) {
      cs.kernel_launches++;
      launch_kv_dedupe(dd, ctx->copy_st);
    }
  }
  if (plan.gather) {
    cs.kernel_launches++;
    launch_kv_gather(kvg_dev + (size_t)b * n, n, plan.max_nu, ctx->Lt, ctx->H, (int)ctx->esz, ctx->copy_st);
  }
  if (plan.gather_q8) {
    cs.kernel_launches++;
    launch_kv_gather_q8(kvq_dev + (size_t)b * n, n, plan.max_nu, ctx->Lt, ctx->H, ctx->d.heads, ctx->copy_st);
  }
  if (ctx->dbg[IG_DBG_CORRUPT_ROW]) {  // fault injection: one staged cached row of the first cache user
    for (int q = 0; q < n; ++q) {
      if (!sr[q].use_cache || sr[q].m->n_m >= ctx->Limg) continue;
      char* dst = (char*)ctx->kv_arena + ((size_t)sr[q].r->slot * ctx->slot_stride + (size_t)buf * ctx->buf_elems) * ctx->esz;
      launch_corrupt_row(dst, (long long)ctx->L * ctx->H, sr[q].m->idx + ctx->Limg, ctx->Lt, ctx->H, (int)ctx->esz,
                         (float)ctx->dbg[IG_DBG_CORRUPT_ROW], ctx->copy_st);
      break;
    }
  }
  ps.bytes = (double)(cs.h2d_bytes + cs.d2d_bytes - by0);
  cudaEventRecord(ctx->ev_copy[buf], ctx->copy_st);
}

// Issue block b's cache copy: on the copy-lane thread when the step runs threaded (the job
// captures the step's request list, which outlives every job: the step drains the lane before
// it returns), else inline.
static void issue_copy(ig_ctx* ctx, const std::vector<StepReq>& sr, const KvGatherReq* kvg_dev,
                       const KvGatherReq* kvq_dev, int b, const CopyPlan& plan) {
  if (!plan.any) return;
  if (!ctx->lane_on) {
    issue_copy_now(ctx, sr, kvg_dev, kvq_dev, b, plan, ctx->stats);
    return;
  }
  const std::vector<StepReq>* srp = &sr;
  const CopyPlan* pp = &plan;
  const long long seq = lane_push(ctx, [ctx, srp, kvg_dev, kvq_dev, b, pp] {
    issue_copy_now(ctx, *srp, kvg_dev, kvq_dev, b, *pp, ctx->cstats);
  });
  if (b >= 0 && b < (int)ctx->job_of_block.size()) ctx->job_of_block[b] = seq;
}

// ---- Algorithm 1 planner on B200 ----------------------------------------------
// Per-block latencies of the batch from the linear models: C_w = comp(masked-rows
// FLOPs), C_w/o = comp(all-rows FLOPs), L = load(cached bytes).  Under the K/V variant the
// dense blocks form a prefix (C-AMB 23), so the exact optimum is a scan over the prefix length
// k of the two-lane pipeline: the copy lane loads cached blocks in order, at most R ahead of
// the compute lane (ring depth); the compute lane runs dense blocks, then each cached block
// once its load landed.  (Algorithm 1's greedy per-block rule, placement.py algorithm1, never
// picks a dense block when C_w/o > L + C_w, which is the B200 + PCIe regime.)
static double block_flops_rows(const ig_ctx* ctx, long long rows) {
  const double H = ctx->H, F = ctx->F;
  if (ctx->d.n_unet > 0)  // qkv + out + q2 + out2 (6 H^2), GEGLU + out (3 F H); self + cross attention
    return 2.0 * rows * (6 * H * H + 3 * H * F) + 4.0 * rows * (ctx->L + ctx->d.ctx_len) * H;
  return 2.0 * rows * (3 * H * H + H * H + 2 * H * F) + 4.0 * rows * ctx->L * H;
}

static int plan_prefix(ig_ctx* ctx, const std::vector<StepReq>& sr, const std::vector<int>& dshared) {
  const int N = ctx->nb;
  long long rows_m = 0, rows_all = 0;
  std::vector<long long> bytes(N, 0), rows_y(N, 0);
  for (auto& s : sr) {
    rows_m += ctx->Lt + s.m->n_m;
    rows_all += ctx->Lt + (s.use_cache ? ctx->Limg : s.m->n_m);
    if (!s.use_cache) continue;
    const ig_cache* c = s.r->cache;
    const long long n_u = ctx->Limg - s.m->n_m;
    long long n_load = n_u - dshared[&s - &sr[0]];  // deduplicated rows cross the link once
    // host-tier DMA groups: the link time of the rows they move plus the calls' fixed cost
    if (c->tier == IG_CACHE_HOST && ctx->o.copy_mode == 1 && n_u > 0 && s.m->dma_rows > 0)
      n_load = (long long)((double)n_load * (double)s.m->dma_rows / (double)n_u);
    for (int b = 0; b < N; ++b) {
      if (y_block(c, b)) {  // one plane; the K/V projection of the unmasked rows is recomputed
        if (b > 0) bytes[b] += c->fp8 ? n_u * (ctx->H + 4LL * ctx->d.heads) : n_load * ctx->H * (long long)ctx->esz;
        rows_y[b] += n_u;
      } else {
        bytes[b] += c->fp8 ? 2LL * n_u * (ctx->H + 4 * ctx->d.heads) : 2LL * n_load * ctx->H * (long long)ctx->esz;
      }
    }
  }
  std::vector<double> cw(N), lt(N);
  for (int b = 0; b < N; ++b) {
    cw[b] = ctx->pm_cs * (block_flops_rows(ctx, rows_m) + 4.0 * rows_y[b] * ctx->H * ctx->H) + ctx->pm_cb;
    lt[b] = bytes[b] > 0 ? ctx->pm_ls * (double)bytes[b] + ctx->pm_lb : 0.0;
  }
  const double cwo = ctx->pm_cs * block_flops_rows(ctx, rows_all) + ctx->pm_cb;
  const int R = ctx->R;
  int best_k = 0;
  double best = 1e300, period0 = 0.0;
  // Steady state of continuous batching: the copy lane is in order and runs into the next
  // step as soon as ring buffers free up (buffer b % R is free once the last cached block
  // that used it finished computing), so the step period is measured over repeated steps.
  std::vector<double> free_at(R);
  for (int k = 0; k <= N; ++k) {
    std::fill(free_at.begin(), free_at.end(), 0.0);
    double comp = 0, load = 0, start = 0;
    for (int rep = 0; rep < 3; ++rep) {
      start = comp;
      for (int b = 0; b < N; ++b) {
        if (b < k) { comp += cwo; continue; }
        load = std::max(load, free_at[b % R]) + lt[b];
        comp = std::max(comp, load) + cw[b];
        free_at[b % R] = comp;
      }
    }
    const double period = comp - start;
    if (k == 0) period0 = period;
    if (period < best - 1e-12) { best = period; best_k = k; }
  }
  // a dense prefix must buy a clear win: when the model's gain is within its own error (the
  // hybrid cache's balanced lanes measured 1% slower with a marginal prefix), keep k = 0
  return best < (1.0 - 0.02) * period0 ? best_k : 0;
}

extern "C" ig_status ig_set_plan(ig_ctx* ctx, int mode, int k, double comp_s_per_flop, double comp_s,
                                 double load_s_per_byte, double load_s) {
  if (!ctx) return set_err(IG_EINVAL, "ctx is NULL");
  if (mode < 0 || mode > 2 || k < 0) return set_err(IG_EINVAL, "bad plan mode/k");
  ctx->plan_mode = mode;
  ctx->plan_k = k;
  ctx->pm_cs = comp_s_per_flop; ctx->pm_cb = comp_s; ctx->pm_ls = load_s_per_byte; ctx->pm_lb = load_s;
  return IG_OK;
}

extern "C" int ig_last_plan(const ig_ctx* ctx) { return ctx ? ctx->last_plan_k : -1; }

// Optional restriction of a step to blocks [b0, b1) on caller-given residual rows (the
// teacher-forced debug hook); defaults run the whole step.
// Eager work after a graph launch: the ring events' latest records were capture nodes, which
// cannot be waited on eagerly; record them again behind the graph on its stream.
static void flush_graph_tail(ig_ctx* ctx) {
  if (!ctx->graph_tail) return;
  for (int i = 0; i < ctx->R; ++i) {
    cudaEventRecord(ctx->ev_comp[i], ctx->graph_st);
    cudaEventRecord(ctx->ev_copy[i], ctx->graph_st);
    cudaEventRecord(ctx->ev_yrec[i], ctx->graph_st);
  }
  ctx->graph_tail = false;
}

struct StepRange {
  int b0 = 0, b1 = -1;
  const float* X_in = nullptr;
  float* X_out = nullptr;
};

template <typename T>
static ig_status run_step(ig_ctx* ctx, const ig_edit_req* reqs, int n, cudaStream_t st,
                          ig_cache* record, int record_step, const StepRange& rng = StepRange()) {
  const int H = ctx->H, F = ctx->F, C = ctx->C, Lt = ctx->Lt, nb = ctx->nb, R = ctx->R;
  const int b0 = rng.b0, b1 = rng.b1 < 0 ? nb : rng.b1;
  const long long es = (long long)ctx->esz;
  const bool unet = ctx->d.n_unet > 0;
  ctx->stats = ig_stats{};
  ctx->copy_err = cudaSuccess;
  ctx->pdl_block = true;  // the step's first GEMM may follow anything the caller enqueued
  auto t_host0 = std::chrono::steady_clock::now();
  // ---- host validation (nothing enqueued before this passes) ----
  if (n < 0 || n > ctx->o.max_batch) return set_err(IG_EINVAL, "n=%d outside [0, max_batch=%d]", n, ctx->o.max_batch);
  if (n > 0 && !reqs) return set_err(IG_EINVAL, "reqs is NULL");
  std::vector<StepReq> sr;
  unsigned slots_seen = 0;
  for (int i = 0; i < n; ++i) {
    const ig_edit_req& r = reqs[i];
    if (r.slot < 0 || r.slot >= ctx->o.max_batch) return set_err(IG_EINVAL, "req %d: slot %d out of range", i, r.slot);
    if (slots_seen & (1u << r.slot)) return set_err(IG_EINVAL, "req %d: duplicate slot %d", i, r.slot);
    slots_seen |= 1u << r.slot;
    if (!r.mask || !r.latent || (!unet && !r.cond_vec) || ((Lt > 0 || unet) && !r.txt))
      return set_err(IG_EINVAL, "req %d: NULL mask/latent/txt/cond_vec", i);
    if (r.mask->L_img != ctx->Limg) return set_err(IG_EINVAL, "req %d: mask built for another model", i);
    const int nm = r.mask->n_m;
    if (nm == 0) continue;  // nothing to compute, latent stays bit-identical
    const bool need = nm < ctx->Limg;
    if (need) {
      if (!r.cache) return set_err(IG_ECACHE_MISS, "req %d: 0 < n_m=%d < L_img and no cache (S:134)", i, nm);
      if (!desc_equal(r.cache->desc, ctx->d)) return set_err(IG_ECACHE_INCOMPAT, "req %d: cache built for another model", i);
      if (r.step < 0 || r.step >= r.cache->n_steps)
        return set_err(IG_ECACHE_INCOMPAT, "req %d: step %d outside the cache schedule [0, %d)", i, r.step, r.cache->n_steps);
      if (r.cache->zombie) return set_err(IG_EINVAL, "req %d: cache was freed", i);
    }
    sr.push_back({&r, r.mask, need});
  }
  const int na = (int)sr.size();
  if (na == 0) return IG_OK;
  const int M_txt = na * Lt;
  int M = M_txt;
  bool any_cache = false;
  int max_nu = 0;
  for (auto& s : sr) {
    M += s.m->n_m;
    any_cache |= s.use_cache;
    if (s.use_cache) max_nu = std::max(max_nu, ctx->Limg - s.m->n_m);
  }
  CopyPlan plan;
  {
    const bool no_dedupe = !ig_tuning_ref().load_dedupe;
    auto dedupable = [&](int q) {
      const ig_cache* c = sr[q].use_cache ? sr[q].r->cache : nullptr;
      return c && c->tier == IG_CACHE_HOST && !c->fp8 && ctx->o.copy_mode == 1;
    };
    const size_t row_b = (size_t)H * es;
    plan.dsrc.assign(na, -1);
    plan.druns.assign(na, {});
    plan.dgroups.assign(na, {});
    plan.dshared.assign(na, 0);
    for (int q = 0; q < na && !no_dedupe; ++q) {
      if (!dedupable(q)) continue;
      for (int q0 = 0; q0 < q; ++q0)
        if (plan.dsrc[q0] < 0 && dedupable(q0) && sr[q0].r->cache == sr[q].r->cache && sr[q0].r->step == sr[q].r->step) {
          if (plan.dd.n >= MAX_DEDUPE) break;
          const auto& bq = sr[q].m->bits;
          const auto& b0 = sr[q0].m->bits;
          int shared = 0;
          auto& runs = plan.druns[q];
          for (int i = 0; i < ctx->Limg;) {  // runs of tokens unmasked in q but masked in q0
            if (bq[i] || !b0[i]) { shared += !bq[i]; ++i; continue; }
            int j = i;
            while (j < ctx->Limg && !bq[j] && b0[j]) ++j;
            runs.push_back({i, j - i});
            i = j;
          }
          make_copy_groups(runs, ctx->Limg, ctx->d.grid_w, copy_call_rows(row_b, 2), plan.dgroups[q]);
          plan.dsrc[q] = q0;
          plan.dshared[q] = shared;
          DedupeEnt& e = plan.dd.e[plan.dd.n++];
          e.idx_u = sr[q].m->idx + ctx->Limg;
          e.n_u = ctx->Limg - sr[q].m->n_m;
          e.bits0 = sr[q0].m->bits_dev;
          e.slot0 = sr[q0].r->slot;
          e.slot = sr[q].r->slot;
          plan.dcache.push_back(sr[q].r->cache);
          plan.dd.max_nu = std::max(plan.dd.max_nu, e.n_u);
          break;
        }
    }
    plan.dd.arena = ctx->kv_arena;
    plan.dd.slot_stride = ctx->slot_stride;
    plan.dd.L = ctx->L;
    plan.dd.Lt = ctx->Lt;
    plan.dd.H = H;
    plan.dd.es = (int)es;
  }
  // ---- Algorithm-1 block plan (C-AMB 23): a dense prefix of k blocks ----
  int kplan = 0;
  if (any_cache && !record && b0 == 0 && b1 == nb) {
    if (ctx->plan_mode == 1) kplan = std::min(ctx->plan_k, nb);
    else if (ctx->plan_mode == 2) kplan = plan_prefix(ctx, sr, plan.dshared);
  }
  ctx->last_plan_k = kplan;
  // unmasked image rows in the row set: Y-cache requests always (their K/V are recomputed from
  // the replenished block inputs), K/V-cache requests only under a dense prefix.  Y requests'
  // rows come first, so a cached block's K/V-recompute rows are the one range [M, M_y).
  // Y requests are ordered by their cache's number of Y blocks (descending); the Y-block sets
  // are nested (y_modes), so block b's Y rows are the one range [M, M + uy[b]).
  int U_y = 0, U_kv = 0;
  std::vector<int> yord;
  for (int q = 0; q < (int)sr.size(); ++q)
    if (sr[q].use_cache) {
      if (sr[q].r->cache->y) { U_y += ctx->Limg - sr[q].m->n_m; yord.push_back(q); }
      else if (kplan > 0) U_kv += ctx->Limg - sr[q].m->n_m;
    }
  std::stable_sort(yord.begin(), yord.end(),
                   [&](int a, int b) { return sr[a].r->cache->kv_blocks < sr[b].r->cache->kv_blocks; });
  std::vector<int> urow0(sr.size(), 0), uy(nb, 0);
  {
    int row = M;
    for (int q : yord) { urow0[q] = row; row += ctx->Limg - sr[q].m->n_m; }
    for (int b = 0; b < nb; ++b)
      for (int q : yord) if (y_block(sr[q].r->cache, b)) uy[b] += ctx->Limg - sr[q].m->n_m;
  }
  const int M_y = M + U_y;
  const int M_full = M_y + U_kv;
  if (M_full > ctx->o.max_rows) return set_err(IG_ENOMEM, "step needs %d rows > max_rows %d", M_full, ctx->o.max_rows);
  const int M_img = M - M_txt;
  ctx->stats.rows = M;

  // ---- descriptors -> pinned staging -> device (one small H2D) ----
  const int si = ctx->stage_i;
  ctx->stage_i = (si + 1) % NSTAGE;
  const unsigned long long step_no = ++ctx->step_no;
  {
    const auto w0 = std::chrono::steady_clock::now();
    CUDA_TRY(cudaEventSynchronize(ctx->ev_stage[si]));  // the step that used this slot is done
    t_host0 += std::chrono::steady_clock::now() - w0;  // back-pressure is not enqueue time
  }
  char* hs = ctx->h_stage[si];
  // a step that runs as a CUDA graph reads its descriptors from ONE fixed device slot, filled from
  // this step's pinned slot just before the graph launch: the graph then does not depend on which
  // of the NSTAGE host slots was used (before: NSTAGE captures per step shape — a new request cost
  // 4+ captures and instantiations, ~100 ms, against ~150 ms of SD3 steps)
  bool graph_ok = ctx->o.use_graphs && st != nullptr && !record && !rng.X_in && !rng.X_out && !ctx->prof &&
                  b0 == 0 && b1 == nb;
  for (auto& s2 : sr)
    if (s2.use_cache && (s2.r->cache->tier != IG_CACHE_DEVICE || ctx->o.copy_mode == 0)) graph_ok = false;
  char* ds = graph_ok ? ctx->d_gstage : ctx->d_stage[si];
  ReqDev* hreq = (ReqDev*)hs;
  // attention segments: [0, 2B) the masked-rows step, [2B, 5B) the dense prefix (+ unmasked)
  AttnSeg* hseg = (AttnSeg*)(hs + ctx->o.max_batch * sizeof(ReqDev));
  AttnSeg* hsegf = hseg + 2 * ctx->o.max_batch;
  // UNet cross-attention: [5B, 6B) masked rows (cached blocks), [6B, 8B) + unmasked (dense prefix)
  AttnSeg* hsegc = hseg + 5 * ctx->o.max_batch;
  AttnSeg* hsegcf = hseg + 6 * ctx->o.max_batch;
  KvGatherReq* hkvg = (KvGatherReq*)((char*)hseg + 8 * ctx->o.max_batch * sizeof(AttnSeg));
  ReqDev* dreq = (ReqDev*)ds;
  AttnSeg* dseg = (AttnSeg*)(ds + ctx->o.max_batch * sizeof(ReqDev));
  AttnSeg* dsegf = dseg + 2 * ctx->o.max_batch;
  AttnSeg* dsegc = dseg + 5 * ctx->o.max_batch;
  AttnSeg* dsegcf = dseg + 6 * ctx->o.max_batch;
  KvGatherReq* dkvg = (KvGatherReq*)((char*)dseg + 8 * ctx->o.max_batch * sizeof(AttnSeg));
  int nseg = 0, max_q = 0, nsegf = 0, max_qf = 0, nsegc = 0, nsegcf = 0, max_qcf = 0;
  int img_row = M_txt, kvrow = M_y;
  for (int q = 0; q < na; ++q) {
    const ig_edit_req* r = sr[q].r;
    ReqDev& d = hreq[q];
    d.slot = r->slot;
    d.n_m = sr[q].m->n_m;
    d.txt_row0 = q * Lt;
    d.img_row0 = img_row;
    d.idx_m = sr[q].m->idx;
    d.idx_u = sr[q].m->idx + ctx->Limg;
    d.latent = r->latent;
    d.txt = r->txt;
    d.cond = r->cond_vec;
    d.sigma = r->sigma;
    d.dsig = r->sigma_next - r->sigma;
    d.has_cache = sr[q].use_cache;
    const bool ycache = sr[q].use_cache && r->cache->y;
    d.n_ui = (sr[q].use_cache && (ycache || kplan > 0)) ? ctx->Limg - d.n_m : 0;
    d.uimg_row0 = ycache ? urow0[q] : kvrow;
    d.tlatent = sr[q].use_cache ? cache_latent_dev(ctx, r->cache, r->step) : nullptr;
    const long long kvb = (long long)r->slot * ctx->slot_stride;
    if (Lt > 0) { hseg[nseg++] = AttnSeg{q * Lt, Lt, kvb}; max_q = std::max(max_q, Lt); }
    hseg[nseg++] = AttnSeg{img_row, d.n_m, kvb};
    max_q = std::max(max_q, d.n_m);
    if (unet) {  // cross-attention segments: the request's context K/V in the cross arena
      const long long ckv = (long long)q * 2 * ctx->d.ctx_len * H;
      hsegc[nsegc++] = AttnSeg{img_row, d.n_m, ckv};
      hsegcf[nsegcf++] = AttnSeg{img_row, d.n_m, ckv};
      if (kplan > 0 && d.n_ui > 0) hsegcf[nsegcf++] = AttnSeg{d.uimg_row0, d.n_ui, ckv};
      max_qcf = std::max(max_qcf, std::max(d.n_m, kplan > 0 ? d.n_ui : 0));
    }
    if (kplan > 0) {
      if (Lt > 0) hsegf[nsegf++] = AttnSeg{q * Lt, Lt, kvb};
      hsegf[nsegf++] = AttnSeg{img_row, d.n_m, kvb};
      if (d.n_ui > 0) hsegf[nsegf++] = AttnSeg{d.uimg_row0, d.n_ui, kvb};
      max_qf = std::max(max_qf, std::max(Lt, std::max(d.n_m, d.n_ui)));
    }
    img_row += d.n_m;
    if (!ycache) kvrow += d.n_ui;
  }
  int npair = 0, npairf = 0, npaircf = 0;  // attention work items (segment, 256-row query-tile pair)
  for (int i = 0; i < nseg; ++i) npair += (hseg[i].q_len + 255) / 256;
  for (int i = 0; i < nsegf; ++i) npairf += (hsegf[i].q_len + 255) / 256;
  for (int i = 0; i < nsegcf; ++i) npaircf += (hsegcf[i].q_len + 255) / 256;
  // copy-lane plan and per-(block, request) gather descriptors (see issue_copy)
  plan.any = any_cache;
  plan.max_nu = max_nu;
  plan.kplan = kplan;

  KvGatherReq* hkvq = hkvg + (size_t)nb * ctx->o.max_batch;
  KvGatherReq* dkvq = dkvg + (size_t)nb * ctx->o.max_batch;
  if (any_cache) {
    for (int q = 0; q < na; ++q) {
      if (!sr[q].use_cache) continue;
      const ig_cache* c = sr[q].r->cache;
      if (c->fp8) plan.gather_q8 = true;
      else if (c->tier == IG_CACHE_DEVICE ? ctx->o.copy_mode != 0 : ctx->o.copy_mode == 2) plan.gather = true;
    }
    for (int b = 0; b < nb; ++b)
      for (int q = 0; q < na; ++q) {
        KvGatherReq g{}, gq{};
        const ig_edit_req* r = sr[q].r;
        if (sr[q].use_cache) {
          const ig_cache* c = r->cache;
          char* dst = (char*)ctx->kv_arena + ((size_t)r->slot * ctx->slot_stride + (size_t)(b % R) * ctx->buf_elems) * es;
          const int n_u = ctx->Limg - sr[q].m->n_m;
          if (c->fp8 && y_block(c, b)) {  // V plane only: dequantize Y_{b-1} rows (after the prefix)
            if (b > kplan) {
              gq.idx_u = sr[q].m->idx + ctx->Limg;
              gq.n_u = n_u;
              gq.srcK = nullptr;
              gq.dstV = dst + (size_t)ctx->L * H * es;
              if (c->tier == IG_CACHE_HOST) {
                const size_t pl = (size_t)ctx->Limg * H, spl = (size_t)ctx->Limg * ctx->d.heads;
                const size_t sb = (size_t)r->slot * R + (b % R);
                gq.srcV = ctx->q8in + sb * 2 * pl + pl;
                gq.sclV = ctx->q8in_scl + sb * 2 * spl + spl;
              } else {
                gq.srcV = cache_plane_dev(ctx, c, r->step, b - 1, 2);
                gq.sclV = cache_scales_dev(ctx, c, r->step, b - 1, 2);
              }
            }
          } else if (c->fp8) {
            gq.idx_u = sr[q].m->idx + ctx->Limg;
            gq.n_u = n_u;
            gq.dstK = dst;
            gq.dstV = dst + (size_t)ctx->L * H * es;
            if (c->tier == IG_CACHE_HOST) {  // dequantize from the staging the DMA lands in
              const size_t pl = (size_t)ctx->Limg * H, spl = (size_t)ctx->Limg * ctx->d.heads;
              const size_t sb = (size_t)r->slot * R + (b % R);
              gq.srcK = ctx->q8in + sb * 2 * pl;
              gq.srcV = ctx->q8in + sb * 2 * pl + pl;
              gq.sclK = ctx->q8in_scl + sb * 2 * spl;
              gq.sclV = ctx->q8in_scl + sb * 2 * spl + spl;
            } else {
              gq.srcK = cache_plane_dev(ctx, c, r->step, b, 0);
              gq.srcV = cache_plane_dev(ctx, c, r->step, b, 1);
              gq.sclK = cache_scales_dev(ctx, c, r->step, b, 0);
              gq.sclV = cache_scales_dev(ctx, c, r->step, b, 1);
            }
          } else if (y_block(c, b)) {  // one plane: Y_{b-1} -> V plane (blocks after the first cached one)
            if ((c->tier == IG_CACHE_DEVICE ? ctx->o.copy_mode != 0 : ctx->o.copy_mode == 2) && b > kplan) {
              g.srcK = nullptr;
              g.srcV = cache_plane_dev(ctx, c, r->step, b - 1, 2);
              g.idx_u = sr[q].m->idx + ctx->Limg;
              g.n_u = n_u;
              g.dstK = dst;
              g.dstV = dst + (size_t)ctx->L * H * es;
            }
          } else if (c->tier == IG_CACHE_DEVICE ? ctx->o.copy_mode != 0 : ctx->o.copy_mode == 2) {
            g.srcK = cache_plane_dev(ctx, c, r->step, b, 0);
            g.srcV = cache_plane_dev(ctx, c, r->step, b, 1);
            g.idx_u = sr[q].m->idx + ctx->Limg;
            g.n_u = n_u;
            g.dstK = dst;
            g.dstV = dst + (size_t)ctx->L * H * es;
          }
        }
        hkvg[(size_t)b * na + q] = g;
        hkvq[(size_t)b * na + q] = gq;
      }
  }
  // the compute stream's descriptors go up on the compute stream; the copy lane's gather
  // descriptors on the copy stream, so the copy lane never waits for the previous step's
  // compute tail before it starts this step's prefetch (no bubble at step boundaries)
  // The compute stream's descriptors are pulled by SM loads from the mapped pinned staging, not
  // by a DMA: a cudaMemcpyAsync here would queue on the copy engine behind the copy lane's
  // cache prefetch (up to R blocks of DMA) and stall the step start (measured: ~85 ms per step
  // with a dense prefix).
  const size_t desc_bytes = (char*)hkvg - hs;
  // ---- CUDA graph of the step (device-tier caches / no cache only: host-tier DMA sources
  // change every step) ----
  // (the legacy default stream cannot be captured)
  std::string gkey;
  if (graph_ok) {
    // this step's descriptors -> the fixed graph slot, stream-ordered after the previous step
    launch_copy_bytes(ds, ctx->m_stage[si], desc_bytes, st);
    if (plan.gather || plan.gather_q8) {
      const size_t off = (char*)hkvg - hs, bytes = (char*)(hkvq + (size_t)nb * na) - (char*)hkvg;
      CUDA_TRY(cudaMemcpyAsync(ds + off, hs + off, bytes, cudaMemcpyHostToDevice, st));
    }
    std::vector<long long> k = {kplan, na, M, M_txt, M_full, nseg, max_q, nsegf, max_qf, max_nu, nsegcf, max_qcf,
                                plan.gather, plan.gather_q8, any_cache, (long long)desc_bytes};
    for (int v : uy) k.push_back(v);
    for (auto& s2 : sr) {
      k.push_back(s2.r->slot); k.push_back(s2.m->n_m); k.push_back(s2.use_cache);
      if (s2.use_cache) { k.push_back(s2.r->cache->y); k.push_back(s2.r->cache->fp8); k.push_back(s2.r->cache->kv_blocks); }
    }
    gkey.assign(reinterpret_cast<const char*>(k.data()), k.size() * sizeof(long long));
    auto it = ctx->graphs.find(gkey);
    if (it != ctx->graphs.end()) {  // replay: the graph pulls this step's descriptors itself
      it->second.last_used = step_no;
      for (auto& s2 : sr) if (s2.use_cache) s2.r->cache->pins.fetch_add(1);
      CUDA_TRY(cudaGraphLaunch(it->second.exec, st));
      ctx->graph_tail = true;
      ctx->graph_st = st;
      ctx->stats = it->second.stats;
      CUDA_TRY(cudaEventRecord(ctx->ev_stage[si], st));
      for (auto& s2 : sr)
        if (s2.use_cache) CUDA_TRY(cudaLaunchHostFunc(st, unpin_cb, (void*)s2.r->cache));
      ctx->stats.host_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t_host0).count();
      return IG_OK;
    }
    CUDA_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    cudaEventRecord(ctx->ev_fork, st);
    cudaStreamWaitEvent(ctx->copy_st, ctx->ev_fork, 0);  // the copy lane joins the capture
    ctx->capturing = true;
    ctx->cap_mask = 0;
  }
  if (!ctx->capturing) flush_graph_tail(ctx);  // eager step after a graph
  // copy lane on its own host thread for host-tier caches (DMA back-pressure), inline otherwise
  // and whenever the main thread itself touches the copy stream (recording, capture, profiling)
  {
    const bool no_lane = !ig_tuning_ref().copy_thread;
    bool any_host = false;
    for (auto& s2 : sr) any_host |= s2.use_cache && s2.r->cache->tier == IG_CACHE_HOST;
    ctx->lane_on = !no_lane && any_host && !ctx->prof && !ctx->capturing && !record && !rng.X_in;
    ctx->cstats = ig_stats{};
    ctx->job_of_block.assign(nb, -1);
  }
  struct LaneGuard {  // every exit path drains the lane before sr / plan go out of scope
    ig_ctx* c;
    ~LaneGuard() {
      if (!c->lane_on) return;
      lane_drain(c);
      c->stats.h2d_bytes += c->cstats.h2d_bytes;
      c->stats.d2d_bytes += c->cstats.d2d_bytes;
      c->stats.kernel_launches += c->cstats.kernel_launches;
      c->stats.dma_calls += c->cstats.dma_calls;
      c->cstats = ig_stats{};
      c->lane_on = false;
    }
  } lane_guard{ctx};
  if (!graph_ok) launch_copy_bytes(ds, ctx->m_stage[si], desc_bytes, st);
  if (!graph_ok && (plan.gather || plan.gather_q8)) {
    const size_t off = (char*)hkvg - hs, bytes = (char*)(hkvq + (size_t)nb * na) - (char*)hkvg;
    if (ctx->lane_on) {
      lane_push(ctx, [ctx, ds, hs, off, bytes] {
        note_copy(ctx, cudaMemcpyAsync(ds + off, hs + off, bytes, cudaMemcpyHostToDevice, ctx->copy_st));
      });
    } else {
      CUDA_TRY(cudaMemcpyAsync(ds + off, hs + off, bytes, cudaMemcpyHostToDevice, ctx->copy_st));
    }
  }
  for (auto& s : sr) if (s.use_cache) { s.r->cache->pins.fetch_add(1); }
  for (auto& s : sr) { s.m->used = true; s.m->last_st = st; }

  // ---- prefetch the first R cached blocks (copy lane); dense-prefix blocks need no cache ----
  const int bc0 = std::max(b0, kplan);
  // sequential loading (Algorithm-1 ablation, fig:pipeline_load): block b's cache copy
  // starts only after block b-1 finished computing, and block b waits for it (no overlap)
  const bool seq_load = ctx->dbg[IG_DBG_SEQUENTIAL] != 0 && !record;
  if (!seq_load)
    for (int b = bc0; b < std::min(bc0 + R, b1); ++b) issue_copy(ctx, sr, dkvg, dkvq, b, plan);

  T* h = (T*)ctx->h;
  T* qkv = (T*)ctx->qkv;
  T* cat = (T*)ctx->cat;
  const long long ldcat = H + F;
  auto& stats = ctx->stats;

  // ---- a2/a4: rows + gather; a3: conditioning ----
  {
    ProfScope ps(ctx, st, IG_K_ROWS, 0.0, (double)M_txt * H * (4 + es) + (double)M_img * C * (4 + es));
    launch_build_rows<T>(dreq, na, Lt, C, H, M_txt, M, ctx->ri, ctx->X, (T*)ctx->Ain, st, M_full, unet ? 1 : 0);
  }
  if (unet) {
    ProfScope ps(ctx, st, IG_K_ROWS, 0.0, 2.0 * na * ctx->d.ctx_len * ctx->d.ctx_dim * es);
    launch_pack_ctx<T>(dreq, na, ctx->d.ctx_len, ctx->d.ctx_dim, (T*)ctx->ctxp, st);
    stats.kernel_launches++;
  }
  if (!unet) {
  ProfScope ps_cond(ctx, st, IG_K_COND, 0.0, (double)ctx->mod_ld * H * es);
  launch_timestep_embed(dreq, na, ctx->temb, st);
  launch_gemv<T>(ctx->gv_t1, 1, (H + 31) / 32, na, 256, st);
  launch_gemv<T>(ctx->gv_t2, 1, (H + 31) / 32, na, H, st);
  launch_add_cond(dreq, na, H, ctx->vec, st);
  if (ctx->modw) {  // bf16: one tensor-core GEMM over the packed modulation weights
    launch_silu(ctx->vec, ctx->svec, (long long)na * H, st, ctx->svec_bf);
    GemmArgs g{};
    g.A = ctx->svec_bf; g.lda = H; g.B = ctx->modw; g.ldb = H; g.bias = ctx->modb;
    g.C = ctx->modbuf; g.ldc = ctx->mod_ld; g.M = na; g.N = (int)ctx->mod_ld; g.K = H;
    g.epi = EPI_STORE; g.out_f32 = 1;
    launch_gemm_tc(g, st);
  } else {
    launch_silu(ctx->vec, ctx->svec, (long long)na * H, st);
    launch_gemv<T>(ctx->gv_mod, (int)ctx->gv_mod_host.size(), ctx->gv_mod_groups, na, H, st);
  }
  }
  if (!unet) stats.kernel_launches += 7;
  if (rng.X_in) {  // teacher-forced residual rows (+ img_in of the template rows, if any)
    CUDA_TRY(cudaMemcpyAsync(ctx->X, rng.X_in, (size_t)M * H * 4, cudaMemcpyDeviceToDevice, st));
    if (M_full > M && !unet) {
      GemmArgs g{};
      g.A = (const char*)ctx->Ain + (long long)(M - M_txt) * C * es; g.lda = C; g.B = ctx->img_in.w; g.ldb = C;
      g.bias = ctx->img_in.b; g.C = ctx->X + (long long)M * H; g.ldc = H; g.M = M_full - M; g.N = H; g.K = C;
      g.epi = EPI_POS; g.ri = ctx->ri; g.ri_off = M; g.pos = ctx->pos_embed; g.pos_ld = H;
      gemm(ctx, g, st);
    }
  } else if (!unet) {  // img_in (+ SD3 pos_embed) into the fp32 residual X
    // (UNet: the masked rows of the level's hidden state are already in X, build_rows)
    GemmArgs g{};
    g.A = ctx->Ain; g.lda = C; g.B = ctx->img_in.w; g.ldb = C; g.bias = ctx->img_in.b;
    g.C = ctx->X + (long long)M_txt * H; g.ldc = H; g.M = M_full - M_txt; g.N = H; g.K = C;
    g.epi = EPI_POS; g.ri = ctx->ri; g.ri_off = M_txt; g.pos = ctx->pos_embed; g.pos_ld = H;
    gemm(ctx, g, st);
  }
  const float* mod = ctx->modbuf;
  const long long mld = ctx->mod_ld;
  auto ln_mod = [&](int r0, int r1, int mod_t, int shift_c, int scale_c) {
    if (r1 <= r0) return;
    const long long off = ctx->mods[mod_t].off;
    ProfScope ps(ctx, st, IG_K_LNMOD, 0.0, (double)(r1 - r0) * H * (4 + es));
    launch_ln_mod<T>(ctx->X, H, r0, r1, ctx->ri, mod + off, (int)mld, shift_c * H, scale_c * H,
                     ctx->d.ln_eps, h, H, st);
    stats.kernel_launches++;
  };
  auto gemm_rows = [&](int r0, int r1, const void* A, long long lda, const void* B, const void* bias,
                       int N, int K, void* Cp, long long ldc, int epi, const float* gate, int out_f32) {
    if (r1 <= r0) return;
    GemmArgs g{};
    g.A = (const char*)A + (long long)r0 * lda * es; g.lda = lda;
    g.B = B; g.ldb = K; g.bias = bias;
    g.M = r1 - r0; g.N = N; g.K = K; g.epi = epi; g.out_f32 = out_f32;
    g.ri = ctx->ri; g.ri_off = r0;
    g.precise_gelu = ig_tuning_ref().precise_gelu != 0;
    if (epi == EPI_GATED_RES) {
      g.C = (float*)Cp + (long long)r0 * ldc; g.gate = gate; g.gate_ld = mld;
    } else {
      g.C = (char*)Cp + (long long)r0 * ldc * (out_f32 ? 4 : es);
    }
    g.ldc = ldc;
    gemm(ctx, g, st);
  };
  auto qkv_post = [&](int r0, int r1, const void* qg, const void* kg, int buf) {
    if (r1 <= r0) return;
    QkvPost p{};
    p.qkv = qkv; p.ld_qkv = 3 * H; p.Q = ctx->Q; p.kv_arena = ctx->kv_arena;
    p.slot_stride = ctx->slot_stride; p.buf_off = (long long)buf * ctx->buf_elems;
    p.L = ctx->L; p.H = H; p.qg = qg; p.kg = kg; p.rope_tab = ctx->rope_tab;
    p.rope_maxpos = ctx->rope_maxpos;
    p.ax1_pair = ctx->d.rope_axes[0] / 2; p.ax2_pair = (ctx->d.rope_axes[0] + ctx->d.rope_axes[1]) / 2;
    p.heads = ctx->d.heads; p.head_dim = ctx->d.head_dim; p.grid_w = ctx->d.grid_w;
    p.qk_norm = ctx->d.qk_norm; p.rope = ctx->d.rope; p.r0 = r0; p.r1 = r1;
    ProfScope ps(ctx, st, IG_K_QKVPOST, 0.0, (double)(r1 - r0) * 6.0 * H * es);
    launch_qkv_post<T>(p, ctx->ri, st);
    stats.kernel_launches++;
  };
  // a6: QKV projection + norm/RoPE/Q-pack/positional K/V merge.  bf16 mode fuses the whole
  // epilogue into the tensor-core GEMM; fp32 parity mode runs the GEMM then qkv_post.
  const bool fused_qkv = ctx->d.dtype == IG_BF16 && g_tc_gemm && ((H % 256) == 0 || unet) &&
                         (ctx->d.head_dim == 128 || ctx->d.head_dim == 64);
  auto qkv_proj = [&](int r0, int r1, const void* W, const void* bias, const void* qg, const void* kg, int buf) {
    if (r1 <= r0) return;
    if (!fused_qkv) {
      gemm_rows(r0, r1, h, H, W, bias, 3 * H, H, qkv, 3 * H, EPI_STORE, nullptr, 0);
      qkv_post(r0, r1, qg, kg, buf);
      return;
    }
    GemmArgs g{};
    g.A = (const char*)h + (long long)r0 * H * es; g.lda = H;
    g.B = W; g.ldb = H; g.bias = bias;
    g.C = ctx->Q; g.ldc = H;
    g.M = r1 - r0; g.N = 3 * H; g.K = H; g.epi = EPI_QKV;
    g.ri = ctx->ri; g.ri_off = r0;
    QkvEpi& e = g.qkv;
    e.Q = ctx->Q; e.kv_arena = ctx->kv_arena; e.slot_stride = ctx->slot_stride;
    e.buf_off = (long long)buf * ctx->buf_elems; e.L = ctx->L; e.H = H; e.qg = qg; e.kg = kg;
    e.rope_tab = ctx->rope_tab; e.rope_maxpos = ctx->rope_maxpos;
    e.ax1_pair = ctx->d.rope_axes[0] / 2; e.ax2_pair = (ctx->d.rope_axes[0] + ctx->d.rope_axes[1]) / 2;
    e.head_dim = ctx->d.head_dim; e.grid_w = ctx->d.grid_w; e.qk_norm = ctx->d.qk_norm; e.rope = ctx->d.rope;
    gemm(ctx, g, st);
  };
  // Y variant: K/V of the replenished unmasked rows only (B = rows [H, 3H) of W_qkv / lin1)
  auto kv_proj = [&](int r0, int r1, const void* W, const void* bias, const void* kg, int buf) {
    if (r1 <= r0) return;
    if (!fused_qkv) {  // parity mode: full [q|k|v] GEMM, the Q rows >= M are never read
      gemm_rows(r0, r1, h, H, W, bias, 3 * H, H, qkv, 3 * H, EPI_STORE, nullptr, 0);
      qkv_post(r0, r1, kg, kg, buf);
      return;
    }
    GemmArgs g{};
    g.A = (const char*)h + (long long)r0 * H * es; g.lda = H;
    g.B = (const char*)W + (long long)H * H * es; g.ldb = H; g.bias = bias ? (const char*)bias + (long long)H * es : nullptr;
    g.C = ctx->Q; g.ldc = H;
    g.M = r1 - r0; g.N = 2 * H; g.K = H; g.epi = EPI_QKV;
    g.ri = ctx->ri; g.ri_off = r0;
    QkvEpi& e = g.qkv;
    e.Q = ctx->Q; e.kv_arena = ctx->kv_arena; e.slot_stride = ctx->slot_stride;
    e.buf_off = (long long)buf * ctx->buf_elems; e.L = ctx->L; e.H = H; e.qg = nullptr; e.kg = kg;
    e.rope_tab = ctx->rope_tab; e.rope_maxpos = ctx->rope_maxpos;
    e.ax1_pair = ctx->d.rope_axes[0] / 2; e.ax2_pair = (ctx->d.rope_axes[0] + ctx->d.rope_axes[1]) / 2;
    e.head_dim = ctx->d.head_dim; e.grid_w = ctx->d.grid_w; e.qk_norm = ctx->d.qk_norm; e.rope = ctx->d.rope;
    e.col_base = H;
    gemm(ctx, g, st);
  };
  // Y variant: replenish the unmasked rows' block input from the staged Y_{b-1} (V plane)
  // Y blocks after the first cached one: LN-modulation of the unmasked rows straight from the
  // staged Y_{b-1} rows (the copy lane's V-plane landing zone), after waiting for the copy
  auto y_staged = [&](int b) { return uy[b] > 0 && b > kplan; };
  int cur_b = 0;  // block being enqueued (the lane job that recorded its ring event must have run)
  auto lane_ready = [&]() {
    if (ctx->lane_on && ctx->job_of_block[cur_b] > 0) lane_wait(ctx, ctx->job_of_block[cur_b]);
  };
  auto ln_mod_y = [&](int b, int buf, int mod_t, int shift_c, int scale_c) {
    if (!ctx->dbg[IG_DBG_DROP_RAW]) {
      lane_ready();
      stream_wait(ctx, st, ctx->ev_copy[buf]);
    }
    const long long off = ctx->mods[mod_t].off;
    ProfScope ps(ctx, st, IG_K_LNMOD, 0.0, (double)uy[b] * H * (es + es));
    launch_ln_mod_staged<T>(ctx->kv_arena, ctx->slot_stride, (long long)buf * ctx->buf_elems, ctx->L, H, M, M + uy[b],
                            ctx->ri, mod + off, (int)mld, shift_c * H, scale_c * H, ctx->d.ln_eps, h, H, st);
    stats.kernel_launches++;
  };
  // Y recording (template pass): the block output's image rows -> compute dtype -> D2H
  auto record_y = [&](int b) {
    if (!record || !record->y || !blk_yrec(record->ymode, b)) return;
    const int yb = b % R;
    const size_t plane = (size_t)ctx->Limg * H * es;
    char* ys = (char*)ctx->yrec + (size_t)yb * plane;
    stream_wait(ctx, st, ctx->ev_yrec[yb]);  // the D2H of block b - R is done
    launch_rows_to<T>(ctx->X + (long long)M_txt * H, ys, (long long)ctx->Limg * H, st);
    stats.kernel_launches++;
    if (record->fp8) {  // quantize per (token, head) into the FP8 Y staging, then D2H data + scales
      const size_t pl = (size_t)ctx->Limg * H, spl = (size_t)ctx->Limg * ctx->d.heads;
      uint8_t* qd = ctx->q8yrec + (size_t)yb * 2 * pl;
      float* qs = ctx->q8yrec_scl + (size_t)yb * 2 * spl;
      launch_kv_quant((const bf16*)ys, (const bf16*)ys, ctx->Limg, H, ctx->d.heads, qd, qd + pl, qs, qs + spl, st);
      stats.kernel_launches++;
      cudaEventRecord(ctx->ev_comp[yb], st);
      cudaStreamWaitEvent(ctx->copy_st, ctx->ev_comp[yb], 0);
      cudaMemcpyAsync(cache_plane(ctx, record, record_step, b, 2), qd, pl, cudaMemcpyDefault, ctx->copy_st);
      cudaMemcpyAsync(cache_scales(ctx, record, record_step, b, 2), qs, spl * 4, cudaMemcpyDefault, ctx->copy_st);
      const long long by = (long long)(pl + spl * 4);
      if (record->tier == IG_CACHE_HOST) stats.d2h_bytes += by; else stats.d2d_bytes += by;
      cudaEventRecord(ctx->ev_yrec[yb], ctx->copy_st);
      return;
    }
    cudaEventRecord(ctx->ev_comp[yb], st);
    cudaStreamWaitEvent(ctx->copy_st, ctx->ev_comp[yb], 0);
    cudaMemcpyAsync(cache_plane(ctx, record, record_step, b, 2), ys, plane, cudaMemcpyDefault, ctx->copy_st);
    if (record->tier == IG_CACHE_HOST) stats.d2h_bytes += plane; else stats.d2d_bytes += plane;
    cudaEventRecord(ctx->ev_yrec[yb], ctx->copy_st);
  };
  auto attn = [&](int buf, bool dense) {
    if (ctx->dbg[IG_DBG_SPIN_COMPUTE_NS]) {  // slow compute lane (WAR race test)
      launch_spin((unsigned long long)ctx->dbg[IG_DBG_SPIN_COMPUTE_NS], st);
      ctx->pdl_block = true;
    }
    AttnArgs a{};
    a.Q = ctx->Q; a.ldq = H; a.O = cat; a.ldo = ldcat; a.kv_arena = ctx->kv_arena;
    a.kv_off = (long long)buf * ctx->buf_elems;
    a.segs = dense ? dsegf : dseg; a.nseg = dense ? nsegf : nseg; a.max_qlen = dense ? max_qf : max_q;
    a.n_pairs = dense ? npairf : npair;
    a.q_rows = dense ? M_full : M;
    a.L = ctx->L; a.heads = ctx->d.heads; a.head_dim = ctx->d.head_dim;
    a.scale = 1.0f / sqrtf((float)ctx->d.head_dim);
    attention(ctx, a, st, 4.0 * (double)(dense ? M_full : M) * ctx->L * H);
  };
  // cache recording (template mode): image-token K/V of ring buffer -> cache[s][b]
  auto record_kv = [&](int b, int buf) {
    if (!record || (record->y && !blk_kv(record->ymode, b))) return;
    cudaEventRecord(ctx->ev_comp[buf], st);
    cudaStreamWaitEvent(ctx->copy_st, ctx->ev_comp[buf], 0);
    const size_t plane = (size_t)ctx->Limg * H * es;
    const char* src = (const char*)ctx->kv_arena + ((size_t)sr[0].r->slot * ctx->slot_stride + (size_t)buf * ctx->buf_elems) * es;
    const size_t txt_off = (size_t)Lt * H * es;
    const size_t vplane = (size_t)ctx->L * H * es;
    if (record->fp8) {  // quantize on the compute stream into the recording staging, then D2H
      const size_t pl = (size_t)ctx->Limg * H, spl = (size_t)ctx->Limg * ctx->d.heads;
      uint8_t* qd = ctx->q8rec + (size_t)buf * 2 * pl;
      float* qs = ctx->q8rec_scl + (size_t)buf * 2 * spl;
      launch_kv_quant((const bf16*)(src + txt_off), (const bf16*)(src + vplane + txt_off), ctx->Limg, H,
                      ctx->d.heads, qd, qd + pl, qs, qs + spl, st);
      cudaEventRecord(ctx->ev_comp[buf], st);
      cudaStreamWaitEvent(ctx->copy_st, ctx->ev_comp[buf], 0);
      for (int w = 0; w < 2; ++w) {
        cudaMemcpyAsync(cache_plane(ctx, record, record_step, b, w), qd + w * pl, pl, cudaMemcpyDefault, ctx->copy_st);
        cudaMemcpyAsync(cache_scales(ctx, record, record_step, b, w), qs + w * spl, spl * 4, cudaMemcpyDefault,
                        ctx->copy_st);
      }
      const long long by = 2LL * (pl + spl * 4);
      if (record->tier == IG_CACHE_HOST) stats.d2h_bytes += by; else stats.d2d_bytes += by;
    } else {
      cudaMemcpyAsync(cache_plane(ctx, record, record_step, b, 0), src + txt_off, plane, cudaMemcpyDefault, ctx->copy_st);
      cudaMemcpyAsync(cache_plane(ctx, record, record_step, b, 1), src + vplane + txt_off, plane, cudaMemcpyDefault,
                      ctx->copy_st);
      if (record->tier == IG_CACHE_HOST) stats.d2h_bytes += 2 * plane; else stats.d2d_bytes += 2 * plane;
    }
    cudaEventRecord(ctx->ev_copy[buf], ctx->copy_st);
  };
  // full-L copies (copy_mode 0) and the host tier's strided DMA groups (copy_mode 1, which may
  // cover masked rows) also write masked rows, so they must land before the fresh K/V merge;
  // the SM gathers touch only unmasked rows and are awaited right before attention
  bool host_dma = false;
  for (auto& q : sr)
    host_dma |= q.use_cache && q.r->cache->tier == IG_CACHE_HOST && ctx->o.copy_mode == 1;
  const bool late_wait = ctx->o.copy_mode != 0 && !record && !host_dma;
  const bool drop_raw = ctx->dbg[IG_DBG_DROP_RAW] != 0;  // negative control of the race tests
  auto wait_copy = [&](int buf) {
    if ((any_cache || record) && !late_wait && !(drop_raw && !record)) {
      lane_ready();
      stream_wait(ctx, st, ctx->ev_copy[buf]);
    }
  };
  auto wait_copy_late = [&](int buf) {
    if (any_cache && late_wait && !drop_raw) {
      lane_ready();
      stream_wait(ctx, st, ctx->ev_copy[buf]);
    }
  };

  // ---- UNet BasicTransformerBlock (config 5; oracle/unet.py unet_block_masked) ----
  // x += SelfAttn(LN1 x) [masked Q x all L_img K/V: fresh rows merged with the cache by mask
  // index]; x += CrossAttn(LN2 x, context K/V computed fresh); x += GEGLU-FF(LN3 x).
  const int Lc = ctx->d.ctx_len, Dc = ctx->d.ctx_dim;
  auto ln_aff = [&](int b, int which, int r0, int r1) {  // LayerNorm affine as LN-modulation (beta, gamma - 1)
    if (r1 <= r0) return;
    ProfScope ps(ctx, st, IG_K_LNMOD, 0.0, (double)(r1 - r0) * H * (4 + es));
    launch_ln_mod<T>(ctx->X, H, r0, r1, ctx->ri, ctx->unet_ln + ((size_t)b * 3 + which) * 2 * H, 0, 0, H,
                     ctx->d.ln_eps, h, H, st);
    stats.kernel_launches++;
  };
  auto ln_aff_y = [&](int b, int buf) {  // Y block: LN1 of the unmasked rows from the staged Y_{b-1}
    lane_ready();
    stream_wait(ctx, st, ctx->ev_copy[buf]);
    ProfScope ps(ctx, st, IG_K_LNMOD, 0.0, (double)uy[b] * H * (es + es));
    launch_ln_mod_staged<T>(ctx->kv_arena, ctx->slot_stride, (long long)buf * ctx->buf_elems, ctx->L, H, M, M + uy[b],
                            ctx->ri, ctx->unet_ln + (size_t)b * 3 * 2 * H, 0, 0, H, ctx->d.ln_eps, h, H, st);
    stats.kernel_launches++;
  };
  // fused (bf16) path: block b's cross K/V live in arena half b % 2 and are produced on the side
  // stream one block ahead (xover); parity mode: half 0, on the compute stream
  const bool no_xover = !ig_tuning_ref().cross_kv_overlap;
  const bool xover = unet && fused_qkv && !no_xover;
  const long long xhalf = (long long)ctx->o.max_batch * 2 * Lc * H;  // elements per arena half
  auto xkv_of = [&](int b) { return (char*)ctx->xkv + (xover ? (long long)(b & 1) * xhalf * es : 0); };
  auto cross_kv_on = [&](const UnetW& u, int b, cudaStream_t s2) {
    const int Mc = na * Lc;
    GemmArgs g{};
    g.A = ctx->ctxp; g.lda = Dc; g.B = u.kv2.w; g.ldb = Dc; g.bias = nullptr;
    g.C = ctx->Q; g.ldc = H; g.M = Mc; g.N = 2 * H; g.K = Dc; g.epi = EPI_QKV;
    g.ri = ctx->ri_c; g.ri_off = 0;
    QkvEpi& e = g.qkv;
    e.Q = ctx->Q; e.kv_arena = xkv_of(b); e.slot_stride = 2LL * Lc * H; e.buf_off = 0; e.L = Lc; e.H = H;
    e.head_dim = ctx->d.head_dim; e.col_base = H;
    if (s2 == st) gemm(ctx, g, st);
    else gemm_side(ctx, g, s2);
  };
  // side stream: produce block b's cross K/V (after block b - 2's cross-attention released the half)
  auto xissue = [&](int b) {
    if (b >= b1) return;
    if (b >= b0 + 2) cudaStreamWaitEvent(ctx->xs, ctx->ev_xuse[b & 1], 0);
    cross_kv_on(ctx->unet[b], b, ctx->xs);
    cudaEventRecord(ctx->ev_xkv[b & 1], ctx->xs);
  };
  auto cross_kv = [&](const UnetW& u) {  // context rows -> K/V planes of the cross arena
    const int Mc = na * Lc;
    if (fused_qkv) {
      cross_kv_on(u, 0, st);
    } else {  // parity mode: K/V GEMM into the [q|k|v] scratch, then the positional write
      GemmArgs g{};
      g.A = ctx->ctxp; g.lda = Dc; g.B = u.kv2.w; g.ldb = Dc;
      g.C = (char*)qkv + (long long)H * es; g.ldc = 3 * H; g.M = Mc; g.N = 2 * H; g.K = Dc; g.epi = EPI_STORE;
      gemm(ctx, g, st);
      QkvPost p{};
      p.qkv = qkv; p.ld_qkv = 3 * H; p.Q = ctx->Q; p.kv_arena = ctx->xkv;
      p.slot_stride = 2LL * Lc * H; p.buf_off = 0; p.L = Lc; p.H = H;
      p.heads = ctx->d.heads; p.head_dim = ctx->d.head_dim; p.r0 = 0; p.r1 = Mc;
      ProfScope ps(ctx, st, IG_K_QKVPOST, 0.0, (double)Mc * 6.0 * H * es);
      launch_qkv_post<T>(p, ctx->ri_c, st);
      stats.kernel_launches++;
    }
  };
  // ys: a Y block after the first cached one (unmasked rows [M, M + uy[b]) enter from the staged
  // Y_{b-1}); Mk: rows through LN1 + the K/V projection (the Y requests' unmasked rows included)
  // dense: an Algorithm-1 prefix block (all rows [0, M_full), own K/V buffer, no cache)
  auto unet_block = [&](int b, int buf, bool ys, int Mk, bool dense) {
    const UnetW& u = ctx->unet[b];
    const int Mc = dense ? M_full : M;
    if (xover) xissue(b + 1);  // next block's cross K/V, concurrently with this block's chain
    else cross_kv(u);  // parity path first: its positional write also stores (unused) Q rows
    ln_aff(b, 0, 0, dense ? M_full : (ys ? M : Mk));
    if (ys) ln_aff_y(b, buf);
    if (!dense) wait_copy(buf);
    qkv_proj(0, Mc, u.qkv, nullptr, nullptr, nullptr, buf);
    if (!dense) {
      kv_proj(M, M + uy[b], u.qkv, nullptr, nullptr, buf);
      wait_copy_late(buf);
    }
    attn(buf, dense);
    record_kv(b, buf);
    if (!dense) {
      cudaEventRecord(ctx->ev_comp[buf], st);
      if (ctx->capturing) ctx->cap_mask |= 1u << buf;
      if (b + R < b1 && !seq_load) issue_copy(ctx, sr, dkvg, dkvq, b + R, plan);
    }
    gemm_rows(0, Mc, cat, ldcat, u.out1.w, u.out1.b, H, H, ctx->X, H, EPI_GATED_RES, ctx->ones, 0);
    ln_aff(b, 1, 0, Mc);
    gemm_rows(0, Mc, h, H, u.q2.w, nullptr, H, H, ctx->Q, H, EPI_STORE, nullptr, 0);
    {
      if (xover) stream_wait(ctx, st, ctx->ev_xkv[b & 1]);
      AttnArgs a{};
      a.Q = ctx->Q; a.ldq = H; a.O = cat; a.ldo = ldcat; a.kv_arena = xkv_of(b); a.kv_off = 0;
      a.segs = dense ? dsegcf : dsegc; a.nseg = dense ? nsegcf : nsegc; a.max_qlen = dense ? max_qcf : max_q;
      a.n_pairs = dense ? npaircf : npair; a.q_rows = Mc;
      a.L = Lc; a.heads = ctx->d.heads; a.head_dim = ctx->d.head_dim;
      a.scale = 1.0f / sqrtf((float)ctx->d.head_dim);
      attention(ctx, a, st, 4.0 * (double)Mc * Lc * H);
      if (xover) cudaEventRecord(ctx->ev_xuse[b & 1], st);
    }
    gemm_rows(0, Mc, cat, ldcat, u.out2.w, u.out2.b, H, H, ctx->X, H, EPI_GATED_RES, ctx->ones, 0);
    ln_aff(b, 2, 0, Mc);
    GemmArgs gg{};  // fused: GEGLU in the tcgen05 epilogue (tile-interleaved weight copy)
    gg.A = h; gg.lda = H; gg.B = u.geglu_w_tc; gg.ldb = H; gg.bias = u.geglu_b_tc;
    gg.C = cat + H; gg.ldc = ldcat; gg.M = Mc; gg.N = 2 * F; gg.K = H; gg.epi = EPI_GEGLU;
    if (u.geglu_w_tc && g_tc_gemm && gemm_tc_supported(gg)) {
      gemm(ctx, gg, st);
    } else {
      gemm_rows(0, Mc, h, H, u.geglu.w, u.geglu.b, 2 * F, H, ctx->u2, 2 * F, EPI_STORE, nullptr, 0);
      ProfScope ps(ctx, st, IG_K_LNMOD, 0.0, (double)Mc * 3 * F * es);
      launch_geglu<T>((const T*)ctx->u2, 2 * F, Mc, F, cat + H, ldcat, st);
      stats.kernel_launches++;
    }
    gemm_rows(0, Mc, cat + H, ldcat, u.ff2.w, u.ff2.b, H, F, ctx->X, H, EPI_GATED_RES, ctx->ones, 0);
  };

  if (xover && b0 < b1) {  // fork the side stream after the packed contexts exist
    cudaEventRecord(ctx->ev_xfork, st);
    cudaStreamWaitEvent(ctx->xs, ctx->ev_xfork, 0);
    xissue(b0);
  }
  // ---- blocks ----
  // Dense-prefix blocks (b < kplan) run every row [0, M_full) with their own K/V buffer (index
  // R, no cache); cached blocks run the masked rows [0, M) with ring buffer b % R.
  for (int b = b0; b < b1; ++b) {
    const bool dense = b < kplan;
    const int Mc = dense ? M_full : M;    // rows through every op of the block
    const int Mk = dense ? M_full : M + uy[b];  // rows through LN-mod and the K/V projection
    const int buf = dense ? R : b % R;
    const bool ys = !dense && y_staged(b);
    cur_b = b;
    if (seq_load && !dense && any_cache) {
      cudaEventRecord(ctx->ev_comp[buf], st);  // everything enqueued so far (block b-1) ...
      issue_copy(ctx, sr, dkvg, dkvq, b, plan);  // ... precedes this block's copy
    }
    if (unet) {
      unet_block(b, buf, ys, Mk, dense);
    } else if (b < ctx->d.n_double) {
      const StreamW& wi = ctx->dimg[b];
      const StreamW& wt = ctx->dtxt[b];
      // text-stream ops on ts, concurrent with the image stream's (rows [0, M_txt) vs [M_txt, Mc))
      // only for small problems (below ~4k rows a stream's GEMMs leave most SMs idle; a batch of
      // 8 Flux requests fills the GPU with either stream: measured neutral), and never in a
      // profiled step (per-launch events would time two streams sharing the SMs)
      const bool tov = ig_tuning_ref().txt_overlap && Lt > 0 && M_txt > 0 && Mc <= 4096 && !ctx->prof;
      auto on_ts = [&](int k, auto&& issue) {
        cudaEventRecord(ctx->ev_tfork[k], st);
        cudaStreamWaitEvent(ctx->ts, ctx->ev_tfork[k], 0);
        cudaStream_t st0 = st;
        st = ctx->ts;
        ctx->pdl_block = true;
        issue();
        cudaEventRecord(ctx->ev_tjoin[k], st);
        st = st0;
        ctx->pdl_block = true;
      };
      auto txt_pre = [&] {
        ln_mod(0, M_txt, wt.mod_t, wt.pre_only ? 1 : 0, wt.pre_only ? 0 : 1);
        qkv_proj(0, M_txt, wt.qkv.w, wt.qkv.b, wt.qg, wt.kg, buf);
      };
      if (tov) on_ts(0, txt_pre);
      ln_mod(M_txt, ys ? M : Mk, wi.mod_t, 0, 1);
      if (ys) ln_mod_y(b, buf, wi.mod_t, 0, 1);
      if (Lt && !tov) ln_mod(0, M_txt, wt.mod_t, wt.pre_only ? 1 : 0, wt.pre_only ? 0 : 1);
      if (!dense) wait_copy(buf);
      qkv_proj(M_txt, Mc, wi.qkv.w, wi.qkv.b, wi.qg, wi.kg, buf);
      if (!dense) kv_proj(M, M + uy[b], wi.qkv.w, wi.qkv.b, wi.kg, buf);
      if (Lt && !tov) qkv_proj(0, M_txt, wt.qkv.w, wt.qkv.b, wt.qg, wt.kg, buf);
      if (tov) stream_wait(ctx, st, ctx->ev_tjoin[0]);
      if (!dense) wait_copy_late(buf);
      attn(buf, dense);
      record_kv(b, buf);
      if (!dense) {
        cudaEventRecord(ctx->ev_comp[buf], st);
        if (ctx->capturing) ctx->cap_mask |= 1u << buf;
        if (b + R < b1 && !seq_load) issue_copy(ctx, sr, dkvg, dkvq, b + R, plan);
      }
      const long long gi = ctx->mods[wi.mod_t].off;
      auto txt_post = [&] {
        const long long gt = ctx->mods[wt.mod_t].off;
        gemm_rows(0, M_txt, cat, ldcat, wt.proj.w, wt.proj.b, H, H, ctx->X, H, EPI_GATED_RES, mod + gt + 2 * H, 0);
        ln_mod(0, M_txt, wt.mod_t, 3, 4);
        gemm_rows(0, M_txt, h, H, wt.fc1.w, wt.fc1.b, F, H, cat + H, ldcat, EPI_GELU, nullptr, 0);
        gemm_rows(0, M_txt, cat + H, ldcat, wt.fc2.w, wt.fc2.b, H, F, ctx->X, H, EPI_GATED_RES, mod + gt + 5 * H, 0);
      };
      const bool tpost = Lt && !wt.pre_only;
      if (tov && tpost) on_ts(1, txt_post);
      gemm_rows(M_txt, Mc, cat, ldcat, wi.proj.w, wi.proj.b, H, H, ctx->X, H, EPI_GATED_RES, mod + gi + 2 * H, 0);
      ln_mod(M_txt, Mc, wi.mod_t, 3, 4);
      gemm_rows(M_txt, Mc, h, H, wi.fc1.w, wi.fc1.b, F, H, cat + H, ldcat, EPI_GELU, nullptr, 0);
      gemm_rows(M_txt, Mc, cat + H, ldcat, wi.fc2.w, wi.fc2.b, H, F, ctx->X, H, EPI_GATED_RES, mod + gi + 5 * H, 0);
      if (tov && tpost) stream_wait(ctx, st, ctx->ev_tjoin[1]);
      else if (tpost) txt_post();
    } else {
      const SingleW& ws = ctx->sgl[b - ctx->d.n_double];
      ln_mod(0, ys ? M : Mk, ws.mod_t, 0, 1);
      if (ys) ln_mod_y(b, buf, ws.mod_t, 0, 1);
      const char* w_u = (const char*)ws.lin1.w + 3LL * H * H * es;
      const char* b_u = (const char*)ws.lin1.b + 3LL * H * es;
      gemm_rows(0, Mc, h, H, w_u, b_u, F, H, cat + H, ldcat, EPI_GELU, nullptr, 0);
      if (!dense) wait_copy(buf);
      qkv_proj(0, Mc, ws.lin1.w, ws.lin1.b, ws.qg, ws.kg, buf);
      if (!dense) kv_proj(M, M + uy[b], ws.lin1.w, ws.lin1.b, ws.kg, buf);
      if (!dense) wait_copy_late(buf);
      attn(buf, dense);
      record_kv(b, buf);
      if (!dense) {
        cudaEventRecord(ctx->ev_comp[buf], st);
        if (ctx->capturing) ctx->cap_mask |= 1u << buf;
        if (b + R < b1 && !seq_load) issue_copy(ctx, sr, dkvg, dkvq, b + R, plan);
      }
      const long long gs = ctx->mods[ws.mod_t].off;
      gemm_rows(0, Mc, cat, ldcat, ws.lin2.w, ws.lin2.b, H, H + F, ctx->X, H, EPI_GATED_RES, mod + gs + 2 * H, 0);
    }
    record_y(b);
  }
  if (rng.X_out) {
    CUDA_TRY(cudaMemcpyAsync(rng.X_out, ctx->X, (size_t)M * H * 4, cudaMemcpyDeviceToDevice, st));
  } else if (unet) {  // exit: the stack's output rows back into the level's hidden state
    ProfScope ps(ctx, st, IG_K_ROWS, 0.0, 2.0 * M * H * 4);
    launch_scatter_rows(dreq, M, ctx->ri, H, ctx->X, st);
    stats.kernel_launches++;
  } else {
    // ---- a11: final layer + Euler scatter ----
    ln_mod(M_txt, M, ctx->fmod_t, 1, 0);  // final chunk order (scale, shift)
    gemm_rows(M_txt, M, h, H, ctx->pout.w, ctx->pout.b, C, H, ctx->vel - (long long)M_txt * C, C, EPI_STORE, nullptr, 1);
    launch_scatter_euler(dreq, na, M_img, ctx->ri, M_txt, C, ctx->vel, st);
    stats.kernel_launches++;
  }
  if (ctx->capturing) {  // end the capture (copy lane joins back), instantiate, launch
    cudaEventRecord(ctx->ev_join, ctx->copy_st);
    cudaStreamWaitEvent(st, ctx->ev_join, 0);
    cudaGraph_t graph = nullptr;
    cudaError_t ce = cudaStreamEndCapture(st, &graph);
    ctx->capturing = false;
    if (ce != cudaSuccess) return set_err(IG_ECUDA, "step capture: %s", cudaGetErrorString(ce));
    cudaGraphExec_t exec = nullptr;
    // a new step shape usually replaces an old one (a request left, another joined): update the
    // least recently used graph of the same topology in place instead of instantiating (measured
    // 16-160 ms per instantiate of a 343-node SD3 step while steps are queued, ~1 ms update).
    // Only graphs not launched in the last NSTAGE steps qualify: the ev_stage wait at the top of
    // this step guarantees those launches completed.
    {
      std::vector<std::pair<unsigned long long, std::string>> cand;
      for (auto& g : ctx->graphs)
        if (g.second.last_used + NSTAGE <= step_no) cand.push_back({g.second.last_used, g.first});
      std::sort(cand.begin(), cand.end());
      for (size_t i = 0; i < cand.size() && i < 4 && !exec; ++i) {
        auto git = ctx->graphs.find(cand[i].second);
        cudaGraphExecUpdateResultInfo info{};
        if (cudaGraphExecUpdate(git->second.exec, graph, &info) == cudaSuccess) {
          exec = git->second.exec;
          ctx->graphs.erase(git);
#ifdef IG_GRAPH_UPDATE_TRACE
          fprintf(stderr, "IG_GRAPH_UPDATE_TRACE: step %llu updated a graph last used at step %llu\n", step_no,
                  cand[i].first);
#endif
        } else {
          // a topology mismatch is not an error of the step; the stale candidate is dropped so
          // that a partially updated exec can never be replayed under its old key
          (void)cudaGetLastError();
          cudaGraphExecDestroy(git->second.exec);
          ctx->graphs.erase(git);
        }
      }
    }
    if (!exec) ce = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ce != cudaSuccess) return set_err(IG_ECUDA, "graph instantiate: %s", cudaGetErrorString(ce));
    if (ctx->graphs.size() >= 64) {  // bounded: batch compositions change under continuous batching
      for (auto& g : ctx->graphs) cudaGraphExecDestroy(g.second.exec);
      ctx->graphs.clear();
    }
    ctx->graphs[gkey] = ig_ctx::GraphEnt{exec, stats, step_no};
    CUDA_TRY(cudaGraphLaunch(exec, st));
    ctx->graph_tail = true;
    ctx->graph_st = st;
  }
  // the copy lane must not run ahead into the next step's buffers before compute is done
  CUDA_TRY(cudaEventRecord(ctx->ev_stage[si], st));
  for (auto& s : sr)
    if (s.use_cache) CUDA_TRY(cudaLaunchHostFunc(st, unpin_cb, (void*)s.r->cache));
  if (record)
    CUDA_TRY(cudaStreamWaitEvent(st, record->y && blk_yrec(record->ymode, b1 - 1) ? ctx->ev_yrec[(b1 - 1) % R]
                                                                                 : ctx->ev_copy[(b1 - 1) % R], 0));
  ctx->pdl_block = true;
  if (ctx->lane_on) {  // every copy of this step enqueued (the jobs reference sr / plan)
    lane_drain(ctx);
    stats.h2d_bytes += ctx->cstats.h2d_bytes;
    stats.d2d_bytes += ctx->cstats.d2d_bytes;
    stats.kernel_launches += ctx->cstats.kernel_launches;
    stats.dma_calls += ctx->cstats.dma_calls;
    ctx->cstats = ig_stats{};
    ctx->lane_on = false;
  }
  if (ctx->copy_err != cudaSuccess) {
    const cudaError_t ce = ctx->copy_err;
    ctx->copy_err = cudaSuccess;
    cudaGetLastError();
    return set_err(IG_ECUDA, "cache prefetch enqueue failed (copy %zu): %s", ctx->copy_err_idx, cudaGetErrorString(ce));
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(IG_ECUDA, "step enqueue: %s", cudaGetErrorString(e));
  stats.host_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t_host0).count();
  return IG_OK;
}

static ig_status step_dispatch(ig_ctx* ctx, const ig_edit_req* reqs, int n, cudaStream_t st,
                               ig_cache* record, int record_step, const StepRange& rng = StepRange()) {
  if (ctx->d.dtype == IG_F32) return run_step<float>(ctx, reqs, n, st, record, record_step, rng);
  return run_step<bf16>(ctx, reqs, n, st, record, record_step, rng);
}

extern "C" ig_status ig_debug_block(ig_ctx* ctx, const ig_edit_req* req, int block, const float* X_in,
                                    float* X_out, void* stream) {
  if (!ctx || !req || !X_in || !X_out) return set_err(IG_EINVAL, "NULL argument");
  if (block < 0 || block >= ctx->nb) return set_err(IG_EINVAL, "block %d out of range", block);
  if (!req->mask || req->mask->n_m == 0) return set_err(IG_EINVAL, "debug block needs n_m > 0");
  CUDA_TRY(cudaSetDevice(ctx->device));
  StepRange rng;
  rng.b0 = block; rng.b1 = block + 1; rng.X_in = X_in; rng.X_out = X_out;
  cudaStream_t st = (cudaStream_t)stream;
  ig_status s = step_dispatch(ctx, req, 1, st, nullptr, 0, rng);
  if (s != IG_OK) return s;
  CUDA_TRY(cudaStreamSynchronize(st));
  return IG_OK;
}

extern "C" ig_status ig_edit_step(ig_ctx* ctx, const ig_edit_req* reqs, int n, void* stream) {
  if (!ctx) return set_err(IG_EINVAL, "ctx is NULL");
  CUDA_TRY(cudaSetDevice(ctx->device));
  reap_zombies(ctx);
  ig_status s = step_dispatch(ctx, reqs, n, (cudaStream_t)stream, nullptr, 0);
  if (s == IG_OK && ctx->o.debug_checks) {
    CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    for (int i = 0; i < n; ++i) {
      std::vector<float> lat((size_t)ctx->Limg * ctx->C);
      CUDA_TRY(cudaMemcpy(lat.data(), reqs[i].latent, lat.size() * 4, cudaMemcpyDefault));
      for (float v : lat)
        if (!std::isfinite(v)) return set_err(IG_ENUMERIC, "req %d: non-finite latent after step", i);
    }
  }
  return s;
}

static ig_status template_record(ig_ctx* ctx, float* latent, const void* txt, const float* cond_vec,
                                 const float* sigmas, int n_steps, ig_cache* c, cudaStream_t st) {
  ig_mask* ones = nullptr;
  ig_status s = get_ones_mask(ctx, &ones);
  if (s != IG_OK) return s;
  ig_stats total{};
  for (int k = 0; k < n_steps; ++k) {
    ig_edit_req r{};
    r.slot = 0; r.latent = latent; r.mask = ones; r.cache = nullptr; r.step = k;
    r.sigma = sigmas[k]; r.sigma_next = sigmas[k + 1]; r.txt = txt; r.cond_vec = cond_vec;
    cudaError_t el = cudaMemcpyAsync(cache_latent(ctx, c, k), latent, (size_t)ctx->Limg * ctx->C * 4,
                                     cudaMemcpyDefault, st);  // the template's input latent of step k
    if (el != cudaSuccess) return set_err(IG_ECUDA, "cache_template: %s", cudaGetErrorString(el));
    s = step_dispatch(ctx, &r, 1, st, c, k);
    if (s != IG_OK) return s;
    total.kernel_launches += ctx->stats.kernel_launches;
    total.d2h_bytes += ctx->stats.d2h_bytes;
    total.d2d_bytes += ctx->stats.d2d_bytes;
    total.rows += ctx->stats.rows;
  }
  cudaError_t e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->copy_st);
  if (e != cudaSuccess) return set_err(IG_ECUDA, "cache_template: %s", cudaGetErrorString(e));
  ctx->stats = total;
  return IG_OK;
}

extern "C" ig_status ig_record_step(ig_ctx* ctx, const ig_edit_req* req, ig_cache* cache, int step, void* stream) {
  if (!ctx || !req || !cache || !req->latent || (!req->cond_vec && ctx->d.n_unet == 0) ||
      ((ctx->Lt > 0 || ctx->d.n_unet > 0) && !req->txt))
    return set_err(IG_EINVAL, "NULL argument");
  if (!desc_equal(cache->desc, ctx->d)) return set_err(IG_ECACHE_INCOMPAT, "cache built for another model");
  if (step < 0 || step >= cache->n_steps) return set_err(IG_ECACHE_INCOMPAT, "step %d outside the cache schedule", step);
  if (cache->y != ctx->o.cache_y || cache->fp8 != ctx->o.cache_fp8) return set_err(IG_ECACHE_INCOMPAT, "cache kind differs from the ctx's");
  CUDA_TRY(cudaSetDevice(ctx->device));
  ig_mask* ones = nullptr;
  ig_status s = get_ones_mask(ctx, &ones);
  if (s != IG_OK) return s;
  cudaStream_t st = (cudaStream_t)stream;
  ig_edit_req r = *req;
  r.slot = 0; r.mask = ones; r.cache = nullptr; r.step = step;
  CUDA_TRY(cudaMemcpyAsync(cache_latent(ctx, cache, step), r.latent, (size_t)ctx->Limg * ctx->C * 4, cudaMemcpyDefault, st));
  return step_dispatch(ctx, &r, 1, st, cache, step);
}

extern "C" ig_status ig_cache_template(ig_ctx* ctx, float* latent, const void* txt, const float* cond_vec,
                                       const float* sigmas, int n_steps, int tier, void* stream,
                                       ig_cache** out) {
  if (!ctx || !latent || (!cond_vec && ctx->d.n_unet == 0) || !sigmas || !out || ((ctx->Lt > 0 || ctx->d.n_unet > 0) && !txt))
    return set_err(IG_EINVAL, "NULL argument");
  *out = nullptr;
  if (n_steps <= 0) return set_err(IG_EINVAL, "n_steps must be positive");
  CUDA_TRY(cudaSetDevice(ctx->device));
  ig_cache* c = nullptr;
  ig_status s = ig_cache_create(ctx, n_steps, tier, &c);
  if (s != IG_OK) return s;
  s = template_record(ctx, latent, txt, cond_vec, sigmas, n_steps, c, (cudaStream_t)stream);
  if (s != IG_OK) { free_cache_now(c); return s; }
  *out = c;
  return IG_OK;
}

extern "C" ig_status ig_cache_template_into(ig_ctx* ctx, float* latent, const void* txt, const float* cond_vec,
                                            const float* sigmas, int n_steps, ig_cache* cache, void* stream) {
  if (!ctx || !latent || (!cond_vec && ctx->d.n_unet == 0) || !sigmas || !cache ||
      ((ctx->Lt > 0 || ctx->d.n_unet > 0) && !txt))
    return set_err(IG_EINVAL, "NULL argument");
  if (!desc_equal(cache->desc, ctx->d)) return set_err(IG_ECACHE_INCOMPAT, "cache built for another model");
  if (n_steps <= 0 || n_steps > cache->n_steps)
    return set_err(IG_ECACHE_INCOMPAT, "n_steps %d outside the cache schedule [1, %d]", n_steps, cache->n_steps);
  if (cache->y != ctx->o.cache_y || cache->fp8 != ctx->o.cache_fp8 ||
      (cache->y && cache->kv_blocks != std::max(0, std::min(ctx->o.cache_kv_blocks, ctx->nb))))
    return set_err(IG_ECACHE_INCOMPAT, "cache kind differs from the ctx's cache options");
  if (cache->pins.load() != 0) return set_err(IG_EINVAL, "cache is in use by an enqueued step");
  CUDA_TRY(cudaSetDevice(ctx->device));
  return template_record(ctx, latent, txt, cond_vec, sigmas, n_steps, cache, (cudaStream_t)stream);
}

extern "C" ig_status ig_debug_set(ig_ctx* ctx, int key, long long value) {
  if (!ctx) return set_err(IG_EINVAL, "ctx is NULL");
  if (key <= 0 || key > IG_DBG_SEQUENTIAL) return set_err(IG_EINVAL, "unknown debug key %d", key);
  CUDA_TRY(cudaSetDevice(ctx->device));
  if (key == IG_DBG_POISON_RING) {  // immediate: every ring buffer of every slot -> NaN
    CUDA_TRY(cudaDeviceSynchronize());
    flush_graph_tail(ctx);
    CUDA_TRY(cudaMemset(ctx->kv_arena, 0xFF, (size_t)ctx->o.max_batch * ctx->slot_stride * ctx->esz));
    CUDA_TRY(cudaDeviceSynchronize());
    for (auto& p : ctx->pref) p = ig_ctx::Pref{};
    return IG_OK;
  }
  if (value < 0) return set_err(IG_EINVAL, "debug value must be >= 0");
  ctx->dbg[key] = value;
  return IG_OK;
}

extern "C" ig_status ig_debug_dump_kv(ig_ctx* ctx, int slot, int block, void* k_out, void* v_out, void* stream) {
  if (!ctx || !k_out || !v_out) return set_err(IG_EINVAL, "NULL argument");
  if (slot < 0 || slot >= ctx->o.max_batch) return set_err(IG_EINVAL, "slot %d out of range", slot);
  if (block < 0 || block >= ctx->nb) return set_err(IG_EINVAL, "block %d out of range", block);
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = (cudaStream_t)stream;
  const size_t plane = (size_t)ctx->L * ctx->H * ctx->esz;
  const char* src = (const char*)ctx->kv_arena + ((size_t)slot * ctx->slot_stride + (size_t)(block % ctx->R) * ctx->buf_elems) * ctx->esz;
  CUDA_TRY(cudaStreamSynchronize(st));
  CUDA_TRY(cudaStreamSynchronize(ctx->copy_st));
  CUDA_TRY(cudaMemcpyAsync(k_out, src, plane, cudaMemcpyDefault, st));
  CUDA_TRY(cudaMemcpyAsync(v_out, src + plane, plane, cudaMemcpyDefault, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return IG_OK;
}

extern "C" ig_status ig_prefetch_layer(ig_ctx* ctx, const ig_edit_req* r, int layer) {
  if (!ctx || !r) return set_err(IG_EINVAL, "NULL argument");
  if (layer < 0 || layer >= ctx->nb) return set_err(IG_EINVAL, "layer %d out of range", layer);
  if (layer >= ctx->R) return set_err(IG_EINVAL, "layer %d beyond the ring depth %d", layer, ctx->R);
  if (r->slot < 0 || r->slot >= ctx->o.max_batch) return set_err(IG_EINVAL, "slot out of range");
  if (!r->cache) return set_err(IG_ECACHE_MISS, "no cache");
  if (!desc_equal(r->cache->desc, ctx->d)) return set_err(IG_ECACHE_INCOMPAT, "cache built for another model");
  if (r->step < 0 || r->step >= r->cache->n_steps) return set_err(IG_ECACHE_INCOMPAT, "step out of range");
  if (ctx->o.copy_mode != 0 || r->cache->fp8 || r->cache->y)
    return set_err(IG_EUNSUPPORTED, "explicit prefetch needs copy_mode 0 and a bf16 K/V cache");
  CUDA_TRY(cudaSetDevice(ctx->device));
  const int buf = layer % ctx->R;
  const size_t es = ctx->esz, H = ctx->H;
  const size_t plane = (size_t)ctx->Limg * H * es;
  flush_graph_tail(ctx);
  CUDA_TRY(cudaStreamWaitEvent(ctx->copy_st, ctx->ev_comp[buf], 0));
  const char* src = cache_plane(ctx, r->cache, r->step, layer, 0);
  char* dst = (char*)ctx->kv_arena + ((size_t)r->slot * ctx->slot_stride + (size_t)buf * ctx->buf_elems) * es;
  const size_t txt_off = (size_t)ctx->Lt * H * es, vplane = (size_t)ctx->L * H * es;
  CUDA_TRY(cudaMemcpyAsync(dst + txt_off, src, plane, cudaMemcpyDefault, ctx->copy_st));
  CUDA_TRY(cudaMemcpyAsync(dst + vplane + txt_off, src + plane, plane, cudaMemcpyDefault, ctx->copy_st));
  CUDA_TRY(cudaEventRecord(ctx->ev_copy[buf], ctx->copy_st));
  ctx->pref[(size_t)r->slot * ctx->R + buf] = ig_ctx::Pref{r->cache, r->step};
  return IG_OK;
}

// ----------------------------------------------------------------------------------------
// per-kernel ops (include/ig_ops.h)
// ----------------------------------------------------------------------------------------
extern "C" ig_status ig_op_gemm(int dtype, const void* A, long long lda, const void* B, long long ldb,
                                const void* bias, void* Cp, long long ldc, int M, int N, int K, int epi,
                                int out_f32, void* stream) {
  if (!A || !B || !Cp) return set_err(IG_EINVAL, "NULL argument");
  if (M < 0 || N <= 0 || K <= 0) return set_err(IG_EINVAL, "bad shape");
  if (epi != EPI_STORE && epi != EPI_GELU && !(epi == EPI_GEGLU && dtype == IG_BF16 && !out_f32))
    return set_err(IG_EINVAL, "ig_op_gemm: epi must be 0 or 1 (or 5 = GEGLU, bf16 output)");
  GemmArgs g{};
  g.A = A; g.lda = lda; g.B = B; g.ldb = ldb; g.bias = bias; g.C = Cp; g.ldc = ldc;
  g.M = M; g.N = N; g.K = K; g.epi = epi; g.out_f32 = out_f32;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == IG_F32) launch_gemm_simt<float>(g, st);
  else if (dtype == IG_BF16) {
    if (!gemm_tc_supported(g)) return set_err(IG_EUNSUPPORTED, "shape not supported by the tcgen05 GEMM");
    launch_gemm_tc(g, st);
  } else return set_err(IG_EINVAL, "bad dtype");
  CUDA_TRY(cudaGetLastError());
  return IG_OK;
}

extern "C" ig_status ig_op_gemm_gated(int dtype, const void* A, long long lda, const void* B, long long ldb,
                                      const void* bias, float* X, long long ldx, const float* gate, int M, int N,
                                      int K, void* stream) {
  if (!A || !B || !X || !gate) return set_err(IG_EINVAL, "NULL argument");
  if (M < 0 || N <= 0 || K <= 0) return set_err(IG_EINVAL, "bad shape");
  cudaStream_t st = (cudaStream_t)stream;
  RowInfo* ri = nullptr;  // every row belongs to request 0
  if (M > 0) {
    CUDA_TRY(cudaMallocAsync((void**)&ri, (size_t)M * sizeof(RowInfo), st));
    CUDA_TRY(cudaMemsetAsync(ri, 0, (size_t)M * sizeof(RowInfo), st));
  }
  GemmArgs g{};
  g.A = A; g.lda = lda; g.B = B; g.ldb = ldb; g.bias = bias; g.C = X; g.ldc = ldx;
  g.M = M; g.N = N; g.K = K; g.epi = EPI_GATED_RES; g.gate = gate; g.gate_ld = 0; g.ri = ri; g.ri_off = 0;
  if (dtype == IG_F32) launch_gemm_simt<float>(g, st);
  else if (dtype == IG_BF16) {
    if (!gemm_tc_supported(g)) { if (ri) cudaFreeAsync(ri, st); return set_err(IG_EUNSUPPORTED, "shape not supported by the tcgen05 GEMM"); }
    launch_gemm_tc(g, st);
  } else return set_err(IG_EINVAL, "bad dtype");
  if (ri) CUDA_TRY(cudaFreeAsync(ri, st));
  CUDA_TRY(cudaGetLastError());
  return IG_OK;
}

extern "C" ig_status ig_op_attention(int dtype, const void* Q, long long ldq, void* O, long long ldo,
                                     const void* kv, const int32_t* segs, int nseg, int L, int heads,
                                     int head_dim, void* stream) {
  if (!Q || !O || !kv || !segs || nseg <= 0 || L <= 0 || heads <= 0) return set_err(IG_EINVAL, "bad argument");
  if (dtype != IG_F32 && dtype != IG_BF16) return set_err(IG_EINVAL, "bad dtype");
  if (head_dim != 16 && head_dim != 64 && head_dim != 128) return set_err(IG_EUNSUPPORTED, "head_dim");
  std::vector<AttnSeg> hs(nseg);
  int maxq = 0;
  const long long H = (long long)heads * head_dim;
  for (int i = 0; i < nseg; ++i) {
    hs[i] = AttnSeg{segs[3 * i], segs[3 * i + 1], (long long)segs[3 * i + 2] * 2 * L * H};
    if (hs[i].q_len < 0 || hs[i].q_start < 0) return set_err(IG_EINVAL, "bad segment");
    maxq = std::max(maxq, hs[i].q_len);
  }
  cudaStream_t st = (cudaStream_t)stream;
  AttnSeg* dsegs = nullptr;
  CUDA_TRY(cudaMallocAsync((void**)&dsegs, nseg * sizeof(AttnSeg), st));
  CUDA_TRY(cudaMemcpyAsync(dsegs, hs.data(), nseg * sizeof(AttnSeg), cudaMemcpyHostToDevice, st));
  AttnArgs a{};
  a.Q = Q; a.ldq = ldq; a.O = O; a.ldo = ldo; a.kv_arena = kv; a.kv_off = 0; a.segs = dsegs;
  a.nseg = nseg; a.max_qlen = maxq; a.L = L; a.heads = heads; a.head_dim = head_dim;
  for (auto& sg : hs) a.n_pairs += (sg.q_len + 255) / 256;
  int qrows = 1;
  for (auto& s : hs) qrows = std::max(qrows, s.q_start + s.q_len);
  a.q_rows = qrows;
  a.scale = 1.0f / sqrtf((float)head_dim);
  const int rep = ig_tuning_ref().op_repeat;  // benchmarking aid: launch the kernel N times
  for (int it = 0; it < rep; ++it) {
    if (dtype == IG_F32) launch_attn_simt<float>(a, st);
    else if (dtype == IG_BF16) {
      if (g_tc_attn && attn_tc_supported(a)) launch_attn_tc(a, st);
      else launch_attn_simt<bf16>(a, st);
    } else return set_err(IG_EINVAL, "bad dtype");
  }
  CUDA_TRY(cudaFreeAsync(dsegs, st));
  CUDA_TRY(cudaStreamSynchronize(st));  // host segment vector lifetime
  CUDA_TRY(cudaGetLastError());
  return IG_OK;
}

extern "C" ig_status ig_op_conv3x3(const void* x_padded, int n_img, int H, int W, int cin, const void* w,
                                   const void* bias, int cout, float* y, void* stream) {
  if (!x_padded || !w || !y) return set_err(IG_EINVAL, "NULL argument");
  if (n_img <= 0 || H <= 0 || W <= 0 || cin <= 0 || cout <= 0 || cin % 8)
    return set_err(IG_EINVAL, "bad shape (C_in must be a multiple of 8)");
  cudaStream_t st = (cudaStream_t)stream;
  GemmArgs g{};
  g.B = w; g.ldb = 9LL * cin; g.bias = bias; g.C = y; g.ldc = cout;
  g.M = n_img * H * W; g.N = cout; g.K = 9 * cin; g.epi = EPI_STORE; g.out_f32 = 1;
  if (cout % 4) return set_err(IG_EUNSUPPORTED, "C_out must be a multiple of 4");
  if (conv3x3_tc_supported(H, W, cin)) {
    g.A = x_padded; g.lda = cin; g.conv_H = H; g.conv_W = W; g.conv_cin = cin;
    launch_conv3x3_tc(g, st);
  } else {  // im2col of the padded input + the tcgen05 GEMM
    bf16* col = nullptr;
    CUDA_TRY(cudaMallocAsync((void**)&col, (size_t)g.M * 9 * cin * 2, st));
    launch_im2col_padded((const bf16*)x_padded, cin, n_img, H, W, 9 * cin, col, st);
    g.A = col; g.lda = 9LL * cin;
    launch_gemm_tc(g, st);
    CUDA_TRY(cudaFreeAsync(col, st));
  }
  CUDA_TRY(cudaGetLastError());
  return IG_OK;
}

extern "C" ig_status ig_stage_input(void* dst, const void* src, size_t bytes, void* stream) {
  if ((!dst || !src) && bytes) return set_err(IG_EINVAL, "NULL argument");
  if (bytes == 0) return IG_OK;
  cudaPointerAttributes pa{};
  if (cudaPointerGetAttributes(&pa, src) != cudaSuccess || pa.type != cudaMemoryTypeHost || !pa.devicePointer) {
    cudaGetLastError();
    return set_err(IG_EINVAL, "ig_stage_input: src must be pinned (page-locked, mapped) host memory");
  }
  launch_copy_bytes(dst, pa.devicePointer, bytes, (cudaStream_t)stream);
  CUDA_TRY(cudaGetLastError());
  return IG_OK;
}

extern "C" ig_status ig_copy(void* dst, const void* src, size_t bytes, void* stream) {
  if ((!dst || !src) && bytes) return set_err(IG_EINVAL, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return IG_OK;
}

// ---- process-wide tuning (include/ig_ops.h) ------------------------------------------------
static std::mutex g_tuning_mu;
static ig_tuning g_tuning;
static std::atomic<bool> g_tuning_init{false};
static void tuning_seed_locked() {
  if (g_tuning_init.load(std::memory_order_relaxed)) return;
  auto off = [](const char* v) { return getenv(v) != nullptr ? 0 : 1; };
  g_tuning.pdl = off("IG_NO_PDL");
  g_tuning.copy_thread = off("IG_NO_COPY_THREAD");
  g_tuning.load_dedupe = off("IG_NO_DEDUPE");
  g_tuning.cross_kv_overlap = off("IG_NO_XOVERLAP");
  g_tuning.gemm_two_cta = off("IG_GEMM_1CTA");
  g_tuning.gemm_small_tiles = off("IG_GEMM_NO_SMALL");
  g_tuning.gemm_bn64 = off("IG_GEMM_NO_BN64");
  g_tuning.conv_two_cta = off("IG_CONV_1CTA");
  g_tuning.precise_gelu = getenv("IG_PRECISE_GELU") != nullptr ? 1 : 0;
  const char* rep = getenv("IG_OP_REPEAT");
  g_tuning.op_repeat = rep ? std::max(1, atoi(rep)) : 1;
  g_tuning.txt_overlap = off("IG_NO_TXT_OVERLAP");
  g_tuning_init.store(true, std::memory_order_release);
}
const ig_tuning& ig_tuning_ref() {
  if (!g_tuning_init.load(std::memory_order_acquire)) {
    std::lock_guard<std::mutex> lk(g_tuning_mu);
    tuning_seed_locked();
  }
  return g_tuning;
}
extern "C" ig_status ig_tuning_get(ig_tuning* out) {
  if (!out) return set_err(IG_EINVAL, "ig_tuning_get: null");
  std::lock_guard<std::mutex> lk(g_tuning_mu);
  tuning_seed_locked();
  *out = g_tuning;
  return IG_OK;
}
extern "C" ig_status ig_tuning_set(const ig_tuning* t) {
  if (!t || t->op_repeat < 1) return set_err(IG_EINVAL, "ig_tuning_set: null or op_repeat < 1");
  std::lock_guard<std::mutex> lk(g_tuning_mu);
  g_tuning = *t;
  g_tuning_init.store(true, std::memory_order_release);
  return IG_OK;
}
