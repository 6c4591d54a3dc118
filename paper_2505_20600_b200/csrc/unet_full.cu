// unet_full.cu — the whole-UNet mask-aware step (include/ig_unet.h; BASELINE config 5, SURVEY
// N2).  Host runtime: parses the SDXL-layout weight table, owns one attention-stack ig_ctx per
// Transformer2D (its blocks on the level's masked rows with the K/V cache: ig_edit_step of
// ig_api.cu), and sequences the dense parts — GroupNorm (+SiLU) into zero-padded NHWC bf16,
// implicit-GEMM tcgen05 3x3 convolutions with fused epilogues (per-image timestep term, bias,
// residual), im2col + tcgen05 GEMM for the strided / 4-channel / narrow-level convolutions,
// nearest upsampling — over the whole batch.  Oracle: oracle/unet_full.py.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ig.h"
#include "../../include/ig_unet.h"
#include "ig_internal.h"
#include "kernels.h"
#include "unet_kernels.h"

using namespace ig;

namespace {

ig_status uerr(ig_status s, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  return ig_internal_err(s, buf);
}
#define UTRY(expr)                                                                              \
  do {                                                                                          \
    cudaError_t e_ = (expr);                                                                    \
    if (e_ != cudaSuccess) return uerr(IG_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)
#define ITRY(expr)                                                                              \
  do {                                                                                          \
    ig_status s_ = (expr);                                                                      \
    if (s_ != IG_OK) return s_;  /* the callee set ig_last_error() */                           \
  } while (0)

struct Lin { const bf16* w = nullptr; const bf16* b = nullptr; int out = 0, in = 0; };

struct Res {
  std::string name;
  int lvl, ci, co;
  const bf16 *gn1g, *gn1b, *gn2g, *gn2b;
  Lin conv1, temb, conv2, skip;  // conv weights [co][9*ci]; skip only when ci != co
  long long temb_off = 0;        // column offset in the packed timestep-projection output
};

struct T2D {
  std::string name;
  int lvl, C, depth;
  const bf16 *gng, *gnb;
  Lin proj_in, proj_out;
  ig_ctx* sub = nullptr;         // the block stack (ig.h UNet model, n_unet = depth)
  long long y_off = 0;           // float offset of this Transformer2D's output plane in a step's Y region
};

enum OpKind { OP_RES, OP_T2D, OP_DOWN, OP_UP, OP_PUSH };
struct Op { OpKind k; int idx; int lvl; };

}  // namespace

struct ig_unet_mask {
  ig_mask* m[3] = {nullptr, nullptr, nullptr};
  int n_m[3] = {0, 0, 0};
  int P[3] = {0, 0, 0};
};

struct ig_unet_cache {
  int n_steps = 0, tier = 0;
  std::vector<ig_cache*> kv;     // per Transformer2D
  float* y = nullptr;            // [n_steps][y_floats] (host pinned mapped or device)
  float* ydev = nullptr;
  size_t y_floats = 0;
  const ig_unet* owner = nullptr;
};

struct ig_unet {
  ig_unet_desc d{};
  int device = 0, B = 8, R = 2;
  int P[3] = {0, 0, 0}, G[3] = {0, 0, 0};
  int E = 0;
  std::vector<const void*> w;
  Lin t1, t2, conv_in, conv_out;
  const bf16 *out_gng = nullptr, *out_gnb = nullptr;
  std::vector<Res> res;
  std::vector<T2D> t2d;
  std::vector<Lin> down, up;     // resampler convs (down.{0,1}, up.{0,1})
  std::vector<Op> ops;
  // packed timestep projections of every ResBlock: [sum co][E] + bias
  bf16* tw = nullptr;
  bf16* tb = nullptr;
  long long t_ld = 0;
  bf16* conv_in_w = nullptr;     // [c0][40] (K = 36 padded to a multiple of 8)
  int conv_in_kp = 0;
  GemvProb* gv = nullptr;        // [2] time MLP GEMVs
  size_t y_floats = 0;
  // workspaces
  float *lat = nullptr, *sinu = nullptr, *tv1 = nullptr, *tv2 = nullptr, *scale = nullptr, *eps = nullptr;
  bf16 *tsilu = nullptr, *tproj = nullptr;
  float* lvl_buf[3][4] = {};      // per level: 4 fp32 [B*P][Cmax_l] working tensors
  std::vector<float*> skip_buf;   // skip tensors (down path), exact sizes
  int skip_C[16] = {};
  int skip_lvl[16] = {};
  bf16* pad = nullptr;            // zero-padded NHWC bf16 (largest level x channels)
  bf16* col = nullptr;            // im2col / packed bf16 rows
  bf16* catb = nullptr;           // [x1 | x2] bf16 (skip projection operand)
  float* pk1 = nullptr;           // packed fp32 rows (proj_in / proj_out outputs)
  float* T[3] = {};               // per level: the stacks' per-request state [B][P][C] fp32
  float2 *gpart = nullptr, *gstats = nullptr, *gcoef = nullptr;
  size_t pad_elems = 0, col_elems = 0;
  ig_mask* ones[3] = {};
  // per-step descriptors (pinned mapped host -> device)
  char* h_desc = nullptr;
  char* d_desc = nullptr;
  size_t desc_bytes = 0;
  cudaEvent_t ev_desc = nullptr;
  ig_stats stats{};
};

namespace {

int rup(int x, int m) { return (x + m - 1) / m * m; }

// ---------------------------------------------------------------------------------------- graph
// The execution order of synth.unet_full_weight_table: ResBlocks, Transformer2Ds, resamplers.
void build_ops(ig_unet* u) {
  const ig_unet_desc& d = u->d;
  int c = d.ch[0];
  std::vector<int> skipc = {c}, skipl = {0};
  auto add_res = [&](const std::string& nm, int lvl, int ci, int co) {
    Res r{};
    r.name = nm; r.lvl = lvl; r.ci = ci; r.co = co;
    u->res.push_back(r);
    u->ops.push_back({OP_RES, (int)u->res.size() - 1, lvl});
  };
  auto add_t2d = [&](const std::string& nm, int lvl) {
    T2D t{};
    t.name = nm; t.lvl = lvl; t.C = d.ch[lvl]; t.depth = d.depth[lvl];
    u->t2d.push_back(t);
    u->ops.push_back({OP_T2D, (int)u->t2d.size() - 1, lvl});
  };
  for (int lvl = 0; lvl < 3; ++lvl) {
    for (int r = 0; r < d.n_res; ++r) {
      add_res("down." + std::to_string(lvl) + ".res." + std::to_string(r), lvl, c, d.ch[lvl]);
      c = d.ch[lvl];
      if (d.depth[lvl]) add_t2d("down." + std::to_string(lvl) + ".attn." + std::to_string(r), lvl);
      u->ops.push_back({OP_PUSH, 0, lvl});
      skipc.push_back(c); skipl.push_back(lvl);
    }
    if (lvl < 2) {
      u->ops.push_back({OP_DOWN, lvl, lvl});
      u->ops.push_back({OP_PUSH, 0, lvl + 1});
      skipc.push_back(c); skipl.push_back(lvl + 1);
    }
  }
  add_res("mid.res.0", 2, c, c);
  add_t2d("mid.attn.0", 2);
  add_res("mid.res.1", 2, c, c);
  const int lvls[3] = {2, 1, 0};
  for (int j = 0; j < 3; ++j) {
    const int lvl = lvls[j];
    for (int r = 0; r <= d.n_res; ++r) {
      const int cs = skipc.back();
      skipc.pop_back(); skipl.pop_back();
      add_res("up." + std::to_string(j) + ".res." + std::to_string(r), lvl, c + cs, d.ch[lvl]);
      c = d.ch[lvl];
      if (d.depth[lvl]) add_t2d("up." + std::to_string(j) + ".attn." + std::to_string(r), lvl);
    }
    if (lvl > 0) u->ops.push_back({OP_UP, j, lvl});
  }
}

}  // namespace

extern "C" int ig_unet_weight_count(const ig_unet_desc* d) {
  if (!d) return -1;
  ig_unet tmp;
  tmp.d = *d;
  build_ops(&tmp);
  int n = 4 + 2;  // time MLP, conv_in
  for (auto& r : tmp.res) n += 10 + (r.ci != r.co ? 2 : 0);
  for (auto& t : tmp.t2d) n += 6 + 17 * t.depth;
  n += 2 * 2 + 2 * 2;  // resamplers
  n += 4;              // out.gn, conv_out
  return n;
}

extern "C" void ig_unet_destroy(ig_unet* u);

extern "C" ig_status ig_unet_create(const ig_unet_desc* desc, const void* const* weights, int n_weights, int device,
                                    int max_batch, int prefetch_depth, ig_unet** out) {
  if (!desc || !weights || !out) return uerr(IG_EINVAL, "NULL argument");
  *out = nullptr;
  const ig_unet_desc& d = *desc;
  for (int l = 0; l < 3; ++l)
    if (d.ch[l] <= 0 || d.ch[l] % 64 || d.depth[l] < 0) return uerr(IG_EUNSUPPORTED, "channels must be positive multiples of 64");
  if (d.depth[0] != 0 || d.depth[2] <= 0) return uerr(IG_EUNSUPPORTED, "depth = (0, d1, d2 > 0) (SDXL layout)");
  if (d.grid % 4 || d.grid < 8 || d.lat_ch <= 0 || d.lat_ch % 4 || d.head_dim != 64 || d.n_res <= 0 ||
      d.gn_groups <= 0 || d.ch[0] % d.gn_groups || d.ctx_len <= 0 || d.ctx_dim % 8)
    return uerr(IG_EUNSUPPORTED, "unsupported UNet shape");
  const int nw = ig_unet_weight_count(desc);
  if (n_weights != nw) return uerr(IG_EINVAL, "expected %d weight pointers, got %d", nw, n_weights);
  for (int i = 0; i < nw; ++i)
    if (!weights[i]) return uerr(IG_EINVAL, "weight %d is NULL", i);
  if (max_batch <= 0 || max_batch > 16) return uerr(IG_EUNSUPPORTED, "max_batch must be in [1, 16]");
  UTRY(cudaSetDevice(device));
  ig_unet* u = new ig_unet();
  u->d = d;
  u->device = device;
  u->B = max_batch;
  u->R = std::max(1, prefetch_depth) + 1;
  u->E = 4 * d.ch[0];
  for (int l = 0; l < 3; ++l) u->P[l] = (d.grid >> l) * (d.grid >> l);
  build_ops(u);
  u->w.assign(weights, weights + nw);
  // ---- resolve the table (synth.unet_full_weight_table order)
  int k = 0;
  auto W = [&]() { return (const bf16*)weights[k++]; };
  auto lin = [&](Lin& l, int o, int i, bool bias = true) { l.w = W(); l.b = bias ? W() : nullptr; l.out = o; l.in = i; };
  lin(u->t1, u->E, d.ch[0]);
  lin(u->t2, u->E, u->E);
  lin(u->conv_in, d.ch[0], 9 * d.lat_ch);
  u->down.resize(2);
  u->up.resize(2);
  size_t yoff = 0;
  for (auto& op : u->ops) {
    if (op.k == OP_RES) {
      Res& r = u->res[op.idx];
      r.gn1g = W(); r.gn1b = W();
      lin(r.conv1, r.co, 9 * r.ci);
      lin(r.temb, r.co, u->E);
      r.gn2g = W(); r.gn2b = W();
      lin(r.conv2, r.co, 9 * r.co);
      if (r.ci != r.co) lin(r.skip, r.co, r.ci);
    } else if (op.k == OP_T2D) {
      T2D& t = u->t2d[op.idx];
      t.gng = W(); t.gnb = W();
      lin(t.proj_in, t.C, t.C);
      std::vector<const void*> sw(weights + k, weights + k + 17 * t.depth);
      k += 17 * t.depth;
      lin(t.proj_out, t.C, t.C);
      t.y_off = (long long)yoff;
      yoff += (size_t)u->P[t.lvl] * t.C;
      // the block stack: ig.h UNet model (n_unet = depth, hidden = C, d = 64)
      ig_model_desc md{};
      md.n_unet = t.depth; md.hidden = t.C; md.heads = t.C / d.head_dim; md.head_dim = d.head_dim;
      md.mlp_hidden = 4 * t.C; md.lat_ch = t.C; md.grid_h = md.grid_w = d.grid >> t.lvl; md.txt_len = 0;
      md.ln_eps = d.ln_eps; md.rope_theta = 10000.f; md.dtype = IG_BF16; md.ctx_len = d.ctx_len; md.ctx_dim = d.ctx_dim;
      ig_ctx_opts o{};
      o.max_batch = max_batch; o.prefetch_depth = std::max(1, prefetch_depth); o.copy_mode = 1;
      ig_status s = ig_ctx_create(&md, sw.data(), (int)sw.size(), device, &o, &t.sub);
      if (s != IG_OK) { const std::string m = ig_last_error(); ig_unet_destroy(u); return ig_internal_err(s, m.c_str()); }
    } else if (op.k == OP_DOWN) {
      lin(u->down[op.idx], d.ch[op.idx], 9 * d.ch[op.idx]);
    } else if (op.k == OP_UP) {
      const int lvl = op.lvl;
      lin(u->up[op.idx], d.ch[lvl], 9 * d.ch[lvl]);
    }
  }
  u->out_gng = W(); u->out_gnb = W();
  lin(u->conv_out, d.lat_ch, 9 * d.ch[0]);
  u->y_floats = yoff;
  if (k != nw) { ig_unet_destroy(u); return uerr(IG_EINVAL, "weight table walk consumed %d of %d", k, nw); }

  // ---- derived weights: packed timestep projections, padded conv_in
  auto dm = [&](void** p, size_t bytes) { return cudaMalloc(p, std::max<size_t>(bytes, 256)) == cudaSuccess; };
  bool ok = true;
  long long tot = 0;
  for (auto& r : u->res) { r.temb_off = tot; tot += r.co; }
  u->t_ld = tot;
  ok &= dm((void**)&u->tw, (size_t)tot * u->E * 2);
  ok &= dm((void**)&u->tb, (size_t)tot * 2);
  u->conv_in_kp = rup(9 * d.lat_ch, 8);
  ok &= dm((void**)&u->conv_in_w, (size_t)d.ch[0] * u->conv_in_kp * 2);
  if (!ok) { ig_unet_destroy(u); return uerr(IG_ENOMEM, "weight pack allocation failed"); }
  for (auto& r : u->res) {
    UTRY(cudaMemcpy(u->tw + r.temb_off * u->E, r.temb.w, (size_t)r.co * u->E * 2, cudaMemcpyDeviceToDevice));
    UTRY(cudaMemcpy(u->tb + r.temb_off, r.temb.b, (size_t)r.co * 2, cudaMemcpyDeviceToDevice));
  }
  UTRY(cudaMemset(u->conv_in_w, 0, (size_t)d.ch[0] * u->conv_in_kp * 2));
  UTRY(cudaMemcpy2D(u->conv_in_w, (size_t)u->conv_in_kp * 2, u->conv_in.w, (size_t)9 * d.lat_ch * 2,
                    (size_t)9 * d.lat_ch * 2, d.ch[0], cudaMemcpyDeviceToDevice));
  // time MLP GEMVs: lin1 (SiLU out) and lin2
  {
    GemvProb p[2];
    p[0] = GemvProb{u->t1.w, u->t1.b, nullptr, nullptr, nullptr, u->E, d.ch[0], d.ch[0], u->E, 0, 1, 0};
    p[1] = GemvProb{u->t2.w, u->t2.b, nullptr, nullptr, nullptr, u->E, u->E, u->E, u->E, 0, 0, 0};
    ok &= dm((void**)&u->gv, sizeof(p));
    ok &= dm((void**)&u->sinu, (size_t)max_batch * d.ch[0] * 4);
    ok &= dm((void**)&u->tv1, (size_t)max_batch * u->E * 4);
    ok &= dm((void**)&u->tv2, (size_t)max_batch * u->E * 4);
    if (!ok) { ig_unet_destroy(u); return uerr(IG_ENOMEM, "workspace allocation failed"); }
    p[0].x = u->sinu; p[0].y = u->tv1;
    p[1].x = u->tv1; p[1].y = u->tv2;
    UTRY(cudaMemcpy(u->gv, p, sizeof(p), cudaMemcpyHostToDevice));
  }
  // ---- workspaces
  const long long B = max_batch;
  int cmax[3] = {0, 0, 0}, cin_max[3] = {0, 0, 0};
  for (auto& r : u->res) {
    cmax[r.lvl] = std::max(cmax[r.lvl], std::max(r.ci, r.co));
    cin_max[r.lvl] = std::max(cin_max[r.lvl], r.ci);
  }
  for (int l = 0; l < 3; ++l) {
    cmax[l] = std::max(cmax[l], d.ch[l]);
    for (int i = 0; i < 4; ++i) ok &= dm((void**)&u->lvl_buf[l][i], (size_t)B * u->P[l] * cmax[l] * 4);
    if (d.depth[l]) ok &= dm((void**)&u->T[l], (size_t)B * u->P[l] * d.ch[l] * 4);
    const int g = d.grid >> l;
    u->pad_elems = std::max(u->pad_elems, (size_t)B * (g + 2) * (g + 2) * cin_max[l]);
    u->pad_elems = std::max(u->pad_elems, (size_t)B * (g + 2) * (g + 2) * cmax[l]);
    u->col_elems = std::max(u->col_elems, (size_t)B * u->P[l] * 9 * cmax[l]);  // generic-path im2col
  }
  u->col_elems = std::max(u->col_elems, (size_t)B * u->P[0] * u->conv_in_kp);
  ok &= dm((void**)&u->pad, u->pad_elems * 2);
  ok &= dm((void**)&u->col, u->col_elems * 2);
  size_t catmax = 0, pkmax = 0;
  for (auto& r : u->res) if (r.ci != r.co) catmax = std::max(catmax, (size_t)B * u->P[r.lvl] * r.ci);
  for (auto& t : u->t2d) pkmax = std::max(pkmax, (size_t)B * u->P[t.lvl] * t.C);
  ok &= dm((void**)&u->catb, catmax * 2);
  ok &= dm((void**)&u->pk1, pkmax * 4);
  ok &= dm((void**)&u->lat, (size_t)B * u->P[0] * d.lat_ch * 4);
  ok &= dm((void**)&u->eps, (size_t)B * u->P[0] * d.lat_ch * 4);
  ok &= dm((void**)&u->scale, (size_t)B * 4);
  ok &= dm((void**)&u->tsilu, (size_t)B * u->E * 2);
  ok &= dm((void**)&u->tproj, (size_t)B * tot * 2);
  ok &= dm((void**)&u->gpart, (size_t)B * ((u->P[0] + 63) / 64) * d.gn_groups * sizeof(float2));
  ok &= dm((void**)&u->gstats, (size_t)B * d.gn_groups * sizeof(float2));
  {
    int cm = 0;
    for (auto& r : u->res) cm = std::max(cm, std::max(r.ci, r.co));
    ok &= dm((void**)&u->gcoef, (size_t)B * cm * sizeof(float2));
  }
  // the down path's skip tensors
  {
    int c = d.ch[0];
    auto add_skip = [&](int lvl, int ch) {
      float* p = nullptr;
      ok &= dm((void**)&p, (size_t)B * u->P[lvl] * ch * 4);
      u->skip_C[u->skip_buf.size()] = ch;
      u->skip_lvl[u->skip_buf.size()] = lvl;
      u->skip_buf.push_back(p);
    };
    add_skip(0, c);
    for (int lvl = 0; lvl < 3; ++lvl) {
      for (int r = 0; r < d.n_res; ++r) { c = d.ch[lvl]; add_skip(lvl, c); }
      if (lvl < 2) add_skip(lvl + 1, c);
    }
  }
  // per-step descriptors: UReq[B] + URows[3 levels][B] + URows unmasked[n_t2d][B] + URows[3][B] unmasked per level
  u->desc_bytes = (size_t)B * sizeof(UReq) + (size_t)(6 + u->t2d.size()) * B * sizeof(URows) + 256;
  ok &= cudaHostAlloc((void**)&u->h_desc, u->desc_bytes, cudaHostAllocMapped | cudaHostAllocPortable) == cudaSuccess;
  ok &= dm((void**)&u->d_desc, u->desc_bytes);
  if (!ok) { ig_unet_destroy(u); return uerr(IG_ENOMEM, "UNet workspace allocation failed"); }
  cudaEventCreateWithFlags(&u->ev_desc, cudaEventDisableTiming);
  // all-ones level masks (dense requests / template)
  for (int l = 0; l < 3; ++l) {
    std::vector<uint8_t> ones(u->P[l], 1);
    ITRY(ig_mask_build_host_L(device, u->P[l], ones.data(), nullptr, &u->ones[l], nullptr));
  }
  UTRY(cudaDeviceSynchronize());
  *out = u;
  return IG_OK;
}

extern "C" void ig_unet_destroy(ig_unet* u) {
  if (!u) return;
  cudaSetDevice(u->device);
  cudaDeviceSynchronize();
  for (auto& t : u->t2d) if (t.sub) ig_ctx_destroy(t.sub);
  for (int l = 0; l < 3; ++l) {
    for (int i = 0; i < 4; ++i) if (u->lvl_buf[l][i]) cudaFree(u->lvl_buf[l][i]);
    if (u->T[l]) cudaFree(u->T[l]);
    if (u->ones[l]) ig_mask_free(u->ones[l]);
  }
  for (float* p : u->skip_buf) if (p) cudaFree(p);
  void* bufs[] = {u->tw, u->tb, u->conv_in_w, u->gv, u->sinu, u->tv1, u->tv2, u->pad, u->col, u->catb, u->pk1,
                  u->lat, u->eps, u->scale, u->tsilu, u->tproj, u->gpart, u->gstats, u->gcoef, u->d_desc};
  for (void* b : bufs) if (b) cudaFree(b);
  if (u->h_desc) cudaFreeHost(u->h_desc);
  if (u->ev_desc) cudaEventDestroy(u->ev_desc);
  delete u;
}

// ------------------------------------------------------------------------------------ masks
static void any_pool2(const std::vector<uint8_t>& in, int g, std::vector<uint8_t>& out) {
  out.assign((size_t)(g / 2) * (g / 2), 0);
  for (int r = 0; r < g / 2; ++r)
    for (int c = 0; c < g / 2; ++c)
      out[(size_t)r * (g / 2) + c] = (in[(size_t)(2 * r) * g + 2 * c] | in[(size_t)(2 * r) * g + 2 * c + 1] |
                                      in[(size_t)(2 * r + 1) * g + 2 * c] | in[(size_t)(2 * r + 1) * g + 2 * c + 1]) != 0;
}

extern "C" ig_status ig_unet_mask_build(ig_unet* u, const uint8_t* mask, void* stream, ig_unet_mask** out, int* n_masked) {
  if (!u || !mask || !out) return uerr(IG_EINVAL, "NULL argument");
  *out = nullptr;
  std::vector<uint8_t> lv[3];
  lv[0].assign(mask, mask + u->P[0]);
  for (auto& v : lv[0]) v = v != 0;
  any_pool2(lv[0], u->d.grid, lv[1]);
  any_pool2(lv[1], u->d.grid / 2, lv[2]);
  ig_unet_mask* m = new ig_unet_mask();
  for (int l = 0; l < 3; ++l) {
    m->P[l] = u->P[l];
    ig_status s = ig_mask_build_host_L(u->device, u->P[l], lv[l].data(), stream, &m->m[l], &m->n_m[l], u->G[l],
                                       u->d.ch[l] * 2);
    if (s != IG_OK) {
      const std::string msg = ig_last_error();
      ig_unet_mask_free(m);
      return ig_internal_err(s, msg.c_str());
    }
  }
  if (n_masked) *n_masked = m->n_m[0];
  *out = m;
  return IG_OK;
}

extern "C" void ig_unet_mask_free(ig_unet_mask* m) {
  if (!m) return;
  for (int l = 0; l < 3; ++l) if (m->m[l]) ig_mask_free(m->m[l]);
  delete m;
}

extern "C" void ig_unet_cache_free(ig_unet_cache* c) {
  if (!c) return;
  for (auto* k : c->kv) if (k) ig_cache_free(k);
  if (c->y) {
    if (c->tier == IG_CACHE_HOST) cudaFreeHost(c->y);
    else cudaFree(c->y);
  }
  delete c;
}

extern "C" ig_status ig_unet_last_stats(const ig_unet* u, ig_stats* out) {
  if (!u || !out) return uerr(IG_EINVAL, "NULL argument");
  *out = u->stats;
  return IG_OK;
}

// ------------------------------------------------------------------------------------ the step
namespace {

struct Ctx {       // one forward pass
  ig_unet* u;
  cudaStream_t st;
  int n;           // requests
  const ig_unet_req* reqs;
  UReq* dreq;      // device descriptors
  URows* drows[3]; // masked rows per level
  URows* durows;   // unmasked rows per (T2D, request): [n_t2d][B]
  int max_rows[3], m_rows[3];
  const float* dscale = nullptr;  // per-image c_in
  std::vector<int> max_u;  // per T2D: max unmasked rows over requests
  ig_unet_cache* record = nullptr;  // template mode (n == 1, dense)
  int record_step = 0;
};

void gemm_launch(ig_unet* u, const GemmArgs& g, cudaStream_t st) {
  u->stats.kernel_launches++;
  launch_gemm_tc(g, st);
}

// y = conv3x3(pad) (+ epilogue): implicit GEMM when the tile walk applies, else im2col + GEMM
void conv(ig_unet* u, cudaStream_t st, int n, int H, int W, int cin, const Lin& w, GemmArgs g) {
  g.B = w.w; g.ldb = 9LL * cin; g.bias = w.b; g.N = w.out; g.K = 9 * cin; g.M = n * H * W;
  if (conv3x3_tc_supported(H, W, cin)) {
    g.A = u->pad; g.lda = cin;
    g.conv_H = H; g.conv_W = W; g.conv_cin = cin;
    u->stats.kernel_launches++;
    launch_conv3x3_tc(g, st);
  } else {
    launch_im2col_padded(u->pad, cin, n, H, W, 9 * cin, u->col, st);
    u->stats.kernel_launches++;
    g.A = u->col; g.lda = 9LL * cin;
    gemm_launch(u, g, st);
  }
}

void gn_stats(ig_unet* u, cudaStream_t st, const float* x1, int C1, const float* x2, int C2, int n, int P, float eps) {
  launch_gn_stats(x1, C1, x2, C2, n, P, u->d.gn_groups, eps, u->gpart, u->gstats, st);
  u->stats.kernel_launches += 2;
}

// ResBlock: out = skip(x) + conv2(SiLU(GN2(conv1(SiLU(GN1(x))) + temb)))
void resblock(Ctx& c, const Res& r, const float* x1, int C1, const float* x2, int C2, float* h1, float* sbuf, float* out) {
  ig_unet* u = c.u;
  const int g = u->d.grid >> r.lvl, P = u->P[r.lvl];
  gn_stats(u, c.st, x1, C1, x2, C2, c.n, P, u->d.gn_eps);
  launch_gn_apply_padded(x1, C1, x2, C2, u->gstats, r.gn1g, r.gn1b, u->d.gn_groups, 1, c.n, g, g, u->pad, u->gcoef, c.st);
  u->stats.kernel_launches += 2;
  GemmArgs a{};
  a.C = h1; a.ldc = r.co; a.epi = EPI_POS; a.pos = u->tproj + r.temb_off; a.pos_ld = u->t_ld; a.pos_div = P;
  conv(u, c.st, c.n, g, g, r.ci, r.conv1, a);
  gn_stats(u, c.st, h1, r.co, nullptr, 0, c.n, P, u->d.gn_eps);
  launch_gn_apply_padded(h1, r.co, nullptr, 0, u->gstats, r.gn2g, r.gn2b, u->d.gn_groups, 1, c.n, g, g, u->pad, u->gcoef, c.st);
  u->stats.kernel_launches += 2;
  const float* res = x1;
  if (r.ci != r.co) {  // 1x1 (linear) skip projection of [x1 | x2]
    launch_cat_bf16(x1, C1, x2, C2, (long long)c.n * P, u->catb, c.st);
    u->stats.kernel_launches++;
    GemmArgs s{};
    s.A = u->catb; s.lda = r.ci; s.B = r.skip.w; s.ldb = r.ci; s.bias = r.skip.b;
    s.C = sbuf; s.ldc = r.co; s.M = c.n * P; s.N = r.co; s.K = r.ci; s.epi = EPI_STORE; s.out_f32 = 1;
    gemm_launch(u, s, c.st);
    res = sbuf;
  }
  GemmArgs b{};
  b.C = out; b.ldc = r.co; b.epi = EPI_ADDRES; b.res = res;
  conv(u, c.st, c.n, g, g, r.co, r.conv2, b);
}

// Transformer2D: masked rows through GN -> proj_in -> the block stack (K/V cache) -> proj_out
// -> residual; unmasked rows from the template's cached output
ig_status transformer2d(Ctx& c, int ti, const float* x, float* out) {
  ig_unet* u = c.u;
  const T2D& t = u->t2d[ti];
  const int l = t.lvl, P = u->P[l], C = t.C;
  gn_stats(u, c.st, x, C, nullptr, 0, c.n, P, u->d.t2d_gn_eps);
  launch_t2d_in_rows(c.drows[l], c.n, c.max_rows[l], x, P, C, u->gstats, t.gng, t.gnb, u->d.gn_groups, u->col, c.st);
  u->stats.kernel_launches++;
  GemmArgs g{};
  g.A = u->col; g.lda = C; g.B = t.proj_in.w; g.ldb = C; g.bias = t.proj_in.b; g.C = u->pk1; g.ldc = C;
  g.M = c.m_rows[l]; g.N = C; g.K = C; g.epi = EPI_STORE; g.out_f32 = 1;
  gemm_launch(u, g, c.st);
  launch_rows_move(c.drows[l], c.n, c.max_rows[l], u->T[l], P, C, u->pk1, nullptr, 0, c.st);
  u->stats.kernel_launches++;
  // the block stack on the masked rows of each request's state (ig_edit_step of the sub-ctx)
  std::vector<ig_edit_req> rq(c.n);
  for (int i = 0; i < c.n; ++i) {
    const ig_unet_req& r = c.reqs[i];
    const bool dense = !r.mask || r.mask->n_m[0] == u->P[0];
    ig_edit_req e{};
    e.slot = i;
    e.latent = u->T[l] + (size_t)i * P * C;
    e.mask = dense ? u->ones[l] : r.mask->m[l];
    e.cache = (dense || !r.cache) ? nullptr : r.cache->kv[ti];
    e.step = r.step;
    e.sigma = r.sigma; e.sigma_next = r.sigma_next;
    e.txt = r.ctx;
    e.cond_vec = nullptr;
    rq[i] = e;
  }
  if (c.record) {
    ITRY(ig_record_step(t.sub, &rq[0], c.record->kv[ti], c.record_step, c.st));
  } else {
    ITRY(ig_edit_step(t.sub, rq.data(), c.n, c.st));
  }
  ig_stats ss{};
  ig_last_stats(t.sub, &ss);
  u->stats.kernel_launches += ss.kernel_launches;
  u->stats.h2d_bytes += ss.h2d_bytes;
  u->stats.d2d_bytes += ss.d2d_bytes;
  launch_rows_move(c.drows[l], c.n, c.max_rows[l], u->T[l], P, C, nullptr, u->col, 1, c.st);
  u->stats.kernel_launches++;
  g = GemmArgs{};
  g.A = u->col; g.lda = C; g.B = t.proj_out.w; g.ldb = C; g.bias = t.proj_out.b; g.C = u->pk1; g.ldc = C;
  g.M = c.m_rows[l]; g.N = C; g.K = C; g.epi = EPI_STORE; g.out_f32 = 1;
  gemm_launch(u, g, c.st);
  launch_t2d_out(c.drows[l], c.durows + (size_t)ti * u->B, c.n, c.max_rows[l] + c.max_u[ti], x, u->pk1, P, C, out, c.st);
  u->stats.kernel_launches++;
  if (c.record) {  // the template's Transformer2D output of this step (all rows) -> Y plane
    float* dst = c.record->y + (size_t)c.record_step * c.record->y_floats + t.y_off;
    UTRY(cudaMemcpyAsync(dst, out, (size_t)P * C * 4, cudaMemcpyDefault, c.st));
    if (c.record->tier == IG_CACHE_HOST) u->stats.d2h_bytes += (long long)P * C * 4;
  }
  return IG_OK;
}

ig_status forward(Ctx& c) {
  ig_unet* u = c.u;
  const ig_unet_desc& d = u->d;
  cudaStream_t st = c.st;
  const int n = c.n;
  // ---- timestep embedding and every ResBlock's projection of it
  launch_unet_sinusoid(c.dreq, n, d.ch[0], u->sinu, st);
  launch_gemv<bf16>(u->gv, 1, (u->E + 31) / 32, n, d.ch[0], st);
  launch_gemv<bf16>(u->gv + 1, 1, (u->E + 31) / 32, n, u->E, st);
  launch_temb_finish(c.dreq, n, u->E, u->tv2, u->tsilu, st);
  u->stats.kernel_launches += 4;
  {
    GemmArgs g{};
    g.A = u->tsilu; g.lda = u->E; g.B = u->tw; g.ldb = u->E; g.bias = u->tb; g.C = u->tproj; g.ldc = u->t_ld;
    g.M = n; g.N = (int)u->t_ld; g.K = u->E; g.epi = EPI_STORE;
    gemm_launch(u, g, st);
  }
  // ---- conv_in on the scaled latents (im2col: 4 channels)
  launch_gather_latents(c.dreq, n, u->P[0], d.lat_ch, u->lat, st);
  launch_im2col(u->lat, d.lat_ch, n, d.grid, d.grid, 1, c.dscale, u->conv_in_kp, u->col, st);
  u->stats.kernel_launches += 2;
  {
    GemmArgs g{};
    g.A = u->col; g.lda = u->conv_in_kp; g.B = u->conv_in_w; g.ldb = u->conv_in_kp; g.bias = u->conv_in.b;
    g.C = u->skip_buf[0]; g.ldc = d.ch[0]; g.M = n * u->P[0]; g.N = d.ch[0]; g.K = u->conv_in_kp;
    g.epi = EPI_STORE; g.out_f32 = 1;
    gemm_launch(u, g, st);
  }
  // ---- the U.  Outputs the down path keeps (ResBlock / Transformer2D outputs followed by a
  // push, downsampler outputs) are written straight into their skip buffers; everything else
  // rotates through the level's four working buffers.
  const float* h = u->skip_buf[0];
  int hc = d.ch[0];
  size_t next_skip = 1;
  std::vector<const float*> stack = {u->skip_buf[0]};
  std::vector<int> stackc = {d.ch[0]};
  auto free_bufs = [&](int lvl, const float* a, const float* b) {
    std::vector<float*> v;
    for (int i = 0; i < 4; ++i) {
      float* p = u->lvl_buf[lvl][i];
      if (p != a && p != b) v.push_back(p);
    }
    return v;
  };
  for (size_t oi = 0; oi < u->ops.size(); ++oi) {
    const Op& op = u->ops[oi];
    const bool next_push = oi + 1 < u->ops.size() && u->ops[oi + 1].k == OP_PUSH;
    if (op.k == OP_RES) {
      const Res& r = u->res[op.idx];
      const float* x2 = nullptr;
      int c2 = 0;
      if (r.name[0] == 'u') {  // up path: [h | skip] concatenation
        x2 = stack.back(); c2 = stackc.back();
        stack.pop_back(); stackc.pop_back();
      }
      auto fb = free_bufs(r.lvl, h, x2);
      float* out = next_push ? u->skip_buf[next_skip] : fb[2];
      resblock(c, r, h, hc, x2, c2, fb[0], fb[1], out);
      h = out;
      hc = r.co;
    } else if (op.k == OP_T2D) {
      float* out = next_push ? u->skip_buf[next_skip] : free_bufs(op.lvl, h, nullptr)[0];
      ig_status s = transformer2d(c, op.idx, h, out);
      if (s != IG_OK) return s;
      h = out;
    } else if (op.k == OP_PUSH) {
      stack.push_back(h); stackc.push_back(hc);
      ++next_skip;
    } else if (op.k == OP_DOWN) {  // conv3x3 stride 2 (im2col + GEMM), output pushed as a skip
      const int lvl = op.lvl, g = d.grid >> lvl, C = d.ch[lvl];
      launch_im2col(h, C, n, g, g, 2, nullptr, 9 * C, u->col, st);
      u->stats.kernel_launches++;
      GemmArgs ga{};
      ga.A = u->col; ga.lda = 9LL * C; ga.B = u->down[op.idx].w; ga.ldb = 9LL * C; ga.bias = u->down[op.idx].b;
      ga.C = u->skip_buf[next_skip]; ga.ldc = C; ga.M = n * u->P[lvl + 1]; ga.N = C; ga.K = 9 * C;
      ga.epi = EPI_STORE; ga.out_f32 = 1;
      gemm_launch(u, ga, st);
      h = u->skip_buf[next_skip];
    } else if (op.k == OP_UP) {  // nearest x2 + conv3x3
      const int lvl = op.lvl, g = d.grid >> lvl, C = d.ch[lvl];
      launch_upsample_padded(h, C, n, g, g, u->pad, st);
      u->stats.kernel_launches++;
      float* out = free_bufs(lvl - 1, nullptr, nullptr)[0];
      GemmArgs ga{};
      ga.C = out; ga.ldc = C; ga.epi = EPI_STORE; ga.out_f32 = 1;
      conv(u, st, n, 2 * g, 2 * g, C, u->up[op.idx], ga);
      h = out;
    }
  }
  // ---- out: GN -> SiLU -> conv_out -> eps; Euler on the masked latent rows
  gn_stats(u, st, h, d.ch[0], nullptr, 0, n, u->P[0], d.gn_eps);
  launch_gn_apply_padded(h, d.ch[0], nullptr, 0, u->gstats, u->out_gng, u->out_gnb, d.gn_groups, 1, n, d.grid, d.grid,
                         u->pad, u->gcoef, st);
  u->stats.kernel_launches += 2;
  GemmArgs go{};
  go.C = u->eps; go.ldc = d.lat_ch; go.epi = EPI_STORE; go.out_f32 = 1;
  conv(u, st, n, d.grid, d.grid, d.ch[0], u->conv_out, go);
  launch_unet_euler(c.dreq, c.drows[0], n, c.max_rows[0], u->P[0], d.lat_ch, u->eps, st);
  u->stats.kernel_launches++;
  return IG_OK;
}

// descriptors of a step -> pinned mapped staging -> device (one SM-driven copy on the stream)
ig_status stage_descriptors(Ctx& c) {
  ig_unet* u = c.u;
  UTRY(cudaEventSynchronize(u->ev_desc));  // the previous step consumed the staging
  const int B = u->B;
  char* hs = u->h_desc;
  UReq* hreq = (UReq*)hs;
  URows* hrows = (URows*)(hs + (size_t)B * sizeof(UReq));
  URows* hurows = hrows + 3 * B;
  for (int l = 0; l < 3; ++l) { c.max_rows[l] = 0; c.m_rows[l] = 0; }
  c.max_u.assign(u->t2d.size(), 0);
  for (int i = 0; i < c.n; ++i) {
    const ig_unet_req& r = c.reqs[i];
    UReq q{};
    q.latent = r.latent; q.cond = r.cond; q.sigma = r.sigma; q.dsig = r.sigma_next - r.sigma;
    q.c_in = (float)(1.0 / std::sqrt((double)r.sigma * r.sigma + 1.0));
    hreq[i] = q;
    const bool dense = !r.mask || r.mask->n_m[0] == u->P[0];
    for (int l = 0; l < 3; ++l) {
      URows w{};
      if (dense) { w.idx = nullptr; w.n = u->P[l]; }
      else {
        const int32_t *im = nullptr, *iu = nullptr;
        int nm = 0;
        ig_mask_indices(r.mask->m[l], &im, &iu, &nm);
        w.idx = im; w.n = nm;
      }
      w.row0 = c.m_rows[l];
      c.m_rows[l] += w.n;
      c.max_rows[l] = std::max(c.max_rows[l], w.n);
      hrows[l * B + i] = w;
    }
    for (size_t ti = 0; ti < u->t2d.size(); ++ti) {
      const int l = u->t2d[ti].lvl;
      URows w{};
      if (!dense) {
        const int32_t *im = nullptr, *iu = nullptr;
        int nm = 0;
        ig_mask_indices(r.mask->m[l], &im, &iu, &nm);
        w.idx = iu; w.n = u->P[l] - nm;
        w.y = r.cache->ydev + (size_t)r.step * r.cache->y_floats + u->t2d[ti].y_off;
      }
      c.max_u[ti] = std::max(c.max_u[ti], w.n);
      hurows[ti * B + i] = w;
    }
  }
  float* hscale = (float*)(hurows + u->t2d.size() * B);
  for (int i = 0; i < c.n; ++i) hscale[i] = hreq[i].c_in;
  launch_copy_bytes(u->d_desc, u->h_desc, u->desc_bytes, c.st);  // mapped staging -> device (SM copy)
  c.dreq = (UReq*)u->d_desc;
  c.drows[0] = (URows*)(u->d_desc + (size_t)B * sizeof(UReq));
  c.drows[1] = c.drows[0] + B;
  c.drows[2] = c.drows[0] + 2 * B;
  c.durows = c.drows[0] + 3 * B;
  // the per-image input scale lives right after the unmasked row lists
  c.dscale = (const float*)(c.durows + u->t2d.size() * B);
  return IG_OK;
}

}  // namespace

extern "C" ig_status ig_unet_step(ig_unet* u, const ig_unet_req* reqs, int n, void* stream) {
  if (!u) return uerr(IG_EINVAL, "NULL argument");
  if (n < 0 || n > u->B) return uerr(IG_EINVAL, "n = %d outside [0, max_batch = %d]", n, u->B);
  if (n > 0 && !reqs) return uerr(IG_EINVAL, "reqs is NULL");
  u->stats = ig_stats{};
  std::vector<ig_unet_req> live;
  for (int i = 0; i < n; ++i) {
    const ig_unet_req& r = reqs[i];
    if (!r.latent || !r.mask || !r.ctx) return uerr(IG_EINVAL, "req %d: NULL latent/mask/ctx", i);
    if (r.mask->P[0] != u->P[0]) return uerr(IG_EINVAL, "req %d: mask built for another UNet", i);
    if (r.mask->n_m[0] == 0) continue;  // nothing to compute, latent bit-identical
    const bool dense = r.mask->n_m[0] == u->P[0];
    if (!dense) {
      if (!r.cache) return uerr(IG_ECACHE_MISS, "req %d: partial mask and no cache (S:134)", i);
      if (r.cache->owner != u) return uerr(IG_ECACHE_INCOMPAT, "req %d: cache recorded by another UNet", i);
      if (r.step < 0 || r.step >= r.cache->n_steps)
        return uerr(IG_ECACHE_INCOMPAT, "req %d: step %d outside the cache schedule [0, %d)", i, r.step, r.cache->n_steps);
    }
    live.push_back(r);
  }
  if (live.empty()) return IG_OK;
  UTRY(cudaSetDevice(u->device));
  Ctx c{};
  c.u = u; c.st = (cudaStream_t)stream; c.n = (int)live.size(); c.reqs = live.data();
  ig_status s = stage_descriptors(c);
  if (s != IG_OK) return s;
  s = forward(c);
  UTRY(cudaEventRecord(u->ev_desc, c.st));
  if (s != IG_OK) return s;
  UTRY(cudaGetLastError());
  return IG_OK;
}

extern "C" ig_status ig_unet_template(ig_unet* u, float* latent, const void* ctx, const float* cond, const float* sigmas,
                                      int n_steps, int tier, void* stream, ig_unet_cache** out) {
  if (!u || !latent || !ctx || !sigmas || !out) return uerr(IG_EINVAL, "NULL argument");
  *out = nullptr;
  if (n_steps <= 0) return uerr(IG_EINVAL, "n_steps must be positive");
  if (tier != IG_CACHE_HOST && tier != IG_CACHE_DEVICE) return uerr(IG_EINVAL, "bad tier");
  UTRY(cudaSetDevice(u->device));
  ig_unet_cache* c = new ig_unet_cache();
  c->n_steps = n_steps; c->tier = tier; c->owner = u; c->y_floats = u->y_floats;
  for (auto& t : u->t2d) {
    ig_cache* k = nullptr;
    ig_status s = ig_cache_create(t.sub, n_steps, tier, &k);
    if (s != IG_OK) { const std::string msg = ig_last_error(); ig_unet_cache_free(c); return ig_internal_err(s, msg.c_str()); }
    c->kv.push_back(k);
  }
  const size_t ybytes = (size_t)n_steps * u->y_floats * 4;
  cudaError_t e = tier == IG_CACHE_HOST ? cudaHostAlloc((void**)&c->y, ybytes, cudaHostAllocMapped | cudaHostAllocPortable)
                                        : cudaMalloc((void**)&c->y, ybytes);
  if (e == cudaSuccess) {
    if (tier == IG_CACHE_HOST) e = cudaHostGetDevicePointer((void**)&c->ydev, c->y, 0);
    else c->ydev = c->y;
  }
  if (e != cudaSuccess) { cudaGetLastError(); ig_unet_cache_free(c); return uerr(IG_ENOMEM, "Y cache allocation: %s", cudaGetErrorString(e)); }
  ig_unet_mask ones;
  for (int l = 0; l < 3; ++l) { ones.m[l] = u->ones[l]; ones.n_m[l] = u->P[l]; ones.P[l] = u->P[l]; }
  cudaStream_t st = (cudaStream_t)stream;
  for (int k = 0; k < n_steps; ++k) {
    ig_unet_req r{};
    r.latent = latent; r.mask = &ones; r.cache = nullptr; r.step = k; r.sigma = sigmas[k]; r.sigma_next = sigmas[k + 1];
    r.ctx = ctx; r.cond = cond;
    Ctx cx{};
    cx.u = u; cx.st = st; cx.n = 1; cx.reqs = &r; cx.record = c; cx.record_step = k;
    ig_status s = stage_descriptors(cx);
    if (s == IG_OK) s = forward(cx);
    cudaEventRecord(u->ev_desc, st);
    if (s != IG_OK) { cudaStreamSynchronize(st); ig_unet_cache_free(c); return s; }
  }
  e = cudaStreamSynchronize(st);
  for (auto& t : u->t2d) if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { ig_unet_cache_free(c); return uerr(IG_ECUDA, "UNet template: %s", cudaGetErrorString(e)); }
  *out = c;
  return IG_OK;
}
