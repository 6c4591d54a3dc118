// k_conv.cu — the dense parts of the whole-UNet step (BASELINE config 5): GroupNorm
// statistics and application (fused SiLU, channel concatenation of the up path's skips, zero-
// padded NHWC output for the implicit-GEMM convolutions), nearest x2 upsampling into a padded
// buffer, im2col for the strided / tiny-channel convolutions, the sinusoidal timestep input,
// row gathers / scatters between a level's full hidden state and the packed masked rows of a
// Transformer2D, and the masked Euler update.  The convolutions themselves are tcgen05 GEMMs
// (k_gemm_tc.cu: launch_conv3x3_tc, launch_gemm_tc).
#include <algorithm>
#include <cstdio>
#include "kernels.h"
#include "unet_kernels.h"

namespace ig {

// ---------------------------------------------------------------------------------------
// GroupNorm statistics over [N images][P pixels][C = C1 + C2 channels] (two fp32 sources:
// the up path's [h | skip] concatenation).  Deterministic: per (image, pixel chunk) partial
// sums per group in a fixed order, then per (image, group) combined in fp64.
// ---------------------------------------------------------------------------------------
constexpr int GN_CHUNK = 64;  // pixels per partial

__global__ void __launch_bounds__(256) gn_partial_kernel(const float* __restrict__ x1, int C1, const float* __restrict__ x2,
                                                         int C2, int P, int G, float2* __restrict__ part) {
  extern __shared__ float sm[];  // [2][C]
  const int C = C1 + C2;
  const int n = blockIdx.y, chunk = blockIdx.x;
  const int p0 = chunk * GN_CHUNK, p1 = min(P, p0 + GN_CHUNK);
  float* ssum = sm;
  float* ssq = sm + C;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const float* base = c < C1 ? x1 + c : x2 + (c - C1);
    const long long ld = c < C1 ? C1 : C2;
    float s0 = 0.f, q0 = 0.f, s1 = 0.f, q1 = 0.f;
    int p = p0;
#pragma unroll 4
    for (; p + 1 < p1; p += 2) {  // two independent chains, loads in flight
      const float v0 = base[((long long)n * P + p) * ld];
      const float v1 = base[((long long)n * P + p + 1) * ld];
      s0 += v0; q0 = fmaf(v0, v0, q0);
      s1 += v1; q1 = fmaf(v1, v1, q1);
    }
    if (p < p1) {
      const float v0 = base[((long long)n * P + p) * ld];
      s0 += v0; q0 = fmaf(v0, v0, q0);
    }
    ssum[c] = s0 + s1;
    ssq[c] = q0 + q1;
  }
  __syncthreads();
  const int cg = C / G;
  for (int gi = threadIdx.x; gi < G; gi += blockDim.x) {
    float s = 0.f, q = 0.f;
    for (int c = gi * cg; c < (gi + 1) * cg; ++c) { s += ssum[c]; q += ssq[c]; }
    part[((long long)n * gridDim.x + chunk) * G + gi] = make_float2(s, q);
  }
}

// float4 variant (C1 % 4 == 0, C2 % 4 == 0): work item = (channel quad, pixel lane); each
// thread walks its lane's pixels of the chunk with 16-byte loads (a warp reads 512 contiguous
// bytes of one pixel row), lanes combined through shared memory in a fixed order
__global__ void __launch_bounds__(256) gn_partial4_kernel(const float* __restrict__ x1, int C1, const float* __restrict__ x2,
                                                          int C2, int P, int G, float2* __restrict__ part) {
  extern __shared__ float4 sm4[];  // [PL][CV] sums, then [PL][CV] sums of squares
  const int C = C1 + C2, CV = C >> 2;
  const int PL = CV >= (int)blockDim.x ? 1 : (int)blockDim.x / CV;
  const int n = blockIdx.y, chunk = blockIdx.x;
  const int p0 = chunk * GN_CHUNK, p1 = min(P, p0 + GN_CHUNK);
  float4* ssum = sm4;
  float4* ssq = sm4 + PL * CV;
  for (int w = threadIdx.x; w < CV * PL; w += blockDim.x) {
    const int cv = w % CV, pl = w / CV, c = 4 * cv;
    const float* base = c < C1 ? x1 + c : x2 + (c - C1);
    const long long ld = c < C1 ? C1 : C2;
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f), q = s;
#pragma unroll 4
    for (int p = p0 + pl; p < p1; p += PL) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(base + ((long long)n * P + p) * ld));
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
      q.x = fmaf(v.x, v.x, q.x); q.y = fmaf(v.y, v.y, q.y); q.z = fmaf(v.z, v.z, q.z); q.w = fmaf(v.w, v.w, q.w);
    }
    ssum[pl * CV + cv] = s;
    ssq[pl * CV + cv] = q;
  }
  __syncthreads();
  const int cg = C / G;
  const float* fs = reinterpret_cast<const float*>(ssum);
  const float* fq = reinterpret_cast<const float*>(ssq);
  for (int gi = threadIdx.x; gi < G; gi += blockDim.x) {
    float s = 0.f, q = 0.f;
    for (int pl = 0; pl < PL; ++pl)
      for (int c = gi * cg; c < (gi + 1) * cg; ++c) { s += fs[pl * C + c]; q += fq[pl * C + c]; }
    part[((long long)n * gridDim.x + chunk) * G + gi] = make_float2(s, q);
  }
}

__global__ void gn_finalize_kernel(const float2* __restrict__ part, int nchunk, int G, long long count, float eps,
                                   float2* __restrict__ stats) {
  const int n = blockIdx.x;
  for (int gi = threadIdx.x; gi < G; gi += blockDim.x) {
    double s = 0.0, q = 0.0;
    for (int k = 0; k < nchunk; ++k) {
      const float2 v = part[((long long)n * nchunk + k) * G + gi];
      s += v.x;
      q += v.y;
    }
    const double mean = s / (double)count;
    double var = q / (double)count - mean * mean;
    if (var < 0.0) var = 0.0;
    stats[n * G + gi] = make_float2((float)mean, (float)(1.0 / sqrt(var + (double)eps)));
  }
}

void launch_gn_stats(const float* x1, int C1, const float* x2, int C2, int N, int P, int G, float eps,
                     float2* partial, float2* stats, cudaStream_t st) {
  const int nchunk = (P + GN_CHUNK - 1) / GN_CHUNK;
  const int C = C1 + C2;
  if (C1 % 4 == 0 && C2 % 4 == 0) {
    const int CV = C / 4, PL = CV >= 256 ? 1 : 256 / CV;
    gn_partial4_kernel<<<dim3(nchunk, N), 256, 2 * PL * CV * sizeof(float4), st>>>(x1, C1, x2, C2, P, G, partial);
  } else {
    gn_partial_kernel<<<dim3(nchunk, N), 256, 2 * C * sizeof(float), st>>>(x1, C1, x2, C2, P, G, partial);
  }
  gn_finalize_kernel<<<N, 64, 0, st>>>(partial, nchunk, G, (long long)P * (C / G), eps, stats);
}

__device__ __forceinline__ float silu_f(float v) { return v / (1.f + __expf(-v)); }

// per (image, channel) affine coefficients of GroupNorm: y = x * a + b with
// a = rstd_g * gamma_c, b = beta_c - mean_g * rstd_g * gamma_c
__global__ void gn_coef_kernel(const float2* __restrict__ stats, const bf16* __restrict__ gamma, const bf16* __restrict__ beta,
                               int G, int C, float2* __restrict__ coef) {
  const int n = blockIdx.x, cg = C / G;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const float2 s = stats[n * G + c / cg];
    const float a = s.y * __bfloat162float(gamma[c]);
    coef[n * C + c] = make_float2(a, __bfloat162float(beta[c]) - s.x * a);
  }
}

// dst: zero-padded NHWC bf16 [N][H+2][W+2][C] (every element written: the borders are zeros,
// so one buffer can be reused with any channel count); value = act(GN([x1 | x2])); 8 channels
// per thread (C1 % 8 == 0: a vector never straddles the two sources)
__global__ void __launch_bounds__(256) gn_apply_padded_kernel(const float* __restrict__ x1, int C1,
                                                              const float* __restrict__ x2, int C2,
                                                              const float2* __restrict__ coef, int do_silu, int N,
                                                              int H, int W, bf16* __restrict__ dst) {
  const int C = C1 + C2;
  const int cv = C / 8;
  const long long total = (long long)N * (H + 2) * (W + 2) * cv;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int v = (int)(i % cv);
    const long long pp = i / cv;
    const int xx = (int)(pp % (W + 2));
    const long long t = pp / (W + 2);
    const int yy = (int)(t % (H + 2));
    const int n = (int)(t / (H + 2));
    uint4 out = make_uint4(0, 0, 0, 0);
    if (yy >= 1 && yy <= H && xx >= 1 && xx <= W) {
      const long long row = ((long long)n * H + (yy - 1)) * W + (xx - 1);
      const int c0 = v * 8;
      const float4* src = c0 < C1 ? reinterpret_cast<const float4*>(x1 + row * C1 + c0)
                                  : reinterpret_cast<const float4*>(x2 + row * C2 + (c0 - C1));
      const float4 a = src[0], b = src[1];
      const float xv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      const float4* cf = reinterpret_cast<const float4*>(coef + (long long)n * C + c0);
      float y[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 k = cf[q];
        y[2 * q] = fmaf(xv[2 * q], k.x, k.y);
        y[2 * q + 1] = fmaf(xv[2 * q + 1], k.z, k.w);
      }
      uint32_t* w = reinterpret_cast<uint32_t*>(&out);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float u0 = do_silu ? silu_f(y[2 * e]) : y[2 * e];
        const float u1 = do_silu ? silu_f(y[2 * e + 1]) : y[2 * e + 1];
        __nv_bfloat162 p = __floats2bfloat162_rn(u0, u1);
        w[e] = *reinterpret_cast<uint32_t*>(&p);
      }
    }
    reinterpret_cast<uint4*>(dst)[i] = out;
  }
}

void launch_gn_apply_padded(const float* x1, int C1, const float* x2, int C2, const float2* stats, const bf16* gamma,
                            const bf16* beta, int G, int do_silu, int N, int H, int W, bf16* dst, float2* coef,
                            cudaStream_t st) {
  gn_coef_kernel<<<N, 256, 0, st>>>(stats, gamma, beta, G, C1 + C2, coef);
  const long long total = (long long)N * (H + 2) * (W + 2) * ((C1 + C2) / 8);
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 16);
  gn_apply_padded_kernel<<<blocks, 256, 0, st>>>(x1, C1, x2, C2, coef, do_silu, N, H, W, dst);
}

// nearest x2 upsampling of x fp32 [N][H][W][C] into zero-padded bf16 [N][2H+2][2W+2][C]
__global__ void __launch_bounds__(256) upsample_padded_kernel(const float* __restrict__ x, int C, int N, int H, int W,
                                                              bf16* __restrict__ dst) {
  const int H2 = 2 * H, W2 = 2 * W, cv = C / 8;
  const long long total = (long long)N * (H2 + 2) * (W2 + 2) * cv;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int v = (int)(i % cv);
    const long long pp = i / cv;
    const int xx = (int)(pp % (W2 + 2));
    const long long t = pp / (W2 + 2);
    const int yy = (int)(t % (H2 + 2));
    const int n = (int)(t / (H2 + 2));
    uint4 out = make_uint4(0, 0, 0, 0);
    if (yy >= 1 && yy <= H2 && xx >= 1 && xx <= W2) {
      const long long row = ((long long)n * H + (yy - 1) / 2) * W + (xx - 1) / 2;
      const float4* s = reinterpret_cast<const float4*>(x + row * C + v * 8);
      const float4 a = s[0], b = s[1];
      uint32_t* w = reinterpret_cast<uint32_t*>(&out);
      __nv_bfloat162 p0 = __floats2bfloat162_rn(a.x, a.y), p1 = __floats2bfloat162_rn(a.z, a.w);
      __nv_bfloat162 p2 = __floats2bfloat162_rn(b.x, b.y), p3 = __floats2bfloat162_rn(b.z, b.w);
      w[0] = *reinterpret_cast<uint32_t*>(&p0);
      w[1] = *reinterpret_cast<uint32_t*>(&p1);
      w[2] = *reinterpret_cast<uint32_t*>(&p2);
      w[3] = *reinterpret_cast<uint32_t*>(&p3);
    }
    reinterpret_cast<uint4*>(dst)[i] = out;
  }
}

void launch_upsample_padded(const float* x, int C, int N, int H, int W, bf16* dst, cudaStream_t st) {
  const long long total = (long long)N * (2 * H + 2) * (2 * W + 2) * (C / 8);
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 16);
  upsample_padded_kernel<<<blocks, 256, 0, st>>>(x, C, N, H, W, dst);
}

// im2col of x fp32 [N][H][W][C] for a 3x3 conv with zero padding 1 and stride s:
// dst[(n*Ho + y)*Wo + x][k] (bf16, row length Kp >= 9C, zero beyond 9C), k = tap*C + c;
// per-image scale (the c_in input scaling of the UNet's latent) when scale != nullptr
__global__ void __launch_bounds__(256) im2col_kernel(const float* __restrict__ x, int C, int N, int H, int W, int s,
                                                     const float* __restrict__ scale, int Kp, bf16* __restrict__ dst) {
  const int Ho = (H - 1) / s + 1, Wo = (W - 1) / s + 1;
  const long long total = (long long)N * Ho * Wo * Kp;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(i % Kp);
    const long long m = i / Kp;
    float v = 0.f;
    if (k < 9 * C) {
      const int tap = k / C, c = k - tap * C;
      const int ky = tap / 3, kx = tap - ky * 3;
      const int xo = (int)(m % Wo);
      const long long t = m / Wo;
      const int yo = (int)(t % Ho);
      const int n = (int)(t / Ho);
      const int yi = yo * s + ky - 1, xi = xo * s + kx - 1;
      if (yi >= 0 && yi < H && xi >= 0 && xi < W) {
        v = x[(((long long)n * H + yi) * W + xi) * C + c];
        if (scale) v *= scale[n];
      }
    }
    dst[i] = __float2bfloat16_rn(v);
  }
}

// 8 consecutive k (one tap, 8 channels) per thread: two float4 loads, one 16-byte store
__global__ void __launch_bounds__(256) im2col8_kernel(const float* __restrict__ x, int C, int N, int H, int W, int s,
                                                      int Kp, bf16* __restrict__ dst) {
  const int Ho = (H - 1) / s + 1, Wo = (W - 1) / s + 1;
  const int kv = Kp / 8;
  const long long total = (long long)N * Ho * Wo * kv;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(i % kv) * 8;
    const long long m = i / kv;
    uint4 out = make_uint4(0, 0, 0, 0);
    if (k < 9 * C) {
      const int tap = k / C, c = k - tap * C;
      const int ky = tap / 3, kx = tap - ky * 3;
      const int xo = (int)(m % Wo);
      const long long t = m / Wo;
      const int yo = (int)(t % Ho);
      const int n = (int)(t / Ho);
      const int yi = yo * s + ky - 1, xi = xo * s + kx - 1;
      if (yi >= 0 && yi < H && xi >= 0 && xi < W) {
        const float4* p = reinterpret_cast<const float4*>(x + (((long long)n * H + yi) * W + xi) * C + c);
        const float4 a = p[0], b = p[1];
        uint32_t* w = reinterpret_cast<uint32_t*>(&out);
        __nv_bfloat162 q0 = __floats2bfloat162_rn(a.x, a.y), q1 = __floats2bfloat162_rn(a.z, a.w);
        __nv_bfloat162 q2 = __floats2bfloat162_rn(b.x, b.y), q3 = __floats2bfloat162_rn(b.z, b.w);
        w[0] = *reinterpret_cast<uint32_t*>(&q0);
        w[1] = *reinterpret_cast<uint32_t*>(&q1);
        w[2] = *reinterpret_cast<uint32_t*>(&q2);
        w[3] = *reinterpret_cast<uint32_t*>(&q3);
      }
    }
    reinterpret_cast<uint4*>(dst)[i] = out;
  }
}

void launch_im2col(const float* x, int C, int N, int H, int W, int stride, const float* scale, int Kp, bf16* dst,
                   cudaStream_t st) {
  const int Ho = (H - 1) / stride + 1, Wo = (W - 1) / stride + 1;
  if (!scale && C % 8 == 0 && Kp % 8 == 0) {
    const long long total = (long long)N * Ho * Wo * (Kp / 8);
    const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 16);
    im2col8_kernel<<<blocks, 256, 0, st>>>(x, C, N, H, W, stride, Kp, dst);
    return;
  }
  const long long total = (long long)N * Ho * Wo * Kp;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 16);
  im2col_kernel<<<blocks, 256, 0, st>>>(x, C, N, H, W, stride, scale, Kp, dst);
}

// im2col from a zero-padded bf16 NHWC buffer [N][H+2][W+2][C] (stride 1): dst[m][k] (row
// length Kp >= 9C), k = tap*C + c — the generic path for convolutions the implicit-GEMM tile
// walk does not cover (narrow levels: (H*W) % 128 != 0 or W < 8)
__global__ void __launch_bounds__(256) im2col_padded_kernel(const bf16* __restrict__ pad, int C, int N, int H, int W,
                                                            int Kp, bf16* __restrict__ dst) {
  const long long total = (long long)N * H * W * Kp;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int k = (int)(i % Kp);
    const long long m = i / Kp;
    bf16 v = __float2bfloat16_rn(0.f);
    if (k < 9 * C) {
      const int tap = k / C, c = k - tap * C;
      const int ky = tap / 3, kx = tap - ky * 3;
      const int x = (int)(m % W);
      const long long t = m / W;
      const int y = (int)(t % H);
      const int n = (int)(t / H);
      v = pad[(((long long)n * (H + 2) + y + ky) * (W + 2) + x + kx) * C + c];
    }
    dst[i] = v;
  }
}

void launch_im2col_padded(const bf16* pad, int C, int N, int H, int W, int Kp, bf16* dst, cudaStream_t st) {
  const long long total = (long long)N * H * W * Kp;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 16);
  im2col_padded_kernel<<<blocks, 256, 0, st>>>(pad, C, N, H, W, Kp, dst);
}

// ---------------------------------------------------------------------------------------
// per-request row lists (UNet batch: request r owns image r of every level buffer)
// ---------------------------------------------------------------------------------------
// dst[r][p][c] = latents[r][p][c] (fp32 copy of each request's latent into the batch buffer)
__global__ void gather_latents_kernel(const UReq* __restrict__ rq, int P, int C, float* __restrict__ dst) {
  const int r = blockIdx.y;
  const float* src = rq[r].latent;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P * C; i += gridDim.x * blockDim.x)
    dst[(long long)r * P * C + i] = src[i];
}
void launch_gather_latents(const UReq* rq, int n, int P, int C, float* dst, cudaStream_t st) {
  gather_latents_kernel<<<dim3(std::max(1, std::min(64, (P * C + 255) / 256)), n), 256, 0, st>>>(rq, P, C, dst);
}

// sinusoid_{dim}(1000 sigma_r), cos first, f_k = exp(-ln(10000) k / (dim / 2)) (double)
__global__ void unet_sinusoid_kernel(const UReq* __restrict__ rq, int dim, float* __restrict__ out) {
  const int r = blockIdx.x, half = dim / 2;
  const double t = 1000.0 * (double)rq[r].sigma;
  for (int k = threadIdx.x; k < half; k += blockDim.x) {
    const double f = exp(-log(10000.0) * (double)k / (double)half);
    out[r * dim + k] = (float)cos(t * f);
    out[r * dim + half + k] = (float)sin(t * f);
  }
}
void launch_unet_sinusoid(const UReq* rq, int n, int dim, float* out, cudaStream_t st) {
  unet_sinusoid_kernel<<<n, 128, 0, st>>>(rq, dim, out);
}

// v[r][c] (+)= cond_r[c] (optional per-request vector), then silu -> bf16 copy
__global__ void temb_finish_kernel(const UReq* __restrict__ rq, int E, float* __restrict__ v, bf16* __restrict__ out) {
  const int r = blockIdx.x;
  for (int c = threadIdx.x; c < E; c += blockDim.x) {
    float a = v[r * E + c];
    if (rq[r].cond) a += rq[r].cond[c];
    v[r * E + c] = a;
    out[r * E + c] = __float2bfloat16_rn(silu_f(a));
  }
}
void launch_temb_finish(const UReq* rq, int n, int E, float* v, bf16* out, cudaStream_t st) {
  temb_finish_kernel<<<n, 256, 0, st>>>(rq, E, v, out);
}

// out = silu(in) elementwise fp32 (in place allowed)
__global__ void silu_inplace_kernel(float* __restrict__ x, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    x[i] = silu_f(x[i]);
}
void launch_silu_inplace(float* x, long long n, cudaStream_t st) {
  silu_inplace_kernel<<<(int)std::min<long long>((n + 255) / 256, 1024), 256, 0, st>>>(x, n);
}

// Transformer2D input: packed rows A[row0_r + j] = GN(x_r[idx_r[j]]) (no activation), bf16;
// rows of request r are its level mask's idx_m (or all tokens when dense)
__global__ void __launch_bounds__(256) t2d_in_rows_kernel(const URows* __restrict__ rl, const float* __restrict__ x, int P,
                                                          int C, const float2* __restrict__ stats,
                                                          const bf16* __restrict__ gamma, const bf16* __restrict__ beta,
                                                          int G, bf16* __restrict__ dst) {
  const int r = blockIdx.y;
  const URows L = rl[r];
  const int cg = C / G;
  const int warps = gridDim.x * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  for (int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < L.n; j += warps) {
    const int tok = L.idx ? L.idx[j] : j;
    const float* src = x + ((long long)r * P + tok) * C;
    bf16* d = dst + (long long)(L.row0 + j) * C;
    for (int c = lane; c < C; c += 32) {
      const float2 s = stats[r * G + c / cg];
      d[c] = __float2bfloat16_rn((src[c] - s.x) * s.y * __bfloat162float(gamma[c]) + __bfloat162float(beta[c]));
    }
  }
}
void launch_t2d_in_rows(const URows* rl, int n, int max_rows, const float* x, int P, int C, const float2* stats,
                        const bf16* gamma, const bf16* beta, int G, bf16* dst, cudaStream_t st) {
  if (max_rows <= 0) return;
  t2d_in_rows_kernel<<<dim3(std::max(1, std::min(128, (max_rows + 7) / 8)), n), 256, 0, st>>>(rl, x, P, C, stats, gamma,
                                                                                                beta, G, dst);
}

// T[r][idx_r[j]][:] = src[row0_r + j][:] (fp32 packed rows -> the stack's per-request state)
// or the reverse gather (to_packed = 1: dst packed bf16 rows from T)
__global__ void __launch_bounds__(256) rows_move_kernel(const URows* __restrict__ rl, float* __restrict__ T, int P, int C,
                                                        const float* __restrict__ src, bf16* __restrict__ dstp,
                                                        int to_packed) {
  const int r = blockIdx.y;
  const URows L = rl[r];
  const int warps = gridDim.x * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  for (int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < L.n; j += warps) {
    const int tok = L.idx ? L.idx[j] : j;
    float* t = T + ((long long)r * P + tok) * C;
    if (to_packed) {
      bf16* d = dstp + (long long)(L.row0 + j) * C;
      for (int c = lane; c < C; c += 32) d[c] = __float2bfloat16_rn(t[c]);
    } else {
      const float* s = src + (long long)(L.row0 + j) * C;
      for (int c = lane; c < C; c += 32) t[c] = s[c];
    }
  }
}
void launch_rows_move(const URows* rl, int n, int max_rows, float* T, int P, int C, const float* src, bf16* dstp,
                      int to_packed, cudaStream_t st) {
  if (max_rows <= 0) return;
  rows_move_kernel<<<dim3(std::max(1, std::min(128, (max_rows + 7) / 8)), n), 256, 0, st>>>(rl, T, P, C, src, dstp,
                                                                                              to_packed);
}

// Transformer2D output: out[r][tok] = x[r][tok] + po[row0 + j] for the masked tokens (rows of
// rl), and = y_r[tok] (the template's Transformer2D output, cache plane) for the others (rlu)
__global__ void __launch_bounds__(256) t2d_out_kernel(const URows* __restrict__ rl, const URows* __restrict__ rlu,
                                                      const float* __restrict__ x, const float* __restrict__ po, int P,
                                                      int C, float* __restrict__ out) {
  const int r = blockIdx.y;
  const int warps = gridDim.x * (blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  const URows L = rl[r], U = rlu[r];
  const int total = L.n + U.n;
  for (int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < total; j += warps) {
    if (j < L.n) {
      const int tok = L.idx ? L.idx[j] : j;
      const long long row = (long long)r * P + tok;
      const float* a = x + row * C;
      const float* b = po + (long long)(L.row0 + j) * C;
      float* o = out + row * C;
      for (int c = lane; c < C; c += 32) o[c] = a[c] + b[c];
    } else {
      const int ju = j - L.n;
      const int tok = U.idx[ju];
      const float* y = U.y + (long long)tok * C;
      float* o = out + ((long long)r * P + tok) * C;
      for (int c = lane; c < C; c += 32) o[c] = y[c];
    }
  }
}
void launch_t2d_out(const URows* rl, const URows* rlu, int n, int max_rows, const float* x, const float* po, int P, int C,
                    float* out, cudaStream_t st) {
  if (max_rows <= 0) return;
  t2d_out_kernel<<<dim3(std::max(1, std::min(128, (max_rows + 7) / 8)), n), 256, 0, st>>>(rl, rlu, x, po, P, C, out);
}

// latent_r[tok][c] += dsig_r * eps[r][tok][c] for the masked tokens of request r (level 0)
__global__ void unet_euler_kernel(const UReq* __restrict__ rq, const URows* __restrict__ rl, int P, int C,
                                  const float* __restrict__ eps) {
  const int r = blockIdx.y;
  const URows L = rl[r];
  const float ds = rq[r].dsig;
  float* lat = rq[r].latent;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < L.n * C; i += gridDim.x * blockDim.x) {
    const int j = i / C, c = i - j * C;
    const int tok = L.idx ? L.idx[j] : j;
    lat[(long long)tok * C + c] += ds * eps[((long long)r * P + tok) * C + c];
  }
}
void launch_unet_euler(const UReq* rq, const URows* rl, int n, int max_rows, int P, int C, const float* eps,
                       cudaStream_t st) {
  if (max_rows <= 0) return;
  unet_euler_kernel<<<dim3(std::max(1, std::min(64, (max_rows * C + 255) / 256)), n), 256, 0, st>>>(rq, rl, P, C, eps);
}

// plain bf16 copy of the [x1 | x2] concatenation (the 1x1 skip projection's A operand)
__global__ void cat_bf16_kernel(const float* __restrict__ x1, int C1, const float* __restrict__ x2, int C2, long long rows,
                                bf16* __restrict__ dst) {
  const int C = C1 + C2, cv = C / 8;  // C1 % 8 == 0: 8-channel vectors never straddle
  const long long total = rows * cv;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long row = i / cv;
    const int c = (int)(i - row * cv) * 8;
    const float4* p = c < C1 ? reinterpret_cast<const float4*>(x1 + row * C1 + c)
                             : reinterpret_cast<const float4*>(x2 + row * C2 + (c - C1));
    const float4 a = p[0], b = p[1];
    uint4 out;
    uint32_t* w = reinterpret_cast<uint32_t*>(&out);
    __nv_bfloat162 q0 = __floats2bfloat162_rn(a.x, a.y), q1 = __floats2bfloat162_rn(a.z, a.w);
    __nv_bfloat162 q2 = __floats2bfloat162_rn(b.x, b.y), q3 = __floats2bfloat162_rn(b.z, b.w);
    w[0] = *reinterpret_cast<uint32_t*>(&q0);
    w[1] = *reinterpret_cast<uint32_t*>(&q1);
    w[2] = *reinterpret_cast<uint32_t*>(&q2);
    w[3] = *reinterpret_cast<uint32_t*>(&q3);
    reinterpret_cast<uint4*>(dst)[i] = out;
  }
}
void launch_cat_bf16(const float* x1, int C1, const float* x2, int C2, long long rows, bf16* dst, cudaStream_t st) {
  const long long total = rows * ((C1 + C2) / 8);
  cat_bf16_kernel<<<(int)std::min<long long>((total + 255) / 256, 148 * 16), 256, 0, st>>>(x1, C1, x2, C2, rows, dst);
}

}  // namespace ig
