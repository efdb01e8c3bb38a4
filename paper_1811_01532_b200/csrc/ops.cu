// Memory-bound kernels of the WAP step: layout moves, im2col/col2im, elementwise
// (BiasAdd/ReLU/GradReLU), AddN, GradBias, MaxPool, LRN, softmax-xent, SGD.
// All are HBM-bound: coalesced along the contiguous channel axis, float4 where
// the layout allows (ld % 4 == 0 always), grid = multiple of the 148 SMs,
// reductions deterministic (fixed order, no atomics) so replicas stay bitwise equal.
#include <atomic>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "../../include/wap_b200.h"

extern std::atomic<long long> g_wap_launches;

namespace {

__host__ __device__ __forceinline__ int64_t lidx(const wap_layout_t& l, int b, int h, int w, int c) {
  return (((int64_t)b * (l.H + l.pad) + h) * (l.W + l.pad) + w) * l.ld + c;
}

int grid_for(int64_t work, int threads) {
  int64_t blocks = (work + threads - 1) / threads;
  const int64_t cap = (int64_t)WAP_NUM_SMS * 16;
  if (blocks > cap) blocks = cap;
  return (int)(blocks < 1 ? 1 : blocks);
}

#define COUNT_LAUNCH() g_wap_launches.fetch_add(1, std::memory_order_relaxed)

int check_layout(const wap_layout_t& l, const char* name) {
  WAP_CHECK_ARG(l.B >= 1 && l.H >= 1 && l.W >= 1 && l.C >= 1, "%s: bad dims", name);
  WAP_CHECK_ARG(l.pad >= 0, "%s: negative pad", name);
  WAP_CHECK_ARG(l.ld >= l.C && l.ld % 4 == 0, "%s: ld=%d must be >= C=%d and a multiple of 4", name, l.ld, l.C);
  return WAP_OK;
}

// ---------------------------------------------------------------------------
// elementwise: one thread per (pixel, 4 channels); lanes >= C written as 0
// ---------------------------------------------------------------------------
template <int OP>
__global__ void elementwise_kernel(const float* __restrict__ x, wap_layout_t xl, const float* __restrict__ aux,
                                   wap_layout_t al, const float* __restrict__ bias, float* __restrict__ y,
                                   wap_layout_t yl) {
  const int c4n = yl.ld / 4;
  const int64_t total = (int64_t)yl.B * yl.H * yl.W * c4n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % c4n) * 4;
    int64_t p = i / c4n;
    const int w = (int)(p % yl.W);
    p /= yl.W;
    const int h = (int)(p % yl.H);
    const int b = (int)(p / yl.H);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (c < xl.ld) v = *reinterpret_cast<const float4*>(x + lidx(xl, b, h, w, c));
    float o[4] = {v.x, v.y, v.z, v.w};
    float m[4] = {1.f, 1.f, 1.f, 1.f};
    if (OP == 3) {
      const float4 a = *reinterpret_cast<const float4*>(aux + lidx(al, b, h, w, c));
      m[0] = a.x; m[1] = a.y; m[2] = a.z; m[3] = a.w;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int cc = c + j;
      if (cc >= yl.C) { o[j] = 0.f; continue; }
      if (OP == 0 || OP == 2) o[j] += __ldg(bias + cc);
      if (OP == 1 || OP == 2) o[j] = fmaxf(o[j], 0.f);
      if (OP == 3) o[j] = m[j] > 0.f ? o[j] : 0.f;
    }
    *reinterpret_cast<float4*>(y + lidx(yl, b, h, w, c)) = make_float4(o[0], o[1], o[2], o[3]);
  }
}

struct PtrPack {
  const float* p[16];
};
__global__ void add_n_kernel_packed(PtrPack xs, int n, float* __restrict__ y, int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 acc = reinterpret_cast<const float4*>(xs.p[0])[i];
    for (int k = 1; k < n; ++k) {
      const float4 v = reinterpret_cast<const float4*>(xs.p[k])[i];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    reinterpret_cast<float4*>(y)[i] = acc;
  }
}

// ---------------------------------------------------------------------------
// GradBias: column sums, pass 1 = per-chunk partials, pass 2 = ordered sum
// ---------------------------------------------------------------------------
// Block = CW float4 column groups (tx) x RL row lanes (ty), CW*RL = 256. Each
// thread streams its rows with four independent float4 loads in flight; the
// row lanes are reduced in a fixed order through shared memory.
__global__ void __launch_bounds__(256) bias_grad_partial(const float* __restrict__ dy, int64_t rows, int ld, int C,
                                                         int64_t rows_per_chunk, int CW, float* __restrict__ part) {
  __shared__ float4 red[256];
  const int RL = 256 / CW;
  const int tx = threadIdx.x % CW, ty = threadIdx.x / CW;
  const int c = (blockIdx.x * CW + tx) * 4;
  const int chunk = blockIdx.y;
  const int64_t r0 = chunk * rows_per_chunk;
  const int64_t r1 = min(rows, r0 + rows_per_chunk);
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  if (c < ld) {
    const float* base = dy + c;
    int64_t r = r0 + ty;
    for (; r + 3 * RL < r1; r += 4 * RL) {
      const float4 a = *reinterpret_cast<const float4*>(base + r * ld);
      const float4 b = *reinterpret_cast<const float4*>(base + (r + RL) * ld);
      const float4 e = *reinterpret_cast<const float4*>(base + (r + 2 * RL) * ld);
      const float4 f = *reinterpret_cast<const float4*>(base + (r + 3 * RL) * ld);
      s.x += (a.x + b.x) + (e.x + f.x);
      s.y += (a.y + b.y) + (e.y + f.y);
      s.z += (a.z + b.z) + (e.z + f.z);
      s.w += (a.w + b.w) + (e.w + f.w);
    }
    for (; r < r1; r += RL) {
      const float4 a = *reinterpret_cast<const float4*>(base + r * ld);
      s.x += a.x; s.y += a.y; s.z += a.z; s.w += a.w;
    }
  }
  red[threadIdx.x] = s;
  __syncthreads();
  if (ty == 0 && c < C) {
    float4 t = red[tx];
    for (int k = 1; k < RL; ++k) {
      const float4 u = red[k * CW + tx];
      t.x += u.x; t.y += u.y; t.z += u.z; t.w += u.w;
    }
    float* o = part + (int64_t)chunk * ld + c;
    o[0] = t.x;
    if (c + 1 < C) o[1] = t.y;
    if (c + 2 < C) o[2] = t.z;
    if (c + 3 < C) o[3] = t.w;
  }
}

int bias_cw(const wap_layout_t& l) {
  const int cols4 = l.ld / 4;
  return cols4 >= 32 ? 32 : (cols4 >= 16 ? 16 : (cols4 >= 8 ? 8 : (cols4 >= 4 ? 4 : (cols4 >= 2 ? 2 : 1))));
}

// One warp per column: lanes take chunks lane, lane + 32, ... and the warp
// reduces in a fixed shuffle order (deterministic for a fixed chunk count).
__global__ void bias_grad_final(const float* __restrict__ part, int chunks, int ld, int C, float* __restrict__ db) {
  const int c = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (c >= C) return;
  float s = 0.f;
  for (int k = lane; k < chunks; k += 32) s += part[(int64_t)k * ld + c];
  s = warp_sum(s);
  if (lane == 0) db[c] = s;
}

int bias_chunks(const wap_layout_t& l) {
  const int64_t rows = (int64_t)l.B * (l.H + l.pad) * (l.W + l.pad);
  const int cw = bias_cw(l);
  const int ctiles = (l.ld / 4 + cw - 1) / cw;
  // enough blocks (8 per SM) to keep ~64 KB of loads in flight per SM
  int64_t chunks = (8 * WAP_NUM_SMS + ctiles - 1) / ctiles;
  const int64_t max_chunks = (rows + 63) / 64;
  if (chunks > max_chunks) chunks = max_chunks;
  if (chunks < 1) chunks = 1;
  return (int)chunks;
}

// ---------------------------------------------------------------------------
// im2col / col2im
// ---------------------------------------------------------------------------
// Rows of `col` enumerate the OUTPUT grid with P trailing halo columns / rows per
// image (halo rows are zero), so a conv whose output must live on a padded grid
// gets GEMM rows that line up with it.
__global__ void im2col_kernel(const float* __restrict__ x, wap_layout_t xl, int k, int s, int p, int Ho, int Wo,
                              int P, float* __restrict__ col, int64_t ldcol) {
  const int C = xl.C;
  const int K = k * k * C;
  const int Hp = Ho + P, Wp = Wo + P;
  const int64_t M = (int64_t)xl.B * Hp * Wp;
  const int64_t total = M * ldcol;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int kk = (int)(i % ldcol);
    const int64_t m = i / ldcol;
    float v = 0.f;
    if (kk < K) {
      const int c = kk % C;
      const int t = kk / C;
      const int u = t / k, vv = t % k;
      const int wo = (int)(m % Wp);
      const int64_t r = m / Wp;
      const int ho = (int)(r % Hp);
      const int b = (int)(r / Hp);
      const int hi = ho * s + u - p, wi = wo * s + vv - p;
      if (ho >= 0 && ho < Ho && wo >= 0 && wo < Wo && hi >= 0 && hi < xl.H && wi >= 0 && wi < xl.W)
        v = __ldg(x + lidx(xl, b, hi, wi, c));
    }
    col[i] = v;
  }
}

// Table-driven im2col: a block owns IM2COL_ROWS output rows; the (u, v, c)
// decode of every column is computed once per block into shared memory, so the
// inner loop is a table lookup + one coalesced store per element.
constexpr int IM2COL_ROWS = 32;
constexpr int IM2COL_MAXK = 4096;

__global__ void __launch_bounds__(256) im2col_table_kernel(const float* __restrict__ x, wap_layout_t xl, int k, int s,
                                                           int p, int Ho, int Wo, int P, float* __restrict__ col,
                                                           int64_t ldcol, int64_t M) {
  __shared__ short tu[IM2COL_MAXK], tv[IM2COL_MAXK];
  __shared__ int toff[IM2COL_MAXK];
  __shared__ int rb[IM2COL_ROWS], rh[IM2COL_ROWS], rw[IM2COL_ROWS];
  __shared__ int64_t rbase[IM2COL_ROWS];
  const int C = xl.C;
  const int K = k * k * C;
  const int Wxp = xl.W + xl.pad;
  for (int kk = threadIdx.x; kk < K; kk += blockDim.x) {
    const int c = kk % C, t = kk / C;
    const int u = t / k, v = t % k;
    tu[kk] = (short)u;
    tv[kk] = (short)v;
    toff[kk] = (u * Wxp + v) * xl.ld + c;
  }
  const int Hp = Ho + P, Wp = Wo + P;
  __syncthreads();
  if (ldcol % 4 == 0) {
    // float4 path: a block sweeps IM2COL_ROWS rows at a time; row geometry comes
    // from a per-row smem table (decoded once per row), columns from the per-block
    // tap table, and the element index is 32-bit (no 64-bit division in the loop).
    const int q4 = (int)(ldcol / 4);
    for (int64_t r0 = (int64_t)blockIdx.x * IM2COL_ROWS; r0 < M; r0 += (int64_t)gridDim.x * IM2COL_ROWS) {
      __syncthreads();
      if (threadIdx.x < IM2COL_ROWS) {
        const int64_t m = r0 + threadIdx.x;
        int64_t base = 0;  // may be negative: taps outside the image are masked per element
        int h0 = 0, w0 = 0, valid = 0;
        if (m < M) {
          const int wo = (int)(m % Wp);
          const int64_t q = m / Wp;
          const int ho = (int)(q % Hp);
          const int bb = (int)(q / Hp);
          if (ho >= 0 && ho < Ho && wo >= 0 && wo < Wo) {
            h0 = ho * s - p;
            w0 = wo * s - p;
            base = (((int64_t)bb * (xl.H + xl.pad) + h0) * Wxp + w0) * xl.ld;
            valid = 1;
          }
        }
        rb[threadIdx.x] = valid;
        rh[threadIdx.x] = h0;
        rw[threadIdx.x] = w0;
        rbase[threadIdx.x] = base;
      }
      __syncthreads();
      const int nrows = (M - r0) < IM2COL_ROWS ? (int)(M - r0) : IM2COL_ROWS;
      float4* out4 = reinterpret_cast<float4*>(col + r0 * ldcol);
      for (int idx = threadIdx.x; idx < nrows * q4; idx += blockDim.x) {
        const int r = idx / q4;
        const int kk0 = (idx - r * q4) * 4;
        float o[4] = {0.f, 0.f, 0.f, 0.f};
        if (rb[r]) {
          const int h0 = rh[r], w0 = rw[r];
          const float* xb = x + rbase[r];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int kk = kk0 + i;
            if (kk < K) {
              const int hi = h0 + tu[kk], wi = w0 + tv[kk];
              if (hi >= 0 && hi < xl.H && wi >= 0 && wi < xl.W) o[i] = __ldg(xb + toff[kk]);
            }
          }
        }
        out4[idx] = make_float4(o[0], o[1], o[2], o[3]);
      }
    }
    return;
  }
  for (int64_t r0 = (int64_t)blockIdx.x * IM2COL_ROWS; r0 < M; r0 += (int64_t)gridDim.x * IM2COL_ROWS) {
    __syncthreads();
    if (threadIdx.x < IM2COL_ROWS) {
      const int64_t m = r0 + threadIdx.x;
      int b = -1, ho = -1, wo = -1;
      if (m < M) {
        wo = (int)(m % Wp);
        const int64_t q = m / Wp;
        ho = (int)(q % Hp);
        b = (int)(q / Hp);
        if (ho < 0 || ho >= Ho || wo < 0 || wo >= Wo) b = -2;  // halo row -> zeros
      }
      rb[threadIdx.x] = b;
      rh[threadIdx.x] = ho * s - p;
      rw[threadIdx.x] = wo * s - p;
    }
    __syncthreads();
    for (int i = 0; i < IM2COL_ROWS; ++i) {
      const int64_t m = r0 + i;
      if (m >= M) break;
      const int b = rb[i], h0 = rh[i], w0 = rw[i];
      float* out = col + m * ldcol;
      // base address of tap (0,0) channel 0 (may be outside; guarded per element)
      const int64_t base = (((int64_t)(b < 0 ? 0 : b) * (xl.H + xl.pad) + h0) * Wxp + w0) * xl.ld;
      for (int kk = threadIdx.x; kk < ldcol; kk += blockDim.x) {
        float v = 0.f;
        if (b >= 0 && kk < K) {
          const int hi = h0 + tu[kk], wi = w0 + tv[kk];
          if (hi >= 0 && hi < xl.H && wi >= 0 && wi < xl.W) v = __ldg(x + base + toff[kk]);
        }
        out[kk] = v;
      }
    }
  }
}

__global__ void col2im_kernel(const float* __restrict__ dcol, int64_t ldcol, int k, int s, int p, int Ho, int Wo,
                              int P, float* __restrict__ dx, wap_layout_t dl, const float* __restrict__ mask,
                              wap_layout_t ml) {
  const int Hp = Ho + P, Wp = Wo + P;
  const int C = dl.C;
  const int64_t total = (int64_t)dl.B * dl.H * dl.W * dl.ld;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % dl.ld);
    int64_t q = i / dl.ld;
    const int w = (int)(q % dl.W);
    q /= dl.W;
    const int h = (int)(q % dl.H);
    const int b = (int)(q / dl.H);
    float acc = 0.f;
    if (c < C) {
      for (int u = 0; u < k; ++u) {
        const int hs = h + p - u;
        if (hs < 0 || hs % s) continue;
        const int ho = hs / s;
        if (ho >= Ho) continue;
        for (int v = 0; v < k; ++v) {
          const int ws = w + p - v;
          if (ws < 0 || ws % s) continue;
          const int wo = ws / s;
          if (wo >= Wo) continue;
          acc += dcol[(((int64_t)b * Hp + ho) * Wp + wo) * ldcol + (u * k + v) * C + c];
        }
      }
      if (mask && !(mask[lidx(ml, b, h, w, c)] > 0.f)) acc = 0.f;
    }
    dx[lidx(dl, b, h, w, c)] = acc;
  }
}

// ---------------------------------------------------------------------------
// Space-to-depth for strided first-layer convs (AlexNet conv1 11x11/4 pad 2)
// ---------------------------------------------------------------------------
// A k x k stride-s conv with zero padding p over x equals a ceil(k/s)^2-tap
// stride-1 VALID conv over xs[b, i, j, (dy*s+dx)*C + c] = xpad[b, s*i+dy, s*j+dx, c]
// with weights ws[a, e, (dy*s+dx)*C + c, o] = w[s*a+dy, s*e+dx, c, o] (0 beyond k).
// On the s2d grid (Hs x Ws rows per image, no halo) the VALID conv is a shifted
// GEMM with tap shifts a*Ws + e whose output grid is the conv output with
// Hs - Ho trailing halo rows / columns: no im2col buffer.
// One thread per output float4 (32-bit indices; the host checks the size): 16
// consecutive threads write one s2d pixel's 64 channels as 256 contiguous bytes,
// the gathered reads hit L1/L2 (neighbouring threads read the same input pixels).
__global__ void __launch_bounds__(256) s2d_input_kernel(const float* __restrict__ x, wap_layout_t xl, int s, int p,
                                                        int Hs, int Wsd, float* __restrict__ xs, int ldc) {
  const int C = xl.C;
  const uint32_t q4n = (uint32_t)ldc / 4;
  const uint32_t total = (uint32_t)xl.B * Hs * Wsd * q4n;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const uint32_t q = e % q4n, pix = e / q4n;
    const uint32_t j = pix % (uint32_t)Wsd, r = pix / (uint32_t)Wsd;
    const int ii = (int)(r % (uint32_t)Hs), b = (int)(r / (uint32_t)Hs);
    float o[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const int cs = (int)q * 4 + l;
      float v = 0.f;
      if (cs < s * s * C) {
        const int t = cs / C, c = cs - t * C;
        const int dy = t / s, dx = t - dy * s;
        const int h = ii * s + dy - p, w = (int)j * s + dx - p;
        if (h >= 0 && h < xl.H && w >= 0 && w < xl.W) v = __ldg(x + lidx(xl, b, h, w, c));
      }
      o[l] = v;
    }
    reinterpret_cast<float4*>(xs)[e] = make_float4(o[0], o[1], o[2], o[3]);
  }
}

// Compile-time stride / channels (AlexNet: s = 4, C = 3, x one float4 per pixel): one
// thread per output float4 (16 per s2d pixel of ldc = 64: the pixel's 256 bytes are
// written by 16 consecutive threads), source channel / pixel decode by constants.
template <int S, int CC>
__global__ void __launch_bounds__(256) s2d_input_const_kernel(const float* __restrict__ x, wap_layout_t xl, int p,
                                                              int Hs, int Wsd, float* __restrict__ xs, int ldc) {
  const uint32_t q4n = (uint32_t)ldc / 4;
  const uint32_t total = (uint32_t)xl.B * Hs * Wsd * q4n;
  const int64_t xrow = (int64_t)(xl.W + xl.pad) * xl.ld;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const uint32_t q = e % q4n, pix = e / q4n;
    const uint32_t j = pix % (uint32_t)Wsd, r = pix / (uint32_t)Wsd;
    const int ii = (int)(r % (uint32_t)Hs), b = (int)(r / (uint32_t)Hs);
    const float* xb = x + lidx(xl, b, 0, 0, 0);
    float o[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const int cs = (int)q * 4 + l;
      const int t = cs / CC, c = cs - t * CC;  // constant divisors
      const int dy = t / S, dx = t - dy * S;
      const int h = ii * S + dy - p, w = (int)j * S + dx - p;
      o[l] = (cs < S * S * CC && h >= 0 && h < xl.H && w >= 0 && w < xl.W)
                 ? __ldg(xb + h * xrow + (int64_t)w * xl.ld + c)
                 : 0.f;
    }
    reinterpret_cast<float4*>(xs)[e] = make_float4(o[0], o[1], o[2], o[3]);
  }
}

// Narrow inputs (C <= 4 stored as one float4 per pixel, e.g. RGB padded to 4):
// one thread per (s2d pixel, source pixel t = dy*s + dx) reads that pixel's float4
// (coalesced along dx) and writes its C channels at t*C; threads t*C >= s*s*C
// zero the channel padding of their s2d pixel.
__global__ void __launch_bounds__(256) s2d_input_px4_kernel(const float* __restrict__ x, wap_layout_t xl, int s,
                                                            int p, int Hs, int Wsd, float* __restrict__ xs,
                                                            int ldc) {
  const int C = xl.C;
  const int ss = s * s;
  const uint32_t per = (uint32_t)(ldc / C > ss ? (ldc + C - 1) / C : ss);  // threads per s2d pixel
  const uint32_t total = (uint32_t)xl.B * Hs * Wsd * per;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const uint32_t t = e % per, pix = e / per;
    float* dst = xs + (int64_t)pix * ldc;
    if ((int)t >= ss) {  // channel padding of this pixel
      for (int c = (int)t * C; c < (int)(t + 1) * C && c < ldc; ++c) dst[c] = 0.f;
      continue;
    }
    const uint32_t j = pix % (uint32_t)Wsd, r = pix / (uint32_t)Wsd;
    const int ii = (int)(r % (uint32_t)Hs), b = (int)(r / (uint32_t)Hs);
    const int dy = (int)t / s, dx = (int)t - dy * s;
    const int h = ii * s + dy - p, w = (int)j * s + dx - p;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (h >= 0 && h < xl.H && w >= 0 && w < xl.W) v = __ldg(reinterpret_cast<const float4*>(x + lidx(xl, b, h, w, 0)));
    const float vv[4] = {v.x, v.y, v.z, v.w};
    for (int c = 0; c < C; ++c) dst[t * C + c] = vv[c];
  }
}

// ws[(a*ks + e)*ldc + cs][o] = w[s*a+dy][s*e+dx][c][o]; grad = 0: forward weight map,
// grad = 1: fold dws back into dw[u][v][c][o] (each (u, v, c) has exactly one source)
__global__ void s2d_weight_kernel(const float* __restrict__ src, float* __restrict__ dst, int k, int C, int Co,
                                  int ldw, int s, int ks, int ldc, int ldws, int grad) {
  const int64_t rows = grad ? (int64_t)k * k * C : (int64_t)ks * ks * ldc;
  const int64_t total = rows * Co;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int o = (int)(i % Co);
    const int64_t row = i / Co;
    if (!grad) {
      const int cs = (int)(row % ldc), tap = (int)(row / ldc);
      const int a = tap / ks, e = tap % ks;
      float v = 0.f;
      if (cs < s * s * C) {
        const int c = cs % C, t = cs / C;
        const int u = a * s + t / s, vv = e * s + t % s;
        if (u < k && vv < k) v = src[((int64_t)(u * k + vv) * C + c) * ldw + o];
      }
      dst[row * ldws + o] = v;
    } else {
      const int c = (int)(row % C), uv = (int)(row / C);
      const int u = uv / k, vv = uv % k;
      const int a = u / s, e = vv / s, cs = ((u % s) * s + (vv % s)) * C + c;
      dst[row * ldw + o] = src[((int64_t)(a * ks + e) * ldc + cs) * ldws + o];
    }
  }
}

// ---------------------------------------------------------------------------
// Direct first-layer conv (Ci <= 4, one float4 per input pixel): CUDA-core fp32
// ---------------------------------------------------------------------------
// A 3-channel stride-1 conv has K = k*k*3 = 27: as a GEMM it is one k-step per
// 128-row tile behind an im2col pass, so its cost is all epilogue and im2col
// traffic. Here each thread computes one output pixel x 32 output channels with
// exact fp32 FMAs (weights of its 32 channels broadcast from shared memory),
// applies bias / ReLU and writes the pixel's 32 channels; halo rows are untouched.
template <int KT, int CT>  // compile-time filter size / channels (0: runtime k, xl.C)
__global__ void __launch_bounds__(256) conv_direct_kernel(const float* __restrict__ x, wap_layout_t xl,
                                                          const float* __restrict__ w, int k_rt, int p, int ldw,
                                                          const float* __restrict__ bias, int relu,
                                                          float* __restrict__ y, wap_layout_t yl,
                                                          uint32_t* __restrict__ mbits, int64_t mbits_ld) {
  extern __shared__ __align__(16) float ws[];  // [k*k*Ci][32] weights of this channel group, then 32 biases
  const int C = CT ? CT : xl.C;
  const int k = KT ? KT : k_rt;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = blockIdx.y;  // 32-channel output group
  const int K = k * k * C;
  for (int i = threadIdx.x; i < K * 32; i += blockDim.x) ws[i] = w[(int64_t)(i >> 5) * ldw + grp * 32 + (i & 31)];
  if (threadIdx.x < 32) ws[K * 32 + threadIdx.x] = bias ? bias[grp * 32 + threadIdx.x] : 0.f;
  __syncthreads();
  const float4* ws4 = reinterpret_cast<const float4*>(ws);
  const uint32_t npix = (uint32_t)yl.B * yl.H * yl.W;
  for (uint32_t pix = (blockIdx.x * 8 + warp) * 32 + lane; pix < npix; pix += gridDim.x * 256) {
    const uint32_t wq = pix % (uint32_t)yl.W, r = pix / (uint32_t)yl.W;
    const int h = (int)(r % (uint32_t)yl.H), bb = (int)(r / (uint32_t)yl.H), wo = (int)wq;
    float acc[32];
#pragma unroll
    for (int o4 = 0; o4 < 8; ++o4) {
      const float4 bq = ws4[K * 8 + o4];
      acc[4 * o4] = bq.x; acc[4 * o4 + 1] = bq.y; acc[4 * o4 + 2] = bq.z; acc[4 * o4 + 3] = bq.w;
    }
#pragma unroll
    for (int u = 0; u < (KT ? KT : 16); ++u) {
      if (!KT && u >= k) break;
      const int hi = h + u - p;
#pragma unroll
      for (int v = 0; v < (KT ? KT : 16); ++v) {
        if (!KT && v >= k) break;
        const int wi = wo + v - p;
        float4 xv = make_float4(0.f, 0.f, 0.f, 0.f);
        if (hi >= 0 && hi < xl.H && wi >= 0 && wi < xl.W)
          xv = __ldg(reinterpret_cast<const float4*>(x + lidx(xl, bb, hi, wi, 0)));
        const float xa[4] = {xv.x, xv.y, xv.z, xv.w};
        const float4* wt = ws4 + (u * k + v) * C * 8;
#pragma unroll
        for (int c = 0; c < (CT ? CT : 4); ++c) {
          if (!CT && c >= C) break;
#pragma unroll
          for (int o4 = 0; o4 < 8; ++o4) {
            const float4 wq4 = wt[c * 8 + o4];  // broadcast: every lane reads the same 16 bytes
            acc[4 * o4] = fmaf(xa[c], wq4.x, acc[4 * o4]);
            acc[4 * o4 + 1] = fmaf(xa[c], wq4.y, acc[4 * o4 + 1]);
            acc[4 * o4 + 2] = fmaf(xa[c], wq4.z, acc[4 * o4 + 2]);
            acc[4 * o4 + 3] = fmaf(xa[c], wq4.w, acc[4 * o4 + 3]);
          }
        }
      }
    }
    const int64_t yrow = ((int64_t)bb * (yl.H + yl.pad) + h) * (yl.W + yl.pad) + wo;
    float* dst = y + yrow * yl.ld + grp * 32;
    uint32_t bits = 0;
#pragma unroll
    for (int o = 0; o < 32; o += 4) {
      float4 q = make_float4(acc[o], acc[o + 1], acc[o + 2], acc[o + 3]);
      if (relu) q = make_float4(fmaxf(q.x, 0.f), fmaxf(q.y, 0.f), fmaxf(q.z, 0.f), fmaxf(q.w, 0.f));
      bits |= ((q.x > 0.f) << o) | ((q.y > 0.f) << (o + 1)) | ((q.z > 0.f) << (o + 2)) | ((q.w > 0.f) << (o + 3));
      *reinterpret_cast<float4*>(dst + o) = q;
    }
    if (mbits) mbits[yrow * mbits_ld + grp] = bits;  // ReLU mask bits, as the GEMM epilogue writes them
  }
}

// conv_direct_kernel<3, 3> with two horizontally adjacent output pixels per thread:
// every broadcast weight load feeds two FMAs (the one-pixel kernel issues one LDS.128
// per 4 FMAs and is shared-memory-issue bound), and the two pixels share 2 of their 3
// input columns (12 loads instead of 18). Per-pixel FMA order is unchanged, so the
// outputs are the same floats as the one-pixel kernel.
__global__ void __launch_bounds__(256, 2) conv_direct_3x3c3_px2_kernel(const float* __restrict__ x, wap_layout_t xl,
                                                                    const float* __restrict__ w, int p, int ldw,
                                                                    const float* __restrict__ bias, int relu,
                                                                    float* __restrict__ y, wap_layout_t yl,
                                                                    uint32_t* __restrict__ mbits, int64_t mbits_ld) {
  constexpr int C = 3, K = 27;
  extern __shared__ __align__(16) float ws[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = blockIdx.y;
  for (int i = threadIdx.x; i < K * 32; i += blockDim.x) ws[i] = w[(int64_t)(i >> 5) * ldw + grp * 32 + (i & 31)];
  if (threadIdx.x < 32) ws[K * 32 + threadIdx.x] = bias ? bias[grp * 32 + threadIdx.x] : 0.f;
  __syncthreads();
  const float4* ws4 = reinterpret_cast<const float4*>(ws);
  const uint32_t Wp = ((uint32_t)yl.W + 1) >> 1;
  const uint32_t npair = (uint32_t)yl.B * yl.H * Wp;
  for (uint32_t pp = (blockIdx.x * 8 + warp) * 32 + lane; pp < npair; pp += gridDim.x * 256) {
    const uint32_t jq = pp % Wp, r = pp / Wp;
    const int h = (int)(r % (uint32_t)yl.H), bb = (int)(r / (uint32_t)yl.H), wo = (int)jq * 2;
    const bool two = wo + 1 < yl.W;
    float acc[2][32];
#pragma unroll
    for (int o4 = 0; o4 < 8; ++o4) {
      const float4 bq = ws4[K * 8 + o4];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        acc[e][4 * o4] = bq.x; acc[e][4 * o4 + 1] = bq.y; acc[e][4 * o4 + 2] = bq.z; acc[e][4 * o4 + 3] = bq.w;
      }
    }
#pragma unroll 1
    for (int u = 0; u < 3; ++u) {
      const int hi = h + u - p;
      float xa[4][4];  // input columns wo-p .. wo-p+3
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const int wi = wo + cc - p;
        float4 xv = make_float4(0.f, 0.f, 0.f, 0.f);
        if (hi >= 0 && hi < xl.H && wi >= 0 && wi < xl.W)
          xv = __ldg(reinterpret_cast<const float4*>(x + lidx(xl, bb, hi, wi, 0)));
        xa[cc][0] = xv.x; xa[cc][1] = xv.y; xa[cc][2] = xv.z; xa[cc][3] = xv.w;
      }
#pragma unroll
      for (int v = 0; v < 3; ++v) {
        const float4* wt = ws4 + (u * 3 + v) * C * 8;
#pragma unroll
        for (int c = 0; c < C; ++c) {
#pragma unroll
          for (int o4 = 0; o4 < 8; ++o4) {
            const float4 wq4 = wt[c * 8 + o4];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const float xe = xa[v + e][c];
              acc[e][4 * o4] = fmaf(xe, wq4.x, acc[e][4 * o4]);
              acc[e][4 * o4 + 1] = fmaf(xe, wq4.y, acc[e][4 * o4 + 1]);
              acc[e][4 * o4 + 2] = fmaf(xe, wq4.z, acc[e][4 * o4 + 2]);
              acc[e][4 * o4 + 3] = fmaf(xe, wq4.w, acc[e][4 * o4 + 3]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      if (e == 1 && !two) break;
      const int64_t yrow = ((int64_t)bb * (yl.H + yl.pad) + h) * (yl.W + yl.pad) + wo + e;
      float* dst = y + yrow * yl.ld + grp * 32;
      uint32_t bits = 0;
#pragma unroll
      for (int o = 0; o < 32; o += 4) {
        float4 q = make_float4(acc[e][o], acc[e][o + 1], acc[e][o + 2], acc[e][o + 3]);
        if (relu) q = make_float4(fmaxf(q.x, 0.f), fmaxf(q.y, 0.f), fmaxf(q.z, 0.f), fmaxf(q.w, 0.f));
        bits |= ((q.x > 0.f) << o) | ((q.y > 0.f) << (o + 1)) | ((q.z > 0.f) << (o + 2)) | ((q.w > 0.f) << (o + 3));
        *reinterpret_cast<float4*>(dst + o) = q;
      }
      if (mbits) mbits[yrow * mbits_ld + grp] = bits;
    }
  }
}

// ---------------------------------------------------------------------------
// MaxPool
// ---------------------------------------------------------------------------
// Row-blocked launches: blockIdx.y = b * H + h (one output row for the forward,
// one input row for the backward), threads sweep (w, 4-channel group) of that row
// with 32-bit indices; row geometry is decoded once per block.
//
// ReLU-fused argmax (flags & WAP_POOL_RELU_FUSED): when the pool input is a ReLU
// output and the backward is fused with that ReLU's GradReLU, the forward stores
// 0xFF for windows whose max is <= 0. The GradReLU mask at the argmax element is
// exactly (max > 0) (the max of ReLU outputs is positive iff its first argmax is),
// so the backward needs no mask read (interp.py:197-198 on the pooled element).
constexpr uint8_t kNoGrad = 0xFF;

__global__ void __launch_bounds__(256) maxpool_fwd_kernel(const float* __restrict__ x, wap_layout_t xl, int win,
                                                          int s, float* __restrict__ y, wap_layout_t yl,
                                                          uint8_t* __restrict__ arg, int relu_fused) {
  const int c4n = yl.ld / 4;
  const int per = yl.W * c4n;
  for (int row = blockIdx.y; row < yl.B * yl.H; row += gridDim.y) {
  const int b = row / yl.H, ho = row - (row / yl.H) * yl.H;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < per; j += gridDim.x * blockDim.x) {
    const int wo = j / c4n;
    const int c = (j - wo * c4n) * 4;
    float best[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    int bi[4] = {0, 0, 0, 0};
    const float* xr = x + lidx(xl, b, ho * s, wo * s, c);
    const int64_t xrow = (int64_t)(xl.W + xl.pad) * xl.ld;
    for (int a2 = 0; a2 < win; ++a2)
      for (int bb = 0; bb < win; ++bb) {
        const float4 v = *reinterpret_cast<const float4*>(xr + a2 * xrow + (int64_t)bb * xl.ld);
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (vv[t] > best[t]) { best[t] = vv[t]; bi[t] = a2 * win + bb; }
      }
    float o[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      o[t] = (c + t < yl.C) ? best[t] : 0.f;
      if (relu_fused && !(best[t] > 0.f)) bi[t] = kNoGrad;
    }
    const int64_t yi = lidx(yl, b, ho, wo, c);
    *reinterpret_cast<float4*>(y + yi) = make_float4(o[0], o[1], o[2], o[3]);
    if (arg) *reinterpret_cast<uchar4*>(arg + yi) = make_uchar4((uint8_t)bi[0], (uint8_t)bi[1], (uint8_t)bi[2],
                                                                (uint8_t)bi[3]);
  }
  }
}

// Gather form (windows may overlap): dx[h, w] = sum over the windows containing
// (h, w) whose argmax is (h, w) of dy. WIN / S as template constants turn the window
// range arithmetic into shifts (AlexNet 3/2, VGG 2/2); 0 / 0 = runtime values.
template <int WINT, int ST>
__global__ void __launch_bounds__(256) maxpool_bwd_kernel(const uint8_t* __restrict__ arg,
                                                          const float* __restrict__ dy, wap_layout_t yl, int win_rt,
                                                          int s_rt, float* __restrict__ dx, wap_layout_t xl,
                                                          const float* __restrict__ mask, wap_layout_t ml) {
  const int win = WINT ? WINT : win_rt, s = ST ? ST : s_rt;
  const int c4n = xl.ld / 4;
  const int64_t yrow_stride = (int64_t)(yl.W + yl.pad) * yl.ld;
  for (int row = blockIdx.y; row < xl.B * xl.H; row += gridDim.y) {
    const int b = row / xl.H, h = row - (row / xl.H) * xl.H;
    // windows (ho, wo) with ho*s <= h < ho*s + win
    const int ho_lo = h >= win ? (h - win) / s + 1 : 0;
    const int ho_hi = min(h / s, yl.H - 1);
    const int64_t y0 = lidx(yl, b, ho_lo, 0, 0);  // start of pooled row ho_lo
    float* dxrow = dx + lidx(xl, b, h, 0, 0);
    const float* mrow = mask ? mask + lidx(ml, b, h, 0, 0) : nullptr;
    const int per = xl.W * c4n;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < per; j += gridDim.x * blockDim.x) {
      const int w = j / c4n;
      const int c = (j - w * c4n) * 4;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      const int wo_lo = w >= win ? (w - win) / s + 1 : 0;
      const int wo_hi = min(w / s, yl.W - 1);
      int64_t yr = y0;
      for (int ho = ho_lo; ho <= ho_hi; ++ho, yr += yrow_stride) {
        const int lh = (h - ho * s) * win;
        for (int wo = wo_lo; wo <= wo_hi; ++wo) {
          const int local = lh + (w - wo * s);
          const int64_t yi = yr + (int64_t)wo * yl.ld + c;
          const uchar4 a4 = *reinterpret_cast<const uchar4*>(arg + yi);
          const float4 g = __ldg(reinterpret_cast<const float4*>(dy + yi));
          if (a4.x == local) acc.x += g.x;
          if (a4.y == local) acc.y += g.y;
          if (a4.z == local) acc.z += g.z;
          if (a4.w == local) acc.w += g.w;
        }
      }
      if (mrow) {
        const float4 m = __ldg(reinterpret_cast<const float4*>(mrow + (int64_t)w * ml.ld + c));
        if (!(m.x > 0.f)) acc.x = 0.f;
        if (!(m.y > 0.f)) acc.y = 0.f;
        if (!(m.z > 0.f)) acc.z = 0.f;
        if (!(m.w > 0.f)) acc.w = 0.f;
      }
      if (c + 0 >= xl.C) acc.x = 0.f;
      if (c + 1 >= xl.C) acc.y = 0.f;
      if (c + 2 >= xl.C) acc.z = 0.f;
      if (c + 3 >= xl.C) acc.w = 0.f;
      *reinterpret_cast<float4*>(dxrow + (int64_t)w * xl.ld + c) = acc;
    }
  }
}

// Stride-2 patch form (AlexNet 3/2, VGG 2/2): one thread owns a 2x2 block of input
// pixels x 4 channels. For s = 2 that block lies in at most (WIN-1)^2 windows
// (ho in {i-1, i} x wo in {j-1, j} for WIN 3; just (i, j) for WIN 2), so each
// pooled (argmax, dy) pair is loaded once per block instead of once per pixel it
// covers (9 -> 4 loads per 4 pixels for 3/2), and the window-relative offsets are
// compile-time. Windows are visited in the per-pixel gather's order (ho, then wo
// ascending), so every dx element is the same float sum, bit for bit.
template <int WIN>
__global__ void __launch_bounds__(256) maxpool_bwd_s2_kernel(const uint8_t* __restrict__ arg,
                                                             const float* __restrict__ dy, wap_layout_t yl,
                                                             float* __restrict__ dx, wap_layout_t xl,
                                                             const float* __restrict__ mask, wap_layout_t ml) {
  constexpr int NW = WIN - 1;  // windows per axis covering a 2-pixel span
  const int c4n = xl.ld / 4;
  const int PH = (xl.H + 1) >> 1, PW = (xl.W + 1) >> 1;
  const int per = PW * c4n;
  const int64_t xrs = (int64_t)(xl.W + xl.pad) * xl.ld;
  const int64_t mrs = (int64_t)(ml.W + ml.pad) * ml.ld;
  for (int prow = blockIdx.y; prow < xl.B * PH; prow += gridDim.y) {
    const int b = prow / PH, i = prow - b * PH;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < per; j += gridDim.x * blockDim.x) {
      const int jj = j / c4n;
      const int c = (j - jj * c4n) * 4;
      float4 acc[2][2];
#pragma unroll
      for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int q = 0; q < 2; ++q) acc[p][q] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int a = 0; a < NW; ++a) {
        const int ho = i - (NW - 1) + a;
        if (ho < 0 || ho >= yl.H) continue;
#pragma unroll
        for (int bb = 0; bb < NW; ++bb) {
          const int wo = jj - (NW - 1) + bb;
          if (wo < 0 || wo >= yl.W) continue;
          const int64_t yi = lidx(yl, b, ho, wo, c);
          const uchar4 a4 = *reinterpret_cast<const uchar4*>(arg + yi);
          const float4 g = __ldg(reinterpret_cast<const float4*>(dy + yi));
#pragma unroll
          for (int p = 0; p < 2; ++p) {
            const int r = 2 * (NW - 1 - a) + p;  // row of pixel (2i+p) inside window ho
            if (r >= WIN) continue;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int cc = 2 * (NW - 1 - bb) + q;
              if (cc >= WIN) continue;
              const int local = r * WIN + cc;
              if (a4.x == local) acc[p][q].x += g.x;
              if (a4.y == local) acc[p][q].y += g.y;
              if (a4.z == local) acc[p][q].z += g.z;
              if (a4.w == local) acc[p][q].w += g.w;
            }
          }
        }
      }
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const int h = 2 * i + p;
        if (h >= xl.H) continue;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int w = 2 * jj + q;
          if (w >= xl.W) continue;
          float4 v = acc[p][q];
          if (mask) {
            const float4 m = __ldg(reinterpret_cast<const float4*>(mask + b * (int64_t)(ml.H + ml.pad) * mrs +
                                                                   h * mrs + (int64_t)w * ml.ld + c));
            if (!(m.x > 0.f)) v.x = 0.f;
            if (!(m.y > 0.f)) v.y = 0.f;
            if (!(m.z > 0.f)) v.z = 0.f;
            if (!(m.w > 0.f)) v.w = 0.f;
          }
          if (c + 0 >= xl.C) v.x = 0.f;
          if (c + 1 >= xl.C) v.y = 0.f;
          if (c + 2 >= xl.C) v.z = 0.f;
          if (c + 3 >= xl.C) v.w = 0.f;
          *reinterpret_cast<float4*>(dx + b * (int64_t)(xl.H + xl.pad) * xrs + h * xrs + (int64_t)w * xl.ld + c) = v;
        }
      }
    }
  }
}

// rows beyond gridDim.y's 65535 limit are covered by the kernels' row loop
dim3 pool_grid(int rows, int per) {
  return dim3((unsigned)std::max(1, std::min((per + 255) / 256, 64)), (unsigned)std::min(rows, 65535));
}

// ---------------------------------------------------------------------------
// LRN: a block handles PIX pixels; channels staged in shared memory
// ---------------------------------------------------------------------------
constexpr int LRN_PIX = 8;

__device__ __forceinline__ void pixel_of(const wap_layout_t& l, int64_t p, int& b, int& h, int& w) {
  // pixel counts of one layer stay below 2^31 (host-checked): 32-bit division
  const uint32_t q = (uint32_t)p;
  const uint32_t r = q / (uint32_t)l.W;
  w = (int)(q - r * (uint32_t)l.W);
  const uint32_t bb = r / (uint32_t)l.H;
  h = (int)(r - bb * (uint32_t)l.H);
  b = (int)bb;
}

__global__ void lrn_fwd_kernel(const float* __restrict__ x, wap_layout_t xl, int size, float alpha, float beta,
                               float k, float* __restrict__ y, wap_layout_t yl) {
  extern __shared__ float sx[];  // [LRN_PIX][C]
  const int C = xl.C;
  const int64_t npix = (int64_t)xl.B * xl.H * xl.W;
  const int half = size / 2;
  for (int64_t p0 = (int64_t)blockIdx.x * LRN_PIX; p0 < npix; p0 += (int64_t)gridDim.x * LRN_PIX) {
    __syncthreads();
    for (int t = threadIdx.x; t < LRN_PIX * C; t += blockDim.x) {
      const int pi = t / C, c = t % C;
      const int64_t p = p0 + pi;
      float v = 0.f;
      if (p < npix) {
        int b, h, w;
        pixel_of(xl, p, b, h, w);
        v = x[lidx(xl, b, h, w, c)];
      }
      sx[t] = v;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < LRN_PIX * yl.ld; t += blockDim.x) {
      const int pi = t / yl.ld, c = t % yl.ld;
      const int64_t p = p0 + pi;
      if (p >= npix) continue;
      int b, h, w;
      pixel_of(yl, p, b, h, w);
      float out = 0.f;
      if (c < C) {
        float ss = 0.f;
        const int lo = max(0, c - half), hi = min(C - 1, c + half);
        for (int j = lo; j <= hi; ++j) ss += sx[pi * C + j] * sx[pi * C + j];
        out = sx[pi * C + c] * powf(k + alpha * ss, -beta);
      }
      y[lidx(yl, b, h, w, c)] = out;
    }
  }
}

__global__ void lrn_bwd_kernel(const float* __restrict__ x, wap_layout_t xl, const float* __restrict__ dy,
                               wap_layout_t dyl, int size, float alpha, float beta, float k, float* __restrict__ dx,
                               wap_layout_t dxl, const float* __restrict__ mask, wap_layout_t ml) {
  extern __shared__ float sh[];  // x, dy, t (= dy*x*s^(-beta-1)), pw (= s^-beta): 4 * [LRN_PIX][C]
  const int C = xl.C;
  float* sx = sh;
  float* sd = sh + LRN_PIX * C;
  float* st = sh + 2 * LRN_PIX * C;
  float* sp = sh + 3 * LRN_PIX * C;
  const int64_t npix = (int64_t)xl.B * xl.H * xl.W;
  const int half = size / 2;
  for (int64_t p0 = (int64_t)blockIdx.x * LRN_PIX; p0 < npix; p0 += (int64_t)gridDim.x * LRN_PIX) {
    __syncthreads();
    for (int t = threadIdx.x; t < LRN_PIX * C; t += blockDim.x) {
      const int pi = t / C, c = t % C;
      const int64_t p = p0 + pi;
      float vx = 0.f, vd = 0.f;
      if (p < npix) {
        int b, h, w;
        pixel_of(xl, p, b, h, w);
        vx = x[lidx(xl, b, h, w, c)];
        vd = dy[lidx(dyl, b, h, w, c)];
      }
      sx[t] = vx;
      sd[t] = vd;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < LRN_PIX * C; t += blockDim.x) {
      const int pi = t / C, c = t % C;
      float ss = 0.f;
      const int lo = max(0, c - half), hi = min(C - 1, c + half);
      for (int j = lo; j <= hi; ++j) ss += sx[pi * C + j] * sx[pi * C + j];
      const float s = k + alpha * ss;
      const float pw = powf(s, -beta);
      sp[t] = pw;
      st[t] = sd[t] * sx[t] * pw / s;
    }
    __syncthreads();
    for (int t = threadIdx.x; t < LRN_PIX * dxl.ld; t += blockDim.x) {
      const int pi = t / dxl.ld, c = t % dxl.ld;
      const int64_t p = p0 + pi;
      if (p >= npix) continue;
      int b, h, w;
      pixel_of(dxl, p, b, h, w);
      float out = 0.f;
      if (c < C) {
        float acc = 0.f;
        const int lo = max(0, c - half), hi = min(C - 1, c + half);
        for (int j = lo; j <= hi; ++j) acc += st[pi * C + j];
        out = sd[pi * C + c] * sp[pi * C + c] - 2.f * alpha * beta * sx[pi * C + c] * acc;
        if (mask && !(mask[lidx(ml, b, h, w, c)] > 0.f)) out = 0.f;
      }
      dx[lidx(dxl, b, h, w, c)] = out;
    }
  }
}

// Fast LRN for compact channels (ld == C, C % 4 == 0, C4 = C/4 known at compile
// time): float4 tile loads into shared memory, per-pixel decode once, fast
// log2/exp2 power. `PIX` pixels per block iteration.
__device__ __forceinline__ float lrn_pow(float s, float e) { return exp2f(e * __log2f(s)); }

template <int C4, int PIX, bool BWD>
__global__ void __launch_bounds__(256) lrn_fast_kernel(const float* __restrict__ x, wap_layout_t xl,
                                                       const float* __restrict__ dy, wap_layout_t dyl, int size,
                                                       float alpha, float beta, float k, float* __restrict__ out,
                                                       wap_layout_t ol, const float* __restrict__ mask,
                                                       wap_layout_t ml) {
  constexpr int C = C4 * 4;
  __shared__ float4 sx[PIX * C4];
  __shared__ float4 sd[BWD ? PIX * C4 : 1];
  __shared__ float st[BWD ? PIX * C : 1];
  __shared__ int64_t px[PIX], pd[BWD ? PIX : 1], po[PIX], pm[BWD ? PIX : 1];
  const int64_t npix = (int64_t)xl.B * xl.H * xl.W;
  const int half = size / 2;
  for (int64_t p0 = (int64_t)blockIdx.x * PIX; p0 < npix; p0 += (int64_t)gridDim.x * PIX) {
    __syncthreads();
    if (threadIdx.x < PIX) {
      int64_t p = p0 + threadIdx.x;
      if (p >= npix) p = npix - 1;
      int b, h, w;
      pixel_of(xl, p, b, h, w);
      px[threadIdx.x] = lidx(xl, b, h, w, 0);
      po[threadIdx.x] = lidx(ol, b, h, w, 0);
      if (BWD) {
        pd[threadIdx.x] = lidx(dyl, b, h, w, 0);
        pm[threadIdx.x] = mask ? lidx(ml, b, h, w, 0) : 0;
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < PIX * C4; i += blockDim.x) {
      const int pi = i / C4, c4 = i % C4;
      sx[i] = *reinterpret_cast<const float4*>(x + px[pi] + 4 * c4);
      if (BWD) sd[i] = *reinterpret_cast<const float4*>(dy + pd[pi] + 4 * c4);
    }
    __syncthreads();
    const float* fx = reinterpret_cast<const float*>(sx);
    if (BWD) {
      const float* fd = reinterpret_cast<const float*>(sd);
      for (int i = threadIdx.x; i < PIX * C; i += blockDim.x) {
        const int pi = i / C, c = i % C;
        const float* row = fx + pi * C;
        float ss = 0.f;
        for (int j = max(0, c - half); j <= min(C - 1, c + half); ++j) ss += row[j] * row[j];
        const float s = k + alpha * ss;
        st[i] = fd[i] * row[c] * lrn_pow(s, -beta - 1.f);
      }
      __syncthreads();
    }
    for (int i = threadIdx.x; i < PIX * C4; i += blockDim.x) {
      const int pi = i / C4, c0 = (i % C4) * 4;
      if (p0 + pi >= npix) continue;
      const float* row = fx + pi * C;
      float o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = c0 + j;
        float ss = 0.f;
        for (int q = max(0, c - half); q <= min(C - 1, c + half); ++q) ss += row[q] * row[q];
        const float s = k + alpha * ss;
        if (!BWD) {
          o[j] = row[c] * lrn_pow(s, -beta);
        } else {
          const float* trow = st + pi * C;
          float acc = 0.f;
          for (int q = max(0, c - half); q <= min(C - 1, c + half); ++q) acc += trow[q];
          const float* drow = reinterpret_cast<const float*>(sd) + pi * C;
          o[j] = drow[c] * lrn_pow(s, -beta) - 2.f * alpha * beta * row[c] * acc;
        }
      }
      if (BWD && mask) {
        const float4 m = *reinterpret_cast<const float4*>(mask + pm[pi] + c0);
        if (!(m.x > 0.f)) o[0] = 0.f;
        if (!(m.y > 0.f)) o[1] = 0.f;
        if (!(m.z > 0.f)) o[2] = 0.f;
        if (!(m.w > 0.f)) o[3] = 0.f;
      }
      *reinterpret_cast<float4*>(out + po[pi] + c0) = make_float4(o[0], o[1], o[2], o[3]);
    }
  }
}

// LRN (size 5) of one lane's 4*VPL contiguous channels of a pixel whose channels are
// spread over 16 lanes (lane sl of its half-warp): forward y = x * s^-beta, backward
// dx = dy * s^-beta - 2*alpha*beta * x * sum_window(dy * x * s^-beta / s), the +-2
// channel window crossing lanes through 16-wide shuffles. Shared by the LRN kernels
// and the fused MaxPool+LRN backward, so both produce the same floats.
template <int VPL, bool BWD>
__device__ __forceinline__ void lrn_lane(const float* v, const float* d, int sl, float alpha, float beta, float k,
                                         float* o) {
  constexpr int NV = 4 * VPL;
  float q[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) q[j] = v[j] * v[j];
    // window sums of squares over channels c-2..c+2
    float pm2 = __shfl_up_sync(0xffffffffu, q[NV - 2], 1, 16), pm1 = __shfl_up_sync(0xffffffffu, q[NV - 1], 1, 16);
    float np0 = __shfl_down_sync(0xffffffffu, q[0], 1, 16), np1 = __shfl_down_sync(0xffffffffu, q[1], 1, 16);
    if (sl == 0) pm2 = pm1 = 0.f;
    if (sl == 15) np0 = np1 = 0.f;
    float s[NV], pw[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      float acc = q[j];
      acc += (j >= 1) ? q[j - 1] : pm1;
      acc += (j >= 2) ? q[j - 2] : (j == 1 ? pm1 : pm2);
      acc += (j + 1 < NV) ? q[j + 1] : np0;
      acc += (j + 2 < NV) ? q[j + 2] : (j + 1 < NV ? np0 : np1);
      s[j] = k + alpha * acc;
      pw[j] = exp2f(-beta * __log2f(s[j]));
    }
    if (!BWD) {
#pragma unroll
      for (int j = 0; j < NV; ++j) o[j] = v[j] * pw[j];
    } else {
      float t[NV];
#pragma unroll
      for (int j = 0; j < NV; ++j) t[j] = __fdividef(d[j] * v[j] * pw[j], s[j]);
      float tm2 = __shfl_up_sync(0xffffffffu, t[NV - 2], 1, 16), tm1 = __shfl_up_sync(0xffffffffu, t[NV - 1], 1, 16);
      float tp0 = __shfl_down_sync(0xffffffffu, t[0], 1, 16), tp1 = __shfl_down_sync(0xffffffffu, t[1], 1, 16);
      if (sl == 0) tm2 = tm1 = 0.f;
      if (sl == 15) tp0 = tp1 = 0.f;
#pragma unroll
      for (int j = 0; j < NV; ++j) {
        float acc = t[j];
        acc += (j >= 1) ? t[j - 1] : tm1;
        acc += (j >= 2) ? t[j - 2] : (j == 1 ? tm1 : tm2);
        acc += (j + 1 < NV) ? t[j + 1] : tp0;
        acc += (j + 2 < NV) ? t[j + 2] : (j + 1 < NV ? tp0 : tp1);
        o[j] = d[j] * pw[j] - 2.f * alpha * beta * v[j] * acc;
      }
    }
}

// Register-only LRN (size 5): 16 lanes per pixel, VPL float4 (4*VPL channels)
// per lane, the +-2 channel window crosses lanes through 16-wide shuffles.
// One coalesced read of x (+dy, mask) and one write per element: HBM-bound.
template <int VPL, bool BWD>
__global__ void __launch_bounds__(256, VPL == 1 ? (BWD ? 6 : 8) : 2) lrn_warp_kernel(const float* __restrict__ x, wap_layout_t xl,
                                                       const float* __restrict__ dy, wap_layout_t dyl, float alpha,
                                                       float beta, float k, float* __restrict__ out, wap_layout_t ol,
                                                       const float* __restrict__ mask, wap_layout_t ml) {
  constexpr int NV = 4 * VPL;
  const int lane = threadIdx.x & 31;
  const int sl = lane & 15;
  const bool mask_is_x = BWD && mask == x && ml.pad == xl.pad && ml.ld == xl.ld;
  const int64_t npix = (int64_t)xl.B * xl.H * xl.W;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int c0 = sl * NV;
  for (int64_t pbase = wid * 2; pbase < npix; pbase += nw * 2) {
    const int64_t p = pbase + (lane >> 4);
    const bool ok = p < npix;
    int b = 0, h = 0, w = 0;
    if (ok) pixel_of(xl, p, b, h, w);
    float v[NV], d[NV];
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f), g = a;
      if (ok) {
        a = *reinterpret_cast<const float4*>(x + lidx(xl, b, h, w, c0 + 4 * i));
        if (BWD) g = *reinterpret_cast<const float4*>(dy + lidx(dyl, b, h, w, c0 + 4 * i));
      }
      v[4 * i] = a.x; v[4 * i + 1] = a.y; v[4 * i + 2] = a.z; v[4 * i + 3] = a.w;
      d[4 * i] = g.x; d[4 * i + 1] = g.y; d[4 * i + 2] = g.z; d[4 * i + 3] = g.w;
    }
    float o[NV];
    lrn_lane<VPL, BWD>(v, d, sl, alpha, beta, k, o);
    if (!ok) continue;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      float4 r = make_float4(o[4 * i], o[4 * i + 1], o[4 * i + 2], o[4 * i + 3]);
      if (BWD && mask_is_x) {
        // GradReLU mask source is the LRN input itself (ReLU -> LRN): reuse the loaded x
        if (!(v[4 * i] > 0.f)) r.x = 0.f;
        if (!(v[4 * i + 1] > 0.f)) r.y = 0.f;
        if (!(v[4 * i + 2] > 0.f)) r.z = 0.f;
        if (!(v[4 * i + 3] > 0.f)) r.w = 0.f;
      } else if (BWD && mask) {
        const float4 m = *reinterpret_cast<const float4*>(mask + lidx(ml, b, h, w, c0 + 4 * i));
        if (!(m.x > 0.f)) r.x = 0.f;
        if (!(m.y > 0.f)) r.y = 0.f;
        if (!(m.z > 0.f)) r.z = 0.f;
        if (!(m.w > 0.f)) r.w = 0.f;
      }
      *reinterpret_cast<float4*>(out + lidx(ol, b, h, w, c0 + 4 * i)) = r;
    }
  }
}

// LRN forward, C = 64: lrn_warp_kernel<1, false> with U pixel pairs per warp
// iteration whose loads are all issued before any math (2x the bytes in flight of
// the one-pair loop). Same lrn_lane math, same floats.
template <int U>
__global__ void __launch_bounds__(256, 8) lrn_fwd_c64_kernel(const float* __restrict__ x, wap_layout_t xl,
                                                             float alpha, float beta, float k,
                                                             float* __restrict__ out, wap_layout_t ol) {
  const int lane = threadIdx.x & 31;
  const int sl = lane & 15;
  const int64_t npix = (int64_t)xl.B * xl.H * xl.W;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int c0 = sl * 4;
  for (int64_t pbase = wid * 2 * U; pbase < npix; pbase += nw * 2 * U) {
    float v[U][4];
    int64_t oi[U];
    bool ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t p = pbase + 2 * u + (lane >> 4);
      ok[u] = p < npix;
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      oi[u] = 0;
      if (ok[u]) {
        int b, h, w;
        pixel_of(xl, p, b, h, w);
        a = *reinterpret_cast<const float4*>(x + lidx(xl, b, h, w, c0));
        oi[u] = lidx(ol, b, h, w, c0);
      }
      v[u][0] = a.x; v[u][1] = a.y; v[u][2] = a.z; v[u][3] = a.w;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float o[4];
      lrn_lane<1, false>(v[u], v[u], sl, alpha, beta, k, o);
      if (ok[u]) *reinterpret_cast<float4*>(out + oi[u]) = make_float4(o[0], o[1], o[2], o[3]);
    }
  }
}

// Fused LRN (size 5) -> MaxPool forward (AlexNet norm1 -> pool1, norm2 -> pool2) when
// the LRN output has no other reader: a half-warp owns one pooled pixel, lane sl the
// 4*VPL channels lrn_lane expects; each window pixel's LRN is computed in registers
// and max-reduced in maxpool_fwd_kernel's order (rows, then columns; first max wins),
// so pooled values and argmax are the same as the two-kernel path, and the LRN output
// tensor is never written or re-read. (Overlapping 3/2 windows recompute 2.25x LRN.)
template <int WIN, int VPL>
__global__ void __launch_bounds__(256) lrn_maxpool_fwd_kernel(const float* __restrict__ x, wap_layout_t xl,
                                                              float alpha, float beta, float k, int s,
                                                              float* __restrict__ y, wap_layout_t yl,
                                                              uint8_t* __restrict__ arg) {
  constexpr int NV = 4 * VPL;
  const int lane = threadIdx.x & 31;
  const int sl = lane & 15;
  const int c0 = sl * NV;
  const int64_t nout = (int64_t)yl.B * yl.H * yl.W;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t pbase = wid * 2; pbase < nout; pbase += nw * 2) {
    const int64_t p = pbase + (lane >> 4);
    const bool ok = p < nout;
    int b = 0, ho = 0, wo = 0;
    if (ok) pixel_of(yl, p, b, ho, wo);
    float best[NV];
    int bi[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) { best[j] = -INFINITY; bi[j] = 0; }
#pragma unroll
    for (int a2 = 0; a2 < WIN; ++a2) {
#pragma unroll
      for (int bb = 0; bb < WIN; ++bb) {
        float v[NV], o[NV];
#pragma unroll
        for (int t = 0; t < VPL; ++t) {
          float4 xa = make_float4(0.f, 0.f, 0.f, 0.f);
          if (ok) xa = *reinterpret_cast<const float4*>(x + lidx(xl, b, ho * s + a2, wo * s + bb, c0 + 4 * t));
          v[4 * t] = xa.x; v[4 * t + 1] = xa.y; v[4 * t + 2] = xa.z; v[4 * t + 3] = xa.w;
        }
        lrn_lane<VPL, false>(v, v, sl, alpha, beta, k, o);
#pragma unroll
        for (int j = 0; j < NV; ++j)
          if (o[j] > best[j]) { best[j] = o[j]; bi[j] = a2 * WIN + bb; }
      }
    }
    if (!ok) continue;
#pragma unroll
    for (int t = 0; t < VPL; ++t) {
      const int64_t yi = lidx(yl, b, ho, wo, c0 + 4 * t);
      *reinterpret_cast<float4*>(y + yi) = make_float4(best[4 * t], best[4 * t + 1], best[4 * t + 2], best[4 * t + 3]);
      if (arg)
        *reinterpret_cast<uchar4*>(arg + yi) = make_uchar4((uint8_t)bi[4 * t], (uint8_t)bi[4 * t + 1],
                                                           (uint8_t)bi[4 * t + 2], (uint8_t)bi[4 * t + 3]);
    }
  }
}

// Row-band form of the fused LRN -> MaxPool forward: a block owns image b and pooled rows
// [ho0, ho0 + R); it computes the LRN of every input pixel of rows
// [ho0*s, (ho0+R-1)*s + WIN) ONCE into shared memory (lrn_lane, so the same floats), then
// pools from shared memory in maxpool_fwd_kernel's order (rows, then columns; first max
// wins). Values and argmax are bitwise those of lrn_maxpool_fwd_kernel, which recomputes
// each LRN up to (WIN/s)^2 = 2.25x for 3/2 windows and measured compute-bound (r01 ncu).
// Recompute here: (R*s + WIN - s) / (R*s) input rows per pooled row (1.25x at R = 2).
template <int WIN, int VPL>
__global__ void __launch_bounds__(256) lrn_maxpool_band_kernel(const float* __restrict__ x, wap_layout_t xl,
                                                               float alpha, float beta, float k, int s, int R,
                                                               float* __restrict__ y, wap_layout_t yl,
                                                               uint8_t* __restrict__ arg) {
  constexpr int NV = 4 * VPL;
  constexpr int C = 64 * VPL;
  extern __shared__ float4 band4[];
  float* band = reinterpret_cast<float*>(band4);
  const int lane = threadIdx.x & 31;
  const int sl = lane & 15;
  const int c0 = sl * NV;
  const int hw = threadIdx.x >> 4;  // half-warp 0..15
  const int bands = (yl.H + R - 1) / R;
  const int b = blockIdx.x / bands;
  const int ho0 = (blockIdx.x - b * bands) * R;
  const int nho = min(R, yl.H - ho0);
  const int h0 = ho0 * s;
  const int nrows = min((nho - 1) * s + WIN, xl.H - h0);
  const int npx = nrows * xl.W;
  // phase 1: LRN of every input pixel of the band, one half-warp per pixel. The two
  // half-warps of a warp iterate together (lrn_lane shuffles with the full-warp mask);
  // the second one idles on the last odd pixel.
  for (int qb = (hw & ~1); qb < npx; qb += 16) {
    const int q = qb + (hw & 1);
    const bool ok = q < npx;
    const int r = ok ? q / xl.W : 0, w = ok ? q - r * xl.W : 0;
    float v[NV], o[NV];
#pragma unroll
    for (int t = 0; t < VPL; ++t) {
      float4 xa = make_float4(0.f, 0.f, 0.f, 0.f);
      if (ok) xa = *reinterpret_cast<const float4*>(x + lidx(xl, b, h0 + r, w, c0 + 4 * t));
      v[4 * t] = xa.x; v[4 * t + 1] = xa.y; v[4 * t + 2] = xa.z; v[4 * t + 3] = xa.w;
    }
    lrn_lane<VPL, false>(v, v, sl, alpha, beta, k, o);
    if (!ok) continue;
    float* dst = band + (int64_t)q * C + c0;
#pragma unroll
    for (int t = 0; t < VPL; ++t)
      *reinterpret_cast<float4*>(dst + 4 * t) = make_float4(o[4 * t], o[4 * t + 1], o[4 * t + 2], o[4 * t + 3]);
  }
  __syncthreads();
  // phase 2: pooled outputs of the band from shared memory
  const int nout = nho * yl.W;
  for (int q = hw; q < nout; q += 16) {
    const int ro = q / yl.W, wo = q - ro * yl.W;
    float best[NV];
    int bi[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) { best[j] = -INFINITY; bi[j] = 0; }
#pragma unroll
    for (int a2 = 0; a2 < WIN; ++a2) {
#pragma unroll
      for (int bb = 0; bb < WIN; ++bb) {
        const float* src = band + ((int64_t)(ro * s + a2) * xl.W + wo * s + bb) * C + c0;
#pragma unroll
        for (int t = 0; t < VPL; ++t) {
          const float4 o4 = *reinterpret_cast<const float4*>(src + 4 * t);
          const float o[4] = {o4.x, o4.y, o4.z, o4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (o[e] > best[4 * t + e]) { best[4 * t + e] = o[e]; bi[4 * t + e] = a2 * WIN + bb; }
        }
      }
    }
#pragma unroll
    for (int t = 0; t < VPL; ++t) {
      const int64_t yi = lidx(yl, b, ho0 + ro, wo, c0 + 4 * t);
      *reinterpret_cast<float4*>(y + yi) = make_float4(best[4 * t], best[4 * t + 1], best[4 * t + 2], best[4 * t + 3]);
      if (arg)
        *reinterpret_cast<uchar4*>(arg + yi) = make_uchar4((uint8_t)bi[4 * t], (uint8_t)bi[4 * t + 1],
                                                           (uint8_t)bi[4 * t + 2], (uint8_t)bi[4 * t + 3]);
    }
  }
}

// Fused MaxPool backward (stride 2) -> LRN backward (size 5) -> GradReLU, for a
// MaxPool whose input is an LRN output (AlexNet norm1 -> pool1, norm2 -> pool2):
// a half-warp owns one 2x2 block of pooled-from pixels, lane sl the 4*VPL contiguous
// channels lrn_lane expects. The pool gradient of the block is gathered exactly as
// maxpool_bwd_s2_kernel does (same window order) and stays in registers as the LRN's
// dy, so the intermediate tensor is never written or re-read.
template <int WIN, int VPL>
__global__ void __launch_bounds__(256, VPL == 1 ? 4 : 2) maxpool_lrn_bwd_kernel(
    const uint8_t* __restrict__ arg, const float* __restrict__ dy, wap_layout_t yl, const float* __restrict__ x,
    wap_layout_t xl, float alpha, float beta, float k, float* __restrict__ out, wap_layout_t ol,
    const float* __restrict__ mask, wap_layout_t ml) {
  constexpr int NW = WIN - 1;
  constexpr int NV = 4 * VPL;
  const int lane = threadIdx.x & 31;
  const int sl = lane & 15;
  const int c0 = sl * NV;
  const bool mask_is_x = mask == x && ml.pad == xl.pad && ml.ld == xl.ld;
  const uint32_t PH = (xl.H + 1) >> 1, PW = (xl.W + 1) >> 1;
  const int64_t nblk = (int64_t)xl.B * PH * PW;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t pbase = wid * 2; pbase < nblk; pbase += nw * 2) {  // warp-uniform trip count
    const int64_t blk = pbase + (lane >> 4);
    const bool ok = blk < nblk;
    int b = 0, i = 0, jj = 0;
    if (ok) {
      const uint32_t q = (uint32_t)blk, r = q / PW;
      jj = (int)(q - r * PW);
      b = (int)(r / PH);
      i = (int)(r - (uint32_t)b * PH);
    }
    float g[2][2][NV];
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
      for (int qq = 0; qq < 2; ++qq)
#pragma unroll
        for (int j = 0; j < NV; ++j) g[p][qq][j] = 0.f;
#pragma unroll
    for (int a = 0; a < NW; ++a) {
      const int ho = i - (NW - 1) + a;
#pragma unroll
      for (int bb = 0; bb < NW; ++bb) {
        const int wo = jj - (NW - 1) + bb;
        if (!ok || ho < 0 || ho >= yl.H || wo < 0 || wo >= yl.W) continue;
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          const int64_t yi = lidx(yl, b, ho, wo, c0 + 4 * v);
          const uchar4 a4 = *reinterpret_cast<const uchar4*>(arg + yi);
          const float4 gv = __ldg(reinterpret_cast<const float4*>(dy + yi));
#pragma unroll
          for (int p = 0; p < 2; ++p) {
            const int r = 2 * (NW - 1 - a) + p;
            if (r >= WIN) continue;
#pragma unroll
            for (int qq = 0; qq < 2; ++qq) {
              const int cc = 2 * (NW - 1 - bb) + qq;
              if (cc >= WIN) continue;
              const int local = r * WIN + cc;
              float* gg = &g[p][qq][4 * v];
              if (a4.x == local) gg[0] += gv.x;
              if (a4.y == local) gg[1] += gv.y;
              if (a4.z == local) gg[2] += gv.z;
              if (a4.w == local) gg[3] += gv.w;
            }
          }
        }
      }
    }
#pragma unroll
    for (int p = 0; p < 2; ++p) {
#pragma unroll
      for (int qq = 0; qq < 2; ++qq) {
        const int h = 2 * i + p, w = 2 * jj + qq;
        const bool pix = ok && h < xl.H && w < xl.W;
        float v[NV], o[NV];
#pragma unroll
        for (int t = 0; t < VPL; ++t) {
          float4 xa = make_float4(0.f, 0.f, 0.f, 0.f);
          if (pix) xa = *reinterpret_cast<const float4*>(x + lidx(xl, b, h, w, c0 + 4 * t));
          v[4 * t] = xa.x; v[4 * t + 1] = xa.y; v[4 * t + 2] = xa.z; v[4 * t + 3] = xa.w;
        }
        lrn_lane<VPL, true>(v, g[p][qq], sl, alpha, beta, k, o);  // every lane: shuffles
        if (!pix) continue;
#pragma unroll
        for (int t = 0; t < VPL; ++t) {
          float4 rr = make_float4(o[4 * t], o[4 * t + 1], o[4 * t + 2], o[4 * t + 3]);
          if (mask_is_x) {
            if (!(v[4 * t] > 0.f)) rr.x = 0.f;
            if (!(v[4 * t + 1] > 0.f)) rr.y = 0.f;
            if (!(v[4 * t + 2] > 0.f)) rr.z = 0.f;
            if (!(v[4 * t + 3] > 0.f)) rr.w = 0.f;
          } else if (mask) {
            const float4 m = *reinterpret_cast<const float4*>(mask + lidx(ml, b, h, w, c0 + 4 * t));
            if (!(m.x > 0.f)) rr.x = 0.f;
            if (!(m.y > 0.f)) rr.y = 0.f;
            if (!(m.z > 0.f)) rr.z = 0.f;
            if (!(m.w > 0.f)) rr.w = 0.f;
          }
          *reinterpret_cast<float4*>(out + lidx(ol, b, h, w, c0 + 4 * t)) = rr;
        }
      }
    }
  }
}

template <bool BWD>
bool launch_lrn_fast(const float* x, wap_layout_t xl, const float* dy, wap_layout_t dyl, int size, float alpha,
                     float beta, float bias, float* out, wap_layout_t ol, const float* mask, wap_layout_t ml,
                     cudaStream_t st) {
  const bool compact = xl.ld == xl.C && ol.ld == xl.C && (!BWD || dyl.ld == xl.C) && (!mask || ml.ld == xl.C);
  if (!compact) return false;
  const int64_t npix = (int64_t)xl.B * xl.H * xl.W;
  if (size == 5 && (xl.C == 64 || xl.C == 192)) {
    const int64_t warps = (npix + 1) / 2;
    int64_t blocks = (warps * 32 + 255) / 256;
    if (blocks > (int64_t)WAP_NUM_SMS * 16) blocks = (int64_t)WAP_NUM_SMS * 16;
    if (xl.C == 64 && !BWD) {
      const int64_t w2 = (npix + 3) / 4;  // two pixel pairs per warp iteration
      int64_t b2 = (w2 * 32 + 255) / 256;
      if (b2 > (int64_t)WAP_NUM_SMS * 8) b2 = (int64_t)WAP_NUM_SMS * 8;
      lrn_fwd_c64_kernel<2><<<(int)b2, 256, 0, st>>>(x, xl, alpha, beta, bias, out, ol);
    } else if (xl.C == 64)
      lrn_warp_kernel<1, BWD><<<(int)blocks, 256, 0, st>>>(x, xl, dy, dyl, alpha, beta, bias, out, ol, mask, ml);
    else
      lrn_warp_kernel<3, BWD><<<(int)blocks, 256, 0, st>>>(x, xl, dy, dyl, alpha, beta, bias, out, ol, mask, ml);
    return true;
  }
  auto blocks = [&](int pix) { return grid_for(npix, pix); };
  if (xl.C == 64) {
    lrn_fast_kernel<16, 32, BWD><<<blocks(32), 256, 0, st>>>(x, xl, dy, dyl, size, alpha, beta, bias, out, ol, mask, ml);
    return true;
  }
  if (xl.C == 192) {
    lrn_fast_kernel<48, 16, BWD><<<blocks(16), 256, 0, st>>>(x, xl, dy, dyl, size, alpha, beta, bias, out, ol, mask, ml);
    return true;
  }
  if (xl.C == 96) {
    lrn_fast_kernel<24, 16, BWD><<<blocks(16), 256, 0, st>>>(x, xl, dy, dyl, size, alpha, beta, bias, out, ol, mask, ml);
    return true;
  }
  return false;
}

// ---------------------------------------------------------------------------
// softmax cross-entropy (+ gradient): one block per row
// ---------------------------------------------------------------------------
__global__ void xent_row_kernel(const float* __restrict__ z, int64_t ldz, const float* __restrict__ y, int64_t ldy,
                                int cols, float inv_denom, float* __restrict__ dz, int64_t ldd,
                                float* __restrict__ row_loss) {
  __shared__ float red[32];
  const int r = blockIdx.x;
  const float* zr = z + r * ldz;
  const float* yr = y + r * ldy;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  float mx = -INFINITY;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) mx = fmaxf(mx, zr[c]);
  mx = warp_max(mx);
  if (lane == 0) red[wid] = mx;
  __syncthreads();
  if (wid == 0) {
    float v = lane < nw ? red[lane] : -INFINITY;
    v = warp_max(v);
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  mx = red[0];
  __syncthreads();
  float se = 0.f;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) se += expf(zr[c] - mx);
  se = warp_sum(se);
  if (lane == 0) red[wid] = se;
  __syncthreads();
  if (wid == 0) {
    float v = lane < nw ? red[lane] : 0.f;
    v = warp_sum(v);
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  se = red[0];
  __syncthreads();
  const float lse = logf(se);
  float l = 0.f;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    const float zc = zr[c] - mx;
    const float yc = yr[c];
    l -= yc * (zc - lse);
    dz[r * ldd + c] = (expf(zc) / se - yc) * inv_denom;
  }
  l = warp_sum(l);
  if (lane == 0) red[wid] = l;
  __syncthreads();
  if (threadIdx.x == 0) {
    float v = 0.f;
    for (int k2 = 0; k2 < nw; ++k2) v += red[k2];
    row_loss[r] = v;
  }
}

__global__ void xent_final_kernel(const float* __restrict__ row_loss, int rows, float* __restrict__ loss) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int r = 0; r < rows; ++r) s += row_loss[r];
    loss[0] = (float)(s / rows);
  }
}

// dense [B,H,W,C] (any C) <-> layout; dir 0 = pack dense->layout, 1 = unpack layout->dense
__global__ void pack_kernel(const float* __restrict__ src, float* __restrict__ dst, wap_layout_t l, int dir) {
  const int64_t total = (int64_t)l.B * l.H * l.W * l.C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % l.C);
    int64_t q = i / l.C;
    const int w = (int)(q % l.W);
    q /= l.W;
    const int h = (int)(q % l.H);
    const int b = (int)(q / l.H);
    const int64_t j = lidx(l, b, h, w, c);
    if (dir == 0) dst[j] = src[i];
    else dst[i] = src[j];
  }
}

// Image upload path (dense NHWC C=3 -> ld=4 layout): blockIdx.y = image row, one
// pixel per thread: a warp reads 384 contiguous bytes (3 coalesced 4-byte loads per
// lane) and writes 512 contiguous bytes (one float4 per lane, padding lane 0).
// No per-pixel index division.
__global__ void __launch_bounds__(256) pack_c3_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                                       wap_layout_t l) {
  for (int row = blockIdx.y; row < l.B * l.H; row += gridDim.y) {
    const int b = row / l.H, h = row - (row / l.H) * l.H;
    const float* s = src + (int64_t)row * l.W * 3;
    float4* d = reinterpret_cast<float4*>(dst + lidx(l, b, h, 0, 0));
    for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < l.W; w += gridDim.x * blockDim.x)
      d[w] = make_float4(__ldg(s + 3 * w), __ldg(s + 3 * w + 1), __ldg(s + 3 * w + 2), 0.f);
  }
}

__global__ void sgd_kernel(const float* __restrict__ w, const float* __restrict__ g, float lr, float* __restrict__ o,
                           int64_t n) {
  const int64_t n4 = n / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 a = reinterpret_cast<const float4*>(w)[i];
    const float4 b = reinterpret_cast<const float4*>(g)[i];
    reinterpret_cast<float4*>(o)[i] = make_float4(a.x - lr * b.x, a.y - lr * b.y, a.z - lr * b.z, a.w - lr * b.w);
  }
  for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    o[i] = w[i] - lr * g[i];
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
#define STREAM(s) reinterpret_cast<cudaStream_t>(s)

extern "C" int wap_elementwise(int op, const float* x, wap_layout_t xl, const float* aux, wap_layout_t al,
                               const float* bias, float* y, wap_layout_t yl, void* stream) {
  int rc;
  if ((rc = check_layout(xl, "x")) || (rc = check_layout(yl, "y"))) return rc;
  WAP_CHECK_ARG(x && y, "null pointer");
  WAP_CHECK_ARG(xl.B == yl.B && xl.H == yl.H && xl.W == yl.W && xl.C == yl.C, "elementwise: shape mismatch");
  if (op == 3) {
    if ((rc = check_layout(al, "aux"))) return rc;
    WAP_CHECK_ARG(aux != nullptr, "GradReLU needs the activation operand");
  }
  if (op == 0 || op == 2) WAP_CHECK_ARG(bias != nullptr, "BiasAdd needs a bias");
  const int threads = 256;
  const int64_t work = (int64_t)yl.B * yl.H * yl.W * (yl.ld / 4);
  const int blocks = grid_for(work, threads);
  switch (op) {
    case 0: elementwise_kernel<0><<<blocks, threads, 0, STREAM(stream)>>>(x, xl, aux, al, bias, y, yl); break;
    case 1: elementwise_kernel<1><<<blocks, threads, 0, STREAM(stream)>>>(x, xl, aux, al, bias, y, yl); break;
    case 2: elementwise_kernel<2><<<blocks, threads, 0, STREAM(stream)>>>(x, xl, aux, al, bias, y, yl); break;
    case 3: elementwise_kernel<3><<<blocks, threads, 0, STREAM(stream)>>>(x, xl, aux, al, bias, y, yl); break;
    case 4: elementwise_kernel<4><<<blocks, threads, 0, STREAM(stream)>>>(x, xl, aux, al, bias, y, yl); break;
    default: WAP_CHECK_ARG(false, "unknown elementwise op %d", op);
  }
  WAP_LAUNCH_CHECK();
  COUNT_LAUNCH();
  return WAP_OK;
}

extern "C" int wap_add_n(const float* const* xs, int n, wap_layout_t l, float* y, void* stream) {
  int rc;
  if ((rc = check_layout(l, "x"))) return rc;
  WAP_CHECK_ARG(n >= 1 && n <= 16, "add_n supports 1..16 operands, got %d", n);
  PtrPack pk;
  for (int i = 0; i < n; ++i) {
    WAP_CHECK_ARG(xs[i] != nullptr, "null operand %d", i);
    pk.p[i] = xs[i];
  }
  const int64_t n4 = (int64_t)l.B * (l.H + l.pad) * (l.W + l.pad) * l.ld / 4;
  add_n_kernel_packed<<<grid_for(n4, 256), 256, 0, STREAM(stream)>>>(pk, n, y, n4);
  WAP_LAUNCH_CHECK();
  COUNT_LAUNCH();
  return WAP_OK;
}

extern "C" int64_t wap_bias_grad_work_floats(wap_layout_t l) { return (int64_t)bias_chunks(l) * l.ld; }

extern "C" int wap_bias_grad(const float* dy, wap_layout_t l, float* db, float* work, void* stream) {
  int rc;
  if ((rc = check_layout(l, "dy"))) return rc;
  WAP_CHECK_ARG(dy && db && work, "null pointer");
  const int64_t rows = (int64_t)l.B * (l.H + l.pad) * (l.W + l.pad);
  const int chunks = bias_chunks(l);
  const int64_t rpc = (rows + chunks - 1) / chunks;
  const int cw = bias_cw(l);
  dim3 grid((l.ld / 4 + cw - 1) / cw, chunks);
  bias_grad_partial<<<grid, 256, 0, STREAM(stream)>>>(dy, rows, l.ld, l.C, rpc, cw, work);
  WAP_LAUNCH_CHECK();
  bias_grad_final<<<(l.C + 3) / 4, 128, 0, STREAM(stream)>>>(work, chunks, l.ld, l.C, db);
  WAP_LAUNCH_CHECK();
  g_wap_launches.fetch_add(2, std::memory_order_relaxed);
  return WAP_OK;
}

// ---------------------------------------------------------------------------
// Direct first-layer weight gradient (GradConv2DW, interp.py:82-91) for a 3x3 stride-1
// conv over a <= 4-channel input (one float4 per pixel): dW[(u,v,c), co] =
// sum_{b,h,w} x[b, h+u-p, w+v-p, c] * dy[b, h, w, co]. As a GEMM it is M = 27 rows
// (4.7 of a 128-row tile busy) over K = B*H*W; here each block owns R image rows of one
// image: the input rows it needs are staged once in shared memory (zero outside the
// image), thread (co, g) accumulates the 27 sums of output channel co over every 4th
// pixel g of the band in fp32 FMAs, the 4 pixel groups are summed in a fixed order, and
// the block writes its [27 x Co] partial; wgrad_direct_final sums the partials in block
// order (deterministic).
// ---------------------------------------------------------------------------
constexpr int kWgdRows = 4;  // image rows per block
__global__ void __launch_bounds__(256) wgrad_direct_3x3_kernel(const float* __restrict__ x, wap_layout_t xl,
                                                               const float* __restrict__ dy, wap_layout_t dl,
                                                               int p, float* __restrict__ part) {
  extern __shared__ float4 xs[];  // (kWgdRows + 2) rows x (W + 2) pixels
  const int Co = dl.C;
  const int W2 = xl.W + 2;
  const int bands = (dl.H + kWgdRows - 1) / kWgdRows;
  const int b = blockIdx.x / bands;
  const int h0 = (blockIdx.x - b * bands) * kWgdRows;
  const int nr = min(kWgdRows, dl.H - h0);
  for (int i = threadIdx.x; i < (nr + 2) * W2; i += blockDim.x) {
    const int r = i / W2, c = i - r * W2;
    const int h = h0 + r - p, w = c - p;  // input pixel of padded column c, row r
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (h >= 0 && h < xl.H && w >= 0 && w < xl.W) v = *reinterpret_cast<const float4*>(x + lidx(xl, b, h, w, 0));
    xs[i] = v;
  }
  __syncthreads();
  // thread = (output channel co, pixel group g); Co <= 64 channels per pass
  const int g = threadIdx.x >> 6;
  const int co = threadIdx.x & 63;
  for (int cbase = 0; cbase < Co; cbase += 64) {
    const int cc = cbase + co;
    float acc[27];
#pragma unroll
    for (int j = 0; j < 27; ++j) acc[j] = 0.f;
    if (cc < Co) {
      // pixels w = g, g + 4, ... of each row; the dy loads of 4 pixels are issued together
      // (one round trip per 4 pixels instead of one per pixel)
      for (int r = 0; r < nr; ++r) {
        const float* dyr = dy + lidx(dl, b, h0 + r, 0, cc);
        const float4* xr = xs + r * W2;
        for (int w0 = g; w0 < dl.W; w0 += 16) {
          float d[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) d[i] = (w0 + 4 * i < dl.W) ? __ldg(dyr + (int64_t)(w0 + 4 * i) * dl.ld) : 0.f;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int w = min(w0 + 4 * i, dl.W - 1);  // d = 0 past the row end
#pragma unroll
            for (int u = 0; u < 3; ++u) {
#pragma unroll
              for (int v = 0; v < 3; ++v) {
                const float4 xv = xr[u * W2 + w + v];
                acc[(u * 3 + v) * 3 + 0] = fmaf(xv.x, d[i], acc[(u * 3 + v) * 3 + 0]);
                acc[(u * 3 + v) * 3 + 1] = fmaf(xv.y, d[i], acc[(u * 3 + v) * 3 + 1]);
                acc[(u * 3 + v) * 3 + 2] = fmaf(xv.z, d[i], acc[(u * 3 + v) * 3 + 2]);
              }
            }
          }
        }
      }
    }
    // sum the 4 pixel groups in order through shared memory (after the staged rows)
    float* red = reinterpret_cast<float*>(xs + (kWgdRows + 2) * W2);  // [4][27][64]
#pragma unroll
    for (int j = 0; j < 27; ++j) red[(g * 27 + j) * 64 + co] = acc[j];
    __syncthreads();
    if (g == 0 && cc < Co) {
#pragma unroll
      for (int j = 0; j < 27; ++j) {
        const float t = ((red[j * 64 + co] + red[(27 + j) * 64 + co]) + red[(54 + j) * 64 + co]) +
                        red[(81 + j) * 64 + co];
        part[((int64_t)blockIdx.x * 27 + j) * Co + cc] = t;
      }
    }
    __syncthreads();
  }
}

// dw[j, co] = sum over blocks (in block order) of part[blk, j, co]; one warp per (j, co)
// run of 32 channels, lanes striding the blocks, fixed shuffle tree (deterministic)
__global__ void wgrad_direct_final_kernel(const float* __restrict__ part, int nblk, int Co, float* __restrict__ dw,
                                          int ldw) {
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= 27 * Co) return;
  const int j = wid / Co, co = wid - j * Co;
  float s = 0.f;
  for (int k = lane; k < nblk; k += 32) s += part[((int64_t)k * 27 + j) * Co + co];
  s = warp_sum(s);
  if (lane == 0) dw[(int64_t)j * ldw + co] = s;
}

extern "C" int64_t wap_conv_wgrad_direct_work_floats(wap_layout_t dyl) {
  const int bands = (dyl.H + kWgdRows - 1) / kWgdRows;
  return (int64_t)dyl.B * bands * 27 * dyl.C;
}

extern "C" int wap_conv_wgrad_direct(const float* x, wap_layout_t xl, const float* dy, wap_layout_t dyl, int k,
                                     int padding, float* dw, int ldw, float* work, void* stream) {
  int rc;
  if ((rc = check_layout(xl, "x")) || (rc = check_layout(dyl, "dy"))) return rc;
  WAP_CHECK_ARG(x && dy && dw && work, "conv_wgrad_direct: null pointer");
  WAP_CHECK_ARG(k == 3 && padding == 1, "conv_wgrad_direct: 3x3 'same' convs only");
  WAP_CHECK_ARG(xl.ld == 4 && xl.C == 3, "conv_wgrad_direct: input must be one float4 per pixel, 3 channels");
  WAP_CHECK_ARG(dyl.H == xl.H && dyl.W == xl.W && dyl.B == xl.B && ldw >= dyl.C,
                "conv_wgrad_direct: shape mismatch");
  const int bands = (dyl.H + kWgdRows - 1) / kWgdRows;
  const int64_t nblk = (int64_t)dyl.B * bands;
  WAP_CHECK_ARG(nblk < (1LL << 31), "conv_wgrad_direct: too many blocks");
  const size_t smem = (size_t)(kWgdRows + 2) * (xl.W + 2) * 16 + (size_t)4 * 27 * 64 * 4;
  WAP_CHECK_ARG(smem <= 96 * 1024, "conv_wgrad_direct: image too wide");
  static bool attr = false;
  if (!attr) {
    WAP_CUDA_TRY(cudaFuncSetAttribute(wgrad_direct_3x3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
    attr = true;
  }
  wgrad_direct_3x3_kernel<<<(unsigned)nblk, 256, smem, STREAM(stream)>>>(x, xl, dy, dyl, padding, work);
  WAP_LAUNCH_CHECK();
  const int warps = 27 * dyl.C;
  wgrad_direct_final_kernel<<<(warps * 32 + 255) / 256, 256, 0, STREAM(stream)>>>(work, (int)nblk, dyl.C, dw, ldw);
  WAP_LAUNCH_CHECK();
  g_wap_launches.fetch_add(2, std::memory_order_relaxed);
  return WAP_OK;
}

extern "C" int wap_conv_direct(const float* x, wap_layout_t xl, const float* w, int k, int padding, int ldw,
                               const float* bias, int relu, float* y, wap_layout_t yl, uint32_t* mbits,
                               int64_t mbits_ld, void* stream) {
  int rc;
  if ((rc = check_layout(xl, "x")) || (rc = check_layout(yl, "y"))) return rc;
  WAP_CHECK_ARG(x && w && y && k >= 1 && padding >= 0, "conv_direct: bad arguments");
  WAP_CHECK_ARG(xl.ld == 4 && xl.C <= 4, "conv_direct: input must be one float4 per pixel (C <= 4)");
  WAP_CHECK_ARG(yl.C % 32 == 0 && yl.ld % 4 == 0 && ldw >= yl.C, "conv_direct: Co must be a multiple of 32");
  WAP_CHECK_ARG(yl.H == xl.H + 2 * padding - k + 1 && yl.W == xl.W + 2 * padding - k + 1 && yl.B == xl.B,
                "conv_direct: output shape mismatch (stride-1 conv)");
  const int64_t npix = (int64_t)yl.B * yl.H * yl.W;
  WAP_CHECK_ARG(npix < (1LL << 31), "conv_direct: too many pixels");
  const int smem = (k * k * xl.C + 1) * 32 * 4;
  WAP_CHECK_ARG(smem <= 48 * 1024, "conv_direct: filter too large");
  int64_t bx = (npix + 255) / 256;
  if (bx > (int64_t)WAP_NUM_SMS * 16) bx = (int64_t)WAP_NUM_SMS * 16;
  const dim3 grid((unsigned)bx, (unsigned)(yl.C / 32));
  if (k == 3 && xl.C == 3 && !getenv("WAP_CONV_DIRECT_PX1")) {
    int64_t b2 = ((int64_t)yl.B * yl.H * ((yl.W + 1) / 2) + 255) / 256;
    if (b2 > (int64_t)WAP_NUM_SMS * 16) b2 = (int64_t)WAP_NUM_SMS * 16;
    conv_direct_3x3c3_px2_kernel<<<dim3((unsigned)b2, (unsigned)(yl.C / 32)), 256, smem, STREAM(stream)>>>(
        x, xl, w, padding, ldw, bias, relu, y, yl, mbits, mbits_ld);
  } else if (k == 3 && xl.C == 3)
    conv_direct_kernel<3, 3><<<grid, 256, smem, STREAM(stream)>>>(x, xl, w, k, padding, ldw, bias, relu, y, yl, mbits,
                                                                mbits_ld);
  else
    conv_direct_kernel<0, 0><<<grid, 256, smem, STREAM(stream)>>>(x, xl, w, k, padding, ldw, bias, relu, y, yl, mbits,
                                                                mbits_ld);
  WAP_LAUNCH_CHECK();
  COUNT_LAUNCH();
  return WAP_OK;
}

extern "C" int wap_s2d_input(const float* x, wap_layout_t xl, int stride, int padding, int Hs, int Ws, float* xs,
                             int ldc, void* stream) {
  int rc;
  if ((rc = check_layout(xl, "x"))) return rc;
  WAP_CHECK_ARG(x && xs && stride >= 1 && padding >= 0 && Hs >= 1 && Ws >= 1, "s2d: bad arguments");
  WAP_CHECK_ARG(ldc % 4 == 0 && ldc >= stride * stride * xl.C, "s2d: ldc must cover s*s*C and be a multiple of 4");
  const int64_t total4 = (int64_t)xl.B * Hs * Ws * (ldc / 4);
  WAP_CHECK_ARG(total4 < (1LL << 31), "s2d: grid too large for 32-bit indexing");
  int64_t blocks = (total4 + 255) / 256;
  if (blocks > (int64_t)WAP_NUM_SMS * 32) blocks = (int64_t)WAP_NUM_SMS * 32;
  if (stride == 4 && xl.C == 3 && xl.ld == 4) {
    s2d_input_const_kernel<4, 3><<<(int)blocks, 256, 0, STREAM(stream)>>>(x, xl, padding, Hs, Ws, xs, ldc);
  } else if (xl.ld == 4 && xl.C <= 4) {
    const int ss = stride * stride;
    const int64_t per = ldc / xl.C > ss ? (ldc + xl.C - 1) / xl.C : ss;
    const int64_t total = (int64_t)xl.B * Hs * Ws * per;
    WAP_CHECK_ARG(total < (1LL << 31), "s2d: grid too large for 32-bit indexing");
    int64_t nb = (total + 255) / 256;
    if (nb > (int64_t)WAP_NUM_SMS * 32) nb = (int64_t)WAP_NUM_SMS * 32;
    s2d_input_px4_kernel<<<(int)nb, 256, 0, STREAM(stream)>>>(x, xl, stride, padding, Hs, Ws, xs, ldc);
  } else {
    s2d_input_kernel<<<(int)blocks, 256, 0, STREAM(stream)>>>(x, xl, stride, padding, Hs, Ws, xs, ldc);
  }
  WAP_LAUNCH_CHECK();
  COUNT_LAUNCH();
  return WAP_OK;
}

extern "C" int wap_s2d_weight(const float* w, float* ws, int k, int C, int Co, int ldw, int stride, int ldc,
                              int ldws, int fold_grad, void* stream) {
  WAP_CHECK_ARG(w && ws && k >= 1 && C >= 1 && Co >= 1 && stride >= 1, "s2d weight: bad arguments");
  WAP_CHECK_ARG(ldw >= Co && ldws >= Co && ldc >= stride * stride * C, "s2d weight: bad strides");
  const int ks = (k + stride - 1) / stride;
  const int64_t rows = fold_grad ? (int64_t)k * k * C : (int64_t)ks * ks * ldc;
  s2d_weight_kernel<<<grid_for(rows * Co, 256), 256, 0, STREAM(stream)>>>(w, ws, k, C, Co, ldw, stride, ks, ldc, ldws,
                                                                          fold_grad);
  WAP_LAUNCH_CHECK();
  COUNT_LAUNCH();
  return WAP_OK;
}

extern "C" int wap_im2col(const float* x, wap_layout_t xl, int k, int stride, int padding, int Ho, int Wo,
                          int out_pad, float* col, int64_t ldcol, void* stream) {
  int rc;
  if ((rc = check_layout(xl, "x"))) return rc;
  WAP_CHECK_ARG(k >= 1 && stride >= 1 && padding >= 0 && Ho >= 1 && Wo >= 1 && out_pad >= 0, "im2col: bad geometry");
  WAP_CHECK_ARG(ldcol >= (int64_t)k * k * xl.C, "im2col: ldcol too small");
  const int64_t M = (int64_t)xl.B * (Ho + out_pad) * (Wo + out_pad);
  const int64_t total = M * ldcol;
  if ((int64_t)k * k * xl.C <= IM2COL_MAXK) {
    int64_t blocks = (M + IM2COL_ROWS - 1) / IM2COL_ROWS;
    if (blocks > WAP_NUM_SMS * 32) blocks = WAP_NUM_SMS * 32;
    im2col_table_kernel<<<(int)blocks, 256, 0, STREAM(stream)>>>(x, xl, k, stride, padding, Ho, Wo, out_pad, col,
                                                                ldcol, M);
  } else {
    im2col_kernel<<<grid_for(total, 256), 256, 0, STREAM(stream)>>>(x, xl, k, stride, padding, Ho, Wo, out_pad, col,
                                                                   ldcol);
  }
  WAP_LAUNCH_CHECK();
  COUNT_LAUNCH();
  return WAP_OK;
}

extern "C" int wap_col2im(const float* dcol, int64_t ldcol, int k, int stride, int padding, int Ho, int Wo,
                          int out_pad, float* dx, wap_layout_t dxl, const float* mask, wap_layout_t ml,
                          void* stream) {
  int rc;
  if ((rc = check_layout(dxl, "dx"))) return rc;
  if (mask && (rc = check_layout(ml, "mask"))) return rc;
  WAP_CHECK_ARG(ldcol >= (int64_t)k * k * dxl.C, "col2im: ldcol too small");
  const int64_t total = (int64_t)dxl.B * dxl.H * dxl.W * dxl.ld;
  col2im_kernel<<<grid_for(total, 256), 256, 0, STREAM(stream)>>>(dcol, ldcol, k, stride, padding, Ho, Wo, out_pad,
                                                                 dx, dxl, mask, ml);
  WAP_LAUNCH_CHECK();
  COUNT_LAUNCH();
  return WAP_OK;
}

extern "C" int wap_maxpool_fwd(const float* x, wap_layout_t xl, int window, int stride, float* y, wap_layout_t yl,
                               uint8_t* argmax, void* stream) {
  return wap_maxpool_fwd_ex(x, xl, window, stride, y, yl, argmax, 0, stream);
}

extern "C" int wap_maxpool_fwd_ex(const float* x, wap_layout_t xl, int window, int stride, float* y, wap_layout_t yl,
                                  uint8_t* argmax, int flags, void* stream) {
  int rc;
  if ((rc = check_layout(xl, "x")) || (rc = check_layout(yl, "y"))) return rc;
  WAP_CHECK_ARG(window >= 1 && window <= 15 && stride >= 1, "maxpool: bad window/stride");
  WAP_CHECK_ARG(yl.H == (xl.H - window) / stride + 1 && yl.W == (xl.W - window) / stride + 1 && yl.C == xl.C &&
                    yl.B == xl.B && xl.ld == yl.ld,
                "maxpool: output layout does not match");
  WAP_CHECK_ARG((int64_t)yl.B * yl.H < 65536 * 1024LL, "maxpool: too many rows");
  const int per = yl.W * (yl.ld / 4);
  maxpool_fwd_kernel<<<pool_grid(yl.B * yl.H, per), 256, 0, STREAM(stream)>>>(
      x, xl, window, stride, y, yl, argmax, (flags & WAP_POOL_RELU_FUSED) ? 1 : 0);
  WAP_LAUNCH_CHECK();
  COUNT_LAUNCH();
  return WAP_OK;
}

extern "C" int wap_maxpool_bwd(const uint8_t* argmax, const float* dy, wap_layout_t dyl, int window, int stride,
                               float* dx, wap_layout_t dxl, const float* mask, wap_layout_t ml, void* stream) {
  int rc;
  if ((rc = check_layout(dyl, "dy")) || (rc = check_layout(dxl, "dx"))) return rc;
  if (mask && (rc = check_layout(ml, "mask"))) return rc;
  WAP_CHECK_ARG(argmax != nullptr, "maxpool backward needs the forward argmax");
  WAP_CHECK_ARG(dxl.ld == dyl.ld, "maxpool: dx/dy ld mismatch");
  const int per = dxl.W * (dxl.ld / 4);
  const dim3 grid = pool_grid(dxl.B * dxl.H, per);
  const bool pixel_form = getenv("WAP_POOL_BWD_PIXEL") != nullptr;  // A/B switch: per-pixel gather
  if (stride == 2 && (window == 3 || window == 2) && !pixel_form) {
    const dim3 g2 = pool_grid(dxl.B * ((dxl.H + 1) / 2), ((dxl.W + 1) / 2) * (dxl.ld / 4));
    if (window == 3)
      maxpool_bwd_s2_kernel<3><<<g2, 256, 0, STREAM(stream)>>>(argmax, dy, dyl, dx, dxl, mask, ml);
    else
      maxpool_bwd_s2_kernel<2><<<g2, 256, 0, STREAM(stream)>>>(argmax, dy, dyl, dx, dxl, mask, ml);
  } else if (window == 3 && stride == 2)
    maxpool_bwd_kernel<3, 2><<<grid, 256, 0, STREAM(stream)>>>(argmax, dy, dyl, window, stride, dx, dxl, mask, ml);
  else if (window == 2 && stride == 2)
    maxpool_bwd_kernel<2, 2><<<grid, 256, 0, STREAM(stream)>>>(argmax, dy, dyl, window, stride, dx, dxl, mask, ml);
  else
    maxpool_bwd_kernel<0, 0><<<grid, 256, 0, STREAM(stream)>>>(argmax, dy, dyl, window, stride, dx, dxl, mask, ml);
  WAP_LAUNCH_CHECK();
  COUNT_LAUNCH();
  return WAP_OK;
}

extern "C" int wap_lrn_maxpool_fwd(const float* x, wap_layout_t xl, int size, float alpha, float beta, float bias,
                                   int window, int stride, float* y, wap_layout_t yl, uint8_t* argmax,
                                   void* stream) {
  int rc;
  if ((rc = check_layout(xl, "x")) || (rc = check_layout(yl, "y"))) return rc;
  WAP_CHECK_ARG(size == 5 && (window == 2 || window == 3) && stride >= 1,
                "fused lrn+maxpool forward: LRN size 5, window 2/3 only");
  WAP_CHECK_ARG(xl.C == 64 || xl.C == 192, "fused lrn+maxpool forward: C must be 64 or 192");
  WAP_CHECK_ARG(xl.ld == xl.C && yl.ld == xl.C, "fused lrn+maxpool forward: compact channel layouts only");
  WAP_CHECK_ARG(yl.H == (xl.H - window) / stride + 1 && yl.W == (xl.W - window) / stride + 1 && yl.C == xl.C &&
                    yl.B == xl.B,
                "fused lrn+maxpool forward: output layout does not match");
  const int64_t nout = (int64_t)yl.B * yl.H * yl.W;
  WAP_CHECK_ARG(nout < (1LL << 31), "fused lrn+maxpool forward: too many pixels");
  int64_t blocks = ((nout + 1) / 2 * 32 + 255) / 256;
  if (blocks > (int64_t)WAP_NUM_SMS * 16) blocks = (int64_t)WAP_NUM_SMS * 16;
  cudaStream_t st = STREAM(stream);
  // row bands (each input LRN computed ~once) when a band of R >= 1 pooled rows fits in
  // <= 72 KB of shared memory (3 blocks per SM). Opt-in (WAP_LRN_POOL_BAND=1): measured r02,
  // AlexNet pool1 0.070 -> 0.084 ms (two serial phases per block, 4 waves), pool2 0.045 ->
  // 0.043 ms; bitwise equal to the per-output form (tests/test_ops_gpu.py)
  static const bool band_on = getenv("WAP_LRN_POOL_BAND") && atoi(getenv("WAP_LRN_POOL_BAND")) != 0;
  int R = 0;
  for (int r = 4; r >= 1 && band_on; --r) {
    const int rows = std::min((r - 1) * stride + window, xl.H);
    if ((int64_t)rows * xl.W * xl.C * 4 <= 72 * 1024) { R = r; break; }
  }
  if (R > 0) {
    const int bands = (yl.H + R - 1) / R;
    const int rows = std::min((R - 1) * stride + window, xl.H);
    const size_t smem = (size_t)rows * xl.W * xl.C * 4;
#define WAP_LRNMPB(WIN, VPL)                                                                                  \
  do {                                                                                                        \
    static bool attr = false;                                                                                 \
    if (!attr) {                                                                                              \
      WAP_CUDA_TRY(cudaFuncSetAttribute(lrn_maxpool_band_kernel<WIN, VPL>,                                    \
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, 72 * 1024));             \
      attr = true;                                                                                            \
    }                                                                                                         \
    lrn_maxpool_band_kernel<WIN, VPL><<<yl.B * bands, 256, smem, st>>>(x, xl, alpha, beta, bias, stride, R, y, \
                                                                       yl, argmax);                          \
  } while (0)
    if (window == 3) {
      if (xl.C == 64) WAP_LRNMPB(3, 1); else WAP_LRNMPB(3, 3);
    } else {
      if (xl.C == 64) WAP_LRNMPB(2, 1); else WAP_LRNMPB(2, 3);
    }
#undef WAP_LRNMPB
    WAP_LAUNCH_CHECK();
    COUNT_LAUNCH();
    return WAP_OK;
  }
#define WAP_LRNMP(WIN, VPL) \
  lrn_maxpool_fwd_kernel<WIN, VPL><<<(int)blocks, 256, 0, st>>>(x, xl, alpha, beta, bias, stride, y, yl, argmax)
  if (window == 3) {
    if (xl.C == 64) WAP_LRNMP(3, 1); else WAP_LRNMP(3, 3);
  } else {
    if (xl.C == 64) WAP_LRNMP(2, 1); else WAP_LRNMP(2, 3);
  }
#undef WAP_LRNMP
  WAP_LAUNCH_CHECK();
  COUNT_LAUNCH();
  return WAP_OK;
}

extern "C" int wap_maxpool_lrn_bwd(const uint8_t* argmax, const float* dy, wap_layout_t dyl, int window,
                                   int stride, const float* x, wap_layout_t xl, int size, float alpha, float beta,
                                   float bias, float* dx, wap_layout_t dxl, const float* mask, wap_layout_t ml,
                                   void* stream) {
  int rc;
  if ((rc = check_layout(dyl, "dy")) || (rc = check_layout(xl, "x")) || (rc = check_layout(dxl, "dx"))) return rc;
  if (mask && (rc = check_layout(ml, "mask"))) return rc;
  WAP_CHECK_ARG(argmax != nullptr, "maxpool backward needs the forward argmax");
  WAP_CHECK_ARG(stride == 2 && (window == 2 || window == 3) && size == 5,
                "fused maxpool+lrn backward: stride 2, window 2/3, LRN size 5 only");
  WAP_CHECK_ARG(xl.C == 64 || xl.C == 192, "fused maxpool+lrn backward: C must be 64 or 192");
  WAP_CHECK_ARG(xl.ld == xl.C && dxl.ld == xl.C && dyl.ld == xl.C && (!mask || ml.ld == xl.C),
                "fused maxpool+lrn backward: compact channel layouts only");
  WAP_CHECK_ARG(dyl.H == (xl.H - window) / 2 + 1 && dyl.W == (xl.W - window) / 2 + 1 && dyl.B == xl.B &&
                    dxl.H == xl.H && dxl.W == xl.W && dxl.B == xl.B && dxl.C == xl.C,
                "fused maxpool+lrn backward: layouts do not match");
  const int64_t nblk = (int64_t)xl.B * ((xl.H + 1) / 2) * ((xl.W + 1) / 2);
  WAP_CHECK_ARG(nblk < (1LL << 31), "fused maxpool+lrn backward: too many pixels");
  int64_t blocks = ((nblk + 1) / 2 * 32 + 255) / 256;
  if (blocks > (int64_t)WAP_NUM_SMS * 16) blocks = (int64_t)WAP_NUM_SMS * 16;
  cudaStream_t st = STREAM(stream);
#define WAP_MPLRN(WIN, VPL)                                                                                    \
  maxpool_lrn_bwd_kernel<WIN, VPL><<<(int)blocks, 256, 0, st>>>(argmax, dy, dyl, x, xl, alpha, beta, bias, dx, \
                                                                  dxl, mask, ml)
  if (window == 3) {
    if (xl.C == 64) WAP_MPLRN(3, 1); else WAP_MPLRN(3, 3);
  } else {
    if (xl.C == 64) WAP_MPLRN(2, 1); else WAP_MPLRN(2, 3);
  }
#undef WAP_MPLRN
  WAP_LAUNCH_CHECK();
  COUNT_LAUNCH();
  return WAP_OK;
}

extern "C" int wap_lrn_fwd(const float* x, wap_layout_t xl, int size, float alpha, float beta, float bias, float* y,
                           wap_layout_t yl, void* stream) {
  int rc;
  if ((rc = check_layout(xl, "x")) || (rc = check_layout(yl, "y"))) return rc;
  WAP_CHECK_ARG(size >= 1 && size % 2 == 1, "LRN size must be odd");
  const int64_t npix = (int64_t)xl.B * xl.H * xl.W;
  WAP_CHECK_ARG(npix < (1LL << 31), "LRN: pixel count must stay below 2^31");
  const int smem = LRN_PIX * xl.C * 4;
  if (!launch_lrn_fast<false>(x, xl, nullptr, xl, size, alpha, beta, bias, y, yl, nullptr, xl, STREAM(stream)))
    lrn_fwd_kernel<<<grid_for(npix, LRN_PIX), 256, smem, STREAM(stream)>>>(x, xl, size, alpha, beta, bias, y, yl);
  WAP_LAUNCH_CHECK();
  COUNT_LAUNCH();
  return WAP_OK;
}

extern "C" int wap_lrn_bwd(const float* x, wap_layout_t xl, const float* dy, wap_layout_t dyl, int size, float alpha,
                           float beta, float bias, float* dx, wap_layout_t dxl, const float* mask, wap_layout_t ml,
                           void* stream) {
  int rc;
  if ((rc = check_layout(xl, "x")) || (rc = check_layout(dyl, "dy")) || (rc = check_layout(dxl, "dx"))) return rc;
  if (mask && (rc = check_layout(ml, "mask"))) return rc;
  const int64_t npix = (int64_t)xl.B * xl.H * xl.W;
  WAP_CHECK_ARG(npix < (1LL << 31), "LRN: pixel count must stay below 2^31");
  const int smem = 4 * LRN_PIX * xl.C * 4;
  if (!launch_lrn_fast<true>(x, xl, dy, dyl, size, alpha, beta, bias, dx, dxl, mask, ml, STREAM(stream)))
    lrn_bwd_kernel<<<grid_for(npix, LRN_PIX), 256, smem, STREAM(stream)>>>(x, xl, dy, dyl, size, alpha, beta, bias,
                                                                           dx, dxl, mask, ml);
  WAP_LAUNCH_CHECK();
  COUNT_LAUNCH();
  return WAP_OK;
}

extern "C" int wap_xent_fwd_bwd(const float* logits, int64_t ldz, const float* labels, int64_t ldy, int rows,
                                int cols, float denominator, float* loss, float* dlogits, int64_t ldd, float* work,
                                void* stream) {
  WAP_CHECK_ARG(logits && labels && loss && dlogits && work, "null pointer");
  WAP_CHECK_ARG(rows >= 1 && cols >= 1 && denominator >= 1.f, "xent: bad shape/denominator");
  xent_row_kernel<<<rows, 256, 0, STREAM(stream)>>>(logits, ldz, labels, ldy, cols, 1.f / denominator, dlogits, ldd,
                                                    work);
  WAP_LAUNCH_CHECK();
  xent_final_kernel<<<1, 32, 0, STREAM(stream)>>>(work, rows, loss);
  WAP_LAUNCH_CHECK();
  g_wap_launches.fetch_add(2, std::memory_order_relaxed);
  return WAP_OK;
}

extern "C" int wap_pack(const float* dense, wap_layout_t l, float* dst, int unpack, void* stream) {
  WAP_CHECK_ARG(dense && dst, "pack: null pointer");
  WAP_CHECK_ARG(l.B >= 1 && l.H >= 1 && l.W >= 1 && l.C >= 1 && l.ld >= l.C && l.pad >= 0, "pack: bad layout");
  const int64_t total = (int64_t)l.B * l.H * l.W * l.C;
  if (unpack) pack_kernel<<<grid_for(total, 256), 256, 0, STREAM(stream)>>>(dst, const_cast<float*>(dense), l, 1);
  else if (l.C == 3 && l.ld == 4 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0)
    pack_c3_kernel<<<dim3((unsigned)((l.W + 255) / 256), (unsigned)std::min(l.B * l.H, 65535)), 256, 0,
                     STREAM(stream)>>>(dense, dst, l);
  else pack_kernel<<<grid_for(total, 256), 256, 0, STREAM(stream)>>>(dense, dst, l, 0);
  WAP_LAUNCH_CHECK();
  COUNT_LAUNCH();
  return WAP_OK;
}

extern "C" int wap_sgd(const float* w, const float* g, float lr, float* w_out, int64_t n, void* stream) {
  WAP_CHECK_ARG(w && g && w_out && n >= 0, "sgd: bad arguments");
  WAP_CHECK_ARG(((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(w_out)) & 15) == 0,
                "sgd: buffers must be 16-byte aligned");
  if (n == 0) return WAP_OK;
  sgd_kernel<<<grid_for(n / 4 + 1, 256), 256, 0, STREAM(stream)>>>(w, g, lr, w_out, n);
  WAP_LAUNCH_CHECK();
  COUNT_LAUNCH();
  return WAP_OK;
}
