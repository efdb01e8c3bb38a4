// tcgen05 (5th-gen tensor core) TF32 / 3xTF32 shifted-GEMM for sm_100a.
//
// One kernel template covers every dense contraction on the WAP hot path
// (SURVEY §8(a) a8-a11):
//   MatMul        Y  = X W            A K-major,  B MN-major   (interp.py:162-163)
//   GradMatMulX   dX = dY W^T         A K-major,  B K-major    (interp.py:185-189)
//   GradMatMulW   dW = X^T dY         A MN-major, B MN-major   (interp.py:183-184)
//   Conv2D        shifted GEMM over the padded-flat NHWC grid, A rows shifted
//                 per filter tap (interp.py:69-79)
//   GradConv2DX   same with the negated shifts and B = W per tap (interp.py:94-102)
//   GradConv2DW   M = (tap, c) with per-tap A shifts (interp.py:82-91)
//
// Pipeline (one CTA per 128 x BN output tile, 256 threads):
//   warp 0      TMA producer (cp.async.bulk.tensor, SWIZZLE_128B) -> smem ring
//   warp 1      single-thread tcgen05.mma issuer, accumulator in TMEM
//   warp 2      TMEM allocator
//   warps 4-7   (3xTF32) split each landed stage into big/small halves,
//               then the epilogue: tcgen05.ld -> bias/ReLU/mask/halo -> global
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <new>

#include "common.cuh"
#include "../../include/wap_b200.h"

extern std::atomic<long long> g_wap_launches;

namespace {

constexpr int BM = 128;
constexpr int BK = 32;  // fp32 elements per 128-byte swizzle row
constexpr int kThreads = 256;
constexpr int kSmemBudget = 200 * 1024;

struct OperandDev {
  int32_t mn_major, tap_period, ntaps;
  int32_t off[WAP_MAX_TAPS];
};

struct GemmArgs {
  int64_t M, N;
  int32_t k_chunks_total, k_chunks_per_split;
  OperandDev a, b;
  float* c;
  int64_t ldc;
  int64_t split_stride;  // elements between split-K slabs in the workspace
  float* partial;        // split-K workspace (null when splits == 1)
  const float* bias;
  int32_t relu;
  const float* mask;
  int64_t ldm;
  int32_t halo_pad, halo_h, halo_w;
};

template <int BN, int PREC>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 4;
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int STAGE_BYTES = (A_BYTES + B_BYTES) * (PREC == 3 ? 2 : 1);
  static constexpr int STAGES_RAW = kSmemBudget / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

// Coordinates of one 32-wide chunk of an operand at (mn, k).
__device__ __forceinline__ void operand_coords(const OperandDev& op, int mn, int k, int& c0, int& c1) {
  if (!op.mn_major) {
    int tap = 0, kin = k;
    if (op.tap_period > 0) {
      tap = k / op.tap_period;
      kin = k - tap * op.tap_period;
    }
    c0 = kin;
    c1 = mn + op.off[tap];
  } else {
    int tap = 0, inner = mn;
    if (op.tap_period > 0) {
      tap = mn / op.tap_period;
      if (tap >= op.ntaps) tap = op.ntaps - 1;  // rows past M only feed masked outputs
      inner = mn - tap * op.tap_period;
    }
    c0 = inner;
    c1 = k + op.off[tap];
  }
}

// Issue the TMA loads of one operand tile (ROWS x BK) for k-chunk starting at k.
template <int ROWS, bool MN>
__device__ __forceinline__ void load_operand(const CUtensorMap* tm, const OperandDev& op, uint32_t dst,
                                             uint32_t bar, int mn0, int k) {
  if constexpr (!MN) {
    int c0, c1;
    operand_coords(op, mn0, k, c0, c1);
    tma_load_2d(dst, tm, bar, c0, c1);  // box {32, ROWS}
  } else {
#pragma unroll
    for (int j = 0; j < ROWS / 32; ++j) {
      int c0, c1;
      operand_coords(op, mn0 + 32 * j, k, c0, c1);
      tma_load_2d(dst + j * (BK * 128), tm, bar, c0, c1);  // box {32, BK}
    }
  }
}

template <bool MN>
__device__ __forceinline__ uint64_t operand_desc(uint32_t base, int kk) {
  // kk = index of the 8-wide k step inside the 32-wide stage.
  if constexpr (!MN) {
    return make_sdesc_sw128(base + kk * 32, 16, 1024);
  } else {
    return make_sdesc_sw128(base + kk * 1024, BK * 128, 512, 1);
  }
}

// Split fp32 words in place into (big = truncated-to-tf32) and write
// small = x - big to `small`; both keep the swizzled positions.
__device__ __forceinline__ void split_tile(uint32_t* raw, uint32_t* small, int nwords, int tid, int nthr) {
  uint4* r4 = reinterpret_cast<uint4*>(raw);
  uint4* s4 = reinterpret_cast<uint4*>(small);
  for (int i = tid; i < nwords / 4; i += nthr) {
    uint4 x = r4[i];
    uint4 b, s;
    b.x = x.x & 0xFFFFE000u;
    b.y = x.y & 0xFFFFE000u;
    b.z = x.z & 0xFFFFE000u;
    b.w = x.w & 0xFFFFE000u;
    s.x = __float_as_uint(__uint_as_float(x.x) - __uint_as_float(b.x));
    s.y = __float_as_uint(__uint_as_float(x.y) - __uint_as_float(b.y));
    s.z = __float_as_uint(__uint_as_float(x.z) - __uint_as_float(b.z));
    s.w = __float_as_uint(__uint_as_float(x.w) - __uint_as_float(b.w));
    r4[i] = b;
    s4[i] = s;
  }
}

__device__ __forceinline__ bool halo_row(const GemmArgs& g, int64_t m) {
  if (g.halo_pad <= 0) return false;
  const int hp = g.halo_h + 2 * g.halo_pad, wp = g.halo_w + 2 * g.halo_pad;
  const int w = (int)(m % wp);
  const int h = (int)((m / wp) % hp);
  return w < g.halo_pad || w >= g.halo_pad + g.halo_w || h < g.halo_pad || h >= g.halo_pad + g.halo_h;
}

template <int BN, bool A_MN, bool B_MN, int PREC>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ GemmArgs g) {
  using C = Cfg<BN, PREC>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES);
  uint64_t* full_bar = bars;
  uint64_t* empty_bar = bars + STAGES;
  uint64_t* conv_bar = bars + 2 * STAGES;
  uint64_t* tmem_full_bar = bars + 3 * STAGES;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 3 * STAGES + 1);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int n_tile = blockIdx.x, m_tile = blockIdx.y, split = blockIdx.z;
  const int m0 = m_tile * BM, n0 = n_tile * BN;
  const int kc_begin = split * g.k_chunks_per_split;
  const int kc_end = min(g.k_chunks_total, kc_begin + g.k_chunks_per_split);

  auto stage_a = [&](int s) { return smem_u32(smem + s * C::STAGE_BYTES); };
  auto stage_b = [&](int s) { return smem_u32(smem + s * C::STAGE_BYTES + C::A_BYTES); };
  auto stage_as = [&](int s) { return smem_u32(smem + s * C::STAGE_BYTES + C::A_BYTES + C::B_BYTES); };
  auto stage_bs = [&](int s) {
    return smem_u32(smem + s * C::STAGE_BYTES + 2 * C::A_BYTES + C::B_BYTES);
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&full_bar[s]), 1);
      mbar_init(smem_u32(&empty_bar[s]), 1);
      mbar_init(smem_u32(&conv_bar[s]), 128);
    }
    mbar_init(smem_u32(tmem_full_bar), 1);
    mbar_fence_init();
  }
  if (warp == 2) tmem_alloc<C::TMEM_COLS>(smem_u32(tmem_holder));
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      int s = 0;
      uint32_t ph = 0;
      for (int kc = kc_begin; kc < kc_end; ++kc) {
        mbar_wait(smem_u32(&empty_bar[s]), ph ^ 1);
        const uint32_t fb = smem_u32(&full_bar[s]);
        mbar_arrive_expect_tx(fb, C::A_BYTES + C::B_BYTES);
        load_operand<BM, A_MN>(&tmA, g.a, stage_a(s), fb, m0, kc * BK);
        load_operand<BN, B_MN>(&tmB, g.b, stage_b(s), fb, n0, kc * BK);
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t idesc = make_idesc_tf32(BM, BN, A_MN, B_MN);
      int s = 0;
      uint32_t ph = 0;
      for (int kc = kc_begin; kc < kc_end; ++kc) {
        if constexpr (PREC == 3) mbar_wait(smem_u32(&conv_bar[s]), ph);
        else mbar_wait(smem_u32(&full_bar[s]), ph);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {
          const uint64_t ad = operand_desc<A_MN>(stage_a(s), kk);
          const uint64_t bd = operand_desc<B_MN>(stage_b(s), kk);
          const uint32_t acc = (kc > kc_begin || kk > 0) ? 1u : 0u;
          if constexpr (PREC == 3) {
            const uint64_t asd = operand_desc<A_MN>(stage_as(s), kk);
            const uint64_t bsd = operand_desc<B_MN>(stage_bs(s), kk);
            umma_tf32(tmem_base, asd, bd, idesc, acc);
            umma_tf32(tmem_base, ad, bsd, idesc, 1u);
            umma_tf32(tmem_base, ad, bd, idesc, 1u);
          } else {
            umma_tf32(tmem_base, ad, bd, idesc, acc);
          }
        }
        umma_commit(smem_u32(&empty_bar[s]));
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
      umma_commit(smem_u32(tmem_full_bar));
    }
  } else if (warp >= 4) {
    const int et = threadIdx.x - 128;  // 0..127
    if constexpr (PREC == 3) {
      // ---------------- 3xTF32 operand split ----------------
      int s = 0;
      uint32_t ph = 0;
      for (int kc = kc_begin; kc < kc_end; ++kc) {
        mbar_wait(smem_u32(&full_bar[s]), ph);
        uint8_t* base = smem + s * C::STAGE_BYTES;
        split_tile(reinterpret_cast<uint32_t*>(base),
                   reinterpret_cast<uint32_t*>(base + C::A_BYTES + C::B_BYTES), BM * BK, et, 128);
        split_tile(reinterpret_cast<uint32_t*>(base + C::A_BYTES),
                   reinterpret_cast<uint32_t*>(base + 2 * C::A_BYTES + C::B_BYTES), BN * BK, et, 128);
        fence_proxy_async_smem();
        mbar_arrive(smem_u32(&conv_bar[s]));
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
    // ---------------- epilogue ----------------
    mbar_wait(smem_u32(tmem_full_bar), 0);
    tc_fence_after();
    const int wq = warp - 4;  // TMEM lane quarter
    const int64_t m = (int64_t)m0 + wq * 32 + lane;
    const bool row_ok = m < g.M;
    const bool halo = row_ok && halo_row(g, m);
    const bool raw_out = g.partial != nullptr;
    float* out_row = raw_out ? g.partial + (int64_t)split * g.split_stride + m * g.ldc : g.c + m * g.ldc;
    const bool vec = (g.ldc % 4) == 0;
#pragma unroll 1
    for (int cb = 0; cb < BN / 32; ++cb) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(wq * 32) << 16) + cb * 32, v);
      tmem_ld_wait();
      if (!row_ok) continue;
      const int nb = n0 + cb * 32;
      float f[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        float x = __uint_as_float(v[j]);
        const int n = nb + j;
        if (!raw_out && n < g.N) {
          if (g.bias) x += __ldg(g.bias + n);
          if (g.relu) x = fmaxf(x, 0.f);
          if (g.mask) x = (__ldg(g.mask + m * g.ldm + n) > 0.f) ? x : 0.f;
          if (halo) x = 0.f;
        }
        f[j] = x;
      }
      if (vec && nb + 32 <= g.N) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(out_row + nb + j) = make_float4(f[j], f[j + 1], f[j + 2], f[j + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (nb + j < g.N) out_row[nb + j] = f[j];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<C::TMEM_COLS>(tmem_base);
}

// Deterministic split-K reduction: fixed slab order, then the epilogue.
__global__ void splitk_reduce_kernel(const GemmArgs g, int splits) {
  const int64_t total = g.M * g.N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / g.N, n = i - m * g.N;
    const float* p = g.partial + m * g.ldc + n;
    float x = p[0];
    for (int s = 1; s < splits; ++s) x += p[(int64_t)s * g.split_stride];
    if (g.bias) x += g.bias[n];
    if (g.relu) x = fmaxf(x, 0.f);
    if (g.mask) x = (g.mask[m * g.ldm + n] > 0.f) ? x : 0.f;
    if (halo_row(g, m)) x = 0.f;
    g.c[m * g.ldc + n] = x;
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int make_tmap(CUtensorMap* tm, const wap_operand_t& op, int box_outer) {
  // K-major tiles use the 16B-chunk 128B swizzle; MN-major tf32 tiles need
  // the 32B-atom variant (the only MN-major tf32 layout tcgen05 accepts).
  const CUtensorMapSwizzle swz = op.mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B;
  auto enc = encode_fn();
  WAP_CHECK_ARG(enc != nullptr, "cuTensorMapEncodeTiled unavailable");
  WAP_CHECK_ARG(op.ptr != nullptr, "operand pointer is null");
  WAP_CHECK_ARG((reinterpret_cast<uintptr_t>(op.ptr) & 15) == 0, "operand must be 16-byte aligned");
  WAP_CHECK_ARG(op.ld % 4 == 0 && op.ld >= op.inner, "operand ld=%lld must be >= inner and a multiple of 4",
                (long long)op.ld);
  WAP_CHECK_ARG(op.inner >= 1 && op.outer >= 1, "operand extents must be positive");
  cuuint64_t dims[2] = {(cuuint64_t)op.inner, (cuuint64_t)op.outer};
  cuuint64_t strides[1] = {(cuuint64_t)op.ld * 4};
  cuuint32_t box[2] = {32u, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(op.ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    wap_set_error("cuTensorMapEncodeTiled failed (%d) inner=%lld outer=%lld ld=%lld box_outer=%d", (int)r,
                  (long long)op.inner, (long long)op.outer, (long long)op.ld, box_outer);
    return WAP_ECUDA;
  }
  return WAP_OK;
}

struct Plan {
  CUtensorMap tmA, tmB;
  GemmArgs args;
  dim3 grid;
  int bn, a_mn, b_mn, prec, splits;
};

int pick_bn(const wap_gemm_desc_t& d) {
  if (d.block_n) return d.block_n;
  if (d.N <= 64) return 64;
  if (d.precision == 1 && d.N >= 256 && d.N % 256 == 0) return 256;
  return 128;
}

int pick_splits(const wap_gemm_desc_t& d, int bn, int k_chunks) {
  if (d.splits > 0) return std::min(d.splits, k_chunks);
  const long long tiles = (long long)wap_ceil_div(d.M, BM) * wap_ceil_div(d.N, bn);
  if (tiles >= WAP_NUM_SMS) return 1;
  // Fill the machine, keep >= 8 k-chunks per split.
  int s = (int)std::max(1LL, (long long)WAP_NUM_SMS / tiles);
  s = std::min(s, std::max(1, k_chunks / 8));
  return std::max(1, s);
}

int validate_operand(const wap_operand_t& op, const char* name) {
  WAP_CHECK_ARG(op.ntaps >= 1 && op.ntaps <= WAP_MAX_TAPS, "%s.ntaps=%d out of [1,%d]", name, op.ntaps,
                WAP_MAX_TAPS);
  WAP_CHECK_ARG(op.tap_period >= 0, "%s.tap_period negative", name);
  WAP_CHECK_ARG(op.tap_period == 0 || op.tap_period % 32 == 0, "%s.tap_period=%d must be a multiple of 32",
                name, op.tap_period);
  return WAP_OK;
}

int build_plan(const wap_gemm_desc_t* desc, Plan* p) {
  WAP_CHECK_ARG(desc != nullptr, "null gemm descriptor");
  const wap_gemm_desc_t& d = *desc;
  WAP_CHECK_ARG(d.M >= 1 && d.N >= 1 && d.K >= 1, "bad GEMM shape M=%lld N=%lld K=%lld", (long long)d.M,
                (long long)d.N, (long long)d.K);
  WAP_CHECK_ARG(d.precision == 1 || d.precision == 3, "precision must be 1 (tf32) or 3 (3xtf32)");
  WAP_CHECK_ARG(d.c != nullptr && d.ldc >= d.N, "bad output");
  int rc;
  if ((rc = validate_operand(d.a, "a")) || (rc = validate_operand(d.b, "b"))) return rc;
  const int bn = pick_bn(d);
  WAP_CHECK_ARG(bn == 64 || bn == 128 || bn == 256, "block_n must be 64/128/256");
  WAP_CHECK_ARG(!(bn == 256 && d.precision == 3), "block_n 256 unsupported with 3xTF32");
  const int k_chunks = wap_ceil_div(d.K, BK);
  const int splits = pick_splits(d, bn, k_chunks);
  const int kps = wap_ceil_div(k_chunks, splits);
  const int eff_splits = wap_ceil_div(k_chunks, kps);
  if ((rc = make_tmap(&p->tmA, d.a, d.a.mn_major ? BK : BM))) return rc;
  if ((rc = make_tmap(&p->tmB, d.b, d.b.mn_major ? BK : bn))) return rc;
  GemmArgs& g = p->args;
  g.M = d.M;
  g.N = d.N;
  g.k_chunks_total = k_chunks;
  g.k_chunks_per_split = kps;
  g.a = {d.a.mn_major, d.a.tap_period, d.a.ntaps, {}};
  g.b = {d.b.mn_major, d.b.tap_period, d.b.ntaps, {}};
  for (int i = 0; i < WAP_MAX_TAPS; ++i) {
    g.a.off[i] = d.a.off[i];
    g.b.off[i] = d.b.off[i];
  }
  g.c = d.c;
  g.ldc = d.ldc;
  g.bias = d.bias;
  g.relu = d.relu;
  g.mask = d.mask;
  g.ldm = d.ldm;
  g.halo_pad = d.halo_pad;
  g.halo_h = d.halo_h;
  g.halo_w = d.halo_w;
  g.partial = nullptr;
  g.split_stride = d.M * d.ldc;
  if (eff_splits > 1) {
    const int64_t need = (int64_t)eff_splits * d.M * d.ldc * 4;
    WAP_CHECK_ARG(d.workspace != nullptr && d.workspace_bytes >= need,
                  "split-K needs a %lld-byte workspace (got %lld)", (long long)need, (long long)d.workspace_bytes);
    g.partial = d.workspace;
  }
  p->grid = dim3(wap_ceil_div(d.N, bn), wap_ceil_div(d.M, BM), eff_splits);
  WAP_CHECK_ARG(p->grid.y <= 65535, "too many M tiles (%u)", p->grid.y);
  p->bn = bn;
  p->a_mn = d.a.mn_major ? 1 : 0;
  p->b_mn = d.b.mn_major ? 1 : 0;
  p->prec = d.precision;
  p->splits = eff_splits;
  return WAP_OK;
}

template <int BN, bool AMN, bool BMN, int PREC>
int launch_t(const Plan& p, cudaStream_t st) {
  using C = Cfg<BN, PREC>;
  auto kern = gemm_tc_kernel<BN, AMN, BMN, PREC>;
  static bool attr_set = false;  // per-instantiation, set once
  if (!attr_set) {
    WAP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr_set = true;
  }
  kern<<<p.grid, kThreads, C::SMEM, st>>>(p.tmA, p.tmB, p.args);
  WAP_LAUNCH_CHECK();
  g_wap_launches.fetch_add(1, std::memory_order_relaxed);
  return WAP_OK;
}

template <int BN, int PREC>
int launch_majors(const Plan& p, cudaStream_t st) {
  if (!p.a_mn && p.b_mn) return launch_t<BN, false, true, PREC>(p, st);
  if (!p.a_mn && !p.b_mn) return launch_t<BN, false, false, PREC>(p, st);
  if (p.a_mn && p.b_mn) return launch_t<BN, true, true, PREC>(p, st);
  return launch_t<BN, true, false, PREC>(p, st);
}

int run_plan(const Plan& p, cudaStream_t st) {
  int rc;
  if (p.prec == 1) {
    if (p.bn == 64) rc = launch_majors<64, 1>(p, st);
    else if (p.bn == 128) rc = launch_majors<128, 1>(p, st);
    else rc = launch_majors<256, 1>(p, st);
  } else {
    if (p.bn == 64) rc = launch_majors<64, 3>(p, st);
    else rc = launch_majors<128, 3>(p, st);
  }
  if (rc) return rc;
  if (p.splits > 1) {
    const int64_t total = p.args.M * p.args.N;
    const int threads = 256;
    const int blocks = (int)std::min<int64_t>((total + threads - 1) / threads, WAP_NUM_SMS * 8);
    splitk_reduce_kernel<<<blocks, threads, 0, st>>>(p.args, p.splits);
    WAP_LAUNCH_CHECK();
    g_wap_launches.fetch_add(1, std::memory_order_relaxed);
  }
  return WAP_OK;
}

}  // namespace

extern "C" int64_t wap_gemm_workspace_bytes(const wap_gemm_desc_t* desc) {
  if (!desc) return -1;
  wap_gemm_desc_t d = *desc;
  const int bn = pick_bn(d);
  const int k_chunks = wap_ceil_div(d.K, BK);
  const int splits = pick_splits(d, bn, k_chunks);
  const int kps = wap_ceil_div(k_chunks, splits);
  const int eff = wap_ceil_div(k_chunks, kps);
  return eff > 1 ? (int64_t)eff * d.M * d.ldc * 4 : 0;
}

extern "C" int wap_gemm(const wap_gemm_desc_t* desc, void* stream) {
  Plan p;
  int rc = build_plan(desc, &p);
  if (rc) return rc;
  return run_plan(p, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int wap_gemm_plan_create(const wap_gemm_desc_t* desc, void** plan) {
  WAP_CHECK_ARG(plan != nullptr, "null plan out-pointer");
  Plan* p = new (std::nothrow) Plan();
  WAP_CHECK_ARG(p != nullptr, "out of host memory");
  int rc = build_plan(desc, p);
  if (rc) {
    delete p;
    return rc;
  }
  *plan = p;
  return WAP_OK;
}

extern "C" int wap_gemm_plan_run(void* plan, void* stream) {
  WAP_CHECK_ARG(plan != nullptr, "null plan");
  return run_plan(*static_cast<Plan*>(plan), reinterpret_cast<cudaStream_t>(stream));
}

extern "C" void wap_gemm_plan_destroy(void* plan) { delete static_cast<Plan*>(plan); }
