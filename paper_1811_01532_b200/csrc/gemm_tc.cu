// Host side of the tcgen05 shifted GEMM: TMA descriptor encoding, tile / split-K /
// cluster planning, dispatch, and the deterministic split-K reduction.
#include <algorithm>
#include <atomic>
#include <mutex>
#include <new>

#include "gemm_tc.cuh"

extern std::atomic<long long> g_wap_launches;

namespace wapgemm {

// Deterministic split-K reduction (slabs summed in split order) with the full
// epilogue: bias, ReLU, GradReLU mask (float or bits), halo zeroing, and the
// [out > 0] bits of the result. One warp per (row, 32-column chunk): lane j owns
// column 32*chunk + j, so the mask-bit word of the chunk is one ballot.
__global__ void splitk_reduce_kernel(const GemmArgs g, int splits) {
  const int lane = threadIdx.x & 31;
  const int64_t nchunks = (g.N + 31) >> 5;
  const int64_t tasks = g.M * nchunks;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < tasks; t += nwarps) {
    const int64_t m = t / nchunks, chunk = t - m * nchunks;
    const int64_t n = chunk * 32 + lane;
    const bool valid = n < g.N;
    float x = 0.f;
    if (valid) {
      const float* p = g.partial + m * g.ldc + n;
      x = p[0];
      for (int s = 1; s < splits; ++s) x += p[(int64_t)s * g.split_stride];
      if (g.bias) x += g.bias[n];
      if (g.relu) x = fmaxf(x, 0.f);
      if (g.mbits_in) x = ((g.mbits_in[m * g.mbits_in_ld + chunk] >> lane) & 1u) ? x : 0.f;
      else if (g.mask) x = (g.mask[m * g.ldm + n] > 0.f) ? x : 0.f;
      if (halo_row(g, m)) x = 0.f;
      g.c[m * g.ldc + n] = x;
    }
    if (g.mbits_out) {
      const uint32_t bits = __ballot_sync(0xffffffffu, valid && x > 0.f);
      if (lane == 0) g.mbits_out[m * g.mbits_out_ld + chunk] = bits;
    }
  }
}

namespace {

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
  auto enc = encode_fn();
  WAP_CHECK_ARG(enc != nullptr, "cuTensorMapEncodeTiled unavailable");
  WAP_CHECK_ARG(op.ptr != nullptr, "operand pointer is null");
  WAP_CHECK_ARG((reinterpret_cast<uintptr_t>(op.ptr) & 15) == 0, "operand must be 16-byte aligned");
  WAP_CHECK_ARG(op.ld % 4 == 0 && op.ld >= op.inner, "operand ld=%lld must be >= inner and a multiple of 4",
                (long long)op.ld);
  WAP_CHECK_ARG(op.inner >= 1 && op.outer >= 1, "operand extents must be positive");
  // K-major tiles: 16B-chunk 128B swizzle; MN-major tf32 tiles: the 32B-atom variant
  // (the only MN-major tf32 layout tcgen05 accepts).
  const CUtensorMapSwizzle swz = op.mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B;
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

int pick_bn(const wap_gemm_desc_t& d) {
  // 3xTF32 holds the accumulator(s), the chain running sum S and the TMEM A slots in
  // 512 columns: BN <= 192
  if (d.block_n) return d.precision == 3 ? std::min(d.block_n, 192) : d.block_n;
  if (d.precision == 3) {
    // 3xTF32: BN = 128 keeps two accumulators next to the chain sum (the epilogue's
    // chain drains overlap the MMAs); 192 (one accumulator) only where it tiles N exactly
    if (d.N <= 64) return 64;
    if (d.N <= 128 || d.N % 128 == 0) return 128;
    if (d.N <= 192) return 192;
    return 128;
  }
  const int widest = 256;
  const int64_t ntiles = (d.N + widest - 1) / widest;
  const int64_t per = (d.N + ntiles - 1) / ntiles;
  for (int bn : {64, 128, 192, 256})
    if (per <= bn) return bn;
  return 256;
}

constexpr int kMaxChainChunks = 64;               // 2048 K per accumulator chain (TF32 split-K rule)
constexpr int kChainChunks = 8;                   // 3xTF32: 256 K per in-kernel accumulator chain
constexpr long long kAccSlabBytes = 64LL << 20;   // split-K workspace the accuracy rule may use

struct Shape {
  int bn, cg, splits, kps, m_tiles, n_tiles, k_chunks;
};

Shape plan_shape(const wap_gemm_desc_t& d) {
  Shape s;
  s.bn = pick_bn(d);
  s.k_chunks = wap_ceil_div(d.K, BK);
  s.n_tiles = wap_ceil_div(d.N, s.bn);
  // CTA pairs (cta_group::2) whenever there are enough 256-row tiles to fill the pairs
  const long long pair_tiles = (long long)wap_ceil_div(d.M, 2 * BM) * s.n_tiles;
  s.cg = (d.M > BM && (pair_tiles >= WAP_NUM_SMS / 4 || d.K >= 64 * BK)) ? 2 : 1;
  if (d.cluster == 1 || d.cluster == 2) s.cg = d.cluster;
  const char* force = getenv("WAP_GEMM_CG");
  if (force) s.cg = atoi(force) == 2 ? 2 : 1;
  if (d.M <= BM) s.cg = 1;
  s.m_tiles = wap_ceil_div(d.M, BM * s.cg);
  const long long tiles = (long long)s.m_tiles * s.n_tiles;
  const long long slots = WAP_NUM_SMS / s.cg;
  int splits = 1;
  if (d.splits > 0) {
    splits = d.splits;  // explicit (autotuned); split-K reduction handles mask bits too
  } else if (d.mbits_out || d.mbits_in) {
    splits = 1;  // automatic plans keep mask-bit GEMMs unsplit
  } else if (tiles < slots) {
    splits = (int)std::max(1LL, slots / tiles);
    splits = std::min(splits, std::max(1, s.k_chunks / 8));
  }
  // accuracy: the tcgen05 accumulator rounds toward zero, about one ulp per MMA
  // (tools/gemm_split_acc.py), so a long K chain drifts (-6.7e-9 x K relative).
  // Automatic plans cut chains longer than kMaxChainChunks into slabs (summed in
  // round-to-nearest fp32 by the deterministic reduction) whenever the slabs are
  // cheap: weight gradients and other small-output / long-K GEMMs.
  // (3xTF32 instead bounds its chains inside the kernel: GemmArgs::chain_chunks)
  if (d.precision != 3 && d.splits <= 0 && !(d.mbits_out || d.mbits_in)) {
    const int need = wap_ceil_div(s.k_chunks, kMaxChainChunks);
    if (need > splits) {
      const long long per_slab = (long long)d.M * d.ldc * 4;
      const long long cap = std::max(1LL, kAccSlabBytes / std::max(1LL, per_slab));
      splits = (int)std::max<long long>(splits, std::min<long long>(need, cap));
    }
  }
  splits = std::max(1, std::min(splits, s.k_chunks));
  s.kps = wap_ceil_div(s.k_chunks, splits);
  s.splits = wap_ceil_div(s.k_chunks, s.kps);
  return s;
}

template <int CG>
int win_smem_cg(int bn, int boxes) {
  switch (bn) {
    case 64: return smem_bytes_for<64, 3, CG, true>(boxes);
    case 128: return smem_bytes_for<128, 3, CG, true>(boxes);
    default: return smem_bytes_for<192, 3, CG, true>(boxes);  // 3xTF32: BN <= 192
  }
}

// Halo-window reuse for a 3xTF32 K-major A with filter taps (see gemm_tc.cuh WIN).
void plan_window(const wap_gemm_desc_t& d, const Shape& s, int& boxes, int& off_min) {
  boxes = 0;
  off_min = 0;
  const wap_operand_t& a = d.a;
  if (d.precision != 3 || a.mn_major || a.tap_period <= 0 || a.ntaps < 2 || d.window < 0) return;
  if ((int64_t)a.ntaps * a.tap_period != d.K) return;
  // the producer reuses the A tap for a tapped K-major B
  if (!d.b.mn_major && d.b.tap_period > 0 && d.b.tap_period != a.tap_period) return;
  int mn = a.off[0], mx = a.off[0];
  for (int t = 1; t < a.ntaps; ++t) {
    mn = std::min(mn, (int)a.off[t]);
    mx = std::max(mx, (int)a.off[t]);
  }
  const int nb = wap_ceil_div(BM + (mx - mn), BM);
  const int smem = s.cg == 2 ? win_smem_cg<2>(s.bn, nb) : win_smem_cg<1>(s.bn, nb);
  if (smem > kMaxDynSmem) return;
  boxes = nb;
  off_min = mn;
}

int validate_operand(const wap_operand_t& op, const char* name) {
  WAP_CHECK_ARG(op.ntaps >= 1 && op.ntaps <= WAP_MAX_TAPS, "%s.ntaps=%d out of [1,%d]", name, op.ntaps,
                WAP_MAX_TAPS);
  WAP_CHECK_ARG(op.tap_period >= 0, "%s.tap_period negative", name);
  WAP_CHECK_ARG(op.tap_period == 0 || op.tap_period % 32 == 0, "%s.tap_period=%d must be a multiple of 32", name,
                op.tap_period);
  return WAP_OK;
}

int build_plan(const wap_gemm_desc_t* desc, Plan* p) {
  WAP_CHECK_ARG(desc != nullptr, "null gemm descriptor");
  const wap_gemm_desc_t& d = *desc;
  WAP_CHECK_ARG(d.M >= 1 && d.N >= 1 && d.K >= 1, "bad GEMM shape M=%lld N=%lld K=%lld", (long long)d.M,
                (long long)d.N, (long long)d.K);
  WAP_CHECK_ARG(d.precision == 1 || d.precision == 3, "precision must be 1 (tf32) or 3 (3xtf32)");
  WAP_CHECK_ARG(d.M < (1LL << 31) && d.N < (1LL << 31), "GEMM extents must stay below 2^31 rows/columns");
  WAP_CHECK_ARG(d.c != nullptr && d.ldc >= d.N, "bad output");
  WAP_CHECK_ARG(!(d.a.mn_major && !d.b.mn_major), "unsupported operand majors (A MN-major, B K-major)");
  int rc;
  if ((rc = validate_operand(d.a, "a")) || (rc = validate_operand(d.b, "b"))) return rc;
  const Shape s = plan_shape(d);
  WAP_CHECK_ARG(s.bn == 64 || s.bn == 128 || s.bn == 192 || s.bn == 256, "block_n must be 64/128/192/256");
  WAP_CHECK_ARG(!(d.precision == 3 && s.bn > 192), "3xTF32 tiles are at most 192 columns wide");
  if ((rc = make_tmap(&p->tmA, d.a, d.a.mn_major ? BK : BM))) return rc;
  if ((rc = make_tmap(&p->tmB, d.b, d.b.mn_major ? BK : s.bn / s.cg))) return rc;
  GemmArgs& g = p->args;
  g.M = d.M;
  g.N = d.N;
  g.k_chunks_total = s.k_chunks;
  g.k_chunks_per_split = s.kps;
  g.m_tiles = s.m_tiles;
  g.n_tiles = s.n_tiles;
  g.splits = s.splits;
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
  plan_window(d, s, g.win_boxes, g.win_off_min);
  p->win = g.win_boxes > 0 ? 1 : 0;
  g.partial = nullptr;
  g.split_stride = d.M * d.ldc;
  g.l2_prefetch = (d.M <= 512 && !getenv("WAP_NO_L2_PREFETCH")) ? 4 : 0;
  // 3xTF32 accumulator chains (accuracy): the tcgen05 accumulator rounds toward zero,
  // about one ulp per MMA (tools/gemm_split_acc.py: bias -6.7e-9 x K relative for a
  // single chain). Chains of kChainChunks k-chunks (3 x 4 x 8 = 96 MMAs) are summed in
  // round-to-nearest fp32 by the epilogue, which bounds the bias independently of K.
  g.chain_chunks = 0;
  if (d.precision == 3) {
    const char* cc = getenv("WAP_CHAIN_CHUNKS");
    // one accumulator buffer (BN = 192): the MMAs wait for every chain drain, so 4x longer chains
    // (one accumulator buffer with BN = 192: the MMAs wait for each 192-column drain, so
    // 2x longer chains; measured AlexNet conv2: 613 / 668 / 737 tensor-pipe TF/s at chains
    // of 8 / 16 / unbounded, tools/gpurun/r2_exp1.sh)
    // The N = 64 pair kernels (one CTA) hold one accumulator next to S as well and issue 2
    // MMAs per k-slice instead of 3, so 16 k-chunks is the same MMA count per chain as 8
    // (AlexNet d_pool1: 493 / 517 / 533 TF/s at chains of 8 / 16 / unbounded, r2_exp2.sh)
    const bool pair = s.bn == 64 && ((s.cg == 1 && WAP_N64_PAIR) || (s.cg == 2 && WAP_N64_PAIR2));
    g.chain_chunks = cc ? std::max(0, atoi(cc)) : ((s.bn == 192 || pair) ? 2 * kChainChunks : kChainChunks);
  }
  g.mbits_out = d.mbits_out;
  g.mbits_out_ld = d.mbits_out_ld;
  g.mbits_in = d.mbits_in;
  g.mbits_in_ld = d.mbits_in_ld;
  // epilogue output through bulk tensor stores when C is TMA-addressable
  g.tma_store = 0;
  if (s.splits == 1 && (reinterpret_cast<uintptr_t>(d.c) & 15) == 0 && d.ldc % 4 == 0 &&
      !getenv("WAP_GEMM_NO_TMA_STORE")) {
    wap_operand_t oc{};
    oc.ptr = d.c;
    oc.inner = d.N;
    oc.outer = d.M;
    oc.ld = d.ldc;
    oc.mn_major = 0;
    oc.ntaps = 1;
    if ((rc = make_tmap(&p->tmC, oc, 32))) return rc;
    g.tma_store = 1;
  } else {
    p->tmC = p->tmA;  // unused
  }
  WAP_CHECK_ARG(!(d.mbits_out || d.mbits_in) || g.tma_store || s.splits > 1,
                "ReLU mask bits need the TMA-store epilogue or split-K");
  if (s.splits > 1) {
    const int64_t need = (int64_t)s.splits * d.M * d.ldc * 4;
    WAP_CHECK_ARG(d.workspace != nullptr && d.workspace_bytes >= need,
                  "split-K needs a %lld-byte workspace (got %lld)", (long long)need, (long long)d.workspace_bytes);
    g.partial = d.workspace;
  }
  const long long tiles = (long long)s.m_tiles * s.n_tiles * s.splits;
  const long long clusters = std::min<long long>(tiles, WAP_NUM_SMS / s.cg);
  p->grid = (int)(clusters * s.cg);
  p->bn = s.bn;
  p->a_mn = d.a.mn_major ? 1 : 0;
  p->b_mn = d.b.mn_major ? 1 : 0;
  p->prec = d.precision;
  p->cg = s.cg;
  p->splits = s.splits;
  return WAP_OK;
}

int run_plan(const Plan& p, cudaStream_t st) {
  int rc = p.prec == 1 ? launch_prec1(p, st) : launch_prec3(p, st);
  if (rc) return rc;
  g_wap_launches.fetch_add(1, std::memory_order_relaxed);
  if (p.splits > 1) {
    const int64_t warps = p.args.M * ((p.args.N + 31) >> 5);
    const int threads = 256;
    const int blocks = (int)std::min<int64_t>((warps * 32 + threads - 1) / threads, WAP_NUM_SMS * 8);
    splitk_reduce_kernel<<<blocks, threads, 0, st>>>(p.args, p.splits);
    WAP_LAUNCH_CHECK();
    g_wap_launches.fetch_add(1, std::memory_order_relaxed);
  }
  return WAP_OK;
}

}  // namespace
}  // namespace wapgemm

using namespace wapgemm;

extern "C" int64_t wap_gemm_workspace_bytes(const wap_gemm_desc_t* desc) {
  if (!desc) return -1;
  const Shape s = plan_shape(*desc);
  return s.splits > 1 ? (int64_t)s.splits * desc->M * desc->ldc * 4 : 0;
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

extern "C" int wap_gemm_plan_info(const void* plan, int64_t out[8]) {
  WAP_CHECK_ARG(plan != nullptr && out != nullptr, "null plan / output");
  const Plan& p = *static_cast<const Plan*>(plan);
  out[0] = p.bn;
  out[1] = p.cg;
  out[2] = p.splits;
  out[3] = p.args.k_chunks_per_split;
  out[4] = p.args.win_boxes;
  out[5] = p.prec;
  out[6] = (p.prec == 3 && p.bn == 64) ? ((p.cg == 1 && WAP_N64_PAIR) ? 1 : ((p.cg == 2 && WAP_N64_PAIR2) ? 2 : 0)) : 0;
  out[7] = p.args.chain_chunks;
  return WAP_OK;
}
