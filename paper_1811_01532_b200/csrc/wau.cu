// Workload Analysis Unit on the GPU: per-layer FLOPs/bytes, Eq. (1) cost model
// and the GPU-count choice, bit-identical to the reference host arithmetic.
//
//   flops   workloads.py:84-117 (int64; companions each cost one forward pass)
//   t_c     planner.py:151-160   work = (fwd+bwd)/d, eff = work/(work+knee), work/(peak*eff)
//   t_s     planner.py:163-177   ring / naive all-to-all
//   T(d)    planner.py:191-192   CPython >= 3.12 sum(): Neumaier compensated, first item seeds;
//                                 WAP_WAU_PLAIN_SUM in `algo`: the plain left fold of CPython < 3.12
//   d*      planner.py:233-238   min over (T, d) -> ties to the smaller d
// Every fp64 operation is an explicit __d*_rn intrinsic so nvcc cannot contract
// a multiply-add into an FMA (which would change the last bit).
#include <atomic>
#include <math.h>

#include "common.cuh"
#include "../../include/wap_b200.h"

extern std::atomic<long long> g_wap_launches;

namespace {

constexpr int kMaxLayers = 256;
constexpr int kMaxDevices = 64;

__device__ __forceinline__ double efficiency(double work, double knee) {
  if (knee == 0.0) return 1.0;
  if (work <= 0.0) return 0.0;
  return __ddiv_rn(work, __dadd_rn(work, knee));
}

struct Neumaier {  // CPython 3.12 builtin sum() over floats (int start 0)
  double s = 0.0, c = 0.0;
  bool first = true;
  bool plain = false;  // CPython < 3.12: sum() is a plain running left fold
  __device__ void add(double x) {
    if (first) {  // 0 + x: the int start is absorbed exactly
      s = x;
      first = false;
      return;
    }
    if (plain) {
      s = __dadd_rn(s, x);
      return;
    }
    const double t = __dadd_rn(s, x);
    if (fabs(s) >= fabs(x)) c = __dadd_rn(c, __dadd_rn(__dadd_rn(s, -t), x));
    else c = __dadd_rn(c, __dadd_rn(__dadd_rn(x, -t), s));
    s = t;
  }
  __device__ double result() const {
    double r = s;
    if (c != 0.0 && isfinite(c)) r = __dadd_rn(r, c);
    return r;
  }
};

__global__ void wau_kernel(const wap_wau_layer_t* __restrict__ layers, int n_layers, int64_t G, int n_dev,
                           wap_wau_profile_t prof, int algo, bool plain_sum, int64_t* __restrict__ flops_out,
                           double* __restrict__ t_c_out, double* __restrict__ t_s_out, double* __restrict__ thr_out,
                           int32_t* __restrict__ d_out) {
  __shared__ long long s_work[kMaxLayers];   // fwd + bwd
  __shared__ long long s_wbytes[kMaxLayers];
  __shared__ double s_total[kMaxDevices];
  // 1) parser: per-layer FLOPs and weight bytes
  for (int l = threadIdx.x; l < n_layers; l += blockDim.x) {
    const wap_wau_layer_t L = layers[l];
    long long fwd, bwd;
    if (L.kind == 2) {  // pre-counted layer: batch = fwd FLOPs, cin = bwd FLOPs
      fwd = L.batch;
      bwd = L.cin;
    } else {
      if (L.kind == 0) fwd = 2LL * L.batch * L.cin * L.cout;
      else fwd = 2LL * L.batch * L.out_h * L.out_w * L.cin * L.cout * L.k * L.k;
      bwd = (long long)L.n_grad * fwd;
    }
    flops_out[2 * l] = fwd;
    flops_out[2 * l + 1] = bwd;
    s_work[l] = fwd + bwd;
    s_wbytes[l] = 4LL * L.weight_elems;
  }
  __syncthreads();
  // 2) cost model, one thread per candidate degree
  for (int d = 1 + threadIdx.x; d <= n_dev; d += blockDim.x) {
    const int i = d - 1;
    if (G % d != 0) {
      t_c_out[i] = t_s_out[i] = thr_out[i] = nan("");
      s_total[i] = INFINITY;
      continue;
    }
    const double dd = (double)d;
    Neumaier tc, ts;
    tc.plain = ts.plain = plain_sum;
    for (int l = 0; l < n_layers; ++l) {
      // compute_time: exact int64 -> double (values < 2^53), correctly rounded division
      const double work = __ddiv_rn((double)s_work[l], dd);
      double t = 0.0;
      if (work != 0.0) t = __ddiv_rn(work, __dmul_rn(prof.peak_flops, efficiency(work, prof.efficiency_knee_flops)));
      tc.add(t);
      // comm_time
      const long long w = s_wbytes[l];
      double u = 0.0;
      if (d > 1 && w != 0) {
        if (algo == 1) {
          u = __dadd_rn(__ddiv_rn((double)(w * (long long)(d - 1) * d), prof.link_bandwidth), prof.link_latency);
        } else {
          const double a = __ddiv_rn(__ddiv_rn((double)(2LL * w * (d - 1)), dd), prof.link_bandwidth);
          u = __dadd_rn(a, __dmul_rn((double)(2 * (d - 1)), prof.allreduce_chunk_latency));
        }
      }
      ts.add(u);
    }
    const double c = tc.result(), s = ts.result();
    const double total = __dadd_rn(c, s);
    t_c_out[i] = c;
    t_s_out[i] = s;
    thr_out[i] = total > 0.0 ? __ddiv_rn((double)G, total) : INFINITY;
    s_total[i] = total;
  }
  __syncthreads();
  // 3) argmin over (T(d), d): strict '<' while scanning d ascending = ties to smaller d
  if (threadIdx.x == 0) {
    int best = 1;
    double bt = INFINITY;
    bool have = false;
    for (int d = 1; d <= n_dev; ++d) {
      if (G % d != 0) continue;
      const double t = s_total[d - 1];
      if (!have || t < bt) {
        bt = t;
        best = d;
        have = true;
      }
    }
    d_out[0] = best;
  }
}

}  // namespace

extern "C" int wap_wau_select(const wap_wau_layer_t* layers, int n_layers, int64_t global_batch, int n_devices,
                              wap_wau_profile_t profile, int algo, int64_t* flops_out, double* t_c, double* t_s,
                              double* thr, int32_t* d_out, void* stream) {
  WAP_CHECK_ARG(n_layers >= 0 && n_layers <= kMaxLayers, "wau: n_layers %d out of [0,%d]", n_layers, kMaxLayers);
  WAP_CHECK_ARG(n_devices >= 1 && n_devices <= kMaxDevices, "device set is empty or too large (%d)", n_devices);
  WAP_CHECK_ARG(global_batch >= 1, "wau: global batch must be positive");
  const bool plain_sum = (algo & WAP_WAU_PLAIN_SUM) != 0;
  algo &= ~WAP_WAU_PLAIN_SUM;
  WAP_CHECK_ARG(algo == 0 || algo == 1, "unknown aggregation algorithm %d", algo);
  WAP_CHECK_ARG(profile.peak_flops > 0 && profile.link_bandwidth > 0, "wau: bad profile");
  WAP_CHECK_ARG(layers || n_layers == 0, "wau: null layers");
  WAP_CHECK_ARG(flops_out && t_c && t_s && thr && d_out, "wau: null output");
  wau_kernel<<<1, 64, 0, reinterpret_cast<cudaStream_t>(stream)>>>(layers, n_layers, global_batch, n_devices, profile,
                                                                   algo, plain_sum, flops_out, t_c, t_s, thr, d_out);
  WAP_LAUNCH_CHECK();
  g_wap_launches.fetch_add(1, std::memory_order_relaxed);
  return WAP_OK;
}
