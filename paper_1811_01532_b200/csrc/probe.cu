// tcgen05.mma kind::tf32 issue-rate probe, launched by bench.py next to every
// measurement so the GEMM roofline's TF32 peak is measured in the same run on the
// same box (MEASURED_PEAKS.json carries only HBM and bf16 figures).
//
// One CTA per SM: one thread issues back-to-back M = 128, N = 256, K = 8 MMAs
// (4 per k-tile of 32) into a TMEM accumulator with both operands resident in
// shared memory (SS form, 128B swizzle), then commits once. Nothing else runs, so
// the kernel time is the tensor pipe's tf32 issue rate times the work:
//   flops = 2 * 128 * 256 * 8 * 4 * iters per CTA (wap_tf32_probe_flops).
// r01 (tools/mma_probe.cu): N >= 128 sustains 2048 MAC/clk/SM on B200.
#include <atomic>

#include "common.cuh"
#include "../../include/wap_b200.h"

extern std::atomic<long long> g_wap_launches;

namespace {

constexpr int kProbeN = 256;
constexpr int kProbeSmem = 48 * 1024 + 1024;  // A 128x32 fp32 + B 256x32 fp32, 1 KB alignment slack

__global__ void __launch_bounds__(128, 1) tf32_probe_kernel(int iters) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int tid = threadIdx.x;
  for (int i = tid; i < (48 * 1024) / 4; i += blockDim.x)
    reinterpret_cast<float*>(sm)[i] = 1.0f + 1e-3f * (float)((i * 2654435761u) % 1000);
  if (tid == 0) {
    mbar_init(smem_u32(&bar), 1);
    mbar_fence_init();
  }
  if (tid < 32) tmem_alloc<512>(smem_u32(&holder));
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = holder;
  if (tid < 32) {
    constexpr uint32_t idesc = make_idesc_tf32(128, kProbeN, false, false);
    const uint64_t ad = make_sdesc_sw128(smem_u32(sm), 16, 1024);
    const uint64_t bd = make_sdesc_sw128(smem_u32(sm + 16384), 16, 1024);
    for (int it = 0; it < iters; ++it) {
      if (tid == 0) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) umma_tf32(tmem, ad + kk * 2, bd + kk * 2, idesc, (it | kk) ? 1u : 0u);
      }
      __syncwarp();
    }
    if (tid == 0) umma_commit(smem_u32(&bar));
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid < 32) tmem_dealloc<512>(tmem);
}

}  // namespace

extern "C" double wap_tf32_probe_flops(int iters) {
  return 2.0 * 128.0 * kProbeN * 8.0 * 4.0 * (double)iters * WAP_NUM_SMS;
}

extern "C" int wap_tf32_probe(int iters, void* stream) {
  WAP_CHECK_ARG(iters >= 1, "probe iterations must be positive");
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(tf32_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kProbeSmem) !=
        cudaSuccess) {
      wap_set_error("probe: cannot set dynamic shared memory");
      return WAP_ECUDA;
    }
    attr = true;
  }
  tf32_probe_kernel<<<WAP_NUM_SMS, 128, kProbeSmem, reinterpret_cast<cudaStream_t>(stream)>>>(iters);
  WAP_LAUNCH_CHECK();
  g_wap_launches.fetch_add(1, std::memory_order_relaxed);
  return WAP_OK;
}
