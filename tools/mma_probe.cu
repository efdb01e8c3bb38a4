// tcgen05.mma kind::tf32 issue-rate probe (diagnostic, not product code).
//
// One CTA (or CTA pair) per SM issues back-to-back MMAs into a TMEM accumulator
// with operands already resident (smem B, smem or TMEM A). Reports MAC/clk/SM
// and the implied TF32 TFLOP/s at the measured clock, for
//   form SS (A, B from smem) / TS (A from TMEM, B from smem),
//   cta_group 1 (M = 128) / 2 (M = 256 over a CTA pair), N in {64 .. 256}.
// This is the ceiling the 3xTF32 GEMM (3 TS MMAs per k-step) can reach.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_probe tools/mma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../paper_1811_01532_b200/csrc/common.cuh"

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int CG>
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (CG == 2)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
  else
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
template <int CG>
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if constexpr (CG == 2)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                 ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
  else
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n"
                 ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
template <int CG>
__device__ __forceinline__ void commit(uint32_t bar) {
  if constexpr (CG == 2)
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(bar), "h"((uint16_t)3) : "memory");
  else
    umma_commit(bar);
}

// smem: A tile 128 x 32 fp32 (16 KB) + B tile 256 x 32 fp32 (32 KB), K-major SW128
template <int N, int CG, bool TS, int NACC = 1>
__global__ void __launch_bounds__(128, 1) probe(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int tid = threadIdx.x;
  for (int i = tid; i < (48 * 1024) / 4; i += blockDim.x)
    reinterpret_cast<float*>(sm)[i] = 1.0f + 1e-3f * (float)((i * 2654435761u) % 1000);
  const uint32_t rank = CG == 2 ? cta_rank() : 0;
  if (tid == 0) {
    mbar_init(smem_u32(&bar), 1);
    mbar_fence_init();
  }
  if (tid < 32) {
    if constexpr (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&holder)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      tmem_alloc<512>(smem_u32(&holder));
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) csync();
  tc_fence_after();
  const uint32_t tmem = holder;
  unsigned long long t0 = 0, t1 = 0;
  if (tid < 32 && rank == 0) {
    constexpr uint32_t idesc = make_idesc_tf32(128 * CG, N, false, false);
    const uint32_t sa = smem_u32(sm), sb = smem_u32(sm + 16384);
    const uint64_t ad = make_sdesc_sw128(sa, 16, 1024), bd = make_sdesc_sw128(sb, 16, 1024);
    const uint32_t a_tmem = tmem + 256;
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (tid == 0) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          // NACC independent accumulators (columns [j*N, j*N+N)) break the RAW chain on D
          const uint32_t d = tmem + (uint32_t)((kk % NACC) * N);
          if constexpr (TS) mma_ts<CG>(d, a_tmem + kk * 8, bd + kk * 2, idesc, (it | kk) ? 1u : 0u);
          else mma_ss<CG>(d, ad + kk * 2, bd + kk * 2, idesc, (it | kk) ? 1u : 0u);
        }
      }
      __syncwarp();
    }
    if (tid == 0) commit<CG>(smem_u32(&bar));
    __syncwarp();
  }
  if (rank == 0 || CG == 1) {
    if (tid < 32) mbar_wait(smem_u32(&bar), 0);
  } else {
    if (tid < 32) mbar_wait(smem_u32(&bar), 0);  // multicast commit arrives here too
  }
  if (tid == 0 && rank == 0) {
    t1 = clock64();
    atomicAdd(cycles, t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) csync();
  if (tid < 32) {
    if constexpr (CG == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else tmem_dealloc<512>(tmem);
  }
}

template <int N, int CG, bool TS, int NACC = 1>
void run(int iters) {
  auto k = probe<N, CG, TS, NACC>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 50 * 1024);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 8);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 50 * 1024;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(cyc, 0, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, k, iters, cyc);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return; }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const int leaders = 148 / CG;
    const double cyc_per = (double)c / leaders;
    const double macs_per_leader = (double)iters * 4 * (128.0 * CG) * N * 8;
    const double mac_clk_sm = macs_per_leader / cyc_per / CG;
    const double tflops = 2.0 * macs_per_leader * leaders / (ms * 1e-3) / 1e12;
    if (rep == 1)
      printf("%s acc=%d cta_group::%d N=%3d: %7.1f MAC/clk/SM  (%5.1f clk per MMA)  %6.1f TFLOP/s  (%.3f ms)\n",
             TS ? "TS" : "SS", NACC, CG, N, mac_clk_sm, cyc_per / (iters * 4.0), tflops, ms);
  }
  cudaFree(cyc);
}

int main() {
  const int iters = 20000;
  // independent accumulators at small N (A in TMEM at column 256: N * NACC <= 256)
  run<64, 1, true, 2>(iters);
  run<64, 1, true, 4>(iters);
  run<64, 2, true, 2>(iters);
  run<64, 2, true, 4>(iters);
  run<64, 1, false, 2>(iters);
  run<128, 2, true, 2>(iters);
  run<64, 1, false>(iters);
  run<128, 1, false>(iters);
  run<256, 1, false>(iters);
  run<64, 1, true>(iters);
  run<128, 1, true>(iters);
  run<256, 1, true>(iters);
  run<64, 2, false>(iters);
  run<128, 2, false>(iters);
  run<256, 2, false>(iters);
  run<64, 2, true>(iters);
  run<128, 2, true>(iters);
  run<192, 2, true>(iters);
  run<256, 2, true>(iters);
  return 0;
}
