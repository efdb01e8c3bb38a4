// Fused gradient allreduce + SGD over peer memory (NVLink / NVSwitch):
// the AllReduceSum of every variable (transform.py:551-571, evaluated as the
// left fold of interp.py:115-119,181-182) followed by its SgdUpdate
// (interp.py:203-204), as ONE kernel per gradient bucket instead of an NCCL
// allreduce plus a separate SGD launch.
//
// Every rank maps every other rank's gradient arena, variable arena and flag
// block into its address space (POSIX-fd handles, host side in
// paper_1811_01532_b200/peer_memory.py), and optionally multicast views of the
// two arenas. Rank r owns the 1/world slice of the bucket that starts at
// r * ceil(n / world) (rounded to 4 floats) and, per element of its slice:
//
//   mode WAP_AR_P2P:  g = grad_0[i] + grad_1[i] + ... + grad_{d-1}[i]
//                     (peer loads, ascending rank = the reference left fold),
//                     w = var_r[i] - lr * scale * g,  var_q[i] = w for every q
//                     (peer stores): reduce-scatter + SGD + all-gather;
//   mode WAP_AR_NVLS: g = multimem.ld_reduce.add(grad_mc + i) (summed in the
//                     switch), w as above, multimem.st(var_mc + i, w) (written
//                     to every rank's copy by the switch).
//
// Each updated weight is computed once and broadcast, so the replicas stay
// bitwise equal by construction. Two flag barriers bracket the data phase:
// entry (every rank's gradients of the bucket are final before anyone reads
// them) and exit (every rank's slice is written before anyone's next step).
// Epochs are device-side counters, so the launch is CUDA-graph replayable; a
// bounded spin turns a missing peer into an error word instead of a hang.
#include <algorithm>
#include <atomic>

#include "common.cuh"
#include "../../include/wap_b200.h"

extern std::atomic<long long> g_wap_launches;

namespace {

constexpr long long kSpinLimit = 1LL << 25;  // x ~200 ns sleeps: a few seconds, then give up

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ float4 mm_ld_reduce_v4(const float* p) {
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void mm_st_v4(float* p, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}

// flag block of a rank: [2 phases][WAP_AR_SLOTS][WAP_AR_MAX_RANKS] u32
__device__ __forceinline__ int flag_index(int phase, int slot, int from) {
  return (phase * WAP_AR_SLOTS + slot) * WAP_AR_MAX_RANKS + from;
}

// One thread: publish `e` into every rank's flag (phase, slot, me), then wait
// until this rank's flags (phase, slot, *) all reached `e`.
__device__ bool flag_barrier(const wap_ar_group_t& G, int phase, int slot, uint32_t e) {
  __threadfence_system();
  for (int q = 0; q < G.world; ++q) st_release_sys(G.flags[q] + flag_index(phase, slot, G.rank), e);
  const uint32_t* mine = G.flags[G.rank];
  for (int q = 0; q < G.world; ++q) {
    long long spins = 0;
    while ((int)(ld_acquire_sys(mine + flag_index(phase, slot, q)) - e) < 0) {
      if (++spins > kSpinLimit) {
        atomicExch(G.status, 1);
        return false;
      }
      __nanosleep(200);
    }
  }
  return true;
}

template <int MODE>
__global__ void __launch_bounds__(256) allreduce_sgd_kernel(const wap_ar_group_t G, int64_t off, int64_t n,
                                                            float lr_scale, int slot) {
  __shared__ uint32_t s_epoch;
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    const uint32_t e = G.epochs[slot] + 1;  // this call's epoch (advanced by the last block)
    s_epoch = e;
    // entry: all ranks' gradients of this bucket are final. One block arrives
    // (block 0), every block waits on its own reads of the local flags.
    bool ok = true;
    if (blockIdx.x == 0) {
      ok = flag_barrier(G, 0, slot, e);
    } else {
      const uint32_t* mine = G.flags[G.rank];
      for (int q = 0; q < G.world && ok; ++q) {
        long long spins = 0;
        while ((int)(ld_acquire_sys(mine + flag_index(0, slot, q)) - e) < 0) {
          if (++spins > kSpinLimit || *(volatile int*)G.status) {
            atomicExch(G.status, 1);
            ok = false;
            break;
          }
          __nanosleep(200);
        }
      }
    }
    s_ok = ok;
  }
  __syncthreads();
  const uint32_t e = s_epoch;
  if (s_ok) {
    // this rank's slice of the bucket, in float4 units (bucket offsets are 16-byte aligned)
    const int64_t n4 = n / 4;
    const int64_t per = (n4 + G.world - 1) / G.world;
    const int64_t lo = per * G.rank < n4 ? per * G.rank : n4, hi = lo + per < n4 ? lo + per : n4;
    for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hi;
         i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t x = off + 4 * i;
      float4 g;
      if constexpr (MODE == WAP_AR_NVLS) {
        g = mm_ld_reduce_v4(G.grad_mc + x);
      } else {
        g = *reinterpret_cast<const float4*>(G.grad[0] + x);
        for (int q = 1; q < G.world; ++q) {  // left fold in ascending rank order (interp.py:115-119)
          const float4 h = *reinterpret_cast<const float4*>(G.grad[q] + x);
          g.x = __fadd_rn(g.x, h.x);
          g.y = __fadd_rn(g.y, h.y);
          g.z = __fadd_rn(g.z, h.z);
          g.w = __fadd_rn(g.w, h.w);
        }
      }
      const float4 w = *reinterpret_cast<const float4*>(G.var[G.rank] + x);
      const float4 o = make_float4(fmaf(-lr_scale, g.x, w.x), fmaf(-lr_scale, g.y, w.y), fmaf(-lr_scale, g.z, w.z),
                                   fmaf(-lr_scale, g.w, w.w));
      if constexpr (MODE == WAP_AR_NVLS) {
        mm_st_v4(G.var_mc + x, o);
      } else {
        for (int q = 0; q < G.world; ++q) *reinterpret_cast<float4*>(G.var[q] + x) = o;
      }
    }
    // tail (n % 4) elements: rank 0 handles them
    if (G.rank == 0 && blockIdx.x == 0 && threadIdx.x < (n & 3)) {
      const int64_t x = off + 4 * n4 + threadIdx.x;
      float g = G.grad[0][x];
      for (int q = 1; q < G.world; ++q) g = __fadd_rn(g, G.grad[q][x]);
      const float o = fmaf(-lr_scale, g, G.var[G.rank][x]);
      for (int q = 0; q < G.world; ++q) G.var[q][x] = o;
    }
  }
  // exit: the last block of this rank to finish arrives at every peer and waits
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const uint32_t done = atomicAdd(G.done + slot, 1u);
    if (done == gridDim.x - 1) {
      if (s_ok) flag_barrier(G, 1, slot, e);
      G.done[slot] = 0;
      G.epochs[slot] = e;
      __threadfence();
    }
  }
}

}  // namespace

extern "C" int wap_allreduce_sgd(const wap_ar_group_t* group, int64_t offset, int64_t n, float lr, float scale,
                                 int slot, void* stream) {
  WAP_CHECK_ARG(group != nullptr, "allreduce_sgd: null group");
  const wap_ar_group_t& G = *group;
  WAP_CHECK_ARG(G.world >= 1 && G.world <= WAP_AR_MAX_RANKS, "allreduce_sgd: world %d out of [1,%d]", G.world,
                WAP_AR_MAX_RANKS);
  WAP_CHECK_ARG(G.rank >= 0 && G.rank < G.world, "allreduce_sgd: rank %d outside [0,%d)", G.rank, G.world);
  WAP_CHECK_ARG(slot >= 0 && slot < WAP_AR_SLOTS, "allreduce_sgd: slot %d out of [0,%d)", slot, WAP_AR_SLOTS);
  WAP_CHECK_ARG(offset >= 0 && n >= 0 && offset % 4 == 0, "allreduce_sgd: offset must be a multiple of 4 floats");
  WAP_CHECK_ARG(G.epochs && G.done && G.status, "allreduce_sgd: null device counters");
  for (int q = 0; q < G.world; ++q)
    WAP_CHECK_ARG(G.grad[q] && G.var[q] && G.flags[q], "allreduce_sgd: rank %d buffers not mapped", q);
  WAP_CHECK_ARG(G.mode == WAP_AR_P2P || (G.mode == WAP_AR_NVLS && G.grad_mc && G.var_mc),
                "allreduce_sgd: mode %d needs multicast addresses", G.mode);
  if (n == 0) return WAP_OK;
  const int64_t per4 = (n / 4 + G.world - 1) / G.world;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((per4 + 255) / 256, 2 * WAP_NUM_SMS));
  const float ls = lr * scale;
  if (G.mode == WAP_AR_NVLS)
    allreduce_sgd_kernel<WAP_AR_NVLS><<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(G, offset, n, ls,
                                                                                                 slot);
  else
    allreduce_sgd_kernel<WAP_AR_P2P><<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(G, offset, n, ls,
                                                                                                slot);
  WAP_LAUNCH_CHECK();
  g_wap_launches.fetch_add(1, std::memory_order_relaxed);
  return WAP_OK;
}
