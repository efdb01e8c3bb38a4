// Probe: can a tcgen05 K-major SWIZZLE_128B smem descriptor start at an arbitrary
// ROW of a 1024-byte-aligned TMA-swizzled tile (row shift s not a multiple of 8)?
//
// This decides the all-SS 3xTF32 conv design: the A halo window of a
// k x k conv is staged once per 32-channel chunk and every filter tap's 128-row A
// tile is addressed as window + shift rows. The swizzle phase of row i is
// ((start >> 7) + i) & 7 if the hardware swizzles on absolute address bits; the
// descriptor's 3-bit "base offset" field (bits 49-51) exists for starts that are
// not pattern-aligned. Both encodings are tried for s = 0..15 against a CPU
// reference with tf32-exact small-integer inputs (exact fp32 sums).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_1811_01532_b200/csrc \
//        -I include tools/desc_shift_probe.cu -o /tmp/desc_shift_probe -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"

constexpr int WROWS = 160;  // window rows (128 + up to 32 shift)
constexpr int N = 128;

__global__ void __launch_bounds__(128, 1) probe(const float* win, const float* b, float* out, int shift, int mode) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = sm;                    // WROWS x 128 B
  uint8_t* sb = sm + WROWS * 128;      // N x 128 B (WROWS*128 = 20480, 1024-aligned)
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  const int tid = threadIdx.x;
  // manual SWIZZLE_128B: 16 B chunk c of row q at q*128 + ((c ^ (q & 7)) << 4)
  for (int i = tid; i < WROWS * 32; i += 128) {
    const int q = i / 32, k = i % 32, c = k / 4, e = k % 4;
    reinterpret_cast<float*>(sa + q * 128 + ((c ^ (q & 7)) << 4))[e] = win[i];
  }
  for (int i = tid; i < N * 32; i += 128) {
    const int q = i / 32, k = i % 32, c = k / 4, e = k % 4;
    reinterpret_cast<float*>(sb + q * 128 + ((c ^ (q & 7)) << 4))[e] = b[i];
  }
  if (tid == 0) {
    mbar_init(smem_u32(&bar), 1);
    mbar_fence_init();
  }
  if (tid < 32) tmem_alloc<128>(smem_u32(&holder));
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = holder;
  if (tid == 0) {
    constexpr uint32_t idesc = make_idesc_tf32(128, N, false, false);
    const uint32_t a0 = smem_u32(sa) + shift * 128;
    uint64_t ad = make_sdesc_sw128(a0, 16, 1024);
    if (mode == 1) ad |= (uint64_t)((a0 >> 7) & 7) << 49;
    if (mode == 2) ad |= (uint64_t)((8 - ((a0 >> 7) & 7)) & 7) << 49;
    const uint64_t bd = make_sdesc_sw128(smem_u32(sb), 16, 1024);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) umma_tf32(tmem, ad + kk * 2, bd + kk * 2, idesc, kk ? 1u : 0u);
    umma_commit(smem_u32(&bar));
  }
  __syncwarp();
  mbar_wait(smem_u32(&bar), 0);
  tc_fence_after();
  const int w = tid / 32;
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t v[32];
    tmem_ld_32x32b_x32(tmem + ((uint32_t)(w * 32) << 16) + c0, v);
    tmem_ld_wait();
    for (int j = 0; j < 32; ++j) out[tid * N + c0 + j] = __uint_as_float(v[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_dealloc<128>(tmem);
}

int main() {
  std::vector<float> win(WROWS * 32), b(N * 32), out(128 * N);
  srand(1);
  for (auto& x : win) x = (float)(rand() % 17 - 8);
  for (auto& x : b) x = (float)(rand() % 17 - 8);
  float *dw, *db, *dout;
  cudaMalloc(&dw, win.size() * 4);
  cudaMalloc(&db, b.size() * 4);
  cudaMalloc(&dout, out.size() * 4);
  cudaMemcpy(dw, win.data(), win.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
  const int smem = WROWS * 128 + N * 128 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 3; ++mode) {
    printf("mode %d (%s):", mode, mode == 0 ? "no base offset" : mode == 1 ? "base offset (addr>>7)&7" : "base offset -(addr>>7)&7");
    for (int s = 0; s < 24; ++s) {
      cudaMemset(dout, 0, out.size() * 4);
      probe<<<1, 128, smem>>>(dw, db, dout, s, mode);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf(" s=%d CUDA %s\n", s, cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
          float r = 0;
          for (int k = 0; k < 32; ++k) r += win[(m + s) * 32 + k] * b[n * 32 + k];
          if (r != out[m * N + n]) ++bad;
        }
      printf(" s%d:%s", s, bad ? "BAD" : "ok");
    }
    printf("\n");
  }
  return 0;
}
