/*
 * wap_b200.h — C ABI of the B200-native WAP data-parallel training step.
 *
 * The reference (arXiv 1811.01532 desk model, /root/reference/pkg/src/wap) has
 * no FFI: its operator boundary is the per-OpKind dispatch inside
 * `interp.execute` (interp.py:160-206). Each entry below replaces one branch of
 * that dispatch (cited per function), plus the WAU arithmetic of
 * planner.py:151-246. Conventions:
 *   - plain pointers + int64 sizes; fp32 device buffers, NHWC activations,
 *     KKIO conv kernels, [in,out] FC weights (the reference layouts, ir.py:351-362);
 *   - every call is stream-ordered on the `stream` argument (a cudaStream_t,
 *     passed as void*), never synchronises the device, never allocates;
 *   - returns 0 on success, <0 on error; wap_last_error() has the message
 *     (thread-local). Status codes map onto the reference exceptions in the
 *     Python shim (EvalError / WorkloadError).
 */
#ifndef WAP_B200_H
#define WAP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WAP_MAX_TAPS 32

/* ---- library ------------------------------------------------------------ */
const char* wap_version(void);
const char* wap_last_error(void);
/* number of kernels launched by this process through the library (for the
 * bench's gpu_launches claim). */
long long wap_launch_count(void);

/* ---- GEMM / implicit-GEMM convolution on tcgen05 (kind::tf32) ----------- */
/* One operand of a (shifted) GEMM. The operand is a row-major 2D view
 * [outer][inner] with row stride `ld` elements (ld % 4 == 0, ptr 16B aligned).
 *   mn_major = 0 (K-major): inner axis is the reduction axis k.
 *       tap = k / tap_period, coordinate (k % tap_period, mn + off[tap]).
 *   mn_major = 1 (MN-major): inner axis is the output axis (m or n).
 *       tap = mn / tap_period, coordinate (mn % tap_period, k + off[tap]).
 * tap_period = 0 disables taps (off[0] is still added).
 * Out-of-range coordinates read as zero (TMA OOB fill) — that is how the
 * zero "same" padding of Conv2D (interp.py:69-79) is realised. */
typedef struct {
  const float* ptr;
  int64_t inner, outer, ld;
  int32_t mn_major;
  int32_t tap_period;
  int32_t ntaps;
  int32_t off[WAP_MAX_TAPS];
} wap_operand_t;

/* C[m, n] = epi( sum_k A[m,k] B[n,k] ).
 * Replaces interp.py:162-163 (MatMul), 183-189 (GradMatMulW/X),
 * 164-165/190-193 (Conv2D, GradConv2DW/X as shifted GEMMs), with the
 * BiasAdd (166-167), ReLU (168-169) and GradReLU (197-198) rules fused into
 * the epilogue: out = acc (+ bias[n]) (relu) (* [mask[m,n] > 0]); rows that
 * fall on the halo of a padded NHWC grid (halo_pad > 0) are written as 0. */
typedef struct {
  int64_t M, N, K;
  wap_operand_t a, b;
  float* c;
  int64_t ldc;
  const float* bias;
  int32_t relu;
  const float* mask;
  int64_t ldm;
  int32_t halo_pad, halo_h, halo_w; /* unpadded H, W of the grid */
  int32_t precision;                /* 1 = TF32, 3 = 3xTF32 (fp32-accurate) */
  int32_t splits;                   /* split-K factor, 0 = automatic */
  int32_t block_n;                  /* 0 = automatic, else 64/128/256 */
  float* workspace;                 /* split-K partials, wap_gemm_workspace_bytes() */
  int64_t workspace_bytes;
} wap_gemm_desc_t;

int64_t wap_gemm_workspace_bytes(const wap_gemm_desc_t* desc);
int wap_gemm(const wap_gemm_desc_t* desc, void* stream);
/* Plans pre-encode the TMA descriptors once (buffers fixed), for the timed loop. */
int wap_gemm_plan_create(const wap_gemm_desc_t* desc, void** plan);
int wap_gemm_plan_run(void* plan, void* stream);
void wap_gemm_plan_destroy(void* plan);

#ifdef __cplusplus
}
#endif
#endif /* WAP_B200_H */
