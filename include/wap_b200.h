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
  int32_t block_n;                  /* 0 = automatic, else 64/128/192/256 */
  int32_t cluster;                  /* 0 = automatic, 1 = one CTA, 2 = CTA pair (cta_group::2) */
  int32_t window;                   /* 3xTF32 shifted A: 0 = halo-window reuse when it fits, -1 = off */
  float* workspace;                 /* split-K partials, wap_gemm_workspace_bytes() */
  int64_t workspace_bytes;
  /* ReLU masks as bits (1 bit per element, 32 columns per word, row stride in words):
   * mbits_out: the epilogue also writes [out > 0] of its final output (forward Conv2D /
   *   MatMul + ReLU; forces split-K off);
   * mbits_in: GradReLU mask read from such bits instead of `mask` (dgrad epilogues). */
  uint32_t* mbits_out;
  int64_t mbits_out_ld;
  const uint32_t* mbits_in;
  int64_t mbits_in_ld;
} wap_gemm_desc_t;

int64_t wap_gemm_workspace_bytes(const wap_gemm_desc_t* desc);
int wap_gemm(const wap_gemm_desc_t* desc, void* stream);
/* Plans pre-encode the TMA descriptors once (buffers fixed), for the timed loop. */
int wap_gemm_plan_create(const wap_gemm_desc_t* desc, void** plan);
int wap_gemm_plan_run(void* plan, void* stream);
void wap_gemm_plan_destroy(void* plan);
/* The launch configuration a plan resolved to, and the part of it that fixes the fp32
 * rounding: out[0..7] = {block_n, cta_group, splits, k_chunks_per_split, window boxes,
 * precision, n64 pair mode (1: one CTA, 2: CTA pair), accumulator chain length in k-chunks}. Two plans of one descriptor with equal
 * {splits, k_chunks_per_split, precision, cta_group, pair mode, window > 0, chain} produce bitwise-equal outputs
 * (same per-element accumulation order); the runtime's autotuner only chooses among
 * those, so tuning never changes results (tests/test_gemm_gpu.py). */
int wap_gemm_plan_info(const void* plan, int64_t out[8]);

/* ---- activation layout --------------------------------------------------- */
/* Logical NHWC [B, H, W, C] stored as [B, H+pad, W+pad, ld] (ld >= C,
 * ld % 4 == 0): each image row is followed by `pad` zero columns and each image
 * by `pad` zero rows. Viewed as a flat [rows, ld] matrix, a filter tap (u, v) of
 * a k x k "same" conv (k/2 <= pad) is the row shift (u-k/2)*(W+pad) + (v-k/2):
 * left/up neighbours of the first column/row land in the previous row's or
 * image's trailing zeros (or before the buffer: TMA OOB zero fill), so one
 * trailing halo serves both sides. A 2D matrix [rows, cols] is B=rows,
 * H=W=1, C=cols, pad=0. Element (b,h,w,c) lives at
 *   ((b*(H+p) + h)*(W+p) + w)*ld + c. */
typedef struct {
  int32_t B, H, W, C;
  int32_t pad;
  int32_t ld;
} wap_layout_t;

/* im2col for Conv2D with any stride/padding (interp.py:69-79 generalised):
 * col[(b,ho,wo), (u,v,c)] = x[b, ho*s+u-p, wo*s+v-p, c] (0 outside), columns
 * K..ldcol-1 zeroed. Rows enumerate the output grid with out_pad trailing halo
 * columns/rows (halo rows zero): col is [B*(Ho+out_pad)*(Wo+out_pad), ldcol]. */
/* Direct stride-1 first-layer conv on CUDA cores (exact fp32 FMA): x has C <= 4
 * channels stored as one float4 per pixel; y = conv(x, w) (+bias) (ReLU) at the
 * valid output pixels of layout yl (halo untouched). w is [k*k*C, ldw] (KKIO),
 * Co = yl.C a multiple of 32. mbits (optional) receives the ReLU mask bits in
 * the GEMM epilogue's format. Replaces im2col + a K = k*k*C GEMM for 3-channel
 * inputs (VGG-16 conv1_1). */
int wap_conv_direct(const float* x, wap_layout_t xl, const float* w, int k, int padding, int ldw,
                    const float* bias, int relu, float* y, wap_layout_t yl, uint32_t* mbits, int64_t mbits_ld,
                    void* stream);
/* Direct first-layer weight gradient (GradConv2DW, interp.py:82-91) of a 3x3 'same'
 * stride-1 conv over a 3-channel float4-per-pixel input: dw[(u,v,c), co] (KKIO rows,
 * row stride ldw) = sum_{b,h,w} x[b,h+u-1,w+v-1,c] * dy[b,h,w,co], fp32 FMAs on CUDA
 * cores, deterministic (per-band partials in `work`, wap_conv_wgrad_direct_work_floats
 * floats, summed in band order). Replaces im2col + an M = 27 GEMM (VGG-16 conv1_1). */
int64_t wap_conv_wgrad_direct_work_floats(wap_layout_t dyl);
int wap_conv_wgrad_direct(const float* x, wap_layout_t xl, const float* dy, wap_layout_t dyl, int k, int padding,
                          float* dw, int ldw, float* work, void* stream);
/* Space-to-depth (first-layer strided conv without im2col): a k x k stride-s conv
 * with padding p over x is a ceil(k/s)^2-tap stride-1 VALID conv over
 *   xs[b, i, j, (dy*s+dx)*C + c] = x[b, s*i+dy-p, s*j+dx-p, c]   (0 outside x)
 * with ws[a, e, (dy*s+dx)*C + c, o] = w[s*a+dy, s*e+dx, c, o] (0 beyond k).
 * xs is dense [B*Hs*Ws, ldc] (ldc >= s*s*C, lanes beyond zeroed); w / dw are
 * [k*k*C, ldw], ws / dws are [ks*ks*ldc, ldws]. fold_grad = 1 maps a dws back to
 * dw (the map is a permutation, so the weight gradient is exact). */
int wap_s2d_input(const float* x, wap_layout_t xl, int stride, int padding, int Hs, int Ws, float* xs, int ldc,
                  void* stream);
int wap_s2d_weight(const float* w, float* ws, int k, int C, int Co, int ldw, int stride, int ldc, int ldws,
                   int fold_grad, void* stream);
int wap_im2col(const float* x, wap_layout_t xl, int k, int stride, int padding, int Ho, int Wo, int out_pad,
               float* col, int64_t ldcol, void* stream);
/* col2im (gather form, deterministic) for GradConv2DX (interp.py:94-102):
 * dx[b,h,w,c] = sum over taps mapping to (h,w) of dcol[(b,ho,wo),(u,v,c)]
 * (dcol rows on the out_pad-padded output grid), optionally times
 * [mask[b,h,w,c] > 0] (fused GradReLU, interp.py:197-198). */
int wap_col2im(const float* dcol, int64_t ldcol, int k, int stride, int padding, int Ho, int Wo, int out_pad,
               float* dx, wap_layout_t dxl, const float* mask, wap_layout_t ml, void* stream);

/* Elementwise (interp.py:166-169,197-198): op 0 = BiasAdd y = x + b[c],
 * 1 = ReLU y = max(x, 0), 2 = BiasAdd+ReLU, 3 = GradReLU y = dy * [x > 0]
 * (x = second operand `aux`), 4 = copy / re-layout. */
int wap_elementwise(int op, const float* x, wap_layout_t xl, const float* aux, wap_layout_t al,
                    const float* bias, float* y, wap_layout_t yl, void* stream);
/* AddN / AllReduceSum evaluated in one process (interp.py:115-119): left fold
 * y = ((x0 + x1) + x2) + ... over n <= 16 inputs of identical layout. */
int wap_add_n(const float* const* xs, int n, wap_layout_t l, float* y, void* stream);
/* GradBias (interp.py:194-196): db[c] = sum over all rows of dy[..., c];
 * deterministic two-pass reduction, `work` >= wap_bias_grad_work_floats(l) floats. */
int64_t wap_bias_grad_work_floats(wap_layout_t l);
int wap_bias_grad(const float* dy, wap_layout_t l, float* db, float* work, void* stream);
/* MaxPool (VALID windows): forward writes y and the argmax position inside
 * each window (uint8, indexed like y's storage; ties -> first maximum in
 * row-major window order). Backward is a deterministic gather of dy through
 * the stored argmax, optionally times [mask > 0] (fused GradReLU). */
int wap_maxpool_fwd(const float* x, wap_layout_t xl, int window, int stride, float* y, wap_layout_t yl,
                    uint8_t* argmax, void* stream);
/* Same with flags. WAP_POOL_RELU_FUSED: x is a ReLU output whose GradReLU is fused
 * into this pool's backward; windows with max <= 0 store argmax 0xFF ("no
 * gradient"), which equals the GradReLU mask at the argmax element, so the fused
 * backward runs with mask == NULL. */
#define WAP_POOL_RELU_FUSED 1
int wap_maxpool_fwd_ex(const float* x, wap_layout_t xl, int window, int stride, float* y, wap_layout_t yl,
                       uint8_t* argmax, int flags, void* stream);
int wap_maxpool_bwd(const uint8_t* argmax, const float* dy, wap_layout_t dyl, int window, int stride,
                    float* dx, wap_layout_t dxl, const float* mask, wap_layout_t ml, void* stream);
/* LRN across channels: y = x / (bias + alpha * sum_{|j-c|<=size/2} x_j^2)^beta. */
int wap_lrn_fwd(const float* x, wap_layout_t xl, int size, float alpha, float beta, float bias, float* y,
                wap_layout_t yl, void* stream);
int wap_lrn_bwd(const float* x, wap_layout_t xl, const float* dy, wap_layout_t dyl, int size, float alpha,
                float beta, float bias, float* dx, wap_layout_t dxl, const float* mask, wap_layout_t ml,
                void* stream);
/* Fused LRN -> MaxPool forward (the LRN output is read by nothing else): y/argmax =
 * MaxPool(LRN(x)) exactly as wap_lrn_fwd followed by wap_maxpool_fwd (same floats and
 * argmax), without writing the LRN output. LRN size 5, window 2 or 3, C = 64 or 192,
 * compact channel layouts. */
int wap_lrn_maxpool_fwd(const float* x, wap_layout_t xl, int size, float alpha, float beta, float bias, int window,
                        int stride, float* y, wap_layout_t yl, uint8_t* argmax, void* stream);
/* Fused GradMaxPool -> GradLRN (-> GradReLU) for a stride-2 MaxPool whose input is the
 * output of an LRN over x (AlexNet norm1 -> pool1, norm2 -> pool2): dx = GradLRN(x,
 * GradMaxPool(argmax, dy)) * [mask > 0], without materialising the pool gradient.
 * Same floats as wap_maxpool_bwd followed by wap_lrn_bwd. Replaces the two
 * interp.py branches for GradMaxPool / GradLRN (extension ops, oracle/interp_ref.py).
 * Window 2 or 3, LRN size 5, C = 64 or 192, compact channel layouts. */
int wap_maxpool_lrn_bwd(const uint8_t* argmax, const float* dy, wap_layout_t dyl, int window, int stride,
                        const float* x, wap_layout_t xl, int size, float alpha, float beta, float bias, float* dx,
                        wap_layout_t dxl, const float* mask, wap_layout_t ml, void* stream);
/* Fused SoftmaxXentLoss + GradSoftmaxXent (interp.py:170-175,199-202):
 * loss[0] = sum_rows -(y . logsoftmax(z)) / rows; dz = (softmax(z) - y) / denominator.
 * `work` holds `rows` floats (per-row losses, summed in row order). */
int wap_xent_fwd_bwd(const float* logits, int64_t ldz, const float* labels, int64_t ldy, int rows, int cols,
                     float denominator, float* loss, float* dlogits, int64_t ldd, float* work, void* stream);
/* Host-facing re-layout: unpack = 0 copies a dense [B,H,W,C] buffer into the
 * layout `l` at `dst` (halo/lane padding untouched); unpack = 1 copies the
 * layout at `dst` back into the dense buffer `dense` (used for graph outputs). */
int wap_pack(const float* dense, wap_layout_t l, float* dst, int unpack, void* stream);
/* SgdUpdate (interp.py:203-204): w_out = w - lr * g over n contiguous floats
 * (w_out may alias w: in-place update of the replicated variable). */
int wap_sgd(const float* w, const float* g, float lr, float* w_out, int64_t n, void* stream);

/* ---- Workload Analysis Unit on device (workloads.py:84-204, planner.py:151-246) */
/* One primary layer as the parser sees it. kind 0 = MatMul ([batch, cin] x
 * [cin, cout]), 1 = Conv2D (output [batch, out_h, out_w, cout], k x k kernel).
 * n_grad = number of gradient companions present (1 for the first layer, else 2);
 * weight_elems = weight + bias-of-BiasAdd elements (4 bytes each). */
typedef struct {
  int32_t kind;
  int32_t n_grad;
  int64_t batch, out_h, out_w, cin, cout, k;
  int64_t weight_elems;
} wap_wau_layer_t;

typedef struct {
  double peak_flops, efficiency_knee_flops, link_bandwidth, link_latency, allreduce_chunk_latency;
} wap_wau_profile_t;

/* Sweep d = 1..n_devices (candidates: d | global_batch), IEEE fp64 with no FMA
 * contraction and CPython-3.12 compensated summation over layers, ties -> smaller d.
 * All pointers are DEVICE pointers: layers[n_layers]; flops_out[2*n_layers]
 * (fwd, bwd per layer); t_c/t_s/thr[n_devices] (NaN for non-candidates);
 * d_out[1]. algo: 0 = ring, 1 = naive all-to-all; OR in WAP_WAU_PLAIN_SUM to sum the
 * per-layer terms with a plain left fold instead (the builtin sum() of CPython < 3.12,
 * which the reference's pyproject still admits). */
#define WAP_WAU_PLAIN_SUM 0x100
int wap_wau_select(const wap_wau_layer_t* layers, int n_layers, int64_t global_batch, int n_devices,
                   wap_wau_profile_t profile, int algo, int64_t* flops_out, double* t_c, double* t_s,
                   double* thr, int32_t* d_out, void* stream);

/* ---- fused gradient allreduce + SGD over peer memory (AllReduceSum + SgdUpdate,
 * transform.py:551-571 / interp.py:115-119,181-182,203-204) ------------------------
 * Every rank maps every rank's gradient arena, variable arena and flag block
 * (peer_memory.py: cuMemCreate + POSIX-fd export, pidfd_getfd import, cuMemMap), and
 * in NVLS mode multicast views of the two arenas (cuMulticastCreate/BindMem). One
 * launch per gradient bucket [offset, offset + n) floats of the arenas: rank r
 * reduces its 1/world slice (P2P: peer loads summed in ascending rank order = the
 * reference left fold; NVLS: multimem.ld_reduce in the switch), applies
 * w -= lr * scale * g once, and writes w to every rank's copy (P2P stores /
 * multimem.st), between an entry and an exit flag barrier. Replicas stay bitwise
 * equal by construction. `slot` (< WAP_AR_SLOTS) names the bucket's barrier
 * counters; epochs live on the device, so launches replay inside CUDA graphs. A
 * peer that never arrives sets *status = 1 after a bounded spin (no hang). */
#define WAP_AR_MAX_RANKS 8
#define WAP_AR_SLOTS 64
#define WAP_AR_P2P 0
#define WAP_AR_NVLS 1
#define WAP_AR_FLAG_WORDS (2 * WAP_AR_SLOTS * WAP_AR_MAX_RANKS)
typedef struct {
  int32_t world, rank, mode, reserved;
  float* grad[WAP_AR_MAX_RANKS];      /* gradient arena of each rank, mapped here */
  float* var[WAP_AR_MAX_RANKS];       /* variable arena of each rank, mapped here */
  float* grad_mc;                     /* multicast view of the gradient arenas (NVLS) */
  float* var_mc;                      /* multicast view of the variable arenas (NVLS) */
  uint32_t* flags[WAP_AR_MAX_RANKS];  /* WAP_AR_FLAG_WORDS barrier words of each rank */
  uint32_t* epochs;                   /* local device counters [WAP_AR_SLOTS], zeroed */
  uint32_t* done;                     /* local device counters [WAP_AR_SLOTS], zeroed */
  int32_t* status;                    /* local device error word, zeroed */
} wap_ar_group_t;
int wap_allreduce_sgd(const wap_ar_group_t* group, int64_t offset, int64_t n, float lr, float scale, int slot,
                      void* stream);

/* Measurement only (bench.py): a tcgen05.mma kind::tf32 issue-rate probe, one CTA
 * per SM issuing M=128 N=256 K=8 MMAs from resident shared-memory operands. Time
 * the launch on `stream`; wap_tf32_probe_flops(iters) is the work it performs. This
 * is the TF32 tensor-pipe peak the GEMM roofline is quoted against. */
double wap_tf32_probe_flops(int iters);
int wap_tf32_probe(int iters, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* WAP_B200_H */
