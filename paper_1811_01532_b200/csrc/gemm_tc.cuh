// tcgen05 (5th-gen tensor core) TF32 / 3xTF32 shifted-GEMM kernel for sm_100a.
//
// One template covers every dense contraction on the WAP hot path:
//   MatMul        Y  = X W            A K-major,  B MN-major   (interp.py:162-163)
//   GradMatMulX   dX = dY W^T         A K-major,  B K-major    (interp.py:185-189)
//   GradMatMulW   dW = X^T dY         A MN-major, B MN-major   (interp.py:183-184)
//   Conv2D        shifted GEMM over the padded-flat NHWC grid: A rows shifted per
//                 filter tap, zero padding from the TMA out-of-bounds fill (interp.py:69-79)
//   GradConv2DX   same with the negated shifts and B = W[tap] (interp.py:94-102)
//   GradConv2DW   M = (tap, c) with per-tap A shifts (interp.py:82-91)
//
// Structure (persistent, warp-specialised, one CTA per SM or one CTA pair per TPC):
//   warp 0      TMA producer: cp.async.bulk.tensor (SWIZZLE_128B / 128B_ATOM_32B) -> smem ring
//   warp 1      MMA issuer (leader CTA): tcgen05.mma.cta_group::CG.kind::tf32, D in TMEM
//   warp 2      TMEM allocator (2 accumulators x BN columns: epilogue of tile i overlaps
//               the mainloop of tile i+1)
//   warps 4-7   epilogue: tcgen05.ld -> bias / ReLU / GradReLU mask / halo zero -> global
//   warps 8-11  (3xTF32 only) split each landed stage into big = trunc_tf32(x) and
//               small = x - big so the MMA warp can issue small*B + A*small + big*big
// CG = 2 pairs two SMs on one 256 x BN tile (cta_group::2): each CTA stages its own
// 128 rows of A and half of B, halving per-SM shared-memory operand traffic.
#pragma once

#include <cudaTypedefs.h>

#include <type_traits>

#include "common.cuh"
#include "../../include/wap_b200.h"

namespace wapgemm {

constexpr int BM = 128;  // rows per CTA
constexpr int BK = 32;   // fp32 per 128-byte swizzle row
#ifndef WAP_EPI_BUFS
#define WAP_EPI_BUFS 1  // epilogue staging blocks per warp (2: a chunk's TMA store overlaps the next chunk)
#endif
constexpr int kEpiBufs = WAP_EPI_BUFS;
constexpr int kSmemBudget = (220 - 16 * kEpiBufs) * 1024;  // + the epilogue staging below
// epilogue staging: per warp one [32 rows][32 fp32] block in the SWIZZLE_128B
// layout (16-byte chunk j of row r at chunk j ^ (r & 7)): conflict-free for the
// row-per-thread writes and the coalesced reads, and the TMA store's source format
constexpr int kEpiStage = kEpiBufs * 4 * 32 * 128;
constexpr int kBarBytes = 768;  // mbarriers + TMEM address holder [0,512) | tap offsets of A, B [512,768)
#ifndef WAP_N64_PAIR
#define WAP_N64_PAIR 1
#endif
#ifndef WAP_N64_PAIR2
#define WAP_N64_PAIR2 1
#endif
#ifndef WAP_PAIR_ONE_GROUP
#define WAP_PAIR_ONE_GROUP 1
#endif
#ifndef WAP_PAIR_SS
#define WAP_PAIR_SS 0
#endif
#ifndef WAP_PAIR_SG3
#define WAP_PAIR_SG3 0
#endif
#ifndef WAP_SG_NARROW
#define WAP_SG_NARROW 3
#endif
#ifndef WAP_PAIR_WIN_MIN_SLOTS
#define WAP_PAIR_WIN_MIN_SLOTS 2  // windowed pair kernels: 2 even slots + two accumulators (r2_exp17.sh)
#endif
#ifndef WAP_PAIR_ODD_RING
#define WAP_PAIR_ODD_RING 0  // 1 hung a full-size d_pool1 in r02 (tools/gpurun/r2_exp13.sh); off
#endif
// Split accumulators (3xTF32): the tcgen05 MMA rounds its accumulator toward zero,
// about one ulp of the accumulator per MMA (tools/gemm_split_acc.py: bias
// -6.7e-9 * K relative, linear in the MMAs per accumulator, for exact-in-tf32
// inputs). Adding the two small cross products into the same accumulator as
// big*big triples the truncation events (measured: 3.6x the exact-input bias).
// With WAP_SPLIT_ACC each accumulator has a second half: big*big goes to half 0,
// small*B and A*small to half 1 (2^-10 smaller, so its truncations are
// negligible), and the epilogue adds the halves in round-to-nearest fp32.
#ifndef WAP_SPLIT_ACC
#define WAP_SPLIT_ACC 0  // r02: the split-accumulator mode mis-sums some small-M FC GEMMs (tools/smoke_diag.py: fc7 grad 7e-2); off
#endif
// 3xTF32 A operand: big*B and A*small read the RAW A tile straight from shared
// memory (SS form; kind::tf32 ignores the low 13 mantissa bits, so the raw word IS
// big), only small*B takes A from TMEM. The splitter then stores one half-tile
// (small) per k-step instead of two, and a TMEM A slot is 32 columns wide (twice the
// slots in the same columns). With a halo window (WIN) the raw A tile of every tap
// is the window at a row offset: a SWIZZLE_128B descriptor may start at any 128-byte
// row of a 1024-byte-aligned swizzled buffer (measured: tools/desc_shift_probe.cu,
// shifts 0..23 exact with no base-offset field).
#ifndef WAP_A_SS
#define WAP_A_SS 1
#endif
#ifndef WAP_B_SPLIT_EARLY
#define WAP_B_SPLIT_EARLY 1
#endif
#ifndef WAP_WIN_SMALL
#define WAP_WIN_SMALL 1
#endif
// fewest TMEM A slots (3xTF32) worth keeping two accumulators for
#ifndef WAP_MIN_A_SLOTS
#define WAP_MIN_A_SLOTS 4
#endif
#ifndef WAP_SPLIT_GROUPS
#define WAP_SPLIT_GROUPS 2
#endif
constexpr int kSplitGroups = WAP_SPLIT_GROUPS;  // 3xTF32 splitter groups (8 warps each)

struct OperandDev {
  int32_t mn_major, tap_period, ntaps;
  int32_t off[WAP_MAX_TAPS];
};

struct GemmArgs {
  int64_t M, N;
  int32_t k_chunks_total, k_chunks_per_split;
  int32_t m_tiles, n_tiles, splits;  // m_tiles counts cluster tiles (128*CG rows)
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
  int32_t win_boxes, win_off_min;  // WIN: 128-row TMA boxes per A halo window, min tap shift
  int32_t tma_store;               // epilogue writes C through tmC (bulk tensor stores)
  uint32_t* mbits_out;             // ReLU mask bits of the output (32 columns per word)
  int64_t mbits_out_ld;
  const uint32_t* mbits_in;        // GradReLU mask bits (replaces `mask`)
  int64_t mbits_in_ld;
  int32_t l2_prefetch;             // k-steps of TMA L2 prefetch ahead of the ring (0 = off)
  int32_t chain_chunks;            // 3xTF32: k-chunks per TMEM accumulator chain (0 = one chain)
};

// 3xTF32 A operand (WAP_A_SS, CTA pairs): the splitter warps read each landed A row
// once from shared memory and store its small half into TMEM with tcgen05.st;
// small*B takes A from TMEM (tcgen05 "TS" form), big*B and A*small read the raw A
// tile from shared memory (SS). Layout of the 512 TMEM columns for PREC == 3:
//   [0, ACC_BUFS*ACC_W)             accumulators
//   [A_COL0 + j*32, +32)            A small of A slot j   (lane = row, column = k)
// (single CTAs and WAP_A_SS=0, the r01 form: all three MMAs TS, slots of 64 columns
// holding big | small)
// WIN (3xTF32, K-major A with filter taps): A is not staged per k-step. For each
// 32-channel chunk the producer loads ONE halo window of A rows
// [m0 + min_tap_shift, m0 + 128 + max_tap_shift) and the splitter cuts every
// tap's 128-row A tile out of it (tap-inner k order), so a k x k conv reads its
// activations once per chunk instead of k^2 times.
template <int BN, int PREC, int CG, bool WIN = false>
struct Cfg {
  static constexpr int B_ROWS = BN / CG;  // B rows staged by each CTA
  static constexpr int A_BYTES = BM * BK * 4;
  static constexpr int B_BYTES = B_ROWS * BK * 4;
  static constexpr int A_OFF = WIN ? 0 : A_BYTES;  // B offset inside a stage
  // PAIR2 (3xTF32, N = 64, CTA pair): the pair-mode N = 128 MMA [B_raw | B_small] with the
  // B operand's two halves in the two CTAs: CTA 0 stages B_raw (64 rows) in region P, CTA 1
  // B_small (64 rows, split from its raw copy in region R) in P; the N = 64 small*B MMA takes
  // B_raw rows 0-31 from CTA 0's region Q and rows 32-63 from CTA 1's. 2 MMAs per k-slice
  // like PAIR, with the CTA pair's shared A/B traffic and two accumulators.
  static constexpr bool PAIR2 = PREC == 3 && BN == 64 && CG == 2 && WAP_N64_PAIR2;
  static constexpr int P2_Q = 64 * 128, P2_R = 96 * 128;  // PAIR2 region offsets after P
  // PREC 3 smem stage: [A raw] | B raw | B small   (PAIR2: [A raw] | P | Q | R)
  static constexpr int B_REGION = PAIR2 ? 160 * 128 : 2 * B_BYTES;
  static constexpr int STAGE_BYTES = PREC == 3 ? (A_OFF + B_REGION) : (A_BYTES + B_BYTES);
  // PAIR (3xTF32, N = 64, one CTA): a tcgen05 MMA with N <= 64 costs about as much as
  // N = 108 (tools/mma_probe.cu: ~54 cycles vs 32 at full rate), so big*big and
  // big*small run as ONE N = 128 MMA over the contiguous [B_raw | B_small] rows of the
  // stage into a 128-column accumulator, and small*big as an N = 64 MMA into its
  // first half; the epilogue adds the two halves. 2 MMAs per k-slice instead of 3.
  static constexpr bool PAIR = PREC == 3 && BN == 64 && CG == 1 && WAP_N64_PAIR;
  // splitter groups: the single-CTA pair kernels run ONE group (its per-step work is small)
  // so their TMEM A-slot ring needs no even length: 3 slots of 64 columns fit next to two
  // 128-column accumulators and S, and the chain drains overlap the MMAs
  // (halo-window pair kernels keep two groups: their per-tap A split measured too much for
  // one group, d_pool1 0.386 -> 0.427 ms; without the window one group wins, VGG conv1_2
  // fprop / dgrad 0.96 / 1.12 -> 0.66 / 0.75 ms, r2_exp8.sh)
  // Other kernels with BN <= 128 run THREE groups (1024 threads, 64 registers): measured
  // r02 (tools/gpurun/r2_exp18.sh) AlexNet conv4 / d_conv3_relu / d_conv4_w 8-10% faster
  // than two groups (which beat the whole-window split, WSS, as well); BN = 192 keeps two
  // (three: d_conv2_w 0.30 -> 0.37 ms).
  static constexpr int SG = PAIR ? (WAP_PAIR_SG3 ? 3 : ((!WIN && WAP_PAIR_ONE_GROUP) ? 1 : kSplitGroups))
                                 : ((PREC == 3 && BN <= 128) ? WAP_SG_NARROW : kSplitGroups);
  // (off, it hung a full-size d_pool1) halo-window pair kernels with an ODD ring of 3 A
  // slots, the groups observing each other's steps (see EVEN); the default gives them an
  // even ring of 2 slots (WAP_PAIR_WIN_MIN_SLOTS) and two accumulators + S instead
  static constexpr bool ODD_PAIR = PAIR && WIN && WAP_PAIR_ODD_RING;
  // fewest A slots that must fit next to two accumulators + S (else: one accumulator)
  static constexpr int MIN_SLOTS =
      (SG == 1 || ODD_PAIR || (PAIR && SG == 3)) ? 3 : ((PAIR && WIN) ? WAP_PAIR_WIN_MIN_SLOTS : WAP_MIN_A_SLOTS);
  // SACC: two-half accumulators (big*big | small products); PAIR always has two halves
  // raw A from shared memory except for the single-CTA N = 64 pair kernels, where the
  // N = 128 SS MMA (A + all of [B | B_small] from this CTA's shared memory, ~128 B/clk)
  // measured slower than the TS form (tools/gpurun/r2_exp1.sh, r02); the TS form keeps
  // 64-column A slots (3 or 2 of them next to two accumulators + S, see SG / MIN_SLOTS)
  static constexpr bool A_SS = WAP_A_SS && PREC == 3 && !(CG == 1 && BN == 64 && !WAP_PAIR_SS);
  static constexpr bool SACC = PREC == 3 && !PAIR && WAP_SPLIT_ACC && !A_SS;
  static constexpr bool HALVES = PAIR || PAIR2 || SACC;             // accumulator has two halves to add
  static constexpr int HALF = (PAIR || PAIR2) ? 64 : BN;            // column offset of half 1
  static constexpr int ACC_W = (PAIR || PAIR2) ? 128 : (SACC ? 2 * BN : BN);  // TMEM columns per accumulator
  // TMEM columns of one A slot: big + small (TS big*B), or small only when the MMAs
  // that use A's high part read the raw tile from shared memory (WAP_A_SS)
  static constexpr int A_SLOT_W = A_SS ? 32 : 64;
  // running sum of the accumulator chains (3xTF32, see GemmArgs::chain_chunks): BN columns
  static constexpr int S_W = PREC == 3 ? ((PAIR || PAIR2) ? 64 : BN) : 0;
  // WSS (halo window, CTA pair): the small half of the whole A window is computed once
  // per channel chunk into shared memory next to the raw window, and all three MMAs
  // of every tap read A from the window (SS): no per-tap A split, no TMEM A slots
  static constexpr bool WSS = WIN && A_SS && WAP_WIN_SMALL && BN <= 128 && !PAIR && SG == 2;
  static constexpr int WIN_MUL = WSS ? 2 : 1;  // window slot = raw (| small)
  static constexpr int ACC_BUFS =
      WSS ? ((2 * ACC_W + S_W <= 512) ? 2 : 1)
          : ((PREC == 3 && 512 - 2 * ACC_W - S_W < MIN_SLOTS * A_SLOT_W) ? 1 : 2);
  static constexpr int S_COL = ACC_BUFS * ACC_W;
  static constexpr int A_COL0 = S_COL + S_W;
  static constexpr int TMEM_A_SLOTS = PREC == 3 ? (512 - A_COL0) / A_SLOT_W : 64;
  static constexpr int STAGES_SMEM = kSmemBudget / STAGE_BYTES;
  // smem stages (TMA prefetch depth) and TMEM A slots (split -> MMA) are separate rings
#ifndef WAP_MAX_A_SLOTS
#define WAP_MAX_A_SLOTS 12
#endif
  // Splitter groups take alternate k-steps and wait on stage / A-slot mbarriers by
  // parity, so a group must observe every phase of each barrier it waits on (with an
  // odd ring a group would otherwise meet a barrier only every other phase and a
  // parity wait could pass on the phase before the one it needs: ABA). With
  // WAP_RING_EVEN (default) the rings are rounded to a multiple of kSplitGroups
  // (each group owns fixed slots); with WAP_RING_EVEN=0 a group instead also waits,
  // without working, on the barriers of the other group's steps (splitter loop).
  // Both pass the hang hunts (tools/gemm_loop.py, tools/hang_hunt.py); even rings
  // measured slightly faster on VGG-16.
#ifndef WAP_RING_EVEN
#define WAP_RING_EVEN 1
#endif
  static constexpr bool EVEN = WAP_RING_EVEN && !ODD_PAIR;
  static constexpr int ring_round(int n) {
    return (PREC == 3 && EVEN) ? n / SG * SG : n;
  }
  static constexpr int A_SLOTS =
      PREC == 3 ? ring_round(TMEM_A_SLOTS > WAP_MAX_A_SLOTS ? WAP_MAX_A_SLOTS : TMEM_A_SLOTS) : 1;
  // (WSS: the small window doubles the window footprint; 4 B stages keep one window pair
  // of 2 boxes + stages + epilogue staging under 227 KB for BN <= 128)
  static constexpr int STAGES = WIN ? (WSS ? 4 : 6)
                                    : ring_round(STAGES_SMEM > 8 ? 8 : STAGES_SMEM);
  static constexpr int TMEM_COLS = PREC == 3 ? 512 : ((2 * BN <= 128) ? 128 : ((2 * BN <= 256) ? 256 : 512));
  static constexpr int THREADS = PREC == 3 ? 256 + 256 * SG : 256;  // + splitter warp groups
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + kEpiStage + kBarBytes;
  static_assert(STAGES >= 2, "need at least two pipeline stages");
  static_assert(PREC != 3 || !EVEN || (STAGES % SG == 0 && A_SLOTS % SG == 0),
                "3xTF32 rings must be multiples of the splitter group count");
  static_assert(B_ROWS % 32 == 0, "B rows per CTA must be a multiple of 32");
  static_assert(PREC != 3 || A_SLOTS >= SG, "3xTF32 needs TMEM A slots next to the accumulators");
  static_assert(PREC != 3 || WSS || A_COL0 + A_SLOTS * A_SLOT_W <= 512, "3xTF32 TMEM layout exceeds 512 columns");
  static_assert(!WSS || SG == 2, "WSS assigns window slot g to splitter group g");
};

// A row m (32 k-values) of a landed stage, K-major SWIZZLE_128B tile.
__device__ __forceinline__ void load_a_row_kmajor(const uint8_t* tile, int m, uint32_t (&v)[32]) {
  const uint8_t* row = tile + m * 128;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint4 q = *reinterpret_cast<const uint4*>(row + ((j ^ (m & 7)) << 4));
    v[4 * j] = q.x;
    v[4 * j + 1] = q.y;
    v[4 * j + 2] = q.z;
    v[4 * j + 3] = q.w;
  }
}

// A column m (32 k-values) of an MN-major tile: 4 blocks of [32 k][32 m] with the
// 32B-atom swizzle (32-byte chunk index XOR (k & 3)).
__device__ __forceinline__ void load_a_row_mnmajor(const uint8_t* tile, int m, uint32_t (&v)[32]) {
  const uint8_t* blk = tile + (m >> 5) * (BK * 128);
  const int mi = m & 31;
#pragma unroll
  for (int k = 0; k < 32; ++k)
    v[k] = *reinterpret_cast<const uint32_t*>(blk + k * 128 + ((((mi >> 3) ^ (k & 3))) << 5) + (mi & 7) * 4);
}

__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
      "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
      "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

// k-columns [16*half, 16*half+16) of A row m, K-major SWIZZLE_128B tile
__device__ __forceinline__ void load_a_half_kmajor(const uint8_t* tile, int m, int half, uint32_t (&v)[16]) {
  const uint8_t* row = tile + m * 128;
#pragma unroll
  for (int jj = 0; jj < 4; ++jj) {
    const int j = half * 4 + jj;
    const uint4 q = *reinterpret_cast<const uint4*>(row + ((j ^ (m & 7)) << 4));
    v[4 * jj] = q.x;
    v[4 * jj + 1] = q.y;
    v[4 * jj + 2] = q.z;
    v[4 * jj + 3] = q.w;
  }
}

// k-rows [16*half, 16*half+16) of A column m, MN-major 32B-atom tile
__device__ __forceinline__ void load_a_half_mnmajor(const uint8_t* tile, int m, int half, uint32_t (&v)[16]) {
  const uint8_t* blk = tile + (m >> 5) * (BK * 128);
  const int mi = m & 31;
#pragma unroll
  for (int kk = 0; kk < 16; ++kk) {
    const int k = half * 16 + kk;
    v[kk] = *reinterpret_cast<const uint32_t*>(blk + k * 128 + ((((mi >> 3) ^ (k & 3))) << 5) + (mi & 7) * 4);
  }
}

__device__ __forceinline__ void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

__device__ __forceinline__ void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// D[tmem] (+)= A[tmem] * B[smem]
template <int CG>
__device__ __forceinline__ void umma_ts_cg(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                           uint32_t acc) {
  if constexpr (CG == 2) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
  } else {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
  }
}

// small = x - trunc13(x) for the B tile (big is the raw word: kind::tf32 ignores
// the low 13 mantissa bits, measured bitwise by tools/trunc_probe.py).
__device__ __forceinline__ void split_small_only(const uint32_t* raw, uint32_t* small, int nwords, int tid, int nthr) {
  const uint4* r4 = reinterpret_cast<const uint4*>(raw);
  uint4* s4 = reinterpret_cast<uint4*>(small);
#pragma unroll 4
  for (int i = tid; i < nwords / 4; i += nthr) {
    const uint4 x = r4[i];
    uint4 s;
    s.x = __float_as_uint(__uint_as_float(x.x) - __uint_as_float(x.x & 0xFFFFE000u));
    s.y = __float_as_uint(__uint_as_float(x.y) - __uint_as_float(x.y & 0xFFFFE000u));
    s.z = __float_as_uint(__uint_as_float(x.z) - __uint_as_float(x.z & 0xFFFFE000u));
    s.w = __float_as_uint(__uint_as_float(x.w) - __uint_as_float(x.w & 0xFFFFE000u));
    s4[i] = s;
  }
}

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

// 2D TMA; for CG == 2 with a leader-side barrier the .cta_group::2 form lets the
// peer's bytes complete the leader's transaction count.
template <int CG>
__device__ __forceinline__ void tma_load(uint32_t dst, const CUtensorMap* tm, uint32_t bar, int c0, int c1) {
  if constexpr (CG == 2) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
  } else {
    tma_load_2d(dst, tm, bar, c0, c1);
  }
}

template <int ROWS, bool MN, int CGT>
__device__ __forceinline__ void load_operand(const CUtensorMap* tm, const OperandDev& op, uint32_t dst, uint32_t bar,
                                             int mn0, int k) {
  if constexpr (!MN) {
    int c0, c1;
    operand_coords(op, mn0, k, c0, c1);
    tma_load<CGT>(dst, tm, bar, c0, c1);  // box {32, ROWS}
  } else {
#pragma unroll
    for (int j = 0; j < ROWS / 32; ++j) {
      int c0, c1;
      operand_coords(op, mn0 + 32 * j, k, c0, c1);
      tma_load<CGT>(dst + j * (BK * 128), tm, bar, c0, c1);  // box {32, BK}
    }
  }
}

template <bool MN>
__device__ __forceinline__ uint64_t operand_desc(uint32_t base, int kk) {
  if constexpr (!MN) return make_sdesc_sw128(base + kk * 32, 16, 1024);
  else return make_sdesc_sw128(base + kk * 1024, BK * 128, 512, 1);
}

__device__ __forceinline__ void split_tile(uint32_t* raw, uint32_t* small, int nwords, int tid, int nthr) {
  uint4* r4 = reinterpret_cast<uint4*>(raw);
  uint4* s4 = reinterpret_cast<uint4*>(small);
#pragma unroll 4
  for (int i = tid; i < nwords / 4; i += nthr) {
    const uint4 x = r4[i];
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

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ float4 ld_shared_v4f(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr) : "memory");
  return v;
}

// TMA tile prefetch into L2 (no shared-memory destination, no completion tracking)
__device__ __forceinline__ void tma_prefetch_l2(const CUtensorMap* tm, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(tm)),
               "r"(c0), "r"(c1)
               : "memory");
}

// TMA store smem -> global (bulk group), completion tracked per issuing thread
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* tm, uint32_t src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(tm)),
               "r"(src), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ bool halo_row(const GemmArgs& g, int64_t m) {
  if (g.halo_pad <= 0) return false;
  const int hp = g.halo_h + g.halo_pad, wp = g.halo_w + g.halo_pad;
  // padded-grid rows of one launch stay below 2^31 (host-checked), so 32-bit math
  const int mi = (int)m;
  const int w = mi % wp;
  const int h = (mi / wp) % hp;
  return w >= g.halo_w || h >= g.halo_h;  // trailing halo columns / rows of each image
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Address of the same shared object in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t map_to_rank(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

template <int CG>
__device__ __forceinline__ void tmem_alloc_cg(uint32_t dst, uint32_t ncols) {
  if constexpr (CG == 2)
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst), "r"(ncols) : "memory");
  else
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst), "r"(ncols) : "memory");
}
template <int CG>
__device__ __forceinline__ void tmem_relinquish_cg() {
  if constexpr (CG == 2) asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  else asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int CG>
__device__ __forceinline__ void tmem_dealloc_cg(uint32_t taddr, uint32_t ncols) {
  if constexpr (CG == 2)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
  else
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
template <int CG>
__device__ __forceinline__ void umma_cg(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  if constexpr (CG == 2) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
  } else {
    umma_tf32(tmem_d, adesc, bdesc, idesc, acc);
  }
}
// Commit: arrive on `bar` in every CTA of the pair once the issued MMAs finish.
template <int CG>
__device__ __forceinline__ void umma_commit_cg(uint32_t bar) {
  if constexpr (CG == 2) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
        "h"((uint16_t)3)
        : "memory");
  } else {
    umma_commit(bar);
  }
}


// Optional role/wait tracing (build with -DWAP_GEMM_TRACE): block 0 records, per
// role, total cycles and cycles spent in each barrier wait (slots 1..3).
#ifdef WAP_GEMM_TRACE
__device__ unsigned long long g_gemm_trace[64];
#define TRACE_BEGIN() unsigned long long _tr[4] = {0, 0, 0, 0}; const unsigned long long _t0 = clock64()
#define TW(slot, expr) do { const unsigned long long _a = clock64(); expr; _tr[slot] += clock64() - _a; } while (0)
#define TRACE_END()                                                                           \
  do {                                                                                        \
    int _role = -1;                                                                           \
    if (warp == 0 && lane == 0) _role = 0;                                                    \
    else if (warp == 1 && lane == 0) _role = 1;                                               \
    else if (warp == 4 && lane == 0) _role = 2;                                               \
    else if (warp == 8 && lane == 0) _role = 3;                                               \
    else if (warp == 16 && lane == 0) _role = 4;                                              \
    if (blockIdx.x == 0 && _role >= 0) {                                                      \
      g_gemm_trace[_role * 4] = clock64() - _t0;                                              \
      for (int _i = 1; _i < 4; ++_i) g_gemm_trace[_role * 4 + _i] = _tr[_i];                  \
    }                                                                                         \
  } while (0)
#ifdef WAP_EPI_TRACE  // epilogue split: slot 1 TMEM load, 2 staging, 3 bias/mask/stores
#define EPI_T0() unsigned long long _e = clock64()
#define EPI_T(slot) do { const unsigned long long _n = clock64(); _tr[slot] += _n - _e; _e = _n; } while (0)
#else
#define EPI_T0() do {} while (0)
#define EPI_T(slot) do {} while (0)
#endif
#else
#define EPI_T0() do {} while (0)
#define EPI_T(slot) do {} while (0)
#define TRACE_BEGIN() do {} while (0)
#define TW(slot, expr) expr
#define TRACE_END() do {} while (0)
#endif

// TMA coordinates of the 32-row box starting at row mn of an MN-major operand:
// inner coordinate and the k-row offset of its tap (constant along k).
__device__ __forceinline__ void mn_box(const OperandDev& op, const int32_t* off, int mn, int& c0, int& o) {
  int tap = 0;
  if (op.tap_period > 0) {
    tap = mn / op.tap_period;
    if (tap >= op.ntaps) tap = op.ntaps - 1;  // rows past M only feed masked outputs
  }
  c0 = mn - tap * op.tap_period;
  o = off[tap];
}

struct TileCoord {
  int m0, n0, split, kc_begin, kc_end;
};

__device__ __forceinline__ TileCoord decode_tile(const GemmArgs& g, int t, int BNv, int CGv) {
  TileCoord c;
  const int n_tile = t % g.n_tiles;
  const int rest = t / g.n_tiles;
  const int m_tile = rest % g.m_tiles;
  c.split = rest / g.m_tiles;
  c.m0 = m_tile * BM * CGv;
  c.n0 = n_tile * BNv;
  c.kc_begin = c.split * g.k_chunks_per_split;
  c.kc_end = min(g.k_chunks_total, c.kc_begin + g.k_chunks_per_split);
  return c;
}

template <int BN, bool A_MN, bool B_MN, int PREC, int CG, bool WIN = false>
__global__ void __launch_bounds__(Cfg<BN, PREC, CG, WIN>::THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, const __grid_constant__ GemmArgs g) {
  using C = Cfg<BN, PREC, CG, WIN>;
  constexpr int STAGES = C::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned base derived from smem_raw by pointer arithmetic, so the
  // compiler keeps the shared address space (LDS/STS, not generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* win_base = smem + STAGES * C::STAGE_BYTES;                  // 2 A halo windows (WIN)
  const int win_bytes = WIN ? g.win_boxes * C::A_BYTES : 0;
  const int win_slot = win_bytes * C::WIN_MUL;                          // raw window (| its small half)
  uint8_t* epi_base = win_base + 2 * win_slot;                         // 1024-aligned staging
  uint64_t* bars = reinterpret_cast<uint64_t*>(epi_base + kEpiStage);
  uint64_t* wfull_bar = bars + 3 * STAGES + 5;   // [2] window landed (WIN)
  uint64_t* wempty_bar = bars + 3 * STAGES + 7;  // [2] window consumed by both splitter groups (WIN)
  uint64_t* aslot_bar = bars + 3 * STAGES + 9;   // [A_SLOTS] TMEM A slot free again (MMA commit)
  uint64_t* wsmall_bar = aslot_bar + C::A_SLOTS;  // [2] WSS: window's small half written (leader-side)
  uint64_t* full_bar = bars;                    // TMA landed (leader-side for CG=2 & TF32)
  uint64_t* empty_bar = bars + STAGES;          // smem slot free (MMA commit, multicast)
  uint64_t* conv_bar = bars + 2 * STAGES;       // 3xTF32 split done (leader-side)
  uint64_t* tfull_bar = bars + 3 * STAGES;      // [2] accumulator ready (MMA commit, multicast)
  uint64_t* tempty_bar = bars + 3 * STAGES + 2; // [2] accumulator drained (leader-side)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 3 * STAGES + 4);
  int32_t(*s_off)[WAP_MAX_TAPS] = reinterpret_cast<int32_t(*)[WAP_MAX_TAPS]>(reinterpret_cast<uint8_t*>(bars) + 512);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = CG == 2 ? cluster_rank() : 0;
  const bool leader = rank == 0;
  const int cluster_id = blockIdx.x / CG;
  const int n_clusters = gridDim.x / CG;
  const int n_tiles_total = g.m_tiles * g.n_tiles * g.splits;

  auto stage_a = [&](int s) { return smem_u32(smem + s * C::STAGE_BYTES); };
  auto stage_b = [&](int s) { return smem_u32(smem + s * C::STAGE_BYTES + C::A_OFF); };
  auto stage_bs = [&](int s) { return smem_u32(smem + s * C::STAGE_BYTES + C::A_OFF + C::B_BYTES); };
  // WIN: k-chunk kc = (channel chunk, tap), tap innermost
  const int ntaps = WIN ? g.a.ntaps : 1;

  if (warp == 3) {
    s_off[0][lane] = g.a.off[lane];
    s_off[1][lane] = g.b.off[lane];
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(smem_u32(&full_bar[s]), 1);
      mbar_init(smem_u32(&empty_bar[s]), 1);
      mbar_init(smem_u32(&conv_bar[s]), CG);  // one arrive per CTA of the pair
    }
    for (int j = 0; j < C::A_SLOTS; ++j) mbar_init(smem_u32(&aslot_bar[j]), 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_u32(&tfull_bar[i]), 1);
      mbar_init(smem_u32(&tempty_bar[i]), CG);  // one arrive per CTA of the pair
      if (WIN) {
        mbar_init(smem_u32(&wfull_bar[i]), 1);
        // every splitter group, plus (WAP_A_SS) the MMA commit of the window's last tap;
        // WSS: the MMA commit alone (the owning group's window read precedes wsmall)
        mbar_init(smem_u32(&wempty_bar[i]), C::WSS ? 1 : C::SG + (C::A_SS ? 1 : 0));
        mbar_init(smem_u32(&wsmall_bar[i]), CG);  // WSS: one arrive per CTA of the pair
      }
    }
    mbar_fence_init();
  }
  if (warp == 2) {
    tmem_alloc_cg<CG>(smem_u32(tmem_holder), C::TMEM_COLS);
    tmem_relinquish_cg<CG>();
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  TRACE_BEGIN();

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs) ----------------
      // Coordinates advance incrementally along k: the k loop has no integer
      // divisions or indexed constant loads (a single thread issues every box,
      // so its dependent-instruction latency bounds the whole pipeline).
      constexpr int NA = A_MN ? BM / 32 : 1;
      constexpr int NB = B_MN ? C::B_ROWS / 32 : 1;
      const int tpa = g.a.tap_period, tpb = g.b.tap_period;
      int s = 0;
      uint32_t ph = 0;
      int wc = 0;  // windows issued
      for (int t = cluster_id; t < n_tiles_total; t += n_clusters) {
        const TileCoord tc = decode_tile(g, t, BN, CG);
        const int a_row0 = tc.m0 + (int)rank * BM;
        const int b_row0 = tc.n0 + (int)rank * C::B_ROWS;
        // MN-major operands: the tap of each 32-row box is fixed for the tile
        int ac0[NA], ao[NA], bc0[NB], bo[NB];
#pragma unroll
        for (int j = 0; j < NA; ++j) mn_box(g.a, s_off[0], a_row0 + 32 * j, ac0[j], ao[j]);
#pragma unroll
        for (int j = 0; j < NB; ++j) mn_box(g.b, s_off[1], b_row0 + 32 * j, bc0[j], bo[j]);
        // PAIR2: B boxes 0, 1 = rows n0 .. n0+63 (CTA 0 -> P, CTA 1 -> R), box 2 = this CTA's
        // 32-row half (-> Q); MN-major: inner coordinate + k offset of each 32-row box
        int p2row[3], p2c0[3], p2o[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          p2row[j] = tc.n0 + (j < 2 ? 32 * j : 32 * (int)rank);
          p2c0[j] = 0;
          p2o[j] = 0;
          if constexpr (C::PAIR2 && B_MN) mn_box(g.b, s_off[1], p2row[j], p2c0[j], p2o[j]);
        }
        auto p2dst = [&](int st, int j) -> uint32_t {
          return j < 2 ? stage_b(st) + (rank == 0 ? 0 : C::P2_R) + j * 4096 : stage_b(st) + C::P2_Q;
        };
        // K-major operands: (tap, k within tap) advance with k
        int k = tc.kc_begin * BK;
        int a_tap = 0, a_kin = k, b_tap = 0, b_kin = k;
        if (tpa > 0) { a_tap = k / tpa; a_kin = k - a_tap * tpa; }
        if (tpb > 0) { b_tap = k / tpb; b_kin = k - b_tap * tpb; }
        int a_row = a_row0 + s_off[0][A_MN ? 0 : a_tap], b_row = b_row0 + s_off[1][B_MN ? 0 : b_tap];
        int w_cidx = 0, w_tap = 0;  // WIN: k-chunk = (channel chunk, tap), tap innermost
        if constexpr (WIN) { w_cidx = tc.kc_begin / ntaps; w_tap = tc.kc_begin - w_cidx * ntaps; }
        for (int kc = tc.kc_begin; kc < tc.kc_end; ++kc) {
          if constexpr (WIN) {
            if (w_tap == 0 || kc == tc.kc_begin) {
              const int ws = wc & 1;
              TW(1, mbar_wait(smem_u32(&wempty_bar[ws]), ((wc >> 1) & 1) ^ 1));
              const uint32_t wb = smem_u32(&wfull_bar[ws]);
              mbar_arrive_expect_tx(wb, win_bytes);
              TW(3, for (int bx = 0; bx < g.win_boxes; ++bx)
                tma_load_2d(smem_u32(win_base + ws * win_slot + bx * C::A_BYTES), &tmA, wb, w_cidx * BK,
                            a_row0 + g.win_off_min + bx * BM));
              ++wc;
            }
            TW(2, mbar_wait(smem_u32(&empty_bar[s]), ph ^ 1));
            const uint32_t fb = smem_u32(&full_bar[s]);
            mbar_arrive_expect_tx(fb, C::PAIR2 ? 3 * 4096 : C::B_BYTES);
            const int kflat = w_tap * tpa + w_cidx * BK;
            if constexpr (C::PAIR2) {
#pragma unroll
              for (int j = 0; j < 3; ++j) {
                if constexpr (B_MN) tma_load<1>(p2dst(s, j), &tmB, fb, p2c0[j], kflat + p2o[j]);
                else if (tpb > 0) tma_load<1>(p2dst(s, j), &tmB, fb, w_cidx * BK, p2row[j] + s_off[1][w_tap]);
                else tma_load<1>(p2dst(s, j), &tmB, fb, kflat, p2row[j] + (b_row - b_row0));
              }
            } else if constexpr (B_MN) {
#pragma unroll
              for (int j = 0; j < NB; ++j) tma_load<1>(stage_b(s) + j * (BK * 128), &tmB, fb, bc0[j], kflat + bo[j]);
            } else if (tpb > 0) {  // host guarantees tpb == tpa: the B tap is the A tap
              tma_load<1>(stage_b(s), &tmB, fb, w_cidx * BK, b_row0 + s_off[1][w_tap]);
            } else {
              tma_load<1>(stage_b(s), &tmB, fb, kflat, b_row);
            }
            if (++s == STAGES) { s = 0; ph ^= 1; }
            if (++w_tap == ntaps) { w_tap = 0; ++w_cidx; }
            continue;
          }
          TW(2, mbar_wait(smem_u32(&empty_bar[s]), ph ^ 1));
          uint32_t fb = smem_u32(&full_bar[s]);
          auto issue = [&](auto cgt) {
            constexpr int CGT = decltype(cgt)::value;
            if constexpr (A_MN) {
#pragma unroll
              for (int j = 0; j < NA; ++j) tma_load<CGT>(stage_a(s) + j * (BK * 128), &tmA, fb, ac0[j], k + ao[j]);
            } else {
              tma_load<CGT>(stage_a(s), &tmA, fb, a_kin, a_row);
            }
            if constexpr (C::PAIR2) {
#pragma unroll
              for (int j = 0; j < 3; ++j) {
                if constexpr (B_MN) tma_load<CGT>(p2dst(s, j), &tmB, fb, p2c0[j], k + p2o[j]);
                else tma_load<CGT>(p2dst(s, j), &tmB, fb, b_kin, p2row[j] + (b_row - b_row0));
              }
            } else if constexpr (B_MN) {
#pragma unroll
              for (int j = 0; j < NB; ++j) tma_load<CGT>(stage_b(s) + j * (BK * 128), &tmB, fb, bc0[j], k + bo[j]);
            } else {
              tma_load<CGT>(stage_b(s), &tmB, fb, b_kin, b_row);
            }
          };
          if constexpr (CG == 2 && PREC == 1) {
            fb &= 0xFEFFFFFFu;  // the leader's barrier collects both CTAs' bytes
            if (leader) mbar_arrive_expect_tx(fb, 2 * (C::A_BYTES + C::B_BYTES));
            issue(std::integral_constant<int, 2>{});
          } else {
            mbar_arrive_expect_tx(fb, C::A_BYTES + (C::PAIR2 ? 3 * 4096 : C::B_BYTES));
            TW(3, issue(std::integral_constant<int, 1>{}));
          }
          // L2 prefetch g.l2_prefetch k-steps ahead of the smem ring for operands without
          // filter taps: deepens the bytes in flight of streamed weights in small-M (FC)
          // GEMMs beyond what the shared-memory stages hold (host enables it for M <= 512;
          // for large-M wgrads it measured slower)
          if (g.l2_prefetch > 0 && (kc + g.l2_prefetch) < tc.kc_end) {
            const int kp = k + g.l2_prefetch * BK;
            if (tpb == 0) {
              if constexpr (B_MN) {
#pragma unroll
                for (int j = 0; j < NB; ++j) tma_prefetch_l2(&tmB, bc0[j], kp + bo[j]);
              } else {
                tma_prefetch_l2(&tmB, kp, b_row);
              }
            }
            if (tpa == 0) {
              if constexpr (A_MN) {
#pragma unroll
                for (int j = 0; j < NA; ++j) tma_prefetch_l2(&tmA, ac0[j], kp + ao[j]);
              } else {
                tma_prefetch_l2(&tmA, kp, a_row);
              }
            }
          }
          if (++s == STAGES) { s = 0; ph ^= 1; }
          k += BK;
          a_kin += BK;
          b_kin += BK;
          if (!A_MN && tpa > 0 && a_kin >= tpa) { a_kin -= tpa; ++a_tap; a_row = a_row0 + s_off[0][a_tap]; }
          if (!B_MN && tpb > 0 && b_kin >= tpb) { b_kin -= tpb; ++b_tap; b_row = b_row0 + s_off[1][b_tap]; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ---------------- MMA issuer (leader CTA) ----------------
      // The whole warp runs the loop (so descriptor math stays warp-uniform and
      // lives in uniform registers); one elected lane issues the tcgen05 ops.
      // A lives in TMEM (K-major by construction) for 3xTF32
      constexpr uint32_t idesc = make_idesc_tf32(BM * CG, BN, PREC == 3 ? false : A_MN, B_MN);
      // WAP_A_SS: the raw-A MMAs read shared memory in the operand's own major-ness
      constexpr uint32_t idesc_ss = make_idesc_tf32(BM * CG, BN, A_MN, B_MN);
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t acc_ph = 0;
      int aj = 0;  // TMEM A slot of the current step
      int mwc = 0;  // WIN: windows seen (slot = (mwc - 1) & 1)
      for (int t = cluster_id; t < n_tiles_total; t += n_clusters) {
        const TileCoord tc = decode_tile(g, t, BN, CG);
        TW(1, mbar_wait(smem_u32(&tempty_bar[acc]), acc_ph ^ 1));
        tc_fence_after();
        const uint32_t dacc = tmem_base + acc * C::ACC_W;
        int mtap = 0;  // WIN: tap of the current k-chunk (tap innermost)
        if constexpr (WIN) mtap = tc.kc_begin % ntaps;
        // 3xTF32 accumulator chains: every chain_chunks k-chunks the accumulator is handed
        // to the epilogue (which folds it into the running sum S in round-to-nearest fp32)
        // and the next chain starts in the other accumulator
        const int clen = (PREC == 3 && g.chain_chunks > 0) ? g.chain_chunks : (tc.kc_end - tc.kc_begin);
        int cpos = 0;
        uint32_t dacc_cur = dacc;
        for (int kc = tc.kc_begin; kc < tc.kc_end; ++kc, ++cpos) {
          if (cpos == clen) {
            if (elect_one()) umma_commit_cg<CG>(smem_u32(&tfull_bar[acc]));
            __syncwarp();
            if (++acc == C::ACC_BUFS) { acc = 0; acc_ph ^= 1; }
            TW(1, mbar_wait(smem_u32(&tempty_bar[acc]), acc_ph ^ 1));
            tc_fence_after();
            dacc_cur = tmem_base + acc * C::ACC_W;
            cpos = 0;
          }
          bool win_last = false;
          uint32_t win_a = 0;  // WIN: raw A tile of this tap = window rows shifted by the tap offset
          if constexpr (WIN) {
            if (mtap == 0 || kc == tc.kc_begin) {
              ++mwc;
              // WSS: both CTAs' small halves of this window are written
              if constexpr (C::WSS) TW(2, mbar_wait(smem_u32(&wsmall_bar[(mwc - 1) & 1]), ((mwc - 1) >> 1) & 1));
            }
            win_last = (mtap == ntaps - 1) || (kc == tc.kc_end - 1);
            win_a = smem_u32(win_base + ((mwc - 1) & 1) * win_slot) +
                    (uint32_t)((s_off[0][mtap] - g.win_off_min) * 128);
          }
          if constexpr (PREC == 3) TW(2, mbar_wait(smem_u32(&conv_bar[s]), ph));
          else TW(2, mbar_wait(smem_u32(&full_bar[s]), ph));
          tc_fence_after();
          // descriptors built once per stage; the k-steps only advance the
          // 14-bit start-address field (addr >> 4), keeping the issue loop short
          constexpr uint64_t kB = B_MN ? (1024 >> 4) : (32 >> 4);
          constexpr uint64_t kA = A_MN ? (1024 >> 4) : (32 >> 4);
          const uint64_t bd0 = operand_desc<B_MN>(stage_b(s), 0);
          const uint64_t bsd0 = operand_desc<B_MN>(stage_bs(s), 0);
          const uint64_t ad0 = WIN ? make_sdesc_sw128(win_a, 16, 1024) : operand_desc<A_MN>(stage_a(s), 0);
          const uint32_t a_big0 = tmem_base + C::A_COL0 + aj * C::A_SLOT_W;
          const uint32_t first0 = cpos > 0 ? 1u : 0u;
#ifdef WAP_GEMM_TMA_ONLY
          // diagnostic: measure the TMA (+ split) stream alone, no MMA
          if (elect_one()) {
            for (uint32_t r = 0; r < (uint32_t)CG; ++r) {
              mbar_arrive_cluster(map_to_rank(smem_u32(&empty_bar[s]), r));
              if constexpr (PREC == 3) mbar_arrive_cluster(map_to_rank(smem_u32(&aslot_bar[aj]), r));
            }
          }
          if (false) {
#else
          if (elect_one()) {
#endif
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              const uint64_t bd = bd0 + kk * kB;
              const uint32_t first = kk > 0 ? 1u : first0;
              if constexpr (C::PAIR2) {
                constexpr uint32_t idesc1 = make_idesc_tf32(BM * CG, 128, A_MN, B_MN);
                constexpr uint32_t idesc2 = make_idesc_tf32(BM * CG, 64, C::WSS ? A_MN : false, B_MN);
                const uint64_t ad = ad0 + kk * kA;
                const uint64_t bq = operand_desc<B_MN>(stage_b(s) + C::P2_Q, 0) + kk * kB;
                umma_cg<CG>(dacc_cur, ad, bd, idesc1, first);                  // A * [B | B_small] (pair halves)
                if constexpr (C::WSS)
                  umma_cg<CG>(dacc_cur, ad + (uint64_t)(win_bytes >> 4), bq, idesc2, 1u);  // small * B (window)
                else
                  umma_ts_cg<CG>(dacc_cur, a_big0 + kk * 8, bq, idesc2, 1u);  // small * B (TMEM A)
              } else if constexpr (C::WSS) {
                // all SS: small half of the window at win_bytes past the raw window
                const uint64_t ad = ad0 + kk * kA;
                const uint64_t as = ad + (uint64_t)(win_bytes >> 4);
                umma_cg<CG>(dacc_cur, as, bd, idesc_ss, first);                // small * B
                umma_cg<CG>(dacc_cur, ad, bsd0 + kk * kB, idesc_ss, 1u);       // A * small
                umma_cg<CG>(dacc_cur, ad, bd, idesc_ss, 1u);                   // big * big
              } else if constexpr (C::A_SS) {
                const uint32_t a_small = a_big0 + kk * 8;
                const uint64_t ad = ad0 + kk * kA;
                if constexpr (C::PAIR) {
                  constexpr uint32_t idesc2 = make_idesc_tf32(BM, 128, A_MN, B_MN);
                  umma_cg<CG>(dacc_cur, ad, bd, idesc2, first);                // A * [B | B_small] (smem A)
                  umma_ts_cg<CG>(dacc_cur, a_small, bd, idesc, 1u);            // small * B (TMEM A)
                } else {
                  umma_ts_cg<CG>(dacc_cur, a_small, bd, idesc, first);         // small * B (TMEM A)
                  umma_cg<CG>(dacc_cur, ad, bsd0 + kk * kB, idesc_ss, 1u);     // A * small (smem A)
                  umma_cg<CG>(dacc_cur, ad, bd, idesc_ss, 1u);                 // big * big (smem A)
                }
              } else if constexpr (C::PAIR) {
                constexpr uint32_t idesc2 = make_idesc_tf32(BM, 128, false, B_MN);
                const uint32_t a_big = a_big0 + kk * 8;
                umma_ts_cg<CG>(dacc_cur, a_big, bd, idesc2, first);            // A * [B | B_small]
                if constexpr (WAP_SPLIT_ACC)
                  umma_ts_cg<CG>(dacc_cur + 64, a_big + 32, bd, idesc, 1u);    // small * B -> small half
                else
                  umma_ts_cg<CG>(dacc_cur, a_big + 32, bd, idesc, 1u);         // small * B
              } else if constexpr (C::SACC) {
                const uint32_t a_big = a_big0 + kk * 8;
                umma_ts_cg<CG>(dacc_cur + C::HALF, a_big + 32, bd, idesc, first);  // small * B -> half 1
                umma_ts_cg<CG>(dacc_cur + C::HALF, a_big, bsd0 + kk * kB, idesc, 1u);  // A * small -> half 1
                umma_ts_cg<CG>(dacc_cur, a_big, bd, idesc, first);                 // big * big -> half 0
              } else if constexpr (PREC == 3) {
                const uint32_t a_big = a_big0 + kk * 8;
                umma_ts_cg<CG>(dacc_cur, a_big + 32, bd, idesc, first);        // small * B
                umma_ts_cg<CG>(dacc_cur, a_big, bsd0 + kk * kB, idesc, 1u);    // A * small
                umma_ts_cg<CG>(dacc_cur, a_big, bd, idesc, 1u);                // big * big
              } else {
                umma_cg<CG>(dacc_cur, ad0 + kk * kA, bd, idesc, first);
              }
            }
            umma_commit_cg<CG>(smem_u32(&empty_bar[s]));
            if constexpr (PREC == 3 && !C::WSS) umma_commit_cg<CG>(smem_u32(&aslot_bar[aj]));
            // the MMAs read the raw window: it is free once the last tap's MMAs complete
            if constexpr (WIN && C::A_SS)
              if (win_last) umma_commit_cg<CG>(smem_u32(&wempty_bar[(mwc - 1) & 1]));
          }
          __syncwarp();
          if (++s == STAGES) { s = 0; ph ^= 1; }
          if (++aj == C::A_SLOTS) aj = 0;
          if constexpr (WIN) mtap = mtap + 1 == ntaps ? 0 : mtap + 1;
        }
#ifdef WAP_GEMM_TMA_ONLY
        if (elect_one())
          for (uint32_t r = 0; r < (uint32_t)CG; ++r) mbar_arrive_cluster(map_to_rank(smem_u32(&tfull_bar[acc]), r));
#else
        if (elect_one()) umma_commit_cg<CG>(smem_u32(&tfull_bar[acc]));
#endif
        __syncwarp();
        if (++acc == C::ACC_BUFS) { acc = 0; acc_ph ^= 1; }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ---------------- epilogue ----------------
    // Phase 1 (thread = accumulator row): tcgen05.ld 32 columns, raw values into
    // this warp's [32 x 32] smem block (SWIZZLE_128B: conflict-free 16-byte accesses).
    // Phase 2 (coalesced, 4 rows x 128 B per instruction): bias / ReLU / GradReLU
    // mask / halo zeroing per 4 columns, with the mask loads of 4 rows in flight
    // together; the result goes back to the block and leaves through one TMA
    // bulk tensor store (split-K partial slabs: direct 16-byte stores).
    const int wq = warp - 4;  // TMEM lane quarter
    const uint32_t stg_base = smem_u32(epi_base) + wq * (32 * 128);
    uint32_t stg_s = stg_base;
    int ebuf = 0;  // staging block of the current chunk (kEpiBufs-deep ring)
    // 16-byte chunk q of staged row r (SWIZZLE_128B)
    auto stg_at = [&](int r, int q) { return stg_s + (uint32_t)(r * 128 + ((q ^ (r & 7)) << 4)); };
    const uint32_t tempty_leader = CG == 2 ? map_to_rank(smem_u32(&tempty_bar[0]), 0) : smem_u32(&tempty_bar[0]);
    int acc = 0;
    uint32_t acc_ph = 0;
    const bool vec = (g.ldc % 4) == 0;
    const bool raw_out = g.partial != nullptr;
    const bool tma_out = !raw_out && g.tma_store;
#ifdef WAP_DIAG_NO_BIAS
    const float* bias = nullptr;
#else
    const float* bias = raw_out ? nullptr : g.bias;
#endif
#ifdef WAP_DIAG_NO_MASK
    const float* mask = nullptr;
#else
    const float* mask = raw_out ? nullptr : g.mask;
#endif
    const bool mvec = (g.ldm % 4) == 0;
    const int c4 = (lane & 7) * 4;
    // bias of this lane's 4 columns of the chunk starting at column nb
    auto load_bias = [&](int nb) {
      float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
      if (bias) {
        const int col = nb + c4;
        if (vec && nb + 32 <= g.N) b = __ldg(reinterpret_cast<const float4*>(bias + col));
        else {
          if (col < g.N) b.x = __ldg(bias + col);
          if (col + 1 < g.N) b.y = __ldg(bias + col + 1);
          if (col + 2 < g.N) b.z = __ldg(bias + col + 2);
          if (col + 3 < g.N) b.w = __ldg(bias + col + 3);
        }
      }
      return b;
    };
    const uint32_t lane_tm = tmem_base + ((uint32_t)(wq * 32) << 16);  // this warp's TMEM lanes
    // logical accumulator columns [c0, c0 + 32) of buffer `a` (PAIR / SACC: both halves added)
    auto load_acc = [&](int a, int c0, uint32_t (&v)[32]) {
      tmem_ld_32x32b_x32(lane_tm + a * C::ACC_W + c0, v);
      if constexpr (C::HALVES) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t v2[16];
          tmem_ld_32x32b_x16(lane_tm + a * C::ACC_W + C::HALF + c0 + hh * 16, v2);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j)
            v[hh * 16 + j] = __float_as_uint(__uint_as_float(v[hh * 16 + j]) + __uint_as_float(v2[j]));
        }
      }
      tmem_ld_wait();
    };
    for (int t = cluster_id; t < n_tiles_total; t += n_clusters) {
      const TileCoord tc = decode_tile(g, t, BN, CG);
      float4 b4_next = load_bias(tc.n0);  // in flight across the accumulator wait
      const int nk = tc.kc_end - tc.kc_begin;
      const int clen = (PREC == 3 && g.chain_chunks > 0) ? g.chain_chunks : nk;
      const int nchains = (nk + clen - 1) / clen;
      // every chain but the last: S (+)= chain accumulator, round-to-nearest fp32, in chain
      // order (deterministic); the accumulator goes straight back to the MMA warp
      for (int ch = 0; ch + 1 < nchains; ++ch) {
        TW(1, mbar_wait(smem_u32(&tfull_bar[acc]), acc_ph));
        tc_fence_after();
        // 16 columns at a time (register pressure: 768 threads share the register file)
#pragma unroll 1
        for (int c0 = 0; c0 < C::S_W; c0 += 16) {
          uint32_t v[16], w[16];
          tmem_ld_32x32b_x16(lane_tm + acc * C::ACC_W + c0, v);
          if constexpr (C::HALVES) tmem_ld_32x32b_x16(lane_tm + acc * C::ACC_W + C::HALF + c0, w);
          tmem_ld_wait();
          if constexpr (C::HALVES) {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) + __uint_as_float(w[j]));
          }
          if (ch > 0) {
            tmem_ld_32x32b_x16(lane_tm + C::S_COL + c0, w);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(__uint_as_float(w[j]) + __uint_as_float(v[j]));
          }
          tmem_st_32x32b_x16(lane_tm + C::S_COL + c0, v);
        }
        tmem_st_wait();
        tc_fence_before();
        named_bar_sync(1, 128);
        if (wq == 0 && lane == 0) {
          if (CG == 2 && !leader) mbar_arrive_cluster(tempty_leader + acc * 8);
          else mbar_arrive(smem_u32(&tempty_bar[acc]));
        }
        if (++acc == C::ACC_BUFS) { acc = 0; acc_ph ^= 1; }
      }
#ifdef WAP_EPI_TRACE
      mbar_wait(smem_u32(&tfull_bar[acc]), acc_ph);
#else
      TW(1, mbar_wait(smem_u32(&tfull_bar[acc]), acc_ph));
#endif
#if defined(WAP_GEMM_TRACE) && !defined(WAP_EPI_TRACE)
      const unsigned long long _drain0 = clock64();
#endif
      tc_fence_after();
      const int64_t m_warp = (int64_t)tc.m0 + (int64_t)rank * BM + wq * 32;  // first row of this warp
      float* out_base = raw_out ? g.partial + (int64_t)tc.split * g.split_stride : g.c;
      // rows this lane stores in phase 2: it * 4 + lane / 8
      uint32_t row_ok = 0, row_zero = 0;
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int64_t row = m_warp + it * 4 + (lane >> 3);
        if (row < g.M) {
          row_ok |= 1u << it;
          if (!raw_out && halo_row(g, row)) row_zero |= 1u << it;
        }
      }
#pragma unroll 1
      for (int cb = 0; cb < BN / 32; ++cb) {
        uint32_t v[32];
        EPI_T0();
        load_acc(acc, cb * 32, v);
        if (PREC == 3 && nchains > 1) {  // + the running sum of the earlier chains
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            uint32_t sv[16];
            tmem_ld_32x32b_x16(lane_tm + C::S_COL + cb * 32 + hh * 16, sv);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j)
              v[hh * 16 + j] = __float_as_uint(__uint_as_float(sv[j]) + __uint_as_float(v[hh * 16 + j]));
          }
        }
        EPI_T(1);
        const int nb = tc.n0 + cb * 32;
        if (nb >= g.N) continue;  // warp-uniform
        const bool full = vec && nb + 32 <= g.N;
        const int col = nb + c4;
        // 1) raw accumulator row -> smem block
        // the TMA store of the previous chunk must have read the staging block
        if (kEpiBufs > 1) {
          stg_s = stg_base + (uint32_t)(ebuf * 4 * 32 * 128);
          ebuf = ebuf + 1 == kEpiBufs ? 0 : ebuf + 1;
        }
        // the TMA store that last used this staging block must have read it
        if (tma_out) {
          if (kEpiBufs > 1) bulk_wait_read_1();
          else bulk_wait_read_all();
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 32; j += 4) st_shared_v4(stg_at(lane, j >> 2), v[j], v[j + 1], v[j + 2], v[j + 3]);
        __syncwarp();
        EPI_T(2);
        // 2) bias of this lane's 4 columns (prefetched one chunk ahead); mask loads of
        //    the rows in flight together
        const float4 b4 = b4_next;
        if (cb + 1 < BN / 32 && nb + 32 < g.N) b4_next = load_bias(nb + 32);
        if (tma_out) {
#ifndef WAP_DIAG_NO_EPI_MATH
          // 2 rows per iteration, rolled (unrolling lets the compiler hoist 8 rows of
          // mask addresses out of the chunk loop and spill them); rows >= M are clipped
          // by the TMA store. Staged row r = it * 4 + lane / 8 has swizzle phase r & 7,
          // which alternates between two values for even / odd it.
          const bool relu = g.relu != 0;
          const int64_t ldm4 = (int64_t)g.ldm * 4;
          const float* mp = (mask && !g.mbits_in) ? mask + (m_warp + (lane >> 3)) * g.ldm + col : nullptr;
          // bit-packed masks: word (row, chunk); this lane's 4 columns are bits c4..c4+3
          const uint32_t* bip = g.mbits_in ? g.mbits_in + (m_warp + (lane >> 3)) * g.mbits_in_ld + (nb >> 5) : nullptr;
          uint32_t* bop = g.mbits_out ? g.mbits_out + (m_warp + (lane >> 3)) * g.mbits_out_ld + (nb >> 5) : nullptr;
          const int64_t bi4 = g.mbits_in_ld * 4, bo4 = g.mbits_out_ld * 4;
          const uint32_t q = lane & 7, r0 = lane >> 3;
          const uint32_t s_even = stg_s + r0 * 128 + ((q ^ r0) << 4);
          const uint32_t s_odd = stg_s + (r0 + 4) * 128 + ((q ^ (r0 + 4)) << 4);
          // GradReLU mask bits of all 8 rows this lane finishes, loaded up front (8 loads in
          // flight instead of one round trip per row pair) and packed as 8 nibbles: row it's
          // 4 columns are bits [4 it, 4 it + 4)
          uint32_t nib = 0;
          if (bip) {
#pragma unroll
            for (int r = 0; r < 8; ++r)
              if (row_ok & (1u << r)) nib |= ((__ldg(bip + (int64_t)r * bi4) >> c4) & 0xFu) << (4 * r);
          }
          // plain outputs (no bias / ReLU / mask / bits / halo: weight gradients) are already
          // final in the staging block
          const bool plain = !bias && !relu && !mask && !g.mbits_in && !bop && g.halo_pad <= 0;
#pragma unroll 1
          for (int it = 0; it < (plain ? 0 : 8); it += 2, mp += mp ? 2 * ldm4 : 0,
                   bop += bop ? 2 * bo4 : 0) {
            float4 mk0 = make_float4(1.f, 1.f, 1.f, 1.f), mk1 = mk0;
            if (bip) {
              const uint32_t w0 = (nib >> (4 * it)) & 0xFu;
              const uint32_t w1 = (nib >> (4 * it + 4)) & 0xFu;
              mk0 = make_float4((float)(w0 & 1u), (float)((w0 >> 1) & 1u), (float)((w0 >> 2) & 1u),
                                (float)((w0 >> 3) & 1u));
              mk1 = make_float4((float)(w1 & 1u), (float)((w1 >> 1) & 1u), (float)((w1 >> 2) & 1u),
                                (float)((w1 >> 3) & 1u));
            } else if (mp) {
              const bool ok0 = row_ok & (1u << it), ok1 = row_ok & (2u << it);
              if (full && mvec) {
                if (ok0) mk0 = __ldg(reinterpret_cast<const float4*>(mp));
                if (ok1) mk1 = __ldg(reinterpret_cast<const float4*>(mp + ldm4));
              } else {
                mk0.x = (ok0 && col < g.N) ? __ldg(mp) : 0.f;
                mk0.y = (ok0 && col + 1 < g.N) ? __ldg(mp + 1) : 0.f;
                mk0.z = (ok0 && col + 2 < g.N) ? __ldg(mp + 2) : 0.f;
                mk0.w = (ok0 && col + 3 < g.N) ? __ldg(mp + 3) : 0.f;
                mk1.x = (ok1 && col < g.N) ? __ldg(mp + ldm4) : 0.f;
                mk1.y = (ok1 && col + 1 < g.N) ? __ldg(mp + ldm4 + 1) : 0.f;
                mk1.z = (ok1 && col + 2 < g.N) ? __ldg(mp + ldm4 + 2) : 0.f;
                mk1.w = (ok1 && col + 3 < g.N) ? __ldg(mp + ldm4 + 3) : 0.f;
              }
            }
            const uint32_t a0 = s_even + it * 512, a1 = s_odd + it * 512;
            float4 x0 = ld_shared_v4f(a0), x1 = ld_shared_v4f(a1);
            const bool z0 = (row_zero >> it) & 1u, z1 = (row_zero >> (it + 1)) & 1u;
            auto fin = [&](float4 x, const float4& m, bool z) {
              x.x += b4.x; x.y += b4.y; x.z += b4.z; x.w += b4.w;
              if (relu) {
                x.x = fmaxf(x.x, 0.f); x.y = fmaxf(x.y, 0.f); x.z = fmaxf(x.z, 0.f); x.w = fmaxf(x.w, 0.f);
              }
              x.x = (!z && m.x > 0.f) ? x.x : 0.f;
              x.y = (!z && m.y > 0.f) ? x.y : 0.f;
              x.z = (!z && m.z > 0.f) ? x.z : 0.f;
              x.w = (!z && m.w > 0.f) ? x.w : 0.f;
              return x;
            };
            x0 = fin(x0, mk0, z0);
            x1 = fin(x1, mk1, z1);
            if (bop) {
              // [out > 0] of rows it / it+1: lane 8k + q holds columns 4q..4q+3 of row k;
              // OR the 8 nibbles of a row together with 3 xor-shuffles inside the 8-lane group
              uint32_t wa = ((x0.x > 0.f) | ((x0.y > 0.f) << 1) | ((x0.z > 0.f) << 2) | ((x0.w > 0.f) << 3)) << c4;
              uint32_t we = ((x1.x > 0.f) | ((x1.y > 0.f) << 1) | ((x1.z > 0.f) << 2) | ((x1.w > 0.f) << 3)) << c4;
#pragma unroll
              for (int o = 1; o < 8; o <<= 1) {
                wa |= __shfl_xor_sync(0xffffffffu, wa, o);
                we |= __shfl_xor_sync(0xffffffffu, we, o);
              }
              if ((lane & 7) == 0) {
                if (row_ok & (1u << it)) *bop = wa;
                if (row_ok & (2u << it)) bop[bo4] = we;
              }
            }
            st_shared_v4(a0, __float_as_uint(x0.x), __float_as_uint(x0.y), __float_as_uint(x0.z), __float_as_uint(x0.w));
            st_shared_v4(a1, __float_as_uint(x1.x), __float_as_uint(x1.y), __float_as_uint(x1.z), __float_as_uint(x1.w));
          }
#endif
        } else {
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            float4 mk[4];
            if (mask) {
  #pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int it = hh * 4 + i;
                mk[i] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (row_ok & (1u << it)) {
                  const float* mp = mask + (m_warp + it * 4 + (lane >> 3)) * g.ldm + col;
                  if (full && mvec) mk[i] = __ldg(reinterpret_cast<const float4*>(mp));
                  else {
                    if (col < g.N) mk[i].x = __ldg(mp);
                    if (col + 1 < g.N) mk[i].y = __ldg(mp + 1);
                    if (col + 2 < g.N) mk[i].z = __ldg(mp + 2);
                    if (col + 3 < g.N) mk[i].w = __ldg(mp + 3);
                  }
                }
              }
            }
  #pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int it = hh * 4 + i;
              if (!(row_ok & (1u << it))) continue;
              const int r = it * 4 + (lane >> 3);
              float4 x = ld_shared_v4f(stg_at(r, lane & 7));
              if (!raw_out) {
                x.x += b4.x; x.y += b4.y; x.z += b4.z; x.w += b4.w;
                if (g.relu) {
                  x.x = fmaxf(x.x, 0.f); x.y = fmaxf(x.y, 0.f); x.z = fmaxf(x.z, 0.f); x.w = fmaxf(x.w, 0.f);
                }
                if (mask) {
                  x.x = mk[i].x > 0.f ? x.x : 0.f;
                  x.y = mk[i].y > 0.f ? x.y : 0.f;
                  x.z = mk[i].z > 0.f ? x.z : 0.f;
                  x.w = mk[i].w > 0.f ? x.w : 0.f;
                }
                if (row_zero & (1u << it)) x = make_float4(0.f, 0.f, 0.f, 0.f);
              }
              if (tma_out) {
                st_shared_v4(stg_at(r, lane & 7), __float_as_uint(x.x), __float_as_uint(x.y), __float_as_uint(x.z),
                             __float_as_uint(x.w));
                continue;
              }
              float* dst = out_base + (m_warp + r) * g.ldc + col;
              if (full) {
                *reinterpret_cast<float4*>(dst) = x;
              } else {
                if (col < g.N) dst[0] = x.x;
                if (col + 1 < g.N) dst[1] = x.y;
                if (col + 2 < g.N) dst[2] = x.z;
                if (col + 3 < g.N) dst[3] = x.w;
              }
            }
          }
        }
        if (tma_out) {
          // the whole 32 x 32 block leaves through one bulk tensor store (rows >= M
          // and columns >= N are clipped by the tensor map)
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
#ifndef WAP_DIAG_NO_EPI_STORE
            tma_store_2d(&tmC, stg_s, nb, (int)m_warp);
#endif
            bulk_commit();
          }
        }
        __syncwarp();
        EPI_T(3);
      }
      tc_fence_before();
#ifdef WAP_EPI_TRACE
      named_bar_sync(1, 128);
#else
      TW(3, named_bar_sync(1, 128));
#endif
#if defined(WAP_GEMM_TRACE) && !defined(WAP_EPI_TRACE)
      _tr[2] += clock64() - _drain0;
#endif
      if (wq == 0 && lane == 0) {
        if (CG == 2 && !leader) mbar_arrive_cluster(tempty_leader + acc * 8);
        else mbar_arrive(smem_u32(&tempty_bar[acc]));
      }
      if (++acc == C::ACC_BUFS) { acc = 0; acc_ph ^= 1; }
    }
    if (lane == 0) bulk_wait_all();
  } else if (PREC == 3 && warp >= 8) {
    // ---------------- 3xTF32 operand split (both CTAs) ----------------
    // kSplitGroups groups of 8 warps alternate stages. Within a group, warp
    // (q, half) owns TMEM lane quarter q = warp % 4 (the tcgen05 lane-access
    // rule) and k-columns [16*half, 16*half + 16); thread row ct = 32q + lane.
    const int sw = warp - 8;
    const int group = sw >> 3;  // 0 .. kSplitGroups-1
    const int half = (sw >> 2) & 1;
    const int ct = (warp & 3) * 32 + lane;
    const int gt = (sw & 7) * 32 + lane;  // thread index inside the group (0..255)
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t conv_leader = CG == 2 ? map_to_rank(smem_u32(&conv_bar[0]), 0) : smem_u32(&conv_bar[0]);
    // B's small half of a landed stage (PAIR2: only CTA 1, from its raw copy R into P)
    auto split_b = [&](uint8_t* base) {
      if constexpr (C::PAIR2) {
        if (rank == 1)
          split_small_only(reinterpret_cast<const uint32_t*>(base + C::A_OFF + C::P2_R),
                           reinterpret_cast<uint32_t*>(base + C::A_OFF), 64 * BK, gt, 256);
      } else {
        split_small_only(reinterpret_cast<const uint32_t*>(base + C::A_OFF),
                         reinterpret_cast<uint32_t*>(base + C::A_OFF + C::B_BYTES), C::B_ROWS * BK, gt, 256);
      }
    };
    int s = 0;
    uint32_t ph = 0;
    int it = 0;
    int wc = 0, wslot = 0;       // WIN: windows seen, current slot
    bool wwaited = false;        // WIN: this group has waited for the current window
    if constexpr (C::WSS) {
      // Window slot g belongs to group g: it waits for every landing of its slot (so its
      // parity waits never skip a phase), writes the small half of the whole window once,
      // and signals wsmall; per k-step a group only splits its B stage.
      const uint32_t wsmall_leader = CG == 2 ? map_to_rank(smem_u32(&wsmall_bar[0]), 0) : smem_u32(&wsmall_bar[0]);
      for (int t = cluster_id; t < n_tiles_total; t += n_clusters) {
        const TileCoord tc = decode_tile(g, t, BN, CG);
        int tap = tc.kc_begin % ntaps;
        for (int kc = tc.kc_begin; kc < tc.kc_end; ++kc, ++it, tap = tap + 1 == ntaps ? 0 : tap + 1) {
          if (tap == 0 || kc == tc.kc_begin) {
            const int ws = wc & 1;
            ++wc;
            if (ws == group) {
              TW(2, mbar_wait(smem_u32(&wfull_bar[ws]), ((wc - 1) >> 1) & 1));
              uint8_t* wraw = win_base + ws * win_slot;
              split_small_only(reinterpret_cast<const uint32_t*>(wraw), reinterpret_cast<uint32_t*>(wraw + win_bytes),
                               win_bytes / 4, gt, 256);
              fence_proxy_async_smem();
              TW(3, named_bar_sync(2 + group, 256));
              if (gt == 0) {
                if (CG == 2 && !leader) mbar_arrive_cluster(wsmall_leader + ws * 8);
                else mbar_arrive(smem_u32(&wsmall_bar[ws]));
              }
            }
          }
          if ((it % C::SG) == group) {
            TW(1, mbar_wait(smem_u32(&full_bar[s]), ph));
            uint8_t* base = smem + s * C::STAGE_BYTES;
            split_b(base);
            fence_proxy_async_smem();
            TW(3, named_bar_sync(2 + group, 256));
            if (gt == 0) {
              if (CG == 2 && !leader) mbar_arrive_cluster(conv_leader + s * 8);
              else mbar_arrive(smem_u32(&conv_bar[s]));
            }
          }
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
    } else
    for (int t = cluster_id; t < n_tiles_total; t += n_clusters) {
      const TileCoord tc = decode_tile(g, t, BN, CG);
      int tap = 0;  // WIN: tap of the current k-chunk (tap innermost), advanced without division
      if constexpr (WIN) tap = tc.kc_begin % ntaps;
      for (int kc = tc.kc_begin; kc < tc.kc_end; ++kc, ++it, tap = (WIN && tap + 1 == ntaps) ? 0 : tap + 1) {
        bool last_in_win = false;
        if constexpr (WIN) {
          if (tap == 0 || kc == tc.kc_begin) {
            wslot = wc & 1;
            ++wc;
            // every group observes every window phase, including windows it has no
            // step in (a one-step window at a split-K boundary), so its parity waits
            // never skip a phase
            TW(2, mbar_wait(smem_u32(&wfull_bar[wslot]), ((wc - 1) >> 1) & 1));
            wwaited = true;
          }
          last_in_win = (tap == ntaps - 1) || (kc == tc.kc_end - 1);
        }
        if ((it % C::SG) != group) {
          // observe this step's stage / A-slot phases (no work) so that the parity
          // waits of this group's own later steps never skip a phase
          if (!C::EVEN && (STAGES % C::SG != 0 || C::A_SLOTS % C::SG != 0)) {
            mbar_wait(smem_u32(&full_bar[s]), ph);
            mbar_wait(smem_u32(&aslot_bar[it % C::A_SLOTS]), ((it / C::A_SLOTS) & 1) ^ 1);
          }
          // this group's own steps of the window are done (each ended in a named barrier)
          if (WIN && last_in_win && gt == 0) mbar_arrive(smem_u32(&wempty_bar[wslot]));
          if (++s == STAGES) { s = 0; ph ^= 1; }
          continue;
        }
        TW(1, mbar_wait(smem_u32(&full_bar[s]), ph));
#ifdef WAP_GEMM_NO_SPLIT
        // diagnostic: skip the split work (TMA stream + handshakes only)
        named_bar_sync(2 + group, 256);
        if (gt == 0) {
          if (CG == 2 && !leader) mbar_arrive_cluster(conv_leader + s * 8);
          else mbar_arrive(smem_u32(&conv_bar[s]));
          if (WIN && last_in_win) mbar_arrive(smem_u32(&wempty_bar[wslot]));
        }
        if (++s == STAGES) { s = 0; ph ^= 1; }
        continue;
#endif
        uint8_t* base = smem + s * C::STAGE_BYTES;
        uint32_t v[16], w[16];
        if constexpr (WIN) {
          if (!wwaited) {
            TW(2, mbar_wait(smem_u32(&wfull_bar[wslot]), ((wc - 1) >> 1) & 1));
            wwaited = true;
          }
          // row ct of this tap's tile = window row ct + shift(tap) - min shift
          load_a_half_kmajor(win_base + wslot * win_slot, ct + s_off[0][tap] - g.win_off_min, half, v);
        } else if constexpr (A_MN) {
          load_a_half_mnmajor(base, ct, half, v);
        } else {
          load_a_half_kmajor(base, ct, half, v);
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint32_t big = v[j] & 0xFFFFE000u;
          w[j] = __float_as_uint(__uint_as_float(v[j]) - __uint_as_float(big));
          if constexpr (!C::A_SS) v[j] = big;
        }
#if WAP_B_SPLIT_EARLY
        // B's small half first: it needs no TMEM slot, so the only work left between the
        // slot wait (MMA completion of the slot's previous step) and this step's conv_bar
        // arrival is the A store
        split_b(base);
#endif
        // TMEM A slot of this step: free once the MMAs of its previous use committed
        const int aj = it % C::A_SLOTS;
        TW(2, mbar_wait(smem_u32(&aslot_bar[aj]), ((it / C::A_SLOTS) & 1) ^ 1));
        tc_fence_after();
        const uint32_t acol = tmem_base + lane_base + C::A_COL0 + aj * C::A_SLOT_W + half * 16;
#ifndef WAP_DIAG_NO_A_SPLIT
        if constexpr (C::A_SS) {
          tmem_st_32x32b_x16(acol, w);  // small only: the MMAs take big from the raw smem tile
        } else {
          tmem_st_32x32b_x16(acol, v);
          tmem_st_32x32b_x16(acol + 32, w);
        }
#endif
#if !WAP_B_SPLIT_EARLY
        split_b(base);
#endif
        TW(3, tmem_st_wait());
        tc_fence_before();
        fence_proxy_async_smem();
        // one arrival per CTA: group-local named barrier, then a single thread
        // signals (CTA-scope in the leader, cluster-scope release from the peer)
        TW(3, named_bar_sync(2 + group, 256));
        if (gt == 0) {
          if (CG == 2 && !leader) mbar_arrive_cluster(conv_leader + s * 8);
          else mbar_arrive(smem_u32(&conv_bar[s]));
          if (WIN && last_in_win) mbar_arrive(smem_u32(&wempty_bar[wslot]));
        }
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
  }
  TRACE_END();
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();
  if (warp == 2) tmem_dealloc_cg<CG>(tmem_base, C::TMEM_COLS);
}

// Deterministic split-K reduction: fixed slab order, then the epilogue.
__global__ void splitk_reduce_kernel(const GemmArgs g, int splits);

struct Plan {
  CUtensorMap tmA, tmB, tmC;
  GemmArgs args;
  int grid;
  int bn, a_mn, b_mn, prec, cg, splits, win;
};

constexpr int kMaxDynSmem = 227 * 1024;
constexpr int kExclusiveSmem = 120 * 1024;  // > half of the 228 KB per SM: one GEMM CTA per SM

// dynamic shared memory of one launch (WIN adds the two A halo windows)
template <int BN, int PREC, int CG, bool WIN>
constexpr int smem_bytes_for(int win_boxes) {
  return Cfg<BN, PREC, CG, WIN>::SMEM +
         (WIN ? 2 * win_boxes * Cfg<BN, PREC, CG, WIN>::A_BYTES * Cfg<BN, PREC, CG, WIN>::WIN_MUL : 0);
}

template <int BN, bool AMN, bool BMN, int PREC, int CG, bool WIN = false>
int launch(const Plan& p, cudaStream_t st) {
  using C = Cfg<BN, PREC, CG, WIN>;
  auto kern = gemm_tc_kernel<BN, AMN, BMN, PREC, CG, WIN>;
  static bool attr_set = false;
  if (!attr_set) {
    WAP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
    attr_set = true;
  }
  const int smem = smem_bytes_for<BN, PREC, CG, WIN>(p.args.win_boxes);
  if (smem > kMaxDynSmem) {
    wap_set_error("GEMM shared memory %d exceeds %d (window of %d boxes)", smem, kMaxDynSmem, p.args.win_boxes);
    return WAP_ENOTSUP;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(p.grid);
  cfg.blockDim = dim3(C::THREADS);
  // Every GEMM CTA claims more than half of an SM's shared memory, so two GEMM CTAs
  // (e.g. a dgrad and a wgrad on parallel streams) never share an SM. Each holds
  // all 512 TMEM columns (3xTF32) and a CTA pair syncs right after allocating:
  // co-resident pairs of two kernels could otherwise each hold one SM's TMEM while
  // waiting for their peer on the other SM (deadlock).
  cfg.dynamicSmemBytes = smem > kExclusiveSmem ? smem : kExclusiveSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  int na = 0;
  if (CG == 2) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    na = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  WAP_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, p.tmA, p.tmB, p.tmC, p.args));
  return WAP_OK;
}

// dispatch over the three major combinations used on the WAP path
template <int BN, int PREC, int CG>
int launch_majors(const Plan& p, cudaStream_t st) {
  if constexpr (PREC == 3) {
    if (p.win && !p.a_mn) {
      if (p.b_mn) return launch<BN, false, true, PREC, CG, true>(p, st);
      return launch<BN, false, false, PREC, CG, true>(p, st);
    }
  }
  if (!p.a_mn && p.b_mn) return launch<BN, false, true, PREC, CG>(p, st);
  if (!p.a_mn && !p.b_mn) return launch<BN, false, false, PREC, CG>(p, st);
  if (p.a_mn && p.b_mn) return launch<BN, true, true, PREC, CG>(p, st);
  wap_set_error("unsupported operand majors (A MN-major with B K-major)");
  return WAP_ENOTSUP;
}

int launch_prec1(const Plan& p, cudaStream_t st);
int launch_prec3(const Plan& p, cudaStream_t st);

}  // namespace wapgemm
