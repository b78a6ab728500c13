// tc.cu -- the tcgen05 engine of libtacsnn: ONE fused kernel per layer call that
// aggregates the K spike frames of a group (A_k = sum_j beta^{K-1-j} S_{kK+j},
// Definition TAC), convolves A_k once on the 5th-generation tensor
// cores (Alg. 1 l.4 / Alg. 2 l.4), and runs the LIF steps (Alg. 1 l.5-7, Alg. 2
// l.5-9, Eq. (1) for dense) with the membrane resident in registers across all
// T/K groups, writing packed (optionally 2x2 OR-pooled) spikes and spike counts.
//
// Exactness of the tensor-core operands:
//   * beta = 2^-m (DVS beta = 0.5) => A_k * 2^{m(K-1)} =
//     sum_j S_{kK+j} 2^{m j} is an exact unsigned integer <= 255 (u8 operand);
//     dense mode (K = 1) has A = S in {0,1} for any beta.
//   * W [C_out][C_in][3][3] fp32 is split per output channel into two int8
//     slices, w ~= s1 q1 + (s1/254) q2, |w - w~| <= max|w| * 1.55e-5; both
//     slices ride in ONE MMA with N = 2 C_out (hi rows on CTA 0, lo rows on CTA
//     1 of the pair), accumulated exactly in s32 in TMEM.
//   * the epilogue forms Y = 2^{-m(K-1)} s1 (D_hi + D_lo/254) + b in fp32.
//
// Tile = 16 output rows x 8 output columns of one sample per CTA (M = 128).
// Halo path (C_in a multiple of 32): the u8 aggregate of the 18 x 10 input halo
// is stored K-major without swizzle, one 16-byte row per halo pixel, halo rows
// 10 pixels apart.  A-operand row i = (g, c) = (i / 8, i % 8) of the tile is read
// at halo pixel (g + r, c + s) for tap (r, s): the 8 rows of a core matrix are
// 16 B apart and core-matrix groups (tile rows) SBO = 160 B apart, so a tap is
// a start-address offset of (10 r + s) * 16 B -- no im2col copies, no junk rows.
// Layers with C_in <= 8 (first layers) use the same halo scheme with 16 fp16
// channels per halo pixel and kind::f16 MMAs: the u8 aggregate (exact in fp16),
// the two fp16 slices of the weights (hi + lo, |error| <= 2^-22 |w|) accumulated
// into ONE fp32 accumulator, and the bias through a constant-1 channel that only
// the centre tap's weights read -- so the epilogue reads Y straight from TMEM.
// TMEM lane i = tile pixel (g, c): epilogue warp q holds tile rows 4q..4q+3, so
// every 2x2 pooling window lies inside one warp (lanes l, l^1, l^8, l^9) and
// spikes are OR-pooled with two shuffles and stored straight from registers.
//
// CTA pair (cluster of 2, tcgen05 cta_group::2, M = 256): each CTA owns one tile
// and half of the B operand (one int8 slice of all 9 taps, resident in smem for
// the whole kernel).  Warp roles per CTA (384 threads):
//   warp 0      : TMEM alloc; in CTA 0 one lane issues all MMAs of the pair
//   warps 1..3  : producers -- load packed spikes, build the u8 aggregate A_k
//   warps 4..11 : epilogue  -- TMEM -> registers, LIF over K steps, pooled /
//                 packed stores, bit-sliced spike counts, v_init / v_final
// Pipelines: A stages (2-3) producer -> MMA, TMEM accumulators (2) MMA -> epilogue.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "ptx.cuh"
#include "tc.cuh"

// host helpers below live in an anonymous namespace and are included by every
// translation unit that instantiates kernels; not all of them use every helper
#pragma GCC diagnostic ignored "-Wunused-function"

namespace tacsnn {

struct TcParams {
  CUtensorMap tmap;  // 4-D [T][B][H][WPR] u32 view of the input spikes (TMA producer), or
                     // 3-D [T][B][H*WPR] (plane mode: whole narrow frames, e.g. 28x28x1 = 112 B)
  int use_tma, raw_bw, nraw;  // use_tma: 0 LDG, 1 halo boxes, 2 whole planes (raw_bw = plane words)
  int warp_stage;             // 1: each producer warp builds whole A stages (stage it -> warp it % 3)
  int prod_refill;            // 1 (plane mode + warp_stage): the warp that consumed raw slot r refills it
  int occ;                    // CTA pairs per SM pair (1, or 2 for small first layers: OCC kernels)
  int c32w;                   // fp16 path, C_out 32: 4 epilogue warps x 32 channels (no atomic sub-word stores)
  int refill_early;           // 1: the MMA warp refills a consumed raw slot before issuing the group
  int sleep_ns;               // > 0: producers / MMA issuer poll their "free slot" barriers with
                              // nanosleep backoff (mbar_wait_sleep) instead of suspend-hint waits
  int prod_step;              // halo-row stride of the pixel-wise producers: 96, or 32 with warp_stage
  uint32_t off_raw, raw_stage_bytes, raw_box_bytes;
  int B, H, W, Cin, Cout, Cout_pad, pad, Ho, Wo, pool;
  int Hq, Wq;  // stored (pooled) extent: floor(H'/2), floor(W'/2) when pool == 2
  int K, G, nsteps, mode, reset;
  int tiles_x, tiles_y, num_tiles, num_pairs, nstages;
  int nkc, ntaps, m_shift;
  int wpr_in, wpr_out, nwo, int_combine;
  long long in_st, in_sb, out_st, out_sb;
  float decay, v_th, v_reset, agg_scale;
  uint32_t off_w, off_a, a_stage_bytes, off_scale, off_bar, smem_bytes;
  uint32_t w_bytes_cta, tmem_cols, n_total, lbo_a, sbo_a, lbo_b;
  int tap_off[9];
  int naccs;             // TMEM accumulators in the MMA -> epilogue ring
  int packed;            // fp16 path, C_in <= 3: hi and lo weight slices share one K=16 MMA
  int split;             // A carried as fp16 hi + lo from the 2^K-entry table lut
  int real;              // continuous input xin (A computed from fp32 frames, then hi + lo)
  const float *xin;      // fp32 [T][B][H][W][C_in], strides in_st / in_sb in floats
  float coef[16];        // A_k weights beta^{K-1-j} or alpha_j (fp32)
  uint32_t off_lut;      // smem copy of the aggregate tables (split path)
  const uint32_t *lut_g; // the tables in the prepared image (see tc_prepare)
  const uint32_t *in;
  uint32_t *out;
  const float *v_init;
  float *v_final;
  uint32_t *counts;
  const unsigned char *w_img;
  const float *scale_bias;
  float ysc, iysc;            // fp16 paths: the Y prescale 2^e and 2^-e (tc_prepare; host-side
                              // from the plan); 1 on int8
  float vth_s;                // v_th 2^e, precomputed so the reset FFMA2 reads it from the
                              // constant bank (no per-thread register, no FMUL)
  float *y_seq;               // training forward: per-group drive [G][B][Ho][Wo][Cout] (or NULL)
  long long yseq_plane;       // B * Ho * Wo * Cout
  unsigned long long *trace;  // optional: per-(group) role timestamps of CTA 0 (debug)
};

namespace {

// 3 producer warps: with 16 epilogue warps + the MMA warp the CTA has 20 warps, 5
// per SM sub-partition, which is what the per-SMSP register file (16 K regs) and
// the setmaxnreg budget below allow (a 21st warp would cap every warp at 80 regs).
constexpr int kProdWarps = 3;
#ifndef TACSNN_HALO_NR
#define TACSNN_HALO_NR 2  // halo producer pixels per pass (K <= 4)
#endif
#ifndef TACSNN_H16_PACK
#define TACSNN_H16_PACK 1
#endif
#ifndef TACSNN_BDESC_OPAQUE
#define TACSNN_BDESC_OPAQUE 1
#endif
#ifndef TACSNN_UT_PREFETCH
#define TACSNN_UT_PREFETCH 0  // 1: double-buffered TMEM loads in the U-in-TMEM loop (round 2: C5 L0 +0.9 %)
#endif
#ifndef TACSNN_REGS_LOW4
#define TACSNN_REGS_LOW4 64    // setmaxnreg of the MMA / producer warps (16 epilogue warps)
#endif
#ifndef TACSNN_REGS_HIGH4
#define TACSNN_REGS_HIGH4 104  // setmaxnreg of the 16 epilogue warps
#endif
#ifndef TACSNN_EPI_HIGH
#define TACSNN_EPI_HIGH 1  // 16-epilogue-warp kernels put the epilogue warps on the high warp ids (C5 L1 -0.9 %, L2 -0.5 %)
#endif
#ifndef TACSNN_EPI_HIGH2
#define TACSNN_EPI_HIGH2 0  // the same for the 8-epilogue-warp kernels (C3 L2 dense -3 %, TAC +1.5 %: off)
#endif
#ifndef TACSNN_UT_MIN_NS
#define TACSNN_UT_MIN_NS 4  // V in TMEM for the fp16 paths from this many LIF steps per group
#endif
#ifndef TACSNN_UT_UNROLL
#define TACSNN_UT_UNROLL 4  // chunks per unrolled body of the U-in-TMEM LIF loop (instruction footprint)
#endif
constexpr int kUtUnroll = TACSNN_UT_UNROLL;
#ifndef TACSNN_H16_ACCS
#define TACSNN_H16_ACCS 3  // TMEM accumulators on the fp16 paths (2 or 3)
#endif
#ifndef TACSNN_UNIFORM_WARP
#define TACSNN_UNIFORM_WARP 1
#endif
#ifndef TACSNN_HALO_MAP
#define TACSNN_HALO_MAP 1  // 1: 8-thread groups own consecutive pixels of one word
#endif
// Warp layout: epilogue warps first (NPART channel parts x 4 TMEM lane quadrants),
// then the MMA warp, then the producer warps.  The SM warp schedulers favour
// higher warp ids, so the warps feeding the tensor pipe (MMA, producers) win
// issue slots over the 16 compute-heavy epilogue warps.
constexpr int epi_warps(int npart) { return 4 * npart; }
// OCC = 2 kernels with 4 epilogue warps (the rate-coded first layers, C_out 32) carry 2
// more producer warps: their row producer builds a whole A stage in one warp and limits
// the group period (scripts/trace_layer.py: 1.6 us per stage, 0.67 us per group), so 5
// warps rotating the stages keep more of them in flight (C3 L1 TAC K=8 75.7 -> 72.4 us,
// C2 L1 -3 %; 4 extra warps cap the registers at 80 and gain nothing).  The extra warps only
// join the one-warp-per-stage (warp_stage) producers; the pixel-wise producers use 3.
#ifndef TACSNN_EXTRA_PW
#define TACSNN_EXTRA_PW 2
#endif
constexpr int extra_prod_warps(int npart, int occ) { return (npart == 1 && occ == 2) ? TACSNN_EXTRA_PW : 0; }
constexpr int kernel_threads(int npart, int occ = 1) {
  return 32 * (1 + kProdWarps + extra_prod_warps(npart, occ) + epi_warps(npart));
}
// A stages / TMEM accumulators: 3 / 2 (int8), 3 / 3 (fp16, C_out 128); the small first
// layers (pixel-wise producers, C_out <= 64) run deeper rings -- their per-group work is
// short, so the producer -> MMA -> epilogue round trip, not any role's busy time, sets
// the period unless more groups are in flight (scripts/trace_layer.py)
constexpr int kMaxStages = 8;
constexpr int kAccs = 6;  // max TMEM accumulators (p.naccs)
constexpr int kMaxSteps = 8;
constexpr int kPlanes = 6;  // bit-sliced spike counters (<= 63 steps per flush)
constexpr int kTileH = 16, kTileW = 8;                 // output pixels per CTA tile
constexpr int kHaloH = kTileH + 2, kHaloW = kTileW + 2;  // 3x3 halo
constexpr int kHaloRows = kHaloH * kHaloW;              // 180 halo pixels
constexpr uint32_t kSmemLimit = 232448;

// int8 halo (C_in % 32 == 0) | fp16 halo (C_in <= 8) | fp16 halo with the split A_hi + A_lo
// aggregate (kernel template only: the host geometry of PATH_SPLIT is that of PATH_H16)
enum { PATH_HALO = 0, PATH_H16 = 1, PATH_SPLIT = 2 };


// trace slots per group iteration (CTA 0 only).  Compiled in only when the library
// is built with -DTACSNN_TRACE (TACSNN_TRACE=1 python -m paper_2603_13810_b200.build
// --force); otherwise trace_mark is empty and costs nothing in the hot loops.
enum { TR_PROD_START = 0, TR_PROD_DONE, TR_MMA_READY, TR_MMA_ISSUED, TR_EPI_FULL, TR_EPI_RELEASED,
       TR_EPI_DONE, TR_PROD_RAW, TR_PROD_ISSUED, TR_MMA_AFULL, TR_MMA_REFILLED,
       TR_P1_START, TR_P1_DONE, TR_P1_RAW, TR_SLOTS = 16 };
__device__ __forceinline__ void trace_mark(const TcParams &p, uint32_t it, int slot) {
#ifdef TACSNN_TRACE
  // CTA 0 records every role; CTA 1 (the pair's other CTA) its producers' events
  const int sl = blockIdx.x == 0 ? slot
                 : (blockIdx.x == 1 && slot == TR_PROD_START) ? TR_P1_START
                 : (blockIdx.x == 1 && slot == TR_PROD_DONE) ? TR_P1_DONE
                 : (blockIdx.x == 1 && slot == TR_PROD_RAW) ? TR_P1_RAW : -1;
  if (p.trace && sl >= 0 && it < 4096) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.trace[it * TR_SLOTS + sl] = t;
  }
#else
  (void)p;
  (void)it;
  (void)slot;
#endif
}

// ------------------------------------------------------------ host helpers --
int beta_shift(float beta) {  // m with beta == 2^-m exactly, else 0
  int e;
  const double mant = std::frexp((double)beta, &e);
  if (mant != 0.5) return 0;
  const int m = 1 - e;
  return m >= 1 ? m : 0;
}

int cout_pad_of(int Cout) {
  if (Cout <= 16) return 16;
  if (Cout <= 32) return 32;
  if (Cout <= 64) return 64;
  return 128;
}

// Split-A (fp16) aggregate: when A_k = sum_j beta^{K-1-j} S_{kK+j} is not an exact
// small integer (beta != 2^-m, e.g. the rate-coded configs' beta = 0.9, or
// m (K-1) > 7), A is carried as two fp16 values A_hi + A_lo (|A - A_hi - A_lo| <=
// 2^-22 |A|) looked up from a 2^K-entry table of the K spike bits of a channel,
// and both ride the fp16 tensor-core path as extra K channels.
constexpr bool templ_k(int K);
bool split_of(const tac_conv_lif_desc *d) {
  if (d->input_kind == TAC_INPUT_REAL) return true;  // continuous input: A is any real
  if (d->mode == TAC_MODE_DENSE) return false;
  if (d->agg_weights) return true;                   // learnable alpha_j: any real
  if (d->K <= 1) return false;
  // a group size without a templated exact producer runs the runtime-K table producer
  // (exact values are exact table entries too); first layers only (envelope)
  if (!templ_k(d->K) && d->C_in <= 2) return true;
  const int m = beta_shift(d->beta);
  return m == 0 || m * (d->K - 1) > 7;
}
// Aggregate tables of the split path: K <= 8: 2^K entries fp16 A_hi | A_lo << 16 indexed
// by the K spike bits of a channel (bit j = frame j); 8 < K <= 16 (first layers, C_in <= 2):
// two fp32 tables, frames 0..K-9 and K-8..K-1, summed in fp32 and split in the producer.
constexpr int kMaxSplitK = 16;
constexpr int kLutWords = 3 << 8;  // [fp16-pair table | fp32 table A | fp32 table B]
// group sizes the templated producers are instantiated for; other K <= 16 run the
// runtime-K split producer (C_in <= 2)
constexpr bool templ_k(int K) { return K == 1 || K == 2 || K == 3 || K == 4 || K == 8; }

int path_of(const tac_conv_lif_desc *d) {
  if (split_of(d)) return PATH_H16;  // (kernel template PATH_SPLIT)
  return (d->C_in % 32 == 0) ? PATH_HALO : PATH_H16;
}


// 16-B K chunks (8 fp16 channels) per halo pixel of the fp16 path: channels
// [A (C_in) | bias 1.0] or, split, [A_hi (C_in) | A_lo (C_in) | bias 1.0]; even
// so that every MMA has K = 16.
int h16_chunks(const tac_conv_lif_desc *d) {
  const int ch = split_of(d) ? 2 * d->C_in + 1 : d->C_in + 1;
  const int nck = (ch + 7) / 8;
  return nck < 2 ? 2 : (nck + 1) / 2 * 2;
}

// fp16 path with both weight slices in one K = 16 MMA per tap (C_in + 1 <= 4 channels each)
// (split aggregate: [A_hi | A_lo | 1 | A_hi | 1] x [W_hi | W_hi | b_hi | W_lo | b_lo], C_in <= 2)
bool packed_of(const tac_conv_lif_desc *d) {
  if (!TACSNN_H16_PACK || path_of(d) != PATH_H16) return false;
  return split_of(d) ? d->C_in <= 2 : d->C_in <= 3;
}

struct Geometry {
  int path, split, nkc, ntaps, cout_pad, nsteps, nstages, use_tma, nraw, raw_bw;
  uint32_t w_bytes_cta, a_stage_bytes, raw_stage_bytes, raw_box_bytes, off_w, off_a, off_raw,
      off_scale, off_lut, off_bar, smem_bytes;
};
constexpr int kMaxRaw = 8;  // raw (TMA) stages: 4 for halo boxes, up to 8 tiny plane boxes
constexpr int kNumBars = 2 * kMaxStages + 2 * kAccs + 1 + 2 * kMaxRaw;

uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

// Shared-memory plan.  With use_tma the producers aggregate from a TMA-loaded
// raw halo ([K][18][raw_bw] u32 per stage) instead of loading from global.
// the row producers (produce_plane_rows / produce_halo_rows) take this layer: C_in <= 2,
// a templated K <= 8, spike input, and a table (split) or an exact beta = 1/2 / dense aggregate
bool rows_ok(const tac_conv_lif_desc *d) {
  const int K = d->mode == TAC_MODE_DENSE ? 1 : d->K;
  const bool exact_m1 = d->mode == TAC_MODE_DENSE || K == 1 || beta_shift(d->beta) == 1;
  return path_of(d) != PATH_HALO && d->C_in <= 2 && templ_k(K) && K <= 8 && d->input_kind == TAC_INPUT_SPIKES &&
         (split_of(d) || exact_m1);
}

Geometry geometry(const tac_conv_lif_desc *d, bool use_tma = false, int plane_words = 0) {
  Geometry g{};
  g.path = path_of(d);
  g.split = split_of(d) ? 1 : 0;
  g.cout_pad = cout_pad_of(d->C_out);
  const int K = d->mode == TAC_MODE_DENSE ? 1 : d->K;
  g.nsteps = d->mode == TAC_MODE_TACTP ? K : 1;
  if (g.path == PATH_HALO) {
    g.nkc = d->C_in / 16;
    g.ntaps = 9;
    g.w_bytes_cta = 9u * d->C_in * g.cout_pad;
    g.a_stage_bytes = align_up((uint32_t)kHaloRows * d->C_in, 128);
    // TMA box start is aligned down to 16 B (4 words): up to 3 extra words in front
    const int nwin = d->C_in / 32;
    g.raw_bw = nwin == 4 ? kHaloW * 4 : (int)align_up(kHaloW * nwin + 3, 4);
  } else {
    g.nkc = h16_chunks(d);                  // 16-B K chunks per halo pixel
    g.ntaps = 9;
    // [hi/lo slice][tap][chunk][C_out_pad/2 rows][16 B] per CTA
    g.w_bytes_cta = 144u * g.nkc * g.cout_pad;
    g.a_stage_bytes = align_up((uint32_t)kHaloRows * 16u * g.nkc, 128);
    // C_in <= 8: 16-B aligned start word + the <= 3 words holding 10 px x C_in bits;
    // C_in = 32: one word per pixel as in the int8 halo path
    g.raw_bw = d->C_in >= 32 ? (int)align_up(kHaloW * (d->C_in / 32) + 3, 4) : 8;
  }
  if (plane_words > 0) g.raw_bw = plane_words;  // plane mode: K whole frames per stage
  g.raw_box_bytes = (uint32_t)K * (plane_words > 0 ? 1 : kHaloH) * g.raw_bw * 4u;
  g.raw_stage_bytes = align_up(g.raw_box_bytes, 128);
  // pixel-wise producers (plane mode or LDG, fp16 paths) try deeper A rings first
  const bool deep = g.path != PATH_HALO && (plane_words > 0 || !use_tma || rows_ok(d));
  const int combos[11][2] = {{8, 8}, {8, 4}, {6, 4}, {4, 4}, {3, 4}, {3, 3}, {3, 2}, {2, 2}, {3, 1}, {2, 1}, {2, 0}};
  for (int ci = deep ? 0 : 4; ci < 11; ++ci) {
    g.nstages = combos[ci][0];
    g.nraw = use_tma ? combos[ci][1] : 0;
    g.off_w = 0;
    g.off_a = align_up(g.w_bytes_cta, 1024);
    g.off_raw = align_up(g.off_a + g.nstages * g.a_stage_bytes, 128);
    g.off_scale = align_up(g.off_raw + g.nraw * g.raw_stage_bytes, 128);
    g.off_lut = align_up(g.off_scale + 4u * g.cout_pad * 4u, 16);
    g.off_bar = align_up(g.off_lut + (g.split ? 4u * kLutWords : 0u), 64);  // split: aggregate tables
    g.smem_bytes = g.off_bar + 8u * kNumBars + 16u;
    if (g.smem_bytes <= kSmemLimit) break;
  }
  g.use_tma = use_tma && g.smem_bytes <= kSmemLimit;
  return g;
}

const char *shape_reason(const tac_conv_lif_desc *d) {
  if (d->R != 3 || d->S != 3) return "needs a 3x3 kernel";
  if (d->stride != 1) return "needs stride 1";
  if (d->pad < 0 || d->pad > 1) return "needs pad 0 or 1";
  if (!((d->C_in % 32 == 0 && d->C_in <= 128) || d->C_in <= 8))
    return "needs C_in <= 8 or a multiple of 32 up to 128";
  if (d->C_out > 128 || !(d->C_out % 32 == 0 || d->C_out == 8 || d->C_out == 16))
    return "needs C_out in {8,16} or a multiple of 32 up to 128";
  const int K = d->mode == TAC_MODE_DENSE ? 1 : d->K;
  if (d->mode == TAC_MODE_TACTP && K > kMaxSteps) return "TAC-TP needs K <= 8";
  if (K > kMaxSplitK) return "needs K <= 16";
  return nullptr;
}

const char *reason(const tac_conv_lif_desc *d) {
  const char *r = shape_reason(d);
  if (r) return r;
  if (d->input_kind == TAC_INPUT_REAL && d->C_in > 2) return "continuous input needs C_in <= 2";
  const int K = d->mode == TAC_MODE_DENSE ? 1 : d->K;
  if (split_of(d)) {
    if (!(d->C_in <= 2 || d->C_in == 32))
      return "split (beta != 2^-m, learnable or continuous) aggregate needs C_in in {1, 2, 32}";
    // any K <= 16 on the first layers (runtime-K producer); the producers are instantiated
    // for K in {1, 2, 3, 4, 8} (3: short last groups, e.g. T = 7, K = 4)
    if (d->C_in == 32 && !templ_k(K)) return "split aggregate with C_in = 32 needs K in {1, 2, 3, 4, 8}";
  } else if (!templ_k(K)) {
    return "needs K in {1, 2, 3, 4, 8} (or a split aggregate on C_in <= 2 with K <= 16)";
  }
  if (geometry(d).smem_bytes > kSmemLimit) return "shared-memory footprint exceeds 227 KB";
  return nullptr;
}

// ------------------------------------------------------------ device code ---
__device__ __forceinline__ void tile_origin(const TcParams &p, int tile, int &b, int &y0, int &x0,
                                            bool &ok) {
  const int per = p.tiles_y * p.tiles_x;
  b = tile / per;
  const int rem = tile - b * per;
  const int ty = rem / p.tiles_x;
  y0 = ty * kTileH;
  x0 = (rem - ty * p.tiles_x) * kTileW;
  ok = tile < p.num_tiles;
}

// origin of one output tile: sample, first output row / column, tile in range
struct TileXY {
  int b, y0, x0;
  bool ok;
};

// Tiles t0, t0 + dt, t0 + 2 dt, ... as (sample, tile row, tile column), advanced
// incrementally: the persistent role loops carry no integer division per tile.
struct TileWalk {
  int b, ty, tx, db, dty, dtx;
  __device__ __forceinline__ TileWalk(const TcParams &p, int t0, int dt) {
    const int per = p.tiles_x * p.tiles_y;
    b = t0 / per;
    ty = (t0 - b * per) / p.tiles_x;
    tx = t0 - b * per - ty * p.tiles_x;
    db = dt / per;
    dty = (dt - db * per) / p.tiles_x;
    dtx = dt - db * per - dty * p.tiles_x;
  }
  __device__ __forceinline__ TileXY at(const TcParams &p, int tile) const {
    return TileXY{b, ty * kTileH, tx * kTileW, tile < p.num_tiles};
  }
  __device__ __forceinline__ void step(const TcParams &p) {
    tx += dtx;
    int cy = tx >= p.tiles_x;
    tx -= cy ? p.tiles_x : 0;
    ty += dty + cy;
    cy = ty >= p.tiles_y;
    ty -= cy ? p.tiles_y : 0;
    b += db + cy;
  }
};

// wait used by roles that normally run ahead of the epilogue (see ptx::mbar_wait_sleep)
__device__ __forceinline__ void wait_ahead(const TcParams &p, uint32_t bar, uint32_t parity) {
  if (p.sleep_ns > 0)
    ptx::mbar_wait_sleep(bar, parity, (uint32_t)p.sleep_ns);
  else
    ptx::mbar_wait(bar, parity);
}

// circular-buffer position (slot, phase parity) advanced by one per use: no integer
// division by the runtime ring sizes in the role loops
struct Ring {
  uint32_t i = 0, ph = 0;
  __device__ __forceinline__ void next(uint32_t n) {
    if (++i == n) {
      i = 0;
      ph ^= 1u;
    }
  }
};

// --- producers: build the u8 aggregate A_k * 2^{m(K-1)} in the MMA layout ---
// byte b of output word q <- input channel (q + 8b) of a 32-channel word; bit
// e_j = m*j of that byte <- frame j (weights 2^{m j}, oldest frame = 1)
template <int K>
__device__ __forceinline__ void agg_word_k(uint32_t (&o)[8], const uint32_t *xj, int m) {
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const uint32_t x = xj[j];
    const int e = m * j;
#pragma unroll
    for (int q = 0; q < 8; ++q) o[q] |= ((x >> q) & 0x01010101u) << e;
  }
}

// Halo producer: the thread owns 32-channel word w of halo pixels row0, row0 +
// rstep, ... (96 % nwin == 0).  Loads are issued in batches of RB pixels x K
// frames before any is consumed, so one memory round trip covers RB pixels.
template <int K>
__device__ __forceinline__ void produce_halo(const TcParams &p, const TileXY &tile, int k, uint32_t a_stage,
                                             int ptid) {
  constexpr int RB = K >= 8 ? 2 : (K >= 4 ? 4 : 8);
  const int nwin = p.Cin >> 5;
  // groups of 8 consecutive threads own 8 consecutive halo pixels of one 32-channel
  // word w: their 16-B A-stage stores are contiguous (no bank conflicts) and their
  // raw-halo loads (pixel stride nwin words, 4 words in a group) hit distinct banks
  const int g8 = ptid >> 3, w = g8 % nwin, row0 = (g8 / nwin) * 8 + (ptid & 7);
  const int rstep = (kProdWarps * 32) / nwin;
  const int b = tile.b, y0 = tile.y0, x0 = tile.x0;
  const bool tok = tile.ok;
  const uint32_t *frame0 = p.in + (long long)(k * K) * p.in_st + (long long)b * p.in_sb + w;
  const long long in_st = p.in_st;
  const int mshift = p.m_shift;
  const int nrows = row0 < kHaloRows ? (kHaloRows - row0 + rstep - 1) / rstep : 0;
  for (int ib = 0; ib < nrows; ib += RB) {
    uint32_t xs[RB][K];
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      const int row = row0 + (ib + r) * rstep;
      const int hy = row / kHaloW, hx = row - (row / kHaloW) * kHaloW;
      const int yi = y0 + hy - p.pad, xi = x0 + hx - p.pad;
      const bool ok = tok && ib + r < nrows && yi >= 0 && yi < p.H && xi >= 0 && xi < p.W;
      const uint32_t *src = frame0 + (long long)yi * p.wpr_in + xi * nwin;
#pragma unroll
      for (int j = 0; j < K; ++j) xs[r][j] = ok ? __ldg(src + j * in_st) : 0u;
    }
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      if (ib + r < nrows) {
        uint32_t o[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        agg_word_k<K>(o, xs[r], mshift);
        const int row = row0 + (ib + r) * rstep;
        const uint32_t dst = a_stage + (uint32_t)(2 * w) * p.lbo_a + (uint32_t)row * 16u;
        ptx::st_shared_v4(dst, o[0], o[1], o[2], o[3]);
        ptx::st_shared_v4(dst + p.lbo_a, o[4], o[5], o[6], o[7]);
      }
    }
  }
}

// --- fp16 halo (C_in <= 8) ---------------------------------------------------
// A halo pixel is a 32-byte K-major row of 16 fp16 channels: the u8 aggregate of
// channels 0..C_in-1, 1.0 at channel C_in (read only by the centre tap's bias
// weights), zeros above.  Bytes are built first (channel c <- byte c of lo/hi)
// and converted exactly: fp16 bits 0x64nn = 1024 + n, minus 1024.
__device__ __forceinline__ void h16_bias_slot(int Cin, uint32_t &lo, uint32_t &hi, uint32_t &c8) {
  lo = Cin < 4 ? 1u << (8 * Cin) : 0u;
  hi = (Cin >= 4 && Cin < 8) ? 1u << (8 * (Cin - 4)) : 0u;
  c8 = Cin == 8 ? 0x3C00u : 0u;  // fp16 1.0 in channel 8 (chunk 1)
}

// spike bits (channel c = bit c, c < 8) of frame weight 2^e -> bytes of lo / hi
__device__ __forceinline__ void h16_acc(uint32_t &lo, uint32_t &hi, uint32_t bits, int e) {
  lo |= (((bits & 0xFu) * 0x204081u) & 0x01010101u) << e;  // bit i -> byte i
  hi |= ((((bits >> 4) & 0xFu) * 0x204081u) & 0x01010101u) << e;
}

// packed slices (C_in <= 3): the C_in + 1 bytes [A | 1] of lo repeated right after
// themselves, so K channels [A | 1 | A | 1] meet [W_hi | b_hi | W_lo | b_lo]
__device__ __forceinline__ void h16_pack_slices(uint32_t &lo, uint32_t &hi, int Cin) {
  uint64_t v = lo;
  v |= v << (8 * (Cin + 1));
  lo = (uint32_t)v;
  hi = (uint32_t)(v >> 32);
}

__device__ __forceinline__ uint32_t u8x2_to_f16x2(uint32_t bytes, uint32_t sel) {
  uint32_t h = __byte_perm(bytes, 0x64646464u, sel), r;
  asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(h), "r"(0x64006400u));
  return r;
}

__device__ __forceinline__ void store_h16_row(uint32_t dst, uint32_t lbo, uint32_t lo, uint32_t hi,
                                              uint32_t c8) {
  ptx::st_shared_v4(dst, u8x2_to_f16x2(lo, 0x5140u), u8x2_to_f16x2(lo, 0x7362u),
                    u8x2_to_f16x2(hi, 0x5140u), u8x2_to_f16x2(hi, 0x7362u));
  ptx::st_shared_v4(dst + lbo, c8, 0u, 0u, 0u);
}

// Source of the pixel-wise producers: packed frames in global memory (LDG, frame stride
// in_st) or, in plane mode, the group's K whole frames staged in shared memory by TMA
// (frame stride = plane words); the indexing is the same.
template <bool SMEM>
__device__ __forceinline__ uint32_t ld_src(const uint32_t *a) {
  if constexpr (SMEM) return *a;
  else return __ldg(a);
}

// LDG fallback: one halo pixel per thread and pass; the C_in <= 8 bits of pixel
// xi start at row bit xi * C_in and straddle at most two words.
template <int K, bool SMEM = false>
__device__ __forceinline__ void produce_h16(const TcParams &p, const TileXY &tile, int k, uint32_t a_stage,
                                            int ptid, const uint32_t *plane = nullptr) {
  const int b = tile.b, y0 = tile.y0, x0 = tile.x0;
  const bool tok = tile.ok;
  const int Cin = p.Cin;
  const uint32_t cmask = (1u << Cin) - 1u;
  uint32_t one_lo, one_hi, c8;
  h16_bias_slot(Cin, one_lo, one_hi, c8);
  const uint32_t *frame0 = SMEM ? plane : p.in + (long long)(k * K) * p.in_st + (long long)b * p.in_sb;
  const long long fst = SMEM ? (long long)p.raw_bw : p.in_st;
  for (int row = ptid; row < kHaloRows; row += p.prod_step) {
    const int hy = row / kHaloW, hx = row - (row / kHaloW) * kHaloW;
    const int yi = y0 + hy - p.pad, xi = x0 + hx - p.pad;
    const bool ok = tok && yi >= 0 && yi < p.H && xi >= 0 && xi < p.W;
    const int bit = ok ? xi * Cin : 0, sh = bit & 31;
    const bool two = ok && sh + Cin > 32;
    const uint32_t *src = frame0 + (long long)(ok ? yi : 0) * p.wpr_in + (bit >> 5);
    uint32_t w0[K], w1[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      w0[j] = ok ? ld_src<SMEM>(src + (long long)j * fst) : 0u;
      w1[j] = two ? ld_src<SMEM>(src + (long long)j * fst + 1) : 0u;
    }
    uint32_t lo = one_lo, hi = one_hi;
#pragma unroll
    for (int j = 0; j < K; ++j) h16_acc(lo, hi, __funnelshift_r(w0[j], w1[j], sh) & cmask, p.m_shift * j);
    if (p.packed) h16_pack_slices(lo, hi, Cin);
    store_h16_row(a_stage + (uint32_t)row * 16u, p.lbo_a, lo, hi, c8);
  }
}

// d | (a & b) in one LOP3
__device__ __forceinline__ uint32_t and_or(uint32_t a, uint32_t b, uint32_t d) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(a), "r"(b), "r"(d));
  return r;
}

// beta = 1/2 aggregate by SWAR bit interleaving (K = 2, 4, 8): byte b of o[q] =
// sum_j 2^j bit(x_j, q + 8b).  Frames are paired into 2-bit fields (e: even
// channels, f: odd), pairs into 4-bit fields per channel class c % 4 (n[r]), and
// nibbles split into bytes: 28 ops per 32-channel word for K = 4 instead of 64.
__device__ __forceinline__ uint32_t bsel(uint32_t m, uint32_t a, uint32_t b) {  // (a & m) | (b & ~m)
  return (a & m) | (b & ~m);
}
__device__ __forceinline__ void pair_fields(uint32_t x0, uint32_t x1, uint32_t &e, uint32_t &f) {
  e = bsel(0x55555555u, x0, x1 << 1);  // channel 2i   -> bits 2i, 2i+1 = (x0, x1)
  f = bsel(0x55555555u, x0 >> 1, x1);  // channel 2i+1 -> bits 2i, 2i+1
}
// 4 frames -> nibble words: n[r] holds channel 4k + r at bits 4k..4k+3
__device__ __forceinline__ void quad_fields(const uint32_t *x, uint32_t (&n)[4]) {
  uint32_t e, f, g, h;
  pair_fields(x[0], x[1], e, f);
  pair_fields(x[2], x[3], g, h);
  n[0] = bsel(0x33333333u, e, g << 2);
  n[2] = bsel(0x33333333u, e >> 2, g);
  n[1] = bsel(0x33333333u, f, h << 2);
  n[3] = bsel(0x33333333u, f >> 2, h);
}
template <int K>
__device__ __forceinline__ void agg_word_swar(uint32_t (&o)[8], const uint32_t (&xj)[K]) {
  static_assert(K == 2 || K == 4 || K == 8, "SWAR aggregate: K in {2, 4, 8}");
  if constexpr (K == 2) {
    uint32_t e, f;
    pair_fields(xj[0], xj[1], e, f);
#pragma unroll
    for (int q = 0; q < 8; q += 2) {
      o[q] = (e >> q) & 0x03030303u;
      o[q + 1] = (f >> q) & 0x03030303u;
    }
  } else {
    uint32_t n[4];
    quad_fields(xj, n);
    if constexpr (K == 8) {
      uint32_t m[4];
      quad_fields(xj + 4, m);
#pragma unroll
      for (int r = 0; r < 4; ++r) {  // frames 0-3 in the low nibble, 4-7 in the high one
        o[r] = bsel(0x0F0F0F0Fu, n[r], m[r] << 4);
        o[r + 4] = bsel(0x0F0F0F0Fu, n[r] >> 4, m[r]);
      }
    } else {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        o[r] = n[r] & 0x0F0F0F0Fu;
        o[r + 4] = (n[r] >> 4) & 0x0F0F0F0Fu;
      }
    }
  }
}

// o[q] (channels q + 8b at byte b) |= frame bit << e with a compile-time frame
// shift e = j (beta = 1/2, or K = 1): one SHF + one LOP3 per (q, frame)
template <int K>
__device__ __forceinline__ void agg_word_m1(uint32_t (&o)[8], const uint32_t (&xj)[K]) {
  if constexpr (K == 2 || K == 4 || K == 8) {
    agg_word_swar<K>(o, xj);
    return;
  }
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const uint32_t mask = 0x01010101u << j;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t t = (q >= j) ? (xj[j] >> (q - j)) : (xj[j] << (j - q));
      o[q] = and_or(t, mask, o[q]);
    }
  }
}

// --- split-A fp16 rows (beta != 2^-m): A_hi / A_lo from the table ---------------
// K-bit table index of one channel: bit j <- channel bit c of frame j
template <int K>
__device__ __forceinline__ uint32_t frame_index(const uint32_t (&bits)[K], int c) {
  uint32_t idx = 0;
#pragma unroll
  for (int j = 0; j < K; ++j) idx |= ((bits[j] >> c) & 1u) << j;
  return idx;
}
// chunk 0 of a C_in <= 2 split row: [A_hi(0..CIN-1) | A_lo(0..CIN-1) | 1.0 | 0 ...]
// e_c = fp16 A_hi | fp16 A_lo << 16 of channel c -> chunk 0 of a split row; packed:
// [A_hi | A_lo | 1 | A_hi | 1] (both weight slices in one MMA), else [A_hi | A_lo | 1]
template <int CIN>
__device__ __forceinline__ uint4 split_row_words(uint32_t e0, uint32_t e1, bool packed) {
  if (CIN == 1)
    return packed ? make_uint4(e0, 0x3C00u | (e0 << 16), 0x3C00u, 0u) : make_uint4(e0, 0x3C00u, 0u, 0u);
  const uint32_t his = __byte_perm(e0, e1, 0x5410u), los = __byte_perm(e0, e1, 0x7632u);
  return packed ? make_uint4(his, los, 0x3C00u | (e0 << 16), (e1 & 0xFFFFu) | 0x3C000000u)
                : make_uint4(his, los, 0x3C00u, 0u);
}
template <int K, int CIN>
__device__ __forceinline__ uint4 split_row_small(const uint32_t (&bits)[K], const uint32_t *lut, bool packed) {
  const uint32_t e0 = lut[frame_index<K>(bits, 0)];
  const uint32_t e1 = CIN == 2 ? lut[frame_index<K>(bits, 1)] : 0u;
  return split_row_words<CIN>(e0, e1, packed);
}
// C_in = 32 split row: 8 index words (byte b of o[q] = channel q + 8b) -> chunks
// 0..3 A_hi, 4..7 A_lo, 8 = {1.0, 0 ...}, 9 = 0
__device__ __forceinline__ void store_split32_row(uint32_t dst, uint32_t lbo, const uint32_t (&o)[8],
                                                  const uint32_t *lut) {
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    uint32_t e[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) e[q] = lut[(o[q] >> (8 * b)) & 0xFFu];
    ptx::st_shared_v4(dst + b * lbo, __byte_perm(e[0], e[1], 0x5410u), __byte_perm(e[2], e[3], 0x5410u),
                      __byte_perm(e[4], e[5], 0x5410u), __byte_perm(e[6], e[7], 0x5410u));
    ptx::st_shared_v4(dst + (4 + b) * lbo, __byte_perm(e[0], e[1], 0x7632u), __byte_perm(e[2], e[3], 0x7632u),
                      __byte_perm(e[4], e[5], 0x7632u), __byte_perm(e[6], e[7], 0x7632u));
  }
  ptx::st_shared_v4(dst + 8 * lbo, 0x3C00u, 0u, 0u, 0u);
  ptx::st_shared_v4(dst + 9 * lbo, 0u, 0u, 0u, 0u);
}

// Runtime group size (any K <= 16; split path, C_in <= 2): the K-bit index of a channel
// is gathered frame by frame; K <= 8 reads the fp16-pair table, 8 < K <= 16 adds the two
// fp32 half tables (frames 0..K-9 | K-8..K-1) and splits the sum into fp16 hi + lo
// (|A - A_hi - A_lo| <= 2^-22 |A| + fp32 rounding of the table sum).
__device__ __forceinline__ uint32_t f32_to_h16pair(float a) {
  const __half hi = __float2half_rn(a);
  const __half lo = __float2half_rn(a - __half2float(hi));
  return (uint32_t)__half_as_ushort(hi) | ((uint32_t)__half_as_ushort(lo) << 16);
}
__device__ __forceinline__ uint32_t split_lookup(uint32_t idx, int K, const uint32_t *lut) {
  if (K <= 8) return lut[idx];
  const int ka = K - 8;
  return f32_to_h16pair(__uint_as_float(lut[256 + (idx & ((1u << ka) - 1u))]) +
                        __uint_as_float(lut[512 + (idx >> ka)]));
}

// continuous-input producer (input_kind REAL, C_in <= 2): A_c = sum_j beta^{K-1-j}
// X_{kK+j, c} in fp32 (the oracle's order), then the same [A_hi | A_lo | 1.0] row as
// the split path
template <int K, int CIN>
__device__ __forceinline__ void produce_h16x(const TcParams &p, const TileXY &tile, int k, uint32_t a_stage,
                                             int ptid) {
  const int b = tile.b, y0 = tile.y0, x0 = tile.x0;
  const bool tok = tile.ok;
  const float *frame0 = p.xin + (long long)(k * (K ? K : p.K)) * p.in_st + (long long)b * p.in_sb;
  for (int row = ptid; row < kHaloRows; row += p.prod_step) {
    const int hy = row / kHaloW, hx = row - (row / kHaloW) * kHaloW;
    const int yi = y0 + hy - p.pad, xi = x0 + hx - p.pad;
    const bool ok = tok && yi >= 0 && yi < p.H && xi >= 0 && xi < p.W;
    const float *src = frame0 + ((long long)(ok ? yi : 0) * p.W + (ok ? xi : 0)) * CIN;
    float a[CIN];
#pragma unroll
    for (int c = 0; c < CIN; ++c) a[c] = 0.f;
    constexpr int KU = K ? K : kMaxSplitK;  // K == 0: runtime p.K <= 16
#pragma unroll
    for (int j = 0; j < KU; ++j)
      if (K || j < p.K) {
#pragma unroll
        for (int c = 0; c < CIN; ++c) a[c] = fmaf(p.coef[j], ok ? __ldg(src + (long long)j * p.in_st + c) : 0.f, a[c]);
      }
    uint32_t e[CIN];
#pragma unroll
    for (int c = 0; c < CIN; ++c) e[c] = f32_to_h16pair(a[c]);
    const uint4 c0 = split_row_words<CIN>(e[0], e[CIN - 1], p.packed);
    const uint32_t dst = a_stage + (uint32_t)row * 16u;
    ptx::st_shared_v4(dst, c0.x, c0.y, c0.z, c0.w);
    ptx::st_shared_v4(dst + p.lbo_a, 0u, 0u, 0u, 0u);
  }
}

// LDG split producers (e.g. MNIST rows, whose 4-B row stride rules out halo-box TMA;
// SMEM: plane mode, the whole frames in shared memory)
template <int K, int CIN, bool SMEM = false>
__device__ __forceinline__ void produce_h16s(const TcParams &p, const uint32_t *lut, const TileXY &tile, int k,
                                             uint32_t a_stage, int ptid, const uint32_t *plane = nullptr) {
  const int b = tile.b, y0 = tile.y0, x0 = tile.x0;
  const bool tok = tile.ok;
  const uint32_t *frame0 = SMEM ? plane : p.in + (long long)(k * K) * p.in_st + (long long)b * p.in_sb;
  const long long fst = SMEM ? (long long)p.raw_bw : p.in_st;
  for (int row = ptid; row < kHaloRows; row += p.prod_step) {
    const int hy = row / kHaloW, hx = row - (row / kHaloW) * kHaloW;
    const int yi = y0 + hy - p.pad, xi = x0 + hx - p.pad;
    const bool ok = tok && yi >= 0 && yi < p.H && xi >= 0 && xi < p.W;
    const int bit = ok ? xi * CIN : 0, sh = bit & 31;
    const bool two = ok && sh + CIN > 32;
    const uint32_t *src = frame0 + (long long)(ok ? yi : 0) * p.wpr_in + (bit >> 5);
    uint32_t bits[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const uint32_t w0 = ok ? ld_src<SMEM>(src + (long long)j * fst) : 0u;
      const uint32_t w1 = two ? ld_src<SMEM>(src + (long long)j * fst + 1) : 0u;
      bits[j] = __funnelshift_r(w0, w1, sh);
    }
    const uint4 c0 = split_row_small<K, CIN>(bits, lut, p.packed);
    const uint32_t dst = a_stage + (uint32_t)row * 16u;
    ptx::st_shared_v4(dst, c0.x, c0.y, c0.z, c0.w);
    ptx::st_shared_v4(dst + p.lbo_a, 0u, 0u, 0u, 0u);
  }
}

template <int CIN, bool SMEM = false>
__device__ __forceinline__ void produce_h16s_rt(const TcParams &p, const uint32_t *lut, const TileXY &tile, int k,
                                                uint32_t a_stage, int ptid, const uint32_t *plane = nullptr) {
  const int b = tile.b, y0 = tile.y0, x0 = tile.x0;
  const bool tok = tile.ok;
  const int K = p.K;
  const uint32_t *frame0 = SMEM ? plane : p.in + (long long)(k * K) * p.in_st + (long long)b * p.in_sb;
  const long long fst = SMEM ? (long long)p.raw_bw : p.in_st;
  for (int row = ptid; row < kHaloRows; row += p.prod_step) {
    const int hy = row / kHaloW, hx = row - (row / kHaloW) * kHaloW;
    const int yi = y0 + hy - p.pad, xi = x0 + hx - p.pad;
    const bool ok = tok && yi >= 0 && yi < p.H && xi >= 0 && xi < p.W;
    const int bit = ok ? xi * CIN : 0, sh = bit & 31;
    const bool two = ok && sh + CIN > 32;
    const uint32_t *src = frame0 + (long long)(ok ? yi : 0) * p.wpr_in + (bit >> 5);
    uint32_t i0 = 0, i1 = 0;
#pragma unroll
    for (int j = 0; j < kMaxSplitK; ++j)
      if (j < K) {
        const uint32_t w0 = ok ? ld_src<SMEM>(src + (long long)j * fst) : 0u;
        const uint32_t w1 = two ? ld_src<SMEM>(src + (long long)j * fst + 1) : 0u;
        const uint32_t bits = __funnelshift_r(w0, w1, sh);
        i0 |= (bits & 1u) << j;
        i1 |= ((bits >> 1) & 1u) << j;
      }
    const uint32_t e0 = split_lookup(i0, K, lut), e1 = CIN == 2 ? split_lookup(i1, K, lut) : 0u;
    const uint4 c0 = split_row_words<CIN>(e0, e1, p.packed);
    const uint32_t dst = a_stage + (uint32_t)row * 16u;
    ptx::st_shared_v4(dst, c0.x, c0.y, c0.z, c0.w);
    ptx::st_shared_v4(dst + p.lbo_a, 0u, 0u, 0u, 0u);
  }
}

// Plane-mode row producer (first layers with C_in <= 2 whose K whole frames sit in smem,
// e.g. MNIST 28 x 28 x 1): lane hy (< 18) builds halo row hy.  The K frame words covering
// the row's 10 halo pixels are funnel-shifted to bit 0 once (K loads per ROW instead of
// per pixel), transposed so that byte b of o[q] is the K-bit frame index of row bit
// q + 8 b, and each pixel's index feeds the aggregate table (split path) or is the
// exact aggregate itself (beta = 1/2 or dense: sum_j bit_j 2^j).  Chunk 1 of every
// row is constant (h16_init_stages), so only chunk 0 is stored.
__device__ __forceinline__ int halo_c0(const TcParams &p, int x0);
// v[j]: frame j's bits of halo row `lane`, halo column 0 at bit 0 -> the row's 10 A rows
// 8 x 8 bit-matrix transpose of a 64-bit word (bit 8 i + j <-> bit 8 j + i): three
// delta swaps (Hacker's Delight 7-3) instead of 8 K shift / mask / or steps
__device__ __forceinline__ uint64_t transpose8x8(uint64_t x) {
  uint64_t t;
  t = (x ^ (x >> 7)) & 0x00AA00AA00AA00AAull;
  x = x ^ t ^ (t << 7);
  t = (x ^ (x >> 14)) & 0x0000CCCC0000CCCCull;
  x = x ^ t ^ (t << 14);
  t = (x ^ (x >> 28)) & 0x00000000F0F0F0F0ull;
  return x ^ t ^ (t << 28);
}

template <int K, int CIN, bool SPLIT>
__device__ __forceinline__ void emit_halo_row(const TcParams &p, const uint32_t *lut, uint32_t a_stage,
                                              int lane, const uint32_t (&v)[K]) {
  // X[b]: byte j = byte b of frame j's row bits -> transposed: byte q = the K-bit frame
  // index of row bit 8 b + q
  constexpr int NB = (kHaloW * CIN + 7) / 8;
  uint64_t X[NB];
#pragma unroll
  for (int bb = 0; bb < NB; ++bb) {
    const uint32_t sel = (uint32_t)bb | ((uint32_t)(4 + bb) << 4);  // byte bb of x, byte bb of y
    uint32_t lo = 0u, hi = 0u;
    if (K >= 2) lo = __byte_perm(v[0], v[K >= 2 ? 1 : 0], sel);
    else lo = (v[0] >> (8 * bb)) & 0xFFu;
    if (K >= 4) lo = __byte_perm(lo, __byte_perm(v[K >= 4 ? 2 : 0], v[K >= 4 ? 3 : 0], sel), 0x5410u);
    else if (K == 3) lo = __byte_perm(lo, (v[K == 3 ? 2 : 0] >> (8 * bb)) & 0xFFu, 0x5410u);
    else lo &= 0xFFFFu;
    if (K >= 6) hi = __byte_perm(v[K >= 6 ? 4 : 0], v[K >= 6 ? 5 : 0], sel);
    else if (K == 5) hi = (v[K == 5 ? 4 : 0] >> (8 * bb)) & 0xFFu;
    if (K == 8) hi = __byte_perm(hi, __byte_perm(v[K == 8 ? 6 : 0], v[K == 8 ? 7 : 0], sel), 0x5410u);
    else if (K == 7) hi = __byte_perm(hi, (v[K == 7 ? 6 : 0] >> (8 * bb)) & 0xFFu, 0x5410u);
    else if (K == 6) hi &= 0xFFFFu;
    X[bb] = transpose8x8(((uint64_t)hi << 32) | lo);
  }
  uint32_t one_lo, one_hi, c8;
  h16_bias_slot(CIN, one_lo, one_hi, c8);
  const uint32_t dst0 = a_stage + (uint32_t)(lane * kHaloW) * 16u;
#pragma unroll
  for (int c = 0; c < kHaloW; ++c) {
    uint32_t idx[CIN];
#pragma unroll
    for (int ch = 0; ch < CIN; ++ch) {
      const int bp = c * CIN + ch;            // compile-time
      idx[ch] = (uint32_t)(X[bp >> 3] >> (8 * (bp & 7))) & 0xFFu;
    }
    if constexpr (SPLIT) {
      const uint4 w = split_row_words<CIN>(lut[idx[0]], CIN == 2 ? lut[idx[CIN - 1]] : 0u, p.packed);
      ptx::st_shared_v4(dst0 + c * 16u, w.x, w.y, w.z, w.w);
    } else {
      uint32_t lo = one_lo | idx[0] | (CIN == 2 ? idx[CIN - 1] << 8 : 0u), hi = one_hi;
      if (p.packed) h16_pack_slices(lo, hi, CIN);
      ptx::st_shared_v4(dst0 + c * 16u, u8x2_to_f16x2(lo, 0x5140u), u8x2_to_f16x2(lo, 0x7362u),
                        u8x2_to_f16x2(hi, 0x5140u), u8x2_to_f16x2(hi, 0x7362u));
    }
  }
}

// The same row producer on a TMA raw HALO box ([K][18][raw_bw] words from the 16-B
// aligned word c0w; the box's out-of-bounds zero fill is the conv padding): the DVS first
// layer (2 x 128 x 128, one producer warp per stage).
template <int K, int CIN, bool SPLIT>
__device__ __forceinline__ void produce_halo_rows(const TcParams &p, const uint32_t *lut, const uint32_t *raw,
                                                  uint32_t a_stage, int lane, int x0) {
  static_assert(K >= 1 && K <= 8 && (CIN == 1 || CIN == 2), "row producer envelope");
  if (lane >= kHaloH) return;
  const int bw = p.raw_bw, fstride = kHaloH * p.raw_bw;
  const int bit0 = (x0 - p.pad) * CIN - (halo_c0(p, x0) & ~3) * 32;  // >= 0
  const uint32_t *row = raw + lane * bw + (bit0 >> 5);
  const int sh = bit0 & 31;
  uint32_t v[K];
#pragma unroll
  for (int j = 0; j < K; ++j) v[j] = __funnelshift_r(row[j * fstride], row[j * fstride + 1], sh);
  emit_halo_row<K, CIN, SPLIT>(p, lut, a_stage, lane, v);
}

template <int K, int CIN, bool SPLIT>
__device__ __forceinline__ void produce_plane_rows(const TcParams &p, const uint32_t *lut, const TileXY &tile,
                                                   uint32_t a_stage, int lane, const uint32_t *plane) {
  static_assert(K >= 1 && K <= 8 && (CIN == 1 || CIN == 2), "row producer envelope");
  if (lane >= kHaloH) return;
  const int b = tile.b, y0 = tile.y0, x0 = tile.x0;
  const bool tok = tile.ok;
  const int yi = y0 + lane - p.pad;
  const bool rok = tok && yi >= 0 && yi < p.H;
  const int bit0 = (x0 - p.pad) * CIN;       // row bit of halo column 0 (-CIN with left padding)
  const int wb = bit0 >> 5, sh = bit0 & 31;  // floor division
  const int wpr = p.wpr_in;
  const uint32_t *row = plane + (rok ? yi : 0) * wpr;
  uint32_t v[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const uint32_t *fr = row + j * p.raw_bw;
    const uint32_t w0 = (rok && wb >= 0 && wb < wpr) ? fr[wb] : 0u;
    const uint32_t w1 = (rok && wb + 1 >= 0 && wb + 1 < wpr) ? fr[wb + 1] : 0u;
    v[j] = __funnelshift_r(w0, w1, sh);      // bits beyond W C_in are 0 in a packed row
  }
  emit_halo_row<K, CIN, SPLIT>(p, lut, a_stage, lane, v);
}

template <int K>
__device__ __forceinline__ void produce_s32(const TcParams &p, const uint32_t *lut, const TileXY &tile, int k,
                                            uint32_t a_stage, int ptid) {
  const int b = tile.b, y0 = tile.y0, x0 = tile.x0;
  const bool tok = tile.ok;
  const uint32_t *frame0 = p.in + (long long)(k * K) * p.in_st + (long long)b * p.in_sb;
  for (int row = ptid; row < kHaloRows; row += p.prod_step) {
    const int hy = row / kHaloW, hx = row - (row / kHaloW) * kHaloW;
    const int yi = y0 + hy - p.pad, xi = x0 + hx - p.pad;
    const bool ok = tok && yi >= 0 && yi < p.H && xi >= 0 && xi < p.W;
    const uint32_t *src = frame0 + (long long)(ok ? yi : 0) * p.wpr_in + (ok ? xi : 0);
    uint32_t x[K];
#pragma unroll
    for (int j = 0; j < K; ++j) x[j] = ok ? __ldg(src + (long long)j * p.in_st) : 0u;
    uint32_t o[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    agg_word_m1<K>(o, x);  // byte b of o[q] = K-bit index of channel q + 8b
    store_split32_row(a_stage + (uint32_t)row * 16u, p.lbo_a, o, lut);
  }
}

// --- TMA producers: aggregate from the raw halo in smem (compact loops) --------
// raw-halo start word of a tile: the TMA box starts 16-B aligned (word c0 & ~3)
__device__ __forceinline__ int halo_c0(const TcParams &p, int x0) {
  return p.Cin >= 32 ? (x0 - p.pad) * (p.Cin >> 5)
                     : ((x0 - p.pad) * p.Cin >= 0 ? ((x0 - p.pad) * p.Cin) >> 5
                                                  : -((31 - (x0 - p.pad) * p.Cin) >> 5));
}

// TMA raw-halo producer (C_in = 32 nwin): thread owns 32-channel word w of halo
// pixels row0, row0 + rstep, ...; NR pixels per pass with all NR K smem loads
// issued before any arithmetic (one smem latency per pass).
template <int K>
__device__ __forceinline__ void produce_halo_tma(const TcParams &p, const uint32_t *raw,
                                                 uint32_t a_stage, int ptid, int x0) {
  const int nwin = p.Cin >> 5, bw = p.raw_bw, fstride = kHaloH * p.raw_bw;
  const int c0 = halo_c0(p, x0);
  raw += c0 - (c0 & ~3);
  // groups of 8 consecutive threads own 8 consecutive halo pixels of one 32-channel
  // word w: their 16-B A-stage stores are contiguous (no bank conflicts) and their
  // raw-halo loads (pixel stride nwin words, 4 words in a group) hit distinct banks
#if TACSNN_HALO_MAP
  const int g8 = ptid >> 3, w = g8 % nwin, row0 = (g8 / nwin) * 8 + (ptid & 7);
#else
  const int w = ptid % nwin, row0 = ptid / nwin;
#endif
  const int rstep = (kProdWarps * 32) / nwin;
  const int mshift = p.m_shift;
  const uint32_t lbo = p.lbo_a;
  constexpr int NR = K <= 4 ? TACSNN_HALO_NR : 2;  // pixels per pass (64 registers per producer thread)
#pragma unroll 1
  for (int row = row0; row < kHaloRows; row += NR * rstep) {
    uint32_t x[NR][K];
#pragma unroll
    for (int r = 0; r < NR; ++r) {  // all NR x K smem loads first
      const int rr = row + r * rstep;
      const bool ok = rr < kHaloRows;
      const int hy = ok ? rr / kHaloW : 0, hx = ok ? rr - hy * kHaloW : 0;
      const uint32_t *src = raw + hy * bw + hx * nwin + w;
#pragma unroll
      for (int j = 0; j < K; ++j) x[r][j] = ok ? src[j * fstride] : 0u;
    }
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int rr = row + r * rstep;
      if (rr < kHaloRows) {
        uint32_t o[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        if (mshift == 1 || K == 1) agg_word_m1<K>(o, x[r]); else agg_word_k<K>(o, x[r], mshift);
        const uint32_t dst = a_stage + (uint32_t)(2 * w) * lbo + (uint32_t)rr * 16u;
        ptx::st_shared_v4(dst, o[0], o[1], o[2], o[3]);
        ptx::st_shared_v4(dst + lbo, o[4], o[5], o[6], o[7]);
      }
    }
  }
}

// The raw box holds words [c0w, c0w + 8) of each halo row (OOB words are zero, and
// so are the bits past W*C_in of a row), so pixel xi sits at box bit
// (xi * C_in - 32 c0w) >= 0 and never straddles past word 7.  Only the first
// 16-B chunk (channels 0..7) of a halo row changes per group; chunk 1 (channels
// 8..15: zeros, or the bias 1.0 when C_in == 8) is written once per A stage by
// h16_init_stages.  CIN4: C_in <= 4, channels 4..7 of chunk 0 hold only the bias.
template <int K, bool CIN4>
__device__ __forceinline__ void produce_h16_tma(const TcParams &p, const uint32_t *raw,
                                                uint32_t a_stage, int ptid, int x0) {
  const int Cin = p.Cin, bw = p.raw_bw, fstride = kHaloH * p.raw_bw;
  const uint32_t cmask = (1u << Cin) - 1u;
  const int c0w = halo_c0(p, x0) & ~3;
  uint32_t one_lo, one_hi, c8;
  h16_bias_slot(Cin, one_lo, one_hi, c8);
  const int mshift = p.m_shift;
  constexpr int RSTEP = kProdWarps * 32;
  constexpr int NR = K <= 4 ? 2 : 1;  // pixels per pass (register budget: 64 per producer thread)
#pragma unroll 1
  for (int row = ptid; row < kHaloRows; row += NR * RSTEP) {
    const int row1 = row + RSTEP;
    const bool two = NR == 2 && row1 < kHaloRows;
    const int r1 = two ? row1 : row;
    const int hy0 = row / kHaloW, hx0 = row - hy0 * kHaloW;
    const int hy1 = r1 / kHaloW, hx1 = r1 - hy1 * kHaloW;
    const int b0 = (x0 + hx0 - p.pad) * Cin - c0w * 32, b1 = (x0 + hx1 - p.pad) * Cin - c0w * 32;
    const uint32_t *s0 = raw + hy0 * bw + (b0 >> 5), *s1 = raw + hy1 * bw + (b1 >> 5);
    const int sh0 = b0 & 31, sh1 = b1 & 31;
    uint32_t a0[K], a1[K], c0[K], c1[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      a0[j] = s0[j * fstride];
      a1[j] = s0[j * fstride + 1];
      c0[j] = NR == 2 ? s1[j * fstride] : 0u;
      c1[j] = NR == 2 ? s1[j * fstride + 1] : 0u;
    }
    uint32_t lo0 = one_lo, hi0 = one_hi, lo1 = one_lo, hi1 = one_hi;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const uint32_t bits0 = __funnelshift_r(a0[j], a1[j], sh0) & cmask;
      const uint32_t bits1 = __funnelshift_r(c0[j], c1[j], sh1) & cmask;
      if (CIN4) {
        lo0 |= ((bits0 * 0x204081u) & 0x01010101u) << (mshift * j);
        lo1 |= ((bits1 * 0x204081u) & 0x01010101u) << (mshift * j);
      } else {
        h16_acc(lo0, hi0, bits0, mshift * j);
        h16_acc(lo1, hi1, bits1, mshift * j);
      }
    }
    if (p.packed) {
      h16_pack_slices(lo0, hi0, Cin);
      h16_pack_slices(lo1, hi1, Cin);
    }
    const uint32_t d0 = a_stage + (uint32_t)row * 16u;
    ptx::st_shared_v4(d0, u8x2_to_f16x2(lo0, 0x5140u), u8x2_to_f16x2(lo0, 0x7362u),
                      u8x2_to_f16x2(hi0, 0x5140u), u8x2_to_f16x2(hi0, 0x7362u));
    if (two) {
      const uint32_t d1 = a_stage + (uint32_t)row1 * 16u;
      ptx::st_shared_v4(d1, u8x2_to_f16x2(lo1, 0x5140u), u8x2_to_f16x2(lo1, 0x7362u),
                        u8x2_to_f16x2(hi1, 0x5140u), u8x2_to_f16x2(hi1, 0x7362u));
    }
  }
}

// TMA split producers (raw halo in smem; see produce_h16_tma / produce_halo_tma)
template <int K, int CIN>
__device__ __forceinline__ void produce_h16s_tma(const TcParams &p, const uint32_t *lut,
                                                 const uint32_t *raw, uint32_t a_stage, int ptid,
                                                 int x0) {
  const int bw = p.raw_bw, fstride = kHaloH * p.raw_bw;
  const int c0w = halo_c0(p, x0) & ~3;
#pragma unroll 1
  for (int row = ptid; row < kHaloRows; row += kProdWarps * 32) {
    const int hy = row / kHaloW, hx = row - hy * kHaloW;
    const int bitoff = (x0 + hx - p.pad) * CIN - c0w * 32;
    const uint32_t *src = raw + hy * bw + (bitoff >> 5);
    const int sh = bitoff & 31;
    uint32_t bits[K];
#pragma unroll
    for (int j = 0; j < K; ++j) bits[j] = __funnelshift_r(src[j * fstride], src[j * fstride + 1], sh);
    const uint4 c = split_row_small<K, CIN>(bits, lut, p.packed);
    ptx::st_shared_v4(a_stage + (uint32_t)row * 16u, c.x, c.y, c.z, c.w);
  }
}

template <int CIN>
__device__ __forceinline__ void produce_h16s_tma_rt(const TcParams &p, const uint32_t *lut,
                                                    const uint32_t *raw, uint32_t a_stage, int ptid,
                                                    int x0) {
  const int bw = p.raw_bw, fstride = kHaloH * p.raw_bw, K = p.K;
  const int c0w = halo_c0(p, x0) & ~3;
#pragma unroll 1
  for (int row = ptid; row < kHaloRows; row += kProdWarps * 32) {
    const int hy = row / kHaloW, hx = row - hy * kHaloW;
    const int bitoff = (x0 + hx - p.pad) * CIN - c0w * 32;
    const uint32_t *src = raw + hy * bw + (bitoff >> 5);
    const int sh = bitoff & 31;
    uint32_t i0 = 0, i1 = 0;
#pragma unroll
    for (int j = 0; j < kMaxSplitK; ++j)
      if (j < K) {
        const uint32_t bits = __funnelshift_r(src[j * fstride], src[j * fstride + 1], sh);
        i0 |= (bits & 1u) << j;
        i1 |= ((bits >> 1) & 1u) << j;
      }
    const uint32_t e0 = split_lookup(i0, K, lut), e1 = CIN == 2 ? split_lookup(i1, K, lut) : 0u;
    const uint4 c = split_row_words<CIN>(e0, e1, p.packed);
    ptx::st_shared_v4(a_stage + (uint32_t)row * 16u, c.x, c.y, c.z, c.w);
  }
}

template <int K>
__device__ __forceinline__ void produce_s32_tma(const TcParams &p, const uint32_t *lut,
                                                const uint32_t *raw, uint32_t a_stage, int ptid,
                                                int x0) {
  const int bw = p.raw_bw, fstride = kHaloH * p.raw_bw;
  const int c0 = halo_c0(p, x0);
  raw += c0 - (c0 & ~3);
#pragma unroll 1
  for (int row = ptid; row < kHaloRows; row += kProdWarps * 32) {
    const int hy = row / kHaloW, hx = row - hy * kHaloW;
    const uint32_t *src = raw + hy * bw + hx;
    uint32_t x[K];
#pragma unroll
    for (int j = 0; j < K; ++j) x[j] = src[j * fstride];
    uint32_t o[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    agg_word_m1<K>(o, x);
    store_split32_row(a_stage + (uint32_t)row * 16u, p.lbo_a, o, lut);
  }
}

// chunk 1 of every halo row of every A stage (constant for the whole kernel)
__device__ __forceinline__ void h16_init_stages(const TcParams &p, uint32_t sbase, int ptid) {
  uint32_t one_lo, one_hi, c8;
  h16_bias_slot(p.Cin, one_lo, one_hi, c8);
  for (int i = ptid; i < p.nstages * kHaloRows; i += kProdWarps * 32) {
    const int st = i / kHaloRows, row = i - st * kHaloRows;
    ptx::st_shared_v4(sbase + p.off_a + st * p.a_stage_bytes + p.lbo_a + (uint32_t)row * 16u, c8,
                      0u, 0u, 0u);
  }
}

// Raw-halo TMA loader, run by one lane of the MMA warp of each CTA: keeps nraw
// raw-halo loads (K frames x 18 halo rows of this CTA's tile) in flight; slot r is
// refilled once the producer warps have arrived on raw_empty[r].
struct RawLoader {
  int ipair, ik;  // next (pair, group) to load
  uint32_t n;     // loads issued
  int b, ty, tx;  // tile coordinates of ipair (advanced incrementally: no divisions per load)
  int db, dty, dtx;
  Ring slot, rel;  // slot of the next load; raw_empty phase of the next refill
  __device__ __forceinline__ void issue(const TcParams &p, uint32_t sbase, uint32_t bar_raw,
                                        int ncl) {
    const uint32_t sl = slot.i;
    slot.next((uint32_t)p.nraw);
    const int x0 = tx * kTileW;
    const int c0 = halo_c0(p, x0) & ~3;  // 16-B aligned box start
    const uint32_t bar = bar_raw + 8 * sl;
    ptx::mbar_arrive_expect_tx(bar, p.raw_box_bytes);
    if (p.use_tma == 2)
      ptx::tma_load_3d(sbase + p.off_raw + sl * p.raw_stage_bytes, &p.tmap, 0, b, ik * p.K, bar);
    else
      ptx::tma_load_4d(sbase + p.off_raw + sl * p.raw_stage_bytes, &p.tmap, c0, ty * kTileH - p.pad, b,
                       ik * p.K, bar);
    if (++ik == p.G) {
      ik = 0;
      ipair += ncl;
      tx += dtx;
      int cy = tx >= p.tiles_x;
      tx -= cy ? p.tiles_x : 0;
      ty += dty + cy;
      cy = ty >= p.tiles_y;
      ty -= cy ? p.tiles_y : 0;
      b += db + cy;
    }
    ++n;
  }
  __device__ __forceinline__ bool more(const TcParams &p) const { return ipair < p.num_pairs; }
  // prime the ring
  __device__ __forceinline__ void start(const TcParams &p, uint32_t sbase, uint32_t bar_raw, int cid,
                                        int ncl, uint32_t rank) {
    ipair = cid;
    ik = 0;
    n = 0;
    slot = Ring();
    rel = Ring();
    const int per = p.tiles_x * p.tiles_y, t0 = 2 * cid + (int)rank, dt = 2 * ncl;
    b = t0 / per;
    ty = (t0 - b * per) / p.tiles_x;
    tx = t0 - b * per - ty * p.tiles_x;
    db = dt / per;
    dty = (dt - db * per) / p.tiles_x;
    dtx = dt - db * per - dty * p.tiles_x;
    for (int r = 0; r < p.nraw && more(p); ++r) issue(p, sbase, bar_raw, ncl);
  }
  // after consumption `it` of slot it % nraw: wait until every producer warp is done
  // with it, then refill the slot
  __device__ __forceinline__ void refill(const TcParams &p, uint32_t sbase, uint32_t bar_raw,
                                         uint32_t bar_raw_empty, uint32_t it, int ncl) {
    (void)it;  // refills come in consumption order: rel tracks it % nraw and its phase
    if (!more(p)) return;
    wait_ahead(p, bar_raw_empty + 8 * rel.i, rel.ph);
    rel.next((uint32_t)p.nraw);
    issue(p, sbase, bar_raw, ncl);
  }
};

// Plane-mode raw refill by the producer warp (p.prod_refill): load number L (the L-th
// (tile pair, group) of this CTA in issue order) into raw slot r.
__device__ __forceinline__ void refill_plane(const TcParams &p, uint32_t sbase, uint32_t bar_raw, uint32_t L,
                                             uint32_t r, int cid, int ncl, uint32_t rank) {
  const int pi = (int)(L / (uint32_t)p.G), k = (int)(L - (uint32_t)pi * (uint32_t)p.G);
  const int pair = cid + pi * ncl;
  if (pair >= p.num_pairs) return;
  int b, y0, x0;
  bool tok;
  tile_origin(p, 2 * pair + (int)rank, b, y0, x0, tok);
  const uint32_t bar = bar_raw + 8 * r;
  ptx::mbar_arrive_expect_tx(bar, p.raw_box_bytes);
  if (p.use_tma == 2)
    ptx::tma_load_3d(sbase + p.off_raw + r * p.raw_stage_bytes, &p.tmap, 0, b, k * p.K, bar);
  else
    ptx::tma_load_4d(sbase + p.off_raw + r * p.raw_stage_bytes, &p.tmap, halo_c0(p, x0) & ~3, y0 - p.pad, b,
                     k * p.K, bar);
}

// TMA producer pipeline: all 96 producer threads aggregate raw stage `it % nraw`
// into A stage `it % nstages`; each warp then releases the raw stage (local
// raw_empty barrier, refilled by the MMA warp's loader) and arrives on the pair's
// A-full barrier in CTA 0.
template <int PATH, int K>
__device__ __forceinline__ void producer_role_tma(const TcParams &p, uint32_t sbase,
                                                  const uint8_t *smem, uint32_t bar_a_full,
                                                  uint32_t bar_a_empty, uint32_t bar_raw,
                                                  uint32_t bar_raw_empty, int cid, int ncl,
                                                  uint32_t rank, uint32_t lane, int ptid, int npw) {
  const uint32_t ns = (uint32_t)p.nstages, nr = (uint32_t)p.nraw;
  const bool ws = p.warp_stage != 0;
  if (!ws) npw = kProdWarps;
  if (ptid >= 32 * npw) return;  // extra producer warps: warp_stage producers only
  if (PATH != PATH_HALO && ptid < 32 * kProdWarps) h16_init_stages(p, sbase, ptid);  // fenced with the first stage
  if (ws) {  // every producer warp's init writes are visible before any warp's first stage
    ptx::fence_proxy_async_smem();
    ptx::named_bar_sync(1, 32 * npw);
  }
  const uint32_t pw = (uint32_t)ptid >> 5;
  const int wptid = ws ? (int)lane : ptid;
  uint32_t it = 0;
  Ring st, rw;
  TileWalk tw(p, 2 * cid + (int)rank, 2 * ncl);
  for (int pair = cid; pair < p.num_pairs; pair += ncl, tw.step(p)) {
    const TileXY tile = tw.at(p, 2 * pair + (int)rank);
    const int x0 = tile.x0;
    for (int k = 0; k < p.G; ++k, ++it) {
      const uint32_t s = st.i, ph = st.ph, r = rw.i, rph = rw.ph;
      st.next(ns);
      rw.next(nr);
      if (ws && it % (uint32_t)npw != pw) continue;  // another producer warp builds this stage
      wait_ahead(p, bar_raw + 8 * r, rph);
      if (wptid == 0) trace_mark(p, it, TR_PROD_RAW);
      wait_ahead(p, bar_a_empty + 8 * s, ph ^ 1u);
      if (wptid == 0) trace_mark(p, it, TR_PROD_START);
      const uint32_t *raw = reinterpret_cast<const uint32_t *>(smem + p.off_raw + r * p.raw_stage_bytes);
      const uint32_t a_stage = sbase + p.off_a + s * p.a_stage_bytes;
      const uint32_t *lut = reinterpret_cast<const uint32_t *>(smem + p.off_lut);
      if (p.use_tma == 2) {  // plane mode: whole frames in smem, pixel-wise producers read them
        if constexpr (PATH != PATH_HALO) {
          if constexpr (K == 0) {
            if (PATH == PATH_SPLIT)
              p.Cin == 1 ? produce_h16s_rt<1, true>(p, lut, tile, k, a_stage, wptid, raw)
                         : produce_h16s_rt<2, true>(p, lut, tile, k, a_stage, wptid, raw);
          } else if (ws && K <= 8 && p.Cin <= 2 && (PATH == PATH_SPLIT || p.m_shift <= 1)) {
            // one warp builds the stage row by row (see produce_plane_rows)
            if constexpr (K <= 8) {
              if (PATH == PATH_SPLIT)
                p.Cin == 1 ? produce_plane_rows<K, 1, true>(p, lut, tile, a_stage, wptid, raw)
                           : produce_plane_rows<K, 2, true>(p, lut, tile, a_stage, wptid, raw);
              else
                p.Cin == 1 ? produce_plane_rows<K, 1, false>(p, lut, tile, a_stage, wptid, raw)
                           : produce_plane_rows<K, 2, false>(p, lut, tile, a_stage, wptid, raw);
            }
          } else if (PATH == PATH_SPLIT) {
            p.Cin == 1 ? produce_h16s<K, 1, true>(p, lut, tile, k, a_stage, wptid, raw)
                       : produce_h16s<K, 2, true>(p, lut, tile, k, a_stage, wptid, raw);
          } else {
            produce_h16<K, true>(p, tile, k, a_stage, wptid, raw);
          }
        }
      } else if constexpr (K == 0) {  // runtime group size: split path, C_in <= 2 (envelope)
        if (PATH == PATH_SPLIT)
          p.Cin == 1 ? produce_h16s_tma_rt<1>(p, lut, raw, a_stage, ptid, x0)
                     : produce_h16s_tma_rt<2>(p, lut, raw, a_stage, ptid, x0);
      } else if (PATH == PATH_HALO) {
        produce_halo_tma<K>(p, raw, a_stage, ptid, x0);
      } else if (ws) {  // halo boxes, one producer warp per stage (host: rows_ok)
        if constexpr (K <= 8) {
          if (PATH == PATH_SPLIT)
            p.Cin == 1 ? produce_halo_rows<K, 1, true>(p, lut, raw, a_stage, wptid, x0)
                       : produce_halo_rows<K, 2, true>(p, lut, raw, a_stage, wptid, x0);
          else
            p.Cin == 1 ? produce_halo_rows<K, 1, false>(p, lut, raw, a_stage, wptid, x0)
                       : produce_halo_rows<K, 2, false>(p, lut, raw, a_stage, wptid, x0);
        }
      } else if (PATH == PATH_SPLIT) {
        p.Cin == 32 ? produce_s32_tma<K>(p, lut, raw, a_stage, ptid, x0)
                    : (p.Cin == 1 ? produce_h16s_tma<K, 1>(p, lut, raw, a_stage, ptid, x0)
                                  : produce_h16s_tma<K, 2>(p, lut, raw, a_stage, ptid, x0));
      } else if (p.Cin <= 4) {
        produce_h16_tma<K, true>(p, raw, a_stage, ptid, x0);
      } else {
        produce_h16_tma<K, false>(p, raw, a_stage, ptid, x0);
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive_local(bar_raw_empty + 8 * r);  // this warp's reads of raw stage r are done
        ptx::mbar_arrive_cluster_cta(bar_a_full + 8 * s, 0);
        // plane mode: this warp was raw slot r's only reader, so it refills the slot with the
        // planes of group it + nraw itself -- the MMA warp's issue loop carries no TMA work
        if (p.prod_refill) refill_plane(p, sbase, bar_raw, it + nr, r, cid, ncl, rank);
      }
      if (wptid == 0) trace_mark(p, it, TR_PROD_DONE);
    }
  }
}

template <int PATH, int K>
__device__ __forceinline__ void producer_role(const TcParams &p, uint32_t sbase, const uint8_t *smem,
                                              uint32_t bar_a_full, uint32_t bar_a_empty, int cid,
                                              int ncl, uint32_t rank, uint32_t lane, int ptid, int npw) {
  const uint32_t *lut = reinterpret_cast<const uint32_t *>(smem + p.off_lut);
  const uint32_t ns = (uint32_t)p.nstages;
  const bool ws = p.warp_stage != 0;
  if (!ws) npw = kProdWarps;
  if (ptid >= 32 * npw) return;  // extra producer warps: warp_stage producers only
  const uint32_t pw = (uint32_t)ptid >> 5;
  if (ws) ptid = (int)lane;  // each warp builds whole stages (stage it -> warp it % 3)
  uint32_t it = 0;
  Ring st;
  TileWalk tw(p, 2 * cid + (int)rank, 2 * ncl);
  for (int pair = cid; pair < p.num_pairs; pair += ncl, tw.step(p)) {
    const TileXY tile = tw.at(p, 2 * pair + (int)rank);
    for (int k = 0; k < p.G; ++k, ++it) {
      const uint32_t s = st.i, ph = st.ph;
      st.next(ns);
      if (ws && it % (uint32_t)npw != pw) continue;
      wait_ahead(p, bar_a_empty + 8 * s, ph ^ 1u);
      const uint32_t a_stage = sbase + p.off_a + s * p.a_stage_bytes;
      if (PATH == PATH_SPLIT && p.real) {
        p.Cin == 1 ? produce_h16x<K, 1>(p, tile, k, a_stage, ptid) : produce_h16x<K, 2>(p, tile, k, a_stage, ptid);
      } else if constexpr (K == 0) {  // runtime group size: split path, C_in <= 2 (envelope)
        if (PATH == PATH_SPLIT)
          p.Cin == 1 ? produce_h16s_rt<1>(p, lut, tile, k, a_stage, ptid)
                     : produce_h16s_rt<2>(p, lut, tile, k, a_stage, ptid);
      } else if (PATH == PATH_HALO) {
        produce_halo<K>(p, tile, k, a_stage, ptid);
      } else if (PATH == PATH_SPLIT) {
        p.Cin == 32 ? produce_s32<K>(p, lut, tile, k, a_stage, ptid)
                    : (p.Cin == 1 ? produce_h16s<K, 1>(p, lut, tile, k, a_stage, ptid)
                                  : produce_h16s<K, 2>(p, lut, tile, k, a_stage, ptid));
      } else {
        produce_h16<K>(p, tile, k, a_stage, ptid);
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_cluster_cta(bar_a_full + 8 * s, 0);
    }
  }
}

// --- epilogue helpers ---------------------------------------------------------
// column popcount of a 32x32 bit matrix held one row per lane (32x32 transpose)
__device__ __forceinline__ uint32_t warp_col_popc(uint32_t x, uint32_t lane) {
  const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    const int s = 16 >> i;
    const uint32_t m = masks[i];
    const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, x, s);
    if (lane & s)
      x = (x & ~m) | ((y >> s) & m);
    else
      x = (x & m) | ((y << s) & ~m);
  }
  return __popc(x);
}

// counts[b][co] += column sums of the bit-sliced per-lane counters (one sample
// per warp: a tile never spans samples); clears the counters
template <int NWT>
__device__ __forceinline__ void flush_counts(const TcParams &p, uint32_t (&planes)[kPlanes][NWT],
                                             int b, int co_base, int nch, uint32_t lane) {
#pragma unroll
  for (int w = 0; w < NWT; ++w) {
    uint32_t total = 0;
#pragma unroll
    for (int pl = 0; pl < kPlanes; ++pl) total += warp_col_popc(planes[pl][w], lane) << pl;
    const int c = w * 32 + (int)lane;
    const int co = co_base + c;
    if (total && c < nch && co < p.Cout) atomicAdd(p.counts + (long long)b * p.Cout + co, total);
  }
#pragma unroll
  for (int pl = 0; pl < kPlanes; ++pl)
#pragma unroll
    for (int w = 0; w < NWT; ++w) planes[pl][w] = 0u;
}

// generic (runtime reset mode) LIF step; inv_bits collects NOT(spike) at `bitmask`
template <int RESET>
__device__ __forceinline__ void lif_step(float &v, float y, float decay, float vth, float vres,
                                         uint32_t &inv_bits, uint32_t bitmask, uint32_t &prev) {
  v = fmaf(decay, v, y);                                    // Alg.1 l.5 / Alg.2 l.6 / Eq.(1)
  if (RESET == 1) v -= (prev & bitmask) ? vth : 0.f;        // delayed: - v_th s_{t-1}
  const float v2 = v - vth;
  const int msk = __float_as_int(v2) >> 31;                 // -1: v < v_th (no spike)
  if (RESET == 0)                                           // subtract: v - v_th on spike
    v = __int_as_float((__float_as_int(v2) & ~msk) | (__float_as_int(v) & msk));
  else if (RESET == 2)                                      // hard: v_reset on spike
    v = __int_as_float((__float_as_int(vres) & ~msk) | (__float_as_int(v) & msk));
  inv_bits |= (uint32_t)msk & bitmask;
  if (RESET == 1) prev = (prev & ~bitmask) | (~(uint32_t)msk & bitmask);
}

// training forward: the drive of one 8-channel chunk as the LIF consumes it -> y_seq
__device__ __forceinline__ void store_yseq8(const TcParams &p, int k, long long vbase, int cc0, int nvalid,
                                            const float (&y)[8]) {
  float *dst = p.y_seq + (long long)k * p.yseq_plane + vbase + cc0;
  if (nvalid >= 8) {  // 32 contiguous bytes (C_out % 8 == 0: 16-B aligned): two vector stores
    reinterpret_cast<float4 *>(dst)[0] = make_float4(y[0], y[1], y[2], y[3]);
    reinterpret_cast<float4 *>(dst)[1] = make_float4(y[4], y[5], y[6], y[7]);
    return;
  }
#pragma unroll
  for (int q = 0; q < 8; ++q)
    if (q < nvalid) dst[q] = y[q];
}

// Y for 8 channels from the two s32 accumulator slices (see file header)
__device__ __forceinline__ void combine8(const TcParams &p, const float *sc, int co,
                                         const uint32_t (&d1)[8], const uint32_t (&d2)[8],
                                         float (&y)[8]) {
  const int Cp = p.Cout_pad;
  if (p.int_combine) {
    // X = 254 D_hi + D_lo exactly in s32;  Y = X * (s1 agg / 254) + b
    const float4 sa = *reinterpret_cast<const float4 *>(sc + co);
    const float4 sb = *reinterpret_cast<const float4 *>(sc + co + 4);
    const float4 ba = *reinterpret_cast<const float4 *>(sc + Cp + co);
    const float4 bb = *reinterpret_cast<const float4 *>(sc + Cp + co + 4);
    const float s8[8] = {sa.x, sa.y, sa.z, sa.w, sb.x, sb.y, sb.z, sb.w};
    const float b8[8] = {ba.x, ba.y, ba.z, ba.w, bb.x, bb.y, bb.z, bb.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int X = (int)d1[i] * 254 + (int)d2[i];
      y[i] = fmaf((float)X, s8[i], b8[i]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float s1 = sc[2 * Cp + co + i], s2 = sc[3 * Cp + co + i], b = sc[Cp + co + i];
      y[i] = fmaf((float)(int)d1[i], s1, fmaf((float)(int)d2[i], s2, b));
    }
  }
}

#define TAC_LOP3(d, a, b, c, lut) asm("lop3.b32 %0, %1, %2, %3, " #lut ";" : "=r"(d) : "r"(a), "r"(b), "r"(c))

// Add a small count (bit-planes v0 + 2 v1 + 4 v2, any of them may be absent) into
// the 6 bit-sliced per-lane counters P (one bit per channel).
__device__ __forceinline__ void planes_add3(uint32_t *P, uint32_t v0, uint32_t v1, uint32_t v2) {
  uint32_t c0, c1, c2, x;
  c0 = P[0] & v0;
  P[0] ^= v0;
  TAC_LOP3(x, P[1], v1, c0, 0x96);   // sum
  TAC_LOP3(c1, P[1], v1, c0, 0xE8);  // majority (carry)
  P[1] = x;
  TAC_LOP3(x, P[2], v2, c1, 0x96);
  TAC_LOP3(c2, P[2], v2, c1, 0xE8);
  P[2] = x;
  const uint32_t c3 = P[3] & c2;
  P[3] ^= c2;
  const uint32_t c4 = P[4] & c3;
  P[4] ^= c3;
  P[5] ^= c4;
}

// carry-save count of 4 spike words -> planes (u + 2 t1 + 4 t2)
__device__ __forceinline__ void planes_add4(uint32_t *P, uint32_t s0, uint32_t s1, uint32_t s2,
                                            uint32_t s3) {
  uint32_t u, v;
  TAC_LOP3(u, s0, s1, s2, 0x96);
  TAC_LOP3(v, s0, s1, s2, 0xE8);
  const uint32_t u2 = u ^ s3, c = u & s3;
  planes_add3(P, u2, v ^ c, v & c);
}

// --- specialised subtract-reset epilogue (NS LIF steps per group) -------------
// State V (membrane after reset); the drive Y'' = Y - v_th is folded into the bias, so
// one FFMA2 gives U = V_pre - v_th directly:
//   U <- decay V + Y''                     FFMA2 (two neurons)
//   no-spike bit = sign(U)  -> shift register  nsp = (nsp << 1) | (U >> 31)   SHF
//   g = sat(-2^127 U) = [U < 0]            FMUL.SAT with an immediate: one register read
//   V <- U + v_th g                        FFMA2 (no spike: V_pre; spike: V_pre - v_th)
// Channels are visited from the highest to the lowest so that channel c of the
// thread's word lands at bit c after NCH shifts: no per-bit masks, no folding.
// (U = -0 would be a tie V == v_th read as "no spike" by the sign but reset by g;
// U = decay V + Y'' is never -0 in round-to-nearest unless both addends are -0, and
// V = U + v_th g is -0 only for v_init = -0 while Y'' = Y - v_th is never -0.)
__device__ __forceinline__ uint32_t shreg(uint32_t acc, float u) {
  return __funnelshift_l(__float_as_uint(u), acc, 1);  // (acc << 1) | sign(u)
}

// g = [u < 0] = sat(-2^127 u): exactly 0 or 1 for every u (ftz)
__device__ __forceinline__ float sat_nospike(float u) {
  float g;
  asm("mul.rn.ftz.sat.f32 %0, %1, 0fFF000000;" : "=f"(g) : "f"(u));
  return g;
}

template <int NS>
__device__ __forceinline__ void lif_pair_sr(float2 &v, float2 y, float2 dec2, float2 th2,
                                            uint32_t (&nsp)[NS]) {
#pragma unroll
  for (int j = 0; j < NS; ++j) {
    const float2 u = __ffma2_rn(dec2, v, y);
    nsp[j] = shreg(nsp[j], u.y);
    nsp[j] = shreg(nsp[j], u.x);
    const float2 g = make_float2(sat_nospike(u.x), sat_nospike(u.y));
    v = __ffma2_rn(g, th2, u);  // scalar v_th in the operand slot that takes a constant
  }
}

// UT (fp16 first-layer path with C_out = 128): the membrane state V lives in TMEM
// columns [naccs n_total, naccs n_total + 128) (after the accumulators), and is
// streamed through registers 8 channels at a time -- 32 registers fewer per thread.
template <int NCH, int PATH, int NPART>
constexpr bool u_in_tmem() { return PATH != PATH_HALO && NPART == 4 && NCH == 32; }

template <int NCH, int PATH, int NPART, int NS, bool TRAIN>
__device__ __forceinline__ void epilogue_sr(const TcParams &p, uint8_t *smem, uint32_t tmem_base,
                                            uint32_t bar_t_full, uint32_t bar_t_empty, int cid,
                                            int ncl, uint32_t rank, uint32_t warp, uint32_t lane) {
  static_assert(NCH <= 32, "one spike word per thread");
  constexpr int NCHUNK = NCH / 8;
  constexpr bool F16 = PATH != PATH_HALO;
  // (V in TMEM only pays when the K LIF steps per group make registers scarce)
  constexpr bool UT = u_in_tmem<NCH, PATH, NPART>() && NS >= TACSNN_UT_MIN_NS;
  constexpr int NBUF = (NPART == 2 || (F16 && NS <= 4)) ? 2 : 1;  // TMEM prefetch depth (registers)
  const float *sc = reinterpret_cast<const float *>(smem + p.off_scale);
  const int e = (int)warp;
  const int quad = (int)(warp & 3);
  const int half = e >> 2;
  const int g = quad * 4 + (int)(lane >> 3);
  const int c = (int)(lane & 7);
  const int co_base = half * NCH;
  const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
  // fp16 paths: TMEM holds Y 2^e (the prescaled operands, tc_prepare); the LIF runs in
  // the scaled state V 2^e with threshold v_th 2^e -- power-of-two scaling commutes with
  // every fp32 rounding, so spikes and membranes are bitwise those of the unscaled update
  const float ysc = p.ysc, iysc = p.iysc;
  const float2 dec2 = make_float2(p.decay, p.decay), th2 = make_float2(p.vth_s, p.vth_s);
  const int G = p.G, Cout = p.Cout, nwo = p.nwo;
  const long long out_st = p.out_st;
  const uint32_t chmask = NCH >= 32 ? 0xFFFFFFFFu : ((1u << NCH) - 1u);
  const bool pooled = p.pool == 2;
  const bool active_half = co_base < Cout;
  // CTA 0's TMEM-empty barriers, mapped once
  const uint32_t t_empty_remote = ptx::mapa_cluster(bar_t_empty, 0);  // CTA 0's TMEM-empty barriers
  uint32_t it = 0;
  Ring ar;
  TileWalk tw(p, 2 * cid + (int)rank, 2 * ncl);
  for (int pair = cid; pair < p.num_pairs; pair += ncl, tw.step(p)) {
    const int tile = 2 * pair + (int)rank;
    const int b = tw.b, y0 = tw.ty * kTileH, x0 = tw.tx * kTileW;
    const bool tok = tile < p.num_tiles;
    const int y = y0 + g, x = x0 + c;
    const bool valid = tok && y < p.Ho && x < p.Wo;
    // fp32 [B][H'][W'][C_out] offset of this lane's first channel: only the v_init /
    // v_final / y_seq paths need it (skipped, with its 64-bit products, otherwise)
    const long long vbase = (TRAIN || p.v_init || p.v_final)
                                ? (((long long)b * p.Ho + y) * p.Wo + x) * Cout + co_base : 0;
    const int yo = pooled ? (y >> 1) : y, xo = pooled ? (x >> 1) : x;
    const bool store_lane = valid && active_half && (!pooled || (lane & 9) == 0) && yo < p.Hq && xo < p.Wq;
    const uint32_t vmask = (valid && active_half) ? chmask : 0u;
    // this lane's output word (NCH == 32) or the word holding its bit field (NCH < 32)
    const long long obit = (long long)xo * Cout + co_base;
    uint32_t *optr = p.out + (long long)b * p.out_sb + (long long)yo * p.wpr_out +
                     (NCH >= 32 ? (long long)xo * nwo + half : (obit >> 5));
    const int osh = NCH >= 32 ? 0 : (int)(obit & 31);
    // pooled whole-word stores (scatter_pool): the 4 lanes of a 2x2 window share its
    // stores -- lane (wb, wc) = (lane & 1, lane >> 3 & 1) stores the steps s with
    // s % 4 == 2 wc + wb (NS >= 4; NS == 2: steps wb, lanes wc == 0)
    constexpr bool SCAT = NCH >= 32 && NS >= 2;
    const int wb = (int)(lane & 1), wc = (int)((lane >> 3) & 1);
    bool store_w = store_lane;
    if (SCAT && pooled) {
      optr += (long long)(NS >= 4 ? 2 * wc + wb : wb) * out_st;
      store_w = valid && active_half && yo < p.Hq && xo < p.Wq && (NS >= 4 || wc == 0);
    }
    float2 U[UT ? 1 : NCH / 2];
    const uint32_t ucol = tmem_base + lane_addr + (uint32_t)p.naccs * p.n_total + (uint32_t)co_base;
    if (p.v_init) {
#pragma unroll
      for (int ch = 0; ch < NCHUNK; ++ch) {
        uint32_t ub[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int cc = ch * 8 + q;
          float v0 = 0.f;
          if (valid && co_base + cc < Cout) v0 = __ldg(p.v_init + vbase + cc);
          const float u0 = v0 * ysc;
          ub[q] = __float_as_uint(u0);
          if (!UT) {
            if (q & 1) U[UT ? 0 : cc / 2].y = u0; else U[UT ? 0 : cc / 2].x = u0;
          }
        }
        if (UT) ptx::tmem_st8(ucol + ch * 8, ub);
      }
    } else {
      // V_0 = 0 (no per-tile loads)
      const float u0 = 0.f;
      uint32_t ub[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) ub[q] = __float_as_uint(u0);
#pragma unroll
      for (int ch = 0; ch < NCHUNK; ++ch) {
        if (UT) ptx::tmem_st8(ucol + ch * 8, ub);
        if (!UT) {
#pragma unroll
          for (int q = 0; q < 4; ++q) U[UT ? 0 : ch * 4 + q] = make_float2(u0, u0);
        }
      }
    }
    if (UT) ptx::tmem_wait_st();
    uint32_t planes[kPlanes];
#pragma unroll
    for (int pl = 0; pl < kPlanes; ++pl) planes[pl] = 0u;
    int steps_acc = 0;
    // spike words of one group -> per-lane bit-sliced counters (pre-pool, valid pixels
    // only; skipped when the caller asked for no counts), flushed before they overflow
    auto count_group = [&](const uint32_t (&spk)[NS], int k) {
      if (!p.counts) return;  // one uniform branch per group when no counts are asked for
      if (NS == 1) {
        uint32_t cy = spk[0];
#pragma unroll
        for (int pl = 0; pl < kPlanes; ++pl) {
          const uint32_t t = planes[pl] & cy;
          planes[pl] ^= cy;
          cy = t;
        }
      } else if (NS == 2) {
        planes_add3(planes, spk[0] ^ spk[NS - 1], spk[0] & spk[NS - 1], 0u);
      } else {
#pragma unroll
        for (int j = 0; j + 3 < NS; j += 4) planes_add4(planes, spk[j], spk[j + 1], spk[j + 2], spk[j + 3]);
      }
      steps_acc += NS;
      if (steps_acc + NS > (1 << kPlanes) - 1 || k == G - 1) {
        if (tok) {
          uint32_t pw[kPlanes][1];
#pragma unroll
          for (int pl = 0; pl < kPlanes; ++pl) pw[pl][0] = planes[pl];
          flush_counts<1>(p, pw, b, co_base, NCH, lane);
        }
#pragma unroll
        for (int pl = 0; pl < kPlanes; ++pl) planes[pl] = 0u;
        steps_acc = 0;
      }
    };
    // in-warp 2x2 OR-pool (all shuffles first), then branch-free packed stores of the
    // group's output steps
    auto pool_store = [&](const uint32_t (&spk)[NS]) {
      if constexpr (SCAT) if (pooled) {
        // reduce-scatter OR over the window: xor-1 partner keeps the other step parity,
        // xor-8 partner the other step pair -- NS/2 + NS/4 shuffles, NS/4 stores per lane
        uint32_t a[NS / 2 > 0 ? NS / 2 : 1];
#pragma unroll
        for (int i = 0; i < NS / 2; ++i) {
          const uint32_t send = wb ? spk[2 * i] : spk[2 * i + 1];
          const uint32_t keep = wb ? spk[2 * i + 1] : spk[2 * i];
          a[i] = keep | __shfl_xor_sync(0xFFFFFFFFu, send, 1);  // step 2 i + wb
        }
        if constexpr (NS == 2) {
          ptx::st_global_pred(optr, a[0] | __shfl_xor_sync(0xFFFFFFFFu, a[0], 8), store_w);
        } else {
#pragma unroll
          for (int i = 0; i < NS / 4; ++i) {
            const uint32_t send = wc ? a[2 * i] : a[2 * i + 1];
            const uint32_t keep = wc ? a[2 * i + 1] : a[2 * i];
            ptx::st_global_pred(optr + (long long)(4 * i) * out_st,
                                keep | __shfl_xor_sync(0xFFFFFFFFu, send, 8), store_w);  // step 4 i + 2 wc + wb
          }
        }
        optr += (long long)NS * out_st;
        return;
      }
      uint32_t pw[NS];
#pragma unroll
      for (int j = 0; j < NS; ++j) pw[j] = spk[j] | (pooled ? __shfl_xor_sync(0xFFFFFFFFu, spk[j], 1) : 0u);
#pragma unroll
      for (int j = 0; j < NS; ++j) pw[j] |= pooled ? __shfl_xor_sync(0xFFFFFFFFu, pw[j], 8) : 0u;
#pragma unroll
      for (int j = 0; j < NS; ++j) {  // one 64-bit pointer step per stored word
        if (NCH >= 32) {
          ptx::st_global_pred(optr, pw[j], store_lane);
        } else if (store_lane && pw[j]) {
          atomicOr(optr, pw[j] << osh);
        }
        optr += out_st;
      }
    };
    for (int k = 0; k < G; ++k, ++it) {
      const uint32_t acc = ar.i, aph = ar.ph;
      ar.next((uint32_t)p.naccs);
      ptx::mbar_wait(bar_t_full + 8 * acc, aph);
      ptx::tc_fence_after();
      if (e == 0 && lane == 0) trace_mark(p, it, TR_EPI_FULL);
      uint32_t nsp[NS];
#pragma unroll
      for (int j = 0; j < NS; ++j) nsp[j] = 0u;
      const uint32_t tcol = tmem_base + lane_addr + acc * p.n_total + (uint32_t)co_base;
      if (UT && TACSNN_UT_PREFETCH) {
        // chunk by chunk (Y and U in, LIF, U out), the next chunk's loads in flight
        uint32_t dy[2][8], du[2][8];
        ptx::tmem_ld8(tcol + (NCHUNK - 1) * 8, dy[0]);
        ptx::tmem_ld8(ucol + (NCHUNK - 1) * 8, du[0]);
        ptx::tmem_wait_ld_dep(dy[0], du[0]);
#pragma unroll kUtUnroll
        for (int i = 0; i < NCHUNK; ++i) {
          const int ch = NCHUNK - 1 - i, cur = i & 1, nxt = cur ^ 1;
          if (ch > 0) {
            ptx::tmem_ld8(tcol + (ch - 1) * 8, dy[nxt]);
            ptx::tmem_ld8(ucol + (ch - 1) * 8, du[nxt]);
          }
#pragma unroll
          for (int q = 3; q >= 0; --q) {
            float2 u = make_float2(__uint_as_float(du[cur][2 * q]), __uint_as_float(du[cur][2 * q + 1]));
            lif_pair_sr<NS>(u, make_float2(__uint_as_float(dy[cur][2 * q]), __uint_as_float(dy[cur][2 * q + 1])),
                            dec2, th2, nsp);
            du[cur][2 * q] = __float_as_uint(u.x);
            du[cur][2 * q + 1] = __float_as_uint(u.y);
          }
          if (TRAIN && valid && active_half) {
            float yv[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) yv[q] = __uint_as_float(dy[cur][q]);
            store_yseq8(p, k, vbase, ch * 8, Cout - co_base - ch * 8, yv);
          }
          ptx::tmem_st8(ucol + ch * 8, du[cur]);
          if (ch > 0) ptx::tmem_wait_ld_dep(dy[nxt], du[nxt]);
        }
      } else if (UT) {
        // one chunk at a time: Y and U in, LIF, U out
#pragma unroll
        for (int i = 0; i < NCHUNK; ++i) {
          const int ch = NCHUNK - 1 - i;
          uint32_t dy[8], du[8];
          ptx::tmem_ld8(tcol + ch * 8, dy);
          ptx::tmem_ld8(ucol + ch * 8, du);
          ptx::tmem_wait_ld_dep(dy, du);
#pragma unroll
          for (int q = 3; q >= 0; --q) {
            float2 u = make_float2(__uint_as_float(du[2 * q]), __uint_as_float(du[2 * q + 1]));
            lif_pair_sr<NS>(u, make_float2(__uint_as_float(dy[2 * q]), __uint_as_float(dy[2 * q + 1])),
                            dec2, th2, nsp);
            du[2 * q] = __float_as_uint(u.x);
            du[2 * q + 1] = __float_as_uint(u.y);
          }
          if (TRAIN && valid && active_half) {
            float yv[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) yv[q] = __uint_as_float(dy[q]);
            store_yseq8(p, k, vbase, ch * 8, Cout - co_base - ch * 8, yv);
          }
          ptx::tmem_st8(ucol + ch * 8, du);
        }
      } else {
        uint32_t d[NBUF][2][8];  // [buffer][hi/lo][col]
        ptx::tmem_ld8(tcol + (NCHUNK - 1) * 8, d[0][0]);
        if (!F16) ptx::tmem_ld8(tcol + p.Cout_pad + (NCHUNK - 1) * 8, d[0][1]);
        ptx::tmem_wait_ld_dep(d[0][0], d[0][1]);
#pragma unroll
        for (int i = 0; i < NCHUNK; ++i) {
          const int ch = NCHUNK - 1 - i;
          const int cur = NBUF == 2 ? (i & 1) : 0, nxt = NBUF == 2 ? (cur ^ 1) : 0;
          if (NBUF == 2 && ch > 0) {  // prefetch the next lower 8 columns
            ptx::tmem_ld8(tcol + (ch - 1) * 8, d[nxt][0]);
            if (!F16) ptx::tmem_ld8(tcol + p.Cout_pad + (ch - 1) * 8, d[nxt][1]);
          }
          float yv[8];
          if (F16) {
#pragma unroll
            for (int q = 0; q < 8; ++q) yv[q] = __uint_as_float(d[cur][0][q]);
          } else {
            combine8(p, sc, co_base + ch * 8, d[cur][0], d[cur][1], yv);
          }
#pragma unroll
          for (int q = 3; q >= 0; --q)
            lif_pair_sr<NS>(U[UT ? 0 : ch * 4 + q], make_float2(yv[2 * q], yv[2 * q + 1]), dec2, th2, nsp);
          if (TRAIN && valid && active_half) store_yseq8(p, k, vbase, ch * 8, Cout - co_base - ch * 8, yv);
          if (ch > 0) {
            if (NBUF == 1) {
              ptx::tmem_ld8(tcol + (ch - 1) * 8, d[0][0]);
              if (!F16) ptx::tmem_ld8(tcol + p.Cout_pad + (ch - 1) * 8, d[0][1]);
            }
            ptx::tmem_wait_ld_dep(d[nxt][0], d[nxt][1]);
          }
        }
      }
      // accumulator consumed: hand TMEM back to the MMA issuer (UT: the U stores of
      // this group complete before the next group's U loads)
      if (UT) ptx::tmem_wait_st();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_remote_relaxed(t_empty_remote + 8 * acc);
      if (e == 0 && lane == 0) trace_mark(p, it, TR_EPI_RELEASED);

      uint32_t spk[NS];
#pragma unroll
      for (int j = 0; j < NS; ++j) TAC_LOP3(spk[j], nsp[j], vmask, vmask, 0x0C);  // ~nsp & vmask, one LOP3
      pool_store(spk);  // output steps t = k NS + j
      count_group(spk, k);
      if (e == 0 && lane == 0) trace_mark(p, it, TR_EPI_DONE);
    }
    if (p.v_final) {
#pragma unroll
      for (int ch = 0; ch < NCHUNK; ++ch) {
        uint32_t du[8];
        if (UT) {
          uint32_t dz[8];
          ptx::tmem_ld8(ucol + ch * 8, du);
          ptx::tmem_wait_ld_dep(du, dz);
        } else {
#pragma unroll
          for (int q = 0; q < 8; q += 2) {
            du[q] = __float_as_uint(U[UT ? 0 : (ch * 8 + q) / 2].x);
            du[q + 1] = __float_as_uint(U[UT ? 0 : (ch * 8 + q) / 2].y);
          }
        }
        if (valid) {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (co_base + ch * 8 + q < Cout) p.v_final[vbase + ch * 8 + q] = __uint_as_float(du[q]) * iysc;
        }
      }
    }
  }
}

// Generic epilogue: any reset form (subtract / delayed / hard) and a runtime number
// of LIF steps per group, V itself in registers (the subtract-reset configurations
// with 1, 2, 4 or 8 steps run epilogue_sr instead).
template <int NCH, int PATH, int NPART, bool TRAIN>
__device__ __forceinline__ void epilogue_generic(const TcParams &p, uint8_t *smem, uint32_t tmem_base,
                                              uint32_t bar_t_full, uint32_t bar_t_empty, int cid,
                                              int ncl, uint32_t rank, uint32_t warp,
                                              uint32_t lane) {
  constexpr int NWT = NCH >= 32 ? NCH / 32 : 1;  // spike words per epilogue thread
  constexpr int NSM = kMaxSteps;
  const float *sc = reinterpret_cast<const float *>(smem + p.off_scale);
  const int e = (int)warp;                   // epilogue warps are 0 .. 4 NPART - 1
  const int quad = (int)(warp & 3);           // TMEM lane quadrant of this warp
  const int half = e >> 2;                    // channel part
  const int g = quad * 4 + (int)(lane >> 3);  // tile row of this lane's pixel
  const int c = (int)(lane & 7);              // tile column
  const int co_base = half * NCH;
  const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
  // fp16 paths: V, v_th, v_reset in the Y 2^e scale (see epilogue_sr)
  const float ysc = p.ysc, iysc = p.iysc;
  const float decay = p.decay, vth = p.v_th * ysc, vres = p.v_reset * ysc;
  const int nsteps = p.nsteps;
  const int G = p.G, K = p.K, mode = p.mode, nwo = p.nwo, Cout = p.Cout, Cp = p.Cout_pad;
  const uint32_t chmask = NCH >= 32 ? 0xFFFFFFFFu : ((1u << NCH) - 1u);
  const bool pooled = p.pool == 2;
  const bool active_half = co_base < Cout;
  uint32_t it = 0;
  Ring ar;
  TileWalk tw(p, 2 * cid + (int)rank, 2 * ncl);
  for (int pair = cid; pair < p.num_pairs; pair += ncl, tw.step(p)) {
    const TileXY tile = tw.at(p, 2 * pair + (int)rank);
    const int b = tile.b, y0 = tile.y0, x0 = tile.x0;
    const bool tok = tile.ok;
    const int y = y0 + g, x = x0 + c;
    const bool valid = tok && y < p.Ho && x < p.Wo;
    const long long vbase = (((long long)b * p.Ho + y) * p.Wo + x) * Cout + co_base;
    // output word address of this lane (pooled: of its 2x2 window; only lanes with
    // (lane & 9) == 0 store, after the in-warp OR)
    const int yo = pooled ? (y >> 1) : y, xo = pooled ? (x >> 1) : x;
    uint32_t *orow = p.out + (long long)b * p.out_sb + (long long)yo * p.wpr_out;
    const bool store_lane = valid && active_half && (!pooled || (lane & 9) == 0) && yo < p.Hq && xo < p.Wq;
    long long obit = (long long)xo * Cout + co_base;  // NCH < 32: bit offset of the field
    float2 V[NCH / 2];
    uint32_t prev[NWT];
    uint32_t planes[kPlanes][NWT];
    int steps_acc = 0;
#pragma unroll
    for (int w = 0; w < NWT; ++w) {
      prev[w] = 0u;
#pragma unroll
      for (int pl = 0; pl < kPlanes; ++pl) planes[pl][w] = 0u;
    }
#pragma unroll
    for (int cc = 0; cc < NCH; cc += 2) {
      float v0 = 0.f, v1 = 0.f;
      if (p.v_init && valid) {
        if (co_base + cc < Cout) v0 = __ldg(p.v_init + vbase + cc) * ysc;
        if (co_base + cc + 1 < Cout) v1 = __ldg(p.v_init + vbase + cc + 1) * ysc;
      }
      V[cc / 2] = make_float2(v0, v1);
      if (p.reset == 1) {  // reading R4
        if (v0 >= vth) prev[cc / 32] |= 1u << (cc % 32);
        if (v1 >= vth) prev[(cc + 1) / 32] |= 1u << ((cc + 1) % 32);
      }
    }
    for (int k = 0; k < G; ++k, ++it) {
      const uint32_t acc = ar.i, aph = ar.ph;
      ar.next((uint32_t)p.naccs);
      ptx::mbar_wait(bar_t_full + 8 * acc, aph);
      ptx::tc_fence_after();
      if (e == 0 && lane == 0) trace_mark(p, it, TR_EPI_FULL);
      uint32_t inv[NSM][NWT];   // NOT(spike) bits
#pragma unroll
      for (int j = 0; j < NSM; ++j)
#pragma unroll
        for (int w = 0; w < NWT; ++w) inv[j][w] = 0u;
      const uint32_t tcol = tmem_base + lane_addr + acc * p.n_total + (uint32_t)co_base;
      constexpr bool F16 = PATH != PATH_HALO;  // fp32 Y straight from TMEM
      constexpr int NBUF = (NPART == 2 || F16) ? 2 : 1;  // TMEM prefetch depth (registers)
      uint32_t d[NBUF][2][8];                    // [buffer][hi/lo][col]
      ptx::tmem_ld8(tcol, d[0][0]);
      if (!F16) ptx::tmem_ld8(tcol + Cp, d[0][1]);
      ptx::tmem_wait_ld_dep(d[0][0], d[0][1]);
#pragma unroll
      for (int ch = 0; ch < NCH / 8; ++ch) {
        const int cur = NBUF == 2 ? (ch & 1) : 0, nxt = NBUF == 2 ? (cur ^ 1) : 0;
        if (NBUF == 2 && ch + 1 < NCH / 8) {  // prefetch the next 8 columns
          ptx::tmem_ld8(tcol + (ch + 1) * 8, d[nxt][0]);
          if (!F16) ptx::tmem_ld8(tcol + Cp + (ch + 1) * 8, d[nxt][1]);
        }
        float yv[8];
        if (F16) {
#pragma unroll
          for (int i = 0; i < 8; ++i) yv[i] = __uint_as_float(d[cur][0][i]);
        } else {
          combine8(p, sc, co_base + ch * 8, d[cur][0], d[cur][1], yv);
        }
        if (TRAIN && valid && active_half) store_yseq8(p, k, vbase, ch * 8, Cout - co_base - ch * 8, yv);
        {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int cc = ch * 8 + i;
            const uint32_t bm = 1u << (cc % 32);
            float v = (i & 1) ? V[cc / 2].y : V[cc / 2].x;
            const int rs = p.reset;
#pragma unroll
            for (int j = 0; j < kMaxSteps; ++j) {
              if (j < nsteps) {
                if (rs == 0) lif_step<0>(v, yv[i], decay, vth, vres, inv[j][cc / 32], bm, prev[cc / 32]);
                else if (rs == 1) lif_step<1>(v, yv[i], decay, vth, vres, inv[j][cc / 32], bm, prev[cc / 32]);
                else lif_step<2>(v, yv[i], decay, vth, vres, inv[j][cc / 32], bm, prev[cc / 32]);
              }
            }
            if (i & 1) V[cc / 2].y = v; else V[cc / 2].x = v;
          }
        }
        if (ch + 1 < NCH / 8) {
          if (NBUF == 1) {
            ptx::tmem_ld8(tcol + (ch + 1) * 8, d[0][0]);
            if (!F16) ptx::tmem_ld8(tcol + Cp + (ch + 1) * 8, d[0][1]);
          }
          ptx::tmem_wait_ld_dep(d[nxt][0], d[nxt][1]);
        }
      }
      // accumulator consumed: hand TMEM back to the MMA issuer
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_cluster_relaxed(bar_t_empty + 8 * acc, 0);
      if (e == 0 && lane == 0) trace_mark(p, it, TR_EPI_RELEASED);

      // spikes: bit-sliced counters, in-warp 2x2 OR-pool, direct packed stores
      uint32_t spk[NSM][NWT];
#pragma unroll
      for (int j = 0; j < NSM; ++j)
#pragma unroll
        for (int w = 0; w < NWT; ++w)
          spk[j][w] = !valid ? 0u : (~inv[j][w] & chmask);
#pragma unroll
      for (int j = 0; j < NSM; ++j) {
        if (j < nsteps) {
          const int t_out = mode == 1 ? k : k * K + j;
          uint32_t *orow_t = orow + (long long)t_out * p.out_st;
#pragma unroll
          for (int w = 0; w < NWT; ++w) {
            uint32_t s = spk[j][w];
            {  // ripple add of one word into the counters
              uint32_t cy = s;
#pragma unroll
              for (int pl = 0; pl < kPlanes; ++pl) {
                const uint32_t t = planes[pl][w] & cy;
                planes[pl][w] ^= cy;
                cy = t;
              }
            }
            if (pooled) {
              s |= __shfl_xor_sync(0xFFFFFFFFu, s, 1);
              s |= __shfl_xor_sync(0xFFFFFFFFu, s, 8);
            }
            if (store_lane) {
              if (NCH >= 32) {
                const int wd = half * NWT + w;
                if (wd < nwo) orow_t[(long long)xo * nwo + wd] = s;
              } else if (s) {
                atomicOr(orow_t + (obit >> 5), s << (obit & 31));
              }
            }
          }
        }
      }
      steps_acc += nsteps;
      if (p.counts && (steps_acc + nsteps > (1 << kPlanes) - 1 || k == G - 1)) {
        if (tok) flush_counts<NWT>(p, planes, b, co_base, NCH, lane);
        steps_acc = 0;
      }
      if (e == 0 && lane == 0) trace_mark(p, it, TR_EPI_DONE);
    }
    if (p.v_final && valid) {
#pragma unroll
      for (int cc = 0; cc < NCH; cc += 2) {
        const float2 v = V[cc / 2];
        if (co_base + cc < Cout) p.v_final[vbase + cc] = v.x * iysc;
        if (co_base + cc + 1 < Cout) p.v_final[vbase + cc + 1] = v.y * iysc;
      }
    }
  }
}

// fp16-path MMAs of one group: 9 taps x {hi, lo} weight slices x NKC2 K=16 steps
template <int NKC2, int NSL>
__device__ __forceinline__ void mma_tap_h16(int tap, uint32_t d_tmem, uint64_t a_base, uint64_t b_desc0,
                                            uint32_t idf, uint32_t lbo16, uint32_t nhb16) {
  const uint32_t toff = (uint32_t)((tap / 3) * kHaloW + (tap % 3));
#pragma unroll
  for (int sl = 0; sl < NSL; ++sl)
#pragma unroll
    for (int kc2 = 0; kc2 < NKC2; ++kc2)
      ptx::mma_f16_cg2(d_tmem, a_base + (uint64_t)(toff + 2u * kc2 * lbo16),
                       b_desc0 + (uint64_t)(((sl * 9 + tap) * 2 * NKC2 + 2 * kc2) * nhb16), idf,
                       (tap | sl | kc2) ? 1u : 0u);
}
// NSL = 1: packed slices (one MMA per tap computes A W_hi + A W_lo + bias)
template <int NKC2, int NSL>
__device__ __forceinline__ void mma_group_h16(uint32_t d_tmem, uint64_t a_base, uint64_t b_desc0,
                                              uint32_t idf, uint32_t lbo16, uint32_t nhb16) {
  if constexpr (NKC2 == 1) {
#ifdef TACSNN_EXP_TAPS
#pragma unroll
    for (int tap = 0; tap < TACSNN_EXP_TAPS; ++tap) mma_tap_h16<NKC2, NSL>(tap, d_tmem, a_base, b_desc0, idf, lbo16, nhb16);
#else
#pragma unroll
    for (int tap = 0; tap < 9; ++tap) mma_tap_h16<NKC2, NSL>(tap, d_tmem, a_base, b_desc0, idf, lbo16, nhb16);
#endif
  } else {
#pragma unroll 1
    for (int tap = 0; tap < 9; ++tap) mma_tap_h16<NKC2, NSL>(tap, d_tmem, a_base, b_desc0, idf, lbo16, nhb16);
  }
}

// OCC = 2: two CTA pairs per SM pair (small first layers: every role of one pipeline is
// latency-bound, so a second independent pipeline per SM fills the idle issue slots);
// the register budget is then 64 K / (2 x threads) per thread and no setmaxnreg.
template <int NCH, int PATH, int NPART, bool TRAIN, int OCC = 1>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kernel_threads(NPART, OCC), OCC)
    tc_conv_lif_kernel(const __grid_constant__ TcParams p) {
  constexpr int kThreads = kernel_threads(NPART, OCC);
  constexpr int kNpw = kProdWarps + extra_prod_warps(NPART, OCC);
  constexpr int kEpiWarps = epi_warps(NPART);
  extern __shared__ __align__(1024) uint8_t smem[];
  // warp index broadcast from lane 0: the compiler then knows it is warp-uniform and keeps
  // the role / TMEM-address arithmetic derived from it in uniform registers
#if TACSNN_UNIFORM_WARP
  const uint32_t warp = __shfl_sync(0xFFFFFFFFu, threadIdx.x >> 5, 0), lane = threadIdx.x & 31;
#else
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#endif
  const uint32_t rank = ptx::cluster_ctarank();
  const uint32_t sbase = ptx::smem_u32(smem);
  const uint32_t bar_a_full = sbase + p.off_bar;
  const uint32_t bar_a_empty = bar_a_full + 8 * kMaxStages;
  const uint32_t bar_t_full = bar_a_empty + 8 * kMaxStages;
  const uint32_t bar_t_empty = bar_t_full + 8 * kAccs;
  const uint32_t bar_w = bar_t_empty + 8 * kAccs;
  const uint32_t bar_raw = bar_w + 8;
  const uint32_t bar_raw_empty = bar_raw + 8 * kMaxRaw;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + p.off_bar + 8 * kNumBars);
  float *sc = reinterpret_cast<float *>(smem + p.off_scale);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kMaxStages; ++s) {
      ptx::mbar_init(bar_a_full + 8 * s, p.warp_stage ? 2 : 2 * kProdWarps);
      ptx::mbar_init(bar_a_empty + 8 * s, 1);
    }
    for (int a = 0; a < kAccs; ++a) {
      ptx::mbar_init(bar_t_full + 8 * a, 1);
      ptx::mbar_init(bar_t_empty + 8 * a, 2 * kEpiWarps);
    }
    ptx::mbar_init(bar_w, 1);
    for (int r = 0; r < kMaxRaw; ++r) {
      ptx::mbar_init(bar_raw + 8 * r, 1);
      ptx::mbar_init(bar_raw_empty + 8 * r, p.warp_stage ? 1 : kProdWarps);
    }
    ptx::fence_mbar_init();
    if (p.use_tma) ptx::prefetch_tmap(&p.tmap);
    // resident weights: this CTA's int8 slice of every tap
    ptx::mbar_arrive_expect_tx(bar_w, p.w_bytes_cta);
    const unsigned char *src = p.w_img + (size_t)rank * p.w_bytes_cta;
    for (uint32_t off = 0; off < p.w_bytes_cta; off += 16384u)
      ptx::bulk_g2s(sbase + p.off_w + off, src + off, min(16384u, p.w_bytes_cta - off), bar_w);
  }
  if (warp == 0) {
    ptx::tmem_alloc_cg2(ptx::smem_u32(tmem_slot), p.tmem_cols);
    ptx::tmem_relinquish_cg2();
  }
  if (p.split && !p.real) {
    uint32_t *lut_s = reinterpret_cast<uint32_t *>(smem + p.off_lut);
    for (int i = threadIdx.x; i < kLutWords; i += kThreads) lut_s[i] = __ldg(p.lut_g + i);
  }
  for (int i = threadIdx.x; i < 4 * p.Cout_pad; i += kThreads) {
    const float f = p.scale_bias[i];
    sc[i] = (i / p.Cout_pad == 1) ? f : f * p.agg_scale;  // [s1/254 | bias | s1 | s2]
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  ptx::mbar_wait(bar_w, 0);
  ptx::cluster_sync();  // both CTAs' weight slices resident before the first MMA

  const int ncl = (int)ptx::nclusters_x();
  const int cid = (int)ptx::cluster_id_x();

  // Register rebalance: the MMA + producer warpgroup gives registers to the
  // epilogue warpgroups.  The sum must not exceed what the launch allocated
  // (threads x kLaunchRegs), or the increase blocks forever.  Each setmaxnreg
  // sits at the top of its role branch so ptxas sees the register regions.
  constexpr uint32_t kLaunchRegs = NPART == 2 ? 168 : 96;  // ptxas allocation at launch
  constexpr uint32_t kRegsLow = NPART == 2 ? 96 : TACSNN_REGS_LOW4, kRegsHigh = NPART == 2 ? 200 : TACSNN_REGS_HIGH4;
  static_assert(32 * (1 + kProdWarps) * kRegsLow + 32 * epi_warps(NPART) * kRegsHigh <=
                    kernel_threads(NPART) * kLaunchRegs, "register budget");
  // Warp layout: epilogue warps first (the schedulers favour higher warp ids, so the MMA
  // and producer warps win issue slots), or -- kEpiHigh, 16-epilogue-warp kernels -- MMA
  // warp 0, producers 1..3 and the epilogue warps 4..19 on top (the epilogue-bound DVS
  // first layer).  Either way an epilogue warp's TMEM lane quadrant is warp & 3.
  constexpr bool kEpiHigh = (NPART == 4 || (NPART == 2 && TACSNN_EPI_HIGH2)) && kNpw == kProdWarps && TACSNN_EPI_HIGH;
  constexpr uint32_t kEpiBase = kEpiHigh ? 1u + (uint32_t)kNpw : 0u;
  static_assert(kEpiBase % 4 == 0, "epilogue warps must start on a TMEM lane-quadrant boundary");
  const uint32_t kMmaWarp = kEpiHigh ? 0u : (uint32_t)kEpiWarps;
  const bool role_warp = kEpiHigh ? warp < kEpiBase : warp >= kMmaWarp;
  if (role_warp) {
    if constexpr (OCC == 1) ptx::setmaxnreg_dec<kRegsLow>();
    if (warp == kMmaWarp) {
      // ================================ MMA issuer (CTA 0 of the pair) =========
      // The whole warp runs the loop converged (warp-uniform descriptors, no
      // waterfall); one elected lane issues.  Descriptors are built once and only
      // their 14-bit start-address field (addr >> 4, always < 2^14) is advanced.
      // Lane 0 also runs this CTA's raw-halo TMA loader (RawLoader): after the MMAs of
      // group `it` (CTA 0) -- or as its only job (CTA 1) -- it refills the raw slot the
      // producers just released.
      RawLoader loader;
      if (p.use_tma && lane == 0) loader.start(p, sbase, bar_raw, cid, ncl, rank);
      if (rank != 0 && p.use_tma && !p.prod_refill && lane == 0) {
        const uint32_t total = (uint32_t)((p.num_pairs - cid + ncl - 1) / ncl) * (uint32_t)p.G;
        for (uint32_t it = 0; it < total; ++it) loader.refill(p, sbase, bar_raw, bar_raw_empty, it, ncl);
      }
      if (rank == 0) {
        const uint32_t idesc = ptx::idesc_i8(256, p.n_total);
        const uint32_t nhb16 = p.lbo_b >> 4;                        // B rows of this CTA x 16 B
        const uint64_t a_desc0 = ptx::smem_desc(sbase + p.off_a, p.lbo_a, p.sbo_a);
#if TACSNN_BDESC_OPAQUE
        const uint64_t b_desc0_ = ptx::smem_desc(sbase + p.off_w, p.lbo_b, 128u);
#else
        const uint64_t b_desc0 = ptx::smem_desc(sbase + p.off_w, p.lbo_b, 128u);
#endif
        const uint32_t lbo16 = p.lbo_a >> 4, stage16 = p.a_stage_bytes >> 4;
        const int nkc = p.nkc, nkc2 = p.nkc >> 1;
        const uint32_t ns = (uint32_t)p.nstages;
        uint32_t it = 0;
        Ring st, ar;
        for (int pair = cid; pair < p.num_pairs; pair += ncl) {
          for (int k = 0; k < p.G; ++k, ++it) {
            const uint32_t s = st.i, ph = st.ph, acc = ar.i, aph = ar.ph;
            st.next(ns);
            ar.next((uint32_t)p.naccs);
            ptx::mbar_wait(bar_a_full + 8 * s, ph);
            if (lane == 0) trace_mark(p, it, TR_MMA_AFULL);
            // A-full(it) implies every producer released raw slot it % nraw: refill it now,
            // before the MMA issue below (which blocks while the tensor queue is full), or
            // after it (p.refill_early = 0, see tc.cu)
            if (p.refill_early && p.use_tma && !p.prod_refill && lane == 0)
              loader.refill(p, sbase, bar_raw, bar_raw_empty, it, ncl);
            __syncwarp();
            if (lane == 0) trace_mark(p, it, TR_MMA_REFILLED);
            wait_ahead(p, bar_t_empty + 8 * acc, aph ^ 1u);
            ptx::tc_fence_after();
            if (lane == 0) trace_mark(p, it, TR_MMA_READY);
            const uint64_t a_base = a_desc0 + (uint64_t)(s * stage16);
#if TACSNN_BDESC_OPAQUE
            // launder the (loop-invariant) B base through an opaque move each group: the
            // compiler then derives the per-MMA B descriptors in uniform registers next to
            // the MMAs instead of hoisting 9-18 of them into vector registers (R2UR each)
            uint64_t b_desc0 = b_desc0_;
            asm volatile("mov.b64 %0, %0;" : "+l"(b_desc0));
#endif
            const uint32_t d_tmem = tmem_base + acc * p.n_total;
            if (ptx::elect_one()) {
              if (PATH == PATH_HALO) {
  #pragma unroll
                for (int tap = 0; tap < 9; ++tap) {
                  const uint32_t toff = (uint32_t)((tap / 3) * kHaloW + (tap % 3));  // 16-B rows
                  for (int kc2 = 0; kc2 < nkc2; ++kc2) {
                    const uint64_t ad = a_base + (uint64_t)(2u * kc2 * lbo16 + toff);
                    const uint64_t bd = b_desc0 + (uint64_t)((tap * nkc + 2 * kc2) * nhb16);
                    ptx::mma_i8_cg2(d_tmem, ad, bd, idesc, (tap | kc2) ? 1u : 0u);
                  }
                }
              } else {
                // D = sum_taps A_tap (W_hi + W_lo) (+ bias via the constant channel of the
                // centre tap): 9 taps x 2 fp16 slices, K = 16 each, into one accumulator
                // (nkc 16-B chunks per halo pixel; K = 16 = two chunks per MMA; the
                // common chunk counts are fully unrolled: no per-MMA address arithmetic)
                const uint32_t idf = ptx::idesc_f16(256, p.n_total);
                if (p.packed)
                  mma_group_h16<1, 1>(d_tmem, a_base, b_desc0, idf, lbo16, nhb16);
                else if (PATH == PATH_H16 || nkc2 == 1)
                  mma_group_h16<1, 2>(d_tmem, a_base, b_desc0, idf, lbo16, nhb16);
                else
                  mma_group_h16<5, 2>(d_tmem, a_base, b_desc0, idf, lbo16, nhb16);
              }
              ptx::mma_commit_cg2_multicast(bar_a_empty + 8 * s);
              ptx::mma_commit_cg2_multicast(bar_t_full + 8 * acc);
            }
            __syncwarp();
            if (lane == 0) trace_mark(p, it, TR_MMA_ISSUED);
            if (!p.refill_early && p.use_tma && !p.prod_refill && lane == 0)
              loader.refill(p, sbase, bar_raw, bar_raw_empty, it, ncl);
            __syncwarp();
          }
        }
      }
      __syncwarp();
    } else {
      // ================================ producers ================================
      const int ptid = (int)(threadIdx.x - 32 * (kMmaWarp + 1));  // producers follow the MMA warp
      if (p.use_tma) {
        switch (p.K) {
          case 1: producer_role_tma<PATH, 1>(p, sbase, smem, bar_a_full, bar_a_empty, bar_raw, bar_raw_empty, cid, ncl, rank, lane, ptid, kNpw); break;
          case 2: producer_role_tma<PATH, 2>(p, sbase, smem, bar_a_full, bar_a_empty, bar_raw, bar_raw_empty, cid, ncl, rank, lane, ptid, kNpw); break;
          case 3: producer_role_tma<PATH, 3>(p, sbase, smem, bar_a_full, bar_a_empty, bar_raw, bar_raw_empty, cid, ncl, rank, lane, ptid, kNpw); break;
          case 4: producer_role_tma<PATH, 4>(p, sbase, smem, bar_a_full, bar_a_empty, bar_raw, bar_raw_empty, cid, ncl, rank, lane, ptid, kNpw); break;
          case 8: producer_role_tma<PATH, 8>(p, sbase, smem, bar_a_full, bar_a_empty, bar_raw, bar_raw_empty, cid, ncl, rank, lane, ptid, kNpw); break;
          default: producer_role_tma<PATH, 0>(p, sbase, smem, bar_a_full, bar_a_empty, bar_raw, bar_raw_empty, cid, ncl, rank, lane, ptid, kNpw); break;
        }
      } else {
        switch (p.K) {
          case 1: producer_role<PATH, 1>(p, sbase, smem, bar_a_full, bar_a_empty, cid, ncl, rank, lane, ptid, kNpw); break;
          case 2: producer_role<PATH, 2>(p, sbase, smem, bar_a_full, bar_a_empty, cid, ncl, rank, lane, ptid, kNpw); break;
          case 3: producer_role<PATH, 3>(p, sbase, smem, bar_a_full, bar_a_empty, cid, ncl, rank, lane, ptid, kNpw); break;
          case 4: producer_role<PATH, 4>(p, sbase, smem, bar_a_full, bar_a_empty, cid, ncl, rank, lane, ptid, kNpw); break;
          case 8: producer_role<PATH, 8>(p, sbase, smem, bar_a_full, bar_a_empty, cid, ncl, rank, lane, ptid, kNpw); break;
          default: producer_role<PATH, 0>(p, sbase, smem, bar_a_full, bar_a_empty, cid, ncl, rank, lane, ptid, kNpw); break;
        }
      }
    }
  } else {
    if constexpr (OCC == 1) ptx::setmaxnreg_inc<kRegsHigh>();
    // ================================ epilogue =================================
    const int ns = p.reset == 0 ? p.nsteps : 0;
    switch (ns) {
      case 1: epilogue_sr<NCH, PATH, NPART, 1, TRAIN>(p, smem, tmem_base, bar_t_full, bar_t_empty, cid, ncl, rank, warp - kEpiBase, lane); break;
      case 2: epilogue_sr<NCH, PATH, NPART, 2, TRAIN>(p, smem, tmem_base, bar_t_full, bar_t_empty, cid, ncl, rank, warp - kEpiBase, lane); break;
      case 4: epilogue_sr<NCH, PATH, NPART, 4, TRAIN>(p, smem, tmem_base, bar_t_full, bar_t_empty, cid, ncl, rank, warp - kEpiBase, lane); break;
      case 8: epilogue_sr<NCH, PATH, NPART, 8, TRAIN>(p, smem, tmem_base, bar_t_full, bar_t_empty, cid, ncl, rank, warp - kEpiBase, lane); break;
      default: epilogue_generic<NCH, PATH, NPART, TRAIN>(p, smem, tmem_base, bar_t_full, bar_t_empty, cid, ncl, rank, warp - kEpiBase, lane); break;
    }
    }

  // teardown: every role done in both CTAs before TMEM is released
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_cg2(tmem_base, p.tmem_cols);
  }
}

template <int NCH, int PATH, int NPART, bool TRAIN, int OCC = 1>
cudaError_t launch_kernel(const TcParams &p, int nclusters, cudaStream_t stream) {
  auto kern = tc_conv_lif_kernel<NCH, PATH, NPART, TRAIN, OCC>;
  cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void *>(kern), (int)p.smem_bytes);
  if (e != cudaSuccess) return e;
  kern<<<dim3(2 * nclusters), dim3(kernel_threads(NPART, OCC)), p.smem_bytes, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace

// Kernel launchers, one translation unit per operand path and inference / training
// variant (tc_k_*.cu, TAC_TC_PATH / TAC_TC_TRAIN) so the instantiations compile in
// parallel; the training variant also writes the per-group drive y_seq.
// C_out 128: 16 epilogue warps x 32 channels; smaller C_out: 8 warps x C_out / 2.
template <int PATH, bool TRAIN>
cudaError_t tc_launch_path(const TcParams &p, int cout_pad, int nclusters, cudaStream_t stream);
template <> cudaError_t tc_launch_path<PATH_HALO, false>(const TcParams &, int, int, cudaStream_t);
template <> cudaError_t tc_launch_path<PATH_HALO, true>(const TcParams &, int, int, cudaStream_t);
template <> cudaError_t tc_launch_path<PATH_H16, false>(const TcParams &, int, int, cudaStream_t);
template <> cudaError_t tc_launch_path<PATH_H16, true>(const TcParams &, int, int, cudaStream_t);
template <> cudaError_t tc_launch_path<PATH_SPLIT, false>(const TcParams &, int, int, cudaStream_t);
template <> cudaError_t tc_launch_path<PATH_SPLIT, true>(const TcParams &, int, int, cudaStream_t);
#ifdef TAC_TC_PATH
template <>
cudaError_t tc_launch_path<TAC_TC_PATH, TAC_TC_TRAIN>(const TcParams &p, int cout_pad, int nclusters,
                                                     cudaStream_t stream) {
  if constexpr (TAC_TC_PATH != PATH_HALO) {
    if (cout_pad == 32 && p.c32w) {  // 4 epilogue warps x 32 channels: whole-word stores
      if (p.occ == 2) return launch_kernel<32, TAC_TC_PATH, 1, TAC_TC_TRAIN, 2>(p, nclusters, stream);
      return launch_kernel<32, TAC_TC_PATH, 1, TAC_TC_TRAIN>(p, nclusters, stream);
    }
    if (p.occ == 2) {
      if (cout_pad == 16) return launch_kernel<8, TAC_TC_PATH, 2, TAC_TC_TRAIN, 2>(p, nclusters, stream);
      if (cout_pad == 32) return launch_kernel<16, TAC_TC_PATH, 2, TAC_TC_TRAIN, 2>(p, nclusters, stream);
    }
  }
  switch (cout_pad) {
    case 16: return launch_kernel<8, TAC_TC_PATH, 2, TAC_TC_TRAIN>(p, nclusters, stream);
    case 32: return launch_kernel<16, TAC_TC_PATH, 2, TAC_TC_TRAIN>(p, nclusters, stream);
    case 64: return launch_kernel<32, TAC_TC_PATH, 2, TAC_TC_TRAIN>(p, nclusters, stream);
    default: return launch_kernel<32, TAC_TC_PATH, 4, TAC_TC_TRAIN>(p, nclusters, stream);
  }
}
#endif

}  // namespace tacsnn
