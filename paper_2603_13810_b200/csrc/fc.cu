// fc.cu -- the tcgen05 fully connected LIF layer of libtacsnn (H = W = R = S = 1: the
// FC(1600->128) / FC(128->10) layers of the MNIST network and the FC(->512) /
// FC(512->110) head of the DVS network).  A fully connected layer is
// the 1x1 conv of a 1x1 image, so the method is unchanged: per group k the K input
// spike vectors are aggregated, A_k = sum_j c_j S_{kK+j} (Definition TAC, PAPER.md:115;
// c_j = beta^{K-1-j} or the learnable alpha_j), one matrix product
// Y_k = W A_k + b per group (Alg. 1 l.4 / Alg. 2 l.4), and the LIF steps (Alg. 1
// l.5-7, Alg. 2 l.5-9, Eq. (1) for dense, K = 1) with V resident across groups.
//
// GEMM mapping (one CTA, cta_group::1): M = 128 samples (TMEM lane = sample), N = the
// CTA's output-channel tile (32, 64 or 128), K = C_in streamed in chunks of 64 inputs.
//   A (per chunk): producers build the aggregate of 128 samples x 64 inputs from the K
//     packed spike words through a 2^K-entry table (fp16 A_hi | A_lo << 16, built on the
//     host in fp64), K-major, no swizzle: [8 16-B K chunks][128 rows][8 fp16].
//   B (per chunk): W 2^e as fp16 hi + lo slices, [slice][8 K chunks][N rows][8 fp16],
//     precomputed in that order by fc_prepare and bulk-copied (cp.async.bulk) per chunk.
//   D (TMEM, fp32, 2 accumulators of N columns): sum over chunks and K16 steps of
//     A_hi W_hi + A_hi W_lo (+ A_lo W_hi when the aggregate is not exact in fp16).
// The epilogue reads Y = D 2^-e + b and integrates V in registers exactly as the SIMT
// fully connected kernel does (same fp32 operation sequence), so the backward replay
// (backward.cu, V domain) and the y_seq of the training forward are shared.
//
// Warp roles (4 NPART + 3 warps): 4 NPART epilogue warps (TMEM lane quadrant x 32-channel
// part), 1 MMA warp (one elected lane issues), 2 producer warps (64 threads, two sample
// rows each per chunk; thread 0 also issues the weight chunk's bulk copy).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "ptx.cuh"
#include "tc.cuh"

namespace tacsnn {
namespace {

constexpr int kFcM = 128;       // samples per CTA tile
constexpr int kFcKc = 64;       // inputs per K chunk (2 packed spike words)
constexpr int kFcStages = 3;    // A / B stages (producers -> MMA)
constexpr int kFcProd = 2;      // producer warps
constexpr int kFcPlanes = 8;    // bit-sliced spike counters (<= 255 output steps)
constexpr int kFcMaxK = 8;      // 2^K-entry aggregate table
constexpr int kFcLut = 256;

struct FcParams {
  int B, Cin, Cout, N, n_tiles, m_tiles, nchunks, wpr_in, K, G, mode, reset, split;
  long long in_st, in_sb, out_st, out_sb;
  float decay, v_th, v_reset, iysc;
  const uint32_t *in;
  uint32_t *out;
  const float *v_init;
  float *v_final;
  uint32_t *counts;
  float *y_seq;
  const unsigned char *w_img;  // [n tile][chunk][slice][8][N][16 B]
  const float *bias;           // fp32 [Cout]
  const uint32_t *lut;         // [256] fp16 A_hi | A_lo << 16
  uint32_t a_bytes, b_bytes, stage_bytes, off_lut, off_bar, smem_bytes, tmem_cols;
  // two-phase mode (few 128-sample tiles): units are (tile, group, K split) GEMMs whose
  // raw accumulators go to ws [S][G][B][C_out]; fc_lif_from_y then runs the LIF
  int splits, cps;             // K splits, chunks per split
  float *ws;
};

// One unit of work: fused mode = a whole (M, N) tile with all its groups in order (V
// stays resident); GEMM mode = one (tile, group, K split).  Every role walks the same
// unit sequence (CTA-strided).
struct FcUnit {
  int mt, nt, k0, k1, c0, c1, s;
};
template <bool GEMM>
__device__ __forceinline__ int fc_units(const FcParams &p) {
  return p.m_tiles * p.n_tiles * (GEMM ? p.G * p.splits : 1);
}
template <bool GEMM>
__device__ __forceinline__ FcUnit fc_unit(const FcParams &p, int u) {
  FcUnit r;
  int tile = u;
  if (GEMM) {
    const int per = p.G * p.splits;
    tile = u / per;
    const int q = u - tile * per;
    r.k0 = q / p.splits;
    r.s = q - r.k0 * p.splits;
    r.k1 = r.k0 + 1;
    r.c0 = r.s * p.cps;
    r.c1 = min(p.nchunks, r.c0 + p.cps);
  } else {
    r.k0 = 0; r.k1 = p.G; r.c0 = 0; r.c1 = p.nchunks; r.s = 0;
  }
  r.mt = tile / p.n_tiles;
  r.nt = tile - r.mt * p.n_tiles;
  return r;
}

constexpr int fc_threads(int npart) { return 32 * (4 * npart + 1 + kFcProd); }

// ---------------------------------------------------------------- producers ---
// byte b of o[q] = the K-bit table index of input (q + 8 b) of a 32-input word
// (bit j <- frame j of the group)
template <int K>
__device__ __forceinline__ void fc_index_bytes(uint32_t (&o)[8], const uint32_t (&x)[K]) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    uint32_t v = 0;
#pragma unroll
    for (int j = 0; j < K; ++j) v |= ((x[j] >> q) & 0x01010101u) << j;
    o[q] = v;
  }
}

// one sample row of one K chunk: 2 words x K frames -> 8 16-B K chunks of A_hi (and A_lo)
template <int K>
__device__ __forceinline__ void fc_produce_row(const FcParams &p, const uint32_t *lut, uint32_t a_hi,
                                               int row, int b, int k, int chunk) {
#pragma unroll
  for (int wi = 0; wi < 2; ++wi) {
    const int w = 2 * chunk + wi;
    uint32_t x[K];
    const bool ok = b < p.B && w < p.wpr_in;
    const uint32_t *src = p.in + (long long)b * p.in_sb + w + (long long)(k * K) * p.in_st;
#pragma unroll
    for (int j = 0; j < K; ++j) x[j] = ok ? __ldg(src + (long long)j * p.in_st) : 0u;
    uint32_t o[8];
    fc_index_bytes<K>(o, x);
#pragma unroll
    for (int kc = 0; kc < 4; ++kc) {  // inputs 8 kc .. 8 kc + 7 of word w
      uint32_t e[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) e[q] = lut[(o[q] >> (8 * kc)) & 0xFFu];
      const uint32_t dst = a_hi + (uint32_t)((wi * 4 + kc) * kFcM + row) * 16u;
      ptx::st_shared_v4(dst, __byte_perm(e[0], e[1], 0x5410u), __byte_perm(e[2], e[3], 0x5410u),
                        __byte_perm(e[4], e[5], 0x5410u), __byte_perm(e[6], e[7], 0x5410u));
      if (p.split)
        ptx::st_shared_v4(dst + 8u * kFcM * 16u, __byte_perm(e[0], e[1], 0x7632u),
                          __byte_perm(e[2], e[3], 0x7632u), __byte_perm(e[4], e[5], 0x7632u),
                          __byte_perm(e[6], e[7], 0x7632u));
    }
  }
}

template <int K, bool GEMM>
__device__ __forceinline__ void fc_producer(const FcParams &p, uint32_t sbase, const uint32_t *lut,
                                            uint32_t bar_full, uint32_t bar_empty, int ptid, uint32_t lane) {
  uint32_t it = 0;
  const int nunits = fc_units<GEMM>(p);
  for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
    const FcUnit w = fc_unit<GEMM>(p, u);
    const int mt = w.mt, nt = w.nt;
    for (int k = w.k0; k < w.k1; ++k)
      for (int c = w.c0; c < w.c1; ++c, ++it) {
        const uint32_t s = it % kFcStages, ph = (it / kFcStages) & 1u;
        ptx::mbar_wait(bar_empty + 8 * s, ph ^ 1u);
        const uint32_t stage = sbase + s * p.stage_bytes;
        if (ptid == 0) {  // this chunk's weights (both slices), one bulk copy
          ptx::mbar_arrive_expect_tx(bar_full + 8 * s, p.b_bytes);
          ptx::bulk_g2s(stage + p.a_bytes, p.w_img + ((size_t)nt * p.nchunks + c) * p.b_bytes, p.b_bytes,
                        bar_full + 8 * s);
        }
#pragma unroll 1
        for (int row = ptid; row < kFcM; row += 32 * kFcProd)
          fc_produce_row<K>(p, lut, stage, row, mt * kFcM + row, k, c);
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_local(bar_full + 8 * s);
      }
  }
}

// ---------------------------------------------------------------- epilogue ----
__device__ __forceinline__ void fc_planes_add(uint32_t (&P)[kFcPlanes], uint32_t v) {
#pragma unroll
  for (int pl = 0; pl < kFcPlanes; ++pl) {
    const uint32_t c = P[pl] & v;
    P[pl] ^= v;
    v = c;
  }
}

// GEMM mode: the raw accumulators of one unit -> ws [s][k][b][co] (fc_lif_from_y adds
// the splits in order, scales and runs the LIF)
template <int NPART>
__device__ __forceinline__ void fc_store_partials(const FcParams &p, uint32_t tmem_base, uint32_t bar_tfull,
                                                  uint32_t bar_tempty, uint32_t warp, uint32_t lane) {
  const int quad = (int)(warp & 3), part = (int)(warp >> 2);
  const int row = quad * 32 + (int)lane;
  const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
  uint32_t it = 0;
  const int nunits = fc_units<true>(p);
  for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++it) {
    const FcUnit w = fc_unit<true>(p, u);
    const int b = w.mt * kFcM + row;
    const int co0 = w.nt * p.N + part * 32;
    const uint32_t acc = it & 1u, aph = (it >> 1) & 1u;
    ptx::mbar_wait(bar_tfull + 8 * acc, aph);
    ptx::tc_fence_after();
    const uint32_t tcol = tmem_base + lane_addr + acc * (uint32_t)p.N + (uint32_t)(part * 32);
    float *dst = p.ws + (((long long)w.s * p.G + w.k0) * p.B + b) * p.Cout + co0;
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      uint32_t d[8], dz[8];
      ptx::tmem_ld8(tcol + cc * 8, d);
      ptx::tmem_wait_ld_dep(d, dz);
      if (b < p.B) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (co0 + cc * 8 + q < p.Cout) dst[cc * 8 + q] = __uint_as_float(d[q]);
      }
    }
    ptx::tc_fence_before();
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive_local(bar_tempty + 8 * acc);
  }
}

template <int NPART, int NS, bool TRAIN>
__device__ __forceinline__ void fc_epilogue(const FcParams &p, uint32_t tmem_base, uint32_t bar_tfull,
                                            uint32_t bar_tempty, uint32_t warp, uint32_t lane) {
  const int quad = (int)(warp & 3), part = (int)(warp >> 2);
  const int row = quad * 32 + (int)lane;
  const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
  const float decay = p.decay, vth = p.v_th, vres = p.v_reset, iysc = p.iysc;
  uint32_t it = 0;
  const int ntiles = p.m_tiles * p.n_tiles;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int mt = tile / p.n_tiles, nt = tile - mt * p.n_tiles;
    const int b = mt * kFcM + row;
    const int co0 = nt * p.N + part * 32;
    const bool bok = b < p.B;
    const int nvalid = min(32, max(0, p.Cout - co0));
    const uint32_t cmask = nvalid >= 32 ? 0xFFFFFFFFu : ((1u << nvalid) - 1u);
    const uint32_t vmask = bok ? cmask : 0u;
    float V[32];
#pragma unroll
    for (int c = 0; c < 32; ++c)
      V[c] = (p.v_init && bok && c < nvalid) ? __ldg(p.v_init + (long long)b * p.Cout + co0 + c) : 0.f;
    uint32_t sprev = 0u;  // pending delayed reset (reading R4): [v_init >= v_th]
    if (p.reset == 1) {
#pragma unroll
      for (int c = 0; c < 32; ++c) sprev |= (V[c] >= vth ? 1u : 0u) << c;
    }
    uint32_t planes[kFcPlanes];
#pragma unroll
    for (int pl = 0; pl < kFcPlanes; ++pl) planes[pl] = 0u;
    uint32_t *optr = p.out + (long long)b * p.out_sb + (co0 >> 5);
    for (int k = 0; k < p.G; ++k, ++it) {
      const uint32_t acc = it & 1u, aph = (it >> 1) & 1u;
      ptx::mbar_wait(bar_tfull + 8 * acc, aph);
      ptx::tc_fence_after();
      uint32_t words[NS];
#pragma unroll
      for (int j = 0; j < NS; ++j) words[j] = 0u;
      const uint32_t tcol = tmem_base + lane_addr + acc * (uint32_t)p.N + (uint32_t)(part * 32);
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        uint32_t d[8], dz[8];
        ptx::tmem_ld8(tcol + cc * 8, d);
        ptx::tmem_wait_ld_dep(d, dz);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int c = cc * 8 + q;
          const int co = co0 + c;
          const float y = fmaf(__uint_as_float(d[q]), iysc, c < nvalid ? __ldg(p.bias + co) : 0.f);
          if (TRAIN && bok && c < nvalid) p.y_seq[((long long)k * p.B + b) * p.Cout + co] = y;
          float v = V[c];
#pragma unroll
          for (int j = 0; j < NS; ++j) {  // the SIMT fc kernel's sequence (Eq. 1 / Alg. 1-2)
            v = fmaf(decay, v, y);
            if (p.reset == 1 && ((sprev >> c) & 1u)) v -= vth;
            const bool s = v >= vth;
            if (s) {
              if (p.reset == 0) v -= vth;
              else if (p.reset == 2) v = vres;
            }
            if (p.reset == 1) sprev = (sprev & ~(1u << c)) | ((s ? 1u : 0u) << c);
            words[j] |= (s ? 1u : 0u) << c;
          }
          V[c] = v;
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_local(bar_tempty + 8 * acc);
#pragma unroll
      for (int j = 0; j < NS; ++j) {
        const uint32_t w = words[j] & vmask;
        if (bok && nvalid > 0) *optr = w;
        optr += p.out_st;
        if (p.counts) fc_planes_add(planes, w);
      }
    }
    if (bok && p.v_final) {
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (c < nvalid) p.v_final[(long long)b * p.Cout + co0 + c] = V[c];
    }
    if (bok && p.counts) {
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        uint32_t n = 0;
#pragma unroll
        for (int pl = 0; pl < kFcPlanes; ++pl) n |= ((planes[pl] >> c) & 1u) << pl;
        if (c < nvalid) p.counts[(long long)b * p.Cout + co0 + c] = n;
      }
    }
  }
}

// ---------------------------------------------------------------- kernel ------
template <int NPART, int NS, bool TRAIN, bool GEMM = false>
__global__ void __launch_bounds__(fc_threads(NPART), 1) fc_lif_tc_kernel(const __grid_constant__ FcParams p) {
  constexpr int kEpiWarps = 4 * NPART;
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t warp = __shfl_sync(0xFFFFFFFFu, threadIdx.x >> 5, 0), lane = threadIdx.x & 31;
  const uint32_t sbase = ptx::smem_u32(smem);
  const uint32_t bar_full = sbase + p.off_bar;
  const uint32_t bar_empty = bar_full + 8 * kFcStages;
  const uint32_t bar_tfull = bar_empty + 8 * kFcStages;
  const uint32_t bar_tempty = bar_tfull + 16;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + p.off_bar + 8 * (2 * kFcStages + 4));
  uint32_t *lut = reinterpret_cast<uint32_t *>(smem + p.off_lut);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kFcStages; ++s) {
      ptx::mbar_init(bar_full + 8 * s, kFcProd + 1);  // producer warps + the weight copy's expect_tx
      ptx::mbar_init(bar_empty + 8 * s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(bar_tfull + 8 * a, 1);
      ptx::mbar_init(bar_tempty + 8 * a, kEpiWarps);
    }
    ptx::fence_mbar_init();
  }
  for (int i = threadIdx.x; i < kFcLut; i += blockDim.x) lut[i] = __ldg(p.lut + i);
  if (warp == (uint32_t)kEpiWarps) {
    ptx::tmem_alloc_cg1(ptx::smem_u32(tmem_slot), p.tmem_cols);
    ptx::tmem_relinquish_cg1();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp < (uint32_t)kEpiWarps) {
    if constexpr (GEMM)
      fc_store_partials<NPART>(p, tmem_base, bar_tfull, bar_tempty, warp, lane);
    else
      fc_epilogue<NPART, NS, TRAIN>(p, tmem_base, bar_tfull, bar_tempty, warp, lane);
  } else if (warp == (uint32_t)kEpiWarps) {
    // MMA issuer: per group, all chunks into one accumulator; commits free the stage
    // and, after the last chunk, hand the accumulator to the epilogue
    const uint32_t idesc = ptx::idesc_f16(kFcM, (uint32_t)p.N);
    const uint32_t lbo_a = kFcM * 16u, lbo_b = (uint32_t)p.N * 16u;
    uint32_t it = 0, g = 0;
    const int nunits = fc_units<GEMM>(p);
    for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
      const FcUnit w = fc_unit<GEMM>(p, u);
      for (int k = w.k0; k < w.k1; ++k, ++g) {
        const uint32_t acc = g & 1u, aph = (g >> 1) & 1u;
        ptx::mbar_wait(bar_tempty + 8 * acc, aph ^ 1u);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * (uint32_t)p.N;
        for (int c = w.c0; c < w.c1; ++c, ++it) {
          const uint32_t s = it % kFcStages, ph = (it / kFcStages) & 1u;
          ptx::mbar_wait(bar_full + 8 * s, ph);
          ptx::tc_fence_after();
          const uint32_t stage = sbase + s * p.stage_bytes;
          if (ptx::elect_one()) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {  // K = 16 per MMA: two 16-B K chunks
              const uint64_t ahi = ptx::smem_desc(stage + ks * 2 * lbo_a, lbo_a, 128u);
              const uint64_t alo = ptx::smem_desc(stage + 8 * lbo_a + ks * 2 * lbo_a, lbo_a, 128u);
              const uint64_t bhi = ptx::smem_desc(stage + p.a_bytes + ks * 2 * lbo_b, lbo_b, 128u);
              const uint64_t blo = ptx::smem_desc(stage + p.a_bytes + 8 * lbo_b + ks * 2 * lbo_b, lbo_b, 128u);
              ptx::mma_f16_cg1(d_tmem, ahi, bhi, idesc, (c != w.c0 || ks) ? 1u : 0u);
              ptx::mma_f16_cg1(d_tmem, ahi, blo, idesc, 1u);
              if (p.split) ptx::mma_f16_cg1(d_tmem, alo, bhi, idesc, 1u);
            }
            ptx::mma_commit_cg1(bar_empty + 8 * s);
            if (c == w.c1 - 1) ptx::mma_commit_cg1(bar_tfull + 8 * acc);
          }
          __syncwarp();
        }
      }
    }
  } else {
    const int ptid = (int)(threadIdx.x - 32 * (kEpiWarps + 1));
    switch (p.K) {
      case 1: fc_producer<1, GEMM>(p, sbase, lut, bar_full, bar_empty, ptid, lane); break;
      case 2: fc_producer<2, GEMM>(p, sbase, lut, bar_full, bar_empty, ptid, lane); break;
      case 3: fc_producer<3, GEMM>(p, sbase, lut, bar_full, bar_empty, ptid, lane); break;
      case 4: fc_producer<4, GEMM>(p, sbase, lut, bar_full, bar_empty, ptid, lane); break;
      case 5: fc_producer<5, GEMM>(p, sbase, lut, bar_full, bar_empty, ptid, lane); break;
      case 6: fc_producer<6, GEMM>(p, sbase, lut, bar_full, bar_empty, ptid, lane); break;
      case 7: fc_producer<7, GEMM>(p, sbase, lut, bar_full, bar_empty, ptid, lane); break;
      default: fc_producer<8, GEMM>(p, sbase, lut, bar_full, bar_empty, ptid, lane); break;
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == (uint32_t)kEpiWarps) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_cg1(tmem_base, p.tmem_cols);
  }
}

template <int NPART, int NS, bool TRAIN, bool GEMM = false>
cudaError_t fc_launch_kernel(const FcParams &p, int grid, cudaStream_t st) {
  auto kern = fc_lif_tc_kernel<NPART, NS, TRAIN, GEMM>;
  cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void *>(kern), (int)p.smem_bytes);
  if (e != cudaSuccess) return e;
  kern<<<grid, fc_threads(NPART), p.smem_bytes, st>>>(p);
  return cudaGetLastError();
}

template <int NPART, bool TRAIN>
cudaError_t fc_launch_ns(const FcParams &p, int ns, int grid, cudaStream_t st) {
  switch (ns) {
    case 1: return fc_launch_kernel<NPART, 1, TRAIN>(p, grid, st);
    case 2: return fc_launch_kernel<NPART, 2, TRAIN>(p, grid, st);
    case 4: return fc_launch_kernel<NPART, 4, TRAIN>(p, grid, st);
    default: return fc_launch_kernel<NPART, 8, TRAIN>(p, grid, st);
  }
}

// Phase 2 of the two-phase mode: one warp per (sample, 32 outputs), lane = output
// channel; Y_k = (sum over the K splits in order) 2^-e + b, then the LIF with the fused
// epilogue's fp32 sequence; spike words by ballot.
template <int NS>
__global__ void __launch_bounds__(32) fc_lif_from_y_kernel(const FcParams p) {
  const int b = blockIdx.x, lane = threadIdx.x, co = blockIdx.y * 32 + lane;
  const bool ok = co < p.Cout;
  float V = (ok && p.v_init) ? __ldg(p.v_init + (long long)b * p.Cout + co) : 0.f;
  bool sprev = p.reset == 1 && V >= p.v_th;
  const float bias = ok ? __ldg(p.bias + co) : 0.f;
  uint32_t cnt = 0;
  uint32_t *optr = p.out + (long long)b * p.out_sb + blockIdx.y;
  for (int k = 0; k < p.G; ++k) {
    float acc = 0.f;
    for (int s = 0; s < p.splits; ++s)
      acc += ok ? __ldg(p.ws + (((long long)s * p.G + k) * p.B + b) * p.Cout + co) : 0.f;
    const float y = fmaf(acc, p.iysc, bias);
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      float v = fmaf(p.decay, V, y);
      if (p.reset == 1 && sprev) v -= p.v_th;
      const bool sp = ok && v >= p.v_th;
      if (sp) {
        if (p.reset == 0) v -= p.v_th;
        else if (p.reset == 2) v = p.v_reset;
        ++cnt;
      }
      sprev = sp;
      V = v;
      const uint32_t bits = __ballot_sync(0xFFFFFFFFu, sp);
      if (lane == 0) *optr = bits;
      optr += p.out_st;
    }
  }
  if (ok && p.v_final) p.v_final[(long long)b * p.Cout + co] = V;
  if (ok && p.counts) p.counts[(long long)b * p.Cout + co] = cnt;
}

// ---------------------------------------------------------------- host --------
int fc_n_tile(int Cout) { return Cout <= 32 ? 32 : (Cout <= 64 ? 64 : 128); }
int fc_nchunks(int Cin) { return (Cin + kFcKc - 1) / kFcKc; }
int fc_group(const tac_conv_lif_desc *d) { return d->mode == TAC_MODE_DENSE ? 1 : d->K; }

// aggregate weights c_j of one group (PAPER.md:115 / :427) and the table of all 2^K sums
std::vector<double> fc_table(const tac_conv_lif_desc *d) {
  const int K = fc_group(d);
  std::vector<double> t(kFcLut, 0.0);
  for (int idx = 0; idx < (1 << K); ++idx) {
    double a = 0.0;
    for (int j = 0; j < K; ++j)
      if ((idx >> j) & 1) {
        const bool alpha = d->agg_weights && d->mode != TAC_MODE_DENSE;
        a += alpha ? (double)d->agg_weights[j] : std::pow((double)d->beta, (double)(K - 1 - j));
      }
    t[idx] = a;
  }
  return t;
}
// the aggregate needs the A_lo term when a table entry is not exact in fp16
bool fc_split(const tac_conv_lif_desc *d) {
  for (double a : fc_table(d))
    if ((double)__half2float(__double2half(a)) != a) return true;
  return false;
}

int fc_groups(const tac_conv_lif_desc *d) {
  const int K = fc_group(d);
  return (d->T + K - 1) / K;
}

// Two-phase plan: 0 = fused (enough (M, N) tiles to fill the GPU), else the number of K
// splits S so that (M tiles x N tiles x groups x S) units cover the 148 SMs
int fc_two_phase_splits(const tac_conv_lif_desc *d) {
  const int N = fc_n_tile(d->C_out), nt = (d->C_out + N - 1) / N, mt = (d->B + kFcM - 1) / kFcM;
  if (mt * nt >= 74) return 0;
  const int units = mt * nt * fc_groups(d);
  return std::max(1, std::min(fc_nchunks(d->C_in), (148 + units - 1) / units));
}

}  // namespace

size_t fc_ws_bytes(const tac_conv_lif_desc *d) {
  const int S = fc_two_phase_splits(d);
  return S ? (size_t)S * fc_groups(d) * d->B * d->C_out * 4 : 0;
}

bool fc_is_fc(const tac_conv_lif_desc *d) {
  return d->H == 1 && d->W == 1 && d->R == 1 && d->S == 1 && d->pad == 0 && d->stride == 1 &&
         d->input_kind == TAC_INPUT_SPIKES;
}

const char *fc_reason(const tac_conv_lif_desc *d) {
  if (!fc_is_fc(d)) return "not a fully connected layer";
  const int K = fc_group(d);
  if (K > kFcMaxK) return "fully connected tcgen05 layer needs K <= 8";
  const int ns = d->mode == TAC_MODE_TACTP ? K : 1;
  if (!(ns == 1 || ns == 2 || ns == 4 || ns == 8)) return "fully connected tcgen05 layer needs 1, 2, 4 or 8 LIF steps per group";
  if (d->out_pool != 1) return "fully connected layers do not pool";
  const int T_out = d->mode == TAC_MODE_TAC ? d->T / K : d->T;
  if (T_out > 255) return "fully connected tcgen05 layer needs <= 255 output steps";
  for (double a : fc_table(d))
    if (std::fabs(a) > 16384.0) return "aggregate exceeds the fp16 operand range";
  return nullptr;
}

size_t fc_weights_bytes(const tac_conv_lif_desc *d) {
  const int N = fc_n_tile(d->C_out), nt = (d->C_out + N - 1) / N;
  return (size_t)nt * fc_nchunks(d->C_in) * 256 * (size_t)N + 4 * kFcLut;
}

int fc_prepare(const tac_conv_lif_desc *d, const float *weight, unsigned char *dst) {
  const int Co = d->C_out, Ci = d->C_in, N = fc_n_tile(Co), nt = (Co + N - 1) / N, nch = fc_nchunks(Ci);
  double mx = 0.0;
  for (size_t i = 0; i < (size_t)Co * Ci; ++i) mx = std::max(mx, std::fabs((double)weight[i]));
  // layer prescale 2^e: the largest |w| lands in [1, 2), so the fp16 hi + lo pair keeps
  // ~22 bits of every weight relative to the layer's scale; the epilogue multiplies by 2^-e
  const int e = mx > 0.0 ? std::max(-60, std::min(60, -std::ilogb(mx))) : 0;
  const double sc = std::ldexp(1.0, e);
  const size_t chunk = 256 * (size_t)N;
  __half *h = reinterpret_cast<__half *>(dst);
  std::memset(dst, 0, fc_weights_bytes(d));
  for (int t = 0; t < nt; ++t)
    for (int c = 0; c < nch; ++c)
      for (int n = 0; n < N; ++n) {
        const int co = t * N + n;
        if (co >= Co) continue;
        for (int kk = 0; kk < kFcKc; ++kk) {
          const int ci = c * kFcKc + kk;
          if (ci >= Ci) break;
          const double w = (double)weight[(size_t)co * Ci + ci] * sc;
          const __half hi = __double2half(w);
          const __half lo = __double2half(w - (double)__half2float(hi));
          // [slice][kc][n][8]: halves index within the chunk
          const size_t base = ((size_t)t * nch + c) * chunk / 2;
          const size_t off = ((size_t)(kk / 8) * N + n) * 8 + kk % 8;
          h[base + off] = hi;
          h[base + (size_t)8 * N * 8 + off] = lo;
        }
      }
  uint32_t *lut = reinterpret_cast<uint32_t *>(dst + (size_t)nt * nch * chunk);
  const std::vector<double> tab = fc_table(d);
  for (int i = 0; i < kFcLut; ++i) {
    const __half hi = __double2half(tab[i]);
    const __half lo = __double2half(tab[i] - (double)__half2float(hi));
    lut[i] = (uint32_t)__half_as_ushort(hi) | ((uint32_t)__half_as_ushort(lo) << 16);
  }
  return e;
}

int fc_launch(const tac_conv_lif_desc *d, const LayerParams &lp, const unsigned char *img, void *stream,
              int *launches) {
  FcParams p{};
  p.B = lp.B; p.Cin = lp.Cin; p.Cout = lp.Cout;
  p.N = fc_n_tile(lp.Cout);
  p.n_tiles = (lp.Cout + p.N - 1) / p.N;
  p.m_tiles = (lp.B + kFcM - 1) / kFcM;
  p.nchunks = fc_nchunks(lp.Cin);
  p.wpr_in = lp.wpr_in;
  p.K = lp.K; p.G = lp.G; p.mode = lp.mode; p.reset = lp.reset;
  p.split = fc_split(d) ? 1 : 0;
  p.in_st = lp.in_st; p.in_sb = lp.in_sb; p.out_st = lp.out_st; p.out_sb = lp.out_sb;
  p.decay = lp.decay; p.v_th = lp.v_th; p.v_reset = lp.v_reset;
  p.iysc = (float)std::ldexp(1.0, -lp.yscale_exp);
  p.in = lp.in; p.out = lp.out; p.v_init = lp.v_init; p.v_final = lp.v_final; p.counts = lp.counts;
  p.y_seq = lp.y_seq;
  p.w_img = img;
  p.bias = lp.bias;
  p.b_bytes = 256u * (uint32_t)p.N;
  p.lut = reinterpret_cast<const uint32_t *>(img + (size_t)p.n_tiles * p.nchunks * p.b_bytes);
  p.a_bytes = 2u * 8u * kFcM * 16u;  // A_hi | A_lo
  p.stage_bytes = p.a_bytes + p.b_bytes;
  p.off_lut = kFcStages * p.stage_bytes;
  p.off_bar = p.off_lut + 4 * kFcLut;
  p.smem_bytes = p.off_bar + 8 * (2 * kFcStages + 4) + 16;
  p.tmem_cols = p.N <= 16 ? 32u : 2u * (uint32_t)p.N;
  const int ns = lp.nsteps;
  cudaStream_t st = (cudaStream_t)stream;
  const bool train = lp.y_seq != nullptr;
  const int npart = p.N / 32;
  cudaError_t e;
  p.splits = train ? 0 : fc_two_phase_splits(d);
  if (p.splits && lp.ws && lp.ws_bytes >= fc_ws_bytes(d)) {
    // two-phase: the GEMM units fill the GPU, then one warp per (sample, 32 outputs) integrates
    p.cps = (p.nchunks + p.splits - 1) / p.splits;
    p.splits = (p.nchunks + p.cps - 1) / p.cps;  // no empty split
    p.ws = static_cast<float *>(lp.ws);
    const int units = p.m_tiles * p.n_tiles * p.G * p.splits;
    const int g1 = std::max(1, std::min(units, 148));
    if (npart == 1) e = fc_launch_kernel<1, 1, false, true>(p, g1, st);
    else if (npart == 2) e = fc_launch_kernel<2, 1, false, true>(p, g1, st);
    else e = fc_launch_kernel<4, 1, false, true>(p, g1, st);
    ++*launches;
    if (e != cudaSuccess) return (int)e;
    const dim3 g2((unsigned)p.B, (unsigned)((p.Cout + 31) / 32));
    switch (ns) {
      case 1: fc_lif_from_y_kernel<1><<<g2, 32, 0, st>>>(p); break;
      case 2: fc_lif_from_y_kernel<2><<<g2, 32, 0, st>>>(p); break;
      case 4: fc_lif_from_y_kernel<4><<<g2, 32, 0, st>>>(p); break;
      default: fc_lif_from_y_kernel<8><<<g2, 32, 0, st>>>(p); break;
    }
    ++*launches;
    return (int)cudaGetLastError();
  }
  p.splits = 1;
  p.cps = p.nchunks;
  const int grid = std::max(1, std::min(p.m_tiles * p.n_tiles, 148));
  if (npart == 1) e = train ? fc_launch_ns<1, true>(p, ns, grid, st) : fc_launch_ns<1, false>(p, ns, grid, st);
  else if (npart == 2) e = train ? fc_launch_ns<2, true>(p, ns, grid, st) : fc_launch_ns<2, false>(p, ns, grid, st);
  else e = train ? fc_launch_ns<4, true>(p, ns, grid, st) : fc_launch_ns<4, false>(p, ns, grid, st);
  ++*launches;
  return (int)e;
}

}  // namespace tacsnn
