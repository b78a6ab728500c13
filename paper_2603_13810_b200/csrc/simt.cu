// simt.cu -- the SIMT engine of libtacsnn: an fp32 direct-convolution Conv-LIF
// kernel for any R/S/stride/pad/K/beta (the engine for layers the tcgen05 path
// does not take, and the GPU parity anchor), plus the packed-format utilities.
//
// One thread owns one PRE-pool output pixel (b, y, x) and up to 32 output
// channels; its membrane V lives in registers for the whole sequence (all G
// groups).  Per group it aggregates the K input frames on the fly
// (A_k = sum_j beta^{K-1-j} S_{kK+j}) while it convolves, so the
// conv runs G = T/K times (Alg. 1 l.3-4, Alg. 2 l.3-4), then it runs the LIF
// steps (Alg. 1 l.5-7 / Alg. 2 l.5-9 / Eq. (1)) and ORs its spike bits into the
// packed output (fused 2x2 OR-pool when pool == 2; the output is zeroed first by
// zero_outputs_kernel in the same stream).
#include <cuda_runtime.h>

#include <algorithm>

#include "layer.cuh"

namespace tacsnn {

namespace {

__global__ void zero_outputs_kernel(uint32_t *out, int T_out, int B, long long plane,
                                    long long st, long long sb, uint32_t *counts,
                                    long long ncounts) {
  const long long per_tb = plane;
  const long long total = (long long)T_out * B * per_tb;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    long long tb = i / per_tb, o = i - tb * per_tb;
    long long t = tb / B, b = tb - t * B;
    out[t * st + b * sb + o] = 0u;
  }
  if (counts)
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < ncounts;
         i += (long long)gridDim.x * blockDim.x)
      counts[i] = 0u;
}

__global__ void add_u32_kernel(uint32_t *dst, const uint32_t *src, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] += src[i];
}

// Fully connected LIF layer (a 1x1 conv of a 1x1 image: H = W = R = S = 1): one block
// per (sample, 32 output channels); the 8 warps split the C_in inputs (lane = output
// channel, weights [C_in][C_out] read coalesced, the group aggregate of input i
// broadcast), partial sums meet in shared memory, warp 0 keeps V in registers for the
// whole sequence and writes each step's 32 spike bits with one ballot.
constexpr int FC_WARPS = 8;
__global__ void __launch_bounds__(32 * FC_WARPS) fc_lif_kernel(const LayerParams p) {
  __shared__ float part[FC_WARPS][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x, co = blockIdx.y * 32 + lane;
  const bool cok = co < p.Cout;
  float V = 0.f;
  int cnt = 0;
  bool sprev = false;  // pending delayed reset (reading R4)
  if (warp == 0 && cok) {
    V = p.v_init ? p.v_init[(long long)b * p.Cout + co] : 0.f;
    sprev = p.reset == RESET_DELAYED && V >= p.v_th;
  }
  const long long rowb = (long long)b * p.in_sb;
  for (int g = 0; g < p.G; ++g) {
    float y = 0.f;
#pragma unroll 4
    for (int i = warp; i < p.Cin; i += FC_WARPS) {
      float a = 0.f;  // A_g of input i
      if (p.xin) {
        for (int j = 0; j < p.K; ++j) a = fmaf(p.coef[j], __ldg(p.xin + (long long)(g * p.K + j) * p.in_st + rowb + i), a);
      } else {
        for (int j = 0; j < p.K; ++j)
          if ((__ldg(p.in + (long long)(g * p.K + j) * p.in_st + rowb + (i >> 5)) >> (i & 31)) & 1u) a += p.coef[j];
      }
      if (a != 0.f && cok) y = fmaf(__ldg(p.w + (long long)i * p.Cout + co), a, y);
    }
    part[warp][lane] = y;
    __syncthreads();
    if (warp == 0) {
      float Y = cok ? __ldg(p.bias + co) : 0.f;
#pragma unroll
      for (int w = 0; w < FC_WARPS; ++w) Y += part[w][lane];
      if (p.y_seq && cok) p.y_seq[((long long)g * p.B + b) * p.Cout + co] = Y;
      for (int j = 0; j < p.nsteps; ++j) {
        float v = fmaf(p.decay, V, Y);
        if (p.reset == RESET_DELAYED && sprev) v -= p.v_th;
        const bool s = cok && v >= p.v_th;
        if (s) {
          if (p.reset == RESET_SUBTRACT) v -= p.v_th;
          else if (p.reset == RESET_HARD) v = p.v_reset;
          ++cnt;
        }
        sprev = s;
        V = v;
        const uint32_t bits = __ballot_sync(0xFFFFFFFFu, s);
        const int t_out = (p.mode == MODE_TAC) ? g : g * p.K + j;
        if (lane == 0)
          p.out[(long long)t_out * p.out_st + (long long)b * p.out_sb + (blockIdx.y * 32 >> 5)] = bits;
      }
    }
    __syncthreads();
  }
  if (warp == 0 && cok) {
    if (p.v_final) p.v_final[(long long)b * p.Cout + co] = V;
    if (p.counts && cnt) atomicAdd(p.counts + (long long)b * p.Cout + co, (uint32_t)cnt);
  }
}

constexpr int CH = 32;  // output channels per thread

__global__ void __launch_bounds__(128) simt_conv_lif_kernel(const LayerParams p) {
  const long long npix = (long long)p.B * p.Ho * p.Wo;
  const long long pix = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (pix >= npix) return;
  const int co0 = blockIdx.y * CH;
  const int nch = min(CH, p.Cout - co0);
  const int b = (int)(pix / ((long long)p.Ho * p.Wo));
  const int rem = (int)(pix - (long long)b * p.Ho * p.Wo);
  const int y = rem / p.Wo, x = rem - (rem / p.Wo) * p.Wo;

  float V[CH];
  int cnt[CH];
  uint32_t sprev = 0u;  // pending delayed reset, one bit per channel
  const long long vbase = pix * p.Cout + co0;  // [B][Ho][Wo][Cout]
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    V[c] = (p.v_init && c < nch) ? p.v_init[vbase + c] : 0.f;
    cnt[c] = 0;
    if (p.reset == RESET_DELAYED && V[c] >= p.v_th) sprev |= 1u << c;  // reading R4
  }

  // output location of this pixel (pooled or not)
  const int yo = p.pool == 2 ? y >> 1 : y, xo = p.pool == 2 ? x >> 1 : x;
  const long long obit = (long long)xo * p.Cout + co0;
  const int ow = (int)(obit >> 5), osh = (int)(obit & 31);

  for (int g = 0; g < p.G; ++g) {
    float Y[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) Y[c] = (c < nch) ? __ldg(p.bias + co0 + c) : 0.f;
    // Y_k = W * A_k with A_k built on the fly from the K packed frames.
    for (int r = 0; r < p.R; ++r) {
      const int yi = y * p.stride + r - p.pad;
      if (yi < 0 || yi >= p.H) continue;
      for (int s = 0; s < p.S; ++s) {
        const int xi = x * p.stride + s - p.pad;
        if (xi < 0 || xi >= p.W) continue;
        const long long rowoff = (long long)b * p.in_sb + (long long)yi * p.wpr_in;
        uint32_t words[kMaxK];
        int cur = -1;
        for (int ci = 0; ci < p.Cin; ++ci) {
          float a = 0.f;
          if (p.xin) {  // continuous input: A = sum_j beta^{K-1-j} X_{gK+j} (fp32)
            const float *xp = p.xin + (long long)b * p.in_sb + ((long long)yi * p.W + xi) * p.Cin + ci;
            for (int j = 0; j < p.K; ++j) a = fmaf(p.coef[j], __ldg(xp + (long long)(g * p.K + j) * p.in_st), a);
          } else {
            const long long bit = (long long)xi * p.Cin + ci;
            const int wi = (int)(bit >> 5), sh = (int)(bit & 31);
            if (wi != cur) {
              for (int j = 0; j < p.K; ++j)
                words[j] = __ldg(p.in + (long long)(g * p.K + j) * p.in_st + rowoff + wi);
              cur = wi;
            }
            for (int j = 0; j < p.K; ++j)
              if ((words[j] >> sh) & 1u) a += p.coef[j];
          }
          if (a != 0.f) {
            const float *wp = p.w + ((long long)(ci * p.R + r) * p.S + s) * p.Cout + co0;
#pragma unroll
            for (int c = 0; c < CH; ++c)
              if (c < nch) Y[c] = fmaf(__ldg(wp + c), a, Y[c]);
          }
        }
      }
    }
    if (p.y_seq) {  // training forward: the group's drive (V-domain, unscaled)
      float *ys = p.y_seq + (long long)g * p.B * p.Ho * p.Wo * p.Cout + vbase;
#pragma unroll
      for (int c = 0; c < CH; ++c)
        if (c < nch) ys[c] = Y[c];
    }
    // LIF steps sharing Y_k
    for (int j = 0; j < p.nsteps; ++j) {
      uint32_t bits = 0u;
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        float v = fmaf(p.decay, V[c], Y[c]);
        if (p.reset == RESET_DELAYED && ((sprev >> c) & 1u)) v -= p.v_th;
        const bool s = (v >= p.v_th) && (c < nch);
        if (s) {
          if (p.reset == RESET_SUBTRACT) v -= p.v_th;
          else if (p.reset == RESET_HARD) v = p.v_reset;
          bits |= 1u << c;
          ++cnt[c];
        }
        V[c] = v;
      }
      if (p.reset == RESET_DELAYED) sprev = bits;
      if (bits && yo < p.Hq && xo < p.Wq) {  // floor pooling drops an odd last row / column
        const int t_out = (p.mode == MODE_TAC) ? g : g * p.K + j;
        uint32_t *row = p.out + (long long)t_out * p.out_st + (long long)b * p.out_sb +
                        (long long)yo * p.wpr_out;
        atomicOr(row + ow, bits << osh);
        if (osh && (osh + nch > 32)) atomicOr(row + ow + 1, bits >> (32 - osh));
      }
    }
  }
  if (p.v_final) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      if (c < nch) p.v_final[vbase + c] = V[c];
  }
  if (p.counts) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      if (cnt[c]) atomicAdd(p.counts + (long long)b * p.Cout + co0 + c, (uint32_t)cnt[c]);
  }
}

__global__ void pack_kernel(const uint8_t *__restrict__ dense, uint32_t *__restrict__ packed,
                            int T, int B, int C, int H, int W, int wpr) {
  const long long nwords = (long long)T * B * H * wpr;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nwords;
       i += (long long)gridDim.x * blockDim.x) {
    const int wi = (int)(i % wpr);
    const long long tby = i / wpr;                 // ((t*B + b)*H + y)
    const int yy = (int)(tby % H);
    const long long tb = tby / H;
    uint32_t word = 0u;
    for (int k = 0; k < 32; ++k) {
      const long long r = (long long)wi * 32 + k;
      if (r >= (long long)W * C) break;
      const int xx = (int)(r / C), c = (int)(r - (long long)(r / C) * C);
      if (dense[((tb * C + c) * H + yy) * (long long)W + xx]) word |= 1u << k;
    }
    packed[i] = word;
  }
}

// Vectorised pack for the input layers (C = 1 or 2, W a multiple of 32 / C): one thread per
// output word reads 32 / C consecutive pixels of each channel plane as 16-B vectors
// (a warp reads 512 contiguous bytes per plane), compacts the 0/1 bytes to bits with one
// multiply per 4 bytes and, for C = 2, interleaves the two planes' bits (bit 2x + c).
__device__ __forceinline__ uint32_t bytes4_to_bits(uint32_t x) {  // nonzero byte k -> bit k
  const uint32_t b = __vcmpne4(x, 0u) & 0x01010101u;
  return ((b * 0x01020408u) >> 24) & 0xFu;
}
__device__ __forceinline__ uint32_t bytes16_to_bits(uint4 v) {
  return bytes4_to_bits(v.x) | (bytes4_to_bits(v.y) << 4) | (bytes4_to_bits(v.z) << 8) | (bytes4_to_bits(v.w) << 12);
}
__device__ __forceinline__ uint32_t spread16(uint32_t x) {  // bit i -> bit 2i
  x = (x | (x << 8)) & 0x00FF00FFu;
  x = (x | (x << 4)) & 0x0F0F0F0Fu;
  x = (x | (x << 2)) & 0x33333333u;
  return (x | (x << 1)) & 0x55555555u;
}
template <int C>
__global__ void pack_vec_kernel(const uint8_t *__restrict__ dense, uint32_t *__restrict__ packed,
                                long long nrows, int H, int W, int wpr) {
  const long long nwords = nrows * wpr;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nwords;
       i += (long long)gridDim.x * blockDim.x) {
    const int wi = (int)(i % wpr);
    const long long tby = i / wpr;  // (t B + b) H + y
    const long long tb = tby / H;
    const int yy = (int)(tby - tb * H);
    const int x0 = wi * (32 / C);
    uint32_t word;
    if (C == 1) {
      const uint4 *src = reinterpret_cast<const uint4 *>(dense + (tb * H + yy) * (long long)W + x0);
      word = bytes16_to_bits(__ldg(src)) | (bytes16_to_bits(__ldg(src + 1)) << 16);
    } else {
      const uint8_t *row0 = dense + ((tb * 2) * H + yy) * (long long)W + x0;
      const uint32_t p0 = bytes16_to_bits(__ldg(reinterpret_cast<const uint4 *>(row0)));
      const uint32_t p1 = bytes16_to_bits(__ldg(reinterpret_cast<const uint4 *>(row0 + (long long)H * W)));
      word = spread16(p0) | (spread16(p1) << 1);
    }
    packed[i] = word;
  }
}

__global__ void unpack_kernel(const uint32_t *__restrict__ packed, uint8_t *__restrict__ dense,
                              int T, int B, int C, int H, int W, int wpr) {
  const long long n = (long long)T * B * C * H * W;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int xx = (int)(i % W);
    long long q = i / W;
    const int yy = (int)(q % H);
    q /= H;
    const int c = (int)(q % C);
    const long long tb = q / C;
    const long long r = (long long)xx * C + c;
    const uint32_t word = packed[(tb * H + yy) * wpr + (r >> 5)];
    dense[i] = (uint8_t)((word >> (r & 31)) & 1u);
  }
}

inline int grid_for(long long n, int block) {
  long long g = (n + block - 1) / block;
  if (g > 148LL * 64) g = 148LL * 64;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

int launch_zero_outputs(const LayerParams &p, void *stream, int *launches) {
  const long long plane = (long long)p.Hq * p.wpr_out;
  const long long total = (long long)p.T_out * p.B * plane;
  zero_outputs_kernel<<<grid_for(total > p.B * (long long)p.Cout ? total : p.B * (long long)p.Cout, 256),
                        256, 0, (cudaStream_t)stream>>>(
      p.out, p.T_out, p.B, plane, p.out_st, p.out_sb, p.counts, (long long)p.B * p.Cout);
  ++*launches;
  return (int)cudaGetLastError();
}

int launch_add_u32(uint32_t *dst, const uint32_t *src, long long n, void *stream) {
  const int grid = (int)std::min<long long>((n + 255) / 256, 148LL * 8);
  add_u32_kernel<<<grid > 0 ? grid : 1, 256, 0, (cudaStream_t)stream>>>(dst, src, n);
  return (int)cudaGetLastError();
}

// VotingLayer (tac_vote): one thread per (sample, class)
__global__ void vote_kernel(const uint32_t *counts, int B, int C, int voters, float inv, float *scores) {
  const int ncls = C / voters;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= (long long)B * ncls) return;
  const long long b = i / ncls, j = i - b * ncls;
  const uint32_t *c = counts + b * C + j * voters;
  uint32_t s = 0;
  for (int v = 0; v < voters; ++v) s += c[v];
  scores[i] = (float)s * inv;
}
int launch_vote(const uint32_t *counts, int B, int C, int voters, int T_out, float *scores, void *stream) {
  const long long n = (long long)B * (C / voters);
  const float inv = (float)(1.0 / ((double)voters * T_out));
  vote_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(counts, B, C, voters, inv, scores);
  return (int)cudaGetLastError();
}

int launch_simt_conv_lif(const LayerParams &p, void *stream, int *launches) {
  if (p.H == 1 && p.W == 1 && p.R == 1 && p.S == 1 && p.pad == 0 && p.pool == 1) {
    fc_lif_kernel<<<dim3((unsigned)p.B, (unsigned)((p.Cout + 31) / 32)), 32 * FC_WARPS, 0,
                    (cudaStream_t)stream>>>(p);
    ++*launches;
    return (int)cudaGetLastError();
  }
  const long long npix = (long long)p.B * p.Ho * p.Wo;
  dim3 grid((unsigned)((npix + 127) / 128), (unsigned)((p.Cout + CH - 1) / CH));
  simt_conv_lif_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(p);
  ++*launches;
  return (int)cudaGetLastError();
}

int launch_pack(const uint8_t *dense, uint32_t *packed, int T, int B, int C, int H, int W,
                void *stream) {
  const int wpr = (W * C + 31) / 32;
  const bool vec = (C == 1 || C == 2) && W % (32 / C) == 0 && reinterpret_cast<uintptr_t>(dense) % 16 == 0;
  if (vec && C == 1)
    pack_vec_kernel<1><<<grid_for((long long)T * B * H * wpr, 256), 256, 0, (cudaStream_t)stream>>>(
        dense, packed, (long long)T * B * H, H, W, wpr);
  else if (vec)
    pack_vec_kernel<2><<<grid_for((long long)T * B * H * wpr, 256), 256, 0, (cudaStream_t)stream>>>(
        dense, packed, (long long)T * B * H, H, W, wpr);
  else
    pack_kernel<<<grid_for((long long)T * B * H * wpr, 256), 256, 0, (cudaStream_t)stream>>>(
        dense, packed, T, B, C, H, W, wpr);
  return (int)cudaGetLastError();
}

int launch_unpack(const uint32_t *packed, uint8_t *dense, int T, int B, int C, int H, int W,
                  void *stream) {
  const int wpr = (W * C + 31) / 32;
  unpack_kernel<<<grid_for((long long)T * B * C * H * W, 256), 256, 0,
                  (cudaStream_t)stream>>>(packed, dense, T, B, C, H, W, wpr);
  return (int)cudaGetLastError();
}

}  // namespace tacsnn
