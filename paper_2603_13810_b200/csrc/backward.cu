// backward.cu -- training side of libtacsnn: surrogate-gradient BPTT through the
// grouped LIF and the gradients of the one-conv-per-group.
//
// The paper trains every network it reports end to end with backpropagation
// through time and a surrogate spike derivative (App. E, P:587-588:
// fast sigmoid slope 25 for MNIST/FMNIST, arctan alpha 2 with a detached reset
// for DVS-Gesture).  For one layer (subtract reset), with U the post-reset state:
//   forward   V_t = decay U_{t-1} + Y_k ;  s_t = Theta(V_t - v_th) ;  U_t = V_t - v_th s_t
//   backward  dV_t = (dL/ds_t - [!detach] v_th gU) h(V_t - v_th) + gU ;  gU <- decay dV_t
//             dL/dY_k = sum over the group's LIF steps of dV_t ;  dL/dv_init = gU
//   conv      dL/dW = sum_k corr(dL/dY_k, A_k) ;  dL/db = sum dL/dY_k
//             dL/dA_k = conv^T(dL/dY_k, W) ;  dL/dS_{kK+j} = a_j dL/dA_k ;
//             dL/da_j = sum_k <dL/dA_k, S_{kK+j}>     (learnable aggregation)
// Because TAC convolves once per group, the backward also runs the conv
// gradients once per group (G = T/K), not per time step -- the same saving as
// the forward.
//
// Kernels:
//   lif_bwd_kernel  one thread per neuron: replays the forward integrator from the
//                   saved per-group drive y_seq (bit-identical arithmetic of the
//                   engine that produced it), keeps V_t - v_th of every step in
//                   registers/local memory, then runs the reverse sweep; writes
//                   dL/dY_k and dL/dv_init.  HBM-bound (reads y_seq + g_spikes once).
//   dgrad_kernel    one thread per input pixel x 32 input channels: dL/dA_k by the
//                   transposed conv, then dL/dS for the K frames of the group and
//                   the dL/da_j partial sums.
//   wgrad_kernel    a block per (32 output ch, 8 input ch) x pixel slice: the
//                   pixel-dimension reduction of dL/dY_k x A_k for all 9 taps staged
//                   through shared memory (A_k rebuilt from the packed frames), then
//                   one atomic add per weight per block.
// plus the OR-pool forward / backward on packed spikes (MaxPool2d semantics: the
// gradient of a 2x2 window goes to its first maximal element in row-major order).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "layer.cuh"

namespace tacsnn {

namespace {

constexpr int kMaxBwdSteps = 64;  // LIF steps per call kept per thread (T <= 64)

__device__ __forceinline__ float surrogate(int kind, float a, float u) {
  if (kind == 0) {  // fast sigmoid: d/du [u / (1 + a|u|)]
    const float d = fmaf(a, fabsf(u), 1.f);
    return 1.f / (d * d);
  }
  const float z = 1.5707963267948966f * a * u;  // arctan: d/du [atan(pi/2 a u) / pi]
  return 0.5f * a / fmaf(z, z, 1.f);
}

__device__ __forceinline__ float sat_nospike(float u) {  // same instruction as the tcgen05 epilogue
  float g;
  asm("mul.rn.ftz.sat.f32 %0, %1, 0fFF000000;" : "=f"(g) : "f"(u));
  return g;
}

__global__ void __launch_bounds__(128) lif_bwd_kernel(const BwdParams p) {
  const long long N = (long long)p.B * p.Ho * p.Wo * p.Cout;
  const long long n = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (n >= N) return;
  const float ysc = p.yscale ? __ldg(p.yscale) : 1.f, iysc = p.yscale ? __ldg(p.yscale + 1) : 1.f;
  const float vth = p.v_th, vths = p.v_th * ysc, d = p.decay;
  const int nsteps = p.nsteps, G = p.G, S = G * nsteps;
  float um[kMaxBwdSteps];  // V_t - v_th (unscaled) of every step
  // forward replay
  float st = p.v_init ? __ldg(p.v_init + n) : 0.f;
  st = st * ysc;
  for (int k = 0; k < G; ++k) {
    const float y = __ldg(p.y_seq + (long long)k * N + n);
    for (int j = 0; j < nsteps; ++j) {
      float pre;
      if (p.udomain) {  // epilogue_sr: U <- d V + Y''; spike = sign(U); V <- U + v_th [U < 0]
        pre = fmaf(d, st, y);
        st = fmaf(sat_nospike(pre), vths, pre);
        um[k * nsteps + j] = pre * iysc;
      } else {  // epilogue_generic / SIMT: V <- d V + Y; spike = V >= v_th; V <- V - v_th
        const float v = fmaf(d, st, y);
        const float v2 = v - vths;
        st = (__float_as_uint(v2) >> 31) ? v : v2;
        um[k * nsteps + j] = v2 * iysc;
      }
    }
  }
  // reverse sweep (unscaled gradients)
  float gU = p.g_vfinal ? __ldg(p.g_vfinal + n) : 0.f;
  const float a = p.sg_alpha;
  for (int k = G - 1; k >= 0; --k) {
    float gy = 0.f;
    for (int j = nsteps - 1; j >= 0; --j) {
      const int t = k * nsteps + j;
      const float h = surrogate(p.surrogate, a, um[t]);
      const float gs = __ldg(p.g_spikes + (long long)t * N + n);
      const float dV = fmaf(p.detach ? gs : fmaf(-vth, gU, gs), h, gU);
      gy += dV;
      gU = d * dV;
    }
    p.g_y[(long long)k * N + n] = gy;
  }
  if (p.g_vinit) p.g_vinit[n] = gU;
}

// A_k[b][yi][xi][ci] of one input pixel / channel (packed spikes or real frames)
__device__ __forceinline__ float agg_at(const BwdParams &p, int k, int b, int yi, int xi, int ci) {
  float a = 0.f;
  if (p.xin) {
    const float *xp = p.xin + (long long)b * p.in_sb + ((long long)yi * p.W + xi) * p.Cin + ci;
    for (int j = 0; j < p.K; ++j) a = fmaf(p.coef[j], __ldg(xp + (long long)(k * p.K + j) * p.in_st), a);
  } else {
    const long long bit = (long long)xi * p.Cin + ci;
    const uint32_t *wp = p.in + (long long)b * p.in_sb + (long long)yi * p.wpr_in + (bit >> 5);
    const int sh = (int)(bit & 31);
    for (int j = 0; j < p.K; ++j)
      if ((__ldg(wp + (long long)(k * p.K + j) * p.in_st) >> sh) & 1u) a += p.coef[j];
  }
  return a;
}

// input frame value S_t[b][yi][xi][ci] (for dL/da_j)
__device__ __forceinline__ float frame_at(const BwdParams &p, int t, int b, int yi, int xi, int ci) {
  if (p.xin)
    return __ldg(p.xin + (long long)t * p.in_st + (long long)b * p.in_sb + ((long long)yi * p.W + xi) * p.Cin + ci);
  const long long bit = (long long)xi * p.Cin + ci;
  const uint32_t w = __ldg(p.in + (long long)t * p.in_st + (long long)b * p.in_sb + (long long)yi * p.wpr_in + (bit >> 5));
  return (float)((w >> (bit & 31)) & 1u);
}

constexpr int kDgradCh = 32;

// dL/dA_k by the transposed conv: thread = (k, b, yi, xi) x 32 input channels
__global__ void __launch_bounds__(128) dgrad_kernel(const BwdParams p) {
  const long long npix = (long long)p.G * p.B * p.H * p.W;
  const long long pix = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const bool live = pix < npix;
  const int ci0 = blockIdx.y * kDgradCh;
  const int nci = min(kDgradCh, p.Cin - ci0);
  __shared__ float s_alpha[kMaxK];
  if (threadIdx.x < kMaxK) s_alpha[threadIdx.x] = 0.f;
  __syncthreads();
  int xi = 0, yi = 0, b = 0, k = 0;
  float gA[kDgradCh];
#pragma unroll
  for (int c = 0; c < kDgradCh; ++c) gA[c] = 0.f;
  if (live) {
    xi = (int)(pix % p.W);
    long long q = pix / p.W;
    yi = (int)(q % p.H);
    q /= p.H;
    b = (int)(q % p.B);
    k = (int)(q / p.B);
    const long long N = (long long)p.B * p.Ho * p.Wo * p.Cout;
    for (int r = 0; r < p.R; ++r) {
      const int ty = yi + p.pad - r;
      if (ty < 0 || ty % p.stride) continue;
      const int y = ty / p.stride;
      if (y >= p.Ho) continue;
      for (int s = 0; s < p.S; ++s) {
        const int tx = xi + p.pad - s;
        if (tx < 0 || tx % p.stride) continue;
        const int x = tx / p.stride;
        if (x >= p.Wo) continue;
        const float *gy = p.g_y + (long long)k * N + (((long long)b * p.Ho + y) * p.Wo + x) * p.Cout;
        const float *wr = p.w + ((long long)(ci0 * p.R + r) * p.S + s) * p.Cout;  // W[ci0][r][s][:]
        const long long wci = (long long)p.R * p.S * p.Cout;                       // ci stride
        for (int co = 0; co < p.Cout; ++co) {
          const float g = __ldg(gy + co);
          if (g == 0.f) continue;
#pragma unroll
          for (int c = 0; c < kDgradCh; ++c)
            if (c < nci) gA[c] = fmaf(g, __ldg(wr + c * wci + co), gA[c]);
        }
      }
    }
  }
  // dL/dS_{kK+j} = a_j dL/dA_k  (channels-last [T][B][H][W][Cin]); dL/da_j partial sums
  const long long plane = (long long)p.H * p.W * p.Cin;
  for (int j = 0; j < p.K; ++j) {
    const int t = k * p.K + j;
    const float aj = p.coef[j];
    float acc = 0.f;
    if (live) {
      float *gi = p.g_in ? p.g_in + ((long long)t * p.B + b) * plane + ((long long)yi * p.W + xi) * p.Cin + ci0
                         : nullptr;
#pragma unroll
      for (int c = 0; c < kDgradCh; ++c)
        if (c < nci) {
          if (gi) gi[c] = aj * gA[c];
          if (p.g_alpha) acc = fmaf(gA[c], frame_at(p, t, b, yi, xi, ci0 + c), acc);
        }
    }
    if (p.g_alpha) {  // uniform branch: every lane of the warp shuffles
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
      if ((threadIdx.x & 31) == 0 && acc != 0.f) atomicAdd(&s_alpha[j], acc);
    }
  }
  if (p.g_alpha) {
    __syncthreads();
    if (threadIdx.x < p.K && s_alpha[threadIdx.x] != 0.f) atomicAdd(p.g_alpha + threadIdx.x, s_alpha[threadIdx.x]);
  }
}

// dL/dW, dL/db: block = (32 output channels) x (8 input channels) x all R x S taps, over a
// contiguous slice of the G*B*Ho output rows; a row is processed in segments of 32
// output pixels: dL/dY of the segment [32 px][32 co] and the A_k patch
// [R][32 + S - 1][8 ci] are staged in shared memory, thread (co, ci) accumulates its
// R*S taps.
constexpr int kWgCo = 32, kWgCi = 8, kWgPx = 32, kWgMaxTaps = 9;
__global__ void __launch_bounds__(256) wgrad_kernel(const BwdParams p, int rows_per_block) {
  __shared__ float s_g[kWgPx][kWgCo + 1];
  __shared__ float s_a[3][kWgPx + 2][kWgCi];  // R, S <= 3 with stride 1 (host checks); else direct
  const int co0 = blockIdx.y * kWgCo, ci0 = blockIdx.z * kWgCi;
  const int tco = threadIdx.x >> 3, tci = threadIdx.x & 7;
  const int co = co0 + tco, ci = ci0 + tci;
  const int taps = p.R * p.S;
  float acc[kWgMaxTaps];
#pragma unroll
  for (int t = 0; t < kWgMaxTaps; ++t) acc[t] = 0.f;
  float accb = 0.f;
  const long long N = (long long)p.B * p.Ho * p.Wo * p.Cout;
  const long long nrows = (long long)p.G * p.B * p.Ho;
  const long long r0 = (long long)blockIdx.x * rows_per_block;
  const long long r1 = min(nrows, r0 + rows_per_block);
  for (long long row = r0; row < r1; ++row) {
    const int y = (int)(row % p.Ho);
    const int b = (int)((row / p.Ho) % p.B);
    const int k = (int)(row / ((long long)p.Ho * p.B));
    for (int x0 = 0; x0 < p.Wo; x0 += kWgPx) {
      __syncthreads();
      // stage dL/dY_k [32 px][32 co]
      for (int i = threadIdx.x; i < kWgPx * kWgCo; i += blockDim.x) {
        const int px = i / kWgCo, c = i % kWgCo;
        const int x = x0 + px;
        float g = 0.f;
        if (x < p.Wo && co0 + c < p.Cout)
          g = __ldg(p.g_y + (long long)k * N + (((long long)b * p.Ho + y) * p.Wo + x) * p.Cout + co0 + c);
        s_g[px][c] = g;
      }
      // stage A_k patch: rows y*stride + r - pad, columns x0 + c - pad (stride 1)
      for (int i = threadIdx.x; i < p.R * (kWgPx + p.S - 1) * kWgCi; i += blockDim.x) {
        const int c8 = i % kWgCi, rest = i / kWgCi;
        const int cx = rest % (kWgPx + p.S - 1), r = rest / (kWgPx + p.S - 1);
        const int yi = y + r - p.pad, xi = x0 + cx - p.pad;
        float a = 0.f;
        if (yi >= 0 && yi < p.H && xi >= 0 && xi < p.W && ci0 + c8 < p.Cin) a = agg_at(p, k, b, yi, xi, ci0 + c8);
        s_a[r][cx][c8] = a;
      }
      __syncthreads();
      const int npx = min(kWgPx, p.Wo - x0);
      for (int px = 0; px < npx; ++px) {
        const float g = s_g[px][tco];
        if (tci == 0) accb += g;
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int s = 0; s < 3; ++s)
            if (r < p.R && s < p.S) acc[r * 3 + s] = fmaf(g, s_a[r][px + s][tci], acc[r * 3 + s]);
      }
    }
  }
  if (co < p.Cout) {
    if (ci < p.Cin)
      for (int r = 0; r < p.R; ++r)
        for (int s = 0; s < p.S; ++s) {
          const float v = acc[r * 3 + s];
          if (v != 0.f) atomicAdd(p.g_w + (((long long)co * p.Cin + ci) * p.R + r) * p.S + s, v);
        }
    if (ci0 == 0 && tci == 0 && accb != 0.f) atomicAdd(p.g_b + co, accb);
  }
}

// generic (any R, S, stride, pad) weight gradient: one thread per weight, full reduction
__global__ void wgrad_direct_kernel(const BwdParams p) {
  const long long nw = (long long)p.Cout * p.Cin * p.R * p.S;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= nw + p.Cout) return;
  const long long N = (long long)p.B * p.Ho * p.Wo * p.Cout;
  if (i >= nw) {  // bias
    const int co = (int)(i - nw);
    float acc = 0.f;
    for (long long n = co; n < (long long)p.G * N; n += p.Cout) acc += __ldg(p.g_y + n);
    p.g_b[co] += acc;
    return;
  }
  const int s = (int)(i % p.S), r = (int)((i / p.S) % p.R);
  const int ci = (int)((i / ((long long)p.S * p.R)) % p.Cin), co = (int)(i / ((long long)p.S * p.R * p.Cin));
  float acc = 0.f;
  for (int k = 0; k < p.G; ++k)
    for (int b = 0; b < p.B; ++b)
      for (int y = 0; y < p.Ho; ++y) {
        const int yi = y * p.stride + r - p.pad;
        if (yi < 0 || yi >= p.H) continue;
        for (int x = 0; x < p.Wo; ++x) {
          const int xi = x * p.stride + s - p.pad;
          if (xi < 0 || xi >= p.W) continue;
          const float g = __ldg(p.g_y + (long long)k * N + (((long long)b * p.Ho + y) * p.Wo + x) * p.Cout + co);
          if (g != 0.f) acc = fmaf(g, agg_at(p, k, b, yi, xi, ci), acc);
        }
      }
  p.g_w[i] += acc;
}

// ---- fully connected layers (H = W = R = S = 1): the backward conv is two plain GEMMs
// over the flattened (group, sample) rows; a shared-memory tiled fp32 GEMM
//   C[m][n] (=) sum_k A(m, k) B(k, n),  A(m, k) = A[m sam + k sak],  B(k, n) = B[k sbk + n sbn]
// (64 x 64 tile, 16-deep K slices, 4 x 4 outputs per thread).
constexpr int kGmT = 64, kGmK = 16;
__global__ void __launch_bounds__(256) gemm_f32_kernel(int M, int N, int K, const float *A, long long sam,
                                                       long long sak, const float *Bm, long long sbk, long long sbn,
                                                       float *C, long long ldc) {
  __shared__ float sA[kGmK][kGmT + 1], sB[kGmK][kGmT + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * kGmT, n0 = blockIdx.x * kGmT;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += kGmK) {
    for (int i = threadIdx.x; i < kGmK * kGmT; i += 256) {
      // consecutive threads walk the unit-stride index of each operand (coalesced loads)
      const int kk = sam == 1 ? i / kGmT : i % kGmK, mm = sam == 1 ? i % kGmT : i / kGmK;
      const int m = m0 + mm, k = k0 + kk;
      sA[kk][mm] = (m < M && k < K) ? __ldg(A + m * sam + k * sak) : 0.f;
      const int nn = sbn == 1 ? i % kGmT : i / kGmK, kb = sbn == 1 ? i / kGmT : i % kGmK;
      const int n = n0 + nn, k2 = k0 + kb;
      sB[kb][nn] = (n < N && k2 < K) ? __ldg(Bm + k2 * sbk + n * sbn) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kGmK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sA[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = sB[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
      if (m < M && n < N) C[m * ldc + n] = acc[i][j];
    }
}

// A_k[kb][c] (fp32) of a fully connected layer's flattened input
__global__ void fc_agg_kernel(const BwdParams p, float *out) {
  const long long n = (long long)p.G * p.B * p.Cin;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % p.Cin);
    const long long kb = i / p.Cin;
    out[i] = agg_at(p, (int)(kb / p.B), (int)(kb % p.B), 0, 0, c);
  }
}

// dL/dS_{kK+j}[b][c] = a_j dA[kb][c]; dL/da_j partial sums (one block-wide reduction per j)
__global__ void fc_gin_kernel(const BwdParams p, const float *dA) {
  __shared__ float red[kMaxK][8];
  const long long n = (long long)p.G * p.B * p.Cin;
  float acc[kMaxK];
#pragma unroll
  for (int j = 0; j < kMaxK; ++j) acc[j] = 0.f;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % p.Cin);
    const long long kb = i / p.Cin;
    const int k = (int)(kb / p.B), b = (int)(kb % p.B);
    const float g = dA[i];
    for (int j = 0; j < p.K; ++j) {
      const int t = k * p.K + j;
      if (p.g_in) p.g_in[((long long)t * p.B + b) * p.Cin + c] = p.coef[j] * g;
      if (p.g_alpha) acc[j] = fmaf(g, frame_at(p, t, b, 0, 0, c), acc[j]);
    }
  }
  if (p.g_alpha) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    for (int j = 0; j < p.K; ++j) {
      float v = acc[j];
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
      if (l == 0) red[j][w] = v;
    }
    __syncthreads();
    if (threadIdx.x < p.K) {
      float v = 0.f;
      for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) v += red[threadIdx.x][w2];
      if (v != 0.f) atomicAdd(p.g_alpha + threadIdx.x, v);
    }
  }
}

__global__ void bias_grad_fc_kernel(const float *g_y, int rows, int Cout, float *g_b) {
  for (int co = threadIdx.x; co < Cout; co += blockDim.x) {
    float acc = 0.f;
    for (int r = blockIdx.x; r < rows; r += gridDim.x) acc += __ldg(g_y + (long long)r * Cout + co);
    if (acc != 0.f) atomicAdd(g_b + co, acc);
  }
}

__global__ void zero_f32_kernel(float *a, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    a[i] = 0.f;
}

// 2x2 OR-pool of packed spikes (floor mode): thread per output word
// C % 32 == 0: a pooled word is the OR of the same channel word of the window's 4 pixels;
// grid (ceil(Wq nw / 128), TB Hq): no 64-bit index arithmetic
__global__ void or_pool2_w32_kernel(const uint32_t *in, uint32_t *out, int C, int H, int W) {
  const int Hq = H / 2, Wq = W / 2, nw = C / 32;
  const int idx = blockIdx.y * blockDim.x + threadIdx.x;
  if (idx >= Wq * nw) return;
  const int xo = idx / nw, wd = idx - xo * nw;
  const long long row = blockIdx.x;  // tb Hq + yo
  const long long tb = row / Hq;
  const int yo = (int)(row - tb * Hq);
  const uint32_t *r0 = in + ((tb * H + 2 * yo) * W + 2 * xo) * nw + wd, *r1 = r0 + (long long)W * nw;
  out[row * Wq * nw + idx] = r0[0] | r0[nw] | r1[0] | r1[nw];
}

__global__ void or_pool2_kernel(const uint32_t *in, uint32_t *out, long long TB, int C, int H, int W) {
  const int Hq = H / 2, Wq = W / 2;
  const int wpr_in = (W * C + 31) / 32, wpr_out = (Wq * C + 31) / 32;
  const long long n = TB * Hq * wpr_out;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int wo = (int)(i % wpr_out);
    const long long q = i / wpr_out;
    const int yo = (int)(q % Hq);
    const long long tb = q / Hq;
    const uint32_t *r0 = in + (tb * H + 2 * yo) * wpr_in, *r1 = r0 + wpr_in;
    uint32_t word = 0u;
    for (int bit = 0; bit < 32; ++bit) {
      const long long ro = (long long)wo * 32 + bit;
      if (ro >= (long long)Wq * C) break;
      const int xo = (int)(ro / C), c = (int)(ro % C);
      uint32_t v = 0u;
      for (int dx = 0; dx < 2; ++dx) {
        const long long ri = (long long)(2 * xo + dx) * C + c;
        v |= ((r0[ri >> 5] | r1[ri >> 5]) >> (ri & 31)) & 1u;
      }
      word |= v << bit;
    }
    out[i] = word;
  }
}

// MaxPool2d backward on binary maps: g_pre[t][b][y][x][c] = g_pooled of its window if
// (y, x) is the window's first maximal element in row-major order, else 0
// C % 32 == 0: one thread per (pooled window, 4 channels) of one unpooled row y: a warp
// stores whole 512-B pixel rows (C = 128), reads the pooled gradient as one 512-B row and the
// window's spike words by broadcast; per channel the gradient goes to the first spiking
// element in row-major order (top-left when none).  Grid (TB H, ceil(Wq C / 4 / 128)).
__global__ void or_pool2_bwd32_kernel(const uint32_t *pre, const float *g_pooled, float *g_pre, long long TB,
                                      int C, int H, int W) {
  const int Hq = H / 2, Wq = W / 2, nw = C / 32, nq = C / 4;
  const int i = blockIdx.y * blockDim.x + threadIdx.x;
  if (i >= Wq * nq) return;
  const int xo = i / nq, q = i - xo * nq;
  const long long rowi = blockIdx.x;
  const long long tb = rowi / H;
  const int y = (int)(rowi - tb * H);
  const int yo = y >> 1, dy = y & 1;
  float4 *d0 = reinterpret_cast<float4 *>(g_pre + ((tb * H + y) * W + 2 * xo) * C) + q;
  float4 *d1 = d0 + nq;
  const bool last_col = (W & 1) && 2 * xo + 2 == W - 1;  // floor mode: the dropped column
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  if (last_col) d1[nq] = z;
  if (yo >= Hq) {  // floor mode: the dropped row
    *d0 = z;
    *d1 = z;
    return;
  }
  const int wd = q >> 3, sh = (q & 7) * 4;
  const uint32_t *r0 = pre + (tb * H + 2 * yo) * (long long)W * nw + wd, *r1 = r0 + (long long)W * nw;
  const uint32_t w00 = (r0[(2 * xo) * nw] >> sh) & 0xFu, w01 = (r0[(2 * xo + 1) * nw] >> sh) & 0xFu;
  const uint32_t w10 = (r1[(2 * xo) * nw] >> sh) & 0xFu, w11 = (r1[(2 * xo + 1) * nw] >> sh) & 0xFu;
  const uint32_t m00 = (w00 | ~(w00 | w01 | w10 | w11)) & 0xFu, m01 = w01 & ~w00;
  const uint32_t m10 = w10 & ~(w00 | w01), m11 = w11 & ~(w00 | w01 | w10);
  const uint32_t ma = dy ? m10 : m00, mb = dy ? m11 : m01;
  const float4 g = __ldg(reinterpret_cast<const float4 *>(g_pooled + ((tb * Hq + yo) * Wq + xo) * C) + q);
  *d0 = make_float4((ma & 1u) ? g.x : 0.f, (ma & 2u) ? g.y : 0.f, (ma & 4u) ? g.z : 0.f, (ma & 8u) ? g.w : 0.f);
  *d1 = make_float4((mb & 1u) ? g.x : 0.f, (mb & 2u) ? g.y : 0.f, (mb & 4u) ? g.z : 0.f, (mb & 8u) ? g.w : 0.f);
}

__global__ void or_pool2_bwd_kernel(const uint32_t *pre, const float *g_pooled, float *g_pre, long long TB,
                                    int C, int H, int W) {
  const int Hq = H / 2, Wq = W / 2;
  const int wpr = (W * C + 31) / 32;
  const long long n = TB * H * W * C;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    long long q = i / C;
    const int x = (int)(q % W);
    q /= W;
    const int y = (int)(q % H);
    const long long tb = q / H;
    const int yo = y >> 1, xo = x >> 1;
    float g = 0.f;
    if (yo < Hq && xo < Wq) {
      int first = 0;  // window index (dy * 2 + dx) of the first spike, 0 if none
      for (int e = 3; e >= 0; --e) {
        const int yy = 2 * yo + (e >> 1), xx = 2 * xo + (e & 1);
        const long long bit = (long long)xx * C + c;
        if ((pre[(tb * H + yy) * wpr + (bit >> 5)] >> (bit & 31)) & 1u) first = e;
      }
      if ((y - 2 * yo) * 2 + (x - 2 * xo) == first) g = g_pooled[((tb * Hq + yo) * Wq + xo) * C + c];
    }
    g_pre[i] = g;
  }
}

inline int grid1(long long n, int block) {
  long long g = (n + block - 1) / block;
  return (int)std::max(1LL, std::min(g, 148LL * 64));
}

}  // namespace

int launch_backward(const BwdParams &p, void *stream, int *launches) {
  cudaStream_t st = (cudaStream_t)stream;
  const long long N = (long long)p.B * p.Ho * p.Wo * p.Cout;
  lif_bwd_kernel<<<(unsigned)((N + 127) / 128), 128, 0, st>>>(p);
  ++*launches;
  const long long nw = (long long)p.Cout * p.Cin * p.R * p.S;
  zero_f32_kernel<<<grid1(nw, 256), 256, 0, st>>>(p.g_w, nw);
  zero_f32_kernel<<<1, 256, 0, st>>>(p.g_b, p.Cout);
  *launches += 2;
  if (p.g_alpha) {
    zero_f32_kernel<<<1, 32, 0, st>>>(p.g_alpha, p.K);
    ++*launches;
  }
  const bool fc = p.H == 1 && p.W == 1 && p.R == 1 && p.S == 1 && p.pad == 0 && p.stride == 1 && p.fc_ws;
  if (fc) {  // fully connected: dW = gY^T A and dA = gY W as tiled GEMMs over the G B rows
    const int KB = p.G * p.B;
    float *Aagg = static_cast<float *>(p.fc_ws), *dA = Aagg + (long long)KB * p.Cin;
    fc_agg_kernel<<<grid1((long long)KB * p.Cin, 256), 256, 0, st>>>(p, Aagg);
    dim3 gw((p.Cin + kGmT - 1) / kGmT, (p.Cout + kGmT - 1) / kGmT);
    gemm_f32_kernel<<<gw, 256, 0, st>>>(p.Cout, p.Cin, KB, p.g_y, 1, p.Cout, Aagg, p.Cin, 1, p.g_w, p.Cin);
    bias_grad_fc_kernel<<<std::min(KB, 148 * 4), 256, 0, st>>>(p.g_y, KB, p.Cout, p.g_b);
    *launches += 3;
    if (p.g_in || p.g_alpha) {
      dim3 gd((p.Cin + kGmT - 1) / kGmT, (KB + kGmT - 1) / kGmT);
      // W(co, ci) = p.w[ci Cout + co] (SIMT layout [Cin][1][1][Cout])
      gemm_f32_kernel<<<gd, 256, 0, st>>>(KB, p.Cin, p.Cout, p.g_y, p.Cout, 1, p.w, 1, p.Cout, dA, p.Cin);
      fc_gin_kernel<<<std::max(1, std::min(grid1((long long)KB * p.Cin, 256), 148 * 4)), 256, 0, st>>>(p, dA);
      *launches += 2;
    }
    return (int)cudaGetLastError();
  }
  static const bool no_wgtc = [] { const char *e = std::getenv("TACSNN_NO_WGRAD_TC"); return e && *e == '1'; }();
  if (p.tc && p.wg_abuf && !no_wgtc && wgrad_tc_ok(p)) {
    const int e = launch_wgrad_tc(p, stream, launches);
    if (e) return e;
    --*launches;  // counted below with the SIMT variants
  } else if (p.stride == 1 && p.R <= 3 && p.S <= 3) {
    const long long nrows = (long long)p.G * p.B * p.Ho;
    const int cob = (p.Cout + kWgCo - 1) / kWgCo, cib = (p.Cin + kWgCi - 1) / kWgCi;
    const long long want = std::max(1LL, 148LL * 4 / (cob * cib));
    const int rpb = (int)std::max(1LL, (nrows + want - 1) / want);
    dim3 grid((unsigned)((nrows + rpb - 1) / rpb), (unsigned)cob, (unsigned)cib);
    wgrad_kernel<<<grid, 256, 0, st>>>(p, rpb);
  } else {
    wgrad_direct_kernel<<<grid1(nw + p.Cout, 128), 128, 0, st>>>(p);
  }
  ++*launches;
  static const bool no_dgtc = [] { const char *e = std::getenv("TACSNN_NO_DGRAD_TC"); return e && *e == '1'; }();
  if ((p.g_in || p.g_alpha) && p.dg_img && !no_dgtc && dgrad_tc_ok(p)) {
    const int e = launch_dgrad_tc(p, p.dg_img, stream, launches);
    if (e) return e;
  } else if (p.g_in || p.g_alpha) {
    const long long npix = (long long)p.G * p.B * p.H * p.W;
    dim3 grid((unsigned)((npix + 127) / 128), (unsigned)((p.Cin + kDgradCh - 1) / kDgradCh));
    dgrad_kernel<<<grid, 128, 0, st>>>(p);
    ++*launches;
  }
  return (int)cudaGetLastError();
}

int launch_or_pool2(const uint32_t *in, uint32_t *out, int T, int B, int C, int H, int W, void *stream) {
  const long long TB = (long long)T * B;
  const long long n = TB * (H / 2) * (((W / 2) * C + 31) / 32);
  if (C % 32 == 0 && W >= 2 && H >= 2 && TB * (H / 2) < (1LL << 31))
    or_pool2_w32_kernel<<<dim3((unsigned)(TB * (H / 2)), (unsigned)(((W / 2) * (C / 32) + 127) / 128)), 128, 0,
                          (cudaStream_t)stream>>>(in, out, C, H, W);
  else
    or_pool2_kernel<<<grid1(n, 256), 256, 0, (cudaStream_t)stream>>>(in, out, TB, C, H, W);
  return (int)cudaGetLastError();
}

int launch_or_pool2_backward(const uint32_t *pre, const float *g_pooled, float *g_pre, int T, int B, int C,
                             int H, int W, void *stream) {
  const long long TB = (long long)T * B;
  if (C % 32 == 0 && (reinterpret_cast<uintptr_t>(g_pre) | reinterpret_cast<uintptr_t>(g_pooled)) % 16 == 0 &&
      TB * H < (1LL << 31))
    or_pool2_bwd32_kernel<<<dim3((unsigned)(TB * H), (unsigned)(((W / 2) * (C / 4) + 127) / 128)), 128, 0,
                            (cudaStream_t)stream>>>(pre, g_pooled, g_pre, TB, C, H, W);
  else
    or_pool2_bwd_kernel<<<grid1(TB * H * W * C, 256), 256, 0, (cudaStream_t)stream>>>(pre, g_pooled, g_pre, TB,
                                                                                      C, H, W);
  return (int)cudaGetLastError();
}

}  // namespace tacsnn
