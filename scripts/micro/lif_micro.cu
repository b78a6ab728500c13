// Micro-benchmark of LIF step formulations (subtract reset, packed fp32x2):
// 16 warps/SM (4 per SMSP, like the epilogue), each thread 32 neurons x NS steps
// per "group" with a fresh drive Y per group.  Reports cycles per neuron-step per SMSP.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t lop3_sel(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d; asm("lop3.b32 %0, %1, %2, %3, 0xD8;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d;
}
template <uint32_t BIT> __device__ __forceinline__ uint32_t mad_bit(uint32_t m, uint32_t inv) {
  uint32_t d; asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(m), "n"(0u - BIT), "r"(inv)); return d;
}
__device__ __forceinline__ float sat_spike(float u) {  // 1 if u >= 0 (ftz), else 0
  float f; asm("fma.rn.ftz.sat.f32 %0, %1, 0f7F000000, 0f3F800000;" : "=f"(f) : "f"(u)); return f;
}
template <uint32_t BIT> __device__ __forceinline__ uint32_t or_bit(uint32_t acc, float f) {
  uint32_t d; asm("lop3.b32 %0, %1, %2, %3, 0xF8;" : "=r"(d) : "r"(acc), "r"(__float_as_uint(f)), "n"(BIT)); return d;
}

// variant 0: current kernel formulation
template <int C0> __device__ __forceinline__ void v0(float2 &v, float2 y, float2 dec2, float2 nth2, uint32_t &inv) {
  v = __ffma2_rn(dec2, v, y);
  const float2 v2 = __fadd2_rn(v, nth2);
  const uint32_t a0 = __float_as_uint(v2.x), a1 = __float_as_uint(v2.y);
  const uint32_t m0 = (uint32_t)((int)a0 >> 31);
  uint32_t m1; asm("mul.hi.s32 %0, %1, 1;" : "=r"(m1) : "r"(a1));
  v.x = __uint_as_float(lop3_sel(a0, __float_as_uint(v.x), m0));
  v.y = __uint_as_float(lop3_sel(a1, __float_as_uint(v.y), m1));
  inv = mad_bit<1u << C0>(m0, inv);
  inv = mad_bit<1u << (C0 + 1)>(m1, inv);
}
// variant 1: U = V - th state; f = sat(U 2^127 + 1); U -= th f; bits via LOP3 (bit 23+k of f)
template <int C0> __device__ __forceinline__ void v1(float2 &u, float2 y, float2 dec2, float2 nth2, uint32_t &acc) {
  u = __ffma2_rn(dec2, u, y);
  float2 f = make_float2(sat_spike(u.x), sat_spike(u.y));
  u = __ffma2_rn(nth2, f, u);
  acc = or_bit<1u << (23 + (C0 % 7))>(acc, f.x);
  acc = or_bit<1u << (23 + ((C0 + 1) % 7))>(acc, f.y);
}
// variant 2: U state; mask from sign (SHF) ; t = th & ~m (LOP3) ; U -= t (FADD2) ; bits IMAD/LOP3
template <int C0> __device__ __forceinline__ void v2(float2 &u, float2 y, float2 dec2, float2 nth2, uint32_t &inv) {
  u = __ffma2_rn(dec2, u, y);
  const uint32_t m0 = (uint32_t)((int)__float_as_uint(u.x) >> 31);
  const uint32_t m1 = (uint32_t)((int)__float_as_uint(u.y) >> 31);
  float2 t;
  t.x = __uint_as_float(__float_as_uint(nth2.x) & ~m0);
  t.y = __uint_as_float(__float_as_uint(nth2.y) & ~m1);
  u = __fadd2_rn(u, t);
  inv = mad_bit<1u << C0>(m0, inv);
  inv |= m1 & (1u << (C0 + 1));
}

// variant 3: scalar, runtime beta / th (uniform operands), sat spike, LOP3 bits
template <int C0> __device__ __forceinline__ void v3(float2 &u, float2 y, float2 dec2, float2 nth2, uint32_t &acc) {
  u.x = fmaf(dec2.x, u.x, y.x);
  u.y = fmaf(dec2.x, u.y, y.y);
  const float f0 = sat_spike(u.x), f1 = sat_spike(u.y);
  u.x = fmaf(nth2.x, f0, u.x);
  u.y = fmaf(nth2.x, f1, u.y);
  acc = or_bit<1u << (23 + (C0 % 7))>(acc, f0);
  acc = or_bit<1u << (23 + ((C0 + 1) % 7))>(acc, f1);
}
// variant 4: scalar, compile-time beta / th immediates
template <int C0> __device__ __forceinline__ void v4(float2 &u, float2 y, float2 dec2, float2 nth2, uint32_t &acc) {
  u.x = fmaf(0.9f, u.x, y.x);
  u.y = fmaf(0.9f, u.y, y.y);
  const float f0 = sat_spike(u.x), f1 = sat_spike(u.y);
  u.x = fmaf(-1.0f, f0, u.x);
  u.y = fmaf(-1.0f, f1, u.y);
  acc = or_bit<1u << (23 + (C0 % 7))>(acc, f0);
  acc = or_bit<1u << (23 + ((C0 + 1) % 7))>(acc, f1);
}
// variant 5: mixed -- FFMA2 update, scalar sat, FFMA2 reset, bits half LOP3 half IMAD.HI
template <int C0> __device__ __forceinline__ void v5(float2 &u, float2 y, float2 dec2, float2 nth2, uint32_t &acc) {
  u = __ffma2_rn(dec2, u, y);
  float2 f = make_float2(sat_spike(u.x), sat_spike(u.y));
  u.x = fmaf(nth2.x, f.x, u.x);
  u.y = fmaf(nth2.x, f.y, u.y);
  acc = or_bit<1u << (23 + (C0 % 7))>(acc, f.x);
  acc = or_bit<1u << (23 + ((C0 + 1) % 7))>(acc, f.y);
}

// variant 6: FFMA2 update, x via SAT (fma pipe), y via sign mask + LOP3 (alu pipe), FFMA2 reset
template <int C0> __device__ __forceinline__ void v6(float2 &u, float2 y, float2 dec2, float2 nth2, uint32_t &acc) {
  u = __ffma2_rn(dec2, u, y);
  float2 f;
  f.x = sat_spike(u.x);
  const uint32_t m1 = (uint32_t)((int)__float_as_uint(u.y) >> 31);
  f.y = __uint_as_float(0x3F800000u & ~m1);
  u = __ffma2_rn(nth2, f, u);
  acc = or_bit<1u << (23 + (C0 % 7))>(acc, f.x);
  acc = or_bit<1u << (23 + ((C0 + 1) % 7))>(acc, f.y);
}


__device__ __forceinline__ uint32_t shreg(uint32_t acc, float u) {  // (acc << 1) | sign(u)
  uint32_t d; asm("shf.l.wrap.b32 %0, %1, %2, 1;" : "=r"(d) : "r"(__float_as_uint(u)), "r"(acc)); return d;
}
// variant 7: FFMA2 update, SAT x2, FFMA2 reset, funnel-shift sign bits
template <int C0> __device__ __forceinline__ void v7(float2 &u, float2 y, float2 dec2, float2 nth2, uint32_t &acc) {
  u = __ffma2_rn(dec2, u, y);
  acc = shreg(acc, u.x); acc = shreg(acc, u.y);
  const float2 f = make_float2(sat_spike(u.x), sat_spike(u.y));
  u = __ffma2_rn(nth2, f, u);
}
// variant 8: scalar update (uniform beta), SAT, FFMA2 reset, funnel
template <int C0> __device__ __forceinline__ void v8(float2 &u, float2 y, float2 dec2, float2 nth2, uint32_t &acc) {
  u.x = fmaf(dec2.x, u.x, y.x); u.y = fmaf(dec2.x, u.y, y.y);
  acc = shreg(acc, u.x); acc = shreg(acc, u.y);
  const float2 f = make_float2(sat_spike(u.x), sat_spike(u.y));
  u = __ffma2_rn(nth2, f, u);
}
// variant 9: all scalar (uniform beta / -th), SAT, funnel
template <int C0> __device__ __forceinline__ void v9(float2 &u, float2 y, float2 dec2, float2 nth2, uint32_t &acc) {
  u.x = fmaf(dec2.x, u.x, y.x); u.y = fmaf(dec2.x, u.y, y.y);
  acc = shreg(acc, u.x); acc = shreg(acc, u.y);
  const float f0 = sat_spike(u.x), f1 = sat_spike(u.y);
  u.x = fmaf(nth2.x, f0, u.x); u.y = fmaf(nth2.x, f1, u.y);
}

// variant 10: FFMA2 update, SAT x2, scalar (uniform) resets, funnel
template <int C0> __device__ __forceinline__ void v10(float2 &u, float2 y, float2 dec2, float2 nth2, uint32_t &acc) {
  u = __ffma2_rn(dec2, u, y);
  acc = shreg(acc, u.y); acc = shreg(acc, u.x);
  const float f0 = sat_spike(u.x), f1 = sat_spike(u.y);
  u.x = fmaf(nth2.x, f0, u.x); u.y = fmaf(nth2.x, f1, u.y);
}

// variant 11: as v7, but the flag is g = [U < 0] = sat(-2^127 U) (FMUL.SAT, one register
// read; the reset becomes P = U + th g with -th folded into the drive)
__device__ __forceinline__ float sat_neg(float u) {
  float g; asm("mul.rn.ftz.sat.f32 %0, %1, 0fFF000000;" : "=f"(g) : "f"(u)); return g;
}
template <int C0> __device__ __forceinline__ void v11(float2 &u, float2 y, float2 dec2, float2 nth2, uint32_t &acc) {
  u = __ffma2_rn(dec2, u, y);
  acc = shreg(acc, u.x); acc = shreg(acc, u.y);
  const float2 g = make_float2(sat_neg(u.x), sat_neg(u.y));
  u = __ffma2_rn(nth2, g, u);
}

template <int V>
#ifndef NP
#define NP 16  // neuron pairs per thread
#endif
#ifndef THREADS
#define THREADS 512
#endif
__global__ void __launch_bounds__(THREADS, 1) bench(const float *ys, uint32_t *sink, int groups, long long *cyc, float beta, float th) {
  float2 u[NP];
  for (int i = 0; i < NP; ++i) u[i] = make_float2(0.f, 0.f);
  const float2 dec2 = make_float2(beta, beta), nth2 = make_float2(-th, -th);
  uint32_t x = 0;
  const float *yp = ys + (threadIdx.x & 31) * 32;
  uint32_t ybits[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) ybits[i] = __float_as_uint(yp[i]);
  long long t0 = clock64();
  for (int g = 0; g < groups; ++g) {
    float yv[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) yv[i] = __uint_as_float(ybits[i] ^ (uint32_t)(g & 7));  // 1 ALU op / neuron / group
    uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int c = 0; c < NP; ++c) {
        const float2 y = make_float2(yv[2 * c], yv[2 * c + 1]);
        if (V == 0) {
          switch (c % 16) {
#define CASE(k) case k: v0<(2 * k) % 32>(u[c], y, dec2, nth2, w[j]); break;
            CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15)
#undef CASE
          }
        } else if (V == 1) {
          switch (c % 16) {
#define CASE(k) case k: v1<(2 * k) % 32>(u[c], y, dec2, nth2, w[j]); break;
            CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15)
#undef CASE
          }
        } else if (V == 3) {
          switch (c % 16) {
#define CASE(k) case k: v3<(2 * k) % 32>(u[c], y, dec2, nth2, w[j]); break;
            CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15)
#undef CASE
          }
        } else if (V == 4) {
          switch (c % 16) {
#define CASE(k) case k: v4<(2 * k) % 32>(u[c], y, dec2, nth2, w[j]); break;
            CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15)
#undef CASE
          }
        } else if (V == 6) {
          switch (c % 16) {
#define CASE(k) case k: v6<(2 * k) % 32>(u[c], y, dec2, nth2, w[j]); break;
            CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15)
#undef CASE
          }
        } else if (V == 7) {
          switch (c % 16) {
#define CASE(k) case k: v7<(2 * k) % 32>(u[c], y, dec2, nth2, w[j]); break;
            CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15)
#undef CASE
          }
        } else if (V == 8) {
          switch (c % 16) {
#define CASE(k) case k: v8<(2 * k) % 32>(u[c], y, dec2, nth2, w[j]); break;
            CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15)
#undef CASE
          }
        } else if (V == 9) {
          switch (c % 16) {
#define CASE(k) case k: v9<(2 * k) % 32>(u[c], y, dec2, nth2, w[j]); break;
            CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15)
#undef CASE
          }
        } else if (V == 11) {
          switch (c % 16) {
#define CASE(k) case k: v11<(2 * k) % 32>(u[c], y, dec2, nth2, w[j]); break;
            CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15)
#undef CASE
          }
        } else if (V == 10) {
          switch (c % 16) {
#define CASE(k) case k: v10<(2 * k) % 32>(u[c], y, dec2, nth2, w[j]); break;
            CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15)
#undef CASE
          }
        } else if (V == 5) {
          switch (c % 16) {
#define CASE(k) case k: v5<(2 * k) % 32>(u[c], y, dec2, nth2, w[j]); break;
            CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15)
#undef CASE
          }
        } else {
          switch (c % 16) {
#define CASE(k) case k: v2<(2 * k) % 32>(u[c], y, dec2, nth2, w[j]); break;
            CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15)
#undef CASE
          }
        }
      }
    }
    x ^= w[0] + 3 * w[1] + 5 * w[2] + 7 * w[3];
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < NP; ++i) s += u[i].x + u[i].y;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = x ^ __float_as_uint(s);
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  const int groups = 2000, blocks = 148, threads = THREADS;
  float *ys; uint32_t *sink; long long *cyc;
  cudaMalloc(&ys, 32 * 32 * 4 * 8); cudaMalloc(&sink, blocks * threads * 4); cudaMalloc(&cyc, blocks * 8);
  static float h[8192]; for (int i = 0; i < 8192; ++i) h[i] = 0.05f + 0.3f * ((i * 37) % 101) / 101.f;
  cudaMemcpy(ys, h, sizeof h, cudaMemcpyHostToDevice);
  for (int v = 0; v < 12; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      if (v == 0) bench<0><<<blocks, threads>>>(ys, sink, groups, cyc, 0.9f, 1.f);
      if (v == 1) bench<1><<<blocks, threads>>>(ys, sink, groups, cyc, 0.9f, 1.f);
      if (v == 2) bench<2><<<blocks, threads>>>(ys, sink, groups, cyc, 0.9f, 1.f);
      if (v == 3) bench<3><<<blocks, threads>>>(ys, sink, groups, cyc, 0.9f, 1.f);
      if (v == 4) bench<4><<<blocks, threads>>>(ys, sink, groups, cyc, 0.9f, 1.f);
      if (v == 6) bench<6><<<blocks, threads>>>(ys, sink, groups, cyc, 0.9f, 1.f);
      if (v == 11) bench<11><<<blocks, threads>>>(ys, sink, groups, cyc, 0.9f, 1.f);
      if (v == 10) bench<10><<<blocks, threads>>>(ys, sink, groups, cyc, 0.9f, 1.f);
      if (v == 7) bench<7><<<blocks, threads>>>(ys, sink, groups, cyc, 0.9f, 1.f);
      if (v == 8) bench<8><<<blocks, threads>>>(ys, sink, groups, cyc, 0.9f, 1.f);
      if (v == 9) bench<9><<<blocks, threads>>>(ys, sink, groups, cyc, 0.9f, 1.f);
      if (v == 5) bench<5><<<blocks, threads>>>(ys, sink, groups, cyc, 0.9f, 1.f);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      // per SMSP: 4 warps x groups x 4 steps x 32 neurons (warp-level neuron-steps)
      double per = (double)c / ((THREADS / 128.0) * groups * 4 * 2 * NP);
      if (rep) printf("variant %d: %.3f ms, %.3f cycles per warp-neuron-step per SMSP (%s)\n", v, ms, per,
                      cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
