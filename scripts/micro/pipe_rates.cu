// Issue-rate micro-benchmark (B200): cycles per warp instruction per SMSP for the
// instruction forms the LIF epilogue is built from.  4 warps per SMSP (16 / SM),
// 8 independent chains per thread so latency never limits.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define N 8
template <int V>
__global__ void __launch_bounds__(512, 1) k(float *sink, int iters, long long *cyc, float a, float b) {
  float x[N]; float2 y[N]; uint32_t u[N];
  for (int i = 0; i < N; ++i) { x[i] = threadIdx.x * 0.001f + i; y[i] = make_float2(x[i], x[i] + 1); u[i] = threadIdx.x * 7 + i; }
  const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < N; ++i) {
        if (V == 0) x[i] = fmaf(x[i], a, b);                       // FFMA reg (uniform operands)
        if (V == 1) y[i] = __ffma2_rn(y[i], a2, b2);               // FFMA2
        if (V == 2) asm volatile("fma.rn.ftz.sat.f32 %0, %0, 0f7F000000, 0f3F800000;" : "+f"(x[i]));
        if (V == 3) asm volatile("lop3.b32 %0, %0, %1, 0x800000, 0xF8;" : "+r"(u[i]) : "r"(u[(i + 1) % N]));
        if (V == 4) { y[i] = __ffma2_rn(y[i], a2, b2); asm volatile("lop3.b32 %0, %0, %1, 0x800000, 0xF8;" : "+r"(u[i]) : "r"(u[(i + 1) % N])); }
        if (V == 5) { x[i] = fmaf(x[i], a, b); asm volatile("lop3.b32 %0, %0, %1, 0x800000, 0xF8;" : "+r"(u[i]) : "r"(u[(i + 1) % N])); }
        if (V == 6) { y[i] = __ffma2_rn(y[i], a2, b2); asm volatile("fma.rn.ftz.sat.f32 %0, %0, 0f7F000000, 0f3F800000;" : "+f"(x[i])); }
        if (V == 7) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x[i]) : "f"(y[i].x), "f"(y[i].y));  // FFMA 3-reg
        if (V == 8) asm volatile("mad.lo.u32 %0, %0, 0xFF7FFFFF, %1;" : "+r"(u[i]) : "r"(u[(i + 1) % N]));   // IMAD
        if (V == 9) { asm volatile("fma.rn.ftz.sat.f32 %0, %0, 0f7F000000, 0f3F800000;" : "+f"(x[i]));
                      asm volatile("lop3.b32 %0, %0, %1, 0x800000, 0xF8;" : "+r"(u[i]) : "r"(u[(i + 1) % N])); }
        if (V == 10) { float2 t = __fadd2_rn(y[i], b2); y[i] = t; }  // FADD2
        if (V == 11) asm volatile("shf.r.wrap.b32 %0, %0, %1, 3;" : "+r"(u[i]) : "r"(u[(i + 1) % N]));   // SHF
        if (V == 12) asm volatile("prmt.b32 %0, %0, %1, 0x3210;" : "+r"(u[i]) : "r"(u[(i + 1) % N]));
        if (V == 14) { y[i] = __ffma2_rn(y[i], a2, b2); asm volatile("fma.rn.ftz.sat.f32 %0, %0, 0f7F000000, 0f3F800000;" : "+f"(x[i]));
                       asm volatile("fma.rn.ftz.sat.f32 %0, %0, 0f7F000000, 0f3F800000;" : "+f"(y[i].x)); }   // FFMA2 + 2 SAT
        if (V == 15) { x[i] = fmaf(x[i], a, b); asm volatile("fma.rn.ftz.sat.f32 %0, %0, 0f7F000000, 0f3F800000;" : "+f"(y[i].x)); }  // FFMA(uniform) + SAT
        if (V == 16) { y[i] = __ffma2_rn(y[i], a2, b2); x[i] = fmaf(x[i], a, b); }   // FFMA2 + FFMA uniform
        if (V == 17) { y[i] = __ffma2_rn(y[i], a2, b2); asm volatile("max.f32 %0, %0, %1;" : "+f"(x[i]) : "f"(y[(i+1)%N].x)); }  // FFMA2 + FMNMX
        if (V == 18) { asm volatile("max.f32 %0, %0, %1;" : "+f"(x[i]) : "f"(y[i].x)); asm volatile("lop3.b32 %0, %0, %1, 0x800000, 0xF8;" : "+r"(u[i]) : "r"(u[(i + 1) % N])); }  // FMNMX + LOP3
        if (V == 19) { x[i] = fmaf(x[i], a, b); asm volatile("max.f32 %0, %0, %1;" : "+f"(y[i].x) : "f"(y[i].y)); }  // FFMA + FMNMX
        if (V == 20) { asm volatile("fma.rn.ftz.sat.f32 %0, %0, 0f7F000000, 0f3F800000;" : "+f"(x[i])); x[i] = fmaf(x[i], a, b); asm volatile("shf.l.wrap.b32 %0, %1, %0, 1;" : "+r"(u[i]) : "r"(__float_as_uint(x[i]))); y[i].x = fmaf(y[i].x, a, b); }  // SAT + 2 FFMA + SHF (scalar LIF mix)
        if (V == 21) { y[i] = __ffma2_rn(y[i], a2, b2); asm volatile("fma.rn.ftz.sat.f32 %0, %0, 0f7F000000, 0f3F800000;" : "+f"(x[i])); asm volatile("shf.l.wrap.b32 %0, %1, %0, 1;" : "+r"(u[i]) : "r"(__float_as_uint(x[i]))); }  // FFMA2 + SAT + SHF (current LIF mix)
        if (V == 22) { asm volatile("{.reg .b32 h; cvt.rn.f16x2.f32 h, %1, %2; fma.rn.sat.f16x2 %0, h, %3, %4;}" : "=r"(u[i]) : "f"(y[i].x), "f"(y[i].y), "r"(0x7BFF7BFFu), "r"(0x3C003C00u)); y[i].x += 1e-30f; }  // F2FP + HFMA2.SAT
        if (V == 13) { asm volatile("max.f32 %0, %0, %1;" : "+f"(x[i]) : "f"(y[i].x)); }
      }
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < N; ++i) s += x[i] + y[i].x + y[i].y + (float)u[i];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int V> void run(const char *name, int per_iter_instr, float *sink, long long *cyc) {
  const int iters = 2000;
  for (int rep = 0; rep < 2; ++rep) {
    k<V><<<148, 512>>>(sink, iters, cyc, 0.999f, 0.001f);
    cudaDeviceSynchronize();
  }
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double instr = 4.0 * iters * 16 * N * per_iter_instr;  // warp instrs per SMSP
  printf("%-34s %.3f cycles / warp-instr / SMSP  (%s)\n", name, c / instr, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  float *sink; long long *cyc;
  cudaMalloc(&sink, 148 * 512 * 4); cudaMalloc(&cyc, 148 * 8);
  run<0>("FFMA (uniform a,b)", 1, sink, cyc);
  run<7>("FFMA 3-reg", 1, sink, cyc);
  run<1>("FFMA2", 1, sink, cyc);
  run<10>("FADD2", 1, sink, cyc);
  run<2>("FFMA.SAT imm,imm", 1, sink, cyc);
  run<3>("LOP3 r,r,imm", 1, sink, cyc);
  run<11>("SHF", 1, sink, cyc);
  run<12>("PRMT", 1, sink, cyc);
  run<13>("FMNMX", 1, sink, cyc);
  run<8>("IMAD imm", 1, sink, cyc);
  run<4>("FFMA2 + LOP3", 2, sink, cyc);
  run<5>("FFMA + LOP3", 2, sink, cyc);
  run<6>("FFMA2 + FFMA.SAT", 2, sink, cyc);
  run<9>("FFMA.SAT + LOP3", 2, sink, cyc);
  run<14>("FFMA2 + 2 SAT", 3, sink, cyc);
  run<15>("FFMA(uni) + SAT", 2, sink, cyc);
  run<16>("FFMA2 + FFMA(uni)", 2, sink, cyc);
  run<17>("FFMA2 + FMNMX", 2, sink, cyc);
  run<18>("FMNMX + LOP3", 2, sink, cyc);
  run<19>("FFMA + FMNMX", 2, sink, cyc);
  run<20>("SAT + 2 FFMA(uni) + SHF", 4, sink, cyc);
  run<21>("FFMA2 + SAT + SHF", 3, sink, cyc);
  run<22>("F2FP + HFMA2.SAT", 2, sink, cyc);
  return 0;
}
