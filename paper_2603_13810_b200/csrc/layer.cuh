// layer.cuh -- device-side parameter block shared by the libtacsnn kernels.
// Built by abi.cu from a validated tac_conv_lif_desc (include/tacsnn.h).
#pragma once
#include <cstdint>

namespace tacsnn {

constexpr int kMaxK = 32;

struct LayerParams {
  // geometry
  int T, B, Cin, H, W, Cout, R, S, stride, pad;
  int K, mode, reset, pool;
  int Ho, Wo;        // pre-pool conv output extent
  int Hq, Wq;        // stored output extent (pooled or not)
  int G;             // number of groups = conv calls = T / K
  int nsteps;        // LIF steps per group: K (TAC-TP), 1 (TAC, dense)
  int T_out;
  int wpr_in, wpr_out;
  long long in_st, in_sb, out_st, out_sb;  // u32-word strides
  // LIF
  float v_th, v_reset;
  float decay;       // beta (dense / TAC-TP) or beta^K (TAC), rounded from fp64
  float coef[kMaxK]; // beta^{K-1-j}, rounded from fp64 (A_k weights)
  // buffers
  const uint32_t *in;     // packed spikes (input_kind SPIKES)
  const float *xin;       // fp32 [T][B][H][W][C_in] (input_kind REAL); strides in floats
  uint32_t *out;
  const float *v_init;
  float *v_final;
  uint32_t *counts;
  const float *w;     // SIMT weights, fp32 [Cin][R][S][Cout]
  const float *bias;  // fp32 [Cout]
};

enum { MODE_DENSE = 0, MODE_TAC = 1, MODE_TACTP = 2 };
enum { RESET_SUBTRACT = 0, RESET_DELAYED = 1, RESET_HARD = 2 };

// Launchers implemented in simt.cu / tc.cu.  Return cudaGetLastError() as int.
int launch_zero_outputs(const LayerParams &p, void *stream, int *launches);
int launch_simt_conv_lif(const LayerParams &p, void *stream, int *launches);
int launch_add_u32(uint32_t *dst, const uint32_t *src, long long n, void *stream);  // dst += src
int launch_pack(const uint8_t *dense, uint32_t *packed, int T, int B, int C, int H,
                int W, void *stream);
int launch_unpack(const uint32_t *packed, uint8_t *dense, int T, int B, int C, int H,
                  int W, void *stream);

}  // namespace tacsnn
