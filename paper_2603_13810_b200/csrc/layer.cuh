// layer.cuh -- device-side parameter block shared by the libtacsnn kernels.
// Built by abi.cu from a validated tac_conv_lif_desc (include/tacsnn.h).
#pragma once
#include <cstdint>

namespace tacsnn {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device, size) instead of
// on every launch (a host-side cost the launch-bound small layers pay per call)
cudaError_t ensure_dyn_smem(const void *kern, int bytes);

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
  float *y_seq;       // training forward: per-group drive [G][B][Ho][Wo][Cout] as the LIF consumed it
  int yscale_exp;     // tcgen05 fp16 paths: the image's operand prescale 2^e (tac_plan::scale_code)
  void *ws;           // the call's device workspace (two-phase FC layers), or NULL
  size_t ws_bytes;
};

enum { MODE_DENSE = 0, MODE_TAC = 1, MODE_TACTP = 2 };
enum { RESET_SUBTRACT = 0, RESET_DELAYED = 1, RESET_HARD = 2 };

// Launchers implemented in simt.cu / tc.cu.  Return cudaGetLastError() as int.
int launch_zero_outputs(const LayerParams &p, void *stream, int *launches);
int launch_simt_conv_lif(const LayerParams &p, void *stream, int *launches);
int launch_add_u32(uint32_t *dst, const uint32_t *src, long long n, void *stream);  // dst += src
int launch_vote(const uint32_t *counts, int B, int C, int voters, int T_out, float *scores, void *stream);
int launch_pack(const uint8_t *dense, uint32_t *packed, int T, int B, int C, int H,
                int W, void *stream);
int launch_unpack(const uint32_t *packed, uint8_t *dense, int T, int B, int C, int H,
                  int W, void *stream);

// ---- backward (backward.cu) ----
struct BwdParams {
  // layer geometry / LIF (as the forward)
  int T, B, Cin, H, W, Cout, R, S, stride, pad, K, mode, G, nsteps, Ho, Wo, wpr_in;
  long long in_st, in_sb;  // packed words (spikes) or floats (real input)
  float decay, v_th, coef[kMaxK];
  // replay of the forward integrator (backward LIF): the tcgen05 subtract epilogue's form
  // (udomain: y = (Y - v_th) s, U = decay V + y, V <- U + v_th s [U < 0]) or the plain
  // V-domain form (y = Y s, V = decay V + y, V <- V - v_th s on a spike); s = 2^e
  int udomain;
  const float *yscale;  // device [s, 1/s] or NULL (= 1)
  // surrogate
  int surrogate, detach;
  float sg_alpha;
  // buffers
  const uint32_t *in;   // packed input spikes, or
  const float *xin;     // fp32 input frames [T][B][H][W][Cin]
  const float *v_init;  // [B][Ho][Wo][Cout] or NULL
  const float *y_seq;   // [G][B][Ho][Wo][Cout]
  const float *g_spikes;  // [nsteps * G][B][Ho][Wo][Cout]
  const float *g_vfinal;  // or NULL
  float *g_y;           // workspace [G][B][Ho][Wo][Cout]
  float *g_vinit;       // or NULL
  const float *w;       // SIMT weights [Cin][R][S][Cout]
  float *g_w;           // [Cout][Cin][R][S]
  float *g_b;           // [Cout]
  float *g_in;          // [T][B][H][W][Cin] or NULL
  float *g_alpha;       // [K] or NULL
  void *dg_img;         // workspace for the tcgen05 input-gradient weights (bwd_tc.cu), or NULL
  int tc;               // the layer's forward ran on tcgen05 (the tcgen05 backward kernels apply)
  void *wg_abuf;        // workspace for the weight gradient's bf16 A_k buffer, or NULL
  void *fc_ws;          // fully connected layers: workspace [A_k | dA] fp32 [G B][C_in] each, or NULL
};
int launch_backward(const BwdParams &p, void *stream, int *launches);
// tcgen05 input gradient (bwd_tc.cu): eligibility, its weight-image bytes, launch
bool dgrad_tc_ok(const BwdParams &p);
size_t dgrad_tc_ws_bytes(int Cin, int Cout);
int launch_dgrad_tc(const BwdParams &p, void *img, void *stream, int *launches);
// tcgen05 weight gradient (bwd_tc.cu)
bool wgrad_tc_ok(const BwdParams &p);
size_t wgrad_tc_ws_bytes(int G, int B, int H, int W, int Cin, int Ho, int Wo, int Cout);
int launch_wgrad_tc(const BwdParams &p, void *stream, int *launches);
int launch_or_pool2(const uint32_t *in, uint32_t *out, int T, int B, int C, int H, int W, void *stream);
int launch_or_pool2_backward(const uint32_t *pre, const float *g_pooled, float *g_pre, int T, int B,
                             int C, int H, int W, void *stream);

}  // namespace tacsnn
