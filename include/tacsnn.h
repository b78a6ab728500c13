/*
 * tacsnn.h -- C ABI of libtacsnn: the Conv-LIF layer of arXiv 2603.13810
 * ("TAC: Temporal Aggregated Convolution") on NVIDIA B200 (sm_100a).
 *
 * One call runs ONE spiking convolutional layer over a whole spike sequence:
 *
 *   dense  (mode 0)  Eq. (1), PAPER.md:101-105 -- T conv calls:
 *            V_t = beta V_{t-1} + W*S_t + b ; s_t = [V_t >= v_th] ; reset
 *   TAC    (mode 1)  Algorithm 1, PAPER.md:135-150 -- T/K conv calls, T/K outputs:
 *            A_k = sum_{j<K} beta^{K-1-j} S_{kK+j}         (Definition)
 *            Y_k = W*A_k + b ; V = beta^K V + Y_k ; s_k = [V >= v_th] ; reset
 *   TAC-TP (mode 2)  Algorithm 2, PAPER.md:170-187 -- T/K conv calls, T outputs:
 *            same A_k, Y_k ; then K times: V = beta V + Y_k ; s = [V >= v_th] ; reset
 *
 * "W*X" is the 2-D cross-correlation with zero padding,
 * W [C_out][C_in][R][S], stride `stride`, padding `pad`; the bias b is added once
 * per conv call (folded inference BatchNorm; R3).
 * Reset forms (R1): SUBTRACT V -= s v_th right after spiking
 * (Alg. 1 l.7 / Alg. 2 l.8, the default); SUBTRACT_DELAYED subtracts
 * v_th s_{t-1} at the next update (Eq. (1), App. A);
 * HARD sets V = v_reset on a spike.  Threshold ties fire.
 *
 * ---------------------------------------------------------------------------
 * Packed spike layout (inputs and outputs), "tac-packed-v1":
 *   u32 words [T][B][H][WPR], WPR = ceil(W*C/32).  The bit of spike
 *   (t, b, c, y, x) is at row offset r = x*C + c: word r>>5, bit r&31 (LSB
 *   first).  Bits past W*C in the last word of a row are zero.  Rows are packed
 *   (row stride WPR); the t and b strides are explicit (in words) so batch
 *   shards are zero-copy views; 0 means the packed default (B*H*WPR, H*WPR).
 *   tac_pack_spikes / tac_unpack_spikes convert from/to u8 {0,1} [T][B][C][H][W]
 *   (the paper's layout, Alg. 1 "Require").
 * Output spikes use the same layout with C = C_out, (H, W) = the layer output
 *   extent -- after the optional fused 2x2 OR-pool (= MaxPool(2) of binary
 *   spikes) when out_pool = 2; odd H', W' pool in floor mode
 *   (H_o = floor(H'/2): the last row / column is dropped, as MaxPool2d).  T_out = T/K for TAC
 *   (ceil(T/K) with partial_last_group), else T.
 * v_init / v_final: fp32 [B][H'][W'][C_out] (channels last, PRE-pool extent
 *   H' = (H+2 pad-R)/stride+1), contiguous.  v_final is V after the last step
 *   (post-reset for SUBTRACT / HARD; R5).  NULL v_init means V=0
 *   (Alg. 1 l.1); with SUBTRACT_DELAYED the pending reset at call start is
 *   [v_init >= v_th] (R4), so chained calls equal one long call
 *   bit for bit (every engine carries V itself across the boundary, scaled by
 *   a power of two at most).
 * counts: u32 [B][C_out] = sum over output steps and PRE-pool pixels of the
 *   spikes (the spike-count readout).
 *
 * ---------------------------------------------------------------------------
 * Conventions for every function:
 *  - Ownership: the caller allocates every buffer (device memory unless a
 *    parameter says host); the library never allocates device memory and keeps
 *    no reference to any buffer after the call returns.
 *  - Ordering: device work is enqueued on `stream` (a cudaStream_t passed as
 *    void*; NULL = legacy default stream) and is asynchronous; results are valid
 *    when the stream reaches the call.  No implicit device synchronisation,
 *    except tac_prepare_weights which copies host data synchronously.
 *  - Errors: all argument checks run on the host before anything is launched
 *    and return a status; on error nothing is launched and outputs are
 *    untouched.  A failed launch returns TAC_ERR_CUDA.  tac_last_error_detail()
 *    (thread-local) names the offending argument.  No C++ exception crosses
 *    this ABI.  Asynchronous device faults surface at the caller's next sync.
 *  - Thread safety: no global mutable state besides the thread-local detail
 *    string and launch counter; distinct calls may run concurrently.
 */
#ifndef TACSNN_H_
#define TACSNN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TACSNN_ABI_VERSION 3 /* 2: input_kind + tac_conv_lif_forward_real;
                                3: tac_plan (prepared image + descriptor fingerprint),
                                   desc.agg_weights (learnable aggregation weights) */

typedef enum { TAC_MODE_DENSE = 0, TAC_MODE_TAC = 1, TAC_MODE_TACTP = 2 } tac_mode;

typedef enum {
  TAC_RESET_SUBTRACT = 0,         /* Alg. 1 l.7 / Alg. 2 l.8 (default)            */
  TAC_RESET_SUBTRACT_DELAYED = 1, /* Eq. (1): V_t = bV_{t-1} + I_t - v_th s_{t-1} */
  TAC_RESET_HARD = 2              /* V = v_reset on spike                         */
} tac_reset;

/* What the layer reads (desc.input_kind).  REAL is the continuous-valued first
 * layer of the paper's DVS network (log-normalised event counts):
 * A_k = sum_j beta^{K-1-j} X_{kK+j} is then real-valued and the conv of the
 * aggregate is still exact by linearity. */
typedef enum { TAC_INPUT_SPIKES = 0, TAC_INPUT_REAL = 1 } tac_input;

typedef enum {
  TAC_ENGINE_AUTO = 0,    /* TCGEN05 when the layer qualifies, else SIMT        */
  TAC_ENGINE_SIMT = 1,    /* fp32 FFMA direct conv + LIF; any R/S/stride/pad/K  */
  TAC_ENGINE_TCGEN05 = 2  /* fused tcgen05/TMEM implicit GEMM   */
} tac_engine;

typedef enum {
  TAC_OK = 0,
  TAC_ERR_NULL = 1,             /* a required pointer is NULL                   */
  TAC_ERR_SHAPE = 2,            /* non-positive extent, H' < 1, pooled extent < 1  */
  TAC_ERR_K_NOT_DIVIDING_T = 3, /* K < 1 or T % K != 0 */
  TAC_ERR_PARAM = 4,            /* beta not in (0,1), v_th <= 0, bad enum        */
  TAC_ERR_NONFINITE = 5,        /* non-finite weight, bias, beta, v_th, v_reset  */
  TAC_ERR_ALIGN = 6,            /* pointer / stride alignment                    */
  TAC_ERR_UNSUPPORTED = 7,      /* layer outside the requested engine's envelope */
  TAC_ERR_WORKSPACE = 8,        /* buffer smaller than required                  */
  TAC_ERR_CUDA = 9              /* CUDA runtime error (detail has the text)      */
} tac_status;

/* Layer descriptor (host struct, passed by pointer to every call). */
typedef struct tac_conv_lif_desc {
  int32_t T, B, C_in, H, W;         /* logical input spikes [T][B][C_in][H][W]      */
  int32_t C_out, R, S, stride, pad; /* kernel [C_out][C_in][R][S]                   */
  int32_t K;                        /* group size; ignored (=1) for DENSE           */
  int32_t mode;                     /* tac_mode                                     */
  float beta;                       /* membrane decay, 0 < beta < 1  */
  float v_th;                       /* threshold > 0                                */
  float v_reset;                    /* HARD reset value                             */
  int32_t reset;                    /* tac_reset                                    */
  int32_t out_pool;                 /* 1 = none, 2 = fused 2x2 OR-pool (floor mode)  */
  int32_t engine;                   /* tac_engine                                   */
  int64_t in_stride_t, in_stride_b; /* u32 words (REAL input: floats); 0 = default  */
  int64_t out_stride_t, out_stride_b;
  int32_t input_kind;               /* tac_input (0 = packed spikes)                */
  int32_t partial_last_group;       /* 0: K must divide T (TAC_ERR_K_NOT_DIVIDING_T);
                                       1: G = ceil(T/K) groups, the last one of
                                       K' = T - (G-1)K frames is a complete group of
                                       size K' (A_k with beta^{K'-1-j}, TAC decay
                                       beta^{K'}, K' TAC-TP steps) -- the paper's
                                       T = 25 with K = 4/8/16.
                                       Runs as the full groups + the short group
                                       chained through the membrane state; needs a
                                       workspace (tac_workspace_bytes); a short group
                                       outside the tcgen05 envelope runs on SIMT.  */
  const float *agg_weights;         /* HOST fp32 [K] or NULL.  Learnable aggregation
                                       weights alpha_j replacing beta^{K-1-j} in
                                       A_k = sum_j alpha_j S_{kK+j} (the paper's
                                       "learnable aggregation weights", PAPER.md:427;
                                       DESIGN.md reading R11).  Read during
                                       tac_prepare_weights and every call that takes
                                       the desc; must be finite.  The membrane decay
                                       (beta^K for TAC, beta per TAC-TP step) is not
                                       affected.  A short last group of K' frames uses
                                       the last K' entries alpha_{K-K'+j} (with the
                                       default alpha_j = beta^{K-1-j} that is exactly
                                       beta^{K'-1-j}, reading D6').  NULL = beta^{K-1-j}. */
} tac_conv_lif_desc;

/* Prepared layer ("plan"): a plain host struct the caller owns (stack, heap, ...),
 * filled by tac_prepare_weights and passed by pointer to every forward call.  It
 * names the caller's device image and carries a fingerprint of the descriptor
 * fields the image depends on (C_in, C_out, R, S, stride, pad, K, mode, beta,
 * v_th, reset, input_kind, the short-group size, agg_weights), so a forward call
 * with a descriptor the image was NOT prepared for -- e.g. weights prepared for TAC
 * run as TAC-TP, whose folded bias and aggregate scale differ -- is refused with
 * TAC_ERR_PARAM before anything is launched.  Fields that do not enter the image
 * (T when K divides it, B, H, W, strides, out_pool, engine, v_reset) may differ
 * between preparation and the call (batch shards, chunked sequences). */
typedef struct tac_plan {
  void *prepared;        /* device image (caller-owned, >= tac_weights_bytes, 256-B aligned) */
  size_t bytes;          /* size of the image                                               */
  uint64_t fingerprint;  /* of the descriptor at preparation (opaque)                       */
  int32_t abi_version;   /* TACSNN_ABI_VERSION of the library that prepared it              */
  int32_t scale_code;    /* library-private: the image's operand prescale exponents; do not modify */
} tac_plan;

/* Validate a descriptor (no device access).  TAC_OK or the first violation. */
tac_status tac_desc_check(const tac_conv_lif_desc *desc);

/* Output geometry: T_out, output (pooled) H_o, W_o and words per output row. */
tac_status tac_out_shape(const tac_conv_lif_desc *desc, int32_t *T_out,
                         int32_t *H_out, int32_t *W_out, int32_t *out_words_per_row);

/* Engine a call with this descriptor runs on (resolves AUTO); -1 if invalid or
 * if an explicitly requested engine cannot run the layer. */
int32_t tac_select_engine(const tac_conv_lif_desc *desc);

/* Size in bytes of the prepared-weights device buffer for this descriptor. */
tac_status tac_weights_bytes(const tac_conv_lif_desc *desc, size_t *bytes);

/* Prepare weights once per (desc, W, b): validates finiteness,
 * builds every engine's device format and copies it into `prepared` (device,
 * >= tac_weights_bytes, 256-B aligned), then fills *plan (host, caller-owned).
 * weight: HOST fp32 [C_out][C_in][R][S]; bias: HOST fp32 [C_out] or NULL (= 0).
 * Synchronous host->device copy.  On error *plan is left untouched. */
tac_status tac_prepare_weights(const tac_conv_lif_desc *desc, const float *weight,
                               const float *bias, void *prepared, size_t bytes,
                               void *stream, tac_plan *plan);

/* Workspace bytes tac_conv_lif_forward uses (device, 256-B aligned):
 *  - partial_last_group with K not dividing T: REQUIRED -- the membrane state between
 *    the full groups and the short last group, fp32 [B][H'][W'][C_out], plus u32
 *    [B][C_out] counts;
 *  - a fully connected layer (H = W = R = S = 1) on tcgen05 whose batch gives few
 *    128-sample tiles: OPTIONAL -- with it the layer runs two-phase (the group GEMMs
 *    split over the SMs into the workspace, fp32 [S][G][B][C_out], then the LIF); with
 *    ws = NULL it runs fused (one CTA per tile, slower for small B).
 *  - otherwise 0. */
tac_status tac_workspace_bytes(const tac_conv_lif_desc *desc, size_t *bytes);

/* The layer (one call = whole sequence, all groups).
 *   plan       host, filled by tac_prepare_weights for a descriptor with the same
 *              image-relevant fields (see tac_plan; TAC_ERR_PARAM otherwise)
 *   spikes_in  device u32, packed layout above (4-B aligned)
 *   v_init     device fp32 [B][H'][W'][C_out] or NULL (= 0)
 *   spikes_out device u32, packed, T_out x B x H_o x WPR_out (with strides)
 *   v_final    device fp32 [B][H'][W'][C_out] or NULL (not written)
 *   counts     device u32 [B][C_out] or NULL (overwritten, not accumulated)
 *   ws         device workspace of ws_bytes >= tac_workspace_bytes (or NULL if 0)
 * spikes_out must not alias spikes_in. */
tac_status tac_conv_lif_forward(const tac_conv_lif_desc *desc, const tac_plan *plan,
                                const uint32_t *spikes_in, const float *v_init,
                                uint32_t *spikes_out, float *v_final,
                                uint32_t *counts, void *ws, size_t ws_bytes,
                                void *stream);

/* The same layer on a continuous-valued input (desc.input_kind = TAC_INPUT_REAL;
 * tac_conv_lif_forward rejects such a descriptor and this call rejects spikes):
 *   x_in  device fp32 [T][B][H][W][C_in] (channels last, 4-B aligned); the t and b
 *         strides (desc.in_stride_t / in_stride_b) are in floats, 0 = contiguous
 *         (H*W*C_in, B*H*W*C_in).
 * Everything else (a plan prepared from a descriptor with the same input_kind,
 * outputs, errors, ordering) as tac_conv_lif_forward.  tcgen05 takes C_in <= 2
 * (the aggregate is carried as fp16 hi + lo, |error| <= 2^-22 |A|); the SIMT engine
 * any shape. */
tac_status tac_conv_lif_forward_real(const tac_conv_lif_desc *desc, const tac_plan *plan,
                                     const float *x_in, const float *v_init,
                                     uint32_t *spikes_out, float *v_final, uint32_t *counts,
                                     void *ws, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * Training: surrogate-gradient backpropagation through time
 * through the grouped LIF, as the paper trains every network it reports
 * (App. E).  Subtract reset (the one the paper
 * trains with), K | T, out_pool = 1 (pool with tac_or_pool2), at most 64 LIF
 * steps per call; other descriptors return TAC_ERR_UNSUPPORTED.
 *
 *   forward   V_t = decay U_{t-1} + Y_k ; s_t = Theta(V_t - v_th) ; U_t = V_t - v_th s_t
 *   surrogate ds_t/dV_t := h(V_t - v_th):
 *               FAST_SIGMOID  h(u) = 1 / (alpha |u| + 1)^2            (MNIST/FMNIST: alpha 25)
 *               ARCTAN        h(u) = (alpha/2) / (1 + (pi/2 alpha u)^2) (DVS-Gesture: alpha 2)
 *   reset     detach_reset = 1: dU_t/dV_t = 1 (DVS, "detach reset"); 0: 1 - v_th h
 *   BPTT      dV_t = (dL/ds_t - [!detach] v_th gU) h + gU ; gU <- decay dV_t ;
 *             dL/dY_k = sum_t in group k dV_t ; dL/dv_init = gU
 *   conv      dL/dW = sum_k corr(dL/dY_k, A_k) ; dL/db = sum dL/dY_k ;
 *             dL/dS_{kK+j} = a_j conv^T(dL/dY_k, W) ; dL/da_j = sum_k <conv^T(dL/dY_k, W), S_{kK+j}>
 * (a_j = desc.agg_weights or beta^{K-1-j}).  The conv gradients run once per group,
 * like the forward conv: G = T/K instead of T.
 * ------------------------------------------------------------------------- */
typedef enum { TAC_SURROGATE_FAST_SIGMOID = 0, TAC_SURROGATE_ARCTAN = 1 } tac_surrogate;

typedef struct tac_grad_desc {
  int32_t surrogate;     /* tac_surrogate                                  */
  float alpha;           /* surrogate sharpness, finite and > 0            */
  int32_t detach_reset;  /* 1: the reset term carries no gradient          */
} tac_grad_desc;

/* Training forward: tac_conv_lif_forward (or _real, by desc.input_kind: `input` is the
 * packed spikes or the fp32 frames) that also writes
 *   y_seq  device fp32 [G][B][H'][W'][C_out], G = T/K: the per-group drive exactly as
 *          the LIF integrator consumed it (engine-specific offset / scale; opaque, read
 *          only by tac_conv_lif_backward with the same desc and plan).
 * Other arguments, ordering and errors as tac_conv_lif_forward. */
tac_status tac_conv_lif_forward_train(const tac_conv_lif_desc *desc, const tac_plan *plan,
                                      const void *input, const float *v_init,
                                      uint32_t *spikes_out, float *v_final, uint32_t *counts,
                                      float *y_seq, void *stream);

/* Workspace of tac_conv_lif_backward: fp32 dL/dY [G][B][H'][W'][C_out]. */
tac_status tac_backward_workspace_bytes(const tac_conv_lif_desc *desc, size_t *bytes);

/* Backward of one training forward (same desc, plan, input, v_init; its y_seq):
 *   g_spikes       device fp32 [T_out][B][H'][W'][C_out] = dL/ds (output spikes, channels last)
 *   g_v_final      device fp32 [B][H'][W'][C_out] = dL/dv_final, or NULL (= 0)
 *   g_weight       device fp32 [C_out][C_in][R][S]   (overwritten)
 *   g_bias         device fp32 [C_out]               (overwritten)
 *   g_input        device fp32 [T][B][H][W][C_in] = dL/d(input frames), or NULL
 *   g_v_init       device fp32 [B][H'][W'][C_out], or NULL
 *   g_agg_weights  device fp32 [K] = dL/da_j, or NULL
 *   ws             device, >= tac_backward_workspace_bytes
 * Gradients are sums over the batch (fp32, atomics: the summation order, and so the
 * last bits, may vary from run to run). */
tac_status tac_conv_lif_backward(const tac_conv_lif_desc *desc, const tac_plan *plan,
                                 const tac_grad_desc *grad, const void *input, const float *v_init,
                                 const float *y_seq, const float *g_spikes, const float *g_v_final,
                                 float *g_weight, float *g_bias, float *g_input, float *g_v_init,
                                 float *g_agg_weights, void *ws, size_t ws_bytes, void *stream);

/* 2x2 OR-pool (= MaxPool(2) of binary spikes; floor mode) of packed spikes
 * [T][B][H][WPR(W, C)] -> [T][B][H/2][WPR(W/2, C)], both contiguous. */
tac_status tac_or_pool2(const uint32_t *in, uint32_t *out, int32_t T, int32_t B, int32_t C,
                        int32_t H, int32_t W, void *stream);

/* Its backward with MaxPool2d semantics: the gradient of a window goes to the window's
 * first maximal element in row-major order (the first spike, or the top-left element of
 * an all-zero window); rows / columns dropped by the floor get 0.
 *   spikes_prepool packed [T][B][H][WPR(W, C)]; g_pooled fp32 [T][B][H/2][W/2][C];
 *   g_prepool fp32 [T][B][H][W][C] (overwritten). */
tac_status tac_or_pool2_backward(const uint32_t *spikes_prepool, const float *g_pooled,
                                 float *g_prepool, int32_t T, int32_t B, int32_t C, int32_t H,
                                 int32_t W, void *stream);

/* VotingLayer readout of the DVS network ("LIF -> VotingLayer(10 voters,
 * 11 classes)", :595): the class score is the mean firing rate of the class's voters,
 *   scores[b][j] = (sum_{v < voters} counts[b][j voters + v]) / (voters T_out)
 * (the sum is exact in u32, one fp32 division).  counts u32 [B][C] (device, e.g. the
 * counts of the last FC-LIF layer), C % voters == 0; scores fp32 [B][C / voters]
 * (device, overwritten).  TAC_ERR_SHAPE on a bad extent, TAC_ERR_NULL / _ALIGN on
 * bad pointers; nothing is launched on error. */
tac_status tac_vote(const uint32_t *counts, int32_t B, int32_t C, int32_t voters, int32_t T_out,
                    float *scores, void *stream);

/* u8 {0,1} [T][B][C][H][W] (device) <-> packed [T][B][H][WPR] (device).
 * pack treats any non-zero byte as a spike. */
tac_status tac_pack_spikes(const uint8_t *dense01, uint32_t *packed, int32_t T,
                           int32_t B, int32_t C, int32_t H, int32_t W, void *stream);
tac_status tac_unpack_spikes(const uint32_t *packed, uint8_t *dense01, int32_t T,
                             int32_t B, int32_t C, int32_t H, int32_t W, void *stream);

const char *tac_status_string(tac_status status);
const char *tac_last_error_detail(void); /* thread-local; "" when none */
int32_t tac_abi_version(void);           /* TACSNN_ABI_VERSION */
/* Device kernels launched by this thread's most recent successful
 * tac_conv_lif_forward / tac_pack_spikes / tac_unpack_spikes call. */
int32_t tac_last_launch_count(void);

/* Diagnostics (not needed for computation): route a per-group role timeline of
 * CTA 0 of every tcgen05 launch into `dev_buffer` (device, >= 4096 x 16 u64,
 * %globaltimer ns; slots: producer start/done, MMA ready/issued, epilogue
 * full/released/done), or stop with NULL.  Process-global; not thread-safe.
 * Only a library built with -DTACSNN_TRACE records anything (scripts/trace_layer.py). */
void tac_debug_set_trace(void *dev_buffer);

#ifdef __cplusplus
}
#endif
#endif /* TACSNN_H_ */
