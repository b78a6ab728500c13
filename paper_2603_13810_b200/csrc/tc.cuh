// tc.cuh -- the tcgen05 engine of libtacsnn (fused aggregation + tcgen05/TMEM
// implicit-GEMM conv + LIF epilogue).  See tc.cu and DESIGN.md.
#pragma once
#include <cstddef>

#include "../../include/tacsnn.h"
#include "layer.cuh"

namespace tacsnn {

// Shape envelope of the tcgen05 kernel (independent of beta / K / mode).
bool tc_shape_ok(const tac_conv_lif_desc *d);
// Full envelope (shape + exactness of the integer aggregate for beta, K, mode).
bool tc_supported(const tac_conv_lif_desc *d);
const char *tc_unsupported_reason(const tac_conv_lif_desc *d);
size_t tc_weights_bytes(const tac_conv_lif_desc *d);
// builds the tcgen05 image; returns the exponent e of the fp16-path operand prescale
// 2^e (0 on the int8 path), which the caller keeps in the plan and passes back in
// LayerParams::yscale_exp
int tc_prepare(const tac_conv_lif_desc *d, const float *weight, const float *bias,
               unsigned char *dst);
// backward replay of the forward integrator: does the subtract epilogue run in the
// shifted state U = V - v_th with the (decay - 1) v_th offset folded into Y (tc.cu)?
bool tc_u_domain(const tac_conv_lif_desc *d);
// device [2^e, 2^-e] Y prescale of the fp16 operand paths, NULL on the int8 path
const float *tc_yscale_ptr(const tac_conv_lif_desc *d, const unsigned char *tc_prep);
int tc_launch(const tac_conv_lif_desc *d, const LayerParams &p, const unsigned char *tc_prep,
              void *stream, int *launches);

// fully connected layers (H = W = R = S = 1) on tcgen05 (fc.cu); the tc_* entry points
// above dispatch to these for such shapes
bool fc_is_fc(const tac_conv_lif_desc *d);
const char *fc_reason(const tac_conv_lif_desc *d);  // NULL when the FC kernel can run it
size_t fc_weights_bytes(const tac_conv_lif_desc *d);
// device workspace of the two-phase FC mode (0: this layer runs fused)
size_t fc_ws_bytes(const tac_conv_lif_desc *d);
int fc_prepare(const tac_conv_lif_desc *d, const float *weight, unsigned char *dst);
int fc_launch(const tac_conv_lif_desc *d, const LayerParams &p, const unsigned char *img, void *stream,
              int *launches);

}  // namespace tacsnn
