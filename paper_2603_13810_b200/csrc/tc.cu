// tc.cu -- tcgen05 engine (placeholder until the fused kernel lands).
#include "tc.cuh"

namespace tacsnn {
bool tc_shape_ok(const tac_conv_lif_desc *) { return false; }
bool tc_supported(const tac_conv_lif_desc *) { return false; }
const char *tc_unsupported_reason(const tac_conv_lif_desc *) { return "tcgen05 engine not built"; }
size_t tc_weights_bytes(const tac_conv_lif_desc *) { return 0; }
void tc_prepare(const tac_conv_lif_desc *, const float *, const float *, unsigned char *) {}
int tc_launch(const tac_conv_lif_desc *, const LayerParams &, const unsigned char *, void *, int *) {
  return 1;
}
}  // namespace tacsnn
