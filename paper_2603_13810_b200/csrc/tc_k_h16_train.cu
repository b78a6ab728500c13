// tcgen05 Conv-LIF kernel instantiations: operand path PATH_H16, training forward (writes the per-group drive y_seq),
// every C_out tile width (see tc_impl.cuh tc_launch_path)
#define TAC_TC_PATH PATH_H16
#define TAC_TC_TRAIN true
#include "tc_impl.cuh"
