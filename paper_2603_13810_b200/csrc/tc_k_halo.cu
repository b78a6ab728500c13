// tcgen05 Conv-LIF kernel instantiations: operand path PATH_HALO, inference,
// every C_out tile width (see tc_impl.cuh tc_launch_path)
#define TAC_TC_PATH PATH_HALO
#define TAC_TC_TRAIN false
#include "tc_impl.cuh"
