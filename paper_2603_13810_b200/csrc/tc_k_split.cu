// tcgen05 Conv-LIF kernel instantiations: operand path PATH_SPLIT, inference,
// every C_out tile width (see tc_impl.cuh tc_launch_path)
#define TAC_TC_PATH PATH_SPLIT
#define TAC_TC_TRAIN false
#include "tc_impl.cuh"
