// fp32 instantiation of the depth-variant correlation kernels.
#include "conv_inst.cuh"
template cudaError_t bd3mg::conv_launch<float>(int, bool, bd3mg::ConvArgs<float>&, int, cudaStream_t);
