// fp64 instantiation of the depth-variant correlation kernels.
#include "conv_inst.cuh"
template cudaError_t bd3mg::conv_launch<double>(int, bool, bd3mg::ConvArgs<double>&, int, cudaStream_t);
