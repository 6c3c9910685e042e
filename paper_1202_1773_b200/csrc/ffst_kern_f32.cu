// float instantiation of the FFST kernels (sm_100a)
#include "ffst_launch.cuh"
namespace ffst { FFST_INSTANTIATE(float) }
