// float instantiation of the arbitrary-n kernels (sm_100a)
#include "ffst_gen_launch.cuh"
namespace ffst { FFST_GEN_INSTANTIATE(float) }
