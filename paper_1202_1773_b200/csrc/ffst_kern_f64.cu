// double instantiation of the FFST kernels (sm_100a); n <= 2048
#include "ffst_launch.cuh"
namespace ffst { FFST_INSTANTIATE(double) }
