// kernels_k4.cu -- all kernels and launchers for K = 4 limbs.
#include "impl.cuh"

template struct Impl<4>;
