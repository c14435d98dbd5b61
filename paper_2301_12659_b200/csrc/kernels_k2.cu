// kernels_k2.cu -- all kernels and launchers for K = 2 limbs.
#include "impl.cuh"

template struct Impl<2>;
