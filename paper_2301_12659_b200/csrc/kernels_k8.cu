// kernels_k8.cu -- all kernels and launchers for K = 8 limbs.
#include "impl.cuh"

template struct Impl<8>;
