// common.cuh -- device-side system descriptor, grid barrier, status word.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "md.cuh"

namespace ns {

// Device status bits (ns_get_status): see include/ns.h
enum : unsigned {
  ST_SINGULAR = 1u,    // an R_jj was exactly zero (reading R15)
  ST_NONFINITE = 2u,   // a norm came out non-finite
};

// Everything a kernel needs about the system; device pointers.
struct DevSys {
  int n;          // dim
  int d;          // D + 1 coefficients
  int M;          // monomials
  int nnz;        // structural Jacobian nonzeros
  int m_max;      // longest monomial
  const int* eq_ptr;    // [n+1]
  const int* mono_ptr;  // [M+1]
  const int* var_idx;   // [sum m]
  const int* mono_dst;  // [sum m] structural entry (index into col_idx) of each occurrence
  const int* row_ptr;   // [n+1]  Jacobian pattern (row CSR)
  const int* col_idx;   // [nnz]
  const int* job_order; // [n] equations by decreasing cost (LPT)
  const double* coeff;  // [K][M]
  const double* rhs;    // [K][n][d]
};

// Sense-reversing grid barrier for a cooperative (co-resident) launch.
// bar[0] = arrival count, bar[1] = generation.
__device__ __forceinline__ void grid_sync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = bar + 1;
    const unsigned gen = *vgen;
    const unsigned nb = gridDim.x * gridDim.y * gridDim.z;
    __threadfence();
    if (atomicAdd(bar, 1u) == nb - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*vgen == gen) {
        __nanosleep(32);
      }
    }
    __threadfence();
  }
  __syncthreads();
}

}  // namespace ns
