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
  int dc;         // active coefficients 0..dc-1 of this step (dc <= d; the staggered window)
  int repeats;    // some monomial repeats a variable (exponent > 1, NEXT-3): partials of one
                  // variable accumulate serially (several occurrences share a Jacobian entry)
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// relaxed (strong, no L1 invalidation) load for spin loops; an acquire fence is
// issued once after the awaited value is seen (an ld.acquire in the loop emits
// CCTL.IVALL on every iteration)
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed_s32(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ unsigned atom_add_acqrel_u32(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_u32(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Grid barrier for a cooperative (co-resident) launch on a monotonic arrival
// counter: barrier i of a launch completes when the counter reaches
// base + i * gridDim.  Each CTA adds 1 with a fire-and-forget release
// reduction and spins on an acquire load: one L2 round trip after the last
// arrival.  The counter is zeroed before the launch (base 0) or, for a kernel
// launched without a memset, advanced by a known amount per launch (base).
struct GridBarrier {
  unsigned* cnt;
  unsigned target;
  __device__ __forceinline__ GridBarrier(unsigned* c, unsigned base) : cnt(c), target(base) {}
  __device__ __forceinline__ void sync() {
    __syncthreads();
    target += gridDim.x * gridDim.y * gridDim.z;
    if (threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
      while ((int)(ld_relaxed_u32(cnt) - target) < 0) {
      }
      (void)ld_acquire_u32(cnt);  // one acquire (one L1 invalidation) once the count is seen
    }
    __syncthreads();
  }
};

// single-use form (counter zeroed before the launch, barriers counted by the caller)
__device__ __forceinline__ void grid_sync(unsigned* bar) {
  // bar[1] holds this CTA-independent barrier index; bar[0] the arrival counter
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned nb = gridDim.x * gridDim.y * gridDim.z;
    const unsigned gen = ld_acquire_u32(bar + 1);
    if (atom_add_acqrel_u32(bar, 1u) == nb - 1) {
      st_relaxed_u32(bar, 0u);
      st_release_u32(bar + 1, gen + 1);
    } else {
      while (ld_acquire_u32(bar + 1) == gen) {
      }
    }
  }
  __syncthreads();
}

}  // namespace ns
