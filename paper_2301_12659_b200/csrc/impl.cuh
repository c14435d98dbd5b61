// impl.cuh -- per-precision launchers (instantiated once per K in kernels_k{2,4,8}.cu).
#pragma once
#include <algorithm>
#include <cstdlib>

#include "batched.cuh"
#include "cqr.cuh"
#include "evaldiff.cuh"
#include "md.cuh"
#include "solve.cuh"
#include "system.h"
#include "wy.cuh"

using ns::DevSys;
#define CK NS_CK
#define dalloc ns_dalloc

namespace {
// device view of the system; dc = active coefficients of this step (window)
inline DevSys devsys(const ns_system* s) {
  return DevSys{s->n, s->d, s->M, s->nnz, s->m_max, s->eq_ptr, s->mono_ptr, s->var_idx, s->mono_dst,
                s->row_ptr, s->col_idx, s->job_order, s->coeff, s->rhs, s->dc, s->repeats ? 1 : 0};
}

template <int K>
ns_status launch_evaldiff(ns_system* s, const double* x, cudaStream_t st) {
  CK(cudaMemsetAsync(s->job_counter, 0, sizeof(int), st));
  CK(cudaMemsetAsync(s->prog, 0, sizeof(int) * 2 * s->M, st));
  CK(cudaMemcpyAsync(s->left, s->left_init, sizeof(int) * s->M, cudaMemcpyDeviceToDevice, st));
  DevSys ds = devsys(s);
  ns::EdJobs J{s->jobs, s->njobs, s->ser_off, s->pool, s->prog, s->prog + s->M, s->left, s->trace,
                 s->conv_terms, s->conv_mode};
  ns::evaldiff_jobs_kernel<K><<<s->grid_ed, 256, s->ed_smem, st>>>(ds, J, x, s->b, s->A, s->A0, s->job_counter);
  s->last_launches += 1;
  CK(cudaGetLastError());
  return NS_OK;
}

template <int K>
ns_status launch_a0(ns_system* s, const double* x, cudaStream_t st) {
  DevSys ds = devsys(s);
  const int blocks = std::max(1, std::min(s->sms, (s->n + 3) / 4));
  ns::a0_kernel<K><<<blocks, 128, 0, st>>>(ds, x, s->A0q);
  s->last_launches += 1;
  CK(cudaGetLastError());
  return NS_OK;
}

// WY path (wy.cuh), after the QR of A_0 alone: R and V row-major, the Gram
// blocks S_p, then T_p = S_p^{-1} and the inverses of R's diagonal blocks in one
// cooperative launch.
template <int K>
ns_status launch_wy_factors(ns_system* s, cudaStream_t st) {
  const int n = s->n, BW = s->wy_BW, P = s->wy_P;
  const long long nn = (long long)n * n;
  const int ub = (int)std::min<long long>((nn + 255) / 256, 4LL * s->sms);
  ns::wy_unpack_kernel<K><<<ub, 256, 0, st>>>(n, BW, P, s->W, s->vhead, s->R, s->Vr, s->wy_blk);
  const long long tasks = (long long)P * BW * BW;
  const int gb = (int)std::min<long long>((tasks + 7) / 8, 8LL * s->sms);
  ns::wy_gram_kernel<K><<<gb, 256, 0, st>>>(n, BW, P, s->W, s->vhead, s->beta, s->qr_owner_beta ? 1 : 0, s->wy_blk);
  CK(cudaMemsetAsync(s->bar + 4, 0, 2 * sizeof(unsigned), st));
  int nblk = 2 * P;
  const double* S = s->wy_blk;
  double *X = s->wy_X, *T1 = s->wy_T1;
  unsigned* bar2 = s->bar + 4;
  void* args[] = {&nblk, (void*)&BW, (void*)&S, &X, &T1, &bar2};
  // wym (n <= 256) runs beside eval/diff: a small cooperative grid that fits
  const int ig = s->wy ? s->sms : std::min(s->sms, 16);
  CK(cudaLaunchCooperativeKernel((const void*)ns::invert_upper_kernel<K>, dim3(ig), dim3(256), args, 0, st));
  s->last_launches += 4;
  if (s->wym) {  // Q^T = I - V (T^T V^T), row-major, for form_m
    const long long lsX = 2LL * P * BW * BW;
    const int zb = (int)std::min<long long>((nn * 8 / 32 + 7) / 8 + 1, 4LL * s->sms);
    ns::wy_z_kernel<K><<<zb, 256, 0, st>>>(n, BW, s->wy_X, lsX, s->Vr, s->Z);
    ns::wy_qt_kernel<K><<<zb, 256, 0, st>>>(n, s->Vr, s->Z, s->Qt);
    s->last_launches += 2;
  }
  CK(cudaGetLastError());
  s->qr_cached = true;
  return NS_OK;
}

// QR of A_0: from A0src (dense row-major) or, with x != nullptr, A_0 formed
// from x inside the QR kernel.
template <int K>
ns_status launch_qr(ns_system* s, const double* A0src, const double* x, cudaStream_t st) {
  // no memsets before the launch: the grid barrier is self-resetting and the
  // reflector flags carry an epoch (launch counter)
  // the epoch advances only with a launch that happened (the grid barrier's
  // base is (epoch - 1) * grid: a failed launch must not skip an epoch)
  int epoch = s->qr_epoch + 1;
  int n = s->n;
  const double* A0 = A0src;
  double *W = s->W, *vh = s->vhead, *be = s->beta, *rd = s->rdiag;
  unsigned *bar = s->bar, *stt = s->status;
  int* fl = s->qr_flags;
  DevSys ds = devsys(s);
  const double* xp = x;
  if (s->cqr_on) {
    ns::CqrShape sh{s->cqr_P, s->cqr_W, s->cqr_CPC, s->cqr_RS, (s->cqr_withM && s->use_m) ? 1 : 0};
    double* Mo = sh.withM ? s->Minv : nullptr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(s->cqr_P);
    cfg.blockDim = dim3(32 * s->cqr_W);
    cfg.dynamicSmemBytes = s->cqr_smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = s->cqr_P;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    double *R = s->R, *Qt = s->Qt;
    long long* tr = s->cqr_trace;
    if (s->cqr_E == 2)
      CK(cudaLaunchKernelEx(&cfg, ns::cluster_qr_kernel<K, 2>, ds, xp, n, A0, W, R, Qt, rd, stt, sh, tr, Mo));
    else
      CK(cudaLaunchKernelEx(&cfg, ns::cluster_qr_kernel<K, 4>, ds, xp, n, A0, W, R, Qt, rd, stt, sh, tr, Mo));
    s->last_launches += 1;
  } else {
    int ob = s->qr_owner_beta ? 1 : 0;
    int ncol = (s->wy || s->wym) ? n : 2 * n;
    int il = s->qr_interleave ? 1 : 0;
    void* args[] = {&ds, (void*)&xp, &n, (void*)&A0, &W, &vh, &be, &rd, &bar, &stt, &fl, &epoch, &ob, &ncol, &il};
    if (s->qr_crit) {
      void* cargs[] = {&ds, (void*)&xp, &n, (void*)&A0, &W, &vh, &be, &rd, &bar, &stt, &fl, &epoch, &ncol, &il};
      CK(cudaLaunchCooperativeKernel((const void*)ns::householder_qr_crit_kernel<K>, dim3(s->grid_qr),
                                     dim3(s->qr_threads), cargs, s->qr_smem_reserve, st));
    } else {
      const void* qk = s->qr_small_regs ? (const void*)ns::householder_qr_kernel<K, 1>
                                        : (const void*)ns::householder_qr_kernel<K>;
      CK(cudaLaunchCooperativeKernel(qk, dim3(s->grid_qr), dim3(s->qr_threads), args, s->qr_smem_reserve, st));
    }
    s->qr_epoch = epoch;
    if (s->wy || s->wym) {
      const ns_status r = launch_wy_factors<K>(s, st);
      if (r || s->wy) return r;
    } else {
      const long long tot = (long long)K * n * n;
      const int blocks = (int)std::min<long long>((tot + 255) / 256, 4LL * s->sms);
      ns::qr_unpack_kernel<K><<<blocks, 256, 0, st>>>(n, s->W, s->R, s->Qt);
      s->last_launches += 1;
    }
    s->last_launches += 1;
  }
  const bool m_done = s->cqr_on && s->cqr_withM && s->use_m;  // M formed inside the cluster QR
  if (!m_done) {
    const size_t inv_smem = sizeof(double) * (size_t)K * (2 * s->TB * s->TB + s->TB * s->TB / 2);
    ns::invert_tiles_kernel<K><<<s->T, 256, inv_smem, st>>>(n, s->TB, s->R, s->invR);
    s->last_launches += 1;
  }
  if (s->use_m && !m_done) {
    CK(cudaMemsetAsync(s->bar + 4, 0, 2 * sizeof(unsigned), st));
    int TB = s->TB;
    const double *R = s->R, *Qt = s->Qt, *iR = s->invR;
    double *M = s->Minv, *Z = s->Z;
    unsigned* bar2 = s->bar + 4;
    void* margs[] = {&n, &TB, (void*)&R, (void*)&Qt, (void*)&iR, &M, &Z, &bar2};
    // 8 warps per SM: the md chains are dependent DADD sequences, one warp per
    // SMSP left the FP64 pipe 90% idle (ncu, C3)
    // wym: on the QR's own SMs (freed when the QR ends), so that M forms beside the
    // still-running eval/diff instead of waiting for a whole-GPU co-resident grid
    const int fg = s->wym ? std::min(s->grid_st, std::max(1, s->grid_qr)) : s->grid_st;
    CK(cudaLaunchCooperativeKernel((const void*)ns::form_m_kernel<K>, dim3(fg), dim3(256), margs, 0, st));
    s->last_launches += 1;
  }
  CK(cudaGetLastError());
  s->qr_cached = true;
  return NS_OK;
}

template <int K>
ns_status launch_stage(ns_system* s, int k_lo, cudaStream_t st) {
  if (s->wy) {
    CK(cudaMemsetAsync(s->bar + 2, 0, 2 * sizeof(unsigned), st));
    DevSys ds = devsys(s);
    ns::WyArgs a{s->b, s->A, s->W, s->Vr, s->vhead, s->R, s->wy_X, s->bp, s->dx, s->y, s->part, s->wy_up, s->wy_u,
                 s->cmax, s->wy_BW, s->wy_P, k_lo};
    unsigned* bar = s->bar + 2;
    void* args[] = {&ds, &a, &bar};
    CK(cudaLaunchCooperativeKernel((const void*)ns::stage_wy_kernel<K>, dim3(s->grid_st), dim3(256), args, 0, st));
    s->last_launches += 1;
    return NS_OK;
  }
  const int wpb2 = s->st2_cwpb;
  const int Q = (s->n + wpb2 - 1) / wpb2;
  if (s->use_m && s->stage_split && Q <= s->grid_st2 / 2 && s->dc - k_lo >= 3) {
    // split design: critical group + right-looking bulk updates
    CK(cudaMemsetAsync(s->bar + 2, 0, 2 * sizeof(unsigned), st));
    CK(cudaMemsetAsync(s->sflags, 0, sizeof(int) * (2 * s->d + 2), st));
    DevSys ds = devsys(s);
    ns::Stage2Args a{s->b, s->A, s->Minv, s->bp, s->dx, s->pend, s->sflags, s->sflags + s->d,
                     (unsigned*)(s->sflags + 2 * s->d), Q, k_lo, s->strace, s->bpart, wpb2};  // sflags[0]: dx published counter
    unsigned* bar = s->bar + 2;
    void* args[] = {&ds, &a, &bar};
    CK(cudaLaunchCooperativeKernel((const void*)ns::stage2_kernel<K>, dim3(s->grid_st2), dim3(s->st2_threads), args,
                                   0, st));
    s->last_launches += 1;
    return NS_OK;
  }
  CK(cudaMemsetAsync(s->bar + 2, 0, 2 * sizeof(unsigned), st));
  CK(cudaMemsetAsync(s->dx, 0, sizeof(double) * (size_t)K * s->d * s->n, st));
  DevSys ds = devsys(s);
  ns::StageArgs a{s->b, s->A, s->Qt, s->R, s->invR, s->bp, s->dx, s->y, s->part, s->use_m ? s->Minv : nullptr,
                  s->cmax, s->TB, k_lo};
  unsigned* bar = s->bar + 2;
  void* args[] = {&ds, &a, &bar};
  CK(cudaLaunchCooperativeKernel((const void*)ns::stage_kernel<K>, dim3(s->grid_st), dim3(s->st_threads), args, 0, st));
  s->last_launches += 1;
  return NS_OK;
}

template <int K>
ns_status launch_residual(ns_system* s, double* x, double* res_out, cudaStream_t st) {
  {
    const int nr = s->n_sample ? s->n_sample : s->n;
    const int* rl = s->n_sample ? s->sample_rows : nullptr;
    const long long rows = (long long)s->dc * nr;
    const int blocks = (int)std::max<long long>(1, std::min<long long>((rows + 7) / 8, 8LL * s->sms));
    // NS_NO_RESIDUAL ("can be omitted"): no residual kernel, ||r|| = 0
    if (!s->no_resid) {
      ns::residual_kernel<K><<<blocks, 256, 0, st>>>(s->n, s->d, s->dc, s->k_lo, rl, nr, s->b, s->bp, s->A0, s->dx,
                                                     s->rbuf, s->knorm);
      s->last_launches += 1;
    }
    ns::knorm_kernel<K><<<s->dc, 128, 0, st>>>(s->n, s->d, s->k_lo, rl, nr, s->b, s->no_resid ? nullptr : s->rbuf,
                                               s->dx, x, s->knorm);
    s->last_launches += 1;
  }
  const long long tot = (long long)s->n * s->d;
  const int blocks = (int)std::max<long long>(1, std::min<long long>((tot + 255) / 256, 2LL * s->sms));
  ns::finalize_kernel<K><<<blocks, 256, 0, st>>>(s->n, s->d, s->dc, x, s->dx, s->knorm,
                                                 res_out ? res_out : s->res_tmp, s->status);
  s->last_launches += 1;
  CK(cudaGetLastError());
  return NS_OK;
}

template <int K>
ns_status setup_grids(ns_system* s) {
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ns::householder_qr_kernel<K>, 128, 0));
  if (occ < 1) return NS_ECUDA;
  // cooperative grids: enough warps for the 2n columns of [A0 | I], never more
  // CTAs than SMs (a grid barrier costs more with every CTA); env overrides for tuning
  // one warp per column of [A0 | I] while that fits in one CTA per SM of 4 warps;
  // larger systems use 8 warps per CTA (the column updates are throughput work)
  // 8 warps per CTA: the grid QR then holds half as many SMs (reserved, below),
  // leaving them to the concurrent eval/diff (C3: 10.25 vs 10.99 ms per step)
  // wym (A_0 alone, n <= 256): 4 warps per CTA, one column-owner warp per SMSP
  s->qr_threads = s->wym ? 128 : 256;
  if (const char* e = getenv("NS_QR_THREADS")) s->qr_threads = atoi(e) >= 256 ? 256 : 128;
  // the owner forms beta once: at 8 warps per CTA the per-consumer reciprocals
  // competed with the owner's chain for the FP64 pipes (C3 QR 7.03 -> 6.92 ms, C4 66.8 -> 63.4)
  s->qr_owner_beta = true;
  if (const char* e = getenv("NS_QR_OWNER_BETA")) s->qr_owner_beta = atoi(e) != 0;
  // large n (more than the 128-row register window): the register-light
  // variant at 2 CTAs per SM (NS_QR_SMALLREGS overrides)
  s->qr_small_regs = s->n > 128;
  // columns spread over the CTAs on the WY path (n > 256, every SM busy to the end);
  // [A0 | I] (n <= 256) keeps contiguous ownership (C3 measured 6.94 vs 7.23 ms)
  s->qr_interleave = s->wy;
  if (const char* e = getenv("NS_QR_INTERLEAVE")) s->qr_interleave = atoi(e) != 0;
  if (const char* e = getenv("NS_QR_SMALLREGS")) s->qr_small_regs = atoi(e) != 0;
  const int qcols = (s->wy || s->wym) ? s->n : 2 * s->n;  // columns of the factored matrix
  s->grid_qr = std::min(s->sms * (s->qr_small_regs ? 2 : 1),
                        std::max(1, (qcols + s->qr_threads / 32 - 1) / (s->qr_threads / 32)));
  // a dedicated CTA for the dependent reflector chain (householder_qr_crit_kernel)
  // plus the column CTAs (NS_QR_CRIT overrides): at C3 ([A0 | I], 8d) measured 9.05
  // against the grid QR's 6.86 ms (the owner warps' column updates bound the step
  // there), so it is off for n <= 256; WY path (n > 256): the critical-chain CTA is the default (C4 QR 32.0 -> 24.0 ms)
  s->qr_crit = s->wy;
  if (const char* e = getenv("NS_QR_CRIT")) s->qr_crit = atoi(e) != 0;
  if (s->qr_crit) {
    s->qr_small_regs = false;
    s->grid_qr = std::min(s->sms, 1 + (qcols - 1 + s->qr_threads / 32 - 1) / (s->qr_threads / 32));
  }
  // The QR is latency-bound and runs concurrently with eval/diff; a large
  // dynamic shared-memory request keeps eval/diff CTAs off the QR's SMs
  // (NS_QR_RESERVE=0 disables).  Default: reserve when the QR grid is small
  // relative to the GPU.
  {
    int optin = 0;
    CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, s->dev));
    bool reserve = 4 * s->grid_qr <= s->sms;
    if (const char* e = getenv("NS_QR_RESERVE")) reserve = atoi(e) != 0;
    s->qr_smem_reserve = reserve ? (size_t)optin : 0;
    if (reserve) {  // static shared memory of the crit kernel: ~1 KiB below the opt-in
      CK(cudaFuncSetAttribute(ns::householder_qr_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
      CK(cudaFuncSetAttribute(ns::householder_qr_kernel<K, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
      CK(cudaFuncSetAttribute(ns::householder_qr_crit_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              optin - 2048));
      if (s->qr_crit) s->qr_smem_reserve = (size_t)optin - 2048;
    }
  }
  // cluster QR: the whole [A0 | I] in the shared memory of one cluster of P CTAs
  {
    int optin = 0;
    CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, s->dev));
    s->cqr_on = false;
    // octo double: the trailing updates outweigh the chain on 16 SMs (C3 measured
    // slower than the grid-wide QR), so the cluster QR is for K <= 4
    bool want = s->n <= 128 && K <= 4 && !s->wy;
    if (const char* e = getenv("NS_CQR")) want = want && atoi(e) != 0;
    int Pforce = 0, RS = 8;
    if (const char* e = getenv("NS_CQR_P")) Pforce = atoi(e);
    if (const char* e = getenv("NS_CQR_RS")) RS = std::max(2, atoi(e));
    const int wmax = (K == 8) ? 8 : 16;
    for (int P : {16, 8}) {
      if (!want || s->cqr_on || (Pforce && P != Pforce)) continue;
      const int CPC = (2 * s->n + P - 1) / P;
      const int W = std::min(wmax, CPC);
      if (2 * W < CPC) continue;
      ns::CqrShape sh{P, W, CPC, RS, 1};
      size_t smem = ns::cqr_smem_bytes(s->n, K, sh);
      bool withM = smem <= (size_t)optin;
      if (const char* e = getenv("NS_CQR_M")) withM = withM && atoi(e) != 0;
      if (!withM) {
        sh.withM = 0;
        smem = ns::cqr_smem_bytes(s->n, K, sh);
      }
      if (smem > (size_t)optin) continue;
      // the QR chain is latency-bound: keep eval/diff CTAs off the cluster's SMs
      // with the full shared-memory request (NS_CQR_RESERVE=0: only what it needs)
      bool reserve = true;
      if (const char* e = getenv("NS_CQR_RESERVE")) reserve = atoi(e) != 0;
      if (reserve) smem = (size_t)optin;
      auto kern = (s->n <= 64) ? ns::cluster_qr_kernel<K, 2> : ns::cluster_qr_kernel<K, 4>;
      if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) continue;
      if (P > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
        cudaGetLastError();
        continue;
      }
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(P);
      cfg.blockDim = dim3(32 * W);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = P;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) != cudaSuccess || ncl < 1) {
        cudaGetLastError();
        continue;
      }
      s->cqr_on = true;
      s->cqr_P = P;
      s->cqr_W = W;
      s->cqr_CPC = CPC;
      s->cqr_RS = RS;
      s->cqr_E = (s->n <= 64) ? 2 : 4;
      s->cqr_smem = smem;
      s->cqr_withM = withM;
      if (getenv("NS_CQR_TRACE") && !s->cqr_trace) {
        if (cudaMalloc(&s->cqr_trace, sizeof(long long) * 8 * s->n) != cudaSuccess) s->cqr_trace = nullptr;
        else cudaMemset(s->cqr_trace, 0, sizeof(long long) * 8 * s->n);
      }
    }
  }
  {
    // co-residency bound of the grid QR at its real launch shape (threads and
    // the reserving dynamic shared memory): an override can not exceed it
    int occq = 0;
    if (s->qr_crit)
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occq, ns::householder_qr_crit_kernel<K>, s->qr_threads,
                                                       s->qr_smem_reserve));
    else if (s->qr_small_regs)
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occq, ns::householder_qr_kernel<K, 1>, s->qr_threads,
                                                       s->qr_smem_reserve));
    else
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occq, ns::householder_qr_kernel<K>, s->qr_threads,
                                                       s->qr_smem_reserve));
    if (occq < 1) return NS_ECUDA;
    if (const char* e = getenv("NS_QR_GRID")) s->grid_qr = std::max(1, atoi(e));
    s->grid_qr = std::min(s->grid_qr, s->sms * occq);
  }
  s->st_threads = 256;
  if (const char* e = getenv("NS_STAGE_THREADS")) s->st_threads = atoi(e) >= 256 ? 256 : 128;
  s->stage_split = true;
  if (const char* e = getenv("NS_CONV_TERMS")) s->conv_terms = std::max(1, atoi(e));
  if (const char* e = getenv("NS_CONV_MODE")) s->conv_mode = atoi(e);
  if (const char* e = getenv("NS_STAGE_SPLIT")) s->stage_split = atoi(e) != 0;
  {
    int occ2 = 0;
    // split stage loop: CTA size and grid (NS_STAGE2_THREADS / NS_STAGE2_GRID)
    s->st2_threads = 256;  // measured: 64 and 128 are not faster (C3 73.6 / 60.3 vs 62.3 us per stage)
    if (const char* e = getenv("NS_STAGE2_THREADS")) s->st2_threads = std::max(32, std::min(256, atoi(e))) / 32 * 32;
    // row-owning warps per critical CTA (NS_STAGE2_CW; default all of them)
    s->st2_cwpb = s->st2_threads / 32;
    if (const char* e = getenv("NS_STAGE2_CW")) s->st2_cwpb = std::max(1, std::min(s->st2_threads / 32, atoi(e)));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, ns::stage2_kernel<K>, s->st2_threads, 0));
    if (occ2 < 1) s->stage_split = false;
    s->grid_st2 = std::min(occ2 * s->sms, s->sms * std::max(1, 256 / s->st2_threads));
    if (const char* e = getenv("NS_STAGE2_GRID")) s->grid_st2 = std::max(1, std::min(s->sms * occ2, atoi(e)));
  }
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ns::stage_kernel<K>, s->st_threads, 0));
  if (occ < 1) return NS_ECUDA;
  if (s->wy || s->wym) {  // cooperative grids of one CTA per SM (256 threads)
    int o1 = 0, o2 = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, ns::stage_wy_kernel<K>, 256, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, ns::invert_upper_kernel<K>, 256, 0));
    if (o1 < 1 || o2 < 1) return NS_ECUDA;
  }
  s->grid_st = s->sms;
  {
    const size_t inv_smem = sizeof(double) * (size_t)K * (2 * s->TB * s->TB + s->TB * s->TB / 2);
    CK(cudaFuncSetAttribute(ns::invert_tiles_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)inv_smem));
  }
  if (const char* e = getenv("NS_STAGE_GRID")) s->grid_st = std::max(1, std::min(s->sms * occ, atoi(e)));
  s->ed_smem = 5 * sizeof(double) * (size_t)K * s->d;  // b accumulator, chain + x double buffers
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ns::evaldiff_jobs_kernel<K>, 256, s->ed_smem));
  if (occ < 1) return NS_ECUDA;
  s->grid_ed = std::min(s->njobs_full, occ * s->sms);
  if (const char* e = getenv("NS_ED_GRID")) s->grid_ed = std::max(1, std::min(occ * s->sms, atoi(e)));
  return NS_OK;
}

}  // namespace
namespace {

// Layout of the batched kernel for this handle (per CTA = per path in
// flight): the small, hot arrays first into shared memory, as long as the
// budget allows `ctas` CTAs per SM; the rest, the structural Jacobian A and
// the per-warp chain series in the CTA's slice of a global workspace.
template <class S, int K>
ns::BLayout batched_layout(const ns_system* s, size_t smem_cap_doubles, int threads) {
  constexpr int C = S::C;
  const size_t n = s->n, d = s->d, NW = threads / 32;
  ns::BLayout L{};
  int TB = 1;
  while (TB * 2 <= std::min<int>(32, s->n)) TB *= 2;
  L.TB = TB;
  const size_t T = (n + TB - 1) / TB, TT = (size_t)TB * TB;
  size_t sz[ns::B_NARR];
  sz[ns::B_X] = C * K * n * d;
  sz[ns::B_B] = C * K * d * n;
  sz[ns::B_DX] = C * K * d * n;
  sz[ns::B_W] = C * K * 2 * n * n;
  sz[ns::B_RI] = C * K * T * TT;
  sz[ns::B_Y] = C * K * std::max(n, TT / 2);
  sz[ns::B_VH] = C * K * n;
  sz[ns::B_BE] = K * n;
  sz[ns::B_KN] = 3 * K * d;
  const int order[ns::B_NARR] = {ns::B_VH, ns::B_BE, ns::B_KN, ns::B_Y, ns::B_X, ns::B_B, ns::B_DX, ns::B_RI, ns::B_W};
  size_t sm = 0;
  size_t g = (size_t)C * K * d * s->nnz + NW * 2 * 3 * (size_t)s->m_max * C * K * d;  // A, per-warp series x 2 eqs
  L.off_A_g = 0;
  L.off_ser_g = (size_t)C * K * d * s->nnz;
  L.in_smem = 0;
  for (int q = 0; q < ns::B_NARR; ++q) {
    const int a = order[q];
    if (sm + sz[a] <= smem_cap_doubles) {
      L.off[a] = sm;
      sm += sz[a];
      L.in_smem |= 1u << a;
    } else {
      L.off[a] = g;
      g += sz[a];
    }
  }
  L.smem_doubles = sm;
  L.gws_doubles = g;
  return L;
}

template <class S, int K, int MB>
ns_status batched_setup_t(ns_system* s) {
  int threads = 256;  // NS_BATCH_THREADS=128: 4 warps per path (more paths in flight per SM)
  if (const char* e = getenv("NS_BATCH_THREADS")) threads = atoi(e) == 128 ? 128 : 256;
  int optin = 0;
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, s->dev));
  int per_sm = 0;
  CK(cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, s->dev));
  // shared-memory budget per CTA: as many CTAs per SM as the layout allows
  // (NS_BATCH_CTAS overrides the target), each CTA's static smem and the
  // per-block reservation (1 KiB) set aside
  int target = 2;
  if (const char* e = getenv("NS_BATCH_CTAS")) target = std::max(1, atoi(e));
  const size_t cap = std::min<size_t>((size_t)optin, (size_t)per_sm / target - 2048) / sizeof(double);
  ns::BLayout L = batched_layout<S, K>(s, cap, threads);
  const size_t smem_bytes = L.smem_doubles * sizeof(double);
  if (cudaFuncSetAttribute(ns::batched_step_kernel<S, K, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem_bytes) != cudaSuccess)
    return NS_ECUDA;
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ns::batched_step_kernel<S, K, MB>, threads, smem_bytes));
  if (occ < 1) return NS_ECUDA;
  s->bl = L;
  s->b_threads = threads;
  s->batched_smem = smem_bytes;
  s->b_grid = std::min(std::max(1, s->max_batch), occ * s->sms);
  if (dalloc(&s->bws, (size_t)s->b_grid * L.gws_doubles) != cudaSuccess) return NS_ENOMEM;
  return NS_OK;
}

template <int K>
ns_status batched_impl(ns_system* s, int batch, double* x, const double* rhs, double* res, uint32_t flags,
                       cudaStream_t st) {
  (void)flags;
  DevSys ds = devsys(s);
  const int grid = std::min(batch, s->b_grid);
  long long* tr = s->btrace_on ? s->strace_b : nullptr;
  if (s->is_complex)
    ns::batched_step_kernel<ns::CplxS<K>, K, 1><<<grid, s->b_threads, s->batched_smem, st>>>(ds, batch, x, rhs, res,
                                                                                              s->bws, s->bl, tr);
  else if (s->b_minb == 2)
    ns::batched_step_kernel<ns::RealS<K>, K, 2><<<grid, s->b_threads, s->batched_smem, st>>>(ds, batch, x, rhs, res,
                                                                                              s->bws, s->bl, tr);
  else
    ns::batched_step_kernel<ns::RealS<K>, K, 1><<<grid, s->b_threads, s->batched_smem, st>>>(ds, batch, x, rhs, res,
                                                                                              s->bws, s->bl, tr);
  s->btrace_grid = grid;
  s->last_launches = 1;
  s->last_stream = st;
  CK(cudaGetLastError());
  return NS_OK;
}

}  // namespace

namespace {
template <int K>
__global__ void md_op_kernel(int op, int n, const double* a, const double* b, double* c) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    md::mdv<K> x = md::load<K>(a, n, i);
    md::mdv<K> y = (op == 4) ? md::zero<K>() : md::load<K>(b, n, i);
    md::mdv<K> r;
    switch (op) {
      case 0: r = md::add<K>(x, y); break;
      case 1: r = md::mul<K>(x, y); break;
      case 2: r = md::fma_acc<K>(md::load<K>(c, n, i), x, y); break;
      case 3: r = md::div<K>(x, y); break;
      case 4: r = md::sqrt<K>(x); break;
      default: r = md::sub<K>(x, y); break;
    }
    md::store<K>(c, n, i, r);
  }
}
}  // namespace

namespace {
// single-warp dependent chains of md ops, timed with the SM clock (latency probe)
template <int K>
__global__ void md_latency_kernel(int op, int iters, const double* in, double* out, long long* cycles) {
  md::mdv<K> a = md::load<K>(in, 4, 0), b = md::load<K>(in, 4, 1), c = md::load<K>(in, 4, 2);
  __syncwarp();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    switch (op) {
      case 0: c = md::fma_acc<K>(c, a, b); break;
      case 1: c = md::add<K>(c, a); break;
      case 2: c = md::mul<K>(c, a); break;
      case 3: c = md::recip<K>(c); break;
      default: c = md::sqrt<K>(md::absv<K>(c)); break;
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) {
    md::store<K>(out, 1, 0, c);
    cycles[0] = t1 - t0;
  }
}
}  // namespace

template <int K>
ns_status Impl<K>::latency(int op, int iters, double* cycles_per_op) {
  double* buf = nullptr;
  long long* cyc = nullptr;
  CK(cudaMalloc(&buf, sizeof(double) * (4 * K + K)));
  CK(cudaMalloc(&cyc, sizeof(long long)));
  double h[4 * K];
  for (int l = 0; l < K; ++l)
    for (int e = 0; e < 4; ++e) h[l * 4 + e] = (l == 0) ? (e == 0 ? 0.999 : (e == 1 ? 1.0001 : 0.5)) : 0.0;
  CK(cudaMemcpy(buf, h, sizeof(h), cudaMemcpyHostToDevice));
  md_latency_kernel<K><<<1, 32>>>(op, 8, buf, buf + 4 * K, cyc);  // warm-up
  md_latency_kernel<K><<<1, 32>>>(op, iters, buf, buf + 4 * K, cyc);
  long long c = 0;
  CK(cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost));
  cudaFree(buf);
  cudaFree(cyc);
  *cycles_per_op = (double)c / iters;
  return NS_OK;
}

template <int K>
ns_status Impl<K>::setup(ns_system* s) { return setup_grids<K>(s); }
template <int K>
ns_status Impl<K>::evaldiff(ns_system* s, const double* x, cudaStream_t st) { return launch_evaldiff<K>(s, x, st); }
template <int K>
ns_status Impl<K>::qr(ns_system* s, const double* A0src, const double* x, cudaStream_t st) {
  return launch_qr<K>(s, A0src, x, st);
}
template <int K>
ns_status Impl<K>::a0(ns_system* s, const double* x, cudaStream_t st) { return launch_a0<K>(s, x, st); }
template <int K>
ns_status Impl<K>::stage(ns_system* s, int k_lo, cudaStream_t st) { return launch_stage<K>(s, k_lo, st); }
template <int K>
ns_status Impl<K>::residual(ns_system* s, double* x, double* r, cudaStream_t st) {
  return launch_residual<K>(s, x, r, st);
}
template <int K>
ns_status Impl<K>::fabry(ns_system* s, const double* x, double* z, cudaStream_t st) {
  ns::fabry_kernel<K><<<(s->n + 127) / 128, 128, 0, st>>>(s->n, s->d, x, z);
  return cudaGetLastError() == cudaSuccess ? NS_OK : NS_ECUDA;
}
template <int K>
ns_status Impl<K>::batched(ns_system* s, int batch, double* x, const double* rhs, double* res, uint32_t flags,
                           cudaStream_t st) {
  return batched_impl<K>(s, batch, x, rhs, res, flags, st);
}
template <int K>
ns_status Impl<K>::batched_setup(ns_system* s) {
  // real: register cap for 2 CTAs per SM (K = 2) unless NS_BATCH_MINB=1
  s->b_minb = (K == 2) ? 2 : 1;
  if (const char* e = getenv("NS_BATCH_MINB")) s->b_minb = atoi(e) == 2 ? 2 : 1;
  if (s->is_complex) return batched_setup_t<ns::CplxS<K>, K, 1>(s);
  return s->b_minb == 2 ? batched_setup_t<ns::RealS<K>, K, 2>(s) : batched_setup_t<ns::RealS<K>, K, 1>(s);
}
template <int K>
ns_status Impl<K>::md_op(int op, int n, const double* a, const double* b, double* c, cudaStream_t st) {
  const int blocks = std::min(1024, (n + 127) / 128);
  md_op_kernel<K><<<blocks, 128, 0, st>>>(op, n, a, b, c);
  return cudaGetLastError() == cudaSuccess ? NS_OK : NS_ECUDA;
}
