// api.cu -- the C ABI of libnewtonmd.so (include/ns.h): descriptor validation,
// workspace, launch sequence of one Newton step.  No allocation and no host
// synchronisation inside a step; everything is ordered on the caller's stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <set>
#include <vector>

#include "../../include/ns.h"
#include "system.h"
#include "common.cuh"

#define CK NS_CK
#define dalloc ns_dalloc

namespace {

int cost_of_eq(const ns_system* s, int i) {
  long long c = 0;
  for (int t = s->h_eq_ptr[i]; t < s->h_eq_ptr[i + 1]; ++t) {
    const int m = s->h_mono_ptr[t + 1] - s->h_mono_ptr[t];
    // critical path ~ (m-1) dependent products plus the cross batch
    c += (m <= 1) ? 1 : (3 * m - 5 > 0 ? 3 * m - 5 : 1);
  }
  return (int)std::min<long long>(c, 1 << 30);
}

ns_status collect_one(ns_system* s);

// FP64 flops of one md multiply-add of md.cuh (static counts; perfmodel.MD_FMA_MIX)
double md_fma_flops(int K) { return K == 2 ? 18.0 : (K == 4 ? 166.0 : 1176.0); }

// algorithmic md multiply-adds of one step on the window [k_lo, dc) (include/ns.h ns_ledger)
void ledger_counts(ns_system* s, bool qr) {
  const long long n = s->n, dc = s->dc, kl = s->k_lo, nnz = s->nnz;
  const long long conv = s->series_products * dc * (dc + 1) / 2 + s->scale_terms * dc;
  long long upd = 0;
  for (long long k = kl; k < dc; ++k) upd += nnz * (k - kl);
  const long long st = upd + (dc - kl) * (2 * n * n + n * n / 2);
  const long long qrc = qr ? 2 * n * n * n / 3 : 0;
  const long long res = nnz * (dc - kl);
  s->ledger.md_fma_convolution += conv;
  s->ledger.md_fma_qr += qrc;
  s->ledger.md_fma_stage += st;
  s->ledger.md_fma_residual += res;
  s->ledger.flops_per_md_fma = md_fma_flops(s->K);
  s->ledger.fp64_flops += md_fma_flops(s->K) * (double)(conv + qrc + st + res);
}

template <int K>
ns_status step_impl(ns_system* s, double* x, double* res_out, uint32_t flags, cudaStream_t st) {
  // Fork: eval/diff on the side stream; on the caller's stream A_0 alone
  // (a0_kernel) then the QR of A_0, concurrently.  Join before the stage loop.
  // Ledger events: e0 start | e1 end eval/diff (side) | e2 end QR | e3 join |
  // e4 end stage loop | e5 end residual.
  const bool ledger = (flags & NS_LEDGER) != 0;
  s->last_launches = 0;
  s->no_resid = (flags & NS_NO_RESIDUAL) != 0;
  cudaEvent_t* ev = nullptr;
  if (ledger) {
    if (s->ledger_count == ns_system::LRING) {  // ring full: read the oldest record (rare)
      ns_status r0 = collect_one(s);
      if (r0) return r0;
    }
    ev = s->ev[(s->ledger_head + s->ledger_count) % ns_system::LRING];
    CK(cudaEventRecord(ev[0], st));
  }
  // the QR (which forms A_0 itself) is launched first so that its co-resident
  // grid is placed before eval/diff fills the SMs
  CK(cudaEventRecord(s->ev_fork, st));
  CK(cudaStreamWaitEvent(s->side, s->ev_fork, 0));
  ns_status r;
  if (!(flags & NS_REUSE_QR)) {
    r = Impl<K>::qr(s, nullptr, x, st);
    if (r) return r;
  }
  if (ledger) CK(cudaEventRecord(ev[2], st));
  r = Impl<K>::evaldiff(s, x, s->side);
  if (r) return r;
  // sharded eval/diff (ns_comm_init): replicate every rank's rows over NVLink
  if (ns_comm_active(s)) {
    r = ns_comm_exchange(s, s->side);
    if (r) return r;
  }
  if (ledger) CK(cudaEventRecord(ev[1], s->side));
  CK(cudaEventRecord(s->ev_join, s->side));
  CK(cudaStreamWaitEvent(st, s->ev_join, 0));
  if (ledger) CK(cudaEventRecord(ev[3], st));
  r = Impl<K>::stage(s, s->k_lo, st);
  if (r) return r;
  if (ledger) CK(cudaEventRecord(ev[4], st));
  r = Impl<K>::residual(s, x, res_out, st);
  if (r) return r;
  if (ledger) {
    CK(cudaEventRecord(ev[5], st));
    s->ledger_count += 1;
    if (!(flags & NS_REUSE_QR)) s->ledger.qr_count += 1;
    ledger_counts(s, !(flags & NS_REUSE_QR));
  }
  s->last_stream = st;
  return NS_OK;
}

ns_status collect_one(ns_system* s) {
  cudaEvent_t* ev = s->ev[s->ledger_head];
  CK(cudaEventSynchronize(ev[5]));
  float conv, qr, stage, resid, total;
  CK(cudaEventElapsedTime(&conv, ev[0], ev[1]));
  CK(cudaEventElapsedTime(&qr, ev[0], ev[2]));
  CK(cudaEventElapsedTime(&stage, ev[3], ev[4]));
  CK(cudaEventElapsedTime(&resid, ev[4], ev[5]));
  CK(cudaEventElapsedTime(&total, ev[0], ev[5]));
  s->ledger.ms_convolution += conv;   // concurrent with the QR (side stream)
  s->ledger.ms_qr += qr;
  s->ledger.ms_stage += stage;
  s->ledger.ms_residual += resid;
  s->ledger.ms_total += total;
  s->ledger.steps += 1;
  s->ledger_head = (s->ledger_head + 1) % ns_system::LRING;
  s->ledger_count -= 1;
  return NS_OK;
}

ns_status collect_ledger(ns_system* s) {
  while (s->ledger_count > 0) {
    ns_status r = collect_one(s);
    if (r) return r;
  }
  return NS_OK;
}

void free_all(ns_system* s) {
  void* ptrs[] = {s->eq_ptr, s->mono_ptr, s->var_idx, s->mono_dst, s->row_ptr, s->col_idx, s->job_order,
                  s->coeff, s->rhs, s->b, s->A, s->A0, s->W, s->vhead, s->beta, s->rdiag, s->R, s->Qt,
                  s->invR, s->bp, s->dx, s->y, s->part, s->Minv, s->Z, s->pend, s->sflags, s->rbuf, s->knorm, s->res_tmp, s->ws, s->job_counter,
                  s->bar, s->status, s->bws, s->A0q, s->qr_flags, s->jobs, s->ser_off, s->pool, s->prog, s->left,
                  s->left_init, s->trace, s->strace, s->sample_rows, s->bpart, s->strace_b,
                  s->wy_blk, s->wy_X, s->wy_T1, s->wy_up, s->wy_u, s->Vr};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  for (auto& row : s->ev)
    for (auto& e : row)
      if (e) cudaEventDestroy(e);
  if (s->ev_fork) cudaEventDestroy(s->ev_fork);
  if (s->ev_join) cudaEventDestroy(s->ev_join);
  if (s->side) cudaStreamDestroy(s->side);
}

}  // namespace

// Job list of the eval/diff job queue for the equations [eq_lo, eq_hi): chains
// longest first (LPT), cross products by the layer their inputs appear at,
// equations by their longest monomial.  ser_off / left cover all monomials.
void ns_build_jobs(const ns_system* s, int eq_lo, int eq_hi, std::vector<int4>& jobs, std::vector<long long>& ser_off,
                std::vector<int>& left, long long& pool_series) {
  const int M = s->M;
  std::vector<int4> chains, cross, eqs;
  ser_off.assign(M, 0);
  left.assign(M, 0);
  pool_series = 0;
  auto prod = [](int m) { return m <= 1 ? 0 : (m == 2 ? 1 : 3 * m - 5); };
  for (int t = 0; t < M; ++t) {
    const int m = s->h_mono_ptr[t + 1] - s->h_mono_ptr[t];
    ser_off[t] = pool_series;
    pool_series += prod(m);
    left[t] = (m <= 1) ? 0 : (m == 2 ? 1 : m);
  }
  for (int i = eq_lo; i < eq_hi; ++i) {
    int mm = 0;
    for (int t = s->h_eq_ptr[i]; t < s->h_eq_ptr[i + 1]; ++t) {
      const int m = s->h_mono_ptr[t + 1] - s->h_mono_ptr[t];
      mm = std::max(mm, m);
      if (m >= 2) chains.push_back(make_int4(0, t, m - 1, 0));
      if (m >= 3) chains.push_back(make_int4(1, t, m - 2, 0));
      for (int j = 2; j <= m - 1; ++j) cross.push_back(make_int4(2, t, j, std::max(j - 2, m - j - 1)));
    }
    eqs.push_back(make_int4(3, i, 0, mm));
  }
  std::stable_sort(chains.begin(), chains.end(), [](int4 a, int4 b) { return a.z > b.z; });
  std::stable_sort(cross.begin(), cross.end(), [](int4 a, int4 b) { return a.w < b.w; });
  std::stable_sort(eqs.begin(), eqs.end(), [](int4 a, int4 b) { return a.w < b.w; });
  jobs = chains;
  jobs.insert(jobs.end(), cross.begin(), cross.end());
  jobs.insert(jobs.end(), eqs.begin(), eqs.end());
}

namespace {

}  // namespace


extern "C" {

const char* ns_strerror(ns_status s) {
  switch (s) {
    case NS_OK: return "ok";
    case NS_EINVAL: return "invalid argument";
    case NS_EPREC: return "precision not in {2,4,8} or not the handle's";
    case NS_EDIM: return "dim/degree/batch mismatch";
    case NS_EMONO: return "malformed monomial list";
    case NS_ESINGULAR: return "zero diagonal entry in R";
    case NS_ENONFINITE: return "non-finite norm";
    case NS_ENOMEM: return "device allocation failed";
    case NS_ECUDA: return "CUDA runtime error";
    case NS_ENCCL: return "NCCL error";
    case NS_ESTATE: return "no cached QR factorisation";
  }
  return "unknown status";
}

const char* ns_build_info(void) {
  return "libnewtonmd sm_100a; md K in {2,4,8}; FP64 CUDA cores; arxiv 2301.12659 Newton step";
}

ns_status ns_system_create(const ns_system_desc* desc, int cuda_device, ns_system** out) {
  if (!out) return NS_EINVAL;
  *out = nullptr;
  if (!desc || !desc->eq_ptr || !desc->mono_ptr || !desc->var_idx || !desc->rhs) return NS_EINVAL;
  const int K = desc->precision;
  if (K != 2 && K != 4 && K != 8) return NS_EPREC;
  const int n = desc->dim, D = desc->degree, M = desc->n_monomials;
  if (n < 1 || D < 0 || M < 1 || desc->max_batch < 0) return NS_EDIM;
  if (desc->eq_ptr[0] != 0 || desc->eq_ptr[n] != M) return NS_EMONO;
  for (int i = 0; i < n; ++i)
    if (desc->eq_ptr[i + 1] < desc->eq_ptr[i]) return NS_EMONO;
  if (desc->mono_ptr[0] != 0) return NS_EMONO;
  int m_max = 1;
  for (int t = 0; t < M; ++t) {
    const int a = desc->mono_ptr[t], b = desc->mono_ptr[t + 1];
    if (b <= a) return NS_EMONO;
    m_max = std::max(m_max, b - a);
    for (int q = a; q < b; ++q) {
      if (desc->var_idx[q] < 0 || desc->var_idx[q] >= n) return NS_EMONO;
      if (q > a && desc->var_idx[q] < desc->var_idx[q - 1]) return NS_EMONO;  // equal: exponent > 1
    }
  }
  if (desc->is_complex != 0 && desc->is_complex != 1) return NS_EINVAL;
  ns_system* s = new (std::nothrow) ns_system();
  if (!s) return NS_ENOMEM;
  s->is_complex = desc->is_complex == 1;
  for (int t = 0; t < M; ++t)
    for (int q = desc->mono_ptr[t] + 1; q < desc->mono_ptr[t + 1]; ++q)
      if (desc->var_idx[q] == desc->var_idx[q - 1]) s->repeats = true;
  s->dev = cuda_device;
  s->n = n;
  s->D = D;
  s->d = D + 1;
  s->dc = s->d;
  s->K = K;
  s->M = M;
  s->m_max = m_max;
  s->max_batch = std::max(1, desc->max_batch);
  for (int t = 0; t < M; ++t) {
    const int m = desc->mono_ptr[t + 1] - desc->mono_ptr[t];
    s->series_products += (m <= 1) ? 0 : (m == 2 ? 1 : 3 * m - 5);
    s->scale_terms += 1 + m;
  }
  s->TB = 32;
  s->T = (n + s->TB - 1) / s->TB;
  // blocked WY solve for large n (wy.cuh): Q^T is not formed (NS_WY=0/1 overrides)
  s->wy = n > 256;
  if (const char* e = getenv("NS_WY")) s->wy = atoi(e) != 0;
  if (const char* e = getenv("NS_WY_BW")) {  // block width: a power of two in [2, 256]
    const int bw = atoi(e);
    if (bw >= 2 && bw <= 256 && (bw & (bw - 1)) == 0) s->wy_BW = bw;
  }
  // n <= 256 (no cluster QR: see setup): QR of A_0 alone and Q^T from one WY block (NS_WYM)
  s->wym = false;  // opt-in: measured slower at C3 (10.96 vs 9.24 ms)
  if (const char* e = getenv("NS_WYM")) s->wym = !s->wy && n <= 256 && atoi(e) != 0;
  if (s->wym) {
    s->wy_BW = 2;
    while (s->wy_BW < n) s->wy_BW *= 2;
  }
  s->wy_P = (n + s->wy_BW - 1) / s->wy_BW;
  const int L = desc->mono_ptr[M];
  s->h_eq_ptr.assign(desc->eq_ptr, desc->eq_ptr + n + 1);
  s->h_mono_ptr.assign(desc->mono_ptr, desc->mono_ptr + M + 1);
  s->h_var_idx.assign(desc->var_idx, desc->var_idx + L);
  // Jacobian pattern: row i = sorted union of the variables of eq i
  s->h_row_ptr.assign(n + 1, 0);
  s->h_mono_dst.assign(L, 0);
  for (int i = 0; i < n; ++i) {
    std::set<int> vs;
    for (int t = s->h_eq_ptr[i]; t < s->h_eq_ptr[i + 1]; ++t)
      for (int q = s->h_mono_ptr[t]; q < s->h_mono_ptr[t + 1]; ++q) vs.insert(s->h_var_idx[q]);
    const int base = (int)s->h_col_idx.size();
    s->h_row_ptr[i] = base;
    std::vector<int> cols(vs.begin(), vs.end());
    s->h_col_idx.insert(s->h_col_idx.end(), cols.begin(), cols.end());
    for (int t = s->h_eq_ptr[i]; t < s->h_eq_ptr[i + 1]; ++t)
      for (int q = s->h_mono_ptr[t]; q < s->h_mono_ptr[t + 1]; ++q)
        s->h_mono_dst[q] = base + (int)(std::lower_bound(cols.begin(), cols.end(), s->h_var_idx[q]) - cols.begin());
  }
  s->h_row_ptr[n] = (int)s->h_col_idx.size();
  s->nnz = s->h_row_ptr[n];
  // LPT order: most expensive equations first
  s->h_job_order.resize(n);
  for (int i = 0; i < n; ++i) s->h_job_order[i] = i;
  std::vector<int> cost(n);
  for (int i = 0; i < n; ++i) cost[i] = cost_of_eq(s, i);
  std::stable_sort(s->h_job_order.begin(), s->h_job_order.end(),
                   [&](int a, int b) { return cost[a] > cost[b]; });

  // eval/diff job queue (see evaldiff.cuh)
  std::vector<int4> jobs;
  std::vector<long long> ser_off;
  std::vector<int> left;
  long long pool_series = 0;
  ns_build_jobs(s, 0, n, jobs, ser_off, left, pool_series);
  s->njobs = (int)jobs.size();
  s->njobs_full = s->njobs;

  ns_status st = NS_OK;
  auto fail = [&](ns_status e) {
    free_all(s);
    delete s;
    return e;
  };
  if (cudaSetDevice(cuda_device) != cudaSuccess) return fail(NS_ECUDA);
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, cuda_device) != cudaSuccess) return fail(NS_ECUDA);
  s->sms = prop.multiProcessorCount;
  const size_t d = s->d, nn = (size_t)n * n;
  bool ok = true;
  ok &= dalloc(&s->eq_ptr, n + 1) == cudaSuccess;
  ok &= dalloc(&s->mono_ptr, M + 1) == cudaSuccess;
  ok &= dalloc(&s->var_idx, L) == cudaSuccess;
  ok &= dalloc(&s->mono_dst, L) == cudaSuccess;
  ok &= dalloc(&s->row_ptr, n + 1) == cudaSuccess;
  ok &= dalloc(&s->col_idx, s->nnz) == cudaSuccess;
  ok &= dalloc(&s->job_order, n) == cudaSuccess;
  const size_t Cc = s->is_complex ? 2 : 1;
  ok &= dalloc(&s->coeff, Cc * K * M) == cudaSuccess;
  ok &= dalloc(&s->rhs, Cc * K * n * d) == cudaSuccess;
  ok &= dalloc(&s->b, (size_t)K * d * n) == cudaSuccess;
  ok &= dalloc(&s->A, (size_t)K * d * s->nnz) == cudaSuccess;
  ok &= dalloc(&s->A0, (size_t)K * nn) == cudaSuccess;
  ok &= dalloc(&s->A0q, (size_t)K * nn) == cudaSuccess;
  ok &= dalloc(&s->qr_flags, 3 * (size_t)n) == cudaSuccess;  // A, B, U flags (epoch valued)
  ok &= cudaMemset(s->qr_flags, 0, sizeof(int) * 3 * n) == cudaSuccess;
  ok &= dalloc(&s->W, (size_t)K * 2 * nn) == cudaSuccess;
  ok &= dalloc(&s->vhead, (size_t)K * n) == cudaSuccess;
  ok &= dalloc(&s->beta, (size_t)K * n) == cudaSuccess;
  ok &= dalloc(&s->rdiag, (size_t)K * n) == cudaSuccess;
  ok &= dalloc(&s->R, (size_t)K * nn) == cudaSuccess;
  ok &= dalloc(&s->Qt, (size_t)K * nn) == cudaSuccess;
  ok &= dalloc(&s->invR, (size_t)K * s->T * s->TB * s->TB) == cudaSuccess;
  ok &= dalloc(&s->bp, (size_t)K * d * n) == cudaSuccess;
  ok &= dalloc(&s->dx, (size_t)K * d * n) == cudaSuccess;
  ok &= dalloc(&s->y, (size_t)K * n) == cudaSuccess;
  ok &= dalloc(&s->Minv, (size_t)K * nn) == cudaSuccess;
  ok &= dalloc(&s->pend, (size_t)K * d * n) == cudaSuccess;
  ok &= dalloc(&s->bpart, (size_t)std::max<long long>(1, (long long)d - 2) * n * K * 32) == cudaSuccess;  // bulk lane partials
  ok &= dalloc(&s->sflags, 2 * d + 2) == cudaSuccess;
  ok &= dalloc(&s->Z, (size_t)K * nn) == cudaSuccess;
  {
    int maxlen = 1;
    for (int i = 0; i < n; ++i) maxlen = std::max(maxlen, s->h_row_ptr[i + 1] - s->h_row_ptr[i]);
    s->cmax = std::max(1, (std::max(1, (int)d - 1) * maxlen + 63) / 64);  // ns::UCH = 64
    ok &= dalloc(&s->part, (size_t)K * n * s->cmax) == cudaSuccess;
  }
  if (s->wy || s->wym) {
    ok &= dalloc(&s->Vr, (size_t)K * nn) == cudaSuccess;
    const size_t nb = (size_t)K * 2 * s->wy_P * s->wy_BW * s->wy_BW;
    ok &= dalloc(&s->wy_blk, nb) == cudaSuccess;
    ok &= dalloc(&s->wy_X, nb) == cudaSuccess;
    ok &= dalloc(&s->wy_T1, nb) == cudaSuccess;
    ok &= dalloc(&s->wy_up, (size_t)K * s->wy_BW) == cudaSuccess;
    ok &= dalloc(&s->wy_u, (size_t)K * s->wy_BW) == cudaSuccess;
  }
  ok &= dalloc(&s->rbuf, (size_t)K * d * n) == cudaSuccess;
  ok &= dalloc(&s->knorm, (size_t)4 * K * d) == cudaSuccess;  // |b_k|, |r_k|, |dx_k|, |x_k|
  ok &= dalloc(&s->res_tmp, (size_t)K * 3) == cudaSuccess;
  ok &= dalloc(&s->job_counter, 1) == cudaSuccess;
  ok &= dalloc(&s->bar, 8) == cudaSuccess;
  ok &= dalloc(&s->status, 1) == cudaSuccess;
  if (!ok) return fail(NS_ENOMEM);
  switch (K) {
    case 2: st = Impl<2>::setup(s); if (!st) st = Impl<2>::batched_setup(s); break;
    case 4: st = Impl<4>::setup(s); if (!st) st = Impl<4>::batched_setup(s); break;
    default: st = Impl<8>::setup(s); if (!st) st = Impl<8>::batched_setup(s); break;
  }
  if (st) return fail(st);
  ok = true;
  ok &= dalloc(&s->jobs, jobs.size()) == cudaSuccess;
  ok &= dalloc(&s->ser_off, M) == cudaSuccess;
  ok &= dalloc(&s->pool, (size_t)std::max<long long>(1, pool_series) * K * d) == cudaSuccess;
  ok &= dalloc(&s->prog, 2 * (size_t)M) == cudaSuccess;
  ok &= dalloc(&s->left, M) == cudaSuccess;
  ok &= dalloc(&s->left_init, M) == cudaSuccess;
  if (const char* e = getenv("NS_STAGE_TRACE"))
    if (atoi(e)) ok &= dalloc(&s->strace, (size_t)5 * s->d) == cudaSuccess;
  if (const char* e = getenv("NS_BATCH_TRACE"))
    if (atoi(e)) {
      s->btrace_on = true;
      ok &= dalloc(&s->strace_b, (size_t)8 * 4 * s->sms * 4) == cudaSuccess;  // up to 16 CTAs per SM
    }
  if (const char* e = getenv("NS_TRACE"))
    if (atoi(e)) ok &= dalloc(&s->trace, 3 * jobs.size() + 6 * 256) == cudaSuccess;
  if (!ok) return fail(NS_ENOMEM);
  ok &= cudaMemcpy(s->jobs, jobs.data(), sizeof(int4) * jobs.size(), cudaMemcpyHostToDevice) == cudaSuccess;
  ok &= cudaMemcpy(s->ser_off, ser_off.data(), sizeof(long long) * M, cudaMemcpyHostToDevice) == cudaSuccess;
  ok &= cudaMemcpy(s->left_init, left.data(), sizeof(int) * M, cudaMemcpyHostToDevice) == cudaSuccess;
  if (!ok) return fail(NS_ECUDA);
  // upload
  std::vector<double> coeff(Cc * K * M, 0.0);
  if (desc->coeff) std::memcpy(coeff.data(), desc->coeff, sizeof(double) * Cc * K * M);
  else
    for (int t = 0; t < M; ++t) coeff[t] = 1.0;
  ok = true;
  ok &= cudaMemcpy(s->eq_ptr, s->h_eq_ptr.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice) == cudaSuccess;
  ok &= cudaMemcpy(s->mono_ptr, s->h_mono_ptr.data(), sizeof(int) * (M + 1), cudaMemcpyHostToDevice) == cudaSuccess;
  ok &= cudaMemcpy(s->var_idx, s->h_var_idx.data(), sizeof(int) * L, cudaMemcpyHostToDevice) == cudaSuccess;
  ok &= cudaMemcpy(s->mono_dst, s->h_mono_dst.data(), sizeof(int) * L, cudaMemcpyHostToDevice) == cudaSuccess;
  ok &= cudaMemcpy(s->row_ptr, s->h_row_ptr.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice) == cudaSuccess;
  ok &= cudaMemcpy(s->col_idx, s->h_col_idx.data(), sizeof(int) * s->nnz, cudaMemcpyHostToDevice) == cudaSuccess;
  ok &= cudaMemcpy(s->job_order, s->h_job_order.data(), sizeof(int) * n, cudaMemcpyHostToDevice) == cudaSuccess;
  ok &= cudaMemcpy(s->coeff, coeff.data(), sizeof(double) * Cc * K * M, cudaMemcpyHostToDevice) == cudaSuccess;
  ok &= cudaMemcpy(s->rhs, desc->rhs, sizeof(double) * Cc * K * n * d, cudaMemcpyHostToDevice) == cudaSuccess;
  ok &= cudaMemset(s->status, 0, sizeof(unsigned)) == cudaSuccess;
  ok &= cudaMemset(s->bar, 0, 8 * sizeof(unsigned)) == cudaSuccess;
  for (auto& row : s->ev)
    for (auto& e : row) ok &= cudaEventCreate(&e) == cudaSuccess;
  ok &= cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming) == cudaSuccess;
  ok &= cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming) == cudaSuccess;
  ok &= cudaStreamCreateWithFlags(&s->side, cudaStreamNonBlocking) == cudaSuccess;
  if (!ok) return fail(NS_ECUDA);
  *out = s;
  return NS_OK;
}

void ns_system_destroy(ns_system* s) {
  if (!s) return;
  cudaSetDevice(s->dev);
  cudaDeviceSynchronize();
  ns_comm_free(s);
  free_all(s);
  if (s->cqr_trace) cudaFree(s->cqr_trace);
  delete s;
}

ns_status ns_newton_series_step(ns_system* s, int precision, int dim, int degree, double* x,
                                double* res_out, uint32_t flags, void* stream) {
  if (!s || !x) return NS_EINVAL;
  if (precision != s->K) return NS_EPREC;
  if (dim != s->n || degree != s->D) return NS_EDIM;
  if (s->is_complex) {  // NEXT-2: the batched kernel on one path (include/ns.h)
    if (flags) return NS_EINVAL;
    if (s->k_lo != 0 || s->dc != s->d) return NS_ESTATE;
    switch (s->K) {
      case 2: return Impl<2>::batched(s, 1, x, nullptr, res_out, 0, (cudaStream_t)stream);
      case 4: return Impl<4>::batched(s, 1, x, nullptr, res_out, 0, (cudaStream_t)stream);
      default: return Impl<8>::batched(s, 1, x, nullptr, res_out, 0, (cudaStream_t)stream);
    }
  }
  if (flags & ~(NS_REUSE_QR | NS_NO_RESIDUAL | NS_LEDGER | NS_TILED_BS)) return NS_EINVAL;
  if ((flags & NS_REUSE_QR) && !s->qr_cached) return NS_ESTATE;
  // M = R^{-1} Q^T (~n^3/2 md-FMA once per QR) saves 2T barriers per stage.
  // With NS_REUSE_QR the cached factorisation keeps the form it was made in.
  if (!(flags & NS_REUSE_QR)) s->use_m = !(flags & NS_TILED_BS);
  cudaStream_t st = (cudaStream_t)stream;
  switch (s->K) {
    case 2: return step_impl<2>(s, x, res_out, flags, st);
    case 4: return step_impl<4>(s, x, res_out, flags, st);
    default: return step_impl<8>(s, x, res_out, flags, st);
  }
}

ns_status ns_newton_series_step_batched(ns_system* s, int precision, int dim, int degree, int batch,
                                        double* x, const double* rhs, double* res, uint32_t flags,
                                        void* stream) {
  if (!s || !x) return NS_EINVAL;
  if (precision != s->K) return NS_EPREC;
  if (dim != s->n || degree != s->D || batch < 0 || batch > s->max_batch) return NS_EDIM;
  if (flags) return NS_EINVAL;
  if (s->k_lo != 0 || s->dc != s->d) return NS_ESTATE;  // the batched kernel runs the full window
  if (batch == 0) return NS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  switch (s->K) {
    case 2: return Impl<2>::batched(s, batch, x, rhs, res, flags, st);
    case 4: return Impl<4>::batched(s, batch, x, rhs, res, flags, st);
    default: return Impl<8>::batched(s, batch, x, rhs, res, flags, st);
  }
}

ns_status ns_eval_diff(ns_system* s, const double* x, double* b, double* A, double* A0, void* stream) {
  if (!s || !x) return NS_EINVAL;
  if (s->is_complex) return NS_EINVAL;  // complex: the batched kernel path only (include/ns.h)
  cudaStream_t st = (cudaStream_t)stream;
  ns_status r;
  s->last_launches = 0;
  switch (s->K) {
    case 2: r = Impl<2>::evaldiff(s, x, st); break;
    case 4: r = Impl<4>::evaldiff(s, x, st); break;
    default: r = Impl<8>::evaldiff(s, x, st); break;
  }
  if (r) return r;
  const size_t K = s->K, d = s->d, n = s->n;
  if (b) CK(cudaMemcpyAsync(b, s->b, sizeof(double) * K * d * n, cudaMemcpyDeviceToDevice, st));
  if (A) CK(cudaMemcpyAsync(A, s->A, sizeof(double) * K * d * s->nnz, cudaMemcpyDeviceToDevice, st));
  if (A0) CK(cudaMemcpyAsync(A0, s->A0, sizeof(double) * K * n * n, cudaMemcpyDeviceToDevice, st));
  s->last_stream = st;
  return NS_OK;
}

int32_t ns_nnz(const ns_system* s) { return s ? s->nnz : -1; }

int32_t ns_get_qr_trace(ns_system* s, int64_t* host, int32_t capacity_steps) {
  if (!s || !s->cqr_trace) return -1;
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  const int ns_ = std::min(capacity_steps, s->n);
  if (host && ns_ > 0 &&
      cudaMemcpy(host, s->cqr_trace, sizeof(long long) * 8 * ns_, cudaMemcpyDeviceToHost) != cudaSuccess)
    return -1;
  return ns_;
}

int32_t ns_get_batch_trace(ns_system* s, int64_t* host, int32_t capacity_ctas) {
  if (!s || !s->strace_b || !host) return -1;
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  const int g = std::min(capacity_ctas, s->btrace_grid);
  if (g > 0 && cudaMemcpy(host, s->strace_b, sizeof(long long) * 8 * g, cudaMemcpyDeviceToHost) != cudaSuccess)
    return -1;
  return g;
}

int32_t ns_get_stage_trace(ns_system* s, int64_t* host) {
  if (!s || !s->strace || !host) return -1;
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  if (cudaMemcpy(host, s->strace, sizeof(long long) * 5 * s->d, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  return s->d;
}

int32_t ns_get_trace(ns_system* s, int64_t* host, int32_t capacity_jobs, int32_t* jobs_out) {
  if (!s || !s->trace) return -1;
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  const int nj = std::min(capacity_jobs, s->njobs);
  if (host && nj > 0) {
    if (cudaMemcpy(host, s->trace, sizeof(long long) * 3 * nj, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    if (capacity_jobs >= s->njobs + 512)  // step stamps of job 0 after the job records
      if (cudaMemcpy(host + 3 * nj, s->trace + 3 * s->njobs, sizeof(long long) * 6 * 256, cudaMemcpyDeviceToHost) !=
          cudaSuccess)
        return -1;
  }
  if (jobs_out) {
    std::vector<int4> jb(nj);
    if (cudaMemcpy(jb.data(), s->jobs, sizeof(int4) * nj, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    for (int i = 0; i < nj; ++i) {
      jobs_out[4 * i] = jb[i].x;
      jobs_out[4 * i + 1] = jb[i].y;
      jobs_out[4 * i + 2] = jb[i].z;
      jobs_out[4 * i + 3] = jb[i].w;
    }
  }
  return nj;
}

ns_status ns_set_partition(ns_system* s, int eq_lo, int eq_hi) {
  if (!s || eq_lo < 0 || eq_hi > s->n || eq_lo >= eq_hi) return NS_EINVAL;
  if (s->is_complex) return NS_EINVAL;  // complex: the batched kernel path only (include/ns.h)
  std::vector<int4> jobs;
  std::vector<long long> ser_off;
  std::vector<int> left;
  long long pool_series = 0;
  ns_build_jobs(s, eq_lo, eq_hi, jobs, ser_off, left, pool_series);
  CK(cudaSetDevice(s->dev));
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(s->jobs, jobs.data(), sizeof(int4) * jobs.size(), cudaMemcpyHostToDevice));
  s->njobs = (int)jobs.size();
  s->eq_lo = eq_lo;
  s->eq_hi = eq_hi;
  return NS_OK;
}

ns_status ns_newton_series_step_from(ns_system* s, int precision, int dim, int degree, double* x, const double* b,
                                     const double* A, const double* A0, double* res_out, uint32_t flags,
                                     void* stream) {
  if (!s || !x || !b || !A || !A0) return NS_EINVAL;
  if (s->is_complex) return NS_EINVAL;  // complex: the batched kernel path only (include/ns.h)
  if (precision != s->K) return NS_EPREC;
  if (dim != s->n || degree != s->D) return NS_EDIM;
  if (flags & ~(NS_REUSE_QR | NS_NO_RESIDUAL | NS_LEDGER | NS_TILED_BS)) return NS_EINVAL;
  if ((flags & NS_REUSE_QR) && !s->qr_cached) return NS_ESTATE;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t K = s->K, d = s->d, n = s->n;
  s->last_launches = 0;
  s->no_resid = (flags & NS_NO_RESIDUAL) != 0;
  CK(cudaMemcpyAsync(s->b, b, sizeof(double) * K * d * n, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(s->A, A, sizeof(double) * K * d * s->nnz, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(s->A0, A0, sizeof(double) * K * n * n, cudaMemcpyDeviceToDevice, st));
  if (!(flags & NS_REUSE_QR)) s->use_m = !(flags & NS_TILED_BS);
  ns_status r = NS_OK;
  switch (s->K) {
    case 2:
      if (!(flags & NS_REUSE_QR)) r = Impl<2>::qr(s, s->A0, nullptr, st);
      if (!r) r = Impl<2>::stage(s, s->k_lo, st);
      if (!r) r = Impl<2>::residual(s, x, res_out, st);
      break;
    case 4:
      if (!(flags & NS_REUSE_QR)) r = Impl<4>::qr(s, s->A0, nullptr, st);
      if (!r) r = Impl<4>::stage(s, s->k_lo, st);
      if (!r) r = Impl<4>::residual(s, x, res_out, st);
      break;
    default:
      if (!(flags & NS_REUSE_QR)) r = Impl<8>::qr(s, s->A0, nullptr, st);
      if (!r) r = Impl<8>::stage(s, s->k_lo, st);
      if (!r) r = Impl<8>::residual(s, x, res_out, st);
      break;
  }
  s->last_stream = st;
  return r;
}

ns_status ns_set_window(ns_system* s, int k_lo, int dc) {
  if (!s || k_lo < 0 || dc > s->d || k_lo >= dc) return NS_EINVAL;
  if (s->is_complex) return NS_EINVAL;  // complex: the batched kernel path only (include/ns.h)
  s->k_lo = k_lo;
  s->dc = dc;
  return NS_OK;
}

ns_status ns_set_residual_sample(ns_system* s, const int32_t* rows, int count) {
  if (!s || count < 0 || count > s->n || (count > 0 && !rows)) return NS_EINVAL;
  if (s->is_complex) return NS_EINVAL;  // complex: the batched kernel path only (include/ns.h)
  if (count == 0) {
    s->n_sample = 0;
    return NS_OK;
  }
  std::vector<char> seen(s->n, 0);
  for (int t = 0; t < count; ++t) {
    if (rows[t] < 0 || rows[t] >= s->n || seen[rows[t]]) return NS_EINVAL;
    seen[rows[t]] = 1;
  }
  CK(cudaSetDevice(s->dev));
  if (!s->sample_rows && dalloc(&s->sample_rows, (size_t)s->n) != cudaSuccess) return NS_ENOMEM;
  // synchronous upload: steps already queued keep their sample (host-side state)
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(s->sample_rows, rows, sizeof(int32_t) * count, cudaMemcpyHostToDevice));
  s->n_sample = count;
  return NS_OK;
}

ns_status ns_fabry_ratio(ns_system* s, const double* x, double* z, void* stream) {
  if (!s || !x || !z || s->d < 2) return NS_EINVAL;
  if (s->is_complex) return NS_EINVAL;  // complex: the batched kernel path only (include/ns.h)
  cudaStream_t st = (cudaStream_t)stream;
  switch (s->K) {
    case 2: return Impl<2>::fabry(s, x, z, st);
    case 4: return Impl<4>::fabry(s, x, z, st);
    default: return Impl<8>::fabry(s, x, z, st);
  }
}

ns_status ns_get_stage_norms(ns_system* s, double* out) {
  if (!s || !out) return NS_EINVAL;
  CK(cudaSetDevice(s->dev));
  if (s->last_stream) CK(cudaStreamSynchronize(s->last_stream));
  else CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(out, s->knorm, sizeof(double) * 4 * s->K * s->d, cudaMemcpyDeviceToHost));
  return NS_OK;
}

// Staggered Newton driver (include/ns.h).  Host loop:
// one windowed step per iteration, then the per-stage norms decide the
// retired stages (reading R34) and the next order (Eq.(10)).
ns_status ns_run_newton(ns_system* s, int precision, int dim, int degree, double* x, int max_iter, double eps,
                        uint32_t flags, void* stream, ns_iter_log* log, ns_run_info* info) {
  if (!s || !x || max_iter < 0) return NS_EINVAL;
  if (s->is_complex) return NS_EINVAL;  // complex: the batched kernel path only (include/ns.h)
  if (precision != s->K) return NS_EPREC;
  if (dim != s->n || degree != s->D) return NS_EDIM;
  if (flags & ~(NS_QR_ONCE | NS_NO_STAGGER | NS_LEDGER | NS_TILED_BS | NS_NO_RESIDUAL)) return NS_EINVAL;
  CK(cudaSetDevice(s->dev));
  cudaStream_t st = (cudaStream_t)stream;
  const int K = s->K, d = s->d;
  if (!(eps > 0.0)) eps = 1e3 * std::ldexp(1.0, K == 2 ? -104 : (K == 4 ? -210 : -423));
  const double sq = std::ldexp(1.0, K == 2 ? -52 : (K == 4 ? -105 : -211));  // sqrt(eps_p)
  std::vector<double> kn((size_t)4 * K * d), prev(d, HUGE_VAL);  // prev: last ||dx_k|| while active
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  int k_lo = 0, dc = (flags & NS_NO_STAGGER) ? d : 1, qr_count = 0, it = 0;
  bool converged = false;
  ns_status r = NS_OK;
  for (it = 1; it <= max_iter; ++it) {
    s->k_lo = k_lo;
    s->dc = dc;
    const bool refactor = qr_count == 0 || (k_lo == 0 && !(flags & NS_QR_ONCE));
    uint32_t sf = (flags & (NS_LEDGER | NS_TILED_BS | NS_NO_RESIDUAL)) | (refactor ? 0u : NS_REUSE_QR);
    if (!refactor) sf &= ~NS_TILED_BS;  // the cached factorisation keeps its form
    else s->use_m = !(flags & NS_TILED_BS);
    if ((r = (cudaEventRecord(e0, st) == cudaSuccess) ? NS_OK : NS_ECUDA)) break;
    switch (K) {
      case 2: r = step_impl<2>(s, x, nullptr, sf, st); break;
      case 4: r = step_impl<4>(s, x, nullptr, sf, st); break;
      default: r = step_impl<8>(s, x, nullptr, sf, st); break;
    }
    if (r) break;
    if (refactor) ++qr_count;
    if (cudaEventRecord(e1, st) != cudaSuccess || cudaEventSynchronize(e1) != cudaSuccess ||
        cudaMemcpy(kn.data(), s->knorm, sizeof(double) * kn.size(), cudaMemcpyDeviceToHost) != cudaSuccess) {
      r = NS_ECUDA;
      break;
    }
    // leading limbs: knorm[w][l][k] at (w * K + l) * d + k
    auto nrm = [&](int w, int k) { return kn[(size_t)w * K * d + k]; };
    double nb = 0, nr = 0, ndx = 0;
    for (int k = 0; k < dc; ++k) {
      nb = std::max(nb, nrm(0, k));
      nr = std::max(nr, nrm(1, k));
      ndx = std::max(ndx, nrm(2, k));
    }
    if (log) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      log[it - 1] = ns_iter_log{it, k_lo, dc, refactor ? 1 : 0, nb, nr, ndx, (double)ms};
    }
    // retire stage k (reading R34) when its correction is negligible,
    // ||dx_k|| <= eps ||x_k|| (x_k was already correct, Eq.(11): b_k = 0 =>
    // dx_k = 0), or when it has reached the rounding floor: below
    // sqrt(eps_p) ||x_k|| and no longer shrinking (quadratic convergence
    // would have cut it by far more than 8; late coefficients carry an
    // amplified floor, kappa_k >> 1, SURVEY c.2 Q26)
    auto retired = [&](int k) {
      const double dxk = nrm(2, k), xk = nrm(3, k);
      if (!std::isfinite(dxk) || !std::isfinite(xk)) return false;
      if (dxk <= eps * xk) return true;
      return dxk <= sq * xk && dxk >= prev[k] * 0.125;
    };
    while (k_lo < dc && retired(k_lo)) ++k_lo;
    for (int k = k_lo; k < dc; ++k) prev[k] = nrm(2, k);
    if (k_lo == d) {
      converged = true;
      break;
    }
    if (!std::isfinite(nb) || !std::isfinite(ndx)) break;
    dc = std::min(d, dc + 1 + dc / 2);  // Eq.(10) "d := d + 1 + d/2", floor division
    if (k_lo >= dc) dc = std::min(d, k_lo + 1);
  }
  if (it > max_iter) it = max_iter;
  s->k_lo = 0;
  s->dc = d;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (info) *info = ns_run_info{it, converged ? 1 : 0, qr_count, k_lo};
  return r;
}

ns_status ns_jacobian_pattern(const ns_system* s, int32_t* row_ptr, int32_t* col_idx) {
  if (!s || !row_ptr || !col_idx) return NS_EINVAL;
  std::memcpy(row_ptr, s->h_row_ptr.data(), sizeof(int) * (s->n + 1));
  std::memcpy(col_idx, s->h_col_idx.data(), sizeof(int) * s->nnz);
  return NS_OK;
}

ns_status ns_toeplitz_solve(ns_system* s, const double* b, const double* A, const double* A0, double* dx,
                            void* stream) {
  if (!s || !b || !A || !A0 || !dx) return NS_EINVAL;
  if (s->is_complex) return NS_EINVAL;  // complex: the batched kernel path only (include/ns.h)
  cudaStream_t st = (cudaStream_t)stream;
  const size_t K = s->K, d = s->d, n = s->n;
  CK(cudaMemcpyAsync(s->b, b, sizeof(double) * K * d * n, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(s->A, A, sizeof(double) * K * d * s->nnz, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(s->A0q, A0, sizeof(double) * K * n * n, cudaMemcpyDeviceToDevice, st));
  ns_status r;
  s->last_launches = 0;
  s->use_m = true;
  switch (s->K) {
    case 2: r = Impl<2>::qr(s, s->A0q, nullptr, st); if (!r) r = Impl<2>::stage(s, s->k_lo, st); break;
    case 4: r = Impl<4>::qr(s, s->A0q, nullptr, st); if (!r) r = Impl<4>::stage(s, s->k_lo, st); break;
    default: r = Impl<8>::qr(s, s->A0q, nullptr, st); if (!r) r = Impl<8>::stage(s, s->k_lo, st); break;
  }
  if (r) return r;
  CK(cudaMemcpyAsync(dx, s->dx, sizeof(double) * K * d * n, cudaMemcpyDeviceToDevice, st));
  s->last_stream = st;
  return NS_OK;
}

ns_status ns_get_r_diag(ns_system* s, double* rdiag, void* stream) {
  if (!s || !rdiag) return NS_EINVAL;
  if (!s->qr_cached) return NS_ESTATE;
  CK(cudaMemcpyAsync(rdiag, s->rdiag, sizeof(double) * s->K * s->n, cudaMemcpyDeviceToDevice,
                     (cudaStream_t)stream));
  return NS_OK;
}

ns_status ns_get_status(ns_system* s, ns_step_info* out) {
  if (!s || !out) return NS_EINVAL;
  CK(cudaSetDevice(s->dev));
  CK(cudaDeviceSynchronize());
  unsigned v = 0;
  CK(cudaMemcpy(&v, s->status, sizeof(unsigned), cudaMemcpyDeviceToHost));
  out->status_bits = v;
  out->qr_cached = s->qr_cached ? 1 : 0;
  return NS_OK;
}

ns_status ns_get_ledger(ns_system* s, ns_ledger* out) {
  if (!s || !out) return NS_EINVAL;
  ns_status r = collect_ledger(s);
  if (r) return r;
  *out = s->ledger;
  return NS_OK;
}

ns_status ns_reset_ledger(ns_system* s) {
  if (!s) return NS_EINVAL;
  ns_status r = collect_ledger(s);
  if (r) return r;
  s->ledger = ns_ledger{};
  s->ledger.flops_per_md_fma = md_fma_flops(s->K);
  return NS_OK;
}

int32_t ns_last_launch_count(const ns_system* s) { return s ? s->last_launches : -1; }

}  // extern "C"

extern "C" ns_status ns_md_op(int precision, int op, int n, const double* a, const double* b, double* c,
                              void* stream) {
  if (n < 0 || op < 0 || op > 5 || !a || !c || (op != 4 && !b)) return NS_EINVAL;
  if (n == 0) return NS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  switch (precision) {
    case 2: return Impl<2>::md_op(op, n, a, b, c, st);
    case 4: return Impl<4>::md_op(op, n, a, b, c, st);
    case 8: return Impl<8>::md_op(op, n, a, b, c, st);
    default: return NS_EPREC;
  }
}

// ------------------------------------------------------------------ FP64 peak probe
namespace {
__global__ void __launch_bounds__(256) fp64_probe_kernel(int op, int iters, double seed, double* sink) {
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 1e-9 + i * 1e-12;
  const double m = 0.999999999, c = 1e-300;
  if (op == 0) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = __fma_rn(a[i], m, c);
    }
  } else {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = __dadd_rn(a[i], c);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678) sink[0] = s;  // keep the chains alive
}
}  // namespace

extern "C" ns_status ns_fp64_peak_probe(int device, int op, double* ginstr, double* ms_out) {
  if (!ginstr || (op != 0 && op != 1)) return NS_EINVAL;
  CK(cudaSetDevice(device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  double* sink = nullptr;
  CK(cudaMalloc(&sink, sizeof(double)));
  const int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  fp64_probe_kernel<<<blocks, threads>>>(op, iters, 1.0, sink);  // warm-up
  CK(cudaEventRecord(e0));
  for (int r = 0; r < 5; ++r) fp64_probe_kernel<<<blocks, threads>>>(op, iters, 1.0, sink);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  const double instr = 5.0 * blocks * threads * (double)iters * 8.0;
  *ginstr = instr / (ms * 1e-3) * 1e-9;
  if (ms_out) *ms_out = ms / 5.0;
  return NS_OK;
}

extern "C" ns_status ns_md_latency_probe(int precision, int op, double* cycles_per_op) {
  if (!cycles_per_op || op < 0 || op > 4) return NS_EINVAL;
  switch (precision) {
    case 2: return Impl<2>::latency(op, 256, cycles_per_op);
    case 4: return Impl<4>::latency(op, 256, cycles_per_op);
    case 8: return Impl<8>::latency(op, 256, cycles_per_op);
    default: return NS_EPREC;
  }
}

// ------------------------------------------------------------------ grid barrier probe
namespace {
__global__ void barrier_probe_kernel(int iters, unsigned* bar) {
  ns::GridBarrier gb(bar, 0u);
  for (int i = 0; i < iters; ++i) gb.sync();
}
}  // namespace

extern "C" ns_status ns_barrier_probe(int device, int blocks, int threads, double* us_per_barrier) {
  if (!us_per_barrier || blocks < 1 || threads < 32) return NS_EINVAL;
  CK(cudaSetDevice(device));
  unsigned* bar = nullptr;
  CK(cudaMalloc(&bar, 2 * sizeof(unsigned)));
  CK(cudaMemset(bar, 0, 2 * sizeof(unsigned)));
  int iters = 8;
  void* args[] = {&iters, &bar};
  CK(cudaLaunchCooperativeKernel((const void*)barrier_probe_kernel, dim3(blocks), dim3(threads), args, 0, 0));
  CK(cudaDeviceSynchronize());
  iters = 2000;
  CK(cudaMemset(bar, 0, 2 * sizeof(unsigned)));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0));
  CK(cudaLaunchCooperativeKernel((const void*)barrier_probe_kernel, dim3(blocks), dim3(threads), args, 0, 0));
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(bar);
  *us_per_barrier = ms * 1e3 / iters;
  return NS_OK;
}
