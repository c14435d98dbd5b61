// comm.cu -- multi-GPU plumbing owned by the library (SURVEY 8(b) ns_nccl_unique_id /
// ns_comm_init, 8(e) C4): one NCCL communicator per handle, the equation
// partition of the sharded eval/diff, and the row replication of (b, A, A_0)
// inside the step.
//
// One large system (north_star: "for one large system the monomial convolution
// jobs, followed by an NCCL reduction of the evaluated and differentiated
// series over NVLink").  Equation-owner sharding: rank r
// evaluates and differentiates the contiguous equations [lo_r, hi_r), balanced
// by the prefix sum of their convolution cost, so every row is complete on
// its owner and the "reduction" is a replication: each rank packs its rows of
// b [K][d][n], A [K][d][nnz] and A_0 [K][n][n] into one contiguous block, and
// a grouped ncclBroadcast (one root per rank; NCCL has no all-gather-v) gives
// every rank every block, which is unpacked in place.  Rows are copied, never
// summed: no ncclSum on limb planes (limb-wise FP64 addition is not md
// addition), so the result is bitwise the one-GPU result whatever N.  The QR
// forms A_0 from x itself (replicated), the stage loop and the residual run
// replicated on every rank.
//
// NCCL is loaded at ns_comm_init time (dlopen of the libnccl.so.2 already in
// the process -- torch's -- or the one on the loader path), so the library
// itself has no link-time NCCL dependency.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/ns.h"
#include "system.h"

namespace {

// the NCCL 2.x C ABI subset used here (types as in nccl.h)
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;  // ncclSuccess = 0
constexpr int kNcclFloat64 = 8;

struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the one torch loaded
  if (!h) {
    const char* p = getenv("NS_NCCL_LIB");
    h = dlopen(p ? p : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  }
  if (!h) return api;
  auto sym = [&](const char* n) { return dlsym(h, n); };
  api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
  api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
  api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
  api.CommGetAsyncError = (decltype(api.CommGetAsyncError))sym("ncclCommGetAsyncError");
  api.Broadcast = (decltype(api.Broadcast))sym("ncclBroadcast");
  api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
  api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
  api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.CommGetAsyncError && api.Broadcast &&
           api.GroupStart && api.GroupEnd;
  return api;
}

// Equation partition: contiguous ranges balanced by the prefix sum of the
// per-equation cost sum_tau P(m_tau) d(d+1)/2 + (m_tau + 1) d (the same rule
// as paper_2301_12659_b200/dist.equation_partition; every rank gets >= 1 row).
std::vector<int> partition_bounds(int n, int d, const int* eq_ptr, const int* mono_ptr, int nranks) {
  const long long tri = (long long)d * (d + 1) / 2;
  std::vector<long long> cost(n, 0);
  long long total = 0;
  for (int i = 0; i < n; ++i) {
    for (int t = eq_ptr[i]; t < eq_ptr[i + 1]; ++t) {
      const int m = mono_ptr[t + 1] - mono_ptr[t];
      const long long p = (m <= 1) ? 0 : (m == 2 ? 1 : 3 * m - 5);
      cost[i] += p * tri + (long long)(m + 1) * d;
    }
    total += cost[i];
  }
  std::vector<int> b{0};
  long long acc = 0;
  int r = 1;
  for (int i = 0; i < n; ++i) {
    acc += cost[i];
    // close range r-1 once its share is reached, leaving a row for every later rank
    while (r < nranks && (double)acc >= (double)total * r / nranks && i + 1 > b.back() && n - (i + 1) >= nranks - r) {
      b.push_back(i + 1);
      ++r;
    }
  }
  while ((int)b.size() < nranks) b.push_back(n - (nranks - (int)b.size()));
  b.push_back(n);
  return b;
}

// rank block layout: [b rows: K d (hi-lo)] [A entries: K d (e1-e0)] [A_0 rows: K (hi-lo) n]
long long block_size(int K, int n, int d, const int* row_ptr, int lo, int hi) {
  const long long rows = hi - lo, ent = row_ptr[hi] - row_ptr[lo];
  return (long long)K * ((long long)d * (rows + ent) + rows * n);
}
long long block_size(const ns_system* s, int lo, int hi) { return block_size(s->K, s->n, s->d, s->h_row_ptr.data(), lo, hi); }

// row pointer of the structural Jacobian pattern from a descriptor (row i =
// the distinct variables of equation i), host only
std::vector<int> desc_row_ptr(const ns_system_desc* desc) {
  std::vector<int> rp(desc->dim + 1, 0), mark(desc->dim, -1);
  for (int i = 0; i < desc->dim; ++i) {
    int c = 0;
    for (int t = desc->eq_ptr[i]; t < desc->eq_ptr[i + 1]; ++t)
      for (int q = desc->mono_ptr[t]; q < desc->mono_ptr[t + 1]; ++q)
        if (mark[desc->var_idx[q]] != i) {
          mark[desc->var_idx[q]] = i;
          ++c;
        }
    rp[i + 1] = rp[i] + c;
  }
  return rp;
}

// one thread per block element; pack: block[t] = src, unpack: dst = block[t]
// (b/A/A0 and bw/Aw/A0w may alias: pack reads the former, unpack writes the latter)
__global__ void pack_rows_kernel(int K, int n, int d, int nnz, int lo, int hi, int e0, int e1, const double* b,
                                 const double* A, const double* A0, double* out, int unpack, double* bw, double* Aw,
                                 double* A0w) {
  const long long rows = hi - lo, ent = e1 - e0;
  const long long nb = (long long)K * d * rows, na = (long long)K * d * ent, n0 = (long long)K * rows * n;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < nb + na + n0;
       t += (long long)gridDim.x * blockDim.x) {
    long long src;
    const double* base;
    double* wbase;
    if (t < nb) {
      const long long lk = t / rows, i = lo + t % rows;  // lk = l d + k
      src = lk * n + i;
      base = b;
      wbase = bw;
    } else if (t < nb + na) {
      const long long u = t - nb, lk = u / ent, e = e0 + u % ent;
      src = lk * nnz + e;
      base = A;
      wbase = Aw;
    } else {
      const long long u = t - nb - na, l = u / (rows * n), r = u % (rows * n);
      src = l * (long long)n * n + (long long)lo * n + r;
      base = A0;
      wbase = A0w;
    }
    if (unpack) wbase[src] = out[t];
    else out[t] = base[src];
  }
}

}  // namespace

struct ns_comm {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  std::vector<int> bounds;         // [nranks + 1] equation ranges
  std::vector<long long> off, cnt;  // block offsets / sizes (doubles) in the gather buffer
  double* gather = nullptr;        // all blocks, [sum cnt]
  int sms = 148;
};

bool ns_comm_active(const ns_system* s) { return s && s->comm && s->comm->nranks > 1; }

void ns_comm_free(ns_system* s) {
  if (!s || !s->comm) return;
  if (s->comm->comm && nccl().ok) nccl().CommDestroy(s->comm->comm);
  if (s->comm->gather) cudaFree(s->comm->gather);
  delete s->comm;
  s->comm = nullptr;
}

// After the sharded eval/diff (stream-ordered on st): pack this rank's rows,
// one grouped ncclBroadcast per rank block, unpack the other ranks' rows.
ns_status ns_comm_exchange(ns_system* s, cudaStream_t st) {
  ns_comm* c = s->comm;
  if (!c || c->nranks <= 1) return NS_OK;
  const int lo = c->bounds[c->rank], hi = c->bounds[c->rank + 1];
  const int threads = 256;
  auto grid = [&](long long tot) { return (int)std::max<long long>(1, std::min<long long>((tot + threads - 1) / threads, 4LL * c->sms)); };
  pack_rows_kernel<<<grid(c->cnt[c->rank]), threads, 0, st>>>(s->K, s->n, s->d, s->nnz, lo, hi, s->h_row_ptr[lo],
                                                               s->h_row_ptr[hi], s->b, s->A, s->A0,
                                                               c->gather + c->off[c->rank], 0, nullptr, nullptr, nullptr);
  s->last_launches += 1;
  if (cudaGetLastError() != cudaSuccess) return NS_ECUDA;
  NcclApi& N = nccl();
  if (N.GroupStart() != 0) return NS_ENCCL;
  for (int r = 0; r < c->nranks; ++r) {
    double* p = c->gather + c->off[r];
    if (N.Broadcast(p, p, (size_t)c->cnt[r], kNcclFloat64, r, c->comm, st) != 0) {
      N.GroupEnd();
      return NS_ENCCL;
    }
  }
  if (N.GroupEnd() != 0) return NS_ENCCL;
  for (int r = 0; r < c->nranks; ++r) {
    if (r == c->rank) continue;
    const int l2 = c->bounds[r], h2 = c->bounds[r + 1];
    pack_rows_kernel<<<grid(c->cnt[r]), threads, 0, st>>>(s->K, s->n, s->d, s->nnz, l2, h2, s->h_row_ptr[l2],
                                                          s->h_row_ptr[h2], nullptr, nullptr, nullptr,
                                                          c->gather + c->off[r], 1, s->b, s->A, s->A0);
    s->last_launches += 1;
  }
  return cudaGetLastError() == cudaSuccess ? NS_OK : NS_ECUDA;
}

extern "C" {

ns_status ns_nccl_unique_id(void* uid128) {
  if (!uid128) return NS_EINVAL;
  NcclApi& N = nccl();
  if (!N.ok) return NS_ENCCL;
  ncclUniqueId id;
  if (N.GetUniqueId(&id) != 0) return NS_ENCCL;
  std::memcpy(uid128, &id, sizeof(id));
  return NS_OK;
}

ns_status ns_exchange_plan(const ns_system_desc* desc, int nranks, int32_t* eq_bounds, int64_t* block_doubles) {
  if (!desc || !desc->eq_ptr || !desc->mono_ptr || !desc->var_idx || nranks < 1 || nranks > desc->dim || !eq_bounds)
    return NS_EINVAL;
  const int n = desc->dim, d = desc->degree + 1;
  const std::vector<int> b = partition_bounds(n, d, desc->eq_ptr, desc->mono_ptr, nranks);
  for (int r = 0; r <= nranks; ++r) eq_bounds[r] = b[r];
  if (block_doubles) {
    const std::vector<int> rp = desc_row_ptr(desc);
    for (int r = 0; r < nranks; ++r) block_doubles[r] = block_size(desc->precision, n, d, rp.data(), b[r], b[r + 1]);
  }
  return NS_OK;
}

ns_status ns_pack_rows(const ns_system* s, int lo, int hi, double* b, double* A, double* A0, double* block, int unpack,
                       void* stream) {
  if (!s || lo < 0 || hi > s->n || lo >= hi || !b || !A || !A0 || !block) return NS_EINVAL;
  const long long tot = block_size(s, lo, hi);
  const int grid = (int)std::max<long long>(1, std::min<long long>((tot + 255) / 256, 4LL * s->sms));
  pack_rows_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(s->K, s->n, s->d, s->nnz, lo, hi, s->h_row_ptr[lo],
                                                            s->h_row_ptr[hi], b, A, A0, block, unpack ? 1 : 0, b, A,
                                                            A0);
  return cudaGetLastError() == cudaSuccess ? NS_OK : NS_ECUDA;
}

ns_status ns_comm_init(ns_system* s, int nranks, int rank, const void* uid128) {
  if (!s || nranks < 1 || rank < 0 || rank >= nranks || nranks > s->n || !uid128 || s->is_complex) return NS_EINVAL;
  if (s->k_lo != 0 || s->dc != s->d) return NS_ESTATE;
  NcclApi& N = nccl();
  if (!N.ok) return NS_ENCCL;
  if (cudaSetDevice(s->dev) != cudaSuccess) return NS_ECUDA;
  ns_comm_free(s);
  ns_comm* c = new ns_comm();
  c->nranks = nranks;
  c->rank = rank;
  c->sms = s->sms;
  c->bounds = partition_bounds(s->n, s->d, s->h_eq_ptr.data(), s->h_mono_ptr.data(), nranks);
  long long tot = 0;
  for (int r = 0; r < nranks; ++r) {
    c->off.push_back(tot);
    c->cnt.push_back(block_size(s, c->bounds[r], c->bounds[r + 1]));
    tot += c->cnt.back();
  }
  s->comm = c;
  if (cudaMalloc(&c->gather, sizeof(double) * std::max<long long>(1, tot)) != cudaSuccess) {
    ns_comm_free(s);
    return NS_ENOMEM;
  }
  ncclUniqueId id;
  std::memcpy(&id, uid128, sizeof(id));
  if (N.CommInitRank(&c->comm, nranks, id, rank) != 0) {
    c->comm = nullptr;
    ns_comm_free(s);
    return NS_ENCCL;
  }
  // this rank's eval/diff job queue: its equations only
  const ns_status r = ns_set_partition(s, c->bounds[rank], c->bounds[rank + 1]);
  if (r) {
    ns_comm_free(s);
    return r;
  }
  return NS_OK;
}

ns_status ns_comm_status(ns_system* s, int32_t* nccl_async_error) {
  if (!s || !nccl_async_error) return NS_EINVAL;
  *nccl_async_error = 0;
  if (!s->comm || !s->comm->comm) return NS_OK;
  ncclResult_t e = 0;
  if (nccl().CommGetAsyncError(s->comm->comm, &e) != 0) return NS_ENCCL;
  *nccl_async_error = e;
  return e == 0 ? NS_OK : NS_ENCCL;
}

}  // extern "C"
