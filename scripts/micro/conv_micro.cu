// Microbenchmarks of the eval/diff convolution on one CTA (development tool,
// not part of the library): FP64 op latencies and conv_batch cycles per call.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_2301_12659_b200/csrc/evaldiff.cuh"

__global__ void lat_kernel(int op, int iters, double a, double b, double* out, long long* cyc) {
  double x = a, y = b, z = a * 0.5, w = b * 0.25;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (op == 0) x = __dadd_rn(x, y);
    else if (op == 1) x = __fma_rn(x, y, b);
    else if (op == 2) { x = __dadd_rn(x, y); z = __dadd_rn(z, y); w = __dadd_rn(w, y); y = __dadd_rn(y, a); }
    else { double s, e; md::two_sum(x, y, s, e); x = s; y = e + b; }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = x + y + z + w; cyc[0] = t1 - t0; }
}

template <int K>
__global__ void conv_kernel(const double* xg, double* out, long long* cyc, int d, int reps, int mt, int mode, int act) {
  __shared__ long long dbg[2];
  long long acc_terms = 0, acc_bfly = 0, acc_tail = 0;
  extern __shared__ double sm[];
  double* A = sm;
  double* B = sm + K * d;
  double* C = sm + 2 * K * d;
  for (int t = threadIdx.x; t < 2 * K * d; t += blockDim.x) sm[t] = xg[t];
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    const long long ts = clock64();
    if ((int)threadIdx.x < act)
      ns::conv_batch<K>(threadIdx.x, act, 1, d,
                        [&](int, ns::SerRef& pa, ns::SerRef& pb, double*& pc) {
                          pa = ns::SerRef{(r & 1) ? C : A, d};
                          pb = ns::SerRef{B, d};
                          pc = (r & 1) ? A : C;
                        },
                        nullptr, mt, mode, dbg);
    const long long te = clock64();
    if (threadIdx.x == 0) { acc_terms += dbg[0] - ts; acc_bfly += dbg[1] - dbg[0]; acc_tail += te - dbg[1]; }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = acc_terms; cyc[2] = acc_bfly; cyc[3] = acc_tail; }
  for (int t = threadIdx.x; t < K * d; t += blockDim.x) out[t] = C[t];
}

template <int K>
void run_conv(int d, int mt, int mode, int threads, int act) {
  std::vector<double> h(2 * K * d);
  srand(1);
  for (int l = 0; l < K; ++l)
    for (int i = 0; i < 2 * d; ++i) h[l * 2 * d + i] = (l == 0 ? 1.0 : 1e-17) * (rand() / (double)RAND_MAX - 0.5);
  double *xg, *out;
  long long* cyc;
  cudaMalloc(&xg, sizeof(double) * h.size());
  cudaMalloc(&out, sizeof(double) * K * d);
  cudaMalloc(&cyc, 32);
  cudaMemcpy(xg, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
  const int reps = 64;
  size_t smem = 3 * K * d * sizeof(double);
  conv_kernel<K><<<1, threads, smem>>>(xg, out, cyc, d, 2, mt, mode, act);
  conv_kernel<K><<<1, threads, smem>>>(xg, out, cyc, d, reps, mt, mode, act);
  long long c[4] = {0, 0, 0, 0};
  cudaMemcpy(c, cyc, 32, cudaMemcpyDeviceToHost);
  printf("{\"K\": %d, \"d\": %d, \"min_terms\": %d, \"mode\": %d, \"threads\": %d, \"active\": %d, \"cycles_per_conv\": %.1f, \"terms\": %.1f, \"butterfly\": %.1f, \"tail\": %.1f, \"err\": \"%s\"}\n",
         K, d, mt, mode, threads, act, (double)c[0] / reps, (double)c[1] / reps, (double)c[2] / reps, (double)c[3] / reps,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(xg); cudaFree(out); cudaFree(cyc);
}

// reflector chain pieces on one warp (K = 4): cycles per iteration
template <int K>
__global__ void refl_kernel(int op, int iters, const double* in, double* out, long long* cyc) {
  const int lane = threadIdx.x & 31;
  md::mdv<K> a = md::load<K>(in, 4, lane % 4);
  double s[K];
  for (int l = 0; l < K; ++l) s[l] = a.x[l];
  md::mdv<K> acc = a;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (op == 0) {  // lazy 32-lane butterfly
      acc = md::group_sum_levels<K>(s, 32);
      s[0] += acc.x[0] * 1e-30;
    } else if (op == 1) {  // sqrt -> sub -> mul -> recip
      md::mdv<K> nrm = md::sqrt<K>(md::absv<K>(acc));
      md::mdv<K> v0 = md::sub<K>(a, nrm);
      acc = md::recip<K>(md::mul<K>(nrm, v0));
    } else if (op == 2) {  // sqrt only
      acc = md::sqrt<K>(md::absv<K>(acc));
    } else if (op == 3) {  // renormalising butterfly (group_sum)
      acc = md::group_sum<K>(acc, 32);
    } else {  // mul -> fma (column update)
      md::mdv<K> nw = md::mul<K>(acc, a);
      acc = md::fma_acc<K>(a, nw, acc);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { md::store<K>(out, 1, 0, acc); cyc[0] = t1 - t0; }
}

int main() {
  {
    double h[16] = {1.5, 0.75, 1.25, 2.0, 1e-17, 2e-17, 3e-17, 1e-17, 1e-34, 1e-34, 1e-34, 1e-34, 0, 0, 0, 0};
    double *in, *out; long long* cyc;
    cudaMalloc(&in, sizeof(h)); cudaMalloc(&out, 64); cudaMalloc(&cyc, 8);
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    const char* nm[] = {"butterfly_lazy", "sqrt_sub_mul_recip", "sqrt", "butterfly_renorm", "mul_fma"};
    for (int op = 0; op < 5; ++op) {
      refl_kernel<4><<<1, 32>>>(op, 4, in, out, cyc);
      refl_kernel<4><<<1, 32>>>(op, 256, in, out, cyc);
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      printf("{\"K\": 4, \"op\": \"%s\", \"cycles\": %.1f}\n", nm[op], c / 256.0);
    }
    for (int op = 0; op < 5; ++op) {
      refl_kernel<2><<<1, 32>>>(op, 4, in, out, cyc);
      refl_kernel<2><<<1, 32>>>(op, 256, in, out, cyc);
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      printf("{\"K\": 2, \"op\": \"%s\", \"cycles\": %.1f}\n", nm[op], c / 256.0);
    }
  }
  double* out; long long* cyc;
  cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
  const char* names[] = {"dadd_chain", "dfma_chain", "dadd_4chains", "two_sum_chain"};
  for (int op = 0; op < 4; ++op) {
    lat_kernel<<<1, 32>>>(op, 16, 1.0, 1e-3, out, cyc);
    lat_kernel<<<1, 32>>>(op, 4096, 1.0, 1e-3, out, cyc);
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("{\"op\": \"%s\", \"cycles_per_iter\": %.2f}\n", names[op], c / 4096.0);
  }
  for (int mode : {0, 1})
    for (int mt : {2, 4, 8}) {
      run_conv<4>(32, mt, mode, 256, 256);
      run_conv<4>(32, mt, mode, 128, 128);
      run_conv<4>(32, mt, mode, 256, 128);
    }
  for (int mode : {0, 1})
    for (int mt : {2, 4, 8}) run_conv<2>(32, mt, mode, 256, 256);
  for (int mode : {0, 1})
    for (int mt : {4, 8}) run_conv<8>(64, mt, mode, 256, 256);
  return 0;
}
