// Microbenchmark: latency and throughput of the device xprec complex ops
// (cmul / cadd in dd and qd) -- guides ILP vs occupancy choices.
// nvcc -O3 -std=c++20 -gencode arch=compute_100a,code=sm_100a -fmad=false -I../../paper_1402_2626_b200/csrc
#include <cstdio>
#include "xprec.cuh"
using namespace pn;

template <class E, int OP, int CH, int LB = 256>
__global__ void __launch_bounds__(LB) k_chain(int iters, const double *in, double *out, long long *cyc) {
  E x[CH], c;
  const double *p = in + (threadIdx.x % 32) * 16;
  for (int i = 0; i < Traits<E>::es; ++i) reinterpret_cast<double *>(&c)[i] = p[i] * 0.5 + 0.25;
  for (int h = 0; h < CH; ++h)
    for (int i = 0; i < Traits<E>::es; ++i) reinterpret_cast<double *>(&x[h])[i] = p[i + 1] + h;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int h = 0; h < CH; ++h) x[h] = OP == 0 ? emul(x[h], c) : eadd(x[h], c);
  }
  long long t1 = clock64();
  double s = 0;
  for (int h = 0; h < CH; ++h) s += reinterpret_cast<double *>(&x[h])[0];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <class E, int OP, int CH, int LB = 256>
void run(const char *name, int blocks, int threads, int iters, double *in, double *out, long long *cyc) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_chain<E, OP, CH, LB><<<blocks, threads>>>(2, in, out, cyc);
  cudaEventRecord(a);
  k_chain<E, OP, CH, LB><<<blocks, threads>>>(iters, in, out, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long hc;
  cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
  if (cudaGetLastError() != cudaSuccess) { printf("%s launch failed\n", name); return; }
  const double ops = (double)blocks * threads * iters * CH;
  printf("%-10s blocks=%4d thr=%4d chains=%d  cycles/op/chain=%8.1f  Gops/s=%9.3f\n", name, blocks, threads, CH,
         (double)hc / iters, ops / (ms * 1e-3) / 1e9);
}

int main() {
  double *in, *out;
  long long *cyc;
  cudaMalloc(&in, 32 * 16 * 8 + 64);
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&cyc, 8);
  double h[32 * 16 + 8];
  for (int i = 0; i < 32 * 16 + 8; ++i) h[i] = 1.0 + 1e-3 * i;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int it = 2000;
  // single warp latency
  run<C<2>, 0, 1>("cdd mul", 1, 32, it, in, out, cyc);
  run<C<2>, 1, 1>("cdd add", 1, 32, it, in, out, cyc);
  run<C<4>, 0, 1>("cqd mul", 1, 32, it / 4, in, out, cyc);
  run<C<4>, 1, 1>("cqd add", 1, 32, it / 4, in, out, cyc);
  run<F<4>, 0, 1>("qd mul", 1, 32, it / 4, in, out, cyc);
  run<C<4>, 0, 2>("cqd mul", 1, 32, it / 4, in, out, cyc);
  // per-SM throughput vs warps (1 CTA per SM)
  for (int w : {1, 2, 4, 8, 16, 32}) run<C<4>, 0, 1>("cqd mul", sms, 32 * w, it / 8, in, out, cyc);
  for (int w : {1, 2, 4, 8, 16, 32}) run<C<2>, 0, 1>("cdd mul", sms, 32 * w, it / 2, in, out, cyc);
  for (int w : {4, 8, 16}) run<C<2>, 0, 4>("cdd mul", sms, 32 * w, it / 8, in, out, cyc);
  for (int w : {1, 2, 4, 8, 16, 32}) run<C<2>, 1, 1>("cdd add", sms, 32 * w, it / 2, in, out, cyc);
  for (int w : {4, 8, 16}) run<C<4>, 1, 1>("cqd add", sms, 32 * w, it / 8, in, out, cyc);
  // more warps per SM at bounded registers
  run<C<4>, 0, 1, 512>("cqd mul", sms, 512, it / 8, in, out, cyc);
  run<C<4>, 0, 1, 768>("cqd mul", sms, 768, it / 8, in, out, cyc);
  run<C<4>, 0, 1, 1024>("cqd mul", sms, 1024, it / 8, in, out, cyc);
  run<C<4>, 1, 1, 512>("cqd add", sms, 512, it / 8, in, out, cyc);
  run<C<4>, 1, 1, 1024>("cqd add", sms, 1024, it / 8, in, out, cyc);
  run<C<2>, 0, 1, 1024>("cdd mul", sms, 1024, it / 2, in, out, cyc);
  return 0;
}
