// Microbenchmark: FP64 pipe rates of DADD, DMUL, DFMA on independent chains
// (is DADD issued at the DFMA rate?).  Each thread runs 8 independent chains.
#include <cstdio>
template <int OP>
__global__ void k_rate(int iters, double c, double d, double *out) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) x[i] = __dadd_rn(x[i], c);
      else if (OP == 1) x[i] = __dmul_rn(x[i], c);
      else x[i] = __fma_rn(x[i], c, d);
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int OP>
void run(const char *name, int sms) {
  double *out;
  cudaMalloc(&out, (size_t)sms * 2048 * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 20000;
  k_rate<OP><<<sms * 2, 1024>>>(10, 1.0000001, 1e-9, out);
  cudaEventRecord(a);
  k_rate<OP><<<sms * 2, 1024>>>(iters, 1.0000001, 1e-9, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("%s: %.2f T instr/s (%s)\n", name, (double)sms * 2 * 1024 * iters * 8 / (ms * 1e-3) / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("DADD", sms);
  run<1>("DMUL", sms);
  run<2>("DFMA", sms);
  return 0;
}
