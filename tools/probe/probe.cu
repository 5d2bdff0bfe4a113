// Probe: fp64 DFMA / DADD / DMUL throughput and HBM copy on the box (sm_100a).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void fp64_fma(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < iters; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void fp64_add(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < iters; ++i) {
    x0 = __dadd_rn(x0, a); x1 = __dadd_rn(x1, a); x2 = __dadd_rn(x2, a); x3 = __dadd_rn(x3, a);
    x4 = __dadd_rn(x4, b); x5 = __dadd_rn(x5, b); x6 = __dadd_rn(x6, b); x7 = __dadd_rn(x7, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void fp64_rcp(double* out, int iters, double a) {
  double x0 = threadIdx.x + 1.5, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  for (int i = 0; i < iters; ++i) {
    x0 = __drcp_rn(x0) + a; x1 = __drcp_rn(x1) + a; x2 = __drcp_rn(x2) + a; x3 = __drcp_rn(x3) + a;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}
__global__ void copyk(const double4* __restrict__ a, double4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s sm %d.%d SMs %d clock %d kHz mem %d kHz l2 %d smem/block optin %zu\n", p.name, p.major, p.minor,
         p.multiProcessorCount, p.clockRate, p.memoryClockRate, p.l2CacheSize, p.sharedMemPerBlockOptin);
  double* out; cudaMalloc(&out, 148 * 8 * 1024 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000; float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); fp64_fma<<<148 * 8, 256>>>(out, iters, 0.999, 1e-3); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA: %.2f T fma/s (%.2f TFLOP/s)\n", 148.0 * 8 * 256 * iters * 8 / ms / 1e9, 2 * 148.0 * 8 * 256 * iters * 8 / ms / 1e9);
    cudaEventRecord(e0); fp64_add<<<148 * 8, 256>>>(out, iters, 0.999, 1e-3); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DADD: %.2f T add/s\n", 148.0 * 8 * 256 * iters * 8 / ms / 1e9);
    cudaEventRecord(e0); fp64_rcp<<<148 * 8, 256>>>(out, iters / 4, 1e-3); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DRCP_RN(+add): %.2f T rcp/s\n", 148.0 * 8 * 256 * (iters / 4) * 4 / ms / 1e9);
  }
  size_t n = (size_t)1 << 28;  // 2^28 double4 = 8 GiB? no: 32 B each -> 8 GiB; use 2^26 -> 2 GiB
  n = (size_t)1 << 26;
  double4 *a, *b; cudaMalloc(&a, n * 32); cudaMalloc(&b, n * 32); cudaMemset(a, 0, n * 32);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); copyk<<<148 * 16, 512>>>(a, b, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("copy: %.1f GB/s\n", 2.0 * n * 32 / ms / 1e6);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
