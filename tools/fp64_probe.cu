// FP64 pipe probe for B200: DFMA vs DMMA (mma.sync m8n8k4 f64) throughput,
// and a layout check for the DMMA fragments. Development tool, not product code.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void dmma_kernel(double* out, int iters) {
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0;
  double a = 1e-3 * threadIdx.x, b = 2e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) dmma(acc[2 * j], acc[2 * j + 1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// layout check: A[i][k] = i*10+k (8x4), B[k][j] = (k==j%4) ? 1 : 0 ... use generic values
__global__ void dmma_layout(double* A, double* B, double* C) {
  int lane = threadIdx.x;
  double a = A[(lane >> 2) * 4 + (lane & 3)];       // row-major 8x4
  double b = B[(lane & 3) * 8 + (lane >> 2)];       // row-major 4x8, element (k=lane%4, n=lane/4)
  double d0 = 0, d1 = 0;
  dmma(d0, d1, a, b);
  C[(lane >> 2) * 8 + (lane & 3) * 2 + 0] = d0;
  C[(lane >> 2) * 8 + (lane & 3) * 2 + 1] = d1;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int optin = 0; cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  printf("{\"name\":\"%s\",\"sms\":%d,\"l2\":%d,\"smem_optin\":%d,\"cc\":\"%d.%d\",\"clock_khz\":%d}\n",
         p.name, p.multiProcessorCount, p.l2CacheSize, optin, p.major, p.minor, p.clockRate);
  double *out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf("DFMA: %.3f ms  %.2f TFLOP/s\n", ms, flops / ms / 1e9);
  }
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * blocks * (threads / 32);
    printf("DMMA: %.3f ms  %.2f TFLOP/s\n", ms, flops / ms / 1e9);
  }
  double hA[32], hB[32], hC[64], ref[64];
  for (int i = 0; i < 32; ++i) { hA[i] = i + 1; hB[i] = (i * 7 % 11) - 5; }
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 8; ++j) {
    double s = 0; for (int k = 0; k < 4; ++k) s += hA[i * 4 + k] * hB[k * 8 + j]; ref[i * 8 + j] = s; }
  double *dA, *dB, *dC; cudaMalloc(&dA, 256); cudaMalloc(&dB, 256); cudaMalloc(&dC, 512);
  cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice);
  dmma_layout<<<1, 32>>>(dA, dB, dC);
  cudaMemcpy(hC, dC, 512, cudaMemcpyDeviceToHost);
  double err = 0; for (int i = 0; i < 64; ++i) err += fabs(hC[i] - ref[i]);
  printf("DMMA layout check abs err = %g (%s)\n", err, err == 0 ? "OK" : "MISMATCH");
  printf("cuda error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
