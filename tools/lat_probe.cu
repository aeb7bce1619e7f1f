#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_chain(double* out, double a, double b, int n, long long* cyc) {
  double x = threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); }
  long long t1 = clock64();
  out[threadIdx.x + blockIdx.x * blockDim.x] = x;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void bar_loop(int n, long long* cyc, double* out) {
  __shared__ double s[256];
  double x = 1.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { s[threadIdx.x] = x; __syncthreads(); x += s[(threadIdx.x + 1) & 255]; __syncthreads(); }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void lds_chain(int n, long long* cyc, int* out) {
  __shared__ int s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i * 7 + 1) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) p = s[p];
  long long t1 = clock64();
  out[threadIdx.x] = p;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void dmma_chain(int n, long long* cyc, double* out) {
  double d0 = 0.0, d1 = 0.0;
  const double a = 1e-3 * threadIdx.x, b = 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  out[threadIdx.x] = d0 + d1;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void rsqrt_chain(int n, long long* cyc, double* out) {
  double x = 1.5 + 1e-3 * threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double y;
    asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    x = y + 1.0;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void shfl_chain(int n, long long* cyc, double* out) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_xor_sync(0xffffffffu, x, 5);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void warp_smem_loop(int n, long long* cyc, double* out) {
  __shared__ double s[32];
  double x = 1.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { s[threadIdx.x] = x; __syncwarp(); x += s[(threadIdx.x + 1) & 31]; __syncwarp(); }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* d; long long* c; int* di; long long h[4];
  cudaMalloc(&d, 1 << 20); cudaMalloc(&c, 64); cudaMalloc(&di, 4096);
  int n = 4096;
  dfma_chain<<<1, 32>>>(d, 0.999, 1e-3, n, c); cudaDeviceSynchronize();
  dfma_chain<<<1, 32>>>(d, 0.999, 1e-3, n, c); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", (double)h[0] / (4.0 * n));
  dfma_chain<<<1, 256>>>(d, 0.999, 1e-3, n, c); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
  printf("DFMA chain, 8 warps: %.2f cycles per dependent op\n", (double)h[0] / (4.0 * n));
  bar_loop<<<1, 256>>>(n, c, d); cudaDeviceSynchronize(); bar_loop<<<1, 256>>>(n, c, d); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
  printf("STS+BAR+LDS+BAR loop (256 thr): %.2f cycles/iter\n", (double)h[0] / n);
  lds_chain<<<1, 32>>>(n, c, di); cudaDeviceSynchronize(); lds_chain<<<1, 32>>>(n, c, di); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
  printf("LDS dependent latency: %.2f cycles\n", (double)h[0] / n);
  dmma_chain<<<1, 32>>>(n, c, d); cudaDeviceSynchronize(); dmma_chain<<<1, 32>>>(n, c, d); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
  printf("DMMA dependent (same accumulator) latency: %.2f cycles\n", (double)h[0] / (4.0 * n));
  rsqrt_chain<<<1, 32>>>(n, c, d); cudaDeviceSynchronize(); rsqrt_chain<<<1, 32>>>(n, c, d); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
  printf("rsqrt.approx.f64 + DADD dependent: %.2f cycles\n", (double)h[0] / n);
  shfl_chain<<<1, 32>>>(n, c, d); cudaDeviceSynchronize(); shfl_chain<<<1, 32>>>(n, c, d); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
  printf("64-bit SHFL dependent: %.2f cycles\n", (double)h[0] / n);
  warp_smem_loop<<<1, 32>>>(n, c, d); cudaDeviceSynchronize(); warp_smem_loop<<<1, 32>>>(n, c, d); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
  printf("STS+syncwarp+LDS+DADD+syncwarp loop (1 warp): %.2f cycles/iter\n", (double)h[0] / n);
  return 0;
}
