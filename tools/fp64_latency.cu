// fp64_latency.cu -- dependent DADD / DFMA / LDS chains on one warp (diagnostic tool).
#include <cuda_runtime.h>
#include <stdint.h>
__global__ void chain_dadd(double* out, double x, int n, long long* cyc) {
  double acc = 0.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, x + i);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = acc; cyc[0] = t1 - t0; }
}
__global__ void chain_dmul_dadd_smem(double* out, int n, long long* cyc) {
  __shared__ double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = 1.0 + i * 1e-3;
  __syncthreads();
  double acc = 0.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, __dmul_rn(sm[i & 4095], sm[(4095 - i) & 4095]));
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = acc; cyc[0] = t1 - t0; }
}
__global__ void chain_fadd(float* out, float x, int n, long long* cyc) {
  float acc = 0.0f;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) acc = __fadd_rn(acc, x + i);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = acc; cyc[0] = t1 - t0; }
}
extern "C" void run_chains(int n, long long* host_cyc) {
  double* d; long long* c; float* f;
  cudaMalloc(&d, 64); cudaMalloc(&c, 64); cudaMalloc(&f, 64);
  chain_dadd<<<1, 32>>>(d, 1.5, n, c); cudaMemcpy(host_cyc + 0, c, 8, cudaMemcpyDeviceToHost);
  chain_dmul_dadd_smem<<<1, 32>>>(d, n, c); cudaMemcpy(host_cyc + 1, c, 8, cudaMemcpyDeviceToHost);
  chain_fadd<<<1, 32>>>(f, 1.5f, n, c); cudaMemcpy(host_cyc + 2, c, 8, cudaMemcpyDeviceToHost);
  cudaFree(d); cudaFree(c); cudaFree(f);
}
