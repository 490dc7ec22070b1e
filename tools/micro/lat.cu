// latency / throughput microbenchmarks of the fp64 ops on the K1/K3 paths (one warp, clock64)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b, float fa) {
  double x = a, y = b;
  long long t0, t1;
  // DFMA dependent chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { x = fma(x, y, 1e-300); x = fma(x, y, 1e-300); x = fma(x, y, 1e-300); x = fma(x, y, 1e-300); }
  t1 = clock64(); cyc[0] = (t1 - t0); out[0] = x;
  // DADD chain
  x = a; t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { x = x + y; x = x + y; x = x + y; x = x + y; }
  t1 = clock64(); cyc[1] = (t1 - t0); out[1] = x;
  // F2F f32->f64 chain (through float)
  float f = fa; t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { double d = (double)f; f = __double2float_rn(d * 1.0000001); }
  t1 = clock64(); cyc[2] = (t1 - t0); out[2] = f;
  // SHFL double chain
  x = a; t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { x = __shfl_xor_sync(0xffffffffu, x, 1); x = __shfl_xor_sync(0xffffffffu, x, 2); }
  t1 = clock64(); cyc[3] = (t1 - t0); out[3] = x;
  // division chain
  x = a; t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) { x = y / (x + 1.5); }
  t1 = clock64(); cyc[4] = (t1 - t0); out[4] = x;
  // DFMA throughput: 8 independent chains
  double c[8];
  for (int j = 0; j < 8; ++j) c[j] = a + j;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j] = fma(c[j], y, 1e-300);
  t1 = clock64(); cyc[5] = (t1 - t0);
  double s = 0; for (int j = 0; j < 8; ++j) s += c[j]; out[5] = s;
}
int main() {
  double* o; long long* c;
  cudaMallocManaged(&o, 64 * 8); cudaMallocManaged(&c, 64 * 8);
  for (int warps : {1, 4, 16, 32}) {
    k<<<1, 32 * warps>>>(o, c, 1.0, 0.999999, 1.0f);
    cudaDeviceSynchronize();
    printf("warps/SM %2d: DFMA lat %.2f  DADD lat %.2f  F2F+F2F+DMUL chain %.2f  SHFL.f64 lat %.2f  DDIV lat %.2f  DFMA x8 indep per inst %.3f\n",
           warps, c[0] / 4096.0, c[1] / 4096.0, c[2] / 1024.0, c[3] / 2048.0, c[4] / 256.0, c[5] / 8192.0);
  }
  return 0;
}
