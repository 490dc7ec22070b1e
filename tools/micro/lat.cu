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
  // REDUX.SUM chain (32-bit)
  int r = (int)a + threadIdx.x; t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { r = __reduce_add_sync(0xffffffffu, r) + 1; r = __reduce_add_sync(0xffffffffu, r) + 1; }
  t1 = clock64(); cyc[6] = (t1 - t0); out[6] = r;
  // F2I.S64.F64 + I2F.F64.S64 round trip
  x = a * 1000.0; t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { long long q = __double2ll_rn(x); x = __ll2double_rn(q + 1); }
  t1 = clock64(); cyc[7] = (t1 - t0); out[7] = x;
  // FRND.F64.FLOOR chain (+ DADD)
  x = a * 1000.5; t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { x = floor(x) + 0.5; x = floor(x) + 0.5; }
  t1 = clock64(); cyc[8] = (t1 - t0); out[8] = x;
  // 3 independent REDUX + recombine (warp_sum_s64 shape)
  long long v = (long long)(a * 1e15) + threadIdx.x; t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
    const int lo = __reduce_add_sync(0xffffffffu, (int)(v & 0x1FFFFF));
    const int mi = __reduce_add_sync(0xffffffffu, (int)((v >> 21) & 0x1FFFFF));
    const int hi = __reduce_add_sync(0xffffffffu, (int)(v >> 42));
    v = ((long long)hi * (1LL << 42) + (long long)mi * (1LL << 21) + (long long)lo) >> 5;
  }
  t1 = clock64(); cyc[9] = (t1 - t0); out[9] = (double)v;
  // LDS dependent chain
  __shared__ int sm[256];
  sm[threadIdx.x & 255] = (threadIdx.x + 1) & 255;
  __syncthreads();
  int ix = threadIdx.x & 255; t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { ix = sm[ix]; ix = sm[ix]; }
  t1 = clock64(); cyc[10] = (t1 - t0); out[10] = ix;
  // DMUL -> F2I.S64 -> (int add) chain ; and I2F -> DMUL
  x = a; t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { x = __dmul_rn(x, 1.0000001); }
  t1 = clock64(); cyc[11] = (t1 - t0); out[11] = x;
  // SHFL 32-bit chain
  int sh = threadIdx.x; t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { sh = __shfl_xor_sync(0xffffffffu, sh, 1) + 1; sh = __shfl_xor_sync(0xffffffffu, sh, 2) + 1; }
  t1 = clock64(); cyc[12] = (t1 - t0); out[12] = sh;
  // IMAD 64-bit chain (xorshift-like int ops)
  unsigned long long u = (unsigned long long)threadIdx.x + 88172645463325252ULL; t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) { u ^= u >> 12; u ^= u << 25; u ^= u >> 27; }
  t1 = clock64(); cyc[13] = (t1 - t0); out[13] = (double)u;
}
int main() {
  double* o; long long* c;
  cudaMallocManaged(&o, 64 * 8); cudaMallocManaged(&c, 64 * 8);
  for (int warps : {1, 4, 16, 32}) {
    k<<<1, 32 * warps>>>(o, c, 1.0, 0.999999, 1.0f);
    cudaDeviceSynchronize();
    printf("warps/SM %2d: DFMA lat %.2f  DADD lat %.2f  F2F+F2F+DMUL chain %.2f  SHFL.f64 lat %.2f  DDIV lat %.2f  DFMA x8 indep per inst %.3f\n",
           warps, c[0] / 4096.0, c[1] / 4096.0, c[2] / 1024.0, c[3] / 2048.0, c[4] / 256.0, c[5] / 8192.0);
    printf("             REDUX+IADD lat %.2f  F2I.S64+IADD+I2F %.2f  FRND.FLOOR+DADD %.2f  warp_sum_s64 (3 REDUX + recombine + shift) %.2f  LDS chain %.2f  DMUL lat %.2f  SHFL32+IADD %.2f  xorshift step (64-bit) %.2f\n",
           c[6] / 2048.0, c[7] / 1024.0, c[8] / 2048.0, c[9] / 1024.0, c[10] / 2048.0, c[11] / 1024.0, c[12] / 2048.0, c[13] / 1024.0);
  }
  return 0;
}
