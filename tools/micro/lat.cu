// dependent-chain latencies on B200 (cycles per op), one warp
#include <cstdio>
#include <cstdint>
#define N 256
__global__ void k(double* out, long long* cyc, double a, double b, int s) {
  double x = a, y = b;
  long long t0, t1;
  __shared__ double sm[64];
  sm[threadIdx.x] = a; __syncwarp();
  // DADD
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) x = x + y;
  t1 = clock64(); cyc[0] = t1 - t0;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) x = fma(x, y, a);
  t1 = clock64(); cyc[1] = t1 - t0;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) x = x * y;
  t1 = clock64(); cyc[2] = t1 - t0;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1 + (i & 15));
  t1 = clock64(); cyc[3] = t1 - t0;
  float f = (float)x;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) f = __shfl_xor_sync(0xffffffffu, f, 1 + (i & 15));
  t1 = clock64(); cyc[4] = t1 - t0;
  int idx = s;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) idx = (int)sm[idx & 31];
  t1 = clock64(); cyc[5] = t1 - t0;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) x = x / y;
  t1 = clock64(); cyc[6] = t1 - t0;
  uint64_t u = (uint64_t)s;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) u = u * 0x2545F4914F6CDD1DULL;
  t1 = clock64(); cyc[7] = t1 - t0;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) x = fmax(x, y);
  t1 = clock64(); cyc[8] = t1 - t0;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) x = floor(x + 0.5);
  t1 = clock64(); cyc[9] = t1 - t0;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) x = (double)(u = (uint64_t)x + 1);
  t1 = clock64(); cyc[10] = t1 - t0;
  float ff = f;
  t0 = clock64();
#pragma unroll
  for (int i = 0; i < N; ++i) ff = ff + (float)s;
  t1 = clock64(); cyc[11] = t1 - t0;
  out[threadIdx.x] = x + idx + f + (double)u + ff;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 64 * 8); cudaMalloc(&c, 16 * 8);
  for (int r = 0; r < 3; ++r) k<<<1, 32>>>(o, c, 1.0000001, 0.9999999, 3);
  long long h[16]; cudaMemcpy(h, c, 16 * 8, cudaMemcpyDeviceToHost);
  const char* nm[] = {"dadd", "dfma", "dmul", "shfl64", "shfl32", "lds(dep)", "ddiv", "imul64", "dmax", "floor+add", "d2u+u2d+add", "fadd"};
  for (int i = 0; i < 12; ++i) printf("%-12s %.1f cyc/op\n", nm[i], h[i] / (double)N);
}
