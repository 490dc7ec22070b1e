// k_datagen.cu -- K6: synthetic datasets for BASELINE.json configs C2..C5,
// generated on the device from a counter-based hash so that 64 GiB never
// has to be produced on the host.  (The reference's own generator,
// make_regression, objectives.cpp:27-45, is sequential; it is restated in
// the oracle for the reference-scale parity cases.)  The bytes produced here
// are copied back to the CPU oracle by the tests.
//
// kind 0: x ~ N(0, x_scale^2), w* ~ N(0,1), y = x.w* + noise_sd * N(0,1)      (C3, C5)
// kind 1: x ~ U[0,1) kept with probability `density`, teacher W ~ N(0,1)
//         (d x C), label = argmax_c (x.W_c + Gumbel)                           (C2)
// kind 2: x ~ N(0, x_scale^2), w* ~ N(0,1), label ~ Bernoulli(sigmoid(x.w*))   (C4)
#include "halp_device.cuh"
#include "kernels.h"

namespace halp {

// Every value is produced by integer hashing and IEEE-exact float/double
// operations (+ - * / sqrt and explicit fma, never contracted: -fmad=false)
// plus the deterministic hexp/hlog, so the host restatement
// oracle/datagen.c (oq_datagen) reproduces the bytes exactly: the reference
// arm of bench.py and the tests regenerate any row range on the CPU without
// touching this library.
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t ctr(uint64_t seed, uint64_t stream, uint64_t i) {
  return mix64(mix64(seed ^ (stream * 0xD1B54A32D192ED03ULL)) + i * 0x9E3779B97F4A7C15ULL);
}
__device__ __forceinline__ double unif64(uint64_t seed, uint64_t stream, uint64_t i) {
  return (double)(ctr(seed, stream, i) >> 11) * 0x1.0p-53;
}
// ln x for x in (0, 1]: x = m 2^e, m in [sqrt(1/2), sqrt(2)), atanh series in f = (m-1)/(m+1)
__device__ __forceinline__ float det_logf(float x) {
  const uint32_t b = __float_as_uint(x);
  int e = (int)((b >> 23) & 255u) - 127;
  float m = __uint_as_float((b & 0x7FFFFFu) | 0x3F800000u);
  if (m > 1.41421356f) {
    m = m * 0.5f;
    e += 1;
  }
  const float f = (m - 1.0f) / (m + 1.0f);
  const float f2 = f * f;
  float q = 0.0909090909f;
  q = q * f2 + 0.111111111f;
  q = q * f2 + 0.142857143f;
  q = q * f2 + 0.2f;
  q = q * f2 + 0.333333333f;
  const float tf = 2.0f * f;
  const float lnm = tf + tf * (f2 * q);
  const float ef = (float)e;
  return ef * 0.693145752f + (ef * 1.42860677e-06f + lnm);
}
// cos(2 pi k / 2^24) for a 24-bit integer k: nearest quarter turn + a polynomial on [-pi/4, pi/4]
__device__ __forceinline__ float det_cos2pi(uint32_t k) {
  const uint32_t qu = (k + (1u << 21)) >> 22;
  const int r = (int)k - (int)(qu << 22);
  const float a = (float)r * 3.74507028e-07f;  // (pi/2) / 2^22
  const float a2 = a * a;
  const float c = 1.0f + a2 * (-0.5f + a2 * (0.0416666667f + a2 * (-0.00138888889f + a2 * 2.48015873e-05f)));
  const float s = a + (a * a2) * (-0.166666667f + a2 * (0.00833333333f + a2 * (-0.000198412698f + a2 * 2.75573192e-06f)));
  const uint32_t q = qu & 3u;
  return q == 0 ? c : q == 1 ? -s : q == 2 ? -c : s;
}
__device__ __forceinline__ float unif32(uint64_t seed, uint64_t stream, uint64_t i) {
  return (float)(ctr(seed, stream, i) >> 40) * 0x1.0p-24f;
}
// Box-Muller from one 64-bit hash: 24 bits for the radius, 24 for the angle
__device__ __forceinline__ float normal32(uint64_t seed, uint64_t stream, uint64_t i) {
  const uint64_t h = ctr(seed, stream, i);
  const float u1 = ((float)(h >> 40) + 0.5f) * 0x1.0p-24f;
  return sqrtf(-2.0f * det_logf(u1)) * det_cos2pi((uint32_t)((h >> 16) & 0xFFFFFFu));
}
__device__ __forceinline__ double normal64(uint64_t seed, uint64_t stream, uint64_t i) {
  return (double)normal32(seed, stream, i);
}

template <class Tx> __device__ __forceinline__ Tx from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ double from_f<double>(float v) { return (double)v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

template <class Tx>
__global__ void k_gen_x(GenParams p) {
  Tx* X = reinterpret_cast<Tx*>(p.X);
  const uint64_t total = (uint64_t)p.n * p.d;
  const float sc = (float)p.x_scale;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (uint64_t)gridDim.x * blockDim.x) {
    float v;
    if (p.kind == 1) {
      const uint64_t h = ctr(p.seed, 1, e);
      const float u = (float)(h >> 40) * 0x1.0p-24f;
      const float keep = (float)((h >> 16) & 0xFFFFFF) * 0x1.0p-24f;
      v = keep < (float)p.density ? u : 0.0f;
    } else {
      v = normal32(p.seed, 1, e) * sc;
    }
    X[e] = from_f<Tx>(v);
  }
}

template <class Tx>
__global__ void k_gen_y(GenParams p) {
  extern __shared__ double wsm[];  // w* (d) or teacher W (d*C, column-major)
  const int d = p.d, C = p.kind == 1 ? p.C : 1;
  for (int k = threadIdx.x; k < d * C; k += blockDim.x) wsm[k] = normal64(p.seed, 2, (uint64_t)k);
  __syncthreads();
  const Tx* X = reinterpret_cast<const Tx*>(p.X);
  const int lane = threadIdx.x & 31, wpb = blockDim.x >> 5;
  for (int64_t i = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); i < p.n; i += (int64_t)gridDim.x * wpb) {
    double acc[kMaxClasses];
    for (int c = 0; c < C; ++c) acc[c] = 0.0;
    for (int j = lane; j < d; j += 32) {
      const double x = to_d<Tx>(X[i * d + j]);
      for (int c = 0; c < C; ++c) acc[c] = fma(x, wsm[c * d + j], acc[c]);
    }
    for (int c = 0; c < C; ++c) acc[c] = warp_allsum(acc[c]);
    if (lane == 0) {
      if (p.kind == 0) {
        p.y[i] = acc[0] + p.noise_sd * normal64(p.seed, 3, (uint64_t)i);
      } else if (p.kind == 1) {
        int best = 0;
        double bv = -1e300;
        for (int c = 0; c < C; ++c) {
          const double u = unif64(p.seed, 4, (uint64_t)i * C + c) + 0x1.0p-54;
          const double v = acc[c] - hlog(-hlog(u));
          if (v > bv) {
            bv = v;
            best = c;
          }
        }
        p.labels[i] = best;
      } else {
        const double pr = 1.0 / (1.0 + hexp(-acc[0]));
        p.labels[i] = unif64(p.seed, 4, (uint64_t)i) < pr ? 1 : 0;
      }
    }
  }
}

template <class Tx>
static cudaError_t gen_t(const GenParams& p, cudaStream_t st) {
  k_gen_x<Tx><<<148 * 8, 256, 0, st>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int C = p.kind == 1 ? p.C : 1;
  const size_t smem = sizeof(double) * (size_t)p.d * C;
  e = cudaFuncSetAttribute(k_gen_y<Tx>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_gen_y<Tx><<<148 * 4, 256, smem, st>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_datagen(const GenParams& p, cudaStream_t st) {
  switch (p.dtype) {
    case 0: return gen_t<double>(p, st);
    case 1: return gen_t<float>(p, st);
    default: return gen_t<__nv_bfloat16>(p, st);
  }
}

// any non-finite bf16 (exponent field all ones) -> *flag = 1; grid-stride,
// 16-byte loads (problem creation only, for the K1 integer-conversion path)
__global__ void k_nonfinite_bf16(const uint4* __restrict__ X, int64_t vecs, int* flag) {
  int bad = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < vecs; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 v = X[i];
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) bad |= ((w[q] & 0x7F80u) == 0x7F80u) | ((w[q] & 0x7F800000u) == 0x7F800000u);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

cudaError_t launch_nonfinite_bf16(const void* X, int64_t elems, int* flag, cudaStream_t st) {
  // rows are padded to 16 bytes with zeros, so elems is a multiple of 8
  const int64_t vecs = elems / 8;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = (vecs + 255) / 256;
  if (blocks > (int64_t)sms * 8) blocks = (int64_t)sms * 8;
  if (blocks < 1) blocks = 1;
  k_nonfinite_bf16<<<(int)blocks, 256, 0, st>>>(reinterpret_cast<const uint4*>(X), vecs, flag);
  return cudaGetLastError();
}

}  // namespace halp
