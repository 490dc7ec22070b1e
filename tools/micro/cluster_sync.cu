// Microbenchmark: per-step cost of the K3 cluster exchange mechanisms (B200).
//  mode 0: barrier.cluster arrive.release/wait.acquire only
//  mode 1: DSMEM stores of 4 doubles per warp to every CTA + cluster barrier
//  mode 2: st.async + mbarrier complete_tx to every CTA, wait on local mbarrier (no cluster barrier)
//  mode 3: __syncthreads only (single CTA reference)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t ctarank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t r) {
  uint32_t ra; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(p)), "r"(r)); return ra;
}

__global__ void __launch_bounds__(256, 1) kern(int mode, int steps, unsigned long long* out) {
  __shared__ double buf[2][16 * 8 * 4];
  __shared__ unsigned long long llbuf[2][16 * 8 * 8];
  __shared__ __align__(8) uint64_t mbar[2];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int NC = gridDim.x;
  const uint32_t rank = ctarank();
  const int NW = blockDim.x / 32;
  const uint32_t bytes = (uint32_t)(NC * NW * 4 * 8);
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < 2 * 16 * 8 * 8; i += blockDim.x) (&llbuf[0][0])[i] = 0ull;
  __syncthreads();
  csync();
  double acc = lane;
  unsigned long long t0 = clock64();
  for (int t = 0; t < steps; ++t) {
    const int par = t & 1;
    if (mode == 0) {
      csync();
    } else if (mode == 1) {
      if ((lane & 7) == 0) {
        const int slot = lane >> 3;
        for (int r = 0; r < NC; ++r) {
          uint32_t a = mapa(&buf[par][(rank * NW + wid) * 4 + slot], r);
          asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(acc) : "memory");
        }
      }
      csync();
      acc += buf[par][lane];
    } else if (mode == 2) {
      if (tid == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar[par])), "r"(bytes) : "memory");
      if ((lane & 7) == 0) {
        const int slot = lane >> 3;
        for (int r = 0; r < NC; ++r) {
          uint32_t a = mapa(&buf[par][(rank * NW + wid) * 4 + slot], r);
          uint32_t b = mapa(&mbar[par], r);
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(a), "d"(acc), "r"(b) : "memory");
        }
      }
      asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(smem_u32(&mbar[par])), "r"((t >> 1) & 1) : "memory");
      acc += buf[par][lane];
    } else if (mode == 5) {
      // LL protocol: each double travels as two 8-byte {32-bit half, 32-bit step flag} words
      const uint32_t flag = (uint32_t)(t + 1);
      const unsigned long long bits = (unsigned long long)__double_as_longlong(acc);
      for (int l0 = lane; l0 < NC * 8; l0 += 32) {
        const int r = l0 >> 3, w8 = l0 & 7;  // 4 doubles = 8 words
        const uint32_t half = (w8 & 1) ? (uint32_t)(bits >> 32) : (uint32_t)bits;
        const unsigned long long word = ((unsigned long long)flag << 32) | half;
        uint32_t a = mapa(&llbuf[par][(rank * NW + wid) * 8 + w8], r);
        asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(a), "l"(word) : "memory");
      }
      // consumer: lane q reads the 8 words of warp q (q < NC*NW) and spins on their flags
      double v = 0.0;
      for (int q = lane; q < NC * NW; q += 32) {
        unsigned long long lo, hi;
        const unsigned long long ts = clock64();
        do {
          asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(lo) : "r"(smem_u32(&llbuf[par][q * 8 + 0])));
          asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(hi) : "r"(smem_u32(&llbuf[par][q * 8 + 1])));
          if (clock64() - ts > 20000000ull) { out[1] = 1000 + t; break; }
        } while ((uint32_t)(lo >> 32) != flag || (uint32_t)(hi >> 32) != flag);
        v += __longlong_as_double((long long)(((hi & 0xFFFFFFFFull) << 32) | (lo & 0xFFFFFFFFull)));
      }
      acc += v;
    } else if (mode == 4) {
      // lane-parallel: lane l stores one double to CTA (l / 4), slot (l % 4)
      if (tid == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar[par])), "r"(bytes) : "memory");
      for (int l0 = lane; l0 < NC * 4; l0 += 32) {
        const int r = l0 >> 2, slot = l0 & 3;
        uint32_t a = mapa(&buf[par][(rank * NW + wid) * 4 + slot], r);
        uint32_t b = mapa(&mbar[par], r);
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(a), "d"(acc), "r"(b) : "memory");
      }
      asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(smem_u32(&mbar[par])), "r"((t >> 1) & 1) : "memory");
      acc += buf[par][lane];
    } else {
      __syncthreads();
      acc += buf[par][lane];
    }
  }
  unsigned long long t1 = clock64();
  if (tid == 0 && rank == 0) out[0] = (t1 - t0) / steps;
  if (acc == 12345.0) out[1] = 1;
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int mode = 0; mode < 6; ++mode)
    for (int nc : {1, 2, 4, 8, 16}) {
      if (mode == 3 && nc > 1) continue;
      if (mode == 4 && nc == 1) continue;
      if (mode < 4 && mode != 2) continue;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(nc);
      cfg.blockDim = dim3(256);
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = nc;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, kern, mode, 20000, d);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h[2];
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("mode %d NC %2d : %llu cycles/step %s flag=%llu\n", mode, nc, h[0], e ? cudaGetErrorString(e) : "", h[1]);
      fflush(stdout);
      cudaMemset(d, 0, 16);
    }
}
// (mode 4 added below via a second kernel)
