// bw_probe.cu — practical HBM read ceiling on this B200 (what the K sweep could
// reach): plain 128-bit loads vs. cp.async.bulk (TMA) streams into a
// shared-memory ring, over a 4 GiB buffer. Build: nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o bw_probe tools/bw_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int UNROLL>
__global__ void read_ldg(const uint4* __restrict__ p, size_t n, unsigned* out) {
  unsigned acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + (UNROLL - 1) * stride < n; i += UNROLL * stride) {
    uint4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const uint4* q = p + i + u * stride;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(q));
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n; i += stride) acc ^= p[i].x;
  if (acc == 0x12345678u) out[0] = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// one CTA per SM streams a contiguous slice through an NS-deep ring of CH-byte
// chunks; one thread produces, all warps consume (xor) and release
template <int NS, int CH>
__global__ void read_tma(const char* __restrict__ p, size_t bytes, unsigned* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)NS * CH);
  uint64_t* empty = full + NS;
  const size_t per = bytes / gridDim.x;
  const char* base = p + per * blockIdx.x;
  const int nchunks = (int)(per / CH);
  const int nw = blockDim.x / 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[s])), "r"(nw));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int q) {
    const int st = q % NS;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[st])), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(sm + (size_t)st * CH)), "l"(base + (size_t)q * CH), "r"(CH), "r"(smem_u32(&full[st])) : "memory");
  };
  if (threadIdx.x == 0)
    for (int q = 0; q < NS && q < nchunks; ++q) issue(q);
  unsigned acc = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int q = 0; q < nchunks; ++q) {
    const int st = q % NS;
    const uint32_t par = (q / NS) & 1;
    asm volatile("{ .reg .pred P; W%=: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W%=; }"
                 ::"r"(smem_u32(&full[st])), "r"(par) : "memory");
    const uint4* v = reinterpret_cast<const uint4*>(sm + (size_t)st * CH);
    for (int i = threadIdx.x; i < CH / 16; i += blockDim.x) {
      const uint4 x = v[i];
      acc ^= x.x ^ x.w;
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[st])) : "memory");
    if (warp == 0 && lane == 0 && q + NS < nchunks) {
      asm volatile("{ .reg .pred P; E%=: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra E%=; }"
                   ::"r"(smem_u32(&empty[st])), "r"(par) : "memory");
      issue(q + NS);
    }
    __syncwarp();
  }
  if (acc == 0x12345678u) out[0] = acc;
}

__global__ void copy_k(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
  const size_t bytes = size_t(4) << 30;
  char* buf;
  unsigned* out;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMalloc(&out, 4));
  CK(cudaMemset(buf, 1, bytes));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch, double traffic) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 8; ++r) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    printf("%-34s %8.3f ms  %8.1f GB/s  %s\n", name, best, traffic / best / 1e6, err == cudaSuccess ? "" : cudaGetErrorString(err));
  };
  const size_t n16 = bytes / 16;
  for (int mult : {1, 2, 4, 8}) {
    char nm[64];
    snprintf(nm, 64, "ldg.v4 unroll8 grid=%dxSM b512", mult);
    timeit(nm, [&] { read_ldg<8><<<sms * mult, 512>>>((const uint4*)buf, n16, out); }, (double)bytes);
    snprintf(nm, 64, "ldg.v4 unroll16 grid=%dxSM b256", mult);
    timeit(nm, [&] { read_ldg<16><<<sms * mult, 256>>>((const uint4*)buf, n16, out); }, (double)bytes);
  }
  {
    constexpr int NS = 6, CH = 32768;
    auto k = read_tma<NS, CH>;
    const int sm_b = NS * CH + 2 * NS * 8;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_b);
    timeit("tma bulk 6x32KB ring, 1 CTA/SM", [&] { k<<<sms, 256, sm_b>>>(buf, bytes, out); }, (double)bytes);
  }
  {
    constexpr int NS = 4, CH = 16384;
    auto k = read_tma<NS, CH>;
    const int sm_b = NS * CH + 2 * NS * 8;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_b);
    timeit("tma bulk 4x16KB ring, 2 CTA/SM", [&] { k<<<sms * 2, 256, sm_b>>>(buf, bytes, out); }, (double)bytes);
  }
  {
    constexpr int NS = 8, CH = 8192;
    auto k = read_tma<NS, CH>;
    const int sm_b = NS * CH + 2 * NS * 8;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm_b);
    timeit("tma bulk 8x8KB ring, 3 CTA/SM", [&] { k<<<sms * 3, 256, sm_b>>>(buf, bytes, out); }, (double)bytes);
  }
  {
    const size_t half = n16 / 2;
    timeit("copy (read+write bytes)", [&] { copy_k<<<sms * 8, 512>>>((const uint4*)buf, (uint4*)buf + half, half); },
           (double)bytes);
  }
  return 0;
}
