// L2-hit gather bandwidth probe (B200): how fast can SMs pull random 128-byte
// rows out of an L2-resident buffer?  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__device__ __forceinline__ void ldg256(const float* p, float4& a, float4& b) {
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w) : "l"(p));
}
// 4 lanes per 128-B row, U rows per group in flight
template <int U>
__global__ void gather4(const float* __restrict__ buf, uint32_t rows_mask, uint32_t iters, float* out, uint32_t local) {
  const int lane = threadIdx.x & 31, j = lane & 3;
  const uint32_t grp = (blockIdx.x * blockDim.x + threadIdx.x) >> 2;
  float acc = 0.f;
  for (uint32_t it = 0; it < iters; ++it) {
    float4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint32_t r = hash32(grp * 7919u + it * U + u);
      if (local) r = (grp * 4 + (r & 1023)) ;  // nearby rows
      r &= rows_mask;
      ldg256(buf + (size_t)r * 32 + 8 * j, a[u], b[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += a[u].x + a[u].y + a[u].z + a[u].w + b[u].x + b[u].y + b[u].z + b[u].w;
  }
  if (acc == 12345.f) out[0] = acc;
}
template <int U>
__global__ void gather8(const float* __restrict__ buf, uint32_t rows_mask, uint32_t iters, float* out) {
  const int lane = threadIdx.x & 31, j = lane & 7;
  const uint32_t grp = (blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  float acc = 0.f;
  for (uint32_t it = 0; it < iters; ++it) {
    float4 a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint32_t r = hash32(grp * 7919u + it * U + u) & rows_mask;
      a[u] = __ldg(reinterpret_cast<const float4*>(buf + (size_t)r * 32 + 4 * j));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += a[u].x + a[u].y + a[u].z + a[u].w;
  }
  if (acc == 12345.f) out[0] = acc;
}
__global__ void copyk(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* buf; float* out;
  const size_t big = 1ull << 30;  // 1 GiB floats region for DRAM tests (4 GB)
  cudaMalloc(&buf, big * 4); cudaMalloc(&out, 64);
  cudaMemset(buf, 0, big * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](auto launch, double bytes, const char* name) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0); for (int i = 0; i < 5; ++i) launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("%-48s %8.3f ms  %8.1f GB/s\n", name, ms, bytes / ms / 1e6);
  };
  const uint32_t iters = 64;
  for (uint32_t mb : {16u, 32u, 64u, 96u, 4096u}) {
    const uint32_t rows = mb * 1024 * 1024 / 128;  // power of two
    for (int bpsm : {4, 8, 16}) {
      const int blocks = sms * bpsm, th = 256;
      const double groups4 = blocks * th / 4.0, groups8 = blocks * th / 8.0;
      char nm[128];
      snprintf(nm, sizeof nm, "gather4 U=4 %uMB blocks/SM=%d", mb, bpsm);
      timeit([&] { gather4<4><<<blocks, th>>>(buf, rows - 1, iters, out, 0); }, groups4 * iters * 4 * 128, nm);
      snprintf(nm, sizeof nm, "gather4 U=8 %uMB blocks/SM=%d", mb, bpsm);
      timeit([&] { gather4<8><<<blocks, th>>>(buf, rows - 1, iters / 2, out, 0); }, groups4 * iters * 4 * 128, nm);
      snprintf(nm, sizeof nm, "gather8 U=4 %uMB blocks/SM=%d", mb, bpsm);
      timeit([&] { gather8<4><<<blocks, th>>>(buf, rows - 1, iters, out); }, groups8 * iters * 4 * 128, nm);
    }
  }
  {
    const int blocks = sms * 8, th = 256;
    timeit([&] { gather4<4><<<blocks, th>>>(buf, (1u << 24) - 1, iters, out, 1); }, blocks * th / 4.0 * iters * 4 * 128, "gather4 local rows (L1-friendly)");
  }
  const size_t n4 = big / 4 / 2;  // float4 count of half the buffer
  timeit([&] { copyk<<<sms * 8, 512>>>(reinterpret_cast<float4*>(buf), reinterpret_cast<float4*>(buf) + n4, n4); },
         n4 * 32.0, "copy 2 GB -> 2 GB (DRAM)");
  return 0;
}
