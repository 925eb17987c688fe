// TMA tile::gather4 semantics + throughput probe (B200, sm_100a).
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c)); }
__device__ __forceinline__ void expect(uint64_t* b, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t done;
  do { asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(done) : "r"(sa(b)), "r"(ph) : "memory"); } while (!done);
}
__device__ __forceinline__ void g4(const CUtensorMap* m, void* dst, uint64_t* bar, int c0, int r0, int r1, int r2, int r3) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
               :: "r"(sa(dst)), "l"(m), "r"(sa(bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3) : "memory");
}

__global__ void sem(const __grid_constant__ CUtensorMap m, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = sm + ((1024 - (sa(sm) & 1023)) & 1023);
  __shared__ uint64_t bar;
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) reinterpret_cast<float*>(s)[i] = -1.f;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  if (threadIdx.x == 0) {
    expect(&bar, 1024);
    g4(&m, s, &bar, 0, 5, 100, 7, 1000);
    g4(&m, s + 512, &bar, 0, 9, 10, 11, 3);
  }
  wait(&bar, 0);
  for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = reinterpret_cast<float*>(s)[i];
}

// throughput: each CTA, one thread issues gather4 of random rows into a ring of S stages x G gathers
template <int S, int G>
__global__ void thr(const __grid_constant__ CUtensorMap m, uint32_t rows_mask, uint32_t iters, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = sm + ((1024 - (sa(sm) & 1023)) & 1023);
  __shared__ uint64_t full[S], empty[S];
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 32); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      for (uint32_t it = 0; it < iters; ++it) {
        const int st = it % S; const uint32_t ph = (it / S) & 1;
        wait(&empty[st], ph ^ 1);
        expect(&full[st], G * 512);
        for (int g = 0; g < G; ++g) {
          uint32_t h = hash32(blockIdx.x * 1000003u + it * G + g);
          g4(&m, s + st * G * 512 + g * 512, &full[st], 0, h & rows_mask, (h >> 3) & rows_mask, (h * 7) & rows_mask, (h * 13) & rows_mask);
        }
      }
    }
  } else if (warp == 1) {
    float acc = 0.f;
    for (uint32_t it = 0; it < iters; ++it) {
      const int st = it % S; const uint32_t ph = (it / S) & 1;
      wait(&full[st], ph);
      acc += reinterpret_cast<float*>(s + st * G * 512)[lane];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[st])) : "memory");
    }
    if (acc == 1234.f) out[0] = acc;
  }
}

template <int S, int G, int W>
__global__ void thrw(const __grid_constant__ CUtensorMap m, uint32_t rows_mask, uint32_t iters, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s0 = sm + ((1024 - (sa(sm) & 1023)) & 1023);
  __shared__ uint64_t fullb[W][S], emptyb[W][S];
  if (threadIdx.x == 0) {
    for (int w = 0; w < W; ++w) for (int i = 0; i < S; ++i) { mbar_init(&fullb[w][i], 1); mbar_init(&emptyb[w][i], 32); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, pair = warp >> 1;
  uint64_t* full = fullb[pair]; uint64_t* empty = emptyb[pair];
  uint8_t* s = s0 + pair * S * G * 512;
  if ((warp & 1) == 0) {
    if (lane == 0) {
      for (uint32_t it = 0; it < iters; ++it) {
        const int st = it % S; const uint32_t ph = (it / S) & 1;
        wait(&empty[st], ph ^ 1);
        expect(&full[st], G * 512);
        for (int g = 0; g < G; ++g) {
          uint32_t h = hash32(blockIdx.x * 1000003u + pair * 7777u + it * G + g);
          g4(&m, s + st * G * 512 + g * 512, &full[st], 0, h & rows_mask, (h >> 3) & rows_mask, (h * 7) & rows_mask, (h * 13) & rows_mask);
        }
      }
    }
  } else {
    float acc = 0.f;
    for (uint32_t it = 0; it < iters; ++it) {
      const int st = it % S; const uint32_t ph = (it / S) & 1;
      wait(&full[st], ph);
      acc += reinterpret_cast<float*>(s + st * G * 512)[lane];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[st])) : "memory");
    }
    if (acc == 1234.f) out[0] = acc;
  }
}
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  EncodeFn enc; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const uint32_t R = 1u << 20;  // 1M rows x 128 B = 128 MB
  std::vector<float> h((size_t)R * 32);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (float)((i / 32) * 100 + (i % 32));
  float* d; cudaMalloc(&d, h.size() * 4); cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  float* out; cudaMalloc(&out, 4096);
  for (int sw = 0; sw < 2; ++sw)
    for (uint32_t boxr : {1u}) {
      CUtensorMap m; cuuint64_t dims[2] = {32, R}, str[1] = {128}; cuuint32_t box[2] = {32, boxr}, es[2] = {1, 1};
      CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      printf("swizzle=%d box rows=%u encode=%d\n", sw, boxr, (int)r);
      if (r) continue;
      cudaMemset(out, 0, 4096);
      sem<<<1, 128, 4096>>>(m, out);
      cudaError_t e = cudaDeviceSynchronize();
      if (e) { printf("  launch error %s\n", cudaGetErrorString(e)); return 1; }
      float o[256]; cudaMemcpy(o, out, 1024, cudaMemcpyDeviceToHost);
      for (int row = 0; row < 8; ++row) {
        printf("  smem row %d:", row);
        for (int c = 0; c < 8; ++c) printf(" %7.0f", o[row * 32 + c * 4]);
        printf("\n");
      }
    }
  // throughput
  CUtensorMap m; cuuint64_t dims[2] = {32, R}, str[1] = {128}; cuuint32_t box[2] = {32, 1}, es[2] = {1, 1};
  enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](auto kern, int S, int G, int ctas_per_sm, uint32_t mask, const char* nm) {
    const uint32_t iters = 2000;
    const int smem = S * G * 512 + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<sms * ctas_per_sm, 64, smem>>>(m, mask, 10, out);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    kern<<<sms * ctas_per_sm, 64, smem>>>(m, mask, iters, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double bytes = (double)sms * ctas_per_sm * iters * G * 512;
    printf("%-40s S=%d G=%d ctas/SM=%d: %.3f ms %.1f GB/s  (%.2f rows/clk/SM at 1.9GHz)  err=%s\n", nm, S, G, ctas_per_sm, ms,
           bytes / ms / 1e6, bytes / 128 / (ms * 1e-3) / sms / 1.9e9, cudaGetErrorString(cudaGetLastError()));
  };
  auto runw = [&](auto kern, int S, int G, int W, uint32_t mask, const char* nm) {
    const uint32_t iters = 2000;
    const int smem = W * S * G * 512 + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<sms, 64 * W, smem>>>(m, mask, 10, out);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    kern<<<sms, 64 * W, smem>>>(m, mask, iters, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double bytes = (double)sms * W * iters * G * 512;
    printf("%-40s S=%d G=%d W=%d: %.3f ms %.1f GB/s  (%.3f rows/clk/SM at 1.9GHz)  err=%s\n", nm, S, G, W, ms,
           bytes / ms / 1e6, bytes / 128 / (ms * 1e-3) / sms / 1.9e9, cudaGetErrorString(cudaGetLastError()));
  };
  runw(thrw<4, 8, 1>, 4, 8, 1, (1u << 19) - 1, "multi-issuer 64MB");
  runw(thrw<4, 8, 2>, 4, 8, 2, (1u << 19) - 1, "multi-issuer 64MB");
  runw(thrw<4, 8, 4>, 4, 8, 4, (1u << 19) - 1, "multi-issuer 64MB");
  runw(thrw<4, 8, 8>, 4, 8, 8, (1u << 19) - 1, "multi-issuer 64MB");
  runw(thrw<2, 8, 8>, 2, 8, 8, (1u << 19) - 1, "multi-issuer 64MB");
  runw(thrw<4, 4, 16>, 4, 4, 16, (1u << 19) - 1, "multi-issuer 64MB");
  run(thr<4, 8>, 4, 8, 1, (1u << 19) - 1, "gather4 64MB L2");
  run(thr<8, 8>, 8, 8, 1, (1u << 19) - 1, "gather4 64MB L2");
  run(thr<8, 16>, 8, 16, 1, (1u << 19) - 1, "gather4 64MB L2");
  run(thr<8, 8>, 8, 8, 2, (1u << 19) - 1, "gather4 64MB L2");
  run(thr<8, 16>, 8, 16, 2, (1u << 19) - 1, "gather4 64MB L2");
  run(thr<8, 16>, 8, 16, 1, (1u << 20) - 1, "gather4 128MB");
  return 0;
}
