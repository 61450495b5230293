// Read-bandwidth probe (diagnostics, not product): how fast can a plain kernel stream a
// mid-size column set from a cold L2?  sum of uint4 loads, grid-stride, U loads in flight per
// thread; one atomicAdd per block so the loads cannot be elided.
#include <cuda_runtime.h>
#include <cstdint>

template <int U>
__global__ void __launch_bounds__(1024) read_kernel(const uint4* __restrict__ p, int64_t n16, unsigned long long* out) {
  unsigned long long acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n16; i += stride) { uint4 v = __ldcs(p + i); acc += v.x ^ v.y ^ v.z ^ v.w; }
  for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, d);
  __shared__ unsigned long long s[32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
    if (t == 0x123456789ull) atomicAdd(out, t);  // (practically never: keeps the loads live)
  }
}

extern "C" int read_probe(const void* p, int64_t bytes, void* out, int blocks, int threads, int unroll, void* stream) {
  const int64_t n16 = bytes / 16;
  cudaStream_t st = (cudaStream_t)stream;
  switch (unroll) {
    case 1: read_kernel<1><<<blocks, threads, 0, st>>>((const uint4*)p, n16, (unsigned long long*)out); break;
    case 4: read_kernel<4><<<blocks, threads, 0, st>>>((const uint4*)p, n16, (unsigned long long*)out); break;
    default: read_kernel<8><<<blocks, threads, 0, st>>>((const uint4*)p, n16, (unsigned long long*)out); break;
  }
  return (int)cudaGetLastError();
}
