// HBM ceilings by access mix, measured with plain 16-byte loads/stores:
// read-only, copy (1:1), write-only and 1 read : 4 writes (the direct
// completion's mix: 2 reads, 8 writes per element of a chunk).
// Build + run: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/hbm_mix scripts/hbm_mix.cu && /tmp/hbm_mix
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_read(const uint4* __restrict__ a, size_t n, uint4* sink) {
  uint4 acc = {0, 0, 0, 0};
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldcs(a + i);
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) *sink = acc;
}
__global__ void k_copy(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(b + i, __ldcs(a + i));
}
__global__ void k_fill(uint4* __restrict__ b, size_t n) {
  const uint4 v = {1, 2, 3, 4};
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) __stcs(b + i, v);
}
__global__ void k_r1w4(const uint4* __restrict__ a, uint4* __restrict__ d0, uint4* __restrict__ d1,
                       uint4* __restrict__ d2, uint4* __restrict__ d3, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldcs(a + i);
    __stcs(d0 + i, v); __stcs(d1 + i, v); __stcs(d2 + i, v); __stcs(d3 + i, v);
  }
}

template <int U>
__global__ void k_fill_plain(uint4* __restrict__ b, size_t n) {
  const uint4 v = {1, 2, 3, 4};
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride * U)
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * stride < n) b[i + u * stride] = v;
}
template <int U>
__global__ void k_r1w4_plain(const uint4* __restrict__ a, uint4* __restrict__ d0, uint4* __restrict__ d1,
                             uint4* __restrict__ d2, uint4* __restrict__ d3, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = (i + u * stride < n) ? a[i + u * stride] : uint4{0, 0, 0, 0};
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * stride < n) {
        d0[i + u * stride] = v[u]; d1[i + u * stride] = v[u]; d2[i + u * stride] = v[u]; d3[i + u * stride] = v[u];
      }
  }
}

template <class F>
float best_ms(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int it = 0; it < 10; ++it) {
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  const size_t bytes = 1ull << 30, n = bytes / 16;   // 1 GiB per array
  uint4 *a, *b[4], *sink;
  cudaMalloc(&a, bytes);
  for (auto& p : b) cudaMalloc(&p, bytes);
  cudaMalloc(&sink, 16);
  cudaMemset(a, 1, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 8, block = 256;
  const double gb = 1e9;
  float t_r = best_ms([&] { k_read<<<grid, block>>>(a, n, sink); });
  float t_c = best_ms([&] { k_copy<<<grid, block>>>(a, b[0], n); });
  float t_w = best_ms([&] { k_fill<<<grid, block>>>(b[0], n); });
  float t_4 = best_ms([&] { k_r1w4<<<grid, block>>>(a, b[0], b[1], b[2], b[3], n); });
  for (int g : {4, 8, 16}) {
    const int gr = sms * g;
    float tf = best_ms([&] { k_fill_plain<4><<<gr, block>>>(b[0], n); });
    float t4 = best_ms([&] { k_r1w4_plain<4><<<gr, block>>>(a, b[0], b[1], b[2], b[3], n); });
    printf("{\"grid_per_sm\": %d, \"write_plain_GBps\": %.1f, \"r1w4_plain_GBps\": %.1f}\n", g,
           bytes / (tf * 1e-3) / gb, 5 * bytes / (t4 * 1e-3) / gb);
  }
  printf("{\"read_GBps\": %.1f, \"copy_GBps\": %.1f, \"write_GBps\": %.1f, \"r1w4_GBps\": %.1f, \"err\": \"%s\"}\n",
         bytes / (t_r * 1e-3) / gb, 2 * bytes / (t_c * 1e-3) / gb, bytes / (t_w * 1e-3) / gb,
         5 * bytes / (t_4 * 1e-3) / gb, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
