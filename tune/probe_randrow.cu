// Random 128-byte row gather throughput on B200 (the access pattern of the
// MTTKRP factor gathers): every 8-lane group reads float4 slices of K rows
// chosen uniformly at random from a `rows` x 32 fp32 matrix, sums them (so
// the loads are live) and writes one float per group. Reports GB/s of row
// bytes for several in-flight depths K and grid shapes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tune/probe_randrow tune/probe_randrow.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

template <int K>
__global__ void gather(const float4* __restrict__ f, uint32_t rows, uint32_t iters, float* out,
                       uint32_t seed) {
  const uint32_t lane = threadIdx.x & 31, q = lane & 7;
  const uint32_t grp = (blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  float4 acc = make_float4(0, 0, 0, 0);
  uint32_t h = hash32(grp * 0x9E3779B9u + seed);
  for (uint32_t it = 0; it < iters; ++it) {
    float4 v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      h = hash32(h + k);
      const uint32_t r = (uint32_t)(((uint64_t)h * rows) >> 32);
      v[k] = __ldg(f + (size_t)r * 8 + q);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) acc.x += v[k].x, acc.y += v[k].y, acc.z += v[k].z, acc.w += v[k].w;
  }
  if (acc.x == 12345.f) out[grp] = acc.y + acc.z + acc.w;
}

template <int K>
void run(const float4* f, uint32_t rows, int blocks, int threads, float* out) {
  const uint32_t iters = 64;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  gather<K><<<blocks, threads>>>(f, rows, iters, out, 1);
  cudaEventRecord(a);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) gather<K><<<blocks, threads>>>(f, rows, iters, out, 7 + r);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = (double)blocks * threads / 8 * iters * K * 128 * reps;
  printf("K=%2d grid=%6d x %4d  rows=%u (%.2f GB)  %.1f GB/s\n", K, blocks, threads, rows,
         rows * 128.0 / 1e9, bytes / (ms * 1e-3) / 1e9);
}

int main() {
  const uint32_t rows = 20000000;  // 2.56 GB: two C5 factors
  float4* f;
  float* out;
  cudaMalloc(&f, (size_t)rows * 128);
  cudaMalloc(&out, 1 << 24);
  cudaMemset(f, 0, (size_t)rows * 128);
  for (int threads : {256, 512}) {
    for (int per_sm : {2, 4, 8}) {
      const int blocks = 148 * per_sm * 512 / threads / 2;
      run<4>(f, rows, blocks, threads, out);
      run<8>(f, rows, blocks, threads, out);
      run<16>(f, rows, blocks, threads, out);
    }
  }
  // small (L2-resident) table for comparison
  run<8>(f, 500000, 148 * 4, 512, out);
  return 0;
}
