// memcpy bandwidth into cudaMallocHost (pinned) memory with 1..16 threads.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main() {
  const size_t n = size_t(32) << 20;
  char* a = (char*)malloc(n * 8); memset(a, 1, n * 8);
  char* p; cudaMallocHost(&p, n);
  for (int t : {1, 4, 8, 16}) {
    double t0 = now();
    for (int r = 0; r < 20; ++r) {
#pragma omp parallel for num_threads(t) schedule(static)
      for (long i = 0; i < 32; ++i) memcpy(p + (i << 20), a + ((r % 8) * n) + (i << 20), 1 << 20);
    }
    printf("to pinned threads=%2d  %.1f GB/s\n", t, 20.0 * n / (now() - t0) / 1e9);
  }
  char* h; cudaHostAlloc(&h, n, cudaHostAllocPortable);
  double t0 = now();
  for (int r = 0; r < 20; ++r) {
#pragma omp parallel for num_threads(8) schedule(static)
    for (long i = 0; i < 32; ++i) memcpy(h + (i << 20), a + (i << 20), 1 << 20);
  }
  printf("to hostalloc(portable) 8 threads  %.1f GB/s\n", 20.0 * n / (now() - t0) / 1e9);
  return 0;
}
