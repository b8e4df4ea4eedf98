// Host memcpy bandwidth with 1..16 OpenMP threads, fresh-page (first touch)
// cost, and pinned-buffer copies: the host side of the drop-in's transfers.
//   g++ -O2 -fopenmp -o tune/probe_hostcopy tune/probe_hostcopy.cpp
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <omp.h>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main() {
  const size_t n = size_t(512) << 20;
  char* a = (char*)malloc(n); char* b = (char*)malloc(n);
  memset(a, 1, n); memset(b, 2, n);
  for (int t : {1, 2, 4, 8, 16}) {
    double t0 = now();
    for (int r = 0; r < 4; ++r) {
#pragma omp parallel for num_threads(t) schedule(static)
      for (long i = 0; i < 512; ++i) memcpy(b + (i << 20), a + (i << 20), 1 << 20);
    }
    printf("memcpy threads=%2d  %.1f GB/s\n", t, 4.0 * n / (now() - t0) / 1e9);
  }
  double t0 = now();
  std::vector<unsigned> v(n / 4);
  printf("vector<unsigned>(n) value-init (fresh pages): %.2f GB/s\n", n / (now() - t0) / 1e9);
  t0 = now();
  char* c = (char*)malloc(n);
#pragma omp parallel for num_threads(8) schedule(static)
  for (long i = 0; i < 512; ++i) memset(c + (i << 20), 0, 1 << 20);
  printf("parallel first touch 8 threads: %.2f GB/s\n", n / (now() - t0) / 1e9);
  printf("omp_get_max_threads=%d\n", omp_get_max_threads());
  return (int)(v[7] + c[5] + b[3]);
}
