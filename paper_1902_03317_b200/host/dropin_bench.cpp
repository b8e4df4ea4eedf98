// End-to-end timing of the C++ drop-in (spten::gpu::*, include/spten/gpu.hpp)
// on host SparseTensorCOO<float> / DenseMatrix<float> data -- the call a user
// of the reference library makes after swapping spten::seq:: for spten::gpu::
// (P/include/spten/kernels_seq.hpp:18-61). Every call uploads its operands
// from the caller's std::vectors, runs the sm_100a kernels and returns its
// result by value, so the timed step includes all host <-> device traffic.
//
//   dropin_bench <dir> <c1|c2|c5> <steps> <warmup>
// <dir> holds the workload's arrays as .npy files (written by bench.py);
// prints one JSON object: mean / median ms per step, bytes up and down.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <malloc.h>
#include <stdexcept>
#include <string>
#include <vector>

#include "spten/gpu.hpp"

using namespace spten;
extern "C" double spten_gpu_copy_probe(const void* src, size_t n);

namespace {

// Minimal .npy reader (little-endian u4 / f4, C order).
template <typename T>
std::vector<T> load_npy(const std::string& path, std::vector<size_t>* shape = nullptr) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open " + path);
  char magic[6];
  in.read(magic, 6);
  uint8_t ver[2];
  in.read(reinterpret_cast<char*>(ver), 2);
  uint32_t hlen = 0;
  if (ver[0] == 1) {
    uint16_t h;
    in.read(reinterpret_cast<char*>(&h), 2);
    hlen = h;
  } else {
    in.read(reinterpret_cast<char*>(&hlen), 4);
  }
  std::string header(hlen, ' ');
  in.read(header.data(), hlen);
  const auto lp = header.find('('), rp = header.find(')');
  std::vector<size_t> shp;
  size_t count = 1;
  for (size_t i = lp + 1; i < rp;) {
    while (i < rp && (header[i] == ' ' || header[i] == ',')) ++i;
    if (i >= rp) break;
    size_t v = 0;
    while (i < rp && header[i] >= '0' && header[i] <= '9') v = v * 10 + (header[i++] - '0');
    shp.push_back(v);
    count *= v;
  }
  if (shape) *shape = shp;
  std::vector<T> data(count);
  in.read(reinterpret_cast<char*>(data.data()), count * sizeof(T));
  if (!in) throw std::runtime_error("short read " + path);
  return data;
}

SparseTensorCOO<float> load_coo(const std::string& dir, const std::string& prefix,
                                const std::vector<Index>& dims,
                                std::vector<unsigned> sort_order) {
  SparseTensorCOO<float> t;
  t.dims = dims;
  for (size_t d = 0; d < dims.size(); ++d)
    t.indices.push_back(load_npy<uint32_t>(dir + "/" + prefix + "i" + std::to_string(d) + ".npy"));
  t.values = load_npy<float>(dir + "/" + prefix + "val.npy");
  t.sort_order = sort_order;
  t.coalesced = true;
  return t;
}

DenseMatrix<float> load_mat(const std::string& path) {
  std::vector<size_t> shp;
  auto v = load_npy<float>(path, &shp);
  DenseMatrix<float> m(shp.at(0), shp.at(1));
  m.data = std::move(v);
  return m;
}

std::vector<Index> read_dims(const std::string& dir) {
  std::ifstream in(dir + "/meta.json");
  std::string s((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  const auto k = s.find("\"dims\"");
  const auto a = s.find('[', k), b = s.find(']', a);
  std::vector<Index> dims;
  for (size_t i = a + 1; i < b;) {
    while (i < b && (s[i] < '0' || s[i] > '9')) ++i;
    if (i >= b) break;
    uint64_t v = 0;
    while (i < b && s[i] >= '0' && s[i] <= '9') v = v * 10 + (s[i++] - '0');
    dims.push_back(static_cast<Index>(v));
  }
  return dims;
}

double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

}  // namespace

int run(int argc, char** argv);

int main(int argc, char** argv) {
  try {
    return run(argc, argv);
  } catch (const std::exception& e) {
    std::printf("{\"error\": \"%s\"}\n", e.what());
    return 1;
  }
}

int run(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: %s <dir> <c1|c2|c5> <steps> <warmup>\n", argv[0]);
    return 2;
  }
  // The app's allocator policy (not the library's): the by-value outputs of
  // the reference API are hundreds of MB; glibc would mmap each one afresh and
  // fault every page in on its single-threaded zero-fill (~2.7 GB/s on the
  // box). From the heap, with trimming off, freed outputs are reused.
  mallopt(M_MMAP_MAX, 0);
  mallopt(M_TRIM_THRESHOLD, -1);
  const std::string dir = argv[1], wl = argv[2];
  const int steps = std::atoi(argv[3]), warmup = std::atoi(argv[4]);
  const std::vector<Index> dims = read_dims(dir);
  const unsigned N = static_cast<unsigned>(dims.size());
  std::vector<unsigned> asc(N);
  for (unsigned d = 0; d < N; ++d) asc[d] = d;

  // one step = the workload's ops through spten::gpu::, results by value
  std::function<void(double&, double&, double&)> step;
  SparseTensorCOO<float> x, y, y2;
  std::vector<DenseMatrix<float>> fs;
  uint64_t units = 0;
  if (wl == "c1") {
    x = load_coo(dir, "x_", dims, asc);
    for (unsigned d = 0; d < N; ++d) fs.push_back(load_mat(dir + "/f" + std::to_string(d) + ".npy"));
    units = 3 * x.nnz();
    step = [&](double& up, double& down, double& chk) {
      auto m = gpu::mttkrp(x, fs, 0);
      auto a = gpu::ts(x, 2.5f, ScalarOp::add);
      auto b = gpu::ts(x, 2.5f, ScalarOp::mul);
      const double t = x.nnz() * 4.0 * (N + 1);
      double fb = 0;
      for (unsigned d = 1; d < N; ++d) fb += fs[d].data.size() * 4.0;
      up += 3 * t + fb;
      down += m.data.size() * 4.0 + 2 * t;
      chk += m.data[0] + a.values.back() + b.values.back();
    };
  } else if (wl == "c2") {
    x = load_coo(dir, "x_", dims, asc);
    y = x;
    y.values = load_npy<float>(dir + "/yval.npy");
    y2 = load_coo(dir, "y2_", dims, asc);
    units = 4 * x.nnz() + 2 * (x.nnz() + y2.nnz());
    step = [&](double& up, double& down, double& chk) {
      const double t = x.nnz() * 4.0 * (N + 1);
      for (int op = 0; op < 4; ++op) {
        auto z = gpu::tew_eq(x, y, static_cast<ElemOp>(op));
        up += 2 * t;
        down += t;
        chk += z.values[0];
      }
      for (ElemOp op : {ElemOp::add, ElemOp::mul}) {
        auto z = gpu::tew(x, y2, op);  // both share the ascending order: no re-sort
        up += t + y2.nnz() * 4.0 * (N + 1);
        down += z.nnz() * 4.0 * (N + 1);
        chk += z.nnz();
      }
    };
  } else if (wl == "c5") {
    x = load_coo(dir, "x_", dims, asc);
    y = x;
    y.values = load_npy<float>(dir + "/yval.npy");
    for (unsigned d = 0; d < N; ++d) fs.push_back(load_mat(dir + "/f" + std::to_string(d) + ".npy"));
    units = 4 * x.nnz();
    step = [&](double& up, double& down, double& chk) {
      const double t = x.nnz() * 4.0 * (N + 1);
      for (unsigned m = 0; m < N; ++m) {
        auto out = gpu::mttkrp(x, fs, m);
        double fb = 0;
        for (unsigned d = 0; d < N; ++d)
          if (d != m) fb += fs[d].data.size() * 4.0;
        up += t + fb;
        down += out.data.size() * 4.0;
        chk += out.data[0];
      }
      auto z = gpu::tew_eq(x, y, ElemOp::mul);
      up += 2 * t;
      down += t;
      chk += z.values[0];
    };
  } else {
    std::fprintf(stderr, "unknown workload %s\n", wl.c_str());
    return 2;
  }
  if (std::getenv("SPT_COPY_PROBE")) {
    std::vector<char> fresh(size_t(256) << 20, 1);
    std::fprintf(stderr, "copy probe: fresh %.1f GB/s, x.indices[0] %.1f GB/s, again %.1f GB/s\n",
                 spten_gpu_copy_probe(fresh.data(), fresh.size()),
                 spten_gpu_copy_probe(x.indices[0].data(), x.indices[0].size() * 4),
                 spten_gpu_copy_probe(x.indices[0].data(), x.indices[0].size() * 4));
  }
  double up = 0, down = 0, chk = 0;
  for (int i = 0; i < warmup; ++i) step(up, down, chk);
  std::vector<double> ms;
  for (int i = 0; i < steps; ++i) {
    up = down = 0;
    const double t0 = now_ms();
    step(up, down, chk);
    ms.push_back(now_ms() - t0);
  }
  std::vector<double> sorted = ms;
  std::sort(sorted.begin(), sorted.end());
  double mean = 0;
  for (double v : ms) mean += v;
  mean /= ms.size();
  std::printf(
      "{\"path\": \"spten::gpu::* (C++ drop-in) on host SparseTensorCOO<float> / "
      "DenseMatrix<float>\", \"ms_per_step\": %.4f, \"ms_median\": %.4f, \"units_per_step\": "
      "%llu, \"h2d_bytes_per_step\": %.0f, \"d2h_bytes_per_step\": %.0f, \"checksum\": %.6g}\n",
      mean, sorted[sorted.size() / 2], static_cast<unsigned long long>(units), up, down, chk);
  return 0;
}
