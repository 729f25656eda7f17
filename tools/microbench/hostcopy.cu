// Host-side costs of the drop-in path (pageable std::vector outputs): vector
// resize (zero fill + first-touch faults), memcpy from pinned staging, and the
// same split over threads; plus pinned vs pageable cudaMemcpy D2H rates.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include <cuda_runtime.h>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main() {
  const size_t bytes = 300u << 20;
  char* pinned; cudaMallocHost(&pinned, bytes);
  memset(pinned, 1, bytes);
  char* dev; cudaMalloc(&dev, bytes); cudaMemset(dev, 2, bytes);
  for (int rep = 0; rep < 2; ++rep) {
    double t = now(); std::vector<double> v; v.resize(bytes / 8); double t_resize = now() - t;
    t = now(); memcpy(v.data(), pinned, bytes); double t_copy = now() - t;
    t = now(); std::vector<double> w(pinned ? (const double*)pinned : nullptr, (const double*)(pinned + bytes)); double t_assign = now() - t;
    for (int nt : {4, 8, 16}) {
      std::vector<double> u; t = now(); u.resize(bytes / 8); double tr = now() - t;
      t = now();
      std::vector<std::thread> th;
      for (int i = 0; i < nt; ++i) th.emplace_back([&, i] { size_t a = bytes * i / nt, b = bytes * (i + 1) / nt; memcpy((char*)u.data() + a, pinned + a, b - a); });
      for (auto& x : th) x.join();
      printf("rep %d threads %d: resize %.1f ms, threaded copy %.1f ms\n", rep, nt, tr * 1e3, (now() - t) * 1e3);
    }
    t = now(); cudaMemcpy(pinned, dev, bytes, cudaMemcpyDeviceToHost); double t_pin = now() - t;
    std::vector<char> pg(bytes);
    t = now(); cudaMemcpy(pg.data(), dev, bytes, cudaMemcpyDeviceToHost); double t_pg = now() - t;
    t = now(); cudaMemcpy(dev, pg.data(), bytes, cudaMemcpyHostToDevice); double t_pgh = now() - t;
    t = now(); cudaMemcpy(dev, pinned, bytes, cudaMemcpyHostToDevice); double t_pinh = now() - t;
    printf("rep %d: resize %.1f ms, memcpy %.1f ms, assign %.1f ms | D2H pinned %.1f GB/s pageable %.1f GB/s | H2D pinned %.1f pageable %.1f GB/s\n",
           rep, t_resize * 1e3, t_copy * 1e3, t_assign * 1e3, bytes / t_pin / 1e9, bytes / t_pg / 1e9, bytes / t_pinh / 1e9, bytes / t_pgh / 1e9);
  }
  printf("hardware threads %u\n", std::thread::hardware_concurrency());
}
