// cub_sort.cu -- measurement only (DESIGN.md §8 "SORT vs CUB"): CUB
// DeviceRadixSort::SortKeys on a key set dumped by libthermo
// (THERMO_DUMP_KEYS), on the same bits the library's onesweep sorts
// ([8, 8 + prefix width)); best and mean of 5 timed runs after 2 warm-ups.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o cub_sort scripts/cub_sort.cu
//   ./cub_sort keys.bin
#include <cub/cub.cuh>
#include <cstdio>
#include <vector>

int main(int argc, char** argv) {
  if (argc < 2) return 1;
  FILE* f = fopen(argv[1], "rb");
  if (!f) return 1;
  unsigned long long hdr[2];
  if (fread(hdr, 8, 2, f) != 2) return 1;
  const size_t n = hdr[0];
  const int bits = (int)hdr[1];
  std::vector<unsigned long long> h(n);
  if (fread(h.data(), 8, n, f) != n) return 1;
  fclose(f);
  unsigned long long *a, *b;
  cudaMalloc(&a, n * 8);
  cudaMalloc(&b, n * 8);
  size_t tmp = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tmp, a, b, (int64_t)n, 8, 8 + bits);
  void* t = nullptr;
  cudaMalloc(&t, tmp);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f, sum = 0;
  for (int it = 0; it < 7; ++it) {
    cudaMemcpy(a, h.data(), n * 8, cudaMemcpyHostToDevice);
    cudaEventRecord(e0);
    cub::DeviceRadixSort::SortKeys(t, tmp, a, b, (int64_t)n, 8, 8 + bits);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (it >= 2) {
      best = ms < best ? ms : best;
      sum += ms;
    }
  }
  printf("{\"keys\": %zu, \"bits\": %d, \"cub_ms_best\": %.4f, \"cub_ms_mean\": %.4f, \"err\": \"%s\"}\n", n, bits, best,
         sum / 5, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
