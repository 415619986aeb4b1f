// fibar_internal.h -- host-side declarations shared by the .cu files.
#pragma once
#include <cuda_runtime.h>

namespace fibar {

// Stream + launch counter (the bench reports how many of our kernels ran).
struct Launcher {
  cudaStream_t stream = nullptr;
  long long launches = 0;
  void count() { ++launches; }
};

int radix_sort_pairs(Launcher &L, unsigned *k_a, unsigned *v_a, unsigned *k_b, unsigned *v_b, unsigned *hist,
                     const long long *n_dev, long long n_max, int bits);

void scan_exclusive_u32(Launcher &L, unsigned *a, int len);

}  // namespace fibar
