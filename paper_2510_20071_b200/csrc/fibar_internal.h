// fibar_internal.h -- host-side declarations shared by the .cu files.
#pragma once
#include <cuda_runtime.h>
#include <string>
#include <vector>

namespace fibar {

// error reporting behind fibar_last_error (thread-local message + FIBAR_E_* code)
extern thread_local std::string g_err;
int fail(int code, const std::string &msg);
int cuda_fail(cudaError_t e, const char *where);

#define CK(call)                                          \
  do {                                                    \
    cudaError_t _e = (call);                              \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);   \
  } while (0)

// Stream + launch counter (the bench reports how many of our kernels ran) and
// an optional per-kernel CUDA-event profiler (bench.py's roofline leg).
struct Launcher {
  cudaStream_t stream = nullptr;
  long long launches = 0;
  bool prof = false;
  struct Rec {
    const char *name;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  void count() { ++launches; }
  cudaEvent_t ev() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
  void begin(const char *name) {
    ++launches;
    if (!prof) return;
    Rec r{name, ev(), ev()};
    cudaEventRecord(r.a, stream);
    recs.push_back(r);
  }
  void end() {
    if (!prof) return;
    cudaEventRecord(recs.back().b, stream);
  }
};

#define FIBAR_LAUNCH(L, name, ...) \
  do {                             \
    (L).begin(name);               \
    __VA_ARGS__;                   \
    (L).end();                     \
  } while (0)

int radix_sort_pairs(Launcher &L, unsigned *k_a, unsigned *v_a, unsigned *k_b, unsigned *v_b, unsigned *hist,
                     const long long *n_dev, long long n_max, int bits);

void scan_exclusive_u32(Launcher &L, unsigned *a, int len);
void scan_exclusive_large(Launcher &L, const unsigned *in, unsigned *out, const long long *n_dev, long long n_fixed,
                          long long n_max, unsigned *part);

}  // namespace fibar
