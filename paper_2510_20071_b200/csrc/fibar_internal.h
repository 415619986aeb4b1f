// fibar_internal.h -- host-side declarations shared by the .cu files.
#pragma once
#include <cuda_runtime.h>
#include <string>
#include <utility>
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
  bool pdl = true;   // programmatic dependent launch between consecutive kernels
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

// Launch with programmatic dependent launch (PDL): the next kernel on the
// stream is scheduled while this one drains, and waits in pdl_wait() (its
// first statement) until this one's memory is visible -- saving the launch
// gap between the ~40 dependent kernels of a batch.
template <typename... KArgs, typename... Args>
inline void fibar_launch(Launcher &L, const char *name, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                         cudaStream_t s, Args &&...args) {
  L.begin(name);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = L.pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  L.end();
}

// A launch of one thread-block cluster of grid.x CTAs (the kernel uses
// cluster barriers), with programmatic dependent launch like fibar_launch.
template <typename... KArgs, typename... Args>
inline void fibar_launch_cluster(Launcher &L, const char *name, void (*kern)(KArgs...), int ctas, dim3 block,
                                 size_t smem, cudaStream_t s, Args &&...args) {
  L.begin(name);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = ctas;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = L.pdl ? 2 : 1;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  L.end();
}

// first statement of every kernel launched by fibar_launch: wait until the
// previous kernel on the stream has completed and its writes are visible
// (a no-op for launches without the PDL attribute)
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef FIBAR_PDL_EARLY
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

int radix_sort_pairs(Launcher &L, unsigned *k_a, unsigned *v_a, unsigned *k_b, unsigned *v_b, unsigned *hist,
                     const long long *n_dev, long long n_max, int bits);

void scan_exclusive_u32(Launcher &L, unsigned *a, int len);
void scan_exclusive_large(Launcher &L, const unsigned *in, unsigned *out, const long long *n_dev, long long n_fixed,
                          long long n_max, unsigned *part);

}  // namespace fibar
