// Small device helpers shared by the kernels.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include <utility>

#include "plan.hpp"

namespace merit_dev {

// Diagnostic knobs (MERIT_CONV_DEBUG, MERIT_SAD_DBG, MERIT_MP_DEBUG) skip work,
// add host synchronisation or print: they exist only in a -DMERIT_DEV_DEBUG
// build, so the product library's results cannot depend on the environment.
// Tuning knobs (kernel variant, ring depths, launch shape) stay environment
// controlled: every setting is parity-tested to give identical results.
inline const char* debug_env(const char* name) {
#ifdef MERIT_DEV_DEBUG
  return getenv(name);
#else
  (void)name;
  return nullptr;
#endif
}

// MERIT_GRID_CAP=n caps a persistent kernel's grid at n CTAs (CTA pairs /
// quads count as one): every CTA then walks many scheduling units, which the
// parity tests use to cover ring-phase carry across units at small sizes.
inline int grid_cap(int grid) {
  if (const char* g = getenv("MERIT_GRID_CAP")) {
    const int c = atoi(g);
    if (c > 0 && grid > c) return c;
  }
  return grid;
}

inline merit_status launch_status(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_check(e, what);
  count_launch();
  note_kernel(what);
  return MERIT_OK;
}

inline int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel,
// size): keeps the per-launch host path short for microsecond-scale kernels.
cudaError_t set_smem_attr_impl(const void* fn, cudaFuncAttribute attr, int bytes);
template <typename K>
inline cudaError_t set_smem_attr(K kernel, cudaFuncAttribute attr, int bytes) {
  return set_smem_attr_impl(reinterpret_cast<const void*>(kernel), attr, bytes);
}

// ---------------------------------------------------------------- PDL --
// Programmatic dependent launch: consecutive MERIT launches on a stream may
// overlap their prologues.  Every PDL kernel executes pdl_wait() (PTX
// griddepcontrol.wait: the previous grid has completed and its memory is
// visible) before its first global load or store, so stream order is kept
// for any chain of launches; only work that touches no global data (barrier
// init, TMEM allocation, L2 prefetch hints) runs before it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// L2 prefetch hint of global bytes [p, p + bytes): no architectural effect,
// so it may precede pdl_wait() (L2 is the coherence point).
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
bool pdl_enabled();  // MERIT_PDL=0 disables

// Launch `kernel` with the PDL attribute (and an optional cluster shape).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              unsigned cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  unsigned n = 0;
  if (pdl_enabled()) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster_x > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster_x;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Clusters of `cluster_x` CTAs of this kernel that can be resident at once
// (cudaOccupancyMaxActiveClusters; 0 if the query fails).  A persistent grid
// of more clusters than this runs its surplus as a second wave.
template <typename... KArgs>
inline int max_active_clusters(void (*kernel)(KArgs...), dim3 block, size_t smem, unsigned cluster_x) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cluster_x * 64);
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = cluster_x;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

}  // namespace merit_dev
