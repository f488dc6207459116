// Host-side launch helpers shared by the translation units of libsrk: every
// per-kernel launch setting that depends on the device (the opt-in shared
// memory attribute, SM count, resident CTAs per SM) is cached per
// (device, kernel), so one process may drive several GPUs (the single-process
// multi-device layout of SURVEY §8e, or a caller that switches
// torch.cuda.set_device between plans).
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <tuple>
#include <utility>

inline int srk_current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

namespace srk_host {
inline std::mutex& mu() {
  static std::mutex m;
  return m;
}
inline std::map<std::pair<int, const void*>, int>& smem_set() {
  static std::map<std::pair<int, const void*>, int> m;
  return m;
}
inline std::map<std::tuple<int, const void*, int, int>, int>& occ() {
  static std::map<std::tuple<int, const void*, int, int>, int> m;
  return m;
}
inline std::map<int, int>& sms() {
  static std::map<int, int> m;
  return m;
}
}  // namespace srk_host

// cudaFuncAttributeMaxDynamicSharedMemorySize >= bytes on the current device,
// set once per (device, kernel) and only raised.  Set even below 48 KB: the
// default limit counts static shared memory too (a 48 KB dynamic ring plus an
// mbarrier needs the opt-in).
inline cudaError_t srk_ensure_smem(const void* fn, int bytes) {
  if (bytes <= 0) return cudaSuccess;
  const int dev = srk_current_device();
  std::lock_guard<std::mutex> lk(srk_host::mu());
  auto& m = srk_host::smem_set();
  auto it = m.find({dev, fn});
  if (it != m.end() && it->second >= bytes) return cudaSuccess;
  cudaError_t err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (err == cudaSuccess) m[{dev, fn}] = bytes;
  return err;
}

inline int srk_sm_count() {
  const int dev = srk_current_device();
  std::lock_guard<std::mutex> lk(srk_host::mu());
  auto& m = srk_host::sms();
  auto it = m.find(dev);
  if (it != m.end()) return it->second;
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  if (n < 1) n = 1;
  m[dev] = n;
  return n;
}

// resident CTAs per SM of fn (nt threads, smem dynamic bytes) on the current device
inline int srk_blocks_per_sm(const void* fn, int nt, int smem) {
  const int dev = srk_current_device();
  {
    std::lock_guard<std::mutex> lk(srk_host::mu());
    auto& m = srk_host::occ();
    auto it = m.find({dev, fn, nt, smem});
    if (it != m.end()) return it->second;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, nt, smem);
  if (per_sm < 1) per_sm = 1;
  std::lock_guard<std::mutex> lk(srk_host::mu());
  srk_host::occ()[{dev, fn, nt, smem}] = per_sm;
  return per_sm;
}

// Kernel launch with programmatic stream serialization (PDL, srk_common.cuh):
// the kernel may begin while the previous kernel of the stream finishes; it
// waits (pdl_wait) before touching data.
inline cudaLaunchConfig_t srk_pdl_config(dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                         cudaLaunchAttribute* attr) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}
inline cudaError_t srk_launch(const void* fn, dim3 grid, dim3 block, void** args, size_t smem, cudaStream_t st) {
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = srk_pdl_config(grid, block, smem, st, attr);
  return cudaLaunchKernelExC(&cfg, fn, args);
}
template <typename... KArgs, typename... Args>
inline cudaError_t srk_launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                Args&&... args) {
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = srk_pdl_config(grid, block, smem, st, attr);
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
