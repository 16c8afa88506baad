// devcache.h -- per-device, thread-safe cache of a launcher's one-time setup
// (the cudaFuncSetAttribute opt-in of dynamic shared memory and the resident
// CTAs per SM from the occupancy calculator).  Both bind to the CURRENT
// device, so a process that drives several GPUs (or switches devices between
// calls) must run the setup once per device, not once per process.
// Host code only; product code (the oracle never sees it).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>

namespace rsa_b200 {

constexpr int kMaxDevices = 64;

struct OccCache {
    std::atomic<int> occ[kMaxDevices];   // 0 = not set up on that device yet
    std::mutex mu;
};

// *occ_out = resident CTAs per SM of the launcher on the current device,
// running `setup(int* occ)` (attribute + occupancy query) the first time this
// device is seen.  Nothing is cached when setup fails, so a retry repeats it.
template <typename Setup>
static inline cudaError_t cached_occupancy(OccCache& c, Setup&& setup, int* occ_out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    int v = c.occ[dev].load(std::memory_order_acquire);
    if (v > 0) {
        *occ_out = v;
        return cudaSuccess;
    }
    std::lock_guard<std::mutex> lk(c.mu);
    v = c.occ[dev].load(std::memory_order_acquire);
    if (v <= 0) {
        int o = 0;
        e = setup(&o);
        if (e != cudaSuccess) return e;
        v = o < 1 ? 1 : o;
        c.occ[dev].store(v, std::memory_order_release);
    }
    *occ_out = v;
    return cudaSuccess;
}

// the usual setup: opt the kernel into `smem` bytes of dynamic shared memory
// (if any) and query its occupancy at `block` threads
template <typename K>
static inline cudaError_t occupancy_with_smem(K kernel, int block, size_t smem, int* occ_out) {
    if (smem) {
        cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ_out, kernel, block, smem);
}

// cudaFuncSetAttribute-only setup (kernels launched with a fixed grid)
struct AttrCache {
    std::atomic<bool> done[kMaxDevices];
    std::mutex mu;
};

template <typename Setup>
static inline cudaError_t cached_attr(AttrCache& c, Setup&& setup) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
    if (c.done[dev].load(std::memory_order_acquire)) return cudaSuccess;
    std::lock_guard<std::mutex> lk(c.mu);
    if (c.done[dev].load(std::memory_order_acquire)) return cudaSuccess;
    e = setup();
    if (e != cudaSuccess) return e;
    c.done[dev].store(true, std::memory_order_release);
    return cudaSuccess;
}

}  // namespace rsa_b200
