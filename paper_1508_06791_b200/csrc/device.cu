// device.cu -- device queries shared by the launchers (thread-safe caches).
#include <atomic>
#include <map>
#include <mutex>
#include <tuple>

#include "kernels.h"

namespace jacc_k {

namespace {
int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}
std::mutex g_mu;
}  // namespace

int sm_count() {
    static std::atomic<int> cache[64];
    int dev = current_device();
    if (dev < 0 || dev >= 64) dev = 0;
    int n = cache[dev].load(std::memory_order_relaxed);
    if (!n) {
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
        cache[dev].store(n, std::memory_order_relaxed);
    }
    return n;
}

cudaError_t set_max_dyn_smem(const void *kernel, int bytes) {
    static std::map<std::tuple<const void *, int, int>, bool> done;
    const auto key = std::make_tuple(kernel, current_device(), bytes);
    std::lock_guard<std::mutex> lk(g_mu);
    if (done.count(key)) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done[key] = true;
    return e;
}

int blocks_per_sm(const void *kernel, int block, int dyn_smem) {
    static std::map<std::tuple<const void *, int, int, int>, int> cache;
    const auto key = std::make_tuple(kernel, current_device(), block, dyn_smem);
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, block, dyn_smem) != cudaSuccess || occ < 1) {
        cudaGetLastError();
        occ = 1;
    }
    cache[key] = occ;
    return occ;
}

}  // namespace jacc_k
