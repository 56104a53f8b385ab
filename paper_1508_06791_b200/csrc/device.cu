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

int max_active_clusters(const void *kernel, const cudaLaunchConfig_t *cfg) {
    // key: kernel, device, block, dynamic smem, cluster shape (the grid does not change the answer)
    static std::map<std::tuple<const void *, int, unsigned, size_t, unsigned, unsigned, unsigned>, int> cache;
    unsigned cx = 1, cy = 1, cz = 1;
    for (unsigned i = 0; i < cfg->numAttrs; ++i)
        if (cfg->attrs[i].id == cudaLaunchAttributeClusterDimension) {
            cx = cfg->attrs[i].val.clusterDim.x;
            cy = cfg->attrs[i].val.clusterDim.y;
            cz = cfg->attrs[i].val.clusterDim.z;
        }
    const auto key = std::make_tuple(kernel, current_device(), cfg->blockDim.x * cfg->blockDim.y * cfg->blockDim.z,
                                     cfg->dynamicSmemBytes, cx, cy, cz);
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kernel, cfg) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    cache[key] = n;
    return n;
}

}  // namespace jacc_k
