// host_runtime.cpp — device-memory and output-placement helpers (host.hpp).
#include "host.hpp"

namespace qmcgpu {
namespace host {

std::string& last_error()
{
    thread_local std::string msg;
    return msg;
}

DevPtr dev_upload(const void* host, size_t bytes)
{
    void* d = nullptr;
    cuda_ok(cudaMalloc(&d, bytes ? bytes : 16), "cudaMalloc");
    DevPtr p(d);
    if (bytes)
        cuda_ok(cudaMemcpy(d, host, bytes, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
    return p;
}

// Fills SmallArgs array `which` (0 = a, 1 = b) by value when it fits the
// parameter space, else stages a device copy through `args`; the device
// address is patched in by finish_small after the upload.
void set_small(SmallArgs& sa, SmallStage& st, int which, const uint32_t* host, uint32_t n,
               CallArgs& args)
{
    if (n <= kSmall) {
        std::memcpy(which ? sa.b : sa.a, host, n * 4);
        (which ? sa.has_b : sa.has_a) = 1;
        return;
    }
    std::vector<uint32_t> pad(std::max<uint32_t>(n, 8) + 8, 0u); // room for 32-B loads
    std::memcpy(pad.data(), host, n * 4);
    st.off[which] = args.add(pad.data(), pad.size() * 4);
}

void finish_small(SmallArgs& sa, const SmallStage& st, const CallArgs& args)
{
    if (st.off[0] != SIZE_MAX) {
        sa.dev_a = args.at<uint32_t>(st.off[0]);
        sa.has_a = 1;
    }
    if (st.off[1] != SIZE_MAX) {
        sa.dev_b = args.at<uint32_t>(st.off[1]);
        sa.has_b = 1;
    }
}

DeviceCtx& device_ctx(int dev)
{
    static std::mutex mu;
    static std::vector<std::unique_ptr<DeviceCtx>> ctxs;
    std::lock_guard<std::mutex> lk(mu);
    if (ctxs.size() <= static_cast<size_t>(dev))
        ctxs.resize(dev + 1);
    if (!ctxs[dev])
        ctxs[dev] = std::make_unique<DeviceCtx>();
    return *ctxs[dev];
}

int current_device()
{
    int dev = 0;
    cuda_ok(cudaGetDevice(&dev), "cudaGetDevice");
    return dev;
}

// Keep up to kPoolKeepBytes of the stream-ordered pool cached across
// synchronizations, so the per-call argument blobs (cudaMallocAsync) never
// remap physical memory in a timed loop (the default release threshold of 0
// returns it at every sync, which cost milliseconds per call). The bound keeps
// large user-sized scratch (host-output render/fill chunks, scene_value,
// quality-metric points) from staying reserved against torch's allocator.
constexpr uint64_t kPoolKeepBytes = 256ull << 20;

void pool_keep_memory()
{
    static std::mutex mu;
    static std::vector<char> done;
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(mu);
    if (done.size() <= static_cast<size_t>(dev))
        done.resize(dev + 1, 0);
    if (done[dev])
        return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = kPoolKeepBytes;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    done[dev] = 1;
}

bool is_device_pointer(const void* p)
{
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

} // namespace host
} // namespace qmcgpu
