// host.hpp — host-side building blocks of libqmcgpu shared by the ABI
// translation units (abi_core.cpp, abi_render.cpp): error handling with the
// reference's exception classes mapped to qmc_status, the immutable tables
// the reference builds on the host (host_tables.cpp), and device-memory /
// output-placement helpers (host_runtime.cpp). No per-sample arithmetic.
#pragma once

#include "qmcgpu.h"

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "device.cuh" // RadicalDim (host-visible layout)
#include "internal.hpp"

namespace qmcgpu {
namespace host {

// ------------------------------------------------------------- errors

// Message of the last failing call on this thread (qmc_last_error()).
std::string& last_error();

struct Fail {
    qmc_status status;
    std::string msg;
};

[[noreturn]] inline void fail(qmc_status s, std::string msg) { throw Fail{s, std::move(msg)}; }

inline void cuda_ok(cudaError_t e, const char* what)
{
    if (e != cudaSuccess)
        fail(QMC_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// make_stream's ConfigError check (imageplane.cpp:296-302).
inline void require(bool ok, const char* what)
{
    if (!ok)
        fail(QMC_CONFIG, what);
}

// Runs f, mapping failures to a status and the thread-local message.
template <typename F>
qmc_status guard(F&& f)
{
    try {
        f();
        return QMC_OK;
    } catch (const Fail& e) {
        last_error() = e.msg;
        return e.status;
    } catch (const std::bad_alloc&) {
        last_error() = "out of host memory";
        return QMC_INTERNAL;
    } catch (const std::exception& e) {
        last_error() = e.what();
        return QMC_INTERNAL;
    }
}

// ------------------------------------------------- tables (host_tables.cpp)

constexpr uint32_t kPrimes = 1000;

struct PrimeTable {
    std::array<uint32_t, kPrimes> p{}, maxpow{};
    PrimeTable()
    {
        uint32_t found = 0;
        for (uint32_t c = 2; found < kPrimes; ++c) {
            bool prime = true;
            for (uint32_t k = 0; k < found && p[k] * p[k] <= c; ++k)
                if (c % p[k] == 0) {
                    prime = false;
                    break;
                }
            if (prime)
                p[found++] = c;
        }
        for (uint32_t k = 0; k < kPrimes; ++k) {
            uint64_t x = p[k];
            while (x * p[k] <= 0xffffffffull)
                x *= p[k];
            maxpow[k] = static_cast<uint32_t>(x);
        }
    }
};

const PrimeTable& primes();
uint32_t prime_at(uint32_t index);              // out_of_range like prime()
std::vector<uint32_t> faure(uint32_t b);        // radical.cpp:50-74

struct DirRow {
    uint32_t s, a;
    std::vector<uint32_t> m;
};

std::vector<DirRow> builtin_rows();                                  // sobol_data.cpp
std::vector<DirRow> parse_rows(const std::string& text);             // digitalnet.cpp:23-65
std::vector<uint32_t> build_columns(const std::vector<DirRow>& rows, uint32_t dims); // :79-109

uint32_t brev_host(uint32_t v);
uint32_t pixel_hash_host(uint32_t j, uint32_t px, uint32_t py);       // lattice.cpp:71-77
std::vector<uint32_t> lfsr(uint32_t seed, uint32_t dims);            // lattice.cpp:81-104
uint32_t hilbert_order(uint32_t w, uint32_t h);                      // render.cpp:28-34

struct HaltonEnum {
    uint32_t sx = 1, sy = 1, ex = 0, ey = 0;
    uint64_t stride = 1, crt_x = 0, crt_y = 0;
};

HaltonEnum halton_enum(uint32_t w, uint32_t h);                      // imageplane.cpp:80-98
uint64_t digit_reverse_host(uint64_t v, uint32_t base, uint32_t digits);
void hilbert_xy_host(uint64_t d, uint32_t order, uint32_t& x, uint32_t& y); // hilbert.hpp:59-78

struct DigitTable {
    const uint32_t* ptr = nullptr;
    uint32_t group = 0;
    // with_quotients: floor(T * 2^32 / group) per entry (the remainder
    // T * 2^32 mod group is -q * group mod 2^32)
    const uint32_t* qx = nullptr;
};

// Widest b^d-entry table (b^d <= max_entries) inverting d >= min_digits
// digits per step with the digit permutation of `mode`; cached per device.
// Random-access users (radical_fixed) keep tables L1-sized; the contiguous
// fills read theirs sequentially and take wider ones (fewer block crossings).
constexpr uint32_t kDigitTableMax = 4096;
constexpr uint32_t kFillTableMax = 65536;
DigitTable digit_table(uint32_t b, uint32_t mode, uint32_t factor, uint32_t min_digits = 2,
                       uint32_t max_entries = kDigitTableMax, bool with_quotients = false);
// floor(2^64 / b^D) for D = 0..32 (0 where b^D >= 2^32), on the current device
const uint64_t* pow_magic(uint32_t b);
// k_render's column order for an image `width` wide (kernels_render.cu).
const uint32_t* render_column_order(uint32_t width);
// phi_3 quotient tables of the render (kernels_render.cu, phi3_q).
const uint32_t* render_phi3_quotients();
constexpr uint32_t kRenderT3Q3Words = 2188 + 2 * 2187 + 2; // 16-B multiple
const uint32_t* render_t3q3();
std::vector<RadicalDim> radical_dims(uint32_t dims, uint32_t first_prime, qmc_radical_scramble sc,
                                     const uint32_t* factors, std::vector<uint32_t>& sigma_pool,
                                     std::vector<size_t>& sigma_off);

// ------------------------------------------------ runtime (host_runtime.cpp)

struct DevFree {
    void operator()(void* p) const { cudaFree(p); }
};
using DevPtr = std::unique_ptr<void, DevFree>;

DevPtr dev_upload(const void* host, size_t bytes);

int current_device();
void pool_keep_memory();
bool is_device_pointer(const void* p);
inline cudaStream_t as_stream(qmc_stream s) { return static_cast<cudaStream_t>(s); }

// NVTX range around a C-ABI entry point (SURVEY §5 tracing): visible in
// Nsight Systems / ncu --nvtx; header-only NVTX3, no cost without a tool.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// RAII: restores the calling thread's current device.
struct DeviceRestoreGuard {
    int prev = 0;
    DeviceRestoreGuard() { cuda_ok(cudaGetDevice(&prev), "cudaGetDevice"); }
    ~DeviceRestoreGuard() { cudaSetDevice(prev); }
    DeviceRestoreGuard(const DeviceRestoreGuard&) = delete;
    DeviceRestoreGuard& operator=(const DeviceRestoreGuard&) = delete;
};

// Small per-call parameter arrays, uploaded with one stream-ordered copy
// and released stream-ordered after the launches.
class CallArgs {
public:
    explicit CallArgs(cudaStream_t s) : s_(s) {}
    ~CallArgs()
    {
        if (dev_)
            cudaFreeAsync(dev_, s_);
    }
    // returns the byte offset of the array inside the blob (16-B aligned)
    size_t add(const void* p, size_t bytes)
    {
        const size_t off = (blob_.size() + 15) & ~size_t(15);
        blob_.resize(off + bytes);
        if (bytes)
            std::memcpy(blob_.data() + off, p, bytes);
        return off;
    }
    void upload()
    {
        if (blob_.empty())
            return;
        pool_keep_memory();
        cuda_ok(cudaMallocAsync(&dev_, blob_.size(), s_), "cudaMallocAsync");
        cuda_ok(cudaMemcpyAsync(dev_, blob_.data(), blob_.size(), cudaMemcpyHostToDevice, s_),
                "cudaMemcpyAsync args");
    }
    template <typename T>
    const T* at(size_t off) const
    {
        return reinterpret_cast<const T*>(static_cast<const char*>(dev_) + off);
    }

private:
    cudaStream_t s_;
    std::vector<char> blob_;
    void* dev_ = nullptr;
};

struct SmallStage {
    size_t off[2] = {SIZE_MAX, SIZE_MAX};
};

void set_small(SmallArgs& sa, SmallStage& st, int which, const uint32_t* host, uint32_t n,
               CallArgs& args);
void finish_small(SmallArgs& sa, const SmallStage& st, const CallArgs& args);

// Per-device resources for the host-output pipeline.
struct DeviceCtx {
    std::mutex mu;
    cudaStream_t streams[2] = {nullptr, nullptr};
    void* staging[2] = {nullptr, nullptr};
    size_t staging_bytes = 0;
};

DeviceCtx& device_ctx(int dev);

constexpr size_t kStagingBytes = size_t(64) << 20;

// Places a fill of n points x dims 32-bit words at `out`. launch(range, s)
// enqueues the kernels writing device memory.
template <typename Launch>
void place_fill(void* out, uint64_t first, uint64_t n, uint32_t dims, cudaStream_t s,
                Launch&& launch)
{
    if (n == 0 || dims == 0)
        return;
    if (!out)
        fail(QMC_INVALID_ARGUMENT, "output pointer is null");
    if (is_device_pointer(out)) {
        cuda_ok(launch(FillRange{first, n, out}, s), "kernel launch");
        return;
    }
    // host output: ordered after prior work on the caller's stream
    cuda_ok(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    DeviceCtx& ctx = device_ctx(current_device());
    std::lock_guard<std::mutex> lk(ctx.mu);
    if (!ctx.streams[0]) {
        for (auto& st : ctx.streams)
            cuda_ok(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
    }
    if (ctx.staging_bytes < kStagingBytes) {
        for (auto& b : ctx.staging) {
            if (b)
                cudaFree(b);
            cuda_ok(cudaMalloc(&b, kStagingBytes), "cudaMalloc staging");
        }
        ctx.staging_bytes = kStagingBytes;
    }
    const uint64_t row = static_cast<uint64_t>(dims) * 4;
    uint64_t chunk = std::max<uint64_t>(1, kStagingBytes / row);
    if (chunk > 4096)
        chunk &= ~uint64_t(4095); // keep chunk starts tile-aligned relative to `first`
    char* host = static_cast<char*>(out);
    uint64_t k = 0;
    for (uint64_t done = 0; done < n; done += chunk, ++k) {
        const uint64_t cnt = std::min(chunk, n - done);
        cudaStream_t st = ctx.streams[k & 1];
        cuda_ok(launch(FillRange{first + done, cnt, ctx.staging[k & 1]}, st), "kernel launch");
        cuda_ok(cudaMemcpyAsync(host + done * row, ctx.staging[k & 1], cnt * row,
                                cudaMemcpyDeviceToHost, st),
                "cudaMemcpyAsync D2H");
    }
    for (auto& st : ctx.streams)
        cuda_ok(cudaStreamSynchronize(st), "cudaStreamSynchronize");
}

// Device copy of a row-major float array (host arrays are staged and freed
// stream-ordered).
struct DevPoints {
    const float* ptr = nullptr;
    float* own = nullptr;
    cudaStream_t s;
    DevPoints(const float* p, uint64_t count, cudaStream_t st) : s(st)
    {
        if (is_device_pointer(p)) {
            ptr = p;
            return;
        }
        cuda_ok(cudaMallocAsync(&own, count * 4 + 4, s), "cudaMallocAsync");
        cuda_ok(cudaMemcpyAsync(own, p, count * 4, cudaMemcpyHostToDevice, s), "H2D");
        ptr = own;
    }
    ~DevPoints()
    {
        if (own)
            cudaFreeAsync(own, s);
    }
};

} // namespace host
} // namespace qmcgpu
