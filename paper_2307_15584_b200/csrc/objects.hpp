// objects.hpp — the opaque ABI handles (qmc_matrices, qmc_xor_tables) and
// the fill/stream helpers the ABI translation units share.
#pragma once

#include "host.hpp"

#include <map>

using qmcgpu::host::brev_host;
using qmcgpu::host::current_device;
using qmcgpu::host::dev_upload;
using qmcgpu::host::DevPtr;

struct qmc_matrices {
    uint32_t dims;
    std::vector<uint32_t> columns; // [dims][52]
    std::mutex mu;
    struct Dev {
        DevPtr colsT, colsT_rev;
    };
    // per (device, dims prefix): the k-major column tables the kernels read
    std::map<std::pair<int, uint32_t>, std::unique_ptr<Dev>> dev;

    // [52][prefix] (and bit-reversed) columns of the first `prefix`
    // dimensions on the current device; built once, then cached.
    const Dev& on_device(uint32_t prefix)
    {
        const int d = current_device();
        std::lock_guard<std::mutex> lk(mu);
        auto& slot = dev[{d, prefix}];
        if (!slot) {
            const uint32_t pd = std::max<uint32_t>(prefix, 8); // room for 32-B loads
            std::vector<uint32_t> t(52 * static_cast<size_t>(pd), 0u), tr(t.size(), 0u);
            for (uint32_t j = 0; j < prefix; ++j)
                for (uint32_t k = 0; k < 52; ++k) {
                    t[k * static_cast<size_t>(prefix) + j] = columns[j * 52 + k];
                    tr[k * static_cast<size_t>(prefix) + j] = brev_host(columns[j * 52 + k]);
                }
            auto e = std::make_unique<Dev>();
            e->colsT = dev_upload(t.data(), t.size() * 4);
            e->colsT_rev = dev_upload(tr.data(), tr.size() * 4);
            slot = std::move(e);
        }
        return *slot;
    }
    const Dev& on_device() { return on_device(dims); }
};

// XOR-table sampler data (imageplane.hpp:92-120): 128x128 reorder words,
// 128x128xdims scramble words and the stored integer-stage point set.
// Immutable; the device copy is built once per GPU.
struct qmc_xor_tables {
    uint32_t dims = 0, point_count = 0;
    std::vector<uint32_t> reorder, scramble; // host
    std::vector<uint32_t> points;            // host (loaded) — empty for white noise
    std::vector<uint32_t> dim_scramble;      // white noise: per-dim XOR of the points
    bool white_noise = false;
    std::mutex mu;
    struct Dev {
        DevPtr reorder, scramble, points;
    };
    std::map<int, std::unique_ptr<Dev>> dev;

    // device copy on the current GPU, built once (abi_core.cpp)
    const Dev& on_device(cudaStream_t s);
};

namespace qmcgpu {
namespace host {

constexpr size_t kXorTile = 128 * 128;

// Device view of the tables a stream / render uses: the caller's handle, or
// white-noise tables made for this call.
struct XorTablesDev {
    uint32_t dims = 0, point_count = 0;
    const uint32_t *reorder = nullptr, *scramble = nullptr, *points = nullptr;
    std::unique_ptr<qmc_xor_tables> own;
};

// build_matrices(builtin_direction_numbers(), dims), cached per dims.
qmc_matrices* builtin_matrices(uint32_t dims);

// Sobol' fill of [first, first+n) x dims into `out` (device or host).
void sobol_fill_impl(qmc_matrices* m, uint64_t first, uint64_t n, uint32_t dims,
                     qmc_sobol_scramble sc, const uint32_t* words, qmc_output kind, void* out,
                     cudaStream_t s);

// white_noise_xor_tables (imageplane.cpp:197-229).
std::unique_ptr<qmc_xor_tables> make_white_noise(uint32_t dims, uint32_t point_count,
                                                 uint32_t seed);

// Device view of `given`, or of white-noise tables made for this call.
XorTablesDev xor_view(const qmc_xor_tables* given, uint32_t dims, uint32_t point_count,
                      uint32_t seed, cudaStream_t s);

} // namespace host
} // namespace qmcgpu
