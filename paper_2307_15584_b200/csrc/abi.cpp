// abi.cpp — the extern "C" boundary (include/qmcgpu.h) of libqmcgpu.
//
// Host responsibilities only: validate arguments with the reference's
// conditions (so callers see the same error classes), build the immutable
// tables the reference builds on the host (primes, direction-number
// matrices, Faure permutations, generator vectors, XOR tables), upload
// per-call parameters, place the output (device pointer: one asynchronous
// launch; host pointer: chunked device fill + D2H pipeline), and launch the
// kernels. No per-sample arithmetic happens here.
#include "qmcgpu.h"

#include <algorithm>
#include <array>
#include <map>
#include <tuple>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "device.cuh" // RadicalDim layout (host-visible struct)
#include "internal.hpp"

using namespace qmcgpu;

namespace {

// ------------------------------------------------------------- errors

thread_local std::string g_error;

struct Fail {
    qmc_status status;
    std::string msg;
};

[[noreturn]] void fail(qmc_status s, std::string msg) { throw Fail{s, std::move(msg)}; }

void cuda_ok(cudaError_t e, const char* what)
{
    if (e != cudaSuccess)
        fail(QMC_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename F>
qmc_status guard(F&& f)
{
    try {
        f();
        return QMC_OK;
    } catch (const Fail& e) {
        g_error = e.msg;
        return e.status;
    } catch (const std::bad_alloc&) {
        g_error = "out of host memory";
        return QMC_INTERNAL;
    } catch (const std::exception& e) {
        g_error = e.what();
        return QMC_INTERNAL;
    }
}

// ---------------------------------------------------------- prime table

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

const PrimeTable& primes()
{
    static const PrimeTable t;
    return t;
}

uint32_t prime_at(uint32_t index)
{
    if (index >= kPrimes)
        fail(QMC_OUT_OF_RANGE, "prime: index beyond the bundled prime table");
    return primes().p[index];
}

// radical.cpp:50-74
std::vector<uint32_t> faure(uint32_t b)
{
    if (b < 2)
        fail(QMC_INVALID_ARGUMENT, "faure_permutation: base must be >= 2");
    if (b == 2)
        return {0u, 1u};
    std::vector<uint32_t> s;
    s.reserve(b);
    if (b % 2 == 0) {
        const auto h = faure(b / 2);
        for (uint32_t v : h)
            s.push_back(2 * v);
        for (uint32_t v : h)
            s.push_back(2 * v + 1);
    } else {
        const auto prev = faure(b - 1);
        const uint32_t mid = (b - 1) / 2;
        for (uint32_t k = 0; k < prev.size(); ++k) {
            if (k == mid)
                s.push_back(mid);
            s.push_back(prev[k] >= mid ? prev[k] + 1 : prev[k]);
        }
    }
    return s;
}

// ------------------------------------------------- direction numbers

struct DirRow {
    uint32_t s, a;
    std::vector<uint32_t> m;
};

struct BuiltinRow {
    uint32_t s, a;
    uint32_t m[32];
};
const BuiltinRow kJoeKuo[] = {
#include "joe_kuo_64.inc"
};

std::vector<DirRow> builtin_rows()
{
    std::vector<DirRow> rows;
    for (const BuiltinRow& r : kJoeKuo)
        rows.push_back(DirRow{r.s, r.a, std::vector<uint32_t>(r.m, r.m + r.s)});
    return rows;
}

// digitalnet.cpp:23-65 — same grammar, checks and ConfigError messages.
std::vector<DirRow> parse_rows(const std::string& text)
{
    std::vector<DirRow> rows;
    std::istringstream in(text);
    std::string line;
    size_t no = 0;
    bool header = false;
    auto bad = [&](const std::string& w) {
        fail(QMC_CONFIG, "direction numbers, line " + std::to_string(no) + ": " + w);
    };
    while (std::getline(in, line)) {
        ++no;
        if (!header) {
            header = true;
            continue;
        }
        std::istringstream ls(line);
        uint32_t d = 0, s = 0, a = 0;
        if (!(ls >> d))
            continue;
        if (!(ls >> s >> a))
            bad("expected 'd s a m_1 ... m_s'");
        if (d != rows.size() + 2)
            bad("dimensions must be consecutive starting at 2");
        if (s == 0 || s > 32)
            bad("degree s out of range");
        if (s > 1 && a >= (1u << (s - 1)))
            bad("coefficient a has more than s-1 bits");
        DirRow row{s, a, {}};
        for (uint32_t k = 1; k <= s; ++k) {
            uint64_t mk = 0;
            if (!(ls >> mk))
                bad("expected " + std::to_string(s) + " direction numbers");
            if (mk % 2 == 0)
                bad("direction number m_" + std::to_string(k) + " is even");
            if (mk >= (1ull << k))
                bad("direction number m_" + std::to_string(k) + " must be < 2^" +
                    std::to_string(k));
            row.m.push_back(static_cast<uint32_t>(mk));
        }
        std::string rest;
        if (ls >> rest)
            bad("trailing tokens after the m values");
        rows.push_back(std::move(row));
    }
    return rows;
}

// digitalnet.cpp:79-109 — MSB-aligned columns, 52 per dimension.
std::vector<uint32_t> build_columns(const std::vector<DirRow>& rows, uint32_t dims)
{
    if (dims > rows.size() + 1)
        fail(QMC_CONFIG, "build_matrices: requested " + std::to_string(dims) +
                             " dimensions, direction numbers provide " +
                             std::to_string(rows.size() + 1));
    std::vector<uint32_t> c(static_cast<size_t>(dims) * 52, 0u);
    if (dims == 0)
        return c;
    for (uint32_t k = 0; k < 32; ++k)
        c[k] = 0x80000000u >> k;
    for (uint32_t j = 1; j < dims; ++j) {
        const DirRow& r = rows[j - 1];
        uint32_t* v = c.data() + static_cast<size_t>(j) * 52;
        for (uint32_t k = 0; k < r.s && k < 52; ++k)
            v[k] = r.m[k] << (31 - k);
        for (uint32_t k = r.s; k < 52; ++k) {
            uint32_t x = v[k - r.s] ^ (v[k - r.s] >> r.s);
            for (uint32_t l = 1; l < r.s; ++l)
                if ((r.a >> (r.s - 1 - l)) & 1u)
                    x ^= v[k - l];
            v[k] = x;
        }
    }
    return c;
}

uint32_t brev_host(uint32_t v)
{
    uint32_t r = 0;
    for (int k = 0; k < 32; ++k)
        r |= ((v >> k) & 1u) << (31 - k);
    return r;
}

// lattice.cpp:59-77
uint32_t fmix_host(uint32_t h)
{
    h = (h ^ (h >> 16)) * 0x85ebca6bu;
    h = (h ^ (h >> 13)) * 0xc2b2ae35u;
    return h ^ (h >> 16);
}
uint32_t pixel_hash_host(uint32_t j, uint32_t px, uint32_t py)
{
    return fmix_host(fmix_host(fmix_host(0x9e3779b9u ^ j) ^ px) ^ py);
}

std::vector<uint32_t> lfsr(uint32_t seed, uint32_t dims)
{
    if (seed == 0)
        fail(QMC_INVALID_ARGUMENT, "lfsr_generator_vector: zero seed is the absorbing state");
    if (dims < 1)
        fail(QMC_INVALID_ARGUMENT, "lfsr_generator_vector: dims must be >= 1");
    std::vector<uint32_t> g{1u};
    uint32_t x = seed;
    for (uint32_t j = 1; j < dims; ++j) {
        x ^= x << 13;
        x ^= x >> 17;
        x ^= x << 5;
        g.push_back(2u * x + 1u);
    }
    return g;
}

uint32_t hilbert_order(uint32_t w, uint32_t h)
{
    uint32_t o = 1;
    while (o < 32 && ((1ull << o) < w || (1ull << o) < h))
        ++o;
    return o;
}

// ------------------------------------------ Halton pixel enumeration

uint64_t inverse_mod(uint64_t a, uint64_t n)
{
    if (n == 1)
        return 0;
    int64_t r0 = static_cast<int64_t>(n), r1 = static_cast<int64_t>(a % n), t0 = 0, t1 = 1;
    while (r1) {
        const int64_t q = r0 / r1;
        const int64_t r2 = r0 - q * r1, t2 = t0 - q * t1;
        r0 = r1;
        r1 = r2;
        t0 = t1;
        t1 = t2;
    }
    const int64_t m = static_cast<int64_t>(n);
    return static_cast<uint64_t>(((t0 % m) + m) % m);
}

struct HaltonEnum {
    uint32_t sx = 1, sy = 1, ex = 0, ey = 0;
    uint64_t stride = 1, crt_x = 0, crt_y = 0;
};

// imageplane.cpp:80-98
HaltonEnum halton_enum(uint32_t w, uint32_t h)
{
    if (w == 0 || h == 0)
        fail(QMC_CONFIG, "HaltonPixelEnumeration: image must be at least 1x1");
    if (w > (1u << 20) || h > 1594323u)
        fail(QMC_CONFIG, "HaltonPixelEnumeration: image too large for the index range");
    HaltonEnum e;
    while (e.sx < w) {
        e.sx *= 2;
        ++e.ex;
    }
    while (e.sy < h) {
        e.sy *= 3;
        ++e.ey;
    }
    e.stride = static_cast<uint64_t>(e.sx) * e.sy;
    e.crt_x = e.sy * inverse_mod(e.sy % e.sx, e.sx);
    e.crt_y = e.sx * inverse_mod(e.sx % e.sy, e.sy);
    return e;
}

uint64_t digit_reverse_host(uint64_t v, uint32_t base, uint32_t digits)
{
    uint64_t r = 0;
    for (uint32_t k = 0; k < digits; ++k) {
        r = r * base + v % base;
        v /= base;
    }
    return r;
}

// ------------------------------------------------------ device buffers

struct DevFree {
    void operator()(void* p) const { cudaFree(p); }
};
using DevPtr = std::unique_ptr<void, DevFree>;

DevPtr dev_upload(const void* host, size_t bytes)
{
    void* d = nullptr;
    cuda_ok(cudaMalloc(&d, bytes ? bytes : 16), "cudaMalloc");
    DevPtr p(d);
    if (bytes)
        cuda_ok(cudaMemcpy(d, host, bytes, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
    return p;
}

// Small per-call parameter arrays, uploaded with one stream-ordered copy
// and released stream-ordered after the launches.
void pool_keep_memory();

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

// Fills SmallArgs array `which` (0 = a, 1 = b) by value when it fits the
// parameter space, else stages a device copy through `args`; the device
// address is patched in by finish_small after the upload.
struct SmallStage {
    size_t off[2] = {SIZE_MAX, SIZE_MAX};
};

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

// Per-device resources for the host-output pipeline.
struct DeviceCtx {
    std::mutex mu;
    cudaStream_t streams[2] = {nullptr, nullptr};
    void* staging[2] = {nullptr, nullptr};
    size_t staging_bytes = 0;
};

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

// Keep the stream-ordered pool's memory cached across synchronizations, so
// the per-call argument blobs (cudaMallocAsync) never remap physical memory
// in a timed loop (the default release threshold of 0 returns it at every
// sync, which cost milliseconds per call).
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
        uint64_t keep = UINT64_MAX;
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

cudaStream_t as_stream(qmc_stream s) { return static_cast<cudaStream_t>(s); }

// Multi-digit tables (tensor_digit_table, radical.cpp:76-110) on the device:
// d = the most base-b digits with b^d <= 4096 (so a table stays 16 KB and
// L1-resident), entry v = the d digits of v permuted by sigma and mirrored.
// Built once per (device, base, scramble) and kept for the process.
struct DigitTable {
    const uint32_t* ptr = nullptr;
    uint32_t group = 0;
};

constexpr uint32_t kDigitTableMax = 4096;

DigitTable digit_table(uint32_t b, uint32_t mode, uint32_t factor)
{
    static std::mutex mu;
    static std::map<std::tuple<int, uint32_t, uint32_t, uint32_t>, std::pair<DevPtr, uint32_t>>
        cache;
    uint32_t d = 0, group = 1;
    while (static_cast<uint64_t>(group) * b <= kDigitTableMax) {
        group *= b;
        ++d;
    }
    if (d < 2)
        return {};
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(mu);
    auto& slot = cache[{dev, b, mode, factor}];
    if (!slot.first) {
        std::vector<uint32_t> sigma(b);
        if (mode == 2) {
            sigma = faure(b);
        } else {
            for (uint32_t a = 0; a < b; ++a)
                sigma[a] = mode == 1 ? static_cast<uint32_t>((uint64_t(factor) * a) % b) : a;
        }
        std::vector<uint32_t> t(group + 8, 0u);
        for (uint32_t v = 0; v < group; ++v) {
            uint32_t rem = v, out = 0;
            for (uint32_t k = 0; k < d; ++k) {
                out = out * b + sigma[rem % b];
                rem /= b;
            }
            t[v] = out;
        }
        slot.first = dev_upload(t.data(), t.size() * 4);
        slot.second = group;
    }
    return {static_cast<const uint32_t*>(slot.first.get()), slot.second};
}

// RadicalDim table for `dims` prime bases (radical.cpp:130-181).
std::vector<RadicalDim> radical_dims(uint32_t dims, uint32_t first_prime, qmc_radical_scramble sc,
                                     const uint32_t* factors, std::vector<uint32_t>& sigma_pool,
                                     std::vector<size_t>& sigma_off)
{
    std::vector<RadicalDim> rd(dims);
    sigma_off.assign(dims, SIZE_MAX);
    for (uint32_t j = 0; j < dims; ++j) {
        const uint32_t pi = first_prime + j;
        const uint32_t b = prime_at(pi);
        RadicalDim& r = rd[j];
        r.base = b;
        r.maxpow = primes().maxpow[pi];
        r.divb = make_div32(b);
        r.divmp = make_div32(r.maxpow);
        r.mode = 0;
        r.factor = 0;
        r.sigma = nullptr;
        r.table = nullptr;
        r.group = 0;
        r.divg = Div32{0, 0};
        if (sc == QMC_RADICAL_LINEAR) {
            const uint32_t f = factors ? factors[j] : b - 1;
            if (f == 0 || f >= b)
                fail(QMC_INVALID_ARGUMENT,
                     "radical_inverse_linscramble: factor must be in [1, base)");
            r.mode = 1;
            r.factor = f;
        } else if (sc == QMC_RADICAL_FAURE) {
            const auto s = faure(b);
            sigma_off[j] = sigma_pool.size();
            sigma_pool.insert(sigma_pool.end(), s.begin(), s.end());
            r.mode = 2;
        }
        if (b > 2) {
            const DigitTable t = digit_table(b, r.mode, r.factor);
            if (t.ptr) {
                r.table = t.ptr;
                r.group = t.group;
                r.divg = make_div32(t.group);
            }
        }
    }
    return rd;
}

} // namespace

// =====================================================================
//                               C ABI
// =====================================================================

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

namespace {

// build_matrices(builtin_direction_numbers(), dims), built once per dims
// and kept for the process (the reference's builtin_direction_numbers() is
// likewise a function-local static, digitalnet.cpp:73-77).
qmc_matrices* builtin_matrices(uint32_t dims)
{
    static std::mutex mu;
    static std::map<uint32_t, std::unique_ptr<qmc_matrices>> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto& m = cache[dims];
    if (!m) {
        auto cols = build_columns(builtin_rows(), dims); // ConfigError beyond 64
        m = std::make_unique<qmc_matrices>();
        m->dims = dims;
        m->columns = std::move(cols);
    }
    return m.get();
}

} // namespace

extern "C" {

const char* qmc_last_error(void) { return g_error.c_str(); }

const char* qmc_status_string(qmc_status s)
{
    switch (s) {
    case QMC_OK: return "ok";
    case QMC_CONFIG: return "config error";
    case QMC_INVALID_ARGUMENT: return "invalid argument";
    case QMC_OUT_OF_RANGE: return "out of range";
    case QMC_OVERFLOW: return "overflow";
    case QMC_CUDA: return "cuda error";
    case QMC_NCCL: return "nccl error";
    default: return "internal error";
    }
}

int qmc_abi_version(void) { return QMCGPU_ABI_VERSION; }

// ------------------------------------------------------------------ L0

qmc_status qmc_map_u32_to_unifloat(const uint32_t* in, float* out, uint64_t n, qmc_stream stream)
{
    return guard([&] {
        if (n == 0)
            return;
        const cudaStream_t s = as_stream(stream);
        if (is_device_pointer(in) && is_device_pointer(out)) {
            cuda_ok(launch_map(in, out, n, s), "launch_map");
            return;
        }
        // host arrays: stage through device memory
        uint32_t* din = nullptr;
        float* dout = nullptr;
        cuda_ok(cudaMallocAsync(&din, n * 4, s), "cudaMallocAsync");
        cuda_ok(cudaMallocAsync(&dout, n * 4, s), "cudaMallocAsync");
        cuda_ok(cudaMemcpyAsync(din, in, n * 4, cudaMemcpyDefault, s), "H2D");
        cuda_ok(launch_map(din, dout, n, s), "launch_map");
        cuda_ok(cudaMemcpyAsync(out, dout, n * 4, cudaMemcpyDefault, s), "D2H");
        cudaFreeAsync(din, s);
        cudaFreeAsync(dout, s);
        cuda_ok(cudaStreamSynchronize(s), "sync");
    });
}

qmc_status qmc_map_selfcheck(uint64_t* mismatches, qmc_stream stream)
{
    return guard([&] {
        const cudaStream_t s = as_stream(stream);
        unsigned long long* d = nullptr;
        cuda_ok(cudaMallocAsync(&d, 8, s), "cudaMallocAsync");
        cuda_ok(cudaMemsetAsync(d, 0, 8, s), "memset");
        cuda_ok(launch_map_selfcheck(d, s), "launch_map_selfcheck");
        unsigned long long h = 0;
        cuda_ok(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, s), "D2H");
        cudaFreeAsync(d, s);
        cuda_ok(cudaStreamSynchronize(s), "sync");
        *mismatches = h;
    });
}

qmc_status qmc_write_probe(void* device_buffer, uint64_t bytes, int mode, qmc_stream stream)
{
    return guard([&] {
        if (!is_device_pointer(device_buffer))
            fail(QMC_INVALID_ARGUMENT, "write probe needs a device buffer");
        cuda_ok(launch_write_probe(device_buffer, bytes & ~uint64_t(31), mode, as_stream(stream)),
                "launch_write_probe");
    });
}

// ------------------------------------------------------------ host setup

qmc_status qmc_prime(uint32_t index, uint32_t* out)
{
    return guard([&] { *out = prime_at(index); });
}

qmc_status qmc_prime_max_power(uint32_t index, uint32_t* out)
{
    return guard([&] {
        if (index >= kPrimes)
            fail(QMC_OUT_OF_RANGE, "prime_max_power: index beyond the bundled prime table");
        *out = primes().maxpow[index];
    });
}

qmc_status qmc_faure_permutation(uint32_t base, uint32_t* out)
{
    return guard([&] {
        const auto s = faure(base);
        std::memcpy(out, s.data(), s.size() * 4);
    });
}

qmc_status qmc_default_linear_factors(uint32_t dims, uint32_t* out)
{
    return guard([&] {
        if (dims > kPrimes)
            fail(QMC_INVALID_ARGUMENT, "default_linear_factors: dims beyond the prime table");
        for (uint32_t j = 0; j < dims; ++j)
            out[j] = primes().p[j] - 1;
    });
}

qmc_status qmc_lfsr_generator_vector(uint32_t seed, uint32_t dims, uint32_t* out)
{
    return guard([&] {
        const auto g = lfsr(seed, dims);
        std::memcpy(out, g.data(), g.size() * 4);
    });
}

uint32_t qmc_pixel_hash(uint32_t j, uint32_t px, uint32_t py) { return pixel_hash_host(j, px, py); }

uint32_t qmc_hilbert_order_for(uint32_t width, uint32_t height)
{
    return hilbert_order(width, height);
}

qmc_status qmc_partition_by_extra_dimension(uint32_t part, uint32_t parts, uint32_t base,
                                            uint64_t* remainder, uint64_t* modulus)
{
    return guard([&] {
        if (base < 2)
            fail(QMC_INVALID_ARGUMENT, "partition_by_extra_dimension: base must be >= 2");
        uint32_t k = 0;
        uint64_t p = 1;
        while (p < parts) {
            p *= base;
            ++k;
        }
        if (p != parts)
            fail(QMC_CONFIG, "partition_by_extra_dimension: parts must be a power of the base");
        if (part >= parts)
            fail(QMC_OUT_OF_RANGE, "partition_by_extra_dimension: part index beyond parts");
        *remainder = digit_reverse_host(part, base, k);
        *modulus = parts;
    });
}

qmc_status qmc_halton_pixel_enumeration(uint32_t width, uint32_t height, uint32_t px, uint32_t py,
                                        qmc_halton_enumeration* e, uint64_t* offset)
{
    return guard([&] {
        const HaltonEnum h = halton_enum(width, height);
        if (px >= h.sx || py >= h.sy)
            fail(QMC_OUT_OF_RANGE, "HaltonPixelEnumeration: pixel outside the scaled grid");
        if (e)
            *e = qmc_halton_enumeration{h.sx, h.sy, h.ex, h.ey, h.stride};
        if (offset) {
            const uint64_t r2 = digit_reverse_host(px, 2, h.ex);
            const uint64_t r3 = digit_reverse_host(py, 3, h.ey);
            *offset = (r2 * h.crt_x % h.stride + r3 * h.crt_y % h.stride) % h.stride;
        }
    });
}

// ------------------------------------------------------------- matrices

static qmc_matrices* new_matrices(std::vector<uint32_t> cols, uint32_t dims)
{
    auto* m = new qmc_matrices();
    m->dims = dims;
    m->columns = std::move(cols);
    return m;
}

qmc_status qmc_matrices_builtin(uint32_t dims, qmc_matrices** out)
{
    return guard([&] { *out = new_matrices(build_columns(builtin_rows(), dims), dims); });
}

qmc_status qmc_matrices_from_text(const char* text, uint32_t dims, qmc_matrices** out)
{
    return guard([&] {
        if (!text)
            fail(QMC_INVALID_ARGUMENT, "direction number text is null");
        *out = new_matrices(build_columns(parse_rows(text), dims), dims);
    });
}

qmc_status qmc_matrices_from_columns(const uint32_t* columns, uint32_t dims, qmc_matrices** out)
{
    return guard([&] {
        if (!columns && dims)
            fail(QMC_INVALID_ARGUMENT, "columns pointer is null");
        *out = new_matrices(std::vector<uint32_t>(columns, columns + static_cast<size_t>(dims) * 52),
                            dims);
    });
}

uint32_t qmc_matrices_dims(const qmc_matrices* m) { return m ? m->dims : 0; }

qmc_status qmc_matrices_columns(const qmc_matrices* m, uint32_t* out)
{
    return guard([&] {
        if (!m)
            fail(QMC_INVALID_ARGUMENT, "matrices handle is null");
        std::memcpy(out, m->columns.data(), m->columns.size() * 4);
    });
}

void qmc_matrices_destroy(qmc_matrices* m) { delete m; }

// ----------------------------------------------------------------- fills

static void sobol_fill_impl(qmc_matrices* m, uint64_t first, uint64_t n, uint32_t dims,
                            qmc_sobol_scramble sc, const uint32_t* words, qmc_output kind,
                            void* out, cudaStream_t s)
{
    if (!m)
        fail(QMC_INVALID_ARGUMENT, "matrices handle is null");
    if (n == 0 || dims == 0)
        return;
    if (first >= (1ull << 52) || n > (1ull << 52) - first)
        fail(QMC_INVALID_ARGUMENT, "sobol_component: index must be below 2^52");
    if (dims > m->dims)
        fail(QMC_OUT_OF_RANGE, "sobol_component: dimension beyond the matrix set");
    if (sc != QMC_SOBOL_NONE && sc != QMC_SOBOL_XOR && sc != QMC_SOBOL_OWEN)
        fail(QMC_INVALID_ARGUMENT, "sobol_fill: unknown scramble kind");
    // the kernels read dims-strided columns: tables for this dims prefix
    const auto& dev = m->on_device(dims);
    const uint32_t* colsT = static_cast<const uint32_t*>(dev.colsT.get());
    const uint32_t* colsT_rev = static_cast<const uint32_t*>(dev.colsT_rev.get());
    CallArgs args(s);
    SmallArgs small{};
    SmallStage stage;
    if (words && sc != QMC_SOBOL_NONE)
        set_small(small, stage, 0, words, dims, args);
    args.upload();
    finish_small(small, stage, args);
    const int mode = sc == QMC_SOBOL_OWEN ? 2 : 0;
    const bool u32 = kind == QMC_OUT_U32;
    place_fill(out, first, n, dims, s, [&](const FillRange& r, cudaStream_t st) {
        return launch_sobol(colsT, colsT_rev, small, dims, mode, u32, r, st);
    });
}

qmc_status qmc_sobol_fill(const qmc_matrices* m, uint64_t first_index, uint64_t n, uint32_t dims,
                          qmc_sobol_scramble scramble, const uint32_t* words, qmc_output kind,
                          void* out, qmc_stream stream)
{
    return guard([&] {
        sobol_fill_impl(const_cast<qmc_matrices*>(m), first_index, n, dims, scramble, words, kind,
                        out, as_stream(stream));
    });
}

static void halton_fill_impl(uint64_t first, uint64_t n, uint32_t dims, uint32_t first_prime,
                             qmc_radical_scramble sc, const uint32_t* factors, qmc_output kind,
                             void* out, cudaStream_t s)
{
    if (sc != QMC_RADICAL_PLAIN && sc != QMC_RADICAL_LINEAR && sc != QMC_RADICAL_FAURE)
        fail(QMC_INVALID_ARGUMENT, "halton: unknown scramble kind");
    const bool u32 = kind == QMC_OUT_U32;
    if (dims == 1 && first_prime == 0) { // van der Corput: every scramble is the identity
        if (sc == QMC_RADICAL_LINEAR && factors && factors[0] != 1)
            fail(QMC_INVALID_ARGUMENT, "radical_inverse_linscramble: factor must be in [1, base)");
        place_fill(out, first, n, 1, s, [&](const FillRange& r, cudaStream_t st) {
            return launch_vdc(u32, r, st);
        });
        return;
    }
    std::vector<uint32_t> pool;
    std::vector<size_t> soff;
    auto rd = radical_dims(dims, first_prime, sc, factors, pool, soff);
    if (n == 0 || dims == 0)
        return;
    CallArgs pargs(s);
    pool.push_back(0u); // never empty
    pargs.add(pool.data(), pool.size() * 4);
    pargs.upload();
    const uint32_t* pool_dev = pargs.at<uint32_t>(0);
    for (size_t j = 0; j < rd.size(); ++j)
        if (soff[j] != SIZE_MAX)
            rd[j].sigma = pool_dev + soff[j];
    CallArgs args(s);
    const size_t off = args.add(rd.data(), rd.size() * sizeof(RadicalDim));
    args.upload();
    const RadicalDim* rdev = args.at<RadicalDim>(off);
    place_fill(out, first, n, dims, s, [&](const FillRange& r, cudaStream_t st) {
        return launch_halton(rdev, dims, u32, r, st);
    });
}

qmc_status qmc_halton_fill(uint64_t first_index, uint64_t n, uint32_t dims,
                           qmc_radical_scramble scramble, const uint32_t* factors,
                           qmc_output kind, void* out, qmc_stream stream)
{
    return guard([&] {
        if (dims > kPrimes)
            fail(QMC_INVALID_ARGUMENT, "halton_point: dims beyond the prime table");
        halton_fill_impl(first_index, n, dims, 0, scramble, factors, kind, out,
                         as_stream(stream));
    });
}

qmc_status qmc_radical_inverse_fill(uint64_t first_index, uint64_t n, uint32_t prime_index,
                                    qmc_radical_scramble scramble, uint32_t factor,
                                    qmc_output kind, void* out, qmc_stream stream)
{
    return guard([&] {
        prime_at(prime_index); // out_of_range like prime()
        halton_fill_impl(first_index, n, 1, prime_index, scramble, &factor, kind, out,
                         as_stream(stream));
    });
}

static void lattice_fill_impl(const uint32_t* g, const uint32_t* shifts, uint32_t dims,
                              uint64_t first, uint64_t n, qmc_output kind, void* out,
                              cudaStream_t s)
{
    if (n == 0 || dims == 0)
        return;
    if (!g)
        fail(QMC_INVALID_ARGUMENT, "generator vector is null");
    CallArgs args(s);
    SmallArgs small{};
    SmallStage stage;
    set_small(small, stage, 0, g, dims, args);
    if (shifts)
        set_small(small, stage, 1, shifts, dims, args);
    args.upload();
    finish_small(small, stage, args);
    const bool u32 = kind == QMC_OUT_U32;
    place_fill(out, first, n, dims, s, [&](const FillRange& r, cudaStream_t st) {
        return launch_lattice(small, dims, u32, r, st);
    });
}

qmc_status qmc_lattice_fill(const uint32_t* g, const uint32_t* shifts, uint32_t dims,
                            uint64_t first_index, uint64_t n, qmc_output kind, void* out,
                            qmc_stream stream)
{
    return guard([&] {
        lattice_fill_impl(g, shifts, dims, first_index, n, kind, out, as_stream(stream));
    });
}

// ------------------------------------------------------ SampleStream façade

static const char* const kKindNames[] = {"sobol",
                                         "halton",
                                         "lattice",
                                         "halton-hilbert",
                                         "pixel-shifted-lattice",
                                         "pixel-random-lattice",
                                         "image-plane-halton",
                                         "sobol-xor-table"};

qmc_status qmc_sampler_kind_from_name(const char* name, qmc_sampler_kind* out)
{
    return guard([&] {
        const std::string n = name ? name : "";
        for (int k = 0; k < 8; ++k)
            if (n == kKindNames[k]) {
                *out = static_cast<qmc_sampler_kind>(k);
                return;
            }
        fail(QMC_CONFIG, "unknown sampler: " + n);
    });
}

const char* qmc_sampler_kind_name(qmc_sampler_kind kind)
{
    return (kind >= 0 && kind < 8) ? kKindNames[kind] : "";
}

namespace {

void require(bool ok, const char* what)
{
    if (!ok)
        fail(QMC_CONFIG, what);
}

} // namespace

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

    const Dev& on_device(cudaStream_t s)
    {
        const int d = current_device();
        std::lock_guard<std::mutex> lk(mu);
        auto& slot = dev[d];
        if (!slot) {
            auto e = std::make_unique<Dev>();
            e->reorder = dev_upload(reorder.data(), reorder.size() * 4);
            e->scramble = dev_upload(scramble.data(), scramble.size() * 4);
            if (white_noise) {
                // the first point_count Sobol' points at the integer stage,
                // XOR-scrambled per dimension when seeded (imageplane.cpp:224-227),
                // generated by the device fill
                void* pts = nullptr;
                cuda_ok(cudaMalloc(&pts, static_cast<size_t>(point_count) * dims * 4 + 32),
                        "cudaMalloc");
                e->points.reset(pts);
                const bool scr = std::any_of(dim_scramble.begin(), dim_scramble.end(),
                                             [](uint32_t w) { return w != 0; });
                sobol_fill_impl(builtin_matrices(dims), 0, point_count, dims,
                                scr ? QMC_SOBOL_XOR : QMC_SOBOL_NONE, dim_scramble.data(),
                                QMC_OUT_U32, pts, s);
                cuda_ok(cudaStreamSynchronize(s), "sync");
            } else {
                e->points = dev_upload(points.data(), points.size() * 4);
            }
            slot = std::move(e);
        }
        return *slot;
    }
};

namespace {

constexpr size_t kXorTile = 128 * 128;

// white_noise_xor_tables (imageplane.cpp:197-229): std::mt19937 words on the
// host, in the reference's draw order.
std::unique_ptr<qmc_xor_tables> make_white_noise(uint32_t dims, uint32_t point_count,
                                                 uint32_t seed)
{
    if (dims == 0)
        fail(QMC_CONFIG, "white_noise_xor_tables: dims must be >= 1");
    if (point_count == 0 || (point_count & (point_count - 1)) != 0)
        fail(QMC_CONFIG, "white_noise_xor_tables: point count must be a power of two");
    auto t = std::make_unique<qmc_xor_tables>();
    t->dims = dims;
    t->point_count = point_count;
    t->white_noise = true;
    std::mt19937 rng(seed);
    t->dim_scramble.assign(dims, 0u);
    if (seed != 0)
        for (auto& w : t->dim_scramble)
            w = rng();
    t->reorder.resize(kXorTile);
    t->scramble.resize(kXorTile * dims);
    for (auto& v : t->reorder)
        v = rng() & (point_count - 1);
    for (auto& v : t->scramble)
        v = rng();
    return t;
}

// Device view of the tables a stream / render uses: the caller's handle, or
// white-noise tables made for this call.
struct XorTablesDev {
    uint32_t dims = 0, point_count = 0;
    const uint32_t *reorder = nullptr, *scramble = nullptr, *points = nullptr;
    std::unique_ptr<qmc_xor_tables> own;
};

XorTablesDev xor_view(const qmc_xor_tables* given, uint32_t dims, uint32_t point_count,
                      uint32_t seed, cudaStream_t s)
{
    XorTablesDev v;
    qmc_xor_tables* t = const_cast<qmc_xor_tables*>(given);
    if (!t) {
        v.own = make_white_noise(dims, point_count, seed);
        t = v.own.get();
    }
    const auto& d = t->on_device(s);
    v.dims = t->dims;
    v.point_count = t->point_count;
    v.reorder = static_cast<const uint32_t*>(d.reorder.get());
    v.scramble = static_cast<const uint32_t*>(d.scramble.get());
    v.points = static_cast<const uint32_t*>(d.points.get());
    return v;
}

} // namespace

namespace {

// make_stream (imageplane.cpp:310-416) for one pixel context: validates the
// parameters with the reference's ConfigError conditions and resolves the
// device-side state the kernels read. Owns every device resource until it
// goes out of scope (callers synchronize before that).
struct ResolvedStream {
    PixelStreamParams q{};
    std::unique_ptr<qmc_matrices> own_matrices;
    qmc_matrices* matrices = nullptr; // sobol
    std::vector<uint32_t> sobol_words; // sobol scrambles (may be empty)
    XorTablesDev xt;
    std::vector<uint32_t> pool;
    std::vector<size_t> soff;
    std::vector<RadicalDim> rd;
    size_t goff = SIZE_MAX, roff = SIZE_MAX, woff = SIZE_MAX;
    qmc_radical_scramble halton_sc = QMC_RADICAL_PLAIN;
};

void resolve_stream(qmc_sampler_kind kind, const qmc_stream_params* p, cudaStream_t s,
                    ResolvedStream& r, CallArgs& args, CallArgs& pargs)
{
    if (!p)
        fail(QMC_INVALID_ARGUMENT, "stream params are null");
    if (kind < 0 || kind > 7)
        fail(QMC_CONFIG, "unknown sampler kind");
    require(p->dims >= 1, "make_stream: dims must be >= 1");
    const uint32_t dims = p->dims;
    auto halton_scramble = [&]() -> qmc_radical_scramble {
        if (p->halton_scramble > 2)
            fail(QMC_CONFIG, "make_stream: scramble must be plain, faure, or linear");
        if (p->halton_scramble == QMC_RADICAL_LINEAR && p->linear_factors)
            require(p->linear_factors_len >= dims,
                    "make_stream: linear factor list shorter than dims");
        return static_cast<qmc_radical_scramble>(p->halton_scramble);
    };
    auto lattice_vector = [&]() {
        require(p->generator && p->generator_dims > 0, "make_stream: generator vector required");
        for (uint32_t j = 0; j < p->generator_dims; ++j)
            require(p->generator[j] & 1u, "make_stream: generator components must be odd");
        require(dims <= p->generator_dims, "make_stream: dims beyond the generator vector");
        r.goff = args.add(p->generator, dims * 4);
    };
    auto validate_pixel = [&]() {
        require(p->order >= 1 && p->order <= 31, "make_stream: pixel order must be in [1, 31]");
        require(p->px < (1u << p->order) && p->py < (1u << p->order),
                "make_stream: pixel outside the 2^order grid");
    };
    PixelStreamParams& q = r.q;
    q.tab3 = digit_table(3, 0, 0).ptr;
    q.kind = kind;
    q.dims = dims;
    q.px = p->px;
    q.py = p->py;
    q.order = p->order;
    q.spp = p->spp;
    q.width = p->width;
    q.height = p->height;
    switch (kind) {
    case QMC_KIND_SOBOL:
        r.matrices = const_cast<qmc_matrices*>(p->matrices);
        if (!r.matrices)
            r.matrices = builtin_matrices(dims);
        require(dims <= r.matrices->dims, "make_stream: dims beyond the generator matrices");
        if (p->sobol_scrambles) {
            require(p->sobol_scrambles_len >= dims, "make_stream: scramble list shorter than dims");
            r.sobol_words.assign(p->sobol_scrambles, p->sobol_scrambles + dims);
            r.woff = args.add(r.sobol_words.data(), dims * 4);
        }
        break;
    case QMC_KIND_HALTON:
        require(dims <= kPrimes, "make_stream: dims beyond the prime table");
        r.halton_sc = halton_scramble();
        r.rd = radical_dims(dims, 0, r.halton_sc, p->linear_factors, r.pool, r.soff);
        break;
    case QMC_KIND_LATTICE:
        lattice_vector();
        break;
    case QMC_KIND_HALTON_HILBERT:
        require(p->spp >= 1, "make_stream: spp must be >= 1");
        validate_pixel();
        require(dims <= kPrimes, "halton_point: dims beyond the prime table");
        r.rd = radical_dims(dims, 0, halton_scramble(), p->linear_factors, r.pool, r.soff);
        break;
    case QMC_KIND_PIXEL_SHIFTED_LATTICE:
        validate_pixel();
        lattice_vector();
        break;
    case QMC_KIND_PIXEL_RANDOM_LATTICE:
        break;
    case QMC_KIND_IMAGE_PLANE_HALTON: {
        require(p->width >= 1 && p->height >= 1,
                "make_stream: image size required for image-plane halton");
        require(p->px < p->width && p->py < p->height, "make_stream: pixel outside the image");
        require(dims <= kPrimes, "make_stream: dims beyond the prime table");
        const HaltonEnum e = halton_enum(p->width, p->height);
        if (p->linear_factors)
            require(p->linear_factors_len >= dims,
                    "make_stream: linear factor list shorter than dims");
        r.rd = radical_dims(dims, 0, QMC_RADICAL_LINEAR, p->linear_factors, r.pool, r.soff);
        q.scale_x = e.sx;
        q.scale_y = e.sy;
        q.exp_x = e.ex;
        q.exp_y = e.ey;
        q.stride = e.stride;
        q.crt_x = e.crt_x;
        q.crt_y = e.crt_y;
        break;
    }
    case QMC_KIND_SOBOL_XOR_TABLE: {
        r.xt = xor_view(p->xor_tables, dims, p->xor_point_count, p->xor_seed, s);
        require(dims <= r.xt.dims, "make_stream: dims beyond the stored point set");
        q.xor_reorder = r.xt.reorder;
        q.xor_scramble = r.xt.scramble;
        q.xor_points = r.xt.points;
        q.xor_point_count = r.xt.point_count;
        q.xor_dims = r.xt.dims;
        break;
    }
    }
    // radical tables: the permutation pool goes first (its device address is
    // patched into the RadicalDim records), then everything else
    if (!r.rd.empty()) {
        r.pool.push_back(0u); // never empty
        pargs.add(r.pool.data(), r.pool.size() * 4);
        pargs.upload();
        const uint32_t* pool_dev = pargs.at<uint32_t>(0);
        for (size_t j = 0; j < r.rd.size(); ++j)
            if (r.soff[j] != SIZE_MAX)
                r.rd[j].sigma = pool_dev + r.soff[j];
        r.roff = args.add(r.rd.data(), r.rd.size() * sizeof(RadicalDim));
    }
    args.upload();
    if (r.goff != SIZE_MAX)
        q.generator = args.at<uint32_t>(r.goff);
    if (r.roff != SIZE_MAX)
        q.radical_dims = args.at<RadicalDim>(r.roff);
}

} // namespace

qmc_status qmc_stream_fill(qmc_sampler_kind kind, const qmc_stream_params* p,
                           uint64_t first_index, uint64_t n, qmc_output out_kind, void* out,
                           qmc_stream stream)
{
    return guard([&] {
        const cudaStream_t s = as_stream(stream);
        if (!p)
            fail(QMC_INVALID_ARGUMENT, "stream params are null");
        const uint32_t dims = p->dims;
        // the non-pixel kinds are the batched fills
        if (kind == QMC_KIND_SOBOL || kind == QMC_KIND_HALTON || kind == QMC_KIND_LATTICE) {
            CallArgs args(s), pargs(s);
            ResolvedStream r;
            resolve_stream(kind, p, s, r, args, pargs);
            if (kind == QMC_KIND_SOBOL) {
                sobol_fill_impl(r.matrices, first_index, n, dims,
                                r.sobol_words.empty() ? QMC_SOBOL_NONE : QMC_SOBOL_XOR,
                                r.sobol_words.empty() ? nullptr : r.sobol_words.data(), out_kind,
                                out, s);
            } else if (kind == QMC_KIND_HALTON) {
                // SampleStream::sample casts the index to 32 bits (the kernel wraps too)
                halton_fill_impl(first_index, n, dims, 0, r.halton_sc, p->linear_factors,
                                 out_kind, out, s);
            } else {
                lattice_fill_impl(p->generator, nullptr, dims, first_index, n, out_kind, out, s);
            }
            cuda_ok(cudaStreamSynchronize(s), "sync");
            return;
        }
        CallArgs args(s), pargs(s);
        ResolvedStream r;
        resolve_stream(kind, p, s, r, args, pargs);
        if (kind == QMC_KIND_HALTON_HILBERT && (first_index >= p->spp || n > p->spp - first_index))
            fail(QMC_OUT_OF_RANGE, "SampleStream: sample index beyond the pixel block");
        if (kind == QMC_KIND_SOBOL_XOR_TABLE &&
            (first_index >= r.q.xor_point_count || n > r.q.xor_point_count - first_index))
            fail(QMC_OUT_OF_RANGE, "xor_table_sample: index beyond the stored point set");
        if (n == 0)
            return;
        const bool u32 = out_kind == QMC_OUT_U32;
        place_fill(out, first_index, n, dims, s, [&](const FillRange& fr, cudaStream_t st) {
            return launch_pixel_stream(r.q, u32, fr, st);
        });
        cuda_ok(cudaStreamSynchronize(s), "sync"); // tables owned by this call
    });
}

// --------------------------------------------------------------- integrate

static const char* const kIntegrandNames[] = {"product-sine", "product-poly", "indicator"};

qmc_status qmc_builtin_integrand(const char* name, uint32_t dims, qmc_integrand_kind* kind,
                                 double* exact_integral)
{
    return guard([&] {
        if (dims == 0)
            fail(QMC_INVALID_ARGUMENT, "builtin_integrands: dims must be >= 1");
        const std::string n = name ? name : "";
        for (int k = 0; k < 3; ++k)
            if (n == kIntegrandNames[k]) {
                if (kind)
                    *kind = static_cast<qmc_integrand_kind>(k);
                if (exact_integral) // quality.cpp:38-66
                    *exact_integral = k == 2 ? std::pow(0.7, static_cast<double>(dims)) : 1.0;
                return;
            }
        fail(QMC_CONFIG, "unknown integrand: " + n);
    });
}

qmc_status qmc_integrate(qmc_sampler_kind kind, const qmc_stream_params* p,
                         qmc_integrand_kind f, uint32_t f_dims, uint64_t n, qmc_accum mode,
                         qmc_integration_row* row, qmc_stream stream)
{
    return guard([&] {
        const auto t0 = std::chrono::steady_clock::now();
        const cudaStream_t s = as_stream(stream);
        if (f < 0 || f > 2)
            fail(QMC_CONFIG, "unknown integrand");
        if (f_dims == 0)
            fail(QMC_INVALID_ARGUMENT, "builtin_integrands: dims must be >= 1");
        if (mode != QMC_ACCUM_KAHAN && mode != QMC_ACCUM_INT)
            fail(QMC_CONFIG, "accumulation mode must be 'kahan' or 'int'");
        if (n == 0)
            fail(QMC_INVALID_ARGUMENT, "integrate: n must be >= 1");
        if (!p)
            fail(QMC_INVALID_ARGUMENT, "stream params are null");
        if (p->dims < f_dims)
            fail(QMC_INVALID_ARGUMENT, "integrate: stream has fewer dimensions than the integrand");
        if (f_dims > integrate_max_dims())
            fail(QMC_INVALID_ARGUMENT, "integrate: at most 64 integrand dimensions on the device");
        CallArgs args(s), pargs(s);
        ResolvedStream r;
        resolve_stream(kind, p, s, r, args, pargs);
        // sample-time preconditions of SampleStream::sample over [0, n)
        if (kind == QMC_KIND_SOBOL && n > (1ull << 52))
            fail(QMC_INVALID_ARGUMENT, "sobol_component: index must be below 2^52");
        if (kind == QMC_KIND_HALTON_HILBERT && n > p->spp)
            fail(QMC_OUT_OF_RANGE, "SampleStream: sample index beyond the pixel block");
        if (kind == QMC_KIND_SOBOL_XOR_TABLE && n > r.q.xor_point_count)
            fail(QMC_OUT_OF_RANGE, "xor_table_sample: index beyond the stored point set");
        if (kind == QMC_KIND_HALTON || kind == QMC_KIND_HALTON_HILBERT ||
            kind == QMC_KIND_IMAGE_PLANE_HALTON)
            for (const RadicalDim& d : r.rd)
                if (d.mode == 1 && (d.factor == 0 || d.factor >= d.base))
                    fail(QMC_INVALID_ARGUMENT,
                         "radical_inverse_linscramble: factor must be in [1, base)");

        const uint32_t dims_of_integrand = p->dims; // stream dims (>= f_dims)
        IntegrateParams ip{};
        ip.pix = r.q;
        ip.fn = f;
        ip.fdims = f_dims;
        ip.n = n;
        if (kind == QMC_KIND_SOBOL) {
            const auto& dev = r.matrices->on_device(dims_of_integrand);
            ip.colsT = static_cast<const uint32_t*>(dev.colsT.get());
            ip.mdims = dims_of_integrand;
            ip.words = r.woff == SIZE_MAX ? nullptr : args.at<uint32_t>(r.woff);
        }
        const uint64_t chunks = (n + 4095) / 4096;
        double* partial = nullptr;
        unsigned long long* scal = nullptr; // [0] int sum, [1] first bad index
        cuda_ok(cudaMallocAsync(&partial, chunks * 8, s), "cudaMallocAsync");
        cuda_ok(cudaMallocAsync(&scal, 16, s), "cudaMallocAsync");
        const unsigned long long init[2] = {0ull, ~0ull};
        cuda_ok(cudaMemcpyAsync(scal, init, 16, cudaMemcpyHostToDevice, s), "H2D");
        cuda_ok(launch_integrate(ip, mode, partial, scal, scal + 1, s), "launch_integrate");
        std::vector<double> hp(mode == QMC_ACCUM_KAHAN ? chunks : 0);
        unsigned long long hs[2] = {0, 0};
        if (!hp.empty())
            cuda_ok(cudaMemcpyAsync(hp.data(), partial, chunks * 8, cudaMemcpyDeviceToHost, s),
                    "D2H");
        cuda_ok(cudaMemcpyAsync(hs, scal, 16, cudaMemcpyDeviceToHost, s), "D2H");
        cudaFreeAsync(partial, s);
        cudaFreeAsync(scal, s);
        cuda_ok(cudaStreamSynchronize(s), "sync");
        if (hs[1] != ~0ull)
            fail(QMC_INTERNAL, std::string("integrate: non-finite value of '") +
                                   kIntegrandNames[f] + "' at index " + std::to_string(hs[1]));
        double estimate;
        if (mode == QMC_ACCUM_KAHAN) { // rank-ordered CompensatedSum, quality.cpp:262-267
            double sum = 0.0, comp = 0.0;
            for (double v : hp) {
                const double t = sum + v;
                if (std::fabs(sum) >= std::fabs(v))
                    comp += (sum - t) + v;
                else
                    comp += (v - t) + sum;
                sum = t;
            }
            estimate = (sum + comp) / static_cast<double>(n);
        } else { // exact 64-bit sum, quality.cpp:268-272
            estimate = static_cast<double>(static_cast<long long>(hs[0])) / 4294967296.0 /
                       static_cast<double>(n);
        }
        double exact = 1.0;
        qmc_builtin_integrand(kIntegrandNames[f], f_dims, nullptr, &exact);
        if (row) {
            row->n = n;
            row->estimate = estimate;
            row->abs_error = std::fabs(estimate - exact);
            row->seconds =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
    });
}

// --------------------------------------------------------------- XOR tables

qmc_status qmc_xor_tables_white_noise(uint32_t dims, uint32_t point_count, uint32_t seed,
                                      qmc_xor_tables** out)
{
    return guard([&] { *out = make_white_noise(dims, point_count, seed).release(); });
}

// load_xor_tables (imageplane.cpp:163-195): "XQT1", 128^2 reorder words (used
// modulo point_count), then 128^2 * dims scramble words, little-endian.
qmc_status qmc_xor_tables_load(const void* bytes, size_t len, uint32_t dims,
                               const uint32_t* points, uint32_t point_count,
                               qmc_xor_tables** out)
{
    return guard([&] {
        if (dims == 0)
            fail(QMC_CONFIG, "load_xor_tables: dims must be >= 1");
        if (point_count == 0 || (point_count & (point_count - 1)) != 0)
            fail(QMC_CONFIG, "load_xor_tables: point count must be a power of two");
        if (!points)
            fail(QMC_CONFIG, "load_xor_tables: point set size does not match point_count * dims");
        const unsigned char* b = static_cast<const unsigned char*>(bytes);
        if (!b || len < 4 || std::memcmp(b, "XQT1", 4) != 0)
            fail(QMC_CONFIG, "xor table file: bad magic, expected XQT1");
        size_t pos = 4;
        auto word = [&]() -> uint32_t {
            if (pos + 4 > len)
                fail(QMC_CONFIG, "xor table file: truncated");
            const uint32_t v = static_cast<uint32_t>(b[pos]) | (static_cast<uint32_t>(b[pos + 1]) << 8) |
                               (static_cast<uint32_t>(b[pos + 2]) << 16) |
                               (static_cast<uint32_t>(b[pos + 3]) << 24);
            pos += 4;
            return v;
        };
        auto t = std::make_unique<qmc_xor_tables>();
        t->dims = dims;
        t->point_count = point_count;
        t->reorder.resize(kXorTile);
        for (auto& v : t->reorder)
            v = word() & (point_count - 1);
        t->scramble.resize(kXorTile * dims);
        for (auto& v : t->scramble)
            v = word();
        t->points.assign(points, points + static_cast<size_t>(point_count) * dims);
        *out = t.release();
    });
}

// write_xor_table_file (imageplane.cpp:154-161).
qmc_status qmc_xor_tables_write(const qmc_xor_tables* t, void* bytes, size_t* len)
{
    return guard([&] {
        if (!t || !len)
            fail(QMC_INVALID_ARGUMENT, "xor tables: null argument");
        const size_t need = 4 + 4 * (t->reorder.size() + t->scramble.size());
        if (!bytes || *len < need) {
            *len = need;
            if (bytes)
                fail(QMC_INVALID_ARGUMENT, "xor tables: output buffer too small");
            return;
        }
        unsigned char* o = static_cast<unsigned char*>(bytes);
        std::memcpy(o, "XQT1", 4);
        size_t pos = 4;
        auto put = [&](uint32_t v) {
            o[pos] = v & 0xff;
            o[pos + 1] = (v >> 8) & 0xff;
            o[pos + 2] = (v >> 16) & 0xff;
            o[pos + 3] = (v >> 24) & 0xff;
            pos += 4;
        };
        for (uint32_t v : t->reorder)
            put(v);
        for (uint32_t v : t->scramble)
            put(v);
        *len = need;
    });
}

uint32_t qmc_xor_tables_dims(const qmc_xor_tables* t) { return t ? t->dims : 0; }
uint32_t qmc_xor_tables_point_count(const qmc_xor_tables* t) { return t ? t->point_count : 0; }
void qmc_xor_tables_destroy(qmc_xor_tables* t) { delete t; }

// ------------------------------------------------------------ quality metrics

namespace {

// Device copy of a row-major float point set (host arrays are staged).
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

double pairwise_metric(const float* points, uint64_t n, uint32_t dims, cudaStream_t s, bool l2)
{
    if (dims > quality_max_dims())
        fail(QMC_INVALID_ARGUMENT, "quality metric: at most 256 dimensions on the device");
    if (n > 0x7fffffffull)
        fail(QMC_INVALID_ARGUMENT, "quality metric: at most 2^31 - 1 points");
    pool_keep_memory();
    DevPoints dp(points, n * dims, s);
    double* scratch = nullptr;
    cuda_ok(cudaMallocAsync(&scratch, (2 * n + 1) * 8, s), "cudaMallocAsync");
    cuda_ok(l2 ? launch_l2star(dp.ptr, n, dims, scratch + 1, scratch, s)
               : launch_mindist(dp.ptr, n, dims, scratch + 1, scratch, s),
            "launch quality");
    double r = 0.0;
    cuda_ok(cudaMemcpyAsync(&r, scratch, 8, cudaMemcpyDeviceToHost, s), "D2H");
    cudaFreeAsync(scratch, s);
    cuda_ok(cudaStreamSynchronize(s), "sync");
    return r;
}

} // namespace

qmc_status qmc_l2_star_discrepancy(const float* points, uint64_t n, uint32_t dims, double* out,
                                   qmc_stream stream)
{
    return guard([&] {
        if (n == 0 || dims == 0)
            fail(QMC_INVALID_ARGUMENT, "l2_star_discrepancy: empty point set");
        if (!points || !out)
            fail(QMC_INVALID_ARGUMENT, "l2_star_discrepancy: null pointer");
        *out = pairwise_metric(points, n, dims, as_stream(stream), true);
    });
}

qmc_status qmc_min_toroidal_distance(const float* points, uint64_t n, uint32_t dims, double* out,
                                     qmc_stream stream)
{
    return guard([&] {
        if (n < 2)
            fail(QMC_INVALID_ARGUMENT, "min_toroidal_distance: need at least two points");
        if (!points || !out)
            fail(QMC_INVALID_ARGUMENT, "min_toroidal_distance: null pointer");
        *out = pairwise_metric(points, n, dims, as_stream(stream), false);
    });
}

qmc_status qmc_check_1d_stratification(qmc_sampler_kind kind, const qmc_stream_params* params,
                                       uint32_t j, uint32_t m, int* ok, uint32_t* histogram,
                                       qmc_stream stream)
{
    return guard([&] {
        if (m > 20)
            fail(QMC_INVALID_ARGUMENT, "check_1d_stratification: m must be <= 20");
        if (!params)
            fail(QMC_INVALID_ARGUMENT, "stream params are null");
        if (j >= params->dims)
            fail(QMC_OUT_OF_RANGE, "SampleStream: dimension beyond the stream");
        const cudaStream_t s = as_stream(stream);
        pool_keep_memory();
        const uint32_t count = 1u << m;
        float* pts = nullptr;
        uint32_t* hist = nullptr;
        unsigned int* bad = nullptr;
        cuda_ok(cudaMallocAsync(&pts, static_cast<size_t>(count) * params->dims * 4 + 32, s),
                "cudaMallocAsync");
        cuda_ok(cudaMallocAsync(&hist, static_cast<size_t>(count) * 4 + 4, s), "cudaMallocAsync");
        cuda_ok(cudaMemsetAsync(hist, 0, static_cast<size_t>(count) * 4 + 4, s), "memset");
        const qmc_status st = qmc_stream_fill(kind, params, 0, count, QMC_OUT_F32, pts, stream);
        if (st != QMC_OK) {
            cudaFreeAsync(pts, s);
            cudaFreeAsync(hist, s);
            fail(st, g_error);
        }
        bad = reinterpret_cast<unsigned int*>(hist + count);
        cuda_ok(launch_stratification(pts, m, params->dims, j, hist, bad, s), "launch");
        unsigned int hbad = 0;
        cuda_ok(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, s), "D2H");
        if (histogram)
            cuda_ok(cudaMemcpyAsync(histogram, hist, static_cast<size_t>(count) * 4,
                                    cudaMemcpyDeviceToHost, s),
                    "D2H");
        cudaFreeAsync(pts, s);
        cudaFreeAsync(hist, s);
        cuda_ok(cudaStreamSynchronize(s), "sync");
        *ok = hbad == 0;
    });
}

// ------------------------------------------------------------------ formats

// load_generator_vector (lattice.cpp:21-46): one decimal component per line,
// '#' comments; ConfigError for components beyond 32 bits, even components,
// or an empty file.
qmc_status qmc_load_generator_vector(const char* text, uint32_t* out, uint32_t capacity,
                                     uint32_t* dims)
{
    return guard([&] {
        if (!text || !dims)
            fail(QMC_INVALID_ARGUMENT, "load_generator_vector: null argument");
        std::istringstream in(text);
        std::string line;
        size_t no = 0;
        std::vector<uint32_t> g;
        while (std::getline(in, line)) {
            ++no;
            const auto hash = line.find('#');
            if (hash != std::string::npos)
                line.erase(hash);
            std::istringstream ls(line);
            uint64_t v = 0;
            if (!(ls >> v))
                continue;
            if (v > 0xffffffffull)
                fail(QMC_CONFIG, "generator vector, line " + std::to_string(no) +
                                     ": component beyond 32 bits");
            if (v % 2 == 0)
                fail(QMC_CONFIG,
                     "generator vector, line " + std::to_string(no) + ": component is even");
            g.push_back(static_cast<uint32_t>(v));
        }
        if (g.empty())
            fail(QMC_CONFIG, "generator vector file holds no components");
        *dims = static_cast<uint32_t>(g.size());
        if (out) {
            if (capacity < g.size())
                fail(QMC_INVALID_ARGUMENT, "load_generator_vector: output capacity too small");
            std::memcpy(out, g.data(), g.size() * 4);
        }
    });
}

// load_linear_factors (radical.cpp:281-306): "base factor" lines override the
// default factor (base - 1) of the matching prime among the first dims.
qmc_status qmc_load_linear_factors(const char* text, uint32_t dims, uint32_t* out)
{
    return guard([&] {
        if (!text || !out)
            fail(QMC_INVALID_ARGUMENT, "load_linear_factors: null argument");
        if (dims > kPrimes)
            fail(QMC_INVALID_ARGUMENT, "default_linear_factors: dims beyond the prime table");
        std::vector<uint32_t> f(dims);
        for (uint32_t j = 0; j < dims; ++j)
            f[j] = primes().p[j] - 1;
        std::istringstream in(text);
        std::string line;
        size_t no = 0;
        while (std::getline(in, line)) {
            ++no;
            const auto hash = line.find('#');
            if (hash != std::string::npos)
                line.erase(hash);
            std::istringstream ls(line);
            uint64_t base = 0, factor = 0;
            if (!(ls >> base))
                continue;
            if (!(ls >> factor))
                fail(QMC_CONFIG, "scramble factor file, line " + std::to_string(no) +
                                     ": expected 'base factor'");
            if (base < 2 || factor == 0 || factor >= base)
                fail(QMC_CONFIG, "scramble factor file, line " + std::to_string(no) +
                                     ": factor must be in [1, base)");
            for (uint32_t j = 0; j < dims; ++j)
                if (primes().p[j] == base)
                    f[j] = static_cast<uint32_t>(factor);
        }
        std::memcpy(out, f.data(), f.size() * 4);
    });
}

// fnv1a64 (image.cpp:54-63) — checksum of serialized output.
uint64_t qmc_fnv1a64(const void* data, uint64_t size)
{
    const unsigned char* p = static_cast<const unsigned char*>(data);
    uint64_t h = 0xcbf29ce484222325ull;
    for (uint64_t k = 0; k < size; ++k) {
        h ^= p[k];
        h *= 0x100000001b3ull;
    }
    return h;
}

// `qmckit points --format csv` rows (qmckit.cpp:225-235): "%.9f" per
// component, comma-separated, one line per point. Host formatting of a
// device or host float array; bytes = NULL queries the size.
qmc_status qmc_write_points_csv(const float* points, uint64_t n, uint32_t dims, void* bytes,
                                size_t* len, qmc_stream stream)
{
    return guard([&] {
        if (!len || (!points && n))
            fail(QMC_INVALID_ARGUMENT, "write_points_csv: null argument");
        std::vector<float> host;
        const float* p = points;
        if (n && is_device_pointer(points)) {
            host.resize(n * dims);
            const cudaStream_t s = as_stream(stream);
            cuda_ok(cudaMemcpyAsync(host.data(), points, host.size() * 4, cudaMemcpyDeviceToHost,
                                    s),
                    "D2H");
            cuda_ok(cudaStreamSynchronize(s), "sync");
            p = host.data();
        }
        std::string text;
        text.reserve(n * dims * 12);
        char buf[32];
        for (uint64_t i = 0; i < n; ++i) {
            for (uint32_t j = 0; j < dims; ++j) {
                std::snprintf(buf, sizeof buf, "%.9f", static_cast<double>(p[i * dims + j]));
                if (j)
                    text += ',';
                text += buf;
            }
            text += '\n';
        }
        if (bytes) {
            if (*len < text.size())
                fail(QMC_INVALID_ARGUMENT, "write_points_csv: output buffer too small");
            std::memcpy(bytes, text.data(), text.size());
        }
        *len = text.size();
    });
}

// write_pgm / write_ppm (image.cpp:34-52): header on the host, the per-pixel
// quantization (image.cpp:25-30) on the device.
qmc_status qmc_write_pnm(const float* image, uint32_t width, uint32_t height, uint32_t channels,
                         void* bytes, size_t* len, qmc_stream stream)
{
    return guard([&] {
        if (!len)
            fail(QMC_INVALID_ARGUMENT, "write_pnm: null length");
        if (channels != 1 && channels != 3)
            fail(QMC_INVALID_ARGUMENT, "write_pnm: channels must be 1 (P5) or 3 (P6)");
        if (width == 0 || height == 0)
            fail(QMC_INVALID_ARGUMENT, "make_image: image must be at least 1x1");
        const std::string header = std::string(channels == 1 ? "P5\n" : "P6\n") +
                                   std::to_string(width) + " " + std::to_string(height) +
                                   "\n255\n";
        const uint64_t npix = static_cast<uint64_t>(width) * height;
        const size_t need = header.size() + npix * channels;
        if (!bytes || *len < need) {
            *len = need;
            if (bytes)
                fail(QMC_INVALID_ARGUMENT, "write_pnm: output buffer too small");
            return;
        }
        if (!image)
            fail(QMC_INVALID_ARGUMENT, "write_pnm: null image");
        const cudaStream_t s = as_stream(stream);
        pool_keep_memory();
        DevPoints dv(image, npix, s);
        unsigned char* d = nullptr;
        cuda_ok(cudaMallocAsync(&d, npix * channels + 1, s), "cudaMallocAsync");
        cuda_ok(launch_quantize(dv.ptr, npix, channels, d, s), "launch_quantize");
        unsigned char* o = static_cast<unsigned char*>(bytes);
        std::memcpy(o, header.data(), header.size());
        cuda_ok(cudaMemcpyAsync(o + header.size(), d, npix * channels, cudaMemcpyDeviceToHost, s),
                "D2H");
        cudaFreeAsync(d, s);
        cuda_ok(cudaStreamSynchronize(s), "sync");
        *len = need;
    });
}

// ------------------------------------------------------------------ render

namespace {

// render() validation and defaults (render.cpp:83-106) resolved into the
// kernel parameters; owns the XOR tables view for the call.
struct ResolvedRender {
    RenderParams p{};
    XorTablesDev xt;
    uint64_t npix = 0;
};

void resolve_render(const qmc_render_job* job, uint32_t row_begin, uint32_t row_end,
                    cudaStream_t s, CallArgs& args, ResolvedRender& rr)
{
    if (!job)
        fail(QMC_INVALID_ARGUMENT, "render job is null");
    if (job->width == 0 || job->height == 0)
        fail(QMC_CONFIG, "render: image must be at least 1x1");
    if (job->spp == 0)
        fail(QMC_CONFIG, "render: spp must be >= 1");
    if (job->kind < 0 || job->kind > 7)
        fail(QMC_CONFIG, "unknown sampler kind");
    if (job->accum != QMC_ACCUM_KAHAN && job->accum != QMC_ACCUM_INT)
        fail(QMC_CONFIG, "accumulation mode must be 'kahan' or 'int'");
    if (row_begin > row_end || row_end > job->height)
        fail(QMC_OUT_OF_RANGE, "render: row band outside the image");
    RenderParams& p = rr.p;
    p.width = job->width;
    p.height = job->height;
    p.spp = job->spp;
    p.order = hilbert_order(job->width, job->height);
    p.row_begin = row_begin;
    p.row_end = row_end;
    p.inv_w = 1.0 / job->width;
    p.inv_h = 1.0 / job->height;
    std::vector<uint32_t> g = job->generator && job->generator_dims
                                  ? std::vector<uint32_t>(job->generator,
                                                          job->generator + job->generator_dims)
                                  : lfsr(job->seed ? job->seed : 0xace1u, 2);
    const uint32_t kind = job->kind;
    if (kind == QMC_KIND_HALTON_HILBERT || kind == QMC_KIND_PIXEL_SHIFTED_LATTICE)
        require(p.order >= 1 && p.order <= 31, "make_stream: pixel order must be in [1, 31]");
    if (kind == QMC_KIND_LATTICE || kind == QMC_KIND_PIXEL_SHIFTED_LATTICE) {
        for (uint32_t v : g)
            require(v & 1u, "make_stream: generator components must be odd");
        require(g.size() >= 2, "make_stream: dims beyond the generator vector");
    }
    if (g.size() < 2)
        g.resize(2, 1u);
    p.g0 = g[0];
    p.g1 = g[1];
    if (kind == QMC_KIND_SOBOL && job->seed != 0) {
        p.scr0 = pixel_hash_host(0, job->seed, 0);
        p.scr1 = pixel_hash_host(1, job->seed, 0);
    }
    p.tab3 = digit_table(3, 0, 0).ptr; // phi_3, seven ternary digits per step
    std::vector<uint32_t> cols2(104, 0u);
    if (job->matrices) {
        require(job->matrices->dims >= 2, "make_stream: dims beyond the generator matrices");
        std::memcpy(cols2.data(), job->matrices->columns.data(), 104 * 4);
    } else {
        cols2 = build_columns(builtin_rows(), 2);
    }
    if (kind == QMC_KIND_IMAGE_PLANE_HALTON) {
        const HaltonEnum he = halton_enum(job->width, job->height);
        p.scale_x = he.sx;
        p.scale_y = he.sy;
        p.exp_x = he.ex;
        p.exp_y = he.ey;
        p.stride = he.stride;
        p.crt_x = he.crt_x;
        p.crt_y = he.crt_y;
    }
    if (kind == QMC_KIND_SOBOL_XOR_TABLE) {
        uint32_t pc = 1;
        while (pc < job->spp)
            pc <<= 1;
        rr.xt = xor_view(job->tables, 2, pc, job->seed, s);
        require(rr.xt.dims >= 2, "make_stream: dims beyond the stored point set");
        p.xor_reorder = rr.xt.reorder;
        p.xor_scramble = rr.xt.scramble;
        p.xor_points = rr.xt.points;
        p.xor_point_count = rr.xt.point_count;
        p.xor_dims = rr.xt.dims;
    }
    const size_t coff = args.add(cols2.data(), cols2.size() * 4);
    args.upload();
    p.cols2 = args.at<uint32_t>(coff);
    rr.npix = static_cast<uint64_t>(row_end - row_begin) * job->width;
}

} // namespace

qmc_status qmc_render(const qmc_render_job* job, uint32_t row_begin, uint32_t row_end, float* out,
                      qmc_stream stream)
{
    return guard([&] {
        const cudaStream_t s = as_stream(stream);
        CallArgs args(s);
        ResolvedRender rr;
        resolve_render(job, row_begin, row_end, s, args, rr);
        if (rr.npix == 0)
            return;
        if (!out)
            fail(QMC_INVALID_ARGUMENT, "output pointer is null");
        if (is_device_pointer(out)) {
            cuda_ok(launch_render(rr.p, job->kind, job->accum, out, s), "launch_render");
            if (job->kind == QMC_KIND_SOBOL_XOR_TABLE && !job->tables)
                cuda_ok(cudaStreamSynchronize(s), "sync"); // temporary tables die with the call
            return;
        }
        float* d = nullptr;
        cuda_ok(cudaMallocAsync(&d, rr.npix * 4, s), "cudaMallocAsync");
        cuda_ok(launch_render(rr.p, job->kind, job->accum, d, s), "launch_render");
        cuda_ok(cudaMemcpyAsync(out, d, rr.npix * 4, cudaMemcpyDeviceToHost, s), "D2H");
        cudaFreeAsync(d, s);
        cuda_ok(cudaStreamSynchronize(s), "sync");
    });
}

qmc_status qmc_render_partial(const qmc_render_job* job, uint32_t part, uint32_t parts,
                              uint32_t row_begin, uint32_t row_end, int64_t* accum,
                              qmc_stream stream)
{
    return guard([&] {
        const cudaStream_t s = as_stream(stream);
        if (job && job->accum != QMC_ACCUM_INT)
            fail(QMC_INVALID_ARGUMENT,
                 "render_partial: sample partitions need the int accumulator (exactly associative)");
        uint64_t rem = 0, mod = 1;
        const qmc_status st = qmc_partition_by_extra_dimension(part, parts, 2, &rem, &mod);
        if (st != QMC_OK)
            fail(st, g_error);
        CallArgs args(s);
        ResolvedRender rr;
        resolve_render(job, row_begin, row_end, s, args, rr);
        if (rr.npix == 0)
            return;
        if (!accum || !is_device_pointer(accum))
            fail(QMC_INVALID_ARGUMENT, "render_partial: accum must be a device buffer");
        cuda_ok(launch_render_partial(rr.p, job->kind, static_cast<uint32_t>(rem),
                                      static_cast<uint32_t>(mod),
                                      reinterpret_cast<long long*>(accum), s),
                "launch_render_partial");
        if (job->kind == QMC_KIND_SOBOL_XOR_TABLE && !job->tables)
            cuda_ok(cudaStreamSynchronize(s), "sync");
    });
}

qmc_status qmc_render_finalize(const int64_t* accum, uint64_t npix, uint32_t spp, float* out,
                               qmc_stream stream)
{
    return guard([&] {
        if (spp == 0)
            fail(QMC_CONFIG, "render: spp must be >= 1");
        if (npix == 0)
            return;
        if (!accum || !out || !is_device_pointer(accum) || !is_device_pointer(out))
            fail(QMC_INVALID_ARGUMENT, "render_finalize: device buffers required");
        cuda_ok(launch_render_finalize(reinterpret_cast<const long long*>(accum), npix, spp, out,
                                       as_stream(stream)),
                "launch_render_finalize");
    });
}

qmc_status qmc_scene_value(const double* xy, double* out, uint64_t n, qmc_stream stream)
{
    return guard([&] {
        if (n == 0)
            return;
        const cudaStream_t s = as_stream(stream);
        if (is_device_pointer(xy) && is_device_pointer(out)) {
            cuda_ok(launch_scene_value(xy, out, n, s), "launch_scene_value");
            return;
        }
        double *dxy = nullptr, *dout = nullptr;
        cuda_ok(cudaMallocAsync(&dxy, n * 16, s), "cudaMallocAsync");
        cuda_ok(cudaMallocAsync(&dout, n * 8, s), "cudaMallocAsync");
        cuda_ok(cudaMemcpyAsync(dxy, xy, n * 16, cudaMemcpyDefault, s), "H2D");
        cuda_ok(launch_scene_value(dxy, dout, n, s), "launch_scene_value");
        cuda_ok(cudaMemcpyAsync(out, dout, n * 8, cudaMemcpyDefault, s), "D2H");
        cudaFreeAsync(dxy, s);
        cudaFreeAsync(dout, s);
        cuda_ok(cudaStreamSynchronize(s), "sync");
    });
}

} // extern "C"
