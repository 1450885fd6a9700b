// abi_bench.cpp — qmc_run_bench_kernel (run_bench_kernel, bench.cpp:79-150,
// the `qmckit bench` comparison of SPEC acceptance 9) and the FP64 probe.
#include "objects.hpp"

#include <string>

using namespace qmcgpu;
using namespace qmcgpu::host;

namespace {

// RAII pair of CUDA events on the current device.
struct EventPair {
    cudaEvent_t a = nullptr, b = nullptr;
    EventPair()
    {
        cuda_ok(cudaEventCreate(&a), "cudaEventCreate");
        cuda_ok(cudaEventCreate(&b), "cudaEventCreate");
    }
    ~EventPair()
    {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
    EventPair(const EventPair&) = delete;
    EventPair& operator=(const EventPair&) = delete;
    double seconds()
    {
        float ms = 0.f;
        cuda_ok(cudaEventElapsedTime(&ms, a, b), "cudaEventElapsedTime");
        return ms * 1e-3;
    }
};

struct BenchKernelName {
    const char* name;
    BenchKind kind;
};

// bench.cpp:85-148, in the reference's order
constexpr BenchKernelName kBenchKernels[] = {
    {"sobol", QMC_BENCH_SOBOL},
    {"halton", QMC_BENCH_HALTON},
    {"halton-tabled", QMC_BENCH_HALTON_TABLED},
    {"lattice", QMC_BENCH_LATTICE},
    {"pixel-shifted-lattice", QMC_BENCH_PIXEL_SHIFTED_LATTICE},
    {"pixel-random-lattice", QMC_BENCH_PIXEL_RANDOM_LATTICE},
};

} // namespace

extern "C" {

qmc_status qmc_run_bench_kernel(const char* kernel, uint64_t count, uint32_t dims,
                                qmc_bench_result* out, qmc_stream stream)
{
    return guard([&] {
        const NvtxRange nvtx("qmc_run_bench_kernel");
        if (!kernel || !out)
            fail(QMC_INVALID_ARGUMENT, "run_bench_kernel: null argument");
        // bench.cpp:82-85
        if (count == 0)
            fail(QMC_CONFIG, "bench: count must be >= 1");
        if (dims == 0)
            fail(QMC_CONFIG, "bench: dims must be >= 1");
        const std::string name(kernel);
        const BenchKernelName* k = nullptr;
        for (const auto& e : kBenchKernels)
            if (name == e.name)
                k = &e;
        if (!k)
            fail(QMC_CONFIG, "bench: unknown kernel '" + name + "'");
        const cudaStream_t s = as_stream(stream);
        BenchParams p{};
        p.count = count;
        p.dims = dims;
        p.kind = k->kind;
        p.tab3 = digit_table(3, 0, 0).ptr;
        CallArgs args(s), pargs(s);
        std::vector<uint32_t> pool;
        std::vector<size_t> soff;
        std::vector<RadicalDim> rd;
        size_t goff = SIZE_MAX, roff = SIZE_MAX;
        switch (k->kind) {
        case QMC_BENCH_SOBOL: // build_matrices(builtin_direction_numbers(), dims)
            p.colsT = static_cast<const uint32_t*>(builtin_matrices(dims)->on_device().colsT.get());
            break;
        case QMC_BENCH_HALTON: // radical_inverse(i, j): prime index j < 1000
        case QMC_BENCH_HALTON_TABLED: // TabledHalton(dims): default linear factors
            if (dims > kPrimes)
                fail(QMC_OUT_OF_RANGE, "prime: index beyond the table");
            rd = radical_dims(dims, 0,
                              k->kind == QMC_BENCH_HALTON ? QMC_RADICAL_PLAIN : QMC_RADICAL_LINEAR,
                              nullptr, pool, soff);
            roff = args.add(rd.data(), rd.size() * sizeof(RadicalDim));
            break;
        case QMC_BENCH_LATTICE:
        case QMC_BENCH_PIXEL_SHIFTED_LATTICE: { // lfsr_generator_vector(kDefaultGeneratorSeed, dims)
            const std::vector<uint32_t> g = lfsr(0xace1u, dims);
            goff = args.add(g.data(), g.size() * 4);
            break;
        }
        case QMC_BENCH_PIXEL_RANDOM_LATTICE:
            break;
        }
        args.upload();
        if (roff != SIZE_MAX)
            p.rd = args.at<RadicalDim>(roff);
        if (goff != SIZE_MAX)
            p.g = args.at<uint32_t>(goff);
        unsigned long long* d = nullptr;
        cuda_ok(cudaMallocAsync(&d, 16, s), "cudaMallocAsync");
        // warm-up walk of count / 8 (bench.cpp:53-54), then the timed walk
        BenchParams warm = p;
        warm.count = std::max<uint64_t>(count / 8, 1);
        cuda_ok(cudaMemsetAsync(d, 0, 16, s), "memset");
        cuda_ok(launch_bench(warm, d + 1, s), "launch_bench");
        EventPair ev;
        cuda_ok(cudaEventRecord(ev.a, s), "cudaEventRecord");
        cuda_ok(launch_bench(p, d, s), "launch_bench");
        cuda_ok(cudaEventRecord(ev.b, s), "cudaEventRecord");
        unsigned long long h = 0;
        cuda_ok(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, s), "D2H");
        cudaFreeAsync(d, s);
        cuda_ok(cudaStreamSynchronize(s), "sync");
        out->evaluations = count;
        out->seconds = ev.seconds();
        out->components_per_second = out->seconds > 0.0 ? count / out->seconds : 0.0;
        out->checksum = h;
    });
}

qmc_status qmc_fp64_probe(uint32_t iters, double* flops_per_second, qmc_stream stream)
{
    return guard([&] {
        if (!flops_per_second || iters == 0)
            fail(QMC_INVALID_ARGUMENT, "fp64_probe: null output or zero iterations");
        const cudaStream_t s = as_stream(stream);
        const uint64_t threads = fp64_probe_threads();
        double* d = nullptr;
        cuda_ok(cudaMallocAsync(&d, threads * 8, s), "cudaMallocAsync");
        cuda_ok(launch_fp64_probe(d, threads, std::max(iters / 8, 1u), s), "launch_fp64_probe");
        EventPair ev;
        cuda_ok(cudaEventRecord(ev.a, s), "cudaEventRecord");
        cuda_ok(launch_fp64_probe(d, threads, iters, s), "launch_fp64_probe");
        cuda_ok(cudaEventRecord(ev.b, s), "cudaEventRecord");
        cudaFreeAsync(d, s);
        cuda_ok(cudaStreamSynchronize(s), "sync");
        *flops_per_second = fp64_probe_flops(threads, iters) / ev.seconds();
    });
}

} // extern "C"
