// abi_render.cpp — the fused per-pixel render of the C ABI (render.cpp:58-143
// on the device): qmc_render, the sample-partitioned qmc_render_partial /
// qmc_render_finalize, and qmc_scene_value.
#include <cstdlib>
#include "objects.hpp"

#include <string>
#include <thread>
#include <vector>

using namespace qmcgpu;
using namespace qmcgpu::host;

extern "C" {

// ------------------------------------------------------------------ render

namespace {

// row bands of a host-image render (D2H of band b overlaps the render of b+1)
constexpr uint32_t kRenderHostBands = 8;

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
    p.divw = job->width >= 2 ? make_div32(job->width) : Div32{0, 0};
    p.small_band = static_cast<uint64_t>(row_end - row_begin) * job->width < (1ull << 32) ? 1u : 0u;
    p.inv_spp = (job->spp & (job->spp - 1)) == 0 ? 1.0 / job->spp : 0.0;
    p.colmap = job->spp >= 8 ? render_column_order(job->width) : nullptr;
    p.q3 = render_phi3_quotients();
    p.t3q3 = render_t3q3();
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
    p.sc = make_scene_consts();
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
        p.stride_magic = p.stride >= 2 && p.stride < (1ull << 32) ? ~0ull / p.stride : 0;
        p.dlo3 = he.sx % 2187u;
        p.dhi3 = he.sx / 2187u;
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
        const NvtxRange nvtx("qmc_render");
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
        // Host image: render in row bands and copy each band to the host on
        // a second stream while the next band renders, so the D2H (PCIe)
        // overlaps the render instead of following it. Small images: one band.
        const uint32_t rows = row_end - row_begin;
        const char* env = std::getenv("QMC_RENDER_BANDS"); // A/B: tools/exp_render_e2e.py
        const uint32_t want = env ? static_cast<uint32_t>(std::atoi(env)) : kRenderHostBands;
        const uint32_t nb = rr.npix >= (1ull << 20) ? std::max(1u, std::min(want, rows)) : 1u;
        if (nb == 1) {
            cuda_ok(launch_render(rr.p, job->kind, job->accum, d, s), "launch_render");
            cuda_ok(cudaMemcpyAsync(out, d, rr.npix * 4, cudaMemcpyDeviceToHost, s), "D2H");
        } else {
            // the copy stream and events die with the call, also on an error
            struct Side {
                cudaStream_t c = nullptr;
                std::vector<cudaEvent_t> ev;
                ~Side()
                {
                    for (cudaEvent_t e : ev)
                        if (e)
                            cudaEventDestroy(e);
                    if (c)
                        cudaStreamDestroy(c);
                }
            } side;
            side.ev.assign(nb + 1, nullptr);
            cuda_ok(cudaStreamCreateWithFlags(&side.c, cudaStreamNonBlocking), "cudaStreamCreate");
            for (auto& e : side.ev)
                cuda_ok(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
            const cudaStream_t c = side.c;
            std::vector<cudaEvent_t>& ev = side.ev;
            for (uint32_t b = 0; b < nb; ++b) {
                const uint32_t rb = row_begin + static_cast<uint32_t>(uint64_t(rows) * b / nb);
                const uint32_t re = row_begin + static_cast<uint32_t>(uint64_t(rows) * (b + 1) / nb);
                RenderParams pb = rr.p;
                pb.row_begin = rb;
                pb.row_end = re;
                const uint64_t off = static_cast<uint64_t>(rb - row_begin) * job->width;
                const uint64_t cnt = static_cast<uint64_t>(re - rb) * job->width;
                cuda_ok(launch_render(pb, job->kind, job->accum, d + off, s), "launch_render");
                cuda_ok(cudaEventRecord(ev[b], s), "cudaEventRecord");
                cuda_ok(cudaStreamWaitEvent(c, ev[b], 0), "cudaStreamWaitEvent");
                cuda_ok(cudaMemcpyAsync(out + off, d + off, cnt * 4, cudaMemcpyDeviceToHost, c),
                        "D2H");
            }
            cuda_ok(cudaEventRecord(ev[nb], c), "cudaEventRecord");
            cuda_ok(cudaStreamWaitEvent(s, ev[nb], 0), "cudaStreamWaitEvent"); // before the free
        }
        cudaFreeAsync(d, s);
        cuda_ok(cudaStreamSynchronize(s), "sync");
    });
}

qmc_status qmc_render_partial(const qmc_render_job* job, uint32_t part, uint32_t parts,
                              uint32_t row_begin, uint32_t row_end, int64_t* accum,
                              qmc_stream stream)
{
    return guard([&] {
        const NvtxRange nvtx("qmc_render_partial");
        const cudaStream_t s = as_stream(stream);
        if (job && job->accum != QMC_ACCUM_INT)
            fail(QMC_INVALID_ARGUMENT,
                 "render_partial: sample partitions need the int accumulator (exactly associative)");
        uint64_t rem = 0, mod = 1;
        const qmc_status st = qmc_partition_by_extra_dimension(part, parts, 2, &rem, &mod);
        if (st != QMC_OK)
            fail(st, last_error());
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
        const NvtxRange nvtx("qmc_render_finalize");
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

qmc_status qmc_render_devices(const qmc_render_job* job, const int* devices, uint32_t n_devices,
                              float* out)
{
    return guard([&] {
        const NvtxRange nvtx("qmc_render_devices");
        if (!job)
            fail(QMC_INVALID_ARGUMENT, "render job is null");
        if (!devices || n_devices == 0)
            fail(QMC_INVALID_ARGUMENT, "qmc_render_devices: the device list is empty");
        if (!out)
            fail(QMC_INVALID_ARGUMENT, "output pointer is null");
        if (is_device_pointer(out))
            fail(QMC_INVALID_ARGUMENT, "qmc_render_devices: out must be host memory");
        int prev = 0;
        cuda_ok(cudaGetDevice(&prev), "cudaGetDevice");
        // one host thread per device renders its row band (the single-GPU
        // per-pixel order, so the assembled image is bit-identical) and
        // copies it into its rows of `out`
        std::vector<qmc_status> st(n_devices, QMC_OK);
        std::vector<std::string> msg(n_devices);
        std::vector<std::thread> workers;
        for (uint32_t k = 0; k < n_devices; ++k) {
            const uint32_t r0 = static_cast<uint32_t>(uint64_t(job->height) * k / n_devices);
            const uint32_t r1 = static_cast<uint32_t>(uint64_t(job->height) * (k + 1) / n_devices);
            workers.emplace_back([&, k, r0, r1] {
                if (cudaSetDevice(devices[k]) != cudaSuccess) {
                    st[k] = QMC_CUDA;
                    msg[k] = "qmc_render_devices: cudaSetDevice failed";
                    return;
                }
                cudaStream_t s = nullptr;
                if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
                    st[k] = QMC_CUDA;
                    msg[k] = "qmc_render_devices: cudaStreamCreate failed";
                    return;
                }
                st[k] = qmc_render(job, r0, r1, out + uint64_t(r0) * job->width, s);
                if (st[k] != QMC_OK)
                    msg[k] = qmc_last_error();
                cudaStreamSynchronize(s);
                cudaStreamDestroy(s);
            });
        }
        for (auto& w : workers)
            w.join();
        cudaSetDevice(prev);
        for (uint32_t k = 0; k < n_devices; ++k)
            if (st[k] != QMC_OK)
                fail(st[k], msg[k]);
    });
}

namespace {

// RAII: a non-blocking stream on the current device, destroyed last.
struct OwnedStream {
    cudaStream_t s = nullptr;
    OwnedStream() { cuda_ok(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate"); }
    ~OwnedStream()
    {
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    }
    OwnedStream(const OwnedStream&) = delete;
    OwnedStream& operator=(const OwnedStream&) = delete;
};

// RAII: restores the calling thread's current device.
struct DeviceRestore {
    int prev = 0;
    DeviceRestore() { cuda_ok(cudaGetDevice(&prev), "cudaGetDevice"); }
    ~DeviceRestore() { cudaSetDevice(prev); }
};

} // namespace

qmc_status qmc_render_samples_devices(const qmc_render_job* job, const int* devices,
                                      uint32_t n_devices, float* out)
{
    return guard([&] {
        const NvtxRange nvtx("qmc_render_samples_devices");
        if (!job)
            fail(QMC_INVALID_ARGUMENT, "render job is null");
        if (job->accum != QMC_ACCUM_INT)
            fail(QMC_INVALID_ARGUMENT,
                 "render_samples: sample partitions need the int accumulator (exactly associative)");
        if (!devices || n_devices == 0 || (n_devices & (n_devices - 1)) != 0)
            fail(QMC_INVALID_ARGUMENT,
                 "qmc_render_samples_devices: the device count must be a power of two");
        if (!out)
            fail(QMC_INVALID_ARGUMENT, "output pointer is null");
        if (is_device_pointer(out))
            fail(QMC_INVALID_ARGUMENT, "qmc_render_samples_devices: out must be host memory");
        const DeviceRestore restore;
        const int home = devices[0];
        cuda_ok(cudaSetDevice(home), "cudaSetDevice");
        const OwnedStream hs; // declared first: destroyed after everything below
        uint64_t npix = 0;
        {
            CallArgs hargs(hs.s);
            ResolvedRender hr; // validates the job
            resolve_render(job, 0, job->height, hs.s, hargs, hr);
            npix = hr.npix;
            cuda_ok(cudaStreamSynchronize(hs.s), "sync");
        }
        if (npix == 0)
            return;
        // the one accumulator, on the first device
        long long* acc = nullptr;
        cuda_ok(cudaMalloc(&acc, npix * 8 + 8), "cudaMalloc");
        const std::unique_ptr<long long, DevFree> acc_own(acc);
        // zeroed on the home stream and waited for before any worker starts:
        // the workers' non-blocking streams (and the peer devices' streams)
        // have no ordering with the legacy stream a plain cudaMemset uses
        cuda_ok(cudaMemsetAsync(acc, 0, npix * 8, hs.s), "cudaMemsetAsync");
        cuda_ok(cudaStreamSynchronize(hs.s), "sync");
        // part k of n (samples i == rev_2(k) mod n) on devices[k]: one kernel
        // renders and atomically adds its int64 partials into the
        // accumulator — over NVLink peer access when the device differs
        std::vector<qmc_status> st(n_devices, QMC_OK);
        std::vector<std::string> msg(n_devices);
        std::vector<std::thread> workers;
        for (uint32_t k = 0; k < n_devices; ++k) {
            workers.emplace_back([&, k] {
                st[k] = guard([&] {
                    cuda_ok(cudaSetDevice(devices[k]), "cudaSetDevice");
                    if (devices[k] != home) {
                        int can = 0;
                        cuda_ok(cudaDeviceCanAccessPeer(&can, devices[k], home),
                                "cudaDeviceCanAccessPeer");
                        if (!can)
                            fail(QMC_CUDA, "qmc_render_samples_devices: no peer access to the "
                                           "accumulator's device");
                        const cudaError_t e = cudaDeviceEnablePeerAccess(home, 0);
                        if (e == cudaErrorPeerAccessAlreadyEnabled)
                            cudaGetLastError(); // clear
                        else
                            cuda_ok(e, "cudaDeviceEnablePeerAccess");
                    }
                    uint64_t rem = 0, mod = 1;
                    const qmc_status ps =
                        qmc_partition_by_extra_dimension(k, n_devices, 2, &rem, &mod);
                    if (ps != QMC_OK)
                        fail(ps, last_error());
                    const OwnedStream s;
                    CallArgs args(s.s);
                    ResolvedRender rr;
                    resolve_render(job, 0, job->height, s.s, args, rr);
                    cuda_ok(launch_render_partial(rr.p, job->kind, static_cast<uint32_t>(rem),
                                                  static_cast<uint32_t>(mod), acc, s.s, true),
                            "launch_render_partial");
                    cuda_ok(cudaStreamSynchronize(s.s), "sync");
                });
                if (st[k] != QMC_OK)
                    msg[k] = qmc_last_error();
            });
        }
        for (auto& w : workers)
            w.join();
        for (uint32_t k = 0; k < n_devices; ++k)
            if (st[k] != QMC_OK)
                fail(st[k], msg[k]);
        cuda_ok(cudaSetDevice(home), "cudaSetDevice");
        float* d = nullptr;
        cuda_ok(cudaMalloc(&d, npix * 4 + 4), "cudaMalloc");
        const DevPtr d_own(d);
        cuda_ok(launch_render_finalize(acc, npix, job->spp, d, hs.s), "launch_render_finalize");
        cuda_ok(cudaMemcpyAsync(out, d, npix * 4, cudaMemcpyDeviceToHost, hs.s), "D2H");
        cuda_ok(cudaStreamSynchronize(hs.s), "sync");
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

