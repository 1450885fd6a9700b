// abi_nccl.cpp — the one collective of the multi-GPU render, inside the
// library. The reference renders with a host worker pool
// (render.cpp:114-139): workers take pixels round-robin and write their own
// pixels of one ImageBuffer. Across GPUs the same job splits either into row
// bands (every pixel keeps the one-GPU summation order, so the image is
// bit-identical) followed by one ncclAllGather of the fp32 bands, or into the
// paper's sample partition (partition_by_extra_dimension, imageplane.cpp:
// 114-130) followed by one ncclAllReduce(sum) of the int64
// per-pixel accumulators and the finalize (exactly associative, so again
// bit-identical to the one-GPU int render).
//
// NCCL is loaded on first use (dlopen "libnccl.so.2"; an already-loaded copy
// — e.g. the one a PyTorch process maps — is preferred; QMC_NCCL_LIBRARY
// overrides the path), so the library has no link-time NCCL dependency and
// never pulls a second NCCL into a process that already has one.
#include "objects.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>

using namespace qmcgpu;
using namespace qmcgpu::host;

struct qmc_comm {
    ncclComm_t comm = nullptr;
    int rank = 0, nranks = 1, device = 0;
    bool owned = true;
};

namespace {

struct NcclApi {
    decltype(&ncclGetVersion) GetVersion = nullptr;
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommInitAll) CommInitAll = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclCommCount) CommCount = nullptr;
    decltype(&ncclCommUserRank) CommUserRank = nullptr;
    decltype(&ncclCommCuDevice) CommCuDevice = nullptr;
    decltype(&ncclAllGather) AllGather = nullptr;
    decltype(&ncclAllReduce) AllReduce = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
    void* handle = nullptr;
    std::string error;
};

const NcclApi& nccl()
{
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = nullptr;
        if (const char* path = std::getenv("QMC_NCCL_LIBRARY"); path && *path)
            h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
        if (!h)
            h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h)
            h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) {
            const char* e = dlerror();
            api.error = std::string("NCCL not available: ") + (e ? e : "dlopen failed");
            return;
        }
        bool ok = true;
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            ok = ok && fn != nullptr;
        };
        sym(api.GetVersion, "ncclGetVersion");
        sym(api.GetUniqueId, "ncclGetUniqueId");
        sym(api.CommInitRank, "ncclCommInitRank");
        sym(api.CommInitAll, "ncclCommInitAll");
        sym(api.CommDestroy, "ncclCommDestroy");
        sym(api.CommCount, "ncclCommCount");
        sym(api.CommUserRank, "ncclCommUserRank");
        sym(api.CommCuDevice, "ncclCommCuDevice");
        sym(api.AllGather, "ncclAllGather");
        sym(api.AllReduce, "ncclAllReduce");
        sym(api.GroupStart, "ncclGroupStart");
        sym(api.GroupEnd, "ncclGroupEnd");
        sym(api.GetErrorString, "ncclGetErrorString");
        if (!ok) {
            api.error = "NCCL library lacks a required symbol";
            return;
        }
        api.handle = h;
    });
    if (!api.handle)
        fail(QMC_NCCL, api.error);
    return api;
}

void nccl_ok(ncclResult_t r, const char* what)
{
    if (r != ncclSuccess)
        fail(QMC_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

void fill_info(qmc_comm& c)
{
    nccl_ok(nccl().CommUserRank(c.comm, &c.rank), "ncclCommUserRank");
    nccl_ok(nccl().CommCount(c.comm, &c.nranks), "ncclCommCount");
    nccl_ok(nccl().CommCuDevice(c.comm, &c.device), "ncclCommCuDevice");
}

// Rows [r0, r1) of rank `rank`'s band: ceil(H / n) rows per rank, the last
// bands clipped (possibly empty), so the all-gather is over equal counts and
// every padding row lands after row H - 1.
struct Band {
    uint32_t per, r0, r1;
};

Band band_of(uint32_t height, int rank, int nranks)
{
    const uint32_t per = (height + nranks - 1) / nranks;
    const uint64_t a = std::min<uint64_t>(uint64_t(per) * rank, height);
    const uint64_t b = std::min<uint64_t>(uint64_t(per) * (rank + 1), height);
    return {per, static_cast<uint32_t>(a), static_cast<uint32_t>(b)};
}

void check_status(qmc_status st)
{
    if (st != QMC_OK)
        fail(st, last_error());
}

// Enqueues this rank's share of the render and the collective on `s`; the
// full image lands in `out` (device memory of the communicator's GPU).
// Scratch is stream-ordered (cudaMallocAsync / cudaFreeAsync on `s`), so the
// call never synchronizes and the pool keeps the buffer between calls.
void render_nccl_enqueue(const qmc_render_job* job, const qmc_comm& c, qmc_partition mode,
                         float* out, cudaStream_t s)
{
    const uint64_t npix = uint64_t(job->height) * job->width;
    if (mode == QMC_PARTITION_ROWS) {
        const Band b = band_of(job->height, c.rank, c.nranks);
        const uint64_t count = uint64_t(b.per) * job->width;
        const bool in_place = uint64_t(b.per) * c.nranks == job->height;
        float* base = out;
        if (!in_place)
            cuda_ok(cudaMallocAsync(reinterpret_cast<void**>(&base), count * c.nranks * 4 + 4, s),
                    "cudaMallocAsync");
        float* mine = base + count * c.rank;
        if (b.r1 > b.r0)
            check_status(qmc_render(job, b.r0, b.r1, mine, s));
        nccl_ok(nccl().AllGather(mine, base, count, ncclFloat, c.comm, s), "ncclAllGather");
        if (!in_place) {
            cuda_ok(cudaMemcpyAsync(out, base, npix * 4, cudaMemcpyDeviceToDevice, s), "D2D");
            cuda_ok(cudaFreeAsync(base, s), "cudaFreeAsync");
        }
        return;
    }
    if (mode != QMC_PARTITION_SAMPLES)
        fail(QMC_INVALID_ARGUMENT, "render_nccl: unknown partition mode");
    int64_t* acc = nullptr;
    cuda_ok(cudaMallocAsync(reinterpret_cast<void**>(&acc), npix * 8 + 8, s), "cudaMallocAsync");
    check_status(qmc_render_partial(job, static_cast<uint32_t>(c.rank),
                                    static_cast<uint32_t>(c.nranks), 0, job->height, acc, s));
    nccl_ok(nccl().AllReduce(acc, acc, npix, ncclInt64, ncclSum, c.comm, s), "ncclAllReduce");
    check_status(qmc_render_finalize(acc, npix, job->spp, out, s));
    cuda_ok(cudaFreeAsync(acc, s), "cudaFreeAsync");
}

void validate_job(const qmc_render_job* job, qmc_partition mode, int nranks)
{
    if (!job)
        fail(QMC_INVALID_ARGUMENT, "render job is null");
    if (mode == QMC_PARTITION_SAMPLES) {
        if (job->accum != QMC_ACCUM_INT)
            fail(QMC_INVALID_ARGUMENT, "render_nccl: sample partitions need the int accumulator "
                                       "(exactly associative)");
        if (nranks <= 0 || (nranks & (nranks - 1)) != 0)
            fail(QMC_INVALID_ARGUMENT,
                 "render_nccl: sample partitions need a power-of-two rank count");
    } else if (mode != QMC_PARTITION_ROWS) {
        fail(QMC_INVALID_ARGUMENT, "render_nccl: unknown partition mode");
    }
}

} // namespace

extern "C" {

qmc_status qmc_nccl_version(int* version)
{
    return guard([&] {
        if (!version)
            fail(QMC_INVALID_ARGUMENT, "version pointer is null");
        nccl_ok(nccl().GetVersion(version), "ncclGetVersion");
    });
}

qmc_status qmc_comm_unique_id(void* id)
{
    return guard([&] {
        if (!id)
            fail(QMC_INVALID_ARGUMENT, "unique id buffer is null");
        ncclUniqueId u;
        nccl_ok(nccl().GetUniqueId(&u), "ncclGetUniqueId");
        std::memcpy(id, &u, sizeof u);
    });
}

qmc_status qmc_comm_init_rank(const void* id, int nranks, int rank, qmc_comm** out)
{
    return guard([&] {
        if (!id || !out)
            fail(QMC_INVALID_ARGUMENT, "qmc_comm_init_rank: null argument");
        if (nranks < 1 || rank < 0 || rank >= nranks)
            fail(QMC_INVALID_ARGUMENT, "qmc_comm_init_rank: rank outside [0, nranks)");
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof u);
        auto c = std::make_unique<qmc_comm>();
        nccl_ok(nccl().CommInitRank(&c->comm, nranks, u, rank), "ncclCommInitRank");
        fill_info(*c);
        *out = c.release();
    });
}

qmc_status qmc_comm_init_all(const int* devices, int n, qmc_comm** out)
{
    return guard([&] {
        if (!devices || n < 1 || !out)
            fail(QMC_INVALID_ARGUMENT, "qmc_comm_init_all: empty device list");
        const DeviceRestoreGuard keep;
        std::vector<ncclComm_t> comms(n);
        nccl_ok(nccl().CommInitAll(comms.data(), n, devices), "ncclCommInitAll");
        for (int k = 0; k < n; ++k) {
            auto c = std::make_unique<qmc_comm>();
            c->comm = comms[k];
            fill_info(*c);
            out[k] = c.release();
        }
    });
}

qmc_status qmc_comm_from_nccl(void* nccl_comm, qmc_comm** out)
{
    return guard([&] {
        if (!nccl_comm || !out)
            fail(QMC_INVALID_ARGUMENT, "qmc_comm_from_nccl: null argument");
        auto c = std::make_unique<qmc_comm>();
        c->comm = static_cast<ncclComm_t>(nccl_comm);
        c->owned = false;
        fill_info(*c);
        *out = c.release();
    });
}

qmc_status qmc_comm_info(const qmc_comm* comm, int* rank, int* nranks, int* device)
{
    return guard([&] {
        if (!comm)
            fail(QMC_INVALID_ARGUMENT, "communicator is null");
        if (rank)
            *rank = comm->rank;
        if (nranks)
            *nranks = comm->nranks;
        if (device)
            *device = comm->device;
    });
}

void qmc_comm_destroy(qmc_comm* comm)
{
    if (!comm)
        return;
    if (comm->owned && comm->comm)
        nccl().CommDestroy(comm->comm);
    delete comm;
}

qmc_status qmc_render_nccl(const qmc_render_job* job, const qmc_comm* comm, qmc_partition mode,
                           float* out, qmc_stream stream)
{
    return guard([&] {
        const NvtxRange nvtx("qmc_render_nccl");
        if (!comm)
            fail(QMC_INVALID_ARGUMENT, "communicator is null");
        validate_job(job, mode, comm->nranks);
        if (uint64_t(job->height) * job->width == 0 || job->spp == 0) {
            // qmc_render's own validation and messages
            check_status(qmc_render(job, 0, job->height, out, stream));
            return;
        }
        if (!out || !is_device_pointer(out))
            fail(QMC_INVALID_ARGUMENT, "render_nccl: out must be device memory");
        const DeviceRestoreGuard keep;
        cuda_ok(cudaSetDevice(comm->device), "cudaSetDevice");
        render_nccl_enqueue(job, *comm, mode, out, as_stream(stream));
    });
}

qmc_status qmc_render_nccl_devices(const qmc_render_job* job, const int* devices,
                                   uint32_t n_devices, qmc_partition mode, float* out)
{
    return guard([&] {
        const NvtxRange nvtx("qmc_render_nccl_devices");
        if (!devices || n_devices == 0)
            fail(QMC_INVALID_ARGUMENT, "qmc_render_nccl_devices: the device list is empty");
        validate_job(job, mode, static_cast<int>(n_devices));
        if (!out)
            fail(QMC_INVALID_ARGUMENT, "output pointer is null");
        if (is_device_pointer(out))
            fail(QMC_INVALID_ARGUMENT, "qmc_render_nccl_devices: out must be host memory");
        const uint64_t npix = uint64_t(job->height) * job->width;
        if (npix == 0 || job->spp == 0) {
            check_status(qmc_render(job, 0, job->height, out, nullptr));
            return;
        }
        const DeviceRestoreGuard keep;
        const uint32_t n = n_devices;
        std::vector<qmc_comm*> comms(n, nullptr);
        check_status(qmc_comm_init_all(devices, static_cast<int>(n), comms.data()));
        struct Rank {
            cudaStream_t s = nullptr;
            DevPtr image, scratch;
        };
        std::vector<Rank> ranks(n);
        auto cleanup = [&] {
            for (uint32_t k = 0; k < n; ++k) {
                cudaSetDevice(devices[k]);
                if (ranks[k].s) {
                    cudaStreamSynchronize(ranks[k].s);
                    cudaStreamDestroy(ranks[k].s);
                }
                ranks[k].image.reset();
                ranks[k].scratch.reset();
                qmc_comm_destroy(comms[k]);
            }
        };
        try {
            for (uint32_t k = 0; k < n; ++k) {
                cuda_ok(cudaSetDevice(devices[k]), "cudaSetDevice");
                cuda_ok(cudaStreamCreateWithFlags(&ranks[k].s, cudaStreamNonBlocking),
                        "cudaStreamCreate");
            }
            // one host thread drives every rank: the renders are launched
            // per device, the collectives of all ranks form one NCCL group
            for (uint32_t k = 0; k < n; ++k) {
                cuda_ok(cudaSetDevice(devices[k]), "cudaSetDevice");
                const qmc_comm& c = *comms[k];
                const cudaStream_t s = ranks[k].s;
                if (mode == QMC_PARTITION_ROWS) {
                    const Band b = band_of(job->height, c.rank, c.nranks);
                    const uint64_t count = uint64_t(b.per) * job->width;
                    void* p = nullptr;
                    cuda_ok(cudaMalloc(&p, count * n * 4 + 4), "cudaMalloc");
                    ranks[k].scratch.reset(p);
                    if (b.r1 > b.r0)
                        check_status(qmc_render(job, b.r0, b.r1,
                                                static_cast<float*>(p) + count * c.rank, s));
                } else {
                    void* p = nullptr;
                    cuda_ok(cudaMalloc(&p, npix * 8 + 8), "cudaMalloc");
                    ranks[k].scratch.reset(p);
                    check_status(qmc_render_partial(job, k, n, 0, job->height,
                                                    static_cast<int64_t*>(p), s));
                }
            }
            nccl_ok(nccl().GroupStart(), "ncclGroupStart");
            for (uint32_t k = 0; k < n; ++k) {
                const qmc_comm& c = *comms[k];
                void* p = ranks[k].scratch.get();
                if (mode == QMC_PARTITION_ROWS) {
                    const Band b = band_of(job->height, c.rank, c.nranks);
                    const uint64_t count = uint64_t(b.per) * job->width;
                    float* base = static_cast<float*>(p);
                    nccl_ok(nccl().AllGather(base + count * c.rank, base, count, ncclFloat, c.comm,
                                             ranks[k].s),
                            "ncclAllGather");
                } else {
                    nccl_ok(nccl().AllReduce(p, p, npix, ncclInt64, ncclSum, c.comm, ranks[k].s),
                            "ncclAllReduce");
                }
            }
            nccl_ok(nccl().GroupEnd(), "ncclGroupEnd");
            // every rank now holds the image; rank 0 finalizes / copies out
            cuda_ok(cudaSetDevice(devices[0]), "cudaSetDevice");
            const cudaStream_t s0 = ranks[0].s;
            const float* src = static_cast<const float*>(ranks[0].scratch.get());
            if (mode == QMC_PARTITION_SAMPLES) {
                void* p = nullptr;
                cuda_ok(cudaMalloc(&p, npix * 4 + 4), "cudaMalloc");
                ranks[0].image.reset(p);
                float* img = static_cast<float*>(p);
                check_status(qmc_render_finalize(static_cast<const int64_t*>(ranks[0].scratch.get()),
                                                 npix, job->spp, img, s0));
                src = img;
            }
            cuda_ok(cudaMemcpyAsync(out, src, npix * 4, cudaMemcpyDeviceToHost, s0), "D2H");
            for (uint32_t k = 0; k < n; ++k) {
                cuda_ok(cudaSetDevice(devices[k]), "cudaSetDevice");
                cuda_ok(cudaStreamSynchronize(ranks[k].s), "sync");
            }
        } catch (...) {
            cleanup();
            throw;
        }
        cleanup();
    });
}

} // extern "C"
