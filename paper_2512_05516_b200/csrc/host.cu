// Host-resident particle orchestration (C4): the paper's stream-vs-in-place
// question (pipelines.cpp:231-296, PAPER §6) re-posed for a PCIe-attached
// B200.
//
//   STREAMED  pinned host AoS, chunked: on each of 3 rotating streams
//             H2D(chunk) -> fused gather+kernel -> [more kernels on SoA]
//             -> scatter-merge write sets into the AoS chunk -> D2H(chunk).
//             The copy engines (H2D, D2H) and the SMs overlap across chunks.
//   MANAGED   cudaMallocManaged AoS (preferred location: host); per chunk
//             cudaMemPrefetchAsync to the GPU, the same kernels run in place
//             on the migrated pages, prefetch back to the host.
//
// Either way the whole record moves each way (88 B/particle at the default
// schema), conversion happens on the GPU, and the AoS in host memory ends up
// exactly as the reference's run_dev_inplace would leave it for a DevSoA
// composition of the same kernels.
#include <cuda_runtime.h>

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "runtime.hpp"

namespace sfb {

namespace {

struct DeviceSlots {
    std::vector<void*> aos, soa;
    std::vector<cudaStream_t> streams;
    size_t aos_bytes = 0, soa_bytes = 0;
    ~DeviceSlots() {
        for (void* p : aos) cudaFree(p);
        for (void* p : soa) cudaFree(p);
        for (auto s : streams) cudaStreamDestroy(s);
    }
};

View with_count(const View& v, uint64_t count) {
    View c = v;
    c.count = count;
    return c;
}

}  // namespace

void run_host(const View& src, void* host, const View& dst, const std::string& kernels, double dt, int math, int mode,
              uint64_t chunk, void* host_soa, double* metrics) {
    require_device();
    if (src.layout != Layout::AoS || src.subset.size() != src.schema->fields.size())
        throw std::invalid_argument("run_host expects an AoS view over the full field set");
    if (dst.layout != Layout::SoA) throw std::invalid_argument("run_host computes on an SoA view");
    std::vector<std::string> ks = split_names(kernels);
    if (ks.empty()) throw std::invalid_argument("no kernels given");
    for (const auto& k : ks)
        if (k != "kick" && k != "drift") throw std::invalid_argument("run_host runs kick and drift");
    if (chunk == 0) chunk = 1ull << 22;
    chunk = (chunk + 127) / 128 * 128;  // 16-B aligned chunk starts for any record width
    const uint64_t n = src.count;
    const uint64_t rb = src.record_bits();
    const int slots = 3;

    cudaPointerAttributes attr{};
    check_cuda(cudaPointerGetAttributes(&attr, host), "pointer attributes");
    if (mode == 0 && attr.type != cudaMemoryTypeHost)
        throw std::invalid_argument("streamed mode needs pinned host memory (sf_b200_host_alloc mode 0)");
    if (mode == 1 && attr.type != cudaMemoryTypeManaged)
        throw std::invalid_argument("managed mode needs cudaMallocManaged memory (sf_b200_host_alloc mode 1)");
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "device");

    static thread_local std::unique_ptr<DeviceSlots> pool;
    const size_t aos_bytes = size_t((chunk * rb + 7) / 8);
    const size_t soa_bytes = size_t(with_count(dst, chunk).total_bytes());
    if (!pool || pool->aos_bytes < aos_bytes || pool->soa_bytes < soa_bytes) {
        pool.reset(new DeviceSlots());
        pool->aos_bytes = aos_bytes;
        pool->soa_bytes = soa_bytes;
        for (int s = 0; s < slots; ++s) {
            void* a = nullptr;
            void* b = nullptr;
            check_cuda(cudaMalloc(&a, aos_bytes), "cudaMalloc");
            check_cuda(cudaMalloc(&b, soa_bytes), "cudaMalloc");
            pool->aos.push_back(a);
            pool->soa.push_back(b);
            cudaStream_t st;
            check_cuda(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
            pool->streams.push_back(st);
        }
    }
    if (mode == 1) {
        const size_t total = size_t((n * rb + 7) / 8);
        cudaMemLocation loc{};
        loc.type = cudaMemLocationTypeHost;
        loc.id = 0;
        (void)loc;
        check_cuda(cudaMemAdvise(host, total, cudaMemAdviseSetPreferredLocation, cudaCpuDeviceId), "advise");
        check_cuda(cudaMemAdvise(host, total, cudaMemAdviseSetAccessedBy, dev), "advise");
    }

    cudaEvent_t t0, t1;
    check_cuda(cudaEventCreate(&t0), "event");
    check_cuda(cudaEventCreate(&t1), "event");
    std::vector<cudaEvent_t> done(slots);
    for (auto& e : done) check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    check_cuda(cudaDeviceSynchronize(), "sync");
    check_cuda(cudaEventRecord(t0, pool->streams[0]), "record");
    for (int s = 1; s < slots; ++s) check_cuda(cudaStreamWaitEvent(pool->streams[s], t0, 0), "wait");

    uint64_t h2d = 0, d2h = 0, nchunks = 0;
    const uint64_t launches0 = launch_count();
    for (uint64_t r0 = 0; r0 < n; r0 += chunk, ++nchunks) {
        const int s = int(nchunks % slots);
        cudaStream_t st = pool->streams[s];
        const uint64_t cnt = std::min(chunk, n - r0);
        const size_t off = size_t(r0 * rb / 8);
        const size_t bytes = size_t((cnt * rb + 7) / 8);
        uint8_t* hchunk = static_cast<uint8_t*>(host) + off;
        void* aos = mode == 0 ? pool->aos[s] : static_cast<void*>(hchunk);
        if (mode == 0) {
            check_cuda(cudaMemcpyAsync(aos, hchunk, bytes, cudaMemcpyHostToDevice, st), "H2D");
        } else {
            check_cuda(cudaMemPrefetchAsync(hchunk, bytes, dev, st), "prefetch");
        }
        h2d += bytes;
        const View sv = with_count(src, cnt), dv = with_count(dst, cnt);
        gather(sv, aos, dv, pool->soa[s], ks[0].c_str(), dt, math, st);
        for (size_t k = 1; k < ks.size(); ++k) run_kernel(dv, pool->soa[s], ks[k], dt, 1, 0, math, st);
        if (host_soa) {
            // SoA result straight to host: one D2H per stream of the chunk
            for (size_t p = 0; p < dv.subset.size(); ++p) {
                const uint64_t lane_bytes = uint64_t(dv.arity(int(p))) * dv.width(int(p)) / 8;
                const uint64_t full_base = dst.lane_base(int(p)) / 8, chunk_base = dv.lane_base(int(p)) / 8;
                check_cuda(cudaMemcpyAsync(static_cast<uint8_t*>(host_soa) + full_base + r0 * lane_bytes,
                                           static_cast<uint8_t*>(pool->soa[s]) + chunk_base, cnt * lane_bytes,
                                           cudaMemcpyDeviceToHost, st),
                           "D2H");
                d2h += cnt * lane_bytes;
            }
            if (mode == 1) check_cuda(cudaMemPrefetchAsync(hchunk, bytes, cudaCpuDeviceId, st), "prefetch");
        } else {
            for (const auto& k : ks) scatter_merge(dv, pool->soa[s], sv, aos, k, st);
            if (mode == 0) {
                check_cuda(cudaMemcpyAsync(hchunk, aos, bytes, cudaMemcpyDeviceToHost, st), "D2H");
            } else {
                check_cuda(cudaMemPrefetchAsync(hchunk, bytes, cudaCpuDeviceId, st), "prefetch");
            }
            d2h += bytes;
        }
    }
    for (int s = 0; s < slots; ++s) {
        check_cuda(cudaEventRecord(done[s], pool->streams[s]), "record");
        check_cuda(cudaStreamWaitEvent(pool->streams[0], done[s], 0), "wait");
    }
    check_cuda(cudaEventRecord(t1, pool->streams[0]), "record");
    check_cuda(cudaEventSynchronize(t1), "sync");
    float ms = 0;
    check_cuda(cudaEventElapsedTime(&ms, t0, t1), "elapsed");
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    for (auto& e : done) cudaEventDestroy(e);
    metrics[0] = ms * 1e-3;
    metrics[1] = double(h2d);
    metrics[2] = double(d2h);
    metrics[3] = double(nchunks);
    metrics[4] = double(launch_count() - launches0);
}

}  // namespace sfb
