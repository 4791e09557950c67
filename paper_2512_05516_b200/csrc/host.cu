// Host-resident particle orchestration (C4): the paper's streaming vs
// in-place question (pipelines.cpp:231-296, §6) re-posed for a
// PCIe-attached B200.  Three modes, all chunked over 3 rotating streams so
// the two copy engines and the SMs overlap (H2D k+1 ∥ compute k ∥ D2H k-1):
//
//   STREAMED (0) pinned host AoS, zero copy: the gather kernel reads only
//                the fields of the SoA view straight from the host records
//                over PCIe (per-lane typed loads of the mapped pinned
//                memory, no whole-record tiles) and the scatter-back writes
//                only the write set's lanes into them — the reference's
//                run_dev_streaming ships just the narrowed records
//                (streamed_bytes_one_way, pipelines.cpp:434-441).  (Round 1
//                narrowed with 2-D DMA rows of the field span: 2.3 GB/s.)
//   MANAGED  (1) cudaMallocManaged AoS, no placement hints; per chunk
//                cudaMemPrefetchAsync to the GPU, kernels run in place on the
//                migrated pages, prefetch back.
//   INPLACE  (2) pinned host AoS, whole records each way (the reference's
//                run_dev_inplace round trip, inplace_bytes_one_way).
//   MANAGED_MAPPED (3) cudaMallocManaged AoS kept on the host (preferred
//                location CPU, accessed-by GPU) and never migrated: the
//                gather's TMA tiles and the scatter-back read and write the
//                host pages over PCIe in place.
//
// Per chunk on the device: fused gather + first kernel (k_gather_warp) ->
// further kernels on the SoA -> either the SoA slice to a host SoA buffer
// (host_soa != NULL) or scatter-merge of every write set into the AoS chunk
// and back to the host.
#include <cuda_runtime.h>

#include <algorithm>
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
    int device = -1;  // the device the slots and streams belong to
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
    if (mode < 0 || mode > 3) throw std::invalid_argument("unknown host orchestration mode");
    const bool managed = mode == 1 || mode == 3;
    const std::vector<std::string> ks = split_names(kernels);
    if (ks.empty()) throw std::invalid_argument("no kernels given");
    for (const auto& k : ks)
        if (k != "kick" && k != "drift") throw std::invalid_argument("run_host runs kick and drift");
    if (chunk == 0) chunk = 1ull << 21;
    chunk = (chunk + 127) / 128 * 128;  // 16-B aligned chunk starts for any record width
    const uint64_t n = src.count;
    const uint64_t rb = src.record_bits();

    for (const auto& k : ks)
        if (!src.schema->kernel(k)) throw std::invalid_argument("no access set declared for kernel '" + k + "'");
    const View& dev_view = src;  // layout of the AoS chunk the kernels address (device slot, or the host records)
    if (mode == 0 && (!src.byte_aligned() || (rb & 7)))
        throw std::invalid_argument("streamed mode needs byte-aligned lanes (use INPLACE for bit-packed AoS)");
    // streamed: the bytes the kernels touch per record, both ways (stored widths)
    uint64_t read_bits = 0, write_bits = 0;
    for (size_t f = 0; f < src.schema->fields.size(); ++f) {
        const FieldDecl& d = src.schema->fields[f];
        const uint64_t w = uint64_t(d.arity) * src.width(src.pos_of(int(f)));
        bool rd = std::find(dst.subset.begin(), dst.subset.end(), int(f)) != dst.subset.end(), wr = false;
        for (const auto& k : ks) {
            const KernelSet* set = src.schema->kernel(k);
            wr |= std::find(set->writes.begin(), set->writes.end(), d.name) != set->writes.end();
        }
        read_bits += rd ? w : 0;
        write_bits += wr ? w : 0;
    }

    cudaPointerAttributes attr{};
    check_cuda(cudaPointerGetAttributes(&attr, host), "pointer attributes");
    if (!managed && attr.type != cudaMemoryTypeHost)
        throw std::invalid_argument("streamed/inplace modes need pinned host memory (sf_b200_host_alloc mode 0)");
    if (managed && attr.type != cudaMemoryTypeManaged)
        throw std::invalid_argument("managed mode needs cudaMallocManaged memory (sf_b200_host_alloc mode 1)");
    int dev = 0;
    check_cuda(cudaGetDevice(&dev), "device");

    const int slots = 3;
    static thread_local std::unique_ptr<DeviceSlots> pool;
    const size_t aos_bytes = size_t((chunk * rb + 7) / 8) + 16;
    const size_t soa_bytes = size_t(with_count(dst, chunk).total_bytes()) + 16;
    if (!pool || pool->device != dev || pool->aos_bytes < aos_bytes || pool->soa_bytes < soa_bytes) {
        if (pool && pool->device != dev) {  // free the old device's slots on that device
            int cur = dev;
            check_cuda(cudaSetDevice(pool->device), "set device");
            pool.reset();
            check_cuda(cudaSetDevice(cur), "set device");
        }
        pool.reset(new DeviceSlots());
        pool->device = dev;
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
    if (managed) {
        // MANAGED_MAPPED keeps the pages on the host and maps them for the GPU; MANAGED migrates them with
        // prefetches and runs best without hints (profiles/r02_managed_probe.log: 356 ms vs 418 ms with
        // PreferredLocation = CPU + AccessedBy; the limiter is the migration back to the host, 25 GB/s
        // against 57 GB/s of pinned D2H DMA)
        const size_t total = size_t((n * rb + 7) / 8);
        if (mode == 3) {
            check_cuda(cudaMemAdvise(host, total, cudaMemAdviseSetPreferredLocation, cudaCpuDeviceId), "advise");
            check_cuda(cudaMemAdvise(host, total, cudaMemAdviseSetAccessedBy, dev), "advise");
        } else {
            check_cuda(cudaMemAdvise(host, total, cudaMemAdviseUnsetPreferredLocation, cudaCpuDeviceId), "advise");
            check_cuda(cudaMemAdvise(host, total, cudaMemAdviseUnsetAccessedBy, dev), "advise");
        }
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
        void* aos = (managed || mode == 0) ? static_cast<void*>(hchunk) : pool->aos[s];
        const bool zero_copy = mode == 0;
        if (mode == 0) {
            h2d += read_bits * cnt / 8;  // the kernels read these lanes in place over PCIe
        } else if (mode == 2) {
            check_cuda(cudaMemcpyAsync(aos, hchunk, bytes, cudaMemcpyHostToDevice, st), "H2D");
            h2d += bytes;
        } else if (mode == 1) {
            check_cuda(cudaMemPrefetchAsync(hchunk, bytes, dev, st), "prefetch");
            h2d += bytes;
        } else {
            h2d += bytes;  // MANAGED_MAPPED: no migration, the kernels read the host pages over PCIe
        }
        const View sv = with_count(dev_view, cnt), dv = with_count(dst, cnt);
        gather(sv, aos, dv, pool->soa[s], ks[0].c_str(), dt, math, st, zero_copy);
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
            for (const auto& k : ks) scatter_merge(dv, pool->soa[s], sv, aos, k, st, zero_copy);
            if (mode == 0) {
                d2h += write_bits * cnt / 8;  // the write set's lanes, stored in place over PCIe
            } else if (mode == 2) {
                check_cuda(cudaMemcpyAsync(hchunk, aos, bytes, cudaMemcpyDeviceToHost, st), "D2H");
                d2h += bytes;
            } else if (mode == 1) {
                check_cuda(cudaMemPrefetchAsync(hchunk, bytes, cudaCpuDeviceId, st), "prefetch");
                d2h += bytes;
            } else {
                d2h += bytes;  // written in place through the mapping
            }
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
