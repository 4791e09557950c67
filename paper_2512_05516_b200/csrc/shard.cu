// One rank of the cell-sharded SPH timestep (BASELINE C5), in
// C++ behind the C ABI (sf_b200_shard_*): the reference's timestep order
// (density, force, kick, drift; pipelines.cpp kernel lists, sph.cpp:176-264)
// followed by particle migration, on an x-slab of cell layers.
//
// Every rank owns ONE persistent device allocation that its +-1 neighbours
// map through CUDA IPC (same node: NVLink / NVSwitch peers, or processes
// sharing a GPU):
//
//   [header | epochs | cell_start | pos (x,y,z,m) | h | h range |
//    vel (v, P/rho^2) | outbox to the left | outbox to the right]
//
// * Halo: the density and force kernels read the neighbours' packed cell
//   blocks in place through the peer pointers (no ghost copy, no send/recv).
// * Migration: after the drift, each rank compacts its leaving particles
//   into the outbox facing their destination; the destination pulls the rows
//   straight out of the neighbour's outbox (one kernel, NVLink loads).  The
//   particles that stay are rewritten in the cell order of this step's
//   binning, so the state stays (nearly) cell-sorted and the next binning /
//   pack gathers are coherent.
// * Ordering between ranks is stream-ordered and device-side: a rank
//   publishes "phase p of step s is done" by a release store of s into an
//   epoch word of its own allocation; a neighbour's stream waits for it with
//   a one-thread acquire spin (k_wait_epochs).  No host barrier; the only
//   host synchronisation per step is reading the new particle count after a
//   migration (world > 1), which sizes the next launches.
//
// The state is an SoA of the reference's default schema at T=32 (x kept in
// binary32 too, the C5 storage) laid out at a fixed capacity: field p's
// stream starts at cap * prefix_bytes(p), so migration never moves streams.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "runtime.hpp"
#include "shard.hpp"

namespace sfb {

namespace {

// the C5 record: the default schema's fields at T=32, declaration order (sph.cpp:446-460)
struct FieldDesc {
    const char* name;
    int bytes;  // per particle
};
constexpr FieldDesc kFields[] = {{"x", 12}, {"id", 8}, {"v", 12}, {"u", 4},  {"m", 4},  {"h", 4},
                                 {"rho", 4}, {"P", 4}, {"cs", 4}, {"a", 12}, {"du", 4}, {"dt", 4}};
constexpr int kNumFields = 12;
__host__ __device__ constexpr int field_bytes(int f) { return (f == 0 || f == 2 || f == 9) ? 12 : f == 1 ? 8 : 4; }
constexpr int kRowBytes = 76;  // one particle, every field
enum { F_X = 0, F_ID, F_V, F_U, F_M, F_H, F_RHO, F_P, F_CS, F_A, F_DU, F_DT };

constexpr uint64_t kMagic = 0x53464232303053ull;  // "SFB200S"
enum Epoch { E_PACKED = 0, E_PACKED_FORCE = 1, E_READ_DONE = 2, E_OUTBOX = 3, E_PULLED = 4, E_COUNT = 8 };

struct Header {
    uint64_t magic, cap, cap_m, ncell;
    int32_t x0, nx, rank, world;
    float x_origin;
    int32_t pad[19];
    uint64_t epoch[E_COUNT];  // offset 128
};
static_assert(sizeof(Header) == 192, "header layout");

uint64_t al256(uint64_t v) { return (v + 255) & ~uint64_t(255); }

struct ShardLayout {
    uint64_t cs, pos, h, hmax, vel, out[2], total;
};
ShardLayout layout_of(uint64_t ncell, uint64_t cap, uint64_t cap_m) {
    ShardLayout L{};
    L.cs = 256;
    L.pos = al256(L.cs + 4 * (ncell + 1));
    L.h = al256(L.pos + 16 * cap);
    L.hmax = al256(L.h + 4 * cap);
    L.vel = al256(L.hmax + 16);
    L.out[0] = al256(L.vel + 16 * cap);
    L.out[1] = al256(L.out[0] + 16 + uint64_t(kRowBytes) * cap_m);
    L.total = al256(L.out[1] + 16 + uint64_t(kRowBytes) * cap_m);
    return L;
}

// ---------------------------------------------------------------- epochs
__global__ void k_signal(uint64_t* epoch, uint64_t value) {
    // every write of the kernels before this one in the stream is visible to the system first
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(epoch), "l"(value) : "memory");
}

// One thread spins (acquire, system scope) until both neighbours' epoch words
// reach `value`.  Bounded: after kWaitNs without progress it raises *timeout
// and returns, so a neighbour that failed (or never started the step) turns
// into an SF_ERROR at this step's end instead of a hung stream.
constexpr uint64_t kWaitNs = 20ull * 1000 * 1000 * 1000;
__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void k_wait_epochs(const uint64_t* a, const uint64_t* b, uint64_t value, int* timeout) {
    const uint64_t t0 = global_ns();
    for (const uint64_t* p : {a, b}) {
        if (!p) continue;
        uint64_t v = 0;
        unsigned ns = 32;
        for (;;) {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
            if (v >= value) break;
            if (global_ns() - t0 > kWaitNs) {
                atomicOr(timeout, 4);
                return;
            }
            __nanosleep(ns);
            ns = ns < 4096 ? ns * 2 : ns;
        }
    }
}

// ---------------------------------------------------------------- migration
struct Streams {
    uint8_t* f[kNumFields];
};

__device__ __forceinline__ int slab_layer(float x, float inv_cell, int nc) {
    return min(max(int(floorf(x * inv_cell)), 0), nc - 1);
}

// Per sorted position k (particle perm[k]): 1 in the class it goes to
// (keep / left / right), prefix-summed afterwards into destination slots.
__global__ void k_mig_classify(const float* __restrict__ x, const int32_t* __restrict__ perm, uint64_t n, float inv_cell,
                               int nc, int x0, int x1, int32_t* __restrict__ keep, int32_t* __restrict__ left,
                               int32_t* __restrict__ right) {
    for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < n; k += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = perm ? uint64_t(perm[k]) : k;
        const int l = slab_layer(x[3 * i], inv_cell, nc);
        keep[k] = l >= x0 && l < x1;
        left[k] = l < x0;
        right[k] = l >= x1;
    }
}

// 4-byte words: rows are 76 B, so a field inside a row is only 4-B aligned
__device__ __forceinline__ void copy_field(uint8_t* __restrict__ d, const uint8_t* __restrict__ s, int bytes) {
    const uint32_t* s4 = reinterpret_cast<const uint32_t*>(s);
    uint32_t* d4 = reinterpret_cast<uint32_t*>(d);
#pragma unroll
    for (int w = 0; w < 3; ++w)
        if (4 * w < bytes) d4[w] = s4[w];
}

// Stayers to their slot of the new state (in sorted order: the state becomes
// cell-sorted), leavers to a row of the outbox facing their destination.
// keep/left/right hold exclusive offsets; totals[3] = their sums.
__global__ void k_mig_scatter(Streams src, Streams dst, const int32_t* __restrict__ perm, uint64_t n,
                              const int32_t* __restrict__ keep, const int32_t* __restrict__ left,
                              const int32_t* __restrict__ right, const float* __restrict__ x, float inv_cell, int nc,
                              int x0, int x1, uint8_t* __restrict__ out_l, uint8_t* __restrict__ out_r,
                              uint64_t cap_m, int* __restrict__ overflow) {
    for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < n; k += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = perm ? uint64_t(perm[k]) : k;
        const int l = slab_layer(x[3 * i], inv_cell, nc);
        if (l >= x0 && l < x1) {
            const uint64_t o = uint64_t(keep[k]);
#pragma unroll
            for (int f = 0; f < kNumFields; ++f)
                copy_field(dst.f[f] + o * field_bytes(f), src.f[f] + i * field_bytes(f), field_bytes(f));
            continue;
        }
        const bool go_l = l < x0;
        const uint64_t o = uint64_t(go_l ? left[k] : right[k]);
        if (o >= cap_m) {
            atomicOr(overflow, 1);
            continue;
        }
        uint8_t* row = (go_l ? out_l : out_r) + 16 + o * kRowBytes;
        int c = 0;
#pragma unroll
        for (int f = 0; f < kNumFields; ++f) {
            copy_field(row + c, src.f[f] + i * field_bytes(f), field_bytes(f));
            c += field_bytes(f);
        }
    }
}

// counts: the outboxes' headers and the number of stayers, from the scans
__global__ void k_mig_counts(const int32_t* __restrict__ keep, const int32_t* __restrict__ left,
                             const int32_t* __restrict__ right, uint64_t n, uint8_t* out_l, uint8_t* out_r,
                             uint64_t* __restrict__ n_keep) {
    // exclusive scans over n + 1 entries: entry n is the total
    *reinterpret_cast<uint64_t*>(out_l) = uint64_t(left[n]);
    *reinterpret_cast<uint64_t*>(out_r) = uint64_t(right[n]);
    *n_keep = uint64_t(keep[n]);
}

// Rows of the neighbours' outboxes facing this rank, appended after the
// stayers: [n_keep, n_keep + c0) from src0, then c1 from src1 (peer memory).
__global__ void k_mig_pull(Streams dst, const uint8_t* __restrict__ src0, const uint8_t* __restrict__ src1,
                           const uint64_t* __restrict__ n_keep, uint64_t cap, uint64_t* __restrict__ n_new,
                           int* __restrict__ overflow) {
    const uint64_t c0 = src0 ? *reinterpret_cast<const volatile uint64_t*>(src0) : 0;
    const uint64_t c1 = src1 ? *reinterpret_cast<const volatile uint64_t*>(src1) : 0;
    const uint64_t base = *n_keep;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *n_new = base + c0 + c1;
        if (base + c0 + c1 > cap) atomicOr(overflow, 2);
    }
    for (uint64_t r = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; r < c0 + c1;
         r += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t o = base + r;
        if (o >= cap) break;
        const uint8_t* row = r < c0 ? src0 + 16 + r * kRowBytes : src1 + 16 + (r - c0) * kRowBytes;
        int c = 0;
#pragma unroll
        for (int f = 0; f < kNumFields; ++f) {
            copy_field(dst.f[f] + o * field_bytes(f), row + c, field_bytes(f));
            c += field_bytes(f);
        }
    }
}

struct DevMem {
    void* p = nullptr;
    DevMem() = default;
    explicit DevMem(uint64_t bytes) { check_cuda(cudaMalloc(&p, bytes), "cudaMalloc"); }
    DevMem(const DevMem&) = delete;
    DevMem& operator=(const DevMem&) = delete;
    ~DevMem() {
        if (p) cudaFree(p);
    }
    template <typename T>
    T* as(uint64_t off = 0) const {
        return reinterpret_cast<T*>(static_cast<uint8_t*>(p) + off);
    }
};

}  // namespace

struct Shard {
    int rank = 0, world = 1, nc = 1, refine = 2, device = 0;
    double cell = 1.0;  // slab cell side (>= 2 h_max)
    uint64_t cap = 0, cap_m = 0, n = 0, step = 0;
    int x0 = 0, x1 = 0;  // coarse layers [x0, x1) owned
    int fx0 = 0, fnx = 0, NF = 0;  // fine layers of the binning grid
    float fine = 0.f;     // binning cell side
    uint64_t ncell = 0;
    ShardLayout L{};
    std::unique_ptr<DevMem> shared, state[2], scratch, perm, classes, misc;
    std::unique_ptr<DevMem> wmask;  // the density's per-window in-support masks for the force
    uint64_t wmask_n = 0;           // homes they hold
    int cur = 0;
    uint64_t bin_bytes = 0, scan_bytes = 0;
    struct Peer {
        int rank = -1;
        void* base = nullptr;
        Header h{};
        ShardLayout L{};
    } peer[2];  // [0] left (rank - 1), [1] right (rank + 1)
    bool connected = false;
    cudaEvent_t ev[12] = {};  // [2k], [2k+1]: around kernel k of the list; [8], [9]: migration

    uint8_t* sbase() const { return shared->as<uint8_t>(); }
    uint64_t* epoch(int e) const { return reinterpret_cast<uint64_t*>(sbase() + offsetof(Header, epoch)) + e; }
    const uint64_t* peer_epoch(int side, int e) const {
        return peer[side].base ? reinterpret_cast<const uint64_t*>(static_cast<uint8_t*>(peer[side].base) +
                                                                   offsetof(Header, epoch)) + e
                               : nullptr;
    }
    uint8_t* field(int s, int f) const {
        uint64_t off = 0;
        for (int q = 0; q < f; ++q) off += cap * kFields[q].bytes;
        return state[s]->as<uint8_t>(off);
    }
    Streams streams(int s) const {
        Streams S{};
        for (int f = 0; f < kNumFields; ++f) S.f[f] = field(s, f);
        return S;
    }
};

Shard* shard_create(int rank, int world, int nc, double cell, int refine, uint64_t capacity) {
    require_device();
    if (world < 1 || rank < 0 || rank >= world || nc < world || !(cell > 0) || refine < 1 || refine > 4 ||
        capacity == 0 || capacity >= (1ull << 30))
        throw std::invalid_argument("shard_create: bad rank / world / grid / capacity");
    std::unique_ptr<Shard> S(new Shard());
    check_cuda(cudaGetDevice(&S->device), "device");
    S->rank = rank, S->world = world, S->nc = nc, S->cell = cell, S->refine = refine;
    S->cap = (capacity + 63) / 64 * 64;  // every stream 16-B aligned (k_update_soa's vector accesses)
    S->cap_m = std::max<uint64_t>(capacity / 8, 65536);
    S->x0 = int(int64_t(rank) * nc / world);
    S->x1 = int(int64_t(rank + 1) * nc / world);
    S->NF = nc * refine;
    S->fx0 = S->x0 * refine;
    S->fnx = (S->x1 - S->x0) * refine;
    S->fine = float(cell / refine);
    S->ncell = uint64_t(S->fnx) * S->NF * S->NF;
    if (S->ncell >= (1ull << 31)) throw std::invalid_argument("shard_create: cell grid too large");
    S->L = layout_of(S->ncell, S->cap, S->cap_m);
    S->shared.reset(new DevMem(S->L.total));
    check_cuda(cudaMemset(S->shared->p, 0, S->L.total), "memset");
    Header h{};
    h.magic = kMagic, h.cap = S->cap, h.cap_m = S->cap_m, h.ncell = S->ncell;
    h.x0 = S->fx0, h.nx = S->fnx, h.rank = rank, h.world = world;
    h.x_origin = float(S->x0 * cell);
    check_cuda(cudaMemcpy(S->shared->p, &h, sizeof(h), cudaMemcpyHostToDevice), "H2D");
    for (int s = 0; s < 2; ++s) S->state[s].reset(new DevMem(uint64_t(kRowBytes) * S->cap + 256));
    S->bin_bytes = bin_scratch_bytes(S->cap, S->fnx, S->NF, S->NF);
    S->scan_bytes = scan_scratch_bytes(int64_t(S->cap) + 1);
    S->scratch.reset(new DevMem(std::max(S->bin_bytes, S->scan_bytes)));
    S->perm.reset(new DevMem(4 * (S->cap + 64)));
    S->classes.reset(new DevMem(3 * 4 * (S->cap + 64)));
    S->misc.reset(new DevMem(256));  // [0] n_keep, [8] n_new, [16] overflow, [20] rho == 0
    check_cuda(cudaMemset(S->misc->p, 0, 256), "memset");
    for (auto& e : S->ev) check_cuda(cudaEventCreate(&e), "event");
    S->connected = world == 1;
    return S.release();
}

void shard_destroy(Shard* S) {
    if (!S) return;
    for (auto& p : S->peer)
        if (p.base) cudaIpcCloseMemHandle(p.base);
    for (auto& e : S->ev)
        if (e) cudaEventDestroy(e);
    delete S;
}

void shard_handle(Shard* S, uint8_t* out) {
    cudaIpcMemHandle_t h;
    check_cuda(cudaIpcGetMemHandle(&h, S->shared->p), "cudaIpcGetMemHandle");
    static_assert(sizeof(h) <= 64, "IPC handle size");
    std::memset(out, 0, 64);
    std::memcpy(out, &h, sizeof(h));
}

void shard_connect(Shard* S, const uint8_t* handles) {
    if (S->world == 1) {
        S->connected = true;
        return;
    }
    for (int side = 0; side < 2; ++side) {
        const int r = S->rank + (side ? 1 : -1);
        if (r < 0 || r >= S->world) continue;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handles + 64 * r, sizeof(h));
        void* p = nullptr;
        check_cuda(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
        Header ph{};
        check_cuda(cudaMemcpy(&ph, p, sizeof(ph), cudaMemcpyDeviceToHost), "peer header");
        if (ph.magic != kMagic || ph.rank != r || ph.world != S->world || ph.cap != S->cap)
            throw std::invalid_argument("shard_connect: handle " + std::to_string(r) +
                                        " is not that rank's shard of the same world and capacity");
        S->peer[side].rank = r;
        S->peer[side].base = p;
        S->peer[side].h = ph;
        S->peer[side].L = layout_of(ph.ncell, ph.cap, ph.cap_m);
    }
    S->connected = true;
}

void shard_load(Shard* S, const void* soa, uint64_t count, cudaStream_t st) {
    if (count > S->cap) throw std::invalid_argument("shard_load: more particles than the shard's capacity");
    // the reference SoA of `count` particles: field p's stream at count * prefix(p)
    uint64_t off = 0;
    for (int f = 0; f < kNumFields; ++f) {
        const uint64_t bytes = count * field_bytes(f);
        if (bytes)
            check_cuda(cudaMemcpyAsync(S->field(S->cur, f), static_cast<const uint8_t*>(soa) + off, bytes,
                                       cudaMemcpyDeviceToDevice, st),
                       "D2D");
        off += bytes;
    }
    S->n = count;
}

void* shard_field(Shard* S, const char* name, int* bytes_per_particle) {
    for (int f = 0; f < kNumFields; ++f)
        if (std::strcmp(kFields[f].name, name) == 0) {
            if (bytes_per_particle) *bytes_per_particle = field_bytes(f);
            return S->field(S->cur, f);
        }
    throw std::invalid_argument(std::string("shard has no field '") + name + "'");
}

uint64_t shard_count(const Shard* S) { return S->n; }

namespace {

void signal(Shard* S, int e, cudaStream_t st) {
    if (S->world == 1) return;
    k_signal<<<1, 1, 0, st>>>(S->epoch(e), S->step);
    count_launches(1);
}

void wait_peers(Shard* S, int e, uint64_t value, cudaStream_t st) {
    if (S->world == 1 || value == 0) return;
    k_wait_epochs<<<1, 1, 0, st>>>(S->peer_epoch(0, e), S->peer_epoch(1, e), value, S->misc->as<int>(16));
    count_launches(1);
}

CellBlockDesc density_block(const uint8_t* base, const ShardLayout& L, int x0, int nx, float x_origin) {
    return CellBlockDesc{base + L.pos, reinterpret_cast<const float*>(base + L.h),
                         reinterpret_cast<const int32_t*>(base + L.cs), reinterpret_cast<const unsigned*>(base + L.hmax),
                         x0, nx, x_origin, 0};
}

ForceBlockDesc force_block(const uint8_t* base, const ShardLayout& L, int x0, int nx, float x_origin) {
    return ForceBlockDesc{base + L.pos, base + L.vel, reinterpret_cast<const float*>(base + L.h),
                          reinterpret_cast<const int32_t*>(base + L.cs),
                          reinterpret_cast<const unsigned*>(base + L.hmax), x0, nx, x_origin, 0};
}

}  // namespace

void shard_step(Shard* S, const std::vector<std::string>& kernels, double dt, cudaStream_t st, double* metrics) {
    require_device();
    if (!S->connected) throw std::invalid_argument("shard_step: sf_b200_shard_connect first");
    for (const auto& k : kernels)
        if (k != "density" && k != "force" && k != "kick" && k != "drift")
            throw std::invalid_argument("shard_step runs density, force, kick and drift, not '" + k + "'");
    ++S->step;
    const uint64_t s = S->step;
    const int c = S->cur;
    uint8_t* base = S->sbase();
    const float* x = reinterpret_cast<const float*>(S->field(c, F_X));
    int32_t* perm = S->perm->as<int32_t>();
    int* overflow = S->misc->as<int>(16);
    unsigned* rho_zero = S->misc->as<unsigned>(20);
    const float lo_yz[2] = {0.f, 0.f};
    const float lo[3] = {float(S->x0 * S->cell), 0.f, 0.f};
    const bool timed = metrics != nullptr;
    auto mark = [&](int i) {
        if (timed) check_cuda(cudaEventRecord(S->ev[i], st), "event");
    };
    if (kernels.size() > 4) throw std::invalid_argument("shard_step: at most four kernels per step");
    bool binned = false;
    auto bin_and_pack = [&] {
        // the neighbours finished reading this block in the previous step
        wait_peers(S, E_READ_DONE, s - 1, st);
        bin_particles(x, S->n, lo, S->fine, S->fnx, S->NF, S->NF, reinterpret_cast<int32_t*>(base + S->L.cs), perm,
                      S->scratch->p, S->bin_bytes, st);
        cells_pack(x, S->field(c, F_M), S->field(c, F_H), 1, S->n, perm, base + S->L.pos,
                   reinterpret_cast<float*>(base + S->L.h), reinterpret_cast<unsigned*>(base + S->L.hmax), st);
        signal(S, E_PACKED, st);
        wait_peers(S, E_PACKED, s, st);
        binned = true;
    };
    std::vector<CellBlockDesc> dblocks;
    std::vector<ForceBlockDesc> fblocks;
    auto blocks = [&] {
        dblocks.clear();
        fblocks.clear();
        const float xo = float(S->x0 * S->cell);
        dblocks.push_back(density_block(base, S->L, S->fx0, S->fnx, xo));
        fblocks.push_back(force_block(base, S->L, S->fx0, S->fnx, xo));
        for (int side = 0; side < 2; ++side) {
            const auto& p = S->peer[side];
            if (!p.base) continue;
            const uint8_t* pb = static_cast<const uint8_t*>(p.base);
            dblocks.push_back(density_block(pb, p.L, p.h.x0, p.h.nx, p.h.x_origin));
            fblocks.push_back(force_block(pb, p.L, p.h.x0, p.h.nx, p.h.x_origin));
        }
    };
    bool force_ran = false;
    // density then force in one step: the density writes every home's per-window in-support masks and the
    // force sweeps exactly those pairs (no culling arithmetic, no out-of-support candidates)
    int32_t* win = nullptr;
    bool win_ready = false;
    {
        const auto di = std::find(kernels.begin(), kernels.end(), "density");
        const auto fi = std::find(kernels.begin(), kernels.end(), "force");
        if (di != kernels.end() && fi != kernels.end() && di < fi && S->refine <= 2 && S->n > 0 &&
            S->n < (1ull << 30)) {  // window masks: reach <= 2
            if (!S->wmask || S->wmask_n < S->n) {
                S->wmask.reset();
                S->wmask_n = S->n + S->n / 8 + 1024;
                S->wmask.reset(new DevMem(window_mask_words(S->wmask_n, S->refine) * 4));
            }
            win = S->wmask->as<int32_t>();
        }
    }
    for (size_t ki = 0; ki < kernels.size(); ++ki) {
        const std::string& k = kernels[ki];
        mark(int(2 * ki));
        if (k == "density" || k == "force") {
            if (!binned) bin_and_pack();
            blocks();
        }
        if (k == "density") {
            density_cells_blocks(dblocks.data(), int(dblocks.size()), S->n, perm, S->n, lo_yz, S->fine, S->NF, S->NF,
                                 S->NF, S->refine, reinterpret_cast<float*>(S->field(c, F_RHO)), st, win);
            win_ready = win != nullptr;
        } else if (k == "force") {
            // the neighbours finished reading this block's (v, P/rho^2) in the previous step (E_READ_DONE,
            // waited in bin_and_pack); rho == 0 -> *rho_zero, checked at the end of the step
            force_pack_async(S->field(c, F_V), S->field(c, F_RHO), S->field(c, F_P), 1, S->n, perm, base + S->L.vel,
                             rho_zero, st);
            signal(S, E_PACKED_FORCE, st);
            wait_peers(S, E_PACKED_FORCE, s, st);
            force_cells_blocks(fblocks.data(), int(fblocks.size()), S->n, perm, S->n, lo_yz, S->fine, S->NF, S->NF,
                               S->NF, S->refine, reinterpret_cast<float*>(S->field(c, F_A)),
                               reinterpret_cast<float*>(S->field(c, F_DU)), st, win_ready ? win : nullptr);
            force_ran = true;
        } else if (k == "kick") {
            // sph.cpp:247-256: v += a dt; u = max(0, u + du dt) in binary64, stored binary32
            check_cuda(launch_update_soa(B_F32, B_F32, S->field(c, F_V), S->field(c, F_A), 3 * S->n, dt, OP_AXPY,
                                         MATH_FP64_EXACT, st),
                       "kick launch");
            check_cuda(launch_update_soa(B_F32, B_F32, S->field(c, F_U), S->field(c, F_DU), S->n, dt,
                                         OP_AXPY_CLAMP0, MATH_FP64_EXACT, st),
                       "kick launch");
            count_launches(2);
        } else {
            // sph.cpp:258-264: x += v dt
            check_cuda(launch_update_soa(B_F32, B_F32, S->field(c, F_X), S->field(c, F_V), 3 * S->n, dt, OP_AXPY,
                                         MATH_FP64_EXACT, st),
                       "drift launch");
            count_launches(1);
        }
        mark(int(2 * ki + 1));
    }
    // nobody reads this rank's block after this point of the step (signalled every step, binned or not:
    // a neighbour that bins in the next step waits for this epoch)
    signal(S, E_READ_DONE, st);
    mark(8);
    uint64_t sent[2] = {0, 0};
    if (S->world > 1) {
        // ---- migration: stayers in cell order into the other state buffer, leavers into the outboxes
        const uint64_t n = S->n;
        int32_t* keep = S->classes->as<int32_t>();
        int32_t* left = keep + (S->cap + 64);
        int32_t* right = left + (S->cap + 64);
        const int32_t* mperm = binned ? perm : nullptr;  // binned positions are pre-drift: still a valid order
        const unsigned g = unsigned(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * 8)));
        const float inv_cell = float(1.0 / S->cell);
        // the neighbours pulled last step's rows out of my outboxes
        wait_peers(S, E_PULLED, s - 1, st);
        k_mig_classify<<<g, 256, 0, st>>>(x, mperm, n, inv_cell, S->nc, S->x0, S->x1, keep, left, right);
        check_cuda(cudaMemsetAsync(keep + n, 0, 4, st), "memset");
        check_cuda(cudaMemsetAsync(left + n, 0, 4, st), "memset");
        check_cuda(cudaMemsetAsync(right + n, 0, 4, st), "memset");
        for (int32_t* a : {keep, left, right})
            exclusive_scan_i32(a, int64_t(n) + 1, S->scratch->as<int32_t>(), st);
        uint8_t* out_l = base + S->L.out[0];
        uint8_t* out_r = base + S->L.out[1];
        const int o = 1 - c;
        k_mig_scatter<<<g, 256, 0, st>>>(S->streams(c), S->streams(o), mperm, n, keep, left, right, x, inv_cell, S->nc,
                                         S->x0, S->x1, out_l, out_r, S->cap_m, overflow);
        k_mig_counts<<<1, 1, 0, st>>>(keep, left, right, n, out_l, out_r, S->misc->as<uint64_t>(0));
        signal(S, E_OUTBOX, st);
        wait_peers(S, E_OUTBOX, s, st);
        // the left neighbour's right outbox and the right neighbour's left outbox face this rank
        const uint8_t* src0 = S->peer[0].base ? static_cast<const uint8_t*>(S->peer[0].base) + S->peer[0].L.out[1]
                                              : nullptr;
        const uint8_t* src1 = S->peer[1].base ? static_cast<const uint8_t*>(S->peer[1].base) + S->peer[1].L.out[0]
                                              : nullptr;
        const unsigned gp = unsigned(std::min<uint64_t>((2 * S->cap_m + 255) / 256, uint64_t(num_sms()) * 4));
        k_mig_pull<<<gp, 256, 0, st>>>(S->streams(o), src0, src1, S->misc->as<uint64_t>(0), S->cap,
                                       S->misc->as<uint64_t>(8), overflow);
        signal(S, E_PULLED, st);
        count_launches(4);
        check_cuda(cudaGetLastError(), "migration launch");
        uint64_t counts[2] = {0, 0};
        check_cuda(cudaMemcpyAsync(counts, S->misc->as<uint64_t>(8), 8, cudaMemcpyDeviceToHost, st), "D2H");
        check_cuda(cudaMemcpyAsync(sent, out_l, 8, cudaMemcpyDeviceToHost, st), "D2H");
        check_cuda(cudaMemcpyAsync(sent + 1, out_r, 8, cudaMemcpyDeviceToHost, st), "D2H");
        int flags[2] = {0, 0};
        check_cuda(cudaMemcpyAsync(flags, overflow, 8, cudaMemcpyDeviceToHost, st), "D2H");
        check_cuda(cudaStreamSynchronize(st), "sync");  // the one host synchronisation of the step
        if (flags[0]) {
            check_cuda(cudaMemset(overflow, 0, 4), "memset");
            if (flags[0] & 4)
                throw std::runtime_error("shard_step: a neighbour did not reach this step within 20 s "
                                         "(failed or not stepping); the shard's state is undefined");
            throw std::runtime_error("shard_step: migration overflowed the outbox or the shard capacity");
        }
        if (flags[1] && force_ran) {
            check_cuda(cudaMemset(rho_zero, 0, 4), "memset");
            throw std::domain_error("force: degenerate state, rho == 0");
        }
        S->n = counts[0];
        S->cur = o;
    } else if (force_ran) {
        unsigned flag = 0;
        check_cuda(cudaMemcpyAsync(&flag, rho_zero, 4, cudaMemcpyDeviceToHost, st), "D2H");
        check_cuda(cudaStreamSynchronize(st), "sync");
        if (flag) {
            check_cuda(cudaMemset(rho_zero, 0, 4), "memset");
            throw std::domain_error("force: degenerate state, rho == 0");
        }
    }
    mark(9);
    if (timed) {
        check_cuda(cudaEventSynchronize(S->ev[9]), "sync");
        auto between = [&](int a, int b) {
            float t = 0;
            check_cuda(cudaEventElapsedTime(&t, S->ev[a], S->ev[b]), "elapsed");
            return double(t);
        };
        // metrics: [0] particles after the step, [1] step ms, [2..5] ms per kernel of the list (in list
        // order, waits on the neighbours included), [6] migration ms, [7] particles sent, [8] step number
        for (int i = 0; i < 9; ++i) metrics[i] = 0.0;
        metrics[0] = double(S->n);
        metrics[1] = kernels.empty() ? 0.0 : between(0, 9);
        for (size_t ki = 0; ki < kernels.size(); ++ki) metrics[2 + ki] = between(int(2 * ki), int(2 * ki + 1));
        metrics[6] = between(8, 9);
        metrics[7] = double(sent[0] + sent[1]);
        metrics[8] = double(S->step);
    }
}

}  // namespace sfb
