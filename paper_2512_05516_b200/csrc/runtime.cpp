#include "runtime.hpp"

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <stdexcept>

namespace sfb {

static std::atomic<uint64_t> g_launches{0};
void count_launches(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

int num_sms() {
    static const int sms = [] {  // thread-safe one-time init
        int dev = 0, n = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        return n > 0 ? n : 148;
    }();
    return sms;
}

void require_device() {
    static const bool have = [] {  // thread-safe one-time init
        int n = 0;
        const bool any = cudaGetDeviceCount(&n) == cudaSuccess && n > 0;
        // Stream-ordered scratch (density_cells) comes from the device's default
        // pool; keep freed blocks cached instead of unmapping them at every
        // synchronize (the default release threshold is 0).
        for (int d = 0; d < n && any; ++d) {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess) {
                uint64_t keep = ~0ull;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
            }
        }
        return any;
    }();
    if (!have) throw std::runtime_error("no CUDA device: libsoaforge_b200 runs on the GPU only (no CPU path)");
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

static void check_ptr(const void* p, const char* what) {
    if (!aligned16(p)) throw std::invalid_argument(std::string(what) + " must be 16-byte aligned");
}

// The per-lane ops of a linear kernel applied to a generic src->dst conversion.
static void fuse_ops(ConvertPlan& p, const View& src, const View& dst, const std::string& kernel, double dt,
                     int math) {
    const KernelPlan kp = plan_kernel(dst, kernel, dt, math);  // validates fields in dst
    p.dt = dt;
    p.math = uint8_t(math);
    for (uint32_t i = 0; i < kp.n; ++i) {
        // find the stream writing the same lanes
        for (uint32_t s = 0; s < p.n; ++s) {
            if (p.s[s].dst.base != kp.s[i].dst.base) continue;
            const int yp_dst = [&] {
                for (size_t q = 0; q < dst.subset.size(); ++q)
                    if (dst.lane_base(int(q)) == kp.s[i].aux.base) return int(q);
                return -1;
            }();
            const int yp_src = src.pos_of(dst.subset[yp_dst]);
            if (yp_src < 0) throw std::invalid_argument("fused operand missing from the source view");
            p.s[s].op = kp.s[i].op;
            p.s[s].aux = src.lanes(yp_src);
            p.s[s].aux_q = dst.fmt[yp_dst];
        }
    }
}

void gather(const View& src, const void* sp, const View& dst, void* dp, const char* kernel, double dt, int math,
            cudaStream_t st, bool zero_copy) {
    require_device();
    check_ptr(sp, "source buffer");
    check_ptr(dp, "destination buffer");
    bool tiled = src.layout == Layout::AoS && dst.layout == Layout::SoA && dst.subset.size() <= size_t(kMaxStreams);
    for (size_t q = 0; q < dst.subset.size() && tiled; ++q)
        tiled = (dst.width(int(q)) == 16 || dst.width(int(q)) == 32 || dst.width(int(q)) == 64) &&
                dst.lane_base(int(q)) % 8 == 0;
    if (tiled) {
        const GatherPlan g = kernel ? plan_gather_fused(src, dst, kernel, dt, math) : plan_gather(src, dst);
        check_cuda(launch_gather(g, sp, src.total_bytes(), dp, st, zero_copy), "gather launch");
        count_launches(1);
        return;
    }
    ConvertPlan p = plan_convert(src, dst, dst.subset);
    if (kernel) fuse_ops(p, src, dst, kernel, dt, math);
    check_cuda(launch_convert(p, sp, dp, st, zero_copy), "convert launch");
    count_launches(1);
}

void convert(const View& src, const void* sp, const View& dst, void* dp, cudaStream_t st) {
    gather(src, sp, dst, dp, nullptr, 0.0, 0, st);
}

void scatter_merge(const View& src, const void* sp, const View& dst, void* dp, const std::string& kernel,
                   cudaStream_t st, bool zero_copy) {
    require_device();
    check_ptr(sp, "source buffer");
    check_ptr(dp, "destination buffer");
    const KernelSet* ks = dst.schema->kernel(kernel);
    if (!ks) throw std::invalid_argument("no access set declared for kernel '" + kernel + "'");
    std::vector<int> fields;
    for (const auto& w : ks->writes) {
        const int f = dst.schema->index(w);
        if (f < 0) throw std::invalid_argument("widen_merge: unknown write field '" + w + "'");
        fields.push_back(f);
    }
    const ConvertPlan p = plan_convert(src, dst, fields);
    check_cuda(launch_convert(p, sp, dp, st, zero_copy), "scatter launch");
    count_launches(1);
}

void convert_fields(const View& src, const void* sp, const View& dst, void* dp, const std::vector<int>& fields,
                    cudaStream_t st, bool zero_copy) {
    require_device();
    check_ptr(sp, "source buffer");
    check_ptr(dp, "destination buffer");
    const ConvertPlan p = plan_convert(src, dst, fields);
    check_cuda(launch_convert(p, sp, dp, st, zero_copy), "convert launch");
    count_launches(1);
}

namespace {
// plain IEEE x/y lanes of one op, naturally aligned inside every record
bool rec_op_ok(const View& v, const CStream& c, const void* p) {
    const uint64_t rb = v.record_bits();
    const auto al = [&](const Lanes& L) { return L.base % L.fmt.width == 0 && rb % L.fmt.width == 0; };
    return fmt_is_ieee(c.dst.fmt) && fmt_is_ieee(c.aux.fmt) && c.dst.arity == c.aux.arity && al(c.dst) &&
           al(c.aux) && (reinterpret_cast<uintptr_t>(p) & 7) == 0;
}

// The ops of one or more kick/drift kernels in one shared-memory pass over the
// AoS records (k_update_rec_tile); false when the layout does not qualify.
bool rec_tile(const View& v, void* p, const std::vector<CStream>& ops, double dt, uint8_t math, cudaStream_t st) {
    const uint64_t stride = v.record_bits() / 8;
    if (v.layout != Layout::AoS || !v.byte_aligned() || ops.empty() || ops.size() > size_t(kMaxSeq) ||
        stride == 0 || stride > kRecTileMaxStride || (reinterpret_cast<uintptr_t>(p) & 31) != 0)
        return false;
    for (const auto& c : ops)
        if (!rec_op_ok(v, c, p)) return false;
    RecSeq q{};
    q.n = int(ops.size());
    uint32_t wlo = uint32_t(stride), whi = 0;  // hull of the written bytes inside a record
    for (int o = 0; o < q.n; ++o) {
        const CStream& c = ops[o];
        q.xoff[o] = uint32_t(c.dst.base / 8);
        q.yoff[o] = uint32_t(c.aux.base / 8);
        if (c.dst.arity != 1 && c.dst.arity != 3) return false;
        q.kind[o] = uint8_t((c.dst.fmt.base * 4 + c.aux.fmt.base) * 2 + (c.dst.arity == 3));
        q.op[o] = c.op;
        wlo = std::min(wlo, q.xoff[o]);
        whi = std::max(whi, q.xoff[o] + uint32_t(c.dst.arity * c.dst.fmt.width / 8));
    }
    check_cuda(launch_update_rec_tile(p, v.count, uint32_t(stride), q, dt, math, wlo, whi, st), "aos update launch");
    count_launches(1);
    return true;
}
}  // namespace

void run_kernel(const View& v, void* p, const std::string& kernel, double dt, uint64_t bs, int per_access, int math,
                cudaStream_t st) {
    require_device();
    check_ptr(p, "buffer");
    if (kernel.find(',') != std::string::npos) {  // "kick,drift": the kernels in order, one pass where possible
        const std::vector<std::string> ks = split_names(kernel);
        if (ks.empty()) throw std::invalid_argument("no kernels given");
        bool linear = v.layout == Layout::AoS && bs != 0 && v.count % bs == 0;
        for (const auto& k : ks) linear = linear && (k == "kick" || k == "drift");
        if (linear) {
            std::vector<CStream> ops;
            uint8_t m = 0;
            for (const auto& k : ks) {
                const KernelPlan kp = plan_kernel(v, k, dt, math);
                m = kp.math;
                for (uint32_t i = 0; i < kp.n; ++i) ops.push_back(kp.s[i]);
            }
            if (rec_tile(v, p, ops, dt, m, st)) return;
        }
        for (const auto& k : ks) run_kernel(v, p, k, dt, bs, per_access, math, st);
        return;
    }
    if (kernel == "density") {
        if (math != MATH_FP64_EXACT) throw std::invalid_argument("buffer-mode density is binary64 (reference semantics)");
        const DensityPlan d = plan_density(v, bs, per_access);
        check_cuda(launch_density_buffer(d, p, st), "density launch");
        count_launches(1);
        return;
    }
    if (kernel == "force") {
        if (math != MATH_FP64_EXACT) throw std::invalid_argument("buffer-mode force is binary64 (reference semantics)");
        const ForcePlan f = plan_force(v, bs, per_access);
        bool degenerate = false;
        check_cuda(launch_force_buffer(f, p, st, &degenerate), "force launch");
        count_launches(1);
        if (degenerate) throw std::domain_error("force: degenerate state, rho == 0");
        return;
    }
    if (bs == 0 || v.count % bs != 0) throw std::invalid_argument("buffer size must divide the particle count");
    if (kernel == "identity") {  // sph.cpp:266-270: x = Q(x), a bitwise no-op on stored lanes
        const int x = v.pos_of("x");
        if (x < 0) throw std::invalid_argument("field 'x' is not present in the buffer view");
        const ConvertPlan cp = plan_convert(v, v, {v.subset[x]});
        check_cuda(launch_convert(cp, p, p, st), "identity launch");
        count_launches(1);
        return;
    }
    const KernelPlan kp = plan_kernel(v, kernel, dt, math);
    if (v.layout == Layout::AoS && rec_tile(v, p, std::vector<CStream>(kp.s, kp.s + kp.n), dt, kp.math, st)) return;
    if (v.layout == Layout::AoS && v.byte_aligned()) {  // typed per-record lanes when every op is plain IEEE
        bool ok = true;
        const uint64_t rb = v.record_bits();
        for (uint32_t i = 0; i < kp.n && ok; ++i) ok = rec_op_ok(v, kp.s[i], p);
        bool same = ok && kp.n <= 2;
        for (uint32_t i = 1; i < kp.n && same; ++i)
            same = fmt_eq(kp.s[i].dst.fmt, kp.s[0].dst.fmt) && fmt_eq(kp.s[i].aux.fmt, kp.s[0].aux.fmt);
        if (same) {  // every op of the kernel in one per-record pass
            RecOps ops{};
            ops.n = int(kp.n);
            for (uint32_t i = 0; i < kp.n; ++i) {
                ops.xoff[i] = uint32_t(kp.s[i].dst.base / 8);
                ops.yoff[i] = uint32_t(kp.s[i].aux.base / 8);
                ops.arity[i] = kp.s[i].dst.arity;
                ops.op[i] = kp.s[i].op;
            }
            check_cuda(launch_update_rec_multi(kp.s[0].dst.fmt.base, kp.s[0].aux.fmt.base, p, v.count,
                                               uint32_t(rb / 8), ops, dt, kp.math, st),
                       "aos update launch");
            count_launches(1);
            return;
        }
        if (ok) {
            for (uint32_t i = 0; i < kp.n; ++i) {
                const CStream& c = kp.s[i];
                check_cuda(launch_update_rec(c.dst.fmt.base, c.aux.fmt.base, c.dst.arity, p, v.count, uint32_t(rb / 8),
                                             uint32_t(c.dst.base / 8), uint32_t(c.aux.base / 8), dt, c.op, kp.math, st),
                           "aos update launch");
            }
            count_launches(kp.n);
            return;
        }
    }
    // SoA streams of plain IEEE lanes: vectorised streaming update per stream pair
    bool vec = v.layout == Layout::SoA;
    for (uint32_t i = 0; i < kp.n && vec; ++i) {
        const CStream& c = kp.s[i];
        vec = fmt_is_ieee(c.dst.fmt) && fmt_is_ieee(c.aux.fmt) && c.dst.fmt.base != B_INT &&
              c.aux.fmt.base != B_INT && c.dst.arity == c.aux.arity && ((c.dst.base | c.aux.base) % 128) == 0 &&
              (reinterpret_cast<uintptr_t>(p) & 15) == 0;
    }
    if (vec) {
        for (uint32_t i = 0; i < kp.n; ++i) {
            const CStream& c = kp.s[i];
            uint8_t* base = static_cast<uint8_t*>(p);
            check_cuda(launch_update_soa(c.dst.fmt.base, c.aux.fmt.base, base + c.dst.base / 8, base + c.aux.base / 8,
                                         v.count * c.dst.arity, dt, c.op, kp.math, st),
                       "update launch");
        }
        count_launches(kp.n);
        return;
    }
    check_cuda(launch_convert(kp, p, p, st), "kernel launch");
    count_launches(1);
}

void permute(const View& v, const void* src, void* dst, const int32_t* perm, cudaStream_t st) {
    require_device();
    if (v.count && (!src || !dst || !perm)) throw std::invalid_argument("null argument");
    if (src == dst) throw std::invalid_argument("permute: source and destination must not alias");
    if (!v.byte_aligned()) throw std::invalid_argument("permute needs a byte-aligned view");
    PermutePlan p;
    p.count = v.count;
    auto unit = [](uint64_t base, uint64_t eb) {
        for (uint8_t u : {8, 4, 2})
            if (base % u == 0 && eb % u == 0) return u;
        return uint8_t(1);
    };
    const uintptr_t a = reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst);
    if (v.layout == Layout::AoS) {
        p.n = 1;
        p.base[0] = 0;
        p.eb[0] = uint32_t(v.record_bits() / 8);
        p.unit[0] = unit(a, p.eb[0]);
    } else {
        for (size_t q = 0; q < v.subset.size(); ++q) {
            p.base[p.n] = v.lane_base(int(q)) / 8;
            p.eb[p.n] = uint32_t(uint64_t(v.arity(int(q))) * v.width(int(q)) / 8);
            p.unit[p.n] = unit(a | p.base[p.n], p.eb[p.n]);
            ++p.n;
        }
    }
    check_cuda(launch_permute(p, src, dst, perm, st), "permute launch");
    count_launches(1);
}

}  // namespace sfb
