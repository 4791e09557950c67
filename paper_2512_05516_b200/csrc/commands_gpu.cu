// The reference's batch commands (bench.cpp:214-604) with every conversion
// and kernel executed by the sm_100a kernels.  CSV / report formats, default
// sweeps, initial conditions and checksums follow the reference, so the
// checksum columns are directly comparable with libsoaforge's
// (tests/test_gpu_commands.py).  Host code here only orchestrates, encodes
// the initial state for upload, and runs the validate battery's independent
// checkers.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <map>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <memory>
#include <random>
#include <sstream>
#include <stdexcept>
#include <vector>

#include "commands.hpp"
#include "runtime.hpp"

namespace sfb {

namespace {

constexpr const char* kVersion = "0.1.0";

// Built-in particle record (the reference's default schema: positions binary64,
// everything else binary32) with its kernel access sets.
const char* builtin_schema_text() {
    return "schema particle {\n"
           "  field x : f64 x3;\n  field id : i64;\n  field v : f32 x3;\n  field u : f32;\n"
           "  field m : f32;\n  field h : f32;\n  field rho : f32;\n  field P : f32;\n  field cs : f32;\n"
           "  field a : f32 x3;\n  field du : f32;\n  field dt : f32;\n}\n"
           "kernel density reads x, m, h writes rho;\n"
           "kernel force reads x, v, m, h, rho, P, cs writes a, du;\n"
           "kernel kick reads v, u, a, du writes v, u;\n"
           "kernel drift reads x, v writes x;\n"
           "kernel identity reads x writes x;\n";
}

std::string header() { return std::string("# soaforge v") + kVersion + "\n"; }

struct DevBuf {
    void* p = nullptr;
    size_t n = 0;
    explicit DevBuf(size_t bytes) : n(bytes + 16) {
        check_cuda(cudaMalloc(&p, n), "cudaMalloc");
        check_cuda(cudaMemset(p, 0, n), "cudaMemset");
    }
    DevBuf(const DevBuf&) = delete;
    ~DevBuf() { cudaFree(p); }
};

// ---- initial conditions (sph.cpp:325-349 semantics) -------------------------
struct State {  // binary64 particle state, field name -> lanes
    uint64_t n = 0;
    std::vector<double> x, v, a, u, m, h, rho, P, cs, du, dt;
    std::vector<int64_t> id;
};

State random_state(uint64_t n, uint64_t seed, double dt) {
    State s;
    s.n = n;
    s.x.resize(3 * n); s.v.resize(3 * n); s.a.assign(3 * n, 0.0);
    s.u.resize(n); s.m.assign(n, 1.0 / 64); s.h.assign(n, 0.5); s.rho.assign(n, 1.0);
    s.P.resize(n); s.cs.resize(n); s.du.assign(n, 0.0); s.dt.assign(n, dt); s.id.resize(n);
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> unit(0.0, 1.0), sym(-1.0, 1.0), energy(0.5, 1.5);
    const double gamma = 5.0 / 3.0;
    for (uint64_t i = 0; i < n; ++i) {
        for (int l = 0; l < 3; ++l) s.x[3 * i + l] = unit(rng);
        for (int l = 0; l < 3; ++l) s.v[3 * i + l] = sym(rng);
        s.u[i] = energy(rng);
        s.P[i] = (gamma - 1.0) * s.rho[i] * s.u[i];
        s.cs[i] = std::sqrt(gamma * s.P[i] / s.rho[i]);
        s.id[i] = int64_t(i);
    }
    return s;
}

// load_initial_conditions_csv (sph.cpp:351-383): rows id,x0,x1,x2,v0,v1,v2,u,m,h;
// blank lines, '#' comments and a header row starting with "id" are skipped;
// rho = 1, P/cs from the EOS, a = du = 0, dt = the run's dt.  Same errors as
// the reference: unreadable file / wrong column count -> runtime_error,
// unparsable number -> std::stod's invalid_argument / out_of_range.
State csv_state(const std::string& path, double dt) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open initial conditions file: " + path);
    State s;
    const double gamma = 5.0 / 3.0;
    std::string line;
    while (std::getline(in, line)) {
        if (line.empty() || line[0] == '#') continue;
        if (line.find_first_not_of(" \t") != std::string::npos && line.rfind("id", 0) == 0) continue;
        std::istringstream row(line);
        std::string cell;
        std::vector<double> vals;
        while (std::getline(row, cell, ',')) vals.push_back(std::stod(cell));
        if (vals.size() != 10) throw std::runtime_error("initial conditions row must have 10 columns: " + line);
        s.id.push_back(int64_t(vals[0]));
        for (int l = 0; l < 3; ++l) s.x.push_back(vals[1 + l]);
        for (int l = 0; l < 3; ++l) s.v.push_back(vals[4 + l]);
        s.u.push_back(vals[7]);
        s.m.push_back(vals[8]);
        s.h.push_back(vals[9]);
        s.rho.push_back(1.0);
        const double P = (gamma - 1.0) * 1.0 * vals[7];  // eos(rho = 1, u), sph.cpp:42-46
        s.P.push_back(P);
        s.cs.push_back(std::sqrt(gamma * P / 1.0));
        for (int l = 0; l < 3; ++l) s.a.push_back(0.0);
        s.du.push_back(0.0);
        s.dt.push_back(dt);
        ++s.n;
    }
    return s;
}

const std::vector<double>* state_field(const State& s, const std::string& f) {
    if (f == "x") return &s.x;
    if (f == "v") return &s.v;
    if (f == "a") return &s.a;
    if (f == "u") return &s.u;
    if (f == "m") return &s.m;
    if (f == "h") return &s.h;
    if (f == "rho") return &s.rho;
    if (f == "P") return &s.P;
    if (f == "cs") return &s.cs;
    if (f == "du") return &s.du;
    if (f == "dt") return &s.dt;
    return nullptr;
}

std::shared_ptr<const Schema> load_schema(const RunConfig& c, int precision, bool all_fields = false) {
    std::string text;
    if (c.schema_path.empty()) {
        text = builtin_schema_text();
    } else {
        std::ifstream in(c.schema_path);
        if (!in) throw std::runtime_error("cannot open schema file: " + c.schema_path);
        std::ostringstream ss;
        ss << in.rdbuf();
        text = ss.str();
    }
    Schema s = parse_schema_text(text);
    if (precision > 0) s = uniform_precision(s, precision, all_fields ? std::vector<std::string>{} : std::vector<std::string>{"x"});
    return std::make_shared<const Schema>(std::move(s));
}

// store_state (sph.cpp:385-412) on the device: the binary64 state as an f64
// SoA buffer, then one conversion kernel into the compressed AoS.
void store_state(const State& st, const View& aos, void* dev_aos) {
    View s64 = make_view(aos.schema, nullptr, Layout::SoA, 64, {}, st.n);
    std::vector<uint8_t> host(s64.total_bytes(), 0);
    for (size_t p = 0; p < s64.subset.size(); ++p) {
        const FieldDecl& f = s64.schema->fields[s64.subset[p]];
        uint8_t* base = host.data() + s64.lane_base(int(p)) / 8;
        if (f.name == "id" && !f.is_float()) {
            memcpy(base, st.id.data(), 8 * st.n);
            continue;
        }
        const std::vector<double>* src = state_field(st, f.name);
        if (src && src->size() == st.n * f.arity) memcpy(base, src->data(), 8 * st.n * f.arity);
    }
    DevBuf d(host.size());
    check_cuda(cudaMemcpy(d.p, host.data(), host.size(), cudaMemcpyHostToDevice), "H2D");
    convert(s64, d.p, aos, dev_aos, nullptr);
}

std::vector<uint8_t> download(const View& v, const void* p) {
    std::vector<uint8_t> h(v.total_bytes());
    check_cuda(cudaDeviceSynchronize(), "sync");
    if (!h.empty()) check_cuda(cudaMemcpy(h.data(), p, h.size(), cudaMemcpyDeviceToHost), "D2H");
    return h;
}

// pipelines.cpp:51-60 FNV-1a over the bytes then the bit length
uint64_t fnv(const std::vector<uint8_t>& bytes, uint64_t length_bits) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (uint8_t b : bytes) h = (h ^ b) * 0x100000001b3ull;
    for (int i = 0; i < 8; ++i) h = (h ^ uint8_t(length_bits >> (8 * i))) * 0x100000001b3ull;
    return h;
}

uint64_t checksum_packed(const View& v, const void* p) {
    // pack (and, for SoA, soa_to_aos) into the compressed AoS, then FNV
    View packed = make_view(v.schema, nullptr, Layout::AoS, kPrecStored, {}, v.count);
    packed.subset = v.subset;
    packed.fmt.clear();
    for (int f : v.subset) {
        const FieldDecl& d = v.schema->fields[f];
        packed.fmt.push_back(d.is_float() ? fmt_compressed(d.stored_width()) : fmt_int());
    }
    DevBuf d(packed.total_bytes());
    convert(v, p, packed, d.p, nullptr);
    return fnv(download(packed, d.p), packed.total_bits());
}

uint64_t host_read_bits(const std::vector<uint8_t>& b, uint64_t off, int w) {
    uint64_t v = 0;
    for (int k = 0; k < w; ++k) v |= uint64_t((b[(off + k) >> 3] >> ((off + k) & 7)) & 1) << k;
    return v;
}

// load_state of one float field (decoded lanes) from a downloaded buffer
std::vector<double> field_values(const View& v, const std::vector<uint8_t>& bytes, const std::string& name) {
    const int p = v.pos_of(name);
    if (p < 0) throw std::invalid_argument("field '" + name + "' missing");
    const Lanes L = v.lanes(p);
    std::vector<double> out(v.count * L.arity);
    for (uint64_t r = 0; r < v.count; ++r)
        for (int l = 0; l < L.arity; ++l)
            out[r * L.arity + l] = decode_lane(host_read_bits(bytes, L.base + r * L.stride + uint64_t(l) * L.fmt.width, L.fmt.width), L.fmt);
    return out;
}

template <typename Fn>
double gpu_seconds(Fn&& fn) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, nullptr);
    fn();
    cudaEventRecord(b, nullptr);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms * 1e-3;
}

void validate_cfg(const RunConfig& c) {
    if (c.buffer_size == 0 || c.particles % c.buffer_size != 0)
        throw std::invalid_argument("buffer size must divide the particle count");
    for (int t : c.precision_sweep)
        if (t < 7 || t > 64) throw std::invalid_argument("precision sweep value " + std::to_string(t) + " outside 7..64");
    if (!(c.latency_s >= 0) || !(c.bandwidth > 0))
        throw std::invalid_argument("interconnect model requires latency >= 0 and bandwidth > 0");
}

struct Population {
    std::shared_ptr<const Schema> schema;
    State ics;
};

Population population(const RunConfig& c, int precision, bool all_fields = false) {
    validate_cfg(c);
    Population p;
    p.schema = load_schema(c, precision, all_fields);
    // bench.cpp:66-70: buffers are sized by the population, the CSV's row count when given
    p.ics = c.ic_csv_path.empty() ? random_state(c.particles, c.seed, c.dt) : csv_state(c.ic_csv_path, c.dt);
    return p;
}

}  // namespace

// -------------------------------------------------------------- bench kernels
// bench.cpp:269-316
std::string cmd_bench_kernels(const RunConfig& c) {
    require_device();
    const std::vector<int> sweep = c.precision_sweep.empty() ? std::vector<int>{64, 32, 16} : c.precision_sweep;
    std::ostringstream out;
    out << header() << "kernel,layout,precision,particles,compute_s,speedup_vs_aos,checksum\n";
    for (int prec : sweep) {
        Population pop = population(c, prec);
        const uint64_t n = pop.ics.n;
        View aos = make_view(pop.schema, nullptr, Layout::AoS, kPrecStored, {}, n);
        View nat = make_view(pop.schema, nullptr, Layout::AoS, kPrecNative, {}, n);
        View soa = make_view(pop.schema, nullptr, Layout::SoA, kPrecNative, {}, n);
        DevBuf state(aos.total_bytes()), native(nat.total_bytes()), streams(soa.total_bytes());
        store_state(pop.ics, aos, state.p);
        convert(aos, state.p, nat, native.p, nullptr);
        gather(aos, state.p, soa, streams.p, nullptr, 0.0, 0, nullptr);
        for (const auto& k : c.kernels) {
            DevBuf work_a(nat.total_bytes()), work_s(soa.total_bytes());
            check_cuda(cudaMemcpy(work_a.p, native.p, nat.total_bytes(), cudaMemcpyDeviceToDevice), "D2D");
            check_cuda(cudaMemcpy(work_s.p, streams.p, soa.total_bytes(), cudaMemcpyDeviceToDevice), "D2D");
            const double ta = gpu_seconds([&] { run_kernel(nat, work_a.p, k, c.dt, c.buffer_size, c.per_access, 0, nullptr); });
            const uint64_t sa = checksum_packed(nat, work_a.p);
            const double ts = gpu_seconds([&] { run_kernel(soa, work_s.p, k, c.dt, c.buffer_size, c.per_access, 0, nullptr); });
            const uint64_t ss = checksum_packed(soa, work_s.p);
            out << k << ",aos," << prec << ',' << c.particles << ',' << ta << ",1," << sa << '\n';
            out << k << ",soa," << prec << ',' << c.particles << ',' << ts << ',' << (ts > 0 ? ta / ts : 0.0) << ',' << ss << '\n';
        }
    }
    return out.str();
}

// -------------------------------------------------------------- bench transform
// bench.cpp:214-267.  Conversion placement on a B200 build: "device" is the
// fused gather kernel after a full-record move; "host" placement would be a
// CPU conversion, which this library deliberately does not contain — its
// convert_s column is reported as nan and only the byte model is given.
std::string cmd_bench_transform(const RunConfig& c) {
    require_device();
    const std::vector<int> sweep = c.precision_sweep.empty() ? std::vector<int>{64, 32, 16} : c.precision_sweep;
    std::ostringstream out;
    out << header() << "kernel,placement,precision,particles,convert_s,bytes_moved,modeled_transfer_s,ratio\n";
    for (int prec : sweep) {
        Population pop = population(c, prec);
        const uint64_t n = pop.ics.n;
        View aos = make_view(pop.schema, nullptr, Layout::AoS, kPrecStored, {}, n);
        DevBuf state(aos.total_bytes());
        store_state(pop.ics, aos, state.p);
        std::vector<std::string> sets = {""};
        for (const auto& k : c.kernels) sets.push_back(k);
        for (const auto& set : sets) {
            View soa = make_view(pop.schema, set.empty() ? nullptr : set.c_str(), Layout::SoA, kPrecNative, {}, n);
            DevBuf streams(soa.total_bytes());
            const double dev_convert = gpu_seconds([&] { gather(aos, state.p, soa, streams.p, nullptr, 0.0, 0, nullptr); });
            const uint64_t host_bytes = soa.total_bytes(), dev_bytes = aos.total_bytes();
            const double host_model = c.latency_s + double(host_bytes) / c.bandwidth;
            const double dev_model = c.latency_s + double(dev_bytes) / c.bandwidth;
            const std::string name = set.empty() ? "full" : set;
            out << name << ",host," << prec << ',' << c.particles << ",nan," << host_bytes << ',' << host_model << ",nan\n";
            out << name << ",device," << prec << ',' << c.particles << ',' << dev_convert << ',' << dev_bytes << ',' << dev_model
                << ",nan\n";
        }
    }
    return out.str();
}

// -------------------------------------------------------------- pipeline
namespace {

enum class Conv { None, Unpack, UnpackSoA };

Conv conv_of(const std::string& v) {
    if (v == "cpu-baseline" || v == "dev-native") return Conv::None;
    if (v == "cpu-soa" || v == "dev-soa" || v == "host-soa-stream") return Conv::UnpackSoA;
    return Conv::Unpack;
}
bool is_cpu(const std::string& v) { return v.rfind("cpu-", 0) == 0; }
bool is_host(const std::string& v) { return v.rfind("host-", 0) == 0; }

struct VariantResult {
    double convert_s = 0, move_s = 0, compute_s = 0, merge_s = 0;
    std::map<std::string, double> kernel_s;
    uint64_t to_dev = 0, to_host = 0, transfers = 0;
    uint64_t checksum = 0;
};

struct PinnedBuf {
    void* p = nullptr;
    explicit PinnedBuf(size_t bytes) { check_cuda(cudaHostAlloc(&p, bytes + 16, cudaHostAllocDefault), "cudaHostAlloc"); }
    PinnedBuf(const PinnedBuf&) = delete;
    ~PinnedBuf() { cudaFreeHost(p); }
};

// pipelines::run_variant (pipelines.cpp:378-405) on the GPU, over real PCIe.
// The state lives in pinned host memory.  dev-* variants: in-place moves the
// whole compressed AoS to the device once, runs every kernel there (through
// the variant's conversions) and moves it back (run_dev_inplace,
// pipelines.cpp:231-249); streaming moves, per kernel, only the narrowed
// fields each way — read from / stored into the host records in place by the
// conversion kernels (zero copy: only the narrowed lanes cross PCIe; 1.6x
// faster than moving them as byte columns with 2-D DMA, measured in round 2)
// — and converts on the device
// (run_dev_streaming, :251-296).  move_s is the measured transfer time and bytes_to_device /
// bytes_to_host the bytes actually copied (= the reference ledger).
// cpu-* variants run on the device with no transfer (their state is where
// the compute is).  host-* variants place the conversion on the host in the
// reference (:298-368), which needs a CPU conversion this library does not
// contain: they keep the ledger byte model with move_s = 0 (bench.py times
// host placement with the reference's own CPU conversion).
VariantResult run_variant_gpu(const RunConfig& c, const Population& pop, const std::string& variant,
                              const std::string& mode, bool fault) {
    const uint64_t n = pop.ics.n;
    View aos = make_view(pop.schema, nullptr, Layout::AoS, kPrecStored, {}, n);
    DevBuf state(aos.total_bytes());
    store_state(pop.ics, aos, state.p);
    VariantResult res;
    const bool dev = variant.rfind("dev-", 0) == 0;
    const bool stream_mode = mode == "streaming" && !is_cpu(variant);
    const size_t abytes = size_t(aos.total_bytes());
    std::unique_ptr<PinnedBuf> hstate;
    if (dev) {  // the state starts (and ends) in pinned host memory
        hstate.reset(new PinnedBuf(abytes));
        check_cuda(cudaMemcpy(hstate->p, state.p, abytes, cudaMemcpyDeviceToHost), "D2H");
        check_cuda(cudaMemset(state.p, 0, abytes), "memset");
    }
    if (!is_cpu(variant) && !stream_mode) {  // one full round trip each way
        // dev variants move the compressed state, host variants the unpacked one
        const uint64_t b = is_host(variant) ? make_view(pop.schema, nullptr, Layout::AoS, kPrecNative, {}, n).total_bytes()
                                            : aos.total_bytes();
        res.to_dev += b;
        res.to_host += b;
        res.transfers += 2;
        if (dev)
            res.move_s += gpu_seconds([&] {
                check_cuda(cudaMemcpyAsync(state.p, hstate->p, abytes, cudaMemcpyHostToDevice, nullptr), "H2D");
            });
    }
    for (const auto& k : c.kernels) {
        const KernelSet* set = pop.schema->kernel(k);
        if (!set) throw std::invalid_argument("no access set declared for kernel '" + k + "'");
        const Conv cv = conv_of(variant);
        if (stream_mode && dev) {
            // N: narrowed compressed AoS of the kernel's fields, straight from the host records
            View nv = make_view(pop.schema, k.c_str(), Layout::AoS, kPrecStored, {}, n);
            DevBuf nb(nv.total_bytes());
            const bool cols = aos.byte_aligned() && nv.byte_aligned() && aos.record_bits() % 8 == 0 &&
                              nv.record_bits() % 8 == 0;
            res.to_dev += nv.total_bytes();
            res.to_host += nv.total_bytes();
            res.transfers += 2;
            res.move_s += gpu_seconds([&] {
                if (cols) {  // the device reads the narrowed lanes of the host records in place
                    gather(aos, hstate->p, nv, nb.p, nullptr, 0.0, 0, nullptr, true);
                } else {  // bit-packed records: whole records over PCIe, narrowed on the device
                    check_cuda(cudaMemcpyAsync(state.p, hstate->p, abytes, cudaMemcpyHostToDevice, nullptr), "H2D");
                    convert(aos, state.p, nv, nb.p, nullptr);
                }
            });
            if (cv == Conv::None) {
                const double t = gpu_seconds([&] { run_kernel(nv, nb.p, k, c.dt, c.buffer_size, c.per_access, 0, nullptr); });
                res.compute_s += t;
                res.kernel_s[k] += t;
            } else {
                View work = make_view(pop.schema, k.c_str(), cv == Conv::UnpackSoA ? Layout::SoA : Layout::AoS,
                                      kPrecNative, {}, n);
                DevBuf w(work.total_bytes());
                res.convert_s += gpu_seconds([&] { gather(nv, nb.p, work, w.p, nullptr, 0.0, 0, nullptr); });
                const double t = gpu_seconds([&] { run_kernel(work, w.p, k, c.dt, c.buffer_size, c.per_access, 0, nullptr); });
                res.compute_s += t;
                res.kernel_s[k] += t;
                if (!set->writes.empty())
                    res.convert_s += gpu_seconds([&] { scatter_merge(work, w.p, nv, nb.p, k, nullptr); });
            }
            // N^T: the narrowed fields back into the host records (read-only fields come back bit-identical)
            res.move_s += gpu_seconds([&] {
                if (cols) {  // ... and stores them back in place
                    convert_fields(nv, nb.p, aos, hstate->p, nv.subset, nullptr, true);
                } else {
                    scatter_merge(nv, nb.p, aos, state.p, k, nullptr);
                    check_cuda(cudaMemcpyAsync(hstate->p, state.p, abytes, cudaMemcpyDeviceToHost, nullptr), "D2H");
                }
            });
            continue;
        }
        if (stream_mode) {  // host-* streaming: ledger only (no CPU conversion in this library)
            View nv = make_view(pop.schema, k.c_str(), Layout::AoS, kPrecNative, {}, n);
            res.to_dev += nv.total_bytes();
            res.to_host += nv.total_bytes();
            res.transfers += 2;
        }
        if (cv == Conv::None) {
            const double t = gpu_seconds([&] { run_kernel(aos, state.p, k, c.dt, c.buffer_size, c.per_access, 0, nullptr); });
            res.compute_s += t;
            res.kernel_s[k] += t;
            continue;
        }
        View work = make_view(pop.schema, k.c_str(), cv == Conv::UnpackSoA ? Layout::SoA : Layout::AoS, kPrecNative, {}, n);
        DevBuf w(work.total_bytes());
        res.convert_s += gpu_seconds([&] { gather(aos, state.p, work, w.p, nullptr, 0.0, 0, nullptr); });
        const double t = gpu_seconds([&] { run_kernel(work, w.p, k, c.dt, c.buffer_size, c.per_access, 0, nullptr); });
        res.compute_s += t;
        res.kernel_s[k] += t;
        if (!set->writes.empty()) res.merge_s += gpu_seconds([&] { scatter_merge(work, w.p, aos, state.p, k, nullptr); });
    }
    std::vector<uint8_t> bytes;
    if (dev) {
        if (!stream_mode)
            res.move_s += gpu_seconds([&] {
                check_cuda(cudaMemcpyAsync(hstate->p, state.p, abytes, cudaMemcpyDeviceToHost, nullptr), "D2H");
            });
        const uint8_t* hp = static_cast<const uint8_t*>(hstate->p);
        bytes.assign(hp, hp + abytes);
    } else {
        bytes = download(aos, state.p);
    }
    if (fault && !bytes.empty()) bytes[0] ^= 0x01;  // bench.cpp:577-578
    res.checksum = fnv(bytes, aos.total_bits());
    return res;
}

}  // namespace

std::string cmd_bench_pipeline(const RunConfig& c) {
    require_device();
    const std::vector<int> sweep = c.precision_sweep.empty() ? std::vector<int>{64, 32, 16} : c.precision_sweep;
    std::ostringstream out;
    out << header()
        << "variant,mode,precision,particles,total_s,convert_s,move_s,compute_s,merge_s,"
           "bytes_to_device,bytes_to_host,modeled_transfer_s,"
           "share_density,share_force,share_kick,share_drift,checksum\n";
    for (int prec : sweep) {
        Population pop = population(c, prec);
        for (const auto& v : c.variants)
            for (const auto& mode : c.modes) {
                VariantResult r = run_variant_gpu(c, pop, v, mode, false);
                auto share = [&](const char* k) {
                    auto it = r.kernel_s.find(k);
                    return it == r.kernel_s.end() || r.compute_s <= 0 ? 0.0 : it->second / r.compute_s;
                };
                const double model = double(r.transfers) * c.latency_s + double(r.to_dev + r.to_host) / c.bandwidth;
                out << v << ',' << mode << ',' << prec << ',' << c.particles << ','
                    << (r.convert_s + r.move_s + r.compute_s + r.merge_s) << ',' << r.convert_s << ',' << r.move_s << ','
                    << r.compute_s << ',' << r.merge_s << ',' << r.to_dev << ',' << r.to_host << ',' << model << ','
                    << share("density") << ',' << share("force") << ',' << share("kick") << ',' << share("drift") << ','
                    << r.checksum << '\n';
            }
    }
    return out.str();
}

// -------------------------------------------------------------- truncation
// bench.cpp:362-418: RMS error of the force acceleration vs the 64-bit run
std::string cmd_study_truncation(const RunConfig& c) {
    require_device();
    static const std::vector<int> kSweep = {64, 56, 48, 40, 34, 33, 32, 24, 17, 16, 12};
    const std::vector<int>& sweep = c.precision_sweep.empty() ? kSweep : c.precision_sweep;
    for (int t : sweep)
        if (t < 7 || t > 64) throw std::invalid_argument("sweep value " + std::to_string(t) + " outside 7..64");
    auto run_once = [&](int prec) {
        Population pop = population(c, prec);
        View aos = make_view(pop.schema, nullptr, Layout::AoS, kPrecStored, {}, pop.ics.n);
        DevBuf state(aos.total_bytes());
        store_state(pop.ics, aos, state.p);
        run_kernel(aos, state.p, "density", c.dt, c.buffer_size, c.per_access, 0, nullptr);
        run_kernel(aos, state.p, "force", c.dt, c.buffer_size, c.per_access, 0, nullptr);
        return field_values(aos, download(aos, state.p), "a");
    };
    const std::vector<double> ref = run_once(64);
    const uint64_t n = ref.size() / 3;
    double norm = 0;
    for (uint64_t i = 0; i < n; ++i)
        norm += std::sqrt(ref[3 * i] * ref[3 * i] + ref[3 * i + 1] * ref[3 * i + 1] + ref[3 * i + 2] * ref[3 * i + 2]);
    norm /= double(n);
    std::ostringstream out;
    out.precision(17);
    out << header() << "total_bits,rmse_rel,max_rel\n";
    for (int prec : sweep) {
        const std::vector<double> a = run_once(prec);
        double sum_sq = 0, max_err = 0;
        for (uint64_t i = 0; i < n; ++i) {
            const double e0 = a[3 * i] - ref[3 * i], e1 = a[3 * i + 1] - ref[3 * i + 1], e2 = a[3 * i + 2] - ref[3 * i + 2];
            const double err = std::sqrt(e0 * e0 + e1 * e1 + e2 * e2);
            sum_sq += err * err;
            max_err = std::max(max_err, err);
        }
        out << prec << ',' << std::sqrt(sum_sq / double(n)) / norm << ',' << max_err / norm << '\n';
    }
    return out.str();
}

// -------------------------------------------------------------- validate
// bench.cpp:420-604, the same PASS/FAIL battery with the GPU path under test
// and independent host restatements as the checkers.
namespace {

double naive_w(double r, double h) {
    const double q = r / h;
    if (q >= 2.0) return 0.0;
    const double norm = (1.0 / 3.14159265358979323846) / (h * h * h);
    if (q < 1.0) return norm * (1.0 - 1.5 * q * q + 0.75 * q * q * q);
    const double t = 2.0 - q;
    return norm * 0.25 * t * t * t;
}
double naive_dwdr(double r, double h) {
    const double q = r / h;
    if (q >= 2.0) return 0.0;
    const double norm = (1.0 / 3.14159265358979323846) / (h * h * h * h);
    if (q < 1.0) return norm * (-3.0 * q + 2.25 * q * q);
    const double t = 2.0 - q;
    return norm * (-0.75 * t * t);
}

}  // namespace

std::string cmd_validate(const RunConfig& c, int& failures) {
    require_device();
    validate_cfg(c);
    failures = 0;
    std::ostringstream rep;
    auto check = [&](const char* name, bool ok) {
        rep << (ok ? "PASS " : "FAIL ") << name << '\n';
        if (!ok) ++failures;
    };
    // fpcodec: frozen values and idempotence (host scalar codec = sf_quantize)
    {
        auto q = [](double x, int t) { const LaneFmt f = fmt_compressed(t); return decode_lane(encode_lane(x, f), f); };
        bool ok = q(3.14159265358979323846, 17) == 3.140625 && q(3.14159265358979323846, 32) == 3.1415927410125732;
        std::mt19937_64 rng(c.seed);
        std::uniform_real_distribution<double> val(-1e4, 1e4);
        std::uniform_int_distribution<int> width(7, 64);
        for (int i = 0; i < 1000 && ok; ++i) {
            const int t = width(rng);
            const double x = q(val(rng), t);
            ok &= q(x, t) == x;
        }
        check("fpcodec-quantize", ok);
    }
    // bit-level lanes on the device: a bit-packed schema round-trips AoS->SoA->AoS
    // and merging one field leaves every other bit alone
    {
        auto s = std::make_shared<const Schema>(parse_schema_text(
            "schema bits { field a : f32 @truncate(7); field b : f64 @truncate(45); field c : f32 x3 @truncate(19);"
            " field d : i64; field e : f32 @truncate(11); }\nkernel touch_c reads c writes c;\n"));
        const uint64_t n = 257;
        View aos = make_view(s, nullptr, Layout::AoS, kPrecStored, {}, n);
        View soa = make_view(s, nullptr, Layout::SoA, kPrecStored, {}, n);
        std::vector<uint8_t> bytes(aos.total_bytes());
        std::mt19937_64 rng(c.seed + 1);
        for (auto& b : bytes) b = uint8_t(rng());
        if (aos.total_bits() % 8) bytes.back() &= uint8_t((1u << (aos.total_bits() % 8)) - 1);
        DevBuf d(bytes.size()), t(soa.total_bytes()), back(bytes.size());
        check_cuda(cudaMemcpy(d.p, bytes.data(), bytes.size(), cudaMemcpyHostToDevice), "H2D");
        convert(aos, d.p, soa, t.p, nullptr);
        convert(soa, t.p, aos, back.p, nullptr);
        bool ok = download(aos, back.p) == bytes;
        // locality: merge field c from a zeroed SoA; only c's bits may change
        check_cuda(cudaMemset(t.p, 0, soa.total_bytes()), "memset");
        scatter_merge(soa, t.p, aos, d.p, "touch_c", nullptr);
        const std::vector<uint8_t> after = download(aos, d.p);
        const int cp = aos.pos_of("c");
        for (uint64_t r = 0; r < n && ok; ++r)
            for (uint64_t bit = r * aos.record_bits(); bit < (r + 1) * aos.record_bits(); ++bit) {
                const uint64_t rel = bit - r * aos.record_bits();
                const bool in_c = rel >= aos.lane_base(cp) && rel < aos.lane_base(cp) + 3 * 19;
                const int was = (bytes[bit >> 3] >> (bit & 7)) & 1, now = (after[bit >> 3] >> (bit & 7)) & 1;
                ok &= in_c ? now == 0 : now == was;
            }
        check("bitpack-roundtrip", ok);
    }
    // lossless operator identities over the active schema
    {
        RunConfig small = c;
        small.particles = std::min<uint64_t>(c.particles, 256);
        small.particles -= small.particles % small.buffer_size;
        if (small.particles == 0) small.particles = small.buffer_size;
        Population pop = population(small, 0);
        const uint64_t n = pop.ics.n;
        View aos = make_view(pop.schema, nullptr, Layout::AoS, kPrecStored, {}, n);
        View soa = make_view(pop.schema, nullptr, Layout::SoA, kPrecStored, {}, n);
        View nat = make_view(pop.schema, nullptr, Layout::AoS, kPrecNative, {}, n);
        DevBuf st(aos.total_bytes()), a(soa.total_bytes()), b(aos.total_bytes()), u(nat.total_bytes());
        store_state(pop.ics, aos, st.p);
        const std::vector<uint8_t> ref = download(aos, st.p);
        convert(aos, st.p, soa, a.p, nullptr);
        convert(soa, a.p, aos, b.p, nullptr);
        bool ok = download(aos, b.p) == ref;
        convert(aos, st.p, nat, u.p, nullptr);
        convert(nat, u.p, aos, b.p, nullptr);
        ok &= download(aos, b.p) == ref;
        check("lossless-identities", ok);
    }
    // density + force in native binary64 vs direct double loops (bit-exact)
    bool momentum_ok = true;
    {
        RunConfig wide = c;
        wide.particles = std::min<uint64_t>(c.particles, 512);
        wide.particles -= wide.particles % wide.buffer_size;
        if (wide.particles == 0) wide.particles = wide.buffer_size;
        Population pop = population(wide, 64, true);
        const uint64_t n = pop.ics.n, bs = wide.buffer_size;
        View aos = make_view(pop.schema, nullptr, Layout::AoS, kPrecStored, {}, n);
        DevBuf st(aos.total_bytes());
        store_state(pop.ics, aos, st.p);
        run_kernel(aos, st.p, "density", c.dt, bs, 0, 0, nullptr);
        run_kernel(aos, st.p, "force", c.dt, bs, 0, 0, nullptr);
        const std::vector<uint8_t> bytes = download(aos, st.p);
        const std::vector<double> rho = field_values(aos, bytes, "rho"), a = field_values(aos, bytes, "a"),
                                  du = field_values(aos, bytes, "du");
        State s = pop.ics;
        bool ok = true;
        for (uint64_t b0 = 0; b0 < n; b0 += bs) {
            for (uint64_t i = b0; i < b0 + bs; ++i) {
                double acc = 0;
                for (uint64_t j = b0; j < b0 + bs; ++j) {
                    const double d0 = s.x[3 * i] - s.x[3 * j], d1 = s.x[3 * i + 1] - s.x[3 * j + 1], d2 = s.x[3 * i + 2] - s.x[3 * j + 2];
                    acc += s.m[j] * naive_w(std::sqrt(d0 * d0 + d1 * d1 + d2 * d2), 0.5 * (s.h[i] + s.h[j]));
                }
                s.rho[i] = acc;
                ok &= rho[i] == acc;
            }
            for (uint64_t i = b0; i < b0 + bs; ++i) {
                const double pr = s.P[i] / (s.rho[i] * s.rho[i]);
                double ac[3] = {0, 0, 0}, compr = 0;
                for (uint64_t j = b0; j < b0 + bs; ++j) {
                    if (j == i) continue;
                    const double d0 = s.x[3 * i] - s.x[3 * j], d1 = s.x[3 * i + 1] - s.x[3 * j + 1], d2 = s.x[3 * i + 2] - s.x[3 * j + 2];
                    const double r = std::sqrt(d0 * d0 + d1 * d1 + d2 * d2);
                    double g0 = 0, g1 = 0, g2 = 0;
                    if (r != 0.0) {
                        const double sc = naive_dwdr(r, 0.5 * (s.h[i] + s.h[j])) / r;
                        g0 = sc * d0, g1 = sc * d1, g2 = sc * d2;
                    }
                    const double pf = pr + s.P[j] / (s.rho[j] * s.rho[j]);
                    ac[0] -= s.m[j] * pf * g0;
                    ac[1] -= s.m[j] * pf * g1;
                    ac[2] -= s.m[j] * pf * g2;
                    compr += s.m[j] * ((s.v[3 * i] - s.v[3 * j]) * g0 + (s.v[3 * i + 1] - s.v[3 * j + 1]) * g1 +
                                       (s.v[3 * i + 2] - s.v[3 * j + 2]) * g2);
                }
                for (int l = 0; l < 3; ++l) ok &= a[3 * i + l] == ac[l];
                ok &= du[i] == pr * compr;
            }
            double net[3] = {0, 0, 0}, scale = 0;
            for (uint64_t i = b0; i < b0 + bs; ++i) {
                const double mag = std::sqrt(a[3 * i] * a[3 * i] + a[3 * i + 1] * a[3 * i + 1] + a[3 * i + 2] * a[3 * i + 2]);
                scale += std::abs(s.m[i]) * mag;
                for (int l = 0; l < 3; ++l) net[l] += s.m[i] * a[3 * i + l];
            }
            momentum_ok &= std::sqrt(net[0] * net[0] + net[1] * net[1] + net[2] * net[2]) <= 1e-12 * scale;
        }
        check("oracle-equivalence", ok);
        check("momentum-conservation", momentum_ok);
    }
    {
        const int steps = 4096;
        const double dr = 2.0 / steps;
        double integral = 0.0;
        for (int i = 0; i <= steps; ++i) {
            const double r = i * dr;
            integral += 4.0 * 3.14159265358979323846 * naive_w(r, 1.0) * r * r * (i == 0 || i == steps ? 1.0 : (i % 2 ? 4.0 : 2.0));
        }
        check("kernel-normalization", std::abs(integral * dr / 3.0 - 1.0) <= 1e-6);
    }
    {
        RunConfig small = c;
        small.particles = std::min<uint64_t>(c.particles, 256);
        small.particles -= small.particles % small.buffer_size;
        if (small.particles == 0) small.particles = small.buffer_size;
        small.kernels = {"density", "force", "kick", "drift"};
        small.per_access = false;
        Population pop = population(small, 0);
        bool ok = true, first = true;
        uint64_t expected = 0;
        for (const auto& v : RunConfig().variants)
            for (const char* mode : {"inplace", "streaming"}) {
                const uint64_t sum =
                    run_variant_gpu(small, pop, v, mode, c.fault && v == "dev-soa" && std::string(mode) == "streaming").checksum;
                if (first) expected = sum, first = false;
                else ok &= sum == expected;
            }
        check("cross-variant-checksums", ok);
        if (c.dump) {
            View aos = make_view(pop.schema, nullptr, Layout::AoS, kPrecStored, {}, pop.ics.n);
            DevBuf st(aos.total_bytes());
            store_state(pop.ics, aos, st.p);
            const std::vector<uint8_t> b = download(aos, st.p);
            const size_t head = std::min<size_t>(b.size(), size_t((small.buffer_size * aos.record_bits() + 7) / 8));
            char hex[4];
            for (size_t i = 0; i < head; ++i) {
                std::snprintf(hex, sizeof hex, "%02x", b[i]);
                rep << hex << ((i % 16 == 15 || i + 1 == head) ? '\n' : ' ');
            }
        }
    }
    return rep.str();
}

}  // namespace sfb
