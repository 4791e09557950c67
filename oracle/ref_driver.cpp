// TEST INFRASTRUCTURE — not part of the product.
//
// A thin extern "C" shim over the *unmodified* reference library
// (soaforge, compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/).  It lets the Python test suite and bench.py's CPU-baseline
// leg drive the reference's own operators:
//   - golden-vector generation (tests/golden/make_golden.py),
//   - oracle pinning (the C restatement in oracle/soa_oracle.c is checked
//     against these outputs),
//   - the `bench.py --impl reference` arm (reference CPU path, timed).
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load this library.
#include <soaforge/bench.hpp>
#include <soaforge/fpcodec.hpp>
#include <soaforge/layout_ops.hpp>
#include <soaforge/pipelines.hpp>
#include <soaforge/schema.hpp>
#include <soaforge/sph.hpp>

#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

using namespace soaforge;
using layoutops::ArenaId;
using layoutops::LayoutTag;
using layoutops::Machine;
using layoutops::PackedBuffer;
using layoutops::PrecisionTag;

namespace {

thread_local std::string g_err;

struct RefBuf {
    PackedBuffer buf;
    std::vector<schema::KernelAccessSet> sets;
};

std::vector<std::string> split_csv(const char* s) {
    std::vector<std::string> out;
    if (!s) return out;
    std::stringstream ss(s);
    std::string item;
    while (std::getline(ss, item, ','))
        if (!item.empty()) out.push_back(item);
    return out;
}

// Schema text (nullptr -> built-in particle schema) optionally rewritten by
// with_uniform_precision(T, exclude).
schema::SchemaFile schema_for(const char* text, int T, const char* exclude_csv) {
    schema::SchemaFile f = schema::parse_file(text ? text : sph::default_schema_text());
    if (T > 0) f.schema = schema::with_uniform_precision(f.schema, T, split_csv(exclude_csv));
    return f;
}

const schema::KernelAccessSet& find_set(const RefBuf& b, const char* name) {
    for (const auto& s : b.sets)
        if (s.kernel == name) return s;
    throw std::invalid_argument(std::string("no access set ") + name);
}

template <typename Fn>
void* guard_ptr(Fn&& fn) {
    try {
        return fn();
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

template <typename Fn>
int guard_int(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

sph::ParticleSoA make_ics(std::uint64_t n, std::uint64_t seed, std::uint64_t accel_seed,
                          double dt) {
    sph::KernelParams p;
    p.dt = dt;
    sph::ParticleSoA s = sph::random_initial_conditions(n, seed, p);
    if (accel_seed != 0) {
        // Seed a and du so kick is not a no-op (the reference ICs zero them).
        std::mt19937_64 rng(accel_seed);
        std::uniform_real_distribution<double> sym(-1.0, 1.0);
        for (std::uint64_t i = 0; i < n; ++i) {
            for (int l = 0; l < 3; ++l) s.a[i][l] = sym(rng);
            s.du[i] = sym(rng);
        }
    }
    return s;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// ---- scalar fpcodec -------------------------------------------------------
uint64_t ref_narrow_to_ieee(double x, int e, int m) { return fpcodec::narrow_to_ieee(x, e, m); }
double ref_widen_from_ieee(uint64_t b, int e, int m) { return fpcodec::widen_from_ieee(b, e, m); }
uint64_t ref_encode_bits(double x, int T) { return fpcodec::encode_bits(x, fpcodec::layout_for(T)); }
double ref_decode_bits(uint64_t b, int T) { return fpcodec::decode_bits(b, fpcodec::layout_for(T)); }
double ref_quantize(double x, int T) { return fpcodec::quantize(x, fpcodec::layout_for(T)); }

void ref_narrow_array(const double* x, uint64_t n, int e, int m, uint64_t* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = fpcodec::narrow_to_ieee(x[i], e, m);
}
void ref_encode_array(const double* x, uint64_t n, int T, uint64_t* out) {
    const auto spec = fpcodec::layout_for(T);
    for (uint64_t i = 0; i < n; ++i) out[i] = fpcodec::encode_bits(x[i], spec);
}

// ---- schema ---------------------------------------------------------------
// Writes record_bits and per-field (offset_bits, width, arity, kind) rows.
int ref_schema_layout(const char* text, int T, const char* exclude, uint64_t* record_bits,
                      int64_t* rows, int max_fields, int* nfields) {
    return guard_int([&] {
        auto f = schema_for(text, T, exclude);
        *record_bits = f.schema.record_bits;
        *nfields = int(f.schema.fields.size());
        for (int i = 0; i < *nfields && i < max_fields; ++i) {
            const auto& d = f.schema.fields[i];
            rows[4 * i + 0] = int64_t(f.schema.slots[i].offset_bits);
            rows[4 * i + 1] = d.stored_width();
            rows[4 * i + 2] = d.arity;
            rows[4 * i + 3] = d.base == schema::BaseKind::F32 ? 0 : d.base == schema::BaseKind::F64 ? 1 : 2;
        }
    });
}

// ---- packed-buffer handles ------------------------------------------------
// make_population + make_state: random ICs (seed) stored through the schema.
void* ref_buf_from_ics(const char* text, int T, const char* exclude, uint64_t n, uint64_t seed,
                       uint64_t accel_seed, double dt) {
    return guard_ptr([&]() -> void* {
        auto f = schema_for(text, T, exclude);
        auto rb = std::make_unique<RefBuf>();
        Machine m;
        auto rs = std::make_shared<schema::RecordSchema>(f.schema);
        rb->buf = layoutops::make_buffer(rs, n, LayoutTag::AoS, PrecisionTag::Compressed,
                                         ArenaId::Host, m);
        rb->sets = f.kernels;
        sph::BufferView view(rb->buf);
        sph::store_state(make_ics(n, seed, accel_seed, dt), view);
        return rb.release();
    });
}

// Compressed AoS over the full field set from raw bytes.
void* ref_buf_from_bytes(const char* text, int T, const char* exclude, uint64_t n,
                         const uint8_t* bytes, uint64_t nbytes) {
    return guard_ptr([&]() -> void* {
        auto f = schema_for(text, T, exclude);
        auto rb = std::make_unique<RefBuf>();
        Machine m;
        auto rs = std::make_shared<schema::RecordSchema>(f.schema);
        rb->buf = layoutops::make_buffer(rs, n, LayoutTag::AoS, PrecisionTag::Compressed,
                                         ArenaId::Host, m);
        rb->sets = f.kernels;
        if (nbytes != rb->buf.data.bytes.size()) throw std::invalid_argument("byte count mismatch");
        std::memcpy(rb->buf.data.bytes.data(), bytes, nbytes);
        return rb.release();
    });
}

// load_state(src) -> store_state(new compressed AoS over schema(T, exclude)).
// This is the reference's f32/f64 -> T-bit narrowing entry (sph.cpp:385-443).
void* ref_buf_restore(void* h, const char* text, int T, const char* exclude) {
    return guard_ptr([&]() -> void* {
        auto* src = static_cast<RefBuf*>(h);
        sph::BufferView sv(src->buf);
        sph::ParticleSoA s = sph::load_state(sv);
        auto f = schema_for(text, T, exclude);
        auto rb = std::make_unique<RefBuf>();
        Machine m;
        auto rs = std::make_shared<schema::RecordSchema>(f.schema);
        rb->buf = layoutops::make_buffer(rs, src->buf.count, LayoutTag::AoS,
                                         PrecisionTag::Compressed, ArenaId::Host, m);
        rb->sets = f.kernels;
        sph::BufferView dv(rb->buf);
        sph::store_state(s, dv);
        return rb.release();
    });
}

void* ref_buf_clone(void* h) {
    return guard_ptr([&]() -> void* { return new RefBuf(*static_cast<RefBuf*>(h)); });
}

// op: unpack | pack | aos_to_soa | soa_to_aos | narrow  (narrow takes `kernel`)
void* ref_buf_op(void* h, const char* op, const char* kernel) {
    return guard_ptr([&]() -> void* {
        auto* b = static_cast<RefBuf*>(h);
        auto out = std::make_unique<RefBuf>();
        out->sets = b->sets;
        const std::string o = op;
        if (o == "unpack") out->buf = layoutops::unpack(b->buf);
        else if (o == "pack") out->buf = layoutops::pack(b->buf);
        else if (o == "aos_to_soa") out->buf = layoutops::aos_to_soa(b->buf);
        else if (o == "soa_to_aos") out->buf = layoutops::soa_to_aos(b->buf);
        else if (o == "narrow") out->buf = layoutops::narrow(b->buf, find_set(*b, kernel));
        else throw std::invalid_argument("unknown op " + o);
        return out.release();
    });
}

int ref_buf_widen_merge(void* narrowed, void* original, const char* kernel) {
    return guard_int([&] {
        auto* o = static_cast<RefBuf*>(original);
        layoutops::widen_merge(static_cast<RefBuf*>(narrowed)->buf, o->buf, find_set(*o, kernel));
    });
}

int ref_buf_run_kernel(void* h, const char* kernel, uint64_t buffer_size, double dt,
                       int per_access, int threads) {
    return guard_int([&] {
        auto* b = static_cast<RefBuf*>(h);
        sph::BufferView view(b->buf);
        sph::KernelParams p;
        p.dt = dt;
        sph::run_kernel_chunked(sph::kernel_from_name(kernel), view, buffer_size, p,
                                per_access ? sph::Writeback::PerAccess : sph::Writeback::Deferred,
                                threads);
    });
}

uint64_t ref_buf_nbytes(void* h) { return static_cast<RefBuf*>(h)->buf.data.bytes.size(); }
uint64_t ref_buf_bits(void* h) { return static_cast<RefBuf*>(h)->buf.data.length_bits; }
void ref_buf_copy_bytes(void* h, uint8_t* out) {
    auto& v = static_cast<RefBuf*>(h)->buf.data.bytes;
    std::memcpy(out, v.data(), v.size());
}
uint64_t ref_buf_checksum(void* h) { return pipelines::checksum(static_cast<RefBuf*>(h)->buf); }
void ref_buf_free(void* h) { delete static_cast<RefBuf*>(h); }

// ---- analytic byte model ----------------------------------------------------
uint64_t ref_streamed_bytes_one_way(const char* text, int T, const char* exclude,
                                    const char* kernel, uint64_t count, const char* variant) {
    auto f = schema_for(text, T, exclude);
    for (const auto& s : f.kernels)
        if (s.kernel == kernel)
            return pipelines::streamed_bytes_one_way(f.schema, s, count,
                                                     pipelines::variant_from_name(variant));
    return 0;
}

// ---- CPU baseline: the reference's own path for the C2 composition ----------
// Per thread: its own slice of `n_per_thread` default-schema particles.
// Timed region (per slice, all threads concurrently):
//   load_state(default AoS) -> store_state(T-bit AoS, x included)      [N: narrowing]
//   -> unpack -> narrow(drift) -> aos_to_soa                           [U, N, C]
//   -> run_kernel_chunked(drift, SoA view, 64, dt)                     [compute]
// Returns wall seconds of the timed region (max over threads == wall).
double ref_time_c2(uint64_t n_per_thread, int threads, int T, uint64_t seed, double dt) {
    try {
        std::vector<std::unique_ptr<RefBuf>> src(threads);
        for (int t = 0; t < threads; ++t)
            src[t].reset(static_cast<RefBuf*>(
                ref_buf_from_ics(nullptr, 0, nullptr, n_per_thread, seed + t, 0, dt)));
        for (auto& s : src)
            if (!s) return -1.0;
        auto work = [&](int t) {
            RefBuf* d = static_cast<RefBuf*>(ref_buf_restore(src[t].get(), nullptr, T, ""));
            RefBuf* u = static_cast<RefBuf*>(ref_buf_op(d, "unpack", nullptr));
            RefBuf* nw = static_cast<RefBuf*>(ref_buf_op(u, "narrow", "drift"));
            RefBuf* so = static_cast<RefBuf*>(ref_buf_op(nw, "aos_to_soa", nullptr));
            ref_buf_run_kernel(so, "drift", 64, dt, 0, 1);
            ref_buf_free(d);
            ref_buf_free(u);
            ref_buf_free(nw);
            ref_buf_free(so);
        };
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t) pool.emplace_back(work, t);
        for (auto& th : pool) th.join();
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1.0;
    }
}

}  // extern "C"
