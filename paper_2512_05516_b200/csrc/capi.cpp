// C ABI of libsoaforge_b200.so (include/soaforge_b200.h).
//
// Error handling mirrors the reference capi.cpp:14-32: exceptions never cross
// the boundary; ParseError -> SF_PARSE_ERROR, std::invalid_argument ->
// SF_INVALID_ARG, anything else (including CUDA failures) -> SF_ERROR, with
// the message in a thread-local buffer.
#include "../../include/soaforge_b200.h"

#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <memory>
#include <sstream>
#include <cstring>
#include <string>
#include <vector>

#include "commands.hpp"
#include "runtime.hpp"
#include "shard.hpp"
#include "schema.hpp"
#include "view.hpp"

using namespace sfb;

namespace {

thread_local std::string g_err;

sf_status fail(sf_status s, const std::string& m) {
    g_err = m;
    return s;
}

template <typename Fn>
sf_status guarded(Fn&& fn) {
    try {
        return fn();
    } catch (const ParseError& e) {
        return fail(SF_PARSE_ERROR, e.what());
    } catch (const std::invalid_argument& e) {
        return fail(SF_INVALID_ARG, e.what());
    } catch (const std::exception& e) {
        return fail(SF_ERROR, e.what());
    }
}

}  // namespace

struct sf_schema {
    std::shared_ptr<const Schema> s;
    std::string printed;
};

struct sf_config {
    RunConfig run;
    std::string last_text;
};

struct sf_view {
    View v;
};

extern "C" {

const char* sf_version(void) { return "0.1.0"; }
const char* sf_last_error(void) { return g_err.c_str(); }

sf_status sf_layout_for(int t, int* s, int* e, int* m) {
    if (!s || !e || !m) return fail(SF_INVALID_ARG, "null output pointer");
    if (t < 7) return fail(SF_INVALID_ARG, "total_bits " + std::to_string(t) + " below minimum width 7");
    if (t > 64) return fail(SF_INVALID_ARG, "total_bits " + std::to_string(t) + " above maximum width 64");
    const LaneFmt f = fmt_compressed(t);
    *s = 1;
    *e = base_ebits(f.base);
    *m = f.mbits;
    return SF_OK;
}

sf_status sf_quantize(double value, int t, double* out) {
    if (!out) return fail(SF_INVALID_ARG, "null output pointer");
    if (t < 7 || t > 64) return fail(SF_INVALID_ARG, "total_bits " + std::to_string(t) + " outside 7..64");
    const LaneFmt f = fmt_compressed(t);
    *out = decode_lane(encode_lane(value, f), f);
    return SF_OK;
}

sf_status sf_schema_parse(const char* text, sf_schema** out) {
    if (!text || !out) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        auto h = std::make_unique<sf_schema>();
        h->s = std::make_shared<const Schema>(parse_schema_text(text));
        *out = h.release();
        return SF_OK;
    });
}

void sf_schema_destroy(sf_schema* s) { delete s; }

sf_status sf_schema_record_bits(const sf_schema* s, uint64_t* out) {
    if (!s || !out) return fail(SF_INVALID_ARG, "null argument");
    *out = s->s->record_bits;
    return SF_OK;
}

sf_status sf_schema_field_count(const sf_schema* s, int* out) {
    if (!s || !out) return fail(SF_INVALID_ARG, "null argument");
    *out = int(s->s->fields.size());
    return SF_OK;
}

sf_status sf_schema_print(sf_schema* s, const char** out) {
    if (!s || !out) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        s->printed = print_schema_text(*s->s);
        *out = s->printed.c_str();
        return SF_OK;
    });
}

sf_status sf_config_create(sf_config** out) {
    if (!out) return fail(SF_INVALID_ARG, "null argument");
    *out = new sf_config();
    return SF_OK;
}

void sf_config_destroy(sf_config* c) { delete c; }

sf_status sf_config_set_string(sf_config* c, const char* key, const char* value) {
    if (!c || !key || !value) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        config_set_string(c->run, key, value);
        return SF_OK;
    });
}

sf_status sf_config_set_int(sf_config* c, const char* key, int64_t value) {
    if (!c || !key) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        config_set_int(c->run, key, value);
        return SF_OK;
    });
}

sf_status sf_config_set_double(sf_config* c, const char* key, double value) {
    if (!c || !key) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        config_set_double(c->run, key, value);
        return SF_OK;
    });
}

static sf_status run_cmd(sf_config* c, const char** out, std::string (*cmd)(const RunConfig&)) {
    if (!c || !out) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        c->last_text = cmd(c->run);
        write_output(c->run, c->last_text);
        *out = c->last_text.c_str();
        return SF_OK;
    });
}

sf_status sf_run_bench_transform(sf_config* c, const char** out) { return run_cmd(c, out, cmd_bench_transform); }
sf_status sf_run_bench_kernels(sf_config* c, const char** out) { return run_cmd(c, out, cmd_bench_kernels); }
sf_status sf_run_bench_pipeline(sf_config* c, const char** out) { return run_cmd(c, out, cmd_bench_pipeline); }
sf_status sf_run_study_truncation(sf_config* c, const char** out) { return run_cmd(c, out, cmd_study_truncation); }

sf_status sf_run_validate(sf_config* c, const char** out) {
    if (!c || !out) return fail(SF_INVALID_ARG, "null argument");
    int failures = 0;
    const sf_status st = guarded([&] {
        c->last_text = cmd_validate(c->run, failures);
        write_output(c->run, c->last_text);
        *out = c->last_text.c_str();
        return SF_OK;
    });
    if (st != SF_OK) return st;
    return failures == 0 ? SF_OK : fail(SF_CHECK_FAILED, "one or more validation checks failed");
}

// ------------------------------------------------------------------- views
sf_status sf_b200_view_create(const sf_schema* s, const char* access_set, int layout, int precision,
                              const char* exclude_csv, uint64_t count, sf_view** out) {
    if (!s || !out) return fail(SF_INVALID_ARG, "null argument");
    if (layout != SF_LAYOUT_AOS && layout != SF_LAYOUT_SOA) return fail(SF_INVALID_ARG, "unknown layout");
    return guarded([&] {
        auto h = std::make_unique<sf_view>();
        h->v = make_view(s->s, access_set, layout == SF_LAYOUT_AOS ? Layout::AoS : Layout::SoA, precision,
                         split_names(exclude_csv ? exclude_csv : ""), count);
        *out = h.release();
        return SF_OK;
    });
}

void sf_b200_view_destroy(sf_view* v) { delete v; }

sf_status sf_b200_view_bytes(const sf_view* v, uint64_t* n) {
    if (!v || !n) return fail(SF_INVALID_ARG, "null argument");
    *n = v->v.total_bytes();
    return SF_OK;
}

sf_status sf_b200_view_lane(const sf_view* v, const char* field, uint64_t* base, uint64_t* stride, int* width,
                            int* arity) {
    if (!v || !field || !base || !stride || !width || !arity) return fail(SF_INVALID_ARG, "null argument");
    const int p = v->v.pos_of(std::string(field));
    if (p < 0) return fail(SF_INVALID_ARG, std::string("field '") + field + "' is not present in the view");
    *base = v->v.lane_base(p);
    *stride = v->v.lane_stride(p);
    *width = v->v.width(p);
    *arity = v->v.arity(p);
    return SF_OK;
}

sf_status sf_b200_gather(const sf_view* src, const void* sp, const sf_view* dst, void* dp, void* stream) {
    if (!src || !dst || !sp || !dp) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        gather(src->v, sp, dst->v, dp, nullptr, 0.0, 0, static_cast<cudaStream_t>(stream));
        return SF_OK;
    });
}

sf_status sf_b200_gather_kernel(const sf_view* src, const void* sp, const sf_view* dst, void* dp, const char* k,
                                double dt, int math, void* stream) {
    if (!src || !dst || !sp || !dp || !k) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        gather(src->v, sp, dst->v, dp, k, dt, math, static_cast<cudaStream_t>(stream));
        return SF_OK;
    });
}

sf_status sf_b200_convert(const sf_view* src, const void* sp, const sf_view* dst, void* dp, void* stream) {
    if (!src || !dst || !sp || !dp) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        convert(src->v, sp, dst->v, dp, static_cast<cudaStream_t>(stream));
        return SF_OK;
    });
}

sf_status sf_b200_permute(const sf_view* v, const void* src_dev, void* dst_dev, const int32_t* perm, void* stream) {
    if (!v) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        permute(v->v, src_dev, dst_dev, perm, static_cast<cudaStream_t>(stream));
        return SF_OK;
    });
}

sf_status sf_b200_scatter_merge(const sf_view* src, const void* sp, const sf_view* dst, void* dp, const char* k,
                                void* stream) {
    if (!src || !dst || !sp || !dp || !k) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        scatter_merge(src->v, sp, dst->v, dp, k, static_cast<cudaStream_t>(stream));
        return SF_OK;
    });
}

sf_status sf_b200_run_kernel(const sf_view* v, void* p, const char* k, double dt, uint64_t bs, int per_access,
                             int math, void* stream) {
    if (!v || !p || !k) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        run_kernel(v->v, p, k, dt, bs, per_access, math, static_cast<cudaStream_t>(stream));
        return SF_OK;
    });
}

sf_status sf_b200_density_cells(const void* x, const void* m, const void* h, int prec, uint64_t n,
                                const int32_t* perm, const int32_t* cell_start, const float* lo, float cell, int nx,
                                int ny, int nz, int reach, uint64_t n_home, float* rho, void* stream) {
    if ((n && (!x || !m || !h || !rho)) || !cell_start || !lo) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        density_cells(x, m, h, prec, n, perm, cell_start, lo, cell, nx, ny, nz, reach, n_home, rho,
                      static_cast<cudaStream_t>(stream));
        return SF_OK;
    });
}

sf_status sf_b200_force_cells(const void* x, const void* v, const void* m, const void* h, const void* rho,
                              const void* P, int prec, uint64_t n, const int32_t* perm, const int32_t* cell_start,
                              const float* lo, float cell, int nx, int ny, int nz, int reach, uint64_t n_home,
                              float* a_out, float* du_out, void* stream) {
    if ((n && (!x || !v || !m || !h || !rho || !P || !a_out || !du_out)) || !cell_start || !lo)
        return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        force_cells(x, v, m, h, rho, P, prec, n, perm, cell_start, lo, cell, nx, ny, nz, reach, n_home, a_out,
                    du_out, static_cast<cudaStream_t>(stream));
        return SF_OK;
    });
}

static_assert(sizeof(sf_cell_block) == sizeof(CellBlockDesc), "sf_cell_block layout");

sf_status sf_b200_cells_pack(const void* x, const void* m, const void* h, int prec, uint64_t n, const int32_t* perm,
                             void* pos_out, float* h_out, uint32_t* hmax_out, void* stream) {
    if ((n && (!x || !m || !h || !pos_out || !h_out)) || !hmax_out) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        cells_pack(x, m, h, prec, n, perm, pos_out, h_out, hmax_out, static_cast<cudaStream_t>(stream));
        return SF_OK;
    });
}

sf_status sf_b200_density_cells_blocks(const sf_cell_block* blocks, int nblocks, uint64_t n, const int32_t* perm,
                                       uint64_t n_home, const float* lo_yz, float cell, int nx_global, int ny, int nz,
                                       int reach, float* rho_out, void* stream) {
    if (!blocks || !lo_yz || (n && !rho_out)) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        std::vector<CellBlockDesc> d(size_t(std::max(nblocks, 0)));
        for (int g = 0; g < nblocks; ++g)
            d[g] = CellBlockDesc{blocks[g].pos,    blocks[g].h,        blocks[g].cell_start, blocks[g].hmax,
                                 blocks[g].x0,     blocks[g].nx,       blocks[g].x_origin,   0};
        density_cells_blocks(d.data(), nblocks, n, perm, n_home, lo_yz, cell, nx_global, ny, nz, reach, rho_out,
                             static_cast<cudaStream_t>(stream));
        return SF_OK;
    });
}

static_assert(sizeof(sf_force_block) == sizeof(ForceBlockDesc), "sf_force_block layout");

sf_status sf_b200_force_pack(const void* v, const void* rho, const void* P, int prec, uint64_t n, const int32_t* perm,
                             void* vel_out, void* stream) {
    if (n && (!v || !rho || !P || !vel_out)) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        force_pack(v, rho, P, prec, n, perm, vel_out, static_cast<cudaStream_t>(stream));
        return SF_OK;
    });
}

sf_status sf_b200_force_cells_blocks(const sf_force_block* blocks, int nblocks, uint64_t n, const int32_t* perm,
                                     uint64_t n_home, const float* lo_yz, float cell, int nx_global, int ny, int nz,
                                     int reach, float* a_out, float* du_out, void* stream) {
    if (!blocks || !lo_yz || (n && (!a_out || !du_out))) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        std::vector<ForceBlockDesc> d(size_t(std::max(nblocks, 0)));
        for (int g = 0; g < nblocks; ++g)
            d[g] = ForceBlockDesc{blocks[g].pos,  blocks[g].vel, blocks[g].h,        blocks[g].cell_start,
                                  blocks[g].hmax, blocks[g].x0,  blocks[g].nx,       blocks[g].x_origin,
                                  0};
        force_cells_blocks(d.data(), nblocks, n, perm, n_home, lo_yz, cell, nx_global, ny, nz, reach, a_out, du_out,
                           static_cast<cudaStream_t>(stream));
        return SF_OK;
    });
}

uint64_t sf_b200_window_mask_bytes(uint64_t n, int reach) {
    return reach >= 1 && reach <= 2 ? 4 * window_mask_words(n, reach) : 0;
}

sf_status sf_b200_density_cells_blocks_masked(const sf_cell_block* blocks, int nblocks, uint64_t n,
                                              const int32_t* perm, uint64_t n_home, const float* lo_yz, float cell,
                                              int nx_global, int ny, int nz, int reach, float* rho_out, void* masks,
                                              void* stream) {
    if (!blocks || !lo_yz || (n && (!rho_out || !masks))) return fail(SF_INVALID_ARG, "null argument");
    if (reach < 1 || reach > 2) return fail(SF_INVALID_ARG, "window masks need reach 1 or 2");
    if (reinterpret_cast<uintptr_t>(masks) & 7) return fail(SF_INVALID_ARG, "masks must be 8-byte aligned");
    return guarded([&] {
        std::vector<CellBlockDesc> d(size_t(std::max(nblocks, 0)));
        for (int g = 0; g < nblocks; ++g)
            d[g] = CellBlockDesc{blocks[g].pos,    blocks[g].h,        blocks[g].cell_start, blocks[g].hmax,
                                 blocks[g].x0,     blocks[g].nx,       blocks[g].x_origin,   0};
        density_cells_blocks(d.data(), nblocks, n, perm, n_home, lo_yz, cell, nx_global, ny, nz, reach, rho_out,
                             static_cast<cudaStream_t>(stream), static_cast<int32_t*>(masks));
        return SF_OK;
    });
}

sf_status sf_b200_force_cells_blocks_masked(const sf_force_block* blocks, int nblocks, uint64_t n,
                                            const int32_t* perm, uint64_t n_home, const float* lo_yz, float cell,
                                            int nx_global, int ny, int nz, int reach, float* a_out, float* du_out,
                                            const void* masks, void* stream) {
    if (!blocks || !lo_yz || (n && (!a_out || !du_out || !masks))) return fail(SF_INVALID_ARG, "null argument");
    if (reach < 1 || reach > 2) return fail(SF_INVALID_ARG, "window masks need reach 1 or 2");
    if (reinterpret_cast<uintptr_t>(masks) & 7) return fail(SF_INVALID_ARG, "masks must be 8-byte aligned");
    return guarded([&] {
        std::vector<ForceBlockDesc> d(size_t(std::max(nblocks, 0)));
        for (int g = 0; g < nblocks; ++g)
            d[g] = ForceBlockDesc{blocks[g].pos,  blocks[g].vel, blocks[g].h,        blocks[g].cell_start,
                                  blocks[g].hmax, blocks[g].x0,  blocks[g].nx,       blocks[g].x_origin,
                                  0};
        force_cells_blocks(d.data(), nblocks, n, perm, n_home, lo_yz, cell, nx_global, ny, nz, reach, a_out, du_out,
                           static_cast<cudaStream_t>(stream), static_cast<const int32_t*>(masks));
        return SF_OK;
    });
}

sf_status sf_b200_dev_alloc(uint64_t bytes, void** out) {
    if (!out) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        require_device();
        *out = nullptr;
        check_cuda(cudaMalloc(out, bytes ? bytes : 1), "cudaMalloc");
        return SF_OK;
    });
}

sf_status sf_b200_dev_free(void* p) {
    return guarded([&] {
        if (p) check_cuda(cudaFree(p), "cudaFree");
        return SF_OK;
    });
}

sf_status sf_b200_ipc_handle(const void* p, uint8_t* handle) {
    if (!p || !handle) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        require_device();
        cudaIpcMemHandle_t hd;
        check_cuda(cudaIpcGetMemHandle(&hd, const_cast<void*>(p)), "cudaIpcGetMemHandle");
        static_assert(sizeof(hd) == SF_IPC_HANDLE_BYTES, "IPC handle size");
        memcpy(handle, &hd, sizeof(hd));
        return SF_OK;
    });
}

sf_status sf_b200_ipc_open(const uint8_t* handle, void** out) {
    if (!handle || !out) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        require_device();
        cudaIpcMemHandle_t hd;
        memcpy(&hd, handle, sizeof(hd));
        check_cuda(cudaIpcOpenMemHandle(out, hd, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
        return SF_OK;
    });
}

sf_status sf_b200_ipc_close(void* p) {
    if (!p) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        check_cuda(cudaIpcCloseMemHandle(p), "cudaIpcCloseMemHandle");
        return SF_OK;
    });
}

// ---------------------------------------------------------------- sharded step
struct sf_shard {
    sfb::Shard* s;
};

sf_status sf_b200_shard_create(int rank, int world, int cells_per_side, double cell, int refine, uint64_t capacity,
                               sf_shard** out) {
    if (!out) return fail(SF_INVALID_ARG, "null argument");
    *out = nullptr;
    return guarded([&] {
        *out = new sf_shard{shard_create(rank, world, cells_per_side, cell, refine, capacity)};
        return SF_OK;
    });
}

void sf_b200_shard_destroy(sf_shard* s) {
    if (!s) return;
    shard_destroy(s->s);
    delete s;
}

sf_status sf_b200_shard_handle(sf_shard* s, uint8_t* handle) {
    if (!s || !handle) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        shard_handle(s->s, handle);
        return SF_OK;
    });
}

sf_status sf_b200_shard_connect(sf_shard* s, const uint8_t* handles) {
    if (!s || !handles) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        shard_connect(s->s, handles);
        return SF_OK;
    });
}

sf_status sf_b200_shard_load(sf_shard* s, const void* soa_dev, uint64_t count, void* stream) {
    if (!s || (count && !soa_dev)) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        shard_load(s->s, soa_dev, count, static_cast<cudaStream_t>(stream));
        return SF_OK;
    });
}

sf_status sf_b200_shard_field(sf_shard* s, const char* field, void** dev, uint64_t* count, int* bytes_per_particle) {
    if (!s || !field || !dev) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        *dev = shard_field(s->s, field, bytes_per_particle);
        if (count) *count = shard_count(s->s);
        return SF_OK;
    });
}

sf_status sf_b200_shard_step(sf_shard* s, const char* kernels, double dt, void* stream, double* metrics) {
    if (!s || !kernels) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        shard_step(s->s, split_names(kernels), dt, static_cast<cudaStream_t>(stream), metrics);
        return SF_OK;
    });
}

uint64_t sf_b200_bin_scratch_bytes(uint64_t n, int nx, int ny, int nz) { return bin_scratch_bytes(n, nx, ny, nz); }

sf_status sf_b200_bin_particles(const float* x, uint64_t n, const float* lo, float cell, int nx, int ny, int nz,
                                int32_t* cell_start, int32_t* perm, void* scratch, uint64_t scratch_bytes,
                                void* stream) {
    // per-particle arrays may be NULL when there are no particles
    if ((n && (!x || !perm)) || !lo || !cell_start || !scratch) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        bin_particles(x, n, lo, cell, nx, ny, nz, cell_start, perm, scratch, scratch_bytes,
                      static_cast<cudaStream_t>(stream));
        return SF_OK;
    });
}

sf_status sf_b200_run_host(const sf_view* src, void* host, const sf_view* dst, const char* kernels, double dt,
                           int math, int mode, uint64_t chunk, void* host_soa, double* metrics) {
    if (!src || !host || !dst || !kernels || !metrics) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        run_host(src->v, host, dst->v, kernels, dt, math, mode, chunk, host_soa, metrics);
        return SF_OK;
    });
}

sf_status sf_b200_host_alloc(uint64_t bytes, int mode, void** out) {
    if (!out) return fail(SF_INVALID_ARG, "null argument");
    return guarded([&] {
        require_device();
        if (mode == SF_MODE_STREAMED) check_cuda(cudaHostAlloc(out, bytes, cudaHostAllocDefault), "cudaHostAlloc");
        else if (mode == SF_MODE_MANAGED) check_cuda(cudaMallocManaged(out, bytes, cudaMemAttachGlobal), "cudaMallocManaged");
        else throw std::invalid_argument("unknown host memory mode");
        return SF_OK;
    });
}

sf_status sf_b200_host_free(void* p, int mode) {
    return guarded([&] {
        if (!p) return SF_OK;
        check_cuda(mode == SF_MODE_STREAMED ? cudaFreeHost(p) : cudaFree(p), "free");
        return SF_OK;
    });
}

uint64_t sf_b200_launch_count(void) { return launch_count(); }

}  // extern "C"
