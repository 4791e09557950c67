#ifndef SOAFORGE_B200_H
#define SOAFORGE_B200_H

/* libsoaforge_b200.so — B200 (sm_100a) drop-in for the reference's
 * AoS->SoA + reduced-precision SPH hot path.
 *
 * Part 1 re-exports the reference C ABI (proj/include/soaforge/soaforge.h:
 * 22-82) with the same names, argument meaning, status codes and
 * thread-local last-error convention, so test_capi-style callers link
 * unchanged.  Part 2 adds the hot-path entry points; every
 * one of them runs on the GPU through hand-written sm_100a kernels — there is
 * no CPU fallback, and a missing device is an SF_ERROR.
 *
 * Conventions (as in the reference): every entry returns sf_status; on
 * failure sf_last_error() holds a thread-local message.  Opaque handles are
 * freed by the matching *_destroy.  Device pointers are caller-owned (the
 * reference's *_into operators, layout_ops.hpp:104-128) and must be 16-byte
 * aligned; `stream` is a cudaStream_t (NULL = legacy default stream).      */

#include <stddef.h>
#include <stdint.h>

#define SF_API __attribute__((visibility("default")))

#ifdef __cplusplus
extern "C" {
#endif

typedef enum sf_status {
    SF_OK = 0,
    SF_ERROR = 1,
    SF_INVALID_ARG = 2,
    SF_PARSE_ERROR = 3,
    SF_CHECK_FAILED = 4
} sf_status;

/* ===================== Part 1: the reference ABI ========================= */
/* replaces soaforge.h:33-34 */
SF_API const char* sf_version(void);
SF_API const char* sf_last_error(void);
/* replaces soaforge.h:39-43 (fpcodec::layout_for / quantize) */
SF_API sf_status sf_layout_for(int total_bits, int* sign_bits, int* exponent_bits, int* mantissa_bits);
SF_API sf_status sf_quantize(double value, int total_bits, double* out);

/* replaces soaforge.h:47-55 (schema DSL, schema.hpp:12-21) */
typedef struct sf_schema sf_schema;
SF_API sf_status sf_schema_parse(const char* text, sf_schema** out);
SF_API void sf_schema_destroy(sf_schema* schema);
SF_API sf_status sf_schema_record_bits(const sf_schema* schema, uint64_t* out);
SF_API sf_status sf_schema_field_count(const sf_schema* schema, int* out);
SF_API sf_status sf_schema_print(sf_schema* schema, const char** out);

/* replaces soaforge.h:59-71 (run configuration, same keys and validation) */
typedef struct sf_config sf_config;
SF_API sf_status sf_config_create(sf_config** out);
SF_API void sf_config_destroy(sf_config* config);
SF_API sf_status sf_config_set_string(sf_config* config, const char* key, const char* value);
SF_API sf_status sf_config_set_int(sf_config* config, const char* key, int64_t value);
SF_API sf_status sf_config_set_double(sf_config* config, const char* key, double value);

/* replaces soaforge.h:77-82 — the commands run their conversions and
 * kernels on the GPU; CSV columns as in bench.cpp:219/275/323-325. */
SF_API sf_status sf_run_bench_transform(sf_config* config, const char** out_text);
SF_API sf_status sf_run_bench_kernels(sf_config* config, const char** out_text);
SF_API sf_status sf_run_bench_pipeline(sf_config* config, const char** out_text);
SF_API sf_status sf_run_study_truncation(sf_config* config, const char** out_text);
SF_API sf_status sf_run_validate(sf_config* config, const char** out_text);

/* ===================== Part 2: B200 hot path ============================= */

/* A view describes one packed particle buffer (the reference PackedBuffer,
 * layout_ops.hpp:76-98): schema, record count, layout, field subset (an
 * access set's reads ∪ writes, or all fields) and per-lane storage format. */
typedef struct sf_view sf_view;

enum { SF_LAYOUT_AOS = 0, SF_LAYOUT_SOA = 1 };
/* precision codes */
enum {
    SF_PREC_STORED = 0,   /* PrecisionTag::Compressed: declared storage widths     */
    SF_PREC_NATIVE = 1,   /* PrecisionTag::Native: unpacked to IEEE widths (U)     */
    /* 7..64: every non-excluded float lane narrowed to T bits (RNE, then
     * mantissa truncation), held in its enclosing IEEE width — the
     * store_state(T) narrowing of sph.cpp:385-412 followed by U            */
    SF_PREC_BF16 = 100,   /* non-excluded float lanes as bfloat16 (RNE)            */
    SF_PREC_PACKED = 1000 /* 1000+T: like T but kept bit-packed at T bits          */
};
enum { SF_MATH_FP64_EXACT = 0, SF_MATH_FP32 = 1 };

/* access_set: a `kernel` name declared in the schema text, or NULL/"" for
 * the full field set (narrow_into, layout_ops.cpp:86-112).
 * exclude_csv: float fields kept at their stored precision (e.g. "x"). */
SF_API sf_status sf_b200_view_create(const sf_schema* schema, const char* access_set, int layout,
                                     int precision, const char* exclude_csv, uint64_t count,
                                     sf_view** out);
SF_API void sf_b200_view_destroy(sf_view* view);
SF_API sf_status sf_b200_view_bytes(const sf_view* view, uint64_t* nbytes);
/* Lane geometry of one field (bits): lane l of record r sits at
 * base + r*stride + l*width (layout_ops.cpp:25-39). */
SF_API sf_status sf_b200_view_lane(const sf_view* view, const char* field, uint64_t* base_bits,
                                   uint64_t* stride_bits, int* width_bits, int* arity);

/* Fused U∘N∘C (+ narrowing): AoS `src` -> SoA `dst` for every field of dst.
 * Replaces narrow_into + unpack_into + aos_to_soa_into (layout_ops.cpp:
 * 86-112, 164-191, 150-162) and the store_state narrowing.  Bit-exact. */
SF_API sf_status sf_b200_gather(const sf_view* src, const void* src_dev, const sf_view* dst,
                                void* dst_dev, void* stream);
/* Gather fused with a linear kernel (kick | drift, sph.cpp:247-264): the
 * kernel consumes the converted lanes straight from the loads and writes the
 * updated SoA; no separate conversion pass. */
SF_API sf_status sf_b200_gather_kernel(const sf_view* src, const void* src_dev, const sf_view* dst,
                                       void* dst_dev, const char* kernel, double dt, int math,
                                       void* stream);
/* Generic lane conversion of every dst field between any two views
 * (AoS<->SoA, any precisions). */
SF_API sf_status sf_b200_convert(const sf_view* src, const void* src_dev, const sf_view* dst,
                                 void* dst_dev, void* stream);
/* Reorder: dst record k = src record perm[k] for every lane of the view
 * (AoS: whole records; SoA: every stream), e.g. a particle population into
 * the cell order of sf_b200_bin_particles' perm.  Byte-aligned views; src
 * and dst must not alias. */
SF_API sf_status sf_b200_permute(const sf_view* view, const void* src_dev, void* dst_dev, const int32_t* perm,
                                 void* stream);
/* Fused C^T∘U^T∘N^T: write only `kernel`'s write set from src into dst
 * (widen_merge, layout_ops.cpp:120-146); read-only lanes stay bit-exact. */
SF_API sf_status sf_b200_scatter_merge(const sf_view* src, const void* src_dev, const sf_view* dst,
                                       void* dst_dev, const char* kernel, void* stream);
/* run_kernel_chunked (sph.cpp:286-308) on a device buffer in place:
 * kick | drift | density | force.  density uses contiguous `buffer_size` neighbour
 * buffers with reference semantics; per_access selects Writeback::PerAccess.
 * A comma-separated list ("kick,drift") runs the kernels in order, with the
 * same result as one call per kernel; on a byte-aligned AoS of plain IEEE
 * lanes the whole list is one pass over the records (k_update_rec_seq). */
SF_API sf_status sf_b200_run_kernel(const sf_view* view, void* dev, const char* kernel, double dt,
                                    uint64_t buffer_size, int per_access, int math, void* stream);

/* Cell-linked density (new algorithm).  x: 3*n, m, h: n lanes
 * in `prec` (SF_PREC_NATIVE -> fp32 streams, 16 -> fp16, SF_PREC_BF16 ->
 * bf16), in particle order; perm[n] / cell_start[ncell+1] from
 * sf_b200_bin_particles over the same grid (lo[3] host floats, cell side,
 * nx*ny*nz cells, x-major).  reach = neighbour cells per side searched
 * (1 when cell >= 2h, 2 when cell >= h).  Only the first n_home particles
 * (particle order) are computed; particles [n_home, n) are neighbours only
 * (ghosts received from other ranks, multi-GPU).  rho_out[i] (fp32,
 * particle order) is written for i < n_home. */
SF_API sf_status sf_b200_density_cells(const void* x, const void* m, const void* h, int prec,
                                       uint64_t n, const int32_t* perm, const int32_t* cell_start,
                                       const float* lo, float cell, int nx, int ny, int nz, int reach,
                                       uint64_t n_home, float* rho_out, void* stream);
/* Multi-block cell-linked density: the homes' own block plus up to two
 * neighbouring slabs' blocks read in place (multi-GPU: peer pointers over
 * NVLink from sf_b200_ipc_open — the halo is never copied).  Every block is
 * one x-slab [x0, x0 + nx) of a global grid (cell side, nx_global x-layers,
 * ny, nz; y/z origin lo_yz[2]) with its own cell list (sf_b200_bin_particles
 * over its layers with lo = {x_origin, lo_yz[0], lo_yz[1]}) and packed
 * particles (sf_b200_cells_pack). */
typedef struct sf_cell_block {
    const void* pos;            /* float4 (x, y, z, m) per particle, cell-sorted */
    const float* h;             /* cell-sorted smoothing lengths */
    const int32_t* cell_start;  /* nx*ny*nz + 1 entries */
    const uint32_t* hmax;       /* h range, 2 words: [0] largest h (float bits), [1] ~bits of the
                                   smallest h (0 = unknown); equal ends select the uniform-h loop,
                                   which reads only pos */
    int32_t x0, nx;             /* global x-layers held by the block */
    float x_origin;             /* the lo[0] its binning used (layer x0 starts there) */
    int32_t reserved;           /* 0 */
} sf_cell_block;
#define SF_IPC_HANDLE_BYTES 64
/* Packs x (3n), m, h (n) in `prec` through perm (sorted position -> particle)
 * into caller-owned pos_out (float4 (x, y, z, m), 16*n bytes, 16-B aligned),
 * h_out (4*n) and hmax_out (two words: the h range of sf_cell_block.hmax). */
SF_API sf_status sf_b200_cells_pack(const void* x, const void* m, const void* h, int prec, uint64_t n,
                                    const int32_t* perm, void* pos_out, float* h_out,
                                    uint32_t* hmax_out, void* stream);
/* rho of the first n_home particles (particle order) of blocks[0] (n particles,
 * perm from its binning); candidates from every block. */
SF_API sf_status sf_b200_density_cells_blocks(const sf_cell_block* blocks, int nblocks, uint64_t n,
                                              const int32_t* perm, uint64_t n_home, const float* lo_yz,
                                              float cell, int nx_global, int ny, int nz, int reach,
                                              float* rho_out, void* stream);
/* The force over the same blocks: a density block plus the same particles'
 * (v, P/rho^2) as float4, packed in its cell-sorted order by
 * sf_b200_force_pack (rho == 0 -> SF_ERROR domain error; synchronizes). */
typedef struct sf_force_block {
    const void* pos;            /* the density block's float4 (x, y, z, m) */
    const void* vel;            /* float4 (vx, vy, vz, P/rho^2) */
    const float* h;             /* the density block's smoothing lengths */
    const int32_t* cell_start;
    const uint32_t* hmax;       /* the density block's h range (2 words) */
    int32_t x0, nx;
    float x_origin;
    int32_t reserved;
} sf_force_block;
SF_API sf_status sf_b200_force_pack(const void* v, const void* rho, const void* P, int prec, uint64_t n,
                                    const int32_t* perm, void* vel_out, void* stream);
SF_API sf_status sf_b200_force_cells_blocks(const sf_force_block* blocks, int nblocks, uint64_t n,
                                            const int32_t* perm, uint64_t n_home, const float* lo_yz,
                                            float cell, int nx_global, int ny, int nz, int reach,
                                            float* a_out, float* du_out, void* stream);
/* One SPH step's density then force over the same blocks, sharing the pair
 * search: the density also writes `masks` (caller-owned device memory of
 * sf_b200_window_mask_bytes(n, reach), 8-B aligned) — for every home and
 * neighbour-column window, the window's first candidate and a bit per
 * in-support candidate — and the force then evaluates exactly those pairs
 * (no culling, no out-of-support candidates; a home with a window of more
 * than 32 candidates falls back to the window sweep).  The masks are valid
 * for the force of the same blocks, perm and grid only.  reach <= 2. */
SF_API uint64_t sf_b200_window_mask_bytes(uint64_t n, int reach);
SF_API sf_status sf_b200_density_cells_blocks_masked(const sf_cell_block* blocks, int nblocks, uint64_t n,
                                                     const int32_t* perm, uint64_t n_home, const float* lo_yz,
                                                     float cell, int nx_global, int ny, int nz, int reach,
                                                     float* rho_out, void* masks, void* stream);
SF_API sf_status sf_b200_force_cells_blocks_masked(const sf_force_block* blocks, int nblocks, uint64_t n,
                                                   const int32_t* perm, uint64_t n_home, const float* lo_yz,
                                                   float cell, int nx_global, int ny, int nz, int reach,
                                                   float* a_out, float* du_out, const void* masks, void* stream);
/* Device memory that another process can map (cudaMalloc base), and CUDA IPC
 * handles for it (same node; NVLink/NVSwitch peers or the same device). */
SF_API sf_status sf_b200_dev_alloc(uint64_t bytes, void** ptr);
SF_API sf_status sf_b200_dev_free(void* ptr);
SF_API sf_status sf_b200_ipc_handle(const void* dev_ptr, uint8_t handle[SF_IPC_HANDLE_BYTES]);
SF_API sf_status sf_b200_ipc_open(const uint8_t handle[SF_IPC_HANDLE_BYTES], void** dev_ptr);
SF_API sf_status sf_b200_ipc_close(void* dev_ptr);
/* Cell-linked force (the reference's force_kernel, sph.cpp:201-245, over
 * cell neighbours instead of 64-particle buffers): x, v: 3*n lanes; m, h,
 * rho, P: n lanes, all in `prec` and particle order; grid, perm and
 * cell_start as for sf_b200_density_cells.  Writes a_out[3*i+l] and
 * du_out[i] (fp32, particle order) for i < n_home (the rest are ghosts).  Any
 * rho == 0 returns SF_ERROR "force: degenerate state, rho == 0" (the
 * reference's std::domain_error); synchronizes `stream` to check it. */
SF_API sf_status sf_b200_force_cells(const void* x, const void* v, const void* m, const void* h,
                                     const void* rho, const void* P, int prec, uint64_t n,
                                     const int32_t* perm, const int32_t* cell_start, const float* lo,
                                     float cell, int nx, int ny, int nz, int reach, uint64_t n_home,
                                     float* a_out, float* du_out, void* stream);
/* One rank of the cell-sharded timestep (BASELINE C5; replaces the
 * reference's threaded run_kernel_chunked, sph.cpp:286-308, for a
 * population decomposed over the GPUs of one node).  The rank owns the
 * x-slab of cell layers [rank*nc/world, (rank+1)*nc/world) of an nc^3 grid
 * of cells of side `cell` (>= 2 h_max) over the unit box, binned `refine`
 * times finer (reach = refine).  Its particles live on the device as an SoA
 * of the default schema at T=32 (x included), at a fixed `capacity`.
 *
 * Setup (host, once): sf_b200_shard_create on every rank; exchange the
 * 64-byte sf_b200_shard_handle of every rank with any transport (MPI,
 * torch.distributed, files) and pass all of them, rank order, to
 * sf_b200_shard_connect; sf_b200_shard_load the rank's particles (a
 * reference SoA buffer of `count` particles, T=32, every field).
 *
 * sf_b200_shard_step runs `kernels` (a list of density, force, kick, drift,
 * the reference's timestep order "density,force,kick,drift") and then
 * migrates the particles whose x-layer left the slab to the +-1 neighbour.
 * The halo is read in place: density and force take the neighbours' packed
 * cell blocks through CUDA IPC peer pointers (NVLink).  Ranks order each
 * other on the device (release/acquire epoch words in peer memory), so a
 * step has no host barrier; with world > 1 it synchronises `stream` once to
 * read the new particle count.  rho == 0 in the force -> SF_ERROR (domain
 * error); an outbox / capacity overflow -> SF_ERROR.
 * metrics (optional, 9 doubles): particles after the step, step ms, ms of
 * each listed kernel (4 slots, list order), migration ms, particles sent,
 * step number. */
typedef struct sf_shard sf_shard;
SF_API sf_status sf_b200_shard_create(int rank, int world, int cells_per_side, double cell, int refine,
                                      uint64_t capacity, sf_shard** out);
SF_API void sf_b200_shard_destroy(sf_shard* shard);
SF_API sf_status sf_b200_shard_handle(sf_shard* shard, uint8_t handle[SF_IPC_HANDLE_BYTES]);
SF_API sf_status sf_b200_shard_connect(sf_shard* shard, const uint8_t* handles /* world x 64 bytes */);
SF_API sf_status sf_b200_shard_load(sf_shard* shard, const void* soa_dev, uint64_t count, void* stream);
/* Device pointer of one field's stream of the current state (binary32 lanes,
 * int64 for id; valid until the next step), the particle count and the
 * field's bytes per particle. */
SF_API sf_status sf_b200_shard_field(sf_shard* shard, const char* field, void** dev, uint64_t* count,
                                     int* bytes_per_particle);
SF_API sf_status sf_b200_shard_step(sf_shard* shard, const char* kernels, double dt, void* stream,
                                    double* metrics);

/* Counting sort of particles into cells (x-major cell id), stable in
 * particle index: writes perm[n] (sorted position -> original index) and
 * cell_start[ncell+1].  scratch must hold sf_b200_bin_scratch_bytes(). */
SF_API sf_status sf_b200_bin_particles(const float* x, uint64_t n, const float* lo, float cell,
                                       int nx, int ny, int nz, int32_t* cell_start, int32_t* perm,
                                       void* scratch, uint64_t scratch_bytes, void* stream);
SF_API uint64_t sf_b200_bin_scratch_bytes(uint64_t n, int nx, int ny, int nz);

/* Host-resident orchestration (the paper's in-place vs streaming question
 * re-posed for PCIe; pipelines.cpp:231-296).  `host_aos` holds `count`
 * records of `src` (full field set, AoS).  One step = gather + `kernels`
 * (comma list of kick,drift) in the dst view's precision + scatter-back of
 * every write set into the AoS, for every record.
 *   mode 0 STREAMED: pinned host memory, zero copy: the gather reads only the
 *                    SoA view's lanes of the host records over PCIe and the
 *                    scatter-back stores only the write set's lanes into them
 *                    (the reference's narrowed streaming transfers);
 *   mode 1 MANAGED:  host_aos is cudaMallocManaged; prefetch to the GPU, kernels
 *                    on the migrated pages, prefetch back (no placement hints);
 *   mode 2 INPLACE:  pinned host memory, whole records each way (the
 *                    reference's in-place round trip).
 *   mode 3 MANAGED_MAPPED: managed memory kept on the host and never
 *                    migrated; the kernels read/write its pages over PCIe.
 * All modes pipeline H2D k+1 ∥ compute k ∥ D2H k-1 over 3 streams.
 * host_soa (optional): when non-NULL the SoA result (dst view, all
 * records) is copied to this host buffer instead of scattering back into
 * the AoS — the end-to-end form of the fused gather+kernel path.
 * metrics[0..4] = {seconds, h2d_bytes, d2h_bytes, chunks, kernel_launches}. */
enum { SF_MODE_STREAMED = 0, SF_MODE_MANAGED = 1, SF_MODE_INPLACE = 2, SF_MODE_MANAGED_MAPPED = 3 };
SF_API sf_status sf_b200_run_host(const sf_view* src, void* host_aos, const sf_view* dst,
                                  const char* kernels, double dt, int math, int mode,
                                  uint64_t chunk_records, void* host_soa, double* metrics);

/* Host buffers for sf_b200_run_host: mode 0 pinned (cudaHostAlloc),
 * mode 1 managed (cudaMallocManaged). */
SF_API sf_status sf_b200_host_alloc(uint64_t bytes, int mode, void** out);
SF_API sf_status sf_b200_host_free(void* p, int mode);

/* Number of sm_100a kernels this library has launched (process-wide). */
SF_API uint64_t sf_b200_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif
