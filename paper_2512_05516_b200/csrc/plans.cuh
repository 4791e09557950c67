// POD launch plans shared between the host planner (view.cpp) and the
// kernels (kernels.cu).  Passed by value as __grid_constant__ parameters.
#pragma once
#include <cstdint>

#include "codec.cuh"

namespace sfb {

enum class Layout : uint8_t { AoS = 0, SoA = 1 };

// Bit geometry of one field's lanes in a buffer: lane l of record r sits at
// base + r*stride + l*fmt.width bits.
struct Lanes {
    uint64_t base = 0, stride = 0;
    LaneFmt fmt{};
    uint8_t arity = 1;
};

enum Op : uint8_t {
    OP_COPY = 0,         // dst = convert(src)
    OP_AXPY = 1,         // dst = Q(Q(x) + Q(y) * dt)          (drift x; kick v)
    OP_AXPY_CLAMP0 = 2,  // dst = Q(max0(Q(x) + Q(y) * dt))    (kick u, sph.cpp:254)
};

enum Math : uint8_t {
    MATH_FP64_EXACT = 0,  // binary64, separately rounded mul/add: bit-exact vs reference
    MATH_FP32 = 1,        // binary32 arithmetic, within 1 ulp of the storage format
};

constexpr int kMaxStreams = 16;

// ---- generic lane-by-lane conversion / in-place update ---------------------
struct CStream {
    Lanes src, dst, aux;  // aux: operand y for the AXPY ops (read from src buffer)
    LaneFmt aux_q;        // y is quantized through this format first
    uint8_t op = OP_COPY;
};

struct ConvertPlan {
    uint64_t count = 0;
    uint32_t n = 0;
    uint8_t dst_byte_aligned = 1;  // plain stores; else bit-level atomics
    uint8_t math = MATH_FP64_EXACT;
    double dt = 0;
    CStream s[kMaxStreams];
};
using KernelPlan = ConvertPlan;

// ---- tiled AoS -> SoA gather (TMA bulk-staged record tiles) ----------------
enum Proc : uint8_t { PROC_GENERIC = 0, PROC_XV_F16 = 1, PROC_XV_BF16 = 2, PROC_XV_F32 = 3 };

struct GStream {
    uint32_t src_off = 0;   // bit offset of lane 0 inside a source record
    uint32_t aux_off = 0;   // operand field, same record
    uint64_t dst_base = 0;  // byte offset of the destination SoA stream
    LaneFmt src{}, dst{}, aux_src{}, aux_dst{};
    uint8_t arity = 1, op = OP_COPY;
    // compile-time-specialised IEEE path (kernels.cu gather_fast_kind);
    // 0 = generic bit-level path
    uint8_t fast = 0;
    // typed direct-load COPY kind of k_gather_multi (set at launch); 0 = none
    uint8_t mkind = 0;
};

struct GatherPlan {
    uint64_t count = 0;
    uint32_t record_bits = 0;
    uint32_t n = 0;
    uint32_t tile_recs = 0;   // per-warp tile: 32*R records, 16-B aligned start
    uint32_t tile_bytes = 0;  // tile_recs * record_bits / 8
    uint32_t out_bytes = 0;   // per-warp SoA staging (largest stream slice)
    uint8_t proc = 0;         // per-tile policy (PROC_*), chosen by view.cpp proc_kind
    uint8_t stages = 4;       // TMA ring depth per warp (set at launch)
    uint8_t math = MATH_FP64_EXACT;
    double dt = 0;
    GStream s[kMaxStreams];
};

// ---- in-place kick/drift on AoS records, all ops in one pass -----------------
struct RecOps {
    uint32_t xoff[2], yoff[2];  // byte offsets of the written field and its operand
    uint8_t arity[2], op[2];
    int n;
};

// ---- kernels (kick | drift | kick,drift ...) in place on AoS records ---------
// Ops run in order per record on the CTA's shared-memory copy of its records.
constexpr int kMaxSeq = 4;
constexpr uint32_t kRecTileMaxStride = 384;  // at most 256 records of at most 384 B per CTA (96 KB)
struct RecSeq {
    uint32_t xoff[kMaxSeq], yoff[kMaxSeq];
    uint8_t kind[kMaxSeq];  // (x base * 4 + y base) * 2 + (arity == 3)
    uint8_t op[kMaxSeq];
    int n;
};

// ---- record permutation (dst record k = src record perm[k]) -----------------
struct PermutePlan {
    uint64_t count = 0;
    int n = 0;                     // element streams (AoS: 1, the whole record)
    uint64_t base[kMaxStreams];    // bytes
    uint32_t eb[kMaxStreams];      // element bytes per record
    uint8_t unit[kMaxStreams];     // 8 / 4 / 2 / 1: widest aligned copy unit
};

// ---- SPH density over 64-particle neighbour buffers (sph.cpp:176-199) -------
struct DensityPlan {
    Lanes x, m, h, rho;
    uint64_t count = 0;
    uint32_t bs = 64;
    uint8_t per_access = 0;
};

// ---- SPH force over 64-particle neighbour buffers (sph.cpp:201-245) ---------
struct ForcePlan {
    Lanes x, v, m, h, rho, P, a, du;
    uint64_t count = 0;
    uint32_t bs = 64;
    uint8_t per_access = 0;
    uint8_t byte_aligned = 1;  // a/du stores: plain or bit-level atomics
};

}  // namespace sfb
