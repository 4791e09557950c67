// Cell-linked SPH density (north-star "density cell-pair neighbour loop").
//
// New algorithm relative to the reference (whose density is all-pairs inside
// contiguous 64-particle buffers, sph.cpp:176-199).  Particles are counting-
// sorted into cells (x-major ids, z fastest; bin_particles below: k_cell_rank
// gives every particle its cell and slot with one returning atomic per (warp,
// cell), a reduce-then-scan turns counts into cell starts, k_place writes the
// permutation without atomics and k_sort_runs orders each cell by particle
// index, so the result is deterministic).  The pass
//
//   k_pack        applies the sort permutation once and packs each particle
//                 as a float4 (x, y, z, m) plus its h (fp16/bf16 stream
//                 values widen exactly), and finds the h range (largest and
//                 smallest h: equal ends select the uniform-h pair loop, which
//                 reads one float4 per candidate and nothing else);
//   k_pairs_c     one thread per PAIR of consecutive homes of the own
//                 x-layers (a contiguous range of the sorted order; the two
//                 usually share a cell): for each of the (2R+1)^2 (dx, dy)
//                 neighbour columns the cells of one z-window are one
//                 contiguous run of the packed array, read through L1/L2
//                 (neighbouring lanes sweep the same runs in lockstep); each
//                 window is culled to the support bound around the pair's box;
//                 every candidate runs the same branch-free pair term against
//                 both homes at once (packed fp32, 1/h_ij hoisted when h is
//                 uniform).  rho is stored back in particle (unsorted) order.
//                 With window masks (one SPH step's density then force), the
//                 sweep also records every home's in-support candidates per
//                 window, and k_force_masked (force section) evaluates exactly
//                 those pairs.
//
// With cells of side >= 2h use reach 1 (27 cells); with cells of side >= h
// reach 2 (125 smaller cells, ~84 after culling).  Pair formula: the
// reference's m_j * W(|x_i - x_j|, (h_i + h_j)/2), M4 spline, sigma = 1/pi,
// evaluated in binary32 (rel <= 1e-5 vs the binary64 oracle).
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <type_traits>
#include <vector>

#include "runtime.hpp"

namespace sfb {

enum StreamPrec { SP_F32 = 0, SP_F16 = 1, SP_BF16 = 2 };

template <int P>
__device__ __forceinline__ float ldf(const void* p, uint64_t i) {
    if constexpr (P == SP_F32) return static_cast<const float*>(p)[i];
    else if constexpr (P == SP_F16) return __half2float(static_cast<const __half*>(p)[i]);
    else return __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
}

// The packed block's smoothing-length range: word [0] = bits of the largest h,
// word [1] = ~bits of the smallest (positive floats order like their bits, so
// both are atomicMax over words zeroed before the pack).  A word [1] of 0
// reads as "range unknown" (no uniform-h fast path).
__device__ __forceinline__ void h_range(float hmax, float hmin, unsigned* __restrict__ words) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        hmax = fmaxf(hmax, __shfl_xor_sync(0xffffffffu, hmax, d));
        hmin = fminf(hmin, __shfl_xor_sync(0xffffffffu, hmin, d));
    }
    if ((threadIdx.x & 31) == 0) {
        if (hmax > 0.0f) atomicMax(words, __float_as_uint(hmax));
        if (hmin < __int_as_float(0x7f800000)) atomicMax(words + 1, ~__float_as_uint(fmaxf(hmin, 0.0f)));
    }
}

// Stored values are exactly representable in binary32, so the packed
// float4 record is lossless for every stream precision.
template <int P>
__global__ void k_pack(const void* __restrict__ x, const void* __restrict__ m, const void* __restrict__ h,
                       const int32_t* __restrict__ perm, uint64_t n, float4* __restrict__ pos,
                       float* __restrict__ hs, unsigned* __restrict__ hmax_bits) {
    float hmax = 0.0f, hmin = __int_as_float(0x7f800000);
    for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < n; k += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = perm ? uint64_t(perm[k]) : k;
        const float hi = ldf<P>(h, i);
        pos[k] = make_float4(ldf<P>(x, 3 * i), ldf<P>(x, 3 * i + 1), ldf<P>(x, 3 * i + 2), ldf<P>(m, i));
        hs[k] = hi;
        hmax = fmaxf(hmax, hi);
        hmin = fminf(hmin, hi);
    }
    h_range(hmax, hmin, hmax_bits);
}

// M4 cubic spline (sph.cpp:17-24) in binary32; caller guarantees q < 2.
__device__ __forceinline__ float w_f32(float q, float inv_h) {
    const float norm = 0.31830988618379067f * inv_h * inv_h * inv_h;
    if (q < 1.0f) return norm * (1.0f - 1.5f * q * q + 0.75f * q * q * q);
    const float t = 2.0f - q;
    return norm * 0.25f * t * t * t;
}

struct CellGrid {
    float lox, loy, loz, inv_cell;
    int nx, ny, nz, reach;
    int64_t n_home;  // particles [0, n_home) (particle order) are homes; the rest neighbours only
};

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float sqrt_approx(float x) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float rsqrt_approx(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// Packed binary32 pairs (sm_100 f32x2: one FADD2 / FMUL2 / FFMA2 issues two
// IEEE binary32 operations, round to nearest, no flush).  A thread evaluates
// one candidate against TWO homes per instruction: the homes' coordinates
// are the pair, the candidate's scalars are broadcast operands.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2(float lo, float hi) {
    f32x2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float lo2(f32x2 a) {
    float l, h;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(l), "=f"(h) : "l"(a));
    (void)h;
    return l;
}
__device__ __forceinline__ float hi2(f32x2 a) {
    float l, h;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(l), "=f"(h) : "l"(a));
    (void)l;
    return h;
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 sub2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
    f32x2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
    f32x2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
// A pair held in one aligned register pair for a whole loop (one FADD2 of +0:
// ptxas keeps the result instead of re-packing the two scalars at every use;
// -0 becomes +0, which no difference or product here can see).
__device__ __forceinline__ f32x2 hold2(float lo, float hi) { return add2(pk2(lo, hi), 0ull); }

// Branch-free M4 spline (sph.cpp:17-24), up to the factor 8 / (4 pi h^3):
//   pi h^3 w(q) / 8 = t^3 - u^3,  t = sat(1 - q/2),  u = sat(c (1 - q)),  c = 2^(-1/3)
// ((2 - q)^3 - 4 (1 - q)^3 = pi h^3 w for q < 1, sph.cpp:20; (2 - q)^3 alone
// for 1 <= q < 2, sph.cpp:22; 0 beyond): saturating FMAs straight from r
// (t = sat(1 + r (-1/2h)), u = sat(c + r (-c/h))), no branch and no support
// test: every candidate runs the same instructions (approximate MUFU forms;
// the sums stay within rel 1e-5 of the binary64 oracle,
// tests/test_gpu_parity.py).  c carries the factor 1/2 of the u^3 term (c^3 =
// 1/2 up to one rounding of c: relative 1e-7 on that term).
constexpr float kC3 = 0.79370052598409974f;  // 2^(-1/3)

__device__ __forceinline__ float spline_w8(float r, float inv_h) {
    const float t = __saturatef(fmaf(-0.5f * inv_h, r, 1.0f));
    const float u = __saturatef(fmaf(-kC3 * inv_h, r, kC3));
    return fmaf(t * t, t, -(u * u) * u);
}

// Two homes (X, Y, Z packed) against one candidate pj: acc += m_j (t^3 - u^3).
// A = -1/(2h), Bc = -c/h of the uniform h.  in0 / in1: the candidate lies
// inside the support of home 0 / 1 (t > 0, i.e. r < 2h).
__device__ __forceinline__ f32x2 density_pair2(f32x2 X, f32x2 Y, f32x2 Z, const float4 pj, float A, float Bc,
                                               f32x2 acc, bool& in0, bool& in1) {
    const f32x2 dx = sub2(X, pk2(pj.x, pj.x)), dy = sub2(Y, pk2(pj.y, pj.y)), dz = sub2(Z, pk2(pj.z, pj.z));
    const f32x2 r2 = fma2(dx, dx, fma2(dy, dy, mul2(dz, dz)));
    const float r0 = sqrt_approx(lo2(r2)), r1 = sqrt_approx(hi2(r2));
    const float t0 = __saturatef(fmaf(A, r0, 1.0f)), t1 = __saturatef(fmaf(A, r1, 1.0f));
    in0 = t0 > 0.0f, in1 = t1 > 0.0f;
    const f32x2 t = pk2(t0, t1);
    const f32x2 u = pk2(__saturatef(fmaf(Bc, r0, kC3)), __saturatef(fmaf(Bc, r1, kC3)));
    const f32x2 w = sub2(mul2(mul2(t, t), t), mul2(mul2(u, u), u));
    return fma2(w, pk2(pj.w, pj.w), acc);
}

// The general (spread-h) pair term for two homes: h_ij = (h_i + h_j) / 2 per
// pair, so 1/h_ij (two MUFU.RCP) and its cube are per pair; HH = (h_0, h_1) / 2.
// acc += m_j / h_ij^3 (t^3 - u^3), t = sat(1 - q/2), u = sat(c (1 - q)).
__device__ __forceinline__ f32x2 density_pair2_h(f32x2 X, f32x2 Y, f32x2 Z, float hh0, float hh1, const float4 pj,
                                                 float hj, f32x2 acc, bool& in0, bool& in1) {
    const f32x2 dx = sub2(X, pk2(pj.x, pj.x)), dy = sub2(Y, pk2(pj.y, pj.y)), dz = sub2(Z, pk2(pj.z, pj.z));
    const f32x2 r2 = fma2(dx, dx, fma2(dy, dy, mul2(dz, dz)));
    const f32x2 ih = pk2(rcp_approx(fmaf(0.5f, hj, hh0)), rcp_approx(fmaf(0.5f, hj, hh1)));
    const f32x2 q = mul2(pk2(sqrt_approx(lo2(r2)), sqrt_approx(hi2(r2))), ih);
    const float q0 = lo2(q), q1 = hi2(q);
    const float t0 = __saturatef(fmaf(-0.5f, q0, 1.0f)), t1 = __saturatef(fmaf(-0.5f, q1, 1.0f));
    in0 = t0 > 0.0f, in1 = t1 > 0.0f;
    const f32x2 t = pk2(t0, t1);
    const f32x2 u = pk2(__saturatef(fmaf(-kC3, q0, kC3)), __saturatef(fmaf(-kC3, q1, kC3)));
    const f32x2 w = sub2(mul2(mul2(t, t), t), mul2(mul2(u, u), u));
    return fma2(w, mul2(mul2(mul2(ih, ih), ih), pk2(pj.w, pj.w)), acc);
}

// The density's in-support bit masks for the force of the same step (which
// needs every rho first, then exactly the same pairs).  For window w (the
// neighbour columns in (dx, dy) row-major order, reach <= 2: 25 windows) of
// the home at sorted position k: occ[k] bit w = the window holds an
// in-support candidate, and then win[w * stride + k] = ((block << 30) | the
// window's first candidate, bits) with bit i set when candidate first + i
// lies inside the home's support; occ[k] bit 31: a window held more than 32
// candidates (that home's force sweeps its windows instead).  Neighbouring
// homes write neighbouring 8-byte words of a window (coalesced); empty
// windows are neither written nor read.
struct WindowMasks {
    int2* win;
    uint32_t* occ;
    int64_t stride;
};
constexpr uint32_t kOccOverflow = 1u << 31;

// The smoothing-length range of the candidate blocks: hmax word [0] = bits of
// the largest h, word [1] = ~bits of the smallest (0 = unknown: not uniform).
template <class BS>
__device__ __forceinline__ bool uniform_h(const BS& B, float* hmax) {
    float hi = 0.0f, lo = __int_as_float(0x7f800000);
#pragma unroll
    for (int g = 0; g < 3; ++g) {
        if (g >= B.nb) break;
        hi = fmaxf(hi, __uint_as_float(B.b[g].hmax[0]));
        const unsigned w1 = B.b[g].hmax[1];
        lo = w1 ? fminf(lo, __uint_as_float(~w1)) : 0.0f;
    }
    *hmax = hi;
    return lo == hi && hi > 0.0f;
}

// Candidate blocks: the homes' own cell-sorted block [0] plus up to two
// neighbouring slabs' blocks [1], [2] (multi-GPU: their packed arrays read in
// place over NVLink through peer pointers, no ghost copy).  Each block covers
// global x-layers [x0, x0 + nx) of one grid (shared origin, cell, ny, nz).
struct CellBlock {
    const float4* pos;  // (x, y, z, m)
    const float* h;
    const int32_t* cs;
    const unsigned* hmax;
    int x0, nx;
    float lox;  // x origin the block was binned with (its layer x0 starts there)
};
struct BlockSet {
    CellBlock b[3];
    int nb, NX;  // blocks in use; global x-layers (faces at 0 and NX)
};

// Two consecutive homes of the cell-sorted order per thread (almost always
// the same cell column, usually the same cell): they share one pass over the
// neighbour columns, each window cut to the support bound around the pair's
// box, and every candidate is evaluated against both homes at once with the
// packed-fp32 pair terms above.  A pair straddling a column boundary takes
// one pass per home.  Homes past n or at/after n_home (ghosts) are not
// written.
struct HomePair {
    float4 p0, p1;  // (x, y, z, m)
    float h0, h1;
    float fx0, fy0, fz0, fx1, fy1, fz1;  // cell coordinates (global x layers)
    int ix0, iy0, ix1, iy1;
    int64_t i0, i1;  // particle indices (i >= n_home: not a home)
};

template <class Blk>
__device__ __forceinline__ HomePair load_pair(const Blk& b0, const int32_t* __restrict__ perm, const CellGrid& G,
                                              int64_t k0, int64_t n) {
    HomePair H;
    const int64_t k1 = k0 + 1 < n ? k0 + 1 : k0;
    H.i0 = perm ? int64_t(perm[k0]) : k0;
    H.i1 = k0 + 1 < n ? (perm ? int64_t(perm[k1]) : k1) : G.n_home;
    H.p0 = b0.pos[k0], H.p1 = b0.pos[k1];
    H.h0 = b0.h[k0], H.h1 = b0.h[k1];
    // the binning formula of the own block (same origin, same rounding), then global layers
    const float fxl0 = (H.p0.x - b0.lox) * G.inv_cell, fxl1 = (H.p1.x - b0.lox) * G.inv_cell;
    H.fy0 = (H.p0.y - G.loy) * G.inv_cell, H.fy1 = (H.p1.y - G.loy) * G.inv_cell;
    H.fz0 = (H.p0.z - G.loz) * G.inv_cell, H.fz1 = (H.p1.z - G.loz) * G.inv_cell;
    H.ix0 = min(max(int(floorf(fxl0)), 0), b0.nx - 1) + b0.x0;
    H.ix1 = min(max(int(floorf(fxl1)), 0), b0.nx - 1) + b0.x0;
    H.fx0 = fxl0 + float(b0.x0), H.fx1 = fxl1 + float(b0.x0);
    H.iy0 = min(max(int(floorf(H.fy0)), 0), G.ny - 1);
    H.iy1 = min(max(int(floorf(H.fy1)), 0), G.ny - 1);
    return H;
}

// The candidate runs of one pass (members m0 / m1 of the pair): for each of
// the (2R+1)^2 neighbour columns the cells of one z-window are one contiguous
// run [b, e) of a block (own, or a neighbouring slab's read in place), cut to
// the support bound rc (cell units, squared) around the members' box;
// columns the bound misses are skipped.  Cells on the grid faces extend to
// infinity (binning clamps), so their distance is measured only on their
// inner side.  Culling removes only candidates at q >= 2 (w = 0; the radius
// margin covers rounding).  Neighbouring threads sweep the same runs in
// lockstep (their homes are neighbours in the sorted order), so candidate
// lines are shared through L1.  visit(w, g, b, e) is called for every window
// w of the (2R+1)^2 (row-major in (dx, dy)); empty ones with b == e.
template <int R, class BS, class Visit>
__device__ __forceinline__ void pass_runs(const BS& B, const CellGrid& G, const HomePair& H, bool m0, bool m1,
                                          float rc2, Visit&& visit) {
    constexpr int W = 2 * R + 1;
    const float fxlo = m0 ? (m1 ? fminf(H.fx0, H.fx1) : H.fx0) : H.fx1;
    const float fxhi = m0 ? (m1 ? fmaxf(H.fx0, H.fx1) : H.fx0) : H.fx1;
    const float fylo = m0 ? (m1 ? fminf(H.fy0, H.fy1) : H.fy0) : H.fy1;
    const float fyhi = m0 ? (m1 ? fmaxf(H.fy0, H.fy1) : H.fy0) : H.fy1;
    const float fzlo = fminf(fmaxf(m0 ? (m1 ? fminf(H.fz0, H.fz1) : H.fz0) : H.fz1, -1e6f), 1e6f);
    const float fzhi = fminf(fmaxf(m0 ? (m1 ? fmaxf(H.fz0, H.fz1) : H.fz0) : H.fz1, -1e6f), 1e6f);
    const int ix = m0 ? H.ix0 : H.ix1, iy = m0 ? H.iy0 : H.iy1;
    const int izl = min(max(int(floorf(fzlo)), 0), G.nz - 1), izh = min(max(int(floorf(fzhi)), 0), G.nz - 1);
    const int zmin = max(izl - R, 0), zmax = min(izh + R, G.nz - 1);
#pragma unroll 1
    for (int dxi = -R; dxi <= R; ++dxi) {
        const int jx = ix + dxi;
        const int w0 = (dxi + R) * W;  // window index of the row's first column
        int g = 0;
        if (jx >= 0 && jx < B.NX)
            while (g < B.nb && (jx < B.b[g].x0 || jx >= B.b[g].x0 + B.b[g].nx)) ++g;
        if (jx < 0 || jx >= B.NX || g == B.nb) {  // outside the grid, or a layer held by no block
            for (int t = 0; t < W; ++t) visit(w0 + t, 0, 0, 0);
            continue;
        }
        const int32_t* __restrict__ cell_start = B.b[g].cs;
        const float ddx =
            fmaxf(fmaxf(jx > 0 ? float(jx) - fxhi : 0.0f, jx < B.NX - 1 ? fxlo - float(jx + 1) : 0.0f), 0.0f);
        const int cx = (jx - B.b[g].x0) * G.ny;  // cell ids fit in int32 (checked on the host)
#pragma unroll 1
        for (int t = 0; t < W; ++t) {
            const int jy = iy - R + t;
            const float ddy =
                fmaxf(fmaxf(jy > 0 ? float(jy) - fyhi : 0.0f, jy < G.ny - 1 ? fylo - float(jy + 1) : 0.0f), 0.0f);
            const float d2 = fmaf(ddx, ddx, ddy * ddy);
            const float dz = sqrt_approx(fmaxf(rc2 - d2, 0.0f));  // rel err ~1e-7, inside the margin
            const int zlo = min(max(int(floorf(fzlo - dz)), zmin), G.nz - 1);
            const int zhi = max(min(int(floorf(fzhi + dz)), zmax), 0);
            if (jy < 0 || jy >= G.ny || !(d2 < rc2) || zlo > zhi) {
                visit(w0 + t, g, 0, 0);
                continue;
            }
            const int c0 = (cx + jy) * G.nz;
            visit(w0 + t, g, __ldg(cell_start + c0 + zlo), __ldg(cell_start + c0 + zhi + 1));
        }
    }
}

template <int R, bool UNI, bool LIST>
__device__ __forceinline__ void pairs_home2(const BlockSet& B, const int32_t* __restrict__ perm, const CellGrid& G,
                                            int64_t k0, int64_t n, float hmax, float* __restrict__ rho,
                                            const WindowMasks& M) {
    const HomePair H = load_pair(B.b[0], perm, G, k0, n);
    const bool live0 = H.i0 < G.n_home, live1 = H.i1 < G.n_home;
    if (!live0 && !live1) return;  // ghosts: neighbours only
    constexpr float k2InvPi = 0.63661977236758134f;  // 8 / (4 pi): spline_w8 carries w / 8
    uint32_t occ0 = 0, occ1 = 0;                     // LIST: windows with in-support candidates, overflow
    // LIST: a home's window (base, in-support bits) for the force, when it holds any
    auto put = [&](bool home, int w, int g, int b, uint32_t bits, bool fit) {
        uint32_t& occ = home ? occ1 : occ0;
        if (!fit) occ |= kOccOverflow;
        if (bits == 0) return;
        occ |= 1u << w;
        // streaming store (evict-first): the masks are read once, by the force, and must not push the
        // candidate lines out of L2
        __stcs(M.win + int64_t(w) * M.stride + k0 + (home ? 1 : 0),
               make_int2(int(uint32_t(g) << 30 | uint32_t(b)), int(bits)));
    };
    if constexpr (UNI) {
        const bool same = H.ix0 == H.ix1 && H.iy0 == H.iy1;
        const float inv_h = rcp_approx(hmax);  // h_ij = h for every pair
        const float A = -0.5f * inv_h, Bc = -kC3 * inv_h;
        const float rc = 2.0f * hmax * G.inv_cell * 1.00001f;  // support bound, cell units
        const f32x2 X = hold2(H.p0.x, H.p1.x), Y = hold2(H.p0.y, H.p1.y), Z = hold2(H.p0.z, H.p1.z);
        float res0 = 0.0f, res1 = 0.0f;
#pragma unroll 1
        for (int pass = 0; pass < (same ? 1 : 2); ++pass) {
            const bool m0 = same || pass == 0, m1 = same || pass == 1;
            f32x2 acc = 0ull, acc2 = 0ull;  // +0.0f pairs; two chains for ILP
            pass_runs<R>(B, G, H, m0, m1, rc * rc, [&](int w, int g, int b, int e) {
                const float4* __restrict__ pos = B.b[g].pos;
                uint32_t mk0 = 0, mk1 = 0, bit = 1;  // LIST: bit of candidate j (0 past 32: no mask)
                const bool fit = e - b <= 32;
                int j = b;
#pragma unroll 1
                for (; j + 1 < e; j += 2) {
                    const float4 p = pos[j], q = pos[j + 1];
                    bool a0, a1, b0, b1;
                    acc = density_pair2(X, Y, Z, p, A, Bc, acc, a0, a1);
                    acc2 = density_pair2(X, Y, Z, q, A, Bc, acc2, b0, b1);
                    if constexpr (LIST) {
                        if (a0) mk0 |= bit;
                        if (a1) mk1 |= bit;
                        if (b0) mk0 |= bit << 1;
                        if (b1) mk1 |= bit << 1;
                        bit <<= 2;
                    }
                }
                if (j < e) {
                    bool a0, a1;
                    acc = density_pair2(X, Y, Z, pos[j], A, Bc, acc, a0, a1);
                    if constexpr (LIST) {
                        if (a0) mk0 |= bit;
                        if (a1) mk1 |= bit;
                    }
                }
                if constexpr (LIST) {
                    if (m0 && live0) put(false, w, g, b, mk0, fit);
                    if (m1 && live1) put(true, w, g, b, mk1, fit);
                }
            });
            acc = add2(acc, acc2);
            if (m0) res0 = lo2(acc);
            if (m1) res1 = hi2(acc);
        }
        const float scale = (inv_h * inv_h) * inv_h * k2InvPi;
        if (live0) rho[H.i0] = res0 * scale;
        if (live1) rho[H.i1] = res1 * scale;
    } else {
        // spread h: h_ij = (h_i + h_j) / 2 per pair, both homes per candidate (packed)
        const bool same = H.ix0 == H.ix1 && H.iy0 == H.iy1;
        const float hh0 = 0.5f * H.h0, hh1 = 0.5f * H.h1;
        const f32x2 X = hold2(H.p0.x, H.p1.x), Y = hold2(H.p0.y, H.p1.y), Z = hold2(H.p0.z, H.p1.z);
        float res0 = 0.0f, res1 = 0.0f;
#pragma unroll 1
        for (int pass = 0; pass < (same ? 1 : 2); ++pass) {
            const bool m0 = same || pass == 0, m1 = same || pass == 1;
            const float hm = m0 ? (m1 ? fmaxf(H.h0, H.h1) : H.h0) : H.h1;
            const float rc = (hm + hmax) * G.inv_cell * 1.00001f;  // support bound, cell units
            f32x2 acc = 0ull;
            pass_runs<R>(B, G, H, m0, m1, rc * rc, [&](int w, int g, int b, int e) {
                const float4* __restrict__ pos = B.b[g].pos;
                const float* __restrict__ hs = B.b[g].h;
                uint32_t mk0 = 0, mk1 = 0, bit = 1;
                const bool fit = e - b <= 32;
#pragma unroll 1
                for (int j = b; j < e; ++j, bit <<= 1) {
                    bool a0, a1;
                    acc = density_pair2_h(X, Y, Z, hh0, hh1, pos[j], __ldg(hs + j), acc, a0, a1);
                    if constexpr (LIST) {
                        if (a0) mk0 |= bit;
                        if (a1) mk1 |= bit;
                    }
                }
                if constexpr (LIST) {
                    if (m0 && live0) put(false, w, g, b, mk0, fit);
                    if (m1 && live1) put(true, w, g, b, mk1, fit);
                }
            });
            if (m0) res0 = lo2(acc);
            if (m1) res1 = hi2(acc);
        }
        if (live0) rho[H.i0] = res0 * k2InvPi;
        if (live1) rho[H.i1] = res1 * k2InvPi;
    }
    if constexpr (LIST) {
        if (live0) M.occ[k0] = occ0;
        if (live1) M.occ[k0 + 1] = occ1;
    }
}

// One thread per pair of homes over a grid of ceil(n/512) CTAs (not a capped
// grid-stride loop): the block scheduler hands out CTAs in index order, so
// the CTAs in flight always cover one compact range of the cell-sorted homes
// and their candidate columns stay in L2 (with the grid capped at 16 CTAs/SM
// the resident CTAs strode through the whole range and the L2 hit rate at C5
// fell from 91% to 46%).
constexpr int kPairThreads = 128;
static unsigned pair_grid(uint64_t n) { return unsigned(((n + 1) / 2 + kPairThreads - 1) / kPairThreads); }

template <int R, bool LIST>
__global__ void __launch_bounds__(kPairThreads, 10) k_pairs_c(const BlockSet B, const int32_t* __restrict__ perm, CellGrid G,
                                                 int64_t n, float* __restrict__ rho, const WindowMasks M) {
    float hmax;
    const bool uni = uniform_h(B, &hmax);
    const int64_t k0 = 2 * (blockIdx.x * int64_t(blockDim.x) + threadIdx.x);
    if (k0 >= n) return;
    if (uni) pairs_home2<R, true, LIST>(B, perm, G, k0, n, hmax, rho, M);
    else pairs_home2<R, false, LIST>(B, perm, G, k0, n, hmax, rho, M);
}

template <bool LIST>
static void launch_pairs_t(const BlockSet& B, const int32_t* perm, const CellGrid& G, int64_t n, int reach,
                           float* rho, const WindowMasks& M, cudaStream_t st) {
    const unsigned grid = pair_grid(uint64_t(n));
    if (reach == 1) k_pairs_c<1, LIST><<<grid, kPairThreads, 0, st>>>(B, perm, G, n, rho, M);
    else if (reach == 2) k_pairs_c<2, LIST><<<grid, kPairThreads, 0, st>>>(B, perm, G, n, rho, M);
    else if constexpr (!LIST) {  // window masks: 25 windows at most (reach <= 2)
        if (reach == 3) k_pairs_c<3, false><<<grid, kPairThreads, 0, st>>>(B, perm, G, n, rho, M);
        else k_pairs_c<4, false><<<grid, kPairThreads, 0, st>>>(B, perm, G, n, rho, M);
    }
}

static void launch_pairs(const BlockSet& B, const int32_t* perm, const CellGrid& G, int64_t n, int reach, float* rho,
                         cudaStream_t st, const WindowMasks* M = nullptr) {
    if (M) launch_pairs_t<true>(B, perm, G, n, reach, rho, *M, st);
    else launch_pairs_t<false>(B, perm, G, n, reach, rho, WindowMasks{nullptr, nullptr, 0}, st);
}


void density_cells(const void* x, const void* m, const void* h, int prec, uint64_t n, const int32_t* perm,
                   const int32_t* cell_start, const float* lo, float cell, int nx, int ny, int nz, int reach,
                   uint64_t n_home, float* rho, cudaStream_t st) {
    require_device();
    if (nx <= 0 || ny <= 0 || nz <= 0 || n_home > n || reach < 1 || reach > 4)
        throw std::invalid_argument("bad cell grid");
    if (n >= (1ull << 31)) throw std::invalid_argument("density_cells: n must be < 2^31 per device");
    if (int64_t(nx) * ny * nz >= (1ll << 31)) throw std::invalid_argument("bad cell grid");
    if (n == 0) return;
    const int sp = (prec == 1 || prec == 32) ? SP_F32 : prec == 16 ? SP_F16 : prec == 100 ? SP_BF16 : -1;
    if (sp < 0) throw std::invalid_argument("density_cells precision must be SF_PREC_NATIVE (fp32), 16 or SF_PREC_BF16");
    float4* pos = nullptr;
    float* hs = nullptr;
    check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&pos), 16 * n, st), "cudaMallocAsync");
    check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&hs), 4 * n + 16, st), "cudaMallocAsync");
    unsigned* hmax = reinterpret_cast<unsigned*>(hs + n);
    check_cuda(cudaMemsetAsync(hmax, 0, 2 * sizeof(unsigned), st), "memset");
    const unsigned blocks = unsigned(std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * 16));
    CellGrid G{lo[0], lo[1], lo[2], 1.0f / cell, nx, ny, nz, reach, int64_t(n_home)};
    const int64_t nn = int64_t(n);
    if (sp == SP_F32) k_pack<SP_F32><<<blocks, 256, 0, st>>>(x, m, h, perm, n, pos, hs, hmax);
    else if (sp == SP_F16) k_pack<SP_F16><<<blocks, 256, 0, st>>>(x, m, h, perm, n, pos, hs, hmax);
    else k_pack<SP_BF16><<<blocks, 256, 0, st>>>(x, m, h, perm, n, pos, hs, hmax);
    BlockSet B{};
    B.b[0] = CellBlock{pos, hs, cell_start, hmax, 0, nx, lo[0]};
    B.nb = 1;
    B.NX = nx;
    launch_pairs(B, perm, G, nn, reach, rho, st);
    check_cuda(cudaGetLastError(), "density_cells launch");
    count_launches(2);
    check_cuda(cudaFreeAsync(pos, st), "cudaFreeAsync");
    check_cuda(cudaFreeAsync(hs, st), "cudaFreeAsync");
}

// Pack for the block API: caller-owned, persistent outputs (so that other
// ranks can read them in place through peer pointers).
void cells_pack(const void* x, const void* m, const void* h, int prec, uint64_t n, const int32_t* perm, void* pos,
                float* hs, unsigned* hmax, cudaStream_t st) {
    require_device();
    if (n >= (1ull << 31)) throw std::invalid_argument("cells_pack: n must be < 2^31 per device");
    const int sp = (prec == 1 || prec == 32) ? SP_F32 : prec == 16 ? SP_F16 : prec == 100 ? SP_BF16 : -1;
    if (sp < 0) throw std::invalid_argument("cells_pack precision must be SF_PREC_NATIVE (fp32), 16 or SF_PREC_BF16");
    check_cuda(cudaMemsetAsync(hmax, 0, 2 * sizeof(unsigned), st), "memset");
    if (n == 0) return;
    if (reinterpret_cast<uintptr_t>(pos) & 15) throw std::invalid_argument("pos must be 16-byte aligned");
    float4* p4 = static_cast<float4*>(pos);
    const unsigned blocks = unsigned(std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * 16));
    if (sp == SP_F32) k_pack<SP_F32><<<blocks, 256, 0, st>>>(x, m, h, perm, n, p4, hs, hmax);
    else if (sp == SP_F16) k_pack<SP_F16><<<blocks, 256, 0, st>>>(x, m, h, perm, n, p4, hs, hmax);
    else k_pack<SP_BF16><<<blocks, 256, 0, st>>>(x, m, h, perm, n, p4, hs, hmax);
    check_cuda(cudaGetLastError(), "cells_pack launch");
    count_launches(1);
}

void density_cells_blocks(const CellBlockDesc* blocks, int nb, uint64_t n, const int32_t* perm, uint64_t n_home,
                          const float* lo_yz, float cell, int NX, int ny, int nz, int reach, float* rho,
                          cudaStream_t st, int32_t* win) {
    require_device();
    if (nb < 1 || nb > 3 || NX <= 0 || ny <= 0 || nz <= 0 || n_home > n || reach < 1 || reach > 4 || !(cell > 0))
        throw std::invalid_argument("bad cell grid");
    if (n >= (1ull << 31)) throw std::invalid_argument("density_cells: n must be < 2^31 per device");
    BlockSet B{};
    B.nb = nb;
    B.NX = NX;
    for (int g = 0; g < nb; ++g) {
        const CellBlockDesc& d = blocks[g];
        if (!d.pos || !d.h || !d.cell_start || !d.hmax) throw std::invalid_argument("null block pointer");
        if (d.nx <= 0 || d.x0 < 0 || d.x0 + d.nx > NX || int64_t(d.nx) * ny * nz >= (1ll << 31))
            throw std::invalid_argument("block layers outside the grid");
        B.b[g] = CellBlock{static_cast<const float4*>(d.pos), d.h, d.cell_start, d.hmax, d.x0, d.nx, d.x_origin};
    }
    if (n == 0) return;
    CellGrid G{blocks[0].x_origin, lo_yz[0], lo_yz[1], 1.0f / cell, NX, ny, nz, reach, int64_t(n_home)};
    if (win && reach <= 2) {  // window bases are tagged (block << 30): every block must hold < 2^30 particles
        if (n >= (1ull << 30)) throw std::invalid_argument("window masks need fewer than 2^30 particles per block");
        const WindowMasks M{reinterpret_cast<int2*>(win), reinterpret_cast<uint32_t*>(win) + window_mask_words(n, reach) - n,
                            int64_t(n)};
        launch_pairs(B, perm, G, int64_t(n), reach, rho, st, &M);
    } else {
        launch_pairs(B, perm, G, int64_t(n), reach, rho, st);
    }
    check_cuda(cudaGetLastError(), "density_cells_blocks launch");
    count_launches(1);
}

// ------------------------------------------------------------------ force
// Cell-linked force (sph.cpp:201-245 restated over cell neighbours; the
// reference evaluates it inside 64-particle buffers).  k_pack_force packs per
// sorted particle (x, y, z, m), (vx, vy, vz, P/rho^2) and h, flags rho == 0
// (the reference's domain_error) and reduces h_max; k_force_c sweeps the same
// culled column runs as k_pairs_c and accumulates, per home particle i,
//   a_i  = -sum_j m_j (P_i/rho_i^2 + P_j/rho_j^2) dW/dr(r, h_ij) dx/r
//   du_i =  P_i/rho_i^2 sum_j m_j (v_i - v_j) . dx dW/dr(r, h_ij) / r
// with the branch-free M4 derivative
//   pi h_ij^4 dW/dr = 3 max(1-q,0)^2 - 0.75 max(2-q,0)^2
// (q < 1: -3q + 2.25q^2, sph.cpp:30; 1 <= q < 2: -0.75 (2-q)^2, sph.cpp:32),
// which is exactly 0 at r = 0, so the self term vanishes as in grad_w
// (sph.cpp:35-40) without a j != i test.  binary32 arithmetic; tolerance
// relative to sum_j |term| (tests/test_gpu_parity.py).
template <int P>
__global__ void k_pack_force(const void* __restrict__ x, const void* __restrict__ v, const void* __restrict__ m,
                             const void* __restrict__ h, const void* __restrict__ rho, const void* __restrict__ pr,
                             const int32_t* __restrict__ perm, uint64_t n, float4* __restrict__ pos,
                             float4* __restrict__ vel, float* __restrict__ hs, unsigned* __restrict__ hmax_bits,
                             unsigned* __restrict__ degenerate) {
    float hmax = 0.0f, hmin = __int_as_float(0x7f800000);
    bool zero = false;
    for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < n; k += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = perm ? uint64_t(perm[k]) : k;
        const float hi = ldf<P>(h, i), ri = ldf<P>(rho, i);
        pos[k] = make_float4(ldf<P>(x, 3 * i), ldf<P>(x, 3 * i + 1), ldf<P>(x, 3 * i + 2), ldf<P>(m, i));
        vel[k] = make_float4(ldf<P>(v, 3 * i), ldf<P>(v, 3 * i + 1), ldf<P>(v, 3 * i + 2), ldf<P>(pr, i) / (ri * ri));
        hs[k] = hi;
        hmax = fmaxf(hmax, hi);
        hmin = fminf(hmin, hi);
        zero |= ri == 0.0f;
    }
    h_range(hmax, hmin, hmax_bits);
    if (__any_sync(0xffffffffu, zero) && (threadIdx.x & 31) == 0) atomicOr(degenerate, 1u);
}

// Candidate blocks of the force: a density block's (x,y,z,m) and h plus the
// same particles' (v, P/rho^2), all in the block's cell-sorted order.
struct ForceBlock {
    const float4* pos;  // (x, y, z, m)
    const float4* vel;  // (vx, vy, vz, P/rho^2)
    const float* h;
    const int32_t* cs;
    const unsigned* hmax;
    int x0, nx;
    float lox;
};
struct ForceBlockSet {
    ForceBlock b[3];
    int nb, NX;
};

// One force term (sph.cpp:201-245) of candidate (pj = (x, m), vj = (v, P/rho^2))
// on home (pi, vi), accumulated into s:
//   (ax, ay, az) += m_j (P_i/rho_i^2 + P_j/rho_j^2) pi h_ij^4 dW/dr / r * dx
//   cp           += m_j pi h_ij^4 dW/dr / r * (v_i - v_j) . dx
// with pi h^4 dW/dr = 3 max(1-q,0)^2 - 0.75 max(2-q,0)^2 (q < 1: -3q + 2.25q^2,
// sph.cpp:30; 1 <= q < 2: -0.75 (2-q)^2, sph.cpp:32), exactly 0 at r = 0, so
// the self term vanishes as in grad_w (sph.cpp:35-40) without a j != i test.
struct ForceSums {
    float ax, ay, az, cp;
};
__device__ __forceinline__ void force_term(const float4 pi, const float4 vi, float inv_h, float ih4, const float4 pj,
                                           const float4 vj, ForceSums& s) {
    const float dx = pi.x - pj.x, dy = pi.y - pj.y, dz = pi.z - pj.z;
    const float r2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    const float inv_r = rsqrt_approx(fmaxf(r2, 1e-30f));
    const float q = (r2 * inv_r) * inv_h;
    const float t = fmaxf(2.0f - q, 0.0f), u = fmaxf(1.0f - q, 0.0f);
    const float dw = fmaf(-0.75f * t, t, 3.0f * u * u);  // pi h^4 dW/dr
    const float msc = pj.w * (dw * ih4 * inv_r);           // m_j pi dW/dr / r
    const float f = msc * (vi.w + vj.w);
    s.ax = fmaf(f, dx, s.ax);
    s.ay = fmaf(f, dy, s.ay);
    s.az = fmaf(f, dz, s.az);
    s.cp = fmaf(msc, fmaf(dz, vi.z - vj.z, fmaf(dy, vi.y - vj.y, dx * (vi.x - vj.x))), s.cp);
}

__device__ __forceinline__ void store_force(const ForceSums& s, float pfi, int64_t i, float* __restrict__ a_out,
                                            float* __restrict__ du_out) {
    constexpr float kInvPi = 0.31830988618379067f;
    a_out[3 * i] = -kInvPi * s.ax;
    a_out[3 * i + 1] = -kInvPi * s.ay;
    a_out[3 * i + 2] = -kInvPi * s.az;
    du_out[i] = pfi * (kInvPi * s.cp);
}

template <int R, int U, bool UNI>
__device__ __forceinline__ void force_home(const ForceBlockSet& B, const int32_t* __restrict__ perm, const CellGrid& G,
                                           int64_t k, float hmax, float* __restrict__ a_out,
                                           float* __restrict__ du_out) {
    constexpr int W = 2 * R + 1;
    const int hx0 = B.b[0].x0, hnx = B.b[0].nx;
    const float hlox = B.b[0].lox;
    const int64_t i_home = perm ? perm[k] : k;
    if (i_home >= G.n_home) return;  // ghosts: neighbours only
    const float4 pi = B.b[0].pos[k];
    const float h_i = B.b[0].h[k];
    const float fxl = (pi.x - hlox) * G.inv_cell, fy = (pi.y - G.loy) * G.inv_cell,
                fz = (pi.z - G.loz) * G.inv_cell;
    const int ix = min(max(int(floorf(fxl)), 0), hnx - 1) + hx0;
    const float fx = fxl + float(hx0);
    const int iy = min(max(int(floorf(fy)), 0), G.ny - 1);
    const int iz = min(max(int(floorf(fz)), 0), G.nz - 1);
    const float4 vi = B.b[0].vel[k];
    const float pfi = vi.w;
    const float rc = (h_i + hmax) * G.inv_cell * 1.00001f;
    const float rc2 = rc * rc;
    const float hh_i = 0.5f * h_i;
    const float inv_hu = rcp_approx(fmaf(0.5f, h_i, hh_i));  // UNI: 1/h_ij for every candidate
    const float ih4u = (inv_hu * inv_hu) * (inv_hu * inv_hu);
    const float fzc = fminf(fmaxf(fz, -1e6f), 1e6f);
    const int zmin = max(iz - R, 0), zmax = min(iz + R, G.nz - 1);
    ForceSums S{0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll 1
    for (int dxi = -R; dxi <= R; ++dxi) {
        const int jx = ix + dxi;
        if (jx < 0 || jx >= B.NX) continue;
        int g = 0;
        while (g < B.nb && (jx < B.b[g].x0 || jx >= B.b[g].x0 + B.b[g].nx)) ++g;
        if (g == B.nb) continue;  // layer held by no block
        const float4* __restrict__ pos = B.b[g].pos;
        const float4* __restrict__ vel = B.b[g].vel;
        const float* __restrict__ hs = B.b[g].h;
        const int32_t* __restrict__ cell_start = B.b[g].cs;
        auto pair = [&](int j) {
            if constexpr (UNI) {
                force_term(pi, vi, inv_hu, ih4u, pos[j], vel[j], S);
            } else {
                const float inv_h = rcp_approx(fmaf(0.5f, __ldg(hs + j), hh_i));
                const float ih2 = inv_h * inv_h;
                force_term(pi, vi, inv_h, ih2 * ih2, pos[j], vel[j], S);
            }
        };
        const float ddx = fmaxf(fmaxf(jx > 0 ? float(jx) - fx : 0.0f, jx < B.NX - 1 ? fx - float(jx + 1) : 0.0f),
                                0.0f);
        int b[W], e[W];
        const int cx = (jx - B.b[g].x0) * G.ny;
#pragma unroll
        for (int t = 0; t < W; ++t) {
            const int jy = iy - R + t;
            const float ddy = fmaxf(
                fmaxf(jy > 0 ? float(jy) - fy : 0.0f, jy < G.ny - 1 ? fy - float(jy + 1) : 0.0f), 0.0f);
            const float d2 = fmaf(ddx, ddx, ddy * ddy);
            const float dzr = sqrt_approx(fmaxf(rc2 - d2, 0.0f));
            const int zlo = min(max(int(floorf(fzc - dzr)), zmin), G.nz - 1);
            const int zhi = max(min(int(floorf(fzc + dzr)), zmax), 0);
            const bool ok = jy >= 0 && jy < G.ny && d2 < rc2 && zlo <= zhi;
            const int c0 = (cx + (ok ? jy : 0)) * G.nz;
            b[t] = ok ? __ldg(cell_start + c0 + zlo) : 0;
            e[t] = ok ? __ldg(cell_start + c0 + zhi + 1) : 0;
        }
#pragma unroll
        for (int t = 0; t < W; ++t) {
            int j = b[t];
            if constexpr (U == 2) {
                for (; j + 1 < e[t]; j += 2) {
                    pair(j);
                    pair(j + 1);
                }
            }
            for (; j < e[t]; ++j) pair(j);
        }
    }
    store_force(S, pfi, i_home, a_out, du_out);
}

// The force of one home from the in-support bit masks the density of the
// same step wrote (exactly the in-support pairs, no culling arithmetic): one
// flattened loop over the home's windows, refilling (base, bits) when the
// current mask is spent, so a lane's iterations are its ~65 pairs plus the
// (2R+1)^2 refills rather than the sum over windows of the warp's longest
// run.  A home with an over-long window falls back to the window sweep.
template <int R, bool UNI>
__device__ __forceinline__ void force_masked_home(const ForceBlockSet& B, const int32_t* __restrict__ perm,
                                                  const CellGrid& G, int64_t k, float hmax, const WindowMasks& M,
                                                  float* __restrict__ a_out, float* __restrict__ du_out) {
    const int64_t i_home = perm ? perm[k] : k;
    if (i_home >= G.n_home) return;  // ghosts: neighbours only
    uint32_t occ = M.occ[k];
    if (occ & kOccOverflow) {
        force_home<R, 2, UNI>(B, perm, G, k, hmax, a_out, du_out);
        return;
    }
    const float4 pi = B.b[0].pos[k], vi = B.b[0].vel[k];
    const float h_i = B.b[0].h[k], hh_i = 0.5f * h_i;
    const float inv_hu = rcp_approx(h_i);
    const float ih4u = (inv_hu * inv_hu) * (inv_hu * inv_hu);
    ForceSums S{0.0f, 0.0f, 0.0f, 0.0f};
    const int2* __restrict__ win = M.win + k;
    int g = 0, base = 0;
    uint32_t bits = 0;
    const float4* __restrict__ pos = B.b[0].pos;
    const float4* __restrict__ vel = B.b[0].vel;
    const float* __restrict__ hs = B.b[0].h;
    auto term = [&](int j, bool real) {
        float4 pj = pos[j];
        if (!real) pj.w = 0.0f;  // padding lane of a pair: zero mass, zero contribution
        if constexpr (UNI) {
            force_term(pi, vi, inv_hu, ih4u, pj, vel[j], S);
        } else {
            const float inv_h = rcp_approx(fmaf(0.5f, __ldg(hs + j), hh_i));
            const float ih2 = inv_h * inv_h;
            force_term(pi, vi, inv_h, ih2 * ih2, pj, vel[j], S);
        }
    };
    // software pipeline: the next occupied window's (base, bits) is loaded while the current one is swept;
    // an exhausted window is replaced by it with register moves only, in the same iteration as the next two
    // terms, so lanes that switch windows do not stall the others
    auto fetch = [&](uint32_t& o) {
        int2 t = make_int2(0, 0);
        if (o) {
            t = __ldg(win + int64_t(__ffs(o) - 1) * M.stride);
            o &= o - 1;
        }
        return t;
    };
    int2 nxt = fetch(occ);
#pragma unroll 1
    while (bits | uint32_t(nxt.y)) {
        if (bits == 0) {  // next occupied window (a block switch is rare: only at slab faces)
            bits = uint32_t(nxt.y);
            base = int(uint32_t(nxt.x) & 0x3fffffffu);
            const int gn = int(uint32_t(nxt.x) >> 30);
            if (gn != g) {
                g = gn;
                pos = B.b[g].pos, vel = B.b[g].vel, hs = B.b[g].h;
            }
            nxt = fetch(occ);
        }
        // two in-support candidates of the window per iteration (independent loads and terms)
        const int j0 = base + __ffs(bits) - 1;
        bits &= bits - 1;
        const bool two = bits != 0;
        const int j1 = two ? base + __ffs(bits) - 1 : j0;
        if (two) bits &= bits - 1;
        term(j0, true);
        term(j1, two);
    }
    store_force(S, vi.w, i_home, a_out, du_out);
}

template <int R, int U>
__global__ void __launch_bounds__(128) k_force_c(const ForceBlockSet B, const int32_t* __restrict__ perm, CellGrid G,
                                                 int64_t n, float* __restrict__ a_out, float* __restrict__ du_out) {
    float hmax;
    const bool uni = uniform_h(B, &hmax);
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        if (uni) force_home<R, U, true>(B, perm, G, k, hmax, a_out, du_out);
        else force_home<R, U, false>(B, perm, G, k, hmax, a_out, du_out);
    }
}

static void launch_force(const ForceBlockSet& B, const int32_t* perm, const CellGrid& G, int64_t n, int reach,
                         float* a, float* du, cudaStream_t st) {
    constexpr unsigned T = 128;
    const unsigned grid = unsigned((uint64_t(n) + T - 1) / T);  // one thread per home, in index order
    if (reach == 1) k_force_c<1, 2><<<grid, T, 0, st>>>(B, perm, G, n, a, du);
    else if (reach == 2) k_force_c<2, 2><<<grid, T, 0, st>>>(B, perm, G, n, a, du);
    else if (reach == 3) k_force_c<3, 2><<<grid, T, 0, st>>>(B, perm, G, n, a, du);
    else k_force_c<4, 2><<<grid, T, 0, st>>>(B, perm, G, n, a, du);
}

template <int R>
__global__ void __launch_bounds__(256) k_force_masked(const ForceBlockSet B, const int32_t* __restrict__ perm,
                                                      CellGrid G, int64_t n, const WindowMasks M,
                                                      float* __restrict__ a_out, float* __restrict__ du_out) {
    float hmax;
    const bool uni = uniform_h(B, &hmax);
    const int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (k >= n) return;
    if (uni) force_masked_home<R, true>(B, perm, G, k, hmax, M, a_out, du_out);
    else force_masked_home<R, false>(B, perm, G, k, hmax, M, a_out, du_out);
}

static void launch_force_masked(const ForceBlockSet& B, const int32_t* perm, const CellGrid& G, int64_t n, int reach,
                                const WindowMasks& M, float* a, float* du, cudaStream_t st) {
    constexpr unsigned T = 256;
    const unsigned grid = unsigned((uint64_t(n) + T - 1) / T);
    if (reach == 1) k_force_masked<1><<<grid, T, 0, st>>>(B, perm, G, n, M, a, du);
    else k_force_masked<2><<<grid, T, 0, st>>>(B, perm, G, n, M, a, du);
}

// (v, P/rho^2) of a packed block, in its cell-sorted order; rho == 0 sets *zero
template <int P>
__global__ void k_pack_vel(const void* __restrict__ v, const void* __restrict__ rho, const void* __restrict__ pr,
                           const int32_t* __restrict__ perm, uint64_t n, float4* __restrict__ vel,
                           unsigned* __restrict__ zero) {
    bool z = false;
    for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < n; k += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = perm ? uint64_t(perm[k]) : k;
        const float ri = ldf<P>(rho, i);
        vel[k] = make_float4(ldf<P>(v, 3 * i), ldf<P>(v, 3 * i + 1), ldf<P>(v, 3 * i + 2), ldf<P>(pr, i) / (ri * ri));
        z |= ri == 0.0f;
    }
    if (__any_sync(0xffffffffu, z) && (threadIdx.x & 31) == 0) atomicOr(zero, 1u);
}

void force_cells(const void* x, const void* v, const void* m, const void* h, const void* rho, const void* pr,
                 int prec, uint64_t n, const int32_t* perm, const int32_t* cell_start, const float* lo, float cell,
                 int nx, int ny, int nz, int reach, uint64_t n_home, float* a, float* du, cudaStream_t st) {
    require_device();
    if (nx <= 0 || ny <= 0 || nz <= 0 || n_home > n || reach < 1 || reach > 4)
        throw std::invalid_argument("bad cell grid");
    if (n >= (1ull << 31)) throw std::invalid_argument("force_cells: n must be < 2^31 per device");
    if (int64_t(nx) * ny * nz >= (1ll << 31)) throw std::invalid_argument("bad cell grid");
    if (n == 0) return;
    const int sp = (prec == 1 || prec == 32) ? SP_F32 : prec == 16 ? SP_F16 : prec == 100 ? SP_BF16 : -1;
    if (sp < 0) throw std::invalid_argument("force_cells precision must be SF_PREC_NATIVE (fp32), 16 or SF_PREC_BF16");
    float4 *pos = nullptr, *vel = nullptr;
    float* hs = nullptr;
    check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&pos), 32 * n, st), "cudaMallocAsync");
    check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&hs), 4 * n + 16, st), "cudaMallocAsync");
    vel = pos + n;
    unsigned* words = reinterpret_cast<unsigned*>(hs + n);  // [0], [1] h range (h_range), [2] rho == 0 flag
    check_cuda(cudaMemsetAsync(words, 0, 3 * sizeof(unsigned), st), "memset");
    const unsigned blocks = unsigned(std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * 16));
    if (sp == SP_F32) k_pack_force<SP_F32><<<blocks, 256, 0, st>>>(x, v, m, h, rho, pr, perm, n, pos, vel, hs, words, words + 2);
    else if (sp == SP_F16) k_pack_force<SP_F16><<<blocks, 256, 0, st>>>(x, v, m, h, rho, pr, perm, n, pos, vel, hs, words, words + 2);
    else k_pack_force<SP_BF16><<<blocks, 256, 0, st>>>(x, v, m, h, rho, pr, perm, n, pos, vel, hs, words, words + 2);
    unsigned flag = 0;
    check_cuda(cudaMemcpyAsync(&flag, words + 2, sizeof(unsigned), cudaMemcpyDeviceToHost, st), "D2H");
    check_cuda(cudaStreamSynchronize(st), "sync");
    if (flag) {
        cudaFreeAsync(pos, st);
        cudaFreeAsync(hs, st);
        throw std::domain_error("force: degenerate state, rho == 0");
    }
    CellGrid G{lo[0], lo[1], lo[2], 1.0f / cell, nx, ny, nz, reach, int64_t(n_home)};
    ForceBlockSet B{};
    B.b[0] = ForceBlock{pos, vel, hs, cell_start, words, 0, nx, lo[0]};
    B.nb = 1;
    B.NX = nx;
    launch_force(B, perm, G, int64_t(n), reach, a, du, st);
    check_cuda(cudaGetLastError(), "force_cells launch");
    count_launches(2);
    check_cuda(cudaFreeAsync(pos, st), "cudaFreeAsync");
    check_cuda(cudaFreeAsync(hs, st), "cudaFreeAsync");
}

// (v, m) and P/rho^2 into a block, stream-ordered: rho == 0 anywhere sets *zero (no host sync)
void force_pack_async(const void* v, const void* rho, const void* pr, int prec, uint64_t n, const int32_t* perm,
                      void* vel, unsigned* zero, cudaStream_t st) {
    require_device();
    if (n >= (1ull << 31)) throw std::invalid_argument("force_pack: n must be < 2^31 per device");
    const int sp = (prec == 1 || prec == 32) ? SP_F32 : prec == 16 ? SP_F16 : prec == 100 ? SP_BF16 : -1;
    if (sp < 0) throw std::invalid_argument("force_pack precision must be SF_PREC_NATIVE (fp32), 16 or SF_PREC_BF16");
    if (n == 0) return;
    if (reinterpret_cast<uintptr_t>(vel) & 15) throw std::invalid_argument("vel must be 16-byte aligned");
    float4* v4 = static_cast<float4*>(vel);
    const unsigned blocks = unsigned(std::min<uint64_t>((n + 255) / 256, uint64_t(num_sms()) * 16));
    if (sp == SP_F32) k_pack_vel<SP_F32><<<blocks, 256, 0, st>>>(v, rho, pr, perm, n, v4, zero);
    else if (sp == SP_F16) k_pack_vel<SP_F16><<<blocks, 256, 0, st>>>(v, rho, pr, perm, n, v4, zero);
    else k_pack_vel<SP_BF16><<<blocks, 256, 0, st>>>(v, rho, pr, perm, n, v4, zero);
    check_cuda(cudaGetLastError(), "force_pack launch");
    count_launches(1);
}

void force_pack(const void* v, const void* rho, const void* pr, int prec, uint64_t n, const int32_t* perm, void* vel,
                cudaStream_t st) {
    require_device();
    if (n == 0) return;
    unsigned* zero = nullptr;
    check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&zero), sizeof(unsigned), st), "cudaMallocAsync");
    check_cuda(cudaMemsetAsync(zero, 0, sizeof(unsigned), st), "memset");
    force_pack_async(v, rho, pr, prec, n, perm, vel, zero, st);
    unsigned flag = 0;
    check_cuda(cudaMemcpyAsync(&flag, zero, sizeof(unsigned), cudaMemcpyDeviceToHost, st), "D2H");
    check_cuda(cudaFreeAsync(zero, st), "cudaFreeAsync");
    check_cuda(cudaStreamSynchronize(st), "sync");
    if (flag) throw std::domain_error("force: degenerate state, rho == 0");
}

void force_cells_blocks(const ForceBlockDesc* blocks, int nb, uint64_t n, const int32_t* perm, uint64_t n_home,
                        const float* lo_yz, float cell, int NX, int ny, int nz, int reach, float* a, float* du,
                        cudaStream_t st, const int32_t* win) {
    require_device();
    if (nb < 1 || nb > 3 || NX <= 0 || ny <= 0 || nz <= 0 || n_home > n || reach < 1 || reach > 4 || !(cell > 0))
        throw std::invalid_argument("bad cell grid");
    if (n >= (1ull << 31)) throw std::invalid_argument("force_cells: n must be < 2^31 per device");
    ForceBlockSet B{};
    B.nb = nb;
    B.NX = NX;
    for (int g = 0; g < nb; ++g) {
        const ForceBlockDesc& d = blocks[g];
        if (!d.pos || !d.vel || !d.h || !d.cell_start || !d.hmax) throw std::invalid_argument("null block pointer");
        if (d.nx <= 0 || d.x0 < 0 || d.x0 + d.nx > NX || int64_t(d.nx) * ny * nz >= (1ll << 31))
            throw std::invalid_argument("block layers outside the grid");
        B.b[g] = ForceBlock{static_cast<const float4*>(d.pos), static_cast<const float4*>(d.vel), d.h, d.cell_start,
                            d.hmax, d.x0, d.nx, d.x_origin};
    }
    if (n == 0) return;
    CellGrid G{blocks[0].x_origin, lo_yz[0], lo_yz[1], 1.0f / cell, NX, ny, nz, reach, int64_t(n_home)};
    if (win && reach <= 2) {  // the window masks the density of this step wrote for the same blocks
        if (n >= (1ull << 30)) throw std::invalid_argument("window masks need fewer than 2^30 particles per block");
        int32_t* w = const_cast<int32_t*>(win);
        const WindowMasks M{reinterpret_cast<int2*>(w), reinterpret_cast<uint32_t*>(w) + window_mask_words(n, reach) - n,
                            int64_t(n)};
        launch_force_masked(B, perm, G, int64_t(n), reach, M, a, du, st);
    } else {
        launch_force(B, perm, G, int64_t(n), reach, a, du, st);
    }
    check_cuda(cudaGetLastError(), "force_cells_blocks launch");
    count_launches(1);
}

// ------------------------------------------------------------------ binning
// Pass 1: cell id of every particle and its slot among the particles of its
// cell (the value its cell counter had when it arrived: one returning atomic
// per (warp, cell), lanes of one cell take consecutive slots in lane order).
__global__ void k_cell_rank(const float* __restrict__ x, uint64_t n, float lox, float loy, float loz, float inv_cell,
                            int nx, int ny, int nz, int32_t* __restrict__ cid, int32_t* __restrict__ rank,
                            int32_t* __restrict__ counts) {
    const int lane = threadIdx.x & 31;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        int cx = int(floorf((x[3 * i] - lox) * inv_cell));
        int cy = int(floorf((x[3 * i + 1] - loy) * inv_cell));
        int cz = int(floorf((x[3 * i + 2] - loz) * inv_cell));
        cx = min(max(cx, 0), nx - 1);
        cy = min(max(cy, 0), ny - 1);
        cz = min(max(cz, 0), nz - 1);
        const int c = (cx * ny + cy) * nz + cz;
        const unsigned peers = __match_any_sync(__activemask(), c);
        const int leader = __ffs(peers) - 1;
        int base = 0;
        if (lane == leader) base = atomicAdd(&counts[c], __popc(peers));
        base = __shfl_sync(peers, base, leader);
        cid[i] = c;
        rank[i] = base + __popc(peers & ((1u << lane) - 1));
    }
}

// Exclusive scan, reduce-then-scan over tiles of kScanTile ints: per-tile
// sums, a scan of the sums (recursively), then each tile scanned in shared
// memory (coalesced striped loads/stores, 16 consecutive values per thread,
// warp-shuffle scan of the thread totals) with its tile offset added.
constexpr int kScanT = 256, kScanV = 16, kScanTile = kScanT * kScanV;

__device__ __forceinline__ int block_exclusive_sum(int v, int* warp_tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += t;
    }
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        int w = lane < kScanT / 32 ? warp_tot[lane] : 0, wi = w;
#pragma unroll
        for (int d = 1; d < kScanT / 32; d <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, wi, d);
            if (lane >= d) wi += t;
        }
        if (lane < kScanT / 32) warp_tot[lane] = wi - w;  // exclusive warp offsets
    }
    __syncthreads();
    return warp_tot[warp] + inc - v;
}

__global__ void __launch_bounds__(kScanT) k_scan_reduce(const int32_t* __restrict__ a, int64_t n,
                                                        int32_t* __restrict__ partial) {
    __shared__ int warp_tot[kScanT / 32];
    const int64_t base = int64_t(blockIdx.x) * kScanTile;
    int sum = 0;
#pragma unroll
    for (int k = 0; k < kScanV; ++k) {
        const int64_t i = base + k * kScanT + threadIdx.x;
        if (i < n) sum += a[i];
    }
    const int excl = block_exclusive_sum(sum, warp_tot);
    if (threadIdx.x == kScanT - 1) partial[blockIdx.x] = excl + sum;
}

__global__ void __launch_bounds__(kScanT) k_scan_apply(int32_t* __restrict__ a, int64_t n,
                                                       const int32_t* __restrict__ offs) {
    __shared__ int sm[kScanTile + kScanTile / 32];
    __shared__ int warp_tot[kScanT / 32];
    const int64_t base = int64_t(blockIdx.x) * kScanTile;
    const int t = threadIdx.x;
#pragma unroll
    for (int k = 0; k < kScanV; ++k) {
        const int i = k * kScanT + t;
        sm[i + (i >> 5)] = base + i < n ? a[base + i] : 0;
    }
    __syncthreads();
    int v[kScanV], tot = 0;
#pragma unroll
    for (int k = 0; k < kScanV; ++k) {
        const int i = t * kScanV + k;
        v[k] = tot;
        tot += sm[i + (i >> 5)];
    }
    const int excl = block_exclusive_sum(tot, warp_tot) + (offs ? offs[blockIdx.x] : 0);
#pragma unroll
    for (int k = 0; k < kScanV; ++k) {
        const int i = t * kScanV + k;
        sm[i + (i >> 5)] = v[k] + excl;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kScanV; ++k) {
        const int i = k * kScanT + t;
        if (base + i < n) a[base + i] = sm[i + (i >> 5)];
    }
}

// scratch: >= ceil(n / kScanTile) ints, plus the same again for every level above
static void exclusive_scan(int32_t* a, int64_t n, int32_t* scratch, cudaStream_t st) {
    const int64_t tiles = (n + kScanTile - 1) / kScanTile;
    if (tiles > 1) {
        k_scan_reduce<<<unsigned(tiles), kScanT, 0, st>>>(a, n, scratch);
        exclusive_scan(scratch, tiles, scratch + ((tiles + 63) / 64) * 64, st);
        count_launches(1);
    }
    k_scan_apply<<<unsigned(tiles), kScanT, 0, st>>>(a, n, tiles > 1 ? scratch : nullptr);
    count_launches(1);
}

void exclusive_scan_i32(int32_t* a, int64_t n, int32_t* scratch, cudaStream_t st) { exclusive_scan(a, n, scratch, st); }
uint64_t scan_scratch_bytes(int64_t n) { return 4 * (2 * (uint64_t(n) / kScanTile + 64) + 64) + 256; }

// Pass 2: every particle to its slot, no atomics.
__global__ void k_place(const int32_t* __restrict__ cid, const int32_t* __restrict__ rank, uint64_t n,
                        const int32_t* __restrict__ start, int32_t* __restrict__ perm) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        perm[start[cid[i]] + rank[i]] = int32_t(i);
}

// Sort a run of <= N particle indices in registers: fully unrolled
// compare-exchange network (branchless min/max), padding with INT_MAX.
template <int N>
__device__ __forceinline__ void sort_run_regs(int32_t* __restrict__ perm, int b, int len) {
    int32_t a[N];
#pragma unroll
    for (int k = 0; k < N; ++k) a[k] = k < len ? perm[b + k] : 0x7fffffff;
#pragma unroll
    for (int i = 1; i < N; ++i)
#pragma unroll
        for (int j = i; j > 0; --j) {
            const int32_t lo = min(a[j - 1], a[j]), hi = max(a[j - 1], a[j]);
            a[j - 1] = lo;
            a[j] = hi;
        }
#pragma unroll
    for (int k = 0; k < N; ++k)
        if (k < len) perm[b + k] = a[k];
}

// make each cell's run ascending in particle index (deterministic order)
__global__ void k_sort_runs(const int32_t* __restrict__ start, int64_t ncell, int32_t* __restrict__ perm) {
    for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < ncell; c += int64_t(gridDim.x) * blockDim.x) {
        const int b = start[c], e = start[c + 1];
        const int len = e - b;
        if (len <= 1) continue;
        if (len <= 8) { sort_run_regs<8>(perm, b, len); continue; }
        if (len <= 24) { sort_run_regs<24>(perm, b, len); continue; }
        for (int i = b + 1; i < e; ++i) {
            const int32_t v = perm[i];
            int j = i - 1;
            while (j >= b && perm[j] > v) { perm[j + 1] = perm[j]; --j; }
            perm[j + 1] = v;
        }
    }
}

uint64_t bin_scratch_bytes(uint64_t n, int nx, int ny, int nz) {
    const uint64_t ncell = uint64_t(nx) * ny * nz;
    // cid[n] + rank[n] + scan partials (ncell / 4096 per level, 64-int padded)
    return 4 * (2 * n + 2 * (ncell / kScanTile + 64) + 64) + 256;
}

void bin_particles(const float* x, uint64_t n, const float* lo, float cell, int nx, int ny, int nz,
                   int32_t* cell_start, int32_t* perm, void* scratch, uint64_t scratch_bytes, cudaStream_t st) {
    require_device();
    if (n >= (1ull << 31)) throw std::invalid_argument("bin_particles: n must be < 2^31 per device");
    const int64_t ncell = int64_t(nx) * ny * nz;
    if (ncell <= 0 || ncell >= (1ll << 31)) throw std::invalid_argument("bad cell grid");
    if (scratch_bytes < bin_scratch_bytes(n, nx, ny, nz)) throw std::invalid_argument("bin scratch too small");
    int32_t* cid = static_cast<int32_t*>(scratch);
    int32_t* rank = cid + n;
    int32_t* scan_tmp = rank + ((n + 63) / 64) * 64;
    check_cuda(cudaMemsetAsync(cell_start, 0, sizeof(int32_t) * (ncell + 1), st), "memset");
    // uncapped grids: the CTAs in flight touch one compact range of particles
    // (and, for cell-sorted input, of cells)
    const unsigned blocks = unsigned((n + 255) / 256);
    if (n) {
        k_cell_rank<<<blocks, 256, 0, st>>>(x, n, lo[0], lo[1], lo[2], 1.0f / cell, nx, ny, nz, cid, rank, cell_start);
        count_launches(1);
    }
    exclusive_scan(cell_start, ncell + 1, scan_tmp, st);  // counts -> starts (last entry = n)
    if (n) {
        k_place<<<blocks, 256, 0, st>>>(cid, rank, n, cell_start, perm);
        k_sort_runs<<<unsigned((ncell + 255) / 256), 256, 0, st>>>(cell_start, ncell, perm);
        count_launches(2);
    }
    check_cuda(cudaGetLastError(), "bin launch");
}

}  // namespace sfb
