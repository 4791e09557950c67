// Cell-linked SPH density (north-star "density cell-pair neighbour loop").
//
// New algorithm relative to the reference (whose density is all-pairs inside
// contiguous 64-particle buffers, sph.cpp:176-199): particles are counting-
// sorted into cells of side >= 2h; each home cell's 27-cell neighbourhood is
// 9 contiguous runs of the sorted arrays (z fastest), staged once per warp
// into shared memory as fp32 (x, y, z, m, h), then every home particle's sum
// is split across the 32 lanes and reduced with warp shuffles.  Pair formula:
// the reference's m_j * W(|x_i - x_j|, (h_i + h_j)/2), M4 spline, sigma=1/pi.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <stdexcept>
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

constexpr int kCellWarps = 4;
constexpr int kCand = 512;  // candidates staged per warp per batch

// M4 cubic spline (sph.cpp:17-24) in binary32; caller guarantees q < 2.
__device__ __forceinline__ float w_f32(float q, float inv_h) {
    const float norm = 0.31830988618379067f * inv_h * inv_h * inv_h;
    if (q < 1.0f) return norm * (1.0f - 1.5f * q * q + 0.75f * q * q * q);
    const float t = 2.0f - q;
    return norm * 0.25f * t * t * t;
}

template <int P>
__global__ void __launch_bounds__(kCellWarps * 32) k_density_cells(const void* __restrict__ x, const void* __restrict__ m,
                                                                   const void* __restrict__ h,
                                                                   const int32_t* __restrict__ cell_start, int nx, int ny,
                                                                   int nz, int own_x0, int own_x1,
                                                                   float* __restrict__ rho) {
    __shared__ float4 s_pos[kCellWarps][kCand];  // x, y, z, m
    __shared__ float s_h[kCellWarps][kCand];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t ncell_own = int64_t(own_x1 - own_x0) * ny * nz;
    for (int64_t wc = int64_t(blockIdx.x) * kCellWarps + warp; wc < ncell_own; wc += int64_t(gridDim.x) * kCellWarps) {
        const int ix = own_x0 + int(wc / (int64_t(ny) * nz));
        const int rem = int(wc % (int64_t(ny) * nz));
        const int iy = rem / nz, iz = rem % nz;
        const int64_t home = (int64_t(ix) * ny + iy) * nz + iz;
        const int hb = cell_start[home], he = cell_start[home + 1];
        if (hb == he) continue;
        // the 9 contiguous (dx, dy) runs covering z-1..z+1
        int rb[9], re[9], tot = 0;
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            const int jx = ix + k / 3 - 1, jy = iy + k % 3 - 1;
            rb[k] = re[k] = 0;
            if (jx < 0 || jx >= nx || jy < 0 || jy >= ny) continue;
            const int64_t c0 = (int64_t(jx) * ny + jy) * nz;
            rb[k] = cell_start[c0 + max(iz - 1, 0)];
            re[k] = cell_start[c0 + min(iz + 1, nz - 1) + 1];
            tot += re[k] - rb[k];
        }
        for (int i = hb; i < he; ++i) {
            // (the candidate set is staged once per batch; with one batch —
            // the common case — it is staged once per home cell)
            const float xi = ldf<P>(x, 3ull * i), yi = ldf<P>(x, 3ull * i + 1), zi = ldf<P>(x, 3ull * i + 2);
            const float hi = ldf<P>(h, i);
            float acc = 0.0f;
            for (int base = 0; base < tot; base += kCand) {
                const int cnt = min(kCand, tot - base);
                if (i == hb || tot > kCand) {
                    __syncwarp();
                    for (int c = lane; c < cnt; c += 32) {
                        int g = base + c, k = 0;
                        while (g >= re[k] - rb[k]) { g -= re[k] - rb[k]; ++k; }
                        const int j = rb[k] + g;
                        s_pos[warp][c] = make_float4(ldf<P>(x, 3ull * j), ldf<P>(x, 3ull * j + 1), ldf<P>(x, 3ull * j + 2),
                                                     ldf<P>(m, j));
                        s_h[warp][c] = ldf<P>(h, j);
                    }
                    __syncwarp();
                }
                for (int c = lane; c < cnt; c += 32) {
                    const float4 pj = s_pos[warp][c];
                    const float dx = xi - pj.x, dy = yi - pj.y, dz = zi - pj.z;
                    const float r2 = dx * dx + dy * dy + dz * dz;
                    const float hij = 0.5f * (hi + s_h[warp][c]);
                    if (r2 < 4.0f * hij * hij) {
                        const float inv_h = __frcp_rn(hij);
                        const float q = sqrtf(r2) * inv_h;
                        if (q < 2.0f) acc += pj.w * w_f32(q, inv_h);
                    }
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) rho[i] = acc;
        }
    }
}

void density_cells(const void* x, const void* m, const void* h, int prec, uint64_t n, const int32_t* cell_start,
                   int nx, int ny, int nz, int own_x0, int own_x1, float* rho, cudaStream_t st) {
    require_device();
    if (nx <= 0 || ny <= 0 || nz <= 0 || own_x0 < 0 || own_x1 > nx || own_x0 > own_x1)
        throw std::invalid_argument("bad cell grid");
    if (n >= (1ull << 31)) throw std::invalid_argument("density_cells: n must be < 2^31 per device");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t cells = int64_t(own_x1 - own_x0) * ny * nz;
    const int blocks = int(std::min<int64_t>((cells + kCellWarps - 1) / kCellWarps, int64_t(sms) * 8));
    if (blocks == 0) return;
    const int T = kCellWarps * 32;
    if (prec == 1 /*native fp32*/ || prec == 32)
        k_density_cells<SP_F32><<<blocks, T, 0, st>>>(x, m, h, cell_start, nx, ny, nz, own_x0, own_x1, rho);
    else if (prec == 16)
        k_density_cells<SP_F16><<<blocks, T, 0, st>>>(x, m, h, cell_start, nx, ny, nz, own_x0, own_x1, rho);
    else if (prec == 100)
        k_density_cells<SP_BF16><<<blocks, T, 0, st>>>(x, m, h, cell_start, nx, ny, nz, own_x0, own_x1, rho);
    else
        throw std::invalid_argument("density_cells precision must be SF_PREC_NATIVE (fp32), 16 or SF_PREC_BF16");
    check_cuda(cudaGetLastError(), "density_cells launch");
    count_launches(1);
}

// ------------------------------------------------------------------ binning
__global__ void k_cell_ids(const float* __restrict__ x, uint64_t n, float lox, float loy, float loz, float inv_cell,
                           int nx, int ny, int nz, int32_t* __restrict__ cid, int32_t* __restrict__ counts) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        int cx = int(floorf((x[3 * i] - lox) * inv_cell));
        int cy = int(floorf((x[3 * i + 1] - loy) * inv_cell));
        int cz = int(floorf((x[3 * i + 2] - loz) * inv_cell));
        cx = min(max(cx, 0), nx - 1);
        cy = min(max(cy, 0), ny - 1);
        cz = min(max(cz, 0), nz - 1);
        const int c = (cx * ny + cy) * nz + cz;
        cid[i] = c;
        atomicAdd(&counts[c], 1);
    }
}

constexpr int kScanBlock = 1024;

// in-place exclusive scan of each 2*kScanBlock segment; segment totals out
__global__ void k_scan_segments(int32_t* __restrict__ a, int64_t n, int32_t* __restrict__ totals) {
    __shared__ int32_t s[2 * kScanBlock];
    const int64_t seg0 = int64_t(blockIdx.x) * 2 * kScanBlock;
    const int t = threadIdx.x;
    for (int k = t; k < 2 * kScanBlock; k += kScanBlock) s[k] = seg0 + k < n ? a[seg0 + k] : 0;
    __syncthreads();
    // Blelloch up-sweep / down-sweep
    int off = 1;
    for (int d = kScanBlock; d > 0; d >>= 1) {
        __syncthreads();
        if (t < d) {
            const int ai = off * (2 * t + 1) - 1, bi = off * (2 * t + 2) - 1;
            s[bi] += s[ai];
        }
        off <<= 1;
    }
    if (t == 0) {
        totals[blockIdx.x] = s[2 * kScanBlock - 1];
        s[2 * kScanBlock - 1] = 0;
    }
    for (int d = 1; d <= kScanBlock; d <<= 1) {
        off >>= 1;
        __syncthreads();
        if (t < d) {
            const int ai = off * (2 * t + 1) - 1, bi = off * (2 * t + 2) - 1;
            const int32_t v = s[ai];
            s[ai] = s[bi];
            s[bi] += v;
        }
    }
    __syncthreads();
    for (int k = t; k < 2 * kScanBlock; k += kScanBlock)
        if (seg0 + k < n) a[seg0 + k] = s[k];
}

__global__ void k_add_offsets(int32_t* __restrict__ a, int64_t n, const int32_t* __restrict__ offs) {
    const int64_t seg = blockIdx.x;
    const int32_t o = offs[seg];
    for (int64_t k = seg * 2 * kScanBlock + threadIdx.x; k < min(n, (seg + 1) * 2 * kScanBlock); k += blockDim.x)
        a[k] += o;
}

static void exclusive_scan(int32_t* a, int64_t n, int32_t* scratch, cudaStream_t st) {
    const int64_t segs = (n + 2 * kScanBlock - 1) / (2 * kScanBlock);
    k_scan_segments<<<unsigned(segs), kScanBlock, 0, st>>>(a, n, scratch);
    count_launches(1);
    if (segs > 1) {
        exclusive_scan(scratch, segs, scratch + ((segs + 15) / 16) * 16, st);
        k_add_offsets<<<unsigned(segs), 256, 0, st>>>(a, n, scratch);
        count_launches(1);
    }
}

__global__ void k_place(const int32_t* __restrict__ cid, uint64_t n, const int32_t* __restrict__ start,
                        int32_t* __restrict__ fill, int32_t* __restrict__ perm) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const int c = cid[i];
        perm[start[c] + atomicAdd(&fill[c], 1)] = int32_t(i);
    }
}

// make each cell's run ascending in particle index (deterministic order)
__global__ void k_sort_runs(const int32_t* __restrict__ start, int64_t ncell, int32_t* __restrict__ perm) {
    for (int64_t c = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; c < ncell; c += int64_t(gridDim.x) * blockDim.x) {
        const int b = start[c], e = start[c + 1];
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
    // cid[n] + fill[ncell] + scan scratch (< ncell/1024 * 2 levels, padded)
    return 4 * (n + ncell + 2 * (ncell / 1024 + 64)) + 256;
}

void bin_particles(const float* x, uint64_t n, const float* lo, float cell, int nx, int ny, int nz,
                   int32_t* cell_start, int32_t* perm, void* scratch, uint64_t scratch_bytes, cudaStream_t st) {
    require_device();
    if (n >= (1ull << 31)) throw std::invalid_argument("bin_particles: n must be < 2^31 per device");
    const int64_t ncell = int64_t(nx) * ny * nz;
    if (ncell <= 0 || ncell >= (1ll << 31)) throw std::invalid_argument("bad cell grid");
    if (scratch_bytes < bin_scratch_bytes(n, nx, ny, nz)) throw std::invalid_argument("bin scratch too small");
    int32_t* cid = static_cast<int32_t*>(scratch);
    int32_t* fill = cid + n;
    int32_t* scan_tmp = fill + ncell;
    check_cuda(cudaMemsetAsync(cell_start, 0, sizeof(int32_t) * (ncell + 1), st), "memset");
    check_cuda(cudaMemsetAsync(fill, 0, sizeof(int32_t) * ncell, st), "memset");
    const unsigned blocks = unsigned(std::min<uint64_t>((n + 255) / 256 + 1, 148ull * 32));
    if (n) {
        k_cell_ids<<<blocks, 256, 0, st>>>(x, n, lo[0], lo[1], lo[2], 1.0f / cell, nx, ny, nz, cid, cell_start);
        count_launches(1);
    }
    exclusive_scan(cell_start, ncell + 1, scan_tmp, st);  // counts -> starts (last entry = n)
    if (n) {
        k_place<<<blocks, 256, 0, st>>>(cid, n, cell_start, fill, perm);
        k_sort_runs<<<unsigned(std::min<int64_t>((ncell + 255) / 256, 148ll * 32)), 256, 0, st>>>(cell_start, ncell, perm);
        count_launches(2);
    }
    check_cuda(cudaGetLastError(), "bin launch");
}

}  // namespace sfb
