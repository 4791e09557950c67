// Host runtime behind the C ABI: validates views, builds plans, launches the
// sm_100a kernels on the caller's stream.  No CPU compute path exists: every
// entry requires a CUDA device and throws otherwise.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "plans.cuh"
#include "view.hpp"

namespace sfb {

// kernels.cu / density.cu launchers
// zero_copy: the host-memory side of the conversion is read / written in place over PCIe (pinned memory
// mapped into the device's address space): only the plan's lanes are touched, never whole records
cudaError_t launch_convert(const ConvertPlan& p, const void* src, void* dst, cudaStream_t st, bool zero_copy = false);
cudaError_t launch_gather(const GatherPlan& p, const void* src, uint64_t src_bytes, void* dst, cudaStream_t st,
                          bool zero_copy = false);
cudaError_t launch_density_buffer(const DensityPlan& p, void* buf, cudaStream_t st);
cudaError_t launch_update_rec(int xb, int yb, int arity, void* buf, uint64_t n, uint32_t stride, uint32_t xoff,
                              uint32_t yoff, double dt, uint8_t op, uint8_t math, cudaStream_t st);
cudaError_t launch_permute(const PermutePlan& p, const void* src, void* dst, const int32_t* perm, cudaStream_t st);
void permute(const View& v, const void* src, void* dst, const int32_t* perm, cudaStream_t st);
cudaError_t launch_update_rec_tile(void* buf, uint64_t n, uint32_t stride, const RecSeq& seq, double dt,
                                   uint8_t math, uint32_t wlo, uint32_t whi, cudaStream_t st);
cudaError_t launch_update_rec_multi(int xb, int yb, void* buf, uint64_t n, uint32_t stride, const RecOps& ops,
                                    double dt, uint8_t math, cudaStream_t st);
cudaError_t launch_update_soa(int xb, int yb, void* x, const void* y, uint64_t n, double dt, uint8_t op, uint8_t math,
                              cudaStream_t st);
cudaError_t launch_force_buffer(const ForcePlan& p, void* buf, cudaStream_t st, bool* degenerate);

void check_cuda(cudaError_t e, const char* what);
void require_device();
int num_sms();  // SM count of the current device
void count_launches(uint64_t n);
uint64_t launch_count();

void gather(const View& src, const void* sp, const View& dst, void* dp, const char* kernel, double dt, int math,
            cudaStream_t st, bool zero_copy = false);
void convert(const View& src, const void* sp, const View& dst, void* dp, cudaStream_t st);
void scatter_merge(const View& src, const void* sp, const View& dst, void* dp, const std::string& kernel,
                   cudaStream_t st, bool zero_copy = false);
void run_kernel(const View& v, void* p, const std::string& kernel, double dt, uint64_t bs, int per_access, int math,
                cudaStream_t st);
// the listed schema fields from src into dst (both views must hold them), nothing else
void convert_fields(const View& src, const void* sp, const View& dst, void* dp, const std::vector<int>& fields,
                    cudaStream_t st, bool zero_copy = false);

// density.cu
void density_cells(const void* x, const void* m, const void* h, int prec, uint64_t n, const int32_t* perm,
                   const int32_t* cell_start, const float* lo, float cell, int nx, int ny, int nz, int reach,
                   uint64_t n_home, float* rho, cudaStream_t st);
// one block of the multi-block density (sf_cell_block)
struct CellBlockDesc {
    const void* pos;   // float4 (x, y, z, m)
    const float* h;
    const int32_t* cell_start;
    const unsigned* hmax;
    int32_t x0, nx;
    float x_origin;
    int32_t reserved;
};
void cells_pack(const void* x, const void* m, const void* h, int prec, uint64_t n, const int32_t* perm, void* pos,
                float* hs, unsigned* hmax, cudaStream_t st);
// win (optional, window_mask_words(n, reach) 32-bit words, 8-byte aligned): every home's per-window
// in-support bit masks, written by the density for the force of the same step (force_cells_blocks(..., win)
// then sweeps exactly those pairs); used for reach <= 2, ignored above
void density_cells_blocks(const CellBlockDesc* blocks, int nb, uint64_t n, const int32_t* perm, uint64_t n_home,
                          const float* lo_yz, float cell, int NX, int ny, int nz, int reach, float* rho,
                          cudaStream_t st, int32_t* win = nullptr);
inline uint64_t window_mask_words(uint64_t n, int reach) {
    return (2 * uint64_t(2 * reach + 1) * (2 * reach + 1) + 1) * n;  // (base, bits) per window + occupancy
}
struct ForceBlockDesc {
    const void* pos;   // float4 (x, y, z, m): the density block's
    const void* vel;   // float4 (vx, vy, vz, P/rho^2)
    const float* h;
    const int32_t* cell_start;
    const unsigned* hmax;
    int32_t x0, nx;
    float x_origin;
    int32_t reserved;
};
void force_pack_async(const void* v, const void* rho, const void* pr, int prec, uint64_t n, const int32_t* perm,
                      void* vel, unsigned* zero, cudaStream_t st);
void force_pack(const void* v, const void* rho, const void* pr, int prec, uint64_t n, const int32_t* perm, void* vel,
                cudaStream_t st);
void force_cells_blocks(const ForceBlockDesc* blocks, int nb, uint64_t n, const int32_t* perm, uint64_t n_home,
                        const float* lo_yz, float cell, int NX, int ny, int nz, int reach, float* a, float* du,
                        cudaStream_t st, const int32_t* win = nullptr);
void force_cells(const void* x, const void* v, const void* m, const void* h, const void* rho, const void* pr,
                 int prec, uint64_t n, const int32_t* perm, const int32_t* cell_start, const float* lo, float cell,
                 int nx, int ny, int nz, int reach, uint64_t n_home, float* a, float* du, cudaStream_t st);
uint64_t bin_scratch_bytes(uint64_t n, int nx, int ny, int nz);
// exclusive prefix sum of n int32 in place (a[n-1] holds the last element's offset); scratch of scan_scratch_bytes
void exclusive_scan_i32(int32_t* a, int64_t n, int32_t* scratch, cudaStream_t st);
uint64_t scan_scratch_bytes(int64_t n);
void bin_particles(const float* x, uint64_t n, const float* lo, float cell, int nx, int ny, int nz,
                   int32_t* cell_start, int32_t* perm, void* scratch, uint64_t scratch_bytes, cudaStream_t st);

// host.cu
void run_host(const View& src, void* host, const View& dst, const std::string& kernels, double dt, int math,
              int mode, uint64_t chunk, void* host_soa, double* metrics);

}  // namespace sfb
