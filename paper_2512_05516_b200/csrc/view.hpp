// Views: host descriptors of packed particle buffers living in device (or
// host/managed) memory.  A view is the B200 counterpart of the reference's
// PackedBuffer (proj/include/soaforge/layout_ops.hpp:76-98): schema, record
// count, layout (AoS | SoA), the field subset (declaration order) and one lane
// format per subset field.  Bytes live in caller-owned memory.
//
// Lane geometry (layout_ops.cpp:25-39): lane l of record r of subset field p
//   AoS:  r*record_bits + prefix(p) + l*width(p)
//   SoA:  stream_base(p) + (r*arity(p) + l)*width(p),
//         stream_base(p) = count * sum_{q<p} arity(q)*width(q)
#pragma once
#include <memory>
#include <string>
#include <vector>

#include "codec.cuh"
#include "plans.cuh"
#include "schema.hpp"

namespace sfb {

// precision codes accepted by sf_b200_view_create (see soaforge_b200.h)
constexpr int kPrecStored = 0;     // compressed stored widths (the AoS on disk)
constexpr int kPrecNative = 1;     // unpacked: enclosing IEEE widths (U)
constexpr int kPrecBF16 = 100;     // every non-excluded float lane as bfloat16
constexpr int kPrecPackedT = 1000; // 1000+T: compressed, uniform T-bit storage

struct View {
    std::shared_ptr<const Schema> schema;
    uint64_t count = 0;
    Layout layout = Layout::AoS;
    std::vector<int> subset;       // schema field indices, declaration order
    std::vector<LaneFmt> fmt;      // per subset position

    int pos_of(int field) const;
    int pos_of(const std::string& name) const;
    int arity(int pos) const { return schema->fields[subset[pos]].arity; }
    int width(int pos) const { return fmt[pos].width; }
    uint64_t record_bits() const;
    uint64_t total_bits() const { return record_bits() * count; }
    uint64_t total_bytes() const { return (total_bits() + 7) / 8; }
    uint64_t lane_base(int pos) const;    // bits
    uint64_t lane_stride(int pos) const;  // bits between consecutive records
    bool byte_aligned() const;            // every lane starts/ends on a byte
    Lanes lanes(int pos) const;
};

View make_view(std::shared_ptr<const Schema> s, const char* access_set, Layout layout,
               int precision, const std::vector<std::string>& exclude, uint64_t count);

// Plans (validated on the host, executed by kernels.cu).
ConvertPlan plan_convert(const View& src, const View& dst, const std::vector<int>& fields);
GatherPlan plan_gather(const View& src, const View& dst);
KernelPlan plan_kernel(const View& v, const std::string& kernel, double dt, int math);
// fused gather + kernel: the kernel's operands are the *converted* lanes.
GatherPlan plan_gather_fused(const View& src, const View& dst, const std::string& kernel, double dt,
                             int math);
DensityPlan plan_density(const View& v, uint64_t buffer_size, int per_access);
ForcePlan plan_force(const View& v, uint64_t buffer_size, int per_access);

}  // namespace sfb
