#include "view.hpp"

#include <algorithm>
#include <numeric>
#include <stdexcept>

namespace sfb {

int View::pos_of(int field) const {
    for (size_t p = 0; p < subset.size(); ++p)
        if (subset[p] == field) return int(p);
    return -1;
}

int View::pos_of(const std::string& name) const { return pos_of(schema->index(name)); }

uint64_t View::record_bits() const {
    uint64_t b = 0;
    for (size_t p = 0; p < subset.size(); ++p) b += uint64_t(arity(int(p))) * width(int(p));
    return b;
}

uint64_t View::lane_base(int pos) const {
    uint64_t b = 0;
    for (int q = 0; q < pos; ++q) b += uint64_t(arity(q)) * width(q);
    return layout == Layout::AoS ? b : b * count;
}

uint64_t View::lane_stride(int pos) const {
    return layout == Layout::AoS ? record_bits() : uint64_t(arity(pos)) * width(pos);
}

bool View::byte_aligned() const {
    for (size_t p = 0; p < subset.size(); ++p)
        if ((lane_base(int(p)) | lane_stride(int(p)) | width(int(p))) & 7) return false;
    return true;
}

Lanes View::lanes(int pos) const {
    Lanes l;
    l.base = lane_base(pos);
    l.stride = lane_stride(pos);
    l.fmt = fmt[pos];
    l.arity = uint8_t(arity(pos));
    return l;
}

static LaneFmt stored_fmt(const FieldDecl& f) {
    return f.is_float() ? fmt_compressed(f.stored_width()) : fmt_int();
}

View make_view(std::shared_ptr<const Schema> s, const char* access_set, Layout layout,
               int precision, const std::vector<std::string>& exclude, uint64_t count) {
    View v;
    v.schema = s;
    v.count = count;
    v.layout = layout;
    const KernelSet* ks = nullptr;
    if (access_set && *access_set) {
        ks = s->kernel(access_set);
        if (!ks) throw std::invalid_argument(std::string("no access set declared for kernel '") + access_set + "'");
    }
    // narrow_into: reads ∪ writes in declaration order (layout_ops.cpp:86-101)
    for (size_t i = 0; i < s->fields.size(); ++i)
        if (!ks || ks->touches(s->fields[i].name)) v.subset.push_back(int(i));
    const bool ok_prec = precision == kPrecStored || precision == kPrecNative || precision == kPrecBF16 ||
                         (precision >= 7 && precision <= 64) ||
                         (precision >= kPrecPackedT + 7 && precision <= kPrecPackedT + 64);
    if (!ok_prec) throw std::invalid_argument("unknown precision code " + std::to_string(precision));
    for (int idx : v.subset) {
        const FieldDecl& f = s->fields[idx];
        const bool excluded = std::find(exclude.begin(), exclude.end(), f.name) != exclude.end();
        LaneFmt fm = stored_fmt(f);
        if (!f.is_float()) {
            v.fmt.push_back(fm);
            continue;
        }
        if (precision == kPrecNative) fm = fmt_native(f.stored_width());
        else if (precision == kPrecBF16) fm = excluded ? fmt_native(f.stored_width()) : fmt_bf16();
        else if (precision >= 7 && precision <= 64) fm = fmt_native(excluded ? f.stored_width() : precision);
        else if (precision >= kPrecPackedT) fm = fmt_compressed(excluded ? f.stored_width() : precision - kPrecPackedT);
        v.fmt.push_back(fm);
    }
    return v;
}

static void check_same_schema(const View& a, const View& b) {
    if (a.schema->fields.size() != b.schema->fields.size())
        throw std::invalid_argument("views over different schemas");
    for (size_t i = 0; i < a.schema->fields.size(); ++i)
        if (a.schema->fields[i].name != b.schema->fields[i].name ||
            a.schema->fields[i].arity != b.schema->fields[i].arity ||
            a.schema->fields[i].is_float() != b.schema->fields[i].is_float())
            throw std::invalid_argument("views over different schemas");
    if (a.count != b.count) throw std::invalid_argument("record count mismatch");
}

ConvertPlan plan_convert(const View& src, const View& dst, const std::vector<int>& fields) {
    check_same_schema(src, dst);
    if (fields.size() > size_t(kMaxStreams)) throw std::invalid_argument("too many fields for one plan");
    ConvertPlan p;
    p.count = src.count;
    p.dst_byte_aligned = dst.byte_aligned();
    for (int f : fields) {
        const int sp = src.pos_of(f), dp = dst.pos_of(f);
        if (sp < 0 || dp < 0)
            throw std::invalid_argument("field '" + src.schema->fields[f].name + "' missing from a view subset");
        CStream& c = p.s[p.n++];
        c.src = src.lanes(sp);
        c.dst = dst.lanes(dp);
        c.op = OP_COPY;
    }
    return p;
}

// Fast-path code of one gather stream: 1 + sb*12 + db*3 + ab, where
// sb in {f64, f32}, db in {f16, bf16, f32, f64}, ab in {none, f64, f32};
// 0 selects the generic path (truncated/bit-packed lanes, ints, odd shapes).
static uint8_t fast_kind(const GStream& s, uint32_t record_bits) {
    auto ieee = [](LaneFmt f) { return fmt_is_ieee(f); };
    auto src_idx = [](LaneFmt f) { return f.base == B_F64 ? 0 : f.base == B_F32 ? 1 : -1; };
    auto dst_idx = [](LaneFmt f) {
        return f.base == B_F16 ? 0 : f.base == B_BF16 ? 1 : f.base == B_F32 ? 2 : f.base == B_F64 ? 3 : -1;
    };
    auto aligned = [&](uint32_t off, LaneFmt f) { return off % f.width == 0 && record_bits % f.width == 0; };
    if (!ieee(s.src) || !ieee(s.dst) || src_idx(s.src) < 0 || dst_idx(s.dst) < 0) return 0;
    if (!aligned(s.src_off, s.src)) return 0;
    int ab = 0;
    if (s.op != OP_COPY) {
        if (!ieee(s.aux_src) || src_idx(s.aux_src) < 0 || !fmt_eq(s.aux_dst, s.dst) || !aligned(s.aux_off, s.aux_src))
            return 0;
        ab = 1 + src_idx(s.aux_src);
    }
    return uint8_t(1 + src_idx(s.src) * 12 + dst_idx(s.dst) * 3 + ab);
}

// Per-tile policy: PROC_XV_* for the drift-set shape (x: f64 x3, v: f32 x3,
// both narrowed to one IEEE format, x optionally drifted by v), else generic.
static uint8_t proc_kind(const GatherPlan& g) {
    if (g.n != 2 || g.tile_recs != 32 || g.record_bits % 64) return PROC_GENERIC;
    const GStream &x = g.s[0], &v = g.s[1];
    const bool x_ok = x.arity == 3 && fmt_is_ieee(x.src) && x.src.base == B_F64 && x.src_off % 64 == 0 &&
                      fmt_is_ieee(x.dst);
    const bool v_ok = v.arity == 3 && fmt_is_ieee(v.src) && v.src.base == B_F32 && v.src_off % 32 == 0 &&
                      v.op == OP_COPY && fmt_eq(v.dst, x.dst);
    const bool op_ok = x.op == OP_COPY ||
                       (x.op == OP_AXPY && x.aux_off == v.src_off && fmt_eq(x.aux_src, v.src) && fmt_eq(x.aux_dst, x.dst));
    if (!x_ok || !v_ok || !op_ok) return PROC_GENERIC;
    switch (x.dst.base) {
        case B_F16: return PROC_XV_F16;
        case B_BF16: return PROC_XV_BF16;
        case B_F32: return PROC_XV_F32;
        default: return PROC_GENERIC;
    }
}

static void finalize_fast(GatherPlan& g) {
    uint32_t out = 16;
    for (uint32_t i = 0; i < g.n; ++i) {
        g.s[i].fast = fast_kind(g.s[i], g.record_bits);
        out = std::max(out, g.tile_recs * g.s[i].arity * (g.s[i].dst.width / 8u));
    }
    g.proc = proc_kind(g);
    if (g.proc != PROC_GENERIC) out = 2 * g.tile_recs * 3 * (g.s[0].dst.width / 8u);  // x and v slices
    g.out_bytes = (out + 15) & ~15u;
}

GatherPlan plan_gather(const View& src, const View& dst) {
    check_same_schema(src, dst);
    if (src.layout != Layout::AoS || dst.layout != Layout::SoA)
        throw std::invalid_argument("tiled gather maps an AoS view to an SoA view");
    if (dst.subset.size() > size_t(kMaxStreams)) throw std::invalid_argument("too many streams");
    GatherPlan g;
    g.count = src.count;
    g.record_bits = uint32_t(src.record_bits());
    // warp tile: 32*R records, R the smallest with 32*R*record_bits % 128 == 0
    const uint32_t period = 128 / std::gcd(g.record_bits, 128u);  // records per 16-B step
    g.tile_recs = 32 * std::max<uint32_t>(1, period / 32);
    g.tile_bytes = uint32_t(g.tile_recs * uint64_t(g.record_bits) / 8);
    if (g.record_bits == 0) throw std::invalid_argument("empty record");
    for (size_t dp = 0; dp < dst.subset.size(); ++dp) {
        const int f = dst.subset[dp];
        const int sp = src.pos_of(f);
        if (sp < 0) throw std::invalid_argument("destination field missing from the source view");
        const int w = dst.width(int(dp));
        if (w != 16 && w != 32 && w != 64) throw std::invalid_argument("SoA gather needs 16/32/64-bit lanes");
        GStream& s = g.s[g.n++];
        s.src_off = uint32_t(src.lane_base(sp));
        s.src = src.fmt[sp];
        s.dst = dst.fmt[dp];
        s.dst_base = dst.lane_base(int(dp)) / 8;
        s.arity = uint8_t(dst.arity(int(dp)));
        s.op = OP_COPY;
    }
    finalize_fast(g);
    return g;
}

namespace {
struct OpSpec { const char* field; const char* operand; uint8_t op; };
const std::vector<OpSpec>& ops_for(const std::string& k) {
    // sph.cpp:247-264 — kick: v += a dt, u = max(0, u + du dt); drift: x += v dt
    static const std::vector<OpSpec> kick = {{"v", "a", OP_AXPY}, {"u", "du", OP_AXPY_CLAMP0}};
    static const std::vector<OpSpec> drift = {{"x", "v", OP_AXPY}};
    if (k == "kick") return kick;
    if (k == "drift") return drift;
    throw std::invalid_argument("kernel '" + k + "' is not a linear streaming kernel (kick|drift)");
}
}  // namespace

KernelPlan plan_kernel(const View& v, const std::string& kernel, double dt, int math) {
    KernelPlan p;
    p.count = v.count;
    p.dt = dt;
    p.math = uint8_t(math);
    p.dst_byte_aligned = v.byte_aligned();
    for (const auto& o : ops_for(kernel)) {
        const int xp = v.pos_of(o.field), yp = v.pos_of(o.operand);
        if (xp < 0 || yp < 0)
            throw std::invalid_argument(std::string("field '") + (xp < 0 ? o.field : o.operand) +
                                        "' is not present in the buffer view");
        CStream& c = p.s[p.n++];
        c.src = c.dst = v.lanes(xp);
        c.aux = v.lanes(yp);
        c.aux_q = v.fmt[yp];
        c.op = o.op;
    }
    return p;
}

GatherPlan plan_gather_fused(const View& src, const View& dst, const std::string& kernel, double dt,
                             int math) {
    GatherPlan g = plan_gather(src, dst);
    g.dt = dt;
    g.math = uint8_t(math);
    for (const auto& o : ops_for(kernel)) {
        const int xf = src.schema->index(o.field), yf = src.schema->index(o.operand);
        const int xd = dst.pos_of(xf), yd = dst.pos_of(yf), ys = src.pos_of(yf);
        if (xd < 0 || yd < 0 || ys < 0)
            throw std::invalid_argument(std::string("fused ") + kernel + " needs fields '" + o.field + "' and '" +
                                        o.operand + "' in both views");
        GStream& s = g.s[xd];
        s.op = o.op;
        s.aux_off = uint32_t(src.lane_base(ys));
        s.aux_src = src.fmt[ys];
        s.aux_dst = dst.fmt[yd];
    }
    finalize_fast(g);
    return g;
}

DensityPlan plan_density(const View& v, uint64_t bs, int per_access) {
    DensityPlan p;
    const int x = v.pos_of("x"), m = v.pos_of("m"), h = v.pos_of("h"), r = v.pos_of("rho");
    if (x < 0 || m < 0 || h < 0 || r < 0)
        throw std::invalid_argument("density needs fields x, m, h, rho in the buffer view");
    if (bs == 0 || bs > 1024 || v.count % bs != 0)
        throw std::invalid_argument("buffer size must divide the particle count (and be <= 1024)");
    p.x = v.lanes(x);
    p.m = v.lanes(m);
    p.h = v.lanes(h);
    p.rho = v.lanes(r);
    p.count = v.count;
    p.bs = uint32_t(bs);
    p.per_access = uint8_t(per_access != 0);
    return p;
}

}  // namespace sfb

namespace sfb {

ForcePlan plan_force(const View& v, uint64_t bs, int per_access) {
    ForcePlan p;
    const char* need[] = {"x", "v", "m", "h", "rho", "P", "a", "du"};
    Lanes* slot[] = {&p.x, &p.v, &p.m, &p.h, &p.rho, &p.P, &p.a, &p.du};
    for (int k = 0; k < 8; ++k) {
        const int pos = v.pos_of(need[k]);
        if (pos < 0) throw std::invalid_argument(std::string("field '") + need[k] + "' is not present in the buffer view");
        *slot[k] = v.lanes(pos);
    }
    if (bs == 0 || bs > 1024 || v.count % bs != 0)
        throw std::invalid_argument("buffer size must divide the particle count (and be <= 1024)");
    p.count = v.count;
    p.bs = uint32_t(bs);
    p.per_access = uint8_t(per_access != 0);
    p.byte_aligned = v.byte_aligned();
    return p;
}

}  // namespace sfb

