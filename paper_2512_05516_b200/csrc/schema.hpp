// Record-schema DSL and padding-free layout (host side).
//
// Same text format and semantics as the reference annotation layer
// (proj/include/soaforge/schema.hpp:12-21, grammar SPEC.md:204):
//
//   schema particle {
//     field x : f64 x3;
//     field rho : f32 @truncate(16);   # comment
//   }
//   kernel density reads x, m, h writes rho;
//
// @truncate(N) means N = total stored bits.  Fields are packed
// in declaration order with no padding (schema.cpp:216-224).
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace sfb {

struct ParseError : std::runtime_error {
    int line, column;
    ParseError(const std::string& msg, int l, int c)
        : std::runtime_error(std::to_string(l) + ":" + std::to_string(c) + ": " + msg), line(l), column(c) {}
};

enum class Kind : uint8_t { F32, F64, I64 };

struct FieldDecl {
    std::string name;
    Kind kind = Kind::F32;
    int arity = 1;
    int trunc = 0;  // 0: none

    bool is_float() const { return kind != Kind::I64; }
    int declared_width() const { return kind == Kind::F32 ? 32 : 64; }
    int stored_width() const { return trunc ? trunc : declared_width(); }
    // width once unpacked: the enclosing IEEE width (schema.hpp:48-51)
    int native_width() const {
        if (!is_float()) return 64;
        const int t = stored_width();
        return t >= 33 ? 64 : t >= 17 ? 32 : 16;
    }
};

struct KernelSet {
    std::string name;
    std::vector<std::string> reads, writes;
    bool touches(const std::string& f) const;
    bool writes_field(const std::string& f) const;
};

struct Schema {
    std::string name;
    std::vector<FieldDecl> fields;
    std::vector<uint64_t> offset_bits;  // per field, stored-width layout
    uint64_t record_bits = 0;
    std::vector<KernelSet> kernels;

    int index(std::string_view n) const;
    const KernelSet* kernel(std::string_view n) const;
    void layout();  // recompute offsets / record_bits
};

Schema parse_schema_text(std::string_view text);
std::string print_schema_text(const Schema& s);
// with_uniform_precision (schema.cpp:296-309)
Schema uniform_precision(const Schema& s, int total_bits, const std::vector<std::string>& exclude);
std::vector<std::string> split_names(const std::string& csv);

}  // namespace sfb
