#include "schema.hpp"

#include <cctype>
#include <sstream>

namespace sfb {

bool KernelSet::touches(const std::string& f) const {
    for (const auto& r : reads) if (r == f) return true;
    return writes_field(f);
}
bool KernelSet::writes_field(const std::string& f) const {
    for (const auto& w : writes) if (w == f) return true;
    return false;
}

int Schema::index(std::string_view n) const {
    for (size_t i = 0; i < fields.size(); ++i)
        if (fields[i].name == n) return int(i);
    return -1;
}

const KernelSet* Schema::kernel(std::string_view n) const {
    for (const auto& k : kernels)
        if (k.name == n) return &k;
    return nullptr;
}

void Schema::layout() {
    offset_bits.assign(fields.size(), 0);
    uint64_t at = 0;
    for (size_t i = 0; i < fields.size(); ++i) {
        offset_bits[i] = at;
        at += uint64_t(fields[i].arity) * fields[i].stored_width();
    }
    record_bits = at;
}

namespace {

struct Tok {
    enum Type { Word, Int, Sym, Eof } type;
    std::string text;
    int line, col;
};

std::vector<Tok> tokenize(std::string_view s) {
    std::vector<Tok> out;
    int line = 1, col = 1;
    size_t i = 0;
    auto bump = [&](size_t n) { i += n; col += int(n); };
    while (i < s.size()) {
        const char c = s[i];
        if (c == '\n') { ++i; ++line; col = 1; continue; }
        if (std::isspace((unsigned char)c)) { bump(1); continue; }
        if (c == '#') { while (i < s.size() && s[i] != '\n') bump(1); continue; }
        Tok t{Tok::Sym, "", line, col};
        size_t j = i;
        if (std::isalpha((unsigned char)c) || c == '_') {
            while (j < s.size() && (std::isalnum((unsigned char)s[j]) || s[j] == '_')) ++j;
            t.type = Tok::Word;
        } else if (std::isdigit((unsigned char)c)) {
            while (j < s.size() && std::isdigit((unsigned char)s[j])) ++j;
            t.type = Tok::Int;
        } else {
            j = i + 1;
        }
        t.text = std::string(s.substr(i, j - i));
        bump(j - i);
        out.push_back(std::move(t));
    }
    out.push_back({Tok::Eof, "", line, col});
    return out;
}

class Parser {
public:
    explicit Parser(std::vector<Tok> toks) : t_(std::move(toks)) {}

    Schema run() {
        Schema s;
        bool seen = false;
        while (cur().type != Tok::Eof) {
            if (word("schema")) {
                if (seen) error("only one schema block per file");
                seen = true;
                schema_block(s);
            } else if (word("kernel")) {
                s.kernels.push_back(kernel_line());
            } else {
                error("expected 'schema' or 'kernel'");
            }
        }
        if (!seen) throw ParseError("no schema block found", 1, 1);
        s.layout();
        for (const auto& k : s.kernels)
            for (const auto* list : {&k.reads, &k.writes})
                for (const auto& n : *list)
                    if (s.index(n) < 0)
                        throw std::invalid_argument("kernel '" + k.name + "' names unknown field '" + n + "'");
        return s;
    }

private:
    const Tok& cur() const { return t_[p_]; }
    [[noreturn]] void error(const std::string& m) const { throw ParseError(m, cur().line, cur().col); }
    bool word(const char* w) {
        if (cur().type == Tok::Word && cur().text == w) { ++p_; return true; }
        return false;
    }
    bool sym(char c) {
        if (cur().type == Tok::Sym && cur().text[0] == c) { ++p_; return true; }
        return false;
    }
    void need(char c) { if (!sym(c)) error(std::string("expected '") + c + "'"); }
    Tok ident(const char* what) {
        if (cur().type != Tok::Word) error(std::string("expected ") + what);
        return t_[p_++];
    }

    void schema_block(Schema& s) {
        s.name = ident("schema name").text;
        need('{');
        while (!sym('}')) {
            if (cur().type == Tok::Eof) error("expected 'field' or '}'");
            const Tok kw = t_[p_++];
            if (kw.type != Tok::Word || kw.text != "field") throw ParseError("expected 'field' or '}'", kw.line, kw.col);
            const Tok at = cur();
            FieldDecl f = field_decl();
            if (s.index(f.name) >= 0) throw ParseError("duplicate field '" + f.name + "'", at.line, at.col);
            s.fields.push_back(std::move(f));
        }
    }

    FieldDecl field_decl() {
        FieldDecl f;
        f.name = ident("field name").text;
        need(':');
        const Tok k = ident("base kind (f32|f64|i64)");
        if (k.text == "f32") f.kind = Kind::F32;
        else if (k.text == "f64") f.kind = Kind::F64;
        else if (k.text == "i64") f.kind = Kind::I64;
        else throw ParseError("unknown base kind '" + k.text + "'", k.line, k.col);
        if (cur().type == Tok::Word && cur().text == "x3") { ++p_; f.arity = 3; }
        if (sym('@')) {
            const Tok a = ident("attribute");
            if (a.text != "truncate") throw ParseError("unknown attribute '@" + a.text + "'", a.line, a.col);
            need('(');
            const Tok n = t_[p_++];
            if (n.type != Tok::Int) throw ParseError("expected truncation width", n.line, n.col);
            if (!f.is_float()) throw ParseError("@truncate is not allowed on i64 field '" + f.name + "'", a.line, a.col);
            const long w = n.text.size() > 3 ? 999 : std::stol(n.text);
            if (w < 7 || w > 64) throw ParseError("truncation width " + n.text + " outside 7..64", n.line, n.col);
            f.trunc = int(w);
            need(')');
        }
        need(';');
        return f;
    }

    std::vector<std::string> name_list() {
        std::vector<std::string> v{ident("field name").text};
        for (;;) {
            if (sym(',')) { v.push_back(ident("field name").text); continue; }
            if (cur().type == Tok::Word && cur().text != "reads" && cur().text != "writes") {
                v.push_back(t_[p_++].text);
                continue;
            }
            return v;
        }
    }

    KernelSet kernel_line() {
        KernelSet k;
        k.name = ident("kernel name").text;
        if (word("reads")) k.reads = name_list();
        if (word("writes")) k.writes = name_list();
        if (k.reads.empty() && k.writes.empty()) error("kernel '" + k.name + "' declares neither reads nor writes");
        need(';');
        return k;
    }

    std::vector<Tok> t_;
    size_t p_ = 0;
};

}  // namespace

Schema parse_schema_text(std::string_view text) { return Parser(tokenize(text)).run(); }

std::string print_schema_text(const Schema& s) {
    std::ostringstream o;
    o << "schema " << s.name << " {\n";
    for (const auto& f : s.fields) {
        o << "  field " << f.name << " : " << (f.kind == Kind::F32 ? "f32" : f.kind == Kind::F64 ? "f64" : "i64");
        if (f.arity == 3) o << " x3";
        if (f.trunc) o << " @truncate(" << f.trunc << ")";
        o << ";\n";
    }
    o << "}\n";
    for (const auto& k : s.kernels) {
        o << "kernel " << k.name;
        const char* sep = " reads ";
        for (const auto& r : k.reads) { o << sep << r; sep = ", "; }
        sep = " writes ";
        for (const auto& w : k.writes) { o << sep << w; sep = ", "; }
        o << ";\n";
    }
    return o.str();
}

Schema uniform_precision(const Schema& s, int t, const std::vector<std::string>& exclude) {
    if (t < 7 || t > 64) throw std::invalid_argument("truncation width outside 7..64");
    Schema out = s;
    for (auto& f : out.fields) {
        if (!f.is_float()) continue;
        bool skip = false;
        for (const auto& e : exclude) skip |= e == f.name;
        if (!skip) f.trunc = t;
    }
    out.layout();
    return out;
}

std::vector<std::string> split_names(const std::string& csv) {
    std::vector<std::string> v;
    std::string cur;
    for (char c : csv) {
        if (c == ',' || std::isspace((unsigned char)c)) {
            if (!cur.empty()) v.push_back(cur);
            cur.clear();
        } else {
            cur += c;
        }
    }
    if (!cur.empty()) v.push_back(cur);
    return v;
}

}  // namespace sfb
