#include "commands.hpp"

#include <fstream>
#include <stdexcept>

#include "schema.hpp"

namespace sfb {

static const char* kVariants[] = {"cpu-baseline", "cpu-unpack", "cpu-soa", "dev-native",
                                  "dev-unpack", "dev-soa", "host-unpack-stream", "host-soa-stream"};
static const char* kKernels[] = {"density", "force", "kick", "drift", "identity"};

template <size_t N>
static void require_member(const std::string& v, const char* (&set)[N], const char* what) {
    for (const char* s : set)
        if (v == s) return;
    throw std::invalid_argument(std::string("unknown ") + what + " '" + v + "'");
}

void config_set_string(RunConfig& c, const std::string& k, const std::string& v) {
    if (k == "schema") c.schema_path = v;
    else if (k == "ic-csv") c.ic_csv_path = v;
    else if (k == "out") c.out_path = v;
    else if (k == "variants") {
        c.variants.clear();
        for (const auto& s : split_names(v)) { require_member(s, kVariants, "pipeline variant"); c.variants.push_back(s); }
    } else if (k == "modes") {
        c.modes.clear();
        for (const auto& s : split_names(v)) {
            if (s != "inplace" && s != "streaming") throw std::invalid_argument("unknown execution mode '" + s + "'");
            c.modes.push_back(s);
        }
    } else if (k == "kernels") {
        c.kernels.clear();
        for (const auto& s : split_names(v)) { require_member(s, kKernels, "kernel"); c.kernels.push_back(s); }
    } else if (k == "writeback") {
        if (v == "deferred") c.per_access = false;
        else if (v == "per-access") c.per_access = true;
        else throw std::invalid_argument("unknown writeback policy: " + v);
    } else if (k == "precision") {
        c.precision_sweep.clear();
        for (const auto& s : split_names(v)) c.precision_sweep.push_back(std::stoi(s));
    } else {
        throw std::invalid_argument("unknown string key: " + k);
    }
}

void config_set_int(RunConfig& c, const std::string& k, int64_t v) {
    if (k == "particles" && v > 0) c.particles = uint64_t(v);
    else if (k == "buffer-size" && v > 0) c.buffer_size = uint64_t(v);
    else if (k == "seed" && v >= 0) c.seed = uint64_t(v);
    else if (k == "threads" && v >= 0) c.threads = int(v);
    else if (k == "fault") c.fault = v != 0;
    else if (k == "dump") c.dump = v != 0;
    else throw std::invalid_argument("unknown integer key or bad value: " + k);
}

void config_set_double(RunConfig& c, const std::string& k, double v) {
    if (k == "dt") c.dt = v;
    else if (k == "latency" && v >= 0) c.latency_s = v;
    else if (k == "bandwidth" && v > 0) c.bandwidth = v;
    else throw std::invalid_argument("unknown real key or bad value: " + k);
}

void write_output(const RunConfig& c, const std::string& text) {
    if (c.out_path.empty()) return;
    std::ofstream o(c.out_path);
    if (!o) throw std::runtime_error("cannot write output file: " + c.out_path);
    o << text;
}

}  // namespace sfb
