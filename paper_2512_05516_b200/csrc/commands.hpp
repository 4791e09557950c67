// Run configuration and the batch commands behind sf_run_* (reference:
// bench.hpp:19-68, capi.cpp:123-198).  Same keys, defaults and validation;
// the conversions and kernels of every command execute on the GPU.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace sfb {

struct RunConfig {
    std::string schema_path, ic_csv_path, out_path;
    uint64_t particles = 4096;
    uint64_t buffer_size = 64;
    uint64_t seed = 42;
    std::vector<int> precision_sweep;
    std::vector<std::string> variants = {"cpu-baseline", "cpu-unpack", "cpu-soa", "dev-native",
                                         "dev-unpack", "dev-soa", "host-unpack-stream", "host-soa-stream"};
    std::vector<std::string> modes = {"inplace", "streaming"};
    std::vector<std::string> kernels = {"density", "force", "kick", "drift"};
    bool per_access = false;
    double latency_s = 5e-6, bandwidth = 64e9, dt = 1e-3;
    int threads = 0;
    bool fault = false, dump = false;
};

void config_set_string(RunConfig& c, const std::string& key, const std::string& value);
void config_set_int(RunConfig& c, const std::string& key, int64_t value);
void config_set_double(RunConfig& c, const std::string& key, double value);
void write_output(const RunConfig& c, const std::string& text);

std::string cmd_bench_transform(const RunConfig& c);
std::string cmd_bench_kernels(const RunConfig& c);
std::string cmd_bench_pipeline(const RunConfig& c);
std::string cmd_study_truncation(const RunConfig& c);
std::string cmd_validate(const RunConfig& c, int& failures);

}  // namespace sfb
