// One rank of the cell-sharded SPH timestep (shard.cu; sf_b200_shard_*).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

namespace sfb {

struct Shard;
Shard* shard_create(int rank, int world, int nc, double cell, int refine, uint64_t capacity);
void shard_destroy(Shard* s);
void shard_handle(Shard* s, uint8_t* out64);
void shard_connect(Shard* s, const uint8_t* handles);  // world x 64 bytes, rank order
void shard_load(Shard* s, const void* soa, uint64_t count, cudaStream_t st);
void* shard_field(Shard* s, const char* name, int* bytes_per_particle);
uint64_t shard_count(const Shard* s);
void shard_step(Shard* s, const std::vector<std::string>& kernels, double dt, cudaStream_t st, double* metrics);

}  // namespace sfb
