// Pure host-side pieces (no CUDA): reference-identical RNG draws, synthetic config
// generators, the symmetric super-tile schedule.
#pragma once

#include <stdint.h>

#include <vector>

namespace krr {

// RffMap ctor (sketches.cpp:24-35) seeded by stage_seed(master, 0) (sketches.cpp:18-20).
void rff_realize(uint64_t master_seed, int64_t d, int64_t s, double sigma, double* W, double* b);

// BASELINE.json configs 1-5, SURVEY.md §8d generators.
void generate_config(int cfg, int64_t n, int64_t d, int64_t t, uint64_t seed, double* X, double* Y);

// rlsc_encode (solver.cpp:152-161).
void rlsc_encode(const int32_t* classes, int64_t n, int32_t num_classes, double* Y);

struct Schedule {
    int64_t st = 0;       // super-tile edge (rows), multiple of 128
    int64_t ns = 0;       // number of super-rows
    int64_t n_pad = 0;    // ns * st
    std::vector<int32_t> tiles;   // flattened (a, b) pairs owned by the rank
    std::vector<uint8_t> owned;   // ns x ns, owned[x*ns + y] = 1 if tile {x, y} is ours
};
Schedule make_schedule(int64_t n, int world, int rank);

// Row shard of the sketch (Z / U) rows: contiguous blocks of ceil(n / world).
void shard_rows(int64_t n, int world, int rank, int64_t* z0, int64_t* z1);

// power_iteration_spectral_norm's start vector (numerics.cpp:160-164): mt19937_64(seed)
// normal(0, 1) draws, normalised.
void power_iteration_start(uint64_t seed, int64_t n, double* v);

// default_initial_sketch_size (precond.cpp:102-104): max(64, ceil(n / 64)).
int64_t default_initial_sketch_size(int64_t n);
// kAttemptSeedStride (sketches.hpp:16): adaptive attempt a uses master + a * stride.
constexpr uint64_t kAttemptSeedStride = 0xD1B54A32D192ED03ULL;

// KRRM model file (io.cpp:192-261), model_io.cpp.
struct ModelMeta {
    int64_t n = 0, d = 0, t = 0;
    double sigma = 0, lambda = 0;
    uint64_t seed = 0;
    std::vector<double> label_map;
};
void model_save(const char* path, double sigma, double lambda, uint64_t seed, const double* label_map,
                int64_t nlabels, const double* X, int64_t n, int64_t d, const double* C, int64_t t);
ModelMeta model_info(const char* path);
void model_load(const char* path, double* label_map, double* X, double* C);

}  // namespace krr
