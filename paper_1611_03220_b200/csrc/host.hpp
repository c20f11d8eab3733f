// Pure host-side pieces (no CUDA): reference-identical RNG draws, synthetic config
// generators, the symmetric super-tile schedule.
#pragma once

#include <stdint.h>

#include <vector>

namespace krr {

// RffMap ctor (sketches.cpp:24-35) seeded by stage_seed(master, 0) (sketches.cpp:18-20).
void rff_realize(uint64_t master_seed, int64_t d, int64_t s, double sigma, double* W, double* b);

// SURVEY 8f4 sketch-stage tables, drawn with the reference's libstdc++ distributions in
// its fixed order; `seed` is the map's own seed (realize_chain applies stage_seed).
// TensorSketchMap ctor (sketches.cpp:51-69): per mode the hash table, then the sign table.
void tensorsketch_realize(uint64_t seed, int64_t in_dim, int64_t s, int degree, uint32_t* hash, double* sign);
// SrhtMap ctor (sketches.cpp:95-109): next_pow2(in_dim) signs, then s rows with replacement.
void srht_realize(uint64_t seed, int64_t in_dim, int64_t s, double* sign, int64_t* rows);
// GaussianMap ctor (sketches.cpp:128-135): s x in_dim standard normals, row by row.
void gaussmap_realize(uint64_t seed, int64_t in_dim, int64_t s, double* proj);
// stage_seed (sketches.cpp:18-20).
uint64_t stage_seed(uint64_t master, int stage);
int64_t next_pow2(int64_t m);
// The radix-2 transform's twiddles, stage by stage (stage of length len at offset
// len/2 - 1; P - 1 complex values as re/im pairs): w_0 = 1, w_{j+1} = w_j * polar(1, ang)
// with ang = -+2 pi / len, the recurrence numerics.cpp:28-40 runs.
void fft_twiddles(int64_t P, bool inverse, double* out);

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
    int family = 0;  // 0 Gaussian (sigma), 1 polynomial (gamma, offset, degree)
    double sigma = 0, gamma = 0, offset = 0;
    int degree = 0;
    double lambda = 0;
    uint64_t seed = 0;
    std::vector<double> label_map;
};
// family 0: sigma; family 1: gamma, offset, degree (io.cpp:73-80 kernel_to_json).
void model_save(const char* path, int family, double sigma, double gamma, double offset, int degree, double lambda,
                uint64_t seed, const double* label_map, int64_t nlabels, const double* X, int64_t n, int64_t d,
                const double* C, int64_t t);
ModelMeta model_info(const char* path);
void model_load(const char* path, double* label_map, double* X, double* C);

}  // namespace krr
