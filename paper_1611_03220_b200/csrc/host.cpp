// Host-side, CUDA-free pieces of the library.
#include "host.hpp"

#include <algorithm>
#include <cmath>
#include <complex>
#include <numbers>
#include <random>
#include <stdexcept>
#include <thread>

#include "../../include/krr_b200.h"

namespace krr {

namespace {
constexpr uint64_t kStageSeedStride = 0x9E3779B97F4A7C15ULL;  // sketches.hpp:14

template <class F>
void parallel_rows(int64_t n, F&& f) {
    unsigned nt = std::max(1u, std::thread::hardware_concurrency());
    nt = unsigned(std::min<int64_t>(nt, std::max<int64_t>(1, n / 1024)));
    if (nt <= 1) {
        f(int64_t(0), n);
        return;
    }
    std::vector<std::thread> th;
    const int64_t chunk = (n + nt - 1) / nt;
    for (unsigned k = 0; k < nt; ++k) {
        const int64_t a = k * chunk, b = std::min(n, a + chunk);
        if (a < b) th.emplace_back([&f, a, b] { f(a, b); });
    }
    for (auto& t : th) t.join();
}

// Column standardisation: mean 0, population std 1.
void standardise(double* X, int64_t n, int64_t d) {
    std::vector<double> mean(size_t(d), 0.0), var(size_t(d), 0.0);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < d; ++j) mean[size_t(j)] += X[i * d + j];
    for (int64_t j = 0; j < d; ++j) mean[size_t(j)] /= double(n);
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < d; ++j) {
            const double c = X[i * d + j] - mean[size_t(j)];
            var[size_t(j)] += c * c;
        }
    for (int64_t j = 0; j < d; ++j) {
        const double sd = std::sqrt(var[size_t(j)] / double(n));
        var[size_t(j)] = sd > 0.0 ? 1.0 / sd : 1.0;
    }
    parallel_rows(n, [&](int64_t a, int64_t b) {
        for (int64_t i = a; i < b; ++i)
            for (int64_t j = 0; j < d; ++j)
                X[i * d + j] = (X[i * d + j] - mean[size_t(j)]) * var[size_t(j)];
    });
}

double dotp(const double* a, const double* b, int64_t d) {
    double s = 0.0;
    for (int64_t k = 0; k < d; ++k) s += a[k] * b[k];
    return s;
}

// Householder QR of a d x d row-major matrix; returns Q (row-major) with the sign
// convention diag(R) > 0.
std::vector<double> householder_q(std::vector<double> a, int64_t d) {
    std::vector<double> q(size_t(d * d), 0.0);
    for (int64_t i = 0; i < d; ++i) q[size_t(i * d + i)] = 1.0;
    std::vector<double> v(static_cast<size_t>(d));
    
    for (int64_t k = 0; k < d; ++k) {
        double norm = 0.0;
        for (int64_t i = k; i < d; ++i) norm += a[size_t(i * d + k)] * a[size_t(i * d + k)];
        norm = std::sqrt(norm);
        if (norm == 0.0) continue;
        const double alpha = a[size_t(k * d + k)] > 0 ? -norm : norm;
        for (int64_t i = 0; i < d; ++i) v[size_t(i)] = 0.0;
        for (int64_t i = k; i < d; ++i) v[size_t(i)] = a[size_t(i * d + k)];
        v[size_t(k)] -= alpha;
        double vn = 0.0;
        for (int64_t i = k; i < d; ++i) vn += v[size_t(i)] * v[size_t(i)];
        if (vn == 0.0) continue;
        // A <- H A, Q <- Q H  (H = I - 2 v v^T / v^T v)
        for (int64_t j = 0; j < d; ++j) {
            double s = 0.0;
            for (int64_t i = k; i < d; ++i) s += v[size_t(i)] * a[size_t(i * d + j)];
            s = 2.0 * s / vn;
            for (int64_t i = k; i < d; ++i) a[size_t(i * d + j)] -= s * v[size_t(i)];
        }
        for (int64_t i = 0; i < d; ++i) {
            double s = 0.0;
            for (int64_t j = k; j < d; ++j) s += q[size_t(i * d + j)] * v[size_t(j)];
            s = 2.0 * s / vn;
            for (int64_t j = k; j < d; ++j) q[size_t(i * d + j)] -= s * v[size_t(j)];
        }
    }
    // Flip columns of Q where R's diagonal is negative.
    for (int64_t k = 0; k < d; ++k)
        if (a[size_t(k * d + k)] < 0.0)
            for (int64_t i = 0; i < d; ++i) q[size_t(i * d + k)] = -q[size_t(i * d + k)];
    return q;
}

}  // namespace

void rff_realize(uint64_t master_seed, int64_t d, int64_t s, double sigma, double* W, double* b) {
    if (s < 1) throw std::invalid_argument("RffMap: need at least one feature");
    if (!(sigma > 0.0)) throw std::invalid_argument("RffMap: sigma must be positive");
    std::mt19937_64 gen(master_seed + 1 * kStageSeedStride);
    std::normal_distribution<double> freq(0.0, 1.0 / sigma);
    std::uniform_real_distribution<double> phase(0.0, 2.0 * std::numbers::pi);
    for (int64_t i = 0; i < s; ++i)
        for (int64_t j = 0; j < d; ++j) W[i * d + j] = freq(gen);
    for (int64_t i = 0; i < s; ++i) b[i] = phase(gen);
}

uint64_t stage_seed(uint64_t master, int stage) { return master + uint64_t(stage + 1) * kStageSeedStride; }

int64_t next_pow2(int64_t m) {
    int64_t p = 1;
    while (p < m) p <<= 1;
    return p;
}

void tensorsketch_realize(uint64_t seed, int64_t in_dim, int64_t s, int degree, uint32_t* hash, double* sign) {
    if (s < 1) throw std::invalid_argument("TensorSketchMap: need at least one feature");
    if (degree < 1) throw std::invalid_argument("TensorSketchMap: degree must be >= 1");
    std::mt19937_64 gen(seed);
    std::uniform_int_distribution<uint32_t> bucket(0, uint32_t(s - 1));
    std::uniform_int_distribution<int> coin(0, 1);
    for (int q = 0; q < degree; ++q) {
        uint32_t* h = hash + int64_t(q) * in_dim;
        double* g = sign + int64_t(q) * in_dim;
        for (int64_t j = 0; j < in_dim; ++j) h[j] = bucket(gen);
        for (int64_t j = 0; j < in_dim; ++j) g[j] = coin(gen) ? 1.0 : -1.0;
    }
}

void srht_realize(uint64_t seed, int64_t in_dim, int64_t s, double* sign, int64_t* rows) {
    if (s < 1) throw std::invalid_argument("SrhtMap: need at least one feature");
    if (in_dim < 1) throw std::invalid_argument("SrhtMap: input dimension must be positive");
    const int64_t P = next_pow2(in_dim);
    std::mt19937_64 gen(seed);
    std::uniform_int_distribution<int> coin(0, 1);
    std::uniform_int_distribution<int64_t> pick(0, P - 1);
    for (int64_t i = 0; i < P; ++i) sign[i] = coin(gen) ? 1.0 : -1.0;
    for (int64_t i = 0; i < s; ++i) rows[i] = pick(gen);
}

void gaussmap_realize(uint64_t seed, int64_t in_dim, int64_t s, double* proj) {
    if (s < 1) throw std::invalid_argument("GaussianMap: need at least one feature");
    std::mt19937_64 gen(seed);
    std::normal_distribution<double> normal(0.0, 1.0);
    for (int64_t i = 0; i < s * in_dim; ++i) proj[i] = normal(gen);
}

void fft_twiddles(int64_t P, bool inverse, double* out) {
    for (int64_t len = 2; len <= P; len <<= 1) {
        const double ang = (inverse ? 2.0 : -2.0) * std::numbers::pi / double(len);
        const std::complex<double> step = std::polar(1.0, ang);
        std::complex<double> w(1.0, 0.0);
        double* o = out + 2 * (len / 2 - 1);
        for (int64_t j = 0; j < len / 2; ++j) {
            o[2 * j] = w.real();
            o[2 * j + 1] = w.imag();
            w *= step;
        }
    }
}

void rlsc_encode(const int32_t* classes, int64_t n, int32_t num_classes, double* Y) {
    if (num_classes < 2) throw std::invalid_argument("rlsc_encode: need at least two classes");
    for (int64_t i = 0; i < n; ++i) {
        const int32_t c = classes[i];
        if (c < 0 || c >= num_classes)
            throw std::invalid_argument("rlsc_encode: class index out of range");
        for (int32_t j = 0; j < num_classes; ++j) Y[i * num_classes + j] = -1.0;
        Y[i * num_classes + c] = 1.0;
    }
}

void generate_config(int cfg, int64_t n, int64_t d, int64_t t, uint64_t seed, double* X,
                     double* Y) {
    if (n < 1 || d < 1 || t < 1) throw std::invalid_argument("generate_config: bad shape");
    if (cfg == 1) {
        if (t != 1) throw std::invalid_argument("config 1 has one right-hand side");
        std::mt19937_64 g0(seed + 0), g1(seed + 1), g2(seed + 2);
        std::normal_distribution<double> n01(0.0, 1.0);
        for (int64_t i = 0; i < n * d; ++i) X[i] = n01(g0);
        std::normal_distribution<double> nw(0.0, 1.0 / std::sqrt(double(d)));
        std::vector<double> w(static_cast<size_t>(d));
        for (auto& x : w) x = nw(g1);
        for (int64_t i = 0; i < n; ++i) Y[i] = std::sin(dotp(w.data(), X + i * d, d)) + 0.1 * n01(g2);
    } else if (cfg == 2) {
        if (t != 1) throw std::invalid_argument("config 2 has one right-hand side");
        constexpr int K = 7;
        std::mt19937_64 g0(seed + 0), g1(seed + 1), g3(seed + 3), g4(seed + 4);
        std::normal_distribution<double> n01(0.0, 1.0), nc(0.0, 2.0);
        std::vector<double> c(static_cast<size_t>(K * d));
        for (auto& x : c) x = nc(g1);
        std::uniform_int_distribution<int> pick(0, K - 1);
        std::vector<int> k(static_cast<size_t>(n));
        for (auto& x : k) x = pick(g3);
        for (int64_t i = 0; i < n; ++i)
            for (int64_t j = 0; j < d; ++j) X[i * d + j] = c[size_t(k[size_t(i)] * d + j)] + n01(g0);
        standardise(X, n, d);
        std::uniform_real_distribution<double> u01(0.0, 1.0);
        for (int64_t i = 0; i < n; ++i) {
            double y = (k[size_t(i)] % 2 == 0) ? 1.0 : -1.0;
            if (u01(g4) < 0.05) y = -y;
            Y[i] = y;
        }
    } else if (cfg == 3 || cfg == 4) {
        if (t != 1) throw std::invalid_argument("configs 3/4 have one right-hand side");
        std::mt19937_64 g0(seed + 0), g1(seed + 1), g2(seed + 2);
        std::normal_distribution<double> n01(0.0, 1.0);
        const double c = std::sqrt(0.75);
        for (int64_t i = 0; i < n; ++i) {
            X[i * d] = n01(g0);
            for (int64_t j = 1; j < d; ++j) X[i * d + j] = 0.5 * X[i * d + j - 1] + c * n01(g0);
        }
        standardise(X, n, d);
        std::normal_distribution<double> nu(0.0, 1.0 / std::sqrt(double(d)));
        std::vector<double> u(static_cast<size_t>(8 * d)), a(8);
        for (auto& x : u) x = nu(g1);
        for (auto& x : a) x = n01(g1);
        std::normal_distribution<double> noise(0.0, 0.5);
        for (int64_t i = 0; i < n; ++i) {
            double y = 0.0;
            for (int k = 0; k < 8; ++k) y += a[size_t(k)] * std::tanh(dotp(u.data() + k * d, X + i * d, d));
            Y[i] = y + noise(g2);
        }
    } else if (cfg == 5) {
        std::mt19937_64 g0(seed + 0), g1(seed + 1), g5(seed + 5);
        std::normal_distribution<double> n01(0.0, 1.0);
        std::vector<double> G(static_cast<size_t>(n * d));
        for (auto& x : G) x = n01(g0);
        std::vector<double> qa(static_cast<size_t>(d * d));
        for (auto& x : qa) x = n01(g5);
        const std::vector<double> Q = householder_q(std::move(qa), d);
        // M = diag(sqrt(1/i)) Q^T, X = G M
        std::vector<double> M(static_cast<size_t>(d * d));
        for (int64_t i = 0; i < d; ++i)
            for (int64_t j = 0; j < d; ++j)
                M[size_t(i * d + j)] = std::sqrt(1.0 / double(i + 1)) * Q[size_t(j * d + i)];
        parallel_rows(n, [&](int64_t a, int64_t b) {
            for (int64_t r = a; r < b; ++r) {
                double* xr = X + r * d;
                for (int64_t j = 0; j < d; ++j) xr[j] = 0.0;
                for (int64_t k = 0; k < d; ++k) {
                    const double gk = G[size_t(r * d + k)];
                    const double* mk = M.data() + k * d;
                    for (int64_t j = 0; j < d; ++j) xr[j] += gk * mk[j];
                }
            }
        });
        standardise(X, n, d);
        std::vector<double> T(static_cast<size_t>(d * t));
        for (auto& x : T) x = n01(g1);
        std::vector<int32_t> labels(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) {
            int best = 0;
            double bv = 0.0;
            for (int64_t c = 0; c < t; ++c) {
                double s = 0.0;
                for (int64_t k = 0; k < d; ++k) s += X[i * d + k] * T[size_t(k * t + c)];
                if (c == 0 || s > bv) {
                    bv = s;
                    best = int(c);
                }
            }
            labels[size_t(i)] = best;
        }
        rlsc_encode(labels.data(), n, int32_t(t), Y);
    } else {
        throw std::invalid_argument("generate_config: cfg must be 1..5");
    }
}

void shard_rows(int64_t n, int world, int rank, int64_t* z0, int64_t* z1) {
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("shard: bad rank");
    const int64_t per = (n + world - 1) / world;
    *z0 = std::min(n, per * rank);
    *z1 = std::min(n, *z0 + per);
}

Schedule make_schedule(int64_t n, int world, int rank) {
    if (n < 1) throw std::invalid_argument("schedule: n must be positive");
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("schedule: bad rank");
    Schedule s;
    auto nsuper = [&](int64_t st) { return (n + st - 1) / st; };
    int64_t st = 128;
    while (st * 2 <= 4096 && nsuper(st * 2) >= 32) st *= 2;
    s.st = st;
    s.ns = nsuper(st);
    s.n_pad = s.ns * st;
    // Heaviest (off-diagonal, full) super-tiles first, diagonal (half) last, dealt
    // round-robin over ranks so every rank gets the same work within one tile.  Blocked
    // order: BLK x BLK blocks of (I, J) super-tile pairs, column-block major, so the ~148
    // CTAs resident at a time share ~BLK row and ~BLK column super-tiles.  The K1 kernels
    // stream the J super-tile once per 128-row pass and read the I super-tile once; with
    // both sets in L2 (2 x 12 x 2.75 MB at n = 1M, d = 90) neither is re-read from HBM.
    // (Column-major alone shared J but gave every resident CTA its own I super-tile:
    // 90 GB of HBM reads per n = 1M mat-vec, 130x the operand bytes.)
    constexpr int64_t BLK = 12;
    std::vector<std::pair<int32_t, int32_t>> order;
    order.reserve(size_t(s.ns * (s.ns + 1) / 2));
    for (int64_t jb = 0; jb * BLK < s.ns; ++jb)
        for (int64_t ib = 0; ib <= jb; ++ib)
            for (int64_t b = jb * BLK; b < std::min(s.ns, (jb + 1) * BLK); ++b)
                for (int64_t a = ib * BLK; a < std::min(b, (ib + 1) * BLK); ++a)
                    order.emplace_back(int32_t(a), int32_t(b));
    for (int64_t a = 0; a < s.ns; ++a) order.emplace_back(int32_t(a), int32_t(a));
    s.owned.assign(size_t(s.ns * s.ns), 0);
    for (size_t q = 0; q < order.size(); ++q) {
        if (int(q % size_t(world)) != rank) continue;
        const auto [a, b] = order[q];
        s.tiles.push_back(a);
        s.tiles.push_back(b);
        s.owned[size_t(a * s.ns + b)] = 1;
        s.owned[size_t(b * s.ns + a)] = 1;
    }
    return s;
}

void power_iteration_start(uint64_t seed, int64_t n, double* v) {
    std::mt19937_64 gen(seed);
    std::normal_distribution<double> normal(0.0, 1.0);
    double ss = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        v[i] = normal(gen);
        ss += v[i] * v[i];
    }
    const double nrm = std::sqrt(ss);
    if (nrm > 0.0)
        for (int64_t i = 0; i < n; ++i) v[i] /= nrm;
}

int64_t default_initial_sketch_size(int64_t n) { return std::max<int64_t>(64, (n + 63) / 64); }

}  // namespace krr
