// the reference's KRRM model file (io.cpp:192-261), byte-identical, so a model
// trained on the B200 path feeds the reference's `krr predict` / `krr eval` unchanged.
//
// Layout: "KRRM" | uint32 version = 1 | uint32 metadata length | metadata JSON (compact,
// keys in std::map order as nlohmann::json dumps them) | X (n x d fp64, row-major) |
// C (n x t fp64, row-major), host byte order.  The metadata for a Gaussian model is
//   {"d":D,"kernel":{"family":"gaussian","sigma":S},"label_map":[...],"lambda":L,"n":N,
//    "seed":SEED,"t":T,"tool_version":"0.1.0"}
// and a polynomial model's kernel object is {"degree":Q,"family":"polynomial","gamma":G,"offset":C}.
// with doubles in nlohmann's shortest-round-trip format (dtoa_impl::format_buffer: fixed
// notation for decimal exponents in (-4, 15], ".0" appended to integral values, otherwise
// d.ddde±XX with at least two exponent digits).  load_model's checks are kept: bad magic,
// unsupported version, trailing bytes, non-finite entries, invalid dimensions.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

#include "../../include/krr_b200.h"
#include "error.hpp"
#include "host.hpp"

namespace krr {
namespace {

constexpr char kMagic[4] = {'K', 'R', 'R', 'M'};
constexpr uint32_t kFormatVersion = 1;
constexpr const char* kToolVersion = "0.1.0";  // io.hpp:14

[[noreturn]] void io_fail(const std::string& msg) { fail(KRR_ERR_IO, msg); }

// nlohmann::json number_float output (shortest digits, dtoa_impl::format_buffer rules).
std::string json_double(double v) {
    if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::scientific);  // shortest
    std::string sci(buf, r.ptr);
    std::string out;
    if (sci[0] == '-') {
        out = "-";
        sci.erase(0, 1);
    }
    const auto epos = sci.find('e');
    std::string digits = sci.substr(0, epos);
    digits.erase(std::remove(digits.begin(), digits.end(), '.'), digits.end());
    const int e10 = std::stoi(sci.substr(epos + 1));
    const int k = int(digits.size());
    const int n = e10 + 1;  // value = 0.d1..dk * 10^n
    constexpr int kMinExp = -4, kMaxExp = 15;
    if (k <= n && n <= kMaxExp) {
        out += digits + std::string(size_t(n - k), '0') + ".0";
    } else if (0 < n && n <= kMaxExp) {
        out += digits.substr(0, size_t(n)) + "." + digits.substr(size_t(n));
    } else if (kMinExp < n && n <= 0) {
        out += "0." + std::string(size_t(-n), '0') + digits;
    } else {
        out += digits.substr(0, 1);
        if (k > 1) out += "." + digits.substr(1);
        const int ex = n - 1;
        out += ex < 0 ? "e-" : "e+";
        const int a = ex < 0 ? -ex : ex;
        if (a < 10) out += "0";
        out += std::to_string(a);
    }
    return out;
}

// ---- a minimal JSON reader for the metadata object (objects, arrays, strings, numbers)
struct JVal;
using JObj = std::map<std::string, JVal>;
using JArr = std::vector<JVal>;
struct JVal {
    // integers without sign / fraction / exponent keep their exact uint64 value (as nlohmann)
    std::variant<std::nullptr_t, double, std::string, std::shared_ptr<JObj>, std::shared_ptr<JArr>, bool, uint64_t> v;
};

struct JParser {
    const std::string& s;
    size_t i = 0;
    void ws() {
        while (i < s.size() && (s[i] == ' ' || s[i] == '\n' || s[i] == '\t' || s[i] == '\r')) ++i;
    }
    [[noreturn]] void bad() { io_fail("model file: bad metadata"); }
    JVal value() {
        ws();
        if (i >= s.size()) bad();
        const char c = s[i];
        if (c == '{') {
            ++i;
            auto o = std::make_shared<JObj>();
            ws();
            if (i < s.size() && s[i] == '}') {
                ++i;
                return {o};
            }
            for (;;) {
                ws();
                const std::string key = str();
                ws();
                if (i >= s.size() || s[i] != ':') bad();
                ++i;
                (*o)[key] = value();
                ws();
                if (i < s.size() && s[i] == ',') {
                    ++i;
                    continue;
                }
                if (i < s.size() && s[i] == '}') {
                    ++i;
                    return {o};
                }
                bad();
            }
        }
        if (c == '[') {
            ++i;
            auto a = std::make_shared<JArr>();
            ws();
            if (i < s.size() && s[i] == ']') {
                ++i;
                return {a};
            }
            for (;;) {
                a->push_back(value());
                ws();
                if (i < s.size() && s[i] == ',') {
                    ++i;
                    continue;
                }
                if (i < s.size() && s[i] == ']') {
                    ++i;
                    return {a};
                }
                bad();
            }
        }
        if (c == '"') return {str()};
        if (s.compare(i, 4, "true") == 0) {
            i += 4;
            return {true};
        }
        if (s.compare(i, 5, "false") == 0) {
            i += 5;
            return {false};
        }
        if (s.compare(i, 4, "null") == 0) {
            i += 4;
            return {nullptr};
        }
        const size_t j0 = i;
        while (i < s.size() && (std::isdigit(static_cast<unsigned char>(s[i])) || s[i] == '-' || s[i] == '+' ||
                                s[i] == '.' || s[i] == 'e' || s[i] == 'E'))
            ++i;
        if (i == j0) bad();
        if (s.find_first_not_of("0123456789", j0) >= i) {
            uint64_t u = 0;
            const auto ru = std::from_chars(s.data() + j0, s.data() + i, u);
            if (ru.ec == std::errc() && ru.ptr == s.data() + i) return {u};
        }
        double d = 0.0;
        const auto r = std::from_chars(s.data() + j0, s.data() + i, d);
        if (r.ec != std::errc() || r.ptr != s.data() + i) bad();
        return {d};
    }
    std::string str() {
        if (i >= s.size() || s[i] != '"') bad();
        ++i;
        std::string out;
        while (i < s.size() && s[i] != '"') {
            if (s[i] == '\\') {
                ++i;
                if (i >= s.size()) bad();
            }
            out += s[i++];
        }
        if (i >= s.size()) bad();
        ++i;
        return out;
    }
};

const JVal& at(const JObj& o, const char* key) {
    auto it = o.find(key);
    if (it == o.end()) io_fail(std::string("model file: bad metadata: missing key '") + key + "'");
    return it->second;
}
double num(const JVal& v) {
    if (auto p = std::get_if<double>(&v.v)) return *p;
    if (auto q = std::get_if<uint64_t>(&v.v)) return double(*q);
    io_fail("model file: bad metadata: expected a number");
}
uint64_t unum(const JVal& v) {
    if (auto q = std::get_if<uint64_t>(&v.v)) return *q;
    io_fail("model file: bad metadata: expected an unsigned integer");
}

void read_exact(std::ifstream& in, void* dst, size_t bytes, const char* what) {
    in.read(static_cast<char*>(dst), std::streamsize(bytes));
    if (size_t(in.gcount()) != bytes) io_fail(std::string("model file: truncated while reading ") + what);
}

ModelMeta read_meta(std::ifstream& in, const std::string& path) {
    if (!in) io_fail("cannot open '" + path + "'");
    char magic[4];
    read_exact(in, magic, 4, "magic");
    if (std::memcmp(magic, kMagic, 4) != 0) io_fail("model file: bad magic");
    uint32_t version = 0, meta_len = 0;
    read_exact(in, &version, 4, "version");
    if (version != kFormatVersion) io_fail("model file: unsupported version " + std::to_string(version));
    read_exact(in, &meta_len, 4, "metadata length");
    std::string text(meta_len, '\0');
    read_exact(in, text.data(), meta_len, "metadata");
    JParser p{text};
    const JVal root = p.value();
    auto obj = std::get_if<std::shared_ptr<JObj>>(&root.v);
    if (!obj) io_fail("model file: bad metadata");
    const JObj& o = **obj;
    ModelMeta m;
    auto kobj = std::get_if<std::shared_ptr<JObj>>(&at(o, "kernel").v);
    if (!kobj) io_fail("model file: bad metadata: kernel");
    auto fam = std::get_if<std::string>(&at(**kobj, "family").v);
    if (!fam) io_fail("model file: bad metadata: kernel family");
    // kernel_from_json (io.cpp:82-90) -> KernelSpec::gaussian / ::polynomial, which validate.
    if (*fam == "gaussian") {
        m.family = 0;
        m.sigma = num(at(**kobj, "sigma"));
        if (!(m.sigma > 0.0)) fail(KRR_ERR_INVALID_ARGUMENT, "KernelSpec: sigma must be positive");
    } else if (*fam == "polynomial") {
        m.family = 1;
        m.gamma = num(at(**kobj, "gamma"));
        m.offset = num(at(**kobj, "offset"));
        m.degree = int(unum(at(**kobj, "degree")));
        if (m.degree < 1) fail(KRR_ERR_INVALID_ARGUMENT, "KernelSpec: degree must be at least 1");
        if (m.offset < 0.0) fail(KRR_ERR_INVALID_ARGUMENT, "KernelSpec: offset must be non-negative");
        if (!(m.gamma > 0.0)) fail(KRR_ERR_INVALID_ARGUMENT, "KernelSpec: gamma must be positive");
    } else {
        io_fail("model file: unknown kernel family '" + *fam + "'");
    }
    m.lambda = num(at(o, "lambda"));
    m.seed = unum(at(o, "seed"));
    auto lm = std::get_if<std::shared_ptr<JArr>>(&at(o, "label_map").v);
    if (!lm) io_fail("model file: bad metadata: label_map");
    for (const JVal& v : **lm) m.label_map.push_back(num(v));
    m.n = int64_t(unum(at(o, "n")));
    m.d = int64_t(unum(at(o, "d")));
    m.t = int64_t(unum(at(o, "t")));
    if (m.n < 1 || m.d < 0 || m.t < 1) io_fail("model file: invalid dimensions");
    return m;
}

}  // namespace
}  // namespace krr

namespace krr {

void model_save(const char* path, int family, double sigma, double gamma, double offset, int degree, double lambda,
                uint64_t seed, const double* label_map, int64_t nlabels, const double* X, int64_t n, int64_t d,
                const double* C, int64_t t) {
    if (!path) fail(KRR_ERR_INVALID_ARGUMENT, "model file: null path");
    if (n < 1 || d < 0 || t < 1 || nlabels < 0) fail(KRR_ERR_DIMENSION_MISMATCH, "model file: bad shapes");
    // kernel_to_json (io.cpp:73-80); nlohmann orders object keys alphabetically.
    const std::string kernel =
        family == 0 ? "{\"family\":\"gaussian\",\"sigma\":" + json_double(sigma) + "}"
                    : "{\"degree\":" + std::to_string(degree) + ",\"family\":\"polynomial\",\"gamma\":" +
                          json_double(gamma) + ",\"offset\":" + json_double(offset) + "}";
    std::string meta = "{\"d\":" + std::to_string(d) + ",\"kernel\":" + kernel + ",\"label_map\":[";
    for (int64_t i = 0; i < nlabels; ++i) meta += (i ? "," : "") + json_double(label_map[i]);
    meta += "],\"lambda\":" + json_double(lambda) + ",\"n\":" + std::to_string(n) + ",\"seed\":" +
            std::to_string(seed) + ",\"t\":" + std::to_string(t) + ",\"tool_version\":\"" + kToolVersion + "\"}";
    std::ofstream out(path, std::ios::binary);
    if (!out) io_fail(std::string("cannot write '") + path + "'");
    const uint32_t version = kFormatVersion, meta_len = uint32_t(meta.size());
    out.write(kMagic, 4);
    out.write(reinterpret_cast<const char*>(&version), 4);
    out.write(reinterpret_cast<const char*>(&meta_len), 4);
    out.write(meta.data(), std::streamsize(meta.size()));
    out.write(reinterpret_cast<const char*>(X), std::streamsize(sizeof(double) * size_t(n * d)));
    out.write(reinterpret_cast<const char*>(C), std::streamsize(sizeof(double) * size_t(n * t)));
    if (!out) io_fail(std::string("write failed for '") + path + "'");
}

ModelMeta model_info(const char* path) {
    std::ifstream in(path ? path : "", std::ios::binary);
    return read_meta(in, path ? path : "");
}

void model_load(const char* path, double* label_map, double* X, double* C) {
    std::ifstream in(path ? path : "", std::ios::binary);
    const ModelMeta m = read_meta(in, path ? path : "");
    for (size_t i = 0; i < m.label_map.size(); ++i) label_map[i] = m.label_map[i];
    read_exact(in, X, sizeof(double) * size_t(m.n * m.d), "X");
    read_exact(in, C, sizeof(double) * size_t(m.n * m.t), "C");
    in.peek();  // io.cpp: declared sizes must account for every payload byte
    if (!in.eof()) io_fail("model file: trailing bytes after payload");
    for (int64_t i = 0; i < m.n * m.d; ++i)
        if (!std::isfinite(X[i])) io_fail("model file: non-finite entries");
    for (int64_t i = 0; i < m.n * m.t; ++i)
        if (!std::isfinite(C[i])) io_fail("model file: non-finite entries");
}

}  // namespace krr
