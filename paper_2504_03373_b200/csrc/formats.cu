// On-disk formats and output records of the localization path (SURVEY §8 row
// f4), behind the C ABI of include/sslgpu.h:
//
//   SSLC correlation tensors  load_correlation / save_correlation
//                             (reference correlation.cpp:133-193): "SSLC", u32le
//                             m, bins, T, then bins x m x m cf32 row-major
//   steering fields           load_steering / save_steering (music.cpp:47-106):
//                             one JSON header line {"bin_max","bin_min",
//                             "directions":[[az,el],..],"m"}, then the raw
//                             [dir][bin][mic] cf32 payload
//   NoiseModel::from_file     (gsvd.cpp:729-734): load + PD gate + inverses,
//                             straight into a device context
//   capture_noise_model       (synth.cpp:329-373) from noise-only PCM: the
//                             device STFT, then K = sum_f x x^H / F accumulated
//                             in FP64 in frame order on the device, narrowed
//                             to cf32 and gated like the reference
//   JSONL estimates           the line run_locate_to_stream writes per block
//                             (pipeline.cpp:265-286): nlohmann::json's dump of
//                             {"estimates":[{"azimuth_deg","direction",
//                             "elevation_deg","low_power","power"}],"frame"} --
//                             sorted keys, shortest round-trip doubles in
//                             nlohmann's layout
//
// File parsing is host I/O; every tensor lands in the device context and all
// arithmetic on it runs on the GPU.
#include "../../include/sslgpu.h"
#include "common.cuh"
#include "kernels.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

namespace sslg {

// K[b] += x_f x_f^H over the frames of one launch, in frame order, with the
// reference's rounding: zi * conj(zj) in the limited-range product form
// (re = ac + bd, im = bc - ad, each product rounded), then the running sum
// (synth.cpp:343-352).  One CTA per bin; acc [bins][m][m] cf64.
__global__ void capture_accum_kernel(const float2* __restrict__ frames, int nframes, int m, int bins,
                                     double2* __restrict__ acc) {
    const int b = blockIdx.x;
    const int mm = m * m;
    double2* a = acc + (size_t)b * mm;
    for (int e = threadIdx.x; e < mm; e += blockDim.x) {
        const int i = e / m, j = e % m;
        double2 s = a[e];
        for (int f = 0; f < nframes; ++f) {
            const float2 xi = frames[((size_t)f * m + i) * bins + b];
            const float2 xj = frames[((size_t)f * m + j) * bins + b];
            const double ar = xi.x, ai = xi.y, br = xj.x, bi = xj.y;
            const double re = __dadd_rn(__dmul_rn(ar, br), __dmul_rn(ai, bi));
            const double im = __dsub_rn(__dmul_rn(ai, br), __dmul_rn(ar, bi));
            s.x = __dadd_rn(s.x, re);
            s.y = __dadd_rn(s.y, im);
        }
        a[e] = s;
    }
}

// kb = float(acc * inv) per component (synth.cpp:361-364)
__global__ void capture_narrow_kernel(const double2* __restrict__ acc, size_t n, double inv, float2* __restrict__ k) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) k[i] = make_float2((float)__dmul_rn(acc[i].x, inv), (float)__dmul_rn(acc[i].y, inv));
}

void launch_capture_accum(const float2* frames, int nframes, int m, int bins, double2* acc, cudaStream_t s) {
    capture_accum_kernel<<<bins, 256, 0, s>>>(frames, nframes, m, bins, acc);
}

void launch_capture_narrow(const double2* acc, size_t n, double inv, float2* k, cudaStream_t s) {
    capture_narrow_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(acc, n, inv, k);
}

}  // namespace sslg

namespace sslg {
int set_error(int code, const std::string& msg);  // engine.cu: the message sslg_last_error returns
}

namespace {

int ferr(int code, const std::string& msg) { return sslg::set_error(code, msg); }

// ---- little-endian u32 (correlation.cpp:135-146) --------------------------------
void put_u32le(std::string& out, uint32_t v) {
    const char b[4] = {char(v & 0xff), char(v >> 8 & 0xff), char(v >> 16 & 0xff), char(v >> 24 & 0xff)};
    out.append(b, 4);
}
uint32_t get_u32le(const unsigned char* b) {
    return uint32_t(b[0]) | uint32_t(b[1]) << 8 | uint32_t(b[2]) << 16 | uint32_t(b[3]) << 24;
}

// ---- nlohmann::json number layout ----------------------------------------------
// Shortest round-trip digits (std::to_chars), laid out as nlohmann's
// format_buffer does (min_exp = -4, max_exp = 15): "40.0", "0.001",
// "1.5e-05", "1e+20"; non-finite values dump as null.
std::string json_double(double x) {
    if (!std::isfinite(x)) return "null";
    if (x == 0) return std::signbit(x) ? "-0.0" : "0.0";
    char sci[64];
    auto res = std::to_chars(sci, sci + sizeof sci, x, std::chars_format::scientific);
    std::string s(sci, res.ptr);
    std::string out;
    if (s[0] == '-') {
        out = "-";
        s.erase(0, 1);
    }
    const size_t epos = s.find('e');
    std::string digits = s.substr(0, epos);
    const int e10 = std::atoi(s.c_str() + epos + 1);
    digits.erase(std::remove(digits.begin(), digits.end(), '.'), digits.end());
    const int k = (int)digits.size();
    const int n = e10 + 1;  // decimal point position
    if (k <= n && n <= 15) {
        out += digits + std::string(n - k, '0') + ".0";
    } else if (0 < n && n <= 15) {
        out += digits.substr(0, n) + "." + digits.substr(n);
    } else if (-4 < n && n <= 0) {
        out += "0." + std::string(-n, '0') + digits;
    } else {
        out += digits.substr(0, 1);
        if (k > 1) out += "." + digits.substr(1);
        const int e = n - 1;
        char eb[8];
        std::snprintf(eb, sizeof eb, "e%c%02d", e < 0 ? '-' : '+', e < 0 ? -e : e);
        out += eb;
    }
    return out;
}

// ---- a minimal JSON reader for the steering header -----------------------------
struct JsonCursor {
    const char* p;
    const char* end;
    bool ok = true;
    void ws() {
        while (p < end && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\n')) ++p;
    }
    bool eat(char c) {
        ws();
        if (p < end && *p == c) {
            ++p;
            return true;
        }
        return false;
    }
    bool str(std::string& out) {
        ws();
        if (p >= end || *p != '"') return ok = false;
        ++p;
        out.clear();
        while (p < end && *p != '"') {
            if (*p == '\\' && p + 1 < end) ++p;
            out.push_back(*p++);
        }
        if (p >= end) return ok = false;
        ++p;
        return true;
    }
    bool num(double& v) {
        ws();
        char* e = nullptr;
        v = std::strtod(p, &e);
        if (e == p) return ok = false;
        p = e;
        return true;
    }
    // skips any value
    bool skip() {
        ws();
        if (p >= end) return ok = false;
        if (*p == '"') {
            std::string s;
            return str(s);
        }
        if (*p == '{' || *p == '[') {
            const char open = *p, close = open == '{' ? '}' : ']';
            ++p;
            if (eat(close)) return true;
            do {
                if (open == '{') {
                    std::string k;
                    if (!str(k) || !eat(':')) return ok = false;
                }
                if (!skip()) return false;
            } while (eat(','));
            return eat(close) || (ok = false);
        }
        if (!std::strncmp(p, "true", 4) || !std::strncmp(p, "null", 4)) {
            p += 4;
            return true;
        }
        if (!std::strncmp(p, "false", 5)) {
            p += 5;
            return true;
        }
        double d;
        return num(d);
    }
};

struct SteeringHeader {
    uint32_t m = 0, bin_min = 0, bin_max = 0;
    std::vector<double> dirs;  // [n][2]
    bool have_m = false, have_min = false, have_max = false, have_dirs = false;
};

bool parse_steering_header(const std::string& line, SteeringHeader& h, std::string& why) {
    JsonCursor c{line.data(), line.data() + line.size()};
    if (!c.eat('{')) {
        why = "expected an object";
        return false;
    }
    if (c.eat('}')) {
        why = "key 'm' not found";
        return false;
    }
    do {
        std::string key;
        if (!c.str(key) || !c.eat(':')) {
            why = "syntax error";
            return false;
        }
        auto get_u32 = [&](uint32_t& dst) {
            double v;
            if (!c.num(v) || !(v >= 0) || v != std::floor(v) || v > 4294967295.0) return false;
            dst = (uint32_t)v;
            return true;
        };
        if (key == "m") {
            if (!get_u32(h.m)) return why = "bad m", false;
            h.have_m = true;
        } else if (key == "bin_min") {
            if (!get_u32(h.bin_min)) return why = "bad bin_min", false;
            h.have_min = true;
        } else if (key == "bin_max") {
            if (!get_u32(h.bin_max)) return why = "bad bin_max", false;
            h.have_max = true;
        } else if (key == "directions") {
            if (!c.eat('[')) return why = "directions must be an array", false;
            if (!c.eat(']')) {
                do {
                    double az, el;
                    if (!c.eat('[') || !c.num(az) || !c.eat(',') || !c.num(el)) return why = "bad direction", false;
                    while (c.eat(',')) c.skip();  // extra components are ignored (at(0), at(1))
                    if (!c.eat(']')) return why = "bad direction", false;
                    h.dirs.push_back(az);
                    h.dirs.push_back(el);
                } while (c.eat(','));
                if (!c.eat(']')) return why = "bad directions array", false;
            }
            h.have_dirs = true;
        } else if (!c.skip()) {
            return why = "syntax error", false;
        }
    } while (c.eat(','));
    if (!c.eat('}')) return why = "syntax error", false;
    if (!h.have_m) return why = "key 'm' not found", false;
    if (!h.have_min) return why = "key 'bin_min' not found", false;
    if (!h.have_max) return why = "key 'bin_max' not found", false;
    if (!h.have_dirs) return why = "key 'directions' not found", false;
    return true;
}

bool read_file(const char* path, std::string& data) {
    std::ifstream in(path, std::ios::binary);
    if (!in) return false;
    data.assign(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
    return true;
}

bool write_file(const char* path, const std::string& data) {
    std::ofstream out(path, std::ios::binary);
    if (!out) return false;
    out.write(data.data(), (std::streamsize)data.size());
    return (bool)out;
}

}  // namespace

extern "C" {

int sslg_read_correlation_file(const char* path, uint32_t* m, uint32_t* bins, uint32_t* t, float* data,
                               uint64_t cap_floats) {
    if (!path) return ferr(SSLG_VALIDATION, "null path");
    std::string d;
    if (!read_file(path, d)) return ferr(SSLG_IO, std::string("cannot open ") + path);
    const auto* u = reinterpret_cast<const unsigned char*>(d.data());
    if (d.size() < 4 || std::memcmp(d.data(), "SSLC", 4) != 0)
        return ferr(SSLG_IO, std::string(path) + ": not a correlation tensor file");
    if (d.size() < 16) return ferr(SSLG_IO, std::string(path) + ": implausible header");
    const uint32_t mm = get_u32le(u + 4), nb = get_u32le(u + 8), tt = get_u32le(u + 12);
    if (mm < 1 || mm > 4096 || nb < 1 || nb > (1u << 20)) return ferr(SSLG_IO, std::string(path) + ": implausible header");
    if (m) *m = mm;
    if (bins) *bins = nb;
    if (t) *t = tt;
    const uint64_t nf = (uint64_t)nb * mm * mm * 2;
    if (d.size() < 16 + nf * 4) return ferr(SSLG_IO, std::string(path) + ": truncated payload");
    if (!data) return SSLG_OK;
    if (cap_floats < nf) return ferr(SSLG_VALIDATION, "buffer too small for the correlation payload");
    std::memcpy(data, d.data() + 16, nf * 4);
    for (uint64_t i = 0; i < nf; ++i)  // CorrelationSet::validate
        if (!std::isfinite(data[i])) return ferr(SSLG_VALIDATION, "non-finite correlation entry");
    return SSLG_OK;
}

int sslg_write_correlation_file(const char* path, uint32_t m, uint32_t bins, uint32_t t, const float* data) {
    if (!path || !data) return ferr(SSLG_VALIDATION, "null argument");
    if (m < 1 || bins < 1) return ferr(SSLG_VALIDATION, "correlation set has no bins");
    const uint64_t nf = (uint64_t)bins * m * m * 2;
    for (uint64_t i = 0; i < nf; ++i)
        if (!std::isfinite(data[i])) return ferr(SSLG_VALIDATION, "non-finite correlation entry");
    std::string out("SSLC", 4);
    put_u32le(out, m);
    put_u32le(out, bins);
    put_u32le(out, t);
    out.append(reinterpret_cast<const char*>(data), nf * 4);
    if (!write_file(path, out)) return ferr(SSLG_IO, std::string("cannot open ") + path + " for writing");
    return SSLG_OK;
}

int sslg_read_steering_file(const char* path, uint32_t* m, uint32_t* bin_min, uint32_t* bin_max, uint32_t* dirs,
                            double* dirs_deg, float* h, uint64_t cap_dirs) {
    if (!path) return ferr(SSLG_VALIDATION, "null path");
    std::string d;
    if (!read_file(path, d)) return ferr(SSLG_IO, std::string("cannot open ") + path);
    const size_t nl = d.find('\n');
    if (d.empty() || nl == 0) return ferr(SSLG_IO, std::string("missing header line in ") + path);
    const std::string line = d.substr(0, nl == std::string::npos ? d.size() : nl);
    SteeringHeader hd;
    std::string why;
    if (!parse_steering_header(line, hd, why))
        return ferr(SSLG_IO, std::string("bad steering header in ") + path + ": " + why);
    if (hd.m == 0 || hd.bin_max < hd.bin_min || hd.dirs.empty())
        return ferr(SSLG_IO, std::string("bad steering header in ") + path);
    const uint32_t nd = (uint32_t)(hd.dirs.size() / 2);
    const uint64_t count = (uint64_t)nd * (hd.bin_max - hd.bin_min + 1) * hd.m;
    const size_t off = nl == std::string::npos ? d.size() : nl + 1;
    if (d.size() - off < count * 8) return ferr(SSLG_IO, std::string("truncated steering payload in ") + path);
    if (m) *m = hd.m;
    if (bin_min) *bin_min = hd.bin_min;
    if (bin_max) *bin_max = hd.bin_max;
    if (dirs) *dirs = nd;
    if (!h && !dirs_deg) return SSLG_OK;
    if (cap_dirs < nd) return ferr(SSLG_VALIDATION, "buffer too small for the steering field");
    if (dirs_deg) std::memcpy(dirs_deg, hd.dirs.data(), hd.dirs.size() * sizeof(double));
    if (h) {
        std::memcpy(h, d.data() + off, count * 8);
        for (uint64_t i = 0; i < count * 2; ++i)  // SteeringField::validate
            if (!std::isfinite(h[i])) return ferr(SSLG_VALIDATION, "non-finite steering value");
    }
    return SSLG_OK;
}

int sslg_write_steering_file(const char* path, uint32_t m, uint32_t bin_min, uint32_t bin_max, uint32_t dirs,
                             const double* dirs_deg, const float* h) {
    if (!path || !dirs_deg || !h) return ferr(SSLG_VALIDATION, "null argument");
    if (m == 0) return ferr(SSLG_VALIDATION, "steering field has no channels");
    if (bin_max < bin_min) return ferr(SSLG_VALIDATION, "steering field bin range is inverted");
    if (dirs == 0) return ferr(SSLG_VALIDATION, "steering field has no directions");
    // nlohmann::json object: keys in sorted order
    std::string out = "{\"bin_max\":" + std::to_string(bin_max) + ",\"bin_min\":" + std::to_string(bin_min) +
                      ",\"directions\":[";
    for (uint32_t i = 0; i < dirs; ++i) {
        if (i) out += ",";
        out += "[" + json_double(dirs_deg[2 * i]) + "," + json_double(dirs_deg[2 * i + 1]) + "]";
    }
    out += "],\"m\":" + std::to_string(m) + "}\n";
    const uint64_t count = (uint64_t)dirs * (bin_max - bin_min + 1) * m;
    out.append(reinterpret_cast<const char*>(h), count * 8);
    if (!write_file(path, out)) return ferr(SSLG_IO, std::string("cannot open ") + path + " for writing");
    return SSLG_OK;
}

int sslg_load_noise_model(sslg_ctx* ctx, const char* path, uint32_t* bad_bin, uint32_t* t) {
    if (!ctx || !path) return ferr(SSLG_VALIDATION, "null argument");
    sslg_config cfg;
    if (int rc = sslg_get_config(ctx, &cfg)) return rc;
    uint32_t m = 0, bins = 0;
    if (int rc = sslg_read_correlation_file(path, &m, &bins, t, nullptr, 0)) return rc;
    if (m != cfg.m) return ferr(SSLG_VALIDATION, "noise model channel count does not match correlation set");
    if (bins != cfg.bins) return ferr(SSLG_VALIDATION, "noise model bin count does not match correlation set");
    std::vector<float> k((size_t)bins * m * m * 2);
    if (int rc = sslg_read_correlation_file(path, nullptr, nullptr, nullptr, k.data(), k.size())) return rc;
    // NoiseModel::from_file checks positive definiteness on load (gsvd.cpp:729-734)
    return sslg_set_noise_model(ctx, k.data(), 1, bad_bin);
}

int sslg_load_steering(sslg_ctx* ctx, const char* path, uint32_t* bin_min) {
    if (!ctx || !path) return ferr(SSLG_VALIDATION, "null argument");
    sslg_config cfg;
    if (int rc = sslg_get_config(ctx, &cfg)) return rc;
    uint32_t m = 0, lo = 0, hi = 0, nd = 0;
    if (int rc = sslg_read_steering_file(path, &m, &lo, &hi, &nd, nullptr, nullptr, 0)) return rc;
    if (m != cfg.m) return ferr(SSLG_VALIDATION, "steering field channel count does not match");
    if (hi - lo + 1 != cfg.bins) return ferr(SSLG_VALIDATION, "steering field bin count does not match factorization");
    std::vector<double> dirs((size_t)nd * 2);
    std::vector<float> h((size_t)nd * cfg.bins * m * 2);
    if (int rc = sslg_read_steering_file(path, nullptr, nullptr, nullptr, nullptr, dirs.data(), h.data(), nd)) return rc;
    if (bin_min) *bin_min = lo;
    return sslg_set_steering(ctx, nd, h.data(), dirs.data(), nullptr, nullptr);
}

int sslg_format_estimates_json(uint64_t frame, uint32_t count, const uint32_t* idx, const double* dirs_deg,
                               const double* power, const uint8_t* low, char* buf, uint64_t cap, uint64_t* len) {
    if (count && (!idx || !dirs_deg || !power || !low)) return ferr(SSLG_VALIDATION, "null argument");
    std::string s = "{\"estimates\":[";
    for (uint32_t i = 0; i < count; ++i) {
        if (i) s += ",";
        const uint32_t j = idx[i];
        s += "{\"azimuth_deg\":" + json_double(dirs_deg[2 * (size_t)j]) + ",\"direction\":" + std::to_string(j) +
             ",\"elevation_deg\":" + json_double(dirs_deg[2 * (size_t)j + 1]) +
             ",\"low_power\":" + (low[i] ? "true" : "false") + ",\"power\":" + json_double(power[i]) + "}";
    }
    s += "],\"frame\":" + std::to_string(frame) + "}";
    if (len) *len = s.size();
    if (!buf) return SSLG_OK;
    if (cap < s.size() + 1) return ferr(SSLG_VALIDATION, "buffer too small for the JSON line");
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return SSLG_OK;
}

}  // extern "C"
