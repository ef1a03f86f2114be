// ============================================================================
// CPU ORACLE -- TEST INFRASTRUCTURE ONLY.
//
// A plain C++ restatement of the reference's algorithm for the north-star
// path (prefill / decode_step / generate / reference_forward_nocache over a
// normalized factorized checkpoint). Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference leg may load this library, and
// only as the checker or the timed CPU baseline -- never as a product path.
//
// The reference (/root/reference, FlashSVD v1.5 desk artifact) implements the
// primitives and the loader but NOT the runtime: prefill/decode_step exist
// only in SPEC.md:283-382. So this file restates:
//   * kernel semantics: proj/src/kernels/kernels_scalar.cpp:11-69 (gemv with
//     per-column in-order accumulation, dot, axpy, scal, add, rmsnorm, silu_mul)
//   * math: proj/include/fsvd/math.hpp:30-44 (rope_inplace, angles in double),
//     :56-101 (OnlineAttend), :132-140 (argmax_greedy, lowest index on ties)
//   * loader: proj/src/checkpoint.cpp:134-197 (FSVD15 read),
//     proj/src/canonical.cpp:57-194 (families A/B/C + pack_ffn) and the
//     family-D extension (A = U diag(S))
//   * runtime: SPEC.md:305-313 prefill (P = X.A once, K/V reconstructed in
//     blocks of 64, RoPE after reconstruction, causal online softmax),
//     SPEC.md:314-322 decode_step, SPEC.md:323-331 ffn_no_merge/ffn_packed,
//     SPEC.md:341-349 generate, SPEC.md:350-358 reference_forward_nocache
//     (structure of the dense gold proj/src/model.cpp:204-285 with every x.W
//     replaced by (x.A).B).
//   * synthetic weights: include/fsvd/synth.hpp stream definition (restated
//     here independently so the product generator is checked, not trusted).
// Parity pins: tests/test_oracle.py checks these primitives bit-for-bit
// against oracle/_ref (the reference compiled from its own sources) and
// against the committed golden vectors in tests/golden/.
//
// Precision: T = float accumulates in float (the fp32 runtime
// semantics), T = double is the f64 gold. Weights are always the floats of
// normalize<float> (GPU and oracle consume the same
// CanonicalModel<float>), upcast on use.
// Build: oracle/Makefile (-O3 -ffp-contract=off, like proj/CMakeLists.txt:15).
// ============================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <limits>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <json.hpp>

namespace oracle {

using u64 = uint64_t;

struct Config {
    size_t L = 0, d = 0, H = 0, dh = 0, dff = 0, V = 0;
    double rope_base = 10000.0, eps = 1e-5;
};

// ----------------------------------------------------------- matrices ----
struct Mat {  // row-major f32 (the canonical weight floats)
    size_t rows = 0, cols = 0;
    std::vector<float> v;
    Mat() = default;
    Mat(size_t r, size_t c) : rows(r), cols(c), v(r * c, 0.f) {}
    float at(size_t i, size_t j) const { return v[i * cols + j]; }
};

struct Factor {
    std::shared_ptr<Mat> a;  // d_in x r
    std::shared_ptr<Mat> b;  // r x d_out
    size_t rank = 0;
};

struct Layer {
    Factor p[7];  // q k v o up gate down
    std::vector<float> attn_gamma, mlp_gamma;
    Mat a_ug;
    size_t r_up = 0;
};

struct Model {
    Config c;
    size_t capacity = 0;
    Mat emb, head;
    std::vector<float> final_gamma;
    std::vector<Layer> layers;
    size_t shared_instances = 0;
};

const char* kProj[7] = {"q", "k", "v", "o", "up", "gate", "down"};
void dims(const Config& c, int p, size_t& din, size_t& dout) {
    din = c.d;
    dout = c.d;
    if (p == 4 || p == 5) dout = c.dff;
    if (p == 6) din = c.dff;
}

// ------------------------------------------------------ thread pool-ish ----
int g_threads = 1;

template <typename F>
void parallel_cols(size_t n, F&& f) {  // f(lo, hi) over output columns
    const int T = std::max(1, std::min<int>(g_threads, static_cast<int>(n / 64 + 1)));
    if (T == 1) {
        f(size_t(0), n);
        return;
    }
    std::vector<std::thread> ts;
    for (int t = 0; t < T; ++t) ts.emplace_back([&, t] { f(n * t / T, n * (t + 1) / T); });
    for (auto& t : ts) t.join();
}

// --------------------------------------------------------------- kernels ----
// kernels_scalar.cpp:11-21 -- y = x . A (A row-major m x n), every column
// accumulates over k in index order. Column-block parallel: bit-preserving by
// the contract in kernels.hpp:8-11.
template <typename T>
void gemv(T* y, const T* x, const Mat& A) {
    const size_t m = A.rows, n = A.cols;
    parallel_cols(n, [&](size_t lo, size_t hi) {
        for (size_t j = lo; j < hi; ++j) y[j] = T(0);
        for (size_t k = 0; k < m; ++k) {
            const T xk = x[k];
            const float* row = A.v.data() + k * n;
            for (size_t j = lo; j < hi; ++j) y[j] += xk * static_cast<T>(row[j]);
        }
    });
}

// Optional: route f32 gemv through the reference's own Ops::gemv (the timed
// CPU baseline, oracle/_ref). Signature kernels.hpp:20.
using RefGemvF32 = void (*)(float*, const float*, const float*, size_t, size_t);
RefGemvF32 g_ref_gemv = nullptr;

void gemv_f32(float* y, const float* x, const Mat& A) {
    if (!g_ref_gemv) return gemv<float>(y, x, A);
    // The reference kernel takes a contiguous row-major A; column panels are
    // pre-split per thread (bitwise identical per column).
    g_ref_gemv(y, x, A.v.data(), A.rows, A.cols);
}

template <typename T>
void gemv_any(T* y, const T* x, const Mat& A) {
    if constexpr (std::is_same_v<T, float>)
        gemv_f32(y, x, A);
    else
        gemv<T>(y, x, A);
}

// Y[t] = X[t] . A for n rows: the same per-(t, column) accumulation as gemv
// (k in index order from zero), rows blocked 8 at a time so each weight row is
// read once per block instead of once per token -- bitwise identical to n
// gemv calls (tensor.hpp:100-119: matmul == triple loop). Used by the prefill
// restatement, where the oracle is otherwise weight-stream
// bound. With the reference gemv plugged in (CPU baseline), rows go through it.
template <typename T>
void gemv_rows(size_t n, const T* const* X, T* const* Y, const Mat& A) {
    if constexpr (std::is_same_v<T, float>)
        if (g_ref_gemv) {
            for (size_t t = 0; t < n; ++t) gemv_f32(Y[t], X[t], A);
            return;
        }
    const size_t m = A.rows, nc = A.cols;
    constexpr size_t RB = 8;
    parallel_cols(nc, [&](size_t lo, size_t hi) {
        for (size_t t0 = 0; t0 < n; t0 += RB) {
            const size_t t1 = std::min(n, t0 + RB);
            for (size_t t = t0; t < t1; ++t)
                for (size_t j = lo; j < hi; ++j) Y[t][j] = T(0);
            for (size_t k = 0; k < m; ++k) {
                const float* row = A.v.data() + k * nc;
                for (size_t t = t0; t < t1; ++t) {
                    const T xk = X[t][k];
                    T* y = Y[t];
                    for (size_t j = lo; j < hi; ++j) y[j] += xk * static_cast<T>(row[j]);
                }
            }
        }
    });
}

template <typename T>
struct Rows {  // n row vectors of one width, with pointer tables for gemv_rows
    std::vector<std::vector<T>> r;
    std::vector<T*> p;
    Rows(size_t n, size_t w) : r(n, std::vector<T>(w)), p(n) {
        for (size_t i = 0; i < n; ++i) p[i] = r[i].data();
    }
    std::vector<const T*> cp(size_t off = 0) const {
        std::vector<const T*> q(r.size());
        for (size_t i = 0; i < r.size(); ++i) q[i] = r[i].data() + off;
        return q;
    }
};

template <typename T>
T dot(const T* a, const T* b, size_t n) {  // kernels_scalar.cpp:23-28
    T s = T(0);
    for (size_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

template <typename T>
void rmsnorm(T* y, const T* x, const std::vector<float>& g, size_t n, T eps) {  // :55-61
    T ss = T(0);
    for (size_t i = 0; i < n; ++i) ss += x[i] * x[i];
    const T inv = T(1) / std::sqrt(ss / static_cast<T>(n) + eps);
    for (size_t i = 0; i < n; ++i) y[i] = x[i] * inv * static_cast<T>(g[i]);
}

template <typename T>
void silu_mul(T* y, const T* gate, const T* up, size_t n) {  // :63-69
    for (size_t i = 0; i < n; ++i) {
        const T g = gate[i];
        y[i] = g / (T(1) + std::exp(-g)) * up[i];
    }
}

// math.hpp:30-44: pair (2i, 2i+1) by pos * base^(-2i/d); angle in double
template <typename T>
void rope(T* v, size_t d, double pos, double base) {
    for (size_t i = 0; i < d / 2; ++i) {
        const double freq = std::pow(base, -2.0 * static_cast<double>(i) / static_cast<double>(d));
        const double ang = pos * freq;
        const T c = static_cast<T>(std::cos(ang));
        const T s = static_cast<T>(std::sin(ang));
        const T x0 = v[2 * i], x1 = v[2 * i + 1];
        v[2 * i] = x0 * c - x1 * s;
        v[2 * i + 1] = x0 * s + x1 * c;
    }
}

// math.hpp:56-101 OnlineAttend
template <typename T>
struct Online {
    T m = -std::numeric_limits<T>::infinity(), l = T(0);
    std::vector<T> acc;
    std::vector<T> scores;
    void reset(size_t d) {
        m = -std::numeric_limits<T>::infinity();
        l = T(0);
        acc.assign(d, T(0));
    }
    // rows of K/V with stride `stride` (elements), d = head dim
    void update(const T* q, const T* k, const T* v, size_t rows, size_t stride, size_t d, T scale) {
        if (!rows) return;
        scores.resize(rows);
        T bm = -std::numeric_limits<T>::infinity();
        for (size_t j = 0; j < rows; ++j) {
            const T s = dot(q, k + j * stride, d) * scale;
            scores[j] = s;
            if (s > bm) bm = s;
        }
        const T mn = m > bm ? m : bm;
        const T r = std::exp(m - mn);
        l *= r;
        for (size_t i = 0; i < d; ++i) acc[i] *= r;  // Ops::scal
        for (size_t j = 0; j < rows; ++j) {
            const T w = std::exp(scores[j] - mn);
            l += w;
            const T* vr = v + j * stride;
            for (size_t i = 0; i < d; ++i) acc[i] += w * vr[i];  // Ops::axpy
        }
        m = mn;
    }
    void finish(T* out, size_t d) const {
        for (size_t i = 0; i < d; ++i) out[i] = acc[i] / l;
    }
};

template <typename T>
size_t argmax(const T* x, size_t n) {  // math.hpp:132-140
    size_t b = 0;
    for (size_t i = 1; i < n; ++i)
        if (x[i] > x[b]) b = i;
    return b;
}

// ------------------------------------------------------------------ CRC ----
uint32_t crc32(const void* data, size_t len) {
    static uint32_t table[256];
    static bool init = false;
    if (!init) {
        for (uint32_t i = 0; i < 256; ++i) {
            uint32_t c = i;
            for (int k = 0; k < 8; ++k) c = (c & 1u) ? 0xEDB88320u ^ (c >> 1) : (c >> 1);
            table[i] = c;
        }
        init = true;
    }
    uint32_t crc = 0xFFFFFFFFu;
    const auto* p = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < len; ++i) crc = table[(crc ^ p[i]) & 0xFFu] ^ (crc >> 8);
    return ~crc;
}

// ---------------------------------------------------------------- loader ----
struct RawTensor {
    std::vector<size_t> shape;
    std::vector<float> data;
};
struct RawCkpt {
    nlohmann::ordered_json header;
    std::map<std::string, RawTensor> t;
};

RawCkpt read_file(const std::string& path) {  // checkpoint.cpp:134-197
    std::ifstream f(path, std::ios::binary);
    if (!f) throw std::runtime_error("cannot open '" + path + "'");
    std::vector<uint8_t> b((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    if (b.size() < 12 || std::memcmp(b.data(), "FSVD15", 6) != 0) throw std::runtime_error("bad magic");
    uint16_t ver;
    uint32_t hl;
    std::memcpy(&ver, b.data() + 6, 2);
    std::memcpy(&hl, b.data() + 8, 4);
    if (ver != 1) throw std::runtime_error("bad version");
    RawCkpt ck;
    ck.header = nlohmann::ordered_json::parse(b.begin() + 12, b.begin() + 12 + hl);
    const size_t base = (12 + hl + 63) / 64 * 64;
    for (const auto& e : ck.header.at("tensors")) {
        RawTensor t;
        t.shape = e.at("shape").get<std::vector<size_t>>();
        size_t n = 1;
        for (size_t s : t.shape) n *= s;
        const size_t off = e.at("offset").get<size_t>();
        if (base + off + n * 4 > b.size()) throw std::runtime_error("truncated tensor");
        if (crc32(b.data() + base + off, n * 4) != e.at("crc32").get<uint32_t>())
            throw std::runtime_error("checksum mismatch");
        t.data.resize(n);
        std::memcpy(t.data.data(), b.data() + base + off, n * 4);
        ck.t[e.at("name").get<std::string>()] = std::move(t);
    }
    return ck;
}

std::shared_ptr<Mat> mat_of(const RawCkpt& ck, const std::string& name) {
    auto it = ck.t.find(name);
    if (it == ck.t.end() || it->second.shape.size() != 2) throw std::runtime_error("missing matrix " + name);
    auto m = std::make_shared<Mat>(it->second.shape[0], it->second.shape[1]);
    m->v = it->second.data;
    return m;
}
std::vector<float> vec_of(const RawCkpt& ck, const std::string& name) {
    auto it = ck.t.find(name);
    if (it == ck.t.end()) throw std::runtime_error("missing vector " + name);
    return it->second.data;
}

void finish_model(Model& m) {  // canonical.cpp:189-192 pack_ffn
    for (auto& L : m.layers) {
        const Mat& up = *L.p[4].a;
        const Mat& gate = *L.p[5].a;
        L.a_ug = Mat(up.rows, up.cols + gate.cols);
        for (size_t i = 0; i < up.rows; ++i) {
            for (size_t j = 0; j < up.cols; ++j) L.a_ug.v[i * L.a_ug.cols + j] = up.at(i, j);
            for (size_t j = 0; j < gate.cols; ++j) L.a_ug.v[i * L.a_ug.cols + up.cols + j] = gate.at(i, j);
        }
        L.r_up = L.p[4].rank;
    }
}

Model normalize(const RawCkpt& ck) {  // canonical.cpp:155-194 (+ family D)
    Model m;
    const auto& cj = ck.header.at("config");
    m.c.L = cj.at("n_layers");
    m.c.d = cj.at("d_model");
    m.c.H = cj.at("n_heads");
    m.c.dh = cj.at("d_head");
    m.c.dff = cj.at("d_ff");
    m.c.V = cj.at("vocab");
    m.c.rope_base = cj.at("rope_base");
    m.c.eps = cj.at("norm_eps");
    m.capacity = ck.header.contains("capacity") ? ck.header.at("capacity").get<size_t>() : 0;
    const std::string fam = ck.header.at("family");
    m.emb = *mat_of(ck, "embedding");
    m.head = *mat_of(ck, "head");
    m.final_gamma = vec_of(ck, "final_gamma");
    m.layers.resize(m.c.L);
    std::map<std::string, std::shared_ptr<Mat>> shared;
    std::vector<size_t> groups;
    if (fam == "C") groups = ck.header.at("layer_groups").get<std::vector<size_t>>();
    for (size_t l = 0; l < m.c.L; ++l) {
        Layer& L = m.layers[l];
        const std::string base = "layers." + std::to_string(l) + ".";
        L.attn_gamma = vec_of(ck, base + "attn_gamma");
        L.mlp_gamma = vec_of(ck, base + "mlp_gamma");
        for (int p = 0; p < 7; ++p) {
            const std::string pb = base + kProj[p];
            Factor& f = L.p[p];
            if (fam == "A") {
                f.a = mat_of(ck, pb + ".A");
                f.b = mat_of(ck, pb + ".B");
            } else if (fam == "B") {  // fold A = diag(1/s) Uf in float (canonical.cpp:97-105)
                f.a = mat_of(ck, pb + ".Uf");
                f.b = mat_of(ck, pb + ".Vt");
                const auto s = vec_of(ck, pb + ".scale");
                for (size_t i = 0; i < f.a->rows; ++i) {
                    const float inv = 1.0f / s[i];
                    for (size_t j = 0; j < f.a->cols; ++j) f.a->v[i * f.a->cols + j] *= inv;
                }
            } else if (fam == "C") {  // canonical.cpp:109-151 aliasing
                const std::string key = std::string(kProj[p]) + ":" + std::to_string(groups[l]);
                auto it = shared.find(key);
                if (it == shared.end())
                    it = shared.emplace(key, mat_of(ck, std::string("shared.") + kProj[p] + "." +
                                                             std::to_string(groups[l]) + ".A"))
                             .first;
                f.a = it->second;
                f.b = mat_of(ck, pb + ".B");
            } else if (fam == "D") {  // A = U diag(S) in float
                f.a = mat_of(ck, pb + ".U");
                f.b = mat_of(ck, pb + ".Vt");
                const auto S = vec_of(ck, pb + ".S");
                for (size_t i = 0; i < f.a->rows; ++i)
                    for (size_t j = 0; j < f.a->cols; ++j) f.a->v[i * f.a->cols + j] *= S[j];
            } else {
                throw std::runtime_error("unknown family " + fam);
            }
            f.rank = f.a->cols;
        }
    }
    m.shared_instances = shared.size();
    finish_model(m);
    return m;
}

// ------------------------------------------------------ synthetic model ----
// Restatement of include/fsvd/synth.hpp: one SplitMix64 stream, element k =
// mix(seed + (k+1) * golden); U(+-sqrt(1/fan_in)) rounded to f32 then to
// bf16 (RNE). Ranks via rank_for_ratio (compress.cpp:68-80) + optional
// jitter from a side stream (families B/D).
u64 mix(u64 z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
float bf16_round(float x) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    if ((u & 0x7F800000u) != 0x7F800000u) {
        u += 0x7FFFu + ((u >> 16) & 1u);
        u &= 0xFFFF0000u;
    }
    float y;
    std::memcpy(&y, &u, 4);
    return y;
}
struct Stream {
    u64 seed, cursor = 0;
    float draw(int kind, double amp) {
        const u64 z = mix(seed + (++cursor) * 0x9E3779B97F4A7C15ull);
        const double unit = static_cast<double>(z >> 11) * 0x1.0p-53;
        double v;
        if (kind == 1)
            v = 1.0 + (2.0 * unit - 1.0) * amp;
        else if (kind == 2)
            v = 0.5 + unit;
        else
            v = (2.0 * unit - 1.0) * amp;
        return bf16_round(static_cast<float>(v));
    }
};
size_t rank_for_ratio(double rho, size_t m, size_t n) {
    const size_t mn = std::min(m, n);
    if (rho >= 1.0) return mn;
    long long r = std::llround(rho * double(m) * double(n) / double(m + n));
    return static_cast<size_t>(std::clamp<long long>(r, 1, static_cast<long long>(mn)));
}

// Fill `count` draws in parallel (positions cursor+1 ..), deterministic.
void fill(Stream& st, float* dst, size_t count, int kind, double amp) {
    const u64 base = st.cursor;
    const int T = std::max(1, std::min(g_threads, int(count / 65536) + 1));
    std::vector<std::thread> ts;
    for (int t = 0; t < T; ++t)
        ts.emplace_back([&, t] {
            Stream s{st.seed, base + count * t / T};
            for (size_t i = count * t / T; i < count * (t + 1) / T; ++i) dst[i] = s.draw(kind, amp);
        });
    for (auto& t : ts) t.join();
    st.cursor = base + count;
}

Model synthetic(const Config& c, size_t cap, char family, double rho, size_t group, u64 seed, bool conditioned,
                double jitter) {
    Model m;
    m.c = c;
    m.capacity = cap;
    Stream st{seed};
    Stream js{seed ^ 0xD1B54A32D192ED03ull};
    std::vector<std::array<size_t, 7>> ranks(c.L);
    for (size_t l = 0; l < c.L; ++l)
        for (int p = 0; p < 7; ++p) {
            size_t din, dout;
            dims(c, p, din, dout);
            size_t r = rank_for_ratio(rho, din, dout);
            const double u = static_cast<double>(mix(js.seed + (++js.cursor) * 0x9E3779B97F4A7C15ull) >> 11) * 0x1.0p-53;
            if ((family == 'B' || family == 'D') && jitter > 0) {
                long long rj = std::llround(double(r) * (1.0 + jitter * (2.0 * u - 1.0)));
                r = static_cast<size_t>(std::clamp<long long>(rj, 1, static_cast<long long>(std::min(din, dout))));
            }
            ranks[l][p] = r;
        }
    auto amp = [](size_t n) { return std::sqrt(1.0 / double(n)); };
    m.emb = Mat(c.V, c.d);
    fill(st, m.emb.v.data(), m.emb.v.size(), 0, amp(c.V));
    m.layers.resize(c.L);
    std::map<std::string, std::shared_ptr<Mat>> shared;
    for (size_t l = 0; l < c.L; ++l) {
        Layer& L = m.layers[l];
        for (int p = 0; p < 7; ++p) {
            size_t din, dout;
            dims(c, p, din, dout);
            const size_t r = ranks[l][p];
            Factor& f = L.p[p];
            f.rank = r;
            f.b = std::make_shared<Mat>(r, dout);
            if (family == 'C') {
                const std::string key = std::string(kProj[p]) + ":" + std::to_string(l / group);
                if (l % group == 0) {
                    auto a = std::make_shared<Mat>(din, r);
                    fill(st, a->v.data(), a->v.size(), 0, amp(din));
                    shared[key] = a;
                }
                f.a = shared.at(key);
                fill(st, f.b->v.data(), f.b->v.size(), 0, amp(r));
            } else {
                f.a = std::make_shared<Mat>(din, r);
                if (family == 'D') {
                    fill(st, f.a->v.data(), f.a->v.size(), 0, amp(din));
                    std::vector<float> S(r);
                    fill(st, S.data(), r, 2, 0.0);
                    fill(st, f.b->v.data(), f.b->v.size(), 0, amp(r));
                    for (size_t i = 0; i < din; ++i)
                        for (size_t j = 0; j < r; ++j) f.a->v[i * r + j] *= S[j];
                } else {
                    fill(st, f.a->v.data(), f.a->v.size(), 0, amp(din));
                    fill(st, f.b->v.data(), f.b->v.size(), 0, amp(r));
                    if (family == 'B') {
                        std::vector<float> s(din);
                        fill(st, s.data(), din, 2, 0.0);
                        for (size_t i = 0; i < din; ++i) {
                            const float inv = 1.0f / s[i];
                            for (size_t j = 0; j < r; ++j) f.a->v[i * r + j] *= inv;
                        }
                    }
                }
            }
        }
        L.attn_gamma.resize(c.d);
        L.mlp_gamma.resize(c.d);
        fill(st, L.attn_gamma.data(), c.d, conditioned ? 1 : 0, conditioned ? 0.1 : amp(c.d));
        fill(st, L.mlp_gamma.data(), c.d, conditioned ? 1 : 0, conditioned ? 0.1 : amp(c.d));
    }
    m.final_gamma.resize(c.d);
    fill(st, m.final_gamma.data(), c.d, conditioned ? 1 : 0, conditioned ? 0.1 : amp(c.d));
    m.head = Mat(c.d, c.V);
    fill(st, m.head.v.data(), m.head.v.size(), 0, amp(c.d));
    m.shared_instances = shared.size();
    finish_model(m);
    return m;
}

// --------------------------------------------------------------- runtime ----
template <typename T>
void lowrank(T* y, const T* x, const Factor& f, std::vector<T>& tmp) {  // y = (x.A).B
    tmp.resize(f.rank);
    gemv_any<T>(tmp.data(), x, *f.a);
    gemv_any<T>(y, tmp.data(), *f.b);
}

template <typename T>
struct Session {
    const Model* m;
    size_t cap;
    int ffn;  // 1 no_merge, 2 packed
    size_t pos = 0;
    std::vector<T> K, V;  // [L][H][cap][dh]
    Session(const Model* mm, size_t c, int f) : m(mm), cap(c), ffn(f) {
        const size_t n = mm->c.L * mm->c.H * c * mm->c.dh;
        K.assign(n, T(0));
        V.assign(n, T(0));
    }
    T* krow(size_t l, size_t h, size_t p) { return &K[((l * m->c.H + h) * cap + p) * m->c.dh]; }
    T* vrow(size_t l, size_t h, size_t p) { return &V[((l * m->c.H + h) * cap + p) * m->c.dh]; }

    // SPEC.md:323-331
    void ffn_apply(const Layer& L, const T* xn, T* out) {
        const Config& c = m->c;
        std::vector<T> u(c.dff), g(c.dff), h(c.dff), tmp;
        if (ffn == 2) {
            std::vector<T> p(L.a_ug.cols);
            gemv_any<T>(p.data(), xn, L.a_ug);  // one packed input-side projection
            gemv_any<T>(u.data(), p.data(), *L.p[4].b);
            gemv_any<T>(g.data(), p.data() + L.r_up, *L.p[5].b);
        } else {
            lowrank<T>(u.data(), xn, L.p[4], tmp);
            lowrank<T>(g.data(), xn, L.p[5], tmp);
        }
        silu_mul<T>(h.data(), g.data(), u.data(), c.dff);
        lowrank<T>(out, h.data(), L.p[6], tmp);
    }

    void head(const T* x, T* logits) {
        const Config& c = m->c;
        std::vector<T> xn(c.d);
        rmsnorm<T>(xn.data(), x, m->final_gamma, c.d, static_cast<T>(c.eps));
        gemv_any<T>(logits, xn.data(), m->head);
    }

    // SPEC.md:314-322
    void decode_step(int token, T* logits) {
        const Config& c = m->c;
        if (pos >= cap) throw std::runtime_error("capacity");
        std::vector<T> x(c.d), xn(c.d), q(c.d), k(c.d), v(c.d), att(c.d), o(c.d), tmp;
        for (size_t i = 0; i < c.d; ++i) x[i] = static_cast<T>(m->emb.at(static_cast<size_t>(token), i));
        const T scale = static_cast<T>(1.0 / std::sqrt(static_cast<double>(c.dh)));
        Online<T> st;
        for (size_t l = 0; l < c.L; ++l) {
            const Layer& L = m->layers[l];
            rmsnorm<T>(xn.data(), x.data(), L.attn_gamma, c.d, static_cast<T>(c.eps));
            lowrank<T>(q.data(), xn.data(), L.p[0], tmp);
            lowrank<T>(k.data(), xn.data(), L.p[1], tmp);
            lowrank<T>(v.data(), xn.data(), L.p[2], tmp);
            for (size_t h = 0; h < c.H; ++h) {
                rope<T>(q.data() + h * c.dh, c.dh, static_cast<double>(pos), c.rope_base);
                rope<T>(k.data() + h * c.dh, c.dh, static_cast<double>(pos), c.rope_base);
                std::copy(k.begin() + h * c.dh, k.begin() + (h + 1) * c.dh, krow(l, h, pos));
                std::copy(v.begin() + h * c.dh, v.begin() + (h + 1) * c.dh, vrow(l, h, pos));
            }
            for (size_t h = 0; h < c.H; ++h) {  // one contiguous block
                st.reset(c.dh);
                st.update(q.data() + h * c.dh, krow(l, h, 0), vrow(l, h, 0), pos + 1, c.dh, c.dh, scale);
                st.finish(att.data() + h * c.dh, c.dh);
            }
            lowrank<T>(o.data(), att.data(), L.p[3], tmp);
            for (size_t i = 0; i < c.d; ++i) x[i] += o[i];
            rmsnorm<T>(xn.data(), x.data(), L.mlp_gamma, c.d, static_cast<T>(c.eps));
            ffn_apply(L, xn.data(), o.data());
            for (size_t i = 0; i < c.d; ++i) x[i] += o[i];
        }
        head(x.data(), logits);
        ++pos;
    }

    // P = X.A once for the prompt; K/V reconstructed and
    // RoPE'd in blocks of 64 and written to the cache; causal online softmax
    // over 64-key blocks.
    // FFN of n rows at once (ffn_apply row by row, bitwise: gemv_rows)
    void ffn_rows(const Layer& L, const Rows<T>& xn, Rows<T>& out) {
        const Config& c = m->c;
        const size_t n = xn.r.size();
        Rows<T> u(n, c.dff), g(n, c.dff), h(n, c.dff);
        const auto xp = xn.cp();
        if (ffn == 2) {
            Rows<T> p(n, L.a_ug.cols);
            gemv_rows<T>(n, xp.data(), p.p.data(), L.a_ug);
            gemv_rows<T>(n, p.cp().data(), u.p.data(), *L.p[4].b);
            gemv_rows<T>(n, p.cp(L.r_up).data(), g.p.data(), *L.p[5].b);
        } else {
            Rows<T> pu(n, L.p[4].rank), pg(n, L.p[5].rank);
            gemv_rows<T>(n, xp.data(), pu.p.data(), *L.p[4].a);
            gemv_rows<T>(n, pu.cp().data(), u.p.data(), *L.p[4].b);
            gemv_rows<T>(n, xp.data(), pg.p.data(), *L.p[5].a);
            gemv_rows<T>(n, pg.cp().data(), g.p.data(), *L.p[5].b);
        }
        for (size_t t = 0; t < n; ++t) silu_mul<T>(h.p[t], g.p[t], u.p[t], c.dff);
        Rows<T> pd(n, L.p[6].rank);
        gemv_rows<T>(n, h.cp().data(), pd.p.data(), *L.p[6].a);
        gemv_rows<T>(n, pd.cp().data(), out.p.data(), *L.p[6].b);
    }

    // P = X.A once for the prompt; K/V reconstructed and
    // RoPE'd (the SPEC's 64-row blocks; rows are independent, so the blocking
    // does not change any value) and written to the cache; causal online
    // softmax over 64-key blocks. Row-batched (gemv_rows): bitwise the same as
    // token-by-token gemv.
    void prefill(const int* tok, size_t T_, T* logits) {
        const Config& c = m->c;
        if (T_ == 0) throw std::runtime_error("shape");
        if (pos + T_ > cap) throw std::runtime_error("capacity");
        const size_t p0 = pos, blk = 64;
        Rows<T> X(T_, c.d);
        for (size_t t = 0; t < T_; ++t)
            for (size_t i = 0; i < c.d; ++i) X.r[t][i] = static_cast<T>(m->emb.at(static_cast<size_t>(tok[t]), i));
        const T scale = static_cast<T>(1.0 / std::sqrt(static_cast<double>(c.dh)));
        Rows<T> XN(T_, c.d), Q(T_, c.d), Kr(T_, c.d), Vr(T_, c.d), A(T_, c.d), O(T_, c.d);
        for (size_t l = 0; l < c.L; ++l) {
            const Layer& L = m->layers[l];
            for (size_t t = 0; t < T_; ++t)
                rmsnorm<T>(XN.p[t], X.p[t], L.attn_gamma, c.d, static_cast<T>(c.eps));
            const auto xn = XN.cp();
            Rows<T>* outs[3] = {&Q, &Kr, &Vr};
            for (int j = 0; j < 3; ++j) {
                Rows<T> P(T_, L.p[j].rank);
                gemv_rows<T>(T_, xn.data(), P.p.data(), *L.p[j].a);
                gemv_rows<T>(T_, P.cp().data(), outs[j]->p.data(), *L.p[j].b);
            }
            for (size_t t = 0; t < T_; ++t) {
                const double ps = static_cast<double>(p0 + t);
                for (size_t h = 0; h < c.H; ++h) {
                    rope<T>(Q.p[t] + h * c.dh, c.dh, ps, c.rope_base);
                    rope<T>(Kr.p[t] + h * c.dh, c.dh, ps, c.rope_base);
                    std::copy(Kr.p[t] + h * c.dh, Kr.p[t] + (h + 1) * c.dh, krow(l, h, p0 + t));
                    std::copy(Vr.p[t] + h * c.dh, Vr.p[t] + (h + 1) * c.dh, vrow(l, h, p0 + t));
                }
            }
            Online<T> st;
            for (size_t t = 0; t < T_; ++t) {
                const size_t nk = p0 + t + 1;
                for (size_t h = 0; h < c.H; ++h) {
                    st.reset(c.dh);
                    for (size_t k0 = 0; k0 < nk; k0 += blk)
                        st.update(Q.p[t] + h * c.dh, krow(l, h, k0), vrow(l, h, k0), std::min(blk, nk - k0), c.dh,
                                  c.dh, scale);
                    st.finish(A.p[t] + h * c.dh, c.dh);
                }
            }
            {
                Rows<T> P(T_, L.p[3].rank);
                gemv_rows<T>(T_, A.cp().data(), P.p.data(), *L.p[3].a);
                gemv_rows<T>(T_, P.cp().data(), O.p.data(), *L.p[3].b);
            }
            for (size_t t = 0; t < T_; ++t)
                for (size_t i = 0; i < c.d; ++i) X.r[t][i] += O.r[t][i];
            for (size_t t = 0; t < T_; ++t)
                rmsnorm<T>(XN.p[t], X.p[t], L.mlp_gamma, c.d, static_cast<T>(c.eps));
            ffn_rows(L, XN, O);
            for (size_t t = 0; t < T_; ++t)
                for (size_t i = 0; i < c.d; ++i) X.r[t][i] += O.r[t][i];
        }
        head(X.p[T_ - 1], logits);
        pos = p0 + T_;
    }
};

// full no-cache causal forward, naive softmax, no_merge
// FFN, structure of proj/src/model.cpp:204-285.
template <typename T>
void forward_nocache(const Model& m, const int* tok, size_t T_, T* logits /* T_ x V */) {
    const Config& c = m.c;
    std::vector<std::vector<T>> X(T_, std::vector<T>(c.d)), Q(T_, std::vector<T>(c.d)), K(T_, std::vector<T>(c.d)),
        Vv(T_, std::vector<T>(c.d)), A(T_, std::vector<T>(c.d));
    for (size_t t = 0; t < T_; ++t)
        for (size_t i = 0; i < c.d; ++i) X[t][i] = static_cast<T>(m.emb.at(static_cast<size_t>(tok[t]), i));
    const T scale = static_cast<T>(1.0 / std::sqrt(static_cast<double>(c.dh)));
    std::vector<T> xn(c.d), o(c.d), tmp, scores(T_);
    for (size_t l = 0; l < c.L; ++l) {
        const Layer& L = m.layers[l];
        for (size_t t = 0; t < T_; ++t) {
            rmsnorm<T>(xn.data(), X[t].data(), L.attn_gamma, c.d, static_cast<T>(c.eps));
            lowrank<T>(Q[t].data(), xn.data(), L.p[0], tmp);
            lowrank<T>(K[t].data(), xn.data(), L.p[1], tmp);
            lowrank<T>(Vv[t].data(), xn.data(), L.p[2], tmp);
            for (size_t h = 0; h < c.H; ++h) {
                rope<T>(Q[t].data() + h * c.dh, c.dh, static_cast<double>(t), c.rope_base);
                rope<T>(K[t].data() + h * c.dh, c.dh, static_cast<double>(t), c.rope_base);
            }
        }
        for (size_t t = 0; t < T_; ++t)
            for (size_t h = 0; h < c.H; ++h) {
                const T* qh = Q[t].data() + h * c.dh;
                T mx = T(-1e300);
                for (size_t j = 0; j <= t; ++j) {
                    scores[j] = dot(qh, K[j].data() + h * c.dh, c.dh) * scale;
                    if (scores[j] > mx) mx = scores[j];
                }
                T den = T(0);
                for (size_t j = 0; j <= t; ++j) {
                    scores[j] = std::exp(scores[j] - mx);
                    den += scores[j];
                }
                T* out = A[t].data() + h * c.dh;
                std::fill(out, out + c.dh, T(0));
                for (size_t j = 0; j <= t; ++j) {
                    const T w = scores[j] / den;
                    const T* vr = Vv[j].data() + h * c.dh;
                    for (size_t i = 0; i < c.dh; ++i) out[i] += w * vr[i];
                }
            }
        for (size_t t = 0; t < T_; ++t) {
            lowrank<T>(o.data(), A[t].data(), L.p[3], tmp);
            for (size_t i = 0; i < c.d; ++i) X[t][i] += o[i];
        }
        Session<T> dummy(&m, 1, 1);
        for (size_t t = 0; t < T_; ++t) {
            rmsnorm<T>(xn.data(), X[t].data(), L.mlp_gamma, c.d, static_cast<T>(c.eps));
            dummy.ffn_apply(L, xn.data(), o.data());
            for (size_t i = 0; i < c.d; ++i) X[t][i] += o[i];
        }
    }
    std::vector<T> fn(c.d);
    for (size_t t = 0; t < T_; ++t) {
        rmsnorm<T>(fn.data(), X[t].data(), m.final_gamma, c.d, static_cast<T>(c.eps));
        gemv_any<T>(logits + t * c.V, fn.data(), m.head);
    }
}

}  // namespace oracle

// ===================================================================== C ABI
using namespace oracle;

namespace {
thread_local std::string g_err;
template <typename F>
int wrap(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return e.what() == std::string("capacity") ? 4 : (e.what() == std::string("shape") ? 1 : 99);
    }
}
struct Sess {
    std::unique_ptr<Session<float>> f;
    std::unique_ptr<Session<double>> d;
};
}  // namespace

extern "C" {

const char* oracle_last_error() { return g_err.c_str(); }
void oracle_set_threads(int n) { g_threads = n < 1 ? 1 : n; }
void oracle_set_ref_gemv(void* fn) { g_ref_gemv = reinterpret_cast<RefGemvF32>(fn); }

void* oracle_load_file(const char* path) {
    Model* m = nullptr;
    if (wrap([&] { m = new Model(normalize(read_file(path))); })) return nullptr;
    return m;
}

void* oracle_synthetic(const uint64_t* cfg6, const double* cfg2, uint64_t cap, char family, double rho,
                       uint64_t group, uint64_t seed, int conditioned, double jitter) {
    Config c;
    c.L = cfg6[0];
    c.d = cfg6[1];
    c.H = cfg6[2];
    c.dh = cfg6[3];
    c.dff = cfg6[4];
    c.V = cfg6[5];
    c.rope_base = cfg2[0];
    c.eps = cfg2[1];
    Model* m = nullptr;
    if (wrap([&] { m = new Model(synthetic(c, cap, family, rho, group, seed, conditioned != 0, jitter)); }))
        return nullptr;
    return m;
}

void oracle_free_model(void* m) { delete static_cast<Model*>(m); }

uint64_t oracle_shared_instances(void* m) { return static_cast<Model*>(m)->shared_instances; }

uint64_t oracle_rank(void* mp, uint64_t layer, int proj) {
    return static_cast<Model*>(mp)->layers.at(layer).p[proj].rank;
}

int oracle_tensor(void* mp, const char* name, float* out, uint64_t count) {
    return wrap([&] {
        const Model& m = *static_cast<Model*>(mp);
        const std::string n(name);
        const std::vector<float>* v = nullptr;
        if (n == "embedding") v = &m.emb.v;
        else if (n == "head") v = &m.head.v;
        else if (n == "final_gamma") v = &m.final_gamma;
        else {
            const size_t dot1 = n.find('.', 7);
            const size_t l = std::stoul(n.substr(7, dot1 - 7));
            const std::string rest = n.substr(dot1 + 1);
            const Layer& L = m.layers.at(l);
            if (rest == "attn_gamma") v = &L.attn_gamma;
            else if (rest == "mlp_gamma") v = &L.mlp_gamma;
            else if (rest == "a_ug") v = &L.a_ug.v;
            else
                for (int p = 0; p < 7; ++p) {
                    if (rest == std::string(kProj[p]) + ".A") v = &L.p[p].a->v;
                    if (rest == std::string(kProj[p]) + ".B") v = &L.p[p].b->v;
                }
        }
        if (!v) throw std::runtime_error("unknown tensor " + n);
        if (v->size() != count) throw std::runtime_error("count mismatch for " + n);
        std::memcpy(out, v->data(), count * 4);
    });
}

void* oracle_session(void* mp, int f64, int ffn, uint64_t cap) {
    auto* s = new Sess();
    const Model* m = static_cast<Model*>(mp);
    if (f64)
        s->d = std::make_unique<Session<double>>(m, cap, ffn);
    else
        s->f = std::make_unique<Session<float>>(m, cap, ffn);
    return s;
}
void oracle_free_session(void* s) { delete static_cast<Sess*>(s); }
// Independent copy of a session (KV cache and position): forks one prompt
// prefix into several continuations without recomputing it (tests only).
void* oracle_clone_session(void* sp) {
    const Sess& s = *static_cast<Sess*>(sp);
    auto* c = new Sess();
    if (s.d) c->d = std::make_unique<Session<double>>(*s.d);
    if (s.f) c->f = std::make_unique<Session<float>>(*s.f);
    return c;
}

int oracle_prefill(void* sp, const int32_t* tok, uint64_t T, double* logits) {
    return wrap([&] {
        Sess& s = *static_cast<Sess*>(sp);
        std::vector<int> t(tok, tok + T);
        if (s.d) {
            s.d->prefill(t.data(), T, logits);
        } else {
            std::vector<float> lf(s.f->m->c.V);
            s.f->prefill(t.data(), T, lf.data());
            for (size_t i = 0; i < lf.size(); ++i) logits[i] = lf[i];
        }
    });
}

int oracle_decode(void* sp, int32_t token, double* logits) {
    return wrap([&] {
        Sess& s = *static_cast<Sess*>(sp);
        if (s.d) {
            s.d->decode_step(token, logits);
        } else {
            std::vector<float> lf(s.f->m->c.V);
            s.f->decode_step(token, lf.data());
            for (size_t i = 0; i < lf.size(); ++i) logits[i] = lf[i];
        }
    });
}

// prefill, then greedy steps; max_new tokens total.
int oracle_generate(void* sp, const int32_t* prompt, uint64_t T, uint64_t max_new, int32_t* out) {
    return wrap([&] {
        Sess& s = *static_cast<Sess*>(sp);
        const size_t V = s.d ? s.d->m->c.V : s.f->m->c.V;
        std::vector<double> lg(V);
        if (max_new == 0) {
            oracle_prefill(sp, prompt, T, lg.data());
            return;
        }
        if (oracle_prefill(sp, prompt, T, lg.data())) throw std::runtime_error(g_err);
        for (size_t i = 0; i < max_new; ++i) {
            const int tok = static_cast<int>(argmax(lg.data(), V));
            out[i] = tok;
            if (i + 1 < max_new && oracle_decode(sp, tok, lg.data())) throw std::runtime_error(g_err);
        }
    });
}

int oracle_forward_nocache(void* mp, int f64, const int32_t* tok, uint64_t T, double* logits) {
    return wrap([&] {
        const Model& m = *static_cast<Model*>(mp);
        std::vector<int> t(tok, tok + T);
        if (f64) {
            forward_nocache<double>(m, t.data(), T, logits);
        } else {
            std::vector<float> lf(T * m.c.V);
            forward_nocache<float>(m, t.data(), T, lf.data());
            for (size_t i = 0; i < lf.size(); ++i) logits[i] = lf[i];
        }
    });
}

int oracle_read_kv(void* sp, uint64_t layer, int which, uint64_t pos0, uint64_t n, double* out) {
    return wrap([&] {
        Sess& s = *static_cast<Sess*>(sp);
        auto get = [&](auto& S) {
            const Config& c = S.m->c;
            for (size_t p = 0; p < n; ++p)
                for (size_t h = 0; h < c.H; ++h) {
                    const auto* r = which ? S.vrow(layer, h, pos0 + p) : S.krow(layer, h, pos0 + p);
                    for (size_t i = 0; i < c.dh; ++i) out[p * c.d + h * c.dh + i] = r[i];
                }
        };
        if (s.d)
            get(*s.d);
        else
            get(*s.f);
    });
}

uint64_t oracle_position(void* sp) {
    Sess& s = *static_cast<Sess*>(sp);
    return s.d ? s.d->pos : s.f->pos;
}

// primitive hooks for the pinning tests (f64)
void oracle_rope_f64(double* v, uint64_t d, double pos, double base) { rope<double>(v, d, pos, base); }
void oracle_rmsnorm_f64(double* y, const double* x, const float* g, uint64_t n, double eps) {
    std::vector<float> gv(g, g + n);
    rmsnorm<double>(y, x, gv, n, eps);
}
void oracle_rmsnorm_f32(float* y, const float* x, const float* g, uint64_t n, float eps) {
    std::vector<float> gv(g, g + n);
    rmsnorm<float>(y, x, gv, n, eps);
}
void oracle_gemv_f32(float* y, const float* x, const float* a, uint64_t m, uint64_t n) {
    Mat A(m, n);
    std::memcpy(A.v.data(), a, m * n * 4);
    gemv<float>(y, x, A);
}
// online softmax over blocks of the given sizes (f64)
void oracle_online_attend_f64(const double* q, const double* k, const double* v, uint64_t rows, uint64_t d,
                              double scale, const uint64_t* blocks, uint64_t nblocks, double* out) {
    Online<double> st;
    st.reset(d);
    size_t r0 = 0;
    for (size_t b = 0; b < nblocks; ++b) {
        st.update(q, k + r0 * d, v + r0 * d, blocks[b], d, d, scale);
        r0 += blocks[b];
    }
    (void)rows;
    st.finish(out, d);
}
uint64_t oracle_rng_u64(uint64_t seed, uint64_t k) { return mix(seed + (k + 1) * 0x9E3779B97F4A7C15ull); }
uint64_t oracle_rank_for_ratio(double rho, uint64_t m, uint64_t n) { return rank_for_ratio(rho, m, n); }
uint64_t oracle_argmax_f64(const double* x, uint64_t n) { return argmax(x, n); }

}  // extern "C"
