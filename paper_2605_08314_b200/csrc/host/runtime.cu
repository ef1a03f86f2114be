// Device model + session runtime (SPEC.md runtime :283-382, plan :384-446).
//
// Decode step = one phase program run by the persistent
// megakernel (csrc/cuda/decode_mk.cu), per layer:
//   qkvA   p_qkv = rmsnorm(x) . [A_q|A_k|A_v]         (packed QKV projection)
//   qkvB   q,k,v = p . B_{q,k,v}; RoPE(q,k) at pos; k,v -> cache row pos
//   attn   dense-KV attention over cache rows [0, pos]
//   oA/oB  x += (attn . A_o) . B_o
//   ugA    p_ug = rmsnorm(x) . [A_up|A_gate]          (packed; no_merge = 2 phases)
//   ugB    h = silu(p_g . B_gate) * (p_u . B_up)
//   dA/dB  x += (h . A_down) . B_down
// framed by the embedding gather and the head + greedy argmax that advances
// the device length register. Plans: eager =
// one launch per phase, per_layer = one CUDA graph per layer, full_step = one
// graph per step -- the same phases, so bitwise identical outputs.
// Prefill runs the chunked GEMM path.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <exception>
#include <mutex>
#include <set>
#include <cstdlib>
#include <cstring>
#include <thread>

#include "runtime.h"
#include "fsvd/crc32.hpp"

namespace fsvd::rt {

void cuda_check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        throw OomError(std::string("CUDA out of memory: ") + what);
    }
    throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------ device model --

DeviceModel::~DeviceModel() {
    if (arena) {
        cudaSetDevice(device);
        cudaFree(arena);
    }
}

void* DeviceModel::alloc(size_t bytes) {
    const size_t a = (used + 255) & ~size_t(255);
    if (a + bytes > arena_bytes) throw OomError("device model arena exhausted");
    used = a + bytes;
    return static_cast<char*>(arena) + a;
}

namespace {

void init_model_shapes(DeviceModel& dm, const ModelConfig& c, size_t cap, fsvd_dtype dt, int device) {
    dm.cfg = c;
    dm.capacity = cap;
    dm.wt = dt == FSVD_DTYPE_BF16 ? k::kBF16 : k::kF32;
    dm.esize = dt == FSVD_DTYPE_BF16 ? 2 : 4;
    dm.device = device;
    dm.ldd = pad64(c.d_model);
    dm.ldff = pad64(c.d_ff);
    FSVD_CUDA(cudaSetDevice(device));
    FSVD_CUDA(cudaDeviceGetAttribute(&dm.sm_count, cudaDevAttrMultiProcessorCount, device));
}

DeviceMatrix make_matrix(int rows, int kk, int esize) {
    DeviceMatrix m;
    m.rows = rows;
    m.k = kk;
    m.kp = k::pad_line(kk, esize);
    return m;
}

// Algorithmic bytes of one B=1 decode step: every layer's
// factors once (a shared basis counts once per layer), head, gammas, one
// embedding row. KV traffic is added by the caller for the context length.
void account(DeviceModel& dm, const std::vector<std::array<size_t, kNumProj>>& ranks) {
    const ModelConfig& c = dm.cfg;
    uint64_t bytes = 0, params = 0;
    for (const auto& lr : ranks)
        for (size_t p = 0; p < kNumProj; ++p) {
            const auto dims = proj_dims(c, p);
            bytes += static_cast<uint64_t>(lr[p]) * (dims[0] + dims[1]) * dm.esize;
            params += static_cast<uint64_t>(lr[p]) * (dims[0] + dims[1]);
        }
    bytes += static_cast<uint64_t>(c.vocab) * c.d_model * dm.esize;      // head
    bytes += static_cast<uint64_t>(c.d_model) * dm.esize;                // embedding row
    bytes += static_cast<uint64_t>(2 * c.n_layers + 1) * c.d_model * 4;  // gammas (fp32)
    dm.decode_weight_bytes = bytes;
    dm.prefill_flops_per_token = 2 * params;
}

// Allocate the arena. keys[l][p] identifies projection p's input factor
// storage (nullptr = unique); equal keys share one device copy.
void allocate(DeviceModel& dm, const std::vector<std::array<size_t, kNumProj>>& ranks,
              const std::vector<std::array<const void*, kNumProj>>& keys) {
    const ModelConfig& c = dm.cfg;
    const int es = dm.esize;
    auto bytes_of = [&](const DeviceMatrix& m) { return m.layout(es).bytes(); };
    // plan sizes
    size_t total = 0;
    auto add = [&](size_t b) { total += (b + 255) & ~size_t(255); };
    add(c.vocab * dm.ldd * es);
    add(bytes_of(make_matrix(static_cast<int>(c.vocab), static_cast<int>(c.d_model), es)));
    add(c.d_model * 4);
    std::map<const void*, bool> seen;
    for (size_t l = 0; l < c.n_layers; ++l)
        for (size_t p = 0; p < kNumProj; ++p) {
            const auto dims = proj_dims(c, p);
            const void* key = keys[l][p];
            if (!key || !seen.count(key)) {
                if (key) seen[key] = true;
                add(bytes_of(make_matrix(static_cast<int>(ranks[l][p]), static_cast<int>(dims[0]), es)));
            }
            add(bytes_of(make_matrix(static_cast<int>(dims[1]), static_cast<int>(ranks[l][p]), es)));
            if (p == 0) add(2 * c.d_model * 4);
        }
    dm.arena_bytes = total + 4096;
    FSVD_CUDA(cudaSetDevice(dm.device));
    cudaError_t e = cudaMalloc(&dm.arena, dm.arena_bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw OomError("cannot allocate " + std::to_string(dm.arena_bytes) + " bytes of device weights");
    }
    FSVD_CUDA(cudaMemset(dm.arena, 0, dm.arena_bytes));
    dm.stored_weight_bytes = total;

    dm.emb = dm.alloc(c.vocab * dm.ldd * es);
    dm.head_t = make_matrix(static_cast<int>(c.vocab), static_cast<int>(c.d_model), es);
    dm.head_t.w = dm.alloc(bytes_of(dm.head_t));
    dm.final_gamma = static_cast<const float*>(dm.alloc(c.d_model * 4));
    std::map<const void*, DeviceMatrix> shared;
    dm.layers.resize(c.n_layers);
    for (size_t l = 0; l < c.n_layers; ++l) {
        DeviceLayer& L = dm.layers[l];
        // input factors first, in projection order: q|k|v and up|gate end up adjacent
        for (size_t p = 0; p < kNumProj; ++p) {
            const auto dims = proj_dims(c, p);
            L.r[p] = static_cast<int>(ranks[l][p]);
            L.rp[p] = pad64(ranks[l][p]);  // 64: the decode planes' k-permutation groups (decode_mk_common.cuh)
            const void* key = keys[l][p];
            auto it = key ? shared.find(key) : shared.end();
            if (it != shared.end()) {
                L.at[p] = it->second;
            } else {
                L.at[p] = make_matrix(L.r[p], static_cast<int>(dims[0]), es);
                L.at[p].w = dm.alloc(bytes_of(L.at[p]));
                if (key) shared[key] = L.at[p];
            }
        }
        for (size_t p = 0; p < kNumProj; ++p) {
            const auto dims = proj_dims(c, p);
            L.bt[p] = make_matrix(static_cast<int>(dims[1]), L.r[p], es);
            L.bt[p].w = dm.alloc(bytes_of(L.bt[p]));
        }
        L.attn_gamma = static_cast<const float*>(dm.alloc(c.d_model * 4));
        L.mlp_gamma = static_cast<const float*>(dm.alloc(c.d_model * 4));
    }
    account(dm, ranks);
}

inline uint16_t bf16_bits(float x) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    if ((u & 0x7F800000u) != 0x7F800000u) u += 0x7FFFu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

template <typename F>
void parallel_for(size_t n, F&& f) {
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> ts;
    for (unsigned w = 0; w < hw; ++w) ts.emplace_back([&, w] { f(n * w / hw, n * (w + 1) / hw); });
    for (auto& t : ts) t.join();
}

// Host-side tile packing: logical (row, k) of W^T = src[k * src_cols + row]
// (the reference's d_in x d_out factor, transposed on the fly).
void upload_tiles(const DeviceModel& dm, const DeviceMatrix& m, const float* src, size_t src_cols) {
    const k::WLayout lay = m.layout(dm.esize);
    std::vector<uint8_t> buf(lay.bytes(), 0);
    parallel_for(static_cast<size_t>(m.rows), [&](size_t lo, size_t hi) {
        for (size_t r = lo; r < hi; ++r)
            for (int kk = 0; kk < m.k; ++kk) {
                const float v = src[static_cast<size_t>(kk) * src_cols + r];
                uint8_t* p = buf.data() + lay.offset(static_cast<int>(r), kk);
                if (dm.esize == 2) {
                    const uint16_t h = bf16_bits(v);
                    std::memcpy(p, &h, 2);
                } else {
                    std::memcpy(p, &v, 4);
                }
            }
    });
    FSVD_CUDA(cudaMemcpy(const_cast<void*>(m.w), buf.data(), buf.size(), cudaMemcpyHostToDevice));
}

void upload_rows(const DeviceModel& dm, const void* dst, const float* src, size_t rows, size_t cols, size_t ld) {
    std::vector<uint8_t> buf(rows * ld * dm.esize, 0);
    for (size_t r = 0; r < rows; ++r)
        for (size_t c = 0; c < cols; ++c) {
            const float v = src[r * cols + c];
            if (dm.esize == 2) {
                const uint16_t h = bf16_bits(v);
                std::memcpy(buf.data() + (r * ld + c) * 2, &h, 2);
            } else {
                std::memcpy(buf.data() + (r * ld + c) * 4, &v, 4);
            }
        }
    FSVD_CUDA(cudaMemcpy(const_cast<void*>(dst), buf.data(), buf.size(), cudaMemcpyHostToDevice));
}

void upload_f32(const void* dst, const float* src, size_t n) {
    FSVD_CUDA(cudaMemcpy(const_cast<void*>(dst), src, n * 4, cudaMemcpyHostToDevice));
}

}  // namespace

std::unique_ptr<DeviceModel> upload_canonical(const CanonicalModel<float>& m, fsvd_dtype dt, int device) {
    auto dm = std::make_unique<DeviceModel>();
    init_model_shapes(*dm, m.config, m.capacity, dt, device);
    const ModelConfig& c = m.config;
    std::vector<std::array<size_t, kNumProj>> ranks(c.n_layers);
    std::vector<std::array<const void*, kNumProj>> keys(c.n_layers);
    for (size_t l = 0; l < c.n_layers; ++l)
        for (size_t p = 0; p < kNumProj; ++p) {
            const auto& f = m.layers[l].proj(p);
            ranks[l][p] = f.rank;
            keys[l][p] = f.shared_group.has_value() ? static_cast<const void*>(f.a.get()) : nullptr;
        }
    allocate(*dm, ranks, keys);
    upload_rows(*dm, dm->emb, m.embedding.data.data(), c.vocab, c.d_model, dm->ldd);
    upload_tiles(*dm, dm->head_t, m.head.data.data(), c.vocab);
    upload_f32(dm->final_gamma, m.final_gamma.data(), c.d_model);
    std::map<const void*, bool> done;
    for (size_t l = 0; l < c.n_layers; ++l) {
        const auto& L = m.layers[l];
        const DeviceLayer& D = dm->layers[l];
        for (size_t p = 0; p < kNumProj; ++p) {
            const auto& f = L.proj(p);
            const auto dims = proj_dims(c, p);
            if (!done.count(D.at[p].w)) {  // A (d_in x r) -> A^T rows r, K d_in
                upload_tiles(*dm, D.at[p], f.a->data.data(), f.rank);
                done[D.at[p].w] = true;
            }
            upload_tiles(*dm, D.bt[p], f.b->data.data(), dims[1]);  // B (r x d_out) -> B^T rows d_out, K r
        }
        upload_f32(D.attn_gamma, L.attn_gamma.data(), c.d_model);
        upload_f32(D.mlp_gamma, L.mlp_gamma.data(), c.d_model);
    }
    FSVD_CUDA(cudaDeviceSynchronize());
    dm->family = 'A';
    return dm;
}

// ------------------------------------------------------ streaming loader --
namespace {

struct FileEntry {
    std::string name;
    std::vector<size_t> shape;
    size_t off = 0;     // absolute file offset of the data
    size_t nbytes = 0;
    uint32_t crc = 0;
    size_t rows() const { return shape.size() == 2 ? shape[0] : 1; }
    size_t cols() const { return shape.size() == 2 ? shape[1] : (shape.empty() ? 0 : shape[0]); }
};

struct PosixFile {
    int fd = -1;
    explicit PosixFile(const std::string& path) : fd(::open(path.c_str(), O_RDONLY)) {}
    ~PosixFile() {
        if (fd >= 0) ::close(fd);
    }
    void read_at(void* dst, size_t n, size_t off) const {
        char* p = static_cast<char*>(dst);
        while (n) {
            const ssize_t r = ::pread(fd, p, n, static_cast<off_t>(off));
            if (r <= 0) throw FormatError("short read from checkpoint");
            p += r;
            n -= static_cast<size_t>(r);
            off += static_cast<size_t>(r);
        }
    }
};

// One destination of a tensor on the device (see k::PackArgs).
struct PackJob {
    const FileEntry* e;
    int mode;
    long long ld;
    k::WLayout lay;
    const float* scale;  // device vector (fold 1 / 2)
    int fold;
    void* dst;
    k::WType dt;
};

}  // namespace

std::unique_ptr<DeviceModel> load_streaming(const std::string& path, fsvd_dtype dt, int device, LoadStats* st) {
    const auto t0 = std::chrono::steady_clock::now();
    PosixFile f(path);
    if (f.fd < 0) throw FormatError("cannot open '" + path + "'");
    struct stat sb {};
    if (::fstat(f.fd, &sb) != 0) throw FormatError("cannot stat '" + path + "'");
    const size_t len = static_cast<size_t>(sb.st_size);
    // ---- container header: the checks and messages of read_checkpoint (checkpoint.cpp) ----
    constexpr size_t kPrefix = 12;
    if (len < kPrefix) throw FormatError("file too short for FSVD15 header");
    uint8_t pre[kPrefix];
    f.read_at(pre, kPrefix, 0);
    if (std::memcmp(pre, kCheckpointMagic, 6) != 0) throw FormatError("bad magic (not an FSVD15 file)");
    uint16_t ver;
    uint32_t hlen;
    std::memcpy(&ver, pre + 6, 2);
    std::memcpy(&hlen, pre + 8, 4);
    if (ver != kCheckpointVersion) throw FormatError("unsupported version " + std::to_string(ver));
    if (kPrefix + static_cast<size_t>(hlen) > len) throw FormatError("truncated header");
    std::string text(hlen, '\0');
    f.read_at(text.data(), hlen, kPrefix);
    Checkpoint meta;  // header + names / shapes only (no tensor data)
    try {
        meta.header = nlohmann::ordered_json::parse(text);
    } catch (const nlohmann::json::exception& e) {
        throw FormatError(std::string("header is not valid JSON: ") + e.what());
    }
    auto idx = meta.header.find("tensors");
    if (idx == meta.header.end() || !idx->is_array()) throw FormatError("header missing tensor index");
    const size_t base = (kPrefix + hlen + 63) / 64 * 64;
    std::vector<FileEntry> ents;
    ents.reserve(idx->size());
    size_t prev_end = 0;
    for (const auto& e : *idx) {
        FileEntry t;
        size_t off;
        try {
            t.name = e.at("name").get<std::string>();
            if (e.at("dtype").get<std::string>() != "f32") throw FormatError("tensor '" + t.name + "' has unsupported dtype");
            t.shape = e.at("shape").get<std::vector<size_t>>();
            off = e.at("offset").get<size_t>();
            t.crc = e.at("crc32").get<uint32_t>();
        } catch (const nlohmann::json::exception& ex) {
            throw FormatError(std::string("malformed tensor index entry: ") + ex.what());
        }
        if (off % 64) throw FormatError("tensor '" + t.name + "' offset not 64-byte aligned");
        if (!ents.empty() && off < prev_end) throw FormatError("tensor '" + t.name + "' overlaps previous tensor");
        size_t n = t.shape.empty() ? 0 : 1;
        for (size_t d : t.shape) n *= d;
        if (n == 0) throw FormatError("tensor '" + t.name + "' has empty shape");
        t.nbytes = n * sizeof(float);
        if (base + off + t.nbytes > len) throw FormatError("tensor '" + t.name + "' extends past end of file");
        t.off = base + off;
        prev_end = off + t.nbytes;
        ents.push_back(std::move(t));
        CheckpointTensor ct;
        ct.name = ents.back().name;
        ct.shape = ents.back().shape;
        meta.tensors.push_back(std::move(ct));
    }
    std::map<std::string, const FileEntry*> by_name;
    for (const auto& e : ents) by_name.emplace(e.name, &e);

    // ---- normalize<float> plan: the checks and messages of canonical.cpp ----
    const char family = meta.family();
    ModelConfig c = meta.config();
    c.validate();
    auto need_mat = [&](const std::string& n, size_t r, size_t cc) -> const FileEntry* {
        auto it = by_name.find(n);
        if (it == by_name.end()) throw NormalizeError("missing tensor '" + n + "'");
        const FileEntry* e = it->second;
        if (e->shape.size() != 2 || e->shape[0] != r || e->shape[1] != cc)
            throw NormalizeError("tensor '" + n + "' has unexpected shape");
        return e;
    };
    auto need_vec = [&](const std::string& n, size_t l) -> const FileEntry* {
        auto it = by_name.find(n);
        if (it == by_name.end()) throw NormalizeError("missing tensor '" + n + "'");
        if (it->second->nbytes / 4 != l) throw NormalizeError("tensor '" + n + "' has unexpected length");
        return it->second;
    };
    auto rank_of = [&](const std::string& n, size_t d_in) -> size_t {
        auto it = by_name.find(n);
        if (it == by_name.end()) throw NormalizeError("missing tensor '" + n + "'");
        if (it->second->shape.size() != 2 || it->second->shape[0] != d_in)
            throw NormalizeError("tensor '" + n + "' has unexpected shape");
        return it->second->shape[1];
    };
    const FileEntry* emb = need_mat("embedding", c.vocab, c.d_model);
    const FileEntry* head = need_mat("head", c.d_model, c.vocab);
    const FileEntry* fgam = need_vec("final_gamma", c.d_model);
    std::vector<std::array<const FileEntry*, 2>> gam(c.n_layers);
    for (size_t l = 0; l < c.n_layers; ++l) {
        const std::string b = "layers." + std::to_string(l) + ".";
        gam[l] = {need_vec(b + "attn_gamma", c.d_model), need_vec(b + "mlp_gamma", c.d_model)};
    }
    struct Proj {
        const FileEntry *a = nullptr, *b = nullptr, *scale = nullptr;
        size_t rank = 0;
        int fold = 0;
    };
    std::vector<std::array<Proj, kNumProj>> pj(c.n_layers);
    std::vector<std::array<size_t, kNumProj>> ranks(c.n_layers);
    std::vector<std::array<const void*, kNumProj>> keys(c.n_layers);
    if (family == 'C') {
        auto it = meta.header.find("layer_groups");
        if (it == meta.header.end() || !it->is_array() || it->size() != c.n_layers)
            throw NormalizeError("family C header missing per-layer group references");
        const auto groups = it->get<std::vector<size_t>>();
        for (size_t p = 0; p < kNumProj; ++p) {
            const auto dims = proj_dims(c, p);
            for (size_t l = 0; l < c.n_layers; ++l) {
                const std::string g = std::to_string(groups[l]);
                const std::string name = std::string("shared.") + kProjNames[p] + "." + g + ".A";
                auto sh = by_name.find(name);
                if (sh == by_name.end())
                    throw NormalizeError("layer " + std::to_string(l) + " references unknown group '" + g + "' (no '" +
                                         name + "')");
                if (sh->second->shape.size() != 2) throw NormalizeError("tensor '" + name + "' has unexpected shape");
                Proj& q = pj[l][p];
                q.a = need_mat(name, dims[0], sh->second->shape[1]);
                q.rank = q.a->shape[1];
                q.b = need_mat("layers." + std::to_string(l) + "." + kProjNames[p] + ".B", q.rank, dims[1]);
                keys[l][p] = q.a;  // one device copy per storage instance
            }
        }
    } else {
        for (size_t l = 0; l < c.n_layers; ++l)
            for (size_t p = 0; p < kNumProj; ++p) {
                const auto dims = proj_dims(c, p);
                const std::string b = "layers." + std::to_string(l) + "." + kProjNames[p];
                Proj& q = pj[l][p];
                const char* an = family == 'A' ? ".A" : family == 'B' ? ".Uf" : ".U";
                q.rank = rank_of(b + an, dims[0]);
                q.a = need_mat(b + an, dims[0], q.rank);
                q.b = need_mat(b + (family == 'A' ? ".B" : ".Vt"), q.rank, dims[1]);
                if (family == 'B') q.scale = need_vec(b + ".scale", dims[0]), q.fold = 1;
                if (family == 'D') q.scale = need_vec(b + ".S", q.rank), q.fold = 2;
                keys[l][p] = nullptr;
            }
    }
    for (size_t l = 0; l < c.n_layers; ++l)
        for (size_t p = 0; p < kNumProj; ++p) ranks[l][p] = pj[l][p].rank;

    auto dm = std::make_unique<DeviceModel>();
    init_model_shapes(*dm, c, meta.capacity(), dt, device);
    allocate(*dm, ranks, keys);
    dm->family = family;

    // fold vectors (small): read and CRC-check now, zero entries are a NormalizeError (canonical.cpp)
    std::map<const FileEntry*, float*> dscale;
    std::vector<void*> scratch;
    for (size_t l = 0; l < c.n_layers; ++l)
        for (size_t p = 0; p < kNumProj; ++p) {
            const FileEntry* se = pj[l][p].scale;
            if (!se || dscale.count(se)) continue;
            std::vector<float> v(se->nbytes / 4);
            f.read_at(v.data(), se->nbytes, se->off);
            if (crc32(v.data(), se->nbytes) != se->crc) throw FormatError("tensor '" + se->name + "' failed checksum");
            if (pj[l][p].fold == 1)
                for (float x : v)
                    if (!(std::abs(static_cast<double>(x)) > 0.0))
                        throw NormalizeError("tensor '" + se->name + "' has zero entry");
            float* d = nullptr;
            FSVD_CUDA(cudaMalloc(&d, se->nbytes));
            scratch.push_back(d);
            FSVD_CUDA(cudaMemcpy(d, v.data(), se->nbytes, cudaMemcpyHostToDevice));
            dscale[se] = d;
        }

    // ---- jobs: every tensor once, to its device destination ----
    const k::WType wt = dm->wt;
    std::vector<PackJob> jobs;
    jobs.push_back({emb, 0, dm->ldd, {}, nullptr, 0, const_cast<void*>(dm->emb), wt});
    jobs.push_back({head, 1, 0, dm->head_t.layout(dm->esize), nullptr, 0, const_cast<void*>(dm->head_t.w), wt});
    jobs.push_back({fgam, 0, static_cast<long long>(c.d_model), {}, nullptr, 0, const_cast<float*>(dm->final_gamma), k::kF32});
    std::set<const void*> done;
    for (size_t l = 0; l < c.n_layers; ++l) {
        const DeviceLayer& D = dm->layers[l];
        for (size_t p = 0; p < kNumProj; ++p) {
            const Proj& q = pj[l][p];
            if (done.insert(D.at[p].w).second)
                jobs.push_back({q.a, 1, 0, D.at[p].layout(dm->esize), q.scale ? dscale[q.scale] : nullptr, q.fold,
                                const_cast<void*>(D.at[p].w), wt});
            jobs.push_back({q.b, 1, 0, D.bt[p].layout(dm->esize), nullptr, 0, const_cast<void*>(D.bt[p].w), wt});
        }
        jobs.push_back({gam[l][0], 0, static_cast<long long>(c.d_model), {}, nullptr, 0, const_cast<float*>(D.attn_gamma), k::kF32});
        jobs.push_back({gam[l][1], 0, static_cast<long long>(c.d_model), {}, nullptr, 0, const_cast<float*>(D.mlp_gamma), k::kF32});
    }
    std::sort(jobs.begin(), jobs.end(), [](const PackJob& a, const PackJob& b) { return a.e->nbytes > b.e->nbytes; });

    // ---- workers: pread -> pinned chunk (+ CRC) -> H2D -> pack kernel, double buffered ----
    constexpr size_t kChunk = 32ull << 20;
    const int nw = static_cast<int>(std::max<size_t>(1, std::min<size_t>({8, jobs.size(), std::max(1u, std::thread::hardware_concurrency() / 2)})));
    std::atomic<size_t> next{0};
    std::atomic<uint64_t> total{0};
    std::mutex err_mu;
    std::exception_ptr err;
    auto worker = [&]() {
        cudaStream_t s = nullptr;
        void* host[2] = {nullptr, nullptr};
        float* dev[2] = {nullptr, nullptr};
        cudaEvent_t ev[2] = {nullptr, nullptr};
        try {
            FSVD_CUDA(cudaSetDevice(device));
            FSVD_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            for (int b = 0; b < 2; ++b) {
                FSVD_CUDA(cudaMallocHost(&host[b], kChunk));
                FSVD_CUDA(cudaMalloc(&dev[b], kChunk));
                FSVD_CUDA(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming));
            }
            bool used[2] = {false, false};
            int b = 0;
            for (size_t j; (j = next.fetch_add(1)) < jobs.size();) {
                const PackJob& job = jobs[j];
                const FileEntry& e = *job.e;
                const size_t rows = e.rows(), cols = e.cols(), row_bytes = cols * 4;
                const size_t rows_per = std::max<size_t>(1, kChunk / row_bytes);
                if (row_bytes > kChunk) throw ConfigError("checkpoint row larger than the loader's staging chunk");
                uint32_t crc = 0;
                for (size_t r0 = 0; r0 < rows; r0 += rows_per) {
                    const size_t nr = std::min(rows_per, rows - r0), nb = nr * row_bytes;
                    if (used[b]) FSVD_CUDA(cudaEventSynchronize(ev[b]));
                    f.read_at(host[b], nb, e.off + r0 * row_bytes);
                    crc = crc32_update(crc, host[b], nb);
                    FSVD_CUDA(cudaMemcpyAsync(dev[b], host[b], nb, cudaMemcpyHostToDevice, s));
                    k::PackArgs a{};
                    a.src = dev[b];
                    a.r0 = static_cast<long long>(r0);
                    a.nrows = static_cast<long long>(nr);
                    a.cols = static_cast<long long>(cols);
                    a.mode = job.mode;
                    a.ld = job.ld;
                    a.lay = job.lay;
                    a.scale = job.scale;
                    a.fold = job.fold;
                    a.dst = job.dst;
                    a.dt = job.dt;
                    k::pack_f32(a, s);
                    FSVD_CUDA(cudaGetLastError());
                    FSVD_CUDA(cudaEventRecord(ev[b], s));
                    used[b] = true;
                    b ^= 1;
                    total += nb;
                }
                if (crc != e.crc) throw FormatError("tensor '" + e.name + "' failed checksum");
            }
            FSVD_CUDA(cudaStreamSynchronize(s));
        } catch (...) {
            std::lock_guard<std::mutex> g(err_mu);
            if (!err) err = std::current_exception();
            next = jobs.size();
        }
        if (s) cudaStreamSynchronize(s);
        for (int b = 0; b < 2; ++b) {
            if (host[b]) cudaFreeHost(host[b]);
            if (dev[b]) cudaFree(dev[b]);
            if (ev[b]) cudaEventDestroy(ev[b]);
        }
        if (s) cudaStreamDestroy(s);
    };
    std::vector<std::thread> ts;
    for (int w = 0; w < nw; ++w) ts.emplace_back(worker);
    for (auto& t : ts) t.join();
    for (void* p : scratch) cudaFree(p);
    if (err) std::rethrow_exception(err);
    FSVD_CUDA(cudaDeviceSynchronize());
    if (st) {
        st->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        st->bytes = total.load();
        st->pinned_bytes = static_cast<uint64_t>(nw) * 2 * kChunk;
    }
    return dm;
}

std::unique_ptr<DeviceModel> generate_synthetic(const SynthSpec& spec, fsvd_dtype dt, int device) {
    const SynthLayout lay = synth_layout(spec);
    auto dm = std::make_unique<DeviceModel>();
    init_model_shapes(*dm, spec.config, spec.capacity, dt, device);
    const ModelConfig& c = spec.config;
    // family C: every projection's input factor is one storage instance per
    // layer group; use the group's first-layer tensor name as the identity
    std::vector<std::array<const void*, kNumProj>> keys(c.n_layers);
    for (size_t l = 0; l < c.n_layers; ++l)
        for (size_t p = 0; p < kNumProj; ++p)
            keys[l][p] = spec.family == 'C'
                             ? static_cast<const void*>(lay.find(std::string("shared.") + kProjNames[p] + "." +
                                                                 std::to_string(l / spec.group_size) + ".A"))
                             : nullptr;
    allocate(*dm, lay.ranks, keys);
    dm->family = spec.family;
    auto need = [&](const std::string& n) -> const SynthTensor& {
        const SynthTensor* t = lay.find(n);
        if (!t) throw ConfigError("synthetic layout lacks '" + n + "'");
        return *t;
    };
    auto fill = [&](const SynthTensor& t, long long rows, long long cols, int mode, const DeviceMatrix* m,
                    const void* dst, long long rs, long long cs, int fold, uint64_t scale_off, k::WType dtype) {
        k::SynthFill f{};
        f.seed = spec.seed;
        f.offset = t.stream_offset;
        f.amp = t.amp;
        f.kind = t.kind;
        f.rows = rows;
        f.cols = cols;
        f.rs = rs;
        f.cs = cs;
        f.mode = mode;
        if (m) f.lay = m->layout(dm->esize);
        f.fold = fold;
        f.scale_offset = scale_off;
        f.dst = const_cast<void*>(dst);
        f.dt = dtype;
        k::synth_fill(f, nullptr);
    };
    const long long V = c.vocab, d = c.d_model;
    fill(need("embedding"), V, d, 0, nullptr, dm->emb, dm->ldd, 1, 0, 0, dm->wt);
    fill(need("head"), d, V, 1, &dm->head_t, dm->head_t.w, 0, 0, 0, 0, dm->wt);
    fill(need("final_gamma"), 1, d, 0, nullptr, dm->final_gamma, 0, 1, 0, 0, k::kF32);
    std::map<const void*, bool> done;
    for (size_t l = 0; l < c.n_layers; ++l) {
        const DeviceLayer& D = dm->layers[l];
        const std::string base = "layers." + std::to_string(l) + ".";
        for (size_t p = 0; p < kNumProj; ++p) {
            const auto dims = proj_dims(c, p);
            const long long din = dims[0], dout = dims[1], r = D.r[p];
            const std::string pb = base + kProjNames[p];
            if (!done.count(D.at[p].w)) {
                done[D.at[p].w] = true;
                switch (spec.family) {
                    case 'A': fill(need(pb + ".A"), din, r, 1, &D.at[p], D.at[p].w, 0, 0, 0, 0, dm->wt); break;
                    case 'B':
                        fill(need(pb + ".Uf"), din, r, 1, &D.at[p], D.at[p].w, 0, 0, 1, need(pb + ".scale").stream_offset,
                             dm->wt);
                        break;
                    case 'C':
                        fill(need(std::string("shared.") + kProjNames[p] + "." + std::to_string(l / spec.group_size) +
                                  ".A"),
                             din, r, 1, &D.at[p], D.at[p].w, 0, 0, 0, 0, dm->wt);
                        break;
                    default:
                        fill(need(pb + ".U"), din, r, 1, &D.at[p], D.at[p].w, 0, 0, 2, need(pb + ".S").stream_offset,
                             dm->wt);
                }
            }
            const SynthTensor& bt = need(pb + (spec.family == 'B' || spec.family == 'D' ? ".Vt" : ".B"));
            fill(bt, r, dout, 1, &D.bt[p], D.bt[p].w, 0, 0, 0, 0, dm->wt);
        }
        fill(need(base + "attn_gamma"), 1, d, 0, nullptr, D.attn_gamma, 0, 1, 0, 0, k::kF32);
        fill(need(base + "mlp_gamma"), 1, d, 0, nullptr, D.mlp_gamma, 0, 1, 0, 0, k::kF32);
    }
    FSVD_CUDA(cudaGetLastError());
    FSVD_CUDA(cudaDeviceSynchronize());
    return dm;
}

void copy_factor(const DeviceModel& dm, size_t layer, size_t proj, bool b, float* out, size_t count) {
    if (layer >= dm.layers.size() || proj >= kNumProj) throw ShapeError("copy_factor: index out of range");
    const DeviceLayer& L = dm.layers[layer];
    const auto dims = proj_dims(dm.cfg, proj);
    const size_t r = L.r[proj];
    const size_t want = b ? r * dims[1] : dims[0] * r;
    if (count != want) throw ShapeError("copy_factor: count mismatch");
    const DeviceMatrix& m = b ? L.bt[proj] : L.at[proj];
    const k::WLayout lay = m.layout(dm.esize);
    std::vector<uint8_t> raw(lay.bytes());
    FSVD_CUDA(cudaMemcpy(raw.data(), m.w, raw.size(), cudaMemcpyDeviceToHost));
    auto get = [&](int row, int kk) -> float {
        const uint8_t* p = raw.data() + lay.offset(row, kk);
        if (dm.esize == 4) {
            float f;
            std::memcpy(&f, p, 4);
            return f;
        }
        uint16_t h;
        std::memcpy(&h, p, 2);
        const uint32_t u = static_cast<uint32_t>(h) << 16;
        float f;
        std::memcpy(&f, &u, 4);
        return f;
    };
    // logical A: d_in x r (= A^T[j][i]); B: r x d_out (= B^T[n][j])
    const size_t rows_out = b ? r : dims[0], cols_out = b ? dims[1] : r;
    for (size_t i = 0; i < rows_out; ++i)
        for (size_t j = 0; j < cols_out; ++j) out[i * cols_out + j] = get(static_cast<int>(j), static_cast<int>(i));
}

// ----------------------------------------------------------------- session --

fsvd_ffn_backend route_ffn_auto(fsvd_plan_mode plan, fsvd_ffn_backend requested) {
    // explicit override wins; auto: eager -> no_merge,
    // per_layer -> packed, split -> no_merge. The full-step graph is a
    // layer-tail graph superset, so it routes like per_layer.
    if (requested != FSVD_FFN_AUTO) return requested;
    return plan == FSVD_PLAN_EAGER || plan == FSVD_PLAN_SPLIT ? FSVD_FFN_NO_MERGE : FSVD_FFN_PACKED;
}

void* Session::dalloc(size_t bytes) {
    void* p = nullptr;
    const size_t n = bytes < 256 ? 256 : bytes;
    cudaError_t e = cudaMalloc(&p, n);
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw OomError("session allocation of " + std::to_string(bytes) + " bytes failed");
    }
    FSVD_CUDA(cudaMemsetAsync(p, 0, n, stream_));
    allocations_.push_back(p);
    return p;
}

k::GemvSeg Session::seg(const DeviceMatrix& mtx, int x_off, int y_off, int epi) const {
    return k::GemvSeg{mtx.w, mtx.rows, mtx.k, mtx.kp, x_off, y_off, epi};
}

// A constructor that throws never runs ~Session: free whatever init() had
// allocated (device buffers, stream, graphs) before rethrowing, so a caller
// retrying with another shape does not leak HBM (ConfigError from the
// megakernel's shared-memory sizing happens after the KV cache allocation).
Session::Session(DeviceModel* m, const fsvd_session_opts& o) : m_(m) {
    try {
        init(o);
    } catch (...) {
        release();
        throw;
    }
}

void Session::init(const fsvd_session_opts& o) {
    DeviceModel* m = m_;
    const ModelConfig& c = m->cfg;
    B_ = static_cast<int>(o.batch);
    if (B_ < 1) throw ConfigError("session batch must be >= 1");
    // B <= 2: the persistent decode megakernel; larger batches: the batched
    // layer engine (FSVD_BATCHED=1 forces it for any batch)
    batched_ = B_ > 2;
    if (const char* e = std::getenv("FSVD_BATCHED"); e && e[0] == '1') batched_ = true;
    if (o.attn_route != FSVD_ATTN_DENSE_KV && o.attn_route != FSVD_ATTN_LOWRANK_HISTORY)
        throw ConfigError("unknown attention route");
    attn_route_ = o.attn_route;
    if (attn_route_ == FSVD_ATTN_LOWRANK_HISTORY) {
        // per-step reconstruction GEMMs over the whole history: shapes change every
        // step, so no static plan can hold them (SPEC.md:405 capture error)
        if (o.plan != FSVD_PLAN_EAGER)
            throw ConfigError("lowrank_history attention route needs the eager plan (dynamic shapes)");
        batched_ = true;  // the layer engine (GEMM launches) hosts the reconstruction
    }
    if (!batched_ && m_->cfg.d_model > 8192)
        throw ConfigError("d_model > 8192 is not supported by the decode megakernel");
    if (!(c.d_head == 32 || c.d_head == 64 || c.d_head == 128))
        throw ConfigError("d_head must be 32, 64 or 128 for the sm_100a kernels");
    cap_ = o.capacity ? o.capacity : (m->capacity ? m->capacity : 8192);
    if (o.plan < FSVD_PLAN_EAGER || o.plan > FSVD_PLAN_SPLIT) throw ConfigError("unknown plan mode");
    if (o.ffn < FSVD_FFN_AUTO || o.ffn > FSVD_FFN_PACKED) throw ConfigError("unknown ffn backend");
    plan_ = o.plan;
    ffn_ = route_ffn_auto(plan_, o.ffn);
    FSVD_CUDA(cudaSetDevice(m->device));
    FSVD_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));

    const size_t H = c.n_heads, dh = c.d_head, L = c.n_layers;
    cache_hstride_ = static_cast<long long>(cap_) * dh;
    cache_bstride_ = static_cast<long long>(H) * cache_hstride_;
    cache_lstride_ = static_cast<long long>(B_) * cache_bstride_;
    const size_t cache_bytes = static_cast<size_t>(cache_lstride_) * L * m->esize;
    kc_ = dalloc(cache_bytes);
    vc_ = dalloc(cache_bytes);

    // RoPE table in double like the reference (math.hpp:34-38), cast to f32
    std::vector<float2> rope(cap_ * (dh / 2));
    for (size_t pos = 0; pos < cap_; ++pos)
        for (size_t i = 0; i < dh / 2; ++i) {
            const double freq = std::pow(c.rope_base, -2.0 * static_cast<double>(i) / static_cast<double>(dh));
            const double ang = static_cast<double>(pos) * freq;
            rope[pos * (dh / 2) + i] = make_float2(static_cast<float>(std::cos(ang)), static_cast<float>(std::sin(ang)));
        }
    rope_ = static_cast<float2*>(dalloc(rope.size() * sizeof(float2)));
    FSVD_CUDA(cudaMemcpyAsync(rope_, rope.data(), rope.size() * sizeof(float2), cudaMemcpyHostToDevice, stream_));

    pos_ = static_cast<int*>(dalloc(4));
    step_ = static_cast<int*>(dalloc(4));
    tokens_ = static_cast<int*>(dalloc(4 * B_));

    // rank-space vectors of the prefill path: segment s of a packed
    // projection starts at the sum of the previous segments' pad64 ranks; the
    // stride covers the last segment's padded (tile-layout) reduction length.
    for (const auto& Ly : m->layers) {
        ld_qkv_ = std::max(ld_qkv_, Ly.rp[kQ] + Ly.rp[kK] + Ly.bt[kV].kp);
        ld_ug_ = std::max(ld_ug_, Ly.rp[kUp] + Ly.bt[kGate].kp);
        ld_o_ = std::max(ld_o_, Ly.bt[kO].kp);
        ld_d_ = std::max(ld_d_, Ly.bt[kDown].kp);
    }
    ld_qkv_ = pad8(ld_qkv_);
    ld_ug_ = pad8(ld_ug_);
    xres_ = static_cast<float*>(dalloc(4ull * B_ * m->ldd));
    x_ = static_cast<float*>(dalloc(4ull * B_ * m->ldd));
    logits_ = static_cast<float*>(dalloc(4ull * B_ * c.vocab));

    mk_grid_ = m->sm_count;
    if (const char* g = std::getenv("FSVD_MK_GRID"); g && std::atoi(g) > 0)  // debugging: fewer CTAs
        mk_grid_ = std::min(mk_grid_, std::atoi(g));
    mk_grid_ = std::min(mk_grid_, 256);
    if (const char* e = std::getenv("FSVD_MK_EXACT")) mk_exact_ = e[0] == '1';  // attention merge scratch is sized for <= 256 pieces per head
    mk_splits_ = mk_grid_;  // attention partial slots per head: one per contributing CTA
    mk_attn_pairs_ = mk_grid_ % 2 == 0 && B_ * static_cast<int>(c.n_heads) <= mk_grid_ / 2;
    // the cooperative launch must fit as clusters of 2 (e.g. not under an SM-limited MPS share)
    if (mk_attn_pairs_ && B_ <= 2 &&
        2 * k::mk_max_active_pairs(m->wt, B_, static_cast<int>(c.d_head), 227 * 1024 - 1024) < mk_grid_)
        mk_attn_pairs_ = false;
    if (const char* e = std::getenv("FSVD_MK_ATTN_PAIRS")) mk_attn_pairs_ = mk_attn_pairs_ && e[0] == '1';
    if (attn_route_ == FSVD_ATTN_LOWRANK_HISTORY) {
        for (const auto& Ly : m->layers) ld_hist_ = std::max({ld_hist_, Ly.r[kK], Ly.r[kV]});
        ld_hist_ = pad8(ld_hist_);
        const size_t hb = static_cast<size_t>(L) * B_ * cap_ * ld_hist_ * m->esize;
        hist_k_ = dalloc(hb);
        hist_v_ = dalloc(hb);
    }
    if (plan_ == FSVD_PLAN_SPLIT) split_buf_ = dalloc(4ull * B_ * m->ldd);
    if (batched_) {
        ensure_prefill_workspace(B_);
        dec_splits_ = k::attn_decode_splits(B_, static_cast<int>(H), static_cast<int>(cap_));
        dec_part_ = static_cast<float*>(dalloc(4ull * B_ * H * dec_splits_ * (dh + 2)));
    } else {
        // the megakernel's work splits multiply in 32 bits (decode_mk_common.cuh RowSplit / MkSplit)
        if (static_cast<unsigned long long>(B_) * H * cap_ * mk_grid_ >= (1ull << 32))
            throw ConfigError("decode megakernel: batch x heads x capacity x grid must stay below 2^32");
        attn_part_ = static_cast<float*>(dalloc(4ull * B_ * H * mk_splits_ * (dh + 2)));
        attn_count_ = static_cast<unsigned*>(dalloc(4ull * B_ * H));
        build_program();
    }
    FSVD_CUDA(cudaStreamSynchronize(stream_));
    stats_.allocs = 0;
}

Session::~Session() { release(); }

void Session::release() {
    cudaSetDevice(m_->device);
    if (stream_) cudaStreamSynchronize(stream_);
    for (auto g : layer_graphs_) cudaGraphExecDestroy(g);
    layer_graphs_.clear();
    if (step_graph_) cudaGraphExecDestroy(step_graph_);
    step_graph_ = nullptr;
    if (bstep_graph_) cudaGraphExecDestroy(bstep_graph_);
    bstep_graph_ = nullptr;
    for (void* p : allocations_) cudaFree(p);
    allocations_.clear();
    if (stream_) cudaStreamDestroy(stream_);
    stream_ = nullptr;
}

void* Session::staging(size_t bytes) {
    if (bytes > staging_bytes_) {
        FSVD_CUDA(cudaStreamSynchronize(stream_));
        if (staging_) {
            allocations_.erase(std::find(allocations_.begin(), allocations_.end(), staging_));
            cudaFree(staging_);
        }
        staging_ = dalloc(bytes);
        staging_bytes_ = bytes;
        stats_.allocs += 1;
    }
    return staging_;
}

// ------------------------------------------------------------ phase program --
// Activation vector in the megakernel's B-operand form (decode_mk.h Planes):
// 4 bytes per element and batch row (bf16 hi + lo, or fp32), zero padded.
k::Planes Session::planes(int len) {
    const int l = pad64(static_cast<size_t>(len));
    x_bytes_ = std::max(x_bytes_, B_ * l * 4);
    return k::Planes{dalloc(4ull * B_ * l), l};
}

// Appends one GEMV phase (weights segs, input planes in); the caller fills
// the output side. Allocates the phase's pieces exchange.
k::MkGemv& Session::add_gemv(const std::vector<k::GemvSeg>& segs, int dual, const k::Planes& in,
                             const float* norm_src, int out_kind) {
    const DeviceModel& m = *m_;
    k::MkPhase p{};
    p.kind = k::kMkGemv;
    k::MkGemv& g = p.g;
    for (size_t i = 0; i < segs.size(); ++i) g.seg[i] = segs[i];
    g.nseg = static_cast<int>(segs.size());
    g.dual = dual;
    g.in = in;
    for (int i = 0; i < g.nseg; ++i)
        if (g.seg[i].x_off + g.seg[i].kp > in.len) throw std::logic_error("megakernel: input planes too short");
    g.norm_src = norm_src;
    g.norm_ld = m.ldd;
    g.norm_len = static_cast<int>(m.cfg.d_model);
    g.eps = static_cast<float>(m.cfg.norm_eps);
    g.out_kind = out_kind;
    // FSVD_MK_EXACT=1: even unit splits (shared boundary tiles through the pieces
    // exchange) for the long-K rank-space projections, whose few large tiles leave
    // tile-aligned splits uneven (1 vs 2 tiles per CTA). Measured slower on C2
    // (3.24 vs 2.90 ms/token: the exchange wait costs more than the imbalance), so
    // tile-aligned splits are the default.
    g.exact_split = out_kind == k::kOutPlanes && mk_exact_;
    int max_pieces = 1;
    k::mk_split_stats(g.seg, g.nseg, dual, m.esize, mk_grid_, g.exact_split, &max_pieces, &g.rec_ntl, &g.rec_c0,
                      &g.rec_c1);
    if (g.rec_ntl > k::kMkMaxLocalTiles)
        throw ConfigError("decode megakernel: a CTA would touch more than 64 output tiles of one phase");
    const int max_chunks = g.rec_ntl * (g.rec_c0 + g.rec_c1);
    const int nt = k::mk_out_tiles(g.seg, g.nseg, dual, m.esize);
    g.max_pieces = max_pieces;
    g.pieces = static_cast<float*>(dalloc(4ull * nt * max_pieces * 2 * k::kTileRows * B_));
    g.count = static_cast<unsigned*>(dalloc(4ull * nt));
    FSVD_CUDA(cudaMemsetAsync(g.count, 0, 4ull * nt, stream_));
    rec_chunks_ = std::max(rec_chunks_, max_chunks);
    if (h_phases_.size() == h_phases_.capacity()) throw std::logic_error("phase program capacity");
    h_phases_.push_back(p);
    return h_phases_.back().g;
}

int Session::add_vec(const void* emb, const float* src, float* xres, const float* gamma, const k::Planes& out) {
    const DeviceModel& m = *m_;
    k::MkPhase p{};
    p.kind = k::kMkVec;
    k::MkVec& v = p.v;
    v.emb = emb;
    v.emb_ld = m.ldd;
    v.tokens = tokens_;
    v.src = src;
    v.src_ld = m.ldd;
    v.len = static_cast<int>(m.cfg.d_model);
    v.xres = xres;
    v.xres_ld = m.ldd;
    v.gamma = gamma;
    v.out = out;
    h_phases_.push_back(p);
    return static_cast<int>(h_phases_.size()) - 1;
}

// One layer. Input: xpl_ = rmsnorm gamma-scaled residual
// planes (the scale 1/rms is applied to the projection outputs); output: the
// residual xres_ and xpl_ scaled by the next norm's gamma (next_gamma).
void Session::add_layer_phases(size_t l, const float* next_gamma) {
    const DeviceModel& m = *m_;
    const ModelConfig& c = m.cfg;
    const DeviceLayer& L = m.layers[l];
    char* kc = static_cast<char*>(kc_) + l * cache_lstride_ * m.esize;
    char* vc = static_cast<char*>(vc_) + l * cache_lstride_ * m.esize;
    const int rq = L.rp[kQ], rk = L.rp[kK];
    // qkvA: p_qkv = rmsnorm(x) . [A_q | A_k | A_v]   (packed QKV projection)
    {
        k::MkGemv& g = add_gemv({seg(L.at[kQ], 0, 0, 0), seg(L.at[kK], 0, 0, 0), seg(L.at[kV], 0, 0, 0)}, 0, xpl_,
                                xres_, k::kOutPlanes);
        g.out = pqkv_;
        g.out_off[0] = 0;
        g.out_off[1] = rq;
        g.out_off[2] = rq + rk;
    }
    // qkvB: q, k, v = p . B with RoPE (q, k) and the dense-KV append at pos
    {
        k::MkGemv& g = add_gemv({seg(L.bt[kQ], 0, 0, 0), seg(L.bt[kK], rq, 0, 0), seg(L.bt[kV], rq + rk, 0, 0)}, 0,
                                pqkv_, nullptr, k::kOutQKV);
        g.qbuf = qbuf_;
        g.q_ld = m.ldd;
        g.rope = rope_;
        g.kcache = kc;
        g.vcache = vc;
        g.cache_bstride = cache_bstride_;
        g.cache_hstride = cache_hstride_;
        g.d_head = static_cast<int>(c.d_head);
        g.pos = pos_;
        g.attn_pairs = mk_attn_pairs_ ? 1 : 0;
    }
    // dense-KV attention over cache rows [0, pos]
    {
        k::MkPhase p{};
        p.kind = k::kMkAttn;
        k::MkAttn& a = p.a;
        a.qbuf = qbuf_;
        a.q_ld = m.ldd;
        a.kcache = kc;
        a.vcache = vc;
        a.cache_bstride = cache_bstride_;
        a.cache_hstride = cache_hstride_;
        a.pos = pos_;
        a.partial = attn_part_;
        a.count = attn_count_;
        a.n_heads = static_cast<int>(c.n_heads);
        a.d_head = static_cast<int>(c.d_head);
        a.splits = mk_splits_;
        a.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(c.d_head)));
        a.out = att_;
        a.pairs = mk_attn_pairs_ ? 1 : 0;
        h_phases_.push_back(p);
    }
    // o projection, residual add (+ the FFN norm's gamma)
    add_gemv({seg(L.at[kO], 0, 0, 0)}, 0, att_, nullptr, k::kOutPlanes).out = po_;
    {
        k::MkGemv& g = add_gemv({seg(L.bt[kO], 0, 0, 0)}, 0, po_, nullptr, k::kOutResid);
        g.out = xpl_;
        g.xres = xres_;
        g.xres_ld = m.ldd;
        g.gamma = L.mlp_gamma;
    }
    // FFN input side: packed = one projection over [A_up | A_gate]
    ph_ffn_begin_.push_back(static_cast<int>(h_phases_.size()));
    if (ffn_ == FSVD_FFN_PACKED) {
        k::MkGemv& g = add_gemv({seg(L.at[kUp], 0, 0, 0), seg(L.at[kGate], 0, 0, 0)}, 0, xpl_, xres_, k::kOutPlanes);
        g.out = pug_;
        g.out_off[1] = L.rp[kUp];
    } else {
        add_gemv({seg(L.at[kUp], 0, 0, 0)}, 0, xpl_, xres_, k::kOutPlanes).out = pug_;
        k::MkGemv& g = add_gemv({seg(L.at[kGate], 0, 0, 0)}, 0, xpl_, xres_, k::kOutPlanes);
        g.out = pug_;
        g.out_off[0] = L.rp[kUp];
    }
    // ugB (dual): up and gate reconstructions, SiLU.mul finalize
    add_gemv({seg(L.bt[kUp], 0, 0, 0), seg(L.bt[kGate], L.rp[kUp], 0, 0)}, 1, pug_, nullptr, k::kOutSilu).out = h_;
    // down projection, residual add (+ the next norm's gamma)
    add_gemv({seg(L.at[kDown], 0, 0, 0)}, 0, h_, nullptr, k::kOutPlanes).out = pd_;
    {
        k::MkGemv& g = add_gemv({seg(L.bt[kDown], 0, 0, 0)}, 0, pd_, nullptr, k::kOutResid);
        g.out = xpl_;
        g.xres = xres_;
        g.xres_ld = m.ldd;
        g.gamma = next_gamma;
    }
}

void Session::build_program() {
    const DeviceModel& m = *m_;
    const ModelConfig& c = m.cfg;
    h_phases_.clear();
    h_phases_.reserve(12 * c.n_layers + 16);
    x_bytes_ = 0;
    rec_chunks_ = 0;
    ph_layer_begin_.clear();
    ph_layer_end_.clear();
    ph_ffn_begin_.clear();
    // activation planes (each a phase's input, written by its producer's finalizers)
    int lq = 0, lo = 0, lug = 0, ld = 0;
    for (const auto& Ly : m.layers) {
        lq = std::max(lq, Ly.rp[kQ] + Ly.rp[kK] + Ly.bt[kV].kp);
        lo = std::max(lo, Ly.bt[kO].kp);
        lug = std::max(lug, Ly.rp[kUp] + Ly.bt[kGate].kp);
        ld = std::max(ld, Ly.bt[kDown].kp);
    }
    xpl_ = planes(m.ldd);
    pqkv_ = planes(lq);
    att_ = planes(m.ldd);
    po_ = planes(lo);
    pug_ = planes(lug);
    h_ = planes(m.ldff);
    pd_ = planes(ld);
    qbuf_ = static_cast<float*>(dalloc(4ull * B_ * m.ldd));
    const int head_tiles = (static_cast<int>(c.vocab) + k::kTileRows - 1) / k::kTileRows;
    cand_v_ = static_cast<float*>(dalloc(4ull * head_tiles * B_));
    cand_i_ = static_cast<int*>(dalloc(4ull * head_tiles * B_));
    mk_bar_ = static_cast<unsigned*>(dalloc(64));

    for (size_t l = 0; l < c.n_layers; ++l) {
        ph_layer_begin_.push_back(static_cast<int>(h_phases_.size()));
        if (l == 0) add_vec(m.emb, nullptr, xres_, m.layers[0].attn_gamma, xpl_);  // embedding row
        add_layer_phases(l, l + 1 < c.n_layers ? m.layers[l + 1].attn_gamma : m.final_gamma);
        ph_layer_end_.push_back(static_cast<int>(h_phases_.size()));
    }
    auto add_head = [&](const float* norm_src, int pos_inc, int& arg_idx) {
        k::MkGemv& g = add_gemv({seg(m.head_t, 0, 0, 0)}, 0, xpl_, norm_src, k::kOutLogits);
        g.logits = logits_;
        g.vocab = static_cast<int>(c.vocab);
        g.cand_v = cand_v_;
        g.cand_i = cand_i_;
        k::MkPhase p{};
        p.kind = k::kMkArgmax;
        p.m.cand_v = cand_v_;
        p.m.cand_i = cand_i_;
        p.m.ntiles = head_tiles;
        p.m.tokens = tokens_;
        p.m.pos = pos_;
        p.m.pos_inc = pos_inc;
        p.m.step = step_;
        arg_idx = static_cast<int>(h_phases_.size());
        h_phases_.push_back(p);
    };
    // decode: the last layer's finalizers leave xpl_ = x * final_gamma
    ph_head_ = static_cast<int>(h_phases_.size());
    add_head(xres_, 1, ph_argmax_);
    // prefill: the last position's hidden state x_ (gathered by the prefill path)
    ph_pf_head_ = add_vec(nullptr, x_, nullptr, m.final_gamma, xpl_);
    add_head(x_, 0, ph_pf_argmax_);

    const int dh = static_cast<int>(c.d_head);
    const int nph_all = static_cast<int>(h_phases_.size());
    mk_stages_ = std::min(12 * 8 / k::kChunkLines, k::mk_max_stages(x_bytes_, rec_chunks_, B_, dh, nph_all));
    if (mk_stages_ < 2)
        throw ConfigError("decode megakernel: shared memory does not fit this (batch, shape): x " +
                          std::to_string(x_bytes_) + " B, " + std::to_string(rec_chunks_) + " chunk records");
    mk_smem_ = k::mk_smem_bytes(mk_stages_, x_bytes_, rec_chunks_, B_, dh, nph_all);
    // L2 prefetch distance (chunks per CTA beyond the ring): 16 x 16 KiB x 148 CTAs = 38 MB of the 126 MB L2
    mk_l2_ahead_ = 64 / k::kChunkLines;  // 128 KiB ahead; measured best of {0, 8, 16, 24, 32, 48} (C2, B200): 3.07 -> 2.94 ms/token
    if (const char* e = std::getenv("FSVD_MK_L2_AHEAD")) mk_l2_ahead_ = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("FSVD_MK_PROGRESS"); e && e[0] == '1') {  // hang diagnosis (debug)
        void* h = nullptr;
        FSVD_CUDA(cudaHostAlloc(&h, 64ull * mk_grid_, cudaHostAllocMapped));
        std::memset(h, 0xff, 64ull * mk_grid_);
        mk_progress_host_ = static_cast<int*>(h);
        void* d = nullptr;
        FSVD_CUDA(cudaHostGetDevicePointer(&d, h, 0));
        mk_progress_ = static_cast<volatile int*>(d);
        std::thread([h = mk_progress_host_, n = mk_grid_] {
            for (int it = 0; it < 600; ++it) {
                std::this_thread::sleep_for(std::chrono::seconds(1));
                if (const char* f = std::getenv("FSVD_MK_PROGRESS_DUMP"); f && it % 2 == 1) {
                    FILE* o = std::fopen(f, "w");
                    if (!o) continue;
                    for (int c = 0; c < n; ++c) { std::fprintf(o, "%d", c); for (int q = 0; q < 16; ++q) std::fprintf(o, " %d", h[16 * c + q]); std::fprintf(o, "\n"); }
                    std::fclose(o);
                }
            }
        }).detach();
    }
    if (const char* tr = std::getenv("FSVD_TRACE"); tr && tr[0] == '1')
        trace_ = static_cast<unsigned long long*>(dalloc(8ull * mk_grid_ * (ph_argmax_ + 1) * 16 + 8ull * 8192 * 4));
    {  // precomputed chunk records of every CTA's weight stream
        std::vector<k::MkChunk> ch;
        std::vector<int> st, tl;
        k::mk_build_chunks(h_phases_.data(), static_cast<int>(h_phases_.size()), mk_grid_, m.esize, ch, st, tl);
        d_chunk_tiles_ = static_cast<int*>(dalloc(sizeof(int) * tl.size()));
        FSVD_CUDA(cudaMemcpyAsync(d_chunk_tiles_, tl.data(), sizeof(int) * tl.size(), cudaMemcpyHostToDevice, stream_));
        d_chunks_ = static_cast<k::MkChunk*>(dalloc(sizeof(k::MkChunk) * std::max<size_t>(1, ch.size())));
        d_chunk_start_ = static_cast<int*>(dalloc(sizeof(int) * st.size()));
        FSVD_CUDA(cudaMemcpyAsync(d_chunks_, ch.data(), sizeof(k::MkChunk) * ch.size(), cudaMemcpyHostToDevice, stream_));
        FSVD_CUDA(cudaMemcpyAsync(d_chunk_start_, st.data(), sizeof(int) * st.size(), cudaMemcpyHostToDevice, stream_));
        FSVD_CUDA(cudaStreamSynchronize(stream_));
    }
    d_phases_ = static_cast<k::MkPhase*>(dalloc(sizeof(k::MkPhase) * h_phases_.size()));
    FSVD_CUDA(cudaMemcpyAsync(d_phases_, h_phases_.data(), sizeof(k::MkPhase) * h_phases_.size(),
                              cudaMemcpyHostToDevice, stream_));
}

void Session::mk_run(int p_begin, int p_end, int reps) {
    k::MkLaunch L{};
    L.phases = d_phases_;
    L.p_begin = p_begin;
    L.p_end = p_end;
    L.reps = reps;
    L.bar = mk_bar_;
    L.grid = mk_grid_;
    L.smem_bytes = mk_smem_;
    L.stages = mk_stages_;
    L.x_bytes = x_bytes_;
    L.rec_chunks = rec_chunks_;
    L.l2_ahead = mk_l2_ahead_;
    L.cluster2 = mk_attn_pairs_ ? 1 : 0;
    L.pos = pos_;
    L.chunks = d_chunks_;
    L.chunk_start = d_chunk_start_;
    L.chunk_tiles = d_chunk_tiles_;
    L.nphases = static_cast<int>(h_phases_.size());
    L.progress = mk_progress_;
    if (trace_ && p_begin == 0 && p_end == ph_argmax_ + 1 && reps == 1) L.trace = trace_;
    if (!k::mk_launch(m_->wt, B_, static_cast<int>(m_->cfg.d_head), L, stream_))
        throw CudaError("megakernel: no instantiation for this (dtype, batch, d_head)");
    FSVD_CUDA(cudaGetLastError());
    ++launches_this_step_;
}

int Session::read_trace(unsigned long long* out, size_t count, int* grid) {
    if (!trace_) throw ConfigError("tracing disabled (set FSVD_TRACE=1 before creating the session)");
    const int nph = ph_argmax_ + 1;
    const size_t n = static_cast<size_t>(mk_grid_) * nph * 16 + 8192 * 4;
    if (count < n) throw ShapeError("trace buffer too small");
    FSVD_CUDA(cudaStreamSynchronize(stream_));
    FSVD_CUDA(cudaMemcpy(out, trace_, n * 8, cudaMemcpyDeviceToHost));
    if (grid) *grid = mk_grid_;
    return nph;
}

void Session::mk_set_out(int32_t* d_out, int out_ld) {
    if (d_out == mk_out_ && out_ld == mk_out_ld_) return;
    k::MkPhase& p = h_phases_[ph_argmax_];
    p.m.out = d_out;
    p.m.out_ld = out_ld;
    FSVD_CUDA(cudaMemcpyAsync(d_phases_ + ph_argmax_, &p, sizeof(k::MkPhase), cudaMemcpyHostToDevice, stream_));
    mk_out_ = d_out;
    mk_out_ld_ = out_ld;
}

// One decode step: eager = one launch per phase, per_layer = one launch
// (captured as one graph) per layer, full_step = one graph for the step.
void Session::mk_decode(int32_t* d_out, int out_ld) {
    mk_set_out(d_out, out_ld);
    const int L = static_cast<int>(m_->cfg.n_layers);
    launches_this_step_ = 0;
    if (plan_ == FSVD_PLAN_EAGER) {
        for (int p = 0; p <= ph_argmax_; ++p) mk_run(p, p + 1);
        stats_.dispatches += launches_this_step_;
        stats_.kernel_launches += launches_this_step_;
        return;
    }
    if (plan_ == FSVD_PLAN_FULL_STEP) {
        if (!step_graph_) {
            cudaGraph_t g;
            FSVD_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
            mk_run(0, ph_argmax_ + 1);
            FSVD_CUDA(cudaStreamEndCapture(stream_, &g));
            FSVD_CUDA(cudaGraphInstantiate(&step_graph_, g, 0));
            cudaGraphDestroy(g);
        }
        FSVD_CUDA(cudaGraphLaunch(step_graph_, stream_));
        stats_.graph_launches += 1;
        stats_.dispatches += 1;
        return;
    }
    // per-layer plans: layer 0 .. L-1 (layer 0 gathers the embedding), [head + argmax];
    // split plans: [attention body], [MLP body] per layer
    const bool split = plan_ == FSVD_PLAN_SPLIT;
    if (layer_graphs_.empty()) {
        std::vector<std::pair<int, int>> ranges;
        for (int l = 0; l < L; ++l) {
            if (split) {
                ranges.push_back({ph_layer_begin_[l], ph_ffn_begin_[l]});
                ranges.push_back({ph_ffn_begin_[l], ph_layer_end_[l]});
            } else {
                ranges.push_back({ph_layer_begin_[l], ph_layer_end_[l]});
            }
        }
        ranges.push_back({ph_head_, ph_argmax_ + 1});
        for (auto [b, e] : ranges) {
            cudaGraph_t g;
            FSVD_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
            mk_run(b, e);
            FSVD_CUDA(cudaStreamEndCapture(stream_, &g));
            cudaGraphExec_t ge;
            FSVD_CUDA(cudaGraphInstantiate(&ge, g, 0));
            cudaGraphDestroy(g);
            layer_graphs_.push_back(ge);
        }
    }
    if (!split) {
        for (auto g : layer_graphs_) FSVD_CUDA(cudaGraphLaunch(g, stream_));
        stats_.graph_launches += layer_graphs_.size();
        stats_.dispatches += layer_graphs_.size();
        return;
    }
    // split: the host boundary between a layer's attention and MLP graphs is an explicit
    // copy of the residual stream (the "graph-boundary traffic" of SPEC.md:406, Fig. 6)
    const size_t cb = 4ull * B_ * m_->ldd;
    for (int l = 0; l < L; ++l) {
        FSVD_CUDA(cudaGraphLaunch(layer_graphs_[2 * l], stream_));
        FSVD_CUDA(cudaMemcpyAsync(split_buf_, xres_, cb, cudaMemcpyDeviceToDevice, stream_));
        FSVD_CUDA(cudaGraphLaunch(layer_graphs_[2 * l + 1], stream_));
        stats_.copy_bytes += cb;
    }
    FSVD_CUDA(cudaGraphLaunch(layer_graphs_.back(), stream_));
    stats_.graph_launches += layer_graphs_.size();
    stats_.dispatches += layer_graphs_.size() + L;
}

void Session::decode_step(const int32_t* d_tokens, float* d_logits) {
    if (position_ == 0) throw ShapeError("decode_step: prefill first (position = 0)");
    if (position_ >= cap_) throw CapacityError("decode_step: KV cache full (capacity " + std::to_string(cap_) + ")");
    if (d_tokens) FSVD_CUDA(cudaMemcpyAsync(tokens_, d_tokens, 4ull * B_, cudaMemcpyDeviceToDevice, stream_));
    const uint64_t before = stats_.dispatches;
    decode_any(nullptr, 0);
    if (d_logits && d_logits != logits_)
        FSVD_CUDA(cudaMemcpyAsync(d_logits, logits_, 4ull * B_ * m_->cfg.vocab, cudaMemcpyDeviceToDevice, stream_));
    FSVD_CUDA(cudaGetLastError());
    stats_.last_dispatches = stats_.dispatches - before;
    stats_.steps += 1;
    position_ += 1;
}

// n greedy decode steps without host round trips (each feeds back its argmax).
// Megakernel + full-step plan: one launch runs up to 256 steps (the phase
// program repeated, pos re-read after each step's argmax): no per-token launch
// gap. Other engines / plans: n single steps. Bitwise identical either way.
void Session::decode_steps(size_t n, int32_t* d_out, int out_ld) {
    if (n == 0) return;
    if (position_ == 0) throw ShapeError("decode_steps: prefill first (position = 0)");
    if (position_ + n > cap_)
        throw CapacityError("decode_steps: " + std::to_string(n) + " steps exceed capacity " + std::to_string(cap_));
    const uint64_t before = stats_.dispatches;
    if (d_out) k::set_int(step_, 0, stream_);  // tokens land in columns 0 .. n-1
    if (batched_ || plan_ != FSVD_PLAN_FULL_STEP) {
        for (size_t i = 0; i < n; ++i) decode_any(d_out, out_ld);
    } else {
        mk_set_out(d_out, out_ld);
        for (size_t i = 0; i < n;) {
            const int r = static_cast<int>(std::min<size_t>(256, n - i));
            launches_this_step_ = 0;
            mk_run(0, ph_argmax_ + 1, r);
            stats_.dispatches += 1;
            stats_.kernel_launches += 1;
            i += r;
        }
    }
    FSVD_CUDA(cudaGetLastError());
    stats_.last_dispatches = (stats_.dispatches - before) / n;
    stats_.steps += n;
    position_ += n;
}

// --------------------------------------------------------------- prefill --
void Session::ensure_prefill_workspace(size_t rows) {
    if (rows <= pf_rows_) return;
    const DeviceModel& m = *m_;
    const size_t es = m.esize;
    pf_x_ = static_cast<float*>(dalloc(rows * m.ldd * 4));
    pf_xn_ = dalloc(rows * m.ldd * es);
    pf_pqkv_ = dalloc(rows * ld_qkv_ * es);
    pf_q_ = dalloc(rows * m.ldd * es);
    pf_att_ = dalloc(rows * m.ldd * es);
    pf_po_ = dalloc(rows * ld_o_ * es);
    pf_pug_ = dalloc(rows * ld_ug_ * es);
    pf_h_ = dalloc(rows * m.ldff * es);
    pf_pd_ = dalloc(rows * ld_d_ * es);
    pf_tok_ = static_cast<int32_t*>(dalloc(rows * 4));
    // split-K scratch (only used while rows <= 1024: few output tiles)
    // (decode-sized M: up to 64 splits per projection, residual adds included)
    pf_ws_floats_ = std::max(4ull * std::min<size_t>(rows, 1024), 64ull * std::min<size_t>(rows, 64)) *
                    std::max({ld_qkv_, ld_o_, ld_ug_, ld_d_, m.ldd});
    pf_ws_ = m.wt == k::kBF16 ? static_cast<float*>(dalloc(4 * pf_ws_floats_)) : nullptr;
    pf_ss_ = static_cast<float*>(dalloc(rows * (m.ldd / 32) * 4));
    pf_rows_ = rows;
    stats_.allocs += 12;
}

// One prefill chunk: tokens [b][t0 .. t0+Tc) of a [B][T_total] prompt.
void Session::prefill_chunk(const int32_t* d_tokens, size_t T_total, size_t t0, size_t Tc) {
    const DeviceModel& m = *m_;
    const ModelConfig& c = m.cfg;
    const int M = static_cast<int>(B_ * Tc);
    const int d = static_cast<int>(c.d_model), ldd = m.ldd;
    FSVD_CUDA(cudaMemcpy2DAsync(pf_tok_, Tc * 4, d_tokens + t0, T_total * 4, Tc * 4, B_, cudaMemcpyDeviceToDevice,
                                stream_));
    k::embed(m.wt, m.emb, ldd, pf_tok_, M, d, pf_x_, ldd, stream_);
    layers_forward(M, static_cast<int>(Tc), static_cast<int>(position_), nullptr);
}

void Session::layers_forward(int M, int Tc, int p0, const int* p0_dev) {
    const DeviceModel& m = *m_;
    const ModelConfig& c = m.cfg;
    const int d = static_cast<int>(c.d_model), ldd = m.ldd, ldff = m.ldff;
    const float eps = static_cast<float>(c.norm_eps);
    const size_t es = m.esize;
    // RMSNorm folded into the GEMMs (prefill, tcgen05 path): the residual-add GEMMs
    // (oB, downB) also emit x_new * gamma_next in bf16 and its per-32-column sums
    // of squares; the next input-factor GEMM (upgateA, next layer's qkvA) reads
    // those and scales its rows by 1 / rms -- no row-RMSNorm launch after layer 0
    const bool fold = m.wt == k::kBF16 && M > 128 && !std::getenv("FSVD_PREFILL_SIMT") &&
                      !std::getenv("FSVD_NO_NORM_FOLD") && d % 128 == 0 && ldd % 32 == 0;
    const void* norm_ss_in = nullptr;  // set for the next plain-store GEMM that consumes a folded norm
    void* norm_xg = nullptr;           // set for the next residual GEMM that emits one
    const float* norm_gamma = nullptr;
    auto gemm = [&](const void* x, int x_ld, int nseg, std::initializer_list<k::GemvSeg> segs, int epi, void* y,
                    int y_ld, char* kc = nullptr, char* vc = nullptr) {
        k::GemmArgs g{};
        g.x = x;
        g.x_ld = x_ld;
        g.M = M;
        int i = 0;
        for (const auto& s : segs) g.seg[i++] = s;
        g.nseg = nseg;
        g.epi = epi;
        g.y = y;
        g.y_ld = y_ld;
        g.rope = rope_;
        g.p0 = p0;
        g.p0_dev = p0_dev;
        g.T = Tc;
        g.d_head = static_cast<int>(c.d_head);
        g.n_heads = static_cast<int>(c.n_heads);
        g.kcache = kc;
        g.vcache = vc;
        g.cache_bstride = cache_bstride_;
        g.cache_hstride = cache_hstride_;
        if (M <= 1024) {
            g.ws = pf_ws_;
            g.ws_floats = pf_ws_floats_;
        }
        if (epi == k::kGemmStore && norm_ss_in) {
            g.norm_ss_in = static_cast<const float*>(norm_ss_in);
            g.norm_ss_ld = ldd / 32;
            g.norm_ss_n = d / 32;
            g.norm_d = d;
            g.norm_eps = eps;
        }
        if (epi == k::kGemmAddF32 && norm_xg) {
            g.norm_xg = norm_xg;
            g.norm_xg_ld = ldd;
            g.norm_gamma = norm_gamma;
            g.norm_ss = pf_ss_;
            g.norm_ss_ld = ldd / 32;
        }
        k::gemm(m.wt, g, stream_);
    };
    for (size_t l = 0; l < c.n_layers; ++l) {
        const DeviceLayer& L = m.layers[l];
        char* kc = static_cast<char*>(kc_) + l * cache_lstride_ * es;
        char* vc = static_cast<char*>(vc_) + l * cache_lstride_ * es;
        const int rq = L.rp[kQ], rk = L.rp[kK];
        if (!fold || l == 0) {
            k::rmsnorm_rows(m.wt, pf_x_, ldd, L.attn_gamma, eps, M, d, pf_xn_, ldd, stream_);
        } else {
            norm_ss_in = pf_ss_;  // pf_xn_ = x * attn_gamma from the previous layer's downB
        }
        gemm(pf_xn_, ldd, 3,
             {seg(L.at[kQ], 0, 0, k::kEpiStore), seg(L.at[kK], 0, rq, k::kEpiStore),
              seg(L.at[kV], 0, rq + rk, k::kEpiStore)},
             k::kGemmStore, pf_pqkv_, ld_qkv_);
        norm_ss_in = nullptr;
        if (attn_route_ == FSVD_ATTN_LOWRANK_HISTORY) {
            // record the pre-RoPE rank-space k / v rows of these positions
            const long long hstride = static_cast<long long>(cap_) * ld_hist_;
            char* hk = static_cast<char*>(hist_k_) + l * B_ * hstride * es;
            char* hv = static_cast<char*>(hist_v_) + l * B_ * hstride * es;
            k::copy_rows_at(pf_pqkv_, ld_qkv_, rq, L.r[kK], hk, hstride, ld_hist_, B_, Tc, p0, p0_dev,
                            static_cast<int>(es), stream_);
            k::copy_rows_at(pf_pqkv_, ld_qkv_, rq + rk, L.r[kV], hv, hstride, ld_hist_, B_, Tc, p0, p0_dev,
                            static_cast<int>(es), stream_);
        }
        if (attn_route_ == FSVD_ATTN_LOWRANK_HISTORY && Tc == 1) {
            // decode: q from its rank-space row; the whole dense K / V history is rebuilt from
            // the rank-space history -- K = P_k B_k with RoPE at every position, V = P_v B_v --
            // then attended like dense_kv (numerically the same, deliberately cost-inferior)
            gemm(pf_pqkv_, ld_qkv_, 1, {seg(L.bt[kQ], 0, 0, k::kEpiRopeQ)}, k::kGemmQKV, pf_q_, ldd, kc, vc);
            const int len = static_cast<int>(position_) + 1;
            const long long hstride = static_cast<long long>(cap_) * ld_hist_;
            for (int b = 0; b < B_; ++b) {
                for (int kv = 0; kv < 2; ++kv) {
                    k::GemmArgs g{};
                    g.x = static_cast<char*>(kv ? hist_v_ : hist_k_) + (l * B_ + b) * hstride * es;
                    g.x_ld = ld_hist_;
                    g.M = len;
                    g.seg[0] = seg(kv ? L.bt[kV] : L.bt[kK], 0, 0, kv ? k::kEpiV : k::kEpiRopeK);
                    g.nseg = 1;
                    g.epi = k::kGemmQKV;
                    g.y = pf_q_;
                    g.y_ld = ldd;
                    g.rope = rope_;
                    g.p0 = 0;
                    g.T = len;
                    g.d_head = static_cast<int>(c.d_head);
                    g.n_heads = static_cast<int>(c.n_heads);
                    g.kcache = kc + b * cache_bstride_ * es;
                    g.vcache = vc + b * cache_bstride_ * es;
                    g.cache_bstride = cache_bstride_;
                    g.cache_hstride = cache_hstride_;
                    k::gemm(m.wt, g, stream_);
                    stats_.recon_flops += 2ull * len * (kv ? L.r[kV] : L.r[kK]) * d;
                }
            }
            launches_this_step_ += 2 * B_;
        } else {
            gemm(pf_pqkv_, ld_qkv_, 3,
                 {seg(L.bt[kQ], 0, 0, k::kEpiRopeQ), seg(L.bt[kK], rq, 0, k::kEpiRopeK),
                  seg(L.bt[kV], rq + rk, 0, k::kEpiV)},
                 k::kGemmQKV, pf_q_, ldd, kc, vc);
        }
        {
            k::AttnPrefillArgs a{};
            a.q = pf_q_;
            a.q_ld = ldd;
            a.kcache = kc;
            a.vcache = vc;
            a.cache_bstride = cache_bstride_;
            a.cache_hstride = cache_hstride_;
            a.out = pf_att_;
            a.out_ld = ldd;
            a.batch = B_;
            a.T = Tc;
            a.p0 = p0;
            a.p0_dev = p0_dev;
            a.n_heads = static_cast<int>(c.n_heads);
            a.d_head = static_cast<int>(c.d_head);
            a.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(c.d_head)));
            // one new query per sequence (batched decode): split-KV flash decode
            if (!(Tc == 1 && dec_part_ && k::attn_decode(m.wt, a, dec_part_, dec_splits_, stream_)))
                k::attn_prefill(m.wt, a, stream_);
        }
        gemm(pf_att_, ldd, 1, {seg(L.at[kO], 0, 0, k::kEpiStore)}, k::kGemmStore, pf_po_, ld_o_);
        if (fold) {
            norm_xg = pf_xn_;
            norm_gamma = L.mlp_gamma;
        }
        gemm(pf_po_, ld_o_, 1, {seg(L.bt[kO], 0, 0, k::kEpiStore)}, k::kGemmAddF32, pf_x_, ldd);
        norm_xg = nullptr;
        if (plan_ == FSVD_PLAN_SPLIT && Tc == 1) {  // split plan: attention | MLP boundary copy
            FSVD_CUDA(cudaMemcpyAsync(split_buf_, pf_x_, 4ull * M * ldd, cudaMemcpyDeviceToDevice, stream_));
            stats_.copy_bytes += 4ull * M * ldd;
            stats_.dispatches += 1;
        }
        if (!fold) {
            k::rmsnorm_rows(m.wt, pf_x_, ldd, L.mlp_gamma, eps, M, d, pf_xn_, ldd, stream_);
        } else {
            norm_ss_in = pf_ss_;  // pf_xn_ = x * mlp_gamma from oB
        }
        if (ffn_ == FSVD_FFN_PACKED) {
            gemm(pf_xn_, ldd, 2, {seg(L.at[kUp], 0, 0, k::kEpiStore), seg(L.at[kGate], 0, L.rp[kUp], k::kEpiStore)},
                 k::kGemmStore, pf_pug_, ld_ug_);
        } else {
            gemm(pf_xn_, ldd, 1, {seg(L.at[kUp], 0, 0, k::kEpiStore)}, k::kGemmStore, pf_pug_, ld_ug_);
            gemm(pf_xn_, ldd, 1, {seg(L.at[kGate], 0, L.rp[kUp], k::kEpiStore)}, k::kGemmStore, pf_pug_, ld_ug_);
        }
        norm_ss_in = nullptr;
        gemm(pf_pug_, ld_ug_, 2, {seg(L.bt[kUp], 0, 0, k::kEpiStore), seg(L.bt[kGate], L.rp[kUp], 0, k::kEpiStore)},
             k::kGemmSilu, pf_h_, ldff);
        gemm(pf_h_, ldff, 1, {seg(L.at[kDown], 0, 0, k::kEpiStore)}, k::kGemmStore, pf_pd_, ld_d_);
        if (fold && l + 1 < c.n_layers) {
            norm_xg = pf_xn_;
            norm_gamma = m.layers[l + 1].attn_gamma;
        }
        gemm(pf_pd_, ld_d_, 1, {seg(L.bt[kDown], 0, 0, k::kEpiStore)}, k::kGemmAddF32, pf_x_, ldd);
        norm_xg = nullptr;
    }
}

// Batched engine head: logits[b] = RMSNorm(x[b]) . head (fp32, zeroed then
// accumulated by the head GEMM's residual-add epilogue), greedy argmax into
// tokens_ (and d_out[b][*step]), then pos += pos_inc, step += 1 -- the same
// contract as the megakernel's head + argmax phases.
void Session::head_rows(const float* x, int32_t* d_out, int out_ld, int pos_inc) {
    const DeviceModel& m = *m_;
    const ModelConfig& c = m.cfg;
    const int V = static_cast<int>(c.vocab);
    k::rmsnorm_rows(m.wt, x, m.ldd, m.final_gamma, static_cast<float>(c.norm_eps), B_, static_cast<int>(c.d_model),
                    pf_xn_, m.ldd, stream_);
    FSVD_CUDA(cudaMemsetAsync(logits_, 0, 4ull * B_ * V, stream_));
    k::GemmArgs g{};
    g.x = pf_xn_;
    g.x_ld = m.ldd;
    g.M = B_;
    g.seg[0] = seg(m.head_t, 0, 0, k::kEpiStore);
    g.nseg = 1;
    g.epi = k::kGemmAddF32;
    g.y = logits_;
    g.y_ld = V;
    g.ws = pf_ws_;
    g.ws_floats = pf_ws_floats_;
    k::gemm(m.wt, g, stream_);
    k::argmax_rows(logits_, V, B_, tokens_, d_out, out_ld, step_, stream_);
    k::advance_pos(pos_, pos_inc, step_, stream_);
    launches_this_step_ += 5;
}

// One batched decode step: embed tokens_ -> every layer at M = B rows, T = 1,
// positions read from the device length register -> head + argmax. Eager
// plan: direct launches; graph plans: the step is captured once (per output
// buffer) and replayed.
void Session::batched_decode(int32_t* d_out, int out_ld) {
    const DeviceModel& m = *m_;
    auto body = [&] {
        k::embed(m.wt, m.emb, m.ldd, tokens_, B_, static_cast<int>(m.cfg.d_model), pf_x_, m.ldd, stream_);
        layers_forward(B_, 1, 0, pos_);
        head_rows(pf_x_, d_out, out_ld, 1);
    };
    launches_this_step_ = 0;
    if (plan_ == FSVD_PLAN_EAGER || plan_ == FSVD_PLAN_SPLIT) {  // (split: eager launches + boundary copies)
        body();
        const uint64_t n = launches_this_step_ + 1 + 10ull * m.cfg.n_layers;
        stats_.dispatches += n;
        stats_.kernel_launches += n;
        return;
    }
    if (bstep_graph_ && (d_out != bstep_out_ || out_ld != bstep_out_ld_)) {
        FSVD_CUDA(cudaGraphExecDestroy(bstep_graph_));
        bstep_graph_ = nullptr;
    }
    if (!bstep_graph_) {
        cudaGraph_t g;
        FSVD_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
        body();
        FSVD_CUDA(cudaStreamEndCapture(stream_, &g));
        FSVD_CUDA(cudaGraphInstantiate(&bstep_graph_, g, 0));
        cudaGraphDestroy(g);
        bstep_out_ = d_out;
        bstep_out_ld_ = out_ld;
    }
    FSVD_CUDA(cudaGraphLaunch(bstep_graph_, stream_));
    stats_.graph_launches += 1;
    stats_.dispatches += 1;
}

void Session::prefill(const int32_t* d_tokens, size_t T, float* d_logits) {
    if (T == 0) throw ShapeError("prefill: empty prompt");
    if (position_ + T > cap_)
        throw CapacityError("prefill: prompt of " + std::to_string(T) + " tokens exceeds capacity " +
                            std::to_string(cap_));
    const ModelConfig& c = m_->cfg;
    // chunk so the workspace stays bounded (<= 16384 rows)
    const size_t max_rows = 16384;
    const size_t Tc_max = std::max<size_t>(1, std::min(T, max_rows / B_));
    ensure_prefill_workspace(B_ * Tc_max);
    for (size_t t0 = 0; t0 < T; t0 += Tc_max) {
        const size_t Tc = std::min(Tc_max, T - t0);
        prefill_chunk(d_tokens, T, t0, Tc);
        if (t0 + Tc == T)
            k::gather_last(pf_x_, m_->ldd, B_, static_cast<int>(Tc), static_cast<int>(c.d_model), x_, m_->ldd,
                           stream_);
        position_ += Tc;
    }
    k::set_int(pos_, static_cast<int>(position_), stream_);
    // head on the last position of every sequence; the argmax phase sets the
    // first generated token (pos_inc = 0: pos already advanced)
    k::set_int(step_, 0, stream_);
    launches_this_step_ = 0;
    if (batched_)
        head_rows(x_, nullptr, 0, 0);
    else
        mk_run(ph_pf_head_, ph_pf_argmax_ + 1);
    if (d_logits && d_logits != logits_)
        FSVD_CUDA(cudaMemcpyAsync(d_logits, logits_, 4ull * B_ * c.vocab, cudaMemcpyDeviceToDevice, stream_));
    FSVD_CUDA(cudaGetLastError());
}

void Session::generate(const int32_t* d_prompt, size_t T, size_t max_new, int32_t* d_out) {
    if (T == 0) throw ShapeError("generate: empty prompt");
    if (position_ + T + (max_new ? max_new - 1 : 0) > cap_)
        throw CapacityError("generate: prompt + max_new exceeds capacity");
    prefill(d_prompt, T, nullptr);
    if (max_new == 0) return;
    // first generated token = argmax of the prefill logits
    FSVD_CUDA(cudaMemcpy2DAsync(d_out, max_new * 4, tokens_, 4, 4, B_, cudaMemcpyDeviceToDevice, stream_));
    k::set_int(step_, 1, stream_);
    for (size_t i = 1; i < max_new; ++i) {
        const uint64_t before = stats_.dispatches;
        decode_any(d_out, static_cast<int>(max_new));
        stats_.last_dispatches = stats_.dispatches - before;
        stats_.steps += 1;
        position_ += 1;
    }
    FSVD_CUDA(cudaGetLastError());
}

void Session::reset() {
    FSVD_CUDA(cudaStreamSynchronize(stream_));
    position_ = 0;
    k::set_int(pos_, 0, stream_);
    k::set_int(step_, 0, stream_);
    stats_ = StepStats{};
    FSVD_CUDA(cudaStreamSynchronize(stream_));
}

void Session::read_kv(size_t layer, size_t b, int which, size_t pos0, size_t npos, float* out) {
    const ModelConfig& c = m_->cfg;
    if (layer >= c.n_layers || b >= static_cast<size_t>(B_) || pos0 + npos > cap_)
        throw ShapeError("read_kv: index out of range");
    FSVD_CUDA(cudaStreamSynchronize(stream_));
    const size_t H = c.n_heads, dh = c.d_head, es = m_->esize;
    const char* base = static_cast<const char*>(which ? vc_ : kc_) + (layer * cache_lstride_ + b * cache_bstride_) * es;
    std::vector<uint8_t> buf(dh * es);
    for (size_t p = 0; p < npos; ++p)
        for (size_t h = 0; h < H; ++h) {
            FSVD_CUDA(cudaMemcpy(buf.data(), base + (h * cache_hstride_ + (pos0 + p) * dh) * es, dh * es,
                                 cudaMemcpyDeviceToHost));
            for (size_t i = 0; i < dh; ++i) {
                float f;
                if (es == 4) {
                    std::memcpy(&f, buf.data() + i * 4, 4);
                } else {
                    uint16_t hb;
                    std::memcpy(&hb, buf.data() + i * 2, 2);
                    const uint32_t u = static_cast<uint32_t>(hb) << 16;
                    std::memcpy(&f, &u, 4);
                }
                out[p * c.d_model + h * dh + i] = f;
            }
        }
}

}  // namespace fsvd::rt
