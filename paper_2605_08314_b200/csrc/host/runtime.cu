// Device model + session runtime (SPEC.md runtime :283-382, plan :384-446).
//
// Decode step (CS3 in SURVEY.md §3), per layer:
//   qkvA   p_qkv = rmsnorm(x) . [A_q|A_k|A_v]         (packed QKV projection)
//   qkvB   q,k,v = p . B_{q,k,v}; RoPE(q,k) at pos; k,v -> cache row pos
//   attn   split-K flash-decode over cache rows [0, pos]
//   oA/oB  x += (attn . A_o) . B_o
//   ugA    p_ug = rmsnorm(x) . [A_up|A_gate]          (packed; no_merge = 2 launches)
//   ugB    h = silu(p_g . B_gate) * (p_u . B_up)
//   dA/dB  x += (h . A_down) . B_down
// then head GEMV (final RMSNorm prologue) and the greedy argmax that advances
// the device length register. Every kernel is launched with PDL; plans
// capture the same launches into CUDA graphs (per layer or per step).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <thread>

#include "runtime.h"

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

struct Plan {
    // byte sizes of every device tensor, computed before allocation
    size_t total = 0;
    void add(size_t b) { total += (b + 255) & ~size_t(255); }
};

void init_model_shapes(DeviceModel& dm, const ModelConfig& c, size_t cap, fsvd_dtype dt, int device) {
    dm.cfg = c;
    dm.capacity = cap;
    dm.wt = dt == FSVD_DTYPE_BF16 ? k::kBF16 : k::kF32;
    dm.esize = dt == FSVD_DTYPE_BF16 ? 2 : 4;
    dm.device = device;
    dm.ldd = pad8(c.d_model);
    FSVD_CUDA(cudaSetDevice(device));
    FSVD_CUDA(cudaDeviceGetAttribute(&dm.sm_count, cudaDevAttrMultiProcessorCount, device));
    dm.ldff = pad8(c.d_ff);
}

size_t ld_in(const DeviceModel& dm, size_t proj) { return proj == kDown ? dm.ldff : dm.ldd; }

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

// Allocate the arena for the given per-layer ranks; A^T buffers deduplicated
// by `key(layer, group_kind)` identity (shared bases).
struct AKeys {
    // per layer: identity keys of the qkv / o / ug / down input factors
    std::vector<std::array<const void*, 4>> keys;
};

void allocate(DeviceModel& dm, const std::vector<std::array<size_t, kNumProj>>& ranks, const AKeys& ak) {
    const ModelConfig& c = dm.cfg;
    const size_t es = dm.esize;
    Plan plan;
    plan.add(c.vocab * dm.ldd * es);  // emb
    plan.add(c.vocab * dm.ldd * es);  // head^T
    plan.add(c.d_model * 4);          // final gamma
    std::map<const void*, bool> seen[4];
    for (size_t l = 0; l < c.n_layers; ++l) {
        const auto& r = ranks[l];
        const size_t a_rows[4] = {r[kQ] + r[kK] + r[kV], r[kO], r[kUp] + r[kGate], r[kDown]};
        const size_t a_ld[4] = {size_t(dm.ldd), size_t(dm.ldd), size_t(dm.ldd), size_t(dm.ldff)};
        for (int g = 0; g < 4; ++g) {
            const void* key = ak.keys[l][g];
            if (key && seen[g].count(key)) continue;
            if (key) seen[g][key] = true;
            plan.add(a_rows[g] * a_ld[g] * es);
        }
        for (size_t p = 0; p < kNumProj; ++p) plan.add(proj_dims(c, p)[1] * pad8(r[p]) * es);
        plan.add(2 * c.d_model * 4);
    }
    dm.arena_bytes = plan.total + 4096;
    FSVD_CUDA(cudaSetDevice(dm.device));
    cudaError_t e = cudaMalloc(&dm.arena, dm.arena_bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw OomError("cannot allocate " + std::to_string(dm.arena_bytes) + " bytes of device weights");
    }
    FSVD_CUDA(cudaMemset(dm.arena, 0, dm.arena_bytes));
    dm.stored_weight_bytes = plan.total;

    dm.emb = dm.alloc(c.vocab * dm.ldd * es);
    dm.head_t = dm.alloc(c.vocab * dm.ldd * es);
    dm.final_gamma = static_cast<const float*>(dm.alloc(c.d_model * 4));
    std::map<const void*, const void*> shared[4];
    dm.layers.resize(c.n_layers);
    for (size_t l = 0; l < c.n_layers; ++l) {
        DeviceLayer& L = dm.layers[l];
        const auto& r = ranks[l];
        for (size_t p = 0; p < kNumProj; ++p) {
            L.r[p] = static_cast<int>(r[p]);
            L.rp[p] = pad8(r[p]);
        }
        const size_t a_rows[4] = {r[kQ] + r[kK] + r[kV], r[kO], r[kUp] + r[kGate], r[kDown]};
        const size_t a_ld[4] = {size_t(dm.ldd), size_t(dm.ldd), size_t(dm.ldd), size_t(dm.ldff)};
        const void* ptrs[4];
        for (int g = 0; g < 4; ++g) {
            const void* key = ak.keys[l][g];
            auto it = key ? shared[g].find(key) : shared[g].end();
            if (it != shared[g].end()) {
                ptrs[g] = it->second;
            } else {
                ptrs[g] = dm.alloc(a_rows[g] * a_ld[g] * es);
                if (key) shared[g][key] = ptrs[g];
            }
        }
        L.at_qkv = ptrs[0];
        L.at_o = ptrs[1];
        L.at_ug = ptrs[2];
        L.at_down = ptrs[3];
        for (size_t p = 0; p < kNumProj; ++p) L.bt[p] = dm.alloc(proj_dims(c, p)[1] * L.rp[p] * es);
        L.attn_gamma = static_cast<const float*>(dm.alloc(c.d_model * 4));
        L.mlp_gamma = static_cast<const float*>(dm.alloc(c.d_model * 4));
    }
    account(dm, ranks);
}

// Base pointer + row offset of projection p's A^T rows inside the packed buffer.
const void* a_rows_ptr(const DeviceModel& dm, const DeviceLayer& L, size_t p) {
    const char* base;
    size_t row0 = 0;
    switch (p) {
        case kQ: base = static_cast<const char*>(L.at_qkv); break;
        case kK: base = static_cast<const char*>(L.at_qkv); row0 = L.r[kQ]; break;
        case kV: base = static_cast<const char*>(L.at_qkv); row0 = L.r[kQ] + L.r[kK]; break;
        case kO: base = static_cast<const char*>(L.at_o); break;
        case kUp: base = static_cast<const char*>(L.at_ug); break;
        case kGate: base = static_cast<const char*>(L.at_ug); row0 = L.r[kUp]; break;
        default: base = static_cast<const char*>(L.at_down); break;
    }
    return base + row0 * ld_in(dm, p) * dm.esize;
}

void to_device_dtype(const float* src, size_t n, k::WType wt, std::vector<uint8_t>& out) {
    if (wt == k::kF32) {
        out.resize(n * 4);
        std::memcpy(out.data(), src, n * 4);
        return;
    }
    out.resize(n * 2);
    uint16_t* o = reinterpret_cast<uint16_t*>(out.data());
    for (size_t i = 0; i < n; ++i) {
        uint32_t u;
        std::memcpy(&u, &src[i], 4);
        if ((u & 0x7F800000u) != 0x7F800000u) u += 0x7FFFu + ((u >> 16) & 1u);
        o[i] = static_cast<uint16_t>(u >> 16);
    }
}

// Upload a host row-major [rows x cols] f32 matrix as transposed [cols][ld]
// (transpose=true) or as [rows][ld] (transpose=false) in the model dtype.
void upload_matrix(const DeviceModel& dm, const void* dst, const float* src, size_t rows, size_t cols, size_t ld,
                   bool transpose) {
    const size_t out_rows = transpose ? cols : rows, out_cols = transpose ? rows : cols;
    std::vector<float> tmp(out_rows * ld, 0.f);
    if (transpose) {
        for (size_t i = 0; i < rows; ++i)
            for (size_t j = 0; j < cols; ++j) tmp[j * ld + i] = src[i * cols + j];
    } else {
        for (size_t i = 0; i < rows; ++i) std::memcpy(&tmp[i * ld], &src[i * cols], cols * 4);
    }
    (void)out_cols;
    std::vector<uint8_t> bytes;
    to_device_dtype(tmp.data(), tmp.size(), dm.wt, bytes);
    FSVD_CUDA(cudaMemcpy(const_cast<void*>(dst), bytes.data(), bytes.size(), cudaMemcpyHostToDevice));
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
    AKeys ak;
    ak.keys.resize(c.n_layers);
    bool any_shared = false;
    for (size_t l = 0; l < c.n_layers; ++l) {
        const auto& L = m.layers[l];
        for (size_t p = 0; p < kNumProj; ++p) ranks[l][p] = L.proj(p).rank;
        for (size_t p = 0; p < kNumProj; ++p) any_shared |= L.proj(p).shared_group.has_value();
    }
    // Shared-basis identity: a packed group is reused only when every member
    // factor aliases the same storage (family C); otherwise per-layer.
    std::map<std::vector<const void*>, const void*> canon[4];
    for (size_t l = 0; l < c.n_layers; ++l) {
        const auto& L = m.layers[l];
        const std::vector<const void*> ids[4] = {{L.q.a.get(), L.k.a.get(), L.v.a.get()},
                                                 {L.o.a.get()},
                                                 {L.up.a.get(), L.gate.a.get()},
                                                 {L.down.a.get()}};
        for (int g = 0; g < 4; ++g) {
            if (!any_shared) {
                ak.keys[l][g] = nullptr;
                continue;
            }
            auto it = canon[g].find(ids[g]);
            if (it == canon[g].end()) it = canon[g].emplace(ids[g], ids[g][0]).first;
            ak.keys[l][g] = it->second;
        }
    }
    allocate(*dm, ranks, ak);

    upload_matrix(*dm, dm->emb, m.embedding.data.data(), c.vocab, c.d_model, dm->ldd, false);
    upload_matrix(*dm, dm->head_t, m.head.data.data(), c.d_model, c.vocab, dm->ldd, true);
    upload_f32(dm->final_gamma, m.final_gamma.data(), c.d_model);
    std::map<const void*, bool> done;
    for (size_t l = 0; l < c.n_layers; ++l) {
        const auto& L = m.layers[l];
        const DeviceLayer& D = dm->layers[l];
        for (size_t p = 0; p < kNumProj; ++p) {
            const auto& f = L.proj(p);
            const auto dims = proj_dims(c, p);
            const void* dst = a_rows_ptr(*dm, D, p);
            if (!done.count(dst)) {
                upload_matrix(*dm, dst, f.a->data.data(), dims[0], f.rank, ld_in(*dm, p), true);
                done[dst] = true;
            }
            upload_matrix(*dm, D.bt[p], f.b->data.data(), f.rank, dims[1], D.rp[p], true);
        }
        upload_f32(D.attn_gamma, L.attn_gamma.data(), c.d_model);
        upload_f32(D.mlp_gamma, L.mlp_gamma.data(), c.d_model);
    }
    FSVD_CUDA(cudaDeviceSynchronize());
    dm->family = 'A';
    return dm;
}

std::unique_ptr<DeviceModel> generate_synthetic(const SynthSpec& spec, fsvd_dtype dt, int device) {
    const SynthLayout lay = synth_layout(spec);
    auto dm = std::make_unique<DeviceModel>();
    init_model_shapes(*dm, spec.config, spec.capacity, dt, device);
    const ModelConfig& c = spec.config;
    AKeys ak;
    ak.keys.resize(c.n_layers);
    // family C: every input factor of a layer group aliases one storage
    // instance; use a synthetic identity per (group) -- all four packed
    // groups share the same layer grouping.
    static const char kTag[4] = {0, 1, 2, 3};
    for (size_t l = 0; l < c.n_layers; ++l)
        for (int g = 0; g < 4; ++g)
            ak.keys[l][g] = spec.family == 'C'
                                ? reinterpret_cast<const void*>(reinterpret_cast<uintptr_t>(&kTag[g]) +
                                                                 (l / spec.group_size) * 4096)
                                : nullptr;
    allocate(*dm, lay.ranks, ak);
    dm->family = spec.family;

    auto fill = [&](const SynthTensor& t, const void* dst, long long rows, long long cols, long long rs,
                    long long cs, int fold, uint64_t scale_off, k::WType dtype) {
        k::SynthFill f{};
        f.seed = spec.seed;
        f.offset = t.stream_offset;
        f.amp = t.amp;
        f.kind = t.kind;
        f.rows = rows;
        f.cols = cols;
        f.rs = rs;
        f.cs = cs;
        f.fold = fold;
        f.scale_offset = scale_off;
        f.dst = const_cast<void*>(dst);
        f.dt = dtype;
        k::synth_fill(f, nullptr);
    };
    auto need = [&](const std::string& n) -> const SynthTensor& {
        const SynthTensor* t = lay.find(n);
        if (!t) throw ConfigError("synthetic layout lacks '" + n + "'");
        return *t;
    };
    const long long V = c.vocab, d = c.d_model;
    fill(need("embedding"), dm->emb, V, d, dm->ldd, 1, 0, 0, dm->wt);
    fill(need("head"), dm->head_t, d, V, 1, dm->ldd, 0, 0, dm->wt);
    fill(need("final_gamma"), dm->final_gamma, 1, d, 0, 1, 0, 0, k::kF32);
    std::map<const void*, bool> done;
    for (size_t l = 0; l < c.n_layers; ++l) {
        const DeviceLayer& D = dm->layers[l];
        const std::string base = "layers." + std::to_string(l) + ".";
        for (size_t p = 0; p < kNumProj; ++p) {
            const auto dims = proj_dims(c, p);
            const long long din = dims[0], dout = dims[1], r = D.r[p];
            const std::string pb = base + kProjNames[p];
            const void* adst = a_rows_ptr(*dm, D, p);
            const long long lda = static_cast<long long>(ld_in(*dm, p));
            if (!done.count(adst)) {
                done[adst] = true;
                switch (spec.family) {
                    case 'A': fill(need(pb + ".A"), adst, din, r, 1, lda, 0, 0, dm->wt); break;
                    case 'B':
                        fill(need(pb + ".Uf"), adst, din, r, 1, lda, 1, need(pb + ".scale").stream_offset, dm->wt);
                        break;
                    case 'C':
                        fill(need(std::string("shared.") + kProjNames[p] + "." + std::to_string(l / spec.group_size) +
                                  ".A"),
                             adst, din, r, 1, lda, 0, 0, dm->wt);
                        break;
                    default: fill(need(pb + ".U"), adst, din, r, 1, lda, 2, need(pb + ".S").stream_offset, dm->wt);
                }
            }
            const SynthTensor& bt = need(pb + (spec.family == 'B' || spec.family == 'D' ? ".Vt" : ".B"));
            fill(bt, D.bt[p], r, dout, 1, D.rp[p], 0, 0, dm->wt);
        }
        fill(need(base + "attn_gamma"), D.attn_gamma, 1, d, 0, 1, 0, 0, k::kF32);
        fill(need(base + "mlp_gamma"), D.mlp_gamma, 1, d, 0, 1, 0, 0, k::kF32);
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
    // A: d_in x r from A^T [r][ld_in]; B: r x d_out from B^T [d_out][rp]
    const size_t rows_t = b ? dims[1] : r, ld = b ? L.rp[proj] : ld_in(dm, proj);
    const size_t want = b ? r * dims[1] : dims[0] * r;
    if (count != want) throw ShapeError("copy_factor: count mismatch");
    const void* src = b ? L.bt[proj] : a_rows_ptr(dm, L, proj);
    std::vector<uint8_t> raw(rows_t * ld * dm.esize);
    FSVD_CUDA(cudaMemcpy(raw.data(), src, raw.size(), cudaMemcpyDeviceToHost));
    auto get = [&](size_t i) -> float {
        if (dm.esize == 4) {
            float f;
            std::memcpy(&f, raw.data() + i * 4, 4);
            return f;
        }
        uint16_t h;
        std::memcpy(&h, raw.data() + i * 2, 2);
        uint32_t u = static_cast<uint32_t>(h) << 16;
        float f;
        std::memcpy(&f, &u, 4);
        return f;
    };
    const size_t cols_out = b ? dims[1] : r;   // logical cols
    const size_t rows_out = b ? r : dims[0];
    for (size_t i = 0; i < rows_out; ++i)
        for (size_t j = 0; j < cols_out; ++j) out[i * cols_out + j] = get(j * ld + i);
}

// ----------------------------------------------------------------- session --

fsvd_ffn_backend route_ffn_auto(fsvd_plan_mode plan, fsvd_ffn_backend requested) {
    // explicit override wins; auto: eager -> no_merge,
    // per_layer -> packed, split -> no_merge. The full-step graph is a
    // layer-tail graph superset, so it routes like per_layer.
    if (requested != FSVD_FFN_AUTO) return requested;
    return plan == FSVD_PLAN_EAGER ? FSVD_FFN_NO_MERGE : FSVD_FFN_PACKED;
}

void* Session::dalloc(size_t bytes) {
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes < 256 ? 256 : bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        throw OomError("session allocation of " + std::to_string(bytes) + " bytes failed");
    }
    FSVD_CUDA(cudaMemsetAsync(p, 0, bytes < 256 ? 256 : bytes, stream_));
    allocations_.push_back(p);
    return p;
}

Session::Session(DeviceModel* m, const fsvd_session_opts& o) : m_(m) {
    const ModelConfig& c = m->cfg;
    B_ = static_cast<int>(o.batch);
    if (B_ < 1) throw ConfigError("session batch must be >= 1");
    if (B_ > 4) throw ConfigError("decode batch > 4 is not supported by the CUDA-core GEMV path yet");
    cap_ = o.capacity ? o.capacity : (m->capacity ? m->capacity : 8192);
    if (o.plan < FSVD_PLAN_EAGER || o.plan > FSVD_PLAN_FULL_STEP) throw ConfigError("unknown plan mode");
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
    tickets_ = static_cast<unsigned*>(dalloc(64));
    counters_ = static_cast<unsigned*>(dalloc(4 * B_ * H));

    int max_rp_qkv = 0, max_ug = 0, max_o = 0, max_d = 0;
    for (const auto& Ly : m->layers) {
        max_rp_qkv = std::max(max_rp_qkv, Ly.rp[kQ] + Ly.rp[kK] + Ly.rp[kV]);
        max_ug = std::max(max_ug, Ly.rp[kUp] + Ly.rp[kGate]);
        max_o = std::max(max_o, Ly.rp[kO]);
        max_d = std::max(max_d, Ly.rp[kDown]);
    }
    ld_qkv_ = max_rp_qkv;
    ld_ug_ = max_ug;
    x_ = static_cast<float*>(dalloc(4ull * B_ * m->ldd));
    p_qkv_ = static_cast<float*>(dalloc(4ull * B_ * ld_qkv_));
    q_ = static_cast<float*>(dalloc(4ull * B_ * m->ldd));
    attn_ = static_cast<float*>(dalloc(4ull * B_ * m->ldd));
    p_o_ = static_cast<float*>(dalloc(4ull * B_ * max_o));
    p_ug_ = static_cast<float*>(dalloc(4ull * B_ * ld_ug_));
    h_ = static_cast<float*>(dalloc(4ull * B_ * m->ldff));
    p_d_ = static_cast<float*>(dalloc(4ull * B_ * max_d));
    logits_ = static_cast<float*>(dalloc(4ull * B_ * c.vocab));

    // split-K: ~2 CTAs per SM, each split <= kAttnMaxChunk rows
    const int bh = B_ * static_cast<int>(H);
    splits_ = std::max((296 + bh - 1) / bh, static_cast<int>((cap_ + k::kAttnMaxChunk - 1) / k::kAttnMaxChunk));
    splits_ = std::min(splits_, 64);
    if (static_cast<size_t>(splits_) * k::kAttnMaxChunk < cap_) throw ConfigError("capacity too large for split-K");
    partial_ = static_cast<float*>(dalloc(4ull * bh * splits_ * (dh + 2)));
    FSVD_CUDA(cudaStreamSynchronize(stream_));
    stats_.allocs = 0;
}

Session::~Session() {
    cudaSetDevice(m_->device);
    if (stream_) cudaStreamSynchronize(stream_);
    for (auto g : layer_graphs_) cudaGraphExecDestroy(g);
    if (step_graph_) cudaGraphExecDestroy(step_graph_);
    for (void* p : allocations_) cudaFree(p);
    if (stream_) cudaStreamDestroy(stream_);
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

void Session::launch_gemv(const k::GemvArgs& a) {
    k::gemv(m_->wt, B_, a, m_->sm_count, stream_, pdl_);
    ++launches_this_step_;
}

void Session::layer_body(size_t l) {
    const DeviceModel& m = *m_;
    const ModelConfig& c = m.cfg;
    const DeviceLayer& L = m.layers[l];
    const int d = static_cast<int>(c.d_model), ldd = m.ldd, ldff = m.ldff;
    const float eps = static_cast<float>(c.norm_eps);
    char* kc = static_cast<char*>(kc_) + l * cache_lstride_ * m.esize;
    char* vc = static_cast<char*>(vc_) + l * cache_lstride_ * m.esize;
    const int rq = L.rp[kQ], rk = L.rp[kK], rv = L.rp[kV];

    // qkvA: p_qkv = rmsnorm(x) . [A_q | A_k | A_v]
    {
        k::GemvArgs a{};
        const char* base = static_cast<const char*>(L.at_qkv);
        a.seg[0] = {base, L.r[kQ], ldd, ldd, 0, 0, k::kEpiStore};
        a.seg[1] = {base + size_t(L.r[kQ]) * ldd * m.esize, L.r[kK], ldd, ldd, 0, rq, k::kEpiStore};
        a.seg[2] = {base + size_t(L.r[kQ] + L.r[kK]) * ldd * m.esize, L.r[kV], ldd, ldd, 0, rq + rk, k::kEpiStore};
        a.nseg = 3;
        a.x = x_;
        a.x_ld = ldd;
        a.x_len = ldd;
        a.gamma = L.attn_gamma;
        a.eps = eps;
        a.norm_len = d;
        a.y = p_qkv_;
        a.y_ld = ld_qkv_;
        launch_gemv(a);
    }
    // qkvB: q, k, v = p . B; RoPE; append k, v at pos
    {
        k::GemvArgs a{};
        a.seg[0] = {L.bt[kQ], d, rq, rq, 0, 0, k::kEpiRopeQ};
        a.seg[1] = {L.bt[kK], d, rk, rk, rq, 0, k::kEpiRopeK};
        a.seg[2] = {L.bt[kV], d, rv, rv, rq + rk, 0, k::kEpiV};
        a.nseg = 3;
        a.x = p_qkv_;
        a.x_ld = ld_qkv_;
        a.x_len = rq + rk + rv;
        a.y = q_;
        a.y_ld = ldd;
        a.rope = rope_;
        a.pos = pos_;
        a.d_head = static_cast<int>(c.d_head);
        a.kcache = kc;
        a.vcache = vc;
        a.cache_bstride = cache_bstride_;
        a.cache_hstride = cache_hstride_;
        launch_gemv(a);
    }
    // attention over the dense cache
    {
        k::AttnDecodeArgs a{};
        a.q = q_;
        a.kcache = kc;
        a.vcache = vc;
        a.cache_bstride = cache_bstride_;
        a.cache_hstride = cache_hstride_;
        a.pos = pos_;
        a.out = attn_;
        a.partial = partial_;
        a.counters = counters_;
        a.batch = B_;
        a.n_heads = static_cast<int>(c.n_heads);
        a.d_head = static_cast<int>(c.d_head);
        a.splits = splits_;
        a.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(c.d_head)));
        k::attn_decode(m.wt, a, stream_, pdl_);
        ++launches_this_step_;
    }
    // oA / oB
    {
        k::GemvArgs a{};
        a.seg[0] = {L.at_o, L.r[kO], ldd, ldd, 0, 0, k::kEpiStore};
        a.nseg = 1;
        a.x = attn_;
        a.x_ld = ldd;
        a.x_len = ldd;
        a.y = p_o_;
        a.y_ld = L.rp[kO];
        launch_gemv(a);
    }
    {
        k::GemvArgs a{};
        a.seg[0] = {L.bt[kO], d, L.rp[kO], L.rp[kO], 0, 0, k::kEpiAdd};
        a.nseg = 1;
        a.x = p_o_;
        a.x_ld = L.rp[kO];
        a.x_len = L.rp[kO];
        a.y = x_;
        a.y_ld = ldd;
        launch_gemv(a);
    }
    // ugA: packed (one launch over [A_up | A_gate]) or no_merge (two)
    {
        const char* base = static_cast<const char*>(L.at_ug);
        const k::GemvSeg up = {base, L.r[kUp], ldd, ldd, 0, 0, k::kEpiStore};
        const k::GemvSeg gate = {base + size_t(L.r[kUp]) * ldd * m.esize, L.r[kGate], ldd, ldd, 0, L.rp[kUp],
                                 k::kEpiStore};
        k::GemvArgs a{};
        a.x = x_;
        a.x_ld = ldd;
        a.x_len = ldd;
        a.gamma = L.mlp_gamma;
        a.eps = eps;
        a.norm_len = d;
        a.y = p_ug_;
        a.y_ld = ld_ug_;
        if (ffn_ == FSVD_FFN_PACKED) {
            a.seg[0] = up;
            a.seg[1] = gate;
            a.nseg = 2;
            launch_gemv(a);
        } else {
            a.seg[0] = up;
            a.nseg = 1;
            launch_gemv(a);
            a.seg[0] = gate;
            launch_gemv(a);
        }
    }
    // ugB: h = silu(p_g . B_gate) * (p_u . B_up)
    {
        k::GemvArgs a{};
        a.seg[0] = {L.bt[kUp], static_cast<int>(c.d_ff), L.rp[kUp], L.rp[kUp], 0, 0, k::kEpiStore};
        a.seg[1] = {L.bt[kGate], static_cast<int>(c.d_ff), L.rp[kGate], L.rp[kGate], L.rp[kUp], 0, k::kEpiStore};
        a.nseg = 2;
        a.dual = 1;
        a.x = p_ug_;
        a.x_ld = ld_ug_;
        a.x_len = L.rp[kUp] + L.rp[kGate];
        a.y = h_;
        a.y_ld = ldff;
        launch_gemv(a);
    }
    // down
    {
        k::GemvArgs a{};
        a.seg[0] = {L.at_down, L.r[kDown], ldff, ldff, 0, 0, k::kEpiStore};
        a.nseg = 1;
        a.x = h_;
        a.x_ld = ldff;
        a.x_len = ldff;
        a.y = p_d_;
        a.y_ld = L.rp[kDown];
        launch_gemv(a);
    }
    {
        k::GemvArgs a{};
        a.seg[0] = {L.bt[kDown], d, L.rp[kDown], L.rp[kDown], 0, 0, k::kEpiAdd};
        a.nseg = 1;
        a.x = p_d_;
        a.x_ld = L.rp[kDown];
        a.x_len = L.rp[kDown];
        a.y = x_;
        a.y_ld = ldd;
        launch_gemv(a);
    }
}

void Session::step_head(float* d_logits, int32_t* d_out, int out_ld) {
    const DeviceModel& m = *m_;
    const ModelConfig& c = m.cfg;
    k::GemvArgs a{};
    a.seg[0] = {m.head_t, static_cast<int>(c.vocab), m.ldd, m.ldd, 0, 0, k::kEpiStore};
    a.nseg = 1;
    a.x = x_;
    a.x_ld = m.ldd;
    a.x_len = m.ldd;
    a.gamma = m.final_gamma;
    a.eps = static_cast<float>(c.norm_eps);
    a.norm_len = static_cast<int>(c.d_model);
    a.y = d_logits;
    a.y_ld = static_cast<int>(c.vocab);
    launch_gemv(a);
    k::argmax_step(d_logits, B_, static_cast<int>(c.vocab), tokens_, pos_, 1, d_out, out_ld, step_, tickets_,
                   stream_, pdl_);
    ++launches_this_step_;
}

void Session::capture_graphs() {
    if (plan_ == FSVD_PLAN_PER_LAYER && layer_graphs_.empty()) {
        for (size_t l = 0; l < m_->cfg.n_layers; ++l) {
            cudaGraph_t g;
            FSVD_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
            layer_body(l);
            FSVD_CUDA(cudaStreamEndCapture(stream_, &g));
            cudaGraphExec_t ge;
            FSVD_CUDA(cudaGraphInstantiate(&ge, g, 0));
            cudaGraphDestroy(g);
            layer_graphs_.push_back(ge);
        }
    }
}

void Session::run_decode(int32_t* d_out, int out_ld, float* d_logits) {
    const uint64_t before = stats_.dispatches;
    launches_this_step_ = 0;
    const ModelConfig& c = m_->cfg;
    if (plan_ == FSVD_PLAN_FULL_STEP) {
        if (!step_graph_ || graph_out_ != d_out || graph_logits_ != d_logits || graph_out_ld_ != out_ld) {
            if (step_graph_) cudaGraphExecDestroy(step_graph_);
            cudaGraph_t g;
            FSVD_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
            k::embed(m_->wt, m_->emb, m_->ldd, tokens_, B_, static_cast<int>(c.d_model), x_, m_->ldd, stream_, pdl_);
            for (size_t l = 0; l < c.n_layers; ++l) layer_body(l);
            step_head(d_logits, d_out, out_ld);
            FSVD_CUDA(cudaStreamEndCapture(stream_, &g));
            FSVD_CUDA(cudaGraphInstantiate(&step_graph_, g, 0));
            cudaGraphDestroy(g);
            graph_out_ = d_out;
            graph_out_ld_ = out_ld;
            graph_logits_ = d_logits;
        }
        FSVD_CUDA(cudaGraphLaunch(step_graph_, stream_));
        stats_.graph_launches += 1;
        stats_.dispatches += 1;
    } else {
        k::embed(m_->wt, m_->emb, m_->ldd, tokens_, B_, static_cast<int>(c.d_model), x_, m_->ldd, stream_, pdl_);
        stats_.dispatches += 1;
        stats_.kernel_launches += 1;
        if (plan_ == FSVD_PLAN_PER_LAYER) {
            capture_graphs();
            for (auto g : layer_graphs_) FSVD_CUDA(cudaGraphLaunch(g, stream_));
            stats_.graph_launches += layer_graphs_.size();
            stats_.dispatches += layer_graphs_.size();
        } else {
            launches_this_step_ = 0;
            for (size_t l = 0; l < c.n_layers; ++l) layer_body(l);
            stats_.dispatches += launches_this_step_;
            stats_.kernel_launches += launches_this_step_;
        }
        launches_this_step_ = 0;
        step_head(d_logits, d_out, out_ld);
        stats_.dispatches += launches_this_step_;
        stats_.kernel_launches += launches_this_step_;
    }
    FSVD_CUDA(cudaGetLastError());
    stats_.last_dispatches = stats_.dispatches - before;
    stats_.steps += 1;
    position_ += 1;
}

void Session::decode_step(const int32_t* d_tokens, float* d_logits) {
    if (position_ == 0) throw ShapeError("decode_step: prefill first (position = 0)");
    if (position_ >= cap_) throw CapacityError("decode_step: KV cache full (capacity " + std::to_string(cap_) + ")");
    if (d_tokens)
        FSVD_CUDA(cudaMemcpyAsync(tokens_, d_tokens, 4ull * B_, cudaMemcpyDeviceToDevice, stream_));
    run_decode(nullptr, 0, d_logits ? d_logits : logits_);
}

void Session::ensure_prefill_workspace(size_t rows) {
    if (rows <= pf_rows_) return;
    const DeviceModel& m = *m_;
    const size_t es = m.esize;
    int max_o = 0, max_d = 0;
    for (const auto& Ly : m.layers) {
        max_o = std::max(max_o, Ly.rp[kO]);
        max_d = std::max(max_d, Ly.rp[kDown]);
    }
    pf_x_ = static_cast<float*>(dalloc(rows * m.ldd * 4));
    pf_xn_ = dalloc(rows * m.ldd * es);
    pf_pqkv_ = dalloc(rows * ld_qkv_ * es);
    pf_q_ = dalloc(rows * m.ldd * es);
    pf_att_ = dalloc(rows * m.ldd * es);
    pf_po_ = dalloc(rows * max_o * es);
    pf_pug_ = dalloc(rows * ld_ug_ * es);
    pf_h_ = dalloc(rows * m.ldff * es);
    pf_pd_ = dalloc(rows * max_d * es);
    pf_tok_ = static_cast<int32_t*>(dalloc(rows * 4));
    pf_rows_ = rows;
    stats_.allocs += 10;
}

// One prefill chunk: tokens [b][t0 .. t0+Tc) of a [B][T_total] prompt.
void Session::prefill_chunk(const int32_t* d_tokens, size_t T_total, size_t t0, size_t Tc) {
    const DeviceModel& m = *m_;
    const ModelConfig& c = m.cfg;
    const int M = static_cast<int>(B_ * Tc);
    const int d = static_cast<int>(c.d_model), ldd = m.ldd, ldff = m.ldff;
    const float eps = static_cast<float>(c.norm_eps);
    const size_t es = m.esize;
    // gather this chunk's tokens into [B*Tc]
    FSVD_CUDA(cudaMemcpy2DAsync(pf_tok_, Tc * 4, d_tokens + t0, T_total * 4, Tc * 4, B_, cudaMemcpyDeviceToDevice,
                                stream_));
    k::embed(m.wt, m.emb, ldd, pf_tok_, M, d, pf_x_, ldd, stream_, false);
    const int p0 = static_cast<int>(position_);
    for (size_t l = 0; l < c.n_layers; ++l) {
        const DeviceLayer& L = m.layers[l];
        char* kc = static_cast<char*>(kc_) + l * cache_lstride_ * es;
        char* vc = static_cast<char*>(vc_) + l * cache_lstride_ * es;
        const int rq = L.rp[kQ], rk = L.rp[kK], rv = L.rp[kV];
        k::rmsnorm_rows(m.wt, pf_x_, ldd, L.attn_gamma, eps, M, d, pf_xn_, ldd, stream_);
        {
            k::GemmArgs g{};
            const char* base = static_cast<const char*>(L.at_qkv);
            g.x = pf_xn_;
            g.x_ld = ldd;
            g.M = M;
            g.seg[0] = {base, L.r[kQ], ldd, ldd, 0, 0, k::kEpiStore};
            g.seg[1] = {base + size_t(L.r[kQ]) * ldd * es, L.r[kK], ldd, ldd, 0, rq, k::kEpiStore};
            g.seg[2] = {base + size_t(L.r[kQ] + L.r[kK]) * ldd * es, L.r[kV], ldd, ldd, 0, rq + rk, k::kEpiStore};
            g.nseg = 3;
            g.epi = k::kGemmStore;
            g.y = pf_pqkv_;
            g.y_ld = ld_qkv_;
            k::gemm(m.wt, g, stream_);
        }
        {
            k::GemmArgs g{};
            g.x = pf_pqkv_;
            g.x_ld = ld_qkv_;
            g.M = M;
            g.seg[0] = {L.bt[kQ], d, rq, rq, 0, 0, k::kEpiRopeQ};
            g.seg[1] = {L.bt[kK], d, rk, rk, rq, 0, k::kEpiRopeK};
            g.seg[2] = {L.bt[kV], d, rv, rv, rq + rk, 0, k::kEpiV};
            g.nseg = 3;
            g.epi = k::kGemmQKV;
            g.y = pf_q_;
            g.y_ld = ldd;
            g.rope = rope_;
            g.p0 = p0;
            g.T = static_cast<int>(Tc);
            g.d_head = static_cast<int>(c.d_head);
            g.n_heads = static_cast<int>(c.n_heads);
            g.kcache = kc;
            g.vcache = vc;
            g.cache_bstride = cache_bstride_;
            g.cache_hstride = cache_hstride_;
            k::gemm(m.wt, g, stream_);
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
            a.T = static_cast<int>(Tc);
            a.p0 = p0;
            a.n_heads = static_cast<int>(c.n_heads);
            a.d_head = static_cast<int>(c.d_head);
            a.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(c.d_head)));
            k::attn_prefill(m.wt, a, stream_);
        }
        {
            k::GemmArgs g{};
            g.x = pf_att_;
            g.x_ld = ldd;
            g.M = M;
            g.seg[0] = {L.at_o, L.r[kO], ldd, ldd, 0, 0, k::kEpiStore};
            g.nseg = 1;
            g.epi = k::kGemmStore;
            g.y = pf_po_;
            g.y_ld = L.rp[kO];
            k::gemm(m.wt, g, stream_);
        }
        {
            k::GemmArgs g{};
            g.x = pf_po_;
            g.x_ld = L.rp[kO];
            g.M = M;
            g.seg[0] = {L.bt[kO], d, L.rp[kO], L.rp[kO], 0, 0, k::kEpiStore};
            g.nseg = 1;
            g.epi = k::kGemmAddF32;
            g.y = pf_x_;
            g.y_ld = ldd;
            k::gemm(m.wt, g, stream_);
        }
        k::rmsnorm_rows(m.wt, pf_x_, ldd, L.mlp_gamma, eps, M, d, pf_xn_, ldd, stream_);
        {
            const char* base = static_cast<const char*>(L.at_ug);
            const k::GemvSeg up = {base, L.r[kUp], ldd, ldd, 0, 0, k::kEpiStore};
            const k::GemvSeg gate = {base + size_t(L.r[kUp]) * ldd * es, L.r[kGate], ldd, ldd, 0, L.rp[kUp],
                                     k::kEpiStore};
            k::GemmArgs g{};
            g.x = pf_xn_;
            g.x_ld = ldd;
            g.M = M;
            g.epi = k::kGemmStore;
            g.y = pf_pug_;
            g.y_ld = ld_ug_;
            if (ffn_ == FSVD_FFN_PACKED) {
                g.seg[0] = up;
                g.seg[1] = gate;
                g.nseg = 2;
                k::gemm(m.wt, g, stream_);
            } else {
                g.seg[0] = up;
                g.nseg = 1;
                k::gemm(m.wt, g, stream_);
                g.seg[0] = gate;
                k::gemm(m.wt, g, stream_);
            }
        }
        {
            k::GemmArgs g{};
            g.x = pf_pug_;
            g.x_ld = ld_ug_;
            g.M = M;
            g.seg[0] = {L.bt[kUp], static_cast<int>(c.d_ff), L.rp[kUp], L.rp[kUp], 0, 0, k::kEpiStore};
            g.seg[1] = {L.bt[kGate], static_cast<int>(c.d_ff), L.rp[kGate], L.rp[kGate], L.rp[kUp], 0, k::kEpiStore};
            g.nseg = 2;
            g.epi = k::kGemmSilu;
            g.y = pf_h_;
            g.y_ld = ldff;
            k::gemm(m.wt, g, stream_);
        }
        {
            k::GemmArgs g{};
            g.x = pf_h_;
            g.x_ld = ldff;
            g.M = M;
            g.seg[0] = {L.at_down, L.r[kDown], ldff, ldff, 0, 0, k::kEpiStore};
            g.nseg = 1;
            g.epi = k::kGemmStore;
            g.y = pf_pd_;
            g.y_ld = L.rp[kDown];
            k::gemm(m.wt, g, stream_);
        }
        {
            k::GemmArgs g{};
            g.x = pf_pd_;
            g.x_ld = L.rp[kDown];
            g.M = M;
            g.seg[0] = {L.bt[kDown], d, L.rp[kDown], L.rp[kDown], 0, 0, k::kEpiStore};
            g.nseg = 1;
            g.epi = k::kGemmAddF32;
            g.y = pf_x_;
            g.y_ld = ldd;
            k::gemm(m.wt, g, stream_);
        }
    }
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
        k::set_int(pos_, static_cast<int>(position_ + Tc), stream_);
        if (t0 + Tc == T) {
            k::gather_last(pf_x_, m_->ldd, B_, static_cast<int>(Tc), static_cast<int>(c.d_model), x_, m_->ldd,
                           stream_);
        }
        position_ += Tc;
    }
    // head on the last position of every sequence; argmax sets the first
    // generated token (pos already advanced: pos_inc = 0)
    launches_this_step_ = 0;
    const DeviceModel& m = *m_;
    k::GemvArgs a{};
    a.seg[0] = {m.head_t, static_cast<int>(c.vocab), m.ldd, m.ldd, 0, 0, k::kEpiStore};
    a.nseg = 1;
    a.x = x_;
    a.x_ld = m.ldd;
    a.x_len = m.ldd;
    a.gamma = m.final_gamma;
    a.eps = static_cast<float>(c.norm_eps);
    a.norm_len = static_cast<int>(c.d_model);
    a.y = d_logits ? d_logits : logits_;
    a.y_ld = static_cast<int>(c.vocab);
    k::gemv(m.wt, B_, a, m.sm_count, stream_, false);
    k::set_int(step_, 0, stream_);
    k::argmax_step(a.y, B_, static_cast<int>(c.vocab), tokens_, pos_, 0, nullptr, 0, step_, tickets_, stream_, false);
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
    for (size_t i = 1; i < max_new; ++i) run_decode(d_out, static_cast<int>(max_new), logits_);
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
